set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/kernel_times.py c2 c4 > gpurun_out/kernel_times.jsonl 2> gpurun_out/kernel_times.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"knn_scan|project_fast" -s 2 -c 2 -o gpurun_out/prof3 python tools/kernel_times.py c2 > gpurun_out/ncu_full3.log 2>&1
ls -la gpurun_out
