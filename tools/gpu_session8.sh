set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -q -p no:cacheprovider -x > gpurun_out/pytest_tc.log 2>&1
timeout 600 python tools/kernel_times.py c2 c4 > gpurun_out/kernel_times.jsonl 2> gpurun_out/kernel_times.err
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"project_reg|knn_tc" -c 2 -o gpurun_out/prof8 python tools/kernel_times.py c4 > gpurun_out/ncu_8.log 2>&1
ls -la gpurun_out
