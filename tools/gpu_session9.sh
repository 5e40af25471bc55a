set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_knn.py -q -p no:cacheprovider -x > gpurun_out/pytest_tc.log 2>&1
timeout 600 python tools/kernel_times.py c2 c4 > gpurun_out/kernel_times.jsonl 2> gpurun_out/kernel_times.err
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"knn_tc|project_reg" -c 2 -o gpurun_out/prof9 python tools/kernel_times.py c2 > gpurun_out/ncu_9.log 2>&1
ls -la gpurun_out
