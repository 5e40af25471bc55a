set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_projection.py -q -p no:cacheprovider -x > gpurun_out/pytest_tc.log 2>&1
timeout 600 python tools/kernel_times.py c2 > gpurun_out/kernel_times.jsonl 2> gpurun_out/kernel_times.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"project_reg" -c 1 -o gpurun_out/prof6p python tools/kernel_times.py c2 > gpurun_out/ncu_6p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"knn_tc" -c 1 -o gpurun_out/prof6t python tools/kernel_times.py c2 > gpurun_out/ncu_6t.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
ls -la gpurun_out
