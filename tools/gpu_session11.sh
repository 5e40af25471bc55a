set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s11_pytest.log 2>&1; echo pytest=$?
timeout 600 python tools/kernel_times.py c2 c4 c5 > gpurun_out/s11_ktimes.log 2>&1
timeout 300 python bench.py > gpurun_out/s11_bench_c2.json 2> gpurun_out/s11_bench_c2.err
tail -3 gpurun_out/s11_pytest.log; cat gpurun_out/s11_ktimes.log gpurun_out/s11_bench_c2.json
