set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s36_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/s36_pytest.log
timeout 300 python tools/kernel_times.py c2 c4 > gpurun_out/s36_kt3.log 2>&1
ESOM_PROJ_V2=1 timeout 300 python tools/kernel_times.py c2 c4 > gpurun_out/s36_kt2.log 2>&1
cat gpurun_out/s36_kt3.log gpurun_out/s36_kt2.log
timeout 300 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/s36_bench_c2.json 2>/dev/null; cat gpurun_out/s36_bench_c2.json
