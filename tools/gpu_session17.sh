set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s17_pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/kernel_times.py c2 c4 > gpurun_out/s17_kt.log 2>&1
timeout 300 python bench.py > gpurun_out/s17_bench_c2.json 2> gpurun_out/s17_bench_c2.err
timeout 300 python bench.py --workload c4 --steps 10 --no-cpu-baseline > gpurun_out/s17_bench_c4.json 2> gpurun_out/s17_bench_c4.err
tail -5 gpurun_out/s17_pytest.log; cat gpurun_out/s17_kt.log gpurun_out/s17_bench_c2.json gpurun_out/s17_bench_c4.json
