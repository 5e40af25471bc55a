mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2a_pytest.log
timeout 600 python bench.py > gpurun_out/r2a_bench_c2.json 2> gpurun_out/r2a_bench_c2.err; echo bench=$?
head -c 1500 gpurun_out/r2a_bench_c2.json
