mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_dropin.py > gpurun_out/r2d_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2d_pytest.log
grep -E "^(FAILED|ERROR)" gpurun_out/r2d_pytest.log | head
timeout 300 python tools/probe_trained.py 40 c2 > gpurun_out/r2d_trained.jsonl 2>&1; cat gpurun_out/r2d_trained.jsonl | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:project_reg2 -s 4 -c 1 -o gpurun_out/r2d_proj_trained python tools/probe_trained.py 40 c2 > /dev/null 2>&1; echo ncu=$?
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r2d_bench_c3.json 2> gpurun_out/r2d_bench_c3.err; echo c3=$?; head -c 400 gpurun_out/r2d_bench_c3.json
