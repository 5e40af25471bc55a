# quick iteration: GPU suite (minus the drop-in subprocess suite), trained probe, C2 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_dropin.py > gpurun_out/it_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/it_pytest.log; grep -E "^(FAILED|ERROR)|Error" gpurun_out/it_pytest.log | head -5
timeout 300 python tools/probe_trained.py 40 c2 2>&1 | tail -2
timeout 300 python tools/probe_trained.py 40 c4 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; echo bench=$?
python -c "import json; j=json.load(open('gpurun_out/it_bench.json')); print(j['value']/1e6, j['ms_per_step'], j['e2e']['value']/1e6, j['e2e_numpy']['value']/1e6, {k: round(v['ms'], 4) for k, v in j['frame']['kernels'].items()})"
