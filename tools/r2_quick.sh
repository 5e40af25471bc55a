# quick timing iteration (no tests): trained probe C2 + C2 bench
mkdir -p gpurun_out
timeout 300 python tools/probe_trained.py 0 c2 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; echo bench=$?
python -c "import json; j=json.load(open('gpurun_out/it_bench.json')); print(j['value']/1e6, j['ms_per_step'], {k: round(v['ms'], 4) for k, v in j['frame']['kernels'].items()})"
