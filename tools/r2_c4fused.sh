mkdir -p gpurun_out
timeout 300 python tools/probe_trained.py 40 c4 2>&1 | tail -2
timeout 900 python bench.py --workload c4 --no-cpu-baseline > gpurun_out/it_bench4.json 2> gpurun_out/it_bench4.err; echo bench=$?
python -c "import json; j=json.load(open('gpurun_out/it_bench4.json')); print(j['value']/1e6, j['ms_per_step'], {k: round(v['ms'], 4) for k, v in j['frame']['kernels'].items()})"
timeout 1200 python -m pytest tests/test_gpu_projection.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py tests/test_gpu_train.py -q -x 2>&1 | tail -2
