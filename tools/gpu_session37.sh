set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s37_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/s37_pytest.log
timeout 600 python bench.py --workload c5 --steps 5 --no-cpu-baseline > gpurun_out/s37_bench_c5.json 2>/dev/null
python -c "
import json
j=json.load(open('gpurun_out/s37_bench_c5.json')); print(round(j['value']/1e6,2), j['ms_per_step'], j['e2e']['value']/1e6, j['gpu_launches'], {k:round(v['ms'],3) for k,v in j['compute_roofline']['kernels'].items()})"
