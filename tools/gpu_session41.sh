set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s42_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/s42_pytest.log
PROBE_VARIANTS=w2,w3,w4 timeout 300 python tools/tc_probe.py c4 > gpurun_out/s42_probe.log 2>&1
ESOM_TC2_FUSED=1 PROBE_VARIANTS=w4 timeout 300 python tools/tc_probe.py c4 >> gpurun_out/s42_probe.log 2>&1
cat gpurun_out/s42_probe.log
timeout 300 python bench.py --workload c4 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); print('c4', round(j['value']/1e6,1), round(j['ms_per_step'],3), j['gpu_launches'], {k:round(v['ms'],3) for k,v in j['compute_roofline']['kernels'].items()})"
