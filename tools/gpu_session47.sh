timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for w in c2 c3 c4; do
timeout 300 python bench.py --workload $w --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); print('$w', round(j['value']/1e6,1), round(j['ms_per_step'],3), 'e2e', round(j['e2e']['value']/1e6,1), j['gpu_launches'], {k:round(v['ms'],3) for k,v in j['compute_roofline']['kernels'].items()})"
done
