set -x
for ch in 393216 1048576 2097152; do
  ESOM_EMBED_CHUNK=$ch timeout 300 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); print('c2 chunk $ch', round(j['value']/1e6,1), round(j['ms_per_step'],3), {k:round(v['ms'],3) for k,v in j['compute_roofline']['kernels'].items()})"
  ESOM_EMBED_CHUNK=$ch timeout 300 python bench.py --workload c4 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); print('c4 chunk $ch', round(j['value']/1e6,1), round(j['ms_per_step'],3), {k:round(v['ms'],3) for k,v in j['compute_roofline']['kernels'].items()})"
done
