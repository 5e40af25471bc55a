for v in "" "ESOM_TC2_KEYCNT=1" "ESOM_TC2_NOSORT=1"; do
env $v timeout 300 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); print('c2 [$v]', round(j['value']/1e6,1), round(j['ms_per_step'],3), {k:round(v['ms'],3) for k,v in j['compute_roofline']['kernels'].items()})"
done
