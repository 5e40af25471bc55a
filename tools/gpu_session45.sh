timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_knn.py -x -q 2>&1 | tail -1
for v in 3 4; do
ESOM_TC2_W=$v ESOM_TC2_SPLIT=1 timeout 300 python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); print('c2 split W=$v', round(j['value']/1e6,1), round(j['ms_per_step'],3), {k:round(v['ms'],3) for k,v in j['compute_roofline']['kernels'].items()})"
done
timeout 300 python bench.py --workload c4 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); print('c4', round(j['value']/1e6,1), round(j['ms_per_step'],3), {k:round(v['ms'],3) for k,v in j['compute_roofline']['kernels'].items()})"
