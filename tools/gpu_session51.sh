for T in 384 256; do
cp sotest/libesom_$T.so paper_2201_00701_b200/libesom.so
timeout 300 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); print('c2 T=$T', round(j['value']/1e6,1), round(j['ms_per_step'],3), {k:round(v['ms'],3) for k,v in j['compute_roofline']['kernels'].items()})"
done
