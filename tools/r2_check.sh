mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_dropin.py -q -rA > gpurun_out/r2c_dropin.log 2>&1; echo dropin=$?
grep -E "^E +FAILED|passed|failed" gpurun_out/r2c_dropin.log | tail -30
for w in "c2" "c2 --trained 40" "c3" "c4" ; do
  tag=$(echo $w | tr ' ' '_' | tr -d '-')
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r2c_bench_$tag.json 2> gpurun_out/r2c_bench_$tag.err; echo bench $w = $?
  python -c "import json,sys; j=json.loads(open('gpurun_out/r2c_bench_$tag.json').read()); print(j['value']/1e6, j['ms_per_step'], j['roofline']['kernel'], j['roofline']['kernel_ms_per_frame'], j['e2e']['value']/1e6, j['e2e_numpy']['value']/1e6, j['cuda_graph'])" || tail -5 gpurun_out/r2c_bench_$tag.err
done
