set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s25_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/s25_pytest.log
for w in c2 c3 c4 c5; do
  st=20; [ $w = c5 ] && st=5
  timeout 600 python bench.py --workload $w --steps $st --no-cpu-baseline > gpurun_out/s25_bench_$w.json 2> gpurun_out/s25_bench_$w.err
  cat gpurun_out/s25_bench_$w.json; tail -3 gpurun_out/s25_bench_$w.err
done
