set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s28_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/s28_pytest.log
for w in c3 c4; do
  timeout 600 python bench.py --workload $w --steps 20 --no-cpu-baseline > gpurun_out/s28_bench_$w.json 2> gpurun_out/s28_bench_$w.err
  tail -2 gpurun_out/s28_bench_$w.err
done
