set -x
# Round evidence run, part 1 (gpurun): GPU tests (incl. the reference's own suites
# through install()), bench lines C2 (+trained), C3 (+trained), C4, C5, the reference
# arm, and the C2 launch list -> gpurun_out/ev_*.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/ev_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/ev_pytest.log
timeout 600 python bench.py > gpurun_out/ev_bench_c2.json 2> gpurun_out/ev_bench_c2.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ev_bench_ref_c2.json 2> gpurun_out/ev_bench_ref_c2.err
timeout 600 python bench.py --trained 40 --no-cpu-baseline > gpurun_out/ev_bench_c2_trained.json 2> gpurun_out/ev_bench_c2_trained.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/ev_bench_c3.json 2> gpurun_out/ev_bench_c3.err
timeout 600 python bench.py --workload c3 --trained 40 --no-cpu-baseline > gpurun_out/ev_bench_c3_trained.json 2> gpurun_out/ev_bench_c3_trained.err
timeout 900 python bench.py --workload c4 --no-cpu-baseline > gpurun_out/ev_bench_c4.json 2> gpurun_out/ev_bench_c4.err
timeout 900 python bench.py --workload c5 --steps 5 > gpurun_out/ev_bench_c5.json 2> gpurun_out/ev_bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
