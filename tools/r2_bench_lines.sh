#!/bin/bash
# bench lines of every workload (the evidence run's part 1 without the test suite / launch list)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python bench.py > gpurun_out/ev_bench_c2.json 2> gpurun_out/ev_bench_c2.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ev_bench_ref_c2.json 2> gpurun_out/ev_bench_ref_c2.err
timeout 600 python bench.py --trained 40 --no-cpu-baseline > gpurun_out/ev_bench_c2_trained.json 2> gpurun_out/ev_bench_c2_trained.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/ev_bench_c3.json 2> gpurun_out/ev_bench_c3.err
timeout 600 python bench.py --workload c3 --trained 40 --no-cpu-baseline > gpurun_out/ev_bench_c3_trained.json 2> gpurun_out/ev_bench_c3_trained.err
timeout 900 python bench.py --workload c4 --no-cpu-baseline > gpurun_out/ev_bench_c4.json 2> gpurun_out/ev_bench_c4.err
timeout 900 python bench.py --workload c5 --steps 5 > gpurun_out/ev_bench_c5.json 2> gpurun_out/ev_bench_c5.err
ls -la gpurun_out/ev_bench_*.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo smoke=$?
