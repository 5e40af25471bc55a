set -x
# Round-end evidence run (gpurun): GPU tests, bench lines C2-C5 + reference arm, launch list,
# ncu --set full captures of the dominant kernels -> gpurun_out/r_* (summarise into profiles/ with
# tools/ncu_summary.py).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r_pytest.log 2>&1; echo pytest=$?
tail -1 gpurun_out/r_pytest.log
timeout 600 python bench.py > gpurun_out/r_bench_c2.json 2> gpurun_out/r_bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r_bench_ref_c2.json 2> gpurun_out/r_bench_ref_c2.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r_bench_c3.json 2> gpurun_out/r_bench_c3.err
timeout 600 python bench.py --workload c4 --no-cpu-baseline > gpurun_out/r_bench_c4.json 2> gpurun_out/r_bench_c4.err
timeout 900 python bench.py --workload c5 --steps 5 > gpurun_out/r_bench_c5.json 2> gpurun_out/r_bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
PROBE_VARIANTS=w4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_exact_bits -c 1 -o gpurun_out/r_exact_c2 python tools/tc_probe.py c2 > /dev/null 2>&1
PROBE_VARIANTS=w4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_tc2 -c 1 -o gpurun_out/r_screen_c2 python tools/tc_probe.py c2 > /dev/null 2>&1
PROBE_VARIANTS=w4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_tc2 -c 1 -o gpurun_out/r_screen_c4 python tools/tc_probe.py c4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:project_reg2 -c 1 -o gpurun_out/r_proj_c2 python tools/kernel_times.py c2 > /dev/null 2>&1
PROBE_VARIANTS=w4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_exact_group -c 1 -o gpurun_out/r_group_c5 python tools/tc_probe.py c5 > /dev/null 2>&1
# rows either side of the path + the on-chip online tick and the far-point projection
timeout 600 python tools/bench_rows.py > gpurun_out/r_rows.jsonl 2> gpurun_out/r_rows.err
timeout 300 python tools/probe_train.py > gpurun_out/r_train.txt 2>&1
timeout 300 python tools/probe_tick.py > gpurun_out/r_tick.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:online_tick_row -c 1 -o gpurun_out/r_tick_c3 python tools/probe_train.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fcs_decode|dim_partial4|transform4|frame_points_pack" -c 4 -o gpurun_out/r_rows python tools/bench_rows.py --rows ingest,engine --steps 2 > /dev/null 2>&1
ls gpurun_out
