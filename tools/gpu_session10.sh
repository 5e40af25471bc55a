set -x
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
timeout 300 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload c4 --steps 10 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"project_reg" -c 1 -o gpurun_out/prof10p python tools/kernel_times.py c2 > gpurun_out/ncu_10p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"knn_scan" -c 1 -o gpurun_out/prof10s python tools/kernel_times.py c2 > gpurun_out/ncu_10s.log 2>&1
ls -la gpurun_out
