set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s20_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/s20_pytest.log
PROBE_VARIANTS=w4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s20_launches_c5.csv python tools/tc_probe.py c5 > /dev/null 2>&1
PROBE_VARIANTS=w4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_gemm -c 1 -o gpurun_out/s20_gemm_c5 python tools/tc_probe.py c5 > gpurun_out/s20_ncu.log 2>&1
PROBE_VARIANTS=w4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_exact_warp -c 1 -o gpurun_out/s20_exact_c5 python tools/tc_probe.py c5 >> gpurun_out/s20_ncu.log 2>&1
tail -2 gpurun_out/s20_ncu.log
