set -x
mkdir -p gpurun_out
timeout 300 python tools/tc_probe.py c2 c4 > gpurun_out/s13_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/s13_pytest_tc.log 2>&1; echo pytest=$?
PROBE_VARIANTS=w3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_tc2 -c 1 -o gpurun_out/s13_tc2_c2 python tools/tc_probe.py c2 > gpurun_out/s13_ncu.log 2>&1
cat gpurun_out/s13_probe.log; tail -5 gpurun_out/s13_pytest_tc.log; tail -3 gpurun_out/s13_ncu.log
