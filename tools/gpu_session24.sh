set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_knn.py -x -q > gpurun_out/s24_pytest.log 2>&1; echo pytest=$?
PROBE_VARIANTS=w4 timeout 300 python tools/tc_probe.py c5 > gpurun_out/s24_probe.log 2>&1
PROBE_VARIANTS=w4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s24_launches_c5.csv python tools/tc_probe.py c5 > /dev/null 2>&1
tail -2 gpurun_out/s24_pytest.log; cat gpurun_out/s24_probe.log
