set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k gemm > gpurun_out/s32_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/s32_pytest.log
PROBE_VARIANTS=w4 timeout 300 python tools/tc_probe.py c5 > gpurun_out/s32_probe1.log 2>&1
ESOM_T3_PASSES=2 PROBE_VARIANTS=w4 timeout 300 python tools/tc_probe.py c5 > gpurun_out/s32_probe2.log 2>&1
PROBE_VARIANTS=w4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s32_launches_c5.csv python tools/tc_probe.py c5 > /dev/null 2>&1
cat gpurun_out/s32_probe1.log gpurun_out/s32_probe2.log
