set -x
mkdir -p gpurun_out
timeout 300 python tools/tc_probe.py c2 c4 > gpurun_out/s15_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_knn.py -x -q > gpurun_out/s15_pytest.log 2>&1; echo pytest=$?
PROBE_VARIANTS=w4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_tc2 -c 1 -o gpurun_out/s15_tc2_c2w4 python tools/tc_probe.py c2 > gpurun_out/s15_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:project_reg -c 1 -o gpurun_out/s15_proj_c2 python tools/kernel_times.py c2 >> gpurun_out/s15_ncu.log 2>&1
cat gpurun_out/s15_probe.log; tail -5 gpurun_out/s15_pytest.log; tail -3 gpurun_out/s15_ncu.log
