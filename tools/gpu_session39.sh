set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_knn.py tests/test_gpu_train.py -x -q > gpurun_out/s39_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/s39_pytest.log
PROBE_VARIANTS=w2,w3,w4 timeout 300 python tools/tc_probe.py c2 c4 > gpurun_out/s39_probe.log 2>&1
cat gpurun_out/s39_probe.log
