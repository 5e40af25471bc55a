set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k gemm > gpurun_out/s38_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/s38_pytest.log
PROBE_VARIANTS=scan,w4 timeout 300 python tools/tc_probe.py c5 > gpurun_out/s38_probe1.log 2>&1
ESOM_T3_COARSE=0 PROBE_VARIANTS=w4 timeout 300 python tools/tc_probe.py c5 > gpurun_out/s38_probe0.log 2>&1
cat gpurun_out/s38_probe1.log gpurun_out/s38_probe0.log
