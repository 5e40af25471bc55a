set -x
mkdir -p gpurun_out
timeout 300 python tools/tc_probe.py c2 c4 > gpurun_out/s12_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/s12_pytest_tc.log 2>&1; echo pytest=$?
timeout 200 python tools/kernel_times.py c2 c4 > gpurun_out/s12_ktimes.log 2>&1
cat gpurun_out/s12_probe.log; tail -5 gpurun_out/s12_pytest_tc.log; cat gpurun_out/s12_ktimes.log
