mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_dropin.py -q -rA > gpurun_out/r2b_dropin.log 2>&1; echo dropin=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/r2b_dropin.log | tail -30
