mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x --durations=5 > gpurun_out/r2f_full.log 2>&1; echo full=$?
tail -15 gpurun_out/r2f_full.log
