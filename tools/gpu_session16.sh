set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_projection.py -x -q > gpurun_out/s16_pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/kernel_times.py c2 c4 > gpurun_out/s16_kt_v2.log 2>&1
ESOM_PROJ_V1=1 timeout 300 python tools/kernel_times.py c2 c4 > gpurun_out/s16_kt_v1.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s16_launches_c2.csv python tools/kernel_times.py c2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:project_reg2 -c 1 -o gpurun_out/s16_proj2_c2 python tools/kernel_times.py c2 > gpurun_out/s16_ncu.log 2>&1
tail -5 gpurun_out/s16_pytest.log; cat gpurun_out/s16_kt_v2.log gpurun_out/s16_kt_v1.log; tail -2 gpurun_out/s16_ncu.log
