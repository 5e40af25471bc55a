mkdir -p gpurun_out
timeout 300 python tools/probe_trained.py 40 c2 2>&1 | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:knn_exact_bits -s 1 -c 1 -o gpurun_out/r2e_exact python tools/probe_trained.py 0 c2 > /dev/null 2>&1; echo ncu1=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:project_reg2 -s 4 -c 1 -o gpurun_out/r2e_proj_trained python tools/probe_trained.py 40 c2 > /dev/null 2>&1; echo ncu2=$?
