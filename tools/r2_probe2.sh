mkdir -p gpurun_out
timeout 300 python tools/probe_trained.py 40 c2 2>&1 | tail -2
timeout 300 python tools/probe_trained.py 40 c4 2>&1 | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:knn_tc2 -s 1 -c 1 -o gpurun_out/r2g_screen_c4 python tools/probe_trained.py 0 c4 > /dev/null 2>&1; echo ncu=$?
