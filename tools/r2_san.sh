mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/san_workload.py > gpurun_out/r2_san_$tool.log 2>&1
  echo $tool=$?; tail -3 gpurun_out/r2_san_$tool.log
done
timeout 600 python -m pytest tests/test_gpu_nccl_graph.py -q > gpurun_out/r2_nccl.log 2>&1; echo nccl=$?; tail -3 gpurun_out/r2_nccl.log
