set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/kernel_times.py c2 c4 > gpurun_out/kernel_times.jsonl 2> gpurun_out/kernel_times.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/bench_dry2.json 2> gpurun_out/bench_dry2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --workload c3 --dist-backend gloo --no-cpu-baseline > gpurun_out/bench_dry2_c3.json 2> gpurun_out/bench_dry2_c3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"project_reg" -c 1 -o gpurun_out/prof7p python tools/kernel_times.py c2 > gpurun_out/ncu_7p.log 2>&1
ls -la gpurun_out
