set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s48_smoke.log 2>&1; echo smoke=$?
tail -2 gpurun_out/s48_smoke.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload c3 --steps 5 --warmup 3 --no-cpu-baseline --dist-backend gloo > gpurun_out/s48_dist.json 2> gpurun_out/s48_dist.err; echo dist=$?
cat gpurun_out/s48_dist.json; tail -3 gpurun_out/s48_dist.err
