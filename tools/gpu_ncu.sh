set -x
# Round evidence run, part 2: ncu --set full captures of the dominant kernels,
# summarised ON THE BOX (tools/ncu_summary.py, tools/ncu_lines.py) so only small
# JSON/text files come back (gpurun returns <= 64 MiB).
mkdir -p gpurun_out/ncu
cap() {  # name, kernel regex, skip, command...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o /tmp/ncu_$name "$@" > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/ncu_$name.ncu-rep gpurun_out/ncu/$name > /dev/null 2>&1
  python tools/ncu_lines.py /tmp/ncu_$name.ncu-rep 30 > gpurun_out/ncu/${name}_lines.txt 2>&1
  rm -f /tmp/ncu_$name.ncu-rep
}
cap fused_c2 embed_fused 1 python tools/probe_trained.py 0 c2
cap screen_c2 knn_tc2 1 python tools/probe_trained.py 0 c2
cap fused_c2_trained embed_fused 3 python tools/probe_trained.py 40 c2 only
cap exact_c4 knn_exact_bits 1 python tools/probe_trained.py 0 c4
cap proj_c4 project_reg3 1 python tools/probe_trained.py 0 c4
cap screen_c4 knn_tc2 1 python tools/probe_trained.py 0 c4
cap gemm_c5 knn_gemm 0 python tools/probe_c5.py
cap group_c5 knn_exact_group 0 python tools/probe_c5.py
ls -la gpurun_out/ncu
# multi-rank dry run on the one GPU (2 processes, gloo): the sharded workloads and
# the max-over-ranks timing path of bench.py (the driver runs N > 1 over NCCL)
for w in c2 c3; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731 \
    bench.py --gpus 2 --steps 5 --warmup 3 --workload $w --dist-backend gloo --no-cpu-baseline \
    > gpurun_out/ncu/dry2_$w.json 2> gpurun_out/ncu/dry2_$w.err; echo dry2_$w=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29732 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/ncu/dry2_ref.json 2> gpurun_out/ncu/dry2_ref.err; echo dry2_ref=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/ncu/smoke.log
