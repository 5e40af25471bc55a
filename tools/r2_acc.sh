mkdir -p gpurun_out/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bmu_accum_smem -s 3 -c 1 -o /tmp/ncu_acc python tools/probe_frame.py c3 > /dev/null 2>&1; echo ncu=$?
python tools/ncu_summary.py /tmp/ncu_acc.ncu-rep gpurun_out/ncu/acc_c3 > /dev/null 2>&1
python tools/ncu_lines.py /tmp/ncu_acc.ncu-rep 20 > gpurun_out/ncu/acc_c3_lines.txt 2>&1
cat gpurun_out/ncu/acc_c3_lines.txt | head -22
python -c "
import json,glob; j=json.load(open(glob.glob('gpurun_out/ncu/acc_c3_0_*.json')[0])); print({k:j[k] for k in ['duration_ns','issue_active_pct','warps_active_avg','dram_bytes']}); print(j['stall_pct'])"
