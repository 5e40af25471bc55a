"""Summarise an ncu report (--set full) into profiles/: one JSON per kernel.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_c2 [--points N]

Key metrics: duration, DRAM bytes (read+write), SM/issue utilisation,
pipe utilisation (FMA, ALU, FP64, XU, tensor), occupancy, executed
instructions and the warp-stall breakdown.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

RAW = {
    "duration_ns": "gpu__time_duration.sum",  # scaled to ns / bytes below
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "tma_pipe_pct": "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active",
    "warps_active_avg": "sm__warps_active.avg.per_cycle_active",
    "registers": "launch__registers_per_thread",
    "inst_executed": "smsp__inst_executed.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
}


SCALE = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    scaled = []
    for r in rows[2:]:
        scaled.append([str(to_float(v) * SCALE[u]) if u in SCALE and to_float(v) is not None else v
                       for v, u in zip(r, units)])
    return hdr, scaled


def to_float(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    points = None
    if "--points" in sys.argv:
        points = int(sys.argv[sys.argv.index("--points") + 1])
    hdr, rows = raw_rows(rep)
    ki = hdr.index("Kernel Name")
    for n, r in enumerate(rows):
        name = r[ki]
        rec = {"kernel": name}
        for key, metric in RAW.items():
            if metric in hdr:
                rec[key] = to_float(r[hdr.index(metric)])
        stalls = {}
        for h, v in zip(hdr, r):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                f = to_float(v)
                if f:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = f
        tot = sum(stalls.values()) or 1.0
        rec["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])}
        rb, wb = rec.get("dram_read_bytes") or 0, rec.get("dram_write_bytes") or 0
        rec["dram_bytes"] = rb + wb
        if points:
            rec["points"] = points
            rec["dram_bytes_per_point"] = (rb + wb) / points
            if rec.get("inst_executed"):
                rec["lane_inst_per_point"] = rec["inst_executed"] * 32 / points
        short = name.split("(")[0].split()[-1].replace("<", "_").replace(">", "").replace(",", "_").replace(" ", "")
        out = Path(f"{prefix}_{n}_{short}.json")
        out.parent.mkdir(parents=True, exist_ok=True)
        out.write_text(json.dumps(rec, indent=1))
        print(out, json.dumps({k: rec.get(k) for k in ("duration_ns", "dram_bytes", "issue_active_pct",
                                                       "tensor_pipe_pct", "fma_pipe_pct", "fp64_pipe_pct")}))


if __name__ == "__main__":
    main()
