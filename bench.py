#!/usr/bin/env python
"""Benchmark of the EmbedSOM hot path on B200 (contract: see DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c4|c5] [--impl ours|reference]

Default workload = BASELINE.json configs[1] (C2): 2^20 x 32-d synthetic
Gaussian-mixture points, 16x16 SOM (256 landmarks), k = 16, projection only.
A step is one full re-projection (one frame) of every point of the rank's
shard.  N > 1 (torchrun) is weak scaling: each rank owns its own 2^20-point
shard; landmarks are replicated; projection has no collective.  c3/c4 add
the batch-SOM training step (fused BMU statistics + one NCCL all-reduce +
landmark update) to every frame.

Rank 0 prints ONE JSON line.  `--impl reference` times the reference's CPU
algorithm (the oracle port, oracle/esom_oracle.c, all host threads) on a
bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "embedded points/sec & fps (1M–10M pts) at 1/2/4/8 B200; % HBM roofline"
UNIT = "points/s"

WORKLOADS = {
    # name: (clusters, n per rank, d, rows, cols, k, train, description)
    "c2": (16, 1 << 20, 32, 16, 16, 16, False,
           "C2: 2^20x32 Gaussian mixture, 16x16 SOM (256 landmarks), k=16, projection only"),
    "c3": (16, 1 << 20, 32, 16, 16, 16, True,
           "C3: 2^20x32, 256 landmarks, k=16, batch-SOM step (BMU stats + all-reduce + update) + re-projection per frame"),
    "c4": (16, 1_250_000, 32, 32, 32, 16, True,
           "C4 shard: 1.25M x32 per GPU (10M over 8), 1024 landmarks, k=16, batch-SOM step + re-projection"),
    "c5": (32, 1 << 20, 512, 64, 64, 32, False,
           "C5: 2^20x512, 4096 landmarks, k=32, projection only (CUDA-core exact path)"),
}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


def make_inputs(workload: str, rank: int):
    from paper_2201_00701_b200 import datagen

    c, n, d, rows, cols, k, train, _ = WORKLOADS[workload]
    # the model comes from the seed-1 dataset on every rank (identical landmarks)
    base = datagen.gaussians_f32(c, n, d, seed=1)
    hi, lo = datagen.som_model(base, rows, cols, seed=2)
    pts = base if rank == 0 else datagen.gaussians_f32(c, n, d, seed=1 + rank)
    return pts, hi, lo, k, train


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every ~2 ms while the
    timed region runs (B200_PROFILING.md clocks recipe, in-process)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001 -- no NVML: report unsampled
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((float(mhz), int(rs)))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({name for _, r in self.samples for name, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(m for m, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "NVML, 2 ms polling"}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return j.get("hbm_gbs", 6541.8), j.get("bf16_tflops", 1649.8), "measured"
    return 6650.0, 1590.0, "fallback"


def ncu_traffic(workload: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        j = json.loads(p.read_text())
        v = j.get(workload)
        if isinstance(v, dict):
            return v.get("dram_bytes_per_launch")
    return None


# ---------------------------------------------------------------------------
# CPU arms (oracle port; test infrastructure, never the measured product)
# ---------------------------------------------------------------------------
def cpu_embed_rate(pts, hi, lo, k, n_sample: int, threads: int):
    from oracle import oracle  # checker / CPU baseline only

    sub = np.ascontiguousarray(pts[:n_sample])
    oracle.embed(sub[:256], hi, lo, k, "base", threads=1)  # warm (page-in)
    t0 = time.perf_counter()
    oracle.embed(sub, hi, lo, k, "base", threads=threads)
    dt = time.perf_counter() - t0
    return n_sample / dt, dt


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    workload = args.workload
    pts, hi, lo, k, train = make_inputs(workload, 0)
    cores = host_cores()
    c, n, d, rows, cols, k, train, desc = WORKLOADS[workload]
    # per-step sample sized for ~1 s of wall time on the host's cores
    per_pt_us = {"c2": 20.0, "c3": 20.0, "c4": 60.0, "c5": 2500.0}[workload]
    n_sample = int(max(256, min(n, cores * 1e6 / per_pt_us)))
    for _ in range(max(0, args.warmup)):
        cpu_embed_rate(pts, hi, lo, k, min(n_sample, 4096), cores)
    rates, times = [], []
    for _ in range(args.steps):
        r, dt = cpu_embed_rate(pts, hi, lo, k, n_sample, cores)
        rates.append(r)
        times.append(dt)
    total_pts = n_sample * args.steps
    value = total_pts / sum(times)
    sample = (f"{n_sample} of {n} points per step ({workload}), oracle port of embed (knn_base + scores + "
              f"projection, ref: projection.py:220-245), {cores} threads, row-sharded")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic (reference datagen.gaussians restated)",
        "config": {"workload": desc, "n_per_rank": n, "d": d, "g": rows * cols, "k": k},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    ndev = max(1, torch.cuda.device_count())
    dev = torch.device("cuda", local % ndev)  # one process per GPU (modulo only for single-GPU dry runs)
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    import paper_2201_00701_b200 as esom
    from paper_2201_00701_b200.batch_som import BatchSomConfig, FrameLoop

    workload = args.workload
    c, n, d, rows, cols, k, train, desc = WORKLOADS[workload]
    pts, hi, lo, k, train = make_inputs(workload, rank)
    g = rows * cols
    X = torch.from_numpy(pts).to(dev)
    loop = FrameLoop(X, hi, lo, k, BatchSomConfig(sigma=1.0, alpha=0.05), train=train)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    stream = torch.cuda.current_stream(dev)
    for _ in range(max(3, args.warmup)):
        loop.frame()
    barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev.index) as clk:
        barrier()
        for s in range(args.steps):
            flush.zero_()  # L2 flush between timed steps, outside the events
            ev[s][0].record(stream)
            loop.frame()
            ev[s][1].record(stream)
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = sum(step_ms) / len(step_ms)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_points = n * world
    value = total_points / (ms_max * 1e-3)

    # ---- dominant kernel: the exact k-NN (tensor-core screened where eligible),
    # timed alone over the whole shard with CUDA events on the launching stream.
    # Algorithmic bytes of the k-NN API per point: 4d (X) + 8k (idx + sqd),
    # SURVEY.md §8d.  The embed-level figure (4d + 8 per point) is reported too.
    from paper_2201_00701_b200 import _dev as _d, _lib as _l

    idx = torch.empty((n, k), dtype=torch.int32, device=dev)
    sqd = torch.empty((n, k), dtype=torch.float32, device=dev)
    wsk = torch.empty(_l.load().esom_workspace_bytes(g, d, k, 0), dtype=torch.uint8, device=dev)
    kflag = _d.new_flag(dev)
    sh = _d.stream_handle(dev)

    def knn_call():
        _l.call("esom_knn", _d.ptr(X), n, d, _d.ptr(loop.model.hi), g, k, _d.ptr(idx), _d.ptr(sqd), _d.ptr(kflag),
                _d.ptr(wsk), wsk.numel(), sh)

    def ev_time(fn, reps=5):
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    knn_call()
    kern = ev_time(knn_call)
    emb = ev_time(lambda: loop.model.embed_into(X, loop.xy, flag=loop.flag))
    del idx, sqd, wsk
    hbm_peak, bf16_peak, peak_kind = measured_peaks()
    alg_bytes = n * (4 * d + 8 * k)
    achieved = alg_bytes / (kern * 1e-3) / 1e9
    clocks = clk.summary()
    sm_mhz = clocks["sm_mhz"] or 1965.0
    fp32_peak = 148 * 128 * sm_mhz * 1e6 / 1e12  # lane-ops/s (T), at the sampled clock
    exact_ops = n * 3.0 * g * d / (emb * 1e-3) / 1e12  # exact-path equivalent sub/mul/add per element
    gemm_tflops = n * 2.0 * g * 16 * ((d + 15) // 16) * 3 / (kern * 1e-3) / 1e12  # split-bf16 screen
    tc_used = d <= 32 and g <= 4096 and k <= 16 and os.environ.get("ESOM_TC", "1") != "0"
    # ---- end to end through the public API: pinned host points in, host xy out ----
    e2e = None
    if True:  # every rank measures; the slowest rank defines the job's e2e time
        host = torch.from_numpy(pts).pin_memory()
        model = esom.LandmarkModel.create(hi, lo)
        params = esom.EmbedParams(k=k)
        esom.embed(host, model, params)  # warm
        times = []
        for _ in range(max(3, min(args.steps, 10))):
            barrier()
            t0 = time.perf_counter()
            out = esom.embed(host, model, params)  # H2D, fused kernel, D2H (numpy back)
            times.append(time.perf_counter() - t0)
        e2e_s = statistics.median(times)
        et = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": total_points / float(et.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(host.numel() * 4), "d2h_bytes_per_step": int(out.nbytes),
               "how": "esom.embed(pinned host tensor, model, EmbedParams) incl. model prep, H2D, kernel, D2H; "
                      "wall clock, median"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cores = host_cores()
        n_s = int(min(n, max(4096, cores * 30_000))) if d <= 64 else 2048
        rate, dt = cpu_embed_rate(pts, hi, lo, k, n_s, cores)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"first {n_s} points of the {workload} workload, oracle port of embed (base backend), "
                         f"{cores} threads, {dt:.2f} s wall"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_max, "fps": 1e3 / ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (exact k-NN), f64 accum",
            "data": "synthetic Gaussian mixture (reference datagen.gaussians restated), SOM-initialised landmarks",
            "config": {"workload": desc, "n_per_rank": n, "d": d, "g": g, "k": k, "train": train,
                       "parallelism": f"points sharded x{world}, landmarks replicated",
                       "l2": "flushed between timed steps (256 MiB write outside the events); X = 128 MiB/rank"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": ncu_traffic(workload), "peak_kind": peak_kind,
                         "kernel": ("knn_tc_kernel (tcgen05 split-bf16 screen + exact f32 recheck)" if tc_used
                                    else "knn_scan_kernel (exact f32, CUDA cores)"),
                         "kernel_ms": kern, "alg_bytes_per_point": 4 * d + 8 * k,
                         "embed_ms": emb, "embed_hbm_frac": n * (4 * d + 8) / (emb * 1e-3) / 1e9 / hbm_peak},
            "compute_roofline": {"exact_equiv_Tops": exact_ops, "fp32_peak_Tops_at_sampled_clock": fp32_peak,
                                 "exact_equiv_frac": exact_ops / fp32_peak,
                                 "tensor_TFLOPs": gemm_tflops if tc_used else 0.0,
                                 "tensor_frac_of_bf16_peak": (gemm_tflops / bf16_peak) if tc_used else 0.0,
                                 "note": "exact_equiv = 3*g*d f32 ops per point / embed time (what the exact "
                                         "CUDA-core path must issue); tensor = split-bf16 x.L^T MMA flops / k-NN time"},
            "clocks": clocks,
            "gpu_launches": args.steps * loop.launches_per_frame,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo only for single-GPU dry runs")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
