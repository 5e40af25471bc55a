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
import ctypes
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
           "C5: 2^20x512, 4096 landmarks, k=32, projection only (tcgen05 split-bf16 GEMM screen + exact re-evaluation)"),
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


def ncu_traffic(workload: str, points_per_launch: float):
    """DRAM bytes per launch of the dominant kernel: the committed ncu capture's
    bytes/point (profiles/traffic.json) x the points one launch processes here."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        j = json.loads(p.read_text())
        v = j.get(workload)
        if isinstance(v, dict) and v.get("points"):
            return v["dram_bytes"] / v["points"] * points_per_launch
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
    # one frame = one CUDA-graph launch (single rank, or no collective in the frame;
    # NCCL inside captured graphs is left out of the multi-rank training loop)
    use_graph = not args.no_graph and (world == 1 or not train)
    if use_graph:
        loop.capture()
        loop.frame()
        barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    from paper_2201_00701_b200 import _lib as _lc

    launches0 = _lc.load().esom_launch_count()
    with ClockSampler(dev.index) as clk:
        barrier()
        for s in range(args.steps):
            flush.zero_()  # L2 flush between timed steps, outside the events
            ev[s][0].record(stream)
            loop.frame()
            ev[s][1].record(stream)
        barrier()
    launches_timed = _lc.load().esom_launch_count() - launches0  # our kernels inside the timed region
    if use_graph:  # replays bypass the host-side counter: kernels captured per frame x frames
        launches_timed = loop.graph_launches * args.steps
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = sum(step_ms) / len(step_ms)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_points = n * world
    value = total_points / (ms_max * 1e-3)

    # ---- dominant kernel of the frame, timed live with CUDA events on the
    # launching stream (libesom's esom_timing_* hooks around each launch),
    # one extra L2-flushed frame after the timed region.  Algorithmic work per
    # point: k-NN kernels 4d (X) + 8k (idx + sqd) bytes, the
    # d > 32 GEMM screen 2 g d flops (one x.L^T), the projection 8k + 8 bytes.
    from paper_2201_00701_b200 import _dev as _d, _lib as _l

    L = _l.load()
    flush.zero_()
    torch.cuda.synchronize(dev)
    L.esom_timing_begin(1)
    loop._eager_frame()  # eager: the timing hooks record events around each launch
    torch.cuda.synchronize(dev)
    ktimes = {}
    for name in ("knn_tc2_kernel", "knn_exact_bits_kernel", "knn_gemm_kernel", "knn_exact_group_kernel",
                 "project_kernel"):
        cnt = ctypes.c_int32(0)
        ms_k = L.esom_timing_query(name.encode(), ctypes.byref(cnt))
        if cnt.value:
            ktimes[name] = {"ms": ms_k, "launches": cnt.value, "share_of_frame": ms_k / ms}
    L.esom_timing_begin(0)
    dom = max(ktimes, key=lambda kk: ktimes[kk]["ms"]) if ktimes else None
    hbm_peak, bf16_peak, peak_kind = measured_peaks()
    clocks = clk.summary()
    sm_mhz = clocks["sm_mhz"] or 1965.0
    fp32_peak = 148 * 128 * sm_mhz * 1e6 / 1e12  # lane-ops/s (T), at the sampled clock
    dk = (d + 31) // 32 * 32
    if dom == "knn_gemm_kernel":
        kms = ktimes[dom]["ms"]
        alg_flops = 2.0 * n * g * d
        mma_flops = 2.0 * n * g * dk * 3 * 2  # split-bf16 (3 products) x two passes, as executed
        roofline = {"bound": "tensor", "achieved": alg_flops / (kms * 1e-3) / 1e12, "peak": bf16_peak,
                    "unit": "TFLOP/s", "frac": alg_flops / (kms * 1e-3) / 1e12 / bf16_peak,
                    "traffic": ncu_traffic(workload, n / ktimes[dom]["launches"]), "peak_kind": peak_kind,
                    "kernel": dom, "kernel_ms_per_frame": kms, "launches": ktimes[dom]["launches"],
                    "alg_flops_per_point": 2 * g * d,
                    "executed_mma_TFLOPs": mma_flops / (kms * 1e-3) / 1e12,
                    "executed_mma_frac_of_bf16_peak": mma_flops / (kms * 1e-3) / 1e12 / bf16_peak,
                    "note": "achieved = algorithmic 2gd flops/point (one x.L^T); the kernel issues 6x that in "
                            "bf16 MMAs (x_hi l_hi + x_hi l_lo + x_lo l_hi, group-min pass + candidate pass)"}
    elif dom is not None:
        kms = ktimes[dom]["ms"]
        per_pt = (4 * d + 8 * k) if dom.startswith("knn") else (8 * k + 8)
        achieved = n * per_pt / (kms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved / hbm_peak, "traffic": ncu_traffic(workload, n / ktimes[dom]["launches"]),
                    "peak_kind": peak_kind,
                    "kernel": dom, "kernel_ms_per_frame": kms, "launches": ktimes[dom]["launches"],
                    "alg_bytes_per_point": per_pt,
                    "note": "issue-bound exact selection (SURVEY §8d: distance intensity >> HBM ridge); "
                            "compute_roofline gives the pipe view"}
    else:
        roofline = None
    embed_frac = n * (4 * d + 8) / (ms * 1e-3) / 1e9 / hbm_peak
    exact_ops = n * 3.0 * g * d / (ms * 1e-3) / 1e12  # exact-path equivalent sub/mul/add per element
    compute_roofline = {"exact_equiv_Tops": exact_ops, "fp32_peak_Tops_at_sampled_clock": fp32_peak,
                        "exact_equiv_frac": exact_ops / fp32_peak, "embed_hbm_frac": embed_frac,
                        "kernels": ktimes,
                        "note": "exact_equiv = 3*g*d f32 ops per point / frame time (what an exact CUDA-core scan "
                                "must issue); kernels: per-kernel device ms inside one frame"}
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
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": ("f32 exact k-NN (bf16x3 tcgen05 screen), f32/f64 projection" if d > 32 else "f32 exact k-NN (bf16x3 tcgen05 screen), f32/f64 projection"),
            "data": "synthetic Gaussian mixture (reference datagen.gaussians restated), SOM-initialised landmarks",
            "config": {"workload": desc, "n_per_rank": n, "d": d, "g": g, "k": k, "train": train,
                       "parallelism": f"points sharded x{world}, landmarks replicated",
                       "l2": "flushed between timed steps (256 MiB write outside the events); X = 128 MiB/rank",
                       "cuda_graph": use_graph},
            "roofline": roofline,
            "compute_roofline": compute_roofline,
            "clocks": clocks,
            "gpu_launches": launches_timed,
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
    ap.add_argument("--no-graph", action="store_true", help="launch each frame's kernels eagerly (no CUDA graph)")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo only for single-GPU dry runs")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
