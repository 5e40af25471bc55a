"""e2e (pinned host -> host) of esom.embed for a workload under pipeline chunk settings."""
import json
import os
import statistics
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import make_inputs  # noqa: E402


def main(w):
    import importlib
    pts, hi, lo, k, _, _ = make_inputs(w, 0, 1)
    host = torch.from_numpy(pts).pin_memory()
    for chunk, depth in [(1 << 16, 4), (1 << 17, 3), (1 << 18, 3), (1 << 19, 2)]:
        os.environ["ESOM_PIPE_CHUNK"] = str(chunk)
        os.environ["ESOM_PIPE_DEPTH"] = str(depth)
        import paper_2201_00701_b200.projection as P
        importlib.reload(P)
        import paper_2201_00701_b200 as esom
        model = esom.LandmarkModel.create(hi, lo)
        params = esom.EmbedParams(k=k)
        P.embed(host, model, params)
        ts = []
        for _ in range(7):
            t0 = time.perf_counter()
            P.embed(host, model, params)
            ts.append(time.perf_counter() - t0)
        ms = statistics.median(ts) * 1e3
        print(json.dumps({"w": w, "chunk": chunk, "depth": depth, "e2e_ms": ms, "Mpts_per_s": host.shape[0] / ms / 1e3}),
              flush=True)


if __name__ == "__main__":
    for w in sys.argv[1:] or ["c2", "c4"]:
        main(w)
