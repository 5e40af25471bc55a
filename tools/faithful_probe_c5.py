import sys, time, torch
sys.path.insert(0, '.')
from bench import make_inputs
import paper_2201_00701_b200 as esom
pts, hi, lo, k, _, _ = make_inputs("c5", 0, 1)
X = torch.from_numpy(pts[: 1 << 16]).cuda()
model = esom.LandmarkModel.create(hi, lo)
esom.embed(X, model, esom.EmbedParams(k=k), mode="faithful"); torch.cuda.synchronize()
t0 = time.perf_counter(); esom.embed(X, model, esom.EmbedParams(k=k), mode="faithful"); torch.cuda.synchronize()
print("c5 faithful 2^16 pts ms", (time.perf_counter() - t0) * 1e3)
