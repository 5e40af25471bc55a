import sys, torch, numpy as np
sys.path.insert(0, '.')
from bench import make_inputs
import paper_2201_00701_b200 as esom
pts, hi, lo, k, _, _ = make_inputs("c4", 0, 1)
X = torch.from_numpy(pts[:2_000_000]).cuda(); H = torch.from_numpy(hi).cuda()
nb = esom.knn(X, H, 16)
idx = nb.indices
order = torch.argsort(idx[:, 0].long(), stable=True)
s = idx[order]
for T in (128, 256, 512):
    n = (s.shape[0] // T) * T
    t = s[:n].view(-1, T * 16).long()
    # unique count per row
    srt = torch.sort(t, dim=1).values
    u = 1 + (srt[:, 1:] != srt[:, :-1]).sum(1)
    q = torch.quantile(u.float(), torch.tensor([0.1, 0.5, 0.9, 0.99], device=u.device))
    print(T, "mean U", u.float().mean().item(), "quantiles", q.tolist())
