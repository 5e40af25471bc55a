import numpy as np, sys, os
sys.path.insert(0,'/root/repo')
import paper_2201_00701_b200 as esom
from paper_2201_00701_b200 import datagen
from oracle import oracle
k=3
gen = np.random.default_rng(k)
pts, _ = datagen.gaussians(6, 3000, 8, seed=k)
hi = pts[gen.choice(3000, 100, replace=False)]
lo = datagen.lattice(10, 10)
model = esom.LandmarkModel.create(hi, lo)
want = oracle.embed(pts, hi, lo, k)
got = esom.embed(pts, model, esom.EmbedParams(k=k), backend="base")
err = np.abs(got-want).max(1)
bad = np.nonzero(err>1e-3)[0]
print("bad", len(bad))
nb = esom.knn_base(pts, hi, k)
for i in bad[:6]:
    print(i, got[i], want[i], nb.indices[i], nb.sqdists[i], lo[nb.indices[i]].tolist())
