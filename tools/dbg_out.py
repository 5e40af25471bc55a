import numpy as np, sys, os
sys.path.insert(0,'/root/repo')
import paper_2201_00701_b200 as esom
from paper_2201_00701_b200 import datagen
from oracle import oracle
gen = np.random.default_rng(11)
hi = gen.normal(size=(64, 16)).astype(np.float32)
lo = datagen.lattice(8, 8)
far = (gen.normal(size=(2000, 16)) * np.repeat([10.0, 100.0, 1000.0, 1.0], 500)[:, None]).astype(np.float32)
model = esom.LandmarkModel.create(hi, lo)
want = oracle.embed(far, hi, lo, 16)
got = esom.embed(far, model, esom.EmbedParams(k=16))
err = np.abs(got-want).max(1)
bad = np.nonzero(err>7e-4)[0]
print("bad", len(bad), "by block", np.bincount(bad//500, minlength=4))
nb = esom.knn_base(far, hi, 16)
for i in bad[:4]:
    print(i, got[i], want[i], err[i], nb.sqdists[i][[0,7,15]])
