import sys; sys.path.insert(0,".")
import torch, numpy as np
import paper_2201_00701_b200 as esom
from paper_2201_00701_b200 import datagen
from paper_2201_00701_b200.core import Rng
n = int(sys.argv[1]); B = int(sys.argv[2])
pts = datagen.gaussians_f32(16, n, 32, seed=1)
hi, lo = datagen.som_model(pts, 16, 16, seed=2)
m = esom.LandmarkModel.create(hi, lo)
print(esom.som_tick(pts, m, esom.SomConfig(batch_size=B), Rng(1))[:1,:4])
