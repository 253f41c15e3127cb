"""One factorisation + one solve (for ncu launch lists)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import h2gen  # noqa: E402
import paper_1705_04601_b200 as h2sp  # noqa: E402
from paper_1705_04601_b200 import solve as sv  # noqa: E402

cfg, N = int(sys.argv[1]), int(sys.argv[2])
h = h2gen.make_config(cfg, N=N)
p = h2gen.pack(h)
plan = h2sp.Plan(p)
sp = h2sp.Sparsifier(plan, p)
sp.build()
fac = sv.factor_chol(sp)
x = sv.solve_chol(sp, fac, torch.from_numpy(np.random.default_rng(1).standard_normal(N)).cuda())
torch.cuda.synchronize()
print("ok")
