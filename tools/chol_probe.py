"""Timing probe of the supernodal Cholesky direct solve on a BASELINE config
recipe: analysis, factor, solve; residual against the oracle's H^2 matvec.
Usage: python tools/chol_probe.py [config] [N]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import h2gen  # noqa: E402
import oracle  # noqa: E402
import paper_1705_04601_b200 as h2sp  # noqa: E402
from paper_1705_04601_b200 import solve as sv  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
h = h2gen.make_config(cfg, N=N)
p = h2gen.pack(h)
plan = h2sp.Plan(p)
sp = h2sp.Sparsifier(plan, p)
sp.build()
torch.cuda.synchronize()
t = time.time()
AM = int(os.environ.get("CHOL_AMALG", "0"))
an = sv.CholAnalysis(plan, AM)
ta = time.time() - t
fac = sv.factor_chol(sp, amalgamate=AM)
torch.cuda.synchronize()
t = time.time()
fac = sv.factor_chol(sp, amalgamate=AM)
torch.cuda.synchronize()
tf = time.time() - t
b = torch.from_numpy(np.random.default_rng(1).standard_normal(N)).cuda()
x = sv.solve_chol(sp, fac, b)
torch.cuda.synchronize()
t = time.time()
for _ in range(3):
    x = sv.solve_chol(sp, fac, b)
torch.cuda.synchronize()
ts = (time.time() - t) / 3
r = oracle.h2_matvec(h, x.cpu().numpy()) - b.cpu().numpy()
print(f"config {cfg} N={N} amalgamate={AM}: S nnz {plan.sizes['s_nnz']:.3e}, supernodes {an.ns}, L panel entries "
      f"{an.panel_doubles:.3e}, flops {an.flops:.3e}; analysis {ta:.2f} s, factor {tf:.3f} s "
      f"({an.flops / tf / 1e12:.2f} TFLOP/s), solve {1e3 * ts:.1f} ms, residual "
      f"{np.linalg.norm(r) / np.linalg.norm(b.cpu().numpy()):.2e}", flush=True)
