"""Small invocations of every libh2sp kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): stored build + applies on configs[0] and a
B = 128 random case, a bench-mode close_gen build (config-5 recipe, N = 8192),
ILUT / triangular solves / SpMV / GMRES on a small problem."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import h2gen  # noqa: E402
import paper_1705_04601_b200 as h2sp  # noqa: E402
from paper_1705_04601_b200 import krylov as kr  # noqa: E402


def stored(h):
    p = h2gen.pack(h)
    plan = h2sp.Plan(p)
    sp = h2sp.Sparsifier(plan, p)
    sp.build()
    b = torch.randn(2, plan.n_tree_local, dtype=torch.float64, device="cuda")
    y = torch.empty(2, plan.s_rows, dtype=torch.float64, device="cuda")
    sp.apply_Ut(b, y)
    sp.apply_V(y, b)
    torch.cuda.synchronize()
    return sp


stored(h2gen.make_config(1))
stored(h2gen.random_h2(4, 128, 3, True, eta=0.7, max_rank=32))
stored(h2gen.random_h2(4, 64, 4, False, eta=0.7, max_rank=32))
# bench mode, matrix-free close blocks (config-5 recipe, B = 128)
h = h2gen.make_config(5, N=8192)
p = h2gen.pack(h)
plan = h2sp.Plan(p, bench=True)
sp = h2sp.Sparsifier(plan, p, close_gen={"points": h.points, "kernel": h.meta["kernel"]})
sp.outputs["bench_w"].copy_(torch.randn(h.N, dtype=torch.float64))
sp.build()
torch.cuda.synchronize()
# ILUT / solves / SpMV / GMRES
rp, ci, v = h2gen.random_sparse(40, 16, 1, density=0.1, shift=0.3)
A = kr.CsrMatrix(torch.from_numpy(rp), torch.from_numpy(ci), torch.from_numpy(v))
F = kr.IlutFactors(A, 1e-2, 8)
bb = torch.randn(A.n, dtype=torch.float64, device="cuda")
F.solve(bb)
A.matvec(bb)
hop = h2gen.make_ifmm(2048, 1e-2, 32, 8)
spo = stored(hop)
Fo = kr.IlutFactors(kr.CsrMatrix.from_sparsifier(spo), 1e-3, -1)
x, info = kr.gmres(spo, torch.randn(2048, dtype=torch.float64, device="cuda"), M=spo, F=Fo, restart=10, maxiter=20)
torch.cuda.synchronize()
print("sanitize cases done", info.iters, flush=True)
