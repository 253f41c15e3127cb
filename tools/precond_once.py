"""One ILUT + one GMRES solve of the preconditioning experiment (ncu capture)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import h2gen  # noqa: E402
import paper_1705_04601_b200 as h2sp  # noqa: E402
from paper_1705_04601_b200 import krylov as kr  # noqa: E402

N, d, tau = int(sys.argv[1]), float(sys.argv[2]), float(sys.argv[3])
sps = []
for r in (32, 8):
    p = h2gen.pack(h2gen.make_ifmm(N, d, 64, r))
    sp = h2sp.Sparsifier(h2sp.Plan(p), p)
    sp.build()
    sps.append(sp)
F = kr.IlutFactors(kr.CsrMatrix.from_sparsifier(sps[1]), tau, -1)
b = torch.from_numpy(np.random.default_rng(1).standard_normal(N)).cuda()
x, info = kr.gmres(sps[0], b, M=sps[1], F=F, restart=30, tol=1e-10, maxiter=300)
torch.cuda.synchronize()
print("ok", info.iters)
