"""Device direct solve x = V S^-1 U^T b on the config-2 recipe: factor / solve
times, factor size and residual against the oracle's H^2 matvec, for S's own
order and a METIS order.  usage (GPU): python tools/solve_experiment.py [N ...]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import h2gen  # noqa: E402
import oracle  # noqa: E402
import paper_1705_04601_b200 as h2sp  # noqa: E402
from paper_1705_04601_b200 import solve as hs  # noqa: E402

for N in [int(a) for a in sys.argv[1:]] or [4096, 16384, 65536]:
    h = h2gen.make_config(2, N=N)
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed)
    sp = h2sp.Sparsifier(plan, packed)
    sp.build()
    torch.cuda.synchronize()
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(N)).cuda()
    for order in ("metis", "s"):
        t0 = time.perf_counter()
        ch = hs.factor(sp, plan, order)
        torch.cuda.synchronize()
        tf = time.perf_counter() - t0
        t0 = time.perf_counter()
        x = hs.solve(sp, ch, b)
        torch.cuda.synchronize()
        ts = time.perf_counter() - t0
        ax = oracle.h2_matvec(h, x.cpu().numpy())
        res = np.linalg.norm(ax - b.cpu().numpy()) / np.linalg.norm(b.cpu().numpy())
        print(f"N={N} order={order} nnz(S)={plan.sizes['s_nnz']:.3e} factor {tf * 1e3:.1f} ms "
              f"(factor storage {ch.internal_bytes / 1e9:.2f} GB) solve {ts * 1e3:.2f} ms residual {res:.2e}", flush=True)
        del ch
