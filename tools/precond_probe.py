"""Timing probe of the preconditioning workload pieces on one GPU (not a bench
line): generation, the two sparsifications, ILUT, triangular solves, SpMV,
applies, GMRES.  Usage: python tools/precond_probe.py N d tau"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import h2gen  # noqa: E402
import paper_1705_04601_b200 as h2sp  # noqa: E402
from paper_1705_04601_b200 import krylov as kr  # noqa: E402


def ev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    d = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2
    tau = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-2
    B = 64
    t = time.time()
    hop = h2gen.make_ifmm(N, d, B, 32)
    hpre = h2gen.make_ifmm(N, d, B, 8)
    print(f"gen {time.time() - t:.1f} s", flush=True)
    sps = []
    for h in (hop, hpre):
        p = h2gen.pack(h)
        plan = h2sp.Plan(p)
        sp = h2sp.Sparsifier(plan, p)
        ms = ev_time(lambda: sp.build(), reps=2)
        print(f"sparsify r={h.meta['r']}: {ms:.2f} ms nnz={plan.sizes['s_nnz']:.3e}", flush=True)
        sps.append(sp)
    spo, spp = sps
    del hop, hpre
    Sp = kr.CsrMatrix.from_sparsifier(spp)
    So = kr.CsrMatrix.from_sparsifier(spo)
    torch.cuda.synchronize()
    t = time.time()
    F = kr.IlutFactors(Sp, tau, -1)
    torch.cuda.synchronize()
    print(f"ilut tau={tau}: {1e3 * (time.time() - t):.1f} ms, factor nnz {F.nnz:.3e} (S nnz {Sp.col.numel():.3e})",
          flush=True)
    b = torch.randn(N, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    print(f"trsv pair: {ev_time(lambda: F.solve(b, x)):.3f} ms", flush=True)
    print(f"spmv op: {ev_time(lambda: So.matvec(b, x)):.3f} ms ({So.col.numel() * 12 / 1e9:.2f} GB)", flush=True)
    y = torch.empty(1, N, dtype=torch.float64, device="cuda")
    print(f"apply_Ut op: {ev_time(lambda: spo.apply_Ut(b.view(1, -1), y)):.3f} ms", flush=True)
    for M, FF, name in ((spp, F, "ilut"), (None, None, "none")):
        torch.cuda.synchronize()
        t = time.time()
        xx, info = kr.gmres(spo, b, M=M, F=FF, restart=30, tol=1e-10, maxiter=300)
        torch.cuda.synchronize()
        print(f"gmres precond={name}: {1e3 * (time.time() - t):.1f} ms, iters {info.iters}, conv {info.converged}",
              flush=True)


if __name__ == "__main__":
    main()
