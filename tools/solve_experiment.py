import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import h2gen, oracle, paper_1705_04601_b200 as h2sp
from paper_1705_04601_b200 import solve as hs
for N in [4096, 16384, 65536]:
    h = h2gen.make_config(2, N=N)
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed); sp = h2sp.Sparsifier(plan, packed); sp.build(); torch.cuda.synchronize()
    t0 = time.perf_counter(); ch = hs.factor(sp, plan); torch.cuda.synchronize(); tf = time.perf_counter() - t0
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(N)).cuda()
    t0 = time.perf_counter(); x = hs.solve(sp, ch, b); torch.cuda.synchronize(); ts = time.perf_counter() - t0
    ax = oracle.h2_matvec(h, x.cpu().numpy())
    res = np.linalg.norm(ax - b.cpu().numpy()) / np.linalg.norm(b.cpu().numpy())
    print(f"N={N} nnz(S)={plan.sizes['s_nnz']:.3e} factor {tf*1e3:.1f} ms (internal {ch.internal_bytes/1e9:.2f} GB) solve {ts*1e3:.2f} ms residual {res:.2e}", flush=True)
