import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import h2gen, paper_1705_04601_b200 as h2sp
from paper_1705_04601_b200 import krylov as kr
from oracle import krylov as okr
N = int(sys.argv[1])
p = h2gen.pack(h2gen.make_ifmm(N, 1e-2, 64, 8)); sp = h2sp.Sparsifier(h2sp.Plan(p), p); sp.build()
p2 = h2gen.pack(h2gen.make_ifmm(N, 1e-2, 64, 32)); spo = h2sp.Sparsifier(h2sp.Plan(p2), p2); spo.build()
S = kr.CsrMatrix.from_sparsifier(sp)
F = kr.IlutFactors(S, 1e-3, -1)
nnz = int(S.col.numel())
t = time.time()
ref = okr.ilut(S.rowptr.cpu().numpy(), S.col.cpu().numpy(), S.val[:nnz].cpu().numpy(), 1e-3, -1)
print("oracle ilut", time.time() - t, flush=True)
lrp, lc, lv, urp, uc, uv, d = F.to_csr()
print("L pattern", np.array_equal(lrp, ref.l_rowptr) and np.array_equal(lc, ref.l_col),
      "U pattern", np.array_equal(urp, ref.u_rowptr) and np.array_equal(uc, ref.u_col),
      "vals", np.array_equal(lv, ref.l_val), np.array_equal(uv, ref.u_val), np.array_equal(d, ref.diag), flush=True)
b = torch.from_numpy(np.random.default_rng(1).standard_normal(N)).cuda()
r = []
for _ in range(2):
    x, info = kr.gmres(spo, b, M=sp, F=F, restart=30, tol=1e-10, maxiter=300)
    r.append((x.cpu().numpy(), info.iters))
print("gmres iters", r[0][1], r[1][1], "x bitwise", np.array_equal(r[0][0], r[1][0]), flush=True)
