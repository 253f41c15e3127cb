"""GPU parity of the preconditioning workload and
of the direct solve's complete LU (§8(f) #1): the CUDA path (libh2sp through
the C ABI) against the plain-C / numpy oracle (oracle/ilut.c, oracle/krylov.py)
on the same seeded inputs.

* ILUT factors: BITWISE equal (pattern and values) -- both sides take every
  dropping decision on the same FP64 values, computed in the same order with
  the same two-rounding updates (reading 25).
* triangular solves, SpMV: 1e-12 relative (summation order differs).
* GMRES: same iteration count (+-1), x within 1e-7 relative, residual of the
  GPU x against the oracle's dense A_H2 below the tolerance."""
import numpy as np
import pytest
import scipy.sparse as sps

import h2gen
import oracle
from oracle import krylov as okr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _gpu_ilut(rp, ci, v, tau, p, pool_cap=None):
    from paper_1705_04601_b200 import krylov as kr
    A = kr.CsrMatrix(torch.from_numpy(rp), torch.from_numpy(ci), torch.from_numpy(v))
    return A, kr.IlutFactors(A, tau, p, pool_cap=pool_cap)


def _assert_bitwise(F, ref):
    lrp, lc, lv, urp, uc, uv, d = F.to_csr()
    assert np.array_equal(lrp, ref.l_rowptr) and np.array_equal(lc, ref.l_col)
    assert np.array_equal(urp, ref.u_rowptr) and np.array_equal(uc, ref.u_col)
    assert np.array_equal(lv.view(np.int64), ref.l_val.view(np.int64))
    assert np.array_equal(uv.view(np.int64), ref.u_val.view(np.int64))
    assert np.array_equal(d.view(np.int64), ref.diag.view(np.int64))


CASES = [
    # (nb, bs, seed, density, decay, shift, tau, p)
    (12, 5, 1, 0.3, 2.0, 1.0, 0.0, -1),     # complete LU
    (12, 5, 2, 0.3, 2.0, 1.0, 1e-2, -1),
    (40, 8, 3, 0.15, 3.0, 0.3, 1e-3, -1),
    (40, 8, 4, 0.15, 3.0, 0.3, 1e-2, 5),
    (40, 8, 5, 0.15, 3.0, 0.3, 5e-2, 0),    # p = 0: diagonal U, unit L
    (64, 33, 6, 0.08, 4.0, 0.2, 2e-2, 12),  # rows span several bitmap words, ragged
    (150, 24, 7, 0.05, 6.0, 0.2, 1e-2, 40),  # n = 3600: more rows than warps
    (150, 24, 8, 0.05, 6.0, 0.2, 0.0, -1),   # complete LU with fill
    (160, 64, 11, 0.25, 8.0, 0.2, 1e-2, -1),  # n = 10240, rows spanning several 4096-column gather groups
    (160, 64, 12, 0.25, 8.0, 0.2, 1e-3, 30),
]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]*c[1]}-tau{c[6]}-p{c[7]}" for c in CASES])
def test_ilut_bitwise(case):
    _need_gpu()
    nb, bs, seed, dens, decay, shift, tau, p = case
    rp, ci, v = h2gen.random_sparse(nb, bs, seed, density=dens, decay=decay, shift=shift)
    ref = okr.ilut(rp, ci, v, tau, p)
    _, F = _gpu_ilut(rp, ci, v, tau, p)
    _assert_bitwise(F, ref)


def test_ilut_edge_cases():
    _need_gpu()
    # n = 1
    rp, ci, v = np.array([0, 1], np.int64), np.array([0], np.int32), np.array([3.0])
    _, F = _gpu_ilut(rp, ci, v, 0.1, -1)
    _assert_bitwise(F, okr.ilut(rp, ci, v, 0.1, -1))
    # diagonal matrix: no L / U entries
    n = 1000
    rp, ci, v = np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.linspace(1, 2, n)
    _, F = _gpu_ilut(rp, ci, v, 0.0, -1)
    _assert_bitwise(F, okr.ilut(rp, ci, v, 0.0, -1))
    # lower bidiagonal with a long dependency chain (every row waits on the previous)
    n = 5000
    A = sps.diags([np.full(n, 2.0), np.full(n - 1, -1.0)], [0, -1]).tocsr()
    A.sort_indices()
    args = (A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.astype(np.float64))
    _, F = _gpu_ilut(*args, 0.0, -1)
    _assert_bitwise(F, okr.ilut(*args, 0.0, -1))


def test_ilut_pool_retry_and_zero_pivot():
    _need_gpu()
    from paper_1705_04601_b200 import H2spError
    rp, ci, v = h2gen.random_sparse(30, 8, 9, density=0.2)
    ref = okr.ilut(rp, ci, v, 0.0, -1)
    _, F = _gpu_ilut(rp, ci, v, 0.0, -1, pool_cap=64)   # far too small: ENOMEM, retried larger
    _assert_bitwise(F, ref)
    # zero pivot: a_00 = 0
    A = np.array([[0.0, 1.0], [1.0, 2.0]])
    S = sps.csr_matrix(A)
    with pytest.raises(H2spError, match="zero pivot at row 0"):
        _gpu_ilut(S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data, 0.0, -1)


def test_ilut_on_S_repeatable():
    """ILUT of a real S (Example mat1, N = 8192, the GPU's S; rows ~6000 wide,
    several gather groups): bitwise the same factors on two runs, and every
    factor row sorted, inside [0, n), L strictly lower, U strictly upper."""
    _need_gpu()
    from paper_1705_04601_b200 import krylov as kr
    sp = _sparsify_gpu(h2gen.make_ifmm(8192, 1e-2, 64, 8))
    S = kr.CsrMatrix.from_sparsifier(sp)
    F1 = kr.IlutFactors(S, 1e-3, -1)
    F2 = kr.IlutFactors(S, 1e-3, -1)
    a, b = F1.to_csr(), F2.to_csr()
    for u, v in zip(a, b):
        assert np.array_equal(np.asarray(u).view(np.uint8), np.asarray(v).view(np.uint8))
    lrp, lc, _, urp, uc, _, d = a
    rows_l = np.repeat(np.arange(F1.n), np.diff(lrp))
    rows_u = np.repeat(np.arange(F1.n), np.diff(urp))
    assert np.all(lc < rows_l) and np.all(lc >= 0) and np.all(uc > rows_u) and np.all(uc < F1.n)
    for rp_, c_ in ((lrp, lc), (urp, uc)):
        same = np.repeat(np.diff(rp_) > 0, np.diff(rp_))
        inc = np.diff(c_.astype(np.int64)) > 0
        brk = np.zeros(len(c_), bool)
        brk[rp_[:-1][np.diff(rp_) > 0]] = True
        assert np.all(inc | brk[1:])
    assert np.all(d != 0)


def test_ilu_solve_and_spmv():
    _need_gpu()
    rp, ci, v = h2gen.random_sparse(100, 20, 10, density=0.06, decay=5.0, shift=0.3)
    ref = okr.ilut(rp, ci, v, 1e-2, 20)
    A, F = _gpu_ilut(rp, ci, v, 1e-2, 20)
    b = np.random.default_rng(1).standard_normal(F.n)
    xg = F.solve(torch.from_numpy(b).cuda()).cpu().numpy()
    xo = okr.ilu_solve(ref, b)
    assert np.linalg.norm(xg - xo) <= 1e-12 * np.linalg.norm(xo)
    # in place (x aliases b)
    bt = torch.from_numpy(b).cuda()
    F.solve(bt, bt)
    assert np.linalg.norm(bt.cpu().numpy() - xo) <= 1e-12 * np.linalg.norm(xo)
    y = A.matvec(torch.from_numpy(b).cuda()).cpu().numpy()
    yo = sps.csr_matrix((v, ci, rp)) @ b
    assert np.linalg.norm(y - yo) <= 1e-13 * np.linalg.norm(yo)


def _sparsify_gpu(h):
    import paper_1705_04601_b200 as h2sp
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed)
    sp = h2sp.Sparsifier(plan, packed)
    sp.build()
    torch.cuda.synchronize()
    return sp


@pytest.mark.parametrize("d,tau", [(1e-3, 2e-2), (1e-2, 1e-2)])
def test_gmres_preconditioned_by_sparsified_ilut(d, tau):
    """The paper's experiment at N = 8192: GMRES on the
    operator H^2 (rank 32) preconditioned by ILUT(tau) of the sparsified rank-8
    H^2 of the same matrix (Example mat1, 3-D)."""
    _need_gpu()
    from paper_1705_04601_b200 import krylov as kr
    N, B = 8192, 64
    hop = h2gen.make_ifmm(N, d, B, 32)
    hpre = h2gen.make_ifmm(N, d, B, 8)
    b = np.random.default_rng(7).standard_normal(N)
    # oracle
    rop, rpre = oracle.sparsify(hop), oracle.sparsify(hpre)
    rp, ci, v = oracle.s_csr(rop)
    Sop = sps.csr_matrix((v, ci, rp), shape=(N, N))
    rp2, ci2, v2 = oracle.s_csr(rpre)
    Fo = okr.ilut(rp2, ci2, v2, tau, -1)

    def mv(x):
        return oracle.apply_V(rop, Sop @ oracle.apply_Ut(rop, x[:, None])[:, 0][:, None], side="row")[:, 0]

    def pc(z):
        return oracle.apply_V(rpre, okr.ilu_solve(Fo, oracle.apply_Ut(rpre, z[:, None])[:, 0])[:, None],
                              side="row")[:, 0]

    ro = okr.gmres(mv, b, precond=pc, restart=30, tol=1e-10, maxiter=300)
    assert ro.converged
    # GPU
    spo, spp = _sparsify_gpu(hop), _sparsify_gpu(hpre)
    F = kr.IlutFactors(kr.CsrMatrix.from_sparsifier(spp), tau, -1)
    x, info = kr.gmres(spo, torch.from_numpy(b).cuda(), M=spp, F=F, restart=30, tol=1e-10, maxiter=300)
    x = x.cpu().numpy()
    assert info.converged
    assert abs(info.iters - ro.iters) <= 1, (info.iters, ro.iters)
    assert np.linalg.norm(x - ro.x) <= 1e-7 * np.linalg.norm(ro.x)
    n_cmp = min(len(info.history), len(ro.history)) - 1
    h_g, h_o = np.array(info.history[:n_cmp]), np.array(ro.history[:n_cmp])
    assert np.all(np.abs(h_g - h_o) <= 1e-6 * h_o + 1e-12)
    # against the dense H^2 matrix (oracle.dense): the residual meets the tolerance
    A = oracle.dense_A(hop)
    assert np.linalg.norm(A @ x - b) <= 2e-10 * np.linalg.norm(b)
    # the preconditioner helps: unpreconditioned GMRES needs more steps
    _, info0 = kr.gmres(spo, torch.from_numpy(b).cuda(), restart=30, tol=1e-10, maxiter=300)
    assert info0.iters > info.iters


def test_direct_solve_complete_lu():
    """§8(f) #1: x = V S^-1 U^T b with S^-1 from the device complete LU (ILUT at
    tau = 0, p < 0) of the GPU S, config-2 recipe at N = 4096: the solution
    against numpy's dense solve of the oracle's dense A_H2, and L U = S on the
    factors (the oracle's complete LU of its own S has the same nonzero count)."""
    _need_gpu()
    from paper_1705_04601_b200 import krylov as kr
    from paper_1705_04601_b200 import solve as sv
    h = h2gen.make_config(2, N=4096)
    sp = _sparsify_gpu(h)
    b = np.random.default_rng(3).standard_normal(4096)
    fac = sv.factor_lu(sp)
    x = sv.solve_lu(sp, fac, torch.from_numpy(b).cuda()).cpu().numpy()
    A = oracle.dense_A(h)
    xd = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xd) <= 1e-9 * np.linalg.norm(xd)
    assert np.linalg.norm(A @ x - b) <= 1e-10 * np.linalg.norm(b)
    lrp, lc, lv, urp, uc, uv, d = fac.to_csr()
    n = fac.n
    L = sps.csr_matrix((lv, lc, lrp), shape=(n, n)) + sps.identity(n)
    U = sps.csr_matrix((uv, uc, urp), shape=(n, n)) + sps.diags(d)
    S = kr.CsrMatrix.from_sparsifier(sp)
    Sd = sps.csr_matrix((S.val.cpu().numpy()[:S.col.numel()], S.col.cpu().numpy(), S.rowptr.cpu().numpy()),
                        shape=(n, n))
    assert abs(L @ U - Sd).max() <= 1e-12 * abs(Sd).max()
    rp, ci, v = oracle.s_csr(oracle.sparsify(h))
    ref = okr.ilut(rp, ci, v, 0.0, -1)
    assert abs(fac.nnz - (len(ref.l_col) + len(ref.u_col) + n)) <= 1e-4 * fac.nnz
