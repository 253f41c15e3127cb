"""GPU parity of the supernodal Cholesky of S (the direct
solve x = V S^-1 U^T b, Eq. sp0): L L^T = S (the GPU's S, dense, small
N), the solution against numpy's dense solve of the oracle's A_H2, and against
the device complete LU of the same S."""
import numpy as np
import pytest
import scipy.sparse as sps

import h2gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _sparsify(h):
    import paper_1705_04601_b200 as h2sp
    p = h2gen.pack(h)
    plan = h2sp.Plan(p)
    sp = h2sp.Sparsifier(plan, p)
    sp.build()
    torch.cuda.synchronize()
    return plan, sp


def test_LLt_equals_S_config1():
    _need_gpu()
    from paper_1705_04601_b200 import solve as sv
    h = h2gen.make_config(1)
    plan, sp = _sparsify(h)
    fac = sv.factor_chol(sp)
    L = fac.dense_L(plan)
    nnz = plan.sizes["s_nnz"]
    S = sps.csr_matrix((sp.outputs["s_val"][:nnz].cpu().numpy(), sp.outputs["s_col"][:nnz].cpu().numpy(),
                        sp.outputs["s_rowptr"].cpu().numpy()), shape=(h.N, h.N)).toarray()
    assert np.allclose(L, np.tril(L), atol=0, rtol=0)
    assert np.all(np.diag(L) > 0)
    assert np.abs(L @ L.T - S).max() <= 1e-12 * np.abs(S).max()
    # the factor's pattern is struct's: L = chol(S) of numpy (same unique factor)
    Lr = np.linalg.cholesky(S)
    assert np.abs(L - Lr).max() <= 1e-10 * np.abs(Lr).max()


CASES = [("cfg1", lambda: h2gen.make_config(1)),
         ("cfg2-4096", lambda: h2gen.make_config(2, N=4096)),
         ("cfg3-4096", lambda: h2gen.make_config(3, N=4096)),
         ("cfg5-8192", lambda: h2gen.make_config(5, N=8192)),
         ("cfg2-16384", lambda: h2gen.make_config(2, N=16384))]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_direct_solve_chol(name, make):
    _need_gpu()
    from paper_1705_04601_b200 import solve as sv
    h = make()
    plan, sp = _sparsify(h)
    fac = sv.factor_chol(sp)
    b = np.random.default_rng(5).standard_normal(h.N)
    x = sv.solve_chol(sp, fac, torch.from_numpy(b).cuda()).cpu().numpy()
    if h.N <= 8192:
        A = oracle.dense_A(h)
        xd = np.linalg.solve(A, b)
        cond = np.linalg.cond(A)
        assert np.linalg.norm(x - xd) <= 1e-13 * cond * np.linalg.norm(xd)
    else:   # the oracle's H^2 matvec (no dense A)
        cond = 1e6
    assert np.linalg.norm(oracle.h2_matvec(h, x) - b) <= 1e-11 * np.linalg.norm(b)
    # same S, the device complete LU (h2sp_ilut at tau = 0)
    lu = sv.factor_lu(sp)
    x2 = sv.solve_lu(sp, lu, torch.from_numpy(b).cuda()).cpu().numpy()
    assert np.linalg.norm(x - x2) <= 1e-13 * cond * np.linalg.norm(x2)
    # repeatable
    x3 = sv.solve_chol(sp, sv.factor_chol(sp), torch.from_numpy(b).cuda()).cpu().numpy()
    assert np.array_equal(x, x3)
