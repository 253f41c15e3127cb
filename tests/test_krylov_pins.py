"""Pins of the preconditioning oracle (oracle/krylov.py, oracle/ilut.c;
SURVEY §8(f) #3) against things other than itself: LAPACK's LU,
a hand-worked example, closed forms and properties of GMRES."""
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sps

import h2gen
from oracle import krylov

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ilut_3x3.txt")


def _csr(A):
    S = sps.csr_matrix(A)
    S.sort_indices()
    return S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data.astype(np.float64)


def test_exact_lu_at_tau_zero():
    """tau = 0, no fill limit: ILUT is the complete LU without pivoting; on a
    diagonally dominant matrix LAPACK's partial pivoting exchanges no rows, so
    its L, U are the same factors."""
    rp, ci, v = h2gen.random_sparse(12, 5, seed=3, density=0.3)
    A = sps.csr_matrix((v, ci, rp)).toarray()
    F = krylov.ilut(rp, ci, v, tau=0.0)
    L, U = F.dense()
    P, Lr, Ur = sla.lu(A)
    assert np.array_equal(P, np.eye(len(A)))
    assert np.abs(L - Lr).max() <= 1e-12
    assert np.abs(U - Ur).max() <= 1e-12 * np.abs(Ur).max()


def test_hand_worked_3x3():
    A = np.zeros((3, 3))
    Lg, Ug = np.eye(3), np.zeros((3, 3))
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        t, i, j, x = line.split()
        {"A": A, "L": Lg, "U": Ug}[t][int(i), int(j)] = float(x)
    F = krylov.ilut(*_csr(A), tau=0.05)
    L, U = F.dense()
    assert np.array_equal(L, Lg) and np.array_equal(U, Ug)
    # the dropped fill (1, 2) and the dropped l_20 are not stored at all
    assert F.u_rowptr[2] - F.u_rowptr[1] == 0 and F.l_rowptr[3] - F.l_rowptr[2] == 0


def test_tridiagonal_closed_form():
    """[-1, 2, -1]: no fill, so any small tau gives the exact factors
    u_ii = (i + 2) / (i + 1), l_{i,i-1} = -i / (i + 1) (0-based), u_{i,i+1} = -1."""
    n = 40
    A = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    F = krylov.ilut(*_csr(A), tau=1e-3)
    i = np.arange(n)
    assert np.allclose(F.diag, (i + 2) / (i + 1), rtol=1e-14, atol=0)
    assert np.array_equal(F.l_col, i[1:] - 1)
    assert np.allclose(F.l_val, -i[1:] / (i[1:] + 1), rtol=1e-14, atol=0)
    assert np.array_equal(F.u_col, i[1:]) and np.all(F.u_val == -1.0)


def test_huge_tau_is_jacobi():
    rp, ci, v = h2gen.random_sparse(8, 4, seed=4, density=0.5)
    A = sps.csr_matrix((v, ci, rp)).toarray()
    F = krylov.ilut(rp, ci, v, tau=1e3)
    assert len(F.l_col) == 0 and len(F.u_col) == 0
    assert np.array_equal(F.diag, np.diag(A))


def test_p_largest_with_ties():
    """Row 0 of an upper-arrow matrix: off-diagonals 1, 3, 2, 3 at columns 1..4.
    p = 2 keeps both 3s; p = 1 keeps the 3 of the smaller column (reading 25);
    p = 3 adds the 2; the diagonal is always kept."""
    n = 5
    A = 10 * np.eye(n)
    A[0, 1:] = [1, 3, 2, 3]
    for p, cols in ((1, [2]), (2, [2, 4]), (3, [2, 3, 4]), (-1, [1, 2, 3, 4])):
        F = krylov.ilut(*_csr(A), tau=0.0, p=p)
        assert list(F.u_col[F.u_rowptr[0]:F.u_rowptr[1]]) == cols
        assert F.diag[0] == 10.0


def test_dropping_reduces_to_lu_of_kept_pattern():
    """Rows without any dropped entry are exact rows of L U = A: for each row
    i, (L U)_i* = a_i* wherever no entry of row i (of L or U) was dropped; with
    every |entry| far above tau the whole factorisation is exact."""
    A = 8 * np.eye(6) + np.ones((6, 6))
    F = krylov.ilut(*_csr(A), tau=1e-6)
    L, U = F.dense()
    assert np.abs(L @ U - A).max() <= 1e-13 * np.abs(A).max()


def test_ilu_solve_is_inverse_of_lu():
    rp, ci, v = h2gen.random_sparse(10, 6, seed=5, density=0.3)
    F = krylov.ilut(rp, ci, v, tau=1e-2, p=8)
    L, U = F.dense()
    b = np.random.default_rng(0).standard_normal(F.n)
    x = krylov.ilu_solve(F, b)
    assert np.abs(L @ (U @ x) - b).max() <= 1e-12 * np.abs(b).max()


def test_gmres_distinct_eigenvalues():
    """A diagonalisable A with k distinct eigenvalues: the Krylov space has
    dimension <= k, so GMRES terminates (to rounding) in <= k steps."""
    rng = np.random.default_rng(1)
    lam = np.repeat([1.0, 2.0, 3.5, 5.0, 8.0], 12)
    Qm, _ = np.linalg.qr(rng.standard_normal((60, 60)))
    A = Qm @ np.diag(lam) @ Qm.T
    b = rng.standard_normal(60)
    r = krylov.gmres(lambda x: A @ x, b, restart=30, tol=1e-12)
    assert r.converged and r.iters <= 5


def test_gmres_matches_direct_solve_and_is_monotone():
    rng = np.random.default_rng(2)
    A = np.eye(80) * 4 + rng.standard_normal((80, 80)) / 4
    b = rng.standard_normal(80)
    r = krylov.gmres(lambda x: A @ x, b, restart=10, tol=1e-12, maxiter=400)
    assert r.converged
    x = np.linalg.solve(A, b)
    assert np.linalg.norm(r.x - x) <= 1e-10 * np.linalg.norm(x)
    h = np.array(r.history)
    assert np.all(np.diff(h[:11]) <= 1e-15)   # minimal residual within a cycle


def test_gmres_exact_preconditioner_one_step():
    rng = np.random.default_rng(3)
    A = np.eye(50) * 3 + rng.standard_normal((50, 50)) / 5
    b = rng.standard_normal(50)
    Ainv = np.linalg.inv(A)
    r = krylov.gmres(lambda x: A @ x, b, precond=lambda v: Ainv @ v, tol=1e-10)
    assert r.converged and r.iters == 1
    assert np.linalg.norm(A @ r.x - b) <= 1e-10 * np.linalg.norm(b)


def test_gmres_ilut_preconditioned_sparse():
    """ILUT as the right preconditioner of a sparse system: fewer iterations
    than without, same solution."""
    rp, ci, v = h2gen.random_sparse(30, 8, seed=6, density=0.15, shift=0.3)
    A = sps.csr_matrix((v, ci, rp))
    b = np.random.default_rng(4).standard_normal(A.shape[0])
    F = krylov.ilut(rp, ci, v, tau=1e-2)
    r0 = krylov.gmres(lambda x: A @ x, b, tol=1e-10, maxiter=2000)
    r1 = krylov.gmres(lambda x: A @ x, b, precond=lambda z: krylov.ilu_solve(F, z), tol=1e-10)
    assert r0.converged and r1.converged and r1.iters < r0.iters
    x = sps.linalg.spsolve(A.tocsc(), b)
    assert np.linalg.norm(r1.x - x) <= 1e-8 * np.linalg.norm(x)
