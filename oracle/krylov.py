"""CPU oracle of the paper's preconditioning workload (
"Sparsification method as a preconditioner"): ILUt of S
(``oracle/ilut.c``, plain C, Saad's ILUT(tau, p), reading 25) and
restarted GMRES with right preconditioning (plain numpy, Saad's Algorithm 9.5
with modified Gram-Schmidt Arnoldi and Givens rotations).

TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT PATH (see oracle/__init__.py).

Pins (tests/test_krylov_pins.py, ``-m "not gpu"``): exact LU at tau = 0
(LAPACK getrf, no row exchanges), a hand-computed 3 x 3 dropping example
(tests/golden/ilut_3x3.txt), the closed-form LU of the [-1, 2, -1]
tridiagonal, Jacobi at a huge tau, the p-largest rule with ties; GMRES: the
number of distinct eigenvalues bounds the iterations, numpy.linalg.solve,
exact preconditioner -> one iteration, monotone residuals.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Callable, List, Optional

import numpy as np

_lib = None


def _load():
    global _lib
    if _lib is None:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libilut.so")
        _lib = ctypes.CDLL(path)
        _lib.oracle_ilut.restype = ctypes.c_int
        _lib.oracle_ilut.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 3 + [ctypes.c_double, ctypes.c_int] + \
            [ctypes.c_void_p] * 3 + [ctypes.c_int64] + [ctypes.c_void_p] * 3 + [ctypes.c_int64] + [ctypes.c_void_p] * 2
        _lib.oracle_ilu_solve.restype = None
        _lib.oracle_ilu_solve.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 9
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class IlutFactors:
    """L strict lower (unit diagonal implied) and U strict upper in CSR with
    ascending columns, and diag = u_ii."""
    n: int
    l_rowptr: np.ndarray
    l_col: np.ndarray
    l_val: np.ndarray
    u_rowptr: np.ndarray
    u_col: np.ndarray
    u_val: np.ndarray
    diag: np.ndarray

    def dense(self):
        n = self.n
        L = np.eye(n)
        U = np.diag(self.diag.copy())
        for i in range(n):
            a, b = self.l_rowptr[i], self.l_rowptr[i + 1]
            L[i, self.l_col[a:b]] = self.l_val[a:b]
            a, b = self.u_rowptr[i], self.u_rowptr[i + 1]
            U[i, self.u_col[a:b]] = self.u_val[a:b]
        return L, U


def ilut(rowptr, col, val, tau: float, p: int = -1, cap: Optional[int] = None) -> IlutFactors:
    """ILUT(tau, p) of the CSR matrix (rowptr int64, col int32 ascending, val
    float64); p < 0 keeps every entry that survives the tau rule."""
    lib = _load()
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    n = len(rowptr) - 1
    cap = cap or max(16, 2 * len(col))
    while True:
        lrp = np.zeros(n + 1, np.int64)
        urp = np.zeros(n + 1, np.int64)
        lci = np.zeros(cap, np.int32)
        uci = np.zeros(cap, np.int32)
        lv = np.zeros(cap)
        uv = np.zeros(cap)
        diag = np.zeros(n)
        bad = np.zeros(1, np.int64)
        rc = lib.oracle_ilut(n, _p(rowptr), _p(col), _p(val), float(tau), int(p), _p(lrp), _p(lci), _p(lv), cap,
                             _p(urp), _p(uci), _p(uv), cap, _p(diag), _p(bad))
        if rc == 1:
            cap *= 2
            continue
        if rc == 2:
            raise ZeroDivisionError(f"ILUT: zero pivot at row {int(bad[0])}")
        nl, nu = int(lrp[n]), int(urp[n])
        return IlutFactors(n, lrp, lci[:nl].copy(), lv[:nl].copy(), urp, uci[:nu].copy(), uv[:nu].copy(), diag)


def ilu_solve(F: IlutFactors, b: np.ndarray) -> np.ndarray:
    """x = (L U)^{-1} b by forward then backward substitution."""
    lib = _load()
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(F.n)
    lib.oracle_ilu_solve(F.n, _p(F.l_rowptr), _p(F.l_col), _p(F.l_val), _p(F.u_rowptr), _p(F.u_col), _p(F.u_val),
                         _p(F.diag), _p(b), _p(x))
    return x


@dataclass
class GmresResult:
    x: np.ndarray
    iters: int                 # Arnoldi steps in total (over all restarts)
    history: List[float]       # ||r_j|| / ||b||: [1.0, estimate after step 1, ...]
    converged: bool


def gmres(matvec: Callable[[np.ndarray], np.ndarray], b: np.ndarray,
          precond: Optional[Callable[[np.ndarray], np.ndarray]] = None, restart: int = 30, tol: float = 1e-10,
          maxiter: int = 500) -> GmresResult:
    """Restarted GMRES(m) with right preconditioning (Saad, Algorithm 9.5):
    solves A x = b as A M^{-1} u = b, x = M^{-1} u, from x0 = 0.  Arnoldi by
    modified Gram-Schmidt; the least-squares problem min ||beta e1 - H y|| is
    reduced by Givens rotations, whose last component |g_{j+1}| is the residual
    norm of step j.  Stops when |g_{j+1}| <= tol ||b|| (or maxiter steps)."""
    M = precond or (lambda v: v)
    n = len(b)
    x = np.zeros(n)
    bnorm = float(np.linalg.norm(b))
    hist = [1.0]
    it = 0
    converged = False
    if bnorm == 0.0:
        return GmresResult(x, 0, hist, True)
    while it < maxiter and not converged:
        r = b - matvec(x)
        beta = float(np.linalg.norm(r))
        if beta <= tol * bnorm:
            converged = True
            break
        m = restart
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        j_done = 0
        for j in range(m):
            w = matvec(M(V[j]))
            for i in range(j + 1):            # modified Gram-Schmidt
                H[i, j] = np.dot(w, V[i])
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] != 0.0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):                # previous rotations on column j
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / den
            sn[j] = H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            it += 1
            j_done = j + 1
            hist.append(abs(g[j + 1]) / bnorm)
            if abs(g[j + 1]) <= tol * bnorm or it >= maxiter:
                break
        k = j_done
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):        # back substitution H[:k, :k] y = g[:k]
            y[i] = (g[i] - np.dot(H[i, i + 1:k], y[i + 1:k])) / H[i, i]
        x = x + M(V[:k].T @ y)
        if abs(g[k]) <= tol * bnorm:
            converged = True
    return GmresResult(x, it, hist, converged)
