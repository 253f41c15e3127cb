"""Binding of the preconditioning workload and of
the direct solve's factorisation (§8(f) #1): ILUT of S, triangular solves,
CSR SpMV and right-preconditioned GMRES, all in ``libh2sp`` (csrc/krylov.cu;
declarations and contracts in include/h2sp.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import H2spError, Sparsifier, _check, _stream_handle, lib

_i32, _i64, _f64, _vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class _Csr(ctypes.Structure):
    _fields_ = [("n", _i64), ("rowptr", _vp), ("col", _vp), ("val", _vp)]


class _Factors(ctypes.Structure):
    _fields_ = [("n", _i64), ("l_start", _vp), ("u_start", _vp), ("l_len", _vp), ("u_len", _vp), ("diag", _vp),
                ("pool_col", _vp), ("pool_val", _vp), ("pool_cap", _i64)]


class _Sparsified(ctypes.Structure):
    _fields_ = [("plan", _vp), ("q", _vp), ("S", _Csr), ("apply_ws", _vp), ("apply_ws_bytes", ctypes.c_size_t)]


class _GmresOpts(ctypes.Structure):
    _fields_ = [("restart", ctypes.c_int), ("maxiter", ctypes.c_int), ("tol", _f64)]


class _GmresInfo(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("restarts", ctypes.c_int), ("converged", ctypes.c_int),
                ("history_len", ctypes.c_int), ("history", ctypes.POINTER(_f64)), ("history_cap", ctypes.c_int)]


lib.h2sp_ilut_ws_bytes.argtypes = [_i64]
lib.h2sp_ilut_ws_bytes.restype = _i64
lib.h2sp_ilut.argtypes = [ctypes.POINTER(_Csr), _f64, ctypes.c_int, ctypes.POINTER(_Factors), _vp, ctypes.c_size_t,
                          ctypes.POINTER(_i64), _vp]
lib.h2sp_ilu_solve_ws_bytes.argtypes = [_i64]
lib.h2sp_ilu_solve_ws_bytes.restype = _i64
lib.h2sp_ilu_solve.argtypes = [ctypes.POINTER(_Factors), _vp, _vp, _vp, ctypes.c_size_t, _vp]
lib.h2sp_csr_spmv.argtypes = [ctypes.POINTER(_Csr), _vp, _vp, _vp]
lib.h2sp_gmres_ws_bytes.argtypes = [_i64, ctypes.c_int]
lib.h2sp_gmres_ws_bytes.restype = _i64
lib.h2sp_gmres.argtypes = [ctypes.POINTER(_Sparsified), ctypes.POINTER(_Sparsified), ctypes.POINTER(_Factors), _vp,
                           _vp, ctypes.POINTER(_GmresOpts), ctypes.POINTER(_GmresInfo), _vp, ctypes.c_size_t, _vp]

H2SP_ENOMEM = 4


def _csr(rowptr, col, val) -> _Csr:
    return _Csr(n=rowptr.numel() - 1, rowptr=rowptr.data_ptr(), col=col.data_ptr(), val=val.data_ptr())


class CsrMatrix:
    """A device CSR matrix (int64 rowptr, int32 col, float64 val)."""

    def __init__(self, rowptr, col, val):
        import torch
        self.rowptr = torch.as_tensor(rowptr).to("cuda", torch.int64).contiguous()
        self.col = torch.as_tensor(col).to("cuda", torch.int32).contiguous()
        self.val = torch.as_tensor(val).to("cuda", torch.float64).contiguous()
        self.n = self.rowptr.numel() - 1
        self.abi = _csr(self.rowptr, self.col, self.val)

    @classmethod
    def from_sparsifier(cls, sp: Sparsifier):
        """S of the last h2sp_build (stored mode), without copying."""
        nnz = int(sp.plan.sizes["s_nnz"])
        m = cls.__new__(cls)
        m.rowptr, m.col, m.val = sp.outputs["s_rowptr"], sp.outputs["s_col"][:max(nnz, 1)], sp.outputs["s_val"]
        m.n = sp.plan.s_rows
        m.abi = _csr(m.rowptr, m.col, m.val)
        return m

    def matvec(self, x, y=None, stream=None):
        import torch
        y = torch.empty_like(x) if y is None else y
        _check(lib.h2sp_csr_spmv(ctypes.byref(self.abi), x.data_ptr(), y.data_ptr(), _stream_handle(stream)),
               "h2sp_csr_spmv")
        return y


class IlutFactors:
    """ILUT(tau, p) factors of a device CSR matrix (h2sp_ilut); tau = 0, p < 0
    gives the complete LU (the direct solve)."""

    def __init__(self, A: CsrMatrix, tau: float, p: int = -1, pool_cap: Optional[int] = None, stream=None):
        import torch
        n = A.n
        self.n, self.tau, self.p = n, float(tau), int(p)
        dev = A.val.device
        self.l_start = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
        self.u_start = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
        self.l_len = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        self.u_len = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        self.diag = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
        nnz = int(A.col.numel())
        if pool_cap:
            cap = int(pool_cap)
        elif p >= 0:
            cap = max(1024, 2 * p * n + n)
        elif tau > 0:   # dropping: start at an eighth of S (grown on H2SP_ENOMEM)
            cap = max(1024, 16 * n, nnz // 8)
        else:           # complete LU: fill
            cap = max(1024, 3 * nnz)
        ws_b = int(lib.h2sp_ilut_ws_bytes(n))
        ws = torch.empty(ws_b + 256, dtype=torch.uint8, device=dev)
        wsp = (ws.data_ptr() + 255) // 256 * 256
        used = _i64(0)
        while True:
            self.pool_col = torch.empty(cap, dtype=torch.int32, device=dev)
            self.pool_val = torch.empty(cap, dtype=torch.float64, device=dev)
            self.abi = _Factors(n=n, l_start=self.l_start.data_ptr(), u_start=self.u_start.data_ptr(),
                                l_len=self.l_len.data_ptr(), u_len=self.u_len.data_ptr(), diag=self.diag.data_ptr(),
                                pool_col=self.pool_col.data_ptr(), pool_val=self.pool_val.data_ptr(), pool_cap=cap)
            st = lib.h2sp_ilut(ctypes.byref(A.abi), self.tau, self.p, ctypes.byref(self.abi), wsp, ws_b,
                               ctypes.byref(used), _stream_handle(stream))
            if st == H2SP_ENOMEM:
                cap = max(2 * cap, 2 * int(used.value))
                del self.pool_col, self.pool_val
                continue
            _check(st, "h2sp_ilut")
            break
        del ws
        self.pool_used = int(used.value)
        sws = int(lib.h2sp_ilu_solve_ws_bytes(n))
        self._sws = torch.empty(sws + 256, dtype=torch.uint8, device=dev)
        self._swsp = (self._sws.data_ptr() + 255) // 256 * 256
        self._swsb = sws

    @property
    def nnz(self) -> int:
        return int(self.l_len.sum().item() + self.u_len.sum().item()) + self.n

    def solve(self, b, x=None, stream=None):
        """x = (L U)^-1 b (device float64 vectors)."""
        import torch
        x = torch.empty_like(b) if x is None else x
        _check(lib.h2sp_ilu_solve(ctypes.byref(self.abi), b.data_ptr(), x.data_ptr(), self._swsp, self._swsb,
                                  _stream_handle(stream)), "h2sp_ilu_solve")
        return x

    def to_csr(self):
        """Host copies as standard CSR (l_rowptr, l_col, l_val, u_rowptr, u_col,
        u_val, diag) -- the pool rows gathered in row order (data movement)."""
        ls, ll = self.l_start.cpu().numpy()[:self.n], self.l_len.cpu().numpy()[:self.n].astype(np.int64)
        us, ul = self.u_start.cpu().numpy()[:self.n], self.u_len.cpu().numpy()[:self.n].astype(np.int64)
        pc, pv = self.pool_col.cpu().numpy(), self.pool_val.cpu().numpy()

        def gather(st, ln):
            rp = np.zeros(self.n + 1, np.int64)
            rp[1:] = np.cumsum(ln)
            idx = np.concatenate([np.arange(s, s + k) for s, k in zip(st, ln)]) if rp[-1] else np.zeros(0, np.int64)
            return rp, pc[idx], pv[idx]

        lrp, lc, lv = gather(ls, ll)
        urp, uc, uv = gather(us, ul)
        return lrp, lc, lv, urp, uc, uv, self.diag.cpu().numpy()[:self.n]


def _sparsified(sp: Sparsifier, S: CsrMatrix) -> _Sparsified:
    ptr, nb = sp.apply_ws(1)
    return _Sparsified(plan=sp.plan.handle, q=sp.outputs["q_row"].data_ptr(), S=S.abi, apply_ws=ptr,
                       apply_ws_bytes=nb)


@dataclass
class GmresInfo:
    iters: int
    restarts: int
    converged: bool
    history: List[float] = field(default_factory=list)


def gmres(A: Sparsifier, b, M: Optional[Sparsifier] = None, F: Optional[IlutFactors] = None, restart: int = 30,
          tol: float = 1e-10, maxiter: int = 500, x=None, stream=None):
    """Solve A_H2 x = b with A_H2 = U S U^T (the sparsified symmetric H^2 matrix
    of ``A``'s last stored-S build) by GMRES(restart), right-preconditioned by
    M^-1 = U_M (L U)^-1 U_M^T (``M``'s sparsification, ``F`` = ILUT of its S);
    b, x in tree order (device float64).  Returns (x, GmresInfo)."""
    import torch
    n = A.plan.s_rows
    x = torch.empty_like(b) if x is None else x
    SA = CsrMatrix.from_sparsifier(A)
    a = _sparsified(A, SA)
    m = None
    if M is not None:
        SM = CsrMatrix.from_sparsifier(M)
        m = _sparsified(M, SM)
    wsb = int(lib.h2sp_gmres_ws_bytes(n, restart))
    ws = torch.empty(wsb + 256, dtype=torch.uint8, device=b.device)
    wsp = (ws.data_ptr() + 255) // 256 * 256
    hist = (_f64 * (maxiter + 2))()
    info = _GmresInfo(history=ctypes.cast(hist, ctypes.POINTER(_f64)), history_cap=maxiter + 2)
    opts = _GmresOpts(restart=restart, maxiter=maxiter, tol=tol)
    _check(lib.h2sp_gmres(ctypes.byref(a), ctypes.byref(m) if m is not None else None,
                          ctypes.byref(F.abi) if F is not None else None, b.data_ptr(), x.data_ptr(),
                          ctypes.byref(opts), ctypes.byref(info), wsp, wsb, _stream_handle(stream)), "h2sp_gmres")
    h = [hist[i] for i in range(min(info.history_len, maxiter + 2))]
    return x, GmresInfo(info.iters, info.restarts, bool(info.converged), h)


__all__ = ["CsrMatrix", "IlutFactors", "GmresInfo", "gmres", "H2spError"]
