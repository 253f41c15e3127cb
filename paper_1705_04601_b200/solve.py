"""Direct solve through the factorisation, x = V S^-1 U^T b (Eq. sp0, P:45-49;
SURVEY §8(f) next #1), on the device.

S is symmetric positive definite when A_H2 is (Proposition) and its
rows are in level-major frozen order: the leaves' frozen unknowns first, each
level's after the levels below, so the upper levels play the separators of a
nested dissection and S is factorised in its own order (no reordering).  The
sparse Cholesky is cuSOLVER's device low-level API (symbolic analysis, numeric
factorisation, triangular solves) -- a library call, like cuBLAS, outside the
sparsification hot path; the applies U^T b and V y are this package's kernels.
"""
import ctypes
import ctypes.util

import torch

from . import Sparsifier

_solver = None
_sparse = None


def _libs():
    global _solver, _sparse
    if _solver is None:
        for name in ("libcusolver.so.11", "libcusolver.so"):
            try:
                _solver = ctypes.CDLL(name)
                break
            except OSError:
                continue
        for name in ("libcusparse.so.12", "libcusparse.so"):
            try:
                _sparse = ctypes.CDLL(name)
                break
            except OSError:
                continue
        if _solver is None or _sparse is None:
            raise RuntimeError("cuSOLVER / cuSPARSE shared libraries not found")
    return _solver, _sparse


def _ck(st, what):
    if st != 0:
        raise RuntimeError(f"{what} failed with status {st}")


class SparseCholesky:
    """S = L L^T of a CSR matrix on the device (int64 row pointers, int32
    columns, float64 values, all CUDA tensors; full symmetric storage)."""

    def __init__(self, rowptr, col, val, n, stream=None):
        sv, sp = _libs()
        vp = ctypes.c_void_p
        self.n = int(n)
        self.nnz = int(col.numel())
        if self.nnz >= 2 ** 31:
            raise ValueError("cuSOLVER sparse Cholesky takes int32 indices (nnz < 2^31)")
        self.rp = rowptr.to(torch.int32).contiguous()
        self.col = col.contiguous()
        self.val = val.contiguous()
        self.handle = vp()
        _ck(sv.cusolverSpCreate(ctypes.byref(self.handle)), "cusolverSpCreate")
        st = stream if stream is not None else torch.cuda.current_stream()
        _ck(sv.cusolverSpSetStream(self.handle, vp(st.cuda_stream)), "cusolverSpSetStream")
        self.descr = vp()
        _ck(sp.cusparseCreateMatDescr(ctypes.byref(self.descr)), "cusparseCreateMatDescr")
        self.info = vp()
        _ck(sv.cusolverSpCreateCsrcholInfo(ctypes.byref(self.info)), "cusolverSpCreateCsrcholInfo")
        n_, nnz_ = ctypes.c_int(self.n), ctypes.c_int(self.nnz)
        _ck(sv.cusolverSpXcsrcholAnalysis(self.handle, n_, nnz_, self.descr, vp(self.rp.data_ptr()),
                                          vp(self.col.data_ptr()), self.info), "cusolverSpXcsrcholAnalysis")
        internal, work = ctypes.c_size_t(), ctypes.c_size_t()
        _ck(sv.cusolverSpDcsrcholBufferInfo(self.handle, n_, nnz_, self.descr, vp(self.val.data_ptr()),
                                            vp(self.rp.data_ptr()), vp(self.col.data_ptr()), self.info,
                                            ctypes.byref(internal), ctypes.byref(work)),
            "cusolverSpDcsrcholBufferInfo")
        self.internal_bytes = int(internal.value)
        self.buffer = torch.empty(max(1, int(work.value)), dtype=torch.uint8, device=val.device)
        _ck(sv.cusolverSpDcsrcholFactor(self.handle, n_, nnz_, self.descr, vp(self.val.data_ptr()),
                                        vp(self.rp.data_ptr()), vp(self.col.data_ptr()), self.info,
                                        vp(self.buffer.data_ptr())), "cusolverSpDcsrcholFactor")
        pos = ctypes.c_int(-1)
        _ck(sv.cusolverSpDcsrcholZeroPivot(self.handle, self.info, ctypes.c_double(0.0), ctypes.byref(pos)),
            "cusolverSpDcsrcholZeroPivot")
        if pos.value >= 0:
            raise RuntimeError(f"S is not positive definite (zero pivot at row {pos.value})")

    def solve(self, b, x=None):
        """x = S^-1 b for one right-hand side (CUDA float64 vectors of length n)."""
        sv, _ = _libs()
        b = b.contiguous()
        x = torch.empty_like(b) if x is None else x
        _ck(sv.cusolverSpDcsrcholSolve(self.handle, ctypes.c_int(self.n), ctypes.c_void_p(b.data_ptr()),
                                       ctypes.c_void_p(x.data_ptr()), self.info, ctypes.c_void_p(self.buffer.data_ptr())),
            "cusolverSpDcsrcholSolve")
        return x

    def __del__(self):
        try:
            sv, sp = _libs()
            sv.cusolverSpDestroyCsrcholInfo(self.info)
            sp.cusparseDestroyMatDescr(self.descr)
            sv.cusolverSpDestroy(self.handle)
        except Exception:
            pass


def metis_order(rowptr, col, n):
    """Fill-reducing symmetric order of the pattern (cuSOLVER's host METIS nested
    dissection); returns the permutation p (new row i = old row p[i]) as int64."""
    import numpy as np
    sv, sp_ = _libs()
    rp = np.ascontiguousarray(rowptr.cpu().numpy().astype(np.int32))
    cl = np.ascontiguousarray(col.cpu().numpy().astype(np.int32))
    perm = np.empty(n, dtype=np.int32)
    h, d = ctypes.c_void_p(), ctypes.c_void_p()
    _ck(sv.cusolverSpCreate(ctypes.byref(h)), "cusolverSpCreate")
    _ck(sp_.cusparseCreateMatDescr(ctypes.byref(d)), "cusparseCreateMatDescr")
    try:
        _ck(sv.cusolverSpXcsrmetisndHost(h, ctypes.c_int(n), ctypes.c_int(cl.size), d,
                                         rp.ctypes.data_as(ctypes.c_void_p), cl.ctypes.data_as(ctypes.c_void_p),
                                         None, perm.ctypes.data_as(ctypes.c_void_p)), "cusolverSpXcsrmetisndHost")
    finally:
        sp_.cusparseDestroyMatDescr(d)
        sv.cusolverSpDestroy(h)
    return perm.astype(np.int64)


class OrderedCholesky:
    """P^T S P = L L^T with a fill-reducing permutation P (METIS); solve
    permutes the right-hand side in and the solution back out on the device."""

    def __init__(self, rowptr, col, val, n):
        import numpy as np
        import scipy.sparse as sps
        self.n = int(n)
        perm = metis_order(rowptr, col, self.n)
        S = sps.csr_matrix((val.cpu().numpy(), col.cpu().numpy(), rowptr.cpu().numpy()), shape=(self.n, self.n))
        Sp = S[perm][:, perm].tocsr()
        Sp.sort_indices()
        dev = val.device
        self.p = torch.from_numpy(perm).to(dev)
        self.chol = SparseCholesky(torch.from_numpy(Sp.indptr.astype(np.int64)).to(dev),
                                   torch.from_numpy(Sp.indices.astype(np.int32)).to(dev),
                                   torch.from_numpy(Sp.data).to(dev), self.n)
        self.internal_bytes = self.chol.internal_bytes

    def solve(self, b, x=None):
        zp = self.chol.solve(b[self.p].contiguous())
        x = torch.empty_like(b) if x is None else x
        x[self.p] = zp
        return x


def factor(sp: Sparsifier, plan, order: str = "s"):
    """Cholesky of the S the last build wrote into sp.outputs (symmetric plans).
    order="s": S's own level-major order; "metis": fill-reducing (host METIS)."""
    if not plan.symmetric:
        raise ValueError("the sparse Cholesky needs a symmetric (SPD) plan")
    nnz = plan.sizes["s_nnz"]
    args = (sp.outputs["s_rowptr"], sp.outputs["s_col"][:nnz], sp.outputs["s_val"][:nnz], plan.s_rows)
    return OrderedCholesky(*args) if order == "metis" else SparseCholesky(*args)


def solve(sp: Sparsifier, chol, b):
    """x = V S^-1 U^T b (Eq. sp0) for one right-hand side b (CUDA float64, length N)."""
    bt = b.reshape(1, -1).contiguous()
    y = torch.empty_like(bt)
    sp.apply_Ut(bt, y)
    z = chol.solve(y[0]).reshape(1, -1)
    x = torch.empty_like(bt)
    sp.apply_V(z, x)
    return x[0]


def factor_lu(sp: Sparsifier, stream=None):
    """The complete LU of the S the last build wrote (h2sp_ilut at tau = 0,
    p < 0: this package's sync-free row-by-row factorisation in S's own
    level-major order, no library call).  Works for symmetric (SPD S,
    Proposition) and general plans with nonzero pivots."""
    from .krylov import CsrMatrix, IlutFactors
    return IlutFactors(CsrMatrix.from_sparsifier(sp), 0.0, -1, stream=stream)


def solve_lu(sp: Sparsifier, fac, b, stream=None):
    """x = V (L U)^-1 U^T b (Eq. sp0) with the device LU of factor_lu;
    b tree order (CUDA float64, length N)."""
    bt = b.reshape(1, -1).contiguous()
    y = torch.empty_like(bt)
    sp.apply_Ut(bt, y, stream=stream)
    fac.solve(y[0], y[0], stream=stream)
    x = torch.empty_like(bt)
    sp.apply_V(y, x, stream=stream)
    return x[0]


# ---------------------------------------------------------------------------
# Supernodal Cholesky (libh2sp, csrc/chol.cu; include/h2sp.h h2sp_chol_*)
# ---------------------------------------------------------------------------
from . import _check, _stream_handle, lib  # noqa: E402

_vp, _i32, _i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
lib.h2sp_chol_analyse.argtypes = [_vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
lib.h2sp_chol_info.argtypes = [_vp, ctypes.POINTER(_i32), _vp, _vp, ctypes.POINTER(ctypes.c_double)]
lib.h2sp_chol_struct.argtypes = [_vp, _i32, _vp, _i32, ctypes.POINTER(_i32)]
lib.h2sp_chol_supernodes.argtypes = [_vp, _vp]
lib.h2sp_chol_upload.argtypes = [_vp, _vp, ctypes.c_size_t, _vp]
lib.h2sp_chol_factor.argtypes = [_vp, _vp, _vp, _vp, _vp]
lib.h2sp_chol_solve.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
lib.h2sp_chol_destroy.argtypes = [_vp]
lib.h2sp_chol_destroy.restype = None


class CholAnalysis:
    """Host analysis of S's supernodal Cholesky (h2sp_chol_analyse): the block
    elimination tree and struct(J) of every supernode (= row group of S)."""

    def __init__(self, plan, amalgamate: int = 0):
        import numpy as np
        self.handle = _vp()
        pd, mb = _i64(), _i64()
        _check(lib.h2sp_chol_analyse(plan.handle, amalgamate, ctypes.byref(self.handle), ctypes.byref(pd),
                                     ctypes.byref(mb)), "h2sp_chol_analyse")
        self.panel_doubles, self.meta_bytes = int(pd.value), int(mb.value)
        ns = _i32()
        fl = ctypes.c_double()
        _check(lib.h2sp_chol_info(self.handle, ctypes.byref(ns), None, None, ctypes.byref(fl)), "h2sp_chol_info")
        self.ns, self.flops = int(ns.value), float(fl.value)
        self.parent = np.zeros(self.ns, np.int32)
        self.panel_rows = np.zeros(self.ns, np.int64)
        _check(lib.h2sp_chol_info(self.handle, None, self.parent.ctypes.data, self.panel_rows.ctypes.data, None),
               "h2sp_chol_info")
        st = np.zeros(self.ns + 1, np.int64)
        _check(lib.h2sp_chol_supernodes(self.handle, st.ctypes.data), "h2sp_chol_supernodes")
        self.starts, self.sizes = st[:-1], np.diff(st)

    def struct(self, J: int):
        import numpy as np
        cnt = _i32()
        _check(lib.h2sp_chol_struct(self.handle, J, None, 0, ctypes.byref(cnt)), "h2sp_chol_struct")
        out = np.zeros(cnt.value, np.int32)
        _check(lib.h2sp_chol_struct(self.handle, J, out.ctypes.data, cnt.value, ctypes.byref(cnt)), "h2sp_chol_struct")
        return out

    def __del__(self):
        try:
            lib.h2sp_chol_destroy(self.handle)
        except Exception:  # noqa: BLE001
            pass


class CholFactor:
    """S = L L^T on the device (h2sp_chol_factor) for the S of the last stored
    build of a symmetric Sparsifier; solve(b) = S^-1 b in S order."""

    def __init__(self, sp: Sparsifier, stream=None, amalgamate: int = 0):
        from .krylov import CsrMatrix
        self.an = CholAnalysis(sp.plan, amalgamate)
        dev = sp.outputs["s_val"].device
        self.meta = torch.empty(self.an.meta_bytes + 256, dtype=torch.uint8, device=dev)
        self.meta_ptr = (self.meta.data_ptr() + 255) // 256 * 256
        self.panel = torch.empty(max(self.an.panel_doubles, 1), dtype=torch.float64, device=dev)
        st = _stream_handle(stream)
        _check(lib.h2sp_chol_upload(self.an.handle, self.meta_ptr, self.an.meta_bytes, st), "h2sp_chol_upload")
        self.S = CsrMatrix.from_sparsifier(sp)
        _check(lib.h2sp_chol_factor(self.an.handle, ctypes.byref(self.S.abi), self.meta_ptr, self.panel.data_ptr(), st),
               "h2sp_chol_factor")

    def solve(self, b, x=None, stream=None):
        x = torch.empty_like(b) if x is None else x
        _check(lib.h2sp_chol_solve(self.an.handle, self.meta_ptr, self.panel.data_ptr(), b.data_ptr(), x.data_ptr(),
                                   _stream_handle(stream)), "h2sp_chol_solve")
        return x

    def dense_L(self, plan):
        """Host dense L assembled from the panels (small N only; data movement)."""
        import numpy as np
        N = plan.N
        off = plan.offsets()["s_off_row"]
        an = self.an
        P = self.panel.cpu().numpy()
        L = np.zeros((N, N))
        starts, ms = an.starts, an.sizes
        po = 0
        for J in range(an.ns):
            mJ = ms[J]
            rows = []
            for I in an.struct(J):
                rows.extend(range(starts[I], starts[I] + ms[I]))
            blk = P[po:po + len(rows) * mJ].reshape(len(rows), mJ)
            L[np.array(rows)[:, None], np.arange(starts[J], starts[J] + mJ)[None, :]] = blk
            po += len(rows) * mJ
        return L


def _groups(plan):
    """(starts, sizes) of S's row groups (clusters with frozen rows), in S order."""
    import numpy as np
    off = plan.offsets()["s_off_row"]
    N = plan.N
    o = np.sort(np.unique(np.append(off, N)))
    starts = o[:-1]
    sizes = np.diff(o)
    keep = sizes > 0
    return starts[keep], sizes[keep]


def factor_chol(sp: Sparsifier, stream=None, amalgamate: int = 0) -> CholFactor:
    """Supernodal Cholesky of the S the last build wrote (symmetric plans);
    amalgamate: merged supernode width bound (0 = the row groups)."""
    return CholFactor(sp, stream=stream, amalgamate=amalgamate)


def solve_chol(sp: Sparsifier, fac: CholFactor, b, stream=None):
    """x = V S^-1 U^T b (Eq. sp0) with the device supernodal Cholesky."""
    bt = b.reshape(1, -1).contiguous()
    y = torch.empty_like(bt)
    sp.apply_Ut(bt, y, stream=stream)
    fac.solve(y[0], y[0], stream=stream)
    x = torch.empty_like(bt)
    sp.apply_V(y, x, stream=stream)
    return x[0]
