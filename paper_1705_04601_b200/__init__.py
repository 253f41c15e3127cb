"""Python binding of ``libh2sp`` -- the B200-native non-extensive sparsification of
an H^2 matrix (arXiv 1705.04601), ``A = U S V^T`` (PAPER.md Eq. main_fact,
P:477-484).

Argument marshalling only: every step of the hot path runs in the CUDA kernels
behind the C ABI declared in ``include/h2sp.h``.  PyTorch provides device
memory and streams.  There is no CPU fallback: importing this package raises
if ``libh2sp.so`` has not been built (``python -c "import __graft_entry__ as g;
g.build()"``), and every call that reaches the device raises if CUDA is
unavailable.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional

import numpy as np

__all__ = ["LIB_PATH", "H2spError", "Plan", "Sparsifier", "lib", "declared_symbols", "close_gen_params",
           "eval_kernel_blocks"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libh2sp.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "h2sp.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build the CUDA library first (__graft_entry__.build())")
lib = ctypes.CDLL(LIB_PATH)

_i32, _i64, _f64, _vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
_P_i32, _P_i64, _P_f64 = ctypes.POINTER(_i32), ctypes.POINTER(_i64), ctypes.POINTER(_f64)


class _Structure(ctypes.Structure):
    _fields_ = [("L", _i32), ("leaf_size", _i32), ("symmetric", _i32), ("rank_row", _P_i32), ("rank_col", _P_i32),
                ("near_ptr", _P_i64), ("near_col", _P_i32), ("adm_ptr", ctypes.POINTER(_P_i64)),
                ("adm_col", ctypes.POINTER(_P_i32))]


class _Sizes(ctypes.Structure):
    _fields_ = [(n, _i64) for n in ("n", "n_clusters", "leaf_row", "transfer_row", "leaf_col", "transfer_col", "close",
                                    "coupling", "q_row", "q_col", "s_nnz", "s_rows", "rank", "world", "first_leaf",
                                    "n_leaves_local", "s_blocks", "workspace_bytes", "meta_bytes",
                                    "levels_active", "launches")] + \
               [(n, _f64) for n in ("flops", "bytes", "flops_congruence", "flops_strips", "flops_executed",
                                    "flops_unique")] + [("bench_parts", _i64)]


class _LaunchInfo(ctypes.Structure):
    _fields_ = [("kind", _i32), ("level", _i32), ("items", _i64), ("flops", _f64), ("bytes", _f64), ("flops_exec", _f64)]


PLAN_EXPLICIT_Q = 1   # include/h2sp.h H2SP_PLAN_EXPLICIT_Q
PLAN_BENCH = 2        # include/h2sp.h H2SP_PLAN_BENCH
LAUNCH_KINDS = ("qr_row", "qr_col", "coupling", "congruence", "strips_row", "strips_col", "csr", "q_form",
                "bench_reduce")


class _ApplyArgs(ctypes.Structure):
    _fields_ = [("b", _vp), ("ldb", _i64), ("y", _vp), ("ldy", _i64), ("w", _vp), ("ldw", _i64), ("x", _vp),
                ("ldx", _i64), ("nrhs", ctypes.c_int), ("ws", _vp), ("ws_bytes", ctypes.c_size_t)]


class _Inputs(ctypes.Structure):
    _fields_ = [(n, _vp) for n in ("leaf_basis_row", "transfer_row", "leaf_basis_col", "transfer_col", "close",
                                   "coupling", "close_gen")]


class _CloseGen(ctypes.Structure):
    _fields_ = [("points", _vp), ("dim", _i32), ("kernel", _i32), ("p0", _f64), ("p1", _f64), ("nodes_row", _vp),
                ("nodes_col", _vp)]


KERNEL_IDS = {"exp": 1, "invh": 2, "laplace": 3}   # include/h2sp.h H2SP_KERNEL_*


def close_gen_params(kspec: dict):
    """(kernel id, p0, p1) of include/h2sp.h h2sp_close_gen for a generator
    kernel spec (h2gen._kernel_spec): exp(-r/ell) + nugget [same];
    1/(r+h) + diag_add [same]; 1/(4 pi r) with 1/(4 pi h) at the same point."""
    kind = kspec["kind"]
    if kind == "exp":
        return KERNEL_IDS[kind], float(kspec["ell"]), float(kspec["nugget"])
    if kind == "invh":
        return KERNEL_IDS[kind], float(kspec["h"]), float(kspec["diag_add"])
    if kind == "laplace":
        return KERNEL_IDS[kind], 0.0, 1.0 / (4.0 * np.pi * float(kspec["h"]))
    raise ValueError(f"no close_gen kernel for {kind!r}")


class _Outputs(ctypes.Structure):
    _fields_ = [(n, _vp) for n in ("q_row", "q_col", "s_rowptr", "s_col", "s_val", "bench_w", "bench_y", "bench_r2")]


_st = ctypes.c_int
lib.h2sp_status_str.restype = ctypes.c_char_p
lib.h2sp_status_str.argtypes = [_st]
lib.h2sp_last_error.restype = ctypes.c_char_p
lib.h2sp_plan_create.argtypes = [ctypes.POINTER(_Structure), ctypes.c_int, ctypes.POINTER(_vp)]
lib.h2sp_plan_create_shard.argtypes = [ctypes.POINTER(_Structure), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(_vp)]
lib.h2sp_plan_local_rows.argtypes = [_vp, _P_i64, _P_i64]
lib.h2sp_plan_sizes.argtypes = [_vp, ctypes.POINTER(_Sizes)]
lib.h2sp_plan_offsets.argtypes = [_vp] + [_P_i64] * 6
lib.h2sp_plan_pattern.argtypes = [_vp, _P_i64, _P_i32]
lib.h2sp_plan_destroy.argtypes = [_vp]
lib.h2sp_plan_destroy.restype = None
lib.h2sp_plan_upload.argtypes = [_vp, _vp, ctypes.c_size_t, _vp]
lib.h2sp_build.argtypes = [_vp, ctypes.POINTER(_Inputs), ctypes.POINTER(_Outputs), _vp, ctypes.c_size_t, _vp]
lib.h2sp_build_ex.argtypes = [_vp, ctypes.POINTER(_Inputs), ctypes.POINTER(_Outputs), _vp, ctypes.c_size_t, _vp,
                              ctypes.POINTER(_vp), _i64]
lib.h2sp_plan_launches.argtypes = [_vp, ctypes.POINTER(_LaunchInfo), _i64, ctypes.POINTER(_i64)]
lib.h2sp_build_apply.argtypes = [_vp, ctypes.POINTER(_Inputs), ctypes.POINTER(_Outputs), _vp, ctypes.c_size_t,
                                 ctypes.POINTER(_ApplyArgs), _vp, ctypes.POINTER(_vp), _i64]
lib.h2sp_build_meta.argtypes = [_vp, ctypes.POINTER(_Inputs), ctypes.POINTER(_Outputs), _vp, _vp, ctypes.c_size_t,
                                ctypes.POINTER(_ApplyArgs), _vp, ctypes.POINTER(_vp), _i64]
lib.h2sp_build_host.argtypes = [_vp, ctypes.POINTER(_Inputs), ctypes.POINTER(_Outputs), ctypes.POINTER(_Inputs),
                                ctypes.POINTER(_Outputs), _vp, ctypes.c_size_t, _vp]
lib.h2sp_eval_kernel_blocks.argtypes = [ctypes.POINTER(_CloseGen), _vp, _vp, _vp, _i64, _vp, _vp]
lib.h2sp_plan_set_qr_mode.argtypes = [_vp, ctypes.c_int]
lib.h2sp_plan_set_qr_mode.restype = ctypes.c_int
QR_NEED, QR_ALL, QR_REUSE = 0, 1, 2
lib.h2sp_apply_ws_bytes.argtypes = [_vp, ctypes.c_int]
lib.h2sp_apply_ws_bytes.restype = _i64
lib.h2sp_apply_Ut.argtypes = [_vp, _vp, _vp, _i64, _vp, _i64, ctypes.c_int, _vp, ctypes.c_size_t, _vp]
lib.h2sp_apply_V.argtypes = [_vp, _vp, _vp, _i64, _vp, _i64, ctypes.c_int, _vp, ctypes.c_size_t, _vp]


class H2spError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = lib.h2sp_status_str(status).decode()
        detail = lib.h2sp_last_error().decode()
        super().__init__(f"{where}: {msg} ({detail})")


def _check(status: int, where: str):
    if status != 0:
        raise H2spError(status, where)


def declared_symbols():
    """Function names declared in include/h2sp.h (for the ABI export test)."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(h2sp_[a-zA-Z_]+)\s*\(", txt)))


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class Plan:
    """Symbolic phase (host): ``h2sp_plan_create`` on the structure arrays of a
    packed H^2 input (``h2gen.pack``-style dict: L, B, symmetric, rank_row,
    rank_col, near_ptr, near_col, adm_ptr[k], adm_col[k]).  ``explicit_q``
    sets H2SP_PLAN_EXPLICIT_Q (no compact-WY level-0 congruence)."""

    def __init__(self, packed: dict, rank: int = 0, world: int = 1, explicit_q: bool = False, bench: bool = False):
        self._keep = []
        L = int(packed["L"])
        rr = np.ascontiguousarray(packed["rank_row"], dtype=np.int32)
        rc = np.ascontiguousarray(packed["rank_col"], dtype=np.int32) if packed.get("rank_col") is not None else None
        npt = np.ascontiguousarray(packed["near_ptr"], dtype=np.int64)
        ncl = np.ascontiguousarray(packed["near_col"], dtype=np.int32)
        aps = [np.ascontiguousarray(a, dtype=np.int64) for a in packed["adm_ptr"]]
        acs = [np.ascontiguousarray(a, dtype=np.int32) for a in packed["adm_col"]]
        self._keep += [rr, rc, npt, ncl, aps, acs]
        ap_arr = (_P_i64 * max(L, 1))(*[_ptr(a, _i64) for a in aps])
        ac_arr = (_P_i32 * max(L, 1))(*[_ptr(a, _i32) for a in acs])
        self._keep += [ap_arr, ac_arr]
        st = _Structure(L=L, leaf_size=int(packed["B"]), symmetric=int(packed["symmetric"]),
                        rank_row=_ptr(rr, _i32), rank_col=_ptr(rc, _i32) if rc is not None else None,
                        near_ptr=_ptr(npt, _i64), near_col=_ptr(ncl, _i32), adm_ptr=ap_arr, adm_col=ac_arr)
        h = _vp()
        flags = (PLAN_EXPLICIT_Q if explicit_q else 0) | (PLAN_BENCH if bench else 0)
        _check(lib.h2sp_plan_create_shard(ctypes.byref(st), int(rank), int(world), flags, ctypes.byref(h)),
               "h2sp_plan_create_shard")
        self.bench = bool(bench)
        self.handle = h
        self._keep = None
        sz = _Sizes()
        _check(lib.h2sp_plan_sizes(self.handle, ctypes.byref(sz)), "h2sp_plan_sizes")
        self.sizes = {f: getattr(sz, f) for f, _ in _Sizes._fields_}
        self.L = L
        self.B = int(packed["B"])
        self.symmetric = bool(packed["symmetric"])
        self.N = self.sizes["n"]
        self.rank, self.world = int(rank), int(world)
        self.s_rows = self.sizes["s_rows"]
        self.n_tree_local = self.sizes["n_leaves_local"] * self.B   # tree-order rows of this shard

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and lib is not None:
            lib.h2sp_plan_destroy(h)
            self.handle = None

    def offsets(self) -> Dict[str, np.ndarray]:
        n = self.sizes["n_clusters"]
        out = {k: np.zeros(n, dtype=np.int64) for k in ("s_off_row", "s_off_col", "q_off_row", "q_off_col",
                                                         "n_row", "n_col")}
        _check(lib.h2sp_plan_offsets(self.handle, *[_ptr(out[k], _i64) for k in ("s_off_row", "s_off_col",
                                                                                   "q_off_row", "q_off_col",
                                                                                   "n_row", "n_col")]),
               "h2sp_plan_offsets")
        return out

    def local_rows(self):
        """Local S row offset of each owned cluster (-1 otherwise), row / column side."""
        n = self.sizes["n_clusters"]
        a, b = np.zeros(n, dtype=np.int64), np.zeros(n, dtype=np.int64)
        _check(lib.h2sp_plan_local_rows(self.handle, _ptr(a, _i64), _ptr(b, _i64)), "h2sp_plan_local_rows")
        return a, b

    def global_rows(self):
        """Global S-order row index of every local S row of this plan."""
        loc, _ = self.local_rows()
        off = self.offsets()
        m = off["n_row"] - np.asarray(self._k_row(), dtype=np.int64)
        out = np.empty(self.s_rows, dtype=np.int64)
        for c in np.nonzero(loc >= 0)[0]:
            out[loc[c]:loc[c] + m[c]] = off["s_off_row"][c] + np.arange(m[c])
        return out

    def _k_row(self):
        off = self.offsets()
        # m = n - k is recovered from consecutive S offsets of the full ordering
        s_off = off["s_off_row"]
        m = np.diff(np.append(s_off, self.N))
        return off["n_row"] - m

    def ranks(self, side: int = 0) -> np.ndarray:
        """Rank k_t of every cluster (level-major), row (0) or column (1) side."""
        off = self.offsets()
        key = "s_off_row" if side == 0 else "s_off_col"
        m = np.diff(np.append(off[key], self.N))
        return (off["n_row" if side == 0 else "n_col"] - m).astype(np.int64)

    def launches(self):
        """Per-launch descriptors of one build (kind, level, items, flops, bytes, flops_exec)."""
        n = _i64()
        _check(lib.h2sp_plan_launches(self.handle, None, 0, ctypes.byref(n)), "h2sp_plan_launches")
        arr = (_LaunchInfo * max(n.value, 1))()
        _check(lib.h2sp_plan_launches(self.handle, arr, n.value, ctypes.byref(n)), "h2sp_plan_launches")
        return [dict(kind=LAUNCH_KINDS[a.kind], level=a.level, items=a.items, flops=a.flops, bytes=a.bytes,
                     flops_exec=a.flops_exec)
                for a in arr[:n.value]]

    def pattern(self, with_cols: bool = True):
        rowptr = np.zeros(self.s_rows + 1, dtype=np.int64)
        col = np.zeros(self.sizes["s_nnz"], dtype=np.int32) if with_cols else None
        _check(lib.h2sp_plan_pattern(self.handle, _ptr(rowptr, _i64), _ptr(col, _i32) if with_cols else None),
               "h2sp_plan_pattern")
        return rowptr, col


def eval_kernel_blocks(kspec: dict, x_nodes, y_nodes, descs, out, stream=None):
    """h2sp_eval_kernel_blocks: out[b] = K(x_nodes[x_off + i], y_nodes[y_off + j]) for
    every block record of ``descs`` (int64 CUDA tensor, 4 words per block, see
    h2gen.coupling_block_descs); x_nodes / y_nodes: (n, d) float64 CUDA tensors."""
    kid, p0, p1 = close_gen_params(kspec)
    g = _CloseGen(points=None, dim=int(x_nodes.shape[1]), kernel=kid, p0=p0, p1=p1)
    _check(lib.h2sp_eval_kernel_blocks(ctypes.byref(g), _dptr(x_nodes), _dptr(y_nodes), _dptr(descs),
                                       int(descs.shape[0]), _dptr(out), _stream_handle(stream)),
           "h2sp_eval_kernel_blocks")
    return out


def _dptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream_handle(stream) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Sparsifier:
    """Device buffers for one plan: inputs (copied once from a packed dict),
    outputs and the uploaded workspace; ``build()`` runs ``h2sp_build``."""

    def __init__(self, plan: Plan, packed: Optional[dict] = None, device="cuda", alloc_inputs: bool = True,
                 close_gen: Optional[dict] = None, inputs: Optional[dict] = None, outputs: Optional[dict] = None,
                 workspace: bool = True):
        """close_gen: {"points": (N, d) tree-ordered array, "kernel": generator
        kernel spec [, "nodes_row": (sum k, d), "nodes_col": ...]} -> matrix-free
        close blocks (h2sp_close_gen); with nodes also matrix-free couplings (no
        coupling buffer).  inputs / outputs: ready device tensors to use instead
        of allocating (e.g. bases built on the device by h2sp construction, or
        the global outputs shared by the virtual shards of one matrix).
        workspace=False: no build workspace (VirtualShards supplies meta + scratch)."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1705_04601_b200 needs a CUDA device (no CPU fallback)")
        self.plan = plan
        self.device = torch.device(device)
        sz = plan.sizes
        f64 = dict(dtype=torch.float64, device=self.device)
        self.inputs = dict(inputs) if inputs else {}
        self._gen = None
        coup_gen = False
        if close_gen is not None:
            def dev(a):
                if isinstance(a, torch.Tensor):
                    return a.to(self.device, dtype=torch.float64).contiguous()
                return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)
            pts = close_gen["points"]
            if pts.ndim != 2 or pts.shape[0] != int(sz["n"]) or not 1 <= pts.shape[1] <= 3:
                raise ValueError(f"close_gen points must be (N={int(sz['n'])}, d<=3), got {tuple(pts.shape)}")
            kid, p0, p1 = close_gen_params(close_gen["kernel"])
            self.inputs["points"] = dev(pts)
            self._gen = _CloseGen(points=self.inputs["points"].data_ptr(), dim=pts.shape[1], kernel=kid, p0=p0, p1=p1)
            if close_gen.get("nodes_row") is not None:
                self.inputs["nodes_row"] = dev(close_gen["nodes_row"])
                self._gen.nodes_row = self.inputs["nodes_row"].data_ptr()
                if not plan.symmetric:
                    self.inputs["nodes_col"] = dev(close_gen["nodes_col"])
                    self._gen.nodes_col = self.inputs["nodes_col"].data_ptr()
                coup_gen = True
        if alloc_inputs:
            names = [("leaf_basis_row", "leaf_row", "leaf_row"), ("transfer_row", "transfer_row", "transfer_row")]
            if not coup_gen:
                names.append(("coupling", "coupling", "coupling"))
            if self._gen is None:
                names.append(("close", "close", "close"))
            if not plan.symmetric:
                names += [("leaf_basis_col", "leaf_col", "leaf_col"), ("transfer_col", "transfer_col", "transfer_col")]
            for abi, key, szk in names:
                if abi in self.inputs:
                    continue
                n = int(sz[szk])
                t = torch.empty(max(n, 1), **f64)
                if packed is not None and n and packed.get(key) is not None:
                    src = np.ascontiguousarray(packed[key], dtype=np.float64).ravel()
                    if src.size != n:
                        raise ValueError(f"input {key}: {src.size} values, plan expects {n}")
                    t[:n].copy_(torch.from_numpy(src))
                self.inputs[abi] = t
        if outputs is not None:
            self.outputs = outputs
        elif plan.bench:
            N = int(sz["n"])
            self.outputs = {
                "q_row": torch.empty(max(int(sz["q_row"]), 1), **f64),
                "q_col": torch.empty(max(int(sz["q_col"]), 1), **f64) if not plan.symmetric else None,
                "s_rowptr": None, "s_col": None, "s_val": None,
                "bench_w": torch.zeros(N, **f64), "bench_y": torch.zeros(N, **f64),
                "bench_r2": torch.zeros(N, **f64),
            }
        else:
            self.outputs = {
                "q_row": torch.empty(max(int(sz["q_row"]), 1), **f64),
                "q_col": torch.empty(max(int(sz["q_col"]), 1), **f64) if not plan.symmetric else None,
                "s_rowptr": torch.empty(plan.s_rows + 1, dtype=torch.int64, device=self.device),
                "s_col": torch.empty(max(int(sz["s_nnz"]), 1), dtype=torch.int32, device=self.device),
                "s_val": torch.empty(max(int(sz["s_nnz"]), 1), **f64),
            }
        self.ws = None
        self.ws_ptr, self.ws_bytes = None, 0
        if workspace:
            self.ws = torch.empty(int(sz["workspace_bytes"]) + 256, dtype=torch.uint8, device=self.device)
            self.ws_ptr = (self.ws.data_ptr() + 255) // 256 * 256
            self.ws_bytes = int(sz["workspace_bytes"])
            _check(lib.h2sp_plan_upload(plan.handle, self.ws_ptr, self.ws_bytes, _stream_handle(None)),
                   "h2sp_plan_upload")

    def _abi_inputs(self, inputs=None):
        src = inputs if inputs is not None else self.inputs
        a = _Inputs(**{k: _dptr(src.get(k)) for k, _ in _Inputs._fields_ if k != "close_gen"})
        if self._gen is not None and self._gen.nodes_row:
            a.coupling = None
        if self._gen is not None:
            a.close_gen = ctypes.addressof(self._gen)
        return a

    def _abi_outputs(self, outputs=None):
        o = outputs if outputs is not None else self.outputs
        return _Outputs(**{k: _dptr(o.get(k)) for k, _ in _Outputs._fields_})

    def build(self, stream=None, write_index: bool = True):
        out = self._abi_outputs()
        if not write_index:
            out.s_rowptr = None
            out.s_col = None
        _check(lib.h2sp_build(self.plan.handle, ctypes.byref(self._abi_inputs()), ctypes.byref(out), self.ws_ptr,
                              self.ws_bytes, _stream_handle(stream)), "h2sp_build")
        return self.outputs

    def capture(self, fn=None):
        """Capture one h2sp_build (plus ``fn()``, e.g. the applies) into a CUDA
        graph on a side stream; returns the torch.cuda.CUDAGraph (replay() runs
        it on the current stream's device).  The library's internal side
        streams fork from and join back into the captured stream."""
        import torch
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.build(stream=s)     # warm-up on the capture stream (lazy init outside capture)
            if fn is not None:
                fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            self.build(stream=s)
            if fn is not None:
                fn()
        return g

    def build_profiled(self, events, stream=None):
        """h2sp_build_ex: records events[i] (torch.cuda.Event) before launch i and
        events[-1] after the last launch, on the launching stream."""
        arr = (_vp * len(events))(*[e.cuda_event for e in events])
        _check(lib.h2sp_build_ex(self.plan.handle, ctypes.byref(self._abi_inputs()),
                                 ctypes.byref(self._abi_outputs()), self.ws_ptr, self.ws_bytes,
                                 _stream_handle(stream), arr, len(events)), "h2sp_build_ex")
        return self.outputs

    def apply_workspace(self, nrhs: int):
        """A separate uploaded workspace for the applies of h2sp_build_apply."""
        import torch
        need = int(lib.h2sp_apply_ws_bytes(self.plan.handle, nrhs))
        ws = torch.empty(need + 256, dtype=torch.uint8, device=self.device)
        ptr = (ws.data_ptr() + 255) // 256 * 256
        _check(lib.h2sp_plan_upload(self.plan.handle, ptr, need, _stream_handle(None)), "h2sp_plan_upload")
        return ws, ptr, need

    def build_apply(self, b, y, w, x, apply_ws, events=None, stream=None):
        """One pass: build + y = U^T b + x = V w (w may be y), the applies
        overlapping the congruence (h2sp_build_apply).  b, x: (nrhs, n_tree_local);
        y, w: (nrhs, s_rows); apply_ws from apply_workspace()."""
        nrhs = b.shape[0] if b is not None else w.shape[0]
        _, ptr, need = apply_ws
        a = _ApplyArgs(b=_dptr(b), ldb=b.shape[-1] if b is not None else 0, y=_dptr(y),
                       ldy=y.shape[-1] if y is not None else 0, w=_dptr(w), ldw=w.shape[-1] if w is not None else 0,
                       x=_dptr(x), ldx=x.shape[-1] if x is not None else 0, nrhs=nrhs, ws=ptr, ws_bytes=need)
        arr = (_vp * len(events))(*[e.cuda_event for e in events]) if events else None
        _check(lib.h2sp_build_apply(self.plan.handle, ctypes.byref(self._abi_inputs()),
                                    ctypes.byref(self._abi_outputs()), self.ws_ptr, self.ws_bytes, ctypes.byref(a),
                                    _stream_handle(stream), arr, len(events) if events else 0), "h2sp_build_apply")
        return self.outputs

    def build_host(self, host_inputs: dict, host_outputs: dict, stream=None):
        """End-to-end: H2D of host (pinned) inputs, build, D2H of all outputs."""
        hi = _Inputs(**{k: _dptr(host_inputs.get(k)) for k, _ in _Inputs._fields_ if k != "close_gen"})
        ho = _Outputs(**{k: _dptr(host_outputs.get(k)) for k, _ in _Outputs._fields_})
        hgen = None
        if self._gen is not None:   # host points (pinned tensor) -> the device points buffer
            hp = host_inputs["points"]
            hgen = _CloseGen(points=_dptr(hp), dim=self._gen.dim, kernel=self._gen.kernel, p0=self._gen.p0,
                             p1=self._gen.p1)
            hi.close_gen = ctypes.addressof(hgen)
        _check(lib.h2sp_build_host(self.plan.handle, ctypes.byref(hi), ctypes.byref(ho),
                                   ctypes.byref(self._abi_inputs()), ctypes.byref(self._abi_outputs()), self.ws_ptr,
                                   self.ws_bytes, _stream_handle(stream)), "h2sp_build_host")

    def apply_ws(self, nrhs: int):
        import torch
        need = int(lib.h2sp_apply_ws_bytes(self.plan.handle, nrhs))
        if need <= self.ws_bytes:
            return self.ws_ptr, self.ws_bytes
        ws = torch.empty(need + 256, dtype=torch.uint8, device=self.device)
        ptr = (ws.data_ptr() + 255) // 256 * 256
        _check(lib.h2sp_plan_upload(self.plan.handle, ptr, need, _stream_handle(None)), "h2sp_plan_upload")
        self._apply_ws = ws
        return ptr, need

    def apply_Ut(self, b, y, stream=None, ws=None):
        """y = U^T b; b: (nrhs, n_tree_local), y: (nrhs, s_rows) contiguous float64 CUDA
        tensors (= column-major with nrhs columns); n_tree_local = s_rows = N unsharded."""
        nrhs = b.shape[0] if b.dim() == 2 else 1
        ptr, nb = ws if ws is not None else self.apply_ws(nrhs)
        _check(lib.h2sp_apply_Ut(self.plan.handle, self.outputs["q_row"].data_ptr(), b.data_ptr(),
                                 b.shape[-1], y.data_ptr(), y.shape[-1], nrhs, ptr, nb, _stream_handle(stream)),
               "h2sp_apply_Ut")
        return y

    def apply_V(self, y, x, stream=None, ws=None):
        """x = V y; y, x: (nrhs, N) contiguous float64 CUDA tensors."""
        nrhs = y.shape[0] if y.dim() == 2 else 1
        ptr, nb = ws if ws is not None else self.apply_ws(nrhs)
        q = self.outputs["q_row"] if self.plan.symmetric else self.outputs["q_col"]
        _check(lib.h2sp_apply_V(self.plan.handle, q.data_ptr(), y.data_ptr(), y.shape[-1], x.data_ptr(),
                                x.shape[-1], nrhs, ptr, nb, _stream_handle(stream)), "h2sp_apply_V")
        return x


class VirtualShards:
    """The virtual shards of ONE matrix processed one after another on one
    device (SURVEY §8(d) config-5 protocol step 2): G sharded plans (top-level
    subtrees), each with its work lists resident in its own device buffer, all
    taking turns on one shared scratch buffer (h2sp_build_meta), with shared
    inputs and global outputs (Q, and in bench mode y = S w and the row norms).
    ``plans``: Plan objects (same matrix, ranks 0..G-1 of world G).
    ``share_qr`` (protocol step 2: "QR/R^ for every cluster depends only on the
    bases, so it runs first for all clusters"): the first shard's build runs the
    QR completion of every cluster (H2SP_QR_ALL), the others reuse its R^ / V, M
    (head of the shared scratch) and Q (H2SP_QR_REUSE) instead of repeating the
    QR of their need sets; results are bitwise the same."""

    def __init__(self, plans, packed: Optional[dict] = None, device="cuda", close_gen: Optional[dict] = None,
                 inputs: Optional[dict] = None, nrhs: int = 1, share_qr: bool = True):
        import torch
        self.plans = list(plans)
        self.share_qr = bool(share_qr) and len(self.plans) > 1
        self.device = torch.device(device)
        first = Sparsifier(self.plans[0], packed, device=device, close_gen=close_gen, inputs=inputs, workspace=False)
        self.shards = [first] + [Sparsifier(p, None, device=device, alloc_inputs=False, close_gen=None,
                                            inputs=first.inputs, outputs=first.outputs, workspace=False)
                                 for p in self.plans[1:]]
        for sp in self.shards[1:]:
            sp._gen = first._gen
        self.inputs, self.outputs = first.inputs, first.outputs
        self._meta = []
        for p in self.plans:   # every shard's work lists stay resident
            mb = int(p.sizes["meta_bytes"])
            buf = torch.empty(mb + 256, dtype=torch.uint8, device=self.device)
            ptr = (buf.data_ptr() + 255) // 256 * 256
            _check(lib.h2sp_plan_upload(p.handle, ptr, mb, _stream_handle(None)), "h2sp_plan_upload")
            self._meta.append((buf, ptr))
        need = max(int(p.sizes["workspace_bytes"]) - int(p.sizes["meta_bytes"]) for p in self.plans)
        self.scratch = torch.empty(need + 256, dtype=torch.uint8, device=self.device)
        self.scratch_ptr = (self.scratch.data_ptr() + 255) // 256 * 256
        self.scratch_bytes = need
        self.nrhs = nrhs
        aneed = max(int(lib.h2sp_apply_ws_bytes(p.handle, nrhs)) - int(p.sizes["meta_bytes"]) for p in self.plans)
        self.apply_scratch = torch.empty(aneed + 256, dtype=torch.uint8, device=self.device)
        self.apply_ptr = (self.apply_scratch.data_ptr() + 255) // 256 * 256
        self.apply_bytes = aneed

    def build(self, applies=None, events=None, stream=None, after_first=None):
        """One pass over all shards.  applies: per shard (b, y, w, x) tensors or
        None (b, x: (nrhs, n_tree_local); y, w: (nrhs, s_rows) of that shard);
        events: per shard a list of 2 * launches torch.cuda.Event or None;
        after_first: called once the first shard's build is enqueued -- with
        share_qr the Q of every cluster is final from there on (the later shards
        do not write it), so a caller may start reading it back beside them."""
        for i, (sp, (_, mptr)) in enumerate(zip(self.shards, self._meta)):
            ap = None
            if applies is not None and applies[i] is not None:
                b, y, w, x = applies[i]
                ap = _ApplyArgs(b=_dptr(b), ldb=b.shape[-1] if b is not None else 0, y=_dptr(y),
                                ldy=y.shape[-1] if y is not None else 0, w=_dptr(w),
                                ldw=w.shape[-1] if w is not None else 0, x=_dptr(x),
                                ldx=x.shape[-1] if x is not None else 0, nrhs=self.nrhs, ws=self.apply_ptr,
                                ws_bytes=self.apply_bytes)
            ev = events[i] if events is not None else None
            arr = (_vp * len(ev))(*[e.cuda_event for e in ev]) if ev else None
            mode = (QR_ALL if i == 0 else QR_REUSE) if self.share_qr else QR_NEED
            _check(lib.h2sp_plan_set_qr_mode(sp.plan.handle, mode), "h2sp_plan_set_qr_mode")
            _check(lib.h2sp_build_meta(sp.plan.handle, ctypes.byref(sp._abi_inputs()),
                                       ctypes.byref(sp._abi_outputs()), mptr, self.scratch_ptr, self.scratch_bytes,
                                       ctypes.byref(ap) if ap is not None else None, _stream_handle(stream), arr,
                                       len(ev) if ev else 0), "h2sp_build_meta")
            if i == 0 and after_first is not None:
                after_first()
        return self.outputs


class _ChebSpec(ctypes.Structure):
    _fields_ = [("dim", _i32), ("orders", _i32 * 3), ("cheb_cos", _f64 * 64)]


lib.h2sp_cheb_construct.argtypes = [_vp, _vp, ctypes.c_int, ctypes.POINTER(_ChebSpec), _vp, _vp, _vp, _vp, _vp, _vp,
                                    _vp]


def cheb_construct(plan: Plan, meta_ptr: int, points, box_lo, box_hi, orders, cos_table, side: int = 0,
                   stream=None) -> dict:
    """h2sp_cheb_construct: the nested Chebyshev bases of one side on the device.
    points (N, d), box_lo / box_hi (n_clusters, d): float64 CUDA tensors;
    orders: base tensor orders (largest-extent axis first); cos_table: the 64
    cosines (h2gen.cheb_cos_table).  Returns {"leaf", "transfer", "nodes"}."""
    import torch
    d = int(points.shape[1])
    sz = plan.sizes
    f64 = dict(dtype=torch.float64, device=points.device)
    leaf = torch.zeros(max(int(sz["leaf_row" if side == 0 else "leaf_col"]), 1), **f64)
    tr = torch.zeros(max(int(sz["transfer_row" if side == 0 else "transfer_col"]), 1), **f64)
    off = plan.offsets()
    n_nodes = int(sum(int(x) for x in (plan.ranks(side))))
    nodes = torch.zeros(max(n_nodes, 1), d, **f64)
    spec = _ChebSpec(dim=d)
    for a in range(3):
        spec.orders[a] = int(orders[a]) if a < d else 1
    for i in range(64):
        spec.cheb_cos[i] = float(cos_table[i])
    _check(lib.h2sp_cheb_construct(plan.handle, meta_ptr, int(side), ctypes.byref(spec), _dptr(points), _dptr(box_lo),
                                   _dptr(box_hi), _dptr(leaf), _dptr(tr), _dptr(nodes), _stream_handle(stream)),
           "h2sp_cheb_construct")
    del off
    return {"leaf": leaf, "transfer": tr, "nodes": nodes}


lib.h2sp_comm_unique_id.argtypes = [_vp]
lib.h2sp_comm_init.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]
lib.h2sp_comm_allreduce.argtypes = [_vp, _vp, _i64, ctypes.c_int, _vp]
lib.h2sp_comm_info.argtypes = [_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
lib.h2sp_comm_destroy.argtypes = [_vp]
lib.h2sp_comm_destroy.restype = None
SUM, MAX = 0, 1


class Comm:
    """NCCL communicator of libh2sp (h2sp_comm_*), bootstrapped through a torch
    process group: rank 0 draws the unique id, the group broadcasts it."""

    def __init__(self, rank: int, world: int, broadcast=None):
        """broadcast(bytes) -> bytes: the caller's rank-0 broadcast (e.g. through
        torch.distributed.broadcast_object_list); None for world == 1."""
        buf = ctypes.create_string_buffer(128)
        if rank == 0:
            _check(lib.h2sp_comm_unique_id(buf), "h2sp_comm_unique_id")
        uid = bytes(buf.raw)
        if world > 1:
            uid = broadcast(uid)
        ctypes.memmove(buf, uid, 128)
        h = _vp()
        _check(lib.h2sp_comm_init(buf, int(rank), int(world), ctypes.byref(h)), "h2sp_comm_init")
        self.handle = h
        self.rank, self.world = rank, world

    def allreduce(self, t, op: int = SUM, stream=None):
        """In-place sum / max of a contiguous float64 CUDA tensor across ranks."""
        _check(lib.h2sp_comm_allreduce(self.handle, t.data_ptr(), t.numel(), op, _stream_handle(stream)),
               "h2sp_comm_allreduce")
        return t

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and lib is not None:
            lib.h2sp_comm_destroy(h)
            self.handle = None


def torch_comm(rank: int, world: int) -> Comm:
    """A Comm bootstrapped from the initialised torch.distributed default group."""
    def bcast(uid: bytes) -> bytes:
        import torch.distributed as dist
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]
    return Comm(rank, world, bcast if world > 1 else None)
