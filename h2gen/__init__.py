"""Seeded synthetic H^2 inputs for the sparsification hot path (setup, untimed).

This module is the ONLY code shared by the CPU oracle (``oracle/``) and the CUDA
path (``paper_1705_04601_b200``): it produces the *inputs* of the method -- the
cluster tree, block cluster tree, leaf bases, transfer matrices, close blocks and
far couplings of an H^2 matrix (§4.1, Def. "H^2 matrix", P:669-675:
``A = C + sum_b R_t D_b E_s^T``).  It holds none of the sparsification
arithmetic (no QR, no congruence, no permutation into S): the paper assumes the
H^2 matrix "is given" and so do both implementations.

Conventions (shared vocabulary, see include/h2sp.h and DESIGN.md):
  * Balanced binary cluster tree with ``L`` levels above the leaves; level 0 =
    leaves (``2^L`` clusters of ``B`` indices each), level ``L`` = root.
  * Cluster ``(k, i)`` has level-major id ``cid = lvl_off[k] + i`` with
    ``lvl_off[k] = 2^(L+1) - 2^(L-k+1)``; children of ``(k, i)`` are
    ``(k-1, 2i)`` and ``(k-1, 2i+1)``.  Leaf ``i`` owns tree-order indices
    ``[iB, (i+1)B)``.
  * ``near`` = inadmissible leaf pairs N_0 (sorted by (t, s)); ``adm[k]`` =
    admissible pairs A_k at level k (sorted); together they are the leaves of
    the block cluster tree.
  * Leaf basis ``R_t`` is ``B x k_t``; transfer ``T_p`` is ``(k_c1 + k_c2) x k_p``
    (child 1's rows first), so the effective basis is
    ``R_p = diag(R_c1, R_c2) T_p`` (nested bases).
  * Close block ``C_ts`` is ``B x B``; coupling ``D_b`` is ``k_t x k_s``.

Input recipes: ``BASELINE.json`` configs 1-5 (points,
kernel, B, r, eta), random H^2 matrices with ragged ranks, the eta=0 case, the
axis-aligned-basis case and the paper's Fig. 1/3 example.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Tuple

import numpy as np

__all__ = [
    "H2Input", "CONFIGS", "lvl_off", "cid", "make_points", "kd_tree", "block_tree",
    "make_config", "random_h2", "axis_aligned_h2", "fig3_h2", "eta0_h2",
    "kernel_matrix", "pack", "make_ifmm", "random_sparse", "coupling_block_descs", "make_structure", "fill_cheb_bases", "cheb_cos_table",
    "cheb_base_orders",
]


# ----------------------------------------------------------------------------
# Cluster numbering
# ----------------------------------------------------------------------------

def lvl_off(L: int, k: int) -> int:
    """First level-major id of level ``k`` (level 0 = leaves)."""
    return (1 << (L + 1)) - (1 << (L - k + 1))


def cid(L: int, k: int, i: int) -> int:
    return lvl_off(L, k) + i


def n_clusters(L: int) -> int:
    return (1 << (L + 1)) - 1


# ----------------------------------------------------------------------------
# Container
# ----------------------------------------------------------------------------

@dataclasses.dataclass
class H2Input:
    """Parameters of an H^2 matrix in tree order.

    ``leaf_row[i]``: B x k leaf basis of leaf i; ``transfer_row[c]``: transfer of
    internal cluster with level-major id c (None for leaves).  Column side
    likewise; in symmetric mode the column lists are the row lists and
    ``C_st = C_ts^T``, ``D_st = D_ts^T`` hold bitwise.
    """
    L: int
    B: int
    symmetric: bool
    rank_row: np.ndarray            # int32 [n_clusters]
    rank_col: np.ndarray            # int32 [n_clusters]
    leaf_row: List[np.ndarray]
    leaf_col: List[np.ndarray]
    transfer_row: List[Optional[np.ndarray]]
    transfer_col: List[Optional[np.ndarray]]
    near: np.ndarray                # int32 [n_near, 2] (t, s) leaf pairs, sorted
    close: np.ndarray               # float64 [n_near, B, B]
    adm: List[np.ndarray]           # per level k=0..L-1: int32 [n_k, 2], sorted
    coupling: List[List[np.ndarray]]  # per level: list of k_t x k_s arrays
    points: Optional[np.ndarray] = None   # tree-ordered points (N, d), if any
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def N(self) -> int:
        return self.B << self.L

    @property
    def n_leaves(self) -> int:
        return 1 << self.L


# ----------------------------------------------------------------------------
# Points, KD tree, block cluster tree
# ----------------------------------------------------------------------------

def make_points(kind: str, N: int, rng: np.random.Generator) -> np.ndarray:
    """Point clouds of BASELINE.json configs (readings 16-17)."""
    if kind == "square":
        return rng.random((N, 2))
    if kind == "cube":
        return rng.random((N, 3))
    if kind == "sphere":
        # Fibonacci lattice + tangent jitter in a disc of radius 0.1*h,
        # renormalised to the unit sphere (SURVEY §8(c) reading 16).
        i = np.arange(N, dtype=np.float64)
        z = 1.0 - (2.0 * i + 1.0) / N
        phi = i * math.pi * (3.0 - math.sqrt(5.0))
        rho = np.sqrt(np.maximum(0.0, 1.0 - z * z))
        p = np.stack([rho * np.cos(phi), rho * np.sin(phi), z], axis=1)
        h = math.sqrt(4.0 * math.pi / N)
        # orthonormal tangent frame
        a = np.where(np.abs(p[:, 2:3]) < 0.9, np.array([[0.0, 0.0, 1.0]]), np.array([[1.0, 0.0, 0.0]]))
        e1 = np.cross(p, a)
        e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
        e2 = np.cross(p, e1)
        rad = 0.1 * h * np.sqrt(rng.random(N))
        ang = 2.0 * math.pi * rng.random(N)
        p = p + (rad * np.cos(ang))[:, None] * e1 + (rad * np.sin(ang))[:, None] * e2
        return p / np.linalg.norm(p, axis=1, keepdims=True)
    raise ValueError(kind)


def kd_tree(points: np.ndarray, L: int):
    """Balanced KD tree: median split along the longest box axis, ties by a
    stable sort on (coordinate, index) (SURVEY §8(c) reading 10).

    Returns ``perm`` (tree order -> original index) and per-cluster tight boxes
    ``lo, hi`` of shape [n_clusters, d] (level-major ids).
    """
    N, d = points.shape
    if N % (1 << L):
        raise ValueError("N must be B * 2^L")
    perm = np.arange(N)
    ncl = n_clusters(L)
    lo = np.zeros((ncl, d))
    hi = np.zeros((ncl, d))
    # rank of every point along each axis in the (coordinate, index) order: a
    # segment sorted by (coordinate, index) is the segment sorted by this rank
    rank = np.empty((d, N), dtype=np.int64)
    for a in range(d):
        rank[a, np.argsort(points[:, a], kind="stable")] = np.arange(N)
    # top-down: at level k the segments have size N >> (L - k)
    for k in range(L, -1, -1):
        M = 1 << (L - k)
        size = N // M
        seg = points[perm].reshape(M, size, d)
        blo = seg.min(axis=1)
        bhi = seg.max(axis=1)
        base = lvl_off(L, k)
        lo[base:base + M] = blo
        hi[base:base + M] = bhi
        if k == 0:
            break
        axis = np.argmax(bhi - blo, axis=1)                        # [M]
        key = np.repeat(np.arange(M, dtype=np.int64) * N, size) + rank[np.repeat(axis, size), perm]
        perm = perm[np.argsort(key)]                                # keys distinct: (segment, coord, index)
    return perm, lo, hi


def _admissible(lo, hi, t, s, eta):
    diam_t = np.linalg.norm(hi[t] - lo[t], axis=1)
    diam_s = np.linalg.norm(hi[s] - lo[s], axis=1)
    gap = np.maximum(0.0, np.maximum(lo[s] - hi[t], lo[t] - hi[s]))
    dist = np.linalg.norm(gap, axis=1)
    return np.maximum(diam_t, diam_s) <= eta * dist


def block_tree(lo, hi, L: int, eta: float):
    """Leaves of the block cluster tree: sons(t) x sons(s) splitting
    of inadmissible pairs, admissibility ``max(diam) <= eta * dist`` on tight
    boxes (SURVEY §8(c) readings 8, 10).  Returns (near N_0 [n,2], adm list)."""
    cand = np.zeros((1, 2), dtype=np.int64)   # (root, root) at level L (in-level index)
    adm: List[np.ndarray] = [None] * L
    near0 = None
    for k in range(L, -1, -1):
        base = lvl_off(L, k)
        if k < L:
            ok = _admissible(lo, hi, base + cand[:, 0], base + cand[:, 1], eta) if len(cand) else np.zeros(0, bool)
            a = cand[ok]
            adm[k] = a[np.lexsort((a[:, 1], a[:, 0]))].astype(np.int32)
            cand = cand[~ok]
        if k == 0:
            near0 = cand[np.lexsort((cand[:, 1], cand[:, 0]))].astype(np.int32)
            break
        # children pairs of inadmissible pairs
        ch = np.empty((len(cand) * 4, 2), dtype=np.int64)
        for a_ in range(2):
            for b_ in range(2):
                j = a_ * 2 + b_
                ch[j::4, 0] = 2 * cand[:, 0] + a_
                ch[j::4, 1] = 2 * cand[:, 1] + b_
        cand = ch
    return near0, adm


def far_ranks(L: int, near0, adm, r_leaf: int, r: int, side: int):
    """Rank r for clusters with an admissible pair at or above them, else 0
    (SURVEY §8(c) reading 5); root rank 0 (reading 4)."""
    ncl = n_clusters(L)
    has = np.zeros(ncl, dtype=bool)
    for k in range(L):
        if len(adm[k]):
            has[lvl_off(L, k) + np.unique(adm[k][:, side])] = True
    # propagate "at or above" downwards
    for k in range(L - 1, -1, -1):
        base, pbase = lvl_off(L, k), lvl_off(L, k + 1)
        M = 1 << (L - k)
        has[base:base + M] |= has[pbase + np.arange(M) // 2]
    rank = np.zeros(ncl, dtype=np.int32)
    rank[has] = r
    rank[:1 << L][has[:1 << L]] = r_leaf
    rank[ncl - 1] = 0
    return rank


# ----------------------------------------------------------------------------
# Kernels (BASELINE.json configs)
# ----------------------------------------------------------------------------

def kernel_matrix(spec: dict, x: np.ndarray, y: np.ndarray, same_index=None) -> np.ndarray:
    """Kernel block K(x_i, y_j); ``same_index`` (bool matrix) marks i == j of
    the point set, where the diagonal self-term replaces/adds (BJ:configs)."""
    diff = x[:, None, :] - y[None, :, :]
    r = np.sqrt(np.einsum("ijk,ijk->ij", diff, diff))
    kind = spec["kind"]
    if kind == "exp":
        K = np.exp(-r / spec["ell"])
        if same_index is not None:
            K = K + spec["nugget"] * same_index
    elif kind == "invh":
        h = spec["h"]
        K = 1.0 / (r + h)
        if same_index is not None:
            K = K + spec["diag_add"] * same_index
    elif kind == "laplace":
        with np.errstate(divide="ignore"):
            K = 1.0 / (4.0 * math.pi * r)
        if same_index is not None:
            K = np.where(same_index, 1.0 / (4.0 * math.pi * spec["h"]), K)
    elif kind == "ifmm":
        K = _ifmm(r, spec["d"])
        if same_index is not None:
            K = np.where(same_index, 1.0, K)
    else:
        raise ValueError(kind)
    return K


def _ifmm(r: np.ndarray, d: float) -> np.ndarray:
    """The interaction matrix of the paper's preconditioning example (Example
    "mat1"): A_ij = 1 if i == j, |r_i - r_j| / d if 0 < |r_i - r_j| < d,
    d / |r_i - r_j| otherwise (the i == j case is applied by the caller, by index)."""
    with np.errstate(divide="ignore"):
        return np.where(r < d, r / d, d / np.maximum(r, 1e-300))


def _kernel_spec(cfg: dict, N: int) -> dict:
    k = dict(cfg["kernel"])
    if k["kind"] == "invh":
        k["h"] = N ** (-1.0 / 3.0)
    if k["kind"] == "laplace":
        k["h"] = math.sqrt(4.0 * math.pi / N)
    return k


CONFIGS: Dict[int, dict] = {
    1: dict(N=2048, points="square", kernel=dict(kind="exp", ell=0.1, nugget=1e-2), B=32, r=8, eta=0.7,
            symmetric=True, method="svd"),
    2: dict(N=65536, points="square", kernel=dict(kind="exp", ell=0.1, nugget=1e-2), B=64, r=16, eta=0.7,
            symmetric=True, method="cheb"),
    3: dict(N=262144, points="cube", kernel=dict(kind="invh", diag_add=1.0), B=64, r=24, eta=0.7,
            symmetric=True, method="cheb"),
    4: dict(N=1048576, points="sphere", kernel=dict(kind="laplace"), B=64, r=32, eta=0.7,
            symmetric=False, method="cheb", orthonormalize=True),
    5: dict(N=4194304, points="cube", kernel=dict(kind="exp", ell=0.05, nugget=1e-2), B=128, r=32, eta=0.7,
            symmetric=True, method="cheb"),
}


# ----------------------------------------------------------------------------
# Nested bases by Chebyshev interpolation (configs 2-5)
# ----------------------------------------------------------------------------

_ORDERS = {(2, 8): (4, 2), (2, 16): (4, 4), (2, 4): (2, 2), (3, 24): (4, 3, 2), (3, 32): (4, 4, 2),
           (3, 8): (2, 2, 2), (3, 16): (4, 2, 2)}


def _orders(d: int, r: int, extent: np.ndarray) -> Tuple[int, ...]:
    base = _ORDERS.get((d, r))
    if base is None:
        raise ValueError(f"no tensor order table for d={d}, r={r}")
    out = [0] * d
    for ax, p in zip(np.argsort(-extent, kind="stable"), base):
        out[int(ax)] = p
    return tuple(out)


def _cheb_nodes(lo: float, hi: float, p: int, kind: int) -> np.ndarray:
    j = np.arange(p)
    if p == 1:
        return np.array([(lo + hi) / 2])
    if kind == 1:   # Chebyshev points of the first kind
        c = np.cos((2 * j + 1) * math.pi / (2 * p))
    else:           # shifted variant for independent column bases (config 4)
        c = np.cos((2 * j + 1.5) * math.pi / (2 * p + 1))
    return (lo + hi) / 2 + (hi - lo) / 2 * c


def _lagrange(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """ell_j(x_i) for 1-D nodes -> [len(x), p]."""
    p = len(nodes)
    out = np.ones((len(x), p))
    for j in range(p):
        for m in range(p):
            if m != j:
                out[:, j] *= (x - nodes[m]) / (nodes[j] - nodes[m])
    return out


def cheb_cos_table(kind: int) -> np.ndarray:
    """[(p - 1) * 8 + j] = the Chebyshev cosine _cheb_nodes uses for order p
    (1..8), node j -- the same numpy expression, so a device construction fed
    with it reproduces the generator's nodes bit for bit (layout only)."""
    out = np.zeros(64)
    for p in range(1, 9):
        j = np.arange(p)
        if kind == 1:
            c = np.cos((2 * j + 1) * math.pi / (2 * p))
        else:
            c = np.cos((2 * j + 1.5) * math.pi / (2 * p + 1))
        out[(p - 1) * 8:(p - 1) * 8 + p] = c
    return out


def cheb_base_orders(d: int, r: int) -> Tuple[int, ...]:
    """Tensor orders of a rank-r cluster, largest-extent axis first."""
    base = _ORDERS.get((d, r))
    if base is None:
        raise ValueError(f"no tensor order table for d={d}, r={r}")
    return tuple(base)


class _ChebCluster:
    def __init__(self, lo, hi, r, kind):
        d = len(lo)
        ext = hi - lo
        pad = np.maximum(ext * 1e-9, 1e-12)
        self.lo, self.hi = lo - pad, hi + pad
        self.ords = _orders(d, r, ext)
        self.axis_nodes = [_cheb_nodes(self.lo[a], self.hi[a], self.ords[a], kind) for a in range(d)]
        grids = np.meshgrid(*self.axis_nodes, indexing="ij")
        self.nodes = np.stack([g.ravel() for g in grids], axis=1)      # [r, d]

    def basis(self, x: np.ndarray) -> np.ndarray:
        """Tensor Lagrange basis at points x -> [len(x), r] (row-major multi-index)."""
        out = None
        for a, nodes in enumerate(self.axis_nodes):
            la = _lagrange(nodes, x[:, a])
            out = la if out is None else (out[:, :, None] * la[:, None, :]).reshape(len(x), -1)
        return out


# ----------------------------------------------------------------------------
# Builders
# ----------------------------------------------------------------------------

def _pairs_same(near0):
    return near0[:, 0] == near0[:, 1]


def make_config(idx: int, seed: Optional[int] = None, N: Optional[int] = None, method: Optional[str] = None,
                with_close: bool = True, with_couplings: bool = True, orthonormalize: Optional[bool] = None) -> H2Input:
    """BASELINE.json ``configs[idx-1]`` with ``seed = idx`` (reading 17).  ``N``
    may be overridden to make smaller instances of the same recipe."""
    cfg = CONFIGS[idx]
    N = N or cfg["N"]
    seed = idx if seed is None else seed
    rng = np.random.default_rng(seed)
    B, r, eta, sym = cfg["B"], cfg["r"], cfg["eta"], cfg["symmetric"]
    L = int(round(math.log2(N // B)))
    assert B << L == N
    pts = make_points(cfg["points"], N, rng)
    perm, lo, hi = kd_tree(pts, L)
    x = pts[perm]
    near0, adm = block_tree(lo, hi, L, eta)
    kspec = _kernel_spec(cfg, N)
    meth = method or cfg["method"]
    if meth == "svd":
        h2 = _svd_h2(x, L, B, r, near0, adm, kspec, sym)
    else:
        h2 = _cheb_h2(x, L, B, r, near0, adm, kspec, lo, hi, sym, with_close, with_couplings)
        h2.meta.update(box_lo=lo, box_hi=hi, r=r, dim=x.shape[1])
        if cfg.get("orthonormalize") if orthonormalize is None else orthonormalize:
            orthonormalize_h2(h2)
    h2.meta.update(config=idx, seed=seed, N=N, eta=eta, method=meth, kernel=kspec)
    return h2


def make_ifmm(N: int, d: float, B: int, r: int, seed: int = 53, eta: float = 0.7) -> H2Input:
    """H^2 input of the paper's preconditioning example (DESIGN.md
    §9e): N uniform points in the unit cube (3-D, "randomly distributed 3D
    data"), kernel of Example mat1 with parameter d, nested Chebyshev
    bases of rank r (the tensor orders of _ORDERS[(3, r)]) and leaves of B
    points, symmetric.  The operator of GMRES and the H^2 matrix behind the
    preconditioner are two such inputs on the same points with different r (the
    paper's eps = 1e-9 and 1e-3 approximations, reading 26)."""
    rng = np.random.default_rng(seed)
    L = int(round(math.log2(N // B)))
    assert B << L == N
    pts = make_points("cube", N, rng)
    perm, lo, hi = kd_tree(pts, L)
    x = pts[perm]
    near0, adm = block_tree(lo, hi, L, eta)
    kspec = dict(kind="ifmm", d=float(d))
    h2 = _cheb_h2(x, L, B, r, near0, adm, kspec, lo, hi, True)
    h2.meta.update(box_lo=lo, box_hi=hi, r=r, dim=3, config="ifmm", seed=seed, N=N, eta=eta, method="cheb",
                   kernel=kspec)
    return h2


def random_sparse(nb: int, bs: int, seed: int, density: float = 0.2, decay: float = 2.0, shift: float = 1.0,
                  symmetric_pattern: bool = True):
    """Seeded block-sparse test matrix in CSR (rowptr int64, col int32 ascending,
    val float64) for the ILUt parity tests: nb x nb blocks of bs x bs, block
    (I, J) present with probability `density` (always for I == J; mirrored when
    `symmetric_pattern`), entries N(0, 1) * exp(-|I - J| / decay), and the
    diagonal raised by `shift` times the row's absolute sum (shift >= 1:
    diagonally dominant, no zero pivot).  Shapes only -- no method arithmetic."""
    rng = np.random.default_rng(seed)
    P = rng.random((nb, nb)) < density
    if symmetric_pattern:
        P = P | P.T
    np.fill_diagonal(P, True)
    n = nb * bs
    rows, cols, vals = [], [], []
    for I in range(nb):
        Js = np.nonzero(P[I])[0]
        blk = rng.standard_normal((bs, len(Js) * bs)) * np.repeat(np.exp(-np.abs(Js - I) / decay), bs)[None, :]
        c = (Js[:, None] * bs + np.arange(bs)[None, :]).ravel()
        for a in range(bs):
            i = I * bs + a
            v = blk[a].copy()
            dpos = np.nonzero(c == i)[0][0]
            v[dpos] = 0.0
            v[dpos] = shift * np.abs(v).sum() + 1.0
            rows.append(np.full(len(c), i))
            cols.append(c)
            vals.append(v)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum([len(c) for c in cols])
    return rowptr, np.concatenate(cols).astype(np.int32), np.concatenate(vals)


def make_structure(idx: int, seed: Optional[int] = None, N: Optional[int] = None) -> H2Input:
    """The STRUCTURE of BASELINE.json ``configs[idx-1]`` only -- tree-ordered
    points, cluster boxes, block cluster tree and ranks, no numeric arrays --
    for instances whose bases / couplings / close blocks are built on the device
    (config 5 at full size: 130 GB of couplings and 980 GB of close blocks are
    never materialised).  Same seed, tree and ranks as make_config."""
    cfg = CONFIGS[idx]
    N = N or cfg["N"]
    seed = idx if seed is None else seed
    rng = np.random.default_rng(seed)
    B, r, eta, sym = cfg["B"], cfg["r"], cfg["eta"], cfg["symmetric"]
    L = int(round(math.log2(N // B)))
    assert B << L == N
    pts = make_points(cfg["points"], N, rng)
    perm, lo, hi = kd_tree(pts, L)
    x = np.ascontiguousarray(pts[perm])
    del pts
    near0, adm = block_tree(lo, hi, L, eta)
    rank_row = far_ranks(L, near0, adm, r, r, 0)
    rank_col = far_ranks(L, near0, adm, r, r, 1)
    if sym:
        rank_row = rank_col = np.maximum(rank_row, rank_col)
    h2 = H2Input(L=L, B=B, symmetric=sym, rank_row=rank_row, rank_col=rank_col, leaf_row=None, leaf_col=None,
                 transfer_row=None, transfer_col=None, near=near0, close=None, adm=adm, coupling=None, points=x)
    h2.meta.update(config=idx, seed=seed, N=N, eta=eta, method="cheb", kernel=_kernel_spec(cfg, N), box_lo=lo,
                   box_hi=hi, r=r, dim=x.shape[1], structure_only=True)
    return h2


def _close_blocks(x, B, near0, kspec):
    nn = len(near0)
    out = np.empty((nn, B, B))
    eye = np.eye(B, dtype=bool)
    chunk = max(1, (1 << 22) // (B * B))
    for c0 in range(0, nn, chunk):
        sl = near0[c0:c0 + chunk]
        xt = x.reshape(-1, B, x.shape[1])[sl[:, 0]]
        xs = x.reshape(-1, B, x.shape[1])[sl[:, 1]]
        diff = xt[:, :, None, :] - xs[:, None, :, :]
        rr = np.sqrt(np.einsum("pijk,pijk->pij", diff, diff))
        same = (sl[:, 0] == sl[:, 1])[:, None, None] & eye[None]
        kind = kspec["kind"]
        if kind == "exp":
            K = np.exp(-rr / kspec["ell"]) + kspec["nugget"] * same
        elif kind == "invh":
            K = 1.0 / (rr + kspec["h"]) + kspec["diag_add"] * same
        elif kind == "laplace":
            with np.errstate(divide="ignore"):
                K = 1.0 / (4.0 * math.pi * rr)
            K = np.where(same, 1.0 / (4.0 * math.pi * kspec["h"]), K)
        elif kind == "ifmm":
            K = np.where(same, 1.0, _ifmm(rr, kspec["d"]))
        out[c0:c0 + chunk] = K
    return out


def _mirror_close(near0, close):
    """Symmetric mode: make C_st = C_ts^T bitwise."""
    key = {(int(t), int(s)): i for i, (t, s) in enumerate(near0)}
    for i, (t, s) in enumerate(near0):
        if t > s:
            close[i] = close[key[(int(s), int(t))]].T
        elif t == s:
            c = close[i]
            close[i] = np.triu(c) + np.triu(c, 1).T
    return close


def _cheb_side(x, L, B, rank, lo, hi, kind):
    """Chebyshev clusters, leaf bases and transfers of one side."""
    ncl = n_clusters(L)
    cl = [None] * ncl
    for c in range(ncl):
        if rank[c] > 0:
            cl[c] = _ChebCluster(lo[c], hi[c], int(rank[c]), kind)
    leaf = []
    for i in range(1 << L):
        c = cid(L, 0, i)
        if rank[c] > 0:
            leaf.append(cl[c].basis(x[i * B:(i + 1) * B]))
        else:
            leaf.append(np.zeros((B, 0)))
    transfer: List[Optional[np.ndarray]] = [None] * ncl
    for k in range(1, L + 1):
        for i in range(1 << (L - k)):
            p = cid(L, k, i)
            c1, c2 = cid(L, k - 1, 2 * i), cid(L, k - 1, 2 * i + 1)
            rows = []
            for c in (c1, c2):
                kc = int(rank[c])
                if rank[p] > 0 and kc > 0:
                    rows.append(cl[p].basis(cl[c].nodes))
                else:
                    rows.append(np.zeros((kc, int(rank[p]))))
            transfer[p] = np.vstack(rows)
    return cl, leaf, transfer


def fill_cheb_bases(h2: H2Input) -> H2Input:
    """Numeric nested bases of a structure-only input (make_structure) with the
    same Chebyshev recipe as make_config -- for the oracle's checks on instances
    whose close blocks / couplings stay matrix-free (config 5 at full size).
    Couplings and close blocks are not built (evaluate them from the points /
    nodes, meta cheb_nodes_*)."""
    x, L, B = h2.points, h2.L, h2.B
    lo, hi = h2.meta["box_lo"], h2.meta["box_hi"]
    clr, h2.leaf_row, h2.transfer_row = _cheb_side(x, L, B, h2.rank_row, lo, hi, 1)
    if h2.symmetric:
        clc, h2.leaf_col, h2.transfer_col = clr, h2.leaf_row, h2.transfer_row
    else:
        clc, h2.leaf_col, h2.transfer_col = _cheb_side(x, L, B, h2.rank_col, lo, hi, 2)
    h2.meta["cheb_nodes_row"] = [c.nodes if c is not None else None for c in clr]
    h2.meta["cheb_nodes_col"] = [c.nodes if c is not None else None for c in clc]
    return h2


def _cheb_h2(x, L, B, r, near0, adm, kspec, lo, hi, sym, with_close=True, with_couplings=True) -> H2Input:
    ncl = n_clusters(L)
    rank_row = far_ranks(L, near0, adm, r, r, 0)
    rank_col = far_ranks(L, near0, adm, r, r, 1)
    if sym:
        rank = np.maximum(rank_row, rank_col)
        rank_row = rank_col = rank

    clr, leaf_row, tr_row = _cheb_side(x, L, B, rank_row, lo, hi, 1)
    if sym:
        clc, leaf_col, tr_col = clr, leaf_row, tr_row
    else:
        clc, leaf_col, tr_col = _cheb_side(x, L, B, rank_col, lo, hi, 2)
    coupling = [] if with_couplings else None
    for k in range(L if with_couplings else 0):
        lst = []
        base = lvl_off(L, k)
        for (t, s) in adm[k]:
            a, b = clr[base + t], clc[base + s]
            D = kernel_matrix(kspec, a.nodes, b.nodes)
            lst.append(D)
        if sym:
            key = {(int(t), int(s)): i for i, (t, s) in enumerate(adm[k])}
            for i, (t, s) in enumerate(adm[k]):
                if t > s:
                    lst[i] = lst[key[(int(s), int(t))]].T.copy()
        coupling.append(lst)
    close = _close_blocks(x, B, near0, kspec) if with_close else None
    if sym and close is not None:
        close = _mirror_close(near0, close)
    h2 = H2Input(L=L, B=B, symmetric=sym, rank_row=rank_row, rank_col=rank_col, leaf_row=leaf_row,
                 leaf_col=leaf_col, transfer_row=tr_row, transfer_col=tr_col, near=near0, close=close,
                 adm=adm, coupling=coupling, points=x)
    # interpolation nodes of every cluster (None where rank 0): the couplings are
    # D_b = K(nodes_t, nodes_s), so they can also be evaluated on the device
    h2.meta["cheb_nodes_row"] = [c.nodes if c is not None else None for c in clr]
    h2.meta["cheb_nodes_col"] = [c.nodes if c is not None else None for c in clc]
    return h2


def coupling_block_descs(h2: H2Input):
    """Layout of the couplings as kernel blocks (pure data movement, no kernel
    arithmetic): flat row / column node arrays, and per admissible pair in the
    `coupling` input order (level-major, CSR by row cluster) the int64 record
    (x_off, y_off, out_off, nx | ny << 32) of include/h2sp.h h2sp_block_desc.
    Needs a Chebyshev-built H2Input (meta cheb_nodes_*)."""
    L = h2.L

    def flat(nodes):
        offs = np.zeros(len(nodes), dtype=np.int64)
        parts, o = [], 0
        for c, nd in enumerate(nodes):
            offs[c] = o
            if nd is not None:
                parts.append(nd)
                o += len(nd)
        d = parts[0].shape[1] if parts else 1
        return (np.ascontiguousarray(np.concatenate(parts), dtype=np.float64) if parts else np.zeros((0, d))), offs

    xr, offr = flat(h2.meta["cheb_nodes_row"])
    xc, offc = flat(h2.meta["cheb_nodes_col"])
    rec = []
    out = 0
    for k in range(L):
        base = lvl_off(L, k)
        for (t, s) in h2.adm[k]:
            ct, cs = base + int(t), base + int(s)
            nx, ny = int(h2.rank_row[ct]), int(h2.rank_col[cs])
            rec.append((offr[ct], offc[cs], out, nx | (ny << 32)))
            out += nx * ny
    desc = np.array(rec, dtype=np.int64).reshape(-1, 4)
    return xr, xc, desc, out


def _svd_h2(x, L, B, r, near0, adm, kspec, sym) -> H2Input:
    """Config 1: exact SVD recompression from the dense kernel matrix
    (SURVEY §8(d) generator; nested orthonormal bases of rank exactly r)."""
    N = x.shape[0]
    A = kernel_matrix(kspec, x, x, np.eye(N, dtype=bool))
    ncl = n_clusters(L)
    rank = far_ranks(L, near0, adm, r, r, 0)
    rank_c = far_ranks(L, near0, adm, r, r, 1)
    rank = np.maximum(rank, rank_c)
    # Far*(t): union of column index sets of admissible blocks at t or ancestors
    far_cols = [np.zeros(N, dtype=bool) for _ in range(ncl)]
    for k in range(L):
        base = lvl_off(L, k)
        sz = B << k
        for (t, s) in adm[k]:
            far_cols[base + t][s * sz:(s + 1) * sz] = True
    for k in range(L - 1, -1, -1):
        base, pbase = lvl_off(L, k), lvl_off(L, k + 1)
        for i in range(1 << (L - k)):
            far_cols[base + i] |= far_cols[pbase + i // 2]
    W = [None] * ncl        # effective orthonormal basis (|t| x k)
    leaf = []
    transfer: List[Optional[np.ndarray]] = [None] * ncl
    for i in range(1 << L):
        c = cid(L, 0, i)
        k_ = int(rank[c])
        blk = A[i * B:(i + 1) * B][:, far_cols[c]]
        if k_ > 0:
            u = np.linalg.svd(blk, full_matrices=True)[0][:, :k_]
        else:
            u = np.zeros((B, 0))
        leaf.append(u)
        W[c] = u
    for k in range(1, L + 1):
        sz = B << k
        for i in range(1 << (L - k)):
            p = cid(L, k, i)
            c1, c2 = cid(L, k - 1, 2 * i), cid(L, k - 1, 2 * i + 1)
            k_ = int(rank[p])
            Wc = np.zeros((sz, W[c1].shape[1] + W[c2].shape[1]))
            Wc[:sz // 2, :W[c1].shape[1]] = W[c1]
            Wc[sz // 2:, W[c1].shape[1]:] = W[c2]
            if k_ > 0:
                blk = Wc.T @ A[i * sz:(i + 1) * sz][:, far_cols[p]]
                t_ = np.linalg.svd(blk, full_matrices=True)[0][:, :k_]
            else:
                t_ = np.zeros((Wc.shape[1], 0))
            transfer[p] = t_
            W[p] = Wc @ t_
    coupling = []
    for k in range(L):
        base = lvl_off(L, k)
        sz = B << k
        lst = []
        for (t, s) in adm[k]:
            lst.append(W[base + t].T @ A[t * sz:(t + 1) * sz, s * sz:(s + 1) * sz] @ W[base + s])
        key = {(int(t), int(s)): i for i, (t, s) in enumerate(adm[k])}
        for i, (t, s) in enumerate(adm[k]):
            if t > s:
                lst[i] = lst[key[(int(s), int(t))]].T.copy()
        coupling.append(lst)
    close = np.stack([A[t * B:(t + 1) * B, s * B:(s + 1) * B] for (t, s) in near0])
    close = _mirror_close(near0, close)
    return H2Input(L=L, B=B, symmetric=sym, rank_row=rank, rank_col=rank, leaf_row=leaf, leaf_col=leaf,
                   transfer_row=transfer, transfer_col=transfer, near=near0, close=close, adm=adm,
                   coupling=coupling, points=x)


def orthonormalize_h2(h2: H2Input) -> H2Input:
    """Rewrite the H^2 parameters with orthonormal nested bases of the SAME rank
    (SVD-based H^2 orthogonalisation, bottom-up): R_t = W_t Z_t, transfers
    T'_p = U_p from [Z_c1 T_p^(1); Z_c2 T_p^(2)] = U_p Z_p, couplings
    D' = Z_t D Z_s^T.  The represented matrix is unchanged in exact arithmetic;
    3-D tensor interpolation restricted to a surface (config 4) gives
    numerically rank-deficient bases (cond ~1e8) whose Householder complement
    is ill-determined, orthonormal bases are perfectly conditioned."""
    L = h2.L
    ncl = n_clusters(L)

    def side(leaf, tr, rank):
        Z = [None] * ncl
        new_leaf, new_tr = [], [None] * ncl
        for i in range(1 << L):
            R = np.asarray(leaf[i])
            if R.shape[1]:
                U, S, Vt = np.linalg.svd(R, full_matrices=False)
                new_leaf.append(U)
                Z[cid(L, 0, i)] = S[:, None] * Vt
            else:
                new_leaf.append(R.copy())
                Z[cid(L, 0, i)] = np.zeros((0, 0))
        for k in range(1, L + 1):
            for i in range(1 << (L - k)):
                p = cid(L, k, i)
                c1, c2 = cid(L, k - 1, 2 * i), cid(L, k - 1, 2 * i + 1)
                T = tr[p]
                k1 = int(rank[c1])
                X = np.vstack([Z[c1] @ T[:k1], Z[c2] @ T[k1:]])
                if X.shape[1]:
                    U, S, Vt = np.linalg.svd(X, full_matrices=False)
                    new_tr[p] = U
                    Z[p] = S[:, None] * Vt
                else:
                    new_tr[p] = X.copy()
                    Z[p] = np.zeros((0, 0))
        return new_leaf, new_tr, Z

    lr, tr_r, Zr = side(h2.leaf_row, h2.transfer_row, h2.rank_row)
    if h2.symmetric:
        lc, tr_c, Zc = lr, tr_r, Zr
    else:
        lc, tr_c, Zc = side(h2.leaf_col, h2.transfer_col, h2.rank_col)
    for k in range(L):
        base = lvl_off(L, k)
        for j, (t, s) in enumerate(h2.adm[k]):
            h2.coupling[k][j] = Zr[base + int(t)] @ h2.coupling[k][j] @ Zc[base + int(s)].T
        if h2.symmetric:
            key = {(int(t), int(s)): j for j, (t, s) in enumerate(h2.adm[k])}
            for j, (t, s) in enumerate(h2.adm[k]):
                if t > s:
                    h2.coupling[k][j] = h2.coupling[k][key[(int(s), int(t))]].T.copy()
    h2.leaf_row, h2.transfer_row, h2.leaf_col, h2.transfer_col = lr, tr_r, lc, tr_c
    h2.meta["orthonormalized"] = True
    return h2


def _random_ranks(L, B, rng, lo_frac=0.0, hi_frac=1.0, zero_prob=0.15, full_prob=0.1, max_rank=None):
    ncl = n_clusters(L)
    rank = np.zeros(ncl, dtype=np.int32)
    nloc = np.zeros(ncl, dtype=np.int64)
    for k in range(L + 1):
        for i in range(1 << (L - k)):
            c = cid(L, k, i)
            if k == 0:
                n = B
            else:
                n = rank[cid(L, k - 1, 2 * i)] + rank[cid(L, k - 1, 2 * i + 1)]
            nloc[c] = n
            u = rng.random()
            if k == L:
                kk = 0
            elif u < zero_prob:
                kk = 0
            elif u < zero_prob + full_prob:
                kk = n
            else:
                kk = int(rng.integers(int(lo_frac * n), int(hi_frac * n) + 1)) if n > 0 else 0
            if max_rank is not None:
                kk = min(kk, max_rank)
            rank[c] = kk
    return rank


def random_h2(L: int, B: int, seed: int, symmetric: bool, eta: float = 0.7, d: int = 2, spd_shift: float = 0.0,
              ragged: bool = True, r: int = None, max_rank: int = None) -> H2Input:
    """Random H^2 matrix on a KD tree of random points: Gaussian bases,
    transfers, couplings and close blocks; ragged per-cluster ranks (including
    k=0, k=n and n=0 clusters) when ``ragged``.  ``spd_shift`` is added to the
    diagonal of the diagonal close blocks (symmetric mode) to make A_H2 SPD."""
    rng = np.random.default_rng(seed)
    N = B << L
    pts = rng.random((N, d))
    perm, lo, hi = kd_tree(pts, L)
    near0, adm = block_tree(lo, hi, L, eta)
    ncl = n_clusters(L)
    if ragged:
        rank_row = _random_ranks(L, B, rng, max_rank=max_rank)
        rank_col = rank_row if symmetric else _random_ranks(L, B, rng, max_rank=max_rank)
    else:
        rr = r if r is not None else max(1, B // 4)
        rank_row = far_ranks(L, near0, adm, rr, rr, 0)
        rank_col = far_ranks(L, near0, adm, rr, rr, 1)
        if symmetric:
            rank_row = rank_col = np.maximum(rank_row, rank_col)

    def bases(rank):
        leaf = [rng.standard_normal((B, int(rank[cid(L, 0, i)]))) for i in range(1 << L)]
        tr: List[Optional[np.ndarray]] = [None] * ncl
        for k in range(1, L + 1):
            for i in range(1 << (L - k)):
                p = cid(L, k, i)
                n = int(rank[cid(L, k - 1, 2 * i)] + rank[cid(L, k - 1, 2 * i + 1)])
                tr[p] = rng.standard_normal((n, int(rank[p])))
        return leaf, tr

    leaf_row, tr_row = bases(rank_row)
    if symmetric:
        leaf_col, tr_col = leaf_row, tr_row
    else:
        leaf_col, tr_col = bases(rank_col)
    coupling = []
    for k in range(L):
        base = lvl_off(L, k)
        lst = [rng.standard_normal((int(rank_row[base + t]), int(rank_col[base + s]))) for (t, s) in adm[k]]
        if symmetric:
            key = {(int(t), int(s)): i for i, (t, s) in enumerate(adm[k])}
            for i, (t, s) in enumerate(adm[k]):
                if t > s:
                    lst[i] = lst[key[(int(s), int(t))]].T.copy()
        coupling.append(lst)
    close = rng.standard_normal((len(near0), B, B))
    if symmetric:
        close = _mirror_close(near0, close)
        if spd_shift:
            for i, (t, s) in enumerate(near0):
                if t == s:
                    close[i] += spd_shift * np.eye(B)
    return H2Input(L=L, B=B, symmetric=symmetric, rank_row=rank_row, rank_col=rank_col, leaf_row=leaf_row,
                   leaf_col=leaf_col, transfer_row=tr_row, transfer_col=tr_col, near=near0, close=close,
                   adm=adm, coupling=coupling, points=pts[perm], meta=dict(seed=seed, eta=eta, random=True))


def structure_h2(L: int, B: int, near0: np.ndarray, adm: List[np.ndarray], rank_row, rank_col, seed: int,
                 symmetric: bool) -> H2Input:
    """Random values on a GIVEN block structure and rank distribution."""
    rng = np.random.default_rng(seed)
    ncl = n_clusters(L)
    rank_row = np.asarray(rank_row, dtype=np.int32)
    rank_col = np.asarray(rank_col, dtype=np.int32)

    def bases(rank):
        leaf = [rng.standard_normal((B, int(rank[cid(L, 0, i)]))) for i in range(1 << L)]
        tr: List[Optional[np.ndarray]] = [None] * ncl
        for k in range(1, L + 1):
            for i in range(1 << (L - k)):
                p = cid(L, k, i)
                n = int(rank[cid(L, k - 1, 2 * i)] + rank[cid(L, k - 1, 2 * i + 1)])
                tr[p] = rng.standard_normal((n, int(rank[p])))
        return leaf, tr

    leaf_row, tr_row = bases(rank_row)
    leaf_col, tr_col = (leaf_row, tr_row) if symmetric else bases(rank_col)
    coupling = []
    for k in range(L):
        base = lvl_off(L, k)
        lst = [rng.standard_normal((int(rank_row[base + t]), int(rank_col[base + s]))) for (t, s) in adm[k]]
        if symmetric:
            key = {(int(t), int(s)): i for i, (t, s) in enumerate(adm[k])}
            for i, (t, s) in enumerate(adm[k]):
                if t > s:
                    lst[i] = lst[key[(int(s), int(t))]].T.copy()
        coupling.append(lst)
    close = rng.standard_normal((len(near0), B, B))
    if symmetric:
        close = _mirror_close(near0, close)
    return H2Input(L=L, B=B, symmetric=symmetric, rank_row=rank_row, rank_col=rank_col, leaf_row=leaf_row,
                   leaf_col=leaf_col, transfer_row=tr_row, transfer_col=tr_col, near=near0, close=close,
                   adm=adm, coupling=coupling, meta=dict(seed=seed))


def fig3_structure():
    """The paper's Fig. 1 / Fig. 3 example: M = 8 leaves,
    C_0 = diagonal + blocks (2,4), (4,2) (0-based, read off the TikZ
    coordinates), all other level-0 blocks far.  Returns (L, near0, adm)."""
    L = 3
    near = [(i, i) for i in range(8)] + [(2, 4), (4, 2)]
    near0 = np.array(sorted(near), dtype=np.int32)
    nearset = set(near)
    n1 = sorted({(t // 2, s // 2) for (t, s) in near})
    adm0 = sorted((2 * p + a, 2 * q + b) for (p, q) in n1 for a in range(2) for b in range(2)
                  if (2 * p + a, 2 * q + b) not in nearset)
    adm1 = sorted((p, q) for p in range(4) for q in range(4) if (p, q) not in set(n1))
    adm = [np.array(adm0, dtype=np.int32).reshape(-1, 2), np.array(adm1, dtype=np.int32).reshape(-1, 2),
           np.zeros((0, 2), dtype=np.int32)]
    return L, near0, adm


def fig3_h2(B: int = 4, seed: int = 0, rank_mode: str = "half", symmetric: bool = True) -> H2Input:
    """Fig. 3 structure with random values.  ``rank_mode='half'``: every
    non-root cluster has rank r = B/2 (the §3 Proposition's hypothesis);
    ``'active'``: rank B/2 only where an admissible pair lies at or above."""
    L, near0, adm = fig3_structure()
    ncl = n_clusters(L)
    if rank_mode == "half":
        rank = np.full(ncl, B // 2, dtype=np.int32)
        rank[ncl - 1] = 0
    else:
        rank = far_ranks(L, near0, adm, B // 2, B // 2, 0)
        rank = np.maximum(rank, far_ranks(L, near0, adm, B // 2, B // 2, 1))
    return structure_h2(L, B, near0, adm, rank, rank, seed, symmetric)


def eta0_h2(L: int, B: int, seed: int, symmetric: bool = True) -> H2Input:
    """eta = 0: no admissible block, all ranks 0 (pin P7)."""
    near0 = np.array([(t, s) for t in range(1 << L) for s in range(1 << L)], dtype=np.int32)
    adm = [np.zeros((0, 2), dtype=np.int32) for _ in range(L)]
    z = np.zeros(n_clusters(L), dtype=np.int32)
    return structure_h2(L, B, near0, adm, z, z, seed, symmetric)


def axis_aligned_h2(L: int, B: int, seed: int, symmetric: bool, eta: float = 0.7) -> H2Input:
    """Pin P8: leaf bases are signed columns of I_B in diagonal position
    (R_t = [diag(+-1); 0]) and transfers are [I; 0]-type selections with signs,
    so every Householder step sees sigma == 0 exactly and every Q = I; the
    whole cascade is then exact (no rounding) and S = P^T A_H2 P bitwise."""
    rng = np.random.default_rng(seed)
    N = B << L
    pts = rng.random((N, 2))
    perm, lo, hi = kd_tree(pts, L)
    near0, adm = block_tree(lo, hi, L, eta)
    h2 = random_h2(L, B, seed, symmetric, eta=eta, ragged=True)
    h2.near, h2.adm = near0, adm
    ncl = n_clusters(L)

    def sel(n, k):
        m = np.zeros((n, k))
        m[np.arange(k), np.arange(k)] = rng.choice([-1.0, 1.0], size=k)
        return m

    def bases(rank):
        leaf = [sel(B, int(rank[cid(L, 0, i)])) for i in range(1 << L)]
        tr: List[Optional[np.ndarray]] = [None] * ncl
        for k in range(1, L + 1):
            for i in range(1 << (L - k)):
                p = cid(L, k, i)
                n = int(rank[cid(L, k - 1, 2 * i)] + rank[cid(L, k - 1, 2 * i + 1)])
                tr[p] = sel(n, int(rank[p]))
        return leaf, tr

    h2.leaf_row, h2.transfer_row = bases(h2.rank_row)
    if symmetric:
        h2.leaf_col, h2.transfer_col = h2.leaf_row, h2.transfer_row
    else:
        h2.leaf_col, h2.transfer_col = bases(h2.rank_col)
    # integer-valued couplings/close blocks keep every product exact as well
    h2.coupling = []
    for k in range(L):
        base = lvl_off(L, k)
        lst = [rng.integers(-8, 9, size=(int(h2.rank_row[base + t]), int(h2.rank_col[base + s]))).astype(float)
               for (t, s) in adm[k]]
        if symmetric:
            key = {(int(t), int(s)): i for i, (t, s) in enumerate(adm[k])}
            for i, (t, s) in enumerate(adm[k]):
                if t > s:
                    lst[i] = lst[key[(int(s), int(t))]].T.copy()
        h2.coupling.append(lst)
    close = rng.integers(-8, 9, size=(len(near0), B, B)).astype(float)
    h2.close = _mirror_close(near0, close) if symmetric else close
    h2.meta = dict(seed=seed, eta=eta, axis_aligned=True)
    return h2


# ----------------------------------------------------------------------------
# Flat packing for the C ABI (include/h2sp.h): layout only, no arithmetic
# ----------------------------------------------------------------------------

def pack(h2: H2Input) -> dict:
    """Flatten to the ABI layout: CSR near/adm lists, concatenated row-major
    leaf bases / transfers / couplings.  Pure data movement."""
    L = h2.L
    nl = 1 << L
    near_ptr = np.zeros(nl + 1, dtype=np.int64)
    np.add.at(near_ptr, h2.near[:, 0].astype(np.int64) + 1, 1)
    near_ptr = np.cumsum(near_ptr)
    near_col = np.ascontiguousarray(h2.near[:, 1], dtype=np.int32)
    adm_ptr, adm_col = [], []
    for k in range(L):
        M = 1 << (L - k)
        p = np.zeros(M + 1, dtype=np.int64)
        a = h2.adm[k]
        if len(a):
            np.add.at(p, a[:, 0].astype(np.int64) + 1, 1)
        adm_ptr.append(np.cumsum(p))
        adm_col.append(np.ascontiguousarray(a[:, 1] if len(a) else np.zeros(0), dtype=np.int32))

    def cat(mats):
        if mats is None:
            return None
        mats = [m for m in mats if m is not None]
        if not mats:
            return np.zeros(0)
        return np.concatenate([np.ascontiguousarray(m, dtype=np.float64).ravel() for m in mats])

    ncl = n_clusters(L)
    out = dict(
        L=L, B=h2.B, symmetric=int(h2.symmetric),
        rank_row=np.ascontiguousarray(h2.rank_row, dtype=np.int32),
        rank_col=np.ascontiguousarray(h2.rank_col, dtype=np.int32),
        near_ptr=near_ptr, near_col=near_col, adm_ptr=adm_ptr, adm_col=adm_col,
        leaf_row=cat(h2.leaf_row),
        transfer_row=cat([h2.transfer_row[c] for c in range(ncl)]) if h2.transfer_row is not None else None,
        leaf_col=cat(h2.leaf_col),
        transfer_col=cat([h2.transfer_col[c] for c in range(ncl)]) if h2.transfer_col is not None else None,
        close=np.ascontiguousarray(h2.close, dtype=np.float64).ravel() if h2.close is not None else None,
        coupling=cat([m for lst in h2.coupling for m in lst]) if h2.coupling is not None else None,
    )
    return out
