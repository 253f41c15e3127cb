"""Algorithm 1 of the paper for a dense matrix (PAPER.md
"Compression algorithm"): the input is a dense A with H^2 structure
 given on the device in cluster-tree order, together with its block
cluster tree; the compression step computes every level's bases from the SVD
of the block rows (row side) / block columns (column side) restricted to the
far field -- the blocks of A that the near part of that level does not cover --
and this package's sparsification (`h2sp_build`, unchanged) then forms
U S V^T level by level exactly as for a given H^2 matrix.

Reading: the paper's U_ki comes from "the SVD of the i-th block
row of A_{b_k b_k}" of the current level's matrix; with nested bases this is
the SVD of the leaf's far-field block row at level 0 and of the children's
projected far-field block row at level k >= 1 (the projection by the
children's bases is what A_{k+1} = U_k^T A_k V_k applies), truncated to rank r
where a far field exists at or above the cluster and 0 elsewhere (reading 5).
The couplings are D_b = W_t^T A_b W_s with the effective orthonormal bases W.

The SVDs and the projections are library calls (torch.linalg.svd / matmul on
the device, like cuBLAS) on the construction side; the sparsification is the
package's kernels.
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np

__all__ = ["compress_dense", "far_ranks"]


def _lvl_off(L: int, k: int) -> int:
    return (1 << (L + 1)) - (1 << (L - k + 1))


def far_ranks(L: int, adm, r: int, side: int) -> np.ndarray:
    """Rank r for every cluster with an admissible pair at or above it, 0
    elsewhere; root rank 0 (readings 4-5)."""
    ncl = (1 << (L + 1)) - 1
    has = np.zeros(ncl, dtype=bool)
    for k in range(L):
        a = np.asarray(adm[k])
        if len(a):
            has[_lvl_off(L, k) + np.unique(a[:, side])] = True
    for k in range(L - 1, -1, -1):
        base, pbase = _lvl_off(L, k), _lvl_off(L, k + 1)
        M = 1 << (L - k)
        has[base:base + M] |= has[pbase + np.arange(M) // 2]
    rank = np.where(has, r, 0).astype(np.int32)
    rank[ncl - 1] = 0
    return rank


def compress_dense(A, L: int, B: int, r: int, near0, adm, symmetric: bool = True) -> dict:
    """Compression step of Algorithm 1 on the device.  A: (N, N) float64 CUDA
    tensor (tree order, N = B 2^L); near0 (n, 2) and adm[k] (n_k, 2): the block
    cluster tree (sorted pairs).  Returns a dict with the structure arrays of
    h2gen.pack (host) and the numeric inputs as device tensors (leaf_row,
    transfer_row, coupling, close and, general mode, the column side), ready for
    `Plan(packed)` and `Sparsifier(plan, inputs=...)`."""
    import torch
    dev = A.device
    N = A.shape[0]
    if N != B << L:
        raise ValueError("A must be (B 2^L) x (B 2^L)")
    ncl = (1 << (L + 1)) - 1
    rank_r = far_ranks(L, adm, r, 0)
    rank_c = far_ranks(L, adm, r, 1)
    if symmetric:
        rank_r = rank_c = np.maximum(rank_r, rank_c)

    def side(At, rank, side_idx):
        # far field of every cluster: the admissible blocks at it or an ancestor
        far: List[np.ndarray] = [np.zeros(N, dtype=bool) for _ in range(ncl)]
        for k in range(L):
            base, sz = _lvl_off(L, k), B << k
            for (t, s) in np.asarray(adm[k]):
                own, oth = (t, s) if side_idx == 0 else (s, t)
                far[base + own][oth * sz:(oth + 1) * sz] = True
        for k in range(L - 1, -1, -1):
            base, pbase = _lvl_off(L, k), _lvl_off(L, k + 1)
            for i in range(1 << (L - k)):
                far[base + i] |= far[pbase + i // 2]
        W: List[Optional[object]] = [None] * ncl
        leaf, transfer = [], [None] * ncl
        for i in range(1 << L):
            c = _lvl_off(L, 0) + i
            k_ = int(rank[c])
            if k_ > 0:
                cols = torch.from_numpy(np.nonzero(far[c])[0]).to(dev)
                u = torch.linalg.svd(At[i * B:(i + 1) * B][:, cols], full_matrices=False)[0][:, :k_]
            else:
                u = torch.zeros(B, 0, dtype=A.dtype, device=dev)
            leaf.append(u.contiguous())
            W[c] = u
        for k in range(1, L + 1):
            sz = B << k
            for i in range(1 << (L - k)):
                p = _lvl_off(L, k) + i
                c1, c2 = _lvl_off(L, k - 1) + 2 * i, _lvl_off(L, k - 1) + 2 * i + 1
                k_ = int(rank[p])
                a, b = W[c1], W[c2]
                Wc = torch.zeros(sz, a.shape[1] + b.shape[1], dtype=A.dtype, device=dev)
                Wc[:sz // 2, :a.shape[1]] = a
                Wc[sz // 2:, a.shape[1]:] = b
                if k_ > 0:
                    cols = torch.from_numpy(np.nonzero(far[p])[0]).to(dev)
                    blk = Wc.T @ At[i * sz:(i + 1) * sz][:, cols]
                    t_ = torch.linalg.svd(blk, full_matrices=False)[0][:, :k_]
                else:
                    t_ = torch.zeros(Wc.shape[1], 0, dtype=A.dtype, device=dev)
                transfer[p] = t_.contiguous()
                W[p] = Wc @ t_
        return leaf, transfer, W

    leaf_r, tr_r, Wr = side(A, rank_r, 0)
    if symmetric:
        leaf_c, tr_c, Wc = leaf_r, tr_r, Wr
    else:
        leaf_c, tr_c, Wc = side(A.T.contiguous(), rank_c, 1)
    coup = []
    for k in range(L):
        base, sz = _lvl_off(L, k), B << k
        blocks = {}
        for (t, s) in np.asarray(adm[k]):
            if symmetric and t > s:
                continue
            blocks[(int(t), int(s))] = Wr[base + t].T @ A[t * sz:(t + 1) * sz, s * sz:(s + 1) * sz] @ Wc[base + s]
        for (t, s) in np.asarray(adm[k]):
            t, s = int(t), int(s)
            coup.append(blocks[(s, t)].T if symmetric and t > s else blocks[(t, s)])
    near0 = np.asarray(near0)
    close = torch.stack([A[t * B:(t + 1) * B, s * B:(s + 1) * B] for (t, s) in near0]) if len(near0) else None
    if symmetric and close is not None:   # C_st = C_ts^T bitwise (only t <= s is read; diagonals symmetrised)
        key = {(int(t), int(s)): j for j, (t, s) in enumerate(near0)}
        for j, (t, s) in enumerate(near0):
            if t > s:
                close[j] = close[key[(int(s), int(t))]].T
            elif t == s:
                close[j] = torch.triu(close[j]) + torch.triu(close[j], 1).T

    def cat(ms):
        ms = [m.reshape(-1) for m in ms if m is not None and m.numel()]
        return torch.cat(ms) if ms else torch.zeros(1, dtype=A.dtype, device=dev)

    nl = 1 << L
    near_ptr = np.zeros(nl + 1, dtype=np.int64)
    np.add.at(near_ptr, near0[:, 0].astype(np.int64) + 1, 1)
    adm_ptr, adm_col = [], []
    for k in range(L):
        a = np.asarray(adm[k]).reshape(-1, 2)
        p_ = np.zeros((1 << (L - k)) + 1, dtype=np.int64)
        if len(a):
            np.add.at(p_, a[:, 0].astype(np.int64) + 1, 1)
        adm_ptr.append(np.cumsum(p_))
        adm_col.append(np.ascontiguousarray(a[:, 1], dtype=np.int32))
    out = dict(L=L, B=B, symmetric=int(symmetric), rank_row=rank_r, rank_col=rank_c, near_ptr=np.cumsum(near_ptr),
               near_col=np.ascontiguousarray(near0[:, 1], dtype=np.int32), adm_ptr=adm_ptr, adm_col=adm_col)
    inputs = {"leaf_basis_row": cat(leaf_r), "transfer_row": cat([tr_r[c] for c in range(ncl)]),
              "coupling": cat(coup), "close": cat([close]) if close is not None else None}
    if not symmetric:
        inputs["leaf_basis_col"] = cat(leaf_c)
        inputs["transfer_col"] = cat([tr_c[c] for c in range(ncl)])
    out["inputs"] = inputs
    return out
