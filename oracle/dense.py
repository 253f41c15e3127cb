"""O0 -- the plain dense definitions (tiny N), and independent checks.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Nothing here is used by
the CUDA path.

  * ``dense_A``: A_H2 = sum_{N_0} C_ts + sum_k sum_{A_k} R_t D_b E_s^T with the
    nested effective bases R_p = diag(R_c1, R_c2) T_p (Def. "H^2
    matrix"; P:76-84 nested bases).
  * ``dense_U``: U with column off(k,t)+a = Phi_t Q_t[:, k_t + a] in the rows of
    cluster t, Phi_leaf = I_B, Phi_p = diag(Phi_c1 Q_c1[:, :k_c1],
    Phi_c2 Q_c2[:, :k_c2]) -- the product of the level factors P_rk U_k
    (Eq. main_uv; §4.2).
  * ``h2_matvec``: the standard upward / coupling / downward H^2 matvec
    (SPEC S:183-191), an independent route to A_H2 x at any N (pin P13).
  * ``frobenius_sq``: ||A_H2||_F^2 from the parameters via Gram matrices
    (pin P5; independent of every QR convention).
  * ``pattern_rule``: the closed-form symbolic pattern of S (pin P10).
"""
from __future__ import annotations

from typing import Dict, List, Set, Tuple

import numpy as np

from h2gen import H2Input, cid, lvl_off, n_clusters


def effective_bases(h2: H2Input, side: str = "row") -> List[np.ndarray]:
    """R_t (|t| x k_t) for every cluster, expanded from leaf bases and transfers."""
    L, B = h2.L, h2.B
    leaf = h2.leaf_row if side == "row" else h2.leaf_col
    tr = h2.transfer_row if side == "row" else h2.transfer_col
    rank = h2.rank_row if side == "row" else h2.rank_col
    R: List[np.ndarray] = [None] * n_clusters(L)
    for i in range(1 << L):
        R[cid(L, 0, i)] = np.asarray(leaf[i])
    for k in range(1, L + 1):
        for i in range(1 << (L - k)):
            p = cid(L, k, i)
            c1, c2 = cid(L, k - 1, 2 * i), cid(L, k - 1, 2 * i + 1)
            a, b = R[c1], R[c2]
            blk = np.zeros((a.shape[0] + b.shape[0], a.shape[1] + b.shape[1]))
            blk[:a.shape[0], :a.shape[1]] = a
            blk[a.shape[0]:, a.shape[1]:] = b
            R[p] = blk @ tr[p] if tr[p].size else np.zeros((blk.shape[0], int(rank[p])))
    return R


def dense_A(h2: H2Input) -> np.ndarray:
    L, B = h2.L, h2.B
    N = B << L
    A = np.zeros((N, N))
    for (t, s), C in zip(h2.near, h2.close):
        A[t * B:(t + 1) * B, s * B:(s + 1) * B] += C
    Rr = effective_bases(h2, "row")
    Rc = effective_bases(h2, "col")
    for k in range(L):
        sz = B << k
        base = lvl_off(L, k)
        for (t, s), D in zip(h2.adm[k], h2.coupling[k]):
            A[t * sz:(t + 1) * sz, s * sz:(s + 1) * sz] += Rr[base + t] @ D @ Rc[base + s].T
    return A


def dense_U(res, side: str = "row") -> np.ndarray:
    L, B = res.L, res.B
    N = B << L
    Q = res.Q_row if side == "row" else res.Q_col
    kk = res.k_row if side == "row" else res.k_col
    off = res.off_row if side == "row" else res.off_col
    U = np.zeros((N, N))
    Phi: Dict[int, np.ndarray] = {}
    for k in range(L + 1):
        sz = B << k
        for i in range(1 << (L - k)):
            c = cid(L, k, i)
            if k == 0:
                Phi[c] = np.eye(B)
            else:
                c1, c2 = cid(L, k - 1, 2 * i), cid(L, k - 1, 2 * i + 1)
                a = Phi[c1] @ Q[c1][:, :kk[c1]]
                b = Phi[c2] @ Q[c2][:, :kk[c2]]
                blk = np.zeros((sz, a.shape[1] + b.shape[1]))
                blk[:sz // 2, :a.shape[1]] = a
                blk[sz // 2:, a.shape[1]:] = b
                Phi[c] = blk
            cols = Phi[c] @ Q[c][:, kk[c]:]
            U[i * sz:(i + 1) * sz, off[c]:off[c] + cols.shape[1]] = cols
    return U


def h2_matvec(h2: H2Input, x: np.ndarray) -> np.ndarray:
    """y = A_H2 x by forward (basis coefficients), coupling and backward passes."""
    L, B = h2.L, h2.B
    x = np.asarray(x, dtype=np.float64)
    y = np.zeros_like(x)
    for (t, s), C in zip(h2.near, h2.close):
        y[t * B:(t + 1) * B] += C @ x[s * B:(s + 1) * B]
    ncl = n_clusters(L)
    xh: List[np.ndarray] = [None] * ncl
    for i in range(1 << L):
        xh[cid(L, 0, i)] = np.asarray(h2.leaf_col[i]).T @ x[i * B:(i + 1) * B]
    for k in range(1, L + 1):
        for i in range(1 << (L - k)):
            p = cid(L, k, i)
            xh[p] = h2.transfer_col[p].T @ np.concatenate([xh[cid(L, k - 1, 2 * i)], xh[cid(L, k - 1, 2 * i + 1)]])
    yh = [np.zeros((int(h2.rank_row[c]),) + x.shape[1:]) for c in range(ncl)]
    for k in range(L):
        base = lvl_off(L, k)
        for (t, s), D in zip(h2.adm[k], h2.coupling[k]):
            yh[base + t] = yh[base + t] + D @ xh[base + int(s)]
    for k in range(L, 0, -1):
        for i in range(1 << (L - k)):
            p = cid(L, k, i)
            c1, c2 = cid(L, k - 1, 2 * i), cid(L, k - 1, 2 * i + 1)
            v = h2.transfer_row[p] @ yh[p]
            k1 = int(h2.rank_row[c1])
            yh[c1] = yh[c1] + v[:k1]
            yh[c2] = yh[c2] + v[k1:]
    for i in range(1 << L):
        y[i * B:(i + 1) * B] += np.asarray(h2.leaf_row[i]) @ yh[cid(L, 0, i)]
    return y


def frobenius_sq(h2: H2Input) -> float:
    """||A_H2||_F^2 = sum_{N_0} ||C||_F^2 + sum_A tr(D^T G^R_t D G^C_s), with
    Gram matrices G_leaf = R^T R, G_p = sum_a T^(a)T G_ca T^(a).  S = U^T A V
    with orthogonal U, V has the same Frobenius norm."""
    L = h2.L
    tot = float(sum(np.sum(C * C) for C in h2.close))

    def grams(leaf, tr, rank):
        G = [None] * n_clusters(L)
        for i in range(1 << L):
            R = np.asarray(leaf[i])
            G[cid(L, 0, i)] = R.T @ R
        for k in range(1, L + 1):
            for i in range(1 << (L - k)):
                p = cid(L, k, i)
                c1, c2 = cid(L, k - 1, 2 * i), cid(L, k - 1, 2 * i + 1)
                k1 = int(rank[c1])
                T = tr[p]
                G[p] = T[:k1].T @ G[c1] @ T[:k1] + T[k1:].T @ G[c2] @ T[k1:]
        return G

    Gr = grams(h2.leaf_row, h2.transfer_row, h2.rank_row)
    Gc = grams(h2.leaf_col, h2.transfer_col, h2.rank_col)
    for k in range(L):
        base = lvl_off(L, k)
        for (t, s), D in zip(h2.adm[k], h2.coupling[k]):
            tot += float(np.trace(D.T @ Gr[base + t] @ D @ Gc[base + s]))
    return tot


def pattern_rule(h2: H2Input) -> Set[Tuple[int, int, int, int]]:
    """Closed-form block pattern of S (SURVEY §8(c) "Symbolic pattern rule"):
    (t@i, s@j) present iff m_t > 0, m_s > 0 and
      i == j and (t, s) in N_i; or
      i > j and some t' below t at level j has (t', s) in N_j with k^R > 0 on
      every row cluster of the path t' .. child-of-t; or the column mirror."""
    L, B = h2.L, h2.B
    kr, kc = np.asarray(h2.rank_row), np.asarray(h2.rank_col)

    def nloc(rank):
        n = np.zeros(n_clusters(L), dtype=np.int64)
        n[:1 << L] = B
        for k in range(1, L + 1):
            for i in range(1 << (L - k)):
                n[cid(L, k, i)] = rank[cid(L, k - 1, 2 * i)] + rank[cid(L, k - 1, 2 * i + 1)]
        return n

    mr = nloc(kr) - kr
    mc = nloc(kc) - kc
    # N_j by the block-tree rule, computed here on its own
    Ns = [set((int(t), int(s)) for (t, s) in h2.near)]
    for j in range(1, L + 1):
        nxt = {(t // 2, s // 2) for (t, s) in Ns[-1]} | {(int(t) // 2, int(s) // 2) for (t, s) in h2.adm[j - 1]}
        Ns.append(nxt)
    out = set()
    for j in range(L + 1):
        for (t0, s0) in Ns[j]:
            ct, cs = cid(L, j, t0), cid(L, j, s0)
            if mr[ct] > 0 and mc[cs] > 0:
                out.add((j, t0, j, s0))
            # row strips: walk t up while the current row cluster keeps basis rows
            t, lvl = t0, j
            while mc[cs] > 0 and lvl < L and kr[cid(L, lvl, t)] > 0:
                t, lvl = t // 2, lvl + 1
                if mr[cid(L, lvl, t)] > 0:
                    out.add((lvl, t, j, s0))
            s, lvl = s0, j
            while mr[ct] > 0 and lvl < L and kc[cid(L, lvl, s)] > 0:
                s, lvl = s // 2, lvl + 1
                if mc[cid(L, lvl, s)] > 0:
                    out.add((j, t0, lvl, s))
    return out


# ---------------------------------------------------------------------------
# Checks at sizes where the close blocks / couplings are never stored (config 5
# at full size): the same definitions, with C_ts and D_b evaluated from the
# points / interpolation nodes (h2gen.kernel_matrix and the plain-C helper
# close_norm.c) instead of read from arrays.
# ---------------------------------------------------------------------------

def _close_lib():
    import ctypes
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libclosenorm.so")
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    lib.oracle_close_frob_sq.argtypes = [P(ctypes.c_double), ctypes.c_int, ctypes.c_int, P(ctypes.c_int32),
                                        P(ctypes.c_int32), ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, P(ctypes.c_double)]
    lib.oracle_close_frob_sq.restype = None
    return lib


_KIND = {"exp": 1, "invh": 2, "laplace": 3}


def close_frob_sq(h2: H2Input, pairs: np.ndarray) -> np.ndarray:
    """||C_ts||_F^2 of each leaf pair (t, s) of ``pairs`` -- from h2.close when the
    blocks are stored, else evaluated from the points (close_norm.c)."""
    import ctypes
    pairs = np.asarray(pairs, dtype=np.int32).reshape(-1, 2)
    if h2.close is not None:
        key = {(int(t), int(s)): i for i, (t, s) in enumerate(h2.near)}
        return np.array([float(np.sum(h2.close[key[(int(t), int(s))]] ** 2)) for (t, s) in pairs])
    ks = h2.meta["kernel"]
    kind = _KIND[ks["kind"]]
    p0, p1 = {"exp": (ks.get("ell"), ks.get("nugget")), "invh": (ks.get("h"), ks.get("diag_add")),
              "laplace": (0.0, 1.0 / (4.0 * np.pi * ks.get("h", 1.0)))}[ks["kind"]]
    x = np.ascontiguousarray(h2.points, dtype=np.float64)
    pt = np.ascontiguousarray(pairs[:, 0])
    ps = np.ascontiguousarray(pairs[:, 1])
    out = np.zeros(len(pairs))
    P = ctypes.POINTER
    _close_lib().oracle_close_frob_sq(x.ctypes.data_as(P(ctypes.c_double)), x.shape[1], h2.B,
                                      pt.ctypes.data_as(P(ctypes.c_int32)), ps.ctypes.data_as(P(ctypes.c_int32)),
                                      len(pairs), kind, float(p0), float(p1), out.ctypes.data_as(P(ctypes.c_double)))
    return out


def _coupling(h2: H2Input, k: int, j: int, t: int, s: int) -> np.ndarray:
    if h2.coupling is not None:
        return h2.coupling[k][j]
    from h2gen import kernel_matrix
    base = lvl_off(h2.L, k)
    return kernel_matrix(h2.meta["kernel"], h2.meta["cheb_nodes_row"][base + t], h2.meta["cheb_nodes_col"][base + s])


def gram_matrices(h2: H2Input, side: str = "row") -> List[np.ndarray]:
    """G_t = R_t^T R_t of every cluster by the nested recursion
    G_p = sum_a T^(a)T G_ca T^(a) (R_p = diag(R_c1, R_c2) T_p)."""
    L = h2.L
    leaf = h2.leaf_row if side == "row" else h2.leaf_col
    tr = h2.transfer_row if side == "row" else h2.transfer_col
    rank = h2.rank_row if side == "row" else h2.rank_col
    G = [None] * n_clusters(L)
    for i in range(1 << L):
        R = np.asarray(leaf[i])
        G[cid(L, 0, i)] = R.T @ R
    for k in range(1, L + 1):
        for i in range(1 << (L - k)):
            p = cid(L, k, i)
            c1, c2 = cid(L, k - 1, 2 * i), cid(L, k - 1, 2 * i + 1)
            k1 = int(rank[c1])
            T = tr[p]
            G[p] = T[:k1].T @ G[c1] @ T[:k1] + T[k1:].T @ G[c2] @ T[k1:]
    return G


def frobenius_sq_rows(h2: H2Input, level: int, index: int) -> float:
    """||A_H2[I_c, :]||_F^2 for the rows I_c of cluster c = (level, index):
    the close blocks with t among c's leaves, tr(D^T G^R_t D G^C_s) for the
    admissible pairs with t inside c (levels <= level), and for the admissible
    pairs of c's ancestors a the same with the Gram of a's basis restricted to
    I_c: R_a[I_c] = R_c T_p1[c's rows] T_p2[p1's rows] ... (nested bases,
    P:76-84), so G = M^T G_c M.  When k_c = 0 the S rows
    of c's subtree, (k', t', a) with t' inside c, are U_c^T A V with U_c an
    orthonormal basis of the coordinates I_c (their count is |I_c| because
    sum m = |I_c| - k_c), so their ||.||_F^2 equals this (pin P5 per subtree,
    P:472-484; QR-independent)."""
    L = h2.L
    lo_leaf, hi_leaf = index << level, (index + 1) << level
    near = np.asarray(h2.near)
    sel = near[(near[:, 0] >= lo_leaf) & (near[:, 0] < hi_leaf)]
    tot = float(np.sum(close_frob_sq(h2, sel)))
    Gr = gram_matrices(h2, "row")
    Gc = Gr if h2.symmetric else gram_matrices(h2, "col")
    for k in range(min(level + 1, L)):
        base = lvl_off(L, k)
        a = np.asarray(h2.adm[k])
        if not len(a):
            continue
        lo_t, hi_t = index << (level - k), (index + 1) << (level - k)
        for j in np.nonzero((a[:, 0] >= lo_t) & (a[:, 0] < hi_t))[0]:
            t, s = int(a[j, 0]), int(a[j, 1])
            D = _coupling(h2, k, int(j), t, s)
            tot += float(np.trace(D.T @ Gr[base + t] @ D @ Gc[base + s]))
    # ancestors of c: their bases restricted to the rows of c
    c = cid(L, level, index)
    M = np.eye(int(h2.rank_row[c]))
    u, ui = c, index
    for k in range(level + 1, L):
        pi = ui >> 1
        p = cid(L, k, pi)
        k1 = int(h2.rank_row[cid(L, k - 1, 2 * pi)])
        T = h2.transfer_row[p]
        M = M @ (T[:k1] if (ui & 1) == 0 else T[k1:])
        G = M.T @ Gr[c] @ M
        a = np.asarray(h2.adm[k])
        if len(a):
            base = lvl_off(L, k)
            for j in np.nonzero(a[:, 0] == pi)[0]:
                s = int(a[j, 1])
                D = _coupling(h2, k, int(j), pi, s)
                tot += float(np.trace(D.T @ G @ D @ Gc[base + s]))
        u, ui = p, pi
    return tot


def h2_matvec_rows(h2: H2Input, x: np.ndarray, leaves) -> Dict[int, np.ndarray]:
    """(A_H2 x) on the rows of the given leaves (pin P13 on a sample at any N):
    close part sum_s C_ts x_s, far part by the standard upward pass (all
    clusters) and the coupling / downward passes along the leaves' root paths
    only.  Close blocks / couplings evaluated when not stored."""
    from h2gen import kernel_matrix
    L, B = h2.L, h2.B
    x = np.asarray(x, dtype=np.float64)
    ncl = n_clusters(L)
    xh: List[np.ndarray] = [None] * ncl
    for i in range(1 << L):
        xh[cid(L, 0, i)] = np.asarray(h2.leaf_col[i]).T @ x[i * B:(i + 1) * B]
    for k in range(1, L + 1):
        for i in range(1 << (L - k)):
            p = cid(L, k, i)
            xh[p] = h2.transfer_col[p].T @ np.concatenate([xh[cid(L, k - 1, 2 * i)], xh[cid(L, k - 1, 2 * i + 1)]])
    near = np.asarray(h2.near)
    adm_rows = []
    for k in range(L):
        a = np.asarray(h2.adm[k])
        adm_rows.append(a)
    out = {}
    for leaf in leaves:
        y = np.zeros(B)
        for j in np.nonzero(near[:, 0] == leaf)[0]:
            s = int(near[j, 1])
            if h2.close is not None:
                C = h2.close[j]
            else:
                same = np.eye(B, dtype=bool) if s == leaf else None
                C = kernel_matrix(h2.meta["kernel"], h2.points[leaf * B:(leaf + 1) * B], h2.points[s * B:(s + 1) * B],
                                  same)
            y += C @ x[s * B:(s + 1) * B]
        yh = np.zeros(0)                  # the root's coefficients (k_root = 0)
        for k in range(L - 1, -1, -1):   # root path, top down
            t = leaf >> k
            p = cid(L, k, t)
            acc = np.zeros(int(h2.rank_row[p]))
            if yh.size:                   # parent's coefficients through its transfer
                v = h2.transfer_row[cid(L, k + 1, t >> 1)] @ yh
                k1 = int(h2.rank_row[cid(L, k, 2 * (t >> 1))])
                acc = acc + (v[:k1] if (t & 1) == 0 else v[k1:])
            a = adm_rows[k]
            if len(a):
                for j in np.nonzero(a[:, 0] == t)[0]:
                    s = int(a[j, 1])
                    acc = acc + _coupling(h2, k, int(j), t, s) @ xh[lvl_off(L, k) + s]
            yh = acc
        y += np.asarray(h2.leaf_row[leaf]) @ yh
        out[int(leaf)] = y
    return out
