"""O1 -- the paper's level-by-level sparsification, written plainly (CPU, fp64).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with the CUDA path (``paper_1705_04601_b200``); the
only common module is the seeded input generator ``h2gen``.

What it computes (PAPER.md = P):
  * step (i)  QR completion of nested bases, P:685-691 ("orthogonalize blocks,
    complete each block to square orthogonal block ... QR decomposition of
    blocks with the square Q factor"), with convention H (reading 1-2,
    LAPACK dgeqrf/dorg2r semantics);
  * far couplings in the orthogonalised bases D~ = R^_t D R^_s^T (P:702,
    reading 11);
  * step (iv) merge of sibling basis parts with the far couplings into the next
    level's close blocks, C_{k+1} = C^_{k+1} + F^_ml,k+1 (Eq. cl1;
    P:698-702);
  * step (ii) congruence H_ts = Q_t^T G_ts Q_s;
  * step (iii) freezing of the non-basis rows/columns into S in the order of
    the permutations P_rk, P_ck, including the basis x frozen
    "strips" rotated by every ancestor (Eq. u1v1; reading 7);
  * the cascade to the root, S = (prod U_k^T) A (prod V_k) (Eq. fin).

Everything is a plain Python loop over clusters / pairs / strips with numpy
matmul as the only library primitive.  Symmetric mode follows DESIGN.md
(canonical pairs t <= s, H_st := H_ts^T, diagonal H_tt symmetrised
upper->lower, row strips only) so that U == V and S is bitwise symmetric
(Proposition).
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Dict, List, Tuple

import numpy as np

from h2gen import H2Input, cid, lvl_off, n_clusters

Pair = Tuple[int, int]


# ----------------------------------------------------------------------------
# Convention H: Householder QR with a square Q, LAPACK semantics
# ----------------------------------------------------------------------------

def householder_complete(X: np.ndarray, record: Optional[list] = None):
    """Q (n x n, orthogonal) and R^ (k x k, upper triangular) with
    X = Q[:, :k] R^.  For j = 0..k-1 on x = X[j:, j]: alpha = x_0,
    sigma = ||x_1:||; sigma == 0 exactly -> tau = 0, beta = alpha; otherwise
    beta = -sgn(alpha) hypot(alpha, sigma) with sgn(+-0) = +1,
    tau = (beta - alpha)/beta, v = [1; x_1:/(alpha - beta)].
    Q = H_0 H_1 ... H_{k-1} I_n (dorg2r order).  k = 0 -> Q = I.
    ``record`` (optional list): receives (alpha, sigma) of every step -- the
    quantities whose sign / zero tests convention H decides (reading 2)."""
    X = np.array(X, dtype=np.float64, copy=True)
    n, k = X.shape
    assert k <= n, (n, k)
    vs: List[np.ndarray] = []
    taus: List[float] = []
    for j in range(k):
        x = X[j:, j]
        alpha = float(x[0])
        sigma = float(np.sqrt(np.dot(x[1:], x[1:]))) if n - j > 1 else 0.0
        if record is not None:
            record.append((alpha, sigma))
        if sigma == 0.0:
            tau = 0.0
            v = np.zeros(n - j)
            v[0] = 1.0
            beta = alpha
        else:
            sgn = -1.0 if alpha < 0.0 else 1.0
            beta = -sgn * float(np.hypot(alpha, sigma))
            tau = (beta - alpha) / beta
            v = np.empty(n - j)
            v[0] = 1.0
            v[1:] = x[1:] / (alpha - beta)
        # apply H_j = I - tau v v^T to the trailing columns
        if tau != 0.0 and j + 1 < k:
            w = v @ X[j:, j + 1:]
            X[j:, j + 1:] -= tau * np.outer(v, w)
        X[j, j] = beta
        X[j + 1:, j] = 0.0
        vs.append(v)
        taus.append(tau)
    Rhat = np.triu(X[:k, :k])
    Q = np.eye(n)
    for j in range(k - 1, -1, -1):
        if taus[j] != 0.0:
            v = vs[j]
            w = v @ Q[j:, :]
            Q[j:, :] -= taus[j] * np.outer(v, w)
    return Q, Rhat


# ----------------------------------------------------------------------------
# Result container
# ----------------------------------------------------------------------------

@dataclasses.dataclass
class OracleResult:
    L: int
    B: int
    symmetric: bool
    n_row: np.ndarray
    k_row: np.ndarray
    n_col: np.ndarray
    k_col: np.ndarray
    Q_row: List[np.ndarray]
    Q_col: List[np.ndarray]
    Rhat_row: List[np.ndarray]
    Rhat_col: List[np.ndarray]
    off_row: np.ndarray            # S-order offset per cluster (row side)
    off_col: np.ndarray
    S: Dict[Tuple[int, int, int, int], np.ndarray]   # (i, t, j, s) -> m_t x m_s
    near_levels: List[List[Pair]]

    @property
    def N(self):
        return self.B << self.L

    @property
    def m_row(self):
        return self.n_row - self.k_row

    @property
    def m_col(self):
        return self.n_col - self.k_col


def _local_sizes(L, B, rank):
    """n_t = B for leaves, k_c1 + k_c2 for internal clusters (reading 3)."""
    n = np.zeros(n_clusters(L), dtype=np.int64)
    n[:1 << L] = B
    for k in range(1, L + 1):
        for i in range(1 << (L - k)):
            n[cid(L, k, i)] = rank[cid(L, k - 1, 2 * i)] + rank[cid(L, k - 1, 2 * i + 1)]
    return n


def s_offsets(L, m):
    """off(k,t) = sum_{k'<k} sum_t' m_t' + sum_{t'<t @k} m_t' -- non-basis
    indices before basis ones, order preserved (P_rk)."""
    off = np.zeros(n_clusters(L), dtype=np.int64)
    acc = 0
    for k in range(L + 1):
        for i in range(1 << (L - k)):
            c = cid(L, k, i)
            off[c] = acc
            acc += int(m[c])
    return off


def near_pairs_next(near_prev: List[Pair], adm_prev: np.ndarray) -> List[Pair]:
    """N_k = parents of N_{k-1} u A_{k-1}: a big block is close if it is not a
    leaf of the block tree at a higher level (reading 9)."""
    par = {(t // 2, s // 2) for (t, s) in near_prev}
    par |= {(int(t) // 2, int(s) // 2) for (t, s) in adm_prev}
    return sorted(par)


# ----------------------------------------------------------------------------
# O1
# ----------------------------------------------------------------------------

def sparsify(h2: H2Input) -> OracleResult:
    L, B, sym = h2.L, h2.B, h2.symmetric
    ncl = n_clusters(L)
    kr = np.asarray(h2.rank_row, dtype=np.int64)
    kc = np.asarray(h2.rank_col, dtype=np.int64)
    nr = _local_sizes(L, B, kr)
    nc = _local_sizes(L, B, kc)
    if np.any(kr > nr) or np.any(kc > nc) or kr[-1] != 0 or kc[-1] != 0:
        raise ValueError("invalid rank distribution")
    off_r = s_offsets(L, nr - kr)
    off_c = s_offsets(L, nc - kc)
    Qr: List[np.ndarray] = [None] * ncl
    Qc: List[np.ndarray] = [None] * ncl
    Rr: List[np.ndarray] = [None] * ncl
    Rc: List[np.ndarray] = [None] * ncl
    S: Dict[Tuple[int, int, int, int], np.ndarray] = {}
    near_levels: List[List[Pair]] = []

    near = [(int(t), int(s)) for (t, s) in h2.near]
    H_prev: Dict[Pair, np.ndarray] = {}
    Dt_prev: Dict[Pair, np.ndarray] = {}
    YR_prev: Dict[Tuple[int, int, int], np.ndarray] = {}    # (c, l, s) -> k_c x m_s
    YC_prev: Dict[Tuple[int, int, int], np.ndarray] = {}    # (l, t, d) -> m_t x k_d

    def X_of(side_rank, Rhat, leaf, transfer, k, i):
        c = cid(L, k, i)
        if k == 0:
            return leaf[i]
        c1, c2 = cid(L, k - 1, 2 * i), cid(L, k - 1, 2 * i + 1)
        k1 = side_rank[c1]
        T = transfer[c]
        return np.vstack([Rhat[c1] @ T[:k1], Rhat[c2] @ T[k1:]])

    for k in range(L + 1):
        M = 1 << (L - k)
        base = lvl_off(L, k)
        if k > 0:
            near = near_pairs_next(near, h2.adm[k - 1])
        near_levels.append(near)
        # ---- step (i): QR completion of the nested bases
        for i in range(M):
            c = base + i
            Qr[c], Rr[c] = householder_complete(X_of(kr, Rr, h2.leaf_row, h2.transfer_row, k, i))
            if sym:
                Qc[c], Rc[c] = Qr[c], Rr[c]
            else:
                Qc[c], Rc[c] = householder_complete(X_of(kc, Rc, h2.leaf_col, h2.transfer_col, k, i))
        # ---- couplings in orthogonalised coordinates (reading 11)
        Dt: Dict[Pair, np.ndarray] = {}
        if k < L:
            for (t, s), D in zip(h2.adm[k], h2.coupling[k]):
                t, s = int(t), int(s)
                if sym and t > s:
                    continue
                Dt[(t, s)] = Rr[base + t] @ D @ Rc[base + s].T
            if sym:
                for (t, s) in h2.adm[k]:
                    t, s = int(t), int(s)
                    if t > s:
                        Dt[(t, s)] = Dt[(s, t)].T
        # ---- steps (iv)+(ii): merge and congruence
        H: Dict[Pair, np.ndarray] = {}
        close_idx = {(int(t), int(s)): j for j, (t, s) in enumerate(h2.near)} if k == 0 else None
        for (t, s) in near:
            if sym and t > s:
                continue
            ct, cs = base + t, base + s
            if k == 0:
                G = h2.close[close_idx[(t, s)]]
            else:
                G = np.zeros((nr[ct], nc[cs]))
                for a in range(2):
                    for b in range(2):
                        ca, db = 2 * t + a, 2 * s + b
                        r0 = 0 if a == 0 else kr[cid(L, k - 1, 2 * t)]
                        c0 = 0 if b == 0 else kc[cid(L, k - 1, 2 * s)]
                        ka, kb = kr[cid(L, k - 1, ca)], kc[cid(L, k - 1, db)]
                        if (ca, db) in H_prev:
                            Y = H_prev[(ca, db)][:ka, :kb]
                        else:
                            Y = Dt_prev[(ca, db)]     # KeyError => block tree not a partition
                        G[r0:r0 + ka, c0:c0 + kb] = Y
            Hts = Qr[ct].T @ G @ Qc[cs]
            if sym and t == s:
                Hts = np.triu(Hts) + np.triu(Hts, 1).T
            H[(t, s)] = Hts
        if sym:
            for (t, s) in near:
                if t > s:
                    H[(t, s)] = H[(s, t)].T
        # ---- step (iii): freeze non-basis x non-basis, start strips
        YR: Dict[Tuple[int, int, int], np.ndarray] = {}
        YC: Dict[Tuple[int, int, int], np.ndarray] = {}
        for (t, s) in near:
            ct, cs = base + t, base + s
            ktt, kss = kr[ct], kc[cs]
            mt, ms = nr[ct] - ktt, nc[cs] - kss
            Hts = H[(t, s)]
            if mt > 0 and ms > 0:
                S[(k, t, k, s)] = Hts[ktt:, kss:]
            if ktt > 0 and ms > 0:
                YR[(t, k, s)] = Hts[:ktt, kss:]
            if not sym and mt > 0 and kss > 0:
                YC[(k, t, s)] = Hts[ktt:, :kss]
        # ---- strips arriving from level k-1 (Eq. u1v1: U_k^T rotates the
        #      whole basis region, including its frozen columns)
        if k > 0:
            groups: Dict[Tuple[int, int, int], List[Tuple[int, np.ndarray]]] = {}
            for (c, l, s), Y in YR_prev.items():
                groups.setdefault((c // 2, l, s), []).append((c % 2, Y))
            for (p, l, s), parts in sorted(groups.items()):
                cp = base + p
                ms = nc[cid(L, l, s)] - kc[cid(L, l, s)]
                Z = np.zeros((nr[cp], ms))
                for a, Y in parts:
                    r0 = 0 if a == 0 else kr[cid(L, k - 1, 2 * p)]
                    Z[r0:r0 + Y.shape[0]] = Y
                W = Qr[cp].T @ Z
                if nr[cp] - kr[cp] > 0:
                    S[(k, p, l, s)] = W[kr[cp]:]
                if kr[cp] > 0:
                    YR[(p, l, s)] = W[:kr[cp]]
            if not sym:
                groups = {}
                for (l, t, d), Y in YC_prev.items():
                    groups.setdefault((l, t, d // 2), []).append((d % 2, Y))
                for (l, t, q), parts in sorted(groups.items()):
                    cq = base + q
                    mt = nr[cid(L, l, t)] - kr[cid(L, l, t)]
                    Z = np.zeros((mt, nc[cq]))
                    for b, Y in parts:
                        c0 = 0 if b == 0 else kc[cid(L, k - 1, 2 * q)]
                        Z[:, c0:c0 + Y.shape[1]] = Y
                    W = Z @ Qc[cq]
                    if nc[cq] - kc[cq] > 0:
                        S[(l, t, k, q)] = W[:, kc[cq]:]
                    if kc[cq] > 0:
                        YC[(l, t, q)] = W[:, :kc[cq]]
        H_prev, Dt_prev, YR_prev, YC_prev = H, Dt, YR, YC

    if sym:
        # column-strip blocks are the transposes of the row-strip blocks
        for (i, t, j, s) in list(S.keys()):
            if i > j:
                S[(j, s, i, t)] = S[(i, t, j, s)].T
    return OracleResult(L=L, B=B, symmetric=sym, n_row=nr, k_row=kr, n_col=nc, k_col=kc, Q_row=Qr, Q_col=Qc,
                        Rhat_row=Rr, Rhat_col=Rc, off_row=off_r, off_col=off_c, S=S, near_levels=near_levels)


# ----------------------------------------------------------------------------
# S as CSR (rows in S order, columns ascending; reading 13: no dropping)
# ----------------------------------------------------------------------------

def s_csr(res: OracleResult):
    """(rowptr int64 [N+1], col int32 [nnz], val float64 [nnz])."""
    L = res.L
    N = res.N
    by_row: Dict[Tuple[int, int], List[Tuple[int, int, int, np.ndarray]]] = {}
    for (i, t, j, s), blk in res.S.items():
        by_row.setdefault((i, t), []).append((int(res.off_col[cid(L, j, s)]), j, s, blk))
    m_r = res.m_row
    m_c = res.m_col
    rowlen = np.zeros(N, dtype=np.int64)
    panels = []
    cols = []
    for k in range(L + 1):
        for t in range(1 << (L - k)):
            c = cid(L, k, t)
            if m_r[c] == 0:
                continue
            blks = sorted(by_row.get((k, t), []), key=lambda e: e[0])
            r0 = int(res.off_row[c])
            if not blks:
                continue
            panel = np.hstack([b[3] for b in blks])
            colidx = np.concatenate([np.arange(b[0], b[0] + m_c[cid(L, b[1], b[2])]) for b in blks])
            rowlen[r0:r0 + m_r[c]] = panel.shape[1]
            panels.append(panel.ravel())
            cols.append(np.tile(colidx, int(m_r[c])))
    rowptr = np.zeros(N + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(rowlen)
    val = np.concatenate(panels) if panels else np.zeros(0)
    col = np.concatenate(cols).astype(np.int32) if cols else np.zeros(0, dtype=np.int32)
    return rowptr, col, val


def s_dense(res: OracleResult) -> np.ndarray:
    """S as a dense N x N matrix (tiny N only)."""
    N = res.N
    out = np.zeros((N, N))
    L = res.L
    for (i, t, j, s), blk in res.S.items():
        r0 = int(res.off_row[cid(L, i, t)])
        c0 = int(res.off_col[cid(L, j, s)])
        out[r0:r0 + blk.shape[0], c0:c0 + blk.shape[1]] = blk
    return out


# ----------------------------------------------------------------------------
# Apply U^T b and V y (Eq. sp0)
# ----------------------------------------------------------------------------

def apply_Ut(res: OracleResult, b: np.ndarray, side: str = "row") -> np.ndarray:
    """y = U^T b: b in tree order (N x nrhs) -> y in S order.  Leaves to root:
    z = Q_t^T x_t; z[k_t:] -> S order; z[:k_t] -> parent's local vector."""
    L, B = res.L, res.B
    Q = res.Q_row if side == "row" else res.Q_col
    kk = res.k_row if side == "row" else res.k_col
    off = res.off_row if side == "row" else res.off_col
    b = np.asarray(b, dtype=np.float64)
    y = np.zeros_like(b)
    xl: Dict[int, np.ndarray] = {}
    for k in range(L + 1):
        for i in range(1 << (L - k)):
            c = cid(L, k, i)
            if k == 0:
                x = b[i * B:(i + 1) * B]
            else:
                x = np.concatenate([xl[cid(L, k - 1, 2 * i)], xl[cid(L, k - 1, 2 * i + 1)]], axis=0)
            z = Q[c].T @ x
            m = z.shape[0] - kk[c]
            y[off[c]:off[c] + m] = z[kk[c]:]
            xl[c] = z[:kk[c]]
    return y


def apply_V(res: OracleResult, y: np.ndarray, side: str = "col") -> np.ndarray:
    """x = V y: y in S order -> x in tree order.  Root to leaves:
    x_t = Q_t [z_basis; y_t]; z_basis comes from the parent."""
    L, B = res.L, res.B
    Q = res.Q_col if side == "col" else res.Q_row
    kk = res.k_col if side == "col" else res.k_row
    off = res.off_col if side == "col" else res.off_row
    y = np.asarray(y, dtype=np.float64)
    x = np.zeros_like(y)
    zb: Dict[int, np.ndarray] = {cid(L, L, 0): y[:0]}
    for k in range(L, -1, -1):
        for i in range(1 << (L - k)):
            c = cid(L, k, i)
            n = Q[c].shape[0]
            m = n - kk[c]
            v = np.concatenate([zb[c], y[off[c]:off[c] + m]], axis=0)
            w = Q[c] @ v
            if k == 0:
                x[i * B:(i + 1) * B] = w
            else:
                k1 = kk[cid(L, k - 1, 2 * i)]
                zb[cid(L, k - 1, 2 * i)] = w[:k1]
                zb[cid(L, k - 1, 2 * i + 1)] = w[k1:]
    return x


def householder_margins(h2: H2Input) -> dict:
    """Survey reading 2 (the Householder tie-break hazard): run the QR pass of
    step (i) on every cluster of both sides, in the paper's order (the same
    X_t as sparsify), and report the smallest relative margin of the two
    decisions convention H takes exactly -- the sign of alpha (alpha_margin =
    min |alpha| / sigma) and sigma == 0 (sigma_margin = min sigma / |alpha|),
    over the steps with alpha != 0 and sigma != 0; min_margin = the smaller.
    Inputs with a margin below 1e-8 are ill-posed for parity (two correct
    implementations may take different branches); exact zeros (axis-aligned pin
    P8) are not hazards."""
    L = h2.L
    ncl = n_clusters(L)
    out = {"min_margin": float("inf"), "alpha_margin": float("inf"), "sigma_margin": float("inf"), "steps": 0,
           "exact_zero_steps": 0, "worst_cluster": None}
    for side in ("row",) + (() if h2.symmetric else ("col",)):
        rank = np.asarray(h2.rank_row if side == "row" else h2.rank_col)
        leaf = h2.leaf_row if side == "row" else h2.leaf_col
        tr = h2.transfer_row if side == "row" else h2.transfer_col
        R: List[np.ndarray] = [None] * ncl
        for k in range(L + 1):
            for i in range(1 << (L - k)):
                c = cid(L, k, i)
                if k == 0:
                    X = np.asarray(leaf[i])
                else:
                    c1, c2 = cid(L, k - 1, 2 * i), cid(L, k - 1, 2 * i + 1)
                    k1 = int(rank[c1])
                    X = np.vstack([R[c1] @ tr[c][:k1], R[c2] @ tr[c][k1:]])
                rec: list = []
                _, R[c] = householder_complete(X, rec)
                for (a, sg) in rec:
                    out["steps"] += 1
                    if a == 0.0 or sg == 0.0:
                        out["exact_zero_steps"] += 1
                        continue
                    out["alpha_margin"] = min(out["alpha_margin"], abs(a) / sg)
                    out["sigma_margin"] = min(out["sigma_margin"], sg / abs(a))
                    m = min(abs(a) / sg, sg / abs(a))
                    if m < out["min_margin"]:
                        out["min_margin"] = m
                        out["worst_cluster"] = (side, k, i)
    return out
