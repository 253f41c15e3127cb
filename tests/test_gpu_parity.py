"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Structure (S order, CSR rowptr/col) bit-exact; S values
within relative Frobenius error 1e-11 and Q blocks within 1e-12 (BASELINE.json
north_star); apply U^T b / V y within 1e-12."""
import numpy as np
import pytest

import h2gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run(h, explicit_q=False):
    import paper_1705_04601_b200 as h2sp
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed, explicit_q=explicit_q)
    sp = h2sp.Sparsifier(plan, packed)
    out = sp.build()
    torch.cuda.synchronize()
    return plan, sp, out


def _level_block_errors(plan, rowptr, col, v, val, tol, per_block=True):
    """Gate the error per level of the S row's cluster (relative, tol) and per
    S block (t@i, s@j): ||dS_b|| <= 1e3 tol ||S_b|| + 10 tol ||S_(t@i, :)|| --
    a wrong block fails even when it is tiny next to ||S||_F, while round-off
    carried from the block's whole strip chain (the block row's scale) passes.
    Returns (worst level error, worst block error relative to the block)."""
    off = plan.offsets()
    N = plan.N
    ncl = len(off["s_off_row"])
    m_r = np.diff(np.append(off["s_off_row"], N))
    m_c = np.diff(np.append(off["s_off_col"], N))
    row_cl = np.repeat(np.arange(ncl), m_r)
    col_cl = np.repeat(np.arange(ncl), m_c)
    L = plan.L
    lvl = np.zeros(ncl, dtype=np.int64)
    for k in range(L + 1):
        lvl[(1 << (L + 1)) - (1 << (L - k + 1)):] = k
    rows = np.repeat(np.arange(N), np.diff(rowptr))
    d2 = (v - val) ** 2
    r2 = val ** 2
    rl = lvl[row_cl[rows]]
    e_l = np.bincount(rl, d2, minlength=L + 1)
    n_l = np.bincount(rl, r2, minlength=L + 1)
    worst_level = 0.0
    for k in range(L + 1):
        if n_l[k] > 0:
            e = np.sqrt(e_l[k] / n_l[k])
            worst_level = max(worst_level, e)
            assert e <= tol, ("level", k, e)
    worst_block = 0.0
    if per_block:
        key = row_cl[rows] * ncl + col_cl[col]
        uq, inv = np.unique(key, return_inverse=True)
        eb = np.sqrt(np.bincount(inv, d2))
        nb = np.sqrt(np.bincount(inv, r2))
        brow = uq // ncl
        nrow = np.sqrt(np.bincount(brow, nb ** 2, minlength=ncl))[brow]
        bad = eb > 1e3 * tol * nb + 10 * tol * nrow
        assert not bad.any(), ("blocks", int(bad.sum()), [(int(uq[i] // ncl), int(uq[i] % ncl)) for i in
                                                         np.nonzero(bad)[0][:5]])
        rel = eb[nb > 0] / nb[nb > 0]
        worst_block = float(rel.max()) if len(rel) else 0.0
    return worst_level, worst_block


def _compare(h, plan, out, res=None, tol=1e-11, qtol=1e-12):
    res = res or oracle.sparsify(h)
    rowptr, col, val = oracle.s_csr(res)
    nnz = len(val)
    assert plan.sizes["s_nnz"] == nnz
    assert np.array_equal(out["s_rowptr"].cpu().numpy(), rowptr)
    assert np.array_equal(out["s_col"][:nnz].cpu().numpy(), col)
    v = out["s_val"][:nnz].cpu().numpy()
    nv = np.linalg.norm(val)
    err = np.linalg.norm(v - val) / nv if nv > 0 else np.linalg.norm(v)
    assert err <= tol, err
    if nv > 0:
        wl, wb = _level_block_errors(plan, rowptr, col, v, val, tol, per_block=nnz <= 60_000_000)
        print(f"parity: global {err:.2e}, worst level {wl:.2e}, worst block (own norm) {wb:.2e}")
    off = plan.offsets()
    qr = out["q_row"].cpu().numpy()
    qc = qr if h.symmetric else out["q_col"].cpu().numpy()
    for c in range(len(res.Q_row)):
        n = int(res.n_row[c])
        if n:
            Q = qr[off["q_off_row"][c]:off["q_off_row"][c] + n * n].reshape(n, n)
            assert np.abs(Q - res.Q_row[c]).max() <= qtol, c
        n = int(res.n_col[c])
        if n:
            Q = qc[off["q_off_col"][c]:off["q_off_col"][c] + n * n].reshape(n, n)
            assert np.abs(Q - res.Q_col[c]).max() <= qtol, c
    return res, v, err


CASES = []
for _sym in (True, False):
    for _seed, _eta in ((0, 0.4), (1, 0.7), (2, 1.5), (3, 0.7)):
        CASES.append((f"rand-{'sym' if _sym else 'gen'}-{_seed}",
                      (lambda sym=_sym, seed=_seed, eta=_eta: h2gen.random_h2(5, 16, seed, sym, eta=eta))))
CASES += [
    ("rand-B64-sym", lambda: h2gen.random_h2(4, 64, 7, True, eta=0.7, max_rank=32)),
    ("rand-B64-gen", lambda: h2gen.random_h2(4, 64, 8, False, eta=0.7, max_rank=32)),
    ("rand-B40-gen-ragged", lambda: h2gen.random_h2(5, 40, 9, False, eta=0.5, max_rank=32)),
    ("rand-B24-sym-uniform", lambda: h2gen.random_h2(5, 24, 10, True, eta=0.7, ragged=False, r=12)),
    ("fig3-half", lambda: h2gen.fig3_h2(8, 0, "half")),
    ("fig3-active-gen", lambda: h2gen.fig3_h2(8, 1, "active", symmetric=False)),
    ("cfg1", lambda: h2gen.make_config(1)),
    ("cfg2-16384", lambda: h2gen.make_config(2, N=16384)),
    ("cfg3-16384", lambda: h2gen.make_config(3, N=16384)),      # 3-D, r = 24: 48-wide internal tiles
    ("cfg4-16384", lambda: h2gen.make_config(4, N=16384)),      # sphere, general mode, r = 32
    # 128-point leaves (pair_wy128_kernel, qr_kernel with V / M output, 128-wide apply tiles)
    ("rand-B128-sym", lambda: h2gen.random_h2(5, 128, 6, True, eta=0.7, max_rank=32)),
    ("rand-B128-gen", lambda: h2gen.random_h2(5, 128, 5, False, eta=0.7, max_rank=32)),
    ("rand-B128-gen-k16", lambda: h2gen.random_h2(5, 128, 11, False, eta=0.7, max_rank=16)),
    ("cfg5-16384", lambda: h2gen.make_config(5, N=16384)),      # config-5 recipe: 3-D, B = 128, r = 32
]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_parity_small(name, make):
    _need_gpu()
    h = make()
    plan, sp, out = _run(h)
    res, v, err = _compare(h, plan, out)
    if h.symmetric:
        # Proposition: S bitwise symmetric in our convention
        import scipy.sparse as sps
        nnz = plan.sizes["s_nnz"]
        S = sps.csr_matrix((v, out["s_col"][:nnz].cpu().numpy(), out["s_rowptr"].cpu().numpy()), shape=(h.N, h.N))
        assert (S != S.T).nnz == 0


@pytest.mark.parametrize("sym", [True, False])
def test_eta0_bitwise(sym):
    """eta = 0: S = C bitwise on the GPU path too."""
    _need_gpu()
    h = h2gen.eta0_h2(3, 16, 5, symmetric=sym)
    plan, sp, out = _run(h)
    A = oracle.dense_A(h)
    rowptr = out["s_rowptr"].cpu().numpy()
    col = out["s_col"].cpu().numpy()
    val = out["s_val"].cpu().numpy()
    D = np.zeros_like(A)
    for r in range(h.N):
        D[r, col[rowptr[r]:rowptr[r + 1]]] = val[rowptr[r]:rowptr[r + 1]]
    assert np.array_equal(D, A)


def test_single_leaf():
    _need_gpu()
    h = h2gen.eta0_h2(0, 32, 6, symmetric=False)
    plan, sp, out = _run(h)
    assert np.array_equal(out["s_val"].cpu().numpy(), h.close[0].ravel())


@pytest.mark.parametrize("sym,seed", [(True, 1), (False, 2)])
def test_axis_aligned_bitwise(sym, seed):
    """Every Q = I exactly, so the GPU cascade is exact: S equals the oracle's
    (= P_r^T A_H2 P_c) bit for bit -- pins all permutation / strip bookkeeping."""
    _need_gpu()
    h = h2gen.axis_aligned_h2(5, 16, seed, sym)
    plan, sp, out = _run(h)
    res = oracle.sparsify(h)
    rowptr, col, val = oracle.s_csr(res)
    assert np.array_equal(out["s_val"][:len(val)].cpu().numpy(), val)


def test_dense_reconstruction_from_gpu_factors():
    """U S V^T = A_H2 with U, V assembled from the GPU's Q blocks (P1 on the GPU path)."""
    _need_gpu()
    h = h2gen.random_h2(4, 16, 12, False, eta=0.7)
    plan, sp, out = _run(h)
    res = oracle.sparsify(h)
    off = plan.offsets()
    qr, qc = out["q_row"].cpu().numpy(), out["q_col"].cpu().numpy()
    res.Q_row = [qr[off["q_off_row"][c]:off["q_off_row"][c] + int(n) ** 2].reshape(int(n), int(n))
                 for c, n in enumerate(res.n_row)]
    res.Q_col = [qc[off["q_off_col"][c]:off["q_off_col"][c] + int(n) ** 2].reshape(int(n), int(n))
                 for c, n in enumerate(res.n_col)]
    U, V = oracle.dense_U(res, "row"), oracle.dense_U(res, "col")
    nnz = plan.sizes["s_nnz"]
    rowptr, col = out["s_rowptr"].cpu().numpy(), out["s_col"].cpu().numpy()
    val = out["s_val"][:nnz].cpu().numpy()
    S = np.zeros((h.N, h.N))
    for r in range(h.N):
        S[r, col[rowptr[r]:rowptr[r + 1]]] = val[rowptr[r]:rowptr[r + 1]]
    A = oracle.dense_A(h)
    assert np.linalg.norm(U @ S @ V.T - A) / np.linalg.norm(A) <= 1e-12


@pytest.mark.parametrize("sym,B", [(True, 16), (False, 16), (True, 128), (False, 128)])
def test_apply_parity(sym, B):
    _need_gpu()
    h = h2gen.random_h2(5, B, 20 + sym, sym, eta=0.7, max_rank=32)
    plan, sp, out = _run(h)
    res = oracle.sparsify(h)
    rng = np.random.default_rng(3)
    b = rng.standard_normal((3, h.N))
    bt = torch.from_numpy(b).cuda()
    y = torch.empty_like(bt)
    sp.apply_Ut(bt, y)
    x = torch.empty_like(bt)
    sp.apply_V(y, x)
    torch.cuda.synchronize()
    yo = oracle.apply_Ut(res, b.T, "row").T
    xo = oracle.apply_V(res, yo.T, "col").T
    assert np.abs(y.cpu().numpy() - yo).max() <= 1e-12 * np.abs(b).max()
    assert np.abs(x.cpu().numpy() - xo).max() <= 1e-12 * np.abs(b).max()


@pytest.mark.parametrize("nrhs", [1, 8, 11, 32])
def test_apply_many_rhs_and_repeatable(nrhs):
    """The applies read each Q once per 8 right-hand sides (apply kernels'
    APPLY_RC): nrhs = 1, 8, 11 (a ragged chunk), 32 against the oracle, config-5
    recipe leaves (B = 128); and bitwise repeatable over 10 runs (the upward pass
    continues through atomic arrival counters -- a race would show here;
    compute-sanitizer is closed on this pool)."""
    _need_gpu()
    h = h2gen.make_config(5, N=8192)
    plan, sp, out = _run(h)
    res = oracle.sparsify(h)
    b = np.random.default_rng(nrhs).standard_normal((nrhs, h.N))
    bt = torch.from_numpy(b).cuda()
    y = torch.empty_like(bt)
    x = torch.empty_like(bt)
    sp.apply_Ut(bt, y)
    sp.apply_V(y, x)
    torch.cuda.synchronize()
    yo = oracle.apply_Ut(res, b.T, "row").T
    xo = oracle.apply_V(res, yo.T, "col").T
    assert np.abs(y.cpu().numpy() - yo).max() <= 1e-12 * np.abs(b).max()
    assert np.abs(x.cpu().numpy() - xo).max() <= 1e-12 * np.abs(b).max()
    y0, x0 = y.clone(), x.clone()
    for _ in range(10):
        sp.apply_Ut(bt, y)
        sp.apply_V(y, x)
        torch.cuda.synchronize()
        assert torch.equal(y, y0) and torch.equal(x, x0)


def test_solve_through_gpu_factors():
    """x = V S^-1 U^T b equals A_H2^-1 b (Eq. sp0) using GPU apply and GPU S."""
    _need_gpu()
    import scipy.sparse as sps
    import scipy.sparse.linalg as spla
    h = h2gen.random_h2(4, 16, 31, True, eta=0.7, spd_shift=60.0)
    plan, sp, out = _run(h)
    nnz = plan.sizes["s_nnz"]
    S = sps.csr_matrix((out["s_val"][:nnz].cpu().numpy(), out["s_col"][:nnz].cpu().numpy(),
                        out["s_rowptr"].cpu().numpy()), shape=(h.N, h.N))
    b = np.random.default_rng(4).standard_normal((1, h.N))
    bt = torch.from_numpy(b).cuda()
    y = torch.empty_like(bt)
    sp.apply_Ut(bt, y)
    z = spla.spsolve(S.tocsc(), y.cpu().numpy()[0])
    x = torch.empty_like(bt)
    sp.apply_V(torch.from_numpy(z[None, :]).cuda(), x)
    A = oracle.dense_A(h)
    xa = np.linalg.solve(A, b[0])
    assert np.linalg.norm(x.cpu().numpy()[0] - xa) / np.linalg.norm(xa) <= np.linalg.cond(A) * 1e-14


def test_build_is_deterministic_and_repeatable():
    _need_gpu()
    h = h2gen.random_h2(5, 16, 40, False, eta=0.7)
    plan, sp, out = _run(h)
    v1 = out["s_val"].clone()
    sp.build()
    torch.cuda.synchronize()
    assert torch.equal(v1, out["s_val"])


def test_build_host_e2e():
    """h2sp_build_host: host inputs -> device -> host outputs equals the device path."""
    _need_gpu()
    import paper_1705_04601_b200 as h2sp
    h = h2gen.random_h2(5, 16, 41, False, eta=0.7)
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed)
    sp = h2sp.Sparsifier(plan, packed)
    ref = {k: (v.clone() if v is not None else None) for k, v in sp.build().items()}
    host_in = {k: v.cpu().pin_memory() for k, v in sp.inputs.items()}
    host_out = {k: (torch.empty_like(v, device="cpu").pin_memory() if v is not None else None)
                for k, v in sp.outputs.items()}
    sp.build_host(host_in, host_out)
    torch.cuda.synchronize()
    for k in ("s_val", "s_col", "s_rowptr", "q_row", "q_col"):
        assert torch.equal(host_out[k], ref[k].cpu()), k


def test_parity_config2_full():
    """BASELINE configs[1] at full size (N = 65536), the bench workload: full S,
    all Q blocks against the oracle."""
    _need_gpu()
    h = h2gen.make_config(2)
    plan, sp, out = _run(h)
    res, v, err = _compare(h, plan, out)
    # Frobenius invariance (P5) of the GPU S
    f = oracle.frobenius_sq(h)
    assert abs(float(np.dot(v, v)) - f) / f <= 1e-12


@pytest.mark.parametrize("name,make,G", [
    ("cfg2-4096-sym", lambda: h2gen.make_config(2, N=4096), 4),
    ("cfg4-8192-gen", lambda: h2gen.make_config(4, N=8192), 2),
    ("rand-gen-uniform", lambda: h2gen.random_h2(6, 8, 4, False, eta=0.7, ragged=False, r=4), 4),
])
def test_virtual_shards_bitwise(name, make, G):
    """SURVEY §8(e) on one GPU: the G subtree shards, built one after the other,
    give exactly (bitwise) the unsharded S rows; sharded apply U^T b / V y equals
    the unsharded apply on the shard's rows.  Also checked against the oracle."""
    _need_gpu()
    import paper_1705_04601_b200 as h2sp
    h = make()
    packed = h2gen.pack(h)
    plan, sp, out = _run(h)
    _compare(h, plan, out)
    full_val = out["s_val"].cpu().numpy()
    frow = out["s_rowptr"].cpu().numpy()
    rng = np.random.default_rng(9)
    b = rng.standard_normal((2, h.N))
    bt = torch.from_numpy(b).cuda()
    yf = torch.empty_like(bt)
    sp.apply_Ut(bt, yf)
    xf = torch.empty_like(bt)
    sp.apply_V(yf, xf)
    seen = np.zeros(h.N, dtype=np.int64)
    for g in range(G):
        sh = h2sp.Plan(packed, g, G)
        ssp = h2sp.Sparsifier(sh, packed)
        o = ssp.build()
        torch.cuda.synchronize()
        rp = o["s_rowptr"].cpu().numpy()
        val = o["s_val"].cpu().numpy()
        gr = sh.global_rows()
        for lr, r in enumerate(gr):
            seen[r] += 1
            assert np.array_equal(val[rp[lr]:rp[lr + 1]], full_val[frow[r]:frow[r + 1]]), (g, r)
        lo = sh.sizes["first_leaf"] * h.B
        bl = bt[:, lo:lo + sh.n_tree_local].contiguous()
        yl = torch.empty(2, sh.s_rows, dtype=torch.float64, device="cuda")
        ssp.apply_Ut(bl, yl)
        torch.cuda.synchronize()
        assert torch.equal(yl.cpu(), yf[:, torch.from_numpy(gr)].cpu())
        xl = torch.empty_like(bl)
        ssp.apply_V(yf[:, torch.from_numpy(gr)].contiguous(), xl)
        torch.cuda.synchronize()
        assert torch.equal(xl.cpu(), xf[:, lo:lo + sh.n_tree_local].cpu())
    assert np.all(seen == 1)


@pytest.mark.parametrize("name,make", [
    ("rand-B16-sym", lambda: h2gen.random_h2(5, 16, 50, True, eta=0.7)),
    ("rand-B64-gen-wy", lambda: h2gen.random_h2(4, 64, 51, False, eta=0.7, max_rank=16)),  # compact-WY path
    ("rand-B128-sym", lambda: h2gen.random_h2(5, 128, 52, True, eta=0.7, max_rank=32)),
])
def test_graph_capture_replay_equals_direct(name, make):
    """The whole build (fork/join over the library's side streams) captured in a
    CUDA graph and replayed gives the direct build's S and Q bitwise; capture
    also proves every side-stream launch is joined back (an unjoined fork is a
    capture error)."""
    _need_gpu()
    import paper_1705_04601_b200 as h2sp
    h = make()
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed)
    sp = h2sp.Sparsifier(plan, packed)
    ref = {k: v.clone() for k, v in sp.build().items() if v is not None}
    torch.cuda.synchronize()
    for v in sp.outputs.values():
        if v is not None:
            v.zero_()
    g = sp.capture()
    g.replay()
    torch.cuda.synchronize()
    for k, v in ref.items():
        assert torch.equal(v, sp.outputs[k]), k


@pytest.mark.parametrize("sym", [True, False])
def test_build_apply_matches_separate_calls(sym):
    """h2sp_build_apply (applies on the QR side stream, overlapping the build)
    equals h2sp_build followed by h2sp_apply_Ut / h2sp_apply_V, bitwise."""
    _need_gpu()
    import paper_1705_04601_b200 as h2sp
    h = h2gen.random_h2(5, 16, 60 + sym, sym, eta=0.7)
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed)
    sp = h2sp.Sparsifier(plan, packed)
    b = torch.from_numpy(np.random.default_rng(5).standard_normal((2, h.N))).cuda()
    y1, x1 = torch.empty_like(b), torch.empty_like(b)
    sp.build()
    sp.apply_Ut(b, y1)
    sp.apply_V(y1, x1)
    torch.cuda.synchronize()
    s1 = sp.outputs["s_val"].clone()
    y2, x2 = torch.zeros_like(b), torch.zeros_like(b)
    aws = sp.apply_workspace(2)
    sp.build_apply(b, y2, y2, x2, aws)
    torch.cuda.synchronize()
    assert torch.equal(s1, sp.outputs["s_val"])
    assert torch.equal(y1, y2) and torch.equal(x1, x2)
    # independent w: V w runs beside U^T b on its own stream
    w = torch.from_numpy(np.random.default_rng(6).standard_normal((2, h.N))).cuda()
    x3 = torch.empty_like(b)
    sp.apply_V(w, x3)
    y4, x4 = torch.zeros_like(b), torch.zeros_like(b)
    sp.build_apply(b, y4, w, x4, aws)
    torch.cuda.synchronize()
    assert torch.equal(y1, y4) and torch.equal(x3, x4)


@pytest.mark.parametrize("name", ["cfg2-16384", "cfg3-16384", "rand-gen-B64"])
def test_explicit_q_and_wy_agree(name):
    """Both level-0 congruence variants (compact-WY, default; explicit Q with
    H2SP_PLAN_EXPLICIT_Q) match the oracle, and each other to rounding."""
    _need_gpu()
    if name == "cfg2-16384":
        h = h2gen.make_config(2, N=16384)
    elif name == "cfg3-16384":
        h = h2gen.make_config(3, N=16384)
    else:
        h = h2gen.random_h2(4, 64, 31, False, eta=0.7, max_rank=16)
    res = oracle.sparsify(h)
    outs = []
    for ex in (False, True):
        plan, sp, out = _run(h, explicit_q=ex)
        lv0 = [l for l in plan.launches() if l["kind"] == "congruence" and l["level"] == 0][0]
        if ex:
            assert lv0["flops_exec"] == lv0["flops"]
        _compare(h, plan, out, res)
        outs.append(out["s_val"].cpu().numpy())
    a, b = outs
    assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b)


@pytest.mark.parametrize("cfg,N", [(1, None), (2, 16384), (3, 16384), (4, 16384), (5, 16384)],
                         ids=["cfg1", "cfg2-16384", "cfg3-16384", "cfg4-16384", "cfg5-16384"])
def test_close_gen_matches_stored_close(cfg, N):
    """Matrix-free close blocks (h2sp_close_gen, SURVEY §8(d) config-5 protocol
    step 1): the level-0 congruence evaluates C_ts from the tree-ordered points.
    S matches the oracle (run on the generator's stored blocks) and the
    stored-close GPU build to rounding (one-ulp differences of exp / sqrt /
    division between numpy and the device); Q does not depend on C (bitwise)."""
    _need_gpu()
    import paper_1705_04601_b200 as h2sp
    h = h2gen.make_config(cfg, N=N)
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed)
    ref = {k: (v.clone() if v is not None else None) for k, v in h2sp.Sparsifier(plan, packed).build().items()}
    sp = h2sp.Sparsifier(plan, packed, close_gen={"points": h.points, "kernel": h.meta["kernel"]})
    assert "close" not in sp.inputs
    out = sp.build()
    torch.cuda.synchronize()
    _compare(h, plan, out)
    assert torch.equal(out["q_row"], ref["q_row"])
    if not h.symmetric:
        assert torch.equal(out["q_col"], ref["q_col"])
    assert torch.equal(out["s_col"], ref["s_col"]) and torch.equal(out["s_rowptr"], ref["s_rowptr"])
    a, b = out["s_val"], ref["s_val"]
    assert float(torch.linalg.norm(a - b)) <= 1e-13 * float(torch.linalg.norm(b))
    if h.symmetric:
        import scipy.sparse as sps
        nnz = plan.sizes["s_nnz"]
        S = sps.csr_matrix((a[:nnz].cpu().numpy(), out["s_col"][:nnz].cpu().numpy(),
                            out["s_rowptr"].cpu().numpy()), shape=(h.N, h.N))
        assert (S != S.T).nnz == 0


def test_close_gen_shards_and_graph_bitwise():
    """close_gen composes with the subtree shards (each shard reads
    its neighbours' points) and with graph capture: shard rows and the replayed
    graph equal the unsharded close_gen build bitwise."""
    _need_gpu()
    import paper_1705_04601_b200 as h2sp
    h = h2gen.make_config(5, N=16384, with_close=False)
    packed = h2gen.pack(h)
    gen = {"points": h.points, "kernel": h.meta["kernel"]}
    plan = h2sp.Plan(packed)
    sp = h2sp.Sparsifier(plan, packed, close_gen=gen)
    ref = {k: v.clone() for k, v in sp.build().items() if v is not None}
    torch.cuda.synchronize()
    full_val = ref["s_val"].cpu().numpy()
    frow = ref["s_rowptr"].cpu().numpy()
    G = 4
    seen = np.zeros(h.N, dtype=np.int64)
    for g in range(G):
        sh = h2sp.Plan(packed, g, G)
        o = h2sp.Sparsifier(sh, packed, close_gen=gen).build()
        torch.cuda.synchronize()
        rp, val = o["s_rowptr"].cpu().numpy(), o["s_val"].cpu().numpy()
        for lr, r in enumerate(sh.global_rows()):
            seen[r] += 1
            assert np.array_equal(val[rp[lr]:rp[lr + 1]], full_val[frow[r]:frow[r + 1]]), (g, r)
    assert np.all(seen == 1)
    for v in sp.outputs.values():
        if v is not None:
            v.zero_()
    gr = sp.capture()
    gr.replay()
    torch.cuda.synchronize()
    for k, v in ref.items():
        assert torch.equal(v, sp.outputs[k]), k


def test_close_gen_build_host_e2e():
    """h2sp_build_host in close_gen mode: the host points are copied in and the
    outputs equal the device-resident close_gen build bitwise."""
    _need_gpu()
    import paper_1705_04601_b200 as h2sp
    h = h2gen.make_config(5, N=4096)
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed)
    sp = h2sp.Sparsifier(plan, packed, close_gen={"points": h.points, "kernel": h.meta["kernel"]})
    ref = {k: (v.clone() if v is not None else None) for k, v in sp.build().items()}
    host_in = {k: v.cpu().pin_memory() for k, v in sp.inputs.items()}
    sp.inputs["points"].zero_()
    host_out = {k: (torch.empty_like(v, device="cpu").pin_memory() if v is not None else None)
                for k, v in sp.outputs.items()}
    sp.build_host(host_in, host_out)
    torch.cuda.synchronize()
    for k in ("s_val", "s_col", "s_rowptr", "q_row"):
        assert torch.equal(host_out[k], ref[k].cpu()), k


@pytest.mark.parametrize("cfg,N", [(2, 16384), (3, 16384), (5, 16384)])
def test_device_couplings_match_generator(cfg, N):
    """SURVEY §8(f) #2, first piece of GPU H^2 construction: h2sp_eval_kernel_blocks
    evaluates the interpolation couplings D_b = K(nodes_t, nodes_s) on the device.
    They match the generator's numpy values to rounding, D_st = D_ts^T bitwise in
    symmetric mode, and a build fed with them matches the oracle."""
    _need_gpu()
    import paper_1705_04601_b200 as h2sp
    h = h2gen.make_config(cfg, N=N)
    packed = h2gen.pack(h)
    xr, xc, desc, n = h2gen.coupling_block_descs(h)
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    h2sp.eval_kernel_blocks(h.meta["kernel"], torch.from_numpy(xr).cuda(), torch.from_numpy(xc).cuda(),
                            torch.from_numpy(desc).cuda(), dev)
    torch.cuda.synchronize()
    ref = torch.from_numpy(packed["coupling"]).cuda()
    assert float(torch.linalg.norm(dev - ref)) <= 1e-14 * float(torch.linalg.norm(ref))
    if h.symmetric:
        from h2gen import lvl_off
        d = desc
        pos = {}
        i = 0
        for k in range(h.L):
            for (t, s) in h.adm[k]:
                pos[(k, int(t), int(s))] = i
                i += 1
        dv = dev.cpu().numpy()
        for (k, t, s), b in list(pos.items())[:4000]:
            if t < s:
                b2 = pos[(k, s, t)]
                nx, ny = int(d[b, 3] & 0xffffffff), int(d[b, 3] >> 32)
                A = dv[d[b, 2]:d[b, 2] + nx * ny].reshape(nx, ny)
                Bm = dv[d[b2, 2]:d[b2, 2] + nx * ny].reshape(ny, nx)
                assert np.array_equal(A, Bm.T)
    plan = h2sp.Plan(packed)
    sp = h2sp.Sparsifier(plan, packed)
    sp.inputs["coupling"][:n].copy_(dev)
    out = sp.build()
    torch.cuda.synchronize()
    _compare(h, plan, out)


def _csr_spmv(out, nnz, n_rows, z, chunks=16):
    """S z with S the GPU CSR output (test infrastructure: torch sparse SpMV over
    row chunks, int32 column indices widened per chunk)."""
    rowptr = out["s_rowptr"]
    res = torch.empty(n_rows, dtype=torch.float64, device=z.device)
    step = (n_rows + chunks - 1) // chunks
    for r0 in range(0, n_rows, step):
        r1 = min(n_rows, r0 + step)
        p0, p1 = int(rowptr[r0]), int(rowptr[r1])
        crow = (rowptr[r0:r1 + 1] - p0).contiguous()
        col = out["s_col"][p0:p1].long()
        val = out["s_val"][p0:p1]
        A = torch.sparse_csr_tensor(crow, col, val, size=(r1 - r0, z.shape[0]))
        res[r0:r1] = torch.mv(A, z)
        del A, col
    return res


def test_config3_full_size_properties():
    """BASELINE configs[2] at its full size (N = 262144; 4.8e9 nnz of S): the
    oracle's O1 pass is out of reach, so the GPU factors are checked through
    properties that hold at any size -- P5 ||S||_F^2 = ||A_H2||_F^2 (Gram
    recursion on the H^2 parameters, QR-independent) and P13 U S U^T x = A_H2 x
    (GPU applies + a CSR SpMV of the GPU S against the oracle's H^2 matvec)."""
    _need_gpu()
    h = h2gen.make_config(3)
    plan, sp, out = _run(h)
    nnz = plan.sizes["s_nnz"]
    v = out["s_val"][:nnz]
    f = oracle.frobenius_sq(h)
    fs = sum(float(torch.dot(c, c)) for c in v.split(1 << 30))   # BLAS dot takes < 2^31 elements
    assert abs(fs - f) / f <= 1e-12
    x = np.random.default_rng(7).standard_normal(h.N)
    xt = torch.from_numpy(x[None, :]).cuda()
    y = torch.empty_like(xt)
    sp.apply_Ut(xt, y)
    z = _csr_spmv(out, nnz, plan.s_rows, y[0])
    w = torch.empty_like(xt)
    sp.apply_V(z[None, :].contiguous(), w)
    ref = oracle.h2_matvec(h, x)
    assert np.linalg.norm(w.cpu().numpy()[0] - ref) / np.linalg.norm(ref) <= 1e-12


def test_config4_general_mode_properties():
    """BASELINE configs[3] recipe (sphere, general mode U != V, r = B/2) at
    N = 65536, beyond the oracle's O1 pass: P5 ||S||_F^2 = ||A_H2||_F^2 and the
    defining identity S y = U^T A_H2 V y (GPU apply_V, the oracle's H^2 matvec,
    GPU apply_Ut) against a CSR SpMV of the GPU S."""
    _need_gpu()
    h = h2gen.make_config(4, N=65536)
    assert not h.symmetric
    plan, sp, out = _run(h)
    nnz = plan.sizes["s_nnz"]
    v = out["s_val"][:nnz]
    f = oracle.frobenius_sq(h)
    fs = sum(float(torch.dot(c, c)) for c in v.split(1 << 30))
    assert abs(fs - f) / f <= 1e-12
    y = np.random.default_rng(8).standard_normal(h.N)
    yt = torch.from_numpy(y[None, :]).cuda()
    vy = torch.empty_like(yt)
    sp.apply_V(yt, vy)
    avy = torch.from_numpy(oracle.h2_matvec(h, vy.cpu().numpy()[0])[None, :]).cuda()
    lhs = torch.empty_like(yt)
    sp.apply_Ut(avy, lhs)
    sy = _csr_spmv(out, nnz, plan.s_rows, yt[0])
    assert float(torch.linalg.norm(lhs[0] - sy) / torch.linalg.norm(sy)) <= 1e-12


def _general_mode_properties(h, qsample=64):
    """P5 (||S||_F^2 = ||A_H2||_F^2), the defining identity S y = U^T A_H2 V y
    (GPU applies, the oracle's H^2 matvec, a CSR SpMV of the GPU S) and the
    orthogonality of a sample of GPU Q blocks -- properties independent of
    which complement the Householder tie-breaks pick (reading 2)."""
    plan, sp, out = _run(h)
    nnz = plan.sizes["s_nnz"]
    v = out["s_val"][:nnz]
    f = oracle.frobenius_sq(h)
    fs = sum(float(torch.dot(c, c)) for c in v.split(1 << 30))
    assert abs(fs - f) / f <= 1e-12, (fs, f)
    y = np.random.default_rng(8).standard_normal(h.N)
    yt = torch.from_numpy(y[None, :]).cuda()
    vy = torch.empty_like(yt)
    sp.apply_V(yt, vy)
    avy = torch.from_numpy(oracle.h2_matvec(h, vy.cpu().numpy()[0])[None, :]).cuda()
    lhs = torch.empty_like(yt)
    sp.apply_Ut(avy, lhs)
    sy = _csr_spmv(out, nnz, plan.s_rows, yt[0])
    assert float(torch.linalg.norm(lhs[0] - sy) / torch.linalg.norm(sy)) <= 1e-12
    off = plan.offsets()
    rng = np.random.default_rng(3)
    for side, q, n_ in (("row", out["q_row"], off["n_row"]), ("col", out["q_col"], off["n_col"])):
        key = "q_off_row" if side == "row" else "q_off_col"
        cl = np.nonzero(n_ > 0)[0]
        for c in rng.choice(cl, size=min(qsample, len(cl)), replace=False):
            n = int(n_[c])
            Q = q[off[key][c]:off[key][c] + n * n].view(n, n)
            e = float((Q.T @ Q - torch.eye(n, dtype=Q.dtype, device=Q.device)).abs().max())
            assert e <= 1e-14 * n, (side, c, e)


def test_config4_raw_chebyshev_properties():
    """BASELINE configs[3]'s recipe with its RAW tensor Chebyshev bases (no
    orthonormalisation; leaf-basis condition ~1e8 on the sphere, Householder
    alpha at round-off level: parity with the oracle is ill-posed there,
    reading 2) -- the GPU result is still exact: P5, S y = U^T A V y, Q orthogonal."""
    _need_gpu()
    h = h2gen.make_config(4, N=65536, orthonormalize=False)
    _general_mode_properties(h)


def test_config4_full_size_properties():
    """BASELINE configs[3] at its full size (N = 1,048,576, general mode, r = B/2)."""
    _need_gpu()
    if torch.cuda.get_device_properties(0).total_memory < 150 * 2 ** 30:
        pytest.skip("needs ~150 GB of device memory")
    import gc
    gc.collect()
    torch.cuda.empty_cache()   # earlier full-size tests' cached blocks
    h = h2gen.make_config(4)
    _general_mode_properties(h, qsample=256)


def test_device_direct_solve():
    """x = V S^-1 U^T b on the device (GPU applies + a sparse
    Cholesky of the GPU S in its own level-major order) solves A_H2 x = b; the
    residual is measured with the oracle's independent H^2 matvec (Eq. sp0)."""
    _need_gpu()
    from paper_1705_04601_b200 import solve as hs
    h = h2gen.make_config(2, N=4096)
    plan, sp, out = _run(h)
    chol = hs.factor(sp, plan)
    b = np.random.default_rng(9).standard_normal(h.N)
    x = hs.solve(sp, chol, torch.from_numpy(b).cuda()).cpu().numpy()
    r = oracle.h2_matvec(h, x) - b
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 1e-10
