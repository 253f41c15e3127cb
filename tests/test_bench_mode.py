"""Bench mode (H2SP_PLAN_BENCH, include/h2sp.h h2sp_outputs): S reduced in the
congruence / strip epilogues to y = S w and the row norms ||S[i,:]||^2 instead
of being stored (SURVEY §8(d) config-5 protocol step 3).

Expected values come from the oracle's S (oracle.sparsify + oracle.s_csr) times
the same seeded w (a library sparse mat-vec): ||y_gpu - S_orc w|| / ||S_orc w||
<= 1e-11 and likewise for the row norms -- the S tolerance of BASELINE.json
north_star carried through one product.  The stored-mode GPU S times w agrees
to ~1e-14 (same arithmetic, different summation), and the reductions are
bitwise reproducible and bitwise independent of the virtual-shard count."""
import numpy as np
import pytest

import h2gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


CASES = [
    ("rand-sym-B16", lambda: h2gen.random_h2(5, 16, 1, True, eta=0.7)),
    ("rand-gen-B16", lambda: h2gen.random_h2(5, 16, 2, False, eta=0.7)),
    ("rand-B40-gen-ragged", lambda: h2gen.random_h2(5, 40, 9, False, eta=0.5, max_rank=32)),
    ("rand-B24-sym-uniform", lambda: h2gen.random_h2(5, 24, 10, True, eta=0.7, ragged=False, r=12)),
    ("fig3-half", lambda: h2gen.fig3_h2(8, 0, "half")),
    ("cfg2-8192", lambda: h2gen.make_config(2, N=8192)),        # compact-WY level 0 (B = 64)
    ("cfg3-8192", lambda: h2gen.make_config(3, N=8192)),        # 48-wide internal tiles
    ("cfg4-8192", lambda: h2gen.make_config(4, N=8192)),        # general mode, column strips
    ("rand-B128-sym", lambda: h2gen.random_h2(5, 128, 6, True, eta=0.7, max_rank=32)),
    ("cfg5-16384", lambda: h2gen.make_config(5, N=16384)),      # config-5 recipe: B = 128, r = 32
]


def _oracle_S(h):
    import scipy.sparse as sps
    res = oracle.sparsify(h)
    rowptr, col, val = oracle.s_csr(res)
    return sps.csr_matrix((val, col, rowptr), shape=(h.N, h.N))


def _bench(h, w, close_gen=None, shards=1, share_qr=True, want_q=False):
    import paper_1705_04601_b200 as h2sp
    packed = h2gen.pack(h)
    if shards == 1:
        plan = h2sp.Plan(packed, bench=True)
        sp = h2sp.Sparsifier(plan, packed, close_gen=close_gen)
        sp.outputs["bench_w"].copy_(torch.from_numpy(w))
        sp.outputs["bench_y"].fill_(np.nan)
        sp.outputs["bench_r2"].fill_(np.nan)
        sp.build()
        torch.cuda.synchronize()
        return sp.outputs["bench_y"].cpu().numpy(), sp.outputs["bench_r2"].cpu().numpy(), plan
    plans = [h2sp.Plan(packed, g, shards, bench=True) for g in range(shards)]
    vs = h2sp.VirtualShards(plans, packed, close_gen=close_gen, share_qr=share_qr)
    vs.outputs["bench_w"].copy_(torch.from_numpy(w))
    vs.outputs["bench_y"].fill_(np.nan)
    vs.outputs["bench_r2"].fill_(np.nan)
    vs.build()
    torch.cuda.synchronize()
    if want_q:
        return (vs.outputs["bench_y"].cpu().numpy(), vs.outputs["bench_r2"].cpu().numpy(),
                vs.outputs["q_row"].cpu().numpy())
    return vs.outputs["bench_y"].cpu().numpy(), vs.outputs["bench_r2"].cpu().numpy(), plans[0]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_bench_y_and_row_norms_vs_oracle(name, make):
    _need_gpu()
    h = make()
    w = np.random.default_rng(7).standard_normal(h.N)
    y, r2, plan = _bench(h, w)
    S = _oracle_S(h)
    y_ref = S @ w
    r2_ref = np.asarray(S.multiply(S).sum(axis=1)).ravel()
    assert np.all(np.isfinite(y)) and np.all(np.isfinite(r2))   # every row written
    ey = np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref)
    er = np.linalg.norm(r2 - r2_ref) / np.linalg.norm(r2_ref)
    assert ey <= 1e-11, ey
    assert er <= 1e-11, er
    # per level of the S row's cluster: no block row family hides below the global norm
    off = plan.offsets()
    L = h.L
    for k in range(L + 1):
        lo = off["s_off_row"][h2gen.lvl_off(L, k)]
        hi = off["s_off_row"][h2gen.lvl_off(L, k + 1)] if k < L else h.N
        if hi > lo and np.linalg.norm(r2_ref[lo:hi]) > 0:
            assert np.linalg.norm(r2[lo:hi] - r2_ref[lo:hi]) <= 1e-11 * np.linalg.norm(r2_ref[lo:hi]), k


def test_bench_matches_stored_gpu_S_and_is_reproducible():
    _need_gpu()
    import paper_1705_04601_b200 as h2sp
    h = h2gen.make_config(5, N=16384)
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed)
    sp = h2sp.Sparsifier(plan, packed)
    out = sp.build()
    torch.cuda.synchronize()
    import scipy.sparse as sps
    nnz = plan.sizes["s_nnz"]
    S = sps.csr_matrix((out["s_val"][:nnz].cpu().numpy(), out["s_col"][:nnz].cpu().numpy(),
                        out["s_rowptr"].cpu().numpy()), shape=(h.N, h.N))
    w = np.random.default_rng(3).standard_normal(h.N)
    y1, r1, _ = _bench(h, w)
    y2, r2, _ = _bench(h, w)
    assert np.array_equal(y1, y2) and np.array_equal(r1, r2)      # no atomics: bitwise reproducible
    y_ref = S @ w
    assert np.linalg.norm(y1 - y_ref) <= 1e-13 * np.linalg.norm(y_ref)


@pytest.mark.parametrize("name,make,G", [
    ("cfg5-16384", lambda: h2gen.make_config(5, N=16384), 4),
    ("cfg2-8192", lambda: h2gen.make_config(2, N=8192), 8),
    ("cfg4-8192", lambda: h2gen.make_config(4, N=8192), 2),
])
def test_virtual_shards_bitwise(name, make, G):
    """G virtual shards (h2sp_build_meta on one scratch buffer) give the
    unsharded y and row norms bit for bit (output independent of G)."""
    _need_gpu()
    h = make()
    w = np.random.default_rng(11).standard_normal(h.N)
    y1, r1, _ = _bench(h, w)
    yg, rg, _ = _bench(h, w, shards=G)
    assert np.array_equal(y1, yg)
    assert np.array_equal(r1, rg)


@pytest.mark.parametrize("name,make,G", [
    ("cfg5-16384", lambda: h2gen.make_config(5, N=16384), 8),
    ("cfg4-8192", lambda: h2gen.make_config(4, N=8192), 4),
])
def test_shared_qr_pass_is_bitwise_the_per_shard_qr(name, make, G):
    """Protocol step 2 (the QR pass runs once for all clusters): the
    first shard's build with H2SP_QR_ALL and the others with H2SP_QR_REUSE give
    the y, row norms and Q of builds that each repeat the QR of their need set."""
    _need_gpu()
    h = make()
    w = np.random.default_rng(13).standard_normal(h.N)
    ya, ra, qa = _bench(h, w, shards=G, share_qr=True, want_q=True)
    yb, rb, qb = _bench(h, w, shards=G, share_qr=False, want_q=True)
    assert np.array_equal(ya, yb) and np.array_equal(ra, rb)
    assert np.array_equal(qa, qb)   # every shard's need sets together cover the Q the applies read


def test_bench_close_gen_matrix_free_couplings():
    """Config-5 protocol inputs: matrix-free close blocks AND couplings
    (h2sp_close_gen.nodes_row) -- nothing but points, nodes and bases stored."""
    _need_gpu()
    h = h2gen.make_config(5, N=16384)
    w = np.random.default_rng(5).standard_normal(h.N)
    xr, xc, _, _ = h2gen.coupling_block_descs(h)
    gen = {"points": h.points, "kernel": h.meta["kernel"], "nodes_row": xr}
    y, r2, _ = _bench(h, w, close_gen=gen)
    S = _oracle_S(h)
    y_ref = S @ w
    r2_ref = np.asarray(S.multiply(S).sum(axis=1)).ravel()
    assert np.linalg.norm(y - y_ref) <= 1e-11 * np.linalg.norm(y_ref)
    assert np.linalg.norm(r2 - r2_ref) <= 1e-11 * np.linalg.norm(r2_ref)
