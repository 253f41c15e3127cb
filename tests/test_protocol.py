"""The config-5 protocol checked through properties that hold at
any size, at N = 262,144 and at BASELINE configs[4]'s full N = 4,194,304 --
in the launch configuration bench.py times (8 virtual shards, device-built
inputs, matrix-free close blocks and couplings, bench-mode S):

* P5 per rank-0 subtree: for a cluster c with k_c = 0 the S rows of c's
  subtree carry ||A_H2[I_c, :]||_F^2 (oracle.frobenius_sq_rows, evaluated from
  the points, nodes and numpy bases of the generator); at N = 262,144 also the
  whole ||S||_F^2 = ||A_H2||_F^2.
* P13 on a sample: U (S (U^T x)) = A_H2 x on sampled leaves' rows
  (oracle.h2_matvec_rows), with U^T x, S w and U y all from the GPU path.
* every row written (finite y and row norms), structure counts of the plan.
"""
import numpy as np
import pytest

import h2gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _need_gpu(min_gb=0):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if min_gb and torch.cuda.get_device_properties(0).total_memory < min_gb * 2 ** 30:
        pytest.skip(f"needs {min_gb} GB of device memory")


def _rank0_level(h):
    L = h.L
    kr = np.asarray(h.rank_row)
    for lev in range(L + 1):
        if not kr[h2gen.lvl_off(L, lev):h2gen.lvl_off(L, lev) + (1 << (L - lev))].any():
            return lev
    return L


def _subtree_rows(plan, L, level, index):
    off = plan.offsets()
    m = np.diff(np.append(off["s_off_row"], plan.N))
    rows = []
    for k in range(level + 1):
        for t in range(index << (level - k), (index + 1) << (level - k)):
            c = h2gen.cid(L, k, t)
            rows.append(np.arange(off["s_off_row"][c], off["s_off_row"][c] + m[c]))
    return np.concatenate(rows)


def _protocol_checks(N, n_subtrees, n_leaves_sample, whole=False):
    from paper_1705_04601_b200.protocol import ProtocolRun
    h = h2gen.make_structure(5, N=N)
    run = ProtocolRun(h, V=8)
    dev = run.device
    # (1) one pass with U^T x through the applies (and any w): Q, row norms, U^T x
    x = np.random.default_rng(21).standard_normal(h.N)
    xt = torch.from_numpy(x).to(dev)
    applies = []
    for i, p in enumerate(run.plans):
        a0, a1 = run.leaf_range(i)
        applies.append((xt[a0:a1].reshape(1, -1).contiguous(), torch.empty(1, p.s_rows, dtype=torch.float64,
                                                                            device=dev), None, None))
    run.outputs["bench_w"].zero_()
    run.build(applies)
    torch.cuda.synchronize()
    r2 = run.outputs["bench_r2"].cpu().numpy()
    assert np.all(np.isfinite(r2))
    w = np.zeros(h.N)
    for i, ap in enumerate(applies):
        w[run.global_rows(i)] = ap[1].cpu().numpy().ravel()
    # (2) y = S w with w = U^T x (bench mode)
    run.outputs["bench_w"].copy_(torch.from_numpy(w))
    run.outputs["bench_y"].fill_(np.nan)
    run.build()
    torch.cuda.synchronize()
    y = run.outputs["bench_y"].cpu().numpy()
    assert np.all(np.isfinite(y))
    # (3) U y through the V apply of a third pass (symmetric: V = U)
    yt = torch.from_numpy(y).to(dev)
    applies = []
    for i, p in enumerate(run.plans):
        a0, a1 = run.leaf_range(i)
        gr = torch.from_numpy(run.global_rows(i)).to(dev)
        applies.append((None, None, yt[gr].reshape(1, -1).contiguous(),
                        torch.empty(1, a1 - a0, dtype=torch.float64, device=dev)))
    run.build(applies)
    torch.cuda.synchronize()
    ux = np.zeros(h.N)
    for i, ap in enumerate(applies):
        a0, a1 = run.leaf_range(i)
        ux[a0:a1] = ap[3].cpu().numpy().ravel()
    plan0 = run.plans[0]
    del run
    torch.cuda.empty_cache()
    # ---- oracle side: numpy bases of the same recipe, C / D evaluated on the fly
    h2gen.fill_cheb_bases(h)
    lev = _rank0_level(h)
    M = 1 << (h.L - lev)
    for index in sorted({0, M - 1, M // 3})[:n_subtrees]:
        ref = oracle.frobenius_sq_rows(h, lev, index)
        got = float(np.sum(r2[_subtree_rows(plan0, h.L, lev, index)]))
        assert abs(got - ref) <= 1e-12 * ref, (lev, index, got, ref)
    if whole:   # the root has rank 0: the whole ||S||_F^2 = ||A_H2||_F^2
        ref = oracle.frobenius_sq_rows(h, h.L, 0)
        assert abs(float(np.sum(r2)) - ref) <= 1e-12 * ref
    nl = h.N // h.B
    leaves = sorted(set(np.random.default_rng(5).integers(0, nl, n_leaves_sample).tolist()) | {0, nl - 1})
    Ax = oracle.h2_matvec_rows(h, x, leaves)
    rms = np.sqrt(np.mean([np.sum(v ** 2) for v in Ax.values()]))   # typical ||(A x)[leaf]||
    for leaf, ref in Ax.items():
        got = ux[leaf * h.B:(leaf + 1) * h.B]
        # P13: relative to the scale of A x (north_star 1e-12 on the whole vector)
        assert np.linalg.norm(got - ref) <= 1e-12 * max(np.linalg.norm(ref), rms), leaf


def test_protocol_config5_N262144():
    _need_gpu()
    _protocol_checks(262144, n_subtrees=3, n_leaves_sample=16, whole=True)


def test_protocol_config5_full_size():
    """BASELINE configs[4] at its full size, N = 4,194,304 (L = 15)."""
    _need_gpu(min_gb=160)
    _protocol_checks(4194304, n_subtrees=2, n_leaves_sample=8)
