"""Host-side checks of the C-ABI library (no GPU needed): exported symbols,
and the symbolic plan (S order, S pattern, CSR) against the oracle bitwise."""
import ctypes

import numpy as np
import pytest

import h2gen
import oracle
import paper_1705_04601_b200 as h2sp


def test_library_exports_every_declared_symbol():
    names = h2sp.declared_symbols()
    assert len(names) >= 12
    for n in names:
        assert hasattr(h2sp.lib, n), n
        ctypes.cast(getattr(h2sp.lib, n), ctypes.c_void_p)


def _cases():
    yield "cfg1", lambda: h2gen.make_config(1)
    yield "cfg2-4096", lambda: h2gen.make_config(2, N=4096)
    for sym in (True, False):
        for seed, eta in ((0, 0.4), (1, 0.7), (2, 1.5)):
            yield f"rand-{'sym' if sym else 'gen'}-{seed}", (lambda sym=sym, seed=seed, eta=eta:
                                                             h2gen.random_h2(5, 8, seed, sym, eta=eta))
    yield "fig3-half", lambda: h2gen.fig3_h2(4, 0, "half")
    yield "fig3-active", lambda: h2gen.fig3_h2(4, 0, "active")
    yield "eta0", lambda: h2gen.eta0_h2(3, 4, 0)
    yield "axis-gen", lambda: h2gen.axis_aligned_h2(4, 8, 2, False)
    yield "L0", lambda: h2gen.eta0_h2(0, 16, 0)
    yield "rand-gen-B128", lambda: h2gen.random_h2(5, 128, 5, False, eta=0.7, max_rank=32)
    yield "rand-sym-B128", lambda: h2gen.random_h2(5, 128, 6, True, eta=0.7, max_rank=32)


CASES = list(_cases())


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_plan_structure_matches_oracle(name, make):
    h = make()
    res = oracle.sparsify(h)
    plan = h2sp.Plan(h2gen.pack(h))
    off = plan.offsets()
    assert np.array_equal(off["s_off_row"], res.off_row)
    assert np.array_equal(off["s_off_col"], res.off_col)
    assert np.array_equal(off["n_row"], res.n_row) and np.array_equal(off["n_col"], res.n_col)
    rowptr, col, val = oracle.s_csr(res)
    prow, pcol = plan.pattern()
    assert np.array_equal(prow, rowptr)
    assert np.array_equal(pcol, col)
    assert plan.sizes["s_nnz"] == len(val)
    assert plan.sizes["s_blocks"] == len(res.S)
    assert plan.sizes["q_row"] == sum(int(n) ** 2 for n in res.n_row)


def _struct_with(h, **kw):
    p = h2gen.pack(h)
    p.update(kw)
    return p


def test_plan_rejects_bad_structures():
    h = h2gen.random_h2(4, 8, 3, True, eta=0.7)
    p = h2gen.pack(h)
    # drop one near pair -> block tree no longer a partition / not symmetric
    npt, ncol = p["near_ptr"].copy(), p["near_col"].copy()
    ncol2 = np.delete(ncol, 1)
    npt2 = npt.copy()
    npt2[1:] -= 1
    npt2[0] = 0
    npt2 = np.maximum(npt2, 0)
    with pytest.raises(h2sp.H2spError) as e:
        h2sp.Plan(_struct_with(h, near_ptr=npt2, near_col=ncol2))
    assert e.value.status == 2
    # rank above the local size
    rr = p["rank_row"].copy()
    rr[0] = h.B + 1
    with pytest.raises(h2sp.H2spError) as e:
        h2sp.Plan(_struct_with(h, rank_row=rr, rank_col=rr))
    assert e.value.status == 3
    # nonzero root rank
    rr = p["rank_row"].copy()
    rr[-1] = 1
    with pytest.raises(h2sp.H2spError) as e:
        h2sp.Plan(_struct_with(h, rank_row=rr, rank_col=rr))
    assert e.value.status == 3
    # unsorted columns
    ncol3 = ncol.copy()
    r0 = slice(npt[0], npt[1])
    ncol3[r0] = ncol3[r0][::-1]
    if npt[1] - npt[0] > 1:
        with pytest.raises(h2sp.H2spError) as e:
            h2sp.Plan(_struct_with(h, near_col=ncol3))
        assert e.value.status == 2
    # a pair both near and admissible at level 1
    gen = h2gen.random_h2(4, 8, 4, False, eta=0.7)
    pg = h2gen.pack(gen)
    adm1 = set(map(tuple, gen.adm[1].tolist()))
    near1 = sorted({(t // 2, s // 2) for (t, s) in gen.near.tolist()} | {(t // 2, s // 2) for (t, s) in gen.adm[0].tolist()})
    extra = [x for x in near1 if x not in adm1][0]
    newadm = np.array(sorted(adm1 | {extra}), dtype=np.int32)
    M = 1 << (gen.L - 1)
    ptr = np.zeros(M + 1, dtype=np.int64)
    np.add.at(ptr, newadm[:, 0] + 1, 1)
    pg["adm_ptr"][1] = np.cumsum(ptr)
    pg["adm_col"][1] = newadm[:, 1].astype(np.int32)
    with pytest.raises(h2sp.H2spError) as e:
        h2sp.Plan(pg)
    assert e.value.status == 2


def test_plan_unsupported_leaf_size():
    """Leaves up to 128 points are supported through the compact-WY level-0
    congruence only (k <= 32); anything else is H2SP_EUNSUPPORTED (7)."""
    h2sp.Plan(h2gen.pack(h2gen.eta0_h2(1, 128, 0)))          # B = 128, k = 0: fine
    cases = [(h2gen.eta0_h2(1, 160, 0), {}),                   # n_t > 128
             (h2gen.eta0_h2(1, 128, 0), {"explicit_q": True}),  # no explicit-Q kernel for n_t > 64
             (h2gen.random_h2(5, 128, 1, True, eta=0.7, r=40, ragged=False), {})]  # k_t > 32 at B = 128
    for h, kw in cases:
        with pytest.raises(h2sp.H2spError) as e:
            h2sp.Plan(h2gen.pack(h), **kw)
        assert e.value.status == 7


@pytest.mark.parametrize("name,make", [c for c in CASES if c[0] in ("cfg1", "rand-sym-1", "rand-gen-2", "fig3-half")],
                         ids=lambda c: c if isinstance(c, str) else "")
def test_plan_flops_match_structural_count(name, make):
    """The plan's algorithmic flop count equals an independent count on the
    oracle's structure (bench.py's reference arm uses the latter)."""
    import bench
    h = make()
    res = oracle.sparsify(h)
    plan = h2sp.Plan(h2gen.pack(h))
    assert plan.sizes["flops"] == pytest.approx(bench._oracle_flops(res, h), rel=1e-12)
    assert sum(l["flops"] for l in plan.launches()) == pytest.approx(plan.sizes["flops"], rel=1e-12)


def test_sparsifier_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    h = h2gen.random_h2(3, 8, 0, True)
    plan = h2sp.Plan(h2gen.pack(h))
    with pytest.raises(RuntimeError):
        h2sp.Sparsifier(plan, h2gen.pack(h))


def test_binding_fails_loudly_without_library(tmp_path):
    """No CPU fallback: the package refuses to import without libh2sp.so."""
    import shutil
    import subprocess
    import sys
    pkg = tmp_path / "paper_1705_04601_b200"
    shutil.copytree(h2sp.__path__[0], pkg, ignore=shutil.ignore_patterns("*.so", "csrc", "__pycache__"))
    (tmp_path / "include").mkdir()
    r = subprocess.run([sys.executable, "-c", "import paper_1705_04601_b200"], cwd=tmp_path, capture_output=True,
                       text=True)
    assert r.returncode != 0 and "libh2sp.so" in r.stderr


def test_wy_congruence_flops():
    """Compact-WY level-0 congruence: executed flops 4 n_t n_s (k_t + k_s) per
    pair; the algorithmic count is unchanged; explicit_q disables it."""
    import paper_1705_04601_b200 as h2sp
    h = h2gen.make_config(2, N=4096, with_close=False)
    packed = h2gen.pack(h)
    for ex in (False, True):
        plan = h2sp.Plan(packed, explicit_q=ex)
        li = [l for l in plan.launches() if l["kind"] == "congruence" and l["level"] == 0][0]
        n, k = 64.0, 16.0
        assert li["flops"] == li["items"] * 2 * n * n * (2 * n)
        want = li["items"] * 4 * n * n * (2 * k) if not ex else li["flops"]
        assert li["flops_exec"] == want
        assert plan.sizes["flops_executed"] == pytest.approx(sum(l["flops_exec"] for l in plan.launches()))
        assert plan.sizes["flops"] == pytest.approx(sum(l["flops"] for l in plan.launches()))


def test_close_gen_descriptor_validation():
    """h2sp_close_gen (matrix-free close blocks) is validated before any device
    work: bad dim / kernel id / NULL points are H2SP_EINVAL (1); the binding maps
    the generator's kernel specs to the header's kernel ids."""
    h = h2gen.random_h2(3, 8, 0, True)
    plan = h2sp.Plan(h2gen.pack(h))
    ws = ctypes.create_string_buffer(int(plan.sizes["workspace_bytes"]) + 512)
    wsp = (ctypes.addressof(ws) + 255) // 256 * 256
    dummy = ctypes.c_double(0.0)
    dp = ctypes.addressof(dummy)
    pts = (ctypes.c_double * (3 * h.N))()
    for dim, kern, p, why in ((5, 1, ctypes.addressof(pts), b"dim"), (3, 9, ctypes.addressof(pts), b"kernel"),
                              (3, 1, None, b"points")):
        g = h2sp._CloseGen(points=p, dim=dim, kernel=kern, p0=0.1, p1=0.01)
        inp = h2sp._Inputs(leaf_basis_row=dp, transfer_row=dp, close=None, coupling=dp,
                           close_gen=ctypes.addressof(g))
        out = h2sp._Outputs(q_row=dp, s_val=dp)
        st = h2sp.lib.h2sp_build(plan.handle, ctypes.byref(inp), ctypes.byref(out), wsp,
                                 int(plan.sizes["workspace_bytes"]), None)
        assert st == 1, (dim, kern)
        assert why in h2sp.lib.h2sp_last_error()
    assert h2sp.close_gen_params({"kind": "exp", "ell": 0.05, "nugget": 1e-2}) == (1, 0.05, 1e-2)
    assert h2sp.close_gen_params({"kind": "invh", "h": 0.5, "diag_add": 1.0}) == (2, 0.5, 1.0)
    k, p0, p1 = h2sp.close_gen_params({"kind": "laplace", "h": 0.25})
    assert k == 3 and p1 == pytest.approx(1.0 / np.pi)


def test_coupling_block_descs_layout():
    """h2gen.coupling_block_descs (the input of h2sp_eval_kernel_blocks) describes
    exactly the generator's coupling layout: evaluating the kernel on the
    described node blocks on the host reproduces pack()'s `coupling` bitwise."""
    h = h2gen.make_config(2, N=4096)
    packed = h2gen.pack(h)
    xr, xc, desc, n = h2gen.coupling_block_descs(h)
    assert n == packed["coupling"].size
    out = np.empty(n)
    for x_off, y_off, o, nn in desc:
        nx, ny = int(nn & 0xffffffff), int(nn >> 32)
        out[o:o + nx * ny] = h2gen.kernel_matrix(h.meta["kernel"], xr[x_off:x_off + nx], xc[y_off:y_off + ny]).ravel()
    assert np.array_equal(out, packed["coupling"])


def test_qr_mode_validation():
    """h2sp_plan_set_qr_mode (include/h2sp.h): NEED / ALL / REUSE accepted, anything else H2SP_EINVAL."""
    import paper_1705_04601_b200 as h2sp
    h = h2gen.random_h2(3, 8, 0, True, eta=0.7)
    plan = h2sp.Plan(h2gen.pack(h))
    for mode in (h2sp.QR_NEED, h2sp.QR_ALL, h2sp.QR_REUSE, h2sp.QR_NEED):
        assert h2sp.lib.h2sp_plan_set_qr_mode(plan.handle, mode) == 0
    assert h2sp.lib.h2sp_plan_set_qr_mode(plan.handle, 7) != 0
    assert h2sp.lib.h2sp_plan_set_qr_mode(None, 0) != 0
