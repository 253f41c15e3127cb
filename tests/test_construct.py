"""GPU H^2 construction: the nested
Chebyshev bases, transfers and interpolation nodes built on the device equal
the numpy generator's (h2gen, the inputs the oracle reads) BIT FOR BIT, and the
matrix-free couplings K(nodes_t, nodes_s) of the build equal the generator's
couplings to rounding (they go through rsqrt / exp on the device)."""
import numpy as np
import pytest

import h2gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _construct(h, side):
    import paper_1705_04601_b200 as h2sp
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed)
    sp = h2sp.Sparsifier(plan, packed, alloc_inputs=False)
    dev = sp.device
    pts = torch.from_numpy(np.ascontiguousarray(h.points)).to(dev)
    lo = torch.from_numpy(np.ascontiguousarray(h.meta["box_lo"])).to(dev)
    hi = torch.from_numpy(np.ascontiguousarray(h.meta["box_hi"])).to(dev)
    d, r = int(h.meta["dim"]), int(h.meta["r"])
    out = h2sp.cheb_construct(plan, sp.ws_ptr, pts, lo, hi, h2gen.cheb_base_orders(d, r),
                              h2gen.cheb_cos_table(1 if side == 0 else 2), side=side)
    torch.cuda.synchronize()
    return packed, out


@pytest.mark.parametrize("cfg,N", [(2, 8192), (3, 8192), (5, 16384), (4, 8192)])
def test_cheb_bases_bitwise(cfg, N):
    _need_gpu()
    h = h2gen.make_config(cfg, N=N, orthonormalize=False)
    for side in ((0,) if h.symmetric else (0, 1)):
        packed, out = _construct(h, side)
        key = "row" if side == 0 else "col"
        nl = packed[f"leaf_{key}"].size
        nt = packed[f"transfer_{key}"].size
        assert np.array_equal(out["leaf"][:nl].cpu().numpy(), packed[f"leaf_{key}"])
        assert np.array_equal(out["transfer"][:nt].cpu().numpy(), packed[f"transfer_{key}"])
        xr, xc, _, _ = h2gen.coupling_block_descs(h)
        ref = xr if side == 0 else xc
        assert np.array_equal(out["nodes"][:len(ref)].cpu().numpy(), ref)


def test_matrix_free_couplings_match_generator():
    """The build's coupling step with D evaluated from the device nodes gives the
    same S as the build reading the generator's stored couplings (<= 1e-13)."""
    _need_gpu()
    import paper_1705_04601_b200 as h2sp
    h = h2gen.make_config(2, N=8192)
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed)
    a = h2sp.Sparsifier(plan, packed)
    va = a.build()["s_val"].clone()
    xr, _, _, _ = h2gen.coupling_block_descs(h)
    b = h2sp.Sparsifier(plan, packed, close_gen={"points": h.points, "kernel": h.meta["kernel"], "nodes_row": xr})
    vb = b.build()["s_val"]
    torch.cuda.synchronize()
    nnz = plan.sizes["s_nnz"]
    err = float(torch.linalg.norm(va[:nnz] - vb[:nnz]) / torch.linalg.norm(va[:nnz]))
    assert err <= 1e-13, err
