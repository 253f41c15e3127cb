"""Algorithm 1 for a dense matrix on the device:
A dense (the generator's kernel matrix) -> bases from SVDs of the far-field
block rows on the device (paper_1705_04601_b200.dense_variant) -> the package's
sparsification -> U S V^T.  Expected value: the numpy generator's config-1 H^2
matrix (the same SVD recompression recipe, h2gen._svd_h2) densified by the
oracle -- the two compressions project onto the same singular subspaces, so
U S V^T must equal it to rounding, whatever signs the two SVDs pick."""
import numpy as np
import pytest

import h2gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dense_usv(h, plan, out, res):
    off = plan.offsets()
    q = out["q_row"].cpu().numpy()
    res.Q_row = [q[off["q_off_row"][c]:off["q_off_row"][c] + int(n) ** 2].reshape(int(n), int(n))
                 for c, n in enumerate(res.n_row)]
    res.Q_col = res.Q_row
    U = oracle.dense_U(res, "row")
    nnz = plan.sizes["s_nnz"]
    rowptr, col = out["s_rowptr"].cpu().numpy(), out["s_col"].cpu().numpy()
    val = out["s_val"][:nnz].cpu().numpy()
    S = np.zeros((h.N, h.N))
    for r in range(h.N):
        S[r, col[rowptr[r]:rowptr[r + 1]]] = val[rowptr[r]:rowptr[r + 1]]
    return U @ S @ U.T


def test_algorithm1_dense_config1():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_04601_b200 as h2sp
    from paper_1705_04601_b200.dense_variant import compress_dense
    h = h2gen.make_config(1)                         # numpy SVD recompression (the expected value)
    A_dense = h2gen.kernel_matrix(h.meta["kernel"], h.points, h.points, np.eye(h.N, dtype=bool))
    At = torch.from_numpy(A_dense).cuda()
    comp = compress_dense(At, h.L, h.B, int(h2gen.CONFIGS[1]["r"]), h.near, h.adm, symmetric=True)
    assert np.array_equal(comp["rank_row"], h.rank_row)
    plan = h2sp.Plan(comp)
    sp = h2sp.Sparsifier(plan, None, inputs=comp["inputs"])
    out = sp.build()
    torch.cuda.synchronize()
    usv = _dense_usv(h, plan, out, oracle.sparsify(h))
    A_h2 = oracle.dense_A(h)
    err = np.linalg.norm(usv - A_h2) / np.linalg.norm(A_h2)
    assert err <= 1e-10, err
    # and the compression is an approximation of A at the generator's level
    assert np.linalg.norm(usv - A_dense) / np.linalg.norm(A_dense) <= 2 * np.linalg.norm(A_h2 - A_dense) / \
        np.linalg.norm(A_dense) + 1e-12
