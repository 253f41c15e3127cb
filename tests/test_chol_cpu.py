"""Host analysis of the supernodal Cholesky (h2sp_chol_analyse, no GPU needed):
struct(J) and the block elimination tree against brute-force symbolic
elimination of S's block pattern (graph elimination on a dense boolean block
matrix: eliminating J connects every pair of its later neighbours)."""
import numpy as np
import pytest

import h2gen
import paper_1705_04601_b200 as h2sp
from paper_1705_04601_b200 import solve as sv


def _brute(plan, starts=None):
    if starts is None:
        starts, _ = sv._groups(plan)
    ns = len(starts)
    rp, col = plan.pattern()
    N = plan.N
    grp = np.searchsorted(starts, np.arange(N), side="right") - 1
    rows = np.repeat(np.arange(N), np.diff(rp))
    Bm = np.zeros((ns, ns), dtype=bool)
    Bm[grp[rows], grp[col]] = True
    Bm = Bm | Bm.T
    structs, parent = [], []
    for J in range(ns):
        below = np.nonzero(Bm[J + 1:, J])[0] + J + 1
        for a in below:
            Bm[a, below] = True
            Bm[below, a] = True
        structs.append(np.concatenate([[J], below]))
        parent.append(below[0] if len(below) else -1)
    return structs, np.array(parent)


CASES = [("cfg1", lambda: h2gen.make_config(1)),
         ("cfg2-4096", lambda: h2gen.make_config(2, N=4096)),
         ("cfg3-4096", lambda: h2gen.make_config(3, N=4096)),
         ("random-sym", lambda: h2gen.random_h2(5, 16, 3, True, eta=0.7)),
         ("eta0", lambda: h2gen.eta0_h2(3, 16, 5, symmetric=True))]


@pytest.mark.parametrize("amalg", [0, 128])
@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_symbolic_matches_graph_elimination(name, make, amalg):
    """amalg = 0: supernodes = S's row groups; 128: relaxed amalgamation -- a
    coarser contiguous partition (merged widths <= 128, each a union of row
    groups) whose structures are again exactly the graph elimination's."""
    plan = h2sp.Plan(h2gen.pack(make()))
    an = sv.CholAnalysis(plan, amalg)
    g0, m0 = sv._groups(plan)
    if amalg == 0:
        assert np.array_equal(an.starts, g0)
    else:
        assert np.all(np.isin(an.starts, g0)) and an.sizes.max() <= max(128, m0.max())
    structs, parent = _brute(plan, an.starts)
    assert an.ns == len(structs)
    assert np.array_equal(an.parent, parent)
    starts, ms = an.starts, an.sizes
    for J in range(an.ns):
        s = an.struct(J)
        assert np.array_equal(s, structs[J]), J
        assert an.panel_rows[J] == ms[s].sum()
    assert an.panel_doubles == sum(int(an.panel_rows[J]) * int(ms[J]) for J in range(an.ns))


def test_rejects_general_and_bench_plans():
    h = h2gen.random_h2(4, 16, 2, False, eta=0.7)
    with pytest.raises(h2sp.H2spError, match="symmetric"):
        sv.CholAnalysis(h2sp.Plan(h2gen.pack(h)))
    h = h2gen.make_config(2, N=4096)
    with pytest.raises(h2sp.H2spError, match="stored-S"):
        sv.CholAnalysis(h2sp.Plan(h2gen.pack(h), bench=True))
