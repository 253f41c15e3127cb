"""Sharded plans, host side: the union of the shards' local S
rows is the full S, each row exactly once, with identical column patterns;
and a world_size-2 gloo run where every rank builds its own shard plan."""
import os

import numpy as np
import pytest

import h2gen
import paper_1705_04601_b200 as h2sp


def _inputs():
    yield "cfg2-4096-sym", lambda: h2gen.make_config(2, N=4096)
    yield "cfg4-8192-gen", lambda: h2gen.make_config(4, N=8192)
    yield "rand-gen-uniform", lambda: h2gen.random_h2(6, 8, 4, False, eta=0.7, ragged=False, r=4)
    yield "rand-sym-uniform", lambda: h2gen.random_h2(6, 8, 5, True, eta=0.7, ragged=False, r=4)


INPUTS = list(_inputs())


def check_union(packed, G):
    full = h2sp.Plan(packed)
    frow, fcol = full.pattern()
    seen = np.zeros(full.N, dtype=np.int64)
    for g in range(G):
        sh = h2sp.Plan(packed, g, G)
        assert sh.sizes["rank"] == g and sh.sizes["world"] == G
        gr = sh.global_rows()
        rp, cl = sh.pattern()
        assert len(gr) == sh.s_rows == len(rp) - 1
        for lr, r in enumerate(gr):
            seen[r] += 1
            assert np.array_equal(cl[rp[lr]:rp[lr + 1]], fcol[frow[r]:frow[r + 1]])
    assert np.all(seen == 1)


@pytest.mark.parametrize("name,make", INPUTS, ids=[i[0] for i in INPUTS])
@pytest.mark.parametrize("G", [2, 4])
def test_shard_union_is_full_pattern(name, make, G):
    check_union(h2gen.pack(make()), G)


def test_shard_flops_add_up_with_cross_pairs():
    """Shards together do at least the full work; symmetric cross pairs are duplicated."""
    p = h2gen.pack(h2gen.make_config(2, N=4096))
    full = h2sp.Plan(p).sizes["flops_congruence"]
    parts = [h2sp.Plan(p, g, 4).sizes["flops_congruence"] for g in range(4)]
    assert sum(parts) >= full
    assert sum(parts) <= 1.5 * full


def test_shard_rejects_bad_world():
    p = h2gen.pack(h2gen.make_config(2, N=4096))
    for rank, world in ((0, 3), (2, 2), (-1, 2)):
        with pytest.raises(h2sp.H2spError):
            h2sp.Plan(p, rank, world)


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    packed = h2gen.pack(h2gen.make_config(2, N=4096))
    sh = h2sp.Plan(packed, rank, world)
    rows = torch.from_numpy(sh.global_rows())
    nnz = torch.tensor([sh.sizes["s_nnz"]], dtype=torch.int64)
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([len(rows)], dtype=torch.int64))
    gathered = [torch.zeros(int(c.item()), dtype=torch.int64) for c in counts]
    dist.all_gather(gathered, rows)
    dist.all_reduce(nnz)
    if rank == 0:
        allrows = torch.cat(gathered).numpy()
        full = h2sp.Plan(packed)
        q.put((sorted(allrows.tolist()) == list(range(full.N)), int(nnz.item()) == full.sizes["s_nnz"]))
    dist.destroy_process_group()


def test_gloo_world2_shards_cover_s():
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.randint(0, 2000)
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in ps)
    rows_ok, nnz_ok = q.get(timeout=5)
    assert rows_ok and nnz_ok


@pytest.mark.parametrize("name,make", INPUTS, ids=[i[0] for i in INPUTS])
@pytest.mark.parametrize("G", [2, 4])
def test_shard_unique_flops_add_up_to_unsharded(name, make, G):
    """flops_unique (work of the shard's own row / rotating clusters) adds up to
    the unsharded plan's algorithmic flops exactly: the job's work for a
    multi-GPU TFLOP/s, without the halo / mirror work done twice."""
    p = h2gen.pack(make())
    full = h2sp.Plan(p).sizes
    assert full["flops_unique"] == full["flops"]
    shards = [h2sp.Plan(p, g, G).sizes for g in range(G)]
    tot = sum(s["flops_unique"] for s in shards)
    assert abs(tot - full["flops"]) <= 1e-9 * full["flops"]
    assert all(s["flops_unique"] <= s["flops"] * (1 + 1e-12) for s in shards)


@pytest.mark.parametrize("name,make", INPUTS, ids=[i[0] for i in INPUTS])
def test_bench_plan_matches_stored_plan(name, make):
    """Bench mode (H2SP_PLAN_BENCH) changes where S goes, not the work: same
    pattern size, blocks and flops; one partial slot per (S row, block); no
    column pattern; the CSR expansion launch replaced by the row-sum launch."""
    p = h2gen.pack(make())
    a, b = h2sp.Plan(p), h2sp.Plan(p, bench=True)
    for k in ("s_nnz", "s_blocks", "s_rows", "q_row", "q_col"):
        assert a.sizes[k] == b.sizes[k], k
    for k in ("flops", "flops_congruence", "flops_strips"):
        assert a.sizes[k] == b.sizes[k], k
    # executed work: bench plans on aligned trees skip the k range of an absent
    # child in the strips (the kernel's loop), so they execute no more
    assert b.sizes["flops_executed"] <= a.sizes["flops_executed"]
    assert a.sizes["bench_parts"] == 0
    # slots: sum over block rows of (rows x blocks) -- every block row's blocks
    # are the column runs of its pattern
    rp, col = a.pattern()
    runs = 0
    for r in range(a.s_rows):
        c = col[rp[r]:rp[r + 1]]
        if len(c):
            runs += 1 + int(np.count_nonzero(np.diff(c) != 1))
    # one slot per (row, block); adjacent blocks of a row may form one column run
    assert runs <= b.sizes["bench_parts"] <= a.sizes["s_nnz"]
    assert b.sizes["bench_parts"] >= a.sizes["s_blocks"]
    kinds_a = [l["kind"] for l in a.launches()]
    kinds_b = [l["kind"] for l in b.launches()]
    assert ("csr" in kinds_a) and ("csr" not in kinds_b) and ("bench_reduce" in kinds_b)
    with pytest.raises(h2sp.H2spError):
        b.pattern(with_cols=True)


def _gloo_protocol_worker(rank, world, port, q):
    """The multi-GPU bench's host logic on gloo: rank g takes virtual shards
    [V g / world, V (g+1) / world) of ONE matrix (bench mode, as bench.py's
    run_protocol), and the job's work is the all-reduced sum of flops_unique."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    V = 4
    packed = h2gen.pack(h2gen.make_structure(5, N=16384))
    mine = list(range(rank * V // world, (rank + 1) * V // world))
    plans = [h2sp.Plan(packed, g, V, bench=True) for g in mine]
    t = torch.tensor([sum(p.sizes["flops_unique"] for p in plans), float(sum(p.s_rows for p in plans))],
                     dtype=torch.float64)
    dist.all_reduce(t)
    shards = torch.zeros(V, dtype=torch.int64)
    for g in mine:
        shards[g] += 1
    dist.all_reduce(shards)
    if rank == 0:
        full = h2sp.Plan(packed, bench=True)
        q.put((abs(float(t[0]) - full.sizes["flops"]) <= 1e-9 * full.sizes["flops"], int(t[1]) == full.N,
               bool((shards == 1).all())))
    dist.destroy_process_group()


def test_gloo_world2_protocol_shard_split():
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31000 + random.randint(0, 2000)
    ps = [ctx.Process(target=_gloo_protocol_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in ps)
    flops_ok, rows_ok, shards_ok = q.get(timeout=5)
    assert flops_ok and rows_ok and shards_ok
