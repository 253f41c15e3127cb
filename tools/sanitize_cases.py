"""Small builds for compute-sanitizer (memcheck / racecheck / synccheck, one tool
per gpurun call): BASELINE configs[0], a random B = 128 general case, the
config-5 recipe in bench mode with matrix-free inputs over 4 virtual shards,
and the applies (apply_ut_kernel's arrival counters)."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import h2gen  # noqa: E402
import paper_1705_04601_b200 as h2sp  # noqa: E402


def stored(h):
    packed = h2gen.pack(h)
    plan = h2sp.Plan(packed)
    sp = h2sp.Sparsifier(plan, packed)
    sp.build()
    b = torch.randn(1, plan.n_tree_local, dtype=torch.float64, device="cuda")
    y = torch.empty(1, plan.s_rows, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    sp.apply_Ut(b, y)
    sp.apply_V(y, x)
    aws = sp.apply_workspace(1)
    sp.build_apply(b, y, torch.randn_like(y), x, aws)
    torch.cuda.synchronize()
    print("stored ok", h.N, flush=True)


def bench_shards(h, G):
    packed = h2gen.pack(h)
    plans = [h2sp.Plan(packed, g, G, bench=True) for g in range(G)]
    xr, _, _, _ = h2gen.coupling_block_descs(h)
    vs = h2sp.VirtualShards(plans, packed, close_gen={"points": h.points, "kernel": h.meta["kernel"], "nodes_row": xr})
    vs.outputs["bench_w"].copy_(torch.from_numpy(np.random.default_rng(1).standard_normal(h.N)))
    vs.build()
    torch.cuda.synchronize()
    print("bench shards ok", h.N, G, flush=True)


if __name__ == "__main__":
    stored(h2gen.make_config(1))
    stored(h2gen.random_h2(4, 128, 5, False, eta=0.7, max_rank=32))
    bench_shards(h2gen.make_config(5, N=8192), 4)
