"""The SURVEY §8(d) config-5 protocol as library calls (orchestration only; every
numeric step runs in libh2sp's kernels):

1. inputs built on the device -- nested Chebyshev bases, transfers and
   interpolation nodes by ``h2sp_cheb_construct``; close blocks and far
   couplings matrix-free (``h2sp_close_gen`` with nodes), so nothing but the
   points, the cluster boxes and the bases is stored;
2. V virtual shards (top-level subtrees, sharded plans) processed one after
   another on one scratch buffer (``h2sp_build_meta``), the shards' work lists
   resident;
3. S in bench mode (``H2SP_PLAN_BENCH``): y = S w and the row norms reduced in
   the epilogues -- config 5's S (~2 TB) is never stored.

A rank of a multi-GPU job takes a contiguous subset of the V shards.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from typing import List, Optional, Sequence

import numpy as np

from . import Plan, VirtualShards, _check, _stream_handle, cheb_construct, lib

__all__ = ["ProtocolRun"]


class ProtocolRun:
    """``h``: a structure-only input (h2gen.make_structure: tree-ordered points,
    cluster boxes, block tree, ranks, kernel spec; symmetric Chebyshev recipe).
    ``shards``: the virtual shard indices (of ``V``) this process builds."""

    def __init__(self, h, V: int = 8, shards: Optional[Sequence[int]] = None, device="cuda", nrhs: int = 1,
                 plan_threads: int = 8, orders=None, cos_table=None):
        import torch
        import h2gen   # seeded input recipe: layout tables only (cosines, base orders)
        if not h.symmetric:
            raise ValueError("the protocol path covers the symmetric (SPD) recipes")
        self.h = h
        self.V = V
        self.shards = list(range(V)) if shards is None else list(shards)
        self.device = torch.device(device)
        self.nrhs = nrhs
        packed = h2gen.pack(h)
        with ThreadPoolExecutor(max(1, min(len(self.shards), plan_threads))) as ex:   # ctypes releases the GIL
            self.plans: List[Plan] = list(ex.map(lambda g: Plan(packed, g, V, bench=True), self.shards))
        del packed
        d, r = int(h.meta["dim"]), int(h.meta["r"])
        self.orders = orders if orders is not None else h2gen.cheb_base_orders(d, r)
        self.cos = cos_table if cos_table is not None else h2gen.cheb_cos_table(1)
        f64 = dict(dtype=torch.float64, device=self.device)
        self.points = torch.from_numpy(np.ascontiguousarray(h.points)).to(**f64)
        self.box_lo = torch.from_numpy(np.ascontiguousarray(h.meta["box_lo"])).to(**f64)
        self.box_hi = torch.from_numpy(np.ascontiguousarray(h.meta["box_hi"])).to(**f64)
        p0 = self.plans[0]
        # the per-cluster arrays every shard plan shares (ranks, basis offsets) on the device
        self._meta0 = torch.empty(int(p0.sizes["meta_bytes"]) + 256, dtype=torch.uint8, device=self.device)
        self._meta0_ptr = (self._meta0.data_ptr() + 255) // 256 * 256
        _check(lib.h2sp_plan_upload(p0.handle, self._meta0_ptr, int(p0.sizes["meta_bytes"]), _stream_handle(None)),
               "h2sp_plan_upload")
        built = self.construct()
        inputs = {"leaf_basis_row": built["leaf"], "transfer_row": built["transfer"]}
        gen = {"points": self.points, "kernel": h.meta["kernel"], "nodes_row": built["nodes"]}
        self.vs = VirtualShards(self.plans, None, device=self.device, close_gen=gen, inputs=inputs, nrhs=nrhs)
        self.outputs = self.vs.outputs
        self.inputs = self.vs.inputs
        self.N = p0.N
        self.B = p0.B

    def construct(self):
        """Nested bases / transfers / nodes of the row side on the device."""
        return cheb_construct(self.plans[0], self._meta0_ptr, self.points, self.box_lo, self.box_hi, self.orders,
                              self.cos, side=0)

    def reconstruct(self):
        """Rebuild the device inputs in place from the (device) points and boxes."""
        b = self.construct()
        self.inputs["leaf_basis_row"].copy_(b["leaf"])
        self.inputs["transfer_row"].copy_(b["transfer"])
        self.inputs["nodes_row"].copy_(b["nodes"])

    def leaf_range(self, i: int):
        p = self.plans[i]
        fl, nl = int(p.sizes["first_leaf"]), int(p.sizes["n_leaves_local"])
        return fl * self.B, (fl + nl) * self.B

    def build(self, applies=None, events=None, stream=None, after_first=None):
        return self.vs.build(applies, events=events, stream=stream, after_first=after_first)

    def global_rows(self, i: int) -> np.ndarray:
        if not hasattr(self, "_grows"):
            self._grows = {}
        if i not in self._grows:
            self._grows[i] = self.plans[i].global_rows()
        return self._grows[i]
