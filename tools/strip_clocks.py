"""Phase attribution of strip_kernel at the bench's full size (attribution build only:
alt/libh2sp_clk.so, kernels.cu compiled with -DH2SP_STRIP_CLOCKS): thread 0 of every 64th
CTA stamps clock64() at the phase boundaries; this prints the mean / median cycles per phase
of the largest launch (level 1 of virtual shard 0).  Run under gpurun from the repo root.

Build the attribution library first (after __graft_entry__.build(), which leaves the other
objects in build/):
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
         -DH2SP_STRIP_CLOCKS -c paper_1705_04601_b200/csrc/kernels.cu -o build/kernels_clk.o
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o alt/libh2sp_clk.so build/plan.cpp.o \
         build/kernels_clk.o build/api.cu.o build/comm.cpp.o build/krylov.cu.o build/chol.cu.o -lcudart -ldl
The script swaps it in for paper_1705_04601_b200/libh2sp.so: rebuild (or restore) the product
library afterwards."""
import ctypes
import shutil
import sys

import numpy as np

shutil.copy("alt/libh2sp_clk.so", "paper_1705_04601_b200/libh2sp.so")
sys.path.insert(0, ".")
import torch  # noqa: E402

import h2gen  # noqa: E402
import paper_1705_04601_b200 as h2sp  # noqa: E402
from paper_1705_04601_b200.protocol import ProtocolRun  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else None
h = h2gen.make_structure(5, N=N)
run = ProtocolRun(h, V=8, shards=[0], device=torch.device("cuda", 0), nrhs=1, plan_threads=8)
run.outputs["bench_w"].normal_()
fn = h2sp.lib.h2sp_debug_strip_clocks
fn.argtypes = [ctypes.c_void_p, ctypes.c_int64]
fn.restype = ctypes.c_int64
rec = np.dtype([("grid", "<u4"), ("smid", "<u4"), ("gt0", "<u8"), ("c", "<i8", (10,))])
buf = np.zeros(16384, dtype=rec)
run.build(None)
fn(buf.ctypes.data, 16384)      # warm-up pass discarded
run.build(None)
n = fn(buf.ctypes.data, 16384)
r = buf[:n]
g = r["grid"].max()
r = r[r["grid"] == g]
names = ["descriptor round trip + barrier", "Q / groups round trip + barrier", "column maps + barrier",
         "gather of Z (issue, wait, barrier)", "product (warp 0)", "panel-row stores (warp 0)",
         "barrier after the product", "slab partials + barrier", "final sums + part stores"]
d = np.diff(r["c"], axis=1).astype(float)
tot = (r["c"][:, 9] - r["c"][:, 0]).astype(float)
print(f"{len(r)} sampled CTAs of the {g}-tile launch; residency mean {tot.mean():.0f} median {np.median(tot):.0f} cycles "
      f"({tot.mean() / 1.965e3:.2f} us)")
for i in range(9):
    print(f"  {names[i]:36s} mean {d[:, i].mean():8.0f}  median {np.median(d[:, i]):8.0f}  ({100 * d[:, i].mean() / tot.mean():4.1f} %)")
# start-time spread of CTAs on one SM (are resident CTAs phase-locked?): gap between consecutive sampled starts
for sm in (0, 1):
    t = np.sort(r["gt0"][r["smid"] == sm].astype(np.int64))
    if len(t) > 2:
        print(f"  SM {sm}: {len(t)} samples, median gap between sampled starts {np.median(np.diff(t)) / 1e3:.1f} us")
