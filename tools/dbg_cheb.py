import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import h2gen, paper_1705_04601_b200 as h2sp
h = h2gen.make_config(2, N=4096)
packed = h2gen.pack(h)
plan = h2sp.Plan(packed)
sp = h2sp.Sparsifier(plan, packed, alloc_inputs=False)
dev = sp.device
pts = torch.from_numpy(np.ascontiguousarray(h.points)).to(dev)
lo = torch.from_numpy(np.ascontiguousarray(h.meta["box_lo"])).to(dev)
hi = torch.from_numpy(np.ascontiguousarray(h.meta["box_hi"])).to(dev)
out = h2sp.cheb_construct(plan, sp.ws_ptr, pts, lo, hi, h2gen.cheb_base_orders(2, 16), h2gen.cheb_cos_table(1), side=0)
torch.cuda.synchronize()
d = out["leaf"][:30].cpu().numpy()
np.set_printoptions(precision=17)
print("x", d[:2], "p", d[2:4], "dim", d[4], "k", d[5])
print("nodes0", d[6:10]); print("nodes1", d[10:14])
print("row", d[14:30])
print("ref row", packed["leaf_row"][:16])
