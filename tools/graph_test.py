import sys, time, json, torch
sys.path.insert(0, '.')
import h2gen, paper_1705_04601_b200 as h2sp
h = h2gen.make_config(2)
packed = h2gen.pack(h)
plan = h2sp.Plan(packed)
sp = h2sp.Sparsifier(plan, packed)
b = torch.randn(1, plan.N, dtype=torch.float64, device='cuda'); y = torch.empty_like(b); x = torch.empty_like(b)
aws = sp.apply_ws(1)
def app():
    sp.apply_Ut(b, y, ws=aws); sp.apply_V(y, x, ws=aws)
def step():
    sp.build(); app()
for _ in range(5): step()
torch.cuda.synchronize()
K = 30
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record();
for _ in range(K): step()
e1.record(); torch.cuda.synchronize(); t_plain = e0.elapsed_time(e1) / K
ref = sp.outputs['s_val'].clone()
g = sp.capture(app)
for _ in range(3): g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(K): g.replay()
e1.record(); torch.cuda.synchronize(); t_graph = e0.elapsed_time(e1) / K
print(json.dumps({"plain_ms": t_plain, "graph_ms": t_graph, "same": bool(torch.equal(ref, sp.outputs['s_val']))}))
