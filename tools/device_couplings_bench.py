"""GPU evaluation of the interpolation couplings (h2sp_eval_kernel_blocks) vs the
numpy generator's coupling loop, on a BASELINE config recipe.  One JSON line.
usage: python tools/device_couplings_bench.py [config] [N]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import h2gen  # noqa: E402
import paper_1705_04601_b200 as h2sp  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
    t0 = time.perf_counter()
    h0 = h2gen.make_config(cfg, N=N, with_close=False, with_couplings=False)
    t_nocoup = time.perf_counter() - t0
    t0 = time.perf_counter()
    h1 = h2gen.make_config(cfg, N=N, with_close=False, with_couplings=True)
    t_coup = time.perf_counter() - t0
    ref = np.concatenate([m.ravel() for lst in h1.coupling for m in lst])
    xr, xc, desc, n = h2gen.coupling_block_descs(h0)
    xr_t, xc_t = torch.from_numpy(xr).cuda(), torch.from_numpy(xc).cuda()
    d_t = torch.from_numpy(desc).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    h2sp.eval_kernel_blocks(h0.meta["kernel"], xr_t, xc_t, d_t, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record()
    for _ in range(reps):
        h2sp.eval_kernel_blocks(h0.meta["kernel"], xr_t, xc_t, d_t, out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    err = float(np.linalg.norm(out.cpu().numpy() - ref) / np.linalg.norm(ref))
    print(json.dumps({"config": cfg, "N": N, "pairs": int(desc.shape[0]), "coupling_doubles": int(n),
                      "gpu_ms": ms, "gpu_gbs_written": n * 8 / (ms * 1e-3) / 1e9,
                      "host_generator_coupling_s": t_coup - t_nocoup, "host_generator_rest_s": t_nocoup,
                      "rel_err_vs_numpy": err}))


if __name__ == "__main__":
    main()
