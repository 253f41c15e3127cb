#!/usr/bin/env python
"""Benchmark of the B200-native H^2 sparsification hot path (arXiv 1705.04601).

One *step* = one pass of the whole hot path of SURVEY.md §8(a) over one
synthetic H^2 matrix: h2sp_build (QR completion, couplings, merge + congruence +
freeze, strips, CSR or the bench-mode S reduction) and the applies y = U^T b,
x = V w (h2sp_apply_Ut / h2sp_apply_V) of the same pass.  The symbolic plan
(row a1, host, structure only) is created once per matrix and reported apart.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config 1..5]

Default workload: BASELINE.json configs[4] at its full size (N = 4,194,304 points
in the unit cube, exp(-|x-y|/0.05) + 1e-2 I, B = 128, r = 32, eta = 0.7, SPD ->
symmetric mode), the configuration the metric is quoted on, by the SURVEY §8(d)
config-5 protocol (inputs built on the device, 8 virtual subtree shards on one
scratch buffer, bench-mode S; run_protocol below).  With N > 1 GPUs (torchrun,
one rank per GPU) the 8 shards of the SAME matrix are split over the ranks
(strong scaling, no data-path collective; the checks go through an NCCL
all_reduce); time = max over ranks.  ``--config 1..4`` run the stored-S path on
one matrix per rank (or ``--shard``: one matrix split in N subtree shards).

``--impl reference`` times the CPU oracle (oracle/, numpy, 1 thread) on a
bounded sample of the workload; only rank 0 works.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H2 sparsification time & FP64 TFLOP/s (frac. of peak) at 1/2/4/8 B200 vs CPU oracle"
UNIT = "TFLOP/s"
# FP64 peaks measured on this pool's B200 (profiles/r01_fp64_peak.txt): DMMA m8n8k4
# microbenchmark 37.0 TFLOP/s (the ceiling used as roofline peak), cuBLAS DGEMM 35.5.
FP64_PEAK_TFLOPS = 37.0
FP64_DGEMM_TFLOPS = 35.5


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "fallback": True}


def workload_desc(cfg_idx: int, N: int, seed) -> str:
    import h2gen
    c = h2gen.CONFIGS[cfg_idx]
    k = c["kernel"]
    kern = {"exp": f"exp(-r/{k.get('ell')})+{k.get('nugget')}*I", "invh": "1/(r+h)+1.0*I (h=N^-1/3)",
            "laplace": "1/(4 pi r), diag 1/(4 pi h)"}[k["kind"]]
    return (f"BASELINE configs[{cfg_idx - 1}]: N={N} {c['points']} points, {kern}, B={c['B']}, r={c['r']}, "
            f"eta={c['eta']}, {'symmetric (SPD)' if c['symmetric'] else 'general'} mode, seed={seed}")


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, dev_index: int, period_s: float = 0.001):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    _NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
              0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
              0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._NAMES.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": [],
                    "note": getattr(self, "err", "no samples")}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def oracle_baseline(h, flops: float, sample: str):
    """The oracle as it stands, single thread, on host cores."""
    import oracle
    try:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(1)
        cores = 1
    except Exception:  # noqa: BLE001
        import contextlib
        ctx = contextlib.nullcontext()
        cores = os.cpu_count()
    with ctx:
        t0 = time.perf_counter()
        res = oracle.sparsify(h)
        oracle.s_csr(res)
        dt = time.perf_counter() - t0
    out = {"value": flops / dt / 1e12, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
           "seconds": dt, "host_cpus": os.cpu_count()}
    # also on all host cores (numpy's BLAS threads unrestricted; the
    # oracle's small per-block products gain little from them)
    t0 = time.perf_counter()
    oracle.s_csr(oracle.sparsify(h))
    dt_all = time.perf_counter() - t0
    out["all_cores"] = {"value": flops / dt_all / 1e12, "cores": os.cpu_count(), "seconds": dt_all}
    return out


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on a bounded sample of the workload."""
    if rank != 0:
        return
    import h2gen
    import oracle
    n_sample = args.ref_n
    h = h2gen.make_config(args.config, N=n_sample)
    # algorithmic flops of the sample, counted from the oracle's own structure
    res0 = oracle.sparsify(h)
    flops = _oracle_flops(res0, h)
    sample = (f"configs[{args.config - 1}] recipe at N={n_sample} (L={h.L}), one full oracle pass "
              f"(sparsify + CSR assembly) per step")
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except Exception:  # noqa: BLE001
        lim = None
    for _ in range(args.warmup):
        oracle.s_csr(oracle.sparsify(h))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.s_csr(oracle.sparsify(h))
    dt = (time.perf_counter() - t0) / args.steps
    del lim
    val = flops / dt / 1e12
    line = {"metric": METRIC, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(args.config, args.n or h2gen.CONFIGS[args.config]["N"], args.config),
                       "sample": sample, "sample_N": n_sample, "flops_per_step": flops},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _oracle_flops(res, h):
    """Algorithmic flops of one build, counted on the oracle's structure with the
    plan's per-unit figures: QR 2nk^2 + 4n^2k, couplings
    2 k_t k_s (k_t + k_s), congruence 2 n_t n_s (n_t + n_s), strip rotation
    2 n_p (sum of present children ranks) m.  Independent of libh2sp."""
    from h2gen import cid
    L = h.L
    f = 0.0
    sides = [(res.n_row, res.k_row)] + ([] if h.symmetric else [(res.n_col, res.k_col)])
    for n, k in sides:
        f += float(sum(2.0 * n[c] * k[c] ** 2 + 4.0 * n[c] ** 2 * k[c] for c in range(len(n))))
    for lvl in range(L):
        for (t, s) in h.adm[lvl]:
            if h.symmetric and t > s:
                continue
            a, b = float(res.k_row[cid(L, lvl, t)]), float(res.k_col[cid(L, lvl, s)])
            f += 2.0 * a * b * (a + b)
    for lvl, near in enumerate(res.near_levels):
        for (t, s) in near:
            if h.symmetric and t > s:
                continue
            a, b = float(res.n_row[cid(L, lvl, t)]), float(res.n_col[cid(L, lvl, s)])
            f += 2.0 * a * b * (a + b)

    def strips(n_rot, k_rot, m_fix, transpose):
        groups = {}
        for j, near in enumerate(res.near_levels):
            for pair in near:
                t0, s0 = (pair[1], pair[0]) if transpose else pair
                if m_fix[cid(L, j, s0)] == 0:
                    continue
                t, lvl = t0, j
                while lvl < L and k_rot[cid(L, lvl, t)] > 0:
                    groups.setdefault((lvl + 1, t // 2, j, s0), set()).add(t % 2)
                    t, lvl = t // 2, lvl + 1
        tot = 0.0
        for (lvl, p, j, s0), kids in groups.items():
            rows = sum(float(k_rot[cid(L, lvl - 1, 2 * p + a)]) for a in kids)
            tot += 2.0 * float(n_rot[cid(L, lvl, p)]) * rows * float(m_fix[cid(L, j, s0)])
        return tot

    f += strips(res.n_row, res.k_row, res.m_col, False)
    if not h.symmetric:
        f += strips(res.n_col, res.k_col, res.m_row, True)
    return f


def _env_knobs():
    """Every H2SP_* environment variable in effect (scheduling experiments only;
    the work-skipping switches exist only in -DH2SP_TIMING_KNOBS builds)."""
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("H2SP_")}


def _cpu_sample_baseline(cfg_idx: int, n_sample: int, full_flops: float):
    """The oracle as it stands, 1 thread, on a bounded sample of the recipe;
    its rate (algorithmic TFLOP/s) is the baseline, extrapolated to the full
    workload by the flop count (labelled as such)."""
    import h2gen
    import oracle
    h = h2gen.make_config(cfg_idx, N=n_sample)
    res0 = oracle.sparsify(h)
    flops = _oracle_flops(res0, h)
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except Exception:  # noqa: BLE001
        lim = None
    t0 = time.perf_counter()
    oracle.s_csr(oracle.sparsify(h))
    dt = time.perf_counter() - t0
    del lim
    rate = flops / dt
    return {"value": rate / 1e12, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": (f"configs[{cfg_idx - 1}] recipe at N={n_sample} (L={h.L}): one full oracle pass (sparsify + "
                       f"CSR assembly), {flops:.3g} algorithmic flops in {dt:.1f} s on 1 host thread; the full "
                       f"workload ({full_flops:.3g} flops) extrapolates to {full_flops / rate / 3600:.1f} h"),
            "extrapolated": True, "seconds": dt, "sample_flops": flops, "host_cpus": os.cpu_count()}


def run_protocol(args, rank, world, local_rank):
    """BASELINE configs[4] at full size (N = 4,194,304) by the SURVEY §8(d)
    config-5 protocol (paper_1705_04601_b200.protocol): inputs built on the
    device (Chebyshev bases / transfers / nodes, h2sp_cheb_construct; close
    blocks and couplings matrix-free), S in bench mode (S w and row norms
    reduced in the epilogues), 8 virtual shards (top-level subtrees) one after
    another on one scratch buffer (h2sp_build_meta).  With N GPUs rank g takes
    shards [8g/N, 8(g+1)/N) of the SAME matrix (strong scaling, no data-path
    collective: halo Q / R^ recomputed per shard; the checks go through an
    NCCL all_reduce); time = max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import h2gen
    from paper_1705_04601_b200.protocol import ProtocolRun

    # H2SP_BENCH_SHARED_GPU=1 (plumbing test only): ranks share the visible GPUs
    # round robin, reduce over gloo, and skip libh2sp's NCCL communicator (NCCL
    # refuses two ranks on one device); every rank still times its own shards
    shared = os.environ.get("H2SP_BENCH_SHARED_GPU") == "1"
    dev_idx = local_rank % torch.cuda.device_count() if shared else local_rank
    torch.cuda.set_device(dev_idx)
    dev = torch.device("cuda", dev_idx)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if shared else dev

    def allreduce(t, op=None):
        if world == 1:
            return t
        x = t.to(red_dev)
        if op is None:
            dist.all_reduce(x)
        else:
            dist.all_reduce(x, op=op)
        t.copy_(x.to(t.device))
        return t

    V = args.virtual_shards
    if V % world:
        raise SystemExit(f"--virtual-shards {V} must be a multiple of the GPU count {world}")
    mine = list(range(rank * V // world, (rank + 1) * V // world))
    t0 = time.perf_counter()
    h = h2gen.make_structure(args.config, N=args.n)
    struct_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    run = ProtocolRun(h, V=V, shards=mine, device=dev, nrhs=args.nrhs, plan_threads=args.plan_threads)
    setup_s = time.perf_counter() - t0
    plans = run.plans
    N, B, nrhs = run.N, run.B, args.nrhs
    f64 = dict(dtype=torch.float64, device=dev)
    gw = torch.Generator(device="cpu").manual_seed(args.config)
    w_host = torch.randn(N, generator=gw, dtype=torch.float64)
    b_host = torch.randn(nrhs, N, generator=gw, dtype=torch.float64)
    run.outputs["bench_w"].copy_(w_host)
    b_full = b_host.to(dev)
    x_full = torch.empty(nrhs, N, **f64)
    applies = []
    for i, p in enumerate(plans):
        a0, a1 = run.leaf_range(i)
        applies.append((b_full[:, a0:a1].contiguous(), torch.empty(nrhs, p.s_rows, **f64),
                        torch.randn(nrhs, p.s_rows, **f64), torch.empty(nrhs, a1 - a0, **f64)))
    launches = [p.launches() for p in plans]
    n_launch = [len(l) for l in launches]
    stream = torch.cuda.current_stream()

    def step(events=None):
        run.build(applies, events=events)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(2 * n)] for n in n_launch] for _ in range(args.steps)]
    for st_ in evs:
        for row in st_:
            for e in row:
                e.record(stream)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev_idx) as clk:
        t_start.record(stream)
        for i in range(args.steps):
            step(evs[i])
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end) / args.steps
    red = torch.tensor([ms], **f64)
    allreduce(red, dist.ReduceOp.MAX)
    ms_max = float(red.item())
    # per-launch durations (per shard, averaged over the timed steps)
    per = [np.zeros(n) for n in n_launch]
    for i in range(args.steps):
        for s_, n in enumerate(n_launch):
            for j in range(n):
                per[s_][j] += evs[i][s_][2 * j].elapsed_time(evs[i][s_][2 * j + 1]) / args.steps
    # the checks (||S||_F^2, ||S w||^2 of this rank's rows) through libh2sp's NCCL
    # communicator (bootstrapped from the torch process group; world 1 included,
    # so the single-GPU run exercises the same path)
    import paper_1705_04601_b200 as h2sp
    nccl_info = None
    chk = torch.stack([run.outputs["bench_r2"].sum(), (run.outputs["bench_y"] ** 2).sum()]).contiguous()
    if shared and world > 1:
        allreduce(chk)
        nccl_info = {"comm_ok": False, "note": "H2SP_BENCH_SHARED_GPU plumbing run: checks over gloo"}
    else:
        try:
            comm = h2sp.torch_comm(rank, world)
            comm.allreduce(chk)
            torch.cuda.synchronize()
            nccl_info = {"comm_nranks": world, "comm_ok": True}
        except h2sp.H2spError as exc:
            # the checks are not on the timed path: fall back to the torch process group's
            # all_reduce and say so rather than lose the run
            nccl_info = {"comm_ok": False, "error": str(exc)[:200]}
            if world > 1:
                allreduce(chk)
                nccl_info["fallback"] = "torch.distributed all_reduce (NCCL process group)"
    offs = plans[0].offsets()
    loc_any = np.zeros(int(plans[0].sizes["n_clusters"]), dtype=bool)
    for p in plans:
        loc_any |= p.local_rows()[0] >= 0
    apply_flops = 2 * 2.0 * nrhs * float(np.sum(offs["n_row"][loc_any].astype(float) ** 2))
    tot = torch.tensor([sum(p.sizes["flops_unique"] for p in plans) + apply_flops,
                        sum(p.sizes["flops"] for p in plans) + apply_flops,
                        sum(p.sizes["flops_executed"] for p in plans) + apply_flops,
                        float(sum(p.sizes["s_nnz"] for p in plans))], **f64)
    allreduce(tot)
    job_flops, job_done, job_exec, s_nnz = (float(v) for v in tot.cpu())
    value = job_flops / (ms_max * 1e-3) / 1e12
    # dominant kernel: the level-0 congruence (pair_wy128_kernel), over this rank's shards
    top_fl = top_ex = top_ms = 0.0
    kinds, per_level = {}, {}
    for s_, lst in enumerate(launches):
        for j, li in enumerate(lst):
            kinds[li["kind"]] = kinds.get(li["kind"], 0.0) + per[s_][j]
            key = f"{li['kind']}@{li['level']}"
            d = per_level.setdefault(key, [0.0, 0.0])
            d[0] += per[s_][j]
            d[1] += li["flops_exec"]
            if li["kind"] == "congruence" and li["level"] == 0:
                top_fl += li["flops"]
                top_ex += li["flops_exec"]
                top_ms += per[s_][j]
    roof = {"bound": "tensor", "achieved": top_fl / (top_ms * 1e-3) / 1e12, "peak": FP64_PEAK_TFLOPS,
            "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = _ncu_traffic_protocol()
    roof.update({"kernel": "congruence@level0 (pair_wy128_kernel<32>, compact-WY, close_gen, bench epilogue)",
                 "launch_ms_summed_over_shards": top_ms, "share_of_step": top_ms / ms,
                 "algorithmic_flops": top_fl, "executed_flops": top_ex,
                 "executed_frac": top_ex / (top_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                 "peak_source": "FP64 DMMA microbenchmark on this pool's B200 (profiles/r01_fp64_peak.txt); "
                                f"cuBLAS DGEMM measured {FP64_DGEMM_TFLOPS}"})
    # ---- e2e: the public API with HOST buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        h_pts = torch.from_numpy(np.ascontiguousarray(h.points)).pin_memory()
        h_lo = torch.from_numpy(np.ascontiguousarray(h.meta["box_lo"])).pin_memory()
        h_hi = torch.from_numpy(np.ascontiguousarray(h.meta["box_hi"])).pin_memory()
        h_w = w_host.pin_memory()
        h_b = b_host.pin_memory()
        h_y = torch.empty(N, dtype=torch.float64).pin_memory()
        h_r2 = torch.empty(N, dtype=torch.float64).pin_memory()
        h_q = torch.empty(run.outputs["q_row"].numel(), dtype=torch.float64).pin_memory()
        h_x = torch.empty(nrhs, N, dtype=torch.float64).pin_memory()

        # Q (5.4 GB, the largest result) is final once the first shard's build -- the shared QR pass --
        # is done (the later shards only read it): its D2H runs on a side stream beside them
        q_stream = torch.cuda.Stream(device=dev)
        q_ready, q_done = torch.cuda.Event(), torch.cuda.Event()
        share_qr = run.vs.share_qr or len(plans) == 1

        def q_readback():
            q_ready.record(stream)
            q_stream.wait_event(q_ready)
            with torch.cuda.stream(q_stream):
                h_q.copy_(run.outputs["q_row"], non_blocking=True)
                q_done.record(q_stream)

        def step_e2e():
            run.points.copy_(h_pts, non_blocking=True)
            run.box_lo.copy_(h_lo, non_blocking=True)
            run.box_hi.copy_(h_hi, non_blocking=True)
            run.outputs["bench_w"].copy_(h_w, non_blocking=True)
            b_full.copy_(h_b, non_blocking=True)
            for i, ap_ in enumerate(applies):
                a0, a1 = run.leaf_range(i)
                ap_[0].copy_(b_full[:, a0:a1])
            run.reconstruct()
            run.build(applies, after_first=q_readback if share_qr else None)
            for i, ap_ in enumerate(applies):
                a0, a1 = run.leaf_range(i)
                x_full[:, a0:a1].copy_(ap_[3])
            h_y.copy_(run.outputs["bench_y"], non_blocking=True)
            h_r2.copy_(run.outputs["bench_r2"], non_blocking=True)
            if share_qr:
                stream.wait_event(q_done)   # the step ends when Q has arrived too
            else:
                h_q.copy_(run.outputs["q_row"], non_blocking=True)
            h_x.copy_(x_full, non_blocking=True)

        step_e2e()
        torch.cuda.synchronize()
        k_e2e = max(2, min(args.steps, 3))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(k_e2e):
            step_e2e()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = torch.tensor([e0.elapsed_time(e1) / k_e2e], **f64)
        allreduce(ems, dist.ReduceOp.MAX)
        h2d = sum(t.numel() * 8 for t in (h_pts, h_lo, h_hi, h_w, h_b))
        d2h = sum(t.numel() * 8 for t in (h_y, h_r2, h_q, h_x))
        e2e = {"value": job_flops / (float(ems.item()) * 1e-3) / 1e12, "unit": UNIT,
               "ms_per_step": float(ems.item()), "steps": k_e2e, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h,
               "api": "pinned host points / boxes / w / b in; h2sp_cheb_construct (bases, transfers, nodes on the "
                      "device), h2sp_build_meta per virtual shard (+ U^T b, V w), y = S w, row norms, Q and x out "
                      "(Q read back on a side stream from the end of the shared QR pass on)"}
    # ---- SURVEY 8(a) a8 alone: y = U^T b and x = V y of one shard (its Q from the
    #      last step), nrhs = 1, 8, 32, against the HBM roofline (every Q_t of the
    #      shard's subtree read once + the vectors)
    apply_info = None
    if rank == 0 and not args.no_apply:
        import paper_1705_04601_b200 as h2sp_
        p0 = plans[0]
        loc0, _ = p0.local_rows()
        qbytes = 8.0 * float(np.sum(offs["n_row"][loc0 >= 0].astype(float) ** 2))
        apply_info = {"shard": 0, "q_bytes": qbytes, "hbm_peak_gbs": _peaks()["hbm_gbs"], "by_nrhs": {}}
        for nr in (1, 8, 32):
            need = int(h2sp_.lib.h2sp_apply_ws_bytes(p0.handle, nr))
            aws = torch.empty(need + 256, dtype=torch.uint8, device=dev)
            aptr = (aws.data_ptr() + 255) // 256 * 256
            h2sp_._check(h2sp_.lib.h2sp_plan_upload(p0.handle, aptr, need, h2sp_._stream_handle(None)), "upload")
            a0, a1 = run.leaf_range(0)
            bb = torch.randn(nr, a1 - a0, **f64)
            yy = torch.empty(nr, p0.s_rows, **f64)
            xx = torch.empty_like(bb)
            q = run.outputs["q_row"]

            def ut():
                h2sp_._check(h2sp_.lib.h2sp_apply_Ut(p0.handle, q.data_ptr(), bb.data_ptr(), bb.shape[-1], yy.data_ptr(),
                                                     yy.shape[-1], nr, aptr, need, h2sp_._stream_handle(None)), "Ut")

            def vv():
                h2sp_._check(h2sp_.lib.h2sp_apply_V(p0.handle, q.data_ptr(), yy.data_ptr(), yy.shape[-1], xx.data_ptr(),
                                                    xx.shape[-1], nr, aptr, need, h2sp_._stream_handle(None)), "V")
            res = {}
            for name, fn in (("ut", ut), ("v", vv)):
                fn()
                e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e_a.record(stream)
                for _ in range(5):
                    fn()
                e_b.record(stream)
                torch.cuda.synchronize()
                ms_ = e_a.elapsed_time(e_b) / 5
                byt = qbytes + 8.0 * nr * ((a1 - a0) + p0.s_rows)
                res[name] = {"us": ms_ * 1e3, "gbs": byt / (ms_ * 1e-3) / 1e9,
                             "frac": byt / (ms_ * 1e-3) / 1e9 / apply_info["hbm_peak_gbs"]}
            apply_info["by_nrhs"][nr] = res
            del aws
    cpu = None
    if rank == 0 and world == 1 and not args.no_oracle:
        cpu = _cpu_sample_baseline(args.config, args.ref_n, job_flops)
    if rank == 0:
        cfgd = h2gen.CONFIGS[args.config]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(args.config, N, h.meta.get("seed")), "N": N, "B": B, "L": h.L,
                       "nrhs": nrhs, "mode": "symmetric" if cfgd["symmetric"] else "general",
                       "protocol": (f"SURVEY 8(d) config-5 protocol: inputs built on the device "
                                    f"(h2sp_cheb_construct; close blocks and couplings matrix-free), S in bench mode "
                                    f"(y = S w and row norms reduced in the epilogues; {s_nnz:.3g} nonzeros = "
                                    f"{s_nnz * 12e-12:.2f} TB of CSR never stored), {V} virtual shards one after "
                                    f"another on one scratch buffer"),
                       "parallelism": (f"{V} virtual subtree shards of one matrix over {world} GPU(s) "
                                       f"({len(mine)} per GPU; no data-path collective: halo Q / R^ recomputed per "
                                       f"shard; NCCL all_reduce of the checks)"),
                       "l2": "inputs (bases 1 GB) and the per-shard intermediates (~100 GB) exceed the 126 MB L2; "
                             "no flush",
                       "structure_s": struct_s, "setup_s": setup_s, "s_nnz": s_nnz,
                       "flops_per_step": job_flops, "flops_done_per_step": job_done,
                       "flops_redundant_frac": job_done / job_flops - 1.0,
                       "executed_flops_per_step": job_exec,
                       "flops_convention": "algorithmic (SURVEY 8(d): explicit-Q congruence 2 n_t n_s (n_t + n_s)), "
                                           "each pair / strip counted once (flops_unique of the shards)",
                       "fp64_frac_of_peak_whole_step": value / world / FP64_PEAK_TFLOPS,
                       "breakdown_ms_summed": {k: round(v, 3) for k, v in kinds.items()},
                       "per_kind_level": {k: {"ms": round(v[0], 3), "tflops_exec": round(v[1] / max(v[0], 1e-9) * 1e-9, 2)}
                                          for k, v in per_level.items()},
                       "checks": {"S_frob2": float(chk[0]), "y_norm2": float(chk[1]),
                                  "collective": ("torch gloo all_reduce (shared-GPU plumbing run)" if shared and world > 1 else "h2sp_comm_allreduce (NCCL) over all ranks")},
                       "nccl": nccl_info,
                       "env": _env_knobs()},
            "roofline": roof,
            "apply_roofline": apply_info,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * sum(n + 2 for n in n_launch),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _ncu_traffic_protocol():
    """dram bytes of one level-0 congruence launch of the protocol run, from the
    committed ncu summary (profiles/*_ncu_top_c5.json), per algorithmic flop
    scaled to... (None when absent)."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_top_c5.json")), reverse=True):
        try:
            with open(p) as f:
                return json.load(f).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            continue
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default 5 for config 5, else 20)")
    ap.add_argument("--warmup", type=int, default=None, help="untimed steps (default 3 for config 5, else 5)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5,
                    help="BASELINE configs[config-1]; 5 (default, the metric's workload) runs the SURVEY 8(d) "
                         "protocol at full size, 1-4 the stored-S path")
    ap.add_argument("--virtual-shards", type=int, default=8, help="config 5: virtual subtree shards of the matrix")
    ap.add_argument("--plan-threads", type=int, default=8, help="config 5: shard plans created in parallel")
    ap.add_argument("--n", "--points", dest="n", type=int, default=None, help="override N (smaller instance of the recipe; --points under torchrun, which claims --n)")
    ap.add_argument("--nrhs", type=int, default=1)
    ap.add_argument("--no-oracle", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-apply", action="store_true", help="skip the standalone apply timing (config 5)")
    ap.add_argument("--graph", action="store_true",
                    help="time CUDA-graph replays of the captured step (launch-bound small configs); the default "
                         "eager steps carry the per-launch events the roofline needs inside the timed region")
    ap.add_argument("--e2e-depth", type=int, default=2,
                    help="e2e leg: jobs in flight (own stream + device buffers each); 1 = strictly one after another")
    ap.add_argument("--ref-n", type=int, default=16384, help="--impl reference sample size")
    ap.add_argument("--timeline", action="store_true", help="print per-launch start/end of the last step (stderr)")
    ap.add_argument("--close-gen", action="store_true",
                    help="matrix-free close blocks (h2sp_close_gen): the level-0 congruence evaluates C_ts from "
                         "the points instead of reading them (SURVEY 8(d) config-5 protocol step 1)")
    ap.add_argument("--stored", action="store_true", help="config 5: the stored-S path (needs a small --n)")
    ap.add_argument("--shard", action="store_true",
                    help="N>1: split ONE matrix into N top-level subtree shards (strong scaling) "
                         "instead of N independent matrices (weak scaling, default)")
    ap.add_argument("--workload", choices=["h2sp", "precond"], default="h2sp",
                    help="precond: the paper's GMRES + sparsified-H2 ILUt experiment (bench_precond.py, SURVEY 8(f) #3)")
    ap.add_argument("--d", type=float, default=1e-3, help="precond: Example mat1 parameter d")
    ap.add_argument("--tau", type=float, default=2e-2, help="precond: ILUt drop tolerance")
    args = ap.parse_args()
    if args.workload == "precond":
        import bench_precond
        args.steps = args.steps or 3
        args.warmup = max(args.warmup or 3, 3)
        bench_precond.run(args, ClockSampler, _peaks())
        return
    if args.steps is None:
        args.steps = 5 if args.config == 5 else 20
    if args.warmup is None:
        args.warmup = 3 if args.config == 5 else 5
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.config == 5 and not args.stored:
        run_protocol(args, rank, world, local_rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    import h2gen
    import paper_1705_04601_b200 as h2sp

    # H2SP_BENCH_SHARED_GPU=1 (plumbing test only): ranks share the visible GPUs
    # round robin and reduce the timings over gloo (every rank still times its own
    # independent build; no rank's kernels wait on another's)
    shared = os.environ.get("H2SP_BENCH_SHARED_GPU") == "1"
    dev_idx = local_rank % torch.cuda.device_count() if shared else local_rank
    torch.cuda.set_device(dev_idx)
    dev = torch.device("cuda", dev_idx)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if shared else dev

    shard = args.shard and world > 1
    seed = args.config + (0 if shard else 1000 * rank)
    h = h2gen.make_config(args.config, seed=seed, N=args.n, with_close=not args.close_gen)
    packed = h2gen.pack(h)
    t0 = time.perf_counter()
    plan = h2sp.Plan(packed, rank, world) if shard else h2sp.Plan(packed)
    plan_ms = (time.perf_counter() - t0) * 1e3
    gen = {"points": h.points, "kernel": h.meta["kernel"]} if args.close_gen else None
    sp = h2sp.Sparsifier(plan, packed, device=dev, close_gen=gen)
    launches = plan.launches()
    close_bytes = 0.0
    if args.close_gen:   # C_ts is evaluated, not read: drop its 8 B^2 per level-0 pair from the byte counts
        for li0 in launches:
            if li0["kind"] == "congruence" and li0["level"] == 0:
                li0["bytes"] -= li0["items"] * 8.0 * plan.B * plan.B
                close_bytes += li0["items"] * 8.0 * plan.B * plan.B
    bytes_step = plan.sizes["bytes"] - close_bytes
    n_launch = len(launches)
    assert n_launch == plan.sizes["launches"]
    nrhs = args.nrhs
    b = torch.randn(nrhs, plan.n_tree_local, dtype=torch.float64, device=dev)
    y = torch.empty(nrhs, plan.s_rows, dtype=torch.float64, device=dev)
    x = torch.empty_like(b)
    wv = torch.randn(nrhs, plan.s_rows, dtype=torch.float64, device=dev)  # the V w input (S order)
    aws = sp.apply_ws(nrhs)
    apply_ws_sep = sp.apply_workspace(nrhs)   # h2sp_build_apply runs the applies concurrently with the build
    offs = plan.offsets()
    n_apply_launch = 2   # one fused kernel per direction (apply_ut_kernel, apply_v_kernel)
    loc_r, _ = plan.local_rows()
    apply_flops = 2 * 2.0 * nrhs * float(np.sum(offs["n_row"][loc_r >= 0].astype(float) ** 2))
    # a shard's share of the job's work: each pair / strip / QR once over the shards (flops_unique;
    # plan.sizes["flops"] also counts the Q / R^ and cross pairs a shard recomputes)
    step_flops = float(plan.sizes.get("flops_unique", plan.sizes["flops"])) + apply_flops
    stream = torch.cuda.current_stream()

    def step(events=None):
        # one pass of the hot path: build + y = U^T b + x = V w (h2sp_build_apply;
        # w an independent seeded S-order vector, so the two applies run side by side)
        sp.build_apply(b, y, wv, x, apply_ws_sep, events=events)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # per-launch events for the roofline of the dominant kernel (same stream)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * n_launch)] for _ in range(args.steps)]
    for row in evs:            # torch creates the CUDA event lazily on first record
        for e in row:
            e.record(stream)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    graph = None
    if args.graph:
        # the whole step (build + applies, fork/join over the library's side
        # streams) captured once into a CUDA graph and replayed; per-launch
        # durations then come from an untimed eager pass below
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(stream)
        with torch.cuda.graph(graph, stream=cap):
            step()
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        t_start.record(stream)
        for i in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                step(evs[i])
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end) / args.steps
    if graph is not None:     # per-launch events: eager steps outside the timed region
        for i in range(args.steps):
            step(evs[i])
        torch.cuda.synchronize()
    ms_t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    # per-launch durations averaged over the timed steps
    per = np.zeros(n_launch)
    for i in range(args.steps):
        for j in range(n_launch):
            per[j] += evs[i][2 * j].elapsed_time(evs[i][2 * j + 1])
    per /= args.steps
    if args.timeline:
        ev = evs[-1]
        base_ev = ev[0]
        for j, li in enumerate(launches):
            st_ms = base_ev.elapsed_time(ev[2 * j])
            en_ms = base_ev.elapsed_time(ev[2 * j + 1])
            print(f"timeline {li['kind']:>11s} L{li['level']:<2d} start {st_ms * 1e3:8.1f} us  end {en_ms * 1e3:8.1f} us "
                  f"dur {(en_ms - st_ms) * 1e3:7.1f} us", file=sys.stderr)
    kinds = {}
    for j, li in enumerate(launches):
        kinds[li["kind"]] = kinds.get(li["kind"], 0.0) + per[j]
    # dominant kernel = the launch with the most algorithmic work (the level-0
    # congruence); durations of concurrent launches are not comparable
    top = int(np.argmax([l["flops"] for l in launches]))
    li = launches[top]
    peaks = _peaks()
    ai = li["flops"] / li["bytes"] if li["bytes"] else float("inf")
    ridge = FP64_PEAK_TFLOPS * 1e12 / (peaks["hbm_gbs"] * 1e9)
    if ai >= ridge:
        roof = {"bound": "tensor", "achieved": li["flops"] / (per[top] * 1e-3) / 1e12, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s"}
    else:
        roof = {"bound": "hbm", "achieved": li["bytes"] / (per[top] * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = _ncu_traffic(li)
    roof.update({"kernel": f"{li['kind']}@level{li['level']}", "launch_ms": per[top],
                 "share_of_step": per[top] / ms, "algorithmic_flops": li["flops"], "algorithmic_bytes": li["bytes"],
                 "arithmetic_intensity": ai,
                 # what the kernel actually issues (compact-WY level-0 congruence:
                 # 4 n_t n_s (k_t + k_s) per pair instead of 2 n_t n_s (n_t + n_s))
                 "executed_flops": li["flops_exec"],
                 "executed_frac": li["flops_exec"] / (per[top] * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                 "peak_source": "FP64 DMMA microbenchmark on this pool's B200 (profiles/r01_fp64_peak.txt); "
                                f"cuBLAS DGEMM measured {FP64_DGEMM_TFLOPS}",
                 "hbm_peak_gbs": peaks["hbm_gbs"]})
    # SURVEY 8(a) a8 on its own: y = U^T b and x = V y timed alone (after the
    # timed region), against the HBM roofline -- algorithmic bytes = every Q_t
    # read once (8 n_t^2) + the vectors in and out (8 N nrhs each)
    def _time_apply(fn, reps=10):
        fn()
        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_a.record(stream)
        for _ in range(reps):
            fn()
        e_b.record(stream)
        torch.cuda.synchronize()
        return e_a.elapsed_time(e_b) / reps
    ut_ms = _time_apply(lambda: sp.apply_Ut(b, y, ws=aws))
    v_ms = _time_apply(lambda: sp.apply_V(y, x, ws=aws))
    loc_rr, loc_cc = plan.local_rows()
    vec_b = 8.0 * nrhs * (plan.n_tree_local + plan.s_rows)
    ut_bytes = 8.0 * float(np.sum(offs["n_row"][loc_rr >= 0].astype(float) ** 2)) + vec_b
    v_bytes = 8.0 * float(np.sum(offs["n_col"][(loc_rr if plan.symmetric else loc_cc) >= 0].astype(float) ** 2)) \
        + vec_b
    apply_info = {"ut_us": ut_ms * 1e3, "v_us": v_ms * 1e3, "ut_bytes": ut_bytes, "v_bytes": v_bytes, "nrhs": nrhs,
                  "ut_gbs": ut_bytes / (ut_ms * 1e-3) / 1e9, "v_gbs": v_bytes / (v_ms * 1e-3) / 1e9,
                  "hbm_peak_gbs": peaks["hbm_gbs"],
                  "note": "h2sp_apply_Ut / h2sp_apply_V timed alone after the timed region (10 reps each); "
                          "algorithmic bytes: every Q_t once + vectors in and out"}
    apply_info["ut_frac"] = apply_info["ut_gbs"] / peaks["hbm_gbs"]
    apply_info["v_frac"] = apply_info["v_gbs"] / peaks["hbm_gbs"]
    # whole-job throughput: the work of every rank (shards: their own flops) / max time
    fl_t = torch.tensor([step_flops], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(fl_t)
    job_flops = float(fl_t.item())
    value = job_flops / (ms_max * 1e-3) / 1e12

    # ---- e2e through the public API with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        # Jobs stream through the public host-buffer API (h2sp_build_host + the
        # applies with host vectors), `depth` of them in flight on their own
        # streams and device buffer sets: job i+1's H2D (inputs) runs while job
        # i's D2H (S, Q, x) drains -- PCIe is full duplex.  Every job still copies
        # all of its inputs in and all of its outputs out inside the timed region.
        depth = max(1, args.e2e_depth)
        # every job in flight needs its own device buffer set and pinned host outputs: full-size
        # configs[2] / configs[3] (58 / 66 GB of S) fit only one of them
        def _nbytes(dct):
            return sum(v.numel() * v.element_size() for v in dct.values() if v is not None)
        set_bytes = _nbytes(sp.inputs) + _nbytes(sp.outputs) + int(plan.sizes["workspace_bytes"])
        free_dev = torch.cuda.mem_get_info(dev)[0]
        import psutil
        free_host = psutil.virtual_memory().available
        while depth > 1 and ((depth - 1) * set_bytes > free_dev - (4 << 30)
                             or _nbytes(sp.inputs) + depth * _nbytes(sp.outputs) > 0.7 * free_host):
            depth -= 1
        host_in = {k: v.cpu().pin_memory() for k, v in sp.inputs.items()}
        hb = b.cpu().pin_memory()
        sets = []
        for d in range(depth):
            spd = sp if d == 0 else h2sp.Sparsifier(plan, packed, device=dev, close_gen=gen)
            sets.append({
                "sp": spd, "stream": torch.cuda.Stream(device=dev),
                "out": {k: (torch.empty(v.shape, dtype=v.dtype).pin_memory() if v is not None else None)
                        for k, v in spd.outputs.items()},
                "b": torch.empty_like(b), "y": torch.empty_like(y), "x": torch.empty_like(x),
                "hx": torch.empty(x.shape, dtype=x.dtype).pin_memory(),
                "aws": aws if d == 0 else spd.apply_ws(nrhs)})

        def step_e2e(i):
            st_ = sets[i % depth]
            with torch.cuda.stream(st_["stream"]):
                st_["sp"].build_host(host_in, st_["out"], stream=st_["stream"])
                st_["b"].copy_(hb, non_blocking=True)
                st_["sp"].apply_Ut(st_["b"], st_["y"], ws=st_["aws"], stream=st_["stream"])
                st_["sp"].apply_V(st_["y"], st_["x"], ws=st_["aws"], stream=st_["stream"])
                st_["hx"].copy_(st_["x"], non_blocking=True)

        def run_e2e(n):
            for st_ in sets:
                st_["stream"].wait_stream(stream)
            for i in range(n):
                step_e2e(i)
            for st_ in sets:
                stream.wait_stream(st_["stream"])

        run_e2e(2 * depth)
        torch.cuda.synchronize()
        k_e2e = max(3, min(args.steps, 10))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        run_e2e(k_e2e)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = torch.tensor([e0.elapsed_time(e1) / k_e2e], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        h2d = sum(int(v.numel()) * v.element_size() for v in host_in.values()) + hb.numel() * 8
        d2h = sum(int(v.numel()) * v.element_size() for v in sets[0]["out"].values() if v is not None) \
            + sets[0]["hx"].numel() * 8
        e2e = {"value": job_flops / (float(ems.item()) * 1e-3) / 1e12, "unit": UNIT,
               "ms_per_step": float(ems.item()), "steps": k_e2e, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "jobs_in_flight": depth,
               "api": "h2sp_build_host + h2sp_apply_Ut/V with pinned host buffers, one stream and device "
                      "buffer set per job in flight"}
        # the link's own ceiling, measured here: pinned 512 MiB copies each way
        # (alone), so e2e can be read against max(H2D, D2H) at full duplex
        try:
            nb = 1 << 26
            hbuf = torch.empty(nb, dtype=torch.float64).pin_memory()
            dbuf = torch.empty(nb, dtype=torch.float64, device=dev)

            def _copy_gbs(fn):
                fn()
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                for _ in range(3):
                    fn()
                b_.record(stream)
                torch.cuda.synchronize()
                return 3 * nb * 8 / (a_.elapsed_time(b_) * 1e-3) / 1e9
            h2d_gbs = _copy_gbs(lambda: dbuf.copy_(hbuf, non_blocking=True))
            d2h_gbs = _copy_gbs(lambda: hbuf.copy_(dbuf, non_blocking=True))
            bound_ms = max(h2d / (h2d_gbs * 1e9), d2h / (d2h_gbs * 1e9)) * 1e3
            e2e["pcie"] = {"h2d_gbs": h2d_gbs, "d2h_gbs": d2h_gbs, "bound_ms": bound_ms,
                           "frac": bound_ms / float(ems.item()),
                           "note": "bound = max(H2D bytes / H2D GB/s, D2H bytes / D2H GB/s), full duplex"}
            del hbuf, dbuf
        except RuntimeError as exc:  # pinned allocation refused: report without the bound
            e2e["pcie"] = {"error": str(exc)[:120]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_oracle and h.close is not None:
        cpu = oracle_baseline(h, plan.sizes["flops"],
                              f"one full oracle pass (sparsify + CSR assembly) of the same matrix "
                              f"(N={plan.N}); build flops only")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong" if shard else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(args.config, plan.N, h.meta.get("seed")), "N": plan.N, "B": plan.B, "L": plan.L,
                       "nrhs": nrhs, "mode": "symmetric" if plan.symmetric else "general",
                       "parallelism": (f"subtree shards x{world} of one matrix (no data-path collective; "
                                       f"Q of halo clusters recomputed per shard)") if shard else
                                      f"replicas x{world} (independent matrices per rank, no collective)",
                       "l2": ("inputs (close blocks %.2f GB) and outputs (S %.2f GB) exceed the 126 MB L2; no flush"
                              % (plan.sizes["close"] * 8e-9, plan.sizes["s_nnz"] * 12e-9)) if not args.close_gen else
                             ("outputs (S %.2f GB) exceed the 126 MB L2; no flush" % (plan.sizes["s_nnz"] * 12e-9)),
                       "close": ("matrix-free: C_ts evaluated in the level-0 congruence from the points "
                                 "(h2sp_close_gen; %.1f GB of close blocks never stored)" % (plan.sizes["close"] * 8e-9))
                                if args.close_gen else "stored (B x B per near pair, read by the level-0 congruence)",
                       "step_launch": ("CUDA graph replay of the captured step (per-launch durations from "
                                       "eager steps run after the timed region)") if args.graph else
                                      "eager (per-launch CUDA events recorded inside the timed steps)",
                       "plan_ms": plan_ms, "s_nnz": plan.sizes["s_nnz"], "s_blocks": plan.sizes["s_blocks"],
                       "flops_per_step": step_flops, "bytes_per_step": bytes_step,
                       "flops_convention": "algorithmic (SURVEY 8(d): explicit-Q congruence 2 n_t n_s (n_t + n_s)); "
                                           "executed_flops_per_step counts what the kernels issue",
                       "executed_flops_per_step": plan.sizes["flops_executed"] + apply_flops,
                       "fp64_frac_of_peak_whole_step": value / world / FP64_PEAK_TFLOPS,
                       "job_flops_per_step": job_flops,
                       "hbm_frac_whole_step": bytes_step / (ms_max * 1e-3) / (peaks["hbm_gbs"] * 1e9),
                       "breakdown_ms": {k: round(v, 4) for k, v in kinds.items()},
                       # every launch of the step, in-run (concurrent launches share the GPU):
                       # duration, executed FP64 TFLOP/s and algorithmic GB/s
                       "per_launch": [{"kind": li["kind"], "level": li["level"], "us": round(per[j] * 1e3, 1),
                                       "tflops": round(li["flops_exec"] / max(per[j], 1e-9) * 1e-9, 2),
                                       "gbs": round(li["bytes"] / max(per[j], 1e-9) * 1e-6, 0)}
                                      for j, li in enumerate(launches)],
                       # the paper's sparsity figures (Fig. 1 nnz/row; §3 Proposition, reading 12:
                       # informational, the printed bound is garbled)
                       "sparsity": {"nnz_per_row": plan.sizes["s_nnz"] / plan.s_rows,
                                    "s_blocks": plan.sizes["s_blocks"], "close_blocks": int(len(h.near)),
                                    "s_blocks_per_close_block": plan.sizes["s_blocks"] / max(1, len(h.near)),
                                    "bound_printed": 4 * plan.L + 6 * (2.0 ** -plan.L - 1),
                                    "bound_corrected": 4 * plan.L - 2 + 3 * 2.0 ** -plan.L}},
            "roofline": roof,
            "apply_roofline": apply_info,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * (n_launch + n_apply_launch),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _ncu_traffic(li):
    """dram bytes per launch of the dominant kernel from the committed ncu
    summary (profiles/*_ncu_top.json), if one exists for this kernel on this
    workload (matched on its algorithmic flop count)."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_top.json")), reverse=True):
        try:
            with open(p) as f:
                d = json.load(f)
            if (d.get("kernel_kind") == li["kind"] and d.get("level") == li["level"]
                    and d.get("algorithmic_flops") == li["flops"]
                    and d.get("executed_flops", li["flops"]) == li["flops_exec"]):
                return d.get("dram_bytes_per_launch")
        except (OSError, ValueError):
            continue
    return None


if __name__ == "__main__":
    main()
