#!/usr/bin/env python
"""Benchmark of the auxiliary-matrix block LDL^T + multi-RHS solve on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl reference]

Default workload: configs[2] (the largest config by factor flops; the north_star target is
">= 50% of measured FP64 tensor peak in the factor phase of the largest config").

Metric (BASELINE.json): "aux-matrix LDL^T factor FP64 GFLOP/s (% of FP64 peak); solve ms
per 1000 RHS".  One step = one pass of the whole hot path over one batch: dd_aux_factor
(a1 load + a2..a6 level-scheduled factorization) followed by dd_aux_solve of the config's
nrhs right-hand sides (a7 sweeps + a8 refinement).  `value` = factor GFLOP/s (algorithmic
flops of the order used / device time of dd_aux_factor), whole job = sum over ranks.
Inputs are device-resident and far larger than L2 (126 MB), so no flush is needed.

Multi-GPU: the path does not shard (north_star: one GPU, no collectives) -> N independent
replicas (weak scaling), torch.distributed only for the barrier and max-over-ranks timing.
`--impl reference` times the CPU oracle (oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import dd_inputs  # noqa: E402

# bounded oracle samples: corner sub-grid of the same workload
SAMPLE_GRID = {"cfg0": (2, 2, 1), "cfg1": (4, 4, 2), "cfg2": (3, 2, 2), "cfg3": (3, 2, 2), "cfg3alt": (3, 2, 2),
               "cfg4": (3, 2, 2)}
WORKLOAD_TXT = {
    "cfg0": "configs[0]: 2x2x1 grid, 4 x 32 real fp64, n=128",
    "cfg1": "configs[1]: 4x4x4 grid, 144 x 256 real fp64, n=36864, ND order",
    "cfg2": "configs[2]: 6x6x6 unstructured-like (L9), sizes U[128,1024], real fp64",
    "cfg3": "configs[3]: 8x8x4 grid (L10), 640 x 512 complex128 symmetric, n=327680",
    "cfg3alt": "configs[3] alt (L10): 3x6x10 grid, 432 x 512 complex128, n=221184",
    "cfg4": "configs[4]: configs[3] matrix, 10 x 1000 complex128 RHS",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("DD_BENCH_CONFIG", "cfg2"))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--refine", type=int, default=1)
    ap.add_argument("--refine-tol", type=float, default=0.0,
                    help="skip a refinement step on the device when every column has berr <= tol (0 = always)")
    ap.add_argument("--nrhs", type=int, default=None)
    ap.add_argument("--complex-4m", action="store_true",
                    help="complex Schur update with 4 real products instead of the default 3M (Gauss)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--trace-out", default=None, help="write the per-kernel trace JSON here")
    return ap.parse_args()


def fp64_peak(cplx):
    """Measured FP64 tensor peak (TFLOP/s): cuBLAS DGEMM / ZGEMM 8192^3 (tools/fp64_peak.py)."""
    path = os.path.join(ROOT, "profiles", "r01_fp64_peak.json")
    d = json.load(open(path))
    return (d["zgemm_tflops_burst"] if cplx else d["dgemm_tflops_burst"]), os.path.relpath(path, ROOT)


def hbm_peak():
    """Measured HBM copy bandwidth (GB/s) of this pool's B200s (driver-written MEASURED_PEAKS.json)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(path))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (b.copy_(a), read+write bytes)"
    except Exception:
        return 7700.0, "fallback: nominal HBM3e 7.7 TB/s (MEASURED_PEAKS.json absent)"


class Clocks:
    """nvidia-smi sampler (B200_PROFILING.md clocks line) running during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(gpu_index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.count(",") >= 8]
        os.unlink(self.f.name)
        if not rows:
            return None
        mhz = sorted(float(r[1]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip().lower() == "active"})
        return {"sm_mhz": mhz[len(mhz) // 2], "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


def berr_check(prob, Bsrc, X, ncols=8):
    """Harness check (not the measured library): per-column backward error
    ||A x - b||_inf / (||A||_inf ||x||_inf) on a few columns, fp64 torch matmuls over the
    caller's original blocks (both triangles), moduli for complex (L6)."""
    import torch
    nrhs = X.shape[1]
    cols = sorted(set(np.linspace(0, nrhs - 1, min(ncols, nrhs)).astype(int).tolist()))
    x = X[:, cols].clone()
    r = Bsrc[:, cols].clone()
    rs = torch.zeros(prob.n, dtype=torch.float64, device=X.device)
    off = prob.dof_offset
    vals = prob.values
    for j in range(prob.nblk):
        for p in range(int(prob.colptr[j]), int(prob.colptr[j + 1])):
            i = int(prob.rowidx[p])
            si, sj = int(prob.blk_size[i]), int(prob.blk_size[j])
            vo = int(prob.val_offset[p])
            blk = vals[vo:vo + si * sj].view(sj, si).t()
            oi, oj = int(off[i]), int(off[j])
            if i == j:
                S = torch.tril(blk) + torch.tril(blk, -1).t()
                r[oi:oi + si] -= S @ x[oi:oi + si]
                rs[oi:oi + si] += S.abs().sum(1)
            else:
                r[oi:oi + si] -= blk @ x[oj:oj + sj]
                r[oj:oj + sj] -= blk.t() @ x[oi:oi + si]
                rs[oi:oi + si] += blk.abs().sum(1)
                rs[oj:oj + sj] += blk.abs().sum(0)
    berr = r.abs().amax(0) / (rs.max() * x.abs().amax(0))
    return float(berr.max()), cols


def oracle_sample(prob, cfg, nrhs, config_flops=None, sub=None):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload: its factor, then
    its solve (O5 sweeps + O6 refinement, refine_steps=1) of one batch of nrhs right-hand sides."""
    import oracle
    from oracle.block_ldlt import flops_factor, flops_solve_per_rhs
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    keep = dd_inputs.corner_interfaces(prob, SAMPLE_GRID[cfg])
    if sub is None:
        sub = dd_inputs.subproblem(prob, keep)
    order = list(range(sub.nblk))
    t0 = time.perf_counter()
    F = oracle.block_factor(sub, order)
    dt = time.perf_counter() - t0
    mu = 4 if sub.is_complex else 1
    fl = flops_factor(sub.blk_size, F.sym, mu)
    B = dd_inputs.random_rhs(sub.n, nrhs, sub.is_complex, 1)
    t0 = time.perf_counter()
    oracle.refine_solve(sub, F, B, 1)
    ds = time.perf_counter() - t0
    g = SAMPLE_GRID[cfg]
    share = fl / config_flops if config_flops else None
    sample = (f"oracle.block_factor + oracle.refine_solve (nrhs={nrhs}, 1 refinement step) on the principal "
              f"sub-matrix of the {len(keep)} interfaces inside the {g[0]}x{g[1]}x{g[2]} corner sub-grid of this "
              f"workload (n={sub.n}, same bytes), natural order: factor {fl:.3g} algorithmic flops in {dt:.2f} s"
              + (f" ({100 * share:.2f}% of the config's factor flops)" if share else "")
              + f", solve {ds:.2f} s")
    return {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": int(cores), "kind": "oracle", "sample": sample,
            "seconds": dt + ds, "factor_s": dt, "solve_s": ds, "sample_n": sub.n, "sample_flops_factor": fl,
            "flops_share_of_config": share,
            "solve_ms_per_1000_rhs": ds * 1e6 / nrhs,
            "solve_gflops": 2 * mu * flops_solve_per_rhs(sub.blk_size, F.sym) * nrhs / ds / 1e9}


def dist_setup(args):
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if args.impl == "reference" else "nccl")
        pg = dist
    return rank, world, local, pg


def reduce_max(values, dist, device="cpu"):
    """Max over ranks of a few per-rank timings (barrier-bracketed device times)."""
    import torch
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def rhs_shard(batches, world, rank):
    """f4: the multi-RHS solve shards by right-hand-side columns with zero
    communication -- every rank holds its own factor replica and solves batches
    rank, rank + world, ... of the job's RHS batches (round robin)."""
    return list(range(rank, batches, world))


def reference_arm(args, rank, world):
    """The oracle on the box's host cores; rank 0 only (others exit 0 without work)."""
    if rank != 0:
        return
    cfg = args.config
    try:
        import torch
        dev = "cuda" if torch.cuda.is_available() else "cpu"
    except Exception:
        dev = "cpu"
    c = dd_inputs.CONFIGS[cfg]
    if dev == "cuda":  # same bytes as our arm's workload, carved on the device
        prob = dd_inputs.config(cfg, seed=args.seed, backend="torch", device="cuda")
    else:
        prob = dd_inputs.config(cfg, seed=args.seed, grid=SAMPLE_GRID[cfg])
    sub = dd_inputs.subproblem(prob, dd_inputs.corner_interfaces(prob, SAMPLE_GRID[cfg]))
    nr = min(c["nrhs"], 256)
    for _ in range(args.warmup):
        oracle_sample(prob, cfg, nr, sub=sub)
    vals, secs = [], 0.0
    cb = None
    for _ in range(args.steps):
        cb = oracle_sample(prob, cfg, nr, sub=sub)
        vals.append(cb["value"])
        secs += cb["seconds"]
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": "aux-matrix LDL^T factor FP64 GFLOP/s (% of FP64 peak); solve ms per 1000 RHS",
            "value": v, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": secs * 1e3 / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128" if c["complex_"] else "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_TXT[cfg], "nrhs": c["nrhs"], "sample": SAMPLE_GRID[cfg]},
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": cb["cores"], "kind": "oracle", "sample": cb["sample"],
                             "solve_ms_per_1000_rhs": cb["solve_ms_per_1000_rhs"]},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def gpu_arm(args, rank, world, local, dist):
    import torch
    import paper_2002_05019_b200 as dd

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = args.config
    c = dd_inputs.CONFIGS[cfg]
    nrhs = args.nrhs or c["nrhs"]
    t0 = time.time()
    # clique form of the workload (one dense S_p per subdomain, drawn on the device)
    prob, Scl, Soff = dd_inputs.config_cliques(cfg, seed=args.seed + rank, device=str(dev))
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    cplx = prob.is_complex
    order = dd.DD_ORDER_ND if c["order"] == "nd" else dd.DD_ORDER_AUTO
    t0 = time.time()
    solver = dd.AuxSolver(prob.blk_size, prob.colptr, prob.rowidx, complex_=cplx, order=order,
                          refine_steps=args.refine, device=str(dev), refine_tol=args.refine_tol,
                          complex_3m=not args.complex_4m)
    analyze_s = time.time() - t0
    info = solver.info
    # f1: the auxiliary matrix is assembled on the device from the cliques by the library
    # (HBM-bound; measured here, outside the factor+solve step), then the cliques are freed
    cl = [c for _, c in prob.cliques]
    vals = solver.assemble(cl, Scl, Soff, prob.val_offset)
    dd.dd_aux_set_trace(solver.h, True)
    dd.dd_aux_get_trace(solver.h, reset=True)
    solver.assemble(cl, Scl, Soff, prob.val_offset, d_vals=vals)
    asm_ms = dd.dd_aux_get_trace(solver.h, reset=True)["assemble"]["ms"]
    dd.dd_aux_set_trace(solver.h, False)
    asm_bytes = dd.dd_aux_last_assemble_bytes(solver.h)
    del Scl
    solver._asm_work = None
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    prob.values = vals
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + args.seed + rank)
    tdt = torch.complex128 if cplx else torch.float64
    Bsrc = torch.randn((nrhs, prob.n), dtype=tdt, device=dev, generator=gen).t()  # column-major n x nrhs
    Bw = torch.empty((nrhs, prob.n), dtype=tdt, device=dev).t()
    batches = c.get("batches", 1)  # configs[4]: many-excitation stress test, batches of nrhs per step
    # f4: with several batches per step and N > 1 ranks, the RHS batches are sharded across the
    # ranks' factor replicas (strong scaling of the solve); a single batch is replicated (weak)
    my_batches = rhs_shard(batches, world, rank) if batches > 1 else [0]
    solver.factor(vals, prob.val_offset)  # allocates factor/work buffers
    solver._work(max(info["work_bytes"], dd.dd_aux_solve_work_bytes(solver.h, nrhs)))
    stream = torch.cuda.current_stream()
    bgen = torch.Generator(device=dev)

    def load_batch(b):
        """Right-hand sides of batch b: batch 0 is Bsrc; configs[4]'s other batches are distinct
        N(0,1) draws (seeded per batch, drawn on the device: 2 ms against a 3.5 s solve)."""
        if b == 0:
            Bw.copy_(Bsrc)
        else:
            bgen.manual_seed(7919 * (b + 1) + args.seed)
            Bw.t().copy_(torch.randn((nrhs, prob.n), dtype=tdt, device=dev, generator=bgen))

    def step(ev):
        ev[0].record(stream)
        rc, fi = solver.factor(vals, prob.val_offset)
        if rc != dd.DD_OK:
            raise RuntimeError(f"factor rc={rc}")
        ev[1].record(stream)
        ev[2].record(stream)
        for b in my_batches:
            load_batch(b)
            solver.solve_(Bw)
        ev[3].record(stream)
        return fi

    mk = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(4)]  # noqa: E731
    for _ in range(args.warmup):
        step(mk())
    torch.cuda.synchronize()
    # ---- timed region: UNTRACED (no per-launch events), CUDA events on the launching stream
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [mk() for _ in range(args.steps)]
    dd.dd_aux_get_trace(solver.h, reset=True)  # launch counters are kept even with tracing off
    start.record(stream)
    finfo = None
    for k in range(args.steps):
        finfo = step(evs[k])
    end.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    total_ms = start.elapsed_time(end)
    fac_ms = sum(e[0].elapsed_time(e[1]) for e in evs)
    sol_ms = sum(e[2].elapsed_time(e[3]) for e in evs)
    launches = sum(v["launches"] for v in dd.dd_aux_get_trace(solver.h, reset=True).values())
    # ---- per-kernel breakdown from a SEPARATE traced pass of the same step (event pair around
    # every launch on its own stream); its step time is reported beside the untraced one
    step_s = total_ms / args.steps / 1e3
    KT = max(1, min(args.steps, int(np.ceil(20.0 / max(step_s, 1e-3)))))
    dd.dd_aux_set_trace(solver.h, True)
    dd.dd_aux_get_trace(solver.h, reset=True)
    tev = [mk() for _ in range(KT)]
    for k in range(KT):
        step(tev[k])
    torch.cuda.synchronize()
    traced_fac_ms = sum(e[0].elapsed_time(e[1]) for e in tev) / KT
    traced_sol_ms = sum(e[2].elapsed_time(e[3]) for e in tev) / KT
    trace = dd.dd_aux_get_trace(solver.h, reset=False)
    lvl = dd.dd_aux_get_level_trace(solver.h)
    dd.dd_aux_get_trace(solver.h, reset=True)
    dd.dd_aux_set_trace(solver.h, False)

    # ---- accuracy evidence (harness, outside the timed region): berr of the timed result and of
    # an unrefined solve of the same right-hand sides; configs[4]: EVERY column of every batch
    load_batch(my_batches[-1])
    Bref = Bw.clone()               # b of the step's last batch
    solver.solve_(Bw)               # x (deterministic: bitwise the timed result)
    berr, cols = berr_check(prob, Bref, Bw)
    berr_all = None
    if batches > 1:  # configs[4] (ledger L15): berr of all nrhs x batches columns
        berr_all = {"max": 0.0, "columns": 0}
        for b in my_batches:
            load_batch(b)
            Bb = Bw.clone()
            solver.solve_(Bw)
            be, cl = berr_check(prob, Bb, Bw, ncols=nrhs)
            berr_all["max"] = max(berr_all["max"], be)
            berr_all["columns"] += len(cl)
            del Bb
        load_batch(0)
        solver.solve_(Bw)
    Bu = torch.empty((len(cols), prob.n), dtype=tdt, device=dev).t()
    Bu.copy_(Bref[:, cols])
    dd.dd_aux_set_refine(solver.h, 0, 0.0)
    solver.solve_(Bu)
    dd.dd_aux_set_refine(solver.h, args.refine, args.refine_tol)
    berr0, _ = berr_check(prob, Bref[:, cols], Bu, ncols=len(cols))
    del Bu, Bref

    # ---- max over ranks (device-timed), NCCL all-reduce of three scalars (plumbing only)
    total_ms, fac_ms, sol_ms = reduce_max([total_ms, fac_ms, sol_ms], dist, dev)

    K = args.steps
    flops = info["flops_factor"]
    value = world * flops * K / (fac_ms * 1e-3) / 1e9
    peak_tf, peak_src = fp64_peak(cplx)
    # ---- roofline of the dominant kernel (largest device time in the step)
    dom = max(trace, key=lambda p: trace[p]["ms"])
    dk = trace[dom]
    achieved = dk["flops"] / (dk["ms"] * 1e-3) / 1e12 if dk["ms"] > 0 else 0.0
    achieved_eff = achieved
    if cplx and not args.complex_4m and dom in ("k3_update", "k2_panel", "fupd", "bupd", "fdiag", "bdiag"):
        achieved = 0.75 * achieved_eff  # 3M executes 3 of the 4 real products the 8-flop convention counts
    traffic, traffic_src = None, None
    asm_traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{cfg}.json")
    if os.path.exists(tpath):  # dram read+write bytes per launch from one ncu --set full capture
        tj = json.load(open(tpath))
        t = tj.get(dom)
        if t:
            traffic, traffic_src = t["dram_bytes_per_launch"], t["launch"]
        if tj.get("k_assemble"):
            asm_traffic = tj["k_assemble"]
    step_ms = total_ms / K

    # ---- e2e: host buffers through the public API (H2D inputs, D2H result inside the region)
    e2e = None
    if not args.no_e2e:
        vh = vals.cpu().pin_memory()
        bh = Bsrc.t().contiguous().cpu().pin_memory()  # (nrhs, n) row-major == column-major n x nrhs
        xh = torch.empty_like(bh).pin_memory()
        evs2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        evs2[0].record(stream)
        vals.copy_(vh, non_blocking=True)
        rc, _ = solver.factor(vals, prob.val_offset)
        evs2[1].record(stream)
        Bw.t().copy_(bh, non_blocking=True)
        solver.solve_(Bw)
        xh.copy_(Bw.t(), non_blocking=True)
        evs2[2].record(stream)
        torch.cuda.synchronize()
        f_ms = evs2[0].elapsed_time(evs2[1])
        s_ms = evs2[1].elapsed_time(evs2[2])
        e2e = {"value": world * flops / (f_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(vh.numel() * vh.element_size() + bh.numel() * bh.element_size()),
               "d2h_bytes_per_step": int(xh.numel() * xh.element_size()),
               "solve_ms_per_1000_rhs": s_ms * 1000.0 / nrhs, "factor_ms": f_ms}
        del vh, bh, xh

    # ---- a5 evidence: the same step replayed from CUDA graphs (options.use_graphs; tracing off, so
    # outside the traced timed region above); reported for the small, launch-bound configs
    graphs = None
    if prob.n <= 100000:
        dd.dd_aux_set_graphs(solver.h, True)
        for _ in range(2):  # capture + one replay
            step(mk())
        torch.cuda.synchronize()
        gev = [mk() for _ in range(K)]
        for k in range(K):
            step(gev[k])
        torch.cuda.synchronize()
        dd.dd_aux_set_graphs(solver.h, False)
        g_fac = sum(e[0].elapsed_time(e[1]) for e in gev) / K
        g_sol = sum(e[2].elapsed_time(e[3]) for e in gev) / K
        graphs = {"factor_ms": g_fac, "solve_ms_per_batch": g_sol / max(1, len(my_batches)),
                  "solve_ms_per_1000_rhs": g_sol * 1000.0 / (nrhs * max(1, len(my_batches))),
                  "what": "same step with use_graphs=1 (factor level loop + solve replayed from CUDA graphs), "
                          "untraced, after the timed region"}
    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(prob, cfg, min(nrhs, 256), config_flops=info["flops_factor"])
        cpu.pop("seconds", None)
    line = {
        "metric": "aux-matrix LDL^T factor FP64 GFLOP/s (% of FP64 peak); solve ms per 1000 RHS",
        "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128" if cplx else "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_TXT[cfg], "n": prob.n, "nblk": prob.nblk, "nrhs": nrhs,
                   "order": ["auto", "nd", "mindeg", "natural", "user"][info["order_used"]],
                   "levels": info["n_levels"], "refine_steps": args.refine, "refine_tol": args.refine_tol,
                   "complex_product": ("4M" if args.complex_4m else "3M (effective GFLOP/s, 8-flop convention)")
                   if cplx else None,
                   "l2": "inputs larger than L2 (no flush needed)",
                   "parallelism": "replicas" if world > 1 else "single GPU"},
        "factor_ms": fac_ms / K, "factor_frac_of_fp64_peak": value / world / 1e3 / peak_tf,
        "solve_ms_per_1000_rhs": (sol_ms / K * 1000.0 / (nrhs * batches)) if batches > 1
        else (sol_ms / K * 1000.0 / nrhs),
        "solve_ms_per_batch": sol_ms / K / max(1, len(my_batches)),
        "solve_batches_per_step": batches,
        "solve_sharding": ({"by": "rhs batches (round robin over the ranks' factor replicas)", "scaling": "strong",
                            "batches_per_rank": [len(rhs_shard(batches, world, r)) for r in range(world)]}
                           if batches > 1 and world > 1 else None),
        # HBM evidence for the solve: each sweep streams the whole factor once (L panels + inverse
        # diagonal blocks); (1 + refine_steps) sweeps per batch; achieved = those bytes / solve time
        "solve_hbm_gbs": (1 + args.refine) * info["factor_value_bytes"] * len(my_batches) * K / (sol_ms * 1e-3) / 1e9,
        "flops_factor": flops, "flops_solve_per_rhs": info["flops_solve_per_rhs"],
        "trace_pass": {"steps": KT, "factor_ms": traced_fac_ms, "solve_ms": traced_sol_ms,
                       "what": "per-kernel ms/launches/flops (phases, roofline) come from this separate "
                               "traced pass (CUDA-event pair around every launch); the timed region above "
                               "runs untraced"},
        "accuracy": {"berr_max": berr, "berr_unrefined_max": berr0, "columns_checked": len(cols),
                     "berr_all_columns": berr_all,
                     "tolerance": 1e-12, "refine_steps": args.refine, "refine_tol": args.refine_tol,
                     "pivots": {"n2x2": finfo["n2x2"], "nswaps": finfo["nswaps"]},
                     "inertia": None if cplx else [finfo["npos"], finfo["nneg"], finfo["nzero"]]},
        "roofline": {"kernel": dom, "bound": "tensor", "achieved": achieved, "achieved_effective_8flop": achieved_eff,
                     "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved / peak_tf, "traffic": traffic, "traffic_src": traffic_src,
                     "peak_src": f"measured cuBLAS {'ZGEMM' if cplx else 'DGEMM'} 8192^3 ({peak_src})"},
        "phases": {p: {"ms_per_step": v["ms"] / KT, "launches_per_step": v["launches"] / KT,
                       "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["ms"] > 0 and v["flops"] > 0 else None}
                   for p, v in trace.items() if v["launches"]},
        "assemble": {"kernel": "k_assemble", "bound": "hbm", "ms": asm_ms, "bytes": asm_bytes,
                     "achieved_gbs": asm_bytes / (asm_ms * 1e-3) / 1e9 if asm_ms > 0 else None,
                     "peak_gbs": hbm_peak()[0], "frac": (asm_bytes / (asm_ms * 1e-3) / 1e9 / hbm_peak()[0])
                     if asm_ms > 0 else None, "peak_src": hbm_peak()[1],
                     "traffic": asm_traffic["dram_bytes_per_launch"] if asm_traffic else None,
                     "traffic_src": asm_traffic["launch"] if asm_traffic else None,
                     "what": "f1: A = sum_p sym(S_p) over the cliques, read S_p blocks + write A (algorithmic bytes)"},
        "gpu_launches": launches,
        "clocks": clk, "cpu_baseline": cpu, "e2e": e2e, "graphs": graphs,
        "setup_s": {"generate": gen_s, "analyze": analyze_s},
    }
    if args.trace_out:
        json.dump({"trace": trace, "line": line, "phases": dd.PHASES,
                   "level_ms": (lvl["ms"] / KT).tolist(), "level_flops": (lvl["flops"] / KT).tolist()},
                  open(args.trace_out, "w"), indent=1)
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ f2/f3 pipeline
FEM_CONFIGS = {  # FEM-like DD models (dd_inputs.fem): grid of a^3-node subdomains, (a-2)^2 duals per face
    "fem1": dict(grid=(4, 4, 4), a=18, leaf=128, complex_=False, nrhs=64,
                 txt="FEM-like DD (dd_inputs.fem): 4x4x4 subdomains of 18^3 primal nodes (373,248 primal DoFs), "
                     "144 interfaces x 256 duals -> the configs[1]-shaped auxiliary matrix from actual eliminations"),
    "fem3": dict(grid=(4, 4, 2), a=18, leaf=128, complex_=True, nrhs=64,
                 txt="FEM-like DD, complex symmetric (lossy): 4x4x2 subdomains of 18^3 nodes, 64 interfaces x 256"),
}


def fem_arm(args, rank, world, local, dist):
    """f3 (subdomain elimination) -> f1 (assembly) -> aux LDL^T -> condense -> aux solve -> f2
    (primal recovery), every step in the library.  value = f3 partial-factorization GFLOP/s."""
    import torch
    import scipy.sparse as sps
    import paper_2002_05019_b200 as dd
    from dd_inputs.fem import fem_dd, schur_block_problem, arrowhead, arrowhead_rhs

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    fc = FEM_CONFIGS[args.config]
    nrhs = args.nrhs or fc["nrhs"]
    t0 = time.time()
    m = fem_dd(*fc["grid"], fc["a"], complex_=fc["complex_"], seed=args.seed + rank, nrhs=nrhs)
    leaf = int(os.environ.get("DD_FEM_LEAF", fc["leaf"]))  # supernode (ND leaf) size: the ordering input
    prob, ns, tgt, grp, auxs, info = schur_block_problem(m, leaf=leaf)
    gen_s = time.time() - t0
    cplx = fc["complex_"]
    tdt = torch.complex128 if cplx else torch.float64
    t0 = time.time()
    ss = dd.SchurSolver(prob.blk_size, prob.colptr, prob.rowidx, tgt, grp, auxs, complex_=cplx, device=str(dev))
    ss._auxs = auxs
    cl = ss.cliques()
    colptr, rowidx = dd_inputs.block_pattern_from_cliques(len(auxs), cl)
    aux_off, aux_tot = dd_inputs._layout(auxs, colptr, rowidx)
    aux = dd.AuxSolver(auxs, colptr, rowidx, complex_=cplx, device=str(dev), order=dd.DD_ORDER_ND)
    analyze_s = time.time() - t0
    vals = torch.from_numpy(prob.values).to(dev)
    F = np.zeros((prob.n, nrhs), dtype=np.complex128 if cplx else np.float64)
    for p in range(m.nsub):
        s0, n_p = info["sub_dof"][p]
        F[s0:s0 + n_p] = m.f[p][info["node_perm"]]
    Fd = torch.from_numpy(np.ascontiguousarray(F.T)).to(dev).t()
    bbd = torch.from_numpy(np.ascontiguousarray(m.bb.T)).to(dev).t()
    G = torch.empty((nrhs, m.n_dual), dtype=tdt, device=dev).t()
    X = torch.empty((nrhs, prob.n), dtype=tdt, device=dev).t()
    avals = torch.empty(aux_tot, dtype=tdt, device=dev)
    ss.factor(vals, prob.val_offset)
    dS, Soff = ss.export()
    aux.assemble(cl, dS, Soff, aux_off, d_vals=avals, symmetrize=False)
    aux.factor(avals, aux_off)
    ss._work(max(ss.info["work_bytes"], dd.dd_aux_solve_work_bytes(ss.h, nrhs)))
    aux._work(max(aux.info["work_bytes"], dd.dd_aux_solve_work_bytes(aux.h, nrhs)))
    stream = torch.cuda.current_stream()

    def step(ev):
        ev[0].record(stream)
        rc, fi = ss.factor(vals, prob.val_offset)                     # f3: partial LDL^T of all subdomains
        if rc != dd.DD_OK:
            raise RuntimeError(f"partial factor rc={rc}")
        ss.export(dS, Soff)                                           # f3: S_p out
        ev[1].record(stream)
        aux.assemble(cl, dS, Soff, aux_off, d_vals=avals, symmetrize=False)   # f1
        rc2, _ = aux.factor(avals, aux_off)                            # aux block LDL^T (hot path)
        if rc2 != dd.DD_OK:
            raise RuntimeError(f"aux factor rc={rc2}")
        ev[2].record(stream)
        G.copy_(bbd)
        ss.condense_(Fd, G)                                           # g = b_b - sum C^T K^-1 f
        aux.solve_(G)                                                 # x_b
        ev[3].record(stream)
        ss.recover(Fd, G, X)                                          # f2: x_p
        ev[4].record(stream)
        return fi

    mk = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(5)]  # noqa: E731
    for _ in range(args.warmup):
        step(mk())
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = Clocks(local)
    evs = [mk() for _ in range(args.steps)]
    dd.dd_aux_get_trace(ss.h, reset=True)
    dd.dd_aux_get_trace(aux.h, reset=True)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    end.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    K = args.steps
    launches = sum(v["launches"] for v in dd.dd_aux_get_trace(ss.h, reset=True).values()) + \
        sum(v["launches"] for v in dd.dd_aux_get_trace(aux.h, reset=True).values())
    tot_ms = start.elapsed_time(end)
    f3_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / K
    aux_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / K
    cond_ms = sum(e[2].elapsed_time(e[3]) for e in evs) / K
    rec_ms = sum(e[3].elapsed_time(e[4]) for e in evs) / K
    f3_ms, aux_ms, cond_ms, rec_ms, tot_ms = reduce_max([f3_ms, aux_ms, cond_ms, rec_ms, tot_ms], dist, dev)
    # traced pass (per-kernel breakdown; separate from the timed region)
    for h in (ss.h, aux.h):
        dd.dd_aux_set_trace(h, True)
        dd.dd_aux_get_trace(h, reset=True)
    step(mk())
    torch.cuda.synchronize()
    tr_s = dd.dd_aux_get_trace(ss.h, reset=True)
    tr_a = dd.dd_aux_get_trace(aux.h, reset=True)
    for h in (ss.h, aux.h):
        dd.dd_aux_set_trace(h, False)
    # e2e: the same step through the public API from pinned HOST buffers (values, F, b_b in; X, x_b out)
    e2e = None
    if not args.no_e2e:
        vh = vals.cpu().pin_memory()
        Fh = Fd.t().contiguous().cpu().pin_memory()
        bh = bbd.t().contiguous().cpu().pin_memory()
        Xh_ = torch.empty((nrhs, prob.n), dtype=tdt).pin_memory()
        Gh_ = torch.empty((nrhs, m.n_dual), dtype=tdt).pin_memory()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        vals.copy_(vh, non_blocking=True)
        Fd.t().copy_(Fh, non_blocking=True)
        bbd.t().copy_(bh, non_blocking=True)
        step(mk())
        Xh_.copy_(X.t(), non_blocking=True)
        Gh_.copy_(G.t(), non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        fl3e = ss.info["flops_factor"]
        e2e = {"value": fl3e / (e_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "step_ms": e_ms,
               "h2d_bytes_per_step": int(vh.numel() * vh.element_size() + Fh.numel() * Fh.element_size() +
                                         bh.numel() * bh.element_size()),
               "d2h_bytes_per_step": int(Xh_.numel() * Xh_.element_size() + Gh_.numel() * Gh_.element_size()),
               "what": "whole f3 -> f1 -> aux -> condense -> aux solve -> f2 step from pinned host buffers; "
                       "value = f3 flops / the whole e2e step time (a lower bound of the f3 rate)"}
        del vh, Fh, bh, Xh_, Gh_
    # accuracy: the global arrowhead residual of the step's solution (harness, scipy on the host)
    Xh = X.cpu().numpy()
    xs = []
    for p in range(m.nsub):
        s0, n_p = info["sub_dof"][p]
        x = np.empty((n_p, nrhs), dtype=Xh.dtype)
        x[info["node_perm"]] = Xh[s0:s0 + n_p]
        xs.append(x)
    got = np.concatenate(xs + [G.cpu().numpy()])
    A = arrowhead(m)
    b = arrowhead_rhs(m)
    nA = float(abs(A).sum(axis=1).max())
    berr = float((np.abs(A @ got - b).max(0) / (nA * np.abs(got).max(0))).max())
    if rank != 0:
        return
    fl3 = ss.info["flops_factor"]
    value = world * fl3 / (f3_ms * 1e-3) / 1e9
    peak_tf, peak_src = fp64_peak(cplx)
    comb = {}
    for nm, tr in (("sub", tr_s), ("aux", tr_a)):
        for ph, v in tr.items():
            if v["launches"]:
                comb[f"{nm}:{ph}"] = v
    dom = max((q for q in comb if q.startswith("sub:")), key=lambda q: comb[q]["ms"])  # the f3 kernels
    dk = comb[dom]
    achieved = dk["flops"] / (dk["ms"] * 1e-3) / 1e12 if dk["ms"] > 0 and dk["flops"] > 0 else None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:  # oracle.dd on a bounded sample: 2 subdomains' S_p
        import oracle.dd as odd
        try:
            from threadpoolctl import threadpool_info
            cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
        except Exception:
            cores = os.cpu_count()
        t0 = time.perf_counter()
        nsamp = 2
        for p in range(nsamp):
            odd.schur_contribution(m, p)
        dt = time.perf_counter() - t0
        per_sub_gpu_flops = fl3 / m.nsub
        cpu = {"value": nsamp * per_sub_gpu_flops / dt / 1e9, "unit": "GFLOP/s (the library's per-subdomain "
               "algorithmic flops / oracle time)", "cores": int(cores), "kind": "oracle",
               "sample": f"oracle.dd.schur_contribution (scipy SuperLU solve of K_p against C_p, then C_p^T W) for "
                         f"{nsamp} of the {m.nsub} subdomains: {dt:.2f} s; the GPU does all {m.nsub} in {f3_ms:.1f} ms",
               "seconds_per_subdomain": dt / nsamp}
    line = {
        "metric": "f3 subdomain elimination (partial block LDL^T of all subdomains + S_p export) FP64 GFLOP/s; "
                  "f2 recovery ms per RHS batch",
        "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": tot_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128" if cplx else "f64", "data": "synthetic",
        "config": {"workload": fc["txt"], "n_arrowhead": int(A.shape[0]), "n_sub_handle": prob.n,
                   "nblk": prob.nblk, "n_schur": ns, "leaf": leaf, "nrhs": nrhs,
                   "levels": ss.info["n_levels"], "aux_n": m.n_dual},
        "f3_ms": f3_ms, "f3_tflops": fl3 / (f3_ms * 1e-3) / 1e12, "f3_frac_of_fp64_peak": fl3 / (f3_ms * 1e-3) / 1e12 / peak_tf,
        "f1_plus_aux_factor_ms": aux_ms, "condense_plus_aux_solve_ms": cond_ms, "f2_recover_ms": rec_ms,
        "f2_recover_ms_per_1000_rhs": rec_ms * 1000.0 / nrhs,
        "flops_f3": fl3, "flops_aux_factor": aux.info["flops_factor"],
        "accuracy": {"global_berr_max": berr, "tolerance": 1e-12, "columns": nrhs},
        "roofline": {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved / peak_tf if achieved else None, "traffic": None,
                     "peak_src": f"measured cuBLAS {'ZGEMM' if cplx else 'DGEMM'} 8192^3 ({peak_src})"},
        "phases": {q: {"ms_per_step": v["ms"], "launches_per_step": v["launches"],
                       "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["ms"] > 0 and v["flops"] > 0 else None}
                   for q, v in comb.items()},
        "gpu_launches": launches, "clocks": clk, "cpu_baseline": cpu,
        "e2e": e2e, "setup_s": {"generate": gen_s, "analyze": analyze_s},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local, dist = dist_setup(args)
    if args.impl == "reference":
        reference_arm(args, rank, world)
    elif args.config in FEM_CONFIGS:
        fem_arm(args, rank, world, local, dist)
    else:
        gpu_arm(args, rank, world, local, dist)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
