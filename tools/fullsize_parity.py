#!/usr/bin/env python
"""Full-size GPU-vs-oracle parity on one BASELINE workload (north_star: "matches the CPU oracle
within the stated tolerances on all five configs").

    python tools/fullsize_parity.py --config cfg3 --nrhs 16 --out profiles/r02_fullsize_parity_cfg3.json

The matrix is drawn on the device exactly as bench.py draws it (dd_inputs torch back-end, seed 0).
The GPU path factors and solves it through the C ABI; then the same bytes go to the host and the
CPU oracle (oracle.block_factor + oracle.refine_solve, as it stands) factors and solves them in
the GPU's block elimination order.  Reported: per-column relative difference, backward error of
both sides (oracle residual code, fp64 on the host), inertia (real), the oracle's wall time and
the host's core count.  Test infrastructure: it is the only tool besides tests/ and bench.py that
executes oracle/.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import dd_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--nrhs", type=int, default=16)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import torch
    import oracle
    from oracle.block_ldlt import residual_berr, norm_inf_A
    import paper_2002_05019_b200 as dd

    c = dd_inputs.CONFIGS[a.config]
    t0 = time.time()
    prob = dd_inputs.config(a.config, seed=0, backend="torch", device="cuda")
    gen_s = time.time() - t0
    s = dd.AuxSolver(prob.blk_size, prob.colptr, prob.rowidx, complex_=c["complex_"],
                     order=dd.DD_ORDER_ND if c["order"] == "nd" else dd.DD_ORDER_AUTO)
    B = dd_inputs.random_rhs(prob.n, a.nrhs, c["complex_"], 21)
    rc, fi = s.factor(prob.values, prob.val_offset)
    assert rc == dd.DD_OK, rc
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().t()
    s.solve_(Bd)
    torch.cuda.synchronize()
    X = Bd.cpu().numpy()
    order = list(s.order())
    info = dict(s.info)
    s.close()
    del Bd
    prob.values = prob.values.cpu().numpy()
    torch.cuda.empty_cache()
    print(f"[gpu] n={prob.n} factor+solve done; oracle starts", flush=True)
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    t0 = time.time()
    F = oracle.block_factor(prob, order)
    of_s = time.time() - t0
    print(f"[oracle] factor {of_s:.1f} s", flush=True)
    t0 = time.time()
    Xo, berr0_o, berr_o = oracle.refine_solve(prob, F, B, 1)
    os_s = time.time() - t0
    nA = norm_inf_A(prob)
    berr_g = residual_berr(prob, X, B, nA)
    rel = np.abs(X - Xo).max(axis=0) / np.abs(Xo).max(axis=0)
    out = {
        "config": a.config, "workload": f"BASELINE {a.config} at full size, seed 0 (bench.py's draws)",
        "n": prob.n, "nblk": prob.nblk, "nrhs": a.nrhs, "order_used": info["order_used"],
        "gpu": {"factor_ms": fi["ms_factor"], "berr_max": float(berr_g.max()), "n2x2": fi["n2x2"],
                "max_abs_L": fi["max_abs_L"],
                "inertia": None if c["complex_"] else [fi["npos"], fi["nneg"], fi["nzero"]]},
        "oracle": {"factor_s": of_s, "solve_s": os_s, "cores": int(cores), "berr_max": float(berr_o.max()),
                   "berr_unrefined_max": float(berr0_o.max()), "n2x2": F.n2x2, "max_abs_L": oracle.max_abs_L(F),
                   "inertia": None if c["complex_"] else list(oracle.inertia(F))},
        "rel_diff_max": float(rel.max()), "rel_diff_per_column": rel.tolist(),
        "tolerances": {"rel_diff": 1e-9, "berr": 1e-12},
        "pass": bool(rel.max() <= 1e-9 and berr_g.max() <= 1e-12 and berr_o.max() <= 1e-12 and
                     (c["complex_"] or [fi["npos"], fi["nneg"], fi["nzero"]] == list(oracle.inertia(F)))),
        "generate_s": gen_s,
    }
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "rel_diff_per_column"}), flush=True)


if __name__ == "__main__":
    main()
