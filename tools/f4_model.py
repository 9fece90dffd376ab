#!/usr/bin/env python
"""f4 timing model from the single-GPU emulation of the subtree-mapped factorization.

Each part's partial factorization (+ S export) and the top's assembly + factorization are timed
separately with CUDA events while the parts run one after the other on one B200.  On N GPUs the
parts run concurrently, so the modeled factor time is
    T_N = max_r T_part(r) + max_r bytes(S_r) / B_link + T_top,
with B_link an assumed 700 GB/s NVLink-5 point-to-point rate (NOT measured here: one GPU only).
It is a model -- the bench reports no multi-GPU factor number.

    python tools/f4_model.py --config cfg2 --parts 2 4 8 --out gpurun_out/r02_f4_model_cfg2.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import dd_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--parts", type=int, nargs="+", default=[2, 4])
    ap.add_argument("--link-gbs", type=float, default=700.0)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import torch
    import paper_2002_05019_b200 as dd
    from paper_2002_05019_b200.multigpu import MultiGPUFactor
    c = dd_inputs.CONFIGS[a.config]
    prob = dd_inputs.config(a.config, seed=0, backend="torch", device="cuda")
    order = dd.DD_ORDER_ND if c["order"] == "nd" else dd.DD_ORDER_AUTO
    s = dd.AuxSolver(prob.blk_size, prob.colptr, prob.rowidx, complex_=c["complex_"], order=order)
    s.factor(prob.values, prob.val_offset)
    rc, fi = s.factor(prob.values, prob.val_offset)
    t1 = fi["ms_factor"]
    s.close()
    del s
    torch.cuda.empty_cache()
    out = {"config": a.config, "n": prob.n, "single_gpu_factor_ms": t1, "link_gbs_assumed": a.link_gbs, "parts": {}}
    for n in a.parts:
        t0 = time.time()
        mf = MultiGPUFactor(prob.blk_size, prob.colptr, prob.rowidx, n, complex_=c["complex_"], order_opt=order)
        plan_s = time.time() - t0
        rc = mf.factor(prob.values, prob.val_offset)
        assert rc == dd.DD_OK, rc
        tm = mf.timings
        tp = max(tm["parts_ms"].values())
        xfer = max(tm["export_bytes"].values()) / (a.link_gbs * 1e9) * 1e3
        tn = tp + xfer + tm["top_ms"]
        P = mf.plan
        tot = sum(P.flops_parts) + P.flops_top
        out["parts"][n] = {"parts_ms": tm["parts_ms"], "top_ms": tm["top_ms"], "max_export_bytes": max(tm["export_bytes"].values()),
                           "modeled_factor_ms": tn, "modeled_speedup": t1 / tn, "top_flop_fraction": P.flops_top / tot,
                           "imbalance": max(P.flops_parts) / (sum(P.flops_parts) / n), "plan_s": plan_s,
                           "top_blocks": len(P.top)}
        print(n, json.dumps(out["parts"][n]), flush=True)
        del mf
        torch.cuda.empty_cache()
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
