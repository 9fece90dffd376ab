#!/usr/bin/env python
"""One small factor + solve through the C ABI, for compute-sanitizer (memcheck / racecheck /
synccheck).  Exercises the level scheduler with its lookahead side streams, the
CUDA-graph path (--graphs), the Schur-mode f3/f2 calls (--schur) and refinement.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py --config cfg0
    compute-sanitizer --tool racecheck python tools/sanitize_case.py --config cfg1 --grid 3 3 2 --size 64
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import dd_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg0")
    ap.add_argument("--grid", type=int, nargs=3, default=None)
    ap.add_argument("--size", type=int, default=None)
    ap.add_argument("--nrhs", type=int, default=3)
    ap.add_argument("--graphs", action="store_true")
    ap.add_argument("--schur", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2002_05019_b200 as dd
    if a.schur:
        from dd_inputs.fem import fem_dd, schur_block_problem
        m = fem_dd(2, 2, 1, 6, seed=0, nrhs=a.nrhs)
        prob, ns, tgt, grp, auxs, info = schur_block_problem(m, leaf=16)
        ss = dd.SchurSolver(prob.blk_size, prob.colptr, prob.rowidx, tgt, grp, auxs)
        ss._auxs = auxs
        rc, _ = ss.factor(torch.from_numpy(prob.values).cuda(), prob.val_offset)
        dS, Soff = ss.export()
        F = torch.randn(a.nrhs, prob.n, dtype=torch.float64, device="cuda").t()
        G = torch.randn(a.nrhs, m.n_dual, dtype=torch.float64, device="cuda").t()
        ss.condense_(F, G)
        X = ss.recover(F, G)
        torch.cuda.synchronize()
        print("schur case ok", rc, float(X.abs().max()))
        return
    kw = {}
    if a.grid:
        kw["grid"] = tuple(a.grid)
    if a.size:
        kw["sizes"] = a.size
    p = dd_inputs.config(a.config, **kw)
    s = dd.AuxSolver(p.blk_size, p.colptr, p.rowidx, complex_=p.is_complex, use_graphs=a.graphs, refine_tol=1e-30)
    vals = torch.from_numpy(p.values).cuda()
    for _ in range(2 if a.graphs else 1):
        rc, fi = s.factor(vals, p.val_offset)
        B = dd_inputs.random_rhs(p.n, a.nrhs, p.is_complex, 0)
        Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().t()
        s.solve_(Bd)
    torch.cuda.synchronize()
    print("case ok", a.config, p.n, rc, fi["npos"], fi["nneg"])


if __name__ == "__main__":
    main()
