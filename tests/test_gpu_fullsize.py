"""Full-size BASELINE workloads (configs[2], configs[3]) in the launch configuration bench.py
times, checked through properties that hold at any size (the oracle cannot factor them):

* backward error ||A x - b||_inf / (||A||_inf ||x||_inf) <= 1e-12 on sampled columns, evaluated
  by an independent fp64 harness product over the caller's original blocks (bench.berr_check);
* real case: Sylvester inertia is a congruence invariant, so the negated matrix must report the
  swapped counts (n_+, n_-) -> (n_-, n_+) with no zero pivots, and n_+ + n_- = n;
* the matrix is assembled on the device by the library (f1) from the seeded cliques.
"""
import numpy as np
import pytest

import dd_inputs

pytestmark = pytest.mark.gpu


def _run(name, nrhs):
    import torch
    import bench
    import paper_2002_05019_b200 as dd
    prob, Scl, Soff = dd_inputs.config_cliques(name, seed=0, device="cuda")
    c = dd_inputs.CONFIGS[name]
    s = dd.AuxSolver(prob.blk_size, prob.colptr, prob.rowidx, complex_=c["complex_"],
                     order=dd.DD_ORDER_ND if c["order"] == "nd" else dd.DD_ORDER_AUTO)
    vals = s.assemble([m for _, m in prob.cliques], Scl, Soff, prob.val_offset)
    del Scl
    s._asm_work = None
    torch.cuda.empty_cache()
    prob.values = vals
    rc, fi = s.factor(vals, prob.val_offset)
    assert rc == dd.DD_OK
    tdt = torch.complex128 if c["complex_"] else torch.float64
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    B = torch.randn((nrhs, prob.n), dtype=tdt, device="cuda", generator=g).t()
    X = torch.empty((nrhs, prob.n), dtype=tdt, device="cuda").t()
    X.copy_(B)
    s.solve_(X)
    torch.cuda.synchronize()
    berr, _ = bench.berr_check(prob, B, X, ncols=6)
    return prob, s, vals, fi, berr


def test_cfg3_full_size_backward_error():
    prob, s, vals, fi, berr = _run("cfg3", 40)
    s.close()
    assert prob.n == 327680
    assert berr <= 1e-12, berr


def test_cfg2_full_size_backward_error_and_inertia():
    import paper_2002_05019_b200 as dd
    prob, s, vals, fi, berr = _run("cfg2", 24)
    assert berr <= 1e-12, berr
    assert fi["nzero"] == 0 and fi["npos"] + fi["nneg"] == prob.n
    vals.neg_()
    rc, fi2 = s.factor(vals, prob.val_offset)
    s.close()
    assert rc == dd.DD_OK
    assert (fi2["npos"], fi2["nneg"], fi2["nzero"]) == (fi["nneg"], fi["npos"], 0)
