"""f4 on the GPU: the subtree-mapped factorization + distributed solve (MultiGPUFactor), run in its
single-process emulation (the parts one after the other on cuda:0 -- no rank waits on another),
against the CPU oracle's factorization of the whole matrix: solution relative difference <= 1e-9,
backward error <= 1e-12, the north_star tolerances.  The multi-process NCCL schedule is the same
code with torch.distributed point-to-point / reduce / broadcast (tests/test_multigpu_host.py runs
its protocol with gloo on CPU)."""
import numpy as np
import pytest

import dd_inputs
from dd_inputs import random_rhs
import oracle
from oracle.block_ldlt import residual_berr

from tests._gpu import rel_diff, to_dev_colmajor

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,grid,sizes,nparts", [
    ("cfg1", (3, 3, 2), 40, 2), ("cfg1", (3, 3, 2), 40, 4),
    ("cfg2", (3, 3, 2), lambda n, r: r.integers(30, 120, n), 3),
    ("cfg3", (3, 2, 2), 48, 2),
])
def test_subtree_mapped_factor_and_solve(name, grid, sizes, nparts):
    import torch
    import paper_2002_05019_b200 as dd
    from paper_2002_05019_b200.multigpu import MultiGPUFactor
    p = dd_inputs.config(name, grid=grid, sizes=sizes)
    mf = MultiGPUFactor(p.blk_size, p.colptr, p.rowidx, nparts, complex_=p.is_complex)
    vals = torch.from_numpy(p.values).cuda()
    rc = mf.factor(vals, p.val_offset)
    assert rc == dd.DD_OK
    B = random_rhs(p.n, 6, p.is_complex, 3)
    X = mf.solve(to_dev_colmajor(B, torch))
    torch.cuda.synchronize()
    X = X.cpu().numpy()
    F = oracle.block_factor(p, list(mf.plan.order))
    Xo, _, _ = oracle.refine_solve(p, F, B, 1)
    berr = residual_berr(p, X, B)
    rd = rel_diff(X, Xo)
    print(f"{name} {grid} nparts={nparts}: top {len(mf.plan.top)} blocks, rel diff {rd:.2e}, berr {berr.max():.2e}")
    assert rd <= 1e-9, rd
    assert berr.max() <= 1e-12, berr.max()
