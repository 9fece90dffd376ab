"""Test helpers: run the CUDA path through the C ABI on a dd_inputs.Problem."""
import numpy as np


def to_dev_colmajor(B, torch):
    B = np.asarray(B)
    return torch.from_numpy(np.ascontiguousarray(B.T)).cuda().t()


def run_gpu(p, B, *, order=None, user_order=None, refine=1, keep=False, perturb_tau=None):
    """Factor + solve on cuda:0. Returns (X, finfo, solver) -- solver only if keep."""
    import torch
    import paper_2002_05019_b200 as dd
    o = dd.DD_ORDER_AUTO if order is None else order
    s = dd.AuxSolver(p.blk_size, p.colptr, p.rowidx, complex_=p.is_complex, order=o, refine_steps=refine,
                     user_order=user_order, perturb_tau=perturb_tau)
    vals = torch.from_numpy(p.values).cuda()
    rc, finfo = s.factor(vals, p.val_offset)
    finfo["rc"] = rc
    X = None
    if B is not None and rc == dd.DD_OK:
        Bd = to_dev_colmajor(B, torch)
        s.solve_(Bd)
        torch.cuda.synchronize()
        X = Bd.cpu().numpy()
    if keep:
        return X, finfo, s
    s.close()
    return X, finfo, None


def rel_diff(X, Xref):
    return float((np.abs(X - Xref).max(axis=0) / np.abs(Xref).max(axis=0)).max())
