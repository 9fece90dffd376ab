"""B200-native auxiliary-matrix solver of arXiv:2002.05019 -- thin Python binding.

The product is the C-ABI library ``libdd_aux.so`` (include/dd_aux.h): hand-written
sm_100a CUDA kernels for the restricted-Bunch-Kaufman block LDL^T of the
block-sparse auxiliary matrix (§II) and its multi-RHS solve.  This
module only marshals arguments to it (same function names as the C ABI); PyTorch
supplies device memory and streams.  There is no CPU fallback: importing this
package on a machine without the built library raises ImportError, and every
compute call needs CUDA device buffers.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

__all__ = ["DD_REAL64", "DD_COMPLEX128", "DD_ORDER_AUTO", "DD_ORDER_ND", "DD_ORDER_MINDEG", "DD_ORDER_NATURAL",
           "DD_ORDER_USER", "DD_OK", "DD_ZERO_PIVOT", "DD_NONFINITE", "DDAuxError", "dd_aux_default_options", "dd_aux_analyze",
           "dd_aux_get_info", "dd_aux_get_order", "dd_aux_get_etree", "dd_aux_solve_work_bytes", "dd_aux_factor",
           "dd_aux_solve", "dd_aux_get_pivots", "dd_aux_destroy", "dd_aux_last_error", "dd_aux_version",
           "dd_aux_set_refine", "dd_aux_set_graphs", "dd_aux_set_trace", "dd_aux_get_trace", "dd_aux_get_level_trace", "dd_aux_assemble_work_bytes", "dd_aux_assemble",
           "dd_aux_last_assemble_bytes", "cliques_to_csr", "AuxSolver", "LIB_PATH", "EXPORTED_SYMBOLS", "PHASES",
           "dd_aux_analyze_partial", "dd_aux_schur_cliques", "dd_aux_schur_export", "dd_aux_condense",
           "dd_aux_recover", "SchurSolver", "dd_aux_get_struct", "dd_aux_assemble_acc", "dd_aux_residual",
           "dd_aux_backward_error"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdd_aux.so")

DD_REAL64, DD_COMPLEX128 = 0, 1
DD_ORDER_AUTO, DD_ORDER_ND, DD_ORDER_MINDEG, DD_ORDER_NATURAL, DD_ORDER_USER = 0, 1, 2, 3, 4
DD_OK, DD_ZERO_PIVOT, DD_NONFINITE = 0, 1, 2
DD_ERR_CUDA, DD_ERR_WORKSPACE, DD_ERR_NOT_FACTORED, DD_ERR_SINGULAR, DD_ERR_PATTERN = -100, -101, -102, -103, -104

EXPORTED_SYMBOLS = ["dd_aux_default_options", "dd_aux_analyze", "dd_aux_get_info", "dd_aux_get_order",
                    "dd_aux_get_etree", "dd_aux_solve_work_bytes", "dd_aux_factor", "dd_aux_solve",
                    "dd_aux_get_pivots", "dd_aux_set_refine", "dd_aux_set_graphs", "dd_aux_set_trace", "dd_aux_get_trace", "dd_aux_get_level_trace", "dd_aux_destroy",
                    "dd_aux_last_error", "dd_aux_version", "dd_aux_assemble_work_bytes", "dd_aux_assemble",
                    "dd_aux_last_assemble_bytes", "dd_aux_analyze_partial", "dd_aux_schur_cliques",
                    "dd_aux_schur_export", "dd_aux_condense", "dd_aux_recover", "dd_aux_get_struct",
                    "dd_aux_assemble_acc", "dd_aux_residual", "dd_aux_backward_error",
                    "dd_aux_validate"]
PHASES = ["load", "k1_diag_bk", "rowperm", "k2_panel", "k3_update", "stats", "perm", "fdiag", "fupd", "dsolve",
          "bupd", "bdiag", "spmv", "linv", "assemble", "schur"]


class DDAuxError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"dd_aux error {code}: {msg}")
        self.code = code


class dd_aux_options(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int32), ("user_order", ctypes.POINTER(ctypes.c_int32)),
                ("refine_steps", ctypes.c_int32), ("use_graphs", ctypes.c_int32), ("refine_tol", ctypes.c_double),
                ("complex_3m", ctypes.c_int32), ("perturb", ctypes.c_int32), ("perturb_tau", ctypes.c_double)]


class dd_aux_info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nblk", ctypes.c_int64), ("nnzb_in", ctypes.c_int64),
                ("nnzb_filled", ctypes.c_int64), ("n_levels", ctypes.c_int64), ("max_front", ctypes.c_int64),
                ("max_level_width", ctypes.c_int64), ("flops_factor", ctypes.c_double),
                ("flops_solve_per_rhs", ctypes.c_double), ("factor_value_bytes", ctypes.c_double),
                ("factor_bytes", ctypes.c_size_t), ("work_bytes", ctypes.c_size_t), ("dtype", ctypes.c_int32),
                ("order_used", ctypes.c_int32), ("n_schur", ctypes.c_int64), ("n_groups", ctypes.c_int64),
                ("n_aux_dof", ctypes.c_int64)]


class dd_aux_factor_info(ctypes.Structure):
    _fields_ = [("npos", ctypes.c_int64), ("nneg", ctypes.c_int64), ("nzero", ctypes.c_int64),
                ("n2x2", ctypes.c_int64), ("nswaps", ctypes.c_int64), ("first_zero_pivot", ctypes.c_int64),
                ("ms_load", ctypes.c_float), ("ms_factor", ctypes.c_float), ("nperturbed", ctypes.c_int64),
                ("nonfinite", ctypes.c_int64), ("max_abs_L", ctypes.c_double)]


class dd_aux_trace(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 16), ("launches", ctypes.c_int64 * 16), ("flops", ctypes.c_double * 16)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python dd_build.py`")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i64, i32 = ctypes.c_int64, ctypes.c_int32
    pi64 = ctypes.POINTER(ctypes.c_int64)
    pi32 = ctypes.POINTER(ctypes.c_int32)
    sig = {
        "dd_aux_default_options": (None, [ctypes.POINTER(dd_aux_options)]),
        "dd_aux_analyze": (ctypes.c_int, [i64, pi64, pi64, pi32, i32, ctypes.POINTER(dd_aux_options), ctypes.POINTER(P)]),
        "dd_aux_get_info": (ctypes.c_int, [P, ctypes.POINTER(dd_aux_info)]),
        "dd_aux_get_order": (ctypes.c_int, [P, pi32]),
        "dd_aux_get_etree": (ctypes.c_int, [P, pi32, pi32, pi64]),
        "dd_aux_solve_work_bytes": (ctypes.c_int, [P, i64, ctypes.POINTER(ctypes.c_size_t)]),
        "dd_aux_factor": (ctypes.c_int, [P, P, pi64, P, P, P, ctypes.POINTER(dd_aux_factor_info)]),
        "dd_aux_solve": (ctypes.c_int, [P, P, P, i64, P, i64, P, P]),
        "dd_aux_get_pivots": (ctypes.c_int, [P, P, pi32, pi32, P, P]),
        "dd_aux_set_refine": (ctypes.c_int, [P, i32, ctypes.c_double]),
        "dd_aux_set_trace": (ctypes.c_int, [P, i32]),
        "dd_aux_set_graphs": (ctypes.c_int, [P, i32]),
        "dd_aux_get_trace": (ctypes.c_int, [P, ctypes.POINTER(dd_aux_trace), i32]),
        "dd_aux_get_level_trace": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
        "dd_aux_assemble_work_bytes": (ctypes.c_int, [P, i64, pi64, pi32, ctypes.POINTER(ctypes.c_size_t)]),
        "dd_aux_assemble": (ctypes.c_int, [P, i64, pi64, pi32, P, pi64, i32, pi64, P, P, P]),
        "dd_aux_last_assemble_bytes": (ctypes.c_double, [P]),
        "dd_aux_analyze_partial": (ctypes.c_int, [i64, pi64, pi64, pi32, i32, ctypes.POINTER(dd_aux_options), i64,
                                                   pi32, pi32, i64, pi64, ctypes.POINTER(P)]),
        "dd_aux_schur_cliques": (ctypes.c_int, [P, pi64, pi64, pi32]),
        "dd_aux_get_struct": (ctypes.c_int, [P, pi64, pi32]),
        "dd_aux_residual": (ctypes.c_int, [P, P, P, i64, P, i64, P, i64, P, i64, P, P]),
        "dd_aux_validate": (ctypes.c_int, [P]),
        "dd_aux_backward_error": (ctypes.c_int, [P, P, P, i64, P, i64, P, i64, P, ctypes.POINTER(ctypes.c_double),
                                                  P]),
        "dd_aux_assemble_acc": (ctypes.c_int, [P, i64, pi64, pi32, P, pi64, i32, pi64, P, P, P]),
        "dd_aux_schur_export": (ctypes.c_int, [P, P, P, pi64, P]),
        "dd_aux_condense": (ctypes.c_int, [P, P, i64, P, i64, P, i64, P, P]),
        "dd_aux_recover": (ctypes.c_int, [P, P, i64, P, i64, P, i64, P, i64, P, P]),
        "dd_aux_destroy": (ctypes.c_int, [P]),
        "dd_aux_last_error": (ctypes.c_char_p, []),
        "dd_aux_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def _np_ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def _check(rc, allow=(DD_OK,)):
    if rc not in allow:
        raise DDAuxError(rc, dd_aux_last_error())
    return rc


def _stream_ptr(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(int(getattr(stream, "cuda_stream", stream)))


def _dev_ptr(t):
    if t is None:
        return None
    if not getattr(t, "is_cuda", False):
        raise ValueError("device buffers must be CUDA tensors (there is no CPU path)")
    return ctypes.c_void_p(t.data_ptr())


def dd_aux_last_error() -> str:
    return _lib.dd_aux_last_error().decode()


def dd_aux_version() -> str:
    return _lib.dd_aux_version().decode()


def dd_aux_default_options(order=DD_ORDER_AUTO, refine_steps=1, user_order=None, refine_tol=None,
                           complex_3m=True, use_graphs=False, perturb_tau=None) -> dd_aux_options:
    o = dd_aux_default_options_raw()
    if perturb_tau is not None:
        o.perturb = 1
        o.perturb_tau = float(perturb_tau)
    o.use_graphs = int(bool(use_graphs))
    o.order = int(order)
    o.complex_3m = int(bool(complex_3m))
    o.refine_steps = int(refine_steps)
    if refine_tol is not None:
        o.refine_tol = float(refine_tol)
    if user_order is not None:
        uo = np.ascontiguousarray(user_order, dtype=np.int32)
        o._user_order_keepalive = uo
        o.user_order = _np_ptr(uo, ctypes.c_int32)
        o.order = DD_ORDER_USER
    return o


def dd_aux_default_options_raw() -> dd_aux_options:
    o = dd_aux_options()
    _lib.dd_aux_default_options(ctypes.byref(o))
    return o


def dd_aux_analyze(blk_size, colptr, rowidx, dtype=DD_REAL64, opt: Optional[dd_aux_options] = None):
    bs = np.ascontiguousarray(blk_size, dtype=np.int64)
    cp = np.ascontiguousarray(colptr, dtype=np.int64)
    ri = np.ascontiguousarray(rowidx, dtype=np.int32)
    h = ctypes.c_void_p()
    rc = _lib.dd_aux_analyze(len(bs), _np_ptr(bs, ctypes.c_int64), _np_ptr(cp, ctypes.c_int64),
                             _np_ptr(ri, ctypes.c_int32), int(dtype), ctypes.byref(opt) if opt is not None else None,
                             ctypes.byref(h))
    _check(rc)
    return h


def dd_aux_get_info(h) -> dict:
    info = dd_aux_info()
    _check(_lib.dd_aux_get_info(h, ctypes.byref(info)))
    return {f: getattr(info, f) for f, _ in dd_aux_info._fields_}


def dd_aux_get_order(h) -> np.ndarray:
    n = dd_aux_get_info(h)["nblk"]
    out = np.empty(n, dtype=np.int32)
    _check(_lib.dd_aux_get_order(h, _np_ptr(out, ctypes.c_int32)))
    return out


def dd_aux_get_etree(h):
    n = dd_aux_get_info(h)["nblk"]
    parent = np.empty(n, dtype=np.int32)
    level = np.empty(n, dtype=np.int32)
    nnz = ctypes.c_int64()
    _check(_lib.dd_aux_get_etree(h, _np_ptr(parent, ctypes.c_int32), _np_ptr(level, ctypes.c_int32),
                                 ctypes.byref(nnz)))
    return parent, level, int(nnz.value)


def dd_aux_get_struct(h):
    """{block id: [struct blocks in elimination order]} as (st_ptr, st_blk) arrays."""
    n = dd_aux_get_info(h)["nblk"]
    ptr = np.empty(n + 1, dtype=np.int64)
    _check(_lib.dd_aux_get_struct(h, _np_ptr(ptr, ctypes.c_int64), None))
    blk = np.empty(max(int(ptr[-1]), 1), dtype=np.int32)
    _check(_lib.dd_aux_get_struct(h, None, _np_ptr(blk, ctypes.c_int32)))
    return ptr, blk[:int(ptr[-1])]


def dd_aux_solve_work_bytes(h, nrhs: int) -> int:
    b = ctypes.c_size_t()
    _check(_lib.dd_aux_solve_work_bytes(h, int(nrhs), ctypes.byref(b)))
    return int(b.value)


def dd_aux_factor(h, d_vals, val_offset, d_factor, d_work, stream=None):
    """Returns (rc, finfo dict); rc is DD_OK, DD_ZERO_PIVOT or DD_NONFINITE, errors raise DDAuxError."""
    vo = np.ascontiguousarray(val_offset, dtype=np.int64)
    fi = dd_aux_factor_info()
    rc = _lib.dd_aux_factor(h, _dev_ptr(d_vals), _np_ptr(vo, ctypes.c_int64), _dev_ptr(d_factor), _dev_ptr(d_work),
                            _stream_ptr(stream), ctypes.byref(fi))
    _check(rc, allow=(DD_OK, DD_ZERO_PIVOT, DD_NONFINITE))
    return rc, {f: getattr(fi, f) for f, _ in dd_aux_factor_info._fields_}


def dd_aux_solve(h, d_factor, d_vals, d_B, d_work, stream=None, nrhs=None, ldb=None):
    """d_B: (n, nrhs) column-major CUDA tensor (stride (1, ldb)); overwritten by X."""
    if nrhs is None:
        nrhs = d_B.shape[1] if d_B.dim() == 2 else 1
    if ldb is None:
        ldb = d_B.stride(1) if d_B.dim() == 2 and d_B.shape[1] > 1 else d_B.shape[0]
        if d_B.dim() == 2 and d_B.shape[1] > 1 and d_B.stride(0) != 1:
            raise ValueError("d_B must be column-major (stride(0) == 1)")
    rc = _lib.dd_aux_solve(h, _dev_ptr(d_factor), _dev_ptr(d_vals), int(nrhs), _dev_ptr(d_B), int(ldb),
                           _dev_ptr(d_work), _stream_ptr(stream))
    return _check(rc)


def dd_aux_get_pivots(h, d_factor, cplx=False) -> dict:
    n = dd_aux_get_info(h)["n"]
    ipiv = np.empty(n, dtype=np.int32)
    perm = np.empty(n, dtype=np.int32)
    dt = np.complex128 if cplx else np.float64
    d = np.empty(n, dtype=dt)
    e = np.empty(n, dtype=dt)
    _check(_lib.dd_aux_get_pivots(h, _dev_ptr(d_factor), _np_ptr(ipiv, ctypes.c_int32), _np_ptr(perm, ctypes.c_int32),
                                  ctypes.c_void_p(d.ctypes.data), ctypes.c_void_p(e.ctypes.data)))
    return dict(ipiv=ipiv, perm=perm, d=d, e=e)


def dd_aux_set_refine(h, refine_steps, refine_tol=0.0):
    _check(_lib.dd_aux_set_refine(h, int(refine_steps), float(refine_tol)))


def dd_aux_set_graphs(h, enable=True):
    _check(_lib.dd_aux_set_graphs(h, int(bool(enable))))


def dd_aux_set_trace(h, enable=True):
    _check(_lib.dd_aux_set_trace(h, int(bool(enable))))


def dd_aux_get_trace(h, reset=True) -> dict:
    """{phase: {"ms", "launches", "flops"}} since the last reset (synchronizes recorded events)."""
    t = dd_aux_trace()
    _check(_lib.dd_aux_get_trace(h, ctypes.byref(t), int(bool(reset))))
    return {name: {"ms": t.ms[i], "launches": int(t.launches[i]), "flops": t.flops[i]} for i, name in enumerate(PHASES)}


def dd_aux_get_level_trace(h) -> dict:
    """Per-level factor trace: {"ms": [n_levels x 16], "flops": [...]} (columns = PHASES)."""
    nl = dd_aux_get_info(h)["n_levels"]
    ms = np.zeros(nl * 16)
    fl = np.zeros(nl * 16)
    _check(_lib.dd_aux_get_level_trace(h, _np_ptr(ms, ctypes.c_double), _np_ptr(fl, ctypes.c_double)))
    return {"ms": ms.reshape(nl, 16)[:, :len(PHASES)], "flops": fl.reshape(nl, 16)[:, :len(PHASES)]}


def cliques_to_csr(cliques):
    """[[block ids], ...] -> (clq_ptr int64[nclq+1], clq_blk int32[...]) (marshalling only)."""
    ptr = np.zeros(len(cliques) + 1, dtype=np.int64)
    for p, members in enumerate(cliques):
        ptr[p + 1] = ptr[p] + len(members)
    blk = np.asarray([int(b) for members in cliques for b in members], dtype=np.int32)
    return ptr, blk


def dd_aux_assemble_work_bytes(h, clq_ptr, clq_blk) -> int:
    cp = np.ascontiguousarray(clq_ptr, dtype=np.int64)
    cb = np.ascontiguousarray(clq_blk, dtype=np.int32)
    b = ctypes.c_size_t()
    _check(_lib.dd_aux_assemble_work_bytes(h, len(cp) - 1, _np_ptr(cp, ctypes.c_int64), _np_ptr(cb, ctypes.c_int32),
                                           ctypes.byref(b)))
    return int(b.value)


def dd_aux_assemble(h, clq_ptr, clq_blk, d_S, S_offset, val_offset, d_vals, d_work, symmetrize=True, stream=None):
    """f1: d_vals <- sum of the cliques' dense contributions (see include/dd_aux.h)."""
    cp = np.ascontiguousarray(clq_ptr, dtype=np.int64)
    cb = np.ascontiguousarray(clq_blk, dtype=np.int32)
    so = np.ascontiguousarray(S_offset, dtype=np.int64)
    vo = np.ascontiguousarray(val_offset, dtype=np.int64)
    rc = _lib.dd_aux_assemble(h, len(cp) - 1, _np_ptr(cp, ctypes.c_int64), _np_ptr(cb, ctypes.c_int32), _dev_ptr(d_S),
                              _np_ptr(so, ctypes.c_int64), int(bool(symmetrize)), _np_ptr(vo, ctypes.c_int64),
                              _dev_ptr(d_vals), _dev_ptr(d_work), _stream_ptr(stream))
    return _check(rc)


def dd_aux_assemble_acc(h, clq_ptr, clq_blk, d_S, S_offset, val_offset, d_vals, d_work, symmetrize=False,
                        stream=None):
    """d_vals += sum of the cliques' contributions (blocks no clique covers are left as they are)."""
    cp = np.ascontiguousarray(clq_ptr, dtype=np.int64)
    cb = np.ascontiguousarray(clq_blk, dtype=np.int32)
    so = np.ascontiguousarray(S_offset, dtype=np.int64)
    vo = np.ascontiguousarray(val_offset, dtype=np.int64)
    rc = _lib.dd_aux_assemble_acc(h, len(cp) - 1, _np_ptr(cp, ctypes.c_int64), _np_ptr(cb, ctypes.c_int32),
                                  _dev_ptr(d_S), _np_ptr(so, ctypes.c_int64), int(bool(symmetrize)),
                                  _np_ptr(vo, ctypes.c_int64), _dev_ptr(d_vals), _dev_ptr(d_work),
                                  _stream_ptr(stream))
    return _check(rc)


def dd_aux_last_assemble_bytes(h) -> float:
    return float(_lib.dd_aux_last_assemble_bytes(h))


def dd_aux_analyze_partial(blk_size, colptr, rowidx, schur_target, schur_group, aux_blk_size, dtype=DD_REAL64,
                           opt: Optional[dd_aux_options] = None):
    """f3: Schur-mode handle; the last len(schur_target) block ids are kept (include/dd_aux.h)."""
    bs = np.ascontiguousarray(blk_size, dtype=np.int64)
    cp = np.ascontiguousarray(colptr, dtype=np.int64)
    ri = np.ascontiguousarray(rowidx, dtype=np.int32)
    st = np.ascontiguousarray(schur_target, dtype=np.int32)
    sg = np.ascontiguousarray(schur_group, dtype=np.int32)
    ab = np.ascontiguousarray(aux_blk_size, dtype=np.int64)
    h = ctypes.c_void_p()
    rc = _lib.dd_aux_analyze_partial(len(bs), _np_ptr(bs, ctypes.c_int64), _np_ptr(cp, ctypes.c_int64),
                                     _np_ptr(ri, ctypes.c_int32), int(dtype),
                                     ctypes.byref(opt) if opt is not None else None, len(st),
                                     _np_ptr(st, ctypes.c_int32), _np_ptr(sg, ctypes.c_int32), len(ab),
                                     _np_ptr(ab, ctypes.c_int64), ctypes.byref(h))
    _check(rc)
    return h


def dd_aux_schur_cliques(h):
    """[[auxiliary block ids of group g, ascending], ...] (the cliques of the exported S_g)."""
    ng = ctypes.c_int64()
    _check(_lib.dd_aux_schur_cliques(h, ctypes.byref(ng), None, None))
    ptr = np.empty(ng.value + 1, dtype=np.int64)
    ns = dd_aux_get_info(h)["n_schur"]
    blk = np.empty(ns, dtype=np.int32)
    _check(_lib.dd_aux_schur_cliques(h, None, _np_ptr(ptr, ctypes.c_int64), _np_ptr(blk, ctypes.c_int32)))
    return [blk[ptr[g]:ptr[g + 1]].tolist() for g in range(ng.value)]


def dd_aux_schur_export(h, d_factor, d_S, S_offset, stream=None):
    so = np.ascontiguousarray(S_offset, dtype=np.int64)
    _check(_lib.dd_aux_schur_export(h, _dev_ptr(d_factor), _dev_ptr(d_S), _np_ptr(so, ctypes.c_int64),
                                    _stream_ptr(stream)))
    return so


def _cm(t):
    """(rows, cols, ld) of a column-major 2-D CUDA tensor (stride (1, ld))."""
    if t.dim() == 1:
        return t.shape[0], 1, t.shape[0]
    if t.shape[1] > 1 and t.stride(0) != 1:
        raise ValueError("buffers must be column-major (stride(0) == 1)")
    return t.shape[0], t.shape[1], (t.stride(1) if t.shape[1] > 1 else t.shape[0])


def dd_aux_condense(h, d_factor, d_F, d_G, d_work, stream=None):
    """G <- G - sum_p R_p^T C_p^T K_p^-1 f_p (column-major CUDA tensors)."""
    _, nrhs, ldf = _cm(d_F)
    _, _, ldg = _cm(d_G)
    _check(_lib.dd_aux_condense(h, _dev_ptr(d_factor), int(nrhs), _dev_ptr(d_F), int(ldf), _dev_ptr(d_G), int(ldg),
                                _dev_ptr(d_work), _stream_ptr(stream)))


def dd_aux_recover(h, d_factor, d_F, d_Xb, d_X, d_work, stream=None):
    """X <- primal K_p^-1 (f_p - C_p R_p x_b) (kept rows: x_b copies)."""
    _, nrhs, ldf = _cm(d_F)
    _, _, ldxb = _cm(d_Xb)
    _, _, ldx = _cm(d_X)
    _check(_lib.dd_aux_recover(h, _dev_ptr(d_factor), int(nrhs), _dev_ptr(d_F), int(ldf), _dev_ptr(d_Xb), int(ldxb),
                               _dev_ptr(d_X), int(ldx), _dev_ptr(d_work), _stream_ptr(stream)))


def dd_aux_residual(h, d_factor, d_vals, d_B, d_X, d_R, d_work, stream=None):
    """R = B - A X over the handle's original blocks (column-major CUDA tensors)."""
    _, nrhs, ldb = _cm(d_B)
    _, _, ldx = _cm(d_X)
    _, _, ldr = _cm(d_R)
    _check(_lib.dd_aux_residual(h, _dev_ptr(d_factor), _dev_ptr(d_vals), int(nrhs), _dev_ptr(d_B), int(ldb),
                                _dev_ptr(d_X), int(ldx), _dev_ptr(d_R), int(ldr), _dev_ptr(d_work),
                                _stream_ptr(stream)))


def dd_aux_backward_error(h, d_factor, d_vals, d_B, d_X, d_work, stream=None) -> np.ndarray:
    """Per-column ||b - A x||_inf / (||A||_inf ||x||_inf) computed on the device (synchronizes)."""
    _, nrhs, ldb = _cm(d_B)
    _, _, ldx = _cm(d_X)
    out = np.empty(nrhs, dtype=np.float64)
    _check(_lib.dd_aux_backward_error(h, _dev_ptr(d_factor), _dev_ptr(d_vals), int(nrhs), _dev_ptr(d_B), int(ldb),
                                      _dev_ptr(d_X), int(ldx), _dev_ptr(d_work), _np_ptr(out, ctypes.c_double),
                                      _stream_ptr(stream)))
    return out


def dd_aux_validate(h):
    """Host-side bounds check of every descriptor table (raises DDAuxError naming the rule)."""
    _check(_lib.dd_aux_validate(h))


def dd_aux_destroy(h):
    if h:
        _lib.dd_aux_destroy(h)


class AuxSolver:
    """Convenience owner of one handle plus its torch-allocated device buffers.

    Marshalling only: analyze -> allocate factor/work with torch -> dd_aux_factor ->
    dd_aux_solve.  Buffers are uint8 CUDA tensors sized by dd_aux_get_info.
    """

    def __init__(self, blk_size, colptr, rowidx, complex_=False, order=DD_ORDER_AUTO, refine_steps=1,
                 user_order=None, device="cuda", refine_tol=None, complex_3m=True, use_graphs=False,
                 perturb_tau=None):
        import torch
        self.torch = torch
        self.cplx = bool(complex_)
        self.opt = dd_aux_default_options(order, refine_steps, user_order, refine_tol, complex_3m, use_graphs,
                                          perturb_tau)
        self.h = dd_aux_analyze(blk_size, colptr, rowidx, DD_COMPLEX128 if self.cplx else DD_REAL64, self.opt)
        self._bs = np.asarray(blk_size, dtype=np.int64)
        self._rows = np.asarray(rowidx, dtype=np.int64)
        self._col = np.repeat(np.arange(len(self._bs)), np.diff(np.asarray(colptr, dtype=np.int64)))
        self.info = dd_aux_get_info(self.h)
        self.device = device
        self.factor_buf = None
        self.work = None
        self.vals = None
        self.finfo = None

    @property
    def n(self):
        return self.info["n"]

    def order(self):
        return dd_aux_get_order(self.h)

    def _work(self, nbytes):
        if self.work is None or self.work.numel() < nbytes:
            self.work = self.torch.empty(max(nbytes, 256), dtype=self.torch.uint8, device=self.device)
        return self.work

    def factor(self, d_vals, val_offset, stream=None):
        torch = self.torch
        if self.factor_buf is None:
            self.factor_buf = torch.empty(self.info["factor_bytes"], dtype=torch.uint8, device=self.device)
        w = self._work(self.info["work_bytes"])
        self.vals = d_vals
        rc, self.finfo = dd_aux_factor(self.h, d_vals, val_offset, self.factor_buf, w, stream)
        return rc, self.finfo

    def solve_(self, d_B, stream=None):
        """In-place solve of a column-major (n, nrhs) CUDA tensor."""
        nrhs = d_B.shape[1] if d_B.dim() == 2 else 1
        w = self._work(dd_aux_solve_work_bytes(self.h, nrhs))
        dd_aux_solve(self.h, self.factor_buf, self.vals, d_B, w, stream)
        return d_B

    def assemble(self, cliques, d_S, S_offset, val_offset, d_vals=None, symmetrize=True, stream=None):
        """f1: assemble the auxiliary matrix on the device from per-clique dense contributions.

        cliques: list of ascending block-id lists; d_S: CUDA tensor holding every S_p (column-major,
        ld = m_p) at element offsets S_offset; returns d_vals (allocated if None) in the layout
        val_offset describes."""
        torch = self.torch
        ptr, blk = cliques_to_csr(cliques)
        if d_vals is None:
            nvals = int(max((int(val_offset[q]) + int(self._bs[self._rows[q]]) * int(self._bs[self._col[q]])
                             for q in range(len(val_offset))), default=0))
            d_vals = torch.empty(nvals, dtype=torch.complex128 if self.cplx else torch.float64, device=self.device)
        w = torch.empty(max(256, dd_aux_assemble_work_bytes(self.h, ptr, blk)), dtype=torch.uint8, device=self.device)
        dd_aux_assemble(self.h, ptr, blk, d_S, S_offset, val_offset, d_vals, w, symmetrize, stream)
        self._asm_work = w  # kept alive until the next assembly (the launch is asynchronous)
        return d_vals

    def pivots(self):
        return dd_aux_get_pivots(self.h, self.factor_buf, self.cplx)

    def close(self):
        if self.h:
            dd_aux_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SchurSolver(AuxSolver):
    """Owner of a Schur-mode (partial factorization) handle: f3 subdomain elimination + f2 primal
    recovery.  Marshalling only (see include/dd_aux.h dd_aux_analyze_partial)."""

    def __init__(self, blk_size, colptr, rowidx, schur_target, schur_group, aux_blk_size, complex_=False,
                 order=DD_ORDER_NATURAL, user_order=None, device="cuda", complex_3m=True):
        import torch
        self.torch = torch
        self.cplx = bool(complex_)
        self.opt = dd_aux_default_options(order, 0, user_order, None, complex_3m, False, None)
        self.h = dd_aux_analyze_partial(blk_size, colptr, rowidx, schur_target, schur_group, aux_blk_size,
                                        DD_COMPLEX128 if self.cplx else DD_REAL64, self.opt)
        self._bs = np.asarray(blk_size, dtype=np.int64)
        self._rows = np.asarray(rowidx, dtype=np.int64)
        self._col = np.repeat(np.arange(len(self._bs)), np.diff(np.asarray(colptr, dtype=np.int64)))
        self.info = dd_aux_get_info(self.h)
        self.device = device
        self.factor_buf = None
        self.work = None
        self.vals = None
        self.finfo = None

    def cliques(self):
        return dd_aux_schur_cliques(self.h)

    def export(self, d_S=None, S_offset=None, stream=None):
        """Dense S_g of every group into one buffer (allocated if None); returns (d_S, S_offset)."""
        torch = self.torch
        cl = self.cliques()
        ms = [int(sum(self._aux_size(I) for I in c)) for c in cl]
        if S_offset is None:
            S_offset = np.concatenate([[0], np.cumsum([m * m for m in ms])[:-1]]).astype(np.int64)
        if d_S is None:
            d_S = torch.empty(int(S_offset[-1] + ms[-1] * ms[-1]),
                              dtype=torch.complex128 if self.cplx else torch.float64, device=self.device)
        dd_aux_schur_export(self.h, self.factor_buf, d_S, S_offset, stream)
        return d_S, S_offset

    def _aux_size(self, I):
        if not hasattr(self, "_auxs"):
            raise RuntimeError("set .aux_sizes")
        return self._auxs[I]

    def condense_(self, d_F, d_G, stream=None):
        w = self._work(dd_aux_solve_work_bytes(self.h, d_F.shape[1] if d_F.dim() == 2 else 1))
        dd_aux_condense(self.h, self.factor_buf, d_F, d_G, w, stream)
        return d_G

    def recover(self, d_F, d_Xb, d_X=None, stream=None):
        if d_X is None:
            d_X = self.torch.empty_like(d_F.t().contiguous()).t() if d_F.dim() == 2 else self.torch.empty_like(d_F)
        w = self._work(dd_aux_solve_work_bytes(self.h, d_F.shape[1] if d_F.dim() == 2 else 1))
        dd_aux_recover(self.h, self.factor_buf, d_F, d_Xb, d_X, w, stream)
        return d_X
