"""B200-native (sm_100a) FP64 tensor-train hot path of arXiv 2509.11890.

Thin ctypes binding of the C-ABI declared in include/tt_hotpath.h: argument marshalling
only — every step of the path runs in the CUDA kernels of libtt_hotpath.so.  PyTorch is
used for device memory and streams.  There is NO CPU fallback: importing this package
without the built library raises, and every call checks that its tensors are CUDA float64.

Function names are the C names.  Tensor shapes (C-contiguous, float64, on one CUDA device):
  phiL (rl,Rl,rl)  A (Rl,n,n,Rr)  phiR (rr,Rr,rr)  x,y (rl,n,rr)  X,Y (rl,n,nvec,rr)
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import torch

__all__ = [
    "TTError", "lib", "LIB_PATH",
    "tt_local_matvec_workspace_size", "tt_local_matvec", "tt_local_matvec_batched",
    "tt_interface_workspace_size", "tt_interface_left", "tt_interface_right",
    "tt_sweep_workspace_size", "tt_sweep_interfaces", "tt_sweep_als_workspace_size",
    "tt_sweep_als", "tt_operator_apply", "tt_last_launch_count",
    "TT_SWEEP_LEFT", "TT_SWEEP_RIGHT", "TT_SWEEP_BOTH", "tt_trace_enable", "tt_trace_disable",
    "tt_trace_count", "tt_trace_read", "tt_fp64_peak_probe", "STAGE_NAMES", "tt_debug_force_v1",
    "tt_debug_set_variant", "tt_debug_set_flags", "tt_debug_set_dag", "tt_debug_set_fused", "tt_debug_dag_trace", "tt_set_graph_cache", "tt_set_matvec_mode", "prepare",
    "PreparedCall",
    "tt_local_gmres",
    "tt_local_gmres_workspace_size",
    "tt_local_matvec_two_site", "tt_local_matvec_two_site_workspace_size",
    "tt_block_local_matvec", "tt_block_local_matvec_workspace_size", "TTBlockTerm",
    "tt_round", "tt_round_async", "tt_compact", "tt_round_workspace_size", "tt_debug_sym_eigen", "tt_debug_svd",
    "tt_local_lobpcg", "tt_local_lobpcg_workspace_size", "tt_merge_operator_cores",
    "tt_orthonormalise", "tt_orthonormalise_workspace_size", "tt_block_move_right",
    "tt_block_move_left", "tt_block_move_right_async", "tt_block_move_left_async", "tt_block_move_workspace_size", "tt_pg_workspace_size",
    "tt_local_matvec_pg", "tt_interface_left_pg", "tt_interface_right_pg", "tt_enrich_right",
    "tt_enrich_right_async",
    "tt_enrich_right_workspace_size", "tt_sweep_w34", "tt_sweep_w34_workspace_size",
]

STAGE_NAMES = {0: "perm", 1: "set", 2: "mv_s1", 3: "mv_s2", 4: "mv_s3", 5: "il_s1", 6: "il_s2",
               7: "il_s3", 8: "ir_s1", 9: "ir_s2", 10: "ir_s3", 11: "apply"}

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtt_hotpath.so")
TT_SWEEP_LEFT, TT_SWEEP_RIGHT, TT_SWEEP_BOTH = 1, 2, 3

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

_i64, _p, _sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
lib = ctypes.CDLL(LIB_PATH)
lib.tt_status_string.restype = ctypes.c_char_p
lib.tt_status_string.argtypes = [ctypes.c_int]
lib.tt_last_error_message.restype = ctypes.c_char_p
lib.tt_version.restype = ctypes.c_char_p
lib.tt_last_launch_count.restype = ctypes.c_int64
lib.tt_local_matvec_workspace_size.restype = _sz
lib.tt_local_matvec_workspace_size.argtypes = [_i64] * 6
lib.tt_local_matvec.argtypes = [_i64] * 5 + [_p] * 6 + [_sz, _p]
lib.tt_local_matvec_batched.argtypes = [_i64] * 6 + [_p] * 6 + [_sz, _p]
lib.tt_interface_workspace_size.restype = _sz
lib.tt_interface_workspace_size.argtypes = [_i64] * 5
lib.tt_interface_left.argtypes = [_i64] * 5 + [_p] * 5 + [_sz, _p]
lib.tt_interface_right.argtypes = [_i64] * 5 + [_p] * 5 + [_sz, _p]
lib.tt_sweep_workspace_size.restype = _sz
lib.tt_sweep_workspace_size.argtypes = [_i64, _p, _p, _p]
lib.tt_sweep_interfaces.argtypes = [_i64, _p, _p, _p, _p, _p, _p, _p, ctypes.c_int, _p, _sz, _p]
lib.tt_sweep_als_workspace_size.restype = _sz
lib.tt_sweep_als_workspace_size.argtypes = [_i64, _p, _p, _p, _i64]
lib.tt_sweep_als.argtypes = [_i64, _p, _p, _p, _i64] + [_p] * 7 + [_p, _sz, _p]
lib.tt_operator_apply.argtypes = [_i64, _p, _p, _p, _p, _p, _p, _p, _p]
lib.tt_trace_enable.argtypes = [_i64]
lib.tt_trace_count.restype = ctypes.c_int64
lib.tt_trace_read.argtypes = [_i64] + [_p] * 6
lib.tt_fp64_peak_probe.argtypes = [_i64, _p, _p]
class TTBlockTerm(ctypes.Structure):
    """tt_block_term: Y[row] += coeff * L_op(L_op2(X[col])) (op2 = -1: single operator)."""
    _fields_ = [("row", ctypes.c_int64), ("col", ctypes.c_int64), ("op", ctypes.c_int64),
                ("op2", ctypes.c_int64), ("coeff", ctypes.c_double)]


lib.tt_round_workspace_size.restype = _sz
lib.tt_round_workspace_size.argtypes = [_i64, _p, _p]
lib.tt_round.argtypes = [_i64, _p, _p, _p, ctypes.c_double, _i64, _p, _p, _p, _sz, _p]
lib.tt_round.restype = ctypes.c_int
lib.tt_round_async.argtypes = [_i64, _p, _p, _p, ctypes.c_double, _i64, _p, _p, _p, _p, _sz, _p]
lib.tt_round_async.restype = ctypes.c_int
lib.tt_debug_sym_eigen.argtypes = [_i64, _p, _p, _p, _p, _sz, _p]
lib.tt_debug_sym_eigen.restype = ctypes.c_int
lib.tt_debug_svd.argtypes = [_i64, _i64, _p, _p, _p, _p, _p, _p]
lib.tt_debug_svd.restype = ctypes.c_int
lib.tt_block_local_matvec_workspace_size.restype = _sz
lib.tt_block_local_matvec_workspace_size.argtypes = [_i64] * 4 + [_p, _p]
lib.tt_block_local_matvec.argtypes = [_i64] * 5 + [_p] * 5 + [_i64, _p, _p, _p, _p, _sz, _p]
lib.tt_block_local_matvec.restype = ctypes.c_int
lib.tt_local_matvec_two_site_workspace_size.restype = _sz
lib.tt_local_matvec_two_site_workspace_size.argtypes = [_i64] * 8
lib.tt_local_matvec_two_site.argtypes = [_i64] * 8 + [_p] * 7 + [_sz, _p]
lib.tt_local_matvec_two_site.restype = ctypes.c_int
lib.tt_local_gmres_workspace_size.restype = _sz
lib.tt_local_gmres_workspace_size.argtypes = [_i64] * 8
lib.tt_local_gmres.argtypes = [_i64] * 9 + [ctypes.c_double] + [_p] * 8 + [_sz, _p]
lib.tt_local_gmres.restype = ctypes.c_int
lib.tt_local_lobpcg_workspace_size.restype = _sz
lib.tt_local_lobpcg_workspace_size.argtypes = [_i64] * 8
lib.tt_local_lobpcg.argtypes = [_i64] * 10 + [ctypes.c_double] + [_p] * 12 + [_sz, _p]
lib.tt_local_lobpcg.restype = ctypes.c_int
lib.tt_merge_operator_cores.argtypes = [_i64] * 5 + [_p] * 4
lib.tt_orthonormalise_workspace_size.restype = _sz
lib.tt_orthonormalise_workspace_size.argtypes = [_i64, _p, _p]
lib.tt_orthonormalise.argtypes = [_i64, _p, _p, _p, ctypes.c_int, _p, _p, _p, _sz, _p]
lib.tt_orthonormalise.restype = ctypes.c_int
lib.tt_block_move_workspace_size.restype = _sz
lib.tt_block_move_workspace_size.argtypes = [_i64] * 6
lib.tt_block_move_right.argtypes = [_i64] * 6 + [ctypes.c_double, _i64] + [_p] * 6 + [_sz, _p]
lib.tt_block_move_right.restype = ctypes.c_int
lib.tt_block_move_left.argtypes = [_i64] * 6 + [ctypes.c_double, _i64] + [_p] * 6 + [_sz, _p]
lib.tt_block_move_left.restype = ctypes.c_int
lib.tt_block_move_right_async.argtypes = [_i64] * 6 + [ctypes.c_double, _i64] + [_p] * 7 + [_sz, _p]
lib.tt_block_move_right_async.restype = ctypes.c_int
lib.tt_block_move_left_async.argtypes = [_i64] * 6 + [ctypes.c_double, _i64] + [_p] * 7 + [_sz, _p]
lib.tt_block_move_left_async.restype = ctypes.c_int
lib.tt_sweep_w34_workspace_size.restype = _sz
lib.tt_sweep_w34_workspace_size.argtypes = [_i64, _p, _p, _p]
lib.tt_sweep_w34.argtypes = [_i64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p]
lib.tt_sweep_w34.restype = ctypes.c_int
lib.tt_pg_workspace_size.restype = _sz
lib.tt_pg_workspace_size.argtypes = [_i64] * 8
lib.tt_local_matvec_pg.argtypes = [_i64] * 8 + [_p] * 6 + [_sz, _p]
lib.tt_local_matvec_pg.restype = ctypes.c_int
lib.tt_interface_left_pg.argtypes = [_i64] * 7 + [_p] * 6 + [_sz, _p]
lib.tt_interface_left_pg.restype = ctypes.c_int
lib.tt_interface_right_pg.argtypes = [_i64] * 7 + [_p] * 6 + [_sz, _p]
lib.tt_interface_right_pg.restype = ctypes.c_int
lib.tt_enrich_right_workspace_size.restype = _sz
lib.tt_enrich_right_workspace_size.argtypes = [_i64] * 6
lib.tt_enrich_right.argtypes = [_i64] * 6 + [ctypes.c_double, _i64] + [_p] * 7 + [_sz, _p]
lib.tt_enrich_right.restype = ctypes.c_int
lib.tt_enrich_right_async.argtypes = [_i64] * 6 + [ctypes.c_double, _i64] + [_p] * 8 + [_sz, _p]
lib.tt_enrich_right_async.restype = ctypes.c_int
lib.tt_merge_operator_cores.restype = ctypes.c_int
lib.tt_debug_force_v1.argtypes = [ctypes.c_int]
lib.tt_debug_force_v1.restype = None
lib.tt_debug_set_variant.argtypes = [ctypes.c_int]
lib.tt_debug_set_variant.restype = None
lib.tt_debug_set_flags.argtypes = [ctypes.c_int]
lib.tt_debug_set_flags.restype = None
lib.tt_debug_set_dag.argtypes = [ctypes.c_int]
lib.tt_debug_set_dag.restype = None
lib.tt_set_matvec_mode.argtypes = [ctypes.c_int]
lib.tt_set_matvec_mode.restype = ctypes.c_int
lib.tt_debug_set_fused.argtypes = [ctypes.c_int]
lib.tt_debug_set_fused.restype = None
lib.tt_set_graph_cache.argtypes = [ctypes.c_int]
lib.tt_set_graph_cache.restype = None
lib.tt_debug_dag_trace.argtypes = [_p, _i64, _p, _i64]
lib.tt_debug_dag_trace.restype = ctypes.c_int64
for _f in ("tt_trace_enable", "tt_trace_disable", "tt_trace_read", "tt_fp64_peak_probe"):
    getattr(lib, _f).restype = ctypes.c_int
for _f in ("tt_local_matvec", "tt_local_matvec_batched", "tt_interface_left",
           "tt_interface_right", "tt_sweep_interfaces", "tt_sweep_als", "tt_operator_apply"):
    getattr(lib, _f).restype = ctypes.c_int


class TTError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{lib.tt_status_string(status).decode()}: {msg}")


def _check(st: int) -> None:
    if st != 0:
        raise TTError(st, lib.tt_last_error_message().decode())


def _dev(t: torch.Tensor, name: str) -> int:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda or t.dtype != torch.float64:
        raise TypeError(f"{name} must be a CUDA float64 tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be C-contiguous")
    return t.data_ptr()


def _expect(t: torch.Tensor, shape, name: str) -> None:
    """Shape check before any pointer reaches the library: the C-ABI takes its extents from
    the x / A arguments, so a wrongly shaped phi / output would be read or written out of
    bounds."""
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if tuple(t.shape) != tuple(int(v) for v in shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(int(v) for v in shape)}")


def _same_device(*ts) -> None:
    """All tensors of one call must live on one CUDA device."""
    devs = {t.device for t in ts if isinstance(t, torch.Tensor)}
    if len(devs) > 1 and any(dv.type != "cuda" for dv in devs):
        raise TypeError("every tensor must be a CUDA float64 tensor (no CPU fallback)")
    if len(devs) > 1:
        raise ValueError(f"tensors of one call are on different devices: {sorted(map(str, devs))}")


def _check_local(phiL, A, phiR, rl, n, rr, nbra_l=None, nbra_r=None) -> None:
    """phiL (rl_bra,Rl,rl), A (Rl,n,n,Rr), phiR (rr_bra,Rr,rr) against the core's (rl, n, rr)."""
    if A.dim() != 4:
        raise ValueError(f"A must be 4-D (Rl, n, n, Rr), got shape {tuple(A.shape)}")
    Rl, Rr = A.shape[0], A.shape[3]
    _expect(A, (Rl, n, n, Rr), "A")
    _expect(phiL, (rl if nbra_l is None else nbra_l, Rl, rl), "phiL")
    _expect(phiR, (rr if nbra_r is None else nbra_r, Rr, rr), "phiR")


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ws(nbytes: int, workspace: Optional[torch.Tensor], device) -> torch.Tensor:
    if workspace is not None:
        return workspace
    ws = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)
    if _RECORD is not None:   # prepare(): the recorded call keeps its workspace alive
        _RECORD_KEEP.append(ws)
    return ws



# ---- prepared calls ------------------------------------------------------------------------
# prepare(fn, ...) runs a hot-path call once and returns a PreparedCall that re-issues the same
# C-ABI call (same device buffers, same marshalled pointer / extent arrays) on a given stream
# with no per-call Python validation or marshalling: the eager-call overhead of an iterative
# solver's repeated sweeps drops to one ctypes call (and the library's graph cache then replays
# the call as one CUDA graph launch).  The PreparedCall keeps every tensor and array alive.
_RECORD: Optional[list] = None
_RECORD_KEEP: list = []


def _invoke(fn, *args) -> None:
    if _RECORD is not None:
        _RECORD.append((fn, args))
    _check(fn(*args))


class PreparedCall:
    """A recorded C-ABI call: ``p()`` / ``p(stream)`` re-issues it; ``p.result`` holds the
    outputs the first call returned (the buffers every re-issue writes)."""

    def __init__(self, fn, args, keep, result):
        self._fn, self._args, self._keep, self.result = fn, args[:-1], keep, result

    def __call__(self, stream=None):
        _check(self._fn(*self._args, _stream(stream)))
        return self.result


def prepare(fn, *args, **kwargs) -> PreparedCall:
    """prepare(tt_sweep_w34, x, A, ...) etc.: validate and marshal once (see PreparedCall).
    fn: tt_local_matvec, tt_local_matvec_batched, tt_interface_left / _right,
    tt_sweep_interfaces, tt_sweep_w34, tt_sweep_als, tt_operator_apply."""
    global _RECORD
    rec: list = []
    _RECORD = rec
    _RECORD_KEEP.clear()
    try:
        result = fn(*args, **kwargs)
        keep = list(_RECORD_KEEP)
    finally:
        _RECORD = None
        _RECORD_KEEP.clear()
    if len(rec) != 1:
        raise ValueError(f"{getattr(fn, '__name__', fn)} is not a single-call hot-path function")
    lfn, largs = rec[0]
    return PreparedCall(lfn, largs, (args, kwargs, largs, keep), result)


def tt_last_launch_count() -> int:
    return int(lib.tt_last_launch_count())


def tt_local_matvec_workspace_size(rl, n, rr, Rl, Rr, nvec=1) -> int:
    return int(lib.tt_local_matvec_workspace_size(rl, n, rr, Rl, Rr, nvec))


def tt_interface_workspace_size(rl, n, rr, Rl, Rr) -> int:
    return int(lib.tt_interface_workspace_size(rl, n, rr, Rl, Rr))


def tt_local_matvec(phiL, A, phiR, x, y=None, workspace=None, stream=None):
    """H1-H3: y = local matvec of core x.  Returns y."""
    if x.dim() != 3:
        raise ValueError(f"x must be (rl, n, rr), got shape {tuple(x.shape)}")
    rl, n, rr = x.shape
    _check_local(phiL, A, phiR, rl, n, rr)
    Rl, Rr = A.shape[0], A.shape[3]
    if y is None:
        y = torch.empty_like(x)
    _expect(y, x.shape, "y")
    _same_device(phiL, A, phiR, x, y, workspace)
    ws = _ws(tt_local_matvec_workspace_size(rl, n, rr, Rl, Rr, 1), workspace, x.device)
    _invoke(lib.tt_local_matvec, rl, n, rr, Rl, Rr, _dev(phiL, "phiL"), _dev(A, "A"),
            _dev(phiR, "phiR"), _dev(x, "x"), _dev(y, "y"), ws.data_ptr(), ws.numel(),
            _stream(stream))
    return y


def tt_local_matvec_batched(phiL, A, phiR, X, Y=None, workspace=None, stream=None):
    """H4: the local matvec on every column of a Block-TT core X (rl,n,nvec,rr)."""
    if X.dim() != 4:
        raise ValueError(f"X must be (rl, n, nvec, rr), got shape {tuple(X.shape)}")
    rl, n, nvec, rr = X.shape
    _check_local(phiL, A, phiR, rl, n, rr)
    Rl, Rr = A.shape[0], A.shape[3]
    if Y is None:
        Y = torch.empty_like(X)
    _expect(Y, X.shape, "Y")
    _same_device(phiL, A, phiR, X, Y, workspace)
    ws = _ws(tt_local_matvec_workspace_size(rl, n, rr, Rl, Rr, nvec), workspace, X.device)
    _invoke(lib.tt_local_matvec_batched, rl, n, rr, Rl, Rr, nvec, _dev(phiL, "phiL"), _dev(A, "A"),
                                       _dev(phiR, "phiR"), _dev(X, "X"), _dev(Y, "Y"),
                                       ws.data_ptr(), ws.numel(), _stream(stream))
    return Y


def tt_interface_left(phiL_prev, A, x, out=None, workspace=None, stream=None):
    """H5: phiL_next (rr,Rr,rr) from phiL_prev (rl,Rl,rl), A_k, x_k."""
    if x.dim() != 3 or A.dim() != 4:
        raise ValueError("x must be (rl, n, rr) and A (Rl, n, n, Rr)")
    rl, n, rr = x.shape
    Rl, Rr = A.shape[0], A.shape[3]
    _expect(A, (Rl, n, n, Rr), "A")
    _expect(phiL_prev, (rl, Rl, rl), "phiL_prev")
    if out is None:
        out = torch.empty((rr, Rr, rr), dtype=x.dtype, device=x.device)
    _expect(out, (rr, Rr, rr), "phiL_next")
    _same_device(phiL_prev, A, x, out, workspace)
    ws = _ws(tt_interface_workspace_size(rl, n, rr, Rl, Rr), workspace, x.device)
    _invoke(lib.tt_interface_left, rl, n, rr, Rl, Rr, _dev(phiL_prev, "phiL_prev"), _dev(A, "A"),
                                 _dev(x, "x"), _dev(out, "phiL_next"), ws.data_ptr(), ws.numel(),
                                 _stream(stream))
    return out


def tt_interface_right(phiR_next, A, x, out=None, workspace=None, stream=None):
    """H6: phiR_prev (rl,Rl,rl) from phiR_next (rr,Rr,rr), A_k, x_k."""
    if x.dim() != 3 or A.dim() != 4:
        raise ValueError("x must be (rl, n, rr) and A (Rl, n, n, Rr)")
    rl, n, rr = x.shape
    Rl, Rr = A.shape[0], A.shape[3]
    _expect(A, (Rl, n, n, Rr), "A")
    _expect(phiR_next, (rr, Rr, rr), "phiR_next")
    if out is None:
        out = torch.empty((rl, Rl, rl), dtype=x.dtype, device=x.device)
    _expect(out, (rl, Rl, rl), "phiR_prev")
    _same_device(phiR_next, A, x, out, workspace)
    ws = _ws(tt_interface_workspace_size(rl, n, rr, Rl, Rr), workspace, x.device)
    _invoke(lib.tt_interface_right, rl, n, rr, Rl, Rr, _dev(phiR_next, "phiR_next"), _dev(A, "A"),
                                  _dev(x, "x"), _dev(out, "phiR_prev"), ws.data_ptr(), ws.numel(),
                                  _stream(stream))
    return out


class _Train:
    """Host-side shape and pointer arrays of a TT train (marshalling only)."""

    def __init__(self, x_cores: Sequence[torch.Tensor], A_cores: Sequence[torch.Tensor]):
        self.d = len(x_cores)
        if len(A_cores) != self.d or self.d == 0:
            raise ValueError("x_cores and A_cores must be non-empty and of the same length")
        for k in range(self.d):
            if x_cores[k].dim() != 3 or A_cores[k].dim() != 4:
                raise ValueError(f"core {k}: x must be (r, n, r') and A (R, n, n, R')")
            n = x_cores[k].shape[1]
            if A_cores[k].shape[1] != n or A_cores[k].shape[2] != n:
                raise ValueError(f"core {k}: A mode sizes {tuple(A_cores[k].shape[1:3])} do not "
                                 f"match the vector mode size {n}")
            if k + 1 < self.d:
                if x_cores[k].shape[2] != x_cores[k + 1].shape[0]:
                    raise ValueError(f"vector bond {k + 1}: core {k} has {x_cores[k].shape[2]}, "
                                     f"core {k + 1} has {x_cores[k + 1].shape[0]}")
                if A_cores[k].shape[3] != A_cores[k + 1].shape[0]:
                    raise ValueError(f"operator bond {k + 1}: core {k} has {A_cores[k].shape[3]}, "
                                     f"core {k + 1} has {A_cores[k + 1].shape[0]}")
        _same_device(*x_cores, *A_cores)
        self.n = [int(c.shape[1]) for c in x_cores]
        self.r = [int(c.shape[0]) for c in x_cores] + [int(x_cores[-1].shape[-1])]
        self.R = [int(c.shape[0]) for c in A_cores] + [int(A_cores[-1].shape[3])]
        self._n = (ctypes.c_int64 * self.d)(*self.n)
        self._r = (ctypes.c_int64 * (self.d + 1))(*self.r)
        self._R = (ctypes.c_int64 * (self.d + 1))(*self.R)
        self._xc, self._Ac = x_cores, A_cores

    @property
    def _x(self):   # pointer arrays built at call time, after every shape check
        return _ptrs(self._xc, "x_cores")

    @property
    def _A(self):
        return _ptrs(self._Ac, "A_cores")


def _check_interfaces(tr: "_Train", phis, name: str) -> None:
    if phis is None:
        return
    if len(phis) != tr.d + 1:
        raise ValueError(f"{name} must hold d+1 = {tr.d + 1} interfaces")
    for k, p in enumerate(phis):
        _expect(p, (tr.r[k], tr.R[k], tr.r[k]), f"{name}[{k}]")


def _check_cores(tr: "_Train", cores, name: str, nvec=None) -> None:
    if cores is None:
        return
    if len(cores) != tr.d:
        raise ValueError(f"{name} must hold d = {tr.d} cores")
    for k, c in enumerate(cores):
        shape = (tr.r[k], tr.n[k], tr.r[k + 1]) if nvec is None else \
            (tr.r[k], tr.n[k], nvec, tr.r[k + 1])
        _expect(c, shape, f"{name}[{k}]")


def _ptrs(ts: Sequence[torch.Tensor], name: str):
    return (ctypes.c_void_p * len(ts))(*[_dev(t, f"{name}[{i}]") for i, t in enumerate(ts)])


def tt_sweep_workspace_size(tr: _Train) -> int:
    return int(lib.tt_sweep_workspace_size(tr.d, tr._n, tr._r, tr._R))


def tt_sweep_als_workspace_size(tr: _Train, nvec: int) -> int:
    return int(lib.tt_sweep_als_workspace_size(tr.d, tr._n, tr._r, tr._R, nvec))


def alloc_interfaces(x_cores, A_cores) -> List[torch.Tensor]:
    tr = _Train(x_cores, A_cores)
    dev = x_cores[0].device
    return [torch.zeros((tr.r[k], tr.R[k], tr.r[k]), dtype=torch.float64, device=dev)
            for k in range(tr.d + 1)]


def tt_sweep_interfaces(x_cores, A_cores, phiL=None, phiR=None, directions=TT_SWEEP_BOTH,
                        workspace=None, stream=None):
    """H7: build phiL[0..d] and/or phiR[0..d] (lists of device tensors).  Returns (phiL, phiR)."""
    tr = _Train(x_cores, A_cores)
    if phiL is None and directions & TT_SWEEP_LEFT:
        phiL = alloc_interfaces(x_cores, A_cores)
    if phiR is None and directions & TT_SWEEP_RIGHT:
        phiR = alloc_interfaces(x_cores, A_cores)
    _check_interfaces(tr, phiL if directions & TT_SWEEP_LEFT else None, "phiL")
    _check_interfaces(tr, phiR if directions & TT_SWEEP_RIGHT else None, "phiR")
    ws = _ws(tt_sweep_workspace_size(tr), workspace, x_cores[0].device)
    pl = _ptrs(phiL, "phiL") if phiL is not None else None
    pr = _ptrs(phiR, "phiR") if phiR is not None else None
    _invoke(lib.tt_sweep_interfaces, tr.d, tr._n, tr._r, tr._R, tr._x, tr._A, pl, pr, directions,
                                   ws.data_ptr(), ws.numel(), _stream(stream))
    return phiL, phiR


def tt_sweep_w34_workspace_size(tr: _Train) -> int:
    return int(lib.tt_sweep_w34_workspace_size(tr.d, tr._n, tr._r, tr._R))


def tt_sweep_w34(x_cores, A_cores, phiL=None, phiR=None, y_cores=None, workspace=None,
                 stream=None):
    """Workload W34 in one DAG-scheduled call: all interfaces and one local matvec per core.
    Returns (y_cores, phiL, phiR)."""
    tr = _Train(x_cores, A_cores)
    if phiL is None:
        phiL = alloc_interfaces(x_cores, A_cores)
    if phiR is None:
        phiR = alloc_interfaces(x_cores, A_cores)
    if y_cores is None:
        y_cores = [torch.empty_like(c) for c in x_cores]
    _check_interfaces(tr, phiL, "phiL")
    _check_interfaces(tr, phiR, "phiR")
    _check_cores(tr, y_cores, "y_cores")
    ws = _ws(tt_sweep_w34_workspace_size(tr), workspace, x_cores[0].device)
    _invoke(lib.tt_sweep_w34, tr.d, tr._n, tr._r, tr._R, tr._x, tr._A, _ptrs(phiL, "phiL"),
                            _ptrs(phiR, "phiR"), _ptrs(y_cores, "y_cores"), ws.data_ptr(),
                            ws.numel(), _stream(stream))
    return y_cores, phiL, phiR


def tt_sweep_als(x_cores, A_cores, X_blocks, Y_fwd=None, Y_bwd=None, phiL=None, phiR=None,
                 workspace=None, stream=None):
    """H7 with interleaved batched matvecs (workload W5).  Returns
    (Y_fwd, Y_bwd, phiL, phiR)."""
    tr = _Train(x_cores, A_cores)
    nvec = int(X_blocks[0].shape[2])
    if Y_fwd is None:
        Y_fwd = [torch.empty_like(X) for X in X_blocks]
    if phiL is None:
        phiL = alloc_interfaces(x_cores, A_cores)
    if phiR is None:
        phiR = alloc_interfaces(x_cores, A_cores)
    _check_cores(tr, X_blocks, "X_blocks", nvec)
    _check_cores(tr, Y_fwd, "Y_fwd", nvec)
    _check_cores(tr, Y_bwd, "Y_bwd", nvec)
    _check_interfaces(tr, phiL, "phiL")
    _check_interfaces(tr, phiR, "phiR")
    ws = _ws(tt_sweep_als_workspace_size(tr, nvec), workspace, x_cores[0].device)
    _invoke(lib.tt_sweep_als, tr.d, tr._n, tr._r, tr._R, nvec, tr._x, tr._A,
                            _ptrs(X_blocks, "X_blocks"), _ptrs(Y_fwd, "Y_fwd"),
                            _ptrs(Y_bwd, "Y_bwd") if Y_bwd is not None else None,
                            _ptrs(phiL, "phiL"), _ptrs(phiR, "phiR"), ws.data_ptr(), ws.numel(),
                            _stream(stream))
    return Y_fwd, Y_bwd, phiL, phiR


def tt_operator_apply(x_cores, A_cores, z_cores=None, stream=None):
    """H8: unrounded TT-matrix x TT-vector product; returns z cores (r R, n_row, r' R')."""
    d = len(x_cores)
    if len(A_cores) != d or d == 0:
        raise ValueError("x_cores and A_cores must be non-empty and of the same length")
    for k in range(d):
        if x_cores[k].dim() != 3 or A_cores[k].dim() != 4:
            raise ValueError(f"core {k}: x must be (r, n_col, r') and A (R, n_row, n_col, R')")
        if A_cores[k].shape[2] != x_cores[k].shape[1]:
            raise ValueError(f"core {k}: A column mode {A_cores[k].shape[2]} != x mode "
                             f"{x_cores[k].shape[1]}")
        if k + 1 < d and (x_cores[k].shape[2] != x_cores[k + 1].shape[0]
                          or A_cores[k].shape[3] != A_cores[k + 1].shape[0]):
            raise ValueError(f"bond {k + 1}: neighbouring cores disagree")
    n_row = [int(c.shape[1]) for c in A_cores]
    n_col = [int(c.shape[2]) for c in A_cores]
    r = [int(c.shape[0]) for c in x_cores] + [int(x_cores[-1].shape[2])]
    R = [int(c.shape[0]) for c in A_cores] + [int(A_cores[-1].shape[3])]
    if z_cores is None:
        z_cores = [torch.empty((r[k] * R[k], n_row[k], r[k + 1] * R[k + 1]), dtype=torch.float64,
                               device=x_cores[0].device) for k in range(d)]
    if len(z_cores) != d:
        raise ValueError(f"z_cores must hold d = {d} cores")
    for k in range(d):
        _expect(z_cores[k], (r[k] * R[k], n_row[k], r[k + 1] * R[k + 1]), f"z_cores[{k}]")
    _same_device(*x_cores, *A_cores, *z_cores)
    a64 = lambda v: (ctypes.c_int64 * len(v))(*v)
    _invoke(lib.tt_operator_apply, d, a64(n_row), a64(n_col), a64(r), a64(R),
                                 _ptrs(x_cores, "x_cores"), _ptrs(A_cores, "A_cores"),
                                 _ptrs(z_cores, "z_cores"), _stream(stream))
    return z_cores


def tt_trace_enable(capacity: int = 4096) -> None:
    """Start recording a CUDA-event pair around every library launch on this thread."""
    _check(lib.tt_trace_enable(int(capacity)))


def tt_trace_disable() -> None:
    _check(lib.tt_trace_disable())


def tt_trace_count() -> int:
    return int(lib.tt_trace_count())


def tt_trace_read(i: int) -> dict:
    """Record i: {stage, tile, M, N, K, ms} (synchronises on the launch's end event)."""
    st, tile = ctypes.c_int(), ctypes.c_int()
    M, N, K = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    ms = ctypes.c_float()
    _check(lib.tt_trace_read(int(i), ctypes.byref(st), ctypes.byref(tile), ctypes.byref(M),
                             ctypes.byref(N), ctypes.byref(K), ctypes.byref(ms)))
    return {"stage": STAGE_NAMES.get(st.value, str(st.value)), "tile": tile.value,
            "M": M.value, "N": N.value, "K": K.value, "ms": ms.value}


def tt_fp64_peak_probe(iters: int, stream=None) -> float:
    """Enqueue the FP64 DMMA probe kernel; returns its flop count (time it on `stream`)."""
    f = ctypes.c_double()
    _check(lib.tt_fp64_peak_probe(int(iters), ctypes.byref(f), _stream(stream)))
    return f.value


def tt_debug_force_v1(on: bool) -> None:
    """Test hook: route this thread's GEMM stages through the generic (v1) kernel."""
    lib.tt_debug_force_v1(1 if on else 0)


def tt_debug_set_variant(v: int) -> None:
    """Benchmark hook: GEMM tiling variant for this thread (-1 default, 0, 1)."""
    lib.tt_debug_set_variant(int(v))


def tt_set_graph_cache(enabled: bool) -> None:
    """Eager multi-launch calls are replayed from a per-thread CUDA graph cache from the second
    identical call on (default on); False disables it and destroys the cached graphs."""
    lib.tt_set_graph_cache(1 if enabled else 0)


_MATVEC_MODES = {"auto": 0, "three_stage": 1, "fused": 2}


def tt_set_matvec_mode(mode) -> None:
    """Evaluation of the local matvec on the calling thread: "auto" (default), "three_stage" or
    "fused" (T1 kept in shared memory: about half the workspace and HBM traffic, same results;
    include/tt_hotpath.h tt_set_matvec_mode).  Workspace sizes follow the mode."""
    _check(lib.tt_set_matvec_mode(int(_MATVEC_MODES.get(mode, mode))))


def tt_debug_set_fused(mode: int) -> None:
    """Fused S1 -> S2 matvec kernel: 0 policy, -1 never, 1 whenever eligible (include/tt_hotpath_debug.h)."""
    lib.tt_debug_set_fused(int(mode))


def tt_debug_set_dag(mode: int) -> None:
    """Benchmark hook: experimental DAG executor for tt_sweep_w34 (0 off = default, 1 / 2 on)."""
    lib.tt_debug_set_dag(int(mode))


def tt_debug_dag_trace(buf=None):
    """Measurement hook: record per-unit timestamps of the next DAG launches into buf (CUDA
    uint64 tensor of 5 x units); returns (tasks, units, unit0 list) of the last DAG launch."""
    import numpy as np
    u0 = np.zeros(4096, dtype=np.int32)
    cap = buf.numel() // 5 if buf is not None else 0
    v = lib.tt_debug_dag_trace(buf.data_ptr() if buf is not None else None, cap,
                               u0.ctypes.data, len(u0))
    nt, nu = int(v >> 32), int(v & 0xffffffff)
    return nt, nu, u0[: nt + 1].tolist()


def tt_debug_set_flags(flags: int) -> None:
    """Benchmark hook (results become wrong): 1 = skip GEMM stores, 2 = skip operand loads."""
    lib.tt_debug_set_flags(int(flags))


def tt_local_gmres_workspace_size(rl, n, rr, Rl, Rr, nvec, m, k_aug=0) -> int:
    return int(lib.tt_local_gmres_workspace_size(rl, n, rr, Rl, Rr, nvec, m, k_aug))


def tt_local_gmres(phiL, A, phiR, F, X=None, m=20, cycles=1, tol=0.0, rel_res=None, iters=None,
                   workspace=None, stream=None, k_aug=0):
    """Restarted GMRES(m) (k_aug = 0) or accelerated LGMRES(m, k_aug) on the projected local
    operator for every column of the Block-TT right-hand side F (rl, n, nvec, rr)
    (PAPER.md:488).  X: initial guess (zeros if None), overwritten with the iterate.
    Returns (X, rel_res, iters) (device tensors)."""
    if F.dim() != 4:
        raise ValueError(f"F must be (rl, n, nvec, rr), got shape {tuple(F.shape)}")
    rl, n, nvec, rr = F.shape
    _check_local(phiL, A, phiR, rl, n, rr)
    Rl, Rr = A.shape[0], A.shape[3]
    if X is None:
        X = torch.zeros_like(F)
    _expect(X, F.shape, "X")
    if rel_res is None:
        rel_res = torch.empty(nvec, dtype=torch.float64, device=F.device)
    if iters is None:
        iters = torch.empty(nvec, dtype=torch.int64, device=F.device)
    _expect(rel_res, (nvec,), "rel_res")
    _expect(iters, (nvec,), "iters")
    _same_device(phiL, A, phiR, F, X, rel_res, iters, workspace)
    ws = _ws(tt_local_gmres_workspace_size(rl, n, rr, Rl, Rr, nvec, m, k_aug), workspace, F.device)
    if iters.dtype != torch.int64 or not iters.is_cuda:
        raise TypeError("iters must be a CUDA int64 tensor")
    _check(lib.tt_local_gmres(rl, n, rr, Rl, Rr, nvec, m, k_aug, cycles, float(tol), _dev(phiL, "phiL"),
                              _dev(A, "A"), _dev(phiR, "phiR"), _dev(F, "F"), _dev(X, "X"),
                              _dev(rel_res, "rel_res"), iters.data_ptr(), ws.data_ptr(),
                              ws.numel(), _stream(stream)))
    return X, rel_res, iters


def tt_local_lobpcg_workspace_size(rl, n, rr, RlA, RrA, RlB, RrB, nb) -> int:
    return int(lib.tt_local_lobpcg_workspace_size(rl, n, rr, RlA, RrA, RlB, RrB, nb))


def tt_local_lobpcg(opA, X, opB=None, maxiter=100, tol=1e-10, lam=None, res=None, iters=None,
                    step=None, workspace=None, stream=None, refresh=20):
    """Block LOBPCG for the nb largest eigenpairs of the projected pencil (L_A, L_B)
    (PAPER.md:556-567).  opA, opB: (phiL, A, phiR) triplets of device tensors; opB None means
    L_B = I.  X (rl, n, nb, rr): initial block, overwritten with the Ritz vectors.
    Returns (X, lam, res, iters, step) (device tensors; step = min(1, 1/lam[0]) or 1)."""
    if X.dim() != 4:
        raise ValueError(f"X must be (rl, n, nb, rr), got shape {tuple(X.shape)}")
    rl, n, nb, rr = X.shape
    phiLA, AA, phiRA = opA
    _check_local(phiLA, AA, phiRA, rl, n, rr)
    RlA, RrA = AA.shape[0], AA.shape[3]
    if opB is not None:
        phiLB, AB, phiRB = opB
        _check_local(phiLB, AB, phiRB, rl, n, rr)
        _same_device(phiLB, AB, phiRB)
        RlB, RrB = AB.shape[0], AB.shape[3]
        pB = (_dev(phiLB, "phiL_B"), _dev(AB, "A_B"), _dev(phiRB, "phiR_B"))
    else:
        RlB = RrB = 0
        pB = (None, None, None)
    dev = X.device
    lam = torch.empty(nb, dtype=torch.float64, device=dev) if lam is None else lam
    res = torch.empty(nb, dtype=torch.float64, device=dev) if res is None else res
    iters = torch.empty(1, dtype=torch.int64, device=dev) if iters is None else iters
    step = torch.empty(1, dtype=torch.float64, device=dev) if step is None else step
    _expect(lam, (nb,), "lam")
    _expect(res, (nb,), "res")
    _expect(iters, (1,), "iters")
    _expect(step, (1,), "step")
    if iters.dtype != torch.int64 or not iters.is_cuda:
        raise TypeError("iters must be a CUDA int64 tensor")
    _same_device(phiLA, AA, phiRA, X, lam, res, iters, step, workspace)
    ws = _ws(tt_local_lobpcg_workspace_size(rl, n, rr, RlA, RrA, RlB, RrB, nb), workspace, dev)
    _check(lib.tt_local_lobpcg(rl, n, rr, RlA, RrA, RlB, RrB, nb, int(maxiter), int(refresh),
                               float(tol),
                               _dev(phiLA, "phiL_A"), _dev(AA, "A_A"), _dev(phiRA, "phiR_A"),
                               pB[0], pB[1], pB[2], _dev(X, "X"), _dev(lam, "lam"),
                               _dev(res, "res"), iters.data_ptr(), _dev(step, "step"),
                               ws.data_ptr(), ws.numel(), _stream(stream)))
    return X, lam, res, iters, step


def tt_merge_operator_cores(A1, A2, A12=None, stream=None):
    """Two-site supercore operator A12 (Rl, n1 n2, n1 n2, Rr) from A1 (Rl,n1,n1,Rm), A2 (Rm,n2,n2,Rr)."""
    if A1.dim() != 4 or A2.dim() != 4:
        raise ValueError("A1 and A2 must be 4-D operator cores")
    Rl, n1, _, Rm = A1.shape
    _, n2, _, Rr = A2.shape
    _expect(A1, (Rl, n1, n1, Rm), "A1")
    _expect(A2, (Rm, n2, n2, Rr), "A2")
    if A12 is None:
        A12 = torch.empty((Rl, n1 * n2, n1 * n2, Rr), dtype=torch.float64, device=A1.device)
    _expect(A12, (Rl, n1 * n2, n1 * n2, Rr), "A12")
    _same_device(A1, A2, A12)
    _check(lib.tt_merge_operator_cores(Rl, n1, n2, Rm, Rr, _dev(A1, "A1"), _dev(A2, "A2"),
                                       _dev(A12, "A12"), _stream(stream)))
    return A12


def tt_local_matvec_two_site_workspace_size(rl, n1, n2, rr, Rl, Rm, Rr, nvec) -> int:
    return int(lib.tt_local_matvec_two_site_workspace_size(rl, n1, n2, rr, Rl, Rm, Rr, nvec))


def tt_local_matvec_two_site(phiL, A1, A2, phiR, W, Y=None, workspace=None, stream=None):
    """Two-site (DMRG supercore) local matvec; W, Y (rl, n1, n2, nvec, rr) or (rl, n1, n2, rr)."""
    single = W.dim() == 4
    Wv = W.unsqueeze(3) if single else W
    if Wv.dim() != 5 or A1.dim() != 4 or A2.dim() != 4:
        raise ValueError("W must be (rl, n1, n2, [nvec,] rr), A1/A2 4-D operator cores")
    rl, n1, n2, nvec, rr = Wv.shape
    Rl, Rm, Rr = A1.shape[0], A1.shape[3], A2.shape[3]
    _expect(A1, (Rl, n1, n1, Rm), "A1")
    _expect(A2, (Rm, n2, n2, Rr), "A2")
    _expect(phiL, (rl, Rl, rl), "phiL")
    _expect(phiR, (rr, Rr, rr), "phiR")
    if Y is None:
        Y = torch.empty_like(W)
    _expect(Y, W.shape, "Y")
    _same_device(phiL, A1, A2, phiR, W, Y, workspace)
    ws = _ws(tt_local_matvec_two_site_workspace_size(rl, n1, n2, rr, Rl, Rm, Rr, nvec), workspace,
             W.device)
    _check(lib.tt_local_matvec_two_site(rl, n1, n2, rr, Rl, Rm, Rr, nvec, _dev(phiL, "phiL"),
                                        _dev(A1, "A1"), _dev(A2, "A2"), _dev(phiR, "phiR"),
                                        _dev(W, "W"), _dev(Y, "Y"), ws.data_ptr(), ws.numel(),
                                        _stream(stream)))
    return Y


def tt_block_local_matvec_workspace_size(rl, n, rr, Rl, Rr) -> int:
    a64 = lambda v: (ctypes.c_int64 * len(v))(*v)
    return int(lib.tt_block_local_matvec_workspace_size(rl, n, rr, len(Rl), a64(Rl), a64(Rr)))


def tt_block_local_matvec(ops, terms, X, Y=None, workspace=None, stream=None):
    """Projected KKT block action.  ops: list of (phiL, A, phiR) device
    tensors sharing the frame; terms: list of (row, col, op, op2, coeff); X (rl, n, nb, rr)."""
    if X.dim() != 4:
        raise ValueError(f"X must be (rl, n, nblocks, rr), got shape {tuple(X.shape)}")
    rl, n, nb, rr = X.shape
    for o, (pL, Ao, pR) in enumerate(ops):
        try:
            _check_local(pL, Ao, pR, rl, n, rr)
        except ValueError as e:
            raise ValueError(f"operator {o}: {e}") from None
    for (row, col, op, op2, _cf) in terms:
        if not (0 <= row < nb and 0 <= col < nb and 0 <= op < len(ops) and -1 <= op2 < len(ops)):
            raise ValueError(f"term {(row, col, op, op2)} indexes outside {nb} blocks / {len(ops)} ops")
    Rl = [int(o[1].shape[0]) for o in ops]
    Rr = [int(o[1].shape[3]) for o in ops]
    if Y is None:
        Y = torch.empty_like(X)
    _expect(Y, X.shape, "Y")
    _same_device(X, Y, workspace, *[t for o in ops for t in o])
    a64 = lambda v: (ctypes.c_int64 * len(v))(*v)
    T = (TTBlockTerm * max(len(terms), 1))(*[TTBlockTerm(int(r), int(c), int(o), int(o2), float(cf))
                                             for (r, c, o, o2, cf) in terms])
    ws = _ws(tt_block_local_matvec_workspace_size(rl, n, rr, Rl, Rr), workspace, X.device)
    _check(lib.tt_block_local_matvec(rl, n, rr, nb, len(ops), a64(Rl), a64(Rr),
                                     _ptrs([o[0] for o in ops], "phiL"),
                                     _ptrs([o[1] for o in ops], "A"),
                                     _ptrs([o[2] for o in ops], "phiR"), len(terms), T,
                                     _dev(X, "X"), _dev(Y, "Y"), ws.data_ptr(), ws.numel(),
                                     _stream(stream)))
    return Y


def tt_round(cores, delta, max_rank=0, workspace=None, stream=None):
    """TT rounding of a TT vector (list of device cores (r_k, n_k, r_{k+1})) to relative
    accuracy delta.  Synchronous.  Returns the list of rounded cores."""
    d = len(cores)
    a64 = lambda v: (ctypes.c_int64 * len(v))(*v)
    _check_vector_train(cores)
    n = [int(c.shape[1]) for c in cores]
    r = [int(c.shape[0]) for c in cores] + [int(cores[-1].shape[2])]
    outs = [torch.empty_like(c) for c in cores]
    rout = (ctypes.c_int64 * (d + 1))()
    ws = _ws(int(lib.tt_round_workspace_size(d, a64(n), a64(r))), workspace, cores[0].device)
    _check(lib.tt_round(d, a64(n), a64(r), _ptrs(cores, "cores"), float(delta), int(max_rank),
                        rout, _ptrs(outs, "cores_out"), ws.data_ptr(), ws.numel(), _stream(stream)))
    ro = list(rout)
    return [outs[k].reshape(-1)[: ro[k] * n[k] * ro[k + 1]].reshape(ro[k], n[k], ro[k + 1])
            for k in range(d)]


def tt_round_async(cores, delta, max_rank=0, workspace=None, stream=None, ranks=None):
    """Asynchronous TT rounding: device-side rank decisions, no host
    synchronisation, graph-capturable.  Returns (padded_cores, ranks): zero-padded cores with
    the host-known storage ranks and a device int64 tensor (d + 1) of the effective ranks;
    tt_compact(padded_cores, ranks) slices them (that reads the ranks: a synchronisation)."""
    d = len(cores)
    a64 = lambda v: (ctypes.c_int64 * len(v))(*v)
    _check_vector_train(cores)
    n = [int(c.shape[1]) for c in cores]
    r = [int(c.shape[0]) for c in cores] + [int(cores[-1].shape[2])]
    outs = [torch.empty_like(c) for c in cores]
    if ranks is None:
        ranks = torch.empty(d + 1, dtype=torch.int64, device=cores[0].device)
    elif ranks.dtype != torch.int64 or ranks.numel() != d + 1 or ranks.device != cores[0].device:
        raise ValueError("ranks must be a device int64 tensor of d + 1 entries")
    rst = (ctypes.c_int64 * (d + 1))()
    ws = _ws(int(lib.tt_round_workspace_size(d, a64(n), a64(r))), workspace, cores[0].device)
    _check(lib.tt_round_async(d, a64(n), a64(r), _ptrs(cores, "cores"), float(delta),
                              int(max_rank), rst, ranks.data_ptr(), _ptrs(outs, "cores_out"),
                              ws.data_ptr(), ws.numel(), _stream(stream)))
    rs = list(rst)
    padded = [outs[k].reshape(-1)[: rs[k] * n[k] * rs[k + 1]].reshape(rs[k], n[k], rs[k + 1])
              for k in range(d)]
    return padded, ranks


def tt_compact(padded_cores, ranks):
    """Slice the zero-padded cores of tt_round_async to their effective ranks (reads `ranks`
    from the device: synchronises)."""
    ro = [int(v) for v in ranks.tolist()]
    return [c[: ro[k], :, : ro[k + 1]].contiguous() for k, c in enumerate(padded_cores)]


def _check_vector_train(cores) -> None:
    if len(cores) == 0:
        raise ValueError("empty train")
    for k, c in enumerate(cores):
        if c.dim() != 3:
            raise ValueError(f"core {k} must be (r, n, r'), got shape {tuple(c.shape)}")
        if k + 1 < len(cores) and c.shape[2] != cores[k + 1].shape[0]:
            raise ValueError(f"bond {k + 1}: core {k} has {c.shape[2]}, core {k + 1} has "
                             f"{cores[k + 1].shape[0]}")
    _same_device(*cores)


def tt_orthonormalise_workspace_size(n, r) -> int:
    a64 = lambda v: (ctypes.c_int64 * len(v))(*v)
    return int(lib.tt_orthonormalise_workspace_size(len(n), a64(n), a64(r)))


def tt_orthonormalise(cores, direction=TT_SWEEP_LEFT, workspace=None, stream=None):
    """Left- (TT_SWEEP_LEFT) or right- (TT_SWEEP_RIGHT) orthonormalisation of a TT vector
    (SURVEY.md 8(f) row 3); the represented tensor is unchanged.  Synchronous.  Returns the
    list of cores (bonds shrink only where the train is exactly rank deficient)."""
    d = len(cores)
    a64 = lambda v: (ctypes.c_int64 * len(v))(*v)
    _check_vector_train(cores)
    n = [int(c.shape[1]) for c in cores]
    r = [int(c.shape[0]) for c in cores] + [int(cores[-1].shape[2])]
    outs = [torch.empty_like(c) for c in cores]
    rout = (ctypes.c_int64 * (d + 1))()
    ws = _ws(int(lib.tt_orthonormalise_workspace_size(d, a64(n), a64(r))), workspace,
             cores[0].device)
    _check(lib.tt_orthonormalise(d, a64(n), a64(r), _ptrs(cores, "cores"), int(direction), rout,
                                 _ptrs(outs, "cores_out"), ws.data_ptr(), ws.numel(),
                                 _stream(stream)))
    ro = list(rout)
    return [outs[k].reshape(-1)[: ro[k] * n[k] * ro[k + 1]].reshape(ro[k], n[k], ro[k + 1])
            for k in range(d)]


def tt_block_move_workspace_size(r0, n0, l, r1, n1, r2) -> int:
    return int(lib.tt_block_move_workspace_size(r0, n0, l, r1, n1, r2))


def tt_block_move_right(Wk_hat, Wk1, delta=0.0, max_rank=0, workspace=None, stream=None):
    """Move the block index of Wk_hat (r0,n0,l,r1) into Wk1 (r1,n1,r2) by one truncated SVD
    step.  Returns (Wk (r0,n0,s) left-orthonormal, Wk1_hat (s,n1,l,r2))."""
    if Wk_hat.dim() != 4 or Wk1.dim() != 3 or Wk1.shape[0] != Wk_hat.shape[3]:
        raise ValueError("Wk_hat must be (r0, n0, l, r1) and Wk1 (r1, n1, r2)")
    _same_device(Wk_hat, Wk1, workspace)
    r0, n0, l, r1 = Wk_hat.shape
    _, n1, r2 = Wk1.shape
    smax = min(r0 * n0, l * r1)
    Wk = torch.empty(r0 * n0 * smax, dtype=torch.float64, device=Wk_hat.device)
    W1 = torch.empty(smax * n1 * l * r2, dtype=torch.float64, device=Wk_hat.device)
    s_out = ctypes.c_int64()
    ws = _ws(tt_block_move_workspace_size(r0, n0, l, r1, n1, r2), workspace, Wk_hat.device)
    _check(lib.tt_block_move_right(r0, n0, l, r1, n1, r2, float(delta), int(max_rank),
                                   _dev(Wk_hat, "Wk_hat"), _dev(Wk1, "Wk1"), _dev(Wk, "Wk_out"),
                                   _dev(W1, "Wk1_hat_out"), ctypes.byref(s_out), ws.data_ptr(),
                                   ws.numel(), _stream(stream)))
    sk = s_out.value
    return (Wk[: r0 * n0 * sk].reshape(r0, n0, sk), W1[: sk * n1 * l * r2].reshape(sk, n1, l, r2))


def tt_block_move_right_async(Wk_hat, Wk1, delta=0.0, max_rank=0, workspace=None, stream=None,
                              rank=None):
    """tt_block_move_right with the truncation decided on the device (no synchronisation,
    graph-capturable).  Returns (Wk (r0,n0,S), Wk1_hat (S,n1,l,r2), rank): zero-padded to the
    storage extent S = min(r0 n0, l r1), `rank` a device int64 tensor (1) with the effective
    rank s; Wk[..., :s] and Wk1_hat[:s] are the synchronous call's outputs."""
    if Wk_hat.dim() != 4 or Wk1.dim() != 3 or Wk1.shape[0] != Wk_hat.shape[3]:
        raise ValueError("Wk_hat must be (r0, n0, l, r1) and Wk1 (r1, n1, r2)")
    _same_device(Wk_hat, Wk1, workspace)
    r0, n0, l, r1 = Wk_hat.shape
    _, n1, r2 = Wk1.shape
    smax = min(r0 * n0, l * r1)
    Wk = torch.empty(r0, n0, smax, dtype=torch.float64, device=Wk_hat.device)
    W1 = torch.empty(smax, n1, l, r2, dtype=torch.float64, device=Wk_hat.device)
    if rank is None:
        rank = torch.empty(1, dtype=torch.int64, device=Wk_hat.device)
    s_st = ctypes.c_int64()
    ws = _ws(tt_block_move_workspace_size(r0, n0, l, r1, n1, r2), workspace, Wk_hat.device)
    _check(lib.tt_block_move_right_async(r0, n0, l, r1, n1, r2, float(delta), int(max_rank),
                                         _dev(Wk_hat, "Wk_hat"), _dev(Wk1, "Wk1"),
                                         _dev(Wk, "Wk_out"), _dev(W1, "Wk1_hat_out"),
                                         ctypes.byref(s_st), rank.data_ptr(), ws.data_ptr(),
                                         ws.numel(), _stream(stream)))
    assert s_st.value == smax
    return Wk, W1, rank


def tt_block_move_left_async(Wkm1, Wk_hat, delta=0.0, max_rank=0, workspace=None, stream=None,
                             rank=None):
    """tt_block_move_left with the truncation decided on the device.  Returns
    (Wkm1_hat (r0,n0,l,S), Wk (S,n1,r2), rank), zero-padded to S = min(r1 l, n1 r2)."""
    if Wkm1.dim() != 3 or Wk_hat.dim() != 4 or Wk_hat.shape[0] != Wkm1.shape[2]:
        raise ValueError("Wkm1 must be (r0, n0, r1) and Wk_hat (r1, n1, l, r2)")
    _same_device(Wkm1, Wk_hat, workspace)
    r0, n0, r1 = Wkm1.shape
    _, n1, l, r2 = Wk_hat.shape
    smax = min(r1 * l, n1 * r2)
    Wh = torch.empty(r0, n0, l, smax, dtype=torch.float64, device=Wk_hat.device)
    Wk = torch.empty(smax, n1, r2, dtype=torch.float64, device=Wk_hat.device)
    if rank is None:
        rank = torch.empty(1, dtype=torch.int64, device=Wk_hat.device)
    s_st = ctypes.c_int64()
    ws = _ws(tt_block_move_workspace_size(r0, n0, l, r1, n1, r2), workspace, Wk_hat.device)
    _check(lib.tt_block_move_left_async(r0, n0, r1, n1, l, r2, float(delta), int(max_rank),
                                        _dev(Wkm1, "Wkm1"), _dev(Wk_hat, "Wk_hat"),
                                        _dev(Wh, "Wkm1_hat_out"), _dev(Wk, "Wk_out"),
                                        ctypes.byref(s_st), rank.data_ptr(), ws.data_ptr(),
                                        ws.numel(), _stream(stream)))
    assert s_st.value == smax
    return Wh, Wk, rank


def tt_block_move_left(Wkm1, Wk_hat, delta=0.0, max_rank=0, workspace=None, stream=None):
    """Move the block index of Wk_hat (r1,n1,l,r2) into Wkm1 (r0,n0,r1).
    Returns (Wkm1_hat (r0,n0,l,s), Wk (s,n1,r2) right-orthonormal)."""
    if Wkm1.dim() != 3 or Wk_hat.dim() != 4 or Wk_hat.shape[0] != Wkm1.shape[2]:
        raise ValueError("Wkm1 must be (r0, n0, r1) and Wk_hat (r1, n1, l, r2)")
    _same_device(Wkm1, Wk_hat, workspace)
    r0, n0, r1 = Wkm1.shape
    _, n1, l, r2 = Wk_hat.shape
    smax = min(r1 * l, n1 * r2)
    Wh = torch.empty(r0 * n0 * l * smax, dtype=torch.float64, device=Wk_hat.device)
    Wk = torch.empty(smax * n1 * r2, dtype=torch.float64, device=Wk_hat.device)
    s_out = ctypes.c_int64()
    ws = _ws(tt_block_move_workspace_size(r0, n0, l, r1, n1, r2), workspace, Wk_hat.device)
    _check(lib.tt_block_move_left(r0, n0, r1, n1, l, r2, float(delta), int(max_rank),
                                  _dev(Wkm1, "Wkm1"), _dev(Wk_hat, "Wk_hat"), _dev(Wh, "Wkm1_hat_out"),
                                  _dev(Wk, "Wk_out"), ctypes.byref(s_out), ws.data_ptr(),
                                  ws.numel(), _stream(stream)))
    sk = s_out.value
    return (Wh[: r0 * n0 * l * sk].reshape(r0, n0, l, sk), Wk[: sk * n1 * r2].reshape(sk, n1, r2))


def tt_pg_workspace_size(rl_bra, rl, n, rr_bra, rr, Rl, Rr, nvec=1) -> int:
    return int(lib.tt_pg_workspace_size(rl_bra, rl, n, rr_bra, rr, Rl, Rr, nvec))


def tt_local_matvec_pg(phiL, A, phiR, X, Y=None, workspace=None, stream=None):
    """Petrov-Galerkin local matvec (bra train != ket train): phiL (rl_bra, Rl, rl),
    phiR (rr_bra, Rr, rr), X (rl, n, nvec, rr) or (rl, n, rr) -> Y (rl_bra, n, [nvec,] rr_bra)."""
    single = X.dim() == 3
    Xv = X.unsqueeze(2) if single else X
    if Xv.dim() != 4 or phiL.dim() != 3 or phiR.dim() != 3:
        raise ValueError("X must be (rl, n, [nvec,] rr); phiL, phiR 3-D")
    rl, n, nvec, rr = Xv.shape
    rlb, rrb = phiL.shape[0], phiR.shape[0]
    _check_local(phiL, A, phiR, rl, n, rr, rlb, rrb)
    Rl, Rr = A.shape[0], A.shape[3]
    shape = (rlb, n, rrb) if single else (rlb, n, nvec, rrb)
    if Y is None:
        Y = torch.empty(shape, dtype=torch.float64, device=X.device)
    _expect(Y, shape, "Y")
    _same_device(phiL, A, phiR, X, Y, workspace)
    ws = _ws(tt_pg_workspace_size(rlb, rl, n, rrb, rr, Rl, Rr, nvec), workspace, X.device)
    _check(lib.tt_local_matvec_pg(rlb, rl, n, rrb, rr, Rl, Rr, nvec, _dev(phiL, "phiL"), _dev(A, "A"),
                                  _dev(phiR, "phiR"), _dev(X, "X"), _dev(Y, "Y"), ws.data_ptr(),
                                  ws.numel(), _stream(stream)))
    return Y


def tt_interface_left_pg(phiL_prev, A, x_bra, x_ket, out=None, workspace=None, stream=None):
    rlb, n, rrb = x_bra.shape
    rl, _, rr = x_ket.shape
    Rl, Rr = A.shape[0], A.shape[3]
    _expect(x_ket, (rl, n, rr), "x_ket")
    _expect(A, (Rl, n, n, Rr), "A")
    _expect(phiL_prev, (rlb, Rl, rl), "phiL_prev")
    if out is None:
        out = torch.empty((rrb, Rr, rr), dtype=torch.float64, device=x_ket.device)
    _expect(out, (rrb, Rr, rr), "phiL_next")
    _same_device(phiL_prev, A, x_bra, x_ket, out, workspace)
    ws = _ws(tt_pg_workspace_size(rlb, rl, n, rrb, rr, Rl, Rr, 1), workspace, x_ket.device)
    _check(lib.tt_interface_left_pg(rlb, rl, n, rrb, rr, Rl, Rr, _dev(phiL_prev, "phiL_prev"),
                                    _dev(A, "A"), _dev(x_bra, "x_bra"), _dev(x_ket, "x_ket"),
                                    _dev(out, "phiL_next"), ws.data_ptr(), ws.numel(),
                                    _stream(stream)))
    return out


def tt_interface_right_pg(phiR_next, A, x_bra, x_ket, out=None, workspace=None, stream=None):
    rlb, n, rrb = x_bra.shape
    rl, _, rr = x_ket.shape
    Rl, Rr = A.shape[0], A.shape[3]
    _expect(x_ket, (rl, n, rr), "x_ket")
    _expect(A, (Rl, n, n, Rr), "A")
    _expect(phiR_next, (rrb, Rr, rr), "phiR_next")
    if out is None:
        out = torch.empty((rlb, Rl, rl), dtype=torch.float64, device=x_ket.device)
    _expect(out, (rlb, Rl, rl), "phiR_prev")
    _same_device(phiR_next, A, x_bra, x_ket, out, workspace)
    ws = _ws(tt_pg_workspace_size(rlb, rl, n, rrb, rr, Rl, Rr, 1), workspace, x_ket.device)
    _check(lib.tt_interface_right_pg(rlb, rl, n, rrb, rr, Rl, Rr, _dev(phiR_next, "phiR_next"),
                                     _dev(A, "A"), _dev(x_bra, "x_bra"), _dev(x_ket, "x_ket"),
                                     _dev(out, "phiR_prev"), ws.data_ptr(), ws.numel(),
                                     _stream(stream)))
    return out


def tt_enrich_right_workspace_size(rl, n, rx, rz, n1, r2) -> int:
    return int(lib.tt_enrich_right_workspace_size(rl, n, rx, rz, n1, r2))


def tt_enrich_right(x_k, z_k, x_k1, delta=0.0, max_rank=0, workspace=None, stream=None):
    """AMEn enrichment: [x_k | z_k] re-orthonormalised, x_{k+1} padded and
    rotated.  Returns (x_k' (rl, n, s) left-orthonormal, x_{k+1}' (s, n1, r2))."""
    if x_k.dim() != 3 or z_k.dim() != 3 or x_k1.dim() != 3:
        raise ValueError("x_k, z_k, x_k1 must be 3-D cores")
    rl, n, rx = x_k.shape
    rz = z_k.shape[2]
    _expect(z_k, (rl, n, rz), "z_k")
    if x_k1.shape[0] != rx:
        raise ValueError(f"x_k1 left bond {x_k1.shape[0]} != x_k right bond {rx}")
    _same_device(x_k, z_k, x_k1, workspace)
    _, n1, r2 = x_k1.shape
    smax = min(rl * n, rx + rz)
    xo = torch.empty(rl * n * smax, dtype=torch.float64, device=x_k.device)
    x1o = torch.empty(smax * n1 * r2, dtype=torch.float64, device=x_k.device)
    s_out = ctypes.c_int64()
    ws = _ws(tt_enrich_right_workspace_size(rl, n, rx, rz, n1, r2), workspace, x_k.device)
    _check(lib.tt_enrich_right(rl, n, rx, rz, n1, r2, float(delta), int(max_rank), _dev(x_k, "x_k"),
                               _dev(z_k, "z_k"), _dev(x_k1, "x_k1"), _dev(xo, "x_k_out"),
                               _dev(x1o, "x_k1_out"), ctypes.byref(s_out), ws.data_ptr(),
                               ws.numel(), _stream(stream)))
    sk = s_out.value
    return xo[: rl * n * sk].reshape(rl, n, sk), x1o[: sk * n1 * r2].reshape(sk, n1, r2)


def tt_enrich_right_async(x_k, z_k, x_k1, delta=0.0, max_rank=0, workspace=None, stream=None,
                          rank=None):
    """tt_enrich_right with the truncation decided on the device (graph-capturable).  Returns
    (x_k' (rl, n, S), x_{k+1}' (S, n1, r2), rank): zero-padded to S = min(rl n, rx + rz), `rank`
    a device int64 tensor (1) with the effective rank."""
    if x_k.dim() != 3 or z_k.dim() != 3 or x_k1.dim() != 3:
        raise ValueError("x_k, z_k, x_k1 must be 3-D cores")
    rl, n, rx = x_k.shape
    rz = z_k.shape[2]
    _expect(z_k, (rl, n, rz), "z_k")
    if x_k1.shape[0] != rx:
        raise ValueError(f"x_k1 left bond {x_k1.shape[0]} != x_k right bond {rx}")
    _same_device(x_k, z_k, x_k1, workspace)
    _, n1, r2 = x_k1.shape
    smax = min(rl * n, rx + rz)
    xo = torch.empty(rl, n, smax, dtype=torch.float64, device=x_k.device)
    x1o = torch.empty(smax, n1, r2, dtype=torch.float64, device=x_k.device)
    if rank is None:
        rank = torch.empty(1, dtype=torch.int64, device=x_k.device)
    s_st = ctypes.c_int64()
    ws = _ws(tt_enrich_right_workspace_size(rl, n, rx, rz, n1, r2), workspace, x_k.device)
    _check(lib.tt_enrich_right_async(rl, n, rx, rz, n1, r2, float(delta), int(max_rank),
                                     _dev(x_k, "x_k"), _dev(z_k, "z_k"), _dev(x_k1, "x_k1"),
                                     _dev(xo, "x_k_out"), _dev(x1o, "x_k1_out"), ctypes.byref(s_st),
                                     rank.data_ptr(), ws.data_ptr(), ws.numel(), _stream(stream)))
    return xo, x1o, rank


def tt_round_workspace_size(n, r) -> int:
    a64 = lambda v: (ctypes.c_int64 * len(v))(*v)
    return int(lib.tt_round_workspace_size(len(n), a64(n), a64(r)))


def tt_debug_svd(B, stream=None):
    """Test hook: one-sided Jacobi SVD of B (rows x c, <= 256) in one thread-block cluster.
    Returns (BJ, J, sigma, sweeps) with B J = BJ (columns u_j sigma_j, unsorted)."""
    rows, c = B.shape
    Bc = B.contiguous()
    BJ = torch.empty_like(Bc)
    J = torch.empty((c, c), dtype=torch.float64, device=B.device)
    sig = torch.empty(c, dtype=torch.float64, device=B.device)
    sw = torch.zeros(1, dtype=torch.int32, device=B.device)
    _check(lib.tt_debug_svd(rows, c, _dev(Bc, "B"), _dev(BJ, "BJ"), _dev(J, "J"), _dev(sig, "sigma"),
                            sw.data_ptr(), _stream(stream)))
    return BJ, J, sig, sw


def tt_debug_sym_eigen(G, stream=None):
    """Eigendecomposition of a symmetric CUDA float64 matrix by the rounding's Jacobi solver.
    Returns (lam descending, V)."""
    n = int(G.shape[0])
    Gc = G.clone()
    V = torch.empty_like(Gc)
    lam = torch.empty(n, dtype=torch.float64, device=G.device)
    npe, npb = (n + 1) // 2 * 2, (n + 63) // 64 * 64
    elems = max(4 * npe * npe, 2 * npb * npb + 64 * npb) + 2 * 4096 + 8
    ws = torch.empty(elems * 8, dtype=torch.uint8, device=G.device)
    _check(lib.tt_debug_sym_eigen(n, _dev(Gc, "G"), _dev(V, "V"), _dev(lam, "lam"), ws.data_ptr(),
                                  ws.numel(), _stream(stream)))
    return lam, V
