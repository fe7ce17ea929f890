"""ctypes binding of the C ABI in include/flowplace_b200.h.

This is the binding a maintainer of the reference would add next to
``flowplace/_simcore``.  There is no fallback: if the
CUDA library is missing or no GPU is visible the calls raise.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

from ._build import LIB as _LIB_PATH

FP_OK, FP_ERR_INVALID, FP_ERR_CUDA, FP_ERR_UNSUPPORTED, FP_ERR_DEADLOCK, FP_ERR_OVERFLOW = range(6)
EP_OK, EP_DEADLOCK, EP_TRACE_OVERFLOW, EP_BAD_ACTION = range(4)
FLAG_WIDE = 1  # force the HBM-resident episode path
FLAG_TIE_RANDOM = 2  # teacher mode: random tie-breaks among equal t-levels
FLAG_PER_STEP = 4  # mp_mode="per_step": re-encode before every decision

_lib = None


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        super().__init__(f"flowplace_b200 error {code}: {msg}")


class FpEvent(ctypes.Structure):
    _fields_ = [("time", ctypes.c_double), ("v", ctypes.c_int32), ("kind", ctypes.c_int8),
                ("etype", ctypes.c_int8), ("a", ctypes.c_int8), ("b", ctypes.c_int8)]


EVENT_DTYPE = np.dtype([("time", "<f8"), ("v", "<i4"), ("kind", "i1"), ("etype", "i1"),
                        ("a", "i1"), ("b", "i1")])
assert EVENT_DTYPE.itemsize == ctypes.sizeof(FpEvent) == 16


class FpGraphDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("d", ctypes.c_int32)] + [
        (name, ctypes.c_void_p) for name in (
            "pred_indptr", "pred_indices", "succ_indptr", "succ_indices", "is_entry", "flops",
            "obytes", "rates", "bw", "eslots", "tslots", "tlev", "blev")] + [
        ("comm_factor", ctypes.c_double)]


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        import os

        path = Path(os.environ.get("FLOWPLACE_B200_LIB", str(_LIB_PATH)))
        if not path.exists():
            raise RuntimeError(
                f"CUDA library {path} is not built; run `python -m paper_2505_23131_b200._build`"
                " (or __graft_entry__.build()). There is no CPU fallback.")
        _lib = ctypes.CDLL(str(path))
        _lib.fp_last_error.restype = ctypes.c_char_p
    return _lib


def check(rc: int) -> int:
    if rc != FP_OK:
        raise NativeError(rc, lib().fp_last_error().decode())
    return rc


def ptr(x) -> ctypes.c_void_p:
    """Raw pointer of a numpy array or torch tensor (None -> NULL)."""
    if x is None:
        return ctypes.c_void_p(0)
    if isinstance(x, np.ndarray):
        return ctypes.c_void_p(x.ctypes.data)
    return ctypes.c_void_p(x.data_ptr())


def stream_ptr(stream=None) -> ctypes.c_void_p:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


EXPORTED = (
    "fp_last_error", "fp_version", "fp_problem_create", "fp_problem_destroy",
    "fp_problem_sim_smem", "fp_sim_workspace_size", "fp_sim_batch", "fp_run_packed", "fp_run_packed_cache_clear",
    "fp_jitter_tables", "fp_static_features",
)


PARAM_ROLES = 78
ROLE_BY_HEAD = {
    "sel.z.w": 64, "sel.z.b": 65, "sel.head1.w": 66, "sel.head1.b": 67, "sel.head2.w": 68,
    "sel.head2.b": 69, "plc.z.w": 70, "plc.z.b": 71, "plc.head1.w": 72, "plc.head1.b": 73,
    "plc.head2.w": 74, "plc.head2.b": 75, "plc.y.w": 76, "plc.y.b": 77,
}
MODE = {"sample": 0, "greedy": 1, "forced": 2, "teacher": 3}
TABLE = {"H_sel": 0, "H_plc": 1, "sel_logit": 2, "A": 3, "G": 4, "M": 5, "c": 6}


def gnn_role(enc: int, k: int, r: int) -> int:
    return (enc * 8 + k) * 4 + r


class FpPolicyDesc(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("k_rounds", ctypes.c_int32),
                ("shared_encoder", ctypes.c_int32), ("leaky_slope", ctypes.c_double)] + [
        (name, ctypes.c_void_p) for name in (
            "x_static", "adj_ptr", "adj_src", "adj_edge", "bpath_ptr", "bpath_idx",
            "tpath_ptr", "tpath_idx", "param_offsets")] + [("n_params", ctypes.c_int64),
                                                           ("bnext", ctypes.c_void_p),
                                                           ("tnext", ctypes.c_void_p)]


class FpRolloutArgs(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("mode", ctypes.c_int32), ("epsilon", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("episode_base", ctypes.c_uint32),
                ("strategy", ctypes.c_int32), ("simulate", ctypes.c_int32)] + [
        (name, ctypes.c_void_p) for name in (
            "forced", "assign", "step_vd", "step_lp", "step_ent", "step_argmax", "step_ncand",
            "makespan", "status", "grad_rows", "grad_ep", "trace")] + [
        ("trace_cap", ctypes.c_int32), ("trace_len", ctypes.c_void_p),
        ("flags", ctypes.c_int32), ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_int64)]


EXPORTED = EXPORTED + (
    "fp_policy_create", "fp_policy_destroy", "fp_policy_set_encoder", "fp_policy_prepare", "fp_policy_table",
    "fp_rollout_workspace_size", "fp_rollout_batch", "fp_grad_ep_stride", "fp_grad_rec_stride",
    "fp_pg_reduce", "fp_pg_reduce_per_step", "fp_policy_backward", "fp_sgd_step", "fp_sgd_step_masked",
    "fp_tc_gemm_selftest", "fp_agg_timer_enable", "fp_agg_timer_read",
)


def agg_timer(on: bool) -> None:
    """Bracket every GNN aggregation launch with an event pair on its stream
    (measurement hook for bench.py; fp_agg_timer_enable)."""
    check(lib().fp_agg_timer_enable(ctypes.c_int32(1 if on else 0)))


def agg_timer_read() -> tuple[float, int]:
    """(summed aggregation-kernel ms, launches) since the last read / enable."""
    ms, cnt = ctypes.c_double(), ctypes.c_int64()
    check(lib().fp_agg_timer_read(ctypes.byref(ms), ctypes.byref(cnt)))
    return ms.value, cnt.value
