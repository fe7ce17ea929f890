"""flowplace/_cudacore.py -- the reference-side binding of the B200 simulator
core (installed into a flowplace tree by integration/install_cuda_backend.py;
see INTEGRATION.md section 1).

Same signature and error behaviour as the Cython core it stands in for,
``_simcore.run_packed`` (flowplace/_simcore.pyx:39-45): borrowed host arrays
in, ``(makespan, [(tkind, v, a, b, time, etype), ...])`` out,
``DeadlockError(time_ms, blocked)`` on a deadlock.  The library call is
``fp_run_packed`` (include/flowplace_b200.h), which caches the packed graph
on the device per host thread, so a caller looping over assignments of one
graph pays one H2D copy, the kernel and the D2H copies per call."""

import ctypes
import os

import numpy as np

from ._simpy import DeadlockError

_LIB_PATH = os.environ.get("FLOWPLACE_B200_LIB", "@FLOWPLACE_B200_LIB@")
_lib = ctypes.CDLL(_LIB_PATH)
_lib.fp_last_error.restype = ctypes.c_char_p
_EV = np.dtype([("time", "<f8"), ("v", "<i4"), ("kind", "i1"), ("etype", "i1"),
                ("a", "i1"), ("b", "i1")])   # fp_event, 16 bytes
_TYPES = (np.int32, np.int32, np.int32, np.int32, np.uint8, np.float64, np.float64, np.int32,
          np.float64, np.float64, np.int32, np.int32, np.float64, np.float64)
FP_ERR_DEADLOCK = 4
_buf = {}


def _events(cap):
    ev = _buf.get(cap)
    if ev is None:
        _buf.clear()
        ev = _buf[cap] = np.empty(cap, dtype=_EV)
    return ev


def run_packed(n, d, pred_indptr, pred_indices, succ_indptr, succ_indices, is_entry, flops,
               obytes, assign, rates, bw, eslots, tslots, tlev, blev, strategy, comm_factor,
               sigma, seed):
    arrs = [np.ascontiguousarray(a, dtype=t) for a, t in zip(
        (pred_indptr, pred_indices, succ_indptr, succ_indices, is_entry, flops, obytes, assign,
         rates, bw, eslots, tslots, tlev, blev), _TYPES)]
    cap = 2 * (n + n * d) + 2
    ev = _events(cap)
    blocked = np.zeros(max(n, 1), dtype=np.uint8)
    mk, ne = ctypes.c_double(), ctypes.c_int64()
    rc = _lib.fp_run_packed(ctypes.c_int32(n), ctypes.c_int32(d),
                            *[ctypes.c_void_p(a.ctypes.data) for a in arrs],
                            ctypes.c_int32(strategy), ctypes.c_double(comm_factor),
                            ctypes.c_double(sigma), ctypes.c_int64(seed), ctypes.byref(mk),
                            ctypes.c_void_p(ev.ctypes.data), ctypes.c_int64(cap),
                            ctypes.byref(ne), ctypes.c_void_p(blocked.ctypes.data))
    if rc == FP_ERR_DEADLOCK:
        raise DeadlockError(mk.value, [int(v) for v in np.flatnonzero(blocked[:n])])
    if rc != 0:
        raise RuntimeError(_lib.fp_last_error().decode())
    e = ev[:ne.value]
    return mk.value, list(zip(e["kind"].tolist(), e["v"].tolist(), e["a"].tolist(),
                              e["b"].tolist(), e["time"].tolist(), e["etype"].tolist()))
