"""ctypes loader for libflowbb_b200.so (the C-ABI of include/flowbb_b200.h)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libflowbb_b200.so")
# FBB_LIB: an alternative build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("FBB_LIB", LIB_PATH)

FBB_OK = 0
FBB_E_ARG = -1
FBB_E_CUDA = -2
FBB_E_RANGE = -3
FBB_E_NOMEM = -4
FBB_E_STATE = -5

EXPORTED = (
    "fbb_create", "fbb_destroy", "fbb_last_error", "fbb_descriptor", "fbb_bound",
    "fbb_bound_device", "fbb_synth_pool", "fbb_expand_bound_prune", "fbb_explorer_reset",
    "fbb_explorer_start_solve", "fbb_explorer_run", "fbb_explorer_state",
    "fbb_explorer_pending", "fbb_explorer_set_residency", "fbb_explorer_set_incumbent",
    "fbb_explorer_best", "fbb_explorer_take", "fbb_explorer_push", "fbb_tuner_create", "fbb_tuner_destroy", "fbb_tuner_target",
    "fbb_tuner_observe", "fbb_tuner_phase", "fbb_tuner_best_batch",
    "fbb_tuner_best_throughput", "fbb_tuner_set_trace", "fbb_version", "fbb_kernels",
    "fbb_group_create", "fbb_group_destroy", "fbb_group_size", "fbb_group_context",
    "fbb_group_last_error", "fbb_group_reset", "fbb_group_start_solve", "fbb_group_run",
    "fbb_group_best", "fbb_plan_transfers",
)


class BackendError(RuntimeError):
    """backend.hpp:19-25 BackendError: a device fault, with the device index."""

    def __init__(self, backend: int, what: str, status: int = FBB_E_CUDA):
        super().__init__(f"backend {backend}: {what}")
        self.backend = backend
        self.status = status


class Descriptor(C.Structure):
    _fields_ = [("grain", C.c_int32), ("base_units", C.c_int32), ("max_batch", C.c_int64)]


class RoundRec(C.Structure):
    """fbb_round_t"""

    _fields_ = [
        ("target", C.c_int64),
        ("branched", C.c_int64),
        ("bounded", C.c_int64),
        ("inserted", C.c_int64),
        ("pruned", C.c_int64),
        ("leaves", C.c_int64),
        ("incumbent", C.c_int32),
        ("k2_ms", C.c_float),
        ("pending", C.c_int64),
        ("round_ms", C.c_float),
        ("launches", C.c_int32),
        ("host_ms", C.c_float),
        ("sync_ms", C.c_float),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("place_ms", C.c_float),
        ("reserved", C.c_int32),
    ]

    def timing(self):
        return {"k2_ms": self.k2_ms, "round_ms": self.round_ms, "launches": self.launches,
                "host_ms": self.host_ms, "sync_ms": self.sync_ms, "h2d_bytes": self.h2d_bytes,
                "d2h_bytes": self.d2h_bytes, "place_ms": self.place_ms}

    def as_tuple(self):
        return (self.target, self.branched, self.bounded, self.inserted, self.pruned,
                self.leaves, self.incumbent, self.pending)


class GroupStats(C.Structure):
    """fbb_group_stats_t"""

    _fields_ = [("steps", C.c_int64), ("rounds", C.c_int64), ("branched", C.c_int64),
                ("bounded", C.c_int64), ("pruned", C.c_int64), ("leaves", C.c_int64),
                ("pending", C.c_int64), ("transfers", C.c_int64), ("incumbent", C.c_int32),
                ("found", C.c_int32), ("seconds", C.c_double), ("device_ms_max", C.c_double),
                ("exchange_ms", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_vp = C.c_void_p
# fbb_tuner_trace_fn(user, window, batch, throughput, decision)
TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_char_p)

_lib = None


def load_library(path: str = LIB_PATH):
    """Loads the product library; raises OSError (loudly) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g;"
                      f" g.build()'` (no CPU fallback exists)")
    L = C.CDLL(path)
    L.fbb_create.argtypes = [C.c_int, _i32p, C.c_int, C.c_int]
    L.fbb_create.restype = _vp
    L.fbb_destroy.argtypes = [_vp]
    L.fbb_destroy.restype = None
    L.fbb_last_error.argtypes = [_vp, C.POINTER(C.c_int), C.c_char_p, C.c_size_t]
    L.fbb_last_error.restype = C.c_int
    L.fbb_descriptor.argtypes = [_vp, C.POINTER(Descriptor)]
    L.fbb_bound.argtypes = [_vp, _u64p, _i32p, _i32p, C.c_int64, _i32p]
    L.fbb_bound_device.argtypes = [_vp, _vp, _vp, _vp, C.c_int64, _vp, _vp]
    L.fbb_synth_pool.argtypes = [_vp, C.c_uint64, C.c_int64, C.c_int32, C.c_int32, _vp, _vp, _vp,
                                 _vp, _vp]
    L.fbb_expand_bound_prune.argtypes = [
        _vp, _u64p, _i32p, _i32p, _u8p, C.c_int64, C.c_int32, C.c_int, _u64p, _i32p, _i32p, _u8p,
        _i32p, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int64), _i32p,
        C.POINTER(RoundRec)]
    L.fbb_explorer_reset.argtypes = [_vp, _u8p, _i32p, C.c_int64, C.c_int32, C.c_int]
    L.fbb_explorer_set_residency.argtypes = [_vp, C.c_int]
    L.fbb_explorer_set_incumbent.argtypes = [_vp, C.c_int32]
    L.fbb_explorer_best.argtypes = [_vp, C.POINTER(C.c_int32), _i32p]
    L.fbb_explorer_take.argtypes = [_vp, C.c_int64, _u8p, _i32p, C.POINTER(C.c_int64)]
    L.fbb_explorer_push.argtypes = [_vp, _u8p, _i32p, C.c_int64]
    L.fbb_explorer_start_solve.argtypes = [_vp, C.c_int32, C.POINTER(RoundRec)]
    L.fbb_explorer_run.argtypes = [_vp, _i64p, C.c_int, C.c_int64, C.c_int64, _vp,
                                   C.POINTER(C.c_int64)]
    L.fbb_explorer_state.argtypes = [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32), _i32p,
                                     C.POINTER(C.c_int64), _i64p]
    L.fbb_explorer_pending.argtypes = [_vp, _u8p, _i32p, C.c_int64, C.POINTER(C.c_int64)]
    L.fbb_tuner_create.argtypes = [C.c_int32, C.c_int32, C.c_int64, C.c_int, C.c_int]
    L.fbb_tuner_create.restype = _vp
    L.fbb_tuner_destroy.argtypes = [_vp]
    L.fbb_tuner_destroy.restype = None
    L.fbb_tuner_target.argtypes = [_vp]
    L.fbb_tuner_target.restype = C.c_int64
    L.fbb_tuner_observe.argtypes = [_vp, C.c_int64, C.c_double]
    L.fbb_tuner_phase.argtypes = [_vp]
    L.fbb_tuner_best_batch.argtypes = [_vp]
    L.fbb_tuner_best_batch.restype = C.c_int64
    L.fbb_tuner_best_throughput.argtypes = [_vp]
    L.fbb_tuner_best_throughput.restype = C.c_double
    L.fbb_version.restype = C.c_char_p
    L.fbb_kernels.argtypes = [_vp, C.c_char_p, C.c_size_t]
    L.fbb_tuner_set_trace.argtypes = [_vp, TRACE_FN, _vp]
    L.fbb_group_create.argtypes = [_i32p, C.c_int, _i32p, C.c_int, C.c_int]
    L.fbb_group_create.restype = _vp
    L.fbb_group_destroy.argtypes = [_vp]
    L.fbb_group_destroy.restype = None
    L.fbb_group_size.argtypes = [_vp]
    L.fbb_group_context.argtypes = [_vp, C.c_int]
    L.fbb_group_context.restype = _vp
    L.fbb_group_last_error.argtypes = [_vp, C.POINTER(C.c_int), C.c_char_p, C.c_size_t]
    L.fbb_group_reset.argtypes = [_vp, _u8p, _i32p, C.c_int64, C.c_int32, C.c_int]
    L.fbb_group_start_solve.argtypes = [_vp, C.c_int32]
    L.fbb_group_run.argtypes = [_vp, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int64,
                                C.POINTER(GroupStats)]
    L.fbb_group_best.argtypes = [_vp, C.POINTER(C.c_int32), _i32p]
    L.fbb_plan_transfers.argtypes = [_i64p, C.c_int, C.c_int64, C.c_int64, _i64p, C.POINTER(C.c_int)]
    _lib = L
    return L


def last_error(ctx) -> tuple[int, int, str]:
    L = load_library()
    dev = C.c_int(-1)
    buf = C.create_string_buffer(512)
    status = L.fbb_last_error(ctx, C.byref(dev), buf, 512)
    return status, dev.value, buf.value.decode(errors="replace")


def check(ctx, rc: int, backend: int = 0) -> None:
    if rc != FBB_OK:
        status, dev, msg = last_error(ctx)
        if status == FBB_E_ARG:
            raise ValueError(msg)
        raise BackendError(dev if dev >= 0 else backend, msg, status)
