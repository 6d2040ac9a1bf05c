"""ctypes binding of the in-tree C-ABI library ``libseghull_b200.so``
(declarations: include/seghull_b200.h).

There is no CPU fallback: if the library (or a CUDA device) is missing,
every hull call raises.
"""

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# SH_LIB: an alternative build of the same library (tuning experiments)
LIB_PATH = os.environ.get("SH_LIB") or os.path.join(_HERE, "libseghull_b200.so")
CSRC = os.path.join(_HERE, "csrc")

SH_OK, SH_CONTRACT, SH_EMPTY, SH_DEGENERATE, SH_ROUND_GUARD, SH_NOMEM, SH_CUDA = 0, 1, 2, 3, 4, 5, 10
SH_FLAG_COLLINEAR = 1

EXPORTED = ("sh_create", "sh_destroy", "sh_hull2d", "sh_hull3d", "sh_hull2d_async",
            "sh_hull3d_async", "sh_fetch", "sh_trace", "sh_reserve", "sh_hypot_host",
            "sh_set_launch_mode", "sh_launch_times", "sh_filter_stats", "sh_bbox", "sh_segmented_scan", "sh_flag_permute",
            "sh_compact", "sh_scatter", "sh_orient_host", "sh_workspace_bytes", "sh_uniform_points", "sh_facet_stats",
            "sh_stats", "sh_stats_reduce", "sh_set_shard", "sh_hull_shard_begin", "sh_hull_shard_end",
            "sh_order_hull_2d", "sh_giftwrap_2d", "sh_set_filter_share",
            "sh_last_error", "sh_version")
SH_STATS, SH_SHARD_EPS, SH_SHARD_SPLIT = 14, 1, 2


class ShResult(ctypes.Structure):
    _fields_ = [("h", ctypes.c_int64), ("iterations", ctypes.c_int64),
                ("candidates", ctypes.c_int64), ("pruned", ctypes.c_int64),
                ("facets", ctypes.c_int64), ("status", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("eps", ctypes.c_double)]


_lib = None
_lock = threading.RLock()


def build(force=False):
    """Compile the CUDA library in-tree for sm_100a (nvcc cross-compiles
    without a GPU)."""
    cmd = ["make", "-s", "-C", CSRC]
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(cmd, check=True)
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `make -C {CSRC}` "
                    "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
            L.sh_create.argtypes = [ctypes.c_int, ctypes.POINTER(P)]
            L.sh_create.restype = ctypes.c_int
            L.sh_destroy.argtypes = [P]
            L.sh_destroy.restype = None
            L.sh_hull2d.argtypes = [P, P, P, I64, I64, D, D, P, ctypes.POINTER(ShResult), P]
            L.sh_hull2d.restype = ctypes.c_int
            L.sh_hull3d.argtypes = [P, P, P, P, I64, I64, D, D, P, P, I64,
                                    ctypes.POINTER(ShResult), P]
            L.sh_hull3d.restype = ctypes.c_int
            L.sh_hull2d_async.argtypes = [P, P, P, I64, I64, D, D, P, P]
            L.sh_hull2d_async.restype = ctypes.c_int
            L.sh_hull3d_async.argtypes = [P, P, P, P, I64, I64, D, D, P, P, I64, P]
            L.sh_hull3d_async.restype = ctypes.c_int
            L.sh_fetch.argtypes = [P, ctypes.POINTER(ShResult), P]
            L.sh_fetch.restype = ctypes.c_int
            L.sh_trace.argtypes = [P, P, P, P, P, I64]
            L.sh_trace.restype = I64
            L.sh_reserve.argtypes = [P, ctypes.c_int, I64]
            L.sh_reserve.restype = ctypes.c_int
            L.sh_hypot_host.argtypes = [P, P, P, I64]
            L.sh_hypot_host.restype = None
            L.sh_set_launch_mode.argtypes = [P, ctypes.c_int]
            L.sh_set_launch_mode.restype = ctypes.c_int
            L.sh_launch_times.argtypes = [P, P, P, I64]
            L.sh_launch_times.restype = I64
            L.sh_bbox.argtypes = [P, P, P, P, I64, I64, ctypes.c_int, P, P]
            L.sh_bbox.restype = ctypes.c_int
            L.sh_segmented_scan.argtypes = [P, P, ctypes.c_int, P, I64, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, P, P]
            L.sh_segmented_scan.restype = ctypes.c_int
            L.sh_flag_permute.argtypes = [P, P, P, I64, I64, P, P, P]
            L.sh_flag_permute.restype = ctypes.c_int
            L.sh_compact.argtypes = [P, P, P, I64, P, ctypes.POINTER(I64), P, P]
            L.sh_compact.restype = ctypes.c_int
            L.sh_scatter.argtypes = [P, P, I64, P, P, I64, I64, P, P]
            L.sh_scatter.restype = ctypes.c_int
            L.sh_orient_host.argtypes = [ctypes.c_int, P, P, I64, ctypes.c_int, P]
            L.sh_orient_host.restype = ctypes.c_int
            L.sh_uniform_points.argtypes = [P, ctypes.c_int, I64, ctypes.c_uint64, I64, ctypes.c_int, P, P]
            L.sh_uniform_points.restype = ctypes.c_int
            L.sh_workspace_bytes.argtypes = [ctypes.c_int, I64]
            L.sh_workspace_bytes.restype = I64
            L.sh_facet_stats.argtypes = [P, P, I64]
            L.sh_facet_stats.restype = ctypes.c_int
            L.sh_filter_stats.argtypes = [P, P, I64]
            L.sh_filter_stats.restype = ctypes.c_int
            L.sh_stats.argtypes = [P, P, P, P, I64, I64, ctypes.c_int, I64, P, P]
            L.sh_stats.restype = ctypes.c_int
            L.sh_stats_reduce.argtypes = [P, P, ctypes.c_int, ctypes.c_int, P, P]
            L.sh_stats_reduce.restype = ctypes.c_int
            L.sh_set_shard.argtypes = [P, P, I64, ctypes.c_int]
            L.sh_set_shard.restype = ctypes.c_int
            L.sh_hull_shard_begin.argtypes = [P, ctypes.c_int, P, P, P, I64, I64, D, D, I64, P, P]
            L.sh_hull_shard_begin.restype = ctypes.c_int
            L.sh_hull_shard_end.argtypes = [P, P, ctypes.c_int, P, ctypes.POINTER(ShResult), P]
            L.sh_hull_shard_end.restype = ctypes.c_int
            L.sh_set_filter_share.argtypes = [P, ctypes.c_int, ctypes.c_int]
            L.sh_set_filter_share.restype = ctypes.c_int
            L.sh_order_hull_2d.argtypes = [P, P, P, I64, P, P]
            L.sh_order_hull_2d.restype = ctypes.c_int
            L.sh_giftwrap_2d.argtypes = [P, P, P, I64, D, P, I64, ctypes.POINTER(I64), P]
            L.sh_giftwrap_2d.restype = ctypes.c_int
            L.sh_last_error.argtypes = []
            L.sh_last_error.restype = ctypes.c_char_p
            L.sh_version.argtypes = []
            L.sh_version.restype = ctypes.c_char_p
            _lib = L
        return _lib


def last_error():
    return lib().sh_last_error().decode()


_ctx = {}
_dev_locks = {}


def device_lock(device: int):
    """The lock serialising use of a device's context: a context (workspace,
    pinned parameter mirror, captured graphs) is not thread-safe, so every
    hull call holds it (including the hull + trace pair of quickhull_3d)."""
    with _lock:
        lk = _dev_locks.get(device)
        if lk is None:
            lk = _dev_locks[device] = threading.RLock()
        return lk


def context(device: int):
    """One C-ABI context per device (workspace + captured CUDA graphs),
    created once under the lock."""
    with _lock:
        c = _ctx.get(device)
        if c is None:
            h = ctypes.c_void_p()
            rc = lib().sh_create(device, ctypes.byref(h))
            if rc != SH_OK:
                raise RuntimeError(f"sh_create failed ({rc}): {last_error()}")
            c = _ctx[device] = h
        return c
