"""ctypes binding of the C ABI in ``include/vfmm.h`` (``libvfmm.so``).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_0809_1810_b200/csrc``).  There is no CPU or Python fallback:
if the library is missing or CUDA is unavailable every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# VFMM_LIB: alternative build of the same library (kernel tuning variants)
LIB_PATH = os.environ.get("VFMM_LIB") or os.path.join(_HERE, "libvfmm.so")

VFMM_OK = 0
VFMM_EINVAL = 1
VFMM_EDOMAIN = 2
VFMM_ECUDA = 3
VFMM_EWORKSPACE = 4

KERNEL_POINT = 0
KERNEL_GAUSSIAN = 1

FLAG_STATS = 1
FLAG_PHASE_TIMES = 64
FLAG_OVERLAP = 2
FLAG_FAR_ONLY = 4
FLAG_PHASE_UP = 8
FLAG_PHASE_DOWN = 16
FLAG_UV_PAIRS = 32
FLAG_SIGMA_SCALAR = 128
FLAG_GRAPH = 256
FLAG_GRAPH_PHASES = 512

ORDER_CAP = 60
LEVELS_CAP = 13

#: every symbol declared in include/vfmm.h
EXPORTED_SYMBOLS = (
    "vfmm_workspace_size",
    "vfmm_layout_of",
    "vfmm_evaluate",
    "vfmm_evaluate_host",
    "vfmm_evaluate_host_streams",
    "vfmm_evaluate_shard",
    "vfmm_shard_exchange_size",
    "vfmm_shard_pack",
    "vfmm_shard_unpack",
    "vfmm_mult_region",
    "vfmm_counts_region",
    "vfmm_read_stats",
    "vfmm_bad_count_async",
    "vfmm_evaluate_at",
    "vfmm_direct_workspace_size",
    "vfmm_direct",
    "vfmm_fp64_probe",
    "vfmm_launch_count",
    "vfmm_graph_phase_times",
    "vfmm_version",
)


class VfmmStats(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("m2l_count", ctypes.c_int64),
        ("near_pair_count", ctypes.c_int64),
        ("levels", ctypes.c_int32),
        ("order", ctypes.c_int32),
        ("sigma_guard_ok", ctypes.c_int32),
        ("bad_count", ctypes.c_int32),
        ("first_bad", ctypes.c_int64),
        ("max_sigma", ctypes.c_double),
        ("sigma_guard", ctypes.c_double),
        ("t_build", ctypes.c_float),
        ("t_upward", ctypes.c_float),
        ("t_m2l", ctypes.c_float),
        ("t_downward", ctypes.c_float),
        ("t_eval", ctypes.c_float),
        ("t_near", ctypes.c_float),
        ("t_total", ctypes.c_float),
        ("overlapped", ctypes.c_int32),
    ]


class VfmmLayout(ctypes.Structure):
    _fields_ = [
        ("perm", ctypes.c_size_t),
        ("leaf_key", ctypes.c_size_t),
        ("leaf_starts", ctypes.c_size_t),
        ("sources", ctypes.c_size_t),
        ("near_uv", ctypes.c_size_t),
        ("mult", ctypes.c_size_t),
        ("loc", ctypes.c_size_t),
        ("leaf_loc", ctypes.c_size_t),
        ("counts", ctypes.c_size_t),
        ("total", ctypes.c_size_t),
    ]


_lock = threading.Lock()
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double
_SZ = ctypes.c_size_t


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load ``libvfmm.so`` and declare the prototypes (no GPU needed to load)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"vfmm CUDA library not built: {path} is missing "
                "(run __graft_entry__.build() or make -C paper_0809_1810_b200/csrc)"
            )
        lib = ctypes.CDLL(path)
        lib.vfmm_workspace_size.argtypes = [_I64, _I, _I, ctypes.POINTER(_SZ)]
        lib.vfmm_layout_of.argtypes = [_I64, _I, _I, ctypes.POINTER(VfmmLayout)]
        lib.vfmm_evaluate.argtypes = [_P, _P, _P, _P, _I64, _D, _D, _D, _I, _I, _I, _P, _P, _P, _SZ,
                                      ctypes.c_uint, ctypes.POINTER(VfmmStats), _P]
        lib.vfmm_evaluate_host.argtypes = lib.vfmm_evaluate.argtypes
        lib.vfmm_evaluate_host_streams.argtypes = [_P, _P, _P, _P, _I64, _D, _D, _D, _I, _I, _I, _P, _P,
                                                   _P, _SZ, ctypes.c_uint, _P, _P, _P]
        lib.vfmm_evaluate_shard.argtypes = [_P, _P, _P, _P, _I64, _D, _D, _D, _I, _I, _I, _I, _I, _P,
                                            _P, _P, _SZ, ctypes.c_uint, ctypes.POINTER(VfmmStats), _P]
        lib.vfmm_shard_exchange_size.argtypes = [_I64, _I, _I, _I, _I, _I, ctypes.POINTER(_SZ),
                                                 ctypes.POINTER(_SZ)]
        lib.vfmm_shard_pack.argtypes = [_I64, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P]
        lib.vfmm_shard_unpack.argtypes = [_I64, _I, _I, _I, _I, _I, _P, _P, _I, _P, _P, _P]
        lib.vfmm_mult_region.argtypes = [_I64, _I, _I, ctypes.POINTER(_SZ), ctypes.POINTER(_SZ)]
        lib.vfmm_counts_region.argtypes = [_I64, _I, _I, ctypes.POINTER(_SZ), ctypes.POINTER(_SZ)]
        lib.vfmm_read_stats.argtypes = [_I64, _I, _I, _I, _D, _P, ctypes.POINTER(VfmmStats), _P]
        lib.vfmm_bad_count_async.argtypes = [_I64, _I, _I, _P, _P, _P]
        lib.vfmm_evaluate_at.argtypes = [_P, _P, _I64, _I64, _D, _D, _D, _I, _I, _I, _P, _P, _P,
                                         ctypes.POINTER(_I64), _P]
        lib.vfmm_direct_workspace_size.argtypes = [_I64, _I64, ctypes.POINTER(_SZ)]
        lib.vfmm_direct.argtypes = [_P, _P, _I64, _P, _P, _P, _P, _I64, _I, _P, _P, _P, _SZ, _P]
        lib.vfmm_fp64_probe.argtypes = [_P, _I, _I, ctypes.POINTER(_D), _P]
        lib.vfmm_version.restype = ctypes.c_char_p
        lib.vfmm_launch_count.argtypes = []
        lib.vfmm_graph_phase_times.argtypes = [_I, ctypes.POINTER(ctypes.c_float)]
        for name in EXPORTED_SYMBOLS:
            if name not in ("vfmm_version", "vfmm_launch_count"):
                getattr(lib, name).restype = _I
        lib.vfmm_launch_count.restype = _I64
        _lib = lib
        return lib


def check(status: int, what: str) -> None:
    if status == VFMM_OK:
        return
    names = {1: "invalid argument", 2: "out of domain", 3: "CUDA error", 4: "workspace too small"}
    raise RuntimeError(f"{what} failed: {names.get(status, status)} (status {status})")


def workspace_size(n: int, levels: int, order: int) -> int:
    out = _SZ()
    check(load().vfmm_workspace_size(n, levels, order, ctypes.byref(out)), "vfmm_workspace_size")
    return out.value


def region(name: str, n: int, levels: int, order: int) -> tuple[int, int]:
    """(offset, bytes) of the 'mult' or 'counts' region of a workspace."""
    off, nbytes = _SZ(), _SZ()
    fn = getattr(load(), f"vfmm_{name}_region")
    check(fn(max(n, 1), levels, order, ctypes.byref(off), ctypes.byref(nbytes)), f"vfmm_{name}_region")
    return off.value, nbytes.value


def layout(n: int, levels: int, order: int) -> VfmmLayout:
    out = VfmmLayout()
    check(load().vfmm_layout_of(n, levels, order, ctypes.byref(out)), "vfmm_layout_of")
    return out
