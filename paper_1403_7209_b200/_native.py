"""ctypes binding of ``libmeshloop_b200.so`` (the C ABI in include/meshloop_b200.h).

The library is loaded from the package directory (built in-tree by
``_build.py`` / ``__graft_entry__.build()``).  Loading fails loudly: there is
no fallback implementation of anything this module exposes.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import numpy as np

from .core import ExecError

_LIB_PATH = Path(__file__).resolve().parent / "libmeshloop_b200.so"
_lib = None
_lock = threading.Lock()

ML_DIRECT, ML_INDIRECT, ML_GLOBAL = 0, 1, 2
MODE_CODE = {"READ": 0, "WRITE": 1, "RW": 2, "INC": 3, "MIN": 4, "MAX": 5}
ML_F64, ML_I64 = 0, 1
ML_AOS, ML_SOA = 0, 1

ML_STREAM_COMPUTE, ML_STREAM_H2D, ML_STREAM_D2H = 0, 1, 2

#: every symbol include/meshloop_b200.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "ml_last_error", "ml_version", "ml_init", "ml_device_info", "ml_synchronize",
    "ml_alloc", "ml_free", "ml_host_alloc", "ml_host_free", "ml_upload", "ml_download",
    "ml_memset", "ml_upload2d", "ml_download2d", "ml_map_upload", "ml_copy_h2d", "ml_copy_d2h",
    "ml_copy_h2d_2d", "ml_copy_d2h_2d", "ml_seg_copy", "ml_seg_params", "ml_order", "ml_sync_all",
    "ml_plan_build", "ml_plan_sizes", "ml_plan_export", "ml_plan_free",
    "ml_gather_build", "ml_gather_export", "ml_gather_free",
    "ml_co_occurrence", "ml_cm_order",
    "ml_functor_lookup", "ml_functor_signature", "ml_functor_count", "ml_functor_name", "ml_chain_lookup",
    "ml_functor_rec_cols",
    "ml_loop_scratch_bytes", "ml_loop_run", "ml_loop_pfold_slot_bytes",
    "ml_program_create", "ml_program_run", "ml_program_replay", "ml_program_loop_times",
    "ml_program_replay_timed",
    "ml_program_free", "ml_program_set_concurrent", "ml_program_deps",
    "ml_pack_rows", "ml_unpack_rows", "ml_combine_ranks", "ml_stream",
    "ml_ipc_handle", "ml_ipc_open", "ml_ipc_close", "ml_put_rows", "ml_wait_flag", "ml_signal_flag",
    "ml_reduce_put", "ml_reduce_fold",
    "ml_flush_l2", "ml_timer_create", "ml_timer_start", "ml_timer_stop", "ml_timer_free",
]


class MlArg(C.Structure):
    _fields_ = [("kind", C.c_int32), ("mode", C.c_int32), ("dim", C.c_int32),
                ("dtype", C.c_int32), ("layout", C.c_int32), ("slot", C.c_int32),
                ("data", C.c_void_p), ("map", C.c_void_p), ("map_from", C.c_int64),
                ("set_size", C.c_int64), ("pitch", C.c_int64), ("seg_shift", C.c_int32)]


class MlPlanDev(C.Structure):
    _fields_ = [("nblocks", C.c_int64), ("ncolors", C.c_int64), ("block_size", C.c_int64),
                ("color_offsets", C.POINTER(C.c_int64)), ("blocks", C.c_void_p),
                ("elem_color", C.c_void_p), ("elem_ncolors", C.c_void_p)]


MAX_ARGS = 16


class MlLoop(C.Structure):
    _fields_ = [("name", C.c_char_p), ("functor", C.c_int32), ("nargs", C.c_int32),
                ("args", C.POINTER(MlArg)), ("n", C.c_int64), ("plan", MlPlanDev),
                ("fconst", C.c_double * 4), ("iconst", C.c_int64 * 4), ("scratch", C.c_void_p),
                ("rlim", C.c_int64),
                ("gather_ntargets", C.c_int64), ("gather_off", C.c_void_p),
                ("gather_elem", C.c_void_p), ("gather_pos", C.c_void_p),
                ("gather_targets", C.c_void_p),
                ("gather_seg", C.c_void_p), ("gather_part", C.c_void_p), ("gather_nhub", C.c_int64),
                ("gather_hub_tl", C.c_void_p), ("gather_hub_off", C.c_void_p),
                ("pf_n1", C.c_int64), ("pf_off1", C.c_void_p), ("pf_elem1", C.c_void_p),
                ("pf_tl1", C.c_void_p), ("pf_n2", C.c_int64), ("pf_off2", C.c_void_p),
                ("pf_elem2", C.c_void_p), ("pf_tl2", C.c_void_p), ("pf_pos2", C.c_void_p),
                ("pf_slots", C.c_void_p), ("pf_slotpos", C.c_void_p),
                ("pf_ncol", C.c_int32), ("pf_rec", C.c_void_p),
                ("pf_rcol", C.c_int8 * 16),
                ("pf_seg1", C.c_void_p), ("pf_seg2", C.c_void_p), ("pf_part1", C.c_void_p),
                ("pf_part2", C.c_void_p), ("pf_nhub1", C.c_int64), ("pf_nhub2", C.c_int64),
                ("pf_hub1_tl", C.c_void_p), ("pf_hub1_off", C.c_void_p), ("pf_hub2_tl", C.c_void_p),
                ("pf_hub2_off", C.c_void_p), ("colour_begin", C.c_int32), ("colour_end", C.c_int32),
                ("rec_fixed", C.c_int32)]


class MlDeviceInfo(C.Structure):
    _fields_ = [("name", C.c_char * 128), ("sm_count", C.c_int32), ("cc_major", C.c_int32),
                ("cc_minor", C.c_int32), ("l2_bytes", C.c_int64), ("hbm_bytes", C.c_int64)]


_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)

_SIGNATURES = {
    "ml_last_error": (C.c_char_p, []),
    "ml_version": (C.c_int, []),
    "ml_init": (C.c_int, [C.c_int]),
    "ml_device_info": (C.c_int, [C.POINTER(MlDeviceInfo)]),
    "ml_synchronize": (C.c_int, []),
    "ml_alloc": (C.c_int, [C.c_uint64, _PP]),
    "ml_free": (C.c_int, [_P]),
    "ml_host_alloc": (C.c_int, [C.c_uint64, _PP]),
    "ml_host_free": (C.c_int, [_P]),
    "ml_upload": (C.c_int, [_P, _P, C.c_uint64]),
    "ml_download": (C.c_int, [_P, _P, C.c_uint64]),
    "ml_memset": (C.c_int, [_P, C.c_int, C.c_uint64]),
    "ml_upload2d": (C.c_int, [_P, C.c_uint64, _P, C.c_uint64, C.c_uint64, C.c_uint64]),
    "ml_download2d": (C.c_int, [_P, C.c_uint64, _P, C.c_uint64, C.c_uint64, C.c_uint64]),
    "ml_copy_h2d_2d": (C.c_int, [_P, C.c_uint64, _P, C.c_uint64, C.c_uint64, C.c_uint64]),
    "ml_copy_d2h_2d": (C.c_int, [_P, C.c_uint64, _P, C.c_uint64, C.c_uint64, C.c_uint64]),
    "ml_seg_copy": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "ml_seg_params": (C.c_int, [_I32P, _I32P, _I32P, _I32P]),
    "ml_map_upload": (C.c_int, [_P, _P, C.c_int64, C.c_int32]),
    "ml_copy_h2d": (C.c_int, [_P, _P, C.c_uint64]),
    "ml_copy_d2h": (C.c_int, [_P, _P, C.c_uint64]),
    "ml_order": (C.c_int, [C.c_int32, C.c_int32]),
    "ml_sync_all": (C.c_int, []),
    "ml_plan_build": (C.c_int, [C.c_int64, C.c_int32, _PP, _I32P, C.c_int64, _PP]),
    "ml_plan_sizes": (C.c_int, [_P, _I64P, _I64P, _I64P]),
    "ml_plan_export": (C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "ml_plan_free": (C.c_int, [_P]),
    "ml_gather_build": (C.c_int, [C.c_int64, C.c_int32, _PP, C.c_int64, _PP]),
    "ml_gather_export": (C.c_int, [_P, _P, _P, _P]),
    "ml_gather_free": (C.c_int, [_P]),
    "ml_co_occurrence": (C.c_int, [C.c_int64, C.c_int32, _PP, _I64P, _I32P, _P, _P, _I64P]),
    "ml_cm_order": (C.c_int, [C.c_int64, _P, _P, _P]),
    "ml_functor_lookup": (C.c_int, [C.c_char_p, C.c_int32, _I32P]),
    "ml_functor_signature": (C.c_int, [C.c_int32, _I32P, _I32P, _I32P, _I32P, _I32P]),
    "ml_functor_count": (C.c_int, [_I32P]),
    "ml_chain_lookup": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int32, _I32P, _P, _I32P, _P]),
    "ml_functor_rec_cols": (C.c_int, [C.c_int32, _P, _I32P]),
    "ml_functor_name": (C.c_int, [C.c_int32, C.c_char_p, C.c_int32, _I32P]),
    "ml_loop_scratch_bytes": (C.c_int, [C.POINTER(MlLoop), C.POINTER(C.c_uint64)]),
    "ml_loop_run": (C.c_int, [C.POINTER(MlLoop)]),
    "ml_loop_pfold_slot_bytes": (C.c_int, [C.POINTER(MlLoop), C.POINTER(C.c_uint64)]),
    "ml_program_create": (C.c_int, [C.POINTER(MlLoop), C.c_int32, _P, _P, C.c_uint64, _PP]),
    "ml_program_run": (C.c_int, [_P, C.c_int32, C.c_int32]),
    "ml_program_replay": (C.c_int, [_P, C.c_int32]),
    "ml_program_loop_times": (C.c_int, [_P, C.POINTER(C.c_float)]),
    "ml_program_replay_timed": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_float)]),
    "ml_program_set_concurrent": (C.c_int, [_P, C.c_int32]),
    "ml_program_deps": (C.c_int, [_P, C.c_int32, _I32P, _P, _I32P]),
    "ml_program_free": (C.c_int, [_P]),
    "ml_pack_rows": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int32, C.c_int64, C.c_int64]),
    "ml_unpack_rows": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int32, C.c_int64, C.c_int64]),
    "ml_combine_ranks": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "ml_stream": (C.c_void_p, []),
    "ml_ipc_handle": (C.c_int, [_P, _P]),
    "ml_ipc_open": (C.c_int, [_P, _PP]),
    "ml_ipc_close": (C.c_int, [_P]),
    "ml_put_rows": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int32, C.c_int64, C.c_int64, _P, _P]),
    "ml_wait_flag": (C.c_int, [_P, _P, C.c_uint64, _P, C.c_int64]),
    "ml_signal_flag": (C.c_int, [_P]),
    "ml_reduce_put": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, C.c_int32, C.c_uint64, _P, C.c_int64]),
    "ml_reduce_fold": (C.c_int, [_P, _P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64,
                                 _P, C.c_int64]),
    "ml_flush_l2": (C.c_int, []),
    "ml_timer_create": (C.c_int, [_PP]),
    "ml_timer_start": (C.c_int, [_P]),
    "ml_timer_stop": (C.c_int, [_P, C.POINTER(C.c_float)]),
    "ml_timer_free": (C.c_int, [_P]),
}


def lib_path() -> Path:
    return _LIB_PATH


def lib():
    """The loaded library; raises ExecError if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise ExecError(f"{_LIB_PATH.name} is not built: run "
                                f"`python -c 'import __graft_entry__ as g; g.build()'` "
                                f"(the B200 backend has no CPU fallback)")
            handle = C.CDLL(str(_LIB_PATH))
            for name, (res, argt) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = argt
            _lib = handle
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().ml_last_error().decode(errors="replace")
        raise ExecError(f"{what}: {msg}" if what else msg)


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


_inited = {}


def init(device: int = 0) -> None:
    if _inited.get("device") == device:
        return
    check(lib().ml_init(device), "ml_init")
    _inited["device"] = device


def device_info() -> dict:
    info = MlDeviceInfo()
    check(lib().ml_device_info(C.byref(info)), "ml_device_info")
    return {"name": info.name.decode(), "sm_count": info.sm_count,
            "cc": (info.cc_major, info.cc_minor), "l2_bytes": info.l2_bytes,
            "hbm_bytes": info.hbm_bytes}


class DeviceBuffer:
    """A device allocation owned by the library (freed with the object)."""

    __slots__ = ("ptr", "nbytes", "__weakref__")

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        check(lib().ml_alloc(int(nbytes), C.byref(p)), f"ml_alloc({nbytes})")
        self.ptr = p.value or 0
        self.nbytes = int(nbytes)

    def upload(self, host: np.ndarray) -> None:
        host = np.ascontiguousarray(host)
        assert host.nbytes <= self.nbytes
        check(lib().ml_upload(self.ptr, ptr(host), host.nbytes), "ml_upload")

    def download(self, host: np.ndarray) -> None:
        assert host.flags.c_contiguous and host.nbytes <= self.nbytes
        check(lib().ml_download(ptr(host), self.ptr, host.nbytes), "ml_download")

    def __del__(self):
        if self.ptr and _lib is not None:
            _lib.ml_free(self.ptr)
            self.ptr = 0


class PinnedArray:
    """A pinned host buffer exposed as a numpy array."""

    def __init__(self, shape, dtype):
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        p = C.c_void_p()
        check(lib().ml_host_alloc(max(nbytes, 8), C.byref(p)), "ml_host_alloc")
        self._ptr = p.value
        buf = (C.c_char * max(nbytes, 8)).from_address(self._ptr)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def __del__(self):
        if getattr(self, "_ptr", None) and _lib is not None:
            _lib.ml_host_free(self._ptr)
            self._ptr = None


def functor_table() -> list[tuple[str, int]]:
    n = C.c_int32()
    check(lib().ml_functor_count(C.byref(n)))
    out = []
    buf = C.create_string_buffer(128)
    for i in range(n.value):
        dt = C.c_int32()
        check(lib().ml_functor_name(i, buf, 128, C.byref(dt)))
        out.append((buf.value.decode(), dt.value))
    return out


def seg_params() -> tuple[int, int, int, int]:
    """(segment shift, component pad, widest and narrowest segmented dim) of
    the library's segmented SOA copies."""
    sh, pad, mx, mn = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    check(lib().ml_seg_params(C.byref(sh), C.byref(pad), C.byref(mx), C.byref(mn)), "ml_seg_params")
    return sh.value, pad.value, mx.value, mn.value
