"""ctypes binding of libhisvsim.so (the C ABI in include/hisvsim.h).

The library is built in-tree by ``build.build_native()`` (``__graft_entry__
.build()``) into ``paper_2205_06973_b200/_lib/libhisvsim.so``. There is no
fallback: if the library is missing or no B200 is visible, every device
entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import (
    DeviceError,
    PartTooWideForLayoutError,
    QubitCountOutOfRangeError,
)

LIB_PATH = Path(os.environ.get("HISVSIM_LIB") or Path(__file__).resolve().parent / "_lib" / "libhisvsim.so")

HS_OK, HS_ERR_INVALID, HS_ERR_CAPACITY, HS_ERR_CUDA, HS_ERR_TOO_WIDE, HS_ERR_UNSUPPORTED = range(6)
HS_C128, HS_C64 = 0, 1
HS_MAX_STAGED = 24

#: every symbol include/hisvsim.h declares (checked by the CPU test suite)
EXPORTS = (
    "hs_last_error", "hs_abi_version", "hs_engine_create", "hs_engine_destroy",
    "hs_engine_query", "hs_engine_set_options", "hs_program_create", "hs_program_create_from_layout",
    "hs_program_destroy",
    "hs_program_num_parts", "hs_program_num_launches", "hs_program_part_info", "hs_program_initial_layout",
    "hs_program_final_layout",
    "hs_program_bind_scratch",
    "hs_program_jit_error", "hs_jit_cache_stats", "hs_program_fuse_switch",
    "hs_program_dump",
    "hs_program_run", "hs_program_run_graph", "hs_plan_part", "hs_plan_program", "hs_plan_program_layouts", "hs_jit_source", "hs_structure_2x2", "hs_dagp_merge", "hs_part_apply",
    "hs_state_init_basis", "hs_bit_permute", "hs_fp64_peak", "hs_max_abs_diff",
    "hs_pack_segments", "hs_unpack_segments", "hs_pack_segments_range", "hs_unpack_segments_range",
    "hs_unpack_segments_range_from", "hs_group_create", "hs_group_destroy", "hs_group_switch",
    "hs_ipc_get_handle", "hs_ipc_open_handle", "hs_ipc_close", "hs_device_alloc", "hs_device_free", "hs_enable_peer_access",
)


class HsGate(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("num_slots", ctypes.c_int32),
        ("slots", ctypes.c_int32 * 3),
        ("reserved", ctypes.c_int32),
        ("params", ctypes.c_double * 3),
    ]


class HsPart(ctypes.Structure):
    _fields_ = [
        ("num_staged", ctypes.c_int32),
        ("staged", ctypes.c_int32 * HS_MAX_STAGED),
        ("gate_offset", ctypes.c_int32),
        ("num_gates", ctypes.c_int32),
    ]


class HsPartInfo(ctypes.Structure):
    _fields_ = [
        ("tile_bits", ctypes.c_int32),
        ("tile_pos", ctypes.c_int32 * 32),
        ("reg_bits", ctypes.c_int32),
        ("phases", ctypes.c_int32),
        ("instructions", ctypes.c_int32),
        ("dense_gates", ctypes.c_int32),
        ("perm_gates", ctypes.c_int32),
        ("diag_gates", ctypes.c_int32),
        ("swaps_relabelled", ctypes.c_int32),
        ("tiles", ctypes.c_int64),
        ("fp_ops_per_amp", ctypes.c_double),
        ("input_gates", ctypes.c_int32),
        ("restore", ctypes.c_int32),
        ("compiled", ctypes.c_int32),
        ("fp64_instr_per_amp", ctypes.c_float),
        ("user_part", ctypes.c_int32),
    ]


_lib = None
_load_error: str | None = None


def _declare(lib) -> None:
    P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    sig = {
        "hs_last_error": (ctypes.c_char_p, []),
        "hs_abi_version": (I, []),
        "hs_engine_create": (I, [I, ctypes.POINTER(P)]),
        "hs_engine_destroy": (I, [P]),
        "hs_engine_query": (I, [P, ctypes.POINTER(I), ctypes.POINTER(I), ctypes.POINTER(I)]),
        "hs_engine_set_options": (I, [P, ctypes.c_uint32]),
        "hs_program_create": (I, [P, I, I, ctypes.POINTER(HsPart), I,
                                  ctypes.POINTER(HsGate), I, ctypes.POINTER(P)]),
        "hs_program_create_from_layout": (I, [P, I, I, ctypes.POINTER(HsPart), I, ctypes.POINTER(HsGate), I,
                                              ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(P)]),
        "hs_program_destroy": (I, [P]),
        "hs_program_num_parts": (I, [P]),
        "hs_program_num_launches": (I, [P]),
        "hs_program_jit_error": (ctypes.c_char_p, [P]),
        "hs_jit_cache_stats": (I, [ctypes.POINTER(I), ctypes.POINTER(I)]),
        "hs_program_fuse_switch": (I, [P, I, I, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_uint64),
                                       ctypes.c_int32]),
        "hs_program_initial_layout": (I, [P, ctypes.POINTER(ctypes.c_int32)]),
        "hs_program_final_layout": (I, [P, ctypes.POINTER(ctypes.c_int32)]),
        "hs_program_bind_scratch": (I, [P, P, ctypes.c_size_t]),
        "hs_program_part_info": (I, [P, I, ctypes.POINTER(HsPartInfo)]),
        "hs_program_dump": (I, [P, I, P, ctypes.c_size_t, ctypes.POINTER(I),
                                ctypes.POINTER(ctypes.c_size_t)]),
        "hs_program_run": (I, [P, P, I64, I, I, P]),
        "hs_program_run_graph": (I, [P, P, I64, P]),
        "hs_plan_part": (I, [I, I, I, ctypes.c_uint32, ctypes.POINTER(ctypes.c_int32), I, ctypes.POINTER(HsGate), I,
                             P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(HsPartInfo)]),
        "hs_plan_program": (I, [I, I, I, ctypes.c_uint32, ctypes.POINTER(HsPart), I, ctypes.POINTER(HsGate), I,
                                P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(I)]),
        "hs_plan_program_layouts": (I, [I, I, I, ctypes.c_uint32, ctypes.POINTER(HsPart), I, ctypes.POINTER(HsGate),
                                        I, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                        ctypes.POINTER(I)]),
        "hs_jit_source": (I, [I, I, I, ctypes.c_uint32, ctypes.POINTER(ctypes.c_int32), I, ctypes.POINTER(HsGate), I,
                              ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
        "hs_structure_2x2": (I, [ctypes.POINTER(D), I, ctypes.POINTER(D), ctypes.POINTER(D)]),
        "hs_dagp_merge": (I, [I, ctypes.POINTER(ctypes.c_uint64), I, ctypes.POINTER(ctypes.c_int32),
                              ctypes.POINTER(ctypes.c_int32), I, ctypes.POINTER(ctypes.c_int32)]),
        "hs_part_apply": (I, [P, P, I64, I, I, ctypes.POINTER(ctypes.c_int32), I,
                              ctypes.POINTER(HsGate), I, P]),
        "hs_state_init_basis": (I, [P, I64, I, I64, P]),
        "hs_bit_permute": (I, [P, P, I, I, ctypes.POINTER(ctypes.c_int32), P]),
        "hs_fp64_peak": (I, [ctypes.POINTER(D), P]),
        "hs_max_abs_diff": (I, [P, I, P, I64, ctypes.POINTER(D), P]),
        "hs_pack_segments": (I, [P, P, I, I, ctypes.POINTER(ctypes.c_int32), I, P]),
        "hs_unpack_segments": (I, [P, P, I, I, ctypes.POINTER(ctypes.c_int32), I, P]),
        "hs_pack_segments_range": (I, [P, P, I, I, ctypes.POINTER(ctypes.c_int32), I, I64, I64, P]),
        "hs_unpack_segments_range": (I, [P, P, I, I, ctypes.POINTER(ctypes.c_int32), I, I64, I64, P]),
        "hs_unpack_segments_range_from": (I, [ctypes.POINTER(P), P, I, I, ctypes.POINTER(ctypes.c_int32), I, I64, I64,
                                              P]),
        "hs_group_create": (I, [I, ctypes.POINTER(ctypes.c_int32), ctypes.c_size_t, ctypes.POINTER(P)]),
        "hs_group_destroy": (I, [P]),
        "hs_group_switch": (I, [P, ctypes.POINTER(P), I, I, ctypes.POINTER(ctypes.c_int32), I,
                                ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(P),
                                ctypes.POINTER(D)]),
        "hs_ipc_get_handle": (I, [P, P]),
        "hs_ipc_open_handle": (I, [P, ctypes.POINTER(P)]),
        "hs_ipc_close": (I, [P]),
        "hs_device_alloc": (I, [ctypes.c_size_t, ctypes.POINTER(P)]),
        "hs_device_free": (I, [P]),
        "hs_enable_peer_access": (I, [I]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load():
    """The loaded library; raises ``DeviceError`` if it cannot be loaded."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise DeviceError(_load_error)
    if not LIB_PATH.exists():
        _load_error = (
            f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
            "there is no CPU fallback"
        )
        raise DeviceError(_load_error)
    try:
        lib = ctypes.CDLL(os.fspath(LIB_PATH))
        _declare(lib)
    except OSError as exc:  # pragma: no cover - depends on the box
        _load_error = f"cannot load {LIB_PATH}: {exc}"
        raise DeviceError(_load_error) from exc
    _lib = lib
    return lib


def check(status: int) -> None:
    """Raise the error class matching a C-ABI status code."""
    if status == HS_OK:
        return
    msg = load().hs_last_error().decode(errors="replace")
    if status == HS_ERR_INVALID:
        raise ValueError(msg)
    if status == HS_ERR_CAPACITY:
        raise QubitCountOutOfRangeError(msg)
    if status == HS_ERR_TOO_WIDE:
        raise PartTooWideForLayoutError(msg)
    raise DeviceError(msg)


_engines: dict[int, int] = {}


def engine(device: int) -> int:
    """Process-wide engine handle for a CUDA device (created on first use)."""
    h = _engines.get(device)
    if h is None:
        lib = load()
        out = ctypes.c_void_p()
        check(lib.hs_engine_create(device, ctypes.byref(out)))
        h = out.value
        _engines[device] = h
    return h


def engine_query(device: int) -> dict:
    lib = load()
    sms, t128, t64 = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    check(lib.hs_engine_query(engine(device), ctypes.byref(sms), ctypes.byref(t128), ctypes.byref(t64)))
    return {"num_sms": sms.value, "tile_bits_c128": t128.value, "tile_bits_c64": t64.value}


HS_PLAN_FUSE_1Q, HS_PLAN_RB3, HS_PLAN_PARITY, HS_PLAN_LAYOUT, HS_PLAN_JIT = 0x1, 0x2, 0x4, 0x8, 0x10
HS_PLAN_INIT_LAYOUT, HS_PLAN_PINGPONG, HS_PLAN_CLUSTER, HS_PLAN_NO_RESTORE = 0x20, 0x40, 0x80, 0x100
HS_PLAN_PART_LOCAL, HS_PLAN_MERGE, HS_PLAN_GLOBAL_DIAG = 0x200, 0x400, 0x800
HS_PLAN_DEFAULT = HS_PLAN_FUSE_1Q | HS_PLAN_PARITY | HS_PLAN_MERGE | HS_PLAN_GLOBAL_DIAG


def set_options(device: int, options: int) -> None:
    """Planner options (HS_PLAN_* bits) for programs created afterwards."""
    check(load().hs_engine_set_options(engine(device), options))


_default_options = HS_PLAN_DEFAULT


def default_options() -> int:
    """Planner bits new programs use unless they pass their own (programs
    run in part ranges, e.g. between distributed layout switches, drop
    HS_PLAN_LAYOUT)."""
    return _default_options


def set_default_options(options: int) -> None:
    global _default_options
    _default_options = int(options)


def jit_cache_stats() -> dict:
    """Compiled-part kernels loaded from the on-disk cubin cache vs compiled
    with NVRTC so far in this process (hs_jit_cache_stats)."""
    hits, comp = ctypes.c_int(), ctypes.c_int()
    check(load().hs_jit_cache_stats(ctypes.byref(hits), ctypes.byref(comp)))
    return {"disk_hits": hits.value, "compiles": comp.value}
