"""ctypes binding of ``libptsbe.so`` (the C ABI in ``include/ptsbe.h``).

The shared library is built in-tree by ``build.py`` / ``__graft_entry__.build()``.
There is deliberately no fallback: if the library or a GPU is missing, the
engine raises ``ExecutionError`` instead of silently computing on the CPU.
ctypes releases the GIL for every foreign call, so worker threads that each
own a handle run concurrently.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import AnnihilatedStateError, ExecutionError, ValidationError

LIB_NAME = "libptsbe.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

PTSBE_OK = 0
PTSBE_ERR_VALIDATION = 1
PTSBE_ERR_ANNIHILATED = 2
PTSBE_ERR_CUDA = 3
PTSBE_ERR_NCCL = 4

PTSBE_C64 = 0
PTSBE_C128 = 1

PTSBE_DEVICE_PTRS = 0x1
PTSBE_NO_SYNC = 0x2
PTSBE_ZERO_VECTOR = 0x4
PTSBE_CONTINUE = 0x8
PTSBE_KEEP_SEL = 0x10
PTSBE_DEFER_NORMS = 0x20
PTSBE_SHARDED = 0x40
PTSBE_HOST_MIRROR = 0x80

RNG_PCG64 = 0
RNG_PHILOX = 1
RNG_KEYS = 2

TRAJ_OK = 0
TRAJ_ANNIHILATED = 2


class Op(C.Structure):
    _fields_ = [("kind", C.c_int32), ("arity", C.c_int32), ("t0", C.c_int32), ("t1", C.c_int32),
                ("ref", C.c_int32), ("pass_", C.c_int32)]


class Channel(C.Structure):
    _fields_ = [("n_outcomes", C.c_int32), ("mat_base", C.c_int32), ("general", C.c_int32),
                ("arity", C.c_int32), ("identity_mask", C.c_uint64)]


class Pass(C.Structure):
    _fields_ = [("qubit_mask", C.c_uint64), ("tile_bits", C.c_int32), ("low_bits", C.c_int32)]


# every exported symbol with (restype, argtypes); tests check the .so exports each
SIGNATURES = {
    "ptsbe_abi_version": (C.c_int, []),
    "ptsbe_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "ptsbe_destroy": (C.c_int, [C.c_void_p]),
    "ptsbe_load_program": (C.c_int, [C.c_void_p, C.POINTER(Op), C.c_int, C.c_void_p, C.c_int,
                                     C.POINTER(Channel), C.c_int, C.c_void_p, C.c_int,
                                     C.POINTER(Pass), C.c_int]),
    "ptsbe_run_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_uint32]),
    "ptsbe_apply_program": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_uint32]),
    "ptsbe_sample": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]),
    "ptsbe_get_state": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint32]),
    "ptsbe_set_state": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint32]),
    "ptsbe_device_memory": (C.c_int, [C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "ptsbe_set_layout": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ptsbe_run_range": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                  C.c_uint32]),
    "ptsbe_run_conventional": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_uint32]),
    "ptsbe_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "ptsbe_shard_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "ptsbe_shard_swap": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "ptsbe_shard_swap_local": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "ptsbe_slot_norms": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "ptsbe_finalize_norms": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "ptsbe_set_host_mirror": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "ptsbe_get_weights": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "ptsbe_gather_amplitudes": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p]),
    "ptsbe_exchange_half": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int]),
    "ptsbe_norm_totals": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "ptsbe_state_ptr": (C.c_void_p, [C.c_void_p, C.c_int]),
    "ptsbe_plan": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64,
                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "ptsbe_synchronize": (C.c_int, [C.c_void_p]),
    "ptsbe_stream": (C.c_void_p, [C.c_void_p]),
    "ptsbe_info": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "ptsbe_pass_info": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int]),
    "ptsbe_last_error": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "ptsbe_launch_count": (C.c_int64, [C.c_void_p]),
    "ptsbe_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "ptsbe_profile_read": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "ptsbe_profile_bytes": (C.c_double, [C.c_void_p]),
    "ptsbe_profile_passes": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "ptsbe_create_host": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "ptsbe_codegen_source": (C.c_int64, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "ptsbe_format_records": (C.c_int64, [C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_int64]),
}

_lib = None


def load_library(path: str | os.PathLike | None = None):
    """Load and type the shared library once; raise ExecutionError if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise ExecutionError(
            f"{p} is missing: build the CUDA engine first (python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ptsbe_abi_version() != 1:
        raise ExecutionError("libptsbe.so ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def last_error(lib, handle) -> str:
    buf = C.create_string_buffer(512)
    lib.ptsbe_last_error(handle, buf, len(buf))
    return buf.value.decode(errors="replace")


def check(lib, handle, status: int, what: str) -> None:
    """Map a C status onto the reference's exception classes (errors.py:17-25)."""
    if status == PTSBE_OK:
        return
    msg = f"{what}: {last_error(lib, handle)}"
    if status == PTSBE_ERR_VALIDATION:
        raise ValidationError(msg)
    if status == PTSBE_ERR_ANNIHILATED:
        raise AnnihilatedStateError(msg)
    raise ExecutionError(msg)
