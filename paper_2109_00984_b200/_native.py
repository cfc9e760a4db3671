"""Loader of the native library libmpc_ring.so (C-ABI in include/mpc_ring.h).

No fallback: a missing or unloadable library raises immediately.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmpc_ring.so")

class ConvGeom(ctypes.Structure):
    """mpc_conv2d_geom (include/mpc_ring.h)."""
    _fields_ = [(f, ctypes.c_int64) for f in ("B", "C", "H", "W", "Cout", "kh", "kw", "sh", "sw", "ph", "pw")]


class Keys(ctypes.Structure):
    """mpc_keys (include/mpc_ring.h): one party's PRZS key pair and, for the dealer, k_ttp."""
    _fields_ = [("przs_self", ctypes.c_uint64), ("przs_prev", ctypes.c_uint64), ("ttp", ctypes.c_uint64),
                ("has_ttp", ctypes.c_int)]


# (name, restype, argtypes); P = void*, I = int, L = int64, U = uint64, S = size_t
_V, _I, _L, _U, _S, _D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_double
SIGNATURES = [
    ("mpc_create", _I, [ctypes.POINTER(_V), _I, _I, _I, _V, _U, _I]),
    ("mpc_derive_keys", _I, [_U, _I, _I, ctypes.POINTER(Keys)]),
    ("mpc_create_with_keys", _I, [ctypes.POINTER(_V), _I, _I, _I, _V, ctypes.POINTER(Keys), _I]),
    ("mpc_destroy", _I, [_V]),
    ("mpc_set_stream", _I, [_V, _V]),
    ("mpc_set_reveal_chunks", _I, [_V, _I]),
    ("mpc_last_error", ctypes.c_char_p, [_V]),
    ("mpc_stats", _I, [_V, ctypes.POINTER(_U), ctypes.POINTER(_U)]),
    ("mpc_world_size", _I, [_V]),
    ("mpc_rank", _I, [_V]),
    ("mpc_nccl_unique_id", _I, [_V]),
    ("mpc_group_create", _I, [ctypes.POINTER(_V), _I]),
    ("mpc_group_destroy", _I, [_V]),
    ("mpc_create_local", _I, [ctypes.POINTER(_V), _V, _I, _I, _U, _I]),
    ("mpc_encode", _I, [_V, _V, _V, _L]),
    ("mpc_encode_async", _I, [_V, _V, _V, _L]),
    ("mpc_check_overflow", _I, [_V]),
    ("mpc_decode", _I, [_V, _V, _V, _L]),
    ("mpc_share", _I, [_V, _V, _I, _U, _V, _L]),
    ("mpc_reveal", _I, [_V, _V, _V, _L]),
    ("mpc_ttp_workspace_bytes", _S, [_V, _L, _L, _L]),
    ("mpc_ttp_triples", _I, [_V, _U, _L, _L, _L, _V, _V, _V, _V, _S]),
    ("mpc_ttp_wrap_pairs", _I, [_V, _U, _L, _V, _V]),
    ("mpc_workspace_bytes", _S, [_V, _L, _L, _L]),
    ("mpc_beaver_matmul", _I, [_V, _V, _V, _V, _V, _V, _V, _L, _L, _L, _I, _U, _V, _S]),
    ("mpc_beaver_mask", _I, [_V, _V, _V, _V, _V, _V, _L, _L, _L]),
    ("mpc_beaver_finish", _I, [_V, _V, _V, _V, _V, _V, _L, _L, _L, _I, _V, _S]),
    ("mpc_workspace_bytes_batched", _S, [_V, _L, _L, _L, _L]),
    ("mpc_beaver_matmul_batched", _I, [_V, _L, _V, _V, _V, _V, _V, _V, _L, _L, _L, _I, _U, _V, _S]),
    ("mpc_beaver_prepare", _I, [_V, _V, _V, _L, _L, _L, _V, _S]),
    ("mpc_beaver_matmul_prepared", _I, [_V, _V, _V, _V, _V, _L, _L, _L, _I, _U, _V, _S]),
    ("mpc_truncate", _I, [_V, _V, _L, _I, _U]),
    ("mpc_truncate_pairs", _I, [_V, _V, _L, _I, _V, _V]),
    ("mpc_ring_matmul_workspace_bytes", _S, [_L, _L, _L]),
    ("mpc_ring_matmul", _I, [_V, _V, _V, _V, _L, _L, _L, _V, _S]),
    ("mpc_ttp_mul_triples", _I, [_V, _U, _L, _V, _V, _V]),
    ("mpc_ttp_square_pairs", _I, [_V, _U, _L, _V, _V]),
    ("mpc_beaver_mul", _I, [_V, _V, _V, _V, _V, _V, _V, _L, _I, _U]),
    ("mpc_beaver_square", _I, [_V, _V, _V, _V, _V, _L, _I, _U]),
    ("mpc_beaver_mul_finish", _I, [_V, _V, _V, _V, _V, _V, _L, _I]),
    ("mpc_beaver_square_finish", _I, [_V, _V, _V, _V, _V, _L, _I]),
    ("mpc_reveal_batch", _I, [_V, _I, ctypes.POINTER(_V), ctypes.POINTER(_V), ctypes.POINTER(_L)]),
    ("mpc_mask", _I, [_V, _V, _V, _L, _V, _V, _L, _V]),
    ("mpc_ttp_conv_workspace_bytes", _S, [_V, ctypes.POINTER(ConvGeom)]),
    ("mpc_ttp_conv_triples", _I, [_V, _U, ctypes.POINTER(ConvGeom), _V, _V, _V, _V, _S]),
    ("mpc_conv2d_workspace_bytes", _S, [_V, ctypes.POINTER(ConvGeom)]),
    ("mpc_beaver_conv2d", _I, [_V, ctypes.POINTER(ConvGeom), _V, _V, _V, _V, _V, _V, _I, _U, _V, _S]),
    ("mpc_beaver_conv2d_finish", _I, [_V, ctypes.POINTER(ConvGeom), _V, _V, _V, _V, _V, _I, _V, _S]),
    ("mpc_relu", _I, [_V, _V, _V, _L, _U, _V]),
    ("mpc_profile_enable", _I, [_V, _I]),
    ("mpc_profile_read", _I, [_V, _I, ctypes.POINTER(_D), ctypes.POINTER(_U)]),
    ("mpc_launch_count", _U, [_V]),
]

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(python -m paper_2109_00984_b200.build) — there is no fallback path")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return [s[0] for s in SIGNATURES]


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = lib().mpc_nccl_unique_id(buf)
    if st != 0:
        raise RuntimeError(f"mpc_nccl_unique_id failed ({st})")
    return buf.raw


def derive_keys(master_seed: int, world_size: int, rank: int) -> Keys:
    """Party `rank`'s keys under the reproducibility convention (mpc_derive_keys; host only)."""
    k = Keys()
    st = lib().mpc_derive_keys(ctypes.c_uint64(master_seed), world_size, rank, ctypes.byref(k))
    if st != 0:
        raise ValueError(f"mpc_derive_keys failed ({st})")
    return k
