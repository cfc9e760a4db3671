"""B200-native Beaver ring-GEMM for CrypTen-style MPC (arXiv 2109.00984).

The hot path is the C-ABI library ``libmpc_ring.so`` (include/mpc_ring.h);
``mpc.Context`` is its thin Python binding.
"""
from .mpc import ALL_PARTIES, Context, Group, Keys, MpcError, create, derive_keys, nccl_unique_id  # noqa: F401

__all__ = ["ALL_PARTIES", "Context", "Group", "Keys", "MpcError", "create", "derive_keys", "nccl_unique_id"]
