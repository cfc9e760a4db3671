"""Thin Python binding of include/mpc_ring.h (argument marshalling only).

Every method below forwards to the C-ABI entry point of the same name in
``libmpc_ring.so``; all arithmetic runs in the library's sm_100a kernels.
PyTorch supplies device memory, the current CUDA stream and (for one party
per GPU) the process group used to broadcast the NCCL unique id.  There is no
CPU or PyTorch fallback: if the native library is missing the import fails.

Tensors are CUDA ``torch.uint64`` (or ``torch.int64``, same bits) and
contiguous.  With ``rank=ALL_PARTIES`` share arguments carry a leading party
dimension ``P``; with one party per process they are that party's share.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _native

ALL_PARTIES = -1
DEFAULT_FRAC_BITS = 16          # P:244 §7, "L = 16 by default"

_STATUS = {0: "MPC_OK", 1: "MPC_ERR_ARG", 2: "MPC_ERR_SHAPE", 3: "MPC_ERR_OVERFLOW", 4: "MPC_ERR_CUDA",
           5: "MPC_ERR_NCCL", 6: "MPC_ERR_STATE", 7: "MPC_ERR_UNSUPPORTED"}

PROFILE_CLASSES = {"gemm": 0, "split": 1, "trunc": 2, "prg": 3, "codec": 4, "comm": 5}


class MpcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libmpc_ring takes CUDA device tensors")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    if t.dtype not in (torch.uint64, torch.int64, torch.float64, torch.uint8, torch.int8):
        raise TypeError(f"unsupported dtype {t.dtype}")
    return t.data_ptr()


def _u64(shape, device) -> torch.Tensor:
    return torch.empty(shape, dtype=torch.uint64, device=device)


def _check_out(t: torch.Tensor, shape, dtype) -> torch.Tensor:
    """Caller-provided output buffer: must match exactly (the library writes through the raw pointer)."""
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype or not t.is_contiguous() or t.device.type != "cuda":
        raise ValueError(f"out tensor {tuple(t.shape)} {t.dtype} does not match {tuple(shape)} {dtype} "
                         "(contiguous, on the context's device)")
    return t


def derive_keys(master_seed: int, world_size: int, rank: int) -> "_native.Keys":
    """Party `rank`'s keys as mpc_create derives them from master_seed (mpc_derive_keys)."""
    return _native.derive_keys(master_seed, world_size, rank)


Keys = _native.Keys


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId from the native library's NCCL (rank 0 calls this)."""
    return _native.nccl_unique_id()


class Prepared:
    """A prepared y operand (delta and b'_p limb planes) of an M x K x N Beaver matmul."""

    def __init__(self, M: int, K: int, N: int, ws: torch.Tensor):
        self.M, self.K, self.N, self.ws = M, K, N, ws


class Group:
    """An mpc_group: P one-party contexts of this process whose reveals meet in
    a host rendezvous instead of NCCL (mpc_create_local).  Drive each party's
    Context from its own thread; destroy the contexts before the group."""

    def __init__(self, world_size: int):
        self._lib = _native.lib()
        self.P = world_size
        h = ctypes.c_void_p()
        st = self._lib.mpc_group_create(ctypes.byref(h), world_size)
        if st != 0:
            raise MpcError(st, "mpc_group_create failed")
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.mpc_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """An mpc_ctx: one party of P (rank >= 0) or all P parties (rank = ALL_PARTIES) on `device`."""

    def __init__(self, world_size: int, rank: int = ALL_PARTIES, device: int = 0,
                 master_seed: int = 210900984, frac_bits: int = DEFAULT_FRAC_BITS,
                 nccl_id: Optional[bytes] = None, group: Optional["Group"] = None,
                 keys: Optional["_native.Keys"] = None):
        """keys: explicit party keys (mpc_create_with_keys; one party per process) instead
        of deriving every key from master_seed (mpc_create)."""
        self._lib = _native.lib()
        self.P = world_size
        self.rank = rank
        self.all_parties = rank == ALL_PARTIES
        self.device = torch.device("cuda", device)
        self.frac_bits = frac_bits
        h = ctypes.c_void_p()
        idbuf = None
        if nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        self._group = group               # keeps the group alive while this party is attached
        if keys is not None:
            if group is not None or rank == ALL_PARTIES:
                raise ValueError("explicit keys: one party per process (no group, no ALL_PARTIES)")
            st = self._lib.mpc_create_with_keys(ctypes.byref(h), world_size, rank, device, idbuf,
                                                ctypes.byref(keys), frac_bits)
        elif group is not None:
            if group.P != world_size:
                raise ValueError(f"group of {group.P} parties, world_size {world_size}")
            st = self._lib.mpc_create_local(ctypes.byref(h), group._h, rank, device, ctypes.c_uint64(master_seed),
                                            frac_bits)
        else:
            st = self._lib.mpc_create(ctypes.byref(h), world_size, rank, device, idbuf,
                                      ctypes.c_uint64(master_seed), frac_bits)
        if st != 0:
            raise MpcError(st, "mpc_create failed (needs an sm_100 GPU; nccl_id for one party per GPU)")
        self._h = h
        self._ws = None
        self._last_stream = None

    # ------------------------------------------------------------ plumbing
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.mpc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _call(self, fn, *args):
        cur = torch.cuda.current_stream(self.device)
        if self._last_stream is not None and self._last_stream != cur:
            # the workspace (and the library's scratch) were last used on another stream
            cur.wait_stream(self._last_stream)
        self._last_stream = cur
        self._lib.mpc_set_stream(self._h, ctypes.c_void_p(cur.cuda_stream))
        st = fn(self._h, *args)
        if st != 0:
            raise MpcError(st, self._lib.mpc_last_error(self._h).decode())

    def _workspace(self, nbytes: int) -> torch.Tensor:
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        return self._ws

    def _lead(self):
        return (self.P,) if self.all_parties else ()

    # ------------------------------------------------------------ fixed point
    def encode(self, x: torch.Tensor, out: Optional[torch.Tensor] = None, check: bool = True) -> torch.Tensor:
        """check=False: no stream synchronisation; overflows are reported by check_overflow()."""
        x = x.to(device=self.device, dtype=torch.float64).contiguous()
        out = _u64(x.shape, self.device) if out is None else _check_out(out, x.shape, torch.uint64)
        fn = self._lib.mpc_encode if check else self._lib.mpc_encode_async
        self._call(fn, _ptr(x), _ptr(out), ctypes.c_int64(x.numel()))
        return out

    def check_overflow(self) -> None:
        """Raises MpcError(MPC_ERR_OVERFLOW) if an encode(check=False) overflowed since the last check."""
        self._call(self._lib.mpc_check_overflow)

    def decode(self, v: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if out is None:
            out = torch.empty(v.shape, dtype=torch.float64, device=self.device)
        else:
            _check_out(out, v.shape, torch.float64)
        self._call(self._lib.mpc_decode, _ptr(v), _ptr(out), ctypes.c_int64(v.numel()))
        return out

    # ------------------------------------------------------------ share / reveal
    def share(self, x: Optional[torch.Tensor], src: int, share_id: int, shape=None,
              out: Optional[torch.Tensor] = None) -> torch.Tensor:
        shape = tuple(x.shape) if x is not None else tuple(shape)
        n = 1
        for s in shape:
            n *= s
        out = _u64(self._lead() + shape, self.device) if out is None else \
            _check_out(out, self._lead() + shape, torch.uint64)
        self._call(self._lib.mpc_share, _ptr(x), src, ctypes.c_uint64(share_id), _ptr(out), ctypes.c_int64(n))
        return out

    def reveal(self, shares: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        shape = tuple(shares.shape[1:]) if self.all_parties else tuple(shares.shape)
        out = _u64(shape, self.device) if out is None else _check_out(out, shape, torch.uint64)
        self._call(self._lib.mpc_reveal, _ptr(shares), _ptr(out), ctypes.c_int64(out.numel()))
        return out

    # ------------------------------------------------------------ offline TTP
    def ttp_triples(self, triple_id: int, M: int, K: int, N: int, out=None):
        if out is None:
            a = _u64(self._lead() + (M, K), self.device)
            b = _u64(self._lead() + (K, N), self.device)
            c = _u64(self._lead() + (M, N), self.device)
        else:
            a, b, c = out
            for t, shp in ((a, (M, K)), (b, (K, N)), (c, (M, N))):
                _check_out(t, self._lead() + shp, torch.uint64)
        nb = self._lib.mpc_ttp_workspace_bytes(self._h, M, K, N)
        ws = self._workspace(nb)
        self._call(self._lib.mpc_ttp_triples, ctypes.c_uint64(triple_id), ctypes.c_int64(M), ctypes.c_int64(K),
                   ctypes.c_int64(N), _ptr(a), _ptr(b), _ptr(c), _ptr(ws), ctypes.c_size_t(ws.numel()))
        return a, b, c

    def ttp_wrap_pairs(self, wrap_id: int, n: int):
        r = _u64(self._lead() + (n,), self.device)
        th = _u64(self._lead() + (n,), self.device)
        self._call(self._lib.mpc_ttp_wrap_pairs, ctypes.c_uint64(wrap_id), ctypes.c_int64(n), _ptr(r), _ptr(th))
        return r, th

    # ------------------------------------------------------------ online
    def set_reveal_chunks(self, chunks: int) -> None:
        """Row chunks of the overlapped eps reveal (one party per GPU; 0 = default policy)."""
        self._call(self._lib.mpc_set_reveal_chunks, int(chunks))

    def workspace_bytes(self, M: int, K: int, N: int) -> int:
        return int(self._lib.mpc_workspace_bytes(self._h, M, K, N))

    def _check_operands(self, lead, M, K, N, x=None, y=None, a=None, b=None, c=None, z=None):
        """Every operand of an M x K x N Beaver step has exactly its shape (the
        library reads and writes through raw pointers)."""
        for t, shp in ((x, (M, K)), (a, (M, K)), (y, (K, N)), (b, (K, N)), (c, (M, N)), (z, (M, N))):
            if t is not None:
                _check_out(t, lead + shp, t.dtype if t.dtype in (torch.uint64, torch.int64) else torch.uint64)

    def beaver_matmul(self, x, y, a, b, c, truncate: bool = True, wrap_id: int = 0,
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
        M, K = x.shape[-2], x.shape[-1]
        N = y.shape[-1]
        z = out if out is not None else _u64(self._lead() + (M, N), self.device)
        self._check_operands(self._lead(), M, K, N, x, y, a, b, c, z)
        ws = self._workspace(self.workspace_bytes(M, K, N))
        self._call(self._lib.mpc_beaver_matmul, _ptr(x), _ptr(y), _ptr(a), _ptr(b), _ptr(c), _ptr(z),
                   ctypes.c_int64(M), ctypes.c_int64(K), ctypes.c_int64(N), int(bool(truncate)),
                   ctypes.c_uint64(wrap_id), _ptr(ws), ctypes.c_size_t(ws.numel()))
        return z

    def beaver_matmul_batched(self, x, y, a, b, c, truncate: bool = True, wrap_id: int = 0,
                              out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """z[i] = x[i] @ y[i] for a batch of one shape: x [(P,) batch, M, K], y [(P,) batch, K, N]
        (mpc_beaver_matmul_batched: one reveal round, one split and one GEMM launch)."""
        B, M, K = x.shape[-3], x.shape[-2], x.shape[-1]
        N = y.shape[-1]
        z = out if out is not None else _u64(self._lead() + (B, M, N), self.device)
        self._check_operands(self._lead() + (B,), M, K, N, x, y, a, b, c, z)
        nb = int(self._lib.mpc_workspace_bytes_batched(self._h, B, M, K, N))
        ws = self._workspace(nb)
        self._call(self._lib.mpc_beaver_matmul_batched, ctypes.c_int64(B), _ptr(x), _ptr(y), _ptr(a), _ptr(b),
                   _ptr(c), _ptr(z), ctypes.c_int64(M), ctypes.c_int64(K), ctypes.c_int64(N), int(bool(truncate)),
                   ctypes.c_uint64(wrap_id), _ptr(ws), ctypes.c_size_t(ws.numel()))
        return z

    def beaver_prepare(self, y, b, M: int, out: Optional["Prepared"] = None) -> "Prepared":
        """The input-independent y side of a Beaver matmul with M x-rows (delta
        reveal + splits, mpc_beaver_prepare); returns the prepared operand, whose
        own workspace feeds beaver_matmul_prepared (`out`: reuse its workspace)."""
        K, N = y.shape[-2], y.shape[-1]
        self._check_operands(self._lead(), M, K, N, y=y, b=b)
        if out is not None:
            if (out.M, out.K, out.N) != (M, K, N):
                raise ValueError("prepared operand of another shape")
            ws = out.ws
        else:
            ws = torch.empty(max(self.workspace_bytes(M, K, N), 256), dtype=torch.uint8, device=self.device)
        self._call(self._lib.mpc_beaver_prepare, _ptr(y), _ptr(b), ctypes.c_int64(M), ctypes.c_int64(K),
                   ctypes.c_int64(N), _ptr(ws), ctypes.c_size_t(ws.numel()))
        return out if out is not None else Prepared(M, K, N, ws)

    def beaver_matmul_prepared(self, x, a, c, prep: "Prepared", truncate: bool = True, wrap_id: int = 0,
                               out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """The x side on a prepared y operand (mpc_beaver_matmul_prepared)."""
        M, K, N = prep.M, prep.K, prep.N
        if x.shape[-2:] != (M, K):
            raise ValueError(f"x {tuple(x.shape)} does not match the prepared {M} x {K}")
        z = out if out is not None else _u64(self._lead() + (M, N), self.device)
        self._check_operands(self._lead(), M, K, N, x=x, a=a, c=c, z=z)
        self._call(self._lib.mpc_beaver_matmul_prepared, _ptr(x), _ptr(a), _ptr(c), _ptr(z), ctypes.c_int64(M),
                   ctypes.c_int64(K), ctypes.c_int64(N), int(bool(truncate)), ctypes.c_uint64(wrap_id),
                   _ptr(prep.ws), ctypes.c_size_t(prep.ws.numel()))
        return z

    def beaver_mask(self, x, y, a, b) -> torch.Tensor:
        """One-party context: [x - a | y - b] (to be revealed by the caller, one round)."""
        M, K = x.shape[-2], x.shape[-1]
        N = y.shape[-1]
        self._check_operands((), M, K, N, x, y, a, b)
        ed = _u64((M * K + K * N,), self.device)
        self._call(self._lib.mpc_beaver_mask, _ptr(x), _ptr(y), _ptr(a), _ptr(b), _ptr(ed),
                   ctypes.c_int64(M), ctypes.c_int64(K), ctypes.c_int64(N))
        return ed

    def beaver_finish(self, ed, a, b, c, truncate: bool = True, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """One-party context: z_p from the revealed [eps | delta] (see mpc_beaver_finish)."""
        M, K = a.shape[-2], a.shape[-1]
        N = b.shape[-1]
        z = out if out is not None else _u64((M, N), self.device)
        self._check_operands((), M, K, N, a=a, b=b, c=c, z=z)
        _check_out(ed, (M * K + K * N,), ed.dtype)
        ws = self._workspace(self.workspace_bytes(M, K, N))
        self._call(self._lib.mpc_beaver_finish, _ptr(ed), _ptr(a), _ptr(b), _ptr(c), _ptr(z), ctypes.c_int64(M),
                   ctypes.c_int64(K), ctypes.c_int64(N), int(bool(truncate)), _ptr(ws), ctypes.c_size_t(ws.numel()))
        return z

    # ------------------------------------------------------------ elementwise
    def ttp_mul_triples(self, triple_id: int, shape, out=None):
        """Elementwise Beaver triple (a, b, c), c = ab (App. A.1.1)."""
        shp = self._lead() + tuple(shape)
        a, b, c = out if out is not None else (_u64(shp, self.device) for _ in range(3))
        for t in (a, b, c):
            _check_out(t, shp, torch.uint64)
        n = a[0].numel() if self.all_parties else a.numel()
        self._call(self._lib.mpc_ttp_mul_triples, ctypes.c_uint64(triple_id), ctypes.c_int64(n), _ptr(a), _ptr(b),
                   _ptr(c))
        return a, b, c

    def ttp_square_pairs(self, pair_id: int, shape, out=None):
        """Beaver pair (a, b), b = a^2."""
        shp = self._lead() + tuple(shape)
        a, b = out if out is not None else (_u64(shp, self.device) for _ in range(2))
        for t in (a, b):
            _check_out(t, shp, torch.uint64)
        n = a[0].numel() if self.all_parties else a.numel()
        self._call(self._lib.mpc_ttp_square_pairs, ctypes.c_uint64(pair_id), ctypes.c_int64(n), _ptr(a), _ptr(b))
        return a, b

    def beaver_mul(self, x, y, a, b, c, truncate: bool = True, wrap_id: int = 0,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Elementwise private product [x][y] (one round; + Alg. 1's round if P > 2 and truncate)."""
        z = _u64(tuple(x.shape), self.device) if out is None else _check_out(out, tuple(x.shape), torch.uint64)
        for t in (y, a, b, c):
            _check_out(t, tuple(x.shape), torch.uint64)
        n = x[0].numel() if self.all_parties else x.numel()
        self._call(self._lib.mpc_beaver_mul, _ptr(x), _ptr(y), _ptr(a), _ptr(b), _ptr(c), _ptr(z),
                   ctypes.c_int64(n), int(bool(truncate)), ctypes.c_uint64(wrap_id))
        return z

    def beaver_square(self, x, a, b, truncate: bool = True, wrap_id: int = 0,
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Private square [x^2] with a Beaver pair (one round; + Alg. 1's round if P > 2 and truncate)."""
        z = _u64(tuple(x.shape), self.device) if out is None else _check_out(out, tuple(x.shape), torch.uint64)
        for t in (a, b):
            _check_out(t, tuple(x.shape), torch.uint64)
        n = x[0].numel() if self.all_parties else x.numel()
        self._call(self._lib.mpc_beaver_square, _ptr(x), _ptr(a), _ptr(b), _ptr(z), ctypes.c_int64(n),
                   int(bool(truncate)), ctypes.c_uint64(wrap_id))
        return z

    def beaver_mul_finish(self, ed, a, b, c, truncate: bool = True) -> torch.Tensor:
        """One-party context: z_p from the revealed [eps | delta] (see mpc_beaver_mul_finish)."""
        z = _u64(tuple(a.shape), self.device)
        self._call(self._lib.mpc_beaver_mul_finish, _ptr(ed), _ptr(a), _ptr(b), _ptr(c), _ptr(z),
                   ctypes.c_int64(a.numel()), int(bool(truncate)))
        return z

    def beaver_square_finish(self, e, a, b, truncate: bool = True) -> torch.Tensor:
        """One-party context: [x^2]_p from the revealed eps (see mpc_beaver_square_finish)."""
        z = _u64(tuple(a.shape), self.device)
        self._call(self._lib.mpc_beaver_square_finish, _ptr(e), _ptr(a), _ptr(b), _ptr(z),
                   ctypes.c_int64(a.numel()), int(bool(truncate)))
        return z

    def reveal_batch(self, shares: list) -> list:
        """Reveal several share tensors in one round."""
        outs = [_u64(tuple(s.shape[1:]) if self.all_parties else tuple(s.shape), self.device) for s in shares]
        cnt = len(shares)
        sp = (ctypes.c_void_p * max(cnt, 1))(*[_ptr(s) for s in shares])
        op = (ctypes.c_void_p * max(cnt, 1))(*[_ptr(o) for o in outs])
        ns = (ctypes.c_int64 * max(cnt, 1))(*[o.numel() for o in outs])
        self._call(self._lib.mpc_reveal_batch, cnt, sp, op, ns)
        return outs

    # ------------------------------------------------------------ conv2d
    @staticmethod
    def conv_geom(B, C, H, W, Cout, kh, kw, stride=1, padding=0):
        """Geometry of x (B,C,H,W) * w (Cout,C,kh,kw), zero padding, stride; output (B,Cout,Ho,Wo)."""
        sh, sw = (stride, stride) if isinstance(stride, int) else stride
        ph, pw = (padding, padding) if isinstance(padding, int) else padding
        return _native.ConvGeom(B, C, H, W, Cout, kh, kw, sh, sw, ph, pw)

    @staticmethod
    def conv_out_shape(g):
        return (g.B, g.Cout, (g.H + 2 * g.ph - g.kh) // g.sh + 1, (g.W + 2 * g.pw - g.kw) // g.sw + 1)

    @staticmethod
    def conv1d_geom(B, C, L, Cout, k, stride=1, padding=0):
        """A 1-D convolution x (B, C, L) * w (Cout, C, k) as the H = kh = 1 case of
        mpc_conv2d_geom (same memory layout: (B, C, 1, L) and (Cout, C, 1, k))."""
        return _native.ConvGeom(B, C, 1, L, Cout, 1, k, 1, stride, 0, padding)

    def ttp_conv1d_triples(self, triple_id: int, g):
        """Conv triple of a 1-D geometry, shaped a (B, C, L), b (Cout, C, k), c (B, Cout, L_out)."""
        a, b, c = self.ttp_conv_triples(triple_id, g)
        lead = self._lead()
        return (a.view(lead + (g.B, g.C, g.W)), b.view(lead + (g.Cout, g.C, g.kw)),
                c.view(lead + (g.B, g.Cout, self.conv_out_shape(g)[3])))

    def beaver_conv1d(self, g, x, y, a, b, c, truncate: bool = True, wrap_id: int = 0,
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Private 1-D convolution: mpc_beaver_conv2d on the (B, C, 1, L) views."""
        if g.H != 1 or g.kh != 1:
            raise ValueError("not a 1-D geometry (conv1d_geom)")
        lead = self._lead()
        v4 = lambda t, shp: t.reshape(lead + shp)  # noqa: E731  (views of contiguous tensors)
        Lo = self.conv_out_shape(g)[3]
        z = self.beaver_conv2d(g, v4(x, (g.B, g.C, 1, g.W)), v4(y, (g.Cout, g.C, 1, g.kw)),
                               v4(a, (g.B, g.C, 1, g.W)), v4(b, (g.Cout, g.C, 1, g.kw)),
                               v4(c, (g.B, g.Cout, 1, Lo)), truncate, wrap_id,
                               None if out is None else v4(out, (g.B, g.Cout, 1, Lo)))
        return z.view(lead + (g.B, g.Cout, Lo))

    def ttp_conv_triples(self, triple_id: int, g):
        """Conv Beaver triple: a (input shape), b (weight shape), c = conv(a, b) (output shape)."""
        a = _u64(self._lead() + (g.B, g.C, g.H, g.W), self.device)
        b = _u64(self._lead() + (g.Cout, g.C, g.kh, g.kw), self.device)
        c = _u64(self._lead() + self.conv_out_shape(g), self.device)
        nb = self._lib.mpc_ttp_conv_workspace_bytes(self._h, ctypes.byref(g))
        ws = self._workspace(nb)
        self._call(self._lib.mpc_ttp_conv_triples, ctypes.c_uint64(triple_id), ctypes.byref(g), _ptr(a), _ptr(b),
                   _ptr(c), _ptr(ws), ctypes.c_size_t(ws.numel()))
        return a, b, c

    def beaver_conv2d(self, g, x, y, a, b, c, truncate: bool = True, wrap_id: int = 0,
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Private convolution [conv(x, y)] (one round at the input/weight shapes; + Alg. 1's if P > 2)."""
        shp = self._lead() + self.conv_out_shape(g)
        z = _u64(shp, self.device) if out is None else _check_out(out, shp, torch.uint64)
        ws = self._workspace(int(self._lib.mpc_conv2d_workspace_bytes(self._h, ctypes.byref(g))))
        self._call(self._lib.mpc_beaver_conv2d, ctypes.byref(g), _ptr(x), _ptr(y), _ptr(a), _ptr(b), _ptr(c), _ptr(z),
                   int(bool(truncate)), ctypes.c_uint64(wrap_id), _ptr(ws), ctypes.c_size_t(ws.numel()))
        return z

    def beaver_conv2d_finish(self, g, ed, a, b, c, truncate: bool = True) -> torch.Tensor:
        """One-party context: z_p from the revealed [eps | delta] (see mpc_beaver_conv2d_finish)."""
        z = _u64(self.conv_out_shape(g), self.device)
        ws = self._workspace(int(self._lib.mpc_conv2d_workspace_bytes(self._h, ctypes.byref(g))))
        self._call(self._lib.mpc_beaver_conv2d_finish, ctypes.byref(g), _ptr(ed), _ptr(a), _ptr(b), _ptr(c), _ptr(z),
                   int(bool(truncate)), _ptr(ws), ctypes.c_size_t(ws.numel()))
        return z

    def mask(self, x, a, y=None, b=None) -> torch.Tensor:
        """[x - a | y - b] as one flat buffer (0 rounds)."""
        n1 = x.numel()
        n2 = y.numel() if y is not None else 0
        ed = _u64((n1 + n2,), self.device)
        self._call(self._lib.mpc_mask, _ptr(x), _ptr(a), ctypes.c_int64(n1), _ptr(y), _ptr(b), ctypes.c_int64(n2),
                   _ptr(ed))
        return ed

    # ------------------------------------------------------------ ReLU
    def relu(self, x: torch.Tensor, relu_id: int, out: Optional[torch.Tensor] = None, want_sign: bool = False):
        """ReLU([x]) = [x][x >= 0] (A2B -> sign bit -> B2A -> Beaver multiplication)."""
        z = _u64(tuple(x.shape), self.device) if out is None else _check_out(out, tuple(x.shape), torch.uint64)
        sign = _u64(tuple(x.shape), self.device) if want_sign else None
        n = x[0].numel() if self.all_parties else x.numel()
        self._call(self._lib.mpc_relu, _ptr(x), _ptr(z), ctypes.c_int64(n), ctypes.c_uint64(relu_id), _ptr(sign))
        return (z, sign) if want_sign else z

    def truncate(self, x: torch.Tensor, bits: Optional[int] = None, wrap_id: int = 0) -> torch.Tensor:
        """In place; returns x."""
        n = x[0].numel() if self.all_parties else x.numel()
        self._call(self._lib.mpc_truncate, _ptr(x), ctypes.c_int64(n), int(bits or self.frac_bits),
                   ctypes.c_uint64(wrap_id))
        return x

    def truncate_pairs(self, x: torch.Tensor, r: torch.Tensor, theta_r: torch.Tensor,
                       bits: Optional[int] = None) -> torch.Tensor:
        """In place with a wrap pair from ttp_wrap_pairs (mpc_truncate_pairs); returns x."""
        n = x[0].numel() if self.all_parties else x.numel()
        for t in (r, theta_r):
            _check_out(t, self._lead() + (n,), torch.uint64)
        self._call(self._lib.mpc_truncate_pairs, _ptr(x), ctypes.c_int64(n), int(bits or self.frac_bits),
                   _ptr(r), _ptr(theta_r))
        return x

    def ring_matmul(self, A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
        M, K = A.shape
        N = B.shape[1]
        C = _u64((M, N), self.device)
        nb = self._lib.mpc_ring_matmul_workspace_bytes(M, K, N)
        ws = self._workspace(nb)
        self._call(self._lib.mpc_ring_matmul, _ptr(A), _ptr(B), _ptr(C), ctypes.c_int64(M), ctypes.c_int64(K),
                   ctypes.c_int64(N), _ptr(ws), ctypes.c_size_t(ws.numel()))
        return C

    # ------------------------------------------------------------ accounting
    def stats(self) -> tuple[int, int]:
        r, b = ctypes.c_uint64(), ctypes.c_uint64()
        self._lib.mpc_stats(self._h, ctypes.byref(r), ctypes.byref(b))
        return int(r.value), int(b.value)

    def profile_enable(self, on: bool = True):
        self._lib.mpc_profile_enable(self._h, int(on))

    def profile_read(self, cls: str) -> tuple[float, int]:
        ms, n = ctypes.c_double(), ctypes.c_uint64()
        self._call(self._lib.mpc_profile_read, PROFILE_CLASSES[cls], ctypes.byref(ms), ctypes.byref(n))
        return float(ms.value), int(n.value)

    def launch_count(self) -> int:
        return int(self._lib.mpc_launch_count(self._h))


def create(world_size: int, rank: int = ALL_PARTIES, **kw) -> Context:
    return Context(world_size, rank, **kw)
