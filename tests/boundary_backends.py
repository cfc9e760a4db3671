"""One protocol script, two libraries behind the same boundary (SURVEY §8(b):
"the oracle library exports the same functions as oracle_mpc_* with host
pointers and identical semantics; the parity harness swaps one library for the
other").

`OracleBackend` drives liboracle.so's oracle_mpc_* on host numpy buffers;
`GpuBackend` drives libmpc_ring.so's mpc_* on CUDA tensors — the C ABI itself,
through ctypes, with the same entry-point names after the prefix.  `run_protocol`
is the script: encode, share, TTP triples, Beaver matmul with truncation, an
extra truncation with an offline wrap pair, reveal, decode.  Test helper only
(argument marshalling; no arithmetic).
"""
from __future__ import annotations

import ctypes

import numpy as np

_V, _I, _L, _U, _S = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t
# name -> argtypes after the context argument (identical for both libraries)
CALLS = {
    "encode": [_V, _V, _L],
    "decode": [_V, _V, _L],
    "share": [_V, _I, _U, _V, _L],
    "reveal": [_V, _V, _L],
    "ttp_triples": [_U, _L, _L, _L, _V, _V, _V, _V, _S],
    "ttp_wrap_pairs": [_U, _L, _V, _V],
    "beaver_matmul": [_V, _V, _V, _V, _V, _V, _L, _L, _L, _I, _U, _V, _S],
    "truncate": [_V, _L, _I, _U],
    "truncate_pairs": [_V, _L, _I, _V, _V],
    "stats": [ctypes.POINTER(_U), ctypes.POINTER(_U)],
}


class _Backend:
    prefix = ""

    def _bind(self, L):
        for name, args in CALLS.items():
            f = getattr(L, self.prefix + name)
            f.restype = _I
            f.argtypes = [_V] + args
        c = getattr(L, self.prefix + "create")
        c.restype = _I
        c.argtypes = [ctypes.POINTER(_V), _I, _I, _I, _V, _U, _I]
        d = getattr(L, self.prefix + "destroy")
        d.restype = _I
        d.argtypes = [_V]
        self.L = L

    def create(self, P, master, frac=16):
        h = _V()
        st = getattr(self.L, self.prefix + "create")(ctypes.byref(h), P, -1, 0, None, _U(master), frac)
        if st != 0:
            raise RuntimeError(f"{self.prefix}create: status {st}")
        self.h, self.P = h, P

    def close(self):
        getattr(self.L, self.prefix + "destroy")(self.h)

    def call(self, name, *args):
        return getattr(self.L, self.prefix + name)(self.h, *args)

    def stats(self):
        r, b = _U(), _U()
        self.call("stats", ctypes.byref(r), ctypes.byref(b))
        return int(r.value), int(b.value)


class OracleBackend(_Backend):
    prefix = "oracle_mpc_"

    def __init__(self):
        import oracle
        self._bind(oracle.lib())

    def buf(self, shape, dtype=np.uint64):
        return np.zeros(shape, dtype=dtype)

    def put(self, a):
        return np.ascontiguousarray(a).copy()

    def get(self, b):
        return np.asarray(b).copy()

    def ptr(self, b):
        return None if b is None else b.ctypes.data

    def ws(self, nbytes):
        return None, 0

    def sync(self):
        pass


class GpuBackend(_Backend):
    prefix = "mpc_"

    def __init__(self):
        import torch
        from paper_2109_00984_b200 import _native
        self.torch = torch
        self._bind(_native.lib())

    def buf(self, shape, dtype=np.uint64):
        t = self.torch
        return t.zeros(shape, dtype=t.float64 if dtype == np.float64 else t.int64, device="cuda")

    def put(self, a):
        a = np.ascontiguousarray(a)
        return self.torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a.copy()).cuda()

    def get(self, b):
        out = b.cpu().numpy()
        return out.view(np.uint64) if out.dtype == np.int64 else out

    def ptr(self, b):
        return None if b is None else b.data_ptr()

    def ws(self, nbytes):
        w = self.torch.empty(max(nbytes, 256), dtype=self.torch.uint8, device="cuda")
        self._ws = w
        return w.data_ptr(), w.numel()

    def sync(self):
        self.torch.cuda.synchronize()


def run_protocol(be, P, M, K, N, Xf, Yf, master, triple_id=1, wrap_id=3):
    """The same sequence of boundary calls on either backend; returns host copies."""
    be.create(P, master)
    out = {}
    p = be.ptr
    xe, ye = be.buf((M, K)), be.buf((K, N))
    hx, hy = be.put(Xf), be.put(Yf)                 # kept alive across the calls
    assert be.call("encode", p(hx), p(xe), M * K) == 0
    assert be.call("encode", p(hy), p(ye), K * N) == 0
    x, y = be.buf((P, M, K)), be.buf((P, K, N))
    assert be.call("share", p(xe), 0, 1, p(x), M * K) == 0
    assert be.call("share", p(ye), 1 % P, 2, p(y), K * N) == 0
    a, b, c = be.buf((P, M, K)), be.buf((P, K, N)), be.buf((P, M, N))
    if isinstance(be, GpuBackend):
        nb = int(be.L.mpc_ttp_workspace_bytes(be.h, M, K, N))
        w, wn = be.ws(nb)
    else:
        w, wn = be.ws(0)
    assert be.call("ttp_triples", triple_id, M, K, N, p(a), p(b), p(c), w, wn) == 0
    z = be.buf((P, M, N))
    if isinstance(be, GpuBackend):
        be.L.mpc_workspace_bytes.restype = _S
        be.L.mpc_workspace_bytes.argtypes = [_V, _L, _L, _L]
        w, wn = be.ws(int(be.L.mpc_workspace_bytes(be.h, M, K, N)))
    assert be.call("beaver_matmul", p(x), p(y), p(a), p(b), p(c), p(z), M, K, N, 1, wrap_id, w, wn) == 0
    # a second truncation with the wrap pair materialised offline (Alg. 1's inputs, P > 2)
    r, th = be.buf((P, M * N)), be.buf((P, M * N))
    assert be.call("ttp_wrap_pairs", wrap_id + 1, M * N, p(r), p(th)) == 0
    z2 = be.buf((P, M, N))
    z2[:] = z
    assert be.call("truncate_pairs", p(z2), M * N, 8, p(r), p(th)) == 0
    zr = be.buf((M, N))
    assert be.call("reveal", p(z), p(zr), M * N) == 0
    dec = be.buf((M, N), np.float64)
    assert be.call("decode", p(zr), p(dec), M * N) == 0
    be.sync()
    for k, v in dict(x=x, y=y, a=a, b=b, c=c, z=z, z2=z2, r=r, th=th, zr=zr, dec=dec).items():
        out[k] = be.get(v)
    out["stats"] = be.stats()
    be.close()
    return out
