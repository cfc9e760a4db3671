"""CPU oracle for the CrypTen Beaver ring-GEMM hot path (arXiv 2109.00984).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It wraps ``oracle/liboracle.so`` (built from ``oracle/oracle.c`` by
``oracle.build()``), which shares no code with the CUDA path.

All functions simulate every party in one process; party-indexed arrays are
numpy ``uint64`` of shape ``(P, ...)``.  Each wrapper only marshals arguments;
the arithmetic, with its citations into PAPER.md, lives in ``oracle.c``.

Parity pins: ``tests/test_oracle_pins.py`` (Philox KAT, frozen PRG table,
numpy / big-int GEMM, the paper's §4.3 float64 block GEMM, Beaver identity,
P=1 closed form, Alg. 1 identity, encode/decode examples).  "Parity unpinned":
only the PRG *layout* choice (any PRG is allowed), which is pinned
to the frozen table of SURVEY.md Appendix A.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

TAG_PRZS, TAG_A, TAG_B, TAG_C, TAG_R, TAG_THETA = 1, 2, 3, 4, 5, 6


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with plain gcc -O2 -fopenmp."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        # compile to a private name, then rename: concurrent importers (spawned
        # test workers) never load a half-written library
        tmp = f"{_LIB}.{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        i64 = ctypes.c_int64
        L.oracle_prg_at.restype = ctypes.c_uint64
        L.oracle_prg_at.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_stream_id.restype = ctypes.c_uint64
        L.oracle_stream_id.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64]
        L.oracle_prg.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, i64, u64p]
        L.oracle_derive_keys.argtypes = [ctypes.c_uint64, ctypes.c_int, u64p, u64p]
        L.oracle_encode.restype = ctypes.c_int
        L.oracle_truncate_local.restype = ctypes.c_int
        L.oracle_truncate_alg1.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_get_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's loops (timing only; results are independent of it)."""
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


# ---------------------------------------------------------------- O1 PRG
def philox4x32_10(ctr, key) -> list[int]:
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, k, o)
    return [int(o[i]) for i in range(4)]


def stream_id(tag: int, party: int, ident: int) -> int:
    return int(lib().oracle_stream_id(tag, party, ident & 0xFFFFFFFFFFFFFFFF))


def prg(key: int, stream: int, n: int, start: int = 0) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    lib().oracle_prg(ctypes.c_uint64(key), ctypes.c_uint64(stream), ctypes.c_uint64(start),
                     ctypes.c_int64(n), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    return out


def derive_keys(master: int, P: int) -> tuple[np.ndarray, int]:
    kp = np.zeros(max(P, 1), dtype=np.uint64)
    kt = np.zeros(1, dtype=np.uint64)
    lib().oracle_derive_keys(ctypes.c_uint64(master), P,
                             kp.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                             kt.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    return kp[:P], int(kt[0])


# ---------------------------------------------------------------- O2
def encode(x, frac_bits: int = 16) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    out = np.zeros(x.shape, dtype=np.uint64)
    rc = lib().oracle_encode(_p(x), _p(out), ctypes.c_int64(x.size), frac_bits)
    if rc != 0:
        raise OverflowError("encode: |x|*2^f >= 2^63")
    return out


def decode(v, frac_bits: int = 16) -> np.ndarray:
    v = _u64(v)
    out = np.zeros(v.shape, dtype=np.float64)
    lib().oracle_decode(_p(v), _p(out), ctypes.c_int64(v.size), frac_bits)
    return out


# ---------------------------------------------------------------- O3 / O8
def share(P: int, master: int, x, src: int, share_id: int, start: int = 0) -> np.ndarray:
    """PRZS shares of the src party's ring tensor x: array (P, *x.shape).
    start > 0: x holds elements [start, start + x.size) of a larger tensor."""
    x = _u64(x)
    kp, _ = derive_keys(master, P)
    kp = np.ascontiguousarray(kp)
    out = np.zeros((P,) + x.shape, dtype=np.uint64)
    lib().oracle_share_range(P, _p(kp), _p(x), src, ctypes.c_uint64(share_id), ctypes.c_int64(start),
                             ctypes.c_int64(x.size), _p(out))
    return out


def reveal(shares) -> np.ndarray:
    s = _u64(shares)
    P = s.shape[0]
    out = np.zeros(s.shape[1:], dtype=np.uint64)
    lib().oracle_reveal(P, _p(s), ctypes.c_int64(out.size), _p(out))
    return out


# ---------------------------------------------------------------- GEMM
def ring_matmul(A, B) -> np.ndarray:
    A, B = _u64(A), _u64(B)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    C = np.zeros((M, N), dtype=np.uint64)
    lib().oracle_ring_matmul(_p(A), _p(B), _p(C), ctypes.c_int64(M), ctypes.c_int64(K), ctypes.c_int64(N))
    return C


# ---------------------------------------------------------------- O4
def ttp_triple(P: int, master: int, triple_id: int, M: int, K: int, N: int, rows=None):
    """Beaver matmul triple (a: (P,R,K), b: (P,K,N), c: (P,R,N)); R = M or len(rows)."""
    _, kt = derive_keys(master, P)
    if rows is None:
        R = M
        rp = None
    else:
        rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        R = rows.size
        rp = _p(rows)
    a = np.zeros((P, R, K), dtype=np.uint64)
    b = np.zeros((P, K, N), dtype=np.uint64)
    c = np.zeros((P, R, N), dtype=np.uint64)
    lib().oracle_ttp_triple(P, ctypes.c_uint64(kt), ctypes.c_uint64(triple_id), ctypes.c_int64(M),
                            ctypes.c_int64(K), ctypes.c_int64(N), rp, ctypes.c_int64(R),
                            _p(a), _p(b), _p(c))
    return a, b, c


def ttp_triple_sampled(P: int, master: int, triple_id: int, M: int, K: int, N: int, rows, cols):
    """The triple restricted to rows of a/c and columns of b/c: a (P,R,K), b (P,K,C), c (P,R,C)."""
    _, kt = derive_keys(master, P)
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    cols = np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
    R, C = rows.size, cols.size
    a = np.zeros((P, R, K), dtype=np.uint64)
    b = np.zeros((P, K, C), dtype=np.uint64)
    c = np.zeros((P, R, C), dtype=np.uint64)
    lib().oracle_ttp_triple_sampled(P, ctypes.c_uint64(kt), ctypes.c_uint64(triple_id), ctypes.c_int64(M),
                                    ctypes.c_int64(K), ctypes.c_int64(N), _p(rows), ctypes.c_int64(R), _p(cols),
                                    ctypes.c_int64(C), _p(a), _p(b), _p(c))
    return a, b, c


def share_indices(P: int, master: int, x_vals, src: int, share_id: int, idx) -> np.ndarray:
    """PRZS shares of the elements at flat indices idx (x_vals = plaintext there): (P, len(idx))."""
    x_vals = _u64(x_vals).ravel()
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64).ravel())
    kp, _ = derive_keys(master, P)
    kp = np.ascontiguousarray(kp)
    out = np.zeros((P, idx.size), dtype=np.uint64)
    lib().oracle_share_indices(P, _p(kp), _p(x_vals), src, ctypes.c_uint64(share_id), _p(idx),
                               ctypes.c_int64(idx.size), _p(out))
    return out


# ---------------------------------------------------------------- O5
def beaver_matmul(x, y, a, b, c, want_intermediates: bool = False):
    """Un-truncated Beaver matmul shares z: (P, M, N) (scale 2^(2f))."""
    x, y, a, b, c = (_u64(t) for t in (x, y, a, b, c))
    P, M, K = x.shape
    N = y.shape[2]
    z = np.zeros((P, M, N), dtype=np.uint64)
    e = np.zeros((P, M, K), dtype=np.uint64)
    d = np.zeros((P, K, N), dtype=np.uint64)
    eps = np.zeros((M, K), dtype=np.uint64)
    delta = np.zeros((K, N), dtype=np.uint64)
    lib().oracle_beaver_matmul(P, _p(x), _p(y), _p(a), _p(b), _p(c), ctypes.c_int64(M), ctypes.c_int64(K),
                               ctypes.c_int64(N), _p(e), _p(d), _p(eps), _p(delta), _p(z))
    if want_intermediates:
        return z, dict(e=e, d=d, eps=eps, delta=delta)
    return z


# ---------------------------------------------------------------- O6 / O7
def truncate_local(x, bits: int = 16) -> np.ndarray:
    x = _u64(x)
    out = np.zeros_like(x)
    rc = lib().oracle_truncate_local(x.shape[0], _p(x), ctypes.c_int64(x[0].size), bits, _p(out))
    if rc != 0:
        raise ValueError("truncate_local: bad bits")
    return out


def wrap_count(x) -> np.ndarray:
    """Exact θ_x = (Σ signed([x]_p) − signed(x)) / 2^64 per element."""
    x = _u64(x)
    th = np.zeros(x.shape[1:], dtype=np.int64)
    lib().oracle_wrap_count(x.shape[0], _p(x), ctypes.c_int64(th.size), _p(th))
    return th


def wrap_pair(P: int, master: int, wrap_id: int, n: int):
    _, kt = derive_keys(master, P)
    r = np.zeros((P, n), dtype=np.uint64)
    th = np.zeros((P, n), dtype=np.uint64)
    lib().oracle_wrap_pair(P, ctypes.c_uint64(kt), ctypes.c_uint64(wrap_id), ctypes.c_int64(n), _p(r), _p(th))
    return r, th


def wrap_pair_indices(P: int, master: int, wrap_id: int, idx):
    _, kt = derive_keys(master, P)
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64).ravel())
    r = np.zeros((P, idx.size), dtype=np.uint64)
    th = np.zeros((P, idx.size), dtype=np.uint64)
    lib().oracle_wrap_pair_indices(P, ctypes.c_uint64(kt), ctypes.c_uint64(wrap_id), _p(idx), ctypes.c_int64(idx.size),
                                   _p(r), _p(th))
    return r, th


def truncate_alg1(x, r, theta_r, bits: int = 16, diagnostics: bool = False):
    x, r, theta_r = _u64(x), _u64(r), _u64(theta_r)
    P = x.shape[0]
    n = x[0].size
    out = np.zeros_like(x)
    z = np.zeros(x.shape[1:], dtype=np.uint64)
    eta = np.zeros(x.shape[1:], dtype=np.int64)
    rc = lib().oracle_truncate_alg1(P, _p(x), _p(r), _p(theta_r), ctypes.c_int64(n), bits, _p(out), _p(z), _p(eta))
    if rc != 0:
        raise ValueError("truncate_alg1: bad arguments")
    if diagnostics:
        return out, dict(z=z, eta=eta)
    return out


def truncate(x, bits: int = 16, master: int | None = None, wrap_id: int = 0, diagnostics: bool = False):
    """Protocol truncation: local for P <= 2, Alg. 1 for P > 2."""
    x = _u64(x)
    P = x.shape[0]
    if P <= 2:
        out = truncate_local(x, bits)
        return (out, dict(theta=wrap_count(x))) if diagnostics else out
    r, th = wrap_pair(P, master, wrap_id, x[0].size)
    r = r.reshape(x.shape)
    th = th.reshape(x.shape)
    return truncate_alg1(x, r, th, bits, diagnostics)


# ---------------------------------------------------------------- O9 - O12
def ttp_mul_triple(P: int, master: int, triple_id: int, shape):
    """Elementwise Beaver triple (a, b, c), each (P, *shape), with Σc = Σa · Σb mod 2^64."""
    _, kt = derive_keys(master, P)
    shape = tuple(shape)
    n = int(np.prod(shape, dtype=np.int64))
    a, b, c = (np.zeros((P,) + shape, dtype=np.uint64) for _ in range(3))
    lib().oracle_ttp_mul_triple(P, ctypes.c_uint64(kt), ctypes.c_uint64(triple_id), ctypes.c_int64(n),
                                _p(a), _p(b), _p(c))
    return a, b, c


def ttp_square_pair(P: int, master: int, pair_id: int, shape):
    """Beaver pair (a, b), each (P, *shape), with Σb = (Σa)^2 mod 2^64."""
    _, kt = derive_keys(master, P)
    shape = tuple(shape)
    n = int(np.prod(shape, dtype=np.int64))
    a, b = (np.zeros((P,) + shape, dtype=np.uint64) for _ in range(2))
    lib().oracle_ttp_square_pair(P, ctypes.c_uint64(kt), ctypes.c_uint64(pair_id), ctypes.c_int64(n), _p(a), _p(b))
    return a, b


def beaver_mul(x, y, a, b, c, want_intermediates: bool = False):
    """Un-truncated elementwise Beaver product shares z: (P, *shape) (scale 2^(2f))."""
    x, y, a, b, c = (_u64(t) for t in (x, y, a, b, c))
    P = x.shape[0]
    n = x[0].size
    z = np.zeros(x.shape, dtype=np.uint64)
    eps = np.zeros(x.shape[1:], dtype=np.uint64)
    delta = np.zeros(x.shape[1:], dtype=np.uint64)
    lib().oracle_beaver_mul(P, _p(x), _p(y), _p(a), _p(b), _p(c), ctypes.c_int64(n), _p(eps), _p(delta), _p(z))
    if want_intermediates:
        return z, dict(eps=eps, delta=delta)
    return z


def beaver_square(x, a, b, want_intermediates: bool = False):
    """Un-truncated Beaver square shares z: (P, *shape) (scale 2^(2f))."""
    x, a, b = (_u64(t) for t in (x, a, b))
    P = x.shape[0]
    n = x[0].size
    z = np.zeros(x.shape, dtype=np.uint64)
    eps = np.zeros(x.shape[1:], dtype=np.uint64)
    lib().oracle_beaver_square(P, _p(x), _p(a), _p(b), ctypes.c_int64(n), _p(eps), _p(z))
    if want_intermediates:
        return z, dict(eps=eps)
    return z


# ---------------------------------------------------------------- O13 / O14
class _ConvGeom(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in ("B", "C", "H", "W", "Cout", "kh", "kw", "sh", "sw", "ph", "pw")]


def conv_geom(B, C, H, W, Cout, kh, kw, stride=1, padding=0):
    sh, sw = (stride, stride) if isinstance(stride, int) else stride
    ph, pw = (padding, padding) if isinstance(padding, int) else padding
    return _ConvGeom(B, C, H, W, Cout, kh, kw, sh, sw, ph, pw)


def conv1d_geom(B, C, L, Cout, k, stride=1, padding=0):
    """A 1-D convolution (Wav2Letter) as the H = kh = 1 case of the 2-D
    geometry: x (B, C, L) = (B, C, 1, L), w (Cout, C, k) = (Cout, C, 1, k)."""
    return conv_geom(B, C, 1, L, Cout, 1, k, (1, stride), (0, padding))


def conv_out_shape(g):
    return (g.B, g.Cout, (g.H + 2 * g.ph - g.kh) // g.sh + 1, (g.W + 2 * g.pw - g.kw) // g.sw + 1)


def conv2d(x, w, g) -> np.ndarray:
    """Ring convolution mod 2^64: x (B,C,H,W), w (Cout,C,kh,kw) -> (B,Cout,Ho,Wo)."""
    x, w = _u64(x), _u64(w)
    out = np.zeros(conv_out_shape(g), dtype=np.uint64)
    lib().oracle_conv2d(_p(x), _p(w), ctypes.byref(g), _p(out))
    return out


def ttp_conv_triple(P: int, master: int, triple_id: int, g):
    """Conv Beaver triple: a (P,B,C,H,W), b (P,Cout,C,kh,kw), c (P,B,Cout,Ho,Wo), Σc = conv(Σa, Σb)."""
    _, kt = derive_keys(master, P)
    a = np.zeros((P, g.B, g.C, g.H, g.W), dtype=np.uint64)
    b = np.zeros((P, g.Cout, g.C, g.kh, g.kw), dtype=np.uint64)
    c = np.zeros((P,) + conv_out_shape(g), dtype=np.uint64)
    lib().oracle_ttp_conv_triple(P, ctypes.c_uint64(kt), ctypes.c_uint64(triple_id), ctypes.byref(g),
                                 _p(a), _p(b), _p(c))
    return a, b, c


def beaver_conv2d(x, y, a, b, c, g, want_intermediates: bool = False):
    """Un-truncated Beaver convolution shares z: (P,B,Cout,Ho,Wo) (scale 2^(2f))."""
    x, y, a, b, c = (_u64(t) for t in (x, y, a, b, c))
    P = x.shape[0]
    z = np.zeros((P,) + conv_out_shape(g), dtype=np.uint64)
    eps = np.zeros(x.shape[1:], dtype=np.uint64)
    delta = np.zeros(y.shape[1:], dtype=np.uint64)
    lib().oracle_beaver_conv2d(P, _p(x), _p(y), _p(a), _p(b), _p(c), ctypes.byref(g), _p(eps), _p(delta), _p(z))
    if want_intermediates:
        return z, dict(eps=eps, delta=delta)
    return z


# ---------------------------------------------------------------- O15 - O19
def bshare(P: int, master: int, x, src: int, share_id: int, shape=None) -> np.ndarray:
    """Binary (XOR) PRZS shares of the src party's words x: (P, *x.shape); x None -> zero-share of `shape`."""
    kp, _ = derive_keys(master, P)
    kp = np.ascontiguousarray(kp)
    if x is None:
        out = np.zeros((P,) + tuple(shape), dtype=np.uint64)
        lib().oracle_bshare(P, _p(kp), None, src, ctypes.c_uint64(share_id), ctypes.c_int64(out[0].size), _p(out))
        return out
    x = _u64(x)
    out = np.zeros((P,) + x.shape, dtype=np.uint64)
    lib().oracle_bshare(P, _p(kp), _p(x), src, ctypes.c_uint64(share_id), ctypes.c_int64(x.size), _p(out))
    return out


def breveal(shares) -> np.ndarray:
    shares = _u64(shares)
    out = np.zeros(shares.shape[1:], dtype=np.uint64)
    lib().oracle_breveal(shares.shape[0], _p(shares), ctypes.c_int64(out.size), _p(out))
    return out


def ttp_binary_triple(P: int, master: int, triple_id: int, shape):
    _, kt = derive_keys(master, P)
    n = int(np.prod(shape, dtype=np.int64))
    a, b, c = (np.zeros((P,) + tuple(shape), dtype=np.uint64) for _ in range(3))
    lib().oracle_ttp_binary_triple(P, ctypes.c_uint64(kt), ctypes.c_uint64(triple_id), ctypes.c_int64(n),
                                   _p(a), _p(b), _p(c))
    return a, b, c


def binary_and(x, y, a, b, c) -> np.ndarray:
    x, y, a, b, c = (_u64(t) for t in (x, y, a, b, c))
    z = np.zeros(x.shape, dtype=np.uint64)
    lib().oracle_binary_and(x.shape[0], _p(x), _p(y), _p(a), _p(b), _p(c), ctypes.c_int64(x[0].size), _p(z))
    return z


def add_ring(P: int, master: int, add_id: int, x, y) -> np.ndarray:
    """Binary shares of (x + y) mod 2^64 from binary shares x, y (Kogge-Stone, triples dealt by add_id)."""
    _, kt = derive_keys(master, P)
    x, y = _u64(x), _u64(y)
    out = np.zeros(x.shape, dtype=np.uint64)
    lib().oracle_add_ring(P, ctypes.c_uint64(kt), ctypes.c_uint64(add_id), _p(x), _p(y), ctypes.c_int64(x[0].size),
                          _p(out))
    return out


def a2b(master: int, a2b_id: int, x) -> np.ndarray:
    """Binary shares (P, *shape) of the value arithmetically shared by x (P, *shape)."""
    x = _u64(x)
    P = x.shape[0]
    kp, kt = derive_keys(master, P)
    kp = np.ascontiguousarray(kp)
    out = np.zeros(x.shape, dtype=np.uint64)
    lib().oracle_a2b(P, _p(kp), ctypes.c_uint64(kt), ctypes.c_uint64(a2b_id), _p(x), ctypes.c_int64(x[0].size),
                     _p(out))
    return out


def ttp_bit_pair(P: int, master: int, pair_id: int, shape):
    _, kt = derive_keys(master, P)
    n = int(np.prod(shape, dtype=np.int64))
    rA, rB = (np.zeros((P,) + tuple(shape), dtype=np.uint64) for _ in range(2))
    lib().oracle_ttp_bit_pair(P, ctypes.c_uint64(kt), ctypes.c_uint64(pair_id), ctypes.c_int64(n), _p(rA), _p(rB))
    return rA, rB


def b2a_bit(b, rA, rB, want_z: bool = False):
    b, rA, rB = (_u64(t) for t in (b, rA, rB))
    out = np.zeros(b.shape, dtype=np.uint64)
    z = np.zeros(b.shape[1:], dtype=np.uint64)
    lib().oracle_b2a_bit(b.shape[0], _p(b), _p(rA), _p(rB), ctypes.c_int64(b[0].size), _p(out), _p(z))
    return (out, z) if want_z else out


def relu(master: int, relu_id: int, x, diagnostics: bool = False):
    """ReLU([x]) = [x][x >= 0] for arithmetic shares x (P, *shape); relu_id < 2^32."""
    x = _u64(x)
    P = x.shape[0]
    kp, kt = derive_keys(master, P)
    kp = np.ascontiguousarray(kp)
    out = np.zeros(x.shape, dtype=np.uint64)
    sign = np.zeros(x.shape, dtype=np.uint64)
    rounds = ctypes.c_int(0)
    lib().oracle_relu(P, _p(kp), ctypes.c_uint64(kt), ctypes.c_uint64(relu_id), _p(x), ctypes.c_int64(x[0].size),
                      _p(out), _p(sign), ctypes.byref(rounds))
    if diagnostics:
        return out, dict(sign=sign, rounds=rounds.value)
    return out
