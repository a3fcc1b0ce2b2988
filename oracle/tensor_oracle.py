"""numpy front end of ``liboracle.so`` (oracle/spmoe_oracle.c).

TEST INFRASTRUCTURE ONLY — the checker for the sm_100a kernels and the timed
CPU restatement for bench.py's reference arm.  See spmoe_oracle.c for the
reference anchors (Eq. 1, Alg. 1-2; trace.py:28-37 tie-break).
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None

_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_u64 = C.c_uint64
_f = C.c_float

_SIGS = {
    "oracle_det_exp": (_f, [_f]),
    "oracle_det_silu": (_f, [_f]),
    "oracle_dot_fixed": (_f, [_p, _p, _i]),
    "oracle_router_topk": (None, [_p, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p]),
    "oracle_moe_permute": (None, [_p, _i, _i, _i, _p, _p, _p]),
    "oracle_expert_ffn": (None, [_p, _p, _i, _i, _i, _i, _p, _p, _p, _p]),
    "oracle_moe_combine": (None, [_p, _p, _p, _i, _i, _i, _p, _p, _p, _p]),
    "oracle_argmax_rows": (None, [_p, _i64, _i, _i, _p]),
    "oracle_greedy_accept": (None, [_p, _i64, _p, _i, _i, _i, _p, _p]),
    "oracle_fill_normal_bf16": (None, [_p, _i64, _u64, _u64, _f]),
    "oracle_set_threads": (None, [_i]),
    "oracle_num_threads": (_i, []),
    "oracle_rms_scale": (_f, [_p, _i, _f]),
    "oracle_rms_norm": (None, [_p, _p, _i, _i, _f, _p]),
    "oracle_linear": (None, [_p, _p, _i64, _i, _i, _i, _p, _f, _p, _i64, _p, _p]),
    "oracle_rope_kv": (None, [_p, _p, _p, _p, _i, _i, _i, _i, _i, _i, _i, _p, _p, _p]),
    "oracle_attention": (None, [_p, _p, _p, _p, _i, _i, _i, _i, _i, _i, _f, _p]),
    "cpu_lm_len": (_i, [_i]),
    "cpu_pack_lm": (None, [_p, _i64, _i, _p]),
    "cpu_pack_blob": (None, [_p, _i, _i, _p]),
    "cpu_blob_lm_elems": (_i64, [_i, _i]),
    "cpu_linear": (None, [_p, _p, _i64, _i, _i, _i, _p, _f, _p, _i64, _p, _p]),
    "cpu_expert_ffn": (None, [_p, _i, _i, _p, _p, _i, _p, _p]),
    "cpu_attn_block": (None, [_p, _i, _i, _i, _p, _p, _p, _f, _i, _i, _i, _p, _p, _i, _p, _p, _p, _i, _f]),
    "cpu_upcycle": (None, [_p, _p, _i64, _f]),
    "cpu_accum": (None, [_p, _p, _i64]),
    "cpu_div_bf16": (None, [_p, _i64, _f, _p]),
    "cpu_scale_bf16": (None, [_p, _i64, _f]),
    "oracle_xc_encode": (_u64, [_p, _i, _p, _p, _u64, _p]),
    "oracle_xc_decode": (_i, [_p, _p]),
}


def build() -> Path:
    srcs = [HERE / n for n in ("spmoe_oracle.c", "forward_oracle.c", "cpu_path.c", "pool.c", "pool.h", "xc_oracle.c",
                               "Makefile")] + [HERE.parent / "include" / "spmoe.h"]
    if not LIB.exists() or any(LIB.stat().st_mtime < s.stat().st_mtime for s in srcs):
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        for n, (r, a) in _SIGS.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def det_exp(x: float) -> float:
    return float(lib().oracle_det_exp(float(x)))


def dot_fixed(a_bf16: np.ndarray, b_bf16: np.ndarray) -> float:
    a = _c(a_bf16, np.uint16)
    b = _c(b_bf16, np.uint16)
    return float(lib().oracle_dot_fixed(_ptr(a), _ptr(b), a.size))


def router_topk(x, wg, k, renorm=True, sg_w=None):
    """x [T,H] uint16(bf16 bits), wg [E,H] -> (weights f32[T,k], idx i32[T,k],
    logits f32[T,E], shared_gate f32[T] | None)."""
    x = _c(x, np.uint16)
    wg = _c(wg, np.uint16)
    T, H = x.shape
    E = wg.shape[0]
    w = np.empty((T, k), np.float32)
    idx = np.empty((T, k), np.int32)
    lg = np.empty((T, E), np.float32)
    sg = None
    sgw = None
    if sg_w is not None:
        sgw = _c(sg_w, np.uint16)
        sg = np.empty((T,), np.float32)
    lib().oracle_router_topk(_ptr(x), _ptr(wg), T, H, E, k, 1 if renorm else 0, _ptr(w), _ptr(idx), _ptr(lg), _ptr(sgw), _ptr(sg))
    return w, idx, lg, sg


def moe_permute(idx, E):
    idx = _c(idx, np.int32)
    T, k = idx.shape
    off = np.empty((E + 1,), np.int32)
    perm = np.empty((T * k,), np.int32)
    inv = np.full((T * k,), -1, np.int32)
    lib().oracle_moe_permute(_ptr(idx), T, k, E, _ptr(off), _ptr(perm), _ptr(inv))
    return off, perm, inv


def expert_ffn(blobs, x, F, offsets, perm, h_out=None, y=None):
    """blobs: list of E uint16 arrays (or None); returns (h [T*k,F] u16, y [T*k,H] f32)."""
    x = _c(x, np.uint16)
    T, H = x.shape
    E = len(blobs)
    n = int(offsets[-1])
    if h_out is None:
        h_out = np.zeros((max(n, 1), F), np.uint16)
    if y is None:
        y = np.zeros((max(n, 1), H), np.float32)
    keep = [None if b is None else _c(b, np.uint16) for b in blobs]
    arr = (C.c_void_p * E)(*[None if b is None else b.ctypes.data for b in keep])
    offsets = _c(offsets, np.int32)
    perm = _c(perm, np.int32)
    lib().oracle_expert_ffn(arr, _ptr(x), T, H, F, E, _ptr(offsets), _ptr(perm), _ptr(h_out), _ptr(y))
    return h_out, y


def moe_combine(y, inv, w, T, H, k, ys=None, sg=None, residual=None):
    out = np.empty((T, H), np.uint16)
    y = _c(y, np.float32)
    inv = _c(inv, np.int32)
    w = None if w is None else _c(w, np.float32)
    ys = None if ys is None else _c(ys, np.float32)
    sg = None if sg is None else _c(sg, np.float32)
    residual = None if residual is None else _c(residual, np.uint16)
    lib().oracle_moe_combine(_ptr(y), _ptr(inv), _ptr(w), T, H, k, _ptr(ys), _ptr(sg), _ptr(residual), _ptr(out))
    return out


def greedy_accept(logits, draft):
    logits = _c(logits, np.float32)
    B, N1, V = logits.shape
    N = N1 - 1
    draft = _c(draft, np.int32).reshape(B, N) if N > 0 else np.zeros((B, 0), np.int32)
    amax = np.empty((B, N1), np.int32)
    res = np.empty((B, 2), np.int32)
    lib().oracle_greedy_accept(_ptr(logits), V, _ptr(draft), B, N, V, _ptr(amax), _ptr(res))
    return amax, res


def argmax_rows(logits):
    logits = _c(logits, np.float32)
    R, V = logits.shape
    out = np.empty((R,), np.int32)
    lib().oracle_argmax_rows(_ptr(logits), V, R, V, _ptr(out))
    return out


def fill_normal_bf16(n, seed, offset=0, std=0.02):
    out = np.empty((n,), np.uint16)
    lib().oracle_fill_normal_bf16(_ptr(out), n, seed & 0xFFFFFFFFFFFFFFFF, offset & 0xFFFFFFFFFFFFFFFF, float(std))
    return out


# ------------------------------------------------- layer block (forward_oracle.c)
def rms_norm(x, w, eps):
    x = _c(x, np.uint16)
    H = x.shape[-1]
    out = np.empty_like(x)
    lib().oracle_rms_norm(_ptr(x), _ptr(_c(w, np.uint16)), x.size // H, H, float(eps), _ptr(out))
    return out


def linear(w, x, norm_w=None, eps=0.0, f32=False, residual=None):
    """Scalar K9: x [T, K] bf16 bits, w [N, K] -> fp32 [T, N] (f32) or bf16
    bits (bf16(residual + bf16(y)) with ``residual``)."""
    w = _c(w, np.uint16)
    x = _c(x, np.uint16)
    N, K = w.shape
    T = x.size // K
    nw = None if norm_w is None else _c(norm_w, np.uint16)
    if f32:
        y = np.empty((T, N), np.float32)
        lib().oracle_linear(_ptr(w), _ptr(x), K, T, K, N, _ptr(nw), float(eps), _ptr(y), N, None, None)
        return y
    out = np.empty((T, N), np.uint16)
    r = None if residual is None else _c(residual, np.uint16).reshape(T, N)
    lib().oracle_linear(_ptr(w), _ptr(x), K, T, K, N, _ptr(nw), float(eps), None, 0, _ptr(out), _ptr(r))
    return out


def rope_kv(qkv, cos, sin, start, nh, nkv, hd, k_cache, v_cache):
    """qkv [B, T, (nh+2nkv)hd] bits; caches [B, nkv, S, hd] updated in place;
    returns q [B, nh, T, hd]."""
    qkv = _c(qkv, np.uint16)
    B, T = qkv.shape[0], qkv.shape[1]
    S = k_cache.shape[2]
    q = np.zeros((B, nh, T, hd), np.uint16)
    st = _c(start, np.int64)
    lib().oracle_rope_kv(_ptr(qkv), _ptr(_c(cos, np.float32)), _ptr(_c(sin, np.float32)), _ptr(st), B, T, nh, nkv,
                         hd, S, cos.shape[0], _ptr(q), _ptr(k_cache), _ptr(v_cache))
    return q


def attention(q, k_cache, v_cache, start, scale):
    q = _c(q, np.uint16)
    B, nh, T, hd = q.shape
    nkv, S = k_cache.shape[1], k_cache.shape[2]
    out = np.empty((B, T, nh * hd), np.uint16)
    lib().oracle_attention(_ptr(q), _ptr(_c(k_cache, np.uint16)), _ptr(_c(v_cache, np.uint16)),
                           _ptr(_c(start, np.int64)), B, T, nh, nkv, hd, S, float(scale), _ptr(out))
    return out


# ------------------------------------------------ lane-major CPU path (cpu_path.c)
def lm_len(K: int) -> int:
    return int(lib().cpu_lm_len(int(K)))


def pack_lm(w):
    """raw [N, K] bf16 bits -> lane-major [N, Kp]."""
    w = _c(w, np.uint16)
    N, K = w.shape
    out = np.empty((N, lm_len(K)), np.uint16)
    lib().cpu_pack_lm(_ptr(w), N, K, _ptr(out))
    return out


def pack_blob(blob, H, F):
    blob = _c(blob, np.uint16).reshape(-1)
    out = np.empty((int(lib().cpu_blob_lm_elems(H, F)),), np.uint16)
    lib().cpu_pack_blob(_ptr(blob), H, F, _ptr(out))
    return out


def lm_linear(w_lm, K, x, norm_w=None, eps=0.0, f32=False, residual=None):
    w_lm = _c(w_lm, np.uint16)
    N = w_lm.shape[0]
    x = _c(x, np.uint16)
    T = x.size // K
    nw = None if norm_w is None else _c(norm_w, np.uint16)
    if f32:
        y = np.empty((T, N), np.float32)
        lib().cpu_linear(_ptr(w_lm), _ptr(x), K, T, K, N, _ptr(nw), float(eps), _ptr(y), N, None, None)
        return y
    out = np.empty((T, N), np.uint16)
    r = None if residual is None else _c(residual, np.uint16).reshape(T, N)
    lib().cpu_linear(_ptr(w_lm), _ptr(x), K, T, K, N, _ptr(nw), float(eps), None, 0, _ptr(out), _ptr(r))
    return out


def lm_expert_ffn(blob_lm, H, F, x, perm=None, n=None):
    """One expert (LM blob) on rows x[perm[q]] -> (h [n, F] bits, y [n, H] f32)."""
    x = _c(x, np.uint16)
    if perm is not None:
        perm = _c(perm, np.int32)
        n = perm.size if n is None else n
    elif n is None:
        n = x.shape[0]
    h = np.empty((max(n, 1), F), np.uint16)
    y = np.empty((max(n, 1), H), np.float32)
    lib().cpu_expert_ffn(_ptr(_c(blob_lm, np.uint16)), H, F, _ptr(x), _ptr(perm), n, _ptr(h), _ptr(y))
    return h[:n], y[:n]


# ---------------------------------------------------------------- bf16 utils
def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bits (same rule as the kernels)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[nan] = 0x7FC0
    return r


def bf16_bits_to_f32(a: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(a, np.uint16).astype(np.uint32) << 16).view(np.float32)


# ---------------------------------------------------------------------------
# XC expert-blob codec (oracle/xc_oracle.c)
# ---------------------------------------------------------------------------
def xc_encode(values, seg_n) -> np.ndarray:
    """bf16 bits (uint16, segments back to back) -> XC blob (uint8)."""
    v = _c(np.asarray(values).reshape(-1), np.uint16)
    segs = np.asarray(seg_n, dtype=np.int64)
    size = lib().oracle_xc_encode(_ptr(v), len(segs), _ptr(segs), None, 0, None)
    if size == 0:
        raise ValueError("segment sizes must be positive multiples of 4096")
    out = np.empty((size,), np.uint8)
    lib().oracle_xc_encode(_ptr(v), len(segs), _ptr(segs), _ptr(out), size, None)
    return out


def xc_decode(blob) -> np.ndarray:
    blob = _c(blob, np.uint8)
    raw = int(np.frombuffer(blob[16:24].tobytes(), dtype=np.uint64)[0])
    out = np.empty((raw // 2,), np.uint16)
    if lib().oracle_xc_decode(_ptr(blob), _ptr(out)) != 0:
        raise ValueError("malformed XC blob")
    return out
