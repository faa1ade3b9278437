"""CPU oracle for the FMPQ steps around the W4Ax GEMM -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` (and the bench's reference legs) may import this module; the
product path never does, and nothing here is shared with ``csrc/``.

Definitions, written out plainly from the paper (PAPER.md, arXiv 2410.12168)
and the SPEC readings listed in DESIGN.md:

* f2 calibration (§3.2, "we first identify channels with outliers
  through data sampling and then use the permutation strategy to cluster these
  channels into a single block"; rule from SPEC S:L139-165):
  score[c] = max over calibration rows |x[m, c]|; median = lower middle of the
  sorted scores; outlier iff score > theta * median (theta = 8); permutation
  perm[new] = old with the outliers first by descending score (ties: ascending
  channel) and the rest in original order; block b (128 channels) is INT8 iff
  it holds an outlier after the permutation.
* f3 KV4 (§3.2 "channel-wise 4-bit quantization strategy for the KV
  cache"; §6.1 "channel-wise asymmetric INT4 group quantization"; the
  asymmetric min-max rule of SPEC S:L62-70 with its degenerate case):
  per (channel, group of G tokens): mn, mx; mn == mx == v -> scale = |v| (1 if
  v == 0), zp = (v < 0); else lo = min(mn, 0), hi = max(mx, 0) (the range
  holds 0, so the zero point lies in [0, 15] and the round-trip bound holds --
  DESIGN.md reading), scale = fp32((hi - lo) / 15),
  zp = clamp(rha(fp32(-lo / scale)), 0, 15); q = clamp(rha(fp32(x / scale)) +
  zp, 0, 15); dequant = fp16_rne(fp32((q - zp) * scale)).  All divisions and
  products in IEEE fp32 (the precision the kernels decide the integers in),
  rha = round half away from zero evaluated exactly.

* f4 static per-block activation scales: see
  static_block_scales / quantize_act_static below.

Parity status: pinned by tests/test_fmpq_aux.py (SPEC worked examples,
lattice round trips, round-trip bound, brute-force reference of the rules).
"""
from __future__ import annotations

import math

import numpy as np

BLOCK = 128


# ------------------------------------------------------------------ f2 ----
def calib_absmax(X: np.ndarray) -> np.ndarray:
    """Per-channel max |x| over the rows of X (fp16 [M x K]) as fp32 (exact)."""
    return np.abs(X.astype(np.float32)).max(axis=0)


def median_lower(score: np.ndarray) -> float:
    s = sorted(float(v) for v in score)
    return s[(len(s) - 1) // 2]


def detect_outliers(score: np.ndarray, theta: float = 8.0) -> np.ndarray:
    """flag iff score > theta * median (theta * median in fp32)."""
    thr = np.float32(np.float32(theta) * np.float32(median_lower(score)))
    return np.array([np.float32(v) > thr for v in score], dtype=bool)


def build_permutation(score: np.ndarray, flags: np.ndarray) -> np.ndarray:
    """outliers first by descending score then ascending index,
    the rest stable.  perm[new] = old."""
    out = [c for c in range(len(score)) if flags[c]]
    out.sort(key=lambda c: (-float(score[c]), c))
    rest = [c for c in range(len(score)) if not flags[c]]
    return np.array(out + rest, dtype=np.int32)


def block_bits_for(perm: np.ndarray, flags: np.ndarray, k: int = BLOCK) -> np.ndarray:
    """S:L157-165 invariant: block b is 8-bit iff it holds >= 1 outlier."""
    nb = len(perm) // k
    return np.array([8 if any(flags[perm[b * k + i]] for i in range(k)) else 4 for b in range(nb)], dtype=np.uint8)


def fmpq_map(score: np.ndarray, theta: float = 8.0):
    flags = detect_outliers(score, theta)
    perm = build_permutation(score, flags)
    return perm, block_bits_for(perm, flags), int(flags.sum())


# ------------------------------------------------------------------ f3 ----
def _rha(v: np.float32) -> int:
    """round half away from zero of an fp32 value (exact: done in fp64)."""
    a = math.floor(abs(float(v)) + 0.5)
    return int(a) if v >= 0 else -int(a)


def kv_params(mn: np.float32, mx: np.float32):
    if mn == mx:
        v = np.float32(mn)
        return (np.float32(1.0) if v == 0 else np.float32(abs(v))), (1 if v < 0 else 0)
    lo, hi = np.float32(min(mn, 0)), np.float32(max(mx, 0))  # the range holds 0 (zp in [0, 15])
    scale = np.float32(np.float32(hi - lo) / np.float32(15.0))
    zp = min(15, max(0, _rha(np.float32(np.float32(-lo) / scale))))
    return scale, zp


def quantize_kv(KV: np.ndarray, group: int):
    """KV fp16 [T x C] -> (q uint8 [T x C] unpacked, scale fp32 [G x C], zp uint8 [G x C])."""
    T, C = KV.shape
    x = KV.astype(np.float32)
    ng = (T + group - 1) // group
    q = np.zeros((T, C), dtype=np.uint8)
    scale = np.zeros((ng, C), dtype=np.float32)
    zp = np.zeros((ng, C), dtype=np.uint8)
    for g in range(ng):
        t0, t1 = g * group, min(T, (g + 1) * group)
        for c in range(C):
            col = x[t0:t1, c]
            s, z = kv_params(np.float32(col.min()), np.float32(col.max()))
            scale[g, c], zp[g, c] = s, z
            for t in range(t0, t1):
                q[t, c] = min(15, max(0, _rha(np.float32(col[t - t0] / s)) + z))
    return q, scale, zp


def quantize_kv_vec(KV: np.ndarray, group: int):
    """Same definition, vectorised over channels (for larger test sizes);
    pinned against quantize_kv on small inputs."""
    T, C = KV.shape
    x = KV.astype(np.float32)
    ng = (T + group - 1) // group
    q = np.zeros((T, C), dtype=np.uint8)
    scale = np.zeros((ng, C), dtype=np.float32)
    zp = np.zeros((ng, C), dtype=np.uint8)
    for g in range(ng):
        t0, t1 = g * group, min(T, (g + 1) * group)
        blk = x[t0:t1]
        mn, mx = blk.min(axis=0), blk.max(axis=0)
        deg = mn == mx
        lo, hi = np.minimum(mn, 0).astype(np.float32), np.maximum(mx, 0).astype(np.float32)
        s = np.where(deg, np.where(mn == 0, np.float32(1), np.abs(mn)),
                     ((hi - lo).astype(np.float32) / np.float32(15)).astype(np.float32)).astype(np.float32)
        with np.errstate(divide="ignore", invalid="ignore"):
            zr = (-lo).astype(np.float32) / s
        zr64 = zr.astype(np.float64)
        z = np.where(deg, (mn < 0).astype(np.int64),
                     np.clip(np.sign(zr64) * np.floor(np.abs(zr64) + 0.5), 0, 15).astype(np.int64))
        scale[g], zp[g] = s, z
        v = (blk / s).astype(np.float32).astype(np.float64)
        r = np.sign(v) * np.floor(np.abs(v) + 0.5)
        q[t0:t1] = np.clip(r + z, 0, 15).astype(np.uint8)
    return q, scale, zp


def pack_kv(q: np.ndarray) -> np.ndarray:
    """[T x C] nibbles -> [T x C/2] bytes, byte j = q[2j] | q[2j+1] << 4."""
    return (q[:, 0::2] | (q[:, 1::2] << 4)).astype(np.uint8)


def dequantize_kv(q: np.ndarray, scale: np.ndarray, zp: np.ndarray, group: int) -> np.ndarray:
    T, C = q.shape
    g = np.arange(T) // group
    y = ((q.astype(np.float32) - zp[g].astype(np.float32)).astype(np.float32) * scale[g]).astype(np.float32)
    return y.astype(np.float16)


def unpack_kv(packed: np.ndarray) -> np.ndarray:
    """[T x C/2] bytes -> [T x C] nibbles (inverse of pack_kv)."""
    T, h = packed.shape
    q = np.zeros((T, 2 * h), dtype=np.uint8)
    q[:, 0::2] = packed & 0xF
    q[:, 1::2] = packed >> 4
    return q


def attention_kv4(q: np.ndarray, K, V, group: int, softmax_scale: float, D: int = 128) -> np.ndarray:
    """f3 dequant-in-attention (§3.2: the KV4 cache serves the
    memory-bound activation-activation operator): one decode query per
    head, K and V given as their KV4 caches (packed [T x C/2], scale [G x C],
    zp [G x C]).  K^, V^ = dequantize_kv(...) (fp16, the values the cache
    stands for); for head h: s_t = softmax_scale * sum_d q[h, d] K^[t, hD + d],
    p = exp(s - max s) / sum exp(s - max s), o[h] = sum_t p_t V^[t, hD : hD + D].
    Everything after the dequantisation in fp64; returns fp64 [H x D]."""
    Kh = dequantize_kv(unpack_kv(K[0]), K[1], K[2], group).astype(np.float64)
    Vh = dequantize_kv(unpack_kv(V[0]), V[1], V[2], group).astype(np.float64)
    H = q.shape[0]
    out = np.zeros((H, D), dtype=np.float64)
    for h in range(H):
        qh = q[h].astype(np.float64)
        s = softmax_scale * (Kh[:, h * D:(h + 1) * D] @ qh)
        e = np.exp(s - s.max())
        p = e / e.sum()
        out[h] = p @ Vh[:, h * D:(h + 1) * D]
    return out


# ------------------------------------------------------------------ f4 ----
# Static per-block activation scales (SPEC S:L157-165
# assign_block_precision: "per-block QuantParams computed from the permuted
# channels' pooled min/max at the block's bit width, symmetric scheme";
# compute_scale S:L62-70: symmetric scale = max(|min|, |max|) / qmax with
# qmax = 2^(b-1) - 1, degenerate -> scale 1; quantize S:L71-78:
# q = clamp(round_half_away(x / scale), -qmax, qmax)).  The runtime absmax of
# the dynamic path is replaced by one calibrated scale per block, the same for
# every token row; Sx[b, m] = scale_b so the GEMM is unchanged.
def static_block_scales(maxabs: np.ndarray, bits, perm=None, k: int = BLOCK) -> np.ndarray:
    """scale_b = fp32(pool_b / qmax_b), pool_b = max of the calibration maxabs
    over the block's channels on the permuted axis; pool_b == 0 -> 1."""
    maxabs = np.asarray(maxabs, dtype=np.float32)
    K = maxabs.size
    order = np.arange(K) if perm is None else np.asarray(perm, dtype=np.int64)
    out = np.zeros(K // k, np.float32)
    for b in range(K // k):
        pool = np.float32(max(float(maxabs[order[b * k + i]]) for i in range(k)))
        qmax = np.float32(127 if int(bits[b]) == 8 else 7)
        out[b] = np.float32(1.0) if pool == 0 else np.float32(pool / qmax)
    return out


def _q_static(x: np.float32, s: np.float32, qmax: int) -> int:
    v = np.float32(x / s)  # IEEE fp32 quotient
    if not np.isfinite(v):
        return qmax if v > 0 else -qmax
    return min(qmax, max(-qmax, _rha(v)))


def quantize_act_static(X: np.ndarray, bits, scales: np.ndarray, perm=None, k: int = BLOCK):
    """X fp16 [M x K] -> (Xq8 int8 [M x K8], Xq4 uint8 [M x K4/2], Sx fp32 [nb x ldsx])
    in the comet plane layout (INT4 nibble order of oracle.pack_int4)."""
    from . import ldsx_for, pack_int4, plane_widths

    X = np.asarray(X, dtype=np.float16)
    M, K = X.shape
    nb = K // k
    order = np.arange(K) if perm is None else np.asarray(perm, dtype=np.int64)
    Xp = X.astype(np.float32)[:, order]
    K8, K4 = plane_widths(bits, k)
    ldsx = ldsx_for(M)
    Xq8 = np.zeros((M, K8), np.int8)
    Xq4 = np.zeros((M, K4 // 2), np.uint8)
    Sx = np.ones((nb, ldsx), np.float32)
    r8 = r4 = 0
    for b in range(nb):
        is8 = int(bits[b]) == 8
        qmax = 127 if is8 else 7
        s = np.float32(scales[b])
        for m in range(M):
            q = np.array([_q_static(Xp[m, b * k + i], s, qmax) for i in range(k)], dtype=np.int8)
            if is8:
                Xq8[m, r8 * k:(r8 + 1) * k] = q
            else:
                Xq4[m, r4 * k // 2:(r4 + 1) * k // 2] = pack_int4(q)
            Sx[b, m] = s
        if is8:
            r8 += 1
        else:
            r4 += 1
    return Xq8, Xq4, Sx


# f4 variant: FP16 weight-scale storage (the group-wise "one FP16 scale
# factor" per group of 128 of the W4A8KV4 baseline; SURVEY 8(f) f4
# "FP16/BF16 scale storage").  Per (output channel n, group j of the permuted
# K axis): a = max |w|; s = fp16_rn(fp32(a / 7)) (a == 0 -> 1; a nonzero scale
# that rounds below the smallest fp16 subnormal -> 2^-24); q = clamp(rha(fp32(
# w / fp32(s))), -7, 7) (the stored scale is the one the weights are
# quantized with, so dequantisation needs no other scale; the clamp catches
# |w / s| up to 7.5 + when fp16 rounding made s < a / 7).  Sw16 [K/group x N]
# fp16, Wq in the O4 nibble order.
def pack_weight_f16s(W: np.ndarray, group: int = BLOCK, perm=None):
    from . import pack_int4

    W = np.asarray(W, dtype=np.float16)
    N, K = W.shape
    order = np.arange(K) if perm is None else np.asarray(perm, dtype=np.int64)
    Wp = W.astype(np.float32)[:, order]
    ng = K // group
    Wq = np.zeros((N, K // 2), np.uint8)
    Sw = np.zeros((ng, N), np.float16)
    for n in range(N):
        row = np.zeros(K, np.int8)
        for j in range(ng):
            g = Wp[n, j * group:(j + 1) * group]
            a = np.float32(np.max(np.abs(g)))
            if a == 0:
                s = np.float16(1.0)
            else:
                s = np.float16(np.float32(a / np.float32(7.0)))
                if s == 0:
                    s = np.float16(2.0 ** -24)
            Sw[j, n] = s
            sf = np.float32(s)
            for i in range(group):
                row[j * group + i] = _q_static(g[i], sf, 7)
        Wq[n] = pack_int4(row)
    return Wq, Sw


# f4, BF16 scale storage: as pack_weight_f16s with s = bf16_rn(fp32(a / 7))
# (round to nearest even on the fp32 bits; bf16 keeps fp32's exponent range,
# so a nonzero a never gives s = 0; a == 0 -> 1).  Sw16 [K/group x N] as
# uint16 bf16 encodings.
def f32_to_bf16_bits(x) -> np.ndarray:
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def pack_weight_bf16s(W: np.ndarray, group: int = BLOCK, perm=None):
    from . import pack_int4

    W = np.asarray(W, dtype=np.float16)
    N, K = W.shape
    order = np.arange(K) if perm is None else np.asarray(perm, dtype=np.int64)
    Wp = W.astype(np.float32)[:, order]
    ng = K // group
    Wq = np.zeros((N, K // 2), np.uint8)
    Sw = np.zeros((ng, N), np.uint16)
    for n in range(N):
        row = np.zeros(K, np.int8)
        for j in range(ng):
            g = Wp[n, j * group:(j + 1) * group]
            a = np.float32(np.max(np.abs(g)))
            sb = f32_to_bf16_bits(np.float32(1.0) if a == 0 else np.float32(a / np.float32(7.0)))
            Sw[j, n] = sb
            sf = bf16_bits_to_f32(sb)
            for i in range(group):
                row[j * group + i] = _q_static(g[i], np.float32(sf), 7)
        Wq[n] = pack_int4(row)
    return Wq, Sw


# f4 variant: bf16 activations.  A bf16 value's bits shifted left by 16 are
# its fp32 encoding (exact); from there the quantization is O3 (the C
# oracle's oracle_quantize_block, via oracle.quantize_block) on the permuted
# row, packed as in oracle.quantize_act.
def bf16_bits_to_f32(bits16: np.ndarray) -> np.ndarray:
    return (np.asarray(bits16, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def quantize_act_bf16(Xbits: np.ndarray, bits, perm=None, k: int = BLOCK):
    """Xbits uint16 [M x K] (bf16 encodings) -> (Xq8, Xq4, Sx) in the comet layout."""
    from . import ldsx_for, pack_int4, plane_widths, quantize_block

    X = bf16_bits_to_f32(Xbits)
    M, K = X.shape
    nb = K // k
    order = np.arange(K) if perm is None else np.asarray(perm, dtype=np.int64)
    Xp = X[:, order]
    K8, K4 = plane_widths(bits, k)
    Xq8 = np.zeros((M, K8), np.int8)
    Xq4 = np.zeros((M, K4 // 2), np.uint8)
    Sx = np.ones((nb, ldsx_for(M)), np.float32)
    r8 = r4 = 0
    for b in range(nb):
        is8 = int(bits[b]) == 8
        for m in range(M):
            q, s = quantize_block(Xp[m, b * k:(b + 1) * k], 127 if is8 else 7)
            if is8:
                Xq8[m, r8 * k:(r8 + 1) * k] = q
            else:
                Xq4[m, r4 * k // 2:(r4 + 1) * k // 2] = pack_int4(q)
            Sx[b, m] = s
        if is8:
            r8 += 1
        else:
            r4 += 1
    return Xq8, Xq4, Sx
