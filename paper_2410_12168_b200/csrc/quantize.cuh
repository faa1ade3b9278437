// quantize.cuh -- a1+a2 (FMPQ activation quantize/pack, P:L185 + P:L194 §3.2)
// and a0 (INT4 weight pack, P:L194 + P:L396) for sm_100a.
//
// Work unit: one (row, 128-channel block) "item" is handled by a half-warp;
// each lane owns 8 consecutive (permuted) channels = one 128-bit fp16 load,
// one 32-bit INT4 store (or one 64-bit INT8 store).  The block absmax is a
// 4-step shuffle reduction inside the half-warp.  Items are ordered
// block-major inside groups of 8 rows so the Sx writes of a warp-pair are
// contiguous.  HBM-bound: algorithmic bytes per element ~ 2 (fp16 in)
// + 0.5..1 (plane out) + 4/128 (scale).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "sm100.cuh"

namespace comet {

struct BlockMap {
  // per 128-channel block: bit 15 = INT8 block, bits 0..14 = rank in its plane
  uint16_t code[512];
};

DEVI float half_bits_to_float(uint32_t h) { return __half2float(__ushort_as_half((unsigned short)h)); }
// activation element bits -> fp32 (exact for both): fp16, or bf16 (f4 variant)
template <bool kBf16>
DEVI float act_bits_to_float(uint32_t h) {
  return kBf16 ? __uint_as_float((h & 0xFFFFu) << 16) : half_bits_to_float(h);
}

// round half away from zero of v, exact for |v| < 2^23:
// floor(RZ(|v| + 0.5)) == floor(|v| + 0.5) because RZ never crosses the
// integer just below the exact sum.
DEVI int32_t round_half_away(float v) {
  int32_t q = __float2int_rz(__fadd_rz(fabsf(v), 0.5f));
  return v < 0.0f ? -q : q;
}

// Quantize 8 values with reciprocal r (already IEEE qmax/a) into int8.
DEVI void quant8(const float (&x)[8], float r, int32_t (&q)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) q[j] = round_half_away(__fmul_rn(x[j], r));
}

// ---- the fast dynamic path (row-staged kernel) ---------------------------
// q = round_half_away(x * r) as the two's-complement bits of M + q in a float
// (M = 1.5 * 2^23: the low byte of the result is q mod 256), without F2I:
//   u = RZ(|v| + 0.5)  (RZ never rounds up to the next integer, so floor(u) ==
//                       floor(|v| + 0.5); round-to-nearest would, for |v| just
//                       below 0.5, where the sum lands in a coarser binade)
//   t = RD(u + M)   = M + floor(u)            (one directed rounding, exact)
//   k = t - M       = floor(|v| + 0.5)        (exact)
//   M + copysign(k, v)                        (exact)
// |v| <= qmax (1 + 2^-22) here (v = x * fl(qmax / a), |x| <= a), so q needs no clamp.
DEVI uint32_t rha_bits(float v) {
  const float M = 12582912.0f;
  const float u = __fadd_rz(fabsf(v), 0.5f);
  const float k = __fadd_rn(__fadd_rd(u, M), -M);
  return __float_as_uint(__fadd_rn(copysignf(k, v), M));
}
// s = a / qmax and r = qmax / a (IEEE, as __fdiv_rn) for an a whose fp32
// mantissa has at most 10 significant fraction bits (an fp16 or bf16 value):
// a = 2^E * m with m in [1, 2), so a / qmax = 2^E * (m / qmax) and the
// correctly rounded quotient is 2^E * RN(m / qmax) while it stays normal;
// tab holds RN(m / qmax) and RN(qmax / m) for the 1024 mantissas (filled with
// __fdiv_rn by the kernel).  Extreme exponents fall back to the division.
// (A compile-time table in global memory instead of each CTA's shared memory
// measured no faster: 8B down projection 138 vs 134 us.)
struct ScaleTab {
  float v[4][1024];  // s7, r7, s127, r127
};
DEVI void fill_scale_tab(ScaleTab* t) {
  for (int i = threadIdx.x; i < 4 * 1024; i += blockDim.x) {
    const int k = i >> 10, j = i & 1023;
    const float m = 1.0f + (float)j * (1.0f / 1024.0f);
    const float qm = k < 2 ? 7.0f : 127.0f;
    t->v[k][j] = (k & 1) ? __fdiv_rn(qm, m) : __fdiv_rn(m, qm);
  }
}
DEVI void scale_recip(float a, bool is8, const ScaleTab* t, float& s, float& r) {
  const uint32_t ab = __float_as_uint(a);
  const uint32_t ex = ab & 0x7F800000u;
  if (a == 0.0f) {
    s = 1.0f;
    r = 0.0f;
  } else if (ex >= 0x1A000000u && ex <= 0x64000000u && (ab & 0x1FFFu) == 0) {  // 2^-75 <= a < 2^73
    const int k = is8 ? 2 : 0, j = (ab >> 13) & 1023;
    const uint32_t d = ex - 0x3F800000u;
    s = __uint_as_float(__float_as_uint(t->v[k][j]) + d);
    r = __uint_as_float(__float_as_uint(t->v[k + 1][j]) - d);
  } else {
    const float qmax = is8 ? 127.0f : 7.0f;
    s = __fdiv_rn(a, qmax);
    r = __fdiv_rn(qmax, a);
  }
}
// 8 values -> the O4 INT4 word (byte j = q_j & 0xF | (q_{j+4} & 0xF) << 4) or
// two INT8 words, from rha_bits results
DEVI uint32_t pack_int4_bits(const uint32_t (&h)[8]) {
  const uint32_t lo = __byte_perm(__byte_perm(h[0], h[1], 0x0040), __byte_perm(h[2], h[3], 0x0040), 0x5410);
  const uint32_t hi = __byte_perm(__byte_perm(h[4], h[5], 0x0040), __byte_perm(h[6], h[7], 0x0040), 0x5410);
  uint32_t w;
  asm("lop3.b32 %0, %1, %2, 0x0F0F0F0F, 0xD8;" : "=r"(w) : "r"(hi << 4), "r"(lo));  // (lo & m) | (hi<<4 & ~m)
  return w;
}
DEVI uint2 pack_int8_bits(const uint32_t (&h)[8]) {
  return make_uint2(__byte_perm(__byte_perm(h[0], h[1], 0x0040), __byte_perm(h[2], h[3], 0x0040), 0x5410),
                    __byte_perm(__byte_perm(h[4], h[5], 0x0040), __byte_perm(h[6], h[7], 0x0040), 0x5410));
}

// e4m3 of q * 2^-9 (sign-magnitude subnormal: byte = sign << 7 | |q|) for 4
// two's-complement nibbles in the low half of each byte of L
DEVI uint32_t e4m3_signed4(uint32_t L) {
  const uint32_t S = L & 0x08080808u;  // sign bits
  const uint32_t m1 = S >> 3;          // 1 per negative byte
  return ((L ^ (m1 * 0x0Fu)) + m1) | (S << 4);  // |q| = 16 - n for a negative nibble n
}
// kE4 output of an INT4 block (the prefill GEMM's operand, written by the
// quantizer in comet_w4ax_linear): 8 e4m3 bytes q * 2^-9 in K order and the
// lane's sum of q (for the 8 * sum(xq) correction)
DEVI uint2 e4m3_int4_bits(const uint32_t (&h)[8], int& qsum) {
  const uint32_t lo = __byte_perm(__byte_perm(h[0], h[1], 0x0040), __byte_perm(h[2], h[3], 0x0040), 0x5410) & 0x0F0F0F0Fu;
  const uint32_t hi = __byte_perm(__byte_perm(h[4], h[5], 0x0040), __byte_perm(h[6], h[7], 0x0040), 0x5410) & 0x0F0F0F0Fu;
  qsum = __dp4a(lo + hi, 0x01010101u, 0u) - 2 * __dp4a((lo & 0x08080808u) + (hi & 0x08080808u), 0x01010101u, 0u);
  return make_uint2(e4m3_signed4(lo), e4m3_signed4(hi));
}

DEVI uint32_t pack_int4_word(const int32_t (&q)[8]) {
  uint32_t w = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) w |= ((uint32_t)(q[j] & 0xF) | ((uint32_t)(q[j + 4] & 0xF) << 4)) << (8 * j);
  return w;
}

// Load the lane's 8 channels of row m, block b (positions 128b + 8*o .. +7
// on the permuted axis).
template <bool kPerm, bool kBf16 = false>
DEVI void load_octet(const __half* __restrict__ X, int64_t ldx, int64_t m, int b, int o, const int32_t* __restrict__ perm,
                     float (&x)[8]) {
  const int i0 = b * 128 + o * 8;
  if (!kPerm) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(X + m * ldx + i0));
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x[2 * j] = act_bits_to_float<kBf16>(w[j] & 0xFFFF);
      x[2 * j + 1] = act_bits_to_float<kBf16>(w[j] >> 16);
    }
  } else {
    int4 p0 = __ldg(reinterpret_cast<const int4*>(perm + i0));
    int4 p1 = __ldg(reinterpret_cast<const int4*>(perm + i0 + 4));
    int p[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
    const unsigned short* row = reinterpret_cast<const unsigned short*>(X + m * ldx);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = act_bits_to_float<kBf16>(__ldg(row + p[j]));
  }
}

// Byte offset of packed byte p (0 <= p < K/2) of weight row n in the tiled
// weight layout (include/comet.h): slab (n/128, p/64) of 128 rows x 64 B is
// contiguous, 16-B chunk c of row r stored at chunk c ^ ((r >> 1) & 3).
DEVI int64_t wq_tiled_offset(int64_t n, int64_t p, int nb) {
  const int64_t tile = n >> 7, r = n & 127, kb = p >> 6, c = (p >> 4) & 3, j = p & 15;
  return ((tile * nb + kb) * 128 + r) * 64 + ((c ^ ((r >> 1) & 3)) << 4) + j;
}

// Activation quantize + pack.  rows = ldsx (rows >= M get only Sx = 1.0).
// kTiledW: the INT4 plane is a weight matrix written in the tiled layout
// (comet_pack_weight, group 128).
// Grid: blockIdx.x = group of 8 rows, blockIdx.y = pair of 128-channel
// blocks; half-warp h of the CTA takes row 8x + (h & 7) of block 2y + (h >> 3)
// (no 64-bit index arithmetic: the previous grid-stride form spent more
// instructions on 64-bit item division than on the quantization).
template <bool kPerm, bool kTiledW = false, bool kBf16 = false>
__global__ void __launch_bounds__(256) quantize_act_kernel(const __half* __restrict__ X, int64_t ldx, int M, int nb,
                                                           int64_t ldsx, const int32_t* __restrict__ perm,
                                                           const __grid_constant__ BlockMap map, int8_t* __restrict__ Xq8,
                                                           int64_t ld8, uint8_t* __restrict__ Xq4, int64_t ld4,
                                                           float* __restrict__ Sx) {
  grid_dep_wait();    // PDL launch: the preceding kernel (which may read this call's outputs) is complete
  grid_dep_launch();  // the GEMM that follows may get scheduled (PDL)
  const int half_id = threadIdx.x >> 4;  // 16 half-warps per CTA
  const int o = threadIdx.x & 15;        // octet within the block
  const unsigned hmask = 0xFFFFu << (threadIdx.x & 16);  // this half-warp's lanes
  const int64_t m = (int64_t)blockIdx.x * 8 + (half_id & 7);
  const int b = blockIdx.y * 2 + (half_id >> 3);
  if (m >= ldsx || b >= nb) return;  // whole half-warps
  if (m >= M) {
    if (o == 0) Sx[(int64_t)b * ldsx + m] = 1.0f;
    return;
  }
  float x[8];
  load_octet<kPerm, kBf16>(X, ldx, m, b, o, perm, x);
  float a = 0.0f;
#pragma unroll
  for (int j = 0; j < 8; ++j) a = fmaxf(a, fabsf(x[j]));
#pragma unroll
  for (int off = 8; off >= 1; off >>= 1) a = fmaxf(a, __shfl_xor_sync(hmask, a, off));
  const uint32_t code = map.code[b];
  const bool is8 = (code >> 15) != 0;
  const int rank = code & 0x7FFF;
  const float qmax = is8 ? 127.0f : 7.0f;
  float s = 1.0f, r = 0.0f;
  if (a != 0.0f) {
    s = __fdiv_rn(a, qmax);
    r = __fdiv_rn(qmax, a);
  }
  int32_t q[8];
  quant8(x, r, q);
  if (is8) {
    uint32_t lo = (uint32_t)(q[0] & 0xFF) | ((uint32_t)(q[1] & 0xFF) << 8) | ((uint32_t)(q[2] & 0xFF) << 16) |
                  ((uint32_t)(q[3] & 0xFF) << 24);
    uint32_t hi = (uint32_t)(q[4] & 0xFF) | ((uint32_t)(q[5] & 0xFF) << 8) | ((uint32_t)(q[6] & 0xFF) << 16) |
                  ((uint32_t)(q[7] & 0xFF) << 24);
    *reinterpret_cast<uint2*>(Xq8 + m * ld8 + (int64_t)rank * 128 + o * 8) = make_uint2(lo, hi);
  } else if (kTiledW) {
    *reinterpret_cast<uint32_t*>(Xq4 + wq_tiled_offset(m, (int64_t)rank * 64 + o * 4, nb)) = pack_int4_word(q);
  } else {
    *reinterpret_cast<uint32_t*>(Xq4 + m * ld4 + (int64_t)rank * 64 + o * 4) = pack_int4_word(q);
  }
  if (o == 0) Sx[(int64_t)b * ldsx + m] = s;
}

// f32x2 helpers (FMUL2 / FADD2 with a rounding mode: two lanes per instruction)
DEVI uint64_t f2_pack(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
DEVI void f2_unpack(uint64_t d, uint32_t& lo, uint32_t& hi) { asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(d)); }
DEVI uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
DEVI uint64_t f2_add_rn(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
DEVI uint64_t f2_add_rz(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
DEVI uint64_t f2_add_rm(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// 0xFF for each negative element (sign replicated by prmt's selector msb;
// __byte_perm drops that bit) of the pairs a (elements 0, 1) and b (2, 3)
DEVI uint32_t sign_bytes4(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, 0xFDB9;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
// |x| of both elements of a packed fp16 / bf16 pair (already sign-cleared)
// as fp32 (exact)
template <bool kBf16>
DEVI uint64_t abs_pair_f32(uint32_t aw) {
  if (kBf16) return f2_pack(__uint_as_float(aw << 16), __uint_as_float(aw & 0xFFFF0000u));
  return f2_pack(half_bits_to_float(aw & 0xFFFFu), half_bits_to_float(aw >> 16));
}

#ifndef COMET_Q_NBUF
#define COMET_Q_NBUF 2  // row buffers per CTA (rows in flight = COMET_Q_NBUF - 1 ahead)
#endif
constexpr int kQNBuf = COMET_Q_NBUF;
// One (row, block) item for the row-staged kernel: 128 / kL lanes, each
// holding kL consecutive channels of the permuted axis; `row` is the row in
// shared memory.  Called warp-uniformly (the absmax and sum(q) reductions are
// full-warp shuffles, each lane group reducing its own item); `valid` false
// (a lane group past the last block) computes on a clamped block and stores
// nothing.
// kStatic (f4): the block's scale is the calibrated sstat[b]; q = clamp(rha(
// fp32(x / s)), -qmax, qmax) (comet_quantize_act_static) instead of the
// runtime absmax and the reciprocal multiply.
// kE4: INT4 blocks are written as the prefill GEMM's e4m3 operand X4e
// [M x n4*128 B] (ld4 = its row stride) plus CX[r4 * ldsx + m] = 8 sum(q)
// instead of the packed plane (comet_w4ax_linear, see gemm_pf.cuh)
//
// Dynamic path, per lane (kL channels as kL/2 packed fp16/bf16 pairs w):
//   a    = max |x| : integer max of the sign-cleared bit patterns (monotone
//          for non-negative floats), then the lane-group shuffle tree;
//   s, r = scale_recip(a)  (IEEE a / qmax and qmax / a);
//   t    = RD(RZ(|x| r + 0.5) + M) on f32x2 pairs: t = M + |q| (see rha_bits,
//          |x| r == |x r|);
//   e4m3 (kE4, INT4 block): byte = |q| | sign(x) << 7, sum(q) by a signed dp4a;
//   INT8 / packed INT4: h = (copysign(t - M, x)) + M, low byte = q.
// A negative x with q == 0 gives the e4m3 byte 0x80 (-0.0): its products
// add exactly zero in the GEMM, the same as +0.
// kPerm: 0 = no permutation, 1 = int32 perm (the API's), 2 = the same
// permutation as uint16 (comet_w4ax_linear converts it once per call into its
// scratch: half the bytes, so a K = 14336 permutation (28 KB) stays in L1
// next to the row buffers, where the int32 one (57 KB) was re-read from L2
// for every row)
template <int kL, int kPerm, bool kStatic = false, bool kBf16 = false, bool kE4 = false>
DEVI void quant_item(const unsigned short* row, const int32_t* __restrict__ gperm, const BlockMap& map, int b, bool valid,
                     int o, int64_t m, int64_t ldsx, int8_t* __restrict__ Xq8, int64_t ld8, uint8_t* __restrict__ Xq4,
                     int64_t ld4, float* __restrict__ Sx, const float* __restrict__ sstat = nullptr,
                     const ScaleTab* tab = nullptr, float* __restrict__ CX = nullptr) {
  static_assert(kL == 8 || kL == 16, "8 or 16 channels per lane");
  constexpr int kW = kL / 2;             // packed pairs per lane
  constexpr int kLanes = 128 / kL;       // lanes per item
  const int i0 = b * 128 + o * kL;
  uint32_t w[kW];  // elements 2j (low half) and 2j + 1 (high half)
  if (kPerm == 2) {
    const uint16_t* p16 = reinterpret_cast<const uint16_t*>(gperm);
#pragma unroll
    for (int v = 0; v < kL / 8; ++v) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(p16 + i0) + v);
      const uint32_t pw[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) w[4 * v + j] = __byte_perm(row[pw[j] & 0xFFFF], row[pw[j] >> 16], 0x5410);
    }
  } else if (kPerm) {
#pragma unroll
    for (int v = 0; v < kL / 4; ++v) {
      const int4 p = __ldg(reinterpret_cast<const int4*>(gperm + i0) + v);
      w[2 * v] = __byte_perm(row[p.x], row[p.y], 0x5410);
      w[2 * v + 1] = __byte_perm(row[p.z], row[p.w], 0x5410);
    }
  } else {
#pragma unroll
    for (int v = 0; v < kL / 8; ++v) {
      const uint4 u = *reinterpret_cast<const uint4*>(row + i0 + 8 * v);
      w[4 * v] = u.x, w[4 * v + 1] = u.y, w[4 * v + 2] = u.z, w[4 * v + 3] = u.w;
    }
  }
  const uint32_t code = map.code[b];
  const bool is8 = (code >> 15) != 0;
  const int rank = code & 0x7FFF;
  if constexpr (kStatic) {
    if (!valid) return;
    const float s = __ldg(sstat + b);
    const int qm = is8 ? 127 : 7;
#pragma unroll
    for (int g = 0; g < kL / 8; ++g) {
      int32_t q[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float v = __fdiv_rn(act_bits_to_float<kBf16>(w[4 * g + (j >> 1)] >> (16 * (j & 1))), s);
        q[j] = fabsf(v) >= 8388608.0f ? (v > 0.0f ? qm : -qm) : min(qm, max(-qm, round_half_away(v)));
      }
      if (is8) {
        uint32_t lo = (uint32_t)(q[0] & 0xFF) | ((uint32_t)(q[1] & 0xFF) << 8) | ((uint32_t)(q[2] & 0xFF) << 16) |
                      ((uint32_t)(q[3] & 0xFF) << 24);
        uint32_t hi = (uint32_t)(q[4] & 0xFF) | ((uint32_t)(q[5] & 0xFF) << 8) | ((uint32_t)(q[6] & 0xFF) << 16) |
                      ((uint32_t)(q[7] & 0xFF) << 24);
        *reinterpret_cast<uint2*>(Xq8 + m * ld8 + (int64_t)rank * 128 + o * kL + 8 * g) = make_uint2(lo, hi);
      } else {
        *reinterpret_cast<uint32_t*>(Xq4 + m * ld4 + (int64_t)rank * 64 + o * (kL / 2) + 4 * g) = pack_int4_word(q);
      }
    }
    if (o == 0) Sx[(int64_t)b * ldsx + m] = s;
    return;
  } else {
    uint32_t aw[kW];
#pragma unroll
    for (int j = 0; j < kW; ++j) aw[j] = w[j] & 0x7FFF7FFFu;
    uint32_t am = aw[0];
#pragma unroll
    for (int j = 1; j < kW; ++j) am = __vmaxu2(am, aw[j]);
    am = max(am & 0xFFFFu, am >> 16);
#pragma unroll
    for (int off = kLanes / 2; off >= 1; off >>= 1) am = max(am, __shfl_xor_sync(0xFFFFFFFFu, am, off));
    float s, r;
    scale_recip(act_bits_to_float<kBf16>(am), is8, tab, s, r);
    const uint64_t r2 = f2_pack(r, r), half2 = f2_pack(0.5f, 0.5f), M2 = f2_pack(12582912.0f, 12582912.0f);
    uint64_t t2[kW];
#pragma unroll
    for (int j = 0; j < kW; ++j) t2[j] = f2_add_rm(f2_add_rz(f2_mul(abs_pair_f32<kBf16>(aw[j]), r2), half2), M2);
    if (kE4) {  // (the sum(q) shuffle runs warp-uniformly: another lane group's block may be INT8)
      uint32_t e[kL / 4];
      int qs = 0;
#pragma unroll
      for (int g = 0; g < kL / 4; ++g) {  // 4 channels per e4m3 word
        uint32_t t0, t1, t2w, t3;
        f2_unpack(t2[2 * g], t0, t1);
        f2_unpack(t2[2 * g + 1], t2w, t3);
        const uint32_t mag = __byte_perm(__byte_perm(t0, t1, 0x0040), __byte_perm(t2w, t3, 0x0040), 0x5410);
        const uint32_t sg = sign_bytes4(w[2 * g], w[2 * g + 1]);
        qs = __dp4a((int)mag, (int)(sg | 0x01010101u), qs);
        e[g] = mag | (sg & 0x80808080u);
      }
#pragma unroll
      for (int off = kLanes / 2; off >= 1; off >>= 1) qs += __shfl_xor_sync(0xFFFFFFFFu, qs, off);
      if (!is8) {
        if (!valid) return;
        uint8_t* dst = Xq4 + m * ld4 + (int64_t)rank * 128 + o * kL;
        if constexpr (kL == 16)
          *reinterpret_cast<uint4*>(dst) = make_uint4(e[0], e[1], e[2], e[3]);
        else
          *reinterpret_cast<uint2*>(dst) = make_uint2(e[0], e[1]);
        if (o == 0) {
          CX[(int64_t)rank * ldsx + m] = 8.0f * (float)qs;
          Sx[(int64_t)b * ldsx + m] = s;
        }
        return;
      }
    }
    if (!valid) return;
    const uint64_t nM2 = f2_pack(-12582912.0f, -12582912.0f);
    uint32_t h[kL];
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      uint32_t klo, khi;
      f2_unpack(f2_add_rn(t2[j], nM2), klo, khi);
      f2_unpack(f2_add_rn(f2_pack(__uint_as_float(klo | ((w[j] << 16) & 0x80000000u)),
                                  __uint_as_float(khi | (w[j] & 0x80000000u))), M2), h[2 * j], h[2 * j + 1]);
    }
#pragma unroll
    for (int g = 0; g < kL / 8; ++g) {
      const uint32_t(&h8)[8] = *reinterpret_cast<const uint32_t(*)[8]>(h + 8 * g);
      if (is8)
        *reinterpret_cast<uint2*>(Xq8 + m * ld8 + (int64_t)rank * 128 + o * kL + 8 * g) = pack_int8_bits(h8);
      else
        *reinterpret_cast<uint32_t*>(Xq4 + m * ld4 + (int64_t)rank * 64 + o * (kL / 2) + 4 * g) = pack_int4_bits(h8);
    }
    if (o == 0) Sx[(int64_t)b * ldsx + m] = s;
  }
}

// Activation quantize + pack, row-staged variant (a1 + a2 for the GEMM
// path): persistent CTAs walk rows; each row (K fp16, contiguous) arrives in
// shared memory by one 1-D bulk copy (the next row's copy is in flight while
// this one is quantized), and the fused channel gather reads the
// permuted positions of the row from shared memory (the permutation itself
// comes through L1/L2) instead of issuing 8 scattered 2-byte global loads per
// lane.  Half-warp per (row, 128-channel block) item, lane = 8 channels, two
// items in flight per half-warp; output identical to quantize_act_kernel.
#ifndef COMET_Q_MINB
#define COMET_Q_MINB 1  // __launch_bounds__ min CTAs per SM (register cap)
#endif
#ifndef COMET_Q_THREADS
#define COMET_Q_THREADS 256
#endif
constexpr int kQThreads = COMET_Q_THREADS;  // threads per CTA of the row-staged kernel
template <int kPerm, bool kStatic = false, bool kBf16 = false, bool kE4 = false>
__global__ void __launch_bounds__(kQThreads, COMET_Q_MINB) quantize_act_rows_kernel(const __half* __restrict__ X, int64_t ldx, int M,
                                                                int nb, int64_t ldsx, const int32_t* __restrict__ perm,
                                                                const __grid_constant__ BlockMap map,
                                                                int8_t* __restrict__ Xq8, int64_t ld8,
                                                                uint8_t* __restrict__ Xq4, int64_t ld4,
                                                                float* __restrict__ Sx,
                                                                const float* __restrict__ sstat = nullptr,
                                                                float* __restrict__ CX = nullptr) {
  extern __shared__ __align__(16) uint8_t qsm[];
  grid_dep_wait();    // PDL launch: the preceding kernel (which may read this call's outputs) is complete
  grid_dep_launch();  // the GEMM that follows may get scheduled (PDL)
  const int K = nb * 128;
  __shared__ uint64_t rbar[kQNBuf];
  __shared__ ScaleTab tab;
  if (!kStatic) fill_scale_tab(&tab);
  // channels per lane: 16 for a contiguous row (two 16-byte smem loads per
  // lane); 8 with the permutation, whose gather is per element: with 16 the
  // lanes of a warp read positions 16 apart, which for the mostly monotone
  // FMPQ permutation (outliers first, the rest in order) piles 8-16
  // lanes onto the same banks (8192 x 4096: 51 vs 45 us; without the
  // permutation 31 vs 35 us)
  constexpr int kL = kPerm ? 8 : 16;
  constexpr int kLanes = 128 / kL;         // lanes per (row, block) item
  constexpr int kS = kQThreads / kLanes;   // items per CTA pass
  const int sub = (threadIdx.x & 31) / kLanes;  // item slot within the warp
  const int o = threadIdx.x % kLanes;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kQNBuf; ++i) mbar_init(&rbar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int64_t m, int buf) {
    mbar_arrive_expect_tx(&rbar[buf], (uint32_t)K * 2);
    bulk_load(qsm + (size_t)buf * K * 2, X + m * ldx, (uint32_t)K * 2, &rbar[buf]);
  };
  int64_t m = blockIdx.x;
  if (threadIdx.x == 0)
    for (int i = 0; i < kQNBuf - 1; ++i)
      if (m + (int64_t)i * gridDim.x < M) issue(m + (int64_t)i * gridDim.x, i);
  for (int it = 0; m < ldsx; ++it, m += gridDim.x) {
    const int buf = it % kQNBuf;
    if (m >= M) {  // padding rows of the scale layout
      for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        Sx[(int64_t)b * ldsx + m] = 1.0f;
        if (kE4 && !(map.code[b] >> 15)) CX[(int64_t)(map.code[b] & 0x7FFF) * ldsx + m] = 0.0f;
      }
      continue;
    }
    // prefetch row it + kQNBuf - 1 into the buffer row it - 1 used (its
    // contents were consumed before the __syncthreads that ended the last
    // iteration)
    const int64_t mp = m + (int64_t)(kQNBuf - 1) * gridDim.x;
    if (threadIdx.x == 0 && mp < M) issue(mp, (it + kQNBuf - 1) % kQNBuf);
    mbar_wait(&rbar[buf], (it / kQNBuf) & 1);
    const unsigned short* row = reinterpret_cast<const unsigned short*>(qsm + (size_t)buf * K * 2);
    // warp w takes blocks b0 .. b0 + 32/kLanes - 1, b0 = (32/kLanes) w + kS i,
    // in warp-uniform steps (the reductions are full-warp shuffles); a lane
    // group past the last block runs on a clamped block and stores nothing
    int b0 = (threadIdx.x >> 5) * (32 / kLanes);
    for (; b0 + kS < nb; b0 += 2 * kS) {
      quant_item<kL, kPerm, kStatic, kBf16, kE4>(row, perm, map, b0 + sub, true, o, m, ldsx, Xq8, ld8, Xq4, ld4, Sx,
                                                 sstat, &tab, CX);
      quant_item<kL, kPerm, kStatic, kBf16, kE4>(row, perm, map, min(b0 + kS + sub, nb - 1), b0 + kS + sub < nb, o, m,
                                                 ldsx, Xq8, ld8, Xq4, ld4, Sx, sstat, &tab, CX);
    }
    if (b0 < nb)
      quant_item<kL, kPerm, kStatic, kBf16, kE4>(row, perm, map, min(b0 + sub, nb - 1), b0 + sub < nb, o, m, ldsx, Xq8,
                                                 ld8, Xq4, ld4, Sx, sstat, &tab, CX);
    __syncthreads();  // every lane group is done with this buffer
  }
}

// perm int32[K] -> uint16[K] (K <= 65536), for the quantizer's kPerm == 2 path
__global__ void __launch_bounds__(256) perm_to_u16_kernel(const int32_t* __restrict__ perm, int K,
                                                          uint16_t* __restrict__ out) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i < K) out[i] = (uint16_t)__ldg(perm + i);
}

// Weight pack with one scale per output channel (group == K): a warp per
// row, pass 1 = absmax over the permuted row, pass 2 = quantize + pack
// (tiled weight layout).
template <bool kPerm>
__global__ void __launch_bounds__(256) pack_weight_rowscale_kernel(const __half* __restrict__ W, int64_t ldw, int N,
                                                                   int K, const int32_t* __restrict__ perm,
                                                                   uint8_t* __restrict__ Wq, float* __restrict__ Sw) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = (int64_t)blockIdx.x * 8 + warp;
  if (n >= N) return;
  const int n_oct = K / 8;
  float a = 0.0f;
  for (int t = lane; t < n_oct; t += 32) {
    float x[8];
    load_octet<kPerm>(W, ldw, n, t >> 4, t & 15, perm, x);
#pragma unroll
    for (int j = 0; j < 8; ++j) a = fmaxf(a, fabsf(x[j]));
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, off));
  float s = 1.0f, r = 0.0f;
  if (a != 0.0f) {
    s = __fdiv_rn(a, 7.0f);
    r = __fdiv_rn(7.0f, a);
  }
  for (int t = lane; t < n_oct; t += 32) {
    float x[8];
    load_octet<kPerm>(W, ldw, n, t >> 4, t & 15, perm, x);
    int32_t q[8];
    quant8(x, r, q);
    *reinterpret_cast<uint32_t*>(Wq + wq_tiled_offset(n, (int64_t)t * 4, K / 128)) = pack_int4_word(q);
  }
  if (lane == 0) Sw[n] = s;
}

}  // namespace comet
