// fmpq_aux.cuh -- the two FMPQ steps around the W4Ax GEMM:
//   f2  calibration: per-channel absmax over calibration activations, the
//       score that identifies outlier channels "through data sampling"
//       (§3.2); the permutation / block mask are built on the host
//       (comet_fmpq_map in comet_api.cu);
//   f3  KV4: "channel-wise asymmetric INT4 group quantization for the KV
//       cache" (§6.1, §3.2) -- quantize-on-append and the
//       dequantization an attention kernel applies.
// All HBM-bound streaming kernels (coalesced 16-byte / 4-byte accesses).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "quantize.cuh"
#include "sm100.cuh"

namespace comet {

// maxabs[c] = max(maxabs[c], max_m |X[m, c]|).  CTA = 32 channel octets (one
// warp-wide 512-byte row segment per load) x 8 row lanes; rows
// 8 * blockIdx.y + lane8, strided by 8 * gridDim.y; the 8 row lanes are
// reduced in shared memory and merged across CTAs with one integer atomicMax
// per channel on the fp32 bit pattern (order-independent, exact for
// non-negative floats).
__global__ void __launch_bounds__(256) calib_absmax_kernel(const __half* __restrict__ X, int64_t ldx, int M, int K,
                                                           float* __restrict__ maxabs) {
  __shared__ float red[8][32 * 8 + 1];
  const int lane = threadIdx.x & 31, rl = threadIdx.x >> 5;  // octet lane, row lane
  const int oct = blockIdx.x * 32 + lane;
  const bool live = oct * 8 < K;
  float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (live) {
    for (int64_t m = (int64_t)blockIdx.y * 8 + rl; m < M; m += (int64_t)gridDim.y * 8) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(X + m * ldx + oct * 8));
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a[2 * j] = fmaxf(a[2 * j], fabsf(half_bits_to_float(w[j] & 0xFFFF)));
        a[2 * j + 1] = fmaxf(a[2 * j + 1], fabsf(half_bits_to_float(w[j] >> 16)));
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[rl][lane * 8 + j] = a[j];
  __syncthreads();
  // thread t merges channel t of this CTA's 256 channels over the 8 row lanes
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c < K) {
    float v = red[0][threadIdx.x];
#pragma unroll
    for (int r = 1; r < 8; ++r) v = fmaxf(v, red[r][threadIdx.x]);
    atomicMax(reinterpret_cast<unsigned int*>(maxabs) + c, __float_as_uint(v));
  }
}

// KV4 quantization of one token group: thread = channel pair (2j, 2j+1)
// (one 4-byte half2 load per token, one packed byte per token out).
// Asymmetric INT4 per (channel, group of G tokens):
//   mn, mx = min, max over the group;  mn == mx == v: scale = |v| (1 if v == 0),
//   zp = (v < 0);  else lo = min(mn, 0), hi = max(mx, 0), scale = (hi - lo) / 15,
//   zp = clamp(rha(-lo / scale), 0, 15);
//   q = clamp(rha(x / scale) + zp, 0, 15)  (IEEE fp32, rha = round half away).
DEVI void kv_params(float mn, float mx, float& scale, int& zp) {
  if (mn == mx) {
    scale = mn == 0.0f ? 1.0f : fabsf(mn);
    zp = mn < 0.0f ? 1 : 0;
  } else {
    // the range holds 0 so the zero point lies in [0, 15] (DESIGN.md reading)
    const float lo = fminf(mn, 0.0f), hi = fmaxf(mx, 0.0f);
    scale = __fdiv_rn(__fsub_rn(hi, lo), 15.0f);
    zp = min(15, max(0, round_half_away(__fdiv_rn(-lo, scale))));
  }
}

// CTA = one token group x 64 channel pairs, 4 token lanes per pair (256
// threads): min/max over the group reduced across the token lanes in shared
// memory, then every thread quantizes its tokens t0 + lane4, +4, ...
__global__ void __launch_bounds__(256) kv4_quantize_kernel(const __half* __restrict__ KV, int64_t ld, int T, int C,
                                                           int G, uint8_t* __restrict__ Q, float* __restrict__ scale,
                                                           uint8_t* __restrict__ zp) {
  __shared__ float red[4][4][64];  // [min0, max0, min1, max1][token lane][pair]
  const int pl = threadIdx.x & 63, tl = threadIdx.x >> 6;
  const int pr = blockIdx.x * 64 + pl;  // channel pair
  const bool live = 2 * pr < C;
  const int g = blockIdx.y;
  const int t0 = g * G, t1 = min(T, t0 + G);
  float mn0 = INFINITY, mx0 = -INFINITY, mn1 = INFINITY, mx1 = -INFINITY;
  if (live) {
    for (int t = t0 + tl; t < t1; t += 4) {
      const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(KV + (int64_t)t * ld + 2 * pr));
      const float x0 = half_bits_to_float(w & 0xFFFF), x1 = half_bits_to_float(w >> 16);
      mn0 = fminf(mn0, x0);
      mx0 = fmaxf(mx0, x0);
      mn1 = fminf(mn1, x1);
      mx1 = fmaxf(mx1, x1);
    }
  }
  red[0][tl][pl] = mn0;
  red[1][tl][pl] = mx0;
  red[2][tl][pl] = mn1;
  red[3][tl][pl] = mx1;
  __syncthreads();
  mn0 = fminf(fminf(red[0][0][pl], red[0][1][pl]), fminf(red[0][2][pl], red[0][3][pl]));
  mx0 = fmaxf(fmaxf(red[1][0][pl], red[1][1][pl]), fmaxf(red[1][2][pl], red[1][3][pl]));
  mn1 = fminf(fminf(red[2][0][pl], red[2][1][pl]), fminf(red[2][2][pl], red[2][3][pl]));
  mx1 = fmaxf(fmaxf(red[3][0][pl], red[3][1][pl]), fmaxf(red[3][2][pl], red[3][3][pl]));
  if (!live) return;
  float s0, s1;
  int z0, z1;
  kv_params(mn0, mx0, s0, z0);
  kv_params(mn1, mx1, s1, z1);
  if (tl == 0) {
    scale[(int64_t)g * C + 2 * pr] = s0;
    scale[(int64_t)g * C + 2 * pr + 1] = s1;
    zp[(int64_t)g * C + 2 * pr] = (uint8_t)z0;
    zp[(int64_t)g * C + 2 * pr + 1] = (uint8_t)z1;
  }
  for (int t = t0 + tl; t < t1; t += 4) {
    const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(KV + (int64_t)t * ld + 2 * pr));
    const float x0 = half_bits_to_float(w & 0xFFFF), x1 = half_bits_to_float(w >> 16);
    const int q0 = min(15, max(0, round_half_away(__fdiv_rn(x0, s0)) + z0));
    const int q1 = min(15, max(0, round_half_away(__fdiv_rn(x1, s1)) + z1));
    Q[(int64_t)t * (C / 2) + pr] = (uint8_t)(q0 | (q1 << 4));
  }
}

// out[t, c] = fp16_rn((q - zp) * scale) for every token t and channel c.
// Thread = 8 packed bytes (16 channels) of one token when C % 16 == 0
// (8-byte load, 32-byte store), else one byte.
__global__ void __launch_bounds__(256) kv4_dequantize_kernel(const uint8_t* __restrict__ Q,
                                                             const float* __restrict__ scale,
                                                             const uint8_t* __restrict__ zp, int T, int C, int G,
                                                             __half* __restrict__ out, int64_t ldo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per = 1;  // bytes per thread (8-byte variant measured slower: serial parameter loads)
  const int64_t units = (int64_t)T * (C / 2) / per;
  if (i >= units) return;
  const int64_t byte0 = i * per;
  const int t = (int)(byte0 / (C / 2)), pr0 = (int)(byte0 % (C / 2));
  const int64_t prow = (int64_t)(t / G) * C;
  uint32_t bytes[8];
  if (per == 8) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(Q + byte0));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      bytes[j] = (v.x >> (8 * j)) & 0xFF;
      bytes[4 + j] = (v.y >> (8 * j)) & 0xFF;
    }
  } else {
    bytes[0] = Q[byte0];
  }
  for (int j = 0; j < per; ++j) {
    const int c = 2 * (pr0 + j);
    const float y0 = __fmul_rn((float)((int)(bytes[j] & 0xF) - (int)zp[prow + c]), scale[prow + c]);
    const float y1 = __fmul_rn((float)((int)(bytes[j] >> 4) - (int)zp[prow + c + 1]), scale[prow + c + 1]);
    *reinterpret_cast<__half2*>(out + (int64_t)t * ldo + c) = __halves2half2(__float2half_rn(y0), __float2half_rn(y1));
  }
}

// Vectorised KV4 quantization (C % 8 == 0, 16-byte aligned rows): CTA = one
// token group x 64 channels (8 channel octets x 32 token lanes: 4 rows of
// 128 B per warp load).  Pass 1: 16-byte loads, per-channel min/max over the
// group reduced across the token lanes in shared memory; one thread per
// channel derives (scale, zp) as kv_params; pass 2 re-reads the group
// (L1/L2-resident) and writes one 4-byte packed word (8 channels) per token.
// Same arithmetic as kv4_quantize_kernel.
__global__ void __launch_bounds__(256) kv4_quantize_v_kernel(const __half* __restrict__ KV, int64_t ld, int T, int C,
                                                             int G, uint8_t* __restrict__ Q, float* __restrict__ scale,
                                                             uint8_t* __restrict__ zp) {
  __shared__ float red[2][32][65];  // [min, max][token lane][channel]
  __shared__ float ps[64];
  __shared__ int pz[64];
  const int ol = threadIdx.x & 7, tl = threadIdx.x >> 3;
  const int c0 = blockIdx.x * 64 + ol * 8;
  const bool live = c0 < C;
  const int g = blockIdx.y;
  const int t0 = g * G, t1 = min(T, t0 + G);
  float mn[8], mx[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) mn[j] = INFINITY, mx[j] = -INFINITY;
  if (live) {
    for (int t = t0 + tl; t < t1; t += 32) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(KV + (int64_t)t * ld + c0));
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float x0 = half_bits_to_float(w[j] & 0xFFFF), x1 = half_bits_to_float(w[j] >> 16);
        mn[2 * j] = fminf(mn[2 * j], x0), mx[2 * j] = fmaxf(mx[2 * j], x0);
        mn[2 * j + 1] = fminf(mn[2 * j + 1], x1), mx[2 * j + 1] = fmaxf(mx[2 * j + 1], x1);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[0][tl][ol * 8 + j] = mn[j], red[1][tl][ol * 8 + j] = mx[j];
  __syncthreads();
  if (threadIdx.x < 64) {
    const int ch = threadIdx.x, c = blockIdx.x * 64 + ch;
    float a = red[0][0][ch], b = red[1][0][ch];
    for (int r = 1; r < 32; ++r) a = fminf(a, red[0][r][ch]), b = fmaxf(b, red[1][r][ch]);
    float sc = 1.0f;
    int z = 0;
    if (c < C) {
      kv_params(a, b, sc, z);
      scale[(int64_t)g * C + c] = sc;
      zp[(int64_t)g * C + c] = (uint8_t)z;
    }
    ps[ch] = sc;
    pz[ch] = z;
  }
  __syncthreads();
  if (!live) return;
  float sv[8];
  int zv[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) sv[j] = ps[ol * 8 + j], zv[j] = pz[ol * 8 + j];
  for (int t = t0 + tl; t < t1; t += 32) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(KV + (int64_t)t * ld + c0));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t packed = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float x0 = half_bits_to_float(w[j] & 0xFFFF), x1 = half_bits_to_float(w[j] >> 16);
      const int q0 = min(15, max(0, round_half_away(__fdiv_rn(x0, sv[2 * j])) + zv[2 * j]));
      const int q1 = min(15, max(0, round_half_away(__fdiv_rn(x1, sv[2 * j + 1])) + zv[2 * j + 1]));
      packed |= (uint32_t)(q0 | (q1 << 4)) << (8 * j);
    }
    *reinterpret_cast<uint32_t*>(Q + (int64_t)t * (C / 2) + c0 / 2) = packed;
  }
}

// Vectorised KV4 dequantization (C % 16 == 0, 16-byte aligned output rows):
// thread = one token x 16 channels: one 8-byte load of the packed row, the
// channels' zero points (16 B) and scales (64 B, L1-resident across the
// group's tokens), two 16-byte stores.  n - zp is formed exactly as a float
// difference of 2^23 + n and 2^23 + zp (no int -> float conversion), then
// fp16_rn(fp32(n - zp) * scale) as kv4_dequantize_kernel.
__global__ void __launch_bounds__(256) kv4_dequantize_v_kernel(const uint8_t* __restrict__ Q,
                                                               const float* __restrict__ scale,
                                                               const uint8_t* __restrict__ zp, int T, int C, int G,
                                                               __half* __restrict__ out, int64_t ldo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nc = C / 16;
  if (i >= (int64_t)T * nc) return;
  const int t = (int)(i / nc), c0 = (int)(i % nc) * 16;
  const int64_t prow = (int64_t)(t / G) * C + c0;
  const uint2 qv = __ldg(reinterpret_cast<const uint2*>(Q + (int64_t)t * (C / 2) + c0 / 2));
  const uint4 zq = __ldg(reinterpret_cast<const uint4*>(zp + prow));
  const float4* sp = reinterpret_cast<const float4*>(scale + prow);
  const float4 s4[4] = {__ldg(sp), __ldg(sp + 1), __ldg(sp + 2), __ldg(sp + 3)};
  const float sc[16] = {s4[0].x, s4[0].y, s4[0].z, s4[0].w, s4[1].x, s4[1].y, s4[1].z, s4[1].w,
                        s4[2].x, s4[2].y, s4[2].z, s4[2].w, s4[3].x, s4[3].y, s4[3].z, s4[3].w};
  const uint32_t qw[2] = {qv.x, qv.y}, zw[4] = {zq.x, zq.y, zq.z, zq.w};
  uint32_t o[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // packed byte j = channels 2j (low nibble), 2j + 1 (high)
    const uint32_t b = (qw[j >> 2] >> (8 * (j & 3))) & 0xFFu;
    const uint32_t z0 = (zw[(2 * j) >> 2] >> (8 * ((2 * j) & 3))) & 0xFFu;
    const uint32_t z1 = (zw[(2 * j + 1) >> 2] >> (8 * ((2 * j + 1) & 3))) & 0xFFu;
    const float d0 = __fsub_rn(__uint_as_float(0x4B000000u | (b & 0xFu)), __uint_as_float(0x4B000000u | z0));
    const float d1 = __fsub_rn(__uint_as_float(0x4B000000u | (b >> 4)), __uint_as_float(0x4B000000u | z1));
    const __half2 h = __floats2half2_rn(__fmul_rn(d0, sc[2 * j]), __fmul_rn(d1, sc[2 * j + 1]));
    o[j] = *reinterpret_cast<const uint32_t*>(&h);
  }
  uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)t * ldo + c0);
  dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
  dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
}

// f4: static per-block activation scales:
// scale[b] = fp32(pool_b / qmax_b), pool_b = max of the calibration maxabs over
// the block's channels on the permuted axis, 1 if pool_b == 0.  CTA = block.
__global__ void __launch_bounds__(128) static_act_scales_kernel(const float* __restrict__ maxabs,
                                                                const int32_t* __restrict__ perm,
                                                                const __grid_constant__ BlockMap map,
                                                                float* __restrict__ scales) {
  __shared__ float red[4];
  const int b = blockIdx.x, i = b * 128 + threadIdx.x;
  float a = __ldg(maxabs + (perm ? __ldg(perm + i) : i));
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    const float pool = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    const float qmax = (map.code[b] >> 15) ? 127.0f : 7.0f;
    scales[b] = pool == 0.0f ? 1.0f : __fdiv_rn(pool, qmax);
  }
}

// f4: activation quantize + pack with static per-block scales:
// q = clamp(rha(fp32(x / scale[b])), -qmax, qmax), Sx[b, m] = scale[b] (so
// the GEMM is unchanged).  Same grid and plane layout as quantize_act_kernel
// (half-warp per (row, block) item, lane = 8 channels), no absmax reduction.
template <bool kPerm>
__global__ void __launch_bounds__(256) quantize_act_static_kernel(const __half* __restrict__ X, int64_t ldx, int M,
                                                                  int nb, int64_t ldsx, const int32_t* __restrict__ perm,
                                                                  const __grid_constant__ BlockMap map,
                                                                  const float* __restrict__ scales,
                                                                  int8_t* __restrict__ Xq8, int64_t ld8,
                                                                  uint8_t* __restrict__ Xq4, int64_t ld4,
                                                                  float* __restrict__ Sx) {
  grid_dep_wait();  // (no-op unless PDL-launched behind a kernel that reads this call's outputs)
  grid_dep_launch();
  const int half_id = threadIdx.x >> 4;
  const int o = threadIdx.x & 15;
  const int64_t m = (int64_t)blockIdx.x * 8 + (half_id & 7);
  const int b = blockIdx.y * 2 + (half_id >> 3);
  if (m >= ldsx || b >= nb) return;
  if (m >= M) {
    if (o == 0) Sx[(int64_t)b * ldsx + m] = 1.0f;
    return;
  }
  float x[8];
  load_octet<kPerm>(X, ldx, m, b, o, perm, x);
  const uint32_t code = map.code[b];
  const bool is8 = (code >> 15) != 0;
  const int rank = code & 0x7FFF;
  const int qmax = is8 ? 127 : 7;
  const float s = __ldg(scales + b);
  int32_t q[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float v = __fdiv_rn(x[j], s);
    // |v| >= 2^23 (incl. inf) is already beyond any qmax: clamp by sign
    q[j] = fabsf(v) >= 8388608.0f ? (v > 0.0f ? qmax : -qmax) : min(qmax, max(-qmax, round_half_away(v)));
  }
  if (is8) {
    uint32_t lo = (uint32_t)(q[0] & 0xFF) | ((uint32_t)(q[1] & 0xFF) << 8) | ((uint32_t)(q[2] & 0xFF) << 16) |
                  ((uint32_t)(q[3] & 0xFF) << 24);
    uint32_t hi = (uint32_t)(q[4] & 0xFF) | ((uint32_t)(q[5] & 0xFF) << 8) | ((uint32_t)(q[6] & 0xFF) << 16) |
                  ((uint32_t)(q[7] & 0xFF) << 24);
    *reinterpret_cast<uint2*>(Xq8 + m * ld8 + (int64_t)rank * 128 + o * 8) = make_uint2(lo, hi);
  } else {
    *reinterpret_cast<uint32_t*>(Xq4 + m * ld4 + (int64_t)rank * 64 + o * 4) = pack_int4_word(q);
  }
  if (o == 0) Sx[(int64_t)b * ldsx + m] = s;
}

// ---- f4: FP16 weight-scale storage ----------------
// Per (row n, group of g permuted channels): a = max |w|, s = fp16_rn(fp32(a /
// 7)) (a == 0 -> 1, a nonzero s that underflows -> 2^-24), q = clamp(rha(fp32(
// w / s)), -7, 7) -- the scale the weights are quantized with is the stored
// fp16 one.  Warp per (row, group) for g = 128 (lane = 4 channels), warp per
// row for g = K; packed into the tiled layout like comet_pack_weight.
template <bool kPerm, bool kBf16S = false>
__global__ void __launch_bounds__(256) pack_weight_f16s_kernel(const __half* __restrict__ W, int64_t ldw, int N, int K,
                                                               int group, const int32_t* __restrict__ perm,
                                                               uint8_t* __restrict__ Wq, uint16_t* __restrict__ Sw) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ng = K / group;
  const int64_t item = (int64_t)blockIdx.x * 8 + warp;  // (row, group)
  if (item >= (int64_t)N * ng) return;
  const int64_t n = item / ng;
  const int j = (int)(item % ng);
  const unsigned short* row = reinterpret_cast<const unsigned short*>(W + n * ldw);
  float a = 0.0f;
  for (int i = lane; i < group; i += 32) {
    const int c = j * group + i;
    a = fmaxf(a, fabsf(half_bits_to_float(row[kPerm ? __ldg(perm + c) : c])));
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, off));
  // the stored scale: fp16 (kBf16S false) or bf16 bits of RN(a / 7)
  uint16_t sbits;
  float sf;
  if (kBf16S) {
    const __nv_bfloat16 sb = __float2bfloat16_rn(a != 0.0f ? __fdiv_rn(a, 7.0f) : 1.0f);  // bf16 keeps fp32's range
    sbits = __bfloat16_as_ushort(sb);
    sf = __bfloat162float(sb);
  } else {
    __half sh = __float2half_rn(1.0f);
    if (a != 0.0f) {
      sh = __float2half_rn(__fdiv_rn(a, 7.0f));
      if (__half2float(sh) == 0.0f) sh = __ushort_as_half((unsigned short)1);  // 2^-24
    }
    sbits = __half_as_ushort(sh);
    sf = __half2float(sh);
  }
  // each lane packs whole 8-value words of the group: word w covers channels 8w .. 8w+7
  for (int w = lane; w < group / 8; w += 32) {
    int32_t q[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = j * group + 8 * w + e;
      const float v = __fdiv_rn(half_bits_to_float(row[kPerm ? __ldg(perm + c) : c]), sf);
      q[e] = fabsf(v) >= 8388608.0f ? (v > 0.0f ? 7 : -7) : min(7, max(-7, round_half_away(v)));
    }
    *reinterpret_cast<uint32_t*>(Wq + wq_tiled_offset(n, ((int64_t)j * group + 8 * w) / 2, K / 128)) =
        pack_int4_word(q);
  }
  if (lane == 0) Sw[(int64_t)j * N + n] = sbits;
}

// fp16 scales -> the fp32 scales the GEMM kernels read (per GEMM call, into the workspace)
template <bool kBf16S>
__global__ void __launch_bounds__(256) widen_scales_kernel(const uint16_t* __restrict__ in, int64_t n,
                                                           float* __restrict__ out) {
  grid_dep_wait();  // PDL: a preceding GEMM on the same workspace may still read the widened scales
  grid_dep_launch();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = kBf16S ? __uint_as_float((uint32_t)in[i] << 16) : __half2float(__ushort_as_half(in[i]));
}

// ---- f3: dequant-in-attention over the KV4 cache (§3.2, §6.1) ----
// One decode query per head: o_h = softmax(scale * q_h . K^_h^T) V^_h with
// K^, V^ = fp16_rn((q - zp) * s) of the KV4 cache (the dequantisation
// kv4_dequantize_kernel applies), never materialised in HBM: the cache is read
// packed (0.5 B per element + its group parameters).  Split over tokens
// (kAttChunk per CTA, flash-decoding style): each CTA writes (max, sum, o[128])
// of its chunk, attn_kv4_combine_kernel merges the splits.  D = 128.
constexpr int kAttD = 128;
constexpr int kAttChunk = 512;  // tokens per CTA: 8 warps x 64 consecutive tokens
constexpr int kAttPart = kAttD + 2;

// 16 channels c .. c+15 of one token from a packed KV4 row (8 bytes, channel
// pairs), dequantised and rounded to fp16 exactly as kv4_dequantize_kernel:
// fp16_rn(fp32((n - zp) * s)); n - zp via the exact 2^23 magic (no I2F)
struct Kv4Par {
  float s[16];
  float zf[16];  // 2^23 + zp
};
DEVI void kv4_load_par(const float* __restrict__ sc, const uint8_t* __restrict__ zp, int64_t off, Kv4Par& p) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 s4 = __ldg(reinterpret_cast<const float4*>(sc + off) + k);
    p.s[4 * k] = s4.x; p.s[4 * k + 1] = s4.y; p.s[4 * k + 2] = s4.z; p.s[4 * k + 3] = s4.w;
  }
  const uint4 z = __ldg(reinterpret_cast<const uint4*>(zp + off));
  const uint32_t zw[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
  for (int j = 0; j < 16; ++j) p.zf[j] = 8388608.0f + (float)((zw[j >> 2] >> (8 * (j & 3))) & 0xFF);
}
DEVI void kv4_deq16(uint2 w, const Kv4Par& p, float (&v)[16]) {
  const uint32_t ww[2] = {w.x, w.y};
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const uint32_t n = (ww[j >> 3] >> (4 * (j & 7))) & 0xF;
    const float d = __fadd_rn(__uint_as_float(0x4B000000u | n), -p.zf[j]);  // n - zp, exact
    v[j] = __half2float(__float2half_rn(__fmul_rn(d, p.s[j])));
  }
}

// CTA = (head, chunk of kAttChunk tokens), 8 warps; a warp walks 64
// consecutive tokens 4 at a time: lanes 8i .. 8i+7 hold token i of the four,
// 16 channels each (one 8-byte load of the packed row), 3-step reduction per
// token for the scores; the values pass keeps 16 running sums per lane.
__global__ void __launch_bounds__(256) attn_kv4_split_kernel(const __half* __restrict__ q,
                                                             const uint8_t* __restrict__ Kq,
                                                             const float* __restrict__ Ks,
                                                             const uint8_t* __restrict__ Kz,
                                                             const uint8_t* __restrict__ Vq,
                                                             const float* __restrict__ Vs,
                                                             const uint8_t* __restrict__ Vz, int T, int H, int G,
                                                             float scale, float* __restrict__ part) {
  __shared__ float sc[kAttChunk];
  __shared__ float red[8][kAttD];
  __shared__ float wred[8];
  const int h = blockIdx.x, split = blockIdx.y;
  const int t0 = split * kAttChunk, t1 = min(T, t0 + kAttChunk);
  const int C = H * kAttD;
  const int64_t rowb = C / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane >> 3, cg = lane & 7;          // token of the four, channel group
  const int c = h * kAttD + 16 * cg;                 // this lane's 16 channels
  for (int i = threadIdx.x; i < kAttChunk; i += blockDim.x) sc[i] = -INFINITY;
  float qv[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) qv[j] = __half2float(q[h * kAttD + 16 * cg + j]) * scale;
  __syncthreads();
  const int w0 = t0 + warp * 64, w1 = min(t1, w0 + 64);
  Kv4Par par;
  int g = -1;
  for (int tb = w0; tb < w1; tb += 4) {
    const int t = tb + sub;
    float d = 0.f;
    if (t < w1) {
      if (t / G != g) {  // warp-divergent only across a group boundary
        g = t / G;
        kv4_load_par(Ks, Kz, (int64_t)g * C + c, par);
      }
      float k[16];
      kv4_deq16(__ldg(reinterpret_cast<const uint2*>(Kq + (int64_t)t * rowb + (c >> 1))), par, k);
#pragma unroll
      for (int j = 0; j < 16; ++j) d = fmaf(k[j], qv[j], d);
    }
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
    if (cg == 0 && t < w1) sc[t - t0] = d;
  }
  __syncthreads();
  float m = -INFINITY;
  for (int i = threadIdx.x; i < kAttChunk; i += blockDim.x) m = fmaxf(m, sc[i]);
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  if (lane == 0) wred[warp] = m;
  __syncthreads();
  m = wred[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) m = fmaxf(m, wred[w]);
  __syncthreads();
  float l = 0.f;
  for (int i = threadIdx.x; i < kAttChunk; i += blockDim.x) {
    const float p = t0 + i < t1 ? expf(sc[i] - m) : 0.f;
    sc[i] = p;
    l += p;
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
  if (lane == 0) wred[warp] = l;
  __syncthreads();
  float o[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j] = 0.f;
  g = -1;
  for (int tb = w0; tb < w1; tb += 4) {
    const int t = tb + sub;
    if (t < w1) {
      if (t / G != g) {
        g = t / G;
        kv4_load_par(Vs, Vz, (int64_t)g * C + c, par);
      }
      float v[16];
      kv4_deq16(__ldg(reinterpret_cast<const uint2*>(Vq + (int64_t)t * rowb + (c >> 1))), par, v);
      const float p = sc[t - t0];
#pragma unroll
      for (int j = 0; j < 16; ++j) o[j] = fmaf(p, v[j], o[j]);
    }
  }
  // the four token lanes of each channel group, then the warps
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    o[j] += __shfl_xor_sync(0xffffffffu, o[j], 8);
    o[j] += __shfl_xor_sync(0xffffffffu, o[j], 16);
  }
  if (sub == 0) {
#pragma unroll
    for (int j = 0; j < 16; ++j) red[warp][16 * cg + j] = o[j];
  }
  __syncthreads();
  float* dst = part + ((int64_t)h * gridDim.y + split) * kAttPart;
  if (threadIdx.x < kAttD) {
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) acc += red[w][threadIdx.x];
    dst[2 + threadIdx.x] = acc;
  }
  if (threadIdx.x == 0) {
    float ls = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) ls += wred[w];
    dst[0] = m;
    dst[1] = ls;
  }
}

// merge the splits of every head: o = sum_s e^(m_s - M) o_s / sum_s e^(m_s - M) l_s
__global__ void __launch_bounds__(kAttD) attn_kv4_combine_kernel(const float* __restrict__ part, int S,
                                                                 __half* __restrict__ out) {
  const int h = blockIdx.x;
  const float* p = part + (int64_t)h * S * kAttPart;
  float M = -INFINITY;
  for (int s = 0; s < S; ++s) M = fmaxf(M, p[s * kAttPart]);
  float L = 0.f, o = 0.f;
  for (int s = 0; s < S; ++s) {
    const float e = expf(p[s * kAttPart] - M);
    L = fmaf(e, p[s * kAttPart + 1], L);
    o = fmaf(e, p[s * kAttPart + 2 + threadIdx.x], o);
  }
  out[h * kAttD + threadIdx.x] = __float2half_rn(o / L);
}

}  // namespace comet
