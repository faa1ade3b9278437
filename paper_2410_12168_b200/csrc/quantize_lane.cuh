// quantize_lane.cuh -- a1 + a2 (FMPQ activation quantize/pack with the fused
// channel gather, P:L185 + P:L194 §3.2) for prefill-sized M (>= 512 rows):
// one THREAD per 64 channels of a (row, 128-channel block) item.
//
// Why lanes own their channels: the half-warp-per-item kernels (quantize.cuh)
// spend more instructions on the per-item shuffle trees (absmax, sum q), the
// scale division and the per-element gather addressing than on the
// quantization itself (~20 lane instructions per element, issue-bound at
// 2 TB/s with the permutation).  Here a lane owns 64 channels of a block (its
// partner lane the other 64): the absmax is a register reduction plus one
// shuffle, the scale pair is computed once per 64 elements.
//
// Data flow (persistent CTAs, as many per SM as shared memory allows):
//   * a stage = R consecutive rows (R * K / 64 sub-items = the compute lanes,
//     ~256 with the permutation, ~512 without); a producer warp brings each
//     row in with one 1-D bulk copy into an S-deep ring of stages (mbarrier
//     complete_tx);
//   * gather: the lane reads its 64 source channels from the staged row with
//     2-byte shared loads at offsets from a per-CTA table built once from the
//     permutation; without one, rotated 16-byte loads of the contiguous run;
//   * bank conflicts: lanes of a warp hold consecutive sub-blocks, whose
//     source positions (for the mostly monotone FMPQ permutation: outliers
//     first, the rest in order) are 128 B apart -- the same bank.  Each
//     sub-block's walk is therefore ROTATED by rho_c (even) so that lane c
//     starts on bank c mod 32: step j reads position (j + rho_c) mod 64, which
//     for a monotone run lands on bank (c + j/2) mod 32.  The table stores the
//     offsets in walk order (u32, per sub-block 16 chunks of 4, XOR-swizzled
//     for conflict-free 16-byte reads);
//   * after all lanes of a ROW finished gathering (named barrier per row),
//     each lane quantizes and writes its 64 output bytes back IN PLACE into
//     its row's staging slot (INT4 plane part first, then the INT8 part),
//     undoing the rotation with one byte-permute per word and a rotated word
//     address;
//   * the producer bulk-stores each row's plane segments to global memory and
//     refills the slot once the store has read it.
// Output is bit-identical to quantize_act_kernel / quantize_act_rows_kernel
// (same rounding sequence: a = max |x|, s = a / qmax, r = qmax / a (IEEE
// divisions), q = round_half_away(fl(x * r)), see quantize.cuh).
//
// Variants: kE4 -- INT4 blocks as the prefill GEMM's e4m3 operand (|q| |
// sign << 7, 128 B per row-block) plus CX = 8 sum(q) (comet_w4ax_linear);
// else the packed INT4 plane (O4 nibble order, 64 B).  INT8 blocks are
// two's-complement bytes in both.  kBf16: bf16 activations (f4).
#pragma once
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "sm100.cuh"
#include "quantize.cuh"

namespace comet {

constexpr int kLaneMaxSmem = 232448;  // sm_100 opt-in dynamic shared memory per CTA
#ifndef COMET_LANE_MIN_ROWS
#define COMET_LANE_MIN_ROWS 512
#endif
constexpr int kLaneMinRows = COMET_LANE_MIN_ROWS;  // below: the row-staged / item kernels (few stages, few CTAs)

struct LanePlan {
  int R = 0;        // rows per stage
  int S = 0;        // stages in the ring
  int lpr = 0;      // lanes per row
  int threads = 0;  // compute threads (multiple of 32) + one producer warp
  int smem = 0;     // dynamic shared memory bytes
  int64_t stages = 0;
};

#ifndef COMET_LANE_SUB
#define COMET_LANE_SUB 64  // channels per lane: 64 (two lanes per 128-channel item) or 128
#endif
constexpr int kLaneSub = COMET_LANE_SUB;
#ifndef COMET_LANE_THREADS
#define COMET_LANE_THREADS 256
#endif
#ifndef COMET_LANE_SMAX
#define COMET_LANE_SMAX 2
#endif
// compute lanes per CTA: the target (small CTAs, several per SM, so their
// stage waits and row barriers interleave) and the most a row may need (a
// row's lanes are whole warps of one CTA)
constexpr int kLaneMaxThreads = COMET_LANE_THREADS;
constexpr int kLaneRowMax = 512;
constexpr int kLaneSMax = COMET_LANE_SMAX;  // stages in the ring at most

// A row is handled by (K / kLaneSub) lanes ("sub-items": one lane per 128 /
// kLaneSub of a 128-channel block).  Lanes are laid out so that a warp never
// straddles two rows when a row needs >= 32 lanes (lpr = that count rounded
// up to 32: the in-place write waits only for the row's own warps); else a
// warp holds whole rows.  R rows per stage so that ~kLaneMaxThreads lanes
// work (one row when a row alone needs more, up to kLaneRowMax); S stages
// next to the gather table (u32 offsets, perm only); S >= 2 or the plan is
// empty (the row-staged kernel takes over).  The launch puts as many CTAs on
// an SM as shared memory allows (cudaOccupancy...).
// Measured (8192 rows, FMPQ permutation; 8B bench step): 256 lanes and
// 2 stages (two CTAs per SM up to K = 14336) against 512 lanes and 3 stages
// (one CTA per SM): K = 4096 42.0 -> 38.9 us, K = 8192 64.5 -> 61.4 us,
// K = 14336 equal, step 2.312 -> 2.284 ms.
// Without a permutation (contiguous 16-byte loads, no table) one big CTA
// per SM with 3 stages stays ahead: 16384 x 8192 65 vs 71 us, 8192 x 28672
// 115-126 vs 128 us.
constexpr int kLaneThreadsNoPerm = 512, kLaneSMaxNoPerm = 3;
inline LanePlan lane_plan(int M, int K, bool perm) {
  LanePlan p;
  const int nb = K / 128;
  const int nsub = K / kLaneSub;
  if (nb <= 0 || nsub > kLaneRowMax) return p;
  const int target = perm ? kLaneMaxThreads : kLaneThreadsNoPerm;
  int ncomp;
  if (nsub >= 32) {
    p.lpr = (nsub + 31) / 32 * 32;
    p.R = std::max(1, target / p.lpr);
    ncomp = p.R * p.lpr;
  } else {
    p.lpr = nsub;
    p.R = (target / 32) * (32 / nsub);
    ncomp = target;
  }
  if (p.lpr > 32 && p.R > 15) return LanePlan{};  // named barriers 1..15
  p.threads = ncomp + 32;
  const int stage = p.R * K * 2;
  const int fixed = (perm ? K * 4 : 0) + ((2 * nb + 15) / 16) * 16 + 128;  // table + rho + barriers (2 x 8)
  p.S = std::min(perm ? kLaneSMax : kLaneSMaxNoPerm, (kLaneMaxSmem - fixed) / stage);
  if (p.S < 2) return LanePlan{};
  p.smem = p.S * stage + fixed;
  p.stages = ((int64_t)M + p.R - 1) / p.R;
  return p;
}

DEVI void lane_bar_sync(int id, int nthreads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }
DEVI uint32_t lds_u16(uint32_t addr) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
DEVI void sts_u32(uint32_t addr, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory"); }
DEVI void sts_u64(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
// 1-D bulk copy own shared memory -> global (bulk-group completion)
DEVI void bulk_store(void* gdst, uint32_t smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(gdst)),
               "r"(smem_src), "r"(bytes)
               : "memory");
}

// |x| of the two halves of a packed bf16 pair as fp32 (exact)
DEVI uint64_t lane_abs_pair_bf16(uint32_t w) {
  const uint32_t aw = w & 0x7FFF7FFFu;
  return f2_pack(__uint_as_float(aw << 16), __uint_as_float(aw & 0xFFFF0000u));
}

// gather of the lane's kLaneSub channels (sub-item c) in walk order into
// packed pairs.  kPerm: 2-byte loads at the table's offsets from the row base
// `ubase` (one add per element: nvcc keeps the [reg + uniform reg] form only
// outside thread-dependent control flow); else rotated 16-byte loads of the
// contiguous sub-block.
template <bool kPerm>
DEVI void lane_gather(uint32_t (&w)[kLaneSub / 2], uint32_t ubase, uint32_t tab_lane, int c) {
  constexpr int kC4 = kLaneSub / 4;  // table chunks of 4 offsets
  if constexpr (kPerm) {
    // the sub-item's table row: kC4 chunks, chunk j4 stored at j4 ^ (c & 7)
    // (the lanes' 16-byte reads spread over all bank groups; the eight chunk
    // bases cover every j4 with immediate offsets)
    uint32_t cb[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) cb[j] = tab_lane + ((j ^ (c & 7)) << 4);
#pragma unroll
    for (int j4 = 0; j4 < kC4; ++j4) {
      const uint4 pe = lds128(cb[j4 & 7] + (j4 >> 3) * 128);
      const uint32_t e0 = lds_u16(ubase + pe.x), e1 = lds_u16(ubase + pe.y);
      const uint32_t e2 = lds_u16(ubase + pe.z), e3 = lds_u16(ubase + pe.w);
      w[2 * j4] = __byte_perm(e0, e1, 0x5410);
      w[2 * j4 + 1] = __byte_perm(e2, e3, 0x5410);
    }
  } else {
    // walk chunk k = chunk (k + c) mod kC8 of the sub-block: the lanes of a
    // warp (consecutive c) spread over the 8 bank groups
    constexpr int kC8 = kLaneSub / 8;
    const uint32_t blk = ubase + c * (kLaneSub * 2);
#pragma unroll
    for (int k = 0; k < kC8; ++k) {
      const uint4 v = lds128(blk + (((k + c) & (kC8 - 1)) << 4));
      w[4 * k] = v.x, w[4 * k + 1] = v.y, w[4 * k + 2] = v.z, w[4 * k + 3] = v.w;
    }
  }
}

// __launch_bounds__ thread counts, i.e. the register caps (the launches use
// <= kLaneMaxThreads + 32 threads either way): the packed-plane variant is
// 5-11% faster capped at 80 registers (bound 672: 8192 x 14336 FMPQ 114 ->
// 102 us, 8192 x 28672 217 -> 203 us, 8192 x 4096 unchanged; a bound of 768,
// also 80 registers, measured slower: the schedule differs); the e4m3
// variant of comet_w4ax_linear at 80 registers (bound 704) saves ~4 us on
// the 8B down projection and is neutral on the K = 4096 layers
#ifndef COMET_LANE_LB_PK
#define COMET_LANE_LB_PK 672
#endif
#ifndef COMET_LANE_LB_E4
#define COMET_LANE_LB_E4 704
#endif
template <bool kE4, bool kBf16, bool kPerm>
__global__ void __launch_bounds__(kE4 ? COMET_LANE_LB_E4 : COMET_LANE_LB_PK, 1)
    quantize_lane_kernel(const __half* __restrict__ X, int64_t ldx, int M, int nb, int64_t ldsx,
                         const int32_t* __restrict__ perm, const __grid_constant__ BlockMap map,
                         int8_t* __restrict__ Xq8, int64_t ld8, uint8_t* __restrict__ Xo4, int64_t ld4,
                         float* __restrict__ Sx, float* __restrict__ CX, int R, int S, int lpr) {
  constexpr int kSub = kLaneSub;
  constexpr int kW = kSub / 2;       // packed pairs per lane
  constexpr int kSpb = 128 / kSub;   // lanes per 128-channel block
  extern __shared__ __align__(128) uint8_t lsm[];
  grid_dep_wait();    // PDL launch: the preceding kernel (which may read this call's outputs) is complete
  grid_dep_launch();  // the GEMM that follows may get scheduled (PDL)
  const int K = nb * 128;
  const int nsub = nb * kSpb;
  const int ncomp = (int)blockDim.x - 32;
  const int stage_bytes = R * K * 2;
  uint8_t* stages = lsm;
  uint32_t* tab = reinterpret_cast<uint32_t*>(lsm + (size_t)S * stage_bytes);
  uint8_t* rho = reinterpret_cast<uint8_t*>(lsm + (size_t)S * stage_bytes + (kPerm ? K * 4 : 0));
  uint64_t* full = reinterpret_cast<uint64_t*>(rho + ((2 * nb + 15) / 16) * 16);
  uint64_t* outready = full + 8;
  const int tid = threadIdx.x;
  const int n4 = [&] {
    int c = 0;
    for (int b = 0; b < nb; ++b) c += (map.code[b] >> 15) ? 0 : 1;
    return c;
  }();
  const int w4 = kE4 ? 128 : 64;  // INT4 bytes per row-block

  // ---- per-CTA gather table (once) ----
  // rho_c: rotation (in elements) of sub-item c's walk.  With the permutation:
  // so that lane (c mod 32) starts on bank c mod 32 (even: whole fp16 pairs; a
  // multiple of 4 for the packed INT4 plane, whose octets must stay
  // word-aligned); the source of the sub-block's middle stands for the run.
  // Without: 8 (c mod kSub/8), the 16-byte chunk rotation of lane_gather.
  for (int c = tid; c < nsub; c += blockDim.x) {
    int rr;
    if (kPerm) {
      const int base = min(max(__ldg(perm + c * kSub + kSub / 2), 0), K - 1) - kSub / 2;
      rr = (2 * (c & 31) - (base & ~1)) & (kSub - 1);
      if (!kE4 && !(map.code[c / kSpb] >> 15)) rr &= ~3;
    } else {
      rr = 8 * (c & (kSub / 8 - 1));
    }
    rho[c] = (uint8_t)rr;
  }
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&outready[i], ncomp / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  const int64_t nst = ((int64_t)M + R - 1) / R;
  const uint32_t stage0 = smem_u32(stages);
  auto load = [&](int64_t st, int buf) {  // (producer thread)
    const int64_t m0 = st * R;
    const int rv = (int)min((int64_t)R, (int64_t)M - m0);
    mbar_arrive_expect_tx(&full[buf], (uint32_t)(rv * K * 2));
    for (int r = 0; r < rv; ++r)
      bulk_load(stages + (size_t)buf * stage_bytes + (size_t)r * K * 2, X + (m0 + r) * ldx, (uint32_t)K * 2,
                &full[buf]);
  };
  // the first S stages are in flight while the table is built
  if (tid == ncomp)
    for (int i = 0; i < S && blockIdx.x + i * G < nst; ++i) load(blockIdx.x + i * G, i);
  if (kPerm) {
    // eight independent permutation loads in flight per thread (the loop is
    // otherwise one L2 round trip per entry)
    for (int i0 = tid; i0 < K; i0 += 8 * blockDim.x) {
      int src[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * blockDim.x;
        src[u] = i < K ? __ldg(perm + (i & ~(kSub - 1)) + (((i & (kSub - 1)) + rho[i / kSub]) & (kSub - 1))) : 0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < K) {
          const int c = i / kSub, p = i & (kSub - 1);
          tab[(c * (kSub / 4) + ((p >> 2) ^ (c & 7))) * 4 + (p & 3)] = (uint32_t)(2 * min(max(src[u], 0), K - 1));
        }
      }
    }
    __syncthreads();
  }

  if (tid >= ncomp) {  // ---- producer warp ----
    if (tid == ncomp) {
      int64_t st = blockIdx.x;
      for (int it = 0; st < nst; ++it, st += G) {
        const int buf = it % S;
        mbar_wait_sleep(&outready[buf], (it / S) & 1);  // (descheduled while it waits: its polling shares an SMSP with compute warps)
        const int64_t m0 = st * R;
        const int rv = (int)min((int64_t)R, (int64_t)M - m0);
        for (int r = 0; r < rv; ++r) {
          const uint32_t src = stage0 + buf * stage_bytes + r * K * 2;
          if (n4) bulk_store(Xo4 + (m0 + r) * ld4, src, (uint32_t)(n4 * w4));
          if (nb - n4) bulk_store(Xq8 + (m0 + r) * ld8, src + n4 * w4, (uint32_t)((nb - n4) * 128));
        }
        bulk_commit_group();
        if (st + S * G < nst) {
          bulk_wait_group_read0();  // the slot is free once the stores have read it
          load(st + S * G, buf);
        }
      }
      bulk_wait_group0();
    }
    return;
  }

  // ---- compute threads: sub-item (r, c), c = kSpb * b + h ----
  const int wid = tid >> 5, lane = tid & 31;
  int r, c;
  bool active;
  if (lpr >= 32) {  // whole warps per row (an idle lane keeps its row: it takes the row's named barrier)
    r = tid / lpr;
    c = tid % lpr;
    active = c < nsub;
    if (!active) c = 0;
  } else {  // whole rows per warp (an idle lane works on the warp's first row and stores nothing)
    const int rpw = 32 / nsub;
    active = lane < rpw * nsub;
    r = wid * rpw + (active ? lane / nsub : 0);
    c = active ? lane % nsub : 0;
  }
  const int b = c / kSpb, h = c % kSpb;
  const uint32_t code = map.code[b];
  const bool is8 = (code >> 15) != 0;
  const int rank = code & 0x7FFF;
  const int rr = rho[c];
  const float qmax = is8 ? 127.0f : 7.0f;
  const uint32_t tab_lane = smem_u32(tab) + c * (kSub * 4);
  // output slot of this sub-item (bytes from the row's staging start)
  const uint32_t out_slot = is8 ? (uint32_t)(n4 * w4 + rank * 128 + h * kSub)
                                : (uint32_t)(rank * w4 + h * (w4 * kSub / 128));

  int it = 0;
  for (int64_t st = blockIdx.x; st < nst; st += G, ++it) {
    const int buf = it % S;
    const int64_t m = st * R + r;
    const bool valid = active && m < M;
    mbar_wait(&full[buf], (it / S) & 1);
    const uint32_t sbase = stage0 + buf * stage_bytes;
    uint32_t w[kW];
    lane_gather<kPerm>(w, sbase + r * K * 2, tab_lane, c);
    // absmax of the block (the lane's values, then its partner lanes')
    float a;
    if constexpr (kBf16) {  // integer max of the sign-cleared patterns (monotone for non-negative floats)
      uint32_t am = 0;
#pragma unroll
      for (int j = 0; j < kW; j += 2) am = __vmaxu2(am, __vmaxu2(w[j] & 0x7FFF7FFFu, w[j + 1] & 0x7FFF7FFFu));
      a = act_bits_to_float<true>(max(am & 0xFFFFu, am >> 16));
    } else {  // three-input |.| max on fp16 pairs (VHMNMX)
      __half2 hm = __habs2(*reinterpret_cast<const __half2*>(&w[0]));
#pragma unroll
      for (int j = 1; j < kW - 1; j += 2)
        hm = __hmax2(hm, __hmax2(__habs2(*reinterpret_cast<const __half2*>(&w[j])),
                                 __habs2(*reinterpret_cast<const __half2*>(&w[j + 1]))));
      hm = __hmax2(hm, __habs2(*reinterpret_cast<const __half2*>(&w[kW - 1])));
      a = fmaxf(__low2float(hm), __high2float(hm));
    }
#pragma unroll
    for (int o = 1; o < kSpb; o <<= 1) a = fmaxf(a, __shfl_xor_sync(0xFFFFFFFFu, a, o));
    float s = 1.0f, rcp = 0.0f;
    if (a != 0.0f) {
      s = __fdiv_rn(a, qmax);
      rcp = __fdiv_rn(qmax, a);
    }
    // the row's lanes all hold their items: its staging slot may be overwritten
    if (lpr > 32)
      lane_bar_sync(1 + r, lpr);
    else
      __syncwarp();
    // quantize: t = RD(RZ(|x| r + 0.5) + M) = M + |q| (quantize.cuh, rha_bits)
    const uint64_t r2 = f2_pack(rcp, rcp), half2 = f2_pack(0.5f, 0.5f), M2 = f2_pack(12582912.0f, 12582912.0f);
    uint32_t ob[kW / 2];  // output bytes in walk order, 4 per word
    int qs = 0;
#pragma unroll
    for (int g = 0; g < kW / 2; ++g) {
      uint32_t t0, t1, t2w, t3;
      uint64_t x01, x23;
      if constexpr (kBf16) {
        x01 = lane_abs_pair_bf16(w[2 * g]);
        x23 = lane_abs_pair_bf16(w[2 * g + 1]);
      } else {  // |x| folded into the fp16 -> fp32 conversion
        const __half2 h01 = *reinterpret_cast<const __half2*>(&w[2 * g]);
        const __half2 h23 = *reinterpret_cast<const __half2*>(&w[2 * g + 1]);
        x01 = f2_pack(__half2float(__habs(__low2half(h01))), __half2float(__habs(__high2half(h01))));
        x23 = f2_pack(__half2float(__habs(__low2half(h23))), __half2float(__habs(__high2half(h23))));
      }
      f2_unpack(f2_add_rm(f2_add_rz(f2_mul(x01, r2), half2), M2), t0, t1);
      f2_unpack(f2_add_rm(f2_add_rz(f2_mul(x23, r2), half2), M2), t2w, t3);
      const uint32_t mag = __byte_perm(__byte_perm(t0, t1, 0x0040), __byte_perm(t2w, t3, 0x0040), 0x5410);
      const uint32_t sg = sign_bytes4(w[2 * g], w[2 * g + 1]);  // 0xFF per negative element
      if (kE4 && !is8) {
        qs = __dp4a((int)mag, (int)(sg | 0x01010101u), qs);
        ob[g] = mag | (sg & 0x80808080u);
      } else {
        // two's complement bytes: -|q| for negative elements with q != 0
        const uint32_t neg = (mag + 0x7F7F7F7Fu) & sg & 0x80808080u;
        const uint32_t m1 = neg >> 7;
        ob[g] = (mag ^ (neg | (neg - m1))) + m1;
      }
    }
    if (kE4) {
#pragma unroll
      for (int o = 1; o < kSpb; o <<= 1) qs += __shfl_xor_sync(0xFFFFFFFFu, qs, o);
    }
    if (valid) {
      constexpr int kOW = kSub / 4;  // output words (byte forms) of the sub-item
      const uint32_t slot = sbase + r * K * 2 + out_slot;
      if (!kPerm) {
        // walk chunk k = output bytes 8 ((k + c) mod kSub/8) .. +7 (packed INT4: 4 bytes)
        constexpr int kC8 = kSub / 8;
        if (kE4 || is8) {
#pragma unroll
          for (int k = 0; k < kC8; ++k) sts_u64(slot + 8 * ((k + c) & (kC8 - 1)), ob[2 * k], ob[2 * k + 1]);
        } else {
#pragma unroll
          for (int k = 0; k < kC8; ++k) {
            uint32_t pk;
            asm("lop3.b32 %0, %1, %2, 0x0F0F0F0F, 0xD8;" : "=r"(pk) : "r"(ob[2 * k + 1] << 4), "r"(ob[2 * k]));
            sts_u32(slot + 4 * ((k + c) & (kC8 - 1)), pk);
          }
        }
      } else if (kE4 || is8) {
        // walk word g holds output bytes 4g + rr .. 4g + rr + 3 (mod kSub)
        const int q = rr >> 2, p = (rr >> 1) & 1;
        const uint32_t sel = p ? 0x5432u : 0x3210u;
#pragma unroll
        for (int g = 0; g < kOW; ++g)
          sts_u32(slot + 4 * ((g + q + p) & (kOW - 1)), __byte_perm(ob[g], ob[(g + 1) & (kOW - 1)], sel));
      } else {
        // packed INT4 (O4: byte j of an octet = q_j | q_{j+4} << 4), rr % 4 == 0
        const int q = rr >> 2, odd = q & 1;
#pragma unroll
        for (int k = 0; k < kOW / 2; ++k) {
          const uint32_t lo = odd ? ob[2 * k + 1] : ob[2 * k];
          const uint32_t hi = odd ? ob[(2 * k + 2) & (kOW - 1)] : ob[2 * k + 1];
          uint32_t pk;
          asm("lop3.b32 %0, %1, %2, 0x0F0F0F0F, 0xD8;" : "=r"(pk) : "r"(hi << 4), "r"(lo));
          sts_u32(slot + 4 * ((k + ((q + 1) >> 1)) & (kOW / 2 - 1)), pk);
        }
      }
      if (h == 0) {
        Sx[(int64_t)b * ldsx + m] = s;
        if (kE4 && !is8) CX[(int64_t)rank * ldsx + m] = 8.0f * (float)qs;
      }
    }
    fence_proxy_async_smem();  // the bulk store (async proxy) reads what this thread wrote
    __syncwarp();
    if (lane == 0) mbar_arrive(&outready[buf]);
  }
  // padding rows of the scale layout
  if (blockIdx.x == 0)
    for (int64_t i = tid; i < (ldsx - M) * nb; i += ncomp) {
      const int64_t mm = M + i / nb;
      const int bb = (int)(i % nb);
      Sx[(int64_t)bb * ldsx + mm] = 1.0f;
      if (kE4 && !(map.code[bb] >> 15)) CX[(int64_t)(map.code[bb] & 0x7FFF) * ldsx + mm] = 0.0f;
    }
}

}  // namespace comet
