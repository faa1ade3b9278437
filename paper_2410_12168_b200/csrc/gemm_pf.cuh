// gemm_pf.cuh -- prefill W4Ax GEMM (M > 128 tokens) on CTA pairs
// (tcgen05 cta_group::2), persistent over pair tiles of 256 tokens x 192
// weight rows, K walked one 128-channel FMPQ block at a time.
//
// Per block, one MMA item of 4 x K=32 tcgen05.mma (M=256, N=192) into one of
// two 192-column TMEM accumulators, so the promotion of block b overlaps the
// MMAs of block b+1 (the paper's overlap of conversion and MMA):
//   INT4 block (W4A4): kind::f8f6f4, e4m3 x e4m3 -> fp32.  Tokens are
//       q * 2^-9 (exact e4m3 subnormals, written by the quantizer in
//       comet_w4ax_linear or by prep_tokens_kernel), weights (q + 8) * 2^-9
//       (the nibble XOR 8: e4m3 bytes 0..15 are exactly u * 2^-9).  Every
//       product is an exact multiple of 2^-18 and the tensor core's fp32 sum
//       of them is exact (|sum| < 2^15 * 2^-18; tools/microbench_fp8.cu checks
//       it against the integer sum), so the accumulator holds
//       D = 2^-18 (acc + 8 sum xq) with acc the INT32 block sum of O6, already
//       in fp32: the promotion needs no int -> float conversion.
//   INT8 block (W4A8): kind::i8, xq x 16*wq -> int32 (the zero extension
//       "multiplied by 16"), promoted with cvt.rn.f32.s32.
// A (tokens) and B (weights) are shared-memory operands (SS MMA): A is a TMA
// box of the CTA's 128 token rows x 128 B (SW128; the INT8 plane or the e4m3
// token plane), B the CTA's 96 packed weight rows expanded by the staging
// warps into a SW128 K-major stage.
//
// Roles per CTA (19 warps = 608 threads, 96 registers; registers are
// allocated to warps in groups of four, so a 21st warp would cost 80):
//   warps 0-11  (a6, a8) promotion: thread = token row (TMEM lane), 64
//           columns read with double-buffered tcgen05.ld x8, the accumulator
//           released after its last load; running sums in registers; at the
//           tile's last block fp16 RNE -> a 32 x 32 smem box per warp -> TMA
//           tensor store
//   warp 12 (a3) token + scale producer: TMA of the token block, bulk copies
//           of Sx, the e4m3 correction 8*sum(xq) and the weight scales
//   warp 13 (a5) MMA issuer (leader CTA only), commits to both CTAs
//   warp 14 (a3) weight producer: 1-D bulk copies of the tiled packed rows
//   warps 15-18 (a4) staging: packed weight chunks -> e4m3 (INT4 block) or
//           INT8 x16 (INT8 block) in the SW128 B stage
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "gemm.cuh"
#include "quantize.cuh"
#include "sm100.cuh"

namespace comet {

// ---- a4: INT4 -> MMA operand bytes (8 values per packed 32-bit word; lo =
// elements 0..3, hi = elements 4..7, the order of the O4 nibble layout) -----
// INT8 x16 (zero extension): lo = (w << 4) & 0xF0F0F0F0, hi = w & 0xF0F0F0F0
DEVI void zext_word(uint32_t w, uint32_t& lo, uint32_t& hi) {
  uint32_t t;
  asm("and.b32 %0, %1, 0x0F0F0F0F;" : "=r"(t) : "r"(w));
  asm("mul.lo.u32 %0, %1, 16;" : "=r"(lo) : "r"(t));
  asm("mad.lo.u32 %0, %1, 0xFFFFFFFF, %2;" : "=r"(hi) : "r"(t), "r"(w));
}
// e4m3 of (q + 8) * 2^-9: the two's-complement nibble XOR 8 is q + 8 in
// [1, 15] (q in [-7, 7]), and e4m3 byte u in [0, 15] encodes u * 2^-9
// exactly (0..7 subnormal, 8..15 the first binade)
DEVI void e4m3_offset_word(uint32_t w, uint32_t& lo, uint32_t& hi) {
  // (x & 0x0F0F0F0F) ^ 0x08080808 as one LOP3 each (LUT 0x6A = (a & b) ^ c)
  asm("lop3.b32 %0, %1, 0x0F0F0F0F, 0x08080808, 0x6A;" : "=r"(lo) : "r"(w));
  asm("lop3.b32 %0, %1, 0x0F0F0F0F, 0x08080808, 0x6A;" : "=r"(hi) : "r"(w >> 4));
}
template <bool kF8>
DEVI void mma_ss_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  if (kF8)
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Instruction descriptor, kind::f8f6f4: D f32, A e4m3, B e4m3, both K-major.
__host__ __device__ constexpr uint32_t idesc_e4m3(uint32_t M, uint32_t N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

DEVI uint64_t add2_u(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// y += (a0, a1) * s for fp32 accumulator values (one FFMA2)
DEVI void fma2_u(uint64_t& y, uint32_t a0, uint32_t a1, uint64_t s) {
  asm("{\n .reg .b64 p;\n mov.b64 p, {%1, %2};\n fma.rn.f32x2 %0, p, %3, %0;\n}\n"
      : "+l"(y)
      : "r"(a0), "r"(a1), "l"(s));
}
// y += ((a0, a1) * s + c) * w  (group-128 weight scales with the e4m3 offset correction c)
DEVI void fma2_corr_u(uint64_t& y, uint32_t a0, uint32_t a1, uint64_t s, uint64_t c, uint64_t w) {
  asm("{\n .reg .b64 p, t;\n mov.b64 p, {%1, %2};\n fma.rn.f32x2 t, p, %3, %4;\n"
      " fma.rn.f32x2 %0, t, %5, %0;\n}\n"
      : "+l"(y)
      : "r"(a0), "r"(a1), "l"(s), "l"(c), "l"(w));
}

struct PfCfg {
#ifndef PF_TILEN
#define PF_TILEN 192
#endif
#ifndef PF_SWARPS
#define PF_SWARPS 4
#endif
#ifndef PF_STAGES
#define PF_STAGES 4
#endif
  static constexpr int kTileN = PF_TILEN;       // weight rows per pair tile (MMA N)
  static constexpr int kRows = kTileN / 2;      // weight rows per CTA
#ifndef PF_PQ
#define PF_PQ (PF_TILEN / 64)
#endif
#ifndef PF_ACCS
#define PF_ACCS 2
#endif
  static constexpr int kPQ = PF_PQ;             // promotion warps per TMEM lane quarter
  static constexpr int kPWarps = 4 * kPQ;       // 16 promotion warps
  static constexpr int kWCols = kTileN / kPQ;   // 64 accumulator columns per promotion warp
  static constexpr int kSWarps = PF_SWARPS;     // staging warps
  static constexpr int kStages = PF_STAGES;     // operand stages (A + B), freed by the MMA commit
  static constexpr int kLStages = PF_STAGES;    // packed weight stages, freed by the staging warps
  static constexpr int kAccs = PF_ACCS;         // kTileN-column accumulators
  static constexpr int kScaleSlots = 8;
  static constexpr int kABytes = 128 * 128;     // token rows x 128 B (SW128)
  static constexpr int kBBytes = kRows * 128;   // expanded weight rows x 128 B (SW128)
  static constexpr int kWPBytes = kRows * 64;   // packed weight rows
  static constexpr int kABase = 0;
  static constexpr int kBBase = kABase + kStages * kABytes;
  static constexpr int kWPBase = kBBase + kStages * kBBytes;
  static constexpr int kScaleBase = kWPBase + kLStages * kWPBytes;
  static constexpr int kCxOff = 512;                          // sx[128] | cx[128] | sw[kTileN]
  static constexpr int kSwOff = 1024;
  static constexpr int kSlotBytes = kSwOff + kTileN * 4;
  static constexpr int kBarBase = kScaleBase + kScaleSlots * kSlotBytes;
  static constexpr int kBarBytes = 512;
  static constexpr int kFacBase = kBarBase + kBarBytes;       // float fac[nb]
  // a8: per promotion warp kYBoxes 32-row x 32-column fp16 boxes (2 KB each,
  // SW64) for the TMA stores of Y
#ifndef PF_YBOXES
#define PF_YBOXES 2
#endif
  static constexpr int kYBoxes = PF_YBOXES;
  static constexpr int kYWarpBytes = kYBoxes * 32 * 64;
  static constexpr int kYBase = (kFacBase + 512 * 4 + 1023) / 1024 * 1024;
  static constexpr int kSmemBytes = kYBase + kPWarps * kYWarpBytes + 1024;
  static_assert(kABase % 1024 == 0 && kBBase % 1024 == 0 && kBBytes % 1024 == 0, "SW128 operand alignment");
  static_assert(kWPBase % 128 == 0 && kScaleBase % 16 == 0, "alignment");
  static_assert(kSmemBytes <= 227 * 1024, "smem budget");
  static_assert(kAccs * kTileN <= 512, "TMEM budget");
  static_assert(kWCols % 16 == 0, "x16 TMEM loads");
  // Warp ids: promotion warps first (the warp schedulers favour low ids and
  // the promotion is the critical path), then the token producer, MMA issuer,
  // weight producer and staging warps.  Measured against producers-first
  // (0 load, 1 MMA, 2 weights, 3-6 staging, 7-18 promotion): 70B gate_up
  // 4041 -> 3906 us; MMA warp first (0 MMA, 1-12 promotion) 3919-3930 us.
  static constexpr int kPBase = 0, kLoadWarp = kPWarps, kMmaWarp = kPWarps + 1, kWLoadWarp = kPWarps + 2,
                       kStageWarp = kPWarps + 3;
  // (warps get registers in groups of four: up to 20 warps keep 96 registers per thread)
  static constexpr int kThreads = 32 * (3 + kSWarps + kPWarps);  // producers + MMA, staging, promotion
  static constexpr int kReadyCount = 2 * kSWarps;   // both CTAs' staging warps
  static constexpr int kTemptyCount = 2 * kPWarps;  // both CTAs' promotion warps
};

// Tile order: groups of group_m token tiles; inside a group the token tile
// runs fastest, then the weight tile.  The host sizes group_m so the group's
// token rows stay resident in L2 while every weight tile passes over them
// (group_m = m_tiles: one group, token tiles fastest, each weight tile read
// once; group_m = 1: weight tiles fastest, each token tile read once).
struct PfSched {
  int m_tiles, n_tiles, tiles, clusters, group_m;
  DEVI void coords(int t, int& m0, int& n0) const {
    const int per = group_m * n_tiles;
    const int g = t / per, r = t - g * per;
    const int gm = min(group_m, m_tiles - g * group_m);
    m0 = (g * group_m + r % gm) * 256;
    n0 = (r / gm) * PfCfg::kTileN;
  }
};

// a4 for the tokens, once per GEMM call: INT4 plane [M x n4*64 B] -> e4m3
// plane X4e [M x n4*128 B] (q * 2^-9, natural K order) and
// CX[r4 * ldsx + m] = 8 * sum_k xq[m, k] over INT4 block r4 (the correction
// of the offset e4m3 weights; 0 for the padding rows m in [M, ldsx)).
// Thread = (row, INT4 block, 16-byte chunk); 4 lanes per (row, block).
__global__ void __launch_bounds__(256) prep_tokens_kernel(const uint8_t* __restrict__ Xq4, int M, int n4,
                                                          int64_t ldsx, uint8_t* __restrict__ X4e,
                                                          float* __restrict__ CX) {
  grid_dep_launch();
  grid_dep_wait();  // the quantizer that wrote Xq4 may still run (PDL)
  const int64_t total = ldsx * n4 * 4;
  const unsigned gmask = 0xFu << (threadIdx.x & 28);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i & 3);
    const int64_t rb = i >> 2;
    const int r4 = (int)(rb % n4);
    const int64_t m = rb / n4;
    int sum = 0;
    if (m < M) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(Xq4 + (m * n4 + r4) * 64 + c * 16));
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      uint32_t o[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t lo = ws[j] & 0x0F0F0F0Fu, hi = (ws[j] >> 4) & 0x0F0F0F0Fu;  // e_j | e_{j+4}
        o[2 * j] = e4m3_signed4(lo);
        o[2 * j + 1] = e4m3_signed4(hi);
        // sum of the 8 signed nibbles: bytes of lo + hi minus 16 per negative one
        sum += __dp4a(lo + hi, 0x01010101u, 0u) - 2 * __dp4a((lo & 0x08080808u) + (hi & 0x08080808u), 0x01010101u, 0u);
      }
      uint4* dst = reinterpret_cast<uint4*>(X4e + (m * n4 + r4) * 128 + c * 32);
      __stcs(dst, make_uint4(o[0], o[1], o[2], o[3]));
      __stcs(dst + 1, make_uint4(o[4], o[5], o[6], o[7]));
    }
    sum += __shfl_xor_sync(gmask, sum, 1);
    sum += __shfl_xor_sync(gmask, sum, 2);
    if (c == 0) CX[(int64_t)r4 * ldsx + m] = 8.0f * (float)sum;
  }
}

// tmXe / tmX8: the e4m3 token plane / the INT8 plane ([M rows x 128 B per
// block], boxes of 128 x 128 B, SW128).  args.CX: prep_tokens_kernel's
// corrections.
// kAccOut: write per-block INT32 accumulators (debug entry).
template <bool kGroupK, bool kAccOut>
#ifndef PF_LB
#define PF_LB 0  // 0: PfCfg::kThreads (tools: a larger bound lowers the register cap)
#endif
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PF_LB > 0 ? PF_LB : PfCfg::kThreads, 1)
    w4ax_gemm_pf_kernel(const __grid_constant__ CUtensorMap tmXe, const __grid_constant__ CUtensorMap tmX8,
                        const __grid_constant__ CUtensorMap tmY, const __grid_constant__ BlockMap map, GemmArgs args,
                        PfSched sched, const __grid_constant__ YPeerMaps ypeers) {
  using C = PfCfg;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t scale_base = sbase + C::kScaleBase;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarBase);
  uint64_t* lfull = bars;                     // [kLStages] packed weights + tokens + scales landed (tx)
  uint64_t* lempty = lfull + C::kLStages;     // [kLStages] the staging warps have read the packed weights
  uint64_t* mdone = lempty + C::kLStages;     // [kStages] MMAs of the block done (commit multicast)
  uint64_t* ready = mdone + C::kStages;       // [kStages] leader: operands of the block staged in both CTAs
  uint64_t* tfull = ready + C::kStages;       // [kAccs] accumulator complete (commit multicast)
  uint64_t* tempty = tfull + C::kAccs;        // [kAccs] leader: 2 CTAs x 16 promotion warps released it
  uint64_t* sempty = tempty + C::kAccs;       // [kScaleSlots] 16 promotion warps done with the slot
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sempty + C::kScaleSlots);
  float* fac = reinterpret_cast<float*>(smem + C::kFacBase);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // warp-uniform for ptxas
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const int cluster = blockIdx.x >> 1;
  const int nb = args.nb;
  const int my_tiles = cluster < sched.tiles ? (sched.tiles - 1 - cluster) / sched.clusters + 1 : 0;
  const int steps = my_tiles * nb;  // (tile, block) steps of this cluster

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&mdone[s], 1);
      mbar_init(&ready[s], C::kReadyCount);
    }
    for (int l = 0; l < C::kLStages; ++l) {
      mbar_init(&lfull[l], 2);  // two producers
      mbar_init(&lempty[l], C::kSWarps);
    }
    for (int a = 0; a < C::kAccs; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], C::kTemptyCount);
    }
    for (int a = 0; a < C::kScaleSlots; ++a) mbar_init(&sempty[a], C::kPWarps);
    fence_mbar_init();
  }
  // per-block factor from accumulator units to logical units: 2^18 (INT4,
  // the two 2^-9 e4m3 scalings) or 1/16 (INT8, the x16 weights)
  for (int i = threadIdx.x; i < nb; i += C::kThreads) fac[i] = (map.code[i] >> 15) ? 0.0625f : 262144.0f;
  if (warp == C::kLoadWarp && lane == 0) {
    tma_prefetch_desc(&tmXe);
    tma_prefetch_desc(&tmX8);
    tma_prefetch_desc(&tmY);
  }
  if (warp == C::kMmaWarp) tmem_alloc_2sm<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();  // orders the allocation's smem write before the reads below for racecheck (cluster_sync does in hardware)
  cluster_sync();
  tc_fence_after();
  // PDL: the next kernel in the stream (e.g. the next layer's quantizer) may
  // be scheduled; its CTAs take SMs as this grid's CTAs exit and wait for
  // this grid's completion before touching memory (griddepcontrol.wait)
  grid_dep_launch();
  const uint32_t tmem_base = *tmem_holder;
  // debug trace of one CTA (-DCOMET_TRACE builds only; tools/gemm_sweep.py trace_pf)
  const bool tr = kTraceBuild && g_cta_times_on && blockIdx.x + 1 == g_cta_times_on;

  if (warp == C::kLoadWarp) {
    // ----------------------------------- a3: token + scale producer ----
    int pt = cluster, pb = 0, pm0 = 0, pn0 = 0;
    sched.coords(pt, pm0, pn0);
    grid_dep_wait();  // the planes and corrections come from the preceding kernels (PDL)
    for (int g = 0; g < steps; ++g) {
      const int b = pb;
      const int l = g % C::kLStages, s = g % C::kStages, a = g & (C::kScaleSlots - 1);
      const uint32_t code = map.code[b];
      const bool is8 = (code >> 15) != 0;
      const int rank = code & 0x7FFF;
      // lfull[l] takes one arrive per block from here and one from the weight
      // refill: wait until the staging warps released block g - kLStages;
      // operand stage s (its A half) is free once the MMAs of block g - kStages
      // are done; scale slot a once the promotion of block g - 8 is
      mbar_wait(&lempty[l], ((g / C::kLStages) & 1) ^ 1);
      mbar_wait(&mdone[s], ((g / C::kStages) & 1) ^ 1);
      mbar_wait(&sempty[a], ((g / C::kScaleSlots) & 1) ^ 1);
      if (elect_one()) {
        trace(tr, 13, g);
        const int my_m0 = pm0 + 128 * (int)crank;
        const int nsx = max(0, min(128, (int)args.ldsx - my_m0));  // multiple of 4
        const bool load_sx = !kAccOut, load_cx = !is8;
        const bool load_sw = !kAccOut && (!kGroupK || b == nb - 1);
        const int nsw = load_sw ? max(0, min(C::kTileN, args.N - pn0)) : 0;  // multiple of 64
        mbar_arrive_expect_tx(&lfull[l], C::kABytes + ((load_sx ? nsx : 0) + (load_cx ? nsx : 0) + nsw) * 4);
        tma_load_2d(smem + C::kABase + s * C::kABytes, is8 ? &tmX8 : &tmXe, &lfull[l], rank * 128, my_m0);
        uint8_t* slot = smem + C::kScaleBase + a * C::kSlotBytes;
        if (load_sx && nsx) bulk_load(slot, args.Sx + (int64_t)b * args.ldsx + my_m0, nsx * 4, &lfull[l]);
        if (load_cx && nsx) bulk_load(slot + C::kCxOff, args.CX + (int64_t)rank * args.ldsx + my_m0, nsx * 4, &lfull[l]);
        if (nsw) bulk_load(slot + C::kSwOff, args.Sw + (kGroupK ? 0 : (int64_t)b * args.N) + pn0, nsw * 4, &lfull[l]);
      }
      __syncwarp();
      if (++pb == nb) {
        pb = 0;
        pt += sched.clusters;
        if (pt < sched.tiles) sched.coords(pt, pm0, pn0);
      }
    }
  } else if (warp == C::kMmaWarp) {
    // -------------------------------------------------- a5: MMA (leader) ----
    constexpr uint32_t idesc8 = idesc_i8(256, C::kTileN), idesc4 = idesc_e4m3(256, C::kTileN);
    int b = 0;
    for (int g = 0; g < steps && crank == 0; ++g) {
      const int s = g % C::kStages, acc = g % C::kAccs;
      const bool is8 = (map.code[b] >> 15) != 0;
      if (++b == nb) b = 0;
      if (lane == 0) trace(tr, 4, g);
      mbar_wait(&ready[s], (g / C::kStages) & 1);
      if (lane == 0) trace(tr, 5, g);
      mbar_wait(&tempty[acc], ((g / C::kAccs) & 1) ^ 1);
      if (lane == 0) trace(tr, 6, g);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t d = tmem_base + acc * C::kTileN;
        const uint32_t ast = sbase + C::kABase + s * C::kABytes, bst = sbase + C::kBBase + s * C::kBBytes;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = umma_desc_sw128_kmajor(ast + 32 * k), bd = umma_desc_sw128_kmajor(bst + 32 * k);
          if (is8)
            mma_ss_2sm<false>(d, ad, bd, idesc8, k > 0 ? 1u : 0u);
          else
            mma_ss_2sm<true>(d, ad, bd, idesc4, k > 0 ? 1u : 0u);
          if (k == 0) trace(tr, 17, g);
        }
        trace(tr, 18, g);
        mma_commit_2sm(&tfull[acc], 0x3);
        trace(tr, 19, g);
        mma_commit_2sm(&mdone[s], 0x3);
        trace(tr, 7, g);
      }
      __syncwarp();
    }
  } else if (warp == C::kWLoadWarp) {
    // ------------------------------------------- a3: weight producer ----
    int pt = cluster, pb = 0, pm0 = 0, pn0 = 0;
    sched.coords(pt, pm0, pn0);
    grid_dep_wait();  // the weights may come from a preceding kernel (PDL)
    for (int g = 0; g < steps; ++g) {
      const int l = g % C::kLStages;
      mbar_wait(&lempty[l], ((g / C::kLStages) & 1) ^ 1);  // the staging warps released block g - kLStages
      if (elect_one()) {
        trace(tr, 12, g);
        // this CTA's weight rows [R, R + v) of the tile (v < kRows at the right
        // edge of N); contiguous within each 128-row slab of the tiled layout
        const int R = pn0 + C::kRows * (int)crank;
        const int v = max(0, min(C::kRows, args.N - R));
        mbar_arrive_expect_tx(&lfull[l], v * 64);
        uint8_t* dst = smem + C::kWPBase + l * C::kWPBytes;
        int r = R, left = v;
        while (left > 0) {
          const int in_slab = min(left, 128 - (r & 127));
          bulk_load(dst, args.Wq + ((int64_t)(r >> 7) * nb + pb) * 8192 + (r & 127) * 64, in_slab * 64, &lfull[l]);
          dst += in_slab * 64;
          r += in_slab;
          left -= in_slab;
        }
      }
      __syncwarp();
      if (++pb == nb) {
        pb = 0;
        pt += sched.clusters;
        if (pt < sched.tiles) sched.coords(pt, pm0, pn0);
      }
    }
  } else if (warp >= C::kStageWarp && warp < C::kStageWarp + C::kSWarps) {
    // ------------- a4 staging: packed weight chunks -> SW128 B operand ----
    const int et = (int)threadIdx.x - 32 * C::kStageWarp;  // 0 .. 32 kSWarps - 1
    const uint32_t leader_ready = mapa_shared(smem_u32(ready), 0);
    constexpr int kChunks = C::kRows * 4 / (32 * C::kSWarps);  // 16-byte packed chunks per thread
    static_assert(kChunks * 32 * C::kSWarps == C::kRows * 4, "staging split");
    int b = 0;
    for (int j = 0; j < steps; ++j) {
      const int l = j % C::kLStages, s = j % C::kStages;
      const bool is8 = (map.code[b] >> 15) != 0;
      if (++b == nb) b = 0;
      const uint32_t wps = sbase + C::kWPBase + l * C::kWPBytes;
      const uint32_t wst = sbase + C::kBBase + s * C::kBBytes;
      const bool tr_s = tr && threadIdx.x == 32 * C::kStageWarp;
      trace(tr_s, 8, j);
      mbar_wait(&lfull[l], (j / C::kLStages) & 1);
      trace(tr_s, 9, j);
      mbar_wait(&mdone[s], ((j / C::kStages) & 1) ^ 1);  // B stage s free
      trace(tr_s, 10, j);
      uint4 wv[kChunks];
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int ch = et + 32 * C::kSWarps * k;
        const int er = ch >> 2, ej = ch & 3;
        wv[k] = lds128(wps + er * 64 + ((ej ^ ((er >> 1) & 3)) << 4));
      }
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int ch = et + 32 * C::kSWarps * k;
        const int er = ch >> 2, ej = ch & 3;
        uint4 o0, o1;
        if (is8) {
          zext_word(wv[k].x, o0.x, o0.y);
          zext_word(wv[k].y, o0.z, o0.w);
          zext_word(wv[k].z, o1.x, o1.y);
          zext_word(wv[k].w, o1.z, o1.w);
        } else {
          e4m3_offset_word(wv[k].x, o0.x, o0.y);
          e4m3_offset_word(wv[k].y, o0.z, o0.w);
          e4m3_offset_word(wv[k].z, o1.x, o1.y);
          e4m3_offset_word(wv[k].w, o1.z, o1.w);
        }
        sts128(wst + er * 128 + (((2 * ej) ^ (er & 7)) << 4), o0);
        sts128(wst + er * 128 + (((2 * ej + 1) ^ (er & 7)) << 4), o1);
      }
      trace(tr_s, 21, j);
      // the packed stage may be refilled once every lane's loads have landed
      __syncwarp();
      if (lane == 0) mbar_arrive(&lempty[l]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_ready + s * 8);
      trace(tr_s, 11, j);

    }
  } else if (warp >= C::kPBase && warp < C::kPBase + C::kPWarps) {
    // ------------------------- warps 0-11: a6 promotion + a8 write-back ----
    const int q = warp & 3;                  // TMEM lane quarter
    const int kw = (warp - C::kPBase) >> 2;  // columns [64 kw, 64 kw + 64) of the tile
    const int row = 32 * q + lane;           // token row within this CTA
    const uint32_t tl = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(C::kWCols * kw);
    const uint32_t leader_tempty = mapa_shared(smem_u32(tempty), 0);
    constexpr int kWC = C::kWCols;
    // per-channel weights: z = sum_b sx_b * fac_b * D_b, zc = sum_b sx_b * 8 sum(xq)_b,
    // y = sw * (z - zc) at the tile end; group 128: y accumulated directly
    uint64_t y[kWC / 2];
#pragma unroll
    for (int j = 0; j < kWC / 2; ++j) y[j] = 0;
    float zc = 0.f;
    int t = cluster, b = 0;
    for (int g = 0; g < steps; ++g) {
      const int a = g & (C::kScaleSlots - 1);
      const int acc = g % C::kAccs;
      const uint32_t slot = scale_base + a * C::kSlotBytes;
      const uint32_t code = map.code[b];
      const bool is8 = (code >> 15) != 0;
      const bool tr_p = tr && lane == 0 && (warp == C::kPBase || warp == C::kPBase + C::kPWarps - 1);
      const int ev0 = warp == C::kPBase ? 0 : 14;
      trace(tr_p && ev0 == 0, 0, g);
      mbar_wait(&tfull[acc], (g / C::kAccs) & 1);
      trace(tr_p, ev0 + 1, g);
      // steps 16..19: every promotion warp's "accumulator seen" / "released" clocks
      trace_at(tr && lane == 0 && g >= 16 && g < 20, 25 + (g - 16), 2 * (warp - C::kPBase));
      tc_fence_after();
      const uint32_t ta = tl + acc * C::kTileN;
      float sxv = 0.f, cxv = 0.f;
      if (!kAccOut) sxv = lds_f32(slot + row * 4) * lds_f32(sbase + C::kFacBase + 4 * b);  // x fac
      if (!is8) cxv = lds_f32(slot + C::kCxOff + row * 4);
      const uint64_t sx2 = pack2(sxv, sxv);
      const float ncx = -sxv * 3.814697265625e-06f * cxv;  // -sx * 8 sum(xq) (sxv carries the 2^18)
      const uint64_t nc2 = pack2(ncx, ncx);
      if (kGroupK) zc -= ncx;
      // one 8-column chunk of the accumulator into the running sums
      auto promote8 = [&](int c, const uint32_t (&r)[8]) {
        uint64_t* yy = &y[4 * c];
        if (kAccOut) {
          int m0, n0;
          sched.coords(t, m0, n0);
          const int m = m0 + 128 * (int)crank + row;
          const int nu = n0 + kWC * kw + 8 * c;
          if (m < args.M) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
              if (nu + jj < args.N)
                args.Acc[((int64_t)b * args.M + m) * args.N + nu + jj] =
                    is8 ? ((int32_t)r[jj] >> 4) : __float2int_rn(__uint_as_float(r[jj]) * 262144.0f) - (int)cxv;
          }
        } else if (kGroupK) {
          if (is8) {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) cvt_fma2(yy[jj], r[2 * jj], r[2 * jj + 1], sx2);
          } else {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) fma2_u(yy[jj], r[2 * jj], r[2 * jj + 1], sx2);
          }
        } else {
          const uint32_t swa = slot + C::kSwOff + (kWC * kw + 8 * c) * 4;
#pragma unroll
          for (int j4 = 0; j4 < 2; ++j4) {
            const float4 w4 = lds_f32x4(swa + 16 * j4);
            const uint64_t w01 = pack2(w4.x, w4.y), w23 = pack2(w4.z, w4.w);
            if (is8) {
              cvt_fma2(yy[2 * j4], r[4 * j4], r[4 * j4 + 1], mul2_u(sx2, w01));
              cvt_fma2(yy[2 * j4 + 1], r[4 * j4 + 2], r[4 * j4 + 3], mul2_u(sx2, w23));
            } else {
              // (D * sx * 2^18 - sx * 8 sum(xq)) * sw = sx * acc * sw
              fma2_corr_u(yy[2 * j4], r[4 * j4], r[4 * j4 + 1], sx2, nc2, w01);
              fma2_corr_u(yy[2 * j4 + 1], r[4 * j4 + 2], r[4 * j4 + 3], sx2, nc2, w23);
            }
          }
        }
      };
      // 8-column chunks, double-buffered: chunk c + 1 is loading while chunk c
      // is promoted; the accumulator is released after its last load
      constexpr int kC8 = kWC / 8;
      uint32_t ra[8], rb[8];
      tmem_ld_32x32b_x8(ta, ra);
      tmem_ld_wait_dep(ra);
#pragma unroll
      for (int c = 0; c < kC8; c += 2) {
        tmem_ld_32x32b_x8(ta + 8 * (c + 1), rb);
        promote8(c, ra);
        tmem_ld_wait_dep(rb);
        if (c + 2 < kC8) {
          tmem_ld_32x32b_x8(ta + 8 * (c + 2), ra);
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(leader_tempty + acc * 8);
          trace(tr_p, ev0 + 2, g);
          trace_at(tr && lane == 0 && g >= 16 && g < 20, 25 + (g - 16), 2 * (warp - C::kPBase) + 1);
        }
        promote8(c + 1, rb);
        if (c + 2 < kC8) tmem_ld_wait_dep(ra);
      }

      if (++b == nb) {
        // -------------------- a8: tile write-back (fp16 RNE, TMA stores) -------
        // y = sw * (z - zc) (per-channel) -> fp16 RNE -> the warp's 2 KB box
        // in shared memory (row = lane, SW64 chunks: conflict-free) -> one
        // TMA store per 32 columns.  (Direct 16-byte stores from the
        // row-per-lane layout touch 32 rows per instruction; their burst at
        // every tile end stalled the staging warps' smem stores and the
        // promotion for ~3 us per tile.)
        if (!kAccOut) {
          int m0, n0;
          sched.coords(t, m0, n0);
          const uint64_t nzc2 = pack2(-zc, -zc);
          const uint32_t swa = slot + C::kSwOff + (kWC * kw) * 4;
          const uint32_t ybuf = sbase + C::kYBase + (warp - C::kPBase) * C::kYWarpBytes;
#pragma unroll
          for (int h = 0; h < kWC / 32; ++h) {
            const uint32_t ybox = ybuf + (h % C::kYBoxes) * 2048;
            if (h % C::kYBoxes == 0) {  // the previous boxes have left the buffer
              if (lane == 0) bulk_wait_group_read0();
              __syncwarp();
            }
#pragma unroll
            for (int v4 = 0; v4 < 4; ++v4) {  // 8 columns: one 16-byte chunk of the row
              const int v = 4 * h + v4;
              uint32_t hw[4];
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int p4 = 2 * v + hh;
                uint64_t v0 = y[2 * p4], v1 = y[2 * p4 + 1];
                if (kGroupK) {  // per-channel weight scales, once per tile
                  const float4 w4 = lds_f32x4(swa + 16 * p4);
                  v0 = mul2_u(add2_u(v0, nzc2), pack2(w4.x, w4.y));
                  v1 = mul2_u(add2_u(v1, nzc2), pack2(w4.z, w4.w));
                }
                __half2 h0 = __float22half2_rn(unpack2(v0));
                __half2 h1 = __float22half2_rn(unpack2(v1));
                hw[2 * hh] = *reinterpret_cast<uint32_t*>(&h0);
                hw[2 * hh + 1] = *reinterpret_cast<uint32_t*>(&h1);
                y[2 * p4] = 0;
                y[2 * p4 + 1] = 0;
              }
              sts128(ybox + lane * 64 + ((v4 ^ ((lane >> 1) & 3)) << 4), make_uint4(hw[0], hw[1], hw[2], hw[3]));
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              const int yx = 2 * (n0 + kWC * kw + 32 * h), yy = m0 + 128 * (int)crank + 32 * q;
              tma_store_2d(&tmY, ybox, yx, yy);
              // f1: the same box into every peer's copy of the output (NVLink
              // P2P stores from the TMA engine; "all-gather fused into
              // the epilogue", one sync before the write-back is consumed)
              for (int i = 0; i < ypeers.n; ++i) tma_store_2d(&ypeers.m[i], ybox, yx, yy);
              bulk_commit_group();
            }
          }
          zc = 0.f;
        }
        b = 0;
        t += sched.clusters;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[a]);
      trace(tr_p && ev0 == 0, 3, g);
    }
  }

  if (warp >= C::kPBase && warp < C::kPBase + C::kPWarps && lane == 0) bulk_wait_group0();  // Y stores complete before the CTA exits
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc_2sm<512>(tmem_base);
}

}  // namespace comet
