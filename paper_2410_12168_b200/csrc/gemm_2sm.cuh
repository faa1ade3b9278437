// gemm_2sm.cuh -- prefill W4Ax GEMM on CTA pairs (tcgen05 cta_group::2),
// persistent over pair tiles.
//
// Pair tile: 256 tokens (MMA M; 128 TMEM lanes in each CTA) x 256 weight
// rows (MMA N; each CTA stages 128 of them); K is walked one 128-channel
// FMPQ block at a time.  One cluster of 2 CTAs stays
// resident per SM pair and walks the tiles t = cluster, cluster + C, ...
// (static round-robin: every tile costs the same, "distribute ... as
// evenly as possible across all SMs"); the per-block pipelines run
// continuously across tile boundaries, so there is no pipeline drain or
// re-fill between tiles and one sync per tile before write-back.
//
// Per block and CTA:
//   a3  warp 16: 1-D bulk copy of the packed weight slab [128 x 64 B] (tiled
//       weight layout) and TMA of the token slab
//       (INT8 blocks [128 x 128 B] straight into the MMA operand with
//       128B swizzle, INT4 blocks packed [128 x 64 B]); 1-D bulk copies of
//       the block's scales into an 8-deep scale ring.
//   a4  warps 0-15 ("compute warps"): INT4 -> INT8 zero-extension
//       of the weights (and INT4 token blocks) of the NEXT block into SW128
//       K-major smem -- one 16-byte packed chunk per thread per operand --
//       then an arrive on the leader CTA's "expanded" barrier;
//   a5  warp 17 of the leader CTA: 4 x tcgen05.mma.cta_group::2.kind::i8
//       (M=256, N=256, K=32) into a fresh INT32 accumulator in both CTAs'
//       TMEM (two 256-column accumulators ping-pong = all 512 columns);
//       tcgen05.commit multicasts to both CTAs' barriers;
//   a6  compute warps: tcgen05.ld 16 columns at a time, I2F, and
//       y += (sx[m,b] 16^-e_b) * acc  with fma.rn.f32x2 (a thread owns a
//       token row, so sx is thread-uniform); group-128 weights also multiply
//       by sw[n,b] (mul.rn.f32x2); per-channel weights apply sw[n] once per
//       tile;
//   a8  after the tile's last block: fp32 -> fp16 RNE, 16-byte stores.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "gemm.cuh"
#include "quantize.cuh"
#include "sm100.cuh"

namespace comet {

struct Gemm2Cfg {
  // 3 stages: operands are resident well before use (L2 hits, one step of
  // ~1800 cycles ahead), and the freed 48 KB hold the output staging below
#ifndef COMET_PF_STAGES
#define COMET_PF_STAGES 3
#endif
  static constexpr int kStages = COMET_PF_STAGES;
  static constexpr int kScaleSlots = 8;
  static constexpr int kABytes = 128 * 128;   // tokens int8, SW128 K-major
  static constexpr int kBBytes = 128 * 128;   // weights int8 (this CTA's half of N)
  static constexpr int kXPBytes = 128 * 64;   // packed INT4 tokens
  static constexpr int kWPBytes = 128 * 64;   // packed INT4 weights
  static constexpr int kStageBytes = kABytes + kBBytes + kXPBytes + kWPBytes;  // 48 KiB
  static constexpr int kSlotBytes = 128 * 4 + 256 * 4;                        // sx[128] + sw[256]
  static constexpr int kScaleBytes = kScaleSlots * kSlotBytes;
  // a8: each compute warp stages its 32 x 64 fp16 output block (128B-swizzled)
  // for one TMA tensor store
  static constexpr int kYWarpBytes = 32 * 64 * 2;
  static constexpr int kYBase = kStages * kStageBytes + kScaleBytes;  // 1024-aligned
#ifndef COMET_PF_TMA_STORE
#define COMET_PF_TMA_STORE 1
#endif
  static constexpr bool kTmaStore = COMET_PF_TMA_STORE;
  static constexpr int kBarBase = kYBase + (kTmaStore ? 16 * kYWarpBytes : 0);
  static constexpr int kBarBytes = 256;
  static constexpr int kSmemBytes = kBarBase + kBarBytes + 1024;
  static_assert(kYBase % 1024 == 0 && kSmemBytes <= 227 * 1024, "smem budget");
  static constexpr int kThreads = 576;  // warps 0-15 compute, 16 TMA producer, 17 MMA issuer
  static constexpr int kLoadWarp = 16;
  static constexpr int kMmaWarp = 17;
  static constexpr int kNumEpiWarps = 16;
};

struct PairSched {
  int m_tiles, n_tiles, tiles, clusters;
  DEVI void coords(int t, int& m0, int& n0) const {
    const int mt = t % m_tiles;  // token tiles fastest: concurrent clusters share weight tiles
    m0 = mt * 256;
    n0 = (t / m_tiles) * 256;
  }
};

// Zero-extension of one packed word w: t = w & 0x0F0F0F0F (LOP3,
// ALU pipe), lo = 16*t = 16*e0..3 and hi = w - t = 16*e4..7 as IMADs (FMA
// pipe) -- the ALU pipe is shared with I2F in the promotion.
DEVI void zext_word(uint32_t w, uint32_t& lo, uint32_t& hi) {
  uint32_t t;
  asm("and.b32 %0, %1, 0x0F0F0F0F;" : "=r"(t) : "r"(w));
  asm("mul.lo.u32 %0, %1, 16;" : "=r"(lo) : "r"(t));
  asm("mad.lo.u32 %0, %1, 0xFFFFFFFF, %2;" : "=r"(hi) : "r"(t), "r"(w));
}
DEVI void expand_chunk(uint4 w, uint32_t dst0, uint32_t dst1) {
  uint4 o0, o1;
  zext_word(w.x, o0.x, o0.y);
  zext_word(w.y, o0.z, o0.w);
  zext_word(w.z, o1.x, o1.y);
  zext_word(w.w, o1.z, o1.w);
  sts128(dst0, o0);  // 16*e0..3 | 16*e4..7 of words 0,1
  sts128(dst1, o1);
}

template <bool kGroupK, bool kAccOut>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(576, 1)
    w4ax_gemm_2sm_kernel(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmX4,
                         const __grid_constant__ CUtensorMap tmX8, const __grid_constant__ BlockMap map, GemmArgs args,
                         PairSched sched) {
  using C = Gemm2Cfg;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t scale_base = sbase + C::kStages * C::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarBase);
  uint64_t* full = bars;                       // [kStages] local TMA tx
  uint64_t* expd = full + C::kStages;          // [kStages] leader: 2 CTAs x 16 compute warps
  uint64_t* empty = expd + C::kStages;         // [kStages] MMA commit (multicast)
  uint64_t* tfull = empty + C::kStages;        // [2] MMA commit (multicast)
  uint64_t* tempty = tfull + 2;                // [2] leader: 2 CTAs x 16 compute warps
  uint64_t* sfull = tempty + 2;                // [kScaleSlots] local bulk tx
  uint64_t* sempty = sfull + C::kScaleSlots;   // [kScaleSlots] local compute warps
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sempty + C::kScaleSlots);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const int cluster = blockIdx.x >> 1;
  const int nb = args.nb;
  // number of (tile, block) steps this cluster runs
  const int my_tiles = cluster < sched.tiles ? (sched.tiles - 1 - cluster) / sched.clusters + 1 : 0;
  const int steps = my_tiles * nb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&expd[s], 2 * C::kNumEpiWarps);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * C::kNumEpiWarps);
    }
    for (int a = 0; a < C::kScaleSlots; ++a) {
      mbar_init(&sfull[a], 1);
      mbar_init(&sempty[a], C::kNumEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == C::kLoadWarp && lane == 0) {
    if (!kAccOut) tma_prefetch_desc(&tmY);
    tma_prefetch_desc(&tmX4);
    tma_prefetch_desc(&tmX8);
  }
  if (warp == C::kMmaWarp) tmem_alloc_2sm<512>(tmem_holder);
  tc_fence_before();
  cluster_sync();  // barrier inits + TMEM allocation visible cluster-wide
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // debug trace of one CTA (comet_debug_cta_times(cta + 1)); see tools/gemm_sweep.py trace2
  const bool tr_cta = g_cta_times_on && blockIdx.x + 1 == g_cta_times_on;

  if (warp == C::kLoadWarp) {
    // ------------------------------------------------- a3: producer ----
    grid_dep_wait();  // PDL: operands come from the preceding kernels
    int t = cluster, b = 0;
    int m0 = 0, n0 = 0;
    sched.coords(t, m0, n0);
    for (int g = 0; g < steps; ++g) {
      const int s = g % C::kStages;
      const uint32_t code = map.code[b];
      const bool is8 = (code >> 15) != 0;
      const int rank = code & 0x7FFF;
      const int my_m0 = m0 + 128 * (int)crank;
      mbar_wait(&empty[s], ((g / C::kStages) & 1) ^ 1);
      trace(tr_cta && lane == 0, 7, g);
      uint8_t* st = smem + s * C::kStageBytes;
      if (elect_one()) {
        // a half-populated pair tile (N % 256 == 128): the second CTA's weight
        // rows are past N -- no load; its (unused) output columns are never stored
        const bool w_valid = n0 + 128 * (int)crank < args.N;
        mbar_arrive_expect_tx(&full[s], (w_valid ? C::kWPBytes : 0) + (is8 ? C::kABytes : C::kXPBytes));
        if (w_valid)
          bulk_load(st + C::kABytes + C::kBBytes + C::kXPBytes,
                    args.Wq + ((int64_t)((n0 >> 7) + (int)crank) * nb + b) * 8192, 8192, &full[s]);
        if (is8)
          tma_load_2d(st, &tmX8, &full[s], rank * 128, my_m0);
        else
          tma_load_2d(st + C::kABytes + C::kBBytes, &tmX4, &full[s], rank * 64, my_m0);
      }
      if (!kAccOut) {
        const int a = g & (C::kScaleSlots - 1);
        mbar_wait(&sempty[a], ((g / C::kScaleSlots) & 1) ^ 1);
        if (elect_one()) {
          const int nsx = max(0, min(128, (int)args.ldsx - my_m0));  // multiple of 4
          const bool load_sw = !kGroupK || b == nb - 1;
          const int nsw = load_sw ? max(0, min(256, args.N - n0)) : 0;
          mbar_arrive_expect_tx(&sfull[a], (nsx + nsw) * 4);
          uint8_t* slot = smem + C::kStages * C::kStageBytes + a * C::kSlotBytes;
          if (nsx) bulk_load(slot, args.Sx + (int64_t)b * args.ldsx + my_m0, nsx * 4, &sfull[a]);
          // group 128: g(b) = b; per-channel: Sw is [1 x N]
          if (nsw) bulk_load(slot + 512, args.Sw + (kGroupK ? 0 : (int64_t)b * args.N) + n0, nsw * 4, &sfull[a]);
        }
      }
      __syncwarp();
      if (++b == nb) {
        b = 0;
        t += sched.clusters;
        if (t < sched.tiles) sched.coords(t, m0, n0);
      }
    }
  } else if (warp == C::kMmaWarp) {
    // --------------------------------------------- a5: MMA (leader) ----
    if (crank == 0) {
      constexpr uint32_t idesc = idesc_i8(256, 256);
      for (int g = 0; g < steps; ++g) {
        const int s = g % C::kStages;
        const int acc = g & 1;
        mbar_wait_cluster(&tempty[acc], ((g >> 1) & 1) ^ 1);
        mbar_wait_cluster(&expd[s], (g / C::kStages) & 1);
        trace(tr_cta && lane == 0, 6, g);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a0 = sbase + s * C::kStageBytes;
          const uint32_t b0 = a0 + C::kABytes;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_i8_ss_2sm(tmem_base + acc * 256, umma_desc_sw128_kmajor(a0 + 32 * k),
                          umma_desc_sw128_kmajor(b0 + 32 * k), idesc, k > 0 ? 1u : 0u);
          mma_commit_2sm(&empty[s], 0x3);
          mma_commit_2sm(&tfull[acc], 0x3);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------ compute warps 0-15: a4 + a6 + a8 ----
    const int ct = threadIdx.x;                   // 0..511
    const int q = warp & 3;                       // TMEM lane quarter
    const int cg = warp >> 2;                     // 64-column group
    const int row = 32 * q + lane;                // token row within this CTA
    const uint32_t tl = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(64 * cg);
    const uint32_t leader_expd = mapa_shared(smem_u32(expd), 0);
    const uint32_t leader_tempty = mapa_shared(smem_u32(tempty), 0);

    const bool tr_on = tr_cta && threadIdx.x == 0;
    // a4: expansion of global step j (block ex_b of its tile); this thread
    // handles packed row ct/4, 16-byte chunk ct%4 of both operands
    int ex_b = 0;
    auto expand = [&](int j) {
      const int s = j % C::kStages;
      const bool is8 = (map.code[ex_b] >> 15) != 0;
      if (++ex_b == nb) ex_b = 0;
      const uint32_t st = sbase + s * C::kStageBytes;
      const int er = ct >> 2, ej = ct & 3;
      const uint32_t e_src = er * 64 + ej * 16;
      const uint32_t w_src = er * 64 + ((ej ^ ((er >> 1) & 3)) << 4);  // tiled weights: 64B swizzle
      const uint32_t e_dst0 = er * 128 + (((2 * ej) ^ (er & 7)) << 4);
      const uint32_t e_dst1 = er * 128 + (((2 * ej + 1) ^ (er & 7)) << 4);
      mbar_wait(&full[s], (j / C::kStages) & 1);
      trace(tr_on, 1, j);
      const uint4 w = lds128(st + C::kABytes + C::kBBytes + C::kXPBytes + w_src);
      if (!is8) {
        const uint4 x = lds128(st + C::kABytes + C::kBBytes + e_src);
        expand_chunk(x, st + e_dst0, st + e_dst1);
      }
      expand_chunk(w, st + C::kABytes + e_dst0, st + C::kABytes + e_dst1);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_expd + s * 8);
      trace(tr_on, 2, j);
    };

    uint64_t y[32];  // fp32 pairs (columns 2j, 2j+1 of this warp's 64)
#pragma unroll
    for (int j = 0; j < 32; ++j) y[j] = 0;
    int t = cluster, b = 0;
    if (steps > 0) expand(0);
    for (int g = 0; g < steps; ++g) {
      trace(tr_on, 0, g);
      if (g + 1 < steps) expand(g + 1);
      // ---- a6: promote block b of tile t -----------------------------------
      const int acc = g & 1;
      const int a = g & (C::kScaleSlots - 1);
      const uint32_t slot = scale_base + a * C::kSlotBytes;
      const bool is8 = (map.code[b] >> 15) != 0;
      float sxv = 0.f;
      if (!kAccOut) {
        mbar_wait(&sfull[a], (g / C::kScaleSlots) & 1);
        sxv = lds_f32(slot + row * 4) * (is8 ? 0.0625f : 0.00390625f);  // fold 16^-e
      }
      trace(tr_on, 3, g);
      const uint64_t sx2 = pack2(sxv, sxv);
      mbar_wait(&tfull[acc], (g >> 1) & 1);
      trace(tr_on, 4, g);
      tc_fence_after();
      if (kAccOut) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(tl + acc * 256 + 16 * c, r);
          tmem_ld_wait();
          int m0, n0;
          sched.coords(t, m0, n0);
          const int sh = is8 ? 4 : 8;
          const int m = m0 + 128 * (int)crank + row;
          if (m < args.M) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int n = n0 + 64 * cg + 16 * c + j;
              if (n < args.N) args.Acc[((int64_t)b * args.M + m) * args.N + n] = ((int32_t)r[j]) >> sh;
            }
          }
        }
      } else {
        // columns [8c, 8c + 8) of this warp's 64; the load of chunk c + 1 is
        // in flight while chunk c is promoted
        auto promote = [&](int c, const uint32_t (&r)[8]) {
          if (kGroupK) {
#pragma unroll
            for (int j = 0; j < 4; ++j) cvt_fma2(y[4 * c + j], r[2 * j], r[2 * j + 1], sx2);
          } else {
            const uint32_t swa = slot + 512 + (64 * cg + 8 * c) * 4;
#pragma unroll
            for (int j4 = 0; j4 < 2; ++j4) {
              const float4 w4 = lds_f32x4(swa + 16 * j4);
              cvt_fma2(y[4 * c + 2 * j4], r[4 * j4], r[4 * j4 + 1], mul2_u(sx2, pack2(w4.x, w4.y)));
              cvt_fma2(y[4 * c + 2 * j4 + 1], r[4 * j4 + 2], r[4 * j4 + 3], mul2_u(sx2, pack2(w4.z, w4.w)));
            }
          }
        };
        uint32_t ra[8], rb[8];
        tmem_ld_32x32b_x8(tl + acc * 256, ra);
        tmem_ld_wait_dep(ra);
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
          tmem_ld_32x32b_x8(tl + acc * 256 + 8 * (c + 1), rb);
          promote(c, ra);
          tmem_ld_wait_dep(rb);
          if (c + 2 < 8) tmem_ld_32x32b_x8(tl + acc * 256 + 8 * (c + 2), ra);
          promote(c + 1, rb);
          if (c + 2 < 8) tmem_ld_wait_dep(ra);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty + acc * 8);
      trace(tr_on, 5, g);

      if (++b == nb) {
        // -------------------------------------------- a8: tile write-back ----
        if (!kAccOut) {
          int m0, n0;
          sched.coords(t, m0, n0);
          const int m = m0 + 128 * (int)crank + row;
          const int nbase = n0 + 64 * cg;
          if (kGroupK) {
            const uint32_t swa = slot + 512 + 64 * cg * 4;
#pragma unroll
            for (int j4 = 0; j4 < 16; ++j4) {
              const float4 w4 = lds_f32x4(swa + 16 * j4);
              y[2 * j4] = mul2_u(y[2 * j4], pack2(w4.x, w4.y));
              y[2 * j4 + 1] = mul2_u(y[2 * j4 + 1], pack2(w4.z, w4.w));
            }
          }
          if (!C::kTmaStore) {
            if (m < args.M && nbase < args.N) {
              __half* yrow = args.Y + (int64_t)m * args.ldy + nbase;
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                __half2 h0 = __float22half2_rn(unpack2(y[4 * v + 0]));
                __half2 h1 = __float22half2_rn(unpack2(y[4 * v + 1]));
                __half2 h2 = __float22half2_rn(unpack2(y[4 * v + 2]));
                __half2 h3 = __float22half2_rn(unpack2(y[4 * v + 3]));
                *reinterpret_cast<uint4*>(yrow + 8 * v) =
                    make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                               *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
              }
            }
          } else {
          // stage this warp's 32 rows x 64 columns (row = lane, 128 B, chunks
          // 128B-swizzled: conflict-free) and hand it to one TMA store, which
          // clips rows >= M and columns >= N
          const uint32_t ybuf = sbase + C::kYBase + warp * C::kYWarpBytes;
          if (lane == 0) bulk_wait_group_read0();  // previous tile's store has left smem
          __syncwarp();
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            __half2 h0 = __float22half2_rn(unpack2(y[4 * v + 0]));
            __half2 h1 = __float22half2_rn(unpack2(y[4 * v + 1]));
            __half2 h2 = __float22half2_rn(unpack2(y[4 * v + 2]));
            __half2 h3 = __float22half2_rn(unpack2(y[4 * v + 3]));
            sts128(ybuf + lane * 128 + ((v ^ (lane & 7)) << 4),
                   make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                              *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3)));
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmY, ybuf, nbase, m - lane);
            bulk_commit_group();
          }
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) y[j] = 0;
        }
        b = 0;
        t += sched.clusters;
      }
      __syncwarp();
      if (!kAccOut && lane == 0) mbar_arrive(&sempty[a]);
    }
  }

  if (C::kTmaStore && !kAccOut && warp < C::kNumEpiWarps && lane == 0) bulk_wait_group0();  // output stores complete
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc_2sm<512>(tmem_base);
}

}  // namespace comet
