// gemm_2sm.cuh -- prefill W4Ax GEMM on a CTA pair (tcgen05 cta_group::2).
//
// Pair tile: 256 tokens (MMA M, 128 TMEM lanes in each CTA) x 256 weight
// rows (MMA N; each CTA stages 128 of them), K walked one 128-channel FMPQ
// block at a time.  Per block and CTA:
//   a3  warp 0: TMA the packed weight slab [128 x 64 B] and the token slab --
//       INT8 blocks [128 x 128 B] straight into the MMA operand (SW128),
//       INT4 blocks packed [128 x 64 B]; 1-D bulk copies of the block's scales
//       into an 8-deep scale ring.
//   a4  warps 2-17 ("compute warps"): INT4 -> INT8 zero-extension
//       of the weights (and of INT4 token blocks) of block i+1 into SW128
//       K-major smem -- one 16-byte packed chunk per thread per operand --
//       then an arrive on the leader CTA's "expanded" barrier ...
//   a5  warp 1 of the leader CTA: 4 x tcgen05.mma.cta_group::2.kind::i8
//       (M=256, N=256, K=32) into a fresh INT32 accumulator in both CTAs'
//       TMEM (two 256-column accumulators ping-pong = all 512 columns);
//       tcgen05.commit multicasts to both CTAs' barriers.
//   a6  ... and promote block i: tcgen05.ld 16 columns at a time, I2F, and
//       y += (sx[m,b] 16^-e_b) * acc  with fma.rn.f32x2 (sx is uniform per
//       thread because a thread owns a token row); group-128 weights also
//       multiply by sw[n,b] (mul.rn.f32x2); per-channel weights apply sw[n]
//       once at the end.
//   a8  fp32 -> fp16 RNE, 16-byte stores of the thread's 64 columns.
// The only inter-SM synchronization is the pair's barrier protocol; tiles
// never wait on each other ("synchronization is only necessary
// after all iterations are completed").
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "gemm.cuh"
#include "quantize.cuh"
#include "sm100.cuh"

namespace comet {

struct Gemm2Cfg {
  static constexpr int kStages = 4;
  static constexpr int kScaleSlots = 8;
  static constexpr int kABytes = 128 * 128;   // tokens int8, SW128 K-major
  static constexpr int kBBytes = 128 * 128;   // weights int8 (this CTA's half of N)
  static constexpr int kXPBytes = 128 * 64;   // packed INT4 tokens
  static constexpr int kWPBytes = 128 * 64;   // packed INT4 weights
  static constexpr int kStageBytes = kABytes + kBBytes + kXPBytes + kWPBytes;  // 48 KiB
  static constexpr int kSlotBytes = 128 * 4 + 256 * 4;                        // sx[128] + sw[256]
  static constexpr int kScaleBytes = kScaleSlots * kSlotBytes + 256 * 4;      // + per-channel sw[256]
  static constexpr int kBarBytes = 256;
  static constexpr int kSmemBytes = kStages * kStageBytes + kScaleBytes + kBarBytes + 1024;
  static constexpr int kThreads = 576;  // 18 warps: TMA, MMA, 16 compute
  static constexpr int kEpiWarp0 = 2;
  static constexpr int kNumEpiWarps = 16;
};

template <bool kGroupK, bool kAccOut>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(576, 1)
    w4ax_gemm_2sm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX4,
                         const __grid_constant__ CUtensorMap tmX8, const __grid_constant__ BlockMap map, GemmArgs args) {
  using C = Gemm2Cfg;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  uint8_t* scale_area = smem + C::kStages * C::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(scale_area + C::kScaleBytes);
  uint64_t* full = bars;                       // [kStages] local TMA tx
  uint64_t* expd = full + C::kStages;          // [kStages] leader: 2 CTAs x 2 expansion warps
  uint64_t* empty = expd + C::kStages;         // [kStages] MMA commit (multicast)
  uint64_t* tfull = empty + C::kStages;        // [2] MMA commit (multicast)
  uint64_t* tempty = tfull + 2;                // [2] leader: 2 CTAs x 16 epilogue warps
  uint64_t* sfull = tempty + 2;                // [kScaleSlots] local bulk tx
  uint64_t* sempty = sfull + C::kScaleSlots;   // [kScaleSlots] local epilogue warps
  uint64_t* swfull = sempty + C::kScaleSlots;  // [1] per-channel weight scales
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(swfull + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const int m0 = (blockIdx.x >> 1) * 256;  // pair's first token
  const int n0 = blockIdx.y * 256;         // pair's first weight row
  const int my_m0 = m0 + 128 * (int)crank;
  const int my_n0 = n0 + 128 * (int)crank;
  const int nb = args.nb;

  auto a_addr = [&](int s) { return sbase + s * C::kStageBytes; };
  auto b_addr = [&](int s) { return sbase + s * C::kStageBytes + C::kABytes; };
  auto xp_ptr = [&](int s) { return smem + s * C::kStageBytes + C::kABytes + C::kBBytes; };
  auto wp_ptr = [&](int s) { return smem + s * C::kStageBytes + C::kABytes + C::kBBytes + C::kXPBytes; };
  auto sx_ptr = [&](int a) { return scale_area + a * C::kSlotBytes; };
  auto sw_ptr = [&](int a) { return scale_area + a * C::kSlotBytes + 128 * 4; };
  uint8_t* swk_ptr = scale_area + C::kScaleSlots * C::kSlotBytes;

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
    mbar_init(swfull, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX4);
    tma_prefetch_desc(&tmX8);
  }
  if (warp == 1) tmem_alloc_2sm<512>(tmem_holder);
  tc_fence_before();
  cluster_sync();  // barrier inits + TMEM allocation visible cluster-wide
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const uint32_t leader_expd = mapa_shared(smem_u32(expd), 0);
  const uint32_t leader_tempty = mapa_shared(smem_u32(tempty), 0);

  if (warp == 0) {
    // ------------------------------------------------------- producer ----
    if (elect_one()) {
      if (kGroupK && !kAccOut) {
        const int nv = min(256, args.N - n0);
        mbar_arrive_expect_tx(swfull, nv * 4);
        bulk_load(swk_ptr, args.Sw + n0, nv * 4, swfull);
      }
      for (int i = 0; i < nb; ++i) {
        const int s = i % C::kStages;
        const uint32_t ph = (i / C::kStages) & 1;
        const uint32_t code = map.code[i];
        const bool is8 = (code >> 15) != 0;
        const int rank = code & 0x7FFF;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], C::kWPBytes + (is8 ? C::kABytes : C::kXPBytes));
        tma_load_2d(wp_ptr(s), &tmW, &full[s], i * 64, my_n0);
        if (is8)
          tma_load_2d(smem + s * C::kStageBytes, &tmX8, &full[s], rank * 128, my_m0);
        else
          tma_load_2d(xp_ptr(s), &tmX4, &full[s], rank * 64, my_m0);
        if (!kAccOut) {
          const int a = i % C::kScaleSlots;
          const uint32_t aph = (i / C::kScaleSlots) & 1;
          mbar_wait(&sempty[a], aph ^ 1);
          const int nsx = max(0, min(128, (int)args.ldsx - my_m0));  // multiple of 4
          const int nsw = kGroupK ? 0 : max(0, min(256, args.N - n0));
          mbar_arrive_expect_tx(&sfull[a], (nsx + nsw) * 4);
          if (nsx) bulk_load(sx_ptr(a), args.Sx + (int64_t)i * args.ldsx + my_m0, nsx * 4, &sfull[a]);
          if (nsw) bulk_load(sw_ptr(a), args.Sw + (int64_t)i * args.N + n0, nsw * 4, &sfull[a]);  // group 128: g(b) = b
        }
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------- MMA (leader CTA) ----
    if (crank == 0) {
      constexpr uint32_t idesc = idesc_i8(256, 256);
      for (int i = 0; i < nb; ++i) {
        const int s = i % C::kStages;
        const uint32_t ph = (i / C::kStages) & 1;
        const int acc = i & 1;
        const uint32_t aph = (i >> 1) & 1;
        mbar_wait_cluster(&tempty[acc], aph ^ 1);
        mbar_wait_cluster(&expd[s], ph);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_i8_ss_2sm(tmem_base + acc * 256, umma_desc_sw128_kmajor(a_addr(s) + 32 * k),
                          umma_desc_sw128_kmajor(b_addr(s) + 32 * k), idesc, k > 0 ? 1u : 0u);
          mma_commit_2sm(&empty[s], 0x3);
          mma_commit_2sm(&tfull[acc], 0x3);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------ compute warps: a4 + a6 + a8 ----
    // Iteration i: expand block i+1 (INT4 -> INT8 into the stage the MMA
    // reads next), then promote block i's accumulator.  The MMA of block i+1
    // overlaps the promotion of block i.
    const int ct = threadIdx.x - 32 * C::kEpiWarp0;  // 0..511
    const int e = warp - C::kEpiWarp0;
    const int q = warp & 3;            // TMEM lane quarter
    const int cg = e >> 2;             // 64-column group
    const int row = 32 * q + lane;     // token row within this CTA
    const int m = my_m0 + row;
    const uint32_t tl = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(64 * cg);
    // this thread's expansion task: packed row ct/4, 16-byte chunk ct%4
    const int er = ct >> 2, ej = ct & 3;
    const uint32_t e_src = er * 64 + ej * 16;
    const uint32_t e_dst0 = er * 128 + (((2 * ej) ^ (er & 7)) << 4);
    const uint32_t e_dst1 = er * 128 + (((2 * ej + 1) ^ (er & 7)) << 4);

    auto expand = [&](int j) {
      const int s = j % C::kStages;
      mbar_wait(&full[s], (j / C::kStages) & 1);
      const uint32_t wp = smem_u32(wp_ptr(s)) + e_src;
      const uint4 w = lds128(wp);
      const bool is8 = (map.code[j] >> 15) != 0;
      uint4 x = make_uint4(0, 0, 0, 0);
      if (!is8) x = lds128(smem_u32(xp_ptr(s)) + e_src);
      {
        const uint32_t t0 = w.x & 0x0F0F0F0Fu, t1 = w.y & 0x0F0F0F0Fu, t2 = w.z & 0x0F0F0F0Fu, t3 = w.w & 0x0F0F0F0Fu;
        sts128(b_addr(s) + e_dst0, make_uint4(t0 << 4, w.x - t0, t1 << 4, w.y - t1));
        sts128(b_addr(s) + e_dst1, make_uint4(t2 << 4, w.z - t2, t3 << 4, w.w - t3));
      }
      if (!is8) {
        const uint32_t t0 = x.x & 0x0F0F0F0Fu, t1 = x.y & 0x0F0F0F0Fu, t2 = x.z & 0x0F0F0F0Fu, t3 = x.w & 0x0F0F0F0Fu;
        sts128(a_addr(s) + e_dst0, make_uint4(t0 << 4, x.x - t0, t1 << 4, x.y - t1));
        sts128(a_addr(s) + e_dst1, make_uint4(t2 << 4, x.z - t2, t3 << 4, x.w - t3));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_expd + s * 8);
    };

    float2 y[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) y[j] = make_float2(0.f, 0.f);

    expand(0);
    for (int i = 0; i < nb; ++i) {
      if (i + 1 < nb) expand(i + 1);
      const int acc = i & 1;
      const uint32_t aph = (i >> 1) & 1;
      const int a = i % C::kScaleSlots;
      const uint32_t sph = (i / C::kScaleSlots) & 1;
      const bool is8 = (map.code[i] >> 15) != 0;
      float sxv = 0.f;
      if (!kAccOut) {
        mbar_wait(&sfull[a], sph);
        sxv = lds_f32(smem_u32(sx_ptr(a)) + row * 4) * (is8 ? 0.0625f : 0.00390625f);
      }
      const float2 sx2 = make_float2(sxv, sxv);
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tl + acc * 256 + 16 * c, r);
        tmem_ld_wait();
        if (kAccOut) {
          const int sh = is8 ? 4 : 8;
          if (m < args.M) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int n = n0 + 64 * cg + 16 * c + j;
              if (n < args.N) args.Acc[((int64_t)i * args.M + m) * args.N + n] = ((int32_t)r[j]) >> sh;
            }
          }
        } else if (kGroupK) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            y[8 * c + j] = fma2(make_float2(i2f(r[2 * j]), i2f(r[2 * j + 1])), sx2, y[8 * c + j]);
        } else {
          const uint32_t swa = smem_u32(sw_ptr(a)) + (64 * cg + 16 * c) * 4;
#pragma unroll
          for (int j4 = 0; j4 < 4; ++j4) {
            const float4 w4 = lds_f32x4(swa + 16 * j4);
            const float2 s01 = mul2(sx2, make_float2(w4.x, w4.y));
            const float2 s23 = mul2(sx2, make_float2(w4.z, w4.w));
            y[8 * c + 2 * j4] = fma2(make_float2(i2f(r[4 * j4]), i2f(r[4 * j4 + 1])), s01, y[8 * c + 2 * j4]);
            y[8 * c + 2 * j4 + 1] = fma2(make_float2(i2f(r[4 * j4 + 2]), i2f(r[4 * j4 + 3])), s23, y[8 * c + 2 * j4 + 1]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_cluster(leader_tempty + acc * 8);
        if (!kAccOut) mbar_arrive(&sempty[a]);
      }
    }

    if (!kAccOut) {
      const int nbase = n0 + 64 * cg;
      if (kGroupK) {
        mbar_wait(swfull, 0);
        const uint32_t swa = smem_u32(swk_ptr) + 64 * cg * 4;
#pragma unroll
        for (int j4 = 0; j4 < 16; ++j4) {
          const float4 w4 = lds_f32x4(swa + 16 * j4);
          y[2 * j4] = mul2(y[2 * j4], make_float2(w4.x, w4.y));
          y[2 * j4 + 1] = mul2(y[2 * j4 + 1], make_float2(w4.z, w4.w));
        }
      }
      if (m < args.M && nbase < args.N) {
        __half* yrow = args.Y + (int64_t)m * args.ldy + nbase;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          __half2 h0 = __float22half2_rn(y[4 * v + 0]);
          __half2 h1 = __float22half2_rn(y[4 * v + 1]);
          __half2 h2 = __float22half2_rn(y[4 * v + 2]);
          __half2 h3 = __float22half2_rn(y[4 * v + 3]);
          uint4 pk = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                                *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
          *reinterpret_cast<uint4*>(yrow + 8 * v) = pk;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_2sm<512>(tmem_base);
}

}  // namespace comet
