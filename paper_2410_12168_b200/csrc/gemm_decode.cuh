// gemm_decode.cuh -- decode-regime W4Ax GEMM (M <= 128 tokens) on sm_100a.
//
// HBM-bound: the packed INT4 weight stream (N*K/2 bytes) dominates.  Swap-AB:
// the 128 weight rows of a tile are the MMA M side and live in TMEM (the A
// operand), the BN tokens are the N side (smem).  Work division is stream-K
// over (tile, K-block) units: CTA c of C owns the contiguous unit range
// [c*U/C, (c+1)*U/C) -- every SM gets the same number of blocks whatever the
// tile count ("tile decomposition ... one-to-many binding between tiles and
// SMs").  A tile split across CTAs is combined by the last
// arriving contributor, summing the partials in CTA order (deterministic),
// after the single inter-CTA sync before write-back.
//
// Per unit (one 128-channel block of one tile):
//   a3  warp 0: 1-D bulk copy of the packed weight slab [128 rows x 64 B],
//       contiguous in the tiled weight layout with the 64B swizzle baked in
//       (evict-first: read once), TMA of the token slab (INT8 blocks
//       straight into the SW128 MMA operand, INT4 blocks packed), plus 1-D
//       bulk copies of the block's scales into a scale ring;
//   a4  warps 4-7 / 8-11 (two groups taking alternate units; thread = weight
//       row): 4 x LDS.128 of the row, INT4->INT8
//       zero-extension in registers, tcgen05.st of the 32 expanded
//       columns into this stage's TMEM A slot; INT4 token blocks are expanded
//       into smem;
//   a5  warp 1: 4 x tcgen05.mma.kind::i8 (A from TMEM, M=128, N=BN, K=32)
//       into a fresh INT32 accumulator (kAcc-deep TMEM ring);
//   a6  epilogue warps (thread = weight row, columns = tokens):
//       y[m] += (sw[n] sx[m,b] 16^-e_b) * acc[m];
//   a7/a8 segment end: fp16 store, or fp32 partial + last-arriver fixup.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "gemm.cuh"
#include "quantize.cuh"
#include "sm100.cuh"

namespace comet {

template <int BN>
struct DecCfg {
  // smem stages set the HBM bytes in flight per SM (a stage is recycled only
  // after HBM latency + expansion + MMA); TMEM A slots only span expansion ->
  // MMA completion, so they are a separate, shorter ring
  static constexpr int kStages = BN <= 16 ? 16 : (BN == 32 ? 14 : (BN == 64 ? 10 : 6));
  static constexpr int kASlots = 4;
  static constexpr int kAcc = BN <= 32 ? 8 : (BN == 64 ? 4 : 2);
  static constexpr int kWPBytes = 128 * 64;  // packed weights, 64B swizzle
  static constexpr int kBBytes = BN * 128;   // tokens int8, SW128 K-major
  static constexpr int kXPBytes = BN * 64;   // packed INT4 tokens
  static constexpr int kStageBytes = kWPBytes + kBBytes + kXPBytes;  // multiple of 1024 (BN >= 16)
  static constexpr int kSlotBytes = BN * 4 + 128 * 4;                // sx[BN] + sw[128]
  static constexpr int kScaleSlots = 16;
  static constexpr int kAOff = kAcc * BN;                            // TMEM column of the A slots
  static constexpr int kTmemCols = 512;
  static constexpr int kEpiWarps = BN >= 128 ? 8 : 4;
  static constexpr int kCW = BN / (kEpiWarps / 4);                   // columns per epilogue warp
  static constexpr int kChunk = kCW >= 16 ? 16 : kCW;
  // expansion groups of 4 warps (one per TMEM lane quarter) take alternate
  // units, so two units' LDS -> zero-extend -> tcgen05.st chains overlap
  static constexpr int kExpGroups = BN >= 128 ? 1 : 2;
  static constexpr int kEpiWarp0 = 4 + 4 * kExpGroups;
  static constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);
  static constexpr int kSmemNeed = kStages * kStageBytes + kScaleSlots * kSlotBytes + 512 + 1024;
  // > half of the SM's 228 KB: exactly one CTA per SM (stream-K divides the
  // work by CTA, and each CTA owns all 512 TMEM columns)
  static constexpr int kSmemBytes = kSmemNeed > 120 * 1024 ? kSmemNeed : 120 * 1024;
  static_assert(kAOff + 32 * kASlots <= kTmemCols, "TMEM budget");
  static_assert(kSmemNeed <= 227 * 1024, "smem budget");
};

struct DecSched {
  int n_tiles, tiles, units, ctas;  // units = tiles * nb
  DEVI int u_begin(int c) const { return (int)(((int64_t)units * c) / ctas); }
};

template <int N>
DEVI void tmem_ld_n(uint32_t taddr, uint32_t (&r)[N]);
template <>
DEVI void tmem_ld_n<16>(uint32_t taddr, uint32_t (&r)[16]) { tmem_ld_32x32b_x16(taddr, r); }
template <>
DEVI void tmem_ld_n<8>(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

DEVI void epi_sync(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }

// debug: per-CTA [start, end, smid] globaltimer stamps (comet_debug_cta_times)
__device__ unsigned long long g_cta_times[3 * 1024];
__device__ int g_cta_times_on;
DEVI unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
DEVI unsigned long long clk64() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
// debug: per-role wait cycles of CTA 0: [role][0..2] = wait A, wait B, total
__device__ unsigned long long g_role_cycles[4][3];
struct RoleTimer {
  bool on;
  unsigned long long t0, w[2];
  DEVI RoleTimer(bool enabled) : on(enabled), t0(enabled ? clk64() : 0) { w[0] = w[1] = 0; }
  DEVI void wait(uint64_t* bar, uint32_t parity, int k) {
    if (!on) {
      mbar_wait(bar, parity);
      return;
    }
    const unsigned long long a = clk64();
    mbar_wait(bar, parity);
    w[k] += clk64() - a;
  }
  DEVI void flush(int role) {
    if (!on) return;
    g_role_cycles[role][0] = w[0];
    g_role_cycles[role][1] = w[1];
    g_role_cycles[role][2] = clk64() - t0;
  }
};
DEVI uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

template <int BN, bool kGroupK, bool kAccOut>
__global__ void __launch_bounds__(DecCfg<BN>::kThreads, 1)
    w4ax_gemm_decode_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX4,
                            const __grid_constant__ CUtensorMap tmX8, const __grid_constant__ BlockMap map,
                            GemmArgs args, DecSched sched) {
  using C = DecCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t scale_base = sbase + C::kStages * C::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes + C::kScaleSlots * C::kSlotBytes);
  uint64_t* full = bars;                      // [kStages]
  uint64_t* expd = full + C::kStages;         // [kStages] 4 expansion warps
  uint64_t* empty = expd + C::kStages;        // [kStages] MMA commit
  uint64_t* tfull = empty + C::kStages;       // [kAcc]
  uint64_t* tempty = tfull + C::kAcc;         // [kAcc] epilogue warps
  uint64_t* sfull = tempty + C::kAcc;         // [kScaleSlots]
  uint64_t* sempty = sfull + C::kScaleSlots;  // [kScaleSlots]
  uint64_t* aempty = sempty + C::kScaleSlots; // [kASlots] MMA commit: TMEM A slot free
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(aempty + C::kASlots);
  int* s_flag = reinterpret_cast<int*>(tmem_holder + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nb = args.nb;
  const int u0 = sched.u_begin(blockIdx.x), u1 = sched.u_begin(blockIdx.x + 1);
  const int nu = u1 - u0;
  if (threadIdx.x == 0 && g_cta_times_on && blockIdx.x < 1024) {
    g_cta_times[3 * blockIdx.x] = global_ns();
    g_cta_times[3 * blockIdx.x + 2] = smid();
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&expd[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::kAcc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], C::kEpiWarps);
    }
    for (int a = 0; a < C::kScaleSlots; ++a) {
      mbar_init(&sfull[a], 1);
      mbar_init(&sempty[a], C::kEpiWarps);
    }
    for (int a = 0; a < C::kASlots; ++a) mbar_init(&aempty[a], 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX4);
    tma_prefetch_desc(&tmX8);
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  auto tile_coords = [&](int t, int& n0, int& m0) {
    n0 = (t % sched.n_tiles) * 128;
    m0 = (t / sched.n_tiles) * BN;
  };

  if (warp == 0) {
    // ------------------------------------------------- a3: producer ----
    const uint64_t pol_w = l2_policy_evict_first();
    RoleTimer rt(g_cta_times_on && blockIdx.x == 0 && lane == 0);
    int t = u0 / nb, b = u0 - t * nb;
    int n0, m0;
    tile_coords(t, n0, m0);
    for (int i = 0; i < nu; ++i) {
      const int s = i % C::kStages;
      const uint32_t code = map.code[b];
      const bool is8 = (code >> 15) != 0;
      const int rank = code & 0x7FFF;
      rt.wait(&empty[s], ((i / C::kStages) & 1) ^ 1, 0);
      uint8_t* st = smem + s * C::kStageBytes;
      if (elect_one()) {
        mbar_arrive_expect_tx(&full[s], C::kWPBytes + (is8 ? C::kBBytes : C::kXPBytes));
        bulk_load_hint(st, args.Wq + ((int64_t)(n0 >> 7) * nb + b) * 8192, 8192, &full[s], pol_w);
        if (is8)
          tma_load_2d(st + C::kWPBytes, &tmX8, &full[s], rank * 128, m0);
        else
          tma_load_2d(st + C::kWPBytes + C::kBBytes, &tmX4, &full[s], rank * 64, m0);
      }
      if (!kAccOut) {
        const int a = i % C::kScaleSlots;
        rt.wait(&sempty[a], ((i / C::kScaleSlots) & 1) ^ 1, 1);
        if (elect_one()) {
          const bool seg_end = (b == nb - 1) || (i == nu - 1);
          const int nsx = max(0, min(BN, (int)args.ldsx - m0));  // multiple of 4
          const int nsw = (!kGroupK || seg_end) ? 128 : 0;
          mbar_arrive_expect_tx(&sfull[a], (nsx + nsw) * 4);
          uint8_t* slot = smem + C::kStages * C::kStageBytes + a * C::kSlotBytes;
          if (nsx) bulk_load(slot, args.Sx + (int64_t)b * args.ldsx + m0, nsx * 4, &sfull[a]);
          if (nsw) bulk_load(slot + BN * 4, args.Sw + (kGroupK ? 0 : (int64_t)b * args.N) + n0, 512, &sfull[a]);
        }
      }
      __syncwarp();
      if (++b == nb) {
        b = 0;
        ++t;
        if (t < sched.tiles) tile_coords(t, n0, m0);
      }
    }
    rt.flush(0);
  } else if (warp == 1) {
    // ------------------------------------------------------ a5: MMA ----
    constexpr uint32_t idesc = idesc_i8(128, BN);
    RoleTimer rt(g_cta_times_on && blockIdx.x == 0 && lane == 0);
    for (int i = 0; i < nu; ++i) {
      const int s = i % C::kStages;
      const int acc = i % C::kAcc;
      rt.wait(&tempty[acc], ((i / C::kAcc) & 1) ^ 1, 0);
      rt.wait(&expd[s], (i / C::kStages) & 1, 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t b0 = sbase + s * C::kStageBytes + C::kWPBytes;
        const int as = i % C::kASlots;
        const uint32_t a0 = tmem_base + C::kAOff + 32 * as;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_i8_ts(tmem_base + acc * BN, a0 + 8 * k, umma_desc_sw128_kmajor(b0 + 32 * k), idesc, k > 0 ? 1u : 0u);
        mma_commit(&empty[s]);
        mma_commit(&aempty[as]);
        mma_commit(&tfull[acc]);
      }
      __syncwarp();
    }
    rt.flush(1);
  } else if (warp >= 4 && warp < C::kEpiWarp0) {
    // ------------------------------------------ a4: expansion warps ----
    const int q = warp & 3;
    const int row = 32 * q + lane;  // weight row of the tile = TMEM lane
    const int grp = (warp - 4) >> 2;
    const int tid = threadIdx.x - 128 - 128 * grp;
    int b = (u0 + grp) % nb;
    RoleTimer rt(g_cta_times_on && blockIdx.x == 0 && warp == 4 && lane == 0);
    for (int i = grp; i < nu; i += C::kExpGroups) {
      const int s = i % C::kStages;
      const bool is8 = (map.code[b] >> 15) != 0;
      b += C::kExpGroups;
      if (b >= nb) b -= nb;
      const uint32_t st = sbase + s * C::kStageBytes;
      rt.wait(&full[s], (i / C::kStages) & 1, 0);
      // own weight row: 4 x 16 B, 64B-swizzled (chunk c at c ^ ((row >> 1) & 3))
      uint32_t e[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 w = lds128(st + row * 64 + ((c ^ ((row >> 1) & 3)) << 4));
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t tt = ww[k] & 0x0F0F0F0Fu;
          e[8 * c + 2 * k] = tt << 4;           // 16*e0..3
          e[8 * c + 2 * k + 1] = ww[k] - tt;    // 16*e4..7
        }
      }
      const int as = i % C::kASlots;
      rt.wait(&aempty[as], ((i / C::kASlots) & 1) ^ 1, 1);  // MMA of unit i - kASlots done
      tc_fence_after();
      tmem_st_32x32b_x32(tmem_base + ((uint32_t)(32 * q) << 16) + C::kAOff + 32 * as, e);
      if (!is8) {
        const uint32_t xp = st + C::kWPBytes + C::kBBytes;
        const uint32_t xb = st + C::kWPBytes;
        for (int tk = tid; tk < BN * 4; tk += 128) {
          const int r = tk >> 2, j = tk & 3;
          const uint4 w = lds128(xp + r * 64 + j * 16);
          uint4 o0, o1;
          uint32_t tt;
          tt = w.x & 0x0F0F0F0Fu; o0.x = tt << 4; o0.y = w.x - tt;
          tt = w.y & 0x0F0F0F0Fu; o0.z = tt << 4; o0.w = w.y - tt;
          tt = w.z & 0x0F0F0F0Fu; o1.x = tt << 4; o1.y = w.z - tt;
          tt = w.w & 0x0F0F0F0Fu; o1.z = tt << 4; o1.w = w.w - tt;
          sts128(xb + r * 128 + (((2 * j) ^ (r & 7)) << 4), o0);
          sts128(xb + r * 128 + (((2 * j + 1) ^ (r & 7)) << 4), o1);
        }
        fence_proxy_async_smem();
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&expd[s]);
    }
    rt.flush(2);
  } else if (warp >= C::kEpiWarp0) {
    // ----------------------------------------- a6-a8: epilogue warps ----
    const int q = warp & 3;
    const int h = (warp - C::kEpiWarp0) >> 2;  // column group
    const int row = 32 * q + lane;
    const int col0 = h * C::kCW;
    const uint32_t tl = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)col0;
    float y[C::kCW];
#pragma unroll
    for (int j = 0; j < C::kCW; ++j) y[j] = 0.f;
    int t = u0 / nb, b = u0 - t * nb;
    int seg_first = b;  // first block of the current segment
    RoleTimer rt(g_cta_times_on && blockIdx.x == 0 && warp == C::kEpiWarp0 && lane == 0);
    for (int i = 0; i < nu; ++i) {
      const int acc = i % C::kAcc;
      const int a = i % C::kScaleSlots;
      const uint32_t slot = scale_base + a * C::kSlotBytes;
      const bool is8 = (map.code[b] >> 15) != 0;
      int n0, m0;
      tile_coords(t, n0, m0);
      const int n = n0 + row;
      float swv = 0.f;
      if (!kAccOut) {
        rt.wait(&sfull[a], (i / C::kScaleSlots) & 1, 0);
        swv = kGroupK ? 1.f : lds_f32(slot + BN * 4 + row * 4);
        swv *= is8 ? 0.0625f : 0.00390625f;  // fold 16^-e
      }
      rt.wait(&tfull[acc], (i / C::kAcc) & 1, 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < C::kCW; c += C::kChunk) {
        uint32_t r[C::kChunk];
        tmem_ld_n<C::kChunk>(tl + acc * BN + c, r);
        tmem_ld_wait();
        if (kAccOut) {
          const int sh = is8 ? 4 : 8;
#pragma unroll
          for (int j = 0; j < C::kChunk; ++j) {
            const int m = m0 + col0 + c + j;
            if (m < args.M) args.Acc[((int64_t)b * args.M + m) * args.N + n] = ((int32_t)r[j]) >> sh;
          }
        } else {
#pragma unroll
          for (int j4 = 0; j4 < C::kChunk; j4 += 4) {
            const float4 sx4 = lds_f32x4(slot + (col0 + c + j4) * 4);
            y[c + j4 + 0] = fmaf(i2f(r[j4 + 0]), sx4.x * swv, y[c + j4 + 0]);
            y[c + j4 + 1] = fmaf(i2f(r[j4 + 1]), sx4.y * swv, y[c + j4 + 1]);
            y[c + j4 + 2] = fmaf(i2f(r[j4 + 2]), sx4.z * swv, y[c + j4 + 2]);
            y[c + j4 + 3] = fmaf(i2f(r[j4 + 3]), sx4.w * swv, y[c + j4 + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);

      const bool tile_end = (b == nb - 1);
      const bool seg_end = tile_end || (i == nu - 1);
      if (!kAccOut && seg_end) {
        if (kGroupK) {
          const float swr = lds_f32(slot + BN * 4 + row * 4);
#pragma unroll
          for (int j = 0; j < C::kCW; ++j) y[j] *= swr;
        }
        if (seg_first == 0 && tile_end) {
          // whole tile in this CTA: direct write-back
#pragma unroll
          for (int j = 0; j < C::kCW; ++j) {
            const int m = m0 + col0 + j;
            if (m < args.M) args.Y[(int64_t)m * args.ldy + n] = __float2half_rn(y[j]);
          }
        } else {
          // ------------------------- a7: stream-K partial + fixup ----
          // slot (cta, 0) = partial of the first tile of this CTA, (cta, 1) = last;
          // layout [row][BN]: this thread's kCW columns are contiguous
          const int which = (seg_first == (u0 % nb) && t == u0 / nb) ? 0 : 1;
          float* part = args.ws_partial + ((int64_t)blockIdx.x * 2 + which) * (128 * BN) + row * BN + col0;
#pragma unroll
          for (int j = 0; j < C::kCW; j += 4)
            __stcg(reinterpret_cast<float4*>(part + j), make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]));
          __threadfence();
          epi_sync(32 * C::kEpiWarps);
          // contributors of tile t: CTAs whose unit range intersects [t*nb, (t+1)*nb)
          const int tu0 = t * nb, tu1 = tu0 + nb;
          int c_lo = (int)(((int64_t)tu0 * sched.ctas) / sched.units);
          while (c_lo > 0 && sched.u_begin(c_lo) > tu0) --c_lo;
          while (sched.u_begin(c_lo + 1) <= tu0) ++c_lo;
          int c_hi = (int)(((int64_t)(tu1 - 1) * sched.ctas) / sched.units);
          while (c_hi > 0 && sched.u_begin(c_hi) > tu1 - 1) --c_hi;
          while (sched.u_begin(c_hi + 1) <= tu1 - 1) ++c_hi;
          if (threadIdx.x == 32 * C::kEpiWarp0) {
            const int prev = atomicAdd(args.ws_counter + t, 1);
            *s_flag = (prev == c_hi - c_lo);
          }
          epi_sync(32 * C::kEpiWarps);
          if (*s_flag) {
            __threadfence();
            // sum the contributors in CTA order (deterministic); each round
            // issues kCW/4 independent 16-byte loads
#pragma unroll
            for (int j = 0; j < C::kCW; ++j) y[j] = 0.f;
            for (int cc = c_lo; cc <= c_hi; ++cc) {
              // the tile is cc's first tile unless cc started in an earlier tile
              const int w = (sched.u_begin(cc) >= tu0) ? 0 : 1;
              const float* src = args.ws_partial + ((int64_t)cc * 2 + w) * (128 * BN) + row * BN + col0;
              float4 v[C::kCW / 4];
#pragma unroll
              for (int j = 0; j < C::kCW; j += 4) v[j / 4] = __ldcg(reinterpret_cast<const float4*>(src + j));
#pragma unroll
              for (int j = 0; j < C::kCW; j += 4) {
                y[j] += v[j / 4].x;
                y[j + 1] += v[j / 4].y;
                y[j + 2] += v[j / 4].z;
                y[j + 3] += v[j / 4].w;
              }
            }
#pragma unroll
            for (int j = 0; j < C::kCW; ++j) {
              const int m = m0 + col0 + j;
              if (m < args.M) args.Y[(int64_t)m * args.ldy + n] = __float2half_rn(y[j]);
            }
            if (threadIdx.x == 32 * C::kEpiWarp0) args.ws_counter[t] = 0;
          }
        }
#pragma unroll
        for (int j = 0; j < C::kCW; ++j) y[j] = 0.f;
      }
      __syncwarp();
      if (!kAccOut && lane == 0) mbar_arrive(&sempty[a]);
      if (++b == nb) {
        b = 0;
        ++t;
      }
      if (seg_end) seg_first = b;
    }
    rt.flush(3);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem_base);
  if (threadIdx.x == 0 && g_cta_times_on && blockIdx.x < 1024) g_cta_times[3 * blockIdx.x + 1] = global_ns();
}

}  // namespace comet
