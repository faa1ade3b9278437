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
// Per unit (up to kUB consecutive 128-channel blocks of one tile):
//   a3  warp 0: one 1-D bulk copy of the unit's packed weight slabs
//       [kUB x 128 rows x 64 B], contiguous in the tiled weight layout with the
//       64B swizzle baked in (evict-first: read once); a TMA of each block's
//       token slab (INT8 blocks straight into the SW128 MMA operand, INT4
//       blocks packed) and a 2-D TMA box of the unit's scales into a scale
//       ring -- the token/scale loads are issued by warp 2 so the weight
//       stream's issue path stays short;
//   a4  warps 4-7 / 8-11 (two groups taking alternate units; thread = weight
//       row): per block 4 x LDS.128 of the row, INT4->INT8 zero-extension in
//       registers, tcgen05.st of the 32 expanded columns into the
//       unit's TMEM A slot; INT4 token blocks are expanded into smem;
//   a5  warp 1: per block 4 x tcgen05.mma.kind::i8 (A from TMEM, M=128, N=BN,
//       K=32) into a fresh INT32 accumulator (kAcc-deep TMEM ring of units);
//   a6  epilogue warps (thread = weight row, columns = tokens):
//       y[m] += (sw[n] sx[m,b] 16^-e_b) * acc_b[m] for each block b;
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
  // a unit is up to kUB consecutive K-blocks of one tile: one contiguous
  // kUB x 8 KB weight copy, one set of barrier hand-offs and one accumulator
  // slot of kUB x BN columns per unit (the fixed per-unit cost of every role
  // is paid once per kUB blocks)
  static constexpr int kUB = BN <= 32 ? 4 : (BN == 64 ? 2 : 1);
  static constexpr int kWPBytes = 128 * 64;  // packed weights of one block, 64B swizzle
  static constexpr int kBBytes = BN * 128;   // tokens int8 of one block, SW128 K-major
  static constexpr int kXPBytes = BN * 64;   // packed INT4 tokens of one block
  // two smem rings: weights [kUB x kWPBytes], released by the expansion warps
  // as soon as they have read them (the MMA never touches packed weights), and
  // tokens [B: kUB x kBBytes][XP: kUB x kXPBytes], released by the MMA commit
  static constexpr int kWStageBytes = kUB * kWPBytes;
  static constexpr int kXStageBytes = kUB * (kBBytes + kXPBytes);
  static constexpr int kXPOff = kUB * kBBytes;  // within a token stage
  // weight stages set the HBM bytes in flight per SM
  static constexpr int kWStages = BN == 16 ? 5 : (BN == 32 ? 4 : (BN == 64 ? 7 : 10));
  static constexpr int kXStages = BN == 128 ? 4 : 3;
  static constexpr int kXBase = kWStages * kWStageBytes;
  // scale slot = [sx: kUB x BN][sw: kUB x 128] fp32
  static constexpr int kSxBytes = kUB * BN * 4;
  static constexpr int kSlotBytes = kSxBytes + kUB * 128 * 4;
  static constexpr int kScaleSlots = BN <= 32 ? 6 : 8;
  static constexpr int kScaleBase = kXBase + kXStages * kXStageBytes;
  static constexpr int kBarBase = kScaleBase + kScaleSlots * kSlotBytes;
  // TMEM: kAcc accumulator slots of kUB x BN columns, then kASlots weight
  // (A operand) slots of kUB x 32 columns
  static constexpr int kASlots = BN == 16 ? 3 : (kUB == 1 ? 4 : 2);
  static constexpr int kAccCols = kUB * BN;
  static constexpr int kAccMax = (512 - kASlots * 32 * kUB) / kAccCols;
  static constexpr int kAcc = kAccMax > 8 ? 8 : kAccMax;
  static constexpr int kAOff = kAcc * kAccCols;  // TMEM column of the A slots
  static constexpr int kTmemCols = 512;
  // two column halves x 4 lane quarters
  static constexpr int kEpiWarps = 8;
  static constexpr int kCW = BN / (kEpiWarps / 4);  // columns per epilogue warp
  static constexpr int kChunk = kCW >= 16 ? 16 : kCW;
  // blocks whose accumulators are loaded before one tcgen05.wait::ld
  static constexpr int kLdG0 = 32 / kCW > 0 ? 32 / kCW : 1;
  static constexpr int kLdG = kLdG0 < kUB ? kLdG0 : kUB;
  // expansion groups of 4 warps (one per TMEM lane quarter) take alternate
  // units, so two units' LDS -> zero-extend -> tcgen05.st chains overlap
  static constexpr int kExpGroups = BN >= 128 ? 1 : 2;
  // warp ids (epilogue warps first measured the same: 70B gate_up M=16 59.4 us)
  static constexpr int kWWarp = 0, kMmaWarp = 1, kXWarp = 2, kExpWarp0 = 4, kEpiWarp0 = 4 + 4 * kExpGroups;
  static constexpr int kThreads = 32 * (4 + 4 * kExpGroups + kEpiWarps);
  static constexpr int kSmemNeed = kBarBase + 1024 + 1024;
  // > half of the SM's 228 KB: exactly one CTA per SM (stream-K divides the
  // work by CTA, and each CTA owns all 512 TMEM columns)
  static constexpr int kSmemBytes = kSmemNeed > 120 * 1024 ? kSmemNeed : 120 * 1024;
  static_assert(kAcc >= 2, "TMEM budget");
  static_assert(kAOff + 32 * kUB * kASlots <= kTmemCols, "TMEM budget");
  static_assert(kSmemNeed <= 227 * 1024, "smem budget");
  static_assert(kXBase % 1024 == 0 && kXStageBytes % 1024 == 0 && kBBytes % 1024 == 0, "SW128 alignment");
};

struct DecSched {
  int n_tiles, tiles, units, ctas;  // units = tiles * nb K-blocks (the stream-K split granularity)
  // 32-bit: the host guarantees units * ctas < 2^32 (tiles <= 16384, nb <= 512)
  DEVI int u_begin(int c) const { return (int)(((uint32_t)units * (uint32_t)c) / (uint32_t)ctas); }
};

// walks a CTA's block range [u, u1) in units of up to KUB blocks that never
// cross a tile boundary; every role replays the same sequence
template <int KUB>
struct UnitIt {
  int u, u1, t, b, len;  // global block index, range end, tile, block in tile, blocks in unit
  int tn, tm, n_tiles;   // tile t = tm * n_tiles + tn (channel tile tn fastest), kept without division
  DEVI UnitIt(int u0_, int u1_, int nb, int n_tiles_) : u(u0_), u1(u1_), n_tiles(n_tiles_) {
    t = u / nb;
    b = u - t * nb;
    tm = t / n_tiles;
    tn = t - tm * n_tiles;
    set_len(nb);
  }
  DEVI void set_len(int nb) { len = min(min(KUB, nb - b), u1 - u); }
  DEVI bool valid() const { return u < u1; }
  DEVI void next(int nb) {
    u += len;
    b += len;
    if (b == nb) {
      b = 0;
      ++t;
      if (++tn == n_tiles) {
        tn = 0;
        ++tm;
      }
    }
    set_len(nb);
  }
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

template <int BN, bool kGroupK, bool kAccOut>
#ifndef DEC_LB
#define DEC_LB 0  // 0: DecCfg<BN>::kThreads (tools: a larger bound lowers the register cap)
#endif
__global__ void __launch_bounds__(DEC_LB > 0 ? DEC_LB : DecCfg<BN>::kThreads, 1)
    w4ax_gemm_decode_kernel(const __grid_constant__ CUtensorMap tmSx, const __grid_constant__ CUtensorMap tmX4,
                            const __grid_constant__ CUtensorMap tmX8, const __grid_constant__ CUtensorMap tmSw,
                            const __grid_constant__ BlockMap map, GemmArgs args, DecSched sched) {
  using C = DecCfg<BN>;
  using It = UnitIt<C::kUB>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t scale_base = sbase + C::kScaleBase;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarBase);
  uint64_t* wfull = bars;                     // [kWStages] weight bytes landed
  uint64_t* wempty = wfull + C::kWStages;     // [kWStages] 4 expansion warps read them
  uint64_t* xfull = wempty + C::kWStages;     // [kXStages] token bytes landed
  uint64_t* xempty = xfull + C::kXStages;     // [kXStages] MMA commit
  uint64_t* expd = xempty + C::kXStages;      // [kXStages] 4 expansion warps
  uint64_t* tfull = expd + C::kXStages;       // [kAcc]
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
  if (threadIdx.x == 0 && g_cta_times_on && blockIdx.x < 1024) {
    g_cta_times[3 * blockIdx.x] = global_ns();
    g_cta_times[3 * blockIdx.x + 2] = smid();
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kWStages; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 4);
    }
    for (int s = 0; s < C::kXStages; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
      mbar_init(&expd[s], 4);
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
  if (warp == C::kXWarp && lane == 0) {
    tma_prefetch_desc(&tmX4);
    tma_prefetch_desc(&tmX8);
    tma_prefetch_desc(&tmSx);
    if (!kGroupK) tma_prefetch_desc(&tmSw);
  }
  if (warp == C::kMmaWarp) tmem_alloc<C::kTmemCols>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  // (no griddepcontrol.launch_dependents here: letting the next layer's
  // quantizer launch early slowed the 70B decode step 0.137 -> 0.158 ms)
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;


  if (warp == C::kWWarp) {
    // ------------------------------------------ a3: weight producer ----
    // only the HBM weight stream: one bulk copy per unit, nothing else on
    // this warp's issue path
    const uint64_t pol_w = l2_policy_evict_first();
    RoleTimer rt(g_cta_times_on && blockIdx.x + 1 == g_cta_times_on && lane == 0);
    int i = 0;
    // PDL: while the quantizer that precedes this GEMM still runs, warm L2 with
    // the first units' weights (an L2 prefetch cannot expose stale data: L2 is
    // the point of coherence), then wait for the predecessor before any load
    // into shared memory (the weights may have been written by it)
    if (elect_one()) {
      int k = 0;
      for (It it(u0, u1, nb, sched.n_tiles); it.valid() && k < C::kWStages; it.next(nb), ++k)
        bulk_prefetch_l2(args.Wq + ((int64_t)it.tn * nb + it.b) * 8192, it.len * 8192);
    }
    grid_dep_wait();
    for (It it(u0, u1, nb, sched.n_tiles); it.valid(); it.next(nb), ++i) {
      const int s = i % C::kWStages;
      rt.wait(&wempty[s], ((i / C::kWStages) & 1) ^ 1, 0);
      trace(rt.on, 0, i);
      if (elect_one()) {
        mbar_arrive_expect_tx(&wfull[s], it.len * C::kWPBytes);
        // the unit's blocks are consecutive 8 KB slabs of the tiled layout
        bulk_load_hint(smem + s * C::kWStageBytes, args.Wq + ((int64_t)it.tn * nb + it.b) * 8192,
                       it.len * 8192, &wfull[s], pol_w);
      }
      __syncwarp();
    }
    rt.flush(0);
  } else if (warp == C::kXWarp) {
    // ---------------------------------- a3: token + scale producer ----
    grid_dep_wait();  // PDL: the planes and scales come from the preceding quantizer
    const bool tr_on = g_cta_times_on && blockIdx.x + 1 == g_cta_times_on && lane == 0;
    int i = 0;
    for (It it(u0, u1, nb, sched.n_tiles); it.valid(); it.next(nb), ++i) {
      const int s = i % C::kXStages;
      const int n0 = it.tn * 128, m0 = it.tm * BN;
      mbar_wait(&xempty[s], ((i / C::kXStages) & 1) ^ 1);
      trace(tr_on, 1, i);
      uint8_t* st = smem + C::kXBase + s * C::kXStageBytes;
      if (elect_one()) {
        uint32_t tx = 0;
#pragma unroll
        for (int j = 0; j < C::kUB; ++j)
          if (j < it.len) tx += (map.code[it.b + j] >> 15) ? C::kBBytes : C::kXPBytes;
        mbar_arrive_expect_tx(&xfull[s], tx);
#pragma unroll
        for (int j = 0; j < C::kUB; ++j) {
          if (j < it.len) {
            const uint32_t code = map.code[it.b + j];
            const int rank = code & 0x7FFF;
            if (code >> 15)
              tma_load_2d(st + j * C::kBBytes, &tmX8, &xfull[s], rank * 128, m0);
            else
              tma_load_2d(st + C::kXPOff + j * C::kXPBytes, &tmX4, &xfull[s], rank * 64, m0);
          }
        }
      }
      if (!kAccOut) {
        const int a = i % C::kScaleSlots;
        mbar_wait(&sempty[a], ((i / C::kScaleSlots) & 1) ^ 1);
        if (elect_one()) {
          const bool seg_end = (it.b + it.len == nb) || (it.u + it.len == u1);
          uint8_t* slot = smem + C::kScaleBase + a * C::kSlotBytes;
          // sx of the unit's blocks: one [kUB x BN] box of Sx [nb x ldsx]
          // (columns >= ldsx and rows >= nb are zero-filled, still counted)
          const uint32_t tx = C::kSxBytes +
                              (kGroupK ? (seg_end ? 512 : 0) : C::kUB * 512);
          mbar_arrive_expect_tx(&sfull[a], tx);
          tma_load_2d(slot, &tmSx, &sfull[a], m0, it.b);
          if (!kGroupK)
            tma_load_2d(slot + C::kSxBytes, &tmSw, &sfull[a], n0, it.b);  // [kUB x 128] box of Sw [nb x N]
          else if (seg_end)
            bulk_load(slot + C::kSxBytes, args.Sw + n0, 512, &sfull[a]);
        }
      }
      __syncwarp();
    }
  } else if (warp == C::kMmaWarp) {
    // ------------------------------------------------------ a5: MMA ----
    constexpr uint32_t idesc = idesc_i8(128, BN);
    RoleTimer rt(g_cta_times_on && blockIdx.x + 1 == g_cta_times_on && lane == 0);
    int i = 0;
    for (It it(u0, u1, nb, sched.n_tiles); it.valid(); it.next(nb), ++i) {
      const int s = i % C::kXStages;
      const int acc = i % C::kAcc;
      rt.wait(&tempty[acc], ((i / C::kAcc) & 1) ^ 1, 0);
      rt.wait(&expd[s], (i / C::kXStages) & 1, 1);
      trace(rt.on, 4, i);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t bst = sbase + C::kXBase + s * C::kXStageBytes;
        const int as = i % C::kASlots;
        const uint32_t a0 = tmem_base + C::kAOff + 32 * C::kUB * as;
        const uint32_t d0 = tmem_base + acc * C::kAccCols;
#pragma unroll
        for (int j = 0; j < C::kUB; ++j) {
          if (j < it.len) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_i8_ts(d0 + j * BN, a0 + 32 * j + 8 * k, umma_desc_sw128_kmajor(bst + j * C::kBBytes + 32 * k), idesc,
                        k > 0 ? 1u : 0u);
          }
        }
        mma_commit(&xempty[s]);
        mma_commit(&aempty[as]);
        mma_commit(&tfull[acc]);
      }
      __syncwarp();
    }
    rt.flush(1);
  } else if (warp >= C::kExpWarp0 && warp < C::kExpWarp0 + 4 * C::kExpGroups) {
    // ------------------------------------------ a4: expansion warps ----
    const int q = warp & 3;
    const int row = 32 * q + lane;  // weight row of the tile = TMEM lane
    const int grp = (warp - C::kExpWarp0) >> 2;
    const int tid = threadIdx.x - 32 * C::kExpWarp0 - 128 * grp;
    RoleTimer rt(g_cta_times_on && blockIdx.x + 1 == g_cta_times_on && warp == C::kExpWarp0 && lane == 0);
    int i = 0;
    for (It it(u0, u1, nb, sched.n_tiles); it.valid(); it.next(nb), ++i) {
      if (C::kExpGroups > 1 && (i % C::kExpGroups) != grp) continue;
      const int ws = i % C::kWStages, s = i % C::kXStages;
      const uint32_t wst = sbase + ws * C::kWStageBytes;
      const uint32_t st = sbase + C::kXBase + s * C::kXStageBytes;
      const int as = i % C::kASlots;
      const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + C::kAOff + 32 * C::kUB * as;
      rt.wait(&wfull[ws], (i / C::kWStages) & 1, 0);
      trace(rt.on, 2, i);
#pragma unroll
      for (int j = 0; j < C::kUB; ++j) {
        if (j < it.len) {
          // own weight row of block j: 4 x 16 B, 64B-swizzled (chunk c at c ^ ((row >> 1) & 3))
          uint32_t e[32];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 w = lds128(wst + j * C::kWPBytes + row * 64 + ((c ^ ((row >> 1) & 3)) << 4));
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t tt = ww[k] & 0x0F0F0F0Fu;
              e[8 * c + 2 * k] = tt << 4;         // 16*e0..3
              e[8 * c + 2 * k + 1] = ww[k] - tt;  // 16*e4..7
            }
          }
          if (j == 0) {
            rt.wait(&aempty[as], ((i / C::kASlots) & 1) ^ 1, 1);  // MMA of unit i - kASlots done
            tc_fence_after();
          }
          tmem_st_32x32b_x32(ta + 32 * j, e);
        }
      }
      // packed weights consumed into registers: release the weight stage now
      __syncwarp();
      if (lane == 0) mbar_arrive(&wempty[ws]);
      mbar_wait(&xfull[s], (i / C::kXStages) & 1);
      bool any4 = false;
#pragma unroll
      for (int j = 0; j < C::kUB; ++j) {
        if (j < it.len && !(map.code[it.b + j] >> 15)) {
          any4 = true;
          const uint32_t xp = st + C::kXPOff + j * C::kXPBytes;
          const uint32_t xb = st + j * C::kBBytes;
          for (int tk = tid; tk < BN * 4; tk += 128) {
            const int r = tk >> 2, jj = tk & 3;
            const uint4 w = lds128(xp + r * 64 + jj * 16);
            uint4 o0, o1;
            uint32_t tt;
            tt = w.x & 0x0F0F0F0Fu; o0.x = tt << 4; o0.y = w.x - tt;
            tt = w.y & 0x0F0F0F0Fu; o0.z = tt << 4; o0.w = w.y - tt;
            tt = w.z & 0x0F0F0F0Fu; o1.x = tt << 4; o1.y = w.z - tt;
            tt = w.w & 0x0F0F0F0Fu; o1.z = tt << 4; o1.w = w.w - tt;
            sts128(xb + r * 128 + (((2 * jj) ^ (r & 7)) << 4), o0);
            sts128(xb + r * 128 + (((2 * jj + 1) ^ (r & 7)) << 4), o1);
          }
        }
      }
      if (any4) fence_proxy_async_smem();
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&expd[s]);
      trace(rt.on, 3, i);
    }
    rt.flush(2);
  } else if (warp >= C::kEpiWarp0 && warp < C::kEpiWarp0 + C::kEpiWarps) {
    // ----------------------------------------- a6-a8: epilogue warps ----
    const int q = warp & 3;
    const int h = (warp - C::kEpiWarp0) >> 2;  // column group
    const int row = 32 * q + lane;
    const int col0 = h * C::kCW;
    const uint32_t tl = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)col0;
    // running sums as packed fp32 pairs (FFMA2 / FMUL2: half the issue slots)
    uint64_t y2[C::kCW / 2];
#pragma unroll
    for (int j = 0; j < C::kCW / 2; ++j) y2[j] = 0ull;
    int seg_first = u0 % nb;  // first block of the current segment
    RoleTimer rt(g_cta_times_on && blockIdx.x + 1 == g_cta_times_on && warp == C::kEpiWarp0 && lane == 0);
    int i = 0;
    for (It it(u0, u1, nb, sched.n_tiles); it.valid(); it.next(nb), ++i) {
      const int acc = i % C::kAcc;
      const int a = i % C::kScaleSlots;
      const uint32_t slot = scale_base + a * C::kSlotBytes;
      const int t = it.t;
      const int n0 = it.tn * 128, m0 = it.tm * BN;
      const int n = n0 + row;
      trace(rt.on, 8, i);
      if (!kAccOut) rt.wait(&sfull[a], (i / C::kScaleSlots) & 1, 0);
      trace(rt.on, 9, i);
      rt.wait(&tfull[acc], (i / C::kAcc) & 1, 1);
      trace(rt.on, 5, i);
      tc_fence_after();
      // one block's chunk of kChunk accumulator columns [c, c + kChunk)
      auto consume = [&](int jb, int c, const uint32_t* r) {
        const int b = it.b + jb;
        const bool is8 = (map.code[b] >> 15) != 0;
        if (kAccOut) {
          const int sh = is8 ? 4 : 8;
#pragma unroll
          for (int j = 0; j < C::kChunk; ++j) {
            const int m = m0 + col0 + c + j;
            if (m < args.M) args.Acc[((int64_t)b * args.M + m) * args.N + n] = ((int32_t)r[j]) >> sh;
          }
        } else {
          float swv = kGroupK ? 1.f : lds_f32(slot + C::kSxBytes + jb * 512 + row * 4);
          swv *= is8 ? 0.0625f : 0.00390625f;  // fold 16^-e
          const uint64_t sw2 = pack2(swv, swv);
#pragma unroll
          for (int j4 = 0; j4 < C::kChunk; j4 += 4) {
            // y[m] += float(acc[m]) * (sx[m] * swv), two columns per instruction
            uint64_t sx01, sx23;
            lds_u64x2(slot + jb * BN * 4 + (col0 + c + j4) * 4, sx01, sx23);
            cvt_fma2(y2[(c + j4) / 2], r[j4 + 0], r[j4 + 1], mul2_u(sx01, sw2));
            cvt_fma2(y2[(c + j4) / 2 + 1], r[j4 + 2], r[j4 + 3], mul2_u(sx23, sw2));
          }
        }
      };
      if constexpr (C::kCW <= 32) {
        // kLdG blocks' accumulators (<= 32 registers) in flight before one wait
#pragma unroll
        for (int jb0 = 0; jb0 < C::kUB; jb0 += C::kLdG) {
          if (jb0 < it.len) {
            uint32_t r[C::kLdG][C::kCW];
#pragma unroll
            for (int g = 0; g < C::kLdG; ++g)
              if (jb0 + g < it.len) {
#pragma unroll
                for (int c = 0; c < C::kCW; c += C::kChunk)
                  tmem_ld_n<C::kChunk>(tl + acc * C::kAccCols + (jb0 + g) * BN + c,
                                       *reinterpret_cast<uint32_t(*)[C::kChunk]>(&r[g][c]));
              }
            tmem_ld_wait();
#pragma unroll
            for (int g = 0; g < C::kLdG; ++g)
              if (jb0 + g < it.len) {
#pragma unroll
                for (int c = 0; c < C::kCW; c += C::kChunk) consume(jb0 + g, c, &r[g][c]);
              }
          }
        }
      } else {
#pragma unroll
        for (int jb = 0; jb < C::kUB; ++jb)
          if (jb < it.len) {
#pragma unroll
            for (int c = 0; c < C::kCW; c += C::kChunk) {
              uint32_t r[C::kChunk];
              tmem_ld_n<C::kChunk>(tl + acc * C::kAccCols + jb * BN + c, r);
              tmem_ld_wait();
              consume(jb, c, r);
            }
          }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      trace(rt.on, 6, i);

      const bool tile_end = (it.b + it.len == nb);
      const bool seg_end = tile_end || (it.u + it.len == u1);
      if (!kAccOut && seg_end) {
        float y[C::kCW];
#pragma unroll
        for (int j = 0; j < C::kCW / 2; ++j) {
          const float2 f = unpack2(y2[j]);
          y[2 * j] = f.x;
          y[2 * j + 1] = f.y;
        }
        if (kGroupK) {
          const float swr = lds_f32(slot + C::kSxBytes + row * 4);
#pragma unroll
          for (int j = 0; j < C::kCW; ++j) y[j] *= swr;
        }
        if (seg_first == 0 && tile_end) {
          // whole tile in this CTA: direct write-back
#pragma unroll
          for (int j = 0; j < C::kCW; ++j) {
            const int m = m0 + col0 + j;
            if (m < args.M) {
              const __half hv = __float2half_rn(y[j]);
              args.Y[(int64_t)m * args.ldy + n] = hv;
              for (int i = 0; i < args.npeer; ++i) args.Ypeer[i][(int64_t)m * args.ldy + n] = hv;  // f1
            }
          }
        } else {
          // ------------------------- a7: stream-K partial + fixup ----
          const unsigned long long tf = rt.now();
          // slot (cta, 0) = partial of the first tile of this CTA, (cta, 1) = last;
          // layout [row][BN]: this thread's kCW columns are contiguous
          const int which = (seg_first == (u0 % nb) && t == u0 / nb) ? 0 : 1;
          float* part = args.ws_partial + ((int64_t)blockIdx.x * 2 + which) * (128 * BN) + row * BN + col0;
#pragma unroll
          for (int j = 0; j < C::kCW; j += 4)
            __stcg(reinterpret_cast<float4*>(part + j), make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]));
          // contributors of tile t: CTAs whose block range intersects [t*nb, (t+1)*nb)
          const int tu0 = t * nb, tu1 = tu0 + nb;
          int c_lo = (int)(((uint32_t)tu0 * (uint32_t)sched.ctas) / (uint32_t)sched.units);
          while (c_lo > 0 && sched.u_begin(c_lo) > tu0) --c_lo;
          while (sched.u_begin(c_lo + 1) <= tu0) ++c_lo;
          int c_hi = (int)(((uint32_t)(tu1 - 1) * (uint32_t)sched.ctas) / (uint32_t)sched.units);
          while (c_hi > 0 && sched.u_begin(c_hi) > tu1 - 1) --c_hi;
          while (sched.u_begin(c_hi + 1) <= tu1 - 1) ++c_hi;
          // the epilogue threads' partial stores are ordered before thread 0's
          // gpu-scope fence by the named barrier (release is cumulative); the
          // last arriver's fence after the atomic orders the reads below
          epi_sync(32 * C::kEpiWarps);
          if (threadIdx.x == 32 * C::kEpiWarp0) {
            __threadfence();
            const int prev = atomicAdd(args.ws_counter + t, 1);
            const bool last = (prev == c_hi - c_lo);
            if (last) __threadfence();
            *s_flag = last;
          }
          epi_sync(32 * C::kEpiWarps);
          if (*s_flag) {
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
              if (m < args.M) {
                const __half hv = __float2half_rn(y[j]);
                args.Y[(int64_t)m * args.ldy + n] = hv;
                for (int i = 0; i < args.npeer; ++i) args.Ypeer[i][(int64_t)m * args.ldy + n] = hv;  // f1
              }
            }
            if (threadIdx.x == 32 * C::kEpiWarp0) args.ws_counter[t] = 0;
          }
          rt.add_fixup(tf);
        }
#pragma unroll
        for (int j = 0; j < C::kCW / 2; ++j) y2[j] = 0ull;
      }
      __syncwarp();
      if (!kAccOut && lane == 0) mbar_arrive(&sempty[a]);
      trace(rt.on, 7, i);
      if (seg_end) seg_first = (it.b + it.len == nb) ? 0 : it.b + it.len;
    }
    rt.flush(3);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc<C::kTmemCols>(tmem_base);
  if (threadIdx.x == 0 && g_cta_times_on && blockIdx.x < 1024) g_cta_times[3 * blockIdx.x + 1] = global_ns();
}

}  // namespace comet
