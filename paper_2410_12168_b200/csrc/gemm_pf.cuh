// gemm_pf.cuh -- prefill W4Ax GEMM (M > 128 tokens) on CTA pairs
// (tcgen05 cta_group::2), persistent over pair tiles, tokens as the TMEM A
// operand.
//
// Pair tile: 256 tokens (MMA M; 128 TMEM lanes in each CTA) x 192 weight rows
// (each CTA stages 96 of them in smem).  K is walked one 128-channel FMPQ
// block at a time; each block is one MMA item of 4 x
// tcgen05.mma.cta_group::2.kind::i8 (M=256, N=192, K=32) into one of two
// 192-column INT32 accumulators, so the promotion of block b overlaps the MMAs
// of block b+1 (the paper's overlap of conversion and MMA, P:L255-259,
// re-cut for TMEM).  TMEM: 2 x 192 accumulator + 4 x 32 A-slot columns.
//
// Roles per CTA (20 warps = 640 threads, 96 registers; lower warp ids first):
//   warps 0 / 2 (a3 producers): weights -- 1-D bulk copies of the CTA's 96
//       packed rows (tiled layout, 64B swizzle baked in) -- and tokens -- a
//       TMA of the block's token slab (INT8 [128 x 128 B] SW128, INT4
//       [128 x 64 B] SW64) plus 1-D copies of the scales; a 5-deep load ring;
//   warp 1 of the leader (a5): waits the block's `ready` and the accumulator's
//       `tempty`, issues the 4 MMAs, commits to both CTAs (warp 3 idles);
//   warps 4-7 (a4 staging; thread = token row of the warp's TMEM lane
//       quarter): the row's token block -- zero-extended INT4 (x16) or
//       raw INT8 -- goes from smem through registers into the block's TMEM A
//       slot (tcgen05.st), and 3 chunks of the packed weight rows are
//       zero-extended into the SW128 K-major B operand; a 4-deep operand ring;
//   warps 8-19 (a6, a8; thread = token row, 64 columns): double-buffered
//       8-column tcgen05.ld, I2F + fma.rn.f32x2 with the thread-uniform row
//       scale; per-channel weight scales once per tile; at the tile's last
//       block fp16 RNE -> smem -> TMA tensor stores.
// Compile-time switches (DESIGN.md section 7 lists what each measured):
// COMET_PF_XPRE (pre-expanded INT4 tokens, SS MMA), COMET_PF_TILEN /
// COMET_PF_ACCS / COMET_PF_PQ (tile shape), COMET_PF_EXP (timing skeletons).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "gemm.cuh"
#include "gemm_2sm.cuh"
#include "quantize.cuh"
#include "sm100.cuh"

namespace comet {

// leader CTA only: D[tmem, both CTAs] (+)= A[tmem, both] . B[smem, both]^T
DEVI void mma_i8_ts_2sm(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

#ifndef COMET_TRACE_EV2
#define COMET_TRACE_EV2 0  // trace builds: events 6/9/10 = token-staging sub-steps instead of MMA/producer
#endif
constexpr bool kTraceEv2 = COMET_TRACE_EV2;

#ifndef COMET_PF_MAGIC
#define COMET_PF_MAGIC 0  // 1: magic-biased accumulators (below; measured 1.6x slower: register spills + refill latency)
#endif
// Magic-biased accumulators (SURVEY 7.3-1 iii): the promotion warps refill
// each accumulator with the bit pattern 0x4B400000 (= 1.5*2^23 as fp32) right
// after reading it, and the MMAs accumulate onto it (enable_input_d = 1 from
// the first K step), so the INT32 result a (|a| < 2^21 for both block kinds)
// arrives as the fp32 value 1.5*2^23 + a: one exact FADD2 converts two
// columns (vs two I2F on the half-rate ALU pipe) -- bit-identical results.
constexpr bool kPfMagic = COMET_PF_MAGIC;

#ifndef COMET_PF_SLEEP
#define COMET_PF_SLEEP 0  // waits that suspend: 1 producer, 2 MMA issuer, 4 staging warps
#endif
template <int kSleep>
DEVI void pf_wait(uint64_t* bar, uint32_t parity) {
  if (kSleep) mbar_wait_sleep(bar, parity); else mbar_wait(bar, parity);
}
#ifndef COMET_PF_CLUSTER_ACQ
#define COMET_PF_CLUSTER_ACQ 0
#endif
// the MMA issuer's waits on barriers the partner CTA arrives on remotely.
// acquire.cta suffices: what they publish is read by the tensor core (smem
// operands after fence.proxy.async, TMEM after tcgen05.fence), not by generic
// loads; an acquire.cluster wait compiles to an L1 invalidation (CCTL.IVALL)
// per completed wait, on the MMA issue path
template <int kSleep>
DEVI void pf_wait_cluster(uint64_t* bar, uint32_t parity) {
  if (COMET_PF_CLUSTER_ACQ) {
    if (kSleep) mbar_wait_cluster_sleep(bar, parity); else mbar_wait_cluster(bar, parity);
  } else {
    if (kSleep) mbar_wait_sleep(bar, parity); else mbar_wait(bar, parity);
  }
}

#ifndef COMET_PF_EXP
#define COMET_PF_EXP 0  // timing experiments only (wrong results): 1 = skip staging work, 2 = skip promotion math, 3 = both, 4 = also skip the accumulator loads, 5 = also skip the operand loads
#endif

#ifndef COMET_PF_SXCHAIN
#define COMET_PF_SXCHAIN 1  // scales complete on the load-ring barrier (no scale barrier wait in the promotion)
#endif
#ifndef COMET_PF_XPRE
#define COMET_PF_XPRE 0
#endif
#ifndef COMET_PF_LDPIPE
#define COMET_PF_LDPIPE 1  // double-buffered 8-column accumulator loads in the promotion
#endif

struct PfCfg {
#ifndef COMET_PF_TILEN
#define COMET_PF_TILEN 192
#endif
  static constexpr int kTileN = COMET_PF_TILEN;  // weight rows per pair tile
  static constexpr int kRows = kTileN / 2;    // weight rows per CTA
#ifndef COMET_PF_ITEMS
#define COMET_PF_ITEMS 1
#endif
  static constexpr int kItems = COMET_PF_ITEMS;  // MMA items per block (1: N=192; 2: N=96 halves)
  static constexpr int kItemN = kTileN / kItems;  // MMA N of one item (kItemN/2 rows from each CTA)
#ifndef COMET_PF_PQ
#define COMET_PF_PQ 3  // measured: 2 (16 warps) -7%, 4 (24 warps, 80 regs) -12%, 6 -22%
#endif
  static constexpr int kPQ = COMET_PF_PQ;         // promotion warps per TMEM lane quarter
  static constexpr int kPWarps = 4 * kPQ;         // promotion warps (0 .. kPWarps - 1)
  static constexpr int kWCols = kItemN / kPQ;     // item columns per promotion warp
#ifndef COMET_PF_LSTAGES
#define COMET_PF_LSTAGES 5
#endif
#ifndef COMET_PF_STAGES
#define COMET_PF_STAGES 4
#endif
  static constexpr int kStages = COMET_PF_STAGES;    // operand stages: SW128 B + TMEM A slot (freed by the MMA)
  static constexpr int kLStages = COMET_PF_LSTAGES;  // load stages: packed weights + raw tokens (freed by staging)
#ifndef COMET_PF_ACCS
#define COMET_PF_ACCS (COMET_PF_ITEMS == 1 ? 2 : 4)
#endif
  static constexpr int kAccs = COMET_PF_ACCS;  // kItemN-column accumulators
  static constexpr int kScaleSlots = 8;
  static constexpr int kWPBytes = kRows * 64;   // packed weights
  static constexpr int kWEBytes = kRows * 128;  // expanded weights, SW128 K-major
  // XPRE: the INT4 token blocks arrive pre-expanded to INT8 (x16, same byte
  // order the staging warps produce) and every token block is TMA-loaded
  // straight into a SW128 smem A stage of the operand ring (SS MMA); the
  // staging warps then only expand weights
  static constexpr bool kXPre = COMET_PF_XPRE;
  static constexpr int kXStageBytes = kXPre ? 0 : 128 * 128;  // INT8 [128 x 128] or packed INT4 [128 x 64]
  static constexpr int kAStageBytes = kXPre ? 128 * 128 : 0;  // token A operand stage (SS MMA)
  static constexpr int kABase = kStages * kWEBytes;
  static constexpr int kWPBase = kABase + kStages * kAStageBytes;
  static constexpr int kXBase = kWPBase + kLStages * kWPBytes;
  static constexpr int kScaleBase = kXBase + kLStages * kXStageBytes;
  static constexpr int kSwOff = 512;                             // sx[128] then sw[192]
  static constexpr int kSlotBytes = kSwOff + kTileN * 4;
  static constexpr int kYBoxBytes = 32 * 16 * 2;                 // 32 rows x 16 fp16
  static constexpr int kYBase = kScaleBase + kScaleSlots * kSlotBytes;
  static constexpr int kYBoxes = kItems * kWCols / 16;           // 32 x 16 output boxes per promotion warp
  static constexpr int kBarBase = kYBase + kPWarps * kYBoxes * kYBoxBytes;
  static constexpr int kBarBytes = 512;
  static constexpr int kFacBase = kBarBase + kBarBytes;  // float fac[nb]: 1/16 (INT8 block) or 1/256 (INT4)
  static constexpr int kSmemBytes = kFacBase + 512 * 4 + 1024;
  static_assert(kWEBytes % 1024 == 0 && kXBase % 1024 == 0 && kWPBase % 512 == 0, "operand alignment");
  static_assert(kScaleBase % 16 == 0 && kYBase % 128 == 0, "alignment");
  static_assert(kSmemBytes <= 227 * 1024, "smem budget");
  static constexpr int kAccCols = kItemN;
  static constexpr int kAOff = kAccs * kAccCols;  // TMEM A slots after the accumulators
  static_assert(kAOff + 32 * kStages <= 512, "TMEM budget");
#ifndef COMET_PF_ROLES_FIRST
#define COMET_PF_ROLES_FIRST 1  // measured neutral (+-0.5%)
#endif
  // warp order = scheduling priority among the warps of an SMSP (lower ids
  // win when several are ready): the latency-critical role warps (producers,
  // MMA issuer) and the staging warps first, the promotion warps last
  static constexpr int kRoleBase = COMET_PF_ROLES_FIRST ? 0 : kPWarps + 4;  // 4 role warps
  static constexpr int kStageWarp = COMET_PF_ROLES_FIRST ? 4 : kPWarps;     // 4 staging warps
  static constexpr int kPBase = COMET_PF_ROLES_FIRST ? 8 : 0;               // promotion warps
  static constexpr int kLoadWarp = kRoleBase;        // weights
  static constexpr int kMmaWarp = kRoleBase + 1;
#ifndef COMET_PF_XWARP
#define COMET_PF_XWARP 6  // 7: token producer on the 4th SMSP (measured neutral)
#endif
  static constexpr int kLoad2Warp = kRoleBase + COMET_PF_XWARP - 4;  // tokens + scales (the 4th warp idles)
  static constexpr int kThreads = 32 * (kPWarps + 8);
  static constexpr int kReadyCount = 2 * 4;  // both CTAs' staging warps
  static constexpr int kTemptyCount = 2 * kPWarps;   // both CTAs' promotion warps
};

struct PfSched {
  int m_tiles, tiles, clusters;
  DEVI void coords(int t, int& m0, int& n0) const {
    const int mt = t % m_tiles;  // token tiles fastest: concurrent clusters share weight tiles
    m0 = mt * 256;
    n0 = (t / m_tiles) * PfCfg::kTileN;
  }
};

// tile-relative weight column of item column j of item h: the first half of
// an item's columns are CTA0's weight rows, the second half CTA1's
__host__ __device__ constexpr int pf_col(int h, int j) {
  return PfCfg::kItems == 1 ? j
                            : (j < PfCfg::kItemN / 2 ? PfCfg::kItemN / 2 * h + j
                                                     : PfCfg::kRows + PfCfg::kItemN / 2 * h + j - PfCfg::kItemN / 2);
}

// kXW: the weights come pre-expanded (INT8 = 16 x INT4, comet_expand_weight)
// and are TMA-loaded straight into the B stage; the staging warps then only
// expand tokens (comet_w4ax_gemm_ex)
template <bool kGroupK, bool kAccOut, bool kXW = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PfCfg::kThreads, 1)
    w4ax_gemm_pf_kernel(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmX4,
                        const __grid_constant__ CUtensorMap tmX8, const __grid_constant__ CUtensorMap tmWE,
                        const __grid_constant__ BlockMap map, GemmArgs args, PfSched sched) {
  using C = PfCfg;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t scale_base = sbase + C::kScaleBase;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarBase);
  uint64_t* lfull = bars;                        // [kLStages] packed weights + tokens landed (tx)
  uint64_t* lempty = lfull + C::kLStages;        // [kLStages] 4 staging warps have read them
  uint64_t* mdone = lempty + C::kLStages;        // [kStages] MMAs of the block done (commit multicast)
  uint64_t* ready = mdone + C::kStages;          // [kStages] leader: operands of the block staged
  uint64_t* tfull = ready + C::kStages;        // [kAccs] item's MMAs done (commit multicast)
  uint64_t* tempty = tfull + C::kAccs;           // [kAccs] leader: 2 CTAs x 12 promotion warps
  uint64_t* sfull = tempty + C::kAccs;           // [kScaleSlots] scales landed (tx)
  uint64_t* sempty = sfull + C::kScaleSlots;     // [kScaleSlots] 12 promotion warps
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sempty + C::kScaleSlots);

  // warp index via shfl from lane 0: ptxas then treats it (and everything
  // derived from it) as warp-uniform
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
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
      mbar_init(&lempty[l], 4);
    }
    for (int a = 0; a < C::kAccs; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], C::kTemptyCount);
    }
    for (int a = 0; a < C::kScaleSlots; ++a) {
      mbar_init(&sfull[a], 1);
      mbar_init(&sempty[a], C::kPWarps);
    }
    fence_mbar_init();
  }
  // per-block activation-scale factor (the x16 / x256 of the expanded operands)
  for (int i = threadIdx.x; i < nb; i += C::kThreads)
    reinterpret_cast<float*>(smem + C::kFacBase)[i] = (map.code[i] >> 15) ? 0.0625f : 0.00390625f;
  if (warp == C::kLoadWarp && lane == 0) {
    if (!kAccOut) tma_prefetch_desc(&tmY);
    tma_prefetch_desc(&tmX4);
    tma_prefetch_desc(&tmX8);
  }
  if (warp == C::kMmaWarp) tmem_alloc_2sm<512>(tmem_holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // debug trace of one CTA (COMET_TRACE builds; tools/gemm_sweep.py trace3)
  const bool tr_cta = kTraceBuild && g_cta_times_on && blockIdx.x + 1 == g_cta_times_on;
  const bool tr_pair = kTraceBuild && g_cta_times_on && (blockIdx.x >> 1) == ((g_cta_times_on - 1) >> 1);

  // (setmaxnreg rebalancing does not help here: ptxas compiles every role to
  // the launch budget of 96 registers, and 24+ warps drop it to 80)
  if (warp >= C::kRoleBase && warp < C::kRoleBase + 4) {
  if (warp == C::kLoadWarp || warp == C::kLoad2Warp) {
    // ------------------- a3: producers (weights | tokens + scales) ----
    // two warps: each TMA / bulk-copy issue costs the issuing thread ~10^2
    // cycles, and one thread issuing all of a block's copies was the rate limit
    const bool wrole = warp == C::kLoadWarp;
    // PDL: both producers wait for the preceding kernel before their first
    // load (the planes, scales and possibly the weights come from it); the
    // prologue above (barrier init, TMEM allocation, descriptor prefetch)
    // already overlapped it.  (An L2 prefetch of the first weight blocks
    // before the wait, as in the decode kernel, measured slower here.)
    int pg = 0, pt = cluster, pb = 0, pm0 = 0, pn0 = 0;
    sched.coords(pt, pm0, pn0);
    __syncwarp();
    grid_dep_wait();
    for (; pg < steps;) {
      const int g = pg, b = pb;
      const int l = g % C::kLStages;
      const int a = g & (C::kScaleSlots - 1);
      // load stage l is free once the staging warps have read block g - kLStages
      // (decoupled from the MMA: loads run ahead of the tensor core by the
      // load ring plus the operand ring)
      // (the producer, MMA and staging warps run ahead of the promotion: their
      // waits suspend instead of polling, leaving issue slots to the promotion)
      pf_wait<COMET_PF_SLEEP & 1>(&lempty[l], ((g / C::kLStages) & 1) ^ 1);
      // XPRE: the tokens land in operand stage g % kStages, free once the MMAs
      // of block g - kStages are done
      if ((C::kXPre && !wrole) || (kXW && wrole))
        pf_wait<COMET_PF_SLEEP & 1>(&mdone[g % C::kStages], ((g / C::kStages) & 1) ^ 1);
      if (elect_one()) trace(tr_cta, wrole ? 14 : 15, g);
      if (!kAccOut && !wrole) pf_wait<COMET_PF_SLEEP & 1>(&sempty[a], ((g / C::kScaleSlots) & 1) ^ 1);
      const uint32_t code = map.code[b];
      const bool is8 = (code >> 15) != 0;
      const int rank = code & 0x7FFF;
      const int my_m0 = pm0 + 128 * (int)crank;
      if (elect_one()) {
        if (wrole && kXW) {
          // pre-expanded weights: one SW128 box of the CTA's kRows rows x 128 B
          // straight into operand stage g % kStages (rows past N zero-filled)
          const int R = pn0 + C::kRows * (int)crank;
          mbar_arrive_expect_tx(&lfull[l], C::kRows * 128);
          tma_load_2d(smem + (g % C::kStages) * C::kWEBytes, &tmWE, &lfull[l], b * 128, R);
        } else if (wrole) {
          // this CTA's weight rows [R, R + v) of the tile (v < 96 at the right
          // edge of N); in the tiled layout they are contiguous within each
          // 128-row slab
          const int R = pn0 + C::kRows * (int)crank;
          const int v = max(0, min(C::kRows, args.N - R));
          mbar_arrive_expect_tx(&lfull[l], COMET_PF_EXP == 5 ? 0 : v * 64);
          uint8_t* dst = smem + C::kWPBase + l * C::kWPBytes;
          int r = R, left = COMET_PF_EXP == 5 ? 0 : v;
          while (left > 0) {
            const int in_slab = min(left, 128 - (r & 127));
            bulk_load(dst, args.Wq + ((int64_t)(r >> 7) * nb + b) * 8192 + (r & 127) * 64, in_slab * 64, &lfull[l]);
            dst += in_slab * 64;
            r += in_slab;
            left -= in_slab;
          }
        } else {
          const int nsx = kAccOut ? 0 : max(0, min(128, (int)args.ldsx - my_m0));  // multiple of 4
          const bool load_sw = !kGroupK || b == nb - 1;
          const int nsw = (kAccOut || !load_sw) ? 0 : max(0, min(C::kTileN, args.N - pn0));  // multiple of 64
          // COMET_PF_SXCHAIN: the scales complete on the load-ring barrier with
          // the tokens; the promotion reads them after the block's tfull, which
          // follows lfull through staging -> ready -> MMA -> commit
          mbar_arrive_expect_tx(&lfull[l], (COMET_PF_EXP >= 5 ? 0 : (is8 || C::kXPre ? 128 * 128 : 128 * 64)) +
                                               (COMET_PF_SXCHAIN ? (nsx + nsw) * 4 : 0));
          uint8_t* xs = C::kXPre ? smem + C::kABase + (g % C::kStages) * C::kAStageBytes
                                 : smem + C::kXBase + l * C::kXStageBytes;
          if (COMET_PF_EXP >= 5) {  // 5: no operand loads, 6: no token loads
          } else if (is8)
            tma_load_2d(xs, &tmX8, &lfull[l], rank * 128, my_m0);
          else
            tma_load_2d(xs, &tmX4, &lfull[l], rank * (C::kXPre ? 128 : 64), my_m0);
          if (!kAccOut) {
            uint64_t* sb = COMET_PF_SXCHAIN ? &lfull[l] : &sfull[a];
            if (!COMET_PF_SXCHAIN) mbar_arrive_expect_tx(&sfull[a], (nsx + nsw) * 4);
            uint8_t* slot = smem + C::kScaleBase + a * C::kSlotBytes;
            if (nsx) bulk_load(slot, args.Sx + (int64_t)b * args.ldsx + my_m0, nsx * 4, sb);
            if (nsw) bulk_load(slot + C::kSwOff, args.Sw + (kGroupK ? 0 : (int64_t)b * args.N) + pn0, nsw * 4, sb);
          }
        }
        trace(!kTraceEv2 && tr_cta, 9, g);
      }
      __syncwarp();
      ++pg;
      if (++pb == nb) {
        pb = 0;
        pt += sched.clusters;
        if (pt < sched.tiles) sched.coords(pt, pm0, pn0);
      }
    }

  } else if (warp == C::kMmaWarp) {
    // --------------------------------------------- a5: MMA (leader) ----
    // a5: MMA items (two N=96 items per block), issued in order when the
    // block is staged and the item's accumulator is free (never blocks)
    constexpr uint32_t idesc = idesc_i8(256, C::kItemN);
    for (int i = 0; i < C::kItems * steps && crank == 0; ++i) {
      const int g = i / C::kItems, h = i % C::kItems;
      const int s = g % C::kStages, acc = i % C::kAccs;
      if (h == 0) pf_wait_cluster<COMET_PF_SLEEP & 2>(&ready[s], (g / C::kStages) & 1);
      if (!kTraceEv2 && C::kItems == 1 && elect_one()) trace(tr_cta, 6, g);
      // magic mode: use k of an accumulator waits for its k-th refill (the
      // promotion warps' initial fill is completion 0)
      pf_wait_cluster<COMET_PF_SLEEP & 2>(&tempty[acc], ((i / C::kAccs) & 1) ^ (kPfMagic ? 0 : 1));
      if (C::kItems == 1 && elect_one()) trace(tr_cta, 8, g);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a_tm = tmem_base + C::kAOff + 32 * s;
        const uint32_t bst = sbase + s * C::kWEBytes;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (C::kXPre)
            mma_i8_ss_2sm(tmem_base + acc * C::kAccCols,
                          umma_desc_sw128_kmajor(sbase + C::kABase + s * C::kAStageBytes + 32 * k),
                          umma_desc_sw128_kmajor(bst + h * (C::kRows / C::kItems) * 128 + 32 * k), idesc,
                          (kPfMagic || k > 0) ? 1u : 0u);
          else
            mma_i8_ts_2sm(tmem_base + acc * C::kAccCols, a_tm + 8 * k,
                          umma_desc_sw128_kmajor(bst + h * (C::kRows / C::kItems) * 128 + 32 * k), idesc,
                          (kPfMagic || k > 0) ? 1u : 0u);
          if (k == 0 && g < 32) trace(tr_cta, 4, 32 + g);
        }
        if (g < 32) trace(tr_cta, 5, 32 + g);
        mma_commit_2sm(&tfull[acc], 0x3);
        if (h == C::kItems - 1) mma_commit_2sm(&mdone[s], 0x3);
        trace(tr_cta, 7 + h, g);
      }
      __syncwarp();
    }
  }  // warp 19: idle
  } else if (warp >= C::kStageWarp && warp < C::kStageWarp + 4) {
    // ---- a4 staging (thread = token row of lane quarter q) ----
    // (XPRE: the tokens arrive expanded in smem; only the weights are staged)
    constexpr bool do_tok = !C::kXPre, do_w = !kXW;
    const int q = warp & 3;
    const int et = (int)threadIdx.x - 32 * C::kStageWarp;  // weight-expanding thread 0..127
    const uint32_t tst = tmem_base + ((uint32_t)(32 * q) << 16) + C::kAOff;
    const uint32_t leader_ready = mapa_shared(smem_u32(ready), 0);
    int sb = 0;
    for (int j = 0; j < steps; ++j) {
      // ---- a4: stage block j: load stage l -> operand stage s ----
      const int l = j % C::kLStages, s = j % C::kStages;
      const bool is8 = (map.code[sb] >> 15) != 0;
      if (++sb == nb) sb = 0;
      const uint32_t xs = sbase + C::kXBase + l * C::kXStageBytes;
      const uint32_t wps = sbase + C::kWPBase + l * C::kWPBytes;
      const uint32_t wst = sbase + s * C::kWEBytes;
      pf_wait<COMET_PF_SLEEP & 4>(&lfull[l], (j / C::kLStages) & 1);
      trace(tr_cta && threadIdx.x == 32 * C::kStageWarp, 12, j);
      // operand stage s (smem B + TMEM A slot) is free once the MMAs of block
      // j - kStages are done
      pf_wait<COMET_PF_SLEEP & 4>(&mdone[s], ((j / C::kStages) & 1) ^ 1);
      trace(tr_cta && threadIdx.x == 32 * C::kStageWarp, 10, j);
      tc_fence_after();
      if (COMET_PF_EXP != 1 && COMET_PF_EXP < 3) {
      // all shared-memory loads of the block first (the loads and stores are
      // volatile asm, kept in program order: interleaving them would expose
      // one load latency per chunk)
      const uint32_t r_ = (32 * q) + (opaque(threadIdx.x) & 31);  // this thread's token row
      uint4 tv[8];
      if (!do_tok) {
      } else if (is8) {
#pragma unroll
        for (int c = 0; c < 8; ++c) tv[c] = lds128(xs + r_ * 128 + ((c ^ (r_ & 7)) << 4));
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) tv[c] = lds128(xs + r_ * 64 + ((c ^ ((r_ >> 1) & 3)) << 4));
      }
      uint4 wv[C::kRows * 4 / 128];
#pragma unroll
      for (int k = 0; k < C::kRows * 4 / 128 && do_w; ++k) {
        const int ch = et + 128 * k;
        const int er = ch >> 2, ej = ch & 3;
        wv[k] = lds128(wps + er * 64 + ((ej ^ ((er >> 1) & 3)) << 4));
      }
      if (kTraceBuild) {  // the LDS results have landed
        uint32_t dep = tv[0].x ^ tv[3].w;
        if (do_w) dep ^= wv[0].x ^ wv[C::kRows * 4 / 128 - 1].w;
        trace(tr_cta && threadIdx.x == 32 * C::kStageWarp && dep != 0x9e3779b9u, 16, j);
      }
      // tokens: 4 chunks of 32 K = 32 TMEM A columns (INT8 raw, INT4 x16)
      if (do_tok) {
        uint32_t e[32];
        if (is8) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            e[4 * c] = tv[c].x; e[4 * c + 1] = tv[c].y; e[4 * c + 2] = tv[c].z; e[4 * c + 3] = tv[c].w;
          }
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            zext_word(tv[c].x, e[8 * c + 0], e[8 * c + 1]);
            zext_word(tv[c].y, e[8 * c + 2], e[8 * c + 3]);
            zext_word(tv[c].z, e[8 * c + 4], e[8 * c + 5]);
            zext_word(tv[c].w, e[8 * c + 6], e[8 * c + 7]);
          }
        }
        if (kTraceBuild) {  // after the zero-extension (its inputs: the LDS results)
          uint32_t dep = 0;
#pragma unroll
          for (int x = 0; x < 32; ++x) dep ^= e[x];
          trace(tr_cta && threadIdx.x == 32 * C::kStageWarp && dep != 0x9e3779b9u, 13, j);
        }
        tmem_st_32x32b_x32(tst + 32 * s, e);
      }
      trace(kTraceEv2 && tr_cta && threadIdx.x == 32 * C::kStageWarp, 6, j);
      // weights: chunks et, et + 128, et + 256 of the packed slab -> SW128 B operand
#pragma unroll
      for (int k = 0; k < C::kRows * 4 / 128 && do_w; ++k) {
        const int ch = et + 128 * k;
        const int er = ch >> 2, ej = ch & 3;
        expand_chunk(wv[k], wst + er * 128 + (((2 * ej) ^ (er & 7)) << 4), wst + er * 128 + (((2 * ej + 1) ^ (er & 7)) << 4));
      }
      }
      // the load stage may be refilled once every lane's loads have landed
      // (the tcgen05.st / st.shared above consumed them; an arrive right after
      // the LDS instructions could overtake them)
      __syncwarp();
      if (lane == 0) mbar_arrive(&lempty[l]);
      trace(kTraceEv2 && tr_cta && threadIdx.x == 32 * C::kStageWarp, 9, j);
      fence_proxy_async_smem();
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_ready + s * 8);
      trace(tr_cta && threadIdx.x == 32 * C::kStageWarp, 1, j);
    }
  } else {

    // ----------------------- warps 8-19: a6 promotion + a8 write-back ----
    const int q = warp & 3;         // TMEM lane quarter
    const int kw = (warp - C::kPBase) >> 2;  // 0..kPQ-1: item columns [kWCols kw, kWCols (kw + 1)) of every item
    const int row = 32 * q + lane;  // token row within this CTA
    const uint32_t tl = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(C::kWCols * kw);
    const uint32_t leader_tempty = mapa_shared(smem_u32(tempty), 0);

    constexpr int kWC = C::kWCols;  // this warp's columns of an item
    uint64_t y[C::kItems * kWC / 2];  // [item h][kWC / 2 pairs]: columns kWC kw + 2p (+1) of item h
#pragma unroll
    for (int j = 0; j < C::kItems * kWC / 2; ++j) y[j] = 0;
    int t = cluster, b = 0;
    // this row's activation scale of block g (x 16^-e_g), fetched one block
    // ahead so its barrier wait and load latency overlap the promotion
    auto fetch_sx = [&](int g, int bb) -> float {
      if (kAccOut || COMET_PF_SXCHAIN || g >= steps) return 0.f;
      const int a = g & (C::kScaleSlots - 1);
      mbar_wait(&sfull[a], (g / C::kScaleSlots) & 1);
      const bool is8 = (map.code[bb] >> 15) != 0;
      return lds_f32(scale_base + a * C::kSlotBytes + row * 4) * (is8 ? 0.0625f : 0.00390625f);
    };
    float sx_next = fetch_sx(0, 0);
    if (kPfMagic) {
      // initial fill of this warp's 32 columns of every accumulator
#pragma unroll
      for (int acc = 0; acc < C::kAccs; ++acc) tmem_fill_32x32b_x32(tl + acc * C::kAccCols, kAccMagic);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        for (int acc = 0; acc < C::kAccs; ++acc) mbar_arrive_cluster(leader_tempty + acc * 8);
    }
    for (int g = 0; g < steps; ++g) {
      trace(tr_cta && threadIdx.x == 32 * C::kPBase, 0, g);
      const int a = g & (C::kScaleSlots - 1);
      const uint32_t slot = scale_base + a * C::kSlotBytes;
      const bool is8 = (map.code[b] >> 15) != 0;
      // (without COMET_PF_SXCHAIN) next block's scale, issued now: its barrier
      // wait and shared load overlap this block's promotion
      uint64_t sx2 = pack2(sx_next, sx_next);
      if (!COMET_PF_SXCHAIN) sx_next = fetch_sx(g + 1, b + 1 == nb ? 0 : b + 1);
      trace(tr_cta && threadIdx.x == 32 * C::kPBase, 11, g);
#pragma unroll
      for (int h = 0; h < C::kItems; ++h) {
        const int i = C::kItems * g + h;
        const int acc = i % C::kAccs;
        pf_wait<COMET_PF_SLEEP & 8>(&tfull[acc], (i / C::kAccs) & 1);
        trace(tr_cta && threadIdx.x == 32 * C::kPBase, 2 + 2 * h, g);
        tc_fence_after();
        if (COMET_PF_SXCHAIN && !kAccOut && h == 0) {
          const float sxv = lds_f32(slot + row * 4) * lds_f32(sbase + C::kFacBase + 4 * b);
          sx2 = pack2(sxv, sxv);
        }
        const uint32_t ta = tl + acc * C::kAccCols;
        if (kAccOut) {
          int m0, n0;
          sched.coords(t, m0, n0);
          const int sh = is8 ? 4 : 8;
          const int m = m0 + 128 * (int)crank + row;
#pragma unroll
          for (int u = 0; u < kWC / 16; ++u) {
            uint32_t r[16];
            tmem_ld_32x32b_x16(ta + 16 * u, r);
            tmem_ld_wait();
            if (kPfMagic && (u & 1)) tmem_fill_32x32b_x32(ta + 16 * (u - 1), kAccMagic);
            if (m < args.M) {
              const int nu = n0 + pf_col(h, kWC * kw + 16 * u);
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (nu + j < args.N)
                  args.Acc[((int64_t)b * args.M + m) * args.N + nu + j] =
                      ((int32_t)(r[j] - (kPfMagic ? kAccMagic : 0u))) >> sh;
            }
          }
        } else if (COMET_PF_LDPIPE && !kPfMagic && COMET_PF_EXP == 0) {
          // 8-column chunks, double-buffered: the load of chunk c + 1 is in
          // flight while chunk c is promoted, so the accumulator's hold time
          // is the load stream, not loads + math; released after the last load
          auto promote8 = [&](int c, const uint32_t (&r)[8]) {
            uint64_t* yy = &y[(kWC / 2) * h + 4 * c];
            if (kGroupK) {
#pragma unroll
              for (int j = 0; j < 4; ++j) cvt_fma2(yy[j], r[2 * j], r[2 * j + 1], sx2);
            } else {
              const uint32_t swa = slot + C::kSwOff + pf_col(h, kWC * kw + 8 * c) * 4;
#pragma unroll
              for (int j4 = 0; j4 < 2; ++j4) {
                const float4 w4 = lds_f32x4(swa + 16 * j4);
                cvt_fma2(yy[2 * j4], r[4 * j4], r[4 * j4 + 1], mul2_u(sx2, pack2(w4.x, w4.y)));
                cvt_fma2(yy[2 * j4 + 1], r[4 * j4 + 2], r[4 * j4 + 3], mul2_u(sx2, pack2(w4.z, w4.w)));
              }
            }
          };
          constexpr int kC = kWC / 8;
          uint32_t ra[8], rb[8];
          tmem_ld_32x32b_x8(ta, ra);
          tmem_ld_wait_dep(ra);
#pragma unroll
          for (int c = 0; c < kC; c += 2) {
            tmem_ld_32x32b_x8(ta + 8 * (c + 1), rb);
            promote8(c, ra);
            tmem_ld_wait_dep(rb);
            if (c + 2 < kC) {
              tmem_ld_32x32b_x8(ta + 8 * (c + 2), ra);
            } else {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(leader_tempty + acc * 8);
              // per-warp release times of steps 10 and 11, both CTAs of the traced pair
              if (C::kItems == 1 && (g == 10 || g == 11)) trace(tr_pair && lane == 0, g - 6, warp - C::kPBase + 16 * (int)crank);
            }
            promote8(c + 1, rb);
            if (c + 2 < kC) tmem_ld_wait_dep(ra);
          }
        } else {
          // 16 columns per tcgen05.ld (the running sums leave room for 16);
          // the accumulator is released as soon as its last load has landed
#pragma unroll
          for (int c2 = 0; c2 < kWC / 16; ++c2) {
            uint32_t r[16];
            if (COMET_PF_EXP >= 4) {
              r[0] = c2;
            } else {
              tmem_ld_32x32b_x16(ta + 16 * c2, r);
              tmem_ld_wait();
            }
            if (kPfMagic && (c2 & 1)) tmem_fill_32x32b_x32(ta + 16 * (c2 - 1), kAccMagic);
            if (c2 == kWC / 16 - 1) {
              if (kPfMagic) tmem_st_wait();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(leader_tempty + acc * 8);
            }
            if (COMET_PF_EXP >= 2) {
              if (r[0] == 0x12345678u) y[0] += 1;  // keep the loads alive
              continue;
            }
#pragma unroll
            for (int c1 = 0; c1 < 2; ++c1) {  // 8-column chunks of this warp's 32 columns
              const int c = 2 * c2 + c1;
              uint64_t* yy = &y[(kWC / 2) * h + 4 * c];
              if (kGroupK) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  if (kPfMagic)
                    magic_fma2(yy[j], r[8 * c1 + 2 * j], r[8 * c1 + 2 * j + 1], sx2);
                  else
                    cvt_fma2(yy[j], r[8 * c1 + 2 * j], r[8 * c1 + 2 * j + 1], sx2);
                }
              } else {
                // group 128: this block's weight scales of the chunk's 8 columns
                const uint32_t swa = slot + C::kSwOff + pf_col(h, kWC * kw + 8 * c) * 4;
#pragma unroll
                for (int j4 = 0; j4 < 2; ++j4) {
                  const float4 w4 = lds_f32x4(swa + 16 * j4);
                  const uint64_t s01 = mul2_u(sx2, pack2(w4.x, w4.y)), s23 = mul2_u(sx2, pack2(w4.z, w4.w));
                  if (kPfMagic) {
                    magic_fma2(yy[2 * j4], r[8 * c1 + 4 * j4], r[8 * c1 + 4 * j4 + 1], s01);
                    magic_fma2(yy[2 * j4 + 1], r[8 * c1 + 4 * j4 + 2], r[8 * c1 + 4 * j4 + 3], s23);
                  } else {
                    cvt_fma2(yy[2 * j4], r[8 * c1 + 4 * j4], r[8 * c1 + 4 * j4 + 1], s01);
                    cvt_fma2(yy[2 * j4 + 1], r[8 * c1 + 4 * j4 + 2], r[8 * c1 + 4 * j4 + 3], s23);
                  }
                }
              }
            }
          }
        }
        if (kAccOut) {
          if (kPfMagic) tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(leader_tempty + acc * 8);
        }
        trace(tr_cta && threadIdx.x == 32 * C::kPBase, 3 + 2 * h, g);
      }

      if (++b == nb) {
        // -------------------------------------------- a8: tile write-back ----
        if (!kAccOut) {
          int m0, n0;
          sched.coords(t, m0, n0);
          const int mw = m0 + 128 * (int)crank + 32 * q;  // first row of this warp's boxes
          const uint32_t ybuf = opaque(sbase + C::kYBase + (warp - C::kPBase) * C::kYBoxes * C::kYBoxBytes);
          if (lane == 0) bulk_wait_group_read0();  // previous tile's stores have left smem
          __syncwarp();
#pragma unroll
          for (int bx = 0; bx < C::kYBoxes; ++bx) {  // box = (item h, unit u): 32 rows x 16 columns
            const int h = bx / (kWC / 16), u = bx % (kWC / 16);
            const uint32_t swa = slot + C::kSwOff + pf_col(h, kWC * kw + 16 * u) * 4;
            uint32_t hw[8];
#pragma unroll
            for (int p4 = 0; p4 < 4; ++p4) {
              uint64_t v0 = y[(kWC / 2) * h + 8 * u + 2 * p4], v1 = y[(kWC / 2) * h + 8 * u + 2 * p4 + 1];
              if (kGroupK) {  // per-channel weight scales, once per tile
                const float4 w4 = lds_f32x4(swa + 16 * p4);
                v0 = mul2_u(v0, pack2(w4.x, w4.y));
                v1 = mul2_u(v1, pack2(w4.z, w4.w));
              }
              __half2 h0 = __float22half2_rn(unpack2(v0));
              __half2 h1 = __float22half2_rn(unpack2(v1));
              hw[2 * p4] = *reinterpret_cast<uint32_t*>(&h0);
              hw[2 * p4 + 1] = *reinterpret_cast<uint32_t*>(&h1);
              y[(kWC / 2) * h + 8 * u + 2 * p4] = 0;
              y[(kWC / 2) * h + 8 * u + 2 * p4 + 1] = 0;
            }
            const uint32_t dst = ybuf + bx * C::kYBoxBytes + (opaque(threadIdx.x) & 31) * 32;
            sts128(dst, make_uint4(hw[0], hw[1], hw[2], hw[3]));
            sts128(dst + 16, make_uint4(hw[4], hw[5], hw[6], hw[7]));
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int bx = 0; bx < C::kYBoxes; ++bx) {
              const int nglob = n0 + pf_col(bx / (kWC / 16), kWC * kw + 16 * (bx % (kWC / 16)));
              if (nglob < args.N) tma_store_2d(&tmY, ybuf + bx * C::kYBoxBytes, nglob, mw);
            }
            bulk_commit_group();
          }
        }
        b = 0;
        t += sched.clusters;
      }
      __syncwarp();
      if (!kAccOut && lane == 0) mbar_arrive(&sempty[a]);
    }
  }

  if (!kAccOut && warp >= C::kPBase && warp < C::kPBase + C::kPWarps && lane == 0) bulk_wait_group0();  // output stores complete
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc_2sm<512>(tmem_base);
}

// XPRE: INT4 token plane [M x n4*64 B] -> INT8 x16 [M x n4*128 B], each
// 4-byte word w -> (w & 0x0F0F0F0F) << 4 | (w & 0xF0F0F0F0) << 32 (the byte
// order the staging warps write into the A operand)
__global__ void __launch_bounds__(256) expand_int4_tokens_kernel(const uint4* __restrict__ in,
                                                                 uint4* __restrict__ out, int64_t n16) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = __ldg(in + i);
    uint4 o0, o1;
    zext_word(w.x, o0.x, o0.y);
    zext_word(w.y, o0.z, o0.w);
    zext_word(w.z, o1.x, o1.y);
    zext_word(w.w, o1.z, o1.w);
    out[2 * i] = o0;
    out[2 * i + 1] = o1;
  }
}

// comet_expand_weight: tiled packed weights -> row-major INT8 We [N x K],
// We[n, k] = 16 * wq[n, k] (the zero-extension of P:L294 done once, offline;
// the nibble order makes lo/hi of each word elements 0-3 / 4-7)
__global__ void __launch_bounds__(256) expand_weights_kernel(const uint8_t* __restrict__ Wq, int N, int K,
                                                             uint4* __restrict__ out) {
  const int nb = K / 128, cpr = K / 32;  // 16-B packed chunks per row
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)N * cpr) return;
  const int64_t n = i / cpr;
  const int c = (int)(i % cpr);
  const uint4 w = *reinterpret_cast<const uint4*>(Wq + wq_tiled_offset(n, (int64_t)c * 16, nb));
  uint4 o0, o1;
  zext_word(w.x, o0.x, o0.y);
  zext_word(w.y, o0.z, o0.w);
  zext_word(w.z, o1.x, o1.y);
  zext_word(w.w, o1.z, o1.w);
  out[2 * i] = o0;
  out[2 * i + 1] = o1;
}

}  // namespace comet
