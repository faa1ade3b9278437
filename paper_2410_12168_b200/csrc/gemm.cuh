// gemm.cuh -- a3..a8: the W4Ax GEMM on sm_100a (§4, §5).
//
// Tile: 128 weight rows (MMA M, = TMEM lanes) x BN tokens (MMA N, = TMEM
// columns), K walked one 128-channel FMPQ block at a time ("a block
// usually contains multiple tiles").  Per block:
//   a3  warp 0 (1 lane): TMA the packed weight slab [128 x 64 B] and either
//       the INT8 activation slab [BN x 128 B] straight into the MMA operand
//       buffer (128B swizzle) or the packed INT4 slab [BN x 64 B].
//   a4  warps 4-7: INT4 -> INT8 zero-extension in shared memory, two word
//       ops per 8 values ((w<<4)&0xF0F0F0F0, w&0xF0F0F0F0 = 16*q),
//       written in the UMMA K-major SWIZZLE_128B layout.
//   a5  warp 1 (1 lane): 4 x tcgen05.mma.kind::i8 (K=32 each) into a fresh
//       INT32 TMEM accumulator (two accumulators ping-pong across blocks).
//   a6  warps 8-15: tcgen05.ld the INT32 block result, promote
//       y += (sx[m,b] * sw[n,g(b)] * 16^-e_b) * acc'  in fp32 registers
//       (the x16 / x256 zero-extension factor folded into the scale,
//       "divide by 16 in the scaling parameter").
//   a7  split-K over the block range when tiles < SMs ("tile decomposition",
//       P:L316-317); partial fp32 tiles combined in a fixed split order by
//       the last-arriving CTA (deterministic; one inter-CTA sync before the
//       write-back).
//   a8  fp32 -> fp16 RNE store of Y.
// Pipelines: smem ring {full (TMA tx), expd (expansion done), empty (MMA
// done, tcgen05.commit)} x STAGES, TMEM ring {tfull (commit), tempty
// (epilogue drained)} x 2.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "quantize.cuh"
#include "sm100.cuh"

namespace comet {

struct GemmArgs {
  int M, N, K, nb;
  int64_t ldsx, ldy;
  const float* Sx;
  const float* Sw;
  int group_blocks;  // 128-blocks per weight-scale group: 1 (group 128) or nb (group K)
  __half* Y;
  int32_t* Acc;  // debug output (kAccOut)
  float* ws_partial;
  int* ws_counter;
  int splits;
};

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN >= 128 ? 4 : 6;
  static constexpr int kABytes = 128 * 128;  // expanded weights, SW128 K-major
  static constexpr int kBBytes = BN * 128;   // activations int8, SW128 K-major
  static constexpr int kWPBytes = 128 * 64;  // packed weights
  static constexpr int kXPBytes = BN * 64;   // packed INT4 activations
  static constexpr int kStageBytes = kABytes + kBBytes + kWPBytes + kXPBytes;
  static constexpr int kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int kCW = BN / 2;  // columns per epilogue warp
  static constexpr int kChunk = kCW >= 32 ? 32 : kCW;
  static constexpr int kThreads = 512;
};

DEVI uint32_t expand_lo(uint32_t w) { return (w << 4) & 0xF0F0F0F0u; }
DEVI uint32_t expand_hi(uint32_t w) { return w & 0xF0F0F0F0u; }

// Expand `rows` rows of packed INT4 (64 B/row) at `src` into int8 rows of
// 128 B at `dst` in the SWIZZLE_128B K-major layout (16-B chunk c of row r
// stored at chunk c ^ (r & 7)).  tid in [0, 128).
DEVI void expand_rows(const uint8_t* src, uint8_t* dst, int rows, int tid) {
  for (int t = tid; t < rows * 4; t += 128) {
    const int r = t >> 2, j = t & 3;
    const uint4 w = *reinterpret_cast<const uint4*>(src + r * 64 + j * 16);
    const uint4 o0 = make_uint4(expand_lo(w.x), expand_hi(w.x), expand_lo(w.y), expand_hi(w.y));
    const uint4 o1 = make_uint4(expand_lo(w.z), expand_hi(w.z), expand_lo(w.w), expand_hi(w.w));
    uint8_t* row = dst + r * 128;
    *reinterpret_cast<uint4*>(row + (((2 * j) ^ (r & 7)) << 4)) = o0;
    *reinterpret_cast<uint4*>(row + (((2 * j + 1) ^ (r & 7)) << 4)) = o1;
  }
}

template <int N>
DEVI void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[N]);
template <>
DEVI void tmem_ld_cols<32>(uint32_t taddr, uint32_t (&r)[32]) { tmem_ld_32x32b_x32(taddr, r); }
template <>
DEVI void tmem_ld_cols<16>(uint32_t taddr, uint32_t (&r)[16]) { tmem_ld_32x32b_x16(taddr, r); }
template <>
DEVI void tmem_ld_cols<8>(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

DEVI void epi_bar_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <int BN, bool kAccOut>
__global__ void __launch_bounds__(512, 1)
    w4ax_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX4,
                     const __grid_constant__ CUtensorMap tmX8, const __grid_constant__ BlockMap map, GemmArgs args) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* full = bars;
  uint64_t* expd = bars + C::kStages;
  uint64_t* empty = bars + 2 * C::kStages;
  uint64_t* tfull = bars + 3 * C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_flag = reinterpret_cast<int*>(tmem_holder + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 128;
  const int m0 = blockIdx.y * BN;
  const int split = blockIdx.z;
  const int kb0 = (int)(((int64_t)args.nb * split) / args.splits);
  const int kb1 = (int)(((int64_t)args.nb * (split + 1)) / args.splits);
  const int nkb = kb1 - kb0;

  auto a_buf = [&](int s) { return smem + s * C::kStageBytes; };
  auto b_buf = [&](int s) { return smem + s * C::kStageBytes + C::kABytes; };
  auto wp_buf = [&](int s) { return smem + s * C::kStageBytes + C::kABytes + C::kBBytes; };
  auto xp_buf = [&](int s) { return smem + s * C::kStageBytes + C::kABytes + C::kBBytes + C::kWPBytes; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&expd[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
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

  if (warp == 0) {
    // ------------------------------------------------ a3: TMA producer ----
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::kStages;
        const uint32_t ph = (i / C::kStages) & 1;
        const int kb = kb0 + i;
        const uint32_t code = map.code[kb];
        const bool is8 = (code >> 15) != 0;
        const int rank = code & 0x7FFF;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], C::kWPBytes + (is8 ? C::kBBytes : C::kXPBytes));
        tma_load_2d(wp_buf(s), &tmW, &full[s], kb * 64, n0);
        if (is8)
          tma_load_2d(b_buf(s), &tmX8, &full[s], rank * 128, m0);
        else
          tma_load_2d(xp_buf(s), &tmX4, &full[s], rank * 64, m0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------- a5: MMA issuer ----
    constexpr uint32_t idesc = idesc_i8(128, BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::kStages;
      const uint32_t ph = (i / C::kStages) & 1;
      const int acc = i & 1;
      const uint32_t aph = (i >> 1) & 1;
      mbar_wait(&tempty[acc], aph ^ 1);
      mbar_wait(&expd[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a_addr = smem_u32(a_buf(s));
        const uint32_t b_addr = smem_u32(b_buf(s));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          mma_i8_ss(tmem_base + acc * BN, umma_desc_sw128_kmajor(a_addr + 32 * k),
                    umma_desc_sw128_kmajor(b_addr + 32 * k), idesc, k > 0 ? 1u : 0u);
        }
        mma_commit(&empty[s]);
        mma_commit(&tfull[acc]);
      }
      __syncwarp();
    }
  } else if (warp >= 4 && warp < 8) {
    // -------------------------------------- a4: INT4 -> INT8 expansion ----
    const int tid = threadIdx.x - 128;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::kStages;
      const uint32_t ph = (i / C::kStages) & 1;
      const bool is8 = (map.code[kb0 + i] >> 15) != 0;
      mbar_wait(&full[s], ph);
      expand_rows(wp_buf(s), a_buf(s), 128, tid);
      if (!is8) expand_rows(xp_buf(s), b_buf(s), BN, tid);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&expd[s]);
    }
  } else if (warp >= 8) {
    // ------------------------------------------ a6: promotion epilogue ----
    const int q = warp & 3;              // TMEM lane quarter (warp % 4)
    const int h = (warp - 8) >> 2;       // column half
    const int row = 32 * q + lane;       // weight row within the tile
    const int n = n0 + row;
    const int col0 = h * C::kCW;         // first token column of this warp
    float y[C::kCW];
#pragma unroll
    for (int j = 0; j < C::kCW; ++j) y[j] = 0.0f;

    for (int i = 0; i < nkb; ++i) {
      const int kb = kb0 + i;
      const int acc = i & 1;
      const uint32_t aph = (i >> 1) & 1;
      const bool is8 = (map.code[kb] >> 15) != 0;
      float sw = 0.0f;
      if (!kAccOut) {
        sw = __ldg(args.Sw + (int64_t)(kb / args.group_blocks) * args.N + n);
        sw *= is8 ? 0.0625f : 0.00390625f;  // fold 16^-e (exact power of two)
      }
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < C::kCW; c += C::kChunk) {
        uint32_t r[C::kChunk];
        const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * BN + col0 + c);
        tmem_ld_cols<C::kChunk>(taddr, r);
        tmem_ld_wait();
        if (kAccOut) {
          const int sh = is8 ? 4 : 8;
#pragma unroll
          for (int j = 0; j < C::kChunk; ++j) {
            const int m = m0 + col0 + c + j;
            if (m < args.M) args.Acc[((int64_t)kb * args.M + m) * args.N + n] = ((int32_t)r[j]) >> sh;
          }
        } else {
          const float* sxp = args.Sx + (int64_t)kb * args.ldsx + m0 + col0 + c;
#pragma unroll
          for (int j4 = 0; j4 < C::kChunk; j4 += 4) {
            float4 sx4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (m0 + col0 + c + j4 < args.ldsx) sx4 = __ldg(reinterpret_cast<const float4*>(sxp + j4));
            y[c + j4 + 0] = fmaf((float)(int32_t)r[j4 + 0], sx4.x * sw, y[c + j4 + 0]);
            y[c + j4 + 1] = fmaf((float)(int32_t)r[j4 + 1], sx4.y * sw, y[c + j4 + 1]);
            y[c + j4 + 2] = fmaf((float)(int32_t)r[j4 + 2], sx4.z * sw, y[c + j4 + 2]);
            y[c + j4 + 3] = fmaf((float)(int32_t)r[j4 + 3], sx4.w * sw, y[c + j4 + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }

    if (!kAccOut) {
      if (args.splits == 1) {
#pragma unroll
        for (int j = 0; j < C::kCW; ++j) {
          const int m = m0 + col0 + j;
          if (m < args.M) args.Y[(int64_t)m * args.ldy + n] = __float2half_rn(y[j]);
        }
      } else {
        // ---------------------------- a7: deterministic split-K fixup ----
        const int tile = blockIdx.y * gridDim.x + blockIdx.x;
        float* part = args.ws_partial + ((int64_t)tile * args.splits) * (BN * 128);
#pragma unroll
        for (int j = 0; j < C::kCW; ++j) part[(int64_t)split * (BN * 128) + (col0 + j) * 128 + row] = y[j];
        __threadfence();
        epi_bar_sync();
        if (threadIdx.x == 256) {
          const int prev = atomicAdd(args.ws_counter + tile, 1);
          *s_flag = (prev == args.splits - 1);
        }
        epi_bar_sync();
        if (*s_flag) {
          __threadfence();
#pragma unroll
          for (int j = 0; j < C::kCW; ++j) {
            const int m = m0 + col0 + j;
            float t = 0.0f;
            for (int sp = 0; sp < args.splits; ++sp) t += __ldcg(part + (int64_t)sp * (BN * 128) + (col0 + j) * 128 + row);
            if (m < args.M) args.Y[(int64_t)m * args.ldy + n] = __float2half_rn(t);
          }
          if (threadIdx.x == 256) args.ws_counter[tile] = 0;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem_base);
}

}  // namespace comet
