// gemm.cuh -- definitions shared by the two W4Ax GEMM kernels (§4,
// P:L321 §5):
//   gemm_decode.cuh  M <= 128 tokens: swap-AB, weights as the TMEM A operand,
//                    stream-K over (tile, K-block) units (HBM-bound regime);
//   gemm_2sm.cuh     M > 128 tokens: persistent CTA-pair (cta_group::2) tiles
//                    of 256 tokens x 256 weight rows (tensor-bound regime).
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
  const uint8_t* Wq;  // tiled packed weights: slab (tile, block) at (tile * nb + block) * 8192
  int32_t* Acc;  // debug output (per-block INT32, logical units)
  float* ws_partial;
  int* ws_counter;
  int splits;
};

}  // namespace comet
