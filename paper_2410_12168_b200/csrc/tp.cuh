// tp.cuh -- the reassembly step of the N-sharded tensor-parallel layer
// (BJ north_star "NCCL all-gather over NVLink is used only to
// reassemble Y"): all_gather_into_tensor leaves the ranks' Y shards
// rank-major, Yall [P x M x per]; the layer's output is Y [M x N] with
// Y[m, r*per + j] = Yall[r, m, j] (columns >= N, the padding of the last
// shard, dropped).  HBM-bound copy, 16-byte vectors (per, N multiples of 128).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "sm100.cuh"

namespace comet {

__global__ void __launch_bounds__(256) gather_shards_kernel(const uint4* __restrict__ Yall, int P, int M, int per,
                                                            int N, uint4* __restrict__ Y, int64_t ldy) {
  grid_dep_wait();
  const int vpr = per / 8;  // 16-byte vectors per shard row
  const int64_t total = (int64_t)P * M * vpr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(i % vpr);
    const int64_t rm = i / vpr;
    const int m = (int)(rm % M), r = (int)(rm / M);
    const int n = r * per + 8 * v;
    if (n < N) Y[((int64_t)m * ldy + n) / 8] = __ldcs(Yall + i);
  }
}

}  // namespace comet
