// microbench_mma.cu -- tcgen05.mma.cta_group::2.kind::i8 issue rate per shape
// (tools only; not part of libcomet.so).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_mma tools/microbench_mma.cu
// One cluster of 2 CTAs per SM pair; the leader's elected thread issues
// ITERS back-to-back MMAs (M=256 across the pair, N, K=32) into one TMEM
// accumulator, A from shared memory (SS) or from TMEM (TS), with a commit
// every kChunk instructions and a wait when kDepth chunks are in flight.
// Reports MACs per SM-clock (nominal kind::i8 peak: 8192).
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2410_12168_b200/csrc/sm100.cuh"

using namespace comet;

constexpr int ITERS = 4096;
constexpr int kChunk = 8;
constexpr int kDepth = 4;

DEVI void mma_ts_2sm(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

template <int N, bool kTS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_kernel(long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[kDepth];
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  const uint32_t crank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kDepth; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  // operands: zeros are fine for timing (A 128 x 128 B, B N/2 x 128 B, SW128)
  for (int i = threadIdx.x; i < (128 + 128) * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc_2sm<512>(&holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = holder;
  long long t0 = clock64();
  if (warp == 0 && crank == 0) {
    const uint32_t a_s = smem_u32(smem), b_s = a_s + 128 * 128;
    constexpr uint32_t idesc = idesc_i8(256, N);
    for (int c = 0; c < ITERS / kChunk; ++c) {
      if (c >= kDepth) mbar_wait(&bars[c % kDepth], ((c / kDepth) - 1) & 1);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
          if (kTS)
            mma_ts_2sm(tmem, tmem + 256 + 8 * (k & 3), umma_desc_sw128_kmajor(b_s + 32 * (k & 3)), idesc, 1);
          else
            mma_i8_ss_2sm(tmem, umma_desc_sw128_kmajor(a_s + 32 * (k & 3)), umma_desc_sw128_kmajor(b_s + 32 * (k & 3)),
                          idesc, 1);
        }
        mma_commit_2sm(&bars[c % kDepth], 0x1);
      }
      __syncwarp();
    }
    for (int c = ITERS / kChunk - kDepth; c < ITERS / kChunk; ++c) mbar_wait(&bars[c % kDepth], (c / kDepth) & 1);
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_2sm<512>(tmem);
  if (threadIdx.x == 0 && crank == 0) cyc[blockIdx.x >> 1] = t1 - t0;
}

template <int N, bool kTS>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 74 * sizeof(long long));
  auto k = mma_kernel<N, kTS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<148, 128, 64 * 1024>>>(d);
  k<<<148, 128, 64 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[74];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 74; ++i) mx = h[i] > mx ? h[i] : mx;
  const double macs_per_sm = (double)ITERS * 256 * N * 32 / 2;
  printf("%-28s N=%3d  %8.1f MAC/clk/SM  (%.1f cyc/instr)  %s\n", name, N, macs_per_sm / mx, mx / ITERS,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<96, false>("SS cta_group::2 kind::i8");
  run<128, false>("SS cta_group::2 kind::i8");
  run<192, false>("SS cta_group::2 kind::i8");
  run<256, false>("SS cta_group::2 kind::i8");
  run<96, true>("TS cta_group::2 kind::i8");
  run<128, true>("TS cta_group::2 kind::i8");
  run<192, true>("TS cta_group::2 kind::i8");
  run<256, true>("TS cta_group::2 kind::i8");
  return 0;
}
