// microbench_l2.cu -- L2 -> shared memory read bandwidth with TMA / bulk copies
// from an L2-resident buffer (tools only; not part of libcomet.so).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_l2 tools/microbench_l2.cu
// One CTA per SM (or two), one elected thread issuing copies into a ring of
// 8 or 16 KB buffers, every copy waited for and the slot reused.  The source
// buffer is `wrap` bytes (L2-resident when << 126 MB).  Reports GB/s over the
// GPU and bytes per SM-clock at the max SM clock.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2410_12168_b200/csrc/sm100.cuh"

using namespace comet;

constexpr int kStages = 12;

template <int MODE, int kBuf>  // 0: 1-D bulk, 1: 2-D SW128 box 128 B x (kBuf/128) rows
__global__ void __launch_bounds__(32, 1) l2_stream(const __grid_constant__ CUtensorMap tm, const uint8_t* base,
                                                   int units_per_cta, long long wrap_units) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[kStages];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  for (int i = 0; i < units_per_cta + kStages; ++i) {
    if (i >= kStages) mbar_wait(&bar[i % kStages], ((i / kStages) - 1) & 1);
    if (i < units_per_cta) {
      const int s = i % kStages;
      const long long u = ((long long)blockIdx.x * 7919 + i) % wrap_units;
      mbar_arrive_expect_tx(&bar[s], kBuf);
      if (MODE == 0)
        bulk_load(smem + s * kBuf, base + u * kBuf, kBuf, &bar[s]);
      else
        tma_load_2d(smem + s * kBuf, &tm, &bar[s], 0, (int)(u * (kBuf / 128)));
    }
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int MODE, int kBuf>
void run(const char* name, uint8_t* buf, size_t wrap, int ctas, EncodeTiledFn enc) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {128, (cuuint64_t)(wrap / 128)};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, (cuuint32_t)(kBuf / 128)};
  cuuint32_t es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  auto k = l2_stream<MODE, kBuf>;
  const int smem = kStages * kBuf + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int units = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    k<<<ctas, 32, smem>>>(tm, buf, units, (long long)(wrap / kBuf));
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double moved = (double)units * ctas * kBuf;
  const double gbs = moved / (best * 1e-3) / 1e9;
  printf("  %-28s wrap %4zu MB ctas %3d  %8.1f GB/s  %6.1f B/SM-clk @1965  (%s)\n", name, wrap >> 20, ctas, gbs,
         gbs * 1e9 / 1.965e9 / 148, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t bytes = 512ull << 20;
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)fp;
  for (size_t wrap : {16ull << 20, 64ull << 20, 512ull << 20}) {
    run<0, 8192>("bulk 8 KB", buf, wrap, 148, enc);
    run<0, 16384>("bulk 16 KB", buf, wrap, 148, enc);
    run<1, 16384>("2-D SW128 128 B x 128 rows", buf, wrap, 148, enc);
    run<1, 16384>("2-D SW128 128 B x 128 rows", buf, wrap, 296, enc);
  }
  return 0;
}
