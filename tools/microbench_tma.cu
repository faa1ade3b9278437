// microbench_tma.cu -- TMA-only streaming rate per box shape (tools only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_tma tools/microbench_tma.cu
// One CTA per SM, one thread issuing loads into a kStages ring of 8 KB
// buffers; every load is waited for and the slot reused.  Reports GB/s over
// the whole GPU for: (a) 2-D box 64 B x 128 rows (row stride = ld),
// (b) 2-D box 128 B x 64 rows, (c) 2-D box 256 B x 32 rows, (d) 1-D bulk 8 KB.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2410_12168_b200/csrc/sm100.cuh"

using namespace comet;

constexpr int kStages = 16;
constexpr int kBuf = 8192;

template <int MODE>
__global__ void __launch_bounds__(32, 1) tma_stream(const __grid_constant__ CUtensorMap tm, const uint8_t* base,
                                                    int units_per_cta, int box_cols, int box_rows, long long rows_total) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[kStages];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const uint64_t pol = l2_policy_evict_first();
  for (int i = 0; i < units_per_cta + kStages; ++i) {
    if (i >= kStages) mbar_wait(&bar[i % kStages], ((i / kStages) - 1) & 1);
    if (i < units_per_cta) {
      const int s = i % kStages;
      const long long u = (long long)blockIdx.x * units_per_cta + i;
      mbar_arrive_expect_tx(&bar[s], kBuf);
      if (MODE == 3) {
        bulk_load(smem + s * kBuf, base + u * kBuf, kBuf, &bar[s]);
      } else {
        // unit u -> (row tile, column block) with the column block fastest
        const long long cols_blocks = 4096 / box_cols;
        const int cb = (int)(u % cols_blocks);
        const long long rt = (u / cols_blocks) % (rows_total / box_rows);
        tma_load_2d_hint(smem + s * kBuf, &tm, &bar[s], cb * box_cols, (int)(rt * box_rows), pol);
      }
    }
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long long ld = 4096;  // bytes per row (K = 8192 packed)
  const long long rows = 57344;
  const size_t bytes = ld * rows;  // 235 MB
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)fp;
  const int units_per_cta = (int)(bytes / kBuf / 148);
  int shapes[3][2] = {{64, 128}, {128, 64}, {256, 32}};
  CUtensorMapSwizzle swz[3] = {CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_SWIZZLE_NONE};
  cudaFuncSetAttribute(tma_stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kBuf + 1024);
  cudaFuncSetAttribute(tma_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kBuf + 1024);
  cudaFuncSetAttribute(tma_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kBuf + 1024);
  cudaFuncSetAttribute(tma_stream<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kBuf + 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 4; ++mode) {
    CUtensorMap tm;
    int bc = 64, br = 128;
    if (mode < 3) {
      bc = shapes[mode][0];
      br = shapes[mode][1];
      cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)ld};
      cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
      cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       swz[mode], CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) printf("encode failed %d\n", r);
    }
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      switch (mode) {
        case 0: tma_stream<0><<<148, 32, kStages * kBuf + 1024>>>(tm, buf, units_per_cta, bc, br, rows); break;
        case 1: tma_stream<1><<<148, 32, kStages * kBuf + 1024>>>(tm, buf, units_per_cta, bc, br, rows); break;
        case 2: tma_stream<2><<<148, 32, kStages * kBuf + 1024>>>(tm, buf, units_per_cta, bc, br, rows); break;
        case 3: tma_stream<3><<<148, 32, kStages * kBuf + 1024>>>(tm, buf, units_per_cta, bc, br, rows); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const double moved = (double)units_per_cta * 148 * kBuf;
    const char* names[4] = {"2-D box 64B x 128 rows", "2-D box 128B x 64 rows", "2-D box 256B x 32 rows", "1-D bulk 8 KB"};
    printf("%-26s %8.1f GB/s  (%s)\n", names[mode], moved / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
