// microbench_l2mc.cu -- is the ~45 B/SM-clk L2 -> SMEM ceiling a chip-wide L2
// limit or a per-SM ingest limit, and does TMA multicast lift it?
// (tools only; not part of libcomet.so)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_l2mc tools/microbench_l2mc.cu
// Cluster of C CTAs (one per SM); every stage is a 16 KB SW128 box
// (128 B x 128 rows) that lands in every CTA of the cluster: each CTA issues
// 128/C rows of it with .multicast::cluster to all C CTAs.  Stage reuse is
// guarded by an empty barrier that collects one arrival from every CTA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2410_12168_b200/csrc/sm100.cuh"

using namespace comet;

constexpr int kStages = 8;
constexpr int kBuf = 16384;

DEVI void tma_load_2d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t x, int32_t y, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "h"(mask)
      : "memory");
}

template <int C>
__global__ void __launch_bounds__(32, 1) mc_stream(const __grid_constant__ CUtensorMap tm, int units, long long wrap_rows) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kStages], empty[kStages];
  const uint32_t rank = C > 1 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C);
    }
    fence_mbar_init();
  }
  if (C > 1) cluster_sync(); else __syncthreads();
  if (threadIdx.x == 0) {
    const int cl = blockIdx.x / C;
    constexpr int D = kStages - 2;  // loads in flight ahead of consumption
    for (int i = 0; i < units + D; ++i) {
      if (i < units) {
        const int s = i % kStages;
        if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], kBuf);
        const long long row = ((long long)(cl * 7919 + i) * 128) % wrap_rows;
        if (C == 1)
          tma_load_2d(smem + s * kBuf, &tm, &full[s], 0, (int)row);
        else
          tma_load_2d_mc(smem + s * kBuf + rank * (kBuf / C), &tm, &full[s], 0, (int)(row + rank * (128 / C)),
                         (uint16_t)((1u << C) - 1));
      }
      const int j = i - D;  // consume: wait for the whole stage here, then release it in every CTA
      if (j >= 0) {
        const int s = j % kStages;
        mbar_wait(&full[s], (j / kStages) & 1);
        if (C == 1) {
          mbar_arrive(&empty[s]);
        } else {
          for (int r = 0; r < C; ++r) mbar_arrive_cluster(mapa_shared(smem_u32(&empty[s]), r));
        }
      }
    }
  }
  if (C > 1) cluster_sync();
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int C>
void run(uint8_t* buf, size_t wrap, int ctas, EncodeTiledFn enc) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {128, (cuuint64_t)(wrap / 128)};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, (cuuint32_t)(128 / C)};
  cuuint32_t es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = kStages * kBuf + 1024;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto k = mc_stream<C>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int units = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, k, tm, units, (long long)(wrap / 128));
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double ingest = (double)units * ctas * kBuf;  // bytes landing in shared memory
  const double secs = best * 1e-3;
  printf("  cluster %d  ctas %3d  wrap %4zu MB: ingest %8.1f GB/s = %5.1f B/SM-clk (per active SM %5.1f), L2 reads %8.1f GB/s  (%s)\n",
         C, ctas, wrap >> 20, ingest / secs / 1e9, ingest / secs / 1.965e9 / 148, ingest / secs / 1.965e9 / ctas,
         ingest / C / secs / 1e9, cudaGetErrorString(cudaGetLastError()));
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
  for (int ctas : {148, 74, 36}) run<1>(buf, 32ull << 20, ctas, enc);
  run<2>(buf, 32ull << 20, 148, enc);
  run<4>(buf, 32ull << 20, 148, enc);
  run<2>(buf, 512ull << 20, 148, enc);
  run<4>(buf, 512ull << 20, 148, enc);
  return 0;
}
