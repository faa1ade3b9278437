// microbench_contend.cu -- does accumulator read-out (tcgen05.ld) or shared-
// memory traffic slow tcgen05.mma? (tools only; not part of libcomet.so)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_contend tools/microbench_contend.cu
// One cluster of 2 CTAs per SM pair, 512 threads. The leader's warp 0 issues
// ITERS MMAs (M=256 across the pair, N=192, K=32, A from TMEM, B from smem)
// into TMEM columns [0, 192), committing every 4 (one "block"); warps 4..15 of
// both CTAs meanwhile run a load: none, tcgen05.ld.32x32b.x8 of columns
// [192, 384) (the other accumulator), or 128-bit shared stores + loads.
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2410_12168_b200/csrc/sm100.cuh"

using namespace comet;

constexpr int ITERS = 4096;
constexpr int kChunk = 4;
constexpr int kDepth = 4;
constexpr int N = 192;

DEVI void mma_ts_2sm(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// kLoad: 0 none, 1 tcgen05.ld x8 (all 12 warps), 2 smem st+ld 128-bit, 3 both
template <int kLoad>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) contend_kernel(long long* cyc, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[kDepth];
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  const uint32_t crank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kDepth; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 128 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc_2sm<512>(&holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = holder;
  float acc = 0.f;
  long long t0 = clock64(), t1 = t0;
  if (warp == 0) {
    if (crank == 0) {
      const uint32_t b_s = smem_u32(smem);
      constexpr uint32_t idesc = idesc_i8(256, N);
      for (int c = 0; c < ITERS / kChunk; ++c) {
        if (c >= kDepth) mbar_wait(&bars[c % kDepth], ((c / kDepth) - 1) & 1);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kChunk; ++k)
            mma_ts_2sm(tmem, tmem + 448 + 8 * k, umma_desc_sw128_kmajor(b_s + 32 * k), idesc, k > 0);
          mma_commit_2sm(&bars[c % kDepth], 0x1);
        }
        __syncwarp();
      }
      for (int c = ITERS / kChunk - kDepth; c < ITERS / kChunk; ++c) mbar_wait(&bars[c % kDepth], (c / kDepth) & 1);
      t1 = clock64();
    }
  } else if (warp >= 4) {
    const int q = warp & 3, kw = (warp - 4) >> 2;  // 3 warps per lane quarter
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16) + 192 + 64 * kw;
    const uint32_t sbuf = smem_u32(smem) + 64 * 1024 + (threadIdx.x - 128) * 16;
    for (int it = 0; it < 3000; ++it) {  // outlasts the MMA loop
      if ((kLoad & 4) && warp < 8) {  // warps 4..7: tcgen05.st x32 into the A region (like the staging warps)
        uint32_t e[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) e[j] = it + j;
        tmem_st_32x32b_x32(tmem + ((uint32_t)(32 * q) << 16) + 384 + 32 * (it & 1), e);
        tmem_st_wait();
        continue;
      }
      if (kLoad & 1) {
        uint32_t r[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          tmem_ld_32x32b_x8(tl + 8 * c, r);
          tmem_ld_wait();
          acc += __int_as_float(r[0] ^ r[7]);
        }
      }
      if (kLoad & 2) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          sts128(sbuf + (c & 1) * 6144, make_uint4(it, c, 0, 0));
          const uint4 v = lds128(sbuf + ((c + 1) & 1) * 6144);
          acc += __int_as_float(v.x);
        }
      }
      if (!kLoad) break;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_2sm<512>(tmem);
  if (threadIdx.x == 0 && crank == 0) cyc[blockIdx.x >> 1] = t1 - t0;
  if (acc == 1.2345f) sink[0] = acc;
}

// latency of one K=128 block (4 MMAs + commit) issued into an idle tensor pipe
template <int kN, bool kTS, int kLd = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) latency_kernel(long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  const uint32_t crank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc_2sm<512>(&holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = holder;
  long long iss = 0, lat = 0;
  if (warp == 0 && crank == 0) {
    const uint32_t a_s = smem_u32(smem) + 32 * 1024, b_s = smem_u32(smem);
    constexpr uint32_t idesc = idesc_i8(256, kN);
    for (int r = 0; r < 64; ++r) {
      long long t0 = clock64(), t1 = t0;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (kTS)
            mma_ts_2sm(tmem, tmem + 448 + 8 * k, umma_desc_sw128_kmajor(b_s + 32 * k), idesc, k > 0);
          else
            mma_i8_ss_2sm(tmem, umma_desc_sw128_kmajor(a_s + 32 * k), umma_desc_sw128_kmajor(b_s + 32 * k), idesc, k > 0);
        }
        mma_commit_2sm(&bar, 0x1);
        t1 = clock64();
      }
      __syncwarp();
      mbar_wait(&bar, r & 1);
      long long t2 = clock64();
      if (r >= 8) { iss += t1 - t0; lat += t2 - t0; }
    }
  } else if (kLd && warp >= 4) {  // concurrent accumulator read-out (x8) / operand stores of other TMEM columns
    const int q = warp & 3, kw = (warp - 4) >> 2;
    float acc = 0.f;
    for (int it = 0; it < 600; ++it) {
      if ((kLd & 2) && warp < 8) {
        uint32_t e[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) e[j] = it + j;
        tmem_st_32x32b_x32(tmem + ((uint32_t)(32 * q) << 16) + 384 + 32 * (it & 1), e);
        tmem_st_wait();
        continue;
      }
      uint32_t rr[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        tmem_ld_32x32b_x8(tmem + ((uint32_t)(32 * q) << 16) + 192 + 64 * kw + 8 * c, rr);
        tmem_ld_wait();
        acc += __int_as_float(rr[0] ^ rr[7]);
      }
    }
    if (acc == 1.2345f) cyc[147] = 1;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_2sm<512>(tmem);
  if (threadIdx.x == 0 && crank == 0) { cyc[2 * (blockIdx.x >> 1)] = iss / 56; cyc[2 * (blockIdx.x >> 1) + 1] = lat / 56; }
}

template <int kN, bool kTS, int kLd = 0>
void run_lat(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  auto k = latency_kernel<kN, kTS, kLd>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<148, 512, 64 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-34s N=%3d issue %5lld cyc, issue->commit arrival %5lld cyc (pair 0; min MMA time %d)  %s\n", name, kN, h[0], h[1],
         4 * kN / 2, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  cudaFree(d);
}

template <int kLoad>
void run(const char* name) {
  long long* d;
  float* s;
  cudaMalloc(&d, 74 * sizeof(long long));
  cudaMalloc(&s, 4);
  auto k = contend_kernel<kLoad>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  k<<<148, 512, 128 * 1024>>>(d, s);
  k<<<148, 512, 128 * 1024>>>(d, s);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[74];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 74; ++i) mx = h[i] > mx ? h[i] : mx;
  const double macs_per_sm = (double)ITERS * 256 * N * 32 / 2;
  printf("%-34s %8.1f MAC/clk/SM  %6.1f cyc per K=128 block  %s\n", name, macs_per_sm / mx, mx / (ITERS / 4),
         e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(s);
}

int main() {
  run_lat<192, true>("latency TS");
  run_lat<192, false>("latency SS");
  run_lat<128, false>("latency SS");
  run_lat<256, false>("latency SS");
  run_lat<64, false>("latency SS");
  run_lat<192, true, 1>("latency TS + 12w ld x8");
  run_lat<192, true, 3>("latency TS + 4w st + 8w ld");
  run_lat<128, false, 1>("latency SS + 12w ld x8");
  run<0>("MMA alone");
  run<1>("MMA + 12 warps tcgen05.ld x8");
  run<2>("MMA + 12 warps smem st/ld 128b");
  run<3>("MMA + both");
  run<4>("MMA + 4 warps tcgen05.st x32");
  run<5>("MMA + st x32 (4w) + ld x8 (8w)");
  run<7>("MMA + st + ld + smem");
  return 0;
}
