// microbench.cu -- per-SM throughput of the instructions the W4Ax promotion
// epilogue is made of (tools only; not part of libcomet.so).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
// Prints ops (or bytes) per SM-clock for: FFMA, FFMA2 (f32x2), FMUL2, FADD2,
// I2FP.F32.S32, IADD3, LOP3, tcgen05.ld.32x32b (TMEM->RF bandwidth).
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2410_12168_b200/csrc/sm100.cuh"

using namespace comet;

constexpr int ITERS = 4096;

// 8 independent dependency chains per thread, one PTX instruction each.
template <int OP>
__global__ void __launch_bounds__(512) alu_kernel(float* out, long long* cyc, float seed) {
  uint32_t v[8];
  unsigned long long w[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    v[j] = __float_as_uint(seed + threadIdx.x * 0.001f + j);
    w[j] = ((unsigned long long)v[j] << 32) | v[j];
  }
  const float c1 = seed * 0.999f, c2 = seed * 1e-3f;
  const unsigned long long c12 = ((unsigned long long)__float_as_uint(c1) << 32) | __float_as_uint(c2);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(v[j]) : "f"(c1), "f"(c2));
      if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(w[j]) : "l"(c12), "l"(c12));
      if (OP == 2) asm volatile("cvt.rn.f32.s32 %0, %0;" : "+r"(v[j]));
      if (OP == 3) asm volatile("add.s32 %0, %0, %1;" : "+r"(v[j]) : "r"(i));
      if (OP == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[j]) : "r"(i), "r"(j));
      if (OP == 5) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(w[j]) : "l"(c12));
      if (OP == 6) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(w[j]) : "l"(c12));
      if (OP == 7) asm volatile("add.rn.f32 %0, %0, %1;" : "+r"(v[j]) : "f"(c1));
      if (OP == 8) asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0f3A83126F;" : "+r"(v[j]));
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += __uint_as_float(v[j]) + __uint_as_float((uint32_t)w[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NWARPS>
__global__ void __launch_bounds__(512) tmem_ld_kernel(float* out, long long* cyc) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t base = holder;
  uint32_t acc = 0;
  long long t0 = clock64();
  if (warp < NWARPS) {
    const uint32_t q = warp & 3;
    for (int i = 0; i < ITERS / 8; ++i) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(base + (q << 16) * 32 + ((i * 32 + (warp >> 2) * 128) & 511), r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += r[j];
    }
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(base);
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NWARPS>
__global__ void __launch_bounds__(512) tmem_st_kernel(float* out, long long* cyc) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t base = holder;
  long long t0 = clock64();
  if (warp < NWARPS) {
    const uint32_t q = warp & 3;
    for (int i = 0; i < ITERS / 8; ++i) {
      tmem_fill_32x32b_x16(base + (q << 16) * 32 + ((i * 16 + (warp >> 2) * 128) & 511), 0x4B400000u + i);
      tmem_fill_32x32b_x16(base + (q << 16) * 32 + ((i * 16 + 16 + (warp >> 2) * 128) & 511), 0x4B400000u + i);
    }
    tmem_st_wait();
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(base);
  out[blockIdx.x * blockDim.x + threadIdx.x] = 0.f;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename F>
void report(const char* name, F launch, double work_per_cta) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  launch(out, cyc);
  cudaDeviceSynchronize();
  launch(out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%-34s %10.1f per SM-clock   (%s)\n", name, work_per_cta / avg, cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  const double lane_ops = 512.0 * ITERS * 8;
  report("FFMA (3-reg) ops", [](float* o, long long* c) { alu_kernel<0><<<148, 512>>>(o, c, 1.0f); }, lane_ops);
  report("FFMA imm ops", [](float* o, long long* c) { alu_kernel<8><<<148, 512>>>(o, c, 1.0f); }, lane_ops);
  report("FFMA2 element-ops (2/lane)", [](float* o, long long* c) { alu_kernel<1><<<148, 512>>>(o, c, 1.0f); }, 2 * lane_ops);
  report("FADD2 element-ops (2/lane)", [](float* o, long long* c) { alu_kernel<5><<<148, 512>>>(o, c, 1.0f); }, 2 * lane_ops);
  report("FMUL2 element-ops (2/lane)", [](float* o, long long* c) { alu_kernel<6><<<148, 512>>>(o, c, 1.0f); }, 2 * lane_ops);
  report("FADD ops", [](float* o, long long* c) { alu_kernel<7><<<148, 512>>>(o, c, 1.0f); }, lane_ops);
  report("I2F (cvt.rn.f32.s32) ops", [](float* o, long long* c) { alu_kernel<2><<<148, 512>>>(o, c, 1.0f); }, lane_ops);
  report("IADD ops", [](float* o, long long* c) { alu_kernel<3><<<148, 512>>>(o, c, 1.0f); }, lane_ops);
  report("LOP3 ops", [](float* o, long long* c) { alu_kernel<4><<<148, 512>>>(o, c, 1.0f); }, lane_ops);
  const double ld_bytes = (ITERS / 8) * 32.0 * 32 * 4;  // per warp
  report("tcgen05.ld B/clk, 4 warps", [](float* o, long long* c) { tmem_ld_kernel<4><<<148, 512>>>(o, c); }, 4 * ld_bytes);
  report("tcgen05.ld B/clk, 8 warps", [](float* o, long long* c) { tmem_ld_kernel<8><<<148, 512>>>(o, c); }, 8 * ld_bytes);
  const double st_bytes = (ITERS / 8) * 2 * 16.0 * 32 * 4;  // per warp
  report("tcgen05.st B/clk, 4 warps", [](float* o, long long* c) { tmem_st_kernel<4><<<148, 512>>>(o, c); }, 4 * st_bytes);
  report("tcgen05.st B/clk, 16 warps", [](float* o, long long* c) { tmem_st_kernel<16><<<148, 512>>>(o, c); }, 16 * st_bytes);
  report("tcgen05.ld B/clk, 16 warps", [](float* o, long long* c) { tmem_ld_kernel<16><<<148, 512>>>(o, c); }, 16 * ld_bytes);
  return 0;
}
