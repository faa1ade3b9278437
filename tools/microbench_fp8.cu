// microbench_fp8.cu -- can the W4A4 blocks run on tcgen05.mma kind::f8f6f4?
// (tools only; not part of libcomet.so)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/microbench_fp8 tools/microbench_fp8.cu
// 1. exactness: D = sum_k A[m,k] B[n,k] over K = 128 (4 x K=32 MMAs,
//    M = N = 128, cta_group::1, SS) for integer-valued e4m3 operands, compared
//    with the exact sum (INT4 x INT4 blocks: |D| <= 49 * 128 = 6272), plus
//    probes of the accumulation precision with larger values;
// 2. issue rate of kind::f8f6f4 vs kind::i8 (cta_group::2, SS and TS);
// 3. pipe rates of PRMT / LOP3 (the nibble -> e4m3 conversion).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2410_12168_b200/csrc/sm100.cuh"

using namespace comet;

__host__ __device__ constexpr uint32_t idesc_mk(uint32_t cfmt, uint32_t afmt, uint32_t bfmt, uint32_t M, uint32_t N) {
  return (cfmt << 4) | (afmt << 7) | (bfmt << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <int KIND>  // 0: f8f6f4 e4m3 -> f32, 1: i8 -> s32
DEVI void mma_ss1(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (KIND == 0)
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
  else
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
}

// A, B: [128 x 128] bytes row-major (K contiguous); out: [128 x 128] 32-bit
template <int KIND>
__global__ void __launch_bounds__(128, 1) exact_kernel(const uint8_t* A, const uint8_t* B, uint32_t* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 128 * 128; i += 128) {
    const int r = i >> 7, k = i & 127;
    const int off = r * 128 + (((k >> 4) ^ (r & 7)) << 4) + (k & 15);
    smem[off] = A[i];
    smem[16384 + off] = B[i];
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<128>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t a = smem_u32(smem), b = a + 16384;
      const uint32_t idesc = KIND == 0 ? idesc_mk(1, 0, 0, 128, 128) : idesc_mk(2, 1, 1, 128, 128);
      for (int k = 0; k < 4; ++k)
        mma_ss1<KIND>(tm, umma_desc_sw128_kmajor(a + 32 * k), umma_desc_sw128_kmajor(b + 32 * k), idesc, k > 0);
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tm + ((uint32_t)(32 * warp) << 16) + 32 * c, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[(32 * warp + (threadIdx.x & 31)) * 128 + 32 * c + j] = r[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tm);
}

double e4m3_val(uint8_t b) {
  const int s = b >> 7, e = (b >> 3) & 15, m = b & 7;
  if (e == 15 && m == 7) return NAN;
  double v = e == 0 ? (m / 8.0) * std::ldexp(1.0, -6) : (1 + m / 8.0) * std::ldexp(1.0, e - 7);
  return s ? -v : v;
}
uint8_t e4m3_enc(double v) {
  for (int b = 0; b < 256; ++b)
    if (e4m3_val((uint8_t)b) == v && !(v == 0 && b != 0)) return (uint8_t)b;
  fprintf(stderr, "not representable: %g\n", v);
  exit(1);
}

struct Case {
  const char* name;
  std::vector<double> a, b;  // values
};

int run_case(const Case& c, bool i8) {
  std::vector<uint8_t> ha(128 * 128), hb(128 * 128);
  for (int i = 0; i < 128 * 128; ++i) {
    if (i8) {
      ha[i] = (uint8_t)(int8_t)c.a[i];
      hb[i] = (uint8_t)(int8_t)c.b[i];
    } else {
      ha[i] = e4m3_enc(c.a[i]);
      hb[i] = e4m3_enc(c.b[i]);
    }
  }
  uint8_t *da, *db;
  uint32_t* dout;
  cudaMalloc(&da, 16384);
  cudaMalloc(&db, 16384);
  cudaMalloc(&dout, 65536);
  cudaMemcpy(da, ha.data(), 16384, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), 16384, cudaMemcpyHostToDevice);
  auto k = i8 ? exact_kernel<1> : exact_kernel<0>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  k<<<1, 128, 40 * 1024>>>(da, db, dout);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<uint32_t> ho(16384);
  cudaMemcpy(ho.data(), dout, 65536, cudaMemcpyDeviceToHost);
  int bad = 0;
  double maxerr = 0, maxabs = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 128; ++n) {
      double ref = 0;  // exact: every product and partial sum is an integer multiple of a power of two < 2^53
      for (int kk = 0; kk < 128; ++kk) ref += c.a[m * 128 + kk] * c.b[n * 128 + kk];
      uint32_t raw = ho[m * 128 + n];
      double got;
      if (i8) got = (double)(int32_t)raw;
      else { float f; memcpy(&f, &raw, 4); got = f; }
      maxabs = std::fmax(maxabs, std::fabs(ref));
      if (got != ref) {
        ++bad;
        maxerr = std::fmax(maxerr, std::fabs(got - ref));
      }
    }
  printf("  %-58s %s  max|ref| %12.6g  mismatches %5d  max err %g\n", c.name, i8 ? "i8  " : "e4m3", maxabs, bad, maxerr);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dout);
  return (e == cudaSuccess ? 0 : 1000) + bad;
}

// ---- throughput -------------------------------------------------------------
constexpr int ITERS = 4096;
template <int KIND, bool kTS, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) rate_kernel(long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[4];
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  const uint32_t crank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (128 + 128) * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x38383838u, 0, 0x38383838u, 0);
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc_2sm<512>(&holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = holder;
  long long t0 = clock64();
  if (warp == 0 && crank == 0) {
    const uint32_t a_s = smem_u32(smem), b_s = a_s + 128 * 128;
    constexpr uint32_t idesc = KIND == 0 ? idesc_mk(1, 0, 0, 256, N) : idesc_mk(2, 1, 1, 256, N);
    for (int c = 0; c < ITERS / 8; ++c) {
      if (c >= 4) mbar_wait(&bars[c % 4], ((c / 4) - 1) & 1);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t bd = umma_desc_sw128_kmajor(b_s + 32 * (k & 3));
          if (KIND == 0 && kTS)
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 1, 0;\n tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                         "r"(tmem + 256 + 8 * (k & 3)), "l"(bd), "r"(idesc) : "memory");
          else if (KIND == 0)
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 1, 0;\n tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                         "l"(umma_desc_sw128_kmajor(a_s + 32 * (k & 3))), "l"(bd), "r"(idesc) : "memory");
          else if (kTS)
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 1, 0;\n tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                         "r"(tmem + 256 + 8 * (k & 3)), "l"(bd), "r"(idesc) : "memory");
          else
            mma_i8_ss_2sm(tmem, umma_desc_sw128_kmajor(a_s + 32 * (k & 3)), bd, idesc, 1);
        }
        mma_commit_2sm(&bars[c % 4], 0x1);
      }
      __syncwarp();
    }
    for (int c = ITERS / 8 - 4; c < ITERS / 8; ++c) mbar_wait(&bars[c % 4], (c / 4) & 1);
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_2sm<512>(tmem);
  if (threadIdx.x == 0 && crank == 0) cyc[blockIdx.x >> 1] = t1 - t0;
}

template <int KIND, bool kTS, int N>
void rate(const char* name) {
  long long* d;
  cudaMalloc(&d, 74 * sizeof(long long));
  auto k = rate_kernel<KIND, kTS, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<148, 128, 64 * 1024>>>(d);
  k<<<148, 128, 64 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[74];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 74; ++i) mx = h[i] > mx ? h[i] : mx;
  const double macs_per_sm = (double)ITERS * 256 * N * 32 / 2;
  printf("  %-34s N=%3d  %8.1f MAC/clk/SM  %s\n", name, N, macs_per_sm / mx, cudaGetErrorString(e));
  cudaFree(d);
}

// ---- ALU pipe: PRMT / LOP3 / SHF lane-op rates ---------------------------------
template <int OP>
__global__ void __launch_bounds__(512) alu_kernel(uint32_t* out, long long* cyc, uint32_t seed) {
  uint32_t v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = seed * (threadIdx.x + 1) + j;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < 4096; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) asm volatile("prmt.b32 %0, %1, %2, %0;" : "+r"(v[j]) : "r"(0x4E4C4A48u), "r"(0x44403800u));
      if (OP == 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0xE8;" : "+r"(v[j]) : "r"(i), "r"(0x77777777u));
      if (OP == 2) asm volatile("shf.l.wrap.b32 %0, %0, %0, 4;" : "+r"(v[j]));
      if (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[j]) : "r"(seed), "r"(i));
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s ^= v[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP>
void alu(const char* name) {
  uint32_t* o;
  long long* c;
  cudaMalloc(&o, 148 * 512 * 4);
  cudaMalloc(&c, 148 * 8);
  alu_kernel<OP><<<148, 512>>>(o, c, 12345u);
  alu_kernel<OP><<<148, 512>>>(o, c, 12345u);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("  %-34s %8.1f lane-ops per SM-clock\n", name, 512.0 * 4096 * 8 / avg);
  cudaFree(o);
  cudaFree(c);
}

int main() {
  srand(1);
  auto rnd = [](int lo, int hi) { return lo + rand() % (hi - lo + 1); };
  int fails = 0;
  printf("exactness (M=N=K=128, 4 x K=32 MMAs, fresh accumulator):\n");
  {
    Case c{"random INT4 x INT4 in [-7,7] (normal codes)", std::vector<double>(16384), std::vector<double>(16384)};
    for (int t = 0; t < 5; ++t) {
      for (auto& x : c.a) x = rnd(-7, 7);
      for (auto& x : c.b) x = rnd(-7, 7);
      fails += run_case(c, false);
      fails += run_case(c, true);
    }
  }
  {
    Case c{"random INT4 x INT4 as q * 2^-9 (subnormal codes)", std::vector<double>(16384), std::vector<double>(16384)};
    for (int t = 0; t < 3; ++t) {
      for (auto& x : c.a) x = rnd(-7, 7) * std::ldexp(1.0, -9);
      for (auto& x : c.b) x = rnd(-7, 7) * std::ldexp(1.0, -9);
      fails += run_case(c, false);
    }
  }
  {
    Case c{"extreme INT4: +-7 x +-7, row/col signs (|D| = 6272)", std::vector<double>(16384), std::vector<double>(16384)};
    for (int i = 0; i < 16384; ++i) {
      c.a[i] = ((i >> 7) & 1) ? -7 : 7;
      c.b[i] = ((i >> 7) % 3) ? 7 : -7;
    }
    fails += run_case(c, false);
    // large first, then small terms
    for (int i = 0; i < 16384; ++i) {
      const int k = i & 127;
      c.a[i] = k < 96 ? 7 : rnd(-1, 1);
      c.b[i] = k < 96 ? 7 : rnd(-7, 7);
    }
    c.name = "INT4: 96 x 49 first, then +-small (|D| ~ 4704)";
    fails += run_case(c, false);
    for (int i = 0; i < 16384; ++i) {
      const int k = i & 127;
      c.a[i] = k >= 32 ? 7 : rnd(-1, 1);
      c.b[i] = k >= 32 ? -7 : rnd(-7, 7);
    }
    c.name = "INT4: +-small first, then 96 x -49";
    fails += run_case(c, false);
  }
  printf("probes (informational -- outside the INT4 x INT4 range):\n");
  {
    Case c{"split INT8: hi in [-8,8] / lo in [0,15] x INT4", std::vector<double>(16384), std::vector<double>(16384)};
    for (auto& x : c.a) x = rnd(0, 15);
    for (auto& x : c.b) x = rnd(-7, 7);
    run_case(c, false);
    for (auto& x : c.a) x = 15;
    for (int i = 0; i < 16384; ++i) c.b[i] = ((i >> 7) & 1) ? 7 : -7;
    c.name = "15 x +-7 everywhere (|D| = 13440)";
    run_case(c, false);
    for (int i = 0; i < 16384; ++i) {
      const int k = i & 127;
      c.a[i] = k == 0 ? 448 : 1;
      c.b[i] = k == 0 ? 448 : ((i >> 7) & 1 ? 1 : -1);
    }
    c.name = "one 448*448 product then 127 x +-1 (same K chunk first)";
    run_case(c, false);
    for (int i = 0; i < 16384; ++i) {
      const int k = i & 127;
      c.a[i] = k < 32 ? 448 : 1;
      c.b[i] = k < 32 ? 448 : ((i >> 7) & 1 ? 1 : -1);
    }
    c.name = "32 x 448*448 (2^22.6) then 96 x +-1";
    run_case(c, false);
    for (int i = 0; i < 16384; ++i) {
      const int k = i & 127;
      c.a[i] = k < 32 ? 16 : 1;
      c.b[i] = k < 32 ? 16 : ((i >> 7) & 1 ? 1 : -1);
    }
    c.name = "32 x 256 (2^13) then 96 x +-1";
    run_case(c, false);
    for (int i = 0; i < 16384; ++i) {
      const int k = i & 127;
      c.a[i] = k < 32 ? 64 : 1;
      c.b[i] = k < 32 ? 64 : ((i >> 7) & 1 ? 1 : -1);
    }
    c.name = "32 x 4096 (2^17) then 96 x +-1";
    run_case(c, false);
  }
  printf("EXACT_FAILS %d\n", fails);
  printf("issue rates (cta_group::2, M=256, K=32; nominal 8192 MAC/clk/SM):\n");
  rate<0, false, 192>("SS f8f6f4 e4m3");
  rate<0, false, 256>("SS f8f6f4 e4m3");
  rate<0, true, 192>("TS f8f6f4 e4m3");
  rate<0, true, 256>("TS f8f6f4 e4m3");
  rate<1, false, 192>("SS i8");
  rate<1, false, 256>("SS i8");
  rate<1, true, 192>("TS i8");
  printf("ALU pipe:\n");
  alu<0>("PRMT");
  alu<1>("LOP3");
  alu<2>("SHF");
  alu<3>("IMAD (fma pipe)");
  return 0;
}
