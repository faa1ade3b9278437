// comet_api.cu -- host side of libcomet.so: argument validation, TMA tensor
// map construction, launch heuristics and the extern "C" entry points
// declared in include/comet.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <algorithm>
#include <vector>

#include "../../include/comet.h"
#include "gemm.cuh"
#include "gemm_pf.cuh"
#include "fmpq_aux.cuh"
#include "gemm_decode.cuh"
#include "quantize.cuh"
#include "quantize_lane.cuh"
#include "tp.cuh"

using namespace comet;

namespace {

thread_local char g_cuda_err[256] = "";
std::atomic<int64_t> g_launches{0};
// tools only (comet_debug_set_pf_clusters): CTA pairs of the prefill grid,
// 0 = one persistent pair per SM pair (the product schedule)
std::atomic<int> g_pf_clusters{0};
// tools only (comet_debug_set_pf_group): token tiles per raster group, 0 = by L2 budget
std::atomic<int> g_pf_group{0};
// tools only (comet_debug_set_prefill_min_m): M above which the prefill kernel runs
// (0 = the product rule)
std::atomic<int> g_pf_min_m{0};

comet_status cuda_fail(cudaError_t e) {
  snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return COMET_ERR_CUDA;
}
// a TMA descriptor the driver refused (bad address, stride or box)
comet_status map_fail(const char* what) {
  snprintf(g_cuda_err, sizeof(g_cuda_err), "cuTensorMapEncodeTiled failed for %s", what);
  return COMET_ERR_CUDA;
}
// launch with the programmatic-stream-serialization (PDL) attribute: the
// kernel may start while its predecessor in the stream still runs; every
// GEMM kernel waits (griddepcontrol.wait) before touching data a predecessor
// may produce
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

comet_status check_launch() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? COMET_OK : cuda_fail(e);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- device capability (cached once per device, thread-safe) -------------
std::mutex g_dev_mu;
int g_dev_ok[64];  // 0 unknown, 1 ok, -1 unsupported
int g_num_sms[64];

comet_status device_check(int* num_sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  if (dev < 0 || dev >= 64) return COMET_ERR_UNSUPPORTED;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (g_dev_ok[dev] == 0) {
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) return cuda_fail(e);
    g_dev_ok[dev] = (prop.major == 10 && prop.minor == 0) ? 1 : -1;
    g_num_sms[dev] = prop.multiProcessorCount;
  }
  if (num_sms) *num_sms = g_num_sms[dev];
  return g_dev_ok[dev] == 1 ? COMET_OK : COMET_ERR_UNSUPPORTED;
}

// ---- TMA tensor maps via the driver entry point (no -lcuda needed) ------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D uint8 tensor [rows x cols] (row stride ld bytes), box [box_rows x box_cols]
bool make_map_u8(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_cols,
                 uint32_t box_rows, CUtensorMapSwizzle swz) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D fp32 tensor [rows x cols] (row stride ld elements), box [box_rows x box_cols],
// out-of-bounds elements zero-filled
bool make_map_f32(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_cols,
                  uint32_t box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// ---- per-device opt-in to large dynamic shared memory -----------------------
// cudaFuncSetAttribute applies to the current device only: remember, per
// kernel and per device, that it succeeded (a failure is not cached)
struct AttrCache {
  std::atomic<uint64_t> done{0};
  cudaError_t set(const void* kern, int smem) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
  }
};

// ---- block map ------------------------------------------------------------
bool build_block_map(const uint8_t* bits, int nb, BlockMap* map, int* n8, int* n4) {
  int r8 = 0, r4 = 0;
  for (int b = 0; b < nb; ++b) {
    if (bits[b] == 8) {
      map->code[b] = (uint16_t)(0x8000u | r8++);
    } else if (bits[b] == 4) {
      map->code[b] = (uint16_t)(r4++);
    } else {
      return false;
    }
  }
  for (int b = nb; b < 512; ++b) map->code[b] = 0;
  if (n8) *n8 = r8;
  if (n4) *n4 = r4;
  return true;
}

// ---- GEMM launch plan -----------------------------------------------------
struct Plan {
  int bn, m_tiles, n_tiles, splits;
  bool two_sm;   // prefill: CTA-pair kernel (256 tokens x 192 weight rows per pair)
  int clusters;  // persistent CTA pairs
  int64_t ws_bytes;
};
constexpr int64_t kCounterBytes = 64 * 1024;
int64_t align256(int64_t x) { return (x + 255) / 256 * 256; }

// Kernel choice by M (per_channel: 1 = weight scales per output channel, 0 =
// group 128, -1 = unknown).  The prefill kernel above 128 tokens; with
// per-channel scales already above 64: there one half-empty 256-token tile of
// the CTA-pair kernel beats the decode kernel's BN = 128 tiles on every
// measured shape (70B gate_up 171 vs 189-194 us, 8B gate_up 60 vs 83-85 us, 8B
// down 66.5 vs 67-71 us at M = 80..128; tools/mband_sweep.py,
// profiles/mband_sweep_r2.txt), while with group-128 scales the decode kernel
// wins on two of the three shapes.  Unknown (the workspace-size query): the
// plan of the two with the larger workspace, so one buffer serves both.
Plan make_plan_for(int M, int N, int K, int num_sms, bool two_sm);
Plan make_plan(int M, int N, int K, int num_sms, int per_channel = -1) {
  const int pf_min = g_pf_min_m.load(std::memory_order_relaxed);
  if (pf_min > 0) return make_plan_for(M, N, K, num_sms, M > pf_min);
  if (M > 128 || M <= 64) return make_plan_for(M, N, K, num_sms, M > 128);
  if (per_channel >= 0) return make_plan_for(M, N, K, num_sms, per_channel == 1);
  const Plan a = make_plan_for(M, N, K, num_sms, true), b = make_plan_for(M, N, K, num_sms, false);
  if (a.ws_bytes < 0 || b.ws_bytes < 0) return a.ws_bytes < 0 ? a : b;
  return a.ws_bytes >= b.ws_bytes ? a : b;
}
Plan make_plan_for(int M, int N, int K, int num_sms, bool two_sm) {
  Plan p;
  p.two_sm = two_sm;
  p.splits = 1;
  if (p.two_sm) {
    p.bn = 128;  // token rows per CTA (TMA box height)
    p.m_tiles = (M + 255) / 256;
    p.n_tiles = (N + PfCfg::kTileN - 1) / PfCfg::kTileN;
    // workspace: [tile counters (kept for decode calls sharing the buffer)]
    // [e4m3 token plane, M x K4 bytes (K4 <= K)] [corrections 8 sum(xq), K/128 x ldsx fp32]
    const int64_t ldsx = ((int64_t)M + 3) / 4 * 4;
    p.ws_bytes = kCounterBytes + align256((int64_t)M * K) + align256((int64_t)(K / 128) * ldsx * 4);
    p.clusters = num_sms / 2;
    return p;
  }
  // decode: stream-K over (tile, K-block) units, one CTA per SM
  p.bn = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : 128;
  p.m_tiles = (M + p.bn - 1) / p.bn;
  p.n_tiles = N / 128;
  const int64_t tiles = (int64_t)p.m_tiles * p.n_tiles;
  const int64_t units = tiles * (K / 128);
  p.clusters = (int)(units < num_sms ? units : num_sms);  // CTAs
  p.ws_bytes = kCounterBytes + (int64_t)p.clusters * 2 * 128 * p.bn * 4;
  if (tiles > kCounterBytes / 4) p.ws_bytes = -1;  // more tiles than tile counters
  if (units * p.clusters >= (int64_t)1 << 32) p.ws_bytes = -1;  // kernel's 32-bit stream-K split arithmetic
  return p;
}

template <bool kGroupK, bool kAcc>
comet_status launch_gemm_pf(const CUtensorMap& tmXe, const CUtensorMap& tmX8, const CUtensorMap& tmY,
                            const BlockMap& map, const GemmArgs& args, const Plan& p, cudaStream_t st,
                            const YPeerMaps& yp) {
  using C = PfCfg;
  auto kern = w4ax_gemm_pf_kernel<kGroupK, kAcc>;
  static AttrCache cache;
  cudaError_t attr_err = cache.set(reinterpret_cast<const void*>(kern), C::kSmemBytes);
  if (attr_err != cudaSuccess) return cuda_fail(attr_err);
  PfSched sched;
  sched.m_tiles = p.m_tiles;
  sched.n_tiles = p.n_tiles;
  sched.tiles = p.m_tiles * p.n_tiles;
  // raster group: as many 256-row token tiles (256 x K operand bytes each) as
  // fit in ~48 MB of the 126 MB L2, so the group's tokens are read from HBM
  // once while the weight tiles stream past (LLaMA-3-8B down projection,
  // K = 14336: one group of all 32 token tiles re-read the 117 MB token plane
  // ~10x, 1.26 GB of DRAM reads per launch)
  const int64_t budget = 48ll << 20;
  int gm = (int)std::min<int64_t>(p.m_tiles, std::max<int64_t>(1, budget / (256ll * args.K)));
  if (g_pf_group.load(std::memory_order_relaxed) > 0) gm = std::min(p.m_tiles, g_pf_group.load());
  sched.group_m = gm;
  const int want = g_pf_clusters.load(std::memory_order_relaxed) > 0 ? g_pf_clusters.load() : p.clusters;
  sched.clusters = sched.tiles < want ? sched.tiles : want;
  // PDL: the prologue (barrier init, TMEM allocation) overlaps the token
  // preparation kernel; the producers wait for it before their first load
  cudaError_t e = launch_pdl(kern, dim3(2 * sched.clusters), dim3(C::kThreads), C::kSmemBytes, st, tmXe, tmX8, tmY,
                             map, args, sched, yp);
  if (e != cudaSuccess) return cuda_fail(e);
  return check_launch();
}

struct DecMaps {
  CUtensorMap sx, sw;  // Sx [nb x ldsx] box [kUB x BN]; Sw [nb x N] box [kUB x 128] (group 128)
};

template <int BN, bool kGroupK, bool kAcc>
comet_status launch_decode(const DecMaps& dm, const CUtensorMap& tmX4, const CUtensorMap& tmX8,
                           const BlockMap& map, const GemmArgs& args, const Plan& p, cudaStream_t st) {
  using C = DecCfg<BN>;
  auto kern = w4ax_gemm_decode_kernel<BN, kGroupK, kAcc>;
  static AttrCache cache;
  cudaError_t attr_err = cache.set(reinterpret_cast<const void*>(kern), C::kSmemBytes);
  if (attr_err != cudaSuccess) return cuda_fail(attr_err);
  DecSched sched;
  sched.n_tiles = p.n_tiles;
  sched.tiles = p.n_tiles * p.m_tiles;
  sched.units = sched.tiles * args.nb;  // K-blocks: the split granularity
  sched.ctas = p.clusters;
  cudaError_t e = launch_pdl(kern, dim3(sched.ctas), dim3(C::kThreads), C::kSmemBytes, st, dm.sx, tmX4, tmX8, dm.sw,
                             map, args, sched);
  if (e != cudaSuccess) return cuda_fail(e);
  return check_launch();
}

template <int BN, bool kGroupK, bool kAcc>
comet_status launch_decode_maps(const CUtensorMap& tmX4, const CUtensorMap& tmX8, const BlockMap& map,
                                const GemmArgs& args, const Plan& p, cudaStream_t st) {
  constexpr int kUB = DecCfg<BN>::kUB;
  DecMaps dm;
  if (!make_map_f32(&dm.sx, args.Sx, (uint64_t)args.ldsx, (uint64_t)args.nb, (uint64_t)args.ldsx, BN, kUB))
    return map_fail("Sx");
  if (!kGroupK && !kAcc) {
    if (!make_map_f32(&dm.sw, args.Sw, (uint64_t)args.N, (uint64_t)args.nb, (uint64_t)args.N, 128, kUB))
      return map_fail("Sw");
  } else {
    dm.sw = dm.sx;  // never dereferenced
  }
  return launch_decode<BN, kGroupK, kAcc>(dm, tmX4, tmX8, map, args, p, st);
}

template <bool kGroupK, bool kAcc>
comet_status launch_decode_bn(const CUtensorMap& tmX4, const CUtensorMap& tmX8, const BlockMap& map,
                              const GemmArgs& args, const Plan& p, cudaStream_t st) {
  switch (p.bn) {
    case 16: return launch_decode_maps<16, kGroupK, kAcc>(tmX4, tmX8, map, args, p, st);
    case 32: return launch_decode_maps<32, kGroupK, kAcc>(tmX4, tmX8, map, args, p, st);
    case 64: return launch_decode_maps<64, kGroupK, kAcc>(tmX4, tmX8, map, args, p, st);
    default: return launch_decode_maps<128, kGroupK, kAcc>(tmX4, tmX8, map, args, p, st);
  }
}

template <bool kAcc>
comet_status launch_gemm(const CUtensorMap& tmXp, const CUtensorMap& tmX8, const CUtensorMap& tmY,
                         const BlockMap& map, const GemmArgs& args, const Plan& p, cudaStream_t st,
                         const YPeerMaps& yp) {
  const bool group_k = args.group_blocks == args.nb;
  if (p.two_sm) {
    if (group_k) return launch_gemm_pf<true, kAcc>(tmXp, tmX8, tmY, map, args, p, st, yp);
    return launch_gemm_pf<false, kAcc>(tmXp, tmX8, tmY, map, args, p, st, yp);
  }
  if (group_k) return launch_decode_bn<true, kAcc>(tmXp, tmX8, map, args, p, st);
  return launch_decode_bn<false, kAcc>(tmXp, tmX8, map, args, p, st);
}

comet_status gemm_common(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx, const uint8_t* bits,
                         int32_t M, int32_t K, const void* Wq, const float* Sw, int32_t N, int32_t group, void* Y,
                         int64_t ldy, int32_t* Acc, void* ws, size_t ws_bytes, cudaStream_t st,
                         bool prepared = false, void* const* ypeers = nullptr, int npeer = 0) {
  // prepared (comet_w4ax_linear): the quantizer already wrote the prefill
  // kernel's e4m3 token plane and corrections into the workspace (Xq4 unused)
  if (!bits || M < 0 || N < 0 || K <= 0) return COMET_ERR_INVALID_ARG;
  if (K % 128 || N % 128 || K > 65536) return COMET_ERR_SHAPE;
  if (group != 128 && group != K) return COMET_ERR_SHAPE;
  if (ldsx < M || ldsx % 4) return COMET_ERR_SHAPE;
  const int nb = K / 128;
  BlockMap map;
  int n8 = 0, n4 = 0;
  if (!build_block_map(bits, nb, &map, &n8, &n4)) return COMET_ERR_INVALID_ARG;
  if (M == 0 || N == 0) return COMET_OK;
  if (!Wq || !Sx || (!Acc && (!Sw || !Y))) return COMET_ERR_INVALID_ARG;
  if (Acc == nullptr && (ldy < N || ldy % 8)) return COMET_ERR_SHAPE;
  if (Acc == nullptr && ((reinterpret_cast<uintptr_t>(Y) & 15) || (reinterpret_cast<uintptr_t>(Sw) & 15)))
    return COMET_ERR_ALIGNMENT;
  if ((n8 && !Xq8) || (n4 && !Xq4 && !prepared)) return COMET_ERR_INVALID_ARG;
  if ((n8 && !aligned16(Xq8)) || (n4 && !aligned16(Xq4)) || !aligned16(Wq) || !aligned16(Sx) || !aligned16(ws))
    return COMET_ERR_ALIGNMENT;
  int num_sms = 148;
  comet_status ds = device_check(&num_sms);
  if (ds != COMET_OK) return ds;
  Plan p = make_plan(M, N, K, num_sms, group == K ? 1 : 0);
  if (p.ws_bytes < 0) return COMET_ERR_SHAPE;
  if (p.ws_bytes > 0 && (ws == nullptr || (int64_t)ws_bytes < p.ws_bytes)) return COMET_ERR_WORKSPACE;

  // token operand maps: the INT8 plane (both kernels, SW128 rows of 128 B);
  // INT4 tokens as the e4m3 plane prepared below (prefill, SW128 rows of
  // 128 B) or the packed plane (decode, unswizzled rows of 64 B)
  CUtensorMap tmXp, tmX8;
  if (n8) {
    if (!make_map_u8(&tmX8, Xq8, (uint64_t)n8 * 128, (uint64_t)M, (uint64_t)n8 * 128, 128, p.bn,
                     CU_TENSOR_MAP_SWIZZLE_128B))
      return map_fail("Xq8");
  }
  uint8_t* x4e = reinterpret_cast<uint8_t*>(ws) + kCounterBytes;
  float* cx = reinterpret_cast<float*>(x4e + align256((int64_t)M * K));
  if (n4 && p.two_sm) {
    if (!make_map_u8(&tmXp, x4e, (uint64_t)n4 * 128, (uint64_t)M, (uint64_t)n4 * 128, 128, p.bn,
                     CU_TENSOR_MAP_SWIZZLE_128B))
      return map_fail("X4e");
  } else if (n4) {
    if (!make_map_u8(&tmXp, Xq4, (uint64_t)n4 * 64, (uint64_t)M, (uint64_t)n4 * 64, 64, p.bn,
                     CU_TENSOR_MAP_SWIZZLE_NONE))
      return map_fail("Xq4");
  }
  if (!n8) tmX8 = tmXp;  // never dereferenced
  if (!n4) tmXp = tmX8;
  // a8 (prefill): Y [M x N] fp16 as bytes, box 32 rows x 64 B (one promotion
  // warp's 32 rows x 32 columns), SW64 so the row-per-lane smem writes are
  // conflict-free; out-of-range rows / columns of a tile are clipped by TMA
  CUtensorMap tmY = tmX8;
  if (p.two_sm && !Acc) {
    if (!make_map_u8(&tmY, Y, (uint64_t)N * 2, (uint64_t)M, (uint64_t)ldy * 2, 64, 32, CU_TENSOR_MAP_SWIZZLE_64B))
      return map_fail("Y");
  }
  // f1: the peers' copies of the output take every Y store too
  if (npeer < 0 || npeer > kMaxYPeers || (npeer && (!ypeers || Acc))) return COMET_ERR_INVALID_ARG;
  YPeerMaps yp;
  memset(&yp, 0, sizeof(yp));
  yp.n = npeer;
  for (int i = 0; i < npeer; ++i) {
    if (!ypeers[i]) return COMET_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(ypeers[i]) & 15) return COMET_ERR_ALIGNMENT;
    if (p.two_sm && !make_map_u8(&yp.m[i], ypeers[i], (uint64_t)N * 2, (uint64_t)M, (uint64_t)ldy * 2, 64, 32,
                                 CU_TENSOR_MAP_SWIZZLE_64B))
      return map_fail("Y peer");
  }
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.npeer = npeer;
  for (int i = 0; i < npeer; ++i) a.Ypeer[i] = reinterpret_cast<__half*>(ypeers[i]);
  a.M = M;
  a.N = N;
  a.K = K;
  a.nb = nb;
  a.ldsx = ldsx;
  a.ldy = ldy;
  a.Sx = Sx;
  a.Sw = Sw;
  a.group_blocks = group / 128;
  a.Y = reinterpret_cast<__half*>(Y);
  a.Wq = reinterpret_cast<const uint8_t*>(Wq);
  a.Acc = Acc;
  a.CX = cx;
  a.splits = p.splits;
  a.ws_counter = reinterpret_cast<int*>(ws);
  a.ws_partial = ws ? reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + kCounterBytes) : nullptr;
  if (n4 && p.two_sm && !prepared) {
    // a4 for the tokens, once per call: INT4 plane -> e4m3 plane + corrections
    const int64_t items = ldsx * n4 * 4;
    int64_t grid = (items + 255) / 256;
    if (grid > (int64_t)num_sms * 8) grid = (int64_t)num_sms * 8;
    cudaError_t e = launch_pdl(prep_tokens_kernel, dim3((unsigned)grid), dim3(256), 0, st,
                               reinterpret_cast<const uint8_t*>(Xq4), (int)M, n4, ldsx, x4e, cx);
    if (e != cudaSuccess) return cuda_fail(e);
    comet_status ls = check_launch();
    if (ls != COMET_OK) return ls;
  }
  if (Acc) return launch_gemm<true>(tmXp, tmX8, tmY, map, a, p, st, yp);
  return launch_gemm<false>(tmXp, tmX8, tmY, map, a, p, st, yp);
}

// comet_w4ax_linear with host buffers: two internal copy streams and their
// events, created once per device and reused (thread-safe creation; one
// host-buffer call at a time per device, which the call's final synchronize
// already implies)
constexpr int kLinMaxChunks = 8;
struct LinStreams {
  cudaStream_t in, out;
  cudaEvent_t ev_start, ev_end, ev_end2, ev_compute, ev_in[kLinMaxChunks], ev_out[kLinMaxChunks];
  // the previous host-buffer call on this device: its stream, whether its
  // output copies are ordered only by ev_end, and the device range of its
  // staged Y (which those copies read)
  bool prev_valid = false;
  cudaStream_t prev_stream = nullptr;
  uintptr_t prev_ys_lo = 0, prev_ys_hi = 0;
};
LinStreams* lin_streams() {
  static LinStreams g_ls[64];
  static bool g_ok[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_ok[dev]) {
    LinStreams& L = g_ls[dev];
    bool ok = cudaStreamCreateWithFlags(&L.in, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&L.out, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&L.ev_start, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&L.ev_end, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&L.ev_end2, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&L.ev_compute, cudaEventDisableTiming) == cudaSuccess;
    for (int c = 0; c < kLinMaxChunks && ok; ++c)
      ok = cudaEventCreateWithFlags(&L.ev_in[c], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&L.ev_out[c], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) return nullptr;
    g_ok[dev] = true;
  }
  return &g_ls[dev];
}

int64_t plane_bytes(int32_t M, int32_t K, const uint8_t* bits, int want) {
  if (M < 0 || K <= 0 || K % 128 || !bits) return -1;
  int64_t cnt = 0;
  for (int b = 0; b < K / 128; ++b) {
    if (bits[b] != 4 && bits[b] != 8) return -1;
    if (bits[b] == want) ++cnt;
  }
  return want == 8 ? (int64_t)M * cnt * 128 : (int64_t)M * cnt * 64;
}

// X4e/CX non-null: INT4 blocks go straight to the prefill GEMM's e4m3 operand
// [M x n4*128 B] and its corrections (comet_w4ax_linear; row-staged kernel only)
template <bool kBf16>
comet_status quantize_act_impl(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                               const uint8_t* block_bits, int8_t* Xq8, void* Xq4, float* Sx, int64_t ldsx,
                               comet_stream_t stream, uint8_t* X4e = nullptr, float* CX = nullptr,
                               const uint16_t* perm16 = nullptr) {
  if (M < 0 || K <= 0 || !block_bits) return COMET_ERR_INVALID_ARG;
  if (K % 128 || K > 65536 || ldx < K || ldx % 8 || ldsx < M || ldsx % 4) return COMET_ERR_SHAPE;
  BlockMap map;
  int n8 = 0, n4 = 0;
  if (!build_block_map(block_bits, K / 128, &map, &n8, &n4)) return COMET_ERR_INVALID_ARG;
  if (M == 0) return COMET_OK;
  if (!X || !Sx || (n8 && !Xq8) || (n4 && !Xq4 && !X4e)) return COMET_ERR_INVALID_ARG;
  if (!aligned16(X) || (n8 && !aligned16(Xq8)) || (n4 && !aligned16(Xq4)) || !aligned16(Sx) ||
      (perm && !aligned16(perm)))
    return COMET_ERR_ALIGNMENT;
  int num_sms = 148;
  comet_status ds = device_check(&num_sms);
  if (ds != COMET_OK) return ds;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const __half* Xh = reinterpret_cast<const __half*>(X);
  if (M >= kLaneMinRows) {
    // thread-per-item kernel (quantize_lane.cuh): persistent, one CTA per SM
    const LanePlan lp = lane_plan(M, K, perm != nullptr);
    if (lp.S) {
      auto kern = X4e ? (perm ? quantize_lane_kernel<true, kBf16, true> : quantize_lane_kernel<true, kBf16, false>)
                      : (perm ? quantize_lane_kernel<false, kBf16, true> : quantize_lane_kernel<false, kBf16, false>);
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lp.smem);
      if (e != cudaSuccess) return cuda_fail(e);
      // persistent: as many CTAs per SM as shared memory / registers allow
      // (one at the default plan sizes)
      int per_sm = 1;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, lp.threads, lp.smem);
      if (e != cudaSuccess) return cuda_fail(e);
      const int64_t grid = std::min<int64_t>((int64_t)num_sms * std::max(1, per_sm), lp.stages);
      e = launch_pdl(kern, dim3((unsigned)grid), dim3(lp.threads), lp.smem, st, Xh, ldx, M, K / 128, ldsx, perm,
                     map, Xq8, (int64_t)n8 * 128, X4e ? X4e : reinterpret_cast<uint8_t*>(Xq4),
                     X4e ? (int64_t)n4 * 128 : (int64_t)n4 * 64, Sx, CX, lp.R, lp.S, lp.lpr);
      if (e != cudaSuccess) return cuda_fail(e);
      return check_launch();
    }
  }
  if (M >= 64) {
    // row-staged kernel: persistent CTAs, double-buffered rows in smem
    const int smem = kQNBuf * K * 2;  // row buffers
    if (smem <= 200 * 1024) {
      auto kern = X4e ? (perm16 ? quantize_act_rows_kernel<2, false, kBf16, true>
                                : perm ? quantize_act_rows_kernel<1, false, kBf16, true>
                                       : quantize_act_rows_kernel<0, false, kBf16, true>)
                      : (perm ? quantize_act_rows_kernel<1, false, kBf16> : quantize_act_rows_kernel<0, false, kBf16>);
      const int32_t* pk = (X4e && perm16) ? reinterpret_cast<const int32_t*>(perm16) : perm;
      // (dynamic smem above the 48 KB default needs the opt-in; set per call,
      // it is a cheap host-side attribute)
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return cuda_fail(e);
      // one wave of persistent CTAs: as many per SM as registers, shared
      // memory (row buffers + the static scale table) and threads allow
      int per_sm = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kQThreads, smem);
      if (e != cudaSuccess) return cuda_fail(e);
      if (per_sm < 1) per_sm = 1;
      int64_t grid = (int64_t)num_sms * per_sm;
      if (grid > ldsx) grid = ldsx;
      e = launch_pdl(kern, dim3((unsigned)grid), dim3(kQThreads), smem, st, Xh, ldx, M, K / 128, ldsx, pk, map, Xq8,
                     (int64_t)n8 * 128, X4e ? X4e : reinterpret_cast<uint8_t*>(Xq4),
                     X4e ? (int64_t)n4 * 128 : (int64_t)n4 * 64, Sx, static_cast<const float*>(nullptr), CX);
      if (e != cudaSuccess) return cuda_fail(e);
      return check_launch();
    }
  }
  if (X4e) return COMET_ERR_UNSUPPORTED;  // the fused output needs the row-staged kernel
  // one CTA per (8 rows, 2 blocks): 16 half-warp items
  const dim3 grid((unsigned)((ldsx + 7) / 8), (unsigned)((K / 128 + 1) / 2));
  cudaError_t e = launch_pdl(perm ? quantize_act_kernel<true, false, kBf16> : quantize_act_kernel<false, false, kBf16>,
                             grid, dim3(256), 0, st, Xh, ldx, M, K / 128, ldsx, perm, map, Xq8, (int64_t)n8 * 128,
                             reinterpret_cast<uint8_t*>(Xq4), (int64_t)n4 * 64, Sx);
  if (e != cudaSuccess) return cuda_fail(e);
  return check_launch();
}

}  // namespace

extern "C" {

int64_t comet_act_plane8_bytes(int32_t M, int32_t K, const uint8_t* block_bits) { return plane_bytes(M, K, block_bits, 8); }
int64_t comet_act_plane4_bytes(int32_t M, int32_t K, const uint8_t* block_bits) { return plane_bytes(M, K, block_bits, 4); }
int64_t comet_act_ldsx(int32_t M) { return M < 0 ? -1 : ((int64_t)M + 3) / 4 * 4; }

int64_t comet_w4ax_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K) {
  if (M < 0 || N < 0 || K <= 0 || K % 128 || N % 128) return -1;
  if (M == 0 || N == 0) return 0;
  int num_sms = 148;
  if (device_check(&num_sms) != COMET_OK) num_sms = 148;
  return make_plan(M, N, K, num_sms).ws_bytes;
}

int64_t comet_w4ax_linear_scratch_bytes(int32_t M, int32_t N, int32_t K, const uint8_t* block_bits) {
  int64_t p8 = plane_bytes(M, K, block_bits, 8), p4 = plane_bytes(M, K, block_bits, 4);
  int64_t ws = comet_w4ax_gemm_workspace_bytes(M, N, K);
  if (p8 < 0 || p4 < 0 || ws < 0) return -1;
  int64_t sx = (K / 128) * comet_act_ldsx(M) * 4;
  int64_t io = align256((int64_t)M * K * 2) + align256((int64_t)M * N * 2);  // staging for host X / Y
  io += align256((int64_t)K * 2);  // the permutation as uint16 (quantizer)
  // the GEMM workspace sits at the scratch base and is never shorter than the
  // stream-K tile counters, so a prefill call (no workspace) never overwrites
  // the counters a later decode call on the same scratch relies on
  return align256(std::max<int64_t>(ws, kCounterBytes)) + align256(p8) + align256(p4) + align256(sx) + align256(io) + 256;
}

comet_status comet_pack_weight(const void* W, int64_t ldw, int32_t N, int32_t K, const int32_t* perm, int32_t group,
                               void* Wq, float* Sw, comet_stream_t stream) {
  if (N < 0 || K <= 0) return COMET_ERR_INVALID_ARG;
  if (K % 128 || K > 65536 || N % 128 || (group != 128 && group != K) || ldw < K || ldw % 8) return COMET_ERR_SHAPE;
  if (N == 0) return COMET_OK;
  if (!W || !Wq || !Sw) return COMET_ERR_INVALID_ARG;
  if (!aligned16(W) || !aligned16(Wq) || (perm && !aligned16(perm))) return COMET_ERR_ALIGNMENT;
  comet_status ds = device_check(nullptr);
  if (ds != COMET_OK) return ds;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const __half* Wh = reinterpret_cast<const __half*>(W);
  if (group == 128) {
    // group-128 weights are "activations" with an all-INT4 mask, Sw = Sx with ldsx = N
    BlockMap map;
    for (int b = 0; b < 512; ++b) map.code[b] = (uint16_t)(b < K / 128 ? b : 0);
    const dim3 grid((unsigned)((N + 7) / 8), (unsigned)((K / 128 + 1) / 2));
    // Sw layout [K/128 x N] is the Sx layout with ldsx == N (no padding rows)
    if (perm)
      quantize_act_kernel<true, true><<<grid, 256, 0, st>>>(Wh, ldw, N, K / 128, N, perm, map, nullptr, 0,
                                                             reinterpret_cast<uint8_t*>(Wq), K / 2, Sw);
    else
      quantize_act_kernel<false, true><<<grid, 256, 0, st>>>(Wh, ldw, N, K / 128, N, perm, map, nullptr, 0,
                                                              reinterpret_cast<uint8_t*>(Wq), K / 2, Sw);
  } else {
    int grid = (N + 7) / 8;
    if (perm)
      pack_weight_rowscale_kernel<true><<<grid, 256, 0, st>>>(Wh, ldw, N, K, perm, reinterpret_cast<uint8_t*>(Wq), Sw);
    else
      pack_weight_rowscale_kernel<false><<<grid, 256, 0, st>>>(Wh, ldw, N, K, perm, reinterpret_cast<uint8_t*>(Wq), Sw);
  }
  return check_launch();
}

comet_status comet_quantize_act(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                                const uint8_t* block_bits, int8_t* Xq8, void* Xq4, float* Sx, int64_t ldsx,
                                comet_stream_t stream) {
  return quantize_act_impl<false>(X, ldx, M, K, perm, block_bits, Xq8, Xq4, Sx, ldsx, stream);
}

comet_status comet_quantize_act_bf16(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                                     const uint8_t* block_bits, int8_t* Xq8, void* Xq4, float* Sx, int64_t ldsx,
                                     comet_stream_t stream) {
  return quantize_act_impl<true>(X, ldx, M, K, perm, block_bits, Xq8, Xq4, Sx, ldsx, stream);
}

comet_status comet_w4ax_gemm(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx,
                             const uint8_t* block_bits, int32_t M, int32_t K, const void* Wq, const float* Sw,
                             int32_t N, int32_t group, void* Y, int64_t ldy, void* workspace, size_t workspace_bytes,
                             comet_stream_t stream) {
  return gemm_common(Xq8, Xq4, Sx, ldsx, block_bits, M, K, Wq, Sw, N, group, Y, ldy, nullptr, workspace,
                     workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}


comet_status comet_w4ax_gemm_acc_i32(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx,
                                     const uint8_t* block_bits, int32_t M, int32_t K, const void* Wq,
                                     const float* Sw, int32_t N, int32_t group, int32_t* Acc, void* workspace,
                                     size_t workspace_bytes, comet_stream_t stream) {
  if (M > 0 && N > 0 && !Acc) return COMET_ERR_INVALID_ARG;
  return gemm_common(Xq8, Xq4, Sx, ldsx, block_bits, M, K, Wq, Sw, N, group, nullptr, N, Acc, workspace,
                     workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

// comet_w4ax_linear and comet_w4ax_linear_allgather (ypeers: further
// destinations of Y, device buffers only)
static comet_status linear_impl(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                                const uint8_t* block_bits, const void* Wq, const float* Sw, int32_t N, int32_t group,
                                void* Y, int64_t ldy, void* scratch, size_t scratch_bytes, comet_stream_t stream,
                                void* const* ypeers, int npeer) {
  if (M < 0 || N < 0 || K <= 0 || !block_bits) return COMET_ERR_INVALID_ARG;
  if (npeer < 0 || npeer > kMaxYPeers || (npeer && !ypeers)) return COMET_ERR_INVALID_ARG;
  if (K % 128 || N % 128 || ldx < K || ldy < N || ldx % 8 || ldy % 8) return COMET_ERR_SHAPE;
  const int64_t need = comet_w4ax_linear_scratch_bytes(M, N, K, block_bits);
  if (need < 0) return COMET_ERR_INVALID_ARG;
  if (M == 0 || N == 0) return COMET_OK;
  if (!X || !Y || !Wq || !Sw) return COMET_ERR_INVALID_ARG;
  if (!scratch || (int64_t)scratch_bytes < need) return COMET_ERR_WORKSPACE;
  // everything comet_quantize_act / comet_w4ax_gemm would reject is checked
  // before the first copy or launch, so a failed call has no side effects
  if (group != 128 && group != K) return COMET_ERR_SHAPE;
  if (K > 65536) return COMET_ERR_SHAPE;
  if (!aligned16(Wq) || !aligned16(Sw) || (perm && !aligned16(perm)) || !aligned16(scratch)) return COMET_ERR_ALIGNMENT;
  if (make_plan(M, N, K, 148, group == K ? 1 : 0).ws_bytes < 0) return COMET_ERR_SHAPE;
  comet_status ds = device_check(nullptr);
  if (ds != COMET_OK) return ds;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaPointerAttributes ax, ay;
  cudaError_t e = cudaPointerGetAttributes(&ax, X);
  if (e != cudaSuccess) return cuda_fail(e);
  e = cudaPointerGetAttributes(&ay, Y);
  if (e != cudaSuccess) return cuda_fail(e);
  const bool x_host = ax.type != cudaMemoryTypeDevice && ax.type != cudaMemoryTypeManaged;
  const bool y_host = ay.type != cudaMemoryTypeDevice && ay.type != cudaMemoryTypeManaged;
  if (npeer && (x_host || y_host)) return COMET_ERR_INVALID_ARG;  // the fused all-gather writes device buffers
  for (int i = 0; i < npeer; ++i)
    if (!ypeers[i] || (reinterpret_cast<uintptr_t>(ypeers[i]) & 15)) return COMET_ERR_ALIGNMENT;

  char* p = reinterpret_cast<char*>(scratch);
  const int64_t ws_bytes = comet_w4ax_gemm_workspace_bytes(M, N, K);
  void* ws = p;  // counters stay at the scratch base (zeroed once, reset by the kernels)
  p += align256(std::max<int64_t>(ws_bytes, kCounterBytes));
  const int64_t p8 = plane_bytes(M, K, block_bits, 8), p4 = plane_bytes(M, K, block_bits, 4);
  int8_t* Xq8 = reinterpret_cast<int8_t*>(p);
  p += align256(p8);
  void* Xq4 = p;
  p += align256(p4);
  float* Sx = reinterpret_cast<float*>(p);
  p += align256((K / 128) * comet_act_ldsx(M) * 4);
  // the permutation as uint16 for the row-staged quantizer (prefill layers)
  const bool use16 = perm && M > 128 && (int64_t)kQNBuf * K * 2 <= 200 * 1024 && !(M >= kLaneMinRows && lane_plan(M, K, true).S);
  uint16_t* perm16 = use16 ? reinterpret_cast<uint16_t*>(p) : nullptr;
  p += align256((int64_t)K * 2);
  char* xs = nullptr;  // host X staged densely (ld = K)
  if (x_host) {
    xs = p;
    p += align256((int64_t)M * K * 2);
  }
  char* ys = y_host ? p : nullptr;  // host Y staged densely (ld = N)

  // one device-resident layer over rows [m0, m0 + mc): quantize + GEMM on st
  auto layer = [&](const void* Xd, int64_t ldxd, int32_t mc, void* Yd, int64_t ldyd) -> comet_status {
    const int64_t ldsx = comet_act_ldsx(mc);
    const int64_t wsb = comet_w4ax_gemm_workspace_bytes(mc, N, K);
    if (make_plan(mc, N, K, 148, group == K ? 1 : 0).two_sm && (int64_t)kQNBuf * K * 2 <= 200 * 1024) {
      // prefill: the quantizer writes the GEMM's e4m3 token operand and its
      // corrections straight into the workspace (no packed INT4 plane, no token
      // preparation kernel); identical results to the two-call path
      uint8_t* x4e = reinterpret_cast<uint8_t*>(ws) + kCounterBytes;
      float* cx = reinterpret_cast<float*>(x4e + align256((int64_t)mc * K));
      comet_status s = quantize_act_impl<false>(Xd, ldxd, mc, K, perm, block_bits, Xq8, nullptr, Sx, ldsx, stream,
                                                x4e, cx, perm16);
      if (s != COMET_OK) return s;
      return gemm_common(Xq8, nullptr, Sx, ldsx, block_bits, mc, K, Wq, Sw, N, group, Yd, ldyd, nullptr, ws,
                         (size_t)wsb, st, true, ypeers, npeer);
    }
    comet_status s = comet_quantize_act(Xd, ldxd, mc, K, perm, block_bits, Xq8, Xq4, Sx, ldsx, stream);
    if (s != COMET_OK) return s;
    return gemm_common(Xq8, Xq4, Sx, ldsx, block_bits, mc, K, Wq, Sw, N, group, Yd, ldyd, nullptr, ws,
                       wsb > 0 ? (size_t)wsb : 0, st, false, ypeers, npeer);
  };

  if (perm16) {
    perm_to_u16_kernel<<<(K + 255) / 256, 256, 0, st>>>(perm, K, perm16);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  if (!x_host && !y_host) {
    // a device-buffer call may use scratch bytes a later host-buffer call
    // stages into: that call must order its input copies after this one
    if (LinStreams* ls = lin_streams()) ls->prev_valid = false;
    return layer(X, ldx, M, Y, ldy);
  }

  // host buffers: row chunks pipeline H2D (copy stream) / compute (stream) /
  // D2H (copy stream), so the PCIe transfers in both directions overlap the
  // layer and each other; chunks of >= 1024 rows keep the prefill kernel's
  // tiles full (a tail under 256 rows joins the previous chunk)
  LinStreams* ls = lin_streams();
  if (!ls) return cuda_fail(cudaGetLastError());
  int nch = M >= 2048 ? std::min<int>(kLinMaxChunks, (int)((M + 1023) / 1024)) : 1;
  std::vector<int> edges(nch + 1);
  for (int c = 0; c <= nch; ++c) edges[c] = (int)(((int64_t)M * c / nch + 255) / 256 * 256);
  edges[nch] = M;
  // input copies: after the caller's earlier work on st -- except right after
  // a host-buffer call on the same stream, whose tail makes st wait for its
  // output copies: then only after that call's compute (and its output
  // copies only if this call's staged X overlaps the Y they read), so this
  // call's H2D overlaps the previous call's D2H
  const uintptr_t xs_lo = reinterpret_cast<uintptr_t>(xs), xs_hi = xs_lo + (x_host ? (uintptr_t)M * K * 2 : 0);
  if (ls->prev_valid && ls->prev_stream == st) {
    if ((e = cudaStreamWaitEvent(ls->in, ls->ev_compute, 0)) != cudaSuccess) return cuda_fail(e);
    if (x_host && xs_lo < ls->prev_ys_hi && ls->prev_ys_lo < xs_hi &&
        (e = cudaStreamWaitEvent(ls->in, ls->ev_end, 0)) != cudaSuccess)
      return cuda_fail(e);
  } else {
    if ((e = cudaEventRecord(ls->ev_start, st)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaStreamWaitEvent(ls->in, ls->ev_start, 0)) != cudaSuccess) return cuda_fail(e);
  }
  for (int c = 0; c < nch; ++c) {
    const int m0 = edges[c], mc = edges[c + 1] - m0;
    if (mc <= 0) continue;
    const void* Xd = reinterpret_cast<const char*>(X) + (int64_t)m0 * ldx * 2;
    int64_t ldxd = ldx;
    if (x_host) {
      e = cudaMemcpy2DAsync(xs + (int64_t)m0 * K * 2, (size_t)K * 2, Xd, (size_t)ldx * 2, (size_t)K * 2, (size_t)mc,
                            cudaMemcpyHostToDevice, ls->in);
      if (e != cudaSuccess) return cuda_fail(e);
      if ((e = cudaEventRecord(ls->ev_in[c], ls->in)) != cudaSuccess) return cuda_fail(e);
      if ((e = cudaStreamWaitEvent(st, ls->ev_in[c], 0)) != cudaSuccess) return cuda_fail(e);
      Xd = xs + (int64_t)m0 * K * 2;
      ldxd = K;
    }
    void* Yd = y_host ? static_cast<void*>(ys + (int64_t)m0 * N * 2)
                      : static_cast<void*>(reinterpret_cast<char*>(Y) + (int64_t)m0 * ldy * 2);
    comet_status s = layer(Xd, ldxd, mc, Yd, y_host ? N : ldy);
    if (s != COMET_OK) return s;
    if (y_host) {
      if ((e = cudaEventRecord(ls->ev_out[c], st)) != cudaSuccess) return cuda_fail(e);
      if ((e = cudaStreamWaitEvent(ls->out, ls->ev_out[c], 0)) != cudaSuccess) return cuda_fail(e);
      e = cudaMemcpy2DAsync(reinterpret_cast<char*>(Y) + (int64_t)m0 * ldy * 2, (size_t)ldy * 2, Yd, (size_t)N * 2,
                            (size_t)N * 2, (size_t)mc, cudaMemcpyDeviceToHost, ls->out);
      if (e != cudaSuccess) return cuda_fail(e);
    }
  }
  // later work on st (and a synchronisation of st) orders after the copies;
  // the call itself does not wait: host Y is complete once st is synchronised
  if ((e = cudaEventRecord(ls->ev_compute, st)) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaEventRecord(ls->ev_end, ls->out)) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaStreamWaitEvent(st, ls->ev_end, 0)) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaEventRecord(ls->ev_end2, ls->in)) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaStreamWaitEvent(st, ls->ev_end2, 0)) != cudaSuccess) return cuda_fail(e);
  ls->prev_valid = true;
  ls->prev_stream = st;
  ls->prev_ys_lo = reinterpret_cast<uintptr_t>(ys);
  ls->prev_ys_hi = ls->prev_ys_lo + (y_host ? (uintptr_t)M * N * 2 : 0);
  return COMET_OK;
}

comet_status comet_w4ax_linear(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                               const uint8_t* block_bits, const void* Wq, const float* Sw, int32_t N, int32_t group,
                               void* Y, int64_t ldy, void* scratch, size_t scratch_bytes, comet_stream_t stream) {
  return linear_impl(X, ldx, M, K, perm, block_bits, Wq, Sw, N, group, Y, ldy, scratch, scratch_bytes, stream,
                     nullptr, 0);
}

// f1: the destinations' column offset col0 applied to every pointer; Ys[0]
// is this rank's copy, Ys[1 ..] the peers'
static comet_status offset_dests(void* const* Ys, int32_t nY, int64_t col0, void** out) {
  if (!Ys || nY < 1 || nY > kMaxYPeers + 1 || col0 < 0 || col0 % 8) return COMET_ERR_INVALID_ARG;
  for (int i = 0; i < nY; ++i) {
    if (!Ys[i]) return COMET_ERR_INVALID_ARG;
    out[i] = reinterpret_cast<char*>(Ys[i]) + col0 * 2;
  }
  return COMET_OK;
}

comet_status comet_w4ax_gemm_allgather(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx,
                                       const uint8_t* block_bits, int32_t M, int32_t K, const void* Wq,
                                       const float* Sw, int32_t N, int32_t group, void* const* Ys, int32_t nY,
                                       int64_t ldy, int64_t col0, void* workspace, size_t workspace_bytes,
                                       comet_stream_t stream) {
  void* d[kMaxYPeers + 1];
  comet_status s = offset_dests(Ys, nY, col0, d);
  if (s != COMET_OK) return s;
  if (ldy < col0 + N) return COMET_ERR_SHAPE;
  return gemm_common(Xq8, Xq4, Sx, ldsx, block_bits, M, K, Wq, Sw, N, group, d[0], ldy, nullptr, workspace,
                     workspace_bytes, reinterpret_cast<cudaStream_t>(stream), false, d + 1, nY - 1);
}

comet_status comet_w4ax_linear_allgather(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                                         const uint8_t* block_bits, const void* Wq, const float* Sw, int32_t N,
                                         int32_t group, void* const* Ys, int32_t nY, int64_t ldy, int64_t col0,
                                         void* scratch, size_t scratch_bytes, comet_stream_t stream) {
  void* d[kMaxYPeers + 1];
  comet_status s = offset_dests(Ys, nY, col0, d);
  if (s != COMET_OK) return s;
  if (ldy < col0 + N) return COMET_ERR_SHAPE;
  for (const void* q : {X, static_cast<const void*>(d[0])}) {  // device buffers only
    cudaPointerAttributes at;
    if (!q) return COMET_ERR_INVALID_ARG;
    cudaError_t e = cudaPointerGetAttributes(&at, q);
    if (e != cudaSuccess) return cuda_fail(e);
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) return COMET_ERR_INVALID_ARG;
  }
  return linear_impl(X, ldx, M, K, perm, block_bits, Wq, Sw, N, group, d[0], ldy, scratch, scratch_bytes, stream,
                     d + 1, nY - 1);
}

comet_status comet_gather_shards(const void* Yall, int32_t P, int32_t M, int32_t per, int32_t N, void* Y,
                                 int64_t ldy, comet_stream_t stream) {
  if (P <= 0 || M < 0 || per < 0 || N < 0) return COMET_ERR_INVALID_ARG;
  if (per % 128 || N % 128 || (int64_t)P * per < N || ldy < N || ldy % 8) return COMET_ERR_SHAPE;
  if (M == 0 || N == 0) return COMET_OK;
  if (!Yall || !Y) return COMET_ERR_INVALID_ARG;
  if (!aligned16(Yall) || !aligned16(Y)) return COMET_ERR_ALIGNMENT;
  int num_sms = 148;
  comet_status ds = device_check(&num_sms);
  if (ds != COMET_OK) return ds;
  const int64_t items = (int64_t)P * M * (per / 8);
  int64_t grid = (items + 255) / 256;
  if (grid > (int64_t)num_sms * 16) grid = (int64_t)num_sms * 16;
  cudaError_t e = launch_pdl(gather_shards_kernel, dim3((unsigned)grid), dim3(256), 0,
                             reinterpret_cast<cudaStream_t>(stream), reinterpret_cast<const uint4*>(Yall), (int)P,
                             (int)M, (int)per, (int)N, reinterpret_cast<uint4*>(Y), ldy);
  if (e != cudaSuccess) return cuda_fail(e);
  return check_launch();
}

// ---- f4: FP16 / BF16 weight-scale storage ---------------------------------
}  // extern "C"
namespace {
template <bool kBf16S>
comet_status pack_weight_h16s(const void* W, int64_t ldw, int32_t N, int32_t K, const int32_t* perm, int32_t group,
                              void* Wq, void* Sw16, comet_stream_t stream) {
  if (N < 0 || K <= 0) return COMET_ERR_INVALID_ARG;
  if (K % 128 || K > 65536 || N % 128 || (group != 128 && group != K) || ldw < K || ldw % 8) return COMET_ERR_SHAPE;
  if (N == 0) return COMET_OK;
  if (!W || !Wq || !Sw16) return COMET_ERR_INVALID_ARG;
  if (!aligned16(W) || !aligned16(Wq) || (perm && !aligned16(perm)) || (reinterpret_cast<uintptr_t>(Sw16) & 1))
    return COMET_ERR_ALIGNMENT;
  comet_status ds = device_check(nullptr);
  if (ds != COMET_OK) return ds;
  const int64_t items = (int64_t)N * (K / group);
  const unsigned grid = (unsigned)((items + 7) / 8);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const __half* Wh = reinterpret_cast<const __half*>(W);
  if (perm)
    pack_weight_f16s_kernel<true, kBf16S><<<grid, 256, 0, st>>>(Wh, ldw, N, K, group, perm,
                                                                 reinterpret_cast<uint8_t*>(Wq),
                                                                 reinterpret_cast<uint16_t*>(Sw16));
  else
    pack_weight_f16s_kernel<false, kBf16S><<<grid, 256, 0, st>>>(Wh, ldw, N, K, group, perm,
                                                                  reinterpret_cast<uint8_t*>(Wq),
                                                                  reinterpret_cast<uint16_t*>(Sw16));
  return check_launch();
}

template <bool kBf16S>
comet_status gemm_h16s(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx, const uint8_t* block_bits,
                       int32_t M, int32_t K, const void* Wq, const void* Sw16, int32_t N, int32_t group, void* Y,
                       int64_t ldy, void* workspace, size_t workspace_bytes, comet_stream_t stream) {
  if (M < 0 || N < 0 || K <= 0 || !block_bits) return COMET_ERR_INVALID_ARG;
  if (K % 128 || N % 128 || (group != 128 && group != K)) return COMET_ERR_SHAPE;
  if (M == 0 || N == 0) return COMET_OK;
  if (!Sw16 || !workspace) return COMET_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(Sw16) & 1) || !aligned16(workspace)) return COMET_ERR_ALIGNMENT;
  const int64_t need = comet_w4ax_gemm_f16s_workspace_bytes(M, N, K, group);
  if (need < 0 || (int64_t)workspace_bytes < need) return COMET_ERR_WORKSPACE;
  const int64_t base = align256(std::max<int64_t>(comet_w4ax_gemm_workspace_bytes(M, N, K), kCounterBytes));
  float* sw32 = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) + base);
  // validate the GEMM's own arguments first (no launch on a failing call)
  if (ldsx < M || ldsx % 4 || ldy < N || ldy % 8) return COMET_ERR_SHAPE;
  if (!Y || !Wq || !Sx) return COMET_ERR_INVALID_ARG;
  int num_sms = 148;
  comet_status ds = device_check(&num_sms);
  if (ds != COMET_OK) return ds;
  const int64_t n = (int64_t)(K / group) * N;
  int64_t grid = (n + 255) / 256;
  if (grid > (int64_t)num_sms * 8) grid = (int64_t)num_sms * 8;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = launch_pdl(widen_scales_kernel<kBf16S>, dim3((unsigned)grid), dim3(256), 0, st,
                             reinterpret_cast<const uint16_t*>(Sw16), n, sw32);
  if (e != cudaSuccess) return cuda_fail(e);
  comet_status ls = check_launch();
  if (ls != COMET_OK) return ls;
  return gemm_common(Xq8, Xq4, Sx, ldsx, block_bits, M, K, Wq, sw32, N, group, Y, ldy, nullptr, workspace,
                     (size_t)base, st);
}
}  // namespace
extern "C" {

comet_status comet_pack_weight_f16s(const void* W, int64_t ldw, int32_t N, int32_t K, const int32_t* perm,
                                    int32_t group, void* Wq, void* Sw16, comet_stream_t stream) {
  return pack_weight_h16s<false>(W, ldw, N, K, perm, group, Wq, Sw16, stream);
}
comet_status comet_pack_weight_bf16s(const void* W, int64_t ldw, int32_t N, int32_t K, const int32_t* perm,
                                     int32_t group, void* Wq, void* Sw16, comet_stream_t stream) {
  return pack_weight_h16s<true>(W, ldw, N, K, perm, group, Wq, Sw16, stream);
}

int64_t comet_w4ax_gemm_f16s_workspace_bytes(int32_t M, int32_t N, int32_t K, int32_t group) {
  const int64_t base = comet_w4ax_gemm_workspace_bytes(M, N, K);
  if (base < 0 || group <= 0 || K % group) return -1;
  return align256(std::max<int64_t>(base, kCounterBytes)) + align256((int64_t)(K / group) * N * 4);
}

comet_status comet_w4ax_gemm_f16s(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx,
                                  const uint8_t* block_bits, int32_t M, int32_t K, const void* Wq, const void* Sw16,
                                  int32_t N, int32_t group, void* Y, int64_t ldy, void* workspace,
                                  size_t workspace_bytes, comet_stream_t stream) {
  return gemm_h16s<false>(Xq8, Xq4, Sx, ldsx, block_bits, M, K, Wq, Sw16, N, group, Y, ldy, workspace,
                          workspace_bytes, stream);
}
comet_status comet_w4ax_gemm_bf16s(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx,
                                   const uint8_t* block_bits, int32_t M, int32_t K, const void* Wq, const void* Sw16,
                                   int32_t N, int32_t group, void* Y, int64_t ldy, void* workspace,
                                   size_t workspace_bytes, comet_stream_t stream) {
  return gemm_h16s<true>(Xq8, Xq4, Sx, ldsx, block_bits, M, K, Wq, Sw16, N, group, Y, ldy, workspace,
                         workspace_bytes, stream);
}


int64_t comet_attention_kv4_workspace_bytes(int32_t T, int32_t H) {
  if (T <= 0 || H <= 0) return -1;
  return (int64_t)H * ((T + kAttChunk - 1) / kAttChunk) * kAttPart * 4;
}

comet_status comet_attention_kv4(const void* q, const void* Kq, const float* Ks, const uint8_t* Kz, const void* Vq,
                                 const float* Vs, const uint8_t* Vz, int32_t T, int32_t H, int32_t D, int32_t group,
                                 float softmax_scale, void* out, void* workspace, size_t workspace_bytes,
                                 comet_stream_t stream) {
  if (T < 0 || H <= 0 || group <= 0) return COMET_ERR_INVALID_ARG;
  if (D != kAttD) return COMET_ERR_SHAPE;
  if (T == 0) return COMET_OK;
  if (!q || !Kq || !Ks || !Kz || !Vq || !Vs || !Vz || !out || !workspace) return COMET_ERR_INVALID_ARG;
  if ((int64_t)workspace_bytes < comet_attention_kv4_workspace_bytes(T, H)) return COMET_ERR_WORKSPACE;
  if (!aligned16(Ks) || !aligned16(Vs) || !aligned16(workspace) || (reinterpret_cast<uintptr_t>(Kz) & 3) ||
      (reinterpret_cast<uintptr_t>(Vz) & 3) || (reinterpret_cast<uintptr_t>(Kq) & 1) ||
      (reinterpret_cast<uintptr_t>(Vq) & 1) || (reinterpret_cast<uintptr_t>(q) & 1) ||
      (reinterpret_cast<uintptr_t>(out) & 1))
    return COMET_ERR_ALIGNMENT;
  comet_status ds = device_check(nullptr);
  if (ds != COMET_OK) return ds;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int S = (T + kAttChunk - 1) / kAttChunk;
  float* part = reinterpret_cast<float*>(workspace);
  attn_kv4_split_kernel<<<dim3((unsigned)H, (unsigned)S), 256, 0, st>>>(
      reinterpret_cast<const __half*>(q), reinterpret_cast<const uint8_t*>(Kq), Ks, Kz,
      reinterpret_cast<const uint8_t*>(Vq), Vs, Vz, T, H, group, softmax_scale, part);
  comet_status ls = check_launch();
  if (ls != COMET_OK) return ls;
  attn_kv4_combine_kernel<<<(unsigned)H, kAttD, 0, st>>>(part, S, reinterpret_cast<__half*>(out));
  return check_launch();
}

const char* comet_status_str(comet_status s) {
  switch (s) {
    case COMET_OK: return "COMET_OK";
    case COMET_ERR_INVALID_ARG: return "COMET_ERR_INVALID_ARG";
    case COMET_ERR_SHAPE: return "COMET_ERR_SHAPE";
    case COMET_ERR_ALIGNMENT: return "COMET_ERR_ALIGNMENT";
    case COMET_ERR_WORKSPACE: return "COMET_ERR_WORKSPACE";
    case COMET_ERR_UNSUPPORTED: return "COMET_ERR_UNSUPPORTED";
    case COMET_ERR_CUDA: return "COMET_ERR_CUDA";
  }
  return "COMET_ERR_UNKNOWN";
}

const char* comet_last_cuda_error(void) { return g_cuda_err; }

// ---- f2: calibration ("identify channels with outliers through data
// sampling") ------------------------------------------------------------------
comet_status comet_calib_absmax(const void* X, int64_t ldx, int32_t M, int32_t K, float* maxabs,
                                comet_stream_t stream) {
  if (M < 0 || K <= 0) return COMET_ERR_INVALID_ARG;
  if (K % 8 || ldx < K || ldx % 8) return COMET_ERR_SHAPE;
  if (M == 0) return COMET_OK;
  if (!X || !maxabs) return COMET_ERR_INVALID_ARG;
  if (!aligned16(X) || (reinterpret_cast<uintptr_t>(maxabs) & 3)) return COMET_ERR_ALIGNMENT;
  comet_status ds = device_check(nullptr);
  if (ds != COMET_OK) return ds;
  // x: 256-channel slices; y: row groups of 8, sized so the grid is ~8 CTAs per SM
  const int xs = (K + 255) / 256;
  int ys = (148 * 8 + xs - 1) / xs;
  if (ys > (M + 7) / 8) ys = (M + 7) / 8;
  const dim3 grid((unsigned)xs, (unsigned)ys);
  calib_absmax_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __half*>(X), ldx, M, K, maxabs);
  return check_launch();
}

comet_status comet_static_act_scales(const float* maxabs, int32_t K, const int32_t* perm, const uint8_t* block_bits,
                                     float* scales, comet_stream_t stream) {
  if (!block_bits || K <= 0) return COMET_ERR_INVALID_ARG;
  if (K % 128 || K > 65536) return COMET_ERR_SHAPE;
  BlockMap map;
  int n8 = 0, n4 = 0;
  if (!build_block_map(block_bits, K / 128, &map, &n8, &n4)) return COMET_ERR_INVALID_ARG;
  if (!maxabs || !scales) return COMET_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(maxabs) & 3) || (reinterpret_cast<uintptr_t>(scales) & 3) ||
      (reinterpret_cast<uintptr_t>(perm) & 3))
    return COMET_ERR_ALIGNMENT;
  comet_status ds = device_check(nullptr);
  if (ds != COMET_OK) return ds;
  static_act_scales_kernel<<<K / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(maxabs, perm, map, scales);
  return check_launch();
}

comet_status comet_quantize_act_static(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                                       const uint8_t* block_bits, const float* scales, int8_t* Xq8, void* Xq4,
                                       float* Sx, int64_t ldsx, comet_stream_t stream) {
  if (M < 0 || K <= 0 || !block_bits) return COMET_ERR_INVALID_ARG;
  if (K % 128 || K > 65536 || ldx < K || ldx % 8 || ldsx < M || ldsx % 4) return COMET_ERR_SHAPE;
  BlockMap map;
  int n8 = 0, n4 = 0;
  if (!build_block_map(block_bits, K / 128, &map, &n8, &n4)) return COMET_ERR_INVALID_ARG;
  if (M == 0) return COMET_OK;
  if (!X || !Sx || !scales || (n8 && !Xq8) || (n4 && !Xq4)) return COMET_ERR_INVALID_ARG;
  if (!aligned16(X) || (n8 && !aligned16(Xq8)) || (n4 && !aligned16(Xq4)) || !aligned16(Sx) ||
      (perm && !aligned16(perm)) || (reinterpret_cast<uintptr_t>(scales) & 3))
    return COMET_ERR_ALIGNMENT;
  comet_status ds = device_check(nullptr);
  if (ds != COMET_OK) return ds;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const __half* Xh = reinterpret_cast<const __half*>(X);
  if (M >= 64 && kQNBuf * K * 2 <= 200 * 1024) {
    // row-staged kernel (as comet_quantize_act), static-scale arithmetic
    const int smem = kQNBuf * K * 2;
    auto kern = perm ? quantize_act_rows_kernel<1, true> : quantize_act_rows_kernel<0, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_fail(e);
    int per_sm = 0;  // one wave of persistent CTAs
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kQThreads, smem);
    if (e != cudaSuccess) return cuda_fail(e);
    if (per_sm < 1) per_sm = 1;
    int num_sms = 148;
    device_check(&num_sms);
    int64_t g = (int64_t)num_sms * per_sm;
    if (g > ldsx) g = ldsx;
    if (perm)
      quantize_act_rows_kernel<1, true><<<(int)g, kQThreads, smem, st>>>(Xh, ldx, M, K / 128, ldsx, perm, map, Xq8,
                                                                      (int64_t)n8 * 128, reinterpret_cast<uint8_t*>(Xq4),
                                                                      (int64_t)n4 * 64, Sx, scales);
    else
      quantize_act_rows_kernel<0, true><<<(int)g, kQThreads, smem, st>>>(Xh, ldx, M, K / 128, ldsx, perm, map, Xq8,
                                                                       (int64_t)n8 * 128, reinterpret_cast<uint8_t*>(Xq4),
                                                                       (int64_t)n4 * 64, Sx, scales);
    return check_launch();
  }
  const dim3 grid((unsigned)((ldsx + 7) / 8), (unsigned)((K / 128 + 1) / 2));
  if (perm)
    quantize_act_static_kernel<true><<<grid, 256, 0, st>>>(Xh, ldx, M, K / 128, ldsx, perm, map, scales, Xq8,
                                                            (int64_t)n8 * 128, reinterpret_cast<uint8_t*>(Xq4),
                                                            (int64_t)n4 * 64, Sx);
  else
    quantize_act_static_kernel<false><<<grid, 256, 0, st>>>(Xh, ldx, M, K / 128, ldsx, perm, map, scales, Xq8,
                                                             (int64_t)n8 * 128, reinterpret_cast<uint8_t*>(Xq4),
                                                             (int64_t)n4 * 64, Sx);
  return check_launch();
}

comet_status comet_fmpq_map(const float* score, int32_t K, float theta, int32_t* perm, uint8_t* block_bits,
                            int32_t* n_outliers) {
  if (!score || !perm || !block_bits || K <= 0 || !(theta > 1.0f)) return COMET_ERR_INVALID_ARG;
  if (K % COMET_BLOCK) return COMET_ERR_SHAPE;
  for (int32_t c = 0; c < K; ++c)
    if (!(score[c] >= 0.0f) || score[c] == INFINITY) return COMET_ERR_INVALID_ARG;  // non-finite or negative
  std::vector<float> sorted(score, score + K);
  std::sort(sorted.begin(), sorted.end());
  const float median = sorted[(K - 1) / 2];  // lower middle for even K
  const float thr = theta * median;
  std::vector<int32_t> out, rest;
  for (int32_t c = 0; c < K; ++c) (score[c] > thr ? out : rest).push_back(c);
  // outliers first by descending score, ties by ascending channel; the rest stable
  std::stable_sort(out.begin(), out.end(), [&](int32_t a, int32_t b) { return score[a] > score[b]; });
  int32_t i = 0;
  for (int32_t c : out) perm[i++] = c;
  for (int32_t c : rest) perm[i++] = c;
  const int32_t n8 = ((int32_t)out.size() + COMET_BLOCK - 1) / COMET_BLOCK;
  for (int32_t b = 0; b < K / COMET_BLOCK; ++b) block_bits[b] = b < n8 ? 8 : 4;
  if (n_outliers) *n_outliers = (int32_t)out.size();
  return COMET_OK;
}

// ---- f3: KV4 cache ("channel-wise asymmetric INT4 group
// quantization for the KV cache") ---------------------------------------------
comet_status comet_quantize_kv(const void* KV, int64_t ld, int32_t T, int32_t C, int32_t group, void* Q,
                               float* scale, uint8_t* zp, comet_stream_t stream) {
  if (T < 0 || C <= 0 || group <= 0) return COMET_ERR_INVALID_ARG;
  if (C % 2 || ld < C || ld % 2) return COMET_ERR_SHAPE;
  if (T == 0) return COMET_OK;
  if (!KV || !Q || !scale || !zp) return COMET_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(KV) & 3) || (reinterpret_cast<uintptr_t>(scale) & 3)) return COMET_ERR_ALIGNMENT;
  comet_status ds = device_check(nullptr);
  if (ds != COMET_OK) return ds;
  if (C % 8 == 0 && ld % 8 == 0 && !(reinterpret_cast<uintptr_t>(KV) & 15) && !(reinterpret_cast<uintptr_t>(Q) & 3)) {
    const dim3 gv((unsigned)((C + 63) / 64), (unsigned)((T + group - 1) / group));
    kv4_quantize_v_kernel<<<gv, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const __half*>(KV), ld, T, C, group, reinterpret_cast<uint8_t*>(Q), scale, zp);
    return check_launch();
  }
  const dim3 grid((unsigned)((C / 2 + 63) / 64), (unsigned)((T + group - 1) / group));
  kv4_quantize_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __half*>(KV), ld, T, C, group, reinterpret_cast<uint8_t*>(Q), scale, zp);
  return check_launch();
}

comet_status comet_dequantize_kv(const void* Q, const float* scale, const uint8_t* zp, int32_t T, int32_t C,
                                 int32_t group, void* out, int64_t ldo, comet_stream_t stream) {
  if (T < 0 || C <= 0 || group <= 0) return COMET_ERR_INVALID_ARG;
  if (C % 2 || ldo < C || ldo % 2) return COMET_ERR_SHAPE;
  if (T == 0) return COMET_OK;
  if (!Q || !scale || !zp || !out) return COMET_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(out) & 3) || (reinterpret_cast<uintptr_t>(scale) & 3)) return COMET_ERR_ALIGNMENT;
  comet_status ds = device_check(nullptr);
  if (ds != COMET_OK) return ds;
  if (C % 16 == 0 && ldo % 8 == 0 && !(reinterpret_cast<uintptr_t>(out) & 15) && !(reinterpret_cast<uintptr_t>(Q) & 7) &&
      !(reinterpret_cast<uintptr_t>(scale) & 15) && !(reinterpret_cast<uintptr_t>(zp) & 15)) {
    const int64_t n = (int64_t)T * (C / 16);
    kv4_dequantize_v_kernel<<<(unsigned)((n + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const uint8_t*>(Q), scale, zp, T, C, group, reinterpret_cast<__half*>(out), ldo);
    return check_launch();
  }
  const int64_t units = (int64_t)T * (C / 2);
  kv4_dequantize_kernel<<<(unsigned)((units + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint8_t*>(Q), scale, zp, T, C, group, reinterpret_cast<__half*>(out), ldo);
  return check_launch();
}

// debug only (not part of comet.h): enable/read per-CTA timestamps of the
// decode kernel, [start_ns, end_ns, smid] x n
int comet_debug_cta_times(int enable, unsigned long long* host, int n) {
  int on = enable;
  if (cudaMemcpyToSymbol(g_cta_times_on, &on, sizeof(int)) != cudaSuccess) return -1;
  if (on) {  // fresh event table for the traced run
    static const unsigned long long zeros[32 * 64] = {};
    if (cudaMemcpyToSymbol(g_trace, zeros, sizeof(zeros)) != cudaSuccess) return -1;
  }
  if (host && n > 0) {
    if (n > 1024) n = 1024;
    if (cudaMemcpyFromSymbol(host, g_cta_times, sizeof(unsigned long long) * 3 * n) != cudaSuccess) return -1;
  }
  return 0;
}
int comet_debug_role_cycles(unsigned long long* host16) {
  return cudaMemcpyFromSymbol(host16, g_role_cycles, sizeof(unsigned long long) * 16) == cudaSuccess ? 0 : -1;
}
int comet_debug_trace(unsigned long long* host2048) {  // 32 x 64 entries
  return cudaMemcpyFromSymbol(host2048, g_trace, sizeof(unsigned long long) * 2048) == cudaSuccess ? 0 : -1;
}
int64_t comet_launch_count(void) { return g_launches.load(); }
// Schedule ablation (tools/a7_ablation.py): the prefill kernel's grid as n CTA
// pairs (n > 74: more pairs than SM pairs, each taking one tile, the
// hardware scheduling them in waves -- the paper's non-persistent "static"
// schedule); 0 restores the persistent grid.  Results are identical.
int comet_debug_set_pf_clusters(int n) {
  g_pf_clusters.store(n < 0 ? 0 : n);
  return 0;
}
// Raster ablation: token tiles per group of the prefill tile order (0 = the
// L2-budget rule).  Results are identical.
int comet_debug_set_pf_group(int n) {
  g_pf_group.store(n < 0 ? 0 : n);
  return 0;
}
// Kernel-choice sweep: M above which the CTA-pair prefill kernel runs instead
// of the decode kernel (0 = the product rule).  Results agree within the Y
// tolerance (the INT32 accumulators are identical).
int comet_debug_set_prefill_min_m(int m) {
  g_pf_min_m.store(m < 0 ? 0 : m);
  return 0;
}

}  // extern "C"
