// gemm.cuh -- definitions shared by the two W4Ax GEMM kernels (§4,
// P:L321 §5):
//   gemm_decode.cuh  M <= 128 tokens: swap-AB, weights as the TMEM A operand,
//                    stream-K over (tile, K-block) units (HBM-bound regime);
//   gemm_pf.cuh      M > 128 tokens: persistent CTA-pair (cta_group::2) tiles
//                    of 256 tokens x 192 weight rows (tensor-bound regime).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "quantize.cuh"
#include "sm100.cuh"

namespace comet {

#ifndef COMET_MAX_YPEERS
#define COMET_MAX_YPEERS 7
#endif
constexpr int kMaxYPeers = COMET_MAX_YPEERS;  // f1: up to 8 ranks (this one + 7 peers)

struct GemmArgs {
  int M, N, K, nb;
  int64_t ldsx, ldy;
  const float* Sx;
  const float* Sw;
  int group_blocks;  // 128-blocks per weight-scale group: 1 (group 128) or nb (group K)
  __half* Y;
  const uint8_t* Wq;  // tiled packed weights: slab (tile, block) at (tile * nb + block) * 8192
  int32_t* Acc;  // debug output (per-block INT32, logical units)
  const float* CX;  // prefill: 8 * sum(xq) per (INT4 block rank, row) [n4 x ldsx]
  float* ws_partial;
  int* ws_counter;
  int splits;
  // f1 (fused all-gather): further destinations of every Y element
  // (peer GPUs' copies of the full output, P2P-mapped), same offsets as Y
  int npeer;
  __half* Ypeer[kMaxYPeers];
};
// the prefill kernel's TMA-store maps of those destinations
struct YPeerMaps {
  CUtensorMap m[kMaxYPeers];
  int n;
};

// ---- debug instrumentation ------------------------------------------------
// Per-CTA start/end stamps are always compiled (once per CTA). Per-role cycle
// counters and per-step event traces exist only in a -DCOMET_TRACE build
// (tools/gemm_sweep.py builds one): even disabled, their code in the hot loops
// cost the prefill kernel ~9% (register pressure).
#ifdef COMET_TRACE
constexpr bool kTraceBuild = true;
#else
constexpr bool kTraceBuild = false;
#endif
// debug: per-CTA [start, end, smid] globaltimer stamps (comet_debug_cta_times)
__device__ unsigned long long g_cta_times[3 * 1024];
__device__ int g_cta_times_on;
DEVI unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
DEVI unsigned long long clk64() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
// debug: per-role cycles of CTA g_cta_times_on - 1:
// [role][0..3] = wait A, wait B, total, stream-K fixup (epilogue)
__device__ unsigned long long g_role_cycles[4][4];
struct RoleTimer {
  bool on;
  unsigned long long t0, w[3];
  DEVI RoleTimer(bool enabled) : on(kTraceBuild && enabled), t0(on ? clk64() : 0) { w[0] = w[1] = w[2] = 0; }
  DEVI unsigned long long now() const { return on ? clk64() : 0; }
  DEVI void add_fixup(unsigned long long since) {
    if (on) w[2] += clk64() - since;
  }
  DEVI void wait(uint64_t* bar, uint32_t parity, int k) {
    if (!on) {
      mbar_wait(bar, parity);
      return;
    }
    const unsigned long long a = clk64();
    mbar_wait(bar, parity);
    w[k] += clk64() - a;
  }
  DEVI void flush(int role) {
    if (!on) return;
    g_role_cycles[role][0] = w[0];
    g_role_cycles[role][1] = w[1];
    g_role_cycles[role][2] = clk64() - t0;
    g_role_cycles[role][3] = w[2];
  }
};
// debug: per-unit event clocks of the traced CTA: [event][unit], unit < 64
// (0 W issue, 1 X issue, 2 data arrived, 3 expanded, 4 MMA issued,
//  5 accumulator ready, 6 accumulator released, 7 unit retired,
//  8 epilogue iteration top, 9 epilogue scales ready)
__device__ unsigned long long g_trace[32][64];
DEVI void trace(bool on, int ev, int i) {
  if (kTraceBuild && on && i < 64) g_trace[ev][i] = clk64();
}
// per-warp clocks of one step: g_trace[row][slot]
DEVI void trace_at(bool on, int row, int slot) {
  if (kTraceBuild && on) g_trace[row][slot] = clk64();
}
DEVI uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

}  // namespace comet
