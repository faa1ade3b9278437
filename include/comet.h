/*
 * comet.h -- C ABI of libcomet.so, the B200 (sm_100a) implementation of
 * COMET's W4Ax mixed-precision GEMM (arXiv 2410.12168; PAPER.md cited as
 * P:L<line> §<section>).
 *
 * The paper's problem statement is the linear layer O = WX with 4-bit
 * weights and FMPQ activations (§5): activations are split along the
 * channel axis into blocks of k = 128 channels (§3.2); outlier
 * channels are clustered by a channel permutation into a few blocks
 * (§3.2) which are quantized to INT8, all other blocks to INT4; the
 * weight reduction axis is permuted identically.  The kernel is
 * "a standalone .so dynamic library" with "a set of C++ APIs"; this
 * header is that API as plain C.
 *
 * Conventions (all entry points):
 *   - Tensor pointers are DEVICE pointers owned by the caller unless stated
 *     otherwise; nothing here allocates, frees or synchronizes.  Work is
 *     enqueued on `stream` (a cudaStream_t; NULL = legacy default stream).
 *   - Every argument is validated on the host before any launch; a call that
 *     returns an error has no side effects.
 *   - block size is fixed at COMET_BLOCK = 128 channels; K % 128 == 0.
 *   - `block_bits` is a HOST array of K/128 entries, each 4 or 8 (the static
 *     per-layer precision mask from calibration); the same array and
 *     the same `perm` must be given to comet_pack_weight/comet_quantize_act
 *     and comet_w4ax_gemm of one layer.
 *   - `perm` is a DEVICE int32[K] with perm[new] = old (a bijection on
 *     [0,K)), or NULL for the identity.
 *   - Inputs must be finite; non-finite input gives unspecified output.
 *   - Results are deterministic (same inputs, shape and device -> identical
 *     bits); no floating-point atomics are used.
 *
 * Data layouts (row-major; "bytes" are leading dimensions in bytes):
 *   X   fp16 [M x K], row stride ldx elements (ldx >= K, ldx % 8 == 0).
 *   Xq8 int8 [M x K8], K8 = 128 * #INT8 blocks; INT8 block b occupies
 *       columns [128*r8(b), 128*r8(b)+128) where r8(b) = number of INT8
 *       blocks before b.
 *   Xq4 packed INT4 [M x K4/2 bytes], K4 = 128 * #INT4 blocks; INT4 block b
 *       occupies bytes [64*r4(b), 64*r4(b)+64).  Nibble order: every 8
 *       consecutive elements e0..e7 form one little-endian 32-bit word whose
 *       byte j = (e_j & 0xF) | (e_{j+4} & 0xF) << 4 -- the 32-bit form of the
 *       paper's W1<->W2 "location switch" (§4.3), so that
 *       (w << 4) & 0xF0F0F0F0 and w & 0xF0F0F0F0 are 16*e0..3 and 16*e4..7
 *       as int8 ("zero extension ... multiplied by 16").
 *   Sx  fp32 [K/128 x ldsx], Sx[b*ldsx + m] = scale of row m, block b;
 *       ldsx >= M, ldsx % 4 == 0; entries m in [M, ldsx) are written as 1.0.
 *   Wq  packed INT4, N*K/2 bytes, same nibble order, K on the permuted axis,
 *       TILED for contiguous streaming (the B200 counterpart of the paper's
 *       offline weight interleave): the slab of output channels
 *       [128*t, 128*t+128) x K-block b (128 rows x 64 bytes) is contiguous at
 *       byte offset (t*(K/128) + b)*8192; inside it, 16-byte chunk c
 *       (channels 32c..32c+31 of the block) of row r is stored at byte
 *       r*64 + ((c ^ ((r >> 1) & 3)) << 4).  Requires N % 128 == 0.
 *   Sw  fp32 [K/group x N], Sw[j*N + n] = scale of output channel n, group j.
 *   Y   fp16 [M x N], row stride ldy elements (ldy >= N, ldy % 8 == 0).
 * Quantization (all blocks, weights and activations): symmetric absmax,
 * a = max|x|, s = a/qmax, r = qmax/a (IEEE fp32), q = round_half_away(x*r),
 * qmax = 7 (INT4) or 127 (INT8); an all-zero block has s = 1, q = 0.
 */
#ifndef COMET_H_
#define COMET_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COMET_BLOCK 128

typedef enum {
  COMET_OK = 0,
  COMET_ERR_INVALID_ARG = 1, /* NULL where required, M/N/K < 0, bad block_bits entry */
  COMET_ERR_SHAPE = 2,       /* K%128, N%128, group not in {128, K}, ld too small, K > 65536 */
  COMET_ERR_ALIGNMENT = 3,   /* pointer or leading dimension not 16-byte aligned */
  COMET_ERR_WORKSPACE = 4,   /* workspace/scratch smaller than the size query returns */
  COMET_ERR_UNSUPPORTED = 5, /* device is not sm_100 (B200) */
  COMET_ERR_CUDA = 6         /* CUDA launch/runtime error (comet_last_cuda_error()) */
} comet_status;

typedef void* comet_stream_t; /* cudaStream_t */

/* ---- size helpers (host, pure; -1 on invalid arguments) ---------------- */
int64_t comet_act_plane8_bytes(int32_t M, int32_t K, const uint8_t* block_bits); /* M*K8   */
int64_t comet_act_plane4_bytes(int32_t M, int32_t K, const uint8_t* block_bits); /* M*K4/2 */
int64_t comet_act_ldsx(int32_t M);                                               /* roundup(M,4) */
/* device workspace comet_w4ax_gemm needs: 64 KiB of stream-K tile counters
 * (decode, M <= 128) followed by the split-K partials (decode) or by the
 * INT4 token plane re-encoded as e4m3 bytes, M*K bytes at most, and its
 * per-(block, row) corrections (prefill, M > 128) */
int64_t comet_w4ax_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K);
/* device scratch comet_w4ax_linear needs (planes + scales + gemm workspace) */
int64_t comet_w4ax_linear_scratch_bytes(int32_t M, int32_t N, int32_t K, const uint8_t* block_bits);

/* ---- a0: offline weight preparation -------------------
 * W fp16 [N x K] (row stride ldw) -> Wq packed INT4 (tiled layout above),
 * Sw fp32 [K/group x N].  N % 128 == 0.  The K axis is permuted by `perm` first (weights are
 * permuted like the activations), then quantized per (n, group of
 * `group` consecutive permuted channels), group in {128, K}. */
comet_status comet_pack_weight(const void* W, int64_t ldw, int32_t N, int32_t K, const int32_t* perm,
                               int32_t group, void* Wq, float* Sw, comet_stream_t stream);

/* ---- a1+a2: FMPQ activation quantization --------------
 * X fp16 [M x K] -> Xq8, Xq4, Sx (layouts above).  The channel permutation
 * is fused (gather) into the quantizer.  Xq8 may be NULL iff K8 == 0 and
 * Xq4 may be NULL iff K4 == 0.  M == 0 is a no-op. */
comet_status comet_quantize_act(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                                const uint8_t* block_bits, int8_t* Xq8, void* Xq4, float* Sx, int64_t ldsx,
                                comet_stream_t stream);
/* f4 variant ("BF16 activations"): identical to
 * comet_quantize_act except that X holds bf16 values (same shape, stride and
 * alignment rules); every bf16 value converts to fp32 exactly, after which
 * the arithmetic, the planes and Sx are those of comet_quantize_act on the
 * same fp32 values. */
comet_status comet_quantize_act_bf16(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                                     const uint8_t* block_bits, int8_t* Xq8, void* Xq4, float* Sx, int64_t ldsx,
                                     comet_stream_t stream);

/* ---- a3..a8: the W4Ax GEMM -------------------------
 * Y[m,n] = sum_b Sx[b,m] * Sw[g(b),n] * sum_{i in block b} xq[m,i]*wq[n,i]
 * with the integer block sums exact (INT32) and the scale applied per block
 * in fp32 ("divide by 16 in the scaling parameter"), rounded once to
 * fp16.  N % 128 == 0.  workspace: device memory of at least
 * comet_w4ax_gemm_workspace_bytes(M, N, K) bytes (16-byte aligned) whose first 64 KiB must be
 * zero on the first use (the kernel leaves it zero again); it may be NULL
 * only if that size is 0.
 * Stream ordering: every library kernel is launched with programmatic stream
 * serialization and executes griddepcontrol.wait before touching memory a
 * preceding kernel may use; the prefill GEMM (M > 128, or M > 64 with
 * per-channel scales) signals griddepcontrol.launch_dependents after its
 * prologue, so a CALLER kernel launched right after it with programmatic
 * stream serialization must itself wait (griddepcontrol.wait /
 * cudaGridDependencySynchronize) before reading Y.  Ordinary launches,
 * events and copies are unaffected. */
comet_status comet_w4ax_gemm(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx,
                             const uint8_t* block_bits, int32_t M, int32_t K, const void* Wq, const float* Sw,
                             int32_t N, int32_t group, void* Y, int64_t ldy, void* workspace,
                             size_t workspace_bytes, comet_stream_t stream);

/* ---- (e) N-sharded tensor parallelism: reassembly of the gathered Y ------
 * BJ north_star: weights are sharded by output channel (N) over P ranks,
 * each rank computes Y_r [M x per] (per = N/P rounded up to 128) and an
 * all-gather (NCCL) leaves Yall = [P x M x per] fp16, rank-major, on every
 * rank.  This writes Y [M x N] (row stride ldy) with
 * Y[m, r*per + j] = Yall[r, m, j] for r*per + j < N.  per % 128 == 0,
 * N % 128 == 0, P*per >= N, ldy >= N, ldy % 8 == 0; Yall and Y 16-byte
 * aligned and not overlapping. */
comet_status comet_gather_shards(const void* Yall, int32_t P, int32_t M, int32_t per, int32_t N, void* Y,
                                 int64_t ldy, comet_stream_t stream);

/* ---- f1: GEMM with the all-gather fused into its epilogue (§4.4:
 * "the all-gather ... overlapped with the GEMM", BJ north_star) ------------
 * Rank r of P computes its N-shard Y_r = comet_w4ax_gemm(...) [M x N] and
 * the epilogue writes every Y_r element into ALL nY destinations: Ys[i] is a
 * full-width output [M x ldy] fp16 (row stride ldy, ldy >= col0 + N,
 * ldy % 8 == 0) and Y_r lands in its columns [col0, col0 + N) (col0 % 8 ==
 * 0, normally r * N).  Ys[0] is this GPU's copy; Ys[1 ..] are other ranks'
 * copies mapped into this process (CUDA IPC / symmetric memory over NVLink:
 * the stores leave this GPU as P2P writes from the TMA engine, tile by tile,
 * overlapping the remaining tiles' MMAs).  1 <= nY <= 8; every Ys[i] 16-byte
 * aligned and writable from the current device.  The call only enqueues:
 * the caller's single cross-rank barrier after it (e.g. the symmetric-memory
 * barrier) makes every rank's copy complete.  Other arguments as for
 * comet_w4ax_gemm. */
comet_status comet_w4ax_gemm_allgather(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx,
                                       const uint8_t* block_bits, int32_t M, int32_t K, const void* Wq,
                                       const float* Sw, int32_t N, int32_t group, void* const* Ys, int32_t nY,
                                       int64_t ldy, int64_t col0, void* workspace, size_t workspace_bytes,
                                       comet_stream_t stream);
/* the whole layer (quantize_act + the fused GEMM above); X and every Ys[i]
 * DEVICE pointers (COMET_ERR_INVALID_ARG for host buffers); scratch as for
 * comet_w4ax_linear. */
comet_status comet_w4ax_linear_allgather(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                                         const uint8_t* block_bits, const void* Wq, const float* Sw, int32_t N,
                                         int32_t group, void* const* Ys, int32_t nY, int64_t ldy, int64_t col0,
                                         void* scratch, size_t scratch_bytes, comet_stream_t stream);

/* ---- test/debug: per-block INT32 accumulators ---------------------------
 * Acc int32 [K/128 x M x N]: Acc[(b*M + m)*N + n] = sum_{i in block b}
 * xq[m,i]*wq[n,i] in LOGICAL units (the x16 zero-extension factor and, in
 * the prefill kernel, the e4m3 offset term removed), computed by the same
 * tcgen05 pipeline as comet_w4ax_gemm; workspace as for comet_w4ax_gemm. */
comet_status comet_w4ax_gemm_acc_i32(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx,
                                     const uint8_t* block_bits, int32_t M, int32_t K, const void* Wq,
                                     const float* Sw, int32_t N, int32_t group, int32_t* Acc, void* workspace,
                                     size_t workspace_bytes, comet_stream_t stream);

/* ---- the whole linear layer (user call): quantize_act + w4ax_gemm ------
 * X and Y may be HOST (pinned or pageable) or DEVICE pointers.  Device X and
 * Y: everything is enqueued on `stream`; at prefill sizes the quantizer
 * writes the GEMM's e4m3 token operand directly (results identical to
 * comet_quantize_act + comet_w4ax_gemm).  Host buffers: the rows are split
 * into chunks (>= 1024 rows, at most 8) whose host->device copy, layer and
 * device->host copy run as a pipeline on two library-internal copy streams
 * ordered after the caller's earlier work on `stream` (X: M*K*2 bytes in,
 * Y: M*N*2 bytes out); later work on `stream` is ordered after the copies.
 * scratch: device memory of at least comet_w4ax_linear_scratch_bytes(M, N,
 * K, block_bits) bytes, first 64 KiB zero on first use.  The call does not
 * synchronize: with host buffers, X must stay unchanged and Y unread until
 * `stream` has been synchronized (as for cudaMemcpyAsync).  The input copies
 * of a host-buffer call that directly follows another host-buffer call on the
 * same stream start once that call's compute is done (not its output
 * copies, unless this call's staged X overlaps the scratch bytes they read),
 * so consecutive layers overlap H2D and D2H; work enqueued on `stream`
 * between two such calls must not write either call's scratch. */
comet_status comet_w4ax_linear(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                               const uint8_t* block_bits, const void* Wq, const float* Sw, int32_t N, int32_t group,
                               void* Y, int64_t ldy, void* scratch, size_t scratch_bytes, comet_stream_t stream);

/* ---- f2: FMPQ calibration (§3.2: outlier channels are identified
 * "through data sampling", then clustered by a permutation) ---------------
 * comet_calib_absmax: maxabs[c] = max(maxabs[c], max_m |X[m, c]|) over the
 * calibration rows X fp16 [M x K] (DEVICE; row stride ldx, ldx % 8 == 0,
 * K % 8 == 0); maxabs is a DEVICE fp32[K] the caller zero-initialises once
 * and may accumulate over several batches (exact, order-independent).
 * comet_fmpq_map (HOST, pure): from per-channel scores (maxabs, HOST fp32[K],
 * K % 128 == 0) and theta > 1: median = lower middle of the sorted scores;
 * channel c is an outlier iff score[c] > theta * median; perm (HOST
 * int32[K], perm[new] = old) puts the outliers first by descending score
 * (ties: ascending channel), the other channels after them in their original
 * order; block_bits (HOST uint8[K/128]) = 8 for the ceil(#outliers/128)
 * leading blocks, 4 otherwise (SPEC S:L139-165 rule, theta = 8 there);
 * *n_outliers (optional) = number of outliers. */
comet_status comet_calib_absmax(const void* X, int64_t ldx, int32_t M, int32_t K, float* maxabs,
                                comet_stream_t stream);
comet_status comet_fmpq_map(const float* score, int32_t K, float theta, int32_t* perm, uint8_t* block_bits,
                            int32_t* n_outliers);

/* ---- f3: KV4 cache (§3.2, §6.1: "channel-wise asymmetric
 * INT4 group quantization for the KV cache") ------------------------------
 * KV fp16 [T x C] (DEVICE; tokens x head-dim channels, row stride ld, C and
 * ld even).  Per (channel c, group j of `group` consecutive tokens):
 *   mn, mx = min, max over the group; if mn == mx == v: scale = |v| (1 if
 *   v == 0), zp = (v < 0); else lo = min(mn, 0), hi = max(mx, 0),
 *   scale = (hi - lo)/15, zp = clamp(rha(-lo / scale), 0, 15);
 *   q = clamp(rha(x / scale) + zp, 0, 15)
 * (IEEE fp32 division, rha = round half away from zero).
 * Q: DEVICE packed [T x C/2] bytes, byte (t, j) = q[t,2j] | q[t,2j+1] << 4;
 * scale fp32 / zp uint8: DEVICE [ceil(T/group) x C].
 * comet_dequantize_kv: out fp16 [T x C] (row stride ldo) = fp16_rn((q - zp) *
 * scale), the dequantisation an attention kernel applies to the cache. */
comet_status comet_quantize_kv(const void* KV, int64_t ld, int32_t T, int32_t C, int32_t group, void* Q,
                               float* scale, uint8_t* zp, comet_stream_t stream);
comet_status comet_dequantize_kv(const void* Q, const float* scale, const uint8_t* zp, int32_t T, int32_t C,
                                 int32_t group, void* out, int64_t ldo, comet_stream_t stream);

/* ---- f4: FP16 weight-scale storage ("the group size is 128 and each
 * group has one FP16 scale factor") ------------------------
 * comet_pack_weight_f16s: as comet_pack_weight (same Wq tiled layout, group
 *   in {128, K}) but the scale of (row n, group j) is stored as fp16 and is
 *   the one the weights are quantized with: a = max |w| over the group,
 *   s = fp16_rn(fp32(a / 7)) (a == 0 -> 1; a nonzero s that underflows ->
 *   2^-24), q = clamp(rha(fp32(w / s)), -7, 7).  Sw16: DEVICE fp16 [K/group x N].
 * comet_w4ax_gemm_f16s: comet_w4ax_gemm with fp16 weight scales (stored at
 *   half the bytes, widened to fp32 per call into the workspace: at least
 *   comet_w4ax_gemm_f16s_workspace_bytes(M, N, K, group) bytes, first 64 KiB
 *   zero on first use).  Results equal comet_w4ax_gemm on the fp32 values of
 *   the fp16 scales. */
comet_status comet_pack_weight_f16s(const void* W, int64_t ldw, int32_t N, int32_t K, const int32_t* perm,
                                    int32_t group, void* Wq, void* Sw16, comet_stream_t stream);
int64_t comet_w4ax_gemm_f16s_workspace_bytes(int32_t M, int32_t N, int32_t K, int32_t group);
comet_status comet_w4ax_gemm_f16s(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx,
                                  const uint8_t* block_bits, int32_t M, int32_t K, const void* Wq, const void* Sw16,
                                  int32_t N, int32_t group, void* Y, int64_t ldy, void* workspace,
                                  size_t workspace_bytes, comet_stream_t stream);
/* BF16 storage (SURVEY 8(f) f4 "FP16/BF16 scale storage"): identical to the
 * fp16 pair above with s = bf16_rn(fp32(a / 7)) (a == 0 -> 1; bf16 keeps
 * fp32's exponent range, so no underflow clamp) stored as bf16 bits [K/group
 * x N]; comet_w4ax_gemm_bf16s takes the workspace of
 * comet_w4ax_gemm_f16s_workspace_bytes and equals comet_w4ax_gemm on the
 * fp32 values of the bf16 scales. */
comet_status comet_pack_weight_bf16s(const void* W, int64_t ldw, int32_t N, int32_t K, const int32_t* perm,
                                     int32_t group, void* Wq, void* Sw16, comet_stream_t stream);
comet_status comet_w4ax_gemm_bf16s(const int8_t* Xq8, const void* Xq4, const float* Sx, int64_t ldsx,
                                   const uint8_t* block_bits, int32_t M, int32_t K, const void* Wq, const void* Sw16,
                                   int32_t N, int32_t group, void* Y, int64_t ldy, void* workspace,
                                   size_t workspace_bytes, comet_stream_t stream);

/* ---- f3: attention over the KV4 cache ("dequant-in-attention") ----------
 * One decode query per head (§3.2: the KV4 cache feeds the
 * memory-bound activation-activation operator): for head h of H (D = 128
 * channels each, C = 128 H),
 *   o[h] = softmax_t(softmax_scale * q[h] . K^[t, h]) . V^[t, h]
 * where K^, V^ = fp16_rn((q - zp) * scale) are the caches produced by
 * comet_quantize_kv on [T x C] (Kq/Vq packed [T x C/2], Ks/Vs fp32 and Kz/Vz
 * uint8 [ceil(T/group) x C]), dequantised on the fly (never written out).
 * q: fp16 [H x 128]; out: fp16 [H x 128]; D must be 128.  workspace: DEVICE,
 * at least comet_attention_kv4_workspace_bytes(T, H) bytes (per-split
 * partials), 16-byte aligned; Ks/Vs 16-byte, Kz/Vz 4-byte aligned.  Softmax
 * and sums in fp32 (expf), result rounded once to fp16. */
int64_t comet_attention_kv4_workspace_bytes(int32_t T, int32_t H);
comet_status comet_attention_kv4(const void* q, const void* Kq, const float* Ks, const uint8_t* Kz, const void* Vq,
                                 const float* Vs, const uint8_t* Vz, int32_t T, int32_t H, int32_t D, int32_t group,
                                 float softmax_scale, void* out, void* workspace, size_t workspace_bytes,
                                 comet_stream_t stream);

/* ---- f4: static per-block activation scales (SPEC
 * S:L157-165 "per-block QuantParams computed from the permuted channels'
 * pooled min/max at the block's bit width, symmetric scheme") ----
 * comet_static_act_scales: scales (DEVICE fp32[K/128]) with
 *   scales[b] = fp32(pool_b / qmax_b), qmax_b = 127 (INT8 block) or 7,
 *   pool_b = max over the block's channels i (permuted axis) of
 *   maxabs[perm[128 b + i]] (maxabs: DEVICE fp32[K] from comet_calib_absmax;
 *   perm as in comet_quantize_act, NULL = identity), 1 if pool_b == 0.
 * comet_quantize_act_static: as comet_quantize_act (same arguments, planes,
 *   Sx layout) but with the calibrated scales instead of the runtime absmax:
 *   q = clamp(rha(fp32(x / scales[b])), -qmax_b, qmax_b) (IEEE division,
 *   round half away from zero; inputs beyond the calibrated range clamp),
 *   Sx[b*ldsx + m] = scales[b] -- the output feeds comet_w4ax_gemm as is.
 *   scales: DEVICE fp32[K/128], every entry > 0. */
comet_status comet_static_act_scales(const float* maxabs, int32_t K, const int32_t* perm, const uint8_t* block_bits,
                                     float* scales, comet_stream_t stream);
comet_status comet_quantize_act_static(const void* X, int64_t ldx, int32_t M, int32_t K, const int32_t* perm,
                                       const uint8_t* block_bits, const float* scales, int8_t* Xq8, void* Xq4,
                                       float* Sx, int64_t ldsx, comet_stream_t stream);

const char* comet_status_str(comet_status s);
const char* comet_last_cuda_error(void);
/* number of kernel launches this library issued since load (host counter) */
int64_t comet_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* COMET_H_ */
