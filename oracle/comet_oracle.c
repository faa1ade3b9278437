/*
 * comet_oracle.c -- plain, slow, obviously-correct CPU oracle for the COMET
 * W4Ax path (FMPQ activation quantization + INT4 weight packing + per-block
 * integer GEMM + dequant), written from the paper (arXiv 2410.12168,
 * /root/reference/PAPER.md, cited as P:L<line> §<section>).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * in paper_2410_12168_b200/csrc/ and never includes anything from there.
 *
 * Arithmetic:
 *   - quantization scale/reciprocal/product are IEEE fp32 (reading A-6: the
 *     paper fixes no precision; s = a/qmax, r = qmax/a, v = x*r, all fp32);
 *   - rounding is round-half-away-from-zero (reading A-4, C roundf);
 *   - the GEMM accumulates exact integers per 128-channel block (P:L248,
 *     "accumulate the compute results of different tiles");
 *   - dequantization sums the per-block products in fp64, blocks ascending
 *     (P:L248), and rounds once to fp16 (round-to-nearest-even).
 *
 * Every function is a direct transcription of a definition; there is no
 * blocking, fusion or reordering.  Parity pins: tests/test_oracle.py.
 *
 * Build: gcc -O2 -fopenmp -fPIC -shared (NO -ffast-math: fp32 semantics
 * must be IEEE; x86-64 SSE gives FLT_EVAL_METHOD == 0).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_ERR_INPUT 1 /* non-finite value, bad bits entry, bad perm */
#define ORACLE_ERR_SHAPE 2 /* block size / group / leading dimension */

/* ------------------------------------------------------------------ fp16 */

/* IEEE binary16 bits -> float, exact (every half is a float). */
float oracle_half_to_float(uint16_t h) {
  int sign = (h >> 15) & 1;
  int e = (h >> 10) & 0x1F;
  int m = h & 0x3FF;
  float v;
  if (e == 0) {
    v = ldexpf((float)m, -24); /* subnormal: m * 2^-24 */
  } else if (e == 31) {
    v = m ? NAN : INFINITY;
  } else {
    v = ldexpf((float)(1024 + m), e - 25); /* (1.m) * 2^(e-15) */
  }
  return sign ? -v : v;
}

/* double -> IEEE binary16 bits, round to nearest, ties to even; values that
 * round beyond the largest finite half become +-inf (IEEE overflow). */
uint16_t oracle_double_to_half(double d) {
  uint16_t sign = 0;
  if (isnan(d)) return 0x7E00;
  if (signbit(d)) {
    sign = 0x8000;
    d = -d;
  }
  if (isinf(d)) return sign | 0x7C00;
  if (d < ldexp(1.0, -14)) {
    /* subnormal range: value = q * 2^-24; q == 1024 is the smallest normal */
    double q = rint(d * ldexp(1.0, 24)); /* exact scaling, RNE rounding */
    return sign | (uint16_t)q;
  }
  int E;
  frexp(d, &E); /* d = f * 2^E, f in [0.5, 1) -> d in [2^(E-1), 2^E) */
  E -= 1;       /* d in [2^E, 2^(E+1)) */
  double q = rint(ldexp(d, 10 - E)); /* mantissa with implicit bit, RNE */
  if (q >= 2048.0) {
    q = 1024.0;
    E += 1;
  }
  if (E + 15 >= 31) return sign | 0x7C00;
  return sign | (uint16_t)(((E + 15) << 10) | ((int)q - 1024));
}

/* --------------------------------------------------------- quantization */

/* O3: symmetric absmax quantization of one block ("divide the
 * activation tensor into ... blocks"; SPEC S:L65 symmetric scale,
 * S:L74 round-half-away + clamp, S:L99 degenerate scale 1).
 *   a = max|x|;  a == 0 -> s = 1, q = 0;
 *   else s = a/qmax, r = qmax/a (fp32 IEEE divisions), v = x*r (fp32),
 *   q = clamp(roundf(v), -qmax, qmax). */
void oracle_quantize_block(const float* x, int n, int qmax, int8_t* q, float* s_out) {
  float a = 0.0f;
  for (int i = 0; i < n; ++i) {
    float ax = fabsf(x[i]);
    if (ax > a) a = ax;
  }
  if (a == 0.0f) {
    for (int i = 0; i < n; ++i) q[i] = 0;
    *s_out = 1.0f;
    return;
  }
  float s = a / (float)qmax;
  float r = (float)qmax / a;
  for (int i = 0; i < n; ++i) {
    float v = x[i] * r;
    float rv = roundf(v);
    if (rv > (float)qmax) rv = (float)qmax;
    if (rv < (float)-qmax) rv = (float)-qmax;
    q[i] = (int8_t)rv;
  }
  *s_out = s;
}

/* O4: INT4 packing, 32-bit form of the paper's W1<->W2 "location switch"
 * (§4.3, Fig 6b).  Per 8 consecutive elements e0..e7 one
 * little-endian 32-bit word with byte j = (e_j & 0xF) | (e_{j+4} & 0xF) << 4.
 * n must be a multiple of 8. */
void oracle_pack_int4(const int8_t* q, int n, uint8_t* out) {
  for (int g = 0; g < n / 8; ++g) {
    for (int j = 0; j < 4; ++j) {
      int lo = q[8 * g + j] & 0xF;
      int hi = q[8 * g + j + 4] & 0xF;
      out[4 * g + j] = (uint8_t)(lo | (hi << 4));
    }
  }
}

/* Inverse of oracle_pack_int4: sign-extend every nibble. */
void oracle_unpack_int4(const uint8_t* p, int n, int8_t* q) {
  for (int g = 0; g < n / 8; ++g) {
    for (int j = 0; j < 4; ++j) {
      int byte = p[4 * g + j];
      int lo = byte & 0xF;
      int hi = (byte >> 4) & 0xF;
      q[8 * g + j] = (int8_t)(lo >= 8 ? lo - 16 : lo);
      q[8 * g + j + 4] = (int8_t)(hi >= 8 ? hi - 16 : hi);
    }
  }
}

static int check_perm(const int32_t* perm, int K) {
  if (!perm) return 1;
  char* seen = (char*)calloc((size_t)K, 1);
  int ok = 1;
  for (int i = 0; i < K && ok; ++i) {
    if (perm[i] < 0 || perm[i] >= K || seen[perm[i]]) ok = 0;
    else seen[perm[i]] = 1;
  }
  free(seen);
  return ok;
}

/* Rank of block b among the blocks with the same precision (its slot in the
 * INT8 or the INT4 plane). */
static int block_rank(const uint8_t* bits, int b) {
  int r = 0;
  for (int i = 0; i < b; ++i)
    if (bits[i] == bits[b]) ++r;
  return r;
}

/* O1-O4: FMPQ activation quantization (P:L185 block-wise mixed precision,
 * P:L194 channel permutation "cluster these channels into a single block").
 *   X    : fp16 bits [M x K], row stride ldx (elements)
 *   k    : block size (128 in the ABI; any multiple of 8 dividing K here)
 *   perm : perm[new] = old, NULL = identity
 *   bits : K/k entries, each 4 or 8 (static per-layer mask, reading A-2)
 *   Xq8  : int8  [M x K8]   (K8 = k * #INT8 blocks),  row stride ld8 bytes
 *   Xq4  : uint8 [M x K4/2] (K4 = k * #INT4 blocks),  row stride ld4 bytes
 *   Sx   : fp32  [K/k x ldsx], Sx[b*ldsx + m]; entries m in [M, ldsx) = 1.0
 * Permuted element i of block b sits at plane column k*rank(b) + (i - k*b)
 * (bytes /2 for the INT4 plane, nibble order of oracle_pack_int4). */
int oracle_quantize_act(const uint16_t* X, int64_t ldx, int M, int K, int k,
                        const int32_t* perm, const uint8_t* bits, int8_t* Xq8,
                        int64_t ld8, uint8_t* Xq4, int64_t ld4, float* Sx,
                        int64_t ldsx) {
  if (M < 0 || K <= 0 || k <= 0 || k % 8 || K % k) return ORACLE_ERR_SHAPE;
  if (ldx < K || ldsx < M) return ORACLE_ERR_SHAPE;
  int nb = K / k;
  for (int b = 0; b < nb; ++b)
    if (bits[b] != 4 && bits[b] != 8) return ORACLE_ERR_INPUT;
  if (!check_perm(perm, K)) return ORACLE_ERR_INPUT;
  for (int64_t m = 0; m < M; ++m)
    for (int i = 0; i < K; ++i) {
      float v = oracle_half_to_float(X[m * ldx + i]);
      if (!isfinite(v)) return ORACLE_ERR_INPUT;
    }
  for (int b = 0; b < nb; ++b)
    for (int64_t m = M; m < ldsx; ++m) Sx[b * ldsx + m] = 1.0f;

#pragma omp parallel
  {
    float* xp = (float*)malloc(sizeof(float) * (size_t)K);
    int8_t* q = (int8_t*)malloc((size_t)k);
#pragma omp for schedule(static)
    for (int m = 0; m < M; ++m) {
      /* O2: Xp[m, i] = X[m, perm[i]] */
      for (int i = 0; i < K; ++i)
        xp[i] = oracle_half_to_float(X[(int64_t)m * ldx + (perm ? perm[i] : i)]);
      for (int b = 0; b < nb; ++b) {
        int qmax = bits[b] == 4 ? 7 : 127;
        float s;
        oracle_quantize_block(xp + (int64_t)b * k, k, qmax, q, &s);
        Sx[(int64_t)b * ldsx + m] = s;
        int rk = block_rank(bits, b);
        if (bits[b] == 8) {
          memcpy(Xq8 + (int64_t)m * ld8 + (int64_t)k * rk, q, (size_t)k);
        } else {
          oracle_pack_int4(q, k, Xq4 + (int64_t)m * ld4 + (int64_t)(k / 2) * rk);
        }
      }
    }
    free(xp);
    free(q);
  }
  return ORACLE_OK;
}

/* O5: INT4 weight quantization on the permuted K axis ("the
 * corresponding positions in the weight matrix also need to be permuted";
 * P:L396 4-bit weights; OmniQuant clipping replaced by symmetric min-max,
 * S:L193-201).  One scale per (n, group of `group` permuted channels).
 *   W  : fp16 bits [N x K], row stride ldw
 *   Wq : uint8 [N x K/2], nibble order of oracle_pack_int4
 *   Sw : fp32 [K/group x N], Sw[j*N + n] */
int oracle_pack_weight(const uint16_t* W, int64_t ldw, int N, int K,
                       const int32_t* perm, int group, uint8_t* Wq, float* Sw) {
  if (N < 0 || K <= 0 || group <= 0 || group % 8 || K % group || ldw < K)
    return ORACLE_ERR_SHAPE;
  if (!check_perm(perm, K)) return ORACLE_ERR_INPUT;
  for (int64_t n = 0; n < N; ++n)
    for (int i = 0; i < K; ++i)
      if (!isfinite(oracle_half_to_float(W[n * ldw + i]))) return ORACLE_ERR_INPUT;
  int ng = K / group;
#pragma omp parallel
  {
    float* wp = (float*)malloc(sizeof(float) * (size_t)K);
    int8_t* q = (int8_t*)malloc((size_t)K);
#pragma omp for schedule(static)
    for (int n = 0; n < N; ++n) {
      for (int i = 0; i < K; ++i)
        wp[i] = oracle_half_to_float(W[(int64_t)n * ldw + (perm ? perm[i] : i)]);
      for (int j = 0; j < ng; ++j) {
        float s;
        oracle_quantize_block(wp + (int64_t)j * group, group, 7, q + (int64_t)j * group, &s);
        Sw[(int64_t)j * N + n] = s;
      }
      oracle_pack_int4(q, K, Wq + (int64_t)n * (K / 2));
    }
    free(wp);
    free(q);
  }
  return ORACLE_OK;
}

/* O6-O7: the W4Ax GEMM Y = dequant(Xq . Wq^T) ("O = WX"; P:L248
 * per-tile partials accumulated by a reduction operator; P:L294 scale
 * applied after integer accumulation).
 *   acc[b][m][n] = sum_{i in block b} xq[m,i] * wq[n,i]      (exact int)
 *   Y64[m][n]    = sum_b (double)Sx[b,m] * (double)Sw[g(b),n] * acc[b][m][n]
 *                  (fp64, b ascending),  Y = fp16_rne(Y64).
 * rows: optional list of nrows row indices to evaluate (NULL = all M rows,
 * nrows ignored); outputs are [nrows x N] (or [M x N]) in that row order.
 * Outputs Y (fp16 bits), Y64, Acc ([nb x R x N]) are each optional.
 * Weight groups must not straddle activation blocks: group % k == 0 or
 * group == K (reading A-9). */
int oracle_w4ax_gemm(const int8_t* Xq8, int64_t ld8, const uint8_t* Xq4,
                     int64_t ld4, const float* Sx, int64_t ldsx,
                     const uint8_t* bits, int M, int K, int k,
                     const uint8_t* Wq, const float* Sw, int N, int group,
                     const int32_t* rows, int nrows, uint16_t* Y, double* Y64,
                     int32_t* Acc) {
  if (M < 0 || N < 0 || K <= 0 || k <= 0 || k % 8 || K % k) return ORACLE_ERR_SHAPE;
  if (group <= 0 || K % group || (group % k && group != K)) return ORACLE_ERR_SHAPE;
  int nb = K / k;
  for (int b = 0; b < nb; ++b)
    if (bits[b] != 4 && bits[b] != 8) return ORACLE_ERR_INPUT;
  int R = rows ? nrows : M;
  for (int r = 0; r < R; ++r)
    if (rows && (rows[r] < 0 || rows[r] >= M)) return ORACLE_ERR_INPUT;

  /* unpack the whole weight matrix once: wq[n][i], i on the permuted axis */
  int8_t* wq = (int8_t*)malloc((size_t)N * (size_t)K);
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n) oracle_unpack_int4(Wq + (int64_t)n * (K / 2), K, wq + (int64_t)n * K);

#pragma omp parallel
  {
    int8_t* xq = (int8_t*)malloc((size_t)K);
#pragma omp for schedule(dynamic, 1)
    for (int r = 0; r < R; ++r) {
      int m = rows ? rows[r] : r;
      /* gather the row's integer activations back onto the permuted axis */
      for (int b = 0; b < nb; ++b) {
        int rk = block_rank(bits, b);
        if (bits[b] == 8)
          memcpy(xq + (int64_t)b * k, Xq8 + (int64_t)m * ld8 + (int64_t)k * rk, (size_t)k);
        else
          oracle_unpack_int4(Xq4 + (int64_t)m * ld4 + (int64_t)(k / 2) * rk, k, xq + (int64_t)b * k);
      }
      for (int n = 0; n < N; ++n) {
        const int8_t* w = wq + (int64_t)n * K;
        double y = 0.0;
        for (int b = 0; b < nb; ++b) {
          int32_t acc = 0;
          for (int i = b * k; i < (b + 1) * k; ++i) acc += (int32_t)xq[i] * (int32_t)w[i];
          if (Acc) Acc[((int64_t)b * R + r) * N + n] = acc;
          int g = (b * k) / group;
          y += (double)Sx[(int64_t)b * ldsx + m] * (double)Sw[(int64_t)g * N + n] * (double)acc;
        }
        if (Y64) Y64[(int64_t)r * N + n] = y;
        if (Y) Y[(int64_t)r * N + n] = oracle_double_to_half(y);
      }
    }
    free(xq);
  }
  free(wq);
  return ORACLE_OK;
}

/* Number of OpenMP threads the oracle will use (reported as cpu cores). */
int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
