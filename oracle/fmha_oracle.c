/*
 * fmha_oracle.c -- CPU restatement of the reference FMHA forward path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernel.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path
 * (paper_2312_11918_b200/) never links or calls it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/proj):
 *
 *   orc_mt19937_64_*      std::mt19937_64 (C++ standard algorithm) used by
 *                         GaussianSource                include/fmhasim/random.hpp:14-42
 *   orc_gaussian_fill     gaussian_tensor               include/fmhasim/random.hpp:44-50
 *   orc_f16_round         float_to_half_bits/half_bits_to_float/f16_round
 *                                                       include/fmhasim/half.hpp:12-72
 *   orc_bf16_round        NEW (the reference has no bf16): IEEE RNE to bfloat16
 *   gemm_nt_accumulate    gemm_nt_accumulate            src/attention.cpp:75-94
 *   online_softmax_step   online_softmax_step           src/attention.cpp:36-66
 *   rowwise_finalize      rowwise_finalize              src/attention.cpp:68-73
 *   fmha_tile             fmha_tile (file-local)        src/attention.cpp:117-133
 *   orc_fmha_forward      fmha_forward                  src/attention.cpp:153-173
 *                         (+ LSE = rowMaxNew + log(rowSum), which the
 *                         reference computes in SoftmaxState but discards)
 *   orc_standard_attention standard_attention (bM=bN=N) src/attention.cpp:137-151
 *   orc_attention_flops   attention_flops               src/attention.cpp:191-193
 *
 * Parity pinning: the restatement is checked bit-for-bit against the
 * reference compiled from its own sources (oracle/_ref, see oracle/Makefile)
 * and against the FNV-1a hashes recorded in SURVEY.md Appendix A
 * (tests/golden/goldens.json, tests/test_oracle.py).
 *
 * Build flags matter: the reference is compiled at -O2 for x86-64 without
 * FMA contraction, so this file must be compiled with -ffp-contract=off (the
 * Makefile does) to reproduce its float rounding sequence exactly.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------ */
/* mt19937_64: the standard C++ engine (N=312, M=156).                 */
/* ------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;

static void mt64_seed(orc_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(orc_mt64* s) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  const uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
  if (s->idx >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
    }
    for (; i < 311; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
    }
    uint64_t x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* GaussianSource::uniform, random.hpp:37-39: 53-bit mantissa uniform. */
static double mt64_uniform(orc_mt64* s) {
  return (double)(mt64_next(s) >> 11) * (1.0 / 9007199254740992.0);
}

/* gaussian_tensor (random.hpp:44-50): one GaussianSource per tensor, values
 * produced in storage order; Box-Muller returns r*cos first and keeps r*sin
 * as the spare (random.hpp:20-34). */
void orc_gaussian_fill(float* out, int64_t count, uint64_t seed) {
  orc_mt64* s = (orc_mt64*)malloc(sizeof(orc_mt64));
  mt64_seed(s, seed);
  int has_spare = 0;
  float spare = 0.0f;
  for (int64_t i = 0; i < count; ++i) {
    if (has_spare) {
      has_spare = 0;
      out[i] = spare;
      continue;
    }
    double u1, u2;
    do {
      u1 = mt64_uniform(s);
    } while (u1 <= 0.0);
    u2 = mt64_uniform(s);
    double r = sqrt(-2.0 * log(u1));
    double theta = 2.0 * M_PI * u2;
    spare = (float)(r * sin(theta));
    has_spare = 1;
    out[i] = (float)(r * cos(theta));
  }
  free(s);
}

/* ------------------------------------------------------------------ */
/* binary16 / bfloat16 rounding                                        */
/* ------------------------------------------------------------------ */
/* float_to_half_bits, half.hpp:12-42 (RNE, saturating to +-65504). */
uint16_t orc_float_to_half_bits(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  int32_t e = (int32_t)((x >> 23) & 0xFF) - 127 + 15;
  uint32_t mant = x & 0x7FFFFFu;
  if (((x >> 23) & 0xFF) == 0xFF) return (uint16_t)(sign | 0x7C00u | (mant ? 0x200u : 0u));
  if (e >= 31) return (uint16_t)(sign | 0x7BFFu);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    mant |= 0x800000u;
    int shift = 14 - e;
    uint32_t hm = mant >> shift;
    uint32_t rem = mant & ((1u << shift) - 1);
    uint32_t halfway = 1u << (shift - 1);
    if (rem > halfway || (rem == halfway && (hm & 1))) ++hm;
    return (uint16_t)(sign | hm);
  }
  uint32_t hm = mant >> 13;
  uint32_t rem = mant & 0x1FFFu;
  uint16_t h = (uint16_t)(sign | ((uint32_t)e << 10) | hm);
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1))) ++h;
  if ((h & 0x7FFFu) >= 0x7C00u) h = (uint16_t)(sign | 0x7BFFu);
  return h;
}

/* half_bits_to_float, half.hpp:44-68. */
float orc_half_bits_to_float(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1F;
  uint32_t mant = h & 0x3FFu;
  uint32_t x;
  if (e == 0) {
    if (mant == 0) {
      x = sign;
    } else {
      int k = -1;
      do {
        ++k;
        mant <<= 1;
      } while ((mant & 0x400u) == 0);
      x = sign | (uint32_t)(127 - 15 - k) << 23 | ((mant & 0x3FFu) << 13);
    }
  } else if (e == 31) {
    x = sign | 0x7F800000u | (mant << 13);
  } else {
    x = sign | ((e - 15 + 127) << 23) | (mant << 13);
  }
  float f;
  memcpy(&f, &x, 4);
  return f;
}

/* f16_round, half.hpp:72. */
float orc_f16_round(float f) { return orc_half_bits_to_float(orc_float_to_half_bits(f)); }

/* bf16 RNE (not in the reference; NaN kept quiet, overflow -> inf as IEEE). */
uint16_t orc_float_to_bf16_bits(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  if ((x & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((x >> 16) | 0x40u);
  uint32_t lsb = (x >> 16) & 1u;
  x += 0x7FFFu + lsb;
  return (uint16_t)(x >> 16);
}
float orc_bf16_bits_to_float(uint16_t b) {
  uint32_t x = (uint32_t)b << 16;
  float f;
  memcpy(&f, &x, 4);
  return f;
}
float orc_bf16_round(float f) { return orc_bf16_bits_to_float(orc_float_to_bf16_bits(f)); }

/* In-place quantisation of a float buffer: mode 1 = f16, 2 = bf16. */
void orc_quantize(float* x, int64_t count, int mode) {
  for (int64_t i = 0; i < count; ++i)
    x[i] = mode == 1 ? orc_f16_round(x[i]) : orc_bf16_round(x[i]);
}
void orc_to_half_bits(const float* x, uint16_t* out, int64_t count, int mode) {
  for (int64_t i = 0; i < count; ++i)
    out[i] = mode == 1 ? orc_float_to_half_bits(x[i]) : orc_float_to_bf16_bits(x[i]);
}
void orc_from_half_bits(const uint16_t* x, float* out, int64_t count, int mode) {
  for (int64_t i = 0; i < count; ++i)
    out[i] = mode == 1 ? orc_half_bits_to_float(x[i]) : orc_bf16_bits_to_float(x[i]);
}

/* ------------------------------------------------------------------ */
/* attention.cpp restatement                                          */
/* ------------------------------------------------------------------ */
enum { ORC_EXACT_F32 = 0, ORC_F16_EMU = 1 };

/* gemm_nt_accumulate, attention.cpp:75-94: C[i][j] += sum_k A[i][k]*B[j][k],
 * sequential-k fp32 accumulation; F16Emu rounds both operands per MAC. */
static void gemm_nt_accumulate(const float* A, const float* B, float* C, int64_t M, int64_t Nc,
                               int64_t Kc, int prec) {
  if (prec == ORC_F16_EMU) {
    for (int64_t i = 0; i < M; ++i)
      for (int64_t j = 0; j < Nc; ++j) {
        float acc = C[i * Nc + j];
        for (int64_t k = 0; k < Kc; ++k)
          acc += orc_f16_round(A[i * Kc + k]) * orc_f16_round(B[j * Kc + k]);
        C[i * Nc + j] = acc;
      }
  } else {
    for (int64_t i = 0; i < M; ++i)
      for (int64_t j = 0; j < Nc; ++j) {
        float acc = C[i * Nc + j];
        for (int64_t k = 0; k < Kc; ++k) acc += A[i * Kc + k] * B[j * Kc + k];
        C[i * Nc + j] = acc;
      }
  }
}

/* SoftmaxState, attention.cpp:29-34. */
typedef struct {
  int64_t bM, d;
  float *rowMaxOld, *rowMaxNew, *rowSum, *O;
} orc_state;

static void state_init(orc_state* s, int64_t bM, int64_t d) {
  s->bM = bM;
  s->d = d;
  s->rowMaxOld = (float*)malloc(sizeof(float) * bM);
  s->rowMaxNew = (float*)malloc(sizeof(float) * bM);
  s->rowSum = (float*)calloc(bM, sizeof(float));
  s->O = (float*)calloc(bM * d, sizeof(float));
  for (int64_t r = 0; r < bM; ++r) s->rowMaxOld[r] = s->rowMaxNew[r] = -FLT_MAX;
}
static void state_free(orc_state* s) {
  free(s->rowMaxOld);
  free(s->rowMaxNew);
  free(s->rowSum);
  free(s->O);
}

/* std::max(a, b) == (a < b) ? b : a */
static inline float std_max(float a, float b) { return (a < b) ? b : a; }

/* online_softmax_step, attention.cpp:36-66. */
static void online_softmax_step(orc_state* st, const float* S, float* P, int64_t bN, int first) {
  for (int64_t r = 0; r < st->bM; ++r) {
    float tileMax = -FLT_MAX;
    for (int64_t c = 0; c < bN; ++c) tileMax = std_max(tileMax, S[r * bN + c]);
    st->rowMaxOld[r] = st->rowMaxNew[r];
    st->rowMaxNew[r] = std_max(st->rowMaxOld[r], tileMax);
    float rowsum = 0.0f;
    for (int64_t c = 0; c < bN; ++c) {
      float e = expf(S[r * bN + c] - st->rowMaxNew[r]);
      P[r * bN + c] = e;
      rowsum += e;
    }
    if (first) {
      st->rowSum[r] = rowsum;
    } else {
      float factor = expf(st->rowMaxOld[r] - st->rowMaxNew[r]);
      st->rowSum[r] = factor * st->rowSum[r] + rowsum;
      for (int64_t k = 0; k < st->d; ++k) st->O[r * st->d + k] *= factor;
    }
  }
}

/* rowwise_finalize, attention.cpp:68-73: O *= 1/Sigma. */
static void rowwise_finalize(orc_state* st) {
  for (int64_t r = 0; r < st->bM; ++r) {
    float inv = 1.0f / st->rowSum[r];
    for (int64_t k = 0; k < st->d; ++k) st->O[r * st->d + k] *= inv;
  }
}

/* fmha_tile, attention.cpp:117-133 (file-local in the reference; restated
 * from its public primitives as SURVEY.md 8(c) step 4 describes). */
static void fmha_tile(const float* Qtile, const float* Kh, const float* Vth, int64_t bM, int64_t bN,
                      int64_t N, int64_t d, float scale, int prec, orc_state* st) {
  float* S = (float*)malloc(sizeof(float) * bM * bN);
  float* P = (float*)malloc(sizeof(float) * bM * bN);
  float* Vt = (float*)malloc(sizeof(float) * d * bN);
  for (int64_t j = 0; j * bN < N; ++j) {
    memset(S, 0, sizeof(float) * bM * bN);
    gemm_nt_accumulate(Qtile, Kh + j * bN * d, S, bM, bN, d, prec);
    for (int64_t i = 0; i < bM * bN; ++i) S[i] *= scale;
    online_softmax_step(st, S, P, bN, j == 0);
    for (int64_t k = 0; k < d; ++k)
      for (int64_t r = 0; r < bN; ++r) Vt[k * bN + r] = Vth[k * N + j * bN + r];
    gemm_nt_accumulate(P, Vt, st->O, bM, d, bN, prec);
  }
  rowwise_finalize(st);
  free(S);
  free(P);
  free(Vt);
}

/* Tensor4::offset, tensor.hpp:20-22: n*d*h + k + head*d + b*h*N*d. */
static inline int64_t t4_off(int64_t N, int64_t h, int64_t d, int64_t b, int64_t n, int64_t head,
                             int64_t k) {
  return n * d * h + k + head * d + b * h * N * d;
}

/* head_matrix / transpose, attention.cpp:98-113. */
static void head_matrices(const float* Q, const float* K, const float* V, int64_t N, int64_t h,
                          int64_t d, int64_t b, int64_t head, float* Qh, float* Kh, float* Vth) {
  for (int64_t n = 0; n < N; ++n)
    for (int64_t k = 0; k < d; ++k) {
      int64_t o = t4_off(N, h, d, b, n, head, k);
      Qh[n * d + k] = Q[o];
      Kh[n * d + k] = K[o];
      Vth[k * N + n] = V[o];
    }
}

/* One unit of work = one Q tile (b, head, i). */
typedef struct {
  const float *Q, *K, *V;
  float *O, *lse;            /* full-problem outputs (BSHD, [L][h][N]) or NULL */
  float *tile_O, *tile_lse;  /* per-requested-tile outputs (sampled mode) or NULL */
  const int64_t* tiles;      /* sampled mode: triples (b, head, i) */
  int64_t n_units;
  int64_t L, N, h, d, bM, bN;
  float scale;
  int prec;
  int n_threads;
  int tid;
} orc_job;

static void run_head_tiles(const orc_job* J, int64_t b, int64_t head, int64_t i_begin,
                           int64_t i_end, int64_t sample_idx) {
  const int64_t N = J->N, h = J->h, d = J->d, bM = J->bM, bN = J->bN;
  float* Qh = (float*)malloc(sizeof(float) * N * d);
  float* Kh = (float*)malloc(sizeof(float) * N * d);
  float* Vth = (float*)malloc(sizeof(float) * N * d);
  head_matrices(J->Q, J->K, J->V, N, h, d, b, head, Qh, Kh, Vth);
  for (int64_t i = i_begin; i < i_end; ++i) {
    orc_state st;
    state_init(&st, bM, d);
    fmha_tile(Qh + i * bM * d, Kh, Vth, bM, bN, N, d, J->scale, J->prec, &st);
    for (int64_t r = 0; r < bM; ++r) {
      /* LSE in scaled-score units: rowMaxNew + ln(rowSum) */
      float lse = st.rowMaxNew[r] + logf(st.rowSum[r]);
      if (sample_idx >= 0) {
        memcpy(J->tile_O + (sample_idx * bM + r) * d, st.O + r * d, sizeof(float) * d);
        if (J->tile_lse) J->tile_lse[sample_idx * bM + r] = lse;
      } else {
        for (int64_t k = 0; k < d; ++k) J->O[t4_off(N, h, d, b, i * bM + r, head, k)] = st.O[r * d + k];
        if (J->lse) J->lse[(b * h + head) * N + i * bM + r] = lse;
      }
    }
    state_free(&st);
  }
  free(Qh);
  free(Kh);
  free(Vth);
}

static void* worker(void* arg) {
  const orc_job* J = (const orc_job*)arg;
  for (int64_t u = J->tid; u < J->n_units; u += J->n_threads) {
    if (J->tiles) {
      const int64_t* t = J->tiles + 3 * u;
      run_head_tiles(J, t[0], t[1], t[2], t[2] + 1, u);
    } else {
      int64_t b = u / J->h, head = u % J->h;
      run_head_tiles(J, b, head, 0, J->N / J->bM, -1);
    }
  }
  return NULL;
}

static void run_jobs(orc_job* proto) {
  int T = proto->n_threads < 1 ? 1 : proto->n_threads;
  if (T > proto->n_units) T = (int)(proto->n_units > 0 ? proto->n_units : 1);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * T);
  orc_job* jobs = (orc_job*)malloc(sizeof(orc_job) * T);
  for (int t = 0; t < T; ++t) {
    jobs[t] = *proto;
    jobs[t].n_threads = T;
    jobs[t].tid = t;
  }
  for (int t = 1; t < T; ++t) pthread_create(&th[t], NULL, worker, &jobs[t]);
  worker(&jobs[0]);
  for (int t = 1; t < T; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
}

/* validate_tiling, attention.cpp:21-27 (+ AttentionProblem checks :16-17).
 * Returns 0 when valid, 2 (the CLI's config exit code) otherwise. */
int orc_validate(int64_t N, int64_t d, int64_t bM, int64_t bN) {
  if (N < 1 || d < 1) return 2;
  if (bM < 1 || bN < 1 || N % bM != 0 || N % bN != 0) return 2;
  return 0;
}

/* AttentionProblem::scale, attention.cpp:18. */
float orc_default_scale(int64_t d) { return (float)(1.0 / sqrt((double)d)); }

/* fmha_forward, attention.cpp:153-173, multi-threaded over independent
 * (b, head) units (bitwise identical to the serial reference: SURVEY 8(c)4). */
int orc_fmha_forward(const float* Q, const float* K, const float* V, int64_t L, int64_t N,
                     int64_t h, int64_t d, int64_t bM, int64_t bN, float scale, int prec, float* O,
                     float* lse, int n_threads) {
  if (orc_validate(N, d, bM, bN)) return 2;
  orc_job J;
  memset(&J, 0, sizeof(J));
  J.Q = Q; J.K = K; J.V = V; J.O = O; J.lse = lse;
  J.n_units = L * h;
  J.L = L; J.N = N; J.h = h; J.d = d; J.bM = bM; J.bN = bN;
  J.scale = scale; J.prec = prec; J.n_threads = n_threads;
  run_jobs(&J);
  return 0;
}

/* Sampled variant: only the listed (b, head, i) Q tiles, each written to
 * tile_O[s][bM][d] and tile_lse[s][bM]. */
int orc_fmha_tiles(const float* Q, const float* K, const float* V, int64_t L, int64_t N, int64_t h,
                   int64_t d, int64_t bM, int64_t bN, float scale, int prec, const int64_t* tiles,
                   int64_t n_tiles, float* tile_O, float* tile_lse, int n_threads) {
  if (orc_validate(N, d, bM, bN)) return 2;
  for (int64_t s = 0; s < n_tiles; ++s) {
    const int64_t* t = tiles + 3 * s;
    if (t[0] < 0 || t[0] >= L || t[1] < 0 || t[1] >= h || t[2] < 0 || t[2] >= N / bM) return 2;
  }
  orc_job J;
  memset(&J, 0, sizeof(J));
  J.Q = Q; J.K = K; J.V = V; J.tile_O = tile_O; J.tile_lse = tile_lse; J.tiles = tiles;
  J.n_units = n_tiles;
  J.L = L; J.N = N; J.h = h; J.d = d; J.bM = bM; J.bN = bN;
  J.scale = scale; J.prec = prec; J.n_threads = n_threads;
  run_jobs(&J);
  return 0;
}

/* standard_attention, attention.cpp:137-151: one tile with bM = bN = N. */
int orc_standard_attention(const float* Q, const float* K, const float* V, int64_t L, int64_t N,
                           int64_t h, int64_t d, float scale, int prec, float* O, float* lse,
                           int n_threads) {
  return orc_fmha_forward(Q, K, V, L, N, h, d, N, N, scale, prec, O, lse, n_threads);
}

/* attention_flops, attention.cpp:191-193. */
int64_t orc_attention_flops(int64_t L, int64_t N, int64_t h, int64_t d) {
  return 4 * N * N * d * h * L;
}

/* FNV-1a-64 over the raw 32-bit float words in storage order (the hash used
 * for SURVEY.md Appendix A: h ^= word; h *= prime). */
uint64_t orc_fnv1a64(const void* data, int64_t nbytes) {
  const uint32_t* p = (const uint32_t*)data;
  uint64_t hsh = 1469598103934665603ULL;
  for (int64_t i = 0; i < nbytes / 4; ++i) {
    hsh ^= p[i];
    hsh *= 1099511628211ULL;
  }
  return hsh;
}
