// fmha_host.cpp -- host side above the C ABI: float <-> 16-bit conversion,
// the fmha_forward_f32 C entry point, and the C++ drop-in adapter
// (include/fmha/fmha.hpp) mirroring fmhasim::fmha_forward
// (/root/reference/proj/include/fmhasim/attention.hpp:58-59).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "../../include/fmha/fmha.h"
#include "../../include/fmha/fmha.hpp"
#include "fmha_errors.hpp"

namespace {

// float -> IEEE binary16, round-to-nearest-even.  Finite values whose
// rounded magnitude exceeds the f16 range SATURATE to +-65504, matching the
// reference's host quantiser (half.hpp:22-24,40) rather than IEEE overflow.
inline uint16_t f32_to_f16_sat(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t ax = x & 0x7FFFFFFFu;
  if (ax >= 0x7F800000u) return static_cast<uint16_t>(sign | 0x7C00u | (ax > 0x7F800000u ? 0x200u : 0u));
  if (ax >= 0x477FF000u) return static_cast<uint16_t>(sign | 0x7BFFu);  // rounds to >= 65520
  if (ax < 0x38800000u) {
    // result is subnormal (or zero): scale into the 10-bit subnormal grid
    // with one float add -- exact RNE because the grid spacing (2^-24) is a
    // power of two and the add rounds in the FPU's default RNE mode.
    float a;
    uint32_t ua = ax;
    std::memcpy(&a, &ua, 4);
    const float biased = a + 0.5f;  // ulp(0.5) = 2^-24 = f16 subnormal step
    uint32_t ub;
    std::memcpy(&ub, &biased, 4);
    return static_cast<uint16_t>(sign | (ub - 0x3F000000u));
  }
  // normal: rebias exponent, round the 13 dropped mantissa bits to even
  const uint32_t mant_odd = (ax >> 13) & 1u;
  const uint32_t r = ax + 0xC8000FFFu + mant_odd;  // -(112 << 23) + 0xFFF + odd
  return static_cast<uint16_t>(sign | (r >> 13));
}

inline float f16_to_f32(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1Fu;
  const uint32_t m = h & 0x3FFu;
  uint32_t x;
  if (e == 0) {
    const float v = static_cast<float>(m) * 5.9604644775390625e-08f;  // m * 2^-24, exact
    std::memcpy(&x, &v, 4);
    x |= sign;
  } else if (e == 31) {
    x = sign | 0x7F800000u | (m << 13);
  } else {
    x = sign | ((e + 112u) << 23) | (m << 13);
  }
  float f;
  std::memcpy(&f, &x, 4);
  return f;
}

inline uint16_t f32_to_bf16(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  if ((x & 0x7FFFFFFFu) > 0x7F800000u) return static_cast<uint16_t>((x >> 16) | 0x40u);
  x += 0x7FFFu + ((x >> 16) & 1u);
  return static_cast<uint16_t>(x >> 16);
}

inline float bf16_to_f32(uint16_t b) {
  const uint32_t x = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &x, 4);
  return f;
}

template <class F>
void parallel_for(int64_t n, F&& fn) {
  const int64_t kGrain = 1 << 20;
  int T = static_cast<int>(std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()),
                                             (n + kGrain - 1) / kGrain));
  if (T <= 1) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t per = (n + T - 1) / T;
  for (int t = 0; t < T; ++t) {
    const int64_t a = t * per, b = std::min(n, a + per);
    if (a < b) th.emplace_back([&, a, b] { fn(a, b); });
  }
  for (auto& x : th) x.join();
}

#if defined(__x86_64__)
// F16C fast paths (8 values per instruction).  vcvtps2ph with round-to-nearest
// -even equals f32_to_f16_sat for every |x| <= 65504 (subnormal results
// included); groups of 8 holding a NaN or a larger magnitude take the scalar
// path, which saturates finite values and keeps inf / canonical NaN.
__attribute__((target("avx2,f16c"))) void to_f16_f16c(const float* src, uint16_t* dst, int64_t a, int64_t b) {
  const __m256 lim = _mm256_set1_ps(65504.0f);
  const __m256 abs_mask = _mm256_castsi256_ps(_mm256_set1_epi32(0x7FFFFFFF));
  int64_t i = a;
  for (; i + 8 <= b; i += 8) {
    const __m256 x = _mm256_loadu_ps(src + i);
    const __m256 special = _mm256_cmp_ps(_mm256_and_ps(x, abs_mask), lim, _CMP_NLE_UQ);  // > lim or NaN
    if (_mm256_movemask_ps(special)) {
      for (int t = 0; t < 8; ++t) dst[i + t] = f32_to_f16_sat(src[i + t]);
      continue;
    }
    _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i), _mm256_cvtps_ph(x, _MM_FROUND_TO_NEAREST_INT));
  }
  for (; i < b; ++i) dst[i] = f32_to_f16_sat(src[i]);
}
__attribute__((target("avx2,f16c"))) void from_f16_f16c(const uint16_t* src, float* dst, int64_t a, int64_t b) {
  int64_t i = a;
  for (; i + 8 <= b; i += 8)
    _mm256_storeu_ps(dst + i, _mm256_cvtph_ps(_mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i))));
  for (; i < b; ++i) dst[i] = f16_to_f32(src[i]);
}
bool has_f16c() {
  static const bool ok = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("f16c");
  return ok;
}
#endif

void to_16(const float* src, uint16_t* dst, int64_t n, fmha_dtype dt) {
  parallel_for(n, [&](int64_t a, int64_t b) {
    if (dt == FMHA_BF16) {
      for (int64_t i = a; i < b; ++i) dst[i] = f32_to_bf16(src[i]);
      return;
    }
#if defined(__x86_64__)
    if (has_f16c()) return to_f16_f16c(src, dst, a, b);
#endif
    for (int64_t i = a; i < b; ++i) dst[i] = f32_to_f16_sat(src[i]);
  });
}

void from_16(const uint16_t* src, float* dst, int64_t n, fmha_dtype dt) {
  parallel_for(n, [&](int64_t a, int64_t b) {
    if (dt == FMHA_BF16) {
      for (int64_t i = a; i < b; ++i) dst[i] = bf16_to_f32(src[i]);
      return;
    }
#if defined(__x86_64__)
    if (has_f16c()) return from_f16_f16c(src, dst, a, b);
#endif
    for (int64_t i = a; i < b; ++i) dst[i] = f16_to_f32(src[i]);
  });
}

// Pinned 16-bit staging for fmha_forward_f32 (Q, K, V, O), kept across calls:
// page-locked buffers let fmha_fwd_host's copies run at the full PCIe rate and
// overlap its kernels; pageable vectors would be staged by the driver.
struct Staging {
  std::mutex mu;
  uint16_t* buf = nullptr;
  size_t elems = 0;
};
Staging& staging() {
  static Staging s;
  return s;
}

}  // namespace

extern "C" {

uint16_t fmha_host_f32_to_16(float x, int bf16) {
  return bf16 ? f32_to_bf16(x) : f32_to_f16_sat(x);
}
float fmha_host_16_to_f32(uint16_t x, int bf16) { return bf16 ? bf16_to_f32(x) : f16_to_f32(x); }

void fmha_host_quantize(const float* src, uint16_t* dst, int64_t n, fmha_dtype dtype) {
  if (src && dst && n > 0) to_16(src, dst, n, dtype);
}
void fmha_host_dequantize(const uint16_t* src, float* dst, int64_t n, fmha_dtype dtype) {
  if (src && dst && n > 0) from_16(src, dst, n, dtype);
}

fmha_status fmha_forward_f32(const float* q, const float* k, const float* v, int64_t L, int64_t N,
                             int64_t h, int64_t d, int64_t bM, int64_t bN, fmha_dtype dtype,
                             float scale, float* o, float* lse, int device) {
  fmha_fwd_params p;
  fmha_params_dense(&p, L, N, h, d, dtype, scale);
  fmha_status s = fmha_fwd_check(&p);
  if (s != FMHA_OK) return s;
  // validate_tiling, attention.cpp:21-27
  if (bM < 1 || bN < 1 || N % bM != 0 || N % bN != 0) {
    fmha_b200::g_last_error = "TileConfig: N = " + std::to_string(N) + " must be divisible by bM = " +
                              std::to_string(bM) + " and bN = " + std::to_string(bN);
    return FMHA_ERR_CONFIG;
  }
  if (!q || !k || !v || !o) {
    fmha_b200::g_last_error = "null tensor pointer";
    return FMHA_ERR_CONFIG;
  }
  const int64_t n = L * N * h * d;
  Staging& stg = staging();
  std::lock_guard<std::mutex> lock(stg.mu);
  std::vector<uint16_t> pageable;  // fallback when page-locked memory is unavailable
  uint16_t* base = nullptr;
  if (stg.elems >= static_cast<size_t>(4 * n)) {
    base = stg.buf;
  } else {
    if (stg.buf) cudaFreeHost(stg.buf);
    stg.buf = nullptr;
    stg.elems = 0;
    void* b = nullptr;
    if (cudaHostAlloc(&b, static_cast<size_t>(4 * n) * 2, cudaHostAllocPortable) == cudaSuccess) {
      stg.buf = static_cast<uint16_t*>(b);
      stg.elems = static_cast<size_t>(4 * n);
      base = stg.buf;
    } else {
      cudaGetLastError();  // clear the allocation error, use pageable memory
      pageable.resize(static_cast<size_t>(4 * n));
      base = pageable.data();
    }
  }
  uint16_t *hq = base, *hk = base + n, *hv = base + 2 * n, *ho = base + 3 * n;
  // quantise each input chunk just before the pipeline copies it, so the
  // conversion of chunk c+1 overlaps the copies / kernels of chunk c
  struct Ctx {
    const float *q, *k, *v;
    uint16_t *hq, *hk, *hv;
    int64_t per_batch;
    fmha_dtype dt;
  } ctx{q, k, v, hq, hk, hv, N * h * d, dtype};
  auto prepare = [](void* c, int64_t b0, int64_t b1) {
    const Ctx& x = *static_cast<const Ctx*>(c);
    const int64_t off = b0 * x.per_batch, cnt = (b1 - b0) * x.per_batch;
    to_16(x.q + off, x.hq + off, cnt, x.dt);
    to_16(x.k + off, x.hk + off, cnt, x.dt);
    to_16(x.v + off, x.hv + off, cnt, x.dt);
  };
  s = fmha_b200::fwd_host_pipeline(&p, hq, hk, hv, ho, lse, device, prepare, &ctx);
  if (s != FMHA_OK) return s;
  from_16(ho, o, n, dtype);
  return FMHA_OK;
}

}  // extern "C"

namespace fmha_b200 {

AttentionProblem::AttentionProblem(Tensor4 q, Tensor4 k, Tensor4 v)
    : Q(std::move(q)), K(std::move(k)), V(std::move(v)) {
  if (Q.L != K.L || Q.N != K.N || Q.h != K.h || Q.d != K.d || Q.L != V.L || Q.N != V.N ||
      Q.h != V.h || Q.d != V.d)
    throw std::invalid_argument("AttentionProblem: Q/K/V shape mismatch");
  if (Q.N < 1 || Q.d < 1) throw std::invalid_argument("AttentionProblem: need N >= 1 and d >= 1");
  scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(Q.d)));
}

void validate_tiling(const AttentionProblem& p, const TileConfig& t) {
  if (t.bM < 1 || t.bN < 1 || p.N() % t.bM != 0 || p.N() % t.bN != 0)
    throw std::invalid_argument("TileConfig: N = " + std::to_string(p.N()) +
                                " must be divisible by bM = " + std::to_string(t.bM) +
                                " and bN = " + std::to_string(t.bN));
}

Tensor4 fmha_forward(const AttentionProblem& p, const TileConfig& t, Precision prec,
                     std::vector<float>* lse, int device) {
  validate_tiling(p, t);
  if (prec == Precision::ExactF32)
    throw std::invalid_argument("fmha_b200: the GPU path is 16-bit (use F16Emu or BF16)");
  const fmha_dtype dt = prec == Precision::BF16 ? FMHA_BF16 : FMHA_F16;
  Tensor4 O(p.L(), p.N(), p.heads(), p.d());
  if (lse) lse->assign(static_cast<size_t>(p.L() * p.heads() * p.N()), 0.0f);
  fmha_status s = fmha_forward_f32(p.Q.data.data(), p.K.data.data(), p.V.data.data(), p.L(), p.N(),
                                   p.heads(), p.d(), t.bM, t.bN, dt, p.scale, O.data.data(),
                                   lse ? lse->data() : nullptr, device);
  if (s == FMHA_ERR_CONFIG || s == FMHA_ERR_UNSUPPORTED)
    throw std::invalid_argument(std::string("fmha_b200: ") + fmha_last_error());
  if (s != FMHA_OK) throw std::runtime_error(std::string("fmha_b200: ") + fmha_last_error());
  return O;
}

Tensor4 fmha_forward(const AttentionProblem& p, const TileConfig& t, Precision prec, int device) {
  return fmha_forward(p, t, prec, nullptr, device);
}

int64_t attention_flops(int64_t L, int64_t N, int64_t h, int64_t d) {
  return fmha_attention_flops(L, N, h, d);
}

}  // namespace fmha_b200
