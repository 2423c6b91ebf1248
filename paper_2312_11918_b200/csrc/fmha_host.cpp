// fmha_host.cpp -- host side above the C ABI: float <-> 16-bit conversion,
// the fmha_forward_f32 C entry point, and the C++ drop-in adapter
// (include/fmha/fmha.hpp) mirroring fmhasim::fmha_forward
// (/root/reference/proj/include/fmhasim/attention.hpp:58-59).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <functional>
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

// Persistent worker pool for the host conversions (the float call shape
// converts ~0.5 GB per call in ~20 pieces: spawning threads per piece cost
// more than the pieces).  One parallel region at a time (callers hold the
// staging lock or run outside it on their own data); the calling thread
// takes part.
class Pool {
 public:
  static Pool& get() {
    static Pool p;
    return p;
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  // fn(t) for t in [0, T), T <= size(); returns when all are done
  void run(int T, const std::function<void(int)>& fn) {
    std::unique_lock<std::mutex> region(region_mu_);
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn;
      tasks_ = T;
      next_ = 1;
      pending_ = T - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  Pool() {
    const int n = std::max(1u, std::thread::hardware_concurrency()) - 1;
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> g(mu_);
      cv_.wait(g, [&] { return stop_ || (gen_ != seen && next_ < tasks_); });
      if (stop_) return;
      const int t = next_++;
      if (next_ >= tasks_) seen = gen_;
      const std::function<void(int)>* fn = fn_;
      g.unlock();
      (*fn)(t);
      g.lock();
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, region_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int tasks_ = 0, next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

template <class F>
void parallel_for(int64_t n, F&& fn) {
  const int64_t kGrain = 1 << 18;
  Pool& pool = Pool::get();
  const int T = static_cast<int>(std::min<int64_t>(pool.size(), (n + kGrain - 1) / kGrain));
  if (T <= 1) {
    fn(0, n);
    return;
  }
  const int64_t per = (n + T - 1) / T;
  pool.run(T, [&](int t) {
    const int64_t a = t * per, b = std::min(n, a + per);
    if (a < b) fn(a, b);
  });
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

// src[a, b) -> dst[a, b), on the calling thread
void from_16_range(const uint16_t* src, float* dst, int64_t a, int64_t b, fmha_dtype dt) {
  if (dt == FMHA_BF16) {
    for (int64_t i = a; i < b; ++i) dst[i] = bf16_to_f32(src[i]);
    return;
  }
#if defined(__x86_64__)
  if (has_f16c()) return from_f16_f16c(src, dst, a, b);
#endif
  for (int64_t i = a; i < b; ++i) dst[i] = f16_to_f32(src[i]);
}

void from_16(const uint16_t* src, float* dst, int64_t n, fmha_dtype dt) {
  parallel_for(n, [&](int64_t a, int64_t b) { from_16_range(src, dst, a, b, dt); });
}

// Pinned staging for fmha_forward_f32 (16-bit Q, K, V, O and fp32 LSE), kept
// across calls: page-locked buffers let fmha_fwd_host's copies run at the full
// PCIe rate and overlap its kernels (a D2H copy into pageable memory would
// also block the calling thread until the copy is done).
struct Staging {
  std::mutex mu;
  uint16_t* buf = nullptr;
  size_t bytes = 0;
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
  const int64_t n_lse = L * h * N;
  const size_t need = static_cast<size_t>(4 * n) * 2 + static_cast<size_t>(n_lse) * 4;
  Staging& stg = staging();
  std::lock_guard<std::mutex> lock(stg.mu);
  std::vector<uint8_t> pageable;  // fallback when page-locked memory is unavailable
  uint8_t* base = nullptr;
  if (stg.bytes >= need) {
    base = reinterpret_cast<uint8_t*>(stg.buf);
  } else {
    if (stg.buf) cudaFreeHost(stg.buf);
    stg.buf = nullptr;
    stg.bytes = 0;
    void* b = nullptr;
    if (cudaHostAlloc(&b, need, cudaHostAllocPortable) == cudaSuccess) {
      stg.buf = static_cast<uint16_t*>(b);
      stg.bytes = need;
      base = static_cast<uint8_t*>(b);
    } else {
      cudaGetLastError();  // clear the allocation error, use pageable memory
      pageable.resize(need);
      base = pageable.data();
    }
  }
  uint16_t* hq = reinterpret_cast<uint16_t*>(base);
  uint16_t *hk = hq + n, *hv = hq + 2 * n, *ho = hq + 3 * n;
  float* hl = lse ? reinterpret_cast<float*>(hq + 4 * n) : nullptr;
  // Quantise each input chunk just before the pipeline copies it (the
  // conversion of chunk c+1 overlaps the copies / kernels of chunk c), and
  // dequantise each piece of O as soon as it is back on the host (while later
  // pieces are still computed / copied).
  struct Ctx {
    const float *q, *k, *v;
    uint16_t *hq, *hk, *hv, *ho;
    const float* hl;
    float *o, *lse;
    int64_t N, h, d;
    fmha_dtype dt;
  } ctx{q, k, v, hq, hk, hv, ho, hl, o, lse, N, h, d, dtype};
  auto prepare = [](void* c, int64_t b0, int64_t b1) {
    const Ctx& x = *static_cast<const Ctx*>(c);
    const int64_t per_batch = x.N * x.h * x.d;
    const int64_t off = b0 * per_batch, cnt = (b1 - b0) * per_batch;
    to_16(x.q + off, x.hq + off, cnt, x.dt);
    to_16(x.k + off, x.hk + off, cnt, x.dt);
    to_16(x.v + off, x.hv + off, cnt, x.dt);
  };
  auto consume = [](void* c, const fmha_b200::OutPiece& pc) {
    const Ctx& x = *static_cast<const Ctx*>(c);
    const int64_t row = x.h * x.d;  // elements per query row (all heads)
    for (int64_t b = pc.b0; b < pc.b1; ++b) {
      if (pc.h0 == 0 && pc.h1 == x.h) {  // whole rows: one contiguous range
        const int64_t off = (b * x.N + pc.n0) * row;
        from_16(x.ho + off, x.o + off, (pc.n1 - pc.n0) * row, x.dt);
      } else {  // a head group: (h1 - h0) * d contiguous elements per row
        const int64_t w = (pc.h1 - pc.h0) * x.d;
        parallel_for((pc.n1 - pc.n0) * w, [&](int64_t a, int64_t e) {
          for (int64_t r = a / w; r * w < e; ++r) {
            const int64_t lo = std::max(a, r * w) - r * w, hi = std::min(e, (r + 1) * w) - r * w;
            const int64_t off = (b * x.N + pc.n0 + r) * row + pc.h0 * x.d;
            from_16_range(x.ho + off, x.o + off, lo, hi, x.dt);
          }
        });
      }
      if (x.lse)
        for (int64_t hh = pc.h0; hh < pc.h1; ++hh) {
          const int64_t off = (b * x.h + hh) * x.N + pc.n0;
          std::memcpy(x.lse + off, x.hl + off, static_cast<size_t>(pc.n1 - pc.n0) * 4);
        }
    }
  };
  return fmha_b200::fwd_host_pipeline(&p, hq, hk, hv, ho, hl, device, prepare, &ctx, consume);
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
