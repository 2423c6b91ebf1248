// ref_shim.cpp -- C ABI over the REFERENCE's public C++ API (TEST INFRASTRUCTURE).
//
// Compiled together with the reference's own sources, where they lie under
// /root/reference/proj (see oracle/Makefile), into oracle/_ref/libfmhasim_ref.so.
// Nothing from the reference is copied here: this file only calls
//   fmhasim::gaussian_tensor          include/fmhasim/random.hpp:44-50
//   fmhasim::AttentionProblem         include/fmhasim/attention.hpp:14-23
//   fmhasim::fmha_forward             include/fmhasim/attention.hpp:58-59
//   fmhasim::standard_attention       include/fmhasim/attention.hpp:54-55
//   fmhasim::SoftmaxState / online_softmax_step / rowwise_finalize /
//   gemm_nt_accumulate                include/fmhasim/attention.hpp:33-75
//   fmhasim::f16_round                include/fmhasim/half.hpp:72
// The per-Q-tile driver below restates the file-local fmha_tile
// (src/attention.cpp:117-133) from those public primitives so that LSE
// (rowMaxNew + log rowSum) is observable; SURVEY.md 8(c) step 4 measured it
// bitwise identical to fmha_forward.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "fmhasim/attention.hpp"
#include "fmhasim/half.hpp"
#include "fmhasim/random.hpp"
#include "fmhasim/tensor.hpp"

using namespace fmhasim;

namespace {

Tensor4 from_buf(const float* p, int64_t L, int64_t N, int64_t h, int64_t d) {
  Tensor4 t(L, N, h, d);
  std::memcpy(t.data.data(), p, sizeof(float) * t.data.size());
  return t;
}

Precision prec_of(int prec) { return prec == 1 ? Precision::F16Emu : Precision::ExactF32; }

// The restated per-Q-tile driver (fmha_tile + head staging, attention.cpp:98-133).
void tile_driver(const AttentionProblem& p, int64_t b, int64_t head, int64_t i, int64_t bM,
                 int64_t bN, Precision prec, float* outO, float* outLse) {
  const int64_t N = p.N(), d = p.d();
  std::vector<float> Qt(size_t(bM) * d), Kh(size_t(N) * d), Vth(size_t(d) * N);
  for (int64_t r = 0; r < bM; ++r)
    for (int64_t k = 0; k < d; ++k) Qt[r * d + k] = p.Q.at(b, i * bM + r, head, k);
  for (int64_t n = 0; n < N; ++n)
    for (int64_t k = 0; k < d; ++k) {
      Kh[n * d + k] = p.K.at(b, n, head, k);
      Vth[k * N + n] = p.V.at(b, n, head, k);
    }
  SoftmaxState state(bM, d);
  std::vector<float> S(size_t(bM) * bN), Vt(size_t(d) * bN);
  for (int64_t j = 0; j * bN < N; ++j) {
    std::fill(S.begin(), S.end(), 0.0f);
    gemm_nt_accumulate(Qt.data(), Kh.data() + j * bN * d, S.data(), bM, bN, d, prec);
    for (auto& s : S) s *= p.scale;
    std::vector<float> P = online_softmax_step(state, S, bN, j == 0);
    for (int64_t k = 0; k < d; ++k)
      for (int64_t r = 0; r < bN; ++r) Vt[k * bN + r] = Vth[k * N + j * bN + r];
    gemm_nt_accumulate(P.data(), Vt.data(), state.O.data(), bM, d, bN, prec);
  }
  rowwise_finalize(state);
  std::memcpy(outO, state.O.data(), sizeof(float) * bM * d);
  for (int64_t r = 0; r < bM; ++r) outLse[r] = state.rowMaxNew[r] + std::log(state.rowSum[r]);
}

}  // namespace

extern "C" {

void ref_gaussian(int64_t L, int64_t N, int64_t h, int64_t d, uint64_t seed, float* out) {
  Tensor4 t = gaussian_tensor(L, N, h, d, seed);
  std::memcpy(out, t.data.data(), sizeof(float) * t.data.size());
}

float ref_f16_round(float x) { return f16_round(x); }

// fmha_forward through the reference's own entry point; 0 ok, 2 invalid_argument.
int ref_fmha_forward(const float* q, const float* k, const float* v, int64_t L, int64_t N,
                     int64_t h, int64_t d, int64_t bM, int64_t bN, int prec, float* out) {
  try {
    AttentionProblem p(from_buf(q, L, N, h, d), from_buf(k, L, N, h, d), from_buf(v, L, N, h, d));
    Tensor4 o = fmha_forward(p, TileConfig{bM, bN}, prec_of(prec));
    std::memcpy(out, o.data.data(), sizeof(float) * o.data.size());
    return 0;
  } catch (const std::invalid_argument&) {
    return 2;
  }
}

int ref_standard_attention(const float* q, const float* k, const float* v, int64_t L, int64_t N,
                           int64_t h, int64_t d, int prec, float* out) {
  try {
    AttentionProblem p(from_buf(q, L, N, h, d), from_buf(k, L, N, h, d), from_buf(v, L, N, h, d));
    Tensor4 o = standard_attention(p, prec_of(prec));
    std::memcpy(out, o.data.data(), sizeof(float) * o.data.size());
    return 0;
  } catch (const std::invalid_argument&) {
    return 2;
  }
}

// Reference fmha_forward over single-(b,head) sub-problems on n_threads host
// threads (harness-side threading; the reference itself is serial).  Inputs
// are one head each: q/k/v hold `heads` packed (N, d) matrices.  Used as the
// bench's CPU baseline ("kind": "reference").
int ref_fmha_forward_heads(const float* q, const float* k, const float* v, int64_t heads, int64_t N,
                           int64_t d, int64_t bM, int64_t bN, float* out, int n_threads) {
  if (n_threads < 1) n_threads = 1;
  int status = 0;
  auto work = [&](int t) {
    for (int64_t u = t; u < heads; u += n_threads) {
      const size_t off = size_t(u) * N * d;
      int s = ref_fmha_forward(q + off, k + off, v + off, 1, N, 1, d, bM, bN, 0, out + off);
      if (s) status = s;
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < n_threads; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  return status;
}

// Restated per-tile driver: O and LSE for the listed (b, head, i) Q tiles.
int ref_fmha_tiles(const float* q, const float* k, const float* v, int64_t L, int64_t N, int64_t h,
                   int64_t d, int64_t bM, int64_t bN, int prec, const int64_t* tiles,
                   int64_t n_tiles, float* tile_O, float* tile_lse, int n_threads) {
  try {
    AttentionProblem p(from_buf(q, L, N, h, d), from_buf(k, L, N, h, d), from_buf(v, L, N, h, d));
    validate_tiling(p, TileConfig{bM, bN});
    if (n_threads < 1) n_threads = 1;
    auto work = [&](int t) {
      for (int64_t s = t; s < n_tiles; s += n_threads)
        tile_driver(p, tiles[3 * s], tiles[3 * s + 1], tiles[3 * s + 2], bM, bN, prec_of(prec),
                    tile_O + s * bM * d, tile_lse + s * bM);
    };
    std::vector<std::thread> th;
    for (int t = 1; t < n_threads; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    return 0;
  } catch (const std::invalid_argument&) {
    return 2;
  }
}

// save_tensor / load_tensor (tensor.cpp:30-84) for the FHMT cross-compat test.
int ref_save_tensor(const char* path, const float* data, int64_t L, int64_t N, int64_t h, int64_t d,
                    int f16) {
  try {
    save_tensor(from_buf(data, L, N, h, d), path, f16 ? "f16" : "f32");
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

int ref_load_tensor(const char* path, float* out, int64_t capacity, int64_t* dims) {
  try {
    Tensor4 t = load_tensor(path);
    dims[0] = t.L;
    dims[1] = t.N;
    dims[2] = t.h;
    dims[3] = t.d;
    if (t.elements() > capacity) return 3;
    std::memcpy(out, t.data.data(), sizeof(float) * t.data.size());
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

}  // extern "C"
