// fmha.hpp -- C++ drop-in adapter for the reference's FMHA entry point.
//
// Reference API (/root/reference/proj/include/fmhasim/attention.hpp):
//   struct AttentionProblem { Tensor4 Q, K, V; float scale; ... }      :14-23
//   struct TileConfig { int64_t bM, bN; }                              :25-28
//   void validate_tiling(const AttentionProblem&, const TileConfig&);  :30
//   Tensor4 fmha_forward(const AttentionProblem&, const TileConfig&,
//                        Precision prec = Precision::ExactF32);        :58-59
//   int64_t attention_flops(int64_t L, int64_t N, int64_t h, int64_t d); :78
//   void save_tensor(...) / Tensor4 load_tensor(...)   (tensor.hpp:36-38)
// and Tensor4 (include/fmhasim/tensor.hpp:12-32).
//
// A reference caller switches `fmhasim::` to `fmha_b200::` and the include
// to "fmha/fmha.hpp"; the call shapes, the BSHD float Tensor4 and the
// std::invalid_argument conventions are the same.  Differences, all explicit:
//   * Precision::ExactF32 throws std::invalid_argument: the GPU path is
//     16-bit in / fp32 accumulate, there is no fp32 or CPU fallback.
//   * Precision::F16Emu maps to fp16 tensor-core math (the reference's
//     f16-operand emulation); Precision::BF16 is new.
//   * TileConfig keeps the reference's divisibility contract (N % bM == 0
//     and N % bN == 0, attention.cpp:21-27) so the same inputs are rejected;
//     the kernel's internal tile shape is its own choice.
//   * an overload also returns the per-row logsumexp ([L][h][N]).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "fmha.h"

namespace fmha_b200 {

enum class Precision { ExactF32, F16Emu, BF16 };

struct Tensor4 {
  int64_t L = 0, N = 0, h = 0, d = 0;
  std::vector<float> data;

  Tensor4() = default;
  Tensor4(int64_t L_, int64_t N_, int64_t h_, int64_t d_)
      : L(L_), N(N_), h(h_), d(d_), data(static_cast<size_t>(L_ * N_ * h_ * d_), 0.0f) {}

  int64_t offset(int64_t b, int64_t n, int64_t head, int64_t k) const {
    return n * d * h + k + head * d + b * h * N * d;
  }
  float& at(int64_t b, int64_t n, int64_t head, int64_t k) { return data[offset(b, n, head, k)]; }
  float at(int64_t b, int64_t n, int64_t head, int64_t k) const {
    return data[offset(b, n, head, k)];
  }
  int64_t elements() const { return static_cast<int64_t>(data.size()); }
  bool operator==(const Tensor4& o) const = default;
};

struct AttentionProblem {
  Tensor4 Q, K, V;
  float scale;  // 1/sqrt(d)

  AttentionProblem(Tensor4 q, Tensor4 k, Tensor4 v);
  int64_t L() const { return Q.L; }
  int64_t N() const { return Q.N; }
  int64_t heads() const { return Q.h; }
  int64_t d() const { return Q.d; }
};

struct TileConfig {
  int64_t bM;
  int64_t bN;
};

void validate_tiling(const AttentionProblem& p, const TileConfig& t);

// GPU FMHA forward on device `device` (default 0).  Throws
// std::invalid_argument for what the reference rejects and for ExactF32,
// std::runtime_error for CUDA failures.
Tensor4 fmha_forward(const AttentionProblem& p, const TileConfig& t,
                     Precision prec = Precision::F16Emu, int device = 0);

// Same, also filling `lse` with L*h*N floats (lse[(b*h + head)*N + n]).
Tensor4 fmha_forward(const AttentionProblem& p, const TileConfig& t, Precision prec,
                     std::vector<float>* lse, int device = 0);

int64_t attention_flops(int64_t L, int64_t N, int64_t h, int64_t d);

// FHMT fixture I/O, same format and exceptions as the reference's
// save_tensor / load_tensor (tensor.hpp:36-38): precision "f32" or "f16".
void save_tensor(const Tensor4& t, const std::string& path, const std::string& precision = "f32");
Tensor4 load_tensor(const std::string& path);

}  // namespace fmha_b200
