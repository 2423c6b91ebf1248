// softmax_math.cuh -- the per-row math of online_softmax_step
// (/root/reference/proj/src/attention.cpp:36-66) tuned for sm_100a:
//
//  * packed fp32x2 FMA / ADD (FFMA2 / FADD2) for x = s*c - m*c and the row sum;
//  * exp2 split between the MUFU unit (ex2.approx) and a degree-4 polynomial
//    on the FMA pipe (Cody-Waite split x = n + f, f in [-1/2, 1/2], 2^f by a
//    minimax polynomial, 2^n added into the exponent field).  At d <= 128 the
//    MUFU ex2 rate (16/clk/SM) otherwise equals the tensor-core rate per score
//    (SURVEY.md 7.2), so moving ~40% of the exponentials to the FMA pipe is
//    what lets the tensor core, not the exponential, set the pace;
//  * P packed to 16-bit pairs for the TMEM store (cvt.rn.{f16,bf16}x2).
//
// Polynomial max relative error 1.0e-4 at degree 3 (2.6e-6 at degree 4; both
// below the fp16 / bf16 rounding of P); inputs are clamped at -125 so fully masked scores give ~2e-38, which
// rounds to 0 in fp16 and contributes < 1e-37 in bf16.
#pragma once

#include <cstdint>

#include "sm100.cuh"

#ifndef FMHA_EXP2_POLY_DEG
#define FMHA_EXP2_POLY_DEG 3  // 4: the degree-4 fit (max rel err 2.6e-6)
#endif

namespace fmha_b200 {

__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^x for a pair, on the FMA + ALU pipes only.
__device__ __forceinline__ uint64_t exp2_poly_x2(uint64_t x) {
  float x0, x1;
  f2_unpack(x, x0, x1);
  x = f2_pack(fmaxf(x0, -125.0f), fmaxf(x1, -125.0f));
  const uint64_t kMagic = f2_pack(12582912.0f, 12582912.0f);  // 1.5 * 2^23: round to integer
  const uint64_t kNegMagic = f2_pack(-12582912.0f, -12582912.0f);
  const uint64_t kMinus1 = f2_pack(-1.0f, -1.0f);
  const uint64_t t = fadd2(x, kMagic);          // low mantissa bits hold n = rint(x)
  const uint64_t n = fadd2(t, kNegMagic);       // n as float
  const uint64_t f = ffma2(n, kMinus1, x);      // f = x - n in [-0.5, 0.5]
#if FMHA_EXP2_POLY_DEG == 3
  // degree-3 relative-error minimax fit on [-1/2, 1/2] with p(0) = 1 exactly
  // (integer exponents stay exact): max rel err 1.0e-4, below the 16-bit
  // rounding of P (fp16 half-ulp 4.9e-4)
  uint64_t p = ffma2(f2_pack(0.0550084225833416f, 0.0550084225833416f), f,
                     f2_pack(0.24220998585224152f, 0.24220998585224152f));
  p = ffma2(p, f, f2_pack(0.6932829022407532f, 0.6932829022407532f));
  p = ffma2(p, f, f2_pack(1.0f, 1.0f));
#else
  uint64_t p = ffma2(f2_pack(0.00957564264535904f, 0.00957564264535904f), f,
                     f2_pack(0.05591900646686554f, 0.05591900646686554f));
  p = ffma2(p, f, f2_pack(0.24024616181850433f, 0.24024616181850433f));
  p = ffma2(p, f, f2_pack(0.693121612071991f, 0.693121612071991f));
  p = ffma2(p, f, f2_pack(0.9999992847442627f, 0.9999992847442627f));
#endif
  float t0, t1, p0, p1;
  f2_unpack(t, t0, t1);
  f2_unpack(p, p0, p1);
  // (t_bits << 23) == n << 23 for |n| < 256; add it into the exponent field
  const uint32_t r0 = __float_as_uint(p0) + (__float_as_uint(t0) << 23);
  const uint32_t r1 = __float_as_uint(p1) + (__float_as_uint(t1) << 23);
  return f2_pack(__uint_as_float(r0), __uint_as_float(r1));
}

__device__ __forceinline__ uint64_t exp2_mufu_x2(uint64_t x) {
  float x0, x1;
  f2_unpack(x, x0, x1);
  return f2_pack(ex2_approx(x0), ex2_approx(x1));
}

template <bool kBF16>
__device__ __forceinline__ uint32_t pack2_x2(uint64_t e) {
  float lo, hi;
  f2_unpack(e, lo, hi);
  return pack2<kBF16>(lo, hi);
}

// Which score pairs take the polynomial: kEmuPer16 of every 16, spread evenly
// (FMHA_EMU_SPREAD=1) so each polynomial chain on the FMA pipe runs beside
// MUFU work, or clustered at the start of each group of 16 pairs (0).
#ifndef FMHA_EMU_SPREAD
#define FMHA_EMU_SPREAD 1
#endif
template <int kEmuPer16>
__device__ __forceinline__ constexpr bool emulate_pair(int i) {
#if FMHA_EMU_SPREAD
  return kEmuPer16 > 0 && ((i & 15) * kEmuPer16) % 16 + kEmuPer16 >= 16;
#else
  return (i & 15) < kEmuPer16;
#endif
}

// kEmuPer16 == kEmuEdgeFree selects a position-dependent pattern over the
// 128-score row (64 pairs in four 16-pair fragments): fragments 0 and 3 stay
// all-MUFU (the first MUFU results are not held up by polynomial chains, the
// last P fragment is not delayed by one), fragments 1 and 2 emulate 6 of 16
// pairs -- 12 of 64 in all (FlashAttention-4's default split for d = 128).
constexpr int kEmuEdgeFree = 17;
template <int kEmuPer16>
__device__ __forceinline__ constexpr bool emulate_pair_at(int ip) {
  if constexpr (kEmuPer16 == kEmuEdgeFree) {
    const int f = ip / 16, k2 = 2 * (ip % 16);
    return f >= 1 && f <= 2 && k2 % 10 >= 6;
  } else {
    return emulate_pair<kEmuPer16>(ip);
  }
}

// P = 2^(s*c - m*c) for the kCols scores s[kOff .. kOff+kCols) of one row;
// returns the fp32 sum of the UNROUNDED P (attention.cpp:50-55) and writes
// the 16-bit packed P.  Pairs selected by emulate_pair use the polynomial.
template <bool kBF16, int kOff, int kCols, int kEmuPer16, int kTotal>
__device__ __forceinline__ float exp_rowsum_pack(const float (&s)[kTotal], float c, float neg_mc,
                                                 uint32_t (&p)[kCols / 2]) {
  const uint64_t c2 = f2_pack(c, c);
  const uint64_t nm2 = f2_pack(neg_mc, neg_mc);
  uint64_t acc0 = f2_pack(0.f, 0.f), acc1 = f2_pack(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < kCols / 2; ++i) {
    const uint64_t x = ffma2(f2_pack(s[kOff + 2 * i], s[kOff + 2 * i + 1]), c2, nm2);
    const bool emu = kEmuPer16 >= kEmuEdgeFree ? emulate_pair_at<kEmuPer16>(kOff / 2 + i) : emulate_pair<kEmuPer16>(i);
    const uint64_t e = emu ? exp2_poly_x2(x) : exp2_mufu_x2(x);
    if (i & 1)
      acc1 = fadd2(acc1, e);
    else
      acc0 = fadd2(acc0, e);
    p[i] = pack2_x2<kBF16>(e);
  }
  float a0, a1, b0, b1;
  f2_unpack(acc0, a0, a1);
  f2_unpack(acc1, b0, b1);
  return (a0 + b0) + (a1 + b1);
}

// P only (no row sum): the kCols exponentials replace their scores in s
// (fp32, unrounded) and are packed to 16-bit pairs; the row sum is taken
// later with row_sum_f32, AFTER P has been published -- the FADD2 chain then
// leaves the S -> P critical path (FlashAttention-4 orders it the same way).
template <bool kBF16, int kOff, int kCols, int kEmuPer16, int kTotal>
__device__ __forceinline__ void exp_pack_inplace(float (&s)[kTotal], float c, float neg_mc,
                                                 uint32_t (&p)[kCols / 2]) {
  const uint64_t c2 = f2_pack(c, c);
  const uint64_t nm2 = f2_pack(neg_mc, neg_mc);
#pragma unroll
  for (int i = 0; i < kCols / 2; ++i) {
    const uint64_t x = ffma2(f2_pack(s[kOff + 2 * i], s[kOff + 2 * i + 1]), c2, nm2);
    const bool emu = kEmuPer16 >= kEmuEdgeFree ? emulate_pair_at<kEmuPer16>(kOff / 2 + i) : emulate_pair<kEmuPer16>(i);
    const uint64_t e = emu ? exp2_poly_x2(x) : exp2_mufu_x2(x);
    f2_unpack(e, s[kOff + 2 * i], s[kOff + 2 * i + 1]);
    p[i] = pack2_x2<kBF16>(e);
  }
}
// fp32 sum of s[0, kTotal) with eight packed accumulators (short dependency chains)
template <int kTotal>
__device__ __forceinline__ float row_sum_f32(const float (&s)[kTotal]) {
  uint64_t acc[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) acc[t] = f2_pack(s[2 * t], s[2 * t + 1]);
#pragma unroll
  for (int i = 8; i < kTotal; i += 8)
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[t] = fadd2(acc[t], f2_pack(s[i + 2 * t], s[i + 2 * t + 1]));
  acc[0] = fadd2(acc[0], acc[1]);
  acc[2] = fadd2(acc[2], acc[3]);
  acc[0] = fadd2(acc[0], acc[2]);
  float a, b;
  f2_unpack(acc[0], a, b);
  return a + b;
}

// exp_rowsum_pack over s[0, 64) with the full 128-column row max of s
// folded into the same instruction stream (FMNMX3 on the ALU pipe fills the
// MUFU / FMA latency slots): the speculative form of a tile's first half,
// exponentiated against the previous tile's max while the new one is reduced.
template <bool kBF16, int kEmuPer16>
__device__ __forceinline__ float exp_rowsum_pack_max(const float (&s)[128], float c, float neg_mc,
                                                     uint32_t (&p)[32], float& row_max) {
  const uint64_t c2 = f2_pack(c, c);
  const uint64_t nm2 = f2_pack(neg_mc, neg_mc);
  uint64_t acc0 = f2_pack(0.f, 0.f), acc1 = f2_pack(0.f, 0.f);
  float mx[4] = {s[0], s[1], s[2], s[3]};
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const uint64_t x = ffma2(f2_pack(s[2 * i], s[2 * i + 1]), c2, nm2);
    const bool emu = kEmuPer16 >= kEmuEdgeFree ? emulate_pair_at<kEmuPer16>(i) : emulate_pair<kEmuPer16>(i);
    const uint64_t e = emu ? exp2_poly_x2(x) : exp2_mufu_x2(x);
    if (i & 1)
      acc1 = fadd2(acc1, e);
    else
      acc0 = fadd2(acc0, e);
    p[i] = pack2_x2<kBF16>(e);
    // 4 more columns of the max per pair (columns 4..127 over the 32 pairs)
    if (i < 31) {
      const int b = 4 + 4 * i;
      mx[i & 3] = fmaxf(mx[i & 3], fmaxf(s[b], fmaxf(s[b + 1], fmaxf(s[b + 2], s[b + 3]))));
    }
  }
  row_max = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
  float a0, a1, b0, b1;
  f2_unpack(acc0, a0, a1);
  f2_unpack(acc1, b0, b1);
  return (a0 + b0) + (a1 + b1);
}

template <uint32_t kRegs>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegs));
}
template <uint32_t kRegs>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegs));
}

}  // namespace fmha_b200
