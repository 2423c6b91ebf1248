// fmha_fwd_st_kernel.cuh -- single-Q-tile FMHA forward with double-buffered S
// (used for head dim 256; D = 64 / 128 instantiations measured).
//
// Same contract as fmha_fwd_kernel.cuh (fmhasim::fmha_forward,
// /root/reference/proj/src/attention.cpp:153-173) but shaped for d = 256,
// where the O accumulator alone needs 256 TMEM columns and a K or V tile is
// kBN x 512 B:
//
//   CTA = one (b, head) and ONE 128-row Q tile; K/V tiles of kBN rows.
//   TMEM: S buffers A [0,kBN) and B [kBN,2kBN) (double-buffered, so the
//         tensor core computes S(j+1) while softmax works on S(j));
//         O [256,512).  P(j) (16-bit) aliases the first kBN/2 columns of its
//         S buffer.
//   smem: Q 64 KB + K/V ring of 128 KB (4 x 32 KB at kBN = 64, 2 x 64 KB at
//         kBN = 128), loaded in the MMA warp's consumption order
//         K0 K1 | V0 K2 | V1 K3 | ... so a 2-slot ring still gives every
//         load one S or PV GEMM (~1k clk) of lead time.
//   warps 0-3 softmax (thread per row), warp 4 TMA producer, warp 5 MMA.
//
// kBN = 128 (default): S GEMMs are M128 N128 (8 KB of shared memory per
// 64-clk MMA, the shared-memory rate); at kBN = 64 the N=64 S GEMMs are
// shared-memory bound at 48 clk per 32-clk MMA (tools/mma_probe.cu).
//
// MMA order: S(0) S(1) | PV(0) S(2) | PV(1) S(3) | ...  PV(j) is committed to
// `pv_done` so the softmax WG can wait for O(j-1) before a conditional
// rescale at step j (with double-buffered S, "S(j) complete" does not imply
// "PV(j-1) complete" here).
#pragma once

#include <cuda.h>
#include <cstdint>

#include "fmha_fwd_kernel.cuh"
#include "sm100.cuh"
#include "softmax_math.cuh"
#include "tmem_ops.cuh"

namespace fmha_b200 {

// Single-Q-tile, double-buffered-S configuration for head dim D and K/V
// step kBN.  TMEM: S buffers [0,kBN) [kBN,2kBN), O [2kBN, 2kBN+D); the
// allocation is the next power of two, so D + 2*kBN <= 256 fits two CTAs per
// SM (their softmax warpgroups then share the SM like a ping-pong, without
// the P -> PV -> S dependency chain between them).
template <int D_, int kBN_>
struct FwdCfgST {
  static constexpr int D = D_;
  static constexpr int kBM = 128;
  static constexpr int kBN = kBN_;
  static_assert(kBN == 64 || kBN == 128, "K/V step of 64 or 128 rows");
  static_assert(D == 64 || D == 128 || D == 256, "head dim");
  static constexpr int kChunks = D / 64;
  static constexpr int kQTileBytes = kBM * D * 2;
  static constexpr int kKVTileBytes = kBN * D * 2;
  static constexpr uint32_t kColO = 2 * kBN;
  static constexpr uint32_t kTmemCols = (2 * kBN + D) <= 256 ? 256u : 512u;
  static constexpr int kCtasPerSm = kTmemCols == 256 ? 2 : 1;
  static constexpr int kRingBudget = (kCtasPerSm == 2 ? 112 * 1024 : 226 * 1024) - kQTileBytes - 1024 - 256;
  static constexpr int kStagesFit = kRingBudget / kKVTileBytes;
  static constexpr int kStages = kStagesFit > 8 ? 8 : kStagesFit;
  static_assert(kStages >= 2, "K/V ring needs two slots");
  static constexpr int kSmemRing = kStages * kKVTileBytes;
  static constexpr int kNumBars = 1 + 2 * kStages + 2 + 2 + 2;
  static constexpr int kSmemBytes = kQTileBytes + kSmemRing + kNumBars * 8 + 16;
  static constexpr int kSmemAlloc = kSmemBytes + 1024;
  static constexpr int kThreads = 192;
  static constexpr int kLoadWarp = 4;
  static constexpr int kMmaWarp = 5;
  __host__ __device__ static constexpr uint32_t col_s(int buf) { return buf ? static_cast<uint32_t>(kBN) : 0u; }
  static_assert(kSmemAlloc <= 227 * 1024, "shared memory budget");
};
template <int kBN_>
using FwdCfgD256 = FwdCfgST<256, kBN_>;

template <int D, bool kBF16, int kBN = 128, int kEmuPer16 = 4>
__global__ void __launch_bounds__(192, FwdCfgST<D, kBN>::kCtasPerSm)
    fmha_fwd_st_kernel(const __grid_constant__ CUtensorMap tmQ,
                       const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV,
                       const __grid_constant__ CUtensorMap tmO,  // box 128 rows (epilogue TMA store)
                       const FwdArgs args) {
  using C = FwdCfgST<D, kBN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sRing = smem + C::kQTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRing + C::kSmemRing);
  uint64_t* bar_q = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;  // [2]
  uint64_t* p_full = s_full + 2;             // [2]
  uint64_t* pv_done = p_full + 2;            // [1]
  uint64_t* o_full = pv_done + 1;            // [1]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const int b = blockIdx.z;
  const int qrow0 = blockIdx.x * C::kBM;
  const int n_kv = args.n_kv_tiles;

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
    }
    mbar_init(pv_done, 1);
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == C::kMmaWarp) tmem_alloc(tmem_holder, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == C::kLoadWarp) {
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      const uint64_t keep = l2_policy_evict_last();
      const uint64_t once = l2_policy_evict_first();
      mbar_arrive_expect_tx(bar_q, C::kQTileBytes);
#pragma unroll
      for (int c = 0; c < C::kChunks; ++c)
        tma_load_4d_hint(&tmQ, bar_q, sQ + c * C::kBM * 128, c * 64, head, qrow0, b, once);
      int slot = 0;
      uint32_t phase = 0;
      auto load = [&](const CUtensorMap* map, int step) {
        mbar_wait(&kv_empty[slot], phase ^ 1);
        mbar_arrive_expect_tx(&kv_full[slot], C::kKVTileBytes);
        uint8_t* dst = sRing + slot * C::kKVTileBytes;
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_4d_hint(map, &kv_full[slot], dst + c * C::kBN * 128, c * 64, head, step * C::kBN, b, keep);
        if (++slot == C::kStages) {
          slot = 0;
          phase ^= 1;
        }
      };
      // consumption order of the MMA warp: K0 K1 | V0 K2 | V1 K3 | ...
      load(&tmK, 0);
      if (n_kv > 1) load(&tmK, 1);
      for (int j = 0; j < n_kv; ++j) {
        load(&tmV, j);
        if (j + 2 < n_kv) load(&tmK, j + 2);
      }
    }
  } else if (warp == C::kMmaWarp) {
    {  // whole warp: uniform control flow, one elected lane issues
      constexpr uint32_t kIdescQK = idesc_f16(kBF16, C::kBM, C::kBN, false, false);
      constexpr uint32_t kIdescPV = idesc_f16(kBF16, C::kBM, D, false, true);
      const uint32_t sQ_addr = smem_u32(sQ);
      const uint32_t ring_addr = smem_u32(sRing);
      int slot = 0;
      uint32_t phase = 0;
      auto next_slot = [&]() -> int {
        const int s = slot;
        mbar_wait(&kv_full[s], phase);
        if (++slot == C::kStages) {
          slot = 0;
          phase ^= 1;
        }
        return s;
      };
      auto mma_qk = [&](int buf, int kslot) {
        const uint32_t b0 = ring_addr + kslot * C::kKVTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off_a = (kk >> 2) * (C::kBM * 128) + (kk & 3) * 32;
          const uint32_t off_b = (kk >> 2) * (C::kBN * 128) + (kk & 3) * 32;
          mma_ss_elect(tmem + C::col_s(buf), sdesc_sw128(sQ_addr + off_a, 16, 1024),
                       sdesc_sw128(b0 + off_b, 16, 1024), kIdescQK, kk > 0 ? 1u : 0u);
        }
      };
      auto mma_pv = [&](int buf, int vslot, bool accumulate) {
        const uint32_t b0 = ring_addr + vslot * C::kKVTileBytes;
#pragma unroll
        for (int kk = 0; kk < C::kBN / 16; ++kk)
          mma_ts_elect(tmem + C::kColO, tmem + C::col_s(buf) + kk * 8,
                       sdesc_sw128(b0 + kk * 16 * 128, C::kBN * 128, 1024), kIdescPV,
                       (accumulate || kk > 0) ? 1u : 0u);
      };

      mbar_wait(bar_q, 0);
      for (int t = 0; t < 2 && t < n_kv; ++t) {
        const int ks = next_slot();
        tc_fence_after();
        mma_qk(t, ks);
        mma_commit_elect(&s_full[t]);
        mma_commit_elect(&kv_empty[ks]);
      }
      for (int j = 0; j < n_kv; ++j) {
        const int buf = j & 1;
        const int vs = next_slot();
        mbar_wait(&p_full[buf], static_cast<uint32_t>(j >> 1) & 1);
        tc_fence_after();
        mma_pv(buf, vs, j > 0);
        mma_commit_elect(pv_done);
        mma_commit_elect(&kv_empty[vs]);
        if (j + 2 < n_kv) {
          const int ks = next_slot();
          tc_fence_after();
          mma_qk(buf, ks);
          mma_commit_elect(&s_full[buf]);
          mma_commit_elect(&kv_empty[ks]);
        }
      }
      mma_commit_elect(o_full);
    }
  } else {
    const int r = threadIdx.x & 127;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tO = tmem + lane_off + C::kColO;
    const float sl2 = args.scale_log2;
    const int N = args.N;
    float m = -INFINITY;
    float l = 0.0f;
    for (int j = 0; j < n_kv; ++j) {
      const int buf = j & 1;
      const uint32_t tS = tmem + lane_off + C::col_s(buf);
      mbar_wait(&s_full[buf], static_cast<uint32_t>(j >> 1) & 1);
      tc_fence_after();
      uint32_t sr[C::kBN];
      if constexpr (C::kBN == 128)
        tmem_ld32x32b_x128(tS, sr);
      else
        tmem_ld32x32b_x64(tS, sr);
      float s[C::kBN];
#pragma unroll
      for (int c = 0; c < C::kBN; ++c) s[c] = __uint_as_float(sr[c]);
      const int valid = N - j * C::kBN;
      if (valid < C::kBN) {
#pragma unroll
        for (int c = 0; c < C::kBN; ++c)
          if (c >= valid) s[c] = -INFINITY;
      }
      float mx[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mx[t] = fmaxf(s[t], s[t + 8]);
#pragma unroll
      for (int c = 16; c < C::kBN; c += 16)
#pragma unroll
        for (int t = 0; t < 8; ++t) mx[t] = fmaxf(mx[t], fmaxf(s[c + t], s[c + t + 8]));
      const float m_new = fmaxf(m, fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                         fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))));
      // conditional rescale (exact: the final (m, Sigma) pair is consistent)
      if (__any_sync(0xffffffffu, (m_new - m) * sl2 > 8.0f)) {
        const float alpha = ex2_approx((m - m_new) * sl2);
        l *= alpha;
        if (j > 0) {
          mbar_wait(pv_done, static_cast<uint32_t>(j - 1) & 1);  // O(j-1) complete
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32x32b_x32(tO + c * 32, o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32x32b_x32(tO + c * 32, o);
          }
        }
        m = m_new;
      }
      const float neg = -m * sl2;
      const bool masked = valid < C::kBN;
      uint32_t p[32];
      float rs;
      if constexpr (C::kBN == 128) {
        uint32_t p0[32], p1[32];
        rs = masked ? exp_rowsum_pack<kBF16, 0, 64, 0>(s, sl2, neg, p0)
                    : exp_rowsum_pack<kBF16, 0, 64, kEmuPer16>(s, sl2, neg, p0);
        tmem_st32x32b_x32(tS, p0);
        rs += masked ? exp_rowsum_pack<kBF16, 64, 64, 0>(s, sl2, neg, p1)
                     : exp_rowsum_pack<kBF16, 64, 64, kEmuPer16>(s, sl2, neg, p1);
        tmem_st32x32b_x32(tS + 32, p1);
        (void)p;
      } else {
        rs = masked ? exp_rowsum_pack<kBF16, 0, 64, 0>(s, sl2, neg, p)
                    : exp_rowsum_pack<kBF16, 0, 64, kEmuPer16>(s, sl2, neg, p);
        tmem_st32x32b_x32(tS, p);
      }
      l += rs;
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&p_full[buf]);
    }

    // epilogue: O staged in the (now free) Q tile buffer, TMA-stored
    mbar_wait(o_full, 0);
    tc_fence_after();
    const int row = qrow0 + r;
    stage_o_tile<D, kBF16>(tO, sQ, r, 1.0f / l);
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int c = 0; c < C::kChunks; ++c) tma_store_4d(&tmO, sQ + c * C::kBM * 128, c * 64, head, qrow0, b);
      tma_store_commit();
      tma_store_wait_all();
    }
    if (row < args.n_q && args.lse != nullptr)
      args.lse[(static_cast<int64_t>(b) * args.H + head) * N + row] = m * args.scale + logf(l);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc(tmem, C::kTmemCols);
}

}  // namespace fmha_b200
