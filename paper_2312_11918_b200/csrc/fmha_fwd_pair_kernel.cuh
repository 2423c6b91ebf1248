// fmha_fwd_pair_kernel.cuh -- forward pass on CTA pairs (cta_group::2): head
// dim 256 (kBN = 128, one CTA per SM) and head dim 128 at long sequence
// lengths (kBN = 64, two CTAs of different pairs per SM).
//
// Same contract as the other forward kernels (fmhasim::fmha_forward,
// /root/reference/proj/src/attention.cpp:153-173); same per-CTA structure as
// fmha_fwd_st_kernel.cuh (one 128-row Q tile per CTA, double-buffered S in
// TMEM), but the two CTAs of a 2-CTA cluster -- adjacent Q tiles of one
// (b, head) -- run every GEMM as ONE M = 256 tcgen05.mma issued by the
// leader CTA (shown for d = 256, kBN = 128):
//
//   S = Q K^T   M256 N128 K256: A = each CTA's own Q tile, B = K tile split
//               by kv rows: CTA r holds K rows [64r, 64r+64) (32 KB);
//   O += P V    M256 N256 K128: A = P from each CTA's own TMEM, B = V tile
//               split by head-dim columns: CTA r holds V[:, 128r, 128r+128).
//
// Each SM therefore streams HALF of every K/V tile (64 KB per 128-row step
// instead of 128 KB) -- at d = 256 the single-CTA kernel is bound by the
// chip's L2 -> SM delivery rate (profiles/r01_microbench.txt) -- and the
// half-tiles make a deeper ring in the same shared memory (5 x 32 KB vs
// 2 x 64 KB).  At d = 128, kBN = 64: M256 N64 S GEMMs, M256 N128 PV GEMMs,
// 8 KB half-tiles in an 8-slot ring, TMEM 256 columns per CTA.
//
// Protocol (mbarriers; "L" = lives in the leader CTA only):
//   bar_q  L  both CTAs' Q TMA complete on it (two Q tiles expected)
//   kv_full[s] L  both halves of slot s
//   kv_empty[s]  per CTA; the leader's MMA commit arrives in both CTAs
//   s_full[2], pv_done, o_full  per CTA; multicast commits from the leader
//   p_full[2] L  one arrival per softmax warp of BOTH CTAs (count 8)
// Only the leader's MMA warp issues; the peer's MMA warp just co-allocates
// TMEM.  Launch: cluster (2,1,1) over the Q-tile axis; an odd Q-tile count
// is padded with one tile past N (zero-filled by TMA, nothing stored).
#pragma once

#include <cuda.h>
#include <cstdint>

#include "fmha_fwd_kernel.cuh"
#include "sm100.cuh"
#include "sm100_pair.cuh"
#include "softmax_math.cuh"
#include "tmem_ops.cuh"

namespace fmha_b200 {

// Head dim D, K/V step kBN.  TMEM per CTA: S buffers [0,kBN) [kBN,2kBN),
// O [2kBN, 2kBN+D), allocated as the next power of two; 2kBN + D <= 256
// fits two CTAs (of two different pairs) per SM.
template <int D_, int kBN_>
struct FwdCfgPair {
  static constexpr int D = D_;
  static constexpr int kBM = 128;  // Q rows per CTA (256 per pair)
  static constexpr int kBN = kBN_;  // K/V rows per step
  static_assert(D == 128 || D == 256, "V is split into 64-column chunks per CTA");
  static_assert(kBN == 64 || kBN == 128, "K/V step");
  static constexpr int kChunks = D / 64;
  static constexpr int kQTileBytes = kBM * D * 2;
  static constexpr int kSlotBytes = kBN * D * 2 / 2;       // half a K or V tile
  static constexpr int kKRowsPerCta = kBN / 2;             // K split by kv rows
  static constexpr int kVColsPerCta = D / 2;               // V split by head-dim columns
  static constexpr uint32_t kTmemCols = (2 * kBN + D) <= 256 ? 256u : 512u;
  static constexpr int kCtasPerSm = kTmemCols == 256 ? 2 : 1;
  static constexpr int kRingBudget = (kCtasPerSm == 2 ? 112 * 1024 : 226 * 1024) - kQTileBytes - 1024 - 256;
  static constexpr int kStagesFit = kRingBudget / kSlotBytes;
  static constexpr int kStages = kStagesFit > 8 ? 8 : kStagesFit;
  static_assert(kStages >= 2, "K/V ring needs two slots");
  static constexpr int kSmemRing = kStages * kSlotBytes;
  static constexpr int kNumBars = 1 + 2 * kStages + 2 + 2 + 2;
  static constexpr int kSmemBytes = kQTileBytes + kSmemRing + kNumBars * 8 + 16;
  static constexpr int kSmemAlloc = kSmemBytes + 1024;
  static constexpr uint32_t kColO = 2 * kBN;
  static constexpr int kThreads = 192;
  static constexpr int kLoadWarp = 4;
  static constexpr int kMmaWarp = 5;
  __host__ __device__ static constexpr uint32_t col_s(int buf) { return buf ? static_cast<uint32_t>(kBN) : 0u; }
  static_assert(kSmemAlloc <= 227 * 1024, "shared memory budget");
};

#ifndef FMHA_PAIR_K4
#define FMHA_PAIR_K4 0  // batched tcgen05 issue (four K-steps per elect.sync; measured neutral: off)
#endif
constexpr bool kPairK4 = FMHA_PAIR_K4 != 0;

template <int D_, int kBN_, bool kBF16, int kEmuPer16 = 4>
__global__ void __launch_bounds__(192, FwdCfgPair<D_, kBN_>::kCtasPerSm)
    fmha_fwd_pair_kernel(const __grid_constant__ CUtensorMap tmQ,  // box 128 rows
                         const __grid_constant__ CUtensorMap tmK,  // box kBN/2 rows
                         const __grid_constant__ CUtensorMap tmV,  // box kBN rows
                         const __grid_constant__ CUtensorMap tmO,  // box 128 rows (epilogue TMA store)
                         const FwdArgs args) {
  using C = FwdCfgPair<D_, kBN_>;
  constexpr int D = C::D;
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
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
    }
    mbar_init(pv_done, 1);
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == C::kMmaWarp) tmem_alloc_pair(tmem_holder, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' barriers initialised before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == C::kLoadWarp) {
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      const uint64_t keep = l2_policy_evict_last();
      const uint64_t once = l2_policy_evict_first();
      if (leader) mbar_arrive_expect_tx(bar_q, 2 * C::kQTileBytes);
      const uint32_t q_bar = mapa_shared(bar_q, 0);
#pragma unroll
      for (int c = 0; c < C::kChunks; ++c)
        tma_load_4d_pair(&tmQ, q_bar, sQ + c * C::kBM * 128, c * 64, head, qrow0, b, once);
      int slot = 0;
      uint32_t phase = 0;
      auto acquire = [&]() -> uint8_t* {
        mbar_wait(&kv_empty[slot], phase ^ 1);
        if (leader) mbar_arrive_expect_tx(&kv_full[slot], 2 * C::kSlotBytes);
        return sRing + slot * C::kSlotBytes;
      };
      auto advance = [&]() {
        if (++slot == C::kStages) {
          slot = 0;
          phase ^= 1;
        }
      };
      auto load_k = [&](int step) {  // kv rows [64 rank, +64) of the tile, 4 d-chunks
        uint8_t* dst = acquire();
        const uint32_t fb = mapa_shared(&kv_full[slot], 0);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_4d_pair(&tmK, fb, dst + c * C::kKRowsPerCta * 128, c * 64, head,
                           step * C::kBN + static_cast<int>(rank) * C::kKRowsPerCta, b, keep);
        advance();
      };
      auto load_v = [&](int step) {  // head-dim columns [128 rank, +128), 2 chunks of 128 rows
        uint8_t* dst = acquire();
        const uint32_t fb = mapa_shared(&kv_full[slot], 0);
#pragma unroll
        for (int c = 0; c < C::kVColsPerCta / 64; ++c)
          tma_load_4d_pair(&tmV, fb, dst + c * C::kBN * 128,
                           (static_cast<int>(rank) * (C::kVColsPerCta / 64) + c) * 64, head, step * C::kBN,
                           b, keep);
        advance();
      };
      // consumption order of the MMA warp: K0 K1 | V0 K2 | V1 K3 | ...
      load_k(0);
      if (n_kv > 1) load_k(1);
      for (int j = 0; j < n_kv; ++j) {
        load_v(j);
        if (j + 2 < n_kv) load_k(j + 2);
      }
      // drain: every slot released, so no commit from the leader is still in
      // flight towards this CTA's barriers when it exits
      for (int s = 0; s < C::kStages; ++s) {
        mbar_wait(&kv_empty[slot], phase ^ 1);
        advance();
      }
    }
  } else if (warp == C::kMmaWarp) {
    if (leader) {  // whole warp: uniform control flow, one elected lane issues
      constexpr uint32_t kIdescQK = idesc_f16(kBF16, 2 * C::kBM, C::kBN, false, false);
      constexpr uint32_t kIdescPV = idesc_f16(kBF16, 2 * C::kBM, D, false, true);
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
        const uint32_t b0 = ring_addr + kslot * C::kSlotBytes;
        if constexpr (kPairK4) {  // four K-steps per elect.sync, one batch per 64-column atom of d
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c)
            mma_pair_ss_k4(tmem + C::col_s(buf), sdesc_sw128(sQ_addr + c * (C::kBM * 128), 16, 1024),
                           sdesc_sw128(b0 + c * (C::kKRowsPerCta * 128), 16, 1024), kIdescQK, c > 0 ? 1u : 0u);
          return;
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off_a = (kk >> 2) * (C::kBM * 128) + (kk & 3) * 32;
          const uint32_t off_b = (kk >> 2) * (C::kKRowsPerCta * 128) + (kk & 3) * 32;
          mma_pair_ss_elect(tmem + C::col_s(buf), sdesc_sw128(sQ_addr + off_a, 16, 1024),
                            sdesc_sw128(b0 + off_b, 16, 1024), kIdescQK, kk > 0 ? 1u : 0u);
        }
      };
      auto mma_pv = [&](int buf, int vslot, bool accumulate) {
        const uint32_t b0 = ring_addr + vslot * C::kSlotBytes;
        if constexpr (kPairK4) {
#pragma unroll
          for (int c = 0; c < C::kBN / 64; ++c)
            mma_pair_ts_k4(tmem + C::kColO, tmem + C::col_s(buf) + c * 32,
                           sdesc_sw128(b0 + c * 4 * 16 * 128, C::kBN * 128, 1024), kIdescPV,
                           (accumulate || c > 0) ? 1u : 0u);
          return;
        }
#pragma unroll
        for (int kk = 0; kk < C::kBN / 16; ++kk)
          mma_pair_ts_elect(tmem + C::kColO, tmem + C::col_s(buf) + kk * 8,
                            sdesc_sw128(b0 + kk * 16 * 128, C::kBN * 128, 1024), kIdescPV,
                            (accumulate || kk > 0) ? 1u : 0u);
      };

      mbar_wait(bar_q, 0);
      tc_fence_after();
      for (int t = 0; t < 2 && t < n_kv; ++t) {
        const int ks = next_slot();
        tc_fence_after();
        mma_qk(t, ks);
        mma_commit_pair_elect(&s_full[t]);
        mma_commit_pair_elect(&kv_empty[ks]);
      }
      for (int j = 0; j < n_kv; ++j) {
        const int buf = j & 1;
        const int vs = next_slot();
        mbar_wait_cluster(&p_full[buf], static_cast<uint32_t>(j >> 1) & 1);
        tc_fence_after();
        mma_pv(buf, vs, j > 0);
        mma_commit_pair_elect(pv_done);
        mma_commit_pair_elect(&kv_empty[vs]);
        if (j + 2 < n_kv) {
          const int ks = next_slot();
          tc_fence_after();
          mma_qk(buf, ks);
          mma_commit_pair_elect(&s_full[buf]);
          mma_commit_pair_elect(&kv_empty[ks]);
        }
      }
      mma_commit_pair_elect(o_full);
    }
  } else {
    const int r = threadIdx.x & 127;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tO = tmem + lane_off + C::kColO;
    const float sl2 = args.scale_log2;
    const int N = args.N;
    const uint32_t p_bar[2] = {mapa_shared(&p_full[0], 0), mapa_shared(&p_full[1], 0)};
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
      uint32_t p0[32];
      float rs = masked ? exp_rowsum_pack<kBF16, 0, 64, 0>(s, sl2, neg, p0)
                        : exp_rowsum_pack<kBF16, 0, 64, kEmuPer16>(s, sl2, neg, p0);
      tmem_st32x32b_x32(tS, p0);
      if constexpr (C::kBN == 128) {
        uint32_t p1[32];
        rs += masked ? exp_rowsum_pack<kBF16, 64, 64, 0>(s, sl2, neg, p1)
                     : exp_rowsum_pack<kBF16, 64, 64, kEmuPer16>(s, sl2, neg, p1);
        tmem_st32x32b_x32(tS + 32, p1);
      }
      l += rs;
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(p_bar[buf]);
    }

    // epilogue: O -> x(1/Sigma) (rowwise_finalize) -> 16-bit -> staged in
    // this CTA's Q tile buffer (free: o_full follows the last S GEMM) in the
    // swizzled TMA layout -> one TMA store per 64 columns (rows past n_q,
    // e.g. a padding CTA's, are clipped by the tensor map)
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
  cluster_sync();  // neither CTA releases TMEM / exits while the pair still works
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc_pair(tmem, C::kTmemCols);
}

}  // namespace fmha_b200
