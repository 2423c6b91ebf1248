// fmha_fwd_split_kernel.cuh -- persistent two-Q-tile ping-pong FMHA forward
// for sm_100a (head dim 64 / 128) with every softmax row split over TWO warps.
//
// Same arithmetic as fmha_fwd_kernel.cuh (fmhasim::fmha_forward,
// /root/reference/proj/src/attention.cpp:153-173: S = Q K^T :123, the online
// softmax step :36-66, O += P V :130, rowwise_finalize :68-73, + LSE), same
// work unit (one (b, head) x two 128-row Q tiles), same TMEM layout and MMA
// issue order.  What changes is the softmax: the per-row exponentials of one
// 128 x 128 score tile are the kernel's critical path (the tensor core waits
// for P before it can run PV and the next S of that Q tile), and one warp per
// TMEM lane quarter leaves each SM sub-partition with a single in-order
// instruction stream per tile.  Here a tile's 32 rows on a sub-partition are
// shared by two warps -- warp c takes score columns [64c, 64c + 64) -- so the
// sub-partition interleaves two independent exp streams:
//
//   warps 0-15  softmax: k = w & 3 (TMEM lane quarter = SM sub-partition),
//               q = (w >> 2) & 1 (Q tile), c = w >> 3 (column half)
//   warp 16     TMA producer (one lane)
//   warp 17     MMA issuer (whole warp, elect.sync issues) + TMEM allocator
//
// Per tile: each warp loads its 64 S columns (tcgen05.ld x64), reduces a
// partial row max, swaps it with its partner warp (w ^ 8: same rows, other
// half) through shared memory under a 64-thread named barrier, decides the
// (conditional) rescale identically, exponentiates its 64 scores and stores
// its P half (packed columns [32c, 32c + 32) of S_q), publishing it on
// p_full[q][c] -- the MMA warp issues the PV K-steps of each half as soon as
// that half lands.  Each warp keeps a partial row sum over its columns; the
// two partials are added in the epilogue.  O_q's rescale and the epilogue are
// split by head-dim columns the same way.  The O tile is staged in the
// swizzled TMA layout and stored by one elected thread per tile.
#pragma once

#include <cuda.h>
#include <cstdint>

#include "fmha_fwd_kernel.cuh"
#include "sm100.cuh"
#include "softmax_math.cuh"
#include "tmem_ops.cuh"

namespace fmha_b200 {

#ifndef FMHA_SPLIT_SHARED
#define FMHA_SPLIT_SHARED 0
#endif

template <int D>
struct SplitCfg {
  static_assert(D == 64 || D == 128, "this kernel handles head dim 64 and 128");
  static constexpr int kBM = 128, kBN = 128;
  static constexpr int kChunks = D / 64;
  static constexpr int kQTileBytes = kBM * D * 2;
  static constexpr int kKVTileBytes = kBN * D * 2;
#ifndef FMHA_SPLIT_STAGES
#define FMHA_SPLIT_STAGES 3
#endif
  static constexpr int kStages = D == 64 ? 8 : FMHA_SPLIT_STAGES;
  static constexpr int kQStages = D == 64 ? 2 : 1;
  static constexpr int kSmemQ = kQStages * 2 * kQTileBytes;
  static constexpr int kSmemO = kQTileBytes;
  static constexpr int kSmemRing = kStages * kKVTileBytes;
  static constexpr int kSmemRed = 2 * 2 * 2 * 128 * 4;  // partial row max / sum exchange [q][c][slot][row]
  static constexpr int kNumBars = 2 * kQStages + 2 * kStages + 2 + 4 + 2 + 2 + 2;
  static constexpr int kSmemBytes = kSmemQ + kSmemO + kSmemRing + kSmemRed + kNumBars * 8 + 16;
  static constexpr int kSmemAlloc = kSmemBytes + 1024;
  // FMHA_SPLIT_SHARED: EIGHT softmax warps, each serving BOTH Q tiles (tile 0's
  // half-rows, then tile 1's, every K/V step), so a tile's exponentials run on
  // two warps of each sub-partition with the whole MUFU to themselves.
  static constexpr bool kShared = FMHA_SPLIT_SHARED != 0;
  static constexpr int kSoftmaxWarps = kShared ? 8 : 16;
  static constexpr int kThreads = kShared ? 320 : 576;
  static constexpr int kLoadWarp = kSoftmaxWarps;
  static constexpr int kMmaWarp = kSoftmaxWarps + 1;
  static constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO0 = 256, kColO1 = 256 + D;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kPairBar = 1;   // named barriers 1..8: (q, k) partner pairs, 64 threads
  static constexpr uint32_t kTileBar = 9;   // 9, 10: the 8 warps of tile q, 256 threads
  static_assert(kSmemAlloc <= 227 * 1024, "shared memory budget");
};

template <int D, bool kBF16, int kEmuPer16>
// 576 threads: each SM sub-partition's 16K-register file holds up to 5 warps
// (sub-partitions 0 and 1: four softmax warps + the load / MMA warp), so 96
// registers per thread; the exponentials go in two 32-column chunks to fit.
__global__ void __launch_bounds__(SplitCfg<D>::kThreads, 1)
    fmha_fwd_split_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                          const FwdArgs args) {
  using C = SplitCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sO = smem + C::kSmemQ;
  uint8_t* sRing = sO + C::kSmemO;
  float* sRed = reinterpret_cast<float*>(sRing + C::kSmemRing);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRing + C::kSmemRing + C::kSmemRed);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + C::kQStages;
  uint64_t* kv_full = bars + 2 * C::kQStages;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;  // [2]
  uint64_t* p_full = s_full + 2;             // [2][2]: (tile q, column half c)
  uint64_t* o_full = p_full + 4;             // [2]
  uint64_t* o_empty = o_full + 2;            // [2]
  uint64_t* stage_free = o_empty + 2;        // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(stage_free + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_kv = args.n_kv_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kQStages; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&s_full[q], 1);
      mbar_init(&p_full[2 * q], 128);      // the 4 column-half-0 warps of tile q
      mbar_init(&p_full[2 * q + 1], 128);  // the 4 column-half-1 warps
      mbar_init(&o_full[q], 1);
      mbar_init(&o_empty[q], 256);
      mbar_init(&stage_free[q], 1);
    }
    fence_mbar_init();
  }
  if (warp == C::kMmaWarp) tmem_alloc(tmem_holder, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == C::kLoadWarp) {
    // ---------------------------------------------------- TMA producer --
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmO);
      const uint64_t keep = l2_policy_evict_last();
      const uint64_t once = l2_policy_evict_first();
      int slot = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int u = blockIdx.x; u < args.n_units; u += gridDim.x, ++i) {
        int b, head, qb;
        decode_unit(u, args.n_qblocks, args.H, b, head, qb);
        const int qrow0 = qb * 2 * C::kBM;
        const int qs = i % C::kQStages;
        mbar_wait(&q_empty[qs], (static_cast<uint32_t>(i / C::kQStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qs], 2 * C::kQTileBytes);
        uint8_t* sQs = sQ + qs * 2 * C::kQTileBytes;
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_4d_hint(&tmQ, &q_full[qs], sQs + q * C::kQTileBytes + c * C::kBM * 128, c * 64, head,
                             qrow0 + q * C::kBM, b, once);
        for (int j = 0; j < n_kv; ++j) {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            mbar_wait(&kv_empty[slot], phase ^ 1);
            mbar_arrive_expect_tx(&kv_full[slot], C::kKVTileBytes);
            uint8_t* dst = sRing + slot * C::kKVTileBytes;
#pragma unroll
            for (int c = 0; c < C::kChunks; ++c)
              tma_load_4d_hint(t == 0 ? &tmK : &tmV, &kv_full[slot], dst + c * C::kBN * 128, c * 64, head,
                               j * C::kBN, b, keep);
            if (++slot == C::kStages) {
              slot = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == C::kMmaWarp) {
    // ------------------------------------------------------ MMA issuer --
    constexpr uint32_t kIdescQK = idesc_f16(kBF16, C::kBM, C::kBN, false, false);
    constexpr uint32_t kIdescPV = idesc_f16(kBF16, C::kBM, D, false, true);
    uint32_t sQ_addr = smem_u32(sQ);
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
    auto mma_qk = [&](int q, int kslot) {
      const uint32_t a0 = sQ_addr + q * C::kQTileBytes;
      const uint32_t b0 = ring_addr + kslot * C::kKVTileBytes;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off_a = (kk >> 2) * (C::kBM * 128) + (kk & 3) * 32;
        const uint32_t off_b = (kk >> 2) * (C::kBN * 128) + (kk & 3) * 32;
        mma_ss_elect(tmem + (q ? C::kColS1 : C::kColS0), sdesc_sw128(a0 + off_a, 16, 1024),
                     sdesc_sw128(b0 + off_b, 16, 1024), kIdescQK, kk > 0 ? 1u : 0u);
      }
    };
    // O_q (+)= P_q V, K-steps 0-3 on P half 0 (kv rows 0-63), 4-7 on half 1
    auto mma_pv = [&](int q, int vslot, bool accumulate, uint32_t par) {
      const uint32_t b0 = ring_addr + vslot * C::kKVTileBytes;
      const uint32_t p0 = tmem + (q ? C::kColS1 : C::kColS0);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        mbar_wait(&p_full[q * 2 + c], par);
        tc_fence_after();
#pragma unroll
        for (int kk = 4 * c; kk < 4 * c + 4; ++kk)
          mma_ts_elect(tmem + (q ? C::kColO1 : C::kColO0), p0 + kk * 8,
                       sdesc_sw128(b0 + kk * 16 * 128, C::kBN * 128, 1024), kIdescPV,
                       (accumulate || kk > 0) ? 1u : 0u);
      }
    };
    uint32_t it = 0;
    int i = 0;
    for (int u = blockIdx.x; u < args.n_units; u += gridDim.x, ++i) {
      const uint32_t ue = (static_cast<uint32_t>(i) & 1) ^ 1;
      const int qs = i % C::kQStages;
      mbar_wait(&q_full[qs], static_cast<uint32_t>(i / C::kQStages) & 1);
      sQ_addr = smem_u32(sQ) + qs * 2 * C::kQTileBytes;
      int ks = next_slot();
      tc_fence_after();
      mma_qk(0, ks);
      mma_commit_elect(&s_full[0]);
      mma_qk(1, ks);
      mma_commit_elect(&s_full[1]);
      if (n_kv == 1) mma_commit_elect(&q_empty[qs]);
      mma_commit_elect(&kv_empty[ks]);
      for (int j = 1; j < n_kv; ++j) {
        const int vs = next_slot();
        ks = next_slot();
        const uint32_t par = it & 1;
        if (j == 1) mbar_wait(&o_empty[0], ue);
        mma_pv(0, vs, j > 1, par);
        mma_qk(0, ks);
        mma_commit_elect(&s_full[0]);
        if (j == 1) mbar_wait(&o_empty[1], ue);
        mma_pv(1, vs, j > 1, par);
        mma_qk(1, ks);
        mma_commit_elect(&s_full[1]);
        if (j == n_kv - 1) mma_commit_elect(&q_empty[qs]);
        mma_commit_elect(&kv_empty[vs]);
        mma_commit_elect(&kv_empty[ks]);
        ++it;
      }
      const int vs = next_slot();
      const uint32_t par = it & 1;
      if (n_kv == 1) mbar_wait(&o_empty[0], ue);
      mma_pv(0, vs, n_kv > 1, par);
      mma_commit_elect(&o_full[0]);
      if (n_kv == 1) mbar_wait(&o_empty[1], ue);
      mma_pv(1, vs, n_kv > 1, par);
      mma_commit_elect(&o_full[1]);
      mma_commit_elect(&kv_empty[vs]);
      ++it;
    }
  } else if constexpr (C::kShared) {
    // ------------------------------------------ softmax (8 shared warps) --
    // warp w: TMEM lane quarter k = w & 3, score columns [64c, 64c + 64) with
    // c = w >> 2, for BOTH Q tiles: per K/V step tile 0's half-rows, then tile
    // 1's.  Partner warp w ^ 4 holds the other 64 columns of the same rows.
    const int k = warp & 3;
    const int c = warp >> 2;
    const int r = k * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(k * 32) << 16;
    constexpr int kOC = D / 2;
    const float sl2 = args.scale_log2;
    const int N = args.N;
    const uint32_t pair_bar = C::kPairBar + k;
    float* red_mine = sRed + c * 256 + r;
    const float* red_other = sRed + (c ^ 1) * 256 + r;
    uint32_t e = 0;
    auto exchange = [&](float x) {
      red_mine[(e & 1) * 128] = x;
      named_bar_sync(pair_bar, 64);
      const float y = red_other[(e & 1) * 128];
      ++e;
      return y;
    };
    uint32_t it = 0;
    int i = 0;
    for (int u = blockIdx.x; u < args.n_units; u += gridDim.x, ++i) {
      int b, head, qb;
      decode_unit(u, args.n_qblocks, args.H, b, head, qb);
      float m[2] = {-INFINITY, -INFINITY};  // running row max per tile (identical in both warps of a pair)
      float l[2] = {0.0f, 0.0f};            // partial running sums over this warp's columns
      for (int j = 0; j < n_kv; ++j, ++it) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const uint32_t tS = tmem + lane_off + (q ? C::kColS1 : C::kColS0);
          const uint32_t tSc = tS + 64 * c, tPc = tS + 32 * c;
          const uint32_t tOc = tmem + lane_off + (q ? C::kColO1 : C::kColO0) + kOC * c;
          mbar_wait(&s_full[q], it & 1);
          tc_fence_after();
          uint32_t sr[64];
          tmem_ld32x32b_x64(tSc, sr);
          float s[64];
#pragma unroll
          for (int t = 0; t < 64; ++t) s[t] = __uint_as_float(sr[t]);
          const int valid = N - j * C::kBN - 64 * c;
          if (valid < 64) {
#pragma unroll
            for (int t = 0; t < 64; ++t)
              if (t >= valid) s[t] = -INFINITY;
          }
          float mx;
          {
            float a[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) a[t] = fmaxf(s[t], s[t + 4]);
#pragma unroll
            for (int t = 8; t < 64; t += 8)
#pragma unroll
              for (int x = 0; x < 4; ++x) a[x] = fmaxf(a[x], fmaxf(s[t + x], s[t + x + 4]));
            mx = fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3]));
          }
          mx = fmaxf(mx, exchange(mx));
          if (__any_sync(0xffffffffu, (mx - m[q]) * sl2 > 8.0f)) {
            const float m_new = fmaxf(mx, m[q]);
            if (j > 0) {  // O_q quiescent: S_q(j) observed => PV_q(j-1) done
              const float alpha = ex2_approx((m[q] - m_new) * sl2);
              l[q] *= alpha;
#pragma unroll
              for (int cc = 0; cc < kOC / 16; ++cc) {
                uint32_t o[16];
                tmem_ld32x32b_x16(tOc + cc * 16, o);
#pragma unroll
                for (int t = 0; t < 16; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * alpha);
                tmem_st32x32b_x16(tOc + cc * 16, o);
              }
            }
            m[q] = m_new;
          }
          const float neg = -m[q] * sl2;
          uint32_t p0[16], p1[16];
          float rs;
          if (valid < 64) {
            rs = exp_rowsum_pack<kBF16, 0, 32, 0>(s, sl2, neg, p0);
            tmem_st32x32b_x16(tPc, p0);
            rs += exp_rowsum_pack<kBF16, 32, 32, 0>(s, sl2, neg, p1);
          } else {
            rs = exp_rowsum_pack<kBF16, 0, 32, kEmuPer16>(s, sl2, neg, p0);
            tmem_st32x32b_x16(tPc, p0);
            rs += exp_rowsum_pack<kBF16, 32, 32, kEmuPer16>(s, sl2, neg, p1);
          }
          tmem_st32x32b_x16(tPc + 16, p1);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&p_full[2 * q + c]);
          l[q] += rs;
        }
      }
      // ------------------------------------------------------- epilogue --
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {
        const float l_tot = l[q] + exchange(l[q]);
        mbar_wait(&o_full[q], i & 1);
        tc_fence_after();
        if (q == 1)
          mbar_wait(&stage_free[0], static_cast<uint32_t>(i) & 1);
        else if (i > 0)
          mbar_wait(&stage_free[1], static_cast<uint32_t>(i - 1) & 1);
        const float inv = 1.0f / l_tot;
        const uint32_t tOc = tmem + lane_off + (q ? C::kColO1 : C::kColO0) + kOC * c;
#pragma unroll
        for (int cc = 0; cc < kOC / 32; ++cc) {
          uint32_t o[32];
          tmem_ld32x32b_x32(tOc + cc * 32, o);
          uint32_t h2[16];
#pragma unroll
          for (int t = 0; t < 16; ++t)
            h2[t] = pack2<kBF16>(__uint_as_float(o[2 * t]) * inv, __uint_as_float(o[2 * t + 1]) * inv);
          const int col = kOC * c + 32 * cc;
          uint8_t* rowp = sO + (col >> 6) * (C::kBM * 128) + r * 128;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int unit = (((col & 63) >> 3) + v) ^ (r & 7);  // 128-B swizzle
            st_shared_v4(rowp + unit * 16, h2[4 * v], h2[4 * v + 1], h2[4 * v + 2], h2[4 * v + 3]);
          }
        }
        tc_fence_before();
        fence_proxy_async_smem();
        mbar_arrive(&o_empty[q]);               // O_q drained from TMEM (256 arrivals)
        named_bar_sync(C::kTileBar, 256);       // all 8 warps have staged their columns
        if (warp == 0 && lane == 0) {
#pragma unroll
          for (int cc = 0; cc < C::kChunks; ++cc)
            tma_store_4d(&tmO, sO + cc * C::kBM * 128, cc * 64, head, qb * 2 * C::kBM + q * C::kBM, b);
          tma_store_commit();
          tma_store_wait_read();
          mbar_arrive(&stage_free[q]);
        }
        const int row = qb * 2 * C::kBM + q * C::kBM + r;
        if (c == 0 && row < args.n_q && args.lse != nullptr)
          args.lse[(static_cast<int64_t>(b) * args.H + head) * N + row] = m[q] * args.scale + logf(l_tot);
      }
    }
    if (warp == 0 && lane == 0) tma_store_wait_all();
  } else {
    // --------------------------------------------------------- softmax --
    const int k = warp & 3;
    const int q = (warp >> 2) & 1;
    const int c = warp >> 3;
    const int r = k * 32 + lane;  // row of the Q tile = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(k * 32) << 16;
    const uint32_t tS = tmem + lane_off + (q ? C::kColS1 : C::kColS0);
    const uint32_t tSc = tS + 64 * c;        // this warp's 64 score columns
    const uint32_t tPc = tS + 32 * c;        // its packed P half
    constexpr int kOC = D / 2;               // O columns per warp
    const uint32_t tOc = tmem + lane_off + (q ? C::kColO1 : C::kColO0) + kOC * c;
    const float sl2 = args.scale_log2;
    const int N = args.N;
    const uint32_t a_s_full = smem_u32(&s_full[q]);
    const uint32_t a_p_full = smem_u32(&p_full[2 * q + c]);
    const uint32_t a_o_full = smem_u32(&o_full[q]);
    const uint32_t a_o_empty = smem_u32(&o_empty[q]);
    const uint32_t pair_bar = C::kPairBar + q * 4 + k;
    // exchange slots with the partner warp, double-buffered: a value written
    // to slot e & 1 is read by the partner after the pair barrier, and the
    // slot is rewritten only after the NEXT exchange's barrier, which the
    // partner reaches only once it has read it -- one barrier per exchange
    float* red_mine = sRed + (q * 2 + c) * 256 + r;
    const float* red_other = sRed + (q * 2 + (c ^ 1)) * 256 + r;
    uint32_t e = 0;
    auto exchange = [&](float x) {
      red_mine[(e & 1) * 128] = x;
      named_bar_sync(pair_bar, 64);
      const float y = red_other[(e & 1) * 128];
      ++e;
      return y;
    };
    uint32_t it = 0;
    int i = 0;
    for (int u = blockIdx.x; u < args.n_units; u += gridDim.x, ++i) {
      int b, head, qb;
      decode_unit(u, args.n_qblocks, args.H, b, head, qb);
      float m = -INFINITY;  // running row max (raw score units), identical in both warps of a pair
      float l = 0.0f;       // partial running sum over this warp's columns

      for (int j = 0; j < n_kv; ++j, ++it) {
        mbar_wait_addr(a_s_full, it & 1);
        tc_fence_after();
        uint32_t sr[64];
        tmem_ld32x32b_x64(tSc, sr);
        float s[64];
#pragma unroll
        for (int t = 0; t < 64; ++t) s[t] = __uint_as_float(sr[t]);
        const int valid = N - j * C::kBN - 64 * c;  // columns >= valid are padding
        if (valid < 64) {
#pragma unroll
          for (int t = 0; t < 64; ++t)
            if (t >= valid) s[t] = -INFINITY;
        }
        float mx;
        {
          float a[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) a[t] = fmaxf(s[t], s[t + 4]);
#pragma unroll
          for (int t = 8; t < 64; t += 8)
#pragma unroll
            for (int e = 0; e < 4; ++e) a[e] = fmaxf(a[e], fmaxf(s[t + e], s[t + e + 4]));
          mx = fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3]));
        }
        // the partner's partial max (same rows, other 64 columns)
        mx = fmaxf(mx, exchange(mx));
        // conditional rescale (exact: the final (m, Sigma) pair is consistent);
        // both warps of a pair see the same rows and take the same decision
        if (__any_sync(0xffffffffu, (mx - m) * sl2 > 8.0f)) {
          const float m_new = fmaxf(mx, m);
          if (j > 0) {  // O_q quiescent: S_q(j) observed => PV_q(j-1) done
            const float alpha = ex2_approx((m - m_new) * sl2);
            l *= alpha;
#pragma unroll
            for (int cc = 0; cc < kOC / 16; ++cc) {
              uint32_t o[16];
              tmem_ld32x32b_x16(tOc + cc * 16, o);
#pragma unroll
              for (int t = 0; t < 16; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * alpha);
              tmem_st32x32b_x16(tOc + cc * 16, o);
            }
          }
          m = m_new;
        }
        const float neg = -m * sl2;
        uint32_t p0[16], p1[16];
        float rs;
        if (valid < 64) {  // padded tile: all-MUFU (exact zeros for -inf scores)
          rs = exp_rowsum_pack<kBF16, 0, 32, 0>(s, sl2, neg, p0);
          tmem_st32x32b_x16(tPc, p0);
          rs += exp_rowsum_pack<kBF16, 32, 32, 0>(s, sl2, neg, p1);
        } else {
          rs = exp_rowsum_pack<kBF16, 0, 32, kEmuPer16>(s, sl2, neg, p0);
          tmem_st32x32b_x16(tPc, p0);
          rs += exp_rowsum_pack<kBF16, 32, 32, kEmuPer16>(s, sl2, neg, p1);
        }
        tmem_st32x32b_x16(tPc + 16, p1);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive_addr(a_p_full);
        l += rs;
      }

      // ------------------------------------------------------- epilogue --
      // total row sum = both warps' partials; O_q columns of this warp ->
      // x(1/Sigma) -> 16-bit -> swizzled staging tile -> TMA store
      const float l_tot = l + exchange(l);
      mbar_wait_addr(a_o_full, i & 1);
      tc_fence_after();
      // staging tile turns: tile 0 of unit i, tile 1 of unit i, tile 0 of unit i+1 ...
      if (q == 1)
        mbar_wait(&stage_free[0], static_cast<uint32_t>(i) & 1);
      else if (i > 0)
        mbar_wait(&stage_free[1], static_cast<uint32_t>(i - 1) & 1);
      const float inv = 1.0f / l_tot;
#pragma unroll
      for (int cc = 0; cc < kOC / 32; ++cc) {
        uint32_t o[32];
        tmem_ld32x32b_x32(tOc + cc * 32, o);
        uint32_t h2[16];
#pragma unroll
        for (int t = 0; t < 16; ++t)
          h2[t] = pack2<kBF16>(__uint_as_float(o[2 * t]) * inv, __uint_as_float(o[2 * t + 1]) * inv);
        const int col = kOC * c + 32 * cc;  // first O column of this chunk
        uint8_t* rowp = sO + (col >> 6) * (C::kBM * 128) + r * 128;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int unit = (((col & 63) >> 3) + v) ^ (r & 7);  // 128-B swizzle
          st_shared_v4(rowp + unit * 16, h2[4 * v], h2[4 * v + 1], h2[4 * v + 2], h2[4 * v + 3]);
        }
      }
      tc_fence_before();
      fence_proxy_async_smem();
      mbar_arrive_addr(a_o_empty);  // O_q drained from TMEM (256 arrivals)
      named_bar_sync(C::kTileBar + q, 256);  // the tile's 8 warps have staged their columns
      if (warp == 4 * q && lane == 0) {
#pragma unroll
        for (int cc = 0; cc < C::kChunks; ++cc)
          tma_store_4d(&tmO, sO + cc * C::kBM * 128, cc * 64, head, qb * 2 * C::kBM + q * C::kBM, b);
        tma_store_commit();
        tma_store_wait_read();
        mbar_arrive(&stage_free[q]);
      }
      const int row = qb * 2 * C::kBM + q * C::kBM + r;
      if (c == 0 && row < args.n_q && args.lse != nullptr)
        args.lse[(static_cast<int64_t>(b) * args.H + head) * N + row] = m * args.scale + logf(l_tot);
    }
    if (warp == 4 * q && lane == 0) tma_store_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc(tmem, C::kTmemCols);
}

}  // namespace fmha_b200
