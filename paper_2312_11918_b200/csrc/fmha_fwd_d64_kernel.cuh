// fmha_fwd_d64_kernel.cuh -- head dim 64: two-Q-tile ping-pong with 64-row
// K/V steps, TWO CTAs per SM.
//
// Same contract as the other forward kernels (fmhasim::fmha_forward,
// /root/reference/proj/src/attention.cpp:153-173).  At d = 64 the tensor core
// has slack (S + PV per 128x128 tile is half the d = 128 work) and the
// softmax alone sets the pace: with one CTA per SM (fmha_fwd_kernel.cuh) each
// SM sub-partition runs two softmax warps that mostly wait on their own
// S -> softmax -> P -> PV -> S chain.  Here the same ping-pong uses 64-column
// S tiles, so a CTA needs S0 S1 O0 O1 = 4 x 64 TMEM columns (256) and two CTAs
// share an SM: four softmax warps per sub-partition, four Q tiles in flight.
//
//   CTA: persistent, units = (b, head, two 128-row Q tiles); 320 threads:
//        warps 0-3 softmax Q tile 0, 4-7 softmax Q tile 1 (thread = row =
//        TMEM lane), warp 8 TMA producer, warp 9 MMA issuer.  No register
//        reallocation (640 threads per SM leave ~100 registers per thread).
//   smem: Q 2 x 16 KB, K/V ring 7 x 8 KB (64 rows x 128 B), one 16 KB O
//        staging tile shared by the two WGs in turns, barriers.
//   TMEM: S0 [0,64) S1 [64,128) O0 [128,192) O1 [192,256); P (16-bit)
//        aliases the first 32 columns of its S tile (TS-form PV MMA).
//   MMA order per unit: S0(0) S1(0) | PV0(j-1) S0(j) PV1(j-1) S1(j) | ... |
//        PV0(n-1) PV1(n-1); in-order completion makes "S_q(j) done" imply
//        "PV_q(j-1) done" (conditional O rescale without an extra barrier).
//   Epilogue: O_q -> x(1/Sigma) -> 16-bit -> the swizzled staging tile (the
//        two WGs take it in turns: WG0 unit i, WG1 unit i, WG0 unit i+1, ...)
//        -> one TMA store issued by the WG's first thread, which releases the
//        tile to the other WG once the store has read it; + LSE.
#pragma once

#include <cuda.h>
#include <cstdint>

#include "fmha_fwd_kernel.cuh"
#include "sm100.cuh"
#include "softmax_math.cuh"
#include "tmem_ops.cuh"

namespace fmha_b200 {

struct FwdCfgD64 {
  static constexpr int D = 64;
  static constexpr int kBM = 128;
  static constexpr int kBN = 64;
  static constexpr int kQTileBytes = kBM * D * 2;    // 16 KB
  static constexpr int kKVTileBytes = kBN * D * 2;   // 8 KB
  static constexpr int kStages = 7;
  static constexpr int kSmemQ = 2 * kQTileBytes;
  static constexpr int kSmemO = kQTileBytes;  // epilogue staging, shared by both WGs
  static constexpr int kSmemRing = kStages * kKVTileBytes;
  static constexpr int kNumBars = 2 + 2 * kStages + 2 + 2 + 2 + 2 + 2;
  static constexpr int kSmemBytes = kSmemQ + kSmemO + kSmemRing + kNumBars * 8 + 16;
  static constexpr int kSmemAlloc = kSmemBytes + 1024;
  static constexpr int kThreads = 320;
  static constexpr int kLoadWarp = 8;
  static constexpr int kMmaWarp = 9;
  static constexpr uint32_t kColS0 = 0, kColS1 = 64, kColO0 = 128, kColO1 = 192;
  static constexpr uint32_t kTmemCols = 256;
  static_assert(kSmemAlloc <= 112 * 1024, "two CTAs per SM");
};

#ifndef FMHA_D64_K4
#define FMHA_D64_K4 1  // batched tcgen05 issue (four K-steps per elect.sync): +1.5 % on Table-1 d=64
#endif
constexpr bool kD64K4 = FMHA_D64_K4 != 0;
#ifndef FMHA_D64_FUSED
#define FMHA_D64_FUSED 0  // PV + S + commit of a tile step in one elect.sync block
#endif
constexpr bool kD64Fused = FMHA_D64_FUSED != 0;

template <bool kBF16, int kEmuPer16 = 4>
__global__ void __launch_bounds__(320, 2)
    fmha_fwd_d64_kernel(const __grid_constant__ CUtensorMap tmQ,  // box 128 rows
                        const __grid_constant__ CUtensorMap tmK,  // box 64 rows
                        const __grid_constant__ CUtensorMap tmV,  // box 64 rows
                        const __grid_constant__ CUtensorMap tmO,  // box 128 rows (epilogue TMA store)
                        const FwdArgs args) {
  using C = FwdCfgD64;
  constexpr int D = C::D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sO = smem + C::kSmemQ;
  uint8_t* sRing = sO + C::kSmemO;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRing + C::kSmemRing);
  uint64_t* q_full = bars;                   // [1]
  uint64_t* q_empty = bars + 1;              // [1]
  uint64_t* kv_full = bars + 2;              // [kStages]
  uint64_t* kv_empty = kv_full + C::kStages;  // [kStages]
  uint64_t* s_full = kv_empty + C::kStages;  // [2]
  uint64_t* p_full = s_full + 2;             // [2]
  uint64_t* o_full = p_full + 2;             // [2]
  uint64_t* o_empty = o_full + 2;            // [2]
  uint64_t* stage_free = o_empty + 2;        // [2]: WG q's use of the staging tile read by its store
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(stage_free + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_kv = args.n_kv_tiles;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&s_full[q], 1);
      mbar_init(&p_full[q], 4);  // one arrival per softmax warp
      mbar_init(&o_full[q], 1);
      mbar_init(&o_empty[q], 4);
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
    // ------------------------------------------------------ TMA producer --
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      const uint64_t keep = l2_policy_evict_last();
      const uint64_t once = l2_policy_evict_first();
      int slot = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int u = blockIdx.x; u < args.n_units; u += gridDim.x, ++i) {
        int b, head, qb;
        decode_unit(u, args.n_qblocks, args.H, b, head, qb);
        const int qrow0 = qb * 2 * C::kBM;
        mbar_wait(q_empty, (static_cast<uint32_t>(i) & 1) ^ 1);  // last S GEMMs of unit i-1 done
        mbar_arrive_expect_tx(q_full, 2 * C::kQTileBytes);
#pragma unroll
        for (int q = 0; q < 2; ++q)
          tma_load_4d_hint(&tmQ, q_full, sQ + q * C::kQTileBytes, 0, head, qrow0 + q * C::kBM, b, once);
        for (int j = 0; j < n_kv; ++j) {
#pragma unroll
          for (int t = 0; t < 2; ++t) {  // K(j), V(j): the MMA warp's consumption order
            mbar_wait(&kv_empty[slot], phase ^ 1);
            mbar_arrive_expect_tx(&kv_full[slot], C::kKVTileBytes);
            tma_load_4d_hint(t == 0 ? &tmK : &tmV, &kv_full[slot], sRing + slot * C::kKVTileBytes, 0, head,
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
    // -------------------------------------------------------- MMA issuer --
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
    // S_q = Q_q K^T: M128 N64, K = 64 in 4 steps of 32 B inside the swizzle atom
    auto mma_qk = [&](int q, int kslot) {
      const uint32_t a0 = sQ_addr + q * C::kQTileBytes;
      const uint32_t b0 = ring_addr + kslot * C::kKVTileBytes;
      if constexpr (kD64K4) {  // the four K-steps in one elect.sync batch
        mma_ss_k4(tmem + (q ? C::kColS1 : C::kColS0), sdesc_sw128(a0, 16, 1024), sdesc_sw128(b0, 16, 1024),
                  kIdescQK, 0u);
        return;
      }
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        mma_ss_elect(tmem + (q ? C::kColS1 : C::kColS0), sdesc_sw128(a0 + kk * 32, 16, 1024),
                     sdesc_sw128(b0 + kk * 32, 16, 1024), kIdescQK, kk > 0 ? 1u : 0u);
    };
    // O_q (+)= P_q V: M128 N64, K = 64 kv rows in 4 steps of 16 (P from TMEM)
    auto mma_pv = [&](int q, int vslot, bool accumulate, uint32_t par) {
      const uint32_t b0 = ring_addr + vslot * C::kKVTileBytes;
      const uint32_t p0 = tmem + (q ? C::kColS1 : C::kColS0);
      mbar_wait(&p_full[q], par);
      tc_fence_after();
      if constexpr (kD64K4) {
        mma_ts_k4(tmem + (q ? C::kColO1 : C::kColO0), p0, sdesc_sw128(b0, C::kBN * 128, 1024), kIdescPV,
                  accumulate ? 1u : 0u);
        return;
      }
#pragma unroll
      for (int kk = 0; kk < C::kBN / 16; ++kk)
        mma_ts_elect(tmem + (q ? C::kColO1 : C::kColO0), p0 + kk * 8,
                     sdesc_sw128(b0 + kk * 16 * 128, C::kBN * 128, 1024), kIdescPV,
                     (accumulate || kk > 0) ? 1u : 0u);
    };

    uint32_t it = 0;  // global K/V-step counter (p_full parity)
    int i = 0;
    for (int u = blockIdx.x; u < args.n_units; u += gridDim.x, ++i) {
      const uint32_t ue = (static_cast<uint32_t>(i) & 1) ^ 1;  // o_empty parity
      mbar_wait(q_full, static_cast<uint32_t>(i) & 1);
      int ks = next_slot();
      tc_fence_after();
      mma_qk(0, ks);
      mma_commit_elect(&s_full[0]);
      mma_qk(1, ks);
      mma_commit_elect(&s_full[1]);
      if (n_kv == 1) mma_commit_elect(q_empty);
      mma_commit_elect(&kv_empty[ks]);
      for (int j = 1; j < n_kv; ++j) {
        const int vs = next_slot();
        ks = next_slot();
        const uint32_t par = it & 1;
        if (j == 1) {  // previous unit's epilogue drained O0 / O1
          mbar_wait(&o_empty[0], ue);
          mbar_wait(&o_empty[1], ue);
        }
        // fixed order (measured: issuing whichever tile's P is ready first,
        // polling both barriers, is 3 % slower)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if constexpr (kD64Fused) {  // PV, S and the s_full commit in one issue block
            mbar_wait(&p_full[q], par);
            tc_fence_after();
            mma_pv_qk_commit_k4(tmem + (q ? C::kColO1 : C::kColO0), tmem + (q ? C::kColS1 : C::kColS0),
                                sdesc_sw128(ring_addr + vs * C::kKVTileBytes, C::kBN * 128, 1024), kIdescPV,
                                j > 1 ? 1u : 0u, tmem + (q ? C::kColS1 : C::kColS0),
                                sdesc_sw128(sQ_addr + q * C::kQTileBytes, 16, 1024),
                                sdesc_sw128(ring_addr + ks * C::kKVTileBytes, 16, 1024), kIdescQK, &s_full[q]);
          } else {
            mma_pv(q, vs, j > 1, par);
            mma_qk(q, ks);
            mma_commit_elect(&s_full[q]);
          }
        }
        if (j == n_kv - 1) mma_commit_elect(q_empty);  // last reads of Q issued
        if constexpr (kD64Fused) {
          mma_commit2_elect(&kv_empty[vs], &kv_empty[ks]);
        } else {
          mma_commit_elect(&kv_empty[vs]);
          mma_commit_elect(&kv_empty[ks]);
        }
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
  } else {
    // ----------------------------------------------- softmax WG 0 / 1 --
    const int q = warp >> 2;
    const int r = threadIdx.x & 127;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_off + (q ? C::kColS1 : C::kColS0);
    const uint32_t tO = tmem + lane_off + (q ? C::kColO1 : C::kColO0);
    const float sl2 = args.scale_log2;
    const int N = args.N;
    uint32_t it = 0;
    int i = 0;
    for (int u = blockIdx.x; u < args.n_units; u += gridDim.x, ++i) {
      int b, head, qb;
      decode_unit(u, args.n_qblocks, args.H, b, head, qb);
      float m = -INFINITY;
      float l = 0.0f;
      for (int j = 0; j < n_kv; ++j, ++it) {
        mbar_wait(&s_full[q], it & 1);
        tc_fence_after();
        uint32_t sr[64];
        tmem_ld32x32b_x64(tS, sr);
        float s[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) s[c] = __uint_as_float(sr[c]);
        const int valid = N - j * C::kBN;
        if (valid < C::kBN) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c >= valid) s[c] = -INFINITY;
        }
        float mx[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) mx[t] = fmaxf(s[t], s[t + 8]);
#pragma unroll
        for (int c = 16; c < 64; c += 16)
#pragma unroll
          for (int t = 0; t < 8; ++t) mx[t] = fmaxf(mx[t], fmaxf(s[c + t], s[c + t + 8]));
        const float m_tile = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                   fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        // conditional rescale (exact: the final (m, Sigma) pair is consistent);
        // O_q is quiescent here: S_q(j) done => PV_q(j-1) done
        if (__any_sync(0xffffffffu, (m_tile - m) * sl2 > 8.0f)) {
          const float m_new = fmaxf(m_tile, m);
          if (j > 0) {
            const float alpha = ex2_approx((m - m_new) * sl2);
            l *= alpha;
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[32];
              tmem_ld32x32b_x32(tO + c * 32, o);
#pragma unroll
              for (int t = 0; t < 32; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * alpha);
              tmem_st32x32b_x32(tO + c * 32, o);
            }
          }
          m = m_new;
        }
        const float neg = -m * sl2;
        uint32_t p[32];
        const float rs = valid < C::kBN ? exp_rowsum_pack<kBF16, 0, 64, 0>(s, sl2, neg, p)
                                        : exp_rowsum_pack<kBF16, 0, 64, kEmuPer16>(s, sl2, neg, p);
        tmem_st32x32b_x32(tS, p);
        l += rs;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[q]);
      }

      // epilogue (rowwise_finalize, attention.cpp:68-73): O_q -> x(1/Sigma)
      // -> 16-bit -> the swizzled staging tile -> TMA store.  The WGs take
      // the tile in strict turns: before writing, wait until the OTHER WG's
      // latest use has been read by its store (that use waited for this WG's
      // previous one, so the parity wait is exact).
      mbar_wait(&o_full[q], static_cast<uint32_t>(i) & 1);
      tc_fence_after();
      if (q == 1)
        mbar_wait(&stage_free[0], static_cast<uint32_t>(i) & 1);
      else if (i > 0)
        mbar_wait(&stage_free[1], static_cast<uint32_t>(i - 1) & 1);
      stage_o_tile<D, kBF16>(tO, sO, r, 1.0f / l);
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[q]);  // O_q drained from TMEM
      named_bar_sync(1 + q, 128);                // the WG's 128 rows staged
      if (r == 0) {
        tma_store_4d(&tmO, sO, 0, head, qb * 2 * C::kBM + q * C::kBM, b);
        tma_store_commit();
        tma_store_wait_read();
        mbar_arrive(&stage_free[q]);
      }
      const int row = qb * 2 * C::kBM + q * C::kBM + r;
      if (row < args.n_q && args.lse != nullptr)
        args.lse[(static_cast<int64_t>(b) * args.H + head) * N + row] = m * args.scale + logf(l);
    }
    if (r == 0) tma_store_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc(tmem, C::kTmemCols);
}

}  // namespace fmha_b200
