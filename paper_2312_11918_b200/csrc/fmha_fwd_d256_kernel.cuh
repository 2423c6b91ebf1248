// fmha_fwd_d256_kernel.cuh -- FMHA forward for head dim 256 on sm_100a.
//
// Same contract as fmha_fwd_kernel.cuh (fmhasim::fmha_forward,
// /root/reference/proj/src/attention.cpp:153-173) but shaped for d = 256,
// where the O accumulator alone needs 256 TMEM columns and a 128 x 256
// 16-bit K or V tile is 64 KB:
//
//   CTA = one (b, head) and ONE 128-row Q tile; K/V tiles of 64 rows.
//   TMEM: S buffers A [0,64) and B [64,128) (double-buffered so the tensor
//         core computes S(j+1) while softmax works on S(j)); O [256,512).
//         P(j) (16-bit) aliases the first 32 columns of its S buffer.
//   smem: Q 64 KB + 4-slot K/V ring of 32 KB = 192 KB.
//   warps 0-3 softmax (thread per row), warp 4 TMA producer, warp 5 MMA.
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
#include "tmem_ops.cuh"

namespace fmha_b200 {

struct FwdCfgD256 {
  static constexpr int D = 256;
  static constexpr int kBM = 128;
  static constexpr int kBN = 64;
  static constexpr int kChunks = 4;
  static constexpr int kQTileBytes = kBM * D * 2;    // 64 KB
  static constexpr int kKVTileBytes = kBN * D * 2;   // 32 KB
  static constexpr int kStages = 4;
  static constexpr int kSmemRing = kStages * kKVTileBytes;
  static constexpr int kNumBars = 1 + 2 * kStages + 2 + 2 + 2;
  static constexpr int kSmemBytes = kQTileBytes + kSmemRing + kNumBars * 8 + 16;
  static constexpr int kSmemAlloc = kSmemBytes + 1024;
  static constexpr int kThreads = 192;
  static constexpr int kLoadWarp = 4;
  static constexpr int kMmaWarp = 5;
  __host__ __device__ static constexpr uint32_t col_s(int buf) { return buf ? 64u : 0u; }
  static constexpr uint32_t kColO = 256;
  static constexpr uint32_t kTmemCols = 512;
};

template <bool kBF16>
__global__ void __launch_bounds__(192, 1)
    fmha_fwd_d256_kernel(const __grid_constant__ CUtensorMap tmQ,
                         const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, const FwdArgs args) {
  using C = FwdCfgD256;
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
      // item t: K_{t/2} (t even) or V_{t/2} (t odd); slot t % S, use (t / S)
      for (int t = 0; t < 2 * n_kv; ++t) {
        const int slot = t % C::kStages;
        const uint32_t use = static_cast<uint32_t>(t / C::kStages);
        mbar_wait(&kv_empty[slot], (use & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[slot], C::kKVTileBytes);
        uint8_t* dst = sRing + slot * C::kKVTileBytes;
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_4d_hint((t & 1) ? &tmV : &tmK, &kv_full[slot], dst + c * C::kBN * 128, c * 64,
                           head, (t >> 1) * C::kBN, b, keep);
      }
    }
  } else if (warp == C::kMmaWarp) {
    {  // whole warp: uniform control flow, one elected lane issues
      constexpr uint32_t kIdescQK = idesc_f16(kBF16, C::kBM, C::kBN, false, false);
      constexpr uint32_t kIdescPV = idesc_f16(kBF16, C::kBM, D, false, true);
      const uint32_t sQ_addr = smem_u32(sQ);
      const uint32_t ring_addr = smem_u32(sRing);
      auto wait_item = [&](int t) -> int {
        const int slot = t % C::kStages;
        mbar_wait(&kv_full[slot], static_cast<uint32_t>(t / C::kStages) & 1);
        return slot;
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
        const int ks = wait_item(2 * t);
        tc_fence_after();
        mma_qk(t, ks);
        mma_commit_elect(&s_full[t]);
        mma_commit_elect(&kv_empty[ks]);
      }
      for (int j = 0; j < n_kv; ++j) {
        const int buf = j & 1;
        const int vs = wait_item(2 * j + 1);
        mbar_wait(&p_full[buf], static_cast<uint32_t>(j >> 1) & 1);
        tc_fence_after();
        mma_pv(buf, vs, j > 0);
        mma_commit_elect(pv_done);
        mma_commit_elect(&kv_empty[vs]);
        if (j + 2 < n_kv) {
          const int ks = wait_item(2 * (j + 2));
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
      float mx0 = s[0], mx1 = s[1], mx2 = s[2], mx3 = s[3];
#pragma unroll
      for (int c = 4; c < 64; c += 4) {
        mx0 = fmaxf(mx0, s[c]);
        mx1 = fmaxf(mx1, s[c + 1]);
        mx2 = fmaxf(mx2, s[c + 2]);
        mx3 = fmaxf(mx3, s[c + 3]);
      }
      const float m_new = fmaxf(m, fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)));
      const bool need = (m_new - m) * sl2 > 8.0f;
      if (__any_sync(0xffffffffu, need)) {
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
      float rs0 = 0.f, rs1 = 0.f, rs2 = 0.f, rs3 = 0.f;
      uint32_t p[32];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float e0 = ex2_approx(fmaf(s[2 * i], sl2, neg));
        const float e1 = ex2_approx(fmaf(s[2 * i + 1], sl2, neg));
        const float e2 = ex2_approx(fmaf(s[2 * i + 2], sl2, neg));
        const float e3 = ex2_approx(fmaf(s[2 * i + 3], sl2, neg));
        rs0 += e0;
        rs1 += e1;
        rs2 += e2;
        rs3 += e3;
        p[i] = pack2<kBF16>(e0, e1);
        p[i + 1] = pack2<kBF16>(e2, e3);
      }
      tmem_st32x32b_x32(tS, p);
      l += (rs0 + rs1) + (rs2 + rs3);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&p_full[buf]);
    }

    mbar_wait(o_full, 0);
    tc_fence_after();
    const int row = qrow0 + r;
    const bool row_ok = row < N;
    const float inv = 1.0f / l;
    uint16_t* orow = reinterpret_cast<uint16_t*>(args.o) + static_cast<int64_t>(b) * args.o_sb +
                     static_cast<int64_t>(row_ok ? row : 0) * args.o_sn +
                     static_cast<int64_t>(head) * args.o_sh;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      tmem_ld32x32b_x32(tO + c * 32, o);
      uint32_t h2[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        h2[i] = pack2<kBF16>(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
      if (row_ok) {
#pragma unroll
        for (int v = 0; v < 4; ++v)
          st_global_v4(orow + c * 32 + v * 8, h2[4 * v], h2[4 * v + 1], h2[4 * v + 2],
                       h2[4 * v + 3]);
      }
    }
    if (row_ok && args.lse != nullptr)
      args.lse[(static_cast<int64_t>(b) * args.H + head) * N + row] = m * args.scale + logf(l);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc(tmem, C::kTmemCols);
}

}  // namespace fmha_b200
