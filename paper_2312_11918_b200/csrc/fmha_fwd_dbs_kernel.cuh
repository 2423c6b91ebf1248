// fmha_fwd_dbs_kernel.cuh -- persistent FMHA forward for sm_100a, head dim
// 128, with DOUBLE-BUFFERED S: one 128-row Q tile per work unit, two S
// accumulators in Tensor Memory, so the tensor core computes S(j+1) while the
// softmax of S(j) runs, and the softmax of one tile is spread over EIGHT warps
// (two per TMEM lane quarter, 16 rows each, a row over the 4 threads of a quad).
//
// Replaces the arithmetic of fmhasim::fmha_forward
// (/root/reference/proj/src/attention.cpp:153-173): per (b, head) and
// 128-row Q tile, stream 128-row K/V tiles (KBLK), S = Q K^T (GEMM-I,
// attention.cpp:123), the online softmax update (online_softmax_step,
// attention.cpp:36-66), O += P V (GEMM-II, attention.cpp:130), the final
// O *= 1/Sigma (rowwise_finalize, attention.cpp:68-73) and LSE = m + ln Sigma.
//
// Why: in the two-Q-tile ping-pong kernel each tile's chain
// softmax(j) -> PV(j) -> S(j+1) -> softmax(j+1) is serial, so the K/V step
// period is the softmax latency (one warp per row group, ~1.9k clk) plus
// 1024 clk of tensor work.  Here S(j+1) is already in TMEM when softmax(j)
// finishes; the period is max(tensor work 1024 clk, softmax latency,
// (tensor + softmax + issue latency) / 2).
//
// The CTA walks a flat sequence of K/V steps g = 0, 1, 2, ... over its units
// (unit i = blockIdx.x + i * gridDim.x, n_kv steps each); S(g) lives in TMEM
// buffer g & 1, so consecutive steps always alternate buffers, also across
// unit boundaries.  MMA issue order:
//     S(0) S(1) | PV(0) S(2) | PV(1) S(3) | ... | PV(G-1)
// (tcgen05 ops from one thread execute in order, so S(g+2) overwrites
// buffer g & 1 only after PV(g) has read P(g) from it).
//
//   warps 0-7   softmax: warp w owns TMEM lanes 32*(w%4) + 16*(w/4) .. +15
//   warps 8-11  epilogue: O(unit) -> x 1/Sigma -> 16-bit -> swizzled smem
//               stage, LSE (one row per thread, lane quarter w%4)
//   warp 12     TMA producer (one lane)      warp 13  MMA issuer + TMEM alloc
//   warp 14     O store (TMA, one lane)      warp 15  idle
//
// Tensor Memory (512 columns):  S0 [0,128)  S1 [128,256)  O0 [256,384)
// O1 [384,512); O alternates per unit so unit i+1's first PV never waits for
// unit i's epilogue.  P(g) (16-bit, packed 2 per column) overwrites the first
// 64 columns of its S buffer.
//
// Shared memory: Q double-buffered (2 x 32 KB, the next unit's Q loads while
// the current unit runs), 4 x 32 KB K/V ring, 32 KB O staging tile, the
// per-row softmax statistics of the finished unit (1 KB), mbarriers.
//
// Rescaling is conditional (FlashAttention-4 style): a warp keeps its stale
// row maxima unless some row's max grew by more than 8 in log2 units; then it
// waits for PV(g-1) to complete (one mbarrier phase per PV) and rescales its
// rows of O in TMEM before publishing P(g).
#pragma once

#include <cuda.h>
#include <cstdint>

#include "fmha_fwd_kernel.cuh"
#include "sm100.cuh"
#include "softmax_math.cuh"
#include "tmem_ops.cuh"

namespace fmha_b200 {

struct FwdCfgDbs {
  static constexpr int D = 128;
  static constexpr int kBM = 128;  // Q rows per unit (UMMA M)
  static constexpr int kBN = 128;  // K/V rows per step
  static constexpr int kChunks = D / 64;
  static constexpr int kQTileBytes = kBM * D * 2;
  static constexpr int kKVTileBytes = kBN * D * 2;
  static constexpr int kStages = 4;   // K/V ring slots (one K or one V tile each)
  static constexpr int kQStages = 2;
  static constexpr int kSmemQ = kQStages * kQTileBytes;
  static constexpr int kSmemO = kQTileBytes;
  static constexpr int kSmemRing = kStages * kKVTileBytes;
  static constexpr int kSmemStats = 2 * kBM * 4;  // m (raw) and Sigma per row
  static constexpr int kNumBars = 2 * kQStages + 2 * kStages + 2 + 4 + 1 + 2 + 2 + 1 + 2;
  static constexpr int kSmemBytes = kSmemQ + kSmemO + kSmemRing + kSmemStats + kNumBars * 8 + 16;
  static constexpr int kSmemAlloc = kSmemBytes + 1024;
  static constexpr int kThreads = 512;
  static constexpr int kEpiWarp0 = 8;
  static constexpr int kLoadWarp = 12;
  static constexpr int kMmaWarp = 13;
  static constexpr int kStoreWarp = 14;
  static constexpr uint32_t kColS = 0, kColO = 256;  // S_b at 128 b, O_u at 256 + 128 u
  static constexpr uint32_t kTmemCols = 512;
  static_assert(kSmemAlloc <= 227 * 1024, "shared memory budget");
};
#ifndef FMHA_IDLE_SLEEP_NS
#define FMHA_IDLE_SLEEP_NS 256  // epilogue / O-store polls (a whole unit of slack)
#endif
#ifndef FMHA_PRODUCER_SLEEP_NS
#define FMHA_PRODUCER_SLEEP_NS 64  // TMA producer polls (~2 K/V steps of slack)
#endif
#ifndef FMHA_SOFTMAX_SLEEP_NS
#define FMHA_SOFTMAX_SLEEP_NS 0  // softmax waits for S: 0 = hardware try_wait loop
#endif
#ifndef FMHA_DBS_SPEC
#define FMHA_DBS_SPEC 1  // speculative first half (exponentials against the previous maxima)
#endif
constexpr bool kDbsSpec = FMHA_DBS_SPEC != 0;
#ifndef FMHA_DBS_LANE_ARRIVE
#define FMHA_DBS_LANE_ARRIVE 1  // P published by lane 0 of each softmax warp (8 arrivals)
#endif
constexpr bool kLaneArrive = FMHA_DBS_LANE_ARRIVE != 0;
constexpr uint32_t kPArrivals = kLaneArrive ? 8 : 256;
#ifndef FMHA_DBS_PREFETCH
#define FMHA_DBS_PREFETCH 4  // K/V L2 prefetch distance in steps (0: off)
#endif
constexpr int kDbsPrefetch = FMHA_DBS_PREFETCH;
constexpr uint32_t kIdleSleepNs = FMHA_IDLE_SLEEP_NS, kProducerSleepNs = FMHA_PRODUCER_SLEEP_NS,
                   kSoftmaxSleepNs = FMHA_SOFTMAX_SLEEP_NS;

// Debug timeline (-DFMHA_TRACE_BUILD, tools/trace_dbs.py): clock64 stamps of
// CTA 0 for its first kTraceSteps K/V steps, trace[g * 16 + k]:
//   softmax warp 0: 0 S observed  1 S in registers  2 max + vote done
//                   3 half-0 exps done  4 P half 0 published  5 P half 1 published
//   softmax warp 4: 6 S observed  7 P half 1 published
//   MMA warp:       8 V(g) ready  9 P(g) half 0 seen  10 P(g) half 1 seen
//                   11 PV(g) issued  12 K(g+2) ready  13 S(g+2) issued
constexpr int kTraceSteps = 64;
__device__ __forceinline__ void dbs_stamp(const FwdArgs& a, bool on, int g, int k) {
#ifdef FMHA_TRACE_BUILD
  if (on && g < kTraceSteps) a.trace[g * 16 + k] = clock64();
#endif
}
// per softmax warp w (lane 0): trace[kTraceSteps * 16 + (g * 8 + w) * 4 + k],
// k = 0 S observed, 1 max + vote done, 2 P half 0 published, 3 P half 1 published
__device__ __forceinline__ void dbs_wstamp(const FwdArgs& a, bool on, int g, int w, int k) {
#ifdef FMHA_TRACE_BUILD
  if (on && g < kTraceSteps) a.trace[kTraceSteps * 16 + (g * 8 + w) * 4 + k] = clock64();
#endif
}

template <bool kBF16, int kEmuPer16 = 4>
__global__ void __launch_bounds__(512, 1)
    fmha_fwd_dbs_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                        const FwdArgs args) {
  using C = FwdCfgDbs;
  constexpr int D = C::D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sO = sQ + C::kSmemQ;
  uint8_t* sRing = sO + C::kSmemO;
  float* stat_m = reinterpret_cast<float*>(sRing + C::kSmemRing);  // [128]
  float* stat_l = stat_m + C::kBM;                                 // [128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(stat_l + C::kBM);
  uint64_t* q_full = bars;                        // [2]
  uint64_t* q_empty = q_full + C::kQStages;       // [2]
  uint64_t* kv_full = q_empty + C::kQStages;      // [kStages]
  uint64_t* kv_empty = kv_full + C::kStages;      // [kStages]
  uint64_t* s_full = kv_empty + C::kStages;       // [2]   S(g) in buffer g & 1
  uint64_t* p_full = s_full + 2;                  // [2][2] (buffer, half of the kv columns)
  uint64_t* pv_done = p_full + 4;                 // one phase per PV
  uint64_t* o_full = pv_done + 1;                 // [2]   O of unit i complete (buffer i & 1)
  uint64_t* o_empty = o_full + 2;                 // [2]   O buffer + statistics read by the epilogue
  uint64_t* stat_full = o_empty + 2;              // statistics of unit i written
  uint64_t* stage_ready = stat_full + 1;          // O staged (128 epilogue threads)
  uint64_t* stage_free = stage_ready + 1;         // staging tile read by the TMA store
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(stage_free + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_kv = args.n_kv_tiles;
  // this CTA's units and K/V steps
  const int n_my = args.n_units > static_cast<int>(blockIdx.x)
                       ? (args.n_units - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                       : 0;
  const int G = n_my * n_kv;
#ifdef FMHA_TRACE_BUILD
  const bool tr = args.trace != nullptr && blockIdx.x == 0;
#else
  constexpr bool tr = false;
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kQStages; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[2 * b], kPArrivals);
      mbar_init(&p_full[2 * b + 1], kPArrivals);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 128);
    }
    mbar_init(pv_done, 1);
    mbar_init(stat_full, 256);
    mbar_init(stage_ready, 128);
    mbar_init(stage_free, 1);
    fence_mbar_init();
  }
  if (warp == C::kMmaWarp) tmem_alloc(tmem_holder, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp >= 12) {
    reg_dealloc<56>();
    if (warp == C::kLoadWarp) {
      // -------------------------------------------------- TMA producer --
      // Ring order = MMA consumption order: K(0) K(1) | V(0) K(2) | V(1) K(3) ...
      // with unit i's Q loaded just before its first K.
      if (lane == 0 && G > 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        tma_prefetch_desc(&tmO);
        const uint64_t keep = l2_policy_evict_last();   // K/V re-read by sibling CTAs
        const uint64_t once = l2_policy_evict_first();  // Q read once
        int slot = 0;
        uint32_t phase = 0;
        // K and V streams walk (unit, step) incrementally: one decode per unit
        struct Cursor {
          int i, j, b, head, qb;
        };
        auto decode = [&](Cursor& c) {
          decode_unit(static_cast<int>(blockIdx.x) + c.i * static_cast<int>(gridDim.x), args.n_qblocks, args.H,
                      c.b, c.head, c.qb);
        };
        auto advance = [&](Cursor& c) {
          if (++c.j == n_kv) {
            c.j = 0;
            ++c.i;
            decode(c);
          }
        };
        Cursor ck{0, 0, 0, 0, 0}, cv{0, 0, 0, 0, 0};
        decode(ck);
        decode(cv);
        auto load = [&](const CUtensorMap* map, const Cursor& c, bool is_k) {
          if (is_k && c.j == 0) {  // first K of unit i: its Q first
            const int qs = c.i & 1;
            mbar_wait_backoff(&q_empty[qs], ((c.i >> 1) & 1) ^ 1, kProducerSleepNs);
            mbar_arrive_expect_tx(&q_full[qs], C::kQTileBytes);
#pragma unroll
            for (int ch = 0; ch < C::kChunks; ++ch)
              tma_load_4d_hint(&tmQ, &q_full[qs], sQ + qs * C::kQTileBytes + ch * C::kBM * 128, ch * 64, c.head,
                               c.qb * C::kBM, c.b, once);
          }
          mbar_wait_backoff(&kv_empty[slot], phase ^ 1, kProducerSleepNs);
          mbar_arrive_expect_tx(&kv_full[slot], C::kKVTileBytes);
          uint8_t* dst = sRing + slot * C::kKVTileBytes;
#pragma unroll
          for (int ch = 0; ch < C::kChunks; ++ch)
            tma_load_4d_hint(map, &kv_full[slot], dst + ch * C::kBN * 128, ch * 64, c.head, c.j * C::kBN, c.b, keep);
          if (++slot == C::kStages) {
            slot = 0;
            phase ^= 1;
          }
        };
        load(&tmK, ck, true);
        advance(ck);
        if (G > 1) {
          load(&tmK, ck, true);
          advance(ck);
        }
        // L2 prefetch of step g + kDbsPrefetch's K and V when step g's V is
        // loaded: the first CTA to touch a K/V tile otherwise pays the HBM
        // latency inside the ring's ~2-step lead (measured: ~2.9k clk TMA
        // latency per tile, tools/trace_dbs.py)
        Cursor cp{0, 0, 0, 0, 0};
        decode(cp);
        for (int t = 0; t < kDbsPrefetch && t < G; ++t) advance(cp);
        for (int g = 0; g < G; ++g) {
          if (kDbsPrefetch > 0 && g + kDbsPrefetch < G) {
#pragma unroll
            for (int ch = 0; ch < C::kChunks; ++ch) {
              tma_prefetch_4d(&tmK, ch * 64, cp.head, cp.j * C::kBN, cp.b);
              tma_prefetch_4d(&tmV, ch * 64, cp.head, cp.j * C::kBN, cp.b);
            }
            advance(cp);
          }
          load(&tmV, cv, false);
          advance(cv);
          if (g + 2 < G) {
            load(&tmK, ck, true);
            advance(ck);
          }
        }
      }
    } else if (warp == C::kMmaWarp) {
      // ---------------------------------------------------- MMA issuer --
      constexpr uint32_t kIdescQK = idesc_f16(kBF16, C::kBM, C::kBN, false, false);
      constexpr uint32_t kIdescPV = idesc_f16(kBF16, C::kBM, D, false, true);
      const uint32_t q_addr = smem_u32(sQ);
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
      // S(g) = Q_i K_j^T into buffer g & 1 (K-major SW128 operands); (si, sj)
      // walk the S stream, two steps ahead of the PV stream
      int si = 0, sj = 0;
      auto issue_s = [&](int g) {
        const int qs = si & 1;
        if (sj == 0) mbar_wait(&q_full[qs], (si >> 1) & 1);
        const int ks = next_slot();
        dbs_stamp(args, tr && lane == 0, g - 2, 12);
        tc_fence_after();
        const uint32_t a0 = q_addr + qs * C::kQTileBytes;
        const uint32_t b0 = ring_addr + ks * C::kKVTileBytes;
        const uint32_t d_tmem = tmem + C::kColS + (g & 1) * 128;
        // two batched issues of four K=16 steps (one per 64-column swizzle atom of d)
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          mma_ss_k4(d_tmem, sdesc_sw128(a0 + c * (C::kBM * 128), 16, 1024), sdesc_sw128(b0 + c * (C::kBN * 128), 16, 1024),
                    kIdescQK, c > 0 ? 1u : 0u);
        dbs_stamp(args, tr && lane == 0, g - 2, 13);
        mma_commit_elect(&s_full[g & 1]);
        mma_commit_elect(&kv_empty[ks]);
        if (sj == n_kv - 1) mma_commit_elect(&q_empty[qs]);  // last read of Q_i issued
        dbs_stamp(args, tr && lane == 0, g - 2, 14);
        if (++sj == n_kv) {
          sj = 0;
          ++si;
        }
      };
      if (G > 0) issue_s(0);
      if (G > 1) issue_s(1);
      int i = 0, j = 0;
      for (int g = 0; g < G; ++g) {
        const int ob = i & 1;
        const int b = g & 1;
        const uint32_t par = static_cast<uint32_t>(g >> 1) & 1;
        dbs_stamp(args, tr && lane == 0, g, 15);
        const int vs = next_slot();
        dbs_stamp(args, tr && lane == 0, g, 8);
        if (j == 0 && i >= 2) mbar_wait(&o_empty[ob], ((i >> 1) & 1) ^ 1);  // epilogue of unit i-2 done
        const uint32_t p0 = tmem + C::kColS + b * 128;
        const uint32_t o_tmem = tmem + C::kColO + ob * 128;
        const uint32_t v0 = ring_addr + vs * C::kKVTileBytes;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mbar_wait(&p_full[2 * b + h], par);
          dbs_stamp(args, tr && lane == 0, g, 9 + h);
          tc_fence_after();
          mma_ts_k4(o_tmem, p0 + h * 32, sdesc_sw128(v0 + h * 64 * 128, C::kBN * 128, 1024), kIdescPV,
                    (j > 0 || h > 0) ? 1u : 0u);
        }
        dbs_stamp(args, tr && lane == 0, g, 11);
        mma_commit_elect(pv_done);
        mma_commit_elect(&kv_empty[vs]);
        if (j == n_kv - 1) mma_commit_elect(&o_full[ob]);
        if (g + 2 < G) issue_s(g + 2);
        if (++j == n_kv) {
          j = 0;
          ++i;
        }
      }
    } else if (warp == C::kStoreWarp) {
      // ------------------------------------------------- O store warp --
      if (lane == 0) {
        for (int i = 0; i < n_my; ++i) {
          int b, head, qb;
          decode_unit(static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x), args.n_qblocks, args.H, b,
                      head, qb);
          mbar_wait_backoff(stage_ready, static_cast<uint32_t>(i) & 1, kIdleSleepNs);
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c)
            tma_store_4d(&tmO, sO + c * C::kBM * 128, c * 64, head, qb * C::kBM, b);
          tma_store_commit();
          tma_store_wait_read();
          mbar_arrive(stage_free);
        }
        tma_store_wait_all();
      }
    }
  } else if (warp >= 8) {
    reg_dealloc<104>();
    // ---------------------------------------------------- epilogue WG --
    // rowwise_finalize (attention.cpp:68-73) + LSE, one row per thread.
    const int r = (warp - C::kEpiWarp0) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    for (int i = 0; i < n_my; ++i) {
      int b, head, qb;
      decode_unit(static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x), args.n_qblocks, args.H, b, head,
                  qb);
      const int ob = i & 1;
      mbar_wait_backoff(&o_full[ob], (i >> 1) & 1, kIdleSleepNs);
      mbar_wait_backoff(stat_full, static_cast<uint32_t>(i) & 1, kIdleSleepNs);
      tc_fence_after();
      const float m = stat_m[r];
      const float l = stat_l[r];
      if (i > 0) mbar_wait_backoff(stage_free, static_cast<uint32_t>(i - 1) & 1, kIdleSleepNs);
      stage_o_tile<D, kBF16>(tmem + lane_off + C::kColO + ob * 128, sO, r, 1.0f / l);
      tc_fence_before();
      fence_proxy_async_smem();  // staged O visible to the TMA (async proxy)
      mbar_arrive(&o_empty[ob]);  // O buffer and statistics consumed
      mbar_arrive(stage_ready);
      const int row = qb * C::kBM + r;
      if (row < args.n_q && args.lse != nullptr)
        args.lse[(static_cast<int64_t>(b) * args.H + head) * args.N + row] = m * args.scale + logf(l);
    }
  } else {
    reg_alloc<176>();
    // -------------------------------------------------- softmax warps --
    // Thread t of warp w: rows r0 = 32*(w%4) + 16*(w/4) + t/4 and r1 = r0 + 8,
    // columns 8c + 2*(t%4) + {0, 1} of each 8-column group c (16x256b shape);
    // a row's maxima / sums combine over the quad with two shuffles.
    const int lb = (warp & 3) * 32 + (warp >> 2) * 16;
    const uint32_t lane_base = static_cast<uint32_t>(lb) << 16;
    const int quad = lane & 3;
    const int r0 = lb + (lane >> 2);
    const float sl2 = args.scale_log2;
    const int N = args.N;
    // P publication: every thread arrives (kLaneArrive = 0) or lane 0 after
    // the warp's TMEM stores are complete (one mbarrier op per warp)
    auto publish_p = [&](uint64_t* bar) {
      if constexpr (kLaneArrive) {
        __syncwarp();
        if (lane == 0) mbar_arrive(bar);
      } else {
        mbar_arrive(bar);
      }
    };
    int g = 0;
    for (int i = 0; i < n_my; ++i) {
      const int ob = i & 1;
      const uint32_t tO = tmem + lane_base + C::kColO + ob * 128;
      float m0 = -INFINITY, m1 = -INFINITY;  // running row maxima (raw score units)
      float l0 = 0.f, l1 = 0.f;              // this thread's partial row sums
      for (int j = 0; j < n_kv; ++j, ++g) {
        const int bsel = g & 1;
        const uint32_t tS = tmem + lane_base + C::kColS + bsel * 128;
        if constexpr (kSoftmaxSleepNs > 0)
          mbar_wait_backoff(&s_full[bsel], static_cast<uint32_t>(g >> 1) & 1, kSoftmaxSleepNs);
        else
          mbar_wait(&s_full[bsel], static_cast<uint32_t>(g >> 1) & 1);
        dbs_stamp(args, tr && threadIdx.x == 0, g, 0);
        dbs_wstamp(args, tr && lane == 0, g, warp, 0);
        dbs_stamp(args, tr && threadIdx.x == 128, g, 6);
        tc_fence_after();
        const int valid = N - j * C::kBN;  // columns >= valid are padding
        const bool masked = valid < C::kBN;
        // s[4c .. 4c+3]: group c (kv columns 8c + 2*quad + {0,1}) of rows r0, r0 + 8
        float s[64];
        // row maxima of groups [c0, c1) into (mx0, mx1), before the quad reduction
        auto group_max = [](const float (&v)[64], int c0, int c1, float& mx0, float& mx1) {
          float a0 = fmaxf(v[4 * c0], v[4 * c0 + 1]), a1 = fmaxf(v[4 * c0 + 2], v[4 * c0 + 3]);
          float b0 = fmaxf(v[4 * c0 + 4], v[4 * c0 + 5]), b1 = fmaxf(v[4 * c0 + 6], v[4 * c0 + 7]);
#pragma unroll
          for (int c = c0 + 2; c < c1; c += 2) {
            a0 = fmaxf(a0, fmaxf(v[4 * c], v[4 * c + 1]));
            a1 = fmaxf(a1, fmaxf(v[4 * c + 2], v[4 * c + 3]));
            b0 = fmaxf(b0, fmaxf(v[4 * c + 4], v[4 * c + 5]));
            b1 = fmaxf(b1, fmaxf(v[4 * c + 6], v[4 * c + 7]));
          }
          mx0 = fmaxf(a0, b0);
          mx1 = fmaxf(a1, b1);
        };
        auto quad_max = [&](float& mx0, float& mx1) {
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        };
        // new running maxima; for j > 0, O must hold PV(g-1): wait for its
        // completion, then rescale this warp's 16 rows of O in TMEM
        auto raise_max = [&](float mx0, float mx1) {
          const float n0 = fmaxf(mx0, m0), n1 = fmaxf(mx1, m1);
          if (j > 0) {
            const float al0 = ex2_approx((m0 - n0) * sl2), al1 = ex2_approx((m1 - n1) * sl2);
            l0 *= al0;
            l1 *= al1;
            mbar_wait(pv_done, static_cast<uint32_t>(g - 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[16];
              tmem_ld16x256b_x4(tO + c * 32, o);
#pragma unroll
              for (int t = 0; t < 16; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * ((t & 2) ? al1 : al0));
              tmem_st16x256b_x4(tO + c * 32, o);
            }
          }
          m0 = n0;
          m1 = n1;
        };
        auto grew = [&](float mx0, float mx1) {
          return __any_sync(0xffffffffu, (mx0 - m0) * sl2 > 8.0f || (mx1 - m1) * sl2 > 8.0f);
        };
        // P = 2^(s*c - m*c): packed pairs, half h = kv columns [64h, 64h+64)
        // = P columns [32h, 32h+32).  16x128b register order: (r0, r1) per group.
        // (padded tiles take an all-MUFU copy: exact zeros for -inf scores;
        // kEmu is a template argument so no predicated-off MUFU is issued)
        const uint64_t c2 = f2_pack(sl2, sl2);
        uint64_t acc0 = f2_pack(0.f, 0.f), acc1 = f2_pack(0.f, 0.f);
        auto exp_half = [&]<int kEmu>(int h, uint32_t (&p)[16]) {
          const uint64_t nm0 = f2_pack(-m0 * sl2, -m0 * sl2), nm1 = f2_pack(-m1 * sl2, -m1 * sl2);
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            const int c = 8 * h + cc;
            const uint64_t x0 = ffma2(f2_pack(s[4 * c], s[4 * c + 1]), c2, nm0);
            const uint64_t x1 = ffma2(f2_pack(s[4 * c + 2], s[4 * c + 3]), c2, nm1);
            const uint64_t e0 = emulate_pair<kEmu>(2 * c) ? exp2_poly_x2(x0) : exp2_mufu_x2(x0);
            const uint64_t e1 = emulate_pair<kEmu>(2 * c + 1) ? exp2_poly_x2(x1) : exp2_mufu_x2(x1);
            acc0 = fadd2(acc0, e0);
            acc1 = fadd2(acc1, e1);
            p[2 * cc] = pack2_x2<kBF16>(e0);
            p[2 * cc + 1] = pack2_x2<kBF16>(e1);
          }
        };
        uint32_t ph0[16], ph1[16];
        if (kDbsSpec && j > 0 && !masked) {
          // Speculative step: kv columns 0-63 are loaded and exponentiated
          // against the previous maxima while columns 64-127 load; the half is
          // redone only if some row's max grew by more than 8 in log2 units.
          uint32_t sra[32], srb[32];
          tmem_ld16x256b_x8(tS, sra);
          tmem_ld16x256b_x8_nowait(tS + 64, srb);
#pragma unroll
          for (int k = 0; k < 32; ++k) s[k] = __uint_as_float(sra[k]);
          dbs_stamp(args, tr && threadIdx.x == 0, g, 1);
          exp_half.template operator()<kEmuPer16>(0, ph0);
          float ma0, ma1, mb0, mb1;
          group_max(s, 0, 8, ma0, ma1);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) s[32 + k] = __uint_as_float(srb[k]);
          group_max(s, 8, 16, mb0, mb1);
          float mx0 = fmaxf(ma0, mb0), mx1 = fmaxf(ma1, mb1);
          quad_max(mx0, mx1);
          dbs_stamp(args, tr && threadIdx.x == 0, g, 2);
          dbs_wstamp(args, tr && lane == 0, g, warp, 1);
          if (grew(mx0, mx1)) {
            raise_max(mx0, mx1);
            acc0 = f2_pack(0.f, 0.f);
            acc1 = f2_pack(0.f, 0.f);
            exp_half.template operator()<kEmuPer16>(0, ph0);
          }
          dbs_stamp(args, tr && threadIdx.x == 0, g, 3);
          tmem_st16x128b_x8(tS, ph0);
          exp_half.template operator()<kEmuPer16>(1, ph1);
        } else {
          uint32_t sr[64];
          tmem_ld16x256b_x16(tS, sr);
#pragma unroll
          for (int k = 0; k < 64; ++k) s[k] = __uint_as_float(sr[k]);
          dbs_stamp(args, tr && threadIdx.x == 0, g, 1);
          if (masked) {
#pragma unroll
            for (int k = 0; k < 64; ++k)
              if ((k >> 2) * 8 + 2 * quad + (k & 1) >= valid) s[k] = -INFINITY;
          }
          float mx0, mx1;
          group_max(s, 0, 16, mx0, mx1);
          quad_max(mx0, mx1);
          if (grew(mx0, mx1)) raise_max(mx0, mx1);
          dbs_stamp(args, tr && threadIdx.x == 0, g, 2);
          dbs_wstamp(args, tr && lane == 0, g, warp, 1);
          if (masked)
            exp_half.template operator()<0>(0, ph0);
          else
            exp_half.template operator()<kEmuPer16>(0, ph0);
          dbs_stamp(args, tr && threadIdx.x == 0, g, 3);
          tmem_st16x128b_x8(tS, ph0);
          if (masked)
            exp_half.template operator()<0>(1, ph1);
          else
            exp_half.template operator()<kEmuPer16>(1, ph1);
        }
        tmem_wait_st();
        tc_fence_before();
        publish_p(&p_full[2 * bsel]);
        dbs_stamp(args, tr && threadIdx.x == 0, g, 4);
        dbs_wstamp(args, tr && lane == 0, g, warp, 2);
        tmem_st16x128b_x8(tS + 32, ph1);
        {
          float x, y;
          f2_unpack(acc0, x, y);
          l0 += x + y;
          f2_unpack(acc1, x, y);
          l1 += x + y;
        }
        tmem_wait_st();
        tc_fence_before();
        publish_p(&p_full[2 * bsel + 1]);
        dbs_stamp(args, tr && threadIdx.x == 0, g, 5);
        dbs_wstamp(args, tr && lane == 0, g, warp, 3);
        dbs_stamp(args, tr && threadIdx.x == 128, g, 7);
      }
      // unit done: row sums over the quad, statistics for the epilogue WG
      l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
      l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
      l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
      l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
      if (i > 0) mbar_wait(&o_empty[(i - 1) & 1], static_cast<uint32_t>((i - 1) >> 1) & 1);  // stats of i-1 read
      if (quad == 0) {
        stat_m[r0] = m0;
        stat_l[r0] = l0;
        stat_m[r0 + 8] = m1;
        stat_l[r0 + 8] = l1;
      }
      mbar_arrive(stat_full);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc(tmem, C::kTmemCols);
}

}  // namespace fmha_b200
