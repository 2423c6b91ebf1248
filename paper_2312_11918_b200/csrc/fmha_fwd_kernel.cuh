// fmha_fwd_kernel.cuh -- persistent, warp-specialised FMHA forward for
// sm_100a, head dim 64 / 128.
//
// Replaces the arithmetic of fmhasim::fmha_forward
// (/root/reference/proj/src/attention.cpp:153-173): for every (b, head) and
// every 128-row Q tile it streams 128-row K/V tiles (the reference's KBLK),
// computes S = Q K^T (GEMM-I, attention.cpp:123), the online softmax update
// (online_softmax_step, attention.cpp:36-66), O += P V (GEMM-II,
// attention.cpp:130) and the final O *= 1/Sigma (rowwise_finalize,
// attention.cpp:68-73), plus LSE = m + ln(Sigma).
//
// Work unit = one (b, head) and TWO 128-row Q tiles (256 query rows) that
// share every K/V tile loaded into shared memory.  The grid is persistent
// (one CTA per SM); CTA c takes units c, c + G, c + 2G, ... so the CTAs
// resident at any time work on neighbouring units of the same heads and K/V
// is served from L2.
//
//   warps 0-3  softmax WG 0: thread t owns row t of Q tile 0 (TMEM lane t)
//   warps 4-7  softmax WG 1: same for Q tile 1
//   warp 8     TMA producer (one lane): Q0 Q1 | K0 V0 K1 V1 ... per unit
//   warp 9     MMA issuer (whole warp, elect.sync issues) + TMEM allocator
//   warp 10    O store warp: TMA-stores each staged O tile, frees the stage
//   warp 11    idle (register donor)
//
// Tensor Memory (512 columns x 128 lanes x 32 bit):
//   S0 [0,128)  S1 [128,256)  O0 [256,256+D)  O1 [256+D,256+2D)
//   P_q (16-bit, packed 2 per column) aliases the first 64 columns of S_q.
//
// Per K/V tile j the MMA warp issues, in order,
//   PV0(j-1) ; S0(j) ; PV1(j-1) ; S1(j)
// so the tensor core runs tile 1's GEMMs while softmax WG 0 works on S0(j)
// and vice versa (two-tile ping-pong).  tcgen05 ops from one thread execute
// in issue order, so when softmax WG q observes "S_q(j) complete" the
// preceding PV_q(j-1) has completed too: the WG may rescale O_q in TMEM
// without any further barrier, and P_q(j) may overwrite S_q(j)'s columns.
// P is published in two halves (kv rows 0-63 / 64-127) so GEMM-II on the
// first half overlaps the end of the softmax; the TMEM store of half 0 is
// waited for (tcgen05.wait::st, ~200 clk) only after half 1's exponentials
// are computed, so the warp never idles on it.
//
// Across units: the producer loads the next unit's Q as soon as the last
// S GEMMs of the current unit have completed (`q_empty`), the MMA warp
// starts the next unit's S(0) while the softmax WGs run their epilogue, and
// only the first PV of a unit waits for the epilogue to have drained O_q
// from TMEM (`o_empty`).  The epilogue stages O in shared memory (the
// swizzled TMA layout) and writes it with one TMA store per 64 columns.
//
// Rescaling is conditional (FlashAttention-4 style): a warp keeps its stale
// row max unless some row's max grew by more than 2^8 in the exp2 domain.
// Exact, because the final (m, Sigma) pair is consistent; P stays <= 256.
#pragma once

#include <cuda.h>
#include <cstdint>

#include "sm100.cuh"
#include "softmax_math.cuh"
#include "tmem_ops.cuh"

namespace fmha_b200 {

struct FwdArgs {
  void* o;                   // BSHD output (informational: every kernel stores O by TMA through tmO)
  int64_t o_sb, o_sn, o_sh;  // output strides (elements)
  float* lse;        // [L][h][N] fp32 or nullptr
  int N, H, L;      // N: key/value length (and the LSE row stride)
  int n_q;           // query rows from the Q/O base (N, or a host-pipeline row slice)
  int n_kv_tiles;    // ceil(N / kBN)
  int n_qblocks;     // Q blocks per head (256 rows for d<=128, 128 for d=256)
  int n_units;       // L * H * n_qblocks
  float scale_log2;  // softmax scale * log2(e)
  float scale;       // softmax scale (natural)
  unsigned long long* trace;  // debug timeline (FMHA_TRACE=1) or nullptr
};

// Debug timeline for the first unit of CTA 0: clock64 stamps written by one
// thread per role.  trace[(q * n_kv + j) * 16 + k]:
//   k=0 softmax woke (S ready)  1 S in registers  8 row max done
//   9 first-half exps done      2 first half published
//   10 second-half exps done    3 second half published
//   4 MMA saw P half 0   11 MMA saw P half 1   12 PV issued   5 S issued
//   [6]/[7] of entry 0: kernel start / setup done; of the last tile:
//   O ready / epilogue done.
// Compiled in only with -DFMHA_TRACE_BUILD (tools/trace_timeline.py builds it).
__device__ __forceinline__ void trace_stamp(const FwdArgs& a, bool on, int q, int j, int k) {
#ifdef FMHA_TRACE_BUILD
  if (on) a.trace[(q * a.n_kv_tiles + j) * 16 + k] = clock64();
#endif
}

// Phase profile (-DFMHA_PROF_BUILD, tools/prof_phases.py): every warp adds
// the clock64 time since its previous mark to accumulator k, and writes the
// totals to trace[(blockIdx.x * 16 + warp) * 8 + k] at exit.  Compiled out
// otherwise.
struct Prof {
#ifdef FMHA_PROF_BUILD
  unsigned long long acc[8];
  long long last;
  static __device__ __forceinline__ long long now() {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    return t;
  }
  __device__ __forceinline__ Prof() : last(now()) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0;
  }
  __device__ __forceinline__ void mark(int k) {
    const long long t = now();
    acc[k] += static_cast<unsigned long long>(t - last);
    last = t;
  }
  __device__ __forceinline__ void flush(const FwdArgs& a, int warp) {
    if ((threadIdx.x & 31) == 0 && a.trace != nullptr)
      for (int k = 0; k < 8; ++k) a.trace[(static_cast<size_t>(blockIdx.x) * 16 + warp) * 8 + k] = acc[k];
  }
#else
  __device__ __forceinline__ void mark(int) {}
  __device__ __forceinline__ void flush(const FwdArgs&, int) {}
#endif
};

#ifndef FMHA_D64_EPI_WG
#define FMHA_D64_EPI_WG 0  // measured slower (profiles/r02_microbench.txt): off
#endif

template <int D>
struct FwdCfg {
  static_assert(D == 64 || D == 128, "this kernel handles head dim 64 and 128");
  static constexpr int kBM = 128;         // Q rows per tile (UMMA M)
  static constexpr int kBN = 128;         // K/V rows per tile
  static constexpr int kChunks = D / 64;  // 128-B swizzle atoms along d
  static constexpr int kQTileBytes = kBM * D * 2;
  static constexpr int kKVTileBytes = kBN * D * 2;
  // Option (FMHA_D64_EPI_WG=1, d = 64): a dedicated epilogue warpgroup drains
  // O (TMEM has room for two O buffers per Q tile, alternating per unit), so
  // the softmax WGs go straight from a unit's last P to the next unit's first
  // S.  Measured 6-8 % slower at N = 256..768: the 512-thread CTA caps the
  // softmax WGs at 176 registers and their exponential phases slow down more
  // than the epilogue overlap saves (profiles/r02_microbench.txt).
  static constexpr bool kEpiWG = D == 64 && FMHA_D64_EPI_WG != 0;
#ifdef FMHA_D64_STAGES
  static constexpr int kStages = D == 64 ? FMHA_D64_STAGES : 4;
#else
  static constexpr int kStages = D == 64 ? (kEpiWG ? 7 : 8) : 4;  // K/V ring depth
#endif
  static constexpr int kQStages = D == 64 ? 2 : 1;  // Q double-buffered when it fits
  static constexpr int kSmemQ = kQStages * 2 * kQTileBytes;
  // O staging for the TMA store: one tile per softmax WG when it fits (d = 64),
  // else one tile the two WGs take in turns (d = 128: 224 KB are in use).
  // (Measured alternative at d = 128, profiles/r02_microbench.txt: staging in
  // the finished unit's Q buffer to buy a fifth K/V slot -- slower.)
  static constexpr int kOBufs = D == 64 ? 2 : 1;
  static constexpr int kSmemO = kOBufs * kQTileBytes;
  static constexpr int kSmemRing = kStages * kKVTileBytes;
  static constexpr int kSmemStats = kEpiWG ? 4 * kBM * 8 : 0;  // (m, Sigma) per row, per (tile, O buffer)
  static constexpr int kPChunks = 2;  // P published in two halves of 64 kv rows
  static constexpr int kOBar = kEpiWG ? 4 : 2;  // o_full / o_empty: per tile (x O buffer)
  static constexpr int kNumBars = 2 * kQStages + 2 * kStages + 2 + 2 * kPChunks + 2 * kOBar + 4 + (kEpiWG ? 4 : 0);
  static constexpr int kSmemBytes = kSmemQ + kSmemO + kSmemRing + kSmemStats + kNumBars * 8 + 16;
  static constexpr int kSmemAlloc = kSmemBytes + 1024;  // slack for 1024-B alignment
  // 3 warpgroups: softmax 0, softmax 1, load/MMA/store (+ the epilogue WG at d = 64)
  static constexpr int kThreads = kEpiWG ? 512 : 384;
  static constexpr int kEpiWarp0 = 8;
  static constexpr int kLoadWarp = kEpiWG ? 12 : 8;
  static constexpr int kMmaWarp = kEpiWG ? 13 : 9;
  static constexpr int kStoreWarp = kEpiWG ? 14 : 10;
  static constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO0 = 256, kColO1 = 256 + D;
  // O of tile q in buffer ob (ob = unit & 1 with the epilogue WG, else 0)
  __host__ __device__ static constexpr uint32_t col_o(int q, int ob) {
    return 256u + static_cast<uint32_t>(q * D + ob * 2 * D);
  }
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kSeqBar = 1;  // named barriers 1, 2: exponential-phase turns of WG 0, 1
  static_assert(kSmemAlloc <= 227 * 1024, "shared memory budget");
};

#ifndef FMHA_SEQ
#define FMHA_SEQ 0
#endif
constexpr bool kSeq = FMHA_SEQ != 0;
#ifndef FMHA_SPEC
#define FMHA_SPEC 0
#endif
constexpr bool kSpec = FMHA_SPEC != 0;  // speculative first half (see the softmax loop)
// FMHA_PP_MASKED_MUFU=0: the padded last K/V tile takes the same exp2 code as
// every other tile (polynomial lanes give 2^-125 instead of 0 for masked
// scores; padded V rows are TMA zero-fill, so O is unchanged) -- one copy of
// the unrolled exponential loop instead of two, a smaller hot loop body.
#ifndef FMHA_PP_MASKED_MUFU
#define FMHA_PP_MASKED_MUFU 1
#endif
constexpr bool kMaskedMufu = FMHA_PP_MASKED_MUFU != 0;
#ifndef FMHA_PP_SOFTMAX_SLEEP_NS
#define FMHA_PP_SOFTMAX_SLEEP_NS 0  // softmax wait for S: nanosleep between polls (0: try_wait loop)
#endif
constexpr uint32_t kSoftmaxWaitNs = FMHA_PP_SOFTMAX_SLEEP_NS;
#ifndef FMHA_PP_STORE_SLEEP_NS
#define FMHA_PP_STORE_SLEEP_NS 0  // O store warp: nanosleep between polls (measured -0.5 % at 256 ns)
#endif
constexpr uint32_t kStoreWaitNs = FMHA_PP_STORE_SLEEP_NS;
#ifndef FMHA_EPI_SLEEP_NS
#define FMHA_EPI_SLEEP_NS 64  // d = 64 epilogue WG: nanosleep between polls (off the critical path)
#endif
constexpr uint32_t kEpiSleepNs = FMHA_EPI_SLEEP_NS;
// Register split of the 384-thread kernel.  The CTA launches with 168 per
// thread (64512 in all); setmaxnreg.inc blocks until the dealloc'd registers
// cover it, so 2 * softmax + role <= 3 * 168 = 504 (else: a hang).
#ifndef FMHA_PP_SOFTMAX_REGS
#define FMHA_PP_SOFTMAX_REGS 192
#endif
#ifndef FMHA_PP_ROLE_REGS
#define FMHA_PP_ROLE_REGS 112
#endif
constexpr uint32_t kSoftmaxRegs = FMHA_PP_SOFTMAX_REGS, kRoleRegs = FMHA_PP_ROLE_REGS;
static_assert(2 * FMHA_PP_SOFTMAX_REGS + FMHA_PP_ROLE_REGS <= 504, "setmaxnreg budget of the 384-thread CTA");
#ifndef FMHA_PP_K4
#define FMHA_PP_K4 2  // MMA issue in batches of four K-steps per elect.sync: 0 off, 1 on, 2 d = 64 only
#endif
#ifndef FMHA_PP_LATE_SUM
#define FMHA_PP_LATE_SUM 0  // row sum of P taken after P is published (off the S -> P chain)
#endif
constexpr bool kLateSum = FMHA_PP_LATE_SUM != 0;
#ifndef FMHA_PP_SPLIT_S
#define FMHA_PP_SPLIT_S 0  // S_q(j+1)'s upper 64 columns issued between PV_q(j)'s two P halves
#endif
constexpr bool kSplitS = FMHA_PP_SPLIT_S != 0;
#ifndef FMHA_UNIT_PREFETCH_MAX_KV
#define FMHA_UNIT_PREFETCH_MAX_KV 0  // next-unit L2 prefetch for units of <= this many K/V steps (measured slower: off)
#endif
constexpr int kUnitPrefetchMaxKv = FMHA_UNIT_PREFETCH_MAX_KV;
#ifndef FMHA_KV_PREFETCH
#define FMHA_KV_PREFETCH 0  // K/V tiles prefetched into L2 this many steps ahead (0: off)
#endif

// Epilogue helper (rowwise_finalize, attention.cpp:68-73): this thread's row
// of a 128-row O tile, TMEM columns [tO, tO + D) -> x inv -> 16-bit -> the
// 128-B-swizzled TMA layout at `stage` (D/64 atoms of 128 rows x 128 B).
template <int D, bool kBF16>
__device__ __forceinline__ void stage_o_tile(uint32_t tO, uint8_t* stage, int r, float inv) {
#pragma unroll
  for (int c = 0; c < D / 32; ++c) {
    uint32_t o[32];
    tmem_ld32x32b_x32(tO + c * 32, o);
    uint32_t h2[16];
#pragma unroll
    for (int t = 0; t < 16; ++t)
      h2[t] = pack2<kBF16>(__uint_as_float(o[2 * t]) * inv, __uint_as_float(o[2 * t + 1]) * inv);
    uint8_t* rowp = stage + (c >> 1) * (128 * 128) + r * 128;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int unit = ((c & 1) * 4 + v) ^ (r & 7);  // 128-B swizzle
      st_shared_v4(rowp + unit * 16, h2[4 * v], h2[4 * v + 1], h2[4 * v + 2], h2[4 * v + 3]);
    }
  }
}

// unit -> (b, head, q-block)
template <bool B>
struct BoolTag {
  static constexpr bool value = B;
};

__device__ __forceinline__ void decode_unit(int u, int n_qb, int H, int& b, int& head, int& qb) {
  qb = u % n_qb;
  const int t = u / n_qb;
  head = t % H;
  b = t / H;
}

// kEmuPer16: of every 16 score pairs, how many take the FMA-pipe exp2.
template <int D, bool kBF16, int kEmuPer16 = 0>
__global__ void __launch_bounds__(FwdCfg<D>::kThreads, 1)
    fmha_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV,
                          const __grid_constant__ CUtensorMap tmO, const FwdArgs args) {
  using C = FwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for the 128-B swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sO = smem + C::kSmemQ;
  uint8_t* sRing = sO + C::kSmemO;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRing + C::kSmemRing + C::kSmemStats);
  uint64_t* q_full = bars;               // [kQStages]
  uint64_t* q_empty = bars + C::kQStages;  // [kQStages]
  uint64_t* kv_full = bars + 2 * C::kQStages;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;  // [2]
  uint64_t* p_full = s_full + 2;             // [2][kPChunks]: (tile q, chunk of kv rows)
  uint64_t* o_full = p_full + 2 * C::kPChunks;  // [kOBar]: tile q (x O buffer ob: index 2q + ob)
  uint64_t* o_empty = o_full + C::kOBar;     // [kOBar]
  uint64_t* stage_free = o_empty + C::kOBar;  // [2]: WG q's use of the O staging tile read by its TMA store
  uint64_t* stage_ready = stage_free + 2;    // [2] O staged (kOBufs == 2: per WG; else [0] in turns)
  uint64_t* stat_full = stage_ready + 2;     // [4] (epilogue WG) unit's (m, Sigma) of tile q, buffer ob
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(stat_full + (C::kEpiWG ? 4 : 0));
  float2* stats = reinterpret_cast<float2*>(sRing + C::kSmemRing);  // [4][128] (epilogue WG)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_kv = args.n_kv_tiles;
  const int n_full = (args.N % C::kBN) ? n_kv - 1 : n_kv;  // K/V steps without padding columns
#ifdef FMHA_TRACE_BUILD
  const bool tr = args.trace != nullptr && blockIdx.x == 0;
#else
  constexpr bool tr = false;
#endif

#ifdef FMHA_TRACE_BUILD
  const unsigned long long t_start = clock64();
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
    for (int q = 0; q < 2; ++q) {
      mbar_init(&s_full[q], 1);
      for (int c = 0; c < C::kPChunks; ++c) mbar_init(&p_full[q * C::kPChunks + c], 128);  // every softmax thread
    }
    for (int t = 0; t < C::kOBar; ++t) {
      mbar_init(&o_full[t], 1);
      mbar_init(&o_empty[t], 128);
    }
    if constexpr (C::kEpiWG)
      for (int t = 0; t < 4; ++t) mbar_init(&stat_full[t], 128);
    mbar_init(&stage_free[0], 1);
    mbar_init(&stage_free[1], 1);
    mbar_init(&stage_ready[0], 128);
    mbar_init(&stage_ready[1], 128);
    fence_mbar_init();
  }
  if (warp == C::kMmaWarp) tmem_alloc(tmem_holder, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // o_full / o_empty index of tile q, O buffer ob
  auto oslot = [](int q, int ob) { return C::kEpiWG ? 2 * q + ob : q; };
#ifdef FMHA_TRACE_BUILD
  if (threadIdx.x == 0 && tr) {
    args.trace[6] = t_start;
    args.trace[7] = clock64();
  }
#endif

  // Register split (setmaxnreg inside each role's branch so ptxas sees one
  // limit per region): the load/MMA warpgroup needs few registers, the
  // softmax warpgroups hold a 128-column S row plus packed P per thread.
  if (C::kEpiWG && warp >= C::kEpiWarp0 && warp < C::kEpiWarp0 + 4) {
    reg_dealloc<72>();
    // ------------------------------------------- epilogue WG (d = 64) --
    // rowwise_finalize (attention.cpp:68-73) + LSE for both Q tiles of every
    // unit: O_q (TMEM buffer i & 1) x 1/Sigma -> 16-bit -> staging tile q ->
    // TMA store by the store warp; one row per thread (lane quarter warp & 3).
    const int r = (warp - C::kEpiWarp0) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    int i = 0;
    // the CTA's last unit is drained by the softmax WGs themselves (they are
    // idle by then; two WGs in parallel keep the kernel's tail short)
    const int last_u = args.n_units - 1 - (args.n_units - 1 - static_cast<int>(blockIdx.x)) % static_cast<int>(gridDim.x);
    for (int u = blockIdx.x; u < last_u; u += gridDim.x, ++i) {
      int b, head, qb;
      decode_unit(u, args.n_qblocks, args.H, b, head, qb);
      const int ob = i & 1;
      const uint32_t par = static_cast<uint32_t>(i >> 1) & 1;
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {
        const int slot = 2 * q + ob;
        mbar_wait_backoff(&o_full[slot], par, kEpiSleepNs);
        mbar_wait_backoff(&stat_full[slot], par, kEpiSleepNs);
        tc_fence_after();
        const float2 st = stats[slot * C::kBM + r];
        if (i > 0) mbar_wait_backoff(&stage_free[q], static_cast<uint32_t>(i - 1) & 1, kEpiSleepNs);
        stage_o_tile<D, kBF16>(tmem + lane_off + C::col_o(q, ob), sO + q * C::kQTileBytes, r, 1.0f / st.y);
        tc_fence_before();
        fence_proxy_async_smem();  // staged O visible to the TMA (async proxy)
        mbar_arrive(&o_empty[slot]);  // O buffer and statistics consumed
        mbar_arrive(&stage_ready[q]);
        const int row = qb * 2 * C::kBM + q * C::kBM + r;
        if (row < args.n_q && args.lse != nullptr)
          args.lse[(static_cast<int64_t>(b) * args.H + head) * args.N + row] = st.x * args.scale + logf(st.y);
      }
    }
  } else if (warp >= 8) {
    reg_dealloc<C::kEpiWG ? 88 : kRoleRegs>();
    if (warp == C::kLoadWarp) {
      // -------------------------------------------------- TMA producer --
      if (lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        tma_prefetch_desc(&tmO);
        const uint64_t keep = l2_policy_evict_last();   // K/V re-read by sibling CTAs
        const uint64_t once = l2_policy_evict_first();  // Q read once
        int slot = 0;
        uint32_t phase = 0;
        int i = 0;
        Prof prof;
        for (int u = blockIdx.x; u < args.n_units; u += gridDim.x, ++i) {
          int b, head, qb;
          decode_unit(u, args.n_qblocks, args.H, b, head, qb);
          const int qrow0 = qb * 2 * C::kBM;
          // Short units (few K/V steps): pull the CTA's NEXT unit's Q and K/V
          // into L2 now, so only each CTA's first unit waits on HBM latency
          // (with a cold L2 the loads at every unit start are latency-bound).
          if (n_kv <= kUnitPrefetchMaxKv && u + static_cast<int>(gridDim.x) < args.n_units) {
            int b2, head2, qb2;
            decode_unit(u + gridDim.x, args.n_qblocks, args.H, b2, head2, qb2);
#pragma unroll
            for (int c = 0; c < C::kChunks; ++c) {
              tma_prefetch_4d(&tmQ, c * 64, head2, qb2 * 2 * C::kBM, b2);
              tma_prefetch_4d(&tmQ, c * 64, head2, qb2 * 2 * C::kBM + C::kBM, b2);
            }
            for (int j = 0; j < n_kv; ++j)
#pragma unroll
              for (int c = 0; c < C::kChunks; ++c) {
                tma_prefetch_4d(&tmK, c * 64, head2, j * C::kBN, b2);
                tma_prefetch_4d(&tmV, c * 64, head2, j * C::kBN, b2);
              }
          }
          // Q stage is free once the last S GEMMs of the unit that used it
          // before have completed
          const int qs = i % C::kQStages;
          const uint32_t qph = static_cast<uint32_t>(i / C::kQStages) & 1;
          mbar_wait(&q_empty[qs], qph ^ 1);
          mbar_arrive_expect_tx(&q_full[qs], 2 * C::kQTileBytes);
          uint8_t* sQs = sQ + qs * 2 * C::kQTileBytes;
#pragma unroll
          for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int c = 0; c < C::kChunks; ++c)
              tma_load_4d_hint(&tmQ, &q_full[qs], sQs + q * C::kQTileBytes + c * C::kBM * 128,
                               c * 64, head, qrow0 + q * C::kBM, b, once);
          for (int j = 0; j < n_kv; ++j) {
#if FMHA_KV_PREFETCH > 0
            // L2 prefetch of the K/V tiles FMHA_KV_PREFETCH steps ahead
            if (j + FMHA_KV_PREFETCH < n_kv)
#pragma unroll
              for (int c = 0; c < C::kChunks; ++c) {
                tma_prefetch_4d(&tmK, c * 64, head, (j + FMHA_KV_PREFETCH) * C::kBN, b);
                tma_prefetch_4d(&tmV, c * 64, head, (j + FMHA_KV_PREFETCH) * C::kBN, b);
              }
#endif
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              prof.mark(3);
              mbar_wait(&kv_empty[slot], phase ^ 1);
              prof.mark(0);
              mbar_arrive_expect_tx(&kv_full[slot], C::kKVTileBytes);
              uint8_t* dst = sRing + slot * C::kKVTileBytes;
#pragma unroll
              for (int c = 0; c < C::kChunks; ++c)
                tma_load_4d_hint(t == 0 ? &tmK : &tmV, &kv_full[slot], dst + c * C::kBN * 128,
                                 c * 64, head, j * C::kBN, b, keep);
              if (++slot == C::kStages) {
                slot = 0;
                phase ^= 1;
              }
            }
          }
        }
        prof.mark(3);
        prof.flush(args, warp);
      }
    } else if (warp == C::kMmaWarp) {
      // ---------------------------------------------------- MMA issuer --
      // whole warp: uniform control flow, one elected lane issues
      constexpr uint32_t kIdescQK = idesc_f16(kBF16, C::kBM, C::kBN, false, false);
      constexpr uint32_t kIdescPV = idesc_f16(kBF16, C::kBM, D, false, true);
      uint32_t sQ_addr = smem_u32(sQ);
      const uint32_t ring_addr = smem_u32(sRing);
      int slot = 0;
      uint32_t phase = 0;
      Prof prof;
      int jj = 0;  // K/V tile index within the unit (profile only)
      auto next_slot = [&]() -> int {
        const int s = slot;
        prof.mark(3);
        mbar_wait(&kv_full[s], phase);
        prof.mark(jj < 2 ? 5 : 0);
        if (++slot == C::kStages) {
          slot = 0;
          phase ^= 1;
        }
        return s;
      };
      // S_q = Q_q K^T : M=128, N=128, K=D in D/16 steps of 32 B inside the
      // 128-B swizzle atom; the next 64 columns of d live in the next atom
      // column (chunk stride = rows * 128 B).
      // batched issue (measured: +2.5 % on c2 at d = 64, neutral at d = 128)
      constexpr bool kK4Issue = FMHA_PP_K4 == 1 || (FMHA_PP_K4 == 2 && D == 64);
      auto mma_qk = [&](int q, int kslot) {
        const uint32_t a0 = sQ_addr + q * C::kQTileBytes;
        const uint32_t b0 = ring_addr + kslot * C::kKVTileBytes;
        if constexpr (kK4Issue) {  // four K=16 steps per elect.sync (one per 64-column atom of d)
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c)
            mma_ss_k4(tmem + (q ? C::kColS1 : C::kColS0), sdesc_sw128(a0 + c * (C::kBM * 128), 16, 1024),
                      sdesc_sw128(b0 + c * (C::kBN * 128), 16, 1024), kIdescQK, c > 0 ? 1u : 0u);
          return;
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off_a = (kk >> 2) * (C::kBM * 128) + (kk & 3) * 32;
          const uint32_t off_b = (kk >> 2) * (C::kBN * 128) + (kk & 3) * 32;
          mma_ss_elect(tmem + (q ? C::kColS1 : C::kColS0), sdesc_sw128(a0 + off_a, 16, 1024),
                       sdesc_sw128(b0 + off_b, 16, 1024), kIdescQK, kk > 0 ? 1u : 0u);
        }
      };
      // Half of S_q = Q_q K^T: N = 64 kv rows [64h, 64h + 64) into S columns
      // [64h, 64h + 64) (FMHA_PP_SPLIT_S: the upper half of S_q(j+1) is issued
      // between the two P halves of PV_q(j) -- those columns no longer hold
      // anything the softmax or GEMM-II still needs once P half 0 is published --
      // so only the lower half (which P_q(j) occupies) waits for PV_q(j)).
      constexpr uint32_t kIdescQK64 = idesc_f16(kBF16, C::kBM, 64, false, false);
      auto mma_qk_half = [&](int q, int kslot, int h) {
        const uint32_t a0 = sQ_addr + q * C::kQTileBytes;
        const uint32_t b0 = ring_addr + kslot * C::kKVTileBytes + h * 64 * 128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off_a = (kk >> 2) * (C::kBM * 128) + (kk & 3) * 32;
          const uint32_t off_b = (kk >> 2) * (C::kBN * 128) + (kk & 3) * 32;
          mma_ss_elect(tmem + (q ? C::kColS1 : C::kColS0) + 64 * h, sdesc_sw128(a0 + off_a, 16, 1024),
                       sdesc_sw128(b0 + off_b, 16, 1024), kIdescQK64, kk > 0 ? 1u : 0u);
        }
      };
      // O_q (+)= P_q V : M=128, N=D, K=128 kv rows in 8 steps of 16 rows.
      // A = P from TMEM (8 columns per step); B = V, MN-major (d contiguous):
      // LBO = chunk stride along d, SBO = 1024 B per 8 kv rows.  P arrives
      // in kPChunks chunks; each chunk's MMAs start as soon as it is stored.
      int ob_cur = 0;  // O buffer of the current unit
      auto mma_pv = [&](int q, int vslot, bool accumulate, uint32_t par, bool trp, int jt, int ks_hi = -1) {
        const uint32_t b0 = ring_addr + vslot * C::kKVTileBytes;
        const uint32_t p0 = tmem + (q ? C::kColS1 : C::kColS0);
        constexpr int kStepsPerChunk = 8 / C::kPChunks;
#pragma unroll
        for (int c = 0; c < C::kPChunks; ++c) {
          prof.mark(3);
#ifdef FMHA_SPIN_P
          mbar_wait_spin(&p_full[q * C::kPChunks + c], par);
#else
          mbar_wait(&p_full[q * C::kPChunks + c], par);
#endif
          prof.mark(1);
          if (c == C::kPChunks - 1) trace_stamp(args, trp, q, jt, 11);
          tc_fence_after();
          if constexpr (kK4Issue && kStepsPerChunk == 4) {
            mma_ts_k4(tmem + C::col_o(q, ob_cur), p0 + c * 32,
                      sdesc_sw128(b0 + c * 4 * 16 * 128, C::kBN * 128, 1024), kIdescPV,
                      (accumulate || c > 0) ? 1u : 0u);
          } else {
#pragma unroll
            for (int kk = c * kStepsPerChunk; kk < (c + 1) * kStepsPerChunk; ++kk)
              mma_ts_elect(tmem + C::col_o(q, ob_cur), p0 + kk * 8,
                           sdesc_sw128(b0 + kk * 16 * 128, C::kBN * 128, 1024), kIdescPV,
                           (accumulate || kk > 0) ? 1u : 0u);
          }
          if (c == 0 && ks_hi >= 0) mma_qk_half(q, ks_hi, 1);
        }
      };

      uint32_t it = 0;  // global K/V-tile counter (p_full parity)
      int i = 0;
      for (int u = blockIdx.x; u < args.n_units; u += gridDim.x, ++i) {
        const bool trm = tr && i == 0;
        // O buffer of this unit and the o_empty phase to wait for: the previous
        // unit's epilogue (one buffer), or unit i-2's (epilogue WG, two buffers)
        const int ob = C::kEpiWG ? (i & 1) : 0;
        const uint32_t ue = C::kEpiWG ? ((static_cast<uint32_t>(i >> 1) & 1) ^ 1) : ((static_cast<uint32_t>(i) & 1) ^ 1);
        ob_cur = ob;
        const int qs = i % C::kQStages;
        prof.mark(3);
        mbar_wait(&q_full[qs], static_cast<uint32_t>(i / C::kQStages) & 1);
        prof.mark(4);
#ifdef FMHA_TRACE_BUILD
        // per-unit timeline of CTA 0 (units 0..7): trace[(3*n_kv)*16 + i*8 + k]
        if (tr && i < 8) args.trace[(3 * n_kv) * 16 + i * 8 + 0] = clock64();
#endif
        sQ_addr = smem_u32(sQ) + qs * 2 * C::kQTileBytes;
        jj = 0;
        int ks = next_slot();
        tc_fence_after();
        mma_qk(0, ks);
        mma_commit_elect(&s_full[0]);
        mma_qk(1, ks);
        mma_commit_elect(&s_full[1]);
        if (n_kv == 1) mma_commit_elect(&q_empty[qs]);
        mma_commit_elect(&kv_empty[ks]);
        for (int j = 1; j < n_kv; ++j) {
          jj = j;
          const int vs = next_slot();
          ks = next_slot();
          const uint32_t par = it & 1;
          if (j == 1) {  // previous unit's epilogue drained O0
            prof.mark(3);
            mbar_wait(&o_empty[oslot(0, ob)], ue);
            prof.mark(2);
          }
          if constexpr (kSplitS) {
            mma_pv(0, vs, j > 1, par, trm, j - 1, ks);
            mma_qk_half(0, ks, 0);
          } else {
            mma_pv(0, vs, j > 1, par, trm, j - 1);
            trace_stamp(args, trm, 0, j - 1, 12);
            mma_qk(0, ks);
          }
          mma_commit_elect(&s_full[0]);
          trace_stamp(args, trm, 0, j - 1, 5);
          if (j == 1) {
            prof.mark(3);
            mbar_wait(&o_empty[oslot(1, ob)], ue);
            prof.mark(2);
          }
          if constexpr (kSplitS) {
            mma_pv(1, vs, j > 1, par, trm, j - 1, ks);
            mma_qk_half(1, ks, 0);
          } else {
            mma_pv(1, vs, j > 1, par, trm, j - 1);
            trace_stamp(args, trm, 1, j - 1, 12);
            mma_qk(1, ks);
          }
          mma_commit_elect(&s_full[1]);
          trace_stamp(args, trm, 1, j - 1, 5);
          if (j == n_kv - 1) mma_commit_elect(&q_empty[qs]);  // last reads of Q issued
          mma_commit_elect(&kv_empty[vs]);
          mma_commit_elect(&kv_empty[ks]);
          ++it;
        }
        const int vs = next_slot();
        const uint32_t par = it & 1;
        if (n_kv == 1) mbar_wait(&o_empty[oslot(0, ob)], ue);
        mma_pv(0, vs, n_kv > 1, par, false, 0);
        mma_commit_elect(&o_full[oslot(0, ob)]);
        if (n_kv == 1) mbar_wait(&o_empty[oslot(1, ob)], ue);
        mma_pv(1, vs, n_kv > 1, par, false, 0);
        mma_commit_elect(&o_full[oslot(1, ob)]);
        mma_commit_elect(&kv_empty[vs]);
        ++it;
      }
      prof.mark(3);
      prof.flush(args, warp);
    } else if (warp == C::kStoreWarp) {
      // ------------------------------------------------- O store warp --
      // Uses of the staging tile alternate WG0, WG1 per unit: use k = 2i+q.
      if (lane == 0) {
        uint32_t k = 0;
        int i = 0;
        for (int u = blockIdx.x; u < args.n_units; u += gridDim.x, ++i) {
          int b, head, qb;
          decode_unit(u, args.n_qblocks, args.H, b, head, qb);
          for (int q = 0; q < 2; ++q, ++k) {
            const bool own = C::kOBufs == 2;  // per-WG tiles: use i of WG q; shared: use k = 2i + q
            // optional sleep between polls (measured: the spin does not cost the
            // softmax warps of this sub-partition anything, profiles/r02_microbench.txt)
            if constexpr (kStoreWaitNs > 0)
              mbar_wait_backoff(&stage_ready[own ? q : 0], own ? (static_cast<uint32_t>(i) & 1) : (k & 1),
                                kStoreWaitNs);
            else
              mbar_wait(&stage_ready[own ? q : 0], own ? (static_cast<uint32_t>(i) & 1) : (k & 1));
            const uint8_t* src = sO + (own ? q : 0) * C::kQTileBytes;
#pragma unroll
            for (int c = 0; c < C::kChunks; ++c)
              tma_store_4d(&tmO, src + c * C::kBM * 128, c * 64, head, qb * 2 * C::kBM + q * C::kBM, b);
            tma_store_commit();
            tma_store_wait_read();
            mbar_arrive(&stage_free[q]);
          }
        }
        tma_store_wait_all();
      }
    }
  } else {
    reg_alloc<C::kEpiWG ? 176 : kSoftmaxRegs>();
    // ------------------------------------------------- softmax WG 0 / 1 --
    const int q = warp >> 2;
    const int r = threadIdx.x & 127;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_off + (q ? C::kColS1 : C::kColS0);
    uint32_t tO = tmem + lane_off + C::col_o(q, 0);  // this unit's O_q (buffer i & 1 with the epilogue WG)
    const float sl2 = args.scale_log2;
    const int N = args.N;
    // shared-window barrier addresses, computed once (hot loop)
    const uint32_t a_s_full = smem_u32(&s_full[q]);
    const uint32_t a_p_full0 = smem_u32(&p_full[q * 2]), a_p_full1 = smem_u32(&p_full[q * 2 + 1]);
    // WG 0 takes the first turn of the exponential phases
    if constexpr (kSeq)
      if (q == 1) named_bar_arrive(C::kSeqBar, 256);
    uint32_t it = 0;
    int i = 0;
    Prof prof;
    for (int u = blockIdx.x; u < args.n_units; u += gridDim.x, ++i) {
      int b, head, qb;
      decode_unit(u, args.n_qblocks, args.H, b, head, qb);
      const bool trq = tr && i == 0 && r == 0;
      if constexpr (C::kEpiWG) tO = tmem + lane_off + C::col_o(q, i & 1);
      float m = -INFINITY;  // running max in raw score units
      float l = 0.0f;       // running sum of exp2((s - m) * sl2)

      // One K/V step of the softmax.  The padded last tile (N % 128 != 0) runs
      // its own instantiation after the loop, so the hot loop body carries no
      // masking code (a smaller unrolled body: fewer instruction-fetch stalls).
      auto kv_step = [&](const int j, auto padded_tag) {
        constexpr bool kPadded = decltype(padded_tag)::value;
        prof.mark(7);
#ifdef FMHA_SPIN_S
        while (!mbar_test_wait(a_s_full, it & 1)) {
        }
#else
        if constexpr (kSoftmaxWaitNs > 0)
          mbar_wait_backoff_addr(a_s_full, it & 1, kSoftmaxWaitNs);  // sleep: leave issue slots to the other WG
        else
          mbar_wait_addr(a_s_full, it & 1);
#endif
        prof.mark(0);
        trace_stamp(args, trq, q, j, 0);
#ifdef FMHA_TRACE_BUILD
        if (tr && i < 8 && r == 0 && j == 0) args.trace[(3 * n_kv) * 16 + i * 8 + 1 + q] = clock64();
#endif
        tc_fence_after();
#ifdef FMHA_PROBE_ONE_WG
        // probe build only (tools/prof_phases.py): WG 1 publishes P (garbage) at
        // once, so WG 0's phase profile shows its softmax without a second
        // softmax on its SM sub-partitions
        if (q == 1) {
          tc_fence_before();
          mbar_arrive_addr(a_p_full0);
          mbar_arrive_addr(a_p_full1);
          prof.mark(5);
          return;
        }
#endif
        uint32_t sr[128];
        if constexpr (C::kThreads > 384)
          tmem_ld32x32b_x64x2(tS, sr);  // base register budget 128: no 129-operand instruction
        else
          tmem_ld32x32b_x128(tS, sr);
        trace_stamp(args, trq, q, j, 1);
        float s[128];
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] = __uint_as_float(sr[c]);
        if constexpr (kPadded) {
          const int valid = N - j * C::kBN;  // columns >= valid are padding
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c >= valid) s[c] = -INFINITY;
        }
        prof.mark(1);
        // Rescale O_q (TMEM) and the running sum by 2^((m - m_new) c); only
        // called while O_q is quiescent (S_q(j) observed => PV_q(j-1) done).
        auto rescale = [&](float m_new) {
          const float alpha = ex2_approx((m - m_new) * sl2);
          l *= alpha;
#pragma unroll
          for (int c = 0; c < D / 16; ++c) {  // x16 chunks: S stays in registers meanwhile
            uint32_t o[16];
            tmem_ld32x32b_x16(tO + c * 16, o);
#pragma unroll
            for (int t = 0; t < 16; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * alpha);
            tmem_st32x32b_x16(tO + c * 16, o);
          }
          m = m_new;
        };
        // full row max, 8 independent chains (short dependency depth)
        auto row_max = [&]() {
          float mx[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) mx[t] = fmaxf(s[t], s[t + 8]);
#pragma unroll
          for (int c = 16; c < 128; c += 16)
#pragma unroll
            for (int t = 0; t < 8; ++t) mx[t] = fmaxf(mx[t], fmaxf(s[c + t], s[c + t + 8]));
          return fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                       fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        };
        // P half h = scores [64h, 64h+64) -> packed TMEM columns [32h, 32h+32)
        // of S_q (S is already in registers).  Padded tiles take an all-MUFU
        // copy (exact zeros for -inf scores).  The TMEM store of half 0 is
        // waited for only after half 1's exponentials: the ~200-clk store
        // latency leaves the critical path; GEMM-II on half 0 then overlaps
        // the store and publication of half 1.
        //
        // Conditional rescale (exact, since the final (m, Sigma) pair is
        // consistent): a warp keeps its stale max unless some row's max grew
        // by more than 8 in log2 units (P stays <= 256).  After the first
        // tile, half 0 is exponentiated speculatively against the stale max
        // while the new row max is reduced in the same instruction stream;
        // only when a row's max grew by more than 8 is the half redone.
        constexpr bool masked = kPadded;
        uint32_t p0[32], p1[32];
        // The exponential phases of the two WGs run in strict turns (named
        // barriers kSeqBar + q): each gets the sub-partitions' MUFU / FMA
        // pipes alone instead of both slowing down when their phases overlap.
        if constexpr (kSeq) named_bar_sync(C::kSeqBar + q, 256);
        float neg, rs;
        bool redo = true;
        if (kSpec && j > 0 && !masked) {
          float mx;
          neg = -m * sl2;
          rs = exp_rowsum_pack_max<kBF16, kEmuPer16>(s, sl2, neg, p0, mx);
          trace_stamp(args, trq, q, j, 8);
          redo = __any_sync(0xffffffffu, (mx - m) * sl2 > 8.0f);
          if (redo) rescale(fmaxf(mx, m));
        } else {
          const float mx = row_max();
          trace_stamp(args, trq, q, j, 8);
          if (__any_sync(0xffffffffu, (mx - m) * sl2 > 8.0f)) {
            const float m_new = fmaxf(mx, m);
            if (j == 0)
              m = m_new;  // l = 0 and the first PV overwrites O
            else
              rescale(m_new);
          }
        }
        prof.mark(2);
        if (kLateSum && !kSpec) {
          neg = -m * sl2;
          if (masked)
            exp_pack_inplace<kBF16, 0, 64, 0>(s, sl2, neg, p0);
          else
            exp_pack_inplace<kBF16, 0, 64, kEmuPer16>(s, sl2, neg, p0);
          trace_stamp(args, trq, q, j, 9);
          prof.mark(3);
          tmem_st32x32b_x32(tS, p0);
          if (masked)
            exp_pack_inplace<kBF16, 64, 64, 0>(s, sl2, neg, p1);
          else
            exp_pack_inplace<kBF16, 64, 64, kEmuPer16>(s, sl2, neg, p1);
          rs = 0.0f;  // the row sum follows the publication below
        } else {
        if (redo) {
          neg = -m * sl2;
          if constexpr (kMaskedMufu)
            rs = masked ? exp_rowsum_pack<kBF16, 0, 64, 0>(s, sl2, neg, p0)
                        : exp_rowsum_pack<kBF16, 0, 64, kEmuPer16>(s, sl2, neg, p0);
          else
            rs = exp_rowsum_pack<kBF16, 0, 64, kEmuPer16>(s, sl2, neg, p0);
        }
        trace_stamp(args, trq, q, j, 9);
        prof.mark(3);
        tmem_st32x32b_x32(tS, p0);
        if constexpr (kMaskedMufu)
          rs += masked ? exp_rowsum_pack<kBF16, 64, 64, 0>(s, sl2, neg, p1)
                       : exp_rowsum_pack<kBF16, 64, 64, kEmuPer16>(s, sl2, neg, p1);
        else
          rs += exp_rowsum_pack<kBF16, 64, 64, kEmuPer16>(s, sl2, neg, p1);
        }
        if constexpr (kSeq) named_bar_arrive(C::kSeqBar + (q ^ 1), 256);
        prof.mark(4);
        trace_stamp(args, trq, q, j, 10);
        // every thread arrives once its own TMEM stores have completed (no
        // lane-0 branch, no warp reconvergence on the critical path)
        auto publish = [&](int half) {
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive_addr(half ? a_p_full1 : a_p_full0);
        };
        publish(0);
        trace_stamp(args, trq, q, j, 2);
        tmem_st32x32b_x32(tS + 32, p1);
        publish(1);
        if constexpr (kLateSum && !kSpec) rs = row_sum_f32(s);  // off the S -> P path
        l += rs;
        prof.mark(5);
        trace_stamp(args, trq, q, j, 3);
#ifdef FMHA_TRACE_BUILD
        // per-warp completion times of the first unit: trace[(2*n_kv + j)*16 + warp]
        if (tr && i == 0 && lane == 0) args.trace[(2 * n_kv + j) * 16 + warp] = clock64();
#endif
      };
      for (int j = 0; j < n_full; ++j, ++it) kv_step(j, BoolTag<false>{});
      if (n_full < n_kv) {
        kv_step(n_kv - 1, BoolTag<true>{});
        ++it;
      }

      if (C::kEpiWG && u + static_cast<int>(gridDim.x) < args.n_units) {
        // hand (m, Sigma) to the epilogue WG; the slot (tile q, buffer i & 1)
        // was last read by unit i-2's epilogue (o_empty, as the MMA warp waits)
        const int slot = 2 * q + (i & 1);
        mbar_wait(&o_empty[slot], (static_cast<uint32_t>(i >> 1) & 1) ^ 1);
        stats[slot * C::kBM + r] = make_float2(m, l);
        mbar_arrive(&stat_full[slot]);
        prof.mark(6);
        continue;
      }
      // ----------------------------------------------------- epilogue --
      // O_q -> registers -> x(1/Sigma) (rowwise_finalize) -> 16-bit -> the
      // swizzled staging tile -> TMA store; TMEM is released as soon as it
      // has been read so the next unit's first PV can start.
      if constexpr (C::kEpiWG)
        mbar_wait(&o_full[2 * q + (i & 1)], static_cast<uint32_t>(i >> 1) & 1);
      else
        mbar_wait(&o_full[q], i & 1);
      tc_fence_after();
      trace_stamp(args, trq, q, n_kv - 1, 6);
      // The two WGs take the staging tile in strict turns (WG0 unit i, WG1
      // unit i, WG0 unit i+1, ...): before writing, wait until the OTHER
      // WG's latest use has been read by its TMA store.  That use itself
      // waited for this WG's previous use, so stage_free[q^1] is at most one
      // phase away from the awaited one and the parity wait is exact.
      if constexpr (C::kOBufs == 2) {  // own tile: wait for this WG's previous store
        if (i > 0) mbar_wait(&stage_free[q], static_cast<uint32_t>(i - 1) & 1);
      } else {
        if (q == 1)
          mbar_wait(&stage_free[0], static_cast<uint32_t>(i) & 1);
        else if (i > 0)
          mbar_wait(&stage_free[1], static_cast<uint32_t>(i - 1) & 1);
      }
      uint8_t* stage = sO + (C::kOBufs == 2 ? q : 0) * C::kQTileBytes;
      stage_o_tile<D, kBF16>(tO, stage, r, 1.0f / l);
      tc_fence_before();
      fence_proxy_async_smem();  // staged O visible to the TMA (async proxy)
      mbar_arrive(&o_empty[C::kEpiWG ? 2 * q + (i & 1) : q]);  // O_q drained from TMEM (all 128 threads)
      mbar_arrive(&stage_ready[C::kOBufs == 2 ? q : 0]);  // this thread's row staged
      const int row = qb * 2 * C::kBM + q * C::kBM + r;
      if (row < args.n_q && args.lse != nullptr)
        args.lse[(static_cast<int64_t>(b) * args.H + head) * N + row] = m * args.scale + logf(l);
      prof.mark(6);
      trace_stamp(args, trq, q, n_kv - 1, 7);
#ifdef FMHA_TRACE_BUILD
      if (tr && i < 8 && r == 0) args.trace[(3 * n_kv) * 16 + i * 8 + 3 + q] = clock64();
#endif
    }
    // consume WG 1's last hand-over so no named barrier is left half-arrived
    if constexpr (kSeq)
      if (q == 0) named_bar_sync(C::kSeqBar, 256);
    prof.flush(args, warp);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc(tmem, C::kTmemCols);
}

}  // namespace fmha_b200
