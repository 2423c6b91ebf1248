// fmha_api.cu -- the C ABI (include/fmha/fmha.h): argument validation, TMA
// descriptor construction, kernel dispatch, and the host-buffer entry points.
//
// The driver entry point cuTensorMapEncodeTiled is resolved at run time via
// cudaGetDriverEntryPoint, so the library links only the CUDA runtime.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fmha/fmha.h"
#include "fmha_errors.hpp"
#include "fmha_fwd_d64_kernel.cuh"
#include "fmha_fwd_pair_kernel.cuh"
#include "fmha_fwd_st_kernel.cuh"
#include "fmha_fwd_kernel.cuh"
#include "fmha_fwd_split_kernel.cuh"
#include "fmha_fwd_dbs_kernel.cuh"

namespace {

using fmha_b200::g_last_error;
using fmha_b200::g_last_launches;

fmha_status fail(fmha_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

fmha_status cuda_fail(cudaError_t e, const char* what) {
  return fail(FMHA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 4-D map over a BSHD tensor: dims (d, h, N, L), box (64, 1, rows, 1), 128-B
// swizzle -- each box lands in shared memory as `rows` x 128 B swizzle atoms,
// exactly the K-major SW128 canonical layout tcgen05 descriptors expect.
// Descriptor cache (per host thread, no locking): small calls re-use the
// same tensors every step, and encoding 4-6 maps per call is a fixed host
// cost of several microseconds.  Keyed by every input of the encoding.
struct MapKey {
  const void* ptr;
  int64_t d, h, N, L, s0, s1, s2;
  int box_rows, dt;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && d == o.d && h == o.h && N == o.N && L == o.L && s0 == o.s0 && s1 == o.s1 &&
           s2 == o.s2 && box_rows == o.box_rows && dt == o.dt;
  }
};
struct MapCache {
  static constexpr int kSize = 32;
  MapKey key[kSize];
  CUtensorMap map[kSize];
  bool used[kSize] = {};
  int next = 0;
};

bool make_map(CUtensorMap* map, const void* ptr, fmha_dtype dt, const fmha_fwd_params* p,
              const int64_t stride[3], int box_rows) {
  thread_local MapCache cache;
  const MapKey k{ptr, p->d, p->h, p->N, p->L, stride[0], stride[1], stride[2], box_rows, static_cast<int>(dt)};
  for (int i = 0; i < MapCache::kSize; ++i)
    if (cache.used[i] && cache.key[i] == k) {
      *map = cache.map[i];
      return true;
    }
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(p->d), static_cast<cuuint64_t>(p->h),
                        static_cast<cuuint64_t>(p->N), static_cast<cuuint64_t>(p->L)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(stride[2]) * 2,
                           static_cast<cuuint64_t>(stride[1]) * 2,
                           static_cast<cuuint64_t>(stride[0]) * 2};
  cuuint32_t box[4] = {64, 1, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, dt == FMHA_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                  4, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  const int slot = cache.next;
  cache.next = (cache.next + 1) % MapCache::kSize;
  cache.key[slot] = k;
  cache.map[slot] = *map;
  cache.used[slot] = true;
  return true;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

float resolve_scale(const fmha_fwd_params* p) {
  // AttentionProblem::scale = float(1.0 / std::sqrt(double(Q.d))), attention.cpp:18
  return p->scale > 0.0f ? p->scale : static_cast<float>(1.0 / std::sqrt(static_cast<double>(p->d)));
}

// Debug timeline buffer (FMHA_TRACE=1): see FwdArgs::trace.
unsigned long long* trace_buffer(size_t n) {
  static unsigned long long* buf = nullptr;
  static size_t cap = 0;
  static const bool on = [] {
    const char* e = std::getenv("FMHA_TRACE");
    return e && e[0] == '1';
  }();
  if (!on) return nullptr;
  if (cap < n) {
    if (buf) cudaFree(buf);
    if (cudaMalloc(&buf, n * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    cudaMemset(buf, 0, n * sizeof(unsigned long long));
    cap = n;
  }
  return buf;
}

// SM count of the current device (cached per device: one process may drive
// several GPUs through the host entry points).
int num_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < 0 || dev >= 64) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// The >48 KB dynamic shared memory opt-in of kernel K on the current device.
// The attribute belongs to the device context, so it is applied once per
// (kernel, device) -- not once per process.
template <auto K>
cudaError_t ensure_smem_attr(int bytes) {
  static std::atomic<uint64_t> done{0};  // bit d: set on device d
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = (dev >= 0 && dev < 64) ? (1ull << dev) : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

template <int D, bool BF16, int EMU = 0>
fmha_status launch_d128(const fmha_fwd_params* p, const CUtensorMap& mq, const CUtensorMap& mk,
                        const CUtensorMap& mv, const CUtensorMap& mo, float* lse, cudaStream_t st, int64_t nq) {
  using Cfg = fmha_b200::FwdCfg<D>;
  auto kern = fmha_b200::fmha_fwd_sm100_kernel<D, BF16, EMU>;
  if (cudaError_t e = ensure_smem_attr<fmha_b200::fmha_fwd_sm100_kernel<D, BF16, EMU>>(Cfg::kSmemAlloc); e != cudaSuccess)
    return cuda_fail(e, "cudaFuncSetAttribute");
  fmha_b200::FwdArgs a{};
  a.lse = lse;
  a.N = static_cast<int>(p->N);
  a.n_q = static_cast<int>(nq);
  a.H = static_cast<int>(p->h);
  a.L = static_cast<int>(p->L);
  a.n_kv_tiles = static_cast<int>((p->N + Cfg::kBN - 1) / Cfg::kBN);
  a.n_qblocks = static_cast<int>((nq + 2 * Cfg::kBM - 1) / (2 * Cfg::kBM));
  a.n_units = a.n_qblocks * a.H * a.L;
  a.scale = resolve_scale(p);
  a.scale_log2 = a.scale * 1.4426950408889634f;
  const int grid = std::min(a.n_units, num_sms());
  a.trace = trace_buffer(std::max<size_t>(static_cast<size_t>(3 * a.n_kv_tiles * 16 + 64),
                                          static_cast<size_t>(grid) * 16 * 8));
  kern<<<grid, Cfg::kThreads, Cfg::kSmemAlloc, st>>>(mq, mk, mv, mo, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  g_last_launches = 1;
  return FMHA_OK;
}

// The double-buffered-S d=128 kernel: one 128-row Q tile per unit, one
// persistent CTA per SM.
template <bool BF16, int EMU>
fmha_status launch_dbs(const fmha_fwd_params* p, const CUtensorMap& mq, const CUtensorMap& mk,
                       const CUtensorMap& mv, const CUtensorMap& mo, float* lse, cudaStream_t st, int64_t nq) {
  using Cfg = fmha_b200::FwdCfgDbs;
  auto kern = fmha_b200::fmha_fwd_dbs_kernel<BF16, EMU>;
  if (cudaError_t e = ensure_smem_attr<fmha_b200::fmha_fwd_dbs_kernel<BF16, EMU>>(Cfg::kSmemAlloc); e != cudaSuccess)
    return cuda_fail(e, "cudaFuncSetAttribute");
  fmha_b200::FwdArgs a{};
  a.lse = lse;
  a.N = static_cast<int>(p->N);
  a.n_q = static_cast<int>(nq);
  a.H = static_cast<int>(p->h);
  a.L = static_cast<int>(p->L);
  a.n_kv_tiles = static_cast<int>((p->N + Cfg::kBN - 1) / Cfg::kBN);
  a.n_qblocks = static_cast<int>((nq + Cfg::kBM - 1) / Cfg::kBM);
  a.n_units = a.n_qblocks * a.H * a.L;
  a.scale = resolve_scale(p);
  a.scale_log2 = a.scale * 1.4426950408889634f;
  a.trace = trace_buffer(fmha_b200::kTraceSteps * 48);
  const int grid = std::min(a.n_units, num_sms());
  kern<<<grid, Cfg::kThreads, Cfg::kSmemAlloc, st>>>(mq, mk, mv, mo, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch (double-buffered S)");
  g_last_launches = 1;
  return FMHA_OK;
}

// The split-row ping-pong kernel (two warps per softmax row): same unit /
// grid as launch_d128.
template <int D, bool BF16, int EMU>
fmha_status launch_split(const fmha_fwd_params* p, const CUtensorMap& mq, const CUtensorMap& mk,
                         const CUtensorMap& mv, const CUtensorMap& mo, float* lse, cudaStream_t st, int64_t nq) {
  using Cfg = fmha_b200::SplitCfg<D>;
  auto kern = fmha_b200::fmha_fwd_split_kernel<D, BF16, EMU>;
  if (cudaError_t e = ensure_smem_attr<fmha_b200::fmha_fwd_split_kernel<D, BF16, EMU>>(Cfg::kSmemAlloc);
      e != cudaSuccess)
    return cuda_fail(e, "cudaFuncSetAttribute");
  fmha_b200::FwdArgs a{};
  a.lse = lse;
  a.N = static_cast<int>(p->N);
  a.n_q = static_cast<int>(nq);
  a.H = static_cast<int>(p->h);
  a.L = static_cast<int>(p->L);
  a.n_kv_tiles = static_cast<int>((p->N + Cfg::kBN - 1) / Cfg::kBN);
  a.n_qblocks = static_cast<int>((nq + 2 * Cfg::kBM - 1) / (2 * Cfg::kBM));
  a.n_units = a.n_qblocks * a.H * a.L;
  a.scale = resolve_scale(p);
  a.scale_log2 = a.scale * 1.4426950408889634f;
  a.trace = nullptr;
  const int grid = std::min(a.n_units, num_sms());
  kern<<<grid, Cfg::kThreads, Cfg::kSmemAlloc, st>>>(mq, mk, mv, mo, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch (split-row)");
  g_last_launches = 1;
  return FMHA_OK;
}

// CTA-pair kernels (cluster 2 x 1 x 1 over the Q-tile axis).  An odd
// Q-tile count gets one padding CTA per (b, head): its Q rows are all past N
// (TMA zero-fills them, nothing is stored).  `mk64` is a K map with 64-row boxes.
// d = 64: two-Q-tile ping-pong with 64-row K/V steps, two persistent CTAs per
// SM.  `mk64` / `mv64` are K / V maps with 64-row boxes.
template <bool BF16, int EMU>
fmha_status launch_d64(const fmha_fwd_params* p, const CUtensorMap& mq, const CUtensorMap& mk64,
                       const CUtensorMap& mv64, const CUtensorMap& mo, void* o, float* lse, cudaStream_t st,
                       int64_t nq) {
  using Cfg = fmha_b200::FwdCfgD64;
  auto kern = fmha_b200::fmha_fwd_d64_kernel<BF16, EMU>;
  if (cudaError_t e = ensure_smem_attr<fmha_b200::fmha_fwd_d64_kernel<BF16, EMU>>(Cfg::kSmemAlloc); e != cudaSuccess)
    return cuda_fail(e, "cudaFuncSetAttribute");
  fmha_b200::FwdArgs a{};
  a.o = o;
  a.lse = lse;
  a.o_sb = p->o_stride[0];
  a.o_sn = p->o_stride[1];
  a.o_sh = p->o_stride[2];
  a.N = static_cast<int>(p->N);
  a.n_q = static_cast<int>(nq);
  a.H = static_cast<int>(p->h);
  a.L = static_cast<int>(p->L);
  a.n_kv_tiles = static_cast<int>((p->N + Cfg::kBN - 1) / Cfg::kBN);
  a.n_qblocks = static_cast<int>((nq + 2 * Cfg::kBM - 1) / (2 * Cfg::kBM));
  a.n_units = a.n_qblocks * a.H * a.L;
  a.scale = resolve_scale(p);
  a.scale_log2 = a.scale * 1.4426950408889634f;
  a.trace = nullptr;
  const int grid = std::min(a.n_units, 2 * num_sms());
  kern<<<grid, Cfg::kThreads, Cfg::kSmemAlloc, st>>>(mq, mk64, mv64, mo, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch (d=64)");
  g_last_launches = 1;
  return FMHA_OK;
}

template <int D, int BN, bool BF16, int EMU>
fmha_status launch_pair(const fmha_fwd_params* p, const CUtensorMap& mq, const CUtensorMap& mk64,
                        const CUtensorMap& mv, const CUtensorMap& mo, void* o, float* lse, cudaStream_t st,
                        int64_t nq) {
  using Cfg = fmha_b200::FwdCfgPair<D, BN>;
  auto kern = fmha_b200::fmha_fwd_pair_kernel<D, BN, BF16, EMU>;
  if (cudaError_t e = ensure_smem_attr<fmha_b200::fmha_fwd_pair_kernel<D, BN, BF16, EMU>>(Cfg::kSmemAlloc); e != cudaSuccess)
    return cuda_fail(e, "cudaFuncSetAttribute");
  fmha_b200::FwdArgs a{};
  a.o = o;
  a.lse = lse;
  a.o_sb = p->o_stride[0];
  a.o_sn = p->o_stride[1];
  a.o_sh = p->o_stride[2];
  a.N = static_cast<int>(p->N);
  a.n_q = static_cast<int>(nq);
  a.H = static_cast<int>(p->h);
  a.n_kv_tiles = static_cast<int>((p->N + Cfg::kBN - 1) / Cfg::kBN);
  a.scale = resolve_scale(p);
  a.scale_log2 = a.scale * 1.4426950408889634f;
  a.trace = nullptr;
  cudaLaunchConfig_t cfg{};
  const unsigned n_qtiles = static_cast<unsigned>((nq + Cfg::kBM - 1) / Cfg::kBM);
  cfg.gridDim = dim3((n_qtiles + 1) & ~1u, static_cast<unsigned>(p->h), static_cast<unsigned>(p->L));
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemAlloc;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mq, mk64, mv, mo, a);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch (CTA pair)");
  g_last_launches = 1;
  return FMHA_OK;
}

template <int D, bool BF16, int BN>
fmha_status launch_st(const fmha_fwd_params* p, const CUtensorMap& mq, const CUtensorMap& mk,
                      const CUtensorMap& mv, const CUtensorMap& mo, void* o, float* lse, cudaStream_t st,
                      int64_t nq) {
  using Cfg = fmha_b200::FwdCfgST<D, BN>;
  auto kern = fmha_b200::fmha_fwd_st_kernel<D, BF16, BN>;
  if (cudaError_t e = ensure_smem_attr<fmha_b200::fmha_fwd_st_kernel<D, BF16, BN>>(Cfg::kSmemAlloc); e != cudaSuccess)
    return cuda_fail(e, "cudaFuncSetAttribute");
  fmha_b200::FwdArgs a{};
  a.o = o;
  a.lse = lse;
  a.o_sb = p->o_stride[0];
  a.o_sn = p->o_stride[1];
  a.o_sh = p->o_stride[2];
  a.N = static_cast<int>(p->N);
  a.n_q = static_cast<int>(nq);
  a.H = static_cast<int>(p->h);
  a.n_kv_tiles = static_cast<int>((p->N + Cfg::kBN - 1) / Cfg::kBN);
  a.scale = resolve_scale(p);
  a.scale_log2 = a.scale * 1.4426950408889634f;
  a.trace = nullptr;
  dim3 grid(static_cast<unsigned>((nq + Cfg::kBM - 1) / Cfg::kBM), static_cast<unsigned>(p->h),
            static_cast<unsigned>(p->L));
  kern<<<grid, Cfg::kThreads, Cfg::kSmemAlloc, st>>>(mq, mk, mv, mo, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    return fail(FMHA_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e) + " (regs " +
                                   std::to_string(fa.numRegs) + ", max threads " +
                                   std::to_string(fa.maxThreadsPerBlock) + ", local " +
                                   std::to_string(fa.localSizeBytes) + " B, launch " +
                                   std::to_string(Cfg::kThreads) + " threads, smem " +
                                   std::to_string(Cfg::kSmemAlloc) + ")");
  }
  g_last_launches = 1;
  return FMHA_OK;
}

// Per-device workspace for the host entry points (grow-only): one device
// buffer, three streams (H2D copies, kernels, D2H copies) and a pool of
// per-chunk events.
struct Workspace {
  std::mutex mu;
  void* dev = nullptr;
  size_t bytes = 0;
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> ev_in;  // event pool (one per chunk and per head group)
};
Workspace& workspace(int device) {
  static Workspace ws[64];
  return ws[device & 63];
}

// One pipeline chunk of the host entry point: batches [b0, b1) x heads [h0, h1).
struct Chunk {
  int64_t b0, b1, h0, h1;
};

// Host-entry pipeline plan.  Inputs are copied in whole-batch chunks of about
// `in_bytes` (contiguous copies run at the full PCIe rate, strided 2-D copies
// at ~80% of it -- measured); a single-batch chunk is computed and copied back
// in head groups of about `out_bytes` of O, so the pipeline tail (the last
// group's kernel and D2H) stays small.  Heads are independent,
// so every group is its own sub-problem.
struct InChunk {
  int64_t b0, b1;
  std::vector<Chunk> groups;
};
std::vector<InChunk> plan_chunks(const fmha_fwd_params* p, size_t in_bytes, size_t out_bytes,
                                 bool head_groups = true) {
  std::vector<InChunk> out;
  const size_t batch_in = static_cast<size_t>(3 * p->N * p->h * p->d * 2);
  const size_t batch_out = static_cast<size_t>(p->N * p->h * p->d * 2);
  const int64_t bpc = std::max<int64_t>(1, static_cast<int64_t>(in_bytes / batch_in));
  for (int64_t b0 = 0; b0 < p->L; b0 += bpc) {
    InChunk c{b0, std::min(p->L, b0 + bpc), {}};
    int64_t groups = 1;
    if (head_groups && c.b1 - c.b0 == 1)
      groups = std::min<int64_t>({p->h, 8, std::max<int64_t>(1, static_cast<int64_t>(batch_out / out_bytes))});
    const int64_t hpg = (p->h + groups - 1) / groups;
    for (int64_t h0 = 0; h0 < p->h; h0 += hpg) c.groups.push_back({c.b0, c.b1, h0, std::min(p->h, h0 + hpg)});
    out.push_back(std::move(c));
  }
  return out;
}

// Copy the [b0,b1) x [h0,h1) slice of a BSHD tensor (strides in elements)
// between host and device buffers that share the same layout.
cudaError_t copy_slice(char* dst, const char* src, const int64_t st[3], const fmha_fwd_params* p,
                       const Chunk& c, cudaMemcpyKind kind, cudaStream_t s) {
  const size_t off = static_cast<size_t>(st[0] * c.b0 + st[2] * c.h0) * 2;
  if (c.h0 == 0 && c.h1 == p->h && st[1] == p->h * p->d && st[0] == p->N * st[1])  // dense rows
    return cudaMemcpyAsync(dst + off, src + off, static_cast<size_t>(st[0] * (c.b1 - c.b0)) * 2, kind, s);
  cudaError_t e = cudaSuccess;
  for (int64_t b = c.b0; b < c.b1 && e == cudaSuccess; ++b) {
    const size_t ob = static_cast<size_t>(st[0] * b + st[2] * c.h0) * 2;
    e = cudaMemcpy2DAsync(dst + ob, static_cast<size_t>(st[1]) * 2, src + ob, static_cast<size_t>(st[1]) * 2,
                          static_cast<size_t>((c.h1 - c.h0 - 1) * st[2] + p->d) * 2, static_cast<size_t>(p->N),
                          kind, s);
  }
  return e;
}

// Copy query rows [n0, n1) of batch b (all heads) of a BSHD tensor between
// host and device buffers that share the same layout.
cudaError_t copy_rows(char* dst, const char* src, const int64_t st[3], const fmha_fwd_params* p, int64_t b,
                      int64_t n0, int64_t n1, cudaMemcpyKind kind, cudaStream_t s) {
  const size_t off = static_cast<size_t>(st[0] * b + st[1] * n0) * 2;
  if (st[1] == p->h * p->d && st[2] == p->d)  // dense rows: one contiguous range
    return cudaMemcpyAsync(dst + off, src + off, static_cast<size_t>((n1 - n0) * st[1]) * 2, kind, s);
  return cudaMemcpy2DAsync(dst + off, static_cast<size_t>(st[1]) * 2, src + off, static_cast<size_t>(st[1]) * 2,
                           static_cast<size_t>((p->h - 1) * st[2] + p->d) * 2, static_cast<size_t>(n1 - n0), kind, s);
}

// ------------------------------------------------------- kernel choice --
// Environment overrides for A/B tuning runs, read once per process:
//   FMHA_TUNE_PAIR=0   no CTA-pair kernels;  FMHA_TUNE_D64=0  no two-CTA d=64
//   kernel;  FMHA_TUNE_EMU / FMHA_TUNE_EMU64  exp2 split of the ping-pong kernel
//   (d = 128 default: kEmuEdgeFree, the position-dependent FlashAttention-4 pattern).
struct Tuning {
  bool pair_ok, d64_ok;
  int emu64, emu128;
  int split;  // split-row ping-pong for d <= 128 (FMHA_TUNE_SPLIT)
  int64_t pair128_min_n;  // d = 128 runs on CTA pairs from this N (FMHA_TUNE_PAIR128_N; default: never)
  int dbs;                // d = 128 below pair128_min_n: double-buffered-S kernel (FMHA_TUNE_DBS)
  int emu64d;             // exp2 split of the two-CTA d = 64 kernel (FMHA_TUNE_EMU64D)
  int64_t d64_min_n;      // d = 64 runs on the two-CTA kernel from this N (FMHA_TUNE_D64_N)
  int64_t tiny_tiles;     // at most this many Q tiles: one CTA per tile (FMHA_TUNE_TINY)
  int64_t tiny2_tiles;    // up to this many Q tiles: one CTA per tile, two per SM (FMHA_TUNE_TINY2)
};
const Tuning& tuning() {
  static const Tuning t = [] {
    auto env = [](const char* n, int dflt) {
      const char* e = std::getenv(n);
      return e ? std::atoi(e) : dflt;
    };
    return Tuning{env("FMHA_TUNE_PAIR", 1) != 0, env("FMHA_TUNE_D64", 1) != 0, env("FMHA_TUNE_EMU64", -1),
                  env("FMHA_TUNE_EMU", fmha_b200::kEmuEdgeFree), env("FMHA_TUNE_SPLIT", 0), env("FMHA_TUNE_PAIR128_N", 1 << 30),
                  env("FMHA_TUNE_DBS", 0), env("FMHA_TUNE_EMU64D", 4),
                  env("FMHA_TUNE_D64_N", 1024), env("FMHA_TUNE_TINY", -1),
                  env("FMHA_TUNE_TINY2", -1)};
  }();
  return t;
}

enum class Kernel { kPingPong64, kD64TwoCta, kPingPong128, kDbs128, kPair128, kPair256, kSingle256, kSingleSmall,
                    kSingleSmall2 };

// Which kernel runs a (valid) problem; thresholds are measured crossovers
// (profiles/r01_microbench.txt):
//  * d = 128: the persistent ping-pong kernel at every N beyond the one-tile
//    paths.  Since its padded-step split it beats the CTA-pair kernel at long
//    sequences too (N = 8192 +4..8 %, N = 16384 +4 %, c5 +2 % at a lower
//    power-capped clock); FMHA_TUNE_PAIR128_N=<N> keeps the pair kernel
//    (one Q tile per CTA, 64-column double-buffered S, two CTAs per SM) as an
//    opt-in from that N;
//  * d = 64, N >= 1024 or enough heads to fill every SM: the two-CTA-per-SM
//    ping-pong with 64-row K/V steps (+4 % at N = 1024 .. +6.8 % at 8192;
//    +1..9 % at N = 128..1000 with 192+ heads; slower on few-head problems);
//  * d = 256, N > 128: CTA pairs (M = 256 MMAs, each SM streams half of every
//    K/V tile; a single Q tile would pay a whole padding CTA);
//  * d <= 128 with at most #SMs Q tiles of 128 rows: the single-CTA kernel
//    (one CTA per Q tile, double-buffered S; +20..55 % on one-wave problems);
//    up to 2 x #SMs tiles (d = 128: N <= 2048) its 64-row-K/V-step form, two
//    CTAs per SM (+0..19 %);
//  * otherwise the persistent ping-pong kernel (d <= 128) or the single-CTA
//    d = 256 kernel.
// The host pipeline runs chunks / row slices of one problem: they must use the
// kernel of the WHOLE problem, so its output is bitwise equal to one device
// launch (tests/test_gpu_parity.py); set for the duration of the pipeline.
thread_local int g_forced_kernel = -1;
struct ForceKernel {
  explicit ForceKernel(int k) { g_forced_kernel = k; }
  ~ForceKernel() { g_forced_kernel = -1; }
};

Kernel select_kernel(const fmha_fwd_params* p) {
  if (g_forced_kernel >= 0) return static_cast<Kernel>(g_forced_kernel);
  const Tuning& t = tuning();
  // Problems of at most one wave of 128-row Q tiles (<= #SMs): one CTA per Q
  // tile with double-buffered S.  The persistent kernels would put two tiles
  // on each of only tiles/2 SMs (measured +20..55 %, tools/exp/tiny2.py).
  // FMHA_TUNE_TINY overrides the tile limit (0: off).
  {
    const int64_t tiles = p->L * p->h * ((p->N + 127) / 128);
    const int64_t limit = t.tiny_tiles >= 0 ? t.tiny_tiles : num_sms();
    if (p->d <= 128 && tiles <= limit && !t.dbs && !t.split) return Kernel::kSingleSmall;
    // up to two waves: one CTA per tile with 64-row K/V steps, two CTAs per SM
    // (d = 64: +0..19 %; d = 128: +4..12 % up to N = 2048, -3 % at N = 4096)
    const int64_t limit2 = t.tiny2_tiles >= 0 ? t.tiny2_tiles : (p->d == 64 || p->N <= 2048 ? 2 * num_sms() : 0);
    if (p->d <= 128 && tiles <= limit2 && !t.dbs && !t.split) return Kernel::kSingleSmall2;
    // (A wave-quantisation rule that sent badly quantised d = 128 mid-N problems
    // to this non-persistent form was +5..8 % before the ping-pong kernel's
    // padded-step split and is 3..6 % slower since: removed,
    // profiles/r02_microbench.txt.)
  }
  if (p->d == 64) {
    // the two-CTA kernel from N = 1024, and below that whenever the ping-pong
    // kernel's 256-row units would fill every SM (measured crossover: many heads
    // win 1-9 % on two CTAs per SM, few-head problems lose 5-10 %)
    const int64_t pp_units = p->L * p->h * ((p->N + 255) / 256);
    const bool many = t.d64_min_n == 1024 && pp_units >= num_sms();
    return t.d64_ok && (p->N >= t.d64_min_n || many) ? Kernel::kD64TwoCta : Kernel::kPingPong64;
  }
  if (p->d == 128)
    return t.pair_ok && p->N >= t.pair128_min_n ? Kernel::kPair128 : t.dbs ? Kernel::kDbs128 : Kernel::kPingPong128;
  return t.pair_ok && p->N > 128 ? Kernel::kPair256 : Kernel::kSingle256;
}

const char* kernel_name(Kernel k) {
  switch (k) {
    case Kernel::kPingPong64: return "fmha_fwd_sm100_kernel<64> (persistent two-Q-tile ping-pong)";
    case Kernel::kD64TwoCta: return "fmha_fwd_d64_kernel (ping-pong, 64-row K/V steps, two CTAs per SM)";
    case Kernel::kPingPong128: return "fmha_fwd_sm100_kernel<128> (persistent two-Q-tile ping-pong)";
    case Kernel::kDbs128: return "fmha_fwd_dbs_kernel<128> (persistent, double-buffered S, eight softmax warps)";
    case Kernel::kPair128: return "fmha_fwd_pair_kernel<128,64> (CTA pairs, two CTAs per SM)";
    case Kernel::kPair256: return "fmha_fwd_pair_kernel<256,128> (CTA pairs)";
    case Kernel::kSingle256: return "fmha_fwd_st_kernel<256,128> (single CTA)";
    case Kernel::kSingleSmall: return "fmha_fwd_st_kernel<64|128,128> (one CTA per Q tile, tiny problems)";
    case Kernel::kSingleSmall2: return "fmha_fwd_st_kernel<64|128,64> (one CTA per Q tile, two CTAs per SM)";
  }
  return "";
}

}  // namespace

extern "C" {

// Debug only: copy the FMHA_TRACE timeline (n entries) to host memory.
int fmha_debug_trace_copy(unsigned long long* host, int64_t n) {
  unsigned long long* b = trace_buffer(static_cast<size_t>(n));
  if (!b) return -1;
  return cudaMemcpy(host, b, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -1;
}

const char* fmha_version(void) { return "paper_2312_11918_b200 0.1.0 (sm_100a)"; }

const char* fmha_last_error(void) { return g_last_error.c_str(); }

int fmha_last_launch_count(void) { return g_last_launches; }

int64_t fmha_attention_flops(int64_t L, int64_t N, int64_t h, int64_t d) {
  return 4 * N * N * d * h * L;
}

void fmha_params_dense(fmha_fwd_params* p, int64_t L, int64_t N, int64_t h, int64_t d,
                       fmha_dtype dtype, float scale) {
  std::memset(p, 0, sizeof(*p));
  p->L = L;
  p->N = N;
  p->h = h;
  p->d = d;
  const int64_t st[3] = {N * h * d, h * d, d};  // Tensor4::offset, tensor.hpp:20-22
  for (int i = 0; i < 3; ++i) p->q_stride[i] = p->k_stride[i] = p->v_stride[i] = p->o_stride[i] = st[i];
  p->scale = scale;
  p->dtype = dtype;
}

fmha_status fmha_fwd_check(const fmha_fwd_params* p) {
  if (p == nullptr) return fail(FMHA_ERR_CONFIG, "null params");
  // AttentionProblem: "need N >= 1 and d >= 1" (attention.cpp:16-17)
  if (p->N < 1 || p->d < 1) return fail(FMHA_ERR_CONFIG, "AttentionProblem: need N >= 1 and d >= 1");
  if (p->L < 1 || p->h < 1) return fail(FMHA_ERR_CONFIG, "need L >= 1 and h >= 1");
  if (p->dtype != FMHA_F16 && p->dtype != FMHA_BF16)
    return fail(FMHA_ERR_CONFIG, "dtype must be FMHA_F16 or FMHA_BF16");
  if (p->d != 64 && p->d != 128 && p->d != 256)
    return fail(FMHA_ERR_UNSUPPORTED, "head dim " + std::to_string(p->d) +
                                          " unsupported by the sm_100a kernel (64, 128, 256)");
  if (p->N > (1ll << 31) - 256 || p->h > 65535 || p->L > 65535)
    return fail(FMHA_ERR_UNSUPPORTED, "problem too large for the launch grid");
  // the persistent kernels index work units (256 query rows of one head) with int32
  if (((p->N + 255) / 256) * p->h * p->L > (1ll << 31) - 1)
    return fail(FMHA_ERR_UNSUPPORTED, "problem too large: more than 2^31 work units");
  const int64_t* strides[4] = {p->q_stride, p->k_stride, p->v_stride, p->o_stride};
  for (auto s : strides)
    for (int i = 0; i < 3; ++i)
      if (s[i] < 1 || (s[i] % 8) != 0)
        return fail(FMHA_ERR_CONFIG, "strides must be positive multiples of 8 elements (16 B)");
  return FMHA_OK;
}

// fmha_fwd on the first `nq` query rows from `q` / `o` (keys and values: all
// p->N rows; LSE rows at `lse` + row with row stride p->N).  nq == p->N is the
// public entry point; the host pipeline also calls it on row slices of Q.
static fmha_status fwd_rows(const fmha_fwd_params* p, const void* q, const void* k, const void* v, void* o,
                            float* lse, void* cuda_stream, int64_t nq) {
  g_last_launches = 0;
  fmha_status s = fmha_fwd_check(p);
  if (s != FMHA_OK) return s;
  if (nq < 1 || nq > p->N) return fail(FMHA_ERR_CONFIG, "query row count out of range");
  fmha_fwd_params pq = *p;  // Q / O maps span the nq rows
  pq.N = nq;
  if (!q || !k || !v || !o) return fail(FMHA_ERR_CONFIG, "null tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
    return fail(FMHA_ERR_CONFIG, "tensor pointers must be 16-byte aligned");
  const int rows = 128;
  const int kv_rows = 128;  // K/V TMA box rows (d = 256 also streams 128-row K/V steps)
  CUtensorMap mq, mk, mv, mo;
  if (!make_map(&mq, q, p->dtype, &pq, p->q_stride, rows) ||
      !make_map(&mk, k, p->dtype, p, p->k_stride, kv_rows) ||
      !make_map(&mv, v, p->dtype, p, p->v_stride, kv_rows) ||
      !make_map(&mo, o, p->dtype, &pq, p->o_stride, rows))
    return fail(FMHA_ERR_CUDA, "cuTensorMapEncodeTiled failed (driver entry point or arguments)");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  const bool bf = p->dtype == FMHA_BF16;
  switch (select_kernel(p)) {
    case Kernel::kPair128: {
      CUtensorMap mkh, mvh;
      if (!make_map(&mkh, k, p->dtype, p, p->k_stride, 32) || !make_map(&mvh, v, p->dtype, p, p->v_stride, 64))
        return fail(FMHA_ERR_CUDA, "cuTensorMapEncodeTiled failed (K/V maps of the CTA-pair kernel)");
      return bf ? launch_pair<128, 64, true, 2>(p, mq, mkh, mvh, mo, o, lse, st, nq)
                : launch_pair<128, 64, false, 2>(p, mq, mkh, mvh, mo, o, lse, st, nq);
    }
    case Kernel::kD64TwoCta: {
      CUtensorMap mk64, mv64;
      if (!make_map(&mk64, k, p->dtype, p, p->k_stride, 64) || !make_map(&mv64, v, p->dtype, p, p->v_stride, 64))
        return fail(FMHA_ERR_CUDA, "cuTensorMapEncodeTiled failed (d=64 K/V maps)");
      // exp2 split of the two-CTA d=64 kernel: FMHA_TUNE_EMU64D (A/B runs), default 4/16
      const int e = tuning().emu64d;
      if (e == 6)
        return bf ? launch_d64<true, 6>(p, mq, mk64, mv64, mo, o, lse, st, nq)
                  : launch_d64<false, 6>(p, mq, mk64, mv64, mo, o, lse, st, nq);
      if (e == 8)
        return bf ? launch_d64<true, 8>(p, mq, mk64, mv64, mo, o, lse, st, nq)
                  : launch_d64<false, 8>(p, mq, mk64, mv64, mo, o, lse, st, nq);
      return bf ? launch_d64<true, 4>(p, mq, mk64, mv64, mo, o, lse, st, nq)
                : launch_d64<false, 4>(p, mq, mk64, mv64, mo, o, lse, st, nq);
    }
    case Kernel::kPingPong64: {
      // exp2 split 6/16 (measured: +1 % over 4/16 at N = 512 / 768, equal at 256)
      const int emu64 = tuning().emu64 >= 0 ? tuning().emu64 : 6;
      if (emu64 == 0)
        return bf ? launch_d128<64, true, 0>(p, mq, mk, mv, mo, lse, st, nq)
                  : launch_d128<64, false, 0>(p, mq, mk, mv, mo, lse, st, nq);
      if (emu64 == 6)
        return bf ? launch_d128<64, true, 6>(p, mq, mk, mv, mo, lse, st, nq)
                  : launch_d128<64, false, 6>(p, mq, mk, mv, mo, lse, st, nq);
      if (emu64 == 8)
        return bf ? launch_d128<64, true, 8>(p, mq, mk, mv, mo, lse, st, nq)
                  : launch_d128<64, false, 8>(p, mq, mk, mv, mo, lse, st, nq);
      return bf ? launch_d128<64, true, 4>(p, mq, mk, mv, mo, lse, st, nq)
                : launch_d128<64, false, 4>(p, mq, mk, mv, mo, lse, st, nq);
    }
    case Kernel::kPingPong128: {
      const int emu = tuning().emu128;
      if (tuning().split) {
        if (emu == 2)
          return bf ? launch_split<128, true, 2>(p, mq, mk, mv, mo, lse, st, nq)
                    : launch_split<128, false, 2>(p, mq, mk, mv, mo, lse, st, nq);
        if (emu == 6)
          return bf ? launch_split<128, true, 6>(p, mq, mk, mv, mo, lse, st, nq)
                    : launch_split<128, false, 6>(p, mq, mk, mv, mo, lse, st, nq);
        return bf ? launch_split<128, true, 4>(p, mq, mk, mv, mo, lse, st, nq)
                  : launch_split<128, false, 4>(p, mq, mk, mv, mo, lse, st, nq);
      }
      if (emu == 0)
        return bf ? launch_d128<128, true, 0>(p, mq, mk, mv, mo, lse, st, nq)
                  : launch_d128<128, false, 0>(p, mq, mk, mv, mo, lse, st, nq);
      if (emu == 2)
        return bf ? launch_d128<128, true, 2>(p, mq, mk, mv, mo, lse, st, nq)
                  : launch_d128<128, false, 2>(p, mq, mk, mv, mo, lse, st, nq);
      if (emu == 6)
        return bf ? launch_d128<128, true, 6>(p, mq, mk, mv, mo, lse, st, nq)
                  : launch_d128<128, false, 6>(p, mq, mk, mv, mo, lse, st, nq);
      if (emu == 8)
        return bf ? launch_d128<128, true, 8>(p, mq, mk, mv, mo, lse, st, nq)
                  : launch_d128<128, false, 8>(p, mq, mk, mv, mo, lse, st, nq);
      if (emu == fmha_b200::kEmuEdgeFree)
        return bf ? launch_d128<128, true, fmha_b200::kEmuEdgeFree>(p, mq, mk, mv, mo, lse, st, nq)
                  : launch_d128<128, false, fmha_b200::kEmuEdgeFree>(p, mq, mk, mv, mo, lse, st, nq);
      return bf ? launch_d128<128, true, 4>(p, mq, mk, mv, mo, lse, st, nq)
                : launch_d128<128, false, 4>(p, mq, mk, mv, mo, lse, st, nq);
    }
    case Kernel::kDbs128: {
      const int emu = tuning().emu128;
      if (emu == 6)
        return bf ? launch_dbs<true, 6>(p, mq, mk, mv, mo, lse, st, nq) : launch_dbs<false, 6>(p, mq, mk, mv, mo, lse, st, nq);
      if (emu == 8)
        return bf ? launch_dbs<true, 8>(p, mq, mk, mv, mo, lse, st, nq) : launch_dbs<false, 8>(p, mq, mk, mv, mo, lse, st, nq);
      return bf ? launch_dbs<true, 4>(p, mq, mk, mv, mo, lse, st, nq) : launch_dbs<false, 4>(p, mq, mk, mv, mo, lse, st, nq);
    }
    case Kernel::kPair256: {
      CUtensorMap mk64;
      if (!make_map(&mk64, k, p->dtype, p, p->k_stride, 64))
        return fail(FMHA_ERR_CUDA, "cuTensorMapEncodeTiled failed (K, 64-row boxes)");
      return bf ? launch_pair<256, 128, true, 4>(p, mq, mk64, mv, mo, o, lse, st, nq)
                : launch_pair<256, 128, false, 4>(p, mq, mk64, mv, mo, o, lse, st, nq);
    }
    case Kernel::kSingleSmall2: {  // 64-row K/V steps: 256 TMEM columns, two CTAs per SM
      CUtensorMap mk64, mv64;
      if (!make_map(&mk64, k, p->dtype, p, p->k_stride, 64) || !make_map(&mv64, v, p->dtype, p, p->v_stride, 64))
        return fail(FMHA_ERR_CUDA, "cuTensorMapEncodeTiled failed (64-row K/V maps)");
      if (p->d == 64)
        return bf ? launch_st<64, true, 64>(p, mq, mk64, mv64, mo, o, lse, st, nq)
                  : launch_st<64, false, 64>(p, mq, mk64, mv64, mo, o, lse, st, nq);
      return bf ? launch_st<128, true, 64>(p, mq, mk64, mv64, mo, o, lse, st, nq)
                : launch_st<128, false, 64>(p, mq, mk64, mv64, mo, o, lse, st, nq);
    }
    case Kernel::kSingleSmall:
      if (p->d == 64)
        return bf ? launch_st<64, true, 128>(p, mq, mk, mv, mo, o, lse, st, nq)
                  : launch_st<64, false, 128>(p, mq, mk, mv, mo, o, lse, st, nq);
      return bf ? launch_st<128, true, 128>(p, mq, mk, mv, mo, o, lse, st, nq)
                : launch_st<128, false, 128>(p, mq, mk, mv, mo, o, lse, st, nq);
    case Kernel::kSingle256:
    default:
      return bf ? launch_st<256, true, 128>(p, mq, mk, mv, mo, o, lse, st, nq)
                : launch_st<256, false, 128>(p, mq, mk, mv, mo, o, lse, st, nq);
  }
}

fmha_status fmha_fwd(const fmha_fwd_params* p, const void* q, const void* k, const void* v, void* o,
                     float* lse, void* cuda_stream) {
  return fwd_rows(p, q, k, v, o, lse, cuda_stream, p ? p->N : 0);
}

const char* fmha_kernel_for(const fmha_fwd_params* p) {
  if (fmha_fwd_check(p) != FMHA_OK) return nullptr;
  return kernel_name(select_kernel(p));
}

fmha_status fmha_fwd_host(const fmha_fwd_params* p, const void* q, const void* k, const void* v,
                          void* o, float* lse, int device) {
  return fmha_b200::fwd_host_pipeline(p, q, k, v, o, lse, device, nullptr, nullptr);
}

}  // extern "C"

fmha_status fmha_b200::fwd_host_pipeline(const fmha_fwd_params* p, const void* q, const void* k, const void* v,
                                         void* o, float* lse, int device,
                                         void (*prepare)(void*, int64_t, int64_t), void* ctx,
                                         void (*consume)(void*, const OutPiece&)) {
  fmha_status s = fmha_fwd_check(p);
  if (s != FMHA_OK) return s;
  if (!q || !k || !v || !o) return fail(FMHA_ERR_CONFIG, "null tensor pointer");
  // every chunk / row slice runs the whole problem's kernel (bitwise equal to one launch)
  ForceKernel force(static_cast<int>(select_kernel(p)));
  // Host buffers are BSHD views of the strides given; the device copies use
  // the same layout, so each region must be batch-major and non-overlapping
  // (the chunked copies move whole batches / row ranges of it).
  const int64_t* all_st[4] = {p->q_stride, p->k_stride, p->v_stride, p->o_stride};
  for (const int64_t* st : all_st)
    if (st[2] < p->d || st[1] < (p->h - 1) * st[2] + p->d || st[0] < (p->N - 1) * st[1] + (p->h - 1) * st[2] + p->d)
      return fail(FMHA_ERR_CONFIG,
                  "host entry point: strides must describe a batch-major, non-overlapping BSHD layout "
                  "(stride[2] >= d, stride[1] >= (h-1)*stride[2]+d, stride[0] >= (N-1)*stride[1]+(h-1)*stride[2]+d)");
  // elements spanned by a view: the last element's offset + 1
  auto extent = [&](const int64_t st[3]) {
    return static_cast<size_t>((p->L - 1) * st[0] + (p->N - 1) * st[1] + (p->h - 1) * st[2] + p->d) * 2;
  };
  const size_t nq = extent(p->q_stride);
  const size_t nk = extent(p->k_stride);
  const size_t nv = extent(p->v_stride);
  const size_t no = extent(p->o_stride);
  const size_t nl = lse ? static_cast<size_t>(p->L * p->h * p->N) * 4 : 0;
  auto up = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
  const size_t total = up(nq) + up(nk) + up(nv) + up(no) + up(nl);
  Workspace& ws = workspace(device);
  std::lock_guard<std::mutex> lock(ws.mu);
  // Restores the caller's current device on every exit, and on an error exit
  // drains the three streams first so no queued copy still touches the
  // caller's host buffers (or the shared staging) after this call returns.
  struct Guard {
    Workspace& ws;
    int prev = -1;
    bool ok = false;
    ~Guard() {
      if (!ok)
        for (cudaStream_t st : {ws.s_in, ws.s_comp, ws.s_out})
          if (st) cudaStreamSynchronize(st);
      if (prev >= 0) cudaSetDevice(prev);
    }
  } guard{ws};
  cudaError_t e = cudaGetDevice(&guard.prev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  for (cudaStream_t* st : {&ws.s_in, &ws.s_comp, &ws.s_out})
    if (!*st && (e = cudaStreamCreateWithFlags(st, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreate");
  if (ws.bytes < total) {
    if (ws.dev) cudaFree(ws.dev);
    ws.dev = nullptr;
    ws.bytes = 0;
    e = cudaMalloc(&ws.dev, total);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc workspace");
    ws.bytes = total;
  }
  char* dq = static_cast<char*>(ws.dev);
  char* dk = dq + up(nq);
  char* dv = dk + up(nk);
  char* dO = dv + up(nv);
  float* dl = lse ? reinterpret_cast<float*>(dO + up(no)) : nullptr;
  // Three-stage pipeline: the H2D stream copies batch chunk c+1 while the
  // kernels of chunk c run and the D2H stream returns earlier head groups
  // (PCIe is full duplex, so the copy-in stream runs back to back and bounds
  // the call).
  // with a consume hook (the float call shape), output pieces stay whole
  // rows (contiguous to dequantise); otherwise single-batch chunks return
  // in head groups of ~4 MB so the D2H tail stays short
  const std::vector<InChunk> plan =
      plan_chunks(p, static_cast<size_t>(16) << 20, static_cast<size_t>(4) << 20, consume == nullptr);
  size_t n_ev = plan.size();
  for (const InChunk& c : plan) n_ev += c.groups.size();
  // The last chunk, when it is one batch of a long sequence, is split by query
  // rows: its K and V go first, then Q in row slices whose kernels and O / LSE
  // copies start as each slice lands, so the work left after the final H2D
  // byte is one slice instead of a whole batch.
  const bool slice_last = plan.back().b1 - plan.back().b0 == 1 && p->N >= 1024;
  const int64_t batch_out = p->N * p->h * p->d * 2;  // ~4 MB of O per slice, 2..16 slices
  const int64_t kSlices = std::min<int64_t>(16, std::max<int64_t>(2, batch_out >> 22));
  n_ev += slice_last ? 2 * kSlices : 0;
  n_ev *= 2;  // + one "piece on the host" event per output piece (consume hook)
  std::vector<std::pair<cudaEvent_t, OutPiece>> pieces;
  while (ws.ev_in.size() < n_ev) {
    cudaEvent_t a;
    if ((e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "cudaEventCreate");
    ws.ev_in.push_back(a);
  }
  int launches = 0;
  size_t ev = 0;
  // FMHA_HOST_PROFILE=1: host-side phase times of this call on stderr
  static const bool host_prof = [] {
    const char* e = std::getenv("FMHA_HOST_PROFILE");
    return e && e[0] == '1';
  }();
  using Clock = std::chrono::steady_clock;
  const auto t_begin = Clock::now();
  double t_prepare = 0, t_wait = 0, t_consume = 0;
  auto ms_since = [](Clock::time_point t) { return std::chrono::duration<double, std::milli>(Clock::now() - t).count(); };
  // (Output pieces are consumed only once every input chunk is issued:
  // consuming finished pieces between the input chunks' conversions was
  // measured slower -- both are host-memory-bound, 10.4 vs 8.3-9.0 ms on c3.)
  size_t consumed = 0;
  for (size_t ci = 0; ci < plan.size(); ++ci) {
    const InChunk& ic = plan[ci];
    const Chunk all{ic.b0, ic.b1, 0, p->h};
    if (prepare) {
      const auto t0 = Clock::now();
      prepare(ctx, ic.b0, ic.b1);
      t_prepare += ms_since(t0);
    }
    if (slice_last && ci + 1 == plan.size()) {
      const int64_t b = ic.b0;
      if ((e = copy_slice(dk, static_cast<const char*>(k), p->k_stride, p, all, cudaMemcpyHostToDevice, ws.s_in)) != cudaSuccess ||
          (e = copy_slice(dv, static_cast<const char*>(v), p->v_stride, p, all, cudaMemcpyHostToDevice, ws.s_in)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpyAsync H2D");
      fmha_fwd_params pc = *p;
      pc.L = 1;
      const int64_t step = ((p->N + kSlices - 1) / kSlices + 255) / 256 * 256;  // whole 256-row Q blocks
      for (int64_t n0 = 0; n0 < p->N; n0 += step) {
        const int64_t n1 = std::min(p->N, n0 + step);
        cudaEvent_t in_done = ws.ev_in[ev++];
        if ((e = copy_rows(dq, static_cast<const char*>(q), p->q_stride, p, b, n0, n1, cudaMemcpyHostToDevice, ws.s_in)) != cudaSuccess ||
            (e = cudaEventRecord(in_done, ws.s_in)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(ws.s_comp, in_done, 0)) != cudaSuccess)
          return cuda_fail(e, "cudaMemcpyAsync H2D");
        auto at = [&](char* base, const int64_t st[3], int64_t row) {
          return base + static_cast<size_t>(st[0] * b + st[1] * row) * 2;
        };
        float* dl_c = dl ? dl + static_cast<size_t>(b * p->h * p->N + n0) : nullptr;
        s = fwd_rows(&pc, at(dq, p->q_stride, n0), at(dk, p->k_stride, 0), at(dv, p->v_stride, 0),
                     at(dO, p->o_stride, n0), dl_c, ws.s_comp, n1 - n0);
        if (s != FMHA_OK) return s;
        ++launches;
        cudaEvent_t comp_done = ws.ev_in[ev++];
        if ((e = cudaEventRecord(comp_done, ws.s_comp)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(ws.s_out, comp_done, 0)) != cudaSuccess ||
            (e = copy_rows(static_cast<char*>(o), dO, p->o_stride, p, b, n0, n1, cudaMemcpyDeviceToHost, ws.s_out)) != cudaSuccess)
          return cuda_fail(e, "cudaMemcpyAsync D2H");
        if (lse) {  // [h] rows of (n1 - n0) floats, pitch N
          const size_t ol = static_cast<size_t>(b * p->h * p->N + n0);
          if ((e = cudaMemcpy2DAsync(lse + ol, static_cast<size_t>(p->N) * 4, dl + ol, static_cast<size_t>(p->N) * 4,
                                     static_cast<size_t>(n1 - n0) * 4, static_cast<size_t>(p->h),
                                     cudaMemcpyDeviceToHost, ws.s_out)) != cudaSuccess)
            return cuda_fail(e, "cudaMemcpyAsync D2H lse");
        }
        if (consume) {
          cudaEvent_t landed = ws.ev_in[ev++];
          if ((e = cudaEventRecord(landed, ws.s_out)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
          pieces.push_back({landed, OutPiece{b, b + 1, 0, p->h, n0, n1}});
        }
      }
      continue;
    }
    cudaEvent_t in_done = ws.ev_in[ev++];
    if ((e = copy_slice(dq, static_cast<const char*>(q), p->q_stride, p, all, cudaMemcpyHostToDevice, ws.s_in)) != cudaSuccess ||
        (e = copy_slice(dk, static_cast<const char*>(k), p->k_stride, p, all, cudaMemcpyHostToDevice, ws.s_in)) != cudaSuccess ||
        (e = copy_slice(dv, static_cast<const char*>(v), p->v_stride, p, all, cudaMemcpyHostToDevice, ws.s_in)) != cudaSuccess ||
        (e = cudaEventRecord(in_done, ws.s_in)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(ws.s_comp, in_done, 0)) != cudaSuccess)
      return cuda_fail(e, "cudaMemcpyAsync H2D");
    for (const Chunk& c : ic.groups) {
      fmha_fwd_params pc = *p;
      pc.L = c.b1 - c.b0;
      pc.h = c.h1 - c.h0;
      auto at = [&](char* base, const int64_t st[3]) {
        return base + static_cast<size_t>(st[0] * c.b0 + st[2] * c.h0) * 2;
      };
      float* dl_c = dl ? dl + static_cast<size_t>((c.b0 * p->h + c.h0) * p->N) : nullptr;
      s = fmha_fwd(&pc, at(dq, p->q_stride), at(dk, p->k_stride), at(dv, p->v_stride), at(dO, p->o_stride),
                   dl_c, ws.s_comp);
      if (s != FMHA_OK) return s;
      ++launches;
      cudaEvent_t comp_done = ws.ev_in[ev++];
      if ((e = cudaEventRecord(comp_done, ws.s_comp)) != cudaSuccess ||
          (e = cudaStreamWaitEvent(ws.s_out, comp_done, 0)) != cudaSuccess ||
          (e = copy_slice(static_cast<char*>(o), dO, p->o_stride, p, c, cudaMemcpyDeviceToHost, ws.s_out)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpyAsync D2H");
      if (lse) {
        // [L][h][N]: the group's rows are one contiguous block per batch
        for (int64_t b = c.b0; b < c.b1; ++b) {
          const size_t ol = static_cast<size_t>((b * p->h + c.h0) * p->N);
          if ((e = cudaMemcpyAsync(lse + ol, dl + ol, static_cast<size_t>((c.h1 - c.h0) * p->N) * 4,
                                   cudaMemcpyDeviceToHost, ws.s_out)) != cudaSuccess)
            return cuda_fail(e, "cudaMemcpyAsync D2H lse");
        }
      }
      if (consume) {
        cudaEvent_t landed = ws.ev_in[ev++];
        if ((e = cudaEventRecord(landed, ws.s_out)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
        pieces.push_back({landed, OutPiece{c.b0, c.b1, c.h0, c.h1, 0, p->N}});
      }
    }
  }
  g_last_launches = launches;
  // hand each output piece to the caller as soon as it is on the host, while
  // the later pieces are still being computed / copied
  const double t_issued = ms_since(t_begin);
  for (; consumed < pieces.size(); ++consumed) {
    auto t0 = Clock::now();
    if ((e = cudaEventSynchronize(pieces[consumed].first)) != cudaSuccess) return cuda_fail(e, "kernel execution");
    t_wait += ms_since(t0);
    t0 = Clock::now();
    consume(ctx, pieces[consumed].second);
    t_consume += ms_since(t0);
  }
  if ((e = cudaStreamSynchronize(ws.s_out)) != cudaSuccess) return cuda_fail(e, "kernel execution");
  if (host_prof)
    std::fprintf(stderr,
                 "fmha host pipeline: %zu input chunks, %zu output pieces | prepare %.2f ms, all issued at %.2f ms, "
                 "waiting for pieces %.2f ms, consume %.2f ms, total %.2f ms\n",
                 plan.size(), pieces.size(), t_prepare, t_issued, t_wait, t_consume, ms_since(t_begin));
  guard.ok = true;
  return FMHA_OK;
}
