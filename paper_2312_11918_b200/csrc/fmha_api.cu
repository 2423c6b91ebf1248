// fmha_api.cu -- the C ABI (include/fmha/fmha.h): argument validation, TMA
// descriptor construction, kernel dispatch, and the host-buffer entry points.
//
// The driver entry point cuTensorMapEncodeTiled is resolved at run time via
// cudaGetDriverEntryPoint, so the library links only the CUDA runtime.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fmha/fmha.h"
#include "fmha_errors.hpp"
#include "fmha_fwd_d256_kernel.cuh"
#include "fmha_fwd_kernel.cuh"

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
bool make_map(CUtensorMap* map, const void* ptr, fmha_dtype dt, const fmha_fwd_params* p,
              const int64_t stride[3], int box_rows) {
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
  return r == CUDA_SUCCESS;
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

int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int D, bool BF16, int EMU = 0>
fmha_status launch_d128(const fmha_fwd_params* p, const CUtensorMap& mq, const CUtensorMap& mk,
                        const CUtensorMap& mv, const CUtensorMap& mo, float* lse, cudaStream_t st) {
  using Cfg = fmha_b200::FwdCfg<D>;
  auto kern = fmha_b200::fmha_fwd_sm100_kernel<D, BF16, EMU>;
  static bool attr_set = false;  // benign race: idempotent attribute set
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::kSmemAlloc);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    attr_set = true;
  }
  fmha_b200::FwdArgs a{};
  a.lse = lse;
  a.N = static_cast<int>(p->N);
  a.H = static_cast<int>(p->h);
  a.L = static_cast<int>(p->L);
  a.n_kv_tiles = static_cast<int>((p->N + Cfg::kBN - 1) / Cfg::kBN);
  a.n_qblocks = static_cast<int>((p->N + 2 * Cfg::kBM - 1) / (2 * Cfg::kBM));
  a.n_units = a.n_qblocks * a.H * a.L;
  a.scale = resolve_scale(p);
  a.scale_log2 = a.scale * 1.4426950408889634f;
  a.trace = trace_buffer(static_cast<size_t>(2 * a.n_kv_tiles * 16));
  const int grid = std::min(a.n_units, num_sms());
  kern<<<grid, Cfg::kThreads, Cfg::kSmemAlloc, st>>>(mq, mk, mv, mo, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  g_last_launches = 1;
  return FMHA_OK;
}

template <bool BF16>
fmha_status launch_d256(const fmha_fwd_params* p, const CUtensorMap& mq, const CUtensorMap& mk,
                        const CUtensorMap& mv, void* o, float* lse, cudaStream_t st) {
  using Cfg = fmha_b200::FwdCfgD256;
  auto kern = fmha_b200::fmha_fwd_d256_kernel<BF16>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::kSmemAlloc);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    attr_set = true;
  }
  fmha_b200::FwdArgs a{};
  a.o = o;
  a.lse = lse;
  a.o_sb = p->o_stride[0];
  a.o_sn = p->o_stride[1];
  a.o_sh = p->o_stride[2];
  a.N = static_cast<int>(p->N);
  a.H = static_cast<int>(p->h);
  a.n_kv_tiles = static_cast<int>((p->N + Cfg::kBN - 1) / Cfg::kBN);
  a.scale = resolve_scale(p);
  a.scale_log2 = a.scale * 1.4426950408889634f;
  a.trace = nullptr;
  dim3 grid(static_cast<unsigned>((p->N + Cfg::kBM - 1) / Cfg::kBM), static_cast<unsigned>(p->h),
            static_cast<unsigned>(p->L));
  kern<<<grid, Cfg::kThreads, Cfg::kSmemAlloc, st>>>(mq, mk, mv, a);
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

// Per-device workspace for the host entry points (grow-only).
struct Workspace {
  std::mutex mu;
  void* dev = nullptr;
  size_t bytes = 0;
  cudaStream_t streams[2] = {nullptr, nullptr};
};
Workspace& workspace(int device) {
  static Workspace ws[64];
  return ws[device & 63];
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
  const int64_t* strides[4] = {p->q_stride, p->k_stride, p->v_stride, p->o_stride};
  for (auto s : strides)
    for (int i = 0; i < 3; ++i)
      if (s[i] < 1 || (s[i] % 8) != 0)
        return fail(FMHA_ERR_CONFIG, "strides must be positive multiples of 8 elements (16 B)");
  return FMHA_OK;
}

fmha_status fmha_fwd(const fmha_fwd_params* p, const void* q, const void* k, const void* v, void* o,
                     float* lse, void* cuda_stream) {
  g_last_launches = 0;
  fmha_status s = fmha_fwd_check(p);
  if (s != FMHA_OK) return s;
  if (!q || !k || !v || !o) return fail(FMHA_ERR_CONFIG, "null tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
    return fail(FMHA_ERR_CONFIG, "tensor pointers must be 16-byte aligned");
  const int rows = 128;
  const int kv_rows = p->d == 256 ? 64 : 128;
  CUtensorMap mq, mk, mv, mo;
  if (!make_map(&mq, q, p->dtype, p, p->q_stride, rows) ||
      !make_map(&mk, k, p->dtype, p, p->k_stride, kv_rows) ||
      !make_map(&mv, v, p->dtype, p, p->v_stride, kv_rows) ||
      !make_map(&mo, o, p->dtype, p, p->o_stride, rows))
    return fail(FMHA_ERR_CUDA, "cuTensorMapEncodeTiled failed (driver entry point or arguments)");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  const bool bf = p->dtype == FMHA_BF16;
  switch (p->d) {
    case 64: {
      // FMHA_TUNE_EMU64 selects the exp2 split for tuning runs (pairs of 16
      // on the polynomial; default 4)
      static const int emu64 = [] {
        const char* e = std::getenv("FMHA_TUNE_EMU64");
        return e ? std::atoi(e) : 4;
      }();
      if (emu64 == 0)
        return bf ? launch_d128<64, true, 0>(p, mq, mk, mv, mo, lse, st)
                  : launch_d128<64, false, 0>(p, mq, mk, mv, mo, lse, st);
      if (emu64 == 6)
        return bf ? launch_d128<64, true, 6>(p, mq, mk, mv, mo, lse, st)
                  : launch_d128<64, false, 6>(p, mq, mk, mv, mo, lse, st);
      return bf ? launch_d128<64, true, 4>(p, mq, mk, mv, mo, lse, st)
                : launch_d128<64, false, 4>(p, mq, mk, mv, mo, lse, st);
    }
    case 128: {
      // FMHA_TUNE_EMU selects the exp2 split for tuning runs (default 4 of 16 pairs)
      static const int emu = [] {
        const char* e = std::getenv("FMHA_TUNE_EMU");
        return e ? std::atoi(e) : 4;
      }();
      if (emu == 0)
        return bf ? launch_d128<128, true, 0>(p, mq, mk, mv, mo, lse, st)
                  : launch_d128<128, false, 0>(p, mq, mk, mv, mo, lse, st);
      if (emu == 2)
        return bf ? launch_d128<128, true, 2>(p, mq, mk, mv, mo, lse, st)
                  : launch_d128<128, false, 2>(p, mq, mk, mv, mo, lse, st);
      return bf ? launch_d128<128, true, 4>(p, mq, mk, mv, mo, lse, st)
                : launch_d128<128, false, 4>(p, mq, mk, mv, mo, lse, st);
    }
    default:
      return bf ? launch_d256<true>(p, mq, mk, mv, o, lse, st)
                : launch_d256<false>(p, mq, mk, mv, o, lse, st);
  }
}

fmha_status fmha_fwd_host(const fmha_fwd_params* p, const void* q, const void* k, const void* v,
                          void* o, float* lse, int device) {
  fmha_status s = fmha_fwd_check(p);
  if (s != FMHA_OK) return s;
  if (!q || !k || !v || !o) return fail(FMHA_ERR_CONFIG, "null tensor pointer");
  // Host buffers are taken as dense BSHD of the strides given (elements
  // spanned = stride[0] * L).
  const size_t nq = static_cast<size_t>(p->q_stride[0] * p->L) * 2;
  const size_t nk = static_cast<size_t>(p->k_stride[0] * p->L) * 2;
  const size_t nv = static_cast<size_t>(p->v_stride[0] * p->L) * 2;
  const size_t no = static_cast<size_t>(p->o_stride[0] * p->L) * 2;
  const size_t nl = lse ? static_cast<size_t>(p->L * p->h * p->N) * 4 : 0;
  auto up = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
  const size_t total = up(nq) + up(nk) + up(nv) + up(no) + up(nl);
  Workspace& ws = workspace(device);
  std::lock_guard<std::mutex> lock(ws.mu);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  for (auto& st : ws.streams)
    if (!st && (e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreate");
  if (ws.bytes < total) {
    if (ws.dev) cudaFree(ws.dev);
    ws.dev = nullptr;
    ws.bytes = 0;
    e = cudaMalloc(&ws.dev, total);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc workspace");
    ws.bytes = total;
  }
  char* base = static_cast<char*>(ws.dev);
  char* dq = base;
  char* dk = dq + up(nq);
  char* dv = dk + up(nk);
  char* dO = dv + up(nv);
  float* dl = lse ? reinterpret_cast<float*>(dO + up(no)) : nullptr;
  // Batch chunks alternate between two streams so the H2D copy of chunk c+1
  // overlaps the kernel and the D2H copy of chunk c (copy engines and SMs
  // work concurrently); each chunk is an independent sub-problem.
  const int64_t n_chunks = std::min<int64_t>(p->L, 4);
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int64_t b0 = p->L * c / n_chunks, b1 = p->L * (c + 1) / n_chunks;
    cudaStream_t st = ws.streams[c & 1];
    fmha_fwd_params pc = *p;
    pc.L = b1 - b0;
    const size_t oq = static_cast<size_t>(p->q_stride[0] * b0) * 2, ok_ = static_cast<size_t>(p->k_stride[0] * b0) * 2,
                 ov = static_cast<size_t>(p->v_stride[0] * b0) * 2, oo = static_cast<size_t>(p->o_stride[0] * b0) * 2;
    const size_t cq = static_cast<size_t>(p->q_stride[0] * pc.L) * 2, ck = static_cast<size_t>(p->k_stride[0] * pc.L) * 2,
                 cv = static_cast<size_t>(p->v_stride[0] * pc.L) * 2, co = static_cast<size_t>(p->o_stride[0] * pc.L) * 2;
    const size_t ol = static_cast<size_t>(b0 * p->h * p->N), cl = static_cast<size_t>(pc.L * p->h * p->N);
    if ((e = cudaMemcpyAsync(dq + oq, static_cast<const char*>(q) + oq, cq, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dk + ok_, static_cast<const char*>(k) + ok_, ck, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dv + ov, static_cast<const char*>(v) + ov, cv, cudaMemcpyHostToDevice, st)) != cudaSuccess)
      return cuda_fail(e, "cudaMemcpyAsync H2D");
    s = fmha_fwd(&pc, dq + oq, dk + ok_, dv + ov, dO + oo, dl ? dl + ol : nullptr, st);
    if (s != FMHA_OK) return s;
    if ((e = cudaMemcpyAsync(static_cast<char*>(o) + oo, dO + oo, co, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      return cuda_fail(e, "cudaMemcpyAsync D2H");
    if (lse && (e = cudaMemcpyAsync(lse + ol, dl + ol, cl * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      return cuda_fail(e, "cudaMemcpyAsync D2H lse");
  }
  g_last_launches = static_cast<int>(n_chunks);
  if ((e = cudaStreamSynchronize(ws.streams[0])) != cudaSuccess ||
      (e = cudaStreamSynchronize(ws.streams[1])) != cudaSuccess)
    return cuda_fail(e, "kernel execution");
  return FMHA_OK;
}

}  // extern "C"
