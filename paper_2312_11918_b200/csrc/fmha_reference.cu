// fmha_reference.cu -- an independent fp32 CUDA-core attention (the
// reference's Alg. 1 `standard_attention` semantics,
// /root/reference/proj/src/attention.cpp:137-151: S in fp32, exact expf,
// unrounded P, O = (P V) / Sigma) used by the CLI's `verify` command as the
// device-side checker of the tensor-core kernels.  It is a verification
// path, not the hot path: one CTA per (32 query rows, head, batch), a warp
// octet per query row, K/V tiles staged in shared memory as fp32.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/fmha/fmha.h"
#include "fmha_errors.hpp"

namespace {

constexpr int kRows = 32;     // query rows per CTA
constexpr int kParts = 8;     // threads per query row
template <int D>
constexpr int keys_per_tile() { return D == 256 ? 16 : 32; }  // fp32 K+V tile <= 33 KB
constexpr int kThreads = kRows * kParts;

__device__ __forceinline__ float load16(const uint16_t* p, bool bf16) {
  const uint16_t h = *p;
  if (bf16) return __uint_as_float(static_cast<uint32_t>(h) << 16);
  return __half2float(__ushort_as_half(h));
}

template <int D>
__global__ void __launch_bounds__(kThreads) reference_kernel(
    const uint16_t* __restrict__ q, const uint16_t* __restrict__ k, const uint16_t* __restrict__ v,
    float* __restrict__ o, float* __restrict__ lse, fmha_fwd_params p, float scale, bool bf16) {
  constexpr int kDP = D / kParts;  // dims per thread
  constexpr int kKeys = keys_per_tile<D>();
  __shared__ float sK[kKeys][D + 1];
  __shared__ float sV[kKeys][D + 1];
  const int head = blockIdx.y, b = blockIdx.z;
  const int r = threadIdx.x / kParts, part = threadIdx.x % kParts;
  const int row = blockIdx.x * kRows + r;
  const bool row_ok = row < p.N;
  float qr[kDP], acc[kDP];
  const uint16_t* qp = q + b * p.q_stride[0] + static_cast<int64_t>(row_ok ? row : 0) * p.q_stride[1] +
                       head * p.q_stride[2];
#pragma unroll
  for (int i = 0; i < kDP; ++i) {
    qr[i] = load16(qp + part * kDP + i, bf16);
    acc[i] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int j0 = 0; j0 < p.N; j0 += kKeys) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < kKeys * D; idx += kThreads) {
      const int jj = idx / D, c = idx % D, j = j0 + jj;
      float kv = 0.f, vv = 0.f;
      if (j < p.N) {
        kv = load16(k + b * p.k_stride[0] + static_cast<int64_t>(j) * p.k_stride[1] + head * p.k_stride[2] + c, bf16);
        vv = load16(v + b * p.v_stride[0] + static_cast<int64_t>(j) * p.v_stride[1] + head * p.v_stride[2] + c, bf16);
      }
      sK[jj][c] = kv;
      sV[jj][c] = vv;
    }
    __syncthreads();
    const int nk = (p.N - j0) < kKeys ? static_cast<int>(p.N - j0) : kKeys;
    for (int jj = 0; jj < nk; ++jj) {
      float dot = 0.f;
#pragma unroll
      for (int i = 0; i < kDP; ++i) dot = fmaf(qr[i], sK[jj][part * kDP + i], dot);
#pragma unroll
      for (int off = kParts / 2; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
      const float s = dot * scale;
      const float m_new = fmaxf(m, s);
      const float alpha = expf(m - m_new);
      const float pj = expf(s - m_new);
      l = l * alpha + pj;
#pragma unroll
      for (int i = 0; i < kDP; ++i) acc[i] = fmaf(pj, sV[jj][part * kDP + i], acc[i] * alpha);
      m = m_new;
    }
  }
  if (!row_ok) return;
  float* op = o + ((static_cast<int64_t>(b) * p.N + row) * p.h + head) * D;
  const float inv = 1.0f / l;
#pragma unroll
  for (int i = 0; i < kDP; ++i) op[part * kDP + i] = acc[i] * inv;
  if (lse && part == 0) lse[(static_cast<int64_t>(b) * p.h + head) * p.N + row] = m + logf(l);
}

}  // namespace

extern "C" fmha_status fmha_fwd_reference(const fmha_fwd_params* p, const void* q, const void* k,
                                          const void* v, float* o, float* lse, void* cuda_stream) {
  fmha_status s = fmha_fwd_check(p);
  if (s != FMHA_OK) return s;
  if (!q || !k || !v || !o) {
    fmha_b200::g_last_error = "null tensor pointer";
    return FMHA_ERR_CONFIG;
  }
  const float scale =
      p->scale > 0.0f ? p->scale : static_cast<float>(1.0 / std::sqrt(static_cast<double>(p->d)));
  dim3 grid(static_cast<unsigned>((p->N + kRows - 1) / kRows), static_cast<unsigned>(p->h),
            static_cast<unsigned>(p->L));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  auto qq = static_cast<const uint16_t*>(q), kk = static_cast<const uint16_t*>(k),
       vv = static_cast<const uint16_t*>(v);
  const bool bf = p->dtype == FMHA_BF16;
  switch (p->d) {
    case 64: reference_kernel<64><<<grid, kThreads, 0, st>>>(qq, kk, vv, o, lse, *p, scale, bf); break;
    case 128: reference_kernel<128><<<grid, kThreads, 0, st>>>(qq, kk, vv, o, lse, *p, scale, bf); break;
    default: reference_kernel<256><<<grid, kThreads, 0, st>>>(qq, kk, vv, o, lse, *p, scale, bf); break;
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fmha_b200::g_last_error = std::string("reference kernel launch: ") + cudaGetErrorString(e);
    return FMHA_ERR_CUDA;
  }
  return FMHA_OK;
}
