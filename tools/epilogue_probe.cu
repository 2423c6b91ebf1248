// epilogue_probe.cu -- store-only timing of the FMHA epilogue (north_star item
// 4: "the HBM GB/s of the epilogue").  Runs exactly the product's epilogue
// path -- stage_o_tile<D> (fmha_fwd_kernel.cuh: O rows from TMEM with
// tcgen05.ld 32x32b, x 1/Sigma, cvt to 16 bit, st.shared into the 128-B
// swizzled TMA layout), fence.proxy.async, one cp.async.bulk.tensor store per
// 64 head-dim columns, plus the per-row LSE write -- over every 128-row Q tile
// of an (L, N, h, d) output, with no mainloop in front of it.  One persistent
// CTA per SM walks the tiles like the product kernels; the staging tile is
// reused once its TMA store has been READ (cp.async.bulk.wait_group.read), as
// in the product's store warp.  Reports O + LSE bytes / kernel time.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_2312_11918_b200/csrc \
//        tools/epilogue_probe.cu -o build/epilogue_probe
//   build/epilogue_probe L N h d [bf16]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fmha_fwd_kernel.cuh"

using namespace fmha_b200;

// Two staging tiles: tile i+1 is staged while tile i's TMA store drains (the
// d = 64 product kernel has one per softmax WG; the d = 128 ping-pong shares
// one between its two WGs; the CTA-pair kernel stages in its Q buffer).
template <int D, bool kBF16>
__global__ void __launch_bounds__(128, 1)
    epilogue_only(const __grid_constant__ CUtensorMap tmO, float* lse, int N, int H, int n_qtiles, int n_units) {
  constexpr int kTile = 128 * D * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x >> 5, r = threadIdx.x;
  constexpr uint32_t kCols = D < 32 ? 32 : D;
  if (warp == 0) tmem_alloc(&tmem_holder, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  // O accumulator rows: some finite values (one tcgen05.st per 32 columns)
  for (int c = 0; c < D / 32; ++c) {
    uint32_t v[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) v[t] = __float_as_uint(0.001f * (r + c * 32 + t));
    tmem_st32x32b_x32(tmem + lane_off + c * 32, v);
  }
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  int k = 0;
  for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++k) {
    const int qt = u % n_qtiles, t = u / n_qtiles, head = t % H, b = t / H;
    uint8_t* stage = smem + (k & 1) * kTile;
    if (k >= 2 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
    __syncthreads();  // stage (k & 1) free again
    const float l = 1.0f + 0.01f * r;
    stage_o_tile<D, kBF16>(tmem + lane_off, stage, r, 1.0f / l);
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int c = 0; c < D / 64; ++c) tma_store_4d(&tmO, stage + c * 128 * 128, c * 64, head, qt * 128, b);
      tma_store_commit();
    }
    const int row = qt * 128 + r;
    if (row < N) lse[(static_cast<int64_t>(b) * H + head) * N + row] = 0.5f * r + logf(l);
  }
  if (threadIdx.x == 0) tma_store_wait_all();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, kCols);
}

template <int D, bool BF16>
float run(int L, int N, int H, int sms, void* o, float* lse, PFN_cuTensorMapEncodeTiled_v12000 enc) {
  CUtensorMap map;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)N, (cuuint64_t)L};
  cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)H * D * 2, (cuuint64_t)N * H * D * 2};
  cuuint32_t box[4] = {64, 1, 128, 1}, es[4] = {1, 1, 1, 1};
  if (enc(&map, BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, o, dims, strides, box,
          es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    fprintf(stderr, "encode failed\n");
    exit(1);
  }
  const int n_qtiles = (N + 127) / 128, n_units = L * H * n_qtiles;
  const int smem = 2 * 128 * D * 2 + 1024;
  auto k = epilogue_only<D, BF16>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = n_units < sms ? n_units : sms;
  for (int i = 0; i < 3; ++i) k<<<grid, 128, smem>>>(map, lse, N, H, n_qtiles, n_units);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20;
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    for (int i = 0; i < iters; ++i) k<<<grid, 128, smem>>>(map, lse, N, H, n_qtiles, n_units);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms / iters < best) best = ms / iters;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  return best;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: %s L N h d [bf16]\n", argv[0]);
    return 2;
  }
  const int L = atoi(argv[1]), N = atoi(argv[2]), H = atoi(argv[3]), D = atoi(argv[4]);
  const bool bf = argc > 5 && argv[5][0] == 'b';
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t o_bytes = static_cast<size_t>(L) * N * H * D * 2, lse_bytes = static_cast<size_t>(L) * H * N * 4;
  void* o;
  float* lse;
  cudaMalloc(&o, o_bytes);
  cudaMalloc(&lse, lse_bytes);
  float ms = 0;
  if (D == 64) ms = bf ? run<64, true>(L, N, H, sms, o, lse, enc) : run<64, false>(L, N, H, sms, o, lse, enc);
  else if (D == 128) ms = bf ? run<128, true>(L, N, H, sms, o, lse, enc) : run<128, false>(L, N, H, sms, o, lse, enc);
  else ms = bf ? run<256, true>(L, N, H, sms, o, lse, enc) : run<256, false>(L, N, H, sms, o, lse, enc);
  const double gbs = (o_bytes + lse_bytes) / (ms * 1e-3) / 1e9;
  printf("{\"L\": %d, \"N\": %d, \"h\": %d, \"d\": %d, \"dtype\": \"%s\", \"o_bytes\": %zu, \"lse_bytes\": %zu, "
         "\"ms\": %.5f, \"GBps\": %.1f}\n",
         L, N, H, D, bf ? "bf16" : "fp16", o_bytes, lse_bytes, ms, gbs);
  return 0;
}
