// issue_probe.cu -- does a warp blocked on tcgen05.mma issue (MMA queue
// full) steal issue bandwidth from the other warps of its SM sub-partition?
// 8 warps per CTA, one CTA per SM.  Warp 1 (SMSP 1) optionally issues a long
// back-to-back stream of M128 N128 K16 MMAs; every other warp runs a fixed
// FFMA/MUFU loop and records its duration.  Compare SMSP 1's compute warp
// (warp 5) with the others, MMA stream on vs off.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//        -I paper_2312_11918_b200/csrc tools/issue_probe.cu -o build/issue_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace fmha_b200;

// 0: no MMA, 1: elect per MMA (mma_ss_elect), 2: batched (mma_ss_k4),
// 3: batched + paced (commit each group of 4 to a barrier, wait for group g-2
//    before issuing group g), 4: paced groups of 2 (elect per MMA)
template <int MODE>
__global__ void __launch_bounds__(256, 1) probe(int n_mma, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint64_t gbar[4];
  __shared__ uint32_t tmem_holder;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&gbar[i], 1);
    fence_mbar_init();
  }
  const int warp = threadIdx.x >> 5;
  if (warp == 1) tmem_alloc(&tmem_holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const long long c0 = clock64();
  if (warp == 1) {
    if (MODE != 0) {
      const uint32_t a = smem_u32(smem), bb = smem_u32(smem + 32768);
      constexpr uint32_t idesc = idesc_f16(false, 128, 128, false, false);
      const uint64_t ad = sdesc_sw128(a, 16, 1024), bd = sdesc_sw128(bb, 16, 1024);
      const int gs = MODE == 4 ? 2 : 4;
      for (int i = 0; i < n_mma / gs; ++i) {
        if (MODE >= 3) {
          if (i >= 2) mbar_wait(&gbar[(i - 2) & 3], ((i - 2) >> 2) & 1);
          if (MODE == 3) {
            mma_ss_k4(tmem, ad, bd, idesc, 1);
          } else {
            mma_ss_elect(tmem, ad, bd, idesc, 1);
            mma_ss_elect(tmem, ad + 2, bd + 2, idesc, 1);
          }
          mma_commit_elect(&gbar[i & 3]);
          continue;
        }
        if (MODE == 1) {
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_ss_elect(tmem, ad + 2 * k, bd + 2 * k, idesc, 1);
        } else {
          mma_ss_k4(tmem, ad, bd, idesc, 1);
        }
      }
      mma_commit_elect(&bar);
      mbar_wait(&bar, 0);
    }
  } else {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5;
    for (int i = 0; i < iters; ++i) {
      x0 = fmaf(x0, 1.0001f, 0.5f);
      x1 = fmaf(x1, 1.0001f, 0.5f);
      x2 = fmaf(x2, 1.0001f, 0.5f);
      x3 = fmaf(x3, 1.0001f, 0.5f);
      x4 = ex2_approx(x4 * 1e-9f);
      x5 = ex2_approx(x5 * 1e-9f);
    }
    if (x0 + x1 + x2 + x3 + x4 + x5 == 12345.f) out[1000] = 1;
  }
  const long long c1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 8 + warp] = c1 - c0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

template <int MODE>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * 8 * 8 + 8 * 1001);
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int n_mma = 2048, iters = 4000;
  probe<MODE><<<148, 256, 80 * 1024>>>(n_mma, iters, d);
  probe<MODE><<<148, 256, 80 * 1024>>>(n_mma, iters, d);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("%s failed\n", name);
    return;
  }
  std::vector<long long> h(148 * 8);
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  printf("%-22s", name);
  for (int w = 0; w < 8; ++w) {
    double s = 0;
    for (int b = 0; b < 148; ++b) s += h[b * 8 + w];
    printf("  w%d %7.0f", w, s / 148);
  }
  printf("   (clk; warp 1 = MMA issuer, SMSP = warp %% 4)\n");
  cudaFree(d);
}

int main() {
  run<0>("no MMA stream");
  run<1>("MMA elect-per-MMA");
  run<2>("MMA batched k4");
  run<3>("MMA paced k4 (g-2)");
  run<4>("MMA paced 2 (g-2)");
  return 0;
}
