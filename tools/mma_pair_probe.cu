// mma_pair_probe.cu -- tcgen05.mma.cta_group::2 throughput (M = 256 over a
// CTA pair) for the d = 256 pair kernel's shapes: SS M256 N128 K16 (S = Q K^T)
// and TS M256 N256 K16 with B MN-major (O += P V).  Cluster (2,1,1), one CTA
// per SM, the leader's thread 0 issues iters x 16 MMAs back to back.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//        -I paper_2312_11918_b200/csrc tools/mma_pair_probe.cu -o build/mma_pair_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"
#include "sm100_pair.cuh"

using namespace fmha_b200;

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* out_clk) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_holder;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc_pair(&tmem_holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  if (cluster_ctarank() == 0 && threadIdx.x < 32) {
    const uint32_t a = smem_u32(smem), bb = smem_u32(smem + 32768);
    constexpr uint32_t idesc_k = idesc_f16(false, 256, 128, false, false);
    constexpr uint32_t idesc_mn = idesc_f16(false, 256, 256, false, true);
    const unsigned long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        if (MODE == 0)
          mma_pair_ss_elect(tmem, sdesc_sw128(a + (kk & 3) * 32, 16, 1024),
                            sdesc_sw128(bb + (kk & 3) * 32, 16, 1024), idesc_k, 1);
        else
          mma_pair_ts_elect(tmem, tmem + 256 + (kk & 7) * 8, sdesc_sw128(bb + (kk & 7) * 2048, 128 * 128, 1024),
                            idesc_mn, 1);
      }
    }
    mma_commit_pair_elect(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long c1 = clock64();
    if (threadIdx.x == 0) out_clk[blockIdx.x / 2] = c1 - c0;
  } else if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc_pair(tmem, 512);
}

template <int MODE>
void run(const char* name, int clusters) {
  const int iters = 2000;
  unsigned long long* dc;
  cudaMalloc(&dc, clusters * 8);
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 100 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, probe<MODE>, 10, dc);
  cudaLaunchKernelEx(&cfg, probe<MODE>, iters, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  std::vector<unsigned long long> c(clusters);
  cudaMemcpy(c.data(), dc, clusters * 8, cudaMemcpyDeviceToHost);
  double cs = 0;
  for (int i = 0; i < clusters; ++i) cs += c[i];
  cs /= clusters;
  const int n = MODE == 0 ? 128 : 256;
  printf("%-30s clusters=%2d  %.1f clk/MMA  (ideal per SM %d)\n", name, clusters, cs / (16.0 * iters), 128 * n / 256);
  cudaFree(dc);
}

int main() {
  for (int cl : {1, 74}) {
    run<0>("pair SS M256 N128 K16", cl);
    run<1>("pair TS M256 N256 K16 (B MN)", cl);
  }
  return 0;
}
