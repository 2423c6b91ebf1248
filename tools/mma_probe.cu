// mma_probe.cu -- microbenchmark: tcgen05.mma throughput per SM for the
// operand modes / shapes the FMHA kernels use (SS = both operands in shared
// memory, TS = A in Tensor Memory).  One CTA per SM, one thread issues
// `iters` x 16 MMAs back to back on fixed operands, then commits.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//        -I paper_2312_11918_b200/csrc tools/mma_probe.cu -o build/mma_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace fmha_b200;

template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* out_clk,
                                                unsigned long long* out_ns) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_holder;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&tmem_holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), bb = smem_u32(smem + 32768);
    constexpr uint32_t idesc_k = idesc_f16(false, 128, N, false, false);
    constexpr uint32_t idesc_mn = idesc_f16(false, 128, N, false, true);
    const unsigned long long c0 = clock64();
    const uint64_t t0 = globaltimer_ns();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        if (MODE == 0) {  // SS, both K-major SW128
          mma_ss(tmem, sdesc_sw128(a + (kk & 3) * 32, 16, 1024), sdesc_sw128(bb + (kk & 3) * 32, 16, 1024),
                 idesc_k, 1);
        } else {  // TS: A from TMEM columns [256, 256+8*...), B MN-major (V-like)
          mma_ts(tmem, tmem + 256 + (kk & 7) * 8, sdesc_sw128(bb + (kk & 7) * 2048, N * 128 / 2, 1024), idesc_mn, 1);
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long c1 = clock64();
    const uint64_t t1 = globaltimer_ns();
    out_clk[blockIdx.x] = c1 - c0;
    out_ns[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int MODE, int N>
void run(const char* name, int ctas) {
  const int iters = 2000;
  unsigned long long *dc, *dn;
  cudaMalloc(&dc, ctas * 8);
  cudaMalloc(&dn, ctas * 8);
  cudaFuncSetAttribute(probe<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  probe<MODE, N><<<ctas, 128, 100 * 1024>>>(10, dc, dn);
  probe<MODE, N><<<ctas, 128, 100 * 1024>>>(iters, dc, dn);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  std::vector<unsigned long long> c(ctas), n(ctas);
  cudaMemcpy(c.data(), dc, ctas * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(n.data(), dn, ctas * 8, cudaMemcpyDeviceToHost);
  double cs = 0, ns = 0;
  for (int i = 0; i < ctas; ++i) {
    cs += c[i];
    ns += n[i];
  }
  cs /= ctas;
  ns /= ctas;
  const double mmas = 16.0 * iters;
  const double flop = 2.0 * 128 * N * 16 * mmas * ctas;
  printf("%-28s ctas=%3d  %.1f clk/MMA  (ideal %d)  %.0f TFLOP/s  clk %.0f MHz\n", name, ctas, cs / mmas,
         128 * N / 256, flop / (ns * 1e-9) / 1e12, cs / ns * 1e3);
  cudaFree(dc);
  cudaFree(dn);
}

int main() {
  for (int ctas : {1, 148}) {
    run<0, 128>("SS M128 N128 K16", ctas);
    run<1, 128>("TS M128 N128 K16 (B MN)", ctas);
    run<0, 256>("SS M128 N256 K16", ctas);
    run<1, 256>("TS M128 N256 K16 (B MN)", ctas);
    run<0, 64>("SS M128 N64 K16", ctas);
  }
  return 0;
}
