// pipe_probe2.cu -- do MUFU.EX2 and the packed FP32 ops (FFMA2 / FADD2) or
// F2FP overlap within one warp?  Each loop iteration issues 8 independent
// ex2.approx (64 clk of MUFU per warp at 8 clk each) plus K independent
// instructions of one other kind; clk per iteration for 1 warp per SMSP.
// overlap => max(64, K * cost);  no overlap => 64 + K * cost.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//        -I paper_2312_11918_b200/csrc tools/pipe_probe2.cu -o build/pipe_probe2
#include <cuda_runtime.h>

#include <cstdio>

#include "softmax_math.cuh"

using namespace fmha_b200;

// KIND 0: FFMA2, 1: FADD2, 2: F2FP pack, 3: scalar FFMA, 4: FMNMX3
template <int NMUFU, int K, int KIND>
__global__ void __launch_bounds__(128, 1) probe(int iters, float seed, long long* clk, float* sink) {
  float m[8];
  uint64_t a[16];
  uint32_t u[16];
  float f[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) m[i] = seed * (i + 1) * 1e-3f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = f2_pack(seed + i, seed - i);
    u[i] = i;
    f[i] = seed + 0.5f * i;
  }
  const uint64_t c2 = f2_pack(0.999f, 1.001f);
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NMUFU; ++i)  // 8 independent MUFU chains
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(m[i & 7]));
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if constexpr (KIND == 0) a[k & 15] = ffma2(a[k & 15], c2, c2);
      if constexpr (KIND == 1) a[k & 15] = fadd2(a[k & 15], c2);
      if constexpr (KIND == 2) u[k & 15] = pack2<false>(f[k & 15], __uint_as_float(u[k & 15]));
      if constexpr (KIND == 3) f[k & 15] = fmaf(f[k & 15], 0.999f, 0.5f);
      if constexpr (KIND == 4) f[k & 15] = fmaxf(fmaxf(f[k & 15], f[(k + 1) & 15]), f[(k + 2) & 15]);
    }
  }
  const long long c1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += m[i];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    float x, y;
    f2_unpack(a[i], x, y);
    s += x + y + __uint_as_float(u[i]) + f[i];
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
}

template <int NMUFU, int K, int KIND>
void run(const char* name) {
  long long* clk;
  float* sink;
  cudaMalloc(&clk, 148 * 8);
  cudaMalloc(&sink, 148 * 128 * 4);
  const int iters = 4096;
  probe<NMUFU, K, KIND><<<148, 128>>>(16, 0.01f, clk, sink);
  probe<NMUFU, K, KIND><<<148, 128>>>(iters, 0.01f, clk, sink);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  printf("%-8s MUFU x%-2d + %2d others : %6.1f clk/iter\n", name, NMUFU, K, double(c) / iters);
  cudaFree(clk);
  cudaFree(sink);
}

int main() {
  run<8, 0, 0>("none");
  run<0, 16, 0>("FFMA2");
  run<8, 16, 0>("FFMA2");
  run<8, 32, 0>("FFMA2");
  run<0, 16, 1>("FADD2");
  run<8, 16, 1>("FADD2");
  run<0, 16, 2>("F2FP");
  run<8, 16, 2>("F2FP");
  run<0, 16, 3>("FFMA");
  run<8, 16, 3>("FFMA");
  run<8, 32, 3>("FFMA");
  run<0, 16, 4>("FMNMX3");
  run<8, 16, 4>("FMNMX3");
  return 0;
}
