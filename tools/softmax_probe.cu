// softmax_probe.cu -- microbenchmark of the per-row softmax math
// (softmax_math.cuh): clocks per 128-score row for a given exp2 split, with
// 1 or 2 warps per SM sub-partition (the FMHA kernel runs two softmax warps
// per SMSP).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//        -I paper_2312_11918_b200/csrc tools/softmax_probe.cu -o build/softmax_probe
#include <cuda_runtime.h>

#include <cstdio>

#include "softmax_math.cuh"

using namespace fmha_b200;

template <int EMU>
__global__ void __launch_bounds__(256, 1) probe(const float* in, uint32_t* out, int iters, long long* clk) {
  float s[128];
#pragma unroll
  for (int c = 0; c < 128; ++c) s[c] = in[(threadIdx.x * 7 + c) & 1023];
  uint32_t acc = 0;
  float sum = 0.f;
  __syncthreads();
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t p[32];
    sum += exp_rowsum_pack<false, 0, 64, EMU>(s, 1.4426950f, -float(it & 7), p);
#pragma unroll
    for (int i = 0; i < 32; ++i) acc ^= p[i];
    sum += exp_rowsum_pack<false, 64, 64, EMU>(s, 1.4426950f, -float(it & 7), p);
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += p[i];
  }
  const long long c1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(sum);
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
}

template <int EMU>
void run(int threads) {
  float* in;
  uint32_t* out;
  long long* clk;
  cudaMalloc(&in, 4096);
  cudaMalloc(&out, 148 * 256 * 4);
  cudaMalloc(&clk, 148 * 8);
  cudaMemset(in, 0, 4096);
  const int iters = 2000;
  probe<EMU><<<148, threads>>>(in, out, 10, clk);
  probe<EMU><<<148, threads>>>(in, out, iters, clk);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  printf("emu %2d/16  warps/SMSP %d : %.0f clk per 128-score row per warp-iteration\n", EMU, threads / 128,
         double(c) / iters);
}

int main() {
  for (int t : {128, 256}) {
    run<0>(t);
    run<4>(t);
    run<6>(t);
    run<8>(t);
    run<16>(t);
  }
  return 0;
}
