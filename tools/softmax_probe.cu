// softmax_probe.cu -- microbenchmark of the per-row softmax math
// (softmax_math.cuh): clocks per 128-score row (row max + exponentials +
// row sum + 16-bit pack) for a given exp2 split and instruction schedule,
// with 1 or 2 warps per SM sub-partition (the FMHA kernel runs two softmax
// warps per SMSP).  Build (register cap as in the kernel's softmax region):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -maxrregcount=192 \
//        -I paper_2312_11918_b200/csrc tools/softmax_probe.cu -o build/softmax_probe
#include <cuda_runtime.h>

#include <cstdio>

#include "softmax_math.cuh"

using namespace fmha_b200;

template <int EMU, int BATCH>
__global__ void __launch_bounds__(256, 1) probe(const float* in, uint32_t* out, int iters, long long* clk) {
  float s[128];
#pragma unroll
  for (int c = 0; c < 128; ++c) s[c] = in[(threadIdx.x * 7 + c) & 1023];
  uint32_t acc = 0;
  float sum = 0.f;
  __syncthreads();
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float mx[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) mx[t] = fmaxf(s[t], s[t + 8]);
#pragma unroll
    for (int c = 16; c < 128; c += 16)
#pragma unroll
      for (int t = 0; t < 8; ++t) mx[t] = fmaxf(mx[t], fmaxf(s[c + t], s[c + t + 8]));
    const float m = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
    uint32_t p[32];
    if (BATCH == 1)
      sum += exp_rowsum_pack<false, 0, 64, EMU>(s, 1.4426950f, -m, p);
    else
      sum += exp_rowsum_pack<false, 0, 64, EMU>(s, 1.4426950f, -m, p);
#pragma unroll
    for (int i = 0; i < 32; ++i) acc ^= p[i];
    if (BATCH == 1)
      sum += exp_rowsum_pack<false, 64, 64, EMU>(s, 1.4426950f, -m, p);
    else
      sum += exp_rowsum_pack<false, 64, 64, EMU>(s, 1.4426950f, -m, p);
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += p[i];
#pragma unroll
    for (int c = 0; c < 128; ++c) s[c] += 1e-7f * float(acc & 1);  // keep s live and changing
  }
  const long long c1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(sum);
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
}

template <int EMU, int BATCH>
void run(int threads) {
  float* in;
  uint32_t* out;
  long long* clk;
  cudaMalloc(&in, 4096);
  cudaMalloc(&out, 148 * 256 * 4);
  cudaMalloc(&clk, 148 * 8);
  cudaMemset(in, 0, 4096);
  const int iters = 2000;
  probe<EMU, BATCH><<<148, threads>>>(in, out, 10, clk);
  probe<EMU, BATCH><<<148, threads>>>(in, out, iters, clk);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  printf("emu %2d/16 batch %2d warps/SMSP %d : %.0f clk per 128-score row (max+exp+sum+pack)\n", EMU, BATCH,
         threads / 128, double(c) / iters);
}

int main() {
  for (int t : {128, 256}) {
    run<0, 1>(t);
    run<0, 4>(t);
    run<0, 8>(t);
    run<0, 16>(t);
    run<4, 1>(t);
    run<4, 8>(t);
    run<4, 16>(t);
  }
  return 0;
}
