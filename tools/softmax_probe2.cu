// softmax_probe2.cu -- the d<=128 kernel's per-tile softmax in isolation, as
// the kernel runs it: tcgen05.ld of a 128-column S row block from TMEM, row
// max (FMNMX3 tree), exponentials + row sum + 16-bit pack, two tcgen05.st of
// P halves.  Clocks per tile per warp, 1 or 2 softmax warps per SM
// sub-partition, for exp-loop variants:
//   V0  exp_rowsum_pack as shipped (emu 4/16 spread)
//   V1  same, emu 6/16
//   V2  V0 + a fake dependency (x * runtime zero) of each polynomial pair on
//       the preceding MUFU pair, to make ptxas interleave the FMA-pipe
//       polynomial with the MUFU stream instead of hoisting it
//   V3  V2 + MUFU inputs of the next group depending on the polynomial
//       result (strict alternation)
//   V5  the ping-pong kernel's step verbatim: x128 load, row max + __any_sync
//       rescale vote, two exp_rowsum_pack halves, P stores each followed by
//       wait::st + fence + a per-thread mbarrier arrive (the p_full publish)
//   V4  the d=128 pair kernel's 64-column tile (x64 load, 64 exps, one x32
//       store), 1-4 warps per sub-partition (clk per 64-column tile)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -maxrregcount=168 \
//        -I paper_2312_11918_b200/csrc tools/softmax_probe2.cu -o build/softmax_probe2
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"
#include "softmax_math.cuh"
#include "tmem_ops.cuh"

using namespace fmha_b200;

// V2/V3: groups of 4 pairs, pair 3 of each group on the polynomial.
template <int kOff, bool kChainMufu>
__device__ __forceinline__ float exp_rowsum_pack_il(const float (&s)[128], float c, float neg_mc, uint64_t zero2,
                                                    uint32_t (&p)[32]) {
  const uint64_t c2 = f2_pack(c, c);
  const uint64_t nm2 = f2_pack(neg_mc, neg_mc);
  uint64_t acc0 = f2_pack(0.f, 0.f), acc1 = f2_pack(0.f, 0.f);
  uint64_t prev_poly = f2_pack(0.f, 0.f);
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    uint64_t e[4];
    uint64_t x[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = g * 4 + t;
      x[t] = ffma2(f2_pack(s[kOff + 2 * i], s[kOff + 2 * i + 1]), c2, nm2);
    }
    if (kChainMufu && g > 0) x[0] = ffma2(prev_poly, zero2, x[0]);
    e[0] = exp2_mufu_x2(x[0]);
    e[1] = exp2_mufu_x2(x[1]);
    e[2] = exp2_mufu_x2(x[2]);
    e[3] = exp2_poly_x2(ffma2(e[0], zero2, x[3]));
    prev_poly = e[3];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (t & 1)
        acc1 = fadd2(acc1, e[t]);
      else
        acc0 = fadd2(acc0, e[t]);
      p[g * 4 + t] = pack2_x2<false>(e[t]);
    }
  }
  float a0, a1, b0, b1;
  f2_unpack(acc0, a0, a1);
  f2_unpack(acc1, b0, b1);
  return (a0 + b0) + (a1 + b1);
}

template <int V>
__global__ void __launch_bounds__(V == 4 ? 512 : 256, 1) probe(int iters, float zero, long long* clk, float* sink) {
  __shared__ uint32_t tmem_holder;
  __shared__ uint64_t pbar[2];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&pbar[0], blockDim.x);
    mbar_init(&pbar[1], blockDim.x);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * (V == 4 ? 128 : 256);
  {  // fill S with scores in [-4, 4)
    uint32_t v[32];
    for (int c = 0; c < 4; ++c) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(((threadIdx.x * 37 + c * 32 + i) % 64) * 0.125f - 4.0f);
      tmem_st32x32b_x32(base + c * 32, v);
    }
    tmem_wait_st();
  }
  const uint64_t zero2 = f2_pack(zero, zero);
  float l = 0.f;
  float m_run = -INFINITY;
  long long h0_clk = 0;
  __syncthreads();
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (V == 4) {  // the d=128 pair kernel's 64-column tile
      uint32_t sr[64];
      tmem_ld32x32b_x64(base, sr);
      float s[64];
#pragma unroll
      for (int c = 0; c < 64; ++c) s[c] = __uint_as_float(sr[c]);
      float mx[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mx[t] = fmaxf(s[t], s[t + 8]);
#pragma unroll
      for (int c = 16; c < 64; c += 16)
#pragma unroll
        for (int t = 0; t < 8; ++t) mx[t] = fmaxf(mx[t], fmaxf(s[c + t], s[c + t + 8]));
      const float m = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      uint32_t p0[32];
      l += exp_rowsum_pack<false, 0, 64, 2>(s, 0.1275f, -m * 0.1275f, p0);
      tmem_st32x32b_x32(base + 64, p0);
      tmem_wait_st();
      __syncwarp();
      continue;
    }
    if constexpr (V == 5) {  // the ping-pong kernel's softmax step
      uint32_t sr[128];
      tmem_ld32x32b_x128(base, sr);
      float s[128];
#pragma unroll
      for (int c = 0; c < 128; ++c) s[c] = __uint_as_float(sr[c]);
      float mx[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mx[t] = fmaxf(s[t], s[t + 8]);
#pragma unroll
      for (int c = 16; c < 128; c += 16)
#pragma unroll
        for (int t = 0; t < 8; ++t) mx[t] = fmaxf(mx[t], fmaxf(s[c + t], s[c + t + 8]));
      const float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      const float sl2 = 0.1275f;
      if (__any_sync(0xffffffffu, (mt - m_run) * sl2 > 8.0f)) {
        const float mn = fmaxf(mt, m_run);
        l *= ex2_approx((m_run - mn) * sl2);
        m_run = mn;
      }
      const float neg = -m_run * sl2;
      uint32_t p0[32], p1[32];
      long long t0;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
      float rs = exp_rowsum_pack<false, 0, 64, 4>(s, sl2, neg, p0);
      long long t1;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
      h0_clk += t1 - t0;
      tmem_st32x32b_x32(base + 128, p0);
      rs += exp_rowsum_pack<false, 64, 64, 4>(s, sl2, neg, p1);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&pbar[0]);
      tmem_st32x32b_x32(base + 160, p1);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&pbar[1]);
      l += rs;
      continue;
    }
    uint32_t sr[128];
    tmem_ld32x32b_x128(base, sr);
    float s[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) s[c] = __uint_as_float(sr[c]);
    float mx[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) mx[t] = fmaxf(s[t], s[t + 8]);
#pragma unroll
    for (int c = 16; c < 128; c += 16)
#pragma unroll
      for (int t = 0; t < 8; ++t) mx[t] = fmaxf(mx[t], fmaxf(s[c + t], s[c + t + 8]));
    const float m = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
    const float sl2 = 0.1275f;
    const float neg = -m * sl2;
    uint32_t p0[32], p1[32];
    float rs;
    if constexpr (V == 0) {
      rs = exp_rowsum_pack<false, 0, 64, 4>(s, sl2, neg, p0);
      tmem_st32x32b_x32(base + 128, p0);
      rs += exp_rowsum_pack<false, 64, 64, 4>(s, sl2, neg, p1);
    } else if constexpr (V == 1) {
      rs = exp_rowsum_pack<false, 0, 64, 6>(s, sl2, neg, p0);
      tmem_st32x32b_x32(base + 128, p0);
      rs += exp_rowsum_pack<false, 64, 64, 6>(s, sl2, neg, p1);
    } else {
      rs = exp_rowsum_pack_il<0, V == 3>(s, sl2, neg, zero2, p0);
      tmem_st32x32b_x32(base + 128, p0);
      rs += exp_rowsum_pack_il<64, V == 3>(s, sl2, neg, zero2, p1);
    }
    tmem_wait_st();
    tmem_st32x32b_x32(base + 160, p1);
    tmem_wait_st();
    l += rs;
    __syncwarp();
  }
  const long long c1 = clock64();
  if ((threadIdx.x & 31) == 0) clk[blockIdx.x * 16 + warp] = c1 - c0;
  if (V == 5 && threadIdx.x == 0 && blockIdx.x == 0) printf("V5 exps half 0: %lld clk per tile (warp 0)\n", h0_clk / iters);
  sink[blockIdx.x * blockDim.x + threadIdx.x] = l;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int V>
void run(int threads) {
  long long* clk;
  float* sink;
  cudaMalloc(&clk, 148 * 16 * 8);
  cudaMalloc(&sink, 148 * 512 * 4);
  const int iters = 2000;
  probe<V><<<148, threads>>>(10, 0.f, clk, sink);
  probe<V><<<148, threads>>>(iters, 0.f, clk, sink);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("V%d failed\n", V);
    return;
  }
  long long c[16];
  cudaMemcpy(c, clk, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int w = 0; w < threads / 32; ++w) avg += c[w];
  avg /= threads / 32;
  printf("V%d warps/SMSP %d : %.0f clk per 128-column tile per warp\n", V, threads / 128, avg / iters);
  cudaFree(clk);
  cudaFree(sink);
}

int main() {
  for (int t : {128, 256}) {
    run<0>(t);
    run<1>(t);
    run<2>(t);
    run<3>(t);
    run<4>(t);
    run<5>(t);
  }
  run<4>(384);  // three warps per SMSP
  run<4>(512);
  return 0;
}
