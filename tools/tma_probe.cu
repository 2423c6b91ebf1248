// tma_probe.cu -- per-SM TMA streaming rate from L2: one CTA per SM, a 4-slot
// ring of 32 KB (two 16 KB 128x128B SWIZZLE_128B boxes per slot, as the FMHA
// K/V tiles), a producer lane and a consumer warp that frees each slot as
// soon as it lands.  MODE 0: every CTA streams its own 2 MB region; MODE 1:
// groups of G consecutive CTAs stream the same region (the FMHA pattern: the
// CTAs of one head read the same K/V tiles); MODE 2: like 1 with a 2-CTA
// cluster multicasting each box to both CTAs (each issues half the boxes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_2312_11918_b200/csrc \
//        tools/tma_probe.cu -o build/tma_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace fmha_b200;

constexpr int kSlots = 4, kSlotBytes = 32768, kTiles = 64;  // 64 tiles x 32 KB = 2 MB per pass

__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap map, int group, int passes,
                                                long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kSlots], empty[kSlots];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int region = group > 0 ? blockIdx.x / group : blockIdx.x;  // which 2 MB region (row block)
  const long long t0 = clock64();
  const int n = kTiles * passes;
  if (warp == 0) {
    if (lane == 0) {
      for (int t = 0; t < n; ++t) {
        const int s = t % kSlots;
        mbar_wait(&empty[s], ((t / kSlots) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], kSlotBytes);
        const int tile = t % kTiles;
        for (int c = 0; c < 2; ++c)
          tma_load_4d(&map, &full[s], smem + s * kSlotBytes + c * 16384, c * 64, 0, tile * 128, region);
      }
    }
  } else {
    for (int t = 0; t < n; ++t) {
      const int s = t % kSlots;
      mbar_wait(&full[s], (t / kSlots) & 1);
      if (lane == 0) mbar_arrive(&empty[s]);
      __syncwarp();
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  const int regions = 148;
  const size_t rows = kTiles * 128;  // per region: 8192 rows x 256 B = 2 MB
  void* buf;
  cudaMalloc(&buf, regions * rows * 256);
  cudaMemset(buf, 1, regions * rows * 256);
  CUtensorMap map;
  cuuint64_t dims[4] = {128, 1, rows, (cuuint64_t)regions};
  cuuint64_t strides[3] = {256, 256, rows * 256};
  cuuint32_t box[4] = {64, 1, 128, 1}, es[4] = {1, 1, 1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = kSlots * kSlotBytes + 1024;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int group : {0, 16, 148}) {
    const int passes = 8;
    stream<<<148, 64, smem>>>(map, group, 1, d);  // warm L2
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    stream<<<148, 64, smem>>>(map, group, passes, d);
    cudaEventRecord(b);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      printf("failed\n");
      return 1;
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> h(148);
    cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto x : h) avg += x;
    avg /= 148;
    const double bytes = 148.0 * kTiles * passes * kSlotBytes;
    printf("group %3d (CTAs sharing a region): %.1f B/clk per SM, chip %.2f TB/s (%.3f ms)\n", group,
           kTiles * passes * kSlotBytes / avg, bytes / (ms * 1e-3) / 1e12, ms);
  }
  return 0;
}
