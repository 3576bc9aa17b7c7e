// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM vs number of warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2510_15964_b200/csrc tmem_bw.cu -o tmem_bw
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace lx;

template <int NW>
__global__ void __launch_bounds__(32 * NW, 1) k_tmem(int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  uint32_t acc = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[4][32];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(base + ((c * 32 + i) & 127), r[c]);
    tmem_ld_wait();
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= r[c][j];
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(slot); }
}

template <int NW>
void run(int iters) {
  unsigned long long* d; uint32_t* s;
  cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 4);
  k_tmem<NW><<<148, 32 * NW>>>(iters, d, s);
  k_tmem<NW><<<148, 32 * NW>>>(iters, d, s);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double bytes = (double)iters * NW * 32 * 128 * 4;  // per CTA (= per SM)
  printf("warps %2d: %.1f B/clk per SM (%llu cycles, err=%s)\n", NW, bytes / h[0], h[0], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<4>(2000);
  run<8>(2000);
  run<16>(1000);
  return 0;
}
