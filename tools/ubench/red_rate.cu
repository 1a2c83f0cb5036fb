// Microbenchmark: LSU fp32 reductions to global (red.global.add.f32 / .v4.f32), coalesced per warp.
#include "common.cuh"
#include <cstdio>
using namespace dkv;

template <int V>
__global__ void k_red(float* g, int iters, long long* clk) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* base = g + (static_cast<int64_t>(blockIdx.x) * 64 + warp) * 4096;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float* p = base + (it & 7) * 128 * V / 4 * 4 + lane * V;
    if (V == 4)
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(2.f), "f"(3.f), "f"(4.f)
                   : "memory");
    else
      asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(1.f) : "memory");
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  float* g;
  cudaMalloc(&g, 148ll * 64 * 4096 * 4);
  long long* clk;
  cudaMalloc(&clk, 8);
  for (int ctas : {148, 74, 37}) {
  for (int warps : {16}) {
    for (int v : {4}) {
      const int iters = 4096;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      if (v == 4) k_red<4><<<ctas, warps * 32>>>(g, 64, clk); else k_red<1><<<ctas, warps * 32>>>(g, 64, clk);
      cudaEventRecord(e0);
      if (v == 4) k_red<4><<<ctas, warps * 32>>>(g, iters, clk); else k_red<1><<<ctas, warps * 32>>>(g, iters, clk);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      long long h;
      cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
      const double bytes = double(warps) * 32 * 4 * v * iters;
      printf("ctas %3d red.global.add%s %2d warps: %6.1f B/clk/SM (%.2f warp-instr/clk), chip %7.1f GB/s\n",
             ctas, v == 4 ? ".v4.f32" : ".f32   ", warps, bytes / h, double(warps) * iters / h,
             bytes * ctas / (ms * 1e-3) / 1e9);
    }
  }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
