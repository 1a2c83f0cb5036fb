// Microbenchmark: does F2FP (cvt.rn.bf16x2.f32) share the MUFU pipe?  16 warps per SM.
#include "common.cuh"
#include <cstdio>
using namespace dkv;

template <int MODE>
__global__ void k(int iters, uint32_t* out, long long* clk) {
  float a[8];
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      if (MODE == 0 || MODE == 2) { a[i] = ex2(a[i]); a[i + 1] = ex2(a[i + 1]); }
      if (MODE == 1 || MODE == 2) acc ^= pack_bf16(a[i], a[i + 1]);
      if (MODE == 3) acc ^= __byte_perm(__float_as_uint(a[i]) + 0x8000u, __float_as_uint(a[i + 1]) + 0x8000u, 0x7632);
      a[i] -= 1e-7f; a[i + 1] -= 1e-7f;
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(a[0] + a[5]);
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  uint32_t* out; long long* clk; long long h;
  cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&clk, 8);
  const int iters = 4096, thr = 512;
  const char* nm[] = {"ex2 only (8/iter)", "cvt only (4 F2FP/iter)", "ex2 8 + cvt 4 per iter", "int round+PRMT 4/iter"};
  for (int m = 0; m < 4; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) k<0><<<148, thr>>>(iters, out, clk);
      if (m == 1) k<1><<<148, thr>>>(iters, out, clk);
      if (m == 2) k<2><<<148, thr>>>(iters, out, clk);
      if (m == 3) k<3><<<148, thr>>>(iters, out, clk);
    }
    cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    printf("%-26s %.1f clk per iteration per warp-slot (%.2f warp-iter/clk/SM)\n", nm[m], double(h) / iters,
           double(thr / 32) * iters / h);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
