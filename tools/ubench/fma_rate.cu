// Microbenchmark: FFMA vs FFMA2 vs FADD2 vs F2FP vs MUFU throughput per SM (16 warps/SM).
#include "common.cuh"
#include <cstdio>
using namespace dkv;

template <int MODE>
__global__ void k(int iters, float* out, long long* clk) {
  float2 a[8];
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = make_float2(1e-3f * threadIdx.x + i, 2e-3f * i);
  const float2 m = make_float2(0.999f, 0.998f), c = make_float2(1e-6f, 2e-6f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) { a[i].x = fmaf(a[i].x, m.x, c.x); a[i].y = fmaf(a[i].y, m.y, c.y); }   // 2 FFMA
      if (MODE == 1) a[i] = __ffma2_rn(a[i], m, c);                                            // 1 FFMA2
      if (MODE == 2) a[i] = __fadd2_rn(a[i], c);                                               // 1 FADD2
      if (MODE == 3) { acc += pack_bf16(a[i].x, a[i].y); a[i].x += 1e-7f; }                    // F2FP + FADD
      if (MODE == 4) { a[i].x = ex2(a[i].x) - 0.5f; }                                          // MUFU + FADD
      if (MODE == 5) { a[i] = __ffma2_rn(a[i], m, c); a[i].x = ex2(a[i].x); }                 // FFMA2 + MUFU
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  float* out; long long* clk; long long h;
  cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&clk, 8);
  const char* nm[] = {"2 FFMA", "1 FFMA2", "1 FADD2", "F2FP+FADD", "MUFU+FADD", "FFMA2+MUFU"};
  for (int m = 0; m < 6; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      const int iters = 4096, thr = 512;
      if (m == 0) k<0><<<148, thr>>>(iters, out, clk);
      if (m == 1) k<1><<<148, thr>>>(iters, out, clk);
      if (m == 2) k<2><<<148, thr>>>(iters, out, clk);
      if (m == 3) k<3><<<148, thr>>>(iters, out, clk);
      if (m == 4) k<4><<<148, thr>>>(iters, out, clk);
      if (m == 5) k<5><<<148, thr>>>(iters, out, clk);
      cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("%-12s: %.2f clk per (warp-op x 8 ops) per SMSP -> %.2f clk per warp-op per SMSP\n", nm[m],
                      double(h) / iters / 4.0, double(h) / iters / 4.0 / 8.0 * 1.0);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
