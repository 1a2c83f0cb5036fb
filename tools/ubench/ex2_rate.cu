// Microbenchmark: exponential throughput per SM -- ex2.approx.f32 (one MUFU op per value) vs
// ex2.approx.f16x2 and ex2.approx.ftz.bf16x2 (two values per instruction).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ex2_rate.cu -o ex2_rate
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void k(int iters, float* out, long long* clk) {
  uint32_t a[8];
  float f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    f[i] = -0.001f * (threadIdx.x + i);
    a[i] = 0xBC00BC00u ^ (threadIdx.x + i);  // small negative halves
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      } else if (MODE == 1) {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
      } else {
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += f[i] + __uint_as_float(a[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&clk, 8);
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int mode = 0; mode < 3; ++mode) {
      if (mode == 0) k<0><<<148, warps * 32>>>(iters, out, clk);
      if (mode == 1) k<1><<<148, warps * 32>>>(iters, out, clk);
      if (mode == 2) k<2><<<148, warps * 32>>>(iters, out, clk);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      const double vals = (double)warps * 32 * iters * 8 * (mode == 0 ? 1 : 2);
      printf("warps %2d %-12s %.1f values/clk/SM\n", warps, mode == 0 ? "f32" : mode == 1 ? "f16x2" : "bf16x2",
             vals / (double)c);
    }
  }
  return 0;
}
