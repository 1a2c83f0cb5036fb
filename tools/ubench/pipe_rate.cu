// Microbenchmark: MUFU ex2 and TMEM ld/st throughput per SM (1 CTA/SM, `warps` warps).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2605_15422_b200/csrc pipe_rate.cu -o pipe_rate
#include "common.cuh"
#include <cstdio>
using namespace dkv;

__global__ void k_ex2(int iters, float* out, long long* clk) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ex2(a[i]) - 1.5f;
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

__global__ void k_tmem(int mode, int iters, float* out, long long* clk) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 256;
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x + i;
  float s = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      tmem_ld32(tm + (it & 3) * 32, r);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) s += __uint_as_float(r[i]);
    } else if (mode == 1) {
      tmem_st32(tm + (it & 3) * 32, r);
      tmem_wait_st();
    } else if (mode == 3) {
      uint32_t q[64];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(q[0]),"=r"(q[1]),"=r"(q[2]),"=r"(q[3]),"=r"(q[4]),"=r"(q[5]),"=r"(q[6]),"=r"(q[7]),"=r"(q[8]),"=r"(q[9]),"=r"(q[10]),"=r"(q[11]),"=r"(q[12]),"=r"(q[13]),"=r"(q[14]),"=r"(q[15]),"=r"(q[16]),"=r"(q[17]),"=r"(q[18]),"=r"(q[19]),"=r"(q[20]),"=r"(q[21]),"=r"(q[22]),"=r"(q[23]),"=r"(q[24]),"=r"(q[25]),"=r"(q[26]),"=r"(q[27]),"=r"(q[28]),"=r"(q[29]),"=r"(q[30]),"=r"(q[31]),"=r"(q[32]),"=r"(q[33]),"=r"(q[34]),"=r"(q[35]),"=r"(q[36]),"=r"(q[37]),"=r"(q[38]),"=r"(q[39]),"=r"(q[40]),"=r"(q[41]),"=r"(q[42]),"=r"(q[43]),"=r"(q[44]),"=r"(q[45]),"=r"(q[46]),"=r"(q[47]),"=r"(q[48]),"=r"(q[49]),"=r"(q[50]),"=r"(q[51]),"=r"(q[52]),"=r"(q[53]),"=r"(q[54]),"=r"(q[55]),"=r"(q[56]),"=r"(q[57]),"=r"(q[58]),"=r"(q[59]),"=r"(q[60]),"=r"(q[61]),"=r"(q[62]),"=r"(q[63])
        : "r"(tm + (it & 1) * 64) : "memory");
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 64; ++i) s += __uint_as_float(q[i]);
    } else if (mode == 4) {
      uint32_t q[32], w[32], x[32];
      tmem_ld32(tm + 0, r);
      tmem_ld32(tm + 32, q);
      tmem_ld32(tm + 64, w);
      tmem_ld32(tm + 96, x);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) s += __uint_as_float(r[i]) + __uint_as_float(q[i]) + __uint_as_float(w[i]) + __uint_as_float(x[i]);
    } else {
      uint32_t q[32];
      tmem_ld32(tm + (it & 3) * 32, r);
      tmem_ld32(tm + ((it + 1) & 3) * 32, q);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) s += __uint_as_float(r[i]) + __uint_as_float(q[i]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + r[3];
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&clk, 8);
  long long h;
  for (int warps : {4, 8, 16}) {
    const int iters = 4096;
    k_ex2<<<148, warps * 32>>>(iters, out, clk);
    k_ex2<<<148, warps * 32>>>(iters, out, clk);
    cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    printf("ex2: %2d warps: %.2f ex2/clk/SM\n", warps, double(warps) * 32 * 8 * iters / h);
  }
  const char* nm[] = {"tcgen05.ld 32x32b.x32", "tcgen05.st 32x32b.x32", "2x tcgen05.ld x32 then wait",
                      "tcgen05.ld 32x32b.x64", "4x tcgen05.ld x32 then wait"};
  for (int mode = 0; mode < 5; ++mode)
    for (int warps : {4, 8}) {
      const int iters = 2048;
      k_tmem<<<148, warps * 32>>>(mode, iters, out, clk);
      k_tmem<<<148, warps * 32>>>(mode, iters, out, clk);
      cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
      const int mult = mode == 2 || mode == 3 ? 2 : mode == 4 ? 4 : 1;
      const double bytes = double(warps) * 32 * 32 * 4 * iters * mult;
      printf("%-28s %d warps: %.1f B/clk/SM  (%.0f clk per iteration)\n", nm[mode], warps, bytes / h,
             double(h) / iters);
    }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
