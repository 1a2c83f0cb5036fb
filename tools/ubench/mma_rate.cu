// Microbenchmark: tcgen05.mma throughput vs operand source (SS/TS), swizzle mode and N.
// One CTA per SM; one elected thread issues `iters` M=128 K=16 bf16 MMAs into TMEM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2605_15422_b200/csrc mma_rate.cu -o mma_rate
#include "common.cuh"
#include <cstdio>
using namespace dkv;

// K-major descriptor for swizzle `sw` bytes (128/64/32): rows of sw bytes, 8-row atoms
__device__ uint64_t kdesc(uint32_t saddr, int sw) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>((8 * sw) >> 4) << 32;
  d |= 1ull << 46;
  const uint64_t lay = sw == 128 ? 2 : sw == 64 ? 4 : 6;
  d |= lay << 61;
  return d;
}

struct Cfg { int ts, n, sw_a, sw_b, b_mn, a_mn; };

__global__ void __launch_bounds__(128, 1) k_rate(Cfg c, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 192 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  fence_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x < 32 && elect_one()) {
    const uint32_t a = smem_u32(base), b = smem_u32(base + 65536);
    const uint32_t id = idesc_bf16_f32(128, c.n, c.a_mn != 0, c.b_mn != 0);
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int kpa = c.sw_a / 32, kpb = c.sw_b / 32;  // K steps per swizzle row
      const uint32_t aoff = c.ts ? 0 : (k / kpa) * (128 * c.sw_a) + (k % kpa) * 32;
      ad[k] = c.ts ? 0 : c.a_mn ? sdesc_sw128(a + k * 2048, 16384, 1024) : kdesc(a + aoff, c.sw_a);
      if (c.b_mn) {
        bd[k] = sdesc_sw128(b + k * 2048, 64 * 128 * 2 /*LBO: next 64-wide MN atom*/, 1024);
      } else {
        const uint32_t boff = (k / kpb) * (c.n * c.sw_b) + (k % kpb) * 32;
        bd[k] = kdesc(b + boff, c.sw_b);
      }
    }
    long long t0 = clock64();
    if (c.ts) {
      for (int i = 0; i < iters; i += 8)
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_ts(tmem + 256, tmem + (k & 3) * 8, bd[k], id, 1u);
    } else {
      for (int i = 0; i < iters; i += 8)
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_ss(tmem, ad[k], bd[k], id, 1u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  Cfg cfgs[] = {
    {0, 128, 128, 128, 0, 0}, {0, 128, 128, 128, 1, 0}, {0, 128, 128, 128, 1, 1}, {0, 128, 128, 128, 0, 1},
    {0, 64, 128, 128, 1, 1}, {1, 128, 0, 128, 1, 0}, {1, 128, 0, 128, 0, 0}, {0, 128, 32, 32, 0, 0},
  };
  for (auto c : cfgs) {
    float best = 1e9; unsigned long long clk = 0;
    for (int rep = 0; rep < 3; ++rep) {
      const int iters = 8192;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k_rate<<<148, 128, 200 * 1024>>>(c, iters, d);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(&clk, d, 8, cudaMemcpyDeviceToHost);
      if (ms < best) best = ms;
    }
    double flop = 2.0 * 128 * c.n * 16 * 8192 * 148;
    printf("%s N%-3d A%s:%s B:%s%-4s clk/mma %6.1f ideal %3d  %5.0f TFLOP/s\n", c.ts ? "TS" : "SS", c.n,
           c.a_mn ? "(MN)" : "", c.ts ? "tmem " : (c.sw_a == 128 ? "sw128" : c.sw_a == 64 ? "sw64 " : "sw32 "),
           c.sw_b == 128 ? "sw128" : c.sw_b == 64 ? "sw64 " : "sw32 ", c.b_mn ? "(MN)" : "", (double)clk / 8192,
           128 * c.n / 256, flop / (best * 1e-3) / 1e12);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
