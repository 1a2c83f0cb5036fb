// Microbenchmark: TMA bulk tensor reduce-add (fp32) throughput from smem to global.
// One CTA per SM, one thread issues `iters` reduce ops of a [rows][128] fp32 box; `share` CTAs
// target the same global region (1 = disjoint).  Prints B/clk/SM and chip-wide GB/s.
#include "common.cuh"
#include "tma_host.h"
#include <cstdio>
using namespace dkv;

__global__ void k_red(const __grid_constant__ CUtensorMap m, int rows, int iters, int share, int inflight,
                      long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* s = reinterpret_cast<float*>(smem);
  for (int i = threadIdx.x; i < rows * 128; i += blockDim.x) s[i] = 1.f;
  fence_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int region = blockIdx.x / share;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      asm volatile(
          "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
              reinterpret_cast<uint64_t>(&m)),
          "r"(smem_u32(s)), "r"(0), "r"(region * 1024 + (it % 8) * rows)
          : "memory");
      bulk_commit();
      if (inflight == 1) bulk_wait_read<0>();
      else if (inflight == 2) bulk_wait_read<1>();
      else bulk_wait_read<3>();
    }
    bulk_wait<0>();
    long long t1 = clock64();
    if (blockIdx.x == 0) *clk = t1 - t0;
  }
}

int main() {
  const int64_t total_rows = 148 * 1024;
  float* g;
  cudaMalloc(&g, total_rows * 128 * 4);
  cudaMemset(g, 0, total_rows * 128 * 4);
  long long* clk;
  cudaMalloc(&clk, 8);
  cudaFuncSetAttribute(k_red, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int rows : {4, 16, 64}) {
    CUtensorMap m;
    // 2-D [total_rows][128] fp32, box (128, rows)
    EncodeTiledFn fn = encode_tiled_fn();
    cuuint64_t gdim[2] = {128, (cuuint64_t)total_rows};
    cuuint64_t gstr[1] = {128 * 4};
    cuuint32_t box[2] = {128, (cuuint32_t)rows};
    cuuint32_t es[2] = {1, 1};
    fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int share : {1, 16}) {
      for (int inflight : {1, 2, 4}) {
        const int iters = 2048 * 16 / rows;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        k_red<<<148, 128, 64 * 1024>>>(m, rows, 64, share, inflight, clk);
        cudaEventRecord(e0);
        k_red<<<148, 128, 64 * 1024>>>(m, rows, iters, share, inflight, clk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long h;
        cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
        const double bytes = double(rows) * 512 * iters;
        printf("box %2d rows (%5d B) share %2d inflight %d: %6.1f B/clk/SM, chip %7.1f GB/s\n", rows, rows * 512,
               share, inflight, bytes / h, bytes * 148 / (ms * 1e-3) / 1e9);
      }
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
