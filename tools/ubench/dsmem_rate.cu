// Microbenchmark: distributed shared memory write bandwidth inside a 2-CTA cluster on B200.
// CTA 1 pushes a 32 KB fp32 tile into CTA 0's shared memory (a) with st.shared::cluster.v4 from
// 128 threads, (b) with one cp.async.bulk.shared::cluster.shared::cta (mbarrier completion), then
// signals CTA 0; clocks per 32 KB tile over many repetitions.  148 clusters... (74 pairs).
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank)); return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) k(int reps, long long* clk) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* src = sm;            // 32 KB local tile
  uint8_t* dst = sm + 32768;    // 32 KB landing zone (written by the peer)
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = ctarank();
  for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(src)[i] = make_uint4(i, 1, 2, 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  cluster_sync();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (rank == 1) {
      if (MODE == 0) {
        const uint32_t rdst = mapa(dst, 0);
        for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) {
          uint4 v = reinterpret_cast<const uint4*>(src)[i];
          asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(rdst + i * 16), "r"(v.x), "r"(v.y),
                       "r"(v.z), "r"(v.w) : "memory");
        }
      } else if (threadIdx.x == 0) {
        // bulk copy local smem -> peer smem, completion as tx bytes on the PEER's barrier
        const uint32_t rbar = mapa(&bar, 0);
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(mapa(dst, 0)), "r"(smem_u32(src)), "r"(32768), "r"(rbar) : "memory");
      }
    } else if (MODE == 1 && threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(32768) : "memory");
      uint32_t ok = 0;
      while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                               : "=r"(ok) : "r"(smem_u32(&bar)), "r"(r & 1) : "memory");
    }
    cluster_sync();  // tile delivered (MODE 0: st.shared::cluster visible after the release/acquire barrier)
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  long long* clk; long long h;
  cudaMalloc(&clk, 8);
  const int reps = 2000;
  for (int m = 0; m < 2; ++m) {
    auto fn = m == 0 ? k<0> : k<1>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    for (int rep = 0; rep < 2; ++rep) fn<<<148, 128, 65536 + 1024>>>(reps, clk);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    printf("%s: %.0f clk per 32 KB tile (incl. a cluster barrier) = %.1f B/clk  [%s]\n",
           m == 0 ? "st.shared::cluster.v4 x 128 thr" : "cp.async.bulk smem->peer smem ", double(h) / reps,
           32768.0 * reps / double(h), cudaGetErrorString(e));
  }
  // cluster barrier alone
  return 0;
}
