// Unit check of the CTA-pair (cta_group::2) tensor-core mechanics used by a 2-CTA kernel:
//   D[256 x 128] = A[256 x 64] * B[128 x 64]^T (bf16 in, fp32 out), one M=256 N=128 MMA chain
//   issued by the leader CTA; CTA r holds A rows [128 r, +128) and B rows (N) [64 r, +64) in its
//   own shared memory at the same offsets; D rows of CTA r land in ITS tensor memory.
// Also checks the TS form (A from TMEM): D2 = D_bf16 * C^T with C[128 x 128] split by N.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../../paper_2605_15422_b200/csrc
//        -I../../include pair_mma.cu -o /tmp/pair_mma && /tmp/pair_mma
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "tma_host.h"
using namespace dkv;

DKV_DEVICE void alloc2(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "n"(512)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
DKV_DEVICE void dealloc2(uint32_t t) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(t), "n"(512) : "memory");
}
DKV_DEVICE void mma_ss2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
DKV_DEVICE void mma_ts2(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
DKV_DEVICE void commit2_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
DKV_DEVICE uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
DKV_DEVICE void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// K-major SW128 tile: row r (128 B = 64 bf16), element k
DKV_DEVICE void put(uint8_t* tile, int r, int k, __nv_bfloat16 v) {
  const uint32_t off = sw128_offset(r, k / 8) + (k % 8) * 2;
  *reinterpret_cast<__nv_bfloat16*>(tile + off) = v;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, const __nv_bfloat16* C, float* D, float* D2) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;              // 128 x 64 bf16 = 16 KB
  uint8_t* sB = base + 16384;      // 64 x 64 bf16 = 8 KB (this CTA's N half)
  uint8_t* sC = base + 24576;      // C as [N = 128 out cols][K = 128] -> this CTA's 64 N rows, 2 K panels: 16 KB
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const uint32_t rank = ctarank();
  for (int i = threadIdx.x; i < 128 * 64; i += 128) {
    const int r = i / 64, k = i % 64;
    put(sA, r, k, A[(rank * 128 + r) * 64 + k]);
  }
  for (int i = threadIdx.x; i < 64 * 64; i += 128) {
    const int r = i / 64, k = i % 64;
    put(sB, r, k, B[(rank * 64 + r) * 64 + k]);
  }
  for (int i = threadIdx.x; i < 64 * 128; i += 128) {
    const int r = i / 128, k = i % 128;
    put(sC + (k / 64) * 8192, r, k % 64, C[(rank * 64 + r) * 128 + k]);
  }
  fence_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) alloc2(&tbase);
  tc_fence_before();
  __syncthreads();
  csync();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t id = idesc_bf16_f32(256, 128, false, false);
    for (int k = 0; k < 4; ++k)
      mma_ss2(tm, sdesc_sw128(smem_u32(sA) + k * 32, 16, 1024), sdesc_sw128(smem_u32(sB) + k * 32, 16, 1024), id,
              k > 0);
    commit2_mc(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = threadIdx.x / 32;
  const uint32_t lane_off = static_cast<uint32_t>(w * 32) << 16;
  const int row = rank * 128 + threadIdx.x;
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t u[32];
    tmem_ld32(tm + lane_off + c0, u);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) D[row * 128 + c0 + i] = __uint_as_float(u[i]);
    // D as bf16 pairs into TMEM columns [128, 192): the TS operand of the second MMA
    uint32_t pk[16];
    for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(__uint_as_float(u[2 * i]), __uint_as_float(u[2 * i + 1]));
    tmem_st16(tm + lane_off + 128 + c0 / 2, pk);
  }
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  csync();  // both CTAs' bf16 D is in TMEM before the leader issues the TS chain
  tc_fence_after();
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t id = idesc_bf16_f32(256, 128, false, false);
    for (int k = 0; k < 8; ++k)
      mma_ts2(tm + 256, tm + 128 + k * 8, sdesc_sw128(smem_u32(sC) + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024),
              id, k > 0);
    commit2_mc(&bar2);
  }
  mbar_wait(&bar2, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t u[32];
    tmem_ld32(tm + lane_off + 256 + c0, u);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) D2[row * 128 + c0 + i] = __uint_as_float(u[i]);
  }
  tc_fence_before();
  __syncthreads();
  csync();
  if (threadIdx.x < 32) dealloc2(tm);
}


// TMA tile load into THIS CTA's smem whose completion is counted on a barrier in the PEER
// (leader) CTA of the pair: the .cta_group::2 form, `rbar` a shared::cluster address
DKV_DEVICE void tma_load_3d_2sm(void* dst, const CUtensorMap* m, uint32_t rbar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(rbar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
DKV_DEVICE uint32_t mapa0(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}

// Same SS product, B halves loaded by TMA in both CTAs, counted on the leader's barrier.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_tma_kernel(const __grid_constant__ CUtensorMap mb, const __nv_bfloat16* A, float* D) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + 16384;
  __shared__ uint64_t full, done;
  __shared__ uint32_t tbase;
  const uint32_t rank = ctarank();
  for (int i = threadIdx.x; i < 128 * 64; i += 128) {
    const int r = i / 64, k = i % 64;
    put(sA, r, k, A[(rank * 128 + r) * 64 + k]);
  }
  fence_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&full, 1);
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) alloc2(&tbase);
  tc_fence_before();
  __syncthreads();
  csync();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    if (rank == 0) mbar_arrive_expect_tx(&full, 2 * 8192);
    tma_load_3d_2sm(sB, &mb, mapa0(&full), 0, 0, rank * 64);
  }
  if (rank == 0 && threadIdx.x == 0) {
    mbar_wait(&full, 0);
    tc_fence_after();
    const uint32_t id = idesc_bf16_f32(256, 128, false, false);
    for (int k = 0; k < 4; ++k)
      mma_ss2(tm, sdesc_sw128(smem_u32(sA) + k * 32, 16, 1024), sdesc_sw128(smem_u32(sB) + k * 32, 16, 1024), id,
              k > 0);
    commit2_mc(&done);
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  const int w = threadIdx.x / 32;
  const uint32_t lane_off = static_cast<uint32_t>(w * 32) << 16;
  const int row = rank * 128 + threadIdx.x;
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t u[32];
    tmem_ld32(tm + lane_off + c0, u);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) D[row * 128 + c0 + i] = __uint_as_float(u[i]);
  }
  tc_fence_before();
  __syncthreads();
  csync();
  if (threadIdx.x < 32) dealloc2(tm);
}

static float bf(float x) {  // round to bf16 and back
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

int main() {
  const int M = 256, N = 128, K = 64, N2 = 128, K2 = 128;
  std::vector<float> a(M * K), b(N * K), c(N2 * K2);
  srand(1);
  for (auto& x : a) x = bf((rand() / (float)RAND_MAX - 0.5f));
  for (auto& x : b) x = bf((rand() / (float)RAND_MAX - 0.5f));
  for (auto& x : c) x = bf((rand() / (float)RAND_MAX - 0.5f));
  std::vector<__nv_bfloat16> ah(a.size()), bh(b.size()), ch(c.size());
  for (size_t i = 0; i < a.size(); ++i) ah[i] = __float2bfloat16(a[i]);
  for (size_t i = 0; i < b.size(); ++i) bh[i] = __float2bfloat16(b[i]);
  for (size_t i = 0; i < c.size(); ++i) ch[i] = __float2bfloat16(c[i]);
  __nv_bfloat16 *ad, *bd, *cd;
  float *dd, *d2;
  cudaMalloc(&ad, ah.size() * 2);
  cudaMalloc(&bd, bh.size() * 2);
  cudaMalloc(&cd, ch.size() * 2);
  cudaMalloc(&dd, M * N * 4);
  cudaMalloc(&d2, M * N2 * 4);
  cudaMemcpy(ad, ah.data(), ah.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(bd, bh.data(), bh.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(cd, ch.data(), ch.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 24576 + 16384 + 1024;
  cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pair_kernel<<<2, 128, smem>>>(ad, bd, cd, dd, d2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> dh(M * N), d2h(M * N2);
  cudaMemcpy(dh.data(), dd, dh.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(d2h.data(), d2, d2h.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0, err2 = 0, mx = 0, mx2 = 0;
  std::vector<float> ref(M * N);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)a[i * K + k] * b[j * K + k];
      ref[i * N + j] = (float)s;
      err = std::max(err, std::abs(s - dh[i * N + j]));
      mx = std::max(mx, std::abs(s));
    }
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N2; ++j) {
      double s = 0;
      for (int k = 0; k < K2; ++k) s += (double)bf(ref[i * N + k]) * c[j * K2 + k];
      err2 = std::max(err2, std::abs(s - d2h[i * N2 + j]));
      mx2 = std::max(mx2, std::abs(s));
    }
  printf("SS M=256 N=128: max abs err %.3e (max |ref| %.3e)\n", err, mx);
  printf("TS M=256 N=128: max abs err %.3e (max |ref| %.3e)\n", err2, mx2);
  printf("%s\n", (err < 1e-3 * mx + 1e-5 && err2 < 1e-2 * mx2) ? "PAIR OK" : "PAIR MISMATCH");
  // B [128 rows (N), 1, 64 (K)] bf16 -> boxes of 64 rows, SW128
  CUtensorMap mb;
  if (!make_map_3d_bf16(&mb, bd, N, 1, K, 1, 64)) {
    printf("tensor map failed\n");
    return 1;
  }
  cudaMemset(dd, 0, M * N * 4);
  cudaFuncSetAttribute(pair_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pair_tma_kernel<<<2, 128, smem>>>(mb, ad, dd);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("tma kernel error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(dh.data(), dd, dh.size() * 4, cudaMemcpyDeviceToHost);
  double err3 = 0;
  for (int i = 0; i < M * N; ++i) err3 = std::max(err3, (double)std::abs(ref[i] - dh[i]));
  printf("SS with 2-SM TMA B halves: max abs err %.3e -> %s\n", err3, err3 < 1e-3 * mx + 1e-5 ? "PAIR TMA OK" : "PAIR TMA MISMATCH");
  return 0;
}
