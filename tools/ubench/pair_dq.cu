// Unit check of the pieces a CTA-pair backward needs for its dQ^T product:
//   D[128 x 64] = A[256 x 128]^T * B[256 x 64]  (bf16 in, fp32 out), ONE cta_group::2 MMA chain
//   with M = 128 (64 rows per CTA), N = 64 (32 columns per CTA), K = 256, issued by the leader.
//   * A is MN-major SW128 (K rows of 64 M-elements = 128 B), CTA r holding M rows [64 r, +64);
//   * B is MN-major SW64 (K rows of 32 N-elements = 64 B), CTA r holding N columns [32 r, +32);
//     half of every CTA's B rows are written by the PEER with st.shared::cluster (the dS^T
//     exchange), made visible to the tensor core by fence.proxy.async + a cluster barrier;
//   * the TMEM lanes that hold a CTA's 64 D rows are discovered by dumping all 128 lanes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../../paper_2605_15422_b200/csrc
//        -I../../include pair_dq.cu -o /tmp/pair_dq && /tmp/pair_dq
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
using namespace dkv;

DKV_DEVICE uint64_t sdesc_sw64(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= 4ull << 61;
  return d;
}
DKV_DEVICE uint32_t sw64_offset(uint32_t r, uint32_t c) { return r * 64u + ((c ^ ((r >> 1) & 3u)) << 4); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_dq_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, float* Dout, int variant) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;          // 256 K rows x 128 B = 32 KB
  uint8_t* sB = base + 32768;  // 256 K rows x 64 B = 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const uint32_t rank = cluster_ctarank();
  // A: this CTA's 64 M columns, MN-major (row = k, element = m)
  for (int i = threadIdx.x; i < 256 * 64; i += 128) {
    const int k = i / 64, m = i % 64;
    const uint32_t off = sw128_offset(k, m / 8) + (m % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sA + off) = A[k * 128 + rank * 64 + m];
  }
  fence_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc2<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' smem exists before any remote store
  tc_fence_after();
  // B rows [128 rank, +128): own N half locally, the other half into the peer (thread = K row)
  {
    const int k = rank * 128 + threadIdx.x;
    for (int half = 0; half < 2; ++half) {
      for (int c = 0; c < 4; ++c) {  // four 16 B chunks = 32 bf16 of this row
        uint32_t w[4];
        for (int j = 0; j < 4; ++j) {
          const __nv_bfloat16 lo = B[k * 64 + half * 32 + c * 8 + 2 * j];
          const __nv_bfloat16 hi = B[k * 64 + half * 32 + c * 8 + 2 * j + 1];
          w[j] = static_cast<uint32_t>(__bfloat16_as_ushort(lo)) | (static_cast<uint32_t>(__bfloat16_as_ushort(hi)) << 16);
        }
        const uint32_t off = sw64_offset(k, c);
        if (half == static_cast<int>(rank)) {
          *reinterpret_cast<uint4*>(sB + off) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
          const uint32_t ra = mapa_shared(sB + off, rank ^ 1);
          asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(ra), "r"(w[0]), "r"(w[1]),
                       "r"(w[2]), "r"(w[3])
                       : "memory");
        }
      }
    }
  }
  if (variant == 0)
    asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
  else
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t id = idesc_bf16_f32(128, 64, true, true);
    for (int k = 0; k < 16; ++k)
      mma_ss2(tm, sdesc_sw128(smem_u32(sA) + k * 2048, 0, 1024), sdesc_sw64(smem_u32(sB) + k * 1024, 0, 512), id,
              k > 0);
    mma_commit2_mc(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = threadIdx.x / 32;
  const uint32_t lane_off = static_cast<uint32_t>(w * 32) << 16;
  for (int c0 = 0; c0 < 64; c0 += 32) {
    uint32_t u[32];
    tmem_ld32(tm + lane_off + c0, u);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) Dout[(rank * 128 + threadIdx.x) * 64 + c0 + i] = __uint_as_float(u[i]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (threadIdx.x < 32) tmem_dealloc2<512>(tm);
}

static float bf(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

int main() {
  const int K = 256, M = 128, N = 64;
  std::vector<float> a(K * M), b(K * N), ref(M * N, 0.f);
  srand(3);
  for (auto& x : a) x = bf(rand() / (float)RAND_MAX - 0.5f);
  for (auto& x : b) x = bf(rand() / (float)RAND_MAX - 0.5f);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)a[k * M + m] * b[k * N + n];
      ref[m * N + n] = (float)s;
    }
  std::vector<__nv_bfloat16> ah(a.size()), bh(b.size());
  for (size_t i = 0; i < a.size(); ++i) ah[i] = __float2bfloat16(a[i]);
  for (size_t i = 0; i < b.size(); ++i) bh[i] = __float2bfloat16(b[i]);
  __nv_bfloat16 *ad, *bd;
  float* dd;
  cudaMalloc(&ad, ah.size() * 2);
  cudaMalloc(&bd, bh.size() * 2);
  cudaMalloc(&dd, 2 * 128 * 64 * 4);
  cudaMemcpy(ad, ah.data(), ah.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(bd, bh.data(), bh.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 49152 + 1024;
  cudaFuncSetAttribute(pair_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(dd, 0, 2 * 128 * 64 * 4);
    pair_dq_kernel<<<2, 128, smem>>>(ad, bd, dd, variant);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("kernel error: %s\n", cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> d(2 * 128 * 64);
    cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
    // where does D row m (CTA m / 64, local row i = m % 64) land?  try lane = i and lane = 32 (i/16) + i%16
    for (int hyp = 0; hyp < 3; ++hyp) {
      double maxerr = 0, maxref = 0;
      for (int m = 0; m < M; ++m) {
        const int r = m / 64, i = m % 64;
        for (int n = 0; n < N; ++n) {
          // hyp 2: lane = local row + 64 (n / 32), column n % 32 (N folded onto the upper 64 lanes)
          const int lane = hyp == 0 ? i : hyp == 1 ? 32 * (i / 16) + i % 16 : i + 64 * (n / 32);
          const int col = hyp == 2 ? n % 32 : n;
          maxerr = fmax(maxerr, fabs(d[(r * 128 + lane) * 64 + col] - ref[m * N + n]));
          maxref = fmax(maxref, fabs(ref[m * N + n]));
        }
      }
      printf("variant %d (%s fence): hypothesis %s: max|err| %.3e (max|ref| %.3e) %s\n", variant,
             variant == 0 ? "cluster" : "cta", hyp == 0 ? "lanes 0-63" : hyp == 1 ? "lanes 0-15 of each quadrant" : "lane = row + 64 (n/32), col n%32", maxerr,
             maxref, maxerr < 1e-3 * maxref ? "MATCH" : "no");
    }
    // unused-lane content (diagnostic): max |value| over lanes 64-127 of each CTA
    double other = 0;
    for (int r = 0; r < 2; ++r)
      for (int lane = 64; lane < 128; ++lane)
        for (int n = 0; n < N; ++n) other = fmax(other, fabs(d[(r * 128 + lane) * 64 + n]));
    printf("  max |D| in lanes 64-127 (cols 32-63 checked below): %.3e\n", other);
  }
  return 0;
}
