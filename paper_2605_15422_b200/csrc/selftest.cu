// selftest.cu -- one-CTA check of every UMMA operand form the attention kernels
// use (K-major / MN-major smem descriptors, A from TMEM, N = 128 / 64), with
// operands staged by the same SWIZZLE_128B TMA boxes.  A debug aid exported
// through the C ABI; tests/test_gpu_selftest.py compares against torch.
//
// Inputs are row-major bf16 matrices as stored in global memory:
//   mode 0: A[M=128][K=128], B[N=128][K=128]        D = A B^T   (K-major / K-major)
//   mode 1: A[M][K],         B[K=128][N=128]        D = A B     (K-major / MN-major)
//   mode 2: A[M][K] via TMEM, B[N][K]               D = A B^T   (TS,      K-major)
//   mode 3: A[K=128][M=128], B[N][K]                D = A^T B^T (MN-major / K-major)
//   mode 4: A[M][K] via TMEM, B[K][N]               D = A B     (TS,      MN-major)
//   mode 5: A[M][K],         B[N=64][K]             D = A B^T   (N = 64)
//   mode 6: A[K][M],         B[K][N=64]             D = A^T B   (MN-major / MN-major, N = 64)
//   mode 7: A[M][K=64],      B[K=64][N=128]         D = A B     (K = 64, MN-major B)
#include "dkv_internal.h"
#include "tma_host.h"

namespace dkv {

struct SelftestParams {
  CUtensorMap ta, tb;
  const __nv_bfloat16* a;
  float* d;
  int mode, n, k, a_rows, b_rows;
};

__global__ void __launch_bounds__(128, 1) selftest_kernel(const __grid_constant__ SelftestParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + 32768;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + 65536);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(base + 65536 + 64);
  const int warp = warp_id();
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;
  const int a_panels = (p.mode == 3 || p.mode == 6) ? 2 : p.k / 64;  // A stored [K][M]: 2 panels of M
  const int b_cols = (p.mode == 1 || p.mode == 4 || p.mode == 6 || p.mode == 7) ? p.n : p.k;
  const int b_panels = b_cols / 64;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bars[0], (a_panels * p.a_rows + b_panels * p.b_rows) * 128);
    for (int pn = 0; pn < a_panels; ++pn) tma_load_3d(sA + pn * p.a_rows * 128, &p.ta, &bars[0], pn * 64, 0, 0);
    for (int pn = 0; pn < b_panels; ++pn) tma_load_3d(sB + pn * p.b_rows * 128, &p.tb, &bars[0], pn * 64, 0, 0);
  }
  mbar_wait(&bars[0], 0);
  const bool a_tmem = p.mode == 2 || p.mode == 4;
  if (a_tmem) {
    // thread m packs row m of A into TMEM columns [256, 256 + K/2)
    const int m = threadIdx.x;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    for (int c0 = 0; c0 < p.k; c0 += 32) {
      uint32_t r[16];
      for (int i = 0; i < 16; ++i) {
        const float lo = __bfloat162float(p.a[m * p.k + c0 + 2 * i]);
        const float hi = __bfloat162float(p.a[m * p.k + c0 + 2 * i + 1]);
        r[i] = pack_bf16(lo, hi);
      }
      tmem_st16(tmem + lane_off + 256 + c0 / 2, r);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    const bool a_mn = p.mode == 3 || p.mode == 6;
    const bool b_mn = p.mode == 1 || p.mode == 4 || p.mode == 6 || p.mode == 7;
    const uint32_t idesc = idesc_bf16_f32(128, p.n, a_mn, b_mn);
    for (int k = 0; k < p.k / 16; ++k) {
      uint64_t bd;
      if (b_mn)
        bd = sdesc_sw128(b0 + k * 2048, p.b_rows * 128, 1024);
      else
        bd = sdesc_sw128(b0 + (k >> 2) * p.b_rows * 128 + (k & 3) * 32, 16, 1024);
      if (a_tmem) {
        mma_ts(tmem, tmem + 256 + k * 8, bd, idesc, k > 0);
      } else {
        uint64_t ad;
        if (a_mn)
          ad = sdesc_sw128(a0 + k * 2048, p.a_rows * 128, 1024);
        else
          ad = sdesc_sw128(a0 + (k >> 2) * p.a_rows * 128 + (k & 3) * 32, 16, 1024);
        mma_ss(tmem, ad, bd, idesc, k > 0);
      }
    }
    mma_commit(&bars[1]);
  }
  mbar_wait(&bars[1], 0);
  tc_fence_after();
  {
    const int m = threadIdx.x;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    for (int c0 = 0; c0 < p.n; c0 += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + c0, r);
      tmem_wait_ld();
      for (int i = 0; i < 32; ++i) p.d[m * p.n + c0 + i] = __uint_as_float(r[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace dkv

using namespace dkv;

extern "C" int32_t dkv_selftest_umma(int32_t mode, const void* a, const void* b, float* d, void* stream) {
  if (mode < 0 || mode > 7 || !a || !b || !d) {
    set_error("dkv_selftest_umma: bad arguments");
    return DKV_ERR_INVALID;
  }
  SelftestParams p{};
  p.mode = mode;
  p.n = (mode == 5 || mode == 6) ? 64 : 128;
  p.k = mode == 7 ? 64 : 128;
  p.a = static_cast<const __nv_bfloat16*>(a);
  p.d = d;
  // global shapes (rows, cols) as stored
  int a_r = 128, a_c = p.k;                                  // A[M][K]
  if (mode == 3 || mode == 6) { a_r = 128; a_c = 128; }      // A[K][M]
  int b_r, b_c;
  if (mode == 1 || mode == 4 || mode == 6 || mode == 7) { b_r = p.k; b_c = p.n; }  // B[K][N]
  else { b_r = p.n; b_c = p.k; }                                                 // B[N][K]
  p.a_rows = a_r;
  p.b_rows = b_r;
  if (!make_map_3d_bf16(&p.ta, a, a_r, 1, a_c, 1, a_r) || !make_map_3d_bf16(&p.tb, b, b_r, 1, b_c, 1, b_r)) {
    set_error("dkv_selftest_umma: tensor map encode failed");
    return DKV_ERR_CUDA;
  }
  const int smem = 65536 + 1024 + 1024;
  cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  selftest_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("dkv_selftest_umma: ") + cudaGetErrorString(e));
    return DKV_ERR_CUDA;
  }
  return DKV_OK;
}
