// qkv_prep.cu -- the step between the QKV projection GEMM and the DualKV op, fused into one HBM
// pass per direction (reference layer.py:182-205 RoPE, positions packing.py:105-120;
// the per-head q/k RMSNorm is Qwen3's, SPEC.md:464 -- the reference toy model has none):
//
//   forward : qkv [T, H + 2 H_k, d] (the GEMM output of the P+NR rows, packed-row order)
//             -> per q / k head: y = x * rsqrt(mean(x^2) + eps) * w   (fp32, skipped without w)
//             -> RoPE at the row's LOGICAL position (angles in fp64 as in rope_rows_kernel)
//             -> written ONCE, rounded to bf16, at row dst[r] of q [T, H, d], k / v [T, H_k, d]
//                (dst = the split layout [all prompts ; all responses] a multi-group launch takes)
//   backward: dq / dk / dv rows gathered from dst[r] -> inverse rotation -> RMSNorm adjoint
//             dx = rstd (w g) - x rstd^3 mean(x w g) -> dqkv [T, H + 2 H_k, d]; the norm weights'
//             gradient sum_rows g x_hat accumulates in registers of a persistent grid and leaves
//             with one fp32 atomic per element per CTA.
//
// Layout per thread: 16-byte vectors (8 bf16); a head (d = 128) is 16 consecutive threads, so the
// head's sum of squares is a 16-lane shuffle reduction.  HBM-bound: 2 x 12 KB per row at Qwen3-8B.
#include "dkv_internal.h"

#include <type_traits>

#include <cmath>

namespace dkv {

namespace {

struct PrepArgs {
  const __nv_bfloat16* qkv;  // [T][HT][D]
  const __nv_bfloat16* wq;   // [D] or null (no norm)
  const __nv_bfloat16* wk;
  const int64_t* pos;        // [T]
  const int64_t* dst;        // [T]
  __nv_bfloat16* q;          // [T][H][D]   (forward outputs / backward inputs)
  __nv_bfloat16* k;          // [T][Hk][D]
  __nv_bfloat16* v;
  __nv_bfloat16* dqkv;       // backward output [T][HT][D]
  float* dwq;                // backward: [D] fp32 accumulators (pre-zeroed)
  float* dwk;
  int64_t rows;
  int heads, kv_heads, head_dim;
  float eps;
  double log2_base;
};

constexpr int kThreads = 256;

DKV_DEVICE void unpack8(const uint4& v, float (&f)[8]) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    f[2 * j] = __uint_as_float(w[j] << 16);
    f[2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
  }
}
DKV_DEVICE uint4 pack8(const float (&f)[8]) {
  uint4 v;
  uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
  for (int j = 0; j < 4; ++j) w[j] = pack_bf16(f[2 * j], f[2 * j + 1]);
  return v;
}

// A thread's vectors all start at the same rotation pair (kThreads is a multiple of VPH, so the
// d-slice of vector i0 + threadIdx.x is fixed): the 4 pair frequencies once per thread, their
// (cos, sin) once per row in registers -- the double-precision angle reduction of rope_rows_kernel
// (aux.cu), without a shared per-row table and the two block barriers per row it needed.
struct ThreadPairs {
  double inv_freq[4];
  __device__ void init(int k0, int head_dim, double log2_base) {
#pragma unroll
    for (int j = 0; j < 4; ++j) inv_freq[j] = exp2(-2.0 * (k0 + j) / static_cast<double>(head_dim) * log2_base);
  }
  __device__ void angles(double pos, bool inverse, float (&c)[4], float (&sn)[4]) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double ang = pos * inv_freq[j];
      ang -= 6.283185307179586 * rint(ang * 0.15915494309189535);  // to [-pi, pi]
      float sf, cf;
      sincosf(static_cast<float>(ang), &sf, &cf);
      c[j] = cf;
      sn[j] = inverse ? -sf : sf;
    }
  }
};
DKV_DEVICE void rotate8r(float (&f)[8], const float (&c)[4], const float (&sn)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float e = f[2 * j], o = f[2 * j + 1];
    f[2 * j] = e * c[j] - o * sn[j];
    f[2 * j + 1] = e * sn[j] + o * c[j];
  }
}


// sum over the VPH lanes that hold one head (VPH = head_dim / 8, a power of two <= 32)
template <int VPH>
DKV_DEVICE float head_sum(float x) {
#pragma unroll
  for (int s = VPH / 2; s > 0; s >>= 1) x += __shfl_xor_sync(0xffffffffu, x, s);
  return x;
}

// one CTA per row (grid-stride): thread i handles vectors i, i + 256, ... of the row
template <int VPH>
__global__ void __launch_bounds__(kThreads) qkv_prep_fwd_kernel(const PrepArgs a) {
  static_assert(kThreads % VPH == 0, "a thread keeps one d-slice");
  const int half = a.head_dim / 2;
  const int ht = a.heads + 2 * a.kv_heads;
  const int nvec = ht * VPH;
  const int hq = a.heads, hqk = a.heads + a.kv_heads;
  ThreadPairs tp;
  tp.init(((threadIdx.x % VPH) * 4) % half, a.head_dim, a.log2_base);
  for (int64_t r = blockIdx.x; r < a.rows; r += gridDim.x) {
    const uint4* src = reinterpret_cast<const uint4*>(a.qkv + r * ht * a.head_dim);
    const int64_t d = a.dst[r];
    float cr[4], sr[4];
    tp.angles(static_cast<double>(a.pos[r]), false, cr, sr);
    for (int i0 = 0; i0 < nvec; i0 += kThreads) {  // whole warps stay in the loop (shuffles)
      const int i = i0 + threadIdx.x;
      const bool live = i < nvec;
      const int head = live ? i / VPH : 0, sub = i % VPH;
      float f[8];
      if (live) unpack8(__ldg(src + i), f);
      const __nv_bfloat16* w = head < hq ? a.wq : (head < hqk ? a.wk : nullptr);
      if (a.wq != nullptr) {  // RMSNorm of the q / k heads; every lane joins the shuffles (a warp
        float ss = 0.f;       // may hold a k and a v head)
        if (live) {
#pragma unroll
          for (int j = 0; j < 8; ++j) ss = fmaf(f[j], f[j], ss);
        }
        ss = head_sum<VPH>(ss);
        if (live && w != nullptr) {
          const float rstd = rsqrtf(ss / static_cast<float>(a.head_dim) + a.eps);
          float wv[8];
          unpack8(__ldg(reinterpret_cast<const uint4*>(w) + sub), wv);
#pragma unroll
          for (int j = 0; j < 8; ++j) f[j] = f[j] * rstd * wv[j];
        }
      }
      if (!live) continue;
      if (head < hqk) rotate8r(f, cr, sr);
      const uint4 out = pack8(f);
      if (head < hq)
        reinterpret_cast<uint4*>(a.q + (d * a.heads + head) * a.head_dim)[sub] = out;
      else if (head < hqk)
        reinterpret_cast<uint4*>(a.k + (d * a.kv_heads + head - hq) * a.head_dim)[sub] = out;
      else
        reinterpret_cast<uint4*>(a.v + (d * a.kv_heads + head - hqk) * a.head_dim)[sub] = out;
    }
  }
}

// kIter >= ceil(nvec / 256): the per-thread dw accumulators cost 8 registers per slot, so the
// launch picks the smallest power of two (Qwen3-8B: 768 vectors -> 4; a fixed 8 held the kernel at
// 119 registers and 2 CTAs per SM, 3.6x the forward's time in tools/profile_layer.py)
template <int VPH, int kIter>
__global__ void __launch_bounds__(kThreads, 4) qkv_prep_bwd_kernel(const PrepArgs a) {
  const int half = a.head_dim / 2;
  const int ht = a.heads + 2 * a.kv_heads;
  const int nvec = ht * VPH;
  const int hq = a.heads, hqk = a.heads + a.kv_heads;
  ThreadPairs tp;
  tp.init(((threadIdx.x % VPH) * 4) % half, a.head_dim, a.log2_base);
  // per-thread partial dw over every row this CTA visits: kThreads is a multiple of VPH, so a
  // thread's d-slice (vector index % VPH) is the same in all its slots -- one accumulator per
  // head kind (q, k) instead of one per slot
  static_assert(kThreads % VPH == 0, "a thread keeps one d-slice");
  float dwacc[2][8];
#pragma unroll
  for (int kd = 0; kd < 2; ++kd)
#pragma unroll
    for (int j = 0; j < 8; ++j) dwacc[kd][j] = 0.f;
  const bool norm = a.wq != nullptr;
  for (int64_t r = blockIdx.x; r < a.rows; r += gridDim.x) {
    const uint4* xsrc = reinterpret_cast<const uint4*>(a.qkv + r * ht * a.head_dim);
    uint4* gdst = reinterpret_cast<uint4*>(a.dqkv + r * ht * a.head_dim);
    const int64_t d = a.dst[r];
    float cr[4], sr[4];
    tp.angles(static_cast<double>(a.pos[r]), true, cr, sr);  // the adjoint (inverse) rotation
#pragma unroll 1
    for (int it = 0; it < kIter; ++it) {
      const int i0 = it * kThreads;
      if (i0 >= nvec) break;
      const int i = i0 + threadIdx.x;
      const bool live = i < nvec;
      const int head = live ? i / VPH : 0, sub = i % VPH;
      float g[8];
      if (live) {
        const uint4* gsrc = head < hq ? reinterpret_cast<const uint4*>(a.q + (d * a.heads + head) * a.head_dim)
                          : head < hqk ? reinterpret_cast<const uint4*>(a.k + (d * a.kv_heads + head - hq) * a.head_dim)
                                       : reinterpret_cast<const uint4*>(a.v + (d * a.kv_heads + head - hqk) * a.head_dim);
        unpack8(gsrc[sub], g);
        if (head < hqk) rotate8r(g, cr, sr);  // the adjoint rotation
      }
      const __nv_bfloat16* w = head < hq ? a.wq : (head < hqk ? a.wk : nullptr);
      if (norm) {  // every lane joins the shuffles; only q / k heads use them
        float x[8], wv[8];
        float ss = 0.f, xu = 0.f;
        const bool nh = live && w != nullptr;
        if (nh) {
          unpack8(__ldg(xsrc + i), x);
          unpack8(__ldg(reinterpret_cast<const uint4*>(w) + sub), wv);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            ss = fmaf(x[j], x[j], ss);
            xu = fmaf(x[j], wv[j] * g[j], xu);
          }
        }
        ss = head_sum<VPH>(ss);
        xu = head_sum<VPH>(xu);
        if (nh) {
          const float inv_d = 1.f / static_cast<float>(a.head_dim);
          const float rstd = rsqrtf(ss * inv_d + a.eps);
          const float c = rstd * rstd * rstd * xu * inv_d;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (head < hq)
              dwacc[0][j] = fmaf(g[j], x[j] * rstd, dwacc[0][j]);  // dw += g * x_hat
            else
              dwacc[1][j] = fmaf(g[j], x[j] * rstd, dwacc[1][j]);
            g[j] = rstd * wv[j] * g[j] - x[j] * c;
          }
        }
      }
      if (live) gdst[i] = pack8(g);
    }
  }
  if (!norm) return;
  const int sub = threadIdx.x % VPH;
  bool has_q = false, has_k = false;  // does any of this thread's slots hold a q / k head
#pragma unroll
  for (int it = 0; it < kIter; ++it) {
    const int i = it * kThreads + threadIdx.x;
    if (i < nvec) {
      has_q |= i / VPH < hq;
      has_k |= i / VPH >= hq && i / VPH < hqk;
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (has_q) atomicAdd(a.dwq + sub * 8 + j, dwacc[0][j]);
    if (has_k) atomicAdd(a.dwk + sub * 8 + j, dwacc[1][j]);
  }
}

int grid_for(int64_t rows) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return static_cast<int>(std::min<int64_t>(rows, static_cast<int64_t>(sms) * 8));
}

int check_args(const PrepArgs& a, const char* fn) {
  const int ht = a.heads + 2 * a.kv_heads;
  if (a.rows < 0 || a.heads <= 0 || a.kv_heads <= 0 || a.heads % a.kv_heads || !a.qkv || !a.pos || !a.dst ||
      !a.q || !a.k || !a.v) {
    set_error(std::string(fn) + ": invalid arguments");
    return DKV_ERR_INVALID;
  }
  if (a.head_dim != 64 && a.head_dim != 128 && a.head_dim != 256) {
    set_error(std::string(fn) + ": head_dim must be 64, 128 or 256");
    return DKV_ERR_UNSUPPORTED;
  }
  if ((a.wq == nullptr) != (a.wk == nullptr)) {
    set_error(std::string(fn) + ": q and k norm weights go together");
    return DKV_ERR_INVALID;
  }
  if (ht * (a.head_dim / 8) > 8 * kThreads) {
    set_error(std::string(fn) + ": too many heads per row");
    return DKV_ERR_UNSUPPORTED;
  }
  return DKV_OK;
}

}  // namespace

}  // namespace dkv

using namespace dkv;

extern "C" int32_t dkv_qkv_prep_fwd(const void* qkv, const void* q_norm_w, const void* k_norm_w, float eps,
                                    const int64_t* positions, const int64_t* dst_rows, void* q, void* k, void* v,
                                    int64_t rows, int64_t heads, int64_t kv_heads, int64_t head_dim, double base,
                                    void* stream) {
  PrepArgs a{};
  a.qkv = static_cast<const __nv_bfloat16*>(qkv);
  a.wq = static_cast<const __nv_bfloat16*>(q_norm_w);
  a.wk = static_cast<const __nv_bfloat16*>(k_norm_w);
  a.pos = positions;
  a.dst = dst_rows;
  a.q = static_cast<__nv_bfloat16*>(q);
  a.k = static_cast<__nv_bfloat16*>(k);
  a.v = static_cast<__nv_bfloat16*>(v);
  a.rows = rows;
  a.heads = static_cast<int>(heads);
  a.kv_heads = static_cast<int>(kv_heads);
  a.head_dim = static_cast<int>(head_dim);
  a.eps = eps;
  a.log2_base = std::log2(base);
  if (rows == 0) return DKV_OK;
  int rc = check_args(a, "dkv_qkv_prep_fwd");
  if (rc) return rc;
  auto st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for(rows);
  if (a.head_dim == 128)
    qkv_prep_fwd_kernel<16><<<grid, kThreads, 0, st>>>(a);
  else if (a.head_dim == 64)
    qkv_prep_fwd_kernel<8><<<grid, kThreads, 0, st>>>(a);
  else
    qkv_prep_fwd_kernel<32><<<grid, kThreads, 0, st>>>(a);
  prof_count(1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("dkv_qkv_prep_fwd: ") + cudaGetErrorString(e));
    return DKV_ERR_CUDA;
  }
  return DKV_OK;
}

extern "C" int32_t dkv_qkv_prep_bwd(const void* dq, const void* dk, const void* dv, const void* qkv,
                                    const void* q_norm_w, const void* k_norm_w, float eps, const int64_t* positions,
                                    const int64_t* dst_rows, void* dqkv, float* dq_norm_w, float* dk_norm_w,
                                    int64_t rows, int64_t heads, int64_t kv_heads, int64_t head_dim, double base,
                                    void* stream) {
  PrepArgs a{};
  a.qkv = static_cast<const __nv_bfloat16*>(qkv);
  a.wq = static_cast<const __nv_bfloat16*>(q_norm_w);
  a.wk = static_cast<const __nv_bfloat16*>(k_norm_w);
  a.pos = positions;
  a.dst = dst_rows;
  a.q = static_cast<__nv_bfloat16*>(const_cast<void*>(dq));
  a.k = static_cast<__nv_bfloat16*>(const_cast<void*>(dk));
  a.v = static_cast<__nv_bfloat16*>(const_cast<void*>(dv));
  a.dqkv = static_cast<__nv_bfloat16*>(dqkv);
  a.dwq = dq_norm_w;
  a.dwk = dk_norm_w;
  a.rows = rows;
  a.heads = static_cast<int>(heads);
  a.kv_heads = static_cast<int>(kv_heads);
  a.head_dim = static_cast<int>(head_dim);
  a.eps = eps;
  a.log2_base = std::log2(base);
  auto st = static_cast<cudaStream_t>(stream);
  if (a.wq && (!a.dwq || !a.dwk)) {
    set_error("dkv_qkv_prep_bwd: norm weight gradients need fp32 accumulators");
    return DKV_ERR_INVALID;
  }
  if (a.wq) {  // the accumulators are summed into: zero them here (stream-ordered)
    cudaMemsetAsync(a.dwq, 0, head_dim * sizeof(float), st);
    cudaMemsetAsync(a.dwk, 0, head_dim * sizeof(float), st);
  }
  if (rows == 0) return DKV_OK;
  int rc = check_args(a, "dkv_qkv_prep_bwd");
  if (rc) return rc;
  if (!a.dqkv) {
    set_error("dkv_qkv_prep_bwd: null dqkv");
    return DKV_ERR_INVALID;
  }
  const int grid = grid_for(rows);
  const int vph = static_cast<int>(head_dim) / 8;
  const int iters = static_cast<int>(((heads + 2 * kv_heads) * vph + kThreads - 1) / kThreads);
  auto launch = [&](auto vph_c) {
    constexpr int V = decltype(vph_c)::value;
    if (iters <= 1)
      qkv_prep_bwd_kernel<V, 1><<<grid, kThreads, 0, st>>>(a);
    else if (iters <= 2)
      qkv_prep_bwd_kernel<V, 2><<<grid, kThreads, 0, st>>>(a);
    else if (iters <= 4)
      qkv_prep_bwd_kernel<V, 4><<<grid, kThreads, 0, st>>>(a);
    else
      qkv_prep_bwd_kernel<V, 8><<<grid, kThreads, 0, st>>>(a);
  };
  if (a.head_dim == 128)
    launch(std::integral_constant<int, 16>{});
  else if (a.head_dim == 64)
    launch(std::integral_constant<int, 8>{});
  else
    launch(std::integral_constant<int, 32>{});
  prof_count(1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("dkv_qkv_prep_bwd: ") + cudaGetErrorString(e));
    return DKV_ERR_CUDA;
  }
  return DKV_OK;
}
