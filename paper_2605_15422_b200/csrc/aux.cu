// aux.cu -- HBM-bound helper kernels around the attention core:
//   * backward preprocess: D = rowsum(dO * O) (fa2.py:232-234), in two layouts
//   * fixed-order fold + single RNE cast of the shared-prompt gradient
//     (kernel.py:279-285 / convert_dkv_context kernel.py:140-148)
//   * f32 -> storage cast (dQ accumulator, generic convert)
//   * row gather / segment-sum for the N(P+R) <-> P+NR repack (packing.py:159-220)
//   * RoPE at logical positions, optionally fused with the repack gather (layer.py:182-205)
#include "dkv_internal.h"

#include <algorithm>
#include <cmath>

namespace dkv {

template <typename T>
DKV_DEVICE float to_f(T v);
template <>
DKV_DEVICE float to_f<float>(float v) { return v; }
template <>
DKV_DEVICE float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

// hi + mid + lo bf16 parts of x (residual <= 2^-24 |x|): lets a K=16 bf16 MMA add an
// fp32-accurate per-column constant to an accumulator
DKV_DEVICE void split3_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& mid, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(hi);
  mid = __float2bfloat16_rn(r1);
  lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
}

// one warp per (token, head).  drow: [H][T] (may be null).  xsplit (may be null): the
// tensor-core backward's per-row additive constants, rows ((hk*tpad + t)*G + g), 32 bf16 each:
// [split3(-lse/scale), 0 x 13, split3(-D), 0 x 13]; rows of padding tokens t >= T are zero.
template <typename T>
__global__ void rowsum_kernel(SimtArgs a, float* drow, __nv_bfloat16* xsplit, int tpad) {
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int rows = xsplit ? tpad : a.total_q;
  if (gw >= static_cast<int64_t>(rows) * a.heads) return;
  const int t = static_cast<int>(gw / a.heads), h = static_cast<int>(gw % a.heads);
  float acc = 0.f;
  if (t < a.total_q) {
    const int64_t off = (static_cast<int64_t>(t) * a.heads + h) * a.head_dim;
    const T* o = static_cast<const T*>(a.out) + off;
    const T* g = static_cast<const T*>(a.dout) + off;
    for (int e = lane; e < a.head_dim; e += 32) acc += to_f(o[e]) * to_f(g[e]);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  }
  if (lane == 0) {
    if (drow && t < a.total_q) drow[static_cast<int64_t>(h) * a.total_q + t] = acc;
    if (xsplit) {
      const int G = a.heads / a.kv_heads;
      const int hk = h / G, gi = h % G;
      __nv_bfloat16 v[32];
      for (int i = 0; i < 32; ++i) v[i] = __float2bfloat16_rn(0.f);
      if (t < a.total_q) {
        const float lse = a.lse[static_cast<int64_t>(h) * a.total_q + t];
        split3_bf16(-lse / a.scale, v[0], v[1], v[2]);
        split3_bf16(-acc, v[16], v[17], v[18]);
      }
      uint4* dst = reinterpret_cast<uint4*>(xsplit + ((static_cast<int64_t>(hk) * tpad + t) * G + gi) * 32);
      const uint4* src = reinterpret_cast<const uint4*>(v);
      for (int i = 0; i < 4; ++i) dst[i] = src[i];
    }
  }
}

// bf16 fast path: LPR = head_dim / 16 lanes per (token, head) row, two 16-byte loads of O and of
// dO per lane (fully coalesced), a log2(LPR)-step shuffle reduction, one 64 B xsplit row store.
template <int LPR>
__global__ void rowsum_bf16_kernel(SimtArgs a, float* drow, __nv_bfloat16* xsplit, int tpad) {
  const int64_t gt = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int sub = threadIdx.x & (LPR - 1);
  const int64_t row = gt / LPR;  // (t, h) row, t-major
  const int rows = xsplit ? tpad : a.total_q;
  const bool live = row < static_cast<int64_t>(rows) * a.heads;
  const int t = live ? static_cast<int>(row / a.heads) : 0, h = live ? static_cast<int>(row % a.heads) : 0;
  float acc = 0.f;
  if (live && t < a.total_q) {
    const int64_t off = row * (LPR * 16) + sub * 16;
    const uint4* o = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.out) + off);
    const uint4* g = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.dout) + off);
    const uint4 o0 = o[0], o1 = o[1], g0 = g[0], g1 = g[1];
    const uint32_t ov[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
    const uint32_t gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc = fmaf(__uint_as_float(ov[i] << 16), __uint_as_float(gv[i] << 16), acc);
      acc = fmaf(__uint_as_float(ov[i] & 0xffff0000u), __uint_as_float(gv[i] & 0xffff0000u), acc);
    }
  }
#pragma unroll
  for (int s = LPR / 2; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (!live || sub != 0) return;
  if (drow && t < a.total_q) drow[static_cast<int64_t>(h) * a.total_q + t] = acc;
  if (xsplit) {
    const int G = a.heads / a.kv_heads;
    const int hk = h / G, gi = h % G;
    __nv_bfloat16 v[32];
    for (int i = 0; i < 32; ++i) v[i] = __float2bfloat16_rn(0.f);
    if (t < a.total_q) {
      const float lse = a.lse[static_cast<int64_t>(h) * a.total_q + t];
      split3_bf16(-lse / a.scale, v[0], v[1], v[2]);
      split3_bf16(-acc, v[16], v[17], v[18]);
    }
    uint4* dst = reinterpret_cast<uint4*>(xsplit + ((static_cast<int64_t>(hk) * tpad + t) * G + gi) * 32);
    const uint4* src = reinterpret_cast<const uint4*>(v);
    for (int i = 0; i < 4; ++i) dst[i] = src[i];
  }
}

void launch_rowsum_do_o(const SimtArgs& a, float* drow, __nv_bfloat16* xsplit, int tpad, cudaStream_t st) {
  const int64_t rows = xsplit ? tpad : a.total_q;
  const int64_t warps = rows * a.heads;
  if (warps == 0) return;
  if (a.dtype == DKV_BF16 && (a.head_dim == 128 || a.head_dim == 64)) {
    const int lpr = a.head_dim / 16;
    const int threads = 256;
    const int64_t blocks = (warps * lpr + threads - 1) / threads;
    if (lpr == 8)
      rowsum_bf16_kernel<8><<<blocks, threads, 0, st>>>(a, drow, xsplit, tpad);
    else
      rowsum_bf16_kernel<4><<<blocks, threads, 0, st>>>(a, drow, xsplit, tpad);
    return;
  }
  const int threads = 256;
  const int64_t blocks = (warps * 32 + threads - 1) / threads;
  if (a.dtype == DKV_F32)
    rowsum_kernel<float><<<blocks, threads, 0, st>>>(a, drow, xsplit, tpad);
  else
    rowsum_kernel<__nv_bfloat16><<<blocks, threads, 0, st>>>(a, drow, xsplit, tpad);
}

// dk/dv[i] = cast(sum_{c < num_parts} partials[c][0/1][i]), fixed chunk order; f32_out (optional)
// receives the fp32 sums [2][plane] (the instrumentation view of the value that is cast once)
__global__ void fold_convert_kernel(const float* __restrict__ parts, int num_parts, int64_t plane, void* dk,
                                    void* dv, int dtype, float* f32_out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= 2 * plane) return;
  const int which = static_cast<int>(i / plane);
  const int64_t e = i % plane;
  float acc = 0.f;
  for (int c = 0; c < num_parts; ++c) acc += parts[(static_cast<int64_t>(c) * 2 + which) * plane + e];
  if (f32_out) f32_out[i] = acc;
  void* dst = which == 0 ? dk : dv;
  if (dtype == DKV_F32)
    static_cast<float*>(dst)[e] = acc;
  else
    static_cast<__nv_bfloat16*>(dst)[e] = __float2bfloat16_rn(acc);
}

void launch_fold_convert(const float* partials, int num_parts, int64_t plane, void* dk, void* dv, int dtype,
                         float* f32_out, cudaStream_t st) {
  if (plane == 0) return;
  const int threads = 256;
  const int64_t blocks = (2 * plane + threads - 1) / threads;
  fold_convert_kernel<<<blocks, threads, 0, st>>>(partials, num_parts, plane, dk, dv, dtype, f32_out);
}

// vectorised f32 -> {bf16, f32}; RNE via __float2bfloat16_rn (== reference bf16_round)
__global__ void convert_kernel(const float* __restrict__ src, void* dst, int dtype, int64_t n, float scale) {
  const int64_t i4 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (i4 >= n) return;
  if (i4 + 4 <= n && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    float4 v = *reinterpret_cast<const float4*>(src + i4);
    v.x *= scale; v.y *= scale; v.z *= scale; v.w *= scale;
    if (dtype == DKV_F32) {
      float* d = static_cast<float*>(dst) + i4;
      d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
    } else {
      __nv_bfloat162* d = reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(dst) + i4);
      d[0] = __floats2bfloat162_rn(v.x, v.y);
      d[1] = __floats2bfloat162_rn(v.z, v.w);
    }
    return;
  }
  for (int64_t i = i4; i < n && i < i4 + 4; ++i) {
    if (dtype == DKV_F32)
      static_cast<float*>(dst)[i] = src[i] * scale;
    else
      static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(src[i] * scale);
  }
}

void launch_convert(const float* src, void* dst, int dtype, int64_t n, cudaStream_t st, float scale) {
  if (n == 0) return;
  const int threads = 256;
  const int64_t blocks = ((n + 3) / 4 + threads - 1) / threads;
  convert_kernel<<<blocks, threads, 0, st>>>(src, dst, dtype, n, scale);
}

// ---------------------------------------------------------------- repack
// one CTA-slice per destination row; 16-byte vectors when rows allow it
__global__ void gather_rows_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                   int64_t row_bytes, const int64_t* __restrict__ idx, int64_t n_rows) {
  const int64_t r = blockIdx.x;
  if (r >= n_rows) return;
  const uint8_t* s = src + idx[r] * row_bytes;
  uint8_t* d = dst + r * row_bytes;
  if ((row_bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    const int64_t n16 = row_bytes >> 4;
    for (int64_t i = threadIdx.x; i < n16; i += blockDim.x)
      reinterpret_cast<int4*>(d)[i] = __ldg(reinterpret_cast<const int4*>(s) + i);
  } else {
    for (int64_t i = threadIdx.x; i < row_bytes; i += blockDim.x) d[i] = s[i];
  }
}

template <typename T>
__global__ void segment_sum_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t row_elems,
                                   const int64_t* __restrict__ seg, const int64_t* __restrict__ sidx,
                                   int64_t n_rows) {
  const int64_t r = blockIdx.x;
  if (r >= n_rows) return;
  const int64_t j0 = seg[r], j1 = seg[r + 1];
  for (int64_t e = threadIdx.x; e < row_elems; e += blockDim.x) {
    float acc = 0.f;
    for (int64_t j = j0; j < j1; ++j) acc += to_f(src[sidx[j] * row_elems + e]);
    if constexpr (sizeof(T) == 4)
      dst[r * row_elems + e] = acc;
    else
      dst[r * row_elems + e] = __float2bfloat16_rn(acc);
  }
}

}  // namespace dkv

using namespace dkv;

extern "C" int32_t dkv_gather_rows(const void* src, void* dst, int64_t row_bytes, const int64_t* idx,
                                   int64_t n_rows, void* stream) {
  if (n_rows < 0 || row_bytes <= 0 || (n_rows > 0 && (!src || !dst || !idx))) {
    set_error("dkv_gather_rows: invalid arguments");
    return DKV_ERR_INVALID;
  }
  if (n_rows == 0) return DKV_OK;
  const int threads = row_bytes >= 4096 ? 256 : 128;
  gather_rows_kernel<<<static_cast<unsigned>(n_rows), threads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), row_bytes, idx, n_rows);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("dkv_gather_rows: ") + cudaGetErrorString(e));
    return DKV_ERR_CUDA;
  }
  return DKV_OK;
}

extern "C" int32_t dkv_segment_sum_rows(const void* src, void* dst, int32_t dtype, int64_t row_elems,
                                        const int64_t* seg, const int64_t* src_idx, int64_t n_rows,
                                        void* stream) {
  if (n_rows < 0 || row_elems <= 0 || (dtype != DKV_BF16 && dtype != DKV_F32)) {
    set_error("dkv_segment_sum_rows: invalid arguments");
    return DKV_ERR_INVALID;
  }
  if (n_rows == 0) return DKV_OK;
  auto st = static_cast<cudaStream_t>(stream);
  if (dtype == DKV_F32)
    segment_sum_kernel<float><<<static_cast<unsigned>(n_rows), 128, 0, st>>>(
        static_cast<const float*>(src), static_cast<float*>(dst), row_elems, seg, src_idx, n_rows);
  else
    segment_sum_kernel<__nv_bfloat16><<<static_cast<unsigned>(n_rows), 128, 0, st>>>(
        static_cast<const __nv_bfloat16*>(src), static_cast<__nv_bfloat16*>(dst), row_elems, seg, src_idx,
        n_rows);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("dkv_segment_sum_rows: ") + cudaGetErrorString(e));
    return DKV_ERR_CUDA;
  }
  return DKV_OK;
}

// RoPE: one CTA per destination row, for up to three tensors of that row (q and k rotated, v
// copied -- the fused repack + RoPE of the QKV projections).  The row's d/2 angles
// pos * base^(-2k/d) are formed in fp64 (|angle| reaches ~2e4 rad at long prompts), reduced
// mod 2 pi in fp64 and only then taken through fp32 sincos; the (cos, sin) pairs are shared by
// every head of q and k.  Pairs move as 16-byte vectors (4 bf16 / 2 fp32 pairs): HBM-bound.
template <typename T>
DKV_DEVICE void rope_vec(uint4& v, const float* cs, int half, int k0) {
  uint32_t* w = reinterpret_cast<uint32_t*>(&v);
  if constexpr (sizeof(T) == 2) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float c = cs[k0 + j], sn = cs[half + k0 + j];
      const float ev = __uint_as_float(w[j] << 16), od = __uint_as_float(w[j] & 0xffff0000u);
      __nv_bfloat162 o = __floats2bfloat162_rn(ev * c - od * sn, ev * sn + od * c);
      w[j] = *reinterpret_cast<uint32_t*>(&o);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float c = cs[k0 + j], sn = cs[half + k0 + j];
      const float ev = __uint_as_float(w[2 * j]), od = __uint_as_float(w[2 * j + 1]);
      w[2 * j] = __float_as_uint(ev * c - od * sn);
      w[2 * j + 1] = __float_as_uint(ev * sn + od * c);
    }
  }
}

struct RopeArgs {
  const void* src[3];
  void* dst[3];
  int64_t nvec[3];   // 16-byte vectors per row of each tensor (0: tensor absent)
  int rotate[3];
  int64_t head_dim;
  const int64_t* positions;
  const int64_t* idx;
  double log2_base;
  int inverse;
};

// Every thread issues its (up to kVecPerThread) 16-byte loads of the row FIRST -- their addresses
// depend only on the gather index -- and computes the row's angles while they are in flight.
constexpr int kRopeVecPerThread = 3;

template <typename T>
__global__ void rope_rows_kernel(const RopeArgs a) {
  extern __shared__ float cs[];  // [d/2] cos, [d/2] sin
  const int64_t r = blockIdx.x;
  const int half = static_cast<int>(a.head_dim / 2);
  constexpr int kPairs = sizeof(T) == 2 ? 4 : 2;  // pairs per 16-byte vector
  const int64_t sr = a.idx ? a.idx[r] : r;
  const int n0 = static_cast<int>(a.nvec[0]), n1 = static_cast<int>(a.nvec[1]), n2 = static_cast<int>(a.nvec[2]);
  const int n01 = n0 + n1, total = n01 + n2;
  // vector i of the row -> (tensor, offset); pointers chosen by selects (a runtime index into
  // the parameter arrays would copy them to local memory)
  struct Loc {
    const uint4* src;
    uint4* dst;
    int off;
    bool rot;
  };
  auto locate = [&](int i) {
    Loc l;
    if (i < n0) {
      l = {reinterpret_cast<const uint4*>(a.src[0]) + sr * n0, reinterpret_cast<uint4*>(a.dst[0]) + r * n0, i,
           a.rotate[0] != 0};
    } else if (i < n01) {
      l = {reinterpret_cast<const uint4*>(a.src[1]) + sr * n1, reinterpret_cast<uint4*>(a.dst[1]) + r * n1, i - n0,
           a.rotate[1] != 0};
    } else {
      l = {reinterpret_cast<const uint4*>(a.src[2]) + sr * n2, reinterpret_cast<uint4*>(a.dst[2]) + r * n2,
           i - n01, a.rotate[2] != 0};
    }
    return l;
  };
  uint4 v[kRopeVecPerThread];
#pragma unroll
  for (int j = 0; j < kRopeVecPerThread; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    if (i < total) v[j] = __ldg(locate(i).src + locate(i).off);
  }
  const double pos = static_cast<double>(a.positions[r]);
  for (int k = threadIdx.x; k < half; k += blockDim.x) {
    const double inv_freq = exp2(-2.0 * k / static_cast<double>(a.head_dim) * a.log2_base);
    double ang = pos * inv_freq;
    ang -= 6.283185307179586 * rint(ang * 0.15915494309189535);  // to [-pi, pi]
    float sf, cf;
    sincosf(static_cast<float>(ang), &sf, &cf);
    cs[k] = cf;
    cs[half + k] = a.inverse ? -sf : sf;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kRopeVecPerThread; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    if (i < total) {
      const Loc l = locate(i);
      if (l.rot) rope_vec<T>(v[j], cs, half, (l.off * kPairs) % half);
      l.dst[l.off] = v[j];
    }
  }
  // rows wider than kRopeVecPerThread x blockDim vectors (not hit by the launch below)
  for (int i = threadIdx.x + kRopeVecPerThread * blockDim.x; i < total; i += blockDim.x) {
    const Loc l = locate(i);
    uint4 w = l.src[l.off];
    if (l.rot) rope_vec<T>(w, cs, half, (l.off * kPairs) % half);
    l.dst[l.off] = w;
  }
}

extern "C" int32_t dkv_rope_qkv_rows(const void* q_src, const void* k_src, const void* v_src, void* q_dst,
                                     void* k_dst, void* v_dst, int32_t dtype, int64_t n_rows, int64_t heads,
                                     int64_t kv_heads, int64_t head_dim, const int64_t* positions,
                                     const int64_t* idx, double base, int32_t inverse, void* stream) {
  const int pairs_per_vec = dtype == DKV_BF16 ? 4 : 2;
  if (n_rows < 0 || heads < 0 || kv_heads < 0 || head_dim <= 0 || !(base > 0.0) ||
      (dtype != DKV_BF16 && dtype != DKV_F32) || (n_rows > 0 && !positions)) {
    set_error("dkv_rope_qkv_rows: invalid arguments");
    return DKV_ERR_INVALID;
  }
  RopeArgs a{};
  const void* srcs[3] = {q_src, k_src, v_src};
  void* dsts[3] = {q_dst, k_dst, v_dst};
  const int64_t hs[3] = {heads, kv_heads, kv_heads};
  int64_t total = 0;
  for (int t = 0; t < 3; ++t) {
    if (!srcs[t] && !dsts[t]) continue;
    if (!srcs[t] || !dsts[t] || hs[t] <= 0 || (srcs[t] == dsts[t] && idx) ||
        (reinterpret_cast<uintptr_t>(srcs[t]) & 15) || (reinterpret_cast<uintptr_t>(dsts[t]) & 15)) {
      set_error("dkv_rope_qkv_rows: tensor pointers must be 16-byte aligned pairs (no in-place gather)");
      return DKV_ERR_INVALID;
    }
    a.src[t] = srcs[t];
    a.dst[t] = dsts[t];
    a.nvec[t] = hs[t] * head_dim / 2 / pairs_per_vec;
    a.rotate[t] = t < 2;
    total += a.nvec[t];
  }
  if ((head_dim / 2) % pairs_per_vec) {
    set_error("dkv_rope_qkv_rows: head_dim must be a multiple of 8 (bf16) / 4 (fp32)");
    return DKV_ERR_UNSUPPORTED;
  }
  if (n_rows == 0 || total == 0) return DKV_OK;
  a.head_dim = head_dim;
  a.positions = positions;
  a.idx = idx;
  a.log2_base = std::log2(base);
  a.inverse = inverse;
  auto st = static_cast<cudaStream_t>(stream);
  const size_t sm = static_cast<size_t>(head_dim) * sizeof(float);
  // enough threads that every vector of the row is one of the up-front loads (<= 1024)
  int64_t want = (total + kRopeVecPerThread - 1) / kRopeVecPerThread;
  want = std::max<int64_t>(want, head_dim / 2);
  const int threads = static_cast<int>(std::min<int64_t>(1024, std::max<int64_t>(256, (want + 31) / 32 * 32)));
  if (dtype == DKV_BF16)
    rope_rows_kernel<__nv_bfloat16><<<static_cast<unsigned>(n_rows), threads, sm, st>>>(a);
  else
    rope_rows_kernel<float><<<static_cast<unsigned>(n_rows), threads, sm, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("dkv_rope_qkv_rows: ") + cudaGetErrorString(e));
    return DKV_ERR_CUDA;
  }
  return DKV_OK;
}

extern "C" int32_t dkv_rope_rows(const void* src, void* dst, int32_t dtype, int64_t n_rows, int64_t heads,
                                 int64_t head_dim, const int64_t* positions, const int64_t* idx, double base,
                                 int32_t inverse, void* stream) {
  if (n_rows > 0 && (!src || !dst)) {
    set_error("dkv_rope_rows: invalid arguments");
    return DKV_ERR_INVALID;
  }
  return dkv_rope_qkv_rows(src, nullptr, nullptr, dst, nullptr, nullptr, dtype, n_rows, heads, 0, head_dim,
                           positions, idx, base, inverse, stream);
}

extern "C" int32_t dkv_convert_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!src || !dst))) {
    set_error("dkv_convert_f32_to_bf16: invalid arguments");
    return DKV_ERR_INVALID;
  }
  launch_convert(src, dst, DKV_BF16, n, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("dkv_convert_f32_to_bf16: ") + cudaGetErrorString(e));
    return DKV_ERR_CUDA;
  }
  return DKV_OK;
}
