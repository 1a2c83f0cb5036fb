// simt_attn.cu -- fp32 SIMT DualKV kernels (any head_dim <= 256, any GQA ratio,
// fp32 or bf16 storage).  These serve the fp32 dtype (BASELINE config C1) and
// shapes the tcgen05 path does not take; compute is fp32 with exact expf.
//
// Semantics follow the reference tile core (fa2.py:112-229, kernel.py:177-305):
// query row r of sequence i (logical position ctx_len + r) sees all context
// keys and own keys 0..r; context gradients are summed over sequences in fp32
// and cast once.
#include "dkv_internal.h"

#include <type_traits>

namespace dkv {

template <typename T>
DKV_DEVICE float ldf(const T* p);
template <>
DKV_DEVICE float ldf<float>(const float* p) { return __ldg(p); }
template <>
DKV_DEVICE float ldf<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

template <typename T>
DKV_DEVICE void stf(T* p, float v);
template <>
DKV_DEVICE void stf<float>(float* p, float v) { *p = v; }
template <>
DKV_DEVICE void stf<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

DKV_DEVICE float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// values per lane of a head_dim row: a template parameter of every kernel (2 / 4 / 8 for head_dim
// <= 64 / 128 / 256), so small head dims do not pay registers for 256
// keys (fwd, dQ) / query rows (dK dV) per step: independent dot products and interleaved shuffle
// reductions (ILP over the L2-latency-bound chain); more for small head dims (fewer registers per row)
template <int kMaxPerLane>
constexpr int key_block() { return kMaxPerLane <= 2 ? 8 : (kMaxPerLane <= 4 ? 4 : 2); }

template <int N>
DKV_DEVICE void warp_sum_n(float (&v)[N]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
}

// cu_seqlens entry i; a null cu means one sequence spanning all total_q rows (the prompt of a
// fused two-call launch)
DKV_DEVICE int cu_at(const SimtArgs& a, int i) { return a.cu ? a.cu[i] : (i == 0 ? 0 : a.total_q); }

// binary search: sequence containing packed row t
DKV_DEVICE int seq_of_row(const int32_t* cu, int n, int t) {
  if (!cu) return 0;
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (cu[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------- forward
// one warp per (packed query row, head); lanes split head_dim
template <typename T, int kMaxPerLane>
__global__ void simt_fwd_kernel(SimtArgs a) {
  constexpr int kKeyBlock = kMaxPerLane <= 4 ? 4 : 2;  // (8 measured slower here: register-bound)
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= a.total_q * a.heads) return;
  const int t = gw / a.heads, h = gw % a.heads;
  const int hk = h / (a.heads / a.kv_heads);
  const int s = seq_of_row(a.cu, a.num_seqs, t);
  const int r = t - cu_at(a, s);
  const int seq0 = cu_at(a, s);
  const int D = a.head_dim;
  const T* q = static_cast<const T*>(a.q) + (static_cast<int64_t>(t) * a.heads + h) * D;
  float qr[kMaxPerLane], acc[kMaxPerLane];
#pragma unroll
  for (int i = 0; i < kMaxPerLane; ++i) {
    int e = lane + 32 * i;
    qr[i] = e < D ? ldf(q + e) : 0.f;
    acc[i] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  // keys j0 .. j0 + cnt - 1 (cnt <= kKeyBlock) in one online-softmax step
  auto visit = [&](const T* kbase, const T* vbase, int j0, int cnt) {
    float sc[kKeyBlock];
#pragma unroll
    for (int b = 0; b < kKeyBlock; ++b) {
      sc[b] = 0.f;
      if (b < cnt) {
        const T* kr = kbase + (static_cast<int64_t>(j0 + b) * a.kv_heads + hk) * D;
#pragma unroll
        for (int i = 0; i < kMaxPerLane; ++i) {
          int e = lane + 32 * i;
          if (e < D) sc[b] += qr[i] * ldf(kr + e);
        }
      }
    }
    warp_sum_n(sc);
    float mn = m;
#pragma unroll
    for (int b = 0; b < kKeyBlock; ++b) {
      sc[b] = b < cnt ? sc[b] * a.scale : -INFINITY;
      mn = fmaxf(mn, sc[b]);
    }
    const float alpha = expf(m - mn);  // m = -inf first time -> 0
    float pb[kKeyBlock];
#pragma unroll
    for (int b = 0; b < kKeyBlock; ++b) pb[b] = b < cnt ? expf(sc[b] - mn) : 0.f;
    float psum = 0.f;
#pragma unroll
    for (int b = 0; b < kKeyBlock; ++b) psum += pb[b];
    l = l * alpha + psum;
#pragma unroll
    for (int i = 0; i < kMaxPerLane; ++i) {
      int e = lane + 32 * i;
      if (e < D) {
        float add = 0.f;
#pragma unroll
        for (int b = 0; b < kKeyBlock; ++b)
          if (b < cnt) add += pb[b] * ldf(vbase + (static_cast<int64_t>(j0 + b) * a.kv_heads + hk) * D + e);
        acc[i] = acc[i] * alpha + add;
      }
    }
    m = mn;
  };
  for (int j = 0; j < a.ctx_len; j += kKeyBlock)
    visit(static_cast<const T*>(a.k_ctx), static_cast<const T*>(a.v_ctx), j, min(kKeyBlock, a.ctx_len - j));
  const T* kown = static_cast<const T*>(a.k) + static_cast<int64_t>(seq0) * a.kv_heads * D;
  const T* vown = static_cast<const T*>(a.v) + static_cast<int64_t>(seq0) * a.kv_heads * D;
  for (int j = 0; j <= r; j += kKeyBlock) visit(kown, vown, j, min(kKeyBlock, r + 1 - j));
  T* o = static_cast<T*>(a.out) + (static_cast<int64_t>(t) * a.heads + h) * D;
  const float inv = 1.f / l;
#pragma unroll
  for (int i = 0; i < kMaxPerLane; ++i) {
    int e = lane + 32 * i;
    if (e < D) stf(o + e, acc[i] * inv);
  }
  if (lane == 0) a.lse[static_cast<int64_t>(h) * a.total_q + t] = m + logf(l);
}

// ---------------------------------------------------------------- backward: dQ
// D_row[h, t] = sum_d dO*O computed by the preprocess kernel (fa2.py:232-234)
template <typename T, int kMaxPerLane>
__global__ void simt_bwd_dq_kernel(SimtArgs a, const float* drow) {
  constexpr int kKeyBlock = key_block<kMaxPerLane>();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= a.total_q * a.heads) return;
  const int t = gw / a.heads, h = gw % a.heads;
  const int hk = h / (a.heads / a.kv_heads);
  const int s = seq_of_row(a.cu, a.num_seqs, t);
  const int r = t - cu_at(a, s);
  const int seq0 = cu_at(a, s);
  const int D = a.head_dim;
  const int64_t qoff = (static_cast<int64_t>(t) * a.heads + h) * D;
  float qr[kMaxPerLane], gr[kMaxPerLane], dq[kMaxPerLane];
#pragma unroll
  for (int i = 0; i < kMaxPerLane; ++i) {
    int e = lane + 32 * i;
    qr[i] = e < D ? ldf(static_cast<const T*>(a.q) + qoff + e) : 0.f;
    gr[i] = e < D ? ldf(static_cast<const T*>(a.dout) + qoff + e) : 0.f;
    dq[i] = 0.f;
  }
  const float lse = a.lse[static_cast<int64_t>(h) * a.total_q + t];
  const float dr = drow[static_cast<int64_t>(h) * a.total_q + t];
  auto visit = [&](const T* kbase, const T* vbase, int j0, int cnt) {
    float sp[kKeyBlock], dp[kKeyBlock];
#pragma unroll
    for (int b = 0; b < kKeyBlock; ++b) {
      sp[b] = 0.f;
      dp[b] = 0.f;
      if (b < cnt) {
        const int64_t ko = (static_cast<int64_t>(j0 + b) * a.kv_heads + hk) * D;
#pragma unroll
        for (int i = 0; i < kMaxPerLane; ++i) {
          int e = lane + 32 * i;
          if (e < D) {
            sp[b] += qr[i] * ldf(kbase + ko + e);
            dp[b] += gr[i] * ldf(vbase + ko + e);
          }
        }
      }
    }
    warp_sum_n(sp);
    warp_sum_n(dp);
#pragma unroll
    for (int b = 0; b < kKeyBlock; ++b) {
      if (b >= cnt) break;
      const float p = expf(sp[b] * a.scale - lse);
      const float ds = p * (dp[b] - dr) * a.scale;
      const int64_t ko = (static_cast<int64_t>(j0 + b) * a.kv_heads + hk) * D;
#pragma unroll
      for (int i = 0; i < kMaxPerLane; ++i) {
        int e = lane + 32 * i;
        if (e < D) dq[i] += ds * ldf(kbase + ko + e);
      }
    }
  };
  for (int j = 0; j < a.ctx_len; j += kKeyBlock)
    visit(static_cast<const T*>(a.k_ctx), static_cast<const T*>(a.v_ctx), j, min(kKeyBlock, a.ctx_len - j));
  const T* kown = static_cast<const T*>(a.k) + static_cast<int64_t>(seq0) * a.kv_heads * D;
  const T* vown = static_cast<const T*>(a.v) + static_cast<int64_t>(seq0) * a.kv_heads * D;
  for (int j = 0; j <= r; j += kKeyBlock) visit(kown, vown, j, min(kKeyBlock, r + 1 - j));
#pragma unroll
  for (int i = 0; i < kMaxPerLane; ++i) {
    int e = lane + 32 * i;
    if (e < D) stf(static_cast<T*>(a.dq) + qoff + e, dq[i]);
  }
}

// ---------------------------------------------------------------- backward: dK/dV
// one warp per (key row, kv head).  Own-region key j of sequence s sums over
// query rows r >= j of s and all G query heads of the group.  Context key j
// sums over every query row of sequences [s_begin, s_end) (a "chunk"), in
// sequence order, into fp32, then either casts once (ctx_out_*) or writes the
// fp32 partial (instrumentation / deterministic fold).
template <typename T, int kMaxPerLane>
__global__ void simt_bwd_dkv_kernel(SimtArgs a, const float* drow, int own_rows, int chunk,
                                    int num_chunks, float* ctx_part, float* own_part) {
  constexpr int kKeyBlock = kMaxPerLane <= 4 ? 4 : 2;  // (8 measured slower here)
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int D = a.head_dim;
  const int G = a.heads / a.kv_heads;
  const int64_t n_own = static_cast<int64_t>(own_rows) * a.kv_heads;
  const int64_t n_ctx = static_cast<int64_t>(a.ctx_len) * a.kv_heads * num_chunks;
  if (gw >= n_own + n_ctx) return;
  const bool is_ctx = gw >= n_own;
  int j, hk, s_lo, s_hi, chunk_id = 0;
  const T *kb, *vb;
  if (!is_ctx) {
    const int t = gw / a.kv_heads;
    hk = gw % a.kv_heads;
    const int s = seq_of_row(a.cu, a.num_seqs, t);
    j = t - cu_at(a, s);
    s_lo = s;
    s_hi = s + 1;
    kb = static_cast<const T*>(a.k);
    vb = static_cast<const T*>(a.v);
  } else {
    int64_t c = gw - n_own;
    chunk_id = static_cast<int>(c / (static_cast<int64_t>(a.ctx_len) * a.kv_heads));
    int rem = static_cast<int>(c % (static_cast<int64_t>(a.ctx_len) * a.kv_heads));
    j = rem / a.kv_heads;
    hk = rem % a.kv_heads;
    s_lo = chunk_id * chunk;
    s_hi = min(a.num_seqs, s_lo + chunk);
    kb = static_cast<const T*>(a.k_ctx);
    vb = static_cast<const T*>(a.v_ctx);
  }
  const int64_t krow = is_ctx ? j : (cu_at(a, s_lo) + j);
  const int64_t ko = (krow * a.kv_heads + hk) * D;
  float kr[kMaxPerLane], vr[kMaxPerLane], dk[kMaxPerLane], dv[kMaxPerLane];
#pragma unroll
  for (int i = 0; i < kMaxPerLane; ++i) {
    int e = lane + 32 * i;
    kr[i] = e < D ? ldf(kb + ko + e) : 0.f;
    vr[i] = e < D ? ldf(vb + ko + e) : 0.f;
    dk[i] = 0.f;
    dv[i] = 0.f;
  }
  for (int s = s_lo; s < s_hi; ++s) {
    const int r0 = cu_at(a, s), r1 = cu_at(a, s + 1);
    const int first = is_ctx ? r0 : r0 + j;
    // (query row, head) pairs of the sequence, kKeyBlock at a time (row-major, head fastest)
    const int n_pairs = (r1 - first) * G;
    for (int q0 = 0; q0 < n_pairs; q0 += kKeyBlock) {
      float sp[kKeyBlock], dp[kKeyBlock];
      float qv[kKeyBlock][kMaxPerLane], gv[kKeyBlock][kMaxPerLane];
#pragma unroll
      for (int b = 0; b < kKeyBlock; ++b) {
        sp[b] = 0.f;
        dp[b] = 0.f;
        const bool live = q0 + b < n_pairs;
        const int t = first + (q0 + b) / G, h = hk * G + (q0 + b) % G;
        const int64_t qo = (static_cast<int64_t>(t) * a.heads + h) * D;
#pragma unroll
        for (int i = 0; i < kMaxPerLane; ++i) {
          int e = lane + 32 * i;
          qv[b][i] = (live && e < D) ? ldf(static_cast<const T*>(a.q) + qo + e) : 0.f;
          gv[b][i] = (live && e < D) ? ldf(static_cast<const T*>(a.dout) + qo + e) : 0.f;
          sp[b] += qv[b][i] * kr[i];
          dp[b] += gv[b][i] * vr[i];
        }
      }
      warp_sum_n(sp);
      warp_sum_n(dp);
#pragma unroll
      for (int b = 0; b < kKeyBlock; ++b) {
        if (q0 + b >= n_pairs) break;
        const int t = first + (q0 + b) / G, h = hk * G + (q0 + b) % G;
        const float p = expf(sp[b] * a.scale - a.lse[static_cast<int64_t>(h) * a.total_q + t]);
        const float ds = p * (dp[b] - drow[static_cast<int64_t>(h) * a.total_q + t]) * a.scale;
#pragma unroll
        for (int i = 0; i < kMaxPerLane; ++i) {
          dv[i] += p * gv[b][i];
          dk[i] += ds * qv[b][i];
        }
      }
    }
  }
  if (!is_ctx && own_part) {
    // fp32 [2][rows][Hk][D] (fused Call 1 of a two-call backward: cast once later, with Call 2's)
    const int64_t plane = static_cast<int64_t>(own_rows) * a.kv_heads * D;
#pragma unroll
    for (int i = 0; i < kMaxPerLane; ++i) {
      int e = lane + 32 * i;
      if (e < D) {
        own_part[ko + e] = dk[i];
        own_part[plane + ko + e] = dv[i];
      }
    }
  } else if (!is_ctx) {
#pragma unroll
    for (int i = 0; i < kMaxPerLane; ++i) {
      int e = lane + 32 * i;
      if (e < D) {
        stf(static_cast<T*>(a.dk) + ko + e, dk[i]);
        stf(static_cast<T*>(a.dv) + ko + e, dv[i]);
      }
    }
  } else {
    // fp32 partial for this chunk: [chunk][2][P][Hk][D]
    const int64_t plane = static_cast<int64_t>(a.ctx_len) * a.kv_heads * D;
    float* pk = ctx_part + static_cast<int64_t>(chunk_id) * 2 * plane + ko;
    float* pv = pk + plane;
#pragma unroll
    for (int i = 0; i < kMaxPerLane; ++i) {
      int e = lane + 32 * i;
      if (e < D) {
        pk[e] = dk[i];
        pv[e] = dv[i];
      }
    }
  }
}

// head_dim -> values per lane
template <typename F>
static void by_lanes(int head_dim, F&& f) {
  if (head_dim <= 64)
    f(std::integral_constant<int, 2>{});
  else if (head_dim <= 128)
    f(std::integral_constant<int, 4>{});
  else
    f(std::integral_constant<int, 8>{});
}

void launch_simt_fwd(const SimtArgs& a, cudaStream_t st) {
  const int64_t warps = a.total_q * a.heads;
  if (warps == 0) return;
  const int threads = 256;
  const int64_t blocks = (warps * 32 + threads - 1) / threads;
  by_lanes(a.head_dim, [&](auto pl) {
    if (a.dtype == DKV_F32)
      simt_fwd_kernel<float, decltype(pl)::value><<<blocks, threads, 0, st>>>(a);
    else
      simt_fwd_kernel<__nv_bfloat16, decltype(pl)::value><<<blocks, threads, 0, st>>>(a);
  });
}

void launch_simt_bwd(const SimtArgs& a, const float* drow, int chunk, int num_chunks, float* ctx_part,
                     float* own_part, cudaStream_t st) {
  const int threads = 256;
  const int64_t w1 = a.total_q * a.heads;
  const int64_t w2 = a.total_q * a.kv_heads + a.ctx_len * a.kv_heads * num_chunks;
  by_lanes(a.head_dim, [&](auto pl) {
    constexpr int PL = decltype(pl)::value;
    if (w1 > 0) {
      const int64_t b1 = (w1 * 32 + threads - 1) / threads;
      if (a.dtype == DKV_F32)
        simt_bwd_dq_kernel<float, PL><<<b1, threads, 0, st>>>(a, drow);
      else
        simt_bwd_dq_kernel<__nv_bfloat16, PL><<<b1, threads, 0, st>>>(a, drow);
    }
    if (w2 > 0) {
      const int64_t b2 = (w2 * 32 + threads - 1) / threads;
      if (a.dtype == DKV_F32)
        simt_bwd_dkv_kernel<float, PL><<<b2, threads, 0, st>>>(a, drow, static_cast<int>(a.total_q), chunk,
                                                               num_chunks, ctx_part, own_part);
      else
        simt_bwd_dkv_kernel<__nv_bfloat16, PL><<<b2, threads, 0, st>>>(a, drow, static_cast<int>(a.total_q),
                                                                       chunk, num_chunks, ctx_part, own_part);
    }
  });
}

}  // namespace dkv
