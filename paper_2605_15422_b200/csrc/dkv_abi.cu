// dkv_abi.cu -- the extern "C" boundary of libdkv.so (declared in include/dkv.h).
//
// Validates the same contract the reference raises ValueError for
// (kernel.py:75-110, :214-218; fa2.py:69-87, :272-275) on the scalar/pointer
// level -- the Python layer additionally validates host-side cu_seqlens
// values -- then dispatches to the tcgen05 kernels (bf16, d in {64,128},
// G | 128) or the fp32 SIMT kernels, all stream-ordered on `stream`.
#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include "dkv_internal.h"

namespace dkv {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

// ---- profiling hooks (bench harness only; off by default)
struct ProfState {
  bool on = false;
  int launches = 0;
  std::vector<std::pair<int, cudaEvent_t>> ev;  // (kind*2 + is_end, event)
};
static ProfState g_prof;

void prof_main_begin(int kind, cudaStream_t st) {
  if (!g_prof.on) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  g_prof.ev.push_back({kind * 2, e});
}
void prof_main_end(int kind, cudaStream_t st) {
  if (!g_prof.on) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  g_prof.ev.push_back({kind * 2 + 1, e});
}
void prof_count(int launches) {
  if (g_prof.on) g_prof.launches += launches;
}

static int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

static int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DKV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return DKV_OK;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

template <typename P>
static int validate_common(const P* p, bool dualkv, const char* fn) {
  if (!p) return fail(DKV_ERR_INVALID, std::string(fn) + ": null params");
  if (p->dtype != DKV_BF16 && p->dtype != DKV_F32) return fail(DKV_ERR_INVALID, std::string(fn) + ": unknown dtype");
  if (p->num_seqs < 1) return fail(DKV_ERR_INVALID, std::string(fn) + ": malformed cu_seqlens (need N >= 1)");
  if (p->total_q < 0) return fail(DKV_ERR_INVALID, std::string(fn) + ": negative token count");
  if (p->ctx_len < 0) return fail(DKV_ERR_INVALID, std::string(fn) + ": context_seqlen must be non-negative");
  if (!dualkv && p->ctx_len != 0) return fail(DKV_ERR_INVALID, std::string(fn) + ": varlen call takes no context");
  if (p->kv_heads <= 0 || p->heads <= 0 || p->heads % p->kv_heads)
    return fail(DKV_ERR_INVALID, std::string(fn) + ": H=" + std::to_string(p->heads) +
                                     " must be a positive multiple of H_k=" + std::to_string(p->kv_heads));
  if (p->head_dim < 1 || p->head_dim > 256)
    return fail(DKV_ERR_UNSUPPORTED, std::string(fn) + ": head_dim must be in [1, 256]");
  if (p->max_seqlen < 0) return fail(DKV_ERR_INVALID, std::string(fn) + ": negative max_seqlen");
  if (p->total_q > 0x7fffffff / std::max<int64_t>(1, p->heads) || p->ctx_len > 0x7fffffff)
    return fail(DKV_ERR_UNSUPPORTED, std::string(fn) + ": problem too large for 32-bit row indexing");
  if (!(p->softmax_scale > 0.f)) return fail(DKV_ERR_INVALID, std::string(fn) + ": softmax_scale must be > 0");
  if (!p->cu_seqlens) return fail(DKV_ERR_INVALID, std::string(fn) + ": null cu_seqlens");
  if (p->total_q > 0 && (!p->q || !p->k || !p->v))
    return fail(DKV_ERR_INVALID, std::string(fn) + ": null q/k/v");
  if (p->ctx_len > 0 && (!p->k_ctx || !p->v_ctx))
    return fail(DKV_ERR_INVALID, std::string(fn) + ": null k_context/v_context");
  return DKV_OK;
}

template <typename P>
static SimtArgs to_args(const P* p) {
  SimtArgs a{};
  a.q = p->q;
  a.k_ctx = p->k_ctx;
  a.v_ctx = p->v_ctx;
  a.k = p->k;
  a.v = p->v;
  a.cu = p->cu_seqlens;
  a.num_seqs = static_cast<int>(p->num_seqs);
  a.total_q = static_cast<int>(p->total_q);
  a.ctx_len = static_cast<int>(p->ctx_len);
  a.heads = static_cast<int>(p->heads);
  a.kv_heads = static_cast<int>(p->kv_heads);
  a.head_dim = static_cast<int>(p->head_dim);
  a.max_seqlen = static_cast<int>(p->max_seqlen);
  a.scale = p->softmax_scale;
  a.dtype = p->dtype;
  return a;
}

static int fwd_impl(const dkv_fwd_params* p, bool dualkv, void* stream, const char* fn) {
  int rc = validate_common(p, dualkv, fn);
  if (rc) return rc;
  if (p->total_q > 0 && (!p->out || !p->lse)) return fail(DKV_ERR_INVALID, std::string(fn) + ": null out/lse");
  SimtArgs a = to_args(p);
  a.out = p->out;
  a.lse = p->lse;
  auto st = static_cast<cudaStream_t>(stream);
  if (a.total_q == 0) return DKV_OK;
  prof_main_begin(0, st);
  if (tc_supported(a.dtype, a.head_dim, a.heads, a.kv_heads)) {
    rc = launch_tc_fwd(a, st);
    if (rc) return rc;
  } else {
    launch_simt_fwd(a, st);
  }
  prof_main_end(0, st);
  prof_count(1);
  return check_launch(fn);
}

// context work chunk (sequences per context work unit) for the tensor-core backward
static int auto_chunk(const dkv_bwd_params* p) {
  if (p->ctx_chunk > 0) return static_cast<int>(std::min<int64_t>(p->ctx_chunk, p->num_seqs));
  if (p->ctx_len == 0) return static_cast<int>(p->num_seqs);
  const bool tc = tc_bwd_supported(p->dtype, static_cast<int>(p->head_dim), static_cast<int>(p->heads),
                                   static_cast<int>(p->kv_heads));
  if (!tc) return static_cast<int>(p->num_seqs);  // SIMT: one ordered fold over all sequences
  // enough context units to fill ~8 waves of 148 SMs, but no more than needed
  const int64_t n_ctx_tiles = (p->ctx_len + 127) / 128;
  const int64_t units_per_chunk = n_ctx_tiles * p->kv_heads;
  int64_t chunks = (148 * 8 + units_per_chunk - 1) / units_per_chunk;
  chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, p->num_seqs));
  return static_cast<int>((p->num_seqs + chunks - 1) / chunks);
}

// dpack row padding: per-KV-head row stride a multiple of 4 tokens (16 B TMA stride)
static int dpack_tpad(size_t T) { return static_cast<int>((T + 3) & ~size_t(3)); }

struct BwdLayout {
  size_t drow, dpack, dq_acc, ctx, total;
  int chunk, num_chunks, num_parts;
};

static BwdLayout bwd_layout(const dkv_bwd_params* p) {
  BwdLayout L{};
  const size_t T = static_cast<size_t>(std::max<int64_t>(0, p->total_q));
  const size_t H = static_cast<size_t>(p->heads), Hk = static_cast<size_t>(std::max<int64_t>(1, p->kv_heads));
  const size_t D = static_cast<size_t>(p->head_dim), P = static_cast<size_t>(p->ctx_len);
  L.chunk = auto_chunk(p);
  L.num_chunks = static_cast<int>((p->num_seqs + L.chunk - 1) / L.chunk);
  const bool tc = tc_bwd_supported(p->dtype, static_cast<int>(p->head_dim), static_cast<int>(p->heads),
                                   static_cast<int>(p->kv_heads));
  // atomic accumulation into one fp32 plane unless the caller wants ordered / per-chunk partials
  L.num_parts = (tc && !p->deterministic && !p->ctx_partials) ? 1 : L.num_chunks;
  size_t off = 0;
  L.drow = off;
  off += align256(H * T * 4);
  L.dpack = off;  // xsplit: H * tpad rows of 32 bf16
  off += align256(H * static_cast<size_t>(dpack_tpad(T)) * 64);
  L.dq_acc = off;
  off += tc ? align256(T * H * D * 4) : 0;
  L.ctx = off;
  off += (p->ctx_partials ? 0 : align256(static_cast<size_t>(L.num_parts) * 2 * P * Hk * D * 4));
  L.total = off;
  return L;
}

static int bwd_impl(const dkv_bwd_params* p, void* ws, size_t ws_bytes, bool dualkv, void* stream,
                    const char* fn) {
  int rc = validate_common(p, dualkv, fn);
  if (rc) return rc;
  if (p->total_q > 0 && (!p->out || !p->lse || !p->dout || !p->dq || !p->dk || !p->dv))
    return fail(DKV_ERR_INVALID, std::string(fn) + ": null out/lse/dout/dq/dk/dv");
  if (p->ctx_len > 0 && (!p->dk_ctx || !p->dv_ctx)) return fail(DKV_ERR_INVALID, std::string(fn) + ": null dk_ctx/dv_ctx");
  BwdLayout L = bwd_layout(p);
  if (ws_bytes < L.total || (L.total > 0 && !ws))
    return fail(DKV_ERR_WORKSPACE, std::string(fn) + ": workspace too small (need " + std::to_string(L.total) + ")");
  auto st = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  SimtArgs a = to_args(p);
  a.out = const_cast<void*>(p->out);
  a.lse = const_cast<float*>(p->lse);
  a.dout = p->dout;
  a.dq = p->dq;
  a.dk = p->dk;
  a.dv = p->dv;
  const int64_t plane = p->ctx_len * p->kv_heads * p->head_dim;
  float* ctx = p->ctx_partials ? p->ctx_partials : reinterpret_cast<float*>(w + L.ctx);
  const bool tc = tc_bwd_supported(a.dtype, a.head_dim, a.heads, a.kv_heads);
  if (a.total_q == 0) {
    // no queries: every gradient is zero (test_dualkv.py:96-102)
    if (plane > 0) {
      cudaMemsetAsync(p->dk_ctx, 0, plane * (a.dtype == DKV_F32 ? 4 : 2), st);
      cudaMemsetAsync(p->dv_ctx, 0, plane * (a.dtype == DKV_F32 ? 4 : 2), st);
      if (p->ctx_partials) cudaMemsetAsync(p->ctx_partials, 0, L.num_chunks * 2 * plane * 4, st);
    }
    return check_launch(fn);
  }
  float* drow = reinterpret_cast<float*>(w + L.drow);
  float* dpack = reinterpret_cast<float*>(w + L.dpack);
  if (tc) {
    float* dq_acc = reinterpret_cast<float*>(w + L.dq_acc);
    cudaMemsetAsync(dq_acc, 0, static_cast<size_t>(a.total_q) * a.heads * a.head_dim * 4, st);
    const bool atomic_ctx = L.num_parts == 1 && L.num_chunks > 1;
    // chunks whose responses are all empty write nothing: start from zero
    if (plane > 0) cudaMemsetAsync(ctx, 0, static_cast<size_t>(L.num_parts) * 2 * plane * 4, st);
    const int tpad = dpack_tpad(static_cast<size_t>(a.total_q));
    __nv_bfloat16* xsplit = reinterpret_cast<__nv_bfloat16*>(dpack);
    launch_rowsum_do_o(a, nullptr, xsplit, tpad, st);
    prof_main_begin(1, st);
    rc = launch_tc_bwd(a, dq_acc, xsplit, tpad, ctx, L.chunk, L.num_chunks, atomic_ctx, st);
    if (rc) return rc;
    prof_main_end(1, st);
    // the kernel accumulates dQ / softmax_scale (the scale is folded into this single cast)
    launch_convert(dq_acc, p->dq, a.dtype, static_cast<int64_t>(a.total_q) * a.heads * a.head_dim, st, a.scale);
    prof_count(3);
  } else {
    launch_rowsum_do_o(a, drow, nullptr, 0, st);
    prof_main_begin(1, st);
    launch_simt_bwd(a, drow, L.chunk, L.num_chunks, ctx, st);
    prof_main_end(1, st);
    prof_count(3);
  }
  if (plane > 0) {
    launch_fold_convert(ctx, L.num_parts, plane, p->dk_ctx, p->dv_ctx, a.dtype, st);
    prof_count(1);
  }
  return check_launch(fn);
}

}  // namespace dkv

using namespace dkv;

extern "C" {

int32_t dkv_abi_version(void) { return DKV_ABI_VERSION; }

int32_t dkv_profile_begin(void) {
  for (auto& e : g_prof.ev) cudaEventDestroy(e.second);
  g_prof.ev.clear();
  g_prof.launches = 0;
  g_prof.on = true;
  return DKV_OK;
}

int32_t dkv_profile_end(double* fwd_ms, int32_t* fwd_launches, double* bwd_ms, int32_t* bwd_launches,
                        int32_t* all_launches) {
  g_prof.on = false;
  double ms[2] = {0, 0};
  int cnt[2] = {0, 0};
  cudaEvent_t open[2] = {nullptr, nullptr};
  for (auto& e : g_prof.ev) {
    const int kind = e.first / 2;
    if ((e.first & 1) == 0) {
      open[kind] = e.second;
    } else if (open[kind]) {
      cudaEventSynchronize(e.second);
      float t = 0.f;
      cudaEventElapsedTime(&t, open[kind], e.second);
      ms[kind] += t;
      cnt[kind] += 1;
      open[kind] = nullptr;
    }
  }
  for (auto& e : g_prof.ev) cudaEventDestroy(e.second);
  g_prof.ev.clear();
  if (fwd_ms) *fwd_ms = ms[0];
  if (fwd_launches) *fwd_launches = cnt[0];
  if (bwd_ms) *bwd_ms = ms[1];
  if (bwd_launches) *bwd_launches = cnt[1];
  if (all_launches) *all_launches = g_prof.launches;
  return check_launch("dkv_profile_end");
}
const char* dkv_last_error(void) { return g_err.c_str(); }
int32_t dkv_uses_tensor_cores(int32_t dtype, int64_t head_dim, int64_t heads, int64_t kv_heads) {
  return tc_supported(dtype, static_cast<int>(head_dim), static_cast<int>(heads), static_cast<int>(kv_heads)) ? 1
                                                                                                              : 0;
}

int32_t dkv_dualkv_fwd(const dkv_fwd_params* p, void* stream) { return fwd_impl(p, true, stream, "dkv_dualkv_fwd"); }
int32_t dkv_varlen_fwd(const dkv_fwd_params* p, void* stream) { return fwd_impl(p, false, stream, "dkv_varlen_fwd"); }

size_t dkv_bwd_workspace_size(const dkv_bwd_params* p) {
  if (!p) return 0;
  return bwd_layout(p).total;
}
int64_t dkv_bwd_num_ctx_chunks(const dkv_bwd_params* p) {
  if (!p) return 0;
  return bwd_layout(p).num_chunks;
}
int32_t dkv_dualkv_bwd(const dkv_bwd_params* p, void* ws, size_t ws_bytes, void* stream) {
  return bwd_impl(p, ws, ws_bytes, true, stream, "dkv_dualkv_bwd");
}
int32_t dkv_varlen_bwd(const dkv_bwd_params* p, void* ws, size_t ws_bytes, void* stream) {
  return bwd_impl(p, ws, ws_bytes, false, stream, "dkv_varlen_bwd");
}

}  // extern "C"
