// dkv_abi.cu -- the extern "C" boundary of libdkv.so (declared in include/dkv.h).
//
// Validates the same contract the reference raises ValueError for
// (kernel.py:75-110, :214-218; fa2.py:69-87, :272-275) on the scalar/pointer
// level -- the Python layer additionally validates host-side cu_seqlens
// values -- then dispatches to the tcgen05 kernels (bf16, d in {64,128},
// G | 128) or the fp32 SIMT kernels, all stream-ordered on `stream`.
#include <algorithm>
#include <cstdio>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "dkv_internal.h"

#include <cstdlib>

namespace dkv {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

bool ensure_smem_optin(const void* kernel, int bytes, const char* name) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    set_error(std::string(name) + ": cudaGetDevice failed");
    return false;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({kernel, dev})) return true;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    set_error(std::string(name) + ": cudaFuncSetAttribute(max dynamic smem) failed: " + cudaGetErrorString(e));
    return false;
  }
  done.insert({kernel, dev});
  return true;
}

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

// SIMT path of the two-call launches: Call 1 (the prompt's self-attention) runs on a side stream
// forked from and joined back into the caller's stream, so its small latency-bound grids overlap
// Call 2's (the tensor-core path fuses both into one launch instead).  One side stream and one
// fork / join event pair per (host thread, device): no state is shared between threads.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static SideStream* side_stream(cudaStream_t st) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return nullptr;
  thread_local std::vector<SideStream> cache;  // (created once, kept for the thread's lifetime)
  if (dev >= static_cast<int>(cache.size())) cache.resize(dev + 1);
  SideStream& x = cache[dev];
  if (!x.s) {
    // never create it inside a stream capture (the fork / join themselves are capture-safe)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return nullptr;
    }
    if (cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      x = SideStream{};
      return nullptr;  // fall back to running Call 1 on the caller's stream
    }
  }
  return &x;
}
static cudaStream_t fork_side(SideStream* sd, cudaStream_t st) {
  if (!sd) return st;
  cudaEventRecord(sd->fork, st);
  cudaStreamWaitEvent(sd->s, sd->fork, 0);
  return sd->s;
}
static void join_side(SideStream* sd, cudaStream_t st) {
  if (!sd) return;
  cudaEventRecord(sd->join, sd->s);
  cudaStreamWaitEvent(st, sd->join, 0);
}

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

// The launch's prompt groups (dkv_group_table, include/dkv.h).  `tc`: the tensor-core kernels
// serve this shape (multi-group launches need them).  Without `fn` (workspace queries) an
// invalid table silently degrades to one group -- the launch itself then reports the error.
template <typename P>
static int parse_groups(const P* p, bool dualkv, bool tc, GroupTable& g, const char* fn) {
  const dkv_group_table& t = p->groups;
  auto bad = [&](const std::string& why) { return fn ? fail(DKV_ERR_INVALID, std::string(fn) + ": " + why) : -1; };
  g.n = 1;
  g.seq[0] = 0;
  g.seq[1] = static_cast<int>(p->num_seqs);
  g.ctx[0] = 0;
  g.ctx[1] = static_cast<int>(std::max<int64_t>(0, p->ctx_len));
  g.max_ctx = g.ctx[1];
  g.max_seqs = g.seq[1];
  if (t.num_groups == 0 || t.num_groups == 1) {
    if (t.num_groups == 1 && t.seq_cu && t.ctx_cu &&
        (t.seq_cu[0] != 0 || t.seq_cu[1] != p->num_seqs || t.ctx_cu[0] != 0 || t.ctx_cu[1] != p->ctx_len))
      return bad("group table inconsistent with num_seqs / ctx_len");
    return DKV_OK;
  }
  if (t.num_groups < 0 || t.num_groups > DKV_MAX_GROUPS)
    return bad("num_groups must be in [0, " + std::to_string(DKV_MAX_GROUPS) + "]");
  if (!dualkv) return bad("a varlen call takes no group table");
  if (!t.seq_cu || !t.ctx_cu) return bad("null group table arrays");
  if (!tc && fn)
    return fail(DKV_ERR_UNSUPPORTED, std::string(fn) +
                                         ": multi-group launches run on the tensor-core path only (bf16, "
                                         "head_dim 64/128)");
  const int n = static_cast<int>(t.num_groups);
  if (t.seq_cu[0] != 0 || t.seq_cu[n] != p->num_seqs)
    return bad("group seq_cu must run from 0 to num_seqs");
  if (t.ctx_cu[0] != 0 || t.ctx_cu[n] != p->ctx_len) return bad("group ctx_cu must run from 0 to ctx_len");
  g.n = n;
  g.max_ctx = 0;
  g.max_seqs = 0;
  for (int i = 0; i <= n; ++i) {
    g.seq[i] = t.seq_cu[i];
    g.ctx[i] = t.ctx_cu[i];
    if (i == 0) continue;
    if (g.seq[i] <= g.seq[i - 1]) return bad("every group needs at least one sequence (seq_cu increasing)");
    if (g.ctx[i] < g.ctx[i - 1]) return bad("group ctx_cu must be non-decreasing");
    g.max_ctx = std::max(g.max_ctx, g.ctx[i] - g.ctx[i - 1]);
    g.max_seqs = std::max(g.max_seqs, g.seq[i] - g.seq[i - 1]);
  }
  return DKV_OK;
}

static int fwd_impl(const dkv_fwd_params* p, bool dualkv, void* stream, const char* fn) {
  int rc = validate_common(p, dualkv, fn);
  if (rc) return rc;
  if (p->total_q > 0 && (!p->out || !p->lse)) return fail(DKV_ERR_INVALID, std::string(fn) + ": null out/lse");
  SimtArgs a = to_args(p);
  a.out = p->out;
  a.lse = p->lse;
  const bool tc = tc_supported(a.dtype, a.head_dim, a.heads, a.kv_heads);
  GroupTable grp;
  rc = parse_groups(p, dualkv, tc, grp, fn);
  if (rc) return rc;
  auto st = static_cast<cudaStream_t>(stream);
  if (a.total_q == 0) return DKV_OK;
  prof_main_begin(0, st);
  if (tc) {
    rc = launch_tc_fwd(a, nullptr, grp, st);
    if (rc) return rc;
  } else {
    launch_simt_fwd(a, st);
  }
  prof_main_end(0, st);
  prof_count(1);
  return check_launch(fn);
}

// SM count of the current device (queried once per device; B200: 148)
static int sm_count() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
  std::lock_guard<std::mutex> lock(mu);
  if (static_cast<int>(cache.size()) <= dev) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

// context work chunk (sequences per context work unit) for the tensor-core backward
// (chunks never span groups: a chunk is `chunk` consecutive sequences of ONE group)
static int auto_chunk(const dkv_bwd_params* p, const GroupTable& g) {
  const int64_t nmax = std::max(1, g.max_seqs);
  if (p->ctx_chunk > 0) return static_cast<int>(std::min<int64_t>(p->ctx_chunk, nmax));
  {
    static const int env_chunk = [] {  // DKV_CTX_CHUNK: tuning experiments only
      const char* e = getenv("DKV_CTX_CHUNK");
      return e ? atoi(e) : 0;
    }();
    if (env_chunk > 0) return static_cast<int>(std::min<int64_t>(env_chunk, nmax));
  }
  if (p->ctx_len == 0) return static_cast<int>(nmax);
  const bool tc = tc_bwd_supported(p->dtype, static_cast<int>(p->head_dim), static_cast<int>(p->heads),
                                   static_cast<int>(p->kv_heads));
  // SIMT: a warp per (prompt key, kv head, chunk) walks the chunk's query rows serially; up to 16
  // chunks (one sequence each for N <= 16) keep those warps short, folded in fixed order
  if (!tc) return static_cast<int>((nmax + 15) / 16);
  // enough context units to fill ~8 waves of the SMs, but no more than needed
  const int64_t n_ctx_tiles = (g.max_ctx + 127) / 128;
  const int64_t units_per_chunk = std::max<int64_t>(1, n_ctx_tiles * p->kv_heads * g.n);
  int64_t chunks = (static_cast<int64_t>(sm_count()) * 8 + units_per_chunk - 1) / units_per_chunk;
  chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, nmax));
  return static_cast<int>((nmax + chunks - 1) / chunks);
}

// dpack row padding: per-KV-head row stride a multiple of 4 tokens (16 B TMA stride)
static int dpack_tpad(size_t T) { return static_cast<int>((T + 3) & ~size_t(3)); }

struct BwdLayout {
  size_t drow, xsplit, dq_acc, drow_s, xsplit_s, dq_acc_s, ctx, total;
  int chunk, num_chunks, num_parts, self_part;
  bool tc, atomic;
};

// Scratch of one backward launch.  `with_self`: the two-call launch, where Call 1 (the prompt's
// causal self-attention) runs in the same launch and adds into the same fp32 prompt scratch.
static BwdLayout bwd_layout(const dkv_bwd_params* p, const GroupTable& g, bool with_self) {
  BwdLayout L{};
  const size_t T = static_cast<size_t>(std::max<int64_t>(0, p->total_q));
  const size_t H = static_cast<size_t>(p->heads), Hk = static_cast<size_t>(std::max<int64_t>(1, p->kv_heads));
  const size_t D = static_cast<size_t>(p->head_dim), P = static_cast<size_t>(std::max<int64_t>(0, p->ctx_len));
  with_self = with_self && P > 0;
  L.chunk = auto_chunk(p, g);
  L.num_chunks = static_cast<int>((std::max(1, g.max_seqs) + L.chunk - 1) / L.chunk);
  L.tc = tc_bwd_supported(p->dtype, static_cast<int>(p->head_dim), static_cast<int>(p->heads),
                          static_cast<int>(p->kv_heads));
  const int writers = L.num_chunks + (with_self ? 1 : 0);  // independent writers of prompt gradients
  // atomic accumulation into one fp32 plane unless the caller wants ordered / per-chunk partials
  L.atomic = L.tc && !p->deterministic && !p->ctx_partials && writers > 1;
  L.num_parts = L.atomic ? 1 : writers;
  L.self_part = L.atomic ? 0 : L.num_chunks;
  size_t off = 0;
  L.drow = off;
  off += L.tc ? 0 : align256(H * T * 4);
  L.xsplit = off;  // H * tpad rows of 32 bf16
  off += L.tc ? align256(H * static_cast<size_t>(dpack_tpad(T)) * 64) : 0;
  L.dq_acc = off;
  off += L.tc ? align256(T * H * D * 4) : 0;
  L.drow_s = off;
  off += (with_self && !L.tc) ? align256(H * P * 4) : 0;
  L.xsplit_s = off;
  off += (with_self && L.tc) ? align256(H * static_cast<size_t>(dpack_tpad(P)) * 64) : 0;
  L.dq_acc_s = off;
  off += (with_self && L.tc) ? align256(P * H * D * 4) : 0;
  L.ctx = off;
  off += (p->ctx_partials ? 0 : align256(static_cast<size_t>(L.num_parts) * 2 * P * Hk * D * 4));
  L.total = off;
  return L;
}

static int bwd_impl(const dkv_bwd_params* p, const CtxSelf* self, void* ws, size_t ws_bytes, bool dualkv,
                    void* stream, const char* fn) {
  int rc = validate_common(p, dualkv, fn);
  if (rc) return rc;
  if (p->total_q > 0 && (!p->out || !p->lse || !p->dout || !p->dq || !p->dk || !p->dv))
    return fail(DKV_ERR_INVALID, std::string(fn) + ": null out/lse/dout/dq/dk/dv");
  if (p->ctx_len > 0 && (!p->dk_ctx || !p->dv_ctx)) return fail(DKV_ERR_INVALID, std::string(fn) + ": null dk_ctx/dv_ctx");
  if (self && p->ctx_len > 0 && (!self->q || !self->out || !self->lse || !self->dout || !self->dq))
    return fail(DKV_ERR_INVALID, std::string(fn) + ": null q_ctx/out_ctx/lse_ctx/dout_ctx/dq_ctx");
  const bool with_self = self && p->ctx_len > 0;
  GroupTable grp;
  rc = parse_groups(p, dualkv,
                    tc_bwd_supported(p->dtype, static_cast<int>(p->head_dim), static_cast<int>(p->heads),
                                     static_cast<int>(p->kv_heads)),
                    grp, fn);
  if (rc) return rc;
  if (grp.n > 1 && p->ctx_partials)
    return fail(DKV_ERR_INVALID, std::string(fn) + ": ctx_partials is a one-group instrumentation hook");
  BwdLayout L = bwd_layout(p, grp, with_self);
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
  // the fused Call 1 problem: the prompt's own queries, keys = the context tensors
  SimtArgs s = a;
  if (with_self) {
    s.q = self->q;
    s.k = p->k_ctx;
    s.v = p->v_ctx;
    s.out = self->out;
    s.lse = self->lse;
    s.dout = self->dout;
    s.dq = self->dq;
    s.total_q = static_cast<int>(p->ctx_len);
    s.num_seqs = 1;
    s.max_seqlen = static_cast<int>(p->ctx_len);
    s.ctx_len = 0;
    s.cu = nullptr;  // one sequence: the prompt
  }
  const int64_t plane = p->ctx_len * p->kv_heads * p->head_dim;
  const size_t esz = a.dtype == DKV_F32 ? 4 : 2;
  float* ctx = p->ctx_partials ? p->ctx_partials : reinterpret_cast<float*>(w + L.ctx);
  if (a.total_q == 0 && !with_self) {
    // no queries: every gradient is zero (test_dualkv.py:96-102)
    if (plane > 0) {
      cudaMemsetAsync(p->dk_ctx, 0, plane * esz, st);
      cudaMemsetAsync(p->dv_ctx, 0, plane * esz, st);
      if (p->ctx_partials) cudaMemsetAsync(p->ctx_partials, 0, L.num_chunks * 2 * plane * 4, st);
      if (p->ctx_grad_f32) cudaMemsetAsync(p->ctx_grad_f32, 0, 2 * plane * 4, st);
    }
    return check_launch(fn);
  }
  // parts nobody writes (chunks of empty responses) must read as zero
  if (plane > 0) cudaMemsetAsync(ctx, 0, static_cast<size_t>(L.num_parts) * 2 * plane * 4, st);
  if (L.tc) {
    BwdScratch sc{};
    sc.dq_acc = reinterpret_cast<float*>(w + L.dq_acc);
    sc.xsplit = reinterpret_cast<__nv_bfloat16*>(w + L.xsplit);
    sc.tpad = dpack_tpad(static_cast<size_t>(a.total_q));
    sc.ctx_acc = ctx;
    sc.chunk = L.chunk;
    sc.num_chunks = L.num_chunks;
    sc.self_part = L.self_part;
    sc.atomic_ctx = L.atomic;
    if (a.total_q > 0) {
      cudaMemsetAsync(sc.dq_acc, 0, static_cast<size_t>(a.total_q) * a.heads * a.head_dim * 4, st);
      launch_rowsum_do_o(a, nullptr, const_cast<__nv_bfloat16*>(sc.xsplit), sc.tpad, st);
      prof_count(1);
    }
    if (with_self) {
      sc.dq_acc_s = reinterpret_cast<float*>(w + L.dq_acc_s);
      sc.xsplit_s = reinterpret_cast<__nv_bfloat16*>(w + L.xsplit_s);
      sc.tpad_s = dpack_tpad(static_cast<size_t>(p->ctx_len));
      cudaMemsetAsync(sc.dq_acc_s, 0, static_cast<size_t>(p->ctx_len) * a.heads * a.head_dim * 4, st);
      launch_rowsum_do_o(s, nullptr, const_cast<__nv_bfloat16*>(sc.xsplit_s), sc.tpad_s, st);
      prof_count(1);
    }
    prof_main_begin(1, st);
    rc = launch_tc_bwd(a, with_self ? self : nullptr, grp, sc, st);
    if (rc) return rc;
    prof_main_end(1, st);
    // the kernel accumulates dQ / softmax_scale (the scale is folded into this single cast)
    if (a.total_q > 0) {
      launch_convert(sc.dq_acc, p->dq, a.dtype, static_cast<int64_t>(a.total_q) * a.heads * a.head_dim, st, a.scale);
      prof_count(1);
    }
    if (with_self) {
      launch_convert(sc.dq_acc_s, self->dq, a.dtype, plane / p->kv_heads * p->heads, st, a.scale);
      prof_count(1);
    }
    prof_count(1);
  } else {
    float* drow = reinterpret_cast<float*>(w + L.drow);
    prof_main_begin(1, st);
    SideStream* sd = with_self && a.total_q > 0 ? side_stream(st) : nullptr;
    const cudaStream_t st1 = fork_side(sd, st);  // Call 1 beside Call 2 (disjoint outputs / parts)
    if (a.total_q > 0) {
      launch_rowsum_do_o(a, drow, nullptr, 0, st);
      launch_simt_bwd(a, drow, L.chunk, L.num_chunks, ctx, nullptr, st);
      prof_count(3);
    }
    if (with_self) {
      // Call 1's prompt-key gradient lands in fp32 as the last part: still one cast in total
      float* drow_s = reinterpret_cast<float*>(w + L.drow_s);
      launch_rowsum_do_o(s, drow_s, nullptr, 0, st1);
      launch_simt_bwd(s, drow_s, 1, 1, nullptr, ctx + static_cast<int64_t>(L.self_part) * 2 * plane, st1);
      prof_count(3);
    }
    join_side(sd, st);
    prof_main_end(1, st);
  }
  if (plane > 0) {
    launch_fold_convert(ctx, L.num_parts, plane, p->dk_ctx, p->dv_ctx, a.dtype, p->ctx_grad_f32, st);
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

static GroupTable groups_of(const dkv_bwd_params* p) {
  GroupTable g;
  parse_groups(p, true, true, g, nullptr);
  return g;
}

size_t dkv_bwd_workspace_size(const dkv_bwd_params* p) {
  if (!p) return 0;
  return bwd_layout(p, groups_of(p), false).total;
}
int64_t dkv_bwd_num_ctx_chunks(const dkv_bwd_params* p) {
  if (!p) return 0;
  return bwd_layout(p, groups_of(p), false).num_chunks;
}
int32_t dkv_dualkv_bwd(const dkv_bwd_params* p, void* ws, size_t ws_bytes, void* stream) {
  return bwd_impl(p, nullptr, ws, ws_bytes, true, stream, "dkv_dualkv_bwd");
}
int32_t dkv_varlen_bwd(const dkv_bwd_params* p, void* ws, size_t ws_bytes, void* stream) {
  return bwd_impl(p, nullptr, ws, ws_bytes, false, stream, "dkv_varlen_bwd");
}

int32_t dkv_twocall_fwd(const dkv_twocall_fwd_params* p, void* stream) {
  if (!p) return fail(DKV_ERR_INVALID, "dkv_twocall_fwd: null params");
  const dkv_fwd_params* c = &p->call2;
  int rc = validate_common(c, true, "dkv_twocall_fwd");
  if (rc) return rc;
  if (c->total_q > 0 && (!c->out || !c->lse)) return fail(DKV_ERR_INVALID, "dkv_twocall_fwd: null out/lse");
  if (c->ctx_len > 0 && (!p->q_ctx || !p->out_ctx || !p->lse_ctx))
    return fail(DKV_ERR_INVALID, "dkv_twocall_fwd: null q_ctx/out_ctx/lse_ctx");
  SimtArgs a = to_args(c);
  a.out = c->out;
  a.lse = c->lse;
  const bool tc = tc_supported(a.dtype, a.head_dim, a.heads, a.kv_heads);
  GroupTable grp;
  rc = parse_groups(c, true, tc, grp, "dkv_twocall_fwd");
  if (rc) return rc;
  auto st = static_cast<cudaStream_t>(stream);
  CtxSelf self{p->q_ctx, p->out_ctx, p->lse_ctx, nullptr, nullptr};
  prof_main_begin(0, st);
  if (tc) {
    rc = launch_tc_fwd(a, c->ctx_len > 0 ? &self : nullptr, grp, st);
    if (rc) return rc;
  } else {
    SideStream* sd = c->ctx_len > 0 && a.total_q > 0 ? side_stream(st) : nullptr;
    const cudaStream_t st1 = fork_side(sd, st);  // Call 1 beside Call 2
    if (a.total_q > 0) launch_simt_fwd(a, st);
    if (c->ctx_len > 0) {
      SimtArgs s = a;
      s.q = p->q_ctx;
      s.k = c->k_ctx;
      s.v = c->v_ctx;
      s.out = p->out_ctx;
      s.lse = p->lse_ctx;
      s.total_q = static_cast<int>(c->ctx_len);
      s.num_seqs = 1;
      s.max_seqlen = s.total_q;
      s.ctx_len = 0;
      s.cu = nullptr;  // one sequence: the prompt
      launch_simt_fwd(s, st1);
    }
    join_side(sd, st);
  }
  prof_main_end(0, st);
  prof_count(1);
  return check_launch("dkv_twocall_fwd");
}

size_t dkv_twocall_bwd_workspace_size(const dkv_twocall_bwd_params* p) {
  if (!p) return 0;
  return bwd_layout(&p->call2, groups_of(&p->call2), true).total;
}

int32_t dkv_twocall_bwd(const dkv_twocall_bwd_params* p, void* ws, size_t ws_bytes, void* stream) {
  if (!p) return fail(DKV_ERR_INVALID, "dkv_twocall_bwd: null params");
  if (p->call2.ctx_partials) return fail(DKV_ERR_INVALID, "dkv_twocall_bwd: ctx_partials is not supported");
  CtxSelf self{p->q_ctx, const_cast<void*>(p->out_ctx), const_cast<float*>(p->lse_ctx), p->dout_ctx, p->dq_ctx};
  return bwd_impl(&p->call2, &self, ws, ws_bytes, true, stream, "dkv_twocall_bwd");
}

}  // extern "C"
