// dkv_internal.h -- declarations shared by the libdkv translation units.
#pragma once
#include <cstdint>
#include <string>

#include "../../include/dkv.h"
#include "common.cuh"

namespace dkv {

// flattened problem description used by every kernel family
struct SimtArgs {
  const void* q;
  const void* k_ctx;
  const void* v_ctx;
  const void* k;
  const void* v;
  const int32_t* cu;  // null: one sequence of total_q rows
  void* out;
  float* lse;
  const void* dout;
  void* dq;
  void* dk;
  void* dv;
  int num_seqs;
  int total_q;
  int ctx_len;
  int heads;
  int kv_heads;
  int head_dim;
  int max_seqlen;
  float scale;
  int dtype;
};

void set_error(const std::string& msg);

// Opt a kernel into `bytes` of dynamic shared memory on the CURRENT device, once per
// (kernel, device); thread-safe.  Returns false (error recorded) if the driver refuses.
bool ensure_smem_optin(const void* kernel, int bytes, const char* name);

// Call 1 of the two-call decomposition fused into a Call 2 launch: the prompt's own queries
// (rows [0, ctx_len) of q/out/dout/dq below) attend causally to the context keys.
struct CtxSelf {
  const void* q;     // [P, H, d]
  void* out;         // [P, H, d]
  float* lse;        // [H, P]
  const void* dout;  // backward only
  void* dq;          // backward only
};

// Prompt groups of one launch (the C ABI's dkv_group_table, validated, with derived maxima).
// Passed by value inside the kernel parameters (~2 KB); one group = {0, num_seqs} / {0, ctx_len}.
struct GroupTable {
  int n;                       // number of groups (>= 1)
  int max_ctx;                 // max prompt rows of a group
  int max_seqs;                // max sequences of a group
  int seq[DKV_MAX_GROUPS + 1]; // sequence ranges
  int ctx[DKV_MAX_GROUPS + 1]; // prompt row ranges in k_ctx / v_ctx / q_ctx
  // group of sequence s (binary search; a single group is the common case)
  __host__ __device__ int group_of(int s) const {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (seq[mid] <= s)
        lo = mid;
      else
        hi = mid - 1;
    }
    return lo;
  }
};

// profiling hooks (dkv_abi.cu): kind 0 = forward main kernel, 1 = backward main kernel
void prof_main_begin(int kind, cudaStream_t st);
void prof_main_end(int kind, cudaStream_t st);
void prof_count(int launches);

// simt_attn.cu
void launch_simt_fwd(const SimtArgs& a, cudaStream_t st);
// own_part (may be null): write own-row dK/dV as fp32 [2][rows][Hk][D] instead of storage dtype
void launch_simt_bwd(const SimtArgs& a, const float* drow, int chunk, int num_chunks, float* ctx_part,
                     float* own_part, cudaStream_t st);

// aux.cu
// D = rowsum(dO*O) into drow [H][T] (SIMT path) and/or the tensor-core path's split-bf16
// additive-constant rows xsplit [Hk][tpad][G][32] (tpad >= T padding tokens, zero rows)
void launch_rowsum_do_o(const SimtArgs& a, float* drow, __nv_bfloat16* xsplit, int tpad, cudaStream_t st);
// f32_out (may be null): also store the folded fp32 sums [2][plane] before the cast
void launch_fold_convert(const float* partials, int num_parts, int64_t plane, void* dk, void* dv, int dtype,
                         float* f32_out, cudaStream_t st);
void launch_convert(const float* src, void* dst, int dtype, int64_t n, cudaStream_t st, float scale = 1.f);

// sm100 tensor-core paths (fwd_sm100.cu / bwd_sm100.cu)
bool force_simt();  // DKV_FORCE_SIMT=1: route everything to the SIMT kernels (cross-checks)
bool tc_supported(int dtype, int head_dim, int heads, int kv_heads);
bool tc_bwd_supported(int dtype, int head_dim, int heads, int kv_heads);
int launch_tc_fwd(const SimtArgs& a, const CtxSelf* self, const GroupTable& grp, cudaStream_t st);
// Backward scratch: dq_acc [T,H,D] f32 (pre-zeroed; accumulates dQ / softmax_scale), xsplit from
// launch_rowsum_do_o; the *_s fields are the fused Call 1's (prompt rows); ctx_acc f32
// [parts][2][P][Hk][D] pre-zeroed: chunk c (of every group) writes part c (or every item red.adds
// part 0 when atomic_ctx), fused Call 1 items write part self_part.
struct BwdScratch {
  float* dq_acc;
  const __nv_bfloat16* xsplit;
  int tpad;
  float* dq_acc_s;
  const __nv_bfloat16* xsplit_s;
  int tpad_s;
  float* ctx_acc;
  int chunk, num_chunks, self_part;
  bool atomic_ctx;
};
int launch_tc_bwd(const SimtArgs& a, const CtxSelf* self, const GroupTable& grp, const BwdScratch& w,
                  cudaStream_t st);
// bwd_pair_sm100.cu: the CTA-pair backward (head_dim 128, G | 32), opt-in (DKV_BWD_PAIR=1)
bool tc_bwd_pair_supported(int head_dim, int heads, int kv_heads);
int launch_tc_bwd_pair(const SimtArgs& a, const CtxSelf* self, const GroupTable& grp, const BwdScratch& w,
                       cudaStream_t st);

}  // namespace dkv
