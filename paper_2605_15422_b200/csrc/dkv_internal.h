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
  const int32_t* cu;
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

// profiling hooks (dkv_abi.cu): kind 0 = forward main kernel, 1 = backward main kernel
void prof_main_begin(int kind, cudaStream_t st);
void prof_main_end(int kind, cudaStream_t st);
void prof_count(int launches);

// simt_attn.cu
void launch_simt_fwd(const SimtArgs& a, cudaStream_t st);
void launch_simt_bwd(const SimtArgs& a, const float* drow, int chunk, int num_chunks, float* ctx_part,
                     cudaStream_t st);

// aux.cu
// D = rowsum(dO*O) into drow [H][T] (SIMT path) and/or the tensor-core path's split-bf16
// additive-constant rows xsplit [Hk][tpad][G][32] (tpad >= T padding tokens, zero rows)
void launch_rowsum_do_o(const SimtArgs& a, float* drow, __nv_bfloat16* xsplit, int tpad, cudaStream_t st);
void launch_fold_convert(const float* partials, int num_parts, int64_t plane, void* dk, void* dv, int dtype,
                         cudaStream_t st);
void launch_convert(const float* src, void* dst, int dtype, int64_t n, cudaStream_t st, float scale = 1.f);

// sm100 tensor-core paths (fwd_sm100.cu / bwd_sm100.cu)
bool force_simt();  // DKV_FORCE_SIMT=1: route everything to the SIMT kernels (cross-checks)
bool tc_supported(int dtype, int head_dim, int heads, int kv_heads);
bool tc_bwd_supported(int dtype, int head_dim, int heads, int kv_heads);
int launch_tc_fwd(const SimtArgs& a, cudaStream_t st);
// dq_acc [T,H,D] f32 (pre-zeroed; holds dQ / softmax_scale), xsplit from launch_rowsum_do_o,
// ctx_acc f32
// [num_parts][2][P][Hk][D] (pre-zeroed when atomic), `atomic_ctx`: parts are red.add'ed.
int launch_tc_bwd(const SimtArgs& a, float* dq_acc, const __nv_bfloat16* xsplit, int tpad, float* ctx_acc, int chunk,
                  int num_chunks, bool atomic_ctx, cudaStream_t st);

}  // namespace dkv
