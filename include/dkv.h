/*
 * dkv.h -- C ABI of the B200 (sm_100a) DualKV attention library (libdkv.so).
 *
 * Plain pointers and sizes only: no torch / Python types cross this
 * boundary.  Every entry point is stream-ordered on the caller's stream,
 * never allocates device memory (the caller passes outputs and workspace),
 * never throws, and returns DKV_OK (0) or a negative error class; the
 * message of the last error on the calling thread is in dkv_last_error().
 *
 * Tensor layouts (all row-major, contiguous, device memory):
 *   q, out, dout, dq      [total_q, heads,    head_dim]
 *   k, v, dk, dv          [total_q, kv_heads, head_dim]   per-sequence keys
 *   k_ctx, v_ctx, dk_ctx  [ctx_len, kv_heads, head_dim]   the ONE shared prompt copy
 *   lse                   [heads, total_q] float32, natural log
 *   cu_seqlens            [num_seqs + 1]   int32, cu[0] = 0, cu[N] = total_q
 * Query row r of sequence i has logical position ctx_len + r; it sees every
 * context key and its own keys 0..r.
 *
 * Reference interfaces each entry point replaces (paths under
 * /root/reference/pkg/src/dualkv/):
 *   dkv_dualkv_fwd      <- kernel.py:177-210  dualkv_fwd(DualKVInput) -> (O, lse)
 *   dkv_dualkv_bwd      <- kernel.py:245-293  dualkv_bwd(inp, O, lse, dO, deterministic, fold_seed)
 *                          (ctx_partials != NULL: kernel.py:296-305 context_grad_contributions)
 *   dkv_varlen_fwd      <- fa2.py:237-265     fa2_varlen_fwd(VarlenBatch) -> (O, lse)
 *   dkv_varlen_bwd      <- fa2.py:268-306     fa2_varlen_bwd(batch, O, lse, dO) -> (dQ, dK, dV)
 *   dkv_convert_f32_to_bf16 <- kernel.py:140-148 convert_dkv_context (one RNE cast, tensor.py:39-58)
 *   dkv_gather_rows / dkv_segment_sum_rows
 *                       <- packing.py:159-220 pack_standard / pack_dualkv as a device
 *                          repack of activations (and its adjoint for gradients)
 */
#ifndef DKV_H_
#define DKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DKV_ABI_VERSION 2

/* Most prompt groups one launch takes (group table entries, see dkv_group_table). */
#define DKV_MAX_GROUPS 256

#if defined(__GNUC__)
#define DKV_API __attribute__((visibility("default")))
#else
#define DKV_API
#endif

enum dkv_status {
  DKV_OK = 0,
  DKV_ERR_INVALID = -1,     /* contract violation (maps to ValueError) */
  DKV_ERR_UNSUPPORTED = -2, /* legal input this build cannot run (maps to ValueError) */
  DKV_ERR_CUDA = -3,        /* launch / driver failure (maps to RuntimeError) */
  DKV_ERR_WORKSPACE = -4    /* workspace too small */
};

enum dkv_dtype { DKV_BF16 = 0, DKV_F32 = 1 };

/* Multi-group launches (SURVEY §8b "group table"): several prompt groups in ONE launch.  The
 * reference runs one group per call and loops over groups in the caller (layer.py:239,
 * SPEC.md:284); here every group's prompt rows are concatenated in k_ctx / v_ctx (and q_ctx of
 * the two-call op) and every group's responses in q / k / v, and the table says which rows
 * belong together.  HOST arrays of num_groups + 1 int32 (copied into the kernel parameters):
 *   seq_cu[g] .. seq_cu[g+1]  the sequences (indices into cu_seqlens) of group g;
 *                             seq_cu[0] = 0, seq_cu[num_groups] = num_seqs, each group >= 1 sequence
 *   ctx_cu[g] .. ctx_cu[g+1]  group g's prompt rows in k_ctx / v_ctx (q_ctx, out_ctx, dq_ctx);
 *                             ctx_cu[0] = 0, ctx_cu[num_groups] = ctx_len
 * num_groups = 0 means one group (every sequence shares rows [0, ctx_len) of the prompt).
 * Multi-group launches run on the tensor-core path only (bf16, head_dim 64 / 128). */
typedef struct dkv_group_table {
  int64_t num_groups;
  const int32_t* seq_cu;
  const int32_t* ctx_cu;
} dkv_group_table;

typedef struct dkv_fwd_params {
  const void* q;
  const void* k_ctx; /* may be NULL when ctx_len == 0 */
  const void* v_ctx;
  const void* k;
  const void* v;
  const int32_t* cu_seqlens;
  void* out;
  float* lse;
  int64_t num_seqs, total_q, ctx_len, heads, kv_heads, head_dim;
  int64_t max_seqlen; /* max_i R_i (bounds the launch grid; must be >= the true max) */
  float softmax_scale;
  int32_t dtype;      /* enum dkv_dtype */
  dkv_group_table groups; /* ABI 2: zero-initialised = one group */
} dkv_fwd_params;

typedef struct dkv_bwd_params {
  const void* q;
  const void* k_ctx;
  const void* v_ctx;
  const void* k;
  const void* v;
  const int32_t* cu_seqlens;
  const void* out;   /* saved forward output */
  const float* lse;  /* saved forward lse [heads, total_q] */
  const void* dout;
  void* dq;
  void* dk_ctx;      /* shared-prompt gradients (NULL when ctx_len == 0) */
  void* dv_ctx;
  void* dk;
  void* dv;
  int64_t num_seqs, total_q, ctx_len, heads, kv_heads, head_dim, max_seqlen;
  float softmax_scale;
  int32_t dtype;
  int32_t deterministic; /* 1: context fold in fixed chunk order (bitwise reproducible dK_c/dV_c) */
  int32_t ctx_chunk;     /* sequences per context work unit; 0 = automatic */
  float* ctx_partials;   /* optional [num_chunks, 2, ctx_len, kv_heads, head_dim] f32 output of the
                            un-folded per-chunk context contributions (instrumentation hook) */
  dkv_group_table groups; /* ABI 2: zero-initialised = one group */
  float* ctx_grad_f32;    /* ABI 2, optional [2, ctx_len, kv_heads, head_dim] f32: the folded prompt
                            gradient (dK_c, dV_c) just before its single cast (instrumentation:
                            the atomic-vs-ordered fold check, SURVEY §8c "determinism") */
} dkv_bwd_params;

DKV_API int32_t dkv_abi_version(void);
DKV_API const char* dkv_last_error(void);
/* 1 when the tensor-core (tcgen05) path serves this shape/dtype, 0 when the SIMT path does. */
DKV_API int32_t dkv_uses_tensor_cores(int32_t dtype, int64_t head_dim, int64_t heads, int64_t kv_heads);

DKV_API int32_t dkv_dualkv_fwd(const dkv_fwd_params* p, void* stream);
DKV_API int32_t dkv_varlen_fwd(const dkv_fwd_params* p, void* stream);

/* Bytes of scratch dkv_*_bwd needs for these parameters (fp32 dQ accumulator,
 * packed (lse, D) rows, fp32 shared-prompt accumulators or per-chunk partials). */
DKV_API size_t dkv_bwd_workspace_size(const dkv_bwd_params* p);
/* Number of context chunks the backward uses (rows of ctx_partials). */
DKV_API int64_t dkv_bwd_num_ctx_chunks(const dkv_bwd_params* p);
DKV_API int32_t dkv_dualkv_bwd(const dkv_bwd_params* p, void* workspace, size_t workspace_bytes, void* stream);
DKV_API int32_t dkv_varlen_bwd(const dkv_bwd_params* p, void* workspace, size_t workspace_bytes, void* stream);

/* Fused two-call launch (layer.py:236-290, §3): Call 1 -- causal self-attention of
 * the prompt's own queries over the single prompt copy -- runs inside the Call 2 launch (its
 * work items fill the tail).  In the backward both calls accumulate the prompt-key gradient in
 * ONE fp32 scratch, cast once into call2.dk_ctx / call2.dv_ctx (the TOTAL prompt gradient;
 * the reference instead adds two separately cast contributions, layer.py:278-279). */
typedef struct dkv_twocall_fwd_params {
  dkv_fwd_params call2; /* the two-region problem; call2.k_ctx / v_ctx are the prompt's keys */
  const void* q_ctx;    /* [ctx_len, heads, head_dim] the prompt's own queries */
  void* out_ctx;        /* [ctx_len, heads, head_dim] */
  float* lse_ctx;       /* [heads, ctx_len] */
} dkv_twocall_fwd_params;

typedef struct dkv_twocall_bwd_params {
  dkv_bwd_params call2; /* ctx_partials must be NULL */
  const void* q_ctx;
  const void* out_ctx;
  const float* lse_ctx;
  const void* dout_ctx;
  void* dq_ctx;         /* [ctx_len, heads, head_dim] */
} dkv_twocall_bwd_params;

DKV_API int32_t dkv_twocall_fwd(const dkv_twocall_fwd_params* p, void* stream);
DKV_API size_t dkv_twocall_bwd_workspace_size(const dkv_twocall_bwd_params* p);
DKV_API int32_t dkv_twocall_bwd(const dkv_twocall_bwd_params* p, void* workspace, size_t workspace_bytes,
                                void* stream);

/* dst[i] = RNE_bf16(src[i]), bit-identical to the reference bf16_round. */
DKV_API int32_t dkv_convert_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream);

/* dst[r, :] = src[idx[r], :] for r < n_rows; rows are row_bytes long (multiple of 16 fastest). */
DKV_API int32_t dkv_gather_rows(const void* src, void* dst, int64_t row_bytes, const int64_t* idx,
                        int64_t n_rows, void* stream);
/* dst[r, :] = sum_{j in [seg[r], seg[r+1])} src[src_idx[j], :], fp32 accumulate, dtype storage. */
DKV_API int32_t dkv_segment_sum_rows(const void* src, void* dst, int32_t dtype, int64_t row_elems,
                             const int64_t* seg, const int64_t* src_idx, int64_t n_rows,
                             void* stream);

/* RoPE at logical positions (reference layer.py:182-205, positions packing.py:105-120), fused
 * with an optional row gather (the N(P+R) -> P+NR repack, packing.py:182-220):
 *   dst[r, h, 2k:2k+2] = R(pos[r] * base^(-2k/d)) src[idx ? idx[r] : r, h, 2k:2k+2]
 * (R the 2x2 rotation, transposed when `inverse` -- the adjoint, rope_bwd).  Angles in fp64,
 * rotation in fp32, dtype storage (bf16 or fp32) for src and dst; `positions` and `idx` are
 * device int64 arrays of n_rows.  head_dim a multiple of 8 (bf16) / 4 (fp32), 16-byte aligned rows. */
DKV_API int32_t dkv_rope_rows(const void* src, void* dst, int32_t dtype, int64_t n_rows, int64_t heads,
                              int64_t head_dim, const int64_t* positions, const int64_t* idx, double base,
                              int32_t inverse, void* stream);
/* The same for a row's q [heads], k [kv_heads] (rotated) and v [kv_heads] (copied) in one pass --
 * the fused repack + RoPE of the QKV projections; any tensor's src/dst may both be NULL. */
DKV_API int32_t dkv_rope_qkv_rows(const void* q_src, const void* k_src, const void* v_src, void* q_dst,
                                  void* k_dst, void* v_dst, int32_t dtype, int64_t n_rows, int64_t heads,
                                  int64_t kv_heads, int64_t head_dim, const int64_t* positions,
                                  const int64_t* idx, double base, int32_t inverse, void* stream);

/* The step between the QKV projection and the DualKV op, one HBM pass (reference
 * layer.py:182-205 for RoPE, packing.py:105-120 for positions; Qwen3's per-head q/k RMSNorm,
 * SPEC.md:464, when the norm weights are given): for every packed row r of
 * qkv [rows, heads + 2 kv_heads, head_dim] (bf16, the GEMM output):
 *   q / k heads: y = RoPE(pos[r]) (x * rsqrt(mean(x^2) + eps) * w)   (fp32, rounded once)
 *   v heads:     copied
 * written at row dst_rows[r] of q [rows, heads, d], k / v [rows, kv_heads, d].  norm weights: bf16
 * [head_dim] each, both NULL for no norm.  head_dim 64 / 128 / 256.  Device int64 arrays. */
DKV_API int32_t dkv_qkv_prep_fwd(const void* qkv, const void* q_norm_w, const void* k_norm_w, float eps,
                                 const int64_t* positions, const int64_t* dst_rows, void* q, void* k, void* v,
                                 int64_t rows, int64_t heads, int64_t kv_heads, int64_t head_dim, double base,
                                 void* stream);
/* Its adjoint: dq / dk / dv (rows in the dst_rows layout) -> dqkv [rows, heads + 2 kv_heads, d] (packed
 * order) and, with norm weights, their fp32 gradients dq_norm_w / dk_norm_w [head_dim] (zeroed and
 * accumulated by the call).  qkv is the forward's input (the norm is recomputed from it). */
DKV_API int32_t dkv_qkv_prep_bwd(const void* dq, const void* dk, const void* dv, const void* qkv,
                                 const void* q_norm_w, const void* k_norm_w, float eps, const int64_t* positions,
                                 const int64_t* dst_rows, void* dqkv, float* dq_norm_w, float* dk_norm_w,
                                 int64_t rows, int64_t heads, int64_t kv_heads, int64_t head_dim, double base,
                                 void* stream);

/* Kernel timing for the bench harness: while enabled, the library records a
 * CUDA event pair (on the launching stream) around every main attention
 * kernel and counts every kernel it launches.  dkv_profile_end synchronises
 * on the recorded events and returns the summed device milliseconds and
 * launch counts of the forward and backward main kernels, plus all launches. */
DKV_API int32_t dkv_profile_begin(void);
DKV_API int32_t dkv_profile_end(double* fwd_ms, int32_t* fwd_launches, double* bwd_ms,
                                int32_t* bwd_launches, int32_t* all_launches);

/* Self-test of the UMMA operand layouts used by the kernels (debug aid):
 * 128x128 (or 128xN) bf16 product through TMA + tcgen05, D fp32 [128][N]. */
DKV_API int32_t dkv_selftest_umma(int32_t mode, const void* a, const void* b, float* d, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DKV_H_ */
