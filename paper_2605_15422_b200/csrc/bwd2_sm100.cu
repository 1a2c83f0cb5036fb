// bwd2_sm100.cu -- tcgen05/TMEM/TMA backward for DualKV attention, 128x128 tiles
// (path 3, and the backward of path 1 / the replicated baseline).
//
// KV-stationary like bwd_sm100.cu (SURVEY §7.4 design (C)): a CTA owns one 128-key tile of one
// KV head and sweeps the GQA-packed 128-row query tiles (128/G tokens x G heads) that see it,
// accumulating dK/dV for all G query heads in TMEM.  What changes versus the 64-row version is
// the MMA shape: every GEMM is M=128 N=128, which the tensor core runs at full rate from shared
// memory (measured, tools/ubench/mma_rate.cu: SS N=64 is smem-read bound at 48 clk per K-step
// instead of 32; N=128 runs at the 64 clk ideal).  TMEM (512 columns) then only fits the four
// 128-column accumulators, so the per-tile intermediates alias:
//   [0,128)   S^T  (P^T bf16 written over [0,64) by the compute warps)
//   [128,256) dP^T (dS^T bf16 over [128,192)); dQ^T = K^T dS^T lands here too, after dK has read dS^T
//   [256,384) dV, [384,512) dK
// and the MMA issue order interleaves two query tiles so the tensor core never waits on the
// compute warps' exponentials:
//   S(0) dP(0) | dV(i) S(i+1) dK(i) dQ(i) dP(i+1) | ...
// (P(i+1) is computed while dK(i)/dQ(i) run; dS(i) while dV(i)/S(i+1) run.)  tcgen05.mma ops
// of one CTA execute in issue order, which makes the write-after-read aliasing safe.
//
// Per query tile (B_q = 128 rows, B_k = 128 keys, d = 128):
//   S^T  = K Q^T  + 1 (-lse/scale)^T   SS  (the additive constant is a K=16 split-bf16 MMA)
//   dP^T = V dO^T + 1 (-D)^T          SS
//   P^T = exp2(S'^T scale log2e), dS^T = P^T dP'^T     (compute warps; softmax scale folded out)
//   dV += P^T dO   TS (A = P^T in TMEM)
//   dK += dS^T Q   TS (A = dS^T in TMEM)
//   dQ^T = K^T dS^T  SS (dS^T also staged in smem), drained and TMA-reduce-added into fp32 dq_acc
// Roles: warps 0-3 compute (thread = key row), 4-7 dQ drain (thread = head-dim lane, one TMA
// reduce per warp per 16-row chunk, double-buffered) + dV epilogue, 8 TMA producer + TMEM
// allocator, 9 MMA issuer.
// Work items and their order: see the decode block below (longest first; co-resident CTAs share
// the query stream in L2: context key tiles fastest, single-sequence items sweep their query
// tiles from the sequence end down so all key tiles of a sequence move in lockstep).
#include "dkv_internal.h"
#include "tma_host.h"
#include "trace.cuh"

#include <cstdlib>

namespace dkv {
namespace bwd2 {

constexpr int kBK = 128;  // keys per tile (MMA M)
constexpr int kBQ = 128;  // query rows per tile (MMA N)
constexpr int D = 128;
constexpr int kThreads = 320;
constexpr int kTile = 128 * 128 * 2;  // bf16 [128 rows][128 cols]
constexpr int kPanel = 128 * 128;     // bf16 [128 rows][64 cols], SW128
constexpr int kX = 128 * 32;          // bf16 [128 rows][16], SW32
constexpr int kChunkRows = 16;        // dQ drain chunk: 16 query rows
constexpr int kStgWarp = kChunkRows * 32 * 4;  // one warp's fp32 [16 rows][32 d] staging (2 KB)
constexpr int kOffK = 0;
constexpr int kOffV = kOffK + kTile;
constexpr int kOffQ = kOffV + kTile;       // 2 stages
constexpr int kOffDO = kOffQ + 2 * kTile;  // 1 stage
constexpr int kOffDS = kOffDO + kTile;     // dS^T [128 keys][128 q] MN-major SW128 (2 panels)
constexpr int kOffXL = kOffDS + kTile;     // 2 stages of split(-lse/scale) rows
constexpr int kOffXD = kOffXL + 2 * kX;    // 1 stage of split(-D) rows
constexpr int kOffOnes = kOffXD + kX;      // [128 keys][16] SW32: (1, 1, 1, 0, ...)
constexpr int kOffStg = kOffOnes + kX;     // [2 buffers][4 warps] dQ staging
constexpr int kOffBar = kOffStg + 2 * 4 * kStgWarp;
constexpr int kSmemBytes = kOffBar + 256 + 1024;
static_assert(kSmemBytes <= 232448, "exceeds the 227 KB opt-in shared memory per block");

struct Params {
  CUtensorMap tm_q, tm_do, tm_k, tm_v, tm_kc, tm_vc, tm_dq, tm_x;
  CUtensorMap tm_qs, tm_dos, tm_xs, tm_dqs;  // fused Call 1 (two-call launch)
  int cu_self[2];     // {0, P}: the prompt as a one-sequence "cu_seqlens"
  int tpad_s, n_self_items, self_part;
  __nv_bfloat16* dk;  // [T][Hk][D]
  __nv_bfloat16* dv;
  float* ctx_acc;     // [parts][2][P][Hk][D]
  const int32_t* cu;
  int num_seqs, total_q, ctx_len, heads, kv_heads, group, tq, tpad;
  int chunk, n_ctx_items, n_ctx_tiles, max_own_tiles;
  int atomic_ctx;
  int chunk_heads, chunk_toks;  // dQ reduce box: 16 rows = chunk_toks tokens x chunk_heads heads
  int ablate;  // timing experiments only (DKV_BWD_ABLATE): 1 no dQ reduce, 2 no dQ staging, 4 no exp
  float scale, scale_log2;
};

struct Bars {
  uint64_t kv_full, kv_done;
  uint64_t q_full[2], q_empty[2];
  uint64_t do_full, do_empty;
  uint64_t s_full, p_full, dp_full, ds_full;
  uint64_t dq_full, dq_empty;
  uint32_t tmem_base;
};

// The query tiles of one work item, walked identically by every role.  Multi-sequence items
// (a chunk of sequences against a context key tile) go forward; single-sequence items go from
// the sequence's last tile down to the first one that sees the key tile.
struct QIter {
  const int32_t* cu;
  int tq, s, s_end, tok, rlen, tok_first;
  bool rev;
  __device__ void begin(const int32_t* cu_, int tq_, int s0, int s1, int tok0, bool reverse) {
    cu = cu_;
    tq = tq_;
    s = s0;
    s_end = s1;
    tok_first = tok0;
    rlen = cu[s + 1] - cu[s];
    rev = reverse;
    if (rev) {
      tok = rlen > tok0 ? ((rlen - 1) / tq) * tq : tok0 - tq;  // no tile: tok < tok_first
    } else {
      tok = tok0;
      skip_empty();
    }
  }
  __device__ void skip_empty() {
    while (s < s_end && tok >= rlen) {
      ++s;
      tok = 0;
      if (s < s_end) rlen = cu[s + 1] - cu[s];
    }
  }
  __device__ bool valid() const { return rev ? tok >= tok_first : s < s_end; }
  __device__ void next() {
    if (rev) {
      tok -= tq;
    } else {
      tok += tq;
      skip_empty();
    }
  }
};

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ float bf16lo(uint32_t x) { return __uint_as_float(x << 16); }
__device__ __forceinline__ float bf16hi(uint32_t x) { return __uint_as_float(x & 0xffff0000u); }

// K-major SW128 operand, K step k (16 elements): panel k/4, 32-byte slice k%4
__device__ __forceinline__ uint64_t kstep_kmajor(uint64_t d0, int k) {
  return d0 + static_cast<uint64_t>((((k >> 2) * kPanel) + (k & 3) * 32) >> 4);
}
// MN-major SW128 operand, K step k: 16 rows of 128 B
__device__ __forceinline__ uint64_t kstep_mnmajor(uint64_t d0, int k) {
  return d0 + static_cast<uint64_t>((k * 2048) >> 4);
}

__global__ void __launch_bounds__(kThreads, 1) dualkv_bwd2_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars& bar = *reinterpret_cast<Bars*>(base + kOffBar);

  // ---- work item (grid order = longest first: kinds 0, 2, 1).
  // kind 0: context key tile x chunk of sequences (Call 2), key tiles fastest;
  // kind 2 (two-call launch only): prompt key tile x the prompt's own causal queries (Call 1),
  //         accumulated into the same fp32 prompt scratch -- one cast for the total gradient;
  // kind 1: own-response key tile of one sequence (Call 2), key tiles fastest.
  const int bid = blockIdx.x;
  const int G = p.group;
  int kind, hk, ktile, s0, s1, tok_first, kv_len, kv_row0, part = 0;
  if (bid < p.n_ctx_items) {
    kind = 0;
    const int per_chunk = p.n_ctx_tiles * p.kv_heads;
    const int chunk_id = bid / per_chunk;
    const int rem = bid % per_chunk;
    ktile = rem % p.n_ctx_tiles;
    hk = rem / p.n_ctx_tiles;
    s0 = chunk_id * p.chunk;
    s1 = min(p.num_seqs, s0 + p.chunk);
    tok_first = 0;
    kv_len = p.ctx_len;
    kv_row0 = 0;
    part = p.atomic_ctx ? 0 : chunk_id;
  } else if (bid >= p.n_ctx_items + p.n_self_items) {
    kind = 1;
    const int b2 = bid - p.n_ctx_items - p.n_self_items;
    ktile = b2 % p.max_own_tiles;
    const int r2 = b2 / p.max_own_tiles;
    hk = r2 % p.kv_heads;
    s0 = r2 / p.kv_heads;
    s1 = s0 + 1;
    kv_len = p.cu[s0 + 1] - p.cu[s0];
    if (ktile * kBK >= kv_len) return;
    tok_first = (ktile * kBK / p.tq) * p.tq;
    kv_row0 = p.cu[s0];
  } else {
    kind = 2;
    const int b3 = bid - p.n_ctx_items;
    ktile = b3 % p.n_ctx_tiles;
    hk = b3 / p.n_ctx_tiles;
    s0 = 0;
    s1 = 1;
    kv_len = p.ctx_len;
    tok_first = (ktile * kBK / p.tq) * p.tq;
    kv_row0 = 0;
    part = p.atomic_ctx ? 0 : p.self_part;
  }
  const bool ctx_keys = kind != 1;  // keys are the shared prompt copy (output -> fp32 scratch)
  const bool causal = kind != 0;
  const bool rev = kind != 0;
  const int32_t* cu = kind == 2 ? p.cu_self : p.cu;
  const CUtensorMap* mq = kind == 2 ? &p.tm_qs : &p.tm_q;
  const CUtensorMap* mdo = kind == 2 ? &p.tm_dos : &p.tm_do;
  const CUtensorMap* mx = kind == 2 ? &p.tm_xs : &p.tm_x;
  const CUtensorMap* mdq = kind == 2 ? &p.tm_dqs : &p.tm_dq;
  const int xtpad = kind == 2 ? p.tpad_s : p.tpad;
  const int kbase = ktile * kBK;  // region-local first key of the tile
  int nq = 0;
  {
    QIter it;
    it.begin(cu, p.tq, s0, s1, tok_first, rev);
    for (; it.valid(); it.next()) ++nq;
  }
  if (nq == 0) return;  // context chunk of empty responses: scratch already zero

  const int warp = warp_id();
  const int lane = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(&bar.kv_full, 1);
    mbar_init(&bar.kv_done, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar.q_full[i], 1);
      mbar_init(&bar.q_empty[i], 1);
    }
    mbar_init(&bar.do_full, 1);
    mbar_init(&bar.do_empty, 1);
    mbar_init(&bar.s_full, 1);
    mbar_init(&bar.p_full, 128);
    mbar_init(&bar.dp_full, 1);
    mbar_init(&bar.ds_full, 128);
    mbar_init(&bar.dq_full, 1);
    mbar_init(&bar.dq_empty, 128);
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<512>(&bar.tmem_base);
  if (warp < 4) {
    // A operand of the additive-constant MMAs: row r = (1, 1, 1, 0, ..., 0) in SW32 K-major layout
    const int r = threadIdx.x;
    const uint32_t ones = 0x3F803F80u;  // two bf16 1.0
    uint8_t* row = base + kOffOnes + r * 32;
    const uint32_t sw = (r >> 2) & 1;   // 16 B chunk index XOR row bit 2
    *reinterpret_cast<uint4*>(row + (0 ^ sw) * 16) = make_uint4(ones, 0x3F80u, 0u, 0u);
    *reinterpret_cast<uint4*>(row + (1 ^ sw) * 16) = make_uint4(0u, 0u, 0u, 0u);
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;

  if (warp == 8) {
    // ================= producer: K/V once, then per query tile Q (+lse rows), dO (+D rows)
    if (lane == 0) {
      const CUtensorMap* mk = ctx_keys ? &p.tm_kc : &p.tm_k;
      const CUtensorMap* mv = ctx_keys ? &p.tm_vc : &p.tm_v;
      tma_prefetch(mq);
      tma_prefetch(mdo);
      tma_prefetch(mx);
      tma_prefetch(mk);
      tma_prefetch(mv);
      mbar_arrive_expect_tx(&bar.kv_full, 2 * kTile);
      for (int pn = 0; pn < 2; ++pn) {
        tma_load_3d(base + kOffK + pn * kPanel, mk, &bar.kv_full, pn * 64, hk, kv_row0 + kbase);
        tma_load_3d(base + kOffV + pn * kPanel, mv, &bar.kv_full, pn * 64, hk, kv_row0 + kbase);
      }
      QIter it;
      it.begin(cu, p.tq, s0, s1, tok_first, rev);
      for (int i = 0; it.valid(); it.next(), ++i) {
        const int st = i & 1;
        const int row0 = cu[it.s] + it.tok;
        const int xrow = (hk * xtpad + row0) * G;
        mbar_wait(&bar.q_empty[st], ((i >> 1) & 1) ^ 1);
        TRACE(T_Q_LOAD, i);
        mbar_arrive_expect_tx(&bar.q_full[st], kTile + kX);
        for (int pn = 0; pn < 2; ++pn)
          tma_load_3d(base + kOffQ + st * kTile + pn * kPanel, mq, &bar.q_full[st], pn * 64, hk * G, row0);
        tma_load_2d(base + kOffXL + st * kX, mx, &bar.q_full[st], 0, xrow);
        mbar_wait(&bar.do_empty, (i & 1) ^ 1);
        TRACE(T_DO_LOAD, i);
        mbar_arrive_expect_tx(&bar.do_full, kTile + kX);
        for (int pn = 0; pn < 2; ++pn)
          tma_load_3d(base + kOffDO + pn * kPanel, mdo, &bar.do_full, pn * 64, hk * G, row0);
        tma_load_2d(base + kOffXD, mx, &bar.do_full, 16, xrow);
      }
    }
  } else if (warp == 9) {
    // ================= MMA issuer (one thread); descriptors built once, K steps added
    if (elect_one()) {
      const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 384;
      const uint32_t id_s = idesc_bf16_f32(kBK, kBQ, false, false);
      const uint32_t id_kv = idesc_bf16_f32(kBK, D, false, true);
      const uint32_t id_dq = idesc_bf16_f32(D, kBQ, true, true);
      const uint64_t dK = sdesc_sw128(smem_u32(base + kOffK), 16, 1024);
      const uint64_t dV = sdesc_sw128(smem_u32(base + kOffV), 16, 1024);
      const uint64_t dKt = sdesc_sw128(smem_u32(base + kOffK), kPanel, 1024);  // K^T, MN-major
      const uint64_t dQk[2] = {sdesc_sw128(smem_u32(base + kOffQ), 16, 1024),
                               sdesc_sw128(smem_u32(base + kOffQ + kTile), 16, 1024)};
      const uint64_t dQm[2] = {sdesc_sw128(smem_u32(base + kOffQ), kPanel, 1024),
                               sdesc_sw128(smem_u32(base + kOffQ + kTile), kPanel, 1024)};
      const uint64_t dOk = sdesc_sw128(smem_u32(base + kOffDO), 16, 1024);
      const uint64_t dOm = sdesc_sw128(smem_u32(base + kOffDO), kPanel, 1024);
      const uint64_t dDS = sdesc_sw128(smem_u32(base + kOffDS), kPanel, 1024);
      const uint64_t dOnes = sdesc_sw32(smem_u32(base + kOffOnes));
      const uint64_t dXL[2] = {sdesc_sw32(smem_u32(base + kOffXL)), sdesc_sw32(smem_u32(base + kOffXL + kX))};
      const uint64_t dXD = sdesc_sw32(smem_u32(base + kOffXD));
      auto issue_s = [&](int st) {  // S^T = K Q^T - lse/scale
#pragma unroll
        for (int k = 0; k < D / 16; ++k) mma_ss(tS, kstep_kmajor(dK, k), kstep_kmajor(dQk[st], k), id_s, k > 0);
        mma_ss(tS, dOnes, dXL[st], id_s, 1u);
      };
      auto issue_dp = [&]() {  // dP^T = V dO^T - D
#pragma unroll
        for (int k = 0; k < D / 16; ++k) mma_ss(tdP, kstep_kmajor(dV, k), kstep_kmajor(dOk, k), id_s, k > 0);
        mma_ss(tdP, dOnes, dXD, id_s, 1u);
      };
      mbar_wait(&bar.kv_full, 0);
      mbar_wait(&bar.q_full[0], 0);
      tc_fence_after();
      TRACE(T_ISS_S, 0);
      issue_s(0);
      mma_commit(&bar.s_full);
      mbar_wait(&bar.do_full, 0);
      tc_fence_after();
      TRACE(T_ISS_DP, 0);
      issue_dp();
      mma_commit(&bar.dp_full);
      for (int i = 0; i < nq; ++i) {
        const int st = i & 1;
        const uint32_t acc0 = i > 0 ? 1u : 0u;
        // dV += P^T dO  (P^T bf16 over the S^T columns)
        mbar_wait(&bar.p_full, i & 1);
        tc_fence_after();
        TRACE(T_ISS_DV, i);
#pragma unroll
        for (int k = 0; k < kBQ / 16; ++k) mma_ts(tdV, tS + k * 8, kstep_mnmajor(dOm, k), id_kv, (acc0 | k) ? 1u : 0u);
        mma_commit(&bar.do_empty);
        // S(i+1): the tensor core works on it while the compute warps build dS(i)
        if (i + 1 < nq) {
          mbar_wait(&bar.q_full[st ^ 1], ((i + 1) >> 1) & 1);
          tc_fence_after();
          TRACE(T_ISS_S, i + 1);
          issue_s(st ^ 1);
          mma_commit(&bar.s_full);
        }
        // dK += dS^T Q, dQ^T = K^T dS^T (dQ^T over the dP^T columns, after dK has read dS^T)
        mbar_wait(&bar.ds_full, i & 1);
        tc_fence_after();
        TRACE(T_ISS_DK, i);
#pragma unroll
        for (int k = 0; k < kBQ / 16; ++k) mma_ts(tdK, tdP + k * 8, kstep_mnmajor(dQm[st], k), id_kv, (acc0 | k) ? 1u : 0u);
        mma_commit(&bar.q_empty[st]);
        TRACE(T_ISS_DQ, i);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) mma_ss(tdP, kstep_mnmajor(dKt, k), kstep_mnmajor(dDS, k), id_dq, k > 0);
        mma_commit(&bar.dq_full);
        // dP(i+1) once the drain has read dQ^T(i) out of those columns
        if (i + 1 < nq) {
          mbar_wait(&bar.dq_empty, i & 1);
          mbar_wait(&bar.do_full, (i + 1) & 1);
          tc_fence_after();
          TRACE(T_ISS_DP, i + 1);
          issue_dp();
          mma_commit(&bar.dp_full);
        }
      }
      mma_commit(&bar.kv_done);
      mbar_wait(&bar.kv_done, 0);
      TRACE(T_MMA_END, 0);
    }
  } else if (warp < 4) {
    // ================= compute WG: thread = key row r of the tile
    const int r = warp * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const uint32_t tS = tmem + lane_off, tdP = tmem + lane_off + 128;
    const int key = kbase + r;  // region-local key index
    uint8_t* sDS = base + kOffDS;
    const float sl2 = p.scale_log2;
    QIter it;
    it.begin(cu, p.tq, s0, s1, tok_first, rev);
    for (int i = 0; it.valid(); it.next(), ++i) {
      // key visible to query column c?  Visible columns form a range [cmin, cmax): context keys
      // (< P) are seen by every row of the sequence; an own key k by query token t >= k, i.e.
      // columns c >= (k - tok0) * G (rows are token-major); columns past the sequence end never
      int cmin;
      if (!causal) {
        cmin = key < kv_len ? 0 : kBQ;
      } else {
        const int dt = key - it.tok;
        cmin = dt <= 0 ? 0 : min(dt * G, kBQ);
      }
      const int cmax = min(kBQ, (it.rlen - it.tok) * G);
      const bool full = __all_sync(0xffffffffu, cmin == 0 && cmax == kBQ);
      // ---- P^T = exp2(S'^T * scale * log2 e), bf16, over the S^T columns (kept packed in pk)
      uint32_t pk[64];
      mbar_wait(&bar.s_full, i & 1);
      tc_fence_after();
      if (threadIdx.x == 0) TRACE(T_C_S, i);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t u[64];
        tmem_ld32(tS + 64 * h, *reinterpret_cast<uint32_t(*)[32]>(&u[0]));
        tmem_ld32(tS + 64 * h + 32, *reinterpret_cast<uint32_t(*)[32]>(&u[32]));
        tmem_wait_ld();
        const float2 s2 = make_float2(sl2, sl2);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 x = __fmul2_rn(make_float2(__uint_as_float(u[2 * j]), __uint_as_float(u[2 * j + 1])), s2);
          float e0 = (p.ablate & 4) ? x.x : ex2(x.x), e1 = (p.ablate & 4) ? x.y : ex2(x.y);
          if (!full) {
            const int c = 64 * h + 2 * j;
            e0 = (c >= cmin && c < cmax) ? e0 : 0.f;
            e1 = (c + 1 >= cmin && c + 1 < cmax) ? e1 : 0.f;
          }
          pk[32 * h + j] = pack_bf16(e0, e1);
        }
        tmem_st32(tS + 32 * h, *reinterpret_cast<uint32_t(*)[32]>(&pk[32 * h]));
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bar.p_full);
      if (threadIdx.x == 0) TRACE(T_C_P, i);
      // ---- dS^T = P^T dP'^T (dP' = dP - D from the MMA), bf16 -> TMEM over dP^T and -> smem
      mbar_wait(&bar.dp_full, i & 1);
      tc_fence_after();
      if (threadIdx.x == 0) TRACE(T_C_DP, i);
      // (the smem dS^T buffer is free: dP(i) was issued after dQ(i-1), its only reader, completed)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t u[64];
        tmem_ld32(tdP + 64 * h, *reinterpret_cast<uint32_t(*)[32]>(&u[0]));
        tmem_ld32(tdP + 64 * h + 32, *reinterpret_cast<uint32_t(*)[32]>(&u[32]));
        tmem_wait_ld();
        uint32_t pd[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint32_t pp = pk[32 * h + j];
          const float2 d2 = __fmul2_rn(make_float2(bf16lo(pp), bf16hi(pp)),
                                       make_float2(__uint_as_float(u[2 * j]), __uint_as_float(u[2 * j + 1])));
          pd[j] = pack_bf16(d2.x, d2.y);
        }
        tmem_st32(tdP + 32 * h, pd);
        uint8_t* panel = sDS + h * kPanel;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          *reinterpret_cast<uint4*>(panel + sw128_offset(r, ch)) =
              make_uint4(pd[4 * ch], pd[4 * ch + 1], pd[4 * ch + 2], pd[4 * ch + 3]);
      }
      tmem_wait_st();
      tc_fence_before();
      fence_async_smem();
      mbar_arrive(&bar.ds_full);
      if (threadIdx.x == 0) TRACE(T_C_DS, i);
    }
  } else {
    // ================= dQ drain: thread = head-dim lane d; each warp reduces its 32 d columns
    const int w4 = warp - 4;
    const uint32_t lane_off = static_cast<uint32_t>(w4 * 32) << 16;
    const uint32_t tdQ = tmem + lane_off + 128;
    float* stg[2] = {reinterpret_cast<float*>(base + kOffStg + w4 * kStgWarp),
                     reinterpret_cast<float*>(base + kOffStg + 4 * kStgWarp + w4 * kStgWarp)};
    int nchunk = 0;
    QIter it;
    it.begin(cu, p.tq, s0, s1, tok_first, rev);
    for (int i = 0; it.valid(); it.next(), ++i) {
      mbar_wait(&bar.dq_full, i & 1);
      tc_fence_after();
      if (threadIdx.x == 128) TRACE(T_D_DQ, i);
      uint32_t u[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tdQ + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&u[32 * c]));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bar.dq_empty);
      if (threadIdx.x == 128) TRACE(T_D_LD, i);
      const int row0 = cu[it.s] + it.tok;
#pragma unroll
      for (int c = 0; c < kBQ / kChunkRows; ++c, ++nchunk) {
        float* sb = stg[nchunk & 1];
        if (p.ablate & 2) continue;
        if (lane == 0) bulk_wait_read<1>();  // this buffer's previous reduce has read it
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kChunkRows; ++j) sb[j * 32 + lane] = __uint_as_float(u[c * kChunkRows + j]);
        fence_async_smem();
        __syncwarp();
        if (lane == 0 && !(p.ablate & 1)) {
          const int rr = c * kChunkRows;  // first tile row of the chunk: token rr / G, head rr % G
          tma_reduce_add_3d(mdq, sb, w4 * 32, hk * G + rr % G, row0 + rr / G);
          bulk_commit();
        }
      }
      if (threadIdx.x == 128) TRACE(T_D_END, i);
    }
    if (lane == 0) bulk_wait<0>();
  }

  // ================= dK / dV epilogue: warps 0-3 dK, warps 4-7 dV (thread = key row)
  if (warp < 8) {
    const bool do_k = warp < 4;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tcol = tmem + lane_off + (do_k ? 384 : 256);
    mbar_wait(&bar.kv_done, 0);
    tc_fence_after();
    const int key = kbase + r;
    const bool ok = key < kv_len;
    const float osc = do_k ? p.scale : 1.f;  // dK = scale * sum dS^T Q
#pragma unroll 1
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t u[32];
      tmem_ld32(tcol + c0, u);
      tmem_wait_ld();
      if (!ok) continue;
#pragma unroll
      for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * osc);
      if (ctx_keys) {
        const int64_t plane = static_cast<int64_t>(p.ctx_len) * p.kv_heads * D;
        float* dst = p.ctx_acc + static_cast<int64_t>(part) * 2 * plane + (do_k ? 0 : plane) +
                     (static_cast<int64_t>(key) * p.kv_heads + hk) * D + c0;
        if (p.atomic_ctx) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            red_add_v4(dst + i, __uint_as_float(u[i]), __uint_as_float(u[i + 1]), __uint_as_float(u[i + 2]),
                       __uint_as_float(u[i + 3]));
        } else {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(dst + i) = make_float4(__uint_as_float(u[i]), __uint_as_float(u[i + 1]),
                                                              __uint_as_float(u[i + 2]), __uint_as_float(u[i + 3]));
        }
      } else {
        __nv_bfloat16* dst = (do_k ? p.dk : p.dv) + ((static_cast<int64_t>(kv_row0) + key) * p.kv_heads + hk) * D + c0;
        uint4 v[4];
        uint32_t* w = reinterpret_cast<uint32_t*>(v);
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = pack_bf16(__uint_as_float(u[2 * i]), __uint_as_float(u[2 * i + 1]));
#pragma unroll
        for (int i = 0; i < 4; ++i) reinterpret_cast<uint4*>(dst)[i] = v[i];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace bwd2

DKV_TRACE_READ_FN(dkv_trace_read)

bool tc_bwd2_supported(int head_dim, int heads, int kv_heads) {
  if (head_dim != bwd2::D || kv_heads <= 0 || heads % kv_heads) return false;
  const int G = heads / kv_heads;
  return G <= bwd2::kBQ && (bwd2::kBQ % G) == 0;
}

int launch_tc_bwd2(const SimtArgs& a, const CtxSelf* self, const BwdScratch& w, cudaStream_t st) {
  using namespace bwd2;
  Params p{};
  const int G = a.heads / a.kv_heads;
  const int tq = kBQ / G;
  p.chunk_heads = G < kChunkRows ? G : kChunkRows;
  p.chunk_toks = kChunkRows / p.chunk_heads;
  if (a.total_q > 0 &&
      (!make_map_3d_bf16(&p.tm_q, a.q, a.total_q, a.heads, D, G, tq) ||
       !make_map_3d_bf16(&p.tm_do, a.dout, a.total_q, a.heads, D, G, tq) ||
       !make_map_3d_bf16(&p.tm_k, a.k, a.total_q, a.kv_heads, D, 1, kBK) ||
       !make_map_3d_bf16(&p.tm_v, a.v, a.total_q, a.kv_heads, D, 1, kBK) ||
       !make_map_3d_f32(&p.tm_dq, w.dq_acc, a.total_q, a.heads, D, p.chunk_heads, p.chunk_toks, 32) ||
       !make_map_2d_bf16_sw32(&p.tm_x, w.xsplit, static_cast<int64_t>(w.tpad) * a.heads, 32, 16, kBQ))) {
    set_error("cuTensorMapEncodeTiled failed (backward q/dO/k/v/dq/x)");
    return DKV_ERR_CUDA;
  }
  if (a.ctx_len > 0) {
    if (!make_map_3d_bf16(&p.tm_kc, a.k_ctx, a.ctx_len, a.kv_heads, D, 1, kBK) ||
        !make_map_3d_bf16(&p.tm_vc, a.v_ctx, a.ctx_len, a.kv_heads, D, 1, kBK)) {
      set_error("cuTensorMapEncodeTiled failed (backward k_ctx/v_ctx)");
      return DKV_ERR_CUDA;
    }
  }
  const bool with_self = self && a.ctx_len > 0;
  if (with_self &&
      (!make_map_3d_bf16(&p.tm_qs, self->q, a.ctx_len, a.heads, D, G, tq) ||
       !make_map_3d_bf16(&p.tm_dos, self->dout, a.ctx_len, a.heads, D, G, tq) ||
       !make_map_3d_f32(&p.tm_dqs, w.dq_acc_s, a.ctx_len, a.heads, D, p.chunk_heads, p.chunk_toks, 32) ||
       !make_map_2d_bf16_sw32(&p.tm_xs, w.xsplit_s, static_cast<int64_t>(w.tpad_s) * a.heads, 32, 16, kBQ))) {
    set_error("cuTensorMapEncodeTiled failed (backward fused Call 1 maps)");
    return DKV_ERR_CUDA;
  }
  p.tpad = w.tpad;
  p.tpad_s = w.tpad_s;
  p.cu_self[0] = 0;
  p.cu_self[1] = a.ctx_len;
  p.dk = static_cast<__nv_bfloat16*>(a.dk);
  p.dv = static_cast<__nv_bfloat16*>(a.dv);
  p.ctx_acc = w.ctx_acc;
  p.cu = a.cu;
  p.num_seqs = a.num_seqs;
  p.total_q = a.total_q;
  p.ctx_len = a.ctx_len;
  p.heads = a.heads;
  p.kv_heads = a.kv_heads;
  p.group = G;
  p.tq = tq;
  p.chunk = w.chunk;
  p.n_ctx_tiles = (a.ctx_len + kBK - 1) / kBK;
  p.n_ctx_items = a.total_q > 0 ? p.n_ctx_tiles * a.kv_heads * w.num_chunks : 0;
  p.n_self_items = with_self ? p.n_ctx_tiles * a.kv_heads : 0;
  p.self_part = w.self_part;
  p.atomic_ctx = w.atomic_ctx ? 1 : 0;
  p.scale = a.scale;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  {
    const char* e = getenv("DKV_BWD_ABLATE");
    p.ablate = e ? atoi(e) : 0;
  }
  p.max_own_tiles = a.total_q > 0 ? (a.max_seqlen + kBK - 1) / kBK : 0;
  const int64_t grid = static_cast<int64_t>(p.n_ctx_items) + p.n_self_items +
                       static_cast<int64_t>(p.max_own_tiles) * a.num_seqs * a.kv_heads;
  if (grid == 0) return DKV_OK;
  if (grid > 0x7fffffff) {
    set_error("backward grid too large");
    return DKV_ERR_UNSUPPORTED;
  }
  if (!ensure_smem_optin(reinterpret_cast<const void*>(dualkv_bwd2_kernel), kSmemBytes, "dualkv_bwd2_kernel"))
    return DKV_ERR_CUDA;
  dualkv_bwd2_kernel<<<static_cast<unsigned>(grid), kThreads, kSmemBytes, st>>>(p);
  return DKV_OK;
}

}  // namespace dkv
