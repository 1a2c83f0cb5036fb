// bwd_sm100.cu -- tcgen05/TMEM/TMA backward for DualKV attention (path 3 and
// the backward of paths 1 / the replicated baseline).
//
// KV-stationary (SURVEY §7.4 design (C)): a CTA owns one 128-key tile of one
// KV head and sweeps the 64-row query tiles that see it, accumulating dK and
// dV in TMEM for ALL G query heads of the group at once (GQA packed into the
// query tile rows, so the reference's per-tile GQA fold, fa2.py:224-227, is
// free).  Work items:
//   * own-region tiles (sequence s, key tile j): query tiles of s from the
//     causal diagonal on; dK_d / dV_d are written once as bf16 (no merge);
//   * shared-prompt tiles (chunk c of sequences, context tile j): all query
//     tiles of the chunk's sequences (no causal mask); the fp32 dK_c / dV_c
//     tile is reduce-added into one fp32 scratch (atomic mode) or stored as
//     the chunk's partial (deterministic mode) -- then folded and cast once
//     (kernel.py:279-285, Alg. 1/2).
// dQ is accumulated across key tiles in fp32: each tile's dQ^T is transposed
// through shared memory and reduce-added into dq_acc by ONE TMA bulk tensor
// reduce (cp.reduce.async.bulk.tensor ... add) -- register-sourced red.global
// measured 2.4-4.7x slower in situ (profiles/r1_microbench.md).
//
// Per query tile (B_q = 64 rows, B_k = 128 keys, d = 128; at d = 64 the K dims of S^T / dP^T
// and the N dims of dV / dK halve, and dQ^T keeps M = 128 over a zero-padded K^T panel):
//   S^T  = K Q^T      (M128 N64  K128)  -> TMEM [0,64)
//   dP^T = V dO^T     (M128 N64  K128)  -> TMEM [64,128)
//   P^T = exp2(S^T*scale*log2e - lse2), dS^T = P^T (dP^T - D) * scale   (compute WG)
//   S^T += 1 (-lse/scale)^T, dP^T += 1 (-D)^T  (K=16 split-bf16 MMAs: no per-column loads)
//   P^T, dS^T (bf16) -> TMEM [128,160), [160,192); dS^T also -> smem
//   dV  += P^T dO     (M128 N128 K64)   TS-MMA, A = P^T (TMEM)  -> TMEM [256,384)
//   dK  += dS^T Q     (M128 N128 K64)   TS-MMA, A = dS^T (TMEM) -> TMEM [384,512)
//   dQ^T = K^T dS^T   (M128 N64  K128)  SS-MMA                  -> TMEM [192,256)
// Roles: warps 0-7 compute (thread = key row; two warps per TMEM lane quadrant,
// 32 query columns each, so TMEM-load latency and MUFU work of one overlap the
// other's), 8-11 dQ drain (thread = head-dim lane), 12 TMA producer + TMEM
// allocator, 13 MMA issuer; warps 0-7 run the dK / dV epilogue.  At C3 the
// kernel runs at the board's 1000 W limit (profiles/r1_microbench.md): what
// moves it is energy per FLOP (L2 bytes), not latency hiding.
#include "dkv_internal.h"
#include "tma_host.h"
#include "trace.cuh"

#include <cstdlib>
#include <type_traits>

namespace dkv {
namespace bwd {

constexpr int kBK = 128;  // keys per tile (MMA M)
constexpr int kBQ = 64;   // query rows per tile (MMA N for S^T / dP^T / dQ^T)
constexpr int kThreads = 448;  // 8 compute warps, 4 dQ-drain warps, producer, MMA issuer
constexpr int kWDrain = 8, kWProd = 12, kWMma = 13;
constexpr int kDrainT0 = kWDrain * 32;  // first drain thread
#ifndef BWD_POLY
#define BWD_POLY 0  // sweep 0/2/4/6: 27.5/27.7/28.1/27.9 ms (noise-level; MUFU is not the limit here)
#endif
constexpr int kPolyPairs = BWD_POLY;    // of every 16 exponential pairs, on the FMA pipe
#ifndef BWD_SPIN
#define BWD_SPIN 0
#endif
#ifndef BWD_OWN_ORDER
// own-response items: 0 kv head fastest, then sequence, then key tile; 1 key tile fastest within
// (sequence, kv head).  A/B at C3 (profiles/r2_ab.md): 1 is 1.5x faster on the causal N-copy
// backward (108 -> 71 ms) and 5 % on the DualKV backward (its own-response items)
#define BWD_OWN_ORDER 1
#endif
#ifndef BWD_KT
// 1: K as a TMEM operand of S^T (d = 128): P^T / dS^T aliased onto the S^T / dP^T columns they
// are computed from, which frees TMEM [128,192) for K; the compute warps report P^T and dS^T
// separately so dV(i) + S^T(i+1) run while they finish dS^T(i) (profiles/r2_energy_ceilings.md)
#define BWD_KT 0
#endif
constexpr int kStages = 3;
constexpr int kKVPanel = kBK * 128;         // 16 KB: one 64-column SW128 panel of a key tile
constexpr int kPBytes = kBK * kBQ * 2;      // 16 KB
constexpr int kXBytes = kBQ * 32;           // [64 rows][16 bf16] SW32 tile (2 KB)

// Shared-memory layout for head dim D (64 or 128).  The K tile always has two panels: dQ^T =
// K^T dS^T runs as an M=128 MMA over the head dim, so at D=64 the second panel holds zeros
// (rows 64-127 of dQ^T come out zero and are not drained).
template <int D>
struct L {
  static constexpr int kKBytes = kBK * 128 * 2;  // 32 KB (two panels)
  static constexpr int kVBytes = kBK * D * 2;
  static constexpr int kQBytes = kBQ * D * 2;
  static constexpr int kQPanel = kBQ * 128;      // 8 KB
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + kKBytes;
  static constexpr int kOffQ = kOffV + kVBytes;
  static constexpr int kOffDO = kOffQ + kStages * kQBytes;
  static constexpr int kOffDS = kOffDO + kStages * kQBytes;
  static constexpr int kOffX = kOffDS + kPBytes;               // per stage: -lse/scale tile, -D tile
  static constexpr int kOffOnes = kOffX + kStages * 2 * kXBytes;  // [128 keys][16 bf16] SW32: 1,1,1,0...
  static constexpr int kOffStage = kOffOnes + kBK * 32;        // dQ staging tile for the TMA reduce
  static constexpr int kStageBytes = kBQ * D * 4;              // [64 rows][D] fp32
  static constexpr int kOffBar = kOffStage + kStageBytes;
  static constexpr int kSmemBytes = kOffBar + 256 + 1024;
  static_assert(kSmemBytes <= 232448, "exceeds the 227 KB opt-in shared memory per block");
};

struct Params {
  CUtensorMap tm_q, tm_do, tm_k, tm_v, tm_kc, tm_vc, tm_dq;
  CUtensorMap tm_x;     // xsplit [Hk*tpad*G rows][32] bf16: split3(-lse/scale) | split3(-D)
  // fused Call 1 (two-call launch): the prompt's own queries, their (lse, D) rows and dQ
  CUtensorMap tm_qs, tm_dos, tm_xs, tm_dqs;
  int tpad_s, n_self_items, self_part;
  float* dq_acc;        // [T][H][D] f32
  __nv_bfloat16* dk;    // [T][Hk][D]
  __nv_bfloat16* dv;
  float* ctx_acc;       // [parts][2][P][Hk][D]
  const int32_t* cu;
  int num_seqs, total_q, ctx_len, heads, kv_heads, group, tq, tpad;
  int chunk, max_chunks, n_ctx_items, n_ctx_tiles;  // n_ctx_tiles: of the longest group prompt
  int max_own_tiles;                               // key tiles of the longest response
  int atomic_ctx;
  int ablate;  // timing experiments only (DKV_BWD_ABLATE): 1 drain I/O, 2 compute math, 4 Q/dO loads,
               // 8 the additive-constant MMAs
  float scale, scale_log2;
  // prompt groups; grp.ctx doubles as the Call 1 "cu_seqlens" (group g's prompt = sequence g)
  GroupTable grp;
};

struct Bars {
  uint64_t kv_full, sdp_full, sdp_empty, pds_full, pds_empty, kv_done;
  uint64_t k_tm, p_ready, dp_full;  // BWD_KT: K in TMEM; P^T(i) stored; dP^T(i) complete
  uint64_t q_full[kStages], q_empty[kStages];
  uint64_t dq_full, dq_empty;
  uint32_t tmem_base;
};

// The query tiles of one work item, walked identically by every role.
struct QIter {
  const int32_t* cu;
  int tq, s, s_end, tok, rlen;
  __device__ void begin(const int32_t* cu_, int tq_, int s0, int s1, int tok0) {
    cu = cu_;
    tq = tq_;
    s = s0;
    s_end = s1;
    tok = tok0;
    rlen = cu[s + 1] - cu[s];
    skip_empty();
  }
  __device__ void skip_empty() {
    while (s < s_end && tok >= rlen) {
      ++s;
      tok = 0;
      if (s < s_end) rlen = cu[s + 1] - cu[s];
    }
  }
  __device__ bool valid() const { return s < s_end; }
  __device__ void next() {
    tok += tq;
    skip_empty();
  }
};

__device__ __forceinline__ void red_add(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) dualkv_bwd_kernel(const __grid_constant__ Params p) {
  using Y = L<D>;
  constexpr bool kKT = BWD_KT && D == 128;
  constexpr int kQBytes = Y::kQBytes, kQPanel = Y::kQPanel, kStageBytes = Y::kStageBytes;
  constexpr int kOffK = Y::kOffK, kOffV = Y::kOffV, kOffQ = Y::kOffQ, kOffDO = Y::kOffDO, kOffDS = Y::kOffDS;
  constexpr int kOffX = Y::kOffX, kOffOnes = Y::kOffOnes, kOffStage = Y::kOffStage, kOffBar = Y::kOffBar;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars& bar = *reinterpret_cast<Bars*>(base + kOffBar);

  // ---- decode the work item (grid order = longest first: kinds 0, 2, 1).
  // kind 0: shared-prompt key tile x chunk of sequences (Call 2);
  // kind 1: own-response key tile of one sequence (Call 2); kind 2 (two-call launch only):
  // prompt key tile x the prompt's own causal queries (Call 1), accumulated into the same fp32
  // shared-prompt scratch so the total prompt gradient is cast once.
  const int bid = blockIdx.x;
  int kind, hk, ktile, s0, s1, tok_first, kv_len, kv_row0, part = 0;
  if (bid < p.n_ctx_items) {
    kind = 0;
    // key tiles fastest: the ~148 co-resident CTAs then share a few (chunk, head) Q/dO streams
    // and dQ-accumulator regions in L2 instead of 8 heads' worth
    // (multi-group launches: then group, then chunk -- every group's chunk 0 first)
    const int per_chunk = p.n_ctx_tiles * p.kv_heads;
    const int cg = bid / per_chunk;  // (chunk, group)
    const int rem = bid % per_chunk;
    ktile = rem % p.n_ctx_tiles;
    hk = rem / p.n_ctx_tiles;
    const int g = cg % p.grp.n;
    const int chunk_id = cg / p.grp.n;
    kv_row0 = p.grp.ctx[g];
    kv_len = p.grp.ctx[g + 1] - kv_row0;
    if (ktile * kBK >= kv_len) return;  // a shorter prompt than the launch's longest
    s0 = p.grp.seq[g] + chunk_id * p.chunk;
    s1 = min(p.grp.seq[g + 1], s0 + p.chunk);
    if (s0 >= s1) return;  // a group with fewer sequences than the largest
    tok_first = 0;
    part = p.atomic_ctx ? 0 : chunk_id;
  } else if (bid >= p.n_ctx_items + p.n_self_items) {
    kind = 1;
    const int b2 = bid - p.n_ctx_items - p.n_self_items;
#if BWD_OWN_ORDER == 1
    // a (sequence, kv head)'s key tiles side by side: co-resident CTAs stream the same Q / dO /
    // (lse, D) rows and reduce into the same dQ accumulator lines in L2
    ktile = b2 % p.max_own_tiles;
    const int r2 = b2 / p.max_own_tiles;
    hk = r2 % p.kv_heads;
    s0 = r2 / p.kv_heads;
#else
    hk = b2 % p.kv_heads;
    const int r2 = b2 / p.kv_heads;
    s0 = r2 % p.num_seqs;
    ktile = r2 / p.num_seqs;
#endif
    s1 = s0 + 1;
    kv_len = p.cu[s0 + 1] - p.cu[s0];
    if (ktile * kBK >= kv_len) return;
    tok_first = (ktile * kBK / p.tq) * p.tq;
    kv_row0 = p.cu[s0];
  } else {
    kind = 2;
    const int b3 = bid - p.n_ctx_items;
    ktile = b3 % p.n_ctx_tiles;
    hk = (b3 / p.n_ctx_tiles) % p.kv_heads;
    s0 = b3 / (p.n_ctx_tiles * p.kv_heads);  // the group = its prompt's "sequence" in grp.ctx
    s1 = s0 + 1;
    kv_row0 = p.grp.ctx[s0];
    kv_len = p.grp.ctx[s0 + 1] - kv_row0;
    if (ktile * kBK >= kv_len) return;
    tok_first = (ktile * kBK / p.tq) * p.tq;
    part = p.atomic_ctx ? 0 : p.self_part;
  }
  const bool ctx_keys = kind != 1;  // keys are the shared prompt copy (output -> fp32 scratch)
  const bool causal = kind != 0;
  const int32_t* cu = kind == 2 ? p.grp.ctx : p.cu;
  const CUtensorMap* mq = kind == 2 ? &p.tm_qs : &p.tm_q;
  const CUtensorMap* mdo = kind == 2 ? &p.tm_dos : &p.tm_do;
  const CUtensorMap* mx = kind == 2 ? &p.tm_xs : &p.tm_x;
  const CUtensorMap* mdq = kind == 2 ? &p.tm_dqs : &p.tm_dq;
  const int xtpad = kind == 2 ? p.tpad_s : p.tpad;
  const int kbase = ktile * kBK;  // region-local first key of the tile
  int nq = 0;
  {
    QIter it;
    it.begin(cu, p.tq, s0, s1, tok_first);
    for (; it.valid(); it.next()) ++nq;
  }
  if (nq == 0) return;  // context chunk of empty responses: scratch already zero

  const int warp = warp_id();
  const int lane = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(&bar.kv_full, 1);
    mbar_init(&bar.sdp_full, 1);
    mbar_init(&bar.sdp_empty, 256);
    mbar_init(&bar.pds_full, 256);
    mbar_init(&bar.pds_empty, 1);
    mbar_init(&bar.kv_done, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&bar.q_full[i], 1);
      mbar_init(&bar.q_empty[i], 1);
    }
    mbar_init(&bar.dq_full, 1);
    mbar_init(&bar.dq_empty, 128);
    mbar_init(&bar.k_tm, 256);
    mbar_init(&bar.p_ready, 256);
    mbar_init(&bar.dp_full, 1);
    fence_mbar_init();
  }
  if (warp == kWProd) tmem_alloc<512>(&bar.tmem_base);
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
  if constexpr (D == 64) {
    // the zero second panel of the key tile (head-dim rows 64-127 of K^T in the dQ^T MMA)
    for (int i = threadIdx.x; i < kKVPanel / 16; i += kThreads)
      reinterpret_cast<uint4*>(base + kOffK + kKVPanel)[i] = make_uint4(0u, 0u, 0u, 0u);
    fence_async_smem();
  }
  // G not dividing 64 (e.g. G = 5): a query tile is tq = 64 / G (floored) tokens x G heads; the
  // TMA boxes fill its first qrows rows only, so the padding rows of every Q / dO stage are zeroed
  // once (their S^T / dP^T columns are then finite and masked to P = dS = 0)
  const int qrows = p.tq * p.group;
  if (qrows < kBQ) {
    for (int st = 0; st < kStages; ++st)
      for (int pn = 0; pn < D / 64; ++pn)
        for (int i = threadIdx.x; i < (kBQ - qrows) * 8; i += kThreads) {
          const int off = (qrows + i / 8) * 128 + (i % 8) * 16;
          *reinterpret_cast<uint4*>(base + kOffQ + st * kQBytes + pn * kQPanel + off) = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(base + kOffDO + st * kQBytes + pn * kQPanel + off) = make_uint4(0u, 0u, 0u, 0u);
        }
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;
  const int G = p.group;

  if (warp == kWProd) {
    // ================= producer: K/V once, then (Q, dO, lse/D) per query tile
    const CUtensorMap* mk = ctx_keys ? &p.tm_kc : &p.tm_k;
    const CUtensorMap* mv = ctx_keys ? &p.tm_vc : &p.tm_v;
    if (lane == 0) {
      tma_prefetch(mq);
      tma_prefetch(mdo);
      tma_prefetch(mdq);
      tma_prefetch(mx);
      tma_prefetch(mk);
      tma_prefetch(mv);
      mbar_arrive_expect_tx(&bar.kv_full, 2 * Y::kVBytes);
      for (int pn = 0; pn < D / 64; ++pn) {
        tma_load_3d(base + kOffK + pn * kKVPanel, mk, &bar.kv_full, pn * 64, hk, kv_row0 + kbase);
        tma_load_3d(base + kOffV + pn * kKVPanel, mv, &bar.kv_full, pn * 64, hk, kv_row0 + kbase);
      }
    }
    if (lane == 0) {
      QIter it;
      it.begin(cu, p.tq, s0, s1, tok_first);
      for (int i = 0; it.valid(); it.next(), ++i) {
        const int st = i % kStages;
        const uint32_t ph = (i / kStages) & 1;
        mbar_wait(&bar.q_empty[st], ph ^ 1);
        TRACE(T_Q_LOAD, i);
        const int row0 = cu[it.s] + it.tok;
        mbar_arrive_expect_tx(&bar.q_full[st], ((DKV_ABL(p.ablate) & 4) ? 0 : 2 * qrows * D * 2) + 2 * kXBytes);
        for (int pn = 0; pn < D / 64 && !(DKV_ABL(p.ablate) & 4); ++pn) {
          tma_load_3d(base + kOffQ + st * kQBytes + pn * kQPanel, mq, &bar.q_full[st], pn * 64, hk * G, row0);
          tma_load_3d(base + kOffDO + st * kQBytes + pn * kQPanel, mdo, &bar.q_full[st], pn * 64, hk * G, row0);
        }
        // the tile's 64 additive-constant rows: -lse/scale (cols 0-15) and -D (cols 16-31)
        const int xrow = (hk * xtpad + row0) * G;
        tma_load_2d(base + kOffX + st * 2 * kXBytes, mx, &bar.q_full[st], 0, xrow);
        tma_load_2d(base + kOffX + st * 2 * kXBytes + kXBytes, mx, &bar.q_full[st], 16, xrow);
#ifdef DKV_TRACE
        mbar_wait(&bar.q_full[st], (i / kStages) & 1);  // trace build: record the load's arrival
        TRACE(T_DO_LOAD, i);
#endif
      }
    }
  } else if (warp == kWMma) {
    // ================= MMA issuer
    if (elect_one()) {
      const uint32_t tS = tmem, tdP = tmem + 64, tP = tmem + 128, tDS = tmem + 160, tdQ = tmem + 192;
      const uint32_t tdV = tmem + 256, tdK = tmem + 384;
      const uint32_t id_sdp = idesc_bf16_f32(kBK, kBQ, false, false);
      const uint32_t id_kv = idesc_bf16_f32(kBK, D, false, true);
      const uint32_t id_dq = idesc_bf16_f32(128, kBQ, true, true);  // M = 128 head-dim rows (zeros past D)
      // descriptors built once; a K step adds its byte offset >> 4 to the start-address field
      const uint64_t dKk = sdesc_sw128(smem_u32(base + kOffK), 16, 1024);
      const uint64_t dVk = sdesc_sw128(smem_u32(base + kOffV), 16, 1024);
      const uint64_t dKt = sdesc_sw128(smem_u32(base + kOffK), kKVPanel, 1024);  // K^T, MN-major
      const uint64_t dDS = sdesc_sw128(smem_u32(base + kOffDS), kPBytes, 1024);
      const uint64_t dOnes = sdesc_sw32(smem_u32(base + kOffOnes));
      auto koff_kv = [](int k) { return static_cast<uint64_t>(((k >> 2) * kKVPanel + (k & 3) * 32) >> 4); };
      auto koff_q = [](int k) { return static_cast<uint64_t>(((k >> 2) * kQPanel + (k & 3) * 32) >> 4); };
      auto koff_mn = [](int k) { return static_cast<uint64_t>((k * 2048) >> 4); };
      // the issuer's waits are on the critical path of the tensor pipe: BWD_SPIN selects how it
      // waits (0 try_wait with a suspend hint, 1 test_wait spin, 2 try_wait without a hint)
      auto issuer_wait = [](uint64_t* b, uint32_t ph) {
        if constexpr (BWD_SPIN == 1)
          mbar_spin(b, ph);
        else if constexpr (BWD_SPIN == 2)
          mbar_wait_nohint(b, ph);
        else if constexpr (BWD_SPIN >= 16)  // a short suspend-time hint of BWD_SPIN ns
          mbar_wait_hint<BWD_SPIN>(b, ph);
        else
          mbar_wait(b, ph);
      };
      issuer_wait(&bar.kv_full, 0);
      if constexpr (kKT) {
        // S^T = K Q^T with A = K from TMEM [128,192); P^T lives in S^T's columns [16,48) and dS^T in
        // dP^T's [80,112) (each compute warp's packed columns land on its own fp32 columns).  Per
        // step i: dV(i-1) -> S^T(i) once P^T(i-1) is stored (the in-order tensor pipe reads P^T
        // before S^T(i) overwrites it); dK(i-1) -> dP^T(i) once dS^T(i-1) is; then dQ^T(i-1).
        const uint32_t tK = tmem + 128, tPa = tS + 16, tDSa = tdP + 16;
        issuer_wait(&bar.k_tm, 0);
        tc_fence_after();
        for (int i = 0; i <= nq; ++i) {
          const int st = i % kStages;
          const int j = i - 1, sj = (i + kStages - 1) % kStages;
          if (i > 0) {
            issuer_wait(&bar.p_ready, j & 1);
            tc_fence_after();
            const uint64_t dOm = sdesc_sw128(smem_u32(base + kOffDO + sj * kQBytes), kQPanel, 1024);
            TRACE(T_ISS_DV, j);
#pragma unroll
            for (int k = 0; k < kBQ / 16; ++k)
              mma_ts(tdV, tPa + k * 8, dOm + koff_mn(k), id_kv, (j > 0 || k > 0) ? 1u : 0u);
          }
          const uint64_t dX = sdesc_sw32(smem_u32(base + kOffX + st * 2 * kXBytes));
          if (i < nq) {
            issuer_wait(&bar.q_full[st], (i / kStages) & 1);
            tc_fence_after();
            const uint64_t dQk = sdesc_sw128(smem_u32(base + kOffQ + st * kQBytes), 16, 1024);
            TRACE(T_ISS_S, i);
#pragma unroll
            for (int k = 0; k < D / 16; ++k) mma_ts(tS, tK + k * 8, dQk + koff_q(k), id_sdp, k > 0);
            mma_ss(tS, dOnes, dX, id_sdp, 1u);
            mma_commit(&bar.sdp_full);
          }
          if (i > 0) {
            issuer_wait(&bar.pds_full, j & 1);
            tc_fence_after();
            const uint64_t dQm = sdesc_sw128(smem_u32(base + kOffQ + sj * kQBytes), kQPanel, 1024);
            TRACE(T_ISS_DK, j);
#pragma unroll
            for (int k = 0; k < kBQ / 16; ++k)
              mma_ts(tdK, tDSa + k * 8, dQm + koff_mn(k), id_kv, (j > 0 || k > 0) ? 1u : 0u);
            mma_commit(&bar.q_empty[sj]);
          }
          if (i < nq) {
            const uint64_t dOk = sdesc_sw128(smem_u32(base + kOffDO + st * kQBytes), 16, 1024);
            TRACE(T_ISS_DP, i);
#pragma unroll
            for (int k = 0; k < D / 16; ++k) mma_ss(tdP, dVk + koff_kv(k), dOk + koff_q(k), id_sdp, k > 0);
            mma_ss(tdP, dOnes, dX + (kXBytes >> 4), id_sdp, 1u);
            mma_commit(&bar.dp_full);
          }
          if (i > 0) {
            issuer_wait(&bar.dq_empty, (j & 1) ^ 1);
            tc_fence_after();
            TRACE(T_ISS_DQ, j);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) mma_ss(tdQ, dKt + koff_mn(k), dDS + koff_mn(k), id_dq, k > 0);
            mma_commit(&bar.dq_full);
            mma_commit(&bar.pds_empty);  // the dS^T shared-memory tile is free
          }
        }
      }
      for (int i = 0; i <= nq && !kKT; ++i) {
        if (i < nq) {
          const int st = i % kStages;
          issuer_wait(&bar.q_full[st], (i / kStages) & 1);
          if (i > 0) issuer_wait(&bar.sdp_empty, (i - 1) & 1);
          tc_fence_after();
          const uint64_t dQk = sdesc_sw128(smem_u32(base + kOffQ + st * kQBytes), 16, 1024);
          const uint64_t dOk = sdesc_sw128(smem_u32(base + kOffDO + st * kQBytes), 16, 1024);
          const uint64_t dX = sdesc_sw32(smem_u32(base + kOffX + st * 2 * kXBytes));
          TRACE(T_ISS_S, i);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            if (DKV_ABL(p.ablate) & 16)  // energy experiment (trace build): A from TMEM (dV columns,
              mma_ts(tS, tdV + k * 8, dQk + koff_q(k), id_sdp, k > 0);  // garbage): no K smem reads
            else
              mma_ss(tS, dKk + koff_kv(k), dQk + koff_q(k), id_sdp, k > 0);
          }
          // S^T[k][c] += -lse[c] / scale  (so that P = exp2(S'^T * scale * log2 e))
          if (!(DKV_ABL(p.ablate) & 8)) mma_ss(tS, dOnes, dX, id_sdp, 1u);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            if (DKV_ABL(p.ablate) & 16)
              mma_ts(tdP, tdK + k * 8, dOk + koff_q(k), id_sdp, k > 0);
            else
              mma_ss(tdP, dVk + koff_kv(k), dOk + koff_q(k), id_sdp, k > 0);
          }
          // dP^T[k][c] += -D[c]  (so that dS^T = P^T * dP'^T)
          if (!(DKV_ABL(p.ablate) & 8)) mma_ss(tdP, dOnes, dX + (kXBytes >> 4), id_sdp, 1u);
          mma_commit(&bar.sdp_full);
        }
        if (i > 0) {
          const int j = i - 1;
          const int sj = j % kStages;
          const uint64_t dQm = sdesc_sw128(smem_u32(base + kOffQ + sj * kQBytes), kQPanel, 1024);
          const uint64_t dOm = sdesc_sw128(smem_u32(base + kOffDO + sj * kQBytes), kQPanel, 1024);
          issuer_wait(&bar.pds_full, j & 1);
          tc_fence_after();
          TRACE(T_ISS_DV, j);
#pragma unroll
          for (int k = 0; k < kBQ / 16; ++k)
            mma_ts(tdV, tP + k * 8, dOm + koff_mn(k), id_kv, (j > 0 || k > 0) ? 1u : 0u);
#pragma unroll
          for (int k = 0; k < kBQ / 16; ++k)
            mma_ts(tdK, tDS + k * 8, dQm + koff_mn(k), id_kv, (j > 0 || k > 0) ? 1u : 0u);
          mma_commit(&bar.q_empty[sj]);
          issuer_wait(&bar.dq_empty, (j & 1) ^ 1);
          tc_fence_after();
          TRACE(T_ISS_DQ, j);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) mma_ss(tdQ, dKt + koff_mn(k), dDS + koff_mn(k), id_dq, k > 0);
          mma_commit(&bar.dq_full);
          mma_commit(&bar.pds_empty);
        }
      }
      mma_commit(&bar.kv_done);
    }
  } else if (warp < kWDrain) {
    // ================= compute warps: thread = key row r of the tile, 32 query columns
    // [c0, c0+32) per warp; two warps per TMEM lane quadrant so one's TMEM-load latency and
    // MUFU work overlap the other's
    const int r = (warp & 3) * 32 + lane;
    const int c0 = (warp >> 2) * 32;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int key = kbase + r;  // region-local key index
    uint8_t* sDS = base + kOffDS;
    if constexpr (kKT) {
      // K row r -> TMEM [128,192) (A operand of S^T): this warp's head-dim half = 32 columns
      mbar_wait(&bar.kv_full, 0);
      const int hh = warp >> 2;
      const uint8_t* kp = base + kOffK + hh * kKVPanel;
      uint32_t u[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 v = *reinterpret_cast<const uint4*>(kp + sw128_offset(r, c));
        u[4 * c] = v.x;
        u[4 * c + 1] = v.y;
        u[4 * c + 2] = v.z;
        u[4 * c + 3] = v.w;
      }
      tmem_st32(tmem + lane_off + 128 + hh * 32, u);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bar.k_tm);
    }
    QIter it;
    it.begin(cu, p.tq, s0, s1, tok_first);
    for (int i = 0; it.valid(); it.next(), ++i) {
      const int st = i % kStages;
      mbar_wait(&bar.q_full[st], (i / kStages) & 1);
      mbar_wait(&bar.sdp_full, i & 1);
      tc_fence_after();
      if constexpr (kKT) {
        // P^T first (-> S^T's own columns, reported on p_ready), then dS^T once dP^T is complete
        uint32_t us[32];
        tmem_ld32(tmem + lane_off + c0, us);
        tmem_wait_ld();
        if (threadIdx.x == 0) TRACE(T_C_S, i);
        int cmin;
        if (!causal) {
          cmin = key < kv_len ? 0 : kBQ;
        } else {
          const int dt = key - it.tok;
          cmin = dt <= 0 ? 0 : min(dt * G, kBQ);
        }
        const int cmax = min(qrows, (it.rlen - it.tok) * G);
        const float2 sl2 = make_float2(p.scale_log2, p.scale_log2);
        uint32_t pp[16];
        auto math_p = [&](auto masked) {
#pragma unroll
          for (int c2 = 0; c2 < 16; ++c2) {
            const float2 x =
                __fmul2_rn(make_float2(__uint_as_float(us[2 * c2]), __uint_as_float(us[2 * c2 + 1])), sl2);
            float2 e;
            if (c2 >= 16 - kPolyPairs) {
              e = ex2_poly2(x);
            } else {
              e.x = ex2(x.x);
              e.y = ex2(x.y);
            }
            if constexpr (decltype(masked)::value) {
              const int c = c0 + 2 * c2;
              e.x = (c >= cmin && c < cmax) ? e.x : 0.f;
              e.y = (c + 1 >= cmin && c + 1 < cmax) ? e.y : 0.f;
            }
            us[2 * c2] = __float_as_uint(e.x);
            us[2 * c2 + 1] = __float_as_uint(e.y);
            pp[c2] = pack_bf16(e.x, e.y);
          }
        };
        if (__all_sync(0xffffffffu, cmin <= c0 && cmax >= c0 + 32))
          math_p(std::false_type{});
        else
          math_p(std::true_type{});
        tmem_st16(tmem + lane_off + 16 + c0 / 2, pp);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bar.p_ready);
        if (threadIdx.x == 0) TRACE(T_C_P, i);
        mbar_wait(&bar.dp_full, i & 1);
        tc_fence_after();
        uint32_t ud[32];
        tmem_ld32(tmem + lane_off + 64 + c0, ud);
        tmem_wait_ld();
        if (threadIdx.x == 0) TRACE(T_C_DP, i);
        uint32_t pd[16];
#pragma unroll
        for (int c2 = 0; c2 < 16; ++c2) {
          const float2 dd = __fmul2_rn(make_float2(__uint_as_float(us[2 * c2]), __uint_as_float(us[2 * c2 + 1])),
                                       make_float2(__uint_as_float(ud[2 * c2]), __uint_as_float(ud[2 * c2 + 1])));
          pd[c2] = pack_bf16(dd.x, dd.y);
        }
        mbar_wait(&bar.pds_empty, (i & 1) ^ 1);  // dQ^T(i-1) is done with the dS^T tile in smem
        tc_fence_after();
        tmem_st16(tmem + lane_off + 80 + c0 / 2, pd);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          const uint32_t off = sw128_offset(r, c0 / 8 + ch);
          *reinterpret_cast<uint4*>(sDS + off) = make_uint4(pd[4 * ch], pd[4 * ch + 1], pd[4 * ch + 2], pd[4 * ch + 3]);
        }
        tmem_wait_st();
        tc_fence_before();
        fence_async_smem();
        mbar_arrive(&bar.pds_full);
        if (threadIdx.x == 0) TRACE(T_C_DS, i);
        continue;
      }
      if (threadIdx.x == 0) TRACE(T_C_S, i);
      uint32_t us[32], ud[32];
      tmem_ld32(tmem + lane_off + c0, us);
      tmem_ld32(tmem + lane_off + 64 + c0, ud);
      tmem_wait_ld();
      if (threadIdx.x == 0) TRACE(T_C_DP, i);
      tc_fence_before();
      mbar_arrive(&bar.sdp_empty);
      // key visible to query column c?  Visible columns form a range [cmin, cmax): context keys
      // (< P) are seen by every row of the sequence; an own key k is seen by query token t >= k,
      // i.e. columns c >= (k - tok0) * G (rows are token-major); columns past the sequence end
      // are never visible
      int cmin;
      if (!causal) {
        cmin = key < kv_len ? 0 : kBQ;
      } else {
        const int dt = key - it.tok;
        cmin = dt <= 0 ? 0 : min(dt * G, kBQ);
      }
      const int cmax = min(qrows, (it.rlen - it.tok) * G);
      const float2 sl2 = make_float2(p.scale_log2, p.scale_log2);
      uint32_t pp[16], pd[16];
      // S' = S - lse/scale and dP' = dP - D arrive from the MMA: P = exp2(S' scale log2e),
      // dS = P dP' (the softmax scale is applied once to dK in the epilogue and dQ in its cast)
      if (DKV_ABL(p.ablate) & 2) {
#pragma unroll
        for (int c2 = 0; c2 < 16; ++c2) {
          pp[c2] = us[2 * c2] ^ us[2 * c2 + 1];
          pd[c2] = ud[2 * c2] ^ ud[2 * c2 + 1];
        }
      } else {
        // the masked / unmasked variants are separate straight-line loops: a per-pair branch
        // inside one unrolled loop keeps ptxas from interleaving the MUFU chains (measured
        // ~2x slower compute warps)
        auto math = [&](auto masked) {
#pragma unroll
          for (int c2 = 0; c2 < 16; ++c2) {
            const float2 x =
                __fmul2_rn(make_float2(__uint_as_float(us[2 * c2]), __uint_as_float(us[2 * c2 + 1])), sl2);
            float2 e;
            if (c2 >= 16 - kPolyPairs) {
              e = ex2_poly2(x);
            } else {
              e.x = ex2(x.x);
              e.y = ex2(x.y);
            }
            if constexpr (decltype(masked)::value) {
              const int c = c0 + 2 * c2;
              e.x = (c >= cmin && c < cmax) ? e.x : 0.f;
              e.y = (c + 1 >= cmin && c + 1 < cmax) ? e.y : 0.f;
            }
            const float2 dd =
                __fmul2_rn(e, make_float2(__uint_as_float(ud[2 * c2]), __uint_as_float(ud[2 * c2 + 1])));
            pp[c2] = pack_bf16(e.x, e.y);
            pd[c2] = pack_bf16(dd.x, dd.y);
          }
        };
        if (__all_sync(0xffffffffu, cmin <= c0 && cmax >= c0 + 32))
          math(std::false_type{});
        else
          math(std::true_type{});
      }
      if (threadIdx.x == 0) TRACE(T_C_P, i);
      mbar_wait(&bar.pds_empty, (i & 1) ^ 1);
      tc_fence_after();
      // P^T and dS^T -> TMEM (A operands of the dV / dK TS-MMAs); dS^T also -> smem (B of dQ^T)
      tmem_st16(tmem + lane_off + 128 + c0 / 2, pp);
      tmem_st16(tmem + lane_off + 160 + c0 / 2, pd);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        const uint32_t off = sw128_offset(r, c0 / 8 + ch);
        *reinterpret_cast<uint4*>(sDS + off) = make_uint4(pd[4 * ch], pd[4 * ch + 1], pd[4 * ch + 2], pd[4 * ch + 3]);
      }
      tmem_wait_st();
      tc_fence_before();
      fence_async_smem();
      mbar_arrive(&bar.pds_full);
      if (threadIdx.x == 0) TRACE(T_C_DS, i);
    }
  } else if (warp < kWProd) {
    // ================= dQ drain WG: thread = head-dim lane d
    const int d = (warp - kWDrain) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>((warp - kWDrain) * 32) << 16;
    QIter it;
    it.begin(cu, p.tq, s0, s1, tok_first);
    for (int i = 0; it.valid(); it.next(), ++i) {
      mbar_wait(&bar.dq_full, i & 1);
      tc_fence_after();
      if (threadIdx.x == kDrainT0) TRACE(T_D_DQ, i);
      uint32_t u[64];
      tmem_ld32(tmem + lane_off + 192, *reinterpret_cast<uint32_t(*)[32]>(&u[0]));
      tmem_ld32(tmem + lane_off + 192 + 32, *reinterpret_cast<uint32_t(*)[32]>(&u[32]));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bar.dq_empty);
      if (threadIdx.x == kDrainT0) TRACE(T_D_LD, i);
      // transpose through smem ([row][d] fp32) and reduce-add into dq_acc with TMA bulk tensor
      // reduces, one per 32-row half: reductions leave an SM at ~25 B/clk (profiles/
      // r1_microbench.md), so the staging of one half overlaps the other half's egress
      if (DKV_ABL(p.ablate) & 1) continue;
      const int row0 = cu[it.s] + it.tok;
      if (qrows < kBQ) {
        // G not dividing 64: one reduce of the tile's tq x G rows (a 32-row half would split a token)
        float* stg = reinterpret_cast<float*>(base + kOffStage);
        if (threadIdx.x == kDrainT0) bulk_wait_read<0>();  // the previous tile's reduce has read it
        named_bar_sync(1, 128);
#pragma unroll
        for (int c = 0; c < kBQ; ++c)
          if (c < qrows && (D == 128 || d < D)) stg[c * D + d] = __uint_as_float(u[c]);
        fence_async_smem();
        named_bar_sync(1, 128);
        if (threadIdx.x == kDrainT0) {
          tma_reduce_add_3d(mdq, stg, 0, hk * G, row0);
          bulk_commit();
        }
        continue;
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float* stg = reinterpret_cast<float*>(base + kOffStage + hh * (kStageBytes / 2));
        if (threadIdx.x == kDrainT0) bulk_wait_read<1>();  // this half's previous reduce has read it
        named_bar_sync(1, 128);
#pragma unroll
        for (int c = 0; c < kBQ / 2; ++c)
          if (D == 128 || d < D) stg[c * D + d] = __uint_as_float(u[hh * (kBQ / 2) + c]);
        fence_async_smem();
        named_bar_sync(1, 128);
        if (threadIdx.x == kDrainT0) {
          const int rr = hh * (kBQ / 2);  // first tile row of the half: token rr / G, head rr % G
          tma_reduce_add_3d(mdq, stg, 0, hk * G + rr % G, row0 + rr / G);
          bulk_commit();
        }
      }
      if (threadIdx.x == kDrainT0) TRACE(T_D_END, i);
    }
    if (threadIdx.x == kDrainT0) bulk_wait<0>();
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
        float* dst = p.ctx_acc + static_cast<int64_t>(part) * 2 * plane +
                     (do_k ? 0 : plane) + ((static_cast<int64_t>(kv_row0) + key) * p.kv_heads + hk) * D + c0;
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
  if (warp == kWProd) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace bwd

DKV_TRACE_READ_FN(dkv_trace_read_v1)

static bool tc_bwd1_supported(int head_dim, int heads, int kv_heads) {
  if ((head_dim != 64 && head_dim != 128) || kv_heads <= 0 || heads % kv_heads) return false;
  const int G = heads / kv_heads;
  return G <= bwd::kBQ;  // a 64-row query tile holds floor(64 / G) tokens x G heads
}

bool tc_bwd_supported(int dtype, int head_dim, int heads, int kv_heads) {
  if (dtype != DKV_BF16 || force_simt()) return false;
  return tc_bwd1_supported(head_dim, heads, kv_heads);
}

namespace bwd {
template <int D>
static int launch(const SimtArgs& a, const CtxSelf* self, const GroupTable& grp, const BwdScratch& w,
                  cudaStream_t st) {
  Params p{};
  const int G = a.heads / a.kv_heads;
  const int tq = kBQ / G;
  // dQ reduce box: one 32-row half when G divides 64, else the tile's whole tq x G rows
  const bool halves = kBQ % G == 0;
  const int hb = !halves ? G : (G < kBQ / 2 ? G : kBQ / 2), tb = !halves ? tq : (kBQ / 2) / hb;
  if (a.total_q > 0 &&
      (!make_map_3d_bf16(&p.tm_q, a.q, a.total_q, a.heads, D, G, tq) ||
       !make_map_3d_bf16(&p.tm_do, a.dout, a.total_q, a.heads, D, G, tq) ||
       !make_map_3d_bf16(&p.tm_k, a.k, a.total_q, a.kv_heads, D, 1, kBK) ||
       !make_map_3d_bf16(&p.tm_v, a.v, a.total_q, a.kv_heads, D, 1, kBK) ||
       !make_map_3d_f32(&p.tm_dq, w.dq_acc, a.total_q, a.heads, D, hb, tb, D) ||
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
       !make_map_3d_f32(&p.tm_dqs, w.dq_acc_s, a.ctx_len, a.heads, D, hb, tb, D) ||
       !make_map_2d_bf16_sw32(&p.tm_xs, w.xsplit_s, static_cast<int64_t>(w.tpad_s) * a.heads, 32, 16, kBQ))) {
    set_error("cuTensorMapEncodeTiled failed (backward fused Call 1 maps)");
    return DKV_ERR_CUDA;
  }
  p.tpad = w.tpad;
  p.tpad_s = w.tpad_s;
  p.grp = grp;
  p.dq_acc = w.dq_acc;
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
  p.max_chunks = w.num_chunks;
  p.n_ctx_tiles = (grp.max_ctx + kBK - 1) / kBK;
  const int64_t n_ctx_items =
      a.total_q > 0 ? static_cast<int64_t>(p.n_ctx_tiles) * a.kv_heads * grp.n * w.num_chunks : 0;
  const int64_t n_self_items = with_self ? static_cast<int64_t>(p.n_ctx_tiles) * a.kv_heads * grp.n : 0;
  if (n_ctx_items + n_self_items > 0x7fffffff) {
    set_error("backward grid too large");
    return DKV_ERR_UNSUPPORTED;
  }
  p.n_ctx_items = static_cast<int>(n_ctx_items);
  p.n_self_items = static_cast<int>(n_self_items);
  p.self_part = w.self_part;
  p.atomic_ctx = w.atomic_ctx ? 1 : 0;
#ifdef DKV_ABLATION  // timing-experiment builds only (libdkv_trace.so); never read by libdkv.so
  {
    const char* e = getenv("DKV_BWD_ABLATE");
    p.ablate = e ? atoi(e) : 0;
  }
#endif
  p.scale = a.scale;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  const int max_tiles = a.total_q > 0 ? (a.max_seqlen + kBK - 1) / kBK : 0;
  p.max_own_tiles = std::max(1, max_tiles);
  const int64_t grid = static_cast<int64_t>(p.n_ctx_items) + p.n_self_items +
                       static_cast<int64_t>(max_tiles) * a.num_seqs * a.kv_heads;
  if (grid == 0) return DKV_OK;
  if (grid > 0x7fffffff) {
    set_error("backward grid too large");
    return DKV_ERR_UNSUPPORTED;
  }
  if (!ensure_smem_optin(reinterpret_cast<const void*>(dualkv_bwd_kernel<D>), L<D>::kSmemBytes, "dualkv_bwd_kernel"))
    return DKV_ERR_CUDA;
  dualkv_bwd_kernel<D><<<static_cast<unsigned>(grid), kThreads, L<D>::kSmemBytes, st>>>(p);
  return DKV_OK;
}
}  // namespace bwd

int launch_tc_bwd(const SimtArgs& a, const CtxSelf* self, const GroupTable& grp, const BwdScratch& w,
                  cudaStream_t st) {
  if (tc_bwd_pair_supported(a.head_dim, a.heads, a.kv_heads)) return launch_tc_bwd_pair(a, self, grp, w, st);
  return a.head_dim == 64 ? bwd::launch<64>(a, self, grp, w, st) : bwd::launch<128>(a, self, grp, w, st);
}

}  // namespace dkv
