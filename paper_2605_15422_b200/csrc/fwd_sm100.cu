// fwd_sm100.cu -- tcgen05/TMEM/TMA forward for DualKV attention (paths 1 & 2).
//
// One kernel serves
//   * Call 2, the fused two-region DualKV forward (kernel.py:177-210): each
//     query tile walks its own causal response tiles, then the shared-prompt
//     tiles (no mask except the partial last tile), carrying one online
//     softmax state across the region boundary and writing lse;
//   * Call 1 / the replicated N-copy baseline (fa2.py:237-265): ctx_len == 0.
//
// Tiling (B200-first, not the reference's loop nest):
//   * GQA packing: the G query heads sharing a KV head are packed into the MMA
//     M dimension -- a 128-row Q tile is (128/G tokens) x (G heads), loaded by
//     ONE 3-D TMA box straight from the [T, H, d] tensor.  Each K/V tile is
//     read once for all G heads (the reference expands K/V with np.repeat,
//     fa2.py:105-109).
//   * Each CTA owns two Q tiles (A, B) of consecutive tokens and ping-pongs the
//     tensor core between them: S_A = Q_A K^T and S_B = Q_B K^T share one K
//     tile in smem; P is written back to TMEM as bf16 (aliasing S) and
//     O += P V runs as a TS-MMA with A from TMEM.
//   * TMEM: S_A [0,128) S_B [128,256) O_A [256,256+d) O_B [384,384+d) columns.
//   * Online softmax in the log2 domain, one query row per thread (TMEM lane),
//     with lazy O rescaling (only when the running max grows by > 8).
//   * Roles: warps 0-7 softmax(A), 8-15 softmax(B) -- two warps per TMEM lane quadrant, one
//     per 64-key half of each row --, 16 TMA producer + TMEM allocator, 17 MMA issuer
//     (18 warps = 5 on some SM sub-partitions, whose 16K registers cap them at 96 per thread;
//     a setmaxnreg split was measured to deadlock or spill).
#include "dkv_internal.h"
#include "tma_host.h"
#include "trace.cuh"

#include <cstdlib>
#include <map>
#include <mutex>

namespace dkv {
namespace fwd {

constexpr int kBM = 128;  // rows per Q tile
constexpr int kBN = 128;  // keys per KV tile
constexpr int kThreads = 576;  // 16 softmax warps, producer, MMA issuer
constexpr int kWProd = 16, kWMma = 17;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef FWD_POLY
#define FWD_POLY 5
#endif
constexpr int kPolyPairs = FWD_POLY;       // of every 16 exponential pairs, on the FMA pipe
#ifndef FWD_EVICT
// L2 hint of the own-region K/V tiles: 0 evict_last (as the prompt's), 1 normal, 2 first
#define FWD_EVICT 1
#endif
#ifndef FWD_SPIN
#define FWD_SPIN 0
#endif
#ifndef FWD_QT_SPLIT
// Q-in-TMEM mode: 1 two warps per row (32 keys each, partial maxima exchanged), 0 one warp per
// row over all 64 keys of the tile (the other eight softmax warps idle).  C3 forward, interleaved
// x3: 0 is 8.6-9.1 ms, 1 is 9.4-9.8 ms (pair default, 128-key tiles: 8.3-8.5 ms)
#define FWD_QT_SPLIT 0
#endif
#ifndef FWD_ORDER
// main work-item order: 0 kv head fastest, then sequence, then q block; 1 q block fastest within
// (sequence, kv head).  A/B at C3 (tools/ab.sh, profiles/r2_ab.md): 1 + evict-normal own K/V is
// 3 % faster for the DualKV forward and 1.3x for the causal (N-copy / Call 1) forward
#define FWD_ORDER 1
#endif

template <int D>
struct Cfg {
  static constexpr int kPanels = D / 64;
  static constexpr int kTileBytes = kBM * D * 2;   // Q, K or V tile (bf16)
  static constexpr int kPanelBytes = kBM * 128;    // one 64-column SW128 panel of 128 rows
  static constexpr int kStages = D == 128 ? 2 : 3; // K ring and V ring depth
  static constexpr int kSmemTiles = (2 + 2 * kStages) * kTileBytes;
  static constexpr int kSmemBytes = kSmemTiles + 8192 /*barriers + row-max exchange*/ + 1024 /*align slack*/;
  // CTA-pair mode (D = 128): each CTA holds half of every K tile (64 keys, two 64-column panels)
  // and half of every V tile (all 128 keys, 64 of the d columns)
  static constexpr int kKHalf = 64 * D * 2;
  static constexpr int kVHalf = kBN * 64 * 2;
  static constexpr int kPairStages = 4;
  static constexpr int kSmemTilesPair = 2 * kTileBytes + kPairStages * (kKHalf + kVHalf);
  static constexpr int kSmemBytesPair = kSmemTilesPair + 8192 + 1024;
  // Q-in-TMEM pair mode (kQT, D = 128): 64-key KV tiles, so S_A / S_B take 64 TMEM columns each and
  // Q_A / Q_B fit beside them as the S MMA's A operand (TS-MMA: no Q reads from shared memory);
  // each CTA holds 32 keys of every K tile and 64 d columns of every V tile
  static constexpr int kKHalfQT = 32 * D * 2;
  static constexpr int kVHalfQT = 64 * 64 * 2;
  static constexpr int kQTStages = 8;
  static constexpr int kSmemTilesQT = 2 * kTileBytes + kQTStages * (kKHalfQT + kVHalfQT);
  static constexpr int kSmemBytesQT = kSmemTilesQT + 8192 + 1024;
};

struct Params {
  CUtensorMap tm_q, tm_k, tm_v, tm_kc, tm_vc;
  CUtensorMap tm_qs;      // fused Call 1: the prompt's own queries [P, H, d]
  CUtensorMap tm_k64, tm_kc64;  // pair mode: K boxes of 64 keys (each CTA loads one half)
  CUtensorMap tm_k32, tm_kc32, tm_v64, tm_vc64;  // Q-in-TMEM pair mode: 32-key K, 64-key V boxes
  __nv_bfloat16* out;
  float* lse;
  __nv_bfloat16* out_s;   // fused Call 1 outputs [P, H, d], lse [H, P]
  float* lse_s;
  const int32_t* cu;
  int num_seqs, total_q, ctx_len, heads, kv_heads, group, tq;
  int n_main_items;       // items >= n_main_items are Call 1 items (causal self-attention over the prompt)
  int blocks_per_seq;     // q blocks (items) per (sequence, kv head) of the longest sequence
  float scale_log2;       // softmax_scale * log2(e)
  int ablate;             // timing experiments only (DKV_FWD_ABLATE): 1 K/V loads, 2 exponentials
  GroupTable grp;         // prompt groups of the launch (one group: {0, num_seqs} / {0, ctx_len})
};

struct Smem {
  uint64_t q_full;
  uint64_t k_full[8], k_empty[8], v_full[8], v_empty[8];
  uint64_t s_full[2], p_full[2], o_full[2];
  uint64_t q_tm[2];       // kQT: Q tile t is in TMEM (one arrival per softmax warp of both CTAs)
  uint32_t tmem_base;
  // the two column halves of a row exchange partial row maxima (and, at the end, row sums)
  float xch[2][2][2][128];  // [tile][iteration parity][column half][row]
};

// kPair: a 2-CTA cluster runs FOUR Q tiles (two per CTA) through M = 256 tcgen05 MMAs issued by
// the leader (cta_group::2): each CTA loads only half of every K tile (64 keys) and half of
// every V tile (64 d columns), so K/V traffic into the SMs and the B-operand shared-memory
// reads per FLOP halve; S, P and O stay in each CTA's own tensor memory.
template <int D, bool kPair, bool kQT = false>
__global__ void __launch_bounds__(kThreads, 1) dualkv_fwd_kernel(const __grid_constant__ Params p) {
  using C = Cfg<D>;
  static_assert(!kPair || D == 128, "pair mode is laid out for d = 128");
  static_assert(!kQT || kPair, "Q-in-TMEM is a pair-mode layout");
  constexpr int BN = kQT ? 64 : kBN;  // keys per KV tile
  constexpr bool kSplit = !kQT || FWD_QT_SPLIT;  // two softmax warps per row (column halves)
  constexpr int kHW = kSplit ? BN / 2 : BN;       // keys per softmax thread
  constexpr int kArr = kSplit ? 16 : 8;           // pair: softmax-warp arrivals (both CTAs) per tile
  constexpr int kSt = kQT ? C::kQTStages : kPair ? C::kPairStages : C::kStages;
  constexpr int kKBytes = kQT ? C::kKHalfQT : kPair ? C::kKHalf : C::kTileBytes;  // per K stage
  constexpr int kVBytes = kQT ? C::kVHalfQT : kPair ? C::kVHalf : C::kTileBytes;  // per V stage
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ[2] = {base, base + C::kTileBytes};
  uint8_t* sK = base + 2 * C::kTileBytes;
  uint8_t* sV = sK + kSt * kKBytes;
  Smem& sm = *reinterpret_cast<Smem*>(base + (kQT ? C::kSmemTilesQT : kPair ? C::kSmemTilesPair : C::kSmemTiles));
  const uint32_t crank = kPair ? cluster_ctarank() : 0;  // 0: the pair's leader (issues the MMAs)
  const int item = kPair ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);

  // ---- work item.  Main items: (q-block pair counted from the sequence end, sequence, kv head)
  // of the two-region problem.  Fused Call 1 items (two-call launch only): the prompt's own
  // queries attend causally to the prompt keys -- one more "sequence" whose own-region K/V are
  // the context tensors and which has no context region.
  // Multi-group launches: a sequence's context region is its group's prompt rows
  // [ctx_row0, ctx_row0 + ctx_len) of the concatenated k_ctx / v_ctx; Call 1 items of group g
  // run the prompt rows of that group.
  const bool self_item = item >= p.n_main_items;
  int hk, jb, seq0, rlen, n_ctx, lse_stride, ctx_row0 = 0, ctx_len = 0;
  const CUtensorMap *mq, *mk_own, *mv_own;
  __nv_bfloat16* out;
  float* lse_out;
  if (!self_item) {
#if FWD_ORDER == 1
    // a (sequence, kv head)'s q blocks side by side: co-resident CTAs share its own K/V stream in L2
    jb = item % p.blocks_per_seq;
    const int rest = item / p.blocks_per_seq;
    hk = rest % p.kv_heads;
    const int seq = rest / p.kv_heads;
#else
    hk = item % p.kv_heads;
    const int rest = item / p.kv_heads;
    const int seq = rest % p.num_seqs;
    jb = rest / p.num_seqs;
#endif
    seq0 = p.cu[seq];
    rlen = p.cu[seq + 1] - seq0;
    const int g = p.grp.group_of(seq);
    ctx_row0 = p.grp.ctx[g];
    ctx_len = p.grp.ctx[g + 1] - ctx_row0;
    n_ctx = (ctx_len + BN - 1) / BN;
    mq = &p.tm_q;
    mk_own = &p.tm_k;
    mv_own = &p.tm_v;
    out = p.out;
    lse_out = p.lse;
    lse_stride = p.total_q;
  } else {
    const int b = item - p.n_main_items;
    hk = b % p.kv_heads;
    const int rest = b / p.kv_heads;
    const int g = rest % p.grp.n;
    jb = rest / p.grp.n;
    seq0 = p.grp.ctx[g];
    rlen = p.grp.ctx[g + 1] - seq0;
    n_ctx = 0;
    mq = &p.tm_qs;
    mk_own = &p.tm_kc;
    mv_own = &p.tm_vc;
    out = p.out_s;
    lse_out = p.lse_s;
    lse_stride = p.ctx_len;
  }
  const int span_tok = (kPair ? 4 : 2) * p.tq;  // tokens of the item (two or four Q tiles)
  const int nblk = (rlen + span_tok - 1) / span_tok;
  if (jb >= nblk) return;  // (both CTAs of a pair: same item)
  const int tok_item = (nblk - 1 - jb) * span_tok;
  const int tok0 = tok_item + static_cast<int>(crank) * 2 * p.tq;  // first token of this CTA's tile A
  // pair mode always runs both tiles (the leader's M = 256 MMAs cover both CTAs); rows past the
  // sequence end are computed on zero / foreign rows and never stored
  const bool has_b = kPair || tok0 + p.tq < rlen;
  const int last_tok = min(tok_item + span_tok, rlen) - 1;  // the item's walk: the whole cluster
  const int n_own = last_tok / BN + 1;
  const int n_iter = n_own + n_ctx;

  const int warp = warp_id();
  const int lane = lane_id();

  if (threadIdx.x == 0) {
    mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kSt; ++i) {
      mbar_init(&sm.k_full[i], 1);
      mbar_init(&sm.k_empty[i], 1);
      mbar_init(&sm.v_full[i], 1);
      mbar_init(&sm.v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.p_full[i], kPair ? kArr : 256);  // pair: one arrival per softmax warp of both CTAs
      mbar_init(&sm.o_full[i], 1);
      mbar_init(&sm.q_tm[i], kArr);
    }
    fence_mbar_init();
  }
  if (warp == kWProd) {
    if constexpr (kPair)
      tmem_alloc2<512>(&sm.tmem_base);
    else
      tmem_alloc<512>(&sm.tmem_base);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync();  // the leader's barriers exist before any 2-SM TMA / arrive
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  // iteration -> (is_ctx, tile index); own tiles from the diagonal down, then context
  auto tile_of = [&](int it, bool& is_ctx) {
    if (it < n_own) {
      is_ctx = false;
      return n_own - 1 - it;
    }
    is_ctx = true;
    return n_ctx - 1 - (it - n_own);
  };

  // teardown without a common tail (each role keeps its own register budget to the end): all
  // warps arrive on barrier 15 when done with TMEM; the allocating warp waits there and frees it
  // (pair mode: a cluster barrier phase instead, so neither CTA frees the pair's TMEM early)
  auto done = [&]() {
    tc_fence_before();
    if constexpr (kPair)
      cluster_arrive();
    else
      named_bar_arrive(15, kThreads);
  };

  if (warp == kWProd) {
    // ================= TMA producer
    if (elect_one()) {
      tma_prefetch(mq);
      tma_prefetch(mk_own);
      tma_prefetch(mv_own);
      if (n_ctx > 0) {
        tma_prefetch(&p.tm_kc);
        tma_prefetch(&p.tm_vc);
      }
      const uint64_t pol_kv = policy_evict_last();
      const uint64_t pol_own = FWD_EVICT == 1 ? policy_evict_normal() : policy_evict_first();
      if constexpr (kQT) {
        // Q is read only by this CTA's own threads (copied into TMEM): a local 1-SM load
        mbar_arrive_expect_tx(&sm.q_full, 2 * C::kTileBytes);
        for (int t = 0; t < 2; ++t)
          for (int pn = 0; pn < C::kPanels; ++pn)
            tma_load_3d(sQ[t] + pn * C::kPanelBytes, mq, &sm.q_full, pn * 64, hk * p.group, seq0 + tok0 + t * p.tq);
      } else if constexpr (kPair) {
        if (crank == 0) mbar_arrive_expect_tx(&sm.q_full, 4 * C::kTileBytes);
        const uint32_t lq = mapa_shared(&sm.q_full, 0);
        for (int t = 0; t < 2; ++t)
          for (int pn = 0; pn < C::kPanels; ++pn)
            tma_load_3d_2sm(sQ[t] + pn * C::kPanelBytes, mq, lq, pn * 64, hk * p.group, seq0 + tok0 + t * p.tq);
      } else {
        // a tile is tq x G rows of 128 B per 64-column panel (< 128 rows when G does not divide 128)
        const int qbytes = p.tq * p.group * 128 * C::kPanels * (has_b ? 2 : 1);
        mbar_arrive_expect_tx(&sm.q_full, qbytes);
        for (int t = 0; t < (has_b ? 2 : 1); ++t)
          for (int pn = 0; pn < C::kPanels; ++pn)
            tma_load_3d(sQ[t] + pn * C::kPanelBytes, mq, &sm.q_full, pn * 64, hk * p.group,
                        seq0 + tok0 + t * p.tq);
      }
      for (int it = 0; it < n_iter; ++it) {
        bool is_ctx;
        const int j = tile_of(it, is_ctx);
        const int slot = it % kSt;
        const uint32_t ph = (it / kSt) & 1;
        const CUtensorMap* mk = is_ctx ? &p.tm_kc : mk_own;
        const CUtensorMap* mv = is_ctx ? &p.tm_vc : mv_own;
        const int row = is_ctx ? ctx_row0 + j * BN : seq0 + j * BN;
        mbar_wait(&sm.k_empty[slot], ph ^ 1);
        TRACE(T_Q_LOAD, it);
        if constexpr (kPair) {
          // this CTA's halves: keys [64 r, +64) of K, d columns [64 r, +64) of V; both counted
          // on the leader's barriers
          const bool ctx_map = is_ctx || self_item;
          const CUtensorMap* mkh = kQT ? (ctx_map ? &p.tm_kc32 : &p.tm_k32) : (ctx_map ? &p.tm_kc64 : &p.tm_k64);
          const CUtensorMap* mvh = kQT ? (ctx_map ? &p.tm_vc64 : &p.tm_v64) : mv;
          if (crank == 0) mbar_arrive_expect_tx(&sm.k_full[slot], 2 * kKBytes);
          const uint32_t lk = mapa_shared(&sm.k_full[slot], 0);
          for (int pn = 0; pn < C::kPanels; ++pn)
            tma_load_3d_2sm(sK + slot * kKBytes + pn * (kKBytes / 2), mkh, lk, pn * 64, hk,
                            row + static_cast<int>(crank) * (BN / 2));
          mbar_wait(&sm.v_empty[slot], ph ^ 1);
          if (crank == 0) mbar_arrive_expect_tx(&sm.v_full[slot], 2 * kVBytes);
          tma_load_3d_2sm(sV + slot * kVBytes, mvh, mapa_shared(&sm.v_full[slot], 0), static_cast<int>(crank) * 64,
                          hk, row);
          continue;
        }
        const bool skip_kv = (DKV_ABL(p.ablate) & 1) || ((DKV_ABL(p.ablate) & 4) && it >= C::kStages);  // 4: reuse the first tiles
        // L2 policy: the shared prompt's K/V is re-read by every sequence's items -> evict_last;
        // a sequence's own K/V only by that sequence's few items (FWD_EVICT selects, see top)
        const uint64_t pol = (is_ctx || FWD_EVICT == 0) ? pol_kv : pol_own;
        mbar_arrive_expect_tx(&sm.k_full[slot], skip_kv ? 0 : C::kTileBytes);
        for (int pn = 0; pn < C::kPanels && !skip_kv; ++pn)
          tma_load_3d_hint(sK + slot * C::kTileBytes + pn * C::kPanelBytes, mk, &sm.k_full[slot], pn * 64, hk,
                           row, pol);
        mbar_wait(&sm.v_empty[slot], ph ^ 1);
        mbar_arrive_expect_tx(&sm.v_full[slot], skip_kv ? 0 : C::kTileBytes);
        for (int pn = 0; pn < C::kPanels && !skip_kv; ++pn)
          tma_load_3d_hint(sV + slot * C::kTileBytes + pn * C::kPanelBytes, mv, &sm.v_full[slot], pn * 64, hk,
                           row, pol);
      }
    }
    __syncwarp();
    tc_fence_before();
    if constexpr (kPair) {
      cluster_arrive();
      cluster_wait();  // every thread of both CTAs is done with the pair's TMEM
      tc_fence_after();
      tmem_dealloc2<512>(tmem);
    } else {
      named_bar_sync(15, kThreads);
      tc_fence_after();
      tmem_dealloc<512>(tmem);
    }
  } else if (warp == kWMma) {
    // ================= MMA issuer (one thread)
    if ((!kPair || crank == 0) && elect_one()) {
      constexpr int kM = kPair ? 2 * kBM : kBM;
      const uint32_t idesc_s = idesc_bf16_f32(kM, BN, false, false);
      const uint32_t idesc_o = idesc_bf16_f32(kM, D, false, true);
      const uint32_t tS[2] = {tmem + 0, tmem + BN};
      const uint32_t tQ[2] = {tmem + 128, tmem + 192};  // kQT only
      const uint32_t tO[2] = {tmem + 256, tmem + 256 + 128};
      const int ntile = has_b ? 2 : 1;
      auto issue_s = [&](int t, int kslot) {
        const uint32_t qa = smem_u32(sQ[t]);
        const uint32_t ka = smem_u32(sK + kslot * kKBytes);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * C::kPanelBytes + (k & 3) * 32;
          if constexpr (kPair) {
            const uint32_t koff = (k >> 2) * (kKBytes / 2) + (k & 3) * 32;  // (BN / 2)-row K panels
            if constexpr (kQT)
              mma_ts2(tS[t], tQ[t] + k * 8, sdesc_sw128(ka + koff, 16, 1024), idesc_s, k > 0);
            else if (DKV_ABL(p.ablate) & 8)  // energy experiment (trace build): A from TMEM (the O
              // columns, garbage values) -- the S MMA without its Q shared-memory reads
              mma_ts2(tS[t], tO[t] + k * 8, sdesc_sw128(ka + koff, 16, 1024), idesc_s, k > 0);
            else
              mma_ss2(tS[t], sdesc_sw128(qa + off, 16, 1024), sdesc_sw128(ka + koff, 16, 1024), idesc_s, k > 0);
          } else {
            mma_ss(tS[t], sdesc_sw128(qa + off, 16, 1024), sdesc_sw128(ka + off, 16, 1024), idesc_s, k > 0);
          }
        }
      };
      auto issue_pv = [&](int t, int vslot, bool accum) {
        const uint32_t va = smem_u32(sV + vslot * kVBytes);
#pragma unroll
        for (int k = 0; k < BN / 16; ++k) {
          if constexpr (kPair)
            mma_ts2(tO[t], tS[t] + k * 8, sdesc_sw128(va + k * 2048, C::kPanelBytes, 1024), idesc_o,
                    (accum || k > 0) ? 1u : 0u);
          else
            mma_ts(tO[t], tS[t] + k * 8, sdesc_sw128(va + k * 2048, C::kPanelBytes, 1024), idesc_o,
                   (accum || k > 0) ? 1u : 0u);
        }
      };
      auto commit = [&](uint64_t* bar) {
        if constexpr (kPair)
          mma_commit2_mc(bar);
        else
          mma_commit(bar);
      };
      // pair mode: these barriers complete from the peer CTA too -> poll (see mbar_wait_poll)
      // (FWD_SPIN: 1 test_wait spin, 2 try_wait without a suspend hint -- see mbar_spin)
      auto wait = [&](uint64_t* bar, uint32_t ph) {
        if constexpr (kPair)
          mbar_wait_poll(bar, ph);
        else if constexpr (FWD_SPIN == 1)
          mbar_spin(bar, ph);
        else if constexpr (FWD_SPIN == 2)
          mbar_wait_nohint(bar, ph);
        else
          mbar_wait(bar, ph);
      };
      if constexpr (!kQT) wait(&sm.q_full, 0);
      wait(&sm.k_full[0], 0);
      tc_fence_after();
      for (int t = 0; t < ntile; ++t) {
        if constexpr (kQT) {
          wait(&sm.q_tm[t], 0);  // both CTAs' softmax warps copied Q tile t into TMEM
          tc_fence_after();
        }
        issue_s(t, 0);
        commit(&sm.s_full[t]);
      }
      commit(&sm.k_empty[0]);
      for (int it = 0; it < n_iter; ++it) {
        const int vslot = it % kSt;
        const uint32_t vph = (it / kSt) & 1;
        const int nslot = (it + 1) % kSt;
        const uint32_t nph = ((it + 1) / kSt) & 1;
        const bool more = it + 1 < n_iter;
        wait(&sm.v_full[vslot], vph);
        if (more) wait(&sm.k_full[nslot], nph);
        for (int t = 0; t < ntile; ++t) {
          wait(&sm.p_full[t], it & 1);  // pair: arrivals from both CTAs
          tc_fence_after();
          TRACE(t == 0 ? T_ISS_DV : T_ISS_DK, it);
          issue_pv(t, vslot, it > 0);
          if (t == ntile - 1) commit(&sm.v_empty[vslot]);
          if (more) {
            TRACE(t == 0 ? T_ISS_S : T_ISS_DP, it + 1);
            issue_s(t, nslot);
            commit(&sm.s_full[t]);
            if (t == ntile - 1) commit(&sm.k_empty[nslot]);
          } else {
            commit(&sm.o_full[t]);
          }
        }
      }
    }
    __syncwarp();
    done();
  } else {
    // ================= softmax: two warps per row quadrant and tile, thread = one row x 64
    // keys (column half h).  One warp per sub-partition is latency-bound (tools/trace_fwd.py:
    // ~2000 clk for a 128-key row), two interleave.  The halves exchange partial row maxima
    // through shared memory (named barrier per warp pair) and take identical rescale decisions;
    // each keeps a partial row sum, combined once in the epilogue.
    const int t = warp >> 3;
    const int h = (warp >> 2) & 1;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int bar_id = 1 + t * 4 + q;  // the two warps (h = 0, 1) of this row quadrant
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t tS = tmem + lane_off + t * BN;
    const uint32_t tO = tmem + lane_off + 256 + t * 128;
    const bool tile_ok = (t == 0) || has_b;
    const int qtok = tok0 + t * p.tq + row / p.group;  // sequence-local token of this row
    const int head = hk * p.group + row % p.group;
    // G not dividing 128 (e.g. Qwen3-14B, G = 5): a tile holds tq = 128 / G (floored) tokens x G
    // heads; its last 128 - tq G rows are padding (stale smem rows, computed, never stored)
    const bool row_valid = tile_ok && qtok < rlen && row < p.tq * p.group;
    const int qmin = tok0 + t * p.tq;                  // first token of the tile
    const int hh = kSplit ? h : 0;                     // column half of this warp (0: whole row)
    const int cb = kHW * hh;                           // first key column of this half
    constexpr int kDH = kSplit ? D / 2 : D;            // O columns this warp rescales / stores
    float m_run = -INFINITY, l_run = 0.f;
    if (!kSplit && h == 1) {
      done();
      return;
    }
    if constexpr (kQT) {
      // Q tile t -> TMEM (the S MMA's A operand): this thread's row, d columns [64 h, +64) = one
      // SW128 panel row = 32 columns of bf16 pairs
      mbar_wait(&sm.q_full, 0);
#pragma unroll 1
      for (int pn = kSplit ? h : 0; pn < (kSplit ? h + 1 : 2); ++pn) {
        const uint8_t* qp = sQ[t] + pn * C::kPanelBytes;
        uint32_t u[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 v = *reinterpret_cast<const uint4*>(qp + sw128_offset(row, c));
          u[4 * c] = v.x;
          u[4 * c + 1] = v.y;
          u[4 * c + 2] = v.z;
          u[4 * c + 3] = v.w;
        }
        tmem_st32(tmem + lane_off + 128 + t * 64 + pn * 32, u);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (crank == 0)
          mbar_arrive(&sm.q_tm[t]);
        else
          mbar_arrive_remote_relaxed(mapa_shared(&sm.q_tm[t], 0));
      }
    }
    if (tile_ok) {
      for (int it = 0; it < n_iter; ++it) {
        bool is_ctx;
        const int j = tile_of(it, is_ctx);
        mbar_wait(&sm.s_full[t], it & 1);
        tc_fence_after();
        if (threadIdx.x == 0) TRACE(T_C_S, it);
        float s[kHW];
        {
          uint32_t u[kHW];
#pragma unroll
          for (int c = 0; c < kHW; c += 32) tmem_ld32(tS + cb + c, *reinterpret_cast<uint32_t(*)[32]>(&u[c]));
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < kHW; ++i) s[i] = __uint_as_float(u[i]);
        }
        if (threadIdx.x == 0) TRACE(T_C_DP, it);
        // masks: own tiles on/after the tile's first token are causal; the last
        // context tile may be partial (keys >= P are out of bounds)
        const int kbase = j * BN + cb;
        const bool need_mask = is_ctx ? (kbase + kHW > ctx_len) : (kbase + kHW - 1 > qmin);
        if (need_mask) {
          const int lim = is_ctx ? ctx_len - 1 - kbase : qtok - kbase;  // last visible column
#pragma unroll
          for (int c = 0; c < kHW; ++c)
            if (c > lim) s[c] = -INFINITY;
        }
        // partial row max (8 independent FMNMX3 chains), then the other half's through smem
        float m8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) m8[i] = fmax3(s[i], s[8 + i], s[16 + i]);
#pragma unroll
        for (int c = 24; c < kHW - 8; c += 16)
#pragma unroll
          for (int i = 0; i < 8; ++i) m8[i] = fmax3(m8[i], s[c + i], s[c + 8 + i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) m8[i] = fmaxf(m8[i], s[kHW - 8 + i]);
        float mx = fmaxf(fmax3(m8[0], m8[1], m8[2]), fmax3(fmax3(m8[3], m8[4], m8[5]), m8[6], m8[7]));
        if constexpr (kSplit) {
          sm.xch[t][it & 1][h][row] = mx;
          named_bar_sync(bar_id, 64);  // also: both halves' S loads are done before P overwrites S
          mx = fmaxf(mx, sm.xch[t][it & 1][h ^ 1][row]);
        }
        if (threadIdx.x == 0) TRACE(T_ISS_DQ, it);
        const float m_tile = mx * p.scale_log2;
        const float m_new = fmaxf(m_run, m_tile);
        float alpha = 1.f;
        if (m_new > m_run + kRescaleThreshold) {
          alpha = ex2(m_run - m_new);
          m_run = m_new;
        }
        const float m_use = m_run == -INFINITY ? 0.f : m_run;
        // x = s * scale * log2(e) - m in packed f32x2 (FFMA2), then 2^x: kPolyPairs of every
        // 16 pairs on the FMA pipe (polynomial, f32x2) to unload the MUFU pipe; row sum in FADD2
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        const float2 nm2 = make_float2(-m_use, -m_use);
        float2 rs2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c0 = 0; c0 < kHW; c0 += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 x = __ffma2_rn(make_float2(s[c0 + 2 * i], s[c0 + 2 * i + 1]), sc2, nm2);
            float2 e;
            if (DKV_ABL(p.ablate) & 2) {
              e = x;
            } else if (i >= 16 - kPolyPairs) {
              e = ex2_poly2(x);
            } else {
              e.x = ex2(x.x);
              e.y = ex2(x.y);
            }
            rs2[i & 3] = __fadd2_rn(rs2[i & 3], e);
            pk[i] = pack_bf16(e.x, e.y);
          }
          tmem_st16(tS + (cb + c0) / 2, pk);  // P (bf16 pairs) over the S columns
        }
        const float2 rsum = __fadd2_rn(__fadd2_rn(rs2[0], rs2[1]), __fadd2_rn(rs2[2], rs2[3]));
        l_run = l_run * alpha + (rsum.x + rsum.y);
        // O holds P V of iterations < it (its MMA completed before S(it) did); each half
        // rescales its D/2 columns
        if (it > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
          for (int c0 = hh * kDH; c0 < (hh + 1) * kDH; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tO + c0, r);
            tmem_wait_ld();
            const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float2 v = __fmul2_rn(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), a2);
              r[i] = __float_as_uint(v.x);
              r[i + 1] = __float_as_uint(v.y);
            }
            tmem_st32(tO + c0, r);
          }
        }
        if (threadIdx.x == 0) TRACE(T_MMA_END, it);
        tmem_wait_st();
        tc_fence_before();
        if constexpr (kPair) {
          __syncwarp();
          if (lane == 0) {
            if (crank == 0)
              mbar_arrive(&sm.p_full[t]);
            else
              mbar_arrive_remote_relaxed(mapa_shared(&sm.p_full[t], 0));  // P in TMEM: nothing to publish
          }
        } else {
          mbar_arrive(&sm.p_full[t]);
        }
        if (threadIdx.x == 0) TRACE(T_C_P, it);
        if (threadIdx.x == 7 * 32) TRACE(T_D_END, it);  // the tile's last softmax warp (trace only)
      }
      // ---- epilogue: l = both halves' partial sums; O / l -> bf16 (each half D/2 columns), lse
      if constexpr (kSplit) {
        sm.xch[t][n_iter & 1][h][row] = l_run;
        named_bar_sync(bar_id, 64);
        l_run += sm.xch[t][n_iter & 1][h ^ 1][row];
      }
      mbar_wait(&sm.o_full[t], 0);
      tc_fence_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      __nv_bfloat16* orow = out + (static_cast<int64_t>(seq0 + qtok) * p.heads + head) * D;
#pragma unroll 1
      for (int c0 = hh * kDH; c0 < (hh + 1) * kDH; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tO + c0, r);
        tmem_wait_ld();
        if (row_valid) {
          uint4 v[4];
          uint32_t* w = reinterpret_cast<uint32_t*>(v);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            w[i] = pack_bf16(__uint_as_float(r[2 * i]) * inv, __uint_as_float(r[2 * i + 1]) * inv);
          uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = v[i];
        }
      }
      if (row_valid && h == 0)
        lse_out[static_cast<int64_t>(head) * lse_stride + seq0 + qtok] =
            (m_run + __log2f(l_run)) * 0.6931471805599453f;
    }
    done();
  }
}

// The CTA-pair (cta_group::2) forward for d = 128 full tiles is the default since the peer's
// P-ready arrive became relaxed (a release at cluster scope was a MEMBAR.ALL.GPU on the chain):
// C3 forward 8.2-8.6 vs 8.5-8.7 ms single-CTA, interleaved (profiles/r2_ab.md).  DKV_FWD_PAIR=0
// selects the single-CTA kernel.
static bool fwd_pairs() {
  static const bool v = [] {
    const char* e = getenv("DKV_FWD_PAIR");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Q as a TMEM operand with 64-key KV tiles (kQT) in the pair forward: DKV_FWD_QT=1.
static bool fwd_qt() {
  static const bool v = [] {
    const char* e = getenv("DKV_FWD_QT");
    return e && e[0] == '1';
  }();
  return v;
}

static const void* pair_fn(bool qt) {
  return qt ? reinterpret_cast<const void*>(dualkv_fwd_kernel<128, true, true>)
            : reinterpret_cast<const void*>(dualkv_fwd_kernel<128, true, false>);
}
static int pair_smem(bool qt) { return qt ? Cfg<128>::kSmemBytesQT : Cfg<128>::kSmemBytesPair; }

// Can a 2-CTA cluster of the pair forward be resident on this device (queried once per device)?
// If not -- e.g. a partitioned device -- the single-CTA kernel runs instead.
static bool pair_launchable(bool qt) {
  static std::mutex mu;
  static std::map<int, bool> ok;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lock(mu);
  const int key = 2 * dev + (qt ? 1 : 0);
  auto it = ok.find(key);
  if (it != ok.end()) return it->second;
  const void* fn = pair_fn(qt);
  bool yes = false;
  if (ensure_smem_optin(fn, pair_smem(qt), "dualkv_fwd_kernel(pair)")) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = pair_smem(qt);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    yes = cudaOccupancyMaxActiveClusters(&n, fn, &cfg) == cudaSuccess && n > 0;
  }
  cudaGetLastError();
  ok[key] = yes;
  return yes;
}

template <int D>
int launch(const SimtArgs& a, const CtxSelf* self, const GroupTable& grp, cudaStream_t st) {
  using C = Cfg<D>;
  Params p{};
  p.grp = grp;
  const int G = a.heads / a.kv_heads;
  const int tq = kBM / G;
  if (a.total_q > 0 &&
      (!make_map_3d_bf16(&p.tm_q, a.q, a.total_q, a.heads, D, G, tq) ||
       !make_map_3d_bf16(&p.tm_k, a.k, a.total_q, a.kv_heads, D, 1, kBN) ||
       !make_map_3d_bf16(&p.tm_v, a.v, a.total_q, a.kv_heads, D, 1, kBN))) {
    set_error("cuTensorMapEncodeTiled failed for q/k/v");
    return DKV_ERR_CUDA;
  }
  if (a.ctx_len > 0) {
    if (!make_map_3d_bf16(&p.tm_kc, a.k_ctx, a.ctx_len, a.kv_heads, D, 1, kBN) ||
        !make_map_3d_bf16(&p.tm_vc, a.v_ctx, a.ctx_len, a.kv_heads, D, 1, kBN)) {
      set_error("cuTensorMapEncodeTiled failed for k_ctx/v_ctx");
      return DKV_ERR_CUDA;
    }
  }
  const bool qt = D == 128 && fwd_qt();
  const bool pair = D == 128 && fwd_pairs() && tq * G == kBM && pair_launchable(qt);  // full tiles only
  if (pair && ((a.total_q > 0 && !make_map_3d_bf16(&p.tm_k64, a.k, a.total_q, a.kv_heads, D, 1, 64)) ||
               (a.ctx_len > 0 && !make_map_3d_bf16(&p.tm_kc64, a.k_ctx, a.ctx_len, a.kv_heads, D, 1, 64)))) {
    set_error("cuTensorMapEncodeTiled failed for the pair-mode K maps");
    return DKV_ERR_CUDA;
  }
  if (pair && qt &&
      ((a.total_q > 0 && (!make_map_3d_bf16(&p.tm_k32, a.k, a.total_q, a.kv_heads, D, 1, 32) ||
                          !make_map_3d_bf16(&p.tm_v64, a.v, a.total_q, a.kv_heads, D, 1, 64))) ||
       (a.ctx_len > 0 && (!make_map_3d_bf16(&p.tm_kc32, a.k_ctx, a.ctx_len, a.kv_heads, D, 1, 32) ||
                          !make_map_3d_bf16(&p.tm_vc64, a.v_ctx, a.ctx_len, a.kv_heads, D, 1, 64))))) {
    set_error("cuTensorMapEncodeTiled failed for the Q-in-TMEM K/V maps");
    return DKV_ERR_CUDA;
  }
  const bool with_self = self && a.ctx_len > 0;
  if (with_self && !make_map_3d_bf16(&p.tm_qs, self->q, a.ctx_len, a.heads, D, G, tq)) {
    set_error("cuTensorMapEncodeTiled failed for q_ctx");
    return DKV_ERR_CUDA;
  }
  p.out = static_cast<__nv_bfloat16*>(a.out);
  p.lse = a.lse;
  p.out_s = with_self ? static_cast<__nv_bfloat16*>(self->out) : nullptr;
  p.lse_s = with_self ? self->lse : nullptr;
  p.cu = a.cu;
  p.num_seqs = a.num_seqs;
  p.total_q = a.total_q;
  p.ctx_len = a.ctx_len;
  p.heads = a.heads;
  p.kv_heads = a.kv_heads;
  p.group = G;
  p.tq = tq;
  p.scale_log2 = a.scale * 1.4426950408889634f;
#ifdef DKV_ABLATION  // timing-experiment builds only (libdkv_trace.so); never read by libdkv.so
  {
    const char* e = getenv("DKV_FWD_ABLATE");
    p.ablate = e ? atoi(e) : 0;
  }
#endif
  const int span = (pair ? 4 : 2) * tq;  // tokens per work item (a CTA, or a CTA pair)
  const int blocks_per_seq = a.total_q > 0 ? (a.max_seqlen + span - 1) / span : 0;
  const int64_t main_items = static_cast<int64_t>(blocks_per_seq) * a.num_seqs * a.kv_heads;
  const int64_t self_items =
      with_self ? static_cast<int64_t>((grp.max_ctx + span - 1) / span) * grp.n * a.kv_heads : 0;
  const int64_t items = main_items + self_items;  // Call 1 items run in the tail of Call 2's
  if (items == 0) return DKV_OK;
  if (items * (pair ? 2 : 1) > 0x7fffffff) {
    set_error("forward grid too large");
    return DKV_ERR_UNSUPPORTED;
  }
  p.n_main_items = static_cast<int>(main_items);
  p.blocks_per_seq = blocks_per_seq;
  if (pair) {
    if (!ensure_smem_optin(pair_fn(qt), pair_smem(qt), "dualkv_fwd_kernel(pair)")) return DKV_ERR_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * items));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = pair_smem(qt);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = qt ? cudaLaunchKernelEx(&cfg, dualkv_fwd_kernel<128, true, true>, p)
                             : cudaLaunchKernelEx(&cfg, dualkv_fwd_kernel<128, true, false>, p);
    if (e != cudaSuccess) {
      set_error(std::string("forward pair launch failed: ") + cudaGetErrorString(e));
      return DKV_ERR_CUDA;
    }
    return DKV_OK;
  }
  if (!ensure_smem_optin(reinterpret_cast<const void*>(dualkv_fwd_kernel<D, false>), C::kSmemBytes,
                         "dualkv_fwd_kernel"))
    return DKV_ERR_CUDA;
  dualkv_fwd_kernel<D, false><<<static_cast<unsigned>(items), kThreads, C::kSmemBytes, st>>>(p);
  return DKV_OK;
}

}  // namespace fwd

DKV_TRACE_READ_FN(dkv_trace_read_fwd)

bool force_simt() {
  static const bool f = [] {
    const char* e = getenv("DKV_FORCE_SIMT");
    return e && e[0] == '1';
  }();
  return f;
}

bool tc_supported(int dtype, int head_dim, int heads, int kv_heads) {
  if (dtype != DKV_BF16 || force_simt()) return false;
  if (head_dim != 64 && head_dim != 128) return false;
  if (kv_heads <= 0 || heads % kv_heads) return false;
  const int G = heads / kv_heads;
  return G <= 128;  // a 128-row query tile holds floor(128 / G) tokens x G heads
}

int launch_tc_fwd(const SimtArgs& a, const CtxSelf* self, const GroupTable& grp, cudaStream_t st) {
  if (a.head_dim == 128) return fwd::launch<128>(a, self, grp, st);
  return fwd::launch<64>(a, self, grp, st);
}

}  // namespace dkv
