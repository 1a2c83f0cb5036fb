// bwd_pair_sm100.cu -- CTA-pair (cta_group::2) backward for DualKV attention, head_dim 128.
//
// Same KV-stationary algorithm as bwd_sm100.cu (SURVEY §7.4 design (C)), but a 2-CTA cluster
// owns TWO adjacent 128-key tiles (CTA r: key tile 2 kp + r) and both CTAs sweep the SAME 64-row
// GQA-packed query tiles.  Every GEMM is one tcgen05.mma.cta_group::2 issued by the leader:
//
//   S^T  = K Q^T      M256 (keys of both CTAs)  N64  K128   B = Q^T split by query half:
//   dP^T = V dO^T     M256                      N64  K128     CTA r streams rows [32 r, +32)
//   dV  += P^T dO     M256  N128 (d halves)  K64   TS, B = dO split by head-dim half
//   dK  += dS^T Q     M256  N128             K64   TS, B = Q split by head-dim half
//   dQ^T = K^T dS^T   M128 (d: 64 per CTA)   N64  K256 (BOTH key tiles)
//
// The last one is the point of the pair: dQ^T of a query tile is summed over 256 keys inside the
// tensor core, so the fp32 dQ reduce-add into dq_acc (the backward's L2 reduction stream,
// profiles/r2_l2_reductions.md) and its shared-memory staging halve.  Its B operand needs each
// CTA's dS^T for the other CTA's query half: the compute warps store that half straight into the
// peer's shared memory (st.shared::cluster, 8 KB per tile), the rest locally.  The B operands of
// S^T / dP^T / dV / dK are split between the CTAs, so shared-memory operand reads per tile drop
// from ~188 KB to ~154 KB.  TMEM per CTA: S^T [0,64) dP^T [64,128) P^T [128,160) dS^T [160,192)
// dQ^T 2 x [192,224) (double-buffered: an M=128 pair tile folds its 64 query columns onto 32
// columns x 128 lanes -- lane = d + 64 (q / 32), column = q % 32, measured by
// tools/ubench/pair_dq.cu) dV [256,384) dK [384,512).
//
// Roles: warps 0-7 compute (thread = key row, 32 query columns per warp), 8-11 dQ drain (two query
// halves, reduced independently), 12 TMA producer, 13 / 14 MMA issuers of the leader (S^T / dP^T;
// dV / dK / dQ^T) -- warp 14 of the peer forwards the arrival of the leader's dS^T half.  Barriers
// the leader's issuers wait on receive arrivals from both CTAs; pair-MMA completions are multicast
// to the same barrier offset in both CTAs.  Cross-CTA arrivals that publish nothing are relaxed (a
// release at cluster scope is a MEMBAR.ALL.GPU); the dS^T exchange uses st.async with complete_tx.
//
// Status (profiles/r2_pair_bwd.md): correct on every GPU test; ncu shows what the design buys --
// tensor-core smem wavefronts 73 % -> 53 %, LSU smem 26 % -> 16 %, L2 throughput 50 % -> 29 %,
// SM clock +11 % at the same 1000 W -- but the cross-CTA handshakes lengthen the per-tile chain
// (tensor pipe 65 % -> 58 % active), and at C3 it runs 26.6 vs 25.9 ms.  Opt-in (DKV_BWD_PAIR=1).
#include "dkv_internal.h"
#include "tma_host.h"
#include "trace.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace dkv {
namespace bwdp {

constexpr int D = 128;
constexpr int kBK = 128;            // keys per CTA
constexpr int kBQ = 64;             // query rows per tile
#ifndef PAIR_CW
#define PAIR_CW 8  // compute warps: 8 (32 query columns each) or 16 (16 columns each)
#endif
constexpr int kCW = PAIR_CW;
constexpr int kCC = 256 / kCW;  // query columns per compute warp (4 lane quadrants x 64 columns)
static_assert(kCW == 8 || kCW == 16, "PAIR_CW: 8 or 16");
constexpr int kWDrain = kCW, kWProd = kCW + 4, kWMma = kCW + 5, kWMma2 = kCW + 6;
constexpr int kThreads = (kCW + 7) * 32;
constexpr int kNSt = 2;  // stages of the query-half operands (S^T / dP^T)
constexpr int kKSt = 2;  // stages of the head-dim-half operands (dV / dK), needed one tile later
constexpr int kPanel = kBK * 128;   // 16 KB: one 64-column SW128 panel of a 128-row key tile
// shared memory (bytes from the 1024-aligned base)
constexpr int kOffK = 0;                      // own K tile, 2 panels (A of S^T, K-major)
constexpr int kOffV = kOffK + 2 * kPanel;     // own V tile
constexpr int kOffKT = kOffV + 2 * kPanel;    // [256 keys][64 d of this CTA's half] (A of dQ^T, MN-major)
constexpr int kQN = 32 * 128 * 2;             // 8 KB: [32 rows][128 d] (2 panels of 4 KB)
constexpr int kQK = kBQ * 128;                // 8 KB: [64 rows][64 d] (one panel)
constexpr int kOffQN = kOffKT + 2 * kPanel;            // per n stage: qn, don
constexpr int kOffQK = kOffQN + kNSt * 2 * kQN;         // per k stage: qk, dok
constexpr int kOffDS = kOffQK + kKSt * 2 * kQK;         // 2 x [256 keys][32 q] SW64 (B of dQ^T)
constexpr int kDSBytes = 256 * 64;
constexpr int kXBytes = 32 * 32;                       // [32 rows][16 bf16] SW32
constexpr int kOffX = kOffDS + 2 * kDSBytes;           // per stage: -lse/scale rows, -D rows
constexpr int kOffOnes = kOffX + kNSt * 2 * kXBytes;
constexpr int kOffStg = kOffOnes + kBK * 32;           // dQ staging [64 q][64 d] fp32
constexpr int kStgBytes = kBQ * 64 * 4;
constexpr int kOffBar = kOffStg + kStgBytes;
constexpr int kSmemBytes = kOffBar + 256 + 1024;
static_assert(kSmemBytes <= 232448, "exceeds the 227 KB opt-in shared memory per block");

struct Params {
  CUtensorMap tm_q, tm_do, tm_qh, tm_doh, tm_k, tm_v, tm_kc, tm_vc, tm_dq, tm_xh;
  CUtensorMap tm_qs, tm_dos, tm_qsh, tm_dosh, tm_xsh, tm_dqs;  // fused Call 1
  int tpad_s, n_self_items, self_part;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  float* ctx_acc;
  const int32_t* cu;
  int num_seqs, total_q, ctx_len, heads, kv_heads, group, tq, tpad;
  int chunk, n_ctx_items, n_ctx_pairs, max_own_pairs;
  int atomic_ctx;
  float scale, scale_log2;
  GroupTable grp;
};

struct Bars {
  // pds_full: P^T / dS^T of a tile in both CTAs' TMEM (+ local dS^T smem writes); p_empty: dV / dK
  // done with them; ds_in[b] / ds_empty[b]: the double-buffered dS^T operand of dQ^T (the other
  // CTA's st.async half arrived / dQ^T done with it)
  uint64_t kv_full, sdp_full, sdp_empty, pds_full, p_empty, kv_done, ds_in[2], ds_empty[2];
  // per stage: the query-half operands of S^T / dP^T (+ the additive-constant rows) are released
  // as soon as those MMAs complete ("n" part), the head-dim-half operands of dV / dK after them
  uint64_t qn_full[kNSt], qn_empty[kNSt], qk_full[kKSt], qk_empty[kKSt];
  uint64_t dq_full[2], dq_empty[2];
  uint32_t tmem_base;
};

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

// SWIZZLE_64B MN-major operand: rows of 64 B (32 bf16), 8-row atoms of 512 B
DKV_DEVICE uint64_t sdesc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(512 >> 4) << 32;  // SBO: next 8-row group along K
  d |= 1ull << 46;
  d |= 4ull << 61;
  return d;
}
DKV_DEVICE uint32_t sw64_offset(uint32_t r, uint32_t c) { return r * 64u + ((c ^ ((r >> 1) & 3u)) << 4); }

DKV_DEVICE void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
// 16 B into the PEER's shared memory, completion (tx bytes) counted on the peer's mbarrier `rbar`
DKV_DEVICE void st_async_v4(uint32_t raddr, uint32_t rbar, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%2, %3, %4, %5}, [%1];" ::"r"(
                   raddr),
               "r"(rbar), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
// Arrivals that only report "my TMEM loads are done" (no memory to publish): relaxed, so a
// remote arrive is a plain SYNCS.ARRIVE.RED -- a release at cluster scope compiles to
// MEMBAR.ALL.GPU, which traced at ~1500 clk per tile in this kernel.
DKV_DEVICE void warp_arrive_leader_relaxed(uint64_t* bar, uint32_t rank) {
  __syncwarp();
  if (lane_id() == 0) {
    if (rank == 0)
      mbar_arrive(bar);
    else
      asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(bar, 0))
                   : "memory");
  }
}

// Waits of the pair kernel.  A thread suspended in try_wait was traced waking several hundred clk
// after an arrival from the other CTA (remote arrive, multicast commit, 2-SM TMA), but polling
// (test_wait.acquire.cluster, with or without a nanosleep backoff) by several warps per
// sub-partition starved the compute warps of issue slots and measured slower overall (C3: spin
// 28.4, 32 ns backoff 27.5, 128 ns 27.9, suspend 27.0 ms).  PAIR_NS: -1 suspend (default), else the
// polling backoff in ns.
#ifndef PAIR_POLY
#define PAIR_POLY 0  // of every 16 exponential pairs, computed on the FMA pipe
#endif
#ifndef PAIR_NS
#define PAIR_NS -1
#endif
#ifndef PAIR_DS_EARLY
#define PAIR_DS_EARLY 1  // dS^T operand stores before the P^T / dS^T TMEM stores (C3: 25.91 vs 26.09 ms)
#endif
#ifndef PAIR_NS_C
#define PAIR_NS_C PAIR_NS  // compute warps' waits (S ready, P^T / dS^T buffers free)
#endif
#ifndef PAIR_NS_I
#define PAIR_NS_I PAIR_NS  // MMA issuers' and the peer forwarder's waits
#endif
template <int NS = PAIR_NS>
DKV_DEVICE void pwait(uint64_t* bar, uint32_t parity) {
  if constexpr (NS < 0) {
    mbar_wait(bar, parity);
  } else {
    for (;;) {
      uint32_t ok;
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(ok)
          : "r"(smem_u32(bar)), "r"(parity)
          : "memory");
      if (ok) break;
      if constexpr (NS > 0) __nanosleep(NS > 0 ? NS : 0);
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) dualkv_bwd_pair_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars& bar = *reinterpret_cast<Bars*>(base + kOffBar);
  const uint32_t rank = cluster_ctarank();
  const int item = static_cast<int>(blockIdx.x >> 1);

  // ---- work item (identical in both CTAs): kind 0 prompt key-tile pair x chunk (Call 2), kind 2
  // prompt key-tile pair x the prompt's causal queries (fused Call 1), kind 1 own-response key-tile
  // pair of one sequence (Call 2).  Grid order: kinds 0, 2, 1 (longest first).
  int kind, hk, kp, s0, s1, tok_first, kv_len, kv_row0, part = 0;
  if (item < p.n_ctx_items) {
    kind = 0;
    const int per_chunk = p.n_ctx_pairs * p.kv_heads;
    const int cg = item / per_chunk;
    const int rem = item % per_chunk;
    kp = rem % p.n_ctx_pairs;
    hk = rem / p.n_ctx_pairs;
    const int g = cg % p.grp.n;
    const int chunk_id = cg / p.grp.n;
    kv_row0 = p.grp.ctx[g];
    kv_len = p.grp.ctx[g + 1] - kv_row0;
    if (2 * kp * kBK >= kv_len) return;
    s0 = p.grp.seq[g] + chunk_id * p.chunk;
    s1 = min(p.grp.seq[g + 1], s0 + p.chunk);
    if (s0 >= s1) return;
    tok_first = 0;
    part = p.atomic_ctx ? 0 : chunk_id;
  } else if (item >= p.n_ctx_items + p.n_self_items) {
    kind = 1;
    const int b2 = item - p.n_ctx_items - p.n_self_items;
    kp = b2 % p.max_own_pairs;
    const int r2 = b2 / p.max_own_pairs;
    hk = r2 % p.kv_heads;
    s0 = r2 / p.kv_heads;
    s1 = s0 + 1;
    kv_len = p.cu[s0 + 1] - p.cu[s0];
    if (2 * kp * kBK >= kv_len) return;
    tok_first = (2 * kp * kBK / p.tq) * p.tq;
    kv_row0 = p.cu[s0];
  } else {
    kind = 2;
    const int b3 = item - p.n_ctx_items;
    kp = b3 % p.n_ctx_pairs;
    hk = (b3 / p.n_ctx_pairs) % p.kv_heads;
    s0 = b3 / (p.n_ctx_pairs * p.kv_heads);
    s1 = s0 + 1;
    kv_row0 = p.grp.ctx[s0];
    kv_len = p.grp.ctx[s0 + 1] - kv_row0;
    if (2 * kp * kBK >= kv_len) return;
    tok_first = (2 * kp * kBK / p.tq) * p.tq;
    part = p.atomic_ctx ? 0 : p.self_part;
  }
  const bool ctx_keys = kind != 1;
  const bool causal = kind != 0;
  const int32_t* cu = kind == 2 ? p.grp.ctx : p.cu;
  const CUtensorMap* mq = kind == 2 ? &p.tm_qs : &p.tm_q;
  const CUtensorMap* mdo = kind == 2 ? &p.tm_dos : &p.tm_do;
  const CUtensorMap* mqh = kind == 2 ? &p.tm_qsh : &p.tm_qh;
  const CUtensorMap* mdoh = kind == 2 ? &p.tm_dosh : &p.tm_doh;
  const CUtensorMap* mxh = kind == 2 ? &p.tm_xsh : &p.tm_xh;
  const CUtensorMap* mdq = kind == 2 ? &p.tm_dqs : &p.tm_dq;
  const int xtpad = kind == 2 ? p.tpad_s : p.tpad;
  const int kbase = (2 * kp + static_cast<int>(rank)) * kBK;  // region-local first key of this CTA
  int nq = 0;
  {
    QIter it;
    it.begin(cu, p.tq, s0, s1, tok_first);
    for (; it.valid(); it.next()) ++nq;
  }
  if (nq == 0) return;  // (both CTAs of the pair: same decision)

  const int warp = warp_id();
  const int lane = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(&bar.kv_full, 1);
    mbar_init(&bar.sdp_full, 1);
    mbar_init(&bar.sdp_empty, 2 * kCW);  // every compute warp of both CTAs
    mbar_init(&bar.pds_full, 2 * kCW);
    mbar_init(&bar.p_empty, 1);
    for (int b = 0; b < 2; ++b) {
      // leader: its issuer's expect_tx arrival, the peer forwarder's (the leader's st.async half
      // landed there) and the 4 + 4 warps that store their half locally; peer: its forwarder's
      mbar_init(&bar.ds_in[b], rank == 0 ? 2 + kCW : 1);
      mbar_init(&bar.ds_empty[b], 1);
    }
    mbar_init(&bar.kv_done, 1);
    for (int i = 0; i < kNSt; ++i) {
      mbar_init(&bar.qn_full[i], 1);
      mbar_init(&bar.qn_empty[i], 1);
    }
    for (int i = 0; i < kKSt; ++i) {
      mbar_init(&bar.qk_full[i], 1);
      mbar_init(&bar.qk_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar.dq_full[i], 1);
      mbar_init(&bar.dq_empty[i], 8);  // 4 drain warps x 2 CTAs
    }
    fence_mbar_init();
  }
  if (warp == kWProd) tmem_alloc2<512>(&bar.tmem_base);
  if (warp < 4) {
    const int r = threadIdx.x;
    const uint32_t ones = 0x3F803F80u;
    uint8_t* row = base + kOffOnes + r * 32;
    const uint32_t sw = (r >> 2) & 1;
    *reinterpret_cast<uint4*>(row + (0 ^ sw) * 16) = make_uint4(ones, 0x3F80u, 0u, 0u);
    *reinterpret_cast<uint4*>(row + (1 ^ sw) * 16) = make_uint4(0u, 0u, 0u, 0u);
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's barriers exist before any remote arrive / 2-SM TMA
  tc_fence_after();
  if (threadIdx.x == 0) TRACE(T_START, 0);
  const uint32_t tmem = bar.tmem_base;
  const int G = p.group;
  const int qrows = p.tq * G;  // 64 (G divides 32)

  if (warp == kWProd) {
    // ================= producer (both CTAs; completions counted on the leader's barriers)
    const CUtensorMap* mk = ctx_keys ? &p.tm_kc : &p.tm_k;
    const CUtensorMap* mv = ctx_keys ? &p.tm_vc : &p.tm_v;
    if (lane == 0) {
      tma_prefetch(mq);
      tma_prefetch(mdo);
      tma_prefetch(mqh);
      tma_prefetch(mdoh);
      tma_prefetch(mdq);
      tma_prefetch(mxh);
      tma_prefetch(mk);
      tma_prefetch(mv);
      const uint32_t lkv = mapa_shared(&bar.kv_full, 0);
      if (rank == 0) mbar_arrive_expect_tx(&bar.kv_full, 2 * 6 * kPanel);
      for (int pn = 0; pn < 2; ++pn) {
        tma_load_3d_2sm(base + kOffK + pn * kPanel, mk, lkv, pn * 64, hk, kv_row0 + kbase);
        tma_load_3d_2sm(base + kOffV + pn * kPanel, mv, lkv, pn * 64, hk, kv_row0 + kbase);
      }
      // A of dQ^T: this CTA's head-dim half of BOTH key tiles (pair order: tile 2 kp first)
      for (int t = 0; t < 2; ++t)
        tma_load_3d_2sm(base + kOffKT + t * kPanel, mk, lkv, static_cast<int>(rank) * 64, hk,
                        kv_row0 + (2 * kp + t) * kBK);
    }
    // lane 0 streams the operands: the query-half ones of tile i (needed first, by S^T / dP^T), then
    // the head-dim-half ones of tile i - 1 (needed by dV / dK one tile later)
    if (lane == 0) {
      QIter it;
      it.begin(cu, p.tq, s0, s1, tok_first);
      int prev_row0 = 0;
      for (int i = 0; i <= nq; ++i) {
        const int row0 = i < nq ? cu[it.s] + it.tok : 0;
        if (i < nq) {
          const int st = i % kNSt;
          const uint32_t ph = (i / kNSt) & 1;
          uint8_t* sq = base + kOffQN + st * 2 * kQN;
          const int tokh = row0 + static_cast<int>(rank) * (p.tq / 2);  // this CTA's query half
          pwait(&bar.qn_empty[st], ph ^ 1);
          TRACE(T_Q_LOAD, i);
          const uint32_t lq = mapa_shared(&bar.qn_full[st], 0);
          if (rank == 0) mbar_arrive_expect_tx(&bar.qn_full[st], 2 * (2 * kQN + 2 * kXBytes));
          for (int pn = 0; pn < 2; ++pn) {
            tma_load_3d_2sm(sq + pn * (kQN / 2), mqh, lq, pn * 64, hk * G, tokh);
            tma_load_3d_2sm(sq + kQN + pn * (kQN / 2), mdoh, lq, pn * 64, hk * G, tokh);
          }
          const int xrow = (hk * xtpad + row0) * G + static_cast<int>(rank) * 32;
          uint8_t* sx = base + kOffX + st * 2 * kXBytes;
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(sx)),
              "l"(reinterpret_cast<uint64_t>(mxh)), "r"(lq), "r"(0), "r"(xrow)
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(sx + kXBytes)),
              "l"(reinterpret_cast<uint64_t>(mxh)), "r"(lq), "r"(16), "r"(xrow)
              : "memory");
        }
        if (i > 0) {
          const int j = i - 1;
          const int st = j % kKSt;
          uint8_t* sq = base + kOffQK + st * 2 * kQK;
          pwait(&bar.qk_empty[st], ((j / kKSt) & 1) ^ 1);
          TRACE(T_KLOAD, j);
          const uint32_t lk = mapa_shared(&bar.qk_full[st], 0);
          if (rank == 0) mbar_arrive_expect_tx(&bar.qk_full[st], 2 * 2 * kQK);
          tma_load_3d_2sm(sq, mq, lk, static_cast<int>(rank) * 64, hk * G, prev_row0);
          tma_load_3d_2sm(sq + kQK, mdo, lk, static_cast<int>(rank) * 64, hk * G, prev_row0);
        }
        prev_row0 = row0;
        if (i < nq) it.next();
      }
    }
  } else if (warp == kWMma || warp == kWMma2) {
    // ================= MMA issuers (leader only), two threads so that neither chain waits behind
    // the other: warp 13 issues S^T / dP^T of tile i as soon as the compute warps have read tile
    // i - 1's, warp 14 issues dV / dK / dQ^T of tile j once its P^T / dS^T are stored.  (Each
    // thread's commits track its own MMAs; the two chains touch disjoint TMEM columns.)
    const uint32_t tS = tmem, tdP = tmem + 64, tP = tmem + 128, tDS = tmem + 160, tdQ = tmem + 192;
    const uint32_t tdV = tmem + 256, tdK = tmem + 384;
    auto koff_kv = [](int k) { return static_cast<uint64_t>(((k >> 2) * kPanel + (k & 3) * 32) >> 4); };
    auto koff_qn = [](int k) { return static_cast<uint64_t>(((k >> 2) * (kQN / 2) + (k & 3) * 32) >> 4); };
    auto koff_mn = [](int k) { return static_cast<uint64_t>((k * 2048) >> 4); };
    if (rank == 0 && warp == kWMma && elect_one()) {
      const uint32_t id_sdp = idesc_bf16_f32(2 * kBK, kBQ, false, false);
      const uint64_t dKk = sdesc_sw128(smem_u32(base + kOffK), 16, 1024);
      const uint64_t dVk = sdesc_sw128(smem_u32(base + kOffV), 16, 1024);
      const uint64_t dOnes = sdesc_sw32(smem_u32(base + kOffOnes));
      pwait<PAIR_NS_I>(&bar.kv_full, 0);
      for (int i = 0; i < nq; ++i) {
        const int st = i % kNSt;
        pwait<PAIR_NS_I>(&bar.qn_full[st], (i / kNSt) & 1);
        if (i > 0) pwait<PAIR_NS_I>(&bar.sdp_empty, (i - 1) & 1);
        tc_fence_after();
        TRACE(T_ISS_S, i);
        const uint32_t sq = smem_u32(base + kOffQN + st * 2 * kQN);
        const uint64_t dQn = sdesc_sw128(sq, 16, 1024);
        const uint64_t dOn = sdesc_sw128(sq + kQN, 16, 1024);
        const uint64_t dX = sdesc_sw32(smem_u32(base + kOffX + st * 2 * kXBytes));
#pragma unroll
        for (int k = 0; k < D / 16; ++k) mma_ss2(tS, dKk + koff_kv(k), dQn + koff_qn(k), id_sdp, k > 0);
        mma_ss2(tS, dOnes, dX, id_sdp, 1u);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) mma_ss2(tdP, dVk + koff_kv(k), dOn + koff_qn(k), id_sdp, k > 0);
        mma_ss2(tdP, dOnes, dX + (kXBytes >> 4), id_sdp, 1u);
        mma_commit2_mc(&bar.sdp_full);
        mma_commit2_mc(&bar.qn_empty[st]);
        TRACE(T_SISS_END, i);
      }
    } else if (rank == 0 && warp == kWMma2 && elect_one()) {
      const uint32_t id_kv = idesc_bf16_f32(2 * kBK, D, false, true);
      const uint32_t id_dq = idesc_bf16_f32(128, kBQ, true, true);
      const uint64_t dKT = sdesc_sw128(smem_u32(base + kOffKT), 0, 1024);
      const uint32_t sDS0 = smem_u32(base + kOffDS);
      auto issue_dq = [&](int j) {
        const int b = j & 1;
        pwait<PAIR_NS_I>(&bar.ds_in[b], (j >> 1) & 1);
        TRACE(T_ISS_DK, j);
        pwait<PAIR_NS_I>(&bar.dq_empty[b], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        fence_async_smem();  // the peer's st.async dS^T half -> visible to the tensor core
        TRACE(T_ISS_DQ, j);
        const uint64_t dDS = sdesc_sw64(sDS0 + b * kDSBytes);
#pragma unroll
        for (int k = 0; k < 2 * kBK / 16; ++k)
          mma_ss2(tdQ + b * 32, dKT + koff_mn(k), dDS + static_cast<uint64_t>((k * 1024) >> 4), id_dq, k > 0);
        mma_commit2_mc(&bar.dq_full[b]);
        mma_commit2_mc(&bar.ds_empty[b]);
      };
      pwait<PAIR_NS_I>(&bar.kv_full, 0);
      for (int j = 0; j < nq; ++j) {
        const int sj = j % kKSt;
        const uint32_t sq = smem_u32(base + kOffQK + sj * 2 * kQK);
        const uint64_t dQm = sdesc_sw128(sq, 0, 1024);
        const uint64_t dOm = sdesc_sw128(sq + kQK, 0, 1024);
        const int b = j & 1;
        mbar_arrive_expect_tx(&bar.ds_in[b], kDSBytes / 2);
        pwait<PAIR_NS_I>(&bar.pds_full, j & 1);
        TRACE(T_ISS_DP, j);
        pwait<PAIR_NS_I>(&bar.qk_full[sj], (j / kKSt) & 1);
        tc_fence_after();
        TRACE(T_ISS_DV, j);
#pragma unroll
        for (int k = 0; k < kBQ / 16; ++k)
          mma_ts2(tdV, tP + k * 8, dOm + koff_mn(k), id_kv, (j > 0 || k > 0) ? 1u : 0u);
#pragma unroll
        for (int k = 0; k < kBQ / 16; ++k)
          mma_ts2(tdK, tDS + k * 8, dQm + koff_mn(k), id_kv, (j > 0 || k > 0) ? 1u : 0u);
        mma_commit2_mc(&bar.qk_empty[sj]);
        mma_commit2_mc(&bar.p_empty);
        // dQ^T of tile j: both CTAs' dS^T halves (ds_in: the peer's st.async bytes here + the peer
        // forwarder's report of the leader's bytes there) and a free dQ^T TMEM buffer.  (Issuing
        // it one tile later, behind the next dV / dK, measured 28.3 vs 26.7 ms.)
        issue_dq(j);
      }
      mma_commit2_mc(&bar.kv_done);
#ifdef DKV_TRACE
    } else if (rank == 1 && warp == kWMma && elect_one()) {
      // trace-only observer: when sdp_full actually completes in the peer (spinning, no suspend)
      for (int i = 0; i < nq; ++i) {
        while (!mbar_test(&bar.sdp_full, i & 1)) {
        }
        TRACE(T_SDONE, i);
      }
#endif
    } else if (rank == 1 && warp == kWMma2 && elect_one()) {
      // the peer's forwarder: once the leader's dS^T half of tile i has landed here (ds_in: st.async
      // bytes), make it visible to the tensor core and report to the leader's MMA issuer
      for (int i = 0; i < nq; ++i) {
        const int b = i & 1;
        const uint32_t lds = mapa_shared(&bar.ds_in[b], 0);
        mbar_arrive_expect_tx(&bar.ds_in[b], kDSBytes / 2);
        pwait<PAIR_NS_I>(&bar.ds_in[b], (i >> 1) & 1);
        TRACE(T_DO_LOAD, i);
        tc_fence_after();
        fence_async_smem();
        tc_fence_before();
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(lds) : "memory");
      }
    }
  } else if (warp < kWDrain) {
    // ================= compute warps (both CTAs): thread = key row r, kCC query columns per warp
    const int r = (warp & 3) * 32 + lane;
    const int c0 = (warp >> 2) * kCC;
    const int qh = c0 >> 5;  // query half of this warp's columns = the CTA whose dQ^T B needs them
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int key = kbase + r;
    // dS^T row of this key in the pair's B operand (pair key order: tile 2 kp first)
    const uint32_t ds_row = rank * kBK + r;
    const bool ds_here = qh == static_cast<int>(rank);
    uint8_t* ds_local0 = base + kOffDS;
    const uint32_t ds_remote0 = mapa_shared(base + kOffDS, rank ^ 1);
    const uint32_t ds_rbar0 = mapa_shared(&bar.ds_in[0], rank ^ 1);
    QIter it;
    it.begin(cu, p.tq, s0, s1, tok_first);
    for (int i = 0; it.valid(); it.next(), ++i) {
      pwait<PAIR_NS_C>(&bar.sdp_full, i & 1);
      tc_fence_after();
      if (threadIdx.x == 0) TRACE(T_C_S, i);
      uint32_t us[kCC], ud[kCC];
      if constexpr (kCC == 32) {
        tmem_ld32(tmem + lane_off + c0, *reinterpret_cast<uint32_t(*)[32]>(us));
        tmem_ld32(tmem + lane_off + 64 + c0, *reinterpret_cast<uint32_t(*)[32]>(ud));
      } else {
        tmem_ld16(tmem + lane_off + c0, *reinterpret_cast<uint32_t(*)[16]>(us));
        tmem_ld16(tmem + lane_off + 64 + c0, *reinterpret_cast<uint32_t(*)[16]>(ud));
      }
      tmem_wait_ld();
      if (threadIdx.x == 0) TRACE(T_C_DP, i);
      tc_fence_before();
      warp_arrive_leader_relaxed(&bar.sdp_empty, rank);
      int cmin;
      if (!causal) {
        cmin = key < kv_len ? 0 : kBQ;
      } else {
        const int dt = key - it.tok;
        cmin = dt <= 0 ? 0 : min(dt * G, kBQ);
      }
      const int cmax = min(qrows, (it.rlen - it.tok) * G);
      const float2 sl2 = make_float2(p.scale_log2, p.scale_log2);
      uint32_t pp[kCC / 2], pd[kCC / 2];
      auto math = [&](auto masked) {
#pragma unroll
        for (int c2 = 0; c2 < kCC / 2; ++c2) {
          const float2 x =
              __fmul2_rn(make_float2(__uint_as_float(us[2 * c2]), __uint_as_float(us[2 * c2 + 1])), sl2);
          float2 e;
          if (c2 >= kCC / 2 - PAIR_POLY) {
            e = ex2_poly2(x);  // on the FMA pipe: the math phase is on the compute warps' critical chain
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
      if (__all_sync(0xffffffffu, cmin <= c0 && cmax >= c0 + kCC))
        math(std::false_type{});
      else
        math(std::true_type{});
      if (threadIdx.x == 0) TRACE(T_C_P, i);
#if PAIR_DS_EARLY
      // dS^T -> the dQ^T operand first (buffer i % 2, free once dQ^T of tile i - 2 is done), so the
      // local writers' proxy fence further down finds these stores complete
      const int b = i & 1;
      pwait<PAIR_NS_C>(&bar.ds_empty[b], ((i >> 1) & 1) ^ 1);
      const int ch0 = (c0 & 31) / 8;
      if (ds_here) {
        uint8_t* ds_local = ds_local0 + b * kDSBytes;
#pragma unroll
        for (int ch = 0; ch < kCC / 8; ++ch)
          *reinterpret_cast<uint4*>(ds_local + sw64_offset(ds_row, ch0 + ch)) =
              make_uint4(pd[4 * ch], pd[4 * ch + 1], pd[4 * ch + 2], pd[4 * ch + 3]);
      } else {
        const uint32_t ds_remote = ds_remote0 + b * kDSBytes;
        const uint32_t ds_rbar = ds_rbar0 + b * 8;  // &ds_in[b] in the peer
#pragma unroll
        for (int ch = 0; ch < kCC / 8; ++ch)
          st_async_v4(ds_remote + sw64_offset(ds_row, ch0 + ch), ds_rbar, pd[4 * ch], pd[4 * ch + 1],
                      pd[4 * ch + 2], pd[4 * ch + 3]);
      }
#endif
      pwait<PAIR_NS_C>(&bar.p_empty, (i & 1) ^ 1);  // dV / dK of tile i - 1 done with P^T / dS^T
      tc_fence_after();
      if (threadIdx.x == 0) TRACE(T_MMA_END, i);
      if constexpr (kCC == 32) {
        tmem_st16(tmem + lane_off + 128 + c0 / 2, *reinterpret_cast<const uint32_t(*)[16]>(pp));
        tmem_st16(tmem + lane_off + 160 + c0 / 2, *reinterpret_cast<const uint32_t(*)[16]>(pd));
      } else {
        tmem_st8(tmem + lane_off + 128 + c0 / 2, *reinterpret_cast<const uint32_t(*)[8]>(pp));
        tmem_st8(tmem + lane_off + 160 + c0 / 2, *reinterpret_cast<const uint32_t(*)[8]>(pd));
      }
      tmem_wait_st();
      tc_fence_before();
      warp_arrive_leader_relaxed(&bar.pds_full, rank);  // dV / dK of tile i may go
#if PAIR_DS_EARLY
      if (ds_here) {
        fence_async_smem();
        warp_arrive_leader_relaxed(&bar.ds_in[i & 1], rank);
      }
#else
      // dS^T (32 query columns of this key) -> buffer i % 2 of the B operand of the CTA owning that
      // query half, once dQ^T of tile i - 2 is done with it; only dQ^T waits for these (ds_in), so
      // the stores and their proxy fence stay off the pds_full -> dV / dK -> p_empty loop
      const int b = i & 1;
      pwait<PAIR_NS_C>(&bar.ds_empty[b], ((i >> 1) & 1) ^ 1);
      const int ch0 = (c0 & 31) / 8;  // first 16 B chunk of these columns in the 64 B query-half row
      if (ds_here) {
        uint8_t* ds_local = ds_local0 + b * kDSBytes;
#pragma unroll
        for (int ch = 0; ch < kCC / 8; ++ch)
          *reinterpret_cast<uint4*>(ds_local + sw64_offset(ds_row, ch0 + ch)) =
              make_uint4(pd[4 * ch], pd[4 * ch + 1], pd[4 * ch + 2], pd[4 * ch + 3]);
        fence_async_smem();
        warp_arrive_leader_relaxed(&bar.ds_in[b], rank);
      } else {
        const uint32_t ds_remote = ds_remote0 + b * kDSBytes;
        const uint32_t ds_rbar = ds_rbar0 + b * 8;  // &ds_in[b] in the peer
#pragma unroll
        for (int ch = 0; ch < kCC / 8; ++ch)
          st_async_v4(ds_remote + sw64_offset(ds_row, ch0 + ch), ds_rbar, pd[4 * ch], pd[4 * ch + 1],
                      pd[4 * ch + 2], pd[4 * ch + 3]);
      }
#endif
      if (threadIdx.x == 4 * 32) TRACE(T_EXTRA, i);  // a warp of the other query half
      if (threadIdx.x == 0) TRACE(T_C_DS, i);
    }
  } else if (warp < kWProd) {
    // ================= dQ drain (both CTAs): lanes [0,64) hold d = lane, queries [0,32); lanes
    // [64,128) the same d, queries [32,64) (M=128 pair layout).  Warps 8-9 drain query half 0,
    // warps 10-11 half 1; each half is staged and reduce-added on its own.
    const int w = warp - kWDrain;
    const int d = (w & 1) * 32 + lane;  // head-dim lane within this CTA's half
    const int h = w >> 1;               // query half
    const uint32_t lane_off = static_cast<uint32_t>(w * 32) << 16;
    const bool issuer = lane == 0 && (w & 1) == 0;
    float* stg = reinterpret_cast<float*>(base + kOffStg) + h * 32 * 64;
    QIter it;
    it.begin(cu, p.tq, s0, s1, tok_first);
    for (int i = 0; it.valid(); it.next(), ++i) {
      const int b = i & 1;
      pwait(&bar.dq_full[b], (i >> 1) & 1);
      tc_fence_after();
      if (threadIdx.x == kWDrain * 32) TRACE(T_D_DQ, i);
      uint32_t u[32];
      tmem_ld32(tmem + lane_off + 192 + b * 32, u);
      tmem_wait_ld();
      tc_fence_before();
      warp_arrive_leader_relaxed(&bar.dq_empty[b], rank);
      if (threadIdx.x == kWDrain * 32) TRACE(T_D_LD, i);
      const int row0 = cu[it.s] + it.tok;
      if (issuer) bulk_wait_read<0>();  // this half's previous reduce has read the staging
      named_bar_sync(1 + h, 64);
#pragma unroll
      for (int c = 0; c < 32; ++c) stg[c * 64 + d] = __uint_as_float(u[c]);
      fence_async_smem();
      named_bar_sync(1 + h, 64);
      if (issuer) {
        const int rr = h * 32;  // first tile row of the half: token rr / G, head rr % G
        tma_reduce_add_3d(mdq, stg, static_cast<int>(rank) * 64, hk * G + rr % G, row0 + rr / G);
        bulk_commit();
      }
      if (threadIdx.x == kWDrain * 32) TRACE(T_D_END, i);
    }
    if (issuer) bulk_wait<0>();
  }

  // ================= dK / dV epilogue (both CTAs, own keys): warps 0-3 dK, 4-7 dV
  if (warp < 8) {
    const bool do_k = warp < 4;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tcol = tmem + lane_off + (do_k ? 384 : 256);
    pwait(&bar.kv_done, 0);
    tc_fence_after();
    const int key = kbase + r;
    const bool ok = key < kv_len;
    const float osc = do_k ? p.scale : 1.f;
#pragma unroll 1
    for (int cc = 0; cc < D; cc += 32) {
      uint32_t u[32];
      tmem_ld32(tcol + cc, u);
      tmem_wait_ld();
      if (!ok) continue;
#pragma unroll
      for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * osc);
      if (ctx_keys) {
        const int64_t plane = static_cast<int64_t>(p.ctx_len) * p.kv_heads * D;
        float* dst = p.ctx_acc + static_cast<int64_t>(part) * 2 * plane + (do_k ? 0 : plane) +
                     ((static_cast<int64_t>(kv_row0) + key) * p.kv_heads + hk) * D + cc;
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
        __nv_bfloat16* dst = (do_k ? p.dk : p.dv) + ((static_cast<int64_t>(kv_row0) + key) * p.kv_heads + hk) * D + cc;
        uint4 v[4];
        uint32_t* wv = reinterpret_cast<uint32_t*>(v);
#pragma unroll
        for (int i = 0; i < 16; ++i) wv[i] = pack_bf16(__uint_as_float(u[2 * i]), __uint_as_float(u[2 * i + 1]));
#pragma unroll
        for (int i = 0; i < 4; ++i) reinterpret_cast<uint4*>(dst)[i] = v[i];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // neither CTA frees the pair's TMEM (or exits) while the other still uses it
  if (warp == kWProd) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem);
  }
}

}  // namespace bwdp

DKV_TRACE_READ_FN(dkv_trace_read_pair)

// DKV_BWD_PAIR=1 routes the d = 128 backward to this kernel (opt-in: measured ~3 % slower than the
// single-CTA kernel at C3 under the power cap, profiles/r2_pair_bwd.md)
static bool bwd_pair_enabled() {
  static const bool v = [] {
    const char* e = getenv("DKV_BWD_PAIR");
    return e && e[0] == '1';
  }();
  return v;
}

bool tc_bwd_pair_supported(int head_dim, int heads, int kv_heads) {
  if (!bwd_pair_enabled() || head_dim != 128 || kv_heads <= 0 || heads % kv_heads) return false;
  const int G = heads / kv_heads;
  return G <= 32 && 32 % G == 0;  // a 32-row query half holds whole tokens
}

int launch_tc_bwd_pair(const SimtArgs& a, const CtxSelf* self, const GroupTable& grp, const BwdScratch& w,
                       cudaStream_t st) {
  using namespace bwdp;
  Params p{};
  const int G = a.heads / a.kv_heads;
  const int tq = kBQ / G;
  if (a.total_q > 0 &&
      (!make_map_3d_bf16(&p.tm_q, a.q, a.total_q, a.heads, D, G, tq) ||
       !make_map_3d_bf16(&p.tm_do, a.dout, a.total_q, a.heads, D, G, tq) ||
       !make_map_3d_bf16(&p.tm_qh, a.q, a.total_q, a.heads, D, G, tq / 2) ||
       !make_map_3d_bf16(&p.tm_doh, a.dout, a.total_q, a.heads, D, G, tq / 2) ||
       !make_map_3d_bf16(&p.tm_k, a.k, a.total_q, a.kv_heads, D, 1, kBK) ||
       !make_map_3d_bf16(&p.tm_v, a.v, a.total_q, a.kv_heads, D, 1, kBK) ||
       !make_map_3d_f32(&p.tm_dq, w.dq_acc, a.total_q, a.heads, D, G, tq / 2, 64) ||
       !make_map_2d_bf16_sw32(&p.tm_xh, w.xsplit, static_cast<int64_t>(w.tpad) * a.heads, 32, 16, 32))) {
    set_error("cuTensorMapEncodeTiled failed (pair backward q/dO/k/v/dq/x)");
    return DKV_ERR_CUDA;
  }
  if (a.ctx_len > 0 && (!make_map_3d_bf16(&p.tm_kc, a.k_ctx, a.ctx_len, a.kv_heads, D, 1, kBK) ||
                        !make_map_3d_bf16(&p.tm_vc, a.v_ctx, a.ctx_len, a.kv_heads, D, 1, kBK))) {
    set_error("cuTensorMapEncodeTiled failed (pair backward k_ctx/v_ctx)");
    return DKV_ERR_CUDA;
  }
  const bool with_self = self && a.ctx_len > 0;
  if (with_self &&
      (!make_map_3d_bf16(&p.tm_qs, self->q, a.ctx_len, a.heads, D, G, tq) ||
       !make_map_3d_bf16(&p.tm_dos, self->dout, a.ctx_len, a.heads, D, G, tq) ||
       !make_map_3d_bf16(&p.tm_qsh, self->q, a.ctx_len, a.heads, D, G, tq / 2) ||
       !make_map_3d_bf16(&p.tm_dosh, self->dout, a.ctx_len, a.heads, D, G, tq / 2) ||
       !make_map_3d_f32(&p.tm_dqs, w.dq_acc_s, a.ctx_len, a.heads, D, G, tq / 2, 64) ||
       !make_map_2d_bf16_sw32(&p.tm_xsh, w.xsplit_s, static_cast<int64_t>(w.tpad_s) * a.heads, 32, 16, 32))) {
    set_error("cuTensorMapEncodeTiled failed (pair backward fused Call 1 maps)");
    return DKV_ERR_CUDA;
  }
  p.tpad = w.tpad;
  p.tpad_s = w.tpad_s;
  p.grp = grp;
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
  const int n_ctx_tiles = (grp.max_ctx + kBK - 1) / kBK;
  p.n_ctx_pairs = (n_ctx_tiles + 1) / 2;
  const int64_t n_ctx_items =
      a.total_q > 0 ? static_cast<int64_t>(p.n_ctx_pairs) * a.kv_heads * grp.n * w.num_chunks : 0;
  const int64_t n_self_items = with_self ? static_cast<int64_t>(p.n_ctx_pairs) * a.kv_heads * grp.n : 0;
  p.n_ctx_items = static_cast<int>(n_ctx_items);
  p.n_self_items = static_cast<int>(n_self_items);
  p.self_part = w.self_part;
  p.atomic_ctx = w.atomic_ctx ? 1 : 0;
  p.scale = a.scale;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  const int max_tiles = a.total_q > 0 ? (a.max_seqlen + kBK - 1) / kBK : 0;
  p.max_own_pairs = std::max(1, (max_tiles + 1) / 2);
  const int64_t items = n_ctx_items + n_self_items +
                        (a.total_q > 0 ? static_cast<int64_t>(p.max_own_pairs) * a.num_seqs * a.kv_heads : 0);
  if (items == 0) return DKV_OK;
  if (2 * items > 0x7fffffff) {
    set_error("pair backward grid too large");
    return DKV_ERR_UNSUPPORTED;
  }
  const void* fn = reinterpret_cast<const void*>(dualkv_bwd_pair_kernel);
  if (!ensure_smem_optin(fn, kSmemBytes, "dualkv_bwd_pair_kernel")) return DKV_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * items));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, dualkv_bwd_pair_kernel, p);
  if (e != cudaSuccess) {
    set_error(std::string("pair backward launch failed: ") + cudaGetErrorString(e));
    return DKV_ERR_CUDA;
  }
  return DKV_OK;
}

}  // namespace dkv
