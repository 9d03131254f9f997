// K3, round-2b structure: 128-query iterations, every GEMM at N = 128.
// (Included by fa_bwd.cu; shares its wait-time instrumentation.)
//
// Same math as fa_bwd_kernel (ref oracle.py:127-152): P = exp(S - LSE),
// dP = dO V^T, dS = P (dP - delta), dV += P^T dO, dK += dS^T Q, dQ += dS K.
//
// Why: the 64-query kernel issues three of its five GEMMs (S^T, dP^T, dQ^T)
// as SS UMMAs with N = 64, which need 192 B/clk of shared-memory operands
// against the 128 B/clk the SM delivers (tools/probes/umma_rate.cu: 66.7 % of
// peak). With 128 queries per iteration every SS GEMM has
// N = 128 (128 B/clk, 100 % in the probe) and the operand bytes per FLOP of
// S^T/dP^T/dQ^T drop by a third.
//
// TMEM (512 columns) holds no double buffers any more; the in-order tensor
// pipe does the hand-off instead:
//   R_S  [0,128)    S^T_i (keys x queries)  -> P^T_i  (bf16, TS A of dV)
//   R_dP [128,256)  dP^T_i                  -> dS^T_i (bf16, TS A of dK)
//                                           -> dQ^T_i = K^T dS^T_i (M = d)
//   [256,256+D) dV,   [256+D,256+2D) dK accumulators.
// Issue order per iteration:  dV_i, S_{i+1}, dK_i, dQ^T_i, dP_{i+1}.
//   S_{i+1} overwrites P^T_i right after dV_i (its only reader) and
//   dQ^T_i overwrites dS^T_i right after dK_i: tcgen05.mma ops of one thread
//   execute in issue order (the 64-query kernel relies on the same property
//   for S^T_{i+2} over P^T_i). S_{i+1} is issued before dK_i/dQ^T_i so the
//   softmax of i+1 (MUFU-bound, ~1000 clk) runs under three GEMMs; the only
//   exposed hand-off is the dQ^T drain's TMEM read before dP_{i+1}.
// Shared memory (D = 128, default staging): K 32 KB, V 32 KB, 2 Q stages
// 64 KB, 1 dO stage 32 KB, dS^T 32 KB, dQ^T drain staging 32 KB = 224 KB (the
// MODE comments below list the alternatives that were measured). The live
// query-tile list is a bitmask (2 x 128 B). D = 64: same structure, dK at
// column 320, dQ^T rows 64-127 unused.
// Warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4-11 two P/dS
// warpgroups (warpgroup hq owns queries [64hq, 64hq+64) of every iteration,
// all 128 keys = TMEM lanes), 12-15 the dQ^T drain (TMEM lane = feature d).

namespace bwd2 {
constexpr int BK = 128;
constexpr int BQ = 128;
constexpr int QST = 2;
constexpr int kThreads = 512;
constexpr int kMaxQTiles = 1024;  // per launch (the C ABI slices at 131072 queries)
constexpr int kWords = kMaxQTiles / 32;
// dQ^T drain staging modes (each box = [D][32 q] fp32, 16 KB at D = 128):
//  kStageHybrid (default): one dO stage; the 32 KB it frees are the drain's
//    own staging for boxes 2,3, and boxes 0,1 go to the dS^T buffer, which is
//    free from dQ^T_i's completion until the softmax stores dS_{i+1} (it waits
//    for those two reduces to finish reading): all four boxes in flight.
//  kStageOwn: one dO stage, all boxes through the own 32 KB (two in flight).
//  kStageDs: two dO stages, all boxes through the dS^T buffer.
constexpr int kStageHybrid = 0, kStageOwn = 1, kStageDs = 2;
template <int D, int MODE>
struct Cfg {
  static constexpr bool kOwn = MODE != kStageDs;
  static constexpr int kDOST = kOwn ? 1 : 2;             // dO stages (Q always has 2)
  static constexpr int kK = 0;
  static constexpr int kV = kK + BK * D * 2;
  static constexpr int kQ = kV + BK * D * 2;             // QST x [D/64 panels][128 q][64] SW128
  static constexpr int kDO = kQ + QST * BQ * D * 2;
  static constexpr int kDS = kDO + kDOST * BQ * D * 2;   // dS^T [2 panels][128 keys][64 q] SW128
  static constexpr int kSTG = kDS + BK * BQ * 2;         // own drain staging: 2 SW128 boxes [D][32 q] fp32
  static constexpr int kStats = kSTG + (kOwn ? 2 * D * 128 : 0);  // QST x (lse2[128], delta[128])
  static constexpr int kMask = kStats + QST * 2 * BQ * 4;  // live bits, full bits
  static constexpr int kBars = kMask + 2 * kWords * 4;
  static constexpr int kBytes = kBars + 256;
  static constexpr int kQStage = BQ * D * 2;              // bytes of one Q (or dO) stage
  static constexpr int kPanels = D / 64;
};
struct Bars {
  uint64_t kv_full;
  uint64_t q_full[QST], q_empty[QST], do_full[QST], do_empty[QST];
  uint64_t s_full, dp_full, p_full, dst_full, dss_full, dq_full, dq_empty, dsbuf_free, dkv_full;
  uint64_t p_part, dst_part;
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "barrier block");

// Live query tiles, highest first (the order every role walks them in).
struct LiveIt {
  const uint32_t* live;
  int wi;
  uint32_t m;
  A2D_DEV void reset(const uint32_t* l, int nwords) {
    live = l;
    wi = nwords - 1;
    m = nwords > 0 ? l[wi] : 0u;
  }
  A2D_DEV int next() {
    while (m == 0u) m = live[--wi];
    const int b = 31 - __clz(m);
    m ^= 1u << b;
    return wi * 32 + b;
  }
};
}  // namespace bwd2

// PX: exp2 pairs computed on the FMA pipe (ex2_poly2) instead of MUFU, out of
// every four pairs of a full tile's P (0, 1 or 2): the P phase is MUFU-bound
// (128 x 128 exps per iteration = 1024 MUFU clk) and gates dV.
// SPL: the P/dS warps release P^T and dS^T in two parts (their first 32-query
// chunk, then the second), so dV / dK start on half of the K steps early.
// CL: CTA pairs (cluster of 2 along the key tiles, an even number of them):
// both CTAs walk the union of their live query tiles; rank 0 loads each Q
// tile and rank 1 each dO tile with TMA multicast into both CTAs, halving the
// SM's L1->L2 load requests (the path the dQ^T reduces saturate). A stage is
// refilled once both CTAs' MMAs released it (multicast commits, count 2).
template <int D, int MODE, int PX, int SPL, bool CL = false>
__global__ void __launch_bounds__(bwd2::kThreads, 1) fa_bwd_q128_kernel(const __grid_constant__ BwdParams p) {
  using namespace bwd2;
  using C = Cfg<D, MODE>;
  constexpr int NDO = C::kDOST;
  static_assert(D == 128 || D == 64, "head dim 64 or 128");
  constexpr int kK = C::kK, kV = C::kV, kQ = C::kQ, kDO = C::kDO, kDS = C::kDS, kStats = C::kStats;
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars& bars = *reinterpret_cast<Bars*>(smem + C::kBars);
  uint32_t* live_mask = reinterpret_cast<uint32_t*>(smem + C::kMask);
  uint32_t* full_mask = live_mask + kWords;

  const int warp = warp_id(), lane = lane_id();
  if ((smem_u32(smem) & 1023u) != 0u) __trap();  // SW128 operands need a 1 KB aligned base
  const int kt = (int)blockIdx.x;
  const int hk = blockIdx.y;
  const int key0 = kt * BK;
  const int nqt64 = (p.Tq + 63) / 64;
  const int nqt = (p.Tq + BQ - 1) / BQ;
  const int nwords = (nqt + 31) / 32;
  const int Tq_pad = p.stats_stride;
  const int2 kb = p.k_bounds[kt];
  const int2 kb_peer = CL ? p.k_bounds[kt ^ 1] : kb;
  const bool causal = p.causal != 0;
  const uint32_t crank = CL ? cluster_rank() : 0u;

  if (threadIdx.x == 0) {
    mbar_init(&bars.kv_full, 1);
    for (int i = 0; i < QST; ++i) {
      mbar_init(&bars.q_full[i], 1); mbar_init(&bars.q_empty[i], CL ? 2 : 1);
      mbar_init(&bars.do_full[i], 1); mbar_init(&bars.do_empty[i], CL ? 2 : 1);
    }
    mbar_init(&bars.s_full, 1);
    mbar_init(&bars.dp_full, 1);
    // P/dS and drain hand-offs arrive once per warp (after __syncwarp): 8 / 4
    // arrivals instead of 256 / 128 serialised shared-memory atomics
    mbar_init(&bars.p_full, 8);
    mbar_init(&bars.p_part, 8);
    mbar_init(&bars.dst_part, 8);
    mbar_init(&bars.dst_full, 8);
    mbar_init(&bars.dss_full, 8);
    mbar_init(&bars.dq_full, 1);
    mbar_init(&bars.dq_empty, 4);
    mbar_init(&bars.dsbuf_free, 1);
    mbar_init(&bars.dkv_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&bars.tmem_base);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tm_q); tma_prefetch(&p.tm_k); tma_prefetch(&p.tm_v); tma_prefetch(&p.tm_do);
    tma_prefetch(&p.tm_dq);
  }
  // ---- live / full bitmasks over 128-query tiles (from the 64-row bounds)
  for (int wi = warp; wi < nwords; wi += 16) {
    const int t = wi * 32 + lane;
    bool lv = false, full = false;
    if (t < nqt) {
      int2 qb = p.q_bounds[2 * t];
      const bool two = 2 * t + 1 < nqt64;
      if (two) {
        const int2 b1 = p.q_bounds[2 * t + 1];
        qb = make_int2(min(qb.x, b1.x), max(qb.y, b1.y));
      }
      lv = qb.x <= qb.y && kb.x <= kb.y && (!causal || kb.x <= qb.y);
      if (CL)  // the pair walks the union (a tile dead here is never full: masked to P = 0)
        lv = lv || (qb.x <= qb.y && kb_peer.x <= kb_peer.y && (!causal || kb_peer.x <= qb.y));
      // full: no mask needed. A tile reaching past the 64-padded stats
      // (single 64-row half) is always masked.
      full = two && (!causal || kb.y <= qb.x);
    }
    const unsigned lm = __ballot_sync(0xffffffffu, lv), fm = __ballot_sync(0xffffffffu, full);
    if (lane == 0) { live_mask[wi] = lm; full_mask[wi] = fm; }
  }
  tc_fence_before();
  __syncthreads();
  if (CL) cluster_sync();  // both CTAs' barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  int n_live = 0;
  for (int wi = 0; wi < nwords; ++wi) n_live += __popc(live_mask[wi]);
  const int n = n_live * p.G;  // iterations: (g, live tile), g-major
  // register budget (setmaxnreg inside each role's branch, so ptxas allocates
  // each role at its own budget): 64 (TMA/MMA/alloc) + 2 x 144 (P/dS) + 160
  // (drain) = 512 per lane x 128
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  (void)prof;
  if (warp < 4) regs_dec<64>();
  if (warp == 0) {
    // -------------------------------------------------------------- producer
    PSTART();
    if (lane == 0 && n > 0) {
      mbar_expect_tx(&bars.kv_full, 2 * BK * D * 2);
      for (int c = 0; c < C::kPanels; ++c) {
        tma_load_3d(smem + kK + c * 16384, &p.tm_k, &bars.kv_full, c * 64, key0, hk);
        tma_load_3d(smem + kV + c * 16384, &p.tm_v, &bars.kv_full, c * 64, key0, hk);
      }
      LiveIt li;
      int it = 0;
      for (int g = 0; g < p.G; ++g) {
        const int h = hk * p.G + g;
        li.reset(live_mask, nwords);
        for (int j = 0; j < n_live; ++j, ++it) {
          const int qt = li.next();
          const int qs = it % QST, ds = it % NDO;
          // Q (+ the stats) once dK_{it-2} freed the stage, dO once dV_{it-NDO} did
          PWAIT(&bars.q_empty[qs], ((it / QST) & 1) ^ 1, 0);
#ifdef A2D_PROFILE
          if ((g_bwd_ablate & 2) && it >= 2) {  // stale tiles: arrive without loading
            mbar_arrive(&bars.q_full[qs]);
            PWAIT(&bars.do_empty[ds], ((it / NDO) & 1) ^ 1, 1);
            mbar_arrive(&bars.do_full[ds]);
            continue;
          }
#endif
          // stats: 128 rows, or 64 when the tile's second half lies past the
          // 64-row padding of the stats (then the tile is on the masked path)
          const int nst = (2 * qt + 1 < nqt64) ? BQ : 64;
          mbar_expect_tx(&bars.q_full[qs], C::kQStage + 2 * nst * 4);
          uint8_t* sq = smem + kQ + qs * C::kQStage;
          if (!CL || crank == 0)
            for (int c = 0; c < C::kPanels; ++c)
              for (int hh = 0; hh < 2; ++hh) {
                if (CL)
                  tma_load_3d_mc(sq + c * 16384 + hh * 8192, &p.tm_q, &bars.q_full[qs], c * 64, qt * BQ + hh * 64, h, 3);
                else
                  tma_load_3d(sq + c * 16384 + hh * 8192, &p.tm_q, &bars.q_full[qs], c * 64, qt * BQ + hh * 64, h);
              }
          float* st = reinterpret_cast<float*>(smem + kStats) + qs * 2 * BQ;
          bulk_g2s(st, p.lse2 + (size_t)h * Tq_pad + qt * BQ, nst * 4, &bars.q_full[qs]);
          bulk_g2s(st + BQ, p.delta + (size_t)h * Tq_pad + qt * BQ, nst * 4, &bars.q_full[qs]);
          PWAIT(&bars.do_empty[ds], ((it / NDO) & 1) ^ 1, 1);
          mbar_expect_tx(&bars.do_full[ds], C::kQStage);
          uint8_t* sd = smem + kDO + ds * C::kQStage;
          if (!CL || crank == 1)
            for (int c = 0; c < C::kPanels; ++c)
              for (int hh = 0; hh < 2; ++hh) {
                if (CL)
                  tma_load_3d_mc(sd + c * 16384 + hh * 8192, &p.tm_do, &bars.do_full[ds], c * 64, qt * BQ + hh * 64, h, 3);
                else
                  tma_load_3d(sd + c * 16384 + hh * 8192, &p.tm_do, &bars.do_full[ds], c * 64, qt * BQ + hh * 64, h);
              }
        }
      }
    }
    PFLUSH(3);
  }
  else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    PSTART();
    if (n > 0) {
      constexpr uint32_t id_s = idesc_bf16(BK, BQ, false, false);  // S^T, dP^T: M=128 keys, N=128 q
      constexpr uint32_t id_kv = idesc_bf16(BK, D, false, true);   // dV, dK: TS, B MN-major
      // dQ^T: M = 128 feature rows always (for D = 64 rows >= 64 read the next
      // smem panel and land in TMEM lanes the drain never reads; M = 64 would
      // cost the same tensor time)
      constexpr uint32_t id_dq = idesc_bf16(128, BQ, true, true);
      const uint32_t sK = smem_u32(smem + kK), sV = smem_u32(smem + kV);
      const uint32_t sQ = smem_u32(smem + kQ), sDO = smem_u32(smem + kDO);
      const uint32_t sDS = smem_u32(smem + kDS);
      const uint32_t tS = tmem, tDP = tmem + 128, tDV = tmem + 256, tDK = tmem + 256 + D;
      const uint64_t dK0 = sdesc_sw128(sK, 16, 1024), dV0 = sdesc_sw128(sV, 16, 1024);
      const uint64_t dQ0 = sdesc_sw128(sQ, 16, 1024), dDO0 = sdesc_sw128(sDO, 16, 1024);
      const uint64_t dKmn = sdesc_sw128(sK, 16384, 1024);   // K as MN-major A (M = d) of dQ^T
      const uint64_t dDSmn = sdesc_sw128(sDS, 16384, 1024); // dS^T as MN-major B (N = q) of dQ^T
      const uint64_t dQmn = sdesc_sw128(sQ, 16384, 1024), dDOmn = sdesc_sw128(sDO, 16384, 1024);
      constexpr uint64_t kStage = (uint64_t)(C::kQStage >> 4);
      // S^T_i (which = 0) or dP^T_i (which = 1): M=128 keys, N=128 q, K=d
      auto issue_sdp = [&](int i, int which) {
        const uint64_t qoff = (uint64_t)(which == 0 ? i % QST : i % NDO) * kStage;
        __syncwarp();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t ka = (uint64_t)(((k / 4) * 16384 + (k % 4) * 32) >> 4);
            if (which == 0)
              umma_ss(tS, dK0 + ka, dQ0 + qoff + ka, id_s, k > 0);
            else
              umma_ss(tDP, dV0 + ka, dDO0 + qoff + ka, id_s, k > 0);
          }
          umma_commit(which == 0 ? &bars.s_full : &bars.dp_full);
        }
        __syncwarp();
      };
      PWAIT(&bars.kv_full, 0, 0);
      PWAIT(&bars.q_full[0], 0, 1);
      tc_fence_after();
      issue_sdp(0, 0);
      PWAIT(&bars.do_full[0], 0, 6);
      tc_fence_after();
      issue_sdp(0, 1);
      for (int i = 0; i < n; ++i) {
        const int qs = i % QST, ds = i % NDO;
        const uint32_t ph = i & 1;
        const uint64_t qoff = (uint64_t)qs * kStage, doff = (uint64_t)ds * kStage;
        // dV += P^T_i dO_i (TS: P^T in R_S; 16 queries per K step at col 32(k/2)+8(k%2))
        // (SPL: K steps {0,1,4,5} = the first chunk of both warpgroups, then {2,3,6,7})
        if (SPL) {
          PWAIT(&bars.p_part, ph, 2);
          tc_fence_after();
          __syncwarp();
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BQ / 16; ++k)
              if ((k / 2) % 2 == 0)
                umma_ts(tDV, tS + (k / 2) * 32 + (k % 2) * 8, dDOmn + doff + (uint64_t)(k * 128), id_kv,
                        (i > 0 || k > 0) ? 1u : 0u);
          }
          __syncwarp();
        }
        PWAIT(&bars.p_full, ph, 2);
        TR(0, i);
        tc_fence_after();
        __syncwarp();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BQ / 16; ++k)
            if (!SPL || (k / 2) % 2 == 1)
              umma_ts(tDV, tS + (k / 2) * 32 + (k % 2) * 8, dDOmn + doff + (uint64_t)(k * 128), id_kv,
                      (i > 0 || k > 0) ? 1u : 0u);
          if (CL) umma_commit_mc(&bars.do_empty[ds], 3); else umma_commit(&bars.do_empty[ds]);  // dO_i's last reader
        }
        __syncwarp();
        // S^T_{i+1} into R_S (after dV_i in the in-order pipe)
        if (i + 1 < n) {
          PWAIT(&bars.q_full[(i + 1) % QST], ((i + 1) / QST) & 1, 1);
          TR(1, i);
          tc_fence_after();
          issue_sdp(i + 1, 0);
        }
        // dK += dS^T_i Q_i (TS: dS^T in R_dP), then release Q_i/dO_i
        if (SPL) {
          PWAIT(&bars.dst_part, ph, 4);
          tc_fence_after();
          __syncwarp();
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BQ / 16; ++k)
              if ((k / 2) % 2 == 0)
                umma_ts(tDK, tDP + (k / 2) * 32 + (k % 2) * 8, dQmn + qoff + (uint64_t)(k * 128), id_kv,
                        (i > 0 || k > 0) ? 1u : 0u);
          }
          __syncwarp();
        }
        PWAIT(&bars.dst_full, ph, 4);
        TR(2, i);
        tc_fence_after();
        __syncwarp();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BQ / 16; ++k)
            if (!SPL || (k / 2) % 2 == 1)
              umma_ts(tDK, tDP + (k / 2) * 32 + (k % 2) * 8, dQmn + qoff + (uint64_t)(k * 128), id_kv,
                      (i > 0 || k > 0) ? 1u : 0u);
          if (CL) umma_commit_mc(&bars.q_empty[qs], 3); else umma_commit(&bars.q_empty[qs]);
        }
        __syncwarp();
        // dQ^T_i = K^T dS^T_i into R_dP (after dK_i); dS^T from shared memory
        PWAIT(&bars.dss_full, ph, 5);
        TR(3, i);
        tc_fence_after();
        __syncwarp();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_ss(tDP, dKmn + (uint64_t)(k * 128), dDSmn + (uint64_t)(k * 128), id_dq, k > 0);
          umma_commit(&bars.dq_full);
        }
        __syncwarp();
        // dP^T_{i+1} into R_dP once the drain has read dQ^T_i
        if (i + 1 < n) {
          PWAIT(&bars.dq_empty, ph, 3);
          TR(4, i);
          PWAIT(&bars.do_full[(i + 1) % NDO], ((i + 1) / NDO) & 1, 6);
          TR(5, i);
          tc_fence_after();
          issue_sdp(i + 1, 1);
        }
      }
      __syncwarp();
      if (elect_one()) umma_commit(&bars.dkv_full);
      __syncwarp();
    }
    PFLUSH(0);
  } else if (warp >= 12) {
    // ------------------------------------------------ dQ^T drain warpgroup
    // Reads all of R_dP (TMEM lane = feature d, column = query) and releases
    // it for dP_{i+1}; then streams the 128 queries as four SW128 boxes
    // [D][32 q] into TMA bulk reduce-adds on the transposed fp32 dq_acc
    // through the staging of MODE (above). The SM's L1->L2 request path is
    // the limit (~2/3 of it is these reduces), so what matters is how many
    // boxes can be in flight while the drain already waits for dQ^T_{i+1}.
    // (red.global from registers measured 2x slower: 1-sector L2 requests.)
    regs_inc<160>();
    const int wq = warp % 4;
    const int d = wq * 32 + lane;
    const bool d_warp_ok = wq * 32 < D;
    PSTART();
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const bool leader = warp == 12 && lane == 0;
    const float scale = p.scale;
    LiveIt li;
    int it = 0;
    for (int g = 0; g < p.G; ++g) {
      const int h = hk * p.G + g;
      li.reset(live_mask, nwords);
      for (int j = 0; j < n_live; ++j, ++it) {
        const int qt = li.next();
        PWAIT(&bars.dq_full, it & 1, 0);
        if (warp == 12) TR(13, it);
        tc_fence_after();
        uint32_t v[4][32];
        if (d_warp_ok) {  // (D = 64: warps 14-15 hold no feature rows)
#pragma unroll
          for (int b = 0; b < 4; ++b) tmem_ld32(tmem + lane_base + 128 + b * 32, v[b]);
          tmem_ld_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.dq_empty);
        if (warp == 12) TR(14, it);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          uint8_t* box;
          bool wait;  // the reduce that last read this slot must be done
          if constexpr (MODE == kStageHybrid) {
            box = smem + (b < 2 ? kDS + b * (D * 128) : C::kSTG + (b - 2) * (D * 128));
            wait = b == 2;  // (boxes 0,1: the dS^T buffer is free once dQ^T_i is done)
          } else {
            box = smem + (MODE == kStageOwn ? C::kSTG : kDS) + (b & 1) * (D * 128);
            wait = MODE == kStageOwn || b >= 2;
          }
          if (wait) {
#ifdef A2D_PROFILE
            const long long tr0 = clock64();
#endif
            if (leader) {
              if (MODE == kStageHybrid)
                bulk_wait_read2();  // only boxes 0,1 of this iteration may still be reading
              else
                bulk_wait_read1();
            }
            named_bar_sync(1, 128);
#ifdef A2D_PROFILE
            prof[1] += clock64() - tr0;
#endif
          }
          uint8_t* row = box + d * 128;
          if (d_warp_ok) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *reinterpret_cast<float4*>(row + ((c ^ (d & 7)) << 4)) =
                  make_float4(__uint_as_float(v[b][4 * c]) * scale, __uint_as_float(v[b][4 * c + 1]) * scale,
                              __uint_as_float(v[b][4 * c + 2]) * scale, __uint_as_float(v[b][4 * c + 3]) * scale);
          }
          fence_async_smem();
          named_bar_sync(1, 128);
          if (leader) {
#ifdef A2D_PROFILE
            if (!(g_bwd_ablate & 1))
#endif
              tma_reduce_add_3d(&p.tm_dq, box, qt * BQ + 32 * b, 0, h);
            bulk_commit();
          }
        }
        if (MODE != kStageOwn && leader) {
          // the dS^T buffer's reduces are done reading: the softmax may store dS_{i+1}
          if (MODE == kStageHybrid)
            bulk_wait_read2();
          else
            bulk_wait_read0();
          mbar_arrive(&bars.dsbuf_free);
        }
        if (warp == 12) TR(15, it);
      }
    }
    if (leader) bulk_wait0();
    if (warp == 12) PFLUSH(2);
  } else if (warp >= 4) {
    // ------------------------------------------------ P/dS warpgroups
    regs_inc<144>();
    const int hq = (warp - 4) / 4;
    const int wq = warp % 4;
    const int r = wq * 32 + lane;
    const int key = key0 + r;
    const bool key_ok = key < p.Tk;
    const int kpos = key_ok ? p.k_pos[key] : INT_MAX;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const float sl2 = p.scale_log2;
    const int* qpos_base = p.q_pos;
    const int Tq = p.Tq;
    PSTART();
    LiveIt li;
    int it = 0;
    for (int g = 0; g < p.G; ++g) {
      li.reset(live_mask, nwords);
      for (int j = 0; j < n_live; ++j, ++it) {
        const int qt = li.next();
        const bool full = (full_mask[qt >> 5] >> (qt & 31)) & 1u;
        const int qs = it % QST;
        const uint32_t ph = it & 1;
        PWAIT(&bars.q_full[qs], (it / QST) & 1, 0);  // stats landed with the Q stage
        const float* stl = reinterpret_cast<const float*>(smem + kStats) + qs * 2 * BQ;
        const float* std_ = stl + BQ;
        PWAIT(&bars.s_full, ph, 1);
        if (warp == 4) TR(6, it);
        tc_fence_after();
        // ---- P (fp32, kept for dS) -> P^T bf16 over the consumed S^T columns
        float pr[2][32];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int q0 = hq * 64 + c * 32;  // query column within the tile
          uint32_t sr[32];
          tmem_ld32(tmem + lane_base + q0, sr);
          tmem_ld_wait();
          if (full) {
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              const float4 l4 = *reinterpret_cast<const float4*>(stl + q0 + e);
              const float x0 = fmaf(__uint_as_float(sr[e + 0]), sl2, -l4.x);
              const float x1 = fmaf(__uint_as_float(sr[e + 1]), sl2, -l4.y);
              const float x2 = fmaf(__uint_as_float(sr[e + 2]), sl2, -l4.z);
              const float x3 = fmaf(__uint_as_float(sr[e + 3]), sl2, -l4.w);
              // pair index within 8 consecutive pairs: (e/2) % 8 and (e/2+1) % 8
              const int pa = (e / 2) % 8;
              if (PX >= 1 && pa == 6) {  // pairs 6 (and 7 for PX 2) of every 8 -> 1/8 or 1/4 of exps
                const float2 y = ex2_poly2(make_float2(x0, x1));
                pr[c][e + 0] = y.x;
                pr[c][e + 1] = y.y;
              } else {
                pr[c][e + 0] = ex2(x0);
                pr[c][e + 1] = ex2(x1);
              }
              if (PX >= 2 && pa == 6) {
                const float2 y = ex2_poly2(make_float2(x2, x3));
                pr[c][e + 2] = y.x;
                pr[c][e + 3] = y.y;
              } else {
                pr[c][e + 2] = ex2(x2);
                pr[c][e + 3] = ex2(x3);
              }
            }
          } else {
            const int qb0 = qt * BQ + q0;
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              const int q = qb0 + e;
              const int qp = __ldg(qpos_base + min(q, Tq - 1));
              const bool keep = key_ok && q < Tq && (!causal || kpos <= qp);
              const float pv = ex2(fmaf(__uint_as_float(sr[e]), sl2, -stl[q0 + e]));
              pr[c][e] = keep ? pv : 0.f;
            }
          }
          uint32_t pw[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) pw[e] = pack_bf16(pr[c][2 * e], pr[c][2 * e + 1]);
          tmem_st16(tmem + lane_base + q0, pw);
          if (SPL && c == 0) {
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars.p_part);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        if (warp == 4) TR(7, it);
        if (warp == 8) TR(12, it);
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.p_full);
        // ---- dS = P (dP - delta) -> dS^T bf16 over the consumed dP^T columns
        PWAIT(&bars.dp_full, ph, 2);
        if (warp == 4) TR(8, it);
        tc_fence_after();
        uint32_t dw[2][16];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int q0 = hq * 64 + c * 32;
          uint32_t dr[32];
          tmem_ld32(tmem + lane_base + 128 + q0, dr);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 d4 = *reinterpret_cast<const float4*>(std_ + q0 + e);
            float ds0 = pr[c][e + 0] * (__uint_as_float(dr[e + 0]) - d4.x);
            float ds1 = pr[c][e + 1] * (__uint_as_float(dr[e + 1]) - d4.y);
            float ds2 = pr[c][e + 2] * (__uint_as_float(dr[e + 2]) - d4.z);
            float ds3 = pr[c][e + 3] * (__uint_as_float(dr[e + 3]) - d4.w);
            if (!full) {  // masked / padded entries: P = 0 and delta may be stale
              ds0 = pr[c][e + 0] != 0.f ? ds0 : 0.f;
              ds1 = pr[c][e + 1] != 0.f ? ds1 : 0.f;
              ds2 = pr[c][e + 2] != 0.f ? ds2 : 0.f;
              ds3 = pr[c][e + 3] != 0.f ? ds3 : 0.f;
            }
            dw[c][e / 2] = pack_bf16(ds0, ds1);
            dw[c][e / 2 + 1] = pack_bf16(ds2, ds3);
          }
          tmem_st16(tmem + lane_base + 128 + q0, dw[c]);
          if (SPL && c == 0) {
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars.dst_part);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        if (warp == 4) TR(9, it);
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.dst_full);
        // ---- dS^T to shared memory (MN-major B of dQ^T) once the drain of
        // dQ^T_{i-1} is off the buffer
        if (MODE != kStageOwn && it >= 1) PWAIT(&bars.dsbuf_free, (it - 1) & 1, 3);
        if (warp == 4) TR(10, it);
        uint8_t* panel = smem + kDS + hq * 16384;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int m = 0; m < 4; ++m)
            *reinterpret_cast<uint4*>(panel + sw128_offset(r, 4 * c + m)) =
                make_uint4(dw[c][4 * m], dw[c][4 * m + 1], dw[c][4 * m + 2], dw[c][4 * m + 3]);
        fence_async_smem();
        if (warp == 4) TR(11, it);
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.dss_full);
      }
    }
    if (warp == 4) PFLUSH(1);
    // ------------------------------------------------ dV (hq=0) / dK (hq=1) epilogue
    if (n > 0) {
      mbar_wait(&bars.dkv_full, 0);
      tc_fence_after();
    }
    float* dst = (hq == 0 ? p.dv : p.dk) + ((size_t)hk * p.Tk + key) * D;
    const float oscale = hq == 0 ? 1.f : p.scale;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t rr[32];
      if (n > 0) {
        tmem_ld32(tmem + lane_base + 256 + hq * D + c * 32, rr);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) rr[j] = 0u;
      }
      if (key_ok) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 val = make_float4(__uint_as_float(rr[j]) * oscale, __uint_as_float(rr[j + 1]) * oscale,
                                   __uint_as_float(rr[j + 2]) * oscale, __uint_as_float(rr[j + 3]) * oscale);
          float4* d4 = reinterpret_cast<float4*>(dst + c * 32 + j);
          if (p.accumulate_kv) {
            const float4 o = *d4;
            val.x += o.x; val.y += o.y; val.z += o.z; val.w += o.w;
          }
          *d4 = val;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (CL) cluster_sync();  // no CTA leaves while its peer may still multicast into it
  if (warp == 2) tmem_dealloc<512>(tmem);
}

template <int D, int MODE, int PX = 0, int SPL = 0, bool CL = false>
static cudaError_t launch_bwd_q128(const BwdParams& p, cudaStream_t s) {
  constexpr int bytes = bwd2::Cfg<D, MODE>::kBytes;
  static_assert(bytes <= 232448, "backward shared memory exceeds 227 KB");
  auto kern = fa_bwd_q128_kernel<D, MODE, PX, SPL, CL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  const int nkt = (p.Tk + bwd2::BK - 1) / bwd2::BK;
  if (CL && (nkt % 2) != 0) return launch_bwd_q128<D, MODE, PX, SPL, false>(p, s);  // pairs need an even count
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nkt, p.Hkv);
  cfg.blockDim = dim3(bwd2::kThreads);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CL ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, kern, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}
