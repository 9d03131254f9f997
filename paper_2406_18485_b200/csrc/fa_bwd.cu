// Chunk flash-attention backward for sm_100a (K3).
//
// Gradients of one ring step's block (Q chunk vs one KV chunk) given the
// FINAL softmax statistics of the query rows (global LSE, and
// delta = rowsum(dO * O) = the reference's row = sum(dP * P), oracle.py:145):
//   P   = exp(S - LSE)               dP = dO V^T
//   dS  = P * (dP - delta) / sqrt(d)   (the 1/sqrt(d) is applied after the GEMMs)
//   dV += P^T dO    dK += dS^T Q    dQ += dS K
// GQA: the CTA walks every query head of its KV head's group, so dK/dV sum
// over the G sharing heads inside TMEM (ref oracle.py:149-151).
//
// One CTA = one 128-key tile of one KV head; it streams the live 64-row query
// tiles (a compacted list built once in shared memory: causal-dead tiles cost
// nothing). Everything is key-major so the key tile owns the 128 TMEM lanes:
//   S^T  = K Q^T      (M=128 keys, N=64 q, K=d)   TMEM region b, cols [0,64)
//   dP^T = V dO^T                                  TMEM region b, cols [64,128)
//   P^T and dS^T (bf16) are written back inside each warpgroup's own S^T
//   columns (warpgroup hq: P^T -> [32hq, 32hq+16), dS^T -> [32hq+16, 32hq+32))
//   and feed dV / dK as TMEM (TS) operands; dQ^T = K^T dS^T (M=d, N=64 q,
//   K=128 keys) lands in the consumed dP^T columns [64,128)
//   dV  += P^T dO     (M=128 keys, N=d, K=64 q)    TMEM [256,384)
//   dK  += dS^T Q                                  TMEM [384,512)
// dS^T also goes through shared memory (SW128) as the MN-major B operand of
// dQ^T; feeding dK from TMEM saves 16 KB of smem operand reads per iteration
// (the backward is shared-memory-bandwidth bound).
// dQ^T is drained TMEM -> smem -> TMA bulk tensor reduce-add into dq_acc (the
// add happens in L2). dq_acc is kept TRANSPOSED, [H][128][Tq_pad] (query
// contiguous), so a drain thread (= one feature d) writes 16-byte runs of 4
// queries straight from its TMEM row: two SW128 boxes of 32 q x 128 d, 16
// vector stores per thread instead of 64 scalar ones (+2.7% sustained).
// Warp roles: 0 TMA, 1 MMA, 2 TMEM alloc, 4-11 two P/dS warpgroups that split
// every 64-query iteration in halves, 12-15 the dQ^T drain warpgroup.
#include "sm100.cuh"
#include "kernels.h"

#include <cstdlib>

namespace a2d {

// Optional wait-time instrumentation (build with -DA2D_PROFILE, see
// build.py --profile): cycles each role spends blocked on each barrier,
// summed over CTAs into g_bwd_prof[role*8 + slot] (role 0 MMA warp, 1 P/dS
// warpgroup 0 (warp 4 lane 0), 2 dQ drain (warp 12 lane 0), 3 TMA producer).
#ifdef A2D_PROFILE
__device__ unsigned long long g_bwd_prof[32];
// ablations for bottleneck measurement only (profile build; results are wrong):
// bit 0: the 128-query kernel skips its dQ^T reduce-adds; bit 1: it loads
// Q/dO only for its first two iterations (stale tiles afterwards)
__device__ int g_bwd_ablate;
// per-event clock64 timeline of one CTA (key tile 0, head 0), iterations
// [kTraceIt0, kTraceIt0 + 32), 16 event slots each (tools/bwd_prof.py --trace)
constexpr int kTraceIt0 = 200;
__device__ long long g_bwd_trace[32 * 16];
#define TR(slot, iter)                                                                                  \
  do {                                                                                                 \
    if (blockIdx.x == 0 && blockIdx.y == 0 && lane == 0 && (iter) >= kTraceIt0 && (iter) < kTraceIt0 + 32) \
      g_bwd_trace[((iter) - kTraceIt0) * 16 + (slot)] = clock64();                                     \
  } while (0)
#ifdef A2D_SPIN
#define A2D_WAIT mbar_spin
#else
#define A2D_WAIT mbar_wait
#endif
#define PWAIT(bar, ph, slot)             \
  do {                                   \
    const long long t0_ = clock64();     \
    A2D_WAIT(bar, ph);                   \
    prof[slot] += clock64() - t0_;       \
  } while (0)
#define PSTART() const long long pt0_ = clock64()
#define PFLUSH(role)                                                                            \
  do {                                                                                          \
    prof[7] = clock64() - pt0_;                                                                 \
    if (lane == 0)                                                                              \
      for (int s_ = 0; s_ < 8; ++s_) atomicAdd(&g_bwd_prof[(role) * 8 + s_], (unsigned long long)prof[s_]); \
  } while (0)
#else
#define PWAIT(bar, ph, slot) mbar_wait(bar, ph)
#define TR(slot, iter)
#define PSTART()
#define PFLUSH(role)
#endif

namespace bwd {
constexpr int BK = 128;  // keys per CTA
constexpr int BQ = 64;   // queries per iteration
constexpr int kQstDefault = 3;  // Q/dO stages (TMA latency off the critical path)
constexpr int kThreads = 512;
constexpr int kMaxQTiles = 2048;                 // live-list capacity per launch (the C ABI slices longer query chunks)
constexpr uint16_t kFullBit = 0x8000;
// smem layout (bytes, from 1 KB aligned base) for head dim D (64 or 128)
// DQ8: per-warp dQ drain in 8-query chunks through 2 x 1 KB staging buffers
// per warp (8 KB in all instead of 32 KB), which is what makes room for a 4th
// Q/dO stage.
template <int D, int QST = kQstDefault, bool DQ8 = false>
struct Cfg {
  static constexpr int kK = 0;
  static constexpr int kV = kK + BK * D * 2;              // 32 KB each at D = 128
  static constexpr int kQ = kV + BK * D * 2;              // QST x 16 KB
  static constexpr int kDO = kQ + QST * BQ * D * 2;       // QST x 16 KB
  static constexpr int kDS = kDO + QST * BQ * D * 2;      // 16 KB  (dS^T, [key][q] SW128)
  static constexpr int kDQ = kDS + BK * BQ * 2;           // fp32 dQ staging: 2 SW128 boxes [D][32 q]
  static constexpr int kStats = kDQ + (DQ8 ? 4 * 2 * 1024 : BQ * D * 4);  // QST x (lse2[64], delta[64])
  static constexpr int kList = kStats + QST * 2 * BQ * 4; // live query tiles (uint16)
  static constexpr int kEnd = kList + kMaxQTiles * 2;
  static constexpr int kBytes = kEnd + 1024;
  static constexpr int kPanels = D / 64;                  // 64-wide SW128 panels per row
  static constexpr uint32_t kTdK = 256 + D;               // TMEM column of the dK accumulator (dV at 256)
};
}  // namespace bwd

template <int QST>
struct BwdBars {
  uint64_t kv_full;
  uint64_t qdo_full[QST], qdo_empty[QST];
  uint64_t s_full[2], ds_full[2], dq_full[2], dq_empty[2], ds_free;
  uint64_t dkv_full;
  uint32_t tmem_base;
  int n_live;
  int warp_cnt[16];
};

A2D_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// D: head dim; QST: Q/dO pipeline stages; PF: L2 prefetch distance (in
// iterations) of upcoming Q/dO tiles issued by the producer (0 = none).
template <int D, int QST, int PF, bool DQ8>
__global__ void __launch_bounds__(bwd::kThreads, 1) fa_bwd_kernel(const __grid_constant__ BwdParams p) {
  using namespace bwd;
  using C = Cfg<D, QST, DQ8>;
  constexpr int kK = C::kK, kV = C::kV, kQ = C::kQ, kDO = C::kDO, kDS = C::kDS, kDQ = C::kDQ;
  constexpr int kStats = C::kStats, kList = C::kList;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in .shared
  __shared__ BwdBars<QST> bars;

  const int warp = warp_id(), lane = lane_id();
  const int nkt = (p.Tk + BK - 1) / BK;
  const int kt = (int)blockIdx.x;  // heavy-first: early keys are seen by the most queries (causal)
  const int hk = blockIdx.y;
  const int key0 = kt * BK;
  const int nqt = (p.Tq + BQ - 1) / BQ;
  const int Tq_pad = p.stats_stride;  // row stride of lse2 / delta (>= round_up(Tq, 64))
  const int2 kb = p.k_bounds[kt];
  const bool causal = p.causal != 0;
  uint16_t* live_list = reinterpret_cast<uint16_t*>(smem + kList);

  if (threadIdx.x == 0) {
    mbar_init(&bars.kv_full, 1);
    for (int i = 0; i < QST; ++i) { mbar_init(&bars.qdo_full[i], 1); mbar_init(&bars.qdo_empty[i], 1); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.s_full[b], 1);
      mbar_init(&bars.ds_full[b], 256);
      mbar_init(&bars.dq_full[b], 1);
      mbar_init(&bars.dq_empty[b], 128);
    }
    mbar_init(&bars.ds_free, 1);
    mbar_init(&bars.dkv_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&bars.tmem_base);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tm_q); tma_prefetch(&p.tm_k); tma_prefetch(&p.tm_v); tma_prefetch(&p.tm_do);
    tma_prefetch(DQ8 ? &p.tm_dq8 : &p.tm_dq);
  }
  // ---- compacted list of live query tiles: every warp scans a contiguous
  // range, counts, then writes its survivors at its prefix offset.
  {
    const int per_warp = (nqt + 15) / 16;
    const int lo = warp * per_warp, hi = min(nqt, lo + per_warp);
    int cnt = 0;
    for (int base = lo; base < hi; base += 32) {
      const int qt = base + lane;
      bool lv = false;
      if (qt < hi) {
        const int2 qb = p.q_bounds[qt];
        lv = qb.x <= qb.y && kb.x <= kb.y && (!causal || kb.x <= qb.y);
      }
      cnt += __popc(__ballot_sync(0xffffffffu, lv));
    }
    if (lane == 0) bars.warp_cnt[warp] = cnt;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; ++w) off += bars.warp_cnt[w];
    if (warp == 15 && lane == 0) bars.n_live = off + cnt;
    for (int base = lo; base < hi; base += 32) {
      const int qt = base + lane;
      bool lv = false, full = false;
      if (qt < hi) {
        const int2 qb = p.q_bounds[qt];
        lv = qb.x <= qb.y && kb.x <= kb.y && (!causal || kb.x <= qb.y);
        full = !causal || kb.y <= qb.x;
      }
      const unsigned m = __ballot_sync(0xffffffffu, lv);
      if (lv) live_list[off + __popc(m & ((1u << lane) - 1u))] = (uint16_t)(qt | (full ? kFullBit : 0));
      off += __popc(m);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const int n_live = bars.n_live;
  const int n = n_live * p.G;  // iterations: (g, live tile) g-major
  // register budget: TMA/MMA warpgroup and drain warpgroup give registers to
  // the two P/dS warpgroups (80*128 + 96*128 + 2*152*128 <= 64K); the
  // drain / P/dS adjustments sit inside their role branches so ptxas
  // allocates each role at its own budget
  if (warp < 4) regs_dec<80>();

  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  (void)prof;
  if (warp == 0) {
    // -------------------------------------------------------------- producer
    PSTART();
    if (lane == 0 && n > 0) {
      mbar_expect_tx(&bars.kv_full, 2 * BK * D * 2);
      for (int c = 0; c < C::kPanels; ++c) {
        tma_load_3d(smem + kK + c * 16384, &p.tm_k, &bars.kv_full, c * 64, key0, hk);
        tma_load_3d(smem + kV + c * 16384, &p.tm_v, &bars.kv_full, c * 64, key0, hk);
      }
      int it = 0;
      if (PF > 0) {  // warm L2 with the first PF iterations' tiles
        for (int j = 0; j < PF && j < n; ++j) {
          const int qt = live_list[n_live - 1 - (j % n_live)] & (kFullBit - 1);
          const int h = hk * p.G + j / n_live;
          for (int c = 0; c < C::kPanels; ++c) {
            tma_prefetch_l2_3d(&p.tm_q, c * 64, qt * BQ, h);
            tma_prefetch_l2_3d(&p.tm_do, c * 64, qt * BQ, h);
          }
        }
      }
      for (int g = 0; g < p.G; ++g) {
        const int h = hk * p.G + g;
        for (int li = 0; li < n_live; ++li, ++it) {
          const int qt = live_list[n_live - 1 - li] & (kFullBit - 1);
          const int qs = it % QST;
          if (PF > 0 && it + PF < n) {  // L2 prefetch PF iterations ahead (no smem needed)
            const int j = it + PF;
            const int qtp = live_list[n_live - 1 - (j % n_live)] & (kFullBit - 1);
            const int hp = hk * p.G + j / n_live;
            for (int c = 0; c < C::kPanels; ++c) {
              tma_prefetch_l2_3d(&p.tm_q, c * 64, qtp * BQ, hp);
              tma_prefetch_l2_3d(&p.tm_do, c * 64, qtp * BQ, hp);
            }
          }
          PWAIT(&bars.qdo_empty[qs], ((it / QST) & 1) ^ 1, 0);
          mbar_expect_tx(&bars.qdo_full[qs], 2 * BQ * D * 2 + 2 * BQ * 4);
          for (int c = 0; c < C::kPanels; ++c) {
            tma_load_3d(smem + kQ + qs * BQ * D * 2 + c * 8192, &p.tm_q, &bars.qdo_full[qs], c * 64, qt * BQ, h);
            tma_load_3d(smem + kDO + qs * BQ * D * 2 + c * 8192, &p.tm_do, &bars.qdo_full[qs], c * 64, qt * BQ,
                        h);
          }
          float* st = reinterpret_cast<float*>(smem + kStats) + qs * 2 * BQ;
          bulk_g2s(st, p.lse2 + (size_t)h * Tq_pad + qt * BQ, BQ * 4, &bars.qdo_full[qs]);
          bulk_g2s(st + BQ, p.delta + (size_t)h * Tq_pad + qt * BQ, BQ * 4, &bars.qdo_full[qs]);
        }
      }
    }
    PFLUSH(3);
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    // The whole (converged) warp runs this loop so descriptors are computed in
    // uniform registers; an elected lane issues each group of tcgen05 ops.
    PSTART();
    if (n > 0) {
      constexpr uint32_t id_s = idesc_bf16(BK, BQ, false, false);   // S^T, dP^T
      constexpr uint32_t id_kv = idesc_bf16(BK, D, false, true);    // dV, dK
      // dQ^T: M = 128 feature rows always (rows >= D read the next smem panel
      // and land in TMEM lanes the drain never reads: M = 64 would cost the
      // same tensor time, max(M,128)*N/256 clocks per K16 step)
      constexpr uint32_t id_dq = idesc_bf16(128, BQ, true, true);
      const uint32_t sK = smem_u32(smem + kK), sV = smem_u32(smem + kV);
      const uint32_t sQ = smem_u32(smem + kQ), sDO = smem_u32(smem + kDO);
      const uint32_t sDS = smem_u32(smem + kDS);
      const uint32_t tDV = tmem + 256, tDK = tmem + C::kTdK;
      // loop-invariant descriptor bases (the start-address field advances by bytes>>4)
      const uint64_t dK0 = sdesc_sw128(sK, 16, 1024), dV0 = sdesc_sw128(sV, 16, 1024);
      const uint64_t dQ0 = sdesc_sw128(sQ, 16, 1024), dDO0 = sdesc_sw128(sDO, 16, 1024);
      const uint64_t dKmn = sdesc_sw128(sK, 16384, 1024);  // K as MN-major A of dQ^T
      const uint64_t dDSmn = sdesc_sw128(sDS, 8192, 1024);  // dS^T as MN-major B of dQ^T
      const uint64_t dQmn = sdesc_sw128(sQ, 8192, 1024), dDOmn = sdesc_sw128(sDO, 8192, 1024);
      // S^T_i and dP^T_i (part 0: both, interleaved per K step) into region
      // i&1, then commit s_full.
      auto issue_s = [&](int i, int part) {
        const int b = i & 1, qs = i % QST;
        const uint32_t tS = tmem + b * 128, tDP = tmem + b * 128 + 64;
        const uint64_t qoff = (uint64_t)((qs * BQ * D * 2) >> 4);
        __syncwarp();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t ka = (uint64_t)(((k / 4) * 16384 + (k % 4) * 32) >> 4);
            const uint64_t kq = qoff + (uint64_t)(((k / 4) * 8192 + (k % 4) * 32) >> 4);
            if (part != 2) umma_ss(tS, dK0 + ka, dQ0 + kq, id_s, k > 0);
            if (part != 1) umma_ss(tDP, dV0 + ka, dDO0 + kq, id_s, k > 0);
          }
          if (part != 1) umma_commit(&bars.s_full[b]);
        }
        __syncwarp();
      };
      PWAIT(&bars.kv_full, 0, 0);
      for (int i = 0; i < 2 && i < n; ++i) {
        PWAIT(&bars.qdo_full[i % QST], (i / QST) & 1, 1);
        tc_fence_after();
        issue_s(i, 0);
      }
      for (int i = 0; i < n; ++i) {
        const int b = i & 1, qs = i % QST;
        const uint64_t qoff = (uint64_t)((qs * BQ * D * 2) >> 4);
        PWAIT(&bars.ds_full[b], (i >> 1) & 1, 2);
        tc_fence_after();
        __syncwarp();
        if (elect_one()) {
          // dQ^T_i = K^T dS^T_i -> region b cols [64,128) (dP^T_i already consumed)
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_ss(tmem + b * 128 + 64, dKmn + (uint64_t)(k * 128), dDSmn + (uint64_t)(k * 128), id_dq, k > 0);
          umma_commit(&bars.dq_full[b]);
          umma_commit(&bars.ds_free);
          // dV += P^T dO and dK += dS^T Q, both TS: the A operand comes from TMEM
          // region b (queries 16k.. of P^T at col (k/2)*32 + (k%2)*8, dS^T at +16)
#pragma unroll
          for (int k = 0; k < BQ / 16; ++k)
            umma_ts(tDV, tmem + b * 128 + (k / 2) * 32 + (k % 2) * 8, dDOmn + qoff + (uint64_t)(k * 128), id_kv,
                    (i > 0 || k > 0) ? 1u : 0u);
#pragma unroll
          for (int k = 0; k < BQ / 16; ++k)
            umma_ts(tDK, tmem + b * 128 + (k / 2) * 32 + 16 + (k % 2) * 8, dQmn + qoff + (uint64_t)(k * 128), id_kv,
                    (i > 0 || k > 0) ? 1u : 0u);
          umma_commit(&bars.qdo_empty[qs]);
        }
        __syncwarp();
        if (i + 2 < n) {
          // (r02: issuing S^T_{i+2} before the dq_empty wait measured 4% slower —
          // it exposes the Q/dO TMA latency the drain wait used to cover)
          PWAIT(&bars.dq_empty[b], (i >> 1) & 1, 3);
          PWAIT(&bars.qdo_full[(i + 2) % QST], ((i + 2) / QST) & 1, 1);
          tc_fence_after();
          issue_s(i + 2, 0);
        }
      }
      __syncwarp();
      if (elect_one()) umma_commit(&bars.dkv_full);
      __syncwarp();
    }
    PFLUSH(0);
  } else if (warp >= 12) {
    // ------------------------------------------------ dQ^T drain warpgroup
    // TMEM lane = feature d; 64 query columns -> two SW128 smem boxes -> TMA
    // bulk reduce-add into the transposed dq_acc. Runs concurrently with the
    // P/dS warpgroups, off their critical path.
    regs_dec<96>();
    const int wq = warp % 4;
    const int d = wq * 32 + lane;
    const bool d_ok = d < D;  // D = 64: warps 14-15 only keep the barriers
    PSTART();
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    float* dq_stage = reinterpret_cast<float*>(smem + kDQ);  // 2 boxes [D][32 q], SW128
    const bool leader = warp == 12 && lane == 0;
    const float scale = p.scale;
    int it = 0;
    for (int g = 0; g < p.G; ++g) {
      const int h = hk * p.G + g;
      for (int li = 0; li < n_live; ++li, ++it) {
        const int qt = live_list[n_live - 1 - li] & (kFullBit - 1);
        const int b = it & 1;
        PWAIT(&bars.dq_full[b], (it >> 1) & 1, 0);
        tc_fence_after();
        uint32_t v0[32], v1[32];
        tmem_ld32(tmem + lane_base + b * 128 + 64, v0);
        tmem_ld32(tmem + lane_base + b * 128 + 96, v1);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bars.dq_empty[b]);
        if constexpr (DQ8) {
          // Each warp drains its own 32 features independently: 8 chunks of 8
          // queries, [32 d][8 q] fp32 (1 KB) through two alternating buffers,
          // one TMA reduce-add per chunk (box {8 q, 32 d}); no cross-warp barrier.
          if (wq * 32 < D) {
            float* wbuf = dq_stage + wq * 512;  // 2 x 256 floats per warp
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              float* buf = wbuf + (c & 1) * 256;
#ifdef A2D_PROFILE
              const long long tr0 = clock64();
#endif
              if (lane == 0) bulk_wait_read1();  // the reduce that read `buf` two chunks ago is done
#ifdef A2D_PROFILE
              prof[1] += clock64() - tr0;
#endif
              __syncwarp();
              const uint32_t* src = c < 4 ? v0 + 8 * c : v1 + 8 * (c - 4);
              float4* dst = reinterpret_cast<float4*>(buf + lane * 8);
              dst[0] = make_float4(__uint_as_float(src[0]) * scale, __uint_as_float(src[1]) * scale,
                                   __uint_as_float(src[2]) * scale, __uint_as_float(src[3]) * scale);
              dst[1] = make_float4(__uint_as_float(src[4]) * scale, __uint_as_float(src[5]) * scale,
                                   __uint_as_float(src[6]) * scale, __uint_as_float(src[7]) * scale);
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_reduce_add_3d(&p.tm_dq8, buf, qt * BQ + 8 * c, wq * 32, h);
                bulk_commit();
              }
            }
          }
          continue;
        }
#ifdef A2D_PROFILE
        const long long tr0 = clock64();
#endif
        if (leader) bulk_wait_read0();  // previous reduce finished reading the stage
#ifdef A2D_PROFILE
        prof[1] += clock64() - tr0;
#endif
        named_bar_sync(1, 128);
        // box b = queries [32b, 32b+32) x all 128 features, SW128: row d, 16-byte
        // chunk j (queries 4j..4j+3) at position j ^ (d & 7)
        if (d_ok) {
          uint8_t* st = reinterpret_cast<uint8_t*>(dq_stage) + d * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<float4*>(st + ((c ^ (d & 7)) << 4)) =
                make_float4(__uint_as_float(v0[4 * c]) * scale, __uint_as_float(v0[4 * c + 1]) * scale,
                            __uint_as_float(v0[4 * c + 2]) * scale, __uint_as_float(v0[4 * c + 3]) * scale);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<float4*>(st + D * 128 + ((c ^ (d & 7)) << 4)) =
                make_float4(__uint_as_float(v1[4 * c]) * scale, __uint_as_float(v1[4 * c + 1]) * scale,
                            __uint_as_float(v1[4 * c + 2]) * scale, __uint_as_float(v1[4 * c + 3]) * scale);
        }
        fence_async_smem();
        named_bar_sync(1, 128);
        if (leader) {
          tma_reduce_add_3d(&p.tm_dq, dq_stage, qt * BQ, 0, h);
          tma_reduce_add_3d(&p.tm_dq, dq_stage + D * 32, qt * BQ + 32, 0, h);
          bulk_commit();
        }
      }
    }
    if (DQ8 ? lane == 0 : leader) bulk_wait0();
    if (warp == 12) PFLUSH(2);
  } else if (warp >= 4) {
    // ------------------------------------------------ P/dS warpgroups
    // Both warpgroups cover all 128 key rows (TMEM lanes); warpgroup hq owns
    // query columns [32*hq, 32*hq+32) of every iteration.
    regs_inc<152>();
    const int hq = (warp - 4) / 4;
    const int wq = warp % 4;
    const int r = wq * 32 + lane;
    const int key = key0 + r;
    const bool key_ok = key < p.Tk;
    const int kpos = key_ok ? p.k_pos[key] : INT_MAX;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const float sl2 = p.scale_log2;
    const int c0 = hq * 32;
    const int* qpos_base = p.q_pos;
    const int Tq = p.Tq;
    PSTART();
    int it = 0;
    for (int g = 0; g < p.G; ++g) {
      for (int li = 0; li < n_live; ++li, ++it) {
        const int ent = live_list[n_live - 1 - li];
        const int qt = ent & (kFullBit - 1);
        const bool full = (ent & kFullBit) != 0;
        const int b = it & 1, qs = it % QST;
        PWAIT(&bars.qdo_full[qs], (it / QST) & 1, 0);  // stats landed with the TMA stage
        const float4* st4 = reinterpret_cast<const float4*>(smem + kStats + qs * 2 * BQ * 4);
        PWAIT(&bars.s_full[b], (it >> 1) & 1, 1);
        tc_fence_after();
        uint32_t sr[32], dr[32];
        tmem_ld32(tmem + lane_base + b * 128 + c0, sr);
        tmem_ld32(tmem + lane_base + b * 128 + 64 + c0, dr);
        tmem_ld_wait();
        uint32_t pw[16], dw[16];
        // dS is kept unscaled here (dS' = P*(dP-delta)); 1/sqrt(d) is applied in
        // the dQ drain and the dK epilogue. Rows/keys past the chunk end need no
        // mask: K/V rows there are zero-filled (their dS feeds dQ through zero
        // K rows, their dK/dV rows are not stored) and padded query columns
        // have lse2 = +inf (P = 0).
        if (full) {
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            const float4 l4 = st4[(c0 + c) / 4];
            const float4 d4 = st4[(BQ + c0 + c) / 4];
            const float p0 = ex2(fmaf(__uint_as_float(sr[c + 0]), sl2, -l4.x));
            const float p1 = ex2(fmaf(__uint_as_float(sr[c + 1]), sl2, -l4.y));
            const float p2 = ex2(fmaf(__uint_as_float(sr[c + 2]), sl2, -l4.z));
            const float p3 = ex2(fmaf(__uint_as_float(sr[c + 3]), sl2, -l4.w));
            pw[c / 2] = pack_bf16(p0, p1);
            pw[c / 2 + 1] = pack_bf16(p2, p3);
            dw[c / 2] = pack_bf16(p0 * (__uint_as_float(dr[c + 0]) - d4.x), p1 * (__uint_as_float(dr[c + 1]) - d4.y));
            dw[c / 2 + 1] =
                pack_bf16(p2 * (__uint_as_float(dr[c + 2]) - d4.z), p3 * (__uint_as_float(dr[c + 3]) - d4.w));
          }
        } else {
          const int qb0 = qt * BQ + c0;
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            const float4 l4 = st4[(c0 + c) / 4];
            const float4 d4 = st4[(BQ + c0 + c) / 4];
            const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
            const float dl[4] = {d4.x, d4.y, d4.z, d4.w};
            float pv[4], dv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int q = qb0 + c + e;
              const int qp = __ldg(qpos_base + min(q, Tq - 1));
              const bool keep = key_ok && q < Tq && kpos <= qp;
              const float pr = ex2(fmaf(__uint_as_float(sr[c + e]), sl2, -lv[e]));
              pv[e] = keep ? pr : 0.f;
              dv[e] = pv[e] * (__uint_as_float(dr[c + e]) - dl[e]);
            }
            pw[c / 2] = pack_bf16(pv[0], pv[1]);
            pw[c / 2 + 1] = pack_bf16(pv[2], pv[3]);
            dw[c / 2] = pack_bf16(dv[0], dv[1]);
            dw[c / 2 + 1] = pack_bf16(dv[2], dv[3]);
          }
        }
        // P^T and dS^T (bf16 pairs) inside this warpgroup's own S^T columns:
        // [c0, c0+16) and [c0+16, c0+32) — the TMEM A operands of dV and dK
        tmem_st16(tmem + lane_base + b * 128 + c0, pw);
        tmem_st16(tmem + lane_base + b * 128 + c0 + 16, dw);
        if (it >= 1) PWAIT(&bars.ds_free, (it - 1) & 1, 2);  // dQ^T of it-1 done reading dS
        uint8_t* dsrow = smem + kDS;
#pragma unroll
        for (int c8 = 0; c8 < 4; ++c8)
          *reinterpret_cast<uint4*>(dsrow + sw128_offset(r, hq * 4 + c8)) =
              make_uint4(dw[4 * c8], dw[4 * c8 + 1], dw[4 * c8 + 2], dw[4 * c8 + 3]);
        fence_async_smem();
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bars.ds_full[b]);
      }
    }
    if (warp == 4) PFLUSH(1);
    // ------------------------------------------------ dV (hq=0) / dK (hq=1) epilogue
    if (n > 0) {
      mbar_wait(&bars.dkv_full, 0);
      tc_fence_after();
    }
    float* dst = (hq == 0 ? p.dv : p.dk) + ((size_t)hk * p.Tk + key) * D;
    const float oscale = hq == 0 ? 1.f : p.scale;  // dK = (dS')^T Q / sqrt(d)
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
  if (warp == 2) tmem_dealloc<512>(tmem);
}

#include "fa_bwd_q128.cuh"

template <int D, int QST, int PF, bool DQ8 = false>
static cudaError_t launch_bwd_d(const BwdParams& p, cudaStream_t s) {
  constexpr int bytes = bwd::Cfg<D, QST, DQ8>::kBytes;
  static_assert(bytes <= 232448, "backward shared memory exceeds 227 KB");
  cudaError_t e =
      cudaFuncSetAttribute(fa_bwd_kernel<D, QST, PF, DQ8>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  dim3 grid((p.Tk + bwd::BK - 1) / bwd::BK, p.Hkv);
  fa_bwd_kernel<D, QST, PF, DQ8><<<grid, bwd::kThreads, bytes, s>>>(p);
  return cudaGetLastError();
}

// Experiment switch (A2D_BWD_VARIANT, read once): 0 default (the 128-query
// kernel, fa_bwd_q128.cuh, own drain staging, CTA pairs with multicast Q/dO
// loads (single CTAs when the key-tile count is odd), D = 64 or 128), 15 =
// the same without pairs, 7 / 8 = the 128-query kernel with the kStageDs /
// kStageHybrid drain staging, 9 / 10 = own staging with 1/8 / 1/4 of the
// P exps on the FMA pipe (7-11 without pairs), 11 = P^T / dS^T released in
// two parts, 6 = the round-2
// 64-query kernel at D = 128 (3 stages, no prefetch), 1 = it with 2 stages,
// 2 = L2 prefetch 4 ahead, 3 = L2 prefetch 8 ahead, 4 = 4 stages with the
// per-warp 8-query dQ drain, 5 = 3 stages with it.
static int bwd_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("A2D_BWD_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

cudaError_t launch_fa_bwd(const BwdParams& p, int head_dim, cudaStream_t s) {
  if (head_dim != 128 && head_dim != 64) return cudaErrorInvalidValue;
  if (p.Tk <= 0 || p.Hkv <= 0) return cudaSuccess;
  if ((p.Tq + bwd::BQ - 1) / bwd::BQ > bwd::kMaxQTiles) return cudaErrorInvalidValue;
  if (head_dim == 64)
    return bwd_variant() == 6    ? launch_bwd_d<64, 3, 0>(p, s)
           : bwd_variant() == 15 ? launch_bwd_q128<64, bwd2::kStageOwn>(p, s)
                                 : launch_bwd_q128<64, bwd2::kStageOwn, 0, 0, true>(p, s);
  switch (bwd_variant()) {
    case 1: return launch_bwd_d<128, 2, 0>(p, s);
    case 2: return launch_bwd_d<128, 3, 4>(p, s);
    case 3: return launch_bwd_d<128, 3, 8>(p, s);
    case 4: return launch_bwd_d<128, 4, 0, true>(p, s);
    case 5: return launch_bwd_d<128, 3, 0, true>(p, s);
    case 6: return launch_bwd_d<128, 3, 0>(p, s);
    case 7: return launch_bwd_q128<128, bwd2::kStageDs>(p, s);
    case 8: return launch_bwd_q128<128, bwd2::kStageHybrid>(p, s);
    case 9: return launch_bwd_q128<128, bwd2::kStageOwn, 1>(p, s);
    case 10: return launch_bwd_q128<128, bwd2::kStageOwn, 2>(p, s);
    case 11: return launch_bwd_q128<128, bwd2::kStageOwn, 0, 1>(p, s);
    case 15: return launch_bwd_q128<128, bwd2::kStageOwn>(p, s);
    default: return launch_bwd_q128<128, bwd2::kStageOwn, 0, 0, true>(p, s);
  }
}

}  // namespace a2d

#ifdef A2D_PROFILE
extern "C" int a2d_prof_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, a2d::g_bwd_trace, sizeof(long long) * 32 * 16) == cudaSuccess ? 0 : 2;
}
extern "C" int a2d_prof_ablate(int bits) {
  return cudaMemcpyToSymbol(a2d::g_bwd_ablate, &bits, sizeof(int)) == cudaSuccess ? 0 : 2;
}
extern "C" int a2d_prof_read(unsigned long long* out, int n) {
  if (n > 32) n = 32;
  if (cudaMemcpyFromSymbol(out, a2d::g_bwd_prof, n * sizeof(unsigned long long)) != cudaSuccess) return 2;
  unsigned long long z[32] = {0};
  return cudaMemcpyToSymbol(a2d::g_bwd_prof, z, sizeof(z)) == cudaSuccess ? 0 : 2;
}
#endif
