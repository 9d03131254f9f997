// Chunk flash-attention forward for sm_100a (K1) with the ring-step LSE merge
// fused into the epilogue (K2).
//
// Computes, for one Q chunk against one KV chunk (one ring step of
// run_double_ring, ref ring.py:64-79 / oracle.py:97-124):
//   blk.out = softmax(mask(Q K^T / sqrt(d))) V,  blk.lse = natural-log LSE
// and either writes blk (mode 0) or folds it into a running fp32 accumulator
// exactly like block_update (mode 1).  The causal mask compares the carried
// original token positions (ref oracle.py:73-75), so zig-zag chunks need no
// special casing: tiles whose keys all lie after every query are skipped,
// tiles entirely in the past run unmasked, only straddling tiles mask.
//
// Structure (one CTA = 2 query tiles of 128 rows of one head, 12 warps):
//   warp 0      TMA producer: Q once, then K/V tiles through 2-stage rings
//   warp 1      MMA issuer (converged warp, elected lane issues): S_t = Q_t K^T
//               into TMEM, O_t += P_t V
//   warp 2      TMEM allocator
//   warps 4-7   softmax for query tile 0 (thread = row = TMEM lane)
//   warps 8-11  softmax for query tile 1
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [384,384+D);
// P_t (bf16) is written over the first 64 columns of S_t and consumed by a
// TMEM-operand (TS) UMMA. The two softmax groups ping-pong so the tensor core
// runs one tile's GEMMs while the other tile's softmax runs.
// Rescaling of O is lazy: the running max only moves when a row max grows by
// more than 2^8, so O is touched on a handful of tiles per row at most.
#include "sm100.cuh"
#include "kernels.h"

#include <cstdlib>

namespace a2d {

// Optional wait-time instrumentation (-DA2D_PROFILE, build.py --profile):
// g_fwd_prof[role*8 + slot], role 0 MMA warp, 1 softmax WG0 (warp 4 lane 0),
// 2 softmax WG1 (warp 8 lane 0), 3 TMA producer; slot 7 = role's total cycles.
#ifdef A2D_PROFILE
__device__ unsigned long long g_fwd_prof[32];
#define FWAIT(bar, ph, slot)         \
  do {                               \
    const long long t0_ = clock64(); \
    mbar_wait(bar, ph);              \
    prof[slot] += clock64() - t0_;   \
  } while (0)
#define FSTART() const long long pt0_ = clock64()
#define FFLUSH(role)                                                                              \
  do {                                                                                            \
    prof[7] = clock64() - pt0_;                                                                   \
    if (lane == 0)                                                                                \
      for (int s_ = 0; s_ < 8; ++s_) atomicAdd(&g_fwd_prof[(role) * 8 + s_], (unsigned long long)prof[s_]); \
  } while (0)
#else
#define FWAIT(bar, ph, slot) mbar_wait(bar, ph)
#define FSTART()
#define FFLUSH(role)
#endif

namespace fwd {
constexpr int BM = 128, BN = 128;
constexpr int kThreads = 384;
constexpr int KST = 2, VST = 2;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr int kMaxKTiles = 8192;           // live-list capacity (Tk <= 1M per chunk)
constexpr uint16_t kMask0 = 0x4000, kMask1 = 0x8000, kIdx = 0x3fff;
}  // namespace fwd

template <int D>
struct FwdSmem {
  static constexpr int kTileBytes = 128 * D * 2;  // one 128-row bf16 tile
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + 2 * kTileBytes;
  static constexpr int kV = kK + fwd::KST * kTileBytes;
  static constexpr int kList = kV + fwd::VST * kTileBytes;  // live KV tiles (uint16 + mask flags)
  static constexpr int kEnd = kList + fwd::kMaxKTiles * 2;
  static constexpr int kBytes = kEnd + 1024;  // + alignment slack
};

struct FwdBars {
  uint64_t q_full;
  uint64_t k_full[fwd::KST], k_empty[fwd::KST];
  uint64_t v_full[fwd::VST], v_empty[fwd::VST];
  uint64_t s_full[2], p_part[2][3], p_full[2], o_full[2];
  uint32_t tmem_base;
  int n_live;
  int warp_cnt[12];
};

// Tile classification against one query tile's position range.
__device__ __forceinline__ bool tile_live(int2 kb, int qmax, bool causal) {
  return kb.x <= kb.y && (!causal || kb.x <= qmax);
}

// Compacted list of the KV tiles (128 keys) that are live for a CTA's two
// query tiles, with per-query-tile "needs mask" flags (kMask0/kMask1). All 12
// warps take part; ends with __syncthreads-visible writes to `list`/`n_live`.
__device__ __forceinline__ void build_live_list(const FwdParams& p, int2 qr0, int2 qr1, int qmax_cta, bool causal,
                                                int nkt, uint16_t* live_list, int* warp_cnt, int* n_live) {
  using namespace fwd;
  const int warp = warp_id(), lane = lane_id();
  auto classify = [&](int j, bool& lv, uint16_t& ent) {
    const int2 kb = p.k_bounds[j];
    lv = tile_live(kb, qmax_cta, causal);
    const bool tail = (j + 1) * BN > p.Tk;
    const bool m0 = tail || (causal && !(qr0.x <= qr0.y && kb.y <= qr0.x));
    const bool m1 = tail || (causal && !(qr1.x <= qr1.y && kb.y <= qr1.x));
    ent = (uint16_t)(j | (m0 ? kMask0 : 0) | (m1 ? kMask1 : 0));
  };
  const int per_warp = (nkt + 11) / 12;
  const int lo = warp * per_warp, hi = min(nkt, lo + per_warp);
  int cnt = 0;
  for (int base = lo; base < hi; base += 32) {
    const int j = base + lane;
    bool lv = false;
    uint16_t ent = 0;
    if (j < hi) classify(j, lv, ent);
    cnt += __popc(__ballot_sync(0xffffffffu, lv));
  }
  if (lane == 0) warp_cnt[warp] = cnt;
  __syncthreads();
  int off = 0;
  for (int w = 0; w < warp; ++w) off += warp_cnt[w];
  if (warp == 11 && lane == 0) *n_live = off + cnt;
  for (int base = lo; base < hi; base += 32) {
    const int j = base + lane;
    bool lv = false;
    uint16_t ent = 0;
    if (j < hi) classify(j, lv, ent);
    const unsigned m = __ballot_sync(0xffffffffu, lv);
    if (lv) live_list[off + __popc(m & ((1u << lane) - 1u))] = ent;
    off += __popc(m);
  }
}

// Row epilogue shared by both forward kernels: normalise O (TMEM) by l_sum,
// LSE, and the fused ring-step merge (ref block_update, oracle.py:111-124).
template <int D>
__device__ __forceinline__ void fwd_epilogue(const FwdParams& p, uint32_t tO, int h, int row, bool row_ok,
                                             float m_used, float l_sum, bool any) {
  const int it = any ? 1 : 0;
  const bool alive = l_sum > 0.f;
  const float inv = alive ? 1.f / l_sum : 0.f;
  const float lse_blk = alive ? (m_used + __log2f(l_sum)) * 0.69314718055994531f : -INFINITY;
  const size_t lrow = (size_t)h * p.Tq + (row_ok ? row : 0);
  float wa = 0.f, wb = inv, lse_new = lse_blk;
  if (p.merge && row_ok) {
    const float la = p.lse[lrow];
    const float mx2 = fmaxf(la, lse_blk);
    if (mx2 == -INFINITY) {
      lse_new = -INFINITY;
      wa = 0.f;
      wb = 0.f;
    } else {
      const float ea = la == -INFINITY ? 0.f : __expf(la - mx2);
      const float eb = lse_blk == -INFINITY ? 0.f : __expf(lse_blk - mx2);
      const float z = ea + eb;
      lse_new = mx2 + __logf(z);
      wa = ea / z;
      wb = eb / z * inv;
    }
  }
  if (row_ok) p.lse[lrow] = lse_new;
  float* acc = (p.acc_o && row_ok) ? p.acc_o + ((size_t)h * p.Tq + row) * D : nullptr;
  __nv_bfloat16* out =
      (p.out && row_ok) ? p.out + (size_t)h * p.out_stride_h + (size_t)row * p.out_stride_t : nullptr;
#pragma unroll 1
  for (int c = 0; c < D / 32; ++c) {
    uint32_t r[32];
    if (it > 0) {
      tmem_ld32(tO + c * 32, r);
      tmem_ld_wait();
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = 0u;
    }
    if (!row_ok) continue;
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[i + e]) * wb;
      if (p.merge) {
        const float4 a0 = *reinterpret_cast<const float4*>(acc + c * 32 + i);
        const float4 a1 = *reinterpret_cast<const float4*>(acc + c * 32 + i + 4);
        v[0] += a0.x * wa; v[1] += a0.y * wa; v[2] += a0.z * wa; v[3] += a0.w * wa;
        v[4] += a1.x * wa; v[5] += a1.y * wa; v[6] += a1.z * wa; v[7] += a1.w * wa;
      }
      if (acc) {
        *reinterpret_cast<float4*>(acc + c * 32 + i) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(acc + c * 32 + i + 4) = make_float4(v[4], v[5], v[6], v[7]);
      }
      if (out) {
        uint4 u;
        u.x = pack_bf16(v[0], v[1]); u.y = pack_bf16(v[2], v[3]);
        u.z = pack_bf16(v[4], v[5]); u.w = pack_bf16(v[6], v[7]);
        *reinterpret_cast<uint4*>(out + c * 32 + i) = u;
      }
    }
  }
}

// NP: the softmax releases P in NP parts of BN/NP keys (1, 2 or 4) so PV's K
// steps (which run over keys) on the released parts start while it still
// computes the rest; the O rescale moves before the exps to keep that legal.
// One barrier per part (each completes once per iteration: a barrier that
// completed twice before its waiter looked would alias its parity), p_full
// for the last.
// PXF: exp2 pairs on the FMA pipe out of every eight (0, 1, 2 = the default 1/4, 3).
template <int D, int NP, int PXF = 2>
__global__ void __launch_bounds__(fwd::kThreads, 1) fa_fwd_kernel(const __grid_constant__ FwdParams p) {
  using namespace fwd;
  using L = FwdSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in .shared
  __shared__ FwdBars bars;

  const int warp = warp_id(), lane = lane_id();
  const int nqb = (p.Tq + 2 * BM - 1) / (2 * BM);
  const int qb = nqb - 1 - (int)blockIdx.x;  // heaviest (latest) query blocks first
  const int h = blockIdx.y;
  const int hk = h / p.G;
  const int q0 = qb * 2 * BM;
  const int nkt = (p.Tk + BN - 1) / BN;

  // query-tile position ranges (tiles beyond Tq have min > max)
  const int nqt = (p.Tq + BM - 1) / BM;
  int2 qr0 = (2 * qb < nqt) ? p.q_bounds[2 * qb] : make_int2(1, 0);
  int2 qr1 = (2 * qb + 1 < nqt) ? p.q_bounds[2 * qb + 1] : make_int2(1, 0);
  const int qmax_cta = max(qr0.x <= qr0.y ? qr0.y : INT_MIN, qr1.x <= qr1.y ? qr1.y : INT_MIN);
  const bool causal = p.causal != 0;

  if (threadIdx.x == 0) {
    mbar_init(&bars.q_full, 1);
    for (int i = 0; i < KST; ++i) { mbar_init(&bars.k_full[i], 1); mbar_init(&bars.k_empty[i], 1); }
    for (int i = 0; i < VST; ++i) { mbar_init(&bars.v_full[i], 1); mbar_init(&bars.v_empty[i], 1); }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bars.s_full[t], 1);
      for (int q = 0; q < 3; ++q) mbar_init(&bars.p_part[t][q], 128);
      mbar_init(&bars.p_full[t], 128);
      mbar_init(&bars.o_full[t], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&bars.tmem_base);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tm_q);
    tma_prefetch(&p.tm_k);
    tma_prefetch(&p.tm_v);
  }
  // ---- compacted list of live KV tiles for this CTA (causal-dead tiles
  // never cost a loop iteration), with per-query-tile "needs mask" flags.
  uint16_t* live_list = reinterpret_cast<uint16_t*>(smem + L::kList);
  build_live_list(p, qr0, qr1, qmax_cta, causal, nkt, live_list, bars.warp_cnt, &bars.n_live);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const int n = bars.n_live;
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  (void)prof;
  // register budget: the TMA/MMA/alloc warpgroup hands registers to the two
  // softmax warpgroups: 88 + 2 x 208 = 504 = the launch allocation (168 x 3
  // warpgroups; setmaxnreg.inc blocks until the pool has the registers, so
  // the sum must not exceed it). The increase sits
  // inside the softmax branch so ptxas allocates that code at 208 (outside
  // the branch it compiled the softmax at the launch budget and spilled).
  if (warp < 4) regs_dec<88>();
  if (warp == 0) {
    // ------------------------------------------------------------ producer
    FSTART();
    if (lane == 0 && n > 0) {
      mbar_expect_tx(&bars.q_full, 2 * L::kTileBytes);
      for (int t = 0; t < 2; ++t)
        for (int c = 0; c < D / 64; ++c)
          tma_load_3d(smem + L::kQ + t * L::kTileBytes + c * 16384, &p.tm_q, &bars.q_full, c * 64,
                      q0 + t * BM, h);
      for (int it = 0; it < n; ++it) {
        const int j = live_list[it] & kIdx;
        const int ks = it % KST, kph = (it / KST) & 1;
        FWAIT(&bars.k_empty[ks], kph ^ 1, 0);
        mbar_expect_tx(&bars.k_full[ks], L::kTileBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_3d(smem + L::kK + ks * L::kTileBytes + c * 16384, &p.tm_k, &bars.k_full[ks], c * 64,
                      j * BN, hk);
        const int vs = it % VST, vph = (it / VST) & 1;
        FWAIT(&bars.v_empty[vs], vph ^ 1, 1);
        mbar_expect_tx(&bars.v_full[vs], L::kTileBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_3d(smem + L::kV + vs * L::kTileBytes + c * 16384, &p.tm_v, &bars.v_full[vs], c * 64,
                      j * BN, hk);
      }
    }
    FFLUSH(3);
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Converged warp (uniform-register descriptors); an elected lane issues.
    FSTART();
    if (n > 0) {
      constexpr uint32_t id_qk = idesc_bf16(BM, BN, false, false);
      constexpr uint32_t id_pv = idesc_bf16(BM, D, false, true);
      const uint32_t tS[2] = {tmem + 0, tmem + 128};
      const uint32_t tO[2] = {tmem + 256, tmem + 384};
      const uint64_t dQ0 = sdesc_sw128(smem_u32(smem + L::kQ), 16, 1024);
      const uint64_t dK0 = sdesc_sw128(smem_u32(smem + L::kK), 16, 1024);
      const uint64_t dV0 = sdesc_sw128(smem_u32(smem + L::kV), 16384, 1024);
      auto issue_qk = [&](int t, int ks) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint64_t off = (uint64_t)(((k / 4) * 16384 + (k % 4) * 32) >> 4);
          umma_ss(tS[t], dQ0 + (uint64_t)((t * L::kTileBytes) >> 4) + off,
                  dK0 + (uint64_t)((ks * L::kTileBytes) >> 4) + off, id_qk, k > 0);
        }
      };
      auto issue_pv = [&](int t, int vs, bool acc, int k0, int k1) {
#pragma unroll
        for (int k = k0; k < k1; ++k)
          umma_ts(tO[t], tS[t] + k * 8, dV0 + (uint64_t)((vs * L::kTileBytes) >> 4) + (uint64_t)(k * 128), id_pv,
                  (acc || k > 0) ? 1u : 0u);
      };
      mbar_wait(&bars.q_full, 0);
      mbar_wait(&bars.k_full[0], 0);
      tc_fence_after();
      __syncwarp();
      if (elect_one()) {
        issue_qk(0, 0);
        umma_commit(&bars.s_full[0]);
        issue_qk(1, 0);
        umma_commit(&bars.s_full[1]);
        umma_commit(&bars.k_empty[0]);
      }
      __syncwarp();
      for (int it = 0; it < n; ++it) {
        const int vs = it % VST;
        FWAIT(&bars.v_full[vs], (it / VST) & 1, 0);
        const bool more = it + 1 < n;
        const int ks1 = (it + 1) % KST;
        for (int part = 0; part < NP - 1; ++part) {  // released parts of P_0 while the rest is computed
          FWAIT(&bars.p_part[0][part], it & 1, 1);
          tc_fence_after();
          __syncwarp();
          if (elect_one()) issue_pv(0, vs, it > 0, part * BN / 16 / NP, (part + 1) * BN / 16 / NP);
          __syncwarp();
        }
        FWAIT(&bars.p_full[0], it & 1, 1);
        if (more) FWAIT(&bars.k_full[ks1], ((it + 1) / KST) & 1, 2);
        tc_fence_after();
        __syncwarp();
        if (elect_one()) {
          issue_pv(0, vs, it > 0, (NP - 1) * BN / 16 / NP, BN / 16);
          if (more) {
            issue_qk(0, ks1);
            umma_commit(&bars.s_full[0]);
          } else {
            umma_commit(&bars.o_full[0]);
          }
        }
        __syncwarp();
        for (int part = 0; part < NP - 1; ++part) {
          FWAIT(&bars.p_part[1][part], it & 1, 3);
          tc_fence_after();
          __syncwarp();
          if (elect_one()) issue_pv(1, vs, it > 0, part * BN / 16 / NP, (part + 1) * BN / 16 / NP);
          __syncwarp();
        }
        FWAIT(&bars.p_full[1], it & 1, 3);
        tc_fence_after();
        __syncwarp();
        if (elect_one()) {
          issue_pv(1, vs, it > 0, (NP - 1) * BN / 16 / NP, BN / 16);
          umma_commit(&bars.v_empty[vs]);
          if (more) {
            issue_qk(1, ks1);
            umma_commit(&bars.s_full[1]);
            umma_commit(&bars.k_empty[ks1]);
          } else {
            umma_commit(&bars.o_full[1]);
          }
        }
        __syncwarp();
      }
    }
    FFLUSH(0);
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax
    regs_inc<208>();
    const int t = (warp - 4) / 4;          // query tile of this warpgroup
    const int wq = warp % 4;               // TMEM lane quarter
    const int row_in_tile = wq * 32 + lane;
    const int row = q0 + t * BM + row_in_tile;
    const bool row_ok = row < p.Tq;
    const int qpos = row_ok ? p.q_pos[row] : INT_MIN;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t tS = tmem + lane_base + t * 128;
    const uint32_t tO = tmem + lane_base + 256 + t * 128;
    const float sl2 = p.scale_log2;

    float m_used = -INFINITY;  // running max, log2 units (scaled)
    float l_sum = 0.f;
    FSTART();
    for (int it = 0; it < n; ++it) {
      const int ent = live_list[it];
      const int j = ent & kIdx;
      const bool full = (ent & (t == 0 ? kMask0 : kMask1)) == 0;

      FWAIT(&bars.s_full[t], it & 1, 0);
      tc_fence_after();
      float s[BN];
      {
        // all four 32-column loads in flight before a single wait
        uint32_t r0[32], r1[32], r2[32], r3[32];
        tmem_ld32(tS + 0, r0);
        tmem_ld32(tS + 32, r1);
        tmem_ld32(tS + 64, r2);
        tmem_ld32(tS + 96, r3);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          s[i] = __uint_as_float(r0[i]);
          s[32 + i] = __uint_as_float(r1[i]);
          s[64 + i] = __uint_as_float(r2[i]);
          s[96 + i] = __uint_as_float(r3[i]);
        }
      }
      if (!full) {  // straddling / tail tile: per-element mask (branch-free)
        const int tk1 = p.Tk - 1;
#pragma unroll
        for (int c = 0; c < BN; ++c) {
          const int col = j * BN + c;
          const int kpos = __ldg(p.k_pos + min(col, tk1));
          const bool keep = col <= tk1 && (!causal || kpos <= qpos);
          s[c] = keep ? s[c] : -INFINITY;
        }
      }
      // row max: four independent chains of three-input max (FMNMX3)
      static_assert(BN % 8 == 0 && BN >= 16, "row max tiling");
      float mq[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) mq[k] = fmax3(s[k], s[k + 4], s[k + 8]);  // columns 0..11
#pragma unroll
      for (int c = 12; c + 8 <= BN - 4; c += 8) {                           // 12 .. BN-5
        mq[0] = fmax3(mq[0], s[c], s[c + 4]);
        mq[1] = fmax3(mq[1], s[c + 1], s[c + 5]);
        mq[2] = fmax3(mq[2], s[c + 2], s[c + 6]);
        mq[3] = fmax3(mq[3], s[c + 3], s[c + 7]);
      }
      const float mx = fmaxf(fmax3(mq[0], mq[1], s[BN - 4]), fmax3(mq[2], mq[3], fmax3(s[BN - 3], s[BN - 2], s[BN - 1])));
      const float m_tile = mx * sl2;  // -inf stays -inf (sl2 > 0)
      float alpha = 1.f;
      bool rescale = false;
      if (m_tile > m_used + kRescaleThreshold) {
        if (m_used != -INFINITY) { alpha = ex2(m_used - m_tile); rescale = true; }
        m_used = m_tile;
        l_sum *= alpha;
      }
      if (__any_sync(0xffffffffu, rescale)) {
        // O (this tile's previous PV) is complete: s_full's commit tracks it.
        // Rescaled before any part of P is released (PV starts on parts).
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tO + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st32(tO + c * 32, r);
        }
      }
      const float neg_m = m_used == -INFINITY ? 0.f : -m_used;
      const float2 sl2x2 = make_float2(sl2, sl2), nm2 = make_float2(neg_m, neg_m);
      float2 part[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      // P in 32-column chunks, each stored to TMEM (16 bf16 pairs) as soon as
      // it is packed: the packed P never has to be live all at once (no spills)
#pragma unroll
      for (int cc = 0; cc < BN; cc += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int c = cc; c < cc + 32; c += 2) {
          const float2 x = __ffma2_rn(make_float2(s[c], s[c + 1]), sl2x2, nm2);
          float2 e;
          if (((c / 2) & 7) >= 8 - PXF) {  // PXF pairs in eight on the FMA pipe (MUFU relief)
            e = ex2_poly2(x);
          } else {
            e.x = ex2(x.x);
            e.y = ex2(x.y);
          }
          part[(c / 2) & 3] = __fadd2_rn(part[(c / 2) & 3], e);
          pk[(c - cc) / 2] = pack_bf16(e.x, e.y);
        }
        tmem_st16(tS + cc / 2, pk);
        if (NP > 1 && cc + 32 < BN && (cc + 32) % (BN / NP) == 0) {  // a part of P is in TMEM
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bars.p_part[t][(cc + 32) / (BN / NP) - 1]);
        }
      }
      {
        const float2 p01 = __fadd2_rn(part[0], part[1]), p23 = __fadd2_rn(part[2], part[3]);
        const float2 pt = __fadd2_rn(p01, p23);
        l_sum += pt.x + pt.y;
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars.p_full[t]);
    }

    if (warp == 4) FFLUSH(1);
    if (warp == 8) FFLUSH(2);
    // ---------------------------------------------------------- epilogue
    const int it = n;
    if (it > 0) {
      mbar_wait(&bars.o_full[t], 0);
      tc_fence_after();
    }
    fwd_epilogue<D>(p, tO, h, row, row_ok, m_used, l_sum, it > 0);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

template <int D, int NP, int PXF = 2>
static cudaError_t launch_fwd_d(const FwdParams& p, cudaStream_t s) {
  if ((p.Tk + fwd::BN - 1) / fwd::BN > fwd::kMaxKTiles) return cudaErrorInvalidValue;
  const int smem = FwdSmem<D>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(fa_fwd_kernel<D, NP, PXF>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int nqb = (p.Tq + 255) / 256;
  dim3 grid(nqb, p.H);
  fa_fwd_kernel<D, NP, PXF><<<grid, fwd::kThreads, smem, s>>>(p);
  return cudaGetLastError();
}

// Experiment switch (A2D_FWD_VARIANT, read once): 0 default (P released in
// four quarters: 1310 vs 1287 TFLOP/s for halves, 1238 for once, sustained
// S = 128K), 1 = P released once (round 2), 2 = in two halves; 3 / 4 / 5 =
// quarters with 0 / 1/8 / 3/8 of the exp pairs on the FMA pipe (default 1/4).
static int fwd_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("A2D_FWD_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

cudaError_t launch_fa_fwd(const FwdParams& p, int head_dim, cudaStream_t s) {
  if (p.Tq <= 0 || p.H <= 0) return cudaSuccess;
  const int v = fwd_variant();
  if (head_dim == 128)
    return v == 1   ? launch_fwd_d<128, 1>(p, s)
           : v == 2 ? launch_fwd_d<128, 2>(p, s)
           : v == 3 ? launch_fwd_d<128, 4, 0>(p, s)
           : v == 4 ? launch_fwd_d<128, 4, 1>(p, s)
           : v == 5 ? launch_fwd_d<128, 4, 3>(p, s)
                    : launch_fwd_d<128, 4>(p, s);
  if (head_dim == 64)
    return v == 1 ? launch_fwd_d<64, 1>(p, s) : v == 2 ? launch_fwd_d<64, 2>(p, s) : launch_fwd_d<64, 4>(p, s);
  return cudaErrorInvalidValue;
}

}  // namespace a2d

#ifdef A2D_PROFILE
extern "C" int a2d_prof_read_fwd(unsigned long long* out, int n) {
  if (n > 32) n = 32;
  if (cudaMemcpyFromSymbol(out, a2d::g_fwd_prof, n * sizeof(unsigned long long)) != cudaSuccess) return 2;
  unsigned long long z[32] = {0};
  return cudaMemcpyToSymbol(a2d::g_fwd_prof, z, sizeof(z)) == cudaSuccess ? 0 : 2;
}
#endif
