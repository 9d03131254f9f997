// Native SPMD 2D-Attention runtime behind the context C ABI:
//   a2d_nccl_unique_id / a2d_ctx_create / a2d_fwd / a2d_bwd / a2d_ctx_destroy.
//
// The same algorithm as the Python runtime dist.Attn2D with its NCCL
// transport (ref run_2d_attention, ring.py:82-119, plus the distributed
// backward designed there): one process per GPU; head-parallel all-to-all as
// grouped ncclSend/ncclRecv inside the HP communicator; Double-Ring KV
// rotation (inner ring w, outer ring d_cp/w) as point-to-point hops on three
// communicators (inner / outer / dK-dV accumulator), each on its own side
// stream and ordered against the compute stream with events, so a hop
// overlaps the attention kernel beside it. The compute is the library's own
// chunk kernels (a2d_fa_fwd_chunk, a2d_fa_bwd_chunk, packs, conversions).
// Scope: head dim 128, head-major [H][L][d] SeqSharded tensors in zig-zag
// token order (layout.seq_positions). The forward's state (the HeadSharded Q,
// K/V chunk, output and LSE the backward needs) lives in a CALLER-OWNED
// buffer of a2d_saved_bytes() bytes, so any number of layers / micro-batches
// can be in flight and the context holds no per-call state (the reference
// operator is a pure function, ring.py:82-119). The context owns only
// workspaces (ring buffers, staging), reused in stream order.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/attn2d_sm100.h"

namespace a2d {
int set_error(int code, const std::string& msg);
}

namespace {

using a2d::set_error;

struct Step {
  int source, inner, outer;
};

struct Ctx {
  int rank = 0, world = 1, d_hp = 1, d_cp = 1, w = 1, placement = 0, H = 0, Hkv = 0, d = 128, causal = 1;
  int64_t S = 0, L = 0, C = 0, C_pad = 0;
  int hp = 0, cp = 0, Hl = 0, Hkl = 0, H_rep = 0, rep = 1, n_outer = 1;
  float scale = 0.f;
  ncclComm_t world_comm = nullptr, hp_comm = nullptr, c_inner = nullptr, c_outer = nullptr, c_dkv = nullptr;
  cudaStream_t s_inner = nullptr, s_outer = nullptr, s_dkv = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_inner = nullptr, ev_outer = nullptr, ev_dkv = nullptr;
  std::vector<Step> steps;
  int inner_to = 0, inner_from = 0, outer_to = 0, outer_from = 0, diag_to = 0, diag_from = 0;
  std::vector<int32_t*> pos, b128, b64;  // per CP chunk j (device)
  int32_t *smap = nullptr, *dmap_k = nullptr, *dmap_v = nullptr;
  std::vector<void*> allocs;
  // workspaces (no per-call state: see Saved)
  uint16_t *kv_send = nullptr, *q_recv = nullptr, *kv_recv = nullptr;
  uint16_t *doh = nullptr, *g_send = nullptr, *dkv_send = nullptr;
  uint16_t* ring[4] = {nullptr, nullptr, nullptr, nullptr};  // inner0, inner1, outer0, outer1
  float *acc = nullptr, *lse2 = nullptr, *delta = nullptr, *dq_acc = nullptr;
  float *dkv = nullptr, *part = nullptr, *dacc[2] = {nullptr, nullptr}, *g32_send = nullptr, *g32_recv = nullptr;
  float* g32_sum = nullptr;
  void* dkv_home = nullptr;
  size_t off_kv = 0, off_out = 0, off_lse = 0, saved_bytes = 0;  // Saved layout
  bool comm = true;  // false: every NCCL call skipped (same kernels / buffers) — exposed-comm measurement only
  // copy-engine head-parallel exchange ("symm"): every HP rank's exchange
  // buffer is IPC-mapped into its peers; a rank writes the chunk for peer p
  // straight into p's buffer with cudaMemcpyAsync (no SMs), then a tiny NCCL
  // all-reduce on the HP communicator is the barrier after which every
  // incoming chunk has landed. IN region: q + kv (fwd) / dO (bwd); OUT: out /
  // dq + dk + dv; consecutive uses of one region are always separated by an
  // exchange (hence a barrier) on the other, so no extra handshake is needed.
  bool symm = false;
  char* xbuf = nullptr;
  size_t x_in = 0, x_out = 0;
  std::vector<char*> xpeer;  // [d_hp]: peers' mapped buffers (own = xbuf)
  std::vector<cudaStream_t> xs;
  std::vector<cudaEvent_t> xe;
  int* xflag = nullptr;
  // optional per-kernel CUDA-event timing of the attention kernels (bench roofline)
  bool timing = false;
  std::vector<cudaEvent_t> tev[2];  // [0] forward, [1] backward: start/end pairs
  size_t tused[2] = {0, 0};
};



// One forward's state inside the caller's saved buffer (256-byte aligned
// regions): HeadSharded Q [Hl][C][128] bf16, K/V chunk [2][Hkl][C][128] bf16,
// output [Hl][C][128] bf16, natural-log LSE [Hl][C] fp32.
struct Saved {
  uint16_t* qh;
  uint16_t* kvh;
  uint16_t* out_h;
  float* lse;
};

Saved saved_view(const Ctx& c, const void* base) {
  char* b = static_cast<char*>(const_cast<void*>(base));
  return {reinterpret_cast<uint16_t*>(b), reinterpret_cast<uint16_t*>(b + c.off_kv),
          reinterpret_cast<uint16_t*>(b + c.off_out), reinterpret_cast<float*>(b + c.off_lse)};
}

#define NCCL_TRY(x)                                                                                  \
  do {                                                                                               \
    ncclResult_t r_ = (x);                                                                           \
    if (r_ != ncclSuccess) return set_error(A2D_ECUDA, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)
#define CUDA_TRY(x)                                                                                  \
  do {                                                                                               \
    cudaError_t e_ = (x);                                                                            \
    if (e_ != cudaSuccess) return set_error(A2D_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define A2D_TRY(x)      \
  do {                  \
    int rc_ = (x);      \
    if (rc_) return rc_; \
  } while (0)

// Bracket one attention-kernel launch with events on `s` when timing is on.
int tmark(Ctx& c, int which, cudaStream_t s) {
  if (!c.timing) return A2D_OK;
  std::vector<cudaEvent_t>& v = c.tev[which];
  if (c.tused[which] == v.size()) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    v.push_back(e);
  }
  CUDA_TRY(cudaEventRecord(v[c.tused[which]++], s));
  return A2D_OK;
}

template <class T>
int dalloc(Ctx& c, T** p, size_t n) {
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T)));
  c.allocs.push_back(*p);
  return A2D_OK;
}

int src_of(int j, int o, int t, int w, int n) {  // ring.py:53-59
  const int ring = j / w, pos = j % w;
  return ((ring - o) % n + n) % n * w + ((pos - t) % w + w) % w;
}

// CP rank j's schedule (schedule.build_ring_schedule) and peers
// (schedule.ring_peers): inner_to, inner_from, outer_to, outer_from, diag_to, diag_from
void ring_plan(int d_cp, int w, int j, std::vector<Step>* steps, int peers[6]) {
  const int n = d_cp / w;
  steps->clear();
  for (int o = 0; o < n; ++o)
    for (int t = 0; t < w; ++t) steps->push_back({src_of(j, o, t, w, n), t, o});
  auto idx = [&](int r, int p) { return ((r % n + n) % n) * w + ((p % w + w) % w); };
  const int ring = j / w, pos = j % w;
  const int v[6] = {idx(ring, pos + 1), idx(ring, pos - 1), idx(ring + 1, pos),
                    idx(ring - 1, pos), idx(ring + 1, pos + 1), idx(ring - 1, pos - 1)};
  std::copy(v, v + 6, peers);
}

// All-to-all of bytes_per_peer between the members of the HP group: chunk p
// of `send` goes to peer p; peer p's chunk for this rank lands at position p.
// NCCL transport: grouped ncclSend/ncclRecv into `recv`. Copy-engine
// transport: into the exchange buffer at byte offset `off` (returned via
// *landed; `recv` is not touched).
int a2a(Ctx& c, const void* send, void* recv, size_t bytes_per_peer, cudaStream_t s, size_t off = 0,
        const void** landed = nullptr) {
  if (landed) *landed = recv;
  if (c.symm) {
    char* dst0 = c.xbuf + off;
    if (landed) *landed = dst0;
    if (!c.comm) return A2D_OK;
    CUDA_TRY(cudaEventRecord(c.ev_ready, s));
    for (int i = 0; i < c.d_hp - 1; ++i) {
      const int p = (c.hp + 1 + i) % c.d_hp;
      CUDA_TRY(cudaStreamWaitEvent(c.xs[i], c.ev_ready, 0));
      CUDA_TRY(cudaMemcpyAsync(c.xpeer[p] + off + (size_t)c.hp * bytes_per_peer,
                               static_cast<const char*>(send) + (size_t)p * bytes_per_peer, bytes_per_peer,
                               cudaMemcpyDeviceToDevice, c.xs[i]));
      CUDA_TRY(cudaEventRecord(c.xe[i], c.xs[i]));
    }
    CUDA_TRY(cudaMemcpyAsync(dst0 + (size_t)c.hp * bytes_per_peer,
                             static_cast<const char*>(send) + (size_t)c.hp * bytes_per_peer, bytes_per_peer,
                             cudaMemcpyDeviceToDevice, s));
    for (int i = 0; i < c.d_hp - 1; ++i) CUDA_TRY(cudaStreamWaitEvent(s, c.xe[i], 0));
    NCCL_TRY(ncclAllReduce(c.xflag, c.xflag, 1, ncclInt32, ncclSum, c.hp_comm, s));  // barrier: all chunks landed
    return A2D_OK;
  }
  if (!c.comm) return A2D_OK;
  NCCL_TRY(ncclGroupStart());
  for (int p = 0; p < c.d_hp; ++p) {
    NCCL_TRY(ncclSend(static_cast<const char*>(send) + p * bytes_per_peer, bytes_per_peer, ncclUint8, p, c.hp_comm, s));
    NCCL_TRY(ncclRecv(static_cast<char*>(recv) + p * bytes_per_peer, bytes_per_peer, ncclUint8, p, c.hp_comm, s));
  }
  NCCL_TRY(ncclGroupEnd());
  return A2D_OK;
}

// a2a whose result must end in `dst` (a caller buffer): copy-engine data is
// moved out of the exchange buffer with one local device copy.
int a2a_to(Ctx& c, const void* send, void* dst, size_t bytes_per_peer, cudaStream_t s, size_t off) {
  const void* landed = nullptr;
  A2D_TRY(a2a(c, send, dst, bytes_per_peer, s, off, &landed));
  if (landed != dst)
    CUDA_TRY(cudaMemcpyAsync(dst, landed, bytes_per_peer * c.d_hp, cudaMemcpyDeviceToDevice, s));
  return A2D_OK;
}

// one ring hop on a side stream, ordered after everything enqueued on `main` so far
int hop(Ctx& c, ncclComm_t comm, cudaStream_t side, cudaStream_t main, const void* send, int to, void* recv, int from,
        size_t bytes, cudaEvent_t done) {
  CUDA_TRY(cudaEventRecord(c.ev_ready, main));
  CUDA_TRY(cudaStreamWaitEvent(side, c.ev_ready, 0));
  if (c.comm) {
    NCCL_TRY(ncclGroupStart());
    NCCL_TRY(ncclSend(send, bytes, ncclUint8, to, comm, side));
    NCCL_TRY(ncclRecv(recv, bytes, ncclUint8, from, comm, side));
    NCCL_TRY(ncclGroupEnd());
  }
  CUDA_TRY(cudaEventRecord(done, side));
  return A2D_OK;
}

// zig-zag positions of CP chunk j (layout.cp_positions)
std::vector<int32_t> cp_positions(int64_t S, int d_cp, int j) {
  const int64_t sigma = S / (2 * d_cp), C = S / d_cp;
  std::vector<int32_t> out(C);
  for (int64_t u = 0; u < C; ++u) {
    const int64_t slot = j * C + u;
    const int64_t jj = slot / (2 * sigma), uu = slot % (2 * sigma);
    const int64_t stripe = uu < sigma ? jj : 2 * d_cp - 1 - jj;
    out[u] = (int32_t)(stripe * sigma + uu % sigma);
  }
  return out;
}

void abort_comms(Ctx& c) {
  for (ncclComm_t* m : {&c.c_dkv, &c.c_outer, &c.c_inner, &c.hp_comm, &c.world_comm})
    if (*m) {
      ncclCommAbort(*m);
      *m = nullptr;
    }
}

int destroy(Ctx* c) {
  if (!c) return A2D_OK;
  cudaDeviceSynchronize();
  for (int p = 0; p < (int)c->xpeer.size(); ++p)
    if (c->xpeer[p] && c->xpeer[p] != c->xbuf) cudaIpcCloseMemHandle(c->xpeer[p]);
  for (cudaStream_t x : c->xs) cudaStreamDestroy(x);
  for (auto& v : c->tev)
    for (cudaEvent_t e : v) cudaEventDestroy(e);
  for (cudaEvent_t x : c->xe) cudaEventDestroy(x);
  for (ncclComm_t* m : {&c->c_dkv, &c->c_outer, &c->c_inner, &c->hp_comm, &c->world_comm})
    if (*m) ncclCommDestroy(*m);
  for (cudaStream_t s : {c->s_inner, c->s_outer, c->s_dkv})
    if (s) cudaStreamDestroy(s);
  for (cudaEvent_t e : {c->ev_ready, c->ev_inner, c->ev_outer, c->ev_dkv})
    if (e) cudaEventDestroy(e);
  for (void* p : c->allocs) cudaFree(p);
  delete c;
  return A2D_OK;
}

// dst = this rank's SeqSharded tensor; src HeadSharded (B heads, C tokens, 128):
// pack [peer][B][L][128] then all-to-all (d_hp = 1: plain copy / conversion)
int gather_bf16(Ctx& c, const uint16_t* src, int B, uint16_t* dst, cudaStream_t s, size_t off) {
  const size_t chunk = (size_t)B * c.L * 128 * 2;
  if (c.d_hp == 1) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, chunk, cudaMemcpyDeviceToDevice, s));
    return A2D_OK;
  }
  A2D_TRY(a2d_permute_blocks(src, c.g_send, B, c.d_hp, (int64_t)c.L * 128 * 2, s));
  return a2a_to(c, c.g_send, dst, chunk, s, off);
}

int gather_f32_to_bf16(Ctx& c, const float* src, int B, uint16_t* dst, cudaStream_t s, size_t off) {
  if (c.d_hp == 1) return a2d_permute_f32_to_bf16(src, dst, 1, 1, (int64_t)B * c.C * 128, s);
  A2D_TRY(a2d_permute_f32_to_bf16(src, c.g_send, B, c.d_hp, (int64_t)c.L * 128, s));
  return a2a_to(c, c.g_send, dst, (size_t)B * c.L * 128 * 2, s, off);
}

int ring_forward(Ctx& c, const Saved& sv, cudaStream_t s) {
  const size_t kv_elems = (size_t)2 * c.Hkl * c.C * 128, kv_bytes = kv_elems * 2, half = kv_elems / 2;
  const int64_t q_rows = (int64_t)c.C;
  if (c.d_cp == 1) {
    A2D_TRY(tmark(c, 0, s));
    A2D_TRY(a2d_fa_fwd_chunk(sv.qh, sv.kvh, sv.kvh + half, c.pos[c.cp], c.pos[c.cp], c.b128[c.cp], c.b128[c.cp], c.Hl,
                             c.Hkl, q_rows, q_rows, 128, c.causal, c.scale, 0, sv.lse, nullptr, sv.out_h, s));
    return tmark(c, 0, s);
  }
  const uint16_t *cur = sv.kvh, *first = sv.kvh;
  uint16_t* nxt_inner = nullptr;
  uint16_t* nxt_outer = nullptr;
  int n_out = 0;
  for (int st = 0; st < c.d_cp; ++st) {
    const Step step = c.steps[st];
    const int t = step.inner, o = step.outer;
    const bool last = st == c.d_cp - 1;
    if (t == 0 && o + 1 < c.n_outer) {
      nxt_outer = c.ring[2 + n_out % 2];
      ++n_out;
      A2D_TRY(hop(c, c.c_outer, c.s_outer, s, first, c.outer_to, nxt_outer, c.outer_from, kv_bytes, c.ev_outer));
    }
    if (t + 1 < c.w) {
      nxt_inner = c.ring[(t + 1) % 2];
      A2D_TRY(hop(c, c.c_inner, c.s_inner, s, cur, c.inner_to, nxt_inner, c.inner_from, kv_bytes, c.ev_inner));
    }
    A2D_TRY(tmark(c, 0, s));
    A2D_TRY(a2d_fa_fwd_chunk(sv.qh, cur, cur + half, c.pos[c.cp], c.pos[step.source], c.b128[c.cp],
                             c.b128[step.source], c.Hl, c.Hkl, q_rows, q_rows, 128, c.causal, c.scale, st > 0 ? 1 : 0,
                             sv.lse, c.acc, last ? sv.out_h : nullptr, s));
    A2D_TRY(tmark(c, 0, s));
    if (t + 1 < c.w) {
      CUDA_TRY(cudaStreamWaitEvent(s, c.ev_inner, 0));
      cur = nxt_inner;
    } else if (!last) {
      CUDA_TRY(cudaStreamWaitEvent(s, c.ev_outer, 0));
      cur = first = nxt_outer;
    }
  }
  return A2D_OK;
}

// returns the home dK/dV buffer ([2][Hkl][C][128]) and whether it is bf16
int ring_backward(Ctx& c, const Saved& sv, const uint16_t* dO, cudaStream_t s, const void** home, bool* home_bf16) {
  const size_t kv_elems = (size_t)2 * c.Hkl * c.C * 128, kv_bytes = kv_elems * 2, half = kv_elems / 2;
  const int64_t T = (int64_t)c.C;
  const uint16_t* kv_own = sv.kvh;
  if (c.d_cp == 1) {
    A2D_TRY(tmark(c, 1, s));
    A2D_TRY(a2d_fa_bwd_chunk(sv.qh, kv_own, kv_own + half, dO, c.pos[c.cp], c.pos[c.cp], c.b64[c.cp], c.b128[c.cp],
                             c.lse2, c.delta, c.dq_acc, c.dkv, c.dkv + half, 0, c.Hl, c.Hkl, T, T, 128, c.causal,
                             c.scale, s));
    A2D_TRY(tmark(c, 1, s));
    *home = c.dkv;
    *home_bf16 = false;
    return A2D_OK;
  }
  const bool hb = c.rep == 1;  // home adds nothing: the last hop may carry bf16 (bit-identical)
  const uint16_t *cur = kv_own, *first = kv_own;
  uint16_t *nxt_inner = nullptr, *nxt_outer = nullptr;
  int n_out = 0;
  for (int st = 0; st < c.d_cp; ++st) {
    const Step step = c.steps[st];
    const int t = step.inner, o = step.outer;
    const bool last = st == c.d_cp - 1;
    if (t == 0 && o + 1 < c.n_outer) {
      nxt_outer = c.ring[2 + n_out % 2];
      ++n_out;
      A2D_TRY(hop(c, c.c_outer, c.s_outer, s, first, c.outer_to, nxt_outer, c.outer_from, kv_bytes, c.ev_outer));
    }
    if (t + 1 < c.w) {
      nxt_inner = c.ring[(t + 1) % 2];
      A2D_TRY(hop(c, c.c_inner, c.s_inner, s, cur, c.inner_to, nxt_inner, c.inner_from, kv_bytes, c.ev_inner));
    }
    float* tgt = st == 0 ? c.dacc[0] : c.part;
    A2D_TRY(tmark(c, 1, s));
    A2D_TRY(a2d_fa_bwd_chunk(sv.qh, cur, cur + half, dO, c.pos[c.cp], c.pos[step.source], c.b64[c.cp],
                             c.b128[step.source], c.lse2, c.delta, c.dq_acc, tgt, tgt + half, 0, c.Hl, c.Hkl, T, T, 128,
                             c.causal, c.scale, s));
    A2D_TRY(tmark(c, 1, s));
    if (st > 0) {  // the travelling accumulator of this chunk arrived in dacc[st % 2]
      CUDA_TRY(cudaStreamWaitEvent(s, c.ev_dkv, 0));
      A2D_TRY(a2d_add_f32(c.dacc[st % 2], c.part, (int64_t)kv_elems, s));
    }
    // next consumer: (r, p+1) inside an outer step, the diagonal (r+1, p+1) across and home
    const bool diag = last || (st + 1) % c.w == 0;
    const int to = diag ? c.diag_to : c.inner_to, from = diag ? c.diag_from : c.inner_from;
    const void* src = c.dacc[st % 2];
    size_t bytes = kv_elems * 4;
    void* dst = last ? c.dkv_home : c.dacc[(st + 1) % 2];
    if (last && hb) {
      A2D_TRY(a2d_f32_to_bf16(c.dacc[st % 2], c.dkv_send, (int64_t)kv_elems, s));
      src = c.dkv_send;
      bytes = kv_elems * 2;
    }
    A2D_TRY(hop(c, c.c_dkv, c.s_dkv, s, src, to, dst, from, bytes, c.ev_dkv));
    if (t + 1 < c.w) {
      CUDA_TRY(cudaStreamWaitEvent(s, c.ev_inner, 0));
      cur = nxt_inner;
    } else if (!last) {
      CUDA_TRY(cudaStreamWaitEvent(s, c.ev_outer, 0));
      cur = first = nxt_outer;
    }
  }
  CUDA_TRY(cudaStreamWaitEvent(s, c.ev_dkv, 0));
  *home = c.dkv_home;
  *home_bf16 = hb;
  return A2D_OK;
}

// Copy-engine exchange setup (collective over the HP group): allocate the
// IN/OUT exchange buffer, share CUDA IPC handles with an NCCL all-gather, map
// the peers' buffers. Every rank must succeed (all-reduce MIN of a flag) or
// all fall back to NCCL together. A2D_TRANSPORT=nccl skips it.
int setup_symm(Ctx& c) {
  const char* tr = getenv("A2D_TRANSPORT");
  if (tr && std::string(tr) == "nccl") return A2D_OK;
  const size_t L128 = (size_t)c.L * 128;
  c.x_in = (size_t)c.d_hp * L128 * 2 * (c.Hl + 2 * c.Hkl);
  c.x_out = (size_t)c.d_hp * L128 * (2 * c.Hl + 2 * c.Hkl * (c.rep == 1 ? 2 : 4));
  c.x_in = (c.x_in + 255) / 256 * 256;
  int ok = 1;
  if (cudaMalloc(&c.xbuf, c.x_in + c.x_out) != cudaSuccess) {
    ok = 0;
    c.xbuf = nullptr;
    cudaGetLastError();
  }
  cudaIpcMemHandle_t h{};
  if (ok && cudaIpcGetMemHandle(&h, c.xbuf) != cudaSuccess) {
    ok = 0;
    cudaGetLastError();
  }
  char* dh = nullptr;
  CUDA_TRY(cudaMalloc(&dh, (c.d_hp + 1) * sizeof(h)));
  CUDA_TRY(cudaMemcpy(dh + c.d_hp * sizeof(h), &h, sizeof(h), cudaMemcpyHostToDevice));
  NCCL_TRY(ncclAllGather(dh + c.d_hp * sizeof(h), dh, sizeof(h), ncclUint8, c.hp_comm, nullptr));
  CUDA_TRY(cudaDeviceSynchronize());
  std::vector<cudaIpcMemHandle_t> hs(c.d_hp);
  CUDA_TRY(cudaMemcpy(hs.data(), dh, c.d_hp * sizeof(h), cudaMemcpyDeviceToHost));
  c.xpeer.assign(c.d_hp, nullptr);
  for (int p = 0; p < c.d_hp && ok; ++p) {
    if (p == c.hp) {
      c.xpeer[p] = c.xbuf;
      continue;
    }
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, hs[p], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      ok = 0;
      cudaGetLastError();
    } else {
      c.xpeer[p] = static_cast<char*>(ptr);
    }
  }
  int* dflag = reinterpret_cast<int*>(dh);
  CUDA_TRY(cudaMemcpy(dflag, &ok, sizeof(int), cudaMemcpyHostToDevice));
  NCCL_TRY(ncclAllReduce(dflag, dflag, 1, ncclInt32, ncclMin, c.hp_comm, nullptr));
  CUDA_TRY(cudaDeviceSynchronize());
  int all = 0;
  CUDA_TRY(cudaMemcpy(&all, dflag, sizeof(int), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaFree(dh));
  if (!all) {  // someone failed: everyone stays on NCCL
    for (int p = 0; p < c.d_hp; ++p)
      if (c.xpeer[p] && c.xpeer[p] != c.xbuf) cudaIpcCloseMemHandle(c.xpeer[p]);
    c.xpeer.clear();
    if (c.xbuf) cudaFree(c.xbuf);
    c.xbuf = nullptr;
    return A2D_OK;
  }
  c.allocs.push_back(c.xbuf);
  A2D_TRY(dalloc(c, &c.xflag, 1));
  CUDA_TRY(cudaMemset(c.xflag, 0, sizeof(int)));
  c.xs.resize(c.d_hp - 1);
  c.xe.resize(c.d_hp - 1);
  for (int i = 0; i < c.d_hp - 1; ++i) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c.xs[i], cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c.xe[i], cudaEventDisableTiming));
  }
  c.symm = true;
  return A2D_OK;
}

int create(const void* id, int rank, int world, int d_hp, int d_cp, int w, int placement, int H, int Hkv, int d,
           int64_t S, int causal, Ctx** out) {
  if (d != 128) return set_error(A2D_EINVAL, "a2d_ctx_create: the native runtime supports head dim 128");
  if (d_hp < 1 || d_cp < 1 || d_hp * d_cp != world) return set_error(A2D_EINVAL, "a2d_ctx_create: world != d_hp*d_cp");
  if (w < 1 || d_cp % w) return set_error(A2D_EINVAL, "inner ring size " + std::to_string(w) + " must divide d_cp=" + std::to_string(d_cp));
  if (H <= 0 || Hkv <= 0 || H % Hkv) return set_error(A2D_EINVAL, "a2d_ctx_create: H must be a multiple of H_kv");
  if (d_hp > H) return set_error(A2D_EINVAL, "d_hp=" + std::to_string(d_hp) + " exceeds H=" + std::to_string(H));
  if (H % d_hp) return set_error(A2D_EINVAL, "a2d_ctx_create: H not divisible by d_hp");
  if (S <= 0 || S % (2 * world)) return set_error(A2D_EINVAL, "a2d_ctx_create: S must be divisible by 2*d_hp*d_cp");
  Ctx* c = new Ctx();
  *out = c;
  c->rank = rank; c->world = world; c->d_hp = d_hp; c->d_cp = d_cp; c->w = w; c->placement = placement;
  c->H = H; c->Hkv = Hkv; c->d = d; c->S = S; c->causal = causal;
  c->H_rep = d_hp <= Hkv ? Hkv : std::lcm(Hkv, d_hp);
  if (c->H_rep % d_hp) return set_error(A2D_EINVAL, "a2d_ctx_create: replicated KV heads not divisible by d_hp");
  c->rep = c->H_rep / Hkv;
  c->Hl = H / d_hp; c->Hkl = c->H_rep / d_hp;
  c->L = S / world; c->C = S / d_cp; c->C_pad = (c->C + 63) / 64 * 64;
  c->n_outer = d_cp / w;
  c->scale = 1.0f / sqrtf((float)d);
  if (placement == 0) { c->cp = rank / d_hp; c->hp = rank % d_hp; }  // head-first: rank = hp + d_hp*cp
  else { c->hp = rank / d_cp; c->cp = rank % d_cp; }                 // context-first: rank = cp + d_cp*hp
  // ---- communicators (ncclCommSplit keeps the key order: HP rank = hp, ring rank = cp)
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  NCCL_TRY(ncclCommInitRank(&c->world_comm, world, uid, rank));
  NCCL_TRY(ncclCommSplit(c->world_comm, c->cp, c->hp, &c->hp_comm, nullptr));
  NCCL_TRY(ncclCommSplit(c->world_comm, c->hp, c->cp, &c->c_inner, nullptr));
  NCCL_TRY(ncclCommSplit(c->world_comm, c->hp, c->cp, &c->c_outer, nullptr));
  NCCL_TRY(ncclCommSplit(c->world_comm, c->hp, c->cp, &c->c_dkv, nullptr));
  for (cudaStream_t* s : {&c->s_inner, &c->s_outer, &c->s_dkv}) CUDA_TRY(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&c->ev_ready, &c->ev_inner, &c->ev_outer, &c->ev_dkv})
    CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  // ---- schedule and peers (schedule.build_ring_schedule / ring_peers)
  int peers[6];
  ring_plan(d_cp, w, c->cp, &c->steps, peers);
  c->inner_to = peers[0]; c->inner_from = peers[1]; c->outer_to = peers[2];
  c->outer_from = peers[3]; c->diag_to = peers[4]; c->diag_from = peers[5];
  // ---- positions and tile bounds of every CP chunk
  const int64_t C = c->C;
  for (int jj = 0; jj < d_cp; ++jj) {
    std::vector<int32_t> hpos = cp_positions(S, d_cp, jj);
    int32_t *p = nullptr, *b1 = nullptr, *b2 = nullptr;
    A2D_TRY(dalloc(*c, &p, C));
    A2D_TRY(dalloc(*c, &b1, 2 * ((C + 127) / 128)));
    A2D_TRY(dalloc(*c, &b2, 2 * ((C + 63) / 64)));
    CUDA_TRY(cudaMemcpy(p, hpos.data(), C * 4, cudaMemcpyHostToDevice));
    A2D_TRY(a2d_tile_bounds(p, C, 128, b1, nullptr));
    A2D_TRY(a2d_tile_bounds(p, C, 64, b2, nullptr));
    c->pos.push_back(p); c->b128.push_back(b1); c->b64.push_back(b2);
  }
  // ---- KV pack maps: block (peer, t, hl) of [d_hp][2][Hkl] reads source head (peer*Hkl + hl) / rep
  std::vector<int32_t> sm, dk, dv;
  for (int p = 0; p < d_hp; ++p)
    for (int hl = 0; hl < c->Hkl; ++hl) {
      sm.push_back((p * c->Hkl + hl) / c->rep);
      dk.push_back(p * 2 * c->Hkl + hl);
      dv.push_back(p * 2 * c->Hkl + c->Hkl + hl);
    }
  A2D_TRY(dalloc(*c, &c->smap, sm.size()));
  A2D_TRY(dalloc(*c, &c->dmap_k, dk.size()));
  A2D_TRY(dalloc(*c, &c->dmap_v, dv.size()));
  CUDA_TRY(cudaMemcpy(c->smap, sm.data(), sm.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->dmap_k, dk.data(), dk.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->dmap_v, dv.data(), dv.size() * 4, cudaMemcpyHostToDevice));
  // ---- buffers
  const size_t qe = (size_t)c->Hl * C * 128, kve = (size_t)2 * c->Hkl * C * 128;
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  c->off_kv = up(qe * 2);
  c->off_out = c->off_kv + up(kve * 2);
  c->off_lse = c->off_out + up(qe * 2);
  c->saved_bytes = c->off_lse + up((size_t)c->Hl * C * 4);
  if (d_hp > 1) {
    A2D_TRY(dalloc(*c, &c->kv_send, kve));
    A2D_TRY(dalloc(*c, &c->q_recv, qe));
    A2D_TRY(dalloc(*c, &c->kv_recv, kve));
    A2D_TRY(dalloc(*c, &c->g_send, std::max(qe, kve / 2)));
    A2D_TRY(dalloc(*c, &c->doh, qe));
  }
  A2D_TRY(dalloc(*c, &c->lse2, (size_t)c->Hl * c->C_pad));
  A2D_TRY(dalloc(*c, &c->delta, (size_t)c->Hl * c->C_pad));
  A2D_TRY(dalloc(*c, &c->dq_acc, (size_t)c->Hl * 128 * c->C_pad));
  A2D_TRY(dalloc(*c, &c->dkv, kve));
  if (d_cp > 1) {
    A2D_TRY(dalloc(*c, &c->acc, qe));
    for (auto& r : c->ring) A2D_TRY(dalloc(*c, &r, kve));
    A2D_TRY(dalloc(*c, &c->part, kve));
    A2D_TRY(dalloc(*c, &c->dacc[0], kve));
    A2D_TRY(dalloc(*c, &c->dacc[1], kve));
    A2D_TRY(dalloc(*c, &c->dkv_send, kve));
    float* home = nullptr;
    A2D_TRY(dalloc(*c, &home, kve));  // fp32-sized: also holds the bf16 home hop
    c->dkv_home = home;
  }
  if (c->rep > 1) {
    const size_t ge = (size_t)c->Hkl * C * 128;  // = H_rep * L * 128
    A2D_TRY(dalloc(*c, &c->g32_send, ge));
    A2D_TRY(dalloc(*c, &c->g32_recv, ge));
    A2D_TRY(dalloc(*c, &c->g32_sum, (size_t)Hkv * c->L * 128));
  }
  if (d_hp > 1) A2D_TRY(setup_symm(*c));
  CUDA_TRY(cudaDeviceSynchronize());
  return A2D_OK;
}

int forward(Ctx& c, const void* q, const void* k, const void* v, void* out, void* saved, cudaStream_t s) {
  const size_t L128 = (size_t)c.L * 128;
  const Saved sv = saved_view(c, saved);
  // KV pack [peer][2][Hkl][L][128] (GQA replication by the head map); with
  // d_hp = 1 the pack IS the HeadSharded KV chunk (written into the state)
  uint16_t* kvp = c.d_hp == 1 ? sv.kvh : c.kv_send;
  A2D_TRY(a2d_gather_blocks(k, kvp, c.smap, c.dmap_k, (int64_t)c.d_hp * c.Hkl, (int64_t)L128 * 2, s));
  A2D_TRY(a2d_gather_blocks(v, kvp, c.smap, c.dmap_v, (int64_t)c.d_hp * c.Hkl, (int64_t)L128 * 2, s));
  if (c.d_hp == 1) {
    // the state owns its Q (no aliasing of the caller's buffer)
    CUDA_TRY(cudaMemcpyAsync(sv.qh, q, (size_t)c.Hl * L128 * 2, cudaMemcpyDeviceToDevice, s));
  } else {
    const size_t qb = (size_t)c.Hl * L128 * 2;
    const void *q_in = nullptr, *kv_in = nullptr;
    A2D_TRY(a2a(c, q, c.q_recv, qb, s, 0, &q_in));
    A2D_TRY(a2a(c, c.kv_send, c.kv_recv, (size_t)2 * c.Hkl * L128 * 2, s, qb * c.d_hp, &kv_in));
    A2D_TRY(a2d_permute_blocks(q_in, sv.qh, c.d_hp, c.Hl, (int64_t)L128 * 2, s));
    A2D_TRY(a2d_permute_blocks(kv_in, sv.kvh, c.d_hp, 2 * c.Hkl, (int64_t)L128 * 2, s));
  }
  A2D_TRY(ring_forward(c, sv, s));
  return gather_bf16(c, sv.out_h, c.Hl, static_cast<uint16_t*>(out), s, c.x_in);
}

int backward(Ctx& c, const void* saved, const void* dout, void* dq, void* dk, void* dv, cudaStream_t s) {
  const size_t L128 = (size_t)c.L * 128;
  const Saved sv = saved_view(c, saved);
  const uint16_t* dO = static_cast<const uint16_t*>(dout);
  if (c.d_hp > 1) {
    const void* d_in = nullptr;
    A2D_TRY(a2a(c, dout, c.q_recv, (size_t)c.Hl * L128 * 2, s, 0, &d_in));
    A2D_TRY(a2d_permute_blocks(d_in, c.doh, c.d_hp, c.Hl, (int64_t)L128 * 2, s));
    dO = c.doh;
  }
  A2D_TRY(a2d_bwd_preprocess(sv.out_h, dO, sv.lse, c.Hl, c.C, 128, c.lse2, c.delta, s));
  CUDA_TRY(cudaMemsetAsync(c.dq_acc, 0, (size_t)c.Hl * 128 * c.C_pad * 4, s));
  const void* home = nullptr;
  bool home_bf16 = false;
  A2D_TRY(ring_backward(c, sv, dO, s, &home, &home_bf16));
  // dQ: transposed accumulator -> bf16 peer-major pack -> all-to-all into the caller's dq
  if (c.d_hp == 1) {
    A2D_TRY(a2d_dqt_to_bf16(c.dq_acc, dq, c.Hl, c.C, c.C_pad, 1, s));
  } else {
    A2D_TRY(a2d_dqt_to_bf16(c.dq_acc, c.g_send, c.Hl, c.C, c.C_pad, c.d_hp, s));
    A2D_TRY(a2a_to(c, c.g_send, dq, (size_t)c.Hl * L128 * 2, s, c.x_in));
  }
  const size_t half = (size_t)c.Hkl * c.C * 128;
  void* outs[2] = {dk, dv};
  // OUT-region offsets: dq at 0, then dk, dv (bf16 chunks, or fp32 for GQA replicas)
  const size_t q_out = (size_t)c.d_hp * c.Hl * L128 * 2;
  const size_t k_out = (size_t)c.d_hp * c.Hkl * L128 * (c.rep == 1 ? 2 : 4);
  for (int t = 0; t < 2; ++t) {
    const size_t off = c.x_in + q_out + t * k_out;
    if (c.rep == 1) {
      if (home_bf16) {
        A2D_TRY(gather_bf16(c, static_cast<const uint16_t*>(home) + t * half, c.Hkl, static_cast<uint16_t*>(outs[t]), s,
                            off));
      } else {
        A2D_TRY(gather_f32_to_bf16(c, static_cast<const float*>(home) + t * half, c.Hkl,
                                   static_cast<uint16_t*>(outs[t]), s, off));
      }
    } else {  // GQA replicas: gather fp32, sum the copies, round once
      const float* src = static_cast<const float*>(home) + t * half;
      const void* g_in = nullptr;
      A2D_TRY(a2d_permute_blocks(src, c.g32_send, c.Hkl, c.d_hp, (int64_t)L128 * 4, s));
      A2D_TRY(a2a(c, c.g32_send, c.g32_recv, (size_t)c.Hkl * L128 * 4, s, off, &g_in));
      A2D_TRY(a2d_sum_replicas_f32(static_cast<const float*>(g_in), c.g32_sum, c.Hkv, c.rep, (int64_t)L128, s));
      A2D_TRY(a2d_f32_to_bf16(c.g32_sum, outs[t], (int64_t)c.Hkv * L128, s));
    }
  }
  return A2D_OK;
}

// Wait for `stream` while polling every communicator for an asynchronous NCCL
// error; on an error or after timeout_ms, abort the communicators (so no rank
// hangs forever on a dead peer) and report.
int sync_checked(Ctx& c, cudaStream_t s, int64_t timeout_ms) {
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return A2D_OK;
    if (q != cudaErrorNotReady) return set_error(A2D_ECUDA, std::string("a2d_sync: ") + cudaGetErrorString(q));
    for (ncclComm_t m : {c.world_comm, c.hp_comm, c.c_inner, c.c_outer, c.c_dkv}) {
      if (!m) continue;
      ncclResult_t r = ncclSuccess;
      if (ncclCommGetAsyncError(m, &r) != ncclSuccess || (r != ncclSuccess && r != ncclInProgress)) {
        abort_comms(c);
        return set_error(A2D_ECUDA, std::string("a2d_sync: NCCL asynchronous error: ") + ncclGetErrorString(r) +
                                        " (communicators aborted)");
      }
    }
    const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms >= 0 && ms > timeout_ms) {
      abort_comms(c);
      return set_error(A2D_ETIMEOUT, "a2d_sync: timed out after " + std::to_string(ms) +
                                         " ms (communicators aborted; the context is no longer usable)");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

}  // namespace

extern "C" {

int a2d_nccl_unique_id(void* out, int64_t out_bytes) {
  if (out_bytes < (int64_t)sizeof(ncclUniqueId)) return set_error(A2D_EINVAL, "a2d_nccl_unique_id: buffer too small");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return A2D_OK;
}

int a2d_ctx_create(const void* nccl_id, int32_t rank, int32_t world, int32_t d_hp, int32_t d_cp, int32_t w,
                   int32_t placement, int32_t H, int32_t H_kv, int32_t d, int64_t S, int32_t causal, void** ctx) {
  Ctx* c = nullptr;
  const int rc = create(nccl_id, rank, world, d_hp, d_cp, w, placement, H, H_kv, d, S, causal, &c);
  if (rc) {
    const std::string msg = a2d_last_error();
    destroy(c);
    *ctx = nullptr;
    return set_error(rc, msg);
  }
  *ctx = c;
  return A2D_OK;
}

int a2d_saved_bytes(void* ctx, int64_t* bytes) {
  if (!ctx || !bytes) return set_error(A2D_EINVAL, "a2d_saved_bytes: null argument");
  *bytes = (int64_t)static_cast<Ctx*>(ctx)->saved_bytes;
  return A2D_OK;
}

int a2d_fwd(void* ctx, const void* q, const void* k, const void* v, void* out, void* saved, void* stream) {
  if (!ctx) return set_error(A2D_EINVAL, "a2d_fwd: null context");
  if (!saved || (reinterpret_cast<uintptr_t>(saved) & 255))
    return set_error(A2D_EINVAL, "a2d_fwd: saved must be a 256-byte aligned buffer of a2d_saved_bytes() bytes");
  Ctx& c = *static_cast<Ctx*>(ctx);
  if (!c.world_comm) return set_error(A2D_EINVAL, "a2d_fwd: context was aborted");
  return forward(c, q, k, v, out, saved, static_cast<cudaStream_t>(stream));
}

int a2d_bwd(void* ctx, const void* saved, const void* dout, void* dq, void* dk, void* dv, void* stream) {
  if (!ctx) return set_error(A2D_EINVAL, "a2d_bwd: null context");
  if (!saved || (reinterpret_cast<uintptr_t>(saved) & 255))
    return set_error(A2D_EINVAL, "a2d_bwd: saved must be the buffer a2d_fwd filled");
  Ctx& c = *static_cast<Ctx*>(ctx);
  if (!c.world_comm) return set_error(A2D_EINVAL, "a2d_bwd: context was aborted");
  return backward(c, saved, dout, dq, dk, dv, static_cast<cudaStream_t>(stream));
}

int a2d_ctx_timing(void* ctx, int32_t enabled) {
  if (!ctx) return set_error(A2D_EINVAL, "a2d_ctx_timing: null context");
  Ctx& c = *static_cast<Ctx*>(ctx);
  c.timing = enabled != 0;
  c.tused[0] = c.tused[1] = 0;
  return A2D_OK;
}

int a2d_ctx_kernel_ms(void* ctx, float* fwd_ms, float* bwd_ms, int64_t* n_fwd, int64_t* n_bwd) {
  if (!ctx || !fwd_ms || !bwd_ms || !n_fwd || !n_bwd) return set_error(A2D_EINVAL, "a2d_ctx_kernel_ms: null argument");
  Ctx& c = *static_cast<Ctx*>(ctx);
  CUDA_TRY(cudaDeviceSynchronize());
  float* outs[2] = {fwd_ms, bwd_ms};
  int64_t* ns[2] = {n_fwd, n_bwd};
  for (int w = 0; w < 2; ++w) {
    float tot = 0.f;
    for (size_t i = 0; i + 1 < c.tused[w]; i += 2) {
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, c.tev[w][i], c.tev[w][i + 1]));
      tot += ms;
    }
    *outs[w] = tot;
    *ns[w] = (int64_t)(c.tused[w] / 2);
  }
  return A2D_OK;
}

int a2d_ctx_transport(void* ctx, int32_t* symm) {
  if (!ctx || !symm) return set_error(A2D_EINVAL, "a2d_ctx_transport: null argument");
  *symm = static_cast<Ctx*>(ctx)->symm ? 1 : 0;
  return A2D_OK;
}

int a2d_ctx_set_comm(void* ctx, int32_t enabled) {
  if (!ctx) return set_error(A2D_EINVAL, "a2d_ctx_set_comm: null context");
  static_cast<Ctx*>(ctx)->comm = enabled != 0;
  return A2D_OK;
}

int a2d_sync(void* ctx, void* stream, int64_t timeout_ms) {
  if (!ctx) return set_error(A2D_EINVAL, "a2d_sync: null context");
  return sync_checked(*static_cast<Ctx*>(ctx), static_cast<cudaStream_t>(stream), timeout_ms);
}

int a2d_ctx_destroy(void* ctx) { return destroy(static_cast<Ctx*>(ctx)); }

int a2d_ring_plan(int32_t d_cp, int32_t w, int32_t j, int32_t* steps_out, int32_t* peers_out) {
  if (d_cp < 1 || w < 1 || d_cp % w || j < 0 || j >= d_cp)
    return set_error(A2D_EINVAL, "a2d_ring_plan: need 0 <= j < d_cp and w | d_cp");
  std::vector<Step> steps;
  int peers[6];
  ring_plan(d_cp, w, j, &steps, peers);
  for (size_t i = 0; i < steps.size(); ++i) {
    steps_out[3 * i] = steps[i].source;
    steps_out[3 * i + 1] = steps[i].outer;
    steps_out[3 * i + 2] = steps[i].inner;
  }
  std::copy(peers, peers + 6, peers_out);
  return A2D_OK;
}

int a2d_zigzag_positions(int64_t S, int32_t d_cp, int32_t j, int32_t* out) {
  if (d_cp < 1 || S <= 0 || S % (2 * d_cp) || j < 0 || j >= d_cp)
    return set_error(A2D_EINVAL, "a2d_zigzag_positions: need S divisible by 2*d_cp and 0 <= j < d_cp");
  const std::vector<int32_t> p = cp_positions(S, d_cp, j);
  std::copy(p.begin(), p.end(), out);
  return A2D_OK;
}

}  // extern "C"
