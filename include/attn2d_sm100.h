/*
 * attn2d_sm100 — C ABI of the B200 (sm_100a) 2D-Attention hot path.
 *
 * Drop-in boundary for the reference operator API of
 * /root/reference/pkg/src/attn2d (a Python package; its "FFI" is a Python
 * call, so the binding a maintainer adds is a ctypes shim — INTEGRATION.md).
 * Each entry point below names the reference function it replaces.
 *
 * Conventions
 *  - All tensor arguments are DEVICE pointers; shapes/sizes are plain ints.
 *  - bf16 tensors are head-major and contiguous: q/out [H][T][D],
 *    k/v [H_kv][T][D] (the reference's DenseTensor.values layout, oracle.py:15-34).
 *  - Positions are int32 original token indices, one per token (DenseTensor.positions).
 *  - LSE is the natural-log log-sum-exp (oracle.py:53-66), fp32 [H][T].
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Calls are
 *    stream-ordered and never synchronise the host.
 *  - Return 0 on success; non-zero on error with a message in
 *    a2d_last_error() (thread-local). Invalid shapes return A2D_EINVAL, the
 *    analogue of the reference's ValueError.
 */
#ifndef ATTN2D_SM100_H_
#define ATTN2D_SM100_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define A2D_OK 0
#define A2D_EINVAL 1
#define A2D_ECUDA 2
#define A2D_ETIMEOUT 3

/* Thread-local message of the last failing call. */
const char* a2d_last_error(void);
/* ABI version (bumped on any signature change). */
int a2d_abi_version(void);
/* Process-wide count of CUDA kernels this library has launched (every entry
 * point below, including those the native runtime calls internally). The
 * bench reads it around its timed region. */
long long a2d_launch_count(void);

/* Per-tile (min, max) of positions: out[2*t], out[2*t+1] for tile t of
 * `tile` tokens; empty tiles get (INT_MAX, INT_MIN). Input to the
 * attention entry points (tile = 128 for keys and forward queries, 64 for
 * backward queries). */
int a2d_tile_bounds(const int32_t* pos, int64_t T, int32_t tile, int32_t* out_minmax, void* stream);

/* One ring step forward: attention of a query chunk against one KV chunk.
 * Replaces ref attention_block (oracle.py:97-101) and, with merge=1, the
 * fold block_update(acc, blk) (oracle.py:111-124) of run_double_ring
 * (ring.py:64-79).
 *   merge=0: lse := blk.lse; acc_o (fp32, nullable) := blk.out;
 *            out_bf16 (nullable) := bf16(blk.out)
 *   merge=1: (acc_o, lse) := block_update((acc_o, lse), blk) in place;
 *            out_bf16 (nullable) := bf16(new acc_o)
 * D in {64, 128}; scale = 1/sqrt(d) of the caller's true head dim. GQA:
 * head h reads KV head h / (H/H_kv) (oracle.py:45-50). */
int a2d_fa_fwd_chunk(const void* q, const void* k, const void* v, const int32_t* q_pos, const int32_t* k_pos,
                     const int32_t* q_bounds128, const int32_t* k_bounds128, int32_t H, int32_t H_kv, int64_t Tq,
                     int64_t Tk, int32_t D, int32_t causal, float scale, int32_t merge, float* lse, float* acc_o,
                     void* out_bf16, void* stream);

/* Backward preprocess for a query chunk: delta[h][t] = sum_d dO*O (the
 * reference's `row`, oracle.py:145) and lse2 = lse*log2(e) (+inf for rows
 * with lse=-inf and for padding). Outputs are [H][Tq_pad], Tq_pad =
 * round_up(Tq, 64). */
int a2d_bwd_preprocess(const void* o, const void* dout, const float* lse, int32_t H, int64_t Tq, int32_t D,
                       float* lse2, float* delta, void* stream);

/* One ring step backward: gradients of the block (query chunk, KV chunk)
 * given the FINAL lse/delta of the query rows. Replaces the per-block part
 * of ref attention_backward (oracle.py:127-152):
 *   dq_acc (fp32, TRANSPOSED [H][D][Tq_pad], Tq_pad = round_up(Tq, 64),
 *          query contiguous) += (dS K / sqrt(d))^T     (L2-side reduce-add);
 *          a2d_dqt_to_bf16(_d) turns it into dQ
 *   dk, dv [H_kv][Tk][D] (fp32) (+)= partial (accumulate_kv selects +=)
 * D must be 64 or 128 (pad other head dims with zeros and pass the true scale). */
int a2d_fa_bwd_chunk(const void* q, const void* k, const void* v, const void* dout, const int32_t* q_pos,
                     const int32_t* k_pos, const int32_t* q_bounds64, const int32_t* k_bounds128, const float* lse2,
                     const float* delta, float* dq_acc, float* dk, float* dv, int32_t accumulate_kv, int32_t H,
                     int32_t H_kv, int64_t Tq, int64_t Tk, int32_t D, int32_t causal, float scale, void* stream);

/* Standalone block_update (oracle.py:111-124) on rows of D fp32 values. */
int a2d_merge(float* acc_o, float* acc_lse, const float* blk_o, const float* blk_lse, int64_t rows, int32_t D,
              void* stream);

/* dst[b][a][:] = src[a][b][:] for blocks of block_bytes (multiple of 16).
 * With A = d_hp peers and B = local heads it is the SeqAlltoAll
 * unpack/pack (ref seq_alltoall_scatter / gather, sharding.py:131-169). */
int a2d_permute_blocks(const void* src, void* dst, int64_t A, int64_t B, int64_t block_bytes, void* stream);

/* dst[dst_map ? dst_map[i] : i][:] = src[map[i]][:] for n blocks — the
 * SeqAlltoAll send-buffer pack with GQA KV replication done by addressing
 * (ref kv_replicate, sharding.py:109-128). Maps are device int32 arrays;
 * dst_map may be NULL. */
int a2d_gather_blocks(const void* src, void* dst, const int32_t* map, const int32_t* dst_map, int64_t n,
                      int64_t block_bytes, void* stream);

/* Strided row copy: for t < n_t, h < n_h, copy row_bytes (multiple of 16)
 * from src + t*src_st + smap(h)*src_sh to dst + t*dst_st + dmap(h)*dst_sh
 * (all strides in BYTES; smap/dmap device int32 maps, NULL = identity).
 * Token-major (L,H,d) <-> head-major (H,L,d) conversion fused with the
 * SeqAlltoAll pack/unpack, including strided views of a fused QKV
 * projection output — the data-loader side of ref shard_sequence
 * (sharding.py:56-79). */
int a2d_copy_rows(const void* src, void* dst, int64_t n_t, int64_t n_h, int64_t src_st, int64_t src_sh,
                  int64_t dst_st, int64_t dst_sh, int64_t row_bytes, const int32_t* smap, const int32_t* dmap,
                  void* stream);

/* Data-loader token gather of ref shard_sequence / unshard (sharding.py:56-106)
 * over all H heads: scatter = 0: dst[h][t] = src[h][idx[t]]; scatter = 1:
 * dst[h][idx[t]] = src[h][t]; t < L, rows of row_bytes (multiple of 16),
 * head strides S_src / S_dst rows. Bit-exact byte move. */
int a2d_gather_tokens(const void* src, void* dst, const int32_t* idx, int64_t H, int64_t S_src, int64_t L,
                      int64_t S_dst, int64_t row_bytes, int32_t scatter, void* stream);

/* dst[h] = sum_r src[h*rep + r] over per_head fp32 values (gradient of kv_replicate). */
int a2d_sum_replicas_f32(const float* src, float* dst, int64_t heads, int32_t rep, int64_t per_head, void* stream);

/* dst[b][a][:] = bf16(src[a][b][:]) for fp32 blocks of block_elems (multiple
 * of 8): the fp32 -> bf16 conversion of dQ / dK / dV fused with the pack of the
 * gradient all-to-all (ref seq_alltoall_gather, sharding.py:155-169). A = 1
 * or B = 1 is a plain conversion. */
int a2d_permute_f32_to_bf16(const float* src, void* dst, int64_t A, int64_t B, int64_t block_elems, void* stream);

/* dQ out of the transposed backward accumulator: dst[a][h][l][d] =
 * bf16(src[h][d][a*L + l]) with L = T/A; A = 1 gives [H][T][128], A = d_hp
 * gives the gradient all-to-all's peer-major pack (sharding.py:155-169). */
int a2d_dqt_to_bf16(const float* src, void* dst, int32_t H, int64_t T, int64_t T_pad, int32_t A, void* stream);
/* Same for a head dim D in {64, 128}: src [H][D][T_pad], dst [a][h][l][D]. */
int a2d_dqt_to_bf16_d(const float* src, void* dst, int32_t H, int64_t T, int64_t T_pad, int32_t A, int32_t D,
                      void* stream);

/* Elementwise helpers (n multiple of 4). */
int a2d_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream);
int a2d_add_f32(float* dst, const float* src, int64_t n, void* stream);

/* ---- Native SPMD runtime (SURVEY §8b "C-ABI to export"): the whole 2D
 * attention layer of one rank, NCCL inside the library. One process per GPU;
 * rank r of a world of d_hp*d_cp ranks, placement 0 = head-first
 * (rank = hp + d_hp*cp), 1 = context-first (rank = cp + d_cp*hp), as the
 * reference's RankGrid (config.py:155-163). Tensors are this rank's
 * SeqSharded chunks, head-major bf16 device arrays: q/out/dout/dq [H][L][d],
 * k/v/dk/dv [H_kv][L][d], L = S/(d_hp*d_cp), tokens in zig-zag order (ref
 * shard_sequence, sharding.py:56-79). Head dim 128.
 * Stateless contexts: a forward's state (HeadSharded Q, K/V chunk, output and
 * natural-log LSE — what the backward needs) is written into a CALLER-OWNED
 * `saved` buffer, so any number of layers / micro-batches can be in flight
 * (the reference operator is a pure function, ring.py:82-119). The context
 * owns only workspaces, reused in stream order: calls on one context must be
 * issued on one stream (or ordered by the caller). */
/* Rank 0 creates the NCCL id (128 bytes) and shares it with the other ranks. */
int a2d_nccl_unique_id(void* out, int64_t out_bytes);
/* Collective over all `world` ranks: communicators (HP all-to-all group; inner,
 * outer and dK/dV ring groups), ring schedule (ring.py:41-61), positions,
 * buffers. Replaces run_2d_attention's setup (ring.py:82-107). */
int a2d_ctx_create(const void* nccl_id, int32_t rank, int32_t world, int32_t d_hp, int32_t d_cp, int32_t w,
                   int32_t placement, int32_t H, int32_t H_kv, int32_t d, int64_t S, int32_t causal, void** ctx);
/* Size of the saved-state buffer one a2d_fwd fills for its a2d_bwd. Layout
 * (256-byte aligned regions, C = S/d_cp, Hl = H/d_hp, Hkl = replicated KV
 * heads/d_hp): Q [Hl][C][128] bf16 | K,V [2][Hkl][C][128] bf16 |
 * out [Hl][C][128] bf16 | LSE [Hl][C] fp32 (natural log, ref oracle.py:94). */
int a2d_saved_bytes(void* ctx, int64_t* bytes);
/* Forward of the layer (ref run_2d_attention, ring.py:82-119): out = this
 * rank's SeqSharded output; `saved` (256-byte aligned, a2d_saved_bytes) gets
 * this call's state. Collective; stream-ordered on `stream`. */
int a2d_fwd(void* ctx, const void* q, const void* k, const void* v, void* out, void* saved, void* stream);
/* Backward of the a2d_fwd that filled `saved`: dq, dk, dv SeqSharded bf16.
 * Collective. `saved` is only read. */
int a2d_bwd(void* ctx, const void* saved, const void* dout, void* dq, void* dk, void* dv, void* stream);
/* Wait for `stream` while polling every communicator of the context with
 * ncclCommGetAsyncError. On an NCCL error, or after timeout_ms (< 0: none),
 * abort the communicators (ncclCommAbort: no rank hangs on a dead peer) and
 * return A2D_ECUDA / A2D_ETIMEOUT; the context then refuses further calls
 * and only a2d_ctx_destroy is valid. */
int a2d_sync(void* ctx, void* stream, int64_t timeout_ms);
/* Measurement only: enabled = 0 skips every NCCL call of the context (same
 * kernels and buffers; receive buffers keep stale data), so a layer timed
 * that way minus the normal layer is the exposed communication
 * (ref timeline.py:152's definition). Results are garbage while disabled. */
int a2d_ctx_set_comm(void* ctx, int32_t enabled);
/* Head-parallel exchange transport the context chose at creation: 1 = copy
 * engines into CUDA-IPC-mapped peer buffers plus an NCCL barrier (default when
 * every HP peer could map the others), 0 = NCCL send/recv (A2D_TRANSPORT=nccl,
 * or any rank failed to map). Ring hops always use NCCL. */
int a2d_ctx_transport(void* ctx, int32_t* symm);
/* Measurement: enabled = 1 brackets every attention-kernel launch of the
 * context with CUDA events on its stream (and resets the record);
 * a2d_ctx_kernel_ms synchronises and returns the summed forward / backward
 * kernel milliseconds and launch counts since then. */
int a2d_ctx_timing(void* ctx, int32_t enabled);
int a2d_ctx_kernel_ms(void* ctx, float* fwd_ms, float* bwd_ms, int64_t* n_fwd, int64_t* n_bwd);
int a2d_ctx_destroy(void* ctx);
/* Host-side plan of the native runtime, exposed for tests and other hosts:
 * CP rank j's ring schedule as (source, outer step, inner step) triples
 * (d_cp of them, ref build_ring_schedule ring.py:41-61) and its peers
 * (inner_to, inner_from, outer_to, outer_from, diag_to, diag_from); and the
 * zig-zag token positions of CP chunk j (ref zigzag_reorder sharding.py:33-53).
 * No GPU needed. */
int a2d_ring_plan(int32_t d_cp, int32_t w, int32_t j, int32_t* steps_out, int32_t* peers_out);
int a2d_zigzag_positions(int64_t S, int32_t d_cp, int32_t j, int32_t* out);

/* UMMA plumbing self-test (one CTA, 128x128x128 bf16 GEMMs in four operand
 * layouts); c is fp32 [4][128][128]. Used by the parity tests. */
int a2d_selftest_umma(const void* a, const void* b, const void* v, const void* at, float* c, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ATTN2D_SM100_H_ */
