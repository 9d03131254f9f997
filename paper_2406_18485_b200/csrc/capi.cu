// extern "C" boundary of libattn2d_sm100.so (declared in include/attn2d_sm100.h).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <atomic>
#include <mutex>
#include <string>

#include "../../include/attn2d_sm100.h"
#include "kernels.h"
#include "tmap.h"

namespace a2d {

// aux.cu
cudaError_t launch_tile_bounds(const int* pos, int T, int tile, int2* out, cudaStream_t s);
cudaError_t launch_bwd_preprocess(const __nv_bfloat16* o, const __nv_bfloat16* dout, int64_t o_sh, int64_t o_st,
                                  int64_t do_sh, int64_t do_st, const float* lse, int H, int Tq, int Tq_pad,
                                  int D, float* lse2, float* delta, cudaStream_t s);
cudaError_t launch_merge_f32(float* acc_o, float* acc_lse, const float* blk_o, const float* blk_lse, int64_t rows,
                             int D, cudaStream_t s);
cudaError_t launch_permute_blocks(const void* src, void* dst, int64_t A, int64_t B, int64_t blk_bytes, int n_sm,
                                  cudaStream_t s);
cudaError_t launch_gather_blocks(const void* src, void* dst, const int* map, const int* dmap, int64_t n,
                                 int64_t blk_bytes, int n_sm, cudaStream_t s);
cudaError_t launch_sum_replicas(const float* src, float* dst, int64_t heads, int rep, int64_t per_head, int n_sm,
                                cudaStream_t s);
cudaError_t launch_f32_to_bf16(const float* src, __nv_bfloat16* dst, int64_t n, int n_sm, cudaStream_t s);
cudaError_t launch_dqt_to_bf16(const float* src, __nv_bfloat16* dst, int H, int64_t T, int64_t T_pad, int A, int D,
                               cudaStream_t s);
cudaError_t launch_permute_f32_bf16(const float* src, __nv_bfloat16* dst, int64_t A, int64_t B, int64_t blk_elems,
                                    int n_sm, cudaStream_t s);
cudaError_t launch_add_f32(float* dst, const float* src, int64_t n, int n_sm, cudaStream_t s);
cudaError_t launch_copy_rows(const void* src, void* dst, int64_t n_t, int64_t n_h, int64_t s_st, int64_t s_sh,
                             int64_t d_st, int64_t d_sh, int64_t row_bytes, const int* smap, const int* dmap,
                             int n_sm, cudaStream_t s);
cudaError_t launch_gather_tokens(const void* src, void* dst, const int* idx, int64_t H, int64_t S_src, int64_t L,
                                 int64_t S_dst, int64_t row_bytes, int scatter, int n_sm, cudaStream_t s);

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};  // kernels launched through this library (a2d_launch_count)

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
static int cuda_status(cudaError_t e, const char* where, int launches = 1) {
  if (e == cudaSuccess) {
    g_launches.fetch_add(launches, std::memory_order_relaxed);
    return A2D_OK;
  }
  return fail(A2D_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tmap_bf16_3d(CUtensorMap* out, const void* base, uint64_t n0, uint64_t n1, uint64_t n2, uint64_t s1,
                      uint64_t s2, uint32_t box1) {
  auto enc = get_encode();
  if (!enc) return fail(A2D_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return fail(A2D_EINVAL, "tensor base not 16-byte aligned");
  cuuint64_t dims[3] = {n0, n1, n2};
  cuuint64_t strides[2] = {s1 * 2, s2 * 2};
  cuuint32_t box[3] = {64, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(A2D_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return A2D_OK;
}

// fp32 [n2][n1][n0] tensor map (row stride s1, plane stride s2 elements), box
// {box0, box1, 1}, SWIZZLE_128B (box0 = 32): the transposed dQ reduce target.
static int make_tmap_f32_3d(CUtensorMap* out, const void* base, uint64_t n0, uint64_t n1, uint64_t n2,
                            uint64_t s1, uint64_t s2, uint32_t box0, uint32_t box1, bool sw128 = true) {
  auto enc = get_encode();
  if (!enc) return fail(A2D_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return fail(A2D_EINVAL, "tensor base not 16-byte aligned");
  cuuint64_t dims[3] = {n0, n1, n2};
  cuuint64_t strides[2] = {s1 * 4, s2 * 4};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(A2D_ECUDA, "cuTensorMapEncodeTiled (f32) failed (" + std::to_string((int)r) + ")");
  return A2D_OK;
}

static int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// for runtime.cu: report through the same thread-local a2d_last_error()
int set_error(int code, const std::string& msg) { return fail(code, msg); }

}  // namespace a2d

using namespace a2d;

extern "C" {

const char* a2d_last_error(void) { return g_err.c_str(); }
int a2d_abi_version(void) { return 2; }
long long a2d_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int a2d_tile_bounds(const int32_t* pos, int64_t T, int32_t tile, int32_t* out_minmax, void* stream) {
  if (T < 0 || tile <= 0 || T > INT32_MAX) return fail(A2D_EINVAL, "a2d_tile_bounds: bad T/tile");
  return cuda_status(launch_tile_bounds(pos, (int)T, tile, reinterpret_cast<int2*>(out_minmax), S(stream)),
                     "a2d_tile_bounds");
}

int a2d_fa_fwd_chunk(const void* q, const void* k, const void* v, const int32_t* q_pos, const int32_t* k_pos,
                     const int32_t* q_bounds128, const int32_t* k_bounds128, int32_t H, int32_t H_kv, int64_t Tq,
                     int64_t Tk, int32_t D, int32_t causal, float scale, int32_t merge, float* lse, float* acc_o,
                     void* out_bf16, void* stream) {
  if (D != 64 && D != 128) return fail(A2D_EINVAL, "a2d_fa_fwd_chunk: head dim must be 64 or 128");
  if (H <= 0 || H_kv <= 0 || H % H_kv != 0)
    return fail(A2D_EINVAL, std::to_string(H) + " query heads not divisible by " + std::to_string(H_kv) + " kv heads");
  if (Tq < 0 || Tk < 0 || Tq > INT32_MAX / 2 || Tk > INT32_MAX / 2) return fail(A2D_EINVAL, "a2d_fa_fwd_chunk: bad T");
  if (!lse) return fail(A2D_EINVAL, "a2d_fa_fwd_chunk: lse is required");
  if (merge && !acc_o) return fail(A2D_EINVAL, "a2d_fa_fwd_chunk: merge needs acc_o");
  if (Tq == 0) return A2D_OK;
  FwdParams p{};
  int rc;
  if (Tk > 0) {
    if ((rc = make_tmap_bf16_3d(&p.tm_q, q, D, Tq, H, D, Tq * D, 128))) return rc;
    if ((rc = make_tmap_bf16_3d(&p.tm_k, k, D, Tk, H_kv, D, Tk * D, 128))) return rc;
    if ((rc = make_tmap_bf16_3d(&p.tm_v, v, D, Tk, H_kv, D, Tk * D, 128))) return rc;
  } else {
    // no keys: still well defined (every row empty); use q for the unused maps
    if ((rc = make_tmap_bf16_3d(&p.tm_q, q, D, Tq, H, D, Tq * D, 128))) return rc;
    p.tm_k = p.tm_q;
    p.tm_v = p.tm_q;
  }
  p.q_pos = q_pos;
  p.k_pos = k_pos;
  p.q_bounds = reinterpret_cast<const int2*>(q_bounds128);
  p.k_bounds = reinterpret_cast<const int2*>(k_bounds128);
  p.Tq = (int)Tq;
  p.Tk = (int)Tk;
  p.H = H;
  p.Hkv = H_kv;
  p.G = H / H_kv;
  p.causal = causal;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.merge = merge;
  p.lse = lse;
  p.acc_o = acc_o;
  p.out = static_cast<__nv_bfloat16*>(out_bf16);
  p.out_stride_h = Tq * D;
  p.out_stride_t = D;
  return cuda_status(launch_fa_fwd(p, D, S(stream)), "a2d_fa_fwd_chunk");
}

int a2d_bwd_preprocess(const void* o, const void* dout, const float* lse, int32_t H, int64_t Tq, int32_t D,
                       float* lse2, float* delta, void* stream) {
  if (D % 64 != 0 || H <= 0 || Tq < 0 || Tq > INT32_MAX / 2) return fail(A2D_EINVAL, "a2d_bwd_preprocess: bad shape");
  const int Tq_pad = (int)((Tq + 63) / 64 * 64);
  return cuda_status(launch_bwd_preprocess(static_cast<const __nv_bfloat16*>(o),
                                           static_cast<const __nv_bfloat16*>(dout), Tq * D, D, Tq * D, D, lse, H,
                                           (int)Tq, Tq_pad, D, lse2, delta, S(stream)),
                     "a2d_bwd_preprocess");
}

int a2d_fa_bwd_chunk(const void* q, const void* k, const void* v, const void* dout, const int32_t* q_pos,
                     const int32_t* k_pos, const int32_t* q_bounds64, const int32_t* k_bounds128, const float* lse2,
                     const float* delta, float* dq_acc, float* dk, float* dv, int32_t accumulate_kv, int32_t H,
                     int32_t H_kv, int64_t Tq, int64_t Tk, int32_t D, int32_t causal, float scale, void* stream) {
  if (D != 128 && D != 64) return fail(A2D_EINVAL, "a2d_fa_bwd_chunk: head dim must be 64 or 128 (zero-pad others)");
  if (H <= 0 || H_kv <= 0 || H % H_kv != 0)
    return fail(A2D_EINVAL, std::to_string(H) + " query heads not divisible by " + std::to_string(H_kv) + " kv heads");
  if (Tq < 0 || Tk < 0 || Tq > INT32_MAX / 2 || Tk > INT32_MAX / 2) return fail(A2D_EINVAL, "a2d_fa_bwd_chunk: bad T");
  if (Tk == 0) return A2D_OK;
  // One launch covers at most 2048 query tiles (128K rows: the kernel's
  // shared-memory live list); longer query chunks run as consecutive slices,
  // later slices accumulating into dk/dv.
  constexpr int64_t kSlice = 2048 * 64;
  const int tq_pad = (int)((Tq + 63) / 64 * 64);
  for (int64_t off = 0; off < (Tq > 0 ? Tq : 1); off += kSlice) {
    const int64_t len = Tq > 0 ? std::min(kSlice, Tq - off) : 0;
    BwdParams p{};
    int rc;
    if ((rc = make_tmap_bf16_3d(&p.tm_k, k, D, Tk, H_kv, D, Tk * D, 128))) return rc;
    if ((rc = make_tmap_bf16_3d(&p.tm_v, v, D, Tk, H_kv, D, Tk * D, 128))) return rc;
    if (len > 0) {
      const __nv_bfloat16* qb = static_cast<const __nv_bfloat16*>(q) + off * D;
      const __nv_bfloat16* db = static_cast<const __nv_bfloat16*>(dout) + off * D;
      if ((rc = make_tmap_bf16_3d(&p.tm_q, qb, D, len, H, D, Tq * D, 64))) return rc;
      if ((rc = make_tmap_bf16_3d(&p.tm_do, db, D, len, H, D, Tq * D, 64))) return rc;
      // dq_acc^T [H][D][tq_pad]: this slice starts at query `off`
      if ((rc = make_tmap_f32_3d(&p.tm_dq, dq_acc + off, len, D, H, tq_pad, (uint64_t)D * tq_pad, 32, D)))
        return rc;
      if ((rc = make_tmap_f32_3d(&p.tm_dq8, dq_acc + off, len, D, H, tq_pad, (uint64_t)D * tq_pad, 8, 32, false)))
        return rc;
    } else {
      p.tm_q = p.tm_k;
      p.tm_do = p.tm_k;
      p.tm_dq = p.tm_k;
      p.tm_dq8 = p.tm_k;
    }
    p.dq = len > 0 ? dq_acc + off : nullptr;
    p.dq_ld = tq_pad;
    p.q_pos = q_pos + off;
    p.k_pos = k_pos;
    p.q_bounds = reinterpret_cast<const int2*>(q_bounds64) + off / 64;
    p.k_bounds = reinterpret_cast<const int2*>(k_bounds128);
    p.lse2 = lse2 + off;
    p.delta = delta + off;
    p.stats_stride = tq_pad;
    p.dk = dk;
    p.dv = dv;
    p.accumulate_kv = (accumulate_kv || off > 0) ? 1 : 0;
    p.Tq = (int)len;
    p.Tk = (int)Tk;
    p.H = H;
    p.Hkv = H_kv;
    p.G = H / H_kv;
    p.causal = causal;
    p.scale = scale;
    p.scale_log2 = scale * 1.4426950408889634f;
    if ((rc = cuda_status(launch_fa_bwd(p, D, S(stream)), "a2d_fa_bwd_chunk"))) return rc;
  }
  return A2D_OK;
}

int a2d_merge(float* acc_o, float* acc_lse, const float* blk_o, const float* blk_lse, int64_t rows, int32_t D,
              void* stream) {
  if (rows < 0 || D <= 0) return fail(A2D_EINVAL, "a2d_merge: bad shape");
  return cuda_status(launch_merge_f32(acc_o, acc_lse, blk_o, blk_lse, rows, D, S(stream)), "a2d_merge");
}

int a2d_permute_blocks(const void* src, void* dst, int64_t A, int64_t B, int64_t block_bytes, void* stream) {
  if (A < 0 || B < 0 || block_bytes % 16 != 0) return fail(A2D_EINVAL, "a2d_permute_blocks: block_bytes % 16 != 0");
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return fail(A2D_EINVAL, "a2d_permute_blocks: pointers must be 16-byte aligned");
  return cuda_status(launch_permute_blocks(src, dst, A, B, block_bytes, sm_count(), S(stream)), "a2d_permute_blocks");
}

int a2d_gather_blocks(const void* src, void* dst, const int32_t* map, const int32_t* dst_map, int64_t n,
                      int64_t block_bytes, void* stream) {
  if (n < 0 || block_bytes % 16 != 0) return fail(A2D_EINVAL, "a2d_gather_blocks: block_bytes % 16 != 0");
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return fail(A2D_EINVAL, "a2d_gather_blocks: pointers must be 16-byte aligned");
  return cuda_status(launch_gather_blocks(src, dst, map, dst_map, n, block_bytes, sm_count(), S(stream)),
                     "a2d_gather_blocks");
}

int a2d_copy_rows(const void* src, void* dst, int64_t n_t, int64_t n_h, int64_t src_st, int64_t src_sh,
                  int64_t dst_st, int64_t dst_sh, int64_t row_bytes, const int32_t* smap, const int32_t* dmap,
                  void* stream) {
  if (n_t < 0 || n_h < 0 || row_bytes <= 0 || row_bytes % 16)
    return fail(A2D_EINVAL, "a2d_copy_rows: row_bytes must be a positive multiple of 16");
  if ((src_st | src_sh | dst_st | dst_sh) % 16 || (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return fail(A2D_EINVAL, "a2d_copy_rows: pointers and strides must be 16-byte aligned");
  return cuda_status(launch_copy_rows(src, dst, n_t, n_h, src_st, src_sh, dst_st, dst_sh, row_bytes, smap, dmap,
                                      sm_count(), S(stream)),
                     "a2d_copy_rows");
}

int a2d_gather_tokens(const void* src, void* dst, const int32_t* idx, int64_t H, int64_t S_src, int64_t L,
                      int64_t S_dst, int64_t row_bytes, int32_t scatter, void* stream) {
  if (H < 0 || L < 0 || S_src < 0 || S_dst < 0 || row_bytes <= 0 || row_bytes % 16)
    return fail(A2D_EINVAL, "a2d_gather_tokens: row_bytes must be a positive multiple of 16");
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return fail(A2D_EINVAL, "a2d_gather_tokens: pointers must be 16-byte aligned");
  if (L > 0 && !idx) return fail(A2D_EINVAL, "a2d_gather_tokens: idx is required");
  return cuda_status(launch_gather_tokens(src, dst, idx, H, S_src, L, S_dst, row_bytes, scatter ? 1 : 0, sm_count(),
                                          S(stream)),
                     "a2d_gather_tokens");
}

int a2d_sum_replicas_f32(const float* src, float* dst, int64_t heads, int32_t rep, int64_t per_head, void* stream) {
  if (heads < 0 || rep <= 0 || per_head < 0) return fail(A2D_EINVAL, "a2d_sum_replicas_f32: bad shape");
  return cuda_status(launch_sum_replicas(src, dst, heads, rep, per_head, sm_count(), S(stream)),
                     "a2d_sum_replicas_f32");
}

int a2d_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream) {
  if (n < 0 || n % 4) return fail(A2D_EINVAL, "a2d_f32_to_bf16: n must be a multiple of 4");
  return cuda_status(launch_f32_to_bf16(src, static_cast<__nv_bfloat16*>(dst), n, sm_count(), S(stream)),
                     "a2d_f32_to_bf16");
}

int a2d_permute_f32_to_bf16(const float* src, void* dst, int64_t A, int64_t B, int64_t block_elems, void* stream) {
  if (A < 0 || B < 0 || block_elems % 8 != 0)
    return fail(A2D_EINVAL, "a2d_permute_f32_to_bf16: block_elems must be a multiple of 8");
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return fail(A2D_EINVAL, "a2d_permute_f32_to_bf16: pointers must be 16-byte aligned");
  return cuda_status(launch_permute_f32_bf16(src, static_cast<__nv_bfloat16*>(dst), A, B, block_elems, sm_count(),
                                             S(stream)),
                     "a2d_permute_f32_to_bf16");
}

int a2d_dqt_to_bf16(const float* src, void* dst, int32_t H, int64_t T, int64_t T_pad, int32_t A, void* stream) {
  return a2d_dqt_to_bf16_d(src, dst, H, T, T_pad, A, 128, stream);
}

int a2d_dqt_to_bf16_d(const float* src, void* dst, int32_t H, int64_t T, int64_t T_pad, int32_t A, int32_t D,
                      void* stream) {
  if (H < 0 || T < 0 || T_pad < T || A <= 0 || T % A || T_pad % 4)
    return fail(A2D_EINVAL, "a2d_dqt_to_bf16: need T_pad >= T, T_pad % 4 == 0 and T divisible by A");
  if (D != 64 && D != 128) return fail(A2D_EINVAL, "a2d_dqt_to_bf16: head dim must be 64 or 128");
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return fail(A2D_EINVAL, "a2d_dqt_to_bf16: pointers must be 16-byte aligned");
  return cuda_status(launch_dqt_to_bf16(src, static_cast<__nv_bfloat16*>(dst), H, T, T_pad, A, D, S(stream)),
                     "a2d_dqt_to_bf16");
}

int a2d_add_f32(float* dst, const float* src, int64_t n, void* stream) {
  if (n < 0 || n % 4) return fail(A2D_EINVAL, "a2d_add_f32: n must be a multiple of 4");
  return cuda_status(launch_add_f32(dst, src, n, sm_count(), S(stream)), "a2d_add_f32");
}

int a2d_selftest_umma(const void* a, const void* b, const void* v, const void* at, float* c, void* stream) {
  SelftestParams p{};
  int rc;
  if ((rc = make_tmap_bf16_3d(&p.tm_a, a, 128, 128, 1, 128, 128 * 128, 128))) return rc;
  if ((rc = make_tmap_bf16_3d(&p.tm_b, b, 128, 128, 1, 128, 128 * 128, 128))) return rc;
  p.a = static_cast<const __nv_bfloat16*>(a);
  p.v = static_cast<const __nv_bfloat16*>(v);
  p.at = static_cast<const __nv_bfloat16*>(at);
  p.c = c;
  return cuda_status(launch_umma_selftest(p, S(stream)), "a2d_selftest_umma");
}

}  // extern "C"
