// Internal launch interface shared by the CUDA translation units.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace a2d {

// Forward chunk attention (one ring step). Tensors are head-major [H][T][D].
struct FwdParams {
  CUtensorMap tm_q, tm_k, tm_v;  // bf16 [H|Hkv][T][D], box {64,128,1}, SW128
  const int* q_pos;              // [Tq] original token positions
  const int* k_pos;              // [Tk]
  const int2* q_bounds;          // [ceil(Tq/128)] (min,max) position per query tile
  const int2* k_bounds;          // [ceil(Tk/128)] per key tile
  int Tq, Tk, H, Hkv, G;
  int causal;
  float scale_log2;              // log2(e) / sqrt(d)
  int merge;                     // 0: write block result; 1: fold into (acc_o, lse)
  float* lse;                    // [H][Tq] natural-log LSE (in/out when merge)
  float* acc_o;                  // [H][Tq][D] fp32 normalised accumulator, nullable
  __nv_bfloat16* out;            // bf16 output, nullable
  int64_t out_stride_h, out_stride_t;
};

cudaError_t launch_fa_fwd(const FwdParams& p, int head_dim, cudaStream_t s);

// Backward chunk attention (one ring step). Uses the final (global) LSE and
// D = rowsum(dO * O) of the query chunk.
struct BwdParams {
  CUtensorMap tm_q, tm_k, tm_v, tm_do;  // box {64,64,1} for q/do, {64,128,1} for k/v
  CUtensorMap tm_dq;                    // fp32 dq_acc^T [H][D][Tq_pad], box {32 q,D d,1}, SW128
  CUtensorMap tm_dq8;                   // same tensor, box {8 q,32 d,1}, no swizzle (per-warp drain)
  float* dq;                            // the same dq_acc^T at this slice's first query (red drain)
  int dq_ld;                            // its row stride (Tq_pad)
  const int* q_pos;
  const int* k_pos;
  const int2* q_bounds;   // per 64-row query tile
  const int2* k_bounds;   // per 128-key tile
  const float* lse2;      // [H][stats_stride] LSE * log2(e) (+inf for dead rows / padding)
  const float* delta;     // [H][stats_stride] rowsum(dO*O)
  int stats_stride;       // row stride of lse2 / delta
  float* dk;              // [Hkv][Tk][D] fp32 output (or accumulated)
  float* dv;
  int accumulate_kv;      // 1: dk/dv += partial, 0: overwrite
  int Tq, Tk, H, Hkv, G;
  int causal;
  float scale;            // 1/sqrt(d)
  float scale_log2;
};

cudaError_t launch_fa_bwd(const BwdParams& p, int head_dim, cudaStream_t s);

// UMMA plumbing self-test (umma_selftest.cu).
struct SelftestParams {
  CUtensorMap tm_a, tm_b;    // [1][128][128] bf16
  const __nv_bfloat16* a;    // [m][k]
  const __nv_bfloat16* v;    // [k][n]
  const __nv_bfloat16* at;   // [k][m]
  float* c;                  // [4][128][128]
};
cudaError_t launch_umma_selftest(const SelftestParams& p, cudaStream_t s);

}  // namespace a2d
