// HBM-bound helper kernels around the attention GEMMs.
//
//  * tile_bounds     : per-tile (min,max) of the carried token positions; the
//                      attention kernels classify tiles (skip / full / masked)
//                      from these, so zig-zag chunks need no special casing.
//  * bwd_preprocess  : delta = rowsum(dO * O) (the reference's `row`,
//                      oracle.py:145) and lse2 = LSE*log2(e) (+inf for dead
//                      rows and tail padding, so P = 0 there).
//  * merge           : standalone block_update (oracle.py:111-124), K2.
//  * permute_blocks  : [A][B][blk] -> [B][A][blk] byte copy with 128-bit
//                      accesses; the pack / unpack around the head-parallel
//                      all-to-all (sharding.py:131-169) are instances of it.
//  * gather_blocks   : dst[i] = src[map[i]] (GQA replication without
//                      materialising kv_replicate's copies, sharding.py:109-128).
//  * sum_replicas    : gradient of that replication (sum of the copies).
//  * cast kernels    : fp32 <-> bf16.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>
#include <cmath>

namespace a2d {

__global__ void tile_bounds_kernel(const int* __restrict__ pos, int T, int tile, int2* __restrict__ out) {
  const int t = blockIdx.x;
  int lo = INT_MAX, hi = INT_MIN;
  for (int i = t * tile + threadIdx.x; i < min(T, (t + 1) * tile); i += blockDim.x) {
    const int v = pos[i];
    lo = min(lo, v);
    hi = max(hi, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ int slo[32], shi[32];
  const int w = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0) { slo[w] = lo; shi[w] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x / 32); ++i) { lo = min(lo, slo[i]); hi = max(hi, shi[i]); }
    out[t] = make_int2(lo, hi);  // empty tile -> (INT_MAX, INT_MIN)
  }
}

cudaError_t launch_tile_bounds(const int* pos, int T, int tile, int2* out, cudaStream_t s) {
  const int n = (T + tile - 1) / tile;
  if (n == 0) return cudaSuccess;
  tile_bounds_kernel<<<n, 128, 0, s>>>(pos, T, tile, out);
  return cudaGetLastError();
}

// delta / lse2 per query row. D/8 lanes per row, one 128-bit load of dO and
// of O per lane (D = 128: 2 rows per warp, each warp load a 512-byte run);
// the row sum is a shuffle reduction inside the lane group.
template <int D>
__global__ void bwd_preprocess_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                      int64_t o_sh, int64_t o_st, int64_t do_sh, int64_t do_st,
                                      const float* __restrict__ lse, int H, int Tq, int Tq_pad,
                                      float* __restrict__ lse2, float* __restrict__ delta) {
  constexpr int kLanes = D / 8;  // lanes per row
  const int64_t rows = (int64_t)H * Tq_pad;
  const int sub = threadIdx.x % kLanes;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kLanes; row < rows;
       row += (int64_t)gridDim.x * blockDim.x / kLanes) {
    const int h = (int)(row / Tq_pad), t = (int)(row % Tq_pad);
    float acc = 0.f;
    if (t < Tq) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(o + h * o_sh + t * o_st) + sub);
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(dout + h * do_sh + t * do_st) + sub);
      const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 x = __bfloat1622float2(pa[i]), y = __bfloat1622float2(pb[i]);
        acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
      }
    }
#pragma unroll
    for (int off = kLanes / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (sub == 0) {
      float l2 = INFINITY;
      if (t < Tq) {
        const float l = lse[(size_t)h * Tq + t];
        l2 = l == -INFINITY ? INFINITY : l * 1.4426950408889634f;
      }
      lse2[row] = l2;
      delta[row] = t < Tq ? acc : 0.f;
    }
  }
}

cudaError_t launch_bwd_preprocess(const __nv_bfloat16* o, const __nv_bfloat16* dout, int64_t o_sh, int64_t o_st,
                                  int64_t do_sh, int64_t do_st, const float* lse, int H, int Tq, int Tq_pad,
                                  int D, float* lse2, float* delta, cudaStream_t s) {
  const int64_t rows = (int64_t)H * Tq_pad;
  if (rows == 0) return cudaSuccess;
  if ((o_st | do_st | o_sh | do_sh) % 8 || ((reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(dout)) & 15))
    return cudaErrorInvalidValue;
  const int threads = 256;
  const int lanes = D / 8;
  int64_t blocks = (rows * lanes + threads - 1) / threads;
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (blocks > (int64_t)n_sm * 16) blocks = (int64_t)n_sm * 16;
  if (D == 128) {
    bwd_preprocess_kernel<128><<<(unsigned)blocks, threads, 0, s>>>(o, dout, o_sh, o_st, do_sh, do_st, lse, H, Tq,
                                                                     Tq_pad, lse2, delta);
  } else if (D == 64) {
    bwd_preprocess_kernel<64><<<(unsigned)blocks, threads, 0, s>>>(o, dout, o_sh, o_st, do_sh, do_st, lse, H, Tq,
                                                                    Tq_pad, lse2, delta);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// acc := block_update(acc, blk) (oracle.py:111-124). acc_o / blk_o fp32
// [R][D], D % 4 == 0: one warp per row, 128-bit loads and stores (D = 128: one
// float4 per lane, 512 contiguous bytes per warp access).
__global__ void merge_kernel(float4* __restrict__ acc_o, float* __restrict__ acc_lse, const float4* __restrict__ blk_o,
                             const float* __restrict__ blk_lse, int64_t rows, int d4) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows; r += warps) {
    const float la = acc_lse[r], lb = blk_lse[r];
    const float m = fmaxf(la, lb);
    float wa = 0.f, wb = 0.f, ln = -INFINITY;
    if (m != -INFINITY) {
      const float ea = la == -INFINITY ? 0.f : expf(la - m);
      const float eb = lb == -INFINITY ? 0.f : expf(lb - m);
      const float z = ea + eb;
      ln = m + logf(z);
      wa = ea / z;
      wb = eb / z;
    }
    for (int c = lane; c < d4; c += 32) {
      const int64_t i = r * d4 + c;
      const float4 a = acc_o[i], b = __ldg(blk_o + i);
      acc_o[i] = make_float4(a.x * wa + b.x * wb, a.y * wa + b.y * wb, a.z * wa + b.z * wb, a.w * wa + b.w * wb);
    }
    __syncwarp();  // every lane has read acc_lse[r]
    if (lane == 0) acc_lse[r] = ln;
  }
}

// any D / alignment (small head dims through the reference-shaped API)
__global__ void merge_scalar_kernel(float* __restrict__ acc_o, float* __restrict__ acc_lse,
                                    const float* __restrict__ blk_o, const float* __restrict__ blk_lse, int64_t rows,
                                    int D) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float la = acc_lse[r], lb = blk_lse[r];
  const float m = fmaxf(la, lb);
  float wa = 0.f, wb = 0.f, ln = -INFINITY;
  if (m != -INFINITY) {
    const float ea = la == -INFINITY ? 0.f : expf(la - m);
    const float eb = lb == -INFINITY ? 0.f : expf(lb - m);
    const float z = ea + eb;
    ln = m + logf(z);
    wa = ea / z;
    wb = eb / z;
  }
  for (int c = lane; c < D; c += 32) acc_o[r * D + c] = acc_o[r * D + c] * wa + blk_o[r * D + c] * wb;
  __syncwarp();
  if (lane == 0) acc_lse[r] = ln;
}

cudaError_t launch_merge_f32(float* acc_o, float* acc_lse, const float* blk_o, const float* blk_lse, int64_t rows,
                             int D, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  if (D % 4 || ((reinterpret_cast<uintptr_t>(acc_o) | reinterpret_cast<uintptr_t>(blk_o)) & 15)) {
    merge_scalar_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(acc_o, acc_lse, blk_o, blk_lse, rows, D);
    return cudaGetLastError();
  }
  int64_t blocks = (rows + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  merge_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<float4*>(acc_o), acc_lse,
                                                reinterpret_cast<const float4*>(blk_o), blk_lse, rows, D / 4);
  return cudaGetLastError();
}

__global__ void permute_blocks_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t A, int64_t B,
                                      int64_t blk_vec) {
  const int64_t total = A * B * blk_vec;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i % blk_vec;
    const int64_t ab = i / blk_vec;  // destination block index = b*A + a
    const int64_t b = ab / A, a = ab % A;
    dst[i] = __ldg(src + (a * B + b) * blk_vec + e);
  }
}

// dst[b][a][:] = src[a][b][:], blocks of blk_bytes (multiple of 16).
cudaError_t launch_permute_blocks(const void* src, void* dst, int64_t A, int64_t B, int64_t blk_bytes, int n_sm,
                                  cudaStream_t s) {
  if (blk_bytes % 16 != 0) return cudaErrorInvalidValue;
  const int64_t total = A * B * (blk_bytes / 16);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = (int64_t)n_sm * 8;
  if (blocks > cap) blocks = cap;
  permute_blocks_kernel<<<(unsigned)blocks, 256, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), A,
                                                         B, blk_bytes / 16);
  return cudaGetLastError();
}

// dst[b][a][:] = bf16(src[a][b][:]) over blocks of blk8*8 fp32 values: the
// fp32 -> bf16 conversion fused into the all-to-all pack of the gradient
// gather (one HBM pass instead of convert + permute).
__global__ void permute_f32_bf16_kernel(const float4* __restrict__ src, uint4* __restrict__ dst, int64_t A, int64_t B,
                                        int64_t blk8) {
  const int64_t total = A * B * blk8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i % blk8;
    const int64_t ab = i / blk8;
    const int64_t b = ab / A, a = ab % A;
    const float4* s2 = src + ((a * B + b) * blk8 + e) * 2;
    const float4 x = __ldg(s2), y = __ldg(s2 + 1);
    __nv_bfloat162 p0 = __floats2bfloat162_rn(x.x, x.y), p1 = __floats2bfloat162_rn(x.z, x.w);
    __nv_bfloat162 p2 = __floats2bfloat162_rn(y.x, y.y), p3 = __floats2bfloat162_rn(y.z, y.w);
    dst[i] = make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                        *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
  }
}

cudaError_t launch_permute_f32_bf16(const float* src, __nv_bfloat16* dst, int64_t A, int64_t B, int64_t blk_elems,
                                    int n_sm, cudaStream_t s) {
  if (blk_elems % 8 != 0) return cudaErrorInvalidValue;
  const int64_t total = A * B * (blk_elems / 8);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = (int64_t)n_sm * 8;
  if (blocks > cap) blocks = cap;
  permute_f32_bf16_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(src),
                                                           reinterpret_cast<uint4*>(dst), A, B, blk_elems / 8);
  return cudaGetLastError();
}

// dQ out of the backward's transposed accumulator: dst[a][h][l][d] =
// bf16(src[h][d][a*L + l]), L = T/A (A = d_hp: the gradient all-to-all's pack;
// A = 1: plain [h][t][d]). A block owns 128 tokens x all D features of one
// head: warp w reads features 8w..8w+7 as float4 runs along the tokens (each
// warp load = 512 contiguous bytes), rounds the 8x4 register block to bf16
// and parks it in shared memory as [token][16-byte feature chunk] (chunk index
// XOR-swizzled by token/4: conflict-free both ways); then every warp store
// writes whole token rows (D*2 bytes each), so the output lines are complete
// when they leave the SM (r02: 6.8 TB/s vs 4.1 TB/s for 16-byte scattered
// stores, tools/probes/hbm_probe.cu).
template <int D>
__global__ void __launch_bounds__(D * 4) dqt_to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                                            int H, int64_t T, int64_t T_pad, int64_t L) {
  constexpr int kChunks = D / 8;  // 16-byte chunks per token row
  __shared__ __align__(16) uint4 tile[128][kChunks];
  const int h = blockIdx.y;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t t0 = (int64_t)blockIdx.x * 128;
  const int64_t t = t0 + 4 * lane;
  if (t < T_pad) {  // T_pad % 4 == 0: the float4 stays inside the row
    const float* s = src + ((size_t)h * D + 8 * w) * T_pad + t;
    float4 r[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = __ldcs(reinterpret_cast<const float4*>(s + (size_t)i * T_pad));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = j == 0 ? r[i].x : j == 1 ? r[i].y : j == 2 ? r[i].z : r[i].w;
      __nv_bfloat162 p0 = __floats2bfloat162_rn(v[0], v[1]), p1 = __floats2bfloat162_rn(v[2], v[3]);
      __nv_bfloat162 p2 = __floats2bfloat162_rn(v[4], v[5]), p3 = __floats2bfloat162_rn(v[6], v[7]);
      tile[4 * lane + j][w ^ (lane % kChunks)] =
          make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                     *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < 128 * kChunks; idx += blockDim.x) {
    const int row = idx / kChunks, c = idx % kChunks;
    const int64_t tok = t0 + row;
    if (tok >= T) continue;
    const int64_t a = tok / L, l = tok % L;
    *reinterpret_cast<uint4*>(dst + (((size_t)a * H + h) * L + l) * D + 8 * c) = tile[row][c ^ ((row >> 2) % kChunks)];
  }
}

cudaError_t launch_dqt_to_bf16(const float* src, __nv_bfloat16* dst, int H, int64_t T, int64_t T_pad, int A, int D,
                               cudaStream_t s) {
  if (H == 0 || T == 0) return cudaSuccess;
  if (T_pad % 4 || ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15))
    return cudaErrorInvalidValue;
  dim3 grid((unsigned)((T + 127) / 128), H);
  if (D == 128)
    dqt_to_bf16_kernel<128><<<grid, 512, 0, s>>>(src, dst, H, T, T_pad, T / A);
  else if (D == 64)
    dqt_to_bf16_kernel<64><<<grid, 256, 0, s>>>(src, dst, H, T, T_pad, T / A);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

__global__ void gather_blocks_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                     const int* __restrict__ map, const int* __restrict__ dmap, int64_t n,
                                     int64_t blk_vec) {
  const int64_t total = n * blk_vec;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = i / blk_vec, e = i % blk_vec;
    const int64_t d = dmap ? (int64_t)dmap[blk] : blk;
    dst[d * blk_vec + e] = __ldg(src + (int64_t)map[blk] * blk_vec + e);
  }
}

// dst[dmap ? dmap[i] : i] = src[map[i]] for n blocks.
cudaError_t launch_gather_blocks(const void* src, void* dst, const int* map, const int* dmap, int64_t n,
                                 int64_t blk_bytes, int n_sm, cudaStream_t s) {
  if (blk_bytes % 16 != 0) return cudaErrorInvalidValue;
  const int64_t total = n * (blk_bytes / 16);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)n_sm * 8) blocks = (int64_t)n_sm * 8;
  gather_blocks_kernel<<<(unsigned)blocks, 256, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), map,
                                                        dmap, n, blk_bytes / 16);
  return cudaGetLastError();
}

// dst[h][e] = sum_r src[h*rep + r][e]   (fp32)
__global__ void sum_replicas_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t heads, int rep,
                                    int64_t per_head) {
  const int64_t total = heads * per_head;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = i / per_head, e = i % per_head;
    float acc = 0.f;
    for (int r = 0; r < rep; ++r) acc += src[(h * rep + r) * per_head + e];
    dst[i] = acc;
  }
}

cudaError_t launch_sum_replicas(const float* src, float* dst, int64_t heads, int rep, int64_t per_head, int n_sm,
                                cudaStream_t s) {
  const int64_t total = heads * per_head;
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)n_sm * 8) blocks = (int64_t)n_sm * 8;
  sum_replicas_kernel<<<(unsigned)blocks, 256, 0, s>>>(src, dst, heads, rep, per_head);
  return cudaGetLastError();
}

__global__ void f32_to_bf16_kernel(const float4* __restrict__ src, uint2* __restrict__ dst, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    dst[i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}

cudaError_t launch_f32_to_bf16(const float* src, __nv_bfloat16* dst, int64_t n, int n_sm, cudaStream_t s) {
  if (n % 4 != 0) return cudaErrorInvalidValue;
  const int64_t n4 = n / 4;
  if (n4 == 0) return cudaSuccess;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks > (int64_t)n_sm * 8) blocks = (int64_t)n_sm * 8;
  f32_to_bf16_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(src),
                                                      reinterpret_cast<uint2*>(dst), n4);
  return cudaGetLastError();
}

// dst (fp32) += src (fp32): the dK/dV accumulate-and-forward step (K4).
__global__ void add_f32_kernel(float4* __restrict__ dst, const float4* __restrict__ src, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = dst[i];
    const float4 b = src[i];
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    dst[i] = a;
  }
}

cudaError_t launch_add_f32(float* dst, const float* src, int64_t n, int n_sm, cudaStream_t s) {
  if (n % 4 != 0) return cudaErrorInvalidValue;
  const int64_t n4 = n / 4;
  if (n4 == 0) return cudaSuccess;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks > (int64_t)n_sm * 8) blocks = (int64_t)n_sm * 8;
  add_f32_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<float4*>(dst), reinterpret_cast<const float4*>(src),
                                                  n4);
  return cudaGetLastError();
}

}  // namespace a2d

namespace a2d {

// dst(t, h) = src(t, smap(h)) for rows of row_vec x 16 bytes, arbitrary
// (t, h) strides in bytes on both sides (dst head slot dmap(h) if given).
// Token-major (L, H, d) <-> head-major (H, L, d) conversions, the fused
// QKV-projection views and the GQA head map are all instances; the layout
// change rides on the all-to-all pack instead of costing its own pass.
__global__ void copy_rows_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t n_t, int64_t n_h,
                                 int64_t s_st, int64_t s_sh, int64_t d_st, int64_t d_sh, int64_t row_vec,
                                 const int* __restrict__ smap, const int* __restrict__ dmap) {
  const int64_t total = n_t * n_h * row_vec;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i % row_vec;
    const int64_t row = i / row_vec;
    const int64_t h = row % n_h, t = row / n_h;
    const int64_t hs = smap ? smap[h] : h, hd = dmap ? dmap[h] : h;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + t * s_st + hs * s_sh) + e);
    reinterpret_cast<uint4*>(dst + t * d_st + hd * d_sh)[e] = v;
  }
}

cudaError_t launch_copy_rows(const void* src, void* dst, int64_t n_t, int64_t n_h, int64_t s_st, int64_t s_sh,
                             int64_t d_st, int64_t d_sh, int64_t row_bytes, const int* smap, const int* dmap,
                             int n_sm, cudaStream_t s) {
  if (row_bytes % 16 != 0) return cudaErrorInvalidValue;
  const int64_t total = n_t * n_h * (row_bytes / 16);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)n_sm * 8) blocks = (int64_t)n_sm * 8;
  copy_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), n_t,
                                                    n_h, s_st, s_sh, d_st, d_sh, row_bytes / 16, smap, dmap);
  return cudaGetLastError();
}

// Data-loader side of ref shard_sequence / unshard (sharding.py:56-106):
// gather (dst[h][t] = src[h][idx[t]]) or scatter (dst[h][idx[t]] = src[h][t])
// of whole token rows, row_vec x 16 bytes, 128-bit accesses, for every head.
__global__ void gather_tokens_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, const int* __restrict__ idx,
                                     int64_t H, int64_t S_src, int64_t L, int64_t S_dst, int64_t row_vec, int scatter) {
  const int64_t total = H * L * row_vec;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i % row_vec;
    const int64_t r = i / row_vec;
    const int64_t t = r % L, h = r / L;
    const int64_t j = __ldg(idx + t);
    if (scatter)
      dst[(h * S_dst + j) * row_vec + e] = __ldg(src + (h * S_src + t) * row_vec + e);
    else
      dst[(h * S_dst + t) * row_vec + e] = __ldg(src + (h * S_src + j) * row_vec + e);
  }
}

cudaError_t launch_gather_tokens(const void* src, void* dst, const int* idx, int64_t H, int64_t S_src, int64_t L,
                                 int64_t S_dst, int64_t row_bytes, int scatter, int n_sm, cudaStream_t s) {
  if (row_bytes % 16 != 0) return cudaErrorInvalidValue;
  const int64_t total = H * L * (row_bytes / 16);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)n_sm * 8) blocks = (int64_t)n_sm * 8;
  gather_tokens_kernel<<<(unsigned)blocks, 256, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), idx, H,
                                                        S_src, L, S_dst, row_bytes / 16, scatter);
  return cudaGetLastError();
}

}  // namespace a2d
