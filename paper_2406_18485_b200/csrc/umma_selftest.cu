// Unit test of the UMMA plumbing used by the attention kernels.
//
// One CTA computes, for 128x128x128 bf16 operands:
//   c[0] = A  * B^T   (SS, A K-major via TMA, B K-major via TMA)      -> like S = Q K^T
//   c[1] = A  * V     (SS, B MN-major, V written to smem by threads)   -> like O = P V
//   c[2] = At^T * B^T (SS, A MN-major written by threads)              -> like dQ^T = K^T dS^T
//   c[3] = A  * V     (TS, A staged into TMEM by tcgen05.st)           -> like O = P(tmem) V
// The host compares each against a reference GEMM.
#include "sm100.cuh"
#include "kernels.h"

namespace a2d {

__global__ void __launch_bounds__(128, 1) umma_selftest_kernel(const __grid_constant__ SelftestParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in .shared
  uint8_t* sA = smem;              // 2 panels x 16 KB
  uint8_t* sB = smem + 32768;      // 2 panels x 16 KB
  uint8_t* sV = smem + 65536;      // MN-major: 2 panels (n 0-63, 64-127) x 16 KB
  uint8_t* sAt = smem + 98304;     // MN-major: 2 panels (m 0-63, 64-127) x 16 KB
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;

  const int warp = warp_id(), lane = lane_id(), tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  // thread-written MN-major operands: row k (K index) holds 128 MN elements,
  // split into two 64-wide panels; within a panel row k is a 128 B SW128 row.
  for (int idx = tid; idx < 128 * 16; idx += 128) {
    int k = idx / 16, chunk16 = idx % 16;     // 16 chunks of 8 elements per row
    int panel = chunk16 / 8, c = chunk16 % 8;
    uint4 vv = *reinterpret_cast<const uint4*>(p.v + k * 128 + chunk16 * 8);
    uint4 tt = *reinterpret_cast<const uint4*>(p.at + k * 128 + chunk16 * 8);
    *reinterpret_cast<uint4*>(sV + panel * 16384 + sw128_offset(k, c)) = vv;
    *reinterpret_cast<uint4*>(sAt + panel * 16384 + sw128_offset(k, c)) = tt;
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  // stage A into TMEM columns [384, 448): row m = lane, 128 bf16 = 64 columns
  {
    uint32_t r[32];
    const int row = warp * 32 + lane;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(p.a + row * 128 + half * 64 + 2 * i);
        r[i] = *reinterpret_cast<uint32_t*>(&x);
      }
      tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 384 + half * 32, r);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (tid == 0) {
    mbar_expect_tx(&bar_tma, 65536);
    tma_load_3d(sA, &p.tm_a, &bar_tma, 0, 0, 0);
    tma_load_3d(sA + 16384, &p.tm_a, &bar_tma, 64, 0, 0);
    tma_load_3d(sB, &p.tm_b, &bar_tma, 0, 0, 0);
    tma_load_3d(sB + 16384, &p.tm_b, &bar_tma, 64, 0, 0);
    mbar_wait(&bar_tma, 0);
    tc_fence_after();
    const uint32_t id_kk = idesc_bf16(128, 128, false, false);
    const uint32_t id_kmn = idesc_bf16(128, 128, false, true);
    const uint32_t id_mnk = idesc_bf16(128, 128, true, false);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB), v0 = smem_u32(sV), t0 = smem_u32(sAt);
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // K = 128 in steps of 16
      uint32_t koff = (k / 4) * 16384 + (k % 4) * 32;  // K-major: panel + 32 B per step
      uint32_t mnoff = k * 2048;                        // MN-major: 16 K-rows = 2 atoms
      umma_ss(tmem + 0, sdesc_sw128(a0 + koff, 16, 1024), sdesc_sw128(b0 + koff, 16, 1024), id_kk, k > 0);
      umma_ss(tmem + 128, sdesc_sw128(a0 + koff, 16, 1024), sdesc_sw128(v0 + mnoff, 16384, 1024), id_kmn, k > 0);
      umma_ss(tmem + 256, sdesc_sw128(t0 + mnoff, 16384, 1024), sdesc_sw128(b0 + koff, 16, 1024), id_mnk, k > 0);
    }
    umma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  // TS: reuse columns [384, 448) as A, accumulate into [448, 512) ... need 128
  // output columns, so write c[3] into columns [0,128) after c[0] is read out.
  tc_fence_after();
  const int row = warp * 32 + lane;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  for (int g = 0; g < 3; ++g) {
    for (int ch = 0; ch < 4; ++ch) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_base + g * 128 + ch * 32, r);
      tmem_ld_wait();
      for (int i = 0; i < 32; ++i) p.c[(g * 128 + row) * 128 + ch * 32 + i] = __uint_as_float(r[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t id_kmn = idesc_bf16(128, 128, false, true);
    const uint32_t v0 = smem_u32(sV);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      umma_ts(tmem + 0, tmem + 384 + k * 8, sdesc_sw128(v0 + k * 2048, 16384, 1024), id_kmn, k > 0);
    umma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 1);
  tc_fence_after();
  for (int ch = 0; ch < 4; ++ch) {
    uint32_t r[32];
    tmem_ld32(tmem + lane_base + ch * 32, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) p.c[(3 * 128 + row) * 128 + ch * 32 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

cudaError_t launch_umma_selftest(const SelftestParams& p, cudaStream_t s) {
  const int smem = 131072 + 1024;
  cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_selftest_kernel<<<1, 128, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace a2d
