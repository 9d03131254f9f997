// Probe (not part of the library): can one kernel mix CTA-pair MMAs
// (tcgen05.mma.cta_group::2, leader-issued, M = 256) with per-CTA MMAs
// (tcgen05.mma.cta_group::1, M = 128) on pair-allocated TMEM? This decides
// whether a pair backward can keep dQ^T as a per-CTA GEMM.
//
//   D_pair = [A0; A1] . B^T      (B's 128 rows split: CTA c holds rows 64c..64c+63)
//   D_c    = A_c . C_c^T         (each CTA alone)
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -shared -Xcompiler -fPIC
//        -I paper_2406_18485_b200/csrc tools/probes/pair_mix_probe.cu -o tools/probes/_pair_mix_probe.so
#include "sm100.cuh"

using namespace a2d;

// copy a [rows][128] bf16 row-major matrix into the SW128 K-major layout (2 panels of 64 k)
__device__ void to_sw128(uint8_t* dst, const __nv_bfloat16* src, int rows) {
  for (int i = threadIdx.x; i < rows * 16; i += blockDim.x) {
    const int r = i / 16, c16 = i % 16;  // 16 chunks of 8 bf16 per row
    const int panel = c16 / 8, c = c16 % 8;
    const uint4 v = *reinterpret_cast<const uint4*>(src + r * 128 + c16 * 8);
    *reinterpret_cast<uint4*>(dst + panel * rows * 128 + sw128_offset(r, c)) = v;
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_mix_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, const __nv_bfloat16* Cm, float* Dpair,
                    float* Down) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar_pair, bar_own;
  __shared__ uint32_t holder;
  const int rank = (int)cluster_rank();
  const int warp = threadIdx.x / 32;
  uint8_t* sA = smem;                  // 32 KB: this CTA's 128 rows of A
  uint8_t* sB = smem + 32768;          // 16 KB: this CTA's 64 rows of B
  uint8_t* sC = smem + 32768 + 16384;  // 32 KB: this CTA's C
  to_sw128(sA, A + rank * 128 * 128, 128);
  to_sw128(sB, B + rank * 64 * 128, 64);
  to_sw128(sC, Cm + rank * 128 * 128, 128);
  fence_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar_pair, 1);
    mbar_init(&bar_own, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_pair<256>(&holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = holder;
  const uint64_t dA = sdesc_sw128(smem_u32(sA), 16, 1024), dB = sdesc_sw128(smem_u32(sB), 16, 1024);
  const uint64_t dC = sdesc_sw128(smem_u32(sC), 16, 1024);
  if (rank == 0 && warp == 0) {
    __syncwarp();
    if (elect_one()) {
      for (int k = 0; k < 8; ++k) {
        const uint64_t oa = (uint64_t)(((k / 4) * 16384 + (k % 4) * 32) >> 4);
        const uint64_t ob = (uint64_t)(((k / 4) * 8192 + (k % 4) * 32) >> 4);
        umma_ss_pair(tmem, dA + oa, dB + ob, idesc_bf16(256, 128, false, false), k > 0);
      }
      umma_commit_pair(&bar_pair);
    }
    __syncwarp();
  }
  mbar_wait(&bar_pair, 0);
  tc_fence_after();
  if (warp == 0) {  // this CTA's own GEMM, into columns [128, 256)
    __syncwarp();
    if (elect_one()) {
      for (int k = 0; k < 8; ++k) {
        const uint64_t o = (uint64_t)(((k / 4) * 16384 + (k % 4) * 32) >> 4);
        umma_ss(tmem + 128, dA + o, dC + o, idesc_bf16(128, 128, false, false), k > 0);
      }
      umma_commit(&bar_own);
    }
    __syncwarp();
  }
  mbar_wait(&bar_own, 0);
  tc_fence_after();
  const int row = (warp % 4) * 32 + (threadIdx.x % 32);
  const uint32_t lane_base = (uint32_t)((warp % 4) * 32) << 16;
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tmem_ld32(tmem + lane_base + c * 32, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) Dpair[(rank * 128 + row) * 128 + c * 32 + i] = __uint_as_float(r[i]);
    tmem_ld32(tmem + lane_base + 128 + c * 32, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) Down[(rank * 128 + row) * 128 + c * 32 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc_pair<256>(tmem);
}

extern "C" int pair_mix_probe(const void* A, const void* B, const void* C, float* Dpair, float* Down) {
  const int smem = 32768 + 16384 + 32768 + 1024;
  cudaFuncSetAttribute(pair_mix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pair_mix_kernel<<<2, 128, smem>>>(static_cast<const __nv_bfloat16*>(A), static_cast<const __nv_bfloat16*>(B),
                                    static_cast<const __nv_bfloat16*>(C), Dpair, Down);
  cudaError_t e = cudaDeviceSynchronize();
  return e == cudaSuccess ? 0 : (int)e;
}
