// Rate of the five GEMMs of the 128-query backward (fa_bwd_q128.cuh) with the
// kernel's exact shared-memory layout, descriptors and TMEM map, issued
// back-to-back by one thread per CTA (one CTA per SM, no other traffic).
// Answers whether the per-iteration GEMM time is 5 x 512 clk when nothing
// else runs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2406_18485_b200/csrc \
//        tools/probes/q128_gemm_rate.cu -o /tmp/q128_gemm_rate && /tmp/q128_gemm_rate
#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace a2d;

// MODE: 0 S^T (SS, K-major, N=128) | 1 dV (TS, B MN-major) | 2 dQ^T (SS, both MN-major)
//       3 all five in the kernel's order: dV, S, dK, dQ^T, dP
// SIDE (MODE 3 only): 0 none | 1 eight warps tcgen05.ld 64 cols + tcgen05.st 16 cols per
// round (the P/dS warps' TMEM traffic) | 2 four warps tcgen05.ld 128 cols (the drain) |
// 3 four warps STS.128 | 4 = 1 + 2 + 3
template <int MODE, int SIDE = 0>
__global__ void __launch_bounds__(512, 1) probe(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ int done;
  const int warp = warp_id(), lane = lane_id();
  for (int i = threadIdx.x; i < (224 * 1024) / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    done = 0;
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 1) {
    constexpr uint32_t id_s = idesc_bf16(128, 128, false, false);
    constexpr uint32_t id_kv = idesc_bf16(128, 128, false, true);
    constexpr uint32_t id_dq = idesc_bf16(128, 128, true, true);
    const uint32_t sK = smem_u32(smem), sV = smem_u32(smem + 32768), sQ = smem_u32(smem + 65536);
    const uint32_t sDO = smem_u32(smem + 131072), sDS = smem_u32(smem + 163840);
    const uint32_t tS = tmem, tDP = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;
    const uint64_t dK0 = sdesc_sw128(sK, 16, 1024), dV0 = sdesc_sw128(sV, 16, 1024);
    const uint64_t dQ0 = sdesc_sw128(sQ, 16, 1024), dDO0 = sdesc_sw128(sDO, 16, 1024);
    const uint64_t dKmn = sdesc_sw128(sK, 16384, 1024), dDSmn = sdesc_sw128(sDS, 16384, 1024);
    const uint64_t dQmn = sdesc_sw128(sQ, 16384, 1024), dDOmn = sdesc_sw128(sDO, 16384, 1024);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      __syncwarp();
      if (elect_one()) {
        if (MODE == 1 || MODE == 3)
#pragma unroll
          for (int k = 0; k < 8; ++k) umma_ts(tDV, tS + (k / 2) * 32 + (k % 2) * 8, dDOmn + (uint64_t)(k * 128), id_kv, 1u);
        if (MODE == 0 || MODE == 3)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t ka = (uint64_t)(((k / 4) * 16384 + (k % 4) * 32) >> 4);
            umma_ss(tS, dK0 + ka, dQ0 + ka, id_s, k > 0);
          }
        if (MODE == 3)
#pragma unroll
          for (int k = 0; k < 8; ++k) umma_ts(tDK, tDP + (k / 2) * 32 + (k % 2) * 8, dQmn + (uint64_t)(k * 128), id_kv, 1u);
        if (MODE == 2 || MODE == 3)
#pragma unroll
          for (int k = 0; k < 8; ++k) umma_ss(tDP, dKmn + (uint64_t)(k * 128), dDSmn + (uint64_t)(k * 128), id_dq, k > 0);
        if (MODE == 3)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t ka = (uint64_t)(((k / 4) * 16384 + (k % 4) * 32) >> 4);
            umma_ss(tDP, dV0 + ka, dDO0 + ka, id_s, k > 0);
          }
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (lane == 0) {
      out[blockIdx.x] = clock64() - t0;
      atomicExch(&done, 1);
    }
  } else if (warp >= 4 && SIDE != 0) {
    const uint32_t lb = (uint32_t)((warp % 4) * 32) << 16;
    uint32_t acc = 0;
    while (!*(volatile int*)&done) {
      if ((SIDE == 1 || SIDE == 4) && warp < 12) {  // P/dS-like: ld 64 cols, st 16 cols
        const uint32_t base = tmem + lb + (warp < 8 ? 0 : 128) + ((warp / 4) & 1) * 64;
        uint32_t r[32];
        tmem_ld32(base, r);
        tmem_ld_wait();
        acc += r[0] ^ r[31];
        tmem_ld32(base + 32, r);
        tmem_ld_wait();
        acc += r[3];
        tmem_st16(base, r);
        tmem_st_wait();
      } else if ((SIDE == 2 || SIDE == 4) && warp >= 12) {  // drain-like: ld 128 cols
        uint32_t r[32];
#pragma unroll 1
        for (int b = 0; b < 4; ++b) {
          tmem_ld32(tmem + lb + 128 + b * 32, r);
          tmem_ld_wait();
          acc += r[1];
        }
        if (SIDE == 4) {
          uint8_t* st = smem + 196608 + (warp % 4) * 4096 + lane * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(st + ((c ^ (lane & 7)) << 4)) = make_uint4(acc, c, 0, 0);
        }
      } else if (SIDE == 3 && warp >= 12) {
        uint8_t* st = smem + 196608 + (warp % 4) * 4096 + lane * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(st + ((c ^ (lane & 7)) << 4)) = make_uint4(acc, c, 0, 0);
      }
    }
    if (acc == 0x9876543u) out[blockIdx.x] = -1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int MODE, int SIDE = 0>
void run(const char* name, int n_sm, int gemms) {
  const int reps = 2048;
  long long* d;
  cudaMalloc(&d, sizeof(long long) * n_sm);
  const int smem = 224 * 1024;
  cudaFuncSetAttribute(probe<MODE, SIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<MODE, SIDE><<<n_sm, 512, smem>>>(8, d);
  cudaDeviceSynchronize();
  probe<MODE, SIDE><<<n_sm, 512, smem>>>(reps, d);
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<long long> h(n_sm);
  cudaMemcpy(h.data(), d, sizeof(long long) * n_sm, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (auto c : h) cyc += c;
  cyc /= n_sm;
  const double per = cyc / reps / gemms;  // clk per 128x128x128 GEMM (ideal 512)
  printf("%-40s %s  %.1f clk per GEMM (ideal 512, %.1f%%)\n", name, err == cudaSuccess ? "ok " : cudaGetErrorString(err),
         per, 100.0 * 512 / per);
  cudaFree(d);
}

int main() {
  int n_sm = 0;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  run<0>("S^T  SS K-major N128", n_sm, 1);
  run<1>("dV   TS, B MN-major LBO 16K", n_sm, 1);
  run<2>("dQ^T SS, A+B MN-major LBO 16K", n_sm, 1);
  run<3>("all five (dV,S,dK,dQ^T,dP)", n_sm, 5);
  run<3, 1>("all five + P/dS-like TMEM ld/st (8 warps)", n_sm, 5);
  run<3, 2>("all five + drain-like TMEM ld (4 warps)", n_sm, 5);
  run<3, 3>("all five + STS.128 (4 warps)", n_sm, 5);
  run<3, 4>("all five + all of the above", n_sm, 5);
  return 0;
}
