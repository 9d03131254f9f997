// UMMA issue-rate probe (B200, sm_100a): how fast do back-to-back
// tcgen05.mma of the shapes the backward uses run, and does concurrent
// shared-memory / TMEM traffic slow them down? Answers whether SS MMAs with
// N=64 are operand-bandwidth bound before redesigning.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2406_18485_b200/csrc \
//        tools/probes/umma_rate.cu -o tools/probes/umma_rate && tools/probes/umma_rate
//
// One CTA per SM; warp 1 issues R x 8 K16-steps of one MMA shape into TMEM,
// commits, waits; optional warps 4-7 hammer LDS.128 / tcgen05.ld meanwhile.
// Prints MACs per clock per SM (peak 4096 for bf16 M=128 cta_group::1).
#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace a2d;

struct Res {
  long long mma_cycles;
  long long side_ops;
};

// mode: 0 SS N64 | 1 SS N128 | 2 SS N256 | 3 TS N64 | 4 TS N128 (B MN-major) | 5 SS N64 A MN-major
// side: 0 none | 1 LDS.128 hammer (4 warps) | 2 tcgen05.ld hammer (4 warps) | 3 STS.128 hammer
template <int MODE, int SIDE>
__global__ void __launch_bounds__(256, 1) probe(int reps, Res* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ int done;
  const int warp = warp_id(), lane = lane_id();
  for (int i = threadIdx.x; i < (160 * 1024) / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
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
  constexpr int N = (MODE == 1 || MODE == 4) ? 128 : (MODE == 2 ? 256 : 64);
  const uint32_t sA = smem_u32(smem), sB = smem_u32(smem + 32768);
  if (warp == 1) {
    const uint32_t id = idesc_bf16(128, N, MODE == 5, MODE == 4);
    const uint64_t dA = sdesc_sw128(sA, MODE == 5 ? 16384 : 16, 1024);
    const uint64_t dB = sdesc_sw128(sB, MODE == 4 ? 8192 : 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      __syncwarp();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t ka = MODE == 5 ? (uint64_t)(k * 128) : (uint64_t)(((k / 4) * 16384 + (k % 4) * 32) >> 4);
          const uint64_t kb = MODE == 4 ? (uint64_t)(k * 128) : (uint64_t)(((k / 4) * N * 128 + (k % 4) * 32) >> 4);
          if (MODE == 3 || MODE == 4)
            umma_ts(tmem, tmem + 256 + k * 8, dB + kb, id, 1u);
          else
            umma_ss(tmem, dA + ka, dB + kb, id, 1u);
        }
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane == 0) {
      out[blockIdx.x].mma_cycles = t1 - t0;
      atomicExch(&done, 1);
    }
  } else if (warp >= 4 && SIDE != 0) {
    long long ops = 0;
    uint32_t acc = 0;
    uint8_t* region = smem + 98304;  // 32 KB side region
    const int wq = warp - 4;
    while (!*(volatile int*)&done) {
#pragma unroll 1
      for (int it = 0; it < 64; ++it) {
        if (SIDE == 1) {
          const uint4 v = *reinterpret_cast<const uint4*>(region + ((it * 32 + lane) & 2047) * 16);
          acc += v.x ^ v.w;
        } else if (SIDE == 3) {
          *reinterpret_cast<uint4*>(region + ((it * 32 + lane + wq * 512) & 2047) * 16) = make_uint4(it, acc, lane, 0);
        } else {
          uint32_t r[32];
          tmem_ld32(tmem + ((uint32_t)(wq * 32) << 16) + 384 + (it & 3) * 32, r);
          tmem_ld_wait();
          acc += r[0] ^ r[31];
        }
      }
      ops += 64;
    }
    if (lane == 0) atomicAdd((unsigned long long*)&out[blockIdx.x].side_ops, (unsigned long long)ops);
    if (acc == 0x12345678) out[blockIdx.x].side_ops = -1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int MODE, int SIDE>
void run(const char* name, int n_sm) {
  const int reps = 4096;
  Res* d;
  cudaMalloc(&d, sizeof(Res) * n_sm);
  cudaMemset(d, 0, sizeof(Res) * n_sm);
  const int smem = 160 * 1024 + 1024;
  cudaFuncSetAttribute(probe<MODE, SIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<MODE, SIDE><<<n_sm, 256, smem>>>(16, d);  // warm-up
  cudaDeviceSynchronize();
  cudaMemset(d, 0, sizeof(Res) * n_sm);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<MODE, SIDE><<<n_sm, 256, smem>>>(reps, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<Res> h(n_sm);
  cudaMemcpy(h.data(), d, sizeof(Res) * n_sm, cudaMemcpyDeviceToHost);
  double cyc = 0, ops = 0;
  for (auto& r : h) {
    cyc += r.mma_cycles;
    ops += r.side_ops;
  }
  cyc /= n_sm;
  ops /= n_sm;
  const int N = (MODE == 1 || MODE == 4) ? 128 : (MODE == 2 ? 256 : 64);
  const double macs = (double)reps * 8 * 128 * N * 16;
  const double side_bytes = SIDE == 2 ? ops * 4 * 32 * 32 * 4 / 4 : ops * 16 * 32;  // per warp-op bytes x 4 warps / 4
  printf("%-34s %s  MAC/clk/SM %7.1f (%.1f%% of 4096)  %.3f ms  TFLOP/s %.0f  side B/clk %.1f\n", name,
         err == cudaSuccess ? "ok " : cudaGetErrorString(err), macs / cyc, 100.0 * macs / cyc / 4096, ms,
         2.0 * macs * n_sm / (ms * 1e-3) / 1e12, SIDE ? side_bytes * 4 / cyc : 0.0);
  cudaFree(d);
}

int main() {
  int n_sm = 0;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  run<0, 0>("SS M128 N64", n_sm);
  run<1, 0>("SS M128 N128", n_sm);
  run<2, 0>("SS M128 N256", n_sm);
  run<3, 0>("TS M128 N64", n_sm);
  run<4, 0>("TS M128 N128 (B MN-major)", n_sm);
  run<5, 0>("SS M128 N64 (A MN-major)", n_sm);
  run<0, 1>("SS N64 + LDS.128 hammer", n_sm);
  run<0, 3>("SS N64 + STS.128 hammer", n_sm);
  run<0, 2>("SS N64 + tcgen05.ld hammer", n_sm);
  run<3, 1>("TS N64 + LDS.128 hammer", n_sm);
  run<1, 1>("SS N128 + LDS.128 hammer", n_sm);
  run<4, 2>("TS N128 + tcgen05.ld hammer", n_sm);
  return 0;
}
