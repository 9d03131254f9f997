// HBM-kernel variant probe (B200): achieved GB/s of candidate layouts for the
// two HBM-bound helpers below roofline in r01 (bwd_preprocess, dqt_to_bf16)
// at the bench shape (H=32, T=131072, D=128), each timed alone with CUDA
// events over 20 launches after warm-up (inputs 2-3 GB >> L2).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probes/hbm_probe.cu -o tools/probes/hbm_probe
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int H = 32, D = 128;
constexpr long long T = 131072;

// ---------------------------------------------------------------- preprocess
template <int RPT>  // rows per lane group per iteration
__global__ void pre_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                           const float* __restrict__ lse, float* __restrict__ lse2, float* __restrict__ delta,
                           long long rows) {
  constexpr int kL = D / 8;
  const int sub = threadIdx.x % kL;
  const long long groups = (long long)gridDim.x * blockDim.x / kL;
  for (long long r0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / kL; r0 < rows; r0 += groups * RPT) {
    uint4 a[RPT], b[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const long long r = r0 + u * groups;
      if (r < rows) {
        a[u] = __ldcs(reinterpret_cast<const uint4*>(o + r * D) + sub);
        b[u] = __ldcs(reinterpret_cast<const uint4*>(dout + r * D) + sub);
      }
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const long long r = r0 + u * groups;
      float acc = 0.f;
      const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a[u]);
      const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b[u]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 x = __bfloat1622float2(pa[i]), y = __bfloat1622float2(pb[i]);
        acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
      }
#pragma unroll
      for (int off = kL / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (sub == 0 && r < rows) {
        lse2[r] = lse[r] * 1.4426950408889634f;
        delta[r] = acc;
      }
    }
  }
}

// ---------------------------------------------------------------- dqt_to_bf16
template <int TPT>  // 4-token groups per thread
__global__ void __launch_bounds__(512) dqt_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                                  long long T_pad) {
  const int h = blockIdx.y;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int f0 = 8 * w;
#pragma unroll
  for (int g = 0; g < TPT; ++g) {
    const long long t = (long long)blockIdx.x * 128 * TPT + g * 128 + 4 * lane;
    const float* s = src + ((size_t)h * D + f0) * T_pad + t;
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
      *reinterpret_cast<uint4*>(dst + ((size_t)h * T + t + j) * D + f0) =
          make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                     *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
    }
  }
}

// smem-staged transpose: block = 64 tokens x 128 features; coalesced float4
// loads along tokens, conflict-free column reads (XOR-swizzled 16-byte chunks),
// each warp writes full 256-byte token rows (16 lanes x 16 B, 2 rows per warp).
__global__ void __launch_bounds__(256) dqt_smem_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                                       long long T_pad) {
  __shared__ float4 tile[128][16];  // [feature][4-token chunk ^ swz]
  const int h = blockIdx.y;
  const long long t0 = (long long)blockIdx.x * 64;
  const float* s = src + (size_t)h * D * T_pad + t0;
  for (int i = threadIdx.x; i < 128 * 16; i += 256) {
    const int f = i / 16, c = i % 16;
    tile[f][c ^ (f & 15)] = __ldcs(reinterpret_cast<const float4*>(s + (size_t)f * T_pad) + c);
  }
  __syncthreads();
  // thread: token tt (0..63), feature chunk fc (0..15) of 8 features
  for (int i = threadIdx.x; i < 64 * 16; i += 256) {
    const int tt = i / 16, fc = i % 16;
    const int c = tt / 4, e = tt % 4;
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int f = fc * 8 + k;
      const float4 q = tile[f][c ^ (f & 15)];
      v[k] = e == 0 ? q.x : e == 1 ? q.y : e == 2 ? q.z : q.w;
    }
    __nv_bfloat162 p0 = __floats2bfloat162_rn(v[0], v[1]), p1 = __floats2bfloat162_rn(v[2], v[3]);
    __nv_bfloat162 p2 = __floats2bfloat162_rn(v[4], v[5]), p3 = __floats2bfloat162_rn(v[6], v[7]);
    *reinterpret_cast<uint4*>(dst + ((size_t)h * T + t0 + tt) * D + fc * 8) =
        make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                   *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
  }
}

// Z: registers -> bf16 -> swizzled smem [token][feature] -> full 256-byte
// token rows to global (each warp store covers two whole rows).
__global__ void __launch_bounds__(512) dqt_z_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                                    long long T_pad) {
  __shared__ __align__(16) uint4 tile[128][16];  // [token][16-byte chunk (8 features), swizzled]
  const int h = blockIdx.y;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long t0 = (long long)blockIdx.x * 128;
  const float* s = src + ((size_t)h * D + 8 * w) * T_pad + t0 + 4 * lane;
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
    const int row = 4 * lane + j;
    tile[row][w ^ (lane & 15)] = make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                                            *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {  // 2048 chunks / 512 threads
    const int idx = k * 512 + threadIdx.x;
    const int row = idx / 16, c = idx % 16;
    const uint4 val = tile[row][c ^ ((row >> 2) & 15)];
    *reinterpret_cast<uint4*>(dst + ((size_t)h * T + t0 + row) * D + 8 * c) = val;
  }
}

template <class F>
void timeit(const char* name, double bytes, F launch) {
  for (int i = 0; i < 3; ++i) launch();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) launch();
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 20;
  printf("%-40s %s %.3f ms  %.0f GB/s (%.1f%% of 6527.5)\n", name, e == cudaSuccess ? "ok" : cudaGetErrorString(e), ms,
         bytes / (ms * 1e-3) / 1e9, 100.0 * bytes / (ms * 1e-3) / 1e9 / 6527.5);
}

int main() {
  int n_sm;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  const long long rows = (long long)H * T;
  __nv_bfloat16 *o, *dout, *dq;
  float *lse, *lse2, *delta, *acc;
  cudaMalloc(&o, rows * D * 2);
  cudaMalloc(&dout, rows * D * 2);
  cudaMalloc(&lse, rows * 4);
  cudaMalloc(&lse2, rows * 4);
  cudaMalloc(&delta, rows * 4);
  cudaMalloc(&acc, rows * D * 4);
  cudaMalloc(&dq, rows * D * 2);
  cudaMemset(o, 0, rows * D * 2);
  cudaMemset(dout, 0, rows * D * 2);
  cudaMemset(acc, 0, rows * D * 4);
  const double pre_bytes = rows * (4.0 * D + 4 + 8);
  for (int blocks_per_sm : {8, 16, 32}) {
    char nm[64];
    snprintf(nm, sizeof nm, "preprocess rpt=1 grid=%dxSM", blocks_per_sm);
    timeit(nm, pre_bytes, [&] { pre_kernel<1><<<n_sm * blocks_per_sm, 256>>>(o, dout, lse, lse2, delta, rows); });
    snprintf(nm, sizeof nm, "preprocess rpt=2 grid=%dxSM", blocks_per_sm);
    timeit(nm, pre_bytes, [&] { pre_kernel<2><<<n_sm * blocks_per_sm, 256>>>(o, dout, lse, lse2, delta, rows); });
    snprintf(nm, sizeof nm, "preprocess rpt=4 grid=%dxSM", blocks_per_sm);
    timeit(nm, pre_bytes, [&] { pre_kernel<4><<<n_sm * blocks_per_sm, 256>>>(o, dout, lse, lse2, delta, rows); });
  }
  timeit("preprocess rpt=1 full grid", pre_bytes,
         [&] { pre_kernel<1><<<(unsigned)(rows * 16 / 256), 256>>>(o, dout, lse, lse2, delta, rows); });
  const double dqt_bytes = rows * D * 6.0;
  timeit("dqt regs tpt=1 (current)", dqt_bytes, [&] { dqt_kernel<1><<<dim3(T / 128, H), 512>>>(acc, dq, T); });
  timeit("dqt regs tpt=2", dqt_bytes, [&] { dqt_kernel<2><<<dim3(T / 256, H), 512>>>(acc, dq, T); });
  timeit("dqt regs tpt=4", dqt_bytes, [&] { dqt_kernel<4><<<dim3(T / 512, H), 512>>>(acc, dq, T); });
  timeit("dqt smem 64x128 swizzled", dqt_bytes, [&] { dqt_smem_kernel<<<dim3(T / 64, H), 256>>>(acc, dq, T); });
  timeit("dqt Z regs->bf16 smem->full rows", dqt_bytes, [&] { dqt_z_kernel<<<dim3(T / 128, H), 512>>>(acc, dq, T); });
  timeit("dqt regs tpt=1 (again)", dqt_bytes, [&] { dqt_kernel<1><<<dim3(T / 128, H), 512>>>(acc, dq, T); });
  timeit("copy f32->f32 (cudaMemcpy D2D ref)", rows * D * 8.0,
         [&] { cudaMemcpyAsync(acc + rows * D / 2, acc, rows * D * 2, cudaMemcpyDeviceToDevice); });
  return 0;
}
