// Host-side TMA tensor-map construction (driver entry point fetched at run time,
// so the library does not link libcuda directly).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace a2d {

// Tensor map over a bf16 tensor [n2][n1][n0] (n0 innermost, contiguous) with
// element strides (s1, s2) for dims 1 and 2, box {64, box1, 1}, SWIZZLE_128B.
// Out-of-bounds rows are zero-filled by the hardware.
int make_tmap_bf16_3d(CUtensorMap* out, const void* base, uint64_t n0, uint64_t n1, uint64_t n2,
                      uint64_t s1, uint64_t s2, uint32_t box1);

}  // namespace a2d
