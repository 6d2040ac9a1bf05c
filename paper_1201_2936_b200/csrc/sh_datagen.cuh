// Device-side synthetic points for the uniform-box benchmark configs
// (reference datagen.py:53-71).
//
// Draw k of seed s is splitmix64's finaliser applied to s + k * gamma
// (64-bit wraparound), mapped to [0, 1) by its top 53 bits times 2^-53.
// That is integer arithmetic plus one exact conversion and one exact
// scaling, so the device values are bit-identical to the host generator
// (paper_1201_2936_b200/datagen.py, itself the reference's stream).  Point
// i (global index start + i) of a `dim`-D uniform box takes draws
// 1 + (start + i) * dim + c for c = 0..dim-1, like the host generator's
// row-major reshape of one stream.  The kinds built on libm (cos, sin,
// cbrt, log1p) are not bit-reproducible on the device and stay on the host.
#pragma once

#include "sh_common.cuh"

namespace sh {

__device__ __forceinline__ double splitmix_unit(unsigned long long seed, unsigned long long k) {
  unsigned long long z = seed + k * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * 0x1.0p-53;
}

// layout 0: structure of arrays, coordinate c of point i at out[c * n + i];
// layout 1: rows, out[i * dim + c] (the PTS1 / (n, dim) tensor layout)
__global__ void __launch_bounds__(BLOCK) k_uniform_points(int dim, uint64_t n, unsigned long long seed,
                                                          uint64_t start, double* out, int layout) {
  const uint64_t total = n * (uint64_t)dim;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    // e enumerates the draws in stream order (point-major)
    const uint64_t i = e / (uint64_t)dim, c = e - i * (uint64_t)dim;
    const double v = splitmix_unit(seed, 1ull + start * (uint64_t)dim + e);
    if (layout == 1) out[e] = v;
    else out[c * n + i] = v;
  }
}

}  // namespace sh
