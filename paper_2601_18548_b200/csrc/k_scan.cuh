// k_scan.cuh -- block-wide exclusive scan shared by the compaction and partition kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gcdf {

// exclusive scan of v over the block (blockDim.x multiple of 32, <= 1024)
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t *total, int64_t *sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t s = lane < nw ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sh[lane] = s;  // inclusive prefix of warp totals
  }
  __syncthreads();
  const int64_t res = x - v + (warp > 0 ? sh[warp - 1] : 0);
  *total = sh[nw - 1];
  __syncthreads();
  return res;
}

}  // namespace gcdf
