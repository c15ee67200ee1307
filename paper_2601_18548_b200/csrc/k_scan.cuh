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

// The scan kernels below are static (internal linkage) so every translation unit that
// includes this header gets its own copy.
namespace scan_detail {
// ---- device-wide exclusive scan (int32 or int64 input -> int64), three launches
template <typename T>
static __global__ void __launch_bounds__(1024) k_scan_blocks(const T *__restrict__ in, int64_t n, int64_t *__restrict__ out,
                                                       int64_t *__restrict__ sums) {
  __shared__ int64_t sh[32];
  const int64_t i = blockIdx.x * 1024ll + threadIdx.x;
  const int64_t v = i < n ? (int64_t)in[i] : 0;
  int64_t tot;
  const int64_t ex = block_excl_scan(v, &tot, sh);
  if (i < n) out[i] = ex;
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}
static __global__ void __launch_bounds__(1024) k_scan_sums(int64_t *sums, int64_t nb, int64_t *__restrict__ total_out) {
  __shared__ int64_t sh[32];
  int64_t carry = 0;
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < nb ? sums[i] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan(v, &tot, sh);
    if (i < nb) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total_out = carry;
}
static __global__ void __launch_bounds__(1024) k_scan_add(int64_t *__restrict__ out, int64_t n, const int64_t *sums) {
  const int64_t i = blockIdx.x * 1024ll + threadIdx.x;
  if (i < n) out[i] += sums[blockIdx.x];
}
template <typename T>
static cudaError_t excl_scan(const T *in, int64_t n, int64_t *out, int64_t *total_out, int64_t *tmp, cudaStream_t s,
                      int *nl) {
  const int64_t nb = (n + 1023) / 1024;
  if (nb <= 0) return cudaSuccess;
  k_scan_blocks<T><<<(unsigned)nb, 1024, 0, s>>>(in, n, out, tmp);
  k_scan_sums<<<1, 1024, 0, s>>>(tmp, nb, total_out);
  k_scan_add<<<(unsigned)nb, 1024, 0, s>>>(out, n, tmp);
  *nl += 3;
  return cudaGetLastError();
}

}  // namespace scan_detail
using scan_detail::excl_scan;

}  // namespace gcdf
