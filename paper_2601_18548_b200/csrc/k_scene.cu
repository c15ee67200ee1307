// k_scene.cu -- K4 scene-update scatter (A9) and K1 standalone pair generation +
// base-frame transform (A2).
//
// A9: online injection/removal of obstacle points without rebuilding the problem
//     (PAPER.md:75 (c), :401).  The host decides the slots; one kernel scatters
//     (x, y, z, live) float4s.  O(n_add + n_remove).
// A2: p' = p - [q_x, q_y, 0] for every (waypoint, local slot) pair (PAPER.md:388,
//     :171).  HBM-bound: 16 B written per pair, points re-read from L2.
#include "gcdf_internal.h"

namespace gcdf {
namespace {

__global__ void k_scatter(const float4 *__restrict__ payload, const int64_t *__restrict__ slots, int64_t n,
                          float4 *__restrict__ pts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    pts[slots[i]] = payload[i];
}

__global__ void k_fill_dead(float4 *__restrict__ pts, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    pts[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// One CTA row-block: each thread writes 4 consecutive pairs (4 x 16 B = 64 B) of one
// waypoint; consecutive threads write consecutive 64 B -> fully coalesced 128-bit stores.
__global__ void __launch_bounds__(256) k_pairgen(const float4 *__restrict__ pts, int64_t lb,
                                                 const float *__restrict__ q, int32_t n_wp,
                                                 float4 *__restrict__ out) {
  const int64_t quads = lb / 4;  // lb is a multiple of 128
  const int64_t total = quads * n_wp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = i / quads;
    const int64_t s = (i - w * quads) * 4;
    const float qx = __ldg(q + w * kNdof), qy = __ldg(q + w * kNdof + 1);
    float4 *o = out + w * lb + s;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 p = __ldg(pts + s + k);
      __stcs(o + k, make_float4(p.x - qx, p.y - qy, p.z, p.w));  // streaming store
    }
  }
}

}  // namespace

cudaError_t launch_scene_scatter(const float4 *payload, const int64_t *slots, int64_t n, float4 *pts,
                                 cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int grid = (int)((n + 255) / 256);
  if (grid > 4096) grid = 4096;
  k_scatter<<<grid, 256, 0, s>>>(payload, slots, n, pts);
  return cudaGetLastError();
}

cudaError_t launch_fill(float4 *pts, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int grid = (int)((n + 255) / 256);
  if (grid > 4096) grid = 4096;
  k_fill_dead<<<grid, 256, 0, s>>>(pts, n);
  return cudaGetLastError();
}

cudaError_t launch_pairgen(const float4 *pts, int64_t local_bound, const float *q, int32_t n_wp, float4 *out,
                           cudaStream_t s) {
  const int64_t total = (local_bound / 4) * n_wp;
  if (total <= 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (total + 255) / 256;
  if (grid > (int64_t)sms * 8) grid = (int64_t)sms * 8;  // 8 resident CTAs per SM, grid-stride
  k_pairgen<<<(unsigned)grid, 256, 0, s>>>(pts, local_bound, q, n_wp, out);
  return cudaGetLastError();
}

}  // namespace gcdf
