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

// grid (slot blocks of 1024, waypoints): each thread writes 4 pairs of one waypoint at
// stride 256 (every store instruction of a warp covers 512 contiguous bytes), the 4
// point loads are issued before the stores (4 x 16 B in flight per thread), and the
// pair index needs no 64-bit division.
__global__ void __launch_bounds__(256) k_pairgen(const float4 *__restrict__ pts, int64_t lb,
                                                 const float *__restrict__ q, int frame, float4 *__restrict__ out) {
  const int64_t w = blockIdx.y;
  const int64_t s0 = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const float qx = __ldg(q + w * kNdof), qy = __ldg(q + w * kNdof + 1);
  float cth = 1.f, sth = 0.f;  // SE(2) frame (R24): p'_xy = R(-theta)(p_xy - b)
  if (frame) sincosf(__ldg(q + w * kNdof + 2), &sth, &cth);
  float4 p[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) p[k] = s0 + 256 * k < lb ? __ldg(pts + s0 + 256 * k) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 *o = out + w * lb;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (s0 + 256 * k < lb) {
      const float dx = p[k].x - qx, dy = p[k].y - qy;
      __stcs(o + s0 + 256 * k, make_float4(cth * dx + sth * dy, -sth * dx + cth * dy, p[k].z, p[k].w));
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

cudaError_t launch_pairgen(const float4 *pts, int64_t local_bound, const float *q, int32_t n_wp, int frame, float4 *out,
                           cudaStream_t s) {
  if (local_bound <= 0 || n_wp <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((local_bound + 1023) / 1024), (unsigned)n_wp);
  k_pairgen<<<grid, 256, 0, s>>>(pts, local_bound, q, frame, out);
  return cudaGetLastError();
}

}  // namespace gcdf
