// k_partition.cu -- NEXT-1 range partition (R23):
// I_{M,i} = { j : |p_j,xy - (x_i, y_i)| <= r } as ordered per-step candidate lists and a
// tile map for the fused detect kernels.
//
//   grid (when the scene or r changed): bbox of the live points -> cell size
//   cs = max(r, extent / 1024) -> counting sort of the live slots by cell.
//   per call: per step, the 3x3 cells around its base (cs >= r covers the disk) are
//   scanned and the slots within r are set in a per-step bitmap; bitmap chunks are
//   counted, scanned in (step, chunk) order and emitted in ascending slot order, so every
//   step's list is sorted and the detect output keeps the canonical (wp, pt) order.
//   Tiles: ceil(m_i / 128) per step, tile_start = their exclusive scan, tile_wp[T] = step.
// All HBM/L2-bound integer work; the points (16 B per slot) stay L2-resident.
#include <algorithm>

#include "gcdf_internal.h"
#include "k_scan.cuh"

namespace gcdf {
namespace {

constexpr int kSub = 2;  // cells per radius: a step scans (2 kSub + 1)^2 cells, pruned by box distance

__device__ __forceinline__ unsigned ord_f(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_f(unsigned u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__global__ void k_bbox_init(unsigned *bbox) {
  if (threadIdx.x == 0) {
    bbox[0] = bbox[1] = 0xffffffffu;  // min x, min y
    bbox[2] = bbox[3] = 0u;           // max x, max y
  }
}

__global__ void __launch_bounds__(256) k_bbox(const float4 *__restrict__ pts, int64_t n, unsigned *bbox) {
  unsigned mnx = 0xffffffffu, mny = 0xffffffffu, mxx = 0u, mxy = 0u;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 p = pts[i];
    if (p.w > 0.f) {
      const unsigned x = ord_f(p.x), y = ord_f(p.y);
      mnx = min(mnx, x); mny = min(mny, y); mxx = max(mxx, x); mxy = max(mxy, y);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mnx = min(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
    mny = min(mny, __shfl_xor_sync(0xffffffffu, mny, o));
    mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
    mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(bbox, mnx); atomicMin(bbox + 1, mny); atomicMax(bbox + 2, mxx); atomicMax(bbox + 3, mxy);
  }
}

// grid parameters: g[0] ox, g[1] oy, g[2] 1/cs, g[3] cs, g[4] r, g[5] nx, g[6] ny (ints as float bits)
__global__ void k_grid_params(const unsigned *bbox, float r, float *g) {
  if (threadIdx.x != 0) return;
  int nx = 0, ny = 0;
  float ox = 0.f, oy = 0.f, cs = r;
  if (bbox[0] != 0xffffffffu) {
    ox = unord_f(bbox[0]);
    oy = unord_f(bbox[1]);
    const float ex = unord_f(bbox[2]) - ox, ey = unord_f(bbox[3]) - oy;
    // cs = r / kSub with a 1e-4 margin: a point within r of a base is at most kSub cells
    // away even after the fp32 rounding of the cell coordinate
    cs = fmaxf(r * 1.0001f / kSub, fmaxf(ex, ey) / 1024.f);
    nx = (int)floorf(ex / cs) + 1;
    ny = (int)floorf(ey / cs) + 1;
    nx = min(nx, 1025);
    ny = min(ny, 1025);
  }
  g[0] = ox; g[1] = oy; g[2] = 1.f / cs; g[3] = cs; g[4] = r;
  g[5] = __int_as_float(nx); g[6] = __int_as_float(ny);
}

__device__ __forceinline__ int cell_of(const float *g, float x, float y, int &cx, int &cy) {
  const int nx = __float_as_int(g[5]), ny = __float_as_int(g[6]);
  cx = min(max((int)floorf((x - g[0]) * g[2]), 0), nx - 1);
  cy = min(max((int)floorf((y - g[1]) * g[2]), 0), ny - 1);
  return cy * nx + cx;
}

// Consecutive slots are mostly points of the same box and hence the same cell: the lanes of
// a warp with equal cells are grouped (match.any) and their leader does one atomic for the
// group (the clutter scenes put ~1e4 points in a cell, so per-point atomics would serialize).
__global__ void __launch_bounds__(256) k_cell_count(const float4 *__restrict__ pts, int64_t n, const float *g,
                                                     int32_t *cell_count) {
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    int c = -1;
    if (i < n) {
      const float4 p = pts[i];
      int cx, cy;
      if (p.w > 0.f) c = cell_of(g, p.x, p.y, cx, cy);
    }
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    if (c >= 0 && lane == __ffs(grp) - 1) atomicAdd(cell_count + c, __popc(grp));
  }
}

__global__ void __launch_bounds__(256) k_cell_fill(const float4 *__restrict__ pts, int64_t n, const float *g,
                                                    const int64_t *__restrict__ cell_start, int32_t *cell_fill,
                                                    int32_t *cell_items, float2 *cell_xy) {
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    int c = -1;
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < n) {
      p = pts[i];
      int cx, cy;
      if (p.w > 0.f) c = cell_of(g, p.x, p.y, cx, cy);
    }
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    const int leader = __ffs(grp) - 1;
    int base = 0;
    if (c >= 0 && lane == leader) base = atomicAdd(cell_fill + c, __popc(grp));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (c >= 0) {
      const int64_t pos = cell_start[c] + base + __popc(grp & ((1u << lane) - 1u));
      cell_items[pos] = (int32_t)i;
      cell_xy[pos] = make_float2(p.x, p.y);
    }
  }
}

// per step: mark the slots of its partition in its bitmap row.  The (2 kSub + 1)^2 cells
// around the base are scanned in cell-sorted order (contiguous xy), cells whose rectangle is
// farther than r from the base are skipped.
__global__ void __launch_bounds__(256) k_part_mark(const float *__restrict__ q, const float *g,
                                                    const int64_t *__restrict__ cell_start,
                                                    const int32_t *__restrict__ cell_items,
                                                    const float2 *__restrict__ cell_xy, int64_t words,
                                                    uint32_t *__restrict__ bitmap) {
  const int w = blockIdx.x;
  const int nx = __float_as_int(g[5]), ny = __float_as_int(g[6]);
  if (nx == 0) return;
  const float bx = q[(int64_t)w * kNdof], by = q[(int64_t)w * kNdof + 1];
  const float ox = g[0], oy = g[1], cs = g[3];
  const float r = g[4], r2 = __fmul_rn(r, r);
  const int cx = (int)floorf((bx - ox) * g[2]), cy = (int)floorf((by - oy) * g[2]);
  uint32_t *row = bitmap + (int64_t)w * words;
  for (int dy = -kSub; dy <= kSub; ++dy) {
    const int y = cy + dy;
    if (y < 0 || y >= ny) continue;
    for (int dx = -kSub; dx <= kSub; ++dx) {
      const int x = cx + dx;
      if (x < 0 || x >= nx) continue;
      // distance from the base to the cell rectangle (with a small slack for rounding)
      const float x0 = ox + x * cs, y0 = oy + y * cs;
      const float ddx = fmaxf(fmaxf(x0 - bx, bx - (x0 + cs)), 0.f);
      const float ddy = fmaxf(fmaxf(y0 - by, by - (y0 + cs)), 0.f);
      if (ddx * ddx + ddy * ddy > r2 * 1.0002f + 1e-6f) continue;
      const int c = y * nx + x;
      for (int64_t k = cell_start[c] + threadIdx.x; k < cell_start[c + 1]; k += blockDim.x) {
        const float2 p = cell_xy[k];
        const float ex = __fsub_rn(p.x, bx), ey = __fsub_rn(p.y, by);
        if (__fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey)) <= r2) {
          const int32_t sl = cell_items[k];
          atomicOr(row + (sl >> 5), 1u << (sl & 31));
        }
      }
    }
  }
}

// popcount per (step, chunk of kPartChunkWords words)
__global__ void __launch_bounds__(256) k_chunk_count(const uint32_t *__restrict__ bitmap, int64_t words,
                                                      int64_t nchunk, int32_t *__restrict__ chunk_cnt) {
  __shared__ int64_t sh[32];
  const int w = blockIdx.y;
  const int64_t c = blockIdx.x;
  const uint32_t *row = bitmap + (int64_t)w * words;
  int64_t s = 0;
  for (int64_t k = c * kPartChunkWords + threadIdx.x; k < min((c + 1) * kPartChunkWords, words); k += blockDim.x)
    s += __popc(row[k]);
  int64_t tot;
  block_excl_scan(s, &tot, sh);
  if (threadIdx.x == 0) chunk_cnt[(int64_t)w * nchunk + c] = (int32_t)tot;
}

// ordered emission: chunk (w, c) writes its set bits' slots at chunk_off[w * nchunk + c] on
__global__ void __launch_bounds__(256) k_chunk_emit(const uint32_t *__restrict__ bitmap, int64_t words,
                                                     int64_t nchunk, const int64_t *__restrict__ chunk_off,
                                                     int32_t *__restrict__ cand, int64_t cap) {
  __shared__ int64_t sh[32];
  const int w = blockIdx.y;
  const int64_t c = blockIdx.x;
  const uint32_t *row = bitmap + (int64_t)w * words;
  constexpr int kPer = kPartChunkWords / 256;  // words per thread, consecutive
  const int64_t k0 = c * kPartChunkWords + (int64_t)threadIdx.x * kPer;
  uint32_t wv[kPer];
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    wv[i] = (k0 + i < words) ? row[k0 + i] : 0u;
    cnt += __popc(wv[i]);
  }
  int64_t tot;
  int64_t pos = chunk_off[(int64_t)w * nchunk + c] + block_excl_scan(cnt, &tot, sh);
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    uint32_t b = wv[i];
    while (b) {
      const int bit = __ffs(b) - 1;
      b &= b - 1;
      if (pos < cap) cand[pos] = (int32_t)((k0 + i) * 32 + bit);
      ++pos;
    }
  }
}

// m_i, list starts, tiles per step and their exclusive scan (single CTA); capacity guard
__global__ void __launch_bounds__(1024) k_part_tiles(const int64_t *__restrict__ chunk_off, int64_t nchunk, int32_t n_wp,
                                                      int64_t cap, int64_t *__restrict__ cand_start,
                                                      int64_t *__restrict__ cand_count, int64_t *__restrict__ tile_start,
                                                      int64_t *__restrict__ n_tiles,
                                                      unsigned long long *__restrict__ overflow) {
  __shared__ int64_t sh[32];
  const int64_t total = chunk_off[(int64_t)n_wp * nchunk];
  const bool over = total > cap;
  int64_t carry = 0;
  for (int base = 0; base < n_wp; base += blockDim.x) {
    const int w = base + threadIdx.x;
    int64_t nt = 0;
    if (w < n_wp) {
      const int64_t a = chunk_off[(int64_t)w * nchunk], b = chunk_off[(int64_t)(w + 1) * nchunk];
      cand_start[w] = a;
      cand_count[w] = b - a;
      nt = over ? 0 : (b - a + kTile - 1) / kTile;
    }
    int64_t tot;
    const int64_t ex = block_excl_scan(nt, &tot, sh);
    if (w < n_wp) tile_start[w] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    tile_start[n_wp] = carry;
    cand_start[n_wp] = total;
    *n_tiles = carry;
    if (over) *overflow = 1ull;
  }
}

__global__ void __launch_bounds__(256) k_part_tile_wp(const int64_t *__restrict__ tile_start, int32_t *__restrict__ tile_wp) {
  const int w = blockIdx.x;
  for (int64_t t = tile_start[w] + threadIdx.x; t < tile_start[w + 1]; t += blockDim.x) tile_wp[t] = w;
}

int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * 8));
}

}  // namespace

int64_t part_scan_tmp_elems(int64_t n) { return (n + 1023) / 1024 + 1; }

cudaError_t launch_part_grid(const float4 *pts, int64_t lb, float r, PartScratch ps, cudaStream_t s, int *nl) {
  k_bbox_init<<<1, 32, 0, s>>>(ps.bbox);
  if (lb > 0) k_bbox<<<grid_for(lb), 256, 0, s>>>(pts, lb, ps.bbox);
  k_grid_params<<<1, 32, 0, s>>>(ps.bbox, r, ps.grid);
  cudaMemsetAsync(ps.cell_count, 0, kPartMaxCells * sizeof(int32_t), s);
  cudaMemsetAsync(ps.cell_fill, 0, kPartMaxCells * sizeof(int32_t), s);
  *nl += 3;
  if (lb > 0) {
    k_cell_count<<<grid_for(lb), 256, 0, s>>>(pts, lb, ps.grid, ps.cell_count);
    ++*nl;
  }
  cudaError_t e = excl_scan(ps.cell_count, kPartMaxCells + 1 - 1, ps.cell_start, ps.cell_start + kPartMaxCells,
                            ps.scan_tmp, s, nl);
  if (e != cudaSuccess) return e;
  if (lb > 0) {
    k_cell_fill<<<grid_for(lb), 256, 0, s>>>(pts, lb, ps.grid, ps.cell_start, ps.cell_fill, ps.cell_items,
                                             ps.cell_xy);
    ++*nl;
  }
  return cudaGetLastError();
}

cudaError_t launch_part_build(const float4 *pts, const float *q, int32_t n_wp, float r, PartScratch ps,
                              unsigned long long *overflow, cudaStream_t s, int *nl) {
  (void)r;
  (void)pts;
  cudaMemsetAsync(ps.bitmap, 0, (size_t)n_wp * ps.words * sizeof(uint32_t), s);
  k_part_mark<<<n_wp, 256, 0, s>>>(q, ps.grid, ps.cell_start, ps.cell_items, ps.cell_xy, ps.words, ps.bitmap);
  k_chunk_count<<<dim3((unsigned)ps.nchunk, (unsigned)n_wp), 256, 0, s>>>(ps.bitmap, ps.words, ps.nchunk, ps.chunk_cnt);
  *nl += 2;
  const int64_t n = (int64_t)n_wp * ps.nchunk;
  cudaError_t e = excl_scan(ps.chunk_cnt, n, ps.chunk_off, ps.chunk_off + n, ps.scan_tmp, s, nl);
  if (e != cudaSuccess) return e;
  k_chunk_emit<<<dim3((unsigned)ps.nchunk, (unsigned)n_wp), 256, 0, s>>>(ps.bitmap, ps.words, ps.nchunk, ps.chunk_off,
                                                                          ps.cand, ps.max_candidates);
  k_part_tiles<<<1, 1024, 0, s>>>(ps.chunk_off, ps.nchunk, n_wp, ps.max_candidates, ps.cand_start, ps.cand_count,
                                  ps.tile_start, ps.n_tiles, overflow);
  k_part_tile_wp<<<n_wp, 256, 0, s>>>(ps.tile_start, ps.tile_wp);
  *nl += 3;
  return cudaGetLastError();
}

}  // namespace gcdf
