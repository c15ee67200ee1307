// k_compact.cu -- K3: threshold + per-waypoint min + stream compaction (A6-A8), the
// finalize pass that turns per-tile staging into the canonical (wp, pt) order, and the
// multi-rank merge of gathered active sets.
//
// Paper: constraint f - delta >= 0, active test R12; union = min
// (PAPER.md:164); c_gcdf "indexed by time step" (Eq. 14).
//
// Min keys: key = ord(f) << 32 | pt, ord() order-preserving float -> uint32, so the
// unsigned minimum is (min f, smallest id on ties) -- one atomicMin per tile.
#include "gcdf_internal.h"
#include "k_scan.cuh"

namespace gcdf {
namespace {

__device__ __forceinline__ unsigned ord_f32(float f) {
  unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(unsigned o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

__global__ void k_detect_init(unsigned long long *wp_key, unsigned long long *counter, int32_t n_wp) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_wp; i += gridDim.x * blockDim.x) wp_key[i] = ~0ull;
  if (blockIdx.x == 0 && threadIdx.x < 2) counter[threadIdx.x] = 0ull;
}


// K3 standalone over dense values: one WARP per tile of 128 slots, 4 slots per lane
// (one 16-B streaming load), no block barrier.  The tile's actives are ranked in slot
// order by a warp prefix scan of per-lane counts (the "warp-ballot and prefix-sum"
// compaction); the per-waypoint min key is a warp-shuffle min + one atomicMin per tile.
// A value of +INF marks a dead slot (gcdf_query_values_grads writes +INF there).
__global__ void __launch_bounds__(256) k_compact_dense(const float *__restrict__ values,
                                                      const float *__restrict__ grads, int64_t stride,
                                                      int32_t n_wp, int32_t tpw, SceneView scene, float delta,
                                                      float tau, DetectScratch ds) {
  const int lane = threadIdx.x & 31;
  const int64_t n_tiles = (int64_t)n_wp * tpw;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t lb = scene.local_bound;
  for (int64_t T = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); T < n_tiles; T += wstride) {
    const int w = (int)(T / tpw);
    const int64_t slot0 = (T - (int64_t)w * tpw) * kTile + 4 * lane;
    const float *vrow = values + (int64_t)w * stride;
    float v[4];
    if (slot0 + 3 < lb) {
      const float4 x = __ldcs(reinterpret_cast<const float4 *>(vrow + slot0));
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = slot0 + k < lb ? vrow[slot0 + k] : __int_as_float(0x7f800000);
    }
    unsigned bits = 0u;
    unsigned long long key = ~0ull;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool live = v[k] != __int_as_float(0x7f800000);
      if (live && v[k] - delta <= tau) bits |= 1u << k;
      if (live) {
        const unsigned long long kk = ((unsigned long long)ord_f32(v[k]) << 32) |
                                      (unsigned long long)local_to_global(slot0 + k, scene.rank, scene.world);
        key = kk < key ? kk : key;
      }
    }
    const int cnt = __popc(bits);
    int incl = cnt;  // warp inclusive scan of the per-lane counts (slot order)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other < key ? other : key;
    }
    int base = 0;
    if (lane == 0) {
      if (key != ~0ull) atomicMin(ds.wp_key + w, key);
      if (total > 0) {
        const unsigned long long b = atomicAdd(ds.counter, (unsigned long long)total);
        if (b + total > (unsigned long long)ds.max_active) {
          atomicOr(ds.counter + 1, 1ull);
          base = -1;
        } else {
          base = (int)b;
        }
      }
      ds.tile_meta[T] = make_int2(base, total);
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    if (bits && base >= 0) {
      int r = base + incl - cnt;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!((bits >> k) & 1u)) continue;
        const int64_t slot = slot0 + k;
        const float *g = grads + ((int64_t)w * stride + slot) * kNdof;
        float4 *dst = reinterpret_cast<float4 *>(ds.staging + r);
        dst[0] = make_float4(v[k], g[0], g[1], g[2]);
        dst[1] = make_float4(g[3], g[4], g[5], g[6]);
        dst[2] = make_float4(g[7], g[8], __uint_as_float((unsigned)w),
                             __uint_as_float((unsigned)local_to_global(slot, scene.rank, scene.world)));
        ++r;
      }
    }
  }
}

// per-waypoint active counts from the tile meta
__global__ void __launch_bounds__(256) k_wp_count(const int2 *__restrict__ meta, int32_t tpw,
                                                  const int64_t *__restrict__ tile_start,
                                                  int64_t *__restrict__ wp_count) {
  __shared__ int64_t sh[32];
  const int w = blockIdx.x;
  const int64_t t0 = tile_start ? tile_start[w] : (int64_t)w * tpw;
  const int64_t nt = tile_start ? tile_start[w + 1] - t0 : tpw;
  int64_t s = 0;
  for (int64_t t = threadIdx.x; t < nt; t += blockDim.x) s += meta[t0 + t].y;
  int64_t tot;
  block_excl_scan(s, &tot, sh);
  if (threadIdx.x == 0) wp_count[w] = tot;
}

// exclusive scan over waypoints + min/argmin/key export (single CTA)
__global__ void __launch_bounds__(1024) k_wp_scan(const int64_t *__restrict__ wp_count, int32_t n_wp,
                                                  int64_t *__restrict__ wp_offsets, int64_t *__restrict__ count,
                                                  const unsigned long long *__restrict__ keys, float *wp_min,
                                                  int64_t *wp_argmin, int64_t *wp_key_out) {
  __shared__ int64_t sh[32];
  int64_t carry = 0;
  for (int base = 0; base < n_wp; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int64_t v = i < n_wp ? wp_count[i] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan(v, &tot, sh);
    if (i < n_wp) wp_offsets[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    wp_offsets[n_wp] = carry;
    *count = carry;
  }
  if (keys) {
    for (int i = threadIdx.x; i < n_wp; i += blockDim.x) {
      const unsigned long long k = keys[i];
      if (wp_min) wp_min[i] = k == ~0ull ? __int_as_float(0x7f800000) : unord_f32((unsigned)(k >> 32));
      if (wp_argmin) wp_argmin[i] = k == ~0ull ? -1 : (int64_t)(k & 0xffffffffull);
      if (wp_key_out) wp_key_out[i] = (int64_t)(k ^ 0x8000000000000000ull);
    }
  }
}

// ordered copy staging -> out: one CTA per waypoint, tiles scanned in order
__global__ void __launch_bounds__(256) k_wp_scatter(const int2 *__restrict__ meta, int32_t tpw,
                                                    const int64_t *__restrict__ tile_start,
                                                    const gcdf_active_t *__restrict__ staging,
                                                    const int64_t *__restrict__ wp_offsets,
                                                    gcdf_active_t *__restrict__ out, int64_t cap) {
  __shared__ int64_t sh[32];
  const int w = blockIdx.x;
  const int64_t tb = tile_start ? tile_start[w] : (int64_t)w * tpw;
  const int64_t nt = tile_start ? tile_start[w + 1] - tb : tpw;
  int64_t carry = wp_offsets[w];
  for (int64_t t0 = 0; t0 < nt; t0 += blockDim.x) {
    const int64_t t = t0 + threadIdx.x;
    int2 m = make_int2(0, 0);
    if (t < nt) m = meta[tb + t];
    int64_t tot;
    const int64_t ex = block_excl_scan(m.y, &tot, sh);
    if (m.y > 0 && m.x >= 0) {
      const float4 *src = reinterpret_cast<const float4 *>(staging + m.x);
      for (int k = 0; k < m.y; ++k) {
        const int64_t o = carry + ex + k;
        if (o < cap) {
          float4 *dst = reinterpret_cast<float4 *>(out + o);
          dst[0] = src[3 * k];
          dst[1] = src[3 * k + 1];
          dst[2] = src[3 * k + 2];
        }
      }
    }
    carry += tot;
  }
}

// ---- multi-rank merge ----
__global__ void k_merge_offsets(int32_t world, int32_t n_wp, const int64_t *__restrict__ offsets,
                                int64_t *__restrict__ wp_offsets, int64_t *__restrict__ count) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w <= n_wp; w += gridDim.x * blockDim.x) {
    int64_t s = 0;
    for (int r = 0; r < world; ++r) s += offsets[(int64_t)r * (n_wp + 1) + w];
    wp_offsets[w] = s;
    if (w == n_wp) *count = s;
  }
}

__global__ void k_merge_records(int32_t world, int32_t n_wp, const gcdf_active_t *__restrict__ recs,
                                int64_t rec_stride, const int64_t *__restrict__ offsets,
                                const int64_t *__restrict__ wp_offsets, gcdf_active_t *__restrict__ out,
                                int64_t cap) {
  const int r = blockIdx.y;
  const int64_t *off = offsets + (int64_t)r * (n_wp + 1);
  const int64_t n = off[n_wp];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    // waypoint of record k: last w with off[w] <= k
    int lo = 0, hi = n_wp - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[mid] <= k) lo = mid; else hi = mid - 1;
    }
    const int w = lo;
    const gcdf_active_t rec = recs[(int64_t)r * rec_stride + k];
    int64_t pos = wp_offsets[w] + (k - off[w]);
    for (int s = 0; s < world; ++s) {
      if (s == r) continue;
      const int64_t *os = offsets + (int64_t)s * (n_wp + 1);
      int64_t a = os[w], b = os[w + 1];  // count records of rank s in wp w with pt < rec.pt
      const gcdf_active_t *rs = recs + (int64_t)s * rec_stride;
      while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (rs[mid].pt < rec.pt) a = mid + 1; else b = mid;
      }
      pos += a - os[w];
    }
    if (pos < cap) out[pos] = rec;
  }
}

__global__ void k_keys_export(const int64_t *__restrict__ skeys, int32_t n_wp, float *wp_min, int64_t *wp_argmin) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_wp; i += gridDim.x * blockDim.x) {
    const unsigned long long k = (unsigned long long)skeys[i] ^ 0x8000000000000000ull;
    if (wp_min) wp_min[i] = k == ~0ull ? __int_as_float(0x7f800000) : unord_f32((unsigned)(k >> 32));
    if (wp_argmin) wp_argmin[i] = k == ~0ull ? -1 : (int64_t)(k & 0xffffffffull);
  }
}

// NEXT-2 (Eq. 14-19, reading R18): c[k] = f_k - delta; CSR row k = the 9 gradient entries
// of record k at columns 2 * 9 * wp_k + t; row_ptr[k] = 9 k.  count read on the device.
__global__ void __launch_bounds__(256) k_sparse_jacobian(const gcdf_active_t *__restrict__ recs,
                                                          const int64_t *__restrict__ count_dev, int64_t cap,
                                                          float delta, float *__restrict__ c,
                                                          int64_t *__restrict__ row_ptr, int32_t *__restrict__ col,
                                                          float *__restrict__ val) {
  const int64_t n = min(*count_dev, cap);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= n; k += (int64_t)gridDim.x * blockDim.x) {
    row_ptr[k] = (int64_t)kNdof * k;
    if (k == n) break;
    const float4 *r = reinterpret_cast<const float4 *>(recs + k);
    const float4 a = r[0], b = r[1], d = r[2];
    const float g[kNdof] = {a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y};
    const int32_t base = 2 * kNdof * (int32_t)__float_as_uint(d.z);
    if (c) c[k] = a.x - delta;
#pragma unroll
    for (int t = 0; t < kNdof; ++t) {
      col[(int64_t)kNdof * k + t] = base + t;
      val[(int64_t)kNdof * k + t] = g[t];
    }
  }
}

}  // namespace

cudaError_t launch_sparse_jacobian(const gcdf_active_t *recs, const int64_t *count, int64_t cap, float delta,
                                   float *c, int64_t *row_ptr, int32_t *col, float *val, int num_sms,
                                   cudaStream_t s) {
  k_sparse_jacobian<<<num_sms * 4, 256, 0, s>>>(recs, count, cap, delta, c, row_ptr, col, val);
  return cudaGetLastError();
}

cudaError_t launch_detect_init(DetectScratch ds, int32_t n_wp, cudaStream_t s) {
  int grid = (n_wp + 255) / 256;
  if (grid < 1) grid = 1;
  k_detect_init<<<grid, 256, 0, s>>>(ds.wp_key, ds.counter, n_wp);
  return cudaGetLastError();
}

cudaError_t launch_compact_dense(const float *values, const float *grads, int64_t stride, int32_t n_wp,
                                 int32_t tiles_per_wp, SceneView scene, float delta, float tau,
                                 DetectScratch ds, cudaStream_t s) {
  const int64_t n_tiles = (int64_t)n_wp * tiles_per_wp;
  if (n_tiles <= 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (n_tiles + 7) / 8;  // 8 warps (tiles) per CTA, 8 CTAs per SM
  const int64_t grid = need < (int64_t)sms * 8 ? need : (int64_t)sms * 8;
  k_compact_dense<<<(unsigned)grid, 256, 0, s>>>(values, grads, stride, n_wp, tiles_per_wp, scene, delta, tau, ds);
  return cudaGetLastError();
}

cudaError_t launch_finalize(DetectScratch ds, int32_t n_wp, int32_t tiles_per_wp, const int64_t *tile_start,
                            gcdf_active_t *out,
                            int64_t out_capacity, int64_t *wp_offsets, float *wp_min, int64_t *wp_argmin,
                            int64_t *wp_key, int64_t *count, int64_t *wp_count_scratch, cudaStream_t s,
                            int *n_launches) {
  if (n_wp <= 0) return cudaSuccess;
  k_wp_count<<<n_wp, 256, 0, s>>>(ds.tile_meta, tiles_per_wp, tile_start, wp_count_scratch);
  k_wp_scan<<<1, 1024, 0, s>>>(wp_count_scratch, n_wp, wp_offsets, count, ds.wp_key, wp_min, wp_argmin, wp_key);
  k_wp_scatter<<<n_wp, 256, 0, s>>>(ds.tile_meta, tiles_per_wp, tile_start, ds.staging, wp_offsets, out,
                                    out_capacity);
  *n_launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_merge(int32_t world, int32_t n_wp, const gcdf_active_t *recs, int64_t rec_stride,
                         const int64_t *offsets, const int64_t *wp_key, gcdf_active_t *out, int64_t out_capacity,
                         int64_t *wp_offsets, float *wp_min, int64_t *wp_argmin, int64_t *count, cudaStream_t s,
                         int *n_launches) {
  int g = (n_wp + 1 + 255) / 256;
  k_merge_offsets<<<g, 256, 0, s>>>(world, n_wp, offsets, wp_offsets, count);
  int gx = (int)((rec_stride + 255) / 256);
  if (gx > 2048) gx = 2048;
  if (gx < 1) gx = 1;
  k_merge_records<<<dim3(gx, world), 256, 0, s>>>(world, n_wp, recs, rec_stride, offsets, wp_offsets, out,
                                                   out_capacity);
  k_keys_export<<<(n_wp + 255) / 256 > 0 ? (n_wp + 255) / 256 : 1, 256, 0, s>>>(wp_key, n_wp, wp_min, wp_argmin);
  *n_launches += 3;
  return cudaGetLastError();
}

}  // namespace gcdf
