// k_compact.cu -- K3: threshold + per-waypoint min + stream compaction (A6-A8), the
// finalize pass that turns per-tile staging into the canonical (wp, pt) order, and the
// multi-rank merge of gathered active sets.
//
// Paper: constraint f - delta >= 0, active test R12; union = min
// (PAPER.md:164); c_gcdf "indexed by time step" (Eq. 14).
//
// Min keys: key = ord(f) << 32 | pt, ord() order-preserving float -> uint32, so the
// unsigned minimum is (min f, smallest id on ties) -- one atomicMin per tile.
#include <algorithm>

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


// ---- standalone K3 (A6-A8 over dense values): ONE pass, decoupled look-back.
// A partition = kLbWarps warps x kLbTW consecutive tiles (128 slots, 4 per lane, one 16-B
// streaming load each) of the flat (step, tile) order; partitions are taken in order from
// a global counter, so a partition only ever waits on partitions already running.  Each
// warp ballots its tiles' actives (f - delta <= tau; dead slots hold +INF and never pass)
// and folds the per-step minimum key; the CTA publishes its active count, looks back over
// the predecessors' published counts / inclusive prefixes (32 at a time, one per lane) for
// its exclusive prefix, publishes its own inclusive prefix, and the lanes with actives read
// their 36-B gradient rows and write their records straight to their final positions --
// the values are read once, the gradients only for actives, nothing else touches HBM.
// Records in (step, slot) order = the canonical (wp, pt) order; wp_offsets[w] is the prefix
// at the step's first tile.
constexpr int kLbWarps = 8, kLbTW = 4, kLbTiles = kLbWarps * kLbTW;
// status word of a partition: [63:40] call epoch, [39:38] 1 = count, 2 = inclusive prefix, [37:0] value
constexpr int kLbAgg = 1, kLbPre = 2;
__device__ __forceinline__ unsigned long long lb_word(uint32_t epoch, int flag, int64_t v) {
  return ((unsigned long long)(epoch & 0xffffffu) << 40) | ((unsigned long long)flag << 38) | (unsigned long long)v;
}
__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// values of tile tw (0-based within step w) for this lane's 4 slots (+INF outside the scene)
__device__ __forceinline__ float4 load_tile_values(const float *__restrict__ values, int64_t stride, int64_t lb,
                                                   int w, int64_t tw, int lane) {
  const int64_t slot0 = tw * kTile + 4 * lane;
  const float *vrow = values + (int64_t)w * stride;
  const float inf = __int_as_float(0x7f800000);
  float4 v = make_float4(inf, inf, inf, inf);
  if (slot0 + 3 < lb) {
    v = __ldcs(reinterpret_cast<const float4 *>(vrow + slot0));
  } else {
    float *pv = reinterpret_cast<float *>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) if (slot0 + k < lb) pv[k] = vrow[slot0 + k];
  }
  return v;
}

__global__ void __launch_bounds__(256) k_compact_lookback(const float *__restrict__ values,
                                                          const float *__restrict__ grads, int64_t stride,
                                                          int32_t n_wp, int32_t tpw, SceneView scene, float delta,
                                                          float tau, unsigned long long *__restrict__ wp_key,
                                                          unsigned long long *part_ctr, unsigned long long *status,
                                                          uint32_t epoch, gcdf_active_t *__restrict__ out, int64_t cap,
                                                          int64_t *__restrict__ wp_offsets, int64_t *__restrict__ count) {
  __shared__ int64_t s_part, s_excl;
  __shared__ int32_t s_wcnt[kLbWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_part = (int64_t)atomicAdd(part_ctr, 1ull);
  __syncthreads();
  const int64_t p = s_part;
  const int64_t n_tiles = (int64_t)n_wp * tpw;
  const int64_t T0 = p * kLbTiles + (int64_t)warp * kLbTW;  // this warp's first flat tile
  const int64_t lb = scene.local_bound;
  const uint32_t lt = (1u << lane) - 1u;
  int w0 = (int)(T0 / tpw);
  int t0 = (int)(T0 - (int64_t)w0 * tpw);
  // ---- loads: the warp's kLbTW tiles, all in flight
  float4 v[kLbTW];
  {
    int w = w0, t = t0;
#pragma unroll
    for (int i = 0; i < kLbTW; ++i) {
      if (T0 + i < n_tiles) v[i] = load_tile_values(values, stride, lb, w, t, lane);
      if (++t == tpw) { t = 0; ++w; }
    }
  }
  // ---- ballots, counts, per-step minimum (one atomicMin per step run of the warp)
  uint32_t bits[kLbTW];  // this lane's 4 active flags per tile (bit k = slot 4 lane + k)
  int below[kLbTW];      // actives of the lower lanes in the tile
  int cnt[kLbTW];        // actives of the tile
  int wtot = 0;
  {
    int w = w0, t = t0;
    unsigned long long key = ~0ull;
    int wk = w0;
    auto flush = [&]() {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
        key = other < key ? other : key;
      }
      if (lane == 0 && key != ~0ull) atomicMin(wp_key + wk, key);
      key = ~0ull;
    };
#pragma unroll
    for (int i = 0; i < kLbTW; ++i) {
      bits[i] = 0u;
      below[i] = cnt[i] = 0;
      if (T0 + i < n_tiles) {  // (uniform over the warp)
        if (w != wk) {
          flush();
          wk = w;
        }
        const float x[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t b = __ballot_sync(0xffffffffu, x[k] - delta <= tau);
          bits[i] |= ((b >> lane) & 1u) << k;
          below[i] += __popc(b & lt);
          cnt[i] += __popc(b);
        }
        // minimum of the lane's four (first slot on ties), as a key with the global id
        const float m4 = fminf(fminf(x[0], x[1]), fminf(x[2], x[3]));
        if (m4 != __int_as_float(0x7f800000)) {
          const int kk = x[0] == m4 ? 0 : x[1] == m4 ? 1 : x[2] == m4 ? 2 : 3;
          const unsigned long long kx =
              ((unsigned long long)ord_f32(m4) << 32) |
              (unsigned long long)local_to_global((int64_t)t * kTile + 4 * lane + kk, scene.rank, scene.world);
          key = kx < key ? kx : key;
        }
        wtot += cnt[i];
      }
      if (++t == tpw) { t = 0; ++w; }
    }
    flush();
  }
  if (lane == 0) s_wcnt[warp] = wtot;
  __syncthreads();
  // ---- decoupled look-back (warp 0): exclusive prefix of this partition
  if (warp == 0) {
    int64_t agg = 0;
#pragma unroll
    for (int j = 0; j < kLbWarps; ++j) agg += s_wcnt[j];
    unsigned long long *const st = status + p;
    if (p == 0) {
      if (lane == 0) st_release(st, lb_word(epoch, kLbPre, agg));
      if (lane == 0) s_excl = 0;
    } else {
      if (lane == 0) st_release(st, lb_word(epoch, kLbAgg, agg));
      int64_t excl = 0;
      for (int64_t base = p - 1;; base -= 32) {
        const int64_t idx = base - lane;
        unsigned long long wd = lb_word(epoch, kLbPre, 0);  // (idx < 0: never reached past partition 0)
        if (idx >= 0) {
          do {
            wd = ld_acquire(status + idx);
          } while ((uint32_t)(wd >> 40) != (epoch & 0xffffffu) || ((wd >> 38) & 3u) == 0u);
        }
        __syncwarp();
        const unsigned pm = __ballot_sync(0xffffffffu, ((wd >> 38) & 3u) == (unsigned)kLbPre);
        const int stop = pm ? __ffs(pm) - 1 : 32;
        int64_t val = lane <= stop ? (int64_t)(wd & ((1ull << 38) - 1ull)) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        excl += val;
        if (pm) break;
      }
      if (lane == 0) {
        st_release(st, lb_word(epoch, kLbPre, excl + agg));
        s_excl = excl;
      }
    }
  }
  __syncthreads();
  int64_t pos = s_excl;
  for (int j = 0; j < warp; ++j) pos += s_wcnt[j];
  // ---- offsets and records
  int w = w0, t = t0;
#pragma unroll
  for (int i = 0; i < kLbTW; ++i) {
    const int64_t T = T0 + i;
    if (T < n_tiles) {
      if (t == 0 && lane == 0) wp_offsets[w] = pos;
      if (T == n_tiles - 1 && lane == 0) {
        wp_offsets[n_wp] = pos + cnt[i];
        *count = pos + cnt[i];
      }
      unsigned b = bits[i];
      int64_t r = pos + below[i];
      while (b) {  // (a lane has ~0.04 actives per tile at 1 % active)
        const int k = __ffs(b) - 1;
        b &= b - 1u;
        const float xk = k == 0 ? v[i].x : k == 1 ? v[i].y : k == 2 ? v[i].z : v[i].w;
        const int64_t slot = (int64_t)t * kTile + 4 * lane + k;
        if (r < cap) {
          const float *g = grads + ((int64_t)w * stride + slot) * kNdof;
          float gg[kNdof];
#pragma unroll
          for (int e = 0; e < kNdof; ++e) gg[e] = __ldcs(g + e);
          float4 *dst = reinterpret_cast<float4 *>(out + r);
          dst[0] = make_float4(xk, gg[0], gg[1], gg[2]);
          dst[1] = make_float4(gg[3], gg[4], gg[5], gg[6]);
          dst[2] = make_float4(gg[7], gg[8], __uint_as_float((unsigned)w),
                               __uint_as_float((unsigned)local_to_global(slot, scene.rank, scene.world)));
        }
        ++r;
      }
      pos += cnt[i];
    }
    if (++t == tpw) { t = 0; ++w; }
  }
}

// per-step min / argmin / key export of the standalone K3; with no tile at all (empty
// scene) also the zero offsets and count
__global__ void k_compact_keys(const unsigned long long *__restrict__ keys, int32_t n_wp, bool no_tiles,
                               float *wp_min, int64_t *wp_argmin, int64_t *wp_key_out, int64_t *wp_offsets,
                               int64_t *count) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w <= n_wp; w += gridDim.x * blockDim.x) {
    if (no_tiles) {
      wp_offsets[w] = 0;
      if (w == n_wp) *count = 0;
    }
    if (w == n_wp) continue;
    const unsigned long long k = keys[w];
    if (wp_min) wp_min[w] = k == ~0ull ? __int_as_float(0x7f800000) : unord_f32((unsigned)(k >> 32));
    if (wp_argmin) wp_argmin[w] = k == ~0ull ? -1 : (int64_t)(k & 0xffffffffull);
    if (wp_key_out) wp_key_out[w] = (int64_t)(k ^ 0x8000000000000000ull);
  }
}

// ---- finalize: per-tile (staging base, count) -> ordered output.  Tiles of step w are
// [t0(w), t0(w) + nt(w)) (tile_start, or w * tpw); each step's tiles are split into chunks of
// kFinChunk tiles (8 per thread) and every (step, chunk) is one CTA, so the ordered copy runs
// on n_wp * nch CTAs instead of n_wp.
constexpr int kFinPer = 8;
constexpr int kFinChunk = 256 * kFinPer;

__device__ __forceinline__ void tile_range(const int64_t *tile_start, int32_t tpw, int w, int64_t &t0, int64_t &nt) {
  t0 = tile_start ? tile_start[w] : (int64_t)w * tpw;
  nt = tile_start ? tile_start[w + 1] - t0 : tpw;
}

// record count of chunk (w, c) -> csum[w * nch + c]
__global__ void __launch_bounds__(256) k_fin_count(const int2 *__restrict__ meta, int32_t tpw,
                                                   const int64_t *__restrict__ tile_start, int64_t nch,
                                                   int64_t *__restrict__ csum) {
  __shared__ int64_t sh[32];
  const int w = blockIdx.y;
  const int64_t c = blockIdx.x;
  int64_t t0, nt;
  tile_range(tile_start, tpw, w, t0, nt);
  int64_t s = 0;
  const int64_t b = c * kFinChunk + (int64_t)threadIdx.x * kFinPer;
#pragma unroll
  for (int i = 0; i < kFinPer; ++i)
    if (b + i < nt) s += meta[t0 + b + i].y;
  int64_t tot;
  block_excl_scan(s, &tot, sh);
  if (threadIdx.x == 0) csum[(int64_t)w * nch + c] = tot;
}

// wp_offsets from the chunk prefix, count, min / argmin / key export
__global__ void __launch_bounds__(256) k_fin_offsets(const int64_t *__restrict__ cpre, int64_t nch, int32_t n_wp,
                                                     int64_t *__restrict__ wp_offsets, int64_t *__restrict__ count,
                                                     const unsigned long long *__restrict__ keys, float *wp_min,
                                                     int64_t *wp_argmin, int64_t *wp_key_out) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w <= n_wp; w += gridDim.x * blockDim.x) {
    wp_offsets[w] = cpre[(int64_t)w * nch];  // cpre[n_wp * nch] = the total
    if (w == n_wp) {
      *count = cpre[(int64_t)n_wp * nch];
      continue;
    }
    if (keys) {
      const unsigned long long k = keys[w];
      if (wp_min) wp_min[w] = k == ~0ull ? __int_as_float(0x7f800000) : unord_f32((unsigned)(k >> 32));
      if (wp_argmin) wp_argmin[w] = k == ~0ull ? -1 : (int64_t)(k & 0xffffffffull);
      if (wp_key_out) wp_key_out[w] = (int64_t)(k ^ 0x8000000000000000ull);
    }
  }
}

// ordered copy staging -> out for chunk (w, c), starting at cpre[w * nch + c]: each thread
// copies the records of its 8 tiles (~1 % of 128 pairs each are active: a few records)
__global__ void __launch_bounds__(256) k_fin_scatter(const int2 *__restrict__ meta, int32_t tpw,
                                                     const int64_t *__restrict__ tile_start, int64_t nch,
                                                     const int64_t *__restrict__ cpre,
                                                     const gcdf_active_t *__restrict__ staging,
                                                     gcdf_active_t *__restrict__ out, int64_t cap) {
  __shared__ int64_t sh[32];
  const int w = blockIdx.y;
  const int64_t c = blockIdx.x;
  int64_t t0, nt;
  tile_range(tile_start, tpw, w, t0, nt);
  if (c * kFinChunk >= nt) return;  // (uniform over the block)
  const int64_t b = c * kFinChunk + (int64_t)threadIdx.x * kFinPer;
  int2 m[kFinPer];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kFinPer; ++i) {
    m[i] = b + i < nt ? meta[t0 + b + i] : make_int2(0, 0);
    s += m[i].y;
  }
  int64_t tot;
  int64_t pos = cpre[(int64_t)w * nch + c] + block_excl_scan(s, &tot, sh);
#pragma unroll
  for (int i = 0; i < kFinPer; ++i) {
    if (m[i].y > 0 && m[i].x >= 0) {
      const float4 *src = reinterpret_cast<const float4 *>(staging + m[i].x);
      for (int k = 0; k < m[i].y; ++k) {
        const int64_t o = pos + k;
        if (o < cap) {
          float4 *dst = reinterpret_cast<float4 *>(out + o);
          dst[0] = src[3 * k];
          dst[1] = src[3 * k + 1];
          dst[2] = src[3 * k + 2];
        }
      }
    }
    pos += m[i].y;
  }
}

// ---- multi-rank merge ----
// Rank r's gathered pieces: offsets at offsets[r * off_stride + 0..n_wp] (its wp_offsets),
// per-waypoint keys at keys[r * key_stride + 0..n_wp-1] (key_stride 0: one already-reduced
// key array), records at recs[r * rec_stride + k] for k < min(its count, rec_stride).
// k_merge_offsets: merged wp_offsets / count (sums over ranks), the MIN of the keys
// (global min / smallest-id argmin) and a rank whose count exceeds rec_stride -> *overflow.
__global__ void k_merge_offsets(int32_t world, int32_t n_wp, const int64_t *__restrict__ offsets, int64_t off_stride,
                                const int64_t *__restrict__ keys, int64_t key_stride, int64_t rec_stride,
                                int64_t *__restrict__ wp_offsets, int64_t *__restrict__ count, int64_t *wp_key,
                                float *wp_min, int64_t *wp_argmin, unsigned long long *overflow) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w <= n_wp; w += gridDim.x * blockDim.x) {
    int64_t s = 0;
    for (int r = 0; r < world; ++r) s += offsets[(int64_t)r * off_stride + w];
    wp_offsets[w] = s;
    if (w == n_wp) {
      *count = s;
      for (int r = 0; r < world; ++r)
        if (overflow && offsets[(int64_t)r * off_stride + n_wp] > rec_stride) atomicOr(overflow, 1ull);
      continue;
    }
    int64_t key = keys[w];
    for (int r = 1; r < world && key_stride; ++r) key = min(key, keys[(int64_t)r * key_stride + w]);
    if (wp_key) wp_key[w] = key;
    const unsigned long long k = (unsigned long long)key ^ 0x8000000000000000ull;
    if (wp_min) wp_min[w] = k == ~0ull ? __int_as_float(0x7f800000) : unord_f32((unsigned)(k >> 32));
    if (wp_argmin) wp_argmin[w] = k == ~0ull ? -1 : (int64_t)(k & 0xffffffffull);
  }
}

// Every rank's records are in canonical (wp, pt) order over its own ids; record k of rank r
// in waypoint w goes to wp_offsets[w] + (k - off_r[w]) + (number of records of the other
// ranks in w with a smaller id), found by binary search -- the merged set equals the
// single-rank result bit for bit (ids are unique across ranks).
__global__ void k_merge_records(int32_t world, int32_t n_wp, const gcdf_active_t *__restrict__ recs,
                                int64_t rec_stride, const int64_t *__restrict__ offsets, int64_t off_stride,
                                const int64_t *__restrict__ wp_offsets, gcdf_active_t *__restrict__ out,
                                int64_t cap) {
  const int r = blockIdx.y;
  const int64_t *off = offsets + (int64_t)r * off_stride;
  const int64_t n = min(off[n_wp], rec_stride);  // (a truncated rank is flagged by k_merge_offsets)
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
      const int64_t *os = offsets + (int64_t)s * off_stride;
      const int64_t a0 = min(os[w], rec_stride);
      int64_t a = a0, b = min(os[w + 1], rec_stride);  // records of rank s in wp w with pt < rec.pt
      const gcdf_active_t *rs = recs + (int64_t)s * rec_stride;
      while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (rs[mid].pt < rec.pt) a = mid + 1; else b = mid;
      }
      pos += a - a0;
    }
    if (pos < cap) out[pos] = rec;
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

int64_t finalize_chunks(int64_t max_tiles_per_wp) { return std::max<int64_t>(1, (max_tiles_per_wp + kFinChunk - 1) / kFinChunk); }

cudaError_t launch_compact_dense(const float *values, const float *grads, int64_t stride, int32_t n_wp,
                                 int32_t tiles_per_wp, SceneView scene, float delta, float tau,
                                 DetectScratch ds, gcdf_active_t *out, int64_t out_capacity, int64_t *wp_offsets,
                                 float *wp_min, int64_t *wp_argmin, int64_t *wp_key, int64_t *count,
                                 uint32_t epoch, cudaStream_t s, int *n_launches) {
  const int64_t n_tiles = (int64_t)n_wp * tiles_per_wp;
  const int64_t n_parts = (n_tiles + kLbTiles - 1) / kLbTiles;
  // the partition counter is ds.counter[0] (zeroed by k_detect_init); the status words live
  // in the tile-bitmap scratch (16 B per tile >= 8 B per partition) and carry the call epoch
  if (n_parts > 0)
    k_compact_lookback<<<(unsigned)n_parts, kLbWarps * 32, 0, s>>>(
        values, grads, stride, n_wp, tiles_per_wp, scene, delta, tau, ds.wp_key, ds.counter,
        reinterpret_cast<unsigned long long *>(ds.tile_bits), epoch, out, out_capacity, wp_offsets, count);
  k_compact_keys<<<(n_wp + 256) / 256, 256, 0, s>>>(ds.wp_key, n_wp, n_parts == 0, wp_min, wp_argmin, wp_key,
                                                    wp_offsets, count);
  *n_launches += n_parts > 0 ? 2 : 1;
  return cudaGetLastError();
}


cudaError_t launch_finalize(DetectScratch ds, int32_t n_wp, int32_t tiles_per_wp, const int64_t *tile_start,
                            int64_t max_tiles_per_wp, gcdf_active_t *out, int64_t out_capacity, int64_t *wp_offsets,
                            float *wp_min, int64_t *wp_argmin, int64_t *wp_key, int64_t *count, int64_t *fin_scratch,
                            cudaStream_t s, int *n_launches) {
  if (n_wp <= 0) return cudaSuccess;
  const int64_t nch = finalize_chunks(tile_start ? max_tiles_per_wp : tiles_per_wp);
  const int64_t n = (int64_t)n_wp * nch;
  int64_t *csum = fin_scratch, *cpre = fin_scratch + n, *tmp = fin_scratch + 2 * n + 1;
  const dim3 grid((unsigned)nch, (unsigned)n_wp);
  k_fin_count<<<grid, 256, 0, s>>>(ds.tile_meta, tiles_per_wp, tile_start, nch, csum);
  cudaError_t e = excl_scan(csum, n, cpre, cpre + n, tmp, s, n_launches);
  if (e != cudaSuccess) return e;
  k_fin_offsets<<<(n_wp + 256) / 256, 256, 0, s>>>(cpre, nch, n_wp, wp_offsets, count, ds.wp_key, wp_min, wp_argmin,
                                                   wp_key);
  k_fin_scatter<<<grid, 256, 0, s>>>(ds.tile_meta, tiles_per_wp, tile_start, nch, cpre, ds.staging, out, out_capacity);
  *n_launches += 3;
  return cudaGetLastError();
}

int64_t finalize_scratch_elems(int64_t max_wp, int64_t max_tiles_per_wp) {
  const int64_t n = max_wp * finalize_chunks(max_tiles_per_wp);
  return 2 * n + 1 + (n + 1023) / 1024 + 1;
}

cudaError_t launch_merge(int32_t world, int32_t n_wp, const gcdf_active_t *recs, int64_t rec_stride,
                         const int64_t *offsets, int64_t off_stride, const int64_t *keys, int64_t key_stride,
                         gcdf_active_t *out, int64_t out_capacity, int64_t *wp_offsets, float *wp_min,
                         int64_t *wp_argmin, int64_t *wp_key, int64_t *count, unsigned long long *overflow,
                         cudaStream_t s, int *n_launches) {
  int g = (n_wp + 1 + 255) / 256;
  k_merge_offsets<<<g, 256, 0, s>>>(world, n_wp, offsets, off_stride, keys, key_stride, rec_stride, wp_offsets, count,
                                    wp_key, wp_min, wp_argmin, overflow);
  int gx = (int)((rec_stride + 255) / 256);
  if (gx > 2048) gx = 2048;
  if (gx < 1) gx = 1;
  k_merge_records<<<dim3(gx, world), 256, 0, s>>>(world, n_wp, recs, rec_stride, offsets, off_stride, wp_offsets, out,
                                                   out_capacity);
  *n_launches += 2;
  return cudaGetLastError();
}

}  // namespace gcdf
