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
#include <cmath>
#include <type_traits>

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


// ---- standalone K3 (A6-A8 over dense values): values read ONCE, in a pure streaming pass.
// A unit = kK3TW consecutive tiles of the flat (step, tile) order = one warp (128 slots, 4 per
// lane, one 16-B streaming load each).
// Mark kernel: each warp ballots its unit's actives (f - delta <= tau; dead slots hold +INF and
// never pass), folds the per-step minimum key (one atomicMin per step run), and writes the
// unit's active bitmap (one 32-bit word per lane: nibble i = tile i's 4 slots of the lane,
// 128 B per unit) and its active count.  No shared memory, no barrier, no atomic round trip:
// the warp's life is its loads and ~200 instructions, so the kernel streams the values at the
// read rate of a plain reduction (tools/probes/read_bw.py).
// Emit kernel, after a scan of the unit counts: one warp per unit ranks its actives from the
// bitmap and writes each record (value, gradient row, ids) straight to its final position.
// HBM traffic: the values once, the bitmaps twice (4 B per 128 values), per active the value
// and the 36-B gradient row read (random 32-B sectors) and the 48-B record written.
// (Measured alternatives: round 2's stage kernel allocating per-CTA staging
// with an atomicAdd and writing records from the streaming warps, plus a place pass: 0.39 ms;
// a decoupled look-back in the mark kernel: its prefix front lags the loads, 0.51 ms for mark
// alone; a separate rank kernel writing pair indices + a thread-per-record gather: 0.40 ms.)
constexpr int kK3TW = 8;           // tiles per unit (warp)
constexpr int kK3MarkWarps = 4;    // warps per mark CTA

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

struct K3Scratch {
  int64_t *ucnt;       // [n_units] actives of the unit
  int64_t *upre;       // [n_units + 1] exclusive prefix of ucnt (+ total)
  uint32_t *bits;      // [n_units][32] active bitmaps
  int64_t *scan_tmp;
};

// The largest float x with fl(x - delta) <= tau (fp32, round to nearest): the active test
// "f - delta <= tau" of K2b (R12) as one compare per value.  fl(x - delta) is non-decreasing
// in x, so {x : fl(x - delta) <= tau} = [-inf, x*] exactly (host side, IEEE single arithmetic).
float k3_threshold(float delta, float tau) {
  if (std::isnan(delta) || std::isnan(tau)) return -INFINITY;
  volatile float d = delta, t = tau;  // (no contraction / excess precision: plain fp32 subtracts)
  auto ok = [&](float x) { volatile float r = x - d; return r <= t; };
  float x = tau + delta;
  if (!std::isfinite(x)) return ok(x) ? x : std::nextafter(x, 0.f);
  while (!ok(x)) x = std::nextafter(x, -INFINITY);
  for (;;) {
    const float y = std::nextafter(x, INFINITY);
    if (!ok(y)) return x;
    x = y;
  }
}

__global__ void __launch_bounds__(kK3MarkWarps * 32, 10) k_k3_mark(const float *__restrict__ values, int64_t stride,
                                                                   int32_t n_wp, int32_t tpw, SceneView scene,
                                                                   float thr, DetectScratch ds, K3Scratch ks) {
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * kK3MarkWarps + (threadIdx.x >> 5);
  const int64_t n_tiles = (int64_t)n_wp * tpw;
  const int64_t T0 = u * kK3TW;  // this warp's first flat tile
  if (T0 >= n_tiles) return;
  const int64_t lb = scene.local_bound;
  const int w0 = (int)(T0 / tpw);
  const int t0 = (int)(T0 - (int64_t)w0 * tpw);
  const int nt = (int)min((int64_t)kK3TW, n_tiles - T0);  // tiles of this warp
  // Fast path (all but ~1 in tpw / 8 warps): 8 full tiles inside one step -- straight loads
  // from one base address, no step change inside, no per-tile bounds checks.
  const bool fast = nt == kK3TW && t0 + kK3TW <= tpw;  // (uniform over the warp)
  float4 v[kK3TW];
  if (fast) {
    const float4 *vb = reinterpret_cast<const float4 *>(values + (int64_t)w0 * stride + (int64_t)t0 * kTile) + lane;
#pragma unroll
    for (int i = 0; i < kK3TW; ++i) v[i] = __ldcs(vb + (kTile / 4) * i);
  } else {
    int w = w0, t = t0;
#pragma unroll
    for (int i = 0; i < kK3TW; ++i) {
      if (i < nt) v[i] = load_tile_values(values, stride, lb, w, t, lane);
      if (++t == tpw) { t = 0; ++w; }
    }
  }
  // per tile: this lane's 4 active flags (nibble i of `bits`) and the lane's running minimum of
  // the step
  uint32_t bits = 0u;
  const float inf = __int_as_float(0x7f800000);
  float lmin = inf;
  uint32_t lslot = 0u;
  auto flush = [&](int wk) {  // the step's minimum over the warp: (min value, then smallest slot)
    float m = lmin;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
    uint32_t sl = lmin == m ? lslot : 0xffffffffu;
    sl = __reduce_min_sync(0xffffffffu, sl);
    if (lane == 0 && m < inf)
      atomicMin(ds.wp_key + wk, ((unsigned long long)ord_f32(m) << 32) |
                                    (unsigned long long)local_to_global(sl, scene.rank, scene.world));
    lmin = inf;
  };
  auto process = [&](auto fc) {
    constexpr bool F = decltype(fc)::value;
    int w = w0, t = t0, wk = w0;
#pragma unroll
    for (int i = 0; i < kK3TW; ++i) {
      if (F || i < nt) {  // (uniform over the warp)
        if (!F && w != wk) {
          flush(wk);
          wk = w;
        }
        const float4 x = v[i];
        const uint32_t b = (x.x <= thr ? 1u : 0u) | (x.y <= thr ? 2u : 0u) | (x.z <= thr ? 4u : 0u) |
                           (x.w <= thr ? 8u : 0u);
        bits |= b << (4 * i);
        const float m4 = fminf(fminf(x.x, x.y), fminf(x.z, x.w));
        if (m4 < lmin) {  // (rare after the first tiles of a step)
          lmin = m4;
          lslot = (uint32_t)t * kTile + 4u * lane + (x.x == m4 ? 0u : x.y == m4 ? 1u : x.z == m4 ? 2u : 3u);
        }
      }
      if (F) {
        ++t;
      } else if (++t == tpw) {
        t = 0;
        ++w;
      }
    }
    flush(wk);
  };
  if (fast) process(std::true_type{});
  else process(std::false_type{});
  ks.bits[u * 32 + lane] = bits;
  const int wtot = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(bits));
  if (lane == 0) ks.ucnt[u] = wtot;
}

// Emit kernel (after a scan of the unit counts): one warp per unit -- its count, prefix and
// bitmap word per lane are loaded together; an active (tile i, lane l, bit q) goes to
//   upre[u] + (actives of tiles < i) + (actives of tile i in lanes < l) + (bits below q)
// from one warp scan of the per-tile counts (8-bit fields, even / odd tiles: a tile has <= 128
// actives, no carries); each lane then loads its actives' values and gradient rows and writes
// their records in place.  A step starting in the unit gets its wp_offsets entry; the first
// n_wp + 1 threads of the grid export the per-step min / argmin / keys and the total.
__global__ void __launch_bounds__(256, 8) k_k3_emit(const float *__restrict__ values, const float *__restrict__ grads,
                                                 int64_t stride, int32_t n_wp, int32_t tpw, int64_t n_units,
                                                 SceneView scene, K3Scratch ks, gcdf_active_t *__restrict__ out,
                                                 int64_t cap, const unsigned long long *__restrict__ keys,
                                                 float *wp_min, int64_t *wp_argmin, int64_t *wp_key_out,
                                                 int64_t *wp_offsets, int64_t *count) {
  const int lane = threadIdx.x & 31;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gt <= n_wp) {
    const int w = (int)gt;
    if (w == n_wp) {
      const int64_t tot = n_units > 0 ? ks.upre[n_units] : 0;
      wp_offsets[n_wp] = tot;
      *count = tot;
    } else {
      if (n_units == 0) wp_offsets[w] = 0;
      const unsigned long long k = keys[w];
      if (wp_min) wp_min[w] = k == ~0ull ? __int_as_float(0x7f800000) : unord_f32((unsigned)(k >> 32));
      if (wp_argmin) wp_argmin[w] = k == ~0ull ? -1 : (int64_t)(k & 0xffffffffull);
      if (wp_key_out) wp_key_out[w] = (int64_t)(k ^ 0x8000000000000000ull);
    }
  }
  const int64_t u = gt >> 5;
  if (u >= n_units) return;
  const int64_t cnt = ks.ucnt[u];
  const int64_t pre = ks.upre[u];
  const uint32_t x = ks.bits[u * 32 + lane];
  const int64_t T0 = u * kK3TW;
  const int w0 = (int)(T0 / tpw);
  const int t0 = (int)(T0 - (int64_t)w0 * tpw);
  const int nt = (int)min((int64_t)kK3TW, (int64_t)n_wp * tpw - T0);
  const bool starts = t0 == 0 || t0 + nt > tpw;  // (a step starts inside the unit: rare)
  if (cnt == 0 && !starts) return;
  uint32_t n = x - ((x >> 1) & 0x55555555u);  // popcount of each nibble = each tile
  n = (n & 0x33333333u) + ((n >> 2) & 0x33333333u);
  const uint32_t ne = n & 0x0f0f0f0fu, no = (n >> 4) & 0x0f0f0f0fu;  // tiles 0, 2, 4, 6 / 1, 3, 5, 7
  uint32_t se = ne, so = no;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t a = __shfl_up_sync(0xffffffffu, se, o), b = __shfl_up_sync(0xffffffffu, so, o);
    if (lane >= o) {
      se += a;
      so += b;
    }
  }
  const uint32_t te = __shfl_sync(0xffffffffu, se, 31), to = __shfl_sync(0xffffffffu, so, 31);
  se -= ne;
  so -= no;
  auto tile_tot = [&](int i) { return (int)((((i & 1) ? to : te) >> (8 * (i >> 1))) & 0xffu); };
  if (starts && lane < nt) {
    const int ti = t0 + lane;
    const int wi = ti / tpw;
    if (ti - wi * tpw == 0) {
      int tp = 0;
#pragma unroll
      for (int i = 0; i < kK3TW; ++i)
        if (i < lane) tp += tile_tot(i);
      wp_offsets[w0 + wi] = pre + tp;
    }
  }
  int tile_pre = 0, last = 0;
  uint32_t y = x;
  while (y) {
    const int b = __ffs(y) - 1;
    y &= y - 1u;
    const int i = b >> 2, q = b & 3;
    for (; last < i; ++last) tile_pre += tile_tot(last);
    const int64_t d = pre + tile_pre + (int)((((i & 1) ? so : se) >> (8 * (i >> 1))) & 0xffu) +
                      __popc((x >> (4 * i)) & ((1u << q) - 1u));
    if (d >= cap) continue;
    const int64_t T = T0 + i;
    const int w = (int)(T / tpw);
    const int64_t slot = (T - (int64_t)w * tpw) * kTile + 4 * lane + q;
    const float *g = grads + ((int64_t)w * stride + slot) * kNdof;
    const float f = __ldcs(values + (int64_t)w * stride + slot);
    float gg[kNdof];
#pragma unroll
    for (int k = 0; k < kNdof; ++k) gg[k] = __ldcs(g + k);
    float4 *dst = reinterpret_cast<float4 *>(out + d);
    dst[0] = make_float4(f, gg[0], gg[1], gg[2]);
    dst[1] = make_float4(gg[3], gg[4], gg[5], gg[6]);
    dst[2] = make_float4(gg[7], gg[8], __uint_as_float((unsigned)w),
                         __uint_as_float((unsigned)local_to_global(slot, scene.rank, scene.world)));
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

// ordered copy staging -> out for chunk (w, c), starting at cpre[w * nch + c]: the chunk's
// per-tile prefix (and staging base) goes to shared memory, then every thread copies records
// r = tid, tid + 256, ... of the chunk (tile found by binary search over the prefix), so all
// of a chunk's record copies are in flight at once.  (One thread per 8 tiles copying their
// records one after the other took ~90 us per detect at C2, a third of its latency.)
__global__ void __launch_bounds__(256) k_fin_scatter(const int2 *__restrict__ meta, int32_t tpw,
                                                     const int64_t *__restrict__ tile_start, int64_t nch,
                                                     const int64_t *__restrict__ cpre,
                                                     const gcdf_active_t *__restrict__ staging,
                                                     gcdf_active_t *__restrict__ out, int64_t cap) {
  __shared__ int64_t sh[32];
  __shared__ int s_pre[kFinChunk + 1];  // exclusive prefix of the records of the chunk's tiles
  __shared__ int s_src[kFinChunk];      // staging base of each tile (-1: dropped by the allocation)
  const int w = blockIdx.y;
  const int64_t c = blockIdx.x;
  int64_t t0, nt;
  tile_range(tile_start, tpw, w, t0, nt);
  if (c * kFinChunk >= nt) return;  // (uniform over the block)
  const int64_t b = c * kFinChunk + (int64_t)threadIdx.x * kFinPer;
  const int ntc = (int)min((int64_t)kFinChunk, nt - c * kFinChunk);  // tiles of this chunk
  int2 m[kFinPer];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kFinPer; ++i) {
    m[i] = b + i < nt ? meta[t0 + b + i] : make_int2(0, 0);
    s += m[i].y;
  }
  int64_t tot;
  int pos = (int)block_excl_scan(s, &tot, sh);
#pragma unroll
  for (int i = 0; i < kFinPer; ++i) {
    const int ti = threadIdx.x * kFinPer + i;
    if (ti < ntc) {
      s_pre[ti] = pos;
      s_src[ti] = m[i].x;
    }
    pos += m[i].y;
  }
  if (threadIdx.x == 0) s_pre[ntc] = (int)tot;
  __syncthreads();
  const int64_t dst0 = cpre[(int64_t)w * nch + c];
  for (int r = threadIdx.x; r < (int)tot; r += blockDim.x) {
    int lo = 0, hi = ntc;  // the tile t with s_pre[t] <= r < s_pre[t + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_pre[mid] <= r) lo = mid;
      else hi = mid;
    }
    const int src = s_src[lo];
    const int64_t o = dst0 + r;
    if (src < 0 || o >= cap) continue;
    const float4 *sp = reinterpret_cast<const float4 *>(staging + src + (r - s_pre[lo]));
    const float4 v0 = sp[0], v1 = sp[1], v2 = sp[2];
    float4 *dst = reinterpret_cast<float4 *>(out + o);
    dst[0] = v0;
    dst[1] = v1;
    dst[2] = v2;
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
                                 int64_t *k3_scratch, cudaStream_t s, int *n_launches) {
  const int64_t n_tiles = (int64_t)n_wp * tiles_per_wp;
  const int64_t n_units = (n_tiles + kK3TW - 1) / kK3TW;
  K3Scratch ks;
  ks.ucnt = k3_scratch;
  ks.upre = ks.ucnt + n_units;
  ks.bits = reinterpret_cast<uint32_t *>(ks.upre + n_units + 1);
  ks.scan_tmp = ks.upre + n_units + 1 + 16 * n_units;
  if (n_units > 0) {
    k_k3_mark<<<(unsigned)((n_units + kK3MarkWarps - 1) / kK3MarkWarps), kK3MarkWarps * 32, 0, s>>>(
        values, stride, n_wp, tiles_per_wp, scene, k3_threshold(delta, tau), ds, ks);
    ++*n_launches;
    cudaError_t e = excl_scan(ks.ucnt, n_units, ks.upre, ks.upre + n_units, ks.scan_tmp, s, n_launches);
    if (e != cudaSuccess) return e;
  }
  const int64_t eblocks = std::max<int64_t>((n_units * 32 + 255) / 256, (n_wp + 256) / 256);
  k_k3_emit<<<(unsigned)eblocks, 256, 0, s>>>(values, grads, stride, n_wp, tiles_per_wp, n_units, scene, ks, out,
                                              out_capacity, ds.wp_key, wp_min, wp_argmin, wp_key, wp_offsets, count);
  ++*n_launches;
  return cudaGetLastError();
}

// scratch (int64 elements) of the standalone K3 for n_wp steps of tiles_per_wp tiles
int64_t k3_scratch_elems(int64_t n_wp, int64_t tiles_per_wp) {
  const int64_t n_units = (n_wp * tiles_per_wp + kK3TW - 1) / kK3TW;
  return 2 * n_units + 1 + 16 * n_units + (n_units + 1023) / 1024 + 1;
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
