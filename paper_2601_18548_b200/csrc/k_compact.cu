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


// K3 standalone over dense values: one WARP per tile of 128 slots, 4 slots per lane
// (one 16-B streaming load), no block barrier.  The tile's actives are ranked in slot
// order by a warp prefix scan of per-lane counts (the "warp-ballot and prefix-sum"
// compaction); the per-waypoint min key is a warp-shuffle min + one atomicMin per tile.
// A value of +INF marks a dead slot (gcdf_query_values_grads writes +INF there).
// ---- standalone K3 (A6-A8 over dense values): two passes, no staging and no global counter.
// Pass 1: a warp takes kGroup consecutive tiles (128 slots, 4 per lane, float4 streaming
// loads all in flight), writes each tile's active count to tile_meta and folds the
// per-waypoint minimum key (one atomicMin per waypoint run in the group).  The chunk scan
// of the finalize turns the counts into output offsets; pass 2 re-reads the values of the
// tiles with records and writes the records straight to their final positions.
constexpr int kGroup = 4;

// values of tile tw (0-based within step w) for this lane's 4 slots (+INF outside the scene)
__device__ __forceinline__ float4 load_tile_values(const float *__restrict__ values, int64_t stride, int64_t lb,
                                                   int w, int64_t tw, int lane, int64_t &slot0) {
  slot0 = tw * kTile + 4 * lane;
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

__global__ void __launch_bounds__(256, 4) k_compact_count(const float *__restrict__ values, int64_t stride,
                                                          int32_t n_wp, int32_t tpw, SceneView scene, float delta,
                                                          float tau, DetectScratch ds) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwb = blockDim.x >> 5;  // warps per CTA
  const int64_t n_tiles = (int64_t)n_wp * tpw;
  const int64_t n_groups = (n_tiles + kGroup - 1) / kGroup;
  // each CTA takes a contiguous range of groups and its warps interleave over it (warp j takes
  // groups j, j + 8, ...): the CTA streams contiguous memory (DRAM row locality, as a grid-
  // stride reduction does), while each warp stays on one step for long runs and folds the
  // step's minimum locally (atomicMin only when the step changes)
  const int64_t per = (n_groups + gridDim.x - 1) / gridDim.x;
  const int64_t C0 = (int64_t)blockIdx.x * per, C1 = min(C0 + per, n_groups);
  const int64_t G0 = C0 + warp;
  if (G0 >= C1) return;
  const int64_t lb = scene.local_bound;
  const int step_tiles = kGroup * nwb;  // tile advance between a warp's consecutive groups
  int wcur = (int)(G0 * kGroup / tpw);
  unsigned long long key = ~0ull;
  float lmin = __int_as_float(0x7f800000);  // this lane's minimum of the current step and its slot
  uint32_t lslot = 0u;
  auto flush_key = [&]() {
    if (lmin != __int_as_float(0x7f800000))
      key = ((unsigned long long)ord_f32(lmin) << 32) |
            (unsigned long long)local_to_global(lslot, scene.rank, scene.world);
    lmin = __int_as_float(0x7f800000);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other < key ? other : key;
    }
    if (lane == 0 && key != ~0ull) atomicMin(ds.wp_key + wcur, key);
    key = ~0ull;
  };
  // (step, tile in step) of the first tile of the next group to load / to process; advanced
  // incrementally (no 64-bit divisions per tile)
  int lw = wcur, pw = wcur;
  int lt = (int)(G0 * kGroup - (int64_t)lw * tpw), pt = lt;
  auto advance = [&](int &w, int &t, int by) {
    t += by;
    while (t >= tpw) {
      t -= tpw;
      ++w;
    }
  };
  auto load_group = [&](int64_t G, float4 (&vv)[kGroup]) {
    if (G < C1) {
      int w = lw, t = lt;
#pragma unroll
      for (int i = 0; i < kGroup; ++i) {
        if (G * kGroup + i < n_tiles) {
          int64_t s0;
          vv[i] = load_tile_values(values, stride, lb, w, t, lane, s0);
        }
        advance(w, t, 1);
      }
    }
    advance(lw, lt, step_tiles);
  };
  auto process = [&](int64_t G, const float4 (&vv)[kGroup]) {
    const int64_t T0 = G * kGroup;
    const int nt = (int)min((int64_t)kGroup, n_tiles - T0);  // tiles of this group in range
    int w = pw, tt = pt;
    advance(pw, pt, step_tiles);
#pragma unroll
    for (int i = 0; i < kGroup; ++i) {
      if (i >= nt) break;
      if (w != wcur) {
        flush_key();
        wcur = w;
      }
      const float4 x = vv[i];
      // minimum: the lane's smallest value and its slot, first (smallest slot) on ties -- a
      // min of the four values, and the slot search only when it improves (rare)
      const float m4 = fminf(fminf(x.x, x.y), fminf(x.z, x.w));
      if (m4 < lmin) {
        lmin = m4;
        lslot = (uint32_t)tt * kTile + 4u * lane + (x.x == m4 ? 0u : x.y == m4 ? 1u : x.z == m4 ? 2u : 3u);
      }
      // active: f - delta <= tau (dead slots are +INF and never pass); the tile's bitmap (word
      // k = ballot of slot 4 lane + k) lets pass 2 skip re-reading the values
      const uint32_t b0 = __ballot_sync(0xffffffffu, x.x - delta <= tau);
      const uint32_t b1 = __ballot_sync(0xffffffffu, x.y - delta <= tau);
      const uint32_t b2 = __ballot_sync(0xffffffffu, x.z - delta <= tau);
      const uint32_t b3 = __ballot_sync(0xffffffffu, x.w - delta <= tau);
      if (lane == 0) {
        const int64_t T = T0 + i;
        ds.tile_meta[T] = make_int2(0, __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3));
        ds.tile_bits[T] = make_uint4(b0, b1, b2, b3);
      }
      advance(w, tt, 1);
    }
  };
  // two register sets in ping-pong (no register copies, which would wait for the loads)
  float4 va[kGroup], vb[kGroup];
  load_group(G0, va);
  for (int64_t G = G0; G < C1; G += 2 * nwb) {
    load_group(G + nwb, vb);
    process(G, va);
    load_group(G + 2 * nwb, va);
    if (G + nwb < C1) process(G + nwb, vb);
  }
  flush_key();
}

// ---- finalize: per-tile (staging base, count) -> ordered output.  Tiles of step w are
// [t0(w), t0(w) + nt(w)) (tile_start, or w * tpw); each step's tiles are split into chunks of
// kFinChunk tiles (8 per thread) and every (step, chunk) is one CTA, so the ordered copy runs
// on n_wp * nch CTAs instead of n_wp.
constexpr int kFinPer = 8;
constexpr int kFinChunk = 256 * kFinPer;
constexpr int kWB = 2;  // tiles per warp step of the standalone K3 write pass

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

// pass 2 of the standalone K3: chunk (w, c) of kFinChunk tiles; the tile offsets come from a
// block scan of the pass-1 counts, then a warp per tile reads the tile's 16-B active bitmap
// (pass 1) -- not its values -- ranks the actives with popcounts of the bitmap words, and the
// lanes with actives read their values and gradients and write the records at
// out[cpre + tile offset + rank].
__global__ void __launch_bounds__(256, 3) k_compact_write(const float *__restrict__ values,
                                                       const float *__restrict__ grads, int64_t stride, int32_t tpw,
                                                       int64_t nch, const int64_t *__restrict__ cpre,
                                                       const int2 *__restrict__ meta,
                                                       const uint4 *__restrict__ tbits, SceneView scene,
                                                       gcdf_active_t *__restrict__ out, int64_t cap) {
  __shared__ int64_t sh[32];
  __shared__ int32_t tpos[kFinChunk];
  const int w = blockIdx.y;
  const int64_t c = blockIdx.x;
  const int64_t t0 = (int64_t)w * tpw, nt = tpw;
  if (c * kFinChunk >= nt) return;  // (uniform over the block)
  const int64_t b = c * kFinChunk + (int64_t)threadIdx.x * kFinPer;
  int cnt[kFinPer];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kFinPer; ++i) {
    cnt[i] = b + i < nt ? meta[t0 + b + i].y : 0;
    s += cnt[i];
  }
  int64_t tot;
  int32_t run = (int32_t)block_excl_scan(s, &tot, sh);
#pragma unroll
  for (int i = 0; i < kFinPer; ++i) {
    tpos[threadIdx.x * kFinPer + i] = cnt[i] > 0 ? run : -1;
    run += cnt[i];
  }
  __syncthreads();
  const int64_t dst0 = cpre[(int64_t)w * nch + c];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t tend = min((int64_t)kFinChunk, nt - c * kFinChunk);
  const float *vrow = values + (int64_t)w * stride;
  // kWB tiles per step: their bitmaps, then their value and gradient loads are in flight
  // before the records are written (a lane has usually 0 or 1 active slot per tile;
  // further ones take the loop at the end)
  auto write_rec = [&](int64_t r, int64_t slot, float v, const float *gg) {
    if (r < cap) {
      float4 *dst = reinterpret_cast<float4 *>(out + r);
      dst[0] = make_float4(v, gg[0], gg[1], gg[2]);
      dst[1] = make_float4(gg[3], gg[4], gg[5], gg[6]);
      dst[2] = make_float4(gg[7], gg[8], __uint_as_float((unsigned)w),
                           __uint_as_float((unsigned)local_to_global(slot, scene.rank, scene.world)));
    }
  };
  for (int64_t tl0 = warp; tl0 < tend; tl0 += 8 * kWB) {
    unsigned bits[kWB];
    int64_t r[kWB];
#pragma unroll
    for (int j = 0; j < kWB; ++j) {
      bits[j] = 0u;
      r[j] = 0;
      const int64_t tl = tl0 + 8 * j;
      const int32_t pos = tl < tend ? tpos[tl] : -1;
      if (pos < 0) continue;  // no records in this tile (uniform over the warp)
      const uint4 bw = __ldg(tbits + t0 + c * kFinChunk + tl);
      const uint32_t wd[4] = {bw.x, bw.y, bw.z, bw.w};
      r[j] = dst0 + pos;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        bits[j] |= ((wd[k] >> lane) & 1u) << k;
        r[j] += __popc(wd[k] & lt);  // actives of the lower lanes (all their slots precede this lane's)
      }
    }
    float4 v4[kWB];
    float gg[kWB][kNdof];
    int kf[kWB];
#pragma unroll
    for (int j = 0; j < kWB; ++j) {  // the first active slot of each tile: value + gradient loads
      kf[j] = __ffs(bits[j]) - 1;
      if (bits[j]) {
        const int64_t slot0 = (c * kFinChunk + tl0 + 8 * j) * kTile + 4 * lane;
        v4[j] = __ldg(reinterpret_cast<const float4 *>(vrow + slot0));
        const float *g = grads + ((int64_t)w * stride + slot0 + kf[j]) * kNdof;
#pragma unroll
        for (int i = 0; i < kNdof; ++i) gg[j][i] = __ldcs(g + i);
      }
    }
#pragma unroll
    for (int j = 0; j < kWB; ++j) {
      if (!bits[j]) continue;
      const int64_t slot0 = (c * kFinChunk + tl0 + 8 * j) * kTile + 4 * lane;
      const float v[4] = {v4[j].x, v4[j].y, v4[j].z, v4[j].w};
      write_rec(r[j], slot0 + kf[j], v[kf[j]], gg[j]);
      unsigned rest = bits[j] & (bits[j] - 1u);
      int64_t rr = r[j] + 1;
      while (rest) {  // rare: more than one active slot in this lane's four
        const int k = __ffs(rest) - 1;
        rest &= rest - 1u;
        const float *g = grads + ((int64_t)w * stride + slot0 + k) * kNdof;
        float g2[kNdof];
#pragma unroll
        for (int i = 0; i < kNdof; ++i) g2[i] = __ldcs(g + i);
        write_rec(rr, slot0 + k, v[k], g2);
        ++rr;
      }
    }
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
                                 int64_t *fin_scratch, cudaStream_t s, int *n_launches) {
  const int64_t n_tiles = (int64_t)n_wp * tiles_per_wp;
  if (n_tiles <= 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one wave: the warps' contiguous tile ranges are sized for the CTAs that are resident at once
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_compact_count, 256, 0) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int64_t need = (n_tiles + 8 * kGroup - 1) / (8 * kGroup);  // 8 warps per CTA, kGroup tiles each
  const int64_t grid = need < (int64_t)sms * per_sm ? need : (int64_t)sms * per_sm;
  k_compact_count<<<(unsigned)grid, 256, 0, s>>>(values, stride, n_wp, tiles_per_wp, scene, delta, tau, ds);
  const int64_t nch = finalize_chunks(tiles_per_wp);
  const int64_t n = (int64_t)n_wp * nch;
  int64_t *csum = fin_scratch, *cpre = fin_scratch + n, *tmp = fin_scratch + 2 * n + 1;
  const dim3 g2((unsigned)nch, (unsigned)n_wp);
  k_fin_count<<<g2, 256, 0, s>>>(ds.tile_meta, tiles_per_wp, nullptr, nch, csum);
  cudaError_t e = excl_scan(csum, n, cpre, cpre + n, tmp, s, n_launches);
  if (e != cudaSuccess) return e;
  k_fin_offsets<<<(n_wp + 256) / 256, 256, 0, s>>>(cpre, nch, n_wp, wp_offsets, count, ds.wp_key, wp_min, wp_argmin,
                                                   wp_key);
  k_compact_write<<<g2, 256, 0, s>>>(values, grads, stride, tiles_per_wp, nch, cpre, ds.tile_meta, ds.tile_bits, scene,
                                     out, out_capacity);
  *n_launches += 4;
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
