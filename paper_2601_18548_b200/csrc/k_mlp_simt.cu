// k_mlp_simt.cu -- K2f: fused pair generation + base-frame transform + 7-layer MLP
// forward + input-gradient backward (+ threshold / min / per-tile compaction in detect
// mode), fp32 on the CUDA cores.  This is the parity path (GCDF_FP32); the tensor-core
// path is k_mlp_tc.cu.
//
// Paper steps (PAPER.md line numbers): base-frame bias :388/:171, MLP :284, value +
// gradient :394, constraint f - delta >= 0 :362-363, union = min :164, c_gcdf order
// :414-435.  DESIGN.md §4 "K2f".
//
// One CTA (256 threads) owns a tile of 128 pairs = 1 waypoint x 128 consecutive local
// point slots.  Each thread computes an 8-pair x (H/16)-unit register tile of every
// layer (units interleaved with stride 16).  Activations live in shared memory as
// [unit][pair] (k-major for the next layer), weights stream from L1/L2 (prepacked so
// that each thread's units are contiguous).  ReLU masks stay in registers (1 bit per
// element), so the backward pass never re-reads forward activations.
#include "gcdf_internal.h"

namespace gcdf {
namespace {

constexpr int LD = kTile + 4;  // smem row stride (floats): conflict-free [unit][pair] stores

__device__ __forceinline__ unsigned ord_f32(float f) {
  unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <int UPT>
__device__ __forceinline__ void load_w(const float *__restrict__ p, float (&w)[UPT]) {
  if constexpr (UPT % 4 == 0) {
#pragma unroll
    for (int i = 0; i < UPT; i += 4) {
      float4 v = __ldg(reinterpret_cast<const float4 *>(p + i));
      w[i] = v.x; w[i + 1] = v.y; w[i + 2] = v.z; w[i + 3] = v.w;
    }
  } else if constexpr (UPT == 2) {
    float2 v = __ldg(reinterpret_cast<const float2 *>(p));
    w[0] = v.x; w[1] = v.y;
  } else {
#pragma unroll
    for (int i = 0; i < UPT; ++i) w[i] = __ldg(p + i);
  }
}

// acc[pp][i] += sum_k X[k][8 tp + pp] * Wp[k][tu][i]
template <int H>
__device__ __forceinline__ void gemm_tile(const float *__restrict__ X, const float *__restrict__ Wp, int tp,
                                          int tu, float (&acc)[8][H / 16]) {
  constexpr int UPT = H / 16;
  const float *xr = X + tp * 8;
  const float *wr = Wp + tu * UPT;
#pragma unroll 16  // (16 k steps in flight: 220M -> 173M SM cycles at C3 vs unroll 4; results identical)
  for (int k = 0; k < H; ++k) {
    const float4 x0 = *reinterpret_cast<const float4 *>(xr + k * LD);
    const float4 x1 = *reinterpret_cast<const float4 *>(xr + k * LD + 4);
    float w[UPT];
    load_w<UPT>(wr + k * H, w);
    const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
    for (int pp = 0; pp < 8; ++pp)
#pragma unroll
      for (int i = 0; i < UPT; ++i) acc[pp][i] = fmaf(x[pp], w[i], acc[pp][i]);
  }
}

template <int H>
__device__ __forceinline__ void store_tile(float *__restrict__ Y, int tp, int tu, const float (&v)[8][H / 16]) {
#pragma unroll
  for (int i = 0; i < H / 16; ++i) {
    float *d = Y + (tu + 16 * i) * LD + tp * 8;
    *reinterpret_cast<float4 *>(d) = make_float4(v[0][i], v[1][i], v[2][i], v[3][i]);
    *reinterpret_cast<float4 *>(d + 4) = make_float4(v[4][i], v[5][i], v[6][i], v[7][i]);
  }
}

// H >= 128: one activation buffer updated in place plus a separate [128][9] gradient staging
// area (H = 256: two buffers would exceed shared memory; H = 128: half the shared memory, so
// two CTAs of 256 threads share an SM at 128 registers -- 173M -> 147M SM cycles at C3 despite
// a few spills); H = 32: two buffers in ping-pong
template <int H>
constexpr bool in_place() { return H >= 128; }
template <int H>
constexpr int smem_bytes_simt() {
  return ((in_place<H>() ? 1 : 2) * H * LD + (in_place<H>() ? kTile * kNdof : 0) + 4 * kTile + H + 16 + kTile + 2 * 4 +
          4 + 4) * 4 + 16;
}

// Hidden activation (ACT = MLPW activation id): 1 = ReLU (R9; masks in registers),
// 2 = softplus (NEXT-4 variant, R26): h = max(z, 0) + log1p(e^-|z|), sigma'(z) = 1/(1 + e^-z)
// kept per element in a per-thread stash (local memory, 6 x 8 x H/16 fp32).
__device__ __forceinline__ float softplus_f32(float z, float &dsig) {
  const float t = expf(-fabsf(z));
  const float r = 1.f / (1.f + t);
  dsig = z >= 0.f ? r : t * r;
  return fmaxf(z, 0.f) + log1pf(t);
}

template <int H, int ACT>
__global__ void __launch_bounds__(256, (H == 128 ? 2 : 1)) k_mlp_simt(const WeightsF32 W, const QueryArgs a) {
  constexpr int UPT = H / 16;
  static_assert(ACT == 1 || ACT == 2, "activation");
  constexpr int MW = (8 * UPT + 31) / 32;
  extern __shared__ __align__(16) float smem[];
  constexpr bool kInPlace = in_place<H>();
  float *buf0 = smem;
  float *buf1 = kInPlace ? smem : smem + H * LD;
  float *gstb = smem + (kInPlace ? H * LD : 0);                   // (in place) [128][9] staging
  float4 *sp = reinterpret_cast<float4 *>(smem + (kInPlace ? H * LD + kTile * kNdof : 2 * H * LD));  // [128] points
  float *c1 = reinterpret_cast<float *>(sp + kTile);            // [H] layer-1 per-waypoint constant
  float *qv = c1 + H;                                            // [16]
  float *fval = qv + 16;                                         // [128]
  unsigned long long *kmin = reinterpret_cast<unsigned long long *>(fval + kTile);  // [4]
  unsigned *actw = reinterpret_cast<unsigned *>(kmin + 4);       // [4]
  int *sbase = reinterpret_cast<int *>(actw + 4);                // [1]

  const int tid = threadIdx.x, tp = tid >> 4, tu = tid & 15;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t n_tiles = query_tiles(a);  // (partitioned: read from the device)
  const int64_t lb = a.scene.local_bound;

  for (int64_t T = blockIdx.x; T < n_tiles; T += gridDim.x) {
    int w;
    int64_t slot0;
    bool v0;
    tile_pair(a, T, 0, w, slot0, v0);  // step of this tile (slot0: dense map only)
    (void)v0;
    __syncthreads();  // smem of the previous tile is free
    if (tid < kNdof) qv[tid] = __ldg(a.q + (int64_t)w * kNdof + tid);
    __syncthreads();
    // A2: pair generation + base-frame bias: p' = p - [q_x, q_y, 0];
    // SE(2) frame (R24): p'_xy = R(-theta)(p_xy - [q_x, q_y])
    float cth = 1.f, sth = 0.f;
    if (a.frame) sincosf(qv[2], &sth, &cth);
    if (tid < kTile) {
      int wt;
      int64_t slot;
      bool valid;
      tile_pair(a, T, tid, wt, slot, valid);
      float4 p = valid ? __ldg(a.scene.pts + slot) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float dx = p.x - qv[0], dy = p.y - qv[1];
      sp[tid] = make_float4(cth * dx + sth * dy, -sth * dx + cth * dy, p.z, p.w);
    }
    // layer-1 constant of this waypoint: c = b1 + W1[:, 5:12] . [theta, j1..j6]
    // (the q^t input channels are fed zero, R2; the theta channel is fed zero in SE(2), R24)
    for (int u = tid; u < H; u += 256) {
      const float *wq = W.w1q + u * 8;
      float c = __ldg(&W.w1p[u].w);
      if (!a.frame) c = fmaf(__ldg(wq), qv[2], c);
#pragma unroll
      for (int i = 1; i < 7; ++i) c = fmaf(__ldg(wq + i), qv[2 + i], c);
      c1[u] = c;
    }
    __syncthreads();

    uint32_t mask[kHidden][MW];
#pragma unroll
    for (int l = 0; l < kHidden; ++l)
#pragma unroll
      for (int m = 0; m < MW; ++m) mask[l][m] = 0u;
    float dsig[ACT == 2 ? kHidden : 1][8][UPT];  // softplus'(z_l) per element (ACT 2)

    float acc[8][UPT];
    // A3: layer 1 (12 -> H) in fp32: z1 = W1[:, 0:3] p' + c
    {
      float4 wv[UPT];
      float cc[UPT];
#pragma unroll
      for (int i = 0; i < UPT; ++i) {
        wv[i] = __ldg(&W.w1p[tu + 16 * i]);
        cc[i] = c1[tu + 16 * i];
      }
#pragma unroll
      for (int pp = 0; pp < 8; ++pp) {
        const float4 x = sp[tp * 8 + pp];
#pragma unroll
        for (int i = 0; i < UPT; ++i) {
          float z = fmaf(wv[i].x, x.x, fmaf(wv[i].y, x.y, fmaf(wv[i].z, x.z, cc[i])));
          const int b = i * 8 + pp;
          if constexpr (ACT == 2) {
            acc[pp][i] = softplus_f32(z, dsig[0][pp][i]);
          } else {
            if (z > 0.f) mask[0][b >> 5] |= 1u << (b & 31);
            acc[pp][i] = fmaxf(z, 0.f);
          }
        }
      }
    }
    float *cur = buf0, *nxt = buf1;
    store_tile<H>(cur, tp, tu, acc);
    __syncthreads();

    // A4: hidden layers 2..6: h_l = ReLU(W_l h_{l-1} + b_l)
    float fpart[8];
#pragma unroll 1
    for (int li = 0; li < 5; ++li) {
      {
        float bv[UPT];
#pragma unroll
        for (int i = 0; i < UPT; ++i) bv[i] = __ldg(W.bias[li] + tu + 16 * i);
#pragma unroll
        for (int pp = 0; pp < 8; ++pp)
#pragma unroll
          for (int i = 0; i < UPT; ++i) acc[pp][i] = bv[i];
      }
      gemm_tile<H>(cur, W.wt[li], tp, tu, acc);
#pragma unroll
      for (int pp = 0; pp < 8; ++pp)
#pragma unroll
        for (int i = 0; i < UPT; ++i) {
          const int b = i * 8 + pp;
          if constexpr (ACT == 2) {
            acc[pp][i] = softplus_f32(acc[pp][i], dsig[li + 1][pp][i]);
          } else {
            if (acc[pp][i] > 0.f) mask[li + 1][b >> 5] |= 1u << (b & 31);
            acc[pp][i] = fmaxf(acc[pp][i], 0.f);
          }
        }
      if (li < 4) {
        if constexpr (kInPlace) __syncthreads();  // every thread has read cur
        store_tile<H>(nxt, tp, tu, acc);
        __syncthreads();
        float *tmp = cur; cur = nxt; nxt = tmp;
      }
    }
    // output layer: f = w7 . h6 + b7 (no activation: signed value)
    {
      float w7v[UPT];
#pragma unroll
      for (int i = 0; i < UPT; ++i) w7v[i] = __ldg(W.w7 + tu + 16 * i);
#pragma unroll
      for (int pp = 0; pp < 8; ++pp) {
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < UPT; ++i) s = fmaf(w7v[i], acc[pp][i], s);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        s += __shfl_xor_sync(0xffffffffu, s, 8);
        fpart[pp] = s + W.b7;
      }
      if (tu == 0) {
#pragma unroll
        for (int pp = 0; pp < 8; ++pp) fval[tp * 8 + pp] = fpart[pp];
      }
      // backward seed: e6 = w7 (.) 1[z6 > 0]
#pragma unroll
      for (int pp = 0; pp < 8; ++pp)
#pragma unroll
        for (int i = 0; i < UPT; ++i) {
          const int b = i * 8 + pp;
          if constexpr (ACT == 2)
            acc[pp][i] = w7v[i] * dsig[5][pp][i];
          else
            acc[pp][i] = (mask[5][b >> 5] >> (b & 31)) & 1u ? w7v[i] : 0.f;
        }
      if constexpr (kInPlace) __syncthreads();  // every thread has read cur
      store_tile<H>(nxt, tp, tu, acc);
      __syncthreads();
      float *tmp = cur; cur = nxt; nxt = tmp;
    }

    // A6/A7 (detect): threshold, per-tile compaction slots, per-waypoint min key
    if (a.detect) {
      if (tid < kTile) {
        int wt;
        int64_t slot;
        bool valid;
        tile_pair(a, T, tid, wt, slot, valid);
        const bool live = valid && sp[tid].w > 0.f;
        const float f = fval[tid];
        const bool act = live && (f - a.delta <= a.tau);
        const unsigned bal = __ballot_sync(0xffffffffu, act);
        unsigned long long key = ~0ull;
        if (live) {
          const unsigned long long gid = (unsigned long long)local_to_global(slot, a.scene.rank, a.scene.world);
          key = ((unsigned long long)ord_f32(f) << 32) | gid;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
          key = other < key ? other : key;
        }
        if (lane == 0) {
          actw[warp] = bal;
          kmin[warp] = key;
        }
      }
      __syncthreads();
      if (tid == 0) {
        unsigned long long km = kmin[0];
        int cnt = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          km = kmin[i] < km ? kmin[i] : km;
          cnt += __popc(actw[i]);
        }
        if (km != ~0ull) atomicMin(a.ds.wp_key + w, km);
        int base = 0;
        if (cnt > 0) {
          unsigned long long b = atomicAdd(a.ds.counter, (unsigned long long)cnt);
          if (b + cnt > (unsigned long long)a.ds.max_active) {
            atomicOr(a.ds.counter + 1, 1ull);
            base = -1;
          } else {
            base = (int)b;
          }
        }
        *sbase = base;
        a.ds.tile_meta[T] = make_int2(base, cnt);
      }
      // (visibility of sbase/actw is ensured by the barriers of the backward pass)
    }

    // A5: input-gradient backward: g_{l-1} = W_l^T e_l, e_{l-1} = g_{l-1} (.) 1[z_{l-1} > 0]
#pragma unroll 1
    for (int li = 4; li >= 0; --li) {
#pragma unroll
      for (int pp = 0; pp < 8; ++pp)
#pragma unroll
        for (int i = 0; i < UPT; ++i) acc[pp][i] = 0.f;
      gemm_tile<H>(cur, W.wb[li], tp, tu, acc);
#pragma unroll
      for (int pp = 0; pp < 8; ++pp)
#pragma unroll
        for (int i = 0; i < UPT; ++i) {
          const int b = i * 8 + pp;
          if constexpr (ACT == 2)
            acc[pp][i] *= dsig[li][pp][i];
          else
            acc[pp][i] = (mask[li][b >> 5] >> (b & 31)) & 1u ? acc[pp][i] : 0.f;
        }
      if constexpr (kInPlace) __syncthreads();  // every thread has read cur
      store_tile<H>(nxt, tp, tu, acc);
      __syncthreads();
      float *tmp = cur; cur = nxt; nxt = tmp;
    }
    // g0 = W1^T e1 restricted to the inputs that depend on q; map to d f / d q (R3):
    //   chain rule:  [-g0[0], -g0[1], g0[5..11]];  q-channel: [g0[3], g0[4], g0[5..11]]
    float *gst = kInPlace ? gstb : nxt;  // [128][9] staging
    {
      const int p = tid & (kTile - 1);
      const int half = tid >> 7;  // warp-uniform
      const float *er = cur + p;
      if (half == 0) {
        const int x0 = a.tgrad ? 3 : 0, x1 = a.tgrad ? 4 : 1;
        float g[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
        for (int k = 0; k < H; ++k) {
          const float e = er[k * LD];
          const float *row = W.w1full + k * kNin;
          g[0] = fmaf(e, __ldg(row + x0), g[0]);
          g[1] = fmaf(e, __ldg(row + x1), g[1]);
          g[2] = fmaf(e, __ldg(row + 5), g[2]);
          g[3] = fmaf(e, __ldg(row + 6), g[3]);
          g[4] = fmaf(e, __ldg(row + 7), g[4]);
        }
        if (a.frame) {
          // SE(2) (R24): df/db = -R(theta) g0_xy, df/dtheta = g0_x p'_y - g0_y p'_x
          const float gx = g[0], gy = g[1];
          g[0] = -(cth * gx - sth * gy);
          g[1] = -(sth * gx + cth * gy);
          g[2] = gx * sp[p].y - gy * sp[p].x;
        } else if (!a.tgrad) {
          g[0] = -g[0];
          g[1] = -g[1];
        }
#pragma unroll
        for (int c = 0; c < 5; ++c) gst[p * 9 + c] = g[c];
      } else {
        float g[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
        for (int k = 0; k < H; ++k) {
          const float e = er[k * LD];
          const float *row = W.w1full + k * kNin;
          g[0] = fmaf(e, __ldg(row + 8), g[0]);
          g[1] = fmaf(e, __ldg(row + 9), g[1]);
          g[2] = fmaf(e, __ldg(row + 10), g[2]);
          g[3] = fmaf(e, __ldg(row + 11), g[3]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) gst[p * 9 + 5 + c] = g[c];
      }
    }
    __syncthreads();

    if (!a.detect) {
      // dense outputs: values [n_wp][lb], grads [n_wp][lb][9]; dead slots -> +INF, 0
      if (tid < kTile) {
        const int64_t slot = slot0 + tid;
        if (slot < lb) a.values[(int64_t)w * lb + slot] = sp[tid].w > 0.f ? fval[tid] : __int_as_float(0x7f800000);
      }
      if (a.grads) {
        const int64_t gbase = ((int64_t)w * lb + slot0) * kNdof;
        for (int idx = tid; idx < kTile * kNdof; idx += 256) {
          const int p = idx / kNdof;
          const int k = idx - p * kNdof;
          // (NEXT-3 projection: q_z = q - f M^{-1} grad_q f, Theorem 1.2)
          const float o = a.project ? qv[k] - (fval[p] * gst[idx]) * a.minv[k] : gst[idx];
          if (slot0 + p < lb) a.grads[gbase + idx] = sp[p].w > 0.f ? o : 0.f;
        }
      }
    } else if (tid < kTile) {
      // A8: ordered per-tile compaction into the staging slots (finalized by k_compact.cu)
      const int base = *sbase;
      const unsigned bits = actw[warp];
      if (base >= 0 && ((bits >> lane) & 1u)) {
        int r = __popc(bits & ((1u << lane) - 1u));
        for (int i = 0; i < warp; ++i) r += __popc(actw[i]);
        int wt;
        int64_t slot;
        bool valid;
        tile_pair(a, T, tid, wt, slot, valid);
        float4 *dst = reinterpret_cast<float4 *>(a.ds.staging + base + r);
        const float *g = gst + tid * 9;
        dst[0] = make_float4(fval[tid], g[0], g[1], g[2]);
        dst[1] = make_float4(g[3], g[4], g[5], g[6]);
        dst[2] = make_float4(g[7], g[8], __uint_as_float((unsigned)w),
                             __uint_as_float((unsigned)local_to_global(slot, a.scene.rank, a.scene.world)));
      }
    }
  }
}

template <int H, int ACT>
cudaError_t launch_h(const WeightsF32 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  const int smem = smem_bytes_simt<H>();
  cudaError_t e = cudaFuncSetAttribute(k_mlp_simt<H, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mlp_simt<H, ACT>, 256, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (!a.part.tile_wp) {  // (a partitioned detect knows its tile count on the device only)
    const int64_t n_tiles = (int64_t)a.n_wp * a.tiles_per_wp;
    if (grid > n_tiles) grid = n_tiles;
  }
  if (grid < 1) return cudaSuccess;
  k_mlp_simt<H, ACT><<<(unsigned)grid, 256, smem, s>>>(w, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mlp_simt(int H, const WeightsF32 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  if (a.act == 2) {
    if (H == 128) return launch_h<128, 2>(w, a, num_sms, s);
    if (H == 32) return launch_h<32, 2>(w, a, num_sms, s);
    if (H == 256) return launch_h<256, 2>(w, a, num_sms, s);
    return cudaErrorInvalidValue;
  }
  if (H == 128) return launch_h<128, 1>(w, a, num_sms, s);
  if (H == 32) return launch_h<32, 1>(w, a, num_sms, s);
  if (H == 256) return launch_h<256, 1>(w, a, num_sms, s);
  return cudaErrorInvalidValue;
}

}  // namespace gcdf
