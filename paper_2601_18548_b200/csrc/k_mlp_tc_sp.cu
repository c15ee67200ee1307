// k_mlp_tc_sp.cu -- K2s: the softplus variant (NEXT-4, R26) of the fused tcgen05
// path: pair generation + base-frame bias + 7-layer MLP forward + input-gradient backward
// (+ threshold / min / per-tile compaction in detect mode), fp16 operands, fp32 accumulation.
//
// Paper steps (PAPER.md lines): base-frame bias :388/:171; "7-layer MLP" on [p, q] :284;
// value + gradient :394; constraint f - delta >= 0 :362-363; union = min :164; c_gcdf
// order :414-435.  The activation is not named by the paper (:284); softplus is SPEC.md:281's
// choice for a smooth field.
//
// What differs from K2b (k_mlp_tc.cu): softplus'(z) is not a 1-bit mask, so the backward
// needs a 16-bit quantity per unit and layer.  K2s keeps the forward activations h_1..h_5
// (the fp16 A operands of layers 2..6) resident in TMEM and recovers
//     softplus'(z) = sigmoid(z) = 1 - e^{-softplus(z)} = 1 - e^{-h}
// from them in the backward; e_l = g_l * sigma'_l then overwrites h_l in place and is the A
// operand of the next backward UMMA.  TMEM (512 columns, one tile in flight):
//     [0, 128)    D: fp32 accumulator of the current phase
//     [128, 448)  h_1 .. h_5 (64 columns each; e_l replaces h_l during the backward)
//     [448, 512)  layer-1 operands x (K = 32, 16 columns) + the "ones" block of the bias
//                 step (8 columns) during the forward; e_6 (64 columns) from phase 5 on
// One tile in flight means the tensor pipe idles during every epilogue; the epilogue is
// bound by the MUFU pipe (2 ops per element forward: ex2 + lg2, 1 backward: ex2), so the
// variant trades throughput for a smooth field ("K2s").
//
// Rounding points (the oracle's EMU_FP16 mode for activation 2, oracle/gcdf_oracle.c):
// A operands h_1..h_5 and e_6..e_1 rounded to fp16 (RN); sigma' of layers 1..5 from the
// rounded h; layer 6's sigma' from the fp32 z_6; f = w7 . h_6 + b7 in fp32; layer 1 in
// split hi/lo operands (~fp32), as in K2b.
#include <cuda_fp16.h>

#include <type_traits>

#include "gcdf_internal.h"
#include "tc_ptx.h"

namespace gcdf {
namespace {

using namespace tc;

constexpr int H = 128;
constexpr int kEpiWarps = 16;                  // warp w: TMEM lane quarter w % 4, unit quarter w / 4
constexpr int kThreads = (kEpiWarps + 1) * 32; // + one MMA warp
constexpr int kEpi = kEpiWarps * 32;           // epilogue threads
constexpr int kEpiHalf = kEpi / 2;             // epi_done[h] arrivals per phase (unit quarters 2h, 2h + 1)
constexpr int kPhases = 12;
constexpr int kWBytes = 5 * H * H * 2;
constexpr int kW1tBytes = 16 * H * 2;
constexpr int kB1Bytes = 32 * H * 2;
constexpr int kBextBytes = 16 * H * 2;
constexpr uint32_t kColH = 128, kColX = 448, kColOnes = 464, kColE6 = 448;
constexpr uint32_t kIdescFwd = idesc_f16kind(128, 64, false, true);  // (output halves: N = 64)
constexpr uint32_t kIdescBwd = idesc_f16kind(128, 64, true, true);
constexpr uint32_t kIdescFin = idesc_f16kind(128, 16, false, true);

struct __align__(1024) SmemSP {
  uint8_t w[kWBytes];           // W_2..W_6 fp16, SW128 (the K2b layout)
  uint8_t w1t[kW1tBytes];       // W1^T [16][128], SW128
  uint8_t b1[kB1Bytes];         // layer-1 split weights [128][32], no swizzle
  uint8_t bext[5][kBextBytes];  // hidden-layer bias blocks [128][16], no swizzle
  float w7[H];
  float fpart[4][H];            // [unit quarter][row] partial output-layer sums
  float4 ptn[H];                // [row] prefetched point of the next tile
  float qn[2][12];              // [tile parity] q row of the tile
  int wtile[2];                 // [tile parity] step (waypoint) of the tile
  uint32_t slotn[2][H];         // [tile parity][row] local scene slot (~0: padding)
  uint64_t mma_done[2];  // [output half]
  uint64_t epi_done[2];
  unsigned act[4];
  unsigned long long kmin[4];
  int sbase;
  uint32_t tmem_base;
};
static_assert(sizeof(SmemSP) + 1024 <= 232448, "SmemSP exceeds the 227 KB of shared memory per CTA");

DEVI float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
DEVI float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
DEVI float rcpf(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2e = 1.4426950408889634f, kLn2 = 0.6931471805599453f;
// softplus(z) = max(z, 0) + log(1 + e^-|z|); t = e^-|z| is returned for the sigmoid
DEVI float softplus_t(float z, float &t) {
  t = ex2f(-fabsf(z) * kLog2e);
  return fmaxf(z, 0.f) + lg2f(1.f + t) * kLn2;
}
// log1p(t) on [0, 1] as a degree-9 polynomial on the FMA pipe (max error 1.24e-7 in fp32;
// coefficients from tools/fit_log1p.py): half of the forward softplus evaluations use it
// instead of the MUFU lg2, so the epilogue's transcendental work is split between the XU
// and the FMA pipes
DEVI float log1p_poly(float t) {
  float r = 3.704979084e-03f;
  r = fmaf(r, t, -2.274715155e-02f);
  r = fmaf(r, t, 6.580121815e-02f);
  r = fmaf(r, t, -1.243493631e-01f);
  r = fmaf(r, t, 1.840040535e-01f);
  r = fmaf(r, t, -2.460547388e-01f);
  r = fmaf(r, t, 3.327418566e-01f);
  r = fmaf(r, t, -4.999519885e-01f);
  r = fmaf(r, t, 9.999983311e-01f);
  return fmaf(r, t, 1.480288958e-08f);
}
DEVI float softplus_t_poly(float z, float &t) {
  t = ex2f(-fabsf(z) * kLog2e);
  return fmaxf(z, 0.f) + log1p_poly(t);
}
DEVI unsigned ord_f32(float f) {
  unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
DEVI float round16(float x) { return __half2float(__float2half_rn(x)); }
// {x_hi, x_lo, x_hi}: the split layer-1 operand of one input (K2b, R16)
DEVI void split3(float x, float *o) {
  const float hi = round16(x);
  o[0] = hi;
  o[1] = x - hi;
  o[2] = hi;
}
DEVI float2 unpack_h2(uint32_t u) {
  __half2 h;
  memcpy(&h, &u, 4);
  return __half22float2(h);
}

// UMMAs of phase p by output half (one elected lane of the converged MMA warp): half h writes
// accumulator columns 64 h .. 64 h + 63 (N = 64, B rows / columns 64 h ..) and is committed to
// mma_done[h], so the epilogue of half 0 starts while the tensor core runs half 1.  Half 0's
// first four K steps read only the units half 0's epilogue wrote (A columns of units 0..63):
// they are issued after epi_done[0]; the rest of the phase after epi_done[1] (wait_half(h)).
template <typename WaitHalf>
DEVI void issue_phase(int p, uint32_t tb, uint32_t sw, uint32_t sw1t, uint32_t sb1, uint32_t sbx, uint64_t *done,
                      WaitHalf &&wait_half) {
  if (p == 0) {  // layer 1: K = 32 split operands (bias included), A = x (written by half 0)
    wait_half(0);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1) wait_half(1);
#pragma unroll
      for (int k = 0; k < 2; ++k)
        mma_ts_elect(tb + 64u * h, tb + kColX + 8u * k, sdesc_nosw(sb1 + k * 2 * 2048 + 1024u * h, 2048, 128), kIdescFwd,
                     k > 0);
      commit_elect(&done[h]);
    }
  } else if (p < 11) {
    const bool fwd = p < 6;
    uint32_t av;
    uint64_t b[2];
    if (fwd) {  // layer l = p + 1: D = h_{l-1} W_l^T + ones x bias (B K-major: output rows 64 h ..)
      av = tb + kColH + 64u * (uint32_t)(p - 1);
      const uint32_t wb = sw + (uint32_t)(p - 1) * (H * H * 2);
      b[0] = sdesc_sw128(wb, 16, 1024);
      b[1] = sdesc_sw128(wb + 8192u, 16, 1024);
    } else {  // backward through layer l = 12 - p: D = e_l W_l (B MN-major: N chunk h)
      av = p == 6 ? tb + kColE6 : tb + kColH + 64u * (uint32_t)(11 - p);
      const uint32_t wb = sw + (uint32_t)(10 - p) * (H * H * 2);
      b[0] = sdesc_sw128(wb, 16384, 1024);
      b[1] = sdesc_sw128(wb + 16384u, 16384, 1024);
    }
    const uint32_t id = fwd ? kIdescFwd : kIdescBwd;
    // (each group of four K steps from one asm block: the lean issue of K2b, tc_ptx.h)
    auto k4 = [&](uint32_t d, uint32_t a, uint64_t bd, uint32_t acc) {
      if (fwd) umma4_sw128_elect(d, a, bd, id, acc);
      else umma4_mn_elect(d, a, bd, id, acc);
    };
    // K steps 4..7: K-major B in the second 64-K chunk (+ 16 KB), MN-major B + 4 x 2 KB
    const uint64_t k47 = fwd ? 1024u : 512u;
    wait_half(0);
    k4(tb, av, b[0], 0u);  // half 0, K steps 0..3 (units 0..63 of A)
    wait_half(1);
    k4(tb, av + 32u, b[0] + k47, 1u);
    if (fwd) mma_ts_elect(tb, tb + kColOnes, sdesc_nosw(sbx + (uint32_t)(p - 1) * kBextBytes, 2048, 128), id, 1u);
    commit_elect(&done[0]);
    k4(tb + 64u, av, b[1], 0u);
    k4(tb + 64u, av + 32u, b[1] + k47, 1u);
    if (fwd)
      mma_ts_elect(tb + 64u, tb + kColOnes, sdesc_nosw(sbx + (uint32_t)(p - 1) * kBextBytes + 1024u, 2048, 128), id,
                   1u);
    commit_elect(&done[1]);
  } else {  // g0 = e1 W1 (N = 16 rows of W1^T): needs all of e1
    wait_half(0);
    wait_half(1);
    umma4_sw128_elect(tb, tb + kColH, sdesc_sw128(sw1t, 16, 1024), kIdescFin, 0u);
    umma4_sw128_elect(tb, tb + kColH + 32u, sdesc_sw128(sw1t + 2048, 16, 1024), kIdescFin, 1u);
    commit_elect(&done[0]);
    commit_elect(&done[1]);
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_mlp_tc_sp(const WeightsBF16 W, const QueryArgs a) {
  extern __shared__ uint8_t smem_raw[];
  SmemSP &S = *reinterpret_cast<SmemSP *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    auto copy16 = [&](void *dst, const void *src, int bytes) {
      const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
      uint4 *d4 = reinterpret_cast<uint4 *>(dst);
      for (int i = tid; i < bytes / 16; i += kThreads) d4[i] = __ldg(s4 + i);
    };
    copy16(S.w, W.w_sw128, kWBytes);
    copy16(S.w1t, W.w1t_sw128, kW1tBytes);
    copy16(S.b1, W.b1_nosw, kB1Bytes);
    copy16(S.bext, W.bext_nosw, 5 * kBextBytes);
    for (int i = tid; i < H; i += kThreads) S.w7[i] = __ldg(W.w7 + i);
  }
  if (warp == 0) {
    tmem_alloc(&S.tmem_base, 512);
    tmem_relinquish();
  }
  if (tid == 32) {
    for (int h = 0; h < 2; ++h) {
      mbar_init(&S.mma_done[h], 1);
      mbar_init(&S.epi_done[h], kEpiHalf);
    }
    fence_barrier_init();
  }
  const int64_t n_tiles = query_tiles(a);
  fence_proxy_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = S.tmem_base;
  const int64_t lb = a.scene.local_bound;
  const int64_t stride = gridDim.x;

  if (warp == kEpiWarps) {
    // ===================== MMA warp ================================================
    const uint32_t sw = smem_u32(S.w), sw1t = smem_u32(S.w1t), sb1 = smem_u32(S.b1), sbx = smem_u32(S.bext);
    uint32_t ph = 0u;  // bit h: parity of epi_done[h]
    auto wait_half = [&](int h) {
      mbar_wait(&S.epi_done[h], (ph >> h) & 1u);
      ph ^= 1u << h;
      fence_after();
    };
    for (int64_t T = blockIdx.x; T < n_tiles; T += stride) {
#pragma unroll 1
      for (int p = 0; p < kPhases; ++p) issue_phase(p, tbase, sw, sw1t, sb1, sbx, S.mma_done, wait_half);
    }
    __syncwarp();
    fence_before();
    __syncthreads();
    return;
  }

  // ===================== epilogue warps ===============================================
  // (the warp index through a lane-0 shuffle: warp-uniform to the compiler, so the TMEM
  // addresses derived from it live in uniform registers, as in K2b)
  const int ew = __shfl_sync(0xffffffffu, warp, 0);
  const int qd = ew & 3;      // TMEM lane quarter (warp % 4)
  const int cq = ew >> 2;     // unit quarter: units 32 cq .. 32 cq + 31
  const int row = qd * 32 + lane;
  const int u0 = 32 * cq;
  const uint32_t tL = tbase + ((uint32_t)(qd * 32) << 16);
  const uint32_t tD = tL + (uint32_t)u0;
  auto tH = [&](int l) { return tL + kColH + 64u * (uint32_t)(l - 1) + 16u * (uint32_t)cq; };  // h_l / e_l, l = 1..5

  const int half = cq >> 1;     // output half of this warp's units
  auto hand_off = [&]() {
    wait_st();
    fence_before();
    mbar_arrive(&S.epi_done[half]);
  };
  // point of row `row` of tile TT -> S.ptn[row] (cp.async), its slot -> S.slotn[par][row];
  // warp 0 also fetches the tile's q row
  auto prefetch = [&](int64_t TT, int par) {
    int wn = 0;
    int64_t sl = 0;
    bool ok = false;
    if (TT < n_tiles) tile_pair(a, TT, row, wn, sl, ok);
    S.slotn[par][row] = ok ? (uint32_t)sl : ~0u;
    cp_async16(&S.ptn[row], ok ? (const void *)(a.scene.pts + sl) : (const void *)a.scene.pts, ok ? 16u : 0u);
    if (warp == 0 && TT < n_tiles) {
      wn = tile_step(a, TT);
      if (lane < kNdof) cp_async4(&S.qn[par][lane], a.q + (int64_t)wn * kNdof + lane);
      if (lane == 0) S.wtile[par] = wn;
    }
    cp_async_commit();
  };
  // layer-1 operands of the tile (x_in split hi/lo, K = 32) and the ones block -> TMEM;
  // unit quarter 0 writes K 0..15, quarter 1 K 16..31, quarter 2 the ones block
  auto stage_a1 = [&](int par) -> bool {
    const float *qw = S.qn[par];
    bool lv = false;
    if (cq == 0) {
      float v[16];
      const float4 pt = S.ptn[row];
      lv = S.slotn[par][row] != ~0u && pt.w > 0.f;
      split3(pt.x - qw[0], v);      // p'_x (A2: base-frame bias)
      split3(pt.y - qw[1], v + 3);  // p'_y
      split3(pt.z, v + 6);
      split3(qw[2], v + 9);         // theta
      split3(qw[3], v + 12);        // j1
      v[15] = round16(qw[4]);
      uint32_t a1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a1[i] = pack_f16(v[2 * i], v[2 * i + 1]);
      st8(tL + kColX, a1);
    } else if (cq == 1) {
      float v[16];
      const float j2 = qw[4];
      const float j2h = round16(j2);
      v[0] = j2 - j2h;
      v[1] = j2h;
#pragma unroll
      for (int i = 0; i < 4; ++i) split3(qw[5 + i], v + 2 + 3 * i);
      v[14] = 1.f;
      v[15] = 1.f;
      uint32_t a1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a1[i] = pack_f16(v[2 * i], v[2 * i + 1]);
      st8(tL + kColX + 8u, a1);
    } else if (cq == 2) {
      const uint32_t ones[8] = {pack_f16(1.f, 1.f), 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      st8(tL + kColOnes, ones);
    }
    hand_off();
    return lv;
  };

  uint32_t ph = 0u;
  int it = 0;
  bool live_n = false;
  if ((int64_t)blockIdx.x < n_tiles) {
    prefetch(blockIdx.x, 0);
    cp_async_wait_all();
    named_bar_sync(1, kEpi);  // S.ptn / S.slotn / S.qn of the first tile are visible
    live_n = stage_a1(0);
  }
  for (int64_t T = blockIdx.x; T < n_tiles; T += stride, ++it) {
    const int par = it & 1;
    const bool live = live_n;
    float f = 0.f;
    int ridx = -1;
    unsigned long long pend_b = 0ull;
    int pend_cnt = 0;
    // one phase of the tile (compile-time phase number, as in K2b: every phase is its own
    // straight code, no run-time dispatch)
    auto phase = [&](auto pc) {
      constexpr int p = decltype(pc)::value;
      mbar_wait(&S.mma_done[half], ph);
      ph ^= 1u;
      fence_after();
      if (p < 5) {
        // ---- forward layer l = p + 1: h = softplus(z) -> fp16 A operand, kept for the backward
        uint32_t r[32];
        ld32(tD, r);
        wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float t0, t1;
          const float h0 = softplus_t(__uint_as_float(r[2 * j]), t0);
          const float h1 = softplus_t_poly(__uint_as_float(r[2 * j + 1]), t1);
          pk[j] = pack_f16(h0, h1);
        }
        st16(tH(p + 1), pk);
        hand_off();
      } else if (p == 5) {
        // ---- layer 6: f = w7 . softplus(z6) + b7 (fp32); e6 = w7 sigmoid(z6) -> A ----
        uint32_t r[32];
        ld32(tD, r);
        wait_ld();
        uint32_t pk[16];
        float fa = 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float e[2];
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const float z = __uint_as_float(r[2 * j + k]);
            float t;
            const float h = k ? softplus_t_poly(z, t) : softplus_t(z, t);
            const float w7 = S.w7[u0 + 2 * j + k];
            fa = fmaf(w7, h, fa);
            // sigmoid(z) = 1 / (1 + e^-z) = (z >= 0 ? 1 : e^-|z|) / (1 + e^-|z|)
            e[k] = w7 * ((z >= 0.f ? 1.f : t) * rcpf(1.f + t));
          }
          pk[j] = pack_f16(e[0], e[1]);
        }
        st16(tL + kColE6 + 16u * (uint32_t)cq, pk);
        hand_off();
        S.fpart[cq][row] = fa;
        named_bar_sync(1, kEpi);
        if (cq == 0) {
          f = (S.fpart[0][row] + S.fpart[1][row]) + (S.fpart[2][row] + S.fpart[3][row]) + W.b7;
          if (!a.detect) {
            const int w = S.wtile[par];
            const int64_t slot = S.slotn[par][row];
            if (slot < lb) a.values[(int64_t)w * lb + slot] = live ? f : __int_as_float(0x7f800000);
          }
        }
      } else if (p < 11) {
        // ---- backward: g_{l-1} = D; e_{l-1} = g (.) (1 - e^{-h~_{l-1}}) overwrites h_{l-1} ----
        const int l = 11 - p;  // layer whose derivative is applied (5 .. 1)
        uint32_t r[32], hp[16];
        ld32(tD, r);
        ld16(tH(l), hp);
        wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 h = unpack_h2(hp[j]);
          const float s0 = 1.f - ex2f(-h.x * kLog2e);
          const float s1 = 1.f - ex2f(-h.y * kLog2e);
          pk[j] = pack_f16(__uint_as_float(r[2 * j]) * s0, __uint_as_float(r[2 * j + 1]) * s1);
        }
        st16(tH(l), pk);
        hand_off();
        if (p == 6 && cq == 0 && a.detect) {
          // A6/A7: threshold, per-tile slots, per-waypoint min key (overlaps the tensor core)
          const int w = S.wtile[par];
          const int64_t slot = S.slotn[par][row];
          const bool act = live && (f - a.delta <= a.tau);
          const unsigned bal = __ballot_sync(0xffffffffu, act);
          unsigned long long key = ~0ull;
          if (live)
            key = ((unsigned long long)ord_f32(f) << 32) |
                  (unsigned long long)local_to_global(slot, a.scene.rank, a.scene.world);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
            key = other < key ? other : key;
          }
          if (lane == 0) {
            S.act[qd] = bal;
            S.kmin[qd] = key;
          }
          named_bar_sync(2, 128);
          int rk = __popc(bal & ((1u << lane) - 1u));
          for (int i = 0; i < qd; ++i) rk += __popc(S.act[i]);
          ridx = act ? rk : -1;
          if (row == 0) {
            unsigned long long km = S.kmin[0];
            int cnt = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              km = S.kmin[i] < km ? S.kmin[i] : km;
              cnt += __popc(S.act[i]);
            }
            if (km != ~0ull) atomicMin(a.ds.wp_key + w, km);
            pend_cnt = cnt;
            pend_b = cnt > 0 ? atomicAdd(a.ds.counter, (unsigned long long)cnt) : 0ull;
          }
        }
        if (p == 7 && cq == 0) prefetch(T + stride, par ^ 1);
        if (p == 8 && cq == 0 && a.detect && row == 0) {
          int base = 0;
          if (pend_cnt > 0) {
            if (pend_b + pend_cnt > (unsigned long long)a.ds.max_active) {
              atomicOr(a.ds.counter + 1, 1ull);
              base = -1;
            } else {
              base = (int)pend_b;
            }
          }
          S.sbase = base;
          a.ds.tile_meta[T] = make_int2(base, pend_cnt);
        }
        if (p == 10 && cq <= 1) {
          // the next tile's point, slot and q row (cp.async by quarter 0 at phase 7) become
          // visible to both staging quarters; S.sbase (phase 8) to quarter 0
          if (cq == 0) cp_async_wait_all();
          named_bar_sync(3, 256);
        }
      } else {
        // ---- g0 = W1^T e1 (16 columns); d f / d q by the chain rule (R3) ----
        uint32_t r[16];
        if (cq == 0) {
          ld16(tL, r);
          wait_ld();
        }
        if (T + stride < n_tiles) live_n = stage_a1(par ^ 1);
        if (cq == 0) {
          const int w = S.wtile[par];
          const int64_t slot = S.slotn[par][row];
          float gq[kNdof];
          gq[0] = a.tgrad ? __uint_as_float(r[3]) : -__uint_as_float(r[0]);
          gq[1] = a.tgrad ? __uint_as_float(r[4]) : -__uint_as_float(r[1]);
#pragma unroll
          for (int i = 0; i < 7; ++i) gq[2 + i] = __uint_as_float(r[5 + i]);
          if (a.detect) {
            const int base = S.sbase;
            ridx = (ridx >= 0 && base >= 0) ? base + ridx : -1;
            if (ridx >= 0) {
              float4 *dst = reinterpret_cast<float4 *>(a.ds.staging + ridx);
              dst[0] = make_float4(f, gq[0], gq[1], gq[2]);
              dst[1] = make_float4(gq[3], gq[4], gq[5], gq[6]);
              dst[2] = make_float4(gq[7], gq[8], __uint_as_float((unsigned)w),
                                   __uint_as_float((unsigned)local_to_global(slot, a.scene.rank, a.scene.world)));
            }
          } else if (a.grads && slot < lb) {
            float *o = a.grads + ((int64_t)w * lb + slot) * kNdof;
            if (a.project) {  // NEXT-3: q_z = q - f M^{-1} grad_q f (Theorem 1.2)
              const float *qw = S.qn[par];
#pragma unroll
              for (int i = 0; i < kNdof; ++i) o[i] = live ? qw[i] - (f * gq[i]) * a.minv[i] : 0.f;
            } else {
#pragma unroll
              for (int i = 0; i < kNdof; ++i) o[i] = live ? gq[i] : 0.f;
            }
          }
        }
      }
    };
    phase(std::integral_constant<int, 0>{});
    phase(std::integral_constant<int, 1>{});
    phase(std::integral_constant<int, 2>{});
    phase(std::integral_constant<int, 3>{});
    phase(std::integral_constant<int, 4>{});
    phase(std::integral_constant<int, 5>{});
    phase(std::integral_constant<int, 6>{});
    phase(std::integral_constant<int, 7>{});
    phase(std::integral_constant<int, 8>{});
    phase(std::integral_constant<int, 9>{});
    phase(std::integral_constant<int, 10>{});
    phase(std::integral_constant<int, 11>{});
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

}  // namespace

cudaError_t launch_mlp_tc_sp(const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  if (a.frame) return cudaErrorInvalidValue;  // (softplus: translation frame only)
  const int smem = (int)sizeof(SmemSP) + 1024;
  cudaError_t e = cudaFuncSetAttribute(k_mlp_tc_sp, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t n_tiles = a.part.tile_wp ? (int64_t)num_sms : (int64_t)a.n_wp * a.tiles_per_wp;
  int64_t grid = n_tiles < num_sms ? n_tiles : num_sms;
  if (grid < 1) return cudaSuccess;
  k_mlp_tc_sp<<<(unsigned)grid, kThreads, smem, s>>>(w, a);
  return cudaGetLastError();
}

}  // namespace gcdf
