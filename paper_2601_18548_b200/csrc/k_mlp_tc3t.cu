// k_mlp_tc3t.cu -- K2t: K2b (k_mlp_tc.cu) with THREE tiles in flight sharing a pool of two
// TMEM accumulators.  Same math, rounding points, UMMA sequence, weight layouts and outputs
// as K2b (translation frame; fp16 or bf16 operands, fp32 accumulation); DESIGN.md section 5
// "K2t" has the schedule arithmetic.
//
// Paper steps (PAPER.md lines): base-frame bias :388/:171; "7-layer MLP" on [p, q] :284;
// value + gradient :394; constraint f - delta >= 0 :362-363; union = min :164; c_gcdf
// order :414-435.
//
// Why: in K2b each slot's chain MMA (576 cycles) -> commit (~300) -> epilogue (~450) ->
// hand-off (~200) must hide behind the other slot's 576 MMA cycles, which caps the tensor
// pipe near 61 %.  A third slot would hide it, but 3 x (128 D + 64 A) TMEM columns do not
// fit in 512.  D, however, is live only from the MMA's start to the epilogue's LAST TMEM
// load; A from the epilogue's stores to the next MMA's end.  So: D is a pool of two buffers
// used by issue order (phase k of the CTA -> D[k % 2]), each slot keeps its own A, and the
// epilogue releases its D buffer ("dfree") as soon as its loads have completed, before the
// ALU work.  TMEM = D[0] [0,128) + D[1] [128,256) + A[s] [256 + 64 s, +64) + ones [448,456).
// The layer-1 operands x are staged in A[s]'s first 16 columns (K2b's original layout).
//
// Issue order (one MMA warp): round r of the CTA holds tiles base + r stride + s, s < a_r
// (a_r = 3 except in the last round); phases p = 0..11 of the round are issued slot by slot,
// so phase p of slot s in round r is the CTA's k = 36 r + p a_r + s-th phase.  Before issuing
// phase k of slot s the MMA warp waits for (1) slot s's previous epilogue (its A; epi_done[s])
// and (2) the epilogue of phase k - 2 to have read D[k % 2] (dfree[k % 2]).
// 24 epilogue warps: warp 8 s + 4 hh + qd = slot s, accumulator column half hh (units
// 64 hh .. 64 hh + 63), TMEM lane quarter qd (the K2b per-thread work).
#include "gcdf_internal.h"
#include "tc_ptx.h"

namespace gcdf {
namespace {

using namespace tc;

constexpr int H = 128;
constexpr int kSlots = 3;
constexpr int kEpiWarps = 8 * kSlots;
constexpr int kMmaWarp = kEpiWarps;   // warps kMmaWarp + (k & 1) issue the CTA's phase k
constexpr int kThreads = (kEpiWarps + 2) * 32;
constexpr int kEpiPerSlot = 256;
constexpr int kPhases = 12;
constexpr int kMasks = 5;
constexpr int kWBytes = 5 * H * H * 2;
constexpr int kW1tBytes = 16 * H * 2;
constexpr int kB1Bytes = 32 * H * 2;
constexpr int kBextCore = H * 16;     // K-core 0 of a [128][16] bias block {b_hi, b_lo, 0..}
constexpr int kBextSrcBytes = 16 * H * 2;  // one K2b bias block (core 0 | zero core 1)
constexpr int kZeroBytes = H * 16;    // shared zero K-core 1 of the five bias blocks
constexpr uint32_t kColA = 256, kColOnes = 448;
template <bool F16> constexpr uint32_t kIdescFwd = idesc_f16kind(128, 128, false, F16);
template <bool F16> constexpr uint32_t kIdescBwd = idesc_f16kind(128, 128, true, F16);
template <bool F16> constexpr uint32_t kIdescFin = idesc_f16kind(128, 16, false, F16);

struct __align__(1024) SmemT {
  uint8_t w[kWBytes];           // W_2..W_6, SW128 (the K2b image)
  uint8_t w1t[kW1tBytes];       // W1^T [16][128], SW128
  uint8_t b1[kB1Bytes];         // layer-1 split weights [128][32], no swizzle
  uint8_t bext[5][kBextCore];   // bias blocks, K-core 0 only
  uint8_t zero[kZeroBytes];     // (after bext: the descriptors' LBO offsets are positive)
  float w7half[H];
  uint32_t w7h[H / 2];
  uint32_t one;
  union {                       // [slot]: the layer-6 partial sums (phase 5), then the point
    float fpart[2][H];          // of the slot's next tile (written after phase 5's barrier,
    float4 ptn[H];              // read at phase 11)
  } pp[kSlots];
  float qn[kSlots][2][12];      // [slot][tile parity] q row
  int wnx[kSlots];
  int wtile[kSlots][2];
  uint32_t slotn[kSlots][2][H]; // [slot][tile parity][row] local scene slot (~0: padding)
  uint32_t mask[kSlots][kMasks][2][kEpiPerSlot];
  uint64_t mma_done[kSlots];
  uint64_t epi_done[kSlots];
  uint64_t dfree[2];
  unsigned act[kSlots][4];
  unsigned long long kmin[kSlots][4];
  int sbase[kSlots];
  uint32_t issued;              // phases issued (the two MMA warps alternate)
  uint32_t tmem_base;
};
static_assert(sizeof(SmemT) + 1024 <= 232448, "SmemT exceeds the 227 KB of shared memory per CTA");

DEVI unsigned ord_f32(float f) {
  unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
template <bool F16>
DEVI float round16(float x) {
  const uint32_t p = pack2<F16>(x, 0.f);
  if constexpr (F16) {
    float f;
    asm("{\n\t.reg .b16 t;\n\tmov.b16 t, %1;\n\tcvt.f32.f16 %0, t;\n\t}" : "=f"(f) : "h"((unsigned short)(p & 0xffffu)));
    return f;
  } else {
    return __uint_as_float(p << 16);
  }
}
template <bool F16>
DEVI void split3(float x, float *o) {
  const float hi = round16<F16>(x);
  o[0] = hi;
  o[1] = x - hi;
  o[2] = hi;
}
DEVI uint32_t add7fff(uint32_t pk, uint32_t one) { return pk * one + 0x7fff7fffu; }
DEVI uint32_t mask_group_f(uint32_t pk01, uint32_t pk23, int k, uint32_t one) {
  const uint32_t x = prmt(add7fff(pk01, one), add7fff(pk23, one), 0x7531u);
  return (x >> k) & (0x80808080u >> k);
}
DEVI uint32_t nz_halves(uint32_t pk, uint32_t one) { return prmt(add7fff(pk, one), 0u, 0xbb99u); }

template <bool F16>
__global__ void __launch_bounds__(kThreads, 1) k_mlp_tc3t(const WeightsBF16 W, const QueryArgs a) {
  extern __shared__ uint8_t smem_raw[];
  SmemT &S = *reinterpret_cast<SmemT *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
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
    for (int l = 0; l < 5; ++l)
      copy16(S.bext[l], static_cast<const uint8_t *>(W.bext_nosw) + l * kBextSrcBytes, kBextCore);
    for (int i = tid; i < kZeroBytes / 16; i += kThreads) reinterpret_cast<uint4 *>(S.zero)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < H; i += kThreads) S.w7half[i] = 0.5f * __ldg(W.w7 + i);
    if (tid == 0) S.one = 1u;
    for (int i = tid; i < H / 2; i += kThreads) S.w7h[i] = pack2<F16>(__ldg(W.w7 + 2 * i), __ldg(W.w7 + 2 * i + 1));
  }
  if (warp == 0) {
    tmem_alloc(&S.tmem_base, 512);
    tmem_relinquish();
  }
  const int64_t n_tiles = query_tiles(a);
  const int64_t base0 = (int64_t)blockIdx.x * kSlots, stride = (int64_t)gridDim.x * kSlots;
  if (tid == 32) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&S.mma_done[s], 1);
      mbar_init(&S.epi_done[s], kEpiPerSlot);
    }
    for (int b = 0; b < 2; ++b) mbar_init(&S.dfree[b], kEpiPerSlot);
    S.issued = 0u;
    fence_barrier_init();
  }
  if (tid < kSlots * kNdof) {  // q rows of the slots' first tiles (later tiles: cp.async, phases 1-3)
    const int s0 = tid / kNdof, i = tid - s0 * kNdof;
    const int64_t T0 = base0 + s0;
    if (T0 < n_tiles) {
      const int w0 = tile_step(a, T0);
      S.qn[s0][0][i] = __ldg(a.q + (int64_t)w0 * kNdof + i);
      if (i == 0) S.wtile[s0][0] = w0;
    }
  }
  fence_proxy_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = S.tmem_base;
  const int64_t lb = a.scene.local_bound;

  if (warp >= kMmaWarp) {
    // ===================== two MMA warps: warp kMmaWarp + (k & 1) issues phase k ==========
    // A tcgen05.commit stalls its issuing thread while the committed UMMAs drain; alternating
    // issuers keep the next phase's issue off that stall (K2b's "two issuers").
    const uint32_t me = (uint32_t)(warp - kMmaWarp);
    const uint32_t sw = smem_u32(S.w), sw1t = smem_u32(S.w1t), sb1 = smem_u32(S.b1), sbx = smem_u32(S.bext);
    const uint32_t szero = smem_u32(S.zero);
    volatile uint32_t *issued = &S.issued;
    uint32_t k = 0;                      // the CTA's phase number
    uint32_t pe[kSlots] = {0u, 0u, 0u};  // epi_done completions per slot (both warps track all)
    for (int64_t rb = base0; rb < n_tiles; rb += stride) {
      const int ar = (int)(n_tiles - rb < kSlots ? n_tiles - rb : kSlots);
#pragma unroll 1
      for (int p = 0; p < kPhases; ++p) {
#pragma unroll 1
        for (int s = 0; s < ar; ++s, ++k) {
          const uint32_t par = pe[s] & 1u;
          ++pe[s];
          if ((k & 1u) != me) continue;
          mbar_wait(&S.epi_done[s], par);
          if (k >= 2) mbar_wait(&S.dfree[k & 1u], ((k >> 1) - 1u) & 1u);
          const long long tw = clock64();
          while (*issued != k) {
            if (clock64() - tw > (1ll << 34)) __trap();
          }
          fence_after();
          const uint32_t d = tbase + 128u * (k & 1u), av = tbase + kColA + 64u * (uint32_t)s;
          // (the UMMAs, then the turn, then the commit: the other warp issues during the commit)
          if (p == 0) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
              mma_ts_elect(d, av + 8u * kk, sdesc_nosw(sb1 + kk * 2 * 2048, 2048, 128), kIdescFwd<F16>, kk > 0);
          } else if (p < 6) {
            const uint32_t wb = sw + (uint32_t)(p - 1) * (H * H * 2);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_ts_elect(d, av + 8u * kk, sdesc_sw128(wb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                           kIdescFwd<F16>, kk > 0);
            const uint32_t st = sbx + (uint32_t)(p - 1) * kBextCore;
            mma_ts_elect(d, tbase + kColOnes, sdesc_nosw(st, szero - st, 128), kIdescFwd<F16>, 1u);
          } else if (p < 11) {
            const uint32_t wb = sw + (uint32_t)(10 - p) * (H * H * 2);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_ts_elect(d, av + 8u * kk, sdesc_sw128(wb + kk * 2048, 16384, 1024), kIdescBwd<F16>, kk > 0);
          } else {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_ts_elect(d, av + 8u * kk, sdesc_sw128(sw1t + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024),
                           kIdescFin<F16>, kk > 0);
          }
          *issued = k + 1u;
          commit_elect(&S.mma_done[s]);
        }
      }
    }
    __syncwarp();
    fence_before();
    __syncthreads();
    return;
  }

  // ===================== epilogue warps ==================================================
  const int s = warp >> 3;          // tile slot
  const int hh = (warp >> 2) & 1;   // accumulator column half
  const int qd = warp & 3;          // TMEM lane quarter (warp % 4)
  const int row = qd * 32 + lane;
  const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
  const uint32_t tL = tbase + lane_off;
  const uint32_t tA = tL + kColA + 64u * (uint32_t)s + 32u * hh;
  const int u0 = 64 * hh;
  uint32_t *mk = &S.mask[s][0][0][hh * 128 + row];
  const uint32_t one = S.one;
  if (s == 0 && hh == 0) {  // the constant ones block of the bias steps (never overwritten)
    const uint32_t ones[8] = {pack2<F16>(1.f, 1.f), 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    st8(tL + kColOnes, ones);
  }
  auto hand_off = [&]() {
    wait_st();
    fence_before();
    mbar_arrive(&S.epi_done[s]);
  };
  auto release_d = [&](int b) {  // this thread's loads of D[b] are complete
    fence_before();
    mbar_arrive(&S.dfree[b]);
  };
  auto next_pt = [&](int64_t TT, int par) {  // (half 0) slot and point of row `row` -> smem
    int wn = 0;
    int64_t sl = 0;
    bool ok = false;
    if (TT < n_tiles) tile_pair(a, TT, row, wn, sl, ok);
    S.slotn[s][par][row] = ok ? (uint32_t)sl : ~0u;
    S.pp[s].ptn[row] = ok ? __ldg(a.scene.pts + sl) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto stage_q = [&](int p, int64_t TT, int par) {  // (K2b) q row of tile TT -> S.qn[s][par]
    if (hh != 0 || qd != 0 || TT >= n_tiles) return;
    if (p == 1) {
      if (a.part.tile_wp && lane == 0) {
        cp_async4(&S.wnx[s], a.part.tile_wp + TT);
        cp_async_commit();
      }
    } else {
      int wn;
      if (a.part.tile_wp) {
        if (lane == 0) cp_async_wait_all();
        __syncwarp();
        wn = S.wnx[s];
      } else {
        wn = (int)(TT / a.tiles_per_wp);
      }
      if (lane < kNdof) cp_async4(&S.qn[s][par][lane], a.q + (int64_t)wn * kNdof + lane);
      cp_async_commit();
      if (lane == 0) S.wtile[s][par] = wn;
    }
  };
  auto stage_a1 = [&](int par) -> bool {  // (K2b) split layer-1 operands -> A
    const float *qw = S.qn[s][par];
    float v[16];
    bool lv = false;
    if (hh == 0) {
      const float4 pt = S.pp[s].ptn[row];
      lv = S.slotn[s][par][row] != ~0u && pt.w > 0.f;
      split3<F16>(pt.x - qw[0], v);  // A2: p' = p - [q_x, q_y, 0]
      split3<F16>(pt.y - qw[1], v + 3);
      split3<F16>(pt.z, v + 6);
      split3<F16>(qw[2], v + 9);
      split3<F16>(qw[3], v + 12);
      v[15] = round16<F16>(qw[4]);
    } else {
      const float j2 = qw[4];
      const float j2h = round16<F16>(j2);
      v[0] = j2 - j2h;
      v[1] = j2h;
#pragma unroll
      for (int i = 0; i < 4; ++i) split3<F16>(qw[5 + i], v + 2 + 3 * i);
      v[14] = 1.f;
      v[15] = 1.f;
    }
    uint32_t a1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a1[i] = pack2<F16>(v[2 * i], v[2 * i + 1]);
    st8(tL + kColA + 64u * (uint32_t)s + 8u * hh, a1);
    return lv;
  };

  uint32_t ph = 0u;  // mma_done[s] parity
  int it = 0;
  bool live_n = false;
  if (base0 + s < n_tiles) {
    if (hh == 0) next_pt(base0 + s, 0);
    live_n = stage_a1(0);
    hand_off();
  }
  for (int64_t rb = base0; rb + s < n_tiles; rb += stride, ++it) {
    const int64_t T = rb + s;
    const int ar = (int)(n_tiles - rb < kSlots ? n_tiles - rb : kSlots);
    const uint32_t k0 = (uint32_t)(36 * it + s);  // the CTA's phase number of this tile's phase 0
    const bool live = live_n;
    float f = 0.f;
    int ridx = -1;
    unsigned long long pend_b = 0ull;
    int pend_cnt = 0;
#pragma unroll 1
    for (int p = 0; p < kPhases; ++p) {
      const int b = (int)((k0 + (uint32_t)(p * ar)) & 1u);  // D buffer of this phase
      const uint32_t tD = tL + 128u * (uint32_t)b + (uint32_t)u0;
      mbar_wait(&S.mma_done[s], ph);
      ph ^= 1u;
      fence_after();
      if (p < 5) {
        // ---- forward layer l = p + 1: h = ReLU(z) -> A, 1-bit masks -> smem ----
        uint32_t rbf[2][16], m = 0u;
        ld16(tD, rbf[0]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < 3) ld16(tD + 16 * (c + 1), rbf[(c + 1) & 1]);
          const uint32_t *rr = rbf[c & 1];
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            pk[j >> 1] = pack2_relu<F16>(__uint_as_float(rr[j]), __uint_as_float(rr[j + 1]));
            pk[(j >> 1) + 1] = pack2_relu<F16>(__uint_as_float(rr[j + 2]), __uint_as_float(rr[j + 3]));
            m |= mask_group_f(pk[j >> 1], pk[(j >> 1) + 1], ((c & 1) * 16 + j) >> 2, one);
          }
          st8(tA + 8 * c, pk);
          if (c & 1) {
            mk[(p * 2 + (c >> 1)) * kEpiPerSlot] = m;
            m = 0u;
          }
          if (c < 3) {
            wait_ld();
            if (c == 2) release_d(b);  // all four chunks of D are in registers
          }
        }
        hand_off();
        if (p == 1 || p == 3) stage_q(p, T + stride, (it + 1) & 1);
      } else if (p == 5) {
        // ---- layer 6: e6 = w7 (.) 1[z6 > 0] -> A; f = w7 . ReLU(z6) + b7 (fp32) ----
        float fa[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t rbf[2][16];
        ld16(tD, rbf[0]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int cb = 16 * c;
          if (c < 3) ld16(tD + cb + 16, rbf[(c + 1) & 1]);
          const uint32_t *rr = rbf[c & 1];
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            const float4 w7 = *reinterpret_cast<const float4 *>(S.w7half + u0 + cb + j);
            const uint2 w2 = *reinterpret_cast<const uint2 *>(S.w7h + (u0 + cb + j) / 2);
            const float z0 = __uint_as_float(rr[j]), z1 = __uint_as_float(rr[j + 1]);
            const float z2 = __uint_as_float(rr[j + 2]), z3 = __uint_as_float(rr[j + 3]);
            pk[j >> 1] = w2.x & nz_halves(pack2_relu<F16>(z0, z1), one);
            pk[(j >> 1) + 1] = w2.y & nz_halves(pack2_relu<F16>(z2, z3), one);
            fa[0] = fmaf(w7.x, z0 + fabsf(z0), fa[0]);
            fa[1] = fmaf(w7.y, z1 + fabsf(z1), fa[1]);
            fa[2] = fmaf(w7.z, z2 + fabsf(z2), fa[2]);
            fa[3] = fmaf(w7.w, z3 + fabsf(z3), fa[3]);
          }
          st8(tA + cb / 2, pk);
          if (c < 3) {
            wait_ld();
            if (c == 2) release_d(b);
          }
        }
        hand_off();
        S.pp[s].fpart[hh][row] = (fa[0] + fa[1]) + (fa[2] + fa[3]);
        if (hh == 0 && qd == 0) cp_async_wait_all();  // S.qn of the next tile (stage_q)
        named_bar_sync(1 + s, kEpiPerSlot);
        if (hh == 0) {
          f = S.pp[s].fpart[0][row] + S.pp[s].fpart[1][row] + W.b7;
          if (!a.detect) {
            const int w = S.wtile[s][it & 1];
            const int64_t slot = S.slotn[s][it & 1][row];
            if (slot < lb) a.values[(int64_t)w * lb + slot] = live ? f : __int_as_float(0x7f800000);
          }
        }
        named_bar_sync(1 + s, kEpiPerSlot);  // fpart read by every row before ptn overwrites it
        if (hh == 0) next_pt(T + stride, (it + 1) & 1);  // the next tile's point, used at phase 11
      } else if (p < 11) {
        // ---- backward: g_{l-1} = D; e_{l-1} = g (.) 1[z_{l-1} > 0] -> A ----
        const int mi = 10 - p;
        const uint32_t mw[2] = {mk[(mi * 2) * kEpiPerSlot], mk[(mi * 2 + 1) * kEpiPerSlot]};
        uint32_t rbf[2][16];
        ld16(tD, rbf[0]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < 3) ld16(tD + 16 * (c + 1), rbf[(c + 1) & 1]);
          const uint32_t *rr = rbf[c & 1];
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            uint32_t lo, hi;
            mask_expand(mw[c >> 1], ((c & 1) * 16 + j) >> 2, lo, hi);
            pk[j >> 1] = pack2<F16>(__uint_as_float(rr[j]), __uint_as_float(rr[j + 1])) & lo;
            pk[(j >> 1) + 1] = pack2<F16>(__uint_as_float(rr[j + 2]), __uint_as_float(rr[j + 3])) & hi;
          }
          st8(tA + 8 * c, pk);
          if (c < 3) {
            wait_ld();
            if (c == 2) release_d(b);
          }
        }
        hand_off();
        if (p == 6 && hh == 0 && a.detect) {
          // A6/A7: threshold, per-tile slots, per-waypoint min key (K2b)
          const int w = S.wtile[s][it & 1];
          const int64_t slot = S.slotn[s][it & 1][row];
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
            S.act[s][qd] = bal;
            S.kmin[s][qd] = key;
          }
          named_bar_sync(4 + s, 128);
          int rk = __popc(bal & ((1u << lane) - 1u));
          for (int i = 0; i < qd; ++i) rk += __popc(S.act[s][i]);
          ridx = act ? rk : -1;
          if (row == 0) {
            unsigned long long km = S.kmin[s][0];
            int cnt = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              km = S.kmin[s][i] < km ? S.kmin[s][i] : km;
              cnt += __popc(S.act[s][i]);
            }
            if (km != ~0ull) atomicMin(a.ds.wp_key + w, km);
            pend_cnt = cnt;
            pend_b = cnt > 0 ? atomicAdd(a.ds.counter, (unsigned long long)cnt) : 0ull;
          }
        }
        if (p == 8 && hh == 0 && a.detect && row == 0) {
          int base = 0;
          if (pend_cnt > 0) {
            if (pend_b + pend_cnt > (unsigned long long)a.ds.max_active) {
              atomicOr(a.ds.counter + 1, 1ull);
              base = -1;
            } else {
              base = (int)pend_b;
            }
          }
          S.sbase[s] = base;
          a.ds.tile_meta[T] = make_int2(base, pend_cnt);
        }
      } else {
        // ---- g0 = W1^T e1 (16 columns of D[b]); the next tile's x; outputs (R3) ----
        uint32_t r[16];
        if (hh == 0) {
          ld16(tL + 128u * (uint32_t)b, r);
          wait_ld();
        }
        release_d(b);
        if (T + stride < n_tiles) {
          live_n = stage_a1((it + 1) & 1);
          hand_off();
        }
        if (hh == 0) {
          const int w = S.wtile[s][it & 1];
          const int64_t slot = S.slotn[s][it & 1][row];
          float gq[kNdof];
          gq[0] = a.tgrad ? __uint_as_float(r[3]) : -__uint_as_float(r[0]);
          gq[1] = a.tgrad ? __uint_as_float(r[4]) : -__uint_as_float(r[1]);
#pragma unroll
          for (int i = 0; i < 7; ++i) gq[2 + i] = __uint_as_float(r[5 + i]);
          if (a.detect) {
            named_bar_sync(4 + s, 128);  // S.sbase[s] (phase 8, row 0) is visible
            const int base = S.sbase[s];
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
              const float *qw = S.qn[s][it & 1];
#pragma unroll
              for (int i = 0; i < kNdof; ++i) o[i] = live ? qw[i] - (f * gq[i]) * a.minv[i] : 0.f;
            } else {
#pragma unroll
              for (int i = 0; i < kNdof; ++i) o[i] = live ? gq[i] : 0.f;
            }
          }
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <bool F16>
cudaError_t launch_t(const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  const int smem = (int)sizeof(SmemT) + 1024;
  cudaError_t e = cudaFuncSetAttribute(k_mlp_tc3t<F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t n_tiles = a.part.tile_wp ? (int64_t)kSlots * num_sms : (int64_t)a.n_wp * a.tiles_per_wp;
  int64_t grid = (n_tiles + kSlots - 1) / kSlots;
  if (grid > num_sms) grid = num_sms;
  if (grid < 1) return cudaSuccess;
  k_mlp_tc3t<F16><<<(unsigned)grid, kThreads, smem, s>>>(w, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mlp_tc3t(bool f16, const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  if (a.frame || a.act != 1) return cudaErrorInvalidValue;
  return f16 ? launch_t<true>(w, a, num_sms, s) : launch_t<false>(w, a, num_sms, s);
}

}  // namespace gcdf
