// k_mlp_tc3.cu -- K2c: the fp32-accurate tensor-core path (GCDF_FP16X3, SURVEY §8(f)
// NEXT-4 "FP32-accurate tensor path via split emulation"): the same fused pair generation
// + base-frame transform + 7-layer MLP forward + input-gradient backward (+ threshold /
// min / per-tile compaction) as K2b (k_mlp_tc.cu), with every hidden GEMM evaluated on
// 3-term split fp16 operands so that the result meets the fp32 tolerances of the
// north star (1e-4 relative / 1e-5 absolute) instead of the 16-bit ones.
//
// Paper steps: as K2b (PAPER.md:388/:171 transform, :284 MLP, :394 value + gradient,
// :362-363 threshold, :164 min, :414-435 order).  DESIGN.md §5 "K2c".
//
// Split arithmetic (R25): x = x_hi + x_lo with x_hi = x truncated to 11
// significant bits (exactly representable in fp16) and x_lo = fp16(x - x_hi); for each
// product  a w ~= a_hi w_hi + a_lo w_hi + a_hi w_lo  (the dropped a_lo w_lo is ~2^-22 |a w|),
// three 128x128x16 UMMAs per K step, fp32 accumulation in TMEM.  Layer 1 already uses this
// split in K2b (K = 32); the biases enter as {1, 1} x {b_hi, b_lo}.
//
// Design differences from K2b (H = 128, one persistent CTA per SM, 576 threads):
//   * TMEM per slot: D [0,128), A_hi [128,192), A_lo [192,256) -- both 256-column slots
//     are full, so the bias step is an SS-mode UMMA with a "ones" A block in shared memory.
//   * W_hi and W_lo of the five hidden layers (320 KB) do not fit in shared memory: they
//     are streamed from L2 through a 2-buffer ring of 64 KB [hi | lo] layer images with
//     1-D cp.async.bulk (measured: ~170 GB/s per SM with all 148 SMs streaming,
//     tools/probes/l2_bulk_probe.cu; a layer is needed once per ~3 us of MMA work).  Both
//     slots run the same phase in turn, so one load serves both tiles; the phase -> layer
//     sequence of a tile is W2 W3 W4 W5 W6 W6 W5 W4 W3 W2, i.e. 8 loads per tile ("runs":
//     W6 is used twice in a row, W2 at the end of a tile and the start of the next).
//     The slot that issues last in a tile pair loads run r + 1 when it starts run r; the
//     buffer it overwrites held run r - 1, whose UMMAs have all completed (its own
//     epilogue saw them complete before handing off, and the tensor pipe runs in order).
//   * The epilogue writes two A operands (hi and lo) per phase.
#include "gcdf_internal.h"
#include "tc_ptx.h"

namespace gcdf {
namespace {

using namespace tc;

constexpr int H = 128;
constexpr int kEpiWarps = 16;
constexpr int kWarps = kEpiWarps + 2;
constexpr int kThreads = kWarps * 32;
constexpr int kEpiPerSlot = 256;
constexpr int kPhases = 12;
constexpr int kMasks = 5;
constexpr int kHalfBytes = H * H * 2;          // one 16-bit SW128 layer image, 32 KB
constexpr int kLayerBytes = 2 * kHalfBytes;    // [hi | lo]
constexpr int kW1tBytes = 16 * H * 2;          // 4 KB (x 2: hi, lo)
constexpr int kB1Bytes = 32 * H * 2;
constexpr int kBextBytes = 16 * H * 2;
constexpr int kOnesBytes = 16 * H * 2;
constexpr uint32_t kColAhi = 128, kColAlo = 192;
// F16: the 16-bit operand type of the split (GCDF_FP16X3: fp16; GCDF_BF16X3: bf16)
template <bool F16> constexpr uint32_t kIdescFwd = idesc_f16kind(128, 128, false, F16);
template <bool F16> constexpr uint32_t kIdescBwd = idesc_f16kind(128, 128, true, F16);
template <bool F16> constexpr uint32_t kIdescFin = idesc_f16kind(128, 16, false, F16);

struct __align__(1024) Smem3 {
  uint8_t ring[2][kLayerBytes];    // streamed W_l images [hi SW128 | lo SW128]
  uint8_t w1t[2][kW1tBytes];       // W1^T [16][128] hi, lo (SW128)
  uint8_t b1[kB1Bytes];            // layer-1 split weights [128][32], no swizzle (as K2b)
  uint8_t bext[5][kBextBytes];     // hidden-layer bias blocks [128][16] {b_hi, b_lo}, no swizzle
  uint8_t ones[kOnesBytes];        // SS-mode A block [128][16]: {1, 1, 0, ...} per row
  float w7half[H];
  uint32_t w7hi[H / 2], w7lo[H / 2];  // w7 split, packed fp16 pairs
  uint32_t one;
  float fpart[2][2][H];
  float4 ptn[2][H];
  float2 pprime[2][2][H];
  float qn[2][2][12];
  int wnx[2];
  int wtile[2][2];
  uint32_t slotn[2][2][H];
  uint32_t mask[2][kMasks][2][kEpiPerSlot];
  uint64_t mma_done[2];
  uint64_t epi_done[2];
  uint64_t ring_full[2][2];        // [buffer][hi, lo] bulk-copy completion
  uint64_t turnb[2];           // [slot] "your turn" (the other slot's phase is issued)
  unsigned act[2][4];
  unsigned long long kmin[2][4];
  int sbase[2];
  uint32_t tmem_base;
};
static_assert(sizeof(Smem3) + 1024 <= 232448, "Smem3 exceeds the 227 KB of shared memory per CTA");

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
// x_hi: x truncated to the type's significand (fp16: 11 significant bits, exact in fp16 in its
// normal range; bf16: 8, exact in bf16 everywhere), same sign as x
template <bool F16>
DEVI float trunc_hi(float x) { return __uint_as_float(__float_as_uint(x) & (F16 ? 0xffffe000u : 0xffff0000u)); }
DEVI uint32_t add7fff(uint32_t pk, uint32_t one) { return pk * one + 0x7fff7fffu; }
DEVI uint32_t mask_group_f(uint32_t pk01, uint32_t pk23, int k, uint32_t one) {
  const uint32_t x = prmt(add7fff(pk01, one), add7fff(pk23, one), 0x7531u);
  return (x >> k) & (0x80808080u >> k);
}
DEVI uint32_t nz_halves(uint32_t pk, uint32_t one) { return prmt(add7fff(pk, one), 0u, 0xbb99u); }

// run (streamed-layer use) of phase p of the CTA's tile number t (phases 1..10), and its layer
DEVI int run_of(int t, int p) { return 8 * t + (p <= 5 ? p - 1 : (p == 6 ? 4 : p - 2)); }
DEVI int layer_of(int r) {
  if (r == 0) return 0;
  const int i = (r - 1) & 7;
  return i < 4 ? i + 1 : 7 - i;  // 1 2 3 4 3 2 1 0
}
DEVI bool starts_run(int t, int p) { return (p >= 2 && p <= 10 && p != 6) || (p == 1 && t == 0); }

template <bool F16, bool kSE2>
__global__ void __launch_bounds__(kThreads, 1) k_mlp_tc3(const WeightsBF16 W, const QueryArgs a) {
  extern __shared__ uint8_t smem_raw[];
  Smem3 &S = *reinterpret_cast<Smem3 *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n_tiles = query_tiles(a);
  const int64_t lb = a.scene.local_bound;
  const int64_t stride = 2 * (int64_t)gridDim.x;
  const uint8_t *w3 = static_cast<const uint8_t *>(W.w3_sw128);

  // ---- one-time setup ----
  {
    auto copy16 = [&](void *dst, const void *src, int bytes) {
      const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
      uint4 *d4 = reinterpret_cast<uint4 *>(dst);
      for (int i = tid; i < bytes / 16; i += kThreads) d4[i] = __ldg(s4 + i);
    };
    copy16(S.w1t, W.w1t3_sw128, 2 * kW1tBytes);
    copy16(S.b1, W.b1_nosw, kB1Bytes);
    copy16(S.bext, W.bext_nosw, 5 * kBextBytes);
    for (int i = tid; i < kOnesBytes / 4; i += kThreads)  // element (row, k) at row*16 + (k/8)*2048 + (k%8)*2
      reinterpret_cast<uint32_t *>(S.ones)[i] = (i % 4 == 0 && i < H * 4) ? pack2<F16>(1.f, 1.f) : 0u;
    for (int i = tid; i < H; i += kThreads) S.w7half[i] = 0.5f * __ldg(W.w7 + i);
    for (int i = tid; i < H / 2; i += kThreads) {
      const float x0 = __ldg(W.w7 + 2 * i), x1 = __ldg(W.w7 + 2 * i + 1);
      const float h0 = trunc_hi<F16>(x0), h1 = trunc_hi<F16>(x1);
      S.w7hi[i] = pack2<F16>(h0, h1);
      S.w7lo[i] = pack2<F16>(x0 - h0, x1 - h1);
    }
    if (tid == 0) S.one = 1u;
  }
  if (warp == 0) {
    tmem_alloc(&S.tmem_base, 512);
    tmem_relinquish();
  }
  if (tid == 32) {
    mbar_init(&S.mma_done[0], 1);
    mbar_init(&S.mma_done[1], 1);
    mbar_init(&S.epi_done[0], kEpiPerSlot);
    mbar_init(&S.epi_done[1], kEpiPerSlot);
    for (int b = 0; b < 2; ++b)
      for (int h = 0; h < 2; ++h) mbar_init(&S.ring_full[b][h], 1);
    mbar_init(&S.turnb[0], 1);
    mbar_init(&S.turnb[1], 1);
    mbar_arrive(&S.turnb[0]);  // slot 0 issues the first phase
    fence_barrier_init();
  }
  if (tid < 2 * kNdof) {
    const int s0 = tid / kNdof, i = tid - s0 * kNdof;
    const int64_t T0 = (int64_t)blockIdx.x * 2 + s0;
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

  // streamed layer run r -> ring buffer r & 1 (hi and lo halves complete separately)
  auto load_run = [&](int r) {
    const int b = r & 1;
    const uint8_t *src = w3 + (size_t)layer_of(r) * kLayerBytes;
    if (lane == 0) {
      mbar_expect_tx(&S.ring_full[b][0], kHalfBytes);
      bulk_g2s(S.ring[b], src, kHalfBytes, &S.ring_full[b][0]);
      mbar_expect_tx(&S.ring_full[b][1], kHalfBytes);
      bulk_g2s(S.ring[b] + kHalfBytes, src + kHalfBytes, kHalfBytes, &S.ring_full[b][1]);
    }
    __syncwarp();
  };

  if (warp >= kEpiWarps) {
    // ===================== MMA warps: warp 16 + s issues slot s's UMMAs =====================
    const int ss = warp - kEpiWarps;
    const uint32_t sw1t = smem_u32(S.w1t), sb1 = smem_u32(S.b1), sbx = smem_u32(S.bext);
    const uint64_t ones_desc = sdesc_nosw(smem_u32(S.ones), 2048, 128);
    const uint32_t d = tbase + (uint32_t)ss * 256u;
    const uint32_t ahi = d + kColAhi, alo = d + kColAlo;
    if (ss == 0 && (int64_t)blockIdx.x * 2 < n_tiles) {  // the first two runs (W2, W3)
      load_run(0);
      load_run(1);
    }
    uint32_t ph = 0u;
    uint32_t seq = (uint32_t)ss;
    int t = 0;
    for (int64_t base = (int64_t)blockIdx.x * 2; base < n_tiles; base += stride, ++t) {
      const bool two = base + 1 < n_tiles;
      if (ss == 1 && !two) break;
      const bool producer = two ? ss == 1 : ss == 0;
      const bool next_tile = base + stride < n_tiles;
#pragma unroll 1
      for (int p = 0; p < kPhases; ++p, seq += 2) {
        mbar_wait(&S.epi_done[ss], ph);
        ph ^= 1u;
        // the turn: an mbarrier (a waiting MMA warp polls try_wait instead of spinning on a
        // shared counter, which took issue slots from the epilogue warps)
        if (two) mbar_wait(&S.turnb[ss], (seq >> 1) & 1u);
        fence_after();
        if (p == 0) {  // layer 1: K = 32 split operands in A_hi (bias included)
#pragma unroll
          for (int k = 0; k < 2; ++k)
            mma_ts_elect(d, ahi + 8u * k, sdesc_nosw(sb1 + k * 2 * 2048, 2048, 128), kIdescFwd<F16>, k > 0);
        } else if (p < 11) {
          const int r = run_of(t, p);
          if (producer && starts_run(t, p) && r >= 1 && (r + 1 <= 8 * t + 8 || next_tile)) load_run(r + 1);
          const int b = r & 1;
          const uint32_t par = (uint32_t)(r >> 1) & 1u;
          const uint32_t whi = smem_u32(S.ring[b]), wlo = whi + kHalfBytes;
          const bool fwd = p < 6;
          auto bdesc = [&](uint32_t wb, int k) {
            return fwd ? sdesc_sw128(wb + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024)
                       : sdesc_sw128(wb + k * 2048, 16384, 1024);
          };
          const uint32_t id = fwd ? kIdescFwd<F16> : kIdescBwd<F16>;
          // (each 8-UMMA group from one asm block: a lean issue stream, see tc_ptx.h)
          mbar_wait(&S.ring_full[b][0], par);
          if (fwd) {
            umma8_kmajor_elect(d, ahi, bdesc(whi, 0), id, 0u);
            umma8_kmajor_elect(d, alo, bdesc(whi, 0), id, 1u);
          } else {
            umma8_mnmajor_elect(d, ahi, bdesc(whi, 0), id, 0u);
            umma8_mnmajor_elect(d, alo, bdesc(whi, 0), id, 1u);
          }
          mbar_wait(&S.ring_full[b][1], par);
          if (fwd) umma8_kmajor_elect(d, ahi, bdesc(wlo, 0), id, 1u);
          else umma8_mnmajor_elect(d, ahi, bdesc(wlo, 0), id, 1u);
          if (fwd) mma_ss_elect(d, ones_desc, sdesc_nosw(sbx + (uint32_t)(p - 1) * kBextBytes, 2048, 128), kIdescFwd<F16>, 1u);
        } else {  // g0 = e1 W1 (N = 16)
          const uint32_t hi1 = sw1t, lo1 = sw1t + kW1tBytes;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            mma_ts_elect(d, ahi + 8u * k, sdesc_sw128(hi1 + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024), kIdescFin<F16>, k > 0);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            mma_ts_elect(d, alo + 8u * k, sdesc_sw128(hi1 + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024), kIdescFin<F16>, 1u);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            mma_ts_elect(d, ahi + 8u * k, sdesc_sw128(lo1 + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024), kIdescFin<F16>, 1u);
        }
        if (two) {
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.turnb[ss ^ 1]);
        }
        commit_elect(&S.mma_done[ss]);
      }
    }
    __syncwarp();
    fence_before();
    __syncthreads();
    return;
  }

  // ===================== epilogue warps =====================
  const int s = warp >> 3;
  const int hh = (warp >> 2) & 1;
  const int qd = warp & 3;
  const int row = qd * 32 + lane;
  const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
  const uint32_t tS = tbase + (uint32_t)s * 256u + lane_off;
  const uint32_t tD = tS + 64u * hh;
  const uint32_t tAh = tS + kColAhi + 32u * hh, tAl = tS + kColAlo + 32u * hh;
  const int u0 = 64 * hh;
  uint32_t *mk = &S.mask[s][0][0][hh * 128 + row];
  auto hand_off = [&]() {
    wait_st();
    fence_before();
    mbar_arrive(&S.epi_done[s]);
  };
  auto prefetch_pt = [&](int64_t TT, int par) {
    int wn = 0;
    int64_t sl = 0;
    bool ok = false;
    if (TT < n_tiles) tile_pair(a, TT, row, wn, sl, ok);
    S.slotn[s][par][row] = ok ? (uint32_t)sl : ~0u;
    cp_async16(&S.ptn[s][row], ok ? (const void *)(a.scene.pts + sl) : (const void *)a.scene.pts, ok ? 16u : 0u);
    cp_async_commit();
  };
  auto stage_q = [&](int p, int64_t TT, int par) {
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
  // A2 + A1 of tile TT (as K2b; the split layer-1 operands go to A_hi, K = 32)
  auto stage_a1 = [&](int par) -> bool {
    const float *qw = S.qn[s][par];
    float v[16];
    bool lv = false;
    if (hh == 0) {
      const float4 pt = S.ptn[s][row];
      lv = S.slotn[s][par][row] != ~0u && pt.w > 0.f;
      float dx = pt.x - qw[0], dy = pt.y - qw[1], th = qw[2];
      if constexpr (kSE2) {
        float sn, cs;
        sincosf(th, &sn, &cs);  // (accurate sincos: this is the fp32-tolerance path)
        const float rx = cs * dx + sn * dy;
        dy = -sn * dx + cs * dy;
        dx = rx;
        th = 0.f;
        S.pprime[s][par][row] = make_float2(dx, dy);
      }
      split3<F16>(dx, v);
      split3<F16>(dy, v + 3);
      split3<F16>(pt.z, v + 6);
      split3<F16>(th, v + 9);
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
    st8(tS + kColAhi + 8u * hh, a1);
    hand_off();
    return lv;
  };
  const uint32_t one = S.one;
  uint32_t ph = 0u;
  int it = 0;
  bool live_n = false;
  if ((int64_t)blockIdx.x * 2 + s < n_tiles) {
    if (hh == 0) {
      prefetch_pt((int64_t)blockIdx.x * 2 + s, 0);
      cp_async_wait_all();
    }
    live_n = stage_a1(0);
  }
  for (int64_t T = (int64_t)blockIdx.x * 2 + s; T < n_tiles; T += stride, ++it) {
    const bool live = live_n;
    float f = 0.f;
    int ridx = -1;
    unsigned long long pend_b = 0ull;
    int pend_cnt = 0;
#pragma unroll 1
    for (int p = 0; p < kPhases; ++p) {
      mbar_wait(&S.mma_done[s], ph);
      ph ^= 1u;
      fence_after();
      if (p < 5) {
        // ---- forward layer p + 1: z = D; h = ReLU(z) -> A_hi, A_lo (3-term split) ----
        uint32_t rb[2][16], m = 0u;
        ld16(tD, rb[0]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < 3) ld16(tD + 16 * (c + 1), rb[(c + 1) & 1]);
          const uint32_t *rr = rb[c & 1];
          uint32_t ph_[8], pl_[8];
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const float z0 = __uint_as_float(rr[j]), z1 = __uint_as_float(rr[j + 1]);
            const float h0 = trunc_hi<F16>(z0), h1 = trunc_hi<F16>(z1);  // same sign as z: ReLU per part
            ph_[j >> 1] = pack2_relu<F16>(h0, h1);
            pl_[j >> 1] = pack2_relu<F16>(z0 - h0, z1 - h1);
          }
#pragma unroll
          for (int j = 0; j < 8; j += 2) m |= mask_group_f(ph_[j], ph_[j + 1], ((c & 1) * 16 + 2 * j) >> 2, one);
          st8(tAh + 8 * c, ph_);
          st8(tAl + 8 * c, pl_);
          if (c & 1) {
            mk[(p * 2 + (c >> 1)) * kEpiPerSlot] = m;
            m = 0u;
          }
          if (c < 3) wait_ld();
        }
        hand_off();
        if (p == 1 || p == 3) stage_q(p, T + stride, (it + 1) & 1);
      } else if (p == 5) {
        // ---- layer 6: e6 = w7 (.) 1[z6 > 0] -> A (w7 split); f = w7 . ReLU(z6) + b7 ----
        float fa[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t rb[2][16];
        ld16(tD, rb[0]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int cb = 16 * c;
          if (c < 3) ld16(tD + cb + 16, rb[(c + 1) & 1]);
          const uint32_t *rr = rb[c & 1];
          uint32_t pkh[8], pkl[8];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            const float4 w7 = *reinterpret_cast<const float4 *>(S.w7half + u0 + cb + j);
            const uint2 wh = *reinterpret_cast<const uint2 *>(S.w7hi + (u0 + cb + j) / 2);
            const uint2 wl = *reinterpret_cast<const uint2 *>(S.w7lo + (u0 + cb + j) / 2);
            const float z0 = __uint_as_float(rr[j]), z1 = __uint_as_float(rr[j + 1]);
            const float z2 = __uint_as_float(rr[j + 2]), z3 = __uint_as_float(rr[j + 3]);
            const uint32_t m01 = nz_halves(pack2_relu<F16>(z0, z1), one);
            const uint32_t m23 = nz_halves(pack2_relu<F16>(z2, z3), one);
            pkh[j >> 1] = wh.x & m01;
            pkh[(j >> 1) + 1] = wh.y & m23;
            pkl[j >> 1] = wl.x & m01;
            pkl[(j >> 1) + 1] = wl.y & m23;
            fa[0] = fmaf(w7.x, z0 + fabsf(z0), fa[0]);
            fa[1] = fmaf(w7.y, z1 + fabsf(z1), fa[1]);
            fa[2] = fmaf(w7.z, z2 + fabsf(z2), fa[2]);
            fa[3] = fmaf(w7.w, z3 + fabsf(z3), fa[3]);
          }
          st8(tAh + cb / 2, pkh);
          st8(tAl + cb / 2, pkl);
          if (c < 3) wait_ld();
        }
        hand_off();
        S.fpart[s][hh][row] = (fa[0] + fa[1]) + (fa[2] + fa[3]);
        if (hh == 0 && qd == 0) cp_async_wait_all();
        named_bar_sync(1 + s, kEpiPerSlot);
        if (hh == 0) {
          f = S.fpart[s][0][row] + S.fpart[s][1][row] + W.b7;
          if (!a.detect) {
            const int w = S.wtile[s][it & 1];
            const int64_t slot = S.slotn[s][it & 1][row];
            if (slot < lb) a.values[(int64_t)w * lb + slot] = live ? f : __int_as_float(0x7f800000);
          }
        }
      } else if (p < 11) {
        // ---- backward: g = D; e = g (.) 1[z > 0] -> A_hi, A_lo ----
        const int mi = 10 - p;
        const uint32_t mw[2] = {mk[(mi * 2) * kEpiPerSlot], mk[(mi * 2 + 1) * kEpiPerSlot]};
        uint32_t rb[2][16];
        ld16(tD, rb[0]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < 3) ld16(tD + 16 * (c + 1), rb[(c + 1) & 1]);
          const uint32_t *rr = rb[c & 1];
          uint32_t pkh[8], pkl[8];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            uint32_t lo, hi;
            mask_expand(mw[c >> 1], ((c & 1) * 16 + j) >> 2, lo, hi);
            const float g0 = __uint_as_float(rr[j]), g1 = __uint_as_float(rr[j + 1]);
            const float g2 = __uint_as_float(rr[j + 2]), g3 = __uint_as_float(rr[j + 3]);
            const float h0 = trunc_hi<F16>(g0), h1 = trunc_hi<F16>(g1), h2 = trunc_hi<F16>(g2), h3 = trunc_hi<F16>(g3);
            pkh[j >> 1] = pack2<F16>(h0, h1) & lo;
            pkh[(j >> 1) + 1] = pack2<F16>(h2, h3) & hi;
            pkl[j >> 1] = pack2<F16>(g0 - h0, g1 - h1) & lo;
            pkl[(j >> 1) + 1] = pack2<F16>(g2 - h2, g3 - h3) & hi;
          }
          st8(tAh + 8 * c, pkh);
          st8(tAl + 8 * c, pkl);
          if (c < 3) wait_ld();
        }
        hand_off();
        if (p == 6 && hh == 0 && a.detect) {
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
          named_bar_sync(3 + s, 128);
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
        if (p == 7 && hh == 0) prefetch_pt(T + stride, (it + 1) & 1);
      } else {
        // ---- g0 = W1^T e1 (16 columns); d f / d q by the chain rule (R3) ----
        uint32_t r[16];
        if (hh == 0) {
          ld16(tS, r);
          wait_ld();
          cp_async_wait_all();
        }
        if (T + stride < n_tiles) live_n = stage_a1((it + 1) & 1);
        if (hh == 0) {
          const int w = S.wtile[s][it & 1];
          const int64_t slot = S.slotn[s][it & 1][row];
          float gq[kNdof];
          gq[0] = a.tgrad ? __uint_as_float(r[3]) : -__uint_as_float(r[0]);
          gq[1] = a.tgrad ? __uint_as_float(r[4]) : -__uint_as_float(r[1]);
#pragma unroll
          for (int i = 0; i < 7; ++i) gq[2 + i] = __uint_as_float(r[5 + i]);
          if constexpr (kSE2) {
            float sn, cs;
            sincosf(S.qn[s][it & 1][2], &sn, &cs);
            const float gx = __uint_as_float(r[0]), gy = __uint_as_float(r[1]);
            const float2 pp = S.pprime[s][it & 1][row];
            gq[0] = -(cs * gx - sn * gy);
            gq[1] = -(sn * gx + cs * gy);
            gq[2] = gx * pp.y - gy * pp.x;
          }
          if (a.detect) {
            named_bar_sync(3 + s, 128);
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
            if (a.project) {
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

template <bool F16, bool kSE2>
cudaError_t launch_t(const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  const int smem = (int)sizeof(Smem3) + 1024;
  cudaError_t e = cudaFuncSetAttribute(k_mlp_tc3<F16, kSE2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t n_tiles = a.part.tile_wp ? 2 * (int64_t)num_sms : (int64_t)a.n_wp * a.tiles_per_wp;
  int64_t grid = (n_tiles + 1) / 2;
  if (grid > num_sms) grid = num_sms;
  if (grid < 1) return cudaSuccess;
  k_mlp_tc3<F16, kSE2><<<(unsigned)grid, kThreads, smem, s>>>(w, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mlp_tc3(bool f16, const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  if (f16) return a.frame ? launch_t<true, true>(w, a, num_sms, s) : launch_t<true, false>(w, a, num_sms, s);
  return a.frame ? launch_t<false, true>(w, a, num_sms, s) : launch_t<false, false>(w, a, num_sms, s);
}

}  // namespace gcdf
