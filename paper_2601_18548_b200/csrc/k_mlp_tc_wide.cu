// k_mlp_tc_wide.cu -- K2w: the H = 256 variant (NEXT-4, R27) of the fused tcgen05
// path: pair generation + base-frame bias + 7-layer MLP [12, 256 x 6, 1] forward + input-
// gradient backward (+ threshold / min / per-tile compaction in detect mode), fp16 operands,
// fp32 accumulation in TMEM.
//
// Paper steps (PAPER.md lines): base-frame bias :388/:171; "7-layer MLP" on [p, q] :284
// (width not given: H = 256 is the wide reading of R8); value + gradient :394; constraint
// f - delta >= 0 :362-363; union = min :164; c_gcdf order :414-435.
//
// What differs from K2b (k_mlp_tc.cu, H = 128):
//   * the five hidden layers are 5 x 128 KB in fp16 -- more than shared memory -- so they are
//     streamed from L2 (where the 1.25 MB chunk sequence stays resident) through a ring of
//     four 32 KB slots by a producer warp (1-D cp.async.bulk completing on the slot's "full"
//     mbarrier); the MMA warp releases a slot with a tcgen05.commit on its "empty" mbarrier
//     once the UMMAs of both output halves that read it complete.  The chunk sequence of a tile is laid out in
//     consumption order: W_2..W_6 K-major [out][in] (forward), then W_6^T..W_2^T K-major
//     [in][out] (backward), 4 chunks of 64 K-columns per layer -- so forward and backward
//     UMMAs use the same descriptor pattern and the producer streams one contiguous image.
//   * one tile in flight (two would need 2 x 384 TMEM columns), pipelined by output half:
//     a layer is two N = 128 UMMA chains (units 0..127, then 128..255; 16 K-steps of
//     128 x 128 x 16 each).  The epilogue warps of half 0 start as soon as half 0's chain
//     completes, while the tensor core runs half 1; the next layer's half-0 chain starts
//     its first 8 K-steps (which read only the units half 0 produced) before half 1's
//     epilogue is done.  That needs the A operand double-buffered by phase parity:
//     TMEM = D [0, 256) fp32 (half h at 128 h) + A[0] [256, 384) + A[1] [384, 512) fp16;
//     the layer-1 operands live in A[0]'s first 16 columns, and the bias steps take their
//     constant "ones" A block from shared memory (SS-mode UMMA).
//   * 16 epilogue warps own 32 rows x 64 units each (warps 8 h .. 8 h + 7: output half h;
//     the K2b per-thread work), ReLU masks in shared memory in K2b's byte-sign form.
// Rounding points: those of K2b (EMU_FP16 in the oracle: W_2..W_6, W_1 (gradient), h_1..h_5,
// e_6..e_1 rounded to fp16; layer 1 split hi/lo; f = w7 . h6 in fp32).
#include <type_traits>

#include "gcdf_internal.h"
#include "tc_ptx.h"

namespace gcdf {
namespace {

using namespace tc;

constexpr int H = 256;
constexpr int kEpiWarps = 16;
constexpr int kMmaWarp = 16, kProdWarp = 17;
constexpr int kThreads = 18 * 32;
constexpr int kEpi = kEpiWarps * 32;
constexpr int kPhases = 12;
constexpr int kMasks = 5;
constexpr int kNS = 4;                      // ring slots
constexpr int kChunk = H * 128;             // 32 KB: [256 rows][64 K-columns] fp16, SW128
constexpr int kChunksPerTile = 40;          // 5 layers x 4 forward + 5 x 4 backward
constexpr int kW1tBytes = 16 * H * 2;       // 8 KB
constexpr int kB1Bytes = 32 * H * 2;        // 16 KB
constexpr int kBextCore = H * 16;           // 4 KB per hidden layer: K-core 0 {b_hi, b_lo, 0..} of [256][16]
constexpr int kZeroBytes = 4096;            // shared all-zero K-core 1 of the bias and ones blocks
constexpr int kOnesBytes = 128 * 16;        // K-core 0 of the ones block [128][16] {1, 1, 0..}
constexpr uint32_t kColA = 256;             // A[b] at 256 + 128 b
constexpr uint32_t kIdescW = idesc_f16kind(128, 128, false, true);
constexpr uint32_t kIdescFin = idesc_f16kind(128, 16, false, true);

struct __align__(1024) SmemW {
  uint8_t ring[kNS][kChunk];
  uint8_t w1t[kW1tBytes];
  uint8_t b1[kB1Bytes];
  uint8_t bext[5][kBextCore];
  uint8_t ones[kOnesBytes];
  uint8_t zero[kZeroBytes];        // (after bext and ones: the descriptors' LBO offsets are positive)
  uint32_t mask[kMasks][2][kEpi];  // ReLU masks [layer][32-unit word][thread]
  uint32_t one;
  float fpart[4][128];
  float4 ptn[128];
  float qn[2][12];
  int wtile[2];
  uint32_t slotn[2][128];
  uint64_t mma_done[2], epi_done[2];  // [output half]
  uint64_t full[kNS], empty[kNS];
  unsigned act[4];
  unsigned long long kmin[4];
  int sbase;
  uint32_t tmem_base;
};
static_assert(sizeof(SmemW) + 1024 <= 232448, "SmemW exceeds the 227 KB of shared memory per CTA");

DEVI unsigned ord_f32(float f) {
  unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
DEVI float round16(float x) {
  const uint32_t p = pack_f16(x, 0.f);
  float f;
  asm("{\n\t.reg .b16 t;\n\tmov.b16 t, %1;\n\tcvt.f32.f16 %0, t;\n\t}" : "=f"(f) : "h"((unsigned short)(p & 0xffffu)));
  return f;
}
DEVI void split3(float x, float *o) {
  const float hi = round16(x);
  o[0] = hi;
  o[1] = x - hi;
  o[2] = hi;
}
// K2b's mask helpers (the "+ 0x7fff7fff" on the FMA pipe through a runtime one)
DEVI uint32_t add7fff(uint32_t pk, uint32_t one) { return pk * one + 0x7fff7fffu; }
DEVI uint32_t mask_group_f(uint32_t pk01, uint32_t pk23, int k, uint32_t one) {
  const uint32_t x = prmt(add7fff(pk01, one), add7fff(pk23, one), 0x7531u);
  return (x >> k) & (0x80808080u >> k);
}

__global__ void __launch_bounds__(kThreads, 1) k_mlp_tc_wide(const WeightsBF16 W, const QueryArgs a) {
  extern __shared__ uint8_t smem_raw[];
  SmemW &S = *reinterpret_cast<SmemW *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    auto copy16 = [&](void *dst, const void *src, int bytes) {
      const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
      uint4 *d4 = reinterpret_cast<uint4 *>(dst);
      for (int i = tid; i < bytes / 16; i += kThreads) d4[i] = __ldg(s4 + i);
    };
    copy16(S.w1t, W.w1t_sw128, kW1tBytes);
    copy16(S.b1, W.b1_nosw, kB1Bytes);
    copy16(S.bext, W.bext_nosw, 5 * kBextCore);
    for (int i = tid; i < kZeroBytes / 16; i += kThreads) reinterpret_cast<uint4 *>(S.zero)[i] = make_uint4(0, 0, 0, 0);
    for (int r = tid; r < 128; r += kThreads)  // ones block, no-swizzle K-major: row r at (r / 8) * 128 + (r % 8) * 16
      *reinterpret_cast<uint4 *>(S.ones + (r >> 3) * 128 + (r & 7) * 16) = make_uint4(pack_f16(1.f, 1.f), 0u, 0u, 0u);
    if (tid == 0) S.one = 1u;
  }
  if (warp == 0) {
    tmem_alloc(&S.tmem_base, 512);
    tmem_relinquish();
  }
  if (tid == 32) {
    for (int h = 0; h < 2; ++h) {
      mbar_init(&S.mma_done[h], 1);
      mbar_init(&S.epi_done[h], kEpi / 2);
    }
    for (int i = 0; i < kNS; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], 1);
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
  const int64_t my_tiles = (int64_t)blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / stride + 1 : 0;

  if (warp == kProdWarp) {
    // ===================== producer: the chunk sequence of every tile through the ring ======
    if (lane == 0) {
      const uint8_t *src = static_cast<const uint8_t *>(W.w_sw128);
      const int64_t total = my_tiles * kChunksPerTile;
      for (int64_t i = 0; i < total; ++i) {
        const int slot = (int)(i % kNS);
        if (i >= kNS) mbar_wait(&S.empty[slot], (uint32_t)((i / kNS - 1) & 1));
        mbar_expect_tx(&S.full[slot], kChunk);
        bulk_g2s(S.ring[slot], src + (i % kChunksPerTile) * kChunk, kChunk, &S.full[slot]);
      }
    }
    __syncwarp();
    fence_before();
    __syncthreads();
    return;
  }
  if (warp == kMmaWarp) {
    // ===================== MMA warp (converged; an elected lane issues) ======================
    const uint32_t sw1t = smem_u32(S.w1t), sb1 = smem_u32(S.b1), sbx = smem_u32(S.bext);
    const uint32_t szero = smem_u32(S.zero), sones = smem_u32(S.ones);
    // bias step of layer l (1..5 = W_2..W_6) for output half h: A = ones (smem), B = rows
    // 128 h.. of the layer's bias block; both K-core 1 halves point at the shared zero block
    const uint64_t a_ones = sdesc_nosw(sones, szero - sones, 128);
    auto b_bias = [&](int l, int h) {
      const uint32_t st = sbx + (uint32_t)(l - 1) * kBextCore + 2048u * (uint32_t)h;
      return sdesc_nosw(st, szero - st, 128);
    };
    uint32_t ph0 = 0u, ph1 = 0u;
    int64_t ci = 0;  // chunks consumed
    auto wait_epi = [&](int h) {
      if (h == 0) { mbar_wait(&S.epi_done[0], ph0); ph0 ^= 1u; }
      else { mbar_wait(&S.epi_done[1], ph1); ph1 ^= 1u; }
      fence_after();
    };
    for (int64_t t = 0; t < my_tiles; ++t) {
#pragma unroll 1
      for (int p = 0; p < kPhases; ++p) {
        const uint32_t ab = tbase + kColA + 128u * (uint32_t)(p & 1);  // A buffer read by phase p
        wait_epi(0);
        if (p == 0) {  // layer 1: K = 32 split operands (bias included), A = A[0] columns 0..15
          wait_epi(1);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int k = 0; k < 2; ++k)
              mma_ts_elect(tbase + 128u * h, ab + 8u * k, sdesc_nosw(sb1 + k * 2 * (H * 16) + 2048 * h, H * 16, 128),
                           kIdescW, k > 0);
            commit_elect(&S.mma_done[h]);
          }
        } else if (p < 11) {
          // hidden layer (forward p = 1..5, backward p = 6..10), 4 streamed chunks of 64 K
          // output half 0: K-steps 0..7 need only the units half 0's epilogue wrote
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            if (c == 2) wait_epi(1);
            const int64_t cc = ci + c;
            mbar_wait(&S.full[cc % kNS], (uint32_t)((cc / kNS) & 1));
            const uint32_t base = smem_u32(S.ring[cc % kNS]);
            umma4_sw128_elect(tbase, ab + 32u * (uint32_t)c, sdesc_sw128(base, 16, 1024), kIdescW, c > 0);
          }
          if (p < 6) mma_ss_elect(tbase, a_ones, b_bias(p, 0), kIdescW, 1u);
          commit_elect(&S.mma_done[0]);
          // output half 1: B rows 128..255 of the same chunks; each chunk's slot is released
          // once these (its last readers) complete
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            const int64_t cc = ci + c;
            const uint32_t base = smem_u32(S.ring[cc % kNS]) + 16384u;
            umma4_sw128_elect(tbase + 128u, ab + 32u * (uint32_t)c, sdesc_sw128(base, 16, 1024), kIdescW, c > 0);
            commit_elect(&S.empty[cc % kNS]);
          }
          if (p < 6) mma_ss_elect(tbase + 128u, a_ones, b_bias(p, 1), kIdescW, 1u);
          commit_elect(&S.mma_done[1]);
          ci += 4;
        } else {  // g0 = e1 W1 (N = 16 rows of W1^T) -> D columns 0..15
          wait_epi(1);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            mma_ts_elect(tbase, ab + 8u * k, sdesc_sw128(sw1t + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024), kIdescFin, k > 0);
          commit_elect(&S.mma_done[0]);
          commit_elect(&S.mma_done[1]);
        }
      }
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
  const int qd = ew & 3;   // TMEM lane quarter
  const int cq = ew >> 2;  // unit quarter: units 64 cq .. 64 cq + 63
  const int row = qd * 32 + lane;
  const int u0 = 64 * cq;
  const uint32_t tL = tbase + ((uint32_t)(qd * 32) << 16);
  const int half = cq >> 1;  // output half of this warp's units
  const uint32_t tD = tL + (uint32_t)u0;
  auto tA = [&](int p) {     // A buffer written by the epilogue of phase p (read by phase p + 1)
    return tL + kColA + 128u * (uint32_t)((p + 1) & 1) + 32u * (uint32_t)cq;
  };
  uint32_t *mk = &S.mask[0][0][tid];  // + (layer * 2 + word) * kEpi
  const uint32_t one = S.one;
  auto hand_off = [&]() {
    wait_st();
    fence_before();
    mbar_arrive(&S.epi_done[half]);
  };
  auto prefetch = [&](int64_t TT, int par) {  // (unit quarter 0) point, slot and q row of tile TT
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
  auto stage_a1 = [&](int par) -> bool {  // layer-1 operands (K2b's split layout) -> TMEM
    const float *qw = S.qn[par];
    bool lv = false;
    if (cq == 0) {
      float v[16];
      const float4 pt = S.ptn[row];
      lv = S.slotn[par][row] != ~0u && pt.w > 0.f;
      split3(pt.x - qw[0], v);  // A2: p' = p - [q_x, q_y, 0]
      split3(pt.y - qw[1], v + 3);
      split3(pt.z, v + 6);
      split3(qw[2], v + 9);
      split3(qw[3], v + 12);
      v[15] = round16(qw[4]);
      uint32_t a1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a1[i] = pack_f16(v[2 * i], v[2 * i + 1]);
      st8(tL + kColA, a1);  // (A[0] columns 0..7: read by phase 0)
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
      st8(tL + kColA + 8u, a1);
    }
    hand_off();
    return lv;
  };

  uint32_t ph = 0u;
  int it = 0;
  bool live_n = false;
  if (my_tiles > 0) {
    if (cq == 0) prefetch(blockIdx.x, 0);
    cp_async_wait_all();
    named_bar_sync(1, kEpi);
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
        // ---- forward layer l = p + 1: h = ReLU(z) -> A (fp16), 1-bit masks -> smem ----
        uint32_t rb[4][16], m = 0u;
        // all four chunks' TMEM loads in flight at once, one wait (K2w has the registers)
#pragma unroll
        for (int c = 0; c < 4; ++c) ld16(tD + 16 * c, rb[c]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t *rr = rb[c];
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            pk[j >> 1] = pack_f16_relu(__uint_as_float(rr[j]), __uint_as_float(rr[j + 1]));
            pk[(j >> 1) + 1] = pack_f16_relu(__uint_as_float(rr[j + 2]), __uint_as_float(rr[j + 3]));
            m |= mask_group_f(pk[j >> 1], pk[(j >> 1) + 1], ((c & 1) * 16 + j) >> 2, one);
          }
          st8(tA(p) + 8 * c, pk);
          if (c & 1) {
            mk[(p * 2 + (c >> 1)) * kEpi] = m;
            m = 0u;
          }
        }
        hand_off();
      } else if (p == 5) {
        // ---- layer 6: e6 = w7 (.) 1[z6 > 0] -> A; f = w7 . ReLU(z6) + b7 (fp32) ----
        float fa[4] = {0.f, 0.f, 0.f, 0.f};
        // the output row from the kernel parameters at compile-time offsets (one body per unit
        // quarter): direct constant-bank operands, no shared-memory loads (as in K2b)
        auto layer6 = [&](auto u0c) {
          constexpr int U0 = decltype(u0c)::value;
          uint32_t rb[4][16];
#pragma unroll
          for (int c = 0; c < 4; ++c) ld16(tD + 16 * c, rb[c]);
          wait_ld();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int cb = 16 * c;
            const uint32_t *rr = rb[c];
            uint32_t pk[8];
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              const int u = U0 + cb + j;
              const float z0 = __uint_as_float(rr[j]), z1 = __uint_as_float(rr[j + 1]);
              const float z2 = __uint_as_float(rr[j + 2]), z3 = __uint_as_float(rr[j + 3]);
              // e6 masks from the sign bytes of the fp32 z6 (as K2b): 1[z >= +0]
              pk[j >> 1] = W.w7h_p[u / 2] & ~prmt(rr[j], rr[j + 1], 0xffbbu);
              pk[(j >> 1) + 1] = W.w7h_p[u / 2 + 1] & ~prmt(rr[j + 2], rr[j + 3], 0xffbbu);
              fa[0] = fmaf(W.w7half_p[u], z0 + fabsf(z0), fa[0]);
              fa[1] = fmaf(W.w7half_p[u + 1], z1 + fabsf(z1), fa[1]);
              fa[2] = fmaf(W.w7half_p[u + 2], z2 + fabsf(z2), fa[2]);
              fa[3] = fmaf(W.w7half_p[u + 3], z3 + fabsf(z3), fa[3]);
            }
            st8(tA(p) + cb / 2, pk);
          }
        };
        switch (cq) {
          case 0: layer6(std::integral_constant<int, 0>{}); break;
          case 1: layer6(std::integral_constant<int, 64>{}); break;
          case 2: layer6(std::integral_constant<int, 128>{}); break;
          default: layer6(std::integral_constant<int, 192>{}); break;
        }
        hand_off();
        S.fpart[cq][row] = (fa[0] + fa[1]) + (fa[2] + fa[3]);
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
        // ---- backward: g_{l-1} = D; e_{l-1} = g (.) 1[z_{l-1} > 0] -> A ----
        const int mi = 10 - p;
        const uint32_t mw[2] = {mk[(mi * 2) * kEpi], mk[(mi * 2 + 1) * kEpi]};
        uint32_t rb[4][16];
        // all four chunks' TMEM loads in flight at once, one wait (K2w has the registers)
#pragma unroll
        for (int c = 0; c < 4; ++c) ld16(tD + 16 * c, rb[c]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t *rr = rb[c];
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            uint32_t lo, hi;
            mask_expand(mw[c >> 1], ((c & 1) * 16 + j) >> 2, lo, hi);
            pk[j >> 1] = pack_f16(__uint_as_float(rr[j]), __uint_as_float(rr[j + 1])) & lo;
            pk[(j >> 1) + 1] = pack_f16(__uint_as_float(rr[j + 2]), __uint_as_float(rr[j + 3])) & hi;
          }
          st8(tA(p) + 8 * c, pk);
        }
        hand_off();
        if (p == 6 && cq == 0 && a.detect) {
          // A6/A7: threshold, per-tile slots, per-waypoint min key
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

cudaError_t launch_mlp_tc_wide(const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  if (a.frame || a.act != 1) return cudaErrorInvalidValue;  // (H = 256: ReLU, translation frame)
  const int smem = (int)sizeof(SmemW) + 1024;
  cudaError_t e = cudaFuncSetAttribute(k_mlp_tc_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t n_tiles = a.part.tile_wp ? (int64_t)num_sms : (int64_t)a.n_wp * a.tiles_per_wp;
  int64_t grid = n_tiles < num_sms ? n_tiles : num_sms;
  if (grid < 1) return cudaSuccess;
  k_mlp_tc_wide<<<(unsigned)grid, kThreads, smem, s>>>(w, a);
  return cudaGetLastError();
}

}  // namespace gcdf
