// k_mlp_tc3.cu -- K2c: the split-operand tensor-core path (GCDF_FP16X3: fp32-accurate;
// GCDF_BF16X3: the bf16 path at the north-star tolerance; SURVEY §8(f) NEXT-4 "FP32-accurate
// tensor path via split emulation"): the same fused pair generation + base-frame transform +
// 7-layer MLP forward + input-gradient backward (+ threshold / min / per-tile compaction) as
// K2b (k_mlp_tc.cu), with every hidden GEMM evaluated on 3-term split 16-bit operands.
//
// Paper steps: as K2b (PAPER.md:388/:171 transform, :284 MLP, :394 value + gradient,
// :362-363 threshold, :164 min, :414-435 order).  DESIGN.md §5 "K2c".
//
// Split arithmetic (R25): x = x_hi + x_lo with x_hi = x truncated to the 16-bit
// type's significand (exact in it) and x_lo = round16(x - x_hi); for each product
// a w ~= a_hi w_hi + a_lo w_hi + a_hi w_lo  (the dropped a_lo w_lo is ~2^-22 |a w| for fp16),
// three 128x128x16 UMMAs per K step, fp32 accumulation in TMEM.  Layer 1 uses the K = 32
// split of K2b; the biases enter as {1, 1} x {b_hi, b_lo}.
//
// Design (H = 128, one persistent CTA per SM, 896 threads = 24 epilogue warps + 3 MMA warps
// + 1 detect warp) -- K2b's three-slot schedule with split operands:
//   * Three tiles in flight, 12 MMA phases per tile; TMEM = four 128-column regions used round
//     robin exactly as in K2b (phase k of the CTA writes D to region k % 4 and reads its A from
//     region (k + 1) % 4, written IN PLACE by the slot's previous epilogue).  With the split,
//     K step k of an A operand takes 16 columns -- hi at 16 k .. 16 k + 7, lo at 16 k + 8 ..
//     16 k + 15 -- i.e. exactly the accumulator columns of its own 16 units, so an epilogue
//     chunk overwrites its own columns and nothing else.  The bias step is an SS-mode UMMA
//     against a "ones" block in shared memory (no free TMEM columns for it).
//   * W_hi and W_lo of the five hidden layers (320 KB) do not fit in shared memory: they are
//     streamed from L2 through a 2-buffer ring of 64 KB [hi | lo] layer images with 1-D
//     cp.async.bulk.  The three slots run the same phase in turn, so one load serves three
//     tiles; the phase -> layer sequence of a tile is W2 W3 W4 W5 W6 W6 W5 W4 W3 W2, i.e. 8
//     loads ("runs") per tile.  The last slot with a tile in the round loads run r + 1 when
//     it starts run r; the buffer it overwrites held run r - 1, whose UMMAs have all completed
//     (its own run r - 1 phase completed before its epilogue handed off, and the other
//     slots' run r - 1 phases were issued before it on the in-order tensor pipe).
//   * The epilogue writes two A operands (hi and lo) per chunk; the per-tile detect
//     bookkeeping (A6-A8 atomics) runs on the detect warp, as in K2b.
#include <type_traits>

#include "gcdf_internal.h"
#include "tc_ptx.h"

namespace gcdf {
namespace {

using namespace tc;

DEVI void wait_bar(uint64_t *bar, uint32_t parity) { mbar_wait(bar, parity); }
DEVI void wait_bar_addr(uint32_t addr, uint32_t parity) {
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(addr, parity)) {
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}

constexpr int H = 128;
constexpr int kSlots = 3;
constexpr int kEpiPerSlot = 256;
constexpr int kEpiWarps = kSlots * kEpiPerSlot / 32;  // warps 0..23
constexpr int kMmaWarp0 = kEpiWarps;                  // warp 24 + s issues slot s's UMMAs
constexpr int kDetectWarp = kEpiWarps + kSlots;       // warp 27
constexpr int kWarps = kDetectWarp + 1;
constexpr int kThreads = kWarps * 32;                 // 896
constexpr int kEpiArrivals = kEpiPerSlot / 32;
constexpr int kPhases = 12;
constexpr int kMasks = 5;
constexpr int kHalfBytes = H * H * 2;          // one 16-bit SW128 layer image, 32 KB
constexpr int kLayerBytes = 2 * kHalfBytes;    // [hi | lo]
constexpr int kW1tBytes = 16 * H * 2;          // 4 KB (x 2: hi, lo)
constexpr int kB1Bytes = 32 * H * 2;
constexpr int kBextBytes = 16 * H * 2;
constexpr int kOnesBytes = 16 * H * 2;
constexpr uint32_t kColX = 16;  // a g0 phase's region: g0 at [0, 16), the next tile's x at [16, 32)
// epilogue chunk c = 0..3 of column half h: accumulator columns (= units) 32h + DC(c) .. + 15;
// their split activations go to 32h + DC(c) (hi, 8 columns) and 32h + DC(c) + 8 (lo): K step
// k = (32h + DC(c)) / 16 of the next UMMA reads hi at 16 k and lo at 16 k + 8
__host__ __device__ constexpr uint32_t DC(int c) { return (uint32_t)((c >> 1) * 64 + (c & 1) * 16); }
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
  uint32_t w7hi[H / 2], w7lo[H / 2];  // w7 split, packed 16-bit pairs
  float fpart[kSlots][2][H];       // [slot][column half][row] partial output-layer sums
  float4 ptn[kSlots][H];           // [slot][row] prefetched point of the slot's next tile
  float qn[kSlots][2][12];         // [slot][tile parity] q row of the slot's tile
  int wnx[kSlots];
  int rnx[kSlots];
  int wtile[kSlots][2];
  uint32_t slotn[kSlots][2][H];    // local slot of the pair (~0: padding; bit 31: removed point)
  uint32_t mask[kSlots][kMasks][2][kEpiPerSlot];
  uint64_t mma_done[kSlots];
  uint64_t epi_done[kSlots];
  uint64_t turn[kSlots];
  uint64_t det_in[kSlots];
  uint64_t det_out[kSlots];
  uint64_t ring_full[2][2];        // [buffer][hi, lo] bulk-copy completion
  uint32_t one;
  unsigned act[kSlots][4];
  unsigned long long kmin[kSlots][4];
  int sbase[kSlots];
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

// run (streamed-layer use) of phase p of the CTA's tile round t (phases 1..10), and its layer
DEVI int run_of(int t, int p) { return 8 * t + (p <= 5 ? p - 1 : (p == 6 ? 4 : p - 2)); }
DEVI int layer_of(int r) {
  if (r == 0) return 0;
  const int i = (r - 1) & 7;
  return i < 4 ? i + 1 : 7 - i;  // 1 2 3 4 3 2 1 0
}
DEVI bool starts_run(int t, int p) { return (p >= 2 && p <= 10 && p != 6) || (p == 1 && t == 0); }

// UMMA groups of one phase from ONE asm block each (one elected lane issues; operands are adds
// of immediates to the phase's base values, see K2b).  A of K step k: hi at av + 16 k, lo at
// av + 16 k + 8.
#define K2C_UMMA(AOFF, DOFF, ACC)                                          \
  "add.u32 ra, %1, " #AOFF ";\n\t"                                         \
  "add.u64 rb, %2, " #DOFF ";\n\t"                                         \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, " ACC ";\n\t"
#define K2C_UMMA_B5(AOFF, DOFF)                                            \
  "add.u32 ra, %1, " #AOFF ";\n\t"                                         \
  "add.u64 rb, %5, " #DOFF ";\n\t"                                         \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, pt;\n\t"
#define K2C_HEAD                                                           \
  "{\n\t.reg .pred e, pf, pt;\n\t.reg .b32 ra;\n\t.reg .b64 rb;\n\t"       \
  "elect.sync _|e, 0xffffffff;\n\t"                                        \
  "setp.ne.b32 pf, %4, %4;\n\tsetp.eq.b32 pt, %4, %4;\n\t"
// forward, W_hi (K-major SW128, 2 x 64-column chunks of 16 KB: K step k at + (k / 4) 16384 +
// (k % 4) 32 bytes): A_hi W_hi and A_lo W_hi
DEVI void umma_fwd_hi(uint32_t d, uint32_t av, uint64_t b0, uint32_t idesc) {
  asm volatile(K2C_HEAD
               K2C_UMMA(0, 0, "pf") K2C_UMMA(8, 0, "pt") K2C_UMMA(16, 2, "pt") K2C_UMMA(24, 2, "pt")
               K2C_UMMA(32, 4, "pt") K2C_UMMA(40, 4, "pt") K2C_UMMA(48, 6, "pt") K2C_UMMA(56, 6, "pt")
               K2C_UMMA(64, 1024, "pt") K2C_UMMA(72, 1024, "pt") K2C_UMMA(80, 1026, "pt") K2C_UMMA(88, 1026, "pt")
               K2C_UMMA(96, 1028, "pt") K2C_UMMA(104, 1028, "pt") K2C_UMMA(112, 1030, "pt") K2C_UMMA(120, 1030, "pt")
               "}" ::"r"(d), "r"(av), "l"(b0), "r"(idesc), "r"(0u)
               : "memory");
}
// forward, W_lo: A_hi W_lo, then the bias step (SS: ones [smem] x {b_hi, b_lo})
DEVI void umma_fwd_lo(uint32_t d, uint32_t av, uint64_t b0, uint32_t idesc, uint64_t ones, uint64_t bias) {
  asm volatile(K2C_HEAD
               K2C_UMMA(0, 0, "pt") K2C_UMMA(16, 2, "pt") K2C_UMMA(32, 4, "pt") K2C_UMMA(48, 6, "pt")
               K2C_UMMA(64, 1024, "pt") K2C_UMMA(80, 1026, "pt") K2C_UMMA(96, 1028, "pt") K2C_UMMA(112, 1030, "pt")
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %6, %3, pt;\n\t"
               "}" ::"r"(d), "r"(av), "l"(b0), "r"(idesc), "r"(0u), "l"(ones), "l"(bias)
               : "memory");
}
// backward, W_hi read MN-major (K step k at + k 2048 bytes): A_hi W_hi and A_lo W_hi
DEVI void umma_bwd_hi(uint32_t d, uint32_t av, uint64_t b0, uint32_t idesc) {
  asm volatile(K2C_HEAD
               K2C_UMMA(0, 0, "pf") K2C_UMMA(8, 0, "pt") K2C_UMMA(16, 128, "pt") K2C_UMMA(24, 128, "pt")
               K2C_UMMA(32, 256, "pt") K2C_UMMA(40, 256, "pt") K2C_UMMA(48, 384, "pt") K2C_UMMA(56, 384, "pt")
               K2C_UMMA(64, 512, "pt") K2C_UMMA(72, 512, "pt") K2C_UMMA(80, 640, "pt") K2C_UMMA(88, 640, "pt")
               K2C_UMMA(96, 768, "pt") K2C_UMMA(104, 768, "pt") K2C_UMMA(112, 896, "pt") K2C_UMMA(120, 896, "pt")
               "}" ::"r"(d), "r"(av), "l"(b0), "r"(idesc), "r"(0u)
               : "memory");
}
// backward, W_lo: A_hi W_lo
DEVI void umma_bwd_lo(uint32_t d, uint32_t av, uint64_t b0, uint32_t idesc) {
  asm volatile(K2C_HEAD
               K2C_UMMA(0, 0, "pt") K2C_UMMA(16, 128, "pt") K2C_UMMA(32, 256, "pt") K2C_UMMA(48, 384, "pt")
               K2C_UMMA(64, 512, "pt") K2C_UMMA(80, 640, "pt") K2C_UMMA(96, 768, "pt") K2C_UMMA(112, 896, "pt")
               "}" ::"r"(d), "r"(av), "l"(b0), "r"(idesc), "r"(0u)
               : "memory");
}
// g0 = e1 W1 (N = 16; W1^T hi at %2, lo at %5, K-major SW128 in 2 chunks of 2 KB)
DEVI void umma_g0(uint32_t d, uint32_t av, uint64_t bhi, uint32_t idesc, uint64_t blo) {
  asm volatile(K2C_HEAD
               K2C_UMMA(0, 0, "pf") K2C_UMMA(8, 0, "pt") K2C_UMMA(16, 2, "pt") K2C_UMMA(24, 2, "pt")
               K2C_UMMA(32, 4, "pt") K2C_UMMA(40, 4, "pt") K2C_UMMA(48, 6, "pt") K2C_UMMA(56, 6, "pt")
               K2C_UMMA(64, 128, "pt") K2C_UMMA(72, 128, "pt") K2C_UMMA(80, 130, "pt") K2C_UMMA(88, 130, "pt")
               K2C_UMMA(96, 132, "pt") K2C_UMMA(104, 132, "pt") K2C_UMMA(112, 134, "pt") K2C_UMMA(120, 134, "pt")
               K2C_UMMA_B5(0, 0) K2C_UMMA_B5(16, 2) K2C_UMMA_B5(32, 4) K2C_UMMA_B5(48, 6)
               K2C_UMMA_B5(64, 128) K2C_UMMA_B5(80, 130) K2C_UMMA_B5(96, 132) K2C_UMMA_B5(112, 134)
               "}" ::"r"(d), "r"(av), "l"(bhi), "r"(idesc), "r"(0u), "l"(blo)
               : "memory");
}
// layer 1: K = 32 split operands at A columns kColX, kColX + 8; B (no swizzle) at + k * 4096 bytes
DEVI void umma_l1(uint32_t d, uint32_t av, uint64_t b0, uint32_t idesc) {
  asm volatile(K2C_HEAD
               K2C_UMMA(16, 0, "pf") K2C_UMMA(24, 256, "pt")
               "}" ::"r"(d), "r"(av), "l"(b0), "r"(idesc), "r"(0u)
               : "memory");
}
static_assert(kColX == 16, "umma_l1 reads x at columns 16..31");
#undef K2C_UMMA
#undef K2C_UMMA_B5
#undef K2C_HEAD

// The MMA warp of slot SS (as K2b's mma_loop, plus the weight ring).  TMEM base address 0.
template <bool F16, int SS>
DEVI void mma_loop(Smem3 &S, const QueryArgs &a, const uint8_t *w3, int64_t n_tiles, int64_t stride, int lane) {
  const uint32_t sw1t = smem_u32(S.w1t), sb1 = smem_u32(S.b1), sbx = smem_u32(S.bext);
  const uint64_t ones_desc = sdesc_nosw(smem_u32(S.ones), 2048, 128);
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
  if (SS == 0 && (int64_t)blockIdx.x * kSlots < n_tiles) {  // the first two runs (W2, W3)
    load_run(0);
    load_run(1);
  }
  uint32_t ph = 0u, seq = (uint32_t)SS;
  int t = 0;
  for (int64_t base = (int64_t)blockIdx.x * kSlots; base < n_tiles; base += stride, ++t) {
    const bool real = base + SS < n_tiles;
    const bool last_was_real = t > 0 && base - stride + SS < n_tiles;
    // the round's last slot with a tile streams the next run
    const bool producer = real && (SS == kSlots - 1 || base + SS + 1 >= n_tiles);
    const bool next_tile = base + stride < n_tiles;
#pragma unroll 1
    for (int p = 0; p < kPhases; ++p, seq += kSlots) {
      if (real || (p == 0 && last_was_real)) {
        wait_bar(&S.epi_done[SS], ph);
        ph ^= 1u;
      }
      auto wait_turn = [&]() {
        wait_bar(&S.turn[SS], (seq / kSlots) & 1u);
        fence_after();
      };
      const uint32_t d = 128u * (seq & 3u), av = 128u * ((seq + 1u) & 3u);
      if (!real) {
        wait_turn();
      } else if (p == 0) {
        const uint64_t b0 = sdesc_nosw(sb1, 2048, 128);
        wait_turn();
        umma_l1(d, av, b0, kIdescFwd<F16>);
      } else if (p < 11) {
        const int r = run_of(t, p);
        if (producer && starts_run(t, p) && r >= 1 && (r + 1 <= 8 * t + 8 || next_tile)) load_run(r + 1);
        const int b = r & 1;
        const uint32_t par = (uint32_t)(r >> 1) & 1u;
        const uint32_t whi = smem_u32(S.ring[b]), wlo = whi + kHalfBytes;
        if (p < 6) {
          const uint64_t bh = sdesc_sw128(whi, 16, 1024), bl = sdesc_sw128(wlo, 16, 1024);
          const uint64_t bx = sdesc_nosw(sbx + (uint32_t)(p - 1) * kBextBytes, 2048, 128);
          wait_turn();
          wait_bar(&S.ring_full[b][0], par);
          umma_fwd_hi(d, av, bh, kIdescFwd<F16>);
          wait_bar(&S.ring_full[b][1], par);
          umma_fwd_lo(d, av, bl, kIdescFwd<F16>, ones_desc, bx);
        } else {
          const uint64_t bh = sdesc_sw128(whi, 16384, 1024), bl = sdesc_sw128(wlo, 16384, 1024);
          wait_turn();
          wait_bar(&S.ring_full[b][0], par);
          umma_bwd_hi(d, av, bh, kIdescBwd<F16>);
          wait_bar(&S.ring_full[b][1], par);
          umma_bwd_lo(d, av, bl, kIdescBwd<F16>);
        }
      } else {
        const uint64_t bh = sdesc_sw128(sw1t, 16, 1024), bl = sdesc_sw128(sw1t + kW1tBytes, 16, 1024);
        wait_turn();
        umma_g0(d, av, bh, kIdescFin<F16>, bl);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.turn[(SS + 1) % kSlots]);
      if (real) commit_elect(&S.mma_done[SS]);
    }
  }
}

// The detect warp: per tile, in slot order, combines the four column-half-1 warps' ballots and
// min keys, publishes the per-waypoint min key and allocates the tile's staging records (as K2b)
DEVI void detect_loop(Smem3 &S, const QueryArgs &a, int64_t n_tiles, int64_t stride, int lane) {
  uint32_t ph = 0u;
  int it = 0;
  for (int64_t base = (int64_t)blockIdx.x * kSlots; base < n_tiles; base += stride, ++it) {
    for (int s = 0; s < kSlots; ++s) {
      const int64_t T = base + s;
      if (T >= n_tiles) break;
      wait_bar(&S.det_in[s], (ph >> s) & 1u);
      ph ^= 1u << s;
      unsigned long long km = lane < 4 ? S.kmin[s][lane] : ~0ull;
      int cnt = lane < 4 ? __popc(S.act[s][lane]) : 0;
#pragma unroll
      for (int o = 2; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, km, o);
        km = other < km ? other : km;
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      }
      if (lane == 0) {
        const int w = S.wtile[s][it & 1];
        if (km != ~0ull) atomicMin(a.ds.wp_key + w, km);
        int b = 0;
        if (cnt > 0) {
          const unsigned long long pb = atomicAdd(a.ds.counter, (unsigned long long)cnt);
          if (pb + cnt > (unsigned long long)a.ds.max_active) {
            atomicOr(a.ds.counter + 1, 1ull);
            b = -1;
          } else {
            b = (int)pb;
          }
        }
        S.sbase[s] = b;
        a.ds.tile_meta[T] = make_int2(b, cnt);
        mbar_arrive(&S.det_out[s]);
      }
      __syncwarp();
    }
  }
}

template <bool F16, bool kSE2>
__global__ void __launch_bounds__(kThreads, 1) k_mlp_tc3(const WeightsBF16 W, const QueryArgs a) {
  extern __shared__ uint8_t smem_raw[];
  Smem3 &S = *reinterpret_cast<Smem3 *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n_tiles = query_tiles(a);
  const int64_t lb = a.scene.local_bound;
  const int64_t stride = kSlots * (int64_t)gridDim.x;

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
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&S.mma_done[i], 1);
      mbar_init(&S.epi_done[i], kEpiArrivals);
      mbar_init(&S.turn[i], 1);
      mbar_init(&S.det_in[i], 4);
      mbar_init(&S.det_out[i], 1);
    }
    for (int b = 0; b < 2; ++b)
      for (int h = 0; h < 2; ++h) mbar_init(&S.ring_full[b][h], 1);
    mbar_arrive(&S.turn[0]);  // slot 0 issues the CTA's first phase
    fence_barrier_init();
  }
  if (tid < kSlots * kNdof) {
    const int s0 = tid / kNdof, i = tid - s0 * kNdof;
    const int64_t T0 = (int64_t)blockIdx.x * kSlots + s0;
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
  if (tbase != 0u) __trap();  // the MMA warps address TMEM from column 0

  if (warp >= kEpiWarps) {
    const uint8_t *w3 = static_cast<const uint8_t *>(W.w3_sw128);
    if (warp == kMmaWarp0) mma_loop<F16, 0>(S, a, w3, n_tiles, stride, lane);
    else if (warp == kMmaWarp0 + 1) mma_loop<F16, 1>(S, a, w3, n_tiles, stride, lane);
    else if (warp == kMmaWarp0 + 2) mma_loop<F16, 2>(S, a, w3, n_tiles, stride, lane);
    else if (a.detect) detect_loop(S, a, n_tiles, stride, lane);
    __syncwarp();
    fence_before();
    __syncthreads();
    return;
  }

  // ===================== epilogue warps =====================
  // (the warp index through a lane-0 shuffle: warp-uniform to the compiler, so the TMEM
  // addresses derived from it live in uniform registers, as in K2b)
  const int ew = __shfl_sync(0xffffffffu, warp, 0);
  const int s = ew >> 3;
  const int hh = (ew >> 2) & 1;
  const int qd = ew & 3;
  const int row = qd * 32 + lane;
  const uint32_t tL = tbase + ((uint32_t)(qd * 32) << 16) + 32u * hh;
  uint32_t seq = (uint32_t)s;
  auto region = [&](uint32_t k) { return tL + 128u * (k & 3u); };
  uint32_t *mk = &S.mask[s][0][0][hh * 128 + row];
  const uint32_t bar_mma = smem_u32(&S.mma_done[s]), bar_epi = smem_u32(&S.epi_done[s]);
  const int u0 = 32 * hh;
  auto hand_off = [&]() {
    wait_st();
    fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_addr(bar_epi);
  };
  auto prefetch_pt = [&](int64_t TT, int par) {
    int wn = 0;
    int64_t sl = 0;
    bool ok = false;
    if (TT < n_tiles) {
      if (a.part.tile_wp) {
        tile_pair(a, TT, row, wn, sl, ok);
      } else {
        sl = (int64_t)S.rnx[s] * kTile + row;
        ok = sl < lb;
      }
    }
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
        if (lane == 0) S.rnx[s] = (int)(TT - (int64_t)wn * a.tiles_per_wp);
      }
      if (lane < kNdof) cp_async4(&S.qn[s][par][lane], a.q + (int64_t)wn * kNdof + lane);
      cp_async_commit();
      if (lane == 0) S.wtile[s][par] = wn;
    }
  };
  // A2 + A1 of a tile (as K2b): split layer-1 operands -> columns kColX.. of the region at tx
  // (hh = 0: K 0..15, hh = 1: K 16..31); SE(2): p'_xy kept in pp (half 0) for phase 11
  float2 pp = make_float2(0.f, 0.f);
  auto stage_a1 = [&](int par, uint32_t tx) -> bool {
    const float *qw = S.qn[s][par];
    float v[16];
    bool lv = false;
    if (hh == 0) {
      const float4 pt = S.ptn[s][row];
      const uint32_t sl = S.slotn[s][par][row];
      lv = sl != ~0u && pt.w > 0.f;
      if (sl != ~0u && !lv) S.slotn[s][par][row] = sl | 0x80000000u;
      float dx = pt.x - qw[0], dy = pt.y - qw[1], th = qw[2];
      if constexpr (kSE2) {
        float sn, cs;
        sincosf(th, &sn, &cs);  // (accurate sincos: the fp32-tolerance path)
        const float rx = cs * dx + sn * dy;
        dy = -sn * dx + cs * dy;
        dx = rx;
        th = 0.f;
        pp = make_float2(dx, dy);
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
    st8(tx - 32u * hh + kColX + 8u * hh, a1);
    return lv;
  };
  const uint32_t one = S.one;
  uint32_t ph = 0u;
  int it = 0;
  if ((int64_t)blockIdx.x * kSlots + s < n_tiles) {
    if (hh == 0) {
      int wn;
      int64_t sl;
      bool ok;
      tile_pair(a, (int64_t)blockIdx.x * kSlots + s, row, wn, sl, ok);
      S.slotn[s][0][row] = ok ? (uint32_t)sl : ~0u;
      cp_async16(&S.ptn[s][row], ok ? (const void *)(a.scene.pts + sl) : (const void *)a.scene.pts, ok ? 16u : 0u);
      cp_async_commit();
      cp_async_wait_all();
    }
    stage_a1(0, region(seq + 1u));
    hand_off();
  }
  for (int64_t T = (int64_t)blockIdx.x * kSlots + s; T < n_tiles; T += stride, ++it) {
    float f = 0.f;
    auto phase = [&](auto pc) {
      constexpr int p = decltype(pc)::value;
      wait_bar_addr(bar_mma, ph);
      ph ^= 1u;
      fence_after();
      const uint32_t tD = region(seq);
      if constexpr (p < 5) {
        // ---- forward layer p + 1: z = D (bias folded in); h = ReLU(z) -> A_hi, A_lo in place
        // (hi = trunc(z) has the sign of z: ReLU per part); masks from h_hi ----
        uint32_t rb[2][16], m = 0u;
        ld16(tD + DC(0), rb[0]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < 3) ld16(tD + DC(c + 1), rb[(c + 1) & 1]);
          const uint32_t *rr = rb[c & 1];
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 2)
            pk[j >> 1] = pack2_relu<F16>(trunc_hi<F16>(__uint_as_float(rr[j])), trunc_hi<F16>(__uint_as_float(rr[j + 1])));
#pragma unroll
          for (int j = 0; j < 8; j += 2) m |= mask_group_f(pk[j], pk[j + 1], ((c & 1) * 16 + 2 * j) >> 2, one);
          st8(tD + DC(c), pk);
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const float z0 = __uint_as_float(rr[j]), z1 = __uint_as_float(rr[j + 1]);
            pk[j >> 1] = pack2_relu<F16>(z0 - trunc_hi<F16>(z0), z1 - trunc_hi<F16>(z1));
          }
          st8(tD + DC(c) + 8u, pk);
          if (c & 1) {
            mk[(p * 2 + (c >> 1)) * kEpiPerSlot] = m;
            m = 0u;
          }
          if (c < 3) wait_ld();
        }
        hand_off();
        if constexpr (p == 1 || p == 3) stage_q(p, T + stride, (it + 1) & 1);
      } else if constexpr (p == 5) {
        // ---- layer 6: e6 = w7 (.) 1[z6 > 0] -> A (w7 split); f = w7 . ReLU(z6) + b7 ----
        float fa[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t rb[2][16];
        ld16(tD + DC(0), rb[0]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int cb = u0 + (int)DC(c);
          if (c < 3) ld16(tD + DC(c + 1), rb[(c + 1) & 1]);
          const uint32_t *rr = rb[c & 1];
          uint32_t pkh[8], pkl[8];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            const float4 w7 = *reinterpret_cast<const float4 *>(S.w7half + cb + j);
            const uint2 wh = *reinterpret_cast<const uint2 *>(S.w7hi + (cb + j) / 2);
            const uint2 wl = *reinterpret_cast<const uint2 *>(S.w7lo + (cb + j) / 2);
            const float z0 = __uint_as_float(rr[j]), z1 = __uint_as_float(rr[j + 1]);
            const float z2 = __uint_as_float(rr[j + 2]), z3 = __uint_as_float(rr[j + 3]);
            // e6 masks from the sign bytes of the fp32 z6 (as K2b): 1[z >= +0]
            const uint32_t m01 = ~prmt(rr[j], rr[j + 1], 0xffbbu);
            const uint32_t m23 = ~prmt(rr[j + 2], rr[j + 3], 0xffbbu);
            pkh[j >> 1] = wh.x & m01;
            pkh[(j >> 1) + 1] = wh.y & m23;
            pkl[j >> 1] = wl.x & m01;
            pkl[(j >> 1) + 1] = wl.y & m23;
            fa[0] = fmaf(w7.x, z0 + fabsf(z0), fa[0]);
            fa[1] = fmaf(w7.y, z1 + fabsf(z1), fa[1]);
            fa[2] = fmaf(w7.z, z2 + fabsf(z2), fa[2]);
            fa[3] = fmaf(w7.w, z3 + fabsf(z3), fa[3]);
          }
          st8(tD + DC(c), pkh);
          st8(tD + DC(c) + 8u, pkl);
          if (c < 3) wait_ld();
        }
        hand_off();
        // (the other half reads this partial sum two hand-offs later, ordered by the
        // mbarrier chain, as in K2b)
        S.fpart[s][hh][row] = (fa[0] + fa[1]) + (fa[2] + fa[3]);
        if (hh == 0) {
          if (qd == 0) cp_async_wait_all();  // S.qn of the next tile (stage_q)
          prefetch_pt(T + stride, (it + 1) & 1);
        }
      } else if constexpr (p < 11) {
        // ---- backward: g_{l-1} = D; e_{l-1} = g (.) 1[z_{l-1} > 0] -> A_hi, A_lo in place ----
        constexpr int mi = 10 - p;
        const uint32_t mw[2] = {mk[(mi * 2) * kEpiPerSlot], mk[(mi * 2 + 1) * kEpiPerSlot]};
        uint32_t rb[2][16];
        ld16(tD + DC(0), rb[0]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < 3) ld16(tD + DC(c + 1), rb[(c + 1) & 1]);
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
          st8(tD + DC(c), pkh);
          st8(tD + DC(c) + 8u, pkl);
          if (c < 3) wait_ld();
        }
        hand_off();
        if constexpr (p == 7) {
          if (hh == 1) {
            f = S.fpart[s][0][row] + S.fpart[s][1][row] + W.b7;
            const uint32_t sl = S.slotn[s][it & 1][row];
            const bool live = (sl >> 31) == 0u;  // (padding rows: ~0; removed points: bit 31)
            if (!a.detect) {
              const int w = S.wtile[s][it & 1];
              const int64_t slot = sl & 0x7fffffffu;
              if (slot < lb) a.values[(int64_t)w * lb + slot] = live ? f : __int_as_float(0x7f800000);
            } else {
              // A6/A7: threshold and the warp's min key -> the detect warp
              const int64_t slot = sl & 0x7fffffffu;
              const bool act = live && (f - a.delta <= a.tau);
              const unsigned bal = __ballot_sync(0xffffffffu, act);
              const unsigned khi = live ? ord_f32(f) : 0xffffffffu;
              const unsigned mhi = __reduce_min_sync(0xffffffffu, khi);
              const unsigned klo = (live && khi == mhi) ? (unsigned)local_to_global(slot, a.scene.rank, a.scene.world)
                                                        : 0xffffffffu;
              const unsigned mlo = __reduce_min_sync(0xffffffffu, klo);
              if (lane == 0) {
                S.act[s][qd] = bal;
                S.kmin[s][qd] = ((unsigned long long)mhi << 32) | mlo;
                mbar_arrive(&S.det_in[s]);
              }
            }
          }
        }
      } else {
        // ---- phase 11: g0 = W1^T e1 (columns 0..15) -> d f / d q (R3) and the outputs; both
        // halves stage the next tile's layer-1 operands (columns kColX.. of this region)
        // before the hand-off (as K2b) ----
        uint32_t r[16];
        if (hh == 0) {
          ld16(tD - 32u * hh, r);
          wait_ld();
        }
        const float2 pp_t = pp;
        if (T + stride < n_tiles) {
          if (hh == 0) cp_async_wait_all();
          stage_a1((it + 1) & 1, tD);
        }
        hand_off();
        if (hh == 0) {
          f = S.fpart[s][0][row] + S.fpart[s][1][row] + W.b7;
          const int w = S.wtile[s][it & 1];
          const uint32_t sl = S.slotn[s][it & 1][row];
          const bool live = (sl >> 31) == 0u;
          const int64_t slot = sl & 0x7fffffffu;
          float gq[kNdof];
          gq[0] = a.tgrad ? __uint_as_float(r[3]) : -__uint_as_float(r[0]);
          gq[1] = a.tgrad ? __uint_as_float(r[4]) : -__uint_as_float(r[1]);
#pragma unroll
          for (int i = 0; i < 7; ++i) gq[2 + i] = __uint_as_float(r[5 + i]);
          if constexpr (kSE2) {
            float sn, cs;
            sincosf(S.qn[s][it & 1][2], &sn, &cs);
            const float gx = __uint_as_float(r[0]), gy = __uint_as_float(r[1]);
            gq[0] = -(cs * gx - sn * gy);
            gq[1] = -(sn * gx + cs * gy);
            gq[2] = gx * pp_t.y - gy * pp_t.x;
          }
          if (a.detect) {
            wait_bar(&S.det_out[s], (uint32_t)it & 1u);
            const bool act = live && (f - a.delta <= a.tau);
            int rk = __popc(S.act[s][qd] & ((1u << lane) - 1u));
            for (int i = 0; i < qd; ++i) rk += __popc(S.act[s][i]);
            const int base = S.sbase[s];
            if (act && base >= 0) {
              float4 *dst = reinterpret_cast<float4 *>(a.ds.staging + base + rk);
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
      seq += kSlots;
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

template <bool F16, bool kSE2>
cudaError_t launch_t(const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  const int smem = (int)sizeof(Smem3) + 1024;
  cudaError_t e = cudaFuncSetAttribute(k_mlp_tc3<F16, kSE2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t n_tiles = a.part.tile_wp ? kSlots * (int64_t)num_sms : (int64_t)a.n_wp * a.tiles_per_wp;
  int64_t grid = (n_tiles + kSlots - 1) / kSlots;
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
