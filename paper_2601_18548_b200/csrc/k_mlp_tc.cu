// k_mlp_tc.cu -- K2b: fused pair generation + base-frame transform + 7-layer MLP forward
// + input-gradient backward (+ threshold / min / per-tile compaction in detect mode) on
// the 5th-generation tensor cores (tcgen05, fp16 or bf16 operands, fp32 accumulation in TMEM).
//
// Paper steps (PAPER.md lines): base-frame bias :388/:171; "7-layer MLP" on [p, q] :284;
// value + gradient :394 (dense gradient R^{NM x n}); constraint f - delta >= 0 :362-363;
// union = min :164; c_gcdf step-major order :414-435.  DESIGN.md §5 "K2b".
//
// Design (H = 128, one persistent CTA per SM, 864 threads = 24 epilogue warps + 3 MMA warps):
//   * Every affine layer of a 128-pair tile is a UMMA with M = 128 pairs, A in TMEM and B
//     resident in shared memory for the whole kernel:
//       - layer 1 (12 -> 128): K = 32 of split hi/lo 16-bit operands (A = {x_hi, x_lo,
//         x_hi}, B = {w_hi, w_hi, w_lo} per input, plus {1, 1} x {b_hi, b_lo}), which
//         keeps the metre-scale point coordinates at ~fp32 accuracy (R16);
//       - layers 2..6 (128 -> 128): K = 128 from the activations + one K = 16 step
//         against a constant "ones" A block that adds the bias {b_hi, b_lo};
//       - backward layers 6..2: D = E W_l with the same smem bytes read MN-major;
//       - g0 = e1 W1: N = 16 rows of W1^T.
//     W_2..W_6 use the UMMA SWIZZLE_128B layout (5 x 32 KB); the small K = 16 / 32 blocks
//     the SWIZZLE_NONE layout (the five bias blocks share one all-zero second K core).
//   * Three tiles in flight (slots), 12 MMA phases per tile (layer 1, layers 2..6, backward
//     6..2, g0).  TMEM is four 128-column regions used round robin: the k-th MMA phase of the
//     CTA (phases interleave slot 0, 1, 2, 0, ...) writes its accumulator D into region k % 4
//     and reads its A operand from region (k + 1) % 4 = the region of the slot's previous
//     phase, where that phase's epilogue wrote the 16-bit activations IN PLACE over the
//     accumulator columns it had already loaded (A of K step k at AK(k)).  So a slot holds
//     one region between phases and a phase needs one fresh region: 3 slots x 128 + 128 =
//     512 columns, where a fixed D + A per slot (192 columns) fits only two slots.  Region
//     k % 4 was last read (as A) by phase k - 1, issued just before phase k by the turn order.
//   * Each slot has 8 epilogue warps: warp (h, q) owns TMEM lanes 32q..32q+31 (the tile's
//     pairs) and accumulator columns 32h + {0..31, 64..95}; one MMA warp per slot issues its
//     phases: it waits on the slot's "A ready" mbarrier (one arrival per epilogue warp) and
//     on its turn (an mbarrier per slot orders the CTA's phases round robin, which the region
//     rotation relies on), an elected lane issues the UMMAs (operands in uniform registers)
//     and commits them to the slot's "D ready" mbarrier.  With three tiles in flight the
//     per-slot chain MMA -> commit -> epilogue -> hand-off (~2k cycles) is
//     covered by the other two slots' tensor work (2 x 576 cycles per phase).
//   * Activations never leave the chip: accumulator D (fp32) -> epilogue registers (ReLU +
//     16-bit pack + byte-sign mask) -> A (TMEM, in place) -> next UMMA.  ReLU masks go to
//     shared memory for the backward pass.
#include <type_traits>

#include "gcdf_internal.h"
#include "tc_ptx.h"

namespace gcdf {
namespace {

using namespace tc;

// Waits of the epilogue / detect / MMA warps: plain try_wait polling.  (A suspend-time hint
// compiles to a NANOSLEEP between polls, which spares the issue slots an idle warp's polls take
// from the busy epilogue warps of its SM sub-partition, but its wake-up latency sits on the
// per-slot chain: measured 105.4M vs 99.8M SM cycles per C5 launch, tools/_runab.sh.)
DEVI void wait_bar(uint64_t *bar, uint32_t parity) { mbar_wait(bar, parity); }
DEVI void wait_bar_addr(uint32_t addr, uint32_t parity) {
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(addr, parity)) {
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}

constexpr int H = 128;
constexpr int kSlots = 3;                         // tiles in flight
constexpr int kEpiPerSlot = 256;                  // 8 epilogue warps per slot
constexpr int kEpiWarps = kSlots * kEpiPerSlot / 32;  // warps 0..23
constexpr int kMmaWarp0 = kEpiWarps;              // warp 24 + s issues slot s's UMMAs
constexpr int kDetectWarp = kEpiWarps + kSlots;   // warp 27: per-tile detect bookkeeping (A6-A8 atomics)
constexpr int kWarps = kDetectWarp + 1;
constexpr int kThreads = kWarps * 32;             // 896
constexpr int kEpiArrivals = kEpiPerSlot / 32;    // epi_done count: one arrival per epilogue warp
constexpr int kRegsIssue = 24, kRegsEpi = 80;     // registers per thread after the split (see k_mlp_tc)
static_assert(kEpiWarps * kRegsEpi + (kWarps - kEpiWarps) * kRegsIssue <= 65536 / 32, "register split");
constexpr int kPhases = 12;                       // MMA phases per tile
constexpr int kMasks = 5;                         // stored ReLU masks: layers 1..5
constexpr int kWBytes = 5 * H * H * 2;            // 163,840
constexpr int kW1tBytes = 16 * H * 2;             // 4,096
constexpr int kB1Bytes = 32 * H * 2;              // 8,192
constexpr int kBextBytes = 16 * H * 2;            // global bias block per hidden layer (2 K cores)
constexpr int kBiasCore = 8 * H * 2;              // 2,048: one K core (8 k) of a bias block
// Region layout (columns relative to the region): the A operand's K step k (16 units, 8
// columns of 16-bit pairs) at AK(k); the "ones" A block of the bias step at kColOnes (written
// by forward epilogues); in a g0 phase's region: g0 at [0, 16) and the next tile's layer-1
// operands x at [kColX, kColX + 16).  All of these are columns the writing warp has loaded.
constexpr uint32_t kColOnes = 48, kColX = 16;
__host__ __device__ constexpr uint32_t AK(int k) {
  return (uint32_t)((k >> 2) * 64 + ((k >> 1) & 1) * 32 + (k & 1) * 8);
}
// epilogue chunk c = 0..3 of column half h: accumulator columns 32h + DC(c) .. + 15 (units of
// the same numbers); their 16-bit activations go to 32h + AC(c) .. + 7 (= AK of their K step)
__host__ __device__ constexpr uint32_t DC(int c) { return (uint32_t)((c >> 1) * 64 + (c & 1) * 16); }
__host__ __device__ constexpr uint32_t AC(int c) { return (uint32_t)((c >> 1) * 64 + (c & 1) * 8); }
static_assert(AK(0) == AC(0) && AK(1) == AC(1) && AK(2) == 32 + AC(0) && AK(3) == 32 + AC(1) && AK(4) == AC(2) &&
                  AK(5) == AC(3) && AK(6) == 32 + AC(2) && AK(7) == 32 + AC(3),
              "K step k holds units 16k..16k+15");
template <bool F16> constexpr uint32_t kIdescFwd = idesc_f16kind(128, 128, false, F16);
template <bool F16> constexpr uint32_t kIdescBwd = idesc_f16kind(128, 128, true, F16);
template <bool F16> constexpr uint32_t kIdescFin = idesc_f16kind(128, 16, false, F16);

struct __align__(1024) SmemTC {
  uint8_t w[kWBytes];          // W_2..W_6, SW128 [2 chunks][128 rows][128 B] each
  uint8_t w1t[kW1tBytes];      // W1^T [16][128], SW128
  uint8_t b1[kB1Bytes];        // layer-1 split weights [128][32], no swizzle
  uint8_t bext[5][kBiasCore];  // hidden-layer bias blocks: K core 0 ({b_hi, b_lo, 0..})
  uint8_t bzero[kBiasCore];    // K core 1 of every bias block (zeros)
  float fpart[kSlots][2][H];   // [slot][column half][row] partial output-layer sums
  float4 ptn[kSlots][H];       // [slot][row] prefetched point of the slot's next tile
  float qn[kSlots][2][12];     // [slot][tile parity] q row of the slot's tile (cp.async, phases 1-3)
  int wnx[kSlots];             // [slot] (partitioned) step of the slot's next tile, staged at phase 1
  int rnx[kSlots];             // [slot] (dense map) tile index within its step of the slot's next tile
  int wtile[kSlots][2];        // [slot][tile parity] step (waypoint) of the slot's tile
  uint32_t slotn[kSlots][2][H];  // [slot][tile parity][row] local scene slot of the pair (~0: padding;
                                 // bit 31: a removed point, set when x is staged)
  uint32_t mask[kSlots][kMasks][2][kEpiPerSlot];  // ReLU masks [slot][layer][32-unit word][thread]
  uint64_t mma_done[kSlots];
  uint64_t epi_done[kSlots];
  uint64_t wbar;               // the resident weights landed (bulk copies, complete_tx)
  uint64_t turn[kSlots];       // [slot] "your turn": the previous slot's phase is issued (round robin)
  uint32_t one;                // 1 (runtime constant, see add7fff)
  uint64_t det_in[kSlots];     // [slot] the 4 column-half-1 warps posted the tile's ballots / min keys
  uint64_t det_out[kSlots];    // [slot] the detect warp posted the tile's staging base
  unsigned act[kSlots][4];
  unsigned long long kmin[kSlots][4];
  int sbase[kSlots];
  uint32_t tmem_base;
};

static_assert(2 * kSlots * kTraceTiles * kTracePhases * 4 + kEpiWarps * kTraceTiles * kPhases <= kTraceLen,
              "trace buffer layout");
// (the dynamic shared memory of a CTA starts 1024-B aligned, after the 1 KB the system
// reserves: checked at kernel entry, so no alignment pad is allocated)
static_assert(sizeof(SmemTC) <= 232448, "SmemTC exceeds the 227 KB of shared memory per CTA");

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

// A1 operand values of the split layer-1 GEMM for one input x: {x_hi, x_lo, x_hi}
template <bool F16>
DEVI void split3(float x, float *o) {
  const float hi = round16<F16>(x);
  o[0] = hi;
  o[1] = x - hi;  // exact in fp32; rounded to 16 bits by the pack
  o[2] = hi;
}

// The epilogue is ALU-pipe bound (F2FP, PRMT, LOP3, SHF); the "+ 0x7fff7fff" of the
// mask tests is written as pk * one + c with a runtime one (read from shared memory) so
// that it compiles to IMAD on the otherwise idle FMA pipe instead of VIADD on the ALU.
DEVI uint32_t add7fff(uint32_t pk, uint32_t one) { return pk * one + 0x7fff7fffu; }
// mask_group (tc_ptx.h) with the adds on the FMA pipe
DEVI uint32_t mask_group_f(uint32_t pk01, uint32_t pk23, int k, uint32_t one) {
  const uint32_t x = prmt(add7fff(pk01, one), add7fff(pk23, one), 0x7531u);
  return (x >> k) & (0x80808080u >> k);
}

// UMMAs of MMA phase p: accumulator in the region at TMEM address d, A operand in the region
// at av (the slot's previous phase's region).  Executed by the whole (converged) MMA warp;
// one elected lane issues all UMMAs of the phase from ONE asm block, the per-UMMA operands
// formed by adds of immediates to the phase's base values (the descriptor's start-address
// field is its low 14 bits, so desc(base + off) = desc(base) + off / 16 for off < 256 KB).
// The issue stream is the tensor pipe's feed: at ~16 instructions per UMMA (operands built
// per UMMA and moved to uniform registers one by one) the MMA warp, sharing its SM
// sub-partition with six busy epilogue warps, issued a 64-cycle UMMA every ~90 cycles.
#define GCDF_UMMA(AOFF, DOFF, ACC)                                         \
  "add.u32 ra, %1, " #AOFF ";\n\t"                                         \
  "add.u64 rb, %2, " #DOFF ";\n\t"                                         \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, " ACC ";\n\t"
#define GCDF_UMMA_HEAD                                                     \
  "{\n\t.reg .pred e, pf, pt;\n\t.reg .b32 ra;\n\t.reg .b64 rb;\n\t"       \
  "elect.sync _|e, 0xffffffff;\n\t"                                        \
  "setp.ne.b32 pf, %4, %4;\n\tsetp.eq.b32 pt, %4, %4;\n\t"
// forward layer (K-major SW128 B, 2 x 64-column chunks of 16 KB): K step k at A column AK(k),
// B at + (k / 4) * 16384 + (k % 4) * 32 bytes; then the bias step (ones at kColOnes)
DEVI void umma_fwd(uint32_t d, uint32_t av, uint64_t b0, uint32_t idesc, uint64_t bias) {
  asm volatile(GCDF_UMMA_HEAD
               GCDF_UMMA(0, 0, "pf") GCDF_UMMA(8, 2, "pt") GCDF_UMMA(32, 4, "pt") GCDF_UMMA(40, 6, "pt")
               GCDF_UMMA(64, 1024, "pt") GCDF_UMMA(72, 1026, "pt") GCDF_UMMA(96, 1028, "pt") GCDF_UMMA(104, 1030, "pt")
               "add.u32 ra, %1, 48;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], %5, %3, pt;\n\t"
               "}" ::"r"(d), "r"(av), "l"(b0), "r"(idesc), "r"(0u), "l"(bias)
               : "memory");
}
static_assert(kColOnes == 48, "umma_fwd's bias step reads the ones block at column 48");
// backward layer (MN-major SW128 B): K step k at B + k * 2048 bytes
DEVI void umma_bwd(uint32_t d, uint32_t av, uint64_t b0, uint32_t idesc) {
  asm volatile(GCDF_UMMA_HEAD
               GCDF_UMMA(0, 0, "pf") GCDF_UMMA(8, 128, "pt") GCDF_UMMA(32, 256, "pt") GCDF_UMMA(40, 384, "pt")
               GCDF_UMMA(64, 512, "pt") GCDF_UMMA(72, 640, "pt") GCDF_UMMA(96, 768, "pt") GCDF_UMMA(104, 896, "pt")
               "}" ::"r"(d), "r"(av), "l"(b0), "r"(idesc), "r"(0u)
               : "memory");
}
// g0 = e1 W1 (N = 16, W1^T K-major SW128 in 2 chunks of 2 KB)
DEVI void umma_g0(uint32_t d, uint32_t av, uint64_t b0, uint32_t idesc) {
  asm volatile(GCDF_UMMA_HEAD
               GCDF_UMMA(0, 0, "pf") GCDF_UMMA(8, 2, "pt") GCDF_UMMA(32, 4, "pt") GCDF_UMMA(40, 6, "pt")
               GCDF_UMMA(64, 128, "pt") GCDF_UMMA(72, 130, "pt") GCDF_UMMA(96, 132, "pt") GCDF_UMMA(104, 134, "pt")
               "}" ::"r"(d), "r"(av), "l"(b0), "r"(idesc), "r"(0u)
               : "memory");
}
// layer 1: K = 32 split operands at A columns kColX, kColX + 8; B (no swizzle) at + k * 4096 bytes
DEVI void umma_l1(uint32_t d, uint32_t av, uint64_t b0, uint32_t idesc) {
  asm volatile(GCDF_UMMA_HEAD
               GCDF_UMMA(16, 0, "pf") GCDF_UMMA(24, 256, "pt")
               "}" ::"r"(d), "r"(av), "l"(b0), "r"(idesc), "r"(0u)
               : "memory");
}
static_assert(kColX == 16, "umma_l1 reads x at columns 16..31");
#undef GCDF_UMMA
#undef GCDF_UMMA_HEAD
static_assert(AK(1) == 8 && AK(2) == 32 && AK(3) == 40 && AK(4) == 64 && AK(5) == 72 && AK(6) == 96 && AK(7) == 104,
              "A column offsets in the umma_* blocks");

// Phase p's UMMAs once the wait returns: the operands (descriptor bases) are formed before
// the wait, so the phase's first UMMA follows the turn by a few instructions.
template <bool F16, typename Wait>
DEVI void issue_phase(int p, uint32_t d, uint32_t av, uint32_t sw, uint32_t sw1t, uint32_t sb1, uint32_t sbx,
                      uint32_t sbz, Wait &&wait) {
  if (p == 0) {
    const uint64_t b0 = sdesc_nosw(sb1, 2048, 128);
    wait();
    umma_l1(d, av, b0, kIdescFwd<F16>);
  } else if (p < 6) {  // layer l = p + 1: D = A W_l^T (B = W_l K-major) + ones x bias
    const uint32_t bb = sbx + (uint32_t)(p - 1) * kBiasCore;
    const uint64_t b0 = sdesc_sw128(sw + (uint32_t)(p - 1) * (H * H * 2), 16, 1024), bx = sdesc_nosw(bb, sbz - bb, 128);
    wait();
    umma_fwd(d, av, b0, kIdescFwd<F16>, bx);
  } else if (p < 11) {  // backward through layer l = 12 - p: D = E W_l, B = W_l MN-major
    const uint64_t b0 = sdesc_sw128(sw + (uint32_t)(10 - p) * (H * H * 2), 16384, 1024);
    wait();
    umma_bwd(d, av, b0, kIdescBwd<F16>);
  } else {  // g0 = e1 W1 (N = 16 rows of W1^T) -> columns 0..15 of the region
    const uint64_t b0 = sdesc_sw128(sw1t, 16, 1024);
    wait();
    umma_g0(d, av, b0, kIdescFin<F16>);
  }
}

// The MMA warp of slot SS.  A commit stalls its issuing thread until the committed MMAs
// drain; with one issuer per slot the other slots' UMMAs keep the tensor pipe busy meanwhile
// (tools/mma_probe.py "two issuers").  Phase k of the CTA (k = 3 j + SS for the slot's j-th
// phase) is issued after phase k - 1 (S.turn[SS], arrived on by the previous slot's MMA warp);
// a slot without a tile in the last round passes its turns.
// TMEM base address 0 (the kernel's single 512-column allocation, checked at setup).
template <bool F16, int SS, bool kTrace>
DEVI void mma_loop(SmemTC &S, const QueryArgs &a, int64_t n_tiles, int64_t stride, int lane) {
  const uint32_t sw = smem_u32(S.w), sw1t = smem_u32(S.w1t), sb1 = smem_u32(S.b1);
  const uint32_t sbx = smem_u32(S.bext), sbz = smem_u32(S.bzero);
  uint32_t ph = 0u, seq = (uint32_t)SS;
  long long *tr = (kTrace && a.trace && blockIdx.x == 0 && lane == 0)
                      ? a.trace + (size_t)SS * kTraceTiles * kTracePhases * 4
                      : nullptr;
  mbar_wait(&S.wbar, 0u);  // the resident weights have landed in shared memory
  int it = 0;
  for (int64_t base = (int64_t)blockIdx.x * kSlots; base < n_tiles; base += stride, ++it) {
    const bool real = base + SS < n_tiles;
    // the slot's last tile hands off once more after its g0 readout: the phase after it (a
    // passed turn) must not let the next phases overwrite the region g0 is read from
    const bool last_was_real = it > 0 && base - stride + SS < n_tiles;
#pragma unroll 1
    for (int p = 0; p < kPhases; ++p, seq += kSlots) {
      long long *t = (tr && it < kTraceTiles) ? tr + ((size_t)it * kTracePhases + p) * 4 : nullptr;
      if (real || (p == 0 && last_was_real)) {
        wait_bar(&S.epi_done[SS], ph);
        ph ^= 1u;
      }
      if (t) t[0] = clock64();
      // the turn (an mbarrier, so a waiting MMA warp sleeps instead of taking issue slots
      // from the epilogue warps of its SM sub-partition)
      auto wait_turn = [&]() {
        wait_bar(&S.turn[SS], (seq / kSlots) & 1u);
        if (t) t[1] = clock64();
        fence_after();
      };
      if (real) issue_phase<F16>(p, 128u * (seq & 3u), 128u * ((seq + 1u) & 3u), sw, sw1t, sb1, sbx, sbz, wait_turn);
      else wait_turn();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.turn[(SS + 1) % kSlots]);  // the next slot may issue now
      if (real) commit_elect(&S.mma_done[SS]);
      if (t) t[2] = clock64();
    }
  }
}

// The detect warp (A6-A8 bookkeeping, detect mode): per tile, in the CTA's slot order, it
// combines the four column-half-1 warps' ballots and min keys (posted after their phase-6
// hand-off), publishes the per-waypoint min key (atomicMin) and allocates the tile's staging
// records (atomicAdd), then posts the tile's staging base for the phase-11 record writes.
// Its global atomics' latency is on no epilogue warp's path.
DEVI void detect_loop(SmemTC &S, const QueryArgs &a, int64_t n_tiles, int64_t stride, int lane) {
  uint32_t ph = 0u;  // bit s: parity of slot s's det_in
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

// kSE2: the SE(2) frame variant (R24) as its own instantiation, so the default
// translation-frame kernel carries none of its code or registers
// kTrace: the diagnostics instantiation (gcdf_debug_trace), the only one with clock64 stamps
template <bool F16, bool kSE2, bool kTrace>
__global__ void __launch_bounds__(kThreads, 1) k_mlp_tc(const WeightsBF16 W, const QueryArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned view (SWIZZLE_128B atoms); pointer arithmetic on the __shared__ array
  // keeps the shared address space visible to the compiler (LDS/STS, not generic LD/ST)
  SmemTC &S = *reinterpret_cast<SmemTC *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (smem_u32(smem_raw) & 1023u) __trap();  // SWIZZLE_128B operands need 1024-B alignment

  // ---- one-time setup: the resident weights (already in their UMMA layouts in global
  // memory) -> smem by 1-D bulk copies (cp.async.bulk, the TMA engine) completing on S.wbar;
  // only the MMA warps wait for them (before their first UMMA), so the copy overlaps the
  // epilogue warps' staging of the first tiles ----
  if (tid == 0) {
    S.one = 1u;
    mbar_init(&S.wbar, 1);
    fence_barrier_init();
    constexpr uint32_t kChunk = 32768;
    mbar_expect_tx(&S.wbar, (uint32_t)(kWBytes + kW1tBytes + kB1Bytes + 5 * kBiasCore));
    for (uint32_t o = 0; o < (uint32_t)kWBytes; o += kChunk)
      bulk_g2s(S.w + o, static_cast<const uint8_t *>(W.w_sw128) + o, kChunk, &S.wbar);
    bulk_g2s(S.w1t, W.w1t_sw128, kW1tBytes, &S.wbar);
    bulk_g2s(S.b1, W.b1_nosw, kB1Bytes, &S.wbar);
    for (int l = 0; l < 5; ++l)  // K core 0 of each bias block (its K core 1 is all zeros)
      bulk_g2s(S.bext[l], static_cast<const uint8_t *>(W.bext_nosw) + l * kBextBytes, kBiasCore, &S.wbar);
  }
  for (int i = tid; i < kBiasCore / 16; i += kThreads) reinterpret_cast<uint4 *>(S.bzero)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) {
    tmem_alloc(&S.tmem_base, 512);
    tmem_relinquish();
  }
  if (tid == 32) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&S.mma_done[i], 1);
      mbar_init(&S.epi_done[i], kEpiArrivals);
    }
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&S.turn[i], 1);
      mbar_init(&S.det_in[i], 4);
      mbar_init(&S.det_out[i], 1);
    }
    mbar_arrive(&S.turn[0]);  // slot 0 issues the CTA's first phase
    fence_barrier_init();
  }
  if (tid < kSlots * kNdof) {  // q rows of the slots' first tiles (later tiles: cp.async, phases 1-3)
    const int s0 = tid / kNdof, i = tid - s0 * kNdof;
    const int64_t T0 = (int64_t)blockIdx.x * kSlots + s0;
    if (T0 < query_tiles(a)) {
      const int w0 = tile_step(a, T0);
      S.qn[s0][0][i] = __ldg(a.q + (int64_t)w0 * kNdof + i);
      if (i == 0) S.wtile[s0][0] = w0;
    }
  }
  fence_proxy_async_smem();  // generic-proxy smem writes (zero K core) -> visible to the tensor core
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = S.tmem_base;
  if (tbase != 0u) __trap();  // the MMA warps address TMEM from column 0 (see mma_loop)
  const int64_t n_tiles = query_tiles(a);  // (partitioned: read from the device)
  const int64_t lb = a.scene.local_bound;
  const int64_t stride = kSlots * (int64_t)gridDim.x;

  // Register split (setmaxnreg, per aligned 4-warp group): the MMA / detect group (warps
  // 24..27) drops to kRegsIssue, the six epilogue groups rise to kRegsEpi (72 at launch:
  // 896 threads share the 64K registers).
  if (warp >= kEpiWarps) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsIssue));
    // ============ three MMA warps: warp 24 + s issues slot s's phases, in CTA order ============
    // (the slot is a template argument, so that the issue loop's operands are warp-uniform to
    // the compiler and live in uniform registers)
    if (warp == kMmaWarp0) mma_loop<F16, 0, kTrace>(S, a, n_tiles, stride, lane);
    else if (warp == kMmaWarp0 + 1) mma_loop<F16, 1, kTrace>(S, a, n_tiles, stride, lane);
    else if (warp == kMmaWarp0 + 2) mma_loop<F16, 2, kTrace>(S, a, n_tiles, stride, lane);
    else if (a.detect) detect_loop(S, a, n_tiles, stride, lane);
    __syncwarp();
    fence_before();
    __syncthreads();
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsEpi));
  // (the warp index through a lane-0 shuffle: warp-uniform to the compiler, so the TMEM
  // addresses derived from it live in uniform registers -- no R2UR before each TMEM load / store)
  const int ew = __shfl_sync(0xffffffffu, warp, 0);
  const int s = ew >> 3;            // tile slot
  const int hh = (ew >> 2) & 1;     // column half: accumulator columns 32 hh + {0..31, 64..95}
  const int qd = ew & 3;            // TMEM lane quarter of this warp (warp % 4)
  const int row = qd * 32 + lane;   // pair within the tile = TMEM lane
  const uint32_t tL = tbase + ((uint32_t)(qd * 32) << 16) + 32u * hh;  // region 0, this lane quarter, column half
  uint32_t seq = (uint32_t)s;       // CTA phase index of the slot's next MMA phase
  auto region = [&](uint32_t k) { return tL + 128u * (k & 3u); };
  uint32_t *mk = &S.mask[s][0][0][hh * 128 + row];  // + (layer * 2 + word) * kEpiPerSlot
  const uint32_t bar_mma = smem_u32(&S.mma_done[s]), bar_epi = smem_u32(&S.epi_done[s]);
  int it = 0;
  // (diagnostics, kTrace only) per-warp hand-off stamps [warp][tile][phase] after the role
  // blocks, and epilogue warp 0's stamps per phase
  long long *twarp = nullptr, *trb = nullptr, *trc = nullptr;
  if constexpr (kTrace) {
    if (a.trace && blockIdx.x == 0 && lane == 0) {
      twarp = a.trace + (size_t)(2 * kSlots) * kTraceTiles * kTracePhases * 4 + (size_t)warp * kTraceTiles * kPhases;
      if (hh == 0 && qd == 0) trb = a.trace + (size_t)(kSlots + s) * kTraceTiles * kTracePhases * 4;
    }
  }
  // epilogue phase done: this warp's TMEM stores complete and ordered before the MMA warp's
  // UMMAs (every lane waits for its stores and fences, then one lane arrives)
  auto hand_off = [&](int p) {
    if constexpr (kTrace) if (trc) trc[2] = clock64();
    wait_st();
    fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_addr(bar_epi);
    if constexpr (kTrace) {
      if (twarp && p >= 0 && it < kTraceTiles) twarp[it * kPhases + p] = clock64();
      if (trc) trc[3] = clock64();
    }
  };
  // cp.async prefetch of this lane's point of tile TT into S.ptn[s][row] (zero if none);
  // issued by the column-half-0 threads, which alone read it
  // (the pair's local slot goes to S.slotn[s][par][row], read back at phases 5, 6 and 11 and
  // by stage_a1: no per-tile index arithmetic on the critical path)
  auto prefetch_pt = [&](int64_t TT, int par) {
    int wn = 0;
    int64_t sl = 0;
    bool ok = false;
    if (TT < n_tiles) {
      if (a.part.tile_wp) {
        tile_pair(a, TT, row, wn, sl, ok);
      } else {  // (step, tile of the step) divided out once, at phase 3, by stage_q
        sl = (int64_t)S.rnx[s] * kTile + row;
        ok = sl < lb;
      }
    }
    S.slotn[s][par][row] = ok ? (uint32_t)sl : ~0u;
    cp_async16(&S.ptn[s][row], ok ? (const void *)(a.scene.pts + sl) : (const void *)a.scene.pts, ok ? 16u : 0u);
    cp_async_commit();
  };
  // q row of the slot's next tile TT -> S.qn[s][par], by lanes 0..8 of warp (half 0,
  // quarter 0) off the critical path: phase 1 stages the step of a partitioned tile, phase
  // 3 copies the row; the copy is waited for before the phase-5 barrier of the slot's 256
  // epilogue threads, which publishes it (stage_a1 reads it at phase 11)
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
  // A2 + A1 of tile TT: pair generation, base-frame bias p' = p - [q_x, q_y, 0]
  // and the split layer-1 operands -> TMEM columns kColX.. of the region at tx
  // (K = 32: half 0 writes K 0..15, half 1 K 16..31).  Returns the pair's liveness
  // (meaningful in half 0).  SE(2) frame (R24): p'_xy = R(-theta)(p_xy - b), theta channel
  // fed 0; p'_xy is kept in pp (half 0's registers) for the theta gradient at phase 11
  // (__sincosf: abs error ~1e-6 on [-pi, pi], far below the 16-bit operand rounding).
  float2 pp = make_float2(0.f, 0.f);
  auto stage_a1 = [&](int par, uint32_t tx) -> bool {
    const float *qw = S.qn[s][par];
    float v[16];
    bool lv = false;
    if (hh == 0) {  // K 0..15: p'_x, p'_y, p_z, theta, j1 (3 each), x_hi of j2
      const float4 pt = S.ptn[s][row];
      const uint32_t sl = S.slotn[s][par][row];
      lv = sl != ~0u && pt.w > 0.f;
      if (sl != ~0u && !lv) S.slotn[s][par][row] = sl | 0x80000000u;
      float dx = pt.x - qw[0], dy = pt.y - qw[1], th = qw[2];
      if constexpr (kSE2) {
        float sn, cs;
        __sincosf(th, &sn, &cs);
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
    } else {        // K 16..31: x_lo, x_hi of j2, j3..j6 (3 each), {1, 1} for b1
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
  if ((int64_t)blockIdx.x * kSlots + s < n_tiles) {
    if (hh == 0) {
      int wn;
      int64_t sl;
      bool ok;
      tile_pair(a, (int64_t)blockIdx.x * kSlots + s, row, wn, sl, ok);  // (the first tile: divided here)
      S.slotn[s][0][row] = ok ? (uint32_t)sl : ~0u;
      cp_async16(&S.ptn[s][row], ok ? (const void *)(a.scene.pts + sl) : (const void *)a.scene.pts, ok ? 16u : 0u);
      cp_async_commit();
      cp_async_wait_all();
    }
    stage_a1(0, region(seq + 1u));  // phase 0's A region
    hand_off(-1);
  }
  for (int64_t T = (int64_t)blockIdx.x * kSlots + s; T < n_tiles; T += stride, ++it) {
    float f = 0.f;
    // one MMA phase of the tile (compile-time phase number: every phase is its own straight
    // code, no run-time dispatch)
    auto phase = [&](auto pc) {
      constexpr int p = decltype(pc)::value;
      if constexpr (kTrace) trc = (trb && it < kTraceTiles) ? trb + ((size_t)it * kTracePhases + p) * 4 : nullptr;
      wait_bar_addr(bar_mma, ph);
      if constexpr (kTrace) if (trc) trc[0] = clock64();
      ph ^= 1u;
      fence_after();
      const uint32_t tD = region(seq);  // this lane quarter's and column half's accumulator
      if constexpr (p < 5) {
        // ---- forward epilogue of layer l = p + 1: z = D (bias folded in); h = ReLU(z) -> A
        // (in place), 1-bit masks -> smem; half 1 also writes the "ones" block of the next
        // phase's bias step.  (16-column chunks, the TMEM load of chunk c + 1 in flight while
        // chunk c is packed) ----
        uint32_t rb[2][16], m = 0u;
        ld16(tD + DC(0), rb[0]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < 3) ld16(tD + DC(c + 1), rb[(c + 1) & 1]);
          const uint32_t *rr = rb[c & 1];
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            pk[j >> 1] = pack2_relu<F16>(__uint_as_float(rr[j]), __uint_as_float(rr[j + 1]));
            pk[(j >> 1) + 1] = pack2_relu<F16>(__uint_as_float(rr[j + 2]), __uint_as_float(rr[j + 3]));
            m |= mask_group_f(pk[j >> 1], pk[(j >> 1) + 1], ((c & 1) * 16 + j) >> 2, one);
          }
          st8(tD + AC(c), pk);
          if (c & 1) {
            mk[(p * 2 + (c >> 1)) * kEpiPerSlot] = m;
            m = 0u;
          }
          if (c < 3) wait_ld();
        }
        if (hh == 1) {  // the constant "ones" A block of the bias step: {1, 1, 0, ...} (columns
                        // 48..55, loaded by this half's chunk 1)
          const uint32_t ones[8] = {pack2<F16>(1.f, 1.f), 0u, 0u, 0u, 0u, 0u, 0u, 0u};
          st8(tD - 32u + kColOnes, ones);
        }
        hand_off(p);
        if constexpr (p == 1 || p == 3) stage_q(p, T + stride, (it + 1) & 1);
      } else if constexpr (p == 5) {
        // ---- layer 6: e6 = w7 (.) 1[z6 > 0] -> A; f = w7 . ReLU(z6) + b7 (fp32) ----
        float fa[4] = {0.f, 0.f, 0.f, 0.f};
        // the output row comes from the kernel parameters with compile-time offsets (one body
        // per column half), i.e. as direct constant-bank operands: no shared-memory loads
        auto layer6 = [&](auto u0c) {
          constexpr int U0 = decltype(u0c)::value;
          uint32_t rb[2][16];
          ld16(tD + DC(0), rb[0]);
          wait_ld();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int cb = (int)DC(c);
            if (c < 3) ld16(tD + DC(c + 1), rb[(c + 1) & 1]);
            const uint32_t *rr = rb[c & 1];
            uint32_t pk[8];
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              const int u = U0 + cb + j;
              const float z0 = __uint_as_float(rr[j]), z1 = __uint_as_float(rr[j + 1]);
              const float z2 = __uint_as_float(rr[j + 2]), z3 = __uint_as_float(rr[j + 3]);
              // e6 = w7 (.) 1[z6 >= 0]: halfword masks from the sign bytes of the fp32 z (one PRMT
              // with sign replication per pair, then w7 & ~sign): the oracle's 1[z > 0] up to
              // z6 = +0 exactly (a kink, R17)
              pk[j >> 1] = W.w7h_p[u / 2] & ~prmt(rr[j], rr[j + 1], 0xffbbu);
              pk[(j >> 1) + 1] = W.w7h_p[u / 2 + 1] & ~prmt(rr[j + 2], rr[j + 3], 0xffbbu);
              // (w7 / 2) (z + |z|) = w7 ReLU(z) exactly (z + |z| = 2 ReLU(z), halving is exact)
              fa[0] = fmaf(W.w7half_p[u], z0 + fabsf(z0), fa[0]);
              fa[1] = fmaf(W.w7half_p[u + 1], z1 + fabsf(z1), fa[1]);
              fa[2] = fmaf(W.w7half_p[u + 2], z2 + fabsf(z2), fa[2]);
              fa[3] = fmaf(W.w7half_p[u + 3], z3 + fabsf(z3), fa[3]);
            }
            st8(tD + AC(c), pk);
            if (c < 3) wait_ld();
          }
        };
        if (hh == 0) layer6(std::integral_constant<int, 0>{});
        else layer6(std::integral_constant<int, 32>{});
        hand_off(p);
        // f = w7 . h6 + b7 (fp32, no output activation: signed value); both
        // column halves form it from the two partial sums (half 0 writes the records, half 1
        // thresholds)
        // (no barrier: the other half reads this partial sum two hand-offs later, at phase 7 /
        // 11, ordered by the mbarrier chain: this warp's arrive -> MMA warp -> commit -> wait)
        S.fpart[s][hh][row] = (fa[0] + fa[1]) + (fa[2] + fa[3]);
        if (hh == 0) {
          if (qd == 0) cp_async_wait_all();  // S.qn of the next tile (stage_q), read at phase 11
          prefetch_pt(T + stride, (it + 1) & 1);  // the next tile's point, needed at phase 11
        }
      } else if constexpr (p < 11) {
        // ---- backward: g_{l-1} = D; e_{l-1} = g (.) 1[z_{l-1} > 0] -> A (in place) ----
        constexpr int mi = 10 - p;
        const uint32_t mw[2] = {mk[(mi * 2) * kEpiPerSlot], mk[(mi * 2 + 1) * kEpiPerSlot]};
        uint32_t rb[2][16];
        ld16(tD + DC(0), rb[0]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < 3) ld16(tD + DC(c + 1), rb[(c + 1) & 1]);
          const uint32_t *rr = rb[c & 1];
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            uint32_t lo, hi;
            mask_expand(mw[c >> 1], ((c & 1) * 16 + j) >> 2, lo, hi);
            pk[j >> 1] = pack2<F16>(__uint_as_float(rr[j]), __uint_as_float(rr[j + 1])) & lo;
            pk[(j >> 1) + 1] = pack2<F16>(__uint_as_float(rr[j + 2]), __uint_as_float(rr[j + 3])) & hi;
          }
          st8(tD + AC(c), pk);
          if (c < 3) wait_ld();
        }
        hand_off(p);
        if constexpr (p == 7) {
          if (hh == 1) {
            f = S.fpart[s][0][row] + S.fpart[s][1][row] + W.b7;
            const uint32_t sl = S.slotn[s][it & 1][row];
            const bool live = (sl >> 31) == 0u;  // (padding rows: ~0; removed points: bit 31)
            const int64_t slot = sl & 0x7fffffffu;
            if (!a.detect) {
              const int w = S.wtile[s][it & 1];
              if (slot < lb) a.values[(int64_t)w * lb + slot] = live ? f : __int_as_float(0x7f800000);
            } else {
              // A6/A7 (overlaps the tensor core): threshold and the warp's min key -> the detect warp
              const bool act = live && (f - a.delta <= a.tau);
              const unsigned bal = __ballot_sync(0xffffffffu, act);
              // the warp's min key (ord f << 32 | id) by two 32-bit warp reductions (REDUX): the
              // min of ord f, then the smallest id among the lanes that hold it
              const unsigned khi = live ? ord_f32(f) : 0xffffffffu;
              const unsigned mhi = __reduce_min_sync(0xffffffffu, khi);
              const unsigned klo = (live && khi == mhi) ? (unsigned)local_to_global(slot, a.scene.rank, a.scene.world)
                                                        : 0xffffffffu;
              const unsigned mlo = __reduce_min_sync(0xffffffffu, klo);
              const unsigned long long key = ((unsigned long long)mhi << 32) | mlo;
              if (lane == 0) {
                S.act[s][qd] = bal;
                S.kmin[s][qd] = key;
                mbar_arrive(&S.det_in[s]);
              }
            }
          }
        }
      } else {
        // ---- phase 11: g0 = W1^T e1 (columns 0..15) -> d f / d q by the chain rule (R3) and
        // the outputs.  Half 0 loads g0 and both halves stage the next tile's layer-1 operands
        // (columns kColX.. of this region, the A operand of the next phase) before the
        // hand-off; the outputs are written after it.  (The hand-off also follows the slot's
        // last tile: it keeps the region, g0 included, from being reused before the load.) ----
        uint32_t r[16];
        if (hh == 0) {
          ld16(tD, r);
          wait_ld();
        }
        const float2 pp_t = pp;  // (SE(2)) p'_xy of this tile; stage_a1 overwrites pp
        if (T + stride < n_tiles) {
          if (hh == 0) cp_async_wait_all();  // this thread's point of the next tile (phase 5)
          stage_a1((it + 1) & 1, tD);
        }
        hand_off(p);
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
          if constexpr (kSE2) {  // SE(2) (R24): df/db = -R(theta) g0_xy, df/dtheta = g0_x p'_y - g0_y p'_x
            float sn, cs;
            __sincosf(S.qn[s][it & 1][2], &sn, &cs);
            const float gx = __uint_as_float(r[0]), gy = __uint_as_float(r[1]);
            gq[0] = -(cs * gx - sn * gy);
            gq[1] = -(sn * gx + cs * gy);
            gq[2] = gx * pp_t.y - gy * pp_t.x;
          }
          if (a.detect) {
            // rank of the pair among the tile's actives (the ballots of the four lane
            // quarters) + the tile's staging base, posted by the detect warp
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
      if constexpr (kTrace) if (trc) trc[1] = clock64();
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

template <bool F16>
cudaError_t launch_tc_t(const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  const int smem = (int)sizeof(SmemTC);
  auto kern = a.trace ? (a.frame ? k_mlp_tc<F16, true, true> : k_mlp_tc<F16, false, true>)
                      : (a.frame ? k_mlp_tc<F16, true, false> : k_mlp_tc<F16, false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  // a partitioned detect knows its tile count on the device only: one CTA per SM
  const int64_t n_tiles = a.part.tile_wp ? kSlots * (int64_t)num_sms : (int64_t)a.n_wp * a.tiles_per_wp;
  int64_t grid = (n_tiles + kSlots - 1) / kSlots;
  if (grid > num_sms) grid = num_sms;
  if (grid < 1) return cudaSuccess;
  kern<<<(unsigned)grid, kThreads, smem, s>>>(w, a);
  return cudaGetLastError();
}

}  // namespace

bool tc_compiled() { return true; }

cudaError_t launch_mlp_tc(int Hh, bool f16, const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  if (Hh != H) return cudaErrorInvalidValue;
  return f16 ? launch_tc_t<true>(w, a, num_sms, s) : launch_tc_t<false>(w, a, num_sms, s);
}

}  // namespace gcdf
