// k_mlp_tc.cu -- K2b: fused pair generation + base-frame transform + 7-layer MLP forward
// + input-gradient backward (+ threshold / min / per-tile compaction in detect mode) on
// the 5th-generation tensor cores (tcgen05, fp16 or bf16 operands, fp32 accumulation in TMEM).
//
// Paper steps (PAPER.md lines): base-frame bias :388/:171; "7-layer MLP" on [p, q] :284;
// value + gradient :394 (dense gradient R^{NM x n}); constraint f - delta >= 0 :362-363;
// union = min :164; c_gcdf step-major order :414-435.  DESIGN.md §5 "K2b".
//
// Design (H = 128, one persistent CTA per SM, 576 threads = 16 epilogue warps + 2 MMA warps):
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
//     the SWIZZLE_NONE layout.
//   * Activations never leave the chip: accumulator D (fp32, 128 TMEM columns) ->
//     epilogue registers (ReLU + 16-bit pack + byte-sign mask) -> A (64 TMEM columns) ->
//     next UMMA.  ReLU masks go to shared memory for the backward pass.
//   * Two tiles in flight: TMEM columns [0,256) belong to slot 0 and [256,512) to slot
//     1 (D [0,128), A [128,192), ones [192,200)).  Each slot has 8 epilogue warps: warp
//     (h, q) owns TMEM lanes 32q..32q+31 (the tile's pairs) and accumulator columns
//     64h..64h+63, so every SM sub-partition runs two warps per slot, and one slot's
//     epilogue overlaps the other slot's tensor-core work.  Warp 16 + s issues slot s's
//     MMAs: after each epilogue phase the slot's 8 warps arrive on the slot's "A ready"
//     mbarrier; the converged MMA warp waits on it (and on its turn: the slots alternate
//     phase by phase) and an elected lane issues the slot's next UMMAs (operands in
//     uniform registers) and commits them to the slot's "D ready" mbarrier.  One issuer
//     per slot keeps the other slot's UMMAs flowing while a commit drains.  12 MMA
//     phases per tile; the next tile's layer-1 operands are staged at the end of the
//     current tile (its point prefetched by cp.async four phases earlier).
//   * Measured (profiles/r1/mma_probe.txt, trace_tc_*.txt): a 128x128x16 UMMA runs at the
//     dense rate (64 cycles) when the issue stream is lean; the kernel is bound by the
//     per-slot chain MMA -> epilogue -> hand-off with two slots.
#include <type_traits>

#include "gcdf_internal.h"
#include "tc_ptx.h"

namespace gcdf {
namespace {

using namespace tc;

constexpr int H = 128;
constexpr int kEpiWarps = 16;             // warps 0..15: epilogue (8 per tile slot)
constexpr int kWarps = kEpiWarps + 2;      // + warp 16 + s: issues tile slot s's UMMAs
constexpr int kThreads = kWarps * 32;
constexpr int kEpiPerSlot = 256;
constexpr int kEpiArrivals = kEpiPerSlot;  // epi_done count: every epilogue thread of the slot
constexpr int kPhases = 12;               // MMA phases per tile
constexpr int kMasks = 5;                 // stored ReLU masks: layers 1..5
constexpr int kWBytes = 5 * H * H * 2;    // 163,840
constexpr int kW1tBytes = 16 * H * 2;     // 4,096
constexpr int kB1Bytes = 32 * H * 2;      // 8,192
constexpr int kBextBytes = 16 * H * 2;    // 4,096 per hidden layer
// per slot: D [0,128), A [128,192), ones [192,200), g0 [200,216), layer-1 operands x [216,232)
// (g0 and x have columns of their own so that the last GEMM of a tile and the first of the
// next one are issued as one phase, see issue_phase)
constexpr uint32_t kColA = 128, kColOnes = 192, kColG0 = 200, kColX = 216;
template <bool F16> constexpr uint32_t kIdescFwd = idesc_f16kind(128, 128, false, F16);
template <bool F16> constexpr uint32_t kIdescBwd = idesc_f16kind(128, 128, true, F16);
template <bool F16> constexpr uint32_t kIdescFin = idesc_f16kind(128, 16, false, F16);

struct __align__(1024) SmemTC {
  uint8_t w[kWBytes];          // W_2..W_6, SW128 [2 chunks][128 rows][128 B] each
  uint8_t w1t[kW1tBytes];      // W1^T [16][128], SW128
  uint8_t b1[kB1Bytes];        // layer-1 split weights [128][32], no swizzle
  uint8_t bext[5][kBextBytes]; // hidden-layer bias blocks [128][16], no swizzle
  uint32_t one;                // 1 (runtime constant, see add7fff)
  float fpart[2][2][H];        // [slot][column half][row] partial output-layer sums
  float4 ptn[2][H];            // [slot][row] prefetched point of the slot's next tile
  float2 pprime[2][2][H];      // [slot][tile parity][row] SE(2) frame: p'_xy kept for d f / d theta (R24)
  float qn[2][2][12];          // [slot][tile parity] q row of the slot's tile (cp.async, phases 1-3)
  int wnx[2];                  // [slot] (partitioned) step of the slot's next tile, staged at phase 1
  int wtile[2][2];             // [slot][tile parity] step (waypoint) of the slot's tile
  uint32_t slotn[2][2][H];     // [slot][tile parity][row] local scene slot of the pair (~0: padding)
  uint32_t mask[2][kMasks][2][kEpiPerSlot];  // ReLU masks [slot][layer][32-unit word][thread]
  uint64_t mma_done[2];
  uint64_t epi_done[2];
  uint64_t wbar;               // the resident weights landed (bulk copies, complete_tx)
  uint32_t turn;               // global issue-order counter of the two MMA warps
  unsigned act[2][4];
  unsigned long long kmin[2][4];
  int sbase[2];
  uint32_t tmem_base;
};

static_assert(sizeof(SmemTC) + 1024 <= 232448, "SmemTC exceeds the 227 KB of shared memory per CTA");

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
// 0xffff half-word masks of the nonzero halves of a packed pair of non-negative 16-bit
// values (bit 15 of v + 0x7fff is set iff v != 0; sign-replicate bytes 1 and 3)
DEVI uint32_t nz_halves(uint32_t pk, uint32_t one) { return prmt(add7fff(pk, one), 0u, 0xbb99u); }

// UMMAs of MMA phase p of the tile whose accumulator starts at TMEM column d, committed
// to bar.  Executed by the whole (converged) MMA warp with warp-uniform operands; one
// elected lane issues.  Uniform operands stay in uniform registers, which keeps the issue
// stream to a few instructions per UMMA: a lane-0-only loop paid a register-to-uniform
// move per operand and issued at ~75-90 cycles per UMMA, slower than the tensor pipe
// (64 cycles per 128x128x16 UMMA, tools/mma_probe.py "lean issue").
// Phase 11 (g0 of this tile, into columns kColG0..) also issues phase 0 of the slot's next
// tile (layer 1, A = x staged at kColX by phase 10's epilogue) when next_l1: one commit,
// one epilogue and one hand-off fewer per tile (11 phases per tile after the first).
template <bool F16, bool kElect = true>
DEVI void issue_phase(int p, uint32_t d, uint32_t sw, uint32_t sw1t, uint32_t sb1, uint32_t sbx, uint64_t *bar,
                      volatile uint32_t *turn = nullptr, uint32_t next_turn = 0u, bool next_l1 = false) {
  auto mma_ts = [](uint32_t dt, uint32_t at, uint64_t bd, uint32_t id, uint32_t acc) {
    if constexpr (kElect) tc::mma_ts_elect(dt, at, bd, id, acc);
    else tc::mma_ts(dt, at, bd, id, acc);
  };
  const uint32_t av = d + kColA;
  auto layer1 = [&]() {  // layer 1: K = 32 split operands (bias included), A = x
#pragma unroll
    for (int k = 0; k < 2; ++k)
      mma_ts(d, d + kColX + 8u * k, sdesc_nosw(sb1 + k * 2 * 2048, 2048, 128), kIdescFwd<F16>, k > 0);
  };
  if (p == 0) {
    layer1();
  } else if (p < 6) {  // layer l = p + 1: D = A W_l^T (B = W_l K-major) + ones x bias
    const uint32_t wb = sw + (uint32_t)(p - 1) * (H * H * 2);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      mma_ts(d, av + 8u * k, sdesc_sw128(wb + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), kIdescFwd<F16>, k > 0);
    mma_ts(d, d + kColOnes, sdesc_nosw(sbx + (uint32_t)(p - 1) * kBextBytes, 2048, 128), kIdescFwd<F16>, 1u);
  } else if (p < 11) {  // backward through layer l = 12 - p: D = E W_l, B = W_l MN-major
    const uint32_t wb = sw + (uint32_t)(10 - p) * (H * H * 2);
#pragma unroll
    for (int k = 0; k < 8; ++k) mma_ts(d, av + 8u * k, sdesc_sw128(wb + k * 2048, 16384, 1024), kIdescBwd<F16>, k > 0);
  } else {  // g0 = e1 W1 (N = 16 rows of W1^T) -> columns kColG0..; then the next tile's layer 1
#pragma unroll
    for (int k = 0; k < 8; ++k)
      mma_ts(d + kColG0, av + 8u * k, sdesc_sw128(sw1t + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024), kIdescFin<F16>,
             k > 0);
    if (next_l1) layer1();
  }
  if (turn) *turn = next_turn;  // (two MMA warps) the other slot may issue now
  if constexpr (kElect) commit_elect(bar);
  else tc::commit(bar);
}

// kSE2: the SE(2) frame variant (R24) as its own instantiation, so the default
// translation-frame kernel carries none of its code or registers
template <bool F16, bool kSE2>
__global__ void __launch_bounds__(kThreads, 1) k_mlp_tc(const WeightsBF16 W, const QueryArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned view (SWIZZLE_128B atoms); pointer arithmetic on the __shared__ array
  // keeps the shared address space visible to the compiler (LDS/STS, not generic LD/ST)
  SmemTC &S = *reinterpret_cast<SmemTC *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- one-time setup: the resident weights (already in their UMMA layouts in global
  // memory, 196 KB) -> smem by 1-D bulk copies (cp.async.bulk, the TMA engine) completing on
  // S.wbar; only the MMA warps wait for them (before their first UMMA), so the copy overlaps
  // the epilogue warps' staging of the first tiles ----
  if (tid == 0) {
    S.one = 1u;
    mbar_init(&S.wbar, 1);
    fence_barrier_init();
    constexpr uint32_t kChunk = 32768;
    mbar_expect_tx(&S.wbar, (uint32_t)(kWBytes + kW1tBytes + kB1Bytes + 5 * kBextBytes));
    for (uint32_t o = 0; o < (uint32_t)kWBytes; o += kChunk)
      bulk_g2s(S.w + o, static_cast<const uint8_t *>(W.w_sw128) + o, kChunk, &S.wbar);
    bulk_g2s(S.w1t, W.w1t_sw128, kW1tBytes, &S.wbar);
    bulk_g2s(S.b1, W.b1_nosw, kB1Bytes, &S.wbar);
    bulk_g2s(S.bext, W.bext_nosw, 5 * kBextBytes, &S.wbar);
  }
  if (warp == 0) {
    tmem_alloc(&S.tmem_base, 512);
    tmem_relinquish();
  }
  if (tid == 32) {
    mbar_init(&S.mma_done[0], 1);
    mbar_init(&S.mma_done[1], 1);
    mbar_init(&S.epi_done[0], kEpiArrivals);
    mbar_init(&S.epi_done[1], kEpiArrivals);
    S.turn = 0u;
    fence_barrier_init();
  }
  if (tid < 2 * kNdof) {  // q rows of the slots' first tiles (later tiles: cp.async, phases 1-3)
    const int s0 = tid / kNdof, i = tid - s0 * kNdof;
    const int64_t T0 = (int64_t)blockIdx.x * 2 + s0;
    if (T0 < query_tiles(a)) {
      const int w0 = tile_step(a, T0);
      S.qn[s0][0][i] = __ldg(a.q + (int64_t)w0 * kNdof + i);
      if (i == 0) S.wtile[s0][0] = w0;
    }
  }
  fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = S.tmem_base;
  const int64_t n_tiles = query_tiles(a);  // (partitioned: read from the device)
  const int64_t lb = a.scene.local_bound;
  const int64_t stride = 2 * (int64_t)gridDim.x;

  if (warp >= kEpiWarps) {
    // ===================== two MMA warps: warp 16 + s issues slot s's UMMAs ================
    // A commit stalls its issuing thread until the committed MMAs drain; with one issuer per
    // slot the other slot's UMMAs keep the tensor pipe busy meanwhile (tools/mma_probe.py
    // "two issuers").  The slots still alternate: a shared turn counter orders slot 0's
    // phase p before slot 1's phase p before slot 0's phase p + 1.
    const int ss = warp - kEpiWarps;
    const uint32_t sw = smem_u32(S.w), sw1t = smem_u32(S.w1t), sb1 = smem_u32(S.b1);
    const uint32_t sbx = smem_u32(S.bext);
    volatile uint32_t *turn = &S.turn;
    uint32_t ph = 0u;
    long long *tr0 = (a.trace && blockIdx.x == 0 && lane == 0) ? a.trace : nullptr;
    uint32_t seq = (uint32_t)ss;  // this slot's position in the global issue order
    int itt = 0;
    mbar_wait(&S.wbar, 0u);  // the resident weights have landed in shared memory
    for (int64_t base = (int64_t)blockIdx.x * 2; base < n_tiles; base += stride, ++itt) {
      const bool two = base + 1 < n_tiles;
      if (ss == 1 && !two) break;
      const bool next_l1 = base + stride + ss < n_tiles;  // this slot has a next tile
#pragma unroll 1
      for (int p = itt == 0 ? 0 : 1; p < kPhases; ++p, seq += 2) {
        long long *t = (tr0 && itt < kTraceTiles) ? tr0 + ((size_t)itt * kTracePhases + p) * 4 + 2 * ss : nullptr;
        long long *t2 = t ? t + (size_t)(kTraceRoles - 1) * kTraceTiles * kTracePhases * 4 : nullptr;
        if (t2) t2[0] = clock64();
        mbar_wait(&S.epi_done[ss], ph);
        ph ^= 1u;
        if (two) {
          const long long tw = clock64();
          while (*turn != seq) {
            if (clock64() - tw > (1ll << 34)) __trap();
          }
        }
        if (t2) t2[1] = clock64();
        fence_after();
        if (t) t[0] = clock64();
        issue_phase<F16>(p, tbase + (uint32_t)ss * 256u, sw, sw1t, sb1, sbx, &S.mma_done[ss], two ? turn : nullptr, seq + 1,
                         next_l1);
        if (t) t[1] = clock64();
      }
    }
    __syncwarp();
    fence_before();
    __syncthreads();
    return;
  }
  const int s = warp >> 3;          // tile slot
  const int hh = (warp >> 2) & 1;   // accumulator column half: units 64 hh .. 64 hh + 63
  const int qd = warp & 3;          // TMEM lane quarter of this warp (warp % 4)
  const int row = qd * 32 + lane;   // pair within the tile = TMEM lane
  const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
  const uint32_t tS = tbase + (uint32_t)s * 256u + lane_off;  // this slot, this lane quarter
  const uint32_t tD = tS + 64u * hh;
  const uint32_t tA = tS + kColA + 32u * hh;
  uint32_t *mk = &S.mask[s][0][0][hh * 128 + row];  // + (layer * 2 + word) * kEpiPerSlot
  if (hh == 0) {  // the constant "ones" A block of the bias GEMM step: {1, 1, 0, ...}
    uint32_t ones[8] = {pack2<F16>(1.f, 1.f), 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    st8(tS + kColOnes, ones);
  }
  // epilogue phase done: TMEM stores complete and ordered before the MMA warp's UMMAs
  auto hand_off = [&](int, bool) {
    wait_st();
    fence_before();
    mbar_arrive(&S.epi_done[s]);
  };
  // cp.async prefetch of this lane's point of tile TT into S.ptn[s][row] (zero if none);
  // issued by the column-half-0 threads, which alone read it
  // (the pair's local slot goes to S.slotn[s][par][row], read back by this same thread at
  // phases 6 and 11 and by stage_a1: no per-tile index arithmetic on the critical path)
  auto prefetch_pt = [&](int64_t TT, int par) {
    int wn = 0;
    int64_t sl = 0;
    bool ok = false;
    if (TT < n_tiles) tile_pair(a, TT, row, wn, sl, ok);
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
      }
      if (lane < kNdof) cp_async4(&S.qn[s][par][lane], a.q + (int64_t)wn * kNdof + lane);
      cp_async_commit();
      if (lane == 0) S.wtile[s][par] = wn;
    }
  };
  // A2 + A1 of tile TT: pair generation, base-frame bias p' = p - [q_x, q_y, 0]
  // and the split layer-1 operands -> TMEM A (K = 32: half 0 writes K 0..15,
  // half 1 K 16..31), then hand off.  Returns the pair's liveness (meaningful in half 0).
  // SE(2) frame (R24): p'_xy = R(-theta)(p_xy - b), theta channel fed 0; p'_xy is kept in
  // S.pprime[s][par] for the theta gradient at phase 11 (__sincosf: abs error ~1e-6 on
  // [-pi, pi], far below the 16-bit operand rounding).
  auto stage_a1 = [&](int64_t TT, int par) -> bool {
    const float *qw = S.qn[s][par];
    float v[16];
    bool lv = false;
    if (hh == 0) {  // K 0..15: p'_x, p'_y, p_z, theta, j1 (3 each), x_hi of j2
      const float4 pt = S.ptn[s][row];
      lv = S.slotn[s][par][row] != ~0u && pt.w > 0.f;
      float dx = pt.x - qw[0], dy = pt.y - qw[1], th = qw[2];
      if constexpr (kSE2) {
        float sn, cs;
        __sincosf(th, &sn, &cs);
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
    st8(tS + kColX + 8u * hh, a1);
    return lv;
  };
  const uint32_t one = S.one;
  // forward epilogue of layer l = p + 1 (p = 0..4): z = D (bias folded in); h = ReLU(z) -> A,
  // 1-bit masks -> smem, then hand off.  (16-column chunks, the TMEM load of chunk c + 1 in
  // flight while chunk c is packed.)  Phase 0 of every tile after the first runs inside the
  // previous tile's phase 11.
  auto fwd_epi = [&](int p, long long *tr) {
    uint32_t rb[2][16], m = 0u;
    ld16(tD, rb[0]);
    wait_ld();
    if (tr) tr[(p + 1) * 4 + 0] = clock64();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c < 3) ld16(tD + 16 * (c + 1), rb[(c + 1) & 1]);
      const uint32_t *rr = rb[c & 1];
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
      if (c < 3) wait_ld();
    }
    if (tr) tr[(p + 1) * 4 + 2] = clock64();
    hand_off(p + 1, true);
    if (tr) tr[(p + 1) * 4 + 3] = clock64();
  };
  uint32_t ph = 0u;
  int it = 0;
  const bool tracer = a.trace && blockIdx.x == 0 && lane == 0;  // lane 0 of every epilogue warp of CTA 0
  bool live_n = false;
  if ((int64_t)blockIdx.x * 2 + s < n_tiles) {
    if (hh == 0) {
      prefetch_pt((int64_t)blockIdx.x * 2 + s, 0);
      cp_async_wait_all();
    }
    live_n = stage_a1((int64_t)blockIdx.x * 2 + s, 0);
    hand_off(0, true);
  }
  for (int64_t T = (int64_t)blockIdx.x * 2 + s; T < n_tiles; T += stride, ++it) {
    long long *tr = (tracer && it < kTraceTiles) ? a.trace + (size_t)((1 + warp) * kTraceTiles + it) * kTracePhases * 4 : nullptr;
    if (tr) tr[0] = clock64();
    const bool live = live_n;
    float f = 0.f;
    int ridx = -1;  // staging record index (detect), -1 = none
    unsigned long long pend_b = 0ull;  // (row 0) staging allocation of this tile, in flight
    int pend_cnt = 0;
#pragma unroll 1
    for (int p = it == 0 ? 0 : 1; p < kPhases; ++p) {
      mbar_wait(&S.mma_done[s], ph);
      if (tr) tr[(p + 1) * 4 + 1] = clock64();
      ph ^= 1u;
      fence_after();
      if (p < 5) {
        fwd_epi(p, tr);
        if (p == 1 || p == 3) stage_q(p, T + stride, (it + 1) & 1);
      } else if (p == 5) {
        // ---- layer 6: e6 = w7 (.) 1[z6 > 0] -> A; f = w7 . ReLU(z6) + b7 (fp32) ----
        // (16-column chunks; the TMEM load of chunk c + 1 in flight while chunk c is used)
        float fa[4] = {0.f, 0.f, 0.f, 0.f};
        // the output row comes from the kernel parameters with compile-time offsets (one body
        // per column half), i.e. as direct constant-bank operands: no shared-memory loads
        auto layer6 = [&](auto u0c) {
          constexpr int U0 = decltype(u0c)::value;
          uint32_t rb[2][16];
          ld16(tD, rb[0]);
          wait_ld();
          if (tr) tr[(p + 1) * 4 + 0] = clock64();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int cb = 16 * c;
            if (c < 3) ld16(tD + cb + 16, rb[(c + 1) & 1]);
            const uint32_t *rr = rb[c & 1];
            uint32_t pk[8];
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              const int u = U0 + cb + j;
              const float z0 = __uint_as_float(rr[j]), z1 = __uint_as_float(rr[j + 1]);
              const float z2 = __uint_as_float(rr[j + 2]), z3 = __uint_as_float(rr[j + 3]);
              pk[j >> 1] = W.w7h_p[u / 2] & nz_halves(pack2_relu<F16>(z0, z1), one);
              pk[(j >> 1) + 1] = W.w7h_p[u / 2 + 1] & nz_halves(pack2_relu<F16>(z2, z3), one);
              // (w7 / 2) (z + |z|) = w7 ReLU(z) exactly (z + |z| = 2 ReLU(z), halving is exact)
              fa[0] = fmaf(W.w7half_p[u], z0 + fabsf(z0), fa[0]);
              fa[1] = fmaf(W.w7half_p[u + 1], z1 + fabsf(z1), fa[1]);
              fa[2] = fmaf(W.w7half_p[u + 2], z2 + fabsf(z2), fa[2]);
              fa[3] = fmaf(W.w7half_p[u + 3], z3 + fabsf(z3), fa[3]);
            }
            st8(tA + cb / 2, pk);
            if (c < 3) wait_ld();
          }
        };
        if (hh == 0) layer6(std::integral_constant<int, 0>{});
        else layer6(std::integral_constant<int, 64>{});
        if (tr) tr[(p + 1) * 4 + 2] = clock64();
        hand_off(p + 1, s == 1 || T + 1 < n_tiles);
        if (tr) tr[(p + 1) * 4 + 3] = clock64();
        // f = w7 . h6 + b7 (fp32, no output activation: signed value)
        S.fpart[s][hh][row] = (fa[0] + fa[1]) + (fa[2] + fa[3]);
        if (hh == 0 && qd == 0) cp_async_wait_all();  // S.qn of the next tile (stage_q)
        named_bar_sync(1 + s, kEpiPerSlot);
        if (hh == 0) {
          f = S.fpart[s][0][row] + S.fpart[s][1][row] + W.b7;
          if (!a.detect) {
            const int w = S.wtile[s][it & 1];
            const int64_t slot = S.slotn[s][it & 1][row];
            if (slot < lb) a.values[(int64_t)w * lb + slot] = live ? f : __int_as_float(0x7f800000);
          }
          prefetch_pt(T + stride, (it + 1) & 1);  // the next tile's point, needed at phase 10
        }
      } else if (p < 11) {
        // ---- backward: g_{l-1} = D; e_{l-1} = g (.) 1[z_{l-1} > 0] -> A ----
        const int mi = 10 - p;
        const uint32_t mw[2] = {mk[(mi * 2) * kEpiPerSlot], mk[(mi * 2 + 1) * kEpiPerSlot]};
        uint32_t rb[2][16];
        ld16(tD, rb[0]);
        wait_ld();
        if (tr) tr[(p + 1) * 4 + 0] = clock64();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < 3) ld16(tD + 16 * (c + 1), rb[(c + 1) & 1]);
          const uint32_t *rr = rb[c & 1];
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            uint32_t lo, hi;
            mask_expand(mw[c >> 1], ((c & 1) * 16 + j) >> 2, lo, hi);
            pk[j >> 1] = pack2<F16>(__uint_as_float(rr[j]), __uint_as_float(rr[j + 1])) & lo;
            pk[(j >> 1) + 1] = pack2<F16>(__uint_as_float(rr[j + 2]), __uint_as_float(rr[j + 3])) & hi;
          }
          st8(tA + 8 * c, pk);
          if (c < 3) wait_ld();
        }
        if (p == 10 && T + stride < n_tiles) {
          // A2 + A1 of the slot's next tile -> x (kColX), issued with this tile's g0 GEMM
          if (hh == 0) cp_async_wait_all();  // this thread's point of the next tile (phase 5)
          live_n = stage_a1(T + stride, (it + 1) & 1);
        }
        if (tr) tr[(p + 1) * 4 + 2] = clock64();
        hand_off(p + 1, s == 1 || T + 1 < n_tiles);
        if (tr) tr[(p + 1) * 4 + 3] = clock64();
        if (p == 6 && hh == 0 && a.detect) {
          // A6/A7 (overlaps the tensor core): threshold, per-tile slots, per-waypoint min key
          const int w = S.wtile[s][it & 1];
          const int64_t slot = S.slotn[s][it & 1][row];  // (live implies a real pair)
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
          ridx = act ? rk : -1;  // rank in the tile; the tile's staging base is added at phase 11
          if (row == 0) {
            unsigned long long km = S.kmin[s][0];
            int cnt = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              km = S.kmin[s][i] < km ? S.kmin[s][i] : km;
              cnt += __popc(S.act[s][i]);
            }
            if (km != ~0ull) atomicMin(a.ds.wp_key + w, km);
            // staging allocation: the (contended) atomic's result is consumed two phases
            // later, so its latency stays off the epilogue's critical path
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
        // ---- phase 11 + phase 0 of the slot's next tile: the UMMAs were issued together ----
        // first the next tile's layer-1 epilogue (so its phase 1 can be issued), then g0 =
        // W1^T e1 (16 columns at kColG0) -> d f / d q by the chain rule (R3) and the outputs
        if (T + stride < n_tiles) fwd_epi(0, nullptr);
        uint32_t r[16];
        if (hh == 0) {
          ld16(tS + kColG0, r);
          wait_ld();
        }
        if (tr) tr[(p + 1) * 4 + 0] = clock64();
        if (tr) tr[(p + 1) * 4 + 2] = clock64();
        if (hh == 0) {
          const int w = S.wtile[s][it & 1];
          const int64_t slot = S.slotn[s][it & 1][row];
          if (tr) tr[1] = clock64();  // (phase-11 detail: step and slot read)
          float gq[kNdof];
          gq[0] = a.tgrad ? __uint_as_float(r[3]) : -__uint_as_float(r[0]);
          gq[1] = a.tgrad ? __uint_as_float(r[4]) : -__uint_as_float(r[1]);
#pragma unroll
          for (int i = 0; i < 7; ++i) gq[2 + i] = __uint_as_float(r[5 + i]);
          if constexpr (kSE2) {  // SE(2) (R24): df/db = -R(theta) g0_xy, df/dtheta = g0_x p'_y - g0_y p'_x
            float sn, cs;
            __sincosf(S.qn[s][it & 1][2], &sn, &cs);
            const float gx = __uint_as_float(r[0]), gy = __uint_as_float(r[1]);
            const float2 pp = S.pprime[s][it & 1][row];
            gq[0] = -(cs * gx - sn * gy);
            gq[1] = -(sn * gx + cs * gy);
            gq[2] = gx * pp.y - gy * pp.x;
          }
          if (a.detect) {
            named_bar_sync(3 + s, 128);  // S.sbase[s] (written at phase 8 by row 0) is visible
            if (tr) tr[2] = clock64();  // (phase-11 detail: barrier passed)
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
        if (tr) tr[(p + 1) * 4 + 3] = clock64();
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <bool F16>
cudaError_t launch_tc_t(const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  const int smem = (int)sizeof(SmemTC) + 1024;
  auto kern = a.frame ? k_mlp_tc<F16, true> : k_mlp_tc<F16, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  // a partitioned detect knows its tile count on the device only: one CTA per SM
  const int64_t n_tiles = a.part.tile_wp ? 2 * (int64_t)num_sms : (int64_t)a.n_wp * a.tiles_per_wp;
  int64_t grid = (n_tiles + 1) / 2;
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
