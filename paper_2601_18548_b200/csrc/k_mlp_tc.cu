// k_mlp_tc.cu -- K2b: fused pair generation + base-frame transform + 7-layer MLP forward
// + input-gradient backward (+ threshold / min / per-tile compaction in detect mode) on
// the 5th-generation tensor cores (tcgen05, fp16 or bf16 operands, fp32 accumulation in TMEM).
//
// Paper steps (PAPER.md lines): base-frame bias :388/:171; "7-layer MLP" on [p, q] :284;
// value + gradient :394 (dense gradient R^{NM x n}); constraint f - delta >= 0 :362-363;
// union = min :164; c_gcdf step-major order :414-435.  DESIGN.md §5 "K2b".
//
// Design (H = 128, one persistent CTA per SM, 640 threads = 20 warps):
//   * The ten H x H hidden-layer GEMMs of a 128-pair tile run as UMMA 128x128x16 with
//     A = activations (16-bit) in TMEM and B = W_l (16-bit) resident in shared memory for
//     the whole kernel (5 x 32 KB, UMMA SWIZZLE_128B).  The same smem bytes are the
//     K-major B of the forward GEMM (D = h W^T) and the MN-major B of the backward GEMM
//     (D = e W).  The last backward GEMM g0 = e1 W1 is a 128x16x128 UMMA against W1^T.
//   * Activations never leave the chip: accumulator D (fp32, 128 TMEM columns) ->
//     epilogue registers (bias, ReLU, 1-bit mask, 16-bit pack) -> A (64 TMEM columns) ->
//     next UMMA.  ReLU masks stay in registers (12 x 32 bit per thread) for the backward.
//   * Two tiles in flight: TMEM columns [0,256) belong to slot 0 and [256,512) to slot
//     1.  Each slot has 8 epilogue warps: warp (h, q) owns TMEM lanes 32q..32q+31 (the
//     tile's pairs) and accumulator columns 64h..64h+63, so every SM sub-partition runs
//     two warps per slot (latency hiding) and one slot's epilogue overlaps the other
//     slot's tensor-core work.  One elected thread of warp 0 issues all UMMAs.
//   * Layer 1 (12 -> H) runs in fp32 on the CUDA cores (3 FMA per unit per pair plus a
//     per-waypoint constant), so the metre-scale point coordinates are never rounded
//     to 16 bits (R16).
//   * Synchronisation: mma_done[s] (tcgen05.commit -> mbarrier, count 1) and epi_done[s]
//     (256 epilogue arrivals); 11 phases per tile.
#include "gcdf_internal.h"
#include "tc_ptx.h"

namespace gcdf {
namespace {

using namespace tc;

constexpr int H = 128;
constexpr int kWarps = 20;
constexpr int kThreads = kWarps * 32;
constexpr int kEpiPerSlot = 256;
constexpr int kWBytes = 5 * H * H * 2;  // 163,840
constexpr int kW1tBytes = 16 * H * 2;   // 4,096
template <bool F16> constexpr uint32_t kIdescFwd = idesc_f16kind(128, 128, false, F16);
template <bool F16> constexpr uint32_t kIdescBwd = idesc_f16kind(128, 128, true, F16);
template <bool F16> constexpr uint32_t kIdescFin = idesc_f16kind(128, 16, false, F16);

struct __align__(1024) SmemTC {
  uint8_t w[kWBytes];        // W_2..W_6, SW128 [2 chunks][128 rows][128 B] each
  uint8_t w1t[kW1tBytes];    // W1^T [16][128], SW128
  float4 w1c[2][H];          // per slot: {W1[u][0], W1[u][1], W1[u][2], c_u(waypoint)}
  float w1q[H * 8];
  float bias[5 * H];
  float w7[H];
  float fpart[2][2][H];      // [slot][half][row] partial output-layer sums
  uint32_t mask[2][kHidden][2][kEpiPerSlot];  // ReLU masks: [slot][layer][32-unit word][thread]
  uint64_t mma_done[2];
  uint64_t epi_done[2];
  unsigned act[2][4];
  unsigned long long kmin[2][4];
  int sbase[2];
  uint32_t tmem_base;
};

DEVI unsigned ord_f32(float f) {
  unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}


template <bool F16>
__global__ void __launch_bounds__(kThreads, 1) k_mlp_tc(const WeightsBF16 W, const QueryArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned view (SWIZZLE_128B atoms); pointer arithmetic on the __shared__ array
  // keeps the shared address space visible to the compiler (LDS/STS, not generic LD/ST)
  SmemTC &S = *reinterpret_cast<SmemTC *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- one-time setup: weights -> smem (already in UMMA layout in global memory) ----
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(W.w_sw128);
    uint4 *dst = reinterpret_cast<uint4 *>(S.w);
    for (int i = tid; i < kWBytes / 16; i += kThreads) dst[i] = __ldg(src + i);
    const uint4 *src1 = reinterpret_cast<const uint4 *>(W.w1t_sw128);
    uint4 *dst1 = reinterpret_cast<uint4 *>(S.w1t);
    for (int i = tid; i < kW1tBytes / 16; i += kThreads) dst1[i] = __ldg(src1 + i);
    for (int i = tid; i < H * 8; i += kThreads) S.w1q[i] = __ldg(W.w1q + i);
    for (int i = tid; i < 5 * H; i += kThreads) S.bias[i] = __ldg(W.bias + i);
    for (int i = tid; i < H; i += kThreads) S.w7[i] = __ldg(W.w7 + i);
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
    fence_barrier_init();
  }
  fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = S.tmem_base;
  const int64_t n_tiles = (int64_t)a.n_wp * a.tiles_per_wp;
  const int64_t lb = a.scene.local_bound;

  if (warp == 0) {
    // =========================== MMA issuer (one thread) ===========================
    if (lane == 0) {
      const uint32_t sw = smem_u32(S.w), sw1t = smem_u32(S.w1t);
      uint32_t phbits = 0u;  // bit s = phase parity of epi_done[s]
      for (int64_t base = (int64_t)blockIdx.x * 2; base < n_tiles; base += 2 * (int64_t)gridDim.x) {
        const int nslots = (base + 1 < n_tiles) ? 2 : 1;
#pragma unroll 1
        for (int p = 0; p < 11; ++p) {
#pragma unroll 1
          for (int s = 0; s < nslots; ++s) {
            mbar_wait(&S.epi_done[s], (phbits >> s) & 1u);
            phbits ^= 1u << s;
            fence_after();
            const uint32_t d = tbase + (uint32_t)s * 256u, av = d + 128u;
            if (p < 5) {  // forward, layer l = p + 2: D = A W_l^T, B = W_l K-major
              const uint32_t wb = sw + (uint32_t)p * (H * H * 2);
#pragma unroll
              for (int k = 0; k < 8; ++k)
                mma_ts(d, av + 8u * k, sdesc_sw128(wb + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), kIdescFwd<F16>,
                       k > 0);
            } else if (p < 10) {  // backward through layer l = 11 - p: D = E W_l, B = W_l MN-major
              const uint32_t wb = sw + (uint32_t)(9 - p) * (H * H * 2);
#pragma unroll
              for (int k = 0; k < 8; ++k)
                mma_ts(d, av + 8u * k, sdesc_sw128(wb + k * 2048, 16384, 1024), kIdescBwd<F16>, k > 0);
            } else {  // g0 = e1 W1 (N = 16 rows of W1^T)
#pragma unroll
              for (int k = 0; k < 8; ++k)
                mma_ts(d, av + 8u * k, sdesc_sw128(sw1t + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024), kIdescFin<F16>,
                       k > 0);
            }
            commit(&S.mma_done[s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // =========================== epilogue warps ===========================
    const int e = warp - 4;
    const int s = e >> 3;             // tile slot
    const int hh = (e >> 2) & 1;      // accumulator column half: units 64 hh .. 64 hh + 63
    const int qd = warp & 3;          // TMEM lane quarter of this warp (warp % 4)
    const int row = qd * 32 + lane;   // pair within the tile = TMEM lane
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const uint32_t tD = tbase + (uint32_t)s * 256u + lane_off + 64u * hh;
    const uint32_t tA = tbase + (uint32_t)s * 256u + 128u + lane_off + 32u * hh;
    const int u0 = 64 * hh;           // first unit of this thread's columns
    uint32_t ph = 0u;
    for (int64_t T = (int64_t)blockIdx.x * 2 + s; T < n_tiles; T += 2 * (int64_t)gridDim.x) {
      const int w = (int)(T / a.tiles_per_wp);
      const int64_t slot = (T % a.tiles_per_wp) * kTile + row;
      const float *qw = a.q + (int64_t)w * kNdof;
      // A2: pair generation + base-frame bias p' = p - [q_x, q_y, 0]
      const float4 pt = slot < lb ? __ldg(a.scene.pts + slot) : make_float4(0.f, 0.f, 0.f, 0.f);
      const bool live = slot < lb && pt.w > 0.f;
      const float px = pt.x - __ldg(qw), py = pt.y - __ldg(qw + 1), pz = pt.z;
      // layer-1 constant of this waypoint for unit u = row: c = b1 + W1[u, 5:12] . [theta, j1..j6]
      if (hh == 0) {
        const float4 wv = __ldg(W.w1p + row);
        float c = wv.w;
#pragma unroll
        for (int i = 0; i < 7; ++i) c = fmaf(S.w1q[row * 8 + i], __ldg(qw + 2 + i), c);
        S.w1c[s][row] = make_float4(wv.x, wv.y, wv.z, c);
      }
      named_bar_sync(1 + s, kEpiPerSlot);

      uint32_t *mk = &S.mask[s][0][0][hh * 128 + row];  // + (layer * 2 + word) * kEpiPerSlot
      // ---- E0: layer 1 in fp32 on CUDA cores -> h1 (16-bit) into TMEM A ----
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        uint32_t pk[16], m = 0u;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float z[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 a0 = S.w1c[s][u0 + c2 * 32 + j + i];
            z[i] = fmaf(a0.x, px, fmaf(a0.y, py, fmaf(a0.z, pz, a0.w)));
          }
          pk[j >> 1] = pack2_relu<F16>(z[0], z[1]);
          pk[(j >> 1) + 1] = pack2_relu<F16>(z[2], z[3]);
          m |= mask_group(pk[j >> 1], pk[(j >> 1) + 1], j >> 2);
        }
        mk[c2 * kEpiPerSlot] = m;
        st16(tA + c2 * 16, pk);
      }
      wait_st();
      fence_before();
      mbar_arrive(&S.epi_done[s]);

      float f = 0.f;
      bool act = false;
      int my_base = -1, my_rank = 0;
#pragma unroll 1
      for (int p = 0; p < 11; ++p) {
        mbar_wait(&S.mma_done[s], ph);
        ph ^= 1u;
        fence_after();
        if (p < 5) {
          // ---- forward hidden layer l = p + 2: z = D + b, h = ReLU(z) -> A ----
          //      (l = 6: f += w7 . h6 in fp32, e6 = w7 (.) 1[z6 > 0] -> A)
          float fp = 0.f;
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            uint32_t m = 0u;
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {  // 16 accumulator columns per TMEM load
              uint32_t r[16], pk[8];
              const int cb = c2 * 32 + hf * 16;
              ld16(tD + cb, r);
              wait_ld();
              const float *bp = S.bias + p * H + u0 + cb;
#pragma unroll
              for (int j = 0; j < 16; j += 4) {
                const float4 b = *reinterpret_cast<const float4 *>(bp + j);
                const float z0 = __uint_as_float(r[j]) + b.x, z1 = __uint_as_float(r[j + 1]) + b.y;
                const float z2 = __uint_as_float(r[j + 2]) + b.z, z3 = __uint_as_float(r[j + 3]) + b.w;
                const int jb = hf * 16 + j;
                if (p < 4) {
                  pk[j >> 1] = pack2_relu<F16>(z0, z1);
                  pk[(j >> 1) + 1] = pack2_relu<F16>(z2, z3);
                  m |= mask_group(pk[j >> 1], pk[(j >> 1) + 1], jb >> 2);
                } else {  // layer 6: its mask is applied right here (e6), never stored
                  const float4 w7 = *reinterpret_cast<const float4 *>(S.w7 + u0 + cb + j);
                  fp = fmaf(w7.x, fmaxf(z0, 0.f), fp);
                  fp = fmaf(w7.y, fmaxf(z1, 0.f), fp);
                  fp = fmaf(w7.z, fmaxf(z2, 0.f), fp);
                  fp = fmaf(w7.w, fmaxf(z3, 0.f), fp);
                  pk[j >> 1] = pack2<F16>(z0 > 0.f ? w7.x : 0.f, z1 > 0.f ? w7.y : 0.f);
                  pk[(j >> 1) + 1] = pack2<F16>(z2 > 0.f ? w7.z : 0.f, z3 > 0.f ? w7.w : 0.f);
                }
              }
              st8(tA + cb / 2, pk);
            }
            if (p < 4) mk[((p + 1) * 2 + c2) * kEpiPerSlot] = m;
          }
          wait_st();
          fence_before();
          mbar_arrive(&S.epi_done[s]);
          if (p == 4) {
            // f = w7 . h6 + b7 (fp32, no output activation: signed value)
            S.fpart[s][hh][row] = fp;
            named_bar_sync(1 + s, kEpiPerSlot);
            f = S.fpart[s][0][row] + S.fpart[s][1][row] + W.b7;
            // A6/A7 (overlaps the next UMMA): threshold, per-tile slots, per-waypoint min key
            if (hh == 0) {
              if (a.detect) {
                act = live && (f - a.delta <= a.tau);
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
                if (row == 0) {
                  unsigned long long km = S.kmin[s][0];
                  int cnt = 0;
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    km = S.kmin[s][i] < km ? S.kmin[s][i] : km;
                    cnt += __popc(S.act[s][i]);
                  }
                  if (km != ~0ull) atomicMin(a.ds.wp_key + w, km);
                  int base = 0;
                  if (cnt > 0) {
                    const unsigned long long b = atomicAdd(a.ds.counter, (unsigned long long)cnt);
                    if (b + cnt > (unsigned long long)a.ds.max_active) {
                      atomicOr(a.ds.counter + 1, 1ull);
                      base = -1;
                    } else {
                      base = (int)b;
                    }
                  }
                  S.sbase[s] = base;
                  a.ds.tile_meta[T] = make_int2(base, cnt);
                }
                named_bar_sync(3 + s, 128);
                my_base = S.sbase[s];
                my_rank = __popc(bal & ((1u << lane) - 1u));
                for (int i = 0; i < qd; ++i) my_rank += __popc(S.act[s][i]);
              } else if (slot < lb) {
                a.values[(int64_t)w * lb + slot] = live ? f : __int_as_float(0x7f800000);
              }
            }
          }
        } else if (p < 10) {
          // ---- backward: g_{l-1} = D; e_{l-1} = g (.) 1[z_{l-1} > 0] -> A ----
          const int mi = 9 - p;
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const uint32_t m = mk[(mi * 2 + c2) * kEpiPerSlot];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              uint32_t r[16], pk[8];
              const int cb = c2 * 32 + hf * 16;
              ld16(tD + cb, r);
              wait_ld();
#pragma unroll
              for (int j = 0; j < 16; j += 4) {
                uint32_t lo, hi;
                mask_expand(m, (hf * 16 + j) >> 2, lo, hi);
                pk[j >> 1] = pack2<F16>(__uint_as_float(r[j]), __uint_as_float(r[j + 1])) & lo;
                pk[(j >> 1) + 1] = pack2<F16>(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])) & hi;
              }
              st8(tA + cb / 2, pk);
            }
          }
          wait_st();
          fence_before();
          mbar_arrive(&S.epi_done[s]);
        } else if (hh == 0) {
          // ---- g0 = W1^T e1 (16 columns); d f / d q by the chain rule (R3) ----
          uint32_t r[16];
          ld16(tbase + (uint32_t)s * 256u + lane_off, r);
          wait_ld();
          float gq[kNdof];
          gq[0] = a.tgrad ? __uint_as_float(r[3]) : -__uint_as_float(r[0]);
          gq[1] = a.tgrad ? __uint_as_float(r[4]) : -__uint_as_float(r[1]);
#pragma unroll
          for (int i = 0; i < 7; ++i) gq[2 + i] = __uint_as_float(r[5 + i]);
          if (a.detect) {
            if (act && my_base >= 0) {
              float4 *dst = reinterpret_cast<float4 *>(a.ds.staging + my_base + my_rank);
              dst[0] = make_float4(f, gq[0], gq[1], gq[2]);
              dst[1] = make_float4(gq[3], gq[4], gq[5], gq[6]);
              dst[2] = make_float4(gq[7], gq[8], __uint_as_float((unsigned)w),
                                   __uint_as_float((unsigned)local_to_global(slot, a.scene.rank, a.scene.world)));
            }
          } else if (a.grads && slot < lb) {
            float *o = a.grads + ((int64_t)w * lb + slot) * kNdof;
#pragma unroll
            for (int i = 0; i < kNdof; ++i) o[i] = live ? gq[i] : 0.f;
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

// ------------------------------------------------------------------ self-test kernel
// One UMMA building block, for unit tests: A fp32 [128][128] -> 16-bit TMEM, B fp32
// [nrows][128] -> 16-bit SW128 smem; mode 0: D = A B^T (K-major B, N = 128); mode 1:
// D = A B (B read MN-major, N = 128); mode 2: D = A B^T with nrows = 16 (N = 16).
template <bool F16>
__global__ void __launch_bounds__(128, 1) k_selftest_umma(const float *A, const float *B, int mode, float *D) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sb = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nrows = mode == 2 ? 16 : 128;
  for (int i = tid; i < nrows * 128; i += 128) {
    const int r = i / 128, c = i % 128;
    const int chunk = c / 64, cb = (c % 64) * 2, g = cb / 16;
    const int byte = chunk * nrows * 128 + r * 128 + ((g ^ (r % 8)) * 16) + (cb % 16);
    const uint32_t v = pack2<F16>(B[i], 0.f);
    *reinterpret_cast<uint16_t *>(sb + byte) = (uint16_t)(v & 0xffffu);
  }
  if (warp == 0) {
    tmem_alloc(&tb, 256);
    tmem_relinquish();
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t0 = tb + ((uint32_t)(warp * 32) << 16);
  {
    const int m = warp * 32 + lane;
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4) {
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) pk[j] = pack2<F16>(A[m * 128 + c4 * 32 + 2 * j], A[m * 128 + c4 * 32 + 2 * j + 1]);
      st16(t0 + 128 + c4 * 16, pk);
    }
    wait_st();
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    const uint32_t sbase = smem_u32(sb);
    for (int k = 0; k < 8; ++k) {
      uint64_t bd;
      uint32_t id;
      if (mode == 0) { bd = sdesc_sw128(sbase + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024); id = kIdescFwd<F16>; }
      else if (mode == 1) { bd = sdesc_sw128(sbase + k * 2048, 16384, 1024); id = kIdescBwd<F16>; }
      else { bd = sdesc_sw128(sbase + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024); id = kIdescFin<F16>; }
      mma_ts(tb, tb + 128 + 8 * k, bd, id, k > 0);
    }
    commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after();
  {
    const int m = warp * 32 + lane;
    if (mode == 2) {
      uint32_t r[16];
      ld16(t0, r);
      wait_ld();
      for (int j = 0; j < 16; ++j) D[m * 128 + j] = __uint_as_float(r[j]);
    } else {
      for (int c4 = 0; c4 < 4; ++c4) {
        uint32_t r[32];
        ld32(t0 + c4 * 32, r);
        wait_ld();
        for (int j = 0; j < 32; ++j) D[m * 128 + c4 * 32 + j] = __uint_as_float(r[j]);
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tb, 256);
}

template <bool F16>
cudaError_t launch_tc_t(const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  const int smem = (int)sizeof(SmemTC) + 1024;
  cudaError_t e = cudaFuncSetAttribute(k_mlp_tc<F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t n_tiles = (int64_t)a.n_wp * a.tiles_per_wp;
  int64_t grid = (n_tiles + 1) / 2;
  if (grid > num_sms) grid = num_sms;
  if (grid < 1) return cudaSuccess;
  k_mlp_tc<F16><<<(unsigned)grid, kThreads, smem, s>>>(w, a);
  return cudaGetLastError();
}

template <bool F16>
cudaError_t selftest_t(int mode, const float *A, const float *B, float *D, cudaStream_t s) {
  const int smem = 32768 + 1024;
  cudaError_t e = cudaFuncSetAttribute(k_selftest_umma<F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k_selftest_umma<F16><<<1, 128, smem, s>>>(A, B, mode, D);
  return cudaGetLastError();
}

}  // namespace

bool tc_compiled() { return true; }

cudaError_t launch_mlp_tc(int Hh, bool f16, const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s) {
  if (Hh != H) return cudaErrorInvalidValue;
  return f16 ? launch_tc_t<true>(w, a, num_sms, s) : launch_tc_t<false>(w, a, num_sms, s);
}

cudaError_t launch_selftest_umma(int mode, const float *A, const float *B, float *D, cudaStream_t s) {
  return (mode & 4) ? selftest_t<true>(mode & 3, A, B, D, s) : selftest_t<false>(mode & 3, A, B, D, s);
}

}  // namespace gcdf
