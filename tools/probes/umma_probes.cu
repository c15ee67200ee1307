// umma_probes.cu -- diagnostics only, NOT part of libgcdf.so: tcgen05 UMMA issue/throughput
// probes (one CTA, back-to-back UMMAs timed with clock64; CTA-pair probes; sub-partition
// interference).  Their measurements are in profiles/r1/mma_probe.txt and DESIGN.md §5.
// Build + run: python tools/mma_probe.py (builds build/probes/libumma_probes.so with nvcc).
#include <cstdint>
#include "../../paper_2601_18548_b200/csrc/gcdf_internal.h"
#include "../../paper_2601_18548_b200/csrc/tc_ptx.h"

namespace gcdf {
namespace {
using namespace tc;
template <bool F16> constexpr uint32_t kIdescFwd = idesc_f16kind(128, 128, false, F16);
template <bool F16> constexpr uint32_t kIdescBwd = idesc_f16kind(128, 128, true, F16);
template <bool F16> constexpr uint32_t kIdescFin = idesc_f16kind(128, 16, false, F16);
}  // namespace
// ------------------------------------------------------------------ UMMA throughput probe
// One CTA, one issuing thread, `reps` back-to-back groups of 8 K-steps (K = 128), then one
// commit; D[0] = clock64 cycles from the first issue to completion, D[1] = MMAs issued.
// variant 0: TS, B K-major SW128, N = 128;  1: TS, B MN-major, N = 128;
// 2: TS, N = 128, two independent accumulators alternating;  3: SS (A in smem, K-major
// SW128), N = 128;  4: TS, N = 256 (B rows 0..255).
namespace {
template <bool F16>
__global__ void __launch_bounds__(128, 1) k_mma_probe(int variant, int reps, float *D) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sb = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 64 KB B + 32 KB A
  __shared__ uint64_t bar, bar2, bar3;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  // operands: zeros, or (variant 18) random fp16 values in [-1, 1) like real weights
  auto rnd16 = [](uint32_t x) -> uint32_t {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return pack2<F16>((float)(x & 0xffff) / 32768.f - 1.f, (float)(x >> 16) / 32768.f - 1.f);
  };
  for (int i = tid; i < (96 * 1024) / 16; i += 128)
    reinterpret_cast<uint4 *>(sb)[i] = variant == 18 ? make_uint4(rnd16(4 * i), rnd16(4 * i + 1), rnd16(4 * i + 2), rnd16(4 * i + 3))
                                                     : make_uint4(0, 0, 0, 0);
  if (warp == 0) {
    tmem_alloc(&tb, 512);
    tmem_relinquish();
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    mbar_init(&bar3, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  if (variant == 18) {  // random A operand in TMEM columns 256..319
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = rnd16(1000003u * tid + i);
    st32(tb + ((uint32_t)(warp * 32) << 16) + 256u, r);
    st32(tb + ((uint32_t)(warp * 32) << 16) + 288u, r);
    wait_st();
    fence_before();
    __syncthreads();
    fence_after();
  }
  __shared__ volatile int stop;
  if (tid == 0) stop = 0;
  __syncthreads();
  if (tid >= 32 && (variant == 16 || variant == 17)) {
    // TMEM traffic of "epilogue" warps (columns 384..511) while warp 0 streams UMMAs
    const uint32_t tq = tb + ((uint32_t)(warp * 32) << 16) + 384u;
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = (uint32_t)i;
    while (!stop) {
      if (variant == 16) {
        ld32(tq, r);
        wait_ld();
      } else {
        st32(tq, r);
        wait_st();
      }
    }
    if (r[5] == 12345u) D[2] = 1.f;  // keep the loads alive
  }
  if (variant == 23 && warp < 2) {
    // two issuing warps (one per slot), each: forward phases (8 K-major + bias) with a
    // commit per phase to its own mbarrier; does a second issuer hide the commit bubble?
    const uint32_t sB = smem_u32(sb), sA = sB + 65536;
    const uint32_t dd = tb + (uint32_t)warp * 256u;
    uint64_t bdk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) bdk[k] = sdesc_sw128(sB + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
    const uint64_t bx = sdesc_nosw(sA, 2048, 128);
    uint64_t *mb = warp == 0 ? &bar2 : &bar3;
    __syncwarp();
    asm volatile("bar.sync 1, 64;" ::: "memory");
    const long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < reps / 2; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_ts_elect(dd, dd + 128 + 8u * k, bdk[k], kIdescFwd<F16>, k > 0);
      mma_ts_elect(dd, dd + 192, bx, kIdescFwd<F16>, 1u);
      commit_elect(mb);
    }
    mbar_wait(mb, (uint32_t)((reps / 2 - 1) & 1));
    asm volatile("bar.sync 1, 64;" ::: "memory");
    const long long t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) {
      D[0] = (float)(t1 - t0);
      D[1] = (float)((reps / 2) * 2 * 9);
    }
  }
  if (tid == 0 && variant != 23) {
    const uint32_t sB = smem_u32(sb), sA = sB + 65536;
    const uint32_t d0 = tb, av = tb + 256;
    long long t0 = clock64();
    int n = 0;
    if (variant >= 13) {  // minimal issue overhead: descriptors precomputed, branch-free loop
      uint64_t bd[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        bd[k] = variant != 14 ? sdesc_sw128(sB + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024)
                              : sdesc_sw128(sB + k * 2048, 16384, 1024);
      const uint32_t idesc = variant != 14 ? kIdescFwd<F16> : kIdescBwd<F16>;
      const uint64_t bx = sdesc_nosw(sA, 2048, 128);
      t0 = clock64();
      if (variant == 19) {  // the kernel's forward phase: 8 K-major steps + a no-swizzle bias step
#pragma unroll 1
        for (int r = 0; r < reps; ++r) {
#pragma unroll
          for (int k = 0; k < 8; ++k) mma_ts(d0, d0 + 128 + 8u * k, bd[k], idesc, k > 0);
          mma_ts(d0, d0 + 192, bx, idesc, 1u);
        }
        n = reps * 9;
      } else if (variant == 24) {  // as 22 with a test_wait spin instead of try_wait
#pragma unroll 1
        for (int r = 0; r < reps; ++r) {
#pragma unroll
          for (int k = 0; k < 8; ++k) mma_ts(d0, d0 + 128 + 8u * k, bd[k], idesc, k > 0);
          mma_ts(d0, d0 + 192, bx, idesc, 1u);
          commit(&bar2);
          mbar_wait_spin(&bar2, (uint32_t)(r & 1));
          fence_after();
        }
        n = reps * 9;
      } else if (variant == 28 || variant == 29) {  // lean M = 64 (28: one D; 29: two D at lanes 0 / 64 alternating)
        const uint32_t id64 = idesc_f16kind(64, 128, false, F16);
#pragma unroll 1
        for (int r = 0; r < reps; ++r) {
          const uint32_t dd = (variant == 29 && (r & 1)) ? d0 + (64u << 16) : d0;
#pragma unroll
          for (int k = 0; k < 8; ++k) mma_ts(dd, av + 8u * k, bd[k], id64, k > 0);
        }
        n = reps * 8;
      } else if (variant == 25) {  // lean N = 64 (two halves of a phase as separate accumulators)
        uint64_t b64[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) b64[k] = sdesc_sw128(sB + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024);
#pragma unroll 1
        for (int r = 0; r < reps; ++r) {
#pragma unroll
          for (int k = 0; k < 8; ++k) mma_ts(d0 + (uint32_t)(r & 1) * 64u, d0 + 128 + 8u * k, b64[k], idesc_f16kind(128, 64, false, F16), k > 0);
        }
        n = reps * 8;
      } else if (variant == 21 || variant == 22) {
        // the kernel's forward phase + a commit to an mbarrier after each phase; 22 also
        // waits for that commit (phase fully serialised: execution + commit latency)
#pragma unroll 1
        for (int r = 0; r < reps; ++r) {
#pragma unroll
          for (int k = 0; k < 8; ++k) mma_ts(d0, d0 + 128 + 8u * k, bd[k], idesc, k > 0);
          mma_ts(d0, d0 + 192, bx, idesc, 1u);
          commit(&bar2);
          if (variant == 22) {
            mbar_wait(&bar2, (uint32_t)(r & 1));
            fence_after();
          }
        }
        n = reps * 9;
      } else if (variant == 20) {  // two slots' phases alternating (D at 0 / 256, A at 128 / 384)
#pragma unroll 1
        for (int r = 0; r < reps; ++r) {
          const uint32_t dd = d0 + (uint32_t)(r & 1) * 256u;
#pragma unroll
          for (int k = 0; k < 8; ++k) mma_ts(dd, dd + 128 + 8u * k, bd[k], idesc, k > 0);
        }
        n = reps * 8;
      } else {
#pragma unroll 1
        for (int r = 0; r < reps; ++r) {
#pragma unroll
          for (int k = 0; k < 8; ++k) mma_ts(d0, av + 8u * k, bd[k], idesc, k > 0);
        }
        n = reps * 8;
      }
    }
    for (int r = 0; r < (variant >= 13 ? 0 : reps); ++r) {
      const uint32_t d = (variant == 2 && (r & 1)) ? tb + 128 : d0;  // (variants 9, 11 use d + 64 / d + 128 too)
      for (int k = 0; k < 8; ++k, ++n) {
        if (variant == 0 || variant == 2)
          mma_ts(d, av + 8u * k, sdesc_sw128(sB + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), kIdescFwd<F16>, k > 0);
        else if (variant == 1)
          mma_ts(d, av + 8u * k, sdesc_sw128(sB + k * 2048, 16384, 1024), kIdescBwd<F16>, k > 0);
        else if (variant == 3) {
          const uint64_t ad = sdesc_sw128(sA + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(sB + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(ad), "l"(bd), "r"(kIdescFwd<F16>), "r"((uint32_t)(k > 0))
              : "memory");
        } else if (variant == 4) {
          mma_ts(d, av + 8u * k, sdesc_sw128(sB + (k >> 2) * 32768 + (k & 3) * 32, 16, 1024),
                 idesc_f16kind(128, 256, false, F16), k > 0);
        } else if (variant == 8 || variant == 9) {  // N = 64 (9: two accumulators, k-step interleaved)
          const uint64_t bd = sdesc_sw128(sB + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024);
          mma_ts(d, av + 8u * k, bd, idesc_f16kind(128, 64, false, F16), k > 0);
          if (variant == 9) {
            mma_ts(d + 64, av + 8u * k, bd, idesc_f16kind(128, 64, false, F16), k > 0);
            ++n;
          }
        } else if (variant == 10) {  // N = 16
          mma_ts(d, av + 8u * k, sdesc_sw128(sB + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024),
                 idesc_f16kind(128, 16, false, F16), k > 0);
        } else if (variant == 11) {  // N = 128, two accumulators (two tiles), k-step interleaved
          const uint64_t bd = sdesc_sw128(sB + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
          mma_ts(d, av + 8u * k, bd, kIdescFwd<F16>, k > 0);
          mma_ts(d + 128, av + 64 + 8u * k, bd, kIdescFwd<F16>, k > 0);
          ++n;
        } else {  // 12: N = 128 K-major, A in TMEM, K = 32 per step pair issued as one phase of 9 incl. a no-swizzle step
          mma_ts(d, av + 8u * k, sdesc_sw128(sB + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), kIdescFwd<F16>, k > 0);
          if (k == 7) {
            mma_ts(d, av, sdesc_nosw(sA, 2048, 128), kIdescFwd<F16>, 1u);
            ++n;
          }
        }
      }
    }
    commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    stop = 1;
    if (blockIdx.x == 0) {
      D[0] = (float)(t1 - t0);
      D[1] = (float)n;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tb, 512);
}
// Does a UMMA issue stream (blocked on the MMA queue) slow down other warps of its SM
// sub-partition?  Warp 0 streams UMMAs (variant 26) or idles (27); warps 4 (same
// sub-partition as warp 0) and 5 (another one) each run a fixed ALU loop.
// D[0] = warp-4 cycles, D[1] = warp-5 cycles, D[2] = UMMA-stream cycles.
template <bool F16>
__global__ void __launch_bounds__(256, 1) k_smsp_probe(int variant, int reps, float *D) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sb = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tb;
  __shared__ uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (64 * 1024) / 16; i += 256) reinterpret_cast<uint4 *>(sb)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) {
    tmem_alloc(&tb, 512);
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
  if (warp == 0 && variant == 26) {
    const uint32_t sB = smem_u32(sb);
    uint64_t bd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) bd[k] = sdesc_sw128(sB + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
    const long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < reps * 4; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_ts_elect(tb, tb + 256 + 8u * k, bd[k], kIdescFwd<F16>, k > 0);
    }
    commit_elect(&bar);
    mbar_wait(&bar, 0);
    if (lane_id() == 0) D[2] = (float)(clock64() - t0);
  } else if (warp == 4 || warp == 5) {
    uint32_t x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (uint32_t)(tid * 8 + i);
    const long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < 4000; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = prmt(x[i], x[(i + 1) & 7], 0x5140u) ^ (x[i] >> 3);
    }
    const long long t1 = clock64();
    uint32_t acc = 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= x[i];
    if (acc == 0x9e3779b9u) D[3] = 1.f;
    if ((tid & 31) == 0) D[warp - 4] = (float)(t1 - t0);
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tb, 512);
}
// 2-CTA (cta_group::2) probe: M = 256 pairs over a CTA pair.  variant 5: TS N = 128;
// 6: SS N = 128; 7: TS N = 256.
template <bool F16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_mma_probe2(int variant, int reps, float *D) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sb = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  uint32_t crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  for (int i = tid; i < (96 * 1024) / 16; i += 128) reinterpret_cast<uint4 *>(sb)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  fence_after();
  const int N = variant == 7 ? 256 : 128;
  const uint32_t idesc = (1u << 4) | ((F16 ? 0u : 1u) << 7) | ((F16 ? 0u : 1u) << 10) | ((uint32_t)(N >> 3) << 17) |
                         ((uint32_t)(256 >> 4) << 24);
  if (crank == 0 && tid == 0) {
    const uint32_t sB = smem_u32(sb), sA = sB + 65536;
    const uint32_t d = tb, av = tb + 256;
    long long t0 = clock64();
    int n = 0;
    for (int r = 0; r < reps; ++r) {
      for (int k = 0; k < 8; ++k, ++n) {
        const uint64_t bd = sdesc_sw128(sB + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
        const uint32_t acc = k > 0;
        if (variant == 6) {
          const uint64_t ad = sdesc_sw128(sA + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
              : "memory");
        } else {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
              "r"(av + 8u * k), "l"(bd), "r"(idesc), "r"(acc)
              : "memory");
        }
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((unsigned short)3)
        : "memory");
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    D[0] = (float)(t1 - t0);
    D[1] = (float)n;
  } else if (tid == 0) {
    mbar_wait(&bar, 0);
  }
  fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512) : "memory");
}
}  // namespace

static cudaError_t launch_probe(int mode, float *D, cudaStream_t s) {
  if (mode >= 26 && mode <= 31) {  // 2-CTA probe: mode = 16 + 2 * variant + f16, variant 5..7
    const int variant = (mode - 16) >> 1;
    const bool f16 = (mode & 1) != 0;
    const int smem = 96 * 1024 + 1024;
    auto k = f16 ? k_mma_probe2<true> : k_mma_probe2<false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k<<<2, 128, smem, s>>>(variant, 200, D);
    return cudaGetLastError();
  }
  if (mode >= 16 + 2 * 26 && mode < 16 + 2 * 28) {  // sub-partition interference probe (variants 26, 27)
    const int variant = (mode - 16) >> 1;
    const bool f16 = (mode & 1) != 0;
    const int smem = 64 * 1024 + 1024;
    auto k = f16 ? k_smsp_probe<true> : k_smsp_probe<false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k<<<1, 256, smem, s>>>(variant, 200, D);
    return cudaGetLastError();
  }
  if (mode >= 16) {  // UMMA throughput probe: mode = 16 + 2 * variant + f16 (variants 0..4, 8..12)
    const int variant = (mode - 16) >> 1;
    const bool f16 = (mode & 1) != 0;
    const int smem = 96 * 1024 + 1024;
    auto k = f16 ? k_mma_probe<true> : k_mma_probe<false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k<<<variant == 15 ? 148 : 1, 128, smem, s>>>(variant, 200, D);
    return cudaGetLastError();
  }
  return cudaErrorInvalidValue;
}



}  // namespace gcdf

// mode = 16 + 2 * variant + f16 (see tools/mma_probe.py); D device fp32 >= 4 floats
extern "C" int probe_umma(int mode, float *D) {
  cudaError_t e = gcdf::launch_probe(mode, D, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return (int)e;
}
