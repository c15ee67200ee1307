// tc_ptx.h -- inline-PTX wrappers for sm_100a: mbarrier, tcgen05 (TMEM alloc, MMA,
// commit, ld/st, fences) and UMMA shared-memory / instruction descriptors.
// Bit layouts follow the PTX ISA for tcgen05 (cross-checked against the CUTLASS headers
// vendored in this image: cute/arch/mma_sm100_desc.hpp, cute/atom/mma_traits_sm100.hpp).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define DEVI __device__ __forceinline__

namespace gcdf {
namespace tc {

DEVI uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
DEVI uint32_t lane_id() { return threadIdx.x & 31u; }

// ------------------------------------------------------------------ mbarrier
DEVI void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
DEVI void mbar_arrive_addr(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
DEVI void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
DEVI bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t"
      "}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking probe of the phase with the given parity (no suspend).
DEVI bool mbar_test(const uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t"
      "}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a protocol bug traps (the launch fails with an error) instead of hanging
// the GPU; the bound (~2^34 cycles, seconds) is far above any legitimate wait.
DEVI void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(addr, parity)) {
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}
// try_wait with an explicit suspend-time hint (ns)
DEVI bool mbar_try_wait_hint(uint32_t addr, uint32_t parity, uint32_t hint_ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t"
      "}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(hint_ns)
      : "memory");
  return ok != 0;
}
template <uint32_t kHintNs>
DEVI void mbar_wait_hint(uint64_t *bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait_hint(addr, parity, kHintNs)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait_hint(addr, parity, kHintNs)) {
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}
// Spin with a short sleep between probes
template <uint32_t kSleepNs>
DEVI void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
  if (mbar_test(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_test(bar, parity)) {
    if (kSleepNs) __nanosleep(kSleepNs);
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}
// Spin variant (test_wait, never suspends): lower wake-up latency for a single polling thread.
DEVI void mbar_wait_spin(uint64_t *bar, uint32_t parity) {
  if (mbar_test(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_test(bar, parity)) {
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}
// expect-tx arrive (one arrival + tx bytes) and a 1-D bulk copy global -> shared that
// completes its bytes on the mbarrier (cp.async.bulk, async proxy)
DEVI void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
DEVI void bulk_g2s(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
DEVI void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
DEVI void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
DEVI void named_bar_sync(uint32_t id, uint32_t n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
DEVI void named_bar_arrive(uint32_t id, uint32_t n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// ------------------------------------------------------------------ cp.async (global -> smem, no registers)
// 16-byte copy; src_bytes = 0 zero-fills the destination (out-of-range source)
DEVI void cp_async16(void *dst_smem, const void *src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst_smem)), "l"(src), "r"(src_bytes)
               : "memory");
}
DEVI void cp_async4(void *dst_smem, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
DEVI void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
DEVI void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ------------------------------------------------------------------ TMEM
DEVI void tmem_alloc(uint32_t *dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
}
DEVI void tmem_relinquish() { asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory"); }
DEVI void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
DEVI void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DEVI void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
DEVI void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
DEVI void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
DEVI void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem desc]; kind::f16 (bf16 in, fp32 accumulate), cta_group::1
DEVI void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t"
      "}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}

// Warp-converged variants: the whole warp executes them with warp-uniform operands and one
// elected lane (elect.sync: the lowest active lane) issues, so the operands can live in
// uniform registers.  commit_elect must be executed by the same warp as the MMAs it tracks.
DEVI void mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t"
      ".reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t"
      "}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}
// SS form (A and B from shared-memory descriptors), warp-converged like mma_ts_elect
DEVI void mma_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t"
      ".reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
// Four UMMAs over one 64-column SWIZZLE_128B K chunk from ONE asm block (a lean issue stream:
// the per-UMMA operands are adds of immediates): A at a + 8 i (TMEM columns), B descriptor
// + 2 i (32 B apart inside the 128-B swizzle atom), the first accumulating iff acc != 0.
DEVI void umma4_sw128_elect(uint32_t d, uint32_t a, uint64_t b0, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred e, p0, pt;\n\t"
      ".reg .b32 ra;\n\t"
      ".reg .b64 rb;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p0, %4, 0;\n\t"
      "setp.eq.b32 pt, %4, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p0;\n\t"
      "add.u32 ra, %1, 8;\n\tadd.u64 rb, %2, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, pt;\n\t"
      "add.u32 ra, %1, 16;\n\tadd.u64 rb, %2, 4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, pt;\n\t"
      "add.u32 ra, %1, 24;\n\tadd.u64 rb, %2, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, pt;\n\t"
      "}" ::"r"(d),
      "r"(a), "l"(b0), "r"(idesc), "r"(acc)
      : "memory");
}
// The same four UMMAs for an MN-major SWIZZLE_128B B operand (B descriptor + 128 = 2048 B per
// K step)
DEVI void umma4_mn_elect(uint32_t d, uint32_t a, uint64_t b0, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred e, p0, pt;\n\t"
      ".reg .b32 ra;\n\t"
      ".reg .b64 rb;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p0, %4, 0;\n\t"
      "setp.eq.b32 pt, %4, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p0;\n\t"
      "add.u32 ra, %1, 8;\n\tadd.u64 rb, %2, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, pt;\n\t"
      "add.u32 ra, %1, 16;\n\tadd.u64 rb, %2, 256;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, pt;\n\t"
      "add.u32 ra, %1, 24;\n\tadd.u64 rb, %2, 384;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, pt;\n\t"
      "}" ::"r"(d),
      "r"(a), "l"(b0), "r"(idesc), "r"(acc)
      : "memory");
}
// Eight UMMAs over K = 128 (8 K steps) from ONE asm block, A at a + 8 k (contiguous TMEM
// columns), B a SWIZZLE_128B operand: K-major (two 64-column chunks of 16 KB: + (k / 4) 16384
// + (k % 4) 32 bytes) or MN-major (+ k 2048 bytes); the first accumulating iff acc != 0.
#define GCDF_UMMA8_STEP(AOFF, DOFF)                  \
  "add.u32 ra, %1, " #AOFF ";\n\t"                    \
  "add.u64 rb, %2, " #DOFF ";\n\t"                    \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ra], rb, %3, pt;\n\t"
#define GCDF_UMMA8_HEAD                                                  \
  "{\n\t.reg .pred e, p0, pt;\n\t.reg .b32 ra;\n\t.reg .b64 rb;\n\t" \
  "elect.sync _|e, 0xffffffff;\n\t"                                      \
  "setp.ne.b32 p0, %4, 0;\n\tsetp.eq.b32 pt, %4, %4;\n\t"               \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p0;\n\t"
DEVI void umma8_kmajor_elect(uint32_t d, uint32_t a, uint64_t b0, uint32_t idesc, uint32_t acc) {
  asm volatile(GCDF_UMMA8_HEAD GCDF_UMMA8_STEP(8, 2) GCDF_UMMA8_STEP(16, 4) GCDF_UMMA8_STEP(24, 6)
                   GCDF_UMMA8_STEP(32, 1024) GCDF_UMMA8_STEP(40, 1026) GCDF_UMMA8_STEP(48, 1028)
                       GCDF_UMMA8_STEP(56, 1030) "}" ::"r"(d),
               "r"(a), "l"(b0), "r"(idesc), "r"(acc)
               : "memory");
}
DEVI void umma8_mnmajor_elect(uint32_t d, uint32_t a, uint64_t b0, uint32_t idesc, uint32_t acc) {
  asm volatile(GCDF_UMMA8_HEAD GCDF_UMMA8_STEP(8, 128) GCDF_UMMA8_STEP(16, 256) GCDF_UMMA8_STEP(24, 384)
                   GCDF_UMMA8_STEP(32, 512) GCDF_UMMA8_STEP(40, 640) GCDF_UMMA8_STEP(48, 768)
                       GCDF_UMMA8_STEP(56, 896) "}" ::"r"(d),
               "r"(a), "l"(b0), "r"(idesc), "r"(acc)
               : "memory");
}
#undef GCDF_UMMA8_STEP
#undef GCDF_UMMA8_HEAD
DEVI void commit_elect(uint64_t *bar) {
  asm volatile(
      "{\n\t"
      ".reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
      "}" ::"r"(smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 bit, 32 consecutive columns -> 32 registers per thread
DEVI void ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
DEVI void ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
DEVI void st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
DEVI void st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
DEVI void st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// ------------------------------------------------------------------ conversions
DEVI uint32_t pack_bf16(float lo, float hi) {  // lo -> bits [0,16) (even column), hi -> [16,32)
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
DEVI uint32_t pack_bf16_relu(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

DEVI uint32_t pack_f16(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
DEVI uint32_t pack_f16_relu(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
// operand type of the tensor-core path: bf16 (8-bit significand) or fp16 (11-bit)
template <bool F16>
DEVI uint32_t pack2(float lo, float hi) {
  if constexpr (F16) return pack_f16(lo, hi);
  else return pack_bf16(lo, hi);
}
template <bool F16>
DEVI uint32_t pack2_relu(float lo, float hi) {
  if constexpr (F16) return pack_f16_relu(lo, hi);
  else return pack_bf16_relu(lo, hi);
}

DEVI uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {  // byte permute; selector bit 3 = sign-replicate
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// ReLU masks in "byte-sign" form.  A 32-unit chunk is stored in one word: unit e (group
// k = e / 4, t = e % 4) at bit 8 t + 7 - k.
// Build (forward): from the two packed ReLU'd 16-bit pairs of units 4k..4k+3 -- a
// non-negative 16-bit value v is nonzero iff bit 15 of v + 0x7fff is set (no carry out of
// the low half: |v| <= 0x7f7f) -- gather those bits into bytes 0..3 (prmt), shift by k.
DEVI uint32_t mask_group(uint32_t pk01, uint32_t pk23, int k) {
  const uint32_t v0 = pk01 + 0x7fff7fffu, v1 = pk23 + 0x7fff7fffu;
  const uint32_t x = prmt(v0, v1, 0x7531u);  // bytes: (v0.b1, v0.b3, v1.b1, v1.b3) -> bit 7 of each
  return (x >> k) & (0x80808080u >> k);
}
// Use (backward): 0xffff half-word masks for units (4k, 4k+1) and (4k+2, 4k+3).
DEVI void mask_expand(uint32_t m, int k, uint32_t &lo, uint32_t &hi) {
  const uint32_t y = m << k;
  lo = prmt(y, 0u, 0x9988u);
  hi = prmt(y, 0u, 0xbbaau);
}

// ------------------------------------------------------------------ descriptors
// Shared-memory matrix descriptor (tcgen05): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version 1 [46,48), base offset 0 [49,52), layout SWIZZLE_128B = 2 [61,64).
// SWIZZLE_NONE (layout 0): 8-row x 16-B core matrices; K-major LBO = distance between the
// two K cores of one K = 16 step, SBO = distance between 8-row groups.
DEVI uint64_t sdesc_nosw(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
DEVI uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor, kind::f16: c_format F32 (1) [4,6), a_format BF16 (1) [7,10),
// b_format BF16 (1) [10,13), a_major K (0) bit 15, b_major bit 16, N>>3 [17,23), M>>4 [24,29).
// a_format / b_format: F16 = 0, BF16 = 1.
__host__ __device__ constexpr uint32_t idesc_f16kind(int M, int N, bool b_mn_major, bool f16) {
  return (1u << 4) | ((f16 ? 0u : 1u) << 7) | ((f16 ? 0u : 1u) << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

}  // namespace tc
}  // namespace gcdf
