// k_selftest.cu -- one UMMA building block for the unit tests (gcdf_selftest_umma): the
// tcgen05 instruction / shared-memory descriptors and TMEM layouts the product kernels use
// (K-major B of the forward GEMMs, MN-major B of the backward GEMMs, N = 16 of the last
// GEMM), checked in isolation against a plain matmul of the 16-bit-rounded operands
// (tests/test_gpu_tensor.py::test_selftest_umma).  Not on the hot path.
#include "gcdf_internal.h"
#include "tc_ptx.h"

namespace gcdf {
namespace {

using namespace tc;

template <bool F16> constexpr uint32_t kIdescFwd = idesc_f16kind(128, 128, false, F16);
template <bool F16> constexpr uint32_t kIdescBwd = idesc_f16kind(128, 128, true, F16);
template <bool F16> constexpr uint32_t kIdescFin = idesc_f16kind(128, 16, false, F16);

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
cudaError_t selftest_t(int mode, const float *A, const float *B, float *D, cudaStream_t s) {
  const int smem = 32768 + 1024;
  cudaError_t e = cudaFuncSetAttribute(k_selftest_umma<F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k_selftest_umma<F16><<<1, 128, smem, s>>>(A, B, mode, D);
  return cudaGetLastError();
}

}  // namespace

// mode bits 0-1: 0 = K-major B (N = 128), 1 = MN-major B (N = 128), 2 = N = 16; bit 2: fp16
cudaError_t launch_selftest_umma(int mode, const float *A, const float *B, float *D, cudaStream_t s) {
  if (mode < 0 || mode > 6 || (mode & 3) > 2) return cudaErrorInvalidValue;
  return (mode & 4) ? selftest_t<true>(mode & 3, A, B, D, s) : selftest_t<false>(mode & 3, A, B, D, s);
}

}  // namespace gcdf
