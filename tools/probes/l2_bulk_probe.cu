// Dev probe: aggregate L2 -> SMEM bandwidth of 1-D cp.async.bulk copies when every SM
// streams 64 KB blocks out of a small (L2-resident) weight image, as a weight-streaming
// kernel would.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2p l2_bulk_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) k_probe(const uint8_t *src, int n_layers, int iters, int chunk, long long *out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const long long t0 = clock64();
  if (tid == 0) {
    uint32_t ph[2] = {0u, 0u};
    for (int it = 0; it < iters + 2; ++it) {
      const int b = it & 1;
      if (it >= 2) {  // wait for the copy issued two iterations ago into this buffer
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                       : "=r"(ok) : "r"(su32(&bar[b])), "r"(ph[b]) : "memory");
        ph[b] ^= 1u;
      }
      if (it < iters) {
        const uint8_t *s = src + (size_t)((blockIdx.x + it) % n_layers) * 65536;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])), "r"(65536) : "memory");
        for (int c = 0; c < 65536; c += chunk)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(sm + b * 65536 + c)), "l"(s + c), "r"(chunk), "r"(su32(&bar[b])) : "memory");
      }
    }
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int n_layers = 5, iters = 2000;
  uint8_t *src;
  long long *out;
  cudaMalloc(&src, (size_t)n_layers * 65536);
  cudaMemset(src, 1, (size_t)n_layers * 65536);
  cudaMalloc(&out, nsm * sizeof(long long));
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536);
  for (int chunk : {16384, 32768, 65536}) {
    for (int grid : {1, nsm / 4, nsm}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      k_probe<<<grid, 128, 2 * 65536>>>(src, n_layers, 50, chunk, out);
      cudaEventRecord(e0);
      k_probe<<<grid, 128, 2 * 65536>>>(src, n_layers, iters, chunk, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)grid * iters * 65536;
      printf("chunk %6d grid %3d: %.3f ms  %.2f TB/s aggregate  %.1f GB/s per SM  (%s)\n", chunk, grid, ms,
             bytes / ms / 1e9, bytes / ms / 1e6 / grid, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
