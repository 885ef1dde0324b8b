// Microbenchmark: the scan kernel's memory pipeline alone.  Each CTA streams
// a contiguous range of an 800 MB buffer through `stages` shared-memory tiles
// with cp.async.bulk + mbarrier (one elected issuing thread), every thread
// touches one word per 32 of each tile, then the CTA syncs and reuses the
// stage — the same structure as scan_topk_kernel minus the scoring.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          (uint32_t)__cvta_generic_to_shared(b)),
      "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(b))
               : "memory");
}

__global__ void stream_kernel(const uint8_t* src, uint64_t total, uint32_t tile, uint32_t stages,
                              uint32_t chunks, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar[8];
  const uint64_t per = (total / gridDim.x) & ~static_cast<uint64_t>(1023);
  const uint8_t* base = src + per * blockIdx.x;
  const uint32_t ntiles = per / tile;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < stages; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint32_t cb = tile / chunks;
  auto issue = [&](uint32_t t) {
    uint64_t* b = &bar[t % stages];
    mbar_expect_tx(b, tile);
    for (uint32_t c = 0; c < chunks; ++c)
      bulk_g2s(smem + (size_t)(t % stages) * tile + c * cb, base + (uint64_t)t * tile + c * cb, cb, b);
  };
  if (threadIdx.x == 0)
    for (uint32_t t = 0; t < min(ntiles, stages - 1); ++t) issue(t);
  uint32_t acc = 0;
  for (uint32_t t = 0; t < ntiles; ++t) {
    if (threadIdx.x == 0 && t + stages - 1 < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;");
      issue(t + stages - 1);
    }
    mbar_wait(&bar[t % stages], (t / stages) & 1u);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(smem + (size_t)(t % stages) * tile);
    for (uint32_t i = threadIdx.x * 32; i < tile / 4; i += blockDim.x * 32) acc += w[i];
    __syncthreads();
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main(int argc, char** argv) {
  const uint64_t total = 800ull << 20;
  uint8_t* d;
  uint32_t* sink;
  cudaMalloc(&d, total);
  cudaMalloc(&sink, 4);
  cudaMemset(d, 1, total);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t tiles[] = {16384, 32768, 40960, 65536, 81920};
  const uint32_t stagess[] = {2, 3, 4, 6};
  const uint32_t chunkss[] = {1, 4, 16};
  const int per_sm[] = {1, 2};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (uint32_t tile : tiles)
    for (uint32_t st : stagess)
      for (uint32_t ch : chunkss)
        for (int ps : per_sm) {
          const size_t sm = (size_t)tile * st;
          if (sm * ps > 220 * 1024) continue;
          cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
          const int grid = sms * ps;
          float best = 1e9f;
          for (int it = 0; it < 6; ++it) {
            cudaEventRecord(e0);
            stream_kernel<<<grid, 512, sm>>>(d, total, tile, st, ch, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it && ms < best) best = ms;
          }
          const cudaError_t err = cudaGetLastError();
          printf("tile %6u stages %u chunks %2u ctas/sm %d: %7.1f us  %7.1f GB/s %s\n", tile, st, ch, ps,
                 best * 1e3, (double)((total / grid) & ~1023ull) * grid / (best * 1e-3) / 1e9,
                 err ? cudaGetErrorString(err) : "");
        }
  return 0;
}
