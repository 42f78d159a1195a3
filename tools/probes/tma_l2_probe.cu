// Per-SM TMA ingest from L2: each CTA streams a window of an L2-resident
// buffer into shared memory with cp.async.bulk (no compute) through `stages`
// mbarrier-tracked buffers of `chunk` bytes; reports aggregate and per-CTA
// GB/s for several grid sizes.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_l2_probe tma_l2_probe.cu
//   ./tma_l2_probe [window_mb=48] [chunk_kb=32] [stages=6]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(128) probe(const char* buf, size_t window, size_t per_cta, int chunk, int stages,
                                             unsigned long long* sink, int issuers, int lanes, int spin) {
  extern __shared__ __align__(1024) char smem_all[];
  // issuer w (warp w / lanes, lane w % lanes) owns stages [w*stages, (w+1)*stages)
  const int lane = threadIdx.x & 31;
  const int w = (threadIdx.x >> 5) * lanes + lane;
  const bool is_issuer = lane < lanes && w < issuers;
  char* smem = smem_all + (size_t)w * stages * chunk;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_all + (size_t)issuers * stages * chunk) + w * stages;
  if (is_issuer) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (!is_issuer) return;
  const size_t n = per_cta / issuers / chunk;
  size_t off = ((size_t)(blockIdx.x * 4 + w) * 7919 * chunk) % window;
  uint32_t phase_bits = 0;
  unsigned long long acc = 0;
  for (size_t i = 0; i < n + stages; ++i) {
    const int s = static_cast<int>(i % stages);
    if (i >= (size_t)stages) {  // consume stage s (issued `stages` iterations ago)
      const uint32_t par = (phase_bits >> s) & 1u;
      uint32_t ok = 0;
      if (spin)
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok)
                       : "r"(su32(&bar[s])), "r"(par)
                       : "memory");
      else
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok)
                       : "r"(su32(&bar[s])), "r"(par)
                       : "memory");
      phase_bits ^= 1u << s;
      acc += *reinterpret_cast<volatile int*>(smem + (size_t)s * chunk);
    }
    if (i < n) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(chunk)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              su32(smem + (size_t)s * chunk)),
          "l"(buf + off), "r"(chunk), "r"(su32(&bar[s]))
          : "memory");
      off += chunk;
      if (off + chunk > window) off = 0;
    }
  }
  sink[blockIdx.x * 8 + w] = acc;
}

int main(int argc, char** argv) {
  const size_t window = (size_t)(argc > 1 ? atoi(argv[1]) : 48) << 20;
  const int chunk = (argc > 2 ? atoi(argv[2]) : 32) << 10;
  const int stages = argc > 3 ? atoi(argv[3]) : 6;
  const int issuers = argc > 4 ? atoi(argv[4]) : 1;
  const int lanes = argc > 5 ? atoi(argv[5]) : 1;  // issuers per warp
  const int spin = argc > 6 ? atoi(argv[6]) : 0;   // 1: mbarrier.test_wait spin instead of try_wait
  const size_t smem = (size_t)issuers * stages * chunk + issuers * stages * 8;
  char* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, window);
  cudaMemset(buf, 1, window);
  cudaMalloc(&sink, 8 * 4096 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("window %zu MB, chunk %d KB, stages %d x %d issuers (%d per warp; %zu KB in flight per CTA), %s\n",
         window >> 20, chunk >> 10, stages, issuers, lanes, (size_t)issuers * stages * chunk >> 10,
         spin ? "test_wait spin" : "try_wait");
  for (int ctas : {1, 8, 32, 74, 148}) {
    const size_t per_cta = (size_t)64 << 20;  // 64 MB per CTA
    probe<<<ctas, 128, smem>>>(buf, window, per_cta / 8, chunk, stages, sink, issuers, lanes, spin);  // warm
    cudaEventRecord(a);
    probe<<<ctas, 128, smem>>>(buf, window, per_cta, chunk, stages, sink, issuers, lanes, spin);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double gbs = (double)per_cta * ctas / (ms * 1e-3) / 1e9;
    printf("ctas %3d: %8.1f GB/s aggregate, %6.1f GB/s per CTA (%.3f ms)  err=%s\n", ctas, gbs, gbs / ctas, ms,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
