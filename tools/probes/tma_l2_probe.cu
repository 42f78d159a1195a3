// Per-SM TMA ingest from L2: each CTA streams a window of an L2-resident
// buffer into shared memory with cp.async.bulk (no compute) through `stages`
// mbarrier-tracked buffers of `chunk` bytes; reports aggregate and per-CTA
// GB/s for several grid sizes.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_l2_probe tma_l2_probe.cu
//   ./tma_l2_probe [window_mb=48] [chunk_kb=32] [stages=6]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
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

// Same stream as 2-D tensor TMA boxes of 128 rows x 64 bf16 (16 KB, 128-byte
// swizzle) over a [rows, 4096] bf16 view of the window: `boxes` per stage, all
// issued by the issuing thread (or rotated over `lanes` lanes of warp 0).
__global__ void __launch_bounds__(128) probe2d(const __grid_constant__ CUtensorMap tm, int rows, size_t per_cta,
                                               int boxes, int stages, int lanes, unsigned long long* sink) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = boxes * 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const size_t n = per_cta / stage_bytes;
  int r0 = (blockIdx.x * 7919 * 128) % rows, c0 = 0;
  uint32_t phase_bits = 0;
  int req = 0;
  unsigned long long acc = 0;
  for (size_t i = 0; i < n + stages; ++i) {
    const int s = static_cast<int>(i % stages);
    if (i >= (size_t)stages) {
      const uint32_t par = (phase_bits >> s) & 1u;
      uint32_t ok = 0;
      if (lane == 0)
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok)
                       : "r"(su32(&bar[s])), "r"(par)
                       : "memory");
      __syncwarp();
      phase_bits ^= 1u << s;
      acc += *reinterpret_cast<volatile int*>(smem + (size_t)s * stage_bytes);
    }
    if (i < n) {
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(stage_bytes)
                     : "memory");
      __syncwarp();
      for (int b = 0; b < boxes; ++b, ++req) {
        if (lane == req % lanes)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                  su32(smem + (size_t)s * stage_bytes + b * 16384)),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&bar[s])), "r"(c0), "r"(r0)
              : "memory");
        c0 += 64;
        if (c0 >= 4096) {
          c0 = 0;
          r0 += 128;
          if (r0 + 128 > rows) r0 = 0;
        }
      }
    }
  }
  if (lane == 0) sink[blockIdx.x] = acc;
}

// FFN-shaped stage: one 1-D bulk copy of `wbytes` (the packed weight tiles)
// plus the token rows either as one 3-D box {64, 128 rows, 2 chunks} (mode 0)
// or as one more 1-D bulk of the same 32 KB (mode 1).  Issued by one thread.
__global__ void __launch_bounds__(128) probe_mix(const __grid_constant__ CUtensorMap tm3, const char* buf,
                                                 size_t window, int rows, size_t per_cta, int stages, int mode,
                                                 unsigned long long* sink) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int half = 32768, stage_bytes = 2 * half;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t n = per_cta / stage_bytes;
  size_t off = ((size_t)blockIdx.x * 7919 * half) % (window / 2);
  int r0 = (blockIdx.x * 7919 * 128) % rows, c0 = 0;
  uint32_t phase_bits = 0;
  unsigned long long acc = 0;
  for (size_t i = 0; i < n + stages; ++i) {
    const int s = static_cast<int>(i % stages);
    if (i >= (size_t)stages) {
      const uint32_t par = (phase_bits >> s) & 1u;
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok)
                     : "r"(su32(&bar[s])), "r"(par)
                     : "memory");
      phase_bits ^= 1u << s;
      acc += *reinterpret_cast<volatile int*>(smem + (size_t)s * stage_bytes);
    }
    if (i < n) {
      char* dst = smem + (size_t)s * stage_bytes;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(stage_bytes)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(dst)),
                   "l"(buf + window / 2 + off), "r"(half), "r"(su32(&bar[s]))
                   : "memory");
      off += half;
      if (off + half > window / 2) off = 0;
      if (mode == 0) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
                su32(dst + half)),
            "l"(reinterpret_cast<uint64_t>(&tm3)), "r"(su32(&bar[s])), "r"(0), "r"(r0), "r"(c0)
            : "memory");
      } else {
        const size_t toff = ((size_t)r0 * 8192 + (size_t)c0 * 128) % (window / 2 - half);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(dst + half)),
                     "l"(buf + toff), "r"(half), "r"(su32(&bar[s]))
                     : "memory");
      }
      c0 += 2;
      if (c0 >= 64) {
        c0 = 0;
        r0 += 128;
        if (r0 + 128 > rows) r0 = 0;
      }
    }
  }
  sink[blockIdx.x] = acc;
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 'm') {  // mixed mode: m <window_mb> <stages> <mode 0 = 3-D box, 1 = bulk>
    const size_t window = (size_t)(argc > 2 ? atoi(argv[2]) : 48) << 20;
    const int stages = argc > 3 ? atoi(argv[3]) : 3, mode = argc > 4 ? atoi(argv[4]) : 0;
    const int rows = (int)(window / 2 / 8192);
    char* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, window);
    cudaMemset(buf, 1, window);
    cudaMalloc(&sink, 4096 * 8);
    CUtensorMap tm;
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, 64};
    cuuint64_t strides[2] = {8192, 128};
    cuuint32_t box[3] = {64, 128, 2};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)r);
      return 1;
    }
    const size_t smem = 1024 + (size_t)stages * 65536 + stages * 8;
    cudaFuncSetAttribute(probe_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("FFN-shaped stages: %d x (32 KB bulk + 32 KB %s)\n", stages, mode ? "bulk" : "3-D box {64,128,2}");
    for (int ctas : {1, 32, 148}) {
      const size_t per_cta = (size_t)64 << 20;
      probe_mix<<<ctas, 128, smem>>>(tm, buf, window, rows, per_cta / 8, stages, mode, sink);
      cudaEventRecord(a);
      probe_mix<<<ctas, 128, smem>>>(tm, buf, window, rows, per_cta, stages, mode, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double gbs = (double)per_cta * ctas / (ms * 1e-3) / 1e9;
      printf("ctas %3d: %8.1f GB/s aggregate, %6.1f GB/s per CTA  err=%s\n", ctas, gbs, gbs / ctas,
             cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
  }
  if (argc > 1 && argv[1][0] == 't') {  // tensor mode: t <window_mb> <boxes/stage> <stages> <lanes>
    const size_t window = (size_t)(argc > 2 ? atoi(argv[2]) : 48) << 20;
    const int boxes = argc > 3 ? atoi(argv[3]) : 2, stages = argc > 4 ? atoi(argv[4]) : 4,
              lanes = argc > 5 ? atoi(argv[5]) : 1;
    const int rows = (int)(window / 8192);
    char* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, window);
    cudaMemset(buf, 1, window);
    cudaMalloc(&sink, 4096 * 8);
    CUtensorMap tm;
    cuuint64_t dims[2] = {4096, (cuuint64_t)rows};
    cuuint64_t strides[1] = {8192};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)r);
      return 1;
    }
    const size_t smem = 1024 + (size_t)stages * boxes * 16384 + stages * 8;
    cudaFuncSetAttribute(probe2d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("tensor TMA: window %zu MB, %d x 16 KB boxes per stage, %d stages, %d issuing lanes\n", window >> 20,
           boxes, stages, lanes);
    for (int ctas : {1, 32, 148}) {
      const size_t per_cta = (size_t)64 << 20;
      probe2d<<<ctas, 128, smem>>>(tm, rows, per_cta / 8, boxes, stages, lanes, sink);
      cudaEventRecord(a);
      probe2d<<<ctas, 128, smem>>>(tm, rows, per_cta, boxes, stages, lanes, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double gbs = (double)per_cta * ctas / (ms * 1e-3) / 1e9;
      printf("ctas %3d: %8.1f GB/s aggregate, %6.1f GB/s per CTA  err=%s\n", ctas, gbs, gbs / ctas,
             cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
  }
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
