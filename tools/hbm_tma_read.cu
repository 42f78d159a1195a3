// HBM read ceiling probe: persistent CTAs stream a large buffer into shared
// memory with 1-D bulk TMA (cp.async.bulk) through an mbarrier ring and
// discard it; also a plain 16-byte-load variant.  Prints GB/s per config.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/bin/hbm_tma_read tools/hbm_tma_read.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void tma_read(const uint8_t* src, size_t bytes, int chunk, int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t n = bytes / chunk;
  uint32_t phase = 0;
  int s = 0;
  size_t issued = 0;
  unsigned long long acc = 0;
  size_t i = blockIdx.x;
  // prologue
  for (int p = 0; p < stages && i + (size_t)p * gridDim.x < n; ++p) {
    const size_t c = i + (size_t)p * gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[p])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(smem + (size_t)p * chunk)), "l"(src + c * chunk), "r"(chunk), "r"(su32(&bar[p])) : "memory");
    ++issued;
  }
  for (size_t c = i; c < n; c += gridDim.x) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar[s])), "r"(phase) : "memory");
    acc += smem[(size_t)s * chunk];
    const size_t nc = c + (size_t)stages * gridDim.x;
    if (nc < n) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(smem + (size_t)s * chunk)), "l"(src + nc * chunk), "r"(chunk), "r"(su32(&bar[s])) : "memory");
    }
    if (++s == stages) { s = 0; phase ^= 1; }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

__global__ void ldg_read(const uint4* src, size_t n16, unsigned long long* sink) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride), d = __ldcs(src + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n16; i += stride) acc ^= __ldcs(src + i).x;
  if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
  const size_t bytes = 8ull << 30;
  uint8_t* buf;
  unsigned long long* sink;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto fn) {
    fn();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 8; ++r) {
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    return bytes / (best * 1e-3) / 1e9;
  };
  cudaFuncSetAttribute(tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const int chunks[] = {8192, 16384, 32768};
  for (int per_sm : {1, 2}) {
    for (int chunk : chunks) {
      for (int inflight_kb : {64, 128, 192}) {
        const int smem_budget = inflight_kb * 1024 / per_sm;
        const int stages = smem_budget / chunk;
        if (stages < 2) continue;
        const size_t smem = (size_t)stages * chunk + 64 * 8;
        if (smem > 220 * 1024) continue;
        double gbs = timeit([&] { tma_read<<<sms * per_sm, 32, smem>>>(buf, bytes, chunk, stages, sink); });
        cudaError_t e = cudaGetLastError();
        printf("tma  ctas/sm=%d chunk=%5d stages=%2d inflight/sm=%3d KB : %7.0f GB/s %s\n", per_sm, chunk, stages,
               stages * chunk * per_sm / 1024, gbs, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  }
  for (int bpsm : {4, 8, 16}) {
    double gbs = timeit([&] { ldg_read<<<sms * bpsm, 256>>>(reinterpret_cast<const uint4*>(buf), bytes / 16, sink); });
    printf("ldg  blocks/sm=%2d x256 thr, 4x16B in flight/thr : %7.0f GB/s\n", bpsm, gbs);
  }
  double gcopy = timeit([&] { cudaMemcpyAsync(buf + bytes / 2, buf, bytes / 2, cudaMemcpyDeviceToDevice); });
  printf("cudaMemcpy D2D (r+w counted as 2x half)          : %7.0f GB/s\n", gcopy);
  return 0;
}
