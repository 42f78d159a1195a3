// HBM read ceiling probe: persistent CTAs stream a large buffer into shared
// memory with 1-D bulk TMA (cp.async.bulk) through an mbarrier ring and
// discard it; also a plain 16-byte-load variant.  Prints GB/s per config.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/bin/hbm_tma_read tools/hbm_tma_read.cu
#include <cuda.h>
#include <cudaTypedefs.h>
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

// 2-D tiled TMA (64 cols x 128 rows, 128-byte swizzle) over a row-major bf16
// matrix [rows, cols]: each CTA walks 128-row blocks (round robin) and, inside
// a block, the 64-column chunks in order -- the weight-streaming pattern of
// the expert GEMM.
__global__ void tma2d_read(const __grid_constant__ CUtensorMap tm, int rows, int cols, int stages,
                           unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int chunk = 128 * 64 * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int kc = cols / 64;
  const long nblk = rows / 128;
  const long n = ((nblk - blockIdx.x + gridDim.x - 1) / gridDim.x) * kc;  // my tiles
  auto coord = [&](long i, int& c0, int& c1) {
    const long b = blockIdx.x + (i / kc) * gridDim.x;
    c0 = (int)(i % kc) * 64;
    c1 = (int)(b * 128);
  };
  unsigned long long acc = 0;
  long issued = 0;
  for (; issued < n && issued < stages; ++issued) {
    int c0, c1;
    coord(issued, c0, c1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[issued])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(smem + issued * chunk)), "l"(&tm), "r"(c0), "r"(c1), "r"(su32(&bar[issued])) : "memory");
  }
  int s = 0;
  uint32_t phase = 0;
  for (long i = 0; i < n; ++i) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar[s])), "r"(phase) : "memory");
    acc += smem[(size_t)s * chunk];
    if (issued < n) {
      int c0, c1;
      coord(issued, c0, c1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(smem + (size_t)s * chunk)), "l"(&tm), "r"(c0), "r"(c1), "r"(su32(&bar[s])) : "memory");
      ++issued;
    }
    if (++s == stages) { s = 0; phase ^= 1; }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

// 3-D view {64, rows, cols/64} of the same matrix, box {64, 128, kch}: one TMA
// brings kch consecutive 64-column chunks of 128 rows (kch*128 B per row).
__global__ void tma3d_read(const __grid_constant__ CUtensorMap tm, int rows, int cols, int kch,
                           int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int chunk = 128 * 64 * 2 * kch;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int kc = cols / 64 / kch;
  const long nblk = rows / 128;
  const long n = ((nblk - blockIdx.x + gridDim.x - 1) / gridDim.x) * kc;
  auto coord = [&](long i, int& c2, int& c1) {
    const long b = blockIdx.x + (i / kc) * gridDim.x;
    c2 = (int)(i % kc) * kch;
    c1 = (int)(b * 128);
  };
  unsigned long long acc = 0;
  long issued = 0;
  for (; issued < n && issued < stages; ++issued) {
    int c2, c1;
    coord(issued, c2, c1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[issued])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(su32(smem + issued * chunk)), "l"(&tm), "r"(0), "r"(c1), "r"(c2), "r"(su32(&bar[issued])) : "memory");
  }
  int s = 0;
  uint32_t phase = 0;
  for (long i = 0; i < n; ++i) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar[s])), "r"(phase) : "memory");
    acc += smem[(size_t)s * chunk];
    if (issued < n) {
      int c2, c1;
      coord(issued, c2, c1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(su32(smem + (size_t)s * chunk)), "l"(&tm), "r"(0), "r"(c1), "r"(c2), "r"(su32(&bar[s])) : "memory");
      ++issued;
    }
    if (++s == stages) { s = 0; phase ^= 1; }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

// The fused FFN's weight stream alone: items of GEMM1 tiles (32 m-blocks x 16
// k-chunks, rows of TD*2 = 2 KB) and GEMM2 tiles (8 m-blocks x 64 chunks, rows
// of 8 KB) interleaved with a lag, tiles round-robin over persistent CTAs.
// packed = 1 reads the same tiles from a tile-contiguous copy (each 128 x 64
// chunk = 16 KB contiguous), i.e. the layout a weight prepack would produce.
__global__ void ffn_pattern(const __grid_constant__ CUtensorMap w1, const __grid_constant__ CUtensorMap w2,
                            int n_items, int lag, int packed, int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int chunk = 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int MT1 = 32, MT2 = 8, KC1 = 16, KC2 = 64;
  const int per = MT1 + MT2, L = lag, n = n_items;
  const int total = n * per;
  int stage = 0;
  uint32_t phase = 0;
  long consumed = 0, issued = 0;
  unsigned long long acc = 0;
  // flatten (tile, kc) into a stream; keep `stages` loads in flight
  int t = blockIdx.x, kc = 0;
  auto next_load = [&](int& gemm, int& c0, int& c1) -> bool {
    if (t >= total) return false;
    int item, g, m;
    const int head = L * MT1, body = head + (n - L) * per;
    if (t < head) { item = t / MT1; g = 0; m = t % MT1; }
    else if (t < body) { const int u = t - head, gg = L + u / per, r = u % per;
      if (r < MT1) { item = gg; g = 0; m = r; } else { item = gg - L; g = 1; m = r - MT1; } }
    else { const int u = t - body; item = n - L + u / MT2; g = 1; m = u % MT2; }
    const int KC = g ? KC2 : KC1, MT = g ? MT2 : MT1;
    gemm = g;
    if (packed) { c0 = 0; c1 = ((item * MT + m) * KC + kc) * 128; }
    else { c0 = kc * 64; c1 = (item * MT + m) * 128; }
    if (++kc == KC) { kc = 0; t += gridDim.x; }
    return true;
  };
  auto issue = [&](int s) -> bool {
    int g, c0, c1;
    if (!next_load(g, c0, c1)) return false;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(smem + (size_t)s * chunk)), "l"(g ? &w2 : &w1), "r"(c0), "r"(c1), "r"(su32(&bar[s])) : "memory");
    return true;
  };
  for (int s = 0; s < stages; ++s) if (issue(s)) ++issued;
  while (consumed < issued) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar[stage])), "r"(phase) : "memory");
    acc += smem[(size_t)stage * chunk];
    ++consumed;
    if (issue(stage)) ++issued;
    if (++stage == stages) { stage = 0; phase ^= 1; }
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
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaFuncSetAttribute(tma2d_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int cols : {1024, 4096}) {
      const long rows = (long)(bytes / 2 / cols);
      CUtensorMap tm;
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
      cuuint32_t box[2] = {64, 128};
      cuuint32_t estr[2] = {1, 1};
      for (int promo : {0, 2, 3}) {
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        for (int stages : {6, 12}) {
          const size_t smem = 1024 + (size_t)stages * 16384 + 64 * 8;
          double gbs = timeit([&] { tma2d_read<<<sms, 32, smem>>>(tm, (int)rows, cols, stages, sink); });
          cudaError_t e = cudaGetLastError();
          printf("tma2d box 64x128 sw128 row=%5d B promo=%d stages=%2d : %7.0f GB/s %s\n", cols * 2, promo, stages, gbs,
                 e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
      }
    }
  }
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaFuncSetAttribute(tma3d_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int cols : {1024, 4096}) {
      const long rows = (long)(bytes / 2 / cols);
      for (int kch : {1, 2, 4}) {
        CUtensorMap tm;
        cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)cols / 64};
        cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
        cuuint32_t box[3] = {64, 128, (cuuint32_t)kch};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode3d failed %d\n", (int)r); continue; }
        for (int inflight_kb : {96, 128, 192}) {
          const int stages = inflight_kb / (16 * kch);
          if (stages < 1) continue;
          const size_t smem = 1024 + (size_t)stages * 16384 * kch + 64 * 8;
          double gbs = timeit([&] { tma3d_read<<<sms, 32, smem>>>(tm, (int)rows, cols, kch, stages, sink); });
          cudaError_t e = cudaGetLastError();
          printf("tma3d box 64x128x%d row=%5d B stages=%2d inflight=%3d KB : %7.0f GB/s %s\n", kch, cols * 2, stages,
                 stages * 16 * kch, gbs, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
      }
    }
  }
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaFuncSetAttribute(ffn_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    const int E = 512, TD = 1024, HD = 4096;
    const size_t wbytes = (size_t)E * TD * HD * 2;  // 4 GiB each
    uint8_t* W1 = buf;
    uint8_t* W2 = buf + wbytes;
    auto mk = [&](CUtensorMap* tm, void* p, cuuint64_t cols, cuuint64_t rows) {
      cuuint64_t dims[2] = {cols, rows};
      cuuint64_t strides[1] = {cols * 2};
      cuuint32_t box[2] = {64, 128};
      cuuint32_t estr[2] = {1, 1};
      return enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUtensorMap r1, r2, p1, p2;
    mk(&r1, W1, TD, (cuuint64_t)E * HD);
    mk(&r2, W2, HD, (cuuint64_t)E * TD);
    mk(&p1, W1, 64, (cuuint64_t)E * HD * TD / 64);
    mk(&p2, W2, 64, (cuuint64_t)E * TD * HD / 64);
    for (int packed : {0, 1}) {
      for (int stages : {6, 8, 12}) {
        const size_t smem = 1024 + (size_t)stages * 16384 + 64 * 8;
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
          cudaEventRecord(a);
          ffn_pattern<<<sms, 32, smem>>>(packed ? p1 : r1, packed ? p2 : r2, E, 30, packed, stages, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (r > 0 && ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("ffn weight stream packed=%d stages=%2d : %.3f ms  %7.0f GB/s %s\n", packed, stages, best,
               2.0 * wbytes / (best * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  }
  double gcopy = timeit([&] { cudaMemcpyAsync(buf + bytes / 2, buf, bytes / 2, cudaMemcpyDeviceToDevice); });
  printf("cudaMemcpy D2D (r+w counted as 2x half)          : %7.0f GB/s\n", gcopy);
  return 0;
}
