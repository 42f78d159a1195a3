// Can a 1-D bulk copy land in THIS CTA's shared memory while counting its
// bytes on the OTHER CTA's mbarrier (cluster of 2)?  Rank 1 copies 32 KB into
// its own smem with mbar = rank 0's barrier; rank 0 waits on its barrier, then
// (after a cluster barrier) rank 1 checks the bytes.  Prints OK / MISMATCH.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __cluster_dims__(2, 1, 1) k(const int4* src, int* ok) {
  __shared__ __align__(128) int4 buf[2048];
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank == 0 && threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(32768) : "memory");
    uint32_t okw = 0;
    while (!okw)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(okw) : "r"(su32(&bar)) : "memory");
  }
  if (rank == 1 && threadIdx.x == 0) {
    uint32_t remote_bar;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote_bar) : "r"(su32(&bar)));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(buf)), "l"(src), "r"(32768), "r"(remote_bar) : "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank == 1) {
    for (int i = threadIdx.x; i < 2048; i += blockDim.x)
      if (buf[i].x != src[i].x || buf[i].w != src[i].w) atomicAdd(ok, 1);
  }
}

int main() {
  int4* src; int* bad;
  cudaMalloc(&src, 32768); cudaMalloc(&bad, 4);
  int4 h[2048];
  for (int i = 0; i < 2048; ++i) h[i] = make_int4(i, 2 * i, 3 * i, 7 * i + 1);
  cudaMemcpy(src, h, 32768, cudaMemcpyHostToDevice);
  cudaMemset(bad, 0, 4);
  k<<<2, 128>>>(src, bad);
  cudaError_t e = cudaDeviceSynchronize();
  int hb = -1;
  cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  printf("%s (launch: %s, mismatched vectors %d)\n", (e == cudaSuccess && hb == 0) ? "OK" : "MISMATCH",
         cudaGetErrorString(e), hb);
  return 0;
}
