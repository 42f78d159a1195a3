// Combine inside a GEMM2 epilogue: the gate-weighted sum of a token's k expert
// outputs (reference moesim::combine<T>, proj/include/moesim/gating.hpp:107-141).
//
// Run by the 4 epilogue warps (tid 0..127) of a CTA after one GEMM2 tile's
// bf16 gate-weighted partials (Yw rows row0 .. row0+len-1, feature block m of
// 128) are stored.  Each row bumps its token's counter for this feature block;
// the k-th arrival is the finisher, which sums the token's k partials in slot
// order (j = 0..k-1) in fp32 and writes the bf16 output row -- the arithmetic
// of combine_kernel (rowops.cu), so the result is bitwise the same whatever
// order the contributions arrive in.  Counters reset themselves.  One fence,
// one round of atomics and one round of partial loads per tile.
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

namespace moe {

__device__ __forceinline__ void combine_rows_epilogue(
    const __nv_bfloat16* Yw, int TD, int k, const int32_t* order, const int32_t* pos,
    int32_t* cnt, __nv_bfloat16* out, int row0, int len, int m, int tid, int* fin_tok,
    int* fin_cnt) {
  const int MT = TD / 128;
  __threadfence();  // this thread's partial stores are visible device-wide
  if (tid == 0) fin_cnt[0] = 0;
  asm volatile("bar.sync 1, 128;" ::: "memory");
  for (int r = tid; r < len; r += 128) {
    const int tk = order[row0 + r] / k;
    int32_t* c = cnt + static_cast<size_t>(tk) * MT + m;
    if (atomicAdd(c, 1) == k - 1) {
      *c = 0;  // self-reset for the next forward
      fin_tok[atomicAdd(fin_cnt, 1)] = tk;
    }
  }
  __threadfence();
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const int nfin = fin_cnt[0];
  const int col = m * 128;
  for (int w = tid; w < nfin * 16; w += 128) {
    const int tk = fin_tok[w >> 4];
    const int c = (w & 15) * 8;  // 8 bf16 = 16 bytes
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < k; ++j) {
      const int p = pos[static_cast<size_t>(tk) * k + j];
      const uint4 v =
          __ldcg(reinterpret_cast<const uint4*>(Yw + static_cast<size_t>(p) * TD + col + c));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        acc[2 * i] += f.x;
        acc[2 * i + 1] += f.y;
      }
    }
    uint4 o;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
    *reinterpret_cast<uint4*>(out + static_cast<size_t>(tk) * TD + col + c) = o;
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");  // fin_tok is reused by the next tile
}

}  // namespace moe
