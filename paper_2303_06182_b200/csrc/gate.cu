// Gate: logits = X Wg^T on tcgen05, fused with softmax + top-k selection.
//
// The paper's gate (a gating function picks the top-1 or
// top-2 experts per token) is absent from the reference (SPEC.md:224 rules the
// gate's linear layer and softmax out of the simulator); the reference only
// fixes what a routing decision must satisfy: k distinct ids in [0,E), weights
// >= 0 summing to 1 (proj/src/trace.cpp:47-67).
//
// Semantics implemented here (and restated by oracle/layer.py):
//   * k largest logits, ties -> lower expert id; slot j orders them by
//     descending logit, so slot 0 is the top choice;
//   * weights = softmax restricted to the selected experts
//     (w_j = exp(l_j - l_0) / sum_i exp(l_i - l_0)); the full-softmax
//     normaliser cancels in the renormalisation, so it is never formed;
//     the last weight is 1 - sum(others) so the pair sums to 1 exactly.
//
// Tile = 128 tokens (TMEM lanes) x E_pad experts (TMEM columns, <= 512).
// Warp 0 = TMA producer, warp 1 = MMA issuer, warp 2 = TMEM allocator,
// warps 4-7 = epilogue, one thread per token: tcgen05.ld 32 logits at a time,
// running top-k in registers, optional fp32 logits store for parity checks.
#include <float.h>

#include <mutex>

#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

constexpr int kBlockM = 128;
constexpr int kBlockK = 64;
constexpr int kABytes = kBlockM * kBlockK * 2;
constexpr int kMaxK = 8;
constexpr int kMaxSmem = 200 * 1024;

struct GateLayout {
  int e_pad;      // E rounded up to 16
  int b_rows;     // rows of Wg staged per k-block (multiple of the box height)
  int box_rows;   // TMA box height for Wg
  int stages;
  int smem;
};

__host__ __device__ inline GateLayout gate_layout(int E) {
  GateLayout L;
  L.e_pad = (E + 15) & ~15;
  L.box_rows = L.e_pad <= 256 ? L.e_pad : 256;
  L.b_rows = (L.e_pad + L.box_rows - 1) / L.box_rows * L.box_rows;
  const int stage = kABytes + L.b_rows * kBlockK * 2;
  int s = (kMaxSmem - 2048) / stage;
  L.stages = s > 8 ? 8 : s;
  L.smem = 1024 + L.stages * stage + (2 * L.stages + 2) * 8 + 16;
  return L;
}

// Insert (v, e) into a list sorted by (descending value, ascending id).  The
// candidate's id is larger than every id already in the list, so on equal
// values it stays behind; once placed, every later entry shifts down.
// Branch-free (selects only) so the 32 lanes never diverge.
template <int K>
__device__ __forceinline__ void topk_insert(float (&bv)[K], int (&bi)[K], float v, int e) {
  bool carry = false;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const bool t = carry || (v > bv[j]);
    const float tv = bv[j];
    const int ti = bi[j];
    bv[j] = t ? v : tv;
    bi[j] = t ? e : ti;
    v = t ? tv : v;
    e = t ? ti : e;
    carry = t;
  }
}

template <int K>
__global__ void __launch_bounds__(256, 1)
    gate_topk_kernel(const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ CUtensorMap tmWg, GateArgs a) {
  const GateLayout L = gate_layout(a.E);
  const int stage_bytes = kABytes + L.b_rows * kBlockK * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.stages * stage_bytes);
  uint64_t* empty = full + L.stages;
  uint64_t* tfull = empty + L.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tok0 = blockIdx.x * kBlockM;
  const int KB = a.TD / kBlockK;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmX);
    ptx::prefetch_tmap(&tmWg);
    for (int s = 0; s < L.stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(tfull, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    if (L.e_pad <= 32) ptx::tmem_alloc<32>(tmem_slot);
    else if (L.e_pad <= 64) ptx::tmem_alloc<64>(tmem_slot);
    else if (L.e_pad <= 128) ptx::tmem_alloc<128>(tmem_slot);
    else if (L.e_pad <= 256) ptx::tmem_alloc<256>(tmem_slot);
    else ptx::tmem_alloc<512>(tmem_slot);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------- TMA producer
      const uint64_t pol_x = ptx::policy_evict_first();
      const uint64_t pol_w = ptx::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < KB; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], stage_bytes);
        uint8_t* st = smem + stage * stage_bytes;
        ptx::tma_load_2d(st, &tmX, &full[stage], kb * kBlockK, tok0, pol_x);
        for (int r = 0; r < L.b_rows; r += L.box_rows)
          ptx::tma_load_2d(st + kABytes + r * kBlockK * 2, &tmWg, &full[stage], kb * kBlockK, r,
                           pol_w);
        if (++stage == L.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------- MMA issuer
      const int n0 = L.e_pad <= 256 ? L.e_pad : 256;
      const int n1 = L.e_pad - n0;
      const uint32_t id0 = ptx::idesc_bf16(kBlockM, n0);
      const uint32_t id1 = ptx::idesc_bf16(kBlockM, n1 > 0 ? n1 : 16);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < KB; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint32_t a0 = ptx::smem_u32(smem + stage * stage_bytes);
        const uint32_t b0 = a0 + kABytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t acc = (kb | kk) != 0 ? 1u : 0u;
          ptx::mma_bf16(tmem_base, ptx::umma_desc_sw128(a0 + kk * 32),
                        ptx::umma_desc_sw128(b0 + kk * 32), id0, acc);
          if (n1 > 0)
            ptx::mma_bf16(tmem_base + 256, ptx::umma_desc_sw128(a0 + kk * 32),
                          ptx::umma_desc_sw128(b0 + 256 * 128 + kk * 32), id1, acc);
        }
        ptx::mma_commit(&empty[stage]);
        if (++stage == L.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      ptx::mma_commit(tfull);
    }
    __syncwarp();
  }

  // -------------------------------------------------------- epilogue (all 8 warps)
  // Warps q and q+4 share TMEM lane quadrant q (tokens 32q..32q+31); warps
  // 0-3 scan the first half of the expert columns, warps 4-7 the second half,
  // then the two partial top-K lists are merged through shared memory.
  ptx::mbar_wait(tfull, 0);
  ptx::tc_fence_after();
  const int q = warp & 3;
  const int half = warp >> 2;
  const int tl = q * 32 + lane;  // token within the tile
  const int tok = tok0 + tl;
  const int nchunk = (a.E + 31) / 32;
  const int split = (nchunk + 1) / 2;
  const int c_begin = half ? split * 32 : 0;
  const int c_end = half ? nchunk * 32 : split * 32;
  float bv[K];
  int bi[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    bv[j] = -INFINITY;
    bi[j] = 0x7fffffff;
  }
  for (int c0 = c_begin; c0 < c_end; c0 += 32) {
    uint32_t r[32];
    ptx::tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + c0, r);
    ptx::tmem_ld_wait();
    if (a.logits && tok < a.S) {
      float* dst = a.logits + static_cast<size_t>(tok) * a.E + c0;
      if (c0 + 32 <= a.E && (a.E & 3) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(dst + i) =
              make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                          __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < a.E) dst[i] = __uint_as_float(r[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float v = (c0 + i < a.E) ? __uint_as_float(r[i]) : -INFINITY;
      if (K == 1) {
        topk_insert<K>(bv, bi, v, c0 + i);
      } else if (__any_sync(0xffffffffu, v > bv[K - 1])) {
        topk_insert<K>(bv, bi, v, c0 + i);
      }
    }
  }
  ptx::tc_fence_before();
  // partial lists of the upper half -> smem (stage buffers are free: all TMA
  // writes landed and all MMAs retired before tfull fired)
  float* pv = reinterpret_cast<float*>(smem);
  int* pi = reinterpret_cast<int*>(smem + kBlockM * K * sizeof(float));
  if (half == 1) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      pv[j * kBlockM + tl] = bv[j];
      pi[j * kBlockM + tl] = bi[j];
    }
  }
  __syncthreads();
  if (half == 0 && tok < a.S) {
    // upper-half ids are all larger, so inserting them in order keeps ties
    // resolved toward the lower id
#pragma unroll
    for (int j = 0; j < K; ++j) topk_insert<K>(bv, bi, pv[j * kBlockM + tl], pi[j * kBlockM + tl]);
    const int k = a.k;
    float ex[K];
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      ex[j] = (j < k) ? expf(bv[j] - bv[0]) : 0.f;
      sum += ex[j];
    }
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (j < k) {
        const float wj = (j < k - 1) ? ex[j] / sum : 1.f - acc;
        acc += wj;
        a.idx[static_cast<size_t>(tok) * k + j] = bi[j];
        a.w[static_cast<size_t>(tok) * k + j] = wj;
      }
    }
  }

  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) {
    if (L.e_pad <= 32) ptx::tmem_dealloc<32>(tmem_base);
    else if (L.e_pad <= 64) ptx::tmem_dealloc<64>(tmem_base);
    else if (L.e_pad <= 128) ptx::tmem_dealloc<128>(tmem_base);
    else if (L.e_pad <= 256) ptx::tmem_dealloc<256>(tmem_base);
    else ptx::tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace

int gate_box_rows(int E) { return gate_layout(E).box_rows; }

cudaError_t gate_prepare(int E) {
  // process-wide kernel attribute: only raise it (see route_prepare)
  static std::mutex mu;
  static int granted = 0;
  const GateLayout L = gate_layout(E);
  std::lock_guard<std::mutex> lock(mu);
  if (L.smem <= granted) return cudaSuccess;
  for (auto fn : {gate_topk_kernel<1>, gate_topk_kernel<2>, gate_topk_kernel<4>, gate_topk_kernel<8>}) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem);
    if (e != cudaSuccess) return e;
  }
  granted = L.smem;
  return cudaSuccess;
}

cudaError_t launch_gate(const CUtensorMap& tmX, const CUtensorMap& tmWg, const GateArgs& a,
                        cudaStream_t stream) {
  if (a.k < 1 || a.k > kMaxK || a.E > 512 || a.E < a.k || (a.TD % kBlockK) != 0)
    return cudaErrorInvalidValue;
  const GateLayout L = gate_layout(a.E);
  const int grid = (a.S + kBlockM - 1) / kBlockM;
  if (a.k == 1) gate_topk_kernel<1><<<grid, 256, L.smem, stream>>>(tmX, tmWg, a);
  else if (a.k == 2) gate_topk_kernel<2><<<grid, 256, L.smem, stream>>>(tmX, tmWg, a);
  else if (a.k <= 4) gate_topk_kernel<4><<<grid, 256, L.smem, stream>>>(tmX, tmWg, a);
  else gate_topk_kernel<8><<<grid, 256, L.smem, stream>>>(tmX, tmWg, a);
  return cudaGetLastError();
}

}  // namespace moe
