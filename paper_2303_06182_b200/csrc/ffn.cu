// Grouped expert FFN on 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// The paper's expert FFN (absent from the reference, which
// only charges a per-assignment cost, proj/src/costmodel.cpp:79-82) is
//   H_e = relu(Xp_e W1_e^T)          Xp_e = rows of expert e, [n_e, TD]
//   Y_e = H_e W2_e^T  (scaled by the gate weight of each row)
// With n_e ~ 32..256 tokens per expert every expert's weights are streamed
// from HBM exactly once and the kernel is HBM-bound on weights.  Hence
// swap-AB: the weight slab is the M=128 operand (A), the expert's tokens are
// the N<=256 operand (B), both K-major, staged by TMA with 128-byte swizzle.
//
// Persistent, warp-specialised CTA (256 threads, one per SM):
//   warp 0   TMA producer  (A: weight tile 128x64, evict-first; B: token rows)
//   warp 1   MMA issuer    (single thread, tcgen05.mma kind::f16, fp32 in TMEM)
//   warp 2   TMEM allocator
//   warps 4-7 epilogue     (tcgen05.ld -> relu / gate-scale -> bf16 ->
//                           smem transpose -> 16-byte coalesced stores)
// Two TMEM accumulators (2 x tile_n columns) let the epilogue of tile i
// overlap the MMAs of tile i+1.  Tiles = (work item, 128-row m-block); the
// work list comes from the route kernel, so no host sync is needed.
#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

constexpr int kBlockM = 128;
constexpr int kBlockK = 64;  // one 128-byte swizzle row of bf16
constexpr int kUmmaK = 16;
constexpr int kABytes = kBlockM * kBlockK * 2;
constexpr int kEpiBytes = 4 * 32 * 32 * 2;
constexpr int kBoxRowsB = 16;

template <int BN, int STAGES>
struct GemmCfg {
  static constexpr int kBBytes = BN * kBlockK * 2;
  static constexpr int kSmem = 1024 + STAGES * (kABytes + kBBytes) + kEpiBytes +
                               (2 * STAGES + 4) * 8 + 16;
  static constexpr int kTmemCols = 2 * BN;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(256, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, GemmArgs g) {
  using Cfg = GemmCfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * kABytes;
  __nv_bfloat16* sEpi = reinterpret_cast<__nv_bfloat16*>(sB + STAGES * Cfg::kBBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sEpi) + kEpiBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // the work list and activations come from the previous kernel

  // optional expert range (expert-cache waves): items of experts [e_lo, e_hi)
  const int item0 = g.item_off ? g.item_off[g.e_lo] : 0;
  const int n_items = g.item_off ? g.item_off[g.e_hi] - item0 : *g.n_items;
  const FfnItem* items = g.items + item0;
  const int MT = g.m_total / kBlockM;
  const int KB = g.k_total / kBlockK;
  const int total = n_items * MT;

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ producer
    // (single thread: a warp-wide producer -- needed for per-lane TMA gather4 --
    // measured 15% slower on the LM shape, profiles/r01_fusion_ab.md)
    const uint64_t pol_a = ptx::policy_evict_first();
    const uint64_t pol_b = ptx::policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const FfnItem it = items[t / MT];
      const int m = t % MT;
      const int nrows = (it.len + 15) & ~15;
      const int wslot = g.slot_of ? g.slot_of[it.expert] : it.expert;
      const int a_row = wslot * g.m_total + m * kBlockM;
      const uint32_t bytes = kABytes + nrows * kBlockK * 2;
      for (int kb = 0; kb < KB; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], bytes);
        ptx::tma_load_2d(sA + stage * kABytes, &tmA, &full[stage], kb * kBlockK, a_row, pol_a);
        uint8_t* b_dst = sB + stage * Cfg::kBBytes;
        for (int r = 0; r < nrows; r += kBoxRowsB)
          ptx::tma_load_2d(b_dst + r * kBlockK * 2, &tmB, &full[stage], kb * kBlockK,
                           it.row0 + r, pol_b);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------ MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const FfnItem it = items[t / MT];
      const int n = (it.len + 15) & ~15;
      const uint32_t idesc = ptx::idesc_bf16(kBlockM, n);
      ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem_base + acc * BN;
      for (int kb = 0; kb < KB; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint32_t a0 = ptx::smem_u32(sA + stage * kABytes);
        const uint32_t b0 = ptx::smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
        for (int kk = 0; kk < kBlockK / kUmmaK; ++kk)
          ptx::mma_bf16(d, ptx::umma_desc_sw128(a0 + kk * kUmmaK * 2),
                        ptx::umma_desc_sw128(b0 + kk * kUmmaK * 2), idesc,
                        (kb | kk) != 0 ? 1u : 0u);
        ptx::mma_commit(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      ptx::mma_commit(&tfull[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quadrant owned by this warp
    __nv_bfloat16* stg = sEpi + q * 32 * 32;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const FfnItem it = items[t / MT];
      const int m = t % MT;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int col0 = m * kBlockM + q * 32;  // output feature of TMEM lane 32q
      for (int c0 = 0; c0 < it.len; c0 += 32) {
        uint32_t r[32];
        ptx::tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c0, r);
        ptx::tmem_ld_wait();
        if (g.mode == kEpiReluBf16) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            stg[i * 32 + lane] = __float2bfloat16_rn(fmaxf(__uint_as_float(r[i]), 0.f));
        } else {  // kEpiScaleBf16: gate weight of the row
          const float wv = (c0 + lane < it.len) ? g.wpos[it.row0 + c0 + lane] : 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            stg[i * 32 + lane] =
                __float2bfloat16_rn(__uint_as_float(r[i]) * __shfl_sync(0xffffffffu, wv, i));
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int tok = j * 8 + (lane >> 2);
          const int ch = lane & 3;
          if (c0 + tok < it.len) {
            const uint4 v = *reinterpret_cast<const uint4*>(stg + tok * 32 + ch * 8);
            int row = it.row0 + c0 + tok;
            if (g.out_rows) row = g.out_rows[row];
            *reinterpret_cast<uint4*>(g.out + static_cast<size_t>(row) * g.m_total + col0 +
                                      ch * 8) = v;
          }
        }
        __syncwarp();
      }
      // TMEM of this tile is no longer needed
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
}

template <int BN, int STAGES>
cudaError_t prepare_one() {
  return cudaFuncSetAttribute(grouped_gemm_kernel<BN, STAGES>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              GemmCfg<BN, STAGES>::kSmem);
}

template <int BN, int STAGES>
cudaError_t launch_one(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& g,
                       int grid, cudaStream_t stream) {
  return launch_chain(grouped_gemm_kernel<BN, STAGES>, dim3(grid), dim3(256),
                      GemmCfg<BN, STAGES>::kSmem, stream, false, tmA, tmB, g);
}

}  // namespace

cudaError_t gemm_prepare() {
  cudaError_t e = prepare_one<128, 6>();
  if (e != cudaSuccess) return e;
  return prepare_one<256, 4>();
}

cudaError_t launch_grouped_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB,
                                const GemmArgs& args, int tile_n, int grid,
                                cudaStream_t stream) {
  if (tile_n == 128) return launch_one<128, 6>(tmA, tmB, args, grid, stream);
  if (tile_n == 256) return launch_one<256, 4>(tmA, tmB, args, grid, stream);
  return cudaErrorInvalidValue;
}

}  // namespace moe
