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
#include <cooperative_groups.h>
#include <float.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

constexpr int kBlockM = 128;
// 32-deep k-blocks (64-byte rows, 64-byte swizzle): a stage is 8 KB of X +
// b_rows x 64 B of Wg (40 KB at E = 512), so five stages fit and the loads of
// four k-blocks are in flight while one is multiplied (at 64-deep stages only
// two 80 KB stages fit and the MMA waited on every load).
constexpr int kBlockK = 32;
constexpr int kABytes = kBlockM * kBlockK * 2;
constexpr int kMaxK = 8;
constexpr int kMaxSmem = 220 * 1024;
// more stages (16) measured equal at MT and cfg1 (same box): the gate is not
// bound by loads in flight
#ifndef MOE_GATE_MAX_STAGES
#define MOE_GATE_MAX_STAGES 8
#endif
constexpr int kMaxStages = MOE_GATE_MAX_STAGES;

struct GateLayout {
  int e_pad;      // E rounded up to 16
  int b_rows;     // rows of Wg staged per k-block (n_box boxes)
  int box_rows;   // TMA box height for Wg
  int n_box;      // 4 when E_pad >= 128 (one box per CTA of a 4-CTA cluster), else 1
  int stages;
  int smem;
};

// Wg k-block slab = n_box boxes; a cluster of C CTAs (C | n_box) splits the
// boxes between its CTAs and multicasts each to all of them.
__host__ __device__ inline GateLayout gate_layout(int E, int bk = kBlockK) {
  GateLayout L;
  L.e_pad = (E + 15) & ~15;
  if (L.e_pad >= 128) {
    L.b_rows = (L.e_pad + 31) & ~31;
    L.n_box = 4;
  } else {
    L.b_rows = L.e_pad;
    L.n_box = 1;
  }
  L.box_rows = L.b_rows / L.n_box;  // multiple of 8: every box starts on a swizzle atom
  const int stage = kBlockM * bk * 2 + L.b_rows * bk * 2;
  int s = (kMaxSmem - 2048) / stage;
  L.stages = s > kMaxStages ? kMaxStages : s;
  L.smem = 1024 + L.stages * stage + (2 * L.stages + 2) * 8 + 16;
  return L;
}

// Insert (v, e) into a list sorted by (descending value, ascending id).  The
// candidate's id is larger than every id already in the list, so on equal
// values it stays behind; once placed, every later entry shifts down.
// Branch-free (selects only) so the 32 lanes never diverge.
__device__ __forceinline__ unsigned long long gate_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

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

// Top-K epilogue of one 128-token tile (all 8 warps of the CTA): TMEM lane =
// token, columns = expert logits.  Warps q and q+4 share TMEM lane quadrant q
// (tokens 32q..32q+31); warps 0-3 scan the first half of the expert columns,
// warps 4-7 the second half, then the two partial top-K lists are merged
// through shared memory (the stage buffers, free once tfull fired).
template <int K>
__device__ __forceinline__ void gate_epilogue(const GateArgs& a, uint32_t tmem_base,
                                              uint64_t* tfull, int tok0, uint8_t* smem, int* s_e,
                                              float* s_w) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  ptx::mbar_wait(tfull, 0);
  ptx::tc_fence_after();
  if (a.prof && threadIdx.x == 0) a.prof[3 * blockIdx.x + 1] = gate_clock();
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
  // K = 2: a second list for the odd columns (two independent compare /
  // select chains instead of one vote-guarded insert per value)
  float ov0 = -INFINITY, ov1 = -INFINITY;
  int oi0 = 0x7fffffff, oi1 = 0x7fffffff;
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
    if constexpr (K == 2) {
      // strict > within a list: ids ascend, so ties keep the lower id
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float v = (c0 + i < a.E) ? __uint_as_float(r[i]) : -INFINITY;
        const float w = (c0 + i + 1 < a.E) ? __uint_as_float(r[i + 1]) : -INFINITY;
        const bool t0 = v > bv[0], t1 = v > bv[1];
        bv[1] = t0 ? bv[0] : (t1 ? v : bv[1]);
        bi[1] = t0 ? bi[0] : (t1 ? c0 + i : bi[1]);
        bv[0] = t0 ? v : bv[0];
        bi[0] = t0 ? c0 + i : bi[0];
        const bool u0 = w > ov0, u1 = w > ov1;
        ov1 = u0 ? ov0 : (u1 ? w : ov1);
        oi1 = u0 ? oi0 : (u1 ? c0 + i + 1 : oi1);
        ov0 = u0 ? w : ov0;
        oi0 = u0 ? c0 + i + 1 : oi0;
      }
    } else {
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
  }
  if constexpr (K == 2) {
    // merge the odd-column list: order by (value desc, id asc)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float v = j ? ov1 : ov0;
      const int e = j ? oi1 : oi0;
      const bool t0 = v > bv[0] || (v == bv[0] && e < bi[0]);
      const bool t1 = v > bv[1] || (v == bv[1] && e < bi[1]);
      bv[1] = t0 ? bv[0] : (t1 ? v : bv[1]);
      bi[1] = t0 ? bi[0] : (t1 ? e : bi[1]);
      bv[0] = t0 ? v : bv[0];
      bi[0] = t0 ? e : bi[0];
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
        if (s_e) {
          s_e[tl * k + j] = bi[j];
          s_w[tl * k + j] = wj;
        }
      }
    }
  }

}

// One 128-token tile of the gate: TMA + tcgen05 logits, top-K epilogue on all
// 8 warps, idx / w written to global; with s_e/s_w the tile's routing is also
// left in shared memory (slot t*k+j of the tile) for a fused dispatch.
// Ends with a block barrier and the TMEM released.
template <int K, int C = 1, int BK = kBlockK>
__device__ __forceinline__ void gate_tile(const CUtensorMap& tmX, const CUtensorMap& tmWg,
                                          const GateArgs& a, uint8_t* smem, int* s_e,
                                          float* s_w) {
  static_assert(C == 1 || C == 2 || C == 4, "cluster of 1, 2 or 4 CTAs");
  static_assert(BK == 32 || BK == 64, "32-deep (64-byte swizzle) or 64-deep (128-byte) k-blocks");
  constexpr int kABytes = kBlockM * BK * 2;
  if (a.prof && threadIdx.x == 0) a.prof[3 * blockIdx.x] = gate_clock();
  const GateLayout L = gate_layout(a.E, BK);
  const int stage_bytes = kABytes + L.b_rows * BK * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.stages * stage_bytes);
  uint64_t* empty = full + L.stages;
  uint64_t* tfull = empty + L.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tok0 = blockIdx.x * kBlockM;
  const int KB = a.TD / BK;
  auto desc = [](uint32_t addr) {
    return BK == 64 ? ptx::umma_desc_sw128(addr) : ptx::umma_desc_sw64(addr);
  };

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmX);
    ptx::prefetch_tmap(&tmWg);
    for (int s = 0; s < L.stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], C);  // one MMA commit from every CTA that reads the stage
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
  if (C > 1) ptx::cluster_sync();  // peers' barriers exist before any multicast lands
  pdl_trigger();
  pdl_wait();  // X and the routing buffers belong to the previous kernel until here

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------- TMA producer
      const uint64_t pol_x = ptx::policy_evict_first();
      const uint64_t pol_w = ptx::policy_evict_last();
      // this CTA's share of the Wg boxes (all of them without a cluster)
      const int per = L.n_box / C;
      const int b_lo = C > 1 ? static_cast<int>(ptx::cluster_ctarank()) * per : 0;
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < KB; ++kb) {
        // free once every CTA of the cluster has consumed the stage
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], stage_bytes);
        uint8_t* st = smem + stage * stage_bytes;
        ptx::tma_load_2d(st, &tmX, &full[stage], kb * BK, tok0, pol_x);
        for (int b = b_lo; b < b_lo + per; ++b) {
          const int r = b * L.box_rows;
          if (C > 1)
            ptx::tma_load_2d_mc(st + kABytes + r * BK * 2, &tmWg, &full[stage], kb * BK, r,
                                static_cast<uint16_t>((1u << C) - 1), pol_w);
          else
            ptx::tma_load_2d(st + kABytes + r * BK * 2, &tmWg, &full[stage], kb * BK, r, pol_w);
        }
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
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint32_t acc = (kb | kk) != 0 ? 1u : 0u;
          ptx::mma_bf16(tmem_base, desc(a0 + kk * 32), desc(b0 + kk * 32), id0, acc);
          if (n1 > 0)
            ptx::mma_bf16(tmem_base + 256, desc(a0 + kk * 32), desc(b0 + 256 * BK * 2 + kk * 32), id1,
                          acc);
        }
        if (C > 1)
          ptx::mma_commit_mc(&empty[stage], static_cast<uint16_t>((1u << C) - 1));
        else
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

  gate_epilogue<K>(a, tmem_base, tfull, tok0, smem, s_e, s_w);

  __syncthreads();
  if (a.prof && threadIdx.x == 0) a.prof[3 * blockIdx.x + 2] = gate_clock();
  ptx::tc_fence_after();
  if (warp == 2) {
    if (L.e_pad <= 32) ptx::tmem_dealloc<32>(tmem_base);
    else if (L.e_pad <= 64) ptx::tmem_dealloc<64>(tmem_base);
    else if (L.e_pad <= 128) ptx::tmem_dealloc<128>(tmem_base);
    else if (L.e_pad <= 256) ptx::tmem_dealloc<256>(tmem_base);
    else ptx::tmem_dealloc<512>(tmem_base);
  }
  // peers' last MMA commits arrive on this CTA's empty barriers: stay alive
  if (C > 1) ptx::cluster_sync();
}

__device__ __forceinline__ uint8_t* aligned_smem() {
  extern __shared__ uint8_t smem_raw[];
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                    ~static_cast<uintptr_t>(1023));
}

// ---------------------------------------------------------------- CTA-pair gate
// For E a multiple of 256 (the LM layer: E = 512) the gate is MMA-bound: a
// cluster of two CTAs covers 256 tokens with tcgen05.mma.cta_group::2
// (M = 256, N = 256 per instruction).  Each CTA stages its own 128 X rows and
// HALF of every 256-expert Wg chunk (the instruction reads the B halves of
// both CTAs); the leader issues the MMAs and commits to both CTAs' barriers;
// each CTA then runs the usual top-K epilogue on its own TMEM lanes.
struct GatePairLayout {
  int nch;         // 256-expert chunks
  int stage;       // bytes per stage and CTA: X 8 KB + nch x 128 Wg rows x 64 B
  int stages;
  int smem;
};
__host__ __device__ inline GatePairLayout gate_pair_layout(int E) {
  GatePairLayout L;
  L.nch = (E + 255) / 256;
  L.stage = kABytes + L.nch * 128 * kBlockK * 2;
  int s = (200 * 1024 - 2048) / L.stage;
  L.stages = s > 8 ? 8 : s;
  L.smem = 1024 + L.stages * L.stage + (2 * L.stages + 2) * 8 + 16;
  return L;
}

template <int K>
__global__ void __launch_bounds__(256, 1)
    gate_pair_kernel(const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ CUtensorMap tmWg, GateArgs a, int box_rows) {
  const GatePairLayout L = gate_pair_layout(a.E);
  uint8_t* smem = aligned_smem();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.stages * L.stage);
  uint64_t* empty = full + L.stages;
  uint64_t* tfull = empty + L.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int tok0 = blockIdx.x * kBlockM;  // consecutive blocks form the pair
  const int KB = a.TD / kBlockK;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmX);
    ptx::prefetch_tmap(&tmWg);
    for (int s = 0; s < L.stages; ++s) {
      ptx::mbar_init(&full[s], 1);   // leader: its producer's arrive (+ both CTAs' bytes)
      ptx::mbar_init(&empty[s], 1);  // the leader's MMA commit
    }
    ptx::mbar_init(tfull, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    if (L.nch > 1)
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       ptx::smem_u32(tmem_slot)) : "memory");
    else
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                       ptx::smem_u32(tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // both CTAs' barriers and TMEM exist before any remote use
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------ producer (both CTAs)
    const uint64_t pol_x = ptx::policy_evict_first();
    const uint64_t pol_w = ptx::policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < KB; ++kb) {
      ptx::mbar_wait(&empty[stage], phase ^ 1);
      const uint32_t fb = ptx::leader_smem_addr(&full[stage]);
      if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * L.stage);
      uint8_t* st = smem + stage * L.stage;
      ptx::tma_load_2d_pair(st, &tmX, fb, kb * kBlockK, tok0, pol_x);
      for (int j = 0; j < L.nch; ++j)
        for (int r = 0; r < 128; r += box_rows)
          ptx::tma_load_2d_pair(st + kABytes + (j * 128 + r) * kBlockK * 2, &tmWg, fb, kb * kBlockK,
                                j * 256 + static_cast<int>(rank) * 128 + r, pol_w);
      if (++stage == L.stages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ------------------------------------------------ MMA issuer (leader)
    const uint32_t idesc = ptx::idesc_bf16(2 * kBlockM, 256);
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < KB; ++kb) {
      ptx::mbar_wait(&full[stage], phase);
      ptx::tc_fence_after();
      const uint32_t a0 = ptx::smem_u32(smem + stage * L.stage);
      const uint32_t b0 = a0 + kABytes;
#pragma unroll
      for (int kk = 0; kk < kBlockK / 16; ++kk)
        for (int j = 0; j < L.nch; ++j)
          ptx::mma_bf16_pair(tmem_base + j * 256, ptx::umma_desc_sw64(a0 + kk * 32),
                             ptx::umma_desc_sw64(b0 + j * 128 * kBlockK * 2 + kk * 32), idesc,
                             (kb | kk) != 0 ? 1u : 0u);
      ptx::mma_commit_pair(&empty[stage]);
      if (++stage == L.stages) {
        stage = 0;
        phase ^= 1;
      }
    }
    ptx::mma_commit_pair(tfull);
  }
  __syncwarp();

  gate_epilogue<K>(a, tmem_base, tfull, tok0, smem, nullptr, nullptr);

  // the leader's last commits into the peer and the peer's TMA completions on
  // the leader's barriers must land before either CTA leaves
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 2) {
    if (L.nch > 1)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem_base) : "memory");
  }
}

template <int K, int C, int BK = kBlockK>
__global__ void __launch_bounds__(256, 1)
    gate_topk_kernel(const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ CUtensorMap tmWg, GateArgs a) {
  gate_tile<K, C, BK>(tmX, tmWg, a, aligned_smem(), nullptr, nullptr);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// peers holding the same key (one ballot per key bit; see route.cu)
__device__ __forceinline__ uint32_t match_key(int key, int nbits) {
  uint32_t m = __ballot_sync(0xffffffffu, key >= 0);
  for (int bit = 0; bit < nbits; ++bit) {
    const bool set = (key >> bit) & 1;
    const uint32_t bm = __ballot_sync(0xffffffffu, set);
    m &= set ? bm : ~bm;
  }
  return m;
}

// Exclusive scan of v[0..n) by the block (256 threads); returns the total.
__device__ int scan_block(int* v, int n, int* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int s = 0;
  for (int i = lo; i < hi; ++i) s += v[i];
  int x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nwarps ? scratch[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    scratch[lane] = w;
  }
  __syncthreads();
  int run = (warp > 0 ? scratch[warp - 1] : 0) + x - s;
  for (int i = lo; i < hi; ++i) {
    const int t = v[i];
    v[i] = run;
    run += t;
  }
  const int total = scratch[nwarps - 1];
  __syncthreads();
  return total;
}

// Gate + dynamic dispatch + gather in one cooperative launch (one CTA per
// 128-token tile, all resident): after the gate tile the CTA histograms its
// 128*k slots, a grid barrier publishes every tile's histogram, each CTA
// derives the global splits and its own stable bases (tiles in token order,
// warps in slot order, ballot-ranked lanes -- the route kernel's order,
// bit-exact to dynamic_dispatch, gating.cpp:58-86), scatters order/pos/wpos
// and copies its tokens' rows into the expert-grouped Xp.  Saves the route
// and gather launches and their HBM round trips of idx/order.
template <int K>
__global__ void __launch_bounds__(256, 1)
    gate_dispatch_kernel(const __grid_constant__ CUtensorMap tmX,
                         const __grid_constant__ CUtensorMap tmWg, GateArgs a, DispatchArgs d) {
  namespace cg = cooperative_groups;
  uint8_t* smem = aligned_smem();
  const int k = a.k, E = a.E;
  int* s_e = reinterpret_cast<int*>(smem + 8192);
  float* s_w = reinterpret_cast<float*>(smem + 8192 + 4096);
  gate_tile<K>(tmX, tmWg, a, smem, s_e, s_w);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x, nb = gridDim.x;
  const int nb4 = (nb + 3) & ~3;
  const int tok0 = b * kBlockM;
  const int nslots = min(kBlockM, a.S - tok0) * k;  // slots of this tile
  // smem after the gate: [0,8K) merge area | s_e | s_w | s_row (4 KB each) | counts
  int* s_row = reinterpret_cast<int*>(smem + 16384);     // [128 * k] row of each slot
  int* warp_cnt = reinterpret_cast<int*>(smem + 20480);  // [8][E]
  int* tot = warp_cnt + 8 * E;                             // [E]
  int* before = tot + E;                                   // [E]
  int* scratch = before + E;                               // [33]
  const int nbits = 32 - __clz(max(E - 1, 1));
  const int per_warp = (((kBlockM * k + 7) / 8) + 31) & ~31;
  const int w_lo = warp * per_warp, w_hi = min(nslots, w_lo + per_warp);
  int* my_cnt = warp_cnt + warp * E;

  // local histogram, per warp
  for (int i = threadIdx.x; i < 8 * E; i += blockDim.x) warp_cnt[i] = 0;
  __syncthreads();
  for (int base = w_lo; base < w_hi; base += 32) {
    const int e = base + lane < w_hi ? s_e[base + lane] : -1;
    const uint32_t peers = match_key(e, nbits);
    if (e >= 0 && (peers & lanemask_lt()) == 0) my_cnt[e] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  if (b == 0)
    for (int i = threadIdx.x; i < E * (nb4 - nb); i += blockDim.x)
      d.block_hist[(size_t)(i / (nb4 - nb)) * nb4 + nb + i % (nb4 - nb)] = 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += warp_cnt[w * E + e];
    d.block_hist[(size_t)e * nb4 + b] = s;
  }
  cg::this_grid().sync();

  // global splits and this tile's bases
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int4* row = reinterpret_cast<const int4*>(d.block_hist + (size_t)e * nb4);
    int s = 0, bf = 0;
#pragma unroll 4
    for (int j4 = 0; j4 < nb4 / 4; ++j4) {
      const int4 x = row[j4];
      const int j = 4 * j4;
      s += x.x + x.y + x.z + x.w;
      bf += (j < b ? x.x : 0) + (j + 1 < b ? x.y : 0) + (j + 2 < b ? x.z : 0) +
            (j + 3 < b ? x.w : 0);
    }
    tot[e] = s;
    before[e] = bf;
  }
  __syncthreads();
  if (b == 0)
    for (int e = threadIdx.x; e < E; e += blockDim.x) d.counts[e] = tot[e];
  const int grand = scan_block(tot, E, scratch);  // tot -> splits
  if (b == 0) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) d.splits[e] = tot[e];
    if (threadIdx.x == 0) d.splits[E] = grand;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int run = tot[e] + before[e];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const int x = warp_cnt[w * E + e];
      warp_cnt[w * E + e] = run;
      run += x;
    }
  }
  __syncthreads();

  // stable scatter of this tile's slots; remember each slot's row for the gather
  for (int base = w_lo; base < w_hi; base += 32) {
    const int sl = base + lane;
    const int e = sl < w_hi ? s_e[sl] : -1;
    const uint32_t peers = match_key(e, nbits);
    if (e >= 0) {
      const int p = my_cnt[e] + __popc(peers & lanemask_lt());
      const int slot = tok0 * k + sl;
      d.order[p] = slot;
      d.pos[slot] = p;
      d.wpos[p] = s_w[sl];
      s_row[sl] = p;
    }
    __syncwarp();
    if (e >= 0 && (peers & lanemask_lt()) == 0) my_cnt[e] += __popc(peers);
    __syncwarp();
  }

  // FFN work items (block 0)
  if (b == 0) {
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x)
      before[e] = (d.counts[e] + d.tile_n - 1) / d.tile_n;
    __syncthreads();
    const int n_items = scan_block(before, E, scratch);
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      const int rows = d.counts[e];
      int it = before[e];
      for (int c = 0; c < rows; c += d.tile_n, ++it) {
        FfnItem item;
        item.expert = e;
        item.row0 = tot[e] + c;
        item.len = min(d.tile_n, rows - c);
        item.pad = 0;
        d.items[it] = item;
      }
      if (d.item_off) d.item_off[e] = before[e];
    }
    if (threadIdx.x == 0) {
      *d.n_items = n_items;
      if (d.item_off) d.item_off[E] = n_items;
    }
  }
  __syncthreads();

  // gather: token rows of this tile -> their expert-grouped rows of Xp
  const int vec = a.TD / 8;  // uint4 per row
  const uint4* X = reinterpret_cast<const uint4*>(d.X);
  uint4* Xp = reinterpret_cast<uint4*>(d.Xp);
  // each warp moves two rows at a time with 4 independent 16-byte loads in
  // flight per lane per row
  for (int sl = warp; sl < nslots; sl += 8) {
    const uint4* src = X + (size_t)(tok0 + sl / k) * vec;
    uint4* dst = Xp + (size_t)s_row[sl] * vec;
    int v = lane;
    for (; v + 96 < vec; v += 128) {
      const uint4 r0 = __ldg(src + v), r1 = __ldg(src + v + 32), r2 = __ldg(src + v + 64),
                  r3 = __ldg(src + v + 96);
      dst[v] = r0;
      dst[v + 32] = r1;
      dst[v + 64] = r2;
      dst[v + 96] = r3;
    }
    for (; v < vec; v += 32) dst[v] = __ldg(src + v);
  }
}

}  // namespace

int gate_box_rows(int E) { return gate_layout(E).box_rows; }
// 64-deep k-blocks with 128-byte rows for E <= 128 (a 32 KB stage at E = 128,
// six stages): 32-deep boxes of 64-byte rows streamed X at ~35-65 GB/s per SM
// (MOE_GATE_PROF); the cooperative gate + dispatch and the CTA-pair gate keep
// 32.  MOE_GATE_WIDE=0 restores 32 everywhere.
bool gate_pair_enabled(int E);
bool gate_wide(int E) {
  static const int env = [] {
    const char* v = getenv("MOE_GATE_WIDE");
    return v ? atoi(v) : 1;
  }();
  return env != 0 && gate_layout(E).e_pad <= 128 && !gate_pair_enabled(E);
}
int gate_box_cols(int E, bool fused_front) { return !fused_front && gate_wide(E) ? 64 : kBlockK; }

template <int C, int BK = kBlockK>
const void* gate_fn(int k) {
  return k == 1   ? reinterpret_cast<const void*>(gate_topk_kernel<1, C, BK>)
         : k == 2 ? reinterpret_cast<const void*>(gate_topk_kernel<2, C, BK>)
         : k <= 4 ? reinterpret_cast<const void*>(gate_topk_kernel<4, C, BK>)
                  : reinterpret_cast<const void*>(gate_topk_kernel<8, C, BK>);
}

cudaError_t gate_prepare(int E) {
  // process-wide kernel attribute: only raise it (see route_prepare)
  static std::mutex mu;
  static int granted = 0;
  const GateLayout L = gate_layout(E);
  std::lock_guard<std::mutex> lock(mu);
  if (L.smem <= granted) return cudaSuccess;
  const void* fns[] = {reinterpret_cast<const void*>(gate_dispatch_kernel<1>),
                       reinterpret_cast<const void*>(gate_dispatch_kernel<2>),
                       reinterpret_cast<const void*>(gate_dispatch_kernel<4>),
                       reinterpret_cast<const void*>(gate_dispatch_kernel<8>)};
  for (const void* fn : fns) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem);
    if (e != cudaSuccess) return e;
  }
  const int wsmem = gate_layout(E, 64).smem;
  for (int k : {1, 2, 4, 8}) {
    for (const void* fn : {gate_fn<1>(k), gate_fn<2>(k), gate_fn<4>(k)}) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem);
      if (e != cudaSuccess) return e;
    }
    for (const void* fn : {gate_fn<1, 64>(k), gate_fn<2, 64>(k), gate_fn<4, 64>(k)}) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           std::max(wsmem, L.smem));
      if (e != cudaSuccess) return e;
    }
  }
  {
    const int psmem = gate_pair_layout(E).smem;
    const void* pfns[] = {reinterpret_cast<const void*>(gate_pair_kernel<1>),
                          reinterpret_cast<const void*>(gate_pair_kernel<2>),
                          reinterpret_cast<const void*>(gate_pair_kernel<4>),
                          reinterpret_cast<const void*>(gate_pair_kernel<8>)};
    for (const void* fn : pfns) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           std::max(psmem, L.smem));
      if (e != cudaSuccess) return e;
    }
  }
  granted = L.smem;
  return cudaSuccess;
}

// Cluster size for the gate: the largest C | n_box (<= MOE_GATE_CLUSTER, default
// 4) for which every cluster of the grid is co-resident (one wave).
int gate_cluster(const GateLayout& L, int tiles, int smem, bool wide = false) {
  static int env = -1;
  if (env < 0) {
    const char* v = getenv("MOE_GATE_CLUSTER");
    env = v ? atoi(v) : 4;
  }
  for (int C = 4; C >= 2; C >>= 1) {
    if (C > env || L.n_box % C != 0 || tiles < C) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((tiles + C - 1) / C * C);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = C;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    const void* fn = wide ? (C == 4 ? gate_fn<4, 64>(2) : gate_fn<2, 64>(2))
                          : (C == 4 ? gate_fn<4>(2) : gate_fn<2>(2));
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (n * C >= tiles) return C;
  }
  return 1;
}

template <int K, int BK = kBlockK>
cudaError_t launch_gate_k(const CUtensorMap& tmX, const CUtensorMap& tmWg, const GateArgs& a,
                          int C, int tiles, int smem, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((tiles + C - 1) / C * C);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeClusterDimension;
  attr[n].val.clusterDim.x = C;
  attr[n].val.clusterDim.y = 1;
  attr[n].val.clusterDim.z = 1;
  ++n;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  if (C == 4) return cudaLaunchKernelEx(&cfg, gate_topk_kernel<K, 4, BK>, tmX, tmWg, a);
  if (C == 2) return cudaLaunchKernelEx(&cfg, gate_topk_kernel<K, 2, BK>, tmX, tmWg, a);
  return cudaLaunchKernelEx(&cfg, gate_topk_kernel<K, 1, BK>, tmX, tmWg, a);
}

template <int K>
cudaError_t launch_gate_pair_k(const CUtensorMap& tmX, const CUtensorMap& tmWg, const GateArgs& a,
                               int tiles, cudaStream_t stream) {
  const GatePairLayout P = gate_pair_layout(a.E);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((tiles + 1) / 2 * 2);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = P.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeClusterDimension;
  attr[n].val.clusterDim.x = 2;
  attr[n].val.clusterDim.y = 1;
  attr[n].val.clusterDim.z = 1;
  ++n;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, gate_pair_kernel<K>, tmX, tmWg, a, gate_layout(a.E).box_rows);
}

// CTA-pair gate for E a multiple of 256: MOE_GATE_PAIR=1.  Off by default:
// correct (all GPU tests pass with it) but measured 31.2 vs 29.7 us at LM
// (same box): the gate is not MMA-bound, and the pair gives up the 4-CTA Wg
// multicast.
bool gate_pair_enabled(int E) {
  static const int v = [] {
    const char* e = getenv("MOE_GATE_PAIR");
    return e ? atoi(e) : 0;
  }();
  return v != 0 && E % 256 == 0 && 128 % gate_layout(E).box_rows == 0;
}

cudaError_t launch_gate(const CUtensorMap& tmX, const CUtensorMap& tmWg, const GateArgs& a,
                        cudaStream_t stream) {
  const bool wide = gate_wide(a.E);
  if (a.k < 1 || a.k > kMaxK || a.E > 512 || a.E < a.k || (a.TD % (wide ? 64 : kBlockK)) != 0)
    return cudaErrorInvalidValue;
  const GateLayout L = gate_layout(a.E, wide ? 64 : kBlockK);
  const int tiles = (a.S + kBlockM - 1) / kBlockM;
  if (gate_pair_enabled(a.E)) {
    if (a.k == 1) return launch_gate_pair_k<1>(tmX, tmWg, a, tiles, stream);
    if (a.k == 2) return launch_gate_pair_k<2>(tmX, tmWg, a, tiles, stream);
    if (a.k <= 4) return launch_gate_pair_k<4>(tmX, tmWg, a, tiles, stream);
    return launch_gate_pair_k<8>(tmX, tmWg, a, tiles, stream);
  }
  // cached per (E, tiles): the occupancy query is not free
  static std::mutex mu;
  static std::map<std::pair<int, int>, int> cache;
  int C;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({L.e_pad, tiles});
    if (it == cache.end()) it = cache.emplace(std::make_pair(L.e_pad, tiles), gate_cluster(L, tiles, L.smem, wide)).first;
    C = it->second;
  }
  static const bool prof = getenv("MOE_GATE_PROF") != nullptr;
  GateArgs b = a;
  static unsigned long long* prof_buf = nullptr;
  if (prof) {
    if (!prof_buf) cudaMalloc(&prof_buf, 3 * 4096 * sizeof(unsigned long long));
    b.prof = prof_buf;
  }
  cudaError_t e;
  if (wide) {
    if (a.k == 1) e = launch_gate_k<1, 64>(tmX, tmWg, b, C, tiles, L.smem, stream);
    else if (a.k == 2) e = launch_gate_k<2, 64>(tmX, tmWg, b, C, tiles, L.smem, stream);
    else if (a.k <= 4) e = launch_gate_k<4, 64>(tmX, tmWg, b, C, tiles, L.smem, stream);
    else e = launch_gate_k<8, 64>(tmX, tmWg, b, C, tiles, L.smem, stream);
  } else if (a.k == 1) e = launch_gate_k<1>(tmX, tmWg, b, C, tiles, L.smem, stream);
  else if (a.k == 2) e = launch_gate_k<2>(tmX, tmWg, b, C, tiles, L.smem, stream);
  else if (a.k <= 4) e = launch_gate_k<4>(tmX, tmWg, b, C, tiles, L.smem, stream);
  else e = launch_gate_k<8>(tmX, tmWg, b, C, tiles, L.smem, stream);
  if (!prof || e != cudaSuccess || tiles > 4096) return e;
  // experiments only: per-CTA mainloop / epilogue split of this launch
  std::vector<unsigned long long> h(3 * (size_t)tiles);
  cudaStreamSynchronize(stream);
  cudaMemcpy(h.data(), prof_buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull, t2 = 0;
  double m = 0, ep = 0;
  for (int i = 0; i < tiles; ++i) {
    t0 = std::min(t0, h[3 * i]);
    t2 = std::max(t2, h[3 * i + 2]);
    m += (double)(h[3 * i + 1] - h[3 * i]);
    ep += (double)(h[3 * i + 2] - h[3 * i + 1]);
  }
  fprintf(stderr, "[gate prof] %d CTAs (cluster %d): mean mainloop %.1f us, mean epilogue %.1f us, span %.1f us\n",
          tiles, C, m / tiles * 1e-3, ep / tiles * 1e-3, (t2 - t0) * 1e-3);
  return e;
}

}  // namespace moe

namespace moe {

// Smem the fused kernel needs beyond the gate stages: merge area + tile
// routing (16 KB) + per-warp histograms and scans.
bool gate_dispatch_supported(int S, int E, int k, int TD, int sms) {
  const GateLayout L = gate_layout(E);
  const int tiles = (S + kBlockM - 1) / kBlockM;
  const size_t need = 20480 + sizeof(int) * (10 * (size_t)E + 64);
  return tiles <= sms && need <= (size_t)L.stages * (kABytes + L.b_rows * kBlockK * 2) &&
         k * kBlockM <= 1024 && TD % 8 == 0;
}

cudaError_t launch_gate_dispatch(const CUtensorMap& tmX, const CUtensorMap& tmWg,
                                 const GateArgs& a, const DispatchArgs& d, cudaStream_t stream) {
  if (a.k < 1 || a.k > kMaxK || a.E > 512 || a.E < a.k || (a.TD % kBlockK) != 0)
    return cudaErrorInvalidValue;
  const GateLayout L = gate_layout(a.E);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.S + kBlockM - 1) / kBlockM);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a.k == 1) return cudaLaunchKernelEx(&cfg, gate_dispatch_kernel<1>, tmX, tmWg, a, d);
  if (a.k == 2) return cudaLaunchKernelEx(&cfg, gate_dispatch_kernel<2>, tmX, tmWg, a, d);
  if (a.k <= 4) return cudaLaunchKernelEx(&cfg, gate_dispatch_kernel<4>, tmX, tmWg, a, d);
  return cudaLaunchKernelEx(&cfg, gate_dispatch_kernel<8>, tmX, tmWg, a, d);
}

}  // namespace moe
