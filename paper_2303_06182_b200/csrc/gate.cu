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
// Warp 0 = TMA producer, warp 1 = MMA issuer, warp 2 = TMEM allocator, then
// all 8 warps run the epilogue, one thread per token: tcgen05.ld 32 logits at
// a time, running top-k in registers, optional fp32 logits store for parity
// checks.  Two grid shapes:
//   * one tile per CTA, clusters of up to 4 CTAs (consecutive token tiles)
//     sharing every Wg k-block by TMA multicast -- when there are enough
//     tiles to fill the GPU (the LM layer: 128 tiles);
//   * split-K (few tiles: MT 48, cfg1 16): a cluster of C CTAs works on ONE
//     tile, each over 1/C of the token dimension; the C-1 followers push
//     their fp32 partial logits into the leader's shared memory over DSMEM
//     (mapa + st.shared::cluster) and the leader adds them in rank order
//     (deterministic) before the top-k -- C times the SMs streaming X.
#include <cudaTypedefs.h>
#include <float.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>
#include <vector>

#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

constexpr int kBlockM = 128;
// 8 warps join the top-K epilogue, two per TMEM lane quadrant, each scanning
// half of the expert columns (16 warps, a quarter each, measured equal: LM
// epilogue 5.0 vs 5.1 us)
constexpr int kThreads = 256;
constexpr int kParts = kThreads / 128;
// 32-deep k-blocks (64-byte rows, 64-byte swizzle): a stage is 8 KB of X +
// b_rows x 64 B of Wg (40 KB at E = 512), so five stages fit and the loads of
// four k-blocks are in flight while one is multiplied (at 64-deep stages only
// two 80 KB stages fit and the MMA waited on every load).
constexpr int kBlockK = 32;
constexpr int kMaxK = 8;
constexpr int kMaxSmem = 220 * 1024;
// split-K partial logits in the leader's smem start past the top-K merge
// scratch of the epilogue ((kParts - 1) x kBlockM x 8 x (4 + 4) bytes)
constexpr int kPartOffset = 16 * 1024;
// more stages (16) measured equal at MT and cfg1 (same box): the gate is not
// bound by loads in flight
#ifndef MOE_GATE_MAX_STAGES
#define MOE_GATE_MAX_STAGES 8
#endif
constexpr int kMaxStages = MOE_GATE_MAX_STAGES;
// MOE_GATE_PROF stamps per CTA: entry, after griddepcontrol.wait, first stage
// full (MMA thread), last MMA committed, accumulator ready (epilogue), end
constexpr int kProf = 6;
#ifndef MOE_GATE_TWO_PASS
#define MOE_GATE_TWO_PASS 1
#endif
constexpr bool kGateTwoPass = MOE_GATE_TWO_PASS;

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

// Top-K epilogue of one 128-token tile (all warps of the CTA): TMEM lane =
// token, columns = expert logits.  Warps q, q+4, ... share TMEM lane quadrant
// q (tokens 32q..32q+31), each scanning 1/kParts of the expert columns; the
// partial top-K lists are then merged
// through shared memory (the stage buffers, free once tfull fired).
// Split-K: `part` holds nparts follower partials, [part][token lane][pstride]
// floats; they are added to this CTA's TMEM logits in rank order.
__device__ __forceinline__ void reg_fence32(uint32_t (&r)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(r[i]));
}

template <int K>
__device__ __forceinline__ void gate_epilogue(const GateArgs& a, uint32_t tmem_base,
                                              uint64_t* tfull, int tok0, uint8_t* smem,
                                              const float* part = nullptr, int nparts = 0,
                                              int pstride = 0) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  ptx::mbar_wait(tfull, 0);
  ptx::tc_fence_after();
  if (a.prof && threadIdx.x == 0) a.prof[kProf * blockIdx.x + 4] = gate_clock();
  const int q = warp & 3;
  const int part_id = warp >> 2;  // column range of this warp
  const int tl = q * 32 + lane;  // token within the tile
  const int tok = tok0 + tl;
  const int nchunk = (a.E + 31) / 32;
  const int c_begin = part_id * nchunk / kParts * 32;
  const int c_end = (part_id + 1) * nchunk / kParts * 32;
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
  // TMEM loads are software-pipelined: the next 32 columns are in flight
  // while this chunk is scanned (tcgen05.wait::ld waits for every load of the
  // thread, so the load of chunk c+1 is issued right after chunk c's wait;
  // the empty asm pins chunk c's registers behind the wait)
  const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
  auto consume = [&](uint32_t (&r)[32], int c0) {
    for (int p = 0; p < nparts; ++p) {
      const float4* src = reinterpret_cast<const float4*>(part + (static_cast<size_t>(p) * kBlockM + tl) * pstride + c0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 v = src[i];
        r[4 * i] = __float_as_uint(__uint_as_float(r[4 * i]) + v.x);
        r[4 * i + 1] = __float_as_uint(__uint_as_float(r[4 * i + 1]) + v.y);
        r[4 * i + 2] = __float_as_uint(__uint_as_float(r[4 * i + 2]) + v.z);
        r[4 * i + 3] = __float_as_uint(__uint_as_float(r[4 * i + 3]) + v.w);
      }
    }
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
  };
  uint32_t ra[32], rb[32];
  int c0 = c_begin;
  if (a.dbg & 48) {  // epilogue ablations: 16 no TMEM loads, 32 no scan (wrong results)
#pragma unroll
    for (int i = 0; i < 32; ++i) ra[i] = __float_as_uint(static_cast<float>(i ^ lane));
    for (; c0 < c_end; c0 += 32) {
      if (!(a.dbg & 16)) {
        ptx::tmem_ld32(trow + c0, ra);
        ptx::tmem_ld_wait();
      }
      reg_fence32(ra);
      if (!(a.dbg & 32)) consume(ra, c0);
    }
    if (a.dbg & 32) bv[0] = __uint_as_float(ra[0] ^ ra[31]);
    c0 = c_end;
  }
  if constexpr (K == 2) {
    // Two-pass top-2 (the scan is issue-bound: ~14 instructions per column
    // in the one-pass form).  Pass 1: the two largest VALUES with min/max
    // only (5 per column pair, 3-input max); pass 2, over the columns again
    // from TMEM in descending order: the lowest id holding the top value and
    // the lowest other id holding the second (equal values -> lower id, as
    // in the one-pass lists).  Full 32-column chunks, no split-K partials
    // and no logits output only.
    if (kGateTwoPass && nparts == 0 && !a.logits && (a.E & 31) == 0 && !(a.dbg & 48)) {
      float m1 = -INFINITY, m2 = -INFINITY;
      auto max3 = [](float x, float y, float z) {
        float r;
        asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(x), "f"(y), "f"(z));
        return r;
      };
      auto values = [&](uint32_t (&r)[32]) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float v = __uint_as_float(r[i]), w = __uint_as_float(r[i + 1]);
          const float hi = fmaxf(v, w), lo = fminf(v, w);
          m2 = max3(m2, lo, fminf(hi, m1));
          m1 = max3(m1, v, w);
        }
      };
      if (c0 < c_end) ptx::tmem_ld32(trow + c0, ra);
      while (c0 < c_end) {
        ptx::tmem_ld_wait();
        reg_fence32(ra);
        if (c0 + 32 < c_end) ptx::tmem_ld32(trow + c0 + 32, rb);
        values(ra);
        c0 += 32;
        if (c0 >= c_end) break;
        ptx::tmem_ld_wait();
        reg_fence32(rb);
        if (c0 + 32 < c_end) ptx::tmem_ld32(trow + c0 + 32, ra);
        values(rb);
        c0 += 32;
      }
      const bool tie = m1 == m2;
      int i1 = 0x7fffffff, i2 = 0x7fffffff;
      auto ids = [&](uint32_t (&r)[32], int cb) {
#pragma unroll
        for (int i = 31; i >= 0; --i) {
          const float v = __uint_as_float(r[i]);
          const bool p1 = v == m1, p2 = v == m2;
          i2 = p2 ? (tie ? i1 : cb + i) : i2;
          i1 = p1 ? cb + i : i1;
        }
      };
      c0 = c_end - 32;
      if (c0 >= c_begin) ptx::tmem_ld32(trow + c0, ra);
      while (c0 >= c_begin) {
        ptx::tmem_ld_wait();
        reg_fence32(ra);
        if (c0 - 32 >= c_begin) ptx::tmem_ld32(trow + c0 - 32, rb);
        ids(ra, c0);
        c0 -= 32;
        if (c0 < c_begin) break;
        ptx::tmem_ld_wait();
        reg_fence32(rb);
        if (c0 - 32 >= c_begin) ptx::tmem_ld32(trow + c0 - 32, ra);
        ids(rb, c0);
        c0 -= 32;
      }
      bv[0] = m1;
      bv[1] = m2;
      bi[0] = i1;
      bi[1] = i2;
      c0 = c_end;  // the one-pass loop below is skipped; the odd list stays empty
    }
  }
  if (c0 < c_end) ptx::tmem_ld32(trow + c0, ra);
  while (c0 < c_end) {
    ptx::tmem_ld_wait();
    reg_fence32(ra);
    if (c0 + 32 < c_end) ptx::tmem_ld32(trow + c0 + 32, rb);
    consume(ra, c0);
    c0 += 32;
    if (c0 >= c_end) break;
    ptx::tmem_ld_wait();
    reg_fence32(rb);
    if (c0 + 32 < c_end) ptx::tmem_ld32(trow + c0 + 32, ra);
    consume(rb, c0);
    c0 += 32;
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
  // partial lists of parts 1.. -> smem (stage buffers are free: all TMA
  // writes landed and all MMAs retired before tfull fired; split-K partials
  // start at kPartOffset, past this scratch)
  float* pv = reinterpret_cast<float*>(smem);
  int* pi = reinterpret_cast<int*>(smem + (kParts - 1) * kBlockM * K * sizeof(float));
  if (part_id > 0) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      pv[((part_id - 1) * K + j) * kBlockM + tl] = bv[j];
      pi[((part_id - 1) * K + j) * kBlockM + tl] = bi[j];
    }
  }
  __syncthreads();
  if (part_id == 0 && tok < a.S) {
    // later parts hold larger ids, so inserting them part by part, each list
    // in its (value desc, id asc) order, keeps ties resolved toward the lower id
    for (int p = 0; p < kParts - 1; ++p)
#pragma unroll
      for (int j = 0; j < K; ++j)
        topk_insert<K>(bv, bi, pv[(p * K + j) * kBlockM + tl], pi[(p * K + j) * kBlockM + tl]);
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

}

// One 128-token tile of the gate: TMA + tcgen05 logits, top-K epilogue on all
// 8 warps, idx / w written to global.  Ends with a block barrier and the TMEM
// released.
//   SPLIT = false: a cluster of C CTAs = C consecutive tiles sharing Wg by
//                  multicast (C = 1, 2, 4);
//   SPLIT = true:  a cluster of C CTAs = one tile, CTA r covering k-blocks
//                  [r*KB/C, (r+1)*KB/C) (C = 2..8), partials reduced into the
//                  leader over DSMEM.
// 3-D views of X and Wg ({BK cols, rows, TD / BK k-blocks}, boxes of 128 /
// b_rows rows x 2 k-blocks): a 2-k-block stage's X and Wg as one request each
struct GateK2Maps {
  CUtensorMap x, w;
  int on;
};

template <int K, int C = 1, int BK = kBlockK, bool SPLIT = false>
__device__ __forceinline__ void gate_tile(const CUtensorMap& tmX, const CUtensorMap& tmWg,
                                          const GateK2Maps& k2m, const GateArgs& a, uint8_t* smem) {
  static_assert(SPLIT ? (C >= 2 && C <= 8) : (C == 1 || C == 2 || C == 4), "cluster shape");
  static_assert(BK == 32 || BK == 64, "32-deep (64-byte swizzle) or 64-deep (128-byte) k-blocks");
  constexpr int kABytes = kBlockM * BK * 2;
  if (a.prof && threadIdx.x == 0) a.prof[kProf * blockIdx.x] = gate_clock();
  const GateLayout L = gate_layout(a.E, BK);
  const int stage_bytes = kABytes + L.b_rows * BK * 2;  // one k-block (X box + Wg boxes)
  // k-blocks per pipeline stage (one barrier phase): more bytes per phase
  // keep more of one SM's TMA stream in flight (tools/probes/tma_l2_probe.cu)
  const int kps = (a.kps > 1 && L.stages >= 2 * a.kps) ? a.kps : 1;
  const int nstages = L.stages / kps;
  // stage s holds its kps X boxes, then their kps Wg slabs
  const int w_bytes = L.b_rows * BK * 2;
  auto x_at = [&](int st, int j) { return smem + st * kps * stage_bytes + j * kABytes; };
  auto w_at = [&](int st, int j) { return smem + st * kps * stage_bytes + kps * kABytes + j * w_bytes; };
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.stages * stage_bytes);
  uint64_t* empty = full + L.stages;
  uint64_t* tfull = empty + L.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  uint64_t* pbar = tfull + 2;  // split-K: the followers' partials landed (leader)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int crank = C > 1 ? static_cast<int>(ptx::cluster_ctarank()) : 0;
  const int tok0 = (SPLIT ? blockIdx.x / C : blockIdx.x) * kBlockM;
  const int KB_all = a.TD / BK;
  const int kb_lo = SPLIT ? crank * KB_all / C : 0;
  const int kb_hi = SPLIT ? (crank + 1) * KB_all / C : KB_all;
  auto desc = [](uint32_t addr) {
    return BK == 64 ? ptx::umma_desc_sw128(addr) : ptx::umma_desc_sw64(addr);
  };

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmX);
    ptx::prefetch_tmap(&tmWg);
    for (int s = 0; s < L.stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], SPLIT ? 1 : C);  // one MMA commit from every CTA that reads the stage
    }
    ptx::mbar_init(tfull, 1);
    if (SPLIT) ptx::mbar_init(pbar, 1);
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
  if (a.prof && threadIdx.x == 0) a.prof[kProf * blockIdx.x + 1] = gate_clock();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------- TMA producer
      // (one issuing thread: rotating the stage's requests over the warp's
      // lanes measured equal, LM 13.3 vs 13.4 us mainloop, same box)
      const uint64_t pol_x = a.x_keep ? ptx::policy_evict_last() : ptx::policy_evict_first();
      const uint64_t pol_w = ptx::policy_evict_last();
      // this CTA's share of the Wg boxes (all of them without multicast)
      constexpr int MC = SPLIT ? 1 : C;  // CTAs sharing each Wg box
      const int per = L.n_box / MC;
      const int b_lo = MC > 1 ? crank * per : 0;
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb_lo; kb < kb_hi; kb += kps) {
        const int nk = min(kps, kb_hi - kb);  // k-blocks in this stage
        // free once every CTA of the cluster has consumed the stage
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (a.dbg & 2) {  // ablation: no loads at all
          ptx::mbar_arrive(&full[stage]);
        } else {
          ptx::mbar_arrive_expect_tx(&full[stage], nk * (stage_bytes - ((a.dbg & 4) ? L.b_rows * BK * 2 : 0) -
                                                         ((a.dbg & 8) ? kABytes : 0)));
          if (MC == 1 && k2m.on && nk == kps) {
            // all k-blocks of the stage: one X request, one Wg request
            if (!(a.dbg & 8)) ptx::tma_load_3d(x_at(stage, 0), &k2m.x, &full[stage], 0, tok0, kb, pol_x);
            if (!(a.dbg & 4)) ptx::tma_load_3d(w_at(stage, 0), &k2m.w, &full[stage], 0, 0, kb, pol_w);
          } else {
            for (int j = 0; j < nk; ++j) {
              if (!(a.dbg & 8)) ptx::tma_load_2d(x_at(stage, j), &tmX, &full[stage], (kb + j) * BK, tok0, pol_x);
              for (int b = b_lo; b < b_lo + per && !(a.dbg & 4); ++b) {
                const int r = b * L.box_rows;
                if (MC > 1)
                  ptx::tma_load_2d_mc(w_at(stage, j) + r * BK * 2, &tmWg, &full[stage], (kb + j) * BK, r,
                                      static_cast<uint16_t>((1u << MC) - 1), pol_w);
                else
                  ptx::tma_load_2d(w_at(stage, j) + r * BK * 2, &tmWg, &full[stage], (kb + j) * BK, r, pol_w);
              }
            }
          }
        }
        if (++stage == nstages) {
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
      for (int kb0 = kb_lo; kb0 < kb_hi; kb0 += kps) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        if (a.prof && kb0 == kb_lo) a.prof[kProf * blockIdx.x + 2] = gate_clock();
        for (int kb = kb0; kb < min(kb0 + kps, kb_hi); ++kb) {
        const uint32_t a0 = ptx::smem_u32(x_at(stage, kb - kb0));
        const uint32_t b0 = ptx::smem_u32(w_at(stage, kb - kb0));
#pragma unroll
        for (int kk = 0; kk < BK / 16 && !(a.dbg & 1); ++kk) {
          const uint32_t acc = (kb != kb_lo || kk != 0) ? 1u : 0u;
          ptx::mma_bf16(tmem_base, desc(a0 + kk * 32), desc(b0 + kk * 32), id0, acc);
          if (n1 > 0)
            ptx::mma_bf16(tmem_base + 256, desc(a0 + kk * 32), desc(b0 + 256 * BK * 2 + kk * 32), id1,
                          acc);
        }
        }
        if (!SPLIT && C > 1)
          ptx::mma_commit_mc(&empty[stage], static_cast<uint16_t>((1u << C) - 1));
        else
          ptx::mma_commit(&empty[stage]);
        if (++stage == nstages) {
          stage = 0;
          phase ^= 1;
        }
      }
      ptx::mma_commit(tfull);
      if (a.prof) a.prof[kProf * blockIdx.x + 3] = gate_clock();
    }
    __syncwarp();
  }

  if constexpr (SPLIT) {
    // Followers: TMEM partial logits -> own smem (their stage buffers are free
    // once their tfull fired), then ONE bulk DSMEM copy into the leader's
    // partial slot, counted on the leader's pbar.  The cluster barrier in
    // between keeps the copies out of the leader's stage buffers until the
    // leader's MMAs retired.  (Per-thread st.shared::cluster stores of the
    // same 64 KB took ~4 us at MT; one bulk copy per follower streams it.)
    const int pstride = (a.E + 31) / 32 * 32 + 4;  // floats per token row (+4: bank spread)
    const uint32_t part_bytes = static_cast<uint32_t>(kBlockM * pstride * 4);
    float* part = reinterpret_cast<float*>(smem + kPartOffset);
    ptx::mbar_wait(tfull, 0);
    ptx::tc_fence_after();
    if (crank != 0) {
      const int q = warp & 3, part_id = warp >> 2, tl = q * 32 + lane;
      const int nchunk = (a.E + 31) / 32;
      const int c_begin = part_id * nchunk / kParts * 32, c_end = (part_id + 1) * nchunk / kParts * 32;
      float* row = reinterpret_cast<float*>(smem) + static_cast<size_t>(tl) * pstride;
      for (int c0 = c_begin; c0 < c_end; c0 += 32) {
        uint32_t r[32];
        ptx::tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + c0, r);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<uint4*>(row + c0 + 4 * i) = make_uint4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
      }
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
    } else if (threadIdx.x == 0) {
      ptx::mbar_arrive_expect_tx(pbar, (C - 1) * part_bytes);
    }
    __syncthreads();
    ptx::cluster_sync();  // leader's stage buffers free; every follower's rows staged
    if (crank != 0 && threadIdx.x == 0)
      ptx::bulk_copy_to_cluster(ptx::cluster_map(ptx::smem_u32(part) + (crank - 1) * part_bytes, 0), smem,
                                part_bytes, ptx::cluster_map(ptx::smem_u32(pbar), 0));
    if (crank == 0) {
      ptx::mbar_wait(pbar, 0);
      gate_epilogue<K>(a, tmem_base, tfull, tok0, smem, part, C - 1, pstride);
    }
  } else {
    gate_epilogue<K>(a, tmem_base, tfull, tok0, smem);
  }

  __syncthreads();
  if (a.prof && threadIdx.x == 0) a.prof[kProf * blockIdx.x + 5] = gate_clock();
  ptx::tc_fence_after();
  if (warp == 2) {
    if (L.e_pad <= 32) ptx::tmem_dealloc<32>(tmem_base);
    else if (L.e_pad <= 64) ptx::tmem_dealloc<64>(tmem_base);
    else if (L.e_pad <= 128) ptx::tmem_dealloc<128>(tmem_base);
    else if (L.e_pad <= 256) ptx::tmem_dealloc<256>(tmem_base);
    else ptx::tmem_dealloc<512>(tmem_base);
  }
  // peers' last MMA commits arrive on this CTA's empty barriers, and the
  // followers' smem is the source of bulk copies until the leader saw pbar:
  // stay alive
  if (C > 1) ptx::cluster_sync();
}

__device__ __forceinline__ uint8_t* aligned_smem() {
  extern __shared__ uint8_t smem_raw[];
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                    ~static_cast<uintptr_t>(1023));
}

template <int K, int C, int BK, bool SPLIT>
__global__ void __launch_bounds__(kThreads, 1)
    gate_topk_kernel(const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ CUtensorMap tmWg, const __grid_constant__ GateK2Maps k2m,
                     GateArgs a) {
  gate_tile<K, C, BK, SPLIT>(tmX, tmWg, k2m, a, aligned_smem());
}

template <int C, int BK, bool SPLIT = false>
const void* gate_fn(int k) {
  return k == 1   ? reinterpret_cast<const void*>(gate_topk_kernel<1, C, BK, SPLIT>)
         : k == 2 ? reinterpret_cast<const void*>(gate_topk_kernel<2, C, BK, SPLIT>)
         : k <= 4 ? reinterpret_cast<const void*>(gate_topk_kernel<4, C, BK, SPLIT>)
                  : reinterpret_cast<const void*>(gate_topk_kernel<8, C, BK, SPLIT>);
}

const void* split_fn(int C, int k) {
  switch (C) {
    case 2: return gate_fn<2, 64, true>(k);
    case 3: return gate_fn<3, 64, true>(k);
    case 4: return gate_fn<4, 64, true>(k);
    default: return gate_fn<8, 64, true>(k);
  }
}

// ---------------------------------------------------------------- small-E gate
// Few experts (E <= 32: configs[0]'s E = 8): the gate is a bandwidth-bound
// GEMV-like pass over X (2 * E flop per byte of X), so it runs on the CUDA
// cores instead of tcgen05: no TMEM allocation, TMA pipeline or cluster
// barriers (whose fixed costs were ~5 us of the 9 us tcgen05 gate at
// configs[0]).  Wg [E, TD] is staged in shared memory BEFORE
// griddepcontrol.wait (weights are never written by the previous kernel of
// the chain); one warp per token then streams its X row with 16-byte loads,
// keeps E fp32 partial sums per lane, all-reduces them with butterflies and
// applies the same top-k / weight rule as the tcgen05 epilogue.
constexpr int kSmallMaxE = 32;
constexpr int kSmallThreads = 512;
constexpr int kSmallMaxSmem = 64 * 1024;
constexpr int kSmallMaxVec = 16;  // 16-byte vectors of an X row per lane: TD <= 4096

__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float (&f)[8]) {
  const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(u[i] << 16);
    f[2 * i + 1] = __uint_as_float(u[i] & 0xffff0000u);
  }
}

template <int EM, int K>
__global__ void __launch_bounds__(kSmallThreads) gate_small_kernel(GateArgs a) {
  extern __shared__ uint4 swg[];  // Wg [E][TD] bf16
  const int vpr = a.TD / 8;       // 16-byte vectors per row
  const uint4* wg = reinterpret_cast<const uint4*>(a.Wg);
  // Wg -> smem with cp.async: the copies are in flight while this warp waits
  // for the previous kernel and then loads its first X row
  for (int i = threadIdx.x; i < a.E * vpr; i += blockDim.x)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(swg + i)), "l"(wg + i)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
  pdl_trigger();
  pdl_wait();  // X belongs to the previous kernel until here
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int stride = gridDim.x * wpb;
  int t = blockIdx.x * wpb + (threadIdx.x >> 5);
  // this lane's 16-byte vectors of the current X row: the smem bound
  // (E * TD * 2 <= 64 KB) caps TD at 4096 / 2048 / 1024 for EM = 8 / 16 / 32
  constexpr int NV = kSmallMaxVec * 8 / EM;
  uint4 xv[NV];
  auto load_x = [&](int tt) {
    const uint4* xr = reinterpret_cast<const uint4*>(a.X) + static_cast<size_t>(tt) * vpr;
#pragma unroll
    for (int u = 0; u < NV; ++u)
      if (lane + 32 * u < vpr) xv[u] = __ldcs(xr + lane + 32 * u);
  };
  if (t < a.S) load_x(t);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  for (; t < a.S; t += stride) {
    float acc[EM];
#pragma unroll
    for (int e = 0; e < EM; ++e) acc[e] = 0.f;
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int v = lane + 32 * u;
      if (v >= vpr) break;
      float xf[8];
      bf16x8_to_f32(xv[u], xf);
#pragma unroll
      for (int e = 0; e < EM; ++e) {
        if (e < a.E) {
          float wf[8];
          bf16x8_to_f32(swg[e * vpr + v], wf);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[e] = fmaf(xf[i], wf[i], acc[e]);
        }
      }
    }
    if (t + stride < a.S) load_x(t + stride);  // the next row is in flight during the reduction
#pragma unroll
    for (int e = 0; e < EM; ++e)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    // every lane holds all E logits: same selection as gate_epilogue
    float bv[K];
    int bi[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      bv[j] = -INFINITY;
      bi[j] = 0x7fffffff;
    }
#pragma unroll
    for (int e = 0; e < EM; ++e)
      if (e < a.E) topk_insert<K>(bv, bi, acc[e], e);
    if (a.logits) {
#pragma unroll
      for (int e = 0; e < EM; ++e)
        if (e == lane && e < a.E) a.logits[static_cast<size_t>(t) * a.E + e] = acc[e];
    }
    if (lane == 0) {
      const int k = a.k;
      float ex[K];
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        ex[j] = (j < k) ? expf(bv[j] - bv[0]) : 0.f;
        sum += ex[j];
      }
      float accw = 0.f;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (j < k) {
          const float wj = (j < k - 1) ? ex[j] / sum : 1.f - accw;
          accw += wj;
          a.idx[static_cast<size_t>(t) * k + j] = bi[j];
          a.w[static_cast<size_t>(t) * k + j] = wj;
        }
      }
    }
  }
}

template <int EM>
cudaError_t launch_gate_small_e(const GateArgs& a, int grid, int smem, cudaStream_t stream) {
  const dim3 g(grid), b(kSmallThreads);
  if (a.k == 1) return launch_chain(gate_small_kernel<EM, 1>, g, b, smem, stream, false, a);
  if (a.k == 2) return launch_chain(gate_small_kernel<EM, 2>, g, b, smem, stream, false, a);
  if (a.k <= 4) return launch_chain(gate_small_kernel<EM, 4>, g, b, smem, stream, false, a);
  return launch_chain(gate_small_kernel<EM, 8>, g, b, smem, stream, false, a);
}

// every gate kernel may use up to the layout maximum (stages are sized to
// kMaxSmem); one attribute value for all of them
constexpr int kSmemAttr = kMaxSmem + 4096;

}  // namespace

int gate_box_rows(int E) { return gate_layout(E).box_rows; }
// 64-deep k-blocks with 128-byte rows for E <= 128 (a 32 KB stage at E = 128,
// six stages): 32-deep boxes of 64-byte rows streamed X at ~35-65 GB/s per SM
// (MOE_GATE_PROF); E > 128 keeps 32 (a 64-deep stage at E = 512 is 80 KB: two
// stages).  MOE_GATE_WIDE=0 restores 32 everywhere (A/B).
bool gate_wide(int E) {
  static const int env = [] {
    const char* v = getenv("MOE_GATE_WIDE");
    return v ? atoi(v) : 1;
  }();
  return env != 0 && gate_layout(E).e_pad <= 128;
}
int gate_box_cols(int E) { return gate_wide(E) ? 64 : kBlockK; }

cudaError_t gate_prepare(int E) {
  (void)E;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    std::vector<const void*> fns;
    for (int k : {1, 2, 4, 8}) {
      for (const void* fn : {gate_fn<1, kBlockK>(k), gate_fn<2, kBlockK>(k), gate_fn<4, kBlockK>(k),
                             gate_fn<1, 64>(k), gate_fn<2, 64>(k), gate_fn<4, 64>(k)})
        fns.push_back(fn);
      for (int C : {2, 3, 4, 8}) fns.push_back(split_fn(C, k));
    }
    for (const void* fn : fns) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAttr);
      if (e != cudaSuccess && err == cudaSuccess) err = e;
    }
    const void* small[] = {
        reinterpret_cast<const void*>(gate_small_kernel<8, 1>), reinterpret_cast<const void*>(gate_small_kernel<8, 2>),
        reinterpret_cast<const void*>(gate_small_kernel<8, 4>), reinterpret_cast<const void*>(gate_small_kernel<8, 8>),
        reinterpret_cast<const void*>(gate_small_kernel<16, 1>), reinterpret_cast<const void*>(gate_small_kernel<16, 2>),
        reinterpret_cast<const void*>(gate_small_kernel<16, 4>), reinterpret_cast<const void*>(gate_small_kernel<16, 8>),
        reinterpret_cast<const void*>(gate_small_kernel<32, 1>), reinterpret_cast<const void*>(gate_small_kernel<32, 2>),
        reinterpret_cast<const void*>(gate_small_kernel<32, 4>), reinterpret_cast<const void*>(gate_small_kernel<32, 8>)};
    for (const void* fn : small) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallMaxSmem);
      if (e != cudaSuccess && err == cudaSuccess) err = e;
    }
  });
  return err;
}

namespace {

bool clusters_fit(const void* fn, int C, int clusters, int smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * C);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = C;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return n >= clusters;
}

// Multicast cluster size: the largest C | n_box (<= MOE_GATE_CLUSTER, default
// 4) for which every cluster of the grid is co-resident (one wave).
int gate_cluster(const GateLayout& L, int tiles, bool wide) {
  static int env = -1;
  if (env < 0) {
    const char* v = getenv("MOE_GATE_CLUSTER");
    env = v ? atoi(v) : 4;
  }
  for (int C = 4; C >= 2; C >>= 1) {
    if (C > env || L.n_box % C != 0 || tiles < C) continue;
    const void* fn = wide ? (C == 4 ? gate_fn<4, 64>(2) : gate_fn<2, 64>(2))
                          : (C == 4 ? gate_fn<4, kBlockK>(2) : gate_fn<2, kBlockK>(2));
    if (clusters_fit(fn, C, (tiles + C - 1) / C, L.smem)) return C;
  }
  return 1;
}

// Split-K cluster size: with fewer tiles than half the SMs (MT: 48, cfg1: 16
// of 148) a tile is shared by C CTAs along the token dimension, the largest
// C in {8, 4, 3, 2} with tiles * C <= SMs, >= 1 k-block per CTA, the
// followers' partials fitting the leader's stage buffers and all clusters
// co-resident.  MOE_GATE_SPLIT=0 disables (A/B), =C forces an upper bound.
int gate_split(int E, int TD, int tiles, int sms) {
  static const int env = [] {
    const char* v = getenv("MOE_GATE_SPLIT");
    return v ? atoi(v) : 8;
  }();
  if (!gate_wide(E) || tiles * 2 > sms || TD % 64) return 1;
  const GateLayout L = gate_layout(E, 64);
  const int stage_bytes = kBlockM * 64 * 2 + L.b_rows * 64 * 2;
  const int pstride = (E + 31) / 32 * 32 + 4;
  for (int C : {8, 4, 3, 2}) {
    if (C > env || tiles * C > sms || TD / 64 < C) continue;
    if (kPartOffset + (C - 1) * kBlockM * pstride * 4 > L.stages * stage_bytes) continue;
    if (clusters_fit(split_fn(C, 2), C, tiles, L.smem)) return C;
  }
  return 1;
}

template <int K, int BK>
cudaError_t launch_gate_k(const CUtensorMap& tmX, const CUtensorMap& tmWg, const GateK2Maps& k2m, const GateArgs& a,
                          int C, bool split, int tiles, int smem, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(split ? tiles * C : (tiles + C - 1) / C * C);
  cfg.blockDim = dim3(kThreads);
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
  if (split) {
    if constexpr (BK == 64) {
      switch (C) {
        case 2: return cudaLaunchKernelEx(&cfg, gate_topk_kernel<K, 2, 64, true>, tmX, tmWg, k2m, a);
        case 3: return cudaLaunchKernelEx(&cfg, gate_topk_kernel<K, 3, 64, true>, tmX, tmWg, k2m, a);
        case 4: return cudaLaunchKernelEx(&cfg, gate_topk_kernel<K, 4, 64, true>, tmX, tmWg, k2m, a);
        default: return cudaLaunchKernelEx(&cfg, gate_topk_kernel<K, 8, 64, true>, tmX, tmWg, k2m, a);
      }
    }
    return cudaErrorInvalidValue;
  }
  if (C == 4) return cudaLaunchKernelEx(&cfg, gate_topk_kernel<K, 4, BK, false>, tmX, tmWg, k2m, a);
  if (C == 2) return cudaLaunchKernelEx(&cfg, gate_topk_kernel<K, 2, BK, false>, tmX, tmWg, k2m, a);
  return cudaLaunchKernelEx(&cfg, gate_topk_kernel<K, 1, BK, false>, tmX, tmWg, k2m, a);
}

template <int BK>
cudaError_t launch_gate_bk(const CUtensorMap& tmX, const CUtensorMap& tmWg, const GateK2Maps& k2m, const GateArgs& a, int C,
                           bool split, int tiles, int smem, cudaStream_t stream) {
  if (a.k == 1) return launch_gate_k<1, BK>(tmX, tmWg, k2m, a, C, split, tiles, smem, stream);
  if (a.k == 2) return launch_gate_k<2, BK>(tmX, tmWg, k2m, a, C, split, tiles, smem, stream);
  if (a.k <= 4) return launch_gate_k<4, BK>(tmX, tmWg, k2m, a, C, split, tiles, smem, stream);
  return launch_gate_k<8, BK>(tmX, tmWg, k2m, a, C, split, tiles, smem, stream);
}

}  // namespace

bool gate_small(int E, int TD) {
  static const int env = [] {
    const char* v = getenv("MOE_GATE_SMALL");
    return v ? atoi(v) : 1;
  }();
  const int em = E <= 8 ? 8 : E <= 16 ? 16 : 32;  // the kernel's E bucket
  return env != 0 && E <= kSmallMaxE && TD % 8 == 0 && TD / 8 <= 32 * (kSmallMaxVec * 8 / em) &&
         E * TD * 2 <= kSmallMaxSmem;
}

// The 3-D X / Wg views of a 64-deep, two-k-blocks-per-stage launch, cached per
// (X, Wg, S, TD, E) (encoding is host work; graph replays reuse the captured
// parameters).  MOE_GATE_K2=0 disables.  False when unavailable.
bool gate_k2_maps(GateK2Maps* m, const void* X, const void* Wg, int S, int TD, int E, int b_rows, int depth) {
  static const bool enabled = [] {
    const char* v = getenv("MOE_GATE_K2");
    return !v || atoi(v) != 0;
  }();
  if (!enabled || TD % 64) return false;
  using Key = std::tuple<const void*, const void*, int, int, int, int>;
  static std::mutex mu;
  static std::map<Key, std::pair<CUtensorMap, CUtensorMap>> cache;
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!enc) return false;
  std::lock_guard<std::mutex> lock(mu);
  const Key key{X, Wg, S, TD, E, depth};
  auto it = cache.find(key);
  if (it == cache.end()) {
    if (cache.size() > 256) cache.clear();
    std::pair<CUtensorMap, CUtensorMap> v;
    auto encode = [&](CUtensorMap* t, const void* p, int rows, int box_rows) {
      cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(TD / 64)};
      cuuint64_t strides[2] = {(cuuint64_t)TD * 2, 128};
      cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)depth};
      cuuint32_t estr[3] = {1, 1, 1};
      return enc(t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(p), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (!encode(&v.first, X, S, kBlockM) || !encode(&v.second, Wg, E, b_rows)) return false;
    it = cache.emplace(key, v).first;
  }
  m->x = it->second.first;
  m->w = it->second.second;
  return true;
}

cudaError_t launch_gate(const CUtensorMap& tmX, const CUtensorMap& tmWg, const GateArgs& a,
                        cudaStream_t stream) {
  if (a.X && a.Wg && a.k >= 1 && a.k <= kMaxK && a.E >= a.k && gate_small(a.E, a.TD)) {
    static int sms_of[64] = {0};  // SM count per device (queried once)
    int dev = 0;
    cudaGetDevice(&dev);
    int& sms = sms_of[dev & 63];
    if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int wpb = kSmallThreads / 32;
    const int grid = std::max(1, std::min((a.S + wpb - 1) / wpb, 2 * sms));
    const int smem = a.E * a.TD * 2;
    if (a.E <= 8) return launch_gate_small_e<8>(a, grid, smem, stream);
    if (a.E <= 16) return launch_gate_small_e<16>(a, grid, smem, stream);
    return launch_gate_small_e<32>(a, grid, smem, stream);
  }
  const bool wide = gate_wide(a.E);
  if (a.k < 1 || a.k > kMaxK || a.E > 512 || a.E < a.k || (a.TD % (wide ? 64 : kBlockK)) != 0)
    return cudaErrorInvalidValue;
  const GateLayout L = gate_layout(a.E, wide ? 64 : kBlockK);
  const int tiles = (a.S + kBlockM - 1) / kBlockM;
  // grid shape cached per (E, TD, tiles): the occupancy queries are not free
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, std::pair<int, bool>> cache;
  std::pair<int, bool> shape;
  {
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(a.E, a.TD, tiles);
    auto it = cache.find(key);
    if (it == cache.end()) {
      int dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int Cs = gate_split(a.E, a.TD, tiles, sms);
      it = cache.emplace(key, Cs > 1 ? std::make_pair(Cs, true)
                                     : std::make_pair(gate_cluster(L, tiles, wide), false)).first;
    }
    shape = it->second;
  }
  const int C = shape.first;
  const bool split = shape.second;
  static const bool prof = getenv("MOE_GATE_PROF") != nullptr;
  static const int dbg = getenv("MOE_GATE_DBG") ? atoi(getenv("MOE_GATE_DBG")) : 0;
  GateArgs b = a;
  b.dbg = dbg;
  static const int kps_env = [] {
    const char* v = getenv("MOE_GATE_KPS");
    return v ? atoi(v) : 0;
  }();
  // measured (ncu, same box): 64-deep path (MT) 2 per stage 16.4 vs 17.5 us
  // (1) / 17.7 (3); 32-deep E = 512 path (LM) 1 per stage 24.8 vs 28.5 (2)
  b.kps = kps_env > 0 ? kps_env : (wide ? 2 : 1);
  // X tiles stay in L2 for the gather, which re-reads X right after the route
  // (same box: LM gather 17.9 -> 16.5 us, MT 16.2 -> 15.3 us; Xp stored with
  // evict-last for the FFN measured no change).  MOE_GATE_X_EVICT_FIRST=1 restores.
  static const bool x_first = getenv("MOE_GATE_X_EVICT_FIRST") && atoi(getenv("MOE_GATE_X_EVICT_FIRST"));
  b.x_keep = x_first ? 0 : 1;
  static unsigned long long* prof_buf = nullptr;
  const int ctas = split ? tiles * C : tiles;
  if (prof) {
    if (!prof_buf) cudaMalloc(&prof_buf, kProf * 4096 * sizeof(unsigned long long));
    if (prof_buf) cudaMemsetAsync(prof_buf, 0, kProf * 4096 * sizeof(unsigned long long), stream);
    b.prof = ctas <= 4096 ? prof_buf : nullptr;
  }
  GateK2Maps k2m;
  k2m.on = 0;
  if (wide && b.kps >= 2 && L.stages >= 2 * b.kps && (split || C == 1) && L.b_rows <= 256 && a.X && a.Wg)
    k2m.on = gate_k2_maps(&k2m, a.X, a.Wg, a.S, a.TD, a.E, L.b_rows, b.kps) ? 1 : 0;
  const cudaError_t e = wide ? launch_gate_bk<64>(tmX, tmWg, k2m, b, C, split, tiles, L.smem, stream)
                             : launch_gate_bk<kBlockK>(tmX, tmWg, k2m, b, C, split, tiles, L.smem, stream);
  if (!b.prof || e != cudaSuccess) return e;
  // experiments only: mean per-CTA phase times of this launch (split
  // followers have no epilogue stamps and are left out)
  std::vector<unsigned long long> h(kProf * (size_t)ctas);
  cudaStreamSynchronize(stream);
  cudaMemcpy(h.data(), prof_buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull, t5 = 0;
  double ph[kProf - 1] = {0, 0, 0, 0, 0};
  int nl = 0;
  for (int i = 0; i < ctas; ++i) {
    if (split && i % C) continue;
    const unsigned long long* p = &h[kProf * (size_t)i];
    ++nl;
    t0 = std::min(t0, p[0]);
    t5 = std::max(t5, p[5]);
    for (int j = 0; j < kProf - 1; ++j) ph[j] += (double)(p[j + 1] - p[j]);
  }
  if (const char* path = getenv("MOE_GATE_PROF_DUMP")) {  // raw stamps, one CTA per line
    if (FILE* f = fopen(path, "a")) {
      for (int i = 0; i < ctas; ++i) {
        fprintf(f, "%d", i);
        for (int j = 0; j < kProf; ++j) fprintf(f, " %llu", h[kProf * (size_t)i + j] - t0);
        fprintf(f, "\n");
      }
      fprintf(f, "--\n");
      fclose(f);
    }
  }
  fprintf(stderr,
          "[gate prof] %d CTAs (cluster %d, %s): mean us: pdl-wait %.1f | first stage %.1f | MMA loop %.1f | "
          "to acc-ready %.1f | epilogue %.1f ; span %.1f\n",
          ctas, C, split ? "split-K" : "multicast", ph[0] / nl * 1e-3, ph[1] / nl * 1e-3, ph[2] / nl * 1e-3,
          ph[3] / nl * 1e-3, ph[4] / nl * 1e-3, (t5 - t0) * 1e-3);
  return e;
}

}  // namespace moe
