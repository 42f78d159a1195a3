// Fused expert FFN on CTA pairs: the same interleaved GEMM1/GEMM2 tile
// sequence as ffn_fused.cu (H kept in L2, per-item done counters, discard of
// consumed H lines), but every tile is a 256-row weight block computed by a
// 2-SM UMMA (tcgen05.mma.cta_group::2, M = 256).
//
// Why: at n_e ~ 64 tokens per expert the FFN streams weights and re-reads
// each expert's token rows (Xp for GEMM1, H for GEMM2) once per 128-row weight
// block.  With the pair, each CTA stages its own 128 weight rows (A) but only
// HALF of the token rows (B is split along N across the two CTAs), so the
// L2->SM token traffic per weight byte halves and one MMA instruction covers
// both SMs.  The smaller B footprint also leaves room for four 32 KB weight
// stages per SM (128 KB of weights in flight).
//
// Pair protocol (cluster of 2; rank 0 = leader):
//   * both CTAs' producers TMA their halves with .cta_group::2, completing on
//     the LEADER's full barrier; the leader's producer alone arms it with the
//     bytes of both CTAs;
//   * the leader's MMA thread issues the M=256 MMAs and commits (multicast)
//     to the empty barrier of both CTAs and, per tile, to both tfull barriers;
//   * each CTA's epilogue drains its own TMEM (its 128 weight rows x all N
//     token columns) and arrives on the leader's tempty barrier (count 8).
#include <cstdio>
#include <cstdlib>

#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

constexpr int kBlockM = 128;  // weight rows per CTA (256 per pair)
constexpr int kChunkK = 64;
constexpr int kUmmaK = 16;
constexpr int kEpiBytes = 4 * 32 * 32 * 2;
constexpr int kAChunk = kBlockM * kChunkK * 2;      // 16 KB

// BN = max tokens per work item (tile_n, 128 or 256); each CTA of the pair
// stages half of the item's token rows.
template <int BN, int STAGES, int KCH>
struct PairCfg {
  static_assert(KCH % 2 == 0, "packed weights: 256-row (two-tile) boxes");
  static constexpr int kBN = BN;
  static constexpr int kBChunk = (BN / 2) * kChunkK * 2;  // half of the token rows
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kStages = STAGES;
  static constexpr int kKch = KCH;  // 64-wide k-chunks per stage
  static constexpr int kStageK = KCH * kChunkK;
  static constexpr int kABytes = KCH * kAChunk;
  static constexpr int kBBytes = KCH * kBChunk;
  static constexpr int kSmem =
      1024 + STAGES * (kABytes + kBBytes) + kEpiBytes + (2 * STAGES + 4) * 8 + 16;
};

struct TileRef {
  int item;
  int gemm;
  int mp;  // 256-row weight block (pair of 128-row blocks)
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ TileRef decode_tile(int t, int n, int L, int P1, int P2) {
  const int head = L * P1;
  if (t < head) return {t / P1, 0, t % P1};
  const int per = P1 + P2;
  const int body = head + (n - L) * per;
  if (t < body) {
    const int u = t - head;
    const int g = L + u / per;
    const int r = u % per;
    if (r < P1) return {g, 0, r};
    return {g - L, 1, r - P1};
  }
  const int u = t - body;
  return {n - L + u / P2, 1, u % P2};
}

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// shared::cluster address of the same smem object in the leader CTA (rank 0)
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(ptx::smem_u32(p)));
  return r;
}

// TMA 2-D load into this CTA's smem, completion counted on the leader's barrier.
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* m,
                                                 uint32_t leader_bar, int32_t c0, int32_t c1,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(ptx::smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// arrive on the barrier at this smem offset in both CTAs of the pair
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(ptx::smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

__device__ __forceinline__ void arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar)
               : "memory");
}

__device__ __forceinline__ void tma_load_3d_pair(void* smem_dst, const CUtensorMap* m,
                                                 uint32_t leader_bar, int32_t c0, int32_t c1, int32_t c2,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(ptx::smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}

// rows [r0, r0 + h) of B (h % 8 == 0) into dst with 64/32/16/8-row boxes
__device__ __forceinline__ void load_rows(uint8_t* dst, const RowMaps* m, uint32_t bar, int k0,
                                          int r0, int h, uint64_t pol) {
  int r = 0;
  for (; r + 64 <= h; r += 64) tma_load_2d_pair(dst + r * 128, &m->m64, bar, k0, r0 + r, pol);
  if (r + 32 <= h) {
    tma_load_2d_pair(dst + r * 128, &m->m32, bar, k0, r0 + r, pol);
    r += 32;
  }
  if (r + 16 <= h) {
    tma_load_2d_pair(dst + r * 128, &m->m16, bar, k0, r0 + r, pol);
    r += 16;
  }
  if (r < h) tma_load_2d_pair(dst + r * 128, &m->m8, bar, k0, r0 + r, pol);
}

template <int BN, int STAGES, int KCH>
__global__ void __launch_bounds__(256, 1)
    fused_ffn_pair_kernel(const __grid_constant__ CUtensorMap tmW1,
                          const __grid_constant__ RowMaps xpm,
                          const __grid_constant__ CUtensorMap tmW2,
                          const __grid_constant__ RowMaps hm, FusedFfnArgs g) {
  using Cfg = PairCfg<BN, STAGES, KCH>;
  constexpr int kStages = Cfg::kStages, kKch = Cfg::kKch, kStageK = Cfg::kStageK;
  constexpr int kABytes = Cfg::kABytes, kBBytes = Cfg::kBBytes;
  constexpr int kBN = Cfg::kBN, kBChunk = Cfg::kBChunk, kTmemCols = Cfg::kTmemCols;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + kStages * kABytes;
  __nv_bfloat16* sEpi = reinterpret_cast<__nv_bfloat16*>(sB + kStages * kBBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sEpi) + kEpiBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ int last_consumer;
  // dynamic tail (as ffn_fused.cu): the leader's producer claims the tail's
  // pair-tiles from a global counter and hands them to its MMA / epilogue
  // warps and to the peer's producer / epilogue warps through this ring
  constexpr int kRing = 4;
  __shared__ int ring_t[kRing];
  __shared__ __align__(8) uint64_t ring_full[kRing], ring_empty[kRing];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmW1);
    ptx::prefetch_tmap(&tmW2);
    for (const RowMaps* m : {&xpm, &hm}) {
      ptx::prefetch_tmap(&m->m8);
      ptx::prefetch_tmap(&m->m16);
      ptx::prefetch_tmap(&m->m32);
      ptx::prefetch_tmap(&m->m64);
    }
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);   // leader: its producer's arrive (+ both CTAs' bytes)
      ptx::mbar_init(&empty[s], 1);  // the leader's MMA commit
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    for (int s = 0; s < kRing; ++s) {
      ptx::mbar_init(&ring_full[s], 1);
      // leader's copy: leader MMA + 4 leader epilogue warps + peer producer + 4 peer epilogue warps
      ptx::mbar_init(&ring_empty[s], 10);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     ptx::smem_u32(tmem_slot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  ptx::tc_fence_before();
  // the CTA barrier orders warp 2's TMEM-slot write before every warp's read
  // (barrier.cluster alone is not a CTA-scope smem barrier to racecheck)
  __syncthreads();
  ptx::cluster_sync();  // barriers and TMEM of both CTAs exist before any remote use
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (!g.late_trigger) pdl_trigger();
  pdl_wait();
  if (g.prof && threadIdx.x == 0) g.prof[2 * blockIdx.x] = globaltimer_ns();

  const int item0 = g.item_off ? g.item_off[g.e_lo] : 0;
  const int n = g.item_off ? g.item_off[g.e_hi] - item0 : *g.n_items;
  const FfnItem* items = g.items + item0;
  int32_t* done1 = g.done1 + item0;
  int32_t* done2 = g.done2 + item0;
  const int MT1 = g.HD / kBlockM, MT2 = g.TD / kBlockM;
  const int P1 = MT1 / 2, P2 = MT2 / 2;
  const int KB1 = g.TD / kStageK, KB2 = g.HD / kStageK;
  const int L = min(g.lag, n);
  const int total = n * (P1 + P2);
  const int cid = blockIdx.x >> 1;
  const int ncl = gridDim.x >> 1;
  // dynamically claimed tail: at least the GEMM2-only segment of the last L
  // items, and at least ~7 waves of pair-tiles (same box, FFN stage: LM
  // 1259.6 -> 1256.5 us, MT 1289.8 -> 1287.9 us, MT seq 256 1682 -> 1644 us
  // against the segment alone (120 pair-tiles); ~1500 and all-dynamic were
  // slower; profiles/r02_s17_ffn_tail_sweep.txt, r02_s18_ffn_tail_default_ab.txt)
  const int t_dyn = g.tile_ctr ? max(0, total - (g.dyn_tail > 0 ? g.dyn_tail / 2 : max(L * P2, 7 * ncl))) : total;
  int rs = 0;
  uint32_t rph = 0;
  // leader producer: claim the next tail tile, publish it in both CTAs' rings
  auto claim = [&]() -> int {
    if (!g.tile_ctr) return -1;
    const int c = t_dyn + atomicAdd(g.tile_ctr, 1);
    const int t = c < total ? c : -1;
    ptx::mbar_wait_cluster(&ring_empty[rs], rph ^ 1);
    ring_t[rs] = t;
    uint32_t peer_t, peer_full;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(peer_t) : "r"(ptx::smem_u32(&ring_t[rs])));
    asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(peer_full) : "r"(ptx::smem_u32(&ring_full[rs])));
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(peer_t), "r"(t) : "memory");
    ptx::mbar_arrive(&ring_full[rs]);
    arrive_remote(peer_full);
    if (++rs == kRing) {
      rs = 0;
      rph ^= 1;
    }
    return t;
  };
  // every other consumer: read the slot, then release it on the leader's copy
  auto take = [&](bool warp_wide) -> int {
    if (!g.tile_ctr) return -1;
    ptx::mbar_wait_cluster(&ring_full[rs], rph);
    const int t = ring_t[rs];
    if (warp_wide) __syncwarp();
    if (!warp_wide || lane == 0) {
      if (leader) ptx::mbar_arrive(&ring_empty[rs]);
      else arrive_remote(leader_addr(&ring_empty[rs]));
    }
    if (++rs == kRing) {
      rs = 0;
      rph ^= 1;
    }
    return t;
  };

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    const uint64_t pol_w = ptx::policy_evict_first();
    const uint64_t pol_x = ptx::policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    auto next = [&]() -> int { return leader ? claim() : take(false); };
    for (int t = cid < t_dyn ? cid : next(); t >= 0; t = t + ncl < t_dyn ? t + ncl : next()) {
      const TileRef tr = decode_tile(t, n, L, P1, P2);
      const FfnItem it = items[tr.item];
      const int nrows = (it.len + 15) & ~15;
      const int half = nrows >> 1;
      const int wslot = g.slot_of ? g.slot_of[it.expert] : it.expert;
      const CUtensorMap* tA = tr.gemm ? &tmW2 : &tmW1;
      const RowMaps* tB = tr.gemm ? &hm : &xpm;
      const int a_row = wslot * (tr.gemm ? g.TD : g.HD) + (2 * tr.mp + rank) * kBlockM;
      const int a_tile = (wslot * (tr.gemm ? MT2 : MT1) + 2 * tr.mp + rank) *
                         ((tr.gemm ? g.HD : g.TD) / kChunkK);
      const int b_row = it.row0 + rank * half;
      const int KB = tr.gemm ? KB2 : KB1;
      if (tr.gemm) {
        uint32_t polls = 0;
        while (ld_acquire(done1 + tr.item) < MT1) {
          __nanosleep(64);
          if (++polls == (1u << 28)) __trap();
        }
        fence_proxy_async_global();
      }
      // both CTAs' A halves + all token rows, counted on the leader's barrier
      const uint32_t bytes = 2 * kABytes + kKch * nrows * kChunkK * 2;
      // this CTA's token rows of the stage (both chunks) as one 3-D box; the
      // chunk stride is then half x 128 B (the MMA issuer uses the same)
      const bool b_k2 = kKch % 2 == 0 && half >= 8 && half <= 128 && tB->has_k2;
      for (int kb = 0; kb < KB; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t fb = leader_addr(&full[stage]);
        // the leader arms its own barrier (CTA-scope arrive: no cluster fence)
        if (leader) ptx::mbar_arrive_expect_tx(&full[stage], bytes);
        // packed weights: the stage's two consecutive (pre-swizzled) tiles as
        // one 256-row box
#pragma unroll
        for (int c2 = 0; c2 < kKch; c2 += 2) {
          if (g.packed)
            tma_load_2d_pair(sA + stage * kABytes + c2 * kAChunk, tA, fb, 0, (a_tile + kb * kKch + c2) * kBlockM,
                             pol_w);
          if (b_k2)
            tma_load_3d_pair(sB + stage * kBBytes + c2 * half * kChunkK * 2, &tB->k2[half / 8 - 1], fb, 0, b_row,
                             kb * kKch + c2, pol_x);
        }
#pragma unroll
        for (int c = 0; c < kKch; ++c) {
          const int k0 = kb * kStageK + c * kChunkK;
          if (!g.packed) tma_load_2d_pair(sA + stage * kABytes + c * kAChunk, tA, fb, k0, a_row, pol_w);
          if (!b_k2) load_rows(sB + stage * kBBytes + c * kBChunk, tB, fb, k0, b_row, half, pol_x);
        }
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ------------------------------------------------------------ MMA issuer (leader)
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cid < t_dyn ? cid : take(false); t >= 0;
         t = t + ncl < t_dyn ? t + ncl : take(false)) {
      const TileRef tr = decode_tile(t, n, L, P1, P2);
      const FfnItem it = items[tr.item];
      const int nn = (it.len + 15) & ~15;
      const uint32_t idesc = ptx::idesc_bf16(2 * kBlockM, nn);
      const int KB = tr.gemm ? KB2 : KB1;
      const int half = nn >> 1;
      const bool b_k2 = kKch % 2 == 0 && half >= 8 && half <= 128 && (tr.gemm ? hm : xpm).has_k2;
      const int bstride = b_k2 ? half * kChunkK * 2 : kBChunk;
      ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem_base + acc * kBN;
      for (int kb = 0; kb < KB; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint64_t da = ptx::umma_desc_sw128(ptx::smem_u32(sA + stage * kABytes));
        const uint64_t db = ptx::umma_desc_sw128(ptx::smem_u32(sB + stage * kBBytes));
#pragma unroll
        for (int c = 0; c < kKch; ++c)
#pragma unroll
          for (int kk = 0; kk < kChunkK / kUmmaK; ++kk)
            mma_bf16_pair(d, da + ((c * kAChunk + kk * kUmmaK * 2) >> 4),
                          db + ((c * bstride + kk * kUmmaK * 2) >> 4), idesc,
                          (kb | c | kk) != 0 ? 1u : 0u);
        commit_pair(&empty[stage]);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      commit_pair(&tfull[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    const int tid = threadIdx.x - 128;
    __nv_bfloat16* stg = sEpi + q * 32 * 32;
    const uint32_t tempty_l[2] = {leader_addr(&tempty[0]), leader_addr(&tempty[1])};
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cid < t_dyn ? cid : take(true); t >= 0;
         t = t + ncl < t_dyn ? t + ncl : take(true)) {
      const TileRef tr = decode_tile(t, n, L, P1, P2);
      const FfnItem it = items[tr.item];
      const int m = 2 * tr.mp + rank;
      const int m_total = tr.gemm ? g.TD : g.HD;
      __nv_bfloat16* out = tr.gemm ? g.Yw : g.H;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int col0 = m * kBlockM + q * 32;
      for (int c0 = 0; c0 < it.len; c0 += 32) {
        uint32_t r[32];
        ptx::tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kBN + c0, r);
        ptx::tmem_ld_wait();
        if (tr.gemm == 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            stg[i * 32 + lane] = __float2bfloat16_rn(fmaxf(__uint_as_float(r[i]), 0.f));
        } else {
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
            if (tr.gemm && g.out_rows) row = g.out_rows[row];
            *reinterpret_cast<uint4*>(out + static_cast<size_t>(row) * m_total + col0 + ch * 8) = v;
          }
        }
        __syncwarp();
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(&tempty[acc]);
        else arrive_remote(tempty_l[acc]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      if (tr.gemm == 0) {
        fence_proxy_async_global();
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (tid == 0) atomicAdd(done1 + tr.item, 1);
      } else {
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (tid == 0) last_consumer = atomicAdd(done2 + tr.item, 1) == MT2 - 1;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (last_consumer && g.discard_h) {
          const int lines_per_row = g.HD * 2 / 128;
          const int lines = it.len * lines_per_row;
          for (int l = tid; l < lines; l += 128)
            discard_l2(g.H + static_cast<size_t>(it.row0 + l / lines_per_row) * g.HD +
                       (l % lines_per_row) * 64);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
  }

  if (g.prof && threadIdx.x == 128) g.prof[2 * blockIdx.x + 1] = globaltimer_ns();
  // the peer's last arrivals on the leader's barriers and the leader's last
  // commits into the peer must land before either CTA leaves
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(kTmemCols)
                 : "memory");
  if (g.late_trigger) pdl_trigger();
}

template <int BN, int STAGES, int KCH>
int pair_grid(int sms) {
  static int grid = -1;
  if (grid >= 0) return grid;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms & ~1);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = PairCfg<BN, STAGES, KCH>::kSmem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fused_ffn_pair_kernel<BN, STAGES, KCH>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  grid = 2 * std::min(n, sms / 2);
  if (getenv("MOE_VERBOSE")) fprintf(stderr, "[moe] ffn pair: %d co-resident clusters -> grid %d\n", n, grid);
  return grid;
}

template <int BN, int STAGES, int KCH>
cudaError_t launch_pair(const CUtensorMap& tmW1, const RowMaps& xp, const CUtensorMap& tmW2,
                        const RowMaps& h, const FusedFfnArgs& args, int sms, cudaStream_t stream) {
  const int grid = pair_grid<BN, STAGES, KCH>(sms);
  if (grid < 2) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = PairCfg<BN, STAGES, KCH>::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = 2;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, fused_ffn_pair_kernel<BN, STAGES, KCH>, tmW1, xp, tmW2, h, args);
}

}  // namespace

// Stage shapes (round 1, same-box A/B, the losing shapes since removed):
// 128-token items 4 stages of 128-deep k (two 64-wide chunks): LM FFN
// 1.303 -> 1.284 ms, MT 1.384 -> 1.340 ms against 8 x 64-deep; 256-token items
// 3 x 128-deep: MT seq 256 FFN 1.82 -> 1.78-1.80 ms, LM static 7.76 ->
// 7.59-7.68 ms against 6 x 64.  Round 2, with one weight box and one 3-D
// token box per two chunks: 2 stages of 256-deep k (KCH = 4, same bytes in
// flight) lost to 4 x 128 (LM FFN 1.2730 vs 1.2630 ms, MT 1.3151 vs 1.2933 ms).
cudaError_t fused_ffn_pair_prepare() {
  cudaError_t e = cudaFuncSetAttribute(fused_ffn_pair_kernel<256, 3, 2>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<256, 3, 2>::kSmem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(fused_ffn_pair_kernel<128, 4, 2>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<128, 4, 2>::kSmem);
}

// CTA pairs for the fused FFN.  MOE_FFN_PAIR: 0 never, 1 always, unset =
// the caller's hint (capi_state.h auto_pair: enough pair-tiles to fill ~8
// waves).  Same box, bitwise-equal outputs: MT seq 256 1.93 -> 1.84 ms, LM
// static 7.95 -> 7.37 ms, LM 1.343 -> 1.306 ms, MT 1.427 -> 1.385 ms.
bool fused_ffn_pair_enabled(int hint) {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("MOE_FFN_PAIR");
    v = e ? atoi(e) : -1;
  }
  return v == 1 || (v == -1 && hint);
}

// Persistent launch on every co-resident CTA pair (all pairs must be resident:
// GEMM2 tiles wait on GEMM1 tiles of other pairs).  Returns
// cudaErrorNotSupported when no pair fits.
cudaError_t launch_fused_ffn_pair(const CUtensorMap& tmW1, const RowMaps& xp,
                                  const CUtensorMap& tmW2, const RowMaps& h,
                                  const FusedFfnArgs& args, int tile_n, int sms,
                                  cudaStream_t stream) {
  if (tile_n == 256) return launch_pair<256, 3, 2>(tmW1, xp, tmW2, h, args, sms, stream);
  return launch_pair<128, 4, 2>(tmW1, xp, tmW2, h, args, sms, stream);
}

}  // namespace moe
