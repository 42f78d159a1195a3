// Fused expert FFN: GEMM1 (relu) and GEMM2 (gate-weighted) tiles in ONE
// persistent tcgen05 kernel, with the hidden activations H kept in L2.
//
// In the two-launch form (ffn.cu) H makes a full HBM round trip: GEMM1 writes
// rows * HD bf16 and GEMM2 reads them back (536 MB per LM layer call, ~82 us of
// a 1.4 ms weight stream).  Here the tile sequence interleaves the two GEMMs:
//
//   group g = [ GEMM1 tiles of item g ] + [ GEMM2 tiles of item g - L ]
//
// so an item's GEMM2 tiles run about one wave of CTAs after its GEMM1 tiles,
// while its H rows (n_e x HD bf16, ~0.5 MB) are still resident in L2.  The
// GEMM2 producer waits on a per-item counter (all HD/128 GEMM1 tiles stored,
// release/acquire + proxy fences) before TMA-loading H; when the last of the
// item's TD/128 GEMM2 tiles has consumed H, its lines are dropped from L2
// with discard.global.L2 so the dead activations are never written back.
//
// Deadlock freedom: every CTA walks its tiles in increasing sequence order and
// a GEMM2 tile only depends on GEMM1 tiles earlier in the sequence, so the
// earliest unfinished tile can always make progress (all CTAs are resident:
// one per SM).
//
// Roles per CTA (256 threads) are those of grouped_gemm_kernel: warp 0 TMA
// producer, warp 1 MMA issuer, warp 2 TMEM allocator, warps 4-7 epilogue.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

constexpr int kBlockM = 128;
constexpr int kChunkK = 64;  // one 128-byte swizzle atom row of bf16
constexpr int kUmmaK = 16;
constexpr int kEpiBytes = 4 * 32 * 32 * 2;

// A stage holds KCH k-chunks of 64 (KCH * 64 = the stage's K extent) for the
// weight tile (128 rows) and the token tile (BN rows), chunk-major: chunk c of
// A at c * 16 KB, chunk c of B at c * BN * 128 B, each a stack of 1024-byte
// swizzle atoms.  Bigger stages amortise the barrier round trip and the MMA
// issue overhead (8 MMAs per wait/commit at KCH = 2).
template <int BN, int STAGES, int KCH>
struct FusedCfg {
  static constexpr int kStageK = KCH * kChunkK;
  static constexpr int kAChunk = kBlockM * kChunkK * 2;
  static constexpr int kBChunk = BN * kChunkK * 2;
  static constexpr int kABytes = KCH * kAChunk;
  static constexpr int kBBytes = KCH * kBChunk;
  static constexpr int kSmem = 1024 + STAGES * (kABytes + kBBytes) + kEpiBytes +
                               (2 * STAGES + 4) * 8 + 16;
  // accumulator column stride (a power of two: TMEM allocations are)
  static constexpr int kAccStride = BN <= 64 ? 64 : (BN <= 128 ? 128 : 256);
  static constexpr int kTmemCols = 2 * kAccStride;
};

struct TileRef {
  int item;
  int gemm;  // 0: GEMM1 (W1 x Xp -> relu -> H), 1: GEMM2 (W2 x H -> scale -> Yw)
  int m;     // 128-row block of the weight matrix
};

// Sequence position -> tile.  n items, lag L (<= n), MT1/MT2 m-blocks.
__device__ __forceinline__ TileRef decode_tile(int t, int n, int L, int MT1, int MT2) {
  const int head = L * MT1;
  if (t < head) return {t / MT1, 0, t % MT1};
  const int per = MT1 + MT2;
  const int body = head + (n - L) * per;
  if (t < body) {
    const int u = t - head;
    const int g = L + u / per;
    const int r = u % per;
    if (r < MT1) return {g, 0, r};
    return {g - L, 1, r - MT1};
  }
  const int u = t - body;
  return {n - L + u / MT2, 1, u % MT2};
}

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_add(int32_t* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

template <int BN, int STAGES, int KCH>
__global__ void __launch_bounds__(256, 1)
    fused_ffn_kernel(const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ RowMaps xpm,
                     const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ RowMaps hm,
                     FusedFfnArgs g) {
  using Cfg = FusedCfg<BN, STAGES, KCH>;
  constexpr int kABytes = Cfg::kABytes;
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
  __shared__ int last_consumer;
  // dynamic tail: tiles [t_dyn, total) are claimed from a global counter by
  // the producer and handed to the MMA / epilogue warps through this ring
  constexpr int kRing = 4;
  __shared__ int ring_t[kRing];
  __shared__ __align__(8) uint64_t ring_full[kRing], ring_empty[kRing];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmW1);
    ptx::prefetch_tmap(&tmW2);
    for (const RowMaps* m : {&xpm, &hm}) {
      ptx::prefetch_tmap(&m->m16);
      ptx::prefetch_tmap(&m->m32);
      ptx::prefetch_tmap(&m->m64);
      ptx::prefetch_tmap(&m->m256);
    }
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 4);
    }
    for (int s = 0; s < kRing; ++s) {
      ptx::mbar_init(&ring_full[s], 1);
      ptx::mbar_init(&ring_empty[s], 5);  // MMA thread + 4 epilogue warps
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (!g.late_trigger) pdl_trigger();
  pdl_wait();  // the work list and activations come from the previous kernel
  if (g.prof && threadIdx.x == 0) g.prof[2 * blockIdx.x] = globaltimer_ns();

  const int item0 = g.item_off ? g.item_off[g.e_lo] : 0;
  const int n = g.item_off ? g.item_off[g.e_hi] - item0 : *g.n_items;
  const FfnItem* items = g.items + item0;
  int32_t* done1 = g.done1 + item0;
  int32_t* done2 = g.done2 + item0;
  const int MT1 = g.HD / kBlockM, MT2 = g.TD / kBlockM;
  const int KB1 = g.TD / Cfg::kStageK, KB2 = g.HD / Cfg::kStageK;
  const int L = min(g.lag, n);
  const int total = n * (MT1 + MT2);
  // Tile order per CTA: round robin over [0, t_dyn), then the tail (the
  // GEMM2-only segment of the last `lag` items: big, equal tiles whose last
  // partial wave left most SMs idle) claimed dynamically, so the CTAs finish
  // together.  Claims are in increasing sequence order, so a GEMM2 tile still
  // only waits for GEMM1 tiles that are claimed and running.
  const int t_dyn = g.tile_ctr ? max(0, total - (g.dyn_tail > 0 ? g.dyn_tail : L * MT2)) : total;
  int rs = 0;
  uint32_t rph = 0;
  // producer: claim the next tail tile and hand it to the consumers
  auto claim = [&]() -> int {
    if (!g.tile_ctr) return -1;  // round robin only: the static sequence is exhausted
    const int c = t_dyn + atomicAdd(g.tile_ctr, 1);
    const int t = c < total ? c : -1;
    ptx::mbar_wait(&ring_empty[rs], rph ^ 1);
    ring_t[rs] = t;
    ptx::mbar_arrive(&ring_full[rs]);
    if (++rs == kRing) {
      rs = 0;
      rph ^= 1;
    }
    return t;
  };
  // MMA thread / epilogue warps: the next tail tile from the ring (a whole
  // epilogue warp reads it, then its lane 0 arrives for the warp)
  auto take = [&](bool warp_wide) -> int {
    if (!g.tile_ctr) return -1;
    ptx::mbar_wait(&ring_full[rs], rph);
    const int t = ring_t[rs];
    if (warp_wide) __syncwarp();
    if (!warp_wide || lane == 0) ptx::mbar_arrive(&ring_empty[rs]);
    if (++rs == kRing) {
      rs = 0;
      rph ^= 1;
    }
    return t;
  };

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ producer
    const uint64_t pol_w = ptx::policy_evict_first();
    const uint64_t pol_x = ptx::policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x < t_dyn ? blockIdx.x : claim(); t >= 0;
         t = t + gridDim.x < t_dyn ? t + gridDim.x : claim()) {
      const TileRef tr = decode_tile(t, n, L, MT1, MT2);
      const FfnItem it = items[tr.item];
      const int nrows = (it.len + 15) & ~15;
      const int wslot = g.slot_of ? g.slot_of[it.expert] : it.expert;
      const CUtensorMap* tA = tr.gemm ? &tmW2 : &tmW1;
      const RowMaps* tB = tr.gemm ? &hm : &xpm;
      const int a_row = wslot * (tr.gemm ? g.TD : g.HD) + tr.m * kBlockM;
      // prepacked: first 128 x 64 tile of this weight block
      const int a_tile = (wslot * (tr.gemm ? MT2 : MT1) + tr.m) * ((tr.gemm ? g.HD : g.TD) / kChunkK);
      const int KB = tr.gemm ? KB2 : KB1;
      if (!tr.gemm && g.arrived) {
        // expert parallelism: this expert's token rows are stored by the peer
        // ranks; wait for all of them (system-scope acquire), then order the
        // generic-proxy stores before this thread's TMA reads
        const unsigned need = static_cast<unsigned>(g.arrived_expect[it.expert]);
        if (ld_acquire_sys_u32(g.arrived + it.expert) < need) {
          const unsigned long long t0 = globaltimer_ns();
          while (ld_acquire_sys_u32(g.arrived + it.expert) < need) {
            if (*reinterpret_cast<volatile int32_t*>(g.arrive_err) != 0) break;
            if (globaltimer_ns() - t0 > g.arrive_timeout_ns) {
              atomicExch(g.arrive_err, 1);
              break;
            }
            __nanosleep(128);
          }
        }
        fence_proxy_async_global();
      }
      if (tr.gemm) {
        // H rows of this item: every GEMM1 tile stored (acquire), then make
        // the generic-proxy stores visible to this thread's TMA reads
        uint32_t polls = 0;
        while (ld_acquire(done1 + tr.item) < MT1) {
          __nanosleep(64);
          if (++polls == (1u << 28)) __trap();
        }
        fence_proxy_async_global();
      }
      // KCH = 1, > 128 rows: the chunk's token rows as one 256-row box (the
      // rows past the item are never multiplied into stored columns)
      const bool b_256 = KCH == 1 && BN == 256 && nrows > 128 && g.rows256 && !(g.dbg & 1);
      const int tok_rows = b_256 ? 256 : nrows;
      const uint32_t bytes = ((g.dbg & 16) ? 0 : kABytes) + ((g.dbg & 1) ? 0 : KCH * tok_rows * kChunkK * 2);
      // packed weights: the stage's KCH tiles are consecutive 16 KB tiles,
      // already in the swizzled smem order -> one 1-D bulk copy
      const uint8_t* wbulk = static_cast<const uint8_t*>(tr.gemm ? g.W2p : g.W1p);
      // KCH = 2 and <= 128 rows: the stage's token rows as one 3-D box (both
      // chunks, chunk stride nrows x 128 B -- the MMA thread uses the same)
      const bool b_k2 = KCH == 2 && nrows <= 128 && tB->has_k2 && !(g.dbg & 1);
      for (int kb = 0; kb < KB; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], bytes);
        if (g.packed && !(g.dbg & 16))
          ptx::bulk_load_hint(sA + stage * kABytes,
                              wbulk + static_cast<size_t>(a_tile + kb * KCH) * Cfg::kAChunk, kABytes,
                              &full[stage], pol_w);
#pragma unroll
        for (int c = 0; c < KCH; ++c) {
          const int k0 = kb * Cfg::kStageK + c * kChunkK;
          if ((g.dbg & 16) || g.packed) {
          } else
            ptx::tma_load_2d(sA + stage * kABytes + c * Cfg::kAChunk, tA, &full[stage], k0, a_row,
                             pol_w);
          uint8_t* b_dst = sB + stage * Cfg::kBBytes + c * Cfg::kBChunk;
          if (g.dbg & 1) continue;
          if (b_k2) {
            if (c == 0) ptx::tma_load_3d(b_dst, &tB->k2[nrows / 8 - 1], &full[stage], 0, it.row0, kb * KCH, pol_x);
            continue;
          }
          if (b_256) {
            ptx::tma_load_2d(b_dst, &tB->m256, &full[stage], k0, it.row0, pol_x);
            continue;
          }
          int r = 0;
          for (; r + 64 <= nrows; r += 64)
            ptx::tma_load_2d(b_dst + r * kChunkK * 2, &tB->m64, &full[stage], k0, it.row0 + r,
                             pol_x);
          if (r + 32 <= nrows) {
            ptx::tma_load_2d(b_dst + r * kChunkK * 2, &tB->m32, &full[stage], k0, it.row0 + r,
                             pol_x);
            r += 32;
          }
          if (r < nrows)
            ptx::tma_load_2d(b_dst + r * kChunkK * 2, &tB->m16, &full[stage], k0, it.row0 + r,
                             pol_x);
        }
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
    for (int t = blockIdx.x < t_dyn ? blockIdx.x : take(false); t >= 0;
         t = t + gridDim.x < t_dyn ? t + gridDim.x : take(false)) {
      const TileRef tr = decode_tile(t, n, L, MT1, MT2);
      const FfnItem it = items[tr.item];
      const int nn = (it.len + 15) & ~15;
      const uint32_t idesc = ptx::idesc_bf16(kBlockM, nn);
      const int KB = tr.gemm ? KB2 : KB1;
      const bool b_k2 = KCH == 2 && nn <= 128 && (tr.gemm ? hm : xpm).has_k2 && !(g.dbg & 1);
      const int bstride = b_k2 ? nn * kChunkK * 2 : Cfg::kBChunk;  // token chunk stride in the stage
      ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem_base + acc * Cfg::kAccStride;
      for (int kb = 0; kb < KB; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        if (g.dbg & 4) {  // experiments: no MMAs, release the stage directly
          ptx::mbar_arrive(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
          continue;
        }
        // descriptors of the stage's first chunk; the start-address field
        // (addr >> 4) of later chunks / k-steps is a plain add (no carry:
        // shared addresses stay below 256 KB)
        const uint64_t da = ptx::umma_desc_sw128(ptx::smem_u32(sA + stage * kABytes));
        const uint64_t db = ptx::umma_desc_sw128(ptx::smem_u32(sB + stage * Cfg::kBBytes));
#pragma unroll
        for (int c = 0; c < KCH; ++c)
#pragma unroll
          for (int kk = 0; kk < kChunkK / kUmmaK; ++kk)
            ptx::mma_bf16(d, da + ((c * Cfg::kAChunk + kk * kUmmaK * 2) >> 4),
                          db + ((c * bstride + kk * kUmmaK * 2) >> 4), idesc,
                          (kb | c | kk) != 0 ? 1u : 0u);
        ptx::mma_commit(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (g.dbg & 4)
        ptx::mbar_arrive(&tfull[acc]);
      else
        ptx::mma_commit(&tfull[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    const int tid = threadIdx.x - 128;
    __nv_bfloat16* stg = sEpi + q * 32 * 32;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x < t_dyn ? blockIdx.x : take(true); t >= 0;
         t = t + gridDim.x < t_dyn ? t + gridDim.x : take(true)) {
      const TileRef tr = decode_tile(t, n, L, MT1, MT2);
      const FfnItem it = items[tr.item];
      const int m_total = tr.gemm ? g.TD : g.HD;
      __nv_bfloat16* out = tr.gemm ? g.Yw : g.H;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int col0 = tr.m * kBlockM + q * 32;
      for (int c0 = 0; c0 < ((g.dbg & 8) ? 0 : it.len); c0 += 32) {
        uint32_t r[32];
        ptx::tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * Cfg::kAccStride + c0, r);
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
          if (c0 + tok < it.len && !(g.dbg & 2)) {
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
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      if (tr.gemm == 0) {
        // publish this GEMM1 tile's H rows
        fence_proxy_async_global();
        if (g.full_fence) {
          __threadfence();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (tid == 0) atomicAdd(done1 + tr.item, 1);
        } else {
          // the named barrier orders the 128 threads' stores before thread 0's
          // release (cumulative): one release instead of 128 fence.sc
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (tid == 0) red_release_add(done1 + tr.item, 1);
        }
      } else {
        // this tile's MMAs (hence its H reads) are complete; the last consumer
        // of the item drops the item's H lines from L2 without write-back
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

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  if (g.late_trigger) pdl_trigger();
  if (g.prof && threadIdx.x == 0) g.prof[2 * blockIdx.x + 1] = globaltimer_ns();
}

template <int BN, int STAGES, int KCH>
cudaError_t prepare_fused() {
  return cudaFuncSetAttribute(fused_ffn_kernel<BN, STAGES, KCH>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              FusedCfg<BN, STAGES, KCH>::kSmem);
}

template <int BN, int STAGES, int KCH>
cudaError_t launch_fused(const CUtensorMap& w1, const RowMaps& xp, const CUtensorMap& w2,
                         const RowMaps& h, const FusedFfnArgs& g, int grid,
                         cudaStream_t stream) {
  return launch_chain(fused_ffn_kernel<BN, STAGES, KCH>, dim3(grid), dim3(256),
                      FusedCfg<BN, STAGES, KCH>::kSmem, stream, false, w1, xp, w2, h, g);
}

}  // namespace

cudaError_t fused_ffn_pair_prepare();
bool fused_ffn_pair_enabled(int hint);
cudaError_t launch_fused_ffn_pair(const CUtensorMap& tmW1, const RowMaps& xp,
                                  const CUtensorMap& tmW2, const RowMaps& h,
                                  const FusedFfnArgs& args, int tile_n, int sms,
                                  cudaStream_t stream);

cudaError_t fused_ffn_prepare() {
  cudaError_t e = fused_ffn_pair_prepare();
  if (e != cudaSuccess) return e;
  // 128-token items: 3 stages of two 64-wide k chunks (round 1 A/B against
  // 6 x 64-deep stages, since removed)
  if ((e = prepare_fused<128, 3, 2>()) != cudaSuccess) return e;
  return prepare_fused<256, 4, 1>();
}

bool fused_ffn_uses_pair(const FusedFfnArgs& args, int tile_n) {
  return (tile_n == 128 || tile_n == 256) && fused_ffn_pair_enabled(args.pair_hint) &&
         !args.arrived && args.HD % 256 == 0 && args.TD % 256 == 0;
}

cudaError_t launch_fused_ffn_impl(const CUtensorMap& tmW1, const RowMaps& xp, const CUtensorMap& tmW2,
                                  const RowMaps& h, const FusedFfnArgs& args, int tile_n, int grid,
                                  cudaStream_t stream) {
  // CTA pairs (M = 256 UMMA) when both GEMMs have an even number of 128-row
  // weight blocks
  if (fused_ffn_uses_pair(args, tile_n)) {
    cudaError_t e = launch_fused_ffn_pair(tmW1, xp, tmW2, h, args, tile_n, grid, stream);
    if (e != cudaErrorNotSupported) return e;
  }
  if (tile_n == 128) return launch_fused<128, 3, 2>(tmW1, xp, tmW2, h, args, grid, stream);
  if (tile_n == 256) return launch_fused<256, 4, 1>(tmW1, xp, tmW2, h, args, grid, stream);
  return cudaErrorInvalidValue;
}

cudaError_t launch_fused_ffn(const CUtensorMap& tmW1, const RowMaps& xp, const CUtensorMap& tmW2,
                             const RowMaps& h, const FusedFfnArgs& args_in, int tile_n, int grid,
                             cudaStream_t stream) {
  static const int full_fence = [] {
    const char* v = getenv("MOE_FFN_FENCE");
    return v ? atoi(v) : 1;
  }();
  static const int prof = [] {
    const char* v = getenv("MOE_FFN_PROF");
    return v ? atoi(v) : 0;
  }();
  // the dependent kernel (combine) is released only as FFN CTAs retire:
  // launched at the FFN's start, its 2048 waiting CTAs measured 11-16 us per
  // LM step slower (same-box A/B); MOE_FFN_LATE_TRIGGER=0 restores it
  static const int late = [] {
    const char* v = getenv("MOE_FFN_LATE_TRIGGER");
    return v ? atoi(v) : 1;
  }();
  static const int rows256 = [] {
    const char* v = getenv("MOE_FFN_ROWS256");
    return v ? atoi(v) : 1;
  }();
  static const int dyn_tail = [] {
    const char* v = getenv("MOE_FFN_DYN_TAIL");  // tiles claimed dynamically; 0 = lag * MT2, <0 = off
    return v ? atoi(v) : 0;
  }();
  FusedFfnArgs args = args_in;
  args.full_fence = full_fence;
  args.dyn_tail = dyn_tail;
  args.rows256 = rows256;
  // packed weights are always loaded as 1-D bulk copies by the 1-SM kernel
  // (the packed tensor maps' 256-row boxes are shaped for the CTA pair)
  if (args.packed && (!args.W1p || !args.W2p)) return cudaErrorInvalidValue;
  if (dyn_tail < 0) args.tile_ctr = nullptr;
  args.late_trigger = late;
  if (!prof) return launch_fused_ffn_impl(tmW1, xp, tmW2, h, args, tile_n, grid, stream);
  // experiments only: per-CTA start/end spread of this launch (eager path)
  static unsigned long long* prof_buf = nullptr;
  if (!prof_buf) cudaMalloc(&prof_buf, 2 * 1024 * sizeof(unsigned long long));
  args.prof = prof_buf;
  cudaError_t e = launch_fused_ffn_impl(tmW1, xp, tmW2, h, args, tile_n, grid, stream);
  if (e != cudaSuccess) return e;
  unsigned long long hb[2 * 1024];
  cudaStreamSynchronize(stream);
  cudaMemcpy(hb, prof_buf, 2 * grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
  double esum = 0;
  for (int i = 0; i < grid; ++i) {
    s0 = std::min(s0, hb[2 * i]);
    s1 = std::max(s1, hb[2 * i]);
    e0 = std::min(e0, hb[2 * i + 1]);
    e1 = std::max(e1, hb[2 * i + 1]);
  }
  for (int i = 0; i < grid; ++i) esum += (double)(hb[2 * i + 1] - s0);
  fprintf(stderr, "[ffn prof] start spread %.1f us, first end %.1f us, mean end %.1f us, last end %.1f us\n",
          (s1 - s0) * 1e-3, (e0 - s0) * 1e-3, esum / grid * 1e-3, (e1 - s0) * 1e-3);
  return cudaSuccess;
}

}  // namespace moe
