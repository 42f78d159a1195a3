// Dynamic / static gating dispatch on the GPU: a deterministic, stable
// counting sort of the k*S assignment slots by expert.
//
// Reference semantics (bit-exact):
//   dynamic_dispatch  proj/src/gating.cpp:58-86  -> counts, splits, order
//   static_dispatch   proj/src/gating.cpp:30-56  -> slots (E x cap), dropped
// Slot id = t*k + j (gating.hpp:33-35); inside an expert segment slot ids
// increase (stability, gating.hpp:49-52); static fills capacity first-come-
// first-served in slot order and records drops in slot order.
//
// Phases (no atomic ever decides an order):
//   1. per-warp histograms, warp-aggregated with ballot-built match masks (the slot
//      ids of a warp are prefetched 8 steps at a time so loads overlap)
//   2. exclusive scan over experts (splits) and over (block, warp) for every
//      expert -> the base position of each warp's run of each expert
//   3. every warp re-walks its slots: stable rank = popc(peers & lanemask_lt)
//      + its running cursor for that expert; scatter to order[] / pos[]
//   4. (static) stable slot-order compaction of the drops, placeholder fill
// Two variants of one kernel template:
//   kSingle  one 1024-thread CTA holds the whole problem (k*S <= 4096 slots):
//            all counts stay in shared memory, no grid barrier, no global
//            scratch.
//   multi    a cooperative grid of 512-thread CTAs for larger batches; the
//            per-block histograms go through global memory between
//            grid-wide barriers.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include <algorithm>

#include "moe_internal.h"

namespace cg = cooperative_groups;

namespace moe {

namespace {

constexpr int kMultiThreads = 512;
constexpr int kSingleThreads = 1024;
// One CTA handles up to this many slots; above it the work is spread over a
// cooperative grid (measured: one SM needs ~76 us for 32K slots at E=512,
// 64 CTAs ~12 us).
constexpr int kSingleMaxSlots = 4096;
constexpr int kPrefetch = 8;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive scan of v[0..n) in place by one block; returns the total.
// Each thread owns a contiguous chunk; chunk sums are scanned with warp
// shuffles, then the per-warp totals by warp 0.  scratch holds >= 33 ints.
__device__ int block_exclusive_scan(int* v, int n, int* scratch) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
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
    scratch[lane] = w;  // inclusive per-warp prefix
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

// Lanes of the warp holding the same key as this lane (the result of
// __match_any_sync), built from one ballot per key bit.  MATCH.ANY costs
// ~2K cycles per call when the 32 keys are mostly distinct (E = 512 routing:
// ncu, profiles/r01_route_match_any.md); nbits ballots + LOP3s are a few
// dozen cycles.  Invalid keys (< 0) match nothing and must not be used.
__device__ __forceinline__ uint32_t match_key(int key, int nbits) {
  uint32_t m = __ballot_sync(0xffffffffu, key >= 0);
  for (int bit = 0; bit < nbits; ++bit) {
    const bool set = (key >> bit) & 1;
    const uint32_t bm = __ballot_sync(0xffffffffu, set);
    m &= set ? bm : ~bm;
  }
  return m;
}

// Sort keys of kPrefetch consecutive 32-slot steps starting at base0
// (-1 for slots past `hi` and, after flagging the error, for invalid ids).
__device__ __forceinline__ void load_keys(const RouteArgs& a, int base0, int hi, int lane,
                                          bool flag_errors, int (&key)[kPrefetch]) {
#pragma unroll
  for (int u = 0; u < kPrefetch; ++u) {
    const int slot = base0 + u * 32 + lane;
    key[u] = slot < hi ? __ldg(a.expert_idx + slot) : -1;
  }
  if (a.key_map) {
#pragma unroll
    for (int u = 0; u < kPrefetch; ++u)
      if (base0 + u * 32 + lane < hi)
        key[u] = (key[u] >= 0 && key[u] < a.num_keys_in) ? __ldg(a.key_map + key[u]) : -2;
  }
#pragma unroll
  for (int u = 0; u < kPrefetch; ++u) {
    const bool valid = base0 + u * 32 + lane < hi;
    if (valid && (key[u] < 0 || key[u] >= a.num_experts)) {
      if (flag_errors) atomicOr(a.error_flag, 1);
      key[u] = -1;
    }
  }
}

__device__ __forceinline__ unsigned long long route_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// MOE_ROUTE_PROF: block 0's thread 0 stamps the phase boundaries
#define ROUTE_STAMP(j) \
  if (a.prof && blockIdx.x == 0 && threadIdx.x == 0) a.prof[j] = route_clock()

template <bool kSingle>
__global__ void __launch_bounds__(kSingle ? kSingleThreads : kMultiThreads)
    route_kernel(RouteArgs a) {
  if (!a.late_trigger) pdl_trigger();
  pdl_wait();
  ROUTE_STAMP(0);
  // zero the FFN's per-item / tile counters for this forward (saves a
  // memset node between the gather and the FFN, which would break the PDL chain)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.zero_n; i += gridDim.x * blockDim.x)
    a.zero[i] = 0;
  constexpr int kWarps = (kSingle ? kSingleThreads : kMultiThreads) / 32;
  extern __shared__ int smem[];
  __shared__ int warp_off[kWarps];
  const int E = a.num_experts;
  const int nb = gridDim.x;
  const int nb4 = (nb + 3) & ~3;  // block_hist row stride (16-byte rows)
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  int* warp_cnt = smem;                 // [warps][E]: histogram, then cursor
  int* tot = warp_cnt + kWarps * E;     // [E]: counts, then splits
  int* before = tot + E;                // [E]: count in earlier blocks
  int* scratch = before + E;            // [33]

  const int total = a.total_slots;
  const int chunk = a.chunk;  // slots per block, multiple of kWarps*32
  const int per_warp = chunk / kWarps;
  const int w_lo = b * chunk + warp * per_warp;
  const int w_hi = min(total, w_lo + per_warp);
  int* my_cnt = warp_cnt + warp * E;
  const int nbits = 32 - __clz(max(E - 1, 1));  // bits needed for keys in [0, E)

  // ---- phase 1: warp-aggregated histogram
  for (int i = threadIdx.x; i < kWarps * E; i += blockDim.x) warp_cnt[i] = 0;
  // a warp whose slots fit one prefetch batch keeps its keys (and the slots'
  // gate weights) in registers for phase 3 instead of re-reading them
  const bool keep = w_hi - w_lo <= 32 * kPrefetch;
  int kept[kPrefetch];
  float kept_w[kPrefetch];
  if (keep && a.wpos)
#pragma unroll
    for (int u = 0; u < kPrefetch; ++u) {
      const int slot = w_lo + u * 32 + lane;
      kept_w[u] = slot < w_hi ? __ldg(a.gate_w + slot) : 0.f;
    }
  __syncthreads();
  for (int base0 = w_lo; base0 < w_hi; base0 += 32 * kPrefetch) {
    int key[kPrefetch];
    load_keys(a, base0, w_hi, lane, true, key);
    if (keep)
#pragma unroll
      for (int u = 0; u < kPrefetch; ++u) kept[u] = key[u];
#pragma unroll
    for (int u = 0; u < kPrefetch; ++u) {
      if (base0 + u * 32 >= w_hi) break;
      const int e = key[u];
      const uint32_t peers = match_key(e, nbits);
      if (e >= 0 && (peers & lanemask_lt()) == 0) my_cnt[e] += __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();

  ROUTE_STAMP(1);
  // ---- phase 2: global scan + per-warp bases
  if constexpr (kSingle) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      int s = 0;
      for (int w = 0; w < kWarps; ++w) s += warp_cnt[w * E + e];
      tot[e] = s;
      before[e] = 0;
    }
  } else {
    if (b == 0)
      for (int i = threadIdx.x; i < E * (nb4 - nb); i += blockDim.x)
        a.block_hist[(size_t)(i / (nb4 - nb)) * nb4 + nb + i % (nb4 - nb)] = 0;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      int s = 0;
      for (int w = 0; w < kWarps; ++w) s += warp_cnt[w * E + e];
      a.block_hist[(size_t)e * nb4 + b] = s;
    }
    cg::this_grid().sync();
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      const int4* row = reinterpret_cast<const int4*>(a.block_hist + (size_t)e * nb4);
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
  }
  __syncthreads();
  if (b == 0)
    for (int e = threadIdx.x; e < E; e += blockDim.x) a.counts[e] = tot[e];
  const int grand = block_exclusive_scan(tot, E, scratch);  // tot -> splits
  if (b == 0) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) a.splits[e] = tot[e];
    if (threadIdx.x == 0) a.splits[E] = grand;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int run = tot[e] + before[e];
    for (int w = 0; w < kWarps; ++w) {
      const int x = warp_cnt[w * E + e];
      warp_cnt[w * E + e] = run;
      run += x;
    }
  }
  __syncthreads();

  ROUTE_STAMP(2);
  // ---- phase 3: stable rank + scatter
  const int cap = a.capacity;  // 0 => dynamic
  int my_drops = 0;
  for (int base0 = w_lo; base0 < w_hi; base0 += 32 * kPrefetch) {
    int key[kPrefetch];
    if (keep) {
#pragma unroll
      for (int u = 0; u < kPrefetch; ++u) key[u] = kept[u];
    } else {
      load_keys(a, base0, w_hi, lane, false, key);
    }
#pragma unroll
    for (int u = 0; u < kPrefetch; ++u) {
      if (base0 + u * 32 >= w_hi) break;
      const int slot = base0 + u * 32 + lane;
      const int e = key[u];
      const float gw = (keep && a.wpos) ? kept_w[u] : 0.f;
      const uint32_t peers = match_key(e, nbits);
      if (e >= 0) {
        const int p = my_cnt[e] + __popc(peers & lanemask_lt());
        if (cap == 0) {
          a.order[p] = slot;
          if (a.pos) a.pos[slot] = p;
          if (a.wpos) a.wpos[p] = keep ? gw : a.gate_w[slot];
        } else {
          const int r = p - tot[e];  // rank inside expert e
          if (r < cap) {
            const long q = (long)e * cap + r;
            a.order[q] = slot;
            if (a.pos) a.pos[slot] = (int)q;
            if (a.wpos) a.wpos[q] = keep ? gw : a.gate_w[slot];
          } else {
            if (a.pos) a.pos[slot] = -1;
            ++my_drops;
          }
          a.drop_mark[slot] = r < cap ? 0 : 1;
        }
      } else if (slot < w_hi) {
        // a rejected (out-of-range) id: the slot has no row, so no stale row
        // index from an earlier forward reaches the gather / combine
        if (a.pos) a.pos[slot] = -1;
        if (cap != 0) a.drop_mark[slot] = 0;
      }
      __syncwarp();
      if (e >= 0 && (peers & lanemask_lt()) == 0) my_cnt[e] += __popc(peers);
      __syncwarp();
    }
  }

  ROUTE_STAMP(3);
  // ---- FFN work items (block 0): expert e contributes ceil(rows_e / tile_n)
  //      items; rows_e = count (dynamic) or capacity (static, placeholders
  //      included -- the waste static gating pays for).
  if (b == 0 && a.items) {
    __syncthreads();
    // counts from the splits in shared memory (tot), not a global read-back
    auto rows_of = [&](int e) { return cap == 0 ? (e + 1 < E ? tot[e + 1] : grand) - tot[e] : cap; };
    for (int e = threadIdx.x; e < E; e += blockDim.x) before[e] = (rows_of(e) + a.tile_n - 1) / a.tile_n;
    __syncthreads();
    const int n_items = block_exclusive_scan(before, E, scratch);
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      const int rows = rows_of(e);
      const int row0 = cap == 0 ? tot[e] : e * cap;
      int it = before[e];
      for (int c = 0; c < rows; c += a.tile_n, ++it) {
        FfnItem item;
        item.expert = e;
        item.row0 = row0 + c;
        item.len = min(a.tile_n, rows - c);
        item.pad = 0;
        a.items[it] = item;
      }
    }
    if (a.item_off) {
      for (int e = threadIdx.x; e < E; e += blockDim.x) a.item_off[e] = before[e];
      if (threadIdx.x == 0) a.item_off[E] = n_items;
    }
    if (threadIdx.x == 0) *a.n_items = n_items;
  }
  ROUTE_STAMP(4);

  if (cap == 0) return;

  // ---- phase 4 (static): stable compaction of drops + placeholder fill
  int wd = my_drops;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wd += __shfl_xor_sync(0xffffffffu, wd, o);
  __syncthreads();
  if (lane == 0) warp_off[warp] = wd;
  __syncthreads();
  if constexpr (!kSingle) {
    // per-block drop counts live past the histogram (other blocks may still
    // be reading the histogram rows: there is no grid barrier after phase 2)
    if (threadIdx.x == 0) {
      int bsum = 0;
      for (int w = 0; w < kWarps; ++w) bsum += warp_off[w];
      a.block_hist[(size_t)E * nb4 + b] = bsum;
    }
    cg::this_grid().sync();
  }
  if (threadIdx.x == 0) {
    int off = 0, tot_d = 0;
    if constexpr (kSingle) {
      for (int w = 0; w < kWarps; ++w) tot_d += warp_off[w];
    } else {
      const int* drop_cnt = a.block_hist + (size_t)E * nb4;
      for (int j = 0; j < nb; ++j) {
        if (j < b) off += drop_cnt[j];
        tot_d += drop_cnt[j];
      }
    }
    if (b == 0) *a.n_dropped = tot_d;
    for (int w = 0; w < kWarps; ++w) {
      const int x = warp_off[w];
      warp_off[w] = off;
      off += x;
    }
  }
  __syncthreads();
  int run = warp_off[warp];
  for (int base = w_lo; base < w_hi; base += 32) {
    const int slot = base + lane;
    bool dropped = false;
    if (slot < w_hi) {
      int e = a.expert_idx[slot];
      if (a.key_map) e = (e >= 0 && e < a.num_keys_in) ? a.key_map[e] : -2;
      if (e >= 0 && e < E) dropped = a.drop_mark[slot] != 0;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, dropped);
    if (dropped) {
      const int at = run + __popc(m & lanemask_lt());
      a.dropped[2 * at] = slot / a.top_k;
      a.dropped[2 * at + 1] = a.expert_idx[slot];
    }
    run += __popc(m);
  }
  // placeholder fill: slots (e, c) with c >= count_e
  const long cells = (long)E * cap;
  for (long q = (long)b * blockDim.x + threadIdx.x; q < cells; q += (long)nb * blockDim.x) {
    const int e = (int)(q / cap), c = (int)(q % cap);
    if (c >= a.counts[e]) {
      a.order[q] = -1;
      if (a.wpos) a.wpos[q] = 0.f;
    }
  }
}

size_t smem_bytes(int E, int warps) { return sizeof(int) * ((size_t)(warps + 2) * E + 64); }

}  // namespace

size_t route_smem_bytes(int E) { return smem_bytes(E, kMultiThreads / 32); }

cudaError_t launch_route(RouteArgs a, int max_blocks, cudaStream_t stream) {
  const int total = a.total_slots;
  static const int late = [] {
    const char* v = getenv("MOE_ROUTE_LATE_TRIGGER");
    return v ? atoi(v) : 0;
  }();
  a.late_trigger = late;
  static const bool prof = getenv("MOE_ROUTE_PROF") != nullptr;
  static unsigned long long* prof_buf = nullptr;
  if (prof && !prof_buf) cudaMalloc(&prof_buf, 8 * sizeof(unsigned long long));
  a.prof = prof ? prof_buf : nullptr;
  struct ProfPrint {  // experiments only: phase times of this launch on exit
    unsigned long long* buf;
    cudaStream_t s;
    ~ProfPrint() {
      if (!buf) return;
      unsigned long long h[5];
      cudaStreamSynchronize(s);
      cudaMemcpy(h, buf, sizeof h, cudaMemcpyDeviceToHost);
      fprintf(stderr, "[route prof] us: histogram %.2f | scan %.2f | scatter %.2f | items %.2f\n",
              (h[1] - h[0]) * 1e-3, (h[2] - h[1]) * 1e-3, (h[3] - h[2]) * 1e-3, (h[4] - h[3]) * 1e-3);
    }
  } pp{a.prof, stream};
  const size_t single_smem = smem_bytes(a.num_experts, kSingleThreads / 32);
  static const int single_max = [] {
    const char* v = getenv("MOE_ROUTE_SINGLE_MAX");  // A/B: largest slot count for the 1-CTA form
    return v ? atoi(v) : kSingleMaxSlots;
  }();
  if (total <= std::min(single_max, kSingleMaxSlots) && single_smem <= 200 * 1024) {
    a.chunk = (total + kSingleThreads - 1) / kSingleThreads * kSingleThreads;
    if (a.chunk == 0) a.chunk = kSingleThreads;
    return launch_chain(route_kernel<true>, dim3(1), dim3(kSingleThreads), single_smem, stream,
                        false, a);
  }
  const int unit = kMultiThreads;  // 32 slots per warp per step
  static const int chunk_units = [] {
    const char* env = getenv("MOE_ROUTE_CHUNK_UNITS");  // tuning knob (units of 512 slots)
    return env ? atoi(env) : 0;
  }();
  // auto: ~32 CTAs' worth of 512-slot units per CTA, at least one (same box:
  // LM 32768 slots 18.1 -> 16.4 us at 2 units, MT 12288 slots best at 1)
  const int units = chunk_units > 0 ? chunk_units : std::max(1, (total + 8192) / 16384);
  int chunk = units * unit;
  while ((total + chunk - 1) / chunk > max_blocks) chunk += unit;
  a.chunk = chunk;
  const int nb = total > 0 ? (total + chunk - 1) / chunk : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(kMultiThreads);
  cfg.dynamicSmemBytes = route_smem_bytes(a.num_experts);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, route_kernel<false>, a);
}

cudaError_t route_prepare(int E, int* max_blocks) {
  // The dynamic-smem limit is a process-wide attribute of the kernel: only
  // ever raise it, so a context prepared for a large E is never undercut by
  // another one preparing a small E.
  static std::mutex mu;
  static size_t granted_multi = 0, granted_single = 0;
  const size_t smem = route_smem_bytes(E);
  const size_t ssmem = smem_bytes(E, kSingleThreads / 32);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (smem > granted_multi) {
      cudaError_t err = cudaFuncSetAttribute(
          route_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (err != cudaSuccess) return err;
      granted_multi = smem;
    }
    if (ssmem <= 200 * 1024 && ssmem > granted_single) {
      cudaError_t err = cudaFuncSetAttribute(
          route_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem);
      if (err != cudaSuccess) return err;
      granted_single = ssmem;
    }
  }
  int per_sm = 0, dev = 0, sms = 0;
  cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, route_kernel<false>,
                                                                  kMultiThreads, smem);
  if (err != cudaSuccess) return err;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  *max_blocks = per_sm * sms;
  return per_sm > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

}  // namespace moe
