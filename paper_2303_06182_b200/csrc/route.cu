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
// One cooperative kernel, three phases separated by grid-wide barriers:
//   1. per-warp histograms (warp-aggregated with __match_any_sync) ->
//      per-block histogram, stored expert-major in global memory
//   2. every block derives the global exclusive scan (splits) and the base
//      offset of each of its warps for every expert
//   3. every warp re-walks its slots: stable rank = popc(peers & lanemask_lt)
//      + running per-(warp, expert) cursor; scatter to order[] / pos[]
// No atomic ever decides an order.  Static mode adds a 4th phase: a stable
// slot-order compaction of the dropped assignments and the placeholder fill.
#include <cooperative_groups.h>

#include <mutex>

#include "moe_internal.h"

namespace cg = cooperative_groups;

namespace moe {

namespace {

constexpr int kRouteThreads = 512;
constexpr int kRouteWarps = kRouteThreads / 32;

// dynamic shared memory layout (ints):
//   warp_cnt[kRouteWarps][E]  per-warp histogram, later per-warp cursor
//   tot[E]                    global count per expert, later splits
//   before[E]                 count of this expert in earlier blocks
//   scratch[kRouteThreads+1]  block-scan scratch

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive scan of v[0..n) in place by one block; returns the total.
__device__ int block_exclusive_scan(int* v, int n, int* scratch) {
  const int tid = threadIdx.x;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int s = 0;
  for (int i = lo; i < hi; ++i) s += v[i];
  scratch[tid] = s;
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const int x = scratch[i];
      scratch[i] = run;
      run += x;
    }
    scratch[blockDim.x] = run;
  }
  __syncthreads();
  int run = scratch[tid];
  for (int i = lo; i < hi; ++i) {
    const int x = v[i];
    v[i] = run;
    run += x;
  }
  const int total = scratch[blockDim.x];
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kRouteThreads)
    route_kernel(RouteArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ int smem[];
  const int E = a.num_experts;
  const int nb = gridDim.x;
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  int* warp_cnt = smem;                             // [warps][E]
  int* tot = warp_cnt + kRouteWarps * E;            // [E]
  int* before = tot + E;                            // [E]
  int* scratch = before + E;                        // [threads + 1]

  const int total = a.total_slots;
  const int chunk = a.chunk;  // slots per block, multiple of kRouteWarps*32
  const int per_warp = chunk / kRouteWarps;
  const int w_lo = b * chunk + warp * per_warp;
  const int w_hi = min(total, w_lo + per_warp);

  // ---- phase 1: warp-aggregated histogram
  for (int i = threadIdx.x; i < kRouteWarps * E; i += blockDim.x) warp_cnt[i] = 0;
  __syncthreads();
  int* my_cnt = warp_cnt + warp * E;
  for (int base = w_lo; base < w_hi; base += 32) {
    const int slot = base + lane;
    int e = -1;
    if (slot < w_hi) {
      e = a.expert_idx[slot];
      if (a.key_map) e = (e >= 0 && e < a.num_keys_in) ? a.key_map[e] : -2;
      if (e < 0 || e >= E) {
        atomicOr(a.error_flag, 1);
        e = -1;
      }
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    if (e >= 0 && (peers & lanemask_lt()) == 0) my_cnt[e] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int s = 0;
    for (int w = 0; w < kRouteWarps; ++w) s += warp_cnt[w * E + e];
    a.block_hist[(size_t)e * nb + b] = s;
  }
  grid.sync();

  // ---- phase 2: global scan + per-warp bases
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int* row = a.block_hist + (size_t)e * nb;
    int s = 0, bf = 0;
    for (int j = 0; j < nb; ++j) {
      const int x = row[j];
      bf += (j < b) ? x : 0;
      s += x;
    }
    tot[e] = s;
    before[e] = bf;
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
    for (int w = 0; w < kRouteWarps; ++w) {
      const int x = warp_cnt[w * E + e];
      warp_cnt[w * E + e] = run;
      run += x;
    }
  }
  __syncthreads();

  // ---- phase 3: stable rank + scatter
  const int cap = a.capacity;  // 0 => dynamic
  int my_drops = 0;
  for (int base = w_lo; base < w_hi; base += 32) {
    const int slot = base + lane;
    int e = -1;
    if (slot < w_hi) {
      e = a.expert_idx[slot];
      if (a.key_map) e = (e >= 0 && e < a.num_keys_in) ? a.key_map[e] : -2;
      if (e < 0 || e >= E) e = -1;
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    if (e >= 0) {
      const int p = my_cnt[e] + __popc(peers & lanemask_lt());
      if (cap == 0) {
        a.order[p] = slot;
        if (a.pos) a.pos[slot] = p;
        if (a.wpos) a.wpos[p] = a.gate_w[slot];
      } else {
        const int r = p - tot[e];  // rank inside expert e
        if (r < cap) {
          const long q = (long)e * cap + r;
          a.order[q] = slot;
          if (a.pos) a.pos[slot] = (int)q;
          if (a.wpos) a.wpos[q] = a.gate_w[slot];
        } else {
          if (a.pos) a.pos[slot] = -1;
          ++my_drops;
        }
        a.drop_mark[slot] = r < cap ? 0 : 1;
      }
    }
    __syncwarp();
    if (e >= 0 && (peers & lanemask_lt()) == 0) my_cnt[e] += __popc(peers);
    __syncwarp();
  }

  // ---- FFN work items (block 0): expert e contributes ceil(rows_e / tile_n)
  //      chunks; rows_e = count (dynamic) or capacity (static, placeholders
  //      included -- the waste static gating pays for).
  if (b == 0 && a.items) {
    // reuse before[] for chunk counts
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      const int rows = cap == 0 ? a.counts[e] : cap;
      before[e] = (rows + a.tile_n - 1) / a.tile_n;
    }
    __syncthreads();
    // counts[] was written by this block; tot[] holds splits
    const int n_items = block_exclusive_scan(before, E, scratch);
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      const int rows = cap == 0 ? a.counts[e] : cap;
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
    if (threadIdx.x == 0) *a.n_items = n_items;
  }

  if (cap == 0) return;

  // ---- phase 4 (static): stable compaction of drops + placeholder fill
  // per-warp drop counts -> block offset
  int wd = my_drops;
  for (int o = 16; o > 0; o >>= 1) wd += __shfl_xor_sync(0xffffffffu, wd, o);
  __syncthreads();
  if (lane == 0) scratch[warp] = wd;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kRouteWarps; ++w) s += scratch[w];
    a.block_hist[b] = s;  // block_hist no longer needed for counts
  }
  grid.sync();
  __shared__ int warp_off[kRouteWarps];
  if (threadIdx.x == 0) {
    int off = 0;
    for (int j = 0; j < b; ++j) off += a.block_hist[j];
    int tot_d = off;
    for (int j = b; j < nb; ++j) tot_d += a.block_hist[j];
    if (b == 0) *a.n_dropped = tot_d;
    for (int w = 0; w < kRouteWarps; ++w) {
      const int x = scratch[w];
      warp_off[w] = off;
      off += x;
    }
  }
  __syncthreads();
  int run = warp_off[warp];
  for (int base = w_lo; base < w_hi; base += 32) {
    const int slot = base + lane;
    bool dropped = false;
    int e = -1;
    if (slot < w_hi) {
      e = a.expert_idx[slot];
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
  // placeholder fill: slots (e, c) with c >= min(count_e, cap)
  const long cells = (long)E * cap;
  for (long q = (long)b * blockDim.x + threadIdx.x; q < cells; q += (long)nb * blockDim.x) {
    const int e = (int)(q / cap), c = (int)(q % cap);
    if (c >= a.counts[e]) {
      a.order[q] = -1;
      if (a.wpos) a.wpos[q] = 0.f;
    }
  }
}

}  // namespace

size_t route_smem_bytes(int E) {
  return sizeof(int) * ((size_t)(kRouteWarps + 2) * E + kRouteThreads + 1);
}

// Grid sizing: one block per `chunk` slots, every block co-resident (the
// kernel uses grid-wide barriers, so it is launched cooperatively).
cudaError_t launch_route(RouteArgs a, int max_blocks, cudaStream_t stream) {
  const int unit = kRouteWarps * 32;
  int chunk = 4 * unit;  // 2048 slots per block by default
  const int total = a.total_slots;
  while ((total + chunk - 1) / chunk > max_blocks) chunk += unit;
  a.chunk = chunk;
  const int nb = total > 0 ? (total + chunk - 1) / chunk : 1;
  const size_t smem = route_smem_bytes(a.num_experts);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(kRouteThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, route_kernel, a);
}

cudaError_t route_prepare(int E, int* max_blocks) {
  // The dynamic-smem limit is a process-wide attribute of the kernel: only
  // ever raise it, so a context prepared for a large E is never undercut by
  // another one preparing a small E.
  static std::mutex mu;
  static size_t granted = 0;
  const size_t smem = route_smem_bytes(E);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (smem > granted) {
      cudaError_t err = cudaFuncSetAttribute(
          route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (err != cudaSuccess) return err;
      granted = smem;
    }
  }
  cudaError_t err;
  int per_sm = 0, dev = 0, sms = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, route_kernel, kRouteThreads, smem);
  if (err != cudaSuccess) return err;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  *max_blocks = per_sm * sms;
  return per_sm > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

}  // namespace moe
