// Expert parallelism with the exchange fused into the layer's own kernels,
// over NVLink peer memory (one CUDA-IPC "window" per rank) -- no NCCL, no host
// synchronisation, graph-capturable.  C ABI: moe_ep_* (include/moe_capi.h).
//
// Reference behaviour replaced (proj/src/exchange.cpp:95-120,
// plan_dynamic_exchange): the "size" phase (E/D int32 counts per (src, dst)
// pair, :100-104) becomes ep_publish_kernel (each rank stores its per-key slot
// counts into every peer's window); the "payload" phase (exact slot counts x
// token bytes, :106-114) becomes ep_dispatch_kernel (gather fused with the
// all-to-all: token rows go from X straight into the peer's receive buffer);
// the return leg ("mirrors the forward plan transposed") and the
// combine (gating.hpp:107-141) become ep_combine_kernel (each token reads its
// k expert outputs from the peers' output buffers, sums in slot order).
//
// Window of rank p (one cudaMalloc, exported with cudaIpcGetMemHandle):
//   EpHdr                   flags: sig_counts[src] (epoch), sig_data (CTA
//                           arrivals, cumulative), sig_ydone[dst] (epoch), epoch
//   counts_all [D][E] i32   row s = rank s's slot count per key
//   recv_w     [R]    f32   gate weight of each received row
//   recv_x     [R+256][TD]  received token rows, grouped by local expert, then
//                           source rank, then source slot order
//   recv_y     [R][TD]      FFN output (gate weight applied) of each row
// Key of an expert: key = device * E/D + local index (local index = rank of
// the expert id among its device's experts), so the keyed route makes every
// destination's rows contiguous and expert-grouped.
//
// Ordering (per step e, all flags monotonic so no reset is needed):
//   publish(e)  stores counts, fence.sys, st.release.sys sig_counts[me] = e at
//               every peer
//   dispatch(e) waits sig_counts[s] >= e for all s; stores rows + weights to
//               peers; fence.sys; red.release.sys sig_data += 1 at every peer
//   recv(e)     waits sig_data >= e * D * dispatch_ctas; builds the FFN work list
//   FFN(e)      local
//   done(e)     st.release.sys sig_ydone[me] = e at every peer
//   combine(e)  waits sig_ydone[p] >= e for all p; reads recv_y remotely
// Buffer reuse across steps is safe without double buffering: a rank starts
// publish/dispatch(e+1) only after its combine(e), which waited for every
// peer's done(e), which follows that peer's dispatch(e)/recv(e)/FFN(e) in its
// stream; and a peer's FFN(e+1) overwrites recv_y only after recv(e+1), i.e.
// after every sender finished combine(e).
#include "ep_state.h"

#include <algorithm>

namespace moe {
namespace {

__device__ __forceinline__ EpHdr* hdr(char* base) { return reinterpret_cast<EpHdr*>(base); }

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Publish the CTA's prior global writes at system scope: the CTA barrier
// orders every thread's stores before thread `t`'s fence + release, which is
// cumulative, so the peers' acquire sees all of them (one fence per CTA
// instead of one per thread; MOE_EP_FENCE=1 adds the per-thread fences back).
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until *p >= target (acquire, system scope).  After timeout_ns, or if
// an earlier wait of this rank already timed out, set err[0] and give up so a
// lost peer never hangs the device.
__device__ bool wait_geq(const unsigned long long* p, unsigned long long target, int32_t* err,
                         unsigned long long timeout_ns) {
  if (ld_acquire_sys(p) >= target) return true;
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(p) < target) {
    if (*reinterpret_cast<volatile int32_t*>(err) != 0) return false;
    if (globaltimer() - t0 > timeout_ns) {
      atomicExch(err, 1);
      return false;
    }
    __nanosleep(100);
  }
  return true;
}

// Inclusive scan of s[0..n) restarted every `seg` entries (blockDim >= n).
__device__ void segmented_scan(int32_t* s, int n, int seg) {
  const int q = threadIdx.x;
  for (int d = 1; d < seg; d <<= 1) {
    int v = 0;
    if (q < n && (q % seg) >= d) v = s[q - d];
    __syncthreads();
    if (q < n) s[q] += v;
    __syncthreads();
  }
}

// ---------------------------------------------------------------- size phase
__global__ void __launch_bounds__(512)
    ep_publish_kernel(EpPeers peers, EpLayout lay, int rank, int D, int E,
                      const int32_t* __restrict__ counts) {
  pdl_trigger();
  pdl_wait();
  EpHdr* me = hdr(peers.base[rank]);
  const unsigned long long e = me->epoch + 1;
  for (int p = 0; p < D; ++p) {
    int32_t* dst = reinterpret_cast<int32_t*>(peers.base[p] + lay.counts_all) + rank * E;
    for (int i = threadIdx.x; i < E; i += blockDim.x) dst[i] = counts[i];
  }
  __syncthreads();
  if (threadIdx.x < D) {
    fence_acq_rel_sys();
    st_release_sys(&hdr(peers.base[threadIdx.x])->sig_counts[rank], e);
  }
  if (threadIdx.x == 0) me->epoch = e;
}

// ---------------------------------------------------------------- payload phase
struct EpDispatchArgs {
  EpPeers peers;
  EpLayout lay;
  int rank, D, E, El, k, rows, vpr, max_recv;
  const uint4* X;          // [S, TD] bf16 token rows
  const int32_t* order;    // [rows] sorted row -> slot
  const int32_t* splits;   // [E+1] key segments of the sorted rows
  const float* wpos;       // [rows] gate weight per sorted row
  int32_t* dest;           // [rows] -> (device << 28) | row at that device
  int32_t* err;            // [0] timeout, [1] receive capacity exceeded
  unsigned long long timeout_ns;
  int full_fence;          // A/B: per-thread fence.sc.sys before the arrival
  int overlap;             // expert-ordered rows + per-expert arrival counters
  // by-token form (default without overlap): one warp per token reads its X
  // row once and stores it to the k destination rows
  const int32_t* idx;      // [S*k] expert ids (null: by-row form)
  const int32_t* pos;      // [S*k] slot -> sorted row
  const int32_t* key_map;  // [E] expert -> key (device * El + local expert)
  const float* w;          // [S*k] gate weight per slot
};

// by-token rows per lane kept in registers (TD <= 4096)
constexpr int kTokVecs = 16;

__device__ __forceinline__ void red_add_release_sys_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(512) ep_dispatch_kernel(EpDispatchArgs a) {
  __shared__ int32_t s_off[512];
  __shared__ int32_t s_split[513];
  __shared__ int32_t s_scan[512];
  __shared__ int32_t s_vstart[513];  // overlap: segment starts in (local expert, device) order
  __shared__ int s_ok;
  pdl_trigger();
  pdl_wait();
  char* mine = a.peers.base[a.rank];
  EpHdr* h = hdr(mine);
  const unsigned long long e = h->epoch;
  if (threadIdx.x == 0) {
    bool ok = true;
    for (int s = 0; s < a.D && ok; ++s) ok = wait_geq(&h->sig_counts[s], e, a.err, a.timeout_ns);
    s_ok = ok;
  }
  __syncthreads();
  if (s_ok) {
    // destination row of sorted row i with key q: s_off[q] + i, where
    //   s_off[q] = (rows of keys before q at q's device, all sources)
    //            + (rows of key q from lower ranks) - splits[q]
    const volatile int32_t* call = reinterpret_cast<const int32_t*>(mine + a.lay.counts_all);
    const int q = threadIdx.x;
    int col = 0, below = 0;
    if (q < a.E) {
      for (int s = 0; s < a.D; ++s) {
        const int c = call[s * a.E + q];
        col += c;
        if (s < a.rank) below += c;
      }
      s_scan[q] = col;
    }
    __syncthreads();
    segmented_scan(s_scan, a.E, a.El);
    if (q < a.E) {
      const int sp = a.splits[q];
      s_split[q] = sp;
      s_off[q] = s_scan[q] - col + below - sp;
    }
    if (q == 0) s_split[a.E] = a.splits[a.E];
    __syncthreads();
    if (a.overlap) {
      // Rows are visited in (local expert, device) order, so every warp sweeps
      // the local experts upward and a destination's expert e completes early
      // when e is small: its FFN starts on expert 0 while later rows still fly.
      // j = e * D + p indexes the segment of key p * El + e.
      if (q < a.E) {
        const int e_ = q / a.D, p_ = q % a.D, key = p_ * a.El + e_;
        s_scan[q] = a.splits[key + 1] - a.splits[key];
      }
      __syncthreads();
      segmented_scan(s_scan, a.E, a.E);
      if (q < a.E) s_vstart[q + 1] = s_scan[q];
      if (q == 0) s_vstart[0] = 0;
      __syncthreads();
    }

    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int nwarps = gridDim.x * wpb;
    if (!a.overlap && a.idx) {
      // ---- by token: X row read once, stored to its k destination rows.
      // Destination of slot t*k+j: key = key_map[idx], sorted row i = pos[slot],
      // row = s_off[key] + i at device key / El (the by-row formula, with the
      // key known directly instead of searched in splits)
      const int S = a.rows / a.k;
      const int nv = a.vpr / 32;  // 16-byte vectors per lane
      for (int t = blockIdx.x * wpb + (threadIdx.x >> 5); t < S; t += nwarps) {
        const uint4* src = a.X + static_cast<size_t>(t) * a.vpr;
        uint4 xv[kTokVecs];
#pragma unroll
        for (int u = 0; u < kTokVecs; ++u)
          if (u < nv) xv[u] = __ldg(src + u * 32 + lane);
        for (int j = 0; j < a.k; ++j) {
          const int slot = t * a.k + j;
          const int i = a.pos[slot];
          if (i < 0) continue;  // rejected id (the route flagged it)
          const int key = a.key_map[a.idx[slot]];
          const int p = key / a.El;
          const int row = s_off[key] + i;
          if (row >= a.max_recv) {
            if (lane == 0) {
              atomicExch(a.err + 1, 1);
              a.dest[i] = -1;
            }
            continue;
          }
          char* peer = a.peers.base[p];
          uint4* dst = reinterpret_cast<uint4*>(peer + a.lay.recv_x) + static_cast<size_t>(row) * a.vpr;
#pragma unroll
          for (int u = 0; u < kTokVecs; ++u)
            if (u < nv) dst[u * 32 + lane] = xv[u];
          if (lane == 0) {
            reinterpret_cast<float*>(peer + a.lay.recv_w)[row] = a.w[slot];
            a.dest[i] = (p << kRowBits) | row;
          }
        }
      }
    }
    for (int v_ = blockIdx.x * wpb + (threadIdx.x >> 5); v_ < a.rows && (a.overlap || !a.idx); v_ += nwarps) {
      int lo, i;
      if (a.overlap) {
        int jl = 0, jh = a.E - 1;  // last (e, p) segment starting at or before v_
        while (jl < jh) {
          const int mid = (jl + jh + 1) >> 1;
          if (s_vstart[mid] <= v_) jl = mid;
          else jh = mid - 1;
        }
        lo = (jl % a.D) * a.El + jl / a.D;
        i = s_split[lo] + (v_ - s_vstart[jl]);
      } else {
        i = v_;
        lo = 0;
        int hi = a.E - 1;  // last key whose segment starts at or before i
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_split[mid] <= i) lo = mid;
          else hi = mid - 1;
        }
      }
      const int p = lo / a.El;
      const int row = s_off[lo] + i;
      if (row >= a.max_recv) {
        if (lane == 0) {
          atomicExch(a.err + 1, 1);
          a.dest[i] = -1;
        }
        continue;
      }
      char* peer = a.peers.base[p];
      uint4* dst = reinterpret_cast<uint4*>(peer + a.lay.recv_x) + static_cast<size_t>(row) * a.vpr;
      const uint4* src = a.X + static_cast<size_t>(a.order[i] / a.k) * a.vpr;
      int v = lane;
      for (; v + 96 < a.vpr; v += 128) {
        const uint4 x0 = __ldg(src + v), x1 = __ldg(src + v + 32), x2 = __ldg(src + v + 64),
                    x3 = __ldg(src + v + 96);
        dst[v] = x0;
        dst[v + 32] = x1;
        dst[v + 64] = x2;
        dst[v + 96] = x3;
      }
      for (; v < a.vpr; v += 32) dst[v] = __ldg(src + v);
      if (lane == 0) {
        reinterpret_cast<float*>(peer + a.lay.recv_w)[row] = a.wpos[i];
        a.dest[i] = (p << kRowBits) | row;
      }
      if (a.overlap) {
        // this row is visible at its owner before the owner's count moves
        __syncwarp();
        if (lane == 0) {
          fence_acq_rel_sys();
          red_add_release_sys_u32(reinterpret_cast<unsigned*>(peer + a.lay.arrived) + lo % a.El, 1u);
        }
      }
    }
  }
  if (a.full_fence) __threadfence_system();
  __syncthreads();
  // every CTA arrives (even on a timeout) so no receiver waits on a dead step
  if (threadIdx.x < a.D) {
    fence_acq_rel_sys();
    red_add_release_sys(&hdr(a.peers.base[threadIdx.x])->sig_data, 1ull);
  }
}

// MOE_EP_DISPATCH_TOKENS=0 restores the by-row dispatch (A/B)
bool ep_dispatch_by_token() {
  static const bool on = [] {
    const char* v = getenv("MOE_EP_DISPATCH_TOKENS");
    return !v || atoi(v) != 0;
  }();
  return on;
}

// ---------------------------------------------------------------- receive side
struct EpRecvArgs {
  char* mine;
  EpLayout lay;
  int rank, D, E, El, tile_n, max_recv, dispatch_ctas;
  int overlap;     // per-expert arrival waits in the FFN instead of a global one here
  int32_t* expect; // [El] rows each local expert receives this step (overlap)
  FfnItem* items;
  int32_t* n_items;
  int32_t* done;  // fused-FFN counters, zeroed here
  int done_n;
  int32_t* err;
  unsigned long long timeout_ns;
};

__global__ void __launch_bounds__(512) ep_recv_kernel(EpRecvArgs a) {
  __shared__ int32_t s_rows[512];
  __shared__ int32_t s_items[512];
  __shared__ int s_ok;
  pdl_trigger();
  pdl_wait();
  EpHdr* h = hdr(a.mine);
  const unsigned long long e = h->epoch;
  if (threadIdx.x == 0)
    s_ok = a.overlap ? 1
                     : wait_geq(&h->sig_data, e * static_cast<unsigned long long>(a.D) * a.dispatch_ctas,
                                a.err, a.timeout_ns);
  for (int i = threadIdx.x; i < a.done_n; i += blockDim.x) a.done[i] = 0;
  __syncthreads();
  const int q = threadIdx.x;  // local expert
  int n = 0;
  if (s_ok && q < a.El) {
    const volatile int32_t* call = reinterpret_cast<const int32_t*>(a.mine + a.lay.counts_all);
    for (int s = 0; s < a.D; ++s) n += call[s * a.E + a.rank * a.El + q];
  }
  if (q < a.El) {
    s_rows[q] = n;
    if (a.expect) a.expect[q] = n;
  }
  __syncthreads();
  segmented_scan(s_rows, a.El, a.El);
  // Rows past the receive capacity were never stored (the sender flagged
  // them and dropped them from its combine): the work list covers exactly the
  // rows that fit, so every row that did arrive is still computed.
  int fit = 0;
  if (q < a.El) fit = max(0, min(n, a.max_recv - (s_rows[q] - n)));
  const int ni = (fit + a.tile_n - 1) / a.tile_n;
  if (q < a.El) s_items[q] = ni;
  __syncthreads();
  segmented_scan(s_items, a.El, a.El);
  if (q < a.El && ni) {
    const int row0 = s_rows[q] - n;
    const int it0 = s_items[q] - ni;
    for (int j = 0; j < ni; ++j) {
      const int r = row0 + j * a.tile_n;
      a.items[it0 + j] = FfnItem{q, r, min(a.tile_n, fit - j * a.tile_n), 0};
    }
  }
  if (q == 0) {
    if (s_rows[a.El - 1] > a.max_recv) atomicExch(a.err + 1, 1);
    *a.n_items = s_ok ? s_items[a.El - 1] : 0;
  }
}

__global__ void ep_done_kernel(EpPeers peers, EpLayout lay, int rank, int D, int El) {
  pdl_wait();
  const unsigned long long e = hdr(peers.base[rank])->epoch;
  // the FFN consumed every arrival of this step: restart the per-expert
  // counts before any sender may start the next step (it waits for this flag)
  unsigned* arrived = reinterpret_cast<unsigned*>(peers.base[rank] + lay.arrived);
  for (int i = threadIdx.x; i < El; i += blockDim.x) arrived[i] = 0;
  __syncwarp();  // every lane's reset is ordered before the releases below
  __threadfence_system();
  if (threadIdx.x < D) st_release_sys(&hdr(peers.base[threadIdx.x])->sig_ydone[rank], e);
}

// ---------------------------------------------------------------- return + combine
struct EpCombineArgs {
  EpPeers peers;
  EpLayout lay;
  int rank, D, S, k, vpr;
  const int32_t* pos;   // [S*k] slot -> sorted row
  const int32_t* dest;  // [S*k] sorted row -> (device << 28) | row
  uint4* out;           // [S, TD]
  int32_t* err;
  unsigned long long timeout_ns;
};

__device__ __forceinline__ void add8(float (&acc)[8], const uint4& v) {
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(b[i]);
    acc[2 * i] += f.x;
    acc[2 * i + 1] += f.y;
  }
}

__global__ void __launch_bounds__(256) ep_combine_kernel(EpCombineArgs a) {
  __shared__ int s_ok;
  // the next step's gate is released only as these CTAs finish (as the
  // single-GPU combine, rowops.cu)
  pdl_wait();
  EpHdr* h = hdr(a.peers.base[a.rank]);
  const unsigned long long e = h->epoch;
  if (threadIdx.x == 0) {
    bool ok = true;
    for (int p = 0; p < a.D && ok; ++p) ok = wait_geq(&h->sig_ydone[p], e, a.err, a.timeout_ns);
    s_ok = ok;
  }
  __syncthreads();
  if (!s_ok) {
    pdl_trigger();
    return;
  }
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int nwarps = gridDim.x * wpb;
  for (int t = blockIdx.x * wpb + (threadIdx.x >> 5); t < a.S; t += nwarps) {
    const uint4* src[8];
    for (int j = 0; j < a.k; ++j) {
      const int d = a.dest[a.pos[static_cast<size_t>(t) * a.k + j]];
      src[j] = d < 0 ? nullptr
                     : reinterpret_cast<const uint4*>(a.peers.base[d >> kRowBits] + a.lay.recv_y) +
                           static_cast<size_t>(d & ((1 << kRowBits) - 1)) * a.vpr;
    }
    for (int v0 = lane; v0 < a.vpr; v0 += 128) {
      float acc[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[u][c] = 0.f;
      for (int j = 0; j < a.k; ++j) {
        if (!src[j]) continue;
        uint4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (v0 + 32 * u < a.vpr) x[u] = __ldcv(src[j] + v0 + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (v0 + 32 * u < a.vpr) add8(acc[u], x[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (v0 + 32 * u >= a.vpr) break;
        uint4 o;
        __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i] = __floats2bfloat162_rn(acc[u][2 * i], acc[u][2 * i + 1]);
        a.out[static_cast<size_t>(t) * a.vpr + v0 + 32 * u] = o;
      }
    }
  }
  pdl_trigger();
}

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

}  // namespace
}  // namespace moe


// Receive side of both transports: FFN work list (items over the received
// rows, grouped by local expert) from the count matrix in the window, and the
// fused FFN's counters zeroed.  wait_for_arrivals: spin until every sender's
// dispatch CTAs arrived (peer-memory transport); the NCCL transport's rows
// are in place when its receive completes in stream order.
int ep_launch_recv(moe_ep* P, cudaStream_t s, bool wait_for_arrivals) {
  const moe_ep_desc& d = P->d;
  const int D = d.world_size, E = d.num_experts;
  EpRecvArgs ra{};
  ra.mine = P->window;
  ra.lay = P->lay;
  ra.rank = d.rank;
  ra.D = D;
  ra.E = E;
  ra.El = P->El;
  ra.tile_n = P->tile_n;
  ra.max_recv = P->max_recv;
  ra.dispatch_ctas = P->dispatch_ctas;
  ra.overlap = wait_for_arrivals ? 0 : 1;
  ra.expect = P->overlap ? P->expect.p : nullptr;
  ra.items = P->items.p;
  ra.n_items = P->n_items.p;
  ra.done = P->done.p;
  ra.done_n = 2 * P->items_max + 1;
  ra.err = P->err.p;
  ra.timeout_ns = P->timeout_ns;
  cudaError_t ce = launch_chain(ep_recv_kernel, dim3(1), dim3(512), 0, s, false, ra);
  if (ce != cudaSuccess) return cuda_fail(ce, "EP receive launch");
  return MOE_OK;
}

// The fused tcgen05 FFN over the received rows (recv_x -> recv_y, gate weight
// applied in the GEMM2 epilogue).
int ep_launch_ffn(moe_ep* P, cudaStream_t s) {
  const moe_ep_desc& d = P->d;
  const int D = d.world_size, E = d.num_experts, TD = d.token_dim, HD = d.hidden_dim;
  FusedFfnArgs fa{};
  fa.items = P->items.p;
  fa.n_items = P->n_items.p;
  fa.TD = TD;
  fa.HD = HD;
  fa.H = P->h.p;
  fa.Yw = reinterpret_cast<__nv_bfloat16*>(P->window + P->lay.recv_y);
  fa.wpos = reinterpret_cast<const float*>(P->window + P->lay.recv_w);
  fa.done1 = P->done.p;
  fa.done2 = P->done.p + P->items_max;
  fa.tile_ctr = P->done.p + 2 * P->items_max;
  if (P->overlap && !P->nccl_comm) {  // GEMM1 tiles wait for their expert's rows, not for every row
    fa.arrived = reinterpret_cast<const unsigned*>(P->window + P->lay.arrived);
    fa.arrived_expect = P->expect.p;
    fa.arrive_err = P->err.p;
    fa.arrive_timeout_ns = P->timeout_ns;
  }
  const int per_item = HD / 128 + TD / 128;
  fa.lag = std::max(2, (8 * P->ctx->sms + per_item - 1) / per_item);
  fa.discard_h = 1;
  fa.packed = 1;
  fa.W1p = P->w1p.p;
  fa.W2p = P->w2p.p;
  fa.pair_hint = auto_pair((double)D * d.max_tokens * d.top_k / E, P->El, TD, HD, P->tile_n,
                           P->ctx->sms);
  cudaError_t ce = launch_fused_ffn(P->tmW1p, P->xpm, P->tmW2p, P->hm, fa, P->tile_n, P->ctx->sms, s);
  if (ce != cudaSuccess) return cuda_fail(ce, "EP fused ffn launch");
  return MOE_OK;
}

extern "C" {

int moe_ep_create(moe_ctx* ctx, const moe_ep_desc* desc, const void* Wg, const void* W1_local,
                  const void* W2_local, const int32_t* device_of, moe_ep** out) {
  if (!ctx || !desc || !out || !Wg || !W1_local || !W2_local || !device_of)
    return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  const moe_ep_desc& d = *desc;
  int st = check_batch(d.max_tokens, d.top_k, d.num_experts);
  if (st) return st;
  const int D = d.world_size, E = d.num_experts;
  if (D < 1 || D > MOE_EP_MAX_RANKS || d.rank < 0 || d.rank >= D)
    return fail(MOE_ERR_INVALID_ARGUMENT, "rank / world_size out of range");
  if (E % D) return fail(MOE_ERR_INVALID_ARGUMENT, "num_experts must divide evenly across devices");
  if (E > 512 || d.top_k > 8)
    return fail(MOE_ERR_UNSUPPORTED, "num_experts <= 512 and top_k <= 8 are supported");
  if (d.token_dim % 128 || d.hidden_dim % 128 || d.token_dim <= 0 || d.hidden_dim <= 0)
    return fail(MOE_ERR_UNSUPPORTED, "token_dim and hidden_dim must be positive multiples of 128");
  const int El = E / D;
  // placement -> keys (balance.cpp:42-57: exactly E/D experts per device)
  std::vector<int32_t> key(E), held(D, 0);
  for (int e = 0; e < E; ++e) {
    const int dev = device_of[e];
    if (dev < 0 || dev >= D || held[dev] >= El)
      return fail(MOE_ERR_INVALID_ARGUMENT, "placement must put exactly E/D experts on every device");
    key[e] = dev * El + held[dev]++;
  }
  const long worst = (long)D * d.max_tokens * d.top_k;
  const long R = d.max_recv_rows > 0 ? d.max_recv_rows : worst;
  if (R > (1L << kRowBits) - 256) return fail(MOE_ERR_UNSUPPORTED, "receive capacity too large");
  MOE_CUDA(cudaSetDevice(ctx->device));
  cudaError_t ce = gate_prepare(E);
  if (ce != cudaSuccess) return cuda_fail(ce, "gate_prepare");

  auto* P = new moe_ep();
  P->ctx = ctx;
  P->d = d;
  P->El = El;
  P->max_recv = (int)R;
  P->Wg = Wg;
  // work-item width: 256-token items (N = 256 MMAs, half the weight re-reads)
  // once the expected rows per local expert (D * S * k / E) pass ~160, as the
  // single-GPU layer picks; MOE_EP_TILE_N overrides
  const double per_expert = (double)D * d.max_tokens * d.top_k / E;
  P->tile_n = auto_tile_n(per_expert, El, d.token_dim, d.hidden_dim, ctx->sms);
  if (const char* v = getenv("MOE_EP_TILE_N")) P->tile_n = atoi(v) == 256 ? 256 : 128;
  P->items_max = (int)(R / P->tile_n + El + 1);
  const size_t TD = d.token_dim, HD = d.hidden_dim, S = d.max_tokens, k = d.top_k;
  size_t off = align256(sizeof(EpHdr));
  P->lay.counts_all = off;
  off = align256(off + sizeof(int32_t) * D * E);
  P->lay.arrived = off;  // [E/D] rows of each local expert stored so far this step
  off = align256(off + sizeof(uint32_t) * El);
  P->lay.recv_w = off;
  off = align256(off + sizeof(float) * R);
  P->lay.recv_x = off;
  off = align256(off + 2 * (R + 256) * TD);
  P->lay.recv_y = off;
  off = align256(off + 2 * R * TD);
  P->lay.total = off;
  auto bail = [&](int s) {
    moe_ep_destroy(P);
    return s;
  };
  if (cudaMalloc(&P->window, P->lay.total) != cudaSuccess) {
    P->window = nullptr;
    return bail(fail(MOE_ERR_OUT_OF_MEMORY, "cudaMalloc (EP window)"));
  }
  if ((ce = cudaMemset(P->window, 0, P->lay.total)) != cudaSuccess)
    return bail(cuda_fail(ce, "clear EP window"));
  const size_t n1 = (size_t)El * HD * TD;
  if ((st = P->key_map.reserve(E)) || (st = P->idx.reserve(S * k)) || (st = P->w.reserve(S * k)) ||
      (st = P->counts.reserve(E)) || (st = P->splits.reserve(E + 1)) ||
      (st = P->order.reserve(S * k)) || (st = P->pos.reserve(S * k)) ||
      (st = P->wpos.reserve(S * k)) || (st = P->dest.reserve(S * k)) ||
      (st = P->n_items.reserve(1)) || (st = P->err.reserve(2)) ||
      (st = P->done.reserve(2 * (size_t)P->items_max + 1)) || (st = P->items.reserve(P->items_max)) ||
      (st = P->h.reserve((R + 256) * HD)) || (st = P->w1p.reserve(n1)) || (st = P->w2p.reserve(n1)) ||
      (st = ctx->prepare_route(E)))
    return bail(st);
  MOE_CUDA(cudaMemcpy(P->key_map.p, key.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice));
  MOE_CUDA(cudaMemset(P->err.p, 0, 2 * sizeof(int32_t)));
  MOE_CUDA(cudaMemset(P->h.p, 0, (R + 256) * HD * 2));
  char* rx = P->window + P->lay.recv_x;
  if ((st = encode_bf16(&P->tmWg, Wg, E, TD, moe::gate_box_rows(E), moe::gate_box_cols(E))) ||
      (st = encode_packed(&P->tmW1p, P->w1p.p, n1)) ||
      (st = encode_packed(&P->tmW2p, P->w2p.p, n1)) ||
      (st = encode_rows(&P->xpm, rx, R + 256, TD)) || (st = encode_rows(&P->hm, P->h.p, R + 256, HD)))
    return bail(st);
  // the fused FFN streams tile-packed weights (contiguous 16 KB 128 x 64 tiles)
  if ((ce = launch_pack_tiles(static_cast<const __nv_bfloat16*>(W1_local), P->w1p.p, (long)El * HD,
                              (int)TD, nullptr)) != cudaSuccess ||
      (ce = launch_pack_tiles(static_cast<const __nv_bfloat16*>(W2_local), P->w2p.p, (long)El * TD,
                              (int)HD, nullptr)) != cudaSuccess ||
      (ce = cudaDeviceSynchronize()) != cudaSuccess)
    return bail(cuda_fail(ce, "EP weight prepack"));
  if (const char* v = getenv("MOE_EP_TIMEOUT_MS")) P->timeout_ns = (unsigned long long)atoll(v) * 1000000ull;
  if (const char* v = getenv("MOE_EP_DISPATCH_CTAS")) P->dispatch_ctas = std::max(1, atoi(v));
  if (const char* v = getenv("MOE_EP_FENCE")) P->full_fence = atoi(v);
  if (const char* v = getenv("MOE_EP_OVERLAP")) P->overlap = atoi(v);
  if ((st = P->expect.reserve(El))) return bail(st);
  if (d.transport != MOE_EP_TRANSPORT_P2P && d.transport != MOE_EP_TRANSPORT_NCCL)
    return bail(fail(MOE_ERR_INVALID_ARGUMENT, "unknown EP transport"));
  if (d.transport == MOE_EP_TRANSPORT_NCCL) P->overlap = 0;  // arrivals are whole NCCL messages
  *out = P;
  return MOE_OK;
}

int moe_ep_destroy(moe_ep* P) {
  if (!P) return MOE_OK;
  cudaSetDevice(P->ctx->device);
  if (P->graph) cudaGraphExecDestroy(P->graph);
  for (cudaEvent_t e : P->tev)
    if (e) cudaEventDestroy(e);
  for (int r = 0; r < MOE_EP_MAX_RANKS; ++r)
    if (P->opened[r]) cudaIpcCloseMemHandle(P->peers.base[r]);
  ep_nccl_release(P);
  if (P->window) cudaFree(P->window);
  P->key_map.release();
  P->idx.release();
  P->counts.release();
  P->splits.release();
  P->order.release();
  P->pos.release();
  P->dest.release();
  P->n_items.release();
  P->done.release();
  P->err.release();
  P->w.release();
  P->wpos.release();
  P->items.release();
  P->h.release();
  P->w1p.release();
  P->w2p.release();
  P->expect.release();
  delete P;
  return MOE_OK;
}

int moe_ep_get_handle(moe_ep* P, void* handle) {
  if (!P || !handle) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) <= MOE_EP_HANDLE_BYTES, "handle size");
  cudaSetDevice(P->ctx->device);
  cudaIpcMemHandle_t h;
  MOE_CUDA(cudaIpcGetMemHandle(&h, P->window));
  memset(handle, 0, MOE_EP_HANDLE_BYTES);
  memcpy(handle, &h, sizeof h);
  return MOE_OK;
}

int moe_ep_connect(moe_ep* P, const void* handles) {
  if (!P || !handles) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (P->connected) return fail(MOE_ERR_INVALID_ARGUMENT, "already connected");
  if (P->d.transport != MOE_EP_TRANSPORT_P2P)
    return fail(MOE_ERR_INVALID_ARGUMENT, "NCCL-transport layer: use moe_ep_connect_nccl");
  cudaSetDevice(P->ctx->device);
  const char* hb = static_cast<const char*>(handles);
  for (int r = 0; r < P->d.world_size; ++r) {
    if (r == P->d.rank) {
      P->peers.base[r] = P->window;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, hb + (size_t)r * MOE_EP_HANDLE_BYTES, sizeof h);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle (peer window)");
    P->peers.base[r] = static_cast<char*>(p);
    P->opened[r] = true;
  }
  P->connected = true;
  return MOE_OK;
}

extern "C++" {
static int ep_forward_impl(moe_ep* P, const void* X, int S, void* out, cudaStream_t s,
                           bool timed = false) {
  const moe_ep_desc& d = P->d;
  auto mark = [&](int i) {
    if (timed && P->timing) cudaEventRecord(P->tev[i], s);
  };
  if (!P->connected) return fail(MOE_ERR_INVALID_ARGUMENT, "moe_ep_connect has not been called");
  if (S < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "empty batch");
  if (S > d.max_tokens) return fail(MOE_ERR_INVALID_ARGUMENT, "S exceeds max_tokens");
  if (P->nccl_comm) return ep_forward_nccl(P, X, S, out, s, timed);
  const int k = d.top_k, E = d.num_experts, TD = d.token_dim, D = d.world_size;
  int st;
  if (X != P->tmX_ptr || S != P->tmX_rows) {
    if ((st = encode_bf16(&P->tmX, X, (uint64_t)S, TD, 128, moe::gate_box_cols(P->d.num_experts)))) return st;
    P->tmX_ptr = X;
    P->tmX_rows = S;
  }
  // 1. gate + keyed route (local)
  GateArgs ga{S, TD, E, k, P->idx.p, P->w.p, nullptr};
  ga.X = X;
  ga.Wg = P->Wg;
  mark(0);
  cudaError_t ce = launch_gate(P->tmX, P->tmWg, ga, s);
  if (ce != cudaSuccess) return cuda_fail(ce, "gate launch");
  st = route_common(P->ctx, P->idx.p, S, k, E, 0, P->counts.p, P->splits.p, P->order.p, P->pos.p,
                    P->w.p, P->wpos.p, nullptr, nullptr, nullptr, nullptr, 128, P->key_map.p, E, s);
  if (st) return st;
  // 2. size phase
  mark(1);
  ce = launch_chain(ep_publish_kernel, dim3(1), dim3(512), 0, s, false, P->peers, P->lay, d.rank, D,
                    E, (const int32_t*)P->counts.p);
  if (ce != cudaSuccess) return cuda_fail(ce, "EP publish launch");
  // 3. payload phase: gather fused with the all-to-all
  EpDispatchArgs da{};
  da.peers = P->peers;
  da.lay = P->lay;
  da.rank = d.rank;
  da.D = D;
  da.E = E;
  da.El = P->El;
  da.k = k;
  da.rows = S * k;
  da.vpr = TD / 8;
  da.max_recv = P->max_recv;
  da.X = static_cast<const uint4*>(X);
  da.order = P->order.p;
  da.splits = P->splits.p;
  da.wpos = P->wpos.p;
  da.dest = P->dest.p;
  da.err = P->err.p;
  da.timeout_ns = P->timeout_ns;
  da.full_fence = P->full_fence;
  da.overlap = P->overlap;
  // the by-token form needs the whole row in registers (TD <= 4096, TD % 256 == 0)
  if (!P->overlap && (TD / 8) % 32 == 0 && TD / 8 <= 32 * kTokVecs && ep_dispatch_by_token()) {
    da.idx = P->idx.p;
    da.pos = P->pos.p;
    da.key_map = P->key_map.p;
    da.w = P->w.p;
  }
  mark(2);
  ce = launch_chain(ep_dispatch_kernel, dim3(P->dispatch_ctas), dim3(512), 0, s, false, da);
  if (ce != cudaSuccess) return cuda_fail(ce, "EP dispatch launch");
  // 4. receive side: work list from the count matrix
  mark(3);
  if ((st = ep_launch_recv(P, s, !P->overlap))) return st;
  // 5. the fused FFN over the received rows (gate weight applied in GEMM2)
  mark(4);
  if ((st = ep_launch_ffn(P, s))) return st;
  // 6. outputs ready -> every peer
  mark(5);
  ce = launch_chain(ep_done_kernel, dim3(1), dim3(32), 0, s, false, P->peers, P->lay, d.rank, D,
                    P->El);
  if (ce != cudaSuccess) return cuda_fail(ce, "EP done launch");
  // 7. return leg fused with the combine
  EpCombineArgs ca{};
  ca.peers = P->peers;
  ca.lay = P->lay;
  ca.rank = d.rank;
  ca.D = D;
  ca.S = S;
  ca.k = k;
  ca.vpr = TD / 8;
  ca.pos = P->pos.p;
  ca.dest = P->dest.p;
  ca.out = static_cast<uint4*>(out);
  ca.err = P->err.p;
  ca.timeout_ns = P->timeout_ns;
  const int grid = std::min(P->ctx->sms * 8, (S + 7) / 8);
  mark(6);
  ce = launch_chain(ep_combine_kernel, dim3(std::max(grid, 1)), dim3(256), 0, s, false, ca);
  if (ce != cudaSuccess) return cuda_fail(ce, "EP combine launch");
  mark(7);
  return MOE_OK;
}
}  // extern "C++"

int moe_ep_forward(moe_ep* P, const void* X, int S, void* out, void* stream) {
  MOE_NVTX("moe.ep_forward");
  if (!P || !X || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  cudaSetDevice(P->ctx->device);
  return ep_forward_impl(P, X, S, out, (cudaStream_t)stream, true);
}

int moe_ep_enable_timing(moe_ep* P, int on) {
  if (!P) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  cudaSetDevice(P->ctx->device);
  if (on && !P->tev[0])
    for (cudaEvent_t& e : P->tev) MOE_CUDA(cudaEventCreate(&e));
  P->timing = on != 0;
  return MOE_OK;
}

int moe_ep_stage_times(moe_ep* P, float* ms) {
  if (!P || !ms) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (!P->tev[0]) return fail(MOE_ERR_INVALID_ARGUMENT, "timing not enabled");
  cudaSetDevice(P->ctx->device);
  MOE_CUDA(cudaEventSynchronize(P->tev[MOE_EP_NUM_STAGES]));
  for (int i = 0; i < MOE_EP_NUM_STAGES; ++i)
    MOE_CUDA(cudaEventElapsedTime(&ms[i], P->tev[i], P->tev[i + 1]));
  return MOE_OK;
}

int moe_ep_forward_graph(moe_ep* P, const void* X, int S, void* out, void* stream) {
  MOE_NVTX("moe.ep_forward_graph");
  if (!P || !X || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  cudaSetDevice(P->ctx->device);
  if (P->nccl_comm) return ep_forward_impl(P, X, S, out, s);  // host sync inside: not capturable
  if (!(P->graph && P->g_x == X && P->g_out == out && P->g_S == S && P->g_stream == s)) {
    if (s == nullptr) return fail(MOE_ERR_INVALID_ARGUMENT, "graph capture needs a non-default stream");
    if (P->graph) cudaGraphExecDestroy(P->graph);
    P->graph = nullptr;
    MOE_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    int st = ep_forward_impl(P, X, S, out, s);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (st) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(e, "end capture");
    e = cudaGraphInstantiate(&P->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      P->graph = nullptr;
      return cuda_fail(e, "graph instantiate");
    }
    P->g_x = X;
    P->g_out = out;
    P->g_S = S;
    P->g_stream = s;
  }
  MOE_CUDA(cudaGraphLaunch(P->graph, s));
  return MOE_OK;
}

int moe_ep_check_errors(moe_ep* P, void* stream) {
  if (!P) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  cudaSetDevice(P->ctx->device);
  MOE_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  int32_t err[2] = {0, 0};
  MOE_CUDA(cudaMemcpy(err, P->err.p, sizeof err, cudaMemcpyDeviceToHost));
  if (err[0]) return fail(MOE_ERR_PEER_TIMEOUT, "expert-parallel peer wait timed out");
  if (err[1]) {
    MOE_CUDA(cudaMemset(P->err.p + 1, 0, sizeof(int32_t)));
    return fail(MOE_ERR_UNSUPPORTED, "expert-parallel receive capacity (max_recv_rows) exceeded");
  }
  return moe_check_errors(P->ctx, stream);
}

int moe_ep_get_view(moe_ep* P, moe_ep_view* v) {
  if (!P || !v) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  v->idx = P->idx.p;
  v->w = P->w.p;
  v->counts = P->counts.p;
  v->counts_all = reinterpret_cast<int32_t*>(P->window + P->lay.counts_all);
  v->dest = P->dest.p;
  v->order = P->order.p;
  v->recv_x = P->window + P->lay.recv_x;
  v->recv_y = P->window + P->lay.recv_y;
  v->recv_w = reinterpret_cast<float*>(P->window + P->lay.recv_w);
  v->n_items = P->n_items.p;
  v->max_recv_rows = P->max_recv;
  return MOE_OK;
}

}  // extern "C"
