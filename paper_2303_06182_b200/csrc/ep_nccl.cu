// Expert parallelism with the exchange over NCCL -- the transport north_star
// names ("variable-count token all-to-all uses NCCL over NVLink, preceded by
// a count exchange"), beside the peer-memory transport of ep_p2p.cu.
// C ABI: moe_nccl_get_unique_id, moe_ep_connect_nccl (include/moe_capi.h);
// moe_ep_forward dispatches here when the layer was created with
// transport = MOE_EP_TRANSPORT_NCCL.
//
// Reference behaviour replaced (proj/src/exchange.cpp:95-120,
// plan_dynamic_exchange), per forward on one stream:
//   size phase    ncclAllGather of every rank's per-key slot counts (E int32:
//                 for each destination its E/D local experts' counts -- the
//                 reference's E/D-count message per (src, dst) pair,
//                 exchange.cpp:100-104), then ONE host sync to size the
//                 payload messages;
//   payload phase gather of the token rows in (destination, local expert,
//                 slot) order, then grouped ncclSend/ncclRecv of exactly the
//                 assigned rows and their gate weights (exchange.cpp:106-114);
//   FFN           the received rows are regrouped by local expert (then
//                 source rank, then slot -- the single-GPU row order) and run
//                 through the same fused tcgen05 FFN as the peer transport;
//   return leg    outputs regrouped back to source order, grouped
//                 ncclSend/ncclRecv, then the weighted combine in slot order.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2; the process's copy
// when torch already loaded one), so the library has no link-time NCCL
// dependency and the peer transport works without it.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "ep_state.h"

namespace moe {
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

int nccl_api(const NcclApi** out) {
  static NcclApi api;
  static int status = -1;
  static std::string why;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (status < 0) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    status = MOE_OK;
    if (!h) {
      status = MOE_ERR_UNSUPPORTED;
      why = std::string("NCCL transport: cannot load libnccl.so.2 (") + dlerror() + ")";
    } else {
      auto sym = [&](auto& fn, const char* name) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
        if (!fn && status == MOE_OK) {
          status = MOE_ERR_UNSUPPORTED;
          why = std::string("NCCL transport: symbol ") + name + " missing";
        }
      };
      sym(api.GetUniqueId, "ncclGetUniqueId");
      sym(api.CommInitRank, "ncclCommInitRank");
      sym(api.CommDestroy, "ncclCommDestroy");
      sym(api.AllGather, "ncclAllGather");
      sym(api.Send, "ncclSend");
      sym(api.Recv, "ncclRecv");
      sym(api.GroupStart, "ncclGroupStart");
      sym(api.GroupEnd, "ncclGroupEnd");
      sym(api.GetErrorString, "ncclGetErrorString");
    }
  }
  if (status != MOE_OK) return fail(status, why);
  *out = &api;
  return MOE_OK;
}

int nccl_fail(const NcclApi* api, ncclResult_t r, const char* what) {
  return fail(MOE_ERR_CUDA, std::string(what) + ": " + api->GetErrorString(r));
}

#define MOE_NCCL(api, call)                                    \
  do {                                                         \
    ncclResult_t _r = (call);                                  \
    if (_r != ncclSuccess) return nccl_fail(api, _r, #call);   \
  } while (0)

// Row order conversion between the source-major receive layout of NCCL
// (source rank, then local expert, then slot) and the expert-grouped layout
// the FFN consumes (local expert, then source rank, then slot).
//   to_grouped = 1: src_major rows -> grouped rows (+ gate weights)
//   to_grouped = 0: grouped rows   -> src_major rows
// c(r, e) = counts_all[r * E + rank * El + e] rows from rank r for local
// expert e.  One warp per row, 16-byte vectors.
struct RegroupArgs {
  const int32_t* counts_all;  // [D, E]
  int rank, D, E, El, vpr, rows;
  uint4* grouped;
  uint4* src_major;
  float* w_grouped;
  const float* w_src_major;
  int to_grouped;
};

__global__ void __launch_bounds__(512) ep_regroup_kernel(RegroupArgs a) {
  __shared__ int32_t g_start[513];  // grouped segment j = e * D + r
  __shared__ int32_t m_start[513];  // source-major segment j = r * El + e
  const int n = a.D * a.El;         // == E <= 512
  const int q = threadIdx.x;
  if (q < n) {
    const int e = q / a.D, r = q % a.D;
    g_start[q + 1] = a.counts_all[r * a.E + a.rank * a.El + e];
    const int r2 = q / a.El, e2 = q % a.El;
    m_start[q + 1] = a.counts_all[r2 * a.E + a.rank * a.El + e2];
  }
  if (q == 0) g_start[0] = m_start[0] = 0;
  __syncthreads();
  // inclusive scans of the sizes (n <= 512: a short Hillis-Steele over smem)
  for (int d = 1; d < n; d <<= 1) {
    int vg = 0, vm = 0;
    if (q < n && q >= d) {
      vg = g_start[q + 1 - d];
      vm = m_start[q + 1 - d];
    }
    __syncthreads();
    if (q < n) {
      g_start[q + 1] += vg;
      m_start[q + 1] += vm;
    }
    __syncthreads();
  }
  const int lane = q & 31;
  const int wpb = blockDim.x >> 5;
  for (int g = blockIdx.x * wpb + (q >> 5); g < a.rows; g += gridDim.x * wpb) {
    int lo = 0, hi = n - 1;  // last grouped segment starting at or before g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (g_start[mid] <= g) lo = mid;
      else hi = mid - 1;
    }
    const int e = lo / a.D, r = lo % a.D;
    const int m = m_start[r * a.El + e] + (g - g_start[lo]);
    const uint4* src = a.to_grouped ? a.src_major + static_cast<size_t>(m) * a.vpr
                                    : a.grouped + static_cast<size_t>(g) * a.vpr;
    uint4* dst = a.to_grouped ? a.grouped + static_cast<size_t>(g) * a.vpr
                              : a.src_major + static_cast<size_t>(m) * a.vpr;
    for (int v = lane; v < a.vpr; v += 32) dst[v] = src[v];
    if (a.to_grouped && lane == 0) a.w_grouped[g] = a.w_src_major[m];
  }
}

int launch_regroup(moe_ep* P, int rows, bool to_grouped, cudaStream_t s) {
  if (rows <= 0) return MOE_OK;
  const moe_ep_desc& d = P->d;
  RegroupArgs a{};
  a.counts_all = reinterpret_cast<const int32_t*>(P->window + P->lay.counts_all);
  a.rank = d.rank;
  a.D = d.world_size;
  a.E = d.num_experts;
  a.El = P->El;
  a.vpr = d.token_dim / 8;
  a.rows = rows;
  a.grouped = reinterpret_cast<uint4*>(P->window + (to_grouped ? P->lay.recv_x : P->lay.recv_y));
  a.src_major = reinterpret_cast<uint4*>(P->recv_xs.p);
  a.w_grouped = reinterpret_cast<float*>(P->window + P->lay.recv_w);
  a.w_src_major = P->recv_ws.p;
  a.to_grouped = to_grouped ? 1 : 0;
  const int grid = std::max(1, std::min(P->ctx->sms * 4, (rows + 15) / 16));
  ep_regroup_kernel<<<grid, 512, 0, s>>>(a);
  MOE_CUDA(cudaGetLastError());
  return MOE_OK;
}

}  // namespace
}  // namespace moe

void ep_nccl_release(moe_ep* P) {
  if (P->nccl_comm) {
    const moe::NcclApi* api = nullptr;
    if (moe::nccl_api(&api) == MOE_OK) api->CommDestroy(static_cast<ncclComm_t>(P->nccl_comm));
    P->nccl_comm = nullptr;
  }
  if (P->host_counts) cudaFreeHost(P->host_counts);
  P->host_counts = nullptr;
  P->send_x.release();
  P->recv_xs.release();
  P->recv_ws.release();
}

int ep_forward_nccl(moe_ep* P, const void* X, int S, void* out, cudaStream_t s, bool timed) {
  using namespace moe;
  const NcclApi* api = nullptr;
  int st = nccl_api(&api);
  if (st) return st;
  const moe_ep_desc& d = P->d;
  auto mark = [&](int i) {
    if (timed && P->timing) cudaEventRecord(P->tev[i], s);
  };
  const int k = d.top_k, E = d.num_experts, TD = d.token_dim, D = d.world_size, El = P->El;
  const int me = d.rank;
  ncclComm_t comm = static_cast<ncclComm_t>(P->nccl_comm);
  if (X != P->tmX_ptr || S != P->tmX_rows) {
    if ((st = encode_bf16(&P->tmX, X, (uint64_t)S, TD, 128, gate_box_cols(E)))) return st;
    P->tmX_ptr = X;
    P->tmX_rows = S;
  }
  // 1. gate + route keyed by (device, local expert) -- local
  mark(0);
  GateArgs ga{S, TD, E, k, P->idx.p, P->w.p, nullptr};
  ga.X = X;
  ga.Wg = P->Wg;
  cudaError_t ce = launch_gate(P->tmX, P->tmWg, ga, s);
  if (ce != cudaSuccess) return cuda_fail(ce, "gate launch");
  st = route_common(P->ctx, P->idx.p, S, k, E, 0, P->counts.p, P->splits.p, P->order.p, P->pos.p,
                    P->w.p, P->wpos.p, nullptr, nullptr, nullptr, nullptr, 128, P->key_map.p, E, s);
  if (st) return st;
  // 2. size phase: every rank's per-key counts everywhere, one host sync
  mark(1);
  int32_t* counts_all = reinterpret_cast<int32_t*>(P->window + P->lay.counts_all);
  MOE_NCCL(api, api->AllGather(P->counts.p, counts_all, (size_t)E, ncclInt32, comm, s));
  MOE_CUDA(cudaMemcpyAsync(P->host_counts, counts_all, sizeof(int32_t) * D * E, cudaMemcpyDeviceToHost, s));
  MOE_CUDA(cudaStreamSynchronize(s));
  // rows[src][dst]: slots of rank src's tokens whose expert lives on dst
  std::vector<long> rows((size_t)D * D, 0);
  for (int src = 0; src < D; ++src)
    for (int dst = 0; dst < D; ++dst)
      for (int e = 0; e < El; ++e) rows[(size_t)src * D + dst] += P->host_counts[(size_t)src * E + dst * El + e];
  // every rank sees the same matrix, so a capacity failure is collective
  for (int dst = 0; dst < D; ++dst) {
    long in = 0;
    for (int src = 0; src < D; ++src) in += rows[(size_t)src * D + dst];
    if (in > P->max_recv)
      return fail(MOE_ERR_UNSUPPORTED, "expert-parallel receive capacity (max_recv_rows) exceeded");
  }
  std::vector<long> soff(D + 1, 0), roff(D + 1, 0);
  for (int p = 0; p < D; ++p) {
    soff[p + 1] = soff[p] + rows[(size_t)me * D + p];
    roff[p + 1] = roff[p] + rows[(size_t)p * D + me];
  }
  const int R = (int)roff[D];
  P->last_recv_rows = R;
  // 3. payload phase: rows in (destination, local expert, slot) order, then
  //    exactly the assigned rows and their gate weights to each owner
  mark(2);
  ce = launch_gather_rows(static_cast<const __nv_bfloat16*>(X), P->order.p, S * k, k, TD, P->send_x.p, s);
  if (ce != cudaSuccess) return cuda_fail(ce, "EP gather launch");
  MOE_NCCL(api, api->GroupStart());
  for (int p = 0; p < D; ++p) {
    const size_t ns = (size_t)(soff[p + 1] - soff[p]), nr = (size_t)(roff[p + 1] - roff[p]);
    if (ns) {
      MOE_NCCL(api, api->Send(P->send_x.p + (size_t)soff[p] * TD, ns * TD, ncclBfloat16, p, comm, s));
      MOE_NCCL(api, api->Send(P->wpos.p + soff[p], ns, ncclFloat32, p, comm, s));
    }
    if (nr) {
      MOE_NCCL(api, api->Recv(P->recv_xs.p + (size_t)roff[p] * TD, nr * TD, ncclBfloat16, p, comm, s));
      MOE_NCCL(api, api->Recv(P->recv_ws.p + roff[p], nr, ncclFloat32, p, comm, s));
    }
  }
  MOE_NCCL(api, api->GroupEnd());
  // 4. regroup by local expert, then the FFN work list
  mark(3);
  if ((st = launch_regroup(P, R, true, s))) return st;
  if ((st = ep_launch_recv(P, s, false))) return st;
  // 5. FFN
  mark(4);
  if ((st = ep_launch_ffn(P, s))) return st;
  // 6. return leg: outputs back to source order, then to their tokens' ranks
  //    (into send_x, which is in the keyed row order `pos` refers to)
  mark(5);
  if ((st = launch_regroup(P, R, false, s))) return st;
  MOE_NCCL(api, api->GroupStart());
  for (int p = 0; p < D; ++p) {
    const size_t ns = (size_t)(roff[p + 1] - roff[p]), nr = (size_t)(soff[p + 1] - soff[p]);
    if (ns) MOE_NCCL(api, api->Send(P->recv_xs.p + (size_t)roff[p] * TD, ns * TD, ncclBfloat16, p, comm, s));
    if (nr) MOE_NCCL(api, api->Recv(P->send_x.p + (size_t)soff[p] * TD, nr * TD, ncclBfloat16, p, comm, s));
  }
  MOE_NCCL(api, api->GroupEnd());
  // 7. weighted combine in slot order
  mark(6);
  ce = launch_combine(P->send_x.p, P->pos.p, S, k, TD, static_cast<__nv_bfloat16*>(out), s);
  if (ce != cudaSuccess) return cuda_fail(ce, "EP combine launch");
  mark(7);
  return MOE_OK;
}

extern "C" {

int moe_nccl_get_unique_id(void* id) {
  if (!id) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  static_assert(sizeof(ncclUniqueId) == MOE_NCCL_ID_BYTES, "NCCL unique id size");
  const moe::NcclApi* api = nullptr;
  int st = moe::nccl_api(&api);
  if (st) return st;
  ncclUniqueId u;
  MOE_NCCL(api, api->GetUniqueId(&u));
  memcpy(id, &u, sizeof u);
  return MOE_OK;
}

int moe_ep_connect_nccl(moe_ep* P, const void* id) {
  if (!P || !id) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (P->d.transport != MOE_EP_TRANSPORT_NCCL)
    return fail(MOE_ERR_INVALID_ARGUMENT, "layer was not created for the NCCL transport");
  if (P->connected) return fail(MOE_ERR_INVALID_ARGUMENT, "already connected");
  const moe::NcclApi* api = nullptr;
  int st = moe::nccl_api(&api);
  if (st) return st;
  MOE_CUDA(cudaSetDevice(P->ctx->device));
  const size_t TD = P->d.token_dim, Sk = (size_t)P->d.max_tokens * P->d.top_k;
  if ((st = P->send_x.reserve(Sk * TD)) || (st = P->recv_xs.reserve((size_t)P->max_recv * TD)) ||
      (st = P->recv_ws.reserve(P->max_recv)))
    return st;
  if (!P->host_counts)
    MOE_CUDA(cudaMallocHost(&P->host_counts, sizeof(int32_t) * P->d.world_size * P->d.num_experts));
  ncclUniqueId u;
  memcpy(&u, id, sizeof u);
  ncclComm_t comm = nullptr;
  MOE_NCCL(api, api->CommInitRank(&comm, P->d.world_size, u, P->d.rank));
  P->nccl_comm = comm;
  P->connected = true;
  return MOE_OK;
}

}  // extern "C"
