// C-ABI implementation: contexts, argument checking (reference error text),
// host-buffer drop-in entry points, TMA descriptor setup and the MoE layer
// (gate -> route -> gather -> grouped FFN x2 -> combine) with its workspace.
#include <mutex>

#include "capi_state.h"

namespace {

__global__ void inverse_order_kernel(const int32_t* order, int64_t n, int32_t* pos) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int s = order[p];
    if (s >= 0) pos[s] = (int32_t)p;
  }
}

// counts[src * D + dst]: slots of tokens resident on src (token t on t % n_src:
// round robin with n_src = D, single source with n_src = 1) routed to an
// expert placed on dst.
__global__ void exchange_counts_kernel(const int32_t* experts, int S, int k, int n_src, int D,
                                       const int32_t* device_of, int E,
                                       unsigned long long* counts, int32_t* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)S * k;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int e = experts[i];
    if (e < 0 || e >= E) {
      atomicOr(err, 1);
      continue;
    }
    const int src = (int)((i / k) % n_src);
    atomicAdd(&counts[(int64_t)src * D + device_of[e]], 1ull);
  }
}

}  // namespace

extern "C" {

int moe_version(void) { return MOE_CAPI_VERSION; }

const char* moe_status_string(int s) {
  switch (s) {
    case MOE_OK: return "ok";
    case MOE_ERR_INVALID_ARGUMENT: return "invalid argument";
    case MOE_ERR_CUDA: return "cuda error";
    case MOE_ERR_UNSUPPORTED: return "unsupported shape";
    case MOE_ERR_OUT_OF_MEMORY: return "out of memory";
    case MOE_ERR_EXPERT_RANGE: return "expert id out of range";
    case MOE_ERR_PEER_TIMEOUT: return "peer timeout";
    default: return "unknown status";
  }
}

const char* moe_last_error(void) { return g_last_error.c_str(); }

int moe_ctx_create(int device, moe_ctx** out) {
  if (!out) return fail(MOE_ERR_INVALID_ARGUMENT, "null output handle");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(MOE_ERR_CUDA, "no CUDA device available");
  if (device < 0 || device >= n) return fail(MOE_ERR_INVALID_ARGUMENT, "device out of range");
  MOE_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  MOE_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(MOE_ERR_UNSUPPORTED, "this library is built for sm_100a (B200) only");
  auto* c = new moe_ctx();
  c->device = device;
  c->sms = prop.multiProcessorCount;
  c->l2_bytes = static_cast<size_t>(prop.l2CacheSize);
  e = gemm_prepare();
  if (e == cudaSuccess) e = fused_ffn_prepare();
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "gemm_prepare");
  }
  int st = get_encoder();
  if (st) {
    delete c;
    return st;
  }
  *out = c;
  return MOE_OK;
}

int moe_ctx_destroy(moe_ctx* ctx) {
  if (!ctx) return MOE_OK;
  cudaSetDevice(ctx->device);
  ctx->block_hist.release();
  ctx->err_flag.release();
  ctx->drop_mark.release();
  ctx->static_splits.release();
  delete ctx;
  return MOE_OK;
}

int moe_ctx_sm_count(const moe_ctx* ctx) { return ctx ? ctx->sms : 0; }

int moe_device_alloc(moe_ctx* ctx, size_t bytes, void** out) {
  if (!ctx || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  MOE_CUDA(cudaSetDevice(ctx->device));
  cudaError_t e = cudaMalloc(out, bytes ? bytes : 1);
  if (e != cudaSuccess) return fail(MOE_ERR_OUT_OF_MEMORY, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return MOE_OK;
}

int moe_device_free(moe_ctx* ctx, void* ptr) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  MOE_CUDA(cudaFree(ptr));
  return MOE_OK;
}

int moe_host_alloc(moe_ctx* ctx, size_t bytes, void** out) {
  if (!ctx || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  cudaError_t e = cudaMallocHost(out, bytes ? bytes : 1);
  if (e != cudaSuccess) return fail(MOE_ERR_OUT_OF_MEMORY, std::string("cudaMallocHost: ") + cudaGetErrorString(e));
  return MOE_OK;
}

int moe_host_free(moe_ctx* ctx, void* ptr) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  MOE_CUDA(cudaFreeHost(ptr));
  return MOE_OK;
}

int moe_memcpy(moe_ctx* ctx, void* dst, const void* src, size_t bytes, int kind, void* stream) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  const cudaMemcpyKind k = kind == 0   ? cudaMemcpyHostToDevice
                           : kind == 1 ? cudaMemcpyDeviceToHost
                                       : cudaMemcpyDeviceToDevice;
  if (kind < 0 || kind > 2) return fail(MOE_ERR_INVALID_ARGUMENT, "bad copy kind");
  MOE_CUDA(cudaMemcpyAsync(dst, src, bytes, k, (cudaStream_t)stream));
  return MOE_OK;
}

int moe_stream_create(moe_ctx* ctx, void** out) {
  if (!ctx || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  MOE_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s;
  MOE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = s;
  return MOE_OK;
}

int moe_stream_destroy(moe_ctx* ctx, void* stream) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  MOE_CUDA(cudaStreamDestroy((cudaStream_t)stream));
  return MOE_OK;
}

int moe_stream_synchronize(moe_ctx* ctx, void* stream) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  MOE_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return MOE_OK;
}

int moe_expert_capacity(double capacity_factor, int seq_len) {
  // gating.cpp:22-28
  const double raw = capacity_factor * seq_len;
  const double nearest = std::round(raw);
  if (std::abs(raw - nearest) < 1e-9 * std::max(1.0, std::abs(raw)))
    return static_cast<int>(nearest);
  return static_cast<int>(std::ceil(raw));
}

extern "C++" {
int moe::capi::route_common(moe_ctx* ctx, const int32_t* expert_idx, int S, int k, int E, int cap,
                        int32_t* counts, int32_t* splits, int32_t* order, int32_t* pos,
                        const float* gate_w, float* wpos, int32_t* dropped, int32_t* n_dropped,
                        FfnItem* items, int32_t* n_items, int tile_n, const int32_t* key_map,
                        int num_keys_in, cudaStream_t stream, int32_t* item_off,
                        int32_t* zero, int zero_n) {
  int st = ctx->prepare_route(E);
  if (st) return st;
  if (cap > 0) {
    st = ctx->drop_mark.reserve((size_t)S * k);
    if (st) return st;
  }
  RouteArgs a{};
  a.expert_idx = expert_idx;
  a.key_map = key_map;
  a.num_keys_in = num_keys_in;
  a.num_experts = E;
  a.total_slots = S * k;
  a.top_k = k;
  a.capacity = cap;
  a.tile_n = tile_n;
  a.counts = counts;
  a.splits = splits;
  a.order = order;
  a.pos = pos;
  a.gate_w = gate_w;
  a.wpos = wpos;
  a.dropped = dropped;
  a.n_dropped = n_dropped;
  a.drop_mark = ctx->drop_mark.p;
  a.block_hist = ctx->block_hist.p;
  a.items = items;
  a.n_items = n_items;
  a.item_off = item_off;
  a.error_flag = ctx->err_flag.p;
  a.zero = zero;
  a.zero_n = zero ? zero_n : 0;
  cudaError_t e = launch_route(a, ctx->route_max_blocks, stream);
  if (e != cudaSuccess) return cuda_fail(e, "route kernel launch");
  return MOE_OK;
}
}  // extern "C++"

int moe_route_dynamic(moe_ctx* ctx, const int32_t* expert_idx, int S, int k, int E,
                      int32_t* counts, int32_t* splits, int32_t* order, int32_t* pos,
                      void* stream) {
  MOE_NVTX("moe.route_dynamic");
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  int st = check_batch(S, k, E);
  if (st) return st;
  if (!expert_idx || !counts || !splits || !order)
    return fail(MOE_ERR_INVALID_ARGUMENT, "null buffer");
  return route_common(ctx, expert_idx, S, k, E, 0, counts, splits, order, pos, nullptr, nullptr,
                      nullptr, nullptr, nullptr, nullptr, 128, nullptr, 0,
                      (cudaStream_t)stream);
}

int moe_route_static(moe_ctx* ctx, const int32_t* expert_idx, int S, int k, int E, int capacity,
                     int32_t* counts, int32_t* slots, int32_t* pos, int32_t* dropped,
                     int32_t* n_dropped, void* stream) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  int st = check_batch(S, k, E);
  if (st) return st;
  if (capacity <= 0) return fail(MOE_ERR_INVALID_ARGUMENT, "zero capacity");
  if (!expert_idx || !counts || !slots || !dropped || !n_dropped)
    return fail(MOE_ERR_INVALID_ARGUMENT, "null buffer");
  st = ctx->prepare_route(E);
  if (st) return st;
  // the splits are not an output of this entry point: context-owned scratch
  // (on the context's device, released with it)
  st = ctx->static_splits.reserve((size_t)E + 1);
  if (st) return st;
  return route_common(ctx, expert_idx, S, k, E, capacity, counts, ctx->static_splits.p, slots, pos, nullptr,
                      nullptr, dropped, n_dropped, nullptr, nullptr, 128, nullptr, 0,
                      (cudaStream_t)stream);
}

int moe_check_errors(moe_ctx* ctx, void* stream) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  MOE_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (!ctx->err_flag.p) return MOE_OK;
  int32_t flag = 0;
  MOE_CUDA(cudaMemcpy(&flag, ctx->err_flag.p, sizeof flag, cudaMemcpyDeviceToHost));
  if (flag) {
    MOE_CUDA(cudaMemset(ctx->err_flag.p, 0, sizeof(int32_t)));
    return fail(MOE_ERR_EXPERT_RANGE, "expert id out of range [0, num_experts)");
  }
  return MOE_OK;
}

int moe_dynamic_dispatch_host(moe_ctx* ctx, const int32_t* experts, int S, int k, int E,
                              int32_t* order, int32_t* counts, int32_t* splits) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  int st = check_batch(S, k, E);
  if (st) return st;
  MOE_CUDA(cudaSetDevice(ctx->device));
  const size_t n = (size_t)S * k;
  int32_t *d_idx = nullptr, *d_order = nullptr, *d_counts = nullptr, *d_splits = nullptr;
  MOE_CUDA(cudaMalloc(&d_idx, n * 4));
  MOE_CUDA(cudaMalloc(&d_order, n * 4));
  MOE_CUDA(cudaMalloc(&d_counts, (size_t)E * 4));
  MOE_CUDA(cudaMalloc(&d_splits, (size_t)(E + 1) * 4));
  int rc = MOE_OK;
  cudaError_t e = cudaMemcpy(d_idx, experts, n * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) rc = cuda_fail(e, "H2D experts");
  if (!rc) rc = moe_route_dynamic(ctx, d_idx, S, k, E, d_counts, d_splits, d_order, nullptr, 0);
  if (!rc) rc = moe_check_errors(ctx, 0);
  if (!rc) {
    cudaMemcpy(order, d_order, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(counts, d_counts, (size_t)E * 4, cudaMemcpyDeviceToHost);
    e = cudaMemcpy(splits, d_splits, (size_t)(E + 1) * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "D2H plan");
  }
  cudaFree(d_idx);
  cudaFree(d_order);
  cudaFree(d_counts);
  cudaFree(d_splits);
  return rc;
}

int moe_static_dispatch_host(moe_ctx* ctx, const int32_t* experts, int S, int k, int E,
                             double capacity_factor, int32_t* capacity, int32_t* slots,
                             int64_t slots_len, int32_t* dropped, int32_t* n_dropped) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  int st = check_batch(S, k, E);
  if (st) return st;
  // gating.cpp:37-42
  if (capacity_factor <= 0.0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "capacity factor must be positive in static mode");
  const int cap = moe_expert_capacity(capacity_factor, S);
  if (cap <= 0) return fail(MOE_ERR_INVALID_ARGUMENT, "zero capacity");
  *capacity = cap;
  if ((int64_t)E * cap > slots_len) return fail(MOE_ERR_INVALID_ARGUMENT, "slots buffer too small");
  MOE_CUDA(cudaSetDevice(ctx->device));
  const size_t n = (size_t)S * k, cells = (size_t)E * cap;
  int32_t *d_idx, *d_slots, *d_counts, *d_drop, *d_nd;
  MOE_CUDA(cudaMalloc(&d_idx, n * 4));
  MOE_CUDA(cudaMalloc(&d_slots, cells * 4));
  MOE_CUDA(cudaMalloc(&d_counts, (size_t)E * 4));
  MOE_CUDA(cudaMalloc(&d_drop, 2 * n * 4));
  MOE_CUDA(cudaMalloc(&d_nd, 4));
  int rc = MOE_OK;
  cudaError_t e = cudaMemcpy(d_idx, experts, n * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) rc = cuda_fail(e, "H2D experts");
  if (!rc) rc = moe_route_static(ctx, d_idx, S, k, E, cap, d_counts, d_slots, nullptr, d_drop, d_nd, 0);
  if (!rc) rc = moe_check_errors(ctx, 0);
  if (!rc) {
    cudaMemcpy(slots, d_slots, cells * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(n_dropped, d_nd, 4, cudaMemcpyDeviceToHost);
    e = cudaMemcpy(dropped, d_drop, (size_t)(*n_dropped) * 2 * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "D2H plan");
  }
  cudaFree(d_idx);
  cudaFree(d_slots);
  cudaFree(d_counts);
  cudaFree(d_drop);
  cudaFree(d_nd);
  return rc;
}

int moe_inverse_order_host(moe_ctx* ctx, const int32_t* order, int64_t n, int32_t* pos,
                           int64_t n_slots) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  if (n < 0 || n_slots < 0) return fail(MOE_ERR_INVALID_ARGUMENT, "negative size");
  for (int64_t i = 0; i < n; ++i)
    if (order[i] < -1 || order[i] >= n_slots)
      return fail(MOE_ERR_INVALID_ARGUMENT, "combine: payload count mismatch vs. plan");
  MOE_CUDA(cudaSetDevice(ctx->device));
  int32_t *d_order = nullptr, *d_pos = nullptr;
  MOE_CUDA(cudaMalloc(&d_order, (size_t)n * 4 + 4));
  MOE_CUDA(cudaMalloc(&d_pos, (size_t)n_slots * 4 + 4));
  int rc = MOE_OK;
  cudaMemcpy(d_order, order, (size_t)n * 4, cudaMemcpyHostToDevice);
  cudaMemset(d_pos, 0xff, (size_t)n_slots * 4);
  if (n > 0) inverse_order_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256>>>(d_order, n, d_pos);
  cudaError_t e = cudaMemcpy(pos, d_pos, (size_t)n_slots * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) rc = cuda_fail(e, "inverse order");
  cudaFree(d_order);
  cudaFree(d_pos);
  return rc;
}

int moe_exchange_counts_host(moe_ctx* ctx, const int32_t* experts, int S, int k, int D,
                             const int32_t* device_of, int E, int residency, int64_t* counts) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  int st = check_batch(S, k, E);
  if (st) return st;
  if (D < 1 || E % D != 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "num_experts must divide evenly across devices");
  if (residency != 0 && residency != 1) return fail(MOE_ERR_INVALID_ARGUMENT, "unknown residency");
  for (int e = 0; e < E; ++e)
    if (device_of[e] < 0 || device_of[e] >= D)
      return fail(MOE_ERR_INVALID_ARGUMENT, "device_of out of range");
  MOE_CUDA(cudaSetDevice(ctx->device));
  st = ctx->prepare_route(E);
  if (st) return st;
  // scratch freed on every path
  struct Scratch {
    DevBuf<int32_t> ids, dev;
    DevBuf<unsigned long long> c;
    ~Scratch() {
      ids.release();
      dev.release();
      c.release();
    }
  } w;
  if ((st = w.ids.reserve((size_t)S * k)) || (st = w.dev.reserve(E)) || (st = w.c.reserve((size_t)D * D)))
    return st;
  MOE_CUDA(cudaMemcpy(w.ids.p, experts, (size_t)S * k * 4, cudaMemcpyHostToDevice));
  MOE_CUDA(cudaMemcpy(w.dev.p, device_of, (size_t)E * 4, cudaMemcpyHostToDevice));
  MOE_CUDA(cudaMemset(w.c.p, 0, (size_t)D * D * 8));
  exchange_counts_kernel<<<std::max(1, std::min(4096, (S * k + 255) / 256)), 256>>>(
      w.ids.p, S, k, residency == 1 ? 1 : D, D, w.dev.p, E, w.c.p, ctx->err_flag.p);
  MOE_CUDA(cudaGetLastError());
  if ((st = moe_check_errors(ctx, 0))) return st;
  MOE_CUDA(cudaMemcpy(counts, w.c.p, (size_t)D * D * 8, cudaMemcpyDeviceToHost));
  return MOE_OK;
}

int moe_gate_topk(moe_ctx* ctx, const void* X, const void* Wg, int S, int TD, int E, int k,
                  int32_t* idx, float* w, float* logits, void* stream) {
  MOE_NVTX("moe.gate_topk");
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  int st = check_batch(S, k, E);
  if (st) return st;
  if (E > 512 || k > 8 || TD % 64 != 0)
    return fail(MOE_ERR_UNSUPPORTED, "gate supports E <= 512, k <= 8, TD % 64 == 0");
  cudaError_t e = gate_prepare(E);
  if (e != cudaSuccess) return cuda_fail(e, "gate_prepare");
  CUtensorMap tmX, tmWg;
  st = encode_bf16(&tmX, X, S, TD, 128, moe::gate_box_cols(E));
  if (st) return st;
  st = encode_bf16(&tmWg, Wg, E, TD, gate_box_rows(E), moe::gate_box_cols(E));
  if (st) return st;
  GateArgs a{S, TD, E, k, idx, w, logits};
  a.X = X;
  a.Wg = Wg;
  e = launch_gate(tmX, tmWg, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "gate launch");
  return MOE_OK;
}

int moe_gather_rows(moe_ctx* ctx, const void* X, const int32_t* order, int rows, int k, int TD,
                    void* Xp, void* stream) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  if (TD % 8 != 0) return fail(MOE_ERR_UNSUPPORTED, "TD must be a multiple of 8");
  cudaError_t e = launch_gather_rows((const __nv_bfloat16*)X, order, rows, k, TD,
                                     (__nv_bfloat16*)Xp, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "gather launch");
  return MOE_OK;
}

int moe_combine(moe_ctx* ctx, const void* Yw, const int32_t* pos, int S, int k, int TD, void* out,
                void* stream) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  if (TD % 8 != 0) return fail(MOE_ERR_UNSUPPORTED, "TD must be a multiple of 8");
  cudaError_t e = launch_combine((const __nv_bfloat16*)Yw, pos, S, k, TD, (__nv_bfloat16*)out,
                                 (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "combine launch");
  return MOE_OK;
}

int moe_fill_uniform_bf16(moe_ctx* ctx, void* dst, int64_t n, uint64_t seed, uint64_t tensor_id,
                          float scale, void* stream) {
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  cudaError_t e = launch_fill_uniform_bf16((__nv_bfloat16*)dst, n, seed, tensor_id, scale,
                                           (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "fill launch");
  return MOE_OK;
}

// ------------------------------------------------------------------ layer

// 256-token work items (many tokens per expert, e.g. cfg1: 8 experts x 256
// tokens) also go through the one-launch fused FFN: measured 0.0943 vs
// 0.1167 ms per cfg1 layer against the two-launch form (same box, A/B);
// MOE_FUSED_256=0 restores the two launches
static bool fused256_enabled() {
  static const int v = [] {
    const char* e = getenv("MOE_FUSED_256");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

int moe_layer_create(moe_ctx* ctx, const moe_layer_desc* desc, const void* Wg, const void* W1,
                     const void* W2, moe_layer** out) {
  if (!ctx || !desc || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  const moe_layer_desc& d = *desc;
  int st = check_batch(d.max_tokens, d.top_k, d.num_experts);
  if (st) return st;
  if (d.token_dim % 128 || d.hidden_dim % 128 || d.token_dim <= 0 || d.hidden_dim <= 0)
    return fail(MOE_ERR_UNSUPPORTED, "token_dim and hidden_dim must be positive multiples of 128");
  if (d.num_experts > 512 || d.top_k > 8)
    return fail(MOE_ERR_UNSUPPORTED, "num_experts <= 512 and top_k <= 8 are supported");
  if (d.mode != MOE_GATING_STATIC && d.mode != MOE_GATING_DYNAMIC)
    return fail(MOE_ERR_INVALID_ARGUMENT, "unknown gating mode");
  if (d.mode == MOE_GATING_STATIC && d.capacity_factor <= 0.0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "capacity factor must be positive in static mode");
  if (!Wg) return fail(MOE_ERR_INVALID_ARGUMENT, "null gate weight pointer");
  if (!W1 != !W2) return fail(MOE_ERR_INVALID_ARGUMENT, "W1 and W2 must both be given or both be NULL");
  const bool pool_only = !W1;
  if (pool_only && (d.mode != MOE_GATING_DYNAMIC || d.weights_packed))
    return fail(MOE_ERR_INVALID_ARGUMENT, "a pool-only layer (no W1/W2) needs dynamic gating, row-major pools");
  if (d.weights_packed && (d.mode != MOE_GATING_DYNAMIC || d.split_ffn || d.keep_layout))
    return fail(MOE_ERR_INVALID_ARGUMENT,
                "pre-packed weights need dynamic gating and the fused FFN (split_ffn, keep_layout 0)");
  if (d.fuse_combine && d.top_k != 1)
    return fail(MOE_ERR_UNSUPPORTED, "fuse_combine (GEMM2 stores the output rows) applies to top-1 layers");
  MOE_CUDA(cudaSetDevice(ctx->device));
  cudaError_t ce = gate_prepare(d.num_experts);
  if (ce != cudaSuccess) return cuda_fail(ce, "gate_prepare");

  auto* L = new moe_layer();
  L->ctx = ctx;
  L->d = d;
  L->Wg = Wg;
  L->W1 = W1;
  L->W2 = W2;
  const int S = d.max_tokens, k = d.top_k, E = d.num_experts;
  int cap = 0;
  if (d.mode == MOE_GATING_STATIC) {
    cap = moe_expert_capacity(d.capacity_factor, S);
    if (cap <= 0) {
      delete L;
      return fail(MOE_ERR_INVALID_ARGUMENT, "zero capacity");
    }
  }
  const long rows_l = d.mode == MOE_GATING_STATIC ? (long)E * cap : (long)S * k;
  if (rows_l > (1L << 30)) {
    delete L;
    return fail(MOE_ERR_UNSUPPORTED, "too many expert rows");
  }
  L->rows_max = (int)rows_l;
  const double avg = (double)L->rows_max / E;
  L->tile_n = d.tile_n ? d.tile_n : auto_tile_n(avg, E, d.token_dim, d.hidden_dim, ctx->sms);
  if (L->tile_n != 128 && L->tile_n != 256) {
    delete L;
    return fail(MOE_ERR_INVALID_ARGUMENT, "tile_n must be 0, 128 or 256");
  }
  L->items_max = d.mode == MOE_GATING_STATIC ? E * ((cap + L->tile_n - 1) / L->tile_n)
                                             : (S * k) / L->tile_n + E + 1;
  const size_t TD = d.token_dim, HD = d.hidden_dim, R = L->rows_max;
  // +16 rows of slack so a B tile of the last item never leaves the tensor
  const size_t Rp = R + 256;
  if ((st = L->idx.reserve((size_t)S * k)) || (st = L->w.reserve((size_t)S * k)) ||
      (st = L->pos.reserve((size_t)S * k)) || (st = L->counts.reserve(E)) ||
      (st = L->splits.reserve(E + 1)) || (st = L->order.reserve(R)) ||
      (st = L->wpos.reserve(R)) || (st = L->items.reserve(L->items_max)) ||
      (st = L->n_items.reserve(1)) || (st = L->err.reserve(1)) ||
      (st = L->item_off.reserve((size_t)E + 1)) ||
      (st = L->done.reserve(2 * (size_t)L->items_max + 1)) ||
      (st = L->xp.reserve(Rp * TD)) || (st = L->h.reserve(Rp * HD)) ||
      (st = L->yw.reserve(R * TD))) {
    moe_layer_destroy(L);
    return st;
  }
  if (d.mode == MOE_GATING_STATIC &&
      ((st = L->dropped.reserve((size_t)2 * S * k)) || (st = L->n_dropped.reserve(1)))) {
    moe_layer_destroy(L);
    return st;
  }
  if (d.keep_logits && (st = L->logits.reserve((size_t)S * E))) {
    moe_layer_destroy(L);
    return st;
  }
  cudaMemset(L->xp.p, 0, Rp * TD * 2);
  // no stale row index before the first forward: a slot whose expert id is
  // rejected (error flag) keeps pos = -1 and is skipped by the gather
  cudaMemset(L->pos.p, 0xff, sizeof(int32_t) * (size_t)S * k);
  cudaMemset(L->order.p, 0xff, sizeof(int32_t) * R);
  cudaMemset(L->h.p, 0, Rp * HD * 2);
  if ((st = encode_bf16(&L->tmWg, Wg, E, TD, moe::gate_box_rows(E), moe::gate_box_cols(E))) ||
      (!pool_only && !d.weights_packed &&
       ((st = encode_bf16(&L->tmW1, W1, (uint64_t)E * HD, TD, 128)) ||
        (st = encode_bf16(&L->tmW2, W2, (uint64_t)E * TD, HD, 128)))) ||
      (st = encode_bf16(&L->tmXp, L->xp.p, Rp, TD, 16)) ||
      (st = encode_bf16(&L->tmH, L->h.p, Rp, HD, 16)) ||
      (st = encode_rows(&L->xpm, L->xp.p, Rp, TD)) || (st = encode_rows(&L->hm, L->h.p, Rp, HD))) {
    moe_layer_destroy(L);
    return st;
  }
  if ((st = ctx->prepare_route(E))) {
    moe_layer_destroy(L);
    return st;
  }
  // weight prepack for the fused FFN's weight stream (contiguous 16 KB tiles
  // read ~5% faster than 128 B row pieces, tools/hbm_tma_read.cu); skipped
  // silently when the copy does not fit
  static const int pack_env = [] {
    const char* v = getenv("MOE_PACK");
    return v ? atoi(v) : 1;
  }();
  L->no_weights = pool_only;
  if (d.weights_packed) {
    // the caller's buffers are the packed tiles: stream them, keep no copy
    const size_t n1 = (size_t)E * HD * TD;
    if ((st = encode_packed(&L->tmW1p, W1, n1)) || (st = encode_packed(&L->tmW2p, W2, n1))) {
      moe_layer_destroy(L);
      return st;
    }
    L->packed = true;
    L->caller_packed = true;
  } else if (!pool_only && !d.keep_layout && pack_env && !d.split_ffn &&
             d.mode == MOE_GATING_DYNAMIC && (L->tile_n == 128 || fused256_enabled())) {
    const size_t n1 = (size_t)E * HD * TD;
    if (L->w1p.reserve(n1) == MOE_OK && L->w2p.reserve(n1) == MOE_OK &&
        encode_packed(&L->tmW1p, L->w1p.p, n1) == MOE_OK &&
        encode_packed(&L->tmW2p, L->w2p.p, n1) == MOE_OK) {
      L->packed = true;
      if ((st = moe_layer_repack(L, nullptr))) {
        moe_layer_destroy(L);
        return st;
      }
    } else {
      L->w1p.release();
      L->w2p.release();
      cudaGetLastError();
      g_last_error.clear();
    }
  }
  if (d.mode == MOE_GATING_STATIC && (st = ctx->drop_mark.reserve((size_t)S * k))) {
    moe_layer_destroy(L);
    return st;
  }
  *out = L;
  return MOE_OK;
}

int moe_layer_repack(moe_layer* L, void* stream) {
  if (!L) return fail(MOE_ERR_INVALID_ARGUMENT, "null layer");
  if (!L->packed || L->caller_packed) return MOE_OK;  // nothing copied: nothing to refresh
  cudaSetDevice(L->ctx->device);
  const moe_layer_desc& d = L->d;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_pack_tiles(static_cast<const __nv_bfloat16*>(L->W1), L->w1p.p,
                                    (long)d.num_experts * d.hidden_dim, d.token_dim, s);
  if (e == cudaSuccess)
    e = launch_pack_tiles(static_cast<const __nv_bfloat16*>(L->W2), L->w2p.p,
                          (long)d.num_experts * d.token_dim, d.hidden_dim, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "weight prepack");
  return MOE_OK;
}

int moe_pack_expert_weights(moe_ctx* ctx, const void* src, void* dst, int64_t rows, int K,
                            void* stream) {
  if (!ctx || !src || !dst) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (rows <= 0 || rows % 128 || K <= 0 || K % 64)
    return fail(MOE_ERR_INVALID_ARGUMENT, "rows must be a multiple of 128 and K a multiple of 64");
  MOE_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  const auto* in = static_cast<const __nv_bfloat16*>(src);
  auto* outp = static_cast<__nv_bfloat16*>(dst);
  cudaError_t e = cudaSuccess;
  if (src != dst) {
    const char *a = static_cast<const char*>(src), *b = static_cast<const char*>(dst);
    const size_t bytes = (size_t)rows * K * 2;
    if (a < b + bytes && b < a + bytes) return fail(MOE_ERR_INVALID_ARGUMENT, "src and dst overlap");
    e = launch_pack_tiles(in, outp, (long)rows, K, s);
  } else {
    // in place: a tile row-block occupies exactly the bytes of its 128 source
    // rows, so blocks of rows pack into a scratch and copy straight back
    const long block = std::max<long>(128, ((64L << 20) / ((long)K * 2)) / 128 * 128);
    DevBuf<__nv_bfloat16> tmp;
    int st = tmp.reserve((size_t)std::min<long>(block, (long)rows) * K);
    if (st) return st;
    for (long r0 = 0; r0 < rows && e == cudaSuccess; r0 += block) {
      const long n = std::min<long>(block, (long)rows - r0);
      e = launch_pack_tiles(in + (size_t)r0 * K, tmp.p, n, K, s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(outp + (size_t)r0 * K, tmp.p, (size_t)n * K * 2, cudaMemcpyDeviceToDevice, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    tmp.release();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "pack expert weights");
  return MOE_OK;
}

int moe_layer_destroy(moe_layer* L) {
  if (!L) return MOE_OK;
  cudaSetDevice(L->ctx->device);
  L->drop_graphs();
  for (cudaEvent_t e : L->tev) cudaEventDestroy(e);
  for (int b = 0; b < moe_layer::kPipeBufs; ++b) {
    if (L->ev_in[b]) cudaEventDestroy(L->ev_in[b]);
    if (L->ev_comp[b]) cudaEventDestroy(L->ev_comp[b]);
    if (L->ev_out[b]) cudaEventDestroy(L->ev_out[b]);
    L->pin[b].release();
    L->pout[b].release();
  }
  if (L->h2d) cudaStreamDestroy(L->h2d);
  if (L->d2h) cudaStreamDestroy(L->d2h);
  L->idx.release();
  L->w.release();
  L->pos.release();
  L->counts.release();
  L->splits.release();
  L->order.release();
  L->wpos.release();
  L->items.release();
  L->n_items.release();
  L->err.release();
  L->item_off.release();
  L->w1p.release();
  L->w2p.release();
  L->done.release();
  L->dropped.release();
  L->n_dropped.release();
  L->logits.release();
  L->xp.release();
  L->h.release();
  L->yw.release();
  L->xin.release();
  L->yout.release();
  delete L;
  return MOE_OK;
}

// Front of the layer: gate (or caller-provided routing), dispatch, gather.
// idx_in/w_in non-null = routed forward (trace replay, skewed workloads).
extern "C++" {
int moe::capi::layer_front(moe_layer* L, const void* X, int S, const int32_t* idx_in,
                       const float* w_in, cudaStream_t s, cudaEvent_t* ev) {
  const moe_layer_desc& d = L->d;
  auto mark = [&](int i) {
    if (ev) cudaEventRecord(ev[i], s);
  };
  if (S < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "empty batch");
  if (S > d.max_tokens) return fail(MOE_ERR_INVALID_ARGUMENT, "S exceeds max_tokens");
  const int k = d.top_k, E = d.num_experts, TD = d.token_dim;
  int st;
  L->counters_zeroed = false;
  const int32_t* idx = idx_in ? idx_in : L->idx.p;
  const float* w = idx_in ? w_in : L->w.p;
  // 1. gate
  mark(0);
  if (X != L->tmX_ptr || S != L->tmX_rows) {
    if ((st = encode_bf16(&L->tmX, X, (uint64_t)S, TD, 128, moe::gate_box_cols(L->d.num_experts))))
      return st;
    L->tmX_ptr = X;
    L->tmX_rows = S;
  }
  if (!idx_in) {
    GateArgs ga{S, TD, E, k, L->idx.p, L->w.p, d.keep_logits ? L->logits.p : nullptr};
    ga.X = X;
    ga.Wg = L->Wg;
    cudaError_t e = launch_gate(L->tmX, L->tmWg, ga, s);
    if (e != cudaSuccess) return cuda_fail(e, "gate launch");
  }
  // 2. route
  int cap = 0, rows = S * k;
  if (d.mode == MOE_GATING_STATIC) {
    cap = moe_expert_capacity(d.capacity_factor, S);
    rows = E * cap;
  }
  L->last_rows = rows;
  L->last_cap = cap;
  mark(1);
  st = route_common(L->ctx, idx, S, k, E, cap, L->counts.p, L->splits.p, L->order.p, L->pos.p, w,
                    L->wpos.p, L->dropped.p, L->n_dropped.p, L->items.p, L->n_items.p, L->tile_n,
                    nullptr, 0, s, L->item_off.p, L->done.p, 2 * L->items_max + 1);
  if (st) return st;
  L->counters_zeroed = true;
  // 3. gather token rows into expert-grouped order
  mark(2);
  cudaError_t e =
      d.mode == MOE_GATING_DYNAMIC && gather_by_token(k)
          ? launch_gather_tokens((const __nv_bfloat16*)X, L->pos.p, S, k, TD, L->xp.p, s)
          : launch_gather_rows((const __nv_bfloat16*)X, L->order.p, rows, k, TD, L->xp.p, s);
  if (e != cudaSuccess) return cuda_fail(e, "gather launch");
  return MOE_OK;
}
}  // extern "C++"

extern "C++" {
// Drop consumed H lines from L2 without write-back only when the layer's H
// does not fit comfortably in L2 (LM: 268 MB, MT: 101-201 MB): there the
// write-back would cost HBM bandwidth the weight stream needs.  A small H
// (configs[0]: 16.8 MB) stays dirty in L2 and the discard loop of the item's
// last consumer sat on the FFN's critical path (same box, cfg1 FFN
// 65.8 -> 61.0 us, step 81.1 -> 76.4 us).  MOE_FFN_DISCARD=0/1 forces it.
static int ffn_discard_h(const moe_ctx* ctx, size_t h_bytes) {
  static const int env = [] {
    const char* v = getenv("MOE_FFN_DISCARD");
    return v ? atoi(v) : -1;
  }();
  if (env >= 0) return env;
  return h_bytes > ctx->l2_bytes / 2 ? 1 : 0;
}

// Grouped FFN over the items of experts [e_lo, e_hi) (all items if e_lo < 0).
int moe::capi::layer_ffn(moe_layer* L, cudaStream_t s, int e_lo, int e_hi, cudaEvent_t* ev) {
  const int TD = L->d.token_dim, HD = L->d.hidden_dim;
  auto mark = [&](int i) {
    if (ev) cudaEventRecord(ev[i], s);
  };
  if (L->no_weights && !L->slot_of)
    return fail(MOE_ERR_INVALID_ARGUMENT, "layer has no expert weights: attach an expert cache (moe_cache_create)");
  const int32_t* off = e_lo >= 0 ? L->item_off.p : nullptr;
  const bool fcomb = layer_fused_combine(L);
  mark(3);
  // fused single launch in the weight-streaming regime (dynamic gating, many
  // small items); compute-bound static batches and few-expert layers (cfg1)
  // measured faster as two launches (profiles/r01_fused_ffn.md)
  // static gating too (capacity-padded items, zero placeholder rows): one
  // launch measured 7.95 vs 8.65 ms (LM CF=0.05) and 46.8 vs 56.6 ms (MT CF=1)
  // against two (same box); MOE_FUSED_STATIC=0 restores the two launches
  static const int fused_static = [] {
    const char* e = getenv("MOE_FUSED_STATIC");
    return e ? atoi(e) : 1;
  }();
  const bool one_launch = !L->d.split_ffn &&
                          (L->d.mode == MOE_GATING_DYNAMIC || fused_static) &&
                          (L->tile_n == 128 || fused256_enabled());
  if (one_launch) {
    // one persistent launch for both GEMMs, H kept in L2 (ffn_fused.cu)
    // the route kernel zeroed the counters for a whole-layer FFN; expert-range
    // waves (expert cache) share the tile counter and need a fresh one each
    if (!(e_lo < 0 && L->counters_zeroed))
      MOE_CUDA(cudaMemsetAsync(L->done.p, 0, sizeof(int32_t) * (2 * (size_t)L->items_max + 1), s));
    L->counters_zeroed = false;
    FusedFfnArgs fa{};
    fa.items = L->items.p;
    fa.n_items = L->n_items.p;
    fa.item_off = off;
    fa.e_lo = e_lo;
    fa.e_hi = e_hi;
    fa.slot_of = L->slot_of;
    fa.TD = TD;
    fa.HD = HD;
    fa.H = L->h.p;
    fa.Yw = L->yw.p;
    fa.wpos = L->wpos.p;
    fa.done1 = L->done.p;
    fa.done2 = L->done.p + L->items_max;
    fa.tile_ctr = L->done.p + 2 * L->items_max;
    // an item's GEMM2 tiles trail its GEMM1 tiles by ~8 waves of CTAs
    // (measured on the LM shape: 4 waves 1.49 ms, 8 waves 1.375 ms, 16 waves
    // 1.43 ms FFN; profiles/r01_fused_ffn.md); MOE_FFN_LAG overrides (items)
    static const int lag_env = [] {
      const char* v = getenv("MOE_FFN_LAG");
      return v ? atoi(v) : 0;
    }();
    const int per_item = HD / 128 + TD / 128;
    // dynamic gating at 256-token items (MT at seq 256: ~1 item per expert,
    // MMA-heavy tiles) runs best with (nearly) every GEMM1 tile ahead of GEMM2:
    // 8x the lag (same box, FFN 1686-1689 -> 1652-1662 us at 4x,
    // profiles/r02_s24_l256_lag_ab.txt; 1637-1647 vs 1653-1664 us at 8x vs 4x,
    // r02_s26_l256_lag_tail.txt;
    // the static capacity-padded items and 128-token items lose 3-6 % with it,
    // profiles/r02_s22_lag_256_items.txt)
    const int lag_mult = (L->d.mode == MOE_GATING_DYNAMIC && L->tile_n == 256) ? 8 : 1;
    const int lag = lag_env > 0 ? lag_env
                                : lag_mult * std::max(2, (8 * L->ctx->sms + per_item - 1) / per_item);
    fa.lag = lag;
    fa.discard_h = ffn_discard_h(L->ctx, (size_t)L->rows_max * HD * 2);
    fa.dbg = getenv("MOE_FFN_DBG") ? atoi(getenv("MOE_FFN_DBG")) : 0;
    // the expert-cache slot pool is row-major: packed tiles only for the layer's own weights
    fa.packed = L->packed && !L->slot_of;
    fa.W1p = L->caller_packed ? L->W1 : L->w1p.p;
    fa.W2p = L->caller_packed ? L->W2 : L->w2p.p;
    fa.pair_hint = auto_pair((double)L->rows_max / L->d.num_experts, L->d.num_experts, TD, HD,
                             L->tile_n, L->ctx->sms);
    if (fcomb) {
      // top-1: one contribution per token, GEMM2 writes the layer output row directly
      fa.Yw = static_cast<__nv_bfloat16*>(L->fwd_out);
      fa.out_rows = L->order.p;
    }
    L->last_ffn_kernel = fused_ffn_uses_pair(fa, L->tile_n) ? 2 : 1;
    cudaError_t e = launch_fused_ffn(fa.packed ? L->tmW1p : L->tmW1, L->xpm,
                                     fa.packed ? L->tmW2p : L->tmW2, L->hm, fa, L->tile_n,
                                     L->ctx->sms, s);
    if (e != cudaSuccess) return cuda_fail(e, "fused ffn launch");
    mark(4);
    return MOE_OK;
  }
  L->last_ffn_kernel = 0;
  GemmArgs g1{L->items.p, L->n_items.p, L->slot_of, HD, TD, kEpiReluBf16, L->h.p, nullptr, nullptr,
              off, e_lo, e_hi};
  cudaError_t e = launch_grouped_gemm(L->tmW1, L->tmXp, g1, L->tile_n, L->ctx->sms, s);
  if (e != cudaSuccess) return cuda_fail(e, "grouped gemm 1 launch");
  mark(4);
  GemmArgs g2{L->items.p, L->n_items.p, L->slot_of, TD, HD, kEpiScaleBf16, L->yw.p, L->wpos.p,
              nullptr, off, e_lo, e_hi};
  if (fcomb) {
    // top-1: one contribution per token, write the layer output directly (row -> token)
    g2.out = static_cast<__nv_bfloat16*>(L->fwd_out);
    g2.out_rows = L->order.p;
  }
  e = launch_grouped_gemm(L->tmW2, L->tmH, g2, L->tile_n, L->ctx->sms, s);
  if (e != cudaSuccess) return cuda_fail(e, "grouped gemm 2 launch");
  return MOE_OK;
}
}  // extern "C++"

extern "C++" {
int moe::capi::layer_back(moe_layer* L, int S, void* out, cudaStream_t s, cudaEvent_t* ev) {
  auto mark = [&](int i) {
    if (ev) cudaEventRecord(ev[i], s);
  };
  mark(5);
  if (!layer_fused_combine(L)) {
    cudaError_t e = launch_combine(L->yw.p, L->pos.p, S, L->d.top_k, L->d.token_dim,
                                   (__nv_bfloat16*)out, s);
    if (e != cudaSuccess) return cuda_fail(e, "combine launch");
  }
  mark(6);
  return MOE_OK;
}
}  // extern "C++"

extern "C++" {
static int layer_forward_impl(moe_layer* L, const void* X, int S, void* out, cudaStream_t s,
                              bool timed = false, const int32_t* idx_in = nullptr,
                              const float* w_in = nullptr) {
  cudaEvent_t* ev = nullptr;
  if (timed && L->t_slots > 0) {
    ev = &L->tev[(size_t)(L->t_calls % L->t_slots) * (MOE_NUM_STAGES + 1)];
    ++L->t_calls;
  }
  int st;
  L->fwd_out = out;
  if ((st = layer_front(L, X, S, idx_in, w_in, s, ev))) return st;
  if ((st = layer_ffn(L, s, -1, -1, ev))) return st;
  return layer_back(L, S, out, s, ev);
}
}  // extern "C++"

int moe_layer_forward_routed(moe_layer* L, const void* X, const int32_t* idx, const float* w, int S,
                             void* out, void* stream) {
  MOE_NVTX("moe.layer_forward_routed");
  if (!L || !X || !out || !idx || !w) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  return layer_forward_impl(L, X, S, out, (cudaStream_t)stream, true, idx, w);
}

int moe_layer_forward(moe_layer* L, const void* X, int S, void* out, void* stream) {
  MOE_NVTX("moe.layer_forward");
  if (!L || !X || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  return layer_forward_impl(L, X, S, out, (cudaStream_t)stream, true);
}

int moe_layer_enable_timing(moe_layer* L, int n_slots) {
  if (!L || n_slots < 0) return fail(MOE_ERR_INVALID_ARGUMENT, "bad timing request");
  for (cudaEvent_t e : L->tev) cudaEventDestroy(e);
  L->tev.clear();
  L->t_slots = 0;
  L->t_calls = 0;
  for (int i = 0; i < n_slots * (MOE_NUM_STAGES + 1); ++i) {
    cudaEvent_t e;
    MOE_CUDA(cudaEventCreate(&e));
    L->tev.push_back(e);
  }
  L->t_slots = n_slots;
  return MOE_OK;
}

int moe_layer_stage_times(moe_layer* L, int slot, float* ms) {
  if (!L || !ms || slot < 0 || slot >= L->t_slots)
    return fail(MOE_ERR_INVALID_ARGUMENT, "bad timing slot");
  cudaEvent_t* ev = &L->tev[(size_t)slot * (MOE_NUM_STAGES + 1)];
  MOE_CUDA(cudaEventSynchronize(ev[MOE_NUM_STAGES]));
  for (int i = 0; i < MOE_NUM_STAGES; ++i) MOE_CUDA(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
  return MOE_OK;
}

int moe_layer_forward_graph(moe_layer* L, const void* X, int S, void* out, void* stream) {
  MOE_NVTX("moe.layer_forward_graph");
  if (!L || !X || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  moe_layer::GraphEntry* hit = nullptr;
  for (moe_layer::GraphEntry& g : L->graphs)
    if (g.exec && g.x == X && g.out == out && g.S == S && g.stream == s) hit = &g;
  if (!hit) {
    if (s == nullptr) return fail(MOE_ERR_INVALID_ARGUMENT, "graph capture needs a non-default stream");
    hit = &L->graphs[0];
    for (moe_layer::GraphEntry& g : L->graphs)
      if (g.used < hit->used) hit = &g;  // LRU (unused entries have used == 0)
    if (hit->exec) cudaGraphExecDestroy(hit->exec);
    *hit = moe_layer::GraphEntry{};
    MOE_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    int st = layer_forward_impl(L, X, S, out, s);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    if (st) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(e, "end capture");
    e = cudaGraphInstantiate(&hit->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      hit->exec = nullptr;
      return cuda_fail(e, "graph instantiate");
    }
    hit->x = X;
    hit->out = out;
    hit->S = S;
    hit->stream = s;
  }
  hit->used = ++L->graph_clock;
  MOE_CUDA(cudaGraphLaunch(hit->exec, s));
  return MOE_OK;
}

int moe_layer_forward_host(moe_layer* L, const void* X_host, int S, void* out_host, void* stream) {
  MOE_NVTX("moe.layer_forward_host");
  if (!L || !X_host || !out_host) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  const size_t bytes = (size_t)L->d.max_tokens * L->d.token_dim * 2;
  int st;
  if ((st = L->xin.reserve(bytes / 2)) || (st = L->yout.reserve(bytes / 2))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t nb = (size_t)S * L->d.token_dim * 2;
  MOE_CUDA(cudaMemcpyAsync(L->xin.p, X_host, nb, cudaMemcpyHostToDevice, s));
  st = layer_forward_impl(L, L->xin.p, S, L->yout.p, s);
  if (st) return st;
  MOE_CUDA(cudaMemcpyAsync(out_host, L->yout.p, nb, cudaMemcpyDeviceToHost, s));
  MOE_CUDA(cudaStreamSynchronize(s));
  return moe_check_errors(L->ctx, s);
}

int moe_layer_forward_host_batches(moe_layer* L, const void* const* X_host, const int* S,
                                   void* const* out_host, int n, void* stream) {
  MOE_NVTX("moe.layer_forward_host_batches");
  if (!L || n < 0 || (n > 0 && (!X_host || !S || !out_host)))
    return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (!stream) return fail(MOE_ERR_INVALID_ARGUMENT, "pipelined forward needs a non-default stream");
  for (int i = 0; i < n; ++i) {
    if (!X_host[i] || !out_host[i]) return fail(MOE_ERR_INVALID_ARGUMENT, "null batch buffer");
    if (S[i] < 1 || S[i] > L->d.max_tokens)
      return fail(MOE_ERR_INVALID_ARGUMENT, "batch size outside [1, max_tokens]");
  }
  cudaSetDevice(L->ctx->device);
  const size_t elems = (size_t)L->d.max_tokens * L->d.token_dim;
  int st;
  constexpr int NB = moe_layer::kPipeBufs;
  for (int b = 0; b < NB; ++b)
    if ((st = L->pin[b].reserve(elems)) || (st = L->pout[b].reserve(elems))) return st;
  if (!L->h2d) {
    MOE_CUDA(cudaStreamCreateWithFlags(&L->h2d, cudaStreamNonBlocking));
    MOE_CUDA(cudaStreamCreateWithFlags(&L->d2h, cudaStreamNonBlocking));
    for (int b = 0; b < NB; ++b) {
      MOE_CUDA(cudaEventCreateWithFlags(&L->ev_in[b], cudaEventDisableTiming));
      MOE_CUDA(cudaEventCreateWithFlags(&L->ev_comp[b], cudaEventDisableTiming));
      MOE_CUDA(cudaEventCreateWithFlags(&L->ev_out[b], cudaEventDisableTiming));
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  // the copy streams start after whatever the caller queued on `stream`
  for (int b = 0; b < NB; ++b) MOE_CUDA(cudaEventRecord(L->ev_comp[b], s));
  MOE_CUDA(cudaStreamWaitEvent(L->h2d, L->ev_comp[0], 0));
  MOE_CUDA(cudaStreamWaitEvent(L->d2h, L->ev_comp[0], 0));
  // experiments (MOE_HOST_PIPE_PROF=1): timing events around every copy and
  // compute, a per-batch timeline printed for a few steady-state batches
  static const bool prof = getenv("MOE_HOST_PIPE_PROF") != nullptr;
  std::vector<cudaEvent_t> pev;
  if (prof) {
    pev.resize((size_t)n * 6);
    for (cudaEvent_t& e : pev) cudaEventCreate(&e);
  }
  auto rec = [&](int i, int j, cudaStream_t st_) {
    if (prof) cudaEventRecord(pev[(size_t)i * 6 + j], st_);
  };
  for (int i = 0; i < n; ++i) {
    const int b = i % NB;
    const size_t nb = (size_t)S[i] * L->d.token_dim * 2;
    // batch i's input lands in pin[b] once batch i-NB's compute has consumed it
    // (three buffers: the upload of batch i overlaps the compute of i-1 and i-2)
    MOE_CUDA(cudaStreamWaitEvent(L->h2d, L->ev_comp[b], 0));
    rec(i, 0, L->h2d);
    MOE_CUDA(cudaMemcpyAsync(L->pin[b].p, X_host[i], nb, cudaMemcpyHostToDevice, L->h2d));
    rec(i, 1, L->h2d);
    MOE_CUDA(cudaEventRecord(L->ev_in[b], L->h2d));
    // compute waits for its input and for batch i-NB's read-back of pout[b]
    MOE_CUDA(cudaStreamWaitEvent(s, L->ev_in[b], 0));
    if (i >= NB) MOE_CUDA(cudaStreamWaitEvent(s, L->ev_out[b], 0));
    rec(i, 2, s);
    if ((st = moe_layer_forward_graph(L, L->pin[b].p, S[i], L->pout[b].p, s))) return st;
    rec(i, 3, s);
    MOE_CUDA(cudaEventRecord(L->ev_comp[b], s));
    MOE_CUDA(cudaStreamWaitEvent(L->d2h, L->ev_comp[b], 0));
    rec(i, 4, L->d2h);
    MOE_CUDA(cudaMemcpyAsync(out_host[i], L->pout[b].p, nb, cudaMemcpyDeviceToHost, L->d2h));
    rec(i, 5, L->d2h);
    MOE_CUDA(cudaEventRecord(L->ev_out[b], L->d2h));
  }
  MOE_CUDA(cudaStreamSynchronize(L->h2d));
  MOE_CUDA(cudaStreamSynchronize(L->d2h));
  MOE_CUDA(cudaStreamSynchronize(s));
  if (prof) {
    for (int i = n / 2; i < std::min(n, n / 2 + 4); ++i) {
      float t[6];
      for (int j = 0; j < 6; ++j) cudaEventElapsedTime(&t[j], pev[0], pev[(size_t)i * 6 + j]);
      fprintf(stderr, "[host pipe] batch %d: h2d %.1f-%.1f  compute %.1f-%.1f  d2h %.1f-%.1f us\n", i,
              t[0] * 1e3, t[1] * 1e3, t[2] * 1e3, t[3] * 1e3, t[4] * 1e3, t[5] * 1e3);
    }
    for (cudaEvent_t e : pev) cudaEventDestroy(e);
  }
  return moe_check_errors(L->ctx, s);
}

int moe_route_dynamic_keyed(moe_ctx* ctx, const int32_t* expert_idx, int S, int k,
                            int num_experts, const int32_t* key_map, int num_keys,
                            int32_t* counts, int32_t* splits, int32_t* order, int32_t* pos,
                            const float* gate_w, float* wpos, void* stream) {
  MOE_NVTX("moe.route_dynamic_keyed");
  if (!ctx) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  int st = check_batch(S, k, num_experts);
  if (st) return st;
  if (num_keys < 1 || !key_map) return fail(MOE_ERR_INVALID_ARGUMENT, "bad key map");
  if (!expert_idx || !counts || !splits || !order)
    return fail(MOE_ERR_INVALID_ARGUMENT, "null buffer");
  return route_common(ctx, expert_idx, S, k, num_keys, 0, counts, splits, order, pos, gate_w, wpos,
                      nullptr, nullptr, nullptr, nullptr, 128, key_map, num_experts,
                      (cudaStream_t)stream);
}

int moe_fill_segments(moe_ctx* ctx, const int32_t* counts, int n_segments, int mod, int32_t* out,
                      void* stream) {
  if (!ctx || mod < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "bad argument");
  cudaError_t e = launch_fill_segments(counts, n_segments, mod, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "fill_segments launch");
  return MOE_OK;
}

int moe_ffn_create(moe_ctx* ctx, const moe_ffn_desc* desc, const void* W1, const void* W2,
                   moe_ffn** out) {
  if (!ctx || !desc || !out || !W1 || !W2) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  const moe_ffn_desc& d = *desc;
  if (d.max_rows < 1 || d.num_experts < 1)
    return fail(MOE_ERR_INVALID_ARGUMENT, "max_rows and num_experts must be positive");
  if (d.token_dim % 128 || d.hidden_dim % 128 || d.token_dim <= 0 || d.hidden_dim <= 0)
    return fail(MOE_ERR_UNSUPPORTED, "token_dim and hidden_dim must be positive multiples of 128");
  MOE_CUDA(cudaSetDevice(ctx->device));
  auto* F = new moe_ffn();
  F->ctx = ctx;
  F->d = d;
  const double avg = (double)d.max_rows / d.num_experts;
  F->tile_n = d.tile_n ? d.tile_n : auto_tile_n(avg, d.num_experts, d.token_dim, d.hidden_dim, ctx->sms);
  if (F->tile_n != 128 && F->tile_n != 256) {
    delete F;
    return fail(MOE_ERR_INVALID_ARGUMENT, "tile_n must be 0, 128 or 256");
  }
  const size_t R = d.max_rows, Rp = R + 256, TD = d.token_dim, HD = d.hidden_dim;
  const size_t items_max = R / F->tile_n + d.num_experts + 1;
  F->items_max = (int)items_max;
  int st;
  if ((st = F->counts.reserve(d.num_experts)) || (st = F->splits.reserve(d.num_experts + 1)) ||
      (st = F->order.reserve(R)) || (st = F->pos.reserve(R)) || (st = F->n_items.reserve(1)) ||
      (st = F->wpos.reserve(R)) || (st = F->ones.reserve(R)) ||
      (st = F->items.reserve(items_max)) || (st = F->xp.reserve(Rp * TD)) ||
      (st = F->done.reserve(2 * items_max + 1)) ||
      (st = F->h.reserve(Rp * HD)) || (st = ctx->prepare_route(d.num_experts))) {
    moe_ffn_destroy(F);
    return st;
  }
  cudaMemset(F->xp.p, 0, Rp * TD * 2);
  cudaMemset(F->h.p, 0, Rp * HD * 2);
  {
    std::vector<float> one(R, 1.0f);
    cudaMemcpy(F->ones.p, one.data(), R * sizeof(float), cudaMemcpyHostToDevice);
  }
  if ((st = encode_bf16(&F->tmW1, W1, (uint64_t)d.num_experts * HD, TD, 128)) ||
      (st = encode_bf16(&F->tmW2, W2, (uint64_t)d.num_experts * TD, HD, 128)) ||
      (st = encode_bf16(&F->tmXp, F->xp.p, Rp, TD, 16)) ||
      (st = encode_bf16(&F->tmH, F->h.p, Rp, HD, 16)) ||
      (st = encode_rows(&F->xpm, F->xp.p, Rp, TD)) || (st = encode_rows(&F->hm, F->h.p, Rp, HD))) {
    moe_ffn_destroy(F);
    return st;
  }
  // packed weight copy for the fused path (as moe_layer_create)
  static const int pack_env = [] {
    const char* v = getenv("MOE_PACK");
    return v ? atoi(v) : 1;
  }();
  if (pack_env && (F->tile_n == 128 || fused256_enabled())) {
    const size_t n1 = (size_t)d.num_experts * HD * TD;
    if (F->w1p.reserve(n1) == MOE_OK && F->w2p.reserve(n1) == MOE_OK &&
        encode_packed(&F->tmW1p, F->w1p.p, n1) == MOE_OK &&
        encode_packed(&F->tmW2p, F->w2p.p, n1) == MOE_OK &&
        launch_pack_tiles(static_cast<const __nv_bfloat16*>(W1), F->w1p.p,
                          (long)d.num_experts * HD, TD, nullptr) == cudaSuccess &&
        launch_pack_tiles(static_cast<const __nv_bfloat16*>(W2), F->w2p.p,
                          (long)d.num_experts * TD, HD, nullptr) == cudaSuccess &&
        cudaDeviceSynchronize() == cudaSuccess) {
      F->packed = true;
    } else {
      F->w1p.release();
      F->w2p.release();
      cudaGetLastError();
      g_last_error.clear();
    }
  }
  *out = F;
  return MOE_OK;
}

int moe_ffn_destroy(moe_ffn* F) {
  if (!F) return MOE_OK;
  F->counts.release();
  F->splits.release();
  F->order.release();
  F->pos.release();
  F->n_items.release();
  F->done.release();
  F->wpos.release();
  F->ones.release();
  F->items.release();
  F->xp.release();
  F->h.release();
  F->w1p.release();
  F->w2p.release();
  delete F;
  return MOE_OK;
}

int moe_ffn_forward(moe_ffn* F, const void* X_rows, const int32_t* keys, const float* row_w,
                    int rows, void* Y_rows, void* stream) {
  if (!F || !X_rows || !keys || !Y_rows) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (rows < 0 || rows > F->d.max_rows) return fail(MOE_ERR_INVALID_ARGUMENT, "rows out of range");
  if (rows == 0) return MOE_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int TD = F->d.token_dim, HD = F->d.hidden_dim;
  int st = route_common(F->ctx, keys, rows, 1, F->d.num_experts, 0, F->counts.p, F->splits.p,
                        F->order.p, F->pos.p, row_w ? row_w : F->ones.p, F->wpos.p, nullptr,
                        nullptr, F->items.p, F->n_items.p, F->tile_n, nullptr, 0, s);
  if (st) return st;
  cudaError_t e = launch_gather_rows((const __nv_bfloat16*)X_rows, F->order.p, rows, 1, TD,
                                     F->xp.p, s);
  if (e != cudaSuccess) return cuda_fail(e, "gather launch");
  if (F->tile_n == 128 || fused256_enabled()) {
    // weight-streaming regime: one persistent launch, H kept in L2, the
    // output rows written straight back to the received order
    MOE_CUDA(cudaMemsetAsync(F->done.p, 0, sizeof(int32_t) * (2 * (size_t)F->items_max + 1), s));
    FusedFfnArgs fa{};
    fa.items = F->items.p;
    fa.n_items = F->n_items.p;
    fa.TD = TD;
    fa.HD = HD;
    fa.H = F->h.p;
    fa.Yw = (__nv_bfloat16*)Y_rows;
    fa.out_rows = F->order.p;
    fa.wpos = F->wpos.p;
    fa.done1 = F->done.p;
    fa.done2 = F->done.p + F->items_max;
    fa.tile_ctr = F->done.p + 2 * F->items_max;
    const int per_item = HD / 128 + TD / 128;
    fa.lag = std::max(2, (8 * F->ctx->sms + per_item - 1) / per_item);
    fa.discard_h = ffn_discard_h(F->ctx, (size_t)F->d.max_rows * HD * 2);
    fa.packed = F->packed;
    fa.W1p = F->w1p.p;
    fa.W2p = F->w2p.p;
    fa.pair_hint = auto_pair((double)F->d.max_rows / F->d.num_experts, F->d.num_experts, TD, HD,
                             F->tile_n, F->ctx->sms);
    e = launch_fused_ffn(F->packed ? F->tmW1p : F->tmW1, F->xpm, F->packed ? F->tmW2p : F->tmW2,
                         F->hm, fa, F->tile_n, F->ctx->sms, s);
    if (e != cudaSuccess) return cuda_fail(e, "fused ffn launch");
    return MOE_OK;
  }
  GemmArgs g1{F->items.p, F->n_items.p, nullptr, HD, TD, kEpiReluBf16, F->h.p, nullptr, nullptr};
  e = launch_grouped_gemm(F->tmW1, F->tmXp, g1, F->tile_n, F->ctx->sms, s);
  if (e != cudaSuccess) return cuda_fail(e, "grouped gemm 1 launch");
  GemmArgs g2{F->items.p, F->n_items.p, nullptr, TD, HD, kEpiScaleBf16, (__nv_bfloat16*)Y_rows,
              F->wpos.p, F->order.p};
  e = launch_grouped_gemm(F->tmW2, F->tmH, g2, F->tile_n, F->ctx->sms, s);
  if (e != cudaSuccess) return cuda_fail(e, "grouped gemm 2 launch");
  return MOE_OK;
}

int moe_layer_get_view(moe_layer* L, moe_layer_view* v) {
  if (!L || !v) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  v->idx = L->idx.p;
  v->w = L->w.p;
  v->logits = L->logits.p;
  v->counts = L->counts.p;
  v->splits = L->splits.p;
  v->order = L->order.p;
  v->pos = L->pos.p;
  v->dropped = L->dropped.p;
  v->n_dropped = L->n_dropped.p;
  v->xp = L->xp.p;
  v->h = L->h.p;
  v->yw = L->yw.p;
  v->n_items = L->n_items.p;
  v->rows = L->last_rows;
  v->capacity = L->last_cap;
  v->tile_n = L->tile_n;
  v->ffn_kernel = L->last_ffn_kernel;
  return MOE_OK;
}

int moe_layer_set_weight_pool(moe_layer* L, const void* W1_pool, const void* W2_pool, int n_slots,
                              const int32_t* slot_of) {
  if (!L) return fail(MOE_ERR_INVALID_ARGUMENT, "null layer");
  const moe_layer_desc& d = L->d;
  int st;
  if (!W1_pool || !W2_pool) {
    // back to the layer's own weights (row-major map only where they are row-major)
    if (!L->no_weights && !L->caller_packed &&
        ((st = encode_bf16(&L->tmW1, L->W1, (uint64_t)d.num_experts * d.hidden_dim, d.token_dim, 128)) ||
         (st = encode_bf16(&L->tmW2, L->W2, (uint64_t)d.num_experts * d.token_dim, d.hidden_dim, 128))))
      return st;
    L->slot_of = nullptr;
  } else {
    if (n_slots < 1 || !slot_of) return fail(MOE_ERR_INVALID_ARGUMENT, "bad weight pool");
    if ((st = encode_bf16(&L->tmW1, W1_pool, (uint64_t)n_slots * d.hidden_dim, d.token_dim, 128)) ||
        (st = encode_bf16(&L->tmW2, W2_pool, (uint64_t)n_slots * d.token_dim, d.hidden_dim, 128)))
      return st;
    L->slot_of = slot_of;
  }
  L->drop_graphs();
  return MOE_OK;
}

}  // extern "C"
