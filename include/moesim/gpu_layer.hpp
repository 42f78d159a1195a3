// C++ host API of the B200 MoE layer: RAII wrappers over the C ABI
// (include/moe_capi.h).  Host code written against this header never touches
// the CUDA runtime -- device memory, pinned host memory, streams and every
// kernel go through libmoe_b200.so.
//
//   moesim::gpu::Context ctx(0);
//   moesim::gpu::DeviceBuffer w1(ctx, bytes), ...;
//   moesim::gpu::MoeLayer layer(ctx, {1024, 4096, 512, 2}, 16384,
//                               moesim::GatingConfig{512, 2, 0.0, moesim::GatingMode::kDynamic},
//                               wg.get(), w1.get(), w2.get());
//   layer.forward(x.get(), 16384, out.get(), stream.get());
//
// Errors: MOE_ERR_INVALID_ARGUMENT -> std::invalid_argument carrying the
// reference's message text, anything else -> moesim::gpu::Error.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "moe_capi.h"
#include "moesim/gating.hpp"

namespace moesim {
namespace gpu {

class Error : public std::runtime_error {
 public:
  Error(int status, const std::string& msg) : std::runtime_error(msg), status_(status) {}
  int status() const { return status_; }

 private:
  int status_;
};

inline void check(int status) {
  if (status == MOE_OK) return;
  const std::string msg = moe_last_error();
  if (status == MOE_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw Error(status, msg);
}

class Context {
 public:
  explicit Context(int device = 0) { check(moe_ctx_create(device, &h_)); }
  ~Context() { moe_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  moe_ctx* get() const { return h_; }
  int sm_count() const { return moe_ctx_sm_count(h_); }

 private:
  moe_ctx* h_ = nullptr;
};

// Owning device (or pinned host) allocation.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(Context& ctx, std::size_t bytes, bool pinned_host = false)
      : ctx_(&ctx), bytes_(bytes), host_(pinned_host) {
    check(host_ ? moe_host_alloc(ctx.get(), bytes, &p_) : moe_device_alloc(ctx.get(), bytes, &p_));
  }
  ~DeviceBuffer() { reset(); }
  DeviceBuffer(DeviceBuffer&& o) noexcept { *this = std::move(o); }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    reset();
    std::swap(ctx_, o.ctx_);
    std::swap(p_, o.p_);
    std::swap(bytes_, o.bytes_);
    std::swap(host_, o.host_);
    return *this;
  }
  void* get() const { return p_; }
  std::size_t bytes() const { return bytes_; }
  void reset() {
    if (p_ && ctx_) host_ ? moe_host_free(ctx_->get(), p_) : moe_device_free(ctx_->get(), p_);
    p_ = nullptr;
  }

 private:
  Context* ctx_ = nullptr;
  void* p_ = nullptr;
  std::size_t bytes_ = 0;
  bool host_ = false;
};

class Stream {
 public:
  explicit Stream(Context& ctx) : ctx_(&ctx) { check(moe_stream_create(ctx.get(), &s_)); }
  ~Stream() { moe_stream_destroy(ctx_->get(), s_); }
  Stream(const Stream&) = delete;
  Stream& operator=(const Stream&) = delete;
  void* get() const { return s_; }
  void synchronize() { check(moe_stream_synchronize(ctx_->get(), s_)); }

 private:
  Context* ctx_;
  void* s_ = nullptr;
};

enum class CopyKind { kHostToDevice = 0, kDeviceToHost = 1, kDeviceToDevice = 2 };

inline void copy(Context& ctx, void* dst, const void* src, std::size_t bytes, CopyKind kind,
                 void* stream = nullptr) {
  check(moe_memcpy(ctx.get(), dst, src, bytes, static_cast<int>(kind), stream));
}

// Counter-based synthetic bf16 (uniform on [-scale, scale)).
inline void fill_uniform_bf16(Context& ctx, void* dst, std::int64_t n, std::uint64_t seed,
                              std::uint64_t tensor_id, float scale, void* stream = nullptr) {
  check(moe_fill_uniform_bf16(ctx.get(), dst, n, seed, tensor_id, scale, stream));
}

struct LayerShape {
  int token_dim = 0;   // TD
  int hidden_dim = 0;  // HD
  int num_experts = 0; // E
  int top_k = 1;       // k
};

struct StageTimes {
  float gate = 0, route = 0, gather = 0, ffn1 = 0, ffn2 = 0, combine = 0;  // ms
  float total() const { return gate + route + gather + ffn1 + ffn2 + combine; }
};

// One MoE layer: gate -> dispatch (gating.hpp semantics,
// dynamic or static) -> grouped expert FFN -> combine, on caller-owned bf16
// device weights Wg [E,TD], W1 [E,HD,TD], W2 [E,TD,HD].
class MoeLayer {
 public:
  // weights_packed: W1/W2 are already tile-packed (pack_expert_weights, e.g.
  // in place) and are streamed as given -- expert weights held once.
  // W1 = W2 = nullptr: a pool-only layer for expert buffering (ExpertCache).
  MoeLayer(Context& ctx, const LayerShape& shape, int max_tokens, const GatingConfig& gating,
           const void* Wg, const void* W1, const void* W2, bool keep_logits = false,
           bool weights_packed = false)
      : ctx_(&ctx), shape_(shape) {
    if (gating.num_experts != shape.num_experts || gating.top_k != shape.top_k)
      throw std::invalid_argument("gating config does not match the layer shape");
    moe_layer_desc d{};
    d.max_tokens = max_tokens;
    d.token_dim = shape.token_dim;
    d.hidden_dim = shape.hidden_dim;
    d.num_experts = shape.num_experts;
    d.top_k = shape.top_k;
    d.mode = gating.mode == GatingMode::kStatic ? MOE_GATING_STATIC : MOE_GATING_DYNAMIC;
    d.capacity_factor = gating.capacity_factor;
    d.keep_logits = keep_logits ? 1 : 0;
    d.weights_packed = weights_packed ? 1 : 0;
    check(moe_layer_create(ctx.get(), &d, Wg, W1, W2, &h_));
  }
  ~MoeLayer() { moe_layer_destroy(h_); }
  MoeLayer(const MoeLayer&) = delete;
  MoeLayer& operator=(const MoeLayer&) = delete;
  moe_layer* get() const { return h_; }
  const LayerShape& shape() const { return shape_; }

  // device buffers, stream-ordered, no host synchronisation
  void forward(const void* X, int S, void* out, void* stream = nullptr) {
    check(moe_layer_forward(h_, X, S, out, stream));
  }
  void forward_graph(const void* X, int S, void* out, void* stream) {
    check(moe_layer_forward_graph(h_, X, S, out, stream));
  }
  // caller-provided routing (device idx [S,k] int32, w [S,k] fp32)
  void forward_routed(const void* X, const std::int32_t* idx, const float* w, int S, void* out,
                      void* stream = nullptr) {
    check(moe_layer_forward_routed(h_, X, idx, w, S, out, stream));
  }
  // host buffers, copies included, synchronous
  void forward_host(const void* X_host, int S, void* out_host, void* stream = nullptr) {
    check(moe_layer_forward_host(h_, X_host, S, out_host, stream));
  }
  // a queue of host batches, copies overlapped with neighbouring batches' compute
  void forward_host_batches(const std::vector<const void*>& X_host, const std::vector<int>& S,
                            const std::vector<void*>& out_host, void* stream) {
    if (X_host.size() != S.size() || S.size() != out_host.size())
      throw std::invalid_argument("one size and one output buffer per batch");
    check(moe_layer_forward_host_batches(h_, X_host.data(), S.data(), out_host.data(),
                                         static_cast<int>(S.size()), stream));
  }
  void check_errors(void* stream = nullptr) { check(moe_check_errors(ctx_->get(), stream)); }

  void enable_timing(int slots) { check(moe_layer_enable_timing(h_, slots)); }
  StageTimes stage_times(int slot) {
    float ms[MOE_NUM_STAGES];
    check(moe_layer_stage_times(h_, slot, ms));
    return StageTimes{ms[0], ms[1], ms[2], ms[3], ms[4], ms[5]};
  }
  moe_layer_view view() {
    moe_layer_view v{};
    check(moe_layer_get_view(h_, &v));
    return v;
  }

 private:
  Context* ctx_;
  LayerShape shape_;
  moe_layer* h_ = nullptr;
};

// Expert weights [rows, K] bf16 -> the tile-packed layout the fused FFN
// streams; dst == src packs in place (moe_pack_expert_weights).
inline void pack_expert_weights(Context& ctx, const void* src, void* dst, std::int64_t rows, int K,
                                void* stream = nullptr) {
  check(moe_pack_expert_weights(ctx.get(), src, dst, rows, K, stream));
}

// GPU-resident LIFO/FIFO expert cache over pinned host weights
// (buffer.hpp access_batch decisions).  While it exists the layer reads its
// experts from the cache's slot pool: run forwards through the cache.
class ExpertCache {
 public:
  ExpertCache(MoeLayer& layer, const void* W1_host, const void* W2_host, int n_slots,
              bool fifo = false) {
    check(moe_cache_create(layer.get(), W1_host, W2_host, n_slots, fifo ? 1 : 0, &h_));
  }
  ~ExpertCache() { moe_cache_destroy(h_); }
  ExpertCache(const ExpertCache&) = delete;
  ExpertCache& operator=(const ExpertCache&) = delete;

  void forward(const void* X, int S, void* out, void* stream = nullptr) {
    check(moe_cache_forward(h_, X, S, out, stream));
  }
  void forward_routed(const void* X, const std::int32_t* idx, const float* w, int S, void* out,
                      void* stream = nullptr) {
    check(moe_cache_forward_routed(h_, X, idx, w, S, out, stream));
  }
  struct Stats {
    std::int64_t accesses = 0, hits = 0, misses = 0, evictions = 0, bytes_copied = 0;
    int last_accesses = 0, last_hits = 0, last_misses = 0, last_evictions = 0, last_waves = 0;
  };
  Stats stats() const {
    std::int64_t t[5];
    int l[5];
    check(moe_cache_stats(h_, t, l));
    return Stats{t[0], t[1], t[2], t[3], t[4], l[0], l[1], l[2], l[3], l[4]};
  }
  std::vector<int> resident() const {
    int n = 0;
    check(moe_cache_resident(h_, nullptr, &n));
    std::vector<std::int32_t> ids(static_cast<std::size_t>(n));
    check(moe_cache_resident(h_, ids.data(), &n));
    return std::vector<int>(ids.begin(), ids.end());
  }

 private:
  moe_cache* h_ = nullptr;
};

// One rank's share of the expert-parallel layer with the exchange over NVLink
// peer memory (moe_ep_*, one process per GPU).  The only host-side collective
// is the exchange of the ranks' window handles at construction, done by the
// caller's transport (`all_gather`: my MOE_EP_HANDLE_BYTES-byte handle in,
// every rank's handle in rank order out -- MPI_Allgather, a file rendezvous,
// torch.distributed, ...).  forward() is then a collective: every rank calls
// it the same number of times; no host synchronisation inside.
class ExpertParallelLayer {
 public:
  using AllGather = std::function<std::vector<std::string>(const std::string& mine)>;

  // NCCL transport (moe_ep_connect_nccl): rank 0's unique id reaches every
  // rank through `broadcast` (called on every rank with rank 0's bytes on
  // rank 0, returns rank 0's bytes everywhere).
  using Broadcast = std::function<std::string(const std::string& root_bytes)>;
  struct Nccl {
    Broadcast broadcast;
  };

  ExpertParallelLayer(Context& ctx, const LayerShape& shape, int rank, int world_size,
                      int max_tokens, const std::vector<std::int32_t>& device_of, const void* Wg,
                      const void* W1_local, const void* W2_local, const Nccl& nccl,
                      int max_recv_rows = 0)
      : ctx_(&ctx), shape_(shape), world_(world_size) {
    create(ctx, shape, rank, world_size, max_tokens, device_of, Wg, W1_local, W2_local, max_recv_rows,
           MOE_EP_TRANSPORT_NCCL);
    std::string id(MOE_NCCL_ID_BYTES, '\0');
    if (rank == 0) check(moe_nccl_get_unique_id(id.data()));
    if (world_size > 1) id = nccl.broadcast(id);
    if (id.size() != MOE_NCCL_ID_BYTES) throw std::invalid_argument("bad NCCL id size");
    check(moe_ep_connect_nccl(h_, id.data()));
  }

  ExpertParallelLayer(Context& ctx, const LayerShape& shape, int rank, int world_size,
                      int max_tokens, const std::vector<std::int32_t>& device_of, const void* Wg,
                      const void* W1_local, const void* W2_local, const AllGather& all_gather,
                      int max_recv_rows = 0)
      : ctx_(&ctx), shape_(shape), world_(world_size) {
    create(ctx, shape, rank, world_size, max_tokens, device_of, Wg, W1_local, W2_local, max_recv_rows,
           MOE_EP_TRANSPORT_P2P);
    std::string mine(MOE_EP_HANDLE_BYTES, '\0');
    check(moe_ep_get_handle(h_, mine.data()));
    std::vector<std::string> all = world_size > 1 ? all_gather(mine) : std::vector<std::string>{mine};
    if (static_cast<int>(all.size()) != world_size)
      throw std::invalid_argument("all_gather must return one handle per rank");
    std::string joined;
    for (const std::string& h : all) {
      if (h.size() != MOE_EP_HANDLE_BYTES) throw std::invalid_argument("bad handle size");
      joined += h;
    }
    check(moe_ep_connect(h_, joined.data()));
  }
  // Callers must make sure no peer still runs a forward (a host barrier)
  // before destroying: the peers map this rank's window.
  ~ExpertParallelLayer() { moe_ep_destroy(h_); }
  ExpertParallelLayer(const ExpertParallelLayer&) = delete;
  ExpertParallelLayer& operator=(const ExpertParallelLayer&) = delete;

  void forward(const void* X, int S, void* out, void* stream = nullptr) {
    check(moe_ep_forward(h_, X, S, out, stream));
  }
  void forward_graph(const void* X, int S, void* out, void* stream) {
    check(moe_ep_forward_graph(h_, X, S, out, stream));
  }
  void check_errors(void* stream = nullptr) { check(moe_ep_check_errors(h_, stream)); }
  moe_ep_view view() {
    moe_ep_view v{};
    check(moe_ep_get_view(h_, &v));
    return v;
  }

 private:
  // the moe_ep object of either transport
  void create(Context& ctx, const LayerShape& shape, int rank, int world_size, int max_tokens,
              const std::vector<std::int32_t>& device_of, const void* Wg, const void* W1_local,
              const void* W2_local, int max_recv_rows, int transport) {
    if (static_cast<int>(device_of.size()) != shape.num_experts)
      throw std::invalid_argument("device_of must have one entry per expert");
    moe_ep_desc d{};
    d.rank = rank;
    d.world_size = world_size;
    d.max_tokens = max_tokens;
    d.token_dim = shape.token_dim;
    d.hidden_dim = shape.hidden_dim;
    d.num_experts = shape.num_experts;
    d.top_k = shape.top_k;
    d.max_recv_rows = max_recv_rows;
    d.transport = transport;
    check(moe_ep_create(ctx.get(), &d, Wg, W1_local, W2_local, device_of.data(), &h_));
  }

  Context* ctx_;
  LayerShape shape_;
  int world_;
  moe_ep* h_ = nullptr;
};

}  // namespace gpu
}  // namespace moesim
