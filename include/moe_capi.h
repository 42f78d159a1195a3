/*
 * moe_capi.h -- the C-ABI boundary of the B200-native MoE-layer inference path.
 *
 * Plain C: opaque handles, plain pointers and sizes, int status codes.  No
 * C++ or torch types cross this boundary.  Every entry point below replaces
 * (or, for the layer arithmetic the reference does not implement, completes)
 * a reference interface, cited as file:line under /root/reference/proj:
 *
 *   moe_dynamic_dispatch_host   dynamic_dispatch    include/moesim/gating.hpp:69,
 *                                                   src/gating.cpp:58-86
 *   moe_static_dispatch_host    static_dispatch     include/moesim/gating.hpp:68,
 *                                                   src/gating.cpp:30-56
 *   moe_expert_capacity         expert_capacity     include/moesim/gating.hpp:31,
 *                                                   src/gating.cpp:22-28
 *   moe_inverse_order_host      combine<T> (its inverse permutation, the part
 *                               that touches every slot) gating.hpp:107-184
 *   moe_route_dynamic/_static   device-resident forms of the two dispatches
 *   moe_gate_topk               (absent in the reference: SPEC.md:224) the gate
 *                               that produces the TokenAssignment of
 *                               include/moesim/trace.hpp:15-18
 *   moe_grouped_ffn             (absent: SPEC.md:8) expert FFN
 *   moe_combine                 weighted combine<T>, gating.hpp:107-184
 *   moe_layer_*                 the whole MoE layer of PAPER.md:178-187 /
 *                               :305-319 (gate -> dispatch -> FFN -> combine)
 *   moe_exchange_counts         plan_dynamic_exchange payload phase,
 *                               include/moesim/exchange.hpp:64-65,
 *                               src/exchange.cpp:95-120
 *   moe_cache_*                 the GPU-resident expert cache driven by
 *                               access_batch, include/moesim/buffer.hpp:53-55
 *
 * Threading: one context per device (like a library handle).  Calls on one
 * context are not thread-safe; different contexts are independent.  Device-
 * pointer entry points are asynchronous and ordered on the caller's stream
 * (a cudaStream_t passed as void*, NULL = legacy default stream); *_host entry
 * points are synchronous.
 *
 * Errors: every call returns MOE_OK (0) or a moe_status; the message of the
 * last failure on the calling thread is available from moe_last_error().  The
 * C++ drop-in layer (include/moesim/gating.hpp) rethrows
 * MOE_ERR_INVALID_ARGUMENT as std::invalid_argument with the reference's
 * exact message text (src/gating.cpp:13-17,33-42,61,90,96,102).
 */
#ifndef MOE_CAPI_H_
#define MOE_CAPI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_CAPI_VERSION 1

typedef enum moe_status {
  MOE_OK = 0,
  MOE_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  MOE_ERR_CUDA = 2,             /* CUDA runtime / driver failure */
  MOE_ERR_UNSUPPORTED = 3,      /* shape outside what the kernels handle */
  MOE_ERR_OUT_OF_MEMORY = 4,
  MOE_ERR_EXPERT_RANGE = 5,     /* an expert id outside [0, E) (UB in the reference) */
  MOE_ERR_PEER_TIMEOUT = 6      /* expert parallelism: a peer rank never signalled */
} moe_status;

typedef enum moe_gating_mode {
  MOE_GATING_STATIC = 0, /* GatingMode::kStatic,  gating.hpp:16 */
  MOE_GATING_DYNAMIC = 1 /* GatingMode::kDynamic, gating.hpp:16 */
} moe_gating_mode;

typedef struct moe_ctx moe_ctx;
typedef struct moe_layer moe_layer;

int moe_version(void);
const char* moe_status_string(int status);
/* Message of the last failing call made by this thread ("" if none). */
const char* moe_last_error(void);

int moe_ctx_create(int device, moe_ctx** out);
int moe_ctx_destroy(moe_ctx* ctx);
/* Number of SMs of the context's device. */
int moe_ctx_sm_count(const moe_ctx* ctx);

/* Device memory, pinned host memory, copies and streams for C/C++ hosts that
 * do not link the CUDA runtime themselves (the C++ layer API,
 * include/moesim/gpu_layer.hpp).  kind: 0 host->device, 1 device->host,
 * 2 device->device.  stream NULL = legacy default stream. */
int moe_device_alloc(moe_ctx* ctx, size_t bytes, void** out);
int moe_device_free(moe_ctx* ctx, void* ptr);
int moe_host_alloc(moe_ctx* ctx, size_t bytes, void** out); /* pinned */
int moe_host_free(moe_ctx* ctx, void* ptr);
int moe_memcpy(moe_ctx* ctx, void* dst, const void* src, size_t bytes, int kind, void* stream);
int moe_stream_create(moe_ctx* ctx, void** out);
int moe_stream_destroy(moe_ctx* ctx, void* stream);
int moe_stream_synchronize(moe_ctx* ctx, void* stream);

/* ---------------------------------------------------------------- routing */

/* gating.cpp:22-28.  Pure host arithmetic; returns the capacity (>= 0). */
int moe_expert_capacity(double capacity_factor, int seq_len);

/* Drop-in, host buffers, synchronous (the GPU does the work).
 *   experts[t*k + j]  expert of assignment slot t*k+j (TokenAssignment::experts)
 *   order[S*k], counts[E], splits[E+1]  exactly DynamicDispatchPlan's fields. */
int moe_dynamic_dispatch_host(moe_ctx* ctx, const int32_t* experts, int S, int k, int E,
                              int32_t* order, int32_t* counts, int32_t* splits);

/* Drop-in static dispatch.  capacity = moe_expert_capacity(C, S); slots is
 * E x capacity EXPERT-MAJOR (slots[e*cap + c] == plan.slots(e, c)), -1 for
 * placeholders; dropped holds (token, expert) pairs in slot order. */
int moe_static_dispatch_host(moe_ctx* ctx, const int32_t* experts, int S, int k, int E,
                             double capacity_factor, int32_t* capacity, int32_t* slots,
                             int64_t slots_len, int32_t* dropped, int32_t* n_dropped);

/* Inverse of a dispatch permutation: pos[order[p]] = p for p < n (entries
 * equal to -1 -- static placeholders -- are skipped).  pos has n_slots
 * entries and is pre-filled with -1.  Host buffers, synchronous. */
int moe_inverse_order_host(moe_ctx* ctx, const int32_t* order, int64_t n, int32_t* pos,
                           int64_t n_slots);

/* Device-resident routing (stream-ordered).  Any out-of-range expert id is
 * reported by the next moe_check_errors(). pos (slot -> row) may be NULL. */
int moe_route_dynamic(moe_ctx* ctx, const int32_t* expert_idx, int S, int k, int E,
                      int32_t* counts, int32_t* splits, int32_t* order, int32_t* pos,
                      void* stream);
int moe_route_static(moe_ctx* ctx, const int32_t* expert_idx, int S, int k, int E, int capacity,
                     int32_t* counts, int32_t* slots, int32_t* pos, int32_t* dropped,
                     int32_t* n_dropped, void* stream);
/* Synchronises `stream`; MOE_ERR_EXPERT_RANGE if a routing call since the
 * last check met an out-of-range expert id (the flag is then cleared). */
int moe_check_errors(moe_ctx* ctx, void* stream);

/* ---------------------------------------------------------------- stages */

/* Gate (bf16 X [S,TD], bf16 Wg [E,TD], both row-major) -> idx [S,k] int32,
 * w [S,k] fp32 (softmax restricted to the chosen k, slot 0 = largest logit,
 * ties -> lower id), optional fp32 logits [S,E].  E <= 512, k <= 8, TD % 64 == 0. */
int moe_gate_topk(moe_ctx* ctx, const void* X, const void* Wg, int S, int TD, int E, int k,
                  int32_t* idx, float* w, float* logits, void* stream);

/* Xp[p] = X[order[p] / k] (zero row where order[p] == -1); bf16, TD % 8 == 0. */
int moe_gather_rows(moe_ctx* ctx, const void* X, const int32_t* order, int rows, int k, int TD,
                    void* Xp, void* stream);

/* out[t] = sum_j Yw[pos[t*k+j]] (pos == -1 skipped), fp32 accumulate in j
 * order, bf16 out. */
int moe_combine(moe_ctx* ctx, const void* Yw, const int32_t* pos, int S, int k, int TD, void* out,
                void* stream);

/* Counter-based synthetic bf16 data, bit-identical to oracle/layer.py::synth:
 * uniform on [-scale, scale). */
int moe_fill_uniform_bf16(moe_ctx* ctx, void* dst, int64_t n, uint64_t seed, uint64_t tensor_id,
                          float scale, void* stream);

/* ---------------------------------------------------------------- layer */

typedef struct moe_layer_desc {
  int max_tokens;         /* S upper bound per forward call */
  int token_dim;          /* TD: multiple of 128 */
  int hidden_dim;         /* HD: multiple of 128 */
  int num_experts;        /* E <= 512 */
  int top_k;              /* k <= 8 */
  int mode;               /* moe_gating_mode */
  double capacity_factor; /* static mode only */
  int tile_n;             /* grouped-FFN item width: 0 = auto, 128 or 256 */
  int keep_logits;        /* 1: keep fp32 gate logits [S,E] for parity checks */
  int fuse_combine;       /* top-1 layers only: 1 = GEMM2 stores each token's
                             output row itself (gate weight applied), no
                             combine kernel; 0 (default): separate combine.
                             (The k >= 2 last-arrival form measured no faster
                             than the combine kernel in round 1 and was
                             removed, profiles/r01_fusion_ab.md.) */
  int split_ffn;          /* 1: GEMM1 and GEMM2 as two launches (H through HBM);
                             0 (default): one fused persistent launch with H
                             kept in L2 */
  int keep_layout;        /* 0 (default): when the fused FFN runs, the layer keeps
                             a copy of W1/W2 repacked into contiguous 128x64
                             tiles (+1x expert-weight memory; weights are
                             snapshotted at create, see moe_layer_repack);
                             1: stream the caller's row-major weights */
  int weights_packed;     /* 1: W1/W2 are already in the tile-packed layout
                             (moe_pack_expert_weights, e.g. packed in place):
                             the FFN streams them directly and the layer keeps
                             NO copy -- expert weights are held once.  Dynamic
                             gating, fused FFN only (split_ffn / keep_layout 0) */
} moe_layer_desc;

/* Weights are caller-owned device buffers (bf16, row-major):
 *   Wg [E, TD], W1 [E, HD, TD] (H = relu(x W1_e^T)), W2 [E, TD, HD].
 * Expert-weight memory:
 *   - default: the layer streams its own tile-packed copy; after create the
 *     caller's W1/W2 are read again only by moe_layer_repack (or by the
 *     split / keep_layout / static forms), so a caller that does not need
 *     those may free them -- or avoid the copy altogether with
 *   - weights_packed = 1: W1/W2 were packed by moe_pack_expert_weights
 *     (in place is fine) and are streamed as they are: one copy in HBM;
 *   - W1 = W2 = NULL: a pool-only layer for expert buffering (dynamic
 *     gating): no expert weights on the device at all until moe_cache_create
 *     attaches its slot pool; a forward without a cache fails. */
int moe_layer_create(moe_ctx* ctx, const moe_layer_desc* desc, const void* Wg, const void* W1,
                     const void* W2, moe_layer** out);
int moe_layer_destroy(moe_layer* layer);

/* Expert weights, row-major [rows, K] bf16 (rows = E * HD for W1 with K = TD,
 * rows = E * TD for W2 with K = HD), -> the tile-packed layout the fused FFN
 * streams (128 x 64 tiles, 16 KB contiguous, each stored in the 128-byte
 * swizzled shared-memory order so consecutive tiles are copied verbatim by
 * one bulk transfer; every expert's tiles stay inside its own row range).  dst == src packs IN PLACE (expert-block-wise through a
 * 64 MB scratch); otherwise the buffers must not overlap.  rows % 128 == 0,
 * K % 64 == 0.  Synchronous on `stream`. */
int moe_pack_expert_weights(moe_ctx* ctx, const void* src, void* dst, int64_t rows, int K,
                            void* stream);

/* Refresh the layer's packed weight copy after the caller changed W1/W2 in
 * place (no-op when the layer streams the caller's weights). */
int moe_layer_repack(moe_layer* layer, void* stream);

/* One forward pass on device buffers: X [S,TD] bf16 -> out [S,TD] bf16.
 * Stream-ordered, no host synchronisation (dynamic and static modes). */
int moe_layer_forward(moe_layer* layer, const void* X, int S, void* out, void* stream);

/* Same, with the forward captured once into a CUDA graph per (X, out, S,
 * stream) and replayed afterwards. */
int moe_layer_forward_graph(moe_layer* layer, const void* X, int S, void* out, void* stream);

/* End-to-end host path: X_host [S,TD] bf16 -> out_host [S,TD] bf16, the H2D
 * and D2H copies included; synchronous.  Host buffers should be pinned. */
int moe_layer_forward_host(moe_layer* layer, const void* X_host, int S, void* out_host,
                           void* stream);

/* End-to-end host path over a stream of n independent batches (a serving
 * queue): batch i's H2D copy, its forward (graph replay on `stream`) and its
 * D2H copy run on three streams with triple-buffered device staging, so batch
 * i+1's upload and batch i-1's read-back overlap batch i's compute.  Every
 * byte of every batch crosses PCIe; synchronous (returns when all out_host[i]
 * are written).  Output of batch i is bitwise equal to
 * moe_layer_forward_host(X_host[i]).  Host buffers should be pinned; `stream`
 * must be non-default. */
int moe_layer_forward_host_batches(moe_layer* layer, const void* const* X_host, const int* S,
                                   void* const* out_host, int n, void* stream);

/* Per-stage CUDA-event timing of moe_layer_forward (eager path only).
 * Stages: 0 gate, 1 route, 2 gather, 3 FFN GEMM1, 4 FFN GEMM2, 5 combine.
 * enable: n_slots > 0 allocates a ring of n_slots event sets; call i records
 * into slot i % n_slots.  stage_times reads slot `slot` (synchronises on its
 * last event) into ms[MOE_NUM_STAGES]. */
#define MOE_NUM_STAGES 6
int moe_layer_enable_timing(moe_layer* layer, int n_slots);
int moe_layer_stage_times(moe_layer* layer, int slot, float* ms);

/* Device pointers of the layer's internal buffers (valid until destroy), for
 * parity checks.  Any field may be NULL when not applicable. */
typedef struct moe_layer_view {
  int32_t* idx;        /* [S*k] */
  float* w;            /* [S*k] */
  float* logits;       /* [S*E] when keep_logits */
  int32_t* counts;     /* [E] */
  int32_t* splits;     /* [E+1] */
  int32_t* order;      /* dynamic [S*k]; static [E*cap] */
  int32_t* pos;        /* [S*k] */
  int32_t* dropped;    /* static [2*S*k] */
  int32_t* n_dropped;  /* static [1] */
  void* xp;            /* bf16 [rows, TD] */
  void* h;             /* bf16 [rows, HD] */
  void* yw;            /* bf16 [rows, TD] */
  int32_t* n_items;    /* [1] */
  int rows;            /* rows of xp/h/yw used by the last forward */
  int capacity;        /* static capacity of the last forward */
  int tile_n;
  int ffn_kernel;      /* FFN of the last forward: 0 two launches, 1 fused
                          one-SM, 2 fused CTA pairs (cta_group::2) */
} moe_layer_view;
int moe_layer_get_view(moe_layer* layer, moe_layer_view* view);

/* Expert cache hook: make the FFN read expert e's weights from slot
 * slot_of[e] of caller-owned pools W1_pool [n_slots, HD, TD] and
 * W2_pool [n_slots, TD, HD] (device).  slot_of is a DEVICE int32 [E] table;
 * pass NULL pools to return to the layer's own W1/W2. */
int moe_layer_set_weight_pool(moe_layer* layer, const void* W1_pool, const void* W2_pool,
                              int n_slots, const int32_t* slot_of);

/* ---------------------------------------------------------------- grouped FFN */

/* Expert FFN over pre-dispatched rows (the expert-parallel receive side, and
 * the building block of the layer): Y_rows[i] = row_w[i] * W2_e relu(W1_e x_i)
 * with e = keys[i] in [0, num_experts).  Rows are grouped by expert on the
 * device (stable counting sort), streamed through the tcgen05 grouped GEMM and
 * written back in input order.  W1 [E, HD, TD], W2 [E, TD, HD] bf16, device.
 * At tile_n 128 the FFN keeps a tile-packed copy of W1/W2 made at create
 * (weights snapshotted; MOE_PACK=0 in the environment streams the caller's
 * buffers instead). */
typedef struct moe_ffn moe_ffn;
typedef struct moe_ffn_desc {
  int max_rows;
  int token_dim;
  int hidden_dim;
  int num_experts;
  int tile_n; /* 0 = auto, 128 or 256 */
} moe_ffn_desc;
int moe_ffn_create(moe_ctx* ctx, const moe_ffn_desc* desc, const void* W1, const void* W2,
                   moe_ffn** out);
int moe_ffn_destroy(moe_ffn* ffn);
/* row_w may be NULL (weight 1).  Stream-ordered, no host synchronisation. */
int moe_ffn_forward(moe_ffn* ffn, const void* X_rows, const int32_t* keys, const float* row_w,
                    int rows, void* Y_rows, void* stream);

/* ---------------------------------------------------------------- expert cache */

/* GPU-resident expert cache for a dynamic-gating layer:
 * all experts' weights live in caller-owned pinned host memory (W1_host
 * [E, HD, TD], W2_host [E, TD, HD] bf16); n_slots of them are resident on the
 * GPU.  Per forward the active experts are visited in increasing id order with
 * the reference's access_batch decisions (include/moesim/buffer.hpp:53-55,
 * src/buffer.cpp:57-130; policy 0 = LIFO, 1 = FIFO); misses are copied with
 * cudaMemcpyAsync on a side stream, in waves so that no slot is overwritten
 * while its expert's FFN is pending.  One host sync per forward (the counts). */
typedef struct moe_cache moe_cache;
int moe_cache_create(moe_layer* layer, const void* W1_host, const void* W2_host, int n_slots,
                     int policy, moe_cache** out);
int moe_cache_destroy(moe_cache* cache);
int moe_cache_forward(moe_cache* cache, const void* X, int S, void* out, void* stream);
int moe_cache_forward_routed(moe_cache* cache, const void* X, const int32_t* idx, const float* w,
                             int S, void* out, void* stream);
/* totals5: accesses, hits, misses, evictions, bytes copied (cumulative);
 * last5: accesses, hits, misses, evictions, waves of the last forward. */
int moe_cache_stats(const moe_cache* cache, int64_t* totals5, int* last5);
/* Resident experts, oldest first (CacheState::insertion_order). */
int moe_cache_resident(const moe_cache* cache, int32_t* experts, int* n);

/* The cache's replacement controller on plain arrays -- access_batch of
 * include/moesim/buffer.hpp:45-55 (src/buffer.cpp:57-130), the same code the
 * GPU cache above runs.  resident[0..*n_resident) are the resident experts
 * oldest first (CacheState::insertion_order; capacity cache_size), updated in
 * place.  policy 0 LIFO, 1 FIFO, 2 MIN (MIN needs future: the flattened later
 * accesses, n_future >= 0; n_future < 0 = no future given).  stats4: accesses,
 * hits, misses, evictions of this batch.  Host only, no device work. */
int moe_cache_policy_access(int32_t* resident, int* n_resident, int cache_size, int policy,
                            const int32_t* active, int n_active, const int32_t* future,
                            int64_t n_future, int32_t* stats4);

/* Forward with caller-provided routing (idx [S,k] int32, w [S,k] fp32 on the
 * device) instead of the gate: trace replay and skewed synthetic workloads. */
int moe_layer_forward_routed(moe_layer* layer, const void* X, const int32_t* idx, const float* w,
                             int S, void* out, void* stream);

/* ---------------------------------------------------------------- EP */

/* Dispatch by a relabelled key: key = key_map[expert] in [0, num_keys)
 * (expert parallelism sorts by (device, local expert) so every destination
 * device's slots are contiguous).  Otherwise identical to moe_route_dynamic;
 * gate_w/wpos (optional) carry the gate weight of each slot to its row. */
int moe_route_dynamic_keyed(moe_ctx* ctx, const int32_t* expert_idx, int S, int k,
                            int num_experts, const int32_t* key_map, int num_keys,
                            int32_t* counts, int32_t* splits, int32_t* order, int32_t* pos,
                            const float* gate_w, float* wpos, void* stream);

/* out[r] = (index of the segment holding r) % mod for back-to-back segments of
 * the given lengths (device int32): local-expert ids of received EP rows. */
int moe_fill_segments(moe_ctx* ctx, const int32_t* counts, int n_segments, int mod, int32_t* out,
                      void* stream);

/* ---------------------------------------------------------------- EP over peer memory
 *
 * The expert-parallel layer with the exchange done by the layer's own kernels
 * through NVLink peer memory (CUDA IPC mappings of one "window" per rank)
 * instead of NCCL: one object per rank (one process per GPU).  Per forward:
 *
 *   gate -> route keyed by (device, local expert)            (local)
 *   publish: my per-key slot counts -> every peer's window    (size phase,
 *            exchange.cpp:100-104), then a release flag per peer
 *   dispatch: wait for every rank's counts, compute each row's destination
 *            row at its device (rows land grouped by local expert, then by
 *            source rank, then by slot -- the single-GPU order), gather the
 *            token row and store it straight into the peer's receive buffer
 *            (payload phase, exchange.cpp:106-114) -- gather and all-to-all
 *            fused, no staging copy
 *   recv:    wait for every sender, build the FFN work list from the count
 *            matrix (no host round trip)
 *   FFN:     the fused tcgen05 FFN over the received rows (gate weight applied)
 *   done:    release flag to every peer
 *   combine: wait for every peer's FFN, each token sums its k expert outputs
 *            read straight from the peers' output buffers (return all-to-all
 *            and combine fused), in slot order j
 *
 * No host synchronisation: the whole forward is stream-ordered and can be
 * captured in a CUDA graph (moe_ep_forward_graph).  Every rank must call
 * forward the same number of times (a collective).  Waits time out after
 * ~20 s (MOE_EP_TIMEOUT_MS) and report MOE_ERR_PEER_TIMEOUT through
 * moe_ep_check_errors instead of hanging the device.
 *
 * Setup: moe_ep_create on every rank, exchange the MOE_EP_HANDLE_BYTES
 * handles (any host transport: torch.distributed all_gather_object, MPI, a
 * file), then moe_ep_connect with all handles in rank order. */
#define MOE_EP_MAX_RANKS 8
#define MOE_EP_HANDLE_BYTES 64

typedef struct moe_ep moe_ep;
typedef struct moe_ep_desc {
  int rank;          /* this process's rank, 0 <= rank < world_size */
  int world_size;    /* D <= MOE_EP_MAX_RANKS; E % D == 0 */
  int max_tokens;    /* S upper bound per rank per forward */
  int token_dim;     /* TD: multiple of 128 */
  int hidden_dim;    /* HD: multiple of 128 */
  int num_experts;   /* global E <= 512 */
  int top_k;         /* k <= 8 */
  int max_recv_rows; /* receive capacity; 0 = world_size * max_tokens * top_k (worst case) */
  int transport;     /* MOE_EP_TRANSPORT_P2P (0, default) or MOE_EP_TRANSPORT_NCCL */
} moe_ep_desc;

#define MOE_EP_TRANSPORT_P2P 0  /* NVLink peer memory (CUDA IPC windows), moe_ep_connect */
#define MOE_EP_TRANSPORT_NCCL 1 /* NCCL count all-gather + grouped send/recv, moe_ep_connect_nccl */

/* Wg [E, TD] (all experts, replicated), W1_local [E/D, HD, TD], W2_local
 * [E/D, TD, HD]: this rank's experts in increasing global id (bf16, device;
 * snapshotted into the FFN's tile-packed copy).  device_of: HOST int32 [E],
 * expert -> rank, exactly E/D per rank (the reference's Placement,
 * include/moesim/balance.hpp:12-21). */
int moe_ep_create(moe_ctx* ctx, const moe_ep_desc* desc, const void* Wg, const void* W1_local,
                  const void* W2_local, const int32_t* device_of, moe_ep** out);
int moe_ep_destroy(moe_ep* ep);
/* This rank's window handle (MOE_EP_HANDLE_BYTES bytes). */
int moe_ep_get_handle(moe_ep* ep, void* handle);
/* handles: world_size * MOE_EP_HANDLE_BYTES, in rank order. */
int moe_ep_connect(moe_ep* ep, const void* handles);
/* NCCL transport (desc.transport = MOE_EP_TRANSPORT_NCCL), north_star's
 * "variable-count token all-to-all uses NCCL over NVLink, preceded by a count
 * exchange": per forward an ncclAllGather of the per-key slot counts (the
 * size phase, exchange.cpp:100-104), one host sync, then grouped
 * ncclSend/ncclRecv of exactly the assigned token rows and gate weights (the
 * payload phase, exchange.cpp:106-114), the same fused FFN, and the reverse
 * send/recv before the weighted combine.  Setup: rank 0 calls
 * moe_nccl_get_unique_id, the MOE_NCCL_ID_BYTES bytes reach every rank over
 * any host transport, then every rank calls moe_ep_connect_nccl (collective)
 * instead of moe_ep_connect.  NCCL is loaded at run time (libnccl.so.2);
 * without it these calls return MOE_ERR_UNSUPPORTED.  Forwards have a host
 * sync, so moe_ep_forward_graph runs them eagerly. */
#define MOE_NCCL_ID_BYTES 128
int moe_nccl_get_unique_id(void* id);
int moe_ep_connect_nccl(moe_ep* ep, const void* nccl_id);
/* X [S, TD] bf16 (this rank's tokens) -> out [S, TD] bf16. */
int moe_ep_forward(moe_ep* ep, const void* X, int S, void* out, void* stream);
int moe_ep_forward_graph(moe_ep* ep, const void* X, int S, void* out, void* stream);
/* Synchronises `stream`; MOE_ERR_PEER_TIMEOUT / MOE_ERR_EXPERT_RANGE /
 * MOE_ERR_UNSUPPORTED (receive capacity exceeded) from the device flags. */
int moe_ep_check_errors(moe_ep* ep, void* stream);

/* Per-stage CUDA-event timing of eager moe_ep_forward calls (not graph
 * replays).  Stages: 0 gate + keyed route, 1 count publish, 2 dispatch
 * (includes the wait for every rank's counts), 3 receive / work list,
 * 4 FFN, 5 done flags, 6 combine (includes the wait for every peer's FFN).
 * stage_times synchronises on the last forward's final event. */
#define MOE_EP_NUM_STAGES 7
int moe_ep_enable_timing(moe_ep* ep, int on);
int moe_ep_stage_times(moe_ep* ep, float* ms);

typedef struct moe_ep_view {
  int32_t* idx;        /* [S*k] top-k expert ids (global) */
  float* w;            /* [S*k] */
  int32_t* counts;     /* [E] slots per key (key = device * E/D + local index) */
  int32_t* counts_all; /* [D, E] every rank's counts (this rank's window) */
  int32_t* dest;       /* [S*k] sorted row -> (device << 28) | row at that device */
  int32_t* order;      /* [S*k] sorted row -> slot */
  void* recv_x;        /* bf16 [max_recv_rows, TD] */
  void* recv_y;        /* bf16 [max_recv_rows, TD] */
  float* recv_w;       /* [max_recv_rows] */
  int32_t* n_items;    /* [1] */
  int max_recv_rows;
} moe_ep_view;
int moe_ep_get_view(moe_ep* ep, moe_ep_view* view);

/* exchange.cpp:95-120, payload phase, as slot counts: counts[src*D + dst] =
 * number of assignment slots whose token lives on src and whose expert lives
 * on dst = device_of[e].  residency 0: token t on t % D (round robin,
 * exchange.cpp:35-37, the EP layer's layout); 1: every token on device 0
 * (Residency::kSingleSource).  Host buffers, synchronous (computed on the
 * GPU; used by the moesim::plan_dynamic_exchange drop-in). */
int moe_exchange_counts_host(moe_ctx* ctx, const int32_t* experts, int S, int k, int D,
                             const int32_t* device_of, int E, int residency, int64_t* counts);

#ifdef __cplusplus
}
#endif

#endif /* MOE_CAPI_H_ */
