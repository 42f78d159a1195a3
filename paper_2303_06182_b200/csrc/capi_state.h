// Internal state of the C ABI: context / layer / FFN objects, device-buffer
// helper, error reporting and TMA descriptor encoding.  Shared by capi.cu
// (routing, layer, FFN entry points) and cache.cu (expert cache).
#pragma once

#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/moe_capi.h"
#include "moe_internal.h"

namespace moe {
int gate_box_rows(int E);
// inner (K) extent of the gate's X / Wg TMA boxes (64 for E <= 128, else 32)
int gate_box_cols(int E);

namespace capi {

inline thread_local std::string g_last_error;

inline int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

inline int cuda_fail(cudaError_t e, const char* what) {
  return fail(MOE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define MOE_CUDA(call)                                         \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);        \
  } while (0)

inline PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

inline int get_encoder() {
  if (g_encode) return MOE_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
    return fail(MOE_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return MOE_OK;
}

// Row-major bf16 matrix [rows, cols] viewed by TMA in boxes of 64 x box_rows
// with the 128-byte swizzle the UMMA descriptors expect.
inline int encode_bf16(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows,
                       uint32_t box_cols = 64) {
  int st = get_encoder();
  if (st) return st;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  // rows of box_cols bf16: 128 B -> 128-byte swizzle, 64 B -> 64-byte swizzle
  const CUtensorMapSwizzle sw = box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu box=%u",
             (int)r, (unsigned long long)rows, (unsigned long long)cols, box_rows);
    return fail(MOE_ERR_CUDA, buf);
  }
  return MOE_OK;
}

// Packed weight tiles (launch_pack_tiles): 128 x 64 bf16 tiles stored already
// in the 128-byte-swizzled shared-memory order, so the tensor map copies them
// verbatim (no swizzle) and a 1-D bulk copy of consecutive tiles lands the same
// bytes.  The box is two tiles (256 rows): the CTA-pair FFN loads a stage's
// weights (KCH = 2 consecutive tiles) as one request.  n = elements.
inline int encode_packed(CUtensorMap* m, const void* ptr, uint64_t n) {
  int st = get_encoder();
  if (st) return st;
  cuuint64_t dims[2] = {64, n / 64};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, 256};  // two consecutive tiles: one CTA-pair stage (KCH = 2)
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MOE_ERR_CUDA, "cuTensorMapEncodeTiled failed (packed weight tiles)");
  return MOE_OK;
}

// [rows, cols] bf16 as a 3-D tensor (64 cols, rows, cols / 64 chunks): a box of
// {64, box_rows, 2} lands as two chunk slabs of box_rows x 128 B, 128-byte swizzled.
inline int encode_rows_k2(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  int st = get_encoder();
  if (st) return st;
  cuuint64_t dims[3] = {64, rows, cols / 64};
  cuuint64_t strides[2] = {cols * 2, 128};
  cuuint32_t box[3] = {64, box_rows, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MOE_ERR_CUDA, "cuTensorMapEncodeTiled failed (3-D row boxes)");
  return MOE_OK;
}

inline int encode_rows(moe::RowMaps* m, const void* ptr, uint64_t rows, uint64_t cols) {
  int st;
  if ((st = encode_bf16(&m->m8, ptr, rows, cols, 8)) ||
      (st = encode_bf16(&m->m16, ptr, rows, cols, 16)) ||
      (st = encode_bf16(&m->m32, ptr, rows, cols, 32)) ||
      (st = encode_bf16(&m->m64, ptr, rows, cols, 64)) ||
      (st = encode_bf16(&m->m256, ptr, rows, cols, 256)))
    return st;
  static const bool k2 = [] {
    const char* v = getenv("MOE_FFN_ROWS_K2");
    return !v || atoi(v) != 0;
  }();
  m->has_k2 = k2 && cols % 128 == 0;
  for (int i = 0; m->has_k2 && i < moe::RowMaps::kK2Maps; ++i)
    if ((st = encode_rows_k2(&m->k2[i], ptr, rows, cols, 8 * (i + 1)))) return st;
  return MOE_OK;
}

// Work-item width of the grouped FFN: 256-token items (N = 256 MMAs, each
// expert's weights streamed once per 256 tokens) once experts average more
// than ~160 rows, unless that leaves fewer than ~4 waves of tiles for the
// persistent grid (few experts, e.g. cfg1: 8 experts x 256 tokens ran 5 %
// faster as 128-token items).  rows_per_expert = expected rows / expert.
inline int auto_tile_n(double rows_per_expert, int experts, int TD, int HD, int sms) {
  if (rows_per_expert <= 160.0) return 128;
  const double items = experts * std::ceil(rows_per_expert / 256.0);
  const double tiles = items * (HD / 128 + TD / 128);
  return tiles >= 4.0 * sms ? 256 : 128;
}

// CTA pairs (M = 256 UMMA) for the fused FFN when there are enough tiles to
// keep every pair busy: >= 8 waves of pair-tiles over sms / 2 pairs.  With
// the dynamic tail, same-box A/B: LM FFN 1.343 -> 1.306 ms, MT 1.427 ->
// 1.385 ms; cfg1 (8 experts, ~2 waves) 0.084 -> 0.093 ms, hence the bound.
inline int auto_pair(double rows_per_expert, int experts, int TD, int HD, int tile_n, int sms) {
  if (TD % 256 || HD % 256) return 0;
  const double items = experts * std::ceil(std::max(rows_per_expert, 1.0) / tile_n);
  const double pair_tiles = items * (HD / 256 + TD / 256);
  return pair_tiles >= 8.0 * (sms / 2) ? 1 : 0;
}

// Reference check_batch (gating.cpp:12-18), verbatim messages.
inline int check_batch(int S, int k, int E) {
  if (E < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "num_experts must be positive");
  if (k < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "top_k must be positive");
  if (k > E) return fail(MOE_ERR_INVALID_ARGUMENT, "top_k exceeds num_experts");
  if (S < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "empty batch");
  return MOE_OK;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  int reserve(size_t count) {
    if (count <= n) return MOE_OK;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T) + 16);
    if (e != cudaSuccess) {
      p = nullptr;
      return fail(MOE_ERR_OUT_OF_MEMORY, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    n = count;
    return MOE_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};


}  // namespace capi
}  // namespace moe

using namespace moe;
using namespace moe::capi;

struct moe_ctx {
  int device = 0;
  int sms = 0;
  size_t l2_bytes = 0;
  int route_max_blocks = 0;
  int route_prepared_E = -1;
  DevBuf<int32_t> block_hist, err_flag, drop_mark;
  DevBuf<int32_t> static_splits;  // moe_route_static's splits scratch (per device)
  cudaStream_t scratch_stream = nullptr;

  int prepare_route(int E) {
    if (E > route_prepared_E) {
      int mb = 0;
      cudaError_t e = route_prepare(E, &mb);
      if (e != cudaSuccess) return cuda_fail(e, "route_prepare");
      route_max_blocks = mb;
      route_prepared_E = E;
    }
    int st = block_hist.reserve((size_t)E * (route_max_blocks + 4) + route_max_blocks);
    if (st) return st;
    if (!err_flag.p) {
      st = err_flag.reserve(1);
      if (st) return st;
      cudaError_t e = cudaMemset(err_flag.p, 0, sizeof(int32_t));
      if (e != cudaSuccess) return cuda_fail(e, "clear error flag");
    }
    return MOE_OK;
  }
};

struct moe_layer {
  moe_ctx* ctx = nullptr;
  moe_layer_desc d{};
  const void* Wg = nullptr;
  const void* W1 = nullptr;
  const void* W2 = nullptr;
  int tile_n = 128;
  int rows_max = 0;
  int items_max = 0;
  CUtensorMap tmWg, tmW1, tmW2, tmXp, tmH;
  moe::RowMaps xpm, hm;  // Xp / H at 8/16/32/64-row boxes (fused FFN)
  // prepacked weights: 128 x 64 tiles, 16 KB contiguous (launch_pack_tiles)
  bool packed = false;
  bool caller_packed = false;  // tmW1p/tmW2p address the caller's pre-packed W1/W2 (no copy)
  bool no_weights = false;     // pool-only layer: expert weights come from an attached cache
  DevBuf<__nv_bfloat16> w1p, w2p;
  CUtensorMap tmW1p, tmW2p;
  CUtensorMap tmX;  // X for the gate (box 64 x 128)
  const void* tmX_ptr = nullptr;
  int tmX_rows = 0;
  DevBuf<int32_t> done;      // fused-FFN per-item counters [2 * items_max]
  void* fwd_out = nullptr;   // output of the forward in flight (fused combine target)
  // optional expert-cache weight pool
  const int32_t* slot_of = nullptr;
  DevBuf<int32_t> idx, pos, counts, splits, order, dropped, n_dropped, n_items, err, item_off;
  DevBuf<float> w, wpos, logits;
  DevBuf<FfnItem> items;
  DevBuf<__nv_bfloat16> xp, h, yw, xin, yout;
  int last_rows = 0;
  int last_cap = 0;
  bool counters_zeroed = false;  // the route kernel of this forward zeroed `done`
  int last_ffn_kernel = 0;       // moe_layer_view::ffn_kernel
  // per-stage timing ring (eager path)
  std::vector<cudaEvent_t> tev;
  int t_slots = 0;
  long t_calls = 0;
  // graph cache: one instantiated graph per (X, out, S, stream), LRU
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    const void* x = nullptr;
    void* out = nullptr;
    int S = -1;
    cudaStream_t stream = nullptr;
    uint64_t used = 0;
  };
  static constexpr int kGraphSlots = 6;
  GraphEntry graphs[kGraphSlots];
  uint64_t graph_clock = 0;
  void drop_graphs() {
    for (GraphEntry& g : graphs) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g = GraphEntry{};
    }
  }
  // pipelined host forward: double-buffered device staging + two copy streams
  static constexpr int kPipeBufs = 3;  // moe_layer_forward_host_batches ring depth
  DevBuf<__nv_bfloat16> pin[kPipeBufs], pout[kPipeBufs];
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_in[kPipeBufs] = {}, ev_comp[kPipeBufs] = {}, ev_out[kPipeBufs] = {};
};

struct moe_ffn {
  moe_ctx* ctx = nullptr;
  moe_ffn_desc d{};
  int tile_n = 128;
  int items_max = 0;
  CUtensorMap tmW1, tmW2, tmXp, tmH;
  moe::RowMaps xpm, hm;
  bool packed = false;
  DevBuf<__nv_bfloat16> w1p, w2p;
  CUtensorMap tmW1p, tmW2p;
  DevBuf<int32_t> counts, splits, order, pos, n_items, done;
  DevBuf<float> wpos, ones;
  DevBuf<FfnItem> items;
  DevBuf<__nv_bfloat16> xp, h;
};


namespace moe {
namespace capi {
int route_common(moe_ctx* ctx, const int32_t* expert_idx, int S, int k, int E, int cap,
                 int32_t* counts, int32_t* splits, int32_t* order, int32_t* pos,
                 const float* gate_w, float* wpos, int32_t* dropped, int32_t* n_dropped,
                 FfnItem* items, int32_t* n_items, int tile_n, const int32_t* key_map,
                 int num_keys_in, cudaStream_t stream, int32_t* item_off = nullptr,
                 int32_t* zero = nullptr, int zero_n = 0);
int layer_front(moe_layer* L, const void* X, int S, const int32_t* idx_in, const float* w_in,
                cudaStream_t s, cudaEvent_t* ev);
int layer_ffn(moe_layer* L, cudaStream_t s, int e_lo, int e_hi, cudaEvent_t* ev);
int layer_back(moe_layer* L, int S, void* out, cudaStream_t s, cudaEvent_t* ev);
// dynamic top-1 gating with fuse_combine: GEMM2 stores each token's output row
// itself (one contribution per token, weight applied), no combine kernel
inline bool layer_fused_combine(const moe_layer* L) {
  return L->d.mode == MOE_GATING_DYNAMIC && L->d.fuse_combine && L->d.top_k == 1;
}
}  // namespace capi
}  // namespace moe
