// Internal (non-ABI) declarations shared by the CUDA translation units.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <nvtx3/nvToolsExt.h>

#include <cstdlib>
#include <utility>

namespace moe {

// NVTX range over a C ABI entry point (host enqueue time; nsys / Nsight
// correlate it with the kernels it launches).  nvtx3 is header-only: with no
// tool attached a push / pop is one call through a null-checked pointer.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define MOE_NVTX(name) ::moe::NvtxRange moe_nvtx_scope_(name)

// ---- programmatic dependent launch (PDL)
// Kernels of the layer chain are launched with programmatic stream
// serialization: the next kernel's CTAs are scheduled while the previous one
// drains, run their prologue (barrier init, TMEM alloc, descriptor prefetch)
// and block in griddepcontrol.wait until the previous grid has completed and
// its memory is visible.  MOE_PDL=0 disables it (A/B).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("MOE_PDL");
    return !v || atoi(v) != 0;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_chain(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                cudaStream_t stream, bool cooperative, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (cooperative) {
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n].val.cooperative = 1;
    ++n;
  } else if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

#ifdef __CUDACC__
// wait for the previous kernel of the stream (no-op without PDL)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// allow the next kernel of the stream to be scheduled early
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif

// One unit of grouped-FFN work: `len` (<= tile_n) consecutive rows of the
// expert-grouped activation matrix, all routed to `expert`.
struct FfnItem {
  int expert;
  int row0;
  int len;
  int pad;
};

struct RouteArgs {
  const int32_t* expert_idx;  // [total_slots] expert id per assignment slot
  const int32_t* key_map;     // optional expert -> sort key relabel (EP); null = identity
  int num_keys_in;            // size of key_map's domain
  int num_experts;            // number of sort keys (E, or E after relabel)
  int total_slots;            // k * S
  int top_k;
  int capacity;               // 0 = dynamic gating, else static capacity per expert
  int chunk;                  // filled by launch_route
  int tile_n;                 // FFN item width (rows per item)
  int32_t* counts;            // [E]
  int32_t* splits;            // [E+1]
  int32_t* order;             // dynamic: [kS]; static: [E*cap] slot table (-1 = placeholder)
  int32_t* pos;               // optional [kS] slot -> row (-1 = dropped)
  const float* gate_w;        // optional [kS] gate weight per slot
  float* wpos;                // optional [rows] gate weight per row (0 for placeholders)
  int32_t* dropped;           // static: [2*kS] (token, expert) pairs in slot order
  int32_t* n_dropped;         // static: [1]
  int32_t* drop_mark;         // static scratch [kS]
  int32_t* block_hist;        // scratch [E * max_blocks]
  FfnItem* items;             // optional [<= E*ceil(rows/tile_n)] FFN work list
  int32_t* n_items;           // [1]
  int32_t* item_off;          // optional [E+1]: first item of each expert (expert cache waves)
  int32_t* error_flag;        // [1] set to 1 on an out-of-range expert id
  int32_t* zero;              // optional [zero_n] buffer zeroed by the kernel (FFN counters)
  int zero_n;
  int late_trigger;           // release the next kernel (gather) only at completion
  unsigned long long* prof = nullptr;  // experiments (MOE_ROUTE_PROF): phase stamps of block 0
};

size_t route_smem_bytes(int E);
cudaError_t route_prepare(int E, int* max_blocks);
cudaError_t launch_route(RouteArgs a, int max_blocks, cudaStream_t stream);

// ---- grouped expert FFN (tcgen05)
enum EpilogueMode { kEpiReluBf16 = 0, kEpiScaleBf16 = 1 };

struct GemmArgs {
  const FfnItem* items;
  const int32_t* n_items;
  const int32_t* slot_of;  // optional expert -> weight-slot (expert cache); null = identity
  int m_total;             // rows of one expert's weight matrix (HD for W1, TD for W2)
  int k_total;             // reduction length (TD for W1, HD for W2)
  int mode;                // EpilogueMode
  __nv_bfloat16* out;      // [rows, m_total]
  const float* wpos;       // kEpiScaleBf16: gate weight per row
  const int32_t* out_rows; // optional row remap of the output (row r -> out_rows[r])
  const int32_t* item_off; // optional: run only the items of experts [e_lo, e_hi)
  int e_lo, e_hi;
};

// Fused GEMM1 + GEMM2 (ffn_fused.cu): one persistent launch, H kept in L2.
struct FusedFfnArgs {
  const FfnItem* items;
  const int32_t* n_items;
  const int32_t* item_off;  // optional expert range [e_lo, e_hi) (cache waves)
  int e_lo, e_hi;
  const int32_t* slot_of;   // optional expert -> weight slot
  int TD, HD;
  __nv_bfloat16* H;         // [rows, HD]
  __nv_bfloat16* Yw;        // [rows, TD]
  const int32_t* out_rows;  // optional: GEMM2 row r is written to Yw row out_rows[r]
  const float* wpos;        // gate weight per row
  int32_t* done1;           // [items] GEMM1 tiles stored (zeroed before launch)
  int32_t* done2;           // [items] GEMM2 tiles finished (zeroed before launch)
  int lag;                  // items between an item's GEMM1 and GEMM2 tiles
  int discard_h;            // drop consumed H lines from L2 (no write-back)
  int dbg;                  // experiments only (MOE_FFN_DBG): 1 = skip B loads, 2 = skip stores,
                            // 4 = skip MMAs, 8 = skip the epilogue
  int packed;               // tmW1/tmW2 address prepacked 128 x 64 tiles (launch_pack_tiles)
  int full_fence;           // A/B: per-thread fence.sc before publishing an H tile
  int32_t* tile_ctr;        // zeroed tile counter for the dynamic tail; null = all round robin
  unsigned long long* prof;  // experiments (MOE_FFN_PROF): per-CTA start/end globaltimer
  int late_trigger;         // let the next kernel launch only as CTAs finish
  int pair_hint;            // the caller expects >= ~8 waves of CTA-pair tiles (see auto_pair)
  int dyn_tail;             // tail tiles claimed dynamically (0 = the last lag * MT2)
  int rows256;              // 1-SM kernel, 256-token items: one 256-row token box per k chunk (MOE_FFN_ROWS256)
  // packed tiles' base addresses: the 1-SM kernel loads a stage's consecutive
  // weight tiles as ONE 1-D bulk copy (null: tensor-map loads)
  const void* W1p = nullptr;
  const void* W2p = nullptr;
  // expert parallelism (ep_p2p.cu): a GEMM1 tile's token rows are loaded only
  // once arrived[expert] >= arrived_expect[expert] (peer stores, acquire.sys);
  // after arrive_timeout_ns the wait gives up and sets arrive_err[0]
  const unsigned* arrived;
  const int32_t* arrived_expect;
  int32_t* arrive_err;
  unsigned long long arrive_timeout_ns;
};
// One activation matrix (Xp or H) seen by TMA at four box heights: a B tile
// of n rows (n % 8 == 0) is n/64 boxes of 64 rows plus at most one each of 32,
// 16 and 8 -- a few TMA issues per k-block instead of n/16.
struct RowMaps {
  CUtensorMap m8, m16, m32, m64;
  // one 2-D box of 256 rows x 64 cols: a 256-token item's rows of one k chunk
  // as ONE request (the 1-SM kernel at 256-token items, KCH = 1)
  CUtensorMap m256;
  // 3-D views [k chunk][row][64 cols] with boxes of two consecutive 64-wide k
  // chunks x 8 (i + 1) rows (k2[i], 8..128 rows): a KCH = 2 stage's token rows
  // as ONE request, landing chunk-major with a chunk stride of rows x 128 B
  static constexpr int kK2Maps = 16;
  CUtensorMap k2[kK2Maps];
  int has_k2;
};
cudaError_t fused_ffn_prepare();
// whether launch_fused_ffn will run the CTA-pair kernel for these arguments
bool fused_ffn_uses_pair(const FusedFfnArgs& args, int tile_n);
cudaError_t launch_fused_ffn(const CUtensorMap& tmW1, const RowMaps& xp, const CUtensorMap& tmW2,
                             const RowMaps& h, const FusedFfnArgs& args, int tile_n, int grid,
                             cudaStream_t stream);

cudaError_t gemm_prepare();
// tmA: weights [slots*m_total, k_total]; tmB: activations [rows, k_total]
cudaError_t launch_grouped_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB,
                                const GemmArgs& args, int tile_n, int grid,
                                cudaStream_t stream);

// ---- gate (tcgen05): logits = X Wg^T, softmax-restricted top-k
struct GateArgs {
  int S, TD, E, k;
  int32_t* idx;     // [S*k]
  float* w;         // [S*k]
  float* logits;    // optional [S*E]
  const void* X = nullptr;   // [S, TD] bf16 (the small-E gate reads it directly)
  const void* Wg = nullptr;  // [E, TD] bf16
  unsigned long long* prof = nullptr;  // experiments (MOE_GATE_PROF): per-CTA phase times
  int dbg = 0;  // ablations (MOE_GATE_DBG, wrong results): 1 no MMAs, 2 no loads, 4 no Wg, 8 no X
  int kps = 1;  // k-blocks per pipeline stage (MOE_GATE_KPS, 64-deep k-block path)
  int x_keep = 0;  // X tiles read with evict-last (the gather re-reads X next) instead of evict-first
};
cudaError_t gate_prepare(int E);
cudaError_t launch_gate(const CUtensorMap& tmX, const CUtensorMap& tmWg, const GateArgs& a,
                        cudaStream_t stream);

// ---- bandwidth kernels
cudaError_t launch_gather_rows(const __nv_bfloat16* X, const int32_t* order, int rows, int k,
                               int TD, __nv_bfloat16* Xp, cudaStream_t stream);
cudaError_t launch_combine(const __nv_bfloat16* Yw, const int32_t* pos, int S, int k, int TD,
                           __nv_bfloat16* out, cudaStream_t stream);
// dynamic gating only (every slot has a row, no placeholders): X[t] -> Xp[pos[t*k+j]]
cudaError_t launch_gather_tokens(const __nv_bfloat16* X, const int32_t* pos, int S, int k,
                                 int TD, __nv_bfloat16* Xp, cudaStream_t stream);
bool gather_by_token(int k);  // launch_gather_tokens applies (MOE_GATHER_TOKENS=0 disables)
// row-major [rows, K] bf16 -> 128 x 64 tiles, 16 KB each, contiguous
cudaError_t launch_pack_tiles(const __nv_bfloat16* src, __nv_bfloat16* dst, long rows, int K,
                              cudaStream_t stream);
cudaError_t launch_fill_segments(const int32_t* counts, int n_segments, int mod, int32_t* out,
                                 cudaStream_t stream);
cudaError_t launch_fill_uniform_bf16(__nv_bfloat16* dst, int64_t n, uint64_t seed,
                                     uint64_t tensor_id, float scale, cudaStream_t stream);

}  // namespace moe
