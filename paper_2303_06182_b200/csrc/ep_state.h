// State of the expert-parallel layer (moe_ep_*), shared by the NVLink
// peer-memory transport (ep_p2p.cu) and the NCCL transport (ep_nccl.cu).
#pragma once

#include "capi_state.h"

namespace moe {

constexpr int kMaxRanks = MOE_EP_MAX_RANKS;
constexpr int kRowBits = 28;

struct EpHdr {
  unsigned long long sig_counts[kMaxRanks];
  unsigned long long sig_data;
  unsigned long long pad0[7];
  unsigned long long sig_ydone[kMaxRanks];
  unsigned long long epoch;  // local step counter (only the owner touches it)
  unsigned long long pad1[7];
};
static_assert(sizeof(EpHdr) <= 512, "header");

struct EpLayout {
  size_t counts_all, arrived, recv_w, recv_x, recv_y, total;
};

struct EpPeers {
  char* base[kMaxRanks];
};

}  // namespace moe

using moe::capi::DevBuf;

struct moe_ep {
  moe_ctx* ctx = nullptr;
  moe_ep_desc d{};
  int El = 0;
  int tile_n = 128;
  int max_recv = 0;
  int items_max = 0;
  moe::EpLayout lay{};
  char* window = nullptr;
  moe::EpPeers peers{};
  bool opened[MOE_EP_MAX_RANKS] = {};
  bool connected = false;
  const void* Wg = nullptr;
  CUtensorMap tmWg, tmX, tmW1p, tmW2p;
  const void* tmX_ptr = nullptr;
  int tmX_rows = 0;
  moe::RowMaps xpm, hm;
  DevBuf<int32_t> key_map, idx, counts, splits, order, pos, dest, n_items, done, err;
  DevBuf<float> w, wpos;
  DevBuf<FfnItem> items;
  DevBuf<__nv_bfloat16> h, w1p, w2p;
  unsigned long long timeout_ns = 20ull * 1000 * 1000 * 1000;
  // CTAs of the dispatch kernel: every rank must use the same count (the
  // receivers wait for D * dispatch_ctas arrivals), hence a constant, one per
  // B200 SM (world 1, ncu: 32 CTAs 106 us, 96 45 us, 148 34 us, 256 48 us,
  // 512 69 us -- every CTA pays the count wait, the scans and a system-scope
  // release); MOE_EP_DISPATCH_CTAS overrides
  int dispatch_ctas = 148;
  int full_fence = 0;
  // MOE_EP_OVERLAP=1: expert-ordered dispatch with per-expert arrival counts,
  // GEMM1 tiles wait only for their expert's rows (the FFN starts while later
  // rows are in flight).  Off by default: at world size 1 the per-row
  // system-scope release costs 41 -> 140 us in the dispatch and the per-tile
  // readiness check +15-19 us in the FFN, and the gain (hiding the
  // all-to-all behind the FFN at D > 1) could not be measured on one GPU.
  int overlap = 0;
  DevBuf<int32_t> expect;
  cudaEvent_t tev[MOE_EP_NUM_STAGES + 1] = {};  // per-stage timing (eager forwards)
  bool timing = false;
  cudaGraphExec_t graph = nullptr;
  const void* g_x = nullptr;
  void* g_out = nullptr;
  int g_S = -1;
  cudaStream_t g_stream = nullptr;
  // NCCL transport (transport == MOE_EP_TRANSPORT_NCCL, ep_nccl.cu)
  void* nccl_comm = nullptr;                 // ncclComm_t
  DevBuf<__nv_bfloat16> send_x, recv_xs;     // [S*k, TD] keyed rows / [R, TD] source-major rows
  DevBuf<float> recv_ws;                     // [R] source-major gate weights
  DevBuf<int32_t> nccl_pos;                  // [S*k] slot -> keyed row (combine)
  int32_t* host_counts = nullptr;            // pinned [D * E]: every rank's per-key counts
  int last_recv_rows = 0;
};


// ep_p2p.cu: the launches both transports share
int ep_launch_recv(moe_ep* P, cudaStream_t s, bool wait_for_arrivals);
int ep_launch_ffn(moe_ep* P, cudaStream_t s);
// ep_nccl.cu
int ep_forward_nccl(moe_ep* P, const void* X, int S, void* out, cudaStream_t s, bool timed);
void ep_nccl_release(moe_ep* P);
