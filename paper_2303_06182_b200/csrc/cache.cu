// Expert buffering: a GPU-resident cache of expert weights
// backed by pinned host memory, filled with cudaMemcpyAsync on a side stream.
//
// Decisions follow the reference's access_batch exactly
// (proj/src/buffer.cpp:57-130, LIFO / FIFO): the batch's active experts are
// visited serially in increasing id order; a miss inserts the expert, and when
// the cache is full it first evicts the most recently inserted resident that
// is inactive in this batch, otherwise the newest (LIFO) / oldest (FIFO).
//
// On the GPU the experts of a batch run concurrently, so the serial semantics
// need one extra rule: a resident whose FFN is scheduled in the current wave
// must not be overwritten before that wave finishes.  The batch is therefore
// split into waves (contiguous expert-id ranges, hence contiguous rows and
// FFN items): a wave closes right before a miss would evict one of its own
// experts.  Copies run on a side stream with per-slot readiness: a copy
// waits only for the FFN of the wave that last read its slot (none for free
// slots and inactive victims, which are all issued up front); each wave's
// FFN waits for its own copies.
// The routing counts reach the host once per layer call (the host sync the
// cache needs to know the active set, shared with the EP count exchange in
// the paper's design).
#include <algorithm>
#include <cstdint>

#include "capi_state.h"

struct moe_cache {
  moe_layer* L = nullptr;
  int n_slots = 0;
  int policy = 0;  // 0 LIFO, 1 FIFO (buffer.hpp:16 CachePolicy order)
  const uint8_t* w1h = nullptr;
  const uint8_t* w2h = nullptr;
  size_t w1_bytes = 0, w2_bytes = 0;
  DevBuf<__nv_bfloat16> pool1, pool2;
  DevBuf<int32_t> slot_dev;
  std::vector<int32_t*> slot_host;  // pinned staging, one table per wave
  int32_t* counts_host = nullptr;   // pinned [E]
  std::vector<int> order;           // residents, oldest first (CacheState::insertion_order)
  std::vector<int> slot_of;         // expert -> slot or -1
  std::vector<int> free_slots;
  int64_t accesses = 0, hits = 0, misses = 0, evictions = 0, copies_bytes = 0;
  int last_stats[5] = {0, 0, 0, 0, 0};  // accesses, hits, misses, evictions, waves
  std::vector<int> last_active;
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> ev_copy, ev_ffn;
};

namespace {

struct Wave {
  int e_lo, e_hi;                              // expert id range [e_lo, e_hi]
  std::vector<std::pair<int, int>> loads;      // (expert, slot) to copy before the wave
  std::vector<std::pair<int, int>> table;      // (expert, slot) of every wave expert
};

int ensure_events(moe_cache* C, size_t n) {
  while (C->ev_copy.size() < n) {
    cudaEvent_t a, b;
    MOE_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    MOE_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    C->ev_copy.push_back(a);
    C->ev_ffn.push_back(b);
  }
  const int E = C->L->d.num_experts;
  while (C->slot_host.size() < n) {
    int32_t* p = nullptr;
    MOE_CUDA(cudaMallocHost(&p, sizeof(int32_t) * E));
    C->slot_host.push_back(p);
  }
  return MOE_OK;
}

// One cache decision, in access order: victim -2 = hit, -1 = miss into a free
// slot, >= 0 = miss that evicts `victim`.
struct CacheStep {
  int expert;
  int victim;
};

// The expert-buffering controller, access_batch semantics
// (proj/src/buffer.cpp:57-130, include/moesim/buffer.hpp:45-55): the sorted,
// distinct active experts are accessed serially; a miss inserts at the back
// of `order` (residents oldest first) and, when the cache is full, evicts
//   LIFO / FIFO: the most recently inserted resident inactive in this batch,
//                else the newest (LIFO) / oldest (FIFO) resident;
//   MIN:         the resident whose next use -- later in this batch, then in
//                `future` -- is farthest; never-used-again first, ties to
//                the lowest id.
// Shared by the GPU cache (plan_batch below) and the moesim::access_batch
// drop-in (through moe_cache_policy_access), so both make the same decisions.
void cache_policy_run(std::vector<int>& order, int cache_size, int policy,
                      const std::vector<int>& active, const int32_t* future, int64_t n_future,
                      std::vector<CacheStep>& steps) {
  steps.clear();
  const int top = active.empty() ? 0 : active.back();
  int hi = top;
  for (int r : order) hi = std::max(hi, r);
  std::vector<char> live((size_t)hi + 1, 0), here((size_t)hi + 1, 0);
  for (int x : active) live[x] = 1;
  for (int r : order) here[r] = 1;
  // MIN: index of each expert's next access.  Within the batch the access
  // sequence is `active` itself; the future stream follows it.
  std::vector<int64_t> next_future;
  if (policy == 2) {
    next_future.assign((size_t)hi + 1, INT64_MAX);
    for (int64_t i = n_future - 1; i >= 0; --i) {
      const int e = future[i];
      if (e >= 0 && e <= hi) next_future[e] = i;
    }
  }
  for (size_t ai = 0; ai < active.size(); ++ai) {
    const int x = active[ai];
    if (here[x]) {
      steps.push_back({x, -2});
      continue;
    }
    int victim = -1;
    if ((int)order.size() >= cache_size) {
      if (policy == 2) {
        int64_t far = -1;
        for (int r : order) {
          int64_t when;
          const auto it = std::lower_bound(active.begin() + ai + 1, active.end(), r);
          if (it != active.end() && *it == r)
            when = it - active.begin();
          else if (next_future[r] != INT64_MAX)
            when = (int64_t)active.size() + next_future[r];
          else
            when = INT64_MAX;
          if (when > far || (when == far && r < victim)) {
            far = when;
            victim = r;
          }
        }
      } else {
        for (auto it = order.rbegin(); it != order.rend() && victim < 0; ++it)
          if (!live[*it]) victim = *it;
        if (victim < 0) victim = policy == 0 ? order.back() : order.front();
      }
      order.erase(std::find(order.begin(), order.end(), victim));
      here[victim] = 0;
    }
    order.push_back(x);
    here[x] = 1;
    steps.push_back({x, victim});
  }
}

// The GPU schedule of one batch from the controller's decisions: slots for
// the misses and the waves (a wave closes right before a miss would evict an
// expert the wave itself still has to run).
std::vector<Wave> plan_batch(moe_cache* C, const std::vector<int>& active, int* stats) {
  std::vector<CacheStep> steps;
  cache_policy_run(C->order, C->n_slots, C->policy, active, nullptr, 0, steps);
  std::vector<Wave> waves;
  Wave cur;
  cur.e_lo = -1;
  std::vector<char> in_wave(C->slot_of.size(), 0);
  auto close_wave = [&]() {
    if (cur.e_lo >= 0) {
      for (auto& es : cur.table) in_wave[es.first] = 0;
      waves.push_back(std::move(cur));
    }
    cur = Wave();
    cur.e_lo = -1;
  };
  for (const CacheStep& st : steps) {
    const int x = st.expert;
    ++stats[0];
    if (st.victim == -2) {
      ++stats[1];
    } else {
      ++stats[2];
      int slot;
      if (st.victim >= 0) {
        if (in_wave[st.victim]) close_wave();  // its weights are still needed by this wave
        slot = C->slot_of[st.victim];
        C->slot_of[st.victim] = -1;
        ++stats[3];
      } else {
        slot = C->free_slots.back();
        C->free_slots.pop_back();
      }
      C->slot_of[x] = slot;
      if (cur.e_lo < 0) cur.e_lo = x;
      cur.loads.emplace_back(x, slot);
    }
    if (cur.e_lo < 0) cur.e_lo = x;
    cur.e_hi = x;
    cur.table.emplace_back(x, C->slot_of[x]);
    in_wave[x] = 1;
  }
  close_wave();
  return waves;
}

int cache_forward(moe_cache* C, const void* X, int S, const int32_t* idx, const float* w, void* out,
                  cudaStream_t s) {
  moe_layer* L = C->L;
  const int E = L->d.num_experts;
  L->fwd_out = out;
  int st = layer_front(L, X, S, idx, w, s, nullptr);
  if (st) return st;
  // the one host sync: which experts are active in this batch
  MOE_CUDA(cudaMemcpyAsync(C->counts_host, L->counts.p, sizeof(int32_t) * E,
                           cudaMemcpyDeviceToHost, s));
  MOE_CUDA(cudaStreamSynchronize(s));
  std::vector<int> active;
  for (int e = 0; e < E; ++e)
    if (C->counts_host[e] > 0) active.push_back(e);
  int stats[4] = {0, 0, 0, 0};
  const std::vector<Wave> waves = plan_batch(C, active, stats);
  if ((st = ensure_events(C, waves.size()))) return st;
  // Per-slot readiness: a copy into slot q must wait only for the FFN of the
  // last wave of THIS batch that read q (earlier batches' FFNs finished
  // before the host sync above).  Copies whose slot no wave of this batch has
  // used yet (free slots, victims inactive in this batch) wait for nothing:
  // they are all issued first, so they stream over PCIe while earlier waves
  // compute; the dependent ones follow wave by wave.
  std::vector<int> slot_wave((size_t)C->n_slots, -1), dep_of_load, wave_dep(waves.size(), -1);
  std::vector<char> wave_has_dep(waves.size(), 0);
  for (size_t wv = 0; wv < waves.size(); ++wv) {
    for (auto& es : waves[wv].loads) {
      const int dep = slot_wave[(size_t)es.second];
      dep_of_load.push_back(dep);
      if (dep >= 0) {
        wave_has_dep[wv] = 1;
        wave_dep[wv] = std::max(wave_dep[wv], dep);
      }
    }
    for (auto& es : waves[wv].table) slot_wave[(size_t)es.second] = (int)wv;
  }
  auto copy_in = [&](const std::pair<int, int>& es) -> int {
    const size_t e = (size_t)es.first, slot = (size_t)es.second;
    MOE_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(C->pool1.p) + slot * C->w1_bytes,
                             C->w1h + e * C->w1_bytes, C->w1_bytes, cudaMemcpyHostToDevice,
                             C->copy_stream));
    MOE_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(C->pool2.p) + slot * C->w2_bytes,
                             C->w2h + e * C->w2_bytes, C->w2_bytes, cudaMemcpyHostToDevice,
                             C->copy_stream));
    C->copies_bytes += (int64_t)(C->w1_bytes + C->w2_bytes);
    return MOE_OK;
  };
  // pass 1: every independent copy, in wave order
  size_t li = 0;
  for (size_t wv = 0; wv < waves.size(); ++wv) {
    for (auto& es : waves[wv].loads)
      if (dep_of_load[li++] < 0 && (st = copy_in(es))) return st;
    if (!wave_has_dep[wv]) MOE_CUDA(cudaEventRecord(C->ev_copy[wv], C->copy_stream));
  }
  // pass 2: per wave, its dependent copies (after the FFN that last read their
  // slots), then its FFN
  li = 0;
  for (size_t wv = 0; wv < waves.size(); ++wv) {
    const Wave& W = waves[wv];
    const size_t l0 = li;
    li += W.loads.size();
    if (wave_has_dep[wv]) {
      MOE_CUDA(cudaStreamWaitEvent(C->copy_stream, C->ev_ffn[(size_t)wave_dep[wv]], 0));
      for (size_t j = 0; j < W.loads.size(); ++j)
        if (dep_of_load[l0 + j] >= 0 && (st = copy_in(W.loads[j]))) return st;
      MOE_CUDA(cudaEventRecord(C->ev_copy[wv], C->copy_stream));
    }
    // compute: the wave's slot table, then its experts' FFN items
    int32_t* tab = C->slot_host[wv];
    for (auto& es : W.table) tab[es.first] = es.second;
    MOE_CUDA(cudaStreamWaitEvent(s, C->ev_copy[wv], 0));
    MOE_CUDA(cudaMemcpyAsync(C->slot_dev.p + W.e_lo, tab + W.e_lo,
                             sizeof(int32_t) * (W.e_hi - W.e_lo + 1), cudaMemcpyHostToDevice, s));
    if ((st = layer_ffn(L, s, W.e_lo, W.e_hi + 1, nullptr))) return st;
    MOE_CUDA(cudaEventRecord(C->ev_ffn[wv], s));
  }
  C->accesses += stats[0];
  C->hits += stats[1];
  C->misses += stats[2];
  C->evictions += stats[3];
  for (int i = 0; i < 4; ++i) C->last_stats[i] = stats[i];
  C->last_stats[4] = (int)waves.size();
  C->last_active = active;
  return layer_back(L, S, out, s, nullptr);
}

}  // namespace

extern "C" {

int moe_cache_create(moe_layer* L, const void* W1_host, const void* W2_host, int n_slots,
                     int policy, moe_cache** out) {
  if (!L || !W1_host || !W2_host || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (n_slots < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "cache_size must be >= 1");
  if (policy != 0 && policy != 1)
    return fail(MOE_ERR_UNSUPPORTED, "the GPU cache implements LIFO (0) and FIFO (1)");
  if (L->d.mode != MOE_GATING_DYNAMIC)
    return fail(MOE_ERR_UNSUPPORTED, "expert buffering is implemented for dynamic gating");
  MOE_CUDA(cudaSetDevice(L->ctx->device));
  auto* C = new moe_cache();
  C->L = L;
  C->n_slots = std::min(n_slots, L->d.num_experts);
  C->policy = policy;
  C->w1h = static_cast<const uint8_t*>(W1_host);
  C->w2h = static_cast<const uint8_t*>(W2_host);
  const size_t TD = L->d.token_dim, HD = L->d.hidden_dim, E = L->d.num_experts;
  C->w1_bytes = HD * TD * 2;
  C->w2_bytes = TD * HD * 2;
  int st;
  if ((st = C->pool1.reserve((size_t)C->n_slots * HD * TD)) ||
      (st = C->pool2.reserve((size_t)C->n_slots * TD * HD)) || (st = C->slot_dev.reserve(E))) {
    moe_cache_destroy(C);
    return st;
  }
  cudaMemset(C->slot_dev.p, 0, sizeof(int32_t) * E);
  if (cudaMallocHost(&C->counts_host, sizeof(int32_t) * E) != cudaSuccess ||
      cudaStreamCreateWithFlags(&C->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
    moe_cache_destroy(C);
    return fail(MOE_ERR_CUDA, "cache host buffers / stream");
  }
  C->slot_of.assign(E, -1);
  for (int i = C->n_slots - 1; i >= 0; --i) C->free_slots.push_back(i);
  if ((st = moe_layer_set_weight_pool(L, C->pool1.p, C->pool2.p, C->n_slots, C->slot_dev.p))) {
    moe_cache_destroy(C);
    return st;
  }
  *out = C;
  return MOE_OK;
}

int moe_cache_destroy(moe_cache* C) {
  if (!C) return MOE_OK;
  if (C->L) moe_layer_set_weight_pool(C->L, nullptr, nullptr, 0, nullptr);
  if (C->copy_stream) {
    cudaStreamSynchronize(C->copy_stream);
    cudaStreamDestroy(C->copy_stream);
  }
  for (auto e : C->ev_copy) cudaEventDestroy(e);
  for (auto e : C->ev_ffn) cudaEventDestroy(e);
  for (auto p : C->slot_host) cudaFreeHost(p);
  if (C->counts_host) cudaFreeHost(C->counts_host);
  C->pool1.release();
  C->pool2.release();
  C->slot_dev.release();
  delete C;
  return MOE_OK;
}

int moe_cache_forward(moe_cache* C, const void* X, int S, void* out, void* stream) {
  MOE_NVTX("moe.cache_forward");
  if (!C || !X || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  return cache_forward(C, X, S, nullptr, nullptr, out, (cudaStream_t)stream);
}

int moe_cache_forward_routed(moe_cache* C, const void* X, const int32_t* idx, const float* w, int S,
                             void* out, void* stream) {
  MOE_NVTX("moe.cache_forward_routed");
  if (!C || !X || !idx || !w || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  return cache_forward(C, X, S, idx, w, out, (cudaStream_t)stream);
}

int moe_cache_stats(const moe_cache* C, int64_t* totals5, int* last5) {
  if (!C) return fail(MOE_ERR_INVALID_ARGUMENT, "null cache");
  if (totals5) {
    totals5[0] = C->accesses;
    totals5[1] = C->hits;
    totals5[2] = C->misses;
    totals5[3] = C->evictions;
    totals5[4] = C->copies_bytes;
  }
  if (last5)
    for (int i = 0; i < 5; ++i) last5[i] = C->last_stats[i];
  return MOE_OK;
}

int moe_cache_policy_access(int32_t* resident, int* n_resident, int cache_size, int policy,
                            const int32_t* active, int n_active, const int32_t* future,
                            int64_t n_future, int32_t* stats4) {
  if (!resident || !n_resident || (!active && n_active > 0) || !stats4)
    return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (cache_size < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "cache_size must be >= 1");
  if (policy < 0 || policy > 2) return fail(MOE_ERR_INVALID_ARGUMENT, "unknown cache policy");
  if (policy == 2 && n_future < 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "MIN policy requires the future access sequence");
  if (n_future > 0 && !future) return fail(MOE_ERR_INVALID_ARGUMENT, "null future");
  if (*n_resident < 0 || *n_resident > cache_size)
    return fail(MOE_ERR_INVALID_ARGUMENT, "resident set larger than the cache");
  std::vector<int> act(active, active + std::max(n_active, 0));
  for (int e : act)
    if (e < 0) return fail(MOE_ERR_INVALID_ARGUMENT, "negative expert id");
  std::sort(act.begin(), act.end());
  act.erase(std::unique(act.begin(), act.end()), act.end());
  std::vector<int> order(resident, resident + *n_resident);
  std::vector<CacheStep> steps;
  cache_policy_run(order, cache_size, policy, act, future, std::max<int64_t>(n_future, 0), steps);
  stats4[0] = stats4[1] = stats4[2] = stats4[3] = 0;
  for (const CacheStep& st : steps) {
    ++stats4[0];
    if (st.victim == -2)
      ++stats4[1];
    else
      ++stats4[2];
    if (st.victim >= 0) ++stats4[3];
  }
  *n_resident = (int)order.size();
  std::copy(order.begin(), order.end(), resident);
  return MOE_OK;
}

int moe_cache_resident(const moe_cache* C, int32_t* experts, int* n) {
  if (!C || !n) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  *n = (int)C->order.size();
  if (experts)
    for (size_t i = 0; i < C->order.size(); ++i) experts[i] = C->order[i];
  return MOE_OK;
}

}  // extern "C"
