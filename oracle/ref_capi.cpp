// ORACLE TEST INFRASTRUCTURE -- never linked into the product library.
//
// extern "C" shims over the reference's own routing / cache / placement /
// exchange code, compiled VERBATIM from /root/reference/proj/src with
// -Dmoesim=moesim_ref (see oracle/Makefile).  Only tests/, bench.py's
// cpu_baseline leg and __graft_entry__.smoke() load the resulting
// oracle/_ref/libmoesim_ref.so, and only as the checker / CPU baseline.
//
// Because the whole translation unit is compiled with -Dmoesim=moesim_ref,
// every `moesim::` below names the reference implementation.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "moesim/balance.hpp"
#include "moesim/buffer.hpp"
#include "moesim/exchange.hpp"
#include "moesim/gating.hpp"
#include "moesim/trace.hpp"

namespace {

thread_local std::string g_err;

moesim::Batch make_batch(const int* experts, const double* weights, int S, int k) {
  moesim::Batch b;
  b.tokens.resize(static_cast<std::size_t>(S));
  for (int t = 0; t < S; ++t) {
    auto& ta = b.tokens[static_cast<std::size_t>(t)];
    ta.experts.assign(experts + static_cast<std::ptrdiff_t>(t) * k,
                      experts + static_cast<std::ptrdiff_t>(t + 1) * k);
    if (weights)
      ta.weights.assign(weights + static_cast<std::ptrdiff_t>(t) * k,
                        weights + static_cast<std::ptrdiff_t>(t + 1) * k);
    else
      ta.weights.assign(static_cast<std::size_t>(k), 1.0 / k);
  }
  return b;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

moesim::GatingConfig cfg_of(int E, int k, double C, bool is_static) {
  moesim::GatingConfig c;
  c.num_experts = E;
  c.top_k = k;
  c.capacity_factor = C;
  c.mode = is_static ? moesim::GatingMode::kStatic : moesim::GatingMode::kDynamic;
  return c;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_expert_capacity(double c, int s) { return moesim::expert_capacity(c, s); }

double ref_waste_factor(int E, double C, int k) {
  double out = -1.0;
  guarded([&] { out = moesim::waste_factor(E, C, k).value; });
  return out;
}

int64_t ref_dispatch_mask_elements(int S, int E, double C) {
  int64_t out = -1;
  guarded([&] { out = moesim::dispatch_mask_elements(S, E, C); });
  return out;
}

// gating.cpp:58-86 -- dynamic_dispatch.  `mode` lets tests hit the mode check.
int ref_dynamic_dispatch(const int* experts, const double* weights, int S, int k, int E,
                         int mode_static, int* order, int* counts, int* splits) {
  return guarded([&] {
    const moesim::Batch b = make_batch(experts, weights, S, k);
    const auto plan = moesim::dynamic_dispatch(b, cfg_of(E, k, 0.0, mode_static != 0));
    std::memcpy(order, plan.order.data(), plan.order.size() * sizeof(int));
    std::memcpy(counts, plan.counts.data(), plan.counts.size() * sizeof(int));
    std::memcpy(splits, plan.splits.data(), plan.splits.size() * sizeof(int));
  });
}

// gating.cpp:30-56 -- static_dispatch.  `slots` is E x capacity expert-major
// (slots[e*cap + c] == plan.slots(e, c)); dropped holds (t, e) pairs.
int ref_static_dispatch(const int* experts, const double* weights, int S, int k, int E,
                        double C, int mode_static, int* capacity, int* slots, int slots_len,
                        int* dropped, int* n_dropped) {
  return guarded([&] {
    const moesim::Batch b = make_batch(experts, weights, S, k);
    const auto plan = moesim::static_dispatch(b, cfg_of(E, k, C, mode_static != 0));
    *capacity = plan.capacity;
    if (static_cast<int64_t>(E) * plan.capacity > slots_len)
      throw std::runtime_error("slots buffer too small");
    for (int e = 0; e < E; ++e)
      for (int c = 0; c < plan.capacity; ++c)
        slots[static_cast<int64_t>(e) * plan.capacity + c] = plan.slots(e, c);
    *n_dropped = static_cast<int>(plan.dropped.size());
    for (std::size_t i = 0; i < plan.dropped.size(); ++i) {
      dropped[2 * i] = plan.dropped[i].first;
      dropped[2 * i + 1] = plan.dropped[i].second;
    }
  });
}

// gating.hpp:107-141 -- dynamic combine<int>.  Output per token t: n[t]
// entries at out_*[t*k + i], in the reference's presentation order.
int ref_combine_dynamic(const int* experts, const double* weights, int S, int k, int E,
                        const int* payload, int payload_len, int* n, int* out_expert,
                        double* out_weight, int* out_payload) {
  return guarded([&] {
    const moesim::Batch b = make_batch(experts, weights, S, k);
    const auto plan = moesim::dynamic_dispatch(b, cfg_of(E, k, 0.0, false));
    const auto res = moesim::combine(plan, b, std::span<const int>(payload, payload_len));
    for (int t = 0; t < S; ++t) {
      n[t] = static_cast<int>(res[t].size());
      for (std::size_t i = 0; i < res[t].size(); ++i) {
        out_expert[t * k + i] = res[t][i].expert;
        out_weight[t * k + i] = res[t][i].weight;
        out_payload[t * k + i] = res[t][i].payload;
      }
    }
  });
}

// gating.hpp:147-184 -- static combine<int>.
int ref_combine_static(const int* experts, const double* weights, int S, int k, int E, double C,
                       const int* payload, int payload_len, int* n, int* out_expert,
                       double* out_weight, int* out_payload) {
  return guarded([&] {
    const moesim::Batch b = make_batch(experts, weights, S, k);
    const auto plan = moesim::static_dispatch(b, cfg_of(E, k, C, true));
    const auto res = moesim::combine(plan, b, std::span<const int>(payload, payload_len));
    for (int t = 0; t < S; ++t) {
      n[t] = static_cast<int>(res[t].size());
      for (std::size_t i = 0; i < res[t].size(); ++i) {
        out_expert[t * k + i] = res[t][i].expert;
        out_weight[t * k + i] = res[t][i].weight;
        out_payload[t * k + i] = res[t][i].payload;
      }
    }
  });
}

// gating.cpp:101-125
int ref_dispatch_cost_counts(const int* experts, int S, int k, int E, int token_dim,
                             int64_t* out3) {
  return guarded([&] {
    const moesim::Batch b = make_batch(experts, nullptr, S, k);
    const auto plan = moesim::dynamic_dispatch(b, cfg_of(E, k, 0.0, false));
    const auto c = moesim::dispatch_cost_counts(plan, token_dim);
    out3[0] = c.comparisons;
    out3[1] = c.count_passes;
    out3[2] = c.gather_elements;
  });
}

// gating.cpp:127-153 -- writes at most buflen-1 chars.
int ref_debug_json(const int* experts, int S, int k, int E, double C, int is_static, char* buf,
                   int buflen) {
  return guarded([&] {
    const moesim::Batch b = make_batch(experts, nullptr, S, k);
    std::string s = is_static ? moesim::debug_json(moesim::static_dispatch(b, cfg_of(E, k, C, true)))
                              : moesim::debug_json(moesim::dynamic_dispatch(b, cfg_of(E, k, 0.0, false)));
    std::strncpy(buf, s.c_str(), static_cast<std::size_t>(buflen - 1));
    buf[buflen - 1] = 0;
  });
}

// ---- expert cache (buffer.cpp:57-130) ------------------------------------
// A cache state lives in an opaque handle; `active` is one batch's active
// expert ids.  Returns the batch stats and the resident set oldest-first.
void* ref_cache_new() { return new moesim::CacheState(); }
void ref_cache_free(void* s) { delete static_cast<moesim::CacheState*>(s); }

int ref_cache_access(void* state, const int* active, int n_active, int cache_size, int policy,
                     const int* future, int n_future, int* stats4, int* resident,
                     int* n_resident) {
  return guarded([&] {
    auto& st = *static_cast<moesim::CacheState*>(state);
    moesim::CacheConfig cfg;
    cfg.cache_size = cache_size;
    cfg.policy = static_cast<moesim::CachePolicy>(policy);
    cfg.expert_bytes = 1.0;
    std::optional<std::span<const int>> fut;
    if (future) fut = std::span<const int>(future, static_cast<std::size_t>(n_future));
    const auto r = moesim::access_batch(st, std::vector<int>(active, active + n_active), cfg, fut);
    stats4[0] = r.accesses;
    stats4[1] = r.hits;
    stats4[2] = r.misses;
    stats4[3] = r.evictions;
    *n_resident = st.size();
    for (int i = 0; i < st.size(); ++i) resident[i] = st.insertion_order[static_cast<std::size_t>(i)];
  });
}

// ---- placement (balance.cpp:59-115) -------------------------------------
// loads is E x B row-major (loads[e*B + b]).
int ref_greedy_place(const double* loads, int E, int B, int D, int* device_of) {
  return guarded([&] {
    moesim::LoadMatrix lm;
    lm.share = Eigen::MatrixXd::Zero(E, B);
    for (int e = 0; e < E; ++e)
      for (int b = 0; b < B; ++b) lm.share(e, b) = loads[static_cast<int64_t>(e) * B + b];
    const auto p = moesim::greedy_place(lm, D);
    for (int e = 0; e < E; ++e) device_of[e] = p.device_of[static_cast<std::size_t>(e)];
  });
}

int ref_contiguous_place(int E, int D, int* device_of) {
  return guarded([&] {
    const auto p = moesim::contiguous_place(E, D);
    for (int e = 0; e < E; ++e) device_of[e] = p.device_of[static_cast<std::size_t>(e)];
  });
}

int ref_anticorr_place(const double* loads, int E, int B, int D, double weight, int* device_of) {
  return guarded([&] {
    moesim::LoadMatrix lm;
    lm.share = Eigen::MatrixXd::Zero(E, B);
    for (int e = 0; e < E; ++e)
      for (int b = 0; b < B; ++b) lm.share(e, b) = loads[static_cast<int64_t>(e) * B + b];
    const auto p = moesim::anticorr_place(lm, D, weight);
    for (int e = 0; e < E; ++e) device_of[e] = p.device_of[static_cast<std::size_t>(e)];
  });
}

// pearson_corr (balance.cpp:69-90); corr is E x E row-major.
int ref_pearson_corr(const double* loads, int E, int B, double* corr) {
  return guarded([&] {
    moesim::LoadMatrix lm;
    lm.share = Eigen::MatrixXd::Zero(E, B);
    for (int e = 0; e < E; ++e)
      for (int b = 0; b < B; ++b) lm.share(e, b) = loads[static_cast<int64_t>(e) * B + b];
    const auto c = moesim::pearson_corr(lm);
    for (int i = 0; i < E; ++i)
      for (int j = 0; j < E; ++j) corr[static_cast<int64_t>(i) * E + j] = c.corr(i, j);
  });
}

// eval_balance (balance.cpp:153-165); out3 = max_load, avg_max_load, objective.
int ref_eval_balance(const int* device_of, int E, int D, const double* loads, int B, double* out3) {
  return guarded([&] {
    moesim::Placement p;
    p.num_devices = D;
    p.device_of.assign(device_of, device_of + E);
    moesim::LoadMatrix lm;
    lm.share = Eigen::MatrixXd::Zero(E, B);
    for (int e = 0; e < E; ++e)
      for (int b = 0; b < B; ++b) lm.share(e, b) = loads[static_cast<int64_t>(e) * B + b];
    const auto r = moesim::eval_balance(p, lm);
    out3[0] = r.max_load;
    out3[1] = r.avg_max_load;
    out3[2] = r.objective;
  });
}

// ---- exchange (exchange.cpp:95-120) -------------------------------------
// Returns the D x D "size" and "payload" byte matrices, row-major src->dst.
int ref_plan_dynamic_exchange(const int* experts, int S, int k, int E, int D,
                              const int* device_of, int64_t token_bytes, int64_t* size_bytes,
                              int64_t* payload_bytes) {
  return guarded([&] {
    const moesim::Batch b = make_batch(experts, nullptr, S, k);
    const auto plan = moesim::dynamic_dispatch(b, cfg_of(E, k, 0.0, false));
    const auto topo = moesim::make_topology(E, D, token_bytes);
    moesim::Placement pl;
    pl.num_devices = D;
    pl.device_of.assign(device_of, device_of + E);
    const auto cp = moesim::plan_dynamic_exchange(plan, topo, pl);
    for (int i = 0; i < D; ++i)
      for (int j = 0; j < D; ++j) {
        size_bytes[i * D + j] = cp.phases[0].bytes(i, j);
        payload_bytes[i * D + j] = cp.phases[1].bytes(i, j);
      }
  });
}

// ---- synthetic skewed routing (trace.cpp:174-259) -------------------------
// Writes num_batches*seq_len*top_k expert ids (batch-major) and weights.
int ref_gen_synthetic_trace(int E, int k, int B, int S, double skew, double persistence,
                            double active_fraction, uint64_t seed, int* experts,
                            double* weights) {
  return guarded([&] {
    moesim::SyntheticSpec spec;
    spec.num_experts = E;
    spec.top_k = k;
    spec.num_batches = B;
    spec.seq_len = S;
    spec.zipf_skew = skew;
    spec.persistence = persistence;
    spec.active_fraction = active_fraction;
    spec.seed = seed;
    const auto tr = moesim::gen_synthetic_trace(spec);
    int64_t i = 0;
    for (const auto& batch : tr.batches)
      for (const auto& ta : batch.tokens)
        for (int j = 0; j < k; ++j, ++i) {
          experts[i] = ta.experts[static_cast<std::size_t>(j)];
          weights[i] = ta.weights[static_cast<std::size_t>(j)];
        }
  });
}

// ---- trace files (trace.cpp:89-157) and load matrix (:158-172) -----------
int ref_save_synthetic_trace(int E, int k, int B, int S, double skew, double persistence,
                             double active_fraction, uint64_t seed, const char* path) {
  return guarded([&] {
    moesim::SyntheticSpec spec;
    spec.num_experts = E;
    spec.top_k = k;
    spec.num_batches = B;
    spec.seq_len = S;
    spec.zipf_skew = skew;
    spec.persistence = persistence;
    spec.active_fraction = active_fraction;
    spec.seed = seed;
    moesim::save_token_trace(moesim::gen_synthetic_trace(spec), path);
  });
}

int ref_trace_roundtrip(const char* in_path, const char* out_path, int* dims) {
  return guarded([&] {
    const auto tr = moesim::load_token_trace(in_path);
    dims[0] = tr.num_experts;
    dims[1] = tr.top_k;
    dims[2] = tr.num_batches();
    if (out_path && *out_path) moesim::save_token_trace(tr, out_path);
  });
}

int ref_trace_loads(const char* path, double* share, int cap) {
  return guarded([&] {
    const auto L = moesim::aggregate_loads(moesim::load_token_trace(path));
    const long n = static_cast<long>(L.share.rows()) * L.share.cols();
    if (n > cap) throw std::runtime_error("load buffer too small");
    for (long j = 0; j < L.share.cols(); ++j)
      for (long i = 0; i < L.share.rows(); ++i) share[j * L.share.rows() + i] = L.share(i, j);
  });
}

// The reference's routing tier timed on one host thread WITHOUT marshalling:
// the Batch (nested std::vector<TokenAssignment>) is built once, untimed, and
// each call below is the reference's own function on it, best of `reps`:
//   sec[0] dynamic_dispatch          gating.cpp:58-86
//   sec[1] combine<float> (dynamic)   gating.hpp:107-141, payload = k*S floats
//   sec[2] static_dispatch (C)       gating.cpp:30-56   (skipped when C <= 0)
//   sec[3] combine<float> (static)   gating.hpp:147-184 (skipped when C <= 0)
int ref_time_routing(const int* experts, const double* weights, int S, int k, int E, double C,
                     int reps, double* sec) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    const moesim::Batch b = make_batch(experts, weights, S, k);
    const std::vector<float> pay(static_cast<std::size_t>(S) * k, 1.0f);
    for (int i = 0; i < 4; ++i) sec[i] = -1.0;
    auto best = [&](int slot, auto&& fn) {
      for (int r = 0; r < reps; ++r) {
        const auto t0 = clk::now();
        fn();
        const double s = std::chrono::duration<double>(clk::now() - t0).count();
        if (sec[slot] < 0 || s < sec[slot]) sec[slot] = s;
      }
    };
    const auto dcfg = cfg_of(E, k, 0.0, false);
    std::size_t sink = 0;
    best(0, [&] { sink += moesim::dynamic_dispatch(b, dcfg).order.size(); });
    const auto dplan = moesim::dynamic_dispatch(b, dcfg);
    best(1, [&] { sink += moesim::combine(dplan, b, std::span<const float>(pay)).size(); });
    if (C > 0) {
      const auto scfg = cfg_of(E, k, C, true);
      best(2, [&] { sink += moesim::static_dispatch(b, scfg).dropped.size(); });
      const auto splan = moesim::static_dispatch(b, scfg);
      const std::vector<float> spay(static_cast<std::size_t>(E) * splan.capacity, 1.0f);
      best(3, [&] { sink += moesim::combine(splan, b, std::span<const float>(spay)).size(); });
    }
    if (sink == static_cast<std::size_t>(-1)) sec[0] = 0;  // keep the calls observable
  });
}

}  // extern "C"
