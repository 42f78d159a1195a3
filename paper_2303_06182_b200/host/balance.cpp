// Expert placement policies (include/moesim/balance.hpp), host side.
//
// Semantics follow the reference's proj/src/balance.cpp (cited per function);
// the output device_of[E] feeds the GPU expert-parallel layer (moe_ep_create)
// and the C entry points at the bottom (moesim_*_place, moesim_eval_balance)
// make this file the placement source of truth for Python hosts as well
// (paper_2303_06182_b200/ep.py).
#include <algorithm>
#include <cmath>
#include <fstream>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "csv_out.hpp"
#include "moesim/balance.hpp"
#include "moesim/placement_c.h"

namespace moesim {

namespace {

// balance.cpp:14-19
void require_divisible(int num_experts, int num_devices) {
  if (num_devices < 1) throw std::invalid_argument("num_devices must be positive");
  if (num_experts < 1) throw std::invalid_argument("num_experts must be positive");
  if (num_experts % num_devices)
    throw std::invalid_argument("num_experts must be divisible by num_devices");
}

// Per-expert mean share over the history's batches.
std::vector<double> mean_share(const LoadMatrix& h) {
  const Eigen::Index E = h.num_experts(), B = h.num_batches();
  std::vector<double> m(static_cast<std::size_t>(E), 0.0);
  for (Eigen::Index e = 0; e < E; ++e) {
    double s = 0.0;
    for (Eigen::Index b = 0; b < B; ++b) s += h.share(e, b);
    m[static_cast<std::size_t>(e)] = B ? s / static_cast<double>(B) : 0.0;
  }
  return m;
}

// Visiting order of the greedy loops: heaviest mean first, ties to the lower
// id (balance.cpp:22-30).
std::vector<int> heaviest_first(const std::vector<double>& mean) {
  std::vector<int> ids(mean.size());
  std::iota(ids.begin(), ids.end(), 0);
  std::stable_sort(ids.begin(), ids.end(), [&](int a, int b) { return mean[a] > mean[b]; });
  return ids;
}

Placement empty_placement(int E, int D) {
  Placement p;
  p.num_devices = D;
  p.device_of.assign(static_cast<std::size_t>(E), -1);
  return p;
}

}  // namespace

Eigen::MatrixXd Placement::matrix() const {
  Eigen::MatrixXd m = Eigen::MatrixXd::Zero(num_experts(), num_devices);
  for (int e = 0; e < num_experts(); ++e) m(e, device_of[static_cast<std::size_t>(e)]) = 1.0;
  return m;
}

// balance.cpp:40-56
void validate(const Placement& placement) {
  const int E = placement.num_experts(), D = placement.num_devices;
  require_divisible(E, D);
  std::vector<int> held(static_cast<std::size_t>(D), 0);
  for (int e = 0; e < E; ++e) {
    const int d = placement.device_of[static_cast<std::size_t>(e)];
    if (d < 0 || d >= D)
      throw std::invalid_argument("expert " + std::to_string(e) + " has invalid device");
    ++held[static_cast<std::size_t>(d)];
  }
  const int want = E / D;
  for (int d = 0; d < D; ++d)
    if (held[static_cast<std::size_t>(d)] != want)
      throw std::invalid_argument("device " + std::to_string(d) + " holds " +
                                  std::to_string(held[static_cast<std::size_t>(d)]) +
                                  " experts, expected " + std::to_string(want));
}

// balance.cpp:59-67
Placement contiguous_place(int num_experts, int num_devices) {
  require_divisible(num_experts, num_devices);
  Placement p = empty_placement(num_experts, num_devices);
  const int per = num_experts / num_devices;
  for (int e = 0; e < num_experts; ++e) p.device_of[static_cast<std::size_t>(e)] = e / per;
  return p;
}

// balance.cpp:69-90: centred rows, cross products over row norms, clamped.
CorrMatrix pearson_corr(const LoadMatrix& history) {
  const Eigen::Index E = history.num_experts(), B = history.num_batches();
  if (B < 2) throw std::invalid_argument("pearson_corr requires at least 2 batches");
  const std::vector<double> mean = mean_share(history);
  std::vector<double> c(static_cast<std::size_t>(E * B));  // centred, row-major
  std::vector<double> len(static_cast<std::size_t>(E), 0.0);
  for (Eigen::Index e = 0; e < E; ++e) {
    double ss = 0.0;
    for (Eigen::Index b = 0; b < B; ++b) {
      const double v = history.share(e, b) - mean[static_cast<std::size_t>(e)];
      c[static_cast<std::size_t>(e * B + b)] = v;
      ss += v * v;
    }
    len[static_cast<std::size_t>(e)] = std::sqrt(ss);
  }
  CorrMatrix out;
  out.corr = Eigen::MatrixXd::Zero(E, E);
  for (Eigen::Index i = 0; i < E; ++i) {
    if (len[static_cast<std::size_t>(i)] == 0.0) continue;  // zero variance: all zeros
    for (Eigen::Index j = 0; j < E; ++j) {
      if (len[static_cast<std::size_t>(j)] == 0.0) continue;
      double dot = 0.0;
      for (Eigen::Index b = 0; b < B; ++b)
        dot += c[static_cast<std::size_t>(i * B + b)] * c[static_cast<std::size_t>(j * B + b)];
      const double r = dot / (len[static_cast<std::size_t>(i)] * len[static_cast<std::size_t>(j)]);
      out.corr(i, j) = std::min(1.0, std::max(-1.0, r));
    }
    out.corr(i, i) = 1.0;
  }
  return out;
}

// balance.cpp:92-115
Placement greedy_place(const LoadMatrix& history, int num_devices) {
  const int E = static_cast<int>(history.num_experts());
  require_divisible(E, num_devices);
  const int cap = E / num_devices;
  const std::vector<double> mean = mean_share(history);
  Placement p = empty_placement(E, num_devices);
  std::vector<double> load(static_cast<std::size_t>(num_devices), 0.0);
  std::vector<int> held(static_cast<std::size_t>(num_devices), 0);
  for (int e : heaviest_first(mean)) {
    int pick = -1;
    for (int d = 0; d < num_devices; ++d)
      if (held[static_cast<std::size_t>(d)] < cap &&
          (pick < 0 || load[static_cast<std::size_t>(d)] < load[static_cast<std::size_t>(pick)]))
        pick = d;
    p.device_of[static_cast<std::size_t>(e)] = pick;
    load[static_cast<std::size_t>(pick)] += mean[static_cast<std::size_t>(e)];
    ++held[static_cast<std::size_t>(pick)];
  }
  return p;
}

Placement anticorr_place(const LoadMatrix& history, int num_devices, double weight) {
  return anticorr_place(history, pearson_corr(history), num_devices, weight);
}

// balance.cpp:117-151
Placement anticorr_place(const LoadMatrix& history, const CorrMatrix& corr, int num_devices,
                         double weight) {
  const int E = static_cast<int>(history.num_experts());
  require_divisible(E, num_devices);
  if (corr.corr.rows() != E || corr.corr.cols() != E)
    throw std::invalid_argument("correlation matrix dimension mismatch");
  const int cap = E / num_devices;
  const std::vector<double> mean = mean_share(history);
  Placement p = empty_placement(E, num_devices);
  std::vector<std::vector<int>> on(static_cast<std::size_t>(num_devices));
  for (int a : heaviest_first(mean)) {
    int pick = -1;
    double pick_score = std::numeric_limits<double>::infinity();
    for (int d = 0; d < num_devices; ++d) {
      const std::vector<int>& members = on[static_cast<std::size_t>(d)];
      if (static_cast<int>(members.size()) >= cap) continue;
      double score = 0.0;
      for (int m : members) score += mean[static_cast<std::size_t>(m)] + weight * corr.corr(a, m);
      if (score < pick_score) {
        pick_score = score;
        pick = d;
      }
    }
    p.device_of[static_cast<std::size_t>(a)] = pick;
    on[static_cast<std::size_t>(pick)].push_back(a);
  }
  return p;
}

// balance.cpp:153-165
BalanceReport eval_balance(const Placement& placement, const LoadMatrix& test) {
  validate(placement);
  if (placement.num_experts() != test.num_experts())
    throw std::invalid_argument("placement/load matrix expert count mismatch");
  const int D = placement.num_devices;
  const Eigen::Index B = test.num_batches();
  BalanceReport r;
  r.device_load = Eigen::MatrixXd::Zero(D, B);
  for (int e = 0; e < placement.num_experts(); ++e) {
    const int d = placement.device_of[static_cast<std::size_t>(e)];
    for (Eigen::Index b = 0; b < B; ++b) r.device_load(d, b) += test.share(e, b);
  }
  const double fair = 1.0 / D;
  double max_all = -std::numeric_limits<double>::infinity(), sum_max = 0.0, dev = 0.0;
  for (Eigen::Index b = 0; b < B; ++b) {
    double col_max = -std::numeric_limits<double>::infinity();
    for (int d = 0; d < D; ++d) {
      const double v = r.device_load(d, b);
      col_max = std::max(col_max, v);
      dev = std::max(dev, std::fabs(v - fair));
    }
    max_all = std::max(max_all, col_max);
    sum_max += col_max;
  }
  r.max_load = max_all;
  r.avg_max_load = B ? sum_max / static_cast<double>(B) : 0.0;
  r.objective = dev;
  return r;
}

void save_placement_csv(const Placement& placement, const std::filesystem::path& path) {
  detail::CsvOut out(path);
  out.line("expert", "device");
  for (int e = 0; e < placement.num_experts(); ++e)
    out.line(e, placement.device_of[static_cast<std::size_t>(e)]);
}

// balance.cpp:175-207: header check, "e,d" rows, then validate().
Placement load_placement_csv(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open placement file: " + path.string());
  std::string text;
  if (!std::getline(in, text) || text.compare(0, 13, "expert,device") != 0)
    throw std::runtime_error(path.string() + ": missing expert,device header");
  std::vector<std::pair<int, int>> rows;
  int top_device = -1;
  for (int lineno = 2; std::getline(in, text); ++lineno) {
    if (text.empty()) continue;
    const std::size_t comma = text.find(',');
    std::size_t used_e = 0, used_d = 0;
    int e = -1, d = -1;
    try {
      if (comma == std::string::npos) throw std::invalid_argument("no comma");
      e = std::stoi(text.substr(0, comma), &used_e);
      d = std::stoi(text.substr(comma + 1), &used_d);
    } catch (const std::exception&) {
      throw std::runtime_error(path.string() + ":" + std::to_string(lineno) +
                               ": malformed placement row");
    }
    rows.emplace_back(e, d);
    top_device = std::max(top_device, d);
  }
  Placement p = empty_placement(static_cast<int>(rows.size()), top_device + 1);
  for (const auto& [e, d] : rows) {
    if (e < 0 || e >= static_cast<int>(rows.size()))
      throw std::runtime_error(path.string() + ": expert id out of range");
    p.device_of[static_cast<std::size_t>(e)] = d;
  }
  validate(p);
  return p;
}

}  // namespace moesim

// ------------------------------------------------------------------ C entry points
namespace {

moesim::LoadMatrix wrap_history(const double* share, int E, int B) {
  moesim::LoadMatrix h;
  h.share = Eigen::MatrixXd::Zero(E, B);
  for (int e = 0; e < E; ++e)
    for (int b = 0; b < B; ++b) h.share(e, b) = share[static_cast<std::size_t>(e) * B + b];
  return h;
}

thread_local std::string g_place_err;

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& ex) {
    g_place_err = ex.what();
    return 1;
  } catch (const std::exception& ex) {
    g_place_err = ex.what();
    return 2;
  }
}

void emit(const moesim::Placement& p, int32_t* device_of) {
  for (std::size_t e = 0; e < p.device_of.size(); ++e) device_of[e] = p.device_of[e];
}

}  // namespace

extern "C" {

const char* moesim_placement_last_error(void) { return g_place_err.c_str(); }

int moesim_contiguous_place(int E, int D, int32_t* device_of) {
  return guarded([&] { emit(moesim::contiguous_place(E, D), device_of); });
}

int moesim_greedy_place(const double* share, int E, int B, int D, int32_t* device_of) {
  return guarded([&] { emit(moesim::greedy_place(wrap_history(share, E, B), D), device_of); });
}

int moesim_anticorr_place(const double* share, int E, int B, int D, double weight,
                          int32_t* device_of) {
  return guarded(
      [&] { emit(moesim::anticorr_place(wrap_history(share, E, B), D, weight), device_of); });
}

int moesim_pearson_corr(const double* share, int E, int B, double* corr) {
  return guarded([&] {
    const moesim::CorrMatrix c = moesim::pearson_corr(wrap_history(share, E, B));
    for (int i = 0; i < E; ++i)
      for (int j = 0; j < E; ++j) corr[static_cast<std::size_t>(i) * E + j] = c.corr(i, j);
  });
}

int moesim_eval_balance(const int32_t* device_of, int E, int D, const double* share, int B,
                        double* device_load, double* max_load, double* avg_max_load,
                        double* objective) {
  return guarded([&] {
    moesim::Placement p;
    p.num_devices = D;
    p.device_of.assign(device_of, device_of + E);
    const moesim::BalanceReport r = moesim::eval_balance(p, wrap_history(share, E, B));
    if (device_load)
      for (int d = 0; d < D; ++d)
        for (int b = 0; b < B; ++b) device_load[static_cast<std::size_t>(d) * B + b] = r.device_load(d, b);
    if (max_load) *max_load = r.max_load;
    if (avg_max_load) *avg_max_load = r.avg_max_load;
    if (objective) *objective = r.objective;
  });
}

}  // extern "C"
