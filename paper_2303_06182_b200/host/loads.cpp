// Load-matrix utilities of include/moesim/trace.hpp (reference
// proj/src/trace.cpp:261-313): the train/test split of the two-half
// placement protocol, sparsity statistics and the load CSV.
#include <algorithm>
#include <cmath>
#include <fstream>
#include <limits>
#include <stdexcept>
#include <string>

#include "csv_out.hpp"
#include "moesim/trace.hpp"

namespace moesim {

// trace.cpp:261-274.  cut = floor(fraction * B), except that a product within
// 1e-9 (relative) of an integer snaps to it.
std::pair<LoadMatrix, LoadMatrix> split_trace(const LoadMatrix& loads, double fraction) {
  const Eigen::Index B = loads.num_batches();
  if (B < 2) throw std::invalid_argument("split requires at least 2 batches");
  if (!(fraction > 0.0 && fraction < 1.0)) throw std::invalid_argument("split fraction must be in (0, 1)");
  const double x = fraction * static_cast<double>(B);
  const double r = std::round(x);
  const Eigen::Index cut = std::fabs(x - r) < 1e-9 * std::max(1.0, x) ? static_cast<Eigen::Index>(r)
                                                                     : static_cast<Eigen::Index>(std::floor(x));
  if (cut <= 0 || cut >= B) throw std::invalid_argument("split produces an empty part");
  const Eigen::Index E = loads.num_experts();
  std::pair<LoadMatrix, LoadMatrix> parts;
  parts.first.share = Eigen::MatrixXd::Zero(E, cut);
  parts.second.share = Eigen::MatrixXd::Zero(E, B - cut);
  for (Eigen::Index e = 0; e < E; ++e)
    for (Eigen::Index b = 0; b < B; ++b)
      (b < cut ? parts.first.share(e, b) : parts.second.share(e, b - cut)) = loads.share(e, b);
  return parts;
}

// trace.cpp:276-299
SparsityReport sparsity_stats(const LoadMatrix& loads) {
  const Eigen::Index E = loads.num_experts(), B = loads.num_batches();
  SparsityReport rep;
  rep.inactive_per_batch.assign(static_cast<std::size_t>(B), 0);
  rep.top_share_per_batch.assign(static_cast<std::size_t>(B), 0.0);
  rep.mean_load = Eigen::VectorXd::Zero(E);
  std::vector<char> ever(static_cast<std::size_t>(E), 0);
  double frac_total = 0.0;
  for (Eigen::Index b = 0; b < B; ++b) {
    int zeros = 0;
    double top = -std::numeric_limits<double>::infinity();
    for (Eigen::Index e = 0; e < E; ++e) {
      const double v = loads.share(e, b);
      zeros += v == 0.0;
      top = std::max(top, v);
    }
    rep.inactive_per_batch[static_cast<std::size_t>(b)] = zeros;
    rep.top_share_per_batch[static_cast<std::size_t>(b)] = top;
    const double f = static_cast<double>(zeros) / static_cast<double>(E);
    frac_total += f;
    rep.max_inactive_fraction = std::max(rep.max_inactive_fraction, f);
  }
  for (Eigen::Index e = 0; e < E; ++e) {
    double s = 0.0;
    for (Eigen::Index b = 0; b < B; ++b) s += loads.share(e, b);
    rep.mean_load[e] = s / static_cast<double>(B);
    rep.never_active += s == 0.0;
  }
  rep.mean_inactive_fraction = B ? frac_total / static_cast<double>(B) : 0.0;
  return rep;
}

// "expert,b0,b1,..." then one row per expert (trace.cpp:301-313).
void save_load_matrix_csv(const LoadMatrix& loads, const std::filesystem::path& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot write file: " + path.string());
  f << "expert";
  for (Eigen::Index b = 0; b < loads.num_batches(); ++b) f << ",b" << b;
  f << '\n';
  for (Eigen::Index e = 0; e < loads.num_experts(); ++e) {
    f << e;
    for (Eigen::Index b = 0; b < loads.num_batches(); ++b)
      f << ',' << detail::CsvOut::number(loads.share(e, b));
    f << '\n';
  }
}

}  // namespace moesim
