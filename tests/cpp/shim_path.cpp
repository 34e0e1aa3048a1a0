// C++ drop-in check: the reference-style fit_path call sequence
// (TensorDesign -> ObservationData -> fit_path) through include/kronglm_b200.hpp.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>

#include "kronglm_b200.hpp"

using namespace kronglm_b200;

int main() {
  Context ctx(0);
  std::vector<double> g1(24), g2(20);
  for (size_t i = 0; i < g1.size(); ++i) g1[i] = static_cast<double>(i) / 23.0;
  for (size_t i = 0; i < g2.size(); ++i) g2[i] = static_cast<double>(i) / 19.0;
  TensorDesign design(ctx, {{bspline_design(g1, 4, 8), bspline_design(g2, 4, 7)}});
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::vector<double> theta(static_cast<size_t>(design.p()), 0.0);
  for (size_t i = 0; i < theta.size(); i += 5) theta[i] = nd(rng);
  std::vector<double> y = h_map(design, theta);
  for (double& v : y) v += 0.3 * nd(rng);
  ObservationData data(design, y);
  PathConfig cfg;
  cfg.cfg.n_lambda = 12;
  cfg.cfg.lambda_min_ratio = 1e-3;
  FitPath path = fit_path(design, FamilySpec::gaussian(), data, PenaltySpec::lasso(), cfg);
  int bad = 0;
  if (path.n_models() != 12 || path.truncated) bad |= 1;
  for (double c : path.fits[0]) bad |= (c != 0.0) ? 2 : 0;  // model 0 sits at lambda_max
  for (Index t = 1; t < path.n_models(); ++t) {
    if (!(path.lambdas[t] < path.lambdas[t - 1])) bad |= 4;
    if (path.objectives[t] > path.objectives[t - 1] + 1e-12) bad |= 8;
  }
  // adjoint identity through the shim
  std::vector<double> u(static_cast<size_t>(design.n()));
  for (double& v : u) v = nd(rng);
  const std::vector<double> gu = g_map(design, u), h = h_map(design, theta);
  double lhs = 0.0, rhs = 0.0;
  for (size_t i = 0; i < u.size(); ++i) lhs += h[i] * u[i];
  for (size_t i = 0; i < gu.size(); ++i) rhs += theta[i] * gu[i];
  if (std::abs(lhs - rhs) > 1e-10 * std::max(1.0, std::abs(rhs))) bad |= 16;
  // error convention: pure ridge needs an explicit grid (path.cpp:33-37)
  try {
    fit_path(design, FamilySpec::gaussian(), data, PenaltySpec::ridge(), cfg);
    bad |= 32;
  } catch (const std::invalid_argument&) {
  }
  // mse_heldout (path.cpp:91-126): a single held-out cell gives the squared residual
  {
    std::vector<double> mask(static_cast<size_t>(design.n()), 0.0);
    mask[5] = 1.0;
    const HeldoutMse ho = mse_heldout(path, design, FamilySpec::gaussian(), y, mask);
    if (ho.mse.size() != static_cast<size_t>(path.n_models())) bad |= 64;
    for (Index t = 0; t < path.n_models(); ++t) {
      const std::vector<double> e = h_map(design, path.fits[static_cast<size_t>(t)]);
      const double d = e[5] - y[5];
      if (std::abs(ho.mse[static_cast<size_t>(t)] - d * d) > 1e-12 * std::max(1.0, d * d)) bad |= 64;
    }
  }
  // bin_scatter (test_bspline.cpp:123-130 corner and boundary conventions)
  {
    const BinnedCounts bc = bin_scatter(ctx, {{0.0, 0.0}, {1.0, 2.0}, {0.499, 1.999}, {1.5, 0.0}}, {{0.0, 1.0}, {0.0, 2.0}},
                                        {2, 4});
    if (bc.dropped != 1 || bc.counts[0] != 1.0 || bc.counts[1 + 2 * 3] != 1.0 || bc.counts[0 + 2 * 3] != 1.0) bad |= 128;
  }
  std::printf("shim_path models=%lld lambda_max=%.6g final_objective=%.9g status=%d\n",
              static_cast<long long>(path.n_models()), path.lambda_max_value, path.objectives.back(), bad);
  return bad;
}
