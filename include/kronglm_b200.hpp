// C++ drop-in for the reference's fitting API (kronglm::fit_path and friends,
// /root/reference/proj/include/kronglm/{array,design,family,penalty,path}.hpp)
// on top of the C ABI in kronglm_b200.h.  Header-only; link libkronglm_b200.so.
//
// Differences from the reference surface, all forced by "no Eigen":
//   * Matrix is an in-house column-major FP64 matrix (same memory layout as
//     Eigen::MatrixXd, array.hpp:11);
//   * coefficient vectors are std::vector<double> (the vec() of the blocks,
//     design.hpp:51-78).
// Error convention mirrors the reference (path.cpp / family.hpp): kg_status is
// turned back into std::invalid_argument, kronglm::EvalError (with the cell),
// std::runtime_error.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "kronglm_b200.h"

namespace kronglm_b200 {

using Index = std::int64_t;

class EvalError : public std::runtime_error {  // family.hpp:53-61
 public:
  EvalError(const std::string& what, Index cell) : std::runtime_error(what), cell_(cell) {}
  Index cell() const { return cell_; }

 private:
  Index cell_;
};

inline void check(kg_status st, const kg_ctx* ctx) {
  if (st == KG_OK) return;
  const std::string msg = ctx ? kg_last_error(ctx) : "kronglm_b200 error";
  switch (st) {
    case KG_EINVAL: throw std::invalid_argument(msg);
    case KG_EEVAL: throw EvalError(msg, kg_last_error_cell(ctx));
    default: throw std::runtime_error(msg);
  }
}

// Column-major FP64 matrix (Eigen::MatrixXd layout).
struct Matrix {
  Index rows = 0, cols = 0;
  std::vector<double> data;
  Matrix() = default;
  Matrix(Index r, Index c) : rows(r), cols(c), data(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(Index i, Index j) { return data[static_cast<size_t>(i + rows * j)]; }
  double operator()(Index i, Index j) const { return data[static_cast<size_t>(i + rows * j)]; }
};

// One CUDA device; owns the stream, workspaces and captured graphs.
class Context {
 public:
  explicit Context(int device = 0) {
    kg_ctx* c = nullptr;
    check(kg_ctx_create(device, &c), nullptr);
    ctx_.reset(c);
  }
  kg_ctx* get() const { return ctx_.get(); }

 private:
  struct Del {
    void operator()(kg_ctx* c) const { kg_ctx_destroy(c); }
  };
  std::unique_ptr<kg_ctx, Del> ctx_;
};

// TensorDesign(std::vector<std::vector<Matrix>>) (design.hpp:17).
class TensorDesign {
 public:
  TensorDesign(Context& ctx, const std::vector<std::vector<Matrix>>& components) : ctx_(&ctx) {
    if (components.empty() || components.front().empty())
      throw std::invalid_argument("TensorDesign: need at least one component and one marginal factor");
    c_ = static_cast<Index>(components.size());
    d_ = static_cast<Index>(components.front().size());
    std::vector<int64_t> n(static_cast<size_t>(d_)), p;
    std::vector<const double*> X;
    for (Index j = 0; j < d_; ++j) n[static_cast<size_t>(j)] = components.front()[static_cast<size_t>(j)].rows;
    for (const auto& comp : components) {
      if (static_cast<Index>(comp.size()) != d_)
        throw std::invalid_argument("TensorDesign: components must share the array order d");
      for (Index j = 0; j < d_; ++j) {
        const Matrix& m = comp[static_cast<size_t>(j)];
        if (m.rows != n[static_cast<size_t>(j)])
          throw std::invalid_argument("TensorDesign: factor row counts differ across components");
        p.push_back(m.cols);
        X.push_back(m.data.data());
      }
    }
    kg_design* h = nullptr;
    check(kg_design_create(ctx.get(), c_, d_, n.data(), p.data(), X.data(), &h), ctx.get());
    h_.reset(h);
    rows_ = n;
  }
  kg_design* get() const { return h_.get(); }
  Context& ctx() const { return *ctx_; }
  Index n() const { return kg_design_n(h_.get()); }
  Index p() const { return kg_design_p(h_.get()); }
  const std::vector<int64_t>& row_dims() const { return rows_; }

 private:
  struct Del {
    void operator()(kg_design* d) const { kg_design_destroy(d); }
  };
  Context* ctx_;
  Index c_ = 0, d_ = 0;
  std::vector<int64_t> rows_;
  std::unique_ptr<kg_design, Del> h_;
};

enum class Family { gaussian = KG_GAUSSIAN, binomial = KG_BINOMIAL, poisson = KG_POISSON, gamma = KG_GAMMA };

struct FamilySpec {  // family.hpp:26-35
  Family family = Family::gaussian;
  double dispersion = 1.0;
  static FamilySpec gaussian() { return {Family::gaussian, 1.0}; }
  static FamilySpec binomial() { return {Family::binomial, 1.0}; }
  static FamilySpec poisson() { return {Family::poisson, 1.0}; }
  static FamilySpec gamma_log() { return {Family::gamma, 1.0}; }
};

struct PenaltySpec {  // penalty.hpp:14-23
  int kind = KG_LASSO;
  double alpha = 0.0;
  static PenaltySpec lasso() { return {KG_LASSO, 0.0}; }
  static PenaltySpec ridge() { return {KG_RIDGE, 0.0}; }
  static PenaltySpec elastic_net(double a) {
    if (!(a >= 0.0)) throw std::invalid_argument("elastic net alpha must be nonnegative");
    return {KG_ELASTIC_NET, a};
  }
};

// ObservationData(y[, a]) (family.hpp:40-47): arrays in column-major order.
class ObservationData {
 public:
  ObservationData(const TensorDesign& design, const std::vector<double>& y, const std::vector<double>* a = nullptr) {
    if (static_cast<Index>(y.size()) != design.n())
      throw std::invalid_argument("ObservationData: response size does not match the design");
    if (a && a->size() != y.size()) throw std::invalid_argument("ObservationData: response and weight dims differ");
    kg_obs* h = nullptr;
    check(kg_obs_create(design.ctx().get(), design.get(), y.data(), a ? a->data() : nullptr, 0, &h),
          design.ctx().get());
    h_.reset(h);
  }
  kg_obs* get() const { return h_.get(); }

 private:
  struct Del {
    void operator()(kg_obs* o) const { kg_obs_destroy(o); }
  };
  std::unique_ptr<kg_obs, Del> h_;
};

struct PathConfig {  // path.hpp:9-13 (+ OuterConfig, InnerConfig)
  kg_path_cfg cfg;
  PathConfig() { kg_path_cfg_default(&cfg); }
};

struct FitPath {  // path.hpp:18-27
  std::vector<double> lambdas;
  std::vector<std::vector<double>> fits;
  std::vector<double> objectives;
  std::vector<Index> outer_iters, inner_iters;
  std::vector<int> status;
  bool truncated = false;
  double lambda_max_value = 0.0;
  Index n_models() const { return static_cast<Index>(lambdas.size()); }
};

namespace detail {
inline FitPath collect(kg_path_result* r, Index p) {
  FitPath out;
  const Index m = kg_result_n_models(r);
  out.truncated = kg_result_truncated(r) != 0;
  out.lambda_max_value = kg_result_lambda_max(r);
  for (Index t = 0; t < m; ++t) {
    out.lambdas.push_back(kg_result_lambda(r, t));
    out.objectives.push_back(kg_result_objective(r, t));
    out.outer_iters.push_back(kg_result_outer_iters(r, t));
    out.inner_iters.push_back(kg_result_inner_iters(r, t));
    out.status.push_back(kg_result_status(r, t));
    std::vector<double> c(static_cast<size_t>(p));
    if (kg_result_coef(r, t, c.data()) != KG_OK) throw std::runtime_error("kg_result_coef failed");
    out.fits.push_back(std::move(c));
  }
  kg_result_free(r);
  return out;
}
}  // namespace detail

// fit_path (path.hpp:36-39): lambda_max and the log grid computed on the device.
inline FitPath fit_path(const TensorDesign& design, const FamilySpec& spec, const ObservationData& data,
                        const PenaltySpec& penalty, const PathConfig& config) {
  kg_path_result* r = nullptr;
  check(kg_fit_path(design.ctx().get(), design.get(), data.get(), static_cast<int>(spec.family), spec.dispersion,
                    penalty.kind, penalty.alpha, &config.cfg, nullptr, 0, &r),
        design.ctx().get());
  return detail::collect(r, design.p());
}

// fit_path over an explicit strictly decreasing grid (path.hpp:41-43).
inline FitPath fit_path(const TensorDesign& design, const FamilySpec& spec, const ObservationData& data,
                        const PenaltySpec& penalty, const PathConfig& config, const std::vector<double>& lambdas) {
  kg_path_result* r = nullptr;
  check(kg_fit_path(design.ctx().get(), design.get(), data.get(), static_cast<int>(spec.family), spec.dispersion,
                    penalty.kind, penalty.alpha, &config.cfg, lambdas.data(), static_cast<int64_t>(lambdas.size()),
                    &r),
        design.ctx().get());
  return detail::collect(r, design.p());
}

// h_map / g_map (design.hpp:83-92) on host vectors.
inline std::vector<double> h_map(const TensorDesign& design, const std::vector<double>& coef) {
  std::vector<double> eta(static_cast<size_t>(design.n()));
  check(kg_h_map(design.ctx().get(), design.get(), coef.data(), eta.data()), design.ctx().get());
  return eta;
}

inline std::vector<double> g_map(const TensorDesign& design, const std::vector<double>& u) {
  std::vector<double> coef(static_cast<size_t>(design.p()));
  check(kg_g_map(design.ctx().get(), design.get(), u.data(), coef.data()), design.ctx().get());
  return coef;
}

// mse_heldout (path.hpp:55-64, path.cpp:91-126): per model the sum over the
// mask == 1 cells of (mean - y_full)^2 and the first minimizing model.  The
// predictions (h_map + inverse link) run on the device via kg_predict.
struct HeldoutMse {
  std::vector<double> mse;
  Index argmin = 0;
};

inline HeldoutMse mse_heldout(const FitPath& path, const TensorDesign& design, const FamilySpec& spec,
                              const std::vector<double>& y_full, const std::vector<double>& heldout_mask) {
  const size_t n = static_cast<size_t>(design.n());
  if (y_full.size() != n || heldout_mask.size() != n)
    throw std::invalid_argument("mse_heldout: array dims do not match the design");
  Index n_held = 0;
  for (double m : heldout_mask) {
    if (m != 0.0 && m != 1.0) throw std::invalid_argument("mse_heldout: mask entries must be 0 or 1");
    if (m == 1.0) ++n_held;
  }
  if (n_held == 0) throw std::invalid_argument("mse_heldout: empty held-out mask");
  if (path.n_models() == 0) throw std::invalid_argument("mse_heldout: empty path");
  HeldoutMse out;
  std::vector<double> eta(n), mu(n);
  for (Index t = 0; t < path.n_models(); ++t) {
    check(kg_predict(design.ctx().get(), design.get(), static_cast<int>(spec.family),
                     path.fits[static_cast<size_t>(t)].data(), eta.data(), mu.data()),
          design.ctx().get());
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i)
      if (heldout_mask[i] == 1.0) {
        const double diff = mu[i] - y_full[i];
        sum += diff * diff;
      }
    out.mse.push_back(sum);
    if (sum < out.mse[static_cast<size_t>(out.argmin)]) out.argmin = t;
  }
  return out;
}

// bspline_design (bspline.hpp:36): clamped uniform basis on the grid points.
inline Matrix bspline_design(const std::vector<double>& points, Index order, Index n_basis) {
  Matrix m(static_cast<Index>(points.size()), n_basis);
  if (kg_bspline_design(static_cast<int64_t>(points.size()), points.data(), order, n_basis, m.data.data()) != KG_OK)
    throw std::invalid_argument("bspline_design: invalid grid or basis specification");
  return m;
}

// bin_scatter (bspline.hpp:33-45) on the device: points are d-vectors, bounds
// (lo, hi) per dimension, bins per dimension; counts are column-major over
// the bins grid (prod bins entries), dropped = points outside the bounds.
struct BinnedCounts {
  std::vector<Index> dims;
  std::vector<double> counts;
  Index dropped = 0;
};

inline BinnedCounts bin_scatter(const Context& ctx, const std::vector<std::vector<double>>& points,
                                const std::vector<std::pair<double, double>>& bounds,
                                const std::vector<Index>& bins) {
  const size_t d = bins.size();
  if (d == 0 || bounds.size() != d)
    throw std::invalid_argument("bin_scatter: bounds and bins must agree on the dimension");
  std::vector<double> flat;
  flat.reserve(points.size() * d);
  for (const auto& pt : points) {
    if (pt.size() != d) throw std::invalid_argument("bin_scatter: point arity does not match the grid");
    flat.insert(flat.end(), pt.begin(), pt.end());
  }
  std::vector<double> lo(d), hi(d);
  std::vector<int64_t> nb(d);
  Index cells = 1;
  for (size_t j = 0; j < d; ++j) {
    lo[j] = bounds[j].first;
    hi[j] = bounds[j].second;
    nb[j] = bins[j];
    cells *= bins[j] > 0 ? bins[j] : 1;
  }
  BinnedCounts out;
  out.dims = bins;
  out.counts.assign(static_cast<size_t>(cells), 0.0);
  int64_t dropped = 0;
  check(kg_bin_scatter(ctx.get(), static_cast<int64_t>(points.size()), static_cast<int64_t>(d), flat.data(),
                       lo.data(), hi.data(), nb.data(), 0, out.counts.data(), &dropped),
        ctx.get());
  out.dropped = dropped;
  return out;
}

}  // namespace kronglm_b200
