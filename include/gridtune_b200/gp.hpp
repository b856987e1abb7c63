// GP surrogate and acquisition API (gp.hpp:12-212, acquisition.hpp:12-92 of
// the reference) with the factor and predictions on the device.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "gridtune_b200/errors.hpp"

namespace gridtune_b200 {

enum class MaternNu { half = GTC_NU_HALF, three_halves = GTC_NU_THREE_HALVES, five_halves = GTC_NU_FIVE_HALVES };

struct MaternKernel {
  MaternNu nu = MaternNu::three_halves;
  double lengthscale = 2.0;
  double output_variance = 1.0;

  MaternKernel() = default;
  MaternKernel(MaternNu n, double l, double s2 = 1.0) : nu(n), lengthscale(l), output_variance(s2) {
    if (!(lengthscale > 0.0)) throw Error("kernel lengthscale must be positive");
    if (!(output_variance > 0.0)) throw Error("kernel output variance must be positive");
  }
  gtc_kernel c() const { return gtc_kernel{static_cast<std::int32_t>(nu), lengthscale, output_variance}; }
};

struct GpPrediction {
  std::vector<double> mean;
  std::vector<double> variance;
  double y_mean = 0.0;
  double y_std = 1.0;
  double raw_mean(std::size_t i) const { return y_mean + y_std * mean[i]; }
};

/// GpModel over arbitrary points (gp.hpp:74-203); X is n x d row-major.
class GpModel {
 public:
  static GpModel fit(const MaternKernel& kernel, const std::vector<double>& X, std::size_t d,
                     const std::vector<double>& y_raw, double noise = 1e-10, double jitter = 1e-6,
                     int device = 0) {
    if (d == 0 || X.size() != y_raw.size() * d)
      throw Error("GP fit: observation count does not match input count");
    gtc_gp* g = nullptr;
    gtc_fit_info info{};
    const gtc_kernel k = kernel.c();
    check(gtc_gp_fit(device, &k, X.data(), y_raw.data(), static_cast<std::int32_t>(y_raw.size()),
                     static_cast<std::int32_t>(d), noise, jitter, &g, &info));
    GpModel m;
    m.h_.reset(g, [](gtc_gp* p) { gtc_gp_destroy(p); });
    m.kernel_ = kernel;
    m.info_ = info;
    m.noise_ = noise;
    m.d_ = d;
    return m;
  }

  const MaternKernel& kernel() const { return kernel_; }
  std::size_t train_size() const { return static_cast<std::size_t>(info_.n); }
  double y_mean() const { return info_.y_mean; }
  double y_std() const { return info_.y_std; }
  double noise() const { return noise_; }
  double jitter() const { return info_.jitter; }
  double standardize(double y_raw) const { return (y_raw - info_.y_mean) / info_.y_std; }

  GpPrediction predict(const std::vector<double>& Xstar) const {
    GpPrediction out;
    const std::size_t m = Xstar.size() / d_;
    out.mean.resize(m);
    out.variance.resize(m);
    out.y_mean = info_.y_mean;
    out.y_std = info_.y_std;
    if (m) check(gtc_gp_predict(h_.get(), Xstar.data(), static_cast<std::int64_t>(m), out.mean.data(), out.variance.data()));
    return out;
  }

 private:
  GpModel() = default;
  std::shared_ptr<gtc_gp> h_;
  MaternKernel kernel_;
  gtc_fit_info info_{};
  double noise_ = 0.0;
  std::size_t d_ = 1;
};

inline double mean_posterior_variance(const GpPrediction& p) {
  if (p.variance.empty()) throw Error("mean_posterior_variance: empty candidate set");
  double s = 0.0;
  for (double v : p.variance) s += v;
  return s / static_cast<double>(p.variance.size());
}

// ---------------------------------------------------------------- acquisition

enum class AcquisitionId { ei = GTC_AF_EI, poi = GTC_AF_POI, lcb = GTC_AF_LCB };

inline const char* to_string(AcquisitionId id) {
  switch (id) {
    case AcquisitionId::ei: return "ei";
    case AcquisitionId::poi: return "poi";
    case AcquisitionId::lcb: return "lcb";
  }
  return "?";
}

struct ExplorationConfig {
  enum class Mode { constant = GTC_LAMBDA_CONSTANT, contextual_variance = GTC_LAMBDA_CONTEXTUAL_VARIANCE };
  Mode mode = Mode::contextual_variance;
  double constant = 0.01;
};

struct ContextualVarianceState {
  double initial_sample_mean = 0.0;
  double initial_mean_variance = 0.0;
};

/// acquisition.hpp:73-83 (the selection kernel evaluates the same expression).
inline std::optional<double> contextual_variance_lambda(const ContextualVarianceState& s,
                                                        double mean_variance, double f_best_raw) {
  if (!(f_best_raw > 0.0) || !(s.initial_sample_mean > 0.0) || !(s.initial_mean_variance > 0.0))
    return std::nullopt;
  const double l = (mean_variance * f_best_raw / s.initial_sample_mean) / s.initial_mean_variance;
  return l > 0.0 ? l : 0.0;
}

/// acquisition.hpp:88-92
inline double discounted_observation_score(std::span<const double> history, double gamma) {
  double score = 0.0;
  for (double o : history) score = score * gamma + o;
  return score;
}

}  // namespace gridtune_b200
