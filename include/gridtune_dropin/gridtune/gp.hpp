// Drop-in replacement of the reference's gridtune/gp.hpp
// (/root/reference/proj/include/gridtune/gp.hpp) with the GP on the B200.
//
// Put include/gridtune_dropin first on the include path (before the
// reference's include/): every `#include "gridtune/gp.hpp"` -- the
// reference's strategies.hpp and its tests -- then gets this header, while
// the other gridtune headers (errors, acquisition, rng, ...) stay the
// reference's own.  The API is the reference's, Eigen-typed:
//   GpModel::fit(const MaternKernel&, const Eigen::MatrixXd& X,
//                const Eigen::VectorXd& y_raw, double noise, double jitter)  gp.hpp:81-83
//   GpPrediction GpModel::predict(const Eigen::MatrixXd&) const             gp.hpp:150
// The factorisation (Gram matrix, jitter escalation) and the posterior run as
// sm_100a kernels behind the C ABI (gtc_gp_fit / gtc_gp_predict,
// include/gridtune_cuda.h); the model holds a device handle (shared by copies,
// GpModel is an immutable value like the reference's, gp.hpp:71-74).  There is
// no CPU fallback: without a device fit() throws gridtune::Error.
#pragma once

#include <Eigen/Dense>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "gridtune/errors.hpp"
#include "gridtune_cuda.h"

namespace gridtune {

namespace b200 {
// The device of every drop-in model (GRIDTUNE_B200_DEVICE, default 0).
inline int device() {
  static const int dev = [] {
    const char* e = std::getenv("GRIDTUNE_B200_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  return dev;
}

// C-ABI status -> the reference's exception types (errors.hpp:9-64).
inline void check(int rc) {
  if (rc == GTC_OK) return;
  const std::string msg = gtc_last_error();
  switch (rc) {
    case GTC_ERR_CONDITIONING: throw ModelConditioningError(msg);
    case GTC_ERR_CONFIG: throw ConfigError(msg);
    case GTC_ERR_SAMPLING: throw SamplingError(msg);
    default: throw Error(msg);
  }
}

// Eigen (column-major) -> row-major n x d for the C ABI.
template <class M>
std::vector<double> row_major(const M& X) {
  const Eigen::Index n = X.rows(), d = X.cols();
  std::vector<double> out(static_cast<std::size_t>(n * d));
  for (Eigen::Index i = 0; i < n; ++i)
    for (Eigen::Index j = 0; j < d; ++j) out[static_cast<std::size_t>(i * d + j)] = X(i, j);
  return out;
}
}  // namespace b200

enum class MaternNu { half, three_halves, five_halves };

inline const char* to_string(MaternNu nu) {
  constexpr const char* names[] = {"1/2", "3/2", "5/2"};
  const int k = static_cast<int>(nu);
  return k >= 0 && k < 3 ? names[k] : "?";
}

/// Matern covariance (gp.hpp:27-56): the closed forms with the reference's
/// constants and evaluation order, also used by the device kernels
/// (gtc_kernels.cu matern<NU>).
struct MaternKernel {
  MaternNu nu = MaternNu::three_halves;
  double lengthscale = 2.0;
  double output_variance = 1.0;

  MaternKernel() = default;
  MaternKernel(MaternNu n, double l, double s2 = 1.0) : nu(n), lengthscale(l), output_variance(s2) {
    if (!(lengthscale > 0.0)) throw Error("kernel lengthscale must be positive");
    if (!(output_variance > 0.0)) throw Error("kernel output variance must be positive");
  }

  double operator()(double r) const {
    const double s = r / lengthscale;
    if (nu == MaternNu::half) return output_variance * std::exp(-s);
    const bool five = nu == MaternNu::five_halves;
    const double a = (five ? 2.2360679774997896 : 1.7320508075688772) * s;
    const double poly = five ? 1.0 + a + a * a / 3.0 : 1.0 + a;
    return output_variance * poly * std::exp(-a);
  }

  gtc_kernel c() const { return gtc_kernel{static_cast<std::int32_t>(nu), lengthscale, output_variance}; }
};

inline double kernel_eval(const MaternKernel& k, double r) { return k(r); }

/// Posterior over a batch of points in standardized units (gp.hpp:62-69).
struct GpPrediction {
  Eigen::VectorXd mean;
  Eigen::VectorXd variance;
  double y_mean = 0.0;
  double y_std = 1.0;

  double raw_mean(Eigen::Index i) const { return y_mean + y_std * mean(i); }
};

class GpModel {
 public:
  /// gp.hpp:81-135: standardisation, Gram matrix with direct differences,
  /// LLT with jitter doubling (at most six times, then
  /// ModelConditioningError), all on the device.
  static GpModel fit(const MaternKernel& kernel, const Eigen::MatrixXd& X, const Eigen::VectorXd& y_raw,
                     double noise = 1e-10, double jitter = 1e-6) {
    if (X.rows() != y_raw.size()) throw Error("GP fit: observation count does not match input count");
    GpModel m;
    m.kernel_ = kernel;
    m.noise_ = noise;
    m.n_ = static_cast<Eigen::Index>(y_raw.size());
    m.d_ = X.cols();
    std::vector<double> y(static_cast<std::size_t>(m.n_));
    for (Eigen::Index i = 0; i < m.n_; ++i) y[static_cast<std::size_t>(i)] = y_raw(i);
    const std::vector<double> x = b200::row_major(X);
    // (a prior model has no points: its handle is created at the first
    // predict, whose inputs fix the dimension)
    const std::int32_t d = static_cast<std::int32_t>(m.d_ > 0 ? m.d_ : 1);
    std::vector<double> xd = m.d_ > 0 ? x : std::vector<double>(static_cast<std::size_t>(m.n_), 0.0);
    gtc_gp* g = nullptr;
    gtc_fit_info info{};
    const gtc_kernel k = kernel.c();
    b200::check(gtc_gp_fit(b200::device(), &k, xd.data(), y.data(), static_cast<std::int32_t>(m.n_), d, noise,
                           jitter, &g, &info));
    m.h_ = std::shared_ptr<gtc_gp>(g, [](gtc_gp* p) { gtc_gp_destroy(p); });
    m.y_mean_ = info.y_mean;
    m.y_std_ = info.y_std;
    m.jitter_ = info.jitter;
    return m;
  }

  const MaternKernel& kernel() const { return kernel_; }
  Eigen::Index train_size() const { return n_; }
  double y_mean() const { return y_mean_; }
  double y_std() const { return y_std_; }
  double noise() const { return noise_; }
  double jitter() const { return jitter_; }

  /// gp.hpp:145
  double standardize(double y_raw) const { return (y_raw - y_mean_) / y_std_; }

  /// gp.hpp:150-168: k* on the fly, forward solve against the device factor,
  /// mean and clamped variance per point (gtc_gp_predict).
  GpPrediction predict(const Eigen::MatrixXd& Xstar) const {
    GpPrediction out;
    out.y_mean = y_mean_;
    out.y_std = y_std_;
    const Eigen::Index m = Xstar.rows();
    out.mean = Eigen::VectorXd(m);
    out.variance = Eigen::VectorXd(m);
    if (m == 0) return out;
    std::vector<double> mean(static_cast<std::size_t>(m)), var(static_cast<std::size_t>(m));
    std::vector<double> xs = b200::row_major(Xstar);
    gtc_gp* g = h_.get();
    std::shared_ptr<gtc_gp> prior;
    if (n_ == 0 && Xstar.cols() != (d_ > 0 ? d_ : 1)) {  // prior at another dimension
      gtc_gp* p = nullptr;
      const gtc_kernel k = kernel_.c();
      b200::check(gtc_gp_fit(b200::device(), &k, nullptr, nullptr, 0,
                             static_cast<std::int32_t>(Xstar.cols() > 0 ? Xstar.cols() : 1), noise_, jitter_, &p,
                             nullptr));
      prior.reset(p, [](gtc_gp* q) { gtc_gp_destroy(q); });
      g = p;
    }
    if (Xstar.cols() == 0) xs.assign(static_cast<std::size_t>(m), 0.0);
    b200::check(gtc_gp_predict(g, xs.data(), static_cast<std::int64_t>(m), mean.data(), var.data()));
    for (Eigen::Index i = 0; i < m; ++i) {
      out.mean(i) = mean[static_cast<std::size_t>(i)];
      out.variance(i) = var[static_cast<std::size_t>(i)];
    }
    return out;
  }

  /// The device model (for callers that go on to the resident-run ABI).
  const gtc_gp* handle() const { return h_.get(); }

 private:
  GpModel() = default;

  MaternKernel kernel_;
  std::shared_ptr<gtc_gp> h_;
  Eigen::Index n_ = 0;
  Eigen::Index d_ = 0;
  double y_mean_ = 0.0;
  double y_std_ = 1.0;
  double noise_ = 0.0;
  double jitter_ = 1e-6;
};

/// gp.hpp:207-212: mean of the posterior variances of a prediction batch
/// (the values are the device's; this is their host-side arithmetic mean).
inline double mean_posterior_variance(const GpPrediction& prediction) {
  const Eigen::Index m = prediction.variance.size();
  if (m == 0) throw Error("mean_posterior_variance: empty candidate set");
  double s = 0.0;
  for (Eigen::Index i = 0; i < m; ++i) s += prediction.variance(i);
  return s / static_cast<double>(m);
}

}  // namespace gridtune
