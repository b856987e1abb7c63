/*
 * gtoracle.c — CPU oracle for the BO surrogate pass. TEST INFRASTRUCTURE ONLY.
 *
 * Restates the reference algorithm in plain C, line by line:
 *   /root/reference/proj/include/gridtune/gp.hpp            (Matern, fit, predict)
 *   /root/reference/proj/include/gridtune/acquisition.hpp   (PI/EI/LCB, CV lambda)
 *   /root/reference/proj/include/gridtune/portfolio.hpp     (best_candidate)
 *   /root/reference/proj/include/gridtune/strategies.hpp    (one run_bo iteration)
 * Eigen's internal operation orders (blocked LLT, vectorised reductions) are
 * not reproducible without Eigen; this file uses the unblocked column
 * recurrence and sequential sums.
 * Compiled with -ffp-contract=off (oracle/Makefile): no FMA contraction.
 */
#include "gtoracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

double gto_matern(int nu, double lengthscale, double s2, double r) {
  /* gp.hpp:40-55 */
  const double s = r / lengthscale;
  if (nu == 0) return s2 * exp(-s);
  if (nu == 1) {
    const double a = 1.7320508075688772 * s;
    return s2 * (1.0 + a) * exp(-a);
  }
  {
    const double a = 2.2360679774997896 * s;
    return s2 * (1.0 + a + a * a / 3.0) * exp(-a);
  }
}

/* Unblocked lower LLT (Eigen's llt_inplace column recurrence). 0 ok, k+1 on
 * the failing pivot k. */
static int llt(double* A, int n) {
  for (int k = 0; k < n; ++k) {
    double x = A[k * n + k];
    for (int m = 0; m < k; ++m) x -= A[k * n + m] * A[k * n + m];
    if (x <= 0.0) return k + 1;
    x = sqrt(x);
    A[k * n + k] = x;
    for (int i = k + 1; i < n; ++i) {
      double s = A[i * n + k];
      for (int m = 0; m < k; ++m) s -= A[i * n + m] * A[k * n + m];
      A[i * n + k] = s / x;
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) A[i * n + j] = 0.0;
  return 0;
}

int gto_gp_fit(int nu, double lengthscale, double s2, const double* X, const double* y, int n,
               int d, double noise, double jitter, double* L, double* alpha, double* scalars) {
  /* gp.hpp:84-89 validation */
  if (!(noise >= 0.0) || !(jitter > 0.0) || n < 0) return -1;
  for (int i = 0; i < n; ++i)
    if (!isfinite(y[i])) return -1;
  double y_mean = 0.0, y_std = 1.0;
  if (n > 0) {
    double sum = 0.0;
    for (int i = 0; i < n; ++i) sum += y[i];
    y_mean = sum / (double)n; /* gp.hpp:98 */
    if (n > 1) {              /* gp.hpp:99-102, population variance */
      double ss = 0.0;
      for (int i = 0; i < n; ++i) ss += (y[i] - y_mean) * (y[i] - y_mean);
      const double var = ss / (double)n;
      y_std = var > 0.0 ? sqrt(var) : 1.0;
    }
  }
  scalars[0] = y_mean;
  scalars[1] = y_std;
  scalars[2] = jitter;
  if (n == 0) return 0;

  double* gram = (double*)malloc(sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n; ++i) { /* gp.hpp:106-114 direct differences */
    gram[i * n + i] = gto_matern(nu, lengthscale, s2, 0.0);
    for (int j = i + 1; j < n; ++j) {
      double ss = 0.0;
      for (int t = 0; t < d; ++t) {
        const double dv = X[i * d + t] - X[j * d + t];
        ss += dv * dv;
      }
      const double k = gto_matern(nu, lengthscale, s2, sqrt(ss));
      gram[i * n + j] = k;
      gram[j * n + i] = k;
    }
  }
  double jit = jitter;
  int attempts = 0;
  for (;;) { /* gp.hpp:116-129 */
    memcpy(L, gram, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i) L[i * n + i] += noise + jit;
    if (llt(L, n) == 0) break;
    if (++attempts > 6) {
      free(gram);
      scalars[2] = jit;
      return -2;
    }
    jit *= 2.0;
  }
  free(gram);
  scalars[2] = jit;
  /* alpha = L^-T L^-1 y_standardized, gp.hpp:103,130 */
  for (int i = 0; i < n; ++i) {
    double s = (y[i] - y_mean) / y_std;
    for (int m = 0; m < i; ++m) s -= L[i * n + m] * alpha[m];
    alpha[i] = s / L[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = alpha[i];
    for (int m = i + 1; m < n; ++m) s -= L[m * n + i] * alpha[m];
    alpha[i] = s / L[i * n + i];
  }
  return 0;
}

void gto_gp_predict(int nu, double lengthscale, double s2, const double* X, int n, int d,
                    const double* L, const double* alpha, const double* Xstar, int64_t m,
                    double* mean, double* var) {
  if (n == 0) { /* prior, gp.hpp:155-158 */
    for (int64_t j = 0; j < m; ++j) {
      mean[j] = 0.0;
      var[j] = s2;
    }
    return;
  }
  double* an = (double*)malloc(sizeof(double) * (size_t)n);
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int t = 0; t < d; ++t) s += X[i * d + t] * X[i * d + t];
    an[i] = s;
  }
  for (int64_t j = 0; j < m; ++j) {
    const double* b = Xstar + j * d;
    double bn = 0.0;
    for (int t = 0; t < d; ++t) bn += b[t] * b[t];
    double mu = 0.0, q = 0.0;
    for (int i = 0; i < n; ++i) {
      /* gp.hpp:176-190: d2 = -2 a.b + |a|^2 + |b|^2, clamp, sqrt, / l, closed form */
      double dot = 0.0;
      for (int t = 0; t < d; ++t) dot += X[i * d + t] * b[t];
      double d2 = -2.0 * dot;
      d2 += an[i];
      d2 += bn;
      const double k = gto_matern(nu, lengthscale, s2, sqrt(d2 > 0.0 ? d2 : 0.0));
      mu += k * alpha[i]; /* mean = kstar^T alpha, gp.hpp:162 */
      /* forward substitution row i, gp.hpp:163-164 */
      double s = k;
      for (int r = 0; r < i; ++r) s -= L[i * n + r] * v[r];
      v[i] = s / L[i * n + i];
      q += v[i] * v[i]; /* colwise squared sum, gp.hpp:165 */
    }
    mean[j] = mu;
    const double vv = s2 - q;
    var[j] = vv > 0.0 ? vv : 0.0; /* gp.hpp:166 */
  }
  free(an);
  free(v);
}

static double normal_pdf(double z) { return 0.3989422804014326779 * exp(-0.5 * z * z); }
static double normal_cdf(double z) { return 0.5 * erfc(-z * 0.70710678118654752440); }

double gto_acq_pi(double mean, double sd, double best_std, double lambda) {
  const double margin = best_std + lambda - mean; /* acquisition.hpp:25-29 */
  if (sd <= 0.0) return margin > 0.0 ? 1.0 : 0.0;
  return normal_cdf(margin / sd);
}

double gto_acq_ei(double mean, double sd, double best_std, double lambda) {
  const double margin = best_std - lambda - mean; /* acquisition.hpp:32-37 */
  if (sd <= 0.0) return margin > 0.0 ? margin : 0.0;
  const double z = margin / sd;
  return margin * normal_cdf(z) + sd * normal_pdf(z);
}

double gto_acq_lcb(double mean, double sd, double lambda) { return mean - lambda * sd; }

int gto_cv_lambda(double mu_s, double var_s, double mean_variance, double f_best_raw, double* lambda) {
  /* acquisition.hpp:73-83 */
  if (!(f_best_raw > 0.0) || !(mu_s > 0.0) || !(var_s > 0.0)) return 0;
  const double l = (mean_variance * f_best_raw / mu_s) / var_s;
  *lambda = l > 0.0 ? l : 0.0;
  return 1;
}

static double score_of(int af, double mean, double sd, double best, double lambda) {
  switch (af) {
    case 0: return gto_acq_ei(mean, sd, best, lambda);
    case 1: return gto_acq_pi(mean, sd, best, lambda);
    case 2: return -gto_acq_lcb(mean, sd, lambda); /* portfolio.hpp:47 */
  }
  return 0.0;
}

int64_t gto_best_candidate(int af, const double* means, const double* stds, int64_t n,
                           double best_std, double lambda, const uint8_t* excluded,
                           double* score_out) {
  /* portfolio.hpp:32-61 */
  int64_t best = -1;
  double best_score = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (excluded && excluded[i]) continue;
    const double s = score_of(af, means[i], stds[i], best_std, lambda);
    if (best == -1 || s > best_score) {
      best = i;
      best_score = s;
    }
  }
  if (score_out) *score_out = best_score;
  return best;
}

double gto_mean(const double* v, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += v[i];
  return s / (double)n;
}

int gto_iteration(int nu, double lengthscale, double s2, const double* coords, int64_t N, int d,
                  const int64_t* train_pos, const double* y, int n, double noise, double jitter,
                  const uint8_t* visited, uint32_t af_mask, int lambda_mode, double lambda_const,
                  double cv_mu_s, double cv_var_s, double f_best_raw, int64_t* pick_out,
                  double* lambda_out) {
  double* X = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * d);
  double* L = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * (n > 0 ? n : 1));
  double* alpha = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double sc[3];
  for (int i = 0; i < n; ++i) memcpy(X + i * d, coords + train_pos[i] * d, sizeof(double) * d);
  int rc = gto_gp_fit(nu, lengthscale, s2, X, y, n, d, noise, jitter, L, alpha, sc);
  if (rc) {
    free(X); free(L); free(alpha);
    return rc;
  }
  int64_t U = 0;
  for (int64_t j = 0; j < N; ++j) U += visited[j] ? 0 : 1;
  int64_t* cand = (int64_t*)malloc(sizeof(int64_t) * (size_t)(U > 0 ? U : 1));
  double* Xs = (double*)malloc(sizeof(double) * (size_t)(U > 0 ? U : 1) * d);
  double* mean = (double*)malloc(sizeof(double) * (size_t)(U > 0 ? U : 1));
  double* var = (double*)malloc(sizeof(double) * (size_t)(U > 0 ? U : 1));
  int64_t u = 0;
  for (int64_t j = 0; j < N; ++j)
    if (!visited[j]) {
      cand[u] = j;
      memcpy(Xs + u * d, coords + j * d, sizeof(double) * d);
      ++u;
    }
  gto_gp_predict(nu, lengthscale, s2, X, n, d, L, alpha, Xs, U, mean, var);
  /* mean posterior variance over the candidates, strategies.hpp:406-407 */
  const double mv = U > 0 ? gto_mean(var, U) : 0.0;
  for (int64_t j = 0; j < U; ++j) var[j] = sqrt(var[j]); /* stds, strategies.hpp:385 */
  double lambda = lambda_const;
  if (lambda_mode == 1) gto_cv_lambda(cv_mu_s, cv_var_s, mv, f_best_raw, &lambda);
  const double best_std = (f_best_raw - sc[0]) / sc[1];
  for (int af = 0; af < 3; ++af) {
    pick_out[af] = -1;
    if (af_mask & (1u << af)) {
      const int64_t p = gto_best_candidate(af, mean, var, U, best_std, lambda, NULL, NULL);
      pick_out[af] = p >= 0 ? cand[p] : -1;
    }
  }
  if (lambda_out) *lambda_out = lambda;
  free(X); free(L); free(alpha); free(cand); free(Xs); free(mean); free(var);
  return 0;
}
