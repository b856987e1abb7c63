"""Dense numpy/LAPACK restatement of the reference surrogate pass — TEST
INFRASTRUCTURE ONLY (the checker for large spaces; never imported by the
product package).

Same mathematics as /root/reference/proj/include/gridtune/ with the dense
kernels Eigen would call replaced by LAPACK/BLAS (a blocked Cholesky and a
blocked triangular solve, like Eigen's own LLT / TriangularView::solve):

  matern                  gp.hpp:27-56
  fit                     gp.hpp:81-135   (direct-difference Gram, jitter x2 up to 6 times)
  predict                 gp.hpp:150-168  (expansion-form cross covariance gp.hpp:175-193,
                                           V = L^-1 K*, var = max(s2 - colsum V^2, 0))
  acquisition_pi/ei/lcb   acquisition.hpp:12-42
  cv_lambda               acquisition.hpp:73-83, strategies.hpp:404-418
  best_candidate          portfolio.hpp:32-61
  initial-sample mean     sampling.hpp:68-72

The plain-C oracle (oracle/gtoracle.c) follows the reference's scalar loops
operation by operation for small cases; this module evaluates the same
formulas vectorised so that 10^5-10^6-candidate states (BASELINE configs C3,
C4) can be checked in seconds.  Pinned against the reference's golden
GpModel outputs in tests/test_oracle_golden.py.
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import solve_triangular
from scipy.special import erfc

SQRT3 = 1.7320508075688772
SQRT5 = 2.2360679774997896


def matern(nu: int, lengthscale: float, s2: float, r):
    """gp.hpp:40-55: s = r/l, (s2 * poly(a)) * exp(-a)."""
    s = np.asarray(r, dtype=np.float64) / lengthscale
    if nu == 0:
        return s2 * np.exp(-s)
    if nu == 1:
        a = SQRT3 * s
        return (s2 * (1.0 + a)) * np.exp(-a)
    a = SQRT5 * s
    return (s2 * (1.0 + a + a * a / 3.0)) * np.exp(-a)


class ConditioningError(Exception):
    pass


def fit(nu: int, lengthscale: float, s2: float, X, y, noise: float = 1e-10, jitter: float = 1e-6) -> dict:
    """GpModel::fit (gp.hpp:81-135)."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    n = len(y)
    model = dict(nu=nu, l=lengthscale, s2=s2, X=X, n=n, y_mean=0.0, y_std=1.0, jitter=jitter, noise=noise)
    if n == 0:
        return model
    y_mean = float(np.sum(y)) / n                                    # gp.hpp:98
    y_std = 1.0
    if n > 1:                                                        # gp.hpp:99-102
        var = float(np.sum((y - y_mean) ** 2)) / n
        y_std = float(np.sqrt(var)) if var > 0.0 else 1.0
    ys = (y - y_mean) / y_std
    diff = X[:, None, :] - X[None, :, :]                             # gp.hpp:105-114 direct differences
    gram = matern(nu, lengthscale, s2, np.sqrt(np.sum(diff * diff, axis=2)))
    np.fill_diagonal(gram, matern(nu, lengthscale, s2, 0.0))
    j = jitter
    attempts = 0
    while True:                                                      # gp.hpp:116-129
        try:
            L = np.linalg.cholesky(gram + (noise + j) * np.eye(n))
            break
        except np.linalg.LinAlgError:
            attempts += 1
            if attempts > 6:
                raise ConditioningError(f"Gram matrix factorization failed after jitter escalation to {j:f}")
            j *= 2.0
    alpha = solve_triangular(L.T, solve_triangular(L, ys, lower=True), lower=False)  # gp.hpp:130
    model.update(y_mean=y_mean, y_std=y_std, jitter=j, L=L, alpha=alpha)
    return model


def cross_covariance(model: dict, Q) -> np.ndarray:
    """gp.hpp:175-193: d2 = -2 A B^T + |a|^2 + |b|^2, clamp, sqrt."""
    A = model["X"]
    Q = np.asarray(Q, dtype=np.float64)
    d2 = -2.0 * (A @ Q.T)
    d2 += np.sum(A * A, axis=1)[:, None]
    d2 += np.sum(Q * Q, axis=1)[None, :]
    return matern(model["nu"], model["l"], model["s2"], np.sqrt(np.maximum(d2, 0.0)))


def predict(model: dict, Q, chunk: int = 65536):
    """GpModel::predict (gp.hpp:150-168), standardized scale; in candidate
    chunks so 10^6-candidate states fit in host memory."""
    Q = np.asarray(Q, dtype=np.float64)
    m = len(Q)
    if model["n"] == 0:
        return np.zeros(m), np.full(m, model["s2"])
    mean = np.empty(m)
    var = np.empty(m)
    for a in range(0, m, chunk):
        ks = cross_covariance(model, Q[a:a + chunk])
        mean[a:a + chunk] = ks.T @ model["alpha"]
        v = solve_triangular(model["L"], ks, lower=True)
        var[a:a + chunk] = np.maximum(model["s2"] - np.sum(v * v, axis=0), 0.0)
    return mean, var


def standardize(model: dict, y_raw: float) -> float:
    return (y_raw - model["y_mean"]) / model["y_std"]               # gp.hpp:145


def normal_cdf(z):
    return 0.5 * erfc(-z * 0.70710678118654752440)                 # acquisition.hpp:12-18


def normal_pdf(z):
    return 0.3989422804014326779 * np.exp(-0.5 * z * z)


def acquisition(af: int, mean, sd, best: float, lam: float):
    """acquisition.hpp:25-42; af 0 EI, 1 PI, 2 LCB.  The LCB slot returns
    -lcb (best_candidate maximises it, portfolio.hpp:47)."""
    mean = np.asarray(mean, dtype=np.float64)
    sd = np.asarray(sd, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        if af == 2:
            return -(mean - lam * sd)
        if af == 1:
            margin = best + lam - mean
            z = margin / np.where(sd > 0.0, sd, 1.0)
            return np.where(sd > 0.0, normal_cdf(z), np.where(margin > 0.0, 1.0, 0.0))
        margin = best - lam - mean
        z = margin / np.where(sd > 0.0, sd, 1.0)
        ei = margin * normal_cdf(z) + sd * normal_pdf(z)
        return np.where(sd > 0.0, ei, np.where(margin > 0.0, margin, 0.0))


def cv_lambda(mu_s: float, var_s: float, mean_var: float, f_best: float):
    """contextual_variance_lambda (acquisition.hpp:73-83); None -> fallback."""
    if not (f_best > 0.0) or not (mu_s > 0.0) or not (var_s > 0.0):
        return None
    lam = (mean_var * f_best / mu_s) / var_s
    return lam if lam > 0.0 else 0.0


def best_candidate(scores) -> int:
    """best_candidate's rule (portfolio.hpp:32-61) over precomputed scores:
    the first candidate unconditionally, then strictly greater non-NaN
    scores (lowest position on ties)."""
    scores = np.asarray(scores)
    if len(scores) == 0:
        raise ValueError("acquisition: no candidates remaining")
    if np.isnan(scores[0]):
        return 0
    finite = np.where(np.isnan(scores), -np.inf, scores)
    return int(np.argmax(finite))  # the first position attaining the maximum


def eps_optimal(scores, pick: int, eps: float = 1e-9) -> bool:
    """SURVEY.md §8(c) parity protocol: `pick` is epsilon-optimal under the
    oracle's scores: score(pick) >= best - eps * max(|best|, 1)."""
    scores = np.asarray(scores)
    finite = scores[~np.isnan(scores)]
    if len(finite) == 0:
        return True
    best = float(np.max(finite))
    s = float(scores[pick])
    return s == s and s >= best - eps * max(abs(best), 1.0)
