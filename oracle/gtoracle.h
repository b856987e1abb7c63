/*
 * gtoracle.h — CPU oracle for the BO surrogate pass. TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference algorithm (citations into
 * /root/reference/proj/include/gridtune/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker — never
 * as the product path.  Pinned by tests/test_oracle_golden.py against golden
 * vectors produced by the unmodified reference (oracle/_ref/ref_tool, see
 * tests/golden/make_golden.py) and against the reference's known-answer tests.
 */
#ifndef GTORACLE_H_
#define GTORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Matern closed forms, gp.hpp:40-55 (nu: 0 = 1/2, 1 = 3/2, 2 = 5/2). */
double gto_matern(int nu, double lengthscale, double s2, double r);

/* GpModel::fit, gp.hpp:81-135.  X n x d row-major.  Outputs: L (n x n row-major
 * lower), alpha (n), scalars[0..2] = y_mean, y_std, jitter.  Returns 0, or -1
 * for bad input, or -2 when the factorisation fails after 6 jitter doublings. */
int gto_gp_fit(int nu, double lengthscale, double s2, const double* X, const double* y, int n,
               int d, double noise, double jitter, double* L, double* alpha, double* scalars);

/* GpModel::predict, gp.hpp:150-193 (expansion-form distances, sequential
 * forward substitution, max(.,0) clamp).  Xstar m x d row-major. */
void gto_gp_predict(int nu, double lengthscale, double s2, const double* X, int n, int d,
                    const double* L, const double* alpha, const double* Xstar, int64_t m,
                    double* mean, double* var);

/* acquisition.hpp:12-42 */
double gto_acq_pi(double mean, double sd, double best_std, double lambda);
double gto_acq_ei(double mean, double sd, double best_std, double lambda);
double gto_acq_lcb(double mean, double sd, double lambda);

/* contextual_variance_lambda, acquisition.hpp:73-83: returns 1 and *lambda, or
 * 0 (nullopt). */
int gto_cv_lambda(double initial_sample_mean, double initial_mean_variance, double mean_variance,
                  double f_best_raw, double* lambda);

/* best_candidate, portfolio.hpp:32-61.  af: 0 ei, 1 poi, 2 lcb.  Returns the
 * position or -1 when every candidate is excluded. */
int64_t gto_best_candidate(int af, const double* means, const double* stds, int64_t n,
                           double best_std, double lambda, const uint8_t* excluded,
                           double* score_out);

/* Sequential arithmetic mean (std::accumulate / size, strategies.hpp:406-407). */
double gto_mean(const double* v, int64_t n);

/* Whole-surrogate reference step for one BO iteration over candidates
 * (strategies.hpp:366-436): predict every unvisited candidate, lambda,
 * best_candidate for each AF in af_mask.  Used by the CPU baseline. */
int gto_iteration(int nu, double lengthscale, double s2, const double* coords, int64_t N, int d,
                  const int64_t* train_pos, const double* y, int n, double noise, double jitter,
                  const uint8_t* visited, uint32_t af_mask, int lambda_mode, double lambda_const,
                  double cv_mu_s, double cv_var_s, double f_best_raw, int64_t* pick_out,
                  double* lambda_out);

#ifdef __cplusplus
}
#endif

#endif
