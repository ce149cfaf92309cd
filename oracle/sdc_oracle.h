/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference
 * hot path (arXiv 2108.13229 reference, /root/reference/proj/core/src).
 * Used only by tests/ (and bench.py's CPU leg) as a checker; the product
 * (paper_2108_13229_b200/) never links it.  Every function cites the
 * reference code it restates; it is pinned against the compiled reference
 * (oracle/_ref/libsdcore_ref.so) by tests/test_oracle.py, bit for bit where
 * the arithmetic order is the same.
 */
#ifndef SDC_ORACLE_H
#define SDC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int n_rows, n_cols;
    const int* rp;
    const int* ci;
    const double* v;
} orc_csr;

/* sparse.cpp:81-90 */
void orc_spmv(const orc_csr* a, const double* x, double* y);
/* sparse.cpp:98-108 */
void orc_spmv_add(const orc_csr* a, const double* x, double* y, double alpha);
/* sparse.cpp:208-222 */
void orc_set_dot_mode(int mode);  /* experiment knob, see sdc_oracle.c */
double orc_dot(int n, const double* x, const double* y);
double orc_norm2(int n, const double* x);
/* precond.cpp:92-108; returns the failing row or -1 */
int orc_sor_sweep(const orc_csr* a, double* z, const double* r, double omega);
/* lu.cpp:178-203 (factors in the reference's CSR layout) */
void orc_lu_solve(int n, const orc_csr* lower, const orc_csr* upper, const int* perm,
                  const double* b, double* y);

/* precond.cpp:122-175; returns the number of aggregates */
int orc_aggregate(const orc_csr* a, double theta, const int* comps, int* agg);

/* One hierarchy level (precond.hpp:77-95) and the coarse LU. */
typedef struct {
    orc_csr a;
    const int* agg; /* NULL on the coarsest level */
    int n_coarse;
} orc_level;

typedef struct {
    int n_levels;
    const orc_level* levels;
    orc_csr lower, upper; /* coarse LU (lu.hpp:20-27) */
    const int* perm;
} orc_hierarchy;

/* precond.cpp:233-259; returns 0 or the failing GS row + 1 */
int orc_vcycle(const orc_hierarchy* h, const double* r, double* z);

/* precond.cpp:289-299: z_v = Vcycle(r_v); z_p = omega (C z_v - r_p) */
int orc_uzawa_apply(const orc_hierarchy* v, const orc_csr* c, double omega, const double* r,
                    double* z);
/* precond.cpp:339-345 (td_bgs) with Uzawa(AMG_V) first and AMG_D' second */
int orc_td_bgs_apply(const orc_hierarchy* v, const orc_csr* c, double omega, const orc_csr* c_prime,
                     const orc_hierarchy* d, int n_v, int n_pff, int n_ppm, const double* r,
                     double* z);

/* generic operator / preconditioner callbacks */
typedef void (*orc_apply_fn)(void* user, const double* x, double* y);

typedef struct {
    int m_init, m_min, m_step, m_max, current_m;
    double previous_rate;
    int has_rate_sample;
    double alpha_p, alpha_d, stall_threshold;
} orc_restart;

typedef struct {
    int iterations;
    int converged;
    double final_residual;
    double* history; /* capacity entries, may be NULL */
    int capacity;
    int length;
} orc_report;

/* krylov.cpp:37-45 */
void orc_restart_update(orc_restart* c, double rate);
/* krylov.cpp:47-184; returns 0, or 2 on a singular Hessenberg block */
int orc_pd_gmres(int n, orc_apply_fn op, void* op_user, orc_apply_fn pre, void* pre_user,
                 const double* b, double tol_abs, int max_restarts, orc_restart ctrl, double* x,
                 orc_report* rep);
/* krylov.cpp:186-292; returns 0, or 3 on repeated breakdown */
int orc_bicgstab(int n, orc_apply_fn op, void* op_user, orc_apply_fn pre, void* pre_user,
                 const double* b, double tol_abs, int max_iters, double* x, orc_report* rep);
/* krylov.cpp:307-339 (std::mt19937 + uniform_real_distribution restated) */
double orc_power_iteration(int n, orc_apply_fn op, void* user, double tol_rel, int max_iters,
                           unsigned seed, int* iterations, int* converged);

/* libstdc++'s std::mt19937 + uniform_real_distribution<double>(-1, 1), as
 * used by tests/support/dense_oracles.hpp:202-208 (random_vector). */
void orc_random_vector(int n, unsigned seed, double* out);

/* convenience callbacks: user = const orc_csr* / a td bundle */
void orc_cb_spmv(void* user, const double* x, double* y);

typedef struct {
    const orc_hierarchy* v;
    const orc_csr* c;
    double omega;
    const orc_csr* c_prime;
    const orc_hierarchy* d;
    int n_v, n_pff, n_ppm;
} orc_td_bundle;
void orc_cb_td_bgs(void* user, const double* r, double* z);
void orc_cb_vcycle(void* user, const double* r, double* z); /* user = orc_hierarchy* */

#ifdef __cplusplus
}
#endif

#endif
