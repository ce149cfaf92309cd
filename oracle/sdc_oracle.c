/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.  Plain-C restatement of the reference's
 * preconditioned Krylov path; see sdc_oracle.h.  The arithmetic order of each
 * loop follows the cited reference lines (gcc -O2 without -mfma, i.e. no FMA
 * contraction, like the reference's own Release build), so results can be
 * compared with the compiled reference bit for bit.
 */
#include "sdc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- sparse kernels: sparse.cpp:81-108, 208-222 ----------------------------- */

void orc_spmv(const orc_csr* a, const double* x, double* y) {
    for (int i = 0; i < a->n_rows; ++i) {
        double acc = 0.0;
        for (int k = a->rp[i]; k < a->rp[i + 1]; ++k) acc += a->v[k] * x[a->ci[k]];
        y[i] = acc;
    }
}

void orc_spmv_add(const orc_csr* a, const double* x, double* y, double alpha) {
    for (int i = 0; i < a->n_rows; ++i) {
        double acc = 0.0;
        for (int k = a->rp[i]; k < a->rp[i + 1]; ++k) acc += a->v[k] * x[a->ci[k]];
        y[i] += alpha * acc;
    }
}

/* Checker-side experiment knob (scripts/ref_dot_experiment.py), default 0 =
 * the reference's sequential sum (sparse.cpp:208-212; every pin of this file
 * runs in that mode).  Mode 1 sums pairwise (blocks of 128, then a binary
 * tree), the error behaviour of a GPU tree reduction: it shows how far the
 * reference's own BiCGSTAB iteration counts depend on the rounding error of
 * its dot products. */
static int g_dot_mode = 0;
void orc_set_dot_mode(int mode) { g_dot_mode = mode; }

static double dot_pairwise(int n, const double* x, const double* y) {
    if (n <= 128) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += x[i] * y[i];
        return s;
    }
    const int h = (n / 2 + 127) / 128 * 128;
    return dot_pairwise(h, x, y) + dot_pairwise(n - h, x + h, y + h);
}

double orc_dot(int n, const double* x, const double* y) {
    if (g_dot_mode == 1) return dot_pairwise(n, x, y);
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
}

double orc_norm2(int n, const double* x) { return sqrt(orc_dot(n, x, x)); }

static void axpy(int n, double alpha, const double* x, double* y) {
    for (int i = 0; i < n; ++i) y[i] += alpha * x[i];
}

static void scale(int n, double* x, double alpha) {
    for (int i = 0; i < n; ++i) x[i] *= alpha;
}

/* ---- Gauss-Seidel: precond.cpp:92-108 --------------------------------------- */

int orc_sor_sweep(const orc_csr* a, double* z, const double* r, double omega) {
    for (int i = 0; i < a->n_rows; ++i) {
        double s = r[i], d = 0.0;
        for (int k = a->rp[i]; k < a->rp[i + 1]; ++k) {
            const int j = a->ci[k];
            if (j == i)
                d = a->v[k];
            else
                s -= a->v[k] * z[j];
        }
        if (d == 0.0) return i;
        z[i] = (1.0 - omega) * z[i] + omega * s / d;
    }
    return -1;
}

/* ---- coarse triangular solves: lu.cpp:178-203 ------------------------------- */

void orc_lu_solve(int n, const orc_csr* lo, const orc_csr* up, const int* perm, const double* b,
                  double* y) {
    for (int k = 0; k < n; ++k) y[k] = b[perm[k]];
    for (int i = 0; i < n; ++i) {
        double s = y[i];
        for (int p = lo->rp[i]; p < lo->rp[i + 1]; ++p) s -= lo->v[p] * y[lo->ci[p]];
        y[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
        const int first = up->rp[i];
        double s = y[i];
        for (int p = first + 1; p < up->rp[i + 1]; ++p) s -= up->v[p] * y[up->ci[p]];
        y[i] = s / up->v[first]; /* the diagonal leads each sorted U row */
    }
}

/* ---- aggregation: precond.cpp:122-175 --------------------------------------- */

int orc_aggregate(const orc_csr* a, double theta, const int* comps, int* agg) {
    const int n = a->n_rows;
    double* dg = (double*)calloc((size_t)n + 1, sizeof(double));
    for (int i = 0; i < n; ++i)
        for (int k = a->rp[i]; k < a->rp[i + 1]; ++k)
            if (a->ci[k] == i) dg[i] = a->v[k];
#define STRONG(i, k)                                                                   \
    (a->ci[k] != (i) && (!comps || comps[i] == comps[a->ci[k]]) &&                     \
     fabs(a->v[k]) >= theta * sqrt(fabs(dg[i] * dg[a->ci[k]])))
    for (int i = 0; i < n; ++i) agg[i] = -1;
    int next = 0;
    for (int i = 0; i < n; ++i) {
        if (agg[i] >= 0) continue;
        int taken = 0;
        for (int k = a->rp[i]; k < a->rp[i + 1]; ++k)
            if (STRONG(i, k) && agg[a->ci[k]] >= 0) taken = 1;
        if (taken) continue;
        agg[i] = next;
        for (int k = a->rp[i]; k < a->rp[i + 1]; ++k)
            if (STRONG(i, k) && agg[a->ci[k]] < 0) agg[a->ci[k]] = next;
        ++next;
    }
    for (int i = 0; i < n; ++i) {
        if (agg[i] >= 0) continue;
        int best = -1;
        double best_w = -1.0;
        for (int k = a->rp[i]; k < a->rp[i + 1]; ++k) {
            const int j = a->ci[k];
            if (j == i || agg[j] < 0) continue;
            const double w = fabs(a->v[k]);
            if (STRONG(i, k) && w > best_w) {
                best_w = w;
                best = agg[j];
            }
        }
        agg[i] = best >= 0 ? best : next++;
    }
#undef STRONG
    free(dg);
    return next;
}

/* ---- V(1,1) cycle: precond.cpp:233-259 -------------------------------------- */

static int vcycle_rec(const orc_hierarchy* h, int lev, const double* r, double* z) {
    const orc_level* L = &h->levels[lev];
    const int n = L->a.n_rows;
    if (lev + 1 == h->n_levels) {
        orc_lu_solve(n, &h->lower, &h->upper, h->perm, r, z);
        return 0;
    }
    for (int i = 0; i < n; ++i) z[i] = 0.0;
    int bad = orc_sor_sweep(&L->a, z, r, 1.0);
    if (bad >= 0) return bad + 1;
    double* res = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(res, r, sizeof(double) * (size_t)n);
    orc_spmv_add(&L->a, z, res, -1.0);
    double* rc = (double*)calloc((size_t)L->n_coarse + 1, sizeof(double));
    double* zc = (double*)calloc((size_t)L->n_coarse + 1, sizeof(double));
    for (int i = 0; i < n; ++i) rc[L->agg[i]] += res[i];
    int rc_err = vcycle_rec(h, lev + 1, rc, zc);
    if (!rc_err) {
        for (int i = 0; i < n; ++i) z[i] += zc[L->agg[i]];
        bad = orc_sor_sweep(&L->a, z, r, 1.0);
        if (bad >= 0) rc_err = bad + 1;
    }
    free(res);
    free(rc);
    free(zc);
    return rc_err;
}

int orc_vcycle(const orc_hierarchy* h, const double* r, double* z) { return vcycle_rec(h, 0, r, z); }

/* ---- Uzawa / td_bgs: precond.cpp:289-299, 339-345 ---------------------------- */

int orc_uzawa_apply(const orc_hierarchy* v, const orc_csr* c, double omega, const double* r,
                    double* z) {
    const int n_v = v->levels[0].a.n_rows, n_p = c->n_rows;
    int err = orc_vcycle(v, r, z);
    if (err) return err;
    double* cz = (double*)malloc(sizeof(double) * ((size_t)n_p + 1));
    orc_spmv(c, z, cz);
    for (int i = 0; i < n_p; ++i) z[n_v + i] = omega * (cz[i] - r[n_v + i]);
    free(cz);
    return 0;
}

int orc_td_bgs_apply(const orc_hierarchy* v, const orc_csr* c, double omega, const orc_csr* c_prime,
                     const orc_hierarchy* d, int n_v, int n_pff, int n_ppm, const double* r,
                     double* z) {
    const int n_ff = n_v + n_pff;
    int err = orc_uzawa_apply(v, c, omega, r, z);
    if (err) return err;
    double* rp = (double*)malloc(sizeof(double) * ((size_t)n_ppm + 1));
    memcpy(rp, r + n_ff, sizeof(double) * (size_t)n_ppm);
    orc_spmv_add(c_prime, z, rp, -1.0);
    err = orc_vcycle(d, rp, z + n_ff);
    free(rp);
    return err;
}

void orc_cb_spmv(void* user, const double* x, double* y) { orc_spmv((const orc_csr*)user, x, y); }

void orc_cb_td_bgs(void* user, const double* r, double* z) {
    const orc_td_bundle* b = (const orc_td_bundle*)user;
    orc_td_bgs_apply(b->v, b->c, b->omega, b->c_prime, b->d, b->n_v, b->n_pff, b->n_ppm, r, z);
}

void orc_cb_vcycle(void* user, const double* r, double* z) {
    orc_vcycle((const orc_hierarchy*)user, r, z);
}

/* ---- restart controller: krylov.cpp:37-45 ----------------------------------- */

static double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }
static int clampi(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }

void orc_restart_update(orc_restart* c, double rate) {
    rate = clampd(rate, -16.0, 16.0);
    const double deriv = c->has_rate_sample ? (rate - c->previous_rate) : 0.0;
    int delta = (int)floor(c->alpha_p * rate + c->alpha_d * deriv);
    if (rate > -c->stall_threshold && delta < c->m_step) delta = c->m_step;
    c->current_m = clampi(c->current_m + delta, c->m_min, c->m_max);
    c->previous_rate = rate;
    c->has_rate_sample = 1;
}

static void hist_push(orc_report* rep, double v) {
    if (rep->history && rep->length < rep->capacity) rep->history[rep->length] = v;
    rep->length++;
}

static void precond_or_copy(int n, orc_apply_fn pre, void* user, const double* r, double* z) {
    if (pre)
        pre(user, r, z);
    else
        memcpy(z, r, sizeof(double) * (size_t)n);
}

/* ---- PD-GMRES: krylov.cpp:47-184 -------------------------------------------- */

int orc_pd_gmres(int n, orc_apply_fn op, void* op_user, orc_apply_fn pre, void* pre_user,
                 const double* b, double tol_abs, int max_restarts, orc_restart ctrl, double* x,
                 orc_report* rep) {
    rep->iterations = 0;
    rep->converged = 0;
    rep->length = 0;
    for (int i = 0; i < n; ++i) x[i] = 0.0;
    const size_t nb = sizeof(double) * (size_t)n;
    double* r = (double*)malloc(nb);
    double* z = (double*)malloc(nb);
    double* w = (double*)malloc(nb);
    double* best_x = (double*)malloc(nb);
    memcpy(r, b, nb);
    double res = orc_norm2(n, r);
    hist_push(rep, res);
    int status = 0;
    if (res <= tol_abs) {
        rep->converged = 1;
        rep->final_residual = res;
        goto done;
    }
    double prev_cycle = res, best_res = res;
    memcpy(best_x, x, nb);
    int trust = 1;
    for (int cycle = 0; cycle < max_restarts; ++cycle) {
        const int m = ctrl.current_m;
        double* V = (double*)malloc(nb * (size_t)(m + 1));
        double* H = (double*)calloc((size_t)(m + 1) * (size_t)m, sizeof(double));
        double* g = (double*)calloc((size_t)m + 1, sizeof(double));
        double* cs = (double*)calloc((size_t)m + 1, sizeof(double));
        double* sn = (double*)calloc((size_t)m + 1, sizeof(double));
#define HH(i, j) H[(size_t)(j) * (size_t)(m + 1) + (size_t)(i)]
        const double beta = orc_norm2(n, r);
        g[0] = beta;
        memcpy(V, r, nb);
        scale(n, V, 1.0 / beta);
        int used = 0, exhausted = 0;
        for (int i = 0; i < m; ++i) {
            double* vi = V + (size_t)i * n;
            precond_or_copy(n, pre, pre_user, vi, z);
            op(op_user, z, w);
            for (int pass = 0; pass < 2; ++pass)
                for (int k = 0; k <= i; ++k) {
                    const double cpk = orc_dot(n, w, V + (size_t)k * n);
                    HH(k, i) += cpk;
                    axpy(n, -cpk, V + (size_t)k * n, w);
                }
            const double wn = orc_norm2(n, w);
            HH(i + 1, i) = wn;
            if (wn > 0.0) {
                double* vn = V + (size_t)(i + 1) * n;
                memcpy(vn, w, nb);
                scale(n, vn, 1.0 / wn);
            }
            for (int k = 0; k < i; ++k) {
                const double t0 = cs[k] * HH(k, i) + sn[k] * HH(k + 1, i);
                const double t1 = -sn[k] * HH(k, i) + cs[k] * HH(k + 1, i);
                HH(k, i) = t0;
                HH(k + 1, i) = t1;
            }
            const double den = hypot(HH(i, i), HH(i + 1, i));
            if (den == 0.0) {
                status = 2;
                break;
            }
            cs[i] = HH(i, i) / den;
            sn[i] = HH(i + 1, i) / den;
            HH(i, i) = den;
            HH(i + 1, i) = 0.0;
            g[i + 1] = -sn[i] * g[i];
            g[i] = cs[i] * g[i];
            rep->iterations++;
            used++;
            const double est = fabs(g[i + 1]);
            hist_push(rep, est);
            if (trust && est <= tol_abs) break;
            if (wn == 0.0) {
                exhausted = 1;
                break;
            }
        }
        double* y = (double*)calloc((size_t)used + 1, sizeof(double));
        for (int i = used - 1; i >= 0 && !status; --i) {
            double s = g[i];
            for (int j = i + 1; j < used; ++j) s -= HH(i, j) * y[j];
            if (HH(i, i) == 0.0) status = 2;
            else y[i] = s / HH(i, i);
        }
#undef HH
        if (!status) {
            for (int i = 0; i < n; ++i) w[i] = 0.0;
            for (int i = 0; i < used; ++i) axpy(n, y[i], V + (size_t)i * n, w);
            precond_or_copy(n, pre, pre_user, w, z);
            for (int i = 0; i < n; ++i) x[i] += z[i];
            op(op_user, x, r);
            for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
            res = orc_norm2(n, r);
            if (res < best_res) {
                best_res = res;
                memcpy(best_x, x, nb);
            }
            if (trust && used < m && res > tol_abs) trust = 0;
            const double rate = log10((res > 1e-300 ? res : 1e-300) / (prev_cycle > 1e-300 ? prev_cycle : 1e-300));
            orc_restart_update(&ctrl, rate);
            prev_cycle = res;
        }
        free(y);
        free(V);
        free(H);
        free(g);
        free(cs);
        free(sn);
        if (status) goto done;
        if (res <= tol_abs || exhausted) break;
    }
    if (best_res < res) {
        memcpy(x, best_x, nb);
        res = best_res;
    }
    hist_push(rep, res);
    rep->final_residual = res;
    rep->converged = res <= tol_abs;
done:
    free(r);
    free(z);
    free(w);
    free(best_x);
    return status;
}

/* ---- BiCGSTAB: krylov.cpp:186-292 ------------------------------------------- */

static void true_residual(int n, orc_apply_fn op, void* user, const double* b, const double* x,
                          double* out) {
    op(user, x, out);
    for (int i = 0; i < n; ++i) out[i] = b[i] - out[i];
}

int orc_bicgstab(int n, orc_apply_fn op, void* op_user, orc_apply_fn pre, void* pre_user,
                 const double* b, double tol_abs, int max_iters, double* x, orc_report* rep) {
    rep->iterations = 0;
    rep->converged = 0;
    rep->length = 0;
    const size_t nb = sizeof(double) * (size_t)n;
    for (int i = 0; i < n; ++i) x[i] = 0.0;
    double* r = (double*)malloc(nb);
    memcpy(r, b, nb);
    double res = orc_norm2(n, r);
    hist_push(rep, res);
    if (res <= tol_abs) {
        rep->converged = 1;
        rep->final_residual = res;
        free(r);
        return 0;
    }
    double* rhat = (double*)malloc(nb);
    double* p = (double*)calloc((size_t)n, sizeof(double));
    double* vv = (double*)calloc((size_t)n, sizeof(double));
    double* s = (double*)malloc(nb);
    double* phat = (double*)malloc(nb);
    double* shat = (double*)malloc(nb);
    double* t = (double*)malloc(nb);
    double* rt = (double*)malloc(nb);
    memcpy(rhat, r, nb);
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    int restarts = 0, replacements = 0, done = 0, status = 0;

#define RESET_DIRECTIONS()                         \
    do {                                           \
        memcpy(rhat, r, nb);                       \
        memset(p, 0, nb);                          \
        memset(vv, 0, nb);                         \
        rho = alpha = omega = 1.0;                 \
    } while (0)
#define HARD_RESTART()                                        \
    do {                                                      \
        if (++restarts > 1) {                                 \
            status = 3;                                       \
            goto out;                                         \
        }                                                     \
        true_residual(n, op, op_user, b, x, r);               \
        RESET_DIRECTIONS();                                   \
    } while (0)

    for (int iter = 0; iter < max_iters && !done; ++iter) {
        const double rho_new = orc_dot(n, rhat, r);
        if (fabs(rho_new) < 1e-300) {
            HARD_RESTART();
            continue;
        }
        const double beta = (rho_new / rho) * (alpha / omega);
        for (int i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - omega * vv[i]);
        precond_or_copy(n, pre, pre_user, p, phat);
        op(op_user, phat, vv);
        const double rv = orc_dot(n, rhat, vv);
        if (fabs(rv) < 1e-300) {
            HARD_RESTART();
            continue;
        }
        alpha = rho_new / rv;
        for (int i = 0; i < n; ++i) s[i] = r[i] - alpha * vv[i];
        rep->iterations++;
        const double snorm = orc_norm2(n, s);
        int check = 0;
        if (snorm <= tol_abs) {
            axpy(n, alpha, phat, x);
            hist_push(rep, snorm);
            check = 1;
        } else {
            precond_or_copy(n, pre, pre_user, s, shat);
            op(op_user, shat, t);
            const double tt = orc_dot(n, t, t);
            if (tt == 0.0) {
                HARD_RESTART();
                continue;
            }
            omega = orc_dot(n, t, s) / tt;
            if (fabs(omega) < 1e-300) {
                HARD_RESTART();
                continue;
            }
            for (int i = 0; i < n; ++i) x[i] += alpha * phat[i] + omega * shat[i];
            for (int i = 0; i < n; ++i) r[i] = s[i] - omega * t[i];
            rho = rho_new;
            res = orc_norm2(n, r);
            hist_push(rep, res);
            check = res <= tol_abs;
        }
        if (check) {
            /* confirmed(): krylov.cpp:225-239 */
            true_residual(n, op, op_user, b, x, rt);
            const double tn = orc_norm2(n, rt);
            if (tn <= tol_abs) break;
            if (replacements++ < 3) {
                memcpy(r, rt, nb);
                RESET_DIRECTIONS();
            } else {
                done = 1;
            }
        }
    }
    true_residual(n, op, op_user, b, x, rt);
    rep->final_residual = orc_norm2(n, rt);
    hist_push(rep, rep->final_residual);
    rep->converged = rep->final_residual <= tol_abs;
out:
#undef HARD_RESTART
#undef RESET_DIRECTIONS
    free(r);
    free(rhat);
    free(p);
    free(vv);
    free(s);
    free(phat);
    free(shat);
    free(t);
    free(rt);
    return status;
}

/* ---- std::mt19937 / uniform_real_distribution<double> (libstdc++) ------------- */

typedef struct {
    uint32_t mt[624];
    int idx;
} mt19937;

static void mt_seed(mt19937* g, uint32_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 624; ++i)
        g->mt[i] = 1812433253u * (g->mt[i - 1] ^ (g->mt[i - 1] >> 30)) + (uint32_t)i;
    g->idx = 624;
}

static uint32_t mt_next(mt19937* g) {
    if (g->idx >= 624) {
        for (int i = 0; i < 624; ++i) {
            const uint32_t y = (g->mt[i] & 0x80000000u) | (g->mt[(i + 1) % 624] & 0x7fffffffu);
            g->mt[i] = g->mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        g->idx = 0;
    }
    uint32_t y = g->mt[g->idx++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

/* generate_canonical<double, 53> over a 32-bit engine: two draws */
static double mt_canonical(mt19937* g) {
    double sum = 0.0, tmp = 1.0;
    for (int k = 0; k < 2; ++k) {
        sum += (double)mt_next(g) * tmp;
        tmp *= 4294967296.0;
    }
    double ret = sum / tmp;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret;
}

static double mt_uniform(mt19937* g, double a, double b) { return mt_canonical(g) * (b - a) + a; }

void orc_random_vector(int n, unsigned seed, double* out) {
    mt19937 g;
    mt_seed(&g, seed);
    for (int i = 0; i < n; ++i) out[i] = mt_uniform(&g, -1.0, 1.0);
}

/* ---- power iteration: krylov.cpp:307-339 ------------------------------------ */

double orc_power_iteration(int n, orc_apply_fn op, void* user, double tol_rel, int max_iters,
                           unsigned seed, int* iterations, int* converged) {
    double* x = (double*)malloc(sizeof(double) * (size_t)n);
    double* y = (double*)malloc(sizeof(double) * (size_t)n);
    orc_random_vector(n, seed, x);
    double xn = orc_norm2(n, x);
    if (xn == 0.0) x[0] = xn = 1.0;
    scale(n, x, 1.0 / xn);
    double value = 0.0, prev = 0.0;
    *iterations = 0;
    *converged = 0;
    for (int k = 0; k < max_iters; ++k) {
        op(user, x, y);
        const double lambda = orc_dot(n, x, y);
        value = lambda;
        *iterations = k + 1;
        if (k > 0 && fabs(lambda - prev) <= tol_rel * fabs(lambda)) {
            *converged = 1;
            break;
        }
        prev = lambda;
        const double yn = orc_norm2(n, y);
        if (yn == 0.0) {
            value = 0.0;
            *converged = 1;
            break;
        }
        for (int i = 0; i < n; ++i) x[i] = y[i] / yn;
    }
    free(x);
    free(y);
    return value;
}
