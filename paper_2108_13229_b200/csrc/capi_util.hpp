// Shared helpers of the extern "C" layer (capi.cu, dist.cu): the opaque
// handle structs, the exception -> return-code guard, argument conversion.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstring>
#include <new>
#include <string>

#include "sdg.h"
#include "setup.hpp"
#include "solver.hpp"

struct sdg_context {
    sdg::CtxPtr p;
};
struct sdg_matrix {
    sdg::MatrixPtr p;
};
struct sdg_precond {
    sdg::PrecondPtr p;
};
struct sdg_lu {
    sdg::CtxPtr ctx;
    sdg::CoarseSolver solver;
    sdg::DevBuf<double> b, x;
};
struct sdg_host_hierarchy {
    std::vector<sdg::HostLevel> levels;
};

namespace sdg_capi {

inline thread_local std::string g_last_error;

template <class F>
inline int guard(F&& f) {
    try {
        f();
        return SDG_OK;
    } catch (const sdg::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return SDG_ENOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SDG_EINVAL;
    }
}

inline void need(const void* p, const char* what) {
    if (!p) sdg::fail(SDG_EINVAL, std::string(what) + ": null argument");
}

inline sdg::HostCsr make_csr(int n_rows, int n_cols, const int* rp, const int* ci, const double* v) {
    if (n_rows < 0 || n_cols < 0) sdg::fail(SDG_EDIM, "SparseMatrix: negative dimension");
    need(rp, "matrix row offsets");
    sdg::HostCsr h(n_rows, n_cols);
    h.rp.assign(rp, rp + n_rows + 1);
    const int nnz = rp[n_rows];
    if (nnz < 0) sdg::fail(SDG_EDIM, "SparseMatrix: negative nnz");
    if (nnz) {
        need(ci, "matrix columns");
        need(v, "matrix values");
    }
    h.ci.assign(ci, ci + nnz);
    h.v.assign(v, v + nnz);
    return h;
}

inline sdg::AmgOpts amg_opts(const sdg_amg_options* o, int n_rows) {
    sdg::AmgOpts a;
    if (!o) return a;
    a.max_levels = o->max_levels;
    a.theta = o->strength_theta;
    a.coarse_threshold = o->coarse_threshold;
    if (o->components) a.components.assign(o->components, o->components + n_rows);
    return a;
}

inline sdg::Restart restart_from(const sdg_restart* c) {
    sdg::Restart r;
    if (!c) return r;
    r.m_init = c->m_init;
    r.m_min = c->m_min;
    r.m_step = c->m_step;
    r.m_max = c->m_max;
    r.current_m = c->current_m;
    r.previous_rate = c->previous_rate;
    r.has_rate_sample = c->has_rate_sample != 0;
    r.alpha_p = c->alpha_p;
    r.alpha_d = c->alpha_d;
    r.stall_threshold = c->stall_threshold;
    return r;
}

inline void fill_report(const sdg::SolveOut& o, double wall, int64_t apps, sdg_report* rep) {
    if (!rep) return;
    rep->iterations = o.iterations;
    rep->converged = o.converged ? 1 : 0;
    rep->final_residual = o.final_residual;
    rep->wall_time = wall;
    rep->device_ms = o.device_ms;
    rep->precond_applications = apps;
    rep->breakdown = o.breakdown ? 1 : 0;
    rep->history_length = static_cast<int>(o.history.size());
    if (rep->residual_history && rep->history_capacity > 0) {
        const int k = std::min(rep->history_capacity, rep->history_length);
        std::memcpy(rep->residual_history, o.history.data(), sizeof(double) * k);
    }
}

inline double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace sdg_capi
