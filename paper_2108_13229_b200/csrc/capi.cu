// extern "C" boundary of libsdgpu.so (include/sdg.h).
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <new>
#include <string>

#include "coarse.hpp"
#include "power.cuh"
#include "sdg.h"
#include "setup.hpp"
#include "solver.hpp"

#include "capi_util.hpp"

using namespace sdg_capi;

namespace {

sdg::AmgPrecond* as_amg(const sdg::PrecondPtr& p) { return dynamic_cast<sdg::AmgPrecond*>(p.get()); }

}  // namespace

extern "C" {

void sdg_restart_defaults(sdg_restart* c) {
    if (!c) return;
    sdg::Restart r;
    c->m_init = r.m_init;
    c->m_min = r.m_min;
    c->m_step = r.m_step;
    c->m_max = r.m_max;
    c->current_m = r.current_m;
    c->previous_rate = r.previous_rate;
    c->has_rate_sample = 0;
    c->alpha_p = r.alpha_p;
    c->alpha_d = r.alpha_d;
    c->stall_threshold = r.stall_threshold;
}

void sdg_amg_defaults(sdg_amg_options* o) {
    if (!o) return;
    o->max_levels = 3;
    o->strength_theta = 0.08;
    o->coarse_threshold = 100;
    o->components = nullptr;
}

void sdg_uzawa_defaults(sdg_uzawa_options* o) {
    if (!o) return;
    sdg_amg_defaults(&o->amg);
    o->power_tol_rel = 1e-3;
    o->power_max_iters = 200;
    o->power_seed = 1729;
    o->omega_override = std::numeric_limits<double>::quiet_NaN();
}

const char* sdg_last_error(void) { return g_last_error.c_str(); }
const char* sdg_version(void) { return "sdgpu 0.1 (sm_100a, fp64)"; }

// ---- context ---------------------------------------------------------------
int sdg_context_create(int device, sdg_context** out) {
    return guard([&] {
        need(out, "sdg_context_create");
        *out = new sdg_context{std::make_shared<sdg::Context>(device)};
    });
}
int sdg_context_destroy(sdg_context* ctx) {
    return guard([&] { delete ctx; });
}
int sdg_context_synchronize(sdg_context* ctx) {
    return guard([&] {
        need(ctx, "sdg_context_synchronize");
        ctx->p->sync();
    });
}
void* sdg_context_stream(sdg_context* ctx) { return ctx ? (void*)ctx->p->stream : nullptr; }
int64_t sdg_context_launches(sdg_context* ctx) { return ctx ? ctx->p->launches.load() : 0; }

int sdg_context_set_profiling(sdg_context* ctx, int enable) {
    return guard([&] {
        need(ctx, "sdg_context_set_profiling");
        auto& c = *ctx->p;
        c.drain_profile();
        for (int f = 0; f < sdg::PF_COUNT; ++f) {
            c.prof_launches[f] = 0;
            c.prof_ms[f] = 0.0;
            c.prof_bytes[f] = 0.0;
        }
        c.profiling = enable != 0;
    });
}

int sdg_context_profile(sdg_context* ctx, int family, int64_t* launches, double* total_ms,
                        double* total_bytes) {
    return guard([&] {
        need(ctx, "sdg_context_profile");
        if (family < 0 || family >= sdg::PF_COUNT) sdg::fail(SDG_EINVAL, "sdg_context_profile: bad family");
        auto& c = *ctx->p;
        c.drain_profile();
        if (launches) *launches = c.prof_launches[family];
        if (total_ms) *total_ms = c.prof_ms[family];
        if (total_bytes) *total_bytes = c.prof_bytes[family];
    });
}

extern "C" int sdg_debug_walk_timeline(unsigned long long* out, int max) { return sdg::walk_timeline(out, max); }
extern "C" double sdg_lattice_check_host(int n, const int* rowptr, const int* col, const double* val,
                                         const double* b) {
    try {
        sdg::HostCsr a(n, n);
        a.rp.assign(rowptr, rowptr + n + 1);
        a.ci.assign(col, col + rowptr[n]);
        a.v.assign(val, val + rowptr[n]);
        return sdg::lattice_check_host(a, b);
    } catch (...) {
        return -2.0;
    }
}
extern "C" int sdg_debug_lattice_sweep(sdg_context* ctx, int n, const int* rowptr, const int* col,
                                       const double* val, const double* b, double* z_host, double* z_dev_out,
                                       int repeats) {
    return guard([&] {
        sdg::HostCsr a(n, n);
        a.rp.assign(rowptr, rowptr + n + 1);
        a.ci.assign(col, col + rowptr[n]);
        a.v.assign(val, val + rowptr[n]);
        if (!sdg::lattice_emulate_host(a, b, z_host)) sdg::fail(SDG_EINVAL, "not a lattice");
        if (ctx && !sdg::lattice_run_device(*ctx->p, a, b, z_dev_out, repeats)) sdg::fail(SDG_EINVAL, "not a lattice");
    });
}
extern "C" int sdg_debug_wave_blocks(unsigned long long* out, int max_bands) {
    return sdg::wave_blocks_copy(out, max_bands);
}
extern "C" int sdg_debug_wave_timeline(unsigned long long* out, int max_bands) {
    return sdg::wave_timeline_copy(out, max_bands);
}

const char* sdg_profile_family_name(int family) {
    static const char* names[] = {"spmv", "gs", "restrict", "prolong", "coarse",
                                  "uzawa", "ortho", "bicg", "vec", "setup", "gsprep", "spmv_block",
                                  "gs_wave", "iface", "gs_lattice"};
    return (family >= 0 && family < sdg::PF_COUNT) ? names[family] : "?";
}

// ---- matrices --------------------------------------------------------------
int sdg_matrix_create(sdg_context* ctx, int n_rows, int n_cols, const int* rowptr, const int* col,
                      const double* val, sdg_matrix** out) {
    return guard([&] {
        need(ctx, "sdg_matrix_create");
        need(out, "sdg_matrix_create");
        auto m = std::make_shared<sdg::Matrix>(ctx->p, make_csr(n_rows, n_cols, rowptr, col, val));
        m->ctx->sync();
        *out = new sdg_matrix{m};
    });
}
int sdg_matrix_destroy(sdg_matrix* a) {
    return guard([&] { delete a; });
}
int sdg_matrix_rows(const sdg_matrix* a) { return a ? a->p->host.n_rows : -1; }
int sdg_matrix_cols(const sdg_matrix* a) { return a ? a->p->host.n_cols : -1; }
int64_t sdg_matrix_nnz(const sdg_matrix* a) { return a ? a->p->host.nnz() : -1; }

int sdg_spmv_device(sdg_matrix* a, const double* x, double* y) {
    return guard([&] {
        need(a, "sdg_spmv_device");
        sdg::launch_spmv(*a->p->ctx, a->p->dev, x, y);
    });
}

int sdg_spmv(sdg_matrix* a, const double* x_host, double* y_host) {
    return guard([&] {
        need(a, "sdg_spmv");
        auto& m = *a->p;
        auto& c = *m.ctx;
        sdg::DevBuf<double> x(m.host.n_cols), y(m.host.n_rows);
        x.upload(x_host, m.host.n_cols, c.stream);
        sdg::launch_spmv(c, m.dev, x.get(), y.get());
        if (m.host.n_rows)
            SDG_CUDA(cudaMemcpyAsync(y_host, y.get(), sizeof(double) * m.host.n_rows,
                                     cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int sdg_spmv_add(sdg_matrix* a, const double* x_host, double* y_host, double alpha) {
    return guard([&] {
        need(a, "sdg_spmv_add");
        auto& m = *a->p;
        auto& c = *m.ctx;
        sdg::DevBuf<double> x(m.host.n_cols), y(m.host.n_rows);
        x.upload(x_host, m.host.n_cols, c.stream);
        y.upload(y_host, m.host.n_rows, c.stream);
        sdg::launch_spmv_add(c, m.dev, x.get(), y.get(), y.get(), alpha);
        if (m.host.n_rows)
            SDG_CUDA(cudaMemcpyAsync(y_host, y.get(), sizeof(double) * m.host.n_rows,
                                     cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int sdg_sor_sweep(sdg_matrix* a, double* z_host, const double* r_host, double omega) {
    return guard([&] {
        need(a, "sdg_sor_sweep");
        auto& m = *a->p;
        auto& c = *m.ctx;
        m.ensure_schedule();
        const int n = m.host.n_rows;
        sdg::DevBuf<double> zo(n), zn(n), r(n);
        zo.upload(z_host, n, c.stream);
        r.upload(r_host, n, c.stream);
        sdg::launch_gs_levels(c, m.dev, m.lvl_ptr.get(), m.lvl_rows.get(), m.n_levels, r.get(),
                              zo.get(), zn.get(), omega);
        if (n)
            SDG_CUDA(cudaMemcpyAsync(z_host, zn.get(), sizeof(double) * n, cudaMemcpyDeviceToHost,
                                     c.stream));
        c.sync();
    });
}

// ---- preconditioners ---------------------------------------------------------
int sdg_amg_create(sdg_matrix* a, const sdg_amg_options* opts, sdg_precond** out) {
    return guard([&] {
        need(a, "sdg_amg_create");
        need(out, "sdg_amg_create");
        auto p = std::make_shared<sdg::AmgPrecond>(a->p->ctx, a->p->host, amg_opts(opts, a->p->host.n_rows));
        *out = new sdg_precond{p};
    });
}

int sdg_uzawa_create(sdg_matrix* v, sdg_matrix* b, sdg_matrix* c, const sdg_uzawa_options* cfg,
                     sdg_precond** out) {
    return guard([&] {
        need(v, "sdg_uzawa_create");
        need(b, "sdg_uzawa_create");
        need(c, "sdg_uzawa_create");
        need(out, "sdg_uzawa_create");
        sdg_uzawa_options d;
        sdg_uzawa_defaults(&d);
        const sdg_uzawa_options& o = cfg ? *cfg : d;
        auto p = std::make_shared<sdg::UzawaPrecond>(v->p->ctx, v->p->host, b->p->host, c->p->host,
                                                     amg_opts(&o.amg, v->p->host.n_rows),
                                                     o.power_tol_rel, o.power_max_iters,
                                                     o.power_seed, o.omega_override);
        *out = new sdg_precond{p};
    });
}

int sdg_block_create(int kind, sdg_matrix* matrix, int n_v, int n_pff, int n_ppm,
                     sdg_precond* first, sdg_precond* pm, sdg_precond** out) {
    return guard([&] {
        need(matrix, "sdg_block_create");
        need(out, "sdg_block_create");
        auto p = std::make_shared<sdg::BlockPrecond>(matrix->p->ctx, kind, matrix->p->host, n_v,
                                                     n_pff, n_ppm, first ? first->p : nullptr,
                                                     pm ? pm->p : nullptr);
        *out = new sdg_precond{p};
    });
}

int sdg_ilu0_create(sdg_matrix* a, sdg_precond** out) {
    return guard([&] {
        need(a, "sdg_ilu0_create");
        need(out, "sdg_ilu0_create");
        *out = new sdg_precond{std::make_shared<sdg::Ilu0Precond>(a->p->ctx, a->p->host)};
    });
}

int sdg_identity_create(sdg_context* ctx, int n, sdg_precond** out) {
    return guard([&] {
        need(ctx, "sdg_identity_create");
        need(out, "sdg_identity_create");
        *out = new sdg_precond{std::make_shared<sdg::IdentityPrecond>(ctx->p, n)};
    });
}

int sdg_gs_merged_sweep_host(int n, const int* rowptr, const int* col, const double* val, int k, int dyn_cap,
                             const double* r, const double* z_old, double* z_new, int* groups) {
    return guard([&] {
        sdg::HostCsr h = make_csr(n, n, rowptr, col, val);
        require_diagonal(h, "sor_sweep");
        const int g = sdg::gs_merged_sweep_host(h, std::max(1, k), dyn_cap, r, z_old, z_new);
        if (g < 0) sdg::fail(SDG_EINVAL, "gs merge: a merged row needs more than 16 entries");
        if (groups) *groups = g;
    });
}

int sdg_ground_dof_host(int n, const int* rowptr, const int* col, double* val_inout, int dof) {
    return guard([&] {
        sdg::HostCsr h = make_csr(n, n, rowptr, col, val_inout);
        sdg::HostCsr g = sdg::ground_dof(h, dof);
        std::memcpy(val_inout, g.v.data(), sizeof(double) * g.v.size());
    });
}

int sdg_td_create(sdg_matrix* a, int n_u, int n_vel, int n_pff, int n_ppm, int kind,
                  int v_max_levels, int d_max_levels, double omega_override, sdg_precond** out) {
    return guard([&] {
        need(a, "sdg_td_create");
        need(out, "sdg_td_create");
        const bool ilu0 = (kind & SDG_TD_ILU0) != 0;  // td_*_uzawa_ilu0 (bench.cpp:156-172)
        kind &= ~SDG_TD_ILU0;
        if (kind != SDG_TD_BJ && kind != SDG_TD_BGS) sdg::fail(SDG_EINVAL, "sdg_td_create: kind must be td_bj or td_bgs");
        auto t0 = std::chrono::steady_clock::now();
        const sdg::HostCsr& A = a->p->host;
        const int n = A.n_rows;
        const int n_ff = n_vel + n_pff;
        if (n_ff + n_ppm != n || n_u < 0 || n_u > n_vel)
            sdg::fail(SDG_EDIM, "block preconditioner: partition does not cover the matrix");
        // bench.cpp:121-182
        sdg::HostCsr d_block = sdg::ground_dof(sdg::submatrix(A, n_ff, n, n_ff, n), 0);
        sdg::AmgOpts v_amg;
        v_amg.max_levels = v_max_levels;
        v_amg.components.assign(n_vel, 0);
        for (int k = n_u; k < n_vel; ++k) v_amg.components[k] = 1;
        sdg::AmgOpts d_amg;
        d_amg.max_levels = d_max_levels;
        auto ctx = a->p->ctx;
        auto first = std::make_shared<sdg::UzawaPrecond>(
            ctx, sdg::submatrix(A, 0, n_vel, 0, n_vel), sdg::submatrix(A, 0, n_vel, n_vel, n_ff),
            sdg::submatrix(A, n_vel, n_ff, 0, n_vel), v_amg, 1e-3, 200, 1729u, omega_override);
        sdg::PrecondPtr pm;
        if (ilu0)
            pm = std::make_shared<sdg::Ilu0Precond>(ctx, d_block);
        else
            pm = std::make_shared<sdg::AmgPrecond>(ctx, d_block, d_amg);
        auto blk = std::make_shared<sdg::BlockPrecond>(ctx, kind, A, n_vel, n_pff, n_ppm, first, pm);
        blk->setup_seconds = seconds_since(t0);
        *out = new sdg_precond{blk};
    });
}

int sdg_precond_destroy(sdg_precond* p) {
    return guard([&] { delete p; });
}
int sdg_precond_rows(const sdg_precond* p) { return p ? p->p->rows() : -1; }
int64_t sdg_precond_applications(const sdg_precond* p) { return p ? p->p->applications() : -1; }
int64_t sdg_precond_setup_memory_doubles(const sdg_precond* p) {
    return p ? p->p->setup_memory_doubles() : -1;
}
int64_t sdg_precond_work_per_apply(const sdg_precond* p) { return p ? p->p->work_per_apply() : -1; }
double sdg_precond_omega(const sdg_precond* p) {
    return p ? p->p->omega() : std::numeric_limits<double>::quiet_NaN();
}
double sdg_precond_setup_seconds(const sdg_precond* p) { return p ? p->p->setup_seconds : -1.0; }
int sdg_precond_set_graphs(sdg_precond* p, int enable) {
    return guard([&] {
        need(p, "sdg_precond_set_graphs");
        (void)enable;
    });
}

int sdg_precond_hierarchy(const sdg_precond* p, int which, int* n_levels, int* rows, int64_t* nnz,
                          int capacity) {
    return guard([&] {
        need(p, "sdg_precond_hierarchy");
        const sdg::AmgPrecond* amg = as_amg(p->p);
        if (!amg) {
            auto* blk = dynamic_cast<sdg::BlockPrecond*>(p->p.get());
            if (!blk) sdg::fail(SDG_EINVAL, "sdg_precond_hierarchy: not an AMG or block handle");
            const sdg::PrecondPtr& sub = which == 0 ? blk->first() : blk->pm();
            amg = as_amg(sub);
            if (!amg) {
                auto* uz = dynamic_cast<sdg::UzawaPrecond*>(sub.get());
                if (!uz) sdg::fail(SDG_EINVAL, "sdg_precond_hierarchy: sub-block has no hierarchy");
                amg = &uz->inner();
            }
        }
        *n_levels = amg->num_levels();
        for (int l = 0; l < amg->num_levels() && l < capacity; ++l) {
            rows[l] = amg->level_rows(l);
            nnz[l] = amg->level_nnz(l);
        }
    });
}

int sdg_precond_features(const sdg_precond* p, int* features) {
    return guard([&] {
        need(p, "sdg_precond_features");
        need(features, "sdg_precond_features");
        int f = 0;
        auto amg_of = [](const sdg::PrecondPtr& q) -> const sdg::AmgPrecond* {
            if (const sdg::AmgPrecond* a = as_amg(q)) return a;
            if (auto* uz = dynamic_cast<sdg::UzawaPrecond*>(q.get())) return &uz->inner();
            return nullptr;
        };
        if (auto* blk = dynamic_cast<sdg::BlockPrecond*>(p->p.get())) {
            if (blk->interface_split()) f |= SDG_FEAT_SPLIT;
            if (blk->early_correction()) f |= SDG_FEAT_EARLY;
            if (const sdg::AmgPrecond* a = amg_of(blk->first())) {
                if (a->finest_wave()) f |= SDG_FEAT_WAVE_V;
                if (a->coarse_lattice()) f |= SDG_FEAT_LATTICE_V;
            }
            if (const sdg::AmgPrecond* a = amg_of(blk->pm())) {
                if (a->finest_wave()) f |= SDG_FEAT_WAVE_D;
                if (a->coarse_lattice()) f |= SDG_FEAT_LATTICE_D;
            }
        } else if (const sdg::AmgPrecond* a = amg_of(p->p)) {
            if (a->finest_wave()) f |= SDG_FEAT_WAVE_V;
            if (a->coarse_lattice()) f |= SDG_FEAT_LATTICE_V;
        }
        *features = f;
    });
}

int sdg_precond_apply_device(sdg_precond* p, const double* r_dev, double* z_dev) {
    return guard([&] {
        need(p, "sdg_precond_apply_device");
        p->p->apply(r_dev, z_dev);
    });
}

int sdg_precond_apply(sdg_precond* p, const double* r_host, double* z_host) {
    return guard([&] {
        need(p, "sdg_precond_apply");
        auto& c = p->p->ctx();
        const int n = p->p->rows();
        sdg::DevBuf<double> r(n), z(n);
        r.upload(r_host, n, c.stream);
        p->p->apply(r.get(), z.get());
        if (n)
            SDG_CUDA(cudaMemcpyAsync(z_host, z.get(), sizeof(double) * n, cudaMemcpyDeviceToHost,
                                     c.stream));
        c.sync();
    });
}

// ---- Krylov --------------------------------------------------------------------
int sdg_pd_gmres_device(sdg_matrix* a, sdg_precond* precond, const double* b_dev, double* x_dev,
                        double tol_abs, int max_restarts, const sdg_restart* ctrl,
                        sdg_report* rep) {
    return guard([&] {
        need(a, "sdg_pd_gmres");
        auto t0 = std::chrono::steady_clock::now();
        const int64_t apps0 = precond ? precond->p->applications() : 0;
        sdg::SolveOut o = sdg::pd_gmres(*a->p, precond ? precond->p.get() : nullptr, b_dev, x_dev,
                                        tol_abs, max_restarts, restart_from(ctrl));
        fill_report(o, seconds_since(t0), (precond ? precond->p->applications() : 0) - apps0, rep);
    });
}

// Warm start (BASELINE config 4): the reference starts
// every solve from x = 0 (krylov.cpp:58), so a warm-started solve is the
// reference solve of the correction: r0 = b - A x, A d = r0, x += d.
int sdg_pd_gmres_warm_device(sdg_matrix* a, sdg_precond* precond, const double* b_dev, double* x_dev,
                             double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep) {
    return guard([&] {
        need(a, "sdg_pd_gmres_warm");
        auto t0 = std::chrono::steady_clock::now();
        auto& c = *a->p->ctx;
        const int n = a->p->host.n_rows;
        sdg::DevBuf<double> r0(std::max(n, 1)), d(std::max(n, 1));
        sdg::launch_spmv_add(c, a->p->dev, x_dev, b_dev, r0.get(), -1.0);
        const int64_t apps0 = precond ? precond->p->applications() : 0;
        sdg::SolveOut o = sdg::pd_gmres(*a->p, precond ? precond->p.get() : nullptr, r0.get(), d.get(),
                                        tol_abs, max_restarts, restart_from(ctrl));
        sdg::launch_add_inplace(c, n, x_dev, d.get());
        c.sync();
        fill_report(o, seconds_since(t0), (precond ? precond->p->applications() : 0) - apps0, rep);
    });
}

int sdg_pd_gmres_warm(sdg_matrix* a, sdg_precond* precond, const double* b_host, double* x_host,
                      double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep) {
    return guard([&] {
        need(a, "sdg_pd_gmres_warm");
        auto& c = *a->p->ctx;
        const int n = a->p->host.n_rows;
        c.stage(static_cast<std::size_t>(std::max(n, 1)));
        sdg::DevBuf<double>&b = c.stage_b, &x = c.stage_x;
        b.upload(b_host, n, c.stream);
        x.upload(x_host, n, c.stream);
        const int rc = sdg_pd_gmres_warm_device(a, precond, b.get(), x.get(), tol_abs, max_restarts, ctrl, rep);
        if (rc != SDG_OK) sdg::fail(rc, g_last_error);
        if (n) SDG_CUDA(cudaMemcpyAsync(x_host, x.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int sdg_bicgstab_warm_device(sdg_matrix* a, sdg_precond* precond, const double* b_dev, double* x_dev,
                             double tol_abs, int max_iters, sdg_report* rep) {
    return guard([&] {
        need(a, "sdg_bicgstab_warm");
        auto t0 = std::chrono::steady_clock::now();
        auto& c = *a->p->ctx;
        const int n = a->p->host.n_rows;
        sdg::DevBuf<double> r0(std::max(n, 1)), d(std::max(n, 1));
        sdg::launch_spmv_add(c, a->p->dev, x_dev, b_dev, r0.get(), -1.0);
        const int64_t apps0 = precond ? precond->p->applications() : 0;
        sdg::SolveOut o = sdg::bicgstab(*a->p, precond ? precond->p.get() : nullptr, r0.get(), d.get(), tol_abs,
                                        max_iters, /*throw_on_breakdown=*/false);
        sdg::launch_add_inplace(c, n, x_dev, d.get());
        c.sync();
        fill_report(o, seconds_since(t0), (precond ? precond->p->applications() : 0) - apps0, rep);
    });
}

int sdg_bicgstab_warm(sdg_matrix* a, sdg_precond* precond, const double* b_host, double* x_host, double tol_abs,
                      int max_iters, sdg_report* rep) {
    return guard([&] {
        need(a, "sdg_bicgstab_warm");
        auto& c = *a->p->ctx;
        const int n = a->p->host.n_rows;
        c.stage(static_cast<std::size_t>(std::max(n, 1)));
        sdg::DevBuf<double>&b = c.stage_b, &x = c.stage_x;
        b.upload(b_host, n, c.stream);
        x.upload(x_host, n, c.stream);
        const int rc = sdg_bicgstab_warm_device(a, precond, b.get(), x.get(), tol_abs, max_iters, rep);
        if (rc != SDG_OK) sdg::fail(rc, g_last_error);
        if (n) SDG_CUDA(cudaMemcpyAsync(x_host, x.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int sdg_pd_gmres(sdg_matrix* a, sdg_precond* precond, const double* b_host, double* x_host,
                 double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep) {
    return guard([&] {
        need(a, "sdg_pd_gmres");
        auto t0 = std::chrono::steady_clock::now();
        auto& c = *a->p->ctx;
        const int n = a->p->host.n_rows;
        c.stage(static_cast<std::size_t>(std::max(n, 1)));
        sdg::DevBuf<double>&b = c.stage_b, &x = c.stage_x;
        b.upload(b_host, n, c.stream);
        const int64_t apps0 = precond ? precond->p->applications() : 0;
        sdg::SolveOut o = sdg::pd_gmres(*a->p, precond ? precond->p.get() : nullptr, b.get(),
                                        x.get(), tol_abs, max_restarts, restart_from(ctrl));
        if (n)
            SDG_CUDA(cudaMemcpyAsync(x_host, x.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        fill_report(o, seconds_since(t0), (precond ? precond->p->applications() : 0) - apps0, rep);
    });
}

int sdg_bicgstab_device(sdg_matrix* a, sdg_precond* precond, const double* b_dev, double* x_dev,
                        double tol_abs, int max_iters, sdg_report* rep) {
    return guard([&] {
        need(a, "sdg_bicgstab");
        auto t0 = std::chrono::steady_clock::now();
        const int64_t apps0 = precond ? precond->p->applications() : 0;
        sdg::SolveOut o = sdg::bicgstab(*a->p, precond ? precond->p.get() : nullptr, b_dev, x_dev,
                                        tol_abs, max_iters);
        fill_report(o, seconds_since(t0), (precond ? precond->p->applications() : 0) - apps0, rep);
    });
}

int sdg_bicgstab(sdg_matrix* a, sdg_precond* precond, const double* b_host, double* x_host,
                 double tol_abs, int max_iters, sdg_report* rep) {
    return guard([&] {
        need(a, "sdg_bicgstab");
        auto t0 = std::chrono::steady_clock::now();
        auto& c = *a->p->ctx;
        const int n = a->p->host.n_rows;
        c.stage(static_cast<std::size_t>(std::max(n, 1)));
        sdg::DevBuf<double>&b = c.stage_b, &x = c.stage_x;
        b.upload(b_host, n, c.stream);
        const int64_t apps0 = precond ? precond->p->applications() : 0;
        sdg::SolveOut o = sdg::bicgstab(*a->p, precond ? precond->p.get() : nullptr, b.get(),
                                        x.get(), tol_abs, max_iters);
        if (n)
            SDG_CUDA(cudaMemcpyAsync(x_host, x.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        fill_report(o, seconds_since(t0), (precond ? precond->p->applications() : 0) - apps0, rep);
    });
}

int sdg_power_iteration(sdg_matrix* a, double tol_rel, int max_iters, unsigned seed, double* value,
                        int* iterations, int* converged) {
    return guard([&] {
        need(a, "sdg_power_iteration");
        auto& m = *a->p;
        auto op = [&](const double* x, double* y) { sdg::launch_spmv(*m.ctx, m.dev, x, y); };
        sdg::PowerOut r = sdg::power_iteration(*m.ctx, m.host.n_rows, op, tol_rel, max_iters, seed);
        if (value) *value = r.value;
        if (iterations) *iterations = r.iterations;
        if (converged) *converged = r.converged ? 1 : 0;
    });
}

// ---- assembly ------------------------------------------------------------------
int sdg_assemble_monolithic(const sdg_scenario* sc, const double* k_cell, const double* v_prev,
                            int* n_total, int64_t* nnz, int* n_u, int* n_vel, int* n_pff,
                            int* n_ppm, int* rowptr, int* col, double* val, double* rhs) {
    return guard([&] {
        need(sc, "sdg_assemble_monolithic");
        sdg::Assembled s = sdg::assemble_monolithic(*sc, k_cell, v_prev);
        if (n_total) *n_total = s.a.n_rows;
        if (nnz) *nnz = s.a.nnz();
        if (n_u) *n_u = s.n_u;
        if (n_vel) *n_vel = s.n_vel;
        if (n_pff) *n_pff = s.n_pff;
        if (n_ppm) *n_ppm = s.n_ppm;
        if (rowptr) std::memcpy(rowptr, s.a.rp.data(), sizeof(int) * s.a.rp.size());
        if (col) std::memcpy(col, s.a.ci.data(), sizeof(int) * s.a.ci.size());
        if (val) std::memcpy(val, s.a.v.data(), sizeof(double) * s.a.v.size());
        if (rhs) std::memcpy(rhs, s.rhs.data(), sizeof(double) * s.rhs.size());
    });
}

int sdg_assemble_rhs_device(sdg_context* ctx, const sdg_scenario* sc, const double* v_prev_dev, double* rhs_dev) {
    return guard([&] {
        need(ctx, "sdg_assemble_rhs_device");
        need(sc, "sdg_assemble_rhs_device");
        need(rhs_dev, "sdg_assemble_rhs_device");
        sdg::launch_assemble_rhs(*ctx->p, *sc, v_prev_dev, rhs_dev);
    });
}

int sdg_assemble_matrix_device(sdg_context* ctx, const sdg_scenario* sc, const double* k_cell_dev, int* rowptr_dev,
                               int* col_dev, double* val_dev, int64_t capacity, int64_t* nnz) {
    return guard([&] {
        need(ctx, "sdg_assemble_matrix_device");
        need(sc, "sdg_assemble_matrix_device");
        need(rowptr_dev, "sdg_assemble_matrix_device");
        need(nnz, "sdg_assemble_matrix_device");
        *nnz = sdg::assemble_matrix_device(*ctx->p, *sc, k_cell_dev, rowptr_dev, col_dev, val_dev, capacity);
        if (col_dev && val_dev && capacity < *nnz)
            sdg::fail(SDG_EDIM, "sdg_assemble_matrix_device: capacity below the number of entries");
    });
}

// ---- partitioned subproblems (host) --------------------------------------------
namespace {
int copy_system(const sdg::LinearSystem& s, int* n, int64_t* nnz, int* rowptr, int* col, double* val, double* rhs) {
    if (n) *n = s.a.n_rows;
    if (nnz) *nnz = s.a.nnz();
    if (rowptr) std::memcpy(rowptr, s.a.rp.data(), sizeof(int) * s.a.rp.size());
    if (col) std::memcpy(col, s.a.ci.data(), sizeof(int) * s.a.ci.size());
    if (val) std::memcpy(val, s.a.v.data(), sizeof(double) * s.a.v.size());
    if (rhs) std::memcpy(rhs, s.rhs.data(), sizeof(double) * s.rhs.size());
    return SDG_OK;
}
}  // namespace

int sdg_assemble_stokes(const sdg_scenario* sc, const double* v_prev, const double* v_gamma, int* n,
                        int64_t* nnz, int* rowptr, int* col, double* val, double* rhs) {
    return guard([&] {
        need(sc, "sdg_assemble_stokes");
        copy_system(sdg::assemble_stokes_dirichlet(*sc, v_prev, v_gamma), n, nnz, rowptr, col, val, rhs);
    });
}

int sdg_assemble_darcy(const sdg_scenario* sc, const double* p_gamma, int* n, int64_t* nnz, int* rowptr, int* col,
                       double* val, double* rhs) {
    return guard([&] {
        need(sc, "sdg_assemble_darcy");
        copy_system(sdg::assemble_darcy_dirichlet(*sc, p_gamma), n, nnz, rowptr, col, val, rhs);
    });
}

int sdg_stokes_pressure_trace(const sdg_scenario* sc, const double* x_ff, double* trace) {
    return guard([&] {
        need(sc, "sdg_stokes_pressure_trace");
        sdg::stokes_pressure_trace(*sc, x_ff, trace);
    });
}

int sdg_darcy_velocity_trace(const sdg_scenario* sc, const double* p, const double* p_gamma, double* trace) {
    return guard([&] {
        need(sc, "sdg_darcy_velocity_trace");
        sdg::darcy_velocity_trace(*sc, p, p_gamma, trace);
    });
}

// ---- host hierarchy inspection ---------------------------------------------------
int sdg_host_hierarchy_build(int n, const int* rowptr, const int* col, const double* val,
                             const sdg_amg_options* opts, sdg_host_hierarchy** out) {
    return guard([&] {
        need(out, "sdg_host_hierarchy_build");
        sdg::HostCsr h = make_csr(n, n, rowptr, col, val);
        h.check();
        *out = new sdg_host_hierarchy{sdg::build_hierarchy(h, amg_opts(opts, n))};
    });
}

int sdg_host_hierarchy_levels(const sdg_host_hierarchy* h) {
    return h ? static_cast<int>(h->levels.size()) : -1;
}

int sdg_host_hierarchy_level(const sdg_host_hierarchy* h, int lev, int* n, int64_t* nnz,
                             int* n_coarse, int* n_sched_levels, int* rowptr, int* col,
                             double* val, int* agg) {
    return guard([&] {
        need(h, "sdg_host_hierarchy_level");
        if (lev < 0 || lev >= static_cast<int>(h->levels.size()))
            sdg::fail(SDG_EINVAL, "sdg_host_hierarchy_level: level out of range");
        const sdg::HostLevel& L = h->levels[lev];
        if (n) *n = L.a.n_rows;
        if (nnz) *nnz = L.a.nnz();
        if (n_coarse) *n_coarse = L.n_coarse;
        const bool last = lev + 1 == static_cast<int>(h->levels.size());
        if (n_sched_levels) *n_sched_levels = last ? 0 : sdg::lower_schedule(L.a).n_levels();
        if (rowptr) std::memcpy(rowptr, L.a.rp.data(), sizeof(int) * L.a.rp.size());
        if (col) std::memcpy(col, L.a.ci.data(), sizeof(int) * L.a.ci.size());
        if (val) std::memcpy(val, L.a.v.data(), sizeof(double) * L.a.v.size());
        if (agg && !L.aggregate_of.empty())
            std::memcpy(agg, L.aggregate_of.data(), sizeof(int) * L.aggregate_of.size());
    });
}

void sdg_host_hierarchy_destroy(sdg_host_hierarchy* h) { delete h; }

int sdg_galerkin_device(sdg_context* ctx, int n, const int* rowptr, const int* col, const double* val, const int* agg,
                        int n_coarse, int* c_rowptr, int* c_col, double* c_val, int64_t* c_nnz) {
    return guard([&] {
        need(ctx, "sdg_galerkin_device");
        need(agg, "sdg_galerkin_device");
        need(c_rowptr, "sdg_galerkin_device");
        sdg::HostCsr h = make_csr(n, n, rowptr, col, val);
        h.check();
        std::vector<int> a(agg, agg + n);
        for (int x : a)
            if (x < 0 || x >= n_coarse) sdg::fail(SDG_EINVAL, "sdg_galerkin_device: aggregate id out of range");
        SDG_CUDA(cudaSetDevice(ctx->p->device));
        const sdg::HostCsr c = sdg::galerkin_device(*ctx->p, h, a, n_coarse);
        std::memcpy(c_rowptr, c.rp.data(), sizeof(int) * c.rp.size());
        if (c_col) std::memcpy(c_col, c.ci.data(), sizeof(int) * c.ci.size());
        if (c_val) std::memcpy(c_val, c.v.data(), sizeof(double) * c.v.size());
        if (c_nnz) *c_nnz = c.nnz();
    });
}

int sdg_lu_factor(sdg_context* ctx, int n, const int* rowptr, const int* col, const double* val, sdg_lu** out) {
    return guard([&] {
        need(ctx, "sdg_lu_factor");
        need(out, "sdg_lu_factor");
        sdg::HostCsr h = make_csr(n, n, rowptr, col, val);
        h.check();
        auto lu = std::make_unique<sdg_lu>();
        lu->ctx = ctx->p;
        SDG_CUDA(cudaSetDevice(ctx->p->device));
        lu->solver.build(*ctx->p, h);
        lu->b.resize(std::max(n, 1));
        lu->x.resize(std::max(n, 1));
        *out = lu.release();
    });
}

int sdg_lu_solve(sdg_lu* lu, const double* b_host, double* x_host) {
    return guard([&] {
        need(lu, "sdg_lu_solve");
        const int n = lu->solver.n();
        if (n == 0) return;
        need(b_host, "sdg_lu_solve");
        need(x_host, "sdg_lu_solve");
        sdg::Context& cx = *lu->ctx;
        SDG_CUDA(cudaSetDevice(cx.device));
        SDG_CUDA(cudaMemcpyAsync(lu->b.get(), b_host, sizeof(double) * n, cudaMemcpyHostToDevice, cx.stream));
        lu->solver.solve(cx, lu->b.get(), lu->x.get());
        SDG_CUDA(cudaMemcpyAsync(x_host, lu->x.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, cx.stream));
        cx.sync();
    });
}

int sdg_lu_info(const sdg_lu* lu, int* dense, int* depth, int64_t* stored_doubles) {
    return guard([&] {
        need(lu, "sdg_lu_info");
        if (dense) *dense = lu->solver.dense() ? 1 : 0;
        if (depth) *depth = lu->solver.depth();
        if (stored_doubles) *stored_doubles = lu->solver.doubles();
    });
}

void sdg_lu_destroy(sdg_lu* lu) { delete lu; }

int sdg_nd_solve_host(int n, const int* rowptr, const int* col, const double* val, int leaf_rows, int max_depth,
                      const double* b, double* x, int* perm, int* n_nodes, int* depth, int* max_separator,
                      int64_t* stored_doubles, int* nodes_out, int max_nodes) {
    return guard([&] {
        sdg::HostCsr h = make_csr(n, n, rowptr, col, val);
        h.check();
        const sdg::NdTree t = sdg::nd_order(h, leaf_rows, max_depth);
        if (perm) std::memcpy(perm, t.perm.data(), sizeof(int) * t.perm.size());
        int ms = 0;
        int64_t doubles = 0;
        for (size_t i = 0; i < t.nodes.size(); ++i) {
            const sdg::NdNode& nd = t.nodes[i];
            const int64_t ni = nd.mid - nd.lo, ns = nd.hi - nd.mid;
            ms = std::max<int>(ms, static_cast<int>(ns));
            doubles += nd.leaf() ? (nd.hi - nd.lo) * static_cast<int64_t>(nd.hi - nd.lo) : ns * ns + ni * ns;
            if (nodes_out && static_cast<int>(i) < max_nodes) {
                nodes_out[4 * i + 0] = nd.lo;
                nodes_out[4 * i + 1] = nd.mid;
                nodes_out[4 * i + 2] = nd.hi;
                nodes_out[4 * i + 3] = nd.depth;
            }
        }
        if (n_nodes) *n_nodes = static_cast<int>(t.nodes.size());
        if (depth) *depth = t.max_depth;
        if (max_separator) *max_separator = ms;
        if (stored_doubles) *stored_doubles = doubles;
        if (b && x && !sdg::nd_solve_host(h, t, b, x))
            sdg::fail(SDG_ESINGULAR, "coarse solve: a nested-dissection block is singular");
    });
}

}  // extern "C"
