// extern "C" boundary of the strip-sharded solve (include/sdg.h, "multi-GPU").
#include <cmath>
#include <limits>

#include "capi_util.hpp"
#include "dist.hpp"

using namespace sdg_capi;

struct sdg_transport {
    sdg::TransportPtr p;
};
struct sdg_dist_system {
    std::unique_ptr<sdg::DistSystem> p;
};
struct sdg_dist_precond {
    std::unique_ptr<sdg::DistTd> p;
};

extern "C" {

int sdg_transport_create_host(int rank, int size, sdg_host_exchange_fn ex, sdg_host_allgather_fn ag, void* user,
                              sdg_transport** out) {
    return guard([&] {
        need(out, "sdg_transport_create_host");
        *out = new sdg_transport{sdg::make_host_transport(rank, size, ex, ag, user)};
    });
}

int sdg_nccl_get_unique_id(unsigned char id[128]) {
    return guard([&] {
        need(id, "sdg_nccl_get_unique_id");
        sdg::nccl_unique_id(id);
    });
}

int sdg_transport_create_nccl(sdg_context* ctx, const unsigned char id[128], int rank, int size,
                              sdg_transport** out) {
    return guard([&] {
        need(ctx, "sdg_transport_create_nccl");
        need(id, "sdg_transport_create_nccl");
        need(out, "sdg_transport_create_nccl");
        *out = new sdg_transport{sdg::make_nccl_transport(*ctx->p, id, rank, size)};
    });
}

int sdg_transport_destroy(sdg_transport* t) {
    return guard([&] { delete t; });
}

int sdg_strip_partition(int n, int n_ranks, int* owner) {
    return guard([&] {
        need(owner, "sdg_strip_partition");
        std::vector<int> o = sdg::strip_partition(n, n_ranks);
        std::copy(o.begin(), o.end(), owner);
    });
}

int sdg_dist_halo_plan(int n_total, const int* rowptr, const int* col, const int* owner, int rank, int size,
                       int* n_ghost, int* ghost_gid, int* recv_counts, int* n_send, int* send_gid,
                       int* send_counts) {
    return guard([&] {
        need(owner, "sdg_dist_halo_plan");
        if (rank < 0 || rank >= size) sdg::fail(SDG_EINVAL, "sdg_dist_halo_plan: bad rank");
        sdg::HostCsr a(n_total, n_total);
        a.rp.assign(rowptr, rowptr + n_total + 1);
        a.ci.assign(col, col + rowptr[n_total]);
        a.v.assign(a.ci.size(), 0.0);
        const sdg::Ownership own = sdg::Ownership::from_owner(std::vector<int>(owner, owner + n_total), size);
        sdg::HostCsr loc;
        sdg::Halo h;
        sdg::build_local(a, own, own, rank, loc, h);
        if (n_ghost) *n_ghost = h.n_ghost();
        if (n_send) *n_send = static_cast<int>(h.send_gid.size());
        if (ghost_gid) std::copy(h.ghost_gid.begin(), h.ghost_gid.end(), ghost_gid);
        if (send_gid) std::copy(h.send_gid.begin(), h.send_gid.end(), send_gid);
        if (recv_counts) std::copy(h.rcount.begin(), h.rcount.end(), recv_counts);
        if (send_counts) std::copy(h.scount.begin(), h.scount.end(), send_counts);
    });
}

int sdg_dist_system_create(sdg_context* ctx, sdg_transport* tr, int n_total, const int* rowptr, const int* col,
                           const double* val, int n_u, int n_vel, int n_pff, int n_ppm, const int* owner,
                           sdg_dist_system** out) {
    return guard([&] {
        need(ctx, "sdg_dist_system_create");
        need(tr, "sdg_dist_system_create");
        need(owner, "sdg_dist_system_create");
        need(out, "sdg_dist_system_create");
        auto s = std::make_unique<sdg::DistSystem>();
        s->ctx = ctx->p;
        s->tr = tr->p;
        s->global = make_csr(n_total, n_total, rowptr, col, val);
        s->global.check();
        if (n_vel + n_pff + n_ppm != n_total || n_u < 0 || n_u > n_vel)
            sdg::fail(SDG_EDIM, "block preconditioner: partition does not cover the matrix");
        s->n_u = n_u;
        s->n_vel = n_vel;
        s->n_pff = n_pff;
        s->n_ppm = n_ppm;
        s->own = sdg::Ownership::from_owner(std::vector<int>(owner, owner + n_total), tr->p->size);
        const int rank = tr->p->rank;
        s->A.build(*s->ctx, s->global, s->own, s->own, rank);
        for (int g : s->own.owned[rank]) {
            if (g < n_vel)
                ++s->n_v_loc;
            else if (g < n_vel + n_pff)
                ++s->n_pff_loc;
            else
                ++s->n_ppm_loc;
        }
        s->ctx->sync();
        *out = new sdg_dist_system{std::move(s)};
    });
}

int sdg_dist_system_destroy(sdg_dist_system* s) {
    return guard([&] { delete s; });
}

int sdg_dist_local_rows(const sdg_dist_system* s, int* n_local, int* global_ids) {
    return guard([&] {
        need(s, "sdg_dist_local_rows");
        const std::vector<int>& g = s->p->own.owned[s->p->tr->rank];
        if (n_local) *n_local = static_cast<int>(g.size());
        if (global_ids) std::copy(g.begin(), g.end(), global_ids);
    });
}

int sdg_dist_spmv(sdg_dist_system* s, const double* x_local, double* y_local) {
    return guard([&] {
        need(s, "sdg_dist_spmv");
        sdg::DistSystem& S = *s->p;
        sdg::Context& c = *S.ctx;
        const int n = S.n_local();
        sdg::DevBuf<double> x(std::max(n, 1)), y(std::max(n, 1));
        x.upload(x_local, n, c.stream);
        S.A.apply(c, *S.tr, x.get(), y.get());
        if (n) SDG_CUDA(cudaMemcpyAsync(y_local, y.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int sdg_dist_td_create(sdg_dist_system* s, int kind, int v_max_levels, int d_max_levels, double omega_override,
                       sdg_dist_precond** out) {
    return guard([&] {
        need(s, "sdg_dist_td_create");
        need(out, "sdg_dist_td_create");
        *out = new sdg_dist_precond{
            std::make_unique<sdg::DistTd>(*s->p, kind, v_max_levels, d_max_levels, omega_override)};
    });
}

int sdg_dist_precond_destroy(sdg_dist_precond* p) {
    return guard([&] { delete p; });
}

double sdg_dist_precond_omega(const sdg_dist_precond* p) {
    return p ? p->p->omega() : std::numeric_limits<double>::quiet_NaN();
}

double sdg_dist_precond_setup_seconds(const sdg_dist_precond* p) { return p ? p->p->setup_seconds : -1.0; }

int sdg_dist_precond_apply(sdg_dist_system* s, sdg_dist_precond* p, const double* r_local, double* z_local) {
    return guard([&] {
        need(s, "sdg_dist_precond_apply");
        need(p, "sdg_dist_precond_apply");
        sdg::DistSystem& S = *s->p;
        sdg::Context& c = *S.ctx;
        const int n = S.n_local();
        sdg::DevBuf<double> r(std::max(n, 1)), z(std::max(n, 1));
        r.upload(r_local, n, c.stream);
        p->p->apply(r.get(), z.get());
        if (n) SDG_CUDA(cudaMemcpyAsync(z_local, z.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int sdg_dist_pd_gmres(sdg_dist_system* s, sdg_dist_precond* p, const double* b_local, double* x_local,
                      double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep) {
    return guard([&] {
        need(s, "sdg_dist_pd_gmres");
        auto t0 = std::chrono::steady_clock::now();
        sdg::DistSystem& S = *s->p;
        sdg::Context& c = *S.ctx;
        const int n = S.n_local();
        sdg::DevBuf<double> b(std::max(n, 1)), x(std::max(n, 1));
        b.upload(b_local, n, c.stream);
        const int64_t apps0 = p ? p->p->applications() : 0;
        sdg::SolveOut o = sdg::dist_pd_gmres(S, p ? p->p.get() : nullptr, b.get(), x.get(), tol_abs, max_restarts,
                                             restart_from(ctrl));
        if (n) SDG_CUDA(cudaMemcpyAsync(x_local, x.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        fill_report(o, seconds_since(t0), (p ? p->p->applications() : 0) - apps0, rep);
    });
}

int sdg_dist_bicgstab(sdg_dist_system* s, sdg_dist_precond* p, const double* b_local, double* x_local,
                      double tol_abs, int max_iters, sdg_report* rep) {
    return guard([&] {
        need(s, "sdg_dist_bicgstab");
        auto t0 = std::chrono::steady_clock::now();
        sdg::DistSystem& S = *s->p;
        sdg::Context& c = *S.ctx;
        const int n = S.n_local();
        sdg::DevBuf<double> b(std::max(n, 1)), x(std::max(n, 1));
        b.upload(b_local, n, c.stream);
        const int64_t apps0 = p ? p->p->applications() : 0;
        sdg::SolveOut o = sdg::dist_bicgstab(S, p ? p->p.get() : nullptr, b.get(), x.get(), tol_abs, max_iters);
        if (n) SDG_CUDA(cudaMemcpyAsync(x_local, x.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        fill_report(o, seconds_since(t0), (p ? p->p->applications() : 0) - apps0, rep);
    });
}

int sdg_dist_pd_gmres_device(sdg_dist_system* s, sdg_dist_precond* p, const double* b_dev, double* x_dev,
                             double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep) {
    return guard([&] {
        need(s, "sdg_dist_pd_gmres_device");
        auto t0 = std::chrono::steady_clock::now();
        const int64_t apps0 = p ? p->p->applications() : 0;
        sdg::SolveOut o = sdg::dist_pd_gmres(*s->p, p ? p->p.get() : nullptr, b_dev, x_dev, tol_abs, max_restarts,
                                             restart_from(ctrl));
        fill_report(o, seconds_since(t0), (p ? p->p->applications() : 0) - apps0, rep);
    });
}

int sdg_dist_bicgstab_device(sdg_dist_system* s, sdg_dist_precond* p, const double* b_dev, double* x_dev,
                             double tol_abs, int max_iters, sdg_report* rep) {
    return guard([&] {
        need(s, "sdg_dist_bicgstab_device");
        auto t0 = std::chrono::steady_clock::now();
        const int64_t apps0 = p ? p->p->applications() : 0;
        sdg::SolveOut o = sdg::dist_bicgstab(*s->p, p ? p->p.get() : nullptr, b_dev, x_dev, tol_abs, max_iters);
        fill_report(o, seconds_since(t0), (p ? p->p->applications() : 0) - apps0, rep);
    });
}

}  // extern "C"

namespace {
// r0 = b - A x over strips, solve A d = r0 from zero, x += d
template <class Solve>
sdg::SolveOut dist_warm(sdg::DistSystem& S, const double* b_dev, double* x_dev, Solve&& solve) {
    sdg::Context& c = *S.ctx;
    const int n = S.n_local();
    sdg::DevBuf<double> r0(std::max(n, 1)), d(std::max(n, 1));
    S.A.apply_add(c, *S.tr, x_dev, b_dev, r0.get(), -1.0);
    sdg::SolveOut o = solve(r0.get(), d.get());
    sdg::launch_add_inplace(c, n, x_dev, d.get());
    c.sync();
    return o;
}
}  // namespace

extern "C" {

int sdg_dist_pd_gmres_warm_device(sdg_dist_system* s, sdg_dist_precond* p, const double* b_dev, double* x_dev,
                                  double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep) {
    return guard([&] {
        need(s, "sdg_dist_pd_gmres_warm_device");
        auto t0 = std::chrono::steady_clock::now();
        const int64_t apps0 = p ? p->p->applications() : 0;
        sdg::SolveOut o = dist_warm(*s->p, b_dev, x_dev, [&](const double* r0, double* d) {
            return sdg::dist_pd_gmres(*s->p, p ? p->p.get() : nullptr, r0, d, tol_abs, max_restarts,
                                      restart_from(ctrl));
        });
        fill_report(o, seconds_since(t0), (p ? p->p->applications() : 0) - apps0, rep);
    });
}

int sdg_dist_bicgstab_warm_device(sdg_dist_system* s, sdg_dist_precond* p, const double* b_dev, double* x_dev,
                                  double tol_abs, int max_iters, sdg_report* rep) {
    return guard([&] {
        need(s, "sdg_dist_bicgstab_warm_device");
        auto t0 = std::chrono::steady_clock::now();
        const int64_t apps0 = p ? p->p->applications() : 0;
        sdg::SolveOut o = dist_warm(*s->p, b_dev, x_dev, [&](const double* r0, double* d) {
            return sdg::dist_bicgstab(*s->p, p ? p->p.get() : nullptr, r0, d, tol_abs, max_iters);
        });
        fill_report(o, seconds_since(t0), (p ? p->p->applications() : 0) - apps0, rep);
    });
}

}  // extern "C"
