// sdc_gpu.hpp -- header-only C++ adapter that plugs libsdgpu.so (include/sdg.h)
// into the reference's own solver API (/root/reference/proj/core/include/sdc).
//
// A reference user keeps assembly, system layout and drivers unchanged and
// swaps the Krylov path:
//
//   sdc::CoupledSystem sys = sdc::assemble_monolithic(grid, cfg, v_prev, t);
//   sdc_gpu::Context gpu;                                  // device 0
//   sdc_gpu::Matrix A(gpu, sys.matrix);                    // LinearOperator::from_matrix
//   auto P = sdc_gpu::td_bgs(A, sys);                      // bench.cpp:121-182 wiring
//   sdc::GmresResult r = sdc_gpu::pd_gmres(A, P.get(), sys.rhs, tol, 400,
//                                           sdc::RestartController::defaults());
//
// The preconditioner is a genuine sdc::Preconditioner subclass (the same
// subclassing pattern as tests/unit/test_precond.cpp:340-352), so it can also
// be handed to the reference's own sdc::pd_gmres / sdc::bicgstab.  Errors are
// rethrown as the exception types the reference throws: SDG_EDIM ->
// std::invalid_argument, SDG_ESINGULAR / SDG_EBREAKDOWN -> std::runtime_error.
#ifndef SDC_GPU_HPP
#define SDC_GPU_HPP

#include <cmath>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "sdc/assembly.hpp"
#include "sdc/krylov.hpp"
#include "sdc/operator.hpp"
#include "sdc/sparse.hpp"
#include "sdg.h"

namespace sdc_gpu {

inline void check(int rc) {
    if (rc == SDG_OK) return;
    const std::string msg = sdg_last_error();
    if (rc == SDG_EDIM) throw std::invalid_argument(msg);
    if (rc == SDG_ESINGULAR || rc == SDG_EBREAKDOWN) throw std::runtime_error(msg);
    throw std::runtime_error("sdgpu: " + msg);
}

class Context {
public:
    explicit Context(int device = 0) { check(sdg_context_create(device, &h_)); }
    ~Context() { sdg_context_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    sdg_context* get() const { return h_; }

private:
    sdg_context* h_ = nullptr;
};

// Device copy of an sdc::SparseMatrix; op() is LinearOperator::from_matrix
// (operator.hpp:24-27) with the product on the GPU.
class Matrix {
public:
    Matrix(Context& ctx, const sdc::SparseMatrix& a) : rows_(a.n_rows) {
        check(sdg_matrix_create(ctx.get(), a.n_rows, a.n_cols, a.row_offsets.data(), a.col_indices.data(),
                                a.values.data(), &h_));
    }
    ~Matrix() { sdg_matrix_destroy(h_); }
    Matrix(const Matrix&) = delete;
    Matrix& operator=(const Matrix&) = delete;
    sdg_matrix* get() const { return h_; }
    int rows() const { return rows_; }
    sdc::LinearOperator op() const {
        sdg_matrix* h = h_;
        return {rows_, [h](std::span<const double> x, std::span<double> y) { check(sdg_spmv(h, x.data(), y.data())); }};
    }

private:
    sdg_matrix* h_ = nullptr;
    int rows_ = 0;
};

// A device preconditioner behind the reference contract (operator.hpp:34-62).
class Preconditioner final : public sdc::Preconditioner {
public:
    explicit Preconditioner(sdg_precond* h) : h_(h) {}
    ~Preconditioner() override { sdg_precond_destroy(h_); }
    int rows() const override { return sdg_precond_rows(h_); }
    std::int64_t setup_memory_doubles() const override { return sdg_precond_setup_memory_doubles(h_); }
    std::int64_t work_per_apply() const override { return sdg_precond_work_per_apply(h_); }
    double omega() const { return sdg_precond_omega(h_); }
    sdg_precond* get() const { return h_; }

protected:
    void do_apply(std::span<const double> r, std::span<double> z) const override {
        check(sdg_precond_apply(h_, r.data(), z.data()));
    }

private:
    sdg_precond* h_;
};

// MonolithicDriver::build_preconditioner (bench.cpp:121-182) for td_bgs / td_bj.
inline std::shared_ptr<Preconditioner> td_bgs(Matrix& a, const sdc::CoupledSystem& sys, int v_max_levels = 3,
                                              int d_max_levels = 3, bool block_jacobi = false) {
    sdg_precond* h = nullptr;
    check(sdg_td_create(a.get(), sys.grid.ff.n_u(), sys.pv_v.size(), sys.pv_pff.size(), sys.pv_ppm.size(),
                        block_jacobi ? SDG_TD_BJ : SDG_TD_BGS, v_max_levels, d_max_levels,
                        std::numeric_limits<double>::quiet_NaN(), &h));
    return std::make_shared<Preconditioner>(h);
}

namespace detail {
inline sdc::GmresResult result(std::vector<double> x, const sdg_report& rep, std::vector<double> hist) {
    sdc::GmresResult out;
    out.x = std::move(x);
    out.report.iterations = rep.iterations;
    out.report.converged = rep.converged != 0;
    out.report.wall_time = rep.wall_time;
    out.report.final_residual = rep.final_residual;
    hist.resize(std::min<std::size_t>(hist.size(), static_cast<std::size_t>(rep.history_length)));
    out.report.residual_history = std::move(hist);
    return out;
}
}  // namespace detail

// Same signature and semantics as sdc::pd_gmres (krylov.hpp:57-59).
inline sdc::GmresResult pd_gmres(const Matrix& a, const Preconditioner* p, std::span<const double> b,
                                 double tol_abs, int max_restarts, sdc::RestartController ctrl) {
    if (static_cast<int>(b.size()) != a.rows()) throw std::invalid_argument("pd_gmres: dimension mismatch");
    sdg_restart c{ctrl.m_init, ctrl.m_min, ctrl.m_step, ctrl.m_max, ctrl.current_m, ctrl.previous_rate,
                  ctrl.has_rate_sample ? 1 : 0, ctrl.alpha_p, ctrl.alpha_d, ctrl.stall_threshold};
    std::vector<double> x(b.size()), hist(static_cast<std::size_t>(max_restarts) * (ctrl.m_max + 1) + 2);
    sdg_report rep{};
    rep.residual_history = hist.data();
    rep.history_capacity = static_cast<int>(hist.size());
    check(sdg_pd_gmres(a.get(), p ? p->get() : nullptr, b.data(), x.data(), tol_abs, max_restarts, &c, &rep));
    return detail::result(std::move(x), rep, std::move(hist));
}

// Same signature and semantics as sdc::bicgstab (krylov.hpp:63-65).
inline sdc::GmresResult bicgstab(const Matrix& a, const Preconditioner* p, std::span<const double> b,
                                 double tol_abs, int max_iters) {
    if (static_cast<int>(b.size()) != a.rows()) throw std::invalid_argument("bicgstab: dimension mismatch");
    std::vector<double> x(b.size()), hist(static_cast<std::size_t>(max_iters) + 8);
    sdg_report rep{};
    rep.residual_history = hist.data();
    rep.history_capacity = static_cast<int>(hist.size());
    check(sdg_bicgstab(a.get(), p ? p->get() : nullptr, b.data(), x.data(), tol_abs, max_iters, &rep));
    return detail::result(std::move(x), rep, std::move(hist));
}

}  // namespace sdc_gpu

#endif  // SDC_GPU_HPP
