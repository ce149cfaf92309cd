// Krylov drivers with device-resident vectors.  The host runs the scalar
// control flow of krylov.cpp verbatim (Givens rotations, estimate-based stop,
// restart controller, best iterate, BiCGSTAB restart/replacement rules) and
// reads a handful of device scalars once per iteration; all O(N) work is in
// the kernels of kernels.cu.
//
// Orthogonalisation: the reference uses modified Gram-Schmidt with one
// reorthogonalisation pass (krylov.cpp:101-111).  Here it is classical
// Gram-Schmidt with one reorthogonalisation pass (CGS2): the same projector
// in exact arithmetic, evaluated as fused multi-dot / multi-axpy kernels
// that stream the basis 4 times per step instead of 2(i+1) separate
// dot+axpy passes (SURVEY.md §7 hard part 5).  The Hessenberg entry is the
// sum of the two passes' coefficients, as in the reference.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <string>

#include "solver.hpp"

namespace sdg {

void Restart::update(double rate) {
    rate = std::clamp(rate, -16.0, 16.0);
    const double derivative = has_rate_sample ? (rate - previous_rate) : 0.0;
    int delta = static_cast<int>(std::floor(alpha_p * rate + alpha_d * derivative));
    if (rate > -stall_threshold) delta = std::max(delta, m_step);
    current_m = std::clamp(current_m + delta, m_min, m_max);
    previous_rate = rate;
    has_rate_sample = true;
}

namespace {

struct EventTimer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t s;
    explicit EventTimer(cudaStream_t st) : s(st) {
        SDG_CUDA(cudaEventCreate(&a));
        SDG_CUDA(cudaEventCreate(&b));
        SDG_CUDA(cudaEventRecord(a, s));
    }
    double stop() {
        SDG_CUDA(cudaEventRecord(b, s));
        SDG_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        SDG_CUDA(cudaEventElapsedTime(&ms, a, b));
        return ms;
    }
    ~EventTimer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

inline void precond_apply(Context& c, Precond* p, const double* r, double* z, int n) {
    if (p)
        p->apply(r, z);
    else
        launch_copy(c, z, r, n);
}

// host <- device scalars, synchronising the stream
inline void read_back(Context& c, double* host, const double* dev, int count) {
    SDG_CUDA(cudaMemcpyAsync(host, dev, sizeof(double) * count, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
}

}  // namespace

// Per-matrix GMRES workspace (basis, work vectors, reduction scratch), kept
// across solves, and one captured graph per Arnoldi step index: step i is
// precond apply -> SpMV -> CGS2 (multi-dot, multi-axpy, twice, the second
// fused with the norm) -> scale into basis vector i + 1, and it reads and
// writes only this workspace, so the graphs replay for every solve with the
// same preconditioner.
struct GmresWork {
    int n = 0, m_cap = 0;
    int64_t ld = 0;
    DevBuf<double> basis, r, z, w, best_x, dd;
    ReduceWs ws;
    std::vector<cudaGraphExec_t> exec;
    std::vector<int64_t> exec_launches;
    const Precond* graph_p = nullptr;
    GmresWork(int n_, int m_cap_, Context& c)
        : n(n_), m_cap(m_cap_), ld((static_cast<int64_t>(n_) + 31) / 32 * 32),
          basis(static_cast<size_t>(ld) * (m_cap_ + 1)), r(n_), z(n_), w(n_), best_x(n_), dd(4 * 64),
          exec(m_cap_, nullptr), exec_launches(m_cap_, 0) {
        ws.init(std::max(reduce_blocks(n_, c.num_sms), 8 * c.num_sms), 64, c.stream);
    }
    void drop_graphs() {
        for (auto& e : exec)
            if (e) {
                cudaGraphExecDestroy(e);
                e = nullptr;
            }
        graph_p = nullptr;
    }
    ~GmresWork() { drop_graphs(); }
};

namespace {

bool graphs_enabled(const Context& c);

}  // namespace

SolveOut pd_gmres(Matrix& A, Precond* P, const double* b, double* x, double tol_abs,
                  int max_restarts, Restart ctrl) {
    Context& c = *A.ctx;
    const int n = A.host.n_rows;
    if (A.host.n_rows != A.host.n_cols) fail(SDG_EDIM, "pd_gmres: dimension mismatch");
    if (P && P->rows() != n) fail(SDG_EDIM, "pd_gmres: preconditioner dimension mismatch");
    const int m_cap = std::max(ctrl.m_max, ctrl.current_m);
    if (m_cap + 1 > 64) fail(SDG_EINVAL, "pd_gmres: restart length above 63 is not supported");

    SolveOut out;
    EventTimer timer(c.stream);
    double* host = c.pinned->as<double>();         // 0..255: reads
    double* host_up = host + 256;                  // 256..511: uploads
    double* host_step = host + 1024;               // 1024..1535: Arnoldi read-backs, two slots

    if (!A.gm_work || A.gm_work->n != n || A.gm_work->m_cap < m_cap)
        A.gm_work = std::make_shared<GmresWork>(n, std::max(m_cap, A.gm_work ? A.gm_work->m_cap : 0), c);
    GmresWork& W = *A.gm_work;
    const int64_t ld = W.ld;
    double* basis = W.basis.get();
    double *r = W.r.get(), *z = W.z.get(), *w = W.w.get(), *best_x = W.best_x.get();
    ReduceWs& ws = W.ws;
    double* h1 = W.dd.get();
    double* h2 = W.dd.get() + 64;
    double* sc = W.dd.get() + 128;   // [0] = ||w||, [1] = beta, [2] = ||r||^2
    double* yv = W.dd.get() + 192;

    // Arnoldi step i (krylov.cpp:99-118, CGS2 form) and the read-back of its
    // Hessenberg column into pinned slot `slot`
    auto enqueue_step = [&](int i) {
        const double* vi = basis + ld * i;
        precond_apply(c, P, vi, z, n);
        launch_spmv(c, A.dev, z, w);
        launch_multidot(c, ws, n, i + 1, basis, ld, w, h1);
        launch_multi_axpy(c, n, i + 1, basis, ld, h1, w);
        launch_multidot(c, ws, n, i + 1, basis, ld, w, h2);
        launch_multi_axpy_norm2(c, ws, n, i + 1, basis, ld, h2, w, sc);
        launch_scale_by_inv(c, n, w, sc, basis + ld * (i + 1));
    };
    const bool use_graph = graphs_enabled(c);
    if (use_graph && W.graph_p != P) W.drop_graphs();
    auto run_step = [&](int i, int slot) {
        if (use_graph) {
            if (!W.exec[i]) {
                const int64_t l0 = c.launches.load();
                cudaGraph_t g = nullptr;
                SDG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
                try {
                    enqueue_step(i);
                } catch (...) {
                    cudaStreamEndCapture(c.stream, &g);
                    if (g) cudaGraphDestroy(g);
                    throw;
                }
                SDG_CUDA(cudaStreamEndCapture(c.stream, &g));
                SDG_CUDA(cudaGraphInstantiate(&W.exec[i], g, 0));
                cudaGraphDestroy(g);
                W.exec_launches[i] = c.launches.load() - l0;
                c.launches.fetch_sub(W.exec_launches[i]);
                if (P) P->add_applications(-1);  // counted at replay
                W.graph_p = P;
            }
            SDG_CUDA(cudaGraphLaunch(W.exec[i], c.stream));
            c.count(static_cast<int>(W.exec_launches[i]));
            if (P) P->add_applications(1);
        } else {
            enqueue_step(i);
        }
        // h1 | h2 | ||w||: ordered before the next step's kernels overwrite them
        SDG_CUDA(cudaMemcpyAsync(host_step + 256 * slot, W.dd.get(), sizeof(double) * 129, cudaMemcpyDeviceToHost,
                                 c.stream));
        SDG_CUDA(cudaEventRecord(c.step_ev[slot], c.stream));
    };

    launch_fill(c, x, 0.0, n);
    launch_copy(c, r, b, n);
    launch_norm2sq(c, ws, n, r, sc + 2);
    read_back(c, host, sc + 2, 1);
    double res_norm = std::sqrt(host[0]);
    out.history.push_back(res_norm);
    if (res_norm <= tol_abs) {
        out.converged = true;
        out.final_residual = res_norm;
        out.device_ms = timer.stop();
        return out;
    }

    double prev_cycle_res = res_norm;
    launch_copy(c, best_x, x, n);
    double best_res = res_norm;
    bool trust_estimate = true;

    for (int cycle = 0; cycle < max_restarts; ++cycle) {
        const int m = ctrl.current_m;
        std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0);
        auto hij = [&](int i, int j) -> double& { return H[static_cast<size_t>(j) * (m + 1) + i]; };
        std::vector<double> g(m + 1, 0.0), cs(m, 0.0), sn(m, 0.0);

        const double beta = res_norm;  // = norm2(r) of the current residual
        g[0] = beta;
        host_up[0] = beta;
        SDG_CUDA(cudaMemcpyAsync(sc + 1, host_up, sizeof(double), cudaMemcpyHostToDevice, c.stream));
        launch_scale_by_inv(c, n, r, sc + 1, basis);

        int used = 0;
        bool basis_exhausted = false;
        // Step i + 1 is enqueued before step i's column is read back: it does
        // not depend on the host's Givens update, so the GPU never waits for
        // the host.  When step i ends the cycle, step i + 1 was speculative:
        // it wrote only basis vector i + 2 and the work vectors, which the
        // cycle end does not read (it reads basis 0..used-1 and overwrites w, z).
        run_step(0, 0);
        for (int i = 0; i < m; ++i) {
            if (i + 1 < m) run_step(i + 1, (i + 1) & 1);
            SDG_CUDA(cudaEventSynchronize(c.step_ev[i & 1]));
            const double* hs = host_step + 256 * (i & 1);
            for (int k = 0; k <= i; ++k) {
                hij(k, i) += hs[k];
                hij(k, i) += hs[64 + k];
            }
            const double wn = hs[128];
            hij(i + 1, i) = wn;
            for (int k = 0; k < i; ++k) {
                const double t0 = cs[k] * hij(k, i) + sn[k] * hij(k + 1, i);
                const double t1 = -sn[k] * hij(k, i) + cs[k] * hij(k + 1, i);
                hij(k, i) = t0;
                hij(k + 1, i) = t1;
            }
            const double denom = std::hypot(hij(i, i), hij(i + 1, i));
            if (denom == 0.0) {
                c.sync();
                fail(SDG_ESINGULAR, "pd_gmres: singular Hessenberg block");
            }
            cs[i] = hij(i, i) / denom;
            sn[i] = hij(i + 1, i) / denom;
            hij(i, i) = denom;
            hij(i + 1, i) = 0.0;
            g[i + 1] = -sn[i] * g[i];
            g[i] = cs[i] * g[i];

            ++out.iterations;
            ++used;
            const double est = std::abs(g[i + 1]);
            out.history.push_back(est);
            if (trust_estimate && est <= tol_abs) break;
            if (wn == 0.0) {
                basis_exhausted = true;
                break;
            }
        }

        if (used < m && P) P->add_applications(-1);  // the speculative step is not an apply of krylov.cpp
        std::vector<double> y(used, 0.0);
        for (int i = used - 1; i >= 0; --i) {
            double s = g[i];
            for (int j = i + 1; j < used; ++j) s -= hij(i, j) * y[j];
            if (hij(i, i) == 0.0) {
                c.sync();
                fail(SDG_ESINGULAR, "pd_gmres: singular Hessenberg block");
            }
            y[i] = s / hij(i, i);
        }
        std::copy(y.begin(), y.end(), host_up);
        SDG_CUDA(cudaMemcpyAsync(yv, host_up, sizeof(double) * std::max(used, 1),
                                 cudaMemcpyHostToDevice, c.stream));
        launch_lincomb(c, n, used, basis, ld, yv, w);
        precond_apply(c, P, w, z, n);
        launch_add_inplace(c, n, x, z);
        launch_spmv_add(c, A.dev, x, b, r, -1.0);  // r = b - A x
        launch_norm2sq(c, ws, n, r, sc + 2);
        read_back(c, host, sc + 2, 1);
        res_norm = std::sqrt(host[0]);
        if (res_norm < best_res) {
            best_res = res_norm;
            launch_copy(c, best_x, x, n);
        }
        if (trust_estimate && used < m && res_norm > tol_abs) trust_estimate = false;
        const double rate =
            std::log10(std::max(res_norm, 1e-300) / std::max(prev_cycle_res, 1e-300));
        ctrl.update(rate);
        prev_cycle_res = res_norm;
        if (res_norm <= tol_abs || basis_exhausted) break;
    }

    if (best_res < res_norm) {
        launch_copy(c, x, best_x, n);
        res_norm = best_res;
    }
    out.history.push_back(res_norm);
    out.final_residual = res_norm;
    out.converged = res_norm <= tol_abs;
    out.device_ms = timer.stop();
    return out;
}

// Per-matrix BiCGSTAB workspace, kept across solves so the captured
// iteration graph (which bakes in these pointers) can be replayed.
struct BiWork {
    int n = 0;
    DevBuf<double> r, rhat, p, vv, s, phat, shat, t, rt, scal;
    DevBuf<BiState> st;
    ReduceWs ws;
    cudaGraphExec_t exec = nullptr;
    const Precond* graph_p = nullptr;
    const double* graph_x = nullptr;
    int64_t graph_launches = 0;
    explicit BiWork(int n_, Context& c)
        : n(n_), r(n_), rhat(n_), p(n_), vv(n_), s(n_), phat(n_), shat(n_), t(n_), rt(n_), scal(4), st(1) {
        ws.init(reduce_blocks(n_, c.num_sms), 2, c.stream);
    }
    ~BiWork() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

namespace {

bool graphs_enabled(const Context& c) {
    static const bool env_off = [] {
        const char* e = std::getenv("SDG_GRAPHS");
        return e && e[0] == '0';
    }();
    return !env_off && !c.profiling;
}

}  // namespace

SolveOut bicgstab(Matrix& A, Precond* P, const double* b, double* x, double tol_abs,
                  int max_iters, bool throw_on_breakdown) {
    Context& c = *A.ctx;
    const int n = A.host.n_rows;
    if (A.host.n_rows != A.host.n_cols) fail(SDG_EDIM, "bicgstab: dimension mismatch");
    if (P && P->rows() != n) fail(SDG_EDIM, "bicgstab: preconditioner dimension mismatch");

    SolveOut out;
    EventTimer timer(c.stream);
    double* host = c.pinned->as<double>();
    BiState* hst = reinterpret_cast<BiState*>(host + 512);

    if (!A.bi_work || A.bi_work->n != n) A.bi_work = std::make_shared<BiWork>(n, c);
    BiWork& W = *A.bi_work;
    DevBuf<double>&r = W.r, &rhat = W.rhat, &p = W.p, &vv = W.vv, &s = W.s, &phat = W.phat,
                   &shat = W.shat, &t = W.t, &rt = W.rt, &scal = W.scal;
    DevBuf<BiState>& st = W.st;
    ReduceWs& ws = W.ws;

    // one iteration (krylov.cpp:241-283) plus the status read-back
    auto enqueue_iteration = [&]() {
        launch_bi_p(c, n, st.get(), r.get(), vv.get(), p.get());
        precond_apply(c, P, p.get(), phat.get(), n);
        launch_spmv(c, A.dev, phat.get(), vv.get());
        launch_bi_rv(c, ws, n, st.get(), rhat.get(), vv.get());
        launch_bi_s(c, ws, n, st.get(), r.get(), vv.get(), s.get());
        precond_apply(c, P, s.get(), shat.get(), n);
        launch_spmv(c, A.dev, shat.get(), t.get());
        launch_bi_t(c, ws, n, st.get(), t.get(), s.get());
        launch_bi_xr(c, ws, n, st.get(), phat.get(), shat.get(), s.get(), t.get(), rhat.get(), x, r.get());
        SDG_CUDA(cudaMemcpyAsync(hst, st.get(), sizeof(BiState), cudaMemcpyDeviceToHost, c.stream));
    };
    const bool use_graph = graphs_enabled(c);
    if (use_graph && (!W.exec || W.graph_p != P || W.graph_x != x)) {
        if (W.exec) {
            cudaGraphExecDestroy(W.exec);
            W.exec = nullptr;
        }
        const int64_t l0 = c.launches.load();
        cudaGraph_t g = nullptr;
        SDG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_iteration();
        } catch (...) {
            cudaStreamEndCapture(c.stream, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        SDG_CUDA(cudaStreamEndCapture(c.stream, &g));
        SDG_CUDA(cudaGraphInstantiate(&W.exec, g, 0));
        cudaGraphDestroy(g);
        W.graph_launches = c.launches.load() - l0;
        c.launches.fetch_sub(W.graph_launches);
        if (P) P->add_applications(-2);  // counted at replay
        W.graph_p = P;
        W.graph_x = x;
    }
    auto run_iteration = [&]() {
        if (use_graph) {
            SDG_CUDA(cudaGraphLaunch(W.exec, c.stream));
            c.count(static_cast<int>(W.graph_launches));
            if (P) P->add_applications(2);
        } else {
            enqueue_iteration();
        }
    };

    auto upload_state = [&](const BiState& s_) {
        *hst = s_;
        SDG_CUDA(cudaMemcpyAsync(st.get(), hst, sizeof(BiState), cudaMemcpyHostToDevice, c.stream));
    };
    auto read_state = [&]() -> BiState {  // the iteration already queued the copy
        c.sync();
        return *hst;
    };
    // true residual b - A x into `dst`, returning its norm
    auto true_residual = [&](double* dst) -> double {
        launch_spmv_add(c, A.dev, x, b, dst, -1.0);
        launch_norm2sq(c, ws, n, dst, scal.get());
        read_back(c, host, scal.get(), 1);
        return std::sqrt(host[0]);
    };

    launch_fill(c, x, 0.0, n);
    launch_copy(c, r.get(), b, n);
    launch_norm2sq(c, ws, n, r.get(), scal.get());
    read_back(c, host, scal.get(), 1);
    double res_norm = std::sqrt(host[0]);
    out.history.push_back(res_norm);
    if (res_norm <= tol_abs) {
        out.converged = true;
        out.final_residual = res_norm;
        out.device_ms = timer.stop();
        return out;
    }

    BiState s0{};
    s0.rho = s0.alpha = s0.omega = 1.0;
    s0.tol = tol_abs;
    s0.flag = BI_OK;
    // rhat = r; p = v = 0 (krylov.cpp:207)
    auto reset_directions = [&](double rho_alpha_omega) {
        launch_copy(c, rhat.get(), r.get(), n);
        launch_fill(c, p.get(), 0.0, n);
        launch_fill(c, vv.get(), 0.0, n);
        BiState s1 = s0;
        s1.rho = s1.alpha = s1.omega = rho_alpha_omega;
        upload_state(s1);
        launch_bi_rho(c, ws, n, st.get(), rhat.get(), r.get());
    };
    reset_directions(1.0);

    int restarts = 0, replacements = 0;
    bool done = false;
    BiState last{};
    static const bool debug = [] {
        const char* e = std::getenv("SDG_DEBUG");
        return e && e[0] == '1';
    }();
    auto hard_restart = [&]() {
        if (debug)
            std::fprintf(stderr, "[sdg] bicgstab hard restart %d: flag %d at iteration %d; rho_new %.3e rho %.3e "
                                 "rv %.3e omega %.3e rn %.3e sn %.3e tt %.3e\n",
                         restarts + 1, last.flag, out.iterations, last.rho_new, last.rho, last.rv, last.omega,
                         last.rn, last.sn, last.tt);
        if (++restarts > 1 && !throw_on_breakdown) {
            out.breakdown = true;
            done = true;
            return;
        }
        if (restarts > 1) {
            static const char* why[] = {"", "rho", "rv", "", "tt", "omega"};
            char msg[256];
            std::snprintf(msg, sizeof msg,
                          "bicgstab: repeated breakdown (%s at iteration %d; rho_new %.3e rho %.3e rv %.3e "
                          "omega %.3e rn %.3e)",
                          why[last.flag], out.iterations, last.rho_new, last.rho, last.rv, last.omega, last.rn);
            fail(SDG_EBREAKDOWN, msg);
        }
        true_residual(r.get());
        reset_directions(1.0);
    };
    auto confirmed = [&]() -> bool {
        const double tn = true_residual(rt.get());
        if (tn <= tol_abs) return true;
        if (replacements++ < 3) {
            launch_copy(c, r.get(), rt.get(), n);
            reset_directions(1.0);
            return false;
        }
        done = true;
        return false;
    };

    for (int iter = 0; iter < max_iters && !done; ++iter) {
        run_iteration();
        BiState cur = read_state();
        last = cur;
        switch (cur.flag) {
        case BI_BREAK_RHO:
        case BI_BREAK_RV:
            hard_restart();
            continue;
        default:
            break;
        }
        ++out.iterations;
        if (cur.flag == BI_S_CONV) {
            launch_bi_x_alpha(c, n, st.get(), phat.get(), x);
            out.history.push_back(cur.sn);
            cur.flag = BI_OK;
            upload_state(cur);
            if (confirmed()) break;
            continue;
        }
        if (cur.flag == BI_BREAK_TT || cur.flag == BI_BREAK_OMEGA) {
            hard_restart();
            continue;
        }
        res_norm = cur.rn;
        out.history.push_back(res_norm);
        if (res_norm <= tol_abs && confirmed()) break;
    }

    const double fin = true_residual(rt.get());
    out.final_residual = fin;
    out.history.push_back(fin);
    out.converged = fin <= tol_abs;
    out.device_ms = timer.stop();
    return out;
}

}  // namespace sdg
