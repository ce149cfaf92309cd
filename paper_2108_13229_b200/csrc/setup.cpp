// Host setup for the device solver.  See setup.hpp.
#include "setup.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>

namespace sdg {

void HostCsr::check() const {
    if (static_cast<int>(rp.size()) != n_rows + 1 || rp.front() != 0)
        fail(SDG_EDIM, "SparseMatrix: row_offsets length mismatch");
    if (rp.back() != static_cast<int>(v.size()) || v.size() != ci.size())
        fail(SDG_EDIM, "SparseMatrix: stored value count mismatch");
    for (int i = 0; i < n_rows; ++i) {
        if (rp[i + 1] < rp[i]) fail(SDG_EDIM, "SparseMatrix: row_offsets not nondecreasing");
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            if (ci[k] < 0 || ci[k] >= n_cols)
                fail(SDG_EDIM, "SparseMatrix: column index out of range");
            if (k > rp[i] && ci[k] <= ci[k - 1])
                fail(SDG_EDIM, "SparseMatrix: columns not strictly increasing");
        }
    }
}

HostCsr submatrix(const HostCsr& a, int rb, int re, int cb, int ce) {
    if (rb < 0 || re > a.n_rows || cb < 0 || ce > a.n_cols || rb > re || cb > ce)
        fail(SDG_EDIM, "submatrix: bad range");
    HostCsr m(re - rb, ce - cb);
    for (int i = rb; i < re; ++i) {
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            const int j = a.ci[k];
            if (j < cb || j >= ce) continue;
            m.ci.push_back(j - cb);
            m.v.push_back(a.v[k]);
        }
        m.rp[i - rb + 1] = static_cast<int>(m.ci.size());
    }
    return m;
}

HostCsr ground_dof(const HostCsr& a, int dof) {
    if (dof < 0 || dof >= a.n_rows) fail(SDG_EDIM, "ground_dof: dof out of range");
    HostCsr g = a;
    double max_abs_diag = 0.0;
    int pos = -1;
    for (int i = 0; i < g.n_rows; ++i)
        for (int k = g.rp[i]; k < g.rp[i + 1]; ++k)
            if (g.ci[k] == i) {
                max_abs_diag = std::max(max_abs_diag, std::abs(g.v[k]));
                if (i == dof) pos = k;
            }
    if (pos < 0) fail(SDG_EDIM, "ground_dof: anchor dof has no stored diagonal");
    g.v[pos] += max_abs_diag > 0.0 ? max_abs_diag : 1.0;
    return g;
}

// ---------------------------------------------------------------------------
// ILU(0) factorization (precond.cpp:13-87): in place on the pattern of a, row
// by row, l_ik = a_ik / u_kk for k < i in column order, then row k's upper part
// merged into the rest of row i (fill outside the pattern dropped); the same
// operation sequence, so the factors are the reference's bit for bit.
void ilu0_factor(const HostCsr& a, HostCsr& lower, HostCsr& upper) {
    if (a.n_rows != a.n_cols) fail(SDG_EDIM, "ilu0: matrix must be square");
    const int n = a.n_rows;
    std::vector<double> f = a.v;
    std::vector<int> diag(n, -1);
    for (int i = 0; i < n; ++i)
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] == i) diag[i] = k;
    for (int i = 0; i < n; ++i) {
        const int row_end = a.rp[i + 1];
        for (int kk = a.rp[i]; kk < row_end; ++kk) {
            const int k = a.ci[kk];
            if (k >= i) break;
            if (diag[k] < 0 || f[diag[k]] == 0.0) fail(SDG_ESINGULAR, "ilu0: zero pivot in row " + std::to_string(k));
            const double lik = f[kk] / f[diag[k]];
            f[kk] = lik;
            int p = diag[k] + 1, q = kk + 1;
            const int k_end = a.rp[k + 1];
            while (p < k_end && q < row_end) {
                if (a.ci[p] == a.ci[q]) {
                    f[q] -= lik * f[p];
                    ++p;
                    ++q;
                } else if (a.ci[p] < a.ci[q]) {
                    ++p;
                } else {
                    ++q;
                }
            }
        }
        if (diag[i] < 0 || f[diag[i]] == 0.0) fail(SDG_ESINGULAR, "ilu0: zero pivot in row " + std::to_string(i));
    }
    lower = HostCsr(n, n);
    upper = HostCsr(n, n);
    for (int i = 0; i < n; ++i) {
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            HostCsr& t = a.ci[k] < i ? lower : upper;
            t.ci.push_back(a.ci[k]);
            t.v.push_back(f[k]);
        }
        lower.rp[i + 1] = static_cast<int>(lower.ci.size());
        upper.rp[i + 1] = static_cast<int>(upper.ci.size());
    }
}

// ---------------------------------------------------------------------------
// aggregation

namespace {

std::vector<double> stored_diagonal(const HostCsr& a) {
    std::vector<double> d(a.n_rows, 0.0);
    for (int i = 0; i < a.n_rows; ++i)
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] == i) d[i] = a.v[k];
    return d;
}

}  // namespace

std::vector<int> aggregate(const HostCsr& a, double theta, const std::vector<int>& comps,
                           int& n_aggregates) {
    const int n = a.n_rows;
    const std::vector<double> d = stored_diagonal(a);
    const bool labelled = !comps.empty();
    // strong coupling test of precond.cpp:132-137
    auto is_strong = [&](int i, int k) -> bool {
        const int j = a.ci[k];
        if (j == i) return false;
        if (labelled && comps[i] != comps[j]) return false;
        return std::abs(a.v[k]) >= theta * std::sqrt(std::abs(d[i] * d[j]));
    };

    std::vector<int> agg(n, -1);
    int next_id = 0;
    // seeding pass (precond.cpp:142-152)
    for (int i = 0; i < n; ++i) {
        if (agg[i] >= 0) continue;
        const int kb = a.rp[i], ke = a.rp[i + 1];
        bool touches_existing = false;
        for (int k = kb; k < ke && !touches_existing; ++k)
            touches_existing = is_strong(i, k) && agg[a.ci[k]] >= 0;
        if (touches_existing) continue;
        agg[i] = next_id;
        for (int k = kb; k < ke; ++k)
            if (is_strong(i, k) && agg[a.ci[k]] < 0) agg[a.ci[k]] = next_id;
        ++next_id;
    }
    // leftovers join the strongest assigned strong neighbour (precond.cpp:154-171)
    for (int i = 0; i < n; ++i) {
        if (agg[i] >= 0) continue;
        int target = -1;
        double strongest = -1.0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            const int j = a.ci[k];
            if (j == i || agg[j] < 0) continue;
            const double w = std::abs(a.v[k]);
            if (is_strong(i, k) && w > strongest) {
                strongest = w;
                target = agg[j];
            }
        }
        agg[i] = target >= 0 ? target : next_id++;
    }
    n_aggregates = next_id;
    return agg;
}

void aggregate_transpose(const std::vector<int>& agg, int n_coarse, std::vector<int>& ptr,
                         std::vector<int>& rows) {
    ptr.assign(n_coarse + 1, 0);
    for (int c : agg) ++ptr[c + 1];
    for (int c = 0; c < n_coarse; ++c) ptr[c + 1] += ptr[c];
    rows.resize(agg.size());
    std::vector<int> fill(ptr.begin(), ptr.end() - 1);
    for (int i = 0; i < static_cast<int>(agg.size()); ++i) rows[fill[agg[i]]++] = i;
}

HostCsr galerkin(const HostCsr& a, const std::vector<int>& agg, int n_coarse) {
    // A_c(c, c') = sum over fine (i, k) with agg[i] = c, agg[col_k] = c' of a_ik,
    // summed in the order the reference's CooBuilder sees them: fine rows
    // ascending, then row entries ascending (stable sort keeps that order).
    std::vector<int> ptr, rows;
    aggregate_transpose(agg, n_coarse, ptr, rows);
    HostCsr c(n_coarse, n_coarse);
    std::vector<double> acc(n_coarse, 0.0);
    std::vector<char> seen(n_coarse, 0);
    std::vector<int> touched;
    c.ci.reserve(a.nnz() / 2);
    c.v.reserve(a.nnz() / 2);
    for (int cr = 0; cr < n_coarse; ++cr) {
        touched.clear();
        for (int q = ptr[cr]; q < ptr[cr + 1]; ++q) {
            const int i = rows[q];
            for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
                const int cc = agg[a.ci[k]];
                if (!seen[cc]) {
                    seen[cc] = 1;
                    acc[cc] = 0.0;
                    touched.push_back(cc);
                }
                acc[cc] += a.v[k];
            }
        }
        std::sort(touched.begin(), touched.end());
        for (int cc : touched) {
            c.ci.push_back(cc);
            c.v.push_back(acc[cc]);
            seen[cc] = 0;
        }
        c.rp[cr + 1] = static_cast<int>(c.ci.size());
    }
    return c;
}

std::vector<HostLevel> build_hierarchy(const HostCsr& a, const AmgOpts& o, const GalerkinFn& product) {
    if (a.n_rows != a.n_cols) fail(SDG_EDIM, "amg_setup: matrix must be square");
    if (!o.components.empty() && static_cast<int>(o.components.size()) != a.n_rows)
        fail(SDG_EDIM, "amg_setup: component label length mismatch");
    std::vector<HostLevel> levels;
    levels.push_back({a, {}, 0, o.components});
    std::vector<int> labels = o.components;
    while (static_cast<int>(levels.size()) < o.max_levels &&
           levels.back().a.n_rows > o.coarse_threshold) {
        int n_coarse = 0;
        std::vector<int> agg = aggregate(levels.back().a, o.theta, labels, n_coarse);
        if (n_coarse >= levels.back().a.n_rows) break;  // no coarsening progress
        HostCsr coarse = product ? product(levels.back().a, agg, n_coarse) : galerkin(levels.back().a, agg, n_coarse);
        if (!labels.empty()) {
            std::vector<int> coarse_labels(n_coarse, 0);
            for (int i = 0; i < levels.back().a.n_rows; ++i) coarse_labels[agg[i]] = labels[i];
            labels.swap(coarse_labels);
        }
        levels.back().aggregate_of = std::move(agg);
        levels.back().n_coarse = n_coarse;
        levels.push_back({std::move(coarse), {}, 0, labels});
    }
    return levels;
}

// ---------------------------------------------------------------------------
// Gauss-Seidel support

LevelSchedule lower_schedule(const HostCsr& a) {
    const int n = a.n_rows;
    std::vector<int> depth(n, 0);
    int max_depth = -1;
    for (int i = 0; i < n; ++i) {
        int d = 0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            const int j = a.ci[k];
            if (j < i) d = std::max(d, depth[j] + 1);
        }
        depth[i] = d;
        max_depth = std::max(max_depth, d);
    }
    LevelSchedule s;
    s.lvl_ptr.assign(max_depth + 2, 0);
    for (int i = 0; i < n; ++i) ++s.lvl_ptr[depth[i] + 1];
    for (int l = 0; l <= max_depth; ++l) s.lvl_ptr[l + 1] += s.lvl_ptr[l];
    s.lvl_rows.resize(n);
    std::vector<int> fill(s.lvl_ptr.begin(), s.lvl_ptr.end() - 1);
    for (int i = 0; i < n; ++i) s.lvl_rows[fill[depth[i]]++] = i;
    if (n == 0) s.lvl_ptr.assign(1, 0);
    return s;
}

void require_diagonal(const HostCsr& a, const char* who) {
    for (int i = 0; i < a.n_rows; ++i) {
        double d = 0.0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] == i) d = a.v[k];
        if (d == 0.0) fail(SDG_ESINGULAR, std::string(who) + ": zero diagonal in row " + std::to_string(i));
    }
}

// ---------------------------------------------------------------------------
// Monolithic assembly on the n x n free-flow box.
//
// Each row is emitted as a list of (column, coefficient) contributions in a
// fixed order; off-diagonal columns are unique within a row, and diagonal
// contributions are summed in emission order starting from 0.0.  That is
// exactly the value the reference's CooBuilder produces (stable sort, sum of
// duplicates in insertion order, sparse.cpp:55-79), so with a uniform
// permeability the matrix and rhs are bitwise those of the reference.

namespace {

struct RowSink {
    HostCsr* out;
    std::vector<std::pair<int, double>> off;
    double diag = 0.0;
    bool has_diag = false;
    int row = 0;

    void begin(int r) {
        row = r;
        off.clear();
        diag = 0.0;
        has_diag = false;
    }
    void d(double x) {
        diag += x;
        has_diag = true;
    }
    void o(int col, double x) { off.emplace_back(col, x); }
    void end() {
        if (has_diag) off.emplace_back(row, diag);
        std::sort(off.begin(), off.end(),
                  [](const auto& p, const auto& q) { return p.first < q.first; });
        for (const auto& [c, x] : off) {
            out->ci.push_back(c);
            out->v.push_back(x);
        }
        out->rp[row + 1] = static_cast<int>(out->ci.size());
    }
};

// harmonic mean with the uniform case kept exact
inline double hmean(double ka, double kb) { return ka == kb ? ka : 2.0 * ka * kb / (ka + kb); }

}  // namespace

Assembled assemble_monolithic(const sdg_scenario& sc, const double* k_cell, const double* v_prev) {
    const int n = sc.n;
    if (n < 1) fail(SDG_EDIM, "assemble_monolithic: n must be positive");
    const double h = 1.0 / n;
    const double mu = sc.nu * sc.rho;
    const double tc = std::isfinite(sc.dt) ? sc.rho / sc.dt : 0.0;
    const double p_in = sc.dp_max * 0.5 * (1.0 - std::cos(M_PI * sc.t / sc.t_end));
    const double p_out = 0.0;
    const double k_uniform = sc.permeability / mu;
    const double slip_uniform = std::sqrt(sc.permeability) / sc.alpha_bj;

    // index maps of the n x n MAC box and the porous square (grid.hpp:28-36,71-78)
    const int nu_ = (n + 1) * n, nv_ = n * (n + 1), np_ = n * n;
    auto U = [&](int i, int j) { return j * (n + 1) + i; };
    auto V = [&](int i, int j) { return nu_ + j * n + i; };
    auto P = [&](int i, int j) { return nu_ + nv_ + j * n + i; };
    const int off_pm = nu_ + nv_ + np_;
    auto D = [&](int i, int j) { return off_pm + j * n + i; };
    auto K = [&](int i, int j) { return k_cell ? k_cell[j * n + i] : sc.permeability; };
    auto prev = [&](int dof) { return v_prev ? v_prev[dof] : 0.0; };

    Assembled out;
    out.n_u = nu_;
    out.n_vel = nu_ + nv_;
    out.n_pff = np_;
    out.n_ppm = np_;
    const int N = off_pm + np_;
    out.a = HostCsr(N, N);
    out.a.ci.reserve(static_cast<size_t>(8) * N);
    out.a.v.reserve(static_cast<size_t>(8) * N);
    out.rhs.assign(N, 0.0);
    RowSink row{&out.a};

    // x-momentum at vertical faces u(i, j)
    for (int j = 0; j < n; ++j) {
        for (int i = 0; i <= n; ++i) {
            const int r = U(i, j);
            const bool edge = (i == 0 || i == n);
            const double vol = h * h * (edge ? 0.5 : 1.0);
            const double len = edge ? 0.5 * h : h;
            const double c = mu * len / h;
            const bool inner_x = i > 0 && i < n;
            double& b = out.rhs[r];
            row.begin(r);
            if (tc != 0.0) {
                row.d(tc * vol);
                b += tc * vol * prev(r);
            }
            if (i < n) {  // east face: viscous flux + pressure
                row.o(U(i + 1, j), -2.0 * mu);
                row.d(2.0 * mu);
                row.o(P(i, j), h);
            } else {
                b -= p_out * h;
            }
            if (i > 0) {  // west face
                row.d(2.0 * mu);
                row.o(U(i - 1, j), -2.0 * mu);
                row.o(P(i - 1, j), -h);
            } else {
                b += p_in * h;
            }
            if (j + 1 < n) {  // north shear
                row.o(U(i, j + 1), -c);
                row.d(c);
            } else {  // no-slip lid over the half distance
                row.d(2.0 * c);
                b += 2.0 * c * 0.0;
            }
            if (inner_x) {
                row.o(V(i, j + 1), -c);
                row.o(V(i - 1, j + 1), c);
            }
            if (j > 0) {  // south shear
                row.d(c);
                row.o(U(i, j - 1), -c);
                if (inner_x) {
                    row.o(V(i, j), c);
                    row.o(V(i - 1, j), -c);
                }
            } else {  // Beavers-Joseph-Saffman slip at the interface
                double slip = slip_uniform;
                if (k_cell) {
                    const double kf = hmean(K(std::max(i - 1, 0), n - 1), K(std::min(i, n - 1), n - 1));
                    slip = std::sqrt(kf) / sc.alpha_bj;
                }
                row.d(mu * len / (0.5 * h + slip));
            }
            row.end();
        }
    }
    // y-momentum at horizontal faces v(i, j)
    for (int j = 0; j <= n; ++j) {
        for (int i = 0; i < n; ++i) {
            const int r = V(i, j);
            row.begin(r);
            if (j == 0) {  // interface: normal-stress continuity + half-cell resistance
                const double kom = k_cell ? K(i, n - 1) / mu : k_uniform;
                row.o(P(i, 0), h);
                row.d(2.0 * mu + h * h / (2.0 * kom));
                row.o(V(i, 1), -2.0 * mu);
                row.o(D(i, n - 1), -h);
                row.end();
                continue;
            }
            if (j == n) {  // lid: Dirichlet v = 0
                row.d(1.0);
                out.rhs[r] = 0.0;
                row.end();
                continue;
            }
            const double vol = h * h * 1.0;
            const double c = mu * h / h;
            if (tc != 0.0) {
                row.d(tc * vol);
                out.rhs[r] += tc * vol * prev(r);
            }
            row.o(V(i, j + 1), -2.0 * mu);  // north
            row.d(2.0 * mu);
            row.o(P(i, j), h);
            row.d(2.0 * mu);  // south
            row.o(V(i, j - 1), -2.0 * mu);
            row.o(P(i, j - 1), -h);
            if (i + 1 < n) {  // east shear (pressure sides contribute nothing)
                row.o(V(i + 1, j), -c);
                row.d(c);
            }
            row.o(U(i + 1, j), -c);
            row.o(U(i + 1, j - 1), c);
            if (i > 0) {  // west shear
                row.d(c);
                row.o(V(i - 1, j), -c);
            }
            row.o(U(i, j), c);
            row.o(U(i, j - 1), -c);
            row.end();
        }
    }
    // free-flow continuity (negated divergence), no gauge pin
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            row.begin(P(i, j));
            row.o(U(i + 1, j), -h);
            row.o(U(i, j), h);
            row.o(V(i, j + 1), -h);
            row.o(V(i, j), h);
            row.end();
        }
    // porous TPFA rows, no-flow outer sides, mass-flux coupling on top
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            row.begin(D(i, j));
            double diag = 0.0;
            auto face = [&](int ii, int jj) {
                const double t = k_cell ? hmean(K(i, j), K(ii, jj)) / mu : k_uniform;
                diag += t;
                row.o(D(ii, jj), -t);
            };
            if (i > 0) face(i - 1, j);
            if (i + 1 < n) face(i + 1, j);
            if (j > 0) face(i, j - 1);
            if (j + 1 < n)
                face(i, j + 1);
            else
                row.o(V(i, 0), h);
            row.d(diag);
            row.end();
        }
    return out;
}

// ---------------------------------------------------------------------------
// Partitioned subproblems (see setup.hpp).

LinearSystem assemble_stokes_dirichlet(const sdg_scenario& sc, const double* v_prev, const double* v_gamma) {
    if (!v_gamma) fail(SDG_EDIM, "assemble_stokes: interface data length mismatch");
    const Assembled m = assemble_monolithic(sc, nullptr, v_prev);
    const int n = sc.n, n_ff = m.n_vel + m.n_pff;
    LinearSystem s;
    s.a = HostCsr(n_ff, n_ff);
    s.rhs.assign(m.rhs.begin(), m.rhs.begin() + n_ff);
    for (int r = 0; r < n_ff; ++r) {
        const int vi = r - m.n_u;
        if (vi >= 0 && vi < n) {  // v(i, 0): Dirichlet row (assembly.cpp:137-141)
            s.a.ci.push_back(r);
            s.a.v.push_back(1.0);
            s.rhs[r] = v_gamma[vi];
        } else {
            for (int k = m.a.rp[r]; k < m.a.rp[r + 1]; ++k) {
                if (m.a.ci[k] >= n_ff) fail(SDG_EINVAL, "assemble_stokes: unexpected coupling column");
                s.a.ci.push_back(m.a.ci[k]);
                s.a.v.push_back(m.a.v[k]);
            }
        }
        s.a.rp[r + 1] = static_cast<int>(s.a.ci.size());
    }
    return s;
}

LinearSystem assemble_darcy_dirichlet(const sdg_scenario& sc, const double* p_gamma) {
    if (!p_gamma) fail(SDG_EDIM, "assemble_darcy: interface data length mismatch");
    const Assembled m = assemble_monolithic(sc, nullptr, nullptr);
    const int n = sc.n, n_ff = m.n_vel + m.n_pff, np_ = m.n_ppm;
    const double t2 = 2.0 * (sc.permeability / (sc.nu * sc.rho));
    LinearSystem s;
    s.a = HostCsr(np_, np_);
    s.rhs.assign(np_, 0.0);
    for (int r = 0; r < np_; ++r) {
        const int g = n_ff + r;
        const bool top = r >= (n - 1) * n;
        for (int k = m.a.rp[g]; k < m.a.rp[g + 1]; ++k) {
            const int c = m.a.ci[k];
            if (c < n_ff) continue;  // the coupled top face becomes Dirichlet
            double v = m.a.v[k];
            if (top && c == g) v += t2;  // diag accumulated W, E, S, then the top face
            s.a.ci.push_back(c - n_ff);
            s.a.v.push_back(v);
        }
        if (top) s.rhs[r] += t2 * p_gamma[r - (n - 1) * n];
        s.a.rp[r + 1] = static_cast<int>(s.a.ci.size());
    }
    return s;
}

void stokes_pressure_trace(const sdg_scenario& sc, const double* x, double* trace) {
    const int n = sc.n;
    const double h = 1.0 / n, mu = sc.nu * sc.rho;
    const int n_u = (n + 1) * n, n_vel = 2 * n * (n + 1);
    for (int i = 0; i < n; ++i) {
        const double dvdy = (x[n_u + n + i] - x[n_u + i]) / h;
        trace[i] = x[n_vel + i] - 2.0 * mu * dvdy;
    }
}

void darcy_velocity_trace(const sdg_scenario& sc, const double* p, const double* p_gamma, double* trace) {
    const int n = sc.n;
    const double h = 1.0 / n, k_over_mu = sc.permeability / (sc.nu * sc.rho);
    for (int i = 0; i < n; ++i) trace[i] = 2.0 * k_over_mu * (p[(n - 1) * n + i] - p_gamma[i]) / h;
}

}  // namespace sdg
