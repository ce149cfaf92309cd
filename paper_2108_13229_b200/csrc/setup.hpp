// Host-side setup that feeds the device: block extraction, aggregation AMG
// hierarchy (aggregation + Galerkin), Gauss-Seidel level schedules and the
// monolithic assembly used to produce bench inputs.  All of it is host C++
// (setup stays host, consumed by the GPU).
#pragma once

#include <functional>
#include <vector>

#include "common.hpp"

namespace sdg {

// sparse.cpp:110-127
HostCsr submatrix(const HostCsr& a, int row_begin, int row_end, int col_begin, int col_end);
// precond.cpp:375-392
HostCsr ground_dof(const HostCsr& a, int dof);
// ILU(0) factors (precond.cpp:13-87, bitwise): strict lower L, upper U with the diagonal first in each row
void ilu0_factor(const HostCsr& a, HostCsr& lower, HostCsr& upper);

struct AmgOpts {
    int max_levels = 3;
    double theta = 0.08;
    int coarse_threshold = 100;
    std::vector<int> components;
};

// One level of the aggregation hierarchy (precond.hpp:77-95).
struct HostLevel {
    HostCsr a;
    std::vector<int> aggregate_of;  // empty on the coarsest level
    int n_coarse = 0;
    std::vector<int> components;    // dof labels of this level (empty: scalar)
};

// amg_setup (precond.cpp:189-217) without the coarse factorization, which
// the device performs (dense LU -> explicit inverse, see precond.cu).
// `product` computes each Galerkin product (default: the host galerkin below;
// the device preconditioners pass galerkin_device, galerkin.cu).
using GalerkinFn = std::function<HostCsr(const HostCsr&, const std::vector<int>&, int)>;
std::vector<HostLevel> build_hierarchy(const HostCsr& a, const AmgOpts& o, const GalerkinFn& product = {});

// Restatement of the greedy aggregation (precond.cpp:122-175).
std::vector<int> aggregate(const HostCsr& a, double theta, const std::vector<int>& comps,
                           int& n_aggregates);
// Restatement of galerkin_product (precond.cpp:177-185), bitwise identical:
// duplicates summed in COO insertion order.
HostCsr galerkin(const HostCsr& a, const std::vector<int>& agg, int n_coarse);
// The same product on the device (galerkin.cu), bitwise equal; returns the host copy.
struct Context;
HostCsr galerkin_device(Context& cx, const HostCsr& a, const std::vector<int>& agg, int n_coarse);

// Level schedule of the strict lower triangle: rows grouped by dependency
// depth so that one level's rows can be relaxed concurrently while the
// lexicographic Gauss-Seidel recurrence of precond.cpp:92-108 is preserved
// exactly (every lower neighbour lies in an earlier level).
struct LevelSchedule {
    std::vector<int> lvl_ptr;   // n_levels + 1
    std::vector<int> lvl_rows;  // rows sorted by (level, row)
    int n_levels() const { return static_cast<int>(lvl_ptr.size()) - 1; }
};
LevelSchedule lower_schedule(const HostCsr& a);
// Throws SDG_ESINGULAR "sor_sweep: zero diagonal in row i" when a row has no
// nonzero stored diagonal (the reference throws the same at apply time).
void require_diagonal(const HostCsr& a, const char* who);

// Transpose of the aggregation map as CSR: coarse c -> fine rows, ascending.
void aggregate_transpose(const std::vector<int>& agg, int n_coarse, std::vector<int>& ptr,
                         std::vector<int>& rows);

// assemble_monolithic (assembly.cpp:327-380) on the n x n free-flow box, with
// an optional per-cell porous permeability field (extension).
struct Assembled {
    HostCsr a;
    std::vector<double> rhs;
    int n_u = 0, n_vel = 0, n_pff = 0, n_ppm = 0;
};
Assembled assemble_monolithic(const sdg_scenario& sc, const double* k_cell, const double* v_prev);

// The partitioned subproblems (coupling.cpp:218-242) on the same boxes:
// assemble_stokes(ff box, ..., &v_gamma) -- Dirichlet normal velocities on the
// interface, slip for the tangential ones (assembly.cpp:134-141, 115-130) --
// and assemble_darcy(pm box, K/mu, {}, &p_gamma) -- Dirichlet interface
// pressures (assembly.cpp:268-270).  Derived from the monolithic rows, which
// they share everywhere else, so uniform-K results are bitwise the reference's.
struct LinearSystem {
    HostCsr a;
    std::vector<double> rhs;
};
LinearSystem assemble_stokes_dirichlet(const sdg_scenario& sc, const double* v_prev, const double* v_gamma);
LinearSystem assemble_darcy_dirichlet(const sdg_scenario& sc, const double* p_gamma);
// stokes_pressure_trace (assembly.cpp:382-391) / darcy_velocity_trace_dirichlet (:393-402)
void stokes_pressure_trace(const sdg_scenario& sc, const double* x_ff, double* trace);
void darcy_velocity_trace(const sdg_scenario& sc, const double* p, const double* p_gamma, double* trace);

}  // namespace sdg
