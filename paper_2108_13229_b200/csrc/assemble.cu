// Device assembly of the monolithic right-hand side (assembly.cpp:327-380,
// restated bitwise by setup.cpp assemble_monolithic).  The matrix of the
// coupled system is step-invariant (the implicit-Euler mass term tc vol sits
// on the diagonal of every step), so the only per-step
// assembly of BASELINE config 4 is the right-hand side, which reads the
// previous velocity: one kernel over the velocity rows instead of a host
// re-assembly and a host-to-device copy per time step.  Every row repeats the
// host's operation sequence with explicitly rounded operations (no FMA
// contraction), so the result is bitwise the host's.
#include "launch.cuh"
#include "solver.hpp"

#include <cmath>

namespace sdg {

namespace {

// u(i, j) row r = j (n+1) + i: b = 0 [+ tc vol u_prev] [- p_out h (i = n)] [+ p_in h (i = 0)]
// [+ 2 c 0 (j = n - 1)];  v(i, j), 0 < j < n: b = 0 + tc h^2 v_prev;  every other row 0
__global__ void k_assemble_rhs(int n, int n_total, double h, double mu, double tc, double p_in, double p_out,
                               const double* __restrict__ prev, double* __restrict__ rhs) {
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_total) return;
    const int nu = (n + 1) * n, nv = n * (n + 1);
    double b = 0.0;
    if (r < nu) {
        const int i = r % (n + 1), j = r / (n + 1);
        const bool edge = (i == 0 || i == n);
        const double vol = __dmul_rn(__dmul_rn(h, h), edge ? 0.5 : 1.0);
        const double len = edge ? __dmul_rn(0.5, h) : h;
        const double c = __ddiv_rn(__dmul_rn(mu, len), h);
        if (tc != 0.0) b = __dadd_rn(b, __dmul_rn(__dmul_rn(tc, vol), prev ? prev[r] : 0.0));
        if (i == n) b = __dsub_rn(b, __dmul_rn(p_out, h));
        if (i == 0) b = __dadd_rn(b, __dmul_rn(p_in, h));
        if (j + 1 == n) b = __dadd_rn(b, __dmul_rn(__dmul_rn(2.0, c), 0.0));
    } else if (r < nu + nv) {
        const int q = r - nu, j = q / n;
        if (j > 0 && j < n && tc != 0.0) {
            const double vol = __dmul_rn(__dmul_rn(h, h), 1.0);
            b = __dadd_rn(b, __dmul_rn(__dmul_rn(tc, vol), prev ? prev[r] : 0.0));
        }
    }
    rhs[r] = b;
}

}  // namespace

void launch_assemble_rhs(Context& c, const sdg_scenario& sc, const double* v_prev, double* rhs) {
    const int n = sc.n;
    if (n < 1) fail(SDG_EDIM, "assemble_rhs: n must be positive");
    const int n_total = 2 * n * (n + 1) + 2 * n * n;
    const double h = 1.0 / n;
    const double mu = sc.nu * sc.rho;
    const double tc = std::isfinite(sc.dt) ? sc.rho / sc.dt : 0.0;
    const double p_in = sc.dp_max * 0.5 * (1.0 - std::cos(M_PI * sc.t / sc.t_end));  // host, as setup.cpp
    ProfScope ps_(c, PF_VEC, 8.0 * (2 * n * (n + 1)) + 8.0 * n_total);
    launch_k(c, k_assemble_rhs, (n_total + 255) / 256, 256, 0, n, n_total, h, mu, tc, p_in, 0.0, v_prev, rhs);
    c.count();
}

}  // namespace sdg
