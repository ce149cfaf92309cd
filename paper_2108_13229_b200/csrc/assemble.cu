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


// ---------------------------------------------------------------------------
// Device assembly of the monolithic matrix (assembly.cpp:17-286 through
// assemble_monolithic, assembly.cpp:327-380, on the n x n box of setup.cpp).
// One thread per row emits the row's contributions in the host's order - the
// off-diagonal (column, value) pairs, the diagonal as a running sum from 0.0
// in emission order, which is what the reference's CooBuilder produces
// (sparse.cpp:55-79) - with every operation explicitly rounded (no FMA
// contraction), then sorts the at most 12 entries by column.  Pass 1 counts
// the entries of a row, a three-kernel scan turns the counts into row offsets,
// pass 2 writes columns and values: bitwise the host CSR (test_host / GPU test).
struct AsmParams {
    int n;
    double h, mu, tc, permeability, alpha_bj, k_uniform, slip_uniform;
    const double* k_cell;  // [n * n] or null
};

struct RowOut {
    int c[12];
    double v[12];
    int k = 0;
    double diag = 0.0;
    bool has_diag = false;
    __device__ void o(int col, double x) {
        c[k] = col;
        v[k] = x;
        ++k;
    }
    __device__ void d(double x) {
        diag = __dadd_rn(diag, x);
        has_diag = true;
    }
};

__device__ __forceinline__ double asm_hmean(double ka, double kb) {
    return ka == kb ? ka : __ddiv_rn(__dmul_rn(__dmul_rn(2.0, ka), kb), __dadd_rn(ka, kb));
}

__device__ void asm_emit_row(const AsmParams& P, int r, RowOut& row) {
    const int n = P.n;
    const double h = P.h, mu = P.mu, tc = P.tc;
    const int nu_ = (n + 1) * n, nv_ = n * (n + 1), np_ = n * n, off_pm = nu_ + nv_ + np_;
    auto U = [&](int i, int j) { return j * (n + 1) + i; };
    auto V = [&](int i, int j) { return nu_ + j * n + i; };
    auto Pr = [&](int i, int j) { return nu_ + nv_ + j * n + i; };
    auto D = [&](int i, int j) { return off_pm + j * n + i; };
    auto K = [&](int i, int j) { return P.k_cell ? P.k_cell[j * n + i] : P.permeability; };
    const double two_mu = __dmul_rn(2.0, mu);
    if (r < nu_) {  // x-momentum at u(i, j)
        const int i = r % (n + 1), j = r / (n + 1);
        const bool edge = (i == 0 || i == n);
        const double vol = __dmul_rn(__dmul_rn(h, h), edge ? 0.5 : 1.0);
        const double len = edge ? __dmul_rn(0.5, h) : h;
        const double c = __ddiv_rn(__dmul_rn(mu, len), h);
        const bool inner_x = i > 0 && i < n;
        if (tc != 0.0) row.d(__dmul_rn(tc, vol));
        if (i < n) {
            row.o(U(i + 1, j), -two_mu);
            row.d(two_mu);
            row.o(Pr(i, j), h);
        }
        if (i > 0) {
            row.d(two_mu);
            row.o(U(i - 1, j), -two_mu);
            row.o(Pr(i - 1, j), -h);
        }
        if (j + 1 < n) {
            row.o(U(i, j + 1), -c);
            row.d(c);
        } else {
            row.d(__dmul_rn(2.0, c));
        }
        if (inner_x) {
            row.o(V(i, j + 1), -c);
            row.o(V(i - 1, j + 1), c);
        }
        if (j > 0) {
            row.d(c);
            row.o(U(i, j - 1), -c);
            if (inner_x) {
                row.o(V(i, j), c);
                row.o(V(i - 1, j), -c);
            }
        } else {
            double slip = P.slip_uniform;
            if (P.k_cell) {
                const double kf = asm_hmean(K(max(i - 1, 0), n - 1), K(min(i, n - 1), n - 1));
                slip = __ddiv_rn(__dsqrt_rn(kf), P.alpha_bj);
            }
            row.d(__ddiv_rn(__dmul_rn(mu, len), __dadd_rn(__dmul_rn(0.5, h), slip)));
        }
    } else if (r < nu_ + nv_) {  // y-momentum at v(i, j)
        const int q = r - nu_, i = q % n, j = q / n;
        if (j == 0) {
            const double kom = P.k_cell ? __ddiv_rn(K(i, n - 1), mu) : P.k_uniform;
            row.o(Pr(i, 0), h);
            row.d(__dadd_rn(two_mu, __ddiv_rn(__dmul_rn(h, h), __dmul_rn(2.0, kom))));
            row.o(V(i, 1), -two_mu);
            row.o(D(i, n - 1), -h);
            return;
        }
        if (j == n) {
            row.d(1.0);
            return;
        }
        const double vol = __dmul_rn(__dmul_rn(h, h), 1.0);
        const double c = __ddiv_rn(__dmul_rn(mu, h), h);
        if (tc != 0.0) row.d(__dmul_rn(tc, vol));
        row.o(V(i, j + 1), -two_mu);
        row.d(two_mu);
        row.o(Pr(i, j), h);
        row.d(two_mu);
        row.o(V(i, j - 1), -two_mu);
        row.o(Pr(i, j - 1), -h);
        if (i + 1 < n) {
            row.o(V(i + 1, j), -c);
            row.d(c);
        }
        row.o(U(i + 1, j), -c);
        row.o(U(i + 1, j - 1), c);
        if (i > 0) {
            row.d(c);
            row.o(V(i - 1, j), -c);
        }
        row.o(U(i, j), c);
        row.o(U(i, j - 1), -c);
    } else if (r < off_pm) {  // free-flow continuity (negated divergence)
        const int q = r - nu_ - nv_, i = q % n, j = q / n;
        row.o(U(i + 1, j), -h);
        row.o(U(i, j), h);
        row.o(V(i, j + 1), -h);
        row.o(V(i, j), h);
    } else {  // porous TPFA rows
        const int q = r - off_pm, i = q % n, j = q / n;
        double diag = 0.0;
        auto face = [&](int ii, int jj) {
            const double t = P.k_cell ? __ddiv_rn(asm_hmean(K(i, j), K(ii, jj)), mu) : P.k_uniform;
            diag = __dadd_rn(diag, t);
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
    }
}

// pass 1 (rowptr_out == the counts array, col == null): entries per row;
// pass 2: columns and values at the row's offset, sorted by column
__global__ void k_assemble_matrix(AsmParams P, int n_total, const int* __restrict__ rowptr, int* __restrict__ counts,
                                  int* __restrict__ col, double* __restrict__ val) {
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_total) return;
    RowOut row;
    asm_emit_row(P, r, row);
    if (row.has_diag) row.o(r, row.diag);
    if (counts) {
        counts[r] = row.k;
        return;
    }
    for (int a = 1; a < row.k; ++a) {  // insertion sort by column (columns are unique within a row)
        const int cc = row.c[a];
        const double vv = row.v[a];
        int b = a - 1;
        while (b >= 0 && row.c[b] > cc) {
            row.c[b + 1] = row.c[b];
            row.v[b + 1] = row.v[b];
            --b;
        }
        row.c[b + 1] = cc;
        row.v[b + 1] = vv;
    }
    const int base = rowptr[r];
    for (int a = 0; a < row.k; ++a) {
        col[base + a] = row.c[a];
        val[base + a] = row.v[a];
    }
}

// exclusive scan of counts[0, n) into out[0, n], three kernels: per-block
// sums, a one-block scan of the sums, per-block scan plus offset
constexpr int kScanBlock = 1024;
__global__ void k_scan_block_sums(const int* __restrict__ in, int n, int* __restrict__ sums) {
    pdl_begin();
    __shared__ int sh[32];
    const int i = blockIdx.x * kScanBlock + threadIdx.x;
    int v = i < n ? in[i] : 0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        int w = sh[threadIdx.x];
        for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (threadIdx.x == 0) sums[blockIdx.x] = w;
    }
}
__global__ void k_scan_sums(int* __restrict__ sums, int nb) {  // one block: exclusive scan in place, total at sums[nb]
    pdl_begin();
    __shared__ int carry;
    __shared__ int sh[kScanBlock];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += kScanBlock) {
        const int i = base + threadIdx.x;
        const int v = i < nb ? sums[i] : 0;
        sh[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < kScanBlock; o <<= 1) {
            const int t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
            __syncthreads();
            sh[threadIdx.x] += t;
            __syncthreads();
        }
        if (i < nb) sums[i] = carry + sh[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 0) carry += sh[kScanBlock - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[nb] = carry;
}
__global__ void k_scan_apply(const int* __restrict__ in, int n, const int* __restrict__ sums, int* __restrict__ out) {
    pdl_begin();
    __shared__ int sh[kScanBlock];
    const int i = blockIdx.x * kScanBlock + threadIdx.x;
    const int v = i < n ? in[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < kScanBlock; o <<= 1) {
        const int t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
        __syncthreads();
        sh[threadIdx.x] += t;
        __syncthreads();
    }
    if (i < n) out[i] = sums[blockIdx.x] + sh[threadIdx.x] - v;
    if (i == n - 1) out[n] = sums[blockIdx.x] + sh[threadIdx.x];
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

// Device assembly of the monolithic matrix: row offsets into rowptr_dev
// [n_total + 1], then - when the caller's capacity holds them - columns and
// values.  Returns the number of entries (one 4-byte read-back).
int64_t assemble_matrix_device(Context& c, const sdg_scenario& sc, const double* k_cell_dev, int* rowptr_dev,
                               int* col_dev, double* val_dev, int64_t capacity) {
    const int n = sc.n;
    if (n < 1) fail(SDG_EDIM, "assemble_matrix_device: n must be positive");
    const int64_t nt64 = 2 * static_cast<int64_t>(n) * (n + 1) + 2 * static_cast<int64_t>(n) * n;
    if (12 * nt64 > INT32_MAX) fail(SDG_EDIM, "assemble_matrix_device: the matrix does not fit int32 offsets");
    const int n_total = static_cast<int>(nt64);
    AsmParams P{};
    P.n = n;
    P.h = 1.0 / n;
    P.mu = sc.nu * sc.rho;
    P.tc = std::isfinite(sc.dt) ? sc.rho / sc.dt : 0.0;
    P.permeability = sc.permeability;
    P.alpha_bj = sc.alpha_bj;
    P.k_uniform = sc.permeability / P.mu;                       // host values, as setup.cpp
    P.slip_uniform = std::sqrt(sc.permeability) / sc.alpha_bj;
    P.k_cell = k_cell_dev;
    const int nb = (n_total + kScanBlock - 1) / kScanBlock;
    DevBuf<int> counts(n_total), sums(nb + 1);
    {
        ProfScope ps_(c, PF_VEC, 4.0 * n_total);
        launch_k(c, k_assemble_matrix, (n_total + 255) / 256, 256, 0, P, n_total, static_cast<const int*>(nullptr),
                 counts.get(), static_cast<int*>(nullptr), static_cast<double*>(nullptr));
        c.count();
    }
    launch_k(c, k_scan_block_sums, nb, kScanBlock, 0, static_cast<const int*>(counts.get()), n_total, sums.get());
    launch_k(c, k_scan_sums, 1, kScanBlock, 0, sums.get(), nb);
    launch_k(c, k_scan_apply, nb, kScanBlock, 0, static_cast<const int*>(counts.get()), n_total,
             static_cast<const int*>(sums.get()), rowptr_dev);
    c.count(3);
    int nnz = 0;
    SDG_CUDA(cudaMemcpyAsync(&nnz, sums.get() + nb, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (col_dev && val_dev && capacity >= nnz) {
        ProfScope ps_(c, PF_VEC, 12.0 * nnz + 4.0 * n_total);
        launch_k(c, k_assemble_matrix, (n_total + 255) / 256, 256, 0, P, n_total, static_cast<const int*>(rowptr_dev),
                 static_cast<int*>(nullptr), col_dev, val_dev);
        c.count();
        c.sync();
    }
    return nnz;
}

}  // namespace sdg

