// Device kernels of the hot path and their launchers.  All arithmetic fp64,
// int32 indices.  Kernels marked BITWISE reproduce the reference's CPU loop
// operation-for-operation (no FMA contraction: __dmul_rn/__dadd_rn/__dsub_rn),
// so their outputs equal the reference's bit for bit on the same inputs.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"

namespace sdg {

// Deterministic reductions write their per-block partials here and the last
// block to finish folds them in a fixed order.
struct ReduceWs {
    DevBuf<double> partials;    // max_blocks * max_vals
    DevBuf<unsigned> ticket;    // one arrival counter
    int max_blocks = 0;
    int max_vals = 0;
    void init(int blocks, int vals, cudaStream_t s);
};

// Scalars of one BiCGSTAB run (device resident; the host reads a copy once
// per iteration).
struct BiState {
    double rho, alpha, omega, rho_new;
    double rv, sn, tt, ts, rn, tn;
    double tol;
    int flag;
    int pad;
};
enum BiFlag { BI_OK = 0, BI_BREAK_RHO = 1, BI_BREAK_RV = 2, BI_S_CONV = 3, BI_BREAK_TT = 4, BI_BREAK_OMEGA = 5 };

int reduce_blocks(int n, int num_sms);

// ---- sparse -------------------------------------------------------------
// BITWISE spmv / spmv_add: y = A x, or y_out = y_in + alpha (A x).
void launch_spmv(Context& c, const DevCsr& a, const double* x, double* y);
// y = A x with x[j] read as packed[bidx[j]] (a Gauss-Seidel walk's staged b), CSR order
void launch_spmv_packed(Context& c, const DevCsr& a, const int* bidx, const double* packed, double* y);
void launch_spmv_add(Context& c, const DevCsr& a, const double* x, const double* y_in,
                     double* y_out, double alpha);
// BITWISE forward SOR sweep over a level schedule; z_old may be null (zero).
void launch_gs_levels(Context& c, const DevCsr& a, const int* lvl_ptr, const int* lvl_rows,
                      int n_levels, const double* r, const double* z_old, double* z_new,
                      double omega);
// BITWISE fused residual + restriction: rc[c] = sum_{i in agg c, ascending} (r - A z)_i.
void launch_resid_restrict(Context& c, const DevCsr& a, const int* pt_ptr, const int* pt_rows,
                           int n_coarse, const double* r, const double* z, double* rc);
// BITWISE prolongation: out[i] = z[i] + zc[agg[i]].
void launch_prolong(Context& c, int n, const int* agg, const double* z, const double* zc,
                    double* out);
// Dense coarse solve y = Ainv x (row-major Ainv).
void launch_dense_gemv(Context& c, int n, const double* ainv, const double* x, double* y);
// z -= K w, K column-major n x m (td_bgs interface response, BlockPrecond)
// z -= K w, K column-major n x m; w is staged in shared memory, so m is bounded
constexpr int kColmajorMaxGamma = 24576;
void launch_colmajor_gemv_sub(Context& c, int n, int m, const double* kmat, const double* w, double* z);
// BITWISE Uzawa pressure step: z_p[i] = omega (sum_k C_ik z_v[k] - r_p[i]).
void launch_uzawa_pressure(Context& c, const DevCsr& cm, const double* z_v, const double* r_p,
                           double omega, double* z_p);
void launch_copy(Context& c, double* dst, const double* src, int64_t n);
void launch_fill(Context& c, double* dst, double v, int64_t n);
// dense scatter of a CSR into a zeroed row-major n x n buffer
void launch_csr_to_dense(Context& c, const DevCsr& a, double* dense);
void launch_set_identity(Context& c, int n, double* dense);

// ---- Krylov vector kernels ------------------------------------------------
// out[v] = sum_i x_v[i] * y[i] for v < k, x_v = X + v*ldx (deterministic).
void launch_multidot(Context& c, ReduceWs& ws, int64_t n, int k, const double* X, int64_t ldx,
                     const double* y, double* out);
// w -= sum_v h[v] X_v  (h in device memory)
void launch_multi_axpy(Context& c, int64_t n, int k, const double* X, int64_t ldx,
                       const double* h, double* w);
// w -= sum_v h[v] X_v, then out[0] = ||w||_2 (the norm itself)
void launch_multi_axpy_norm2(Context& c, ReduceWs& ws, int64_t n, int k, const double* X,
                             int64_t ldx, const double* h, double* w, double* out);
// dst = src * (1/den[0]) when den[0] > 0  (reference: scale(v, 1.0 / wn))
void launch_scale_by_inv(Context& c, int64_t n, const double* src, const double* den, double* dst);
// BITWISE w = sum_{v<k} y[v] X_v, sequential in v from 0.0 (fill + axpy loop)
void launch_lincomb(Context& c, int64_t n, int k, const double* X, int64_t ldx, const double* y,
                    double* w);
// BITWISE x += z
void launch_add_inplace(Context& c, int64_t n, double* x, const double* z);
// BITWISE y += alpha x  (axpy, sparse.cpp:216-218); alpha from device
void launch_axpy_dev(Context& c, int64_t n, const double* alpha, const double* x, double* y);
// out[0] = ||x||^2 (deterministic)
void launch_norm2sq(Context& c, ReduceWs& ws, int64_t n, const double* x, double* out);
void launch_dot(Context& c, ReduceWs& ws, int64_t n, const double* x, const double* y, double* out);
// BITWISE x = y / yn[0]  (power iteration normalisation, krylov.cpp:337)
void launch_div_scalar(Context& c, int64_t n, const double* y, const double* yn, double* x);

// ---- fused BiCGSTAB steps (krylov.cpp:240-283) -----------------------------
void launch_bi_p(Context& c, int64_t n, BiState* st, const double* r, const double* v, double* p);
void launch_bi_rv(Context& c, ReduceWs& ws, int64_t n, BiState* st, const double* rhat,
                  const double* v);
void launch_bi_s(Context& c, ReduceWs& ws, int64_t n, BiState* st, const double* r,
                 const double* v, double* s);
void launch_bi_t(Context& c, ReduceWs& ws, int64_t n, BiState* st, const double* t,
                 const double* s);
void launch_bi_xr(Context& c, ReduceWs& ws, int64_t n, BiState* st, const double* phat,
                  const double* shat, const double* s, const double* t, const double* rhat,
                  double* x, double* r);
// restart helpers: rho_new = dot(rhat, r) into st
void launch_bi_rho(Context& c, ReduceWs& ws, int64_t n, BiState* st, const double* rhat,
                   const double* r);
void launch_bi_x_alpha(Context& c, int64_t n, BiState* st, const double* phat, double* x);

}  // namespace sdg
