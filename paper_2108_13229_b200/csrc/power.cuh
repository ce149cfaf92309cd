// power_iteration (krylov.cpp:307-339) with the operator on the device.
// The start vector is drawn on the host with the reference's generator
// (std::mt19937 + std::uniform_real_distribution<double>(-1, 1)) and
// normalised there exactly as the reference does; iterations run on the GPU.
#pragma once

#include <cmath>
#include <random>
#include <vector>

#include "solver.hpp"

namespace sdg {

template <class Op>
PowerOut power_iteration(Context& c, int n, Op&& op, double tol_rel, int max_iters, unsigned seed) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    std::vector<double> xh(n);
    for (double& t : xh) t = dist(rng);
    double ss = 0.0;
    for (double t : xh) ss += t * t;
    double xn = std::sqrt(ss);
    if (xn == 0.0) xh[0] = xn = 1.0;
    const double inv = 1.0 / xn;
    for (double& t : xh) t *= inv;

    DevBuf<double> x(n), y(n), scal(2);
    ReduceWs ws;
    ws.init(reduce_blocks(n, c.num_sms), 2, c.stream);
    x.upload(xh.data(), n, c.stream);
    double* host = c.pinned->as<double>();

    PowerOut res;
    double prev = 0.0;
    for (int k = 0; k < max_iters; ++k) {
        op(x.get(), y.get());
        launch_dot(c, ws, n, x.get(), y.get(), scal.get());
        launch_norm2sq(c, ws, n, y.get(), scal.get() + 1);
        SDG_CUDA(cudaMemcpyAsync(host, scal.get(), 2 * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        const double lambda = host[0];
        const double yn = std::sqrt(host[1]);
        res.value = lambda;
        res.iterations = k + 1;
        if (k > 0 && std::abs(lambda - prev) <= tol_rel * std::abs(lambda)) {
            res.converged = true;
            return res;
        }
        prev = lambda;
        if (yn == 0.0) {
            res.value = 0.0;
            res.converged = true;
            return res;
        }
        // x = y / ||y||: put the norm (not its square) on the device first
        host[2] = yn;
        SDG_CUDA(cudaMemcpyAsync(scal.get(), &host[2], sizeof(double), cudaMemcpyHostToDevice, c.stream));
        launch_div_scalar(c, n, y.get(), scal.get(), x.get());
        c.sync();  // host[2] is reused next iteration
    }
    return res;
}

}  // namespace sdg
