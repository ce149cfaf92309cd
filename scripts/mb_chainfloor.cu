// Dev micro-benchmark: latency floor of the lane-chain lower solve (no record
// loads; coefficients constant), one CTA of W warps.  Cross-warp values go
// through a shared array with a NaN sentinel as the per-value flag (no
// fences).  Prints cycles per step.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double ld_vol(const double* p) {
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}

template <int U, int MODE>
__global__ void k_floor(int nx, int ny, double* out, long long* cyc) {
    extern __shared__ double bnd[];  // [warps][nx]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = threadIdx.x; k < nw * nx; k += blockDim.x) bnd[k] = __longlong_as_double(0x7ff4000000000000ull);
    __syncthreads();
    long long t0 = clock64();
    const double cw = -0.25, cs = -0.24;
    double west = 0.0, zl = 0.0, acc = 0.0;
    const int steps = nx + 31;
    const double* src = w > 0 ? bnd + (w - 1) * nx : nullptr;
    double* dst = bnd + w * nx;
    for (int s0 = 0; s0 < steps; s0 += U) {
        double bv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = s0 + u;
            bv[u] = 0.0;
            if (MODE == 0) {
                if (lane == 0 && w > 0 && c < nx) {
                    double v;
                    do { v = ld_vol(src + c); } while (__double_as_longlong(v) == 0x7ff4000000000000ll);
                    bv[u] = v;
                }
            } else if (MODE == 1) {  // no wait (timing only)
                if (lane == 0 && w > 0 && c < nx) bv[u] = ld_vol(src + c);
            } else {  // whole warp spins on the same address (uniform)
                if (w > 0 && c < nx) {
                    double v;
                    do { v = ld_vol(src + c); } while (__double_as_longlong(v) == 0x7ff4000000000000ll);
                    bv[u] = lane == 0 ? v : 0.0;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int s = s0 + u;
            double south = __shfl_up_sync(0xffffffffu, zl, 1);
            if (lane == 0) south = bv[u];
            const int i = s - lane;
            double v = fma(cs, south, 1.0);
            v = fma(cw, west, v);
            const bool act = i >= 0 && i < nx;
            v = act ? v : 0.0;
            zl = v;
            west = v;
            acc += v;
            if (lane == 31 && act) dst[i] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[0] = clock64() - t0;
    out[threadIdx.x] = acc;
}

int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 8 * 1024);
    cudaMalloc(&c, 8);
    int nxs[] = {160, 500};
    for (int nx : nxs) {
        for (int nw : {1, 2, 5, 16}) {
            const int ny = 32 * nw;
            long long h = 0;
            const int depth = nx + ny - 1;
            for (int r = 0; r < 3; ++r) k_floor<4, 0><<<1, 32 * nw, nw * nx * 8>>>(nx, ny, o, c);
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("lane0-spin nx=%d warps=%2d: %.1f per step %s\n", nx, nw, (double)h / depth, cudaGetErrorString(cudaDeviceSynchronize()));
            for (int r = 0; r < 3; ++r) k_floor<4, 1><<<1, 32 * nw, nw * nx * 8>>>(nx, ny, o, c);
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("no-wait    nx=%d warps=%2d: %.1f per step\n", nx, nw, (double)h / depth);
            for (int r = 0; r < 3; ++r) k_floor<4, 2><<<1, 32 * nw, nw * nx * 8>>>(nx, ny, o, c);
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("warp-spin  nx=%d warps=%2d: %.1f per step\n", nx, nw, (double)h / depth);
        }
    }
    return 0;
}
