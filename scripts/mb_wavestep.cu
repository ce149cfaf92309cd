// Dev micro-benchmark: cycles per step of the MAC wavefront's register chain
// (no record loads, no stores): which part of the ~275 cycles per step of
// k_gs_wave<2> is the dependent chain shuffle -> select -> DFMA -> DFMA.
//   A: three 64-bit shuffles, selects for lane 0, 8 DFMA + 1 DADD (the kernel's step)
//   B: two shuffles (u(i-1, j-1) kept from the previous step)
//   C: B without the lane-0 selects
//   D: the u chain alone (one shuffle, two DFMA)
//   E: D with the shuffle split in two independent 32-bit halves issued back to back (same thing, reference)
//   F: B + 10 LDS.128 per two steps (records from shared memory)
// nvcc -arch=sm_100a -O3 -o mb_wavestep mb_wavestep.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_step(long long* out, double* sink, int n) {
    extern __shared__ double2 rec[];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 10 * 4 * 32; i += blockDim.x) rec[i] = make_double2(1e-3 * (i % 7), -1e-3 * (i % 5));
    __syncthreads();
    double u_last = sink[0], u_last2 = 0.0, v_last = sink[1], su_prev = 0.0;
    const double c0 = 1e-3 + sink[2], c1 = -0.25 + sink[3], c2 = -0.24, c3 = 2e-3, c4 = -0.1, c5 = -0.11, c6 = -0.12,
                 c7 = -0.13, c8 = -0.2, c9 = -0.21;
    const double bnd = sink[4];
    long long t0 = clock64();
    for (int s = 0; s < n; s += 2) {
        double2 R[10];
        if (MODE == 5) {
#pragma unroll
            for (int f = 0; f < 10; ++f) R[f] = rec[(f * 4 + ((s >> 1) & 3)) * 32 + lane];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            auto r = [&](int f, double c) { return MODE == 5 ? (h ? R[f].y : R[f].x) : c; };
            if (MODE == 3) {
                double su1 = __shfl_up_sync(0xffffffffu, u_last, 1);
                u_last = fma(c2, u_last, fma(c1, su1, c0));
                continue;
            }
            double su1 = __shfl_up_sync(0xffffffffu, u_last, 1);
            double su2 = MODE == 0 ? __shfl_up_sync(0xffffffffu, u_last2, 1) : su_prev;
            double sv1 = __shfl_up_sync(0xffffffffu, v_last, 1);
            if (MODE != 2 && lane == 0) {
                su1 = bnd;
                if (MODE == 0) su2 = bnd;
                sv1 = bnd;
            }
            su_prev = su1;
            const double un = fma(r(2, c2), u_last, fma(r(1, c1), su1, r(0, c0)));
            double acc = fma(r(4, c4), su2, 0.0);
            acc = fma(r(5, c5), su1, acc);
            acc = fma(r(6, c6), u_last, acc);
            acc = fma(r(7, c7), un, acc);
            const double vn = fma(r(9, c9), v_last, fma(r(8, c8), sv1, r(3, c3) + acc));
            u_last2 = u_last;
            u_last = un;
            v_last = vn;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[8 + threadIdx.x] = u_last + v_last + u_last2 + su_prev;
}

int main() {
    long long* d;
    double* sink;
    cudaMalloc(&d, 8);
    cudaMalloc(&sink, 4096 * 8);
    cudaMemset(sink, 0, 4096 * 8);
    const int n = 8192;
    const char* names[] = {"A 3 shfl + sel", "B 2 shfl + sel", "C 2 shfl no sel", "D u chain only", "-", "F B + LDS records"};
    auto run = [&](int mode, void (*k)(long long*, double*, int)) {
        for (int rep = 0; rep < 2; ++rep) k<<<1, 32, 10 * 4 * 32 * 16>>>(d, sink, n);
        long long c;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("%-20s %7.1f cycles/step\n", names[mode], double(c) / n);
    };
    run(0, k_step<0>);
    run(1, k_step<1>);
    run(2, k_step<2>);
    run(3, k_step<3>);
    run(5, k_step<5>);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
