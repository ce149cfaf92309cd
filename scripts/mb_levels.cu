// Dev micro-benchmark: per-level cost of a single-CTA level walk on B200.
// Variants: barrier only; + smem gather/FMA chain; named-barrier variant.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_bar_only(int levels, long long* out) {
    long long t0 = clock64();
    for (int l = 0; l < levels; ++l) __syncthreads();
    if (threadIdx.x == 0) out[0] = clock64() - t0;
}

__global__ void k_chain(int levels, int width, long long* out, double* sink) {
    __shared__ double ring[4096];
    const int t = threadIdx.x;
    for (int i = t; i < 4096; i += blockDim.x) ring[i] = 1.0 + i * 1e-6;
    __syncthreads();
    long long t0 = clock64();
    double v[8];
    int s[8];
    for (int k = 0; k < 8; ++k) {
        v[k] = 0.1 * (k + 1);
        s[k] = (t * 7 + k * 131) & 4095;
    }
    for (int l = 0; l < levels; ++l) {
        if (t < width) {
            double p[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) p[k] = v[k] * ring[s[k]];
            double acc = 1.0 - (((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7])));
            ring[(l * width + t) & 4095] = acc * 1e-3;
#pragma unroll
            for (int k = 0; k < 8; ++k) s[k] = (s[k] + width) & 4095;
        }
        __syncthreads();
    }
    if (t == 0) out[0] = clock64() - t0;
    if (t == 0) sink[0] = ring[5];
}

__global__ void k_chain2(int levels, int width, long long* out, double* sink) {
    __shared__ double ring[4096];
    const int t = threadIdx.x;
    for (int i = t; i < 4096; i += blockDim.x) ring[i] = 1.0 + i * 1e-6;
    __syncthreads();
    long long t0 = clock64();
    double v0 = 0.3, v1 = 0.2;
    int s0 = (t * 7) & 4095, s1 = (t * 7 + 1) & 4095;
    for (int l = 0; l < levels; ++l) {
        if (t < width) {
            double acc = 1.0 - fma(v1, ring[s1], v0 * ring[s0]);
            ring[(l * width + t) & 4095] = acc * 1e-3;
            s0 = (s0 + width) & 4095;
            s1 = (s1 + width) & 4095;
        }
        __syncthreads();
    }
    if (t == 0) out[0] = clock64() - t0;
    if (t == 0) sink[0] = ring[5];
}

int main() {
    long long* d;
    double* sink;
    cudaMalloc(&d, 64);
    cudaMalloc(&sink, 64);
    const int levels = 10000;
    int threads_list[] = {64, 128, 192, 384, 512, 1024};
    for (int th : threads_list) {
        long long h;
        k_bar_only<<<1, th>>>(levels, d);
        k_bar_only<<<1, th>>>(levels, d);
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("threads %4d  barrier only      : %6.1f cycles/level\n", th, (double)h / levels);
        k_chain<<<1, th>>>(levels, th, d, sink);
        k_chain<<<1, th>>>(levels, th, d, sink);
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("threads %4d  8-term gather+bar : %6.1f cycles/level\n", th, (double)h / levels);
        k_chain2<<<1, th>>>(levels, th, d, sink);
        k_chain2<<<1, th>>>(levels, th, d, sink);
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("threads %4d  2-term gather+bar : %6.1f cycles/level\n", th, (double)h / levels);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
