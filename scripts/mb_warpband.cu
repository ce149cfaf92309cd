// Dev micro-benchmark: per-level cost of a lexicographic 5-point lower solve
// (z_ij = b - a_w z_{i-1,j} - a_s z_{i,j-1}) on an nx x ny grid, one CTA.
//   bar : one thread per grid row, __syncthreads per anti-diagonal level
//   wb  : warp bands (each warp owns h grid rows, lane = row), warp-synchronous
//         levels, cross-warp dependencies through smem z + progress counters
//   wbr : wb with the in-row (west) dependency kept in a register
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int ld_vol(const int* p) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}
__device__ __forceinline__ int ld_acq(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
    asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

__global__ void k_bar(int nx, int ny, long long* out, double* zout) {
    extern __shared__ double z[];
    const int j = threadIdx.x;
    for (int k = threadIdx.x; k < nx * ny; k += blockDim.x) z[k] = 0.0;
    __syncthreads();
    long long t0 = clock64();
    const int levels = nx + ny - 1;
    for (int L = 0; L < levels; ++L) {
        const int i = L - j;
        if (j < ny && i >= 0 && i < nx) {
            const int r = j * nx + i;
            const double w = i > 0 ? z[r - 1] : 0.0;
            const double s = j > 0 ? z[r - nx] : 0.0;
            z[r] = 1.0 - fma(0.25, w, 0.25 * s);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = clock64() - t0;
    for (int k = threadIdx.x; k < nx * ny; k += blockDim.x) zout[k] = z[k];
}

template <bool REG, bool ACQ>
__global__ void k_wb(int nx, int ny, int h, long long* out, double* zout) {
    extern __shared__ double z[];
    __shared__ int prog[32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    for (int k = threadIdx.x; k < nx * ny; k += blockDim.x) z[k] = 0.0;
    if (threadIdx.x < 32) prog[threadIdx.x] = 0;
    __syncthreads();
    long long t0 = clock64();
    const int j = w * h + lane;
    const bool act = lane < h && j < ny;
    const int levels = nx + h - 1;
    double west = 0.0;
    for (int L = 0; L < levels; ++L) {
        // level L of this warp reads row w*h-1 of warp w-1 at column L (its local level L + h - 1)
        if (w > 0 && lane == 0) {
            const int need = min(L + h, nx + h - 1);
            if (ACQ) {
                while (ld_acq(&prog[w - 1]) < need) {}
            } else {
                while (ld_vol(&prog[w - 1]) < need) {}
            }
        }
        __syncwarp();
        const int i = L - lane;
        if (act && i >= 0 && i < nx) {
            const int r = j * nx + i;
            const double wv = REG ? west : (i > 0 ? z[r - 1] : 0.0);
            const double s = j > 0 ? z[r - nx] : 0.0;
            const double v = 1.0 - fma(0.25, wv, 0.25 * s);
            z[r] = v;
            west = v;
        }
        __syncwarp();
        if (lane == 0) {
            if (ACQ) {
                st_rel(&prog[w], L + 1);
            } else {
                __threadfence_block();
                asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&prog[w])), "r"(L + 1) : "memory");
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[0] = clock64() - t0;
    for (int k = threadIdx.x; k < nx * ny; k += blockDim.x) zout[k] = z[k];
}

int main() {
    long long* d;
    double *z1, *z2;
    const int nx = 160, ny = 160;
    cudaMalloc(&d, 64);
    cudaMalloc(&z1, nx * ny * 8);
    cudaMalloc(&z2, nx * ny * 8);
    const size_t sm = nx * ny * 8;
    cudaFuncSetAttribute(k_bar, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_wb<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_wb<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_wb<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    long long h;
    const int depth = nx + ny - 1;
    for (int rep = 0; rep < 2; ++rep) k_bar<<<1, 160, sm>>>(nx, ny, d, z1);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("bar  160 threads: %8lld cycles, %6.1f cycles/level (depth %d)\n", h, (double)h / depth, depth);
    double* hz1 = new double[nx * ny];
    double* hz2 = new double[nx * ny];
    cudaMemcpy(hz1, z1, sm, cudaMemcpyDeviceToHost);
    int hs[] = {5, 8, 10, 16, 20, 32};
    for (int hh : hs) {
        const int warps = (ny + hh - 1) / hh;
        if (warps > 32) continue;
        for (int var = 0; var < 3; ++var) {
            for (int rep = 0; rep < 2; ++rep) {
                if (var == 0) k_wb<false, false><<<1, warps * 32, sm>>>(nx, ny, hh, d, z2);
                if (var == 1) k_wb<true, false><<<1, warps * 32, sm>>>(nx, ny, hh, d, z2);
                if (var == 2) k_wb<true, true><<<1, warps * 32, sm>>>(nx, ny, hh, d, z2);
            }
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(hz2, z2, sm, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int k = 0; k < nx * ny; ++k) bad += hz1[k] != hz2[k];
            printf("wb h=%2d warps=%2d %s: %8lld cycles, %6.1f cycles/level, mismatches %d (%s)\n", hh, warps,
                   var == 0 ? "smem-west    " : var == 1 ? "reg-west     " : "reg-west+acq ", h, (double)h / depth,
                   bad, cudaGetErrorString(e));
        }
    }
    return 0;
}
