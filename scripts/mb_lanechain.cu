// Dev micro-benchmark: lexicographic 5-point lower solve
//   z_ij = b_ij + cw_ij z_{i-1,j} + cs_ij z_{i,j-1}
// as a "lane chain": lane = grid row, lanes skewed by one column, the west
// value in a register, the south value by shfl.up from the previous step.
//   A: one CTA, W warps, warp boundary through a shared ring + progress counter
//   B: one warp per CTA in a cluster, boundary through DSMEM stores + remote
//      release counter
// Records are laid out [band][step][lane] (coalesced), prefetched one unrolled
// block (U steps) ahead.  Prints cycles per step and checks bits against a
// sequential host solve.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int U = 4;
constexpr int RING = 512;

__device__ __forceinline__ unsigned ld_acq_cl(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acq_cta(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}

struct Rec { double b, cw, cs; };

// steps per band = nx + 31
template <bool CLUSTER>
__global__ void k_chain(int nx, int ny, const double* __restrict__ B, const double* __restrict__ CW,
                        const double* __restrict__ CS, double* __restrict__ z, long long* cyc) {
    extern __shared__ double ringbuf[];
    __shared__ unsigned prog[32];
    auto ring = reinterpret_cast<double (*)[RING]>(ringbuf);
    const int lane = threadIdx.x & 31;
    int band, wib;
    if (CLUSTER) { band = blockIdx.x; wib = 0; } else { band = threadIdx.x >> 5; wib = band; }
    const int nb = (ny + 31) / 32;
    if (lane == 0) prog[wib] = 0;
    if (CLUSTER) cg::this_cluster().sync(); else __syncthreads();
    const int steps = nx + 31;
    const int sp = (steps + U - 1) / U * U;
    const size_t base = (size_t)band * sp * 32;
    const int j = band * 32 + lane;
    long long t0 = clock64();
    double west = 0.0, zlast = 0.0;
    Rec cur[U], nxt[U];
    double bnd[U], bndn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const size_t k = base + (size_t)u * 32 + lane;
        cur[u] = {B[k], CW[k], CS[k]};
    }
    // consumer side: remote column values for block 0
    double* myring = ring[wib];
    unsigned seen = 0;
    auto need = [&](int col_hi) {  // wait until producer published columns < col_hi
        if (band == 0) return;
        const unsigned want = min(col_hi, nx);
        if (seen >= want) return;
        if (lane == 0) {
            unsigned v;
            do { v = CLUSTER ? ld_acq_cl(&prog[wib]) : ld_acq_cta(&prog[wib - 1]); } while (v < want);
            seen = v;
        }
        seen = __shfl_sync(0xffffffffu, seen, 0);
    };
    const double* rsrc = CLUSTER ? myring : ring[wib - (band > 0)];
    need(U);
#pragma unroll
    for (int u = 0; u < U; ++u) bnd[u] = (band > 0 && u < nx) ? rsrc[u % RING] : 0.0;
    for (int s0 = 0; s0 < sp; s0 += U) {
        const bool more = s0 + U < sp;
        if (more) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const size_t k = base + (size_t)(s0 + U + u) * 32 + lane;
                nxt[u] = {B[k], CW[k], CS[k]};
            }
            need(s0 + 2 * U);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = s0 + U + u;
                bndn[u] = (band > 0 && c < nx) ? rsrc[c % RING] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int s = s0 + u;
            double south = __shfl_up_sync(0xffffffffu, zlast, 1);
            if (lane == 0) south = bnd[u];  // column s of row j-1
            const int i = s - lane;
            double v = fma(cur[u].cs, south, cur[u].b);
            v = fma(cur[u].cw, west, v);
            const bool act = i >= 0 && i < nx && j < ny;
            if (!act) v = 0.0;
            if (act) z[(size_t)j * nx + i] = v;
            zlast = v;
            west = (i >= 0 && i < nx) ? v : 0.0;
            // producer: lane 31 publishes column i
            if (lane == 31 && act && band + 1 < nb) {
                if (CLUSTER) {
                    cg::cluster_group cl = cg::this_cluster();
                    double* rr = cl.map_shared_rank(ringbuf, band + 1);
                    rr[i % RING] = v;
                } else {
                    ring[wib][i % RING] = v;
                }
            }
        }
        if (lane == 31 && band + 1 < nb) {
            const int done = min(max(s0 + U - 31, 0), nx);
            if (CLUSTER) {
                cg::cluster_group cl = cg::this_cluster();
                unsigned* rp = cl.map_shared_rank(&prog[0], band + 1);
                asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(rp)), "r"((unsigned)done) : "memory");
            } else {
                asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&prog[wib])), "r"((unsigned)done) : "memory");
            }
        }
        if (more) {
#pragma unroll
            for (int u = 0; u < U; ++u) { cur[u] = nxt[u]; bnd[u] = bndn[u]; }
        }
    }
    if (CLUSTER) cg::this_cluster().sync(); else __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = clock64() - t0;
}

int main() {
    int sizes[][2] = {{160, 160}, {161, 160}, {500, 500}};
    for (auto& sz : sizes) {
        const int nx = sz[0], ny = sz[1];
        const int nb = (ny + 31) / 32;
        const int steps = nx + 31, sp = (steps + U - 1) / U * U;
        std::vector<double> hb(nx * ny), hw(nx * ny), hs(nx * ny), zr(nx * ny);
        srand(1);
        for (int k = 0; k < nx * ny; ++k) {
            hb[k] = rand() / (double)RAND_MAX;
            hw[k] = -0.3 * rand() / (double)RAND_MAX;
            hs[k] = -0.3 * rand() / (double)RAND_MAX;
        }
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                const int k = j * nx + i;
                double v = fma(hs[k], j > 0 ? zr[k - nx] : 0.0, hb[k]);
                zr[k] = fma(hw[k], i > 0 ? zr[k - 1] : 0.0, v);
            }
        // packed [band][step][lane]
        size_t np = (size_t)nb * sp * 32;
        std::vector<double> pb(np, 0), pw(np, 0), ps(np, 0);
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                const int band = j / 32, lane = j % 32, s = i + lane;
                const size_t p = ((size_t)band * sp + s) * 32 + lane;
                pb[p] = hb[j * nx + i];
                pw[p] = hw[j * nx + i];
                ps[p] = hs[j * nx + i];
            }
        double *db, *dw, *ds, *dz;
        long long* dc;
        cudaMalloc(&db, np * 8); cudaMalloc(&dw, np * 8); cudaMalloc(&ds, np * 8);
        cudaMalloc(&dz, nx * ny * 8); cudaMalloc(&dc, 8);
        cudaMemcpy(db, pb.data(), np * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dw, pw.data(), np * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(ds, ps.data(), np * 8, cudaMemcpyHostToDevice);
        for (int var = 0; var < 2; ++var) {
            if (var == 0 && nb > 32) continue;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            float ms = 0;
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(dz, 0, nx * ny * 8);
                cudaEventRecord(e0);
                if (var == 0) {
                    cudaFuncSetAttribute(k_chain<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, nb * RING * 8);
                    k_chain<false><<<1, nb * 32, nb * RING * 8>>>(nx, ny, db, dw, ds, dz, dc);
                } else {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(nb); cfg.blockDim = dim3(32); cfg.dynamicSmemBytes = RING * 8;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = nb; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                    cfg.attrs = at; cfg.numAttrs = 1;
                    cudaFuncSetAttribute(k_chain<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                    cudaError_t le = cudaLaunchKernelEx(&cfg, k_chain<true>, nx, ny, (const double*)db, (const double*)dw, (const double*)ds, dz, dc);
                    if (le != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(le));
                }
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            cudaError_t e = cudaDeviceSynchronize();
            long long h;
            cudaMemcpy(&h, dc, 8, cudaMemcpyDeviceToHost);
            std::vector<double> hz(nx * ny);
            cudaMemcpy(hz.data(), dz, nx * ny * 8, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int k = 0; k < nx * ny; ++k) bad += hz[k] != zr[k];
            const int depth = nx + ny - 1;
            printf("%dx%d %s bands=%d: %lld cycles (%.1f/level of %d), %.1f us event, mismatches %d (%s)\n", nx, ny,
                   var ? "cluster" : "1-CTA  ", nb, h, (double)h / depth, depth, ms * 1e3, bad, cudaGetErrorString(e));
        }
        cudaFree(db); cudaFree(dw); cudaFree(ds); cudaFree(dz); cudaFree(dc);
    }
    return 0;
}
