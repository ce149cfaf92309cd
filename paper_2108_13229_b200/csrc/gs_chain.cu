// Lane-chain lower solve for the structured finest levels of the smoother.
//
// The finest velocity block (MAC u / v, grid.hpp:28-36) and the finest Darcy
// block (TPFA, 5-point) have a lexicographic lower triangle whose
// dependencies all point one cell west or one cell south (plus, for a v row,
// four u neighbours of the same or the previous cell row).  That is a 2-D
// wavefront with one short recurrence per grid row, so instead of the level
// walk (gs_walk.cu: every level a CTA barrier + shared-memory gathers, ~250-600
// cycles) each grid row is a lane: lane L owns cell row j = L and walks its
// row west to east one cell per step, one step behind lane L-1.  The west
// value stays in a register, the south values come from lane L-1's previous
// step by warp shuffle, and only the first lane of each warp reads its south
// values from a shared-memory row written by the last lane of the warp below.
// That row is initialised with a NaN sentinel; the reader spins on the
// sentinel one unrolled block ahead, so no fence or barrier sits on the
// recurrence.  The exact lexicographic Gauss-Seidel order is kept: every row
// still sees the new values of all its lower neighbours.
//
// Records are laid out [band][step][lane] per field (coalesced 256-byte
// loads per warp) and prefetched one unrolled block (kU steps) ahead into
// registers.  b (the prep kernels' output) lives in the plan's `packed`
// array in the same layout, so the prep kernels (gs.cu) are unchanged.
#include "gs.cuh"
#include "launch.cuh"
#include "ptx.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace sdg {

namespace {

constexpr int kU = 4;           // steps per unrolled block (MAC)
constexpr int k5U = 16;         // steps per unrolled block (5-point)
constexpr int kMaxBands = 8;    // warps of the one-CTA kernel

__device__ __forceinline__ void bar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ptx::smem_addr(bar)) : "memory");
}

// Predicated stores / arrive without a branch around them: the step loop of a
// warp stays convergent (a divergent branch per step costs more than the step).
__device__ __forceinline__ void st_global_if(double* p, double v, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global.f64 [%0], %1;\n}" ::"l"(p), "d"(v),
                 "r"(static_cast<int>(pred))
                 : "memory");
}
__device__ __forceinline__ void st_shared_if(double* p, double v, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.shared.f64 [%0], %1;\n}" ::"r"(ptx::smem_addr(p)),
                 "d"(v), "r"(static_cast<int>(pred))
                 : "memory");
}
__device__ __forceinline__ void arrive_if(uint64_t* bar, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %1, 0;\n@q mbarrier.arrive.shared::cta.b64 _, [%0];\n}" ::"r"(
                     ptx::smem_addr(bar)),
                 "r"(static_cast<int>(pred))
                 : "memory");
}

// ---- 5-point (TPFA) -------------------------------------------------------
// z_r = b_r + cs_r z_south + cw_r z_west, row r = j * nx + i, lane = j.
// MODE (dev knob SDG_CHAIN_MODE, timing experiments only): 1 = no z stores,
// 2 = no boundary waits, 4 = no record loads after the first block
template <int MODE, int kU>
__global__ void __launch_bounds__(kMaxBands * 32)
k_chain5(int nx, int ny, int steps, const double* __restrict__ B, const double* __restrict__ CW,
         const double* __restrict__ CS, double* __restrict__ z) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nb = blockDim.x >> 5;
    const int nblk = (nx + kU - 1) / kU;  // column blocks: one single-use mbarrier each
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);                   // [bands - 1][nblk]
    double* ring = reinterpret_cast<double*>(bars + (nb - 1) * nblk);         // [bands - 1][nx]
    for (int k = threadIdx.x; k < (nb - 1) * nblk; k += blockDim.x) ptx::mbar_init(bars + k, 1);
    __syncthreads();
    pdl_wait();
    const int j = w * 32 + lane;
    const double* src = w > 0 ? ring + (w - 1) * nx : nullptr;
    uint64_t* sbar = w > 0 ? bars + (w - 1) * nblk : nullptr;
    double* dst = (w + 1 < nb) ? ring + w * nx : nullptr;
    uint64_t* dbar = dst ? bars + w * nblk : nullptr;
    // the south values of the block starting at column c0 (warp-uniform wait, then lane 0 reads)
    auto south_block = [&](int c0, double (&out)[kU]) {
#pragma unroll
        for (int u = 0; u < kU; ++u) out[u] = 0.0;
        if (!src || c0 >= nx) return;
        ptx::mbar_wait(sbar + c0 / kU, 0);
        if (lane == 0) {
#pragma unroll
            for (int u = 0; u < kU; ++u) out[u] = c0 + u < nx ? src[c0 + u] : 0.0;
        }
    };
    const size_t base = static_cast<size_t>(w) * steps * 32 + lane;
    double b[kU], cw[kU], cs[kU], nb_[kU], ncw[kU], ncs[kU], sr[kU], nsr[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        const size_t k = base + static_cast<size_t>(u) * 32;
        b[u] = B[k];
        cw[u] = CW[k];
        cs[u] = CS[k];
    }
    south_block(0, sr);
    double west = 0.0, last = 0.0;
    long long t_begin = clock64();
    for (int s0 = 0; s0 < steps; s0 += kU) {
        const bool more = s0 + kU < steps;
        if (more && !(MODE & 4)) {
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const size_t k = base + static_cast<size_t>(s0 + kU + u) * 32;
                nb_[u] = B[k];
                ncw[u] = CW[k];
                ncs[u] = CS[k];
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int s = s0 + u;
            double south = __shfl_up_sync(0xffffffffu, last, 1);
            if (lane == 0) south = sr[u];
            const double v = fma(cw[u], west, fma(cs[u], south, b[u]));
            const int i = s - lane;
            const bool act = i >= 0 && i < nx && j < ny;
            if (!(MODE & 1)) st_global_if(z + static_cast<size_t>(j) * nx + i, v, act);
            if (dst) {  // warp-uniform
                const bool pub = act && lane == 31;
                st_shared_if(dst + i, v, pub);
                arrive_if(dbar + i / kU, pub && (i % kU == kU - 1 || i == nx - 1));
            }
            last = act ? v : 0.0;
            west = last;
        }
        if (more) {
            // the south values of the next block (lane 0 only; spins on the sentinel)
            south_block(s0 + kU, nsr);
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (!(MODE & 4)) {
                    b[u] = nb_[u];
                    cw[u] = ncw[u];
                    cs[u] = ncs[u];
                }
                sr[u] = nsr[u];
            }
        }
    }
    if (MODE & 8) {
        if (lane == 0) {
            z[static_cast<size_t>(nx) * ny + 2 * w] = static_cast<double>(t_begin);
            z[static_cast<size_t>(nx) * ny + 2 * w + 1] = static_cast<double>(clock64());
        }
    }
    pdl_trigger();
}

// ---- MAC velocity ----------------------------------------------------------
// Lane L = cell row j.  At step s lane l computes u(i = s - l, j) and then
// v(i' = s - l - 1, j):
//   u = bu + cus u(i, j-1) + cuw u(i-1, j)
//   v = bv + cv4 u(i', j-1) + cv3 u(i', j) + cvw v(i'-1, j) + cvs v(i', j-1)
//          + cv2 u(i'+1, j-1) + cv1 u(i'+1, j)
// u rows: r = j (m+1) + i (j < m); v rows: n_u + j m + i' (j <= m).
struct MacCoef {
    const double *cuw, *cus, *cvw, *cvs, *cv1, *cv2, *cv3, *cv4;
};

template <int MODE>
__global__ void __launch_bounds__(kMaxBands * 32)
k_chain_mac(int m, int steps, const double* __restrict__ BU, const double* __restrict__ BV, MacCoef cf,
            double* __restrict__ z) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nb = blockDim.x >> 5;
    const int len = m + 1;
    const int nblk = (len + kU - 1) / kU;  // block q: u and v columns <= (q + 1) kU - 1
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);                    // [bands - 1][nblk]
    double* ring = reinterpret_cast<double*>(bars + (nb - 1) * nblk);          // [bands - 1][2][m + 1]
    for (int k = threadIdx.x; k < (nb - 1) * nblk; k += blockDim.x) ptx::mbar_init(bars + k, 1);
    __syncthreads();
    pdl_wait();
    const int j = w * 32 + lane;
    const int n_u = m * (m + 1);
    const double* su_ring = w > 0 ? ring + (w - 1) * 2 * len : nullptr;
    const double* sv_ring = w > 0 ? su_ring + len : nullptr;
    double* du_ring = (w + 1 < nb) ? ring + w * 2 * len : nullptr;
    double* dv_ring = du_ring ? du_ring + len : nullptr;
    uint64_t* sbar = w > 0 ? bars + (w - 1) * nblk : nullptr;
    uint64_t* dbar = du_ring ? bars + w * nblk : nullptr;
    const size_t base = static_cast<size_t>(w) * steps * 32 + lane;

    double r[kU][10], nr[kU][10];
    double ru[kU], ru2[kU], rv[kU];  // lane 0: u(s, j-1), u(s-1, j-1), v(s-1, j-1)
    auto load = [&](double (&d)[kU][10], int s0) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const size_t k = base + static_cast<size_t>(s0 + u) * 32;
            d[u][0] = BU[k];
            d[u][1] = cf.cuw[k];
            d[u][2] = cf.cus[k];
            d[u][3] = BV[k];
            d[u][4] = cf.cvw[k];
            d[u][5] = cf.cvs[k];
            d[u][6] = cf.cv1[k];
            d[u][7] = cf.cv2[k];
            d[u][8] = cf.cv3[k];
            d[u][9] = cf.cv4[k];
        }
    };
    load(r, 0);
    // lane 0's boundary values of a block starting at s0: u columns s0-1 .. s0+kU-1, v columns s0-1 .. s0+kU-2
    auto boundary = [&](int s0) {
        double bu[kU + 1], bv[kU];
#pragma unroll
        for (int k = 0; k <= kU; ++k) bu[k] = 0.0;
#pragma unroll
        for (int k = 0; k < kU; ++k) bv[k] = 0.0;
        if (su_ring && s0 < len) {
            ptx::mbar_wait(sbar + s0 / kU, 0);  // u, v columns <= s0 + kU - 1 are in
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k <= kU; ++k) {
                    const int c = s0 - 1 + k;
                    bu[k] = (c >= 0 && c < len) ? su_ring[c] : 0.0;
                }
#pragma unroll
                for (int k = 0; k < kU; ++k) {
                    const int c = s0 - 1 + k;
                    bv[k] = (c >= 0 && c < m) ? sv_ring[c] : 0.0;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            ru[u] = bu[u + 1];
            ru2[u] = bu[u];
            rv[u] = bv[u];
        }
    };
    boundary(0);
    double u_last = 0.0, u_last2 = 0.0, v_last = 0.0;
    for (int s0 = 0; s0 < steps; s0 += kU) {
        const bool more = s0 + kU < steps;
        if (more && !(MODE & 4)) load(nr, s0 + kU);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int s = s0 + u;
            double su1 = __shfl_up_sync(0xffffffffu, u_last, 1);
            double su2 = __shfl_up_sync(0xffffffffu, u_last2, 1);
            double sv1 = __shfl_up_sync(0xffffffffu, v_last, 1);
            if (lane == 0) {
                su1 = ru[u];
                su2 = ru2[u];
                sv1 = rv[u];
            }
            const double* q = r[u];
            const double un = fma(q[1], u_last, fma(q[2], su1, q[0]));
            double t = fma(q[9], su2, q[3]);
            t = fma(q[8], u_last, t);
            t = fma(q[4], v_last, t);
            t = fma(q[5], sv1, t);
            t = fma(q[7], su1, t);
            const double vn = fma(q[6], un, t);
            const int i = s - lane;
            const bool ua = i >= 0 && i <= m && j < m;
            const bool va = i - 1 >= 0 && i - 1 < m && j <= m;
            if (!(MODE & 1)) {
                st_global_if(z + static_cast<size_t>(j) * (m + 1) + i, un, ua);
                st_global_if(z + n_u + static_cast<size_t>(j) * m + (i - 1), vn, va);
            }
            if (du_ring) {  // warp-uniform
                st_shared_if(du_ring + i, un, ua && lane == 31);
                const int c = i - 1;  // v column c; u column c + 1 went in this step too
                const bool pub = va && lane == 31;
                st_shared_if(dv_ring + c, vn, pub);
                arrive_if(dbar + c / kU, pub && (c % kU == kU - 1));
                if (pub && c == m - 1)
                    for (int q = c / kU + (c % kU == kU - 1); q < nblk; ++q) bar_arrive(dbar + q);
            }
            u_last2 = u_last;
            u_last = ua ? un : 0.0;
            v_last = va ? vn : 0.0;
        }
        if (more) {
            boundary(s0 + kU);
            if (!(MODE & 4)) {
#pragma unroll
                for (int u = 0; u < kU; ++u)
#pragma unroll
                    for (int f = 0; f < 10; ++f) r[u][f] = nr[u][f];
            }
        }
    }
    pdl_trigger();
}

}  // namespace

// Detects the two structured patterns on the plan's matrix and lays out the
// records; returns false (plan untouched) for anything else.
bool GsPlan::build_chain(const HostCsr& a, const std::vector<int>& comps, const std::vector<double>& dinv_h,
                         cudaStream_t s) {
    // SDG_GS_CHAIN: 0 off (default: the walk measures as fast at c2), 1 the 5-point chain, 2 also the MAC chain
    const char* env = std::getenv("SDG_GS_CHAIN");
    const int allow = env ? std::atoi(env) : 0;
    if (allow <= 0) return false;
    const int nn = a.n_rows;
    if (nn < 64) return false;
    int kind = 0, nx = 0, ny = 0, m = 0, lanes = 0;
    if (!comps.empty()) {
        if (allow < 2) return false;  // measured slower than the walk at c2 (bandwidth of one SM)
        int n_u = 0;
        while (n_u < nn && comps[n_u] == 0) ++n_u;
        m = static_cast<int>(std::floor(std::sqrt(static_cast<double>(n_u))));
        while (static_cast<int64_t>(m) * (m + 1) > n_u) --m;
        if (m < 2 || static_cast<int64_t>(m) * (m + 1) != n_u || 2 * n_u != nn) return false;
        for (int r = n_u; r < nn; ++r)
            if (comps[r] != 1) return false;
        kind = 2;
        lanes = m + 1;
    } else {
        nx = static_cast<int>(std::lround(std::sqrt(static_cast<double>(nn))));
        if (static_cast<int64_t>(nx) * nx != nn) return false;
        ny = nx;
        kind = 1;
        lanes = ny;
    }
    const int nb = (lanes + 31) / 32;
    if (nb > kMaxBands || nb < 2) return false;
    int steps = kind == 1 ? nx + 31 : m + 32;
    const int unroll = kind == 1 ? k5U : kU;
    steps = (steps + unroll - 1) / unroll * unroll;
    const size_t slots = static_cast<size_t>(nb) * steps * 32;
    auto slot = [&](int j, int step) { return (static_cast<size_t>(j / 32) * steps + step) * 32 + (j % 32); };
    const int nf = kind == 1 ? 2 : 8;
    std::vector<double> coef(nf * slots, 0.0);
    std::vector<int> bx(nn, -1);
    auto put = [&](int field, size_t at, double v) { coef[static_cast<size_t>(field) * slots + at] = v; };
    for (int r = 0; r < nn; ++r) {
        size_t at;
        int expect[6] = {-1, -1, -1, -1, -1, -1};
        int field[6] = {0, 0, 0, 0, 0, 0};
        if (kind == 1) {
            const int i = r % nx, j = r / nx;
            at = slot(j, i + j % 32);
            bx[r] = static_cast<int>(at);
            expect[0] = i > 0 ? r - 1 : -1;
            field[0] = 0;
            expect[1] = j > 0 ? r - nx : -1;
            field[1] = 1;
        } else if (r < m * (m + 1)) {
            const int i = r % (m + 1), j = r / (m + 1);
            at = slot(j, i + j % 32);
            bx[r] = static_cast<int>(at);
            expect[0] = i > 0 ? r - 1 : -1;
            field[0] = 0;
            expect[1] = j > 0 ? r - (m + 1) : -1;
            field[1] = 1;
        } else {
            const int q = r - m * (m + 1), i = q % m, j = q / m;
            at = slot(j, i + j % 32 + 1);
            bx[r] = static_cast<int>(slots + at);
            auto urow = [&](int ii, int jj) { return (jj >= 0 && jj < m && ii >= 0 && ii <= m) ? jj * (m + 1) + ii : -1; };
            expect[0] = i > 0 ? r - 1 : -1;        // v(i-1, j)
            field[0] = 2;
            expect[1] = j > 0 ? r - m : -1;        // v(i, j-1)
            field[1] = 3;
            expect[2] = urow(i + 1, j);            // u(i+1, j)
            field[2] = 4;
            expect[3] = urow(i + 1, j - 1);        // u(i+1, j-1)
            field[3] = 5;
            expect[4] = urow(i, j);                // u(i, j)
            field[4] = 6;
            expect[5] = urow(i, j - 1);            // u(i, j-1)
            field[5] = 7;
        }
        for (int k = a.rp[r]; k < a.rp[r + 1]; ++k) {
            const int c = a.ci[k];
            if (c >= r) continue;
            int hit = -1;
            for (int e = 0; e < 6; ++e)
                if (expect[e] == c) hit = e;
            if (hit < 0) return false;  // not the structured pattern
            put(field[hit], at, -a.v[k] * dinv_h[r]);
        }
    }
    packed.resize(kind == 1 ? slots : 2 * slots);
    SDG_CUDA(cudaMemsetAsync(packed.get(), 0, packed.size() * sizeof(double), s));
    chain_coef.upload(coef, s);
    bidx.upload(bx, s);
    chain = true;
    chain_kind = kind;
    chain_nx = kind == 1 ? nx : m;
    chain_ny = kind == 1 ? ny : m + 1;
    chain_steps = steps;
    chain_bands = nb;
    {
        const int cols = kind == 1 ? nx : m + 1;
        const int nblk = (cols + unroll - 1) / unroll;
        chain_smem = static_cast<size_t>(nb - 1) * (nblk * sizeof(uint64_t) + (kind == 1 ? 1 : 2) * cols * sizeof(double));
    }
    walk = false;
    usable = true;
    if (std::getenv("SDG_DEBUG"))
        std::fprintf(stderr, "[sdg] gs chain: kind %d, %d lanes in %d warps, %d steps, %zu B ring\n", kind, lanes,
                     nb, steps, chain_smem);
    return true;
}

template <int MODE>
void launch_chain_mode(Context& c, const GsPlan& g, double* z_new) {
    const size_t slots = static_cast<size_t>(g.chain_bands) * g.chain_steps * 32;
    const double* cf = g.chain_coef.get();
    if (g.chain_kind == 1) {
        launch_k(c, k_chain5<MODE, k5U>, 1, g.chain_bands * 32, g.chain_smem, g.chain_nx, g.chain_ny, g.chain_steps,
                 g.packed.get(), cf, cf + slots, z_new);
    } else {
        MacCoef m{cf, cf + slots, cf + 2 * slots, cf + 3 * slots, cf + 4 * slots, cf + 5 * slots, cf + 6 * slots,
                  cf + 7 * slots};
        launch_k(c, k_chain_mac<MODE>, 1, g.chain_bands * 32, g.chain_smem, g.chain_nx, g.chain_steps,
                 g.packed.get(), g.packed.get() + slots, m, z_new);
    }
}

void launch_gs_chain(Context& c, const GsPlan& g, double* z_new) {
    static const int mode = [] {
        const char* e = std::getenv("SDG_CHAIN_MODE");
        return e ? std::atoi(e) : 0;
    }();
    switch (mode) {
    case 1: launch_chain_mode<1>(c, g, z_new); break;
    case 2: launch_chain_mode<2>(c, g, z_new); break;
    case 3: launch_chain_mode<3>(c, g, z_new); break;
    case 4: launch_chain_mode<4>(c, g, z_new); break;
    case 7: launch_chain_mode<7>(c, g, z_new); break;
    case 8: launch_chain_mode<8>(c, g, z_new); break;
    case 9: launch_chain_mode<9>(c, g, z_new); break;
    case 12: launch_chain_mode<12>(c, g, z_new); break;
    case 13: launch_chain_mode<13>(c, g, z_new); break;
    default: launch_chain_mode<0>(c, g, z_new); break;
    }
    c.count();
}

}  // namespace sdg
