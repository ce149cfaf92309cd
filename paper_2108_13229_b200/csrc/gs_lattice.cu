// Multi-SM lattice lower solve for the aggregated coarse levels of the
// smoother (sor_sweep, precond.cpp:92-108, lower part of one forward sweep).
//
// The first coarse levels of the velocity and porous hierarchies are
// aggregations of the structured finest grids (precond.cpp:122-175): the
// aggregates form rows, and the lexicographic lower triangle of a coarse
// level is a lattice -- every aggregate depends on its west neighbour in its
// own aggregate row and on two or three aggregates of the row below.  The
// level walk (gs_walk.cu) pays a CTA-wide hand-off per dependency level
// (~300-500 cycles, one SM); here the rows are cut into CHAINS and each
// chain is a lane, as the wavefront does for the finest grids (gs_wave.cu):
//
//   * a chain is a sequence of rows each of which depends on its predecessor
//     (row i joins the chain whose last row is i's most recent lower
//     neighbour; otherwise it starts a chain).  Chains ordered by their first
//     row are the lanes; 32 consecutive chains are a band, one warp, one CTA;
//   * every row gets a step: one after its chain predecessor and one after
//     each lower neighbour in its band (the schedule is a topological order
//     of the lower triangle, so the sweep stays the exact lexicographic
//     Gauss-Seidel sweep).  Lanes with nothing to do at a step run a zero
//     record;
//   * within a band every lane stores its value of step t into a shared-
//     memory ring (32 lanes x R steps) and reads its lower neighbours from it
//     (a __syncwarp per step); across bands only the last chain of band b - 1
//     may feed band b: its lane 31 stores each step's value into a boundary
//     buffer that holds a sentinel until written (the value is its own flag,
//     as in gs_wave.cu), and band b loads a 32-step window of it per block,
//     one block ahead, into shared memory;
//   * records [block][field][KU/2 step pairs][32 lanes][2] are streamed by
//     1-D TMA bulk copies into a shared-memory ring, as in gs_wave.cu.
//
// Arithmetic: the level walk's, bit for bit -- the lower entries in column
// order, c = -a_ij / d_i; rows with <= 2 lower entries
//   z = fma(c1, z1, fma(c0, z0, b)),
// wider rows (the walk's wide record, pairs then a balanced tree)
//   z = (fma(c1, z1, fma(c0, z0, b)) + fma(c3, z3, c2 z2)) + 0.
// Levels that are not such a lattice (more than 4 lower entries in a row,
// a dependency on another band than the previous one's last chain, a window
// wider than 32 steps) keep the level walk.
#include "gs.cuh"
#include "launch.cuh"
#include "ptx.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unordered_map>

namespace sdg {

namespace {

constexpr int kLatKU = 8;       // steps per block
constexpr int kLatF = 8;        // record fields: b, c0..c3, src01, src23, (rowid, wide)
constexpr int kLatDepth = 4;    // blocks of records in flight
constexpr int kLatR = 64;       // ring steps per lane
constexpr int kLatW = 32;       // window steps of the previous band's last chain
constexpr int kLatZero = 32 * kLatR;           // index of the constant zero in the value array
constexpr int kLatWin = kLatZero + 1;          // two windows (block parity) follow
constexpr int kLatVals = kLatWin + 2 * kLatW;  // doubles of the value array
constexpr unsigned long long kLatSent = 0x7ff4deadbeefcafeull;

struct LatArgs {
    const double* rec;            // [band][block][F][KU/2][32][2]
    const int* win;               // [band][block]: window of the previous band's last chain (first step * 64 + steps)
    double* z;
    double* bnd;                  // [2 parities][nbands][T]
    unsigned long long* ticket;
    int nbands, nblocks;
};

__device__ __forceinline__ bool lat_ready(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) != kLatSent;
}
__device__ __forceinline__ double lat_ld_if(const double* p, bool pred) {
    double v;
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\nmov.b64 %0, 0;\n@q ld.relaxed.gpu.global.f64 %0, [%1];\n}"
                 : "=d"(v)
                 : "l"(p), "r"(static_cast<int>(pred))
                 : "memory");
    return v;
}
__device__ __forceinline__ void lat_st_relaxed_if(double* p, double v, bool pred) {
    const double w = v + 0.0;  // quiets a signalling NaN: a stored value is never the sentinel
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.relaxed.gpu.global.f64 [%0], %1;\n}" ::"l"(p),
                 "d"(w), "r"(static_cast<int>(pred)));
}
__device__ __forceinline__ void lat_st_if(double* p, double v, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global.f64 [%0], %1;\n}" ::"l"(p), "d"(v),
                 "r"(static_cast<int>(pred)));
}
__device__ __forceinline__ void lat_tma_if(double* dst, const double* src, unsigned bytes, uint64_t* bar, bool pred) {
    asm volatile(
        "{\n.reg .pred q;\nsetp.ne.b32 q, %4, 0;\n"
        "@q fence.proxy.async.shared::cta;\n"
        "@q mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n"
        "@q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}" ::"r"(
            ptx::smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(ptx::smem_addr(bar)), "r"(static_cast<int>(pred))
        : "memory");
}

// One warp per band; all control flow warp-uniform (per-lane work predicated).
__global__ void __launch_bounds__(32, 1) k_gs_lattice(LatArgs a) {
    constexpr int KU = kLatKU, F = kLatF, BLK = F * KU * 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* ring = reinterpret_cast<double*>(smem_raw);      // records
    double* vals = ring + kLatDepth * BLK;                   // value ring | zero | windows
    uint64_t* bars = reinterpret_cast<uint64_t*>(vals + kLatVals + 1);
    const int lane = threadIdx.x;
    unsigned long long t = 0;
    if (lane == 0) {
        t = atomicAdd(a.ticket, 1ull);
#pragma unroll
        for (int d = 0; d < kLatDepth; ++d) ptx::mbar_init(bars + d, 1);
        ptx::fence_mbar_init();
    }
    for (int k = lane; k < kLatVals; k += 32) vals[k] = 0.0;
    t = __shfl_sync(0xffffffffu, t, 0);
    __syncwarp();
    const int band = static_cast<int>(t % static_cast<unsigned long long>(a.nbands));
    const int par = static_cast<int>((t / static_cast<unsigned long long>(a.nbands)) & 1ull);
    pdl_wait();  // b is written by the prep kernel; the previous launch of this plan is complete
    pdl_trigger();
    const double* src = a.rec + static_cast<size_t>(band) * a.nblocks * BLK;
    for (int d = 0; d < kLatDepth && d < a.nblocks; ++d)
        lat_tma_if(ring + d * BLK, src + static_cast<size_t>(d) * BLK, BLK * 8, bars + d, lane == 0);
    const int T = a.nblocks * KU;
    const bool has_src = band > 0, has_dst = band + 1 < a.nbands;
    const size_t pstride = static_cast<size_t>(a.nbands) * T;
    const double* b_in = a.bnd + par * pstride + static_cast<size_t>(has_src ? band - 1 : 0) * T;
    double* b_out = a.bnd + par * pstride + static_cast<size_t>(band) * T;
    if (has_src) {  // the other parity's input slots, for the next launch
        double* rs = a.bnd + (par ^ 1) * pstride + static_cast<size_t>(band - 1) * T;
        for (int k = lane; k < T; k += 32) rs[k] = __longlong_as_double(static_cast<long long>(kLatSent));
    }
    const int* win = a.win + static_cast<size_t>(band) * a.nblocks;
    // window of block q: steps win[q] .. win[q] + 31 of the previous band's last chain
    // win[q] = first step * 64 + steps needed (<= 32), or -1: no window
    auto load_win = [&](int q) {
        const int w = q < a.nblocks ? win[q] : -1;
        return lat_ld_if(b_in + (w >> 6) + lane, has_src && w >= 0 && lane < (w & 63));
    };
    auto settle = [&](int q, double& v) {
        const int w = q < a.nblocks ? win[q] : -1;
        while (!__all_sync(0xffffffffu, lat_ready(v)))
            v = lat_ld_if(b_in + (w >> 6) + lane, has_src && w >= 0 && lane < (w & 63));
        vals[kLatWin + (q & 1) * kLatW + lane] = v;
    };
    double wv = load_win(0);
    settle(0, wv);
    const bool pub = has_dst && lane == 31;
    for (int q = 0; q < a.nblocks; ++q) {
        double wn = load_win(q + 1);  // in flight during this block
        const int slot = q % kLatDepth;
        ptx::mbar_wait(bars + slot, (q / kLatDepth) & 1);
        __syncwarp();  // the window stored at the end of the previous block
        const double2* B = reinterpret_cast<const double2*>(ring + slot * BLK) + lane;
#pragma unroll
        for (int u2 = 0; u2 < KU / 2; ++u2) {
            double2 R[F];
#pragma unroll
            for (int f = 0; f < F; ++f) R[f] = B[(f * KU / 2 + u2) * 32];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                auto r = [&](int f) { return h ? R[f].y : R[f].x; };
                auto ri = [&](int f) {
                    const int2 v = *reinterpret_cast<const int2*>(h ? &R[f].y : &R[f].x);
                    return v;
                };
                const int2 s01 = ri(5), s23 = ri(6), rw = ri(7);
                const double z0 = vals[s01.x], z1 = vals[s01.y], z2 = vals[s23.x], z3 = vals[s23.y];
                const double acc = fma(r(2), z1, fma(r(1), z0, r(0)));
                const double wide = (acc + fma(r(4), z3, r(3) * z2)) + 0.0;
                const double res = rw.y ? wide : acc;
                const int step = q * KU + 2 * u2 + h;
                // no lane reads a slot written in this step (same-band sources are
                // at least one and less than kLatR steps old, GsPlan::build_lattice)
                vals[lane * kLatR + (step & (kLatR - 1))] = res;
                lat_st_if(a.z + rw.x, res, rw.x >= 0);
                lat_st_relaxed_if(b_out + step, res, pub);
                __syncwarp();  // the step's values are visible to the next step
            }
        }
        __syncwarp();  // every lane has read the record slot
        lat_tma_if(ring + slot * BLK, src + static_cast<size_t>(q + kLatDepth) * BLK, BLK * 8, bars + slot,
                   lane == 0 && q + kLatDepth < a.nblocks);
        if (q + 1 < a.nblocks) settle(q + 1, wn);
    }
}

size_t lat_smem_bytes() {
    return static_cast<size_t>(kLatDepth) * kLatF * kLatKU * 32 * sizeof(double) + (kLatVals + 1) * sizeof(double) +
           kLatDepth * sizeof(uint64_t);
}

}  // namespace

// Host plan of the lattice (no device work): records, b slots, windows.
struct LatticeHost {
    int nb = 0, nblocks = 0, nch = 0;
    std::vector<double> rec;
    std::vector<int> bidx, win;
};

// Plans the lattice for the lower triangle of `a` (all of it: a label block's
// own matrix when called from build_parts).  Returns false when the level is
// not such a lattice.
static bool plan_lattice(const HostCsr& a, const std::vector<double>& dinv_h, LatticeHost& out) {
    const int nn = a.n_rows;
    if (nn < 256) return false;
    // lower entries in column order
    std::vector<int> lp(nn + 1, 0);
    std::vector<int> lc;
    std::vector<double> lv;
    for (int i = 0; i < nn; ++i) {
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] < i) {
                lc.push_back(a.ci[k]);
                lv.push_back(-(a.v[k] * dinv_h[i]));
            }
        lp[i + 1] = static_cast<int>(lc.size());
        if (lp[i + 1] - lp[i] > 4) return false;
    }
    // chains: row i joins the chain whose last row is i's most recent lower neighbour
    std::vector<int> chain(nn), tail_chain(nn, -1);  // tail_chain[r] = chain whose last row is r
    int nch = 0;
    for (int i = 0; i < nn; ++i) {
        int pick = -1;
        for (int k = lp[i]; k < lp[i + 1]; ++k)
            if (tail_chain[lc[k]] >= 0) pick = std::max(pick, lc[k]);
        if (pick >= 0) {
            chain[i] = tail_chain[pick];
            tail_chain[pick] = -1;
        } else {
            chain[i] = nch++;
        }
        tail_chain[i] = chain[i];
    }
    const int nb = (nch + 31) / 32;
    if (nb < 2) return false;  // one band: the single-CTA walk is as good
    // steps: after the chain predecessor and after every lower neighbour of the same band
    std::vector<int> step(nn), last_step(nch, -1);
    int tmax = 0;
    for (int i = 0; i < nn; ++i) {
        const int c = chain[i], b = c / 32;
        int tt = last_step[c] + 1;
        for (int k = lp[i]; k < lp[i + 1]; ++k) {
            const int j = lc[k], cj = chain[j], bj = cj / 32;
            if (bj == b)
                tt = std::max(tt, step[j] + 1);
            else if (!(bj == b - 1 && cj % 32 == 31))
                return false;  // only the previous band's last chain may feed a band
        }
        step[i] = tt;
        last_step[c] = tt;
        tmax = std::max(tmax, tt);
    }
    const int nblocks = (tmax + 1 + kLatKU - 1) / kLatKU;
    // windows: per consumer block, the steps of the previous band's last chain it reads
    std::vector<int> wlo(static_cast<size_t>(nb) * nblocks, INT32_MAX), whi(static_cast<size_t>(nb) * nblocks, -1);
    for (int i = 0; i < nn; ++i) {
        const int b = chain[i] / 32;
        for (int k = lp[i]; k < lp[i + 1]; ++k) {
            const int j = lc[k];
            if (chain[j] / 32 == b) {
                if (step[i] - step[j] >= kLatR) return false;  // older than the ring
                continue;
            }
            const size_t q = static_cast<size_t>(b) * nblocks + step[i] / kLatKU;
            wlo[q] = std::min(wlo[q], step[j]);
            whi[q] = std::max(whi[q], step[j]);
        }
    }
    std::vector<int>& win = out.win;
    win.assign(static_cast<size_t>(nb) * nblocks, -1);
    for (size_t q = 0; q < win.size(); ++q) {
        if (whi[q] < 0) continue;
        if (whi[q] - wlo[q] >= kLatW || wlo[q] >= (1 << 24)) return false;
        win[q] = wlo[q] * 64 + (whi[q] - wlo[q] + 1);
    }
    // records
    const int T = nblocks * kLatKU;
    const size_t blk = static_cast<size_t>(kLatF) * kLatKU * 32;
    auto slot = [&](int f, int b, int lane, int t) {
        const int q = t / kLatKU, u = t % kLatKU;
        return (static_cast<size_t>(b) * nblocks + q) * blk + static_cast<size_t>(f) * kLatKU * 32 +
               static_cast<size_t>(u / 2) * 64 + 2 * lane + (u % 2);
    };
    std::vector<double>& rec = out.rec;
    rec.assign(static_cast<size_t>(nb) * nblocks * blk, 0.0);
    if (rec.size() > static_cast<size_t>(INT32_MAX)) return false;
    auto put_int2 = [&](size_t at, int x, int y) {
        int v[2] = {x, y};
        std::memcpy(&rec[at], v, sizeof v);
    };
    // idle slots: zero coefficients reading the zero cell, no row
    for (int b = 0; b < nb; ++b)
        for (int l = 0; l < 32; ++l)
            for (int t = 0; t < T; ++t) {
                put_int2(slot(5, b, l, t), kLatZero, kLatZero);
                put_int2(slot(6, b, l, t), kLatZero, kLatZero);
                put_int2(slot(7, b, l, t), -1, 0);
            }
    out.bidx.assign(nn, 0);
    for (int i = 0; i < nn; ++i) {
        const int c = chain[i], b = c / 32, l = c % 32, t = step[i];
        out.bidx[i] = static_cast<int>(slot(0, b, l, t));
        int src[4] = {kLatZero, kLatZero, kLatZero, kLatZero};
        int m = 0;
        for (int k = lp[i]; k < lp[i + 1]; ++k, ++m) {
            const int j = lc[k], cj = chain[j];
            rec[slot(1 + m, b, l, t)] = lv[k];
            if (cj / 32 == b)
                src[m] = (cj % 32) * kLatR + (step[j] & (kLatR - 1));
            else
                src[m] = kLatWin + ((t / kLatKU) & 1) * kLatW +
                         (step[j] - (win[static_cast<size_t>(b) * nblocks + t / kLatKU] >> 6));
        }
        put_int2(slot(5, b, l, t), src[0], src[1]);
        put_int2(slot(6, b, l, t), src[2], src[3]);
        put_int2(slot(7, b, l, t), i, lp[i + 1] - lp[i] > 2 ? 1 : 0);
    }
    out.nb = nb;
    out.nblocks = nblocks;
    out.nch = nch;
    return true;
}

// CPU emulation of k_gs_lattice over a host plan (same records, ring, windows,
// boundary buffer and arithmetic), bands in order: the check of the planner.
static void emulate_lattice(const LatticeHost& h, const double* b_nat, double* z) {
    const int KU = kLatKU, T = h.nblocks * KU;
    const size_t blk = static_cast<size_t>(kLatF) * KU * 32;
    std::vector<double> rec = h.rec;
    for (size_t i = 0; i < h.bidx.size(); ++i) rec[h.bidx[i]] = b_nat[i];
    std::vector<double> bnd(static_cast<size_t>(h.nb) * T, 0.0);
    for (int band = 0; band < h.nb; ++band) {
        std::vector<double> vals(kLatVals, 0.0);
        for (int q = 0; q < h.nblocks; ++q) {
            const int w = h.win[static_cast<size_t>(band) * h.nblocks + q];
            for (int l = 0; l < 32; ++l)
                vals[kLatWin + (q & 1) * kLatW + l] =
                    (band > 0 && w >= 0 && l < (w & 63)) ? bnd[static_cast<size_t>(band - 1) * T + (w >> 6) + l] : 0.0;
            const double* B = rec.data() + (static_cast<size_t>(band) * h.nblocks + q) * blk;
            for (int u = 0; u < KU; ++u) {
                const int step = q * KU + u;
                double res[32];
                int rows[32];
                for (int l = 0; l < 32; ++l) {
                    auto f = [&](int fld) { return B[static_cast<size_t>(fld) * KU * 32 + (u / 2) * 64 + 2 * l + u % 2]; };
                    auto fi = [&](int fld) {
                        int v[2];
                        const double d = f(fld);
                        std::memcpy(v, &d, sizeof v);
                        return std::pair<int, int>(v[0], v[1]);
                    };
                    const auto s01 = fi(5), s23 = fi(6), rw = fi(7);
                    const double z0 = vals[s01.first], z1 = vals[s01.second], z2 = vals[s23.first],
                                 z3 = vals[s23.second];
                    const double acc = std::fma(f(2), z1, std::fma(f(1), z0, f(0)));
                    const double wide = (acc + std::fma(f(4), z3, f(3) * z2)) + 0.0;
                    res[l] = rw.second ? wide : acc;
                    rows[l] = rw.first;
                }
                for (int l = 0; l < 32; ++l) {
                    vals[l * kLatR + (step & (kLatR - 1))] = res[l];
                    if (rows[l] >= 0) z[rows[l]] = res[l];
                }
                bnd[static_cast<size_t>(band) * T + step] = res[31];
            }
        }
    }
}

// SDG_GS_LATTICE=0 disables the lattice (GsPlan::build / build_parts; the level walks then run).
bool GsPlan::build_lattice(const HostCsr& a, const std::vector<double>& dinv_h, cudaStream_t s) {
    LatticeHost h;
    if (!plan_lattice(a, dinv_h, h)) return false;
    const int T = h.nblocks * kLatKU;
    n = a.n_rows;  // (build_parts builds its parts through this entry point)
    packed.upload(h.rec, s);
    bidx.upload(h.bidx, s);
    lat_win.upload(h.win, s);
    lat_ticket.resize(1);
    SDG_CUDA(cudaMemsetAsync(lat_ticket.get(), 0, sizeof(unsigned long long), s));
    {
        double sent;
        std::memcpy(&sent, &kLatSent, sizeof sent);
        lat_bnd.upload(std::vector<double>(static_cast<size_t>(2) * h.nb * T, sent), s);
    }
    lattice = true;
    lat_bands = h.nb;
    lat_blocks = h.nblocks;
    walk = false;
    wave = false;
    usable = true;
    if (std::getenv("SDG_DEBUG"))
        std::fprintf(stderr, "[sdg gs lattice] n=%d: %d chains in %d bands, %d steps\n", a.n_rows, h.nch, h.nb, T);
    return true;
}

// Host check of the planner (no GPU): plans the lattice of `a`, runs the
// emulation on b and returns the max |z - z_seq| against the sequential lower
// solve z_i = b_i + sum_{j<i} c_ij z_j (c = -a_ij / d_i); -1 when `a` is not a lattice.
// dev aids: the emulated sweep (host) and the kernel's sweep (device) of the
// lattice of `a` for right-hand side b (the lower solve z = b + C z)
bool lattice_emulate_host(const HostCsr& a, const double* b, double* z) {
    const int n = a.n_rows;
    std::vector<double> dinv(n, 1.0);
    for (int i = 0; i < n; ++i)
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] == i) dinv[i] = 1.0 / a.v[k];
    LatticeHost h;
    if (!plan_lattice(a, dinv, h)) return false;
    emulate_lattice(h, b, z);
    return true;
}

bool lattice_run_device(Context& c, const HostCsr& a, const double* b, double* z, int repeats) {
    const int n = a.n_rows;
    std::vector<double> dinv(n, 1.0);
    for (int i = 0; i < n; ++i)
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] == i) dinv[i] = 1.0 / a.v[k];
    GsPlan g;
    g.n = n;
    if (!g.build_lattice(a, dinv, c.stream)) return false;
    std::vector<double> rec(g.packed.size());
    std::vector<int> bx(n);
    SDG_CUDA(cudaMemcpy(rec.data(), g.packed.get(), rec.size() * 8, cudaMemcpyDeviceToHost));
    SDG_CUDA(cudaMemcpy(bx.data(), g.bidx.get(), n * sizeof(int), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) rec[bx[i]] = b[i];
    SDG_CUDA(cudaMemcpy(g.packed.get(), rec.data(), rec.size() * 8, cudaMemcpyHostToDevice));
    DevBuf<double> zd(n);
    for (int r = 0; r < repeats; ++r) launch_gs_lattice(c, g, zd.get());
    SDG_CUDA(cudaStreamSynchronize(c.stream));
    SDG_CUDA(cudaMemcpy(z, zd.get(), n * 8, cudaMemcpyDeviceToHost));
    return true;
}

double lattice_check_host(const HostCsr& a, const double* b) {
    const int n = a.n_rows;
    std::vector<double> dinv(n, 1.0);
    for (int i = 0; i < n; ++i)
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] == i) dinv[i] = 1.0 / a.v[k];
    LatticeHost h;
    if (!plan_lattice(a, dinv, h)) return -1.0;
    std::vector<double> z(n, 0.0), zs(n, 0.0);
    emulate_lattice(h, b, z.data());
    for (int i = 0; i < n; ++i) {
        double acc = b[i];
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] < i) acc += -(a.v[k] * dinv[i]) * zs[a.ci[k]];
        zs[i] = acc;
    }
    double err = 0.0;
    for (int i = 0; i < n; ++i) err = std::max(err, std::abs(z[i] - zs[i]));
    return err;
}

void launch_gs_lattice(Context& c, const GsPlan& g, double* z_new) {
    static const bool attr = [] {
        SDG_CUDA(cudaFuncSetAttribute(k_gs_lattice, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(lat_smem_bytes())));
        return true;
    }();
    (void)attr;
    LatArgs a{g.records(), g.lat_win.get(), z_new, g.lat_bnd.get(), g.lat_ticket.get(), g.lat_bands, g.lat_blocks};
    launch_k(c, k_gs_lattice, g.lat_bands, 32, lat_smem_bytes(), a);
}

}  // namespace sdg
