// Multi-SM lattice lower solve for the aggregated coarse levels of the
// smoother (sor_sweep, precond.cpp:92-108, lower part of one forward sweep).
//
// The first coarse levels of the velocity and porous hierarchies are
// aggregations of the structured finest grids (precond.cpp:122-175): the
// aggregates form rows, and the lexicographic lower triangle of a coarse
// level is a lattice -- every aggregate depends on its west neighbour in its
// own aggregate row and on two or three aggregates of the row below.  The
// level walk (gs_walk.cu) pays a CTA-wide hand-off per dependency level
// (~300-500 cycles, one SM); here the rows are cut into CHAINS and each chain
// is a lane, as the wavefront does for the finest grids (gs_wave.cu):
//
//   * a chain is a sequence of rows each of which depends on its predecessor
//     (row i joins the chain whose last row is i's most recent lower
//     neighbour; otherwise it starts a chain).  Chains ordered by their first
//     row are the lanes; 32 consecutive chains are a band, one warp, one CTA;
//   * every row gets a step: one after its chain predecessor and one after
//     each lower neighbour in its band, so the schedule is a topological
//     order of the lower triangle and the sweep stays the exact lexicographic
//     Gauss-Seidel sweep.  A lane with no row at a step runs a zero record;
//   * a lane keeps its last three values in registers (h1..h3) and the last
//     four values of the lane below in a shift register fed by one warp
//     shuffle per step (p1..p4): a row may depend on its own chain 1..3 steps
//     back and on the chain below 1..4 steps back (the lattices of the c3
//     coarse levels need exactly that).  Lane 0's chain-below is the last
//     chain of the previous band: its lane 31 stores every step's value into
//     a boundary buffer that holds a sentinel until written (the value is its
//     own flag, as in gs_wave.cu), and lane 0 reads a window of it, loaded one
//     block ahead into shared memory;
//   * records [block][field][KU/2 step pairs][32 lanes][2] are streamed by
//     1-D TMA bulk copies into a shared-memory ring, as in gs_wave.cu.
//
// Arithmetic: z = b + sum c_s v_s over the seven sources in a fixed order
// (p4, p3, p2, p1, h3, h2, h1; fma chain, c = -a_ij / d_i, zero coefficients
// for absent sources), so the newest values enter last.  That is a
// reassociation of the row sum (the level walk sums in column order): equal to
// the reference sweep to rounding, like the rest of the fast smoother.  Levels
// that are not such a lattice keep the level walk.
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
constexpr int kLatF = 9;        // record fields: b, c_h1..c_h3, c_p1..c_p4, (rowid, lane-0 window slots)
constexpr int kLatDepth = 4;    // blocks of records in flight
constexpr int kLatW = 32;       // window steps of the previous band's last chain
constexpr int kLatVals = 2 * kLatW;  // the two windows (block parity) in shared memory
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
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\nmov.b64 %0, 0;\n@q ld.relaxed.gpu.f64 %0, [%1];\n}"
                 : "=d"(v)
                 : "l"(p), "r"(static_cast<int>(pred))
                 : "memory");
    return v;
}
__device__ __forceinline__ void lat_st_relaxed_if(double* p, double v, bool pred) {
    const double w = v + 0.0;  // quiets a signalling NaN: a stored value is never the sentinel
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.relaxed.gpu.f64 [%0], %1;\n}" ::"l"(p),
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

// One warp per band, W consecutive bands per CTA, D blocks of records in flight
// per band; all control flow warp-uniform (per-lane work predicated).  Two
// bands of one CTA hand the last chain's values over through shared memory
// (value-as-flag slots filled with the sentinel at kernel start); the first
// band of a CTA polls the previous CTA's boundary in L2.  Generic-address
// loads and stores serve both.
template <int W, int D>
__global__ void __launch_bounds__(32 * W, 1) k_gs_lattice(LatArgs a) {
    constexpr int KU = kLatKU, F = kLatF, BLK = F * KU * 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ unsigned long long s_ticket;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* base = reinterpret_cast<double*>(smem_raw);
    double* ring = base + warp * (D * BLK);                              // records
    double* wins = base + W * D * BLK + warp * kLatVals;                 // two windows
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + W * D * BLK + W * kLatVals) + warp * D;
    double* sh_bnd = base + W * D * BLK + W * kLatVals + W * D;          // inbound boundaries of warps 1 .. W-1
    const int T = a.nblocks * KU;
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.ticket, 1ull);
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) ptx::mbar_init(bars + d, 1);
        ptx::fence_mbar_init();
    }
    if (W > 1 && warp > 0) {
        double* mine = sh_bnd + static_cast<size_t>(warp - 1) * T;
        for (int k = lane; k < T; k += 32) mine[k] = __longlong_as_double(static_cast<long long>(kLatSent));
    }
    __syncthreads();
    const unsigned long long t = s_ticket;
    const unsigned long long nctas = static_cast<unsigned long long>((a.nbands + W - 1) / W);
    const int band = static_cast<int>(t % nctas) * W + warp;
    const int par = static_cast<int>((t / nctas) & 1ull);
    if (band >= a.nbands) return;
    pdl_wait();  // b is written by the prep kernel; the previous launch of this plan is complete
    pdl_trigger();
    const double* src = a.rec + static_cast<size_t>(band) * a.nblocks * BLK;
    for (int d = 0; d < D && d < a.nblocks; ++d)
        lat_tma_if(ring + d * BLK, src + static_cast<size_t>(d) * BLK, BLK * 8, bars + d, lane == 0);
    const bool has_src = band > 0, has_dst = band + 1 < a.nbands;
    const bool src_sh = W > 1 && warp > 0, dst_sh = W > 1 && warp + 1 < W && has_dst;
    const size_t pstride = static_cast<size_t>(a.nbands) * T;
    const double* b_in = src_sh ? sh_bnd + static_cast<size_t>(warp - 1) * T
                                : a.bnd + par * pstride + static_cast<size_t>(has_src ? band - 1 : 0) * T;
    double* b_out = dst_sh ? sh_bnd + static_cast<size_t>(warp) * T : a.bnd + par * pstride + static_cast<size_t>(band) * T;
    if (has_src && !src_sh) {  // the other parity's input slots, for the next launch
        double* rs = a.bnd + (par ^ 1) * pstride + static_cast<size_t>(band - 1) * T;
        for (int k = lane; k < T; k += 32) rs[k] = __longlong_as_double(static_cast<long long>(kLatSent));
    }
    const int* win = a.win + static_cast<size_t>(band) * a.nblocks;
    // win[q] = first step * 64 + steps needed (<= 32), or -1: no window
    auto load_win = [&](int q) {
        const int w = q < a.nblocks ? win[q] : -1;
        return lat_ld_if(b_in + (w >> 6) + lane, has_src && w >= 0 && lane < (w & 63));
    };
    auto settle = [&](int q, double& v) {
        const int w = q < a.nblocks ? win[q] : -1;
        while (!__all_sync(0xffffffffu, lat_ready(v)))
            v = lat_ld_if(b_in + (w >> 6) + lane, has_src && w >= 0 && lane < (w & 63));
        wins[(q & 1) * kLatW + lane] = v;
    };
    double wv = load_win(0);
    settle(0, wv);
    const bool pub = has_dst && lane == 31;
    double h1 = 0.0, h2 = 0.0, h3 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0, p4 = 0.0;
    for (int q = 0; q < a.nblocks; ++q) {
        double wn = load_win(q + 1);  // in flight during this block
        const int slot = q % D;
        ptx::mbar_wait(bars + slot, (q / D) & 1);
        __syncwarp();  // the window stored at the end of the previous block
        const double2* B = reinterpret_cast<const double2*>(ring + slot * BLK) + lane;
        const double* W = wins + (q & 1) * kLatW;
#pragma unroll
        for (int u2 = 0; u2 < KU / 2; ++u2) {
            double2 R[F];
#pragma unroll
            for (int f = 0; f < F; ++f) R[f] = B[(f * KU / 2 + u2) * 32];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                auto r = [&](int f) { return h ? R[f].y : R[f].x; };
                const int2 rw = *reinterpret_cast<const int2*>(h ? &R[8].y : &R[8].x);
                // the lane below, one step back (lane 0: its register is lane 31's, unused)
                const double pn = __shfl_up_sync(0xffffffffu, h1, 1);
                p4 = p3;
                p3 = p2;
                p2 = p1;
                p1 = pn;
                double P1 = p1, P2 = p2, P3 = p3, P4 = p4;
                if (has_src) {  // lane 0: the previous band's last chain, from the window
                    const unsigned ws = static_cast<unsigned>(rw.y);
                    const double w1 = W[ws & 31], w2 = W[(ws >> 8) & 31], w3 = W[(ws >> 16) & 31],
                                 w4 = W[(ws >> 24) & 31];
                    if (lane == 0) {
                        P1 = w1;
                        P2 = w2;
                        P3 = w3;
                        P4 = w4;
                    }
                }
                double acc = fma(r(7), P4, r(0));
                acc = fma(r(6), P3, acc);
                acc = fma(r(5), P2, acc);
                acc = fma(r(4), P1, acc);
                acc = fma(r(3), h3, acc);
                acc = fma(r(2), h2, acc);
                const double res = fma(r(1), h1, acc);
                h3 = h2;
                h2 = h1;
                h1 = res;
                const int step = q * KU + 2 * u2 + h;
                lat_st_if(a.z + rw.x, res, rw.x >= 0);
                lat_st_relaxed_if(b_out + step, res, pub);
            }
        }
        __syncwarp();  // every lane has read the record slot and the window
        lat_tma_if(ring + slot * BLK, src + static_cast<size_t>(q + D) * BLK, BLK * 8, bars + slot,
                   lane == 0 && q + D < a.nblocks);
        if (q + 1 < a.nblocks) settle(q + 1, wn);
    }
}

size_t lat_smem_bytes(int w, int d, int steps) {
    return static_cast<size_t>(w) * (static_cast<size_t>(d) * kLatF * kLatKU * 32 * sizeof(double) +
                                     kLatVals * sizeof(double) + d * sizeof(uint64_t)) +
           static_cast<size_t>(w - 1) * steps * sizeof(double);
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
        if (lp[i + 1] - lp[i] > 7) return false;
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
            else if (!(bj == b - 1 && cj % 32 == 31 && c % 32 == 0))
                return false;  // across bands only: lane 0 <- the previous band's last chain
        }
        step[i] = tt;
        last_step[c] = tt;
        tmax = std::max(tmax, tt);
    }
    const int nblocks = (tmax + 1 + kLatKU - 1) / kLatKU;
    // windows: per consumer block, the steps of the previous band's last chain lane 0 reads
    std::vector<int> wlo(static_cast<size_t>(nb) * nblocks, INT32_MAX), whi(static_cast<size_t>(nb) * nblocks, -1);
    for (int i = 0; i < nn; ++i) {
        const int b = chain[i] / 32;
        for (int k = lp[i]; k < lp[i + 1]; ++k) {
            const int j = lc[k];
            if (chain[j] / 32 == b) continue;
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
    for (int b = 0; b < nb; ++b)  // no row: no store
        for (int l = 0; l < 32; ++l)
            for (int t = 0; t < T; ++t) put_int2(slot(8, b, l, t), -1, 0);
    out.bidx.assign(nn, 0);
    for (int i = 0; i < nn; ++i) {
        const int c = chain[i], b = c / 32, l = c % 32, t = step[i];
        out.bidx[i] = static_cast<int>(slot(0, b, l, t));
        // window deps of lane 0, newest first -> P1, P2, ...
        std::vector<std::pair<int, double>> wdeps;
        for (int k = lp[i]; k < lp[i + 1]; ++k) {
            const int j = lc[k], cj = chain[j];
            if (cj / 32 != b) {
                wdeps.push_back({step[j], lv[k]});
                continue;
            }
            const int age = t - step[j];
            int field;
            if (cj == c) {  // own chain, age 1..3 -> h1..h3
                if (age < 1 || age > 3) return false;
                field = age;
            } else if (cj % 32 == l - 1) {  // the chain below, age 1..4 -> p1..p4
                if (age < 1 || age > 4) return false;
                field = 3 + age;
            } else {
                return false;
            }
            rec[slot(field, b, l, t)] = lv[k];
        }
        unsigned ws = 0;
        if (!wdeps.empty()) {
            if (wdeps.size() > 4) return false;
            std::sort(wdeps.begin(), wdeps.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
            const int w0 = win[static_cast<size_t>(b) * nblocks + t / kLatKU] >> 6;
            for (size_t k = 0; k < wdeps.size(); ++k) {
                rec[slot(4 + static_cast<int>(k), b, l, t)] = wdeps[k].second;
                ws |= static_cast<unsigned>(wdeps[k].first - w0) << (8 * k);
            }
        }
        put_int2(slot(8, b, l, t), i, static_cast<int>(ws));
    }
    out.nb = nb;
    out.nblocks = nblocks;
    out.nch = nch;
    return true;
}

// CPU emulation of k_gs_lattice over a host plan (same records, registers,
// windows, boundary buffer and arithmetic), bands in order: the check of the
// planner.
static void emulate_lattice(const LatticeHost& h, const double* b_nat, double* z) {
    const int KU = kLatKU, T = h.nblocks * KU;
    const size_t blk = static_cast<size_t>(kLatF) * KU * 32;
    std::vector<double> rec = h.rec;
    for (size_t i = 0; i < h.bidx.size(); ++i) rec[h.bidx[i]] = b_nat[i];
    std::vector<double> bnd(static_cast<size_t>(h.nb) * T, 0.0);
    for (int band = 0; band < h.nb; ++band) {
        double H[32][3] = {}, Pp[32][4] = {};
        double Wn[kLatW];
        for (int q = 0; q < h.nblocks; ++q) {
            const int w = h.win[static_cast<size_t>(band) * h.nblocks + q];
            for (int l = 0; l < kLatW; ++l)
                Wn[l] = (band > 0 && w >= 0 && l < (w & 63)) ? bnd[static_cast<size_t>(band - 1) * T + (w >> 6) + l]
                                                             : 0.0;
            const double* B = rec.data() + (static_cast<size_t>(band) * h.nblocks + q) * blk;
            for (int u = 0; u < KU; ++u) {
                const int step = q * KU + u;
                double pn[32];
                for (int l = 0; l < 32; ++l) pn[l] = l > 0 ? H[l - 1][0] : H[31][0];
                double res[32];
                for (int l = 0; l < 32; ++l) {
                    auto f = [&](int fld) { return B[static_cast<size_t>(fld) * KU * 32 + (u / 2) * 64 + 2 * l + u % 2]; };
                    int rw[2];
                    const double d8 = f(8);
                    std::memcpy(rw, &d8, sizeof rw);
                    double* P = Pp[l];
                    P[3] = P[2];
                    P[2] = P[1];
                    P[1] = P[0];
                    P[0] = pn[l];
                    double v[4] = {P[0], P[1], P[2], P[3]};
                    if (band > 0 && l == 0) {
                        const unsigned ws = static_cast<unsigned>(rw[1]);
                        for (int k = 0; k < 4; ++k) v[k] = Wn[(ws >> (8 * k)) & 31];
                    }
                    double acc = std::fma(f(7), v[3], f(0));
                    acc = std::fma(f(6), v[2], acc);
                    acc = std::fma(f(5), v[1], acc);
                    acc = std::fma(f(4), v[0], acc);
                    acc = std::fma(f(3), H[l][2], acc);
                    acc = std::fma(f(2), H[l][1], acc);
                    res[l] = std::fma(f(1), H[l][0], acc);
                    if (rw[0] >= 0) z[rw[0]] = res[l];
                }
                for (int l = 0; l < 32; ++l) {
                    H[l][2] = H[l][1];
                    H[l][1] = H[l][0];
                    H[l][0] = res[l];
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
    // bands (warps) per CTA and blocks in flight per band: (2, 4) by default,
    // (3, 3) / (4, 2) trade record look-ahead for fewer hand-offs through L2
    // (SDG_LAT_W = 1..4); whatever shared memory holds
    {
        constexpr size_t kSmemMax = 226 * 1024;  // 227 KB per CTA minus the static words
        int w = 2;
        if (const char* e = std::getenv("SDG_LAT_W")) w = std::max(1, std::min(4, std::atoi(e)));
        w = std::min(w, h.nb);
        auto depth = [](int ww) { return ww <= 2 ? 4 : ww == 3 ? 3 : 2; };
        while (w > 1 && lat_smem_bytes(w, depth(w), T) > kSmemMax) --w;
        lat_w = w;
        lat_depth = depth(w);
        lat_smem = lat_smem_bytes(lat_w, lat_depth, T);
    }
    walk = false;
    wave = false;
    usable = true;
    if (std::getenv("SDG_DEBUG"))
        std::fprintf(stderr, "[sdg gs lattice] n=%d: %d chains in %d bands (%d per CTA), %d steps\n", a.n_rows, h.nch,
                     h.nb, lat_w, T);
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
        for (auto k : {k_gs_lattice<1, 4>, k_gs_lattice<2, 4>, k_gs_lattice<3, 3>, k_gs_lattice<4, 2>})
            SDG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
        return true;
    }();
    (void)attr;
    LatArgs a{g.records(), g.lat_win.get(), z_new, g.lat_bnd.get(), g.lat_ticket.get(), g.lat_bands, g.lat_blocks};
    void (*k)(LatArgs) = g.lat_w == 4 ? k_gs_lattice<4, 2> : g.lat_w == 3 ? k_gs_lattice<3, 3>
                         : g.lat_w == 2 ? k_gs_lattice<2, 4> : k_gs_lattice<1, 4>;
    launch_k(c, k, (g.lat_bands + g.lat_w - 1) / g.lat_w, 32 * g.lat_w, g.lat_smem, a);
}

}  // namespace sdg
