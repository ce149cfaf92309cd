// Multi-SM wavefront lower solve for the structured finest levels of the
// smoother (sor_sweep, precond.cpp:92-108, lower part of one forward sweep).
//
// The finest velocity block (MAC u / v, grid.hpp:28-36) and the finest Darcy
// block (TPFA, 5-point) have a lexicographic lower triangle whose
// dependencies point one cell west or one cell south, plus, for a v row, the
// four u neighbours of the same and the previous cell row (assembly.cpp:
// 134-215).  That is a 2-D wavefront with one short recurrence per grid row:
//
//   * lane L of a band (one warp) owns grid row j = 32 * band + L and walks it
//     west to east, one cell per step, one step behind lane L - 1: the west
//     value stays in a register, the south values come from lane L - 1's
//     previous step by warp shuffle;
//   * bands are separate CTAs (one warp each) on separate SMs.  Lane 31 of a
//     band also stores each value of its row into a boundary buffer whose
//     slots hold a sentinel until written, and lane 0 of the band above polls
//     those slots (L2, relaxed loads, one block of KU columns ahead): the
//     value is its own ready flag, so the hand-off needs no fence, no flag
//     and no acquire.  Bands run as a pipeline whose depth is the wavefront's
//     own (columns + rows steps) plus about one block and one L2 round trip
//     per band;
//   * band ids come from a ticket counter (atomicAdd), so the band a CTA waits
//     for always belongs to a CTA that started earlier (no co-residency
//     assumption); the boundary buffer has two parities (launch e uses e % 2
//     and resets the other), so a captured CUDA graph replays the kernel
//     unchanged;
//   * the records of a band, [block][field][KU/2 step pairs][32 lanes][2], are streamed
//     into a shared-memory ring by 1-D TMA bulk copies (cp.async.bulk +
//     mbarrier), one copy per block, so every step reads its coefficients
//     from shared memory with conflict-free 8-byte loads.
//
// b (the prep kernels' output, gs.cu) lives in the same record array: the
// plan's bidx points each row at its b slot, so the prep kernels are shared
// with every other plan.
//
// Arithmetic (bitwise equal to the level walk of gs_walk.cu, and for the MAC
// block to its label-block form, u block then v block with the coupling step
// k_gs_couple in between): the lower entries of a row in column order,
//   5-point / u row:  z = fma(c_W, z_W, fma(c_S, z_S, b))
//   v row:            acc = 0; acc = fma(c_u, u, acc) over the four u
//                     neighbours in column order; b' = b + acc;
//                     z = fma(c_W, v_W, fma(c_S, v_S, b'))
// with c = -a_ij / d_i.  The exact lexicographic Gauss-Seidel order is kept:
// every row still sees the new values of all its lower neighbours.
#include "gs.cuh"
#include "launch.cuh"
#include "ptx.cuh"

#include <algorithm>
#include <cstring>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace sdg {

namespace {

constexpr int kWaveDepth = 4;  // blocks of records in flight per band

template <int KIND>
struct WaveShape;
template <>
struct WaveShape<1> {  // 5-point: b, c_S, c_W
    static constexpr int F = 3, KU = 16;
};
template <>
struct WaveShape<2> {  // MAC: bu, cu_S, cu_W, bv, c_u(i',j-1), c_u(i'+1,j-1), c_u(i',j), c_u(i'+1,j), cv_S, cv_W
    static constexpr int F = 10, KU = 8;
};

struct WaveArgs {
    const double* rec;              // [band][block][F][KU / 2][32][2]
    double* z;                      // natural order
    double* bnd;                    // [2 parities][nbands - 1][fields][bcols]: top rows of the bands
    unsigned long long* ticket;     // band tickets handed out so far
    int nbands, nblocks;
    int nx;                         // 5-point: columns; MAC: m (u rows have m + 1 cells, v rows m)
    int ny;                         // grid rows (5-point ny; MAC m + 1)
    int n_u;                        // MAC: m (m + 1)
    int bcols;                      // boundary slots per field (5-point nx; MAC m + 1)
    unsigned long long* tl;         // dev timeline (SDG_WAVE_TL=1): per band {start, first block, end, wait ns}
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// The hand-off between bands carries no flags: a slot of the boundary buffer
// holds kSent until the band below stores the value, and the value is its own
// ready flag (8-byte single-copy atomic stores and loads, relaxed at gpu
// scope, so neither side needs a fence).  Launch e uses parity e % 2 and
// resets parity (e + 1) % 2, which launch e - 1 used and launch e + 1 will
// use; launches of one plan are ordered (each starts with griddepcontrol.wait).
constexpr unsigned long long kSent = 0x7ff4deadbeefcafeull;  // a signalling-NaN payload arithmetic never makes

__device__ __forceinline__ bool not_sent(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) != kSent;
}
// Everything inside the step loop is warp-uniform control flow; per-lane work
// (lane 0's boundary loads, lane 31's boundary stores, the elected bulk copy)
// is predicated, never branched: a lane-divergent branch there makes the
// compiler's divergent-warp fallback (collective shuffles) run the block.
__device__ __forceinline__ double ld_relaxed_if(const double* p, bool pred) {
    double v;
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\nmov.b64 %0, 0;\n@q ld.relaxed.gpu.f64 %0, [%1];\n}"
                 : "=d"(v)
                 : "l"(p), "r"(static_cast<int>(pred))
                 : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_if(double* p, double v, bool pred) {
    // v + 0 quiets a signalling NaN, so a stored value is never the sentinel
    // (and it equals v otherwise, up to the sign of a zero)
    const double w = v + 0.0;
    // no "memory" clobber: nothing this thread reads depends on the store, so
    // the compiler may keep scheduling the next step's shared loads across it
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.relaxed.gpu.f64 [%0], %1;\n}" ::"l"(p),
                 "d"(w), "r"(static_cast<int>(pred)));
}
// predicated store without a branch around it (the step loop stays convergent)
__device__ __forceinline__ void st_global_if(double* p, double v, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global.f64 [%0], %1;\n}" ::"l"(p), "d"(v),
                 "r"(static_cast<int>(pred)));
}
// refill a ring slot: order the slot's shared loads before the async-proxy
// write, arm the slot's mbarrier and issue the 1-D bulk copy (one lane)
__device__ __forceinline__ void tma_block_if(double* dst, const double* src, unsigned bytes, uint64_t* bar,
                                             bool pred) {
    asm volatile(
        "{\n.reg .pred q;\nsetp.ne.b32 q, %4, 0;\n"
        "@q fence.proxy.async.shared::cta;\n"
        "@q mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n"
        "@q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}" ::"r"(
            ptx::smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(ptx::smem_addr(bar)), "r"(static_cast<int>(pred))
        : "memory");
}

// W warps per CTA, one band each (consecutive bands).  The hand-off between
// two bands of one CTA goes through shared memory (the same value-as-flag
// slots, filled with the sentinel at kernel start); only the first band of a
// CTA polls the previous CTA's boundary in L2.  The loads and stores use
// generic addresses, so one code path serves both.
template <int KIND, int W>
__global__ void __launch_bounds__(32 * W, 1) k_gs_wave(WaveArgs a) {
    constexpr int F = WaveShape<KIND>::F, KU = WaveShape<KIND>::KU;
    constexpr int NBF = KIND == 1 ? 1 : 2;  // boundary fields: z, or u and v
    constexpr int BLK = F * KU * 32;        // doubles per block
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ unsigned long long s_ticket;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* ring = reinterpret_cast<double*>(smem_raw) + warp * (kWaveDepth * BLK);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(smem_raw) + W * kWaveDepth * BLK) +
                     warp * kWaveDepth;
    const size_t bstride = static_cast<size_t>(NBF) * a.bcols;                 // one band boundary
    // inbound boundaries of warps 1 .. W-1 (shared memory)
    double* sh_bnd = reinterpret_cast<double*>(smem_raw) + W * kWaveDepth * BLK + W * kWaveDepth;
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.ticket, 1ull);
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < kWaveDepth; ++d) ptx::mbar_init(bars + d, 1);
        ptx::fence_mbar_init();
    }
    if (W > 1 && warp > 0) {
        double* mine = sh_bnd + (warp - 1) * bstride;
        for (size_t k = lane; k < bstride; k += 32) mine[k] = __longlong_as_double(static_cast<long long>(kSent));
    }
    __syncthreads();
    const unsigned long long t = s_ticket;
    const unsigned long long nctas = static_cast<unsigned long long>((a.nbands + W - 1) / W);
    const int band = static_cast<int>(t % nctas) * W + warp;
    const int par = static_cast<int>((t / nctas) & 1ull);
    if (band >= a.nbands) return;
    pdl_wait();  // b is written by the prep kernel before this launch; the previous launch is done
    pdl_trigger();
    const double* src = a.rec + static_cast<size_t>(band) * a.nblocks * BLK;
    for (int d = 0; d < kWaveDepth && d < a.nblocks; ++d)
        tma_block_if(ring + d * BLK, src + static_cast<size_t>(d) * BLK, BLK * 8, bars + d, lane == 0);
    const int j = band * 32 + lane;
    const bool has_src = band > 0, has_dst = band + 1 < a.nbands;
    const bool src_sh = W > 1 && warp > 0, dst_sh = W > 1 && warp + 1 < W && has_dst;
    unsigned long long wait_ns = 0, t_start = a.tl ? gtimer() : 0, t_first = 0, tma_cyc = 0, comp_cyc = 0;
    const size_t pstride = static_cast<size_t>(a.nbands - 1) * bstride;         // one parity
    const double* sb_in = src_sh    ? sh_bnd + (warp - 1) * bstride
                          : has_src ? a.bnd + par * pstride + (band - 1) * bstride
                                    : a.bnd;                                                 // read (lane 0)
    double* sb_out = dst_sh ? sh_bnd + warp * bstride
                            : a.bnd + par * pstride + (has_dst ? band : 0) * bstride;        // written (lane 31)
    if (has_src && !src_sh) {  // reset the input slots of the other parity for the next launch
        double* rs = a.bnd + (par ^ 1) * pstride + (band - 1) * bstride;
        for (size_t k = lane; k < bstride; k += 32) rs[k] = __longlong_as_double(static_cast<long long>(kSent));
    }

    if constexpr (KIND == 1) {
        const int nx = a.nx;
        // block q, step s = q KU + u: lane 0 reads z(s, j - 1) = sb[u]
        double sb[KU], nsb[KU];
        auto load_bnd = [&](int q, double (&o)[KU]) {
            const bool on = has_src && lane == 0 && q < a.nblocks;
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                const int c = q * KU + u;
                o[u] = ld_relaxed_if(sb_in + c, on && c < nx);
            }
        };
        // warp-uniform wait until every value of the block has been stored
        auto settle = [&](int q, double (&o)[KU]) {
            const unsigned long long t0 = a.tl ? gtimer() : 0;
            for (;;) {
                bool ok = true;
#pragma unroll
                for (int u = 0; u < KU; ++u) ok = ok && not_sent(o[u]);
                if (__all_sync(0xffffffffu, ok)) break;
                load_bnd(q, o);
            }
            if (a.tl) wait_ns += gtimer() - t0;
        };
        load_bnd(0, sb);
        settle(0, sb);
        if (a.tl) t_first = gtimer();
        double last = 0.0;
        double* zrow = a.z + static_cast<size_t>(j) * nx;
        const bool row_ok = j < a.ny;
        const bool pub = has_dst && lane == 31;
        for (int q = 0; q < a.nblocks; ++q) {
            load_bnd(q + 1, nsb);  // in flight during this block
            const int slot = q % kWaveDepth;
            ptx::mbar_wait(bars + slot, (q / kWaveDepth) & 1);
            const double2* B = reinterpret_cast<const double2*>(ring + slot * BLK) + lane;
            auto run_block = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
            for (int u2 = 0; u2 < KU / 2; ++u2) {
                const double2 b2 = B[(0 * KU / 2 + u2) * 32], cs2 = B[(1 * KU / 2 + u2) * 32],
                              cw2 = B[(2 * KU / 2 + u2) * 32];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int u = 2 * u2 + h;
                    double south = __shfl_up_sync(0xffffffffu, last, 1);
                    if (lane == 0) south = sb[u];
                    // padding slots (before a lane's first column, after its
                    // last) hold zero records, so they compute 0: no select
                    last = fma(h ? cw2.y : cw2.x, last, fma(h ? cs2.y : cs2.x, south, h ? b2.y : b2.x));
                    const int i = q * KU + u - lane;
                    const bool act = FULL ? row_ok : (row_ok && i >= 0 && i < nx);
                    st_global_if(zrow + i, last, act);
                    st_relaxed_if(sb_out + i, last, act && pub);
                }
            }
            };
            if (q * KU - 31 >= 0 && q * KU + KU - 1 < nx)
                run_block(std::true_type{});
            else
                run_block(std::false_type{});
            __syncwarp();  // every lane has read the slot
            tma_block_if(ring + slot * BLK, src + static_cast<size_t>(q + kWaveDepth) * BLK, BLK * 8, bars + slot,
                         lane == 0 && q + kWaveDepth < a.nblocks);
            settle(q + 1, nsb);
#pragma unroll
            for (int u = 0; u < KU; ++u) sb[u] = nsb[u];
        }
    } else {
        const int m = a.nx;
        const double* su_in = sb_in;              // u(., j-1), m + 1 slots
        const double* sv_in = sb_in + a.bcols;    // v(., j-1), m slots
        double* su_out = sb_out;
        double* sv_out = sb_out + a.bcols;
        double bu[KU + 1], bv[KU], nbu[KU + 1], nbv[KU];
        // block q, step s = q KU + u (lane 0: u column s, v column s - 1) reads
        // u(s, j-1) = bu[u + 1], u(s - 1, j-1) = bu[u], v(s - 1, j-1) = bv[u]
        auto load_bnd = [&](int q, double (&ou)[KU + 1], double (&ov)[KU]) {
            const bool on = has_src && lane == 0 && q < a.nblocks;
#pragma unroll
            for (int k = 0; k <= KU; ++k) {
                const int c = q * KU - 1 + k;
                ou[k] = ld_relaxed_if(su_in + c, on && c >= 0 && c <= m);
            }
#pragma unroll
            for (int k = 0; k < KU; ++k) {
                const int c = q * KU - 1 + k;
                ov[k] = ld_relaxed_if(sv_in + c, on && c >= 0 && c < m);
            }
        };
        auto settle = [&](int q, double (&ou)[KU + 1], double (&ov)[KU]) {
            const unsigned long long t0 = a.tl ? gtimer() : 0;
            for (;;) {
                bool ok = not_sent(ou[KU]);
#pragma unroll
                for (int k = 0; k < KU; ++k) ok = ok && not_sent(ou[k]) && not_sent(ov[k]);
                if (__all_sync(0xffffffffu, ok)) break;
                load_bnd(q, ou, ov);
            }
            if (a.tl) wait_ns += gtimer() - t0;
        };
        load_bnd(0, bu, bv);
        settle(0, bu, bv);
        if (a.tl) t_first = gtimer();
        double u_last = 0.0, u_last2 = 0.0, v_last = 0.0;
        double* zu = a.z + static_cast<size_t>(j) * (m + 1);
        double* zv = a.z + a.n_u + static_cast<size_t>(j) * m - 1;  // indexed by u column i = v column + 1
        const bool u_row = j < m, v_row = j <= m;
        const bool pub = has_dst && lane == 31;
        for (int q = 0; q < a.nblocks; ++q) {
            load_bnd(q + 1, nbu, nbv);  // in flight during this block
            const int slot = q % kWaveDepth;
            const long long c0 = a.tl ? clock64() : 0;
            ptx::mbar_wait(bars + slot, (q / kWaveDepth) & 1);
            const long long c1 = a.tl ? clock64() : 0;
            const double2* B = reinterpret_cast<const double2*>(ring + slot * BLK) + lane;
            // every lane inside its u and v rows for the whole block: no
            // per-step column tests (the interior blocks, most of the sweep)
            auto run_block = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
            for (int u2 = 0; u2 < KU / 2; ++u2) {
                double2 R[F];
#pragma unroll
                for (int f = 0; f < F; ++f) R[f] = B[(f * KU / 2 + u2) * 32];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int u = 2 * u2 + h;
                    auto r = [&](int f) { return h ? R[f].y : R[f].x; };
                    double su1 = __shfl_up_sync(0xffffffffu, u_last, 1);   // u(i, j-1)
                    double su2 = __shfl_up_sync(0xffffffffu, u_last2, 1);  // u(i-1, j-1)
                    double sv1 = __shfl_up_sync(0xffffffffu, v_last, 1);   // v(i-1, j-1)
                    if (lane == 0) {
                        su1 = bu[u + 1];
                        su2 = bu[u];
                        sv1 = bv[u];
                    }
                    // u(i, j); padding slots hold zero records and compute 0
                    const double un = fma(r(2), u_last, fma(r(1), su1, r(0)));
                    // v(i' = i - 1, j): u neighbours in column order
                    double acc = fma(r(4), su2, 0.0);   // u(i', j-1)
                    acc = fma(r(5), su1, acc);          // u(i'+1, j-1)
                    acc = fma(r(6), u_last, acc);       // u(i', j)
                    acc = fma(r(7), un, acc);           // u(i'+1, j)
                    const double vn = fma(r(9), v_last, fma(r(8), sv1, r(3) + acc));
                    const int i = q * KU + u - lane;
                    const bool ua = FULL ? u_row : (u_row && i >= 0 && i <= m);
                    const bool va = FULL ? v_row : (v_row && i >= 1 && i <= m);
                    st_global_if(zu + i, un, ua);
                    st_global_if(zv + i, vn, va);
                    st_relaxed_if(su_out + i, un, ua && pub);
                    st_relaxed_if(sv_out + i - 1, vn, va && pub);
                    u_last2 = u_last;
                    u_last = un;
                    v_last = vn;
                }
            }
            };
            if (q * KU - 31 >= 1 && q * KU + KU - 1 <= m)
                run_block(std::true_type{});
            else
                run_block(std::false_type{});
            if (a.tl) {
                const long long c2 = clock64();
                tma_cyc += c1 - c0;
                comp_cyc += c2 - c1;
            }
            __syncwarp();  // every lane has read the slot
            tma_block_if(ring + slot * BLK, src + static_cast<size_t>(q + kWaveDepth) * BLK, BLK * 8, bars + slot,
                         lane == 0 && q + kWaveDepth < a.nblocks);
            settle(q + 1, nbu, nbv);
#pragma unroll
            for (int k = 0; k <= KU; ++k) bu[k] = nbu[k];
#pragma unroll
            for (int k = 0; k < KU; ++k) bv[k] = nbv[k];
        }
    }
    if (a.tl && lane == 0) {
        unsigned long long* o = a.tl + 8 * band;
        o[4] = tma_cyc;
        o[5] = comp_cyc;
        o[0] = t_start;
        o[1] = t_first;
        o[2] = gtimer();
        o[3] = wait_ns;
    }
}

template <int KIND>
size_t wave_smem_bytes(int w, int bcols) {
    const size_t nbf = KIND == 1 ? 1 : 2;
    return static_cast<size_t>(w) * (static_cast<size_t>(kWaveDepth) * WaveShape<KIND>::F * WaveShape<KIND>::KU * 32 *
                                         sizeof(double) +
                                     kWaveDepth * sizeof(uint64_t)) +
           static_cast<size_t>(w - 1) * nbf * bcols * sizeof(double);
}

}  // namespace

// Detects the two structured patterns on the plan's matrix and lays out the
// records; returns false (plan untouched) for anything else.  SDG_GS_WAVE=0
// disables it (GsPlan::build; the level walks then run).
bool GsPlan::build_wave(const HostCsr& a, const std::vector<int>& comps, const std::vector<double>& dinv_h,
                        cudaStream_t s) {
    const int nn = a.n_rows;
    if (nn < 64) return false;
    int kind = 0, nx = 0, ny = 0, m = 0;
    if (!comps.empty()) {
        int n_u = 0;
        while (n_u < nn && comps[n_u] == 0) ++n_u;
        m = static_cast<int>(std::floor(std::sqrt(static_cast<double>(n_u))));
        while (static_cast<int64_t>(m) * (m + 1) > n_u) --m;
        if (m < 2 || static_cast<int64_t>(m) * (m + 1) != n_u || 2 * n_u != nn) return false;
        for (int r = n_u; r < nn; ++r)
            if (comps[r] != 1) return false;
        kind = 2;
        nx = m;
        ny = m + 1;
    } else {
        nx = static_cast<int>(std::lround(std::sqrt(static_cast<double>(nn))));
        if (static_cast<int64_t>(nx) * nx != nn) return false;
        ny = nx;
        kind = 1;
    }
    const int F = kind == 1 ? WaveShape<1>::F : WaveShape<2>::F;
    const int KU = kind == 1 ? WaveShape<1>::KU : WaveShape<2>::KU;
    const int nb = (ny + 31) / 32;
    const int cols = kind == 1 ? nx : m + 1;  // u rows of the MAC block have m + 1 cells (v: m, one step later)
    const int steps = cols + 32;              // lane 31 finishes column cols - 1 (v: m - 1) at step cols + 31
    const int nblocks = (steps + KU - 1) / KU;
    const size_t blk = static_cast<size_t>(F) * KU * 32;
    // record slot of (field f, band-local lane l, step s) of band b: per block
    // and field, [step pair][lane][2], so a lane loads two steps at once
    auto slot = [&](int f, int j, int step) {
        const int b = j / 32, l = j % 32, q = step / KU, u = step % KU;
        return (static_cast<size_t>(b) * nblocks + q) * blk + static_cast<size_t>(f) * KU * 32 +
               static_cast<size_t>(u / 2) * 64 + 2 * l + (u % 2);
    };
    std::vector<double> rec(static_cast<size_t>(nb) * nblocks * blk, 0.0);
    std::vector<int> bx(nn, -1);
    for (int r = 0; r < nn; ++r) {
        int i, j, step, fb;
        int expect[6] = {-1, -1, -1, -1, -1, -1};
        int field[6] = {0, 0, 0, 0, 0, 0};
        if (kind == 1) {
            i = r % nx;
            j = r / nx;
            step = i + j % 32;
            fb = 0;
            expect[0] = j > 0 ? r - nx : -1;  // south (first in column order)
            field[0] = 1;
            expect[1] = i > 0 ? r - 1 : -1;   // west
            field[1] = 2;
        } else if (r < m * (m + 1)) {
            i = r % (m + 1);
            j = r / (m + 1);
            step = i + j % 32;
            fb = 0;
            expect[0] = j > 0 ? r - (m + 1) : -1;
            field[0] = 1;
            expect[1] = i > 0 ? r - 1 : -1;
            field[1] = 2;
        } else {
            const int qq = r - m * (m + 1);
            i = qq % m;
            j = qq / m;
            step = i + 1 + j % 32;  // v(i, j) in the step of u(i + 1, j)
            fb = 3;
            auto urow = [&](int ii, int jj) {
                return (jj >= 0 && jj < m && ii >= 0 && ii <= m) ? jj * (m + 1) + ii : -1;
            };
            expect[0] = urow(i, j - 1);
            field[0] = 4;
            expect[1] = urow(i + 1, j - 1);
            field[1] = 5;
            expect[2] = urow(i, j);
            field[2] = 6;
            expect[3] = urow(i + 1, j);
            field[3] = 7;
            expect[4] = j > 0 ? r - m : -1;  // v(i, j-1)
            field[4] = 8;
            expect[5] = i > 0 ? r - 1 : -1;  // v(i-1, j)
            field[5] = 9;
        }
        bx[r] = static_cast<int>(slot(fb, j, step));
        for (int k = a.rp[r]; k < a.rp[r + 1]; ++k) {
            const int c = a.ci[k];
            if (c >= r) continue;
            int hit = -1;
            for (int e = 0; e < 6; ++e)
                if (expect[e] == c) hit = e;
            if (hit < 0) return false;  // not the structured pattern
            rec[slot(field[hit], j, step)] = -(a.v[k] * dinv_h[r]);
        }
    }
    if (rec.size() > static_cast<size_t>(INT32_MAX)) return false;  // bidx is int
    packed.upload(rec, s);
    bidx.upload(bx, s);
    wave_ticket.resize(1);
    SDG_CUDA(cudaMemsetAsync(wave_ticket.get(), 0, sizeof(unsigned long long), s));
    {   // boundary slots, both parities, all holding the sentinel
        const size_t nbnd = static_cast<size_t>(2) * std::max(nb - 1, 1) * (kind == 1 ? 1 : 2) * cols;
        double sent;
        std::memcpy(&sent, &kSent, sizeof sent);
        wave_bnd.upload(std::vector<double>(nbnd, sent), s);
    }
    wave = true;
    wave_kind = kind;
    wave_nx = nx;
    wave_ny = ny;
    wave_bands = nb;
    wave_blocks = nblocks;
    // warps (bands) per CTA: as many as shared memory holds, at most one per
    // SM sub-partition; the MAC ring is 80 KB per band (SDG_WAVE_W overrides)
    {
        const int bc = kind == 1 ? nx : nx + 1;
        constexpr size_t kSmemMax = 226 * 1024;  // 227 KB per CTA minus the static words
        int w = kind == 1 ? 4 : 2;
        if (const char* e = std::getenv("SDG_WAVE_W")) w = std::max(1, std::min(w, std::atoi(e)));
        while (w > 1 && (kind == 1 ? wave_smem_bytes<1>(w, bc) : wave_smem_bytes<2>(w, bc)) > kSmemMax) w /= 2;
        w = std::min(w, nb >= 4 ? 4 : nb >= 2 ? 2 : 1);
        wave_w = w;
        wave_smem = kind == 1 ? wave_smem_bytes<1>(w, bc) : wave_smem_bytes<2>(w, bc);
    }
    walk = false;
    usable = true;
    if (std::getenv("SDG_DEBUG"))
        std::fprintf(stderr,
                     "[sdg] gs wave: kind %d, %d x %d grid, %d bands (%d per CTA), %d blocks of %d steps, %zu B smem\n",
                     kind, nx, ny, nb, wave_w, nblocks, KU, wave_smem);
    return true;
}

// dev aid: SDG_WAVE_TL=1 makes every launch write {start, first block, end,
// waiting ns} per band into a device buffer; sdg_wave_timeline copies the last
// launch's records out
namespace {
unsigned long long* g_wave_tl = nullptr;
int g_wave_tl_bands = 0;
unsigned long long* wave_timeline(int bands) {
    static const bool on = [] {
        const char* e = std::getenv("SDG_WAVE_TL");
        return e && e[0] == '1';
    }();
    if (!on) return nullptr;
    if (!g_wave_tl) SDG_CUDA(cudaMalloc(&g_wave_tl, 8 * 1024 * sizeof(unsigned long long)));
    g_wave_tl_bands = std::min(bands, 1024);
    return g_wave_tl;
}
}  // namespace

int wave_timeline_copy(unsigned long long* out, int max_bands) {
    if (!g_wave_tl) return 0;
    const int nb = std::min(max_bands, g_wave_tl_bands);
    SDG_CUDA(cudaDeviceSynchronize());
    SDG_CUDA(cudaMemcpy(out, g_wave_tl, 8 * nb * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    return nb;
}

void launch_gs_wave(Context& c, const GsPlan& g, double* z_new) {
    WaveArgs a{g.packed.get(), z_new, g.wave_bnd.get(), g.wave_ticket.get(), g.wave_bands, g.wave_blocks,
               g.wave_nx, g.wave_ny, g.wave_kind == 2 ? g.wave_nx * (g.wave_nx + 1) : 0,
               g.wave_kind == 1 ? g.wave_nx : g.wave_nx + 1, wave_timeline(g.wave_bands)};
    const int ctas = (g.wave_bands + g.wave_w - 1) / g.wave_w;
    static const bool attr = [] {  // every instantiation may use the whole shared memory of an SM
        for (auto k : {k_gs_wave<1, 1>, k_gs_wave<1, 2>, k_gs_wave<1, 4>, k_gs_wave<2, 1>, k_gs_wave<2, 2>})
            SDG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
        return true;
    }();
    (void)attr;
    auto go = [&](void (*kernel)(WaveArgs)) { launch_k(c, kernel, ctas, 32 * g.wave_w, g.wave_smem, a); };
    if (g.wave_kind == 1) {
        if (g.wave_w == 4) go(k_gs_wave<1, 4>);
        else if (g.wave_w == 2) go(k_gs_wave<1, 2>);
        else go(k_gs_wave<1, 1>);
    } else {
        if (g.wave_w == 2) go(k_gs_wave<2, 2>);
        else go(k_gs_wave<2, 1>);
    }
}

}  // namespace sdg
