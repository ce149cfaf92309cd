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
//   * bands run as a pipeline over SMs, W bands (warps) per CTA.  A band reads
//     the top row of the band below from an *inbound row* in its CTA's shared
//     memory, one block of KU steps at a time; the values are loaded early
//     (from the middle of the previous block) and tested when the block
//     starts, so a band that is not right behind the band below never waits.
//     The inbound row is filled by the band below itself when it is a warp of
//     the same CTA, otherwise by a *poller warp* that copies the band below's
//     L2 boundary buffer (st.relaxed.gpu by its lane 31) into shared memory
//     slot by slot.  Every slot - in L2 and in shared memory - holds a
//     sentinel until written: the value is its own ready flag, so the
//     hand-off needs no fence, no flag and no acquire, and the compute warps
//     never wait on an L2 round trip.  The pipeline's depth is the wavefront's
//     own (columns + rows steps) plus about KU steps per band;
//   * band ids come from a ticket counter (atomicAdd), so the band a CTA waits
//     for always belongs to a CTA that started earlier (no co-residency
//     assumption); the L2 boundary buffer has two parities (launch e uses
//     e % 2 and resets the other), so a captured CUDA graph replays the kernel
//     unchanged;
//   * the records of a band, [block][field][KU/2 step pairs][32 lanes][2], are
//     streamed into a shared-memory ring by 1-D TMA bulk copies (cp.async.bulk
//     + mbarrier), one copy per block, and read with 16-byte shared loads one
//     step pair ahead of their use;
//   * the MAC block runs its u and v recurrences on two warps per band
//     (k_gs_wave_mac below); k_gs_wave<2> is the same sweep on one warp
//     (SDG_WAVE_SPLIT=0), kept as the bitwise cross-check.
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
// MAC block: steps per block and ring depth of the two-warp kernel.  Measured
// at c3 (velocity V-cycle): 8 steps x 4 blocks, two bands per CTA 820 us;
// 16 x 2, two bands per CTA 823 us (refills arrive late); 16 x 3, one band per
// CTA 765 us: the per-block work (inbound test, mbarrier probes, ring refill)
// is a third of a block of 8 steps.
#ifndef SDG_WAVE_MAC_KU
#define SDG_WAVE_MAC_KU 16
#endif
#ifndef SDG_WAVE_MAC_DEPTH
#define SDG_WAVE_MAC_DEPTH 3
#endif
constexpr int kMacDepth = SDG_WAVE_MAC_DEPTH;  // the same for the two-warp MAC kernel

template <int KIND>
struct WaveShape;
template <>
struct WaveShape<1> {  // 5-point: b, c_S, c_W
    static constexpr int F = 3, KU = 16;
};
template <>
struct WaveShape<2> {  // MAC: bu, cu_S, cu_W, bv, c_u(i',j-1), c_u(i'+1,j-1), c_u(i',j), c_u(i'+1,j), cv_S, cv_W
    static constexpr int F = 10, KU = SDG_WAVE_MAC_KU;
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

// Everything inside the step loop is warp-uniform control flow; per-lane work
// (lane 31's boundary stores, the elected bulk copy) is predicated, never
// branched: a lane-divergent branch there makes the compiler's divergent-warp
// fallback (collective shuffles) run the block.
__device__ __forceinline__ void st_relaxed_if(double* p, double v, bool pred) {
    // every stored value is the result of an fma, which never returns a
    // signalling NaN, so a stored value is never the sentinel
    const double w = v;
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
// refill a ring slot: arm the slot's mbarrier and issue the 1-D bulk copy (one
// lane).  No proxy fence: the slot's shared loads have delivered their values
// (the steps that used them are done, every lane has passed __syncwarp), and a
// fence.proxy.async here also waits for the warp's outstanding global stores,
// several hundred cycles on every block (measured: see DESIGN.md).
__device__ __forceinline__ void tma_block_if(double* dst, const double* src, unsigned bytes, uint64_t* bar,
                                             bool pred) {
    asm volatile(
        "{\n.reg .pred q;\nsetp.ne.b32 q, %4, 0;\n"
        "@q mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n"
        "@q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}" ::"r"(
            ptx::smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(ptx::smem_addr(bar)), "r"(static_cast<int>(pred))
        : "memory");
}

// non-blocking test of a ring slot's mbarrier, issued a few steps before the
// slot is needed so that its latency hides behind the steps (test_wait, not
// try_wait: try_wait may suspend the warp for microseconds when the phase is
// not complete)
__device__ __forceinline__ bool mbar_try(uint64_t* bar, unsigned parity) {
    unsigned ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok)
                 : "r"(ptx::smem_addr(bar)), "r"(parity)
                 : "memory");
    return ok != 0;
}

// Boundary hand-off, round-2 form.  A band reads the top row of the band below
// from an *inbound row* in its CTA's shared memory, one block of KU steps at a
// time, just before the block starts (the values of a step: 5-point z(s, j-1);
// MAC the pair {u(s, j-1), v(s-1, j-1)}, 16 bytes).  Who fills the inbound row:
//   * the band below, directly (st.shared by its lane 31), when it is a warp
//     of the same CTA;
//   * otherwise the CTA's poller warp (warp W): the band below stores into the
//     L2 boundary buffer (st.relaxed.gpu), the poller's lanes each spin on one
//     slot of the current 32-slot window (ld.relaxed.gpu) and copy it into
//     the inbound row the moment it stops being the sentinel.
// Every slot, in L2 and in shared memory, is its own ready flag (kSent until
// written), so there is no fence, flag or acquire anywhere; the compute warps
// never wait on an L2 round trip, only on shared memory.  Slots past a row's
// last column are never written and hold 0, so no load needs a bounds test.
// A row has S = nblocks * KU slots (steps), NBF doubles each.
__device__ __forceinline__ bool is_sent_hi(double v) {
    // the sentinel's high word belongs to a NaN that arithmetic never produces
    return static_cast<unsigned>(__double2hiint(v)) == static_cast<unsigned>(kSent >> 32);
}
// relaxed (strong) shared load: ptxas may hoist a weak load out of the spin
// loop that re-reads the same addresses
__device__ __forceinline__ double2 lds_v2(unsigned addr) {
    double2 v;
    asm volatile("ld.relaxed.cta.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void st_pair_if(double* p, double x, double y, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q st.relaxed.gpu.v2.f64 [%0], {%1, %2};\n}" ::"l"(p),
                 "d"(x), "d"(y), "r"(static_cast<int>(pred)));
}

// W compute warps per CTA, one band each (consecutive bands), plus the poller.
// TL: the dev timeline (SDG_WAVE_TL=1) is a separate instantiation, so the
// product kernel carries no test of it in its loops
template <int KIND, int W, bool TL>
__global__ void __launch_bounds__(32 * (W + 1), 1) k_gs_wave(WaveArgs a) {
    constexpr int F = WaveShape<KIND>::F, KU = WaveShape<KIND>::KU;
    constexpr int NBF = KIND == 1 ? 1 : 2;  // doubles per boundary slot: z, or {u, v}
    constexpr int BLK = F * KU * 32;        // doubles per block
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ unsigned long long s_ticket;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int S = a.nblocks * KU;                              // steps = slots per boundary row
    const size_t bstride = static_cast<size_t>(NBF) * S;       // doubles per boundary row
    double* ring_all = reinterpret_cast<double*>(smem_raw);
    uint64_t* bars_all = reinterpret_cast<uint64_t*>(ring_all + W * kWaveDepth * BLK);
    double* inb_all = reinterpret_cast<double*>(bars_all + W * kWaveDepth);  // [W][S][NBF], 16-byte aligned
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.ticket, 1ull);
    if (warp < W && lane == 0) {
#pragma unroll
        for (int d = 0; d < kWaveDepth; ++d) ptx::mbar_init(bars_all + warp * kWaveDepth + d, 1);
        ptx::fence_mbar_init();
    }
    // inbound rows: the sentinel where a value will arrive, 0 past the row's end
    const int valid = a.bcols;  // slots that receive a value (5-point nx; MAC m + 1)
    for (size_t k = threadIdx.x; k < static_cast<size_t>(W) * bstride; k += blockDim.x) {
        const int slot = static_cast<int>((k % bstride) / NBF);
        inb_all[k] = slot < valid ? __longlong_as_double(static_cast<long long>(kSent)) : 0.0;
    }
    __syncthreads();
    const unsigned long long t = s_ticket;
    const unsigned long long nctas = static_cast<unsigned long long>((a.nbands + W - 1) / W);
    const int band0 = static_cast<int>(t % nctas) * W;
    const int par = static_cast<int>((t / nctas) & 1ull);
    const size_t pstride = static_cast<size_t>(a.nbands - 1) * bstride;  // one parity of the L2 buffer

    if (warp == W) {  // ---- the poller
        if (band0 == 0 || band0 >= a.nbands) return;
        pdl_wait();  // the previous launch has read its parity; this launch may reset it
        {   // reset this boundary's slots of the other parity for the next launch
            double* rs = a.bnd + (par ^ 1) * pstride + static_cast<size_t>(band0 - 1) * bstride;
            for (size_t k = lane; k < static_cast<size_t>(valid) * NBF; k += 32)
                rs[k] = __longlong_as_double(static_cast<long long>(kSent));
        }
        const double* srcb = a.bnd + par * pstride + static_cast<size_t>(band0 - 1) * bstride;
        double* dst = inb_all;  // inbound row of warp 0
        const int nslots = valid * NBF;
        for (int base = 0; base < nslots; base += 32) {
            const int k = base + lane;
            if (k < nslots) {
                for (;;) {
                    double v;
                    asm volatile("ld.relaxed.gpu.f64 %0, [%1];" : "=d"(v) : "l"(srcb + k) : "memory");
                    if (!is_sent_hi(v)) {
                        asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(ptx::smem_addr(dst + k)), "d"(v)
                                     : "memory");
                        break;
                    }
                }
            }
            __syncwarp();
        }
        return;
    }

    const int band = band0 + warp;
    if (band >= a.nbands) return;
    double* ring = ring_all + warp * (kWaveDepth * BLK);
    uint64_t* bars = bars_all + warp * kWaveDepth;
    pdl_wait();  // b is written by the prep kernel before this launch; the previous launch is done
    pdl_trigger();
    const double* src = a.rec + static_cast<size_t>(band) * a.nblocks * BLK;
    for (int d = 0; d < kWaveDepth && d < a.nblocks; ++d)
        tma_block_if(ring + d * BLK, src + static_cast<size_t>(d) * BLK, BLK * 8, bars + d, lane == 0);
    const int j = band * 32 + lane;
    const bool has_src = band > 0, has_dst = band + 1 < a.nbands;
    const bool dst_sh = warp + 1 < W && has_dst;
    const double* inb = inb_all + warp * bstride;                                         // read (all lanes, same address)
    double* sb_out = dst_sh ? inb_all + (warp + 1) * bstride
                            : a.bnd + par * pstride + static_cast<size_t>(has_dst ? band : 0) * bstride;  // written (lane 31)
    unsigned long long t_start = TL ? gtimer() : 0, t_first = 0, t_b4 = 0, t_b12 = 0;
    long long wait_cyc = 0, comp_cyc = 0;
    const bool pub = has_dst && lane == 31;

    // the records of a step pair are loaded one pair ahead (R: this pair, Rn:
    // the next one, across block boundaries too), so the shared-memory latency
    // of the loads hides behind the previous pair's arithmetic
    double2 R[F];
    auto load_pair = [&](int slot, int u2, double2 (&dst)[F]) {
        const double2* B = reinterpret_cast<const double2*>(ring + slot * BLK) + lane;
#pragma unroll
        for (int f = 0; f < F; ++f) dst[f] = B[(f * KU / 2 + u2) * 32];
    };
    // The inbound values of block q: loaded early (from the middle of block
    // q - 1, into bn) and tested when block q starts; only if one is still the
    // sentinel the band spins on reloads.  Every lane reads the same
    // addresses, so the test is warp-uniform.  A band that is not right behind
    // the band below pays no load latency for its inbound values.
    double bz[NBF * KU], bn[NBF * KU];
    const unsigned inb_addr = ptx::smem_addr(inb);
    auto load_bnd = [&](int q, double (&o)[NBF * KU]) {
        const unsigned p = inb_addr + static_cast<unsigned>(q) * (KU * NBF * 8);
#pragma unroll
        for (int k = 0; k < NBF * KU / 2; ++k) {
            const double2 v = lds_v2(p + 16 * k);
            o[2 * k] = v.x;
            o[2 * k + 1] = v.y;
        }
    };
    auto take_bnd = [&](int q) {  // bz = the inbound values of block q
        if (!has_src) return;
        const long long c0 = TL ? clock64() : 0;
        for (;;) {
            // four independent chains of compares, not one of NBF * KU
            bool ok0 = true, ok1 = true, ok2 = true, ok3 = true;
#pragma unroll
            for (int k = 0; k < NBF * KU; k += 4) {
                ok0 &= !is_sent_hi(bn[k]);
                ok1 &= !is_sent_hi(bn[k + 1]);
                ok2 &= !is_sent_hi(bn[k + 2]);
                ok3 &= !is_sent_hi(bn[k + 3]);
            }
            if (__all_sync(0xffffffffu, (ok0 && ok1) && (ok2 && ok3))) break;
            load_bnd(q, bn);
        }
#pragma unroll
        for (int k = 0; k < NBF * KU; ++k) bz[k] = bn[k];
        if (TL) wait_cyc += clock64() - c0;
    };
#pragma unroll
    for (int k = 0; k < NBF * KU; ++k) bz[k] = bn[k] = 0.0;
    if (has_src) load_bnd(0, bn);

    if constexpr (KIND == 1) {
        const int nx = a.nx;
        double last = 0.0;
        double* zrow = a.z + static_cast<size_t>(j) * nx;
        const bool row_ok = j < a.ny;
        take_bnd(0);
        if (TL) t_first = gtimer();
        ptx::mbar_wait(bars + 0, 0);
        load_pair(0, 0, R);
        for (int q = 0; q < a.nblocks; ++q) {
            if (q > 0) take_bnd(q);
            if (TL && lane == 0 && q < 128) a.tl[8 * 1024 + band * 128 + q] = gtimer();
            const int slot = q % kWaveDepth, nslot = (q + 1) % kWaveDepth;
            const unsigned npar = ((q + 1) / kWaveDepth) & 1;
            const bool more = q + 1 < a.nblocks;
            const long long c1 = TL ? clock64() : 0;
            auto run_block = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
            bool landed = true;
#pragma unroll
            for (int u2 = 0; u2 < KU / 2; ++u2) {
                double2 Rn[F];
                if (u2 == 0 && more) landed = mbar_try(bars + nslot, npar);
                if (u2 == KU / 4 && has_src && more) load_bnd(q + 1, bn);
                if (u2 + 1 < KU / 2) {
                    load_pair(slot, u2 + 1, Rn);
                } else if (more) {  // the next block's first pair
                    if (!__all_sync(0xffffffffu, landed)) ptx::mbar_wait(bars + nslot, npar);
                    load_pair(nslot, 0, Rn);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int u = 2 * u2 + h;
                    double south = __shfl_up_sync(0xffffffffu, last, 1);
                    if (lane == 0) south = bz[u];
                    // padding slots (before a lane's first column, after its
                    // last) hold zero records, so they compute 0: no select
                    last = fma(h ? R[2].y : R[2].x, last, fma(h ? R[1].y : R[1].x, south, h ? R[0].y : R[0].x));
                    const int i = q * KU + u - lane;
                    const bool act = FULL ? row_ok : (row_ok && i >= 0 && i < nx);
                    st_global_if(zrow + i, last, act);
                    st_relaxed_if(sb_out + i, last, act && pub);
                }
                if (u2 + 1 < KU / 2 || more) {
#pragma unroll
                    for (int f = 0; f < F; ++f) R[f] = Rn[f];
                }
            }
            };
            if (q * KU - 31 >= 0 && q * KU + KU - 1 < nx)
                run_block(std::true_type{});
            else
                run_block(std::false_type{});
            if (TL) {
                comp_cyc += clock64() - c1;
                if (q == 2) t_b4 = gtimer();
                if (q == 6) t_b12 = gtimer();
            }
            __syncwarp();  // every lane has read the slot
            tma_block_if(ring + slot * BLK, src + static_cast<size_t>(q + kWaveDepth) * BLK, BLK * 8, bars + slot,
                         lane == 0 && q + kWaveDepth < a.nblocks);
        }
    } else {
        const int m = a.nx;
        // step s = q KU + u of lane 0 (u column s, v column s - 1) reads the
        // pair {u(s, j-1), v(s-1, j-1)} = bz[2u], bz[2u + 1]; u(s-1, j-1) is
        // the previous step's u(s, j-1) (su_prev: what a shuffle of the lane's
        // own previous u would return, lane 0 included)
        double u_last = 0.0, su_prev = 0.0, v_last = 0.0;
        double* zu = a.z + static_cast<size_t>(j) * (m + 1);
        double* zv = a.z + a.n_u + static_cast<size_t>(j) * m - 1;  // indexed by u column i = v column + 1
        const bool u_row = j < m, v_row = j <= m;
        take_bnd(0);
        if (TL) t_first = gtimer();
        ptx::mbar_wait(bars + 0, 0);
        load_pair(0, 0, R);
        for (int q = 0; q < a.nblocks; ++q) {
            if (q > 0) take_bnd(q);
            if (TL && lane == 0 && q < 128) a.tl[8 * 1024 + band * 128 + q] = gtimer();
            const int slot = q % kWaveDepth, nslot = (q + 1) % kWaveDepth;
            const unsigned npar = ((q + 1) / kWaveDepth) & 1;
            const bool more = q + 1 < a.nblocks;
            const long long c1 = TL ? clock64() : 0;
            // FULL: every lane inside its u and v rows for the whole block, no
            // per-step column tests (the interior blocks, most of the sweep)
            auto run_block = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
            bool landed = true;
#pragma unroll
            for (int u2 = 0; u2 < KU / 2; ++u2) {
                double2 Rn[F];
                if (u2 == 0 && more) landed = mbar_try(bars + nslot, npar);
                if (u2 == KU / 4 && has_src && more) load_bnd(q + 1, bn);
                if (u2 + 1 < KU / 2) {
                    load_pair(slot, u2 + 1, Rn);
                } else if (more) {  // the next block's first pair
                    if (!__all_sync(0xffffffffu, landed)) ptx::mbar_wait(bars + nslot, npar);
                    load_pair(nslot, 0, Rn);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int u = 2 * u2 + h;
                    auto r = [&](int f) { return h ? R[f].y : R[f].x; };
                    double su1 = __shfl_up_sync(0xffffffffu, u_last, 1);   // u(i, j-1)
                    const double su2 = su_prev;                            // u(i-1, j-1)
                    double sv1 = __shfl_up_sync(0xffffffffu, v_last, 1);   // v(i-1, j-1)
                    if (lane == 0) {
                        su1 = bz[2 * u];
                        sv1 = bz[2 * u + 1];
                    }
                    su_prev = su1;
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
                    // one 16-byte store for the band above: at i = 0 the v
                    // half is the 0 of a padding record, which is what it reads
                    st_pair_if(sb_out + 2 * i, un, vn, ua && pub);
                    u_last = un;
                    v_last = vn;
                }
                if (u2 + 1 < KU / 2 || more) {
#pragma unroll
                    for (int f = 0; f < F; ++f) R[f] = Rn[f];
                }
            }
            };
            if (q * KU - 31 >= 1 && q * KU + KU - 1 <= m)
                run_block(std::true_type{});
            else
                run_block(std::false_type{});
            if (TL) {
                comp_cyc += clock64() - c1;
                if (q == 4) t_b4 = gtimer();
                if (q == 12) t_b12 = gtimer();
            }
            __syncwarp();  // every lane has read the slot
            tma_block_if(ring + slot * BLK, src + static_cast<size_t>(q + kWaveDepth) * BLK, BLK * 8, bars + slot,
                         lane == 0 && q + kWaveDepth < a.nblocks);
        }
    }
    if (TL && lane == 0) {
        unsigned long long* o = a.tl + 8 * band;
        o[0] = t_start;
        o[1] = t_first;
        o[2] = gtimer();
        o[3] = static_cast<unsigned long long>(wait_cyc);
        o[4] = 0;
        o[5] = static_cast<unsigned long long>(comp_cyc);
        o[6] = t_b4;
        o[7] = t_b12;
    }
}

// ---------------------------------------------------------------------------
// MAC wavefront with the u and v recurrences on separate warps ("split").
//
// The u rows of the MAC block never read a v value (assembly.cpp:134-170), so
// a band's u recurrence can run ahead of its v recurrence, and everything a v
// row takes from u rows can be summed where the u values are.  Each band gets
// two warps on two SM sub-partitions:
//   * the U warp walks u(i, j) like the 5-point kernel and, with the values it
//     holds anyway (u(i, j), u(i-1, j), and the row below from its shuffle),
//     also forms t = b_v + (the four u neighbours of v(i-1, j) in column
//     order) - off its own dependent chain - and drops t into an exchange ring
//     in shared memory, X[XD blocks][KU steps][32 lanes] (record fields 0-7);
//   * the V warp follows at least one block behind, takes t from the ring and
//     runs the v recurrence v = fma(c_W, v_W, fma(c_S, v_S, t)) (fields 8-9).
// Same operations on the same operands in the same order as the fused kernel,
// hence the same bits.  Per block the U warp arrives on xfull[slot] after its
// stores and waits on xempty[slot] before it reuses a ring slot; the V warp
// does the opposite (mbarriers, one arrive by lane 0 after __syncwarp).
// Boundary rows are separate for u and v ([U row S | V row S], v indexed by
// the u column i = v column + 1, slot 0 of the V row is a constant 0), each
// polled by its own poller warp, so the u chain across bands never waits for
// the v chain.  Threads: 2 W compute warps + 2 pollers.
template <int W, bool TL>
__global__ void __launch_bounds__(32 * (2 * W + 2), 1) k_gs_wave_mac(WaveArgs a) {
    constexpr int KU = WaveShape<2>::KU, FU = 8, FV = 2, D = kMacDepth, XD = 4;
    constexpr int UBLK = FU * KU * 32, VBLK = FV * KU * 32, BLK = UBLK + VBLK, XBLK = KU * 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ unsigned long long s_ticket;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int S = a.nblocks * KU;
    const size_t bstride = 2 * static_cast<size_t>(S);  // [U row | V row]
    double* uring_all = reinterpret_cast<double*>(smem_raw);
    double* vring_all = uring_all + W * D * UBLK;
    double* x_all = vring_all + W * D * VBLK;
    double* inb_all = x_all + W * XD * XBLK;                                  // [W][2][S]
    uint64_t* bars_all = reinterpret_cast<uint64_t*>(inb_all + W * bstride);  // per band: U ring D, V ring D, xfull XD, xempty XD
    constexpr int NBAR = 2 * D + 2 * XD;
    const int m = a.nx, valid = a.bcols;  // valid = m + 1 u columns
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.ticket, 1ull);
    if (warp < W && lane == 0) {
        for (int d = 0; d < NBAR; ++d) ptx::mbar_init(bars_all + warp * NBAR + d, 1);
        ptx::fence_mbar_init();
    }
    auto expects = [&](size_t k) {  // does slot k of a boundary row pair receive a value?
        const size_t r = k % bstride;
        const int slot = static_cast<int>(r % S);
        return r < static_cast<size_t>(S) ? slot < valid : (slot >= 1 && slot < valid);
    };
    for (size_t k = threadIdx.x; k < static_cast<size_t>(W) * bstride; k += blockDim.x)
        inb_all[k] = expects(k) ? __longlong_as_double(static_cast<long long>(kSent)) : 0.0;
    __syncthreads();
    const unsigned long long t = s_ticket;
    const unsigned long long nctas = static_cast<unsigned long long>((a.nbands + W - 1) / W);
    const int band0 = static_cast<int>(t % nctas) * W;
    const int par = static_cast<int>((t / nctas) & 1ull);
    const size_t pstride = static_cast<size_t>(a.nbands - 1) * bstride;

    if (warp >= 2 * W) {  // ---- the pollers: warp 2W the U row, warp 2W + 1 the V row
        if (band0 == 0 || band0 >= a.nbands) return;
        const int row = warp - 2 * W;
        pdl_wait();
        const size_t off = static_cast<size_t>(band0 - 1) * bstride + static_cast<size_t>(row) * S;
        {   // reset this row of the other parity for the next launch
            double* rs = a.bnd + (par ^ 1) * pstride + off;
            for (int k = lane + row; k < valid; k += 32) rs[k] = __longlong_as_double(static_cast<long long>(kSent));
        }
        const double* srcb = a.bnd + par * pstride + off;
        double* dst = inb_all + static_cast<size_t>(row) * S;  // inbound rows of band 0 of the CTA
        for (int base = row; base < valid; base += 32) {
            const int k = base + lane;
            if (k < valid) {
                for (;;) {
                    double v;
                    asm volatile("ld.relaxed.gpu.f64 %0, [%1];" : "=d"(v) : "l"(srcb + k) : "memory");
                    if (!is_sent_hi(v)) {
                        asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(ptx::smem_addr(dst + k)), "d"(v)
                                     : "memory");
                        break;
                    }
                }
            }
            __syncwarp();
        }
        return;
    }

    const int w = warp >> 1;
    const bool is_v = warp & 1;
    const int band = band0 + w;
    if (band >= a.nbands) return;
    uint64_t* bars = bars_all + w * NBAR + (is_v ? D : 0);
    uint64_t* xfull = bars_all + w * NBAR + 2 * D;
    uint64_t* xempty = xfull + XD;
    double* X = x_all + w * XD * XBLK;
    pdl_wait();
    pdl_trigger();
    const int j = band * 32 + lane;
    const bool has_src = band > 0, has_dst = band + 1 < a.nbands;
    const bool dst_sh = w + 1 < W && has_dst;
    const bool pub = has_dst && lane == 31;
    const unsigned inb_u = ptx::smem_addr(inb_all + w * bstride), inb_v = inb_u + static_cast<unsigned>(S) * 8;
    double* out = dst_sh ? inb_all + (w + 1) * bstride
                         : a.bnd + par * pstride + static_cast<size_t>(has_dst ? band : 0) * bstride;
    unsigned long long t_start = TL ? gtimer() : 0, t_first = 0;
    const double* src = a.rec + static_cast<size_t>(band) * a.nblocks * BLK + (is_v ? UBLK : 0);

    if (!is_v) {
        // ------------------------------------------------------------- U warp
        double* ring = uring_all + w * D * UBLK;
        for (int d = 0; d < D && d < a.nblocks; ++d)
            tma_block_if(ring + d * UBLK, src + static_cast<size_t>(d) * BLK, UBLK * 8, bars + d, lane == 0);
        double bz[KU], bn[KU];
        auto load_bnd = [&](int q, double (&o)[KU]) {
            const unsigned p = inb_u + static_cast<unsigned>(q) * (KU * 8);
#pragma unroll
            for (int k = 0; k < KU / 2; ++k) {
                const double2 v = lds_v2(p + 16 * k);
                o[2 * k] = v.x;
                o[2 * k + 1] = v.y;
            }
        };
        auto take_bnd = [&](int q) {
            if (!has_src) return;
            for (;;) {
                bool ok = true;
#pragma unroll
                for (int k = 0; k < KU; ++k) ok &= !is_sent_hi(bn[k]);
                if (__all_sync(0xffffffffu, ok)) break;
                load_bnd(q, bn);
            }
#pragma unroll
            for (int k = 0; k < KU; ++k) bz[k] = bn[k];
        };
#pragma unroll
        for (int k = 0; k < KU; ++k) bz[k] = bn[k] = 0.0;
        if (has_src) load_bnd(0, bn);
        double2 R[FU];
        auto load_pair = [&](int slot, int u2, double2 (&dst)[FU]) {
            const double2* B = reinterpret_cast<const double2*>(ring + slot * UBLK) + lane;
#pragma unroll
            for (int f = 0; f < FU; ++f) dst[f] = B[(f * KU / 2 + u2) * 32];
        };
        double u_last = 0.0, su_prev = 0.0;
        bool x_free = false;
        double* zu = a.z + static_cast<size_t>(j) * (m + 1);
        const bool u_row = j < m;
        take_bnd(0);
        if (TL) t_first = gtimer();
        ptx::mbar_wait(bars + 0, 0);
        load_pair(0, 0, R);
        for (int q = 0; q < a.nblocks; ++q) {
            if (q > 0) take_bnd(q);
            const int slot = q % D, nslot = (q + 1) % D, xs = q % XD;
            const unsigned npar = ((q + 1) / D) & 1;
            const bool more = q + 1 < a.nblocks;
            // the V warp is done with this ring slot (probed during the previous block)
            if (q >= XD && !__all_sync(0xffffffffu, x_free)) ptx::mbar_wait(xempty + xs, ((q / XD) - 1) & 1);
            double* Xq = X + xs * XBLK + lane;
            auto run_block = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
            bool landed = true;
#pragma unroll
            for (int u2 = 0; u2 < KU / 2; ++u2) {
                double2 Rn[FU];
                if (u2 == 0 && more) landed = mbar_try(bars + nslot, npar);
                if (u2 == KU / 4 && has_src && more) load_bnd(q + 1, bn);
                if (u2 == KU / 4 && q + 1 >= XD && more)
                    x_free = mbar_try(xempty + (q + 1) % XD, (((q + 1) / XD) - 1) & 1);
                if (u2 + 1 < KU / 2) {
                    load_pair(slot, u2 + 1, Rn);
                } else if (more) {
                    if (!__all_sync(0xffffffffu, landed)) ptx::mbar_wait(bars + nslot, npar);
                    load_pair(nslot, 0, Rn);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int u = 2 * u2 + h;
                    auto r = [&](int f) { return h ? R[f].y : R[f].x; };
                    double su1 = __shfl_up_sync(0xffffffffu, u_last, 1);  // u(i, j-1)
                    if (lane == 0) su1 = bz[u];
                    const double su2 = su_prev;                           // u(i-1, j-1)
                    su_prev = su1;
                    const double un = fma(r(2), u_last, fma(r(1), su1, r(0)));
                    // for v(i' = i - 1, j): its u neighbours in column order, then b_v
                    double acc = fma(r(4), su2, 0.0);   // u(i', j-1)
                    acc = fma(r(5), su1, acc);          // u(i'+1, j-1)
                    acc = fma(r(6), u_last, acc);       // u(i', j)
                    acc = fma(r(7), un, acc);           // u(i'+1, j)
                    const double tv = r(3) + acc;
                    const int i = q * KU + u - lane;
                    const bool ua = FULL ? u_row : (u_row && i >= 0 && i <= m);
                    Xq[u * 32] = tv;
                    st_global_if(zu + i, un, ua);
                    st_relaxed_if(out + i, un, ua && pub);
                    u_last = un;
                }
                if (u2 + 1 < KU / 2 || more) {
#pragma unroll
                    for (int f = 0; f < FU; ++f) R[f] = Rn[f];
                }
            }
            };
            if (q * KU - 31 >= 1 && q * KU + KU - 1 <= m)
                run_block(std::true_type{});
            else
                run_block(std::false_type{});
            __syncwarp();  // every lane has stored its X values and read the record slot
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ptx::smem_addr(xfull + xs)) : "memory");
            tma_block_if(ring + slot * UBLK, src + static_cast<size_t>(q + D) * BLK, UBLK * 8, bars + slot,
                         lane == 0 && q + D < a.nblocks);
        }
        if (TL && lane == 0) {
            unsigned long long* o = a.tl + 8 * band;
            o[0] = t_start;
            o[1] = t_first;
            o[2] = gtimer();
        }
    } else {
        // ------------------------------------------------------------- V warp
        double* ring = vring_all + w * D * VBLK;
        for (int d = 0; d < D && d < a.nblocks; ++d)
            tma_block_if(ring + d * VBLK, src + static_cast<size_t>(d) * BLK, VBLK * 8, bars + d, lane == 0);
        double bz[KU], bn[KU];  // v(s-1, j-1)
        auto load_bnd = [&](int q, double (&o)[KU]) {
            const unsigned pv = inb_v + static_cast<unsigned>(q) * (KU * 8);
#pragma unroll
            for (int k = 0; k < KU / 2; ++k) {
                const double2 b2 = lds_v2(pv + 16 * k);
                o[2 * k] = b2.x;
                o[2 * k + 1] = b2.y;
            }
        };
        auto take_bnd = [&](int q) {
            if (!has_src) return;
            for (;;) {
                bool ok = true;
#pragma unroll
                for (int k = 0; k < KU; ++k) ok &= !is_sent_hi(bn[k]);
                if (__all_sync(0xffffffffu, ok)) break;
                load_bnd(q, bn);
            }
#pragma unroll
            for (int k = 0; k < KU; ++k) bz[k] = bn[k];
        };
#pragma unroll
        for (int k = 0; k < KU; ++k) bz[k] = bn[k] = 0.0;
        if (has_src) load_bnd(0, bn);
        double2 R[FV];  // cv_S, cv_W
        auto load_pair = [&](int slot, int u2, double2 (&dst)[FV]) {
            const double2* B = reinterpret_cast<const double2*>(ring + slot * VBLK) + lane;
#pragma unroll
            for (int f = 0; f < FV; ++f) dst[f] = B[(f * KU / 2 + u2) * 32];
        };
        double v_last = 0.0;
        double* zv = a.z + a.n_u + static_cast<size_t>(j) * m - 1;  // indexed by u column i = v column + 1
        const bool v_row = j <= m;
        double* outv = out + S;
        take_bnd(0);
        ptx::mbar_wait(bars + 0, 0);
        load_pair(0, 0, R);
        for (int q = 0; q < a.nblocks; ++q) {
            if (q > 0) take_bnd(q);
            const int slot = q % D, nslot = (q + 1) % D, xs = q % XD;
            const unsigned npar = ((q + 1) / D) & 1;
            const bool more = q + 1 < a.nblocks;
            ptx::mbar_wait(xfull + xs, (q / XD) & 1);  // the U warp has stored this block's values
            const double* Xq = X + xs * XBLK + lane;
            auto run_block = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
            bool landed = true;
#pragma unroll
            for (int u2 = 0; u2 < KU / 2; ++u2) {
                double2 Rn[FV];
                if (u2 == 0 && more) landed = mbar_try(bars + nslot, npar);
                if (u2 == KU / 4 && has_src && more) load_bnd(q + 1, bn);
                if (u2 + 1 < KU / 2) {
                    load_pair(slot, u2 + 1, Rn);
                } else if (more) {
                    if (!__all_sync(0xffffffffu, landed)) ptx::mbar_wait(bars + nslot, npar);
                    load_pair(nslot, 0, Rn);
                }
                const double t0 = Xq[(2 * u2) * 32], t1 = Xq[(2 * u2 + 1) * 32];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int u = 2 * u2 + h;
                    double sv1 = __shfl_up_sync(0xffffffffu, v_last, 1);   // v(i-1, j-1)
                    if (lane == 0) sv1 = bz[u];
                    const double vn = fma(h ? R[1].y : R[1].x, v_last, fma(h ? R[0].y : R[0].x, sv1, h ? t1 : t0));
                    const int i = q * KU + u - lane;
                    const bool va = FULL ? v_row : (v_row && i >= 1 && i <= m);
                    st_global_if(zv + i, vn, va);
                    st_relaxed_if(outv + i, vn, va && pub);
                    v_last = vn;
                }
                if (u2 + 1 < KU / 2 || more) {
#pragma unroll
                    for (int f = 0; f < FV; ++f) R[f] = Rn[f];
                }
            }
            };
            if (q * KU - 31 >= 1 && q * KU + KU - 1 <= m)
                run_block(std::true_type{});
            else
                run_block(std::false_type{});
            __syncwarp();  // every lane has read the X values and the record slot
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ptx::smem_addr(xempty + xs)) : "memory");
            tma_block_if(ring + slot * VBLK, src + static_cast<size_t>(q + D) * BLK, VBLK * 8, bars + slot,
                         lane == 0 && q + D < a.nblocks);
        }
        if (TL && lane == 0) a.tl[8 * band + 3] = gtimer();
    }
}

size_t wave_mac_smem_bytes(int w, int nblocks) {
    constexpr int KU = WaveShape<2>::KU;
    return static_cast<size_t>(w) * (static_cast<size_t>(kMacDepth) * 10 * KU * 32 * sizeof(double) +   // record rings
                                     4 * KU * 32 * sizeof(double) +                                     // exchange ring
                                     2 * static_cast<size_t>(nblocks) * KU * sizeof(double) +           // inbound rows
                                     (2 * kMacDepth + 8) * sizeof(uint64_t));
}

// slots (steps) of a boundary row and shared memory of a CTA of w bands
template <int KIND>
size_t wave_smem_bytes(int w, int nblocks) {
    const size_t nbf = KIND == 1 ? 1 : 2;
    return static_cast<size_t>(w) * (static_cast<size_t>(kWaveDepth) * WaveShape<KIND>::F * WaveShape<KIND>::KU * 32 *
                                         sizeof(double) +
                                     kWaveDepth * sizeof(uint64_t) +
                                     nbf * nblocks * WaveShape<KIND>::KU * sizeof(double));
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
    int pick_w = 1;
    size_t pick_smem = 0;
    // MAC: the split kernel (u and v on separate warps) unless SDG_WAVE_SPLIT=0
    bool split = kind == 2;
    if (const char* e = std::getenv("SDG_WAVE_SPLIT")) split = split && e[0] != '0';
    // warps (bands) per CTA: as many as shared memory holds, at most two (the
    // MAC rings are 80 KB per band; four 5-point bands on one SM measured
    // slower than two); SDG_WAVE_W overrides
    {
        constexpr size_t kSmemMax = 226 * 1024;  // 227 KB per CTA minus the static words
        int w = 2;
        if (const char* e = std::getenv("SDG_WAVE_W")) w = std::max(1, std::min(kind == 1 ? 4 : 2, std::atoi(e)));
        auto bytes = [&](int ww) {
            return kind == 1 ? wave_smem_bytes<1>(ww, nblocks)
                   : split   ? wave_mac_smem_bytes(ww, nblocks)
                             : wave_smem_bytes<2>(ww, nblocks);
        };
        while (w > 1 && bytes(w) > kSmemMax) w /= 2;
        if (bytes(w) > kSmemMax) return false;  // a row too long for one inbound row: the walks run
        w = std::min(w, nb >= 4 ? 4 : nb >= 2 ? 2 : 1);
        pick_w = w;
        pick_smem = bytes(w);
    }
    if (rec.size() > static_cast<size_t>(INT32_MAX)) return false;  // bidx is int
    packed.upload(rec, s);
    bidx.upload(bx, s);
    wave_ticket.resize(1);
    SDG_CUDA(cudaMemsetAsync(wave_ticket.get(), 0, sizeof(unsigned long long), s));
    {   // L2 boundary rows [2 parities][nb - 1][row]: the sentinel where a value will arrive,
        // 0 elsewhere (see the kernels' hand-off comments).  A row is [S slots][NBF] for the
        // 5-point and the fused MAC kernel, [U row S | V row S] for the split MAC kernel
        // (slot 0 of the V row never receives a value)
        const size_t nbf = kind == 1 ? 1 : 2, S = static_cast<size_t>(nblocks) * KU;
        double sent;
        std::memcpy(&sent, &kSent, sizeof sent);
        std::vector<double> row(nbf * S, 0.0);
        if (split) {
            std::fill(row.begin(), row.begin() + cols, sent);
            std::fill(row.begin() + S + 1, row.begin() + S + cols, sent);
        } else {
            std::fill(row.begin(), row.begin() + nbf * cols, sent);
        }
        std::vector<double> all;
        for (int k = 0; k < 2 * std::max(nb - 1, 1); ++k) all.insert(all.end(), row.begin(), row.end());
        wave_bnd.upload(all, s);
    }
    wave = true;
    wave_kind = kind;
    wave_nx = nx;
    wave_ny = ny;
    wave_bands = nb;
    wave_blocks = nblocks;
    wave_w = pick_w;
    wave_smem = pick_smem;
    wave_split = split;
    walk = false;
    usable = true;
    if (std::getenv("SDG_DEBUG"))
        std::fprintf(stderr,
                     "[sdg] gs wave: kind %d%s, %d x %d grid, %d bands (%d per CTA), %d blocks of %d steps, %zu B smem\n",
                     kind, wave_split ? " (u/v split)" : "", nx, ny, nb, wave_w, nblocks, KU, wave_smem);
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
    if (!g_wave_tl) SDG_CUDA(cudaMalloc(&g_wave_tl, (8 + 128) * 1024 * sizeof(unsigned long long)));
    g_wave_tl_bands = std::min(bands, 1024);
    return g_wave_tl;
}
}  // namespace

int wave_blocks_copy(unsigned long long* out, int max_bands) {  // [band][128] block start times
    if (!g_wave_tl) return 0;
    const int nb = std::min(max_bands, g_wave_tl_bands);
    SDG_CUDA(cudaDeviceSynchronize());
    SDG_CUDA(cudaMemcpy(out, g_wave_tl + 8 * 1024, 128 * nb * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    return nb;
}

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
    const bool tl = a.tl != nullptr;
    static const bool attr = [] {  // every instantiation may use the whole shared memory of an SM
        for (auto k : {k_gs_wave<1, 1, false>, k_gs_wave<1, 2, false>, k_gs_wave<1, 4, false>, k_gs_wave<2, 1, false>,
                       k_gs_wave<2, 2, false>, k_gs_wave<1, 1, true>, k_gs_wave<1, 2, true>, k_gs_wave<1, 4, true>,
                       k_gs_wave<2, 1, true>, k_gs_wave<2, 2, true>})
            SDG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
        return true;
    }();
    (void)attr;
    auto go = [&](void (*kernel)(WaveArgs), void (*kernel_tl)(WaveArgs)) {
        launch_k(c, tl ? kernel_tl : kernel, ctas, 32 * (g.wave_w + 1), g.wave_smem, a);
    };
    if (g.wave_split) {
        static const bool attr2 = [] {
            for (auto k : {k_gs_wave_mac<1, false>, k_gs_wave_mac<2, false>, k_gs_wave_mac<1, true>, k_gs_wave_mac<2, true>})
                SDG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
            return true;
        }();
        (void)attr2;
        auto kern = g.wave_w == 2 ? (tl ? k_gs_wave_mac<2, true> : k_gs_wave_mac<2, false>)
                                  : (tl ? k_gs_wave_mac<1, true> : k_gs_wave_mac<1, false>);
        launch_k(c, kern, ctas, 32 * (2 * g.wave_w + 2), g.wave_smem, a);
        return;
    }
    if (g.wave_kind == 1) {
        if (g.wave_w == 4) go(k_gs_wave<1, 4, false>, k_gs_wave<1, 4, true>);
        else if (g.wave_w == 2) go(k_gs_wave<1, 2, false>, k_gs_wave<1, 2, true>);
        else go(k_gs_wave<1, 1, false>, k_gs_wave<1, 1, true>);
    } else {
        if (g.wave_w == 2) go(k_gs_wave<2, 2, false>, k_gs_wave<2, 2, true>);
        else go(k_gs_wave<2, 1, false>, k_gs_wave<2, 1, true>);
    }
}

}  // namespace sdg
