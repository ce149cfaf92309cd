// Fast Gauss-Seidel smoother: plan (host) + prep / lower / restrict kernels.
// See gs.cuh for the algorithm; this file holds the data layout and kernels.
//
// Bands and clusters.  The rows are cut into B bands (B = cluster size, one
// CTA per band, B <= 8).  Every row's band is its component-relative height
// (row rank inside its label) raised to the largest band of any of its lower
// dependencies, so dependencies only ever point to the same or an earlier
// band.  Values a later band needs are pushed into its shared-memory halo
// with DSMEM st.async stores that complete single-use "packet" mbarriers
// there (one packet per upstream band level); a band waits for a packet
// before the first level that reads it.
//
// Packed layout (per band level, contiguous, 16-byte aligned):
//   [nS small records of 48 B][nL large records of 112 B][nE exports of 16 B]
// small record (rows with <= 2 lower entries):
//   { double b; int rowid; int wpos; double val[2]; int src[2]; int pad[2] }
// large record (rows with 3..8 lower entries):
//   { double b; int rowid; int wpos; double val[8]; int src[8] }
// export entry (a value of the PREVIOUS level needed downstream):
//   { int local ring slot; int destination band | packet << 8; int destination halo index; int pad }
// b = (r - U z_old)_i / d_i (written by the prep kernels), val = a_ij / d_i,
// src = slot in [z ring | zero slot | halo], or -(j+1) for the rare in-band
// dependency older than the ring (read back from global z_new).  48 and 112
// are odd multiples of 16 bytes, so 16-byte shared loads of consecutive
// records are bank-conflict free.
#include "gs.cuh"
#include "launch.cuh"
#include "ptx.cuh"
#include "rowdot.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>

namespace cg = cooperative_groups;

namespace sdg {

using namespace ptx;

namespace {

constexpr int kMaxSmem = 227 * 1024;
constexpr int kSmallBytes = 48;
constexpr int kLargeBytes = 112;
constexpr int kExportBytes = 16;
constexpr int kMaxLower = 8;

__host__ __device__ inline int pad16(int64_t b) { return static_cast<int>((b + 15) / 16 * 16); }

// ---- prep kernels ----------------------------------------------------------

__global__ void k_gs_prep_pre(int n, const double* __restrict__ r, const double* __restrict__ dinv,
                              const int* __restrict__ bidx, double* __restrict__ packed) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) packed[bidx[i]] = r[i] * dinv[i];
}

// b_i += sum_j (-a_ij / d_i) z_j over the earlier label blocks (GsPlan::couple)
__global__ void k_gs_couple(int rows, int r0, const int* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, const double* __restrict__ z,
                            const int* __restrict__ bidx, double* __restrict__ packed) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    double acc = 0.0;
    row_fold<8>(ci, v, rp[i], rp[i + 1], [&](int j) { return z[j]; },
                [&](double a, double x) { acc = fma(a, x, acc); });
    packed[bidx[r0 + i]] += acc;
}

// merged label block: b'_i = sum_q T_iq b_q (T: the group-local substitution of merge_levels,
// unit diagonal), from the block's temporary b slots into the records of its walk
__global__ void k_gs_tapply(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, const double* __restrict__ tmp,
                            const int* __restrict__ pbidx, double* __restrict__ packed) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    double acc = 0.0;
    row_fold<8>(ci, v, rp[i], rp[i + 1], [&](int j) { return tmp[j]; },
                [&](double a, double x) { acc = fma(a, x, acc); });
    packed[pbidx[i]] = acc;
}

__global__ void k_gs_prep_post(int n, const int* __restrict__ urp, const int* __restrict__ uci,
                               const double* __restrict__ uv, const double* __restrict__ r,
                               const double* __restrict__ z, const double* __restrict__ zc,
                               const int* __restrict__ agg, const double* __restrict__ dinv,
                               const int* __restrict__ bidx, double* __restrict__ packed) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = r[i];
    const int e = urp[i + 1];
    auto f = [&](double a, double x) { s = fma(-a, x, s); };
    if (zc)
        row_fold<8>(uci, uv, urp[i], e, [&](int j) { return z[j] + zc[agg[j]]; }, f);
    else if (z)
        row_fold<8>(uci, uv, urp[i], e, [&](int j) { return z[j]; }, f);
    packed[bidx[i]] = s * dinv[i];
}

// merged plans (GsPlan::merged): b'_i = sum_q W_iq r_q [- sum_u WU_iu z_old_u].
// The rows of W and WU are long (group fill), so kGroup lanes share a row
// and fold their partial sums with shuffles.
constexpr int kGroup = 8;

__global__ void k_gs_prep_m(int n, const int* __restrict__ wrp, const int* __restrict__ wci,
                            const double* __restrict__ wv, const int* __restrict__ urp,
                            const int* __restrict__ uci, const double* __restrict__ uv,
                            const double* __restrict__ r, const double* __restrict__ z,
                            const double* __restrict__ zc, const int* __restrict__ agg,
                            const int* __restrict__ bidx, double* __restrict__ packed) {
    pdl_begin();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = t / kGroup, lane = t % kGroup;
    double s = 0.0;
    if (i < n) {
        for (int k = wrp[i] + lane; k < wrp[i + 1]; k += kGroup) s = fma(wv[k], r[wci[k]], s);
        if (z) {
            const int e = urp[i + 1];
            if (zc) {
                for (int k = urp[i] + lane; k < e; k += kGroup) {
                    const int j = uci[k];
                    s = fma(-uv[k], z[j] + zc[agg[j]], s);
                }
            } else {
                for (int k = urp[i] + lane; k < e; k += kGroup) s = fma(-uv[k], z[uci[k]], s);
            }
        }
    }
#pragma unroll
    for (int o = kGroup / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, kGroup);
    if (i < n && lane == 0) packed[bidx[i]] = s;
}

// ---- the lower solve -------------------------------------------------------

// Load row t of a level segment into registers.  Small records fill the
// unused entries with the zero slot, so every row can use the same formula.
__device__ __forceinline__ bool load_row(const unsigned char* seg, int nS, int nL, int t, int zero_slot,
                                         double& b, int& rowid, int& wpos, double (&v)[kMaxLower],
                                         int (&sr)[kMaxLower]) {
    if (t >= nS + nL) return false;
    if (t < nS) {
        const unsigned char* q = seg + static_cast<size_t>(t) * kSmallBytes;
        const int4 h = *reinterpret_cast<const int4*>(q);
        const double2 vv = *reinterpret_cast<const double2*>(q + 16);
        const int4 ss = *reinterpret_cast<const int4*>(q + 32);
        b = __hiloint2double(h.y, h.x);
        rowid = h.z;
        wpos = h.w;
        v[0] = vv.x;
        v[1] = vv.y;
        sr[0] = ss.x;
        sr[1] = ss.y;
#pragma unroll
        for (int k = 2; k < kMaxLower; ++k) {
            v[k] = 0.0;
            sr[k] = zero_slot;
        }
    } else {
        const unsigned char* q = seg + static_cast<size_t>(nS) * kSmallBytes +
                                 static_cast<size_t>(t - nS) * kLargeBytes;
        const int4 h = *reinterpret_cast<const int4*>(q);
        b = __hiloint2double(h.y, h.x);
        rowid = h.z;
        wpos = h.w;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 vv = *reinterpret_cast<const double2*>(q + 16 + 16 * k);
            v[2 * k] = vv.x;
            v[2 * k + 1] = vv.y;
        }
        const int4 s0 = *reinterpret_cast<const int4*>(q + 80);
        const int4 s1 = *reinterpret_cast<const int4*>(q + 96);
        sr[0] = s0.x; sr[1] = s0.y; sr[2] = s0.z; sr[3] = s0.w;
        sr[4] = s1.x; sr[5] = s1.y; sr[6] = s1.z; sr[7] = s1.w;
    }
    return true;
}

template <bool GLOBAL>
__device__ __forceinline__ double zref(const double* zring, const double* z_new, int s) {
    if (GLOBAL) return s >= 0 ? zring[s] : __ldcg(z_new - s - 1);
    return zring[s];
}

// z_i = b_i - sum_k v_k z_{src_k}; TWO: the level has only small rows.
template <bool GLOBAL, bool TWO>
__device__ __forceinline__ void solve_row(double b, int rowid, int wpos, const double (&v)[kMaxLower],
                                          const int (&sr)[kMaxLower], double* zring, double* z_new) {
    double acc;
    if (TWO) {
        acc = b - fma(v[1], zref<GLOBAL>(zring, z_new, sr[1]), v[0] * zref<GLOBAL>(zring, z_new, sr[0]));
    } else {
        double p[kMaxLower];
#pragma unroll
        for (int k = 0; k < kMaxLower; ++k) p[k] = v[k] * zref<GLOBAL>(zring, z_new, sr[k]);
        acc = b - (((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7])));
    }
    zring[wpos] = acc;
    z_new[rowid] = acc;
}

// One CTA per band, the bands forming one thread-block cluster.  Shared
// memory: [D chunk mbarriers | per-level meta + req_ptr + chunk table of the
// band | packet mbarriers | z ring, zero slot, halo | D chunk slots].  The
// level segments are grouped into chunks of several consecutive levels that
// one TMA bulk copy brings in, so warp 0 lane 0 (the producer) works once per
// chunk, keeping D chunks in flight; warps 1.. are consumers, one row each
// per level (wider levels loop), pulling their next-level row into registers
// before the level barrier.
__global__ void __launch_bounds__(512, 1)
k_gs_cluster(const int4* __restrict__ meta_g, const int4* __restrict__ band_info,
             const int* __restrict__ req_ptr_g, const int* __restrict__ req,
             const int* __restrict__ packet_bytes, const int4* __restrict__ chunks_g,
             const double* __restrict__ packed, int ring, int halo, int depth, int max_chunk,
             int meta_bytes, int chunk_tab_bytes, int pbar_bytes, double* z_new) {
    pdl_begin();
    extern __shared__ __align__(128) unsigned char sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int band = static_cast<int>(cluster.block_rank());
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
    int4* meta = reinterpret_cast<int4*>(sm + 128);
    int* reqp = reinterpret_cast<int*>(sm + 128 + meta_bytes);
    int4* chunks = reinterpret_cast<int4*>(sm + 128 + 2 * meta_bytes);
    uint64_t* pbars = reinterpret_cast<uint64_t*>(sm + 128 + 2 * meta_bytes + chunk_tab_bytes);
    double* zring = reinterpret_cast<double*>(sm + 128 + 2 * meta_bytes + chunk_tab_bytes + pbar_bytes);
    const int zero_slot = ring;
    const int zbytes = pad16(static_cast<int64_t>(ring + 1 + halo) * 8);
    unsigned char* slots = reinterpret_cast<unsigned char*>(zring) + zbytes;
    const int tid = threadIdx.x;
    const int ct = tid - 32;
    const int ncons = blockDim.x - 32;

    const int4 bi = band_info[band];          // {meta base, n levels, packet base, n packets}
    const int4 bc = band_info[gridDim.x + band];  // {chunk base, n chunks, -, -}
    const int mbase = bi.x, n_levels = bi.y, n_chunks = bc.y;
    const bool has_packets = bi.w > 0;
    for (int l = tid; l < n_levels; l += blockDim.x) {
        int4 m = meta_g[mbase + l];
        m.x = (m.w % depth) * max_chunk + m.x * 16;  // byte offset of the level in the slot area
        meta[l] = m;
    }
    for (int l = tid; l <= n_levels; l += blockDim.x) reqp[l] = req_ptr_g[mbase + l];
    for (int c = tid; c < n_chunks; c += blockDim.x) chunks[c] = chunks_g[bc.x + c];
    for (int q = tid; q < bi.w; q += blockDim.x) {
        mbar_init(&pbars[q], 1);
        mbar_expect_tx(&pbars[q], static_cast<unsigned>(packet_bytes[bi.z + q]));
    }
    if (tid == 0) {
        for (int s = 0; s < depth; ++s) mbar_init(&bars[s], 1);
        zring[zero_slot] = 0.0;  // zero slot for padded entries
    }
    fence_mbar_init();
    cluster.sync();  // every packet barrier is armed before any remote store

    const unsigned char* gbase = reinterpret_cast<const unsigned char*>(packed);
    auto slot_of = [&](int chunk) { return slots + static_cast<size_t>(chunk % depth) * max_chunk; };
    auto seg_of = [&](int L) {
        return static_cast<const unsigned char*>(slots) + meta[L].x;  // {slot offset, nS | flag, nL | nE << 16, chunk}
    };
    auto issue = [&](int c) {
        const int4 ch = chunks[c];  // {off16, bytes16, first level, levels}
        uint64_t* bar = &bars[c % depth];
        const unsigned bytes = static_cast<unsigned>(ch.y) * 16u;
        mbar_expect_tx(bar, bytes);
        if (bytes) tma_load_1d(slot_of(c), gbase + static_cast<size_t>(ch.x) * 16, bytes, bar);
    };
    auto wait_chunk = [&](int c) { mbar_wait(&bars[c % depth], static_cast<unsigned>(c / depth) & 1u); };
    auto satisfy = [&](int L) {
        for (int q = reqp[L]; q < reqp[L + 1]; ++q) mbar_wait(&pbars[req[q]], 0);
    };
    if (tid == 0) {
        for (int c = 0; c < depth && c < n_chunks; ++c) issue(c);
        if (n_levels > 0) {
            wait_chunk(meta[0].w);
            if (has_packets) satisfy(0);
        }
        if (n_levels > 1 && meta[1].w != meta[0].w) wait_chunk(meta[1].w);
    }
    __syncthreads();

    double rb = 0.0, v[kMaxLower];
    int rowid = 0, wpos = 0, sr[kMaxLower];
    bool live = false;
    if (ct >= 0 && n_levels > 0) {
        const int4 m0 = meta[0];
        live = load_row(seg_of(0), m0.y & 0x7fffffff, m0.z & 0xffff, ct, zero_slot, rb, rowid, wpos, v, sr);
    }

    for (int L = 0; L < n_levels; ++L) {
        if (ct >= 0) {
            const int4 m = meta[L];
            const int nS = m.y & 0x7fffffff, nL = m.z & 0xffff, nE = m.z >> 16;
            const unsigned char* seg = seg_of(L);
            // exports of the previous level (its values are in the ring)
            for (int e = ct; e < nE; e += ncons) {
                const int4 x = *reinterpret_cast<const int4*>(seg + static_cast<size_t>(nS) * kSmallBytes +
                                                              static_cast<size_t>(nL) * kLargeBytes +
                                                              static_cast<size_t>(e) * kExportBytes);
                const unsigned dst = static_cast<unsigned>(x.y) & 0xffu;
                const unsigned pkt = static_cast<unsigned>(x.y) >> 8;
                st_async_f64(cluster_addr(zring + zero_slot + 1 + x.z, dst), zring[x.x],
                             cluster_addr(&pbars[pkt], dst));
            }
            if (live) {
                if (m.y < 0)
                    solve_row<true, false>(rb, rowid, wpos, v, sr, zring, z_new);
                else if (nL == 0)
                    solve_row<false, true>(rb, rowid, wpos, v, sr, zring, z_new);
                else
                    solve_row<false, false>(rb, rowid, wpos, v, sr, zring, z_new);
            }
            if (nS + nL > ncons) {  // wider than the block
                for (int t = ct + ncons; t < nS + nL; t += ncons) {
                    double eb, ev[kMaxLower];
                    int er, ew, es[kMaxLower];
                    load_row(seg, nS, nL, t, zero_slot, eb, er, ew, ev, es);
                    solve_row<true, false>(eb, er, ew, ev, es, zring, z_new);
                }
            }
            // then the next level's row (its segment landed before the last barrier)
            if (L + 1 < n_levels) {
                const int4 mn = meta[L + 1];
                live = load_row(seg_of(L + 1), mn.y & 0x7fffffff, mn.z & 0xffff, ct, zero_slot, rb, rowid,
                                wpos, v, sr);
            }
        } else if (tid == 0) {
            // consumers read level L+2 during level L+1: its chunk must land first
            if (L + 2 < n_levels && meta[L + 2].w != meta[L + 1].w) wait_chunk(meta[L + 2].w);
            if (has_packets && L + 1 < n_levels) satisfy(L + 1);
        }
        __syncthreads();
        // chunk(L) is done once level L+1 starts in the next chunk: recycle it
        if (tid == 0 && L + 1 < n_levels && meta[L + 1].w != meta[L].w && meta[L].w + depth < n_chunks) {
            fence_proxy_async();
            issue(meta[L].w + depth);
        }
    }
    cluster.sync();  // no CTA leaves while others may still write into it
}

__device__ __forceinline__ double warp_shfl(double x, int src) {
    return __shfl_sync(0xffffffffu, x, src);
}

// BITWISE with precond.cpp:241-244: kRestrictGroup lanes per aggregate
// (aggregates hold ~4-8 fine rows), the lanes compute the fine residuals
// (row loads issued up front, rowdot.cuh), lane 0 of the group accumulates
// them in ascending fine-row order.
constexpr int kRestrictGroup = 8;

__global__ void k_restrict_warp(int n_coarse, const int* __restrict__ pt_ptr,
                                const int* __restrict__ pt_rows, const int* __restrict__ rp,
                                const int* __restrict__ ci, const double* __restrict__ v,
                                const double* __restrict__ r, const double* __restrict__ z,
                                double* __restrict__ rc, const double* __restrict__ next_dinv,
                                const int* __restrict__ next_bidx, double* __restrict__ next_packed) {
    pdl_begin();
    constexpr int G = kRestrictGroup;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int ag = t / G, lane = t % G;
    const bool live = ag < n_coarse;
    const int q0 = live ? pt_ptr[ag] : 0, q1 = live ? pt_ptr[ag + 1] : 0;
    // every group of the warp takes part in the shuffles of the longest one
    const int rounds = __reduce_max_sync(0xffffffffu, (q1 - q0 + G - 1) / G);
    double acc = 0.0;
    for (int b = 0; b < rounds; ++b) {
        const int base = q0 + b * G;
        double res = 0.0;
        if (base + lane < q1) {
            const int i = pt_rows[base + lane];
            double sum = 0.0;
            row_fold<8>(ci, v, rp[i], rp[i + 1], [&](int j) { return z[j]; },
                        [&](double a, double x) { sum = __dadd_rn(sum, __dmul_rn(a, x)); });
            res = __dadd_rn(r[i], __dmul_rn(-1.0, sum));
        }
        const int cnt = q1 - base;
#pragma unroll
        for (int k = 0; k < G; ++k) {
            const double x = __shfl_sync(0xffffffffu, res, k, G);
            if (k < cnt) acc = __dadd_rn(acc, x);
        }
    }
    if (live && lane == 0) {
        rc[ag] = acc;
        if (next_packed) next_packed[next_bidx[ag]] = acc * next_dinv[ag];
    }
}

int smem_budget() {
    int dev = 0, optin = 0;
    SDG_CUDA(cudaGetDevice(&dev));
    SDG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    SDG_CUDA(cudaFuncGetAttributes(&fa, k_gs_cluster));
    return std::min(kMaxSmem, optin - static_cast<int>(fa.sharedSizeBytes) - 1024);
}

// ---- level merging ---------------------------------------------------------
//
// The walk's cost is per dependency level (a latency chain), so k consecutive
// levels are merged into one group: with  z_i = bh_i - sum_{j<i} c_ij z_j
// (bh = (r - U z_old) / d, c_ij = a_ij / d_i), every lower dependency j in
// the same group is replaced by its own expression, giving
//   z_i = sum_q T_iq bh_q - sum_{j in earlier groups} G_ij z_j,
//   T_i = e_i - sum_{j int} c_ij T_j,   G_i = sum_{j ext} c_ij e_j - sum_{j int} c_ij G_j.
// The walk runs over G (one level per group); the prep computes
// b'_i = sum_q T_iq bh_q = (W r - WU z_old)_i with W = T D^{-1}, WU = T D^{-1} U.
// Exact in exact arithmetic (the same lexicographic Gauss-Seidel sweep,
// precond.cpp:92-108); rounding differs like the rest of the fast smoother.
struct MergedLower {
    HostCsr g, w, wu, t;
    std::vector<int> nlow;
    int max_k = 0;
    int groups = 0;
};

// Groups: fixed (level / k), or dynamic (dyn_cap > 0): consecutive levels
// join the open group (at most k of them) while every row's substituted lower
// part keeps <= dyn_cap entries, so the records stay narrow.
bool merge_levels(const HostCsr& a, const std::vector<double>& dinv, const HostCsr& up, int k, int cap,
                  MergedLower& out, int dyn_cap = 0) {
    const int n = a.n_rows;
    std::vector<int> lev(n, 0);
    int nlv = 0;
    for (int i = 0; i < n; ++i) {
        int d = 0;
        for (int e = a.rp[i]; e < a.rp[i + 1]; ++e)
            if (a.ci[e] < i) d = std::max(d, lev[a.ci[e]] + 1);
        lev[i] = d;
        nlv = std::max(nlv, d + 1);
    }
    std::vector<int> grp(n);
    int ng = 0;
    if (dyn_cap <= 0) {
        for (int i = 0; i < n; ++i) {
            grp[i] = lev[i] / k;
            ng = std::max(ng, grp[i] + 1);
        }
    } else {
        std::vector<int> lptr(nlv + 1, 0), lrows(n);
        for (int i = 0; i < n; ++i) ++lptr[lev[i] + 1];
        for (int l = 0; l < nlv; ++l) lptr[l + 1] += lptr[l];
        {
            std::vector<int> fill(lptr.begin(), lptr.end() - 1);
            for (int i = 0; i < n; ++i) lrows[fill[lev[i]]++] = i;
        }
        std::vector<std::vector<int>> gset(n);  // substituted lower columns (rows of the open group)
        std::vector<int> mark(n, -1);
        int cur = 0, in_group = 0;
        std::vector<int> tmp;
        auto try_level = [&](int l, bool fresh) {
            for (int p = lptr[l]; p < lptr[l + 1]; ++p) {
                const int i = lrows[p];
                tmp.clear();
                for (int e = a.rp[i]; e < a.rp[i + 1]; ++e) {
                    const int j = a.ci[e];
                    if (j >= i) continue;
                    if (!fresh && grp[j] == cur) {
                        for (int q : gset[j])
                            if (mark[q] != i) { mark[q] = i; tmp.push_back(q); }
                    } else if (mark[j] != i) {
                        mark[j] = i;
                        tmp.push_back(j);
                    }
                }
                for (int q : tmp) mark[q] = -1;
                if (!fresh && static_cast<int>(tmp.size()) > dyn_cap) return false;
                gset[i] = tmp;
            }
            return true;
        };
        for (int l = 0; l < nlv; ++l) {
            bool fresh = in_group == 0;
            if (!fresh && (in_group >= k || !try_level(l, false))) {
                ++cur;
                in_group = 0;
                fresh = true;
            }
            if (fresh) try_level(l, true);
            for (int p = lptr[l]; p < lptr[l + 1]; ++p) grp[lrows[p]] = cur;
            ++in_group;
        }
        ng = cur + 1;
    }
    // sparse accumulators (dense value + marker + touched list)
    std::vector<double> accT(n, 0.0), accG(n, 0.0);
    std::vector<int> mkT(n, -1), mkG(n, -1), lT, lG;
    HostCsr T(n, n), G(n, n);
    auto addT = [&](int i, int q, double v) {
        if (mkT[q] != i) { mkT[q] = i; accT[q] = 0.0; lT.push_back(q); }
        accT[q] += v;
    };
    auto addG = [&](int i, int j, double v) {
        if (mkG[j] != i) { mkG[j] = i; accG[j] = 0.0; lG.push_back(j); }
        accG[j] += v;
    };
    out.nlow.assign(n, 0);
    out.max_k = 0;
    for (int i = 0; i < n; ++i) {
        lT.clear();
        lG.clear();
        addT(i, i, 1.0);
        for (int e = a.rp[i]; e < a.rp[i + 1]; ++e) {
            const int j = a.ci[e];
            if (j >= i) continue;
            const double c = a.v[e] * dinv[i];
            if (grp[j] < grp[i]) {
                addG(i, j, c);
            } else {
                for (int f = T.rp[j]; f < T.rp[j + 1]; ++f) addT(i, T.ci[f], -c * T.v[f]);
                for (int f = G.rp[j]; f < G.rp[j + 1]; ++f) addG(i, G.ci[f], -c * G.v[f]);
            }
        }
        if (static_cast<int>(lG.size()) > cap) return false;
        std::sort(lT.begin(), lT.end());
        std::sort(lG.begin(), lG.end());
        for (int q : lT) { T.ci.push_back(q); T.v.push_back(accT[q]); }
        for (int j : lG) { G.ci.push_back(j); G.v.push_back(accG[j]); }
        T.rp[i + 1] = static_cast<int>(T.ci.size());
        G.rp[i + 1] = static_cast<int>(G.ci.size());
        out.nlow[i] = static_cast<int>(lG.size());
        out.max_k = std::max(out.max_k, out.nlow[i]);
    }
    // W = T D^{-1}, WU = T D^{-1} U
    HostCsr W(n, n), WU(n, up.n_cols);
    std::vector<double> accU(std::max(n, up.n_cols), 0.0);
    std::vector<int> mkU(accU.size(), -1), lU;
    for (int i = 0; i < n; ++i) {
        lU.clear();
        for (int f = T.rp[i]; f < T.rp[i + 1]; ++f) {
            const int q = T.ci[f];
            const double wq = T.v[f] * dinv[q];
            W.ci.push_back(q);
            W.v.push_back(wq);
            for (int e = up.rp[q]; e < up.rp[q + 1]; ++e) {
                const int u = up.ci[e];
                if (mkU[u] != i) { mkU[u] = i; accU[u] = 0.0; lU.push_back(u); }
                accU[u] += wq * up.v[e];
            }
        }
        std::sort(lU.begin(), lU.end());
        for (int u : lU) { WU.ci.push_back(u); WU.v.push_back(accU[u]); }
        W.rp[i + 1] = static_cast<int>(W.ci.size());
        WU.rp[i + 1] = static_cast<int>(WU.ci.size());
    }
    out.g = std::move(G);
    out.t = std::move(T);
    out.w = std::move(W);
    out.wu = std::move(WU);
    out.groups = ng;
    return true;
}

}  // namespace

// Host evaluation of one merged forward sweep (checker of merge_levels, used
// by the CPU tests through sdg_gs_merged_sweep_host): b' = W r - WU z_old,
// then z_i = b'_i - sum_j G_ij z_j in row order (G refers to earlier groups
// only).  Returns the number of groups, or -1 when a row exceeds 16 entries.
int gs_merged_sweep_host(const HostCsr& a, int k, int dyn_cap, const double* r, const double* z_old,
                         double* z_new) {
    const int n = a.n_rows;
    std::vector<double> dinv(n, 0.0);
    HostCsr up(n, n);
    for (int i = 0; i < n; ++i) {
        for (int e = a.rp[i]; e < a.rp[i + 1]; ++e) {
            if (a.ci[e] == i) dinv[i] = 1.0 / a.v[e];
            if (a.ci[e] > i) {
                up.ci.push_back(a.ci[e]);
                up.v.push_back(a.v[e]);
            }
        }
        up.rp[i + 1] = static_cast<int>(up.ci.size());
    }
    MergedLower m;
    if (!merge_levels(a, dinv, up, k, 16, m, dyn_cap)) return -1;
    for (int i = 0; i < n; ++i) {
        double b = 0.0;
        for (int e = m.w.rp[i]; e < m.w.rp[i + 1]; ++e) b += m.w.v[e] * r[m.w.ci[e]];
        if (z_old)
            for (int e = m.wu.rp[i]; e < m.wu.rp[i + 1]; ++e) b -= m.wu.v[e] * z_old[m.wu.ci[e]];
        for (int e = m.g.rp[i]; e < m.g.rp[i + 1]; ++e) b -= m.g.v[e] * z_new[m.g.ci[e]];
        z_new[i] = b;
    }
    return m.groups;
}

// ---------------------------------------------------------------------------
// plan

void GsPlan::build(const HostCsr& a, const std::vector<int>& comps, cudaStream_t s, int bands_hint,
                   bool allow_merge) {
    n = a.n_rows;
    std::vector<double> dinv_h(n);
    std::vector<int> nlow(n, 0);
    HostCsr up(n, n);
    int max_k = 0;
    for (int i = 0; i < n; ++i) {
        double d = 0.0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            if (a.ci[k] == i) d = a.v[k];
            if (a.ci[k] < i) ++nlow[i];
            if (a.ci[k] > i) {
                up.ci.push_back(a.ci[k]);
                up.v.push_back(a.v[k]);
            }
        }
        dinv_h[i] = 1.0 / d;
        up.rp[i + 1] = static_cast<int>(up.ci.size());
        max_k = std::max(max_k, nlow[i]);
    }

    // ---- bands: one for small systems, more once a single SM's bandwidth
    // becomes the bound (SDG_GS_BANDS overrides) -----------------------------
    // the single-CTA walk first (gs_walk.cu); the banded cluster kernel when
    // the walk does not fit or bands are requested (bands_hint, SDG_GS_BANDS)
    const char* bands_env = std::getenv("SDG_GS_BANDS");
    const char* walk_env = std::getenv("SDG_GS_WALK");
    const bool want_walk = bands_hint <= 0 && !bands_env && !(walk_env && walk_env[0] == '0');
    int nb = bands_hint > 0 ? bands_hint : (n >= 200000 ? 8 : n >= 80000 ? 4 : 1);
    if (bands_env) nb = std::max(1, std::atoi(bands_env));
    nb = std::max(1, std::min({nb, 8, std::max(1, n / 256)}));
    // contiguous label blocks (e.g. u / v of the velocity block)
    std::vector<int> r0{0};
    bool contiguous = comps.size() == static_cast<size_t>(n) && n > 0;
    if (contiguous) {
        std::vector<int> seen;
        for (int i = 1; i < n; ++i)
            if (comps[i] != comps[i - 1]) r0.push_back(i);
        for (size_t k = 0; k < r0.size(); ++k) {
            if (std::find(seen.begin(), seen.end(), comps[r0[k]]) != seen.end()) contiguous = false;
            seen.push_back(comps[r0[k]]);
        }
        r0.push_back(n);
    }
    auto finish = [&]() {
        dinv.upload(dinv_h, s);
        upper.upload(up, s);
        SDG_CUDA(cudaStreamSynchronize(s));
    };
    // test knobs (SDG_GS_SPLIT, SDG_GS_PIPE, SDG_GS_MERGE, SDG_GS_WAVE) apply to
    // every matrix, or only to those with SDG_GS_KNOB_ROWS rows
    const char* knob_rows = std::getenv("SDG_GS_KNOB_ROWS");
    const bool knobs = !knob_rows || std::atoi(knob_rows) == n;
    auto knob = [&](const char* name) { return knobs ? std::getenv(name) : nullptr; };
    const char* split_env = knob("SDG_GS_SPLIT");  // sequential label-block walks
    const bool force_split = split_env && split_env[0] == '1';
    const char* pipe_env = knob("SDG_GS_PIPE");
    const bool try_pipe = !force_split && pipe_env && pipe_env[0] == '1';  // opt-in
    const char* wave_env = knob("SDG_GS_WAVE");
    const bool wave_off = wave_env && wave_env[0] == '0';
    row_has_lower.assign(n, 0);
    for (int i = 0; i < n; ++i) row_has_lower[i] = nlow[i] > 0;
    // 0. the multi-SM wavefront, when the matrix is a structured finest level
    // (the knobs that force another plan skip it)
    if (want_walk && !wave_off && !force_split && !try_pipe && !knob("SDG_GS_MERGE") &&
        build_wave(a, comps, dinv_h, s))
        return finish();
    // 0a. the multi-SM lattice, when the level is an aggregated lattice
    //     (gs_lattice.cu; opt-in, SDG_GS_LATTICE=1, here and in build_parts:
    //     bitwise equal to the level walks but measured slower than them at c3,
    //     DESIGN.md §3)
    // SDG_GS_LATTICE: 0 never, 1 wherever a level (or label block) is a
    // lattice, unset: per label block the faster of the level walk and the
    // lattice, timed on the device at setup (build_parts; needs `tune`)
    const char* lat_env = knob("SDG_GS_LATTICE");
    lattice_mode_ = lat_env ? (lat_env[0] == '1' ? 1 : 0) : (tune ? 2 : 0);
    // a forced plan shape (tests pin one: SDG_GS_SPLIT / _PIPE / _MERGE) keeps the plain walks it names
    if (lattice_mode_ == 2 && (knob("SDG_GS_SPLIT") || knob("SDG_GS_PIPE") || knob("SDG_GS_MERGE"))) lattice_mode_ = 0;
    lattice_off_ = lattice_mode_ != 1;
    if (want_walk && !lattice_off_ && !force_split && !try_pipe && !knob("SDG_GS_MERGE") &&
        build_lattice(a, dinv_h, s))
        return finish();
    // 0b. one walk over merged levels: the first candidate, in the order
    //     (dynamic groups of <= 4 levels with <= 8 entries per row, fixed
    //     k = 4, 3, 2), whose modelled sweep (walk_model_cost, corrected form)
    //     is at least 10 % cheaper than the plain walk.  The model ranks merged
    //     against plain walks but not candidates among themselves (c2 launch
    //     lists: the Darcy levels gain most with 4-level groups, the velocity
    //     levels not at all once the extra prep of a merged coarse level is
    //     counted), hence the fixed order.  SDG_GS_MERGE=k forces fixed k
    //     (with SDG_GS_MERGE_CAP=c: dynamic groups of <= k levels, <= c
    //     entries), 1 disables.
    if (want_walk && allow_merge && !force_split && !try_pipe) {
        const char* me = knob("SDG_GS_MERGE");
        const char* ce = knob("SDG_GS_MERGE_CAP");
        const int kforce = me ? std::atoi(me) : 0;
        // merging pays where a level is latency-bound, i.e. narrow; wide levels
        // (> kMergeRows rows on average, c3+) are throughput-bound and only get
        // wider records, so they are not even evaluated (setup time at c4)
        constexpr int kMergeRows = 200;
        const int depth = lower_schedule(a).n_levels();
        if (kforce != 1 && (kforce > 1 || static_cast<int64_t>(depth) * kMergeRows >= n)) {
            const double base_cost = walk_model_cost(a, nlow, max_k);
            int best_k = 1;
            MergedLower bm;
            std::vector<std::pair<int, int>> cands = {{4, 8}, {4, 0}, {3, 0}, {2, 0}};  // (k, dynamic cap)
            if (kforce > 1) cands = {{kforce, ce ? std::atoi(ce) : 0}};
            for (const auto& kc : cands) {
                MergedLower m;
                if (!merge_levels(a, dinv_h, up, kc.first, 16, m, kc.second)) continue;
                const double c = walk_model_cost(m.g, m.nlow, m.max_k);
                if (std::getenv("SDG_DEBUG"))
                    std::fprintf(stderr,
                                 "[sdg gs merge] n=%d k=%d cap=%d groups=%d max_k=%d cost=%.0f (unmerged %.0f)\n", n,
                                 kc.first, kc.second, m.groups, m.max_k, c, base_cost);
                if ((kforce > 1 && c < 1e300) || c <= 0.9 * base_cost) {
                    best_k = kc.first;
                    bm = std::move(m);
                    break;
                }
            }
            if (best_k > 1) {
                const std::vector<double> ones(n, 1.0);
                if (build_walk(bm.g, ones, bm.nlow, bm.max_k, s)) {
                    merged = true;
                    merge_k = best_k;
                    wmat.upload(bm.w, s);
                    wumat.upload(bm.wu, s);
                    return finish();
                }
            }
        }
    }
    // 1. two label blocks walked concurrently on a 2-CTA cluster
    if (want_walk && try_pipe && contiguous && r0.size() == 3 && build_pipe(a, r0, dinv_h, s)) return finish();
    // 2. one walk over the whole matrix
    if (want_walk && !force_split && build_walk(a, dinv_h, nlow, max_k, s)) return finish();
    // 3. one walk per label block, in sequence, with a coupling step
    if (want_walk && contiguous && r0.size() > 2 && build_parts(a, r0, dinv_h, s)) return finish();
    walk = false;
    const int global_depth = lower_schedule(a).n_levels();
    std::vector<int> rank_in_comp(n), comp_size;
    for (int i = 0; i < n; ++i) {
        const int c = comps.empty() ? 0 : comps[i];
        if (c >= static_cast<int>(comp_size.size())) comp_size.resize(c + 1, 0);
        rank_in_comp[i] = comp_size[c]++;
    }
    std::vector<int> band_of(n);
    for (int i = 0; i < n; ++i) {
        const int c = comps.empty() ? 0 : comps[i];
        int b = static_cast<int>(static_cast<int64_t>(rank_in_comp[i]) * nb / std::max(1, comp_size[c]));
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] < i) b = std::max(b, band_of[a.ci[k]]);
        band_of[i] = b;
    }
    bands = nb;

    // ---- band-local level schedules --------------------------------------
    std::vector<int> lev(n, 0), nlev(nb, 0);
    for (int i = 0; i < n; ++i) {
        int d = 0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            const int j = a.ci[k];
            if (j < i && band_of[j] == band_of[i]) d = std::max(d, lev[j] + 1);
        }
        lev[i] = d;
        nlev[band_of[i]] = std::max(nlev[band_of[i]], d + 1);
    }
    // a band that exports gets one extra (row-less) level for its last exports
    std::vector<int> blev(nb);
    for (int b = 0; b < nb; ++b) blev[b] = nlev[b] + (nb > 1 ? 1 : 0);
    std::vector<int> lbase(nb + 1, 0);
    for (int b = 0; b < nb; ++b) lbase[b + 1] = lbase[b] + blev[b];
    n_levels = lbase[nb];
    max_band_levels = *std::max_element(blev.begin(), blev.end());

    std::vector<int> nS_of(n_levels, 0), nr_of(n_levels, 0);
    for (int i = 0; i < n; ++i) {
        const int q = lbase[band_of[i]] + lev[i];
        ++nr_of[q];
        if (nlow[i] <= 2) ++nS_of[q];
    }
    std::vector<int> lptr(n_levels + 1, 0);
    for (int q = 0; q < n_levels; ++q) lptr[q + 1] = lptr[q] + nr_of[q];
    std::vector<int> order(n), fillS(n_levels), fillL(n_levels);
    for (int q = 0; q < n_levels; ++q) {
        fillS[q] = lptr[q];
        fillL[q] = lptr[q] + nS_of[q];
    }
    for (int i = 0; i < n; ++i) {
        const int q = lbase[band_of[i]] + lev[i];
        order[nlow[i] <= 2 ? fillS[q]++ : fillL[q]++] = i;
    }
    std::vector<int> pos(n);  // band-local position in level order
    for (int b = 0; b < nb; ++b)
        for (int p = lptr[lbase[b]]; p < lptr[lbase[b + 1]]; ++p) pos[order[p]] = p - lptr[lbase[b]];

    // ---- halo imports, packets, exports, requirements ------------------------
    // A packet = the values band b imports from one level of one upstream
    // band; it completes a single-use mbarrier in band b.
    std::vector<std::vector<std::pair<int, int>>> imports(nb);  // (row j, halo index)
    std::vector<int> halo_n(nb, 0);
    std::vector<std::vector<int4>> exports(n_levels);  // keyed by the level that executes them
    std::vector<int> req_ptr_h(n_levels + 1, 0);
    std::vector<int> req_h;
    std::vector<int> pkt_base(nb + 1, 0);
    std::vector<int> pkt_bytes_h;
    {
        std::vector<int> halo_band(n, -1);
        cross_refs = 0;
        for (int b = 0; b < nb; ++b) {
            pkt_base[b] = static_cast<int>(pkt_bytes_h.size());
            std::map<std::pair<int, int>, int> pkt_of;  // (upstream band, its level) -> packet
            std::vector<char> waited;
            for (int L = 0; L < blev[b]; ++L) {
                const int q = lbase[b] + L;
                for (int p = lptr[q]; p < lptr[q + 1]; ++p) {
                    const int i = order[p];
                    for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
                        const int j = a.ci[k];
                        if (j >= i || band_of[j] == b) continue;
                        ++cross_refs;
                        const int bj = band_of[j];
                        const auto key = std::make_pair(bj, lev[j]);
                        auto it = pkt_of.find(key);
                        if (it == pkt_of.end()) {
                            it = pkt_of.emplace(key, static_cast<int>(pkt_bytes_h.size()) - pkt_base[b]).first;
                            pkt_bytes_h.push_back(0);
                            waited.push_back(0);
                        }
                        const int pk = it->second;
                        if (halo_band[j] != b) {  // first import of j into band b
                            halo_band[j] = b;
                            const int h = halo_n[b]++;
                            imports[b].push_back({j, h});
                            pkt_bytes_h[pkt_base[b] + pk] += 8;
                            // exported by band bj while it walks level lev[j] + 1
                            exports[lbase[bj] + lev[j] + 1].push_back(make_int4(0, b | (pk << 8), h, j));
                        }
                        if (!waited[pk]) {  // the first level that reads a packet waits for it
                            waited[pk] = 1;
                            req_h.push_back(pk);
                        }
                    }
                }
                req_ptr_h[q + 1] = static_cast<int>(req_h.size());
            }
        }
        pkt_base[nb] = static_cast<int>(pkt_bytes_h.size());
    }
    halo = std::max(1, *std::max_element(halo_n.begin(), halo_n.end()));
    max_packets = 1;
    for (int b = 0; b < nb; ++b) max_packets = std::max(max_packets, pkt_base[b + 1] - pkt_base[b]);

    // ---- segments and chunks -------------------------------------------------
    // level q's segment: [small records][large records][exports]; consecutive
    // levels of a band are grouped into chunks of about kChunkTarget bytes,
    // each brought in by one TMA copy
    constexpr int kChunkTarget = 24 * 1024;
    std::vector<int> lvl_abs16(n_levels), lvl_bytes(n_levels);
    std::vector<int4> mh(n_levels);   // {local off16, nS | flag, nL | nE << 16, band-local chunk}
    std::vector<int4> ch_h;           // {off16, bytes16, first level, levels}
    std::vector<int> ch_base(nb + 1, 0);
    int64_t off = 0;
    int max_rows = 1, max_exp = 0;
    max_seg = 16;
    for (int b = 0; b < nb; ++b) {
        ch_base[b] = static_cast<int>(ch_h.size());
        int chunk_bytes = 0;
        for (int L = 0; L < blev[b]; ++L) {
            const int q = lbase[b] + L;
            const int nS = nS_of[q], nL = nr_of[q] - nS_of[q], nE = static_cast<int>(exports[q].size());
            if (nL > 0xffff || nE > 0x7fff) fail(SDG_EINVAL, "gs plan: level too wide");
            const int bytes = nS * kSmallBytes + nL * kLargeBytes + nE * kExportBytes;
            if (L == 0 || chunk_bytes + bytes > kChunkTarget) {
                ch_h.push_back(make_int4(static_cast<int>(off / 16), 0, L, 0));
                chunk_bytes = 0;
            }
            int4& ch = ch_h.back();
            lvl_abs16[q] = static_cast<int>(off / 16);
            lvl_bytes[q] = bytes;
            mh[q] = make_int4(chunk_bytes / 16, nS, nL | (nE << 16), static_cast<int>(ch_h.size()) - 1 - ch_base[b]);
            chunk_bytes += bytes;
            ch.y = chunk_bytes / 16;
            ch.w += 1;
            off += bytes;
            max_seg = std::max(max_seg, chunk_bytes);
            max_rows = std::max(max_rows, nr_of[q]);
            max_exp = std::max(max_exp, nE);
        }
    }
    ch_base[nb] = static_cast<int>(ch_h.size());
    if (off / 8 + 2 > (static_cast<int64_t>(1) << 31)) fail(SDG_EINVAL, "gs plan: packed buffer too large");

    int max_dist = 2;      // in-band dependency distance in level-order positions
    int max_exp_dist = 2;  // exports read the ring one level after the value was written
    for (int b = 0; b < nb; ++b)
        for (int q = lbase[b]; q < lbase[b + 1]; ++q) {
            const int band_end = lptr[q + 1] - lptr[lbase[b]];
            for (int p = lptr[q]; p < lptr[q + 1]; ++p) {
                const int i = order[p];
                for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
                    const int j = a.ci[k];
                    if (j < i && band_of[j] == b) max_dist = std::max(max_dist, band_end - pos[j]);
                }
                if (q + 1 < lbase[b + 1])
                    max_exp_dist = std::max(max_exp_dist, lptr[q + 2] - lptr[lbase[b]] - pos[i]);
            }
        }

    int max_band_chunks = 1;
    for (int b = 0; b < nb; ++b) max_band_chunks = std::max(max_band_chunks, ch_base[b + 1] - ch_base[b]);
    const int budget = smem_budget();
    const int meta_bytes = pad16(static_cast<int64_t>(max_band_levels + 1) * 16);
    const int chunk_tab_bytes = pad16(static_cast<int64_t>(max_band_chunks) * 16);
    const int pbar_bytes = pad16(static_cast<int64_t>(max_packets) * 8);
    const int base_bytes = 128 + 2 * meta_bytes + chunk_tab_bytes + pbar_bytes;
    // z ring: large enough for every in-band dependency when four chunk slots
    // still fit, else the largest power of two that does
    const int ring_room = (budget - base_bytes - (halo + 2) * 8 - 16 - 4 * max_seg) / 8;
    int min_ring = 64;
    while (min_ring < max_exp_dist) min_ring <<= 1;  // exports must find their values
    ring = 1;
    while (ring < max_dist && ring < 32768) ring <<= 1;
    while (ring > min_ring && ring > ring_room) ring >>= 1;
    ring = std::max(ring, min_ring);

    std::vector<double> pk(static_cast<size_t>(off / 8 + 2), 0.0);
    unsigned char* base = reinterpret_cast<unsigned char*>(pk.data());
    std::vector<int> bidx_h(n);
    global_refs = 0;
    lower_entries = 0;
    std::vector<int> halo_lookup(n, -1);
    for (int b = 0; b < nb; ++b) {
        for (auto& jh : imports[b]) halo_lookup[jh.first] = jh.second;
        for (int L = 0; L < blev[b]; ++L) {
            const int q = lbase[b] + L;
            int4& m = mh[q];
            const int band_end = lptr[q + 1] - lptr[lbase[b]];
            const int nS = m.y, nL = m.z & 0xffff;
            unsigned char* seg = base + static_cast<size_t>(lvl_abs16[q]) * 16;
            for (int p = lptr[q]; p < lptr[q + 1]; ++p) {
                const int t = p - lptr[q];
                const int i = order[p];
                const bool small = t < nS;
                unsigned char* rec = seg + (small ? static_cast<size_t>(t) * kSmallBytes
                                                  : static_cast<size_t>(nS) * kSmallBytes +
                                                        static_cast<size_t>(t - nS) * kLargeBytes);
                double* recd = reinterpret_cast<double*>(rec);
                int* reci = reinterpret_cast<int*>(rec);
                bidx_h[i] = static_cast<int>((rec - base) / 8);
                reci[2] = i;                      // rowid
                reci[3] = pos[i] & (ring - 1);    // wpos
                const int kcap = small ? 2 : kMaxLower;
                double* val = recd + 2;
                int* src = reci + (small ? 8 : 20);
                int k2 = 0;
                for (int k = a.rp[i]; k < a.rp[i + 1] && k2 < kcap; ++k) {
                    const int j = a.ci[k];
                    if (j >= i) continue;
                    val[k2] = a.v[k] * dinv_h[i];
                    if (band_of[j] != b) {
                        src[k2] = ring + 1 + halo_lookup[j];
                    } else if (band_end - pos[j] <= ring) {
                        src[k2] = pos[j] & (ring - 1);
                    } else {
                        src[k2] = -(j + 1);
                        ++global_refs;
                        m.y |= static_cast<int>(0x80000000u);
                    }
                    ++k2;
                    ++lower_entries;
                }
                for (; k2 < kcap; ++k2) {
                    val[k2] = 0.0;
                    src[k2] = ring;  // zero slot
                }
            }
            // export entries executed at this level (values of level L-1)
            int* ex = reinterpret_cast<int*>(seg + static_cast<size_t>(nS) * kSmallBytes +
                                             static_cast<size_t>(nL) * kLargeBytes);
            for (size_t e = 0; e < exports[q].size(); ++e) {
                const int4 x = exports[q][e];
                ex[4 * e + 0] = pos[x.w] & (ring - 1);  // local ring slot of row j
                ex[4 * e + 1] = x.y;                    // destination band | packet << 8
                ex[4 * e + 2] = x.z;                    // destination halo index
                ex[4 * e + 3] = 0;
            }
        }
        for (auto& jh : imports[b]) halo_lookup[jh.first] = -1;
    }

    nthreads = 32 + std::min(480, (std::max(max_rows, max_exp) + 31) / 32 * 32);
    const int fixed = base_bytes + pad16(static_cast<int64_t>(ring + 1 + halo) * 8);
    depth = std::min(6, std::max(0, (budget - fixed) / std::max(max_seg, 16)));
    usable = depth >= 3 && max_k <= kMaxLower && ring >= max_exp_dist;
    smem = static_cast<size_t>(fixed) + static_cast<size_t>(std::max(depth, 0)) * max_seg;
    if (std::getenv("SDG_DEBUG"))
        std::fprintf(stderr,
                     "[sdg gs plan] n=%d bands=%d levels(max/band)=%d global_depth=%d threads=%d ring=%d "
                     "halo=%d chunks=%zu depth=%d max_chunk=%d smem=%zu cross_refs=%lld global_refs=%lld "
                     "packets=%zu packed=%.1fKB usable=%d max_k=%d\n",
                     n, nb, max_band_levels, global_depth, nthreads, ring, halo, ch_h.size(), depth, max_seg,
                     smem, (long long)cross_refs, (long long)global_refs, pkt_bytes_h.size(), off / 1024.0,
                     (int)usable, max_k);

    std::vector<int4> binfo(2 * nb);
    for (int b = 0; b < nb; ++b) {
        binfo[b] = make_int4(lbase[b], blev[b], pkt_base[b], pkt_base[b + 1] - pkt_base[b]);
        binfo[nb + b] = make_int4(ch_base[b], ch_base[b + 1] - ch_base[b], 0, 0);
    }
    if (req_h.empty()) req_h.push_back(0);
    if (pkt_bytes_h.empty()) pkt_bytes_h.push_back(0);
    meta.upload(mh, s);
    band_info.upload(binfo, s);
    req_ptr.upload(req_ptr_h, s);
    req.upload(req_h, s);
    packet_bytes.upload(pkt_bytes_h, s);
    chunk_tab.upload(ch_h, s);
    packed.upload(pk, s);
    bidx.upload(bidx_h, s);
    dinv.upload(dinv_h, s);
    upper.upload(up, s);
    meta_bytes_ = meta_bytes;
    chunk_tab_bytes_ = chunk_tab_bytes;
    pbar_bytes_ = pbar_bytes;
    if (usable) {
        SDG_CUDA(cudaFuncSetAttribute(k_gs_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
        SDG_CUDA(cudaFuncSetAttribute(k_gs_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    SDG_CUDA(cudaStreamSynchronize(s));  // host staging vectors die here
}

// mean device time (ms) of one lower solve of a stand-alone plan (its own records)
static double time_lower(Context& c, const GsPlan& g) {
    DevBuf<double> z(std::max(g.n, 1)), tmp;
    if (g.merged_part) {  // stand-alone: b' = T b from a zero scratch into the plan's own records
        tmp.resize(std::max(g.n, 1));
        SDG_CUDA(cudaMemsetAsync(tmp.get(), 0, sizeof(double) * std::max(g.n, 1), c.stream));
    }
    auto sweep = [&]() {
        if (g.merged_part)
            launch_k(c, k_gs_tapply, (g.n + 255) / 256, 256, 0, g.n, g.tmat.rp.get(), g.tmat.ci.get(), g.tmat.v.get(),
                     static_cast<const double*>(tmp.get()), static_cast<const int*>(g.bidx.get()),
                     const_cast<double*>(g.packed.get()));
        launch_gs_lower(c, g, z.get());
    };
    cudaEvent_t e0, e1;
    SDG_CUDA(cudaEventCreate(&e0));
    SDG_CUDA(cudaEventCreate(&e1));
    for (int r = 0; r < 2; ++r) sweep();
    constexpr int kReps = 6;
    SDG_CUDA(cudaEventRecord(e0, c.stream));
    for (int r = 0; r < kReps; ++r) sweep();
    SDG_CUDA(cudaEventRecord(e1, c.stream));
    SDG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    SDG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ms / kReps;
}

bool GsPlan::build_parts(const HostCsr& a, const std::vector<int>& r0, const std::vector<double>& dinv_h,
                         cudaStream_t s) {
    const int nparts = static_cast<int>(r0.size()) - 1;
    std::vector<std::unique_ptr<GsPlan>> ps;
    for (int k = 0; k < nparts; ++k) {
        const int lo = r0[k], hi = r0[k + 1], m = hi - lo;
        HostCsr sub(m, m);
        std::vector<double> dsub(dinv_h.begin() + lo, dinv_h.begin() + hi);
        std::vector<int> nlow(m, 0);
        int max_k = 0;
        for (int i = lo; i < hi; ++i) {
            for (int e = a.rp[i]; e < a.rp[i + 1]; ++e) {
                const int j = a.ci[e];
                if (j < lo || j >= hi) continue;
                sub.ci.push_back(j - lo);
                sub.v.push_back(a.v[e]);
                if (j < i) ++nlow[i - lo];
            }
            sub.rp[i - lo + 1] = static_cast<int>(sub.ci.size());
            max_k = std::max(max_k, nlow[i - lo]);
        }
        auto p = std::make_unique<GsPlan>();
        if (lattice_mode_ == 2 && tune) {
            // measured choice between the plain level walk, the multi-SM lattice and a walk over
            // merged levels: every candidate sweeps its own (zero) records a few times
            if (!p->build_walk(sub, dsub, nlow, max_k, s)) return false;
            std::vector<std::unique_ptr<GsPlan>> cand;
            std::vector<const char*> names;
            {
                auto q = std::make_unique<GsPlan>();
                if (q->build_lattice(sub, dsub, s)) {
                    cand.push_back(std::move(q));
                    names.push_back("lattice");
                }
            }
            const char* pm_env = std::getenv("SDG_GS_PART_MERGE");
            if (!(pm_env && pm_env[0] == '0')) {
                HostCsr upsub(m, m);  // the block's own upper part: only T and G of the merge are used
                const std::pair<int, int> kc[4] = {{4, 8}, {2, 0}, {3, 0}, {4, 0}};  // (levels, dynamic entry cap)
                static const char* const kc_names[4] = {"merged walk (<= 4 levels, <= 8 entries)", "merged walk (2 levels)",
                                                        "merged walk (3 levels)", "merged walk (4 levels)"};
                for (int ic = 0; ic < 4; ++ic) {
                    const auto& c = kc[ic];
                    MergedLower ml;
                    if (!merge_levels(sub, dsub, upsub, c.first, 16, ml, c.second)) continue;
                    auto q = std::make_unique<GsPlan>();
                    const std::vector<double> ones(m, 1.0);
                    if (!q->build_walk(ml.g, ones, ml.nlow, ml.max_k, s)) continue;
                    q->merged_part = true;
                    q->merge_k = c.first;
                    q->tmat.upload(ml.t, s);
                    cand.push_back(std::move(q));
                    names.push_back(kc_names[ic]);
                }
            }
            if (!cand.empty()) {
                // the first decision for a block of this shape holds for the process: two
                // preconditioners of one system must run the same plan (their applies are
                // compared bit for bit), whatever the timer says the second time
                static std::mutex mu;
                static std::map<std::tuple<int, int64_t, int>, int> decided;
                const auto key = std::make_tuple(m, sub.nnz(), k);
                int choice = -2;  // -1: the plain walk, >= 0: cand[choice]
                {
                    std::lock_guard<std::mutex> g(mu);
                    auto it = decided.find(key);
                    if (it != decided.end()) choice = it->second;
                }
                if (choice == -2) {
                    const double tw = time_lower(*tune, *p);
                    double best = 0.9 * tw;  // an alternative must win by 10 %
                    choice = -1;
                    for (size_t q = 0; q < cand.size(); ++q) {
                        const double tq = time_lower(*tune, *cand[q]);
                        if (std::getenv("SDG_DEBUG"))
                            std::fprintf(stderr, "[sdg gs plan] label block %d (%d rows): walk %.1f us, %s %.1f us\n", k, m,
                                         tw * 1e3, names[q], tq * 1e3);
                        if (tq < best) {
                            best = tq;
                            choice = static_cast<int>(q);
                        }
                    }
                    std::lock_guard<std::mutex> g(mu);
                    decided.emplace(key, choice);
                }
                if (choice >= 0 && choice < static_cast<int>(cand.size())) p = std::move(cand[choice]);
            }
        } else if (!(lattice_mode_ == 1 && p->build_lattice(sub, dsub, s)) &&
                   !p->build_walk(sub, dsub, nlow, max_k, s)) {
            return false;
        }
        ps.push_back(std::move(p));
    }
    // one record buffer; the prep kernels write b through the global bidx
    size_t total = 0;
    std::vector<size_t> off(nparts);
    for (int k = 0; k < nparts; ++k) {
        off[k] = total;
        total += (ps[k]->packed.size() + 31) / 32 * 32;  // 256-byte aligned parts: TMA sources
        if (ps[k]->merged_part) {  // the plain b of a merged block lands in a temporary region first
            ps[k]->part_tmp_off = total;
            total += (static_cast<size_t>(ps[k]->n) + 31) / 32 * 32;
        }
    }
    if (total > static_cast<size_t>(INT32_MAX)) return false;  // bidx is int
    packed.resize(total);
    SDG_CUDA(cudaMemsetAsync(packed.get(), 0, total * sizeof(double), s));
    std::vector<int> bidx_h(n);
    for (int k = 0; k < nparts; ++k) {
        GsPlan& p = *ps[k];
        SDG_CUDA(cudaMemcpyAsync(packed.get() + off[k], p.packed.get(), p.packed.size() * 8,
                                 cudaMemcpyDeviceToDevice, s));
        std::vector<int> lb(p.n);
        SDG_CUDA(cudaMemcpyAsync(lb.data(), p.bidx.get(), p.n * sizeof(int), cudaMemcpyDeviceToHost, s));
        SDG_CUDA(cudaStreamSynchronize(s));
        if (p.merged_part) {
            for (int i = 0; i < p.n; ++i) {
                bidx_h[r0[k] + i] = static_cast<int>(p.part_tmp_off) + i;
                lb[i] += static_cast<int>(off[k]);
            }
            p.part_bidx.upload(lb, s);
            SDG_CUDA(cudaStreamSynchronize(s));
        } else {
            for (int i = 0; i < p.n; ++i) bidx_h[r0[k] + i] = static_cast<int>(off[k]) + lb[i];
        }
        p.part_doubles = p.packed.size();
        p.packed.release();
        p.bidx.release();
        p.packed_ptr = packed.get() + off[k];
    }
    bidx.upload(bidx_h, s);
    couple.resize(nparts);
    for (int k = 1; k < nparts; ++k) {
        HostCsr cp(r0[k + 1] - r0[k], n);
        for (int i = r0[k]; i < r0[k + 1]; ++i) {
            for (int e = a.rp[i]; e < a.rp[i + 1]; ++e)
                if (a.ci[e] < r0[k]) {
                    cp.ci.push_back(a.ci[e]);
                    cp.v.push_back(-(a.v[e] * dinv_h[i]));
                }
            cp.rp[i - r0[k] + 1] = static_cast<int>(cp.ci.size());
        }
        couple[k].upload(cp, s);
    }
    parts = std::move(ps);
    part_r0 = r0;
    walk = false;
    usable = true;
    bands = 1;
    n_levels = 0;
    for (auto& p : parts) n_levels += p->n_levels;
    if (std::getenv("SDG_DEBUG"))
        std::fprintf(stderr, "[sdg gs plan] n=%d: %d label blocks, one walk each (%d levels in sequence)\n", n, nparts,
                     n_levels);
    return true;
}

// Two label blocks walked concurrently: CTA 0 walks block 0 and pushes the
// values block 1 needs into CTA 1's import slots (a ring of kImportRing slots,
// in export order); CTA 1 walks block 1, waiting at each level for the block-0
// levels its imports come from.  Back-pressure: before a block-0 level
// overwrites import slots, CTA 0 waits for the block-1 levels that last read
// them.  A host simulation of the two schedules rules out a deadlock.
bool GsPlan::build_pipe(const HostCsr& a, const std::vector<int>& r0, const std::vector<double>& dinv_h,
                        cudaStream_t s) {
    const int lo1 = r0[1], n0 = r0[1], n1 = n - r0[1];
    auto debug = std::getenv("SDG_DEBUG");
    auto reject = [&](const char* why) {
        if (debug) std::fprintf(stderr, "[sdg gs plan] n=%d: no 2-CTA pipe (%s)\n", n, why);
        return false;
    };
    // block matrices: A00 (local), A11 (local), L10 (block-1 rows x block-0 columns, lower by construction)
    HostCsr a0(n0, n0), a1(n1, n1), l10(n1, n0);
    std::vector<int> nlow0(n0, 0), nlow1(n1, 0);
    int maxk0 = 0, maxk1 = 0;
    for (int i = 0; i < n; ++i) {
        for (int e = a.rp[i]; e < a.rp[i + 1]; ++e) {
            const int j = a.ci[e];
            if (i < lo1) {
                if (j < lo1) {
                    a0.ci.push_back(j);
                    a0.v.push_back(a.v[e]);
                    if (j < i) ++nlow0[i];
                }
            } else if (j >= lo1) {
                a1.ci.push_back(j - lo1);
                a1.v.push_back(a.v[e]);
                if (j < i) ++nlow1[i - lo1];
            } else {
                l10.ci.push_back(j);
                l10.v.push_back(a.v[e]);
                ++nlow1[i - lo1];
            }
        }
        if (i < lo1) {
            a0.rp[i + 1] = static_cast<int>(a0.ci.size());
            maxk0 = std::max(maxk0, nlow0[i]);
        } else {
            a1.rp[i - lo1 + 1] = static_cast<int>(a1.ci.size());
            l10.rp[i - lo1 + 1] = static_cast<int>(l10.ci.size());
            maxk1 = std::max(maxk1, nlow1[i - lo1]);
        }
    }
    std::vector<double> d0(dinv_h.begin(), dinv_h.begin() + lo1), d1(dinv_h.begin() + lo1, dinv_h.end());

    // pass 1: each block's own shape -> one common kernel shape and record width
    Link s0, s1;
    s0.role = 1;
    s1.role = 2;
    s1.ext = &l10;
    std::vector<int> zero_slot_of(n0, 0), zero_plv(n0, 0);
    s1.ext_slot = &zero_slot_of;
    s1.ext_plv = &zero_plv;
    s1.import_slots = 1;
    {
        GsPlan t0, t1;
        if (!t0.build_walk(a0, d0, nlow0, maxk0, s, &s0)) return reject("block 0 does not fit a walk");
        if (!t1.build_walk(a1, d1, nlow1, maxk1, s, &s1)) return reject("block 1 does not fit a walk");
    }
    Link f0, f1;
    f0.force_w = f1.force_w = std::max(s0.shape[0], s1.shape[0]);
    f0.force_r2 = f1.force_r2 = std::max(s0.shape[1], s1.shape[1]);
    f0.force_r8 = f1.force_r8 = std::max(s0.shape[2], s1.shape[2]);
    f0.force_kw = f1.force_kw = std::max(s0.shape[3], s1.shape[3]);
    // pass 2: block 0's levels -> exports in level order -> import slots (a ring)
    std::vector<int> plv0, plv1;
    f0.role = 1;
    f0.plv_out = &plv0;
    {
        GsPlan t0;
        if (!t0.build_walk(a0, d0, nlow0, maxk0, s, &f0)) return reject("block 0 with the common shape");
    }
    std::vector<char> needed(n0, 0);
    for (int j : l10.ci) needed[j] = 1;
    std::vector<int> exported;
    for (int j = 0; j < n0; ++j)
        if (needed[j]) exported.push_back(j);
    std::stable_sort(exported.begin(), exported.end(), [&](int x, int y) { return plv0[x] < plv0[y]; });
    const int nexp = static_cast<int>(exported.size());
    int per_level = 1, nlev0 = 0;
    for (int j = 0; j < n0; ++j) nlev0 = std::max(nlev0, plv0[j] + 1);
    {
        std::vector<int> cnt(nlev0 + 1, 0);
        for (int j : exported) per_level = std::max(per_level, ++cnt[plv0[j]]);
    }
    int ring_slots = 1024;
    while (ring_slots < 24 * per_level && ring_slots < 8192) ring_slots <<= 1;
    std::vector<int> slot(n0, -1);
    for (int k = 0; k < nexp; ++k) slot[exported[k]] = k % ring_slots;
    // block 1 with its imports
    f1.role = 2;
    f1.ext = &l10;
    f1.ext_slot = &slot;
    f1.ext_plv = &plv0;
    f1.import_slots = ring_slots;
    f1.plv_out = &plv1;
    std::vector<int> peer_bytes(nlev0, 0);
    for (int j : exported) peer_bytes[plv0[j]] += 8;
    f1.peer_bytes = &peer_bytes;
    auto q1 = std::make_unique<GsPlan>();
    if (!q1->build_walk(a1, d1, nlow1, maxk1, s, &f1)) return reject("block 1 with its imports");
    // back-pressure: block-0 level X may overwrite export k - ring_slots once
    // the block-1 levels reading it are done
    std::vector<int> last_read(n0, -1);
    for (int i = 0; i < n1; ++i)
        for (int e = l10.rp[i]; e < l10.rp[i + 1]; ++e)
            last_read[l10.ci[e]] = std::max(last_read[l10.ci[e]], plv1[i]);
    std::vector<int> need(nlev0, 0);
    for (int k = ring_slots; k < nexp; ++k) {
        const int x = plv0[exported[k]];
        need[x] = std::max(need[x], last_read[exported[k - ring_slots]] + 1);
    }
    // no deadlock: both schedules advance whenever allowed and finish
    {
        std::vector<int> sync1(q1->n_levels, 0);
        for (int i = 0; i < n1; ++i)
            for (int e = l10.rp[i]; e < l10.rp[i + 1]; ++e)
                sync1[plv1[i]] = std::max(sync1[plv1[i]], plv0[l10.ci[e]] + 1);
        int d0l = 0, d1l = 0;
        while (d0l < nlev0 || d1l < q1->n_levels) {
            bool moved = false;
            while (d0l < nlev0 && need[d0l] <= d1l) ++d0l, moved = true;
            while (d1l < q1->n_levels && sync1[d1l] <= d0l) ++d1l, moved = true;
            if (!moved) return reject("the import ring would deadlock");
        }
    }
    // pass 3: block 0 with its exports and back-pressure levels
    std::vector<int> plv0b;
    f0.plv_out = &plv0b;
    f0.export_slot = &slot;
    f0.export_need = &need;
    f0.export_base = q1->walk_import_base;
    auto q0 = std::make_unique<GsPlan>();
    if (!q0->build_walk(a0, d0, nlow0, maxk0, s, &f0)) return reject("block 0 with its exports");
    if (plv0b != plv0) return reject("block 0 changed its level split");
    if (nlev0 > 4096) return reject("too many block-0 levels for the mbarriers");
    const int w = f0.force_w, r2 = f0.force_r2, r8 = f0.force_r8, kw = f0.force_kw;
    if (r2 > 2 || r8 > 2) return reject("no pipe instantiation for the shape");
    // one record buffer (as build_parts), global bidx for the prep kernels
    std::vector<std::unique_ptr<GsPlan>> ps;
    ps.push_back(std::move(q0));
    ps.push_back(std::move(q1));
    size_t total = 0;
    std::vector<size_t> off(2);
    for (int k = 0; k < 2; ++k) {
        off[k] = total;
        total += ps[k]->packed.size();
    }
    packed.resize(total);
    std::vector<int> bidx_h(n);
    for (int k = 0; k < 2; ++k) {
        GsPlan& p = *ps[k];
        SDG_CUDA(cudaMemcpyAsync(packed.get() + off[k], p.packed.get(), p.packed.size() * 8,
                                 cudaMemcpyDeviceToDevice, s));
        std::vector<int> lb(p.n);
        SDG_CUDA(cudaMemcpyAsync(lb.data(), p.bidx.get(), p.n * sizeof(int), cudaMemcpyDeviceToHost, s));
        SDG_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < p.n; ++i) bidx_h[r0[k] + i] = static_cast<int>(off[k]) + lb[i];
        p.part_doubles = p.packed.size();
        p.packed.release();
        p.bidx.release();
        p.packed_ptr = packed.get() + off[k];
    }
    bidx.upload(bidx_h, s);
    parts = std::move(ps);
    part_r0 = r0;
    couple.clear();
    pipe = true;
    walk = false;
    usable = true;
    bands = 2;
    n_levels = std::max(parts[0]->n_levels, parts[1]->n_levels);
    if (debug)
        std::fprintf(stderr,
                     "[sdg gs plan] n=%d: 2-CTA pipe, blocks %d + %d rows, %d + %d levels, %d exports, import ring %d, "
                     "shape warps=%d rows/thread=%d+%d wide=%d\n",
                     n, n0, n1, parts[0]->n_levels, parts[1]->n_levels, nexp, ring_slots, w, r2, r8, kw);
    return true;
}

// ---------------------------------------------------------------------------
// launchers

#define SDG_GS_CHECK()                                                                      \
    do {                                                                                    \
        c.count();                                                                          \
        cudaError_t e_ = cudaGetLastError();                                                \
        if (e_ != cudaSuccess) fail(SDG_ECUDA, std::string(__func__) + ": " + cudaGetErrorString(e_)); \
    } while (0)

void launch_gs_prep_pre(Context& c, const GsPlan& g, const double* r) {
    if (g.merged) {
        ProfScope ps_(c, PF_GSPREP, 12.0 * g.wmat.nnz + 4.0 * (g.n + 1) + 16.0 * g.n);
        if (g.n == 0) return;
        launch_k(c, k_gs_prep_m, (g.n * kGroup + 255) / 256, 256, 0, g.n, g.wmat.rp.get(), g.wmat.ci.get(),
                 g.wmat.v.get(), g.wumat.rp.get(), g.wumat.ci.get(), g.wumat.v.get(), r,
                 static_cast<const double*>(nullptr), static_cast<const double*>(nullptr),
                 static_cast<const int*>(nullptr), g.bidx.get(), const_cast<double*>(g.packed.get()));
        SDG_GS_CHECK();
        return;
    }
    ProfScope ps_(c, PF_GSPREP, 24.0 * g.n + 8.0 * g.n);
    if (g.n == 0) return;
    launch_k(c, k_gs_prep_pre, (g.n + 255) / 256, 256, 0, g.n, r, g.dinv.get(), g.bidx.get(),
                                                            const_cast<double*>(g.packed.get()));
    SDG_GS_CHECK();
}

void launch_gs_prep_post(Context& c, const GsPlan& g, const double* r, const double* z,
                         const double* zc, const int* agg) {
    if (g.merged) {
        ProfScope ps_(c, PF_GSPREP,
                      12.0 * (g.wmat.nnz + g.wumat.nnz) + 8.0 * (g.n + 1) + 8.0 * g.n * (z ? 2 : 1) +
                          (zc ? 12.0 * g.n : 0.0) + 16.0 * g.n);
        if (g.n == 0) return;
        launch_k(c, k_gs_prep_m, (g.n * kGroup + 255) / 256, 256, 0, g.n, g.wmat.rp.get(), g.wmat.ci.get(),
                 g.wmat.v.get(), g.wumat.rp.get(), g.wumat.ci.get(), g.wumat.v.get(), r, z, zc, agg,
                 g.bidx.get(), const_cast<double*>(g.packed.get()));
        SDG_GS_CHECK();
        return;
    }
    ProfScope ps_(c, PF_GSPREP,
                  12.0 * g.upper.nnz + 4.0 * (g.n + 1) + 8.0 * g.n * (z ? 2 : 1) + (zc ? 12.0 * g.n : 0.0) +
                      16.0 * g.n);
    if (g.n == 0) return;
    launch_k(c, k_gs_prep_post, (g.n + 255) / 256, 256, 0, 
        g.n, g.upper.rp.get(), g.upper.ci.get(), g.upper.v.get(), r, z, zc, agg, g.dinv.get(),
        g.bidx.get(), const_cast<double*>(g.packed.get()));
    SDG_GS_CHECK();
}

void launch_gs_lower(Context& c, const GsPlan& g, double* z_new, cudaEvent_t mark) {
    if (g.pipe) {
        ProfScope ps_(c, PF_GS, g.packed_bytes() + 8.0 * g.n);
        launch_gs_pipe(c, g, z_new);
        return;
    }
    if (!g.parts.empty()) {
        for (size_t k = 0; k < g.parts.size(); ++k) {
            if (k > 0) {
                const DevCsr& cp = g.couple[k];
                ProfScope ps_(c, PF_GSPREP, 12.0 * cp.nnz + 4.0 * (cp.n_rows + 1) + 28.0 * cp.n_rows);
                launch_k(c, k_gs_couple, (cp.n_rows + 255) / 256, 256, 0, 
                    cp.n_rows, g.part_r0[k], cp.rp.get(), cp.ci.get(), cp.v.get(), z_new, g.bidx.get(),
                    const_cast<double*>(g.packed.get()));
                SDG_GS_CHECK();
            }
            const GsPlan& part = *g.parts[k];
            if (part.merged_part) {
                ProfScope ps_(c, PF_GSPREP, 12.0 * part.tmat.nnz + 4.0 * (part.n + 1) + 16.0 * part.n);
                launch_k(c, k_gs_tapply, (part.n + 255) / 256, 256, 0, part.n, part.tmat.rp.get(), part.tmat.ci.get(),
                         part.tmat.v.get(), g.packed.get() + part.part_tmp_off,
                         static_cast<const int*>(part.part_bidx.get()), const_cast<double*>(g.packed.get()));
                SDG_GS_CHECK();
            }
            launch_gs_lower(c, part, z_new + g.part_r0[k], k + 1 == g.parts.size() ? mark : nullptr);
        }
        return;
    }
    if (g.lattice) {
        ProfScope ps_(c, PF_GS_LATTICE, g.packed_bytes() + 8.0 * g.n);
        launch_gs_lattice(c, g, z_new);
        SDG_GS_CHECK();
        return;
    }
    if (g.wave) {
        // algorithmic bytes: the band records (b and the scaled lower
        // coefficients, [band][block][field][step][lane] incl. the skew
        // padding) streamed once, z written once, lane 0's south row read once
        ProfScope ps_(c, PF_GS_WAVE, g.packed_bytes() + 8.0 * g.n + 16.0 * g.wave_nx * g.wave_bands);
        if (mark) SDG_CUDA(cudaEventRecord(mark, c.stream));
        launch_gs_wave(c, g, z_new);
        SDG_GS_CHECK();
        return;
    }
    ProfScope ps_(c, PF_GS, g.packed_bytes() + 8.0 * g.n);
    if (g.n == 0) return;
    if (g.walk) {
        if (mark) SDG_CUDA(cudaEventRecord(mark, c.stream));
        launch_gs_walk(c, g, z_new);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(g.bands);
    cfg.blockDim = dim3(g.nthreads);
    cfg.dynamicSmemBytes = g.smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = g.bands;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const double* packed = g.packed.get();
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_gs_cluster, g.meta.get(), g.band_info.get(), g.req_ptr.get(),
                                       g.req.get(), g.packet_bytes.get(), g.chunk_tab.get(), packed, g.ring,
                                       g.halo, g.depth, g.max_seg, g.meta_bytes_, g.chunk_tab_bytes_,
                                       g.pbar_bytes_, z_new);
    if (e != cudaSuccess) fail(SDG_ECUDA, std::string("launch_gs_lower: ") + cudaGetErrorString(e));
    SDG_GS_CHECK();
}

void launch_restrict_warp(Context& c, const DevCsr& a, const int* pt_ptr, const int* pt_rows,
                          int n_coarse, const double* r, const double* z, double* rc,
                          const GsPlan* next) {
    ProfScope ps_(c, PF_RESTRICT,
                  12.0 * a.nnz + 4.0 * (a.n_rows + 1) + 16.0 * a.n_rows + 4.0 * a.n_rows +
                      4.0 * (n_coarse + 1) + 8.0 * n_coarse);
    if (n_coarse == 0) return;
    const int threads = 256;
    const int blocks = static_cast<int>((static_cast<int64_t>(n_coarse) * kRestrictGroup + threads - 1) / threads);
    launch_k(c, k_restrict_warp, blocks, threads, 0, 
        n_coarse, pt_ptr, pt_rows, a.rp.get(), a.ci.get(), a.v.get(), r, z, rc,
        next ? next->dinv.get() : nullptr, next ? next->bidx.get() : nullptr,
        next ? const_cast<double*>(next->packed.get()) : nullptr);
    SDG_GS_CHECK();
}

}  // namespace sdg
