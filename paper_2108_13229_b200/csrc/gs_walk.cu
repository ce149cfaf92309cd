// Single-CTA lower solve of the fast Gauss-Seidel smoother (one band; see
// gs.cuh for the prep / lower split and gs.cu for the banded cluster kernel).
//
// Rows are walked level by level (a level = rows whose lower dependencies are
// all in earlier levels).  The rows of a level are split into two classes,
// each an array of fixed-size records (16-byte vector loads with immediate
// offsets; 48 and 112 are odd multiples of 16, so a warp's loads are
// bank-conflict free):
//   K2 (<= 2 lower entries, 48 B): { double b; int rowid; int pin; double v[2]; int src[2]; int pad[2] }
//   K8 (3..8 lower entries, 112 B): { double b; int rowid; int pin; double v[8]; int src[8] }
// b = (r - U z_old)_i / d_i (written by the prep kernels), v = -a_ij / d_i, so
// z_i = b_i + sum_k v_k z_src_k.  src is a shared-memory slot: a ring indexed
// by level-order position (recent values), the zero slot (padding), or a
// pinned slot holding a value that is needed long after it left the ring;
// `pin` is where a row also stores its value (a dummy slot when nobody needs
// it late).  The ring slot of a row is its level-order position.
//
// W consumer warps each hold R2 K2 rows and R8 K8 rows per level (row slot
// r * 32W + 32 * warp + lane); a level wider than that is split into several
// consecutive pseudo-levels (its rows are independent).  Slots past the end
// of a class point at a null record (b = 0, sources = zero slot, stores to a
// dummy slot, rowid -1), so the per-row path has no branches.  With W = 1 the
// level hand-off is a __syncwarp: no CTA barrier at all.  The host plan picks
// (W, R2, R8) per system from a cost model.
//
// Consecutive levels are grouped into chunks that one TMA bulk copy brings
// into a byte ring of shared memory.  A producer thread (warp 0, lane 0)
// issues each copy once the consumers' published progress shows that the
// bytes it overwrites are dead, and publishes a `landed` count as copies
// complete; a consumer checks it only at the first level of a chunk.  The
// producer is not part of the level barrier.  Each level of a consumer warp:
// gathers + coefficient loads for all its rows, FMAs, ring stores, prefetch
// of the next level's records, level hand-off.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>

#include "gs.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace sdg {

using namespace ptx;

namespace {

#ifndef SDG_WALK_EXP
#define SDG_WALK_EXP 0  // dev knock-out experiments (scripts/mb_real2.cu); 0 in the product
#endif

#ifdef SDG_WALK_TRACE  // dev aid (scripts/mb_real2.cu): per-level clocks of lane 0 of every warp
__device__ long long g_walk_trace[1024 * 16 * 4];
#define WALK_CLK(L, k)                                          \
    if ((threadIdx.x & 31) == 0 && (L) < 1024)                  \
    g_walk_trace[((L) * 16 + (threadIdx.x >> 5)) * 4 + (k)] = clock64()
#else
#define WALK_CLK(L, k)
#endif

#ifdef SDG_WALK_TL  // dev aid: kernel timeline {start, after pdl wait, end, smid | n_levels << 16}
__device__ unsigned long long g_walk_tl[4096 * 4];
__device__ unsigned g_walk_tl_n;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

constexpr int kBars = 32;  // chunk mbarriers (chunks in flight at most)
constexpr int kK2Bytes = 48;
constexpr int kMaxK = 16;
constexpr int kPseudoBytes = 24 * 1024;  // records per pseudo-level (staging granularity)

// wide records: <= 6 entries (80 B, 16-bit sources), <= 8 (112 B, 32-bit
// sources) or <= 16 (176 B, 16-bit sources); all odd multiples of 16 bytes
__host__ __device__ constexpr int wide_bytes(int kw) { return kw == 6 ? 80 : kw == 8 ? 112 : 176; }
__host__ __device__ constexpr int wide_src_off(int kw) { return kw == 6 ? 64 : kw == 8 ? 80 : 144; }
constexpr int kMaxR2 = 6, kMaxR8 = 3;
constexpr int kChunkBytes = 16 * 1024;
constexpr int kSmemCap = 227 * 1024;
constexpr int kNullBytes = 320;  // null small record at +0, null wide record at +128

inline int pad16(int64_t b) { return static_cast<int>((b + 15) / 16 * 16); }

// threads per CTA an instantiation may use (register budget)
constexpr int max_threads(int r2, int r8, int kw) {
    const int load = r2 + (kw == 16 ? 4 : 2) * r8;
    return load <= 3 ? 512 : load <= 5 ? 384 : load <= 7 ? 256 : 128;
}

// shapes whose instantiation fits the register file without spills (ptxas -v)
constexpr bool shape_ok(int r2, int r8, int kw) {
    return kw == 16 ? (r8 <= 1 && r2 <= 4) : (r2 + 2 * r8 <= 9 && !(r8 == 3 && r2 >= 4));
}

__device__ __forceinline__ int ld_volatile(const int* p) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}

// acquire: the staged records read after observing `landed` must not be
// hoisted above it (plain shared loads may be reordered before a volatile one)
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}

__device__ __forceinline__ int ld_acquire_cluster(const int* p) {
    int v;
    asm volatile("ld.acquire.cluster.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_cluster(unsigned cluster_addr, int v) {
    asm volatile("st.release.cluster.shared::cluster.s32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_cluster(unsigned cluster_addr, int v) {
    asm volatile("st.relaxed.cluster.shared::cluster.s32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned cluster_ctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void st_volatile(int* p, int v) {
    asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
    unsigned done;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return done != 0;
}

struct WalkArgs {
    const int4* meta_g;   // per level (+2 sentinels) {K2 stage off | peer level << 18, K8 stage off | chunk-start
                          //   << 18, K2 pos | n2 << 20, K8 pos | n8 << 20}
    const int4* chunk_g;  // per chunk {global off / 16, bytes, stage off, may issue once this level is done}
    const unsigned char* packed;
    int n_levels, n_chunks, ring, meta_bytes, chunk_bytes, zbytes;
    double* z_new;
    // 0: one CTA.  In a 2-CTA pipe (two label blocks walked concurrently on a
    // cluster): 1 = the earlier block, whose small rows push the values the
    // other block needs into the peer's import slots with st.async, each
    // completing the transaction count of the peer's mbarrier for that level;
    // 2 = the later block.  The peer-level field of a level is the peer's
    // progress it needs first (role 2: the producer levels its imports come
    // from; role 1: the consumer levels that last read the import slots it is
    // about to overwrite).
    int role;
    int n_peer;               // role 2: levels of the peer (one single-use mbarrier each)
    int pbar_bytes;           // role 2: shared bytes of those mbarriers
    const int* peer_bytes_g;  // role 2: bytes the peer pushes at each of its levels
};

struct WalkPair {
    WalkArgs a[2];  // indexed by the CTA's rank in the cluster (a[0] only without a cluster)
};

// 32-bit shared-memory accesses through explicit addresses (kept in
// registers; the compiler would otherwise re-derive them from the kernel
// parameters with constant loads on the critical path)
__device__ __forceinline__ unsigned keep(unsigned x) {
    unsigned y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ int4 lds4(unsigned a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ int2 lds2(unsigned a) {
    int2 v;
    asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double ldsd(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double2 ldsd2(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void stsd(unsigned a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// A thread's rows for one level in two forms: the raw record words just
// loaded from the stage (Raw) and the ready-to-use addresses derived from
// them one level later (Rows: gather sources, ring and pin stores, global z,
// coefficients).  Splitting the two keeps the record loads' latency off the
// in-order issue stream.
template <int R2, int R8, int KW>
struct WalkRaw {
    int4 h2[R2 > 0 ? R2 : 1], h8[R8 > 0 ? R8 : 1];       // {b lo, b hi, rowid, pin}
    int4 s2[R2 > 0 ? R2 : 1];                            // small rows: {source, source, export slot, -}
    int4 s8[R8 > 0 ? R8 : 1][KW == 8 ? 2 : (KW + 7) / 8];  // sources of wide rows (32- or 16-bit)
    unsigned q2[R2 > 0 ? R2 : 1], q8[R8 > 0 ? R8 : 1];   // record addresses
    int4 m;                                              // the level's meta
};

template <int R2, int R8, int KW>
struct WalkRows {
    double b2[R2 > 0 ? R2 : 1], b8[R8 > 0 ? R8 : 1];
    unsigned s2[R2 > 0 ? R2 : 1][2], s8[R8 > 0 ? R8 : 1][KW];
    unsigned wa2[R2 > 0 ? R2 : 1], pa2[R2 > 0 ? R2 : 1], va2[R2 > 0 ? R2 : 1];
    unsigned wa8[R8 > 0 ? R8 : 1], pa8[R8 > 0 ? R8 : 1], va8[R8 > 0 ? R8 : 1];
    int rid2[R2 > 0 ? R2 : 1], rid8[R8 > 0 ? R8 : 1];
    unsigned ex2[R2 > 0 ? R2 : 1];  // shared::cluster address of the export slot in the peer (0: none)
    int sync;                       // peer progress this level needs (pipe roles)
};

// The level loop of one consumer warp (see the file comment).  Three-stage
// software pipeline per level L: solve level L (gathers -> FMAs -> ring/pin
// stores, global z), turn level L+1's raw record words into addresses, load
// level L+2's raw records; then the level hand-off.  The critical path per
// level is gathers -> FMAs -> ring store -> hand-off.
template <int R2, int R8, int KW, bool PIPE, bool ROLES>
__device__ __forceinline__ void walk_consumer(const WalkArgs& a, const int4* meta, const unsigned char* stage,
                                              const unsigned char* nullrec, double* zr, int* flags,
                                              unsigned peer_zr, unsigned peer_flag, unsigned peer_pbar,
                                              uint64_t* pbars_l) {
    const int mask = a.ring - 1, dummy = a.ring + 1;
    const int nw = (blockDim.x >> 5) - 1;  // consumer warps
    const int nbar = 32 * nw;              // threads in the level barrier
    // ROLES (WalkArgs::roles): the first half of the consumer warps walk the
    // small rows of every level (this instantiation has R8 = 0), the second
    // half the wide rows (R2 = 0)
    const int stride = ROLES ? nbar / 2 : nbar;  // row slots of one kind per pass
    const int t0 = threadIdx.x - 32 - (ROLES && R2 == 0 ? stride : 0);
    const int n_levels = a.n_levels;
    const unsigned stage_s = smem_addr(stage), null_s = smem_addr(nullrec), zr_s = smem_addr(zr);
    const unsigned dummy_s = zr_s + 8u * dummy;
    double* const z_new = a.z_new;
    int* progress = flags;
    const int* landed = flags + 1;
    const int role = PIPE ? a.role : 0;  // compile-time 0 outside pipes (no cost on the plain walk)
    // peer progress: role 1 reads flags[2] (the peer's level count, stored
    // remotely), role 2 flags[3] (peer levels whose pushes have all landed,
    // published by its own producer thread from the mbarriers)
    int peer_seen = 0;
    auto wait_peer = [&](int need) {
        if (need > peer_seen) {
            if (role == 1) {
                while ((peer_seen = ld_volatile(flags + 2)) < need) {
                }
            } else {
                for (int l = peer_seen; l < need; ++l) mbar_wait(pbars_l + l, 0);
                peer_seen = need;
            }
        }
    };
    using Raw = WalkRaw<R2, R8, KW>;
    using Rows = WalkRows<R2, R8, KW>;
    constexpr int WB = wide_bytes(KW);
    auto wait_landed = [&](const int4 m) {
        const int need = static_cast<unsigned>(m.y) >> 18;  // chunk id + 1 when the level starts a chunk
        if (need)
            while (ld_acquire(landed) < need) {
            }
    };
    auto load_raw = [&](Raw& w, const int4 m) {
        w.m = m;
#pragma unroll
        for (int r = 0; r < R2; ++r) {
            const int u = r * stride + t0;
            const unsigned q = u < (m.z >> 20) ? stage_s + (m.x & 0x3ffff) + u * kK2Bytes : null_s;
            w.q2[r] = q;
            w.h2[r] = lds4(q);
            w.s2[r] = lds4(q + 32);
        }
#pragma unroll
        for (int r = 0; r < R8; ++r) {
            const int u = r * stride + t0;
            const unsigned q = u < (m.w >> 20) ? stage_s + (m.y & 0x3ffff) + u * WB : null_s + 128;
            w.q8[r] = q;
            w.h8[r] = lds4(q);
#pragma unroll
            for (int j = 0; j < (KW == 8 ? 2 : (KW + 7) / 8); ++j)
                w.s8[r][j] = lds4(q + (KW == 8 ? 80 : wide_src_off(KW)) + 16 * j);
        }
    };
    auto unpack = [&](Rows& x, const Raw& w) {
        const int4 m = w.m;
        x.sync = static_cast<unsigned>(m.x) >> 18;
#pragma unroll
        for (int r = 0; r < R2; ++r) {
            const int u = r * stride + t0;
            const bool ok = u < (m.z >> 20);
            x.b2[r] = __hiloint2double(w.h2[r].y, w.h2[r].x);
            x.rid2[r] = w.h2[r].z;
            x.pa2[r] = zr_s + 8u * w.h2[r].w;
            x.s2[r][0] = zr_s + 8u * w.s2[r].x;
            x.s2[r][1] = zr_s + 8u * w.s2[r].y;
            x.ex2[r] = PIPE && w.s2[r].z >= 0 ? peer_zr + 8u * w.s2[r].z : 0u;
            x.va2[r] = w.q2[r] + 16;
            x.wa2[r] = zr_s + 8u * (ok ? (((m.z & 0xfffff) + u) & mask) : dummy);
        }
#pragma unroll
        for (int r = 0; r < R8; ++r) {
            const int u = r * stride + t0;
            const bool ok = u < (m.w >> 20);
            x.b8[r] = __hiloint2double(w.h8[r].y, w.h8[r].x);
            x.rid8[r] = w.h8[r].z;
            x.pa8[r] = zr_s + 8u * w.h8[r].w;
            if constexpr (KW == 8) {
                const int sv[8] = {w.s8[r][0].x, w.s8[r][0].y, w.s8[r][0].z, w.s8[r][0].w,
                                   w.s8[r][1 % 2].x, w.s8[r][1 % 2].y, w.s8[r][1 % 2].z, w.s8[r][1 % 2].w};
#pragma unroll
                for (int k = 0; k < KW; ++k) x.s8[r][k] = zr_s + 8u * sv[k % 8];
            } else {
                unsigned wd[(KW + 7) / 8 * 4];
#pragma unroll
                for (int j = 0; j < (KW + 7) / 8; ++j) {
                    wd[4 * j] = w.s8[r][j].x;
                    wd[4 * j + 1] = w.s8[r][j].y;
                    wd[4 * j + 2] = w.s8[r][j].z;
                    wd[4 * j + 3] = w.s8[r][j].w;
                }
#pragma unroll
                for (int k = 0; k < KW; ++k) x.s8[r][k] = zr_s + 8u * ((wd[k / 2] >> (16 * (k % 2))) & 0xffff);
            }
            x.va8[r] = w.q8[r] + 16;
            x.wa8[r] = zr_s + 8u * (ok ? (((m.w & 0xfffff) + u) & mask) : dummy);
        }
    };
    // solve level L (rows in x), unpack level L+1 (raw w) into y, load level L+2 into w
    auto step = [&](int L, const Rows& x, Rows& y, Raw& w) {
        WALK_CLK(L, 0);
        if (role == 2) wait_peer(x.sync);  // the imported values of this level have arrived
        double z2[R2 > 0 ? R2 : 1][2], v2[R2 > 0 ? R2 : 1][2];
        double z8[R8 > 0 ? R8 : 1][KW], v8[R8 > 0 ? R8 : 1][KW];
#pragma unroll
        for (int r = 0; r < R2; ++r) {
            z2[r][0] = ldsd(x.s2[r][0]);
            z2[r][1] = ldsd(x.s2[r][1]);
            const double2 c = ldsd2(x.va2[r]);
            v2[r][0] = c.x;
            v2[r][1] = c.y;
        }
#pragma unroll
        for (int r = 0; r < R8; ++r) {
#pragma unroll
            for (int k = 0; k < KW; ++k) z8[r][k] = ldsd(x.s8[r][k]);
#pragma unroll
            for (int k = 0; k < KW / 2; ++k) {
                const double2 c = ldsd2(x.va8[r] + 16 * k);
                v8[r][2 * k] = c.x;
                v8[r][2 * k + 1] = c.y;
            }
        }
        const int4 m2 = meta[L + 2];
        if (role == 1) wait_peer(x.sync);  // the import slots about to be overwritten have been read
#pragma unroll
        for (int r = 0; r < R2; ++r) {
            const double acc = fma(v2[r][1], z2[r][1], fma(v2[r][0], z2[r][0], x.b2[r]));
            stsd(x.wa2[r], acc);
            if (x.pa2[r] != dummy_s) stsd(x.pa2[r], acc);  // most rows are not pinned
            if (PIPE && x.ex2[r]) st_async_f64(x.ex2[r], acc, peer_pbar + 8u * L);
            if (!(SDG_WALK_EXP & 2) && x.rid2[r] >= 0) z_new[x.rid2[r]] = acc;
        }
#pragma unroll
        for (int r = 0; r < R8; ++r) {
            const double* v = v8[r];
            const double* z = z8[r];
            // pairs, then a balanced tree: (q0 + q1) + q2 for 6, ((q0+q1)+(q2+q3)) for 8, ...
            double qq[KW / 2];
            qq[0] = fma(v[1], z[1], fma(v[0], z[0], x.b8[r]));
#pragma unroll
            for (int j = 1; j < KW / 2; ++j) qq[j] = fma(v[2 * j + 1], z[2 * j + 1], v[2 * j] * z[2 * j]);
#pragma unroll
            for (int j2 = 1; j2 < KW / 2; j2 *= 2)
#pragma unroll
                for (int j = 0; j + j2 < KW / 2; j += 2 * j2) qq[j] += qq[j + j2];
            const double acc = qq[0];
            stsd(x.wa8[r], acc);
            if (x.pa8[r] != dummy_s) stsd(x.pa8[r], acc);
            if (!(SDG_WALK_EXP & 2) && x.rid8[r] >= 0) z_new[x.rid8[r]] = acc;
        }
        WALK_CLK(L, 1);
        unpack(y, w);
        if (!(SDG_WALK_EXP & 8)) {
            wait_landed(m2);
            load_raw(w, m2);
        }
        WALK_CLK(L, 2);
        if (nw == 1)
            __syncwarp();
        else
            asm volatile("bar.sync 1, %0;" ::"r"(nbar) : "memory");
        if (threadIdx.x == 32) {
            st_volatile(progress, L + 1);
            if (role == 2) st_relaxed_cluster(peer_flag, L + 1);  // back-pressure for the peer
        }
    };
    Rows x, y;
    Raw w;
    {
        const int4 m0 = meta[0], m1 = meta[1];
        wait_landed(m0);
        load_raw(w, m0);
        unpack(x, w);
        wait_landed(m1);
        load_raw(w, m1);
    }
    for (int L = 0; L < n_levels; L += 2) {
        step(L, x, y, w);
        if (L + 1 < n_levels) step(L + 1, y, x, w);
    }
}

// TMA producer (thread 0): issue chunk copies once the consumers' progress
// frees their ring space, publish each chunk once it has landed
__device__ __forceinline__ void walk_producer(const WalkArgs& a, uint64_t* bars, int* flags, const int4* ctab,
                                              unsigned char* stage, uint64_t* pbars) {
    const int nc = a.n_chunks, np = 0;  // consumers wait on the peer mbarriers themselves
    int pl = 0;  // peer levels whose pushes have landed
    // the records' b values come from the previous kernel (prep / restriction):
    // the setup above overlapped it, the copies wait for it.  Consumers touch
    // global memory only after `landed` shows copies issued after this wait.
    pdl_wait();
    int ci = 0, cw = 0;
    while (cw < nc || pl < np) {
        if (pl < np && mbar_test(&pbars[pl], 0)) {
            int q = pl + 1;
            while (q < np && mbar_test(&pbars[q], 0)) ++q;
            pl = q;
            asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(smem_addr(&flags[3])), "r"(pl) : "memory");
        }
        const int done = ld_volatile(&flags[0]) - 1;  // last completed level
        while (ci < nc && ci < cw + kBars && ctab[ci].w <= done) {
            const int4 cd = ctab[ci];
            uint64_t* bar = &bars[ci % kBars];
            mbar_expect_tx(bar, static_cast<unsigned>(cd.y));
            tma_load_1d(stage + cd.z, a.packed + static_cast<size_t>(cd.x) * 16, static_cast<unsigned>(cd.y), bar);
            ++ci;
        }
        if (cw < ci && mbar_test(&bars[cw % kBars], static_cast<unsigned>(cw / kBars) & 1u)) {
            ++cw;
            asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(smem_addr(&flags[1])), "r"(cw) : "memory");
        } else if (pl >= np) {
            __nanosleep(20);
        }
    }
}

template <int R2, int R8, int KW, bool PIPE, bool ROLES = false>
__global__ void __launch_bounds__(max_threads(R2, R8, KW), 1) k_gs_walk(WalkPair pair) {
    const unsigned rank = PIPE ? cluster_ctarank() : 0u;
    const WalkArgs a = rank ? pair.a[1] : pair.a[0];  // a copy: no dynamically indexed parameter loads
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
    // {levels done, chunks landed, peer levels done (role 1), peer levels landed (role 2)}
    int* flags = reinterpret_cast<int*>(sm + kBars * 8);
    unsigned char* nullrec = sm + kBars * 8 + 16;
    int4* meta = reinterpret_cast<int4*>(nullrec + kNullBytes);
    int4* ctab = reinterpret_cast<int4*>(reinterpret_cast<unsigned char*>(meta) + a.meta_bytes);
    uint64_t* pbars = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(ctab) + a.chunk_bytes);
    double* zr = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(pbars) + a.pbar_bytes);
    unsigned char* stage = reinterpret_cast<unsigned char*>(zr) + a.zbytes;
    const int tid = threadIdx.x;
    const int nl = a.n_levels, nc = a.n_chunks;
    const int zero_slot = a.ring, dummy = a.ring + 1;
#ifdef SDG_WALK_TL
    __shared__ unsigned tl_slot;
    if (tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        tl_slot = atomicAdd(&g_walk_tl_n, 1u) % 4096u;
        g_walk_tl[tl_slot * 4 + 0] = gtimer();
        g_walk_tl[tl_slot * 4 + 3] = smid | (static_cast<unsigned long long>(nl) << 16);
    }
#endif

    for (int l = tid; l <= nl + 1; l += blockDim.x) meta[l] = a.meta_g[l];
    for (int c = tid; c < nc; c += blockDim.x) ctab[c] = a.chunk_g[c];
    if (tid < kBars) mbar_init(&bars[tid], 1);
    if (PIPE && a.role == 2)
        for (int l = tid; l < a.n_peer; l += blockDim.x) {
            mbar_init(&pbars[l], 1);
            mbar_expect_tx(&pbars[l], static_cast<unsigned>(a.peer_bytes_g[l]));
        }
    if (tid < 2) {  // null records: b = 0, v = 0, sources = zero slot, stores to the dummy slot
        int* nr = reinterpret_cast<int*>(nullrec + 128 * tid);
        for (int k = 0; k < (tid ? wide_bytes(KW) : 48) / 4; ++k) nr[k] = 0;
        nr[2] = -1;     // rowid
        nr[3] = dummy;  // pin
        if (tid == 0) {
            nr[8] = nr[9] = zero_slot;
            nr[10] = -1;  // no export
        } else if (KW == 8) {
            for (int k = 0; k < 8; ++k) nr[20 + k] = zero_slot;
        } else {
            for (int k = 0; k < KW / 2; ++k) nr[wide_src_off(KW) / 4 + k] = zero_slot | (zero_slot << 16);
        }
    }
    if (tid == 0) {
        zr[zero_slot] = 0.0;
        flags[0] = 0;
        flags[1] = 0;
        flags[2] = 0;
        flags[3] = 0;
    }
    fence_mbar_init();
    if (PIPE)
        asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
    else
        __syncthreads();
    pdl_trigger();  // the next kernel may launch (it waits for this grid itself)

    if (tid >= 32) {
        // the peer CTA's mbarriers, z slots and progress word (in its own layout)
        unsigned peer_zr = 0, peer_flag = 0, peer_pbar = 0;
        if (PIPE) {
            const WalkArgs& pa = rank ? pair.a[0] : pair.a[1];
            const unsigned char* pb = sm + kBars * 8 + 16 + kNullBytes + pa.meta_bytes + pa.chunk_bytes;
            peer_pbar = cluster_addr(pb, rank ^ 1u);
            peer_zr = cluster_addr(pb + pa.pbar_bytes, rank ^ 1u);
            peer_flag = cluster_addr(flags + 2, rank ^ 1u);
        }
        if constexpr (ROLES) {
            if (tid - 32 < (static_cast<int>(blockDim.x) - 32) / 2)
                walk_consumer<R2, 0, KW, false, true>(a, meta, stage, nullrec, zr, flags, 0u, 0u, 0u, pbars);
            else
                walk_consumer<0, R8, KW, false, true>(a, meta, stage, nullrec, zr, flags, 0u, 0u, 0u, pbars);
        } else {
            walk_consumer<R2, R8, KW, PIPE, false>(a, meta, stage, nullrec, zr, flags, peer_zr, peer_flag, peer_pbar,
                                                   pbars);
        }
#ifdef SDG_WALK_TL
        if (tid == 32) g_walk_tl[tl_slot * 4 + 2] = gtimer();
#endif
    } else if (tid == 0) {
#ifdef SDG_WALK_TL
        pdl_wait();
        g_walk_tl[tl_slot * 4 + 1] = gtimer();
#endif
        walk_producer(a, bars, flags, ctab, stage, pbars);
    }
    // no CTA of a pipe leaves while its peer may still store into it
    if (PIPE) asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
}

using WalkKernel = void (*)(WalkPair);

constexpr int kw_of(int i) { return i == 0 ? 6 : i == 1 ? 8 : 16; }

template <int I>
constexpr WalkKernel kernel_at() {
    return &k_gs_walk<I / (3 * (kMaxR8 + 1)) + 1, (I / 3) % (kMaxR8 + 1), kw_of(I % 3), false>;
}

// 2-CTA pipe instantiations: R2 <= 2, R8 <= 2
template <int I>
constexpr WalkKernel pipe_kernel_at() {
    return &k_gs_walk<I / 9 + 1, (I / 3) % 3, kw_of(I % 3), true>;
}

// all instantiations, indexed [R2 - 1][R8][wide width 6 / 8 / 16]
template <int... I>
constexpr auto make_table(std::integer_sequence<int, I...>) {
    struct T {
        WalkKernel k[sizeof...(I)];
    };
    return T{{kernel_at<I>()...}};
}

template <int... I>
constexpr auto make_pipe_table(std::integer_sequence<int, I...>) {
    struct T {
        WalkKernel k[sizeof...(I)];
    };
    return T{{pipe_kernel_at<I>()...}};
}

// roles instantiations: R2 <= 2, 1 <= R8 <= 2, wide width 6 / 8
template <int I>
constexpr WalkKernel roles_kernel_at() {
    return &k_gs_walk<I / 4 + 1, (I / 2) % 2 + 1, I % 2 ? 8 : 6, false, true>;
}

template <int... I>
constexpr auto make_roles_table(std::integer_sequence<int, I...>) {
    struct T {
        WalkKernel k[sizeof...(I)];
    };
    return T{{roles_kernel_at<I>()...}};
}

bool has_roles_kernel(int r2, int r8, int kw) { return r2 >= 1 && r2 <= 2 && r8 >= 1 && r8 <= 2 && kw != 16; }

WalkKernel walk_kernel(int r2, int r8, int kw, bool pipe = false, bool roles = false) {
    const int kwi = kw == 6 ? 0 : kw == 8 ? 1 : 2;
    if (roles) {
        static const auto rtable = make_roles_table(std::make_integer_sequence<int, 8>{});
        if (!has_roles_kernel(r2, r8, kw)) fail(SDG_EINVAL, "gs walk: no roles instantiation for this shape");
        return rtable.k[((r2 - 1) * 2 + (r8 - 1)) * 2 + (kw == 8 ? 1 : 0)];
    }
    if (pipe) {
        static const auto ptable = make_pipe_table(std::make_integer_sequence<int, 2 * 3 * 3>{});
        if (r2 < 1 || r2 > 2 || r8 > 2) fail(SDG_EINVAL, "gs pipe: no instantiation for this shape");
        return ptable.k[((r2 - 1) * 3 + r8) * 3 + kwi];
    }
    static const auto table = make_table(std::make_integer_sequence<int, kMaxR2 * (kMaxR8 + 1) * 3>{});
    return table.k[((r2 - 1) * (kMaxR8 + 1) + r8) * 3 + kwi];
}

}  // namespace

// Returns false when the system does not fit the walk (rows with more than 8
// lower entries, a level too large for the staging ring); the caller then
// builds the banded plan.
// (W, R2, R8) from a cost model in cycles per pseudo-level, fitted to B200
// measurements (scripts/mb_real2.cu): a latency chain that grows slowly with
// the warps and rows per thread, or the shared-memory traffic (records staged
// and read back, gathers) when that is larger.  Returns the modelled cycles
// of one sweep (1e300 when no shape fits).
//
// `corrected` is the form used to compare plans (GsPlan::build, level
// merging): refitted on the c2 launch lists of merged and unmerged walks,
// where 16-entry records cost ~400 cycles more per level than the chain term
// and staging-heavy levels ~1.8x the traffic term.
double walk_shape_cost(const std::vector<int>& c2, const std::vector<int>& c8, int kw, int* w_out, int* r2_out,
                       int* r8_out, bool corrected) {
    const int nlv = static_cast<int>(c2.size());
    const int WB = wide_bytes(kw);
    int best_w = 0, best_r2 = 0, best_r8 = 0;
    double best_cost = 1e300;
    for (int w : {1, 2, 3, 4, 5, 6, 8, 11, 15})
        for (int r2 = 1; r2 <= kMaxR2; ++r2)
            for (int r8 = 0; r8 <= kMaxR8; ++r8) {
                if (32 + 32 * w > max_threads(r2, r8, kw) || !shape_ok(r2, r8, kw)) continue;
                const int cap2 = 32 * w * r2, cap8 = 32 * w * r8;
                const double chain = 220.0 + 15.0 * w + 35.0 * (r2 - 1) + 60.0 * r8 +
                                     (corrected && kw == 16 && r8 ? 400.0 : 0.0);
                const double bw_scale = corrected ? 1.8 : 1.0;
                double cost = 0;
                bool ok = true;
                for (int q = 0; q < nlv && ok; ++q) {
                    if (c8[q] > 0 && r8 == 0) ok = false;
                    const int p = std::max({1, (c2[q] + cap2 - 1) / cap2, r8 ? (c8[q] + cap8 - 1) / cap8 : 1,
                                            (c2[q] * kK2Bytes + c8[q] * WB + kPseudoBytes - 1) / kPseudoBytes});
                    const double bw = (2.0 * (c2[q] * kK2Bytes + c8[q] * WB) + 40.0 * c2[q] + 100.0 * c8[q]) /
                                      (128.0 * p);
                    cost += p * std::max(chain, bw_scale * bw);
                }
                if (ok && cost < best_cost) {
                    best_cost = cost;
                    best_w = w;
                    best_r2 = r2;
                    best_r8 = r8;
                }
            }
    if (w_out) *w_out = best_w;
    if (r2_out) *r2_out = best_r2;
    if (r8_out) *r8_out = best_r8;
    return best_cost;
}

double walk_model_cost(const HostCsr& a, const std::vector<int>& nlow, int max_k) {
    if (max_k > kMaxK) return 1e300;
    const int n = a.n_rows;
    std::vector<int> lev(n, 0);
    int nlv = 0;
    for (int i = 0; i < n; ++i) {
        int d = 0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] < i) d = std::max(d, lev[a.ci[k]] + 1);
        lev[i] = d;
        nlv = std::max(nlv, d + 1);
    }
    std::vector<int> c2(nlv, 0), c8(nlv, 0);
    for (int i = 0; i < n; ++i) ++(nlow[i] <= 2 ? c2 : c8)[lev[i]];
    const int kw = max_k <= 6 ? 6 : max_k <= 8 ? 8 : 16;
    return walk_shape_cost(c2, c8, kw, nullptr, nullptr, nullptr, true);
}

bool GsPlan::build_walk(const HostCsr& a, const std::vector<double>& dinv_h, const std::vector<int>& nlow,
                        int max_k, cudaStream_t s, Link* link) {
    auto reject = [&](const char* why) {
        if (std::getenv("SDG_DEBUG")) std::fprintf(stderr, "[sdg gs walk] n=%d: not used (%s)\n", a.n_rows, why);
        return false;
    };
    if (max_k > kMaxK) return reject("a row has more than 16 lower entries");
    n = a.n_rows;
    if (n >= (1 << 20)) return reject("too many rows for the meta packing");
    std::vector<int> lev(n, 0);
    int nlv = 0;
    for (int i = 0; i < n; ++i) {
        int d = 0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] < i) d = std::max(d, lev[a.ci[k]] + 1);
        lev[i] = d;
        nlv = std::max(nlv, d + 1);
    }
    std::vector<int> c2(nlv, 0), c8(nlv, 0);
    for (int i = 0; i < n; ++i) ++(nlow[i] <= 2 ? c2 : c8)[lev[i]];
    // wide rows: the narrowest record that holds every row (see wide_bytes)
    const int kw = link && link->force_kw ? link->force_kw : max_k <= 6 ? 6 : max_k <= 8 ? 8 : 16;
    if (max_k > kw) return reject("forced record width too small");
    const int WB = wide_bytes(kw);

    // (W, R2, R8) from the cost model (walk_shape_cost)
    int best_w = 0, best_r2 = 0, best_r8 = 0;
    const double best_cost = walk_shape_cost(c2, c8, kw, &best_w, &best_r2, &best_r8, false);
    if (const char* e = std::getenv("SDG_WALK_SHAPE")) {  // dev override "warps,r2,r8[,rows]" (rows: only that n)
        int w = 0, r2 = 0, r8 = 0, only_n = 0;
        const int got = std::sscanf(e, "%d,%d,%d,%d", &w, &r2, &r8, &only_n);
        if (got == 4 && only_n != n) w = 0;
        if (got >= 3 && w >= 1 && r2 >= 1 && r2 <= kMaxR2 && r8 >= 0 &&
            r8 <= kMaxR8) {
            bool ok = 32 + 32 * w <= max_threads(r2, r8, kw) && shape_ok(r2, r8, kw);
            for (int q = 0; q < nlv; ++q) ok = ok && (r8 > 0 || c8[q] == 0);
            if (ok) {
                best_w = w;
                best_r2 = r2;
                best_r8 = r8;
            }
        }
    }
    if (link && link->force_w) {
        const int w = link->force_w, r2 = link->force_r2, r8 = link->force_r8;
        bool ok = 32 + 32 * w <= max_threads(r2, r8, kw) && shape_ok(r2, r8, kw);
        for (int q = 0; q < nlv; ++q) ok = ok && (r8 > 0 || c8[q] == 0);
        if (!ok) return reject("forced shape does not fit");
        best_w = w;
        best_r2 = r2;
        best_r8 = r8;
    }
    if (best_w == 0) return reject("no (warps, rows per thread) shape fits");
    const int cap2 = 32 * best_w * best_r2, cap8 = 32 * best_w * best_r8;

    // pseudo-levels: a level wider than one pass of the block, or with more
    // record bytes than kPseudoBytes, is split evenly (its rows are independent)
    std::vector<int> plv_of(n);   // pseudo-level of each row
    std::vector<int> n2, n8;      // per pseudo-level
    {
        std::vector<int> first_plv(nlv), parts(nlv);
        for (int q = 0; q < nlv; ++q) {
            const int p = std::max({1, (c2[q] + cap2 - 1) / cap2, best_r8 ? (c8[q] + cap8 - 1) / cap8 : 1,
                                    (c2[q] * kK2Bytes + c8[q] * WB + kPseudoBytes - 1) / kPseudoBytes});
            first_plv[q] = static_cast<int>(n2.size());
            parts[q] = p;
            for (int k = 0; k < p; ++k) {
                n2.push_back(0);
                n8.push_back(0);
            }
        }
        std::vector<int> seen2(nlv, 0), seen8(nlv, 0);
        for (int i = 0; i < n; ++i) {
            const int q = lev[i];
            const int pl = nlow[i] <= 2
                               ? first_plv[q] + static_cast<int>(static_cast<int64_t>(seen2[q]++) * parts[q] / c2[q])
                               : first_plv[q] + static_cast<int>(static_cast<int64_t>(seen8[q]++) * parts[q] / c8[q]);
            plv_of[i] = pl;
            ++(nlow[i] <= 2 ? n2 : n8)[pl];
        }
    }
    const int nl = static_cast<int>(n2.size());
    if (nl >= (1 << 13)) return reject("too many levels for the meta packing");
    std::vector<int> lptr(nl + 1, 0), fill2(nl), fill8(nl), order(n), pos(n);
    for (int q = 0; q < nl; ++q) lptr[q + 1] = lptr[q] + n2[q] + n8[q];
    for (int q = 0; q < nl; ++q) {
        fill2[q] = lptr[q];
        fill8[q] = lptr[q] + n2[q];
    }
    for (int i = 0; i < n; ++i) {
        const int p = (nlow[i] <= 2 ? fill2 : fill8)[plv_of[i]]++;
        order[p] = i;
        pos[i] = p;
    }
    int max_rows = 1;
    std::vector<int> lbytes(nl);
    std::vector<int64_t> goff(nl);
    int64_t off = 0;
    for (int q = 0; q < nl; ++q) {
        max_rows = std::max(max_rows, n2[q] + n8[q]);
        lbytes[q] = n2[q] * kK2Bytes + n8[q] * WB;
        goff[q] = off;
        off += lbytes[q];
    }
    if (off / 16 >= (static_cast<int64_t>(1) << 31)) return reject("packed buffer too large");

    // chunks of consecutive levels
    std::vector<int> cfirst, cbytes;
    std::vector<int> chunk_of(nl), in_chunk(nl);
    for (int q = 0; q < nl; ++q) {
        if (cfirst.empty() || cbytes.back() + lbytes[q] > kChunkBytes) {
            cfirst.push_back(q);
            cbytes.push_back(0);
        }
        chunk_of[q] = static_cast<int>(cfirst.size()) - 1;
        in_chunk[q] = cbytes.back();
        cbytes.back() += lbytes[q];
    }
    const int nc = static_cast<int>(cfirst.size());
    int max_chunk = 16;
    for (int c = 0; c < nc; ++c) max_chunk = std::max(max_chunk, cbytes[c]);

    // ring: every dependency distance (in level-order positions) when it fits,
    // else smaller with the older dependencies going through pinned slots
    int max_dist = 1;
    for (int q = 0; q < nl; ++q)
        for (int p = lptr[q]; p < lptr[q + 1]; ++p) {
            const int i = order[p];
            for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
                if (a.ci[k] < i) max_dist = std::max(max_dist, lptr[q + 1] - pos[a.ci[k]]);
        }
    int dev = 0, optin = 0;
    SDG_CUDA(cudaGetDevice(&dev));
    SDG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const int budget = std::min(kSmemCap, optin - 1024);
    const int meta_bytes = pad16(static_cast<int64_t>(nl + 2) * 16);
    const int chunk_bytes = pad16(static_cast<int64_t>(nc) * 16);
    const int pbar_bytes = link && link->peer_bytes ? pad16(static_cast<int64_t>(link->peer_bytes->size()) * 8) : 0;
    const int min_stage = 3 * max_chunk;
    ring = 64;
    while (ring < max_dist && ring < 8192) ring <<= 1;
    std::vector<int> pin_of;
    int npin = 0, zbytes = 0, fixed = 0, R = 0;
    for (;;) {
        pin_of.assign(n, -1);
        npin = 0;
        for (int q = 0; q < nl; ++q)
            for (int p = lptr[q]; p < lptr[q + 1]; ++p) {
                const int i = order[p];
                for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
                    const int j = a.ci[k];
                    if (j < i && lptr[q + 1] - pos[j] > ring && pin_of[j] < 0) pin_of[j] = npin++;
                }
            }
        zbytes = pad16(static_cast<int64_t>(ring + 2 + npin + (link ? link->import_slots : 0)) * 8);
        fixed = kBars * 8 + 16 + kNullBytes + meta_bytes + chunk_bytes + pbar_bytes + zbytes;
        R = (budget - fixed) / 16 * 16;
        if (R >= min_stage) break;
        if (ring <= 64 || ring / 2 < 2 * max_rows) return reject("shared memory: ring + pinned values + staging");
        ring >>= 1;
    }
    const int zero_slot = ring, dummy_slot = ring + 1, pin_base = ring + 2, import_base = pin_base + npin;
    const int nslots = import_base + (link ? link->import_slots : 0);
    if (kw != 8 && nslots >= 65536) return reject("too many shared slots for 16-bit sources");

    // staging ring placement and issue points of the chunks
    std::vector<int> roff(nc), after(nc);
    int cur = 0;
    for (int c = 0; c < nc; ++c) {
        const int sz = cbytes[c];
        if (cur + sz > R) cur = 0;
        roff[c] = cur;
        int aft = c > 0 ? after[c - 1] : -1;
        int64_t scanned = 0;
        for (int x = c - 1; x >= 0 && scanned <= 2LL * R; --x) {
            scanned += cbytes[x];
            if (roff[x] < cur + sz && cur < roff[x] + cbytes[x]) {
                const int last = x + 1 < nc ? cfirst[x + 1] - 1 : nl - 1;
                aft = std::max(aft, last);
                break;
            }
        }
        if (aft >= 0 && aft > cfirst[c] - 4) return reject("staging ring too small for the look-ahead");
        after[c] = aft;
        cur += sz;
    }

    std::vector<double> pk(static_cast<size_t>(off / 8 + 2), 0.0);
    unsigned char* base = reinterpret_cast<unsigned char*>(pk.data());
    std::vector<int> bidx_h(n);
    std::vector<int> sync_of(nl, 0);  // peer progress a level needs (pipe roles)
    if (link && link->export_need)
        for (int q = 0; q < nl; ++q) sync_of[q] = (*link->export_need)[q];
    std::vector<int4> meta_h(nl + 2), ctab_h(nc);
    lower_entries = 0;
    global_refs = 0;
    cross_refs = npin;
    for (int q = 0; q < nl; ++q) {
        unsigned char* seg = base + goff[q];
        for (int p = lptr[q]; p < lptr[q + 1]; ++p) {
            const int t = p - lptr[q];
            const int i = order[p];
            const bool k2 = t < n2[q];
            unsigned char* rec = k2 ? seg + static_cast<size_t>(t) * kK2Bytes
                                    : seg + static_cast<size_t>(n2[q]) * kK2Bytes +
                                          static_cast<size_t>(t - n2[q]) * WB;
            double* recd = reinterpret_cast<double*>(rec);
            int* reci = reinterpret_cast<int*>(rec);
            bidx_h[i] = static_cast<int>((rec - base) / 8);
            reci[2] = i;
            reci[3] = pin_of[i] >= 0 ? pin_base + pin_of[i] : dummy_slot;
            const int exp = link && link->export_slot && (*link->export_slot)[i] >= 0
                                ? link->export_base + (*link->export_slot)[i]
                                : -1;
            if (k2)
                reci[10] = exp;
            else if (exp >= 0)
                return reject("a wide row exports to the peer");
            const int cap = k2 ? 2 : kw;
            double* val = recd + 2;
            int* src = reci + (k2 ? 8 : 20);
            uint16_t* src16 = reinterpret_cast<uint16_t*>(rec + wide_src_off(kw));
            const bool narrow_src = !k2 && kw != 8;
            int m = 0;
            for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
                const int j = a.ci[k];
                if (j >= i) continue;
                val[m] = -(a.v[k] * dinv_h[i]);
                const int slot = lptr[q + 1] - pos[j] <= ring ? (pos[j] & (ring - 1)) : pin_base + pin_of[j];
                if (narrow_src)
                    src16[m] = static_cast<uint16_t>(slot);
                else
                    src[m] = slot;
                ++m;
                ++lower_entries;
            }
            if (link && link->ext) {  // lower entries to the peer block: its values arrive in import slots
                const HostCsr& x = *link->ext;
                for (int k = x.rp[i]; k < x.rp[i + 1]; ++k) {
                    const int j = x.ci[k];
                    val[m] = -(x.v[k] * dinv_h[i]);
                    const int slot = import_base + (*link->ext_slot)[j];
                    if (narrow_src)
                        src16[m] = static_cast<uint16_t>(slot);
                    else
                        src[m] = slot;
                    ++m;
                    ++lower_entries;
                    sync_of[q] = std::max(sync_of[q], (*link->ext_plv)[j] + 1);
                }
            }
            for (; m < cap; ++m) {
                val[m] = 0.0;
                if (narrow_src)
                    src16[m] = static_cast<uint16_t>(zero_slot);
                else
                    src[m] = zero_slot;
            }
        }
        const int starts = cfirst[chunk_of[q]] == q ? chunk_of[q] + 1 : 0;  // chunk id + 1 if q starts a chunk
        const int o2 = roff[chunk_of[q]] + in_chunk[q], o8 = o2 + n2[q] * kK2Bytes;
        if (sync_of[q] >= (1 << 14)) return reject("peer level out of the meta packing");
        meta_h[q] = make_int4(o2 | (sync_of[q] << 18), o8 | (starts << 18), lptr[q] | (n2[q] << 20),
                              (lptr[q] + n2[q]) | (n8[q] << 20));
    }
    meta_h[nl] = meta_h[nl + 1] = make_int4(0, 0, 0, 0);  // sentinels: prefetches past the end read null rows
    for (int c = 0; c < nc; ++c)
        ctab_h[c] = make_int4(static_cast<int>(goff[cfirst[c]] / 16), cbytes[c], roff[c], after[c]);

    walk_import_base = import_base;
    walk_pbar_bytes = pbar_bytes;
    walk_n_peer = 0;
    if (link && link->peer_bytes) {
        walk_n_peer = static_cast<int>(link->peer_bytes->size());
        walk_peer_bytes.upload(*link->peer_bytes, s);
    }
    if (link) {
        if (link->plv_out) *link->plv_out = plv_of;
        link->shape[0] = best_w;
        link->shape[1] = best_r2;
        link->shape[2] = best_r8;
        link->shape[3] = kw;
        walk_role = link->role;
    }
    walk = true;
    usable = true;
    bands = 1;
    n_levels = nl;
    max_band_levels = nl;
    // roles (k_gs_walk<..., ROLES>): twice the consumer warps, each taking one
    // kind of row, so a warp issues one row path per level instead of both.
    // Measured on every c2 walk (ncu, one td_bgs apply): V0 98.4 -> 93.2 us,
    // V1 44.7 -> 41.4, porous D0 52.6 -> 48.7, the rest unchanged; apply 380 ->
    // 363 us.  Bitwise the same sweep.  SDG_WALK_ROLES=0 disables.
    const char* re = std::getenv("SDG_WALK_ROLES");
    walk_roles = !(re && re[0] == '0') && !link && has_roles_kernel(best_r2, best_r8, kw) &&
                 32 + 64 * best_w <= max_threads(best_r2, best_r8, kw);
    nthreads = 32 + 32 * best_w * (walk_roles ? 2 : 1);
    walk_r2 = best_r2;
    walk_r8 = best_r8;
    walk_kw = kw;
    walk_meta_bytes = meta_bytes;
    walk_chunk_bytes = chunk_bytes;
    walk_zbytes = zbytes;
    walk_chunks = nc;
    max_seg = max_chunk;
    halo = npin;
    smem = static_cast<size_t>(fixed) + R;
    if (std::getenv("SDG_DEBUG"))
        std::fprintf(stderr,
                     "[sdg gs walk] n=%d levels=%d pseudo-levels=%d warps=%d%s rows/thread=%d+%d wide=%d chunks=%d "
                     "ring=%d pinned=%d stage=%d smem=%zu packed=%.1fKB model=%.0f cycles\n",
                     n, nlv, nl, best_w, walk_roles ? "x2 (roles)" : "", best_r2, best_r8, kw, nc, ring, npin, R,
                     smem, off / 1024.0, best_cost);
    meta.upload(meta_h, s);
    walk_iss.upload(ctab_h, s);
    packed.upload(pk, s);
    bidx.upload(bidx_h, s);
    SDG_CUDA(cudaFuncSetAttribute(walk_kernel(best_r2, best_r8, kw, false, walk_roles != 0),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
    if (link && link->role && best_r2 <= 2 && best_r8 <= 2)
        SDG_CUDA(cudaFuncSetAttribute(walk_kernel(best_r2, best_r8, kw, true),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
    SDG_CUDA(cudaStreamSynchronize(s));  // host staging vectors die here
    return true;
}

namespace {
WalkArgs walk_args(const GsPlan& g, double* z_new) {
    return WalkArgs{g.meta.get(), g.walk_iss.get(), reinterpret_cast<const unsigned char*>(g.records()),
                    g.n_levels, g.walk_chunks, g.ring, g.walk_meta_bytes, g.walk_chunk_bytes, g.walk_zbytes,
                    z_new, g.walk_role, g.walk_n_peer, g.walk_pbar_bytes, g.walk_peer_bytes.get()};
}
}  // namespace

#ifdef SDG_WALK_TL
int walk_timeline(unsigned long long* out, int max) {
    unsigned n = 0;
    cudaMemcpyFromSymbol(&n, g_walk_tl_n, sizeof(n));
    const int m = std::min<int>(std::min<unsigned>(n, 4096u), max);
    cudaMemcpyFromSymbol(out, g_walk_tl, sizeof(unsigned long long) * 4 * m);
    unsigned z = 0;
    cudaMemcpyToSymbol(g_walk_tl_n, &z, sizeof(z));
    return m;
}
#else
int walk_timeline(unsigned long long*, int) { return 0; }
#endif

void launch_gs_walk(Context& c, const GsPlan& g, double* z_new) {
    WalkPair pair{};
    pair.a[0] = walk_args(g, z_new);
    launch_k(c, walk_kernel(g.walk_r2, g.walk_r8, g.walk_kw, false, g.walk_roles != 0), 1, g.nthreads, g.smem, pair);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(SDG_ECUDA, std::string("launch_gs_walk: ") + cudaGetErrorString(e));
    c.count();
}

void launch_gs_pipe(Context& c, const GsPlan& g, double* z_new) {
    const GsPlan& p0 = *g.parts[0];
    const GsPlan& p1 = *g.parts[1];
    WalkPair pair{};
    pair.a[0] = walk_args(p0, z_new + g.part_r0[0]);
    pair.a[1] = walk_args(p1, z_new + g.part_r0[1]);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(p0.nthreads);
    cfg.dynamicSmemBytes = std::max(p0.smem, p1.smem);
    cfg.stream = c.stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = c.pdl ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, walk_kernel(p0.walk_r2, p0.walk_r8, p0.walk_kw, true), pair);
    if (e != cudaSuccess) fail(SDG_ECUDA, std::string("launch_gs_pipe: ") + cudaGetErrorString(e));
    c.count();
}

}  // namespace sdg
