// Single-CTA lower solve of the fast Gauss-Seidel smoother (one band; see
// gs.cuh for the prep / lower split and gs.cu for the banded cluster kernel).
//
// The rows of each dependency level are split into two classes, each an array
// of fixed-size records (16-byte vector loads with immediate offsets; 48 and
// 112 are odd multiples of 16, so a warp's loads are bank-conflict free):
//   K2 (<= 2 lower entries, 48 B): { double b; int rowid; int pin; double v[2]; int src[2]; int pad[2] }
//   K8 (3..8 lower entries, 112 B): { double b; int rowid; int pin; double v[8]; int src[8] }
// b = (r - U z_old)_i / d_i (written by the prep kernels), v = -a_ij / d_i, so
// z_i = b_i + sum_k v_k z_src_k.  src is a shared-memory slot: a ring indexed
// by level-order position (recent values), the zero slot (padding), or a
// pinned slot holding a value that is needed long after it left the ring;
// `pin` is where a row also stores its value (a dummy slot when nobody needs
// it late).  The ring slot of a row is its level-order position.
//
// Warps own one class for a whole level (the first ceil(n2/32) consumer warps
// take K2 rows, the next ceil(n8/32) K8 rows); lanes past the end of their
// class point at a null record in shared memory (b = 0, sources = zero slot,
// stores to a dummy slot, rowid -1), so the per-row path has no branches.
// Consecutive levels are grouped into chunks that one TMA bulk copy (issued by
// thread 0) brings into a byte ring of shared memory; the host plan places
// every chunk and names the level after whose barrier it may overwrite older
// bytes.  Thread 0 also waits for the chunk of the level two ahead before
// joining the level barrier, so consumers never touch mbarriers.  Consumers
// hold the next level's row in registers (ping-pong between two register
// sets), and the per-level critical path is
//   barrier -> shared gathers -> two FMAs -> shared store -> barrier.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "gs.cuh"
#include "ptx.cuh"

namespace sdg {

using namespace ptx;

namespace {

#ifdef SDG_WALK_TRACE  // dev aid (scripts/mb_real2.cu): per-level clocks of lane 0 of every warp
__device__ long long g_walk_trace[1024 * 16 * 4];
#define WALK_CLK(L, k)                                          \
    if ((threadIdx.x & 31) == 0 && (L) < 1024)                  \
    g_walk_trace[((L) * 16 + (threadIdx.x >> 5)) * 4 + (k)] = clock64()
#else
#define WALK_CLK(L, k)
#endif

constexpr int kBars = 32;      // chunk mbarriers (chunks in flight at most)
constexpr int kK2Bytes = 48;
constexpr int kK8Bytes = 112;
constexpr int kMaxK = 8;
constexpr int kMaxWarps = 15;  // consumer warps (512 threads with the producer warp)
constexpr int kChunkBytes = 16 * 1024;
constexpr int kSmemCap = 227 * 1024;
constexpr int kNullBytes = 256;  // null K2 record at +0, null K8 record at +128

inline int pad16(int64_t b) { return static_cast<int>((b + 15) / 16 * 16); }

struct WalkArgs {
    const int4* meta_g;    // per level (+1 sentinel) {stage off, n2, n8, pos base}
    const int4* chunk_g;   // per chunk {global off / 16, bytes, stage off, may issue after the barrier of this level}
    const int* cfirst_g;   // per chunk: its first level
    const unsigned char* packed;
    int n_levels, n_chunks, ring, meta_bytes, chunk_bytes, cfirst_bytes, zbytes;
    int w2;                // consumer warps that own K2 rows (the rest own K8 rows)
    double* z_new;
};

__device__ __forceinline__ int ld_volatile(const int* p) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
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

// The level loop of one consumer warp.  Every warp owns one class for the
// whole sweep (thread t of the class: t-th row of that class at every level),
// so the loop has no class branches.  Per level: the gathers, coefficient and
// next-level meta loads are issued together, the row is finished and stored,
// and the next level's record is requested before the barrier (it lands while
// the barrier completes).  The level barrier is a named barrier of the
// consumer warps only; a level that starts a chunk first checks the
// producer's `landed` counter.
template <bool K2>
__device__ __forceinline__ void walk_consumer(const WalkArgs& a, const int4* meta, const unsigned char* stage,
                                              const unsigned char* nullrec, double* zr, int* flags, int t) {
    const int mask = a.ring - 1, dummy = a.ring + 1;
    const unsigned ncons = blockDim.x - 32;
    constexpr int K = K2 ? 2 : kMaxK;
    constexpr int RB = K2 ? kK2Bytes : kK8Bytes;
    double b;
    int s[K], rowid, pin, wpos;
    const unsigned char* vrec;
    // meta = {K2 stage offset, K8 stage offset | chunk-start << 18, K2 pos | n2 << 20, K8 pos | n8 << 20}
    const unsigned char* nrec = nullrec + (K2 ? 0 : 128);
    const int toff = t * RB;
    auto fetch = [&](const int4 m) {
        const int off = K2 ? m.x : (m.y & 0x3ffff);
        const int pn = K2 ? m.z : m.w;
        const bool ok = t < (pn >> 20);
        const unsigned char* q = ok ? stage + off + toff : nrec;
        const int4 h = *reinterpret_cast<const int4*>(q);
        if (K2) {
            const int2 ss = *reinterpret_cast<const int2*>(q + 32);
            s[0] = ss.x;
            s[1] = ss.y;
        } else {
            const int4 s0 = *reinterpret_cast<const int4*>(q + 80);
            const int4 s1 = *reinterpret_cast<const int4*>(q + 96);
            s[0] = s0.x; s[1] = s0.y; s[2 % K] = s0.z; s[3 % K] = s0.w;
            s[4 % K] = s1.x; s[5 % K] = s1.y; s[6 % K] = s1.z; s[7 % K] = s1.w;
        }
        b = __hiloint2double(h.y, h.x);
        rowid = h.z;
        pin = h.w;
        vrec = q + 16;
        wpos = ok ? (((pn & 0xfffff) + t) & mask) : dummy;
    };
    int* progress = flags;
    const int* landed = flags + 1;
    {
        const int4 m0 = meta[0];
        const int need = static_cast<unsigned>(m0.y) >> 18;
        while (ld_volatile(landed) < need) {
        }
        fetch(m0);
    }
    for (int L = 0; L < a.n_levels; ++L) {
        WALK_CLK(L, 0);
        double z[K], v[K];
#pragma unroll
        for (int k = 0; k < K; ++k) z[k] = zr[s[k]];
#pragma unroll
        for (int k = 0; k < K / 2; ++k) {
            const double2 c = reinterpret_cast<const double2*>(vrec)[k];
            v[2 * k] = c.x;
            v[2 * k + 1] = c.y;
        }
        const int4 mn = meta[L + 1];
        const int need = static_cast<unsigned>(mn.y) >> 18;  // chunk id + 1 when level L+1 starts a chunk
        if (need)
            while (ld_volatile(landed) < need) {
            }
        double acc;
        if (K2) {
            acc = fma(v[1], z[1], fma(v[0], z[0], b));
        } else {
            const double q0 = fma(v[1], z[1], fma(v[0], z[0], b));
            const double q1 = fma(v[3 % K], z[3 % K], v[2 % K] * z[2 % K]);
            const double q2 = fma(v[5 % K], z[5 % K], v[4 % K] * z[4 % K]);
            const double q3 = fma(v[7 % K], z[7 % K], v[6 % K] * z[6 % K]);
            acc = (q0 + q1) + (q2 + q3);
        }
        zr[wpos] = acc;
        zr[pin] = acc;
        if (rowid >= 0) a.z_new[rowid] = acc;
        WALK_CLK(L, 1);
        fetch(mn);
        WALK_CLK(L, 2);
        asm volatile("bar.sync 1, %0;" ::"r"(ncons) : "memory");
        if (threadIdx.x == 32) st_volatile(progress, L + 1);
    }
}

__global__ void __launch_bounds__(512, 1) k_gs_walk(WalkArgs a) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
    int* flags = reinterpret_cast<int*>(sm + kBars * 8);  // {levels done, chunks landed}
    unsigned char* nullrec = sm + kBars * 8 + 16;
    int4* meta = reinterpret_cast<int4*>(nullrec + kNullBytes);
    int4* ctab = reinterpret_cast<int4*>(reinterpret_cast<unsigned char*>(meta) + a.meta_bytes);
    int* cfirst = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(ctab) + a.chunk_bytes);
    double* zr = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(cfirst) + a.cfirst_bytes);
    unsigned char* stage = reinterpret_cast<unsigned char*>(zr) + a.zbytes;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int wc = (tid >> 5) - 1;  // consumer warp index (-1: producer warp)
    const int nl = a.n_levels, nc = a.n_chunks;
    const int zero_slot = a.ring, dummy = a.ring + 1;

    for (int l = tid; l <= nl; l += blockDim.x) meta[l] = a.meta_g[l];
    for (int c = tid; c < nc; c += blockDim.x) ctab[c] = a.chunk_g[c];
    if (tid < kBars) mbar_init(&bars[tid], 1);
    if (tid < 2) {  // null records
        int* nr = reinterpret_cast<int*>(nullrec + 128 * tid);
        for (int k = 0; k < 32; ++k) nr[k] = 0;
        nr[2] = -1;     // rowid
        nr[3] = dummy;  // pin
        for (int k = 0; k < kMaxK; ++k) nr[(tid ? 20 : 8) + k] = zero_slot;
    }
    if (tid == 0) {
        zr[zero_slot] = 0.0;
        flags[0] = 0;
        flags[1] = 0;
    }
    fence_mbar_init();
    __syncthreads();

    if (wc >= 0) {
        if (wc < a.w2)
            walk_consumer<true>(a, meta, stage, nullrec, zr, flags, wc * 32 + lane);
        else
            walk_consumer<false>(a, meta, stage, nullrec, zr, flags, (wc - a.w2) * 32 + lane);
        return;
    }
    if (tid != 0) return;
    // producer: issue chunk copies once the consumers' progress frees their
    // ring space, publish each chunk once it has landed
    int ci = 0, cw = 0;
    while (cw < nc) {
        const int done = ld_volatile(&flags[0]) - 1;  // last completed level
        while (ci < nc && ci < cw + kBars && ctab[ci].w <= done) {
            const int4 cd = ctab[ci];
            uint64_t* bar = &bars[ci % kBars];
            mbar_expect_tx(bar, static_cast<unsigned>(cd.y));
            tma_load_1d(stage + cd.z, a.packed + static_cast<size_t>(cd.x) * 16, static_cast<unsigned>(cd.y), bar);
            ++ci;
        }
        if (cw < ci && mbar_test(&bars[cw % kBars], static_cast<unsigned>(cw / kBars) & 1u)) {
            __threadfence_block();
            ++cw;
            st_volatile(&flags[1], cw);
        } else {
            __nanosleep(20);
        }
    }
}

}  // namespace

// Returns false when the system does not fit the walk (rows with more than 8
// lower entries, levels wider than the block, a level too large for the
// staging ring); the caller then builds the banded plan.
bool GsPlan::build_walk(const HostCsr& a, const std::vector<double>& dinv_h, const std::vector<int>& nlow,
                        int max_k, cudaStream_t s) {
    auto reject = [&](const char* why) {
        if (std::getenv("SDG_DEBUG")) std::fprintf(stderr, "[sdg gs walk] n=%d: not used (%s)\n", a.n_rows, why);
        return false;
    };
    if (max_k > kMaxK) return reject("a row has more than 8 lower entries");
    n = a.n_rows;
    std::vector<int> lev(n, 0);
    int nl = 0;
    for (int i = 0; i < n; ++i) {
        int d = 0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] < i) d = std::max(d, lev[a.ci[k]] + 1);
        lev[i] = d;
        nl = std::max(nl, d + 1);
    }
    // classes: w2 warps take rows with <= 2 lower entries (48-byte records),
    // the other warps everything else (112-byte records), including the
    // small rows of a level that has more of them than the w2 warps hold;
    // w2 minimises the consumer warp count
    std::vector<int> c2(nl, 0), c8(nl, 0);
    for (int i = 0; i < n; ++i) ++(nlow[i] <= 2 ? c2 : c8)[lev[i]];
    int w2 = 0, w8 = 1 << 20;
    for (int cand = 0; cand <= kMaxWarps; ++cand) {
        int need8 = 0;
        for (int q = 0; q < nl; ++q)
            need8 = std::max(need8, (c8[q] + std::max(0, c2[q] - 32 * cand) + 31) / 32);
        if (cand + need8 < w2 + w8 || (cand + need8 == w2 + w8 && cand > w2)) {
            w2 = cand;
            w8 = need8;
        }
    }
    const int max_warps = std::max(1, w2 + w8);
    if (max_warps > kMaxWarps) return reject("levels wider than the block");
    std::vector<int> n2(nl), n8(nl);
    for (int q = 0; q < nl; ++q) {
        n2[q] = std::min(c2[q], 32 * w2);
        n8[q] = c8[q] + c2[q] - n2[q];
    }
    std::vector<int> lptr(nl + 1, 0), fill2(nl), fill8(nl), order(n), pos(n), seen2(nl, 0);
    for (int q = 0; q < nl; ++q) lptr[q + 1] = lptr[q] + n2[q] + n8[q];
    for (int q = 0; q < nl; ++q) {
        fill2[q] = lptr[q];
        fill8[q] = lptr[q] + n2[q];
    }
    for (int i = 0; i < n; ++i) {
        const int q = lev[i];
        const bool small = nlow[i] <= 2 && seen2[q]++ < n2[q];
        const int p = (small ? fill2 : fill8)[q]++;
        order[p] = i;
        pos[i] = p;
    }
    int max_rows = 1;
    std::vector<int> lbytes(nl);
    std::vector<int64_t> goff(nl);
    int64_t off = 0;
    for (int q = 0; q < nl; ++q) {
        max_rows = std::max(max_rows, n2[q] + n8[q]);
        lbytes[q] = n2[q] * kK2Bytes + n8[q] * kK8Bytes;
        goff[q] = off;
        off += lbytes[q];
    }
    if (off / 16 >= (static_cast<int64_t>(1) << 31)) return reject("packed buffer too large");
    if (n >= (1 << 20) || nl >= (1 << 13)) return reject("too many rows or levels for the meta packing");

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
    const int meta_bytes = pad16(static_cast<int64_t>(nl + 1) * 16);
    const int chunk_bytes = pad16(static_cast<int64_t>(nc) * 16);
    const int cfirst_bytes = pad16(static_cast<int64_t>(nc) * 4);
    const int min_stage = std::max(3 * max_chunk, kMaxWarps * 32 * kK8Bytes);
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
        zbytes = pad16(static_cast<int64_t>(ring + 2 + npin) * 8);
        fixed = kBars * 8 + 16 + kNullBytes + meta_bytes + chunk_bytes + cfirst_bytes + zbytes;
        R = (budget - fixed) / 16 * 16;
        if (R >= min_stage) break;
        if (ring <= 64 || ring / 2 < 2 * max_rows) return reject("shared memory: ring + pinned values + staging");
        ring >>= 1;
    }
    const int zero_slot = ring, dummy_slot = ring + 1, pin_base = ring + 2;

    // staging ring placement and issue points of the chunks
    std::vector<int> roff(nc), after(nc);
    int cur = 0;
    for (int c = 0; c < nc; ++c) {
        const int sz = cbytes[c];
        if (cur + sz > R) cur = 0;
        roff[c] = cur;
        int aft = c > 0 ? after[c - 1] : -1;
        if (c >= kBars - 2) aft = std::max(aft, cfirst[c - (kBars - 2)]);  // its mbarrier was waited on
        int64_t scanned = 0;
        for (int x = c - 1; x >= 0 && scanned <= 2LL * R; --x) {
            scanned += cbytes[x];
            if (roff[x] < cur + sz && cur < roff[x] + cbytes[x]) {
                const int last = x + 1 < nc ? cfirst[x + 1] - 1 : nl - 1;
                aft = std::max(aft, last);
                break;
            }
        }
        if (aft >= 0 && aft > cfirst[c] - 3) return reject("staging ring too small for the look-ahead");
        after[c] = aft;
        cur += sz;
    }

    std::vector<double> pk(static_cast<size_t>(off / 8 + 2), 0.0);
    unsigned char* base = reinterpret_cast<unsigned char*>(pk.data());
    std::vector<int> bidx_h(n);
    std::vector<int4> meta_h(nl + 1), ctab_h(nc);
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
                                          static_cast<size_t>(t - n2[q]) * kK8Bytes;
            double* recd = reinterpret_cast<double*>(rec);
            int* reci = reinterpret_cast<int*>(rec);
            bidx_h[i] = static_cast<int>((rec - base) / 8);
            reci[2] = i;
            reci[3] = pin_of[i] >= 0 ? pin_base + pin_of[i] : dummy_slot;
            const int cap = k2 ? 2 : kMaxK;
            double* val = recd + 2;
            int* src = reci + (k2 ? 8 : 20);
            int m = 0;
            for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
                const int j = a.ci[k];
                if (j >= i) continue;
                val[m] = -(a.v[k] * dinv_h[i]);
                src[m] = lptr[q + 1] - pos[j] <= ring ? (pos[j] & (ring - 1)) : pin_base + pin_of[j];
                ++m;
                ++lower_entries;
            }
            for (; m < cap; ++m) {
                val[m] = 0.0;
                src[m] = zero_slot;
            }
        }
        const int starts = cfirst[chunk_of[q]] == q ? chunk_of[q] + 1 : 0;  // chunk id + 1 if q starts a chunk
        const int o2 = roff[chunk_of[q]] + in_chunk[q], o8 = o2 + n2[q] * kK2Bytes;
        meta_h[q] = make_int4(o2, o8 | (starts << 18), lptr[q] | (n2[q] << 20), (lptr[q] + n2[q]) | (n8[q] << 20));
    }
    meta_h[nl] = make_int4(0, 0, 0, 0);  // sentinel: the prefetch past the last level reads null rows
    for (int c = 0; c < nc; ++c)
        ctab_h[c] = make_int4(static_cast<int>(goff[cfirst[c]] / 16), cbytes[c], roff[c], after[c]);

    walk = true;
    usable = true;
    bands = 1;
    n_levels = nl;
    max_band_levels = nl;
    nthreads = 32 + 32 * max_warps;
    walk_meta_bytes = meta_bytes;
    walk_chunk_bytes = chunk_bytes;
    walk_cfirst_bytes = cfirst_bytes;
    walk_zbytes = zbytes;
    walk_chunks = nc;
    walk_w2 = w2;
    max_seg = max_chunk;
    halo = npin;
    smem = static_cast<size_t>(fixed) + R;
    if (std::getenv("SDG_DEBUG"))
        std::fprintf(stderr,
                     "[sdg gs walk] n=%d levels=%d chunks=%d threads=%d ring=%d pinned=%d stage=%d max_chunk=%d "
                     "smem=%zu packed=%.1fKB\n",
                     n, nl, nc, nthreads, ring, npin, R, max_chunk, smem, off / 1024.0);
    meta.upload(meta_h, s);
    walk_iss.upload(ctab_h, s);
    walk_cfirst.upload(cfirst, s);
    packed.upload(pk, s);
    bidx.upload(bidx_h, s);
    SDG_CUDA(cudaFuncSetAttribute(k_gs_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
    SDG_CUDA(cudaStreamSynchronize(s));  // host staging vectors die here
    return true;
}

void launch_gs_walk(Context& c, const GsPlan& g, double* z_new) {
    WalkArgs a{g.meta.get(), g.walk_iss.get(), g.walk_cfirst.get(),
               reinterpret_cast<const unsigned char*>(g.packed.get()), g.n_levels, g.walk_chunks, g.ring,
               g.walk_meta_bytes, g.walk_chunk_bytes, g.walk_cfirst_bytes, g.walk_zbytes, g.walk_w2, z_new};
    k_gs_walk<<<1, g.nthreads, g.smem, c.stream>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(SDG_ECUDA, std::string("launch_gs_walk: ") + cudaGetErrorString(e));
    c.count();
}

}  // namespace sdg
