// Strip-sharded solve across GPUs: transports, ownership / halo plans,
// distributed operators, AMG V-cycle, td_bgs and PD-GMRES (see dist.hpp).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <unordered_map>

#include "dist.hpp"
#include "launch.cuh"

namespace sdg {

// ---------------------------------------------------------------------------
// small kernels of the exchange path

namespace {

constexpr int kT = 256;
inline int nblk(int64_t n) { return static_cast<int>(std::max<int64_t>(1, (n + kT - 1) / kT)); }

__global__ void k_gather(int n, const int* __restrict__ idx, const double* __restrict__ src,
                         double* __restrict__ dst) {
    pdl_begin();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) dst[k] = src[idx[k]];
}

// dst[idx[k]] = src[k] for idx[k] >= 0
__global__ void k_scatter(int n, const int* __restrict__ idx, const double* __restrict__ src,
                          double* __restrict__ dst) {
    pdl_begin();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n && idx[k] >= 0) dst[idx[k]] = src[k];
}

// acc[t] += recv[src[q]] for q in [ptr[t], ptr[t+1]), in order
__global__ void k_add_gathered(int n, const int* __restrict__ ptr, const int* __restrict__ src,
                               const double* __restrict__ recv, double* __restrict__ acc) {
    pdl_begin();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int e = ptr[t + 1];
    if (ptr[t] == e) return;
    double a = acc[t];
    for (int q = ptr[t]; q < e; ++q) a = __dadd_rn(a, recv[src[q]]);
    acc[t] = a;
}

// BiCGSTAB vector updates with host scalars, in the reference's operation
// order (krylov.cpp:246,255,278-279)
__global__ void k_dbi_p(int n, double beta, double omega, const double* __restrict__ r,
                        const double* __restrict__ vv, double* __restrict__ p) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = __dadd_rn(r[i], __dmul_rn(beta, __dsub_rn(p[i], __dmul_rn(omega, vv[i]))));
}

__global__ void k_dbi_s(int n, double alpha, const double* __restrict__ r, const double* __restrict__ vv,
                        double* __restrict__ s) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) s[i] = __dsub_rn(r[i], __dmul_rn(alpha, vv[i]));
}

__global__ void k_dbi_xr(int n, double alpha, double omega, const double* __restrict__ phat,
                         const double* __restrict__ shat, const double* __restrict__ s,
                         const double* __restrict__ t, double* __restrict__ x, double* __restrict__ r) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    x[i] = __dadd_rn(x[i], __dadd_rn(__dmul_rn(alpha, phat[i]), __dmul_rn(omega, shat[i])));
    r[i] = __dsub_rn(s[i], __dmul_rn(omega, t[i]));
}

__global__ void k_daxpy(int n, double alpha, const double* __restrict__ x, double* __restrict__ y) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = __dadd_rn(y[i], __dmul_rn(alpha, x[i]));
}

void launch_gather(Context& c, int n, const int* idx, const double* src, double* dst) {
    ProfScope ps_(c, PF_VEC, 16.0 * n);
    if (n <= 0) return;
    launch_k(c, k_gather, nblk(n), kT, 0, n, idx, src, dst);
    c.count();
}

void launch_scatter(Context& c, int n, const int* idx, const double* src, double* dst) {
    ProfScope ps_(c, PF_VEC, 20.0 * n);
    if (n <= 0) return;
    launch_k(c, k_scatter, nblk(n), kT, 0, n, idx, src, dst);
    c.count();
}

void launch_add_gathered(Context& c, int n, const int* ptr, const int* src, const double* recv, double* acc) {
    ProfScope ps_(c, PF_RESTRICT, 20.0 * n);
    if (n <= 0) return;
    launch_k(c, k_add_gathered, nblk(n), kT, 0, n, ptr, src, recv, acc);
    c.count();
}

int total(const std::vector<int>& v) {
    int s = 0;
    for (int x : v) s += x;
    return s;
}

template <class T>
void upload_vec(DevBuf<T>& d, const std::vector<T>& h, cudaStream_t s) {
    d.resize(std::max<size_t>(h.size(), 1));
    d.upload(h.data(), h.size(), s);
}

bool env_on(const char* name) {
    const char* e = std::getenv(name);
    return e && e[0] == '1';
}

}  // namespace

// ---------------------------------------------------------------------------
// transports

void Transport::allreduce(Context& c, const double* partial, int k, double* host_out) {
    const size_t need = static_cast<size_t>(size) * k;
    if (gather_.size() < need) gather_.resize(need);
    allgather(c, partial, k, gather_.get());
    host_.resize(need);
    SDG_CUDA(cudaMemcpyAsync(host_.data(), gather_.get(), need * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    for (int j = 0; j < k; ++j) {
        double s = 0.0;
        for (int p = 0; p < size; ++p) s += host_[static_cast<size_t>(p) * k + j];
        host_out[j] = s;
    }
}

namespace {

// out[j] = sum over ranks p in rank order of g[p * k + j] (the order the host
// fold of Transport::allreduce uses, so both give the same bits)
__global__ void k_fold_ranks(int k, int size, const double* __restrict__ g, double* __restrict__ out, int take_sqrt) {
    pdl_begin();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    double s = 0.0;
    for (int p = 0; p < size; ++p) s += g[static_cast<size_t>(p) * k + j];
    out[j] = take_sqrt ? sqrt(s) : s;
}

}  // namespace

void Transport::allreduce_device(Context& c, const double* partial, int k, double* out, bool take_sqrt) {
    if (k <= 0) return;
    const size_t need = static_cast<size_t>(size) * k;
    if (gather_.size() < need) gather_.resize(need);
    allgather(c, partial, k, gather_.get());
    launch_k(c, k_fold_ranks, (k + 127) / 128, 128, 0, k, size, static_cast<const double*>(gather_.get()), out,
             take_sqrt ? 1 : 0);
    c.count();
}

namespace {

struct HostTransport final : Transport {
    HostExchangeFn ex;
    HostAllgatherFn ag;
    void* user;
    std::unique_ptr<PinnedBuf> sbuf, rbuf;

    double* stage(std::unique_ptr<PinnedBuf>& b, size_t doubles) {
        const size_t bytes = std::max<size_t>(doubles, 1) * sizeof(double);
        if (!b || b->bytes() < bytes) b = std::make_unique<PinnedBuf>(bytes * 2);
        return b->as<double>();
    }

    void exchange(Context& c, const double* send, const std::vector<int>& scount, double* recv,
                  const std::vector<int>& rcount) override {
        const int ns = total(scount), nr = total(rcount);
        double* hs = stage(sbuf, ns);
        double* hr = stage(rbuf, nr);
        if (ns) SDG_CUDA(cudaMemcpyAsync(hs, send, ns * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        if (ex(user, hs, scount.data(), hr, rcount.data()) != 0) fail(SDG_ENCCL, "transport: exchange callback failed");
        if (nr) SDG_CUDA(cudaMemcpyAsync(recv, hr, nr * sizeof(double), cudaMemcpyHostToDevice, c.stream));
        c.sync();
    }

    void allgather(Context& c, const double* send, int count, double* recv) override {
        if (size == 1) {
            launch_copy(c, recv, send, count);
            return;
        }
        double* hs = stage(sbuf, count);
        double* hr = stage(rbuf, static_cast<size_t>(count) * size);
        if (count) SDG_CUDA(cudaMemcpyAsync(hs, send, count * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        if (ag(user, hs, count, hr) != 0) fail(SDG_ENCCL, "transport: allgather callback failed");
        if (count)
            SDG_CUDA(cudaMemcpyAsync(recv, hr, static_cast<size_t>(count) * size * sizeof(double),
                                     cudaMemcpyHostToDevice, c.stream));
        c.sync();
    }
};

// NCCL, resolved at run time so the library loads where NCCL is absent.
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;

    static NcclApi& get() {
        static NcclApi api = [] {
            NcclApi a;
            for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
                a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
                if (a.h) break;
            }
            if (!a.h) return a;
            auto sym = [&](const char* s) { return dlsym(a.h, s); };
            a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(sym("ncclGetUniqueId"));
            a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(sym("ncclCommInitRank"));
            a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(sym("ncclCommDestroy"));
            a.send = reinterpret_cast<decltype(a.send)>(sym("ncclSend"));
            a.recv = reinterpret_cast<decltype(a.recv)>(sym("ncclRecv"));
            a.groupStart = reinterpret_cast<decltype(a.groupStart)>(sym("ncclGroupStart"));
            a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(sym("ncclGroupEnd"));
            a.allGather = reinterpret_cast<decltype(a.allGather)>(sym("ncclAllGather"));
            a.errStr = reinterpret_cast<decltype(a.errStr)>(sym("ncclGetErrorString"));
            return a;
        }();
        if (!api.h || !api.commInitRank || !api.send || !api.allGather)
            fail(SDG_ENCCL, "NCCL transport: libnccl.so.2 not found");
        return api;
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess)
            fail(SDG_ENCCL, std::string(what) + ": " + (errStr ? errStr(r) : "NCCL error"));
    }
};

struct NcclTransport final : Transport {
    ncclComm_t comm = nullptr;
    ~NcclTransport() override {
        if (comm) NcclApi::get().commDestroy(comm);
    }
    void exchange(Context& c, const double* send, const std::vector<int>& scount, double* recv,
                  const std::vector<int>& rcount) override {
        NcclApi& n = NcclApi::get();
        n.check(n.groupStart(), "ncclGroupStart");
        size_t so = 0, ro = 0;
        for (int p = 0; p < size; ++p) {
            if (scount[p]) n.check(n.send(send + so, scount[p], ncclDouble, p, comm, c.stream), "ncclSend");
            if (rcount[p]) n.check(n.recv(recv + ro, rcount[p], ncclDouble, p, comm, c.stream), "ncclRecv");
            so += scount[p];
            ro += rcount[p];
        }
        n.check(n.groupEnd(), "ncclGroupEnd");
    }
    void allgather(Context& c, const double* send, int count, double* recv) override {
        NcclApi& n = NcclApi::get();
        n.check(n.allGather(send, recv, count, ncclDouble, comm, c.stream), "ncclAllGather");
    }
};

}  // namespace

TransportPtr make_host_transport(int rank, int size, HostExchangeFn ex, HostAllgatherFn ag, void* user) {
    if (size < 1 || rank < 0 || rank >= size) fail(SDG_EINVAL, "transport: bad rank / size");
    if (!ex || !ag) fail(SDG_EINVAL, "transport: null callback");
    auto t = std::make_shared<HostTransport>();
    t->rank = rank;
    t->size = size;
    t->ex = ex;
    t->ag = ag;
    t->user = user;
    return t;
}

void nccl_unique_id(unsigned char out[128]) {
    NcclApi& n = NcclApi::get();
    ncclUniqueId id;
    n.check(n.getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, 128);
}

TransportPtr make_nccl_transport(Context& c, const unsigned char id[128], int rank, int size) {
    if (size < 1 || rank < 0 || rank >= size) fail(SDG_EINVAL, "transport: bad rank / size");
    NcclApi& n = NcclApi::get();
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    auto t = std::make_shared<NcclTransport>();
    t->rank = rank;
    t->size = size;
    SDG_CUDA(cudaSetDevice(c.device));
    n.check(n.commInitRank(&t->comm, size, uid, rank), "ncclCommInitRank");
    return t;
}

// ---------------------------------------------------------------------------
// ownership and halo plans

Ownership Ownership::from_owner(std::vector<int> owner_in, int size_in) {
    Ownership o;
    o.size = size_in;
    o.owner = std::move(owner_in);
    o.lidx.assign(o.owner.size(), -1);
    o.owned.assign(size_in, {});
    for (int g = 0; g < static_cast<int>(o.owner.size()); ++g) {
        const int p = o.owner[g];
        if (p < 0 || p >= size_in) fail(SDG_EINVAL, "partition: owner rank out of range at dof " + std::to_string(g));
        o.lidx[g] = static_cast<int>(o.owned[p].size());
        o.owned[p].push_back(g);
    }
    return o;
}

Ownership Ownership::slice(int g0, int g1) const {
    return from_owner(std::vector<int>(owner.begin() + g0, owner.begin() + g1), size);
}

void build_local(const HostCsr& a, const Ownership& R, const Ownership& Cc, int rank, HostCsr& loc, Halo& h) {
    if (R.n() != a.n_rows || Cc.n() != a.n_cols) fail(SDG_EDIM, "distributed operator: partition does not cover the matrix");
    const int P = R.size;
    const std::vector<int>& rows = R.owned[rank];
    h.n_owned = static_cast<int>(Cc.owned[rank].size());
    std::vector<int> gh;
    for (int g : rows)
        for (int k = a.rp[g]; k < a.rp[g + 1]; ++k)
            if (Cc.owner[a.ci[k]] != rank) gh.push_back(a.ci[k]);
    auto by_owner = [&](int x, int y) { return Cc.owner[x] != Cc.owner[y] ? Cc.owner[x] < Cc.owner[y] : x < y; };
    std::sort(gh.begin(), gh.end(), by_owner);
    gh.erase(std::unique(gh.begin(), gh.end()), gh.end());
    h.ghost_gid = gh;
    h.rcount.assign(P, 0);
    std::unordered_map<int, int> gpos;
    gpos.reserve(gh.size() * 2 + 1);
    for (int k = 0; k < static_cast<int>(gh.size()); ++k) {
        gpos[gh[k]] = h.n_owned + k;
        ++h.rcount[Cc.owner[gh[k]]];
    }
    loc = HostCsr(static_cast<int>(rows.size()), h.n_owned + static_cast<int>(gh.size()));
    loc.ci.reserve(rows.size() * 8);
    loc.v.reserve(rows.size() * 8);
    for (int r = 0; r < static_cast<int>(rows.size()); ++r) {
        const int g = rows[r];
        for (int k = a.rp[g]; k < a.rp[g + 1]; ++k) {
            const int j = a.ci[k];
            loc.ci.push_back(Cc.owner[j] == rank ? Cc.lidx[j] : gpos[j]);
            loc.v.push_back(a.v[k]);
        }
        loc.rp[r + 1] = static_cast<int>(loc.ci.size());
    }
    // what each peer needs from this rank (same rule, evaluated on its rows)
    h.scount.assign(P, 0);
    h.send_gid.clear();
    for (int p = 0; p < P; ++p) {
        if (p == rank) continue;
        std::vector<int> need;
        for (int g : R.owned[p])
            for (int k = a.rp[g]; k < a.rp[g + 1]; ++k)
                if (Cc.owner[a.ci[k]] == rank) need.push_back(a.ci[k]);
        std::sort(need.begin(), need.end());
        need.erase(std::unique(need.begin(), need.end()), need.end());
        h.scount[p] = static_cast<int>(need.size());
        h.send_gid.insert(h.send_gid.end(), need.begin(), need.end());
    }
}

void Halo::update(Context& c, Transport& t, double* x_ext) {
    if (t.size == 1) return;
    const int ns = static_cast<int>(send_gid.size());
    launch_gather(c, ns, send_idx.get(), x_ext, send_buf.get());
    t.exchange(c, send_buf.get(), scount, x_ext + n_owned, rcount);
}

void DistOp::build(Context& c, const HostCsr& global, const Ownership& rows, const Ownership& cols, int rank) {
    build_local(global, rows, cols, rank, host, halo);
    n_rows = host.n_rows;
    a.upload(host, c.stream);
    std::vector<int> sidx(halo.send_gid.size());
    for (size_t k = 0; k < sidx.size(); ++k) sidx[k] = cols.lidx[halo.send_gid[k]];
    upload_vec(halo.send_idx, sidx, c.stream);
    halo.send_buf.resize(std::max<size_t>(sidx.size(), 1));
    x_ext.resize(std::max(host.n_cols, 1));
}

double* DistOp::load(Context& c, Transport& t, const double* x) {
    launch_copy(c, x_ext.get(), x, halo.n_owned);
    halo.update(c, t, x_ext.get());
    return x_ext.get();
}

void DistOp::apply(Context& c, Transport& t, const double* x, double* y) {
    const double* xe = load(c, t, x);
    launch_spmv(c, a, xe, y);
}

void DistOp::apply_add(Context& c, Transport& t, const double* x, const double* y_in, double* y_out, double alpha) {
    const double* xe = load(c, t, x);
    launch_spmv_add(c, a, xe, y_in, y_out, alpha);
}

std::vector<int> strip_partition(int n, int size) {
    if (n < 1 || size < 1 || size > n) fail(SDG_EINVAL, "strip_partition: need 1 <= ranks <= cells per side");
    const int n_u = (n + 1) * n, n_v = n * (n + 1), n_p = n * n;
    std::vector<int> owner(n_u + n_v + 2 * n_p);
    auto strip = [&](int j) { return static_cast<int>(static_cast<int64_t>(j) * size / n); };
    int g = 0;
    for (int j = 0; j < n; ++j)            // u(i, j), i = 0..n  (grid.hpp: j-major)
        for (int i = 0; i <= n; ++i) owner[g++] = strip(j);
    for (int j = 0; j <= n; ++j)           // v(i, j), j = 0..n (top wall row joins the top strip)
        for (int i = 0; i < n; ++i) owner[g++] = strip(std::min(j, n - 1));
    for (int j = 0; j < n; ++j)            // p_ff(i, j)
        for (int i = 0; i < n; ++i) owner[g++] = strip(j);
    for (int j = 0; j < n; ++j)            // p_pm(i, j): rank 0 at the top, next to the interface
        for (int i = 0; i < n; ++i) owner[g++] = size - 1 - strip(j);
    return owner;
}

// ---------------------------------------------------------------------------
// AMG over strips

DistAmg::DistAmg(CtxPtr c, TransportPtr t, const HostCsr& a, const Ownership& own, const AmgOpts& o)
    : ctx_(std::move(c)), tr_(std::move(t)) {
    Context& cx = *ctx_;
    const int rank = tr_->rank, P = tr_->size;
    std::vector<HostLevel> hl = build_hierarchy(a, o);
    n_levels_ = static_cast<int>(hl.size());
    n_rows_ = static_cast<int>(own.owned[rank].size());
    const bool exact = env_on("SDG_GS_EXACT");

    // ownership per level: a coarse dof belongs to the owner of the first
    // (lowest) fine row of its aggregate
    std::vector<Ownership> O(n_levels_);
    O[0] = own;
    for (int l = 0; l + 1 < n_levels_; ++l) {
        const std::vector<int>& agg = hl[l].aggregate_of;
        std::vector<int> oc(hl[l].n_coarse, -1);
        for (int i = 0; i < static_cast<int>(agg.size()); ++i)
            if (oc[agg[i]] < 0) oc[agg[i]] = O[l].owner[i];
        O[l + 1] = Ownership::from_owner(std::move(oc), P);
    }

    lv_.resize(std::max(n_levels_ - 1, 0));
    for (int l = 0; l + 1 < n_levels_; ++l) {
        Level& V = lv_[l];
        const HostCsr& A = hl[l].a;
        require_diagonal(A, "sor_sweep");
        V.A.build(cx, A, O[l], O[l], rank);
        const int n = V.A.n_rows;
        const int ng = V.A.halo.n_ghost();
        // owned block (lower triangle for the smoother) and the ghost columns
        HostCsr blk(n, n), G(n, std::max(ng, 1));
        for (int r = 0; r < n; ++r) {
            for (int k = V.A.host.rp[r]; k < V.A.host.rp[r + 1]; ++k) {
                const int j = V.A.host.ci[k];
                if (j < n) {
                    blk.ci.push_back(j);
                    blk.v.push_back(V.A.host.v[k]);
                } else {
                    G.ci.push_back(j - n);
                    G.v.push_back(V.A.host.v[k]);
                }
            }
            blk.rp[r + 1] = static_cast<int>(blk.ci.size());
            G.rp[r + 1] = static_cast<int>(G.ci.size());
        }
        V.G.upload(G, cx.stream);
        if (!exact && n > 0) {
            std::vector<int> comps;
            if (!hl[l].components.empty()) {
                comps.resize(n);
                for (int r = 0; r < n; ++r) comps[r] = hl[l].components[O[l].owned[rank][r]];
            }
            V.gs.build(blk, comps, cx.stream);
            V.fast = V.gs.usable;
        }
        if (!V.fast) {
            LevelSchedule s = lower_schedule(blk);
            upload_vec(V.lvl_ptr, s.lvl_ptr, cx.stream);
            upload_vec(V.lvl_rows, s.lvl_rows, cx.stream);
            V.n_sched = s.n_levels();
        }

        // restriction / prolongation plan with level l + 1
        const std::vector<int>& agg = hl[l].aggregate_of;
        const Ownership& Oc = O[l + 1];
        const std::vector<int>& fine = O[l].owned[rank];
        V.n_c_owned = static_cast<int>(Oc.owned[rank].size());
        std::vector<int> rem;
        for (int g : fine)
            if (Oc.owner[agg[g]] != rank) rem.push_back(agg[g]);
        std::sort(rem.begin(), rem.end(), [&](int x, int y) {
            return Oc.owner[x] != Oc.owner[y] ? Oc.owner[x] < Oc.owner[y] : x < y;
        });
        rem.erase(std::unique(rem.begin(), rem.end()), rem.end());
        V.n_c_remote = static_cast<int>(rem.size());
        V.rem_scount.assign(P, 0);
        std::unordered_map<int, int> rslot;
        for (int k = 0; k < V.n_c_remote; ++k) {
            rslot[rem[k]] = V.n_c_owned + k;
            ++V.rem_scount[Oc.owner[rem[k]]];
        }
        const int n_ext = V.n_c_owned + V.n_c_remote;
        std::vector<int> agg_local(n), cnt(n_ext + 1, 0);
        for (int r = 0; r < n; ++r) {
            const int cg = agg[fine[r]];
            agg_local[r] = Oc.owner[cg] == rank ? Oc.lidx[cg] : rslot[cg];
            ++cnt[agg_local[r] + 1];
        }
        for (int k = 0; k < n_ext; ++k) cnt[k + 1] += cnt[k];
        std::vector<int> pt_rows(n), fillp(cnt.begin(), cnt.end() - 1);
        for (int r = 0; r < n; ++r) pt_rows[fillp[agg_local[r]]++] = r;
        upload_vec(V.agg_local, agg_local, cx.stream);
        upload_vec(V.pt_ptr, cnt, cx.stream);
        upload_vec(V.pt_rows, pt_rows, cx.stream);
        // partial sums this rank receives, and the coarse values it returns
        V.rem_rcount.assign(P, 0);
        std::vector<int> back, pos_target;
        for (int p = 0; p < P; ++p) {
            if (p == rank) continue;
            std::vector<int> lp;
            for (int g : O[l].owned[p])
                if (Oc.owner[agg[g]] == rank) lp.push_back(agg[g]);
            std::sort(lp.begin(), lp.end());
            lp.erase(std::unique(lp.begin(), lp.end()), lp.end());
            V.rem_rcount[p] = static_cast<int>(lp.size());
            for (int cg : lp) {
                back.push_back(Oc.lidx[cg]);
                pos_target.push_back(Oc.lidx[cg]);
            }
        }
        std::vector<int> aptr(V.n_c_owned + 1, 0);
        for (int t2 : pos_target) ++aptr[t2 + 1];
        for (int k = 0; k < V.n_c_owned; ++k) aptr[k + 1] += aptr[k];
        std::vector<int> asrc(pos_target.size()), afill(aptr.begin(), aptr.end() - 1);
        for (int q = 0; q < static_cast<int>(pos_target.size()); ++q) asrc[afill[pos_target[q]]++] = q;
        upload_vec(V.add_ptr, aptr, cx.stream);
        upload_vec(V.add_src, asrc, cx.stream);
        upload_vec(V.back_idx, back, cx.stream);
        V.c_ext_gid = Oc.owned[rank];
        V.c_ext_gid.insert(V.c_ext_gid.end(), rem.begin(), rem.end());
        upload_vec(V.c_ext_gid_dev, V.c_ext_gid, cx.stream);
        V.rc_ext.resize(std::max(n_ext, 1));
        V.zc_ext.resize(std::max(n_ext, 1));
        V.recv_buf.resize(std::max<size_t>(back.size(), 1));
        V.back_buf.resize(std::max<size_t>(back.size(), 1));
        V.zt_ext.resize(std::max(n + ng, 1));
        V.reff.resize(std::max(n, 1));
    }

    // coarsest level: replicated direct solve (coarse.hpp), allgathered right-hand side
    const HostCsr& Ac = hl.back().a;
    n_c_ = Ac.n_rows;
    coarse_.build(cx, Ac);
    const Ownership& Oc = O.back();
    c_owned_ = static_cast<int>(Oc.owned[rank].size());
    c_max_ = 1;
    for (int p = 0; p < P; ++p) c_max_ = std::max<int>(c_max_, static_cast<int>(Oc.owned[p].size()));
    std::vector<int> slot(static_cast<size_t>(P) * c_max_, -1);
    for (int p = 0; p < P; ++p)
        for (int k = 0; k < static_cast<int>(Oc.owned[p].size()); ++k) slot[static_cast<size_t>(p) * c_max_ + k] = Oc.owned[p][k];
    upload_vec(c_slot_gid_, slot, cx.stream);
    upload_vec(c_own_gid_, Oc.owned[rank], cx.stream);
    c_send_.resize(c_max_);
    c_gather_.resize(static_cast<size_t>(P) * c_max_);
    c_full_.resize(std::max(n_c_, 1));
    c_sol_.resize(std::max(n_c_, 1));
    cx.sync();
}

void DistAmg::coarse_solve(const double* r_owned) {
    Context& cx = *ctx_;
    launch_fill(cx, c_send_.get(), 0.0, c_max_);
    launch_copy(cx, c_send_.get(), r_owned, c_owned_);
    tr_->allgather(cx, c_send_.get(), c_max_, c_gather_.get());
    launch_scatter(cx, tr_->size * c_max_, c_slot_gid_.get(), c_gather_.get(), c_full_.get());
    coarse_.solve(cx, c_full_.get(), c_sol_.get());
}

void DistAmg::vcycle(int l, const double* r, double* z) {
    Context& cx = *ctx_;
    Transport& t = *tr_;
    if (l + 1 == n_levels_) {  // single-level hierarchy
        coarse_solve(r);
        launch_gather(cx, c_owned_, c_own_gid_.get(), c_sol_.get(), z);
        return;
    }
    Level& V = lv_[l];
    const int n = V.A.n_rows;
    // pre-smoother: z_old = 0 on every rank, so ghost columns contribute nothing
    if (V.fast) {
        launch_gs_prep_pre(cx, V.gs, r);
        launch_gs_lower(cx, V.gs, z);
    } else {
        launch_gs_levels(cx, V.A.a, V.lvl_ptr.get(), V.lvl_rows.get(), V.n_sched, r, nullptr, z, 1.0);
    }
    // residual + restriction (own aggregates and partial sums for remote ones)
    const double* zx = V.A.load(cx, t, z);
    launch_resid_restrict(cx, V.A.a, V.pt_ptr.get(), V.pt_rows.get(), V.n_c_owned + V.n_c_remote, r, zx,
                          V.rc_ext.get());
    if (t.size > 1) {
        t.exchange(cx, V.rc_ext.get() + V.n_c_owned, V.rem_scount, V.recv_buf.get(), V.rem_rcount);
        launch_add_gathered(cx, V.n_c_owned, V.add_ptr.get(), V.add_src.get(), V.recv_buf.get(), V.rc_ext.get());
    }
    // coarse correction, then the coarse ghosts this rank's aggregates need
    if (l + 2 == n_levels_) {
        coarse_solve(V.rc_ext.get());
        launch_gather(cx, V.n_c_owned + V.n_c_remote, V.c_ext_gid_dev.get(), c_sol_.get(), V.zc_ext.get());
    } else {
        vcycle(l + 1, V.rc_ext.get(), V.zc_ext.get());
        if (t.size > 1) {
            const int nb = static_cast<int>(total(V.rem_rcount));
            launch_gather(cx, nb, V.back_idx.get(), V.zc_ext.get(), V.back_buf.get());
            t.exchange(cx, V.back_buf.get(), V.rem_rcount, V.zc_ext.get() + V.n_c_owned, V.rem_scount);
        }
    }
    // post-smoother from z_old = z + P zc, ghosts = the neighbours' z + P zc
    launch_prolong(cx, n, V.agg_local.get(), z, V.zc_ext.get(), V.zt_ext.get());
    V.A.halo.update(cx, t, V.zt_ext.get());
    if (V.fast) {
        launch_spmv_add(cx, V.G, V.zt_ext.get() + n, r, V.reff.get(), -1.0);
        launch_gs_prep_post(cx, V.gs, V.reff.get(), z, V.zc_ext.get(), V.agg_local.get());
        launch_gs_lower(cx, V.gs, z);
    } else {
        launch_gs_levels(cx, V.A.a, V.lvl_ptr.get(), V.lvl_rows.get(), V.n_sched, r, V.zt_ext.get(), z, 1.0);
    }
}

// ---------------------------------------------------------------------------
// td_bgs over strips

DistTd::DistTd(DistSystem& s, int kind, int v_levels, int d_levels, double omega_override) : s_(s), kind_(kind) {
    auto t0 = std::chrono::steady_clock::now();
    if (kind != SDG_TD_BJ && kind != SDG_TD_BGS && kind != SDG_DIST_UZAWA && kind != SDG_DIST_AMG)
        fail(SDG_EINVAL, "dist td: kind must be td_bj, td_bgs, SDG_DIST_UZAWA or SDG_DIST_AMG");
    Context& cx = *s.ctx;
    Transport& tr = *s.tr;
    const int rank = tr.rank;
    const HostCsr& A = s.global;
    const int n = A.n_rows, n_vel = s.n_vel, n_ff = s.n_vel + s.n_pff;
    if (kind == SDG_DIST_AMG) {
        // the porous subdomain solve of the partitioned driver (coupling.cpp:140-146):
        // AMG on the matrix as it is
        if (n_ff != 0) fail(SDG_EDIM, "dist amg: the system must be one block (n_vel = n_pff = 0)");
        AmgOpts da;
        da.max_levels = d_levels;
        d_ = std::make_unique<DistAmg>(s.ctx, s.tr, A, s.own, da);
        cx.sync();
        setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return;
    }
    if (kind == SDG_DIST_UZAWA && s.n_ppm != 0) fail(SDG_EDIM, "dist uzawa: the system must have no porous block");
    // bench.cpp:121-182
    const HostCsr V = submatrix(A, 0, n_vel, 0, n_vel);
    const HostCsr B = submatrix(A, 0, n_vel, n_vel, n_ff);
    const HostCsr C = submatrix(A, n_vel, n_ff, 0, n_vel);
    const Ownership Ov = s.own.slice(0, n_vel), Op = s.own.slice(n_vel, n_ff);
    AmgOpts va;
    va.max_levels = v_levels;
    va.components.assign(n_vel, 0);
    for (int k = s.n_u; k < n_vel; ++k) va.components[k] = 1;
    v_ = std::make_unique<DistAmg>(s.ctx, s.tr, V, Ov, va);
    c_.build(cx, C, Op, Ov, rank);
    b_.build(cx, B, Ov, Op, rank);
    if (kind != SDG_DIST_UZAWA) {
        const HostCsr D = ground_dof(submatrix(A, n_ff, n, n_ff, n), 0);
        const Ownership Off = s.own.slice(0, n_ff), Opm = s.own.slice(n_ff, n);
        AmgOpts da;
        da.max_levels = d_levels;
        d_ = std::make_unique<DistAmg>(s.ctx, s.tr, D, Opm, da);
        if (kind_ == SDG_TD_BGS) cp_.build(cx, submatrix(A, n_ff, n, 0, n_ff), Opm, Off, rank);
        tmp_.resize(std::max(s.n_ppm_loc, 1));
    }

    if (!std::isnan(omega_override)) {
        omega_ = omega_override;
    } else {
        // power_iteration (krylov.cpp:307-339) on C Vtilde^{-1} B, seed 1729,
        // tol 1e-3, 200 iterations (UzawaConfig defaults, precond.hpp:126-128);
        // the start vector is the reference's global one, sliced per rank.
        std::mt19937 rng(1729u);
        std::uniform_real_distribution<double> dist(-1.0, 1.0);
        std::vector<double> xg(s.n_pff);
        for (double& v : xg) v = dist(rng);
        double ss = 0.0;
        for (double v : xg) ss += v * v;
        double xn = std::sqrt(ss);
        if (xn == 0.0) xg[0] = xn = 1.0;
        const double inv = 1.0 / xn;
        for (double& v : xg) v *= inv;
        const int np = s.n_pff_loc, nv = s.n_v_loc;
        std::vector<double> xl(np);
        for (int k = 0; k < np; ++k) xl[k] = xg[Op.owned[rank][k]];
        DevBuf<double> x(std::max(np, 1)), y(std::max(np, 1)), t1(std::max(nv, 1)), t2(std::max(nv, 1)), part(2), scal(1);
        x.upload(xl.data(), np, cx.stream);
        ReduceWs ws;
        ws.init(reduce_blocks(std::max(np, 1), cx.num_sms), 2, cx.stream);
        double prev = 0.0, lambda = 0.0, hv[2];
        for (int k = 0; k < 200; ++k) {
            b_.apply(cx, tr, x.get(), t1.get());
            v_->apply(t1.get(), t2.get());
            c_.apply(cx, tr, t2.get(), y.get());
            launch_dot(cx, ws, np, x.get(), y.get(), part.get());
            launch_norm2sq(cx, ws, np, y.get(), part.get() + 1);
            tr.allreduce(cx, part.get(), 2, hv);
            lambda = hv[0];
            const double yn = std::sqrt(hv[1]);
            if (k > 0 && std::abs(lambda - prev) <= 1e-3 * std::abs(lambda)) break;
            prev = lambda;
            if (yn == 0.0) {
                lambda = 0.0;
                break;
            }
            SDG_CUDA(cudaMemcpyAsync(scal.get(), &yn, sizeof(double), cudaMemcpyHostToDevice, cx.stream));
            launch_div_scalar(cx, np, y.get(), scal.get(), x.get());
            cx.sync();
        }
        omega_ = (std::abs(lambda) > 1e-300) ? 1.0 / lambda : 1.0;
    }
    cx.sync();
    setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void DistTd::apply(const double* r, double* z) {
    Context& cx = *s_.ctx;
    Transport& tr = *s_.tr;
    ++apps_;
    if (kind_ == SDG_DIST_AMG) {
        d_->apply(r, z);
        return;
    }
    const int nv = s_.n_v_loc, nff = s_.n_v_loc + s_.n_pff_loc;
    v_->apply(r, z);                                              // z_v = Vtilde^{-1} r_v
    const double* zx = c_.load(cx, tr, z);
    launch_uzawa_pressure(cx, c_.a, zx, r + nv, omega_, z + nv);  // z_p = omega (C z_v - r_p)
    if (kind_ == SDG_DIST_UZAWA) return;
    if (kind_ == SDG_TD_BGS) {                                    // precond.cpp:339-345
        cp_.apply_add(cx, tr, z, r + nff, tmp_.get(), -1.0);
        d_->apply(tmp_.get(), z + nff);
    } else {
        d_->apply(r + nff, z + nff);
    }
}

// ---------------------------------------------------------------------------
// PD-GMRES over strips (krylov.cpp:47-184; CGS2 as in krylov.cu)

SolveOut dist_pd_gmres(DistSystem& S, DistTd* P, const double* b, double* x, double tol_abs, int max_restarts,
                       Restart ctrl) {
    Context& c = *S.ctx;
    Transport& t = *S.tr;
    const int n = S.n_local();
    const int m_cap = std::max(ctrl.m_max, ctrl.current_m);
    if (m_cap + 1 > 64) fail(SDG_EINVAL, "pd_gmres: restart length above 63 is not supported");
    auto t0 = std::chrono::steady_clock::now();
    (void)t0;
    cudaEvent_t ea, eb;
    SDG_CUDA(cudaEventCreate(&ea));
    SDG_CUDA(cudaEventCreate(&eb));
    SDG_CUDA(cudaEventRecord(ea, c.stream));

    SolveOut out;
    const int nn = std::max(n, 1);
    const int64_t ld = (static_cast<int64_t>(nn) + 31) / 32 * 32;
    DevBuf<double> basis(static_cast<size_t>(ld) * (m_cap + 1));
    DevBuf<double> r(nn), z(nn), w(nn), best_x(nn), dd(4 * 64);
    ReduceWs ws;
    ws.init(reduce_blocks(nn, c.num_sms), 64, c.stream);
    double* h1 = dd.get();
    double* h2 = dd.get() + 64;
    double* sc = dd.get() + 128;
    double* yv = dd.get() + 192;
    double hh[64], up[64];
    double* hcol = c.pinned->as<double>() + 2048;  // h1 | h2 | ||w|| read-back of one step
    auto precond = [&](const double* in, double* o) {
        if (P)
            P->apply(in, o);
        else
            launch_copy(c, o, in, n);
    };
    auto upload = [&](double* dev, const double* host, int k) {
        SDG_CUDA(cudaMemcpyAsync(dev, host, sizeof(double) * k, cudaMemcpyHostToDevice, c.stream));
        c.sync();  // host buffer is reused
    };

    launch_fill(c, x, 0.0, n);
    launch_copy(c, r.get(), b, n);
    launch_norm2sq(c, ws, n, r.get(), sc);
    t.allreduce(c, sc, 1, hh);
    double res_norm = std::sqrt(hh[0]);
    out.history.push_back(res_norm);
    auto finish = [&]() {
        SDG_CUDA(cudaEventRecord(eb, c.stream));
        SDG_CUDA(cudaEventSynchronize(eb));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ea, eb);
        out.device_ms = ms;
        cudaEventDestroy(ea);
        cudaEventDestroy(eb);
    };
    if (res_norm <= tol_abs) {
        out.converged = true;
        out.final_residual = res_norm;
        finish();
        return out;
    }
    double prev_cycle_res = res_norm;
    launch_copy(c, best_x.get(), x, n);
    double best_res = res_norm;
    bool trust_estimate = true;

    for (int cycle = 0; cycle < max_restarts; ++cycle) {
        const int m = ctrl.current_m;
        std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0);
        auto hij = [&](int i, int j) -> double& { return H[static_cast<size_t>(j) * (m + 1) + i]; };
        std::vector<double> g(m + 1, 0.0), cs(m, 0.0), sn(m, 0.0);
        g[0] = res_norm;
        up[0] = res_norm;
        upload(sc + 1, up, 1);
        launch_scale_by_inv(c, n, r.get(), sc + 1, basis.get());
        int used = 0;
        bool basis_exhausted = false;
        for (int i = 0; i < m; ++i) {
            // the Arnoldi step runs on the device end to end: each CGS2 pass's
            // partial dots are all-gathered and folded in rank order by a
            // kernel (Transport::allreduce_device), and the host reads the
            // Hessenberg column once per step
            const double* vi = basis.get() + ld * i;
            precond(vi, z.get());
            S.A.apply(c, t, z.get(), w.get());
            launch_multidot(c, ws, n, i + 1, basis.get(), ld, w.get(), h1);
            t.allreduce_device(c, h1, i + 1, h1);
            launch_multi_axpy(c, n, i + 1, basis.get(), ld, h1, w.get());
            launch_multidot(c, ws, n, i + 1, basis.get(), ld, w.get(), h2);
            t.allreduce_device(c, h2, i + 1, h2);
            launch_multi_axpy(c, n, i + 1, basis.get(), ld, h2, w.get());
            launch_norm2sq(c, ws, n, w.get(), sc);
            t.allreduce_device(c, sc, 1, sc, /*take_sqrt=*/true);
            launch_scale_by_inv(c, n, w.get(), sc, basis.get() + ld * (i + 1));
            SDG_CUDA(cudaMemcpyAsync(hcol, dd.get(), sizeof(double) * 129, cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            for (int k = 0; k <= i; ++k) hij(k, i) += hcol[k];
            for (int k = 0; k <= i; ++k) hij(k, i) += hcol[64 + k];
            const double wn = hcol[128];
            hij(i + 1, i) = wn;
            for (int k = 0; k < i; ++k) {
                const double a0 = cs[k] * hij(k, i) + sn[k] * hij(k + 1, i);
                const double a1 = -sn[k] * hij(k, i) + cs[k] * hij(k + 1, i);
                hij(k, i) = a0;
                hij(k + 1, i) = a1;
            }
            const double denom = std::hypot(hij(i, i), hij(i + 1, i));
            if (denom == 0.0) fail(SDG_ESINGULAR, "pd_gmres: singular Hessenberg block");
            cs[i] = hij(i, i) / denom;
            sn[i] = hij(i + 1, i) / denom;
            hij(i, i) = denom;
            hij(i + 1, i) = 0.0;
            g[i + 1] = -sn[i] * g[i];
            g[i] = cs[i] * g[i];
            ++out.iterations;
            ++used;
            const double est = std::abs(g[i + 1]);
            out.history.push_back(est);
            if (trust_estimate && est <= tol_abs) break;
            if (wn == 0.0) {
                basis_exhausted = true;
                break;
            }
        }
        std::vector<double> y(used, 0.0);
        for (int i = used - 1; i >= 0; --i) {
            double sum = g[i];
            for (int j = i + 1; j < used; ++j) sum -= hij(i, j) * y[j];
            if (hij(i, i) == 0.0) fail(SDG_ESINGULAR, "pd_gmres: singular Hessenberg block");
            y[i] = sum / hij(i, i);
        }
        std::copy(y.begin(), y.end(), up);
        upload(yv, up, std::max(used, 1));
        launch_lincomb(c, n, used, basis.get(), ld, yv, w.get());
        precond(w.get(), z.get());
        launch_add_inplace(c, n, x, z.get());
        S.A.apply_add(c, t, x, b, r.get(), -1.0);  // r = b - A x
        launch_norm2sq(c, ws, n, r.get(), sc);
        t.allreduce(c, sc, 1, hh);
        res_norm = std::sqrt(hh[0]);
        if (res_norm < best_res) {
            best_res = res_norm;
            launch_copy(c, best_x.get(), x, n);
        }
        if (trust_estimate && used < m && res_norm > tol_abs) trust_estimate = false;
        const double rate = std::log10(std::max(res_norm, 1e-300) / std::max(prev_cycle_res, 1e-300));
        ctrl.update(rate);
        prev_cycle_res = res_norm;
        if (res_norm <= tol_abs || basis_exhausted) break;
    }
    if (best_res < res_norm) {
        launch_copy(c, x, best_x.get(), n);
        res_norm = best_res;
    }
    out.history.push_back(res_norm);
    out.final_residual = res_norm;
    out.converged = res_norm <= tol_abs;
    finish();
    return out;
}

// ---------------------------------------------------------------------------
// BiCGSTAB over strips (krylov.cpp:186-292): host scalars, reductions as
// deterministic all-gathers of per-rank partials

SolveOut dist_bicgstab(DistSystem& S, DistTd* P, const double* b, double* x, double tol_abs, int max_iters) {
    Context& c = *S.ctx;
    Transport& tr = *S.tr;
    const int n = S.n_local();
    const int nn = std::max(n, 1);
    cudaEvent_t ea, eb;
    SDG_CUDA(cudaEventCreate(&ea));
    SDG_CUDA(cudaEventCreate(&eb));
    SDG_CUDA(cudaEventRecord(ea, c.stream));
    SolveOut out;
    DevBuf<double> r(nn), rhat(nn), p(nn), vv(nn), s(nn), phat(nn), shat(nn), t(nn), rt(nn), part(4);
    ReduceWs ws;
    ws.init(reduce_blocks(nn, c.num_sms), 2, c.stream);
    double hv[4];
    auto precond = [&](const double* in, double* o) {
        if (P)
            P->apply(in, o);
        else
            launch_copy(c, o, in, n);
    };
    auto dot1 = [&](const double* a, const double* bb) {
        launch_dot(c, ws, n, a, bb, part.get());
        tr.allreduce(c, part.get(), 1, hv);
        return hv[0];
    };
    auto norm = [&](const double* a) {
        launch_norm2sq(c, ws, n, a, part.get());
        tr.allreduce(c, part.get(), 1, hv);
        return std::sqrt(hv[0]);
    };
    auto residual = [&](double* dst) { S.A.apply_add(c, tr, x, b, dst, -1.0); };
    const int g = nblk(n);

    launch_fill(c, x, 0.0, n);
    launch_copy(c, r.get(), b, n);
    double res_norm = norm(r.get());
    out.history.push_back(res_norm);
    auto finish = [&]() {
        SDG_CUDA(cudaEventRecord(eb, c.stream));
        SDG_CUDA(cudaEventSynchronize(eb));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ea, eb);
        out.device_ms = ms;
        cudaEventDestroy(ea);
        cudaEventDestroy(eb);
    };
    if (res_norm <= tol_abs) {
        out.converged = true;
        out.final_residual = res_norm;
        finish();
        return out;
    }
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    auto reset = [&]() {
        launch_copy(c, rhat.get(), r.get(), n);
        launch_fill(c, p.get(), 0.0, n);
        launch_fill(c, vv.get(), 0.0, n);
        rho = alpha = omega = 1.0;
    };
    reset();
    int restarts = 0, replacements = 0;
    bool done = false;
    auto hard_restart = [&]() {
        if (++restarts > 1) fail(SDG_EBREAKDOWN, "bicgstab: repeated breakdown");
        residual(r.get());
        reset();
    };
    auto confirmed = [&]() {
        residual(rt.get());
        const double tn = norm(rt.get());
        if (tn <= tol_abs) return true;
        if (replacements++ < 3) {
            launch_copy(c, r.get(), rt.get(), n);
            reset();
            return false;
        }
        done = true;
        return false;
    };
    for (int iter = 0; iter < max_iters && !done; ++iter) {
        const double rho_new = dot1(rhat.get(), r.get());
        if (std::abs(rho_new) < 1e-300) {
            hard_restart();
            continue;
        }
        const double beta = (rho_new / rho) * (alpha / omega);
        launch_k(c, k_dbi_p, g, kT, 0, n, beta, omega, r.get(), vv.get(), p.get());
        c.count();
        precond(p.get(), phat.get());
        S.A.apply(c, tr, phat.get(), vv.get());
        const double rv = dot1(rhat.get(), vv.get());
        if (std::abs(rv) < 1e-300) {
            hard_restart();
            continue;
        }
        alpha = rho_new / rv;
        launch_k(c, k_dbi_s, g, kT, 0, n, alpha, r.get(), vv.get(), s.get());
        c.count();
        ++out.iterations;
        const double sn = norm(s.get());
        if (sn <= tol_abs) {
            launch_k(c, k_daxpy, g, kT, 0, n, alpha, phat.get(), x);
            c.count();
            out.history.push_back(sn);
            if (confirmed()) break;
            continue;
        }
        precond(s.get(), shat.get());
        S.A.apply(c, tr, shat.get(), t.get());
        launch_dot(c, ws, n, t.get(), t.get(), part.get());
        launch_dot(c, ws, n, t.get(), s.get(), part.get() + 1);
        tr.allreduce(c, part.get(), 2, hv);
        const double tt = hv[0];
        if (tt == 0.0) {
            hard_restart();
            continue;
        }
        omega = hv[1] / tt;
        if (std::abs(omega) < 1e-300) {
            hard_restart();
            continue;
        }
        launch_k(c, k_dbi_xr, g, kT, 0, n, alpha, omega, phat.get(), shat.get(), s.get(), t.get(), x, r.get());
        c.count();
        rho = rho_new;
        res_norm = norm(r.get());
        out.history.push_back(res_norm);
        if (res_norm <= tol_abs && confirmed()) break;
    }
    residual(rt.get());
    const double fin = norm(rt.get());
    out.final_residual = fin;
    out.history.push_back(fin);
    out.converged = fin <= tol_abs;
    finish();
    return out;
}

}  // namespace sdg
