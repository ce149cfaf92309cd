// Strip-sharded solve across GPUs: one process per GPU,
// each rank owning one horizontal strip of the free-flow box and one of the
// porous box (rank 0 holds both strips that touch the interface).
//
// Everything is expressed over a row ownership (owner rank per global dof),
// so the same machinery serves the monolithic operator of the Krylov solve,
// every AMG level of the velocity and Darcy hierarchies (coarse ownership is
// inherited from the first fine row of each aggregate) and the coupling
// blocks C (Uzawa) and C' (td_bgs).  Per rank and operator:
//   - the owned rows, with columns renumbered [owned | ghosts] (ghosts sorted
//     by (owner, global id), entries kept in global column order so row sums
//     run in the reference's order);
//   - a halo plan: which owned values each peer needs (send lists), computed
//     from replicated knowledge of the global sparsity -- no plan exchange.
// The AMG hierarchy itself is built from the global level matrices exactly as
// amg_setup does (precond.cpp:189-217), so aggregates, Galerkin products and
// the coarsest matrix are the reference's.  What changes with P > 1 is the
// smoother: lexicographic Gauss-Seidel inside each strip, the previous
// iterate across strip boundaries (processor-block Gauss-Seidel, SURVEY.md
// §8(e): +-4 % GMRES iterations for P <= 8).  P = 1 is the single-GPU
// smoother exactly.  The coarsest level is solved redundantly on every rank
// (allgather of the coarse residual + the replicated explicit inverse).
//
// Communication goes through a Transport: a built-in NCCL one (dlopen'd
// libnccl, grouped ncclSend/ncclRecv for halos, ncclAllGather for the
// deterministic reductions) or host callbacks (the caller's own runtime,
// e.g. torch.distributed/gloo in the tests).  Reductions are deterministic:
// per-rank partials are all-gathered and folded in rank order.
#pragma once

#include <memory>
#include <vector>

#include "gs.cuh"
#include "solver.hpp"

namespace sdg {

struct Transport {
    int rank = 0;
    int size = 1;
    virtual ~Transport() = default;
    // send[soff_p .. soff_p + scount[p]) goes to p, rcount[p] doubles from p
    // land at recv + roff_p (offsets = prefix sums in peer order).  Device
    // pointers on c's device; on return the data is usable in c's stream order.
    virtual void exchange(Context& c, const double* send, const std::vector<int>& scount, double* recv,
                          const std::vector<int>& rcount) = 0;
    // recv[p * count + k] = rank p's send[k]
    virtual void allgather(Context& c, const double* send, int count, double* recv) = 0;

    // Sum of k per-rank partials (device), folded in rank order on the host.
    void allreduce(Context& c, const double* partial, int k, double* host_out);
    // The same sum folded in rank order by a device kernel into out (device;
    // may alias partial), stream-ordered: no host synchronisation.  take_sqrt:
    // out = sqrt(sum) (a norm from squared partials).
    void allreduce_device(Context& c, const double* partial, int k, double* out, bool take_sqrt = false);

private:
    DevBuf<double> gather_;
    std::vector<double> host_;
};
using TransportPtr = std::shared_ptr<Transport>;

// Calls back into the host runtime with host buffers (staged through pinned
// memory by the library).
using HostExchangeFn = sdg_host_exchange_fn;
using HostAllgatherFn = sdg_host_allgather_fn;
TransportPtr make_host_transport(int rank, int size, HostExchangeFn ex, HostAllgatherFn ag, void* user);
void nccl_unique_id(unsigned char out[128]);
TransportPtr make_nccl_transport(Context& c, const unsigned char id[128], int rank, int size);

// Owner rank of every global dof and its index among its owner's rows.
struct Ownership {
    int size = 1;
    std::vector<int> owner;
    std::vector<int> lidx;
    std::vector<std::vector<int>> owned;  // per rank, ascending global ids
    static Ownership from_owner(std::vector<int> owner, int size);
    Ownership slice(int g0, int g1) const;  // the sub-space [g0, g1), renumbered from 0
    int n() const { return static_cast<int>(owner.size()); }
};

// Halo plan of one operator on one rank.
struct Halo {
    int n_owned = 0;                 // owned entries of the column space
    std::vector<int> ghost_gid;      // sorted by (owner, gid)
    std::vector<int> rcount, scount; // per peer
    std::vector<int> send_gid;       // grouped by peer, ascending gid inside a group
    DevBuf<int> send_idx;            // owned local indices of send_gid
    DevBuf<double> send_buf;
    int n_ghost() const { return static_cast<int>(ghost_gid.size()); }
    // x_ext[0, n_owned) holds the owned values; fills x_ext[n_owned, ...)
    void update(Context& c, Transport& t, double* x_ext);
};

// Rows of `a` owned by `rank` with columns renumbered [owned | ghosts].
// Host-only (used by the C-ABI plan inspection and the CPU tests).
void build_local(const HostCsr& a, const Ownership& rows, const Ownership& cols, int rank, HostCsr& local,
                 Halo& halo);

// A distributed sparse operator: owned rows x (owned columns | ghosts).
struct DistOp {
    int n_rows = 0;
    HostCsr host;   // local rectangular matrix
    DevCsr a;
    Halo halo;
    DevBuf<double> x_ext;
    void build(Context& c, const HostCsr& global, const Ownership& rows, const Ownership& cols, int rank);
    // copies the owned x into x_ext, exchanges the ghosts, returns x_ext
    double* load(Context& c, Transport& t, const double* x);
    void apply(Context& c, Transport& t, const double* x, double* y);
    void apply_add(Context& c, Transport& t, const double* x, const double* y_in, double* y_out, double alpha);
};

// Aggregation AMG V(1,1) (precond.cpp:233-259) over strips.
class DistAmg {
public:
    DistAmg(CtxPtr c, TransportPtr t, const HostCsr& a, const Ownership& own, const AmgOpts& o);
    int rows() const { return n_rows_; }
    void apply(const double* r, double* z) { vcycle(0, r, z); }
    int num_levels() const { return n_levels_; }

private:
    struct Level {
        DistOp A;
        DevCsr G;                         // owned rows x ghost columns (post-smoother)
        GsPlan gs;
        bool fast = false;
        DevBuf<int> lvl_ptr, lvl_rows;    // bitwise smoother schedule (owned lower triangle)
        int n_sched = 0;
        // restriction / prolongation with the next level
        int n_c_owned = 0, n_c_remote = 0;
        DevBuf<int> pt_ptr, pt_rows;      // (owned coarse | remote slots) -> local fine rows
        std::vector<int> rem_scount;      // remote slots per owning peer
        std::vector<int> rem_rcount;      // contributions received per peer
        DevBuf<int> add_ptr, add_src;     // owned coarse -> positions in recv_buf (peer order)
        DevBuf<int> back_idx;             // owned coarse values returned to contributors
        DevBuf<double> rc_ext, recv_buf, back_buf, zc_ext;
        DevBuf<int> agg_local;            // owned fine row -> zc_ext index
        std::vector<int> c_ext_gid;       // global ids of zc_ext entries
        DevBuf<int> c_ext_gid_dev;
        DevBuf<double> zt_ext, reff, z_own;
    };
    void vcycle(int l, const double* r, double* z);
    void coarse_solve(const double* r_owned);

    CtxPtr ctx_;
    TransportPtr tr_;
    int n_rows_ = 0;
    int n_levels_ = 0;
    std::vector<Level> lv_;
    // coarsest level, solved redundantly on every rank
    int n_c_ = 0, c_max_ = 0, c_owned_ = 0;
    CoarseSolver coarse_;
    DevBuf<double> c_send_, c_gather_, c_full_, c_sol_;
    DevBuf<int> c_slot_gid_;              // gathered slot -> global coarse id (-1 = padding)
    DevBuf<int> c_own_gid_;               // owned coarse rows (global ids), when the hierarchy has one level
};

// The whole system on one rank: monolithic operator + layout.
struct DistSystem {
    CtxPtr ctx;
    TransportPtr tr;
    HostCsr global;   // replicated assembled system (host)
    int n_u = 0, n_vel = 0, n_pff = 0, n_ppm = 0;
    Ownership own;
    DistOp A;
    int n_v_loc = 0, n_pff_loc = 0, n_ppm_loc = 0;
    int n_local() const { return A.n_rows; }
};

// td_bj / td_bgs(Uzawa(AMG_V), AMG_D') over strips (bench.cpp:121-182,
// precond.cpp:264-299, 339-345).
class DistTd {
public:
    DistTd(DistSystem& s, int kind, int v_levels, int d_levels, double omega_override);
    void apply(const double* r, double* z);
    double omega() const { return omega_; }
    int64_t applications() const { return apps_; }
    double setup_seconds = 0.0;

private:
    DistSystem& s_;
    int kind_;
    std::unique_ptr<DistAmg> v_, d_;
    DistOp c_, b_, cp_;
    double omega_ = 1.0;
    DevBuf<double> tmp_;
    int64_t apps_ = 0;
};

// pd_gmres (krylov.cpp:47-184) over strips; vectors are the rank's owned rows.
SolveOut dist_pd_gmres(DistSystem& s, DistTd* p, const double* b, double* x, double tol_abs, int max_restarts,
                       Restart ctrl);

// bicgstab (krylov.cpp:186-292) over strips.
SolveOut dist_bicgstab(DistSystem& s, DistTd* p, const double* b, double* x, double tol_abs, int max_iters);

// Horizontal strips of the n x n free-flow box (rank r: cell rows of strip r
// from the bottom) and of the porous box (rank r: strip r from the top).
std::vector<int> strip_partition(int n, int size);

}  // namespace sdg
