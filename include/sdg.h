/*
 * sdg.h -- C-ABI of libsdgpu.so, the B200-native (sm_100a, fp64) replacement
 * for the reference's preconditioned Krylov path (arXiv 2108.13229 reference,
 * /root/reference/proj/core).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * Every entry point names the reference interface it replaces (file:line,
 * relative to /root/reference/proj/core).  A header-only C++ adapter that
 * turns these handles back into the reference's own types
 * (sdc::LinearOperator, sdc::Preconditioner subclasses, sdc::pd_gmres /
 * sdc::bicgstab signatures) is include/sdc_gpu.hpp; the Python mirror is
 * paper_2108_13229_b200/sdc.py.
 *
 * Memory contract (mirrors operator.hpp:30-33 and SURVEY.md §8(b)):
 *   - `*_host` pointers are borrowed for the duration of the call only;
 *   - `*_dev` pointers are device pointers on the handle's device, consumed
 *     in stream order on the handle's stream (no implicit synchronisation);
 *   - handles own their device memory; all handles created from one context
 *     share that context's CUDA stream, and calls on a context are serialised.
 *
 * Error contract: every function returning int returns SDG_OK (0) or one of
 * the codes below; sdg_last_error() returns a thread-local message.  The C++
 * adapter rethrows SDG_EDIM as std::invalid_argument and SDG_ESINGULAR /
 * SDG_EBREAKDOWN as std::runtime_error, which is what the reference throws
 * (krylov.cpp:52-55,126,150,215; precond.cpp:104-105; lu.cpp:141-143).
 */
#ifndef SDG_H
#define SDG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDG_OK 0
#define SDG_EDIM 1        /* dimension / contract violation (std::invalid_argument) */
#define SDG_ESINGULAR 2   /* zero diagonal, zero pivot, singular Hessenberg (std::runtime_error) */
#define SDG_EBREAKDOWN 3  /* repeated BiCGSTAB breakdown (std::runtime_error) */
#define SDG_ECUDA 4       /* CUDA runtime / library failure */
#define SDG_ENOMEM 5      /* device allocation failure */
#define SDG_ENCCL 6       /* NCCL failure (strip-sharded handles) */
#define SDG_EINVAL 7      /* bad handle / argument */

typedef struct sdg_context sdg_context;
typedef struct sdg_matrix sdg_matrix;
typedef struct sdg_precond sdg_precond;

/* Block preconditioner kinds: precond.hpp:162 (BlockPrecondKind). */
#define SDG_TD_BJ 0
#define SDG_TD_BGS 1
#define SDG_PV_BJ 2
#define SDG_PV_BGS 3
/* OR-ed into sdg_td_create's kind: ILU(0) instead of AMG on the grounded
 * porous block D' (the td_*_uzawa_ilu0 choices, bench.cpp:156-172) */
#define SDG_TD_ILU0 16
/* sdg_dist_td_create only: the two subdomain preconditioners of the partitioned
 * Dirichlet-Neumann driver over strips (coupling.cpp:115-146): inexact
 * Uzawa(AMG_V) on a Stokes system [V B; C 0] (n_ppm = 0), and AMG on a single
 * matrix (n_vel = n_pff = 0, no grounding: the Dirichlet Darcy problem is regular) */
#define SDG_DIST_UZAWA 32
#define SDG_DIST_AMG 33

/* RestartController (krylov.hpp:23-47). Updated in place by sdg_pd_gmres
 * only on the caller's copy semantics of the reference: the reference takes
 * the controller by value, so sdg_pd_gmres never writes it back. */
typedef struct sdg_restart {
    int m_init;
    int m_min;
    int m_step;
    int m_max;
    int current_m;
    double previous_rate;
    int has_rate_sample;
    double alpha_p;
    double alpha_d;
    double stall_threshold;
} sdg_restart;

/* SolveReport (krylov.hpp:12-18).  residual_history is caller-owned with
 * capacity history_capacity (may be NULL / 0); history_length reports the
 * full length the reference would have produced. */
typedef struct sdg_report {
    int iterations;
    int converged;
    double wall_time;       /* seconds, host clock around the whole call */
    double final_residual;
    double* residual_history;
    int history_capacity;
    int history_length;
    int64_t precond_applications; /* applications made by this solve */
    double device_ms;       /* CUDA-event time of the device-resident part */
    int breakdown;          /* warm-started BiCGSTAB only: ended by a repeated breakdown (x = last iterate) */
} sdg_report;

/* AmgOptions (precond.hpp:64-72).  components: NULL or one label per row. */
typedef struct sdg_amg_options {
    int max_levels;
    double strength_theta;
    int coarse_threshold;
    const int* components;
} sdg_amg_options;

/* UzawaConfig (precond.hpp:122-129), inexact mode only (exact mode is the
 * test-only DirectSolvePreconditioner, out of scope per SURVEY.md §2).
 * omega_override: NaN -> estimate by power iteration as the reference does
 * (precond.cpp:278-286); otherwise use the given relaxation directly. */
typedef struct sdg_uzawa_options {
    sdg_amg_options amg;
    double power_tol_rel;
    int power_max_iters;
    unsigned power_seed;
    double omega_override;
} sdg_uzawa_options;

/* Fills the reference defaults: RestartController::defaults(),
 * AmgOptions{}, UzawaConfig{}. */
void sdg_restart_defaults(sdg_restart* c);
void sdg_amg_defaults(sdg_amg_options* o);
void sdg_uzawa_defaults(sdg_uzawa_options* o);

const char* sdg_last_error(void);
const char* sdg_version(void);

/* ---- context ----------------------------------------------------------- */
int sdg_context_create(int device, sdg_context** out);
int sdg_context_destroy(sdg_context* ctx);
int sdg_context_synchronize(sdg_context* ctx);
/* The context's cudaStream_t, as void* (for callers that order their own
 * copies against the solver, e.g. the e2e bench leg). */
void* sdg_context_stream(sdg_context* ctx);
/* Number of this library's kernels launched on the context so far. */
int64_t sdg_context_launches(sdg_context* ctx);

/* Live kernel profiler.  When enabled, every launch is bracketed by CUDA
 * events on the context stream and tagged with its algorithmic bytes
 * (SURVEY.md §8(d) byte model); sdg_context_profile folds them per kernel
 * family.  Enabling clears previous totals.  Families: 0 spmv, 1 gs,
 * 2 restrict, 3 prolong, 4 coarse, 5 uzawa, 6 ortho, 7 bicg, 8 vec, 9 setup,
 * 10 gsprep, 11 spmv_block, 12 gs_wave (the multi-SM wavefront smoother of
 * the structured finest levels), 13 iface (td_bgs interface GEMV),
 * 14 gs_lattice (the multi-SM lattice smoother of the aggregated coarse levels). */
#define SDG_PROF_FAMILIES 15
int sdg_context_set_profiling(sdg_context* ctx, int enable);
int sdg_context_profile(sdg_context* ctx, int family, int64_t* launches, double* total_ms,
                        double* total_bytes);
const char* sdg_profile_family_name(int family);

/* ---- matrices / LinearOperator ------------------------------------------
 * Replaces SparseMatrix (sparse.hpp:17-46) as the operand and
 * LinearOperator::from_matrix (operator.hpp:24-27) as the operator.  CSR,
 * int32 offsets/columns, fp64 values; the host arrays are copied. */
int sdg_matrix_create(sdg_context* ctx, int n_rows, int n_cols, const int* rowptr,
                      const int* col, const double* val, sdg_matrix** out);
int sdg_matrix_destroy(sdg_matrix* a);
int sdg_matrix_rows(const sdg_matrix* a);
int sdg_matrix_cols(const sdg_matrix* a);
int64_t sdg_matrix_nnz(const sdg_matrix* a);

/* spmv (sparse.cpp:81-90): y = A x. */
int sdg_spmv(sdg_matrix* a, const double* x_host, double* y_host);
/* spmv_add (sparse.cpp:98-108): y = y + alpha A x. */
int sdg_spmv_add(sdg_matrix* a, const double* x_host, double* y_host, double alpha);
int sdg_spmv_device(sdg_matrix* a, const double* x_dev, double* y_dev);
/* sor_sweep (precond.cpp:92-108): one forward sweep, z updated in place. */
int sdg_sor_sweep(sdg_matrix* a, double* z_host, const double* r_host, double omega);

/* ---- preconditioners (operator.hpp:34-62) ------------------------------- */
/* AmgPreconditioner(a, opts) (precond.hpp:101-120): amg_setup
 * (precond.cpp:189-217) on the host, V(1,1) apply (precond.cpp:233-259) on
 * the device. */
int sdg_amg_create(sdg_matrix* a, const sdg_amg_options* opts, sdg_precond** out);
/* UzawaPreconditioner(v, b, c, cfg) (precond.cpp:264-299). */
int sdg_uzawa_create(sdg_matrix* v, sdg_matrix* b, sdg_matrix* c, const sdg_uzawa_options* cfg,
                     sdg_precond** out);
/* BlockPreconditioner(kind, matrix, n_v, n_pff, n_ppm, first, pm)
 * (precond.cpp:304-363).  Retains `first` and `pm` (shared ownership, as the
 * reference's shared_ptr<const Preconditioner>). */
int sdg_block_create(int kind, sdg_matrix* matrix, int n_v, int n_pff, int n_ppm,
                     sdg_precond* first, sdg_precond* pm, sdg_precond** out);
/* IdentityPreconditioner(n) (operator.hpp:64-76). */
/* Ilu0Preconditioner(a) (precond.hpp:18-30, precond.cpp:13-87): factors
 * bitwise the reference's; apply = the two triangular solves on the device. */
int sdg_ilu0_create(sdg_matrix* a, sdg_precond** out);
int sdg_identity_create(sdg_context* ctx, int n, sdg_precond** out);
/* ground_dof (precond.cpp:375-392) applied on the host to a CSR copy. */
int sdg_ground_dof_host(int n, const int* rowptr, const int* col, double* val_inout, int dof);

/* Host check of the fast smoother's level merging (no GPU): one forward
 * Gauss-Seidel sweep (precond.cpp:92-108, omega = 1, z_old may be NULL = 0)
 * evaluated in the merged form the device walk uses, with groups of k
 * dependency levels (dyn_cap > 0: dynamic groups of <= k levels whose rows
 * keep <= dyn_cap entries).  *groups receives the group count.  Equal to the
 * plain sweep up to rounding. */
int sdg_gs_merged_sweep_host(int n, const int* rowptr, const int* col, const double* val, int k, int dyn_cap,
                             const double* r, const double* z_old, double* z_new, int* groups);

/* The whole MonolithicDriver::build_preconditioner wiring (bench.cpp:121-182)
 * for kind td_bj / td_bgs in one call: D' = ground_dof(A[pm,pm]), V labels
 * u = 0 / v = 1, Uzawa(AMG_V) on [v | p_ff], AMG on D'.  v_max_levels /
 * d_max_levels set AmgOptions.max_levels of the two hierarchies (SURVEY.md
 * §8(d) makes them per-config parity inputs).  omega_override as above. */
int sdg_td_create(sdg_matrix* a, int n_u, int n_vel, int n_pff, int n_ppm, int kind,
                  int v_max_levels, int d_max_levels, double omega_override,
                  sdg_precond** out);

int sdg_precond_destroy(sdg_precond* p);
int sdg_precond_rows(const sdg_precond* p);
/* Preconditioner::apply (operator.hpp:40-43). */
int sdg_precond_apply(sdg_precond* p, const double* r_host, double* z_host);
int sdg_precond_apply_device(sdg_precond* p, const double* r_dev, double* z_dev);
/* Preconditioner::applications() (operator.hpp:55). */
int64_t sdg_precond_applications(const sdg_precond* p);
/* setup_memory_doubles / work_per_apply (operator.hpp:51-53). */
int64_t sdg_precond_setup_memory_doubles(const sdg_precond* p);
int64_t sdg_precond_work_per_apply(const sdg_precond* p);
/* UzawaPreconditioner::omega() (precond.hpp:141); for a td_* block, the
 * omega of its Uzawa first block; NaN otherwise. */
double sdg_precond_omega(const sdg_precond* p);
/* Host seconds spent in setup (aggregation, Galerkin, coarse factor, omega). */
double sdg_precond_setup_seconds(const sdg_precond* p);
/* Hierarchy shape of an AMG handle (or of the V / D' hierarchies of a td_*
 * handle, which = 0 / 1): number of levels, rows and nnz per level. */
int sdg_precond_hierarchy(const sdg_precond* p, int which, int* n_levels, int* rows,
                          int64_t* nnz, int capacity);
/* Use CUDA-graph capture for device applies (default on). */
int sdg_precond_set_graphs(sdg_precond* p, int enable);
/* Which fast paths a handle runs (diagnostic / test query; no reference
 * counterpart).  Bits: the td_bgs interface split, the early interface
 * correction (both BlockPrecond), the multi-SM wavefront smoother on the
 * finest velocity / porous level (an AMG or Uzawa handle reports its own
 * finest level in SDG_FEAT_WAVE_V). */
#define SDG_FEAT_SPLIT 1
#define SDG_FEAT_EARLY 2
#define SDG_FEAT_WAVE_V 4
#define SDG_FEAT_WAVE_D 8
#define SDG_FEAT_LATTICE_V 16 /* a coarse velocity (or AMG handle's) level on the multi-SM lattice smoother */
#define SDG_FEAT_LATTICE_D 32
int sdg_precond_features(const sdg_precond* p, int* features);

/* ---- Krylov solvers (krylov.cpp) ----------------------------------------
 * precond may be NULL (identity, krylov.cpp:19-25).  x starts at zero
 * (krylov.cpp:58,194).  tol_abs is absolute, as in the reference. */
/* pd_gmres (krylov.hpp:57-59, krylov.cpp:47-184). */
int sdg_pd_gmres(sdg_matrix* a, sdg_precond* precond, const double* b_host, double* x_host,
                 double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep);
int sdg_pd_gmres_device(sdg_matrix* a, sdg_precond* precond, const double* b_dev,
                        double* x_dev, double tol_abs, int max_restarts,
                        const sdg_restart* ctrl, sdg_report* rep);
/* Warm-started pd_gmres (BASELINE config 4): x is the initial guess on entry
 * and the solution on exit.  Exactly the reference solve of the correction
 * (x0 = 0 is hard-coded at krylov.cpp:58): r0 = b - A x, A d = r0 with
 * tol_abs, x += d.  rep describes the correction solve. */
int sdg_pd_gmres_warm(sdg_matrix* a, sdg_precond* precond, const double* b_host, double* x_host,
                      double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep);
int sdg_pd_gmres_warm_device(sdg_matrix* a, sdg_precond* precond, const double* b_dev, double* x_dev,
                             double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep);
/* Warm-started bicgstab, same correction form (x0 = 0 at krylov.cpp:194).
 * A repeated breakdown (the reference throws, krylov.cpp:215) is reported
 * instead: rep->breakdown = 1, rep->converged = 0 and x = x0 + the last
 * iterate, so a driver can restart from there (which re-seeds the shadow
 * residual, as the reference's hard restart does). */
int sdg_bicgstab_warm(sdg_matrix* a, sdg_precond* precond, const double* b_host, double* x_host,
                      double tol_abs, int max_iters, sdg_report* rep);
int sdg_bicgstab_warm_device(sdg_matrix* a, sdg_precond* precond, const double* b_dev, double* x_dev,
                             double tol_abs, int max_iters, sdg_report* rep);
/* bicgstab (krylov.hpp:63-65, krylov.cpp:186-292). */
int sdg_bicgstab(sdg_matrix* a, sdg_precond* precond, const double* b_host, double* x_host,
                 double tol_abs, int max_iters, sdg_report* rep);
int sdg_bicgstab_device(sdg_matrix* a, sdg_precond* precond, const double* b_dev,
                        double* x_dev, double tol_abs, int max_iters, sdg_report* rep);
/* power_iteration (krylov.hpp:79-80, krylov.cpp:307-339) on y = A x. */
int sdg_power_iteration(sdg_matrix* a, double tol_rel, int max_iters, unsigned seed,
                        double* value, int* iterations, int* converged);

/* ---- host-side input producer (stays host C++) ----------
 * assemble_monolithic (assembly.cpp:327-380) on the n x n free-flow box
 * over the n x n porous square, restated in this library so the bench can
 * build inputs without the reference.  k_cell: NULL for the scalar
 * permeability `permeability` (bitwise identical to the reference), or n*n
 * per-cell porous permeabilities (row-major, j*n+i; the log-normal
 * extension of BASELINE.json configs 2/4 -- parity unpinned, see
 * DESIGN.md).  Two-phase: call with NULL outputs to get sizes. */
typedef struct sdg_scenario {
    int n;
    double permeability;
    double alpha_bj;
    double nu;
    double rho;
    double dt;      /* +inf -> stationary */
    double t_end;
    double dp_max;
    double t;       /* inflow_pressure(t) = dp_max/2 (1 - cos(pi t / t_end)) */
} sdg_scenario;

int sdg_assemble_monolithic(const sdg_scenario* sc, const double* k_cell, const double* v_prev,
                            int* n_total, int64_t* nnz, int* n_u, int* n_vel, int* n_pff,
                            int* n_ppm, int* rowptr, int* col, double* val, double* rhs);

/* ---- partitioned Dirichlet-Neumann subproblems (host, BASELINE config 5) ---
 * assemble_stokes(ff box, FlowParams, v_prev, {p_in(t), p=0, wall}, &v_gamma)
 * (assembly.cpp:287-303) and assemble_darcy(pm box, K/mu, {}, &p_gamma)
 * (assembly.cpp:305-325) on the n x n boxes; uniform permeability, bitwise
 * the reference.  Two-phase like sdg_assemble_monolithic.  The traces that
 * close the coupling loop (coupling.cpp:218-242): stokes_pressure_trace
 * (assembly.cpp:382-391) of the free-flow solution and
 * darcy_velocity_trace_dirichlet (assembly.cpp:393-402) of the porous one. */
/* The right-hand side of assemble_monolithic on the device (the matrix is
 * step-invariant, so BASELINE config 4 re-assembles only this each time step):
 * rhs_dev[n_total] from the previous velocity v_prev_dev[n_vel] (device, or NULL
 * for zero), on the context's stream; bitwise the host assembly's rhs.
 * Replaces the per-step assemble_monolithic call of MonolithicDriver::advance
 * (bench.cpp:187, assembly.cpp:327-380). */
int sdg_assemble_rhs_device(sdg_context* ctx, const sdg_scenario* sc, const double* v_prev_dev, double* rhs_dev);
/* The matrix of assemble_monolithic on the device (StokesAssembler / DarcyAssembler /
 * coupling rows, assembly.cpp:17-286 and 327-380), CSR with int32 offsets, bitwise the
 * host assembly (sdg_assemble_monolithic), with the per-cell permeability extension
 * (k_cell_dev: n*n device doubles, or NULL for the scenario's uniform K).  One thread per
 * row emits the row's contributions in the reference's order with explicitly rounded
 * operations; a count pass and a device scan give the row offsets.
 * rowptr_dev: n_total + 1 device ints, always written; *nnz receives the number of
 * entries.  col_dev / val_dev (capacity entries) are written when capacity >= *nnz; with
 * NULL col_dev / val_dev the call only counts (then size the arrays and call again). */
int sdg_assemble_matrix_device(sdg_context* ctx, const sdg_scenario* sc, const double* k_cell_dev, int* rowptr_dev,
                               int* col_dev, double* val_dev, int64_t capacity, int64_t* nnz);
int sdg_assemble_stokes(const sdg_scenario* sc, const double* v_prev, const double* v_gamma, int* n,
                        int64_t* nnz, int* rowptr, int* col, double* val, double* rhs);
int sdg_assemble_darcy(const sdg_scenario* sc, const double* p_gamma, int* n, int64_t* nnz, int* rowptr,
                       int* col, double* val, double* rhs);
int sdg_stokes_pressure_trace(const sdg_scenario* sc, const double* x_ff, double* trace);
int sdg_darcy_velocity_trace(const sdg_scenario* sc, const double* p, const double* p_gamma, double* trace);

/* ---- host-side setup inspection (no GPU needed) ----------------------------
 * The aggregation hierarchy exactly as the device preconditioner builds it
 * (amg_setup, precond.cpp:189-217, minus the coarse factorization), so the
 * setup can be checked bit for bit against the reference on a CPU-only box.
 * sdg_host_hierarchy_level: NULL outputs are skipped; n_sched_levels is the
 * Gauss-Seidel level-schedule depth of the level (0 on the coarsest). */
typedef struct sdg_host_hierarchy sdg_host_hierarchy;
int sdg_host_hierarchy_build(int n, const int* rowptr, const int* col, const double* val,
                             const sdg_amg_options* opts, sdg_host_hierarchy** out);
int sdg_host_hierarchy_levels(const sdg_host_hierarchy* h);
int sdg_host_hierarchy_level(const sdg_host_hierarchy* h, int lev, int* n, int64_t* nnz,
                             int* n_coarse, int* n_sched_levels, int* rowptr, int* col,
                             double* val, int* agg);
void sdg_host_hierarchy_destroy(sdg_host_hierarchy* h);

/* Galerkin product of an aggregation on the device (galerkin_product,
 * precond.cpp:177-185; csrc/galerkin.cu): A_c = P^T A P for agg (fine row ->
 * aggregate, n_coarse aggregates), bitwise equal to the reference's CooBuilder
 * sum order.  The device AMG setup uses it for every level.  Outputs: c_rowptr
 * (n_coarse + 1), c_col / c_val (capacity nnz(A) suffices), *c_nnz. */
int sdg_galerkin_device(sdg_context* ctx, int n, const int* rowptr, const int* col, const double* val, const int* agg,
                        int n_coarse, int* c_rowptr, int* c_col, double* c_val, int64_t* c_nnz);

/* ---- direct solve (lu.hpp:38-41: lu_factor / lu_solve) ----------------------
 * The factorization the AMG hierarchies use on their coarsest level, as its own
 * handle: a nested-dissection block elimination with explicit inverses of small
 * dense blocks (batched Gauss-Jordan with partial pivoting on the device;
 * csrc/coarse.hpp), or one dense inverse for small systems.  A singular matrix
 * returns SDG_ESINGULAR like lu_factor's std::runtime_error (lu.cpp:142).
 * sdg_lu_info: dense = 1 when a single dense inverse is kept, depth = levels of
 * the dissection, stored_doubles = dense block storage. */
typedef struct sdg_lu sdg_lu;
int sdg_lu_factor(sdg_context* ctx, int n, const int* rowptr, const int* col, const double* val, sdg_lu** out);
int sdg_lu_solve(sdg_lu* lu, const double* b_host, double* x_host);
int sdg_lu_info(const sdg_lu* lu, int* dense, int* depth, int64_t* stored_doubles);
void sdg_lu_destroy(sdg_lu* lu);

/* Host check of the coarse direct solve (no GPU): the nested-dissection block
 * elimination that replaces lu_factor / lu_solve on the coarsest AMG level
 * (lu.cpp:91-203; csrc/coarse.hpp).  Orders the matrix (nodes split while they
 * have more than leaf_rows rows, at most max_depth times), solves A x = b
 * through the ordering and reports the tree: perm (new -> old, n ints, may be
 * NULL), node count, depth, the widest separator and the doubles a device
 * build stores.  nodes_out (may be NULL, up to max_nodes x 4 ints): lo, mid,
 * hi, depth per node in post-order.  SDG_ESINGULAR when a block is singular. */
int sdg_nd_solve_host(int n, const int* rowptr, const int* col, const double* val, int leaf_rows, int max_depth,
                      const double* b, double* x, int* perm, int* n_nodes, int* depth, int* max_separator,
                      int64_t* stored_doubles, int* nodes_out, int max_nodes);

/* ---- strip-sharded multi-GPU solve ----------------------
 * One process (and one sdg_context) per GPU.  Every rank passes the same
 * assembled system and the same ownership map (owner rank per global dof;
 * sdg_strip_partition gives the horizontal strips: rank r owns free-flow
 * cell rows of strip r from the bottom and porous strip r from the top, so
 * rank 0 holds the interface).  Vectors at this boundary are the rank's own
 * rows in ascending global order (sdg_dist_local_rows).  Replaces, per rank,
 * the same reference entry points as the single-GPU calls (pd_gmres
 * krylov.hpp:57-59, BlockPreconditioner td_* precond.cpp:304-363,
 * MonolithicDriver::build_preconditioner bench.cpp:121-182).
 * The smoother is Gauss-Seidel inside each strip with the previous iterate
 * across strip boundaries (processor-block GS; identical to the single-GPU
 * smoother for one rank).  The coarsest AMG level is solved redundantly.
 *
 * Transport: NCCL (grouped send/recv for halos, all-gather for the
 * deterministic reductions), or host callbacks from the caller's runtime
 * (buffers are host memory staged by the library; return 0 on success):
 *   exchange: send[soff_p .. + send_counts[p]) to rank p, recv_counts[p]
 *             doubles from rank p into recv + roff_p (offsets = prefix sums
 *             in rank order; counts are symmetric by construction);
 *   allgather: recv[p * count + k] = rank p's send[k]. */
typedef struct sdg_transport sdg_transport;
typedef struct sdg_dist_system sdg_dist_system;
typedef struct sdg_dist_precond sdg_dist_precond;
typedef int (*sdg_host_exchange_fn)(void* user, const double* send, const int* send_counts, double* recv,
                                    const int* recv_counts);
typedef int (*sdg_host_allgather_fn)(void* user, const double* send, int count, double* recv);

int sdg_transport_create_host(int rank, int size, sdg_host_exchange_fn exchange, sdg_host_allgather_fn allgather,
                              void* user, sdg_transport** out);
/* NCCL: rank 0 creates the id, the caller distributes it (128 bytes). */
int sdg_nccl_get_unique_id(unsigned char id[128]);
int sdg_transport_create_nccl(sdg_context* ctx, const unsigned char id[128], int rank, int size,
                              sdg_transport** out);
int sdg_transport_destroy(sdg_transport* t);

/* owner[n_total] for the n x n monolithic layout (sdg_assemble_monolithic). */
int sdg_strip_partition(int n, int n_ranks, int* owner);

/* Host-only inspection (no GPU): the halo plan of the monolithic operator on
 * `rank` -- ghost columns sorted by (owner, id) with per-owner counts, and
 * the rows each peer needs from this rank, grouped by peer.  NULL outputs
 * are skipped (call once with NULL arrays to size them). */
int sdg_dist_halo_plan(int n_total, const int* rowptr, const int* col, const int* owner, int rank, int size,
                       int* n_ghost, int* ghost_gid, int* recv_counts, int* n_send, int* send_gid,
                       int* send_counts);

int sdg_dist_system_create(sdg_context* ctx, sdg_transport* tr, int n_total, const int* rowptr, const int* col,
                           const double* val, int n_u, int n_vel, int n_pff, int n_ppm, const int* owner,
                           sdg_dist_system** out);
int sdg_dist_system_destroy(sdg_dist_system* s);
int sdg_dist_local_rows(const sdg_dist_system* s, int* n_local, int* global_ids);
/* spmv (sparse.cpp:81-90) on the rank's rows; collective. */
int sdg_dist_spmv(sdg_dist_system* s, const double* x_local, double* y_local);
/* td_bj / td_bgs as sdg_td_create, over strips; or SDG_DIST_UZAWA /
 * SDG_DIST_AMG for the subdomain solves of the partitioned driver (v_max_levels
 * resp. d_max_levels set the AMG depth).  Collective.  The system must outlive
 * the preconditioner. */
int sdg_dist_td_create(sdg_dist_system* s, int kind, int v_max_levels, int d_max_levels, double omega_override,
                       sdg_dist_precond** out);
int sdg_dist_precond_destroy(sdg_dist_precond* p);
double sdg_dist_precond_omega(const sdg_dist_precond* p);
double sdg_dist_precond_setup_seconds(const sdg_dist_precond* p);
int sdg_dist_precond_apply(sdg_dist_system* s, sdg_dist_precond* p, const double* r_local, double* z_local);
/* pd_gmres over strips; collective; tol_abs is the global absolute tolerance. */
int sdg_dist_pd_gmres(sdg_dist_system* s, sdg_dist_precond* p, const double* b_local, double* x_local,
                      double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep);

/* bicgstab over strips; collective. */
int sdg_dist_bicgstab(sdg_dist_system* s, sdg_dist_precond* p, const double* b_local, double* x_local,
                      double tol_abs, int max_iters, sdg_report* rep);

/* device-pointer variants (b, x on the context's device, stream-ordered). */
int sdg_dist_pd_gmres_device(sdg_dist_system* s, sdg_dist_precond* p, const double* b_dev, double* x_dev,
                             double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep);
int sdg_dist_bicgstab_device(sdg_dist_system* s, sdg_dist_precond* p, const double* b_dev, double* x_dev,
                             double tol_abs, int max_iters, sdg_report* rep);
/* Warm-started strip solves (BASELINE config 4 over strips; MonolithicDriver::
 * advance, bench.cpp:183-238): x_dev holds this rank's rows of the previous
 * solution; the reference solve of the correction (x0 = 0 is hard-coded,
 * krylov.cpp:58/194) on r0 = b - A x, then x += d.  Collective. */
int sdg_dist_pd_gmres_warm_device(sdg_dist_system* s, sdg_dist_precond* p, const double* b_dev, double* x_dev,
                                  double tol_abs, int max_restarts, const sdg_restart* ctrl, sdg_report* rep);
int sdg_dist_bicgstab_warm_device(sdg_dist_system* s, sdg_dist_precond* p, const double* b_dev, double* x_dev,
                                  double tol_abs, int max_iters, sdg_report* rep);

#ifdef __cplusplus
}
#endif

#endif /* SDG_H */
