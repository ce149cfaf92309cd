// Fast lexicographic Gauss-Seidel for the AMG smoother (precond.cpp:92-108,
// omega = 1).  One forward sweep  z_new = (D + L)^{-1} (r - U z_old)  is
// split into
//   prep  (all SMs, bandwidth-bound): b_i = (r_i - sum_{j>i} a_ij z_old_j) / d_i
//         written straight into the level-ordered packed buffer; for the
//         post-smoother z_old = z + P zc, i.e. the prolongation is fused here;
//   lower (latency-bound): the exact lexicographic recurrence
//         z_i = b_i - sum_{j<i} (a_ij / d_i) z_j.
//
// The lower solve is chosen per matrix by GsPlan::build, in this order:
//   * a merged single-CTA walk (gs.cu merge_levels): k dependency levels per
//     group, rows substituted inside a group, prep b' = W r - WU z_old;
//   * a single-CTA walk (gs_walk.cu): the level-ordered records streamed into
//     shared memory by TMA bulk copies from a producer thread, recent z values
//     in a shared-memory ring, per level gathers -> FMAs -> ring store ->
//     named-barrier hand-off;
//   * one such walk per labelled block (u, v) in sequence with a coupling
//     step, when the whole matrix does not fit one CTA's shared memory;
//   * the banded cluster kernel (gs.cu k_gs_cluster): B bands on a
//     thread-block cluster, values crossing bands pushed with DSMEM st.async
//     packets completing single-use mbarriers, bands as a skewed pipeline.
// Structured finest levels (MAC velocity, 5-point TPFA) take the multi-SM
// wavefront instead (gs_wave.cu, tried first; SDG_GS_WAVE=0 disables).
// Opt-in experiment: the 2-CTA pipe (SDG_GS_PIPE=1).  Every variant keeps
// the exact lexicographic order.
//
// Arithmetic is reassociated versus the reference (upper part first, 1/d
// folded into the coefficients), so results agree to rounding; the BITWISE
// single-CTA kernel (kernels.cu, k_gs_levels) remains the checker path of
// sdg_sor_sweep and SDG_GS_EXACT=1.
#pragma once

#include <memory>
#include <vector>

#include "common.hpp"
#include "setup.hpp"

namespace sdg {

struct GsPlan {
    int n = 0;
    int bands = 1;          // = cluster size of the lower kernel
    int n_levels = 0;       // sum over bands of band levels (+1 export level when banded)
    int max_band_levels = 0;
    int nthreads = 64;
    int ring = 0;           // local z ring per band, power of two
    int halo = 0;           // imported boundary values per band (max)
    int depth = 0;          // segments in flight (D)
    int max_seg = 0;        // bytes of the largest chunk
    int max_packets = 1;    // imported DSMEM packets per band (max)
    size_t smem = 0;        // dynamic shared memory of the lower kernel
    bool usable = false;    // false -> fall back to the bitwise kernel
    int64_t lower_entries = 0;
    int64_t cross_refs = 0;
    int64_t global_refs = 0;
    int meta_bytes_ = 0, chunk_tab_bytes_ = 0, pbar_bytes_ = 0;
    bool walk = false;         // single-CTA walk (gs_walk.cu) instead of the banded cluster kernel
    int walk_meta_bytes = 0, walk_chunk_bytes = 0, walk_zbytes = 0, walk_chunks = 0;
    int walk_r2 = 1, walk_r8 = 0;  // rows per consumer thread and level (<= 2-entry / wider rows)
    int walk_kw = 8;               // entries of a wide record (6 or 8)
    DevBuf<int4> walk_iss;     // per chunk {global off16, bytes, stage off, issue after level}
    DevBuf<int4> meta;         // per (band, level) {chunk-local off16, nS | global flag << 31, nL | nE << 16, chunk}
    DevBuf<int4> chunk_tab;    // per (band, chunk) {off16, bytes16, first level, levels}
    DevBuf<int4> band_info;    // per band {meta base, n levels, packet base, n packets}, then {chunk base, n chunks}
    DevBuf<int> req_ptr;       // per (band, level) + 1: CSR into req
    DevBuf<int> req;           // band-local packet ids a level waits for
    DevBuf<int> packet_bytes;  // expected bytes per packet (all bands)
    DevBuf<double> packed;     // all segments, 16-byte aligned
    DevBuf<int> bidx;          // natural row -> index (in doubles) of its b slot
    DevBuf<double> dinv;
    DevCsr upper;              // strict upper triangle (natural order), unscaled

    // Block forward substitution over contiguous label blocks, used when the
    // whole lower solve does not fit one walk (exact: every row of block k
    // precedes every row of block k+1).  parts[k] walks rows
    // [part_r0[k], part_r0[k+1]); before it, couple[k] (rows of block k,
    // columns of the earlier blocks, values -a_ij / d_i) adds the earlier
    // blocks' new values to its b.  All records live in this plan's `packed`.
    std::vector<std::unique_ptr<GsPlan>> parts;
    std::vector<int> part_r0;
    std::vector<DevCsr> couple;
    bool pipe = false;   // two parts walked concurrently on a 2-CTA cluster (no coupling step)
    int walk_role = 0;   // WalkArgs::role of a pipe part
    int walk_roles = 0;  // WalkArgs::roles (small / wide rows on separate warps)
    int walk_import_base = 0;  // first import slot of a walk (pipe role 2)
    int walk_n_peer = 0, walk_pbar_bytes = 0;
    DevBuf<int> walk_peer_bytes;  // pipe role 2: bytes the peer pushes at each of its levels
    // multi-SM wavefront lower solve of a structured finest level (gs_wave.cu);
    // its records (b and the scaled lower coefficients) live in `packed`
    bool wave = false;
    int wave_kind = 0;                   // 1: 5-point grid, 2: MAC velocity (u and v rows in one pass)
    int wave_nx = 0, wave_ny = 0;        // grid columns (m for MAC) / grid rows
    int wave_bands = 0, wave_blocks = 0, wave_w = 1;  // wave_w: bands (warps) per CTA
    size_t wave_smem = 0;
    bool wave_split = false;             // MAC: u and v recurrences on separate warps (k_gs_wave_mac)
    DevBuf<unsigned long long> wave_ticket;  // band tickets handed out (gs_wave.cu)
    DevBuf<double> wave_bnd;                 // band boundary rows, two parities, sentinel until written
    // multi-SM lattice lower solve of an aggregated coarse level (gs_lattice.cu);
    // records in `packed`
    bool lattice = false;
    int lat_bands = 0, lat_blocks = 0, lat_w = 1, lat_depth = 4;  // lat_w bands (warps) per CTA
    size_t lat_smem = 0;
    DevBuf<int> lat_win;                     // per (band, block): first window step of the previous band
    DevBuf<unsigned long long> lat_ticket;   // band tickets handed out
    DevBuf<double> lat_bnd;                  // last-chain values of every band, two parities, sentinel until written
    // per row: 1 when it has entries left of the diagonal (its lower solve reads other rows)
    std::vector<unsigned char> row_has_lower;
    bool lattice_off_ = false;  // SDG_GS_LATTICE=0 (build_parts asks its parts too)
    int lattice_mode_ = 0;      // 0 off, 1 wherever the level is a lattice, 2 the faster of walk and lattice (timed)
    Context* tune = nullptr;    // set by the owner before build(): lets the planner time candidate plans
    // level merging (gs.cu, merge_levels): groups of k consecutive dependency
    // levels are walked as one; rows inside a group are substituted into each
    // other, so the walk reads only earlier groups and the prep computes the
    // group-local combination  b' = W r - WU z_old  instead of (r - U z_old)/d
    bool merged = false;
    int merge_k = 1;
    DevCsr wmat, wumat;
    // a label block walked over merged levels (build_parts): the parent's prep / coupling steps
    // write the plain b = (r - U z_old - L_prev z_new) / d into a temporary region of the parent's
    // buffer (part_tmp_off), k_gs_tapply turns it into the group-local combination b' = T b
    // inside the walk's records (through part_bidx), then the walk over the merged rows runs
    bool merged_part = false;
    DevCsr tmat;
    DevBuf<int> part_bidx;       // local row -> slot of b' in the parent's buffer
    size_t part_tmp_off = 0;     // first temporary slot in the parent's buffer (local row i -> + i)
    const double* packed_ptr = nullptr;  // records of a part inside its parent's buffer
    size_t part_doubles = 0;             // size of a part's records

    // components: per-row labels (e.g. u = 0 / v = 1 of the MAC velocity
    // block) so that bands cut every component at the same relative height.
    // allow_merge: the caller runs launch_gs_prep_pre for every sweep that
    // starts from z = 0 (no restriction seeding into a merged plan)
    void build(const HostCsr& a, const std::vector<int>& components, cudaStream_t s,
               int bands_hint = 0, bool allow_merge = false);
    double packed_bytes() const {
        return static_cast<double>(packed_ptr ? part_doubles : packed.size()) * 8.0;
    }
    const double* records() const { return packed_ptr ? packed_ptr : packed.get(); }
    // a plain walk, or label-block walks: launch_gs_lower can record its mark
    // after the last write to packed (prep, coupling steps) and before the last walk
    bool can_mark() const {
        if (pipe || merged) return false;
        if (parts.empty()) return (walk || wave) && !merged;
        for (const auto& p : parts)
            if (!p->walk || !p->parts.empty() || p->merged) return false;
        return true;
    }

    // optional inputs / outputs of build_walk for the parts of a pipe
    struct Link {
        int force_w = 0, force_r2 = 0, force_r8 = 0, force_kw = 0;  // shape (0: the cost model's)
        int role = 0;
        const std::vector<int>* export_slot = nullptr;  // role 1: per row, import slot in the peer (-1 none)
        const std::vector<int>* export_need = nullptr;  // role 1: per pseudo-level, peer levels done first
        int export_base = 0;                            // role 1: the peer's first import slot
        const HostCsr* ext = nullptr;                   // role 2: rows x peer rows, lower entries to the peer
        const std::vector<int>* ext_slot = nullptr;     // role 2: peer row -> import slot
        const std::vector<int>* ext_plv = nullptr;      // role 2: peer row -> its pseudo-level
        const std::vector<int>* peer_bytes = nullptr;   // role 2: bytes pushed at each peer level
        int import_slots = 0;
        std::vector<int>* plv_out = nullptr;  // pseudo-level of every row
        int shape[4] = {0, 0, 0, 0};          // out: chosen W, R2, R8, wide width
    };

    // the lattice plan of a whole matrix (gs_lattice.cu); false if it is not one
    bool build_lattice(const HostCsr& a, const std::vector<double>& dinv_h, cudaStream_t s);

private:
    bool build_wave(const HostCsr& a, const std::vector<int>& comps, const std::vector<double>& dinv_h,
                    cudaStream_t s);
    bool build_parts(const HostCsr& a, const std::vector<int>& r0, const std::vector<double>& dinv_h,
                     cudaStream_t s);
    bool build_pipe(const HostCsr& a, const std::vector<int>& r0, const std::vector<double>& dinv_h,
                    cudaStream_t s);
    bool build_walk(const HostCsr& a, const std::vector<double>& dinv_h, const std::vector<int>& nlow, int max_k,
                    cudaStream_t s, Link* link = nullptr);
};

// host check of level merging (gs.cu): one merged forward sweep; returns the
// number of groups (-1: a row needs more than 16 entries)
int gs_merged_sweep_host(const HostCsr& a, int k, int dyn_cap, const double* r, const double* z_old,
                         double* z_new);

// dev aid (built with -DSDG_WALK_TL): walk kernel timeline, 4 words per launch
int walk_timeline(unsigned long long* out, int max);

// modelled cycles of one walk sweep over a (gs_walk.cu); 1e300 if it cannot walk
double walk_model_cost(const HostCsr& a, const std::vector<int>& nlow, int max_k);
double walk_shape_cost(const std::vector<int>& c2, const std::vector<int>& c8, int kw, int* w_out, int* r2_out,
                       int* r8_out, bool corrected);

// packed[bidx[i]] = r[i] * dinv[i]                      (pre-smoother, z_old = 0)
void launch_gs_prep_pre(Context& c, const GsPlan& g, const double* r);
// packed[bidx[i]] = (r_i - sum_{j>i} a_ij (z_j [+ zc[agg_j]])) * dinv_i
void launch_gs_prep_post(Context& c, const GsPlan& g, const double* r, const double* z,
                         const double* zc, const int* agg);
// the level walk; writes z_new (natural order)
// mark: recorded on the stream right before the last walk of the sweep is
// launched, i.e. once every packed b of the sweep is final (GsPlan::can_mark)
void launch_gs_lower(Context& c, const GsPlan& g, double* z_new, cudaEvent_t mark = nullptr);
// multi-SM wavefront variant (plans with wave == true; gs_wave.cu)
void launch_gs_wave(Context& c, const GsPlan& g, double* z_new);
// multi-SM lattice variant (plans with lattice == true; gs_lattice.cu)
void launch_gs_lattice(Context& c, const GsPlan& g, double* z_new);
// host check of the lattice planner: emulated sweep vs sequential lower solve
// (max abs difference; -1 when the matrix is not a lattice)
double lattice_check_host(const HostCsr& a, const double* b);
bool lattice_emulate_host(const HostCsr& a, const double* b, double* z);
bool lattice_run_device(Context& c, const HostCsr& a, const double* b, double* z, int repeats);
// dev aid (SDG_WAVE_TL=1): per band {start, first block, end, waiting ns} of the last wave launch
int wave_timeline_copy(unsigned long long* out, int max_bands);
int wave_blocks_copy(unsigned long long* out, int max_bands);
// single-CTA variant (plans with walk == true; gs_walk.cu)
void launch_gs_walk(Context& c, const GsPlan& g, double* z_new);
// the two parts of a pipe on a 2-CTA cluster (gs_walk.cu)
void launch_gs_pipe(Context& c, const GsPlan& g, double* z_new);
// fused residual + restriction, one warp per aggregate (bit-identical to
// precond.cpp:241-244); optionally also seeds the next level's packed b
// (rc * dinv) for its pre-smoother.
void launch_restrict_warp(Context& c, const DevCsr& a, const int* pt_ptr, const int* pt_rows,
                          int n_coarse, const double* r, const double* z, double* rc,
                          const GsPlan* next);

}  // namespace sdg
