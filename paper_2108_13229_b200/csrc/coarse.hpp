// Coarsest-level direct solve (the reference's lu_factor / lu_solve,
// lu.cpp:91-203, used by amg_setup precond.cpp:215 and vcycle precond.cpp:235).
//
// The reference factors the coarsest matrix with a sparse LU and runs two
// sequential triangular solves per V-cycle.  On the GPU a triangular solve is
// a latency chain, so the solve is reorganised as a nested-dissection block
// elimination whose every step is a batch of small dense products:
//
//   order the unknowns  [ subtree(A) | subtree(B) | separator S ]  recursively
//   (post-order), so the interior I of a tree node is a contiguous range that
//   is followed by its separator.  With  A = [A_II A_IS; A_SI A_SS]:
//       y_I = A_II^{-1} b_I                       (the two subtrees, recursively)
//       x_S = Sc^{-1} (b_S - A_SI y_I),   Sc = A_SS - A_SI A_II^{-1} A_IS
//       x_I = y_I - W x_S,                W  = A_II^{-1} A_IS
//   Leaves keep the explicit inverse of their diagonal block, internal nodes
//   keep Sc^{-1} (dense |S|^2) and W (dense |I| x |S|); A_SI stays sparse.
//
// One solve is 1 + 2 * depth launches (leaves; then per depth, bottom-up, the
// separator solves and the W corrections), each fully parallel, and reads
// ~ n^2 / 2^depth + n * sum|S| doubles instead of the n^2 of one dense
// inverse (c3 velocity: 1.2 GB -> ~0.1 GB; c4 porous: 9.9 GB -> ~0.3 GB).
// Small systems (n < kNdMinRows) keep one dense inverse: a single leaf.
//
// All dense inverses are computed on the device by a batched in-place
// Gauss-Jordan elimination with partial pivoting (coarse.cu); nothing here
// calls a library.  A singular block (possible for an indefinite matrix even
// when the matrix itself is regular) makes build() fall back to the dense
// inverse of the whole matrix, which pivots like the reference's lu_factor.
#pragma once

#include <vector>

#include "common.hpp"

namespace sdg {

struct NdNode {
    int lo = 0, mid = 0, hi = 0;   // interior [lo, mid), separator [mid, hi) in the new numbering
    int depth = 0;
    int left = -1, right = -1;     // children (-1: leaf; a leaf has mid == hi and owns [lo, hi))
    bool leaf() const { return left < 0; }
};

struct NdTree {
    std::vector<int> perm;         // new index -> old index
    std::vector<NdNode> nodes;     // post-order: children before parents, root last
    int max_depth = 0;             // depth of the deepest node
};

constexpr int kNdMinRows = 3000;   // below this one dense inverse is cheaper than the extra launches
constexpr int kNdLeafRows = 1024;  // split while a node has more rows than this

// Nested-dissection ordering of the symmetrised graph of `a` by breadth-first
// level sets from a pseudo-peripheral vertex: the separator is the median
// level, thinned to the vertices that see the next level.
NdTree nd_order(const HostCsr& a, int leaf_rows, int max_depth);

// Host evaluation of the block elimination above (dense blocks inverted by
// Gauss-Jordan with partial pivoting): the algebra check of the CPU test
// suite.  Returns false when a block is singular.
bool nd_solve_host(const HostCsr& a, const NdTree& t, const double* b, double* x);

// P A P^T for perm (new -> old), columns sorted.
HostCsr permute_symmetric(const HostCsr& a, const std::vector<int>& perm);

struct NdNodeDev {
    int lo, mid, hi, pad;
    long long inv;   // pool offset: leaf inverse (n_l^2) or Sc^{-1} (|S|^2), row-major
    long long w;     // pool offset: W (|I| x |S|, row-major); unused for leaves
};

class CoarseSolver {
public:
    void build(Context& cx, const HostCsr& a);
    // z = A^{-1} r on the context's stream
    void solve(Context& cx, const double* r, double* z);
    int n() const { return n_; }
    bool dense() const { return dense_; }
    int depth() const { return dense_ ? 0 : tree_.max_depth; }
    int64_t doubles() const { return static_cast<int64_t>(pool_.size()); }
    int64_t sparse_entries() const { return ap_.nnz; }

private:
    void build_dense(Context& cx, const HostCsr& a);
    void build_nd(Context& cx, const HostCsr& a);
    // the phases of depths > above (leaves first) on m right-hand sides, u -> y (both n x m, column-major)
    void run_phases(Context& cx, int above, const double* u, const int* perm, double* y, double* xout, int m);

    int n_ = 0;
    bool dense_ = true;
    DevBuf<double> pool_;
    NdTree tree_;
    DevCsr ap_;                           // P A P^T
    DevBuf<NdNodeDev> nodes_;
    DevBuf<int> perm_, leaf_of_;
    std::vector<DevBuf<int>> node_of_;    // per depth: row -> internal node of that depth (or -1)
    std::vector<DevBuf<int>> ids_;        // per depth: internal node ids
    std::vector<int> n_ids_, max_s_;      // per depth: node count, widest separator
    std::vector<double> bytes_sep_, bytes_down_;
    double bytes_leaf_ = 0;
    DevBuf<double> y_;
};

// Batched dense inversion in place (row-major, partial pivoting): the items'
// matrices are overwritten by their inverses.  Throws SDG_ESINGULAR naming
// `what` when a pivot column is exactly zero.
struct GjItem {
    double* a;
    int n;
};
void batched_inverse(Context& cx, const std::vector<GjItem>& items, const char* what);

}  // namespace sdg
