// Host side of the coarse direct solve (coarse.hpp): the nested-dissection
// ordering and a host evaluation of the block elimination for the CPU tests.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>

#include "coarse.hpp"

namespace sdg {

namespace {

struct Graph {
    std::vector<int> ptr, adj;  // symmetrised pattern without the diagonal
};

Graph symmetric_graph(const HostCsr& a) {
    const int n = a.n_rows;
    std::vector<int> deg(n, 0);
    for (int i = 0; i < n; ++i)
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            const int j = a.ci[k];
            if (j == i) continue;
            ++deg[i];
            ++deg[j];
        }
    Graph g;
    g.ptr.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) g.ptr[i + 1] = g.ptr[i] + deg[i];
    g.adj.resize(g.ptr[n]);
    std::vector<int> fill(g.ptr.begin(), g.ptr.end() - 1);
    for (int i = 0; i < n; ++i)
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            const int j = a.ci[k];
            if (j == i) continue;
            g.adj[fill[i]++] = j;
            g.adj[fill[j]++] = i;
        }
    // duplicates (entries present in both triangles) are harmless for the searches below
    return g;
}

class Dissector {
public:
    Dissector(const Graph& g, int n, int leaf_rows, int max_depth)
        : g_(g), leaf_rows_(leaf_rows), max_depth_(max_depth), region_(n, -1), dist_(n, -1) {}

    int dissect(std::vector<int>& verts, int depth, NdTree& t) {
        std::vector<int> a, b, s;
        if (static_cast<int>(verts.size()) > leaf_rows_ && depth < max_depth_) split(verts, a, b, s);
        NdNode nd;
        nd.depth = depth;
        nd.lo = static_cast<int>(t.perm.size());
        if (a.empty() || b.empty()) {
            std::sort(verts.begin(), verts.end());
            t.perm.insert(t.perm.end(), verts.begin(), verts.end());
            nd.mid = nd.hi = static_cast<int>(t.perm.size());
        } else {
            verts.clear();
            verts.shrink_to_fit();
            nd.left = dissect(a, depth + 1, t);
            nd.right = dissect(b, depth + 1, t);
            nd.mid = static_cast<int>(t.perm.size());
            std::sort(s.begin(), s.end());
            t.perm.insert(t.perm.end(), s.begin(), s.end());
            nd.hi = static_cast<int>(t.perm.size());
        }
        t.max_depth = std::max(t.max_depth, depth);
        t.nodes.push_back(nd);
        return static_cast<int>(t.nodes.size()) - 1;
    }

private:
    // breadth-first search inside the current region; returns the visit order
    void bfs(int root, std::vector<int>& order) {
        order.clear();
        order.push_back(root);
        dist_[root] = 0;
        for (size_t h = 0; h < order.size(); ++h) {
            const int v = order[h];
            for (int k = g_.ptr[v]; k < g_.ptr[v + 1]; ++k) {
                const int w = g_.adj[k];
                if (region_[w] == stamp_ && dist_[w] < 0) {
                    dist_[w] = dist_[v] + 1;
                    order.push_back(w);
                }
            }
        }
    }

    void split(const std::vector<int>& verts, std::vector<int>& a, std::vector<int>& b, std::vector<int>& s) {
        ++stamp_;
        for (int v : verts) {
            region_[v] = stamp_;
            dist_[v] = -1;
        }
        std::vector<int> order;
        bfs(verts[0], order);
        if (order.size() < verts.size()) {
            // disconnected: whole components go to the lighter side, no separator
            std::vector<std::vector<int>> comps;
            comps.push_back(order);
            for (int v : verts)
                if (dist_[v] < 0) {
                    bfs(v, order);
                    comps.push_back(order);
                }
            std::sort(comps.begin(), comps.end(),
                      [](const std::vector<int>& x, const std::vector<int>& y) { return x.size() > y.size(); });
            for (auto& c : comps) {
                auto& side = a.size() <= b.size() ? a : b;
                side.insert(side.end(), c.begin(), c.end());
            }
            return;
        }
        // pseudo-peripheral root: restart twice from the farthest vertex
        for (int pass = 0; pass < 2; ++pass) {
            const int far = order.back();
            for (int v : verts) dist_[v] = -1;
            bfs(far, order);
        }
        const int depth = dist_[order.back()];
        if (depth < 2) return;  // no level can separate two non-empty sides
        std::vector<int> count(depth + 1, 0);
        for (int v : verts) ++count[dist_[v]];
        int d = 0, cum = 0;
        const int half = static_cast<int>(verts.size()) / 2;
        for (; d <= depth; ++d) {
            cum += count[d];
            if (cum >= half) break;
        }
        d = std::min(std::max(d, 1), depth - 1);
        for (int v : verts) {
            if (dist_[v] < d) {
                a.push_back(v);
            } else if (dist_[v] > d) {
                b.push_back(v);
            } else {
                bool sees_next = false;
                for (int k = g_.ptr[v]; k < g_.ptr[v + 1] && !sees_next; ++k) {
                    const int w = g_.adj[k];
                    sees_next = region_[w] == stamp_ && dist_[w] == d + 1;
                }
                (sees_next ? s : a).push_back(v);
            }
        }
    }

    const Graph& g_;
    int leaf_rows_, max_depth_;
    std::vector<int> region_, dist_;
    int stamp_ = 0;
};

// in-place Gauss-Jordan inverse with partial pivoting (row-major n x n);
// the same operation sequence as the device kernels of coarse.cu
bool gj_inverse_host(std::vector<double>& m, int n) {
    std::vector<int> piv(n);
    std::vector<double> row(n), col(n);
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::fabs(m[static_cast<size_t>(k) * n + k]);
        for (int i = k + 1; i < n; ++i) {
            const double v = std::fabs(m[static_cast<size_t>(i) * n + k]);
            if (v > best) {
                best = v;
                p = i;
            }
        }
        if (best == 0.0) return false;
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < n; ++j) std::swap(m[static_cast<size_t>(k) * n + j], m[static_cast<size_t>(p) * n + j]);
        const double d = m[static_cast<size_t>(k) * n + k];
        for (int j = 0; j < n; ++j) row[j] = j == k ? 1.0 / d : m[static_cast<size_t>(k) * n + j] / d;
        for (int i = 0; i < n; ++i) col[i] = m[static_cast<size_t>(i) * n + k];
        for (int i = 0; i < n; ++i) {
            double* mi = &m[static_cast<size_t>(i) * n];
            if (i == k) {
                for (int j = 0; j < n; ++j) mi[j] = row[j];
            } else {
                const double f = col[i];
                for (int j = 0; j < n; ++j) mi[j] = (j == k ? 0.0 : mi[j]) - f * row[j];
            }
        }
    }
    for (int k = n - 1; k >= 0; --k)
        if (piv[k] != k)
            for (int i = 0; i < n; ++i) std::swap(m[static_cast<size_t>(i) * n + k], m[static_cast<size_t>(i) * n + piv[k]]);
    return true;
}

}  // namespace

NdTree nd_order(const HostCsr& a, int leaf_rows, int max_depth) {
    if (a.n_rows != a.n_cols) fail(SDG_EDIM, "nd_order: matrix must be square");
    const int n = a.n_rows;
    NdTree t;
    t.perm.reserve(n);
    const Graph g = symmetric_graph(a);
    Dissector ds(g, n, std::max(leaf_rows, 1), max_depth);
    std::vector<int> all(n);
    std::iota(all.begin(), all.end(), 0);
    ds.dissect(all, 0, t);
    return t;
}

HostCsr permute_symmetric(const HostCsr& a, const std::vector<int>& perm) {
    const int n = a.n_rows;
    std::vector<int> inv(n);
    for (int i = 0; i < n; ++i) inv[perm[i]] = i;
    HostCsr p(n, n);
    p.ci.reserve(a.ci.size());
    p.v.reserve(a.v.size());
    std::vector<std::pair<int, double>> row;
    for (int i = 0; i < n; ++i) {
        const int o = perm[i];
        row.clear();
        for (int k = a.rp[o]; k < a.rp[o + 1]; ++k) row.emplace_back(inv[a.ci[k]], a.v[k]);
        std::sort(row.begin(), row.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
        for (const auto& e : row) {
            p.ci.push_back(e.first);
            p.v.push_back(e.second);
        }
        p.rp[i + 1] = static_cast<int>(p.ci.size());
    }
    return p;
}

bool nd_solve_host(const HostCsr& a, const NdTree& t, const double* b, double* x) {
    const int n = a.n_rows;
    const HostCsr ap = permute_symmetric(a, t.perm);
    struct Blocks {
        std::vector<double> inv, w;
    };
    std::vector<Blocks> blk(t.nodes.size());
    // dense multi-column work: apply the subtree solve of node `id` to the columns of rhs (rows [lo, hi))
    // rhs/out are (hi - lo) x m row-major
    std::function<void(int, std::vector<double>&, int)> subtree = [&](int id, std::vector<double>& rhs, int m) {
        const NdNode& nd = t.nodes[id];
        const int lo = nd.lo, ni = nd.mid - nd.lo, ns = nd.hi - nd.mid, nl = nd.hi - nd.lo;
        if (nd.leaf()) {
            std::vector<double> out(static_cast<size_t>(nl) * m, 0.0);
            for (int r = 0; r < nl; ++r)
                for (int c = 0; c < nl; ++c) {
                    const double f = blk[id].inv[static_cast<size_t>(r) * nl + c];
                    if (f != 0.0)
                        for (int q = 0; q < m; ++q) out[static_cast<size_t>(r) * m + q] += f * rhs[static_cast<size_t>(c) * m + q];
                }
            rhs.swap(out);
            return;
        }
        for (int child : {nd.left, nd.right}) {
            const NdNode& ch = t.nodes[child];
            const int cl = ch.hi - ch.lo, off = ch.lo - lo;
            std::vector<double> sub(rhs.begin() + static_cast<size_t>(off) * m, rhs.begin() + static_cast<size_t>(off + cl) * m);
            subtree(child, sub, m);
            std::copy(sub.begin(), sub.end(), rhs.begin() + static_cast<size_t>(off) * m);
        }
        // t = b_S - A_SI y_I ; x_S = Sc^{-1} t
        std::vector<double> ts(static_cast<size_t>(ns) * m);
        for (int s = 0; s < ns; ++s) {
            for (int q = 0; q < m; ++q) ts[static_cast<size_t>(s) * m + q] = rhs[static_cast<size_t>(ni + s) * m + q];
            const int row = nd.mid + s;
            for (int k = ap.rp[row]; k < ap.rp[row + 1]; ++k) {
                const int j = ap.ci[k];
                if (j < lo || j >= nd.mid) continue;
                for (int q = 0; q < m; ++q) ts[static_cast<size_t>(s) * m + q] -= ap.v[k] * rhs[static_cast<size_t>(j - lo) * m + q];
            }
        }
        for (int r = 0; r < ns; ++r)
            for (int q = 0; q < m; ++q) {
                double acc = 0.0;
                for (int c = 0; c < ns; ++c) acc += blk[id].inv[static_cast<size_t>(r) * ns + c] * ts[static_cast<size_t>(c) * m + q];
                rhs[static_cast<size_t>(ni + r) * m + q] = acc;
            }
        for (int i = 0; i < ni; ++i)
            for (int q = 0; q < m; ++q) {
                double acc = 0.0;
                for (int c = 0; c < ns; ++c) acc += blk[id].w[static_cast<size_t>(i) * ns + c] * rhs[static_cast<size_t>(ni + c) * m + q];
                rhs[static_cast<size_t>(i) * m + q] -= acc;
            }
    };
    for (size_t id = 0; id < t.nodes.size(); ++id) {  // post-order: children are ready
        const NdNode& nd = t.nodes[id];
        const int lo = nd.lo, ni = nd.mid - nd.lo, ns = nd.hi - nd.mid;
        if (nd.leaf()) {
            const int nl = nd.hi - nd.lo;
            blk[id].inv.assign(static_cast<size_t>(nl) * nl, 0.0);
            for (int r = 0; r < nl; ++r)
                for (int k = ap.rp[lo + r]; k < ap.rp[lo + r + 1]; ++k) {
                    const int j = ap.ci[k];
                    if (j >= lo && j < nd.hi) blk[id].inv[static_cast<size_t>(r) * nl + (j - lo)] = ap.v[k];
                }
            if (!gj_inverse_host(blk[id].inv, nl)) return false;
            continue;
        }
        // W = A_II^{-1} A_IS through the two child subtrees
        std::vector<double> w(static_cast<size_t>(ni) * ns, 0.0);
        for (int i = 0; i < ni; ++i)
            for (int k = ap.rp[lo + i]; k < ap.rp[lo + i + 1]; ++k) {
                const int j = ap.ci[k];
                if (j >= nd.mid && j < nd.hi) w[static_cast<size_t>(i) * ns + (j - nd.mid)] = ap.v[k];
            }
        for (int child : {nd.left, nd.right}) {
            const NdNode& ch = t.nodes[child];
            const int cl = ch.hi - ch.lo, off = ch.lo - lo;
            std::vector<double> sub(w.begin() + static_cast<size_t>(off) * ns, w.begin() + static_cast<size_t>(off + cl) * ns);
            subtree(child, sub, ns);
            std::copy(sub.begin(), sub.end(), w.begin() + static_cast<size_t>(off) * ns);
        }
        std::vector<double> sc(static_cast<size_t>(ns) * ns, 0.0);
        for (int s = 0; s < ns; ++s) {
            const int row = nd.mid + s;
            for (int k = ap.rp[row]; k < ap.rp[row + 1]; ++k) {
                const int j = ap.ci[k];
                if (j >= nd.mid && j < nd.hi) {
                    sc[static_cast<size_t>(s) * ns + (j - nd.mid)] += ap.v[k];
                } else if (j >= lo && j < nd.mid) {
                    for (int c = 0; c < ns; ++c) sc[static_cast<size_t>(s) * ns + c] -= ap.v[k] * w[static_cast<size_t>(j - lo) * ns + c];
                }
            }
        }
        if (!gj_inverse_host(sc, ns)) return false;
        blk[id].inv.swap(sc);
        blk[id].w.swap(w);
    }
    std::vector<double> rhs(n);
    for (int i = 0; i < n; ++i) rhs[i] = b[t.perm[i]];
    subtree(static_cast<int>(t.nodes.size()) - 1, rhs, 1);
    for (int i = 0; i < n; ++i) x[t.perm[i]] = rhs[i];
    return true;
}

}  // namespace sdg
