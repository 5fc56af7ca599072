// partition.cpp -- host side of the index build: the vertex-separator
// partition and the per-part minimum-degree orders.
//
// Native restatement of the reference partitioner (partition.py:82-248) and
// of factor._min_degree_order (factor.py:31-55) with the same tie rules, so
// the permutation, part boundaries and elimination orders are identical to
// the reference's for the same graph and configuration:
//   * a piece is split by BFS levels from its smallest node; levels are
//     accumulated until they hold at least half the piece (never all of it);
//   * the cut edges (level k -> not yet taken) get a greedy vertex cover that
//     repeatedly takes the endpoint with the most uncovered edges, ties to
//     the smaller id; the cover joins the separator;
//   * both sides are split into connected components ordered by smallest
//     node (each sorted), pushed on a LIFO stack b-side first;
//   * pieces of size <= limit (or depth exhausted, or < 2 nodes) are parts.
// Sets of the reference become stamp arrays and a lazy max-heap.
#include <algorithm>
#include <cstdint>
#include <queue>
#include <utility>
#include <vector>

#include "katzb200.h"

namespace {

struct Csr {
    int64_t n;
    const int64_t* rp;
    const int64_t* ci;
};

struct Stamps {
    std::vector<uint32_t> s;
    uint32_t cur = 0;
    explicit Stamps(int64_t n) : s(n, 0) {}
    void next() {
        if (++cur == 0) {
            std::fill(s.begin(), s.end(), 0);
            cur = 1;
        }
    }
    bool has(int64_t v) const { return s[v] == cur; }
    void add(int64_t v) { s[v] = cur; }
};

// _bfs_levels (partition.py:82-97)
void bfs_levels(const Csr& g, const std::vector<char>& in_sub, int64_t start, Stamps& seen,
                std::vector<std::vector<int64_t>>& levels) {
    levels.clear();
    seen.next();
    seen.add(start);
    levels.push_back({start});
    while (true) {
        std::vector<int64_t> nxt;
        for (int64_t u : levels.back())
            for (int64_t e = g.rp[u]; e < g.rp[u + 1]; ++e) {
                const int64_t w = g.ci[e];
                if (in_sub[w] && !seen.has(w)) {
                    seen.add(w);
                    nxt.push_back(w);
                }
            }
        if (nxt.empty()) return;
        std::sort(nxt.begin(), nxt.end());
        levels.push_back(std::move(nxt));
    }
}

// _greedy_vertex_cover (partition.py:100-127): most uncovered edges first,
// ties to the smaller id; returns the cover sorted.
std::vector<int64_t> greedy_cover(const std::vector<std::pair<int64_t, int64_t>>& cut) {
    std::vector<int64_t> verts;
    verts.reserve(cut.size() * 2);
    for (auto& e : cut) {
        verts.push_back(e.first);
        verts.push_back(e.second);
    }
    std::sort(verts.begin(), verts.end());
    verts.erase(std::unique(verts.begin(), verts.end()), verts.end());
    auto vid = [&](int64_t v) { return std::lower_bound(verts.begin(), verts.end(), v) - verts.begin(); };
    const size_t nv = verts.size();
    std::vector<std::vector<int32_t>> inc(nv);
    for (size_t e = 0; e < cut.size(); ++e) {
        inc[vid(cut[e].first)].push_back(static_cast<int32_t>(e));
        inc[vid(cut[e].second)].push_back(static_cast<int32_t>(e));
    }
    std::vector<int64_t> cnt(nv);
    // heap of (count, -id): largest count, then smallest id
    std::priority_queue<std::pair<int64_t, int64_t>> heap;
    for (size_t i = 0; i < nv; ++i) {
        cnt[i] = static_cast<int64_t>(inc[i].size());
        heap.push({cnt[i], -static_cast<int64_t>(i)});
    }
    std::vector<char> covered(cut.size(), 0), taken(nv, 0);
    size_t left = cut.size();
    std::vector<int64_t> cover;
    while (left > 0 && !heap.empty()) {
        auto top = heap.top();
        heap.pop();
        const size_t i = static_cast<size_t>(-top.second);
        if (taken[i] || top.first != cnt[i]) continue;  // stale entry
        taken[i] = 1;
        cover.push_back(verts[i]);
        for (int32_t e : inc[i]) {
            if (covered[e]) continue;
            covered[e] = 1;
            --left;
            const int64_t other = cut[e].first == verts[i] ? cut[e].second : cut[e].first;
            const size_t o = vid(other);
            if (!taken[o]) {
                --cnt[o];
                heap.push({cnt[o], -static_cast<int64_t>(o)});
            }
        }
        cnt[i] = 0;
    }
    std::sort(cover.begin(), cover.end());
    return cover;
}

// _components_of (partition.py:153-175)
void components_of(const Csr& g, const std::vector<int64_t>& nodes, const std::vector<char>& in_sub,
                   Stamps& seen, std::vector<std::vector<int64_t>>& comps) {
    comps.clear();
    seen.next();
    for (int64_t s : nodes) {
        if (seen.has(s)) continue;
        seen.add(s);
        std::vector<int64_t> comp{s}, frontier{s};
        while (!frontier.empty()) {
            std::vector<int64_t> nxt;
            for (int64_t u : frontier)
                for (int64_t e = g.rp[u]; e < g.rp[u + 1]; ++e) {
                    const int64_t w = g.ci[e];
                    if (in_sub[w] && !seen.has(w)) {
                        seen.add(w);
                        nxt.push_back(w);
                    }
                }
            comp.insert(comp.end(), nxt.begin(), nxt.end());
            frontier.swap(nxt);
        }
        std::sort(comp.begin(), comp.end());
        comps.push_back(std::move(comp));
    }
}

}  // namespace

// partition_vertex_separator (partition.py:178-248) for a connected graph
// in CSR (int64 arrays, host memory).  Outputs: perm[n] (new position ->
// node), bounds[num_parts+1] (caller allocates n+1), *num_parts, *n1, *n2.
extern "C" int kz_partition(int64_t n, const int64_t* rowptr, const int64_t* colidx, int64_t limit,
                            int64_t max_depth, int64_t* perm, int64_t* bounds, int64_t* num_parts,
                            int64_t* n1_out, int64_t* n2_out) {
    if (n < 1 || !rowptr || !perm || !bounds || !num_parts || !n1_out || !n2_out || limit < 1)
        return KZ_EARG;
    const Csr g{n, rowptr, colidx};
    std::vector<char> in_sub(n, 0);
    Stamps seen(n), aset(n), sepset(n);
    std::vector<std::vector<int64_t>> parts, levels, comps_a, comps_b;
    std::vector<int64_t> separator;
    std::vector<std::pair<std::vector<int64_t>, int64_t>> stack;
    std::vector<int64_t> all(n);
    for (int64_t i = 0; i < n; ++i) all[i] = i;
    stack.push_back({std::move(all), max_depth});
    while (!stack.empty()) {
        auto item = std::move(stack.back());
        stack.pop_back();
        std::vector<int64_t>& nodes = item.first;
        const int64_t depth = item.second;
        if (static_cast<int64_t>(nodes.size()) <= limit || depth <= 0 || nodes.size() < 2) {
            parts.push_back(std::move(nodes));
            continue;
        }
        for (int64_t u : nodes) in_sub[u] = 1;
        // _split_once (partition.py:130-150)
        bfs_levels(g, in_sub, nodes[0], seen, levels);
        const double half = static_cast<double>(nodes.size()) / 2.0;
        int64_t cum = 0, k = static_cast<int64_t>(levels.size());
        for (size_t i = 0; i < levels.size(); ++i) {
            cum += static_cast<int64_t>(levels[i].size());
            if (static_cast<double>(cum) >= half) {
                k = static_cast<int64_t>(i);
                break;
            }
        }
        if (k >= static_cast<int64_t>(levels.size()) - 1) k = static_cast<int64_t>(levels.size()) - 2;
        aset.next();
        for (int64_t l = 0; l <= k; ++l)
            for (int64_t u : levels[l]) aset.add(u);
        std::vector<std::pair<int64_t, int64_t>> cut;
        for (int64_t u : levels[k])
            for (int64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
                const int64_t w = colidx[e];
                if (in_sub[w] && !aset.has(w)) cut.push_back({u, w});
            }
        std::vector<int64_t> sep = greedy_cover(cut);
        sepset.next();
        for (int64_t u : sep) sepset.add(u);
        std::vector<int64_t> side_a, side_b;
        for (int64_t u : nodes) {
            if (sepset.has(u)) continue;
            (aset.has(u) ? side_a : side_b).push_back(u);
        }
        separator.insert(separator.end(), sep.begin(), sep.end());
        for (int64_t u : sep) in_sub[u] = 0;
        components_of(g, side_a, in_sub, seen, comps_a);
        components_of(g, side_b, in_sub, seen, comps_b);
        for (int64_t u : side_a) in_sub[u] = 0;
        for (int64_t u : side_b) in_sub[u] = 0;
        for (auto it = comps_b.rbegin(); it != comps_b.rend(); ++it) stack.push_back({std::move(*it), depth - 1});
        for (auto it = comps_a.rbegin(); it != comps_a.rend(); ++it) stack.push_back({std::move(*it), depth - 1});
    }
    std::sort(separator.begin(), separator.end());
    int64_t pos = 0;
    bounds[0] = 0;
    for (size_t p = 0; p < parts.size(); ++p) {
        for (int64_t u : parts[p]) perm[pos++] = u;
        bounds[p + 1] = pos;
    }
    const int64_t n1 = pos;
    for (int64_t u : separator) perm[pos++] = u;
    if (pos != n) return KZ_EARG;
    *num_parts = static_cast<int64_t>(parts.size());
    *n1_out = n1;
    *n2_out = n - n1;
    return KZ_OK;
}

namespace {

// Minimum-degree elimination of one part whose rows are [s, s+m) of a CSR
// with global columns (entries outside [s, s+m) are ignored).
void min_degree_part(int64_t s, int64_t m, const int64_t* rowptr, const int64_t* colidx, int64_t* order) {
    std::vector<std::vector<char>> nb(m, std::vector<char>(m, 0));
    std::vector<int64_t> deg(m, 0);
    for (int64_t i = 0; i < m; ++i)
        for (int64_t e = rowptr[s + i]; e < rowptr[s + i + 1]; ++e) {
            const int64_t j = colidx[e] - s;
            if (j >= 0 && j < m && j != i && !nb[i][j]) {
                nb[i][j] = 1;
                ++deg[i];
            }
        }
    std::vector<char> alive(m, 1);
    std::vector<int64_t> clique;
    for (int64_t step = 0; step < m; ++step) {
        int64_t u = -1;
        for (int64_t v = 0; v < m; ++v)
            if (alive[v] && (u < 0 || deg[v] < deg[u])) u = v;
        order[step] = u;
        alive[u] = 0;
        clique.clear();
        for (int64_t x = 0; x < m; ++x)
            if (nb[u][x]) clique.push_back(x);
        for (int64_t x : clique)
            if (nb[x][u]) {
                nb[x][u] = 0;
                --deg[x];
            }
        for (int64_t x : clique)
            for (int64_t y : clique)
                if (y != x && !nb[x][y]) {
                    nb[x][y] = 1;
                    ++deg[x];
                }
    }
}

}  // namespace

// _min_degree_order (factor.py:31-55) of one part: its internal adjacency
// in local CSR (m nodes).  Elimination simulation on dense boolean rows
// (parts are small); ties to the smallest index.
extern "C" int kz_min_degree_order(int64_t m, const int64_t* rowptr, const int64_t* colidx, int64_t* order) {
    if (m < 0 || (m > 0 && (!rowptr || !order))) return KZ_EARG;
    if (m > 0) min_degree_part(0, m, rowptr, colidx, order);
    return KZ_OK;
}

// All parts at once: rows [bounds[p], bounds[p+1]) of the partition-ordered
// adjacency (global columns) form part p; orders[bounds[p] + k] receives the
// k-th eliminated local index of part p.
extern "C" int kz_min_degree_orders(int64_t nparts, const int64_t* bounds, const int64_t* rowptr,
                                    const int64_t* colidx, int64_t* orders) {
    if (nparts < 0 || (nparts > 0 && (!bounds || !rowptr || !orders))) return KZ_EARG;
    for (int64_t p = 0; p < nparts; ++p) {
        const int64_t s = bounds[p], m = bounds[p + 1] - s;
        if (m < 0) return KZ_EARG;
        if (m == 1) orders[s] = 0;
        else if (m > 1) min_degree_part(s, m, rowptr, colidx, orders + s);
    }
    return KZ_OK;
}
