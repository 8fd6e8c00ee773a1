// partition.cpp -- NEXT-4: graph partitioning orders for
// irregular matrices.  PAPER.md §2.2: for matrices not from a regular
// grid "the rows of the matrix are switched first and all the nonzero entries
// are put along the diagonal as close as possible", with the "quasi-optimal
// partition method METIS".  METIS is not installable offline (reading A21), so
// this file builds the two orders SPEC.md's partitioner contract allows
// (S:136-140):
//
//   HEC_ORDER_BISECT      SPEC's default: recursive bisection by BFS level
//                         sets from a pseudo-peripheral vertex, parts balanced
//                         by rows, lowest index first on ties.
//   HEC_ORDER_MULTILEVEL  a multilevel k-way partitioner (the METIS scheme):
//                         heavy-edge matching coarsens the graph, the coarsest
//                         graph is split by weighted level-set bisection, and
//                         every level is refined by greedy boundary moves on
//                         the way back, parts balanced by nonzeros.
//
// Both return perm[new] = old with the parts contiguous in the new order and
// part_ptr[P+1]; B = P A P^T (hec_permute) is then partitioned with
// HEC_PART_EXPLICIT.  The graph is the pattern of A + A^T without the
// diagonal; an edge's weight is the number of stored entries it stands for (1
// or 2), i.e. the halo entries it costs when cut.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <cstdlib>
#include <vector>

#include "hec_internal.h"

namespace hec {

struct Graph {
    int32_t n = 0;
    std::vector<int64_t> xadj;  // [n+1]
    std::vector<int32_t> adj;   // ascending per vertex
    std::vector<int32_t> ew;    // edge weights
    std::vector<int64_t> vw;    // vertex weights
    int64_t total = 0;          // sum of vw
};

// Pattern of A + A^T without the diagonal, with multiplicity as edge weight.
static Graph build_graph(const CsrView& A, bool unit_vertex_weights) {
    const int32_t n = A.n_rows;
    Graph g;
    g.n = n;
    std::vector<int64_t> deg((size_t)n + 1, 0);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k)
            if (A.col[k] != i) { deg[i]++; deg[A.col[k]]++; }
    std::vector<int64_t> ptr((size_t)n + 1, 0);
    for (int32_t i = 0; i < n; ++i) ptr[i + 1] = ptr[i] + deg[i];
    std::vector<int32_t> tmp((size_t)ptr[n]);
    std::vector<int64_t> pos(ptr.begin(), ptr.end() - 1);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) {
            const int32_t j = A.col[k];
            if (j == i) continue;
            tmp[(size_t)pos[i]++] = j;
            tmp[(size_t)pos[j]++] = i;
        }
    g.xadj.assign((size_t)n + 1, 0);
    g.adj.reserve(tmp.size());
    g.ew.reserve(tmp.size());
    for (int32_t i = 0; i < n; ++i) {
        auto b = tmp.begin() + ptr[i], e = tmp.begin() + ptr[i + 1];
        std::sort(b, e);
        for (auto it = b; it != e;) {
            auto jt = it;
            while (jt != e && *jt == *it) ++jt;
            g.adj.push_back(*it);
            g.ew.push_back((int32_t)(jt - it));
            it = jt;
        }
        g.xadj[i + 1] = (int64_t)g.adj.size();
    }
    g.vw.resize(n);
    for (int32_t i = 0; i < n; ++i)
        g.vw[i] = unit_vertex_weights ? 1 : std::max<int64_t>(1, A.row_ptr[i + 1] - A.row_ptr[i]);
    g.total = std::accumulate(g.vw.begin(), g.vw.end(), (int64_t)0);
    return g;
}

// BFS over the vertices with in[v] == stamp from root; appends to `out` in
// level order (neighbours ascending), marks them seen; returns the last level.
static std::vector<int32_t> bfs(const Graph& g, int32_t root, const std::vector<int32_t>& in, int32_t stamp,
                                std::vector<int32_t>& seen, int32_t seen_stamp, std::vector<int32_t>* out,
                                int32_t* depth) {
    std::vector<int32_t> level{root}, next;
    seen[root] = seen_stamp;
    if (out) out->push_back(root);
    *depth = 0;
    while (true) {
        next.clear();
        for (int32_t v : level)
            for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k) {
                const int32_t u = g.adj[(size_t)k];
                if (in[u] == stamp && seen[u] != seen_stamp) {
                    seen[u] = seen_stamp;
                    next.push_back(u);
                    if (out) out->push_back(u);
                }
            }
        if (next.empty()) return level;
        ++*depth;
        level.swap(next);
    }
}

// Level-set order of the vertex subset V (in[v] == stamp): for each connected
// piece, a pseudo-peripheral start (George-Liu: BFS, move to the
// lowest-(degree, index) vertex of the last level while the depth grows),
// then its BFS order; pieces in order of their lowest-(degree, index) vertex.
static void levelset_order(const Graph& g, const std::vector<int32_t>& V, std::vector<int32_t>& in, int32_t stamp,
                           std::vector<int32_t>& seen, int32_t& seen_stamp, std::vector<int32_t>* order) {
    order->clear();
    std::vector<int32_t> cand(V);
    auto deg = [&](int32_t v) { return g.xadj[v + 1] - g.xadj[v]; };
    std::sort(cand.begin(), cand.end(), [&](int32_t a, int32_t b) { return deg(a) != deg(b) ? deg(a) < deg(b) : a < b; });
    const int32_t done_stamp = ++seen_stamp;  // vertices already ordered
    for (int32_t s : cand) {
        if (seen[s] == done_stamp) continue;
        // pseudo-peripheral vertex of s's piece (scratch marks, not done_stamp)
        int32_t root = s, depth = -1;
        for (int it = 0; it < 8; ++it) {
            int32_t d = 0;
            const int32_t st = ++seen_stamp;
            std::vector<int32_t> last = bfs(g, root, in, stamp, seen, st, nullptr, &d);
            // the BFS overwrote done marks only inside this piece (none done yet)
            if (d <= depth) break;
            depth = d;
            int32_t best = last[0];
            for (int32_t v : last)
                if (deg(v) < deg(best) || (deg(v) == deg(best) && v < best)) best = v;
            root = best;
        }
        // the final BFS from root, marking the piece done
        std::vector<int32_t> piece;
        int32_t d = 0;
        const int32_t st = ++seen_stamp;
        bfs(g, root, in, stamp, seen, st, &piece, &d);
        for (int32_t v : piece) seen[v] = done_stamp;
        order->insert(order->end(), piece.begin(), piece.end());
    }
}

// Recursive bisection of V into P parts [part0, part0 + P): level-set order,
// split where the prefix weight reaches the proportional share.
static void recursive_bisect(const Graph& g, const std::vector<int32_t>& V, int32_t P, int32_t part0,
                             std::vector<int32_t>& part, std::vector<int32_t>& in, int32_t& in_stamp,
                             std::vector<int32_t>& seen, int32_t& seen_stamp, std::vector<int32_t>* emit) {
    if (P == 1 || V.size() <= 1) {
        for (int32_t v : V) part[v] = part0;
        if (emit) emit->insert(emit->end(), V.begin(), V.end());
        return;
    }
    const int32_t stamp = ++in_stamp;
    for (int32_t v : V) in[v] = stamp;
    std::vector<int32_t> order;
    levelset_order(g, V, in, stamp, seen, seen_stamp, &order);
    const int32_t P1 = P / 2;
    int64_t W = 0;
    for (int32_t v : V) W += g.vw[v];
    const int64_t target = W * P1 / P;
    size_t k = 0;
    int64_t acc = 0;
    while (k < order.size() && acc + g.vw[order[k]] <= target) acc += g.vw[order[k++]];
    if (k < order.size() && (target - acc) * 2 > g.vw[order[k]]) acc += g.vw[order[k++]];  // nearer the target
    // every side keeps at least as many vertices as parts
    k = std::max<size_t>(k, (size_t)P1);
    k = std::min<size_t>(k, order.size() - (size_t)(P - P1));
    std::vector<int32_t> L(order.begin(), order.begin() + k), R(order.begin() + k, order.end());
    recursive_bisect(g, L, P1, part0, part, in, in_stamp, seen, seen_stamp, emit);
    recursive_bisect(g, R, P - P1, part0 + P1, part, in, in_stamp, seen, seen_stamp, emit);
}

// Spectral order of a small graph (n <= kSpectralMax): vertices sorted by
// the Fiedler vector of the weighted Laplacian (cyclic Jacobi on the dense
// matrix; ties by index).  On a chain with uniformly spread "noise" edges the
// noise shifts every non-constant eigenvalue alike, so the order is the
// chain's -- the case the coarsest graph of a banded matrix with far
// couplings is, where BFS level sets see one level.
constexpr int32_t kSpectralMax = 512;
static std::vector<int32_t> spectral_order(const Graph& g) {
    const int32_t n = g.n;
    std::vector<double> a((size_t)n * n, 0.0), V((size_t)n * n, 0.0);
    for (int32_t i = 0; i < n; ++i) {
        V[(size_t)i * n + i] = 1.0;
        for (int64_t k = g.xadj[i]; k < g.xadj[i + 1]; ++k) {
            const int32_t j = g.adj[(size_t)k];
            a[(size_t)i * n + j] -= g.ew[(size_t)k];
            a[(size_t)i * n + i] += g.ew[(size_t)k];
        }
    }
    for (int sweep = 0; sweep < 30; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int32_t i = 0; i < n; ++i)
            for (int32_t j = 0; j < n; ++j) {
                const double v = a[(size_t)i * n + j] * a[(size_t)i * n + j];
                tot += v;
                if (i != j) off += v;
            }
        if (off <= 1e-16 * tot) break;  // the order needs the Fiedler vector to ~1e-8, not to rounding
        for (int32_t p = 0; p < n - 1; ++p)
            for (int32_t q = p + 1; q < n; ++q) {
                const double apq = a[(size_t)p * n + q];
                if (apq == 0.0) continue;
                const double app = a[(size_t)p * n + p], aqq = a[(size_t)q * n + q];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
                for (int32_t k = 0; k < n; ++k) {  // columns p, q
                    const double akp = a[(size_t)k * n + p], akq = a[(size_t)k * n + q];
                    a[(size_t)k * n + p] = c * akp - sn * akq;
                    a[(size_t)k * n + q] = sn * akp + c * akq;
                }
                for (int32_t k = 0; k < n; ++k) {  // rows p, q
                    const double apk = a[(size_t)p * n + k], aqk = a[(size_t)q * n + k];
                    a[(size_t)p * n + k] = c * apk - sn * aqk;
                    a[(size_t)q * n + k] = sn * apk + c * aqk;
                }
                for (int32_t k = 0; k < n; ++k) {
                    const double vkp = V[(size_t)k * n + p], vkq = V[(size_t)k * n + q];
                    V[(size_t)k * n + p] = c * vkp - sn * vkq;
                    V[(size_t)k * n + q] = sn * vkp + c * vkq;
                }
            }
    }
    std::vector<int32_t> ev(n);
    std::iota(ev.begin(), ev.end(), 0);
    std::sort(ev.begin(), ev.end(), [&](int32_t x, int32_t y) {
        const double ax = a[(size_t)x * n + x], ay = a[(size_t)y * n + y];
        return ax != ay ? ax < ay : x < y;
    });
    const int32_t f = n > 1 ? ev[1] : ev[0];  // second smallest: the Fiedler vector
    std::vector<int32_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
        const double fx = V[(size_t)x * n + f], fy = V[(size_t)y * n + f];
        return fx != fy ? fx < fy : x < y;
    });
    return order;
}

// Recursive spectral bisection of the vertex subset V (a small coarse graph):
// each split orders V by the Fiedler vector of V's own induced subgraph and
// cuts where the prefix weight reaches the proportional share.  A chain
// segment's own Fiedler vector is sharper than the whole chain's (lambda_2
// grows as the segment shortens, the far couplings' noise does not), so the
// deeper splits fold less than one P-way cut of the global order.
static void spectral_bisect(const Graph& g, const std::vector<int32_t>& V, int32_t P, int32_t part0,
                            std::vector<int32_t>& part, std::vector<int32_t>& loc) {
    if (P == 1 || V.size() <= 1) {
        for (int32_t v : V) part[v] = part0;
        return;
    }
    Graph h;
    h.n = (int32_t)V.size();
    for (int32_t i = 0; i < h.n; ++i) loc[V[i]] = i;
    h.xadj.assign((size_t)h.n + 1, 0);
    h.vw.resize(h.n);
    for (int32_t i = 0; i < h.n; ++i) {
        const int32_t v = V[i];
        h.vw[i] = g.vw[v];
        for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k) {
            const int32_t u = g.adj[(size_t)k];
            if (loc[u] >= 0) {
                h.adj.push_back(loc[u]);
                h.ew.push_back(g.ew[(size_t)k]);
            }
        }
        h.xadj[i + 1] = (int64_t)h.adj.size();
    }
    std::vector<int32_t> ord = spectral_order(h);
    for (int32_t v : V) loc[v] = -1;
    const int32_t P1 = P / 2;
    int64_t W = 0;
    for (int32_t v : V) W += g.vw[v];
    const int64_t target = W * P1 / P;
    size_t k = 0;
    int64_t acc = 0;
    while (k < ord.size() && acc + h.vw[ord[k]] <= target) acc += h.vw[ord[k++]];
    if (k < ord.size() && (target - acc) * 2 > h.vw[ord[k]]) acc += h.vw[ord[k++]];
    k = std::max<size_t>(k, (size_t)P1);
    k = std::min<size_t>(k, ord.size() - (size_t)(P - P1));
    std::vector<int32_t> L, R;
    for (size_t i = 0; i < ord.size(); ++i) (i < k ? L : R).push_back(V[ord[i]]);
    spectral_bisect(g, L, P1, part0, part, loc);
    spectral_bisect(g, R, P - P1, part0 + P1, part, loc);
}

static uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Heavy-edge matching (vertices visited in a seeded order; ties to the lowest
// index) and contraction: cmap[v] = coarse vertex.
static Graph coarsen(const Graph& g, uint64_t seed, std::vector<int32_t>* cmap) {
    const int32_t n = g.n;
    std::vector<int32_t> visit(n);
    std::iota(visit.begin(), visit.end(), 0);
    std::vector<uint64_t> key(n);
    for (int32_t v = 0; v < n; ++v) key[v] = mix64(seed ^ (uint64_t)v);
    std::sort(visit.begin(), visit.end(), [&](int32_t a, int32_t b) { return key[a] < key[b]; });
    std::vector<int32_t> match(n, -1);
    const int64_t capdiv = std::getenv("HEC_PART_CAPDIV") ? std::atoll(std::getenv("HEC_PART_CAPDIV")) : 64;
    const int64_t cap = std::max<int64_t>(1, g.total / capdiv);  // no coarse vertex heavier than ~1/64 of the graph
    for (int32_t v : visit) {
        if (match[v] >= 0) continue;
        int32_t best = -1, bw = -1;
        for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k) {
            const int32_t u = g.adj[(size_t)k];
            if (match[u] >= 0 || g.vw[u] + g.vw[v] > cap) continue;
            if (g.ew[(size_t)k] > bw) { bw = g.ew[(size_t)k]; best = u; }
        }
        if (best < 0) match[v] = v;
        else { match[v] = best; match[best] = v; }
    }
    cmap->assign(n, -1);
    int32_t nc = 0;
    for (int32_t v = 0; v < n; ++v)
        if ((*cmap)[v] < 0) {
            (*cmap)[v] = nc;
            (*cmap)[match[v]] = nc;
            ++nc;
        }
    Graph c;
    c.n = nc;
    c.vw.assign(nc, 0);
    for (int32_t v = 0; v < n; ++v) c.vw[(*cmap)[v]] += g.vw[v];
    c.total = g.total;
    // members of each coarse vertex, then merge their adjacency
    std::vector<int32_t> first(nc, -1), second(nc, -1);
    for (int32_t v = 0; v < n; ++v) {
        const int32_t cv = (*cmap)[v];
        if (first[cv] < 0) first[cv] = v;
        else second[cv] = v;
    }
    c.xadj.assign((size_t)nc + 1, 0);
    std::vector<int32_t> accw(nc, 0), touched;
    for (int32_t cv = 0; cv < nc; ++cv) {
        touched.clear();
        for (int32_t v : {first[cv], second[cv]}) {
            if (v < 0) continue;
            for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k) {
                const int32_t cu = (*cmap)[g.adj[(size_t)k]];
                if (cu == cv) continue;
                if (accw[cu] == 0) touched.push_back(cu);
                accw[cu] += g.ew[(size_t)k];
            }
        }
        for (int32_t cu : touched) {  // first-touch order: deterministic, no sort needed
            c.adj.push_back(cu);
            c.ew.push_back(accw[cu]);
            accw[cu] = 0;
        }
        c.xadj[cv + 1] = (int64_t)c.adj.size();
    }
    return c;
}

// Greedy k-way boundary refinement: move a vertex to the adjacent part it is
// most connected to when that cuts fewer edge weights (or as many, towards a
// lighter part) and keeps the target under the balance bound; overweight
// parts first shed vertices to their lightest adjacent part.
static void refine(const Graph& g, int32_t P, std::vector<int32_t>& part, int passes) {
    const int64_t maxw = (int64_t)((double)g.total / P * 1.03) + 1;
    std::vector<int64_t> pw(P, 0);
    for (int32_t v = 0; v < g.n; ++v) pw[part[v]] += g.vw[v];
    std::vector<int64_t> conn(P, 0);
    std::vector<int32_t> touched;
    for (int pass = 0; pass < passes; ++pass) {
        int64_t moved = 0;
        for (int32_t v = 0; v < g.n; ++v) {
            const int32_t own = part[v];
            touched.clear();
            bool boundary = false;
            for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k) {
                const int32_t q = part[g.adj[(size_t)k]];
                if (q != own) boundary = true;
                if (conn[q] == 0) touched.push_back(q);
                conn[q] += g.ew[(size_t)k];
            }
            if (boundary || pw[own] > maxw) {
                const int64_t internal = conn[own];
                int32_t best = own;
                int64_t bgain = pw[own] > maxw ? INT64_MIN : 0;
                for (int32_t q : touched) {
                    if (q == own || pw[q] + g.vw[v] > maxw) continue;
                    const int64_t gain = conn[q] - internal;
                    if (gain > bgain || (gain == bgain && best != own && pw[q] < pw[best]) ||
                        (gain == 0 && best == own && pw[q] + g.vw[v] < pw[own])) {
                        bgain = gain;
                        best = q;
                    }
                }
                if (best != own && pw[own] > g.vw[v]) {  // never empty a part
                    part[v] = best;
                    pw[own] -= g.vw[v];
                    pw[best] += g.vw[v];
                    ++moved;
                }
            }
            for (int32_t q : touched) conn[q] = 0;
        }
        if (moved == 0) break;
    }
}

// FM refinement with hill climbing (Fiduccia-Mattheyses, k-way) for the
// small coarse levels: moves the unlocked vertex with the best gain to an
// adjacent part -- also when the gain is negative -- under a balance bound of
// the average part weight + one heaviest vertex, locks it, and after the
// pass rolls back to the prefix of moves with the smallest edge cut.  A
// negative first move lets a whole run of vertices follow, which the greedy
// refine() (gain >= 0 only) cannot: the folds the coarsest spectral order
// leaves are such runs.
static void fm_refine(const Graph& g, int32_t P, std::vector<int32_t>& part, int passes) {
    const int32_t n = g.n;
    int64_t maxv = 0;
    for (int32_t v = 0; v < n; ++v) maxv = std::max(maxv, g.vw[v]);
    const int64_t maxw = (int64_t)((double)g.total / P * 1.03) + maxv;
    std::vector<int64_t> pw(P, 0), conn((size_t)n * P, 0);
    for (int pass = 0; pass < passes; ++pass) {
        std::fill(pw.begin(), pw.end(), 0);
        std::fill(conn.begin(), conn.end(), 0);
        for (int32_t v = 0; v < n; ++v) {
            pw[part[v]] += g.vw[v];
            for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k)
                conn[(size_t)v * P + part[g.adj[(size_t)k]]] += g.ew[(size_t)k];
        }
        std::vector<char> locked(n, 0);
        std::vector<std::pair<int32_t, int32_t>> moves;  // (vertex, from)
        int64_t cut = 0, best = 0;
        size_t best_len = 0;
        for (int32_t step = 0; step < n; ++step) {
            int32_t bv = -1, bq = -1;
            int64_t bg = INT64_MIN;
            for (int32_t v = 0; v < n; ++v) {
                if (locked[v]) continue;
                const int32_t own = part[v];
                if (pw[own] - g.vw[v] <= 0) continue;  // never empty a part
                const int64_t in = conn[(size_t)v * P + own];
                for (int32_t q = 0; q < P; ++q) {
                    if (q == own || conn[(size_t)v * P + q] == 0 || pw[q] + g.vw[v] > maxw) continue;
                    const int64_t gain = conn[(size_t)v * P + q] - in;
                    if (gain > bg) { bg = gain; bv = v; bq = q; }
                }
            }
            if (bv < 0) break;
            const int32_t from = part[bv];
            part[bv] = bq;
            pw[from] -= g.vw[bv];
            pw[bq] += g.vw[bv];
            for (int64_t k = g.xadj[bv]; k < g.xadj[bv + 1]; ++k) {
                const int32_t u = g.adj[(size_t)k];
                conn[(size_t)u * P + from] -= g.ew[(size_t)k];
                conn[(size_t)u * P + bq] += g.ew[(size_t)k];
            }
            locked[bv] = 1;
            moves.emplace_back(bv, from);
            cut -= bg;  // relative to the pass's start
            if (cut < best) { best = cut; best_len = moves.size(); }
        }
        for (size_t i = moves.size(); i > best_len; --i) part[moves[i - 1].first] = moves[i - 1].second;
        if (best_len == 0) break;
    }
}

// Final order: parts in order, inside a part the vertices keep the order of
// their coarsest ancestors (a level-set order of the coarse graph), children
// of one coarse vertex adjacent -- locality for the x gathers.
static hec_status order_from_parts(const std::vector<Graph>& G, const std::vector<std::vector<int32_t>>& cmaps,
                                   const std::vector<int32_t>& coarse_order, const std::vector<int32_t>& part, int32_t P,
                                   int32_t* perm, int32_t* part_ptr) {
    const int L = (int)G.size();
    // rank of every vertex at the coarsest level, then refined level by level
    std::vector<int64_t> rank(G[L - 1].n);
    for (size_t i = 0; i < coarse_order.size(); ++i) rank[coarse_order[i]] = (int64_t)i;
    for (int l = L - 2; l >= 0; --l) {
        std::vector<int64_t> fr(G[l].n);
        std::vector<int32_t> idx(G[l].n);
        std::iota(idx.begin(), idx.end(), 0);
        for (int32_t v = 0; v < G[l].n; ++v) fr[v] = rank[cmaps[l][v]];
        std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return fr[a] < fr[b]; });
        for (int32_t i = 0; i < G[l].n; ++i) fr[idx[i]] = i;
        rank.swap(fr);
    }
    const int32_t n = G[0].n;
    std::vector<int32_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
        return part[a] != part[b] ? part[a] < part[b] : rank[a] < rank[b];
    });
    std::memcpy(perm, idx.data(), sizeof(int32_t) * (size_t)n);
    std::vector<int32_t> cnt(P + 1, 0);
    for (int32_t v = 0; v < n; ++v) cnt[part[v] + 1]++;
    for (int32_t p = 0; p < P; ++p) cnt[p + 1] += cnt[p];
    std::memcpy(part_ptr, cnt.data(), sizeof(int32_t) * (size_t)(P + 1));
    for (int32_t p = 0; p < P; ++p)
        if (part_ptr[p + 1] == part_ptr[p]) return fail(HEC_ERR_PARTS, "a part came out empty");
    return HEC_OK;
}

}  // namespace hec

using namespace hec;

extern "C" {

hec_status hec_partition_order(const hec_csr* A, int32_t n_parts, int32_t method, int32_t* perm, int32_t* part_ptr) {
    if (!perm || !part_ptr) return fail(HEC_ERR_ARG, "NULL output");
    CsrView v;
    hec_status st = validate_csr(A, &v);
    if (st != HEC_OK) return st;
    if (v.n_rows != v.n_cols) return fail(HEC_ERR_DIM, "partition orders need a square matrix");
    if (n_parts < 1 || n_parts > v.n_rows) return fail(HEC_ERR_PARTS, "n_parts must be in [1, n_rows]");
    if (method != HEC_ORDER_BISECT && method != HEC_ORDER_MULTILEVEL) return fail(HEC_ERR_ARG, "unknown method");
    if (n_parts == 1) {  // one part: the identity order
        for (int32_t i = 0; i < v.n_rows; ++i) perm[i] = i;
        part_ptr[0] = 0;
        part_ptr[1] = v.n_rows;
        return HEC_OK;
    }
    try {
        const Graph g0 = build_graph(v, method == HEC_ORDER_BISECT);
        if (method == HEC_ORDER_BISECT) {
            std::vector<int32_t> part(g0.n, 0), in(g0.n, 0), seen(g0.n, 0), order, all(g0.n);
            int32_t in_stamp = 0, seen_stamp = 0;
            std::iota(all.begin(), all.end(), 0);
            recursive_bisect(g0, all, n_parts, 0, part, in, in_stamp, seen, seen_stamp, &order);
            return order_from_parts({g0}, {}, order, part, n_parts, perm, part_ptr);
        }
        // multilevel: a few independent trials (matching orders), the smallest
        // edge cut wins -- the result of one trial depends on where the
        // coarsening happens to fold the graph
        // (each matching order is run twice: plain greedy refinement, and with
        // FM hill climbing on the small levels first -- neither wins always)
        int trials = 3;
        if (const char* e = std::getenv("HEC_PART_TRIALS")) trials = std::max(1, std::atoi(e));
        int32_t fm_max = 2048;  // FM on the levels up to this many vertices (HEC_PART_FM, tuning; 0: off)
        if (const char* e = std::getenv("HEC_PART_FM")) fm_max = std::max(0, std::atoi(e));
        // and a third time from a recursive spectral bisection of the coarsest graph
        const int runs = (fm_max > 0 ? 2 : 1) * trials + trials;
        int64_t best_cut = -1, best_vol = -1;
        std::vector<int32_t> seen_part(n_parts, 0);
        std::vector<int32_t> bperm(v.n_rows), bpp(n_parts + 1);
        for (int run = 0; run < runs; ++run) {
            const int trial = run % trials;
            const bool rsb = run >= runs - trials;
            const int32_t fm_lvl = (run >= trials && !rsb) || (rsb && fm_max > 0) ? fm_max : 0;
            std::vector<Graph> G;
            G.push_back(g0);
            std::vector<std::vector<int32_t>> cmaps;
            int32_t stop = std::max<int32_t>(32 * n_parts, 256);
            if (const char* e = std::getenv("HEC_PART_STOP")) stop = std::max(2 * n_parts, std::atoi(e));  // tuning
            const char* sd = std::getenv("HEC_PART_SEED");  // matching order seed (tuning)
            const uint64_t seed = (sd ? std::atoll(sd) : 1606) + 7919ULL * trial;
            while (G.back().n > stop) {
                std::vector<int32_t> cmap;
                Graph c = coarsen(G.back(), seed + G.size(), &cmap);
                if (c.n > (int32_t)(0.95 * G.back().n)) break;  // matching stalled
                cmaps.push_back(std::move(cmap));
                G.push_back(std::move(c));
            }
            const Graph& gc = G.back();
            std::vector<int32_t> part(gc.n, 0), in(gc.n, 0), seen(gc.n, 0), coarse_order;
            int32_t in_stamp = 0, seen_stamp = 0;
            if (gc.n <= kSpectralMax) coarse_order = spectral_order(gc);
            if (rsb && !coarse_order.empty()) {
                std::vector<int32_t> all(gc.n), loc(gc.n, -1);
                std::iota(all.begin(), all.end(), 0);
                spectral_bisect(gc, all, n_parts, 0, part, loc);
            } else if (!coarse_order.empty()) {
                // the coarsest order cut into n_parts consecutive pieces of (nearly) equal weight
                int64_t acc = 0;
                int32_t p = 0;
                for (size_t i = 0; i < coarse_order.size(); ++i) {
                    const int32_t u = coarse_order[i];
                    // advance while this vertex's midpoint lies past part p's share
                    // (and enough vertices remain for the parts after it)
                    while (p < n_parts - 1 && (acc + gc.vw[u] / 2) * n_parts >= (int64_t)(p + 1) * gc.total &&
                           (int64_t)(coarse_order.size() - i) >= n_parts - p)
                        ++p;
                    part[u] = p;
                    acc += gc.vw[u];
                }
            } else {
                std::vector<int32_t> all(gc.n);
                std::iota(all.begin(), all.end(), 0);
                recursive_bisect(gc, all, n_parts, 0, part, in, in_stamp, seen, seen_stamp, &coarse_order);
            }
            if (gc.n <= fm_lvl) fm_refine(gc, n_parts, part, 8);
            refine(gc, n_parts, part, 8);
            for (int l = (int)G.size() - 2; l >= 0; --l) {
                std::vector<int32_t> fine(G[l].n);
                for (int32_t u = 0; u < G[l].n; ++u) fine[u] = part[cmaps[l][u]];
                part.swap(fine);
                if (G[l].n <= fm_lvl) fm_refine(G[l], n_parts, part, 4);
                refine(G[l], n_parts, part, 4);
            }
            // the run's halo volume: sum over vertices u of the other parts
            // adjacent to u (each is one x entry that part receives) -- what
            // the exchange moves; the edge cut breaks ties
            int64_t cut = 0, vol = 0;
            for (int32_t u = 0; u < g0.n; ++u) {
                const int32_t pu = part[u];
                for (int64_t k = g0.xadj[u]; k < g0.xadj[u + 1]; ++k) {
                    const int32_t q = part[g0.adj[(size_t)k]];
                    if (q == pu) continue;
                    cut += g0.ew[(size_t)k];
                    if (seen_part[q] != u + 1) { seen_part[q] = u + 1; ++vol; }
                }
            }
            if (best_cut < 0 || vol < best_vol || (vol == best_vol && cut < best_cut)) {
                st = order_from_parts(G, cmaps, coarse_order, part, n_parts, bperm.data(), bpp.data());
                if (st != HEC_OK) continue;
                best_cut = cut;
                best_vol = vol;
            }
        }
        if (best_cut < 0) return fail(HEC_ERR_PARTS, "a part came out empty");
        std::memcpy(perm, bperm.data(), sizeof(int32_t) * (size_t)v.n_rows);
        std::memcpy(part_ptr, bpp.data(), sizeof(int32_t) * (size_t)(n_parts + 1));
        return HEC_OK;
    } catch (const std::bad_alloc&) {
        return fail(HEC_ERR_NOMEM, "host allocation failed in hec_partition_order");
    }
}

}  // extern "C"
