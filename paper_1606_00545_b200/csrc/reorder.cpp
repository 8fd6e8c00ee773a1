// reorder.cpp -- NEXT-4: bandwidth-reducing row/column
// reordering for irregular matrices.  PAPER.md §2.2: for matrices that
// are not from a regular grid, "the rows of the matrix are switched first and
// all the nonzero entries are put along the diagonal as close as possible"
// (the paper uses METIS, which cannot be installed offline here).  This is a
// deterministic reverse Cuthill-McKee ordering (reading A21) plus the
// symmetric permutation B = P A P^T, after which the contiguous partitions of
// hec_partition have small halos.
#include <algorithm>
#include <cstring>
#include <vector>

#include "hec_internal.h"

namespace hec {

// Undirected adjacency of the pattern of A + A^T without the diagonal, each
// list ascending.
static void sym_adjacency(const CsrView& A, std::vector<int64_t>* ptr, std::vector<int32_t>* adj) {
    const int32_t n = A.n_rows;
    std::vector<int64_t> deg(n + 1, 0);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) {
            const int32_t j = A.col[k];
            if (j == i) continue;
            deg[i]++;
            deg[j]++;
        }
    ptr->assign(n + 1, 0);
    for (int32_t i = 0; i < n; ++i) (*ptr)[i + 1] = (*ptr)[i] + deg[i];
    std::vector<int32_t> tmp((size_t)(*ptr)[n]);
    std::vector<int64_t> pos(ptr->begin(), ptr->end() - 1);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) {
            const int32_t j = A.col[k];
            if (j == i) continue;
            tmp[pos[i]++] = j;
            tmp[pos[j]++] = i;
        }
    // sort + unique each list (A_ij and A_ji both stored give duplicates)
    adj->clear();
    adj->reserve(tmp.size());
    std::vector<int64_t> nptr(n + 1, 0);
    for (int32_t i = 0; i < n; ++i) {
        auto b = tmp.begin() + (*ptr)[i], e = tmp.begin() + (*ptr)[i + 1];
        std::sort(b, e);
        auto u = std::unique(b, e);
        adj->insert(adj->end(), b, u);
        nptr[i + 1] = (int64_t)adj->size();
    }
    ptr->swap(nptr);
}

// BFS levels from `root` inside the unvisited set; returns the last level.
static std::vector<int32_t> bfs_last_level(int32_t root, const std::vector<int64_t>& ptr,
                                           const std::vector<int32_t>& adj, const std::vector<char>& done,
                                           std::vector<int32_t>* mark, int32_t stamp, int32_t* depth) {
    std::vector<int32_t> level{root}, next;
    (*mark)[root] = stamp;
    *depth = 0;
    while (true) {
        next.clear();
        for (int32_t v : level)
            for (int64_t k = ptr[v]; k < ptr[v + 1]; ++k) {
                const int32_t u = adj[k];
                if (!done[u] && (*mark)[u] != stamp) {
                    (*mark)[u] = stamp;
                    next.push_back(u);
                }
            }
        if (next.empty()) return level;
        level.swap(next);
        ++*depth;
    }
}

// Reading A21.  For each connected component in order of its lowest vertex:
//  1. start = its lowest-degree vertex (ties: lowest index); repeat: BFS from
//     start, take the last level's lowest-degree vertex (ties: lowest index);
//     stop when the depth no longer increases (George-Liu pseudo-peripheral);
//  2. Cuthill-McKee BFS from it, each vertex's unvisited neighbours appended in
//     increasing (degree, index) order;
// then reverse the whole sequence.  perm[new] = old.
void rcm_order(const CsrView& A, int32_t* perm) {
    const int32_t n = A.n_rows;
    std::vector<int64_t> ptr;
    std::vector<int32_t> adj;
    sym_adjacency(A, &ptr, &adj);
    auto degree = [&](int32_t v) { return ptr[v + 1] - ptr[v]; };
    auto less_deg = [&](int32_t a, int32_t b) {
        const int64_t da = degree(a), db = degree(b);
        return da != db ? da < db : a < b;
    };
    std::vector<char> done(n, 0);
    std::vector<int32_t> mark(n, -1), order;
    order.reserve(n);
    int32_t stamp = 0;
    for (int32_t seed = 0; seed < n; ++seed) {
        if (done[seed]) continue;
        // the component of `seed`
        std::vector<int32_t> comp{seed};
        ++stamp;
        mark[seed] = stamp;
        for (size_t h = 0; h < comp.size(); ++h)
            for (int64_t k = ptr[comp[h]]; k < ptr[comp[h] + 1]; ++k) {
                const int32_t u = adj[k];
                if (mark[u] != stamp) { mark[u] = stamp; comp.push_back(u); }
            }
        int32_t start = *std::min_element(comp.begin(), comp.end(), less_deg);
        int32_t depth = -1;
        while (true) {
            int32_t d = 0;
            ++stamp;
            std::vector<int32_t> last = bfs_last_level(start, ptr, adj, done, &mark, stamp, &d);
            const int32_t cand = *std::min_element(last.begin(), last.end(), less_deg);
            if (d <= depth || cand == start) break;
            depth = d;
            start = cand;
        }
        // Cuthill-McKee from start
        const size_t base = order.size();
        order.push_back(start);
        done[start] = 1;
        std::vector<int32_t> nb;
        for (size_t h = base; h < order.size(); ++h) {
            const int32_t v = order[h];
            nb.clear();
            for (int64_t k = ptr[v]; k < ptr[v + 1]; ++k)
                if (!done[adj[k]]) nb.push_back(adj[k]);
            std::sort(nb.begin(), nb.end(), less_deg);
            for (int32_t u : nb) { done[u] = 1; order.push_back(u); }
        }
    }
    for (int32_t i = 0; i < n; ++i) perm[i] = order[n - 1 - i];
}

}  // namespace hec

using namespace hec;

extern "C" {

hec_status hec_reorder_rcm(const hec_csr* A, int32_t* perm) {
    if (!perm && A && A->n_rows > 0) return fail(HEC_ERR_ARG, "NULL perm");
    CsrView v;
    hec_status st = validate_csr(A, &v);
    if (st != HEC_OK) return st;
    if (v.n_rows != v.n_cols) return fail(HEC_ERR_DIM, "reordering needs a square matrix");
    try {
        rcm_order(v, perm);
    } catch (...) {
        return fail(HEC_ERR_NOMEM, "host allocation failed in hec_reorder_rcm");
    }
    return HEC_OK;
}

hec_status hec_permute(const hec_csr* A, const int32_t* perm, int32_t* row_ptr_out, int32_t* col_out,
                       double* val_out) {
    CsrView v;
    hec_status st = validate_csr(A, &v);
    if (st != HEC_OK) return st;
    if (v.n_rows != v.n_cols) return fail(HEC_ERR_DIM, "symmetric permutation needs a square matrix");
    const int32_t n = v.n_rows;
    if (n > 0 && (!perm || !row_ptr_out)) return fail(HEC_ERR_ARG, "NULL argument");
    if (v.nnz > 0 && (!col_out || !val_out)) return fail(HEC_ERR_ARG, "NULL argument");
    std::vector<int32_t> inv(n, -1);
    for (int32_t i = 0; i < n; ++i) {
        if (perm[i] < 0 || perm[i] >= n || inv[perm[i]] != -1) return fail(HEC_ERR_ARG, "perm is not a permutation");
        inv[perm[i]] = i;
    }
    // B[i][inv[j]] = A[perm[i]][j]
    row_ptr_out[0] = 0;
    std::vector<std::pair<int32_t, double>> row;
    int64_t p = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t o = perm[i];
        row.clear();
        for (int32_t k = v.row_ptr[o]; k < v.row_ptr[o + 1]; ++k) row.emplace_back(inv[v.col[k]], v.val[k]);
        std::sort(row.begin(), row.end(),
                  [](const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b) { return a.first < b.first; });
        for (const auto& e : row) { col_out[p] = e.first; val_out[p] = e.second; ++p; }
        row_ptr_out[i + 1] = (int32_t)p;
    }
    return HEC_OK;
}

}  // extern "C"
