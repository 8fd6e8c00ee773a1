// plan.cpp -- row partition and halo plan (host).
//
// PAPER.md §2.2: the matrix is partitioned by rows ("sequence
// partition" for FDM/FVM matrices), the vector is split into conformal
// segments, and each part receives the x entries its segment "can not
// provide".  Readings A9-A12 fix the partition rules, the halo
// ordering and the interior/boundary split.
#include <algorithm>
#include <cstring>
#include <memory>

#include "hec_internal.h"

namespace hec {

static hec_status make_part_ptr(const CsrView& A, int32_t P, int32_t kind, const int32_t* grid,
                                std::vector<int32_t>* pp) {
    const int32_t n = A.n_rows;
    pp->assign((size_t)P + 1, 0);
    (*pp)[P] = n;
    if (kind == HEC_PART_CONTIG_ROWS) {
        for (int32_t p = 1; p < P; ++p) (*pp)[p] = (int32_t)(((int64_t)p * n) / P);
    } else if (kind == HEC_PART_GRID) {
        if (!grid) return fail(HEC_ERR_ARG, "GRID partition needs grid dims");
        const int64_t nx = grid[0], ny = grid[1], nz = grid[2];
        if (nx < 1 || ny < 1 || nz < 1 || nx * ny * nz != n)
            return fail(HEC_ERR_PARTS, "grid dims do not match n_rows");
        int64_t ext, plane;
        if (nz > 1) { ext = nz; plane = nx * ny; }
        else if (ny > 1) { ext = ny; plane = nx; }
        else { ext = nx; plane = 1; }
        if (P > ext) return fail(HEC_ERR_PARTS, "more parts than grid planes");
        for (int32_t p = 1; p < P; ++p) (*pp)[p] = (int32_t)(((int64_t)p * ext / P) * plane);
    } else if (kind == HEC_PART_CONTIG_NNZ) {
        const int64_t nnz = A.nnz;
        for (int32_t p = 1; p < P; ++p) {
            const int64_t t = ((int64_t)p * nnz + P - 1) / P;  // ceil(p nnz / P)
            const int32_t* lb = std::lower_bound(A.row_ptr, A.row_ptr + n + 1, t,
                                                 [](int32_t a, int64_t b) { return (int64_t)a < b; });
            int32_t r = (int32_t)(lb - A.row_ptr);
            r = std::max(r, (*pp)[p - 1] + 1);
            r = std::min(r, n - (P - p));
            (*pp)[p] = r;
        }
    } else if (kind == HEC_PART_CONTIG_COST) {
        // Modeled-cost balance: row i of part p costs
        // kCostSlot * w_p + kCostTail * max(len_i - w_p, 0) with w_p the part's
        // own BG3 width (A1/A12: padded ELL slots + tail entries); start from
        // CONTIG_NNZ and re-balance kCostIters times (fixed count: deterministic).
        constexpr int64_t kCostSlot = 3, kCostTail = 4;
        constexpr int kCostIters = 4;
        std::vector<int32_t> cur;
        hec_status st = make_part_ptr(A, P, HEC_PART_CONTIG_NNZ, nullptr, &cur);
        if (st != HEC_OK) return st;
        hec_opts o;
        hec_opts_default(&o);
        std::vector<int64_t> S((size_t)n + 1);
        for (int it = 0; it < kCostIters; ++it) {
            S[0] = 0;
            for (int32_t p = 0; p < P; ++p) {
                CsrView v;
                v.n_rows = cur[p + 1] - cur[p];
                v.n_cols = A.n_cols;
                v.row_ptr = A.row_ptr + cur[p];  // lengths only (differences)
                v.nnz = A.row_ptr[cur[p + 1]] - A.row_ptr[cur[p]];
                const int64_t w = choose_width(v, o);
                for (int32_t i = cur[p]; i < cur[p + 1]; ++i) {
                    const int64_t len = A.row_ptr[i + 1] - A.row_ptr[i];
                    S[i + 1] = S[i] + kCostSlot * w + kCostTail * std::max<int64_t>(len - w, 0);
                }
            }
            std::vector<int32_t> nxt((size_t)P + 1, 0);
            nxt[P] = n;
            const int64_t C = S[n];
            for (int32_t p = 1; p < P; ++p) {
                const int64_t t = (p * C + P - 1) / P;  // ceil(p C / P)
                int32_t r = (int32_t)(std::lower_bound(S.begin(), S.end(), t) - S.begin());
                r = std::max(r, nxt[p - 1] + 1);
                r = std::min(r, n - (P - p));
                nxt[p] = r;
            }
            if (nxt == cur) break;
            cur.swap(nxt);
        }
        *pp = cur;
    } else if (kind == HEC_PART_EXPLICIT) {
        if (!grid) return fail(HEC_ERR_ARG, "EXPLICIT partition needs part_ptr");
        if (grid[0] != 0 || grid[P] != n) return fail(HEC_ERR_PARTS, "part_ptr must run from 0 to n_rows");
        for (int32_t p = 0; p < P; ++p) {
            if (grid[p + 1] <= grid[p]) return fail(HEC_ERR_PARTS, "part_ptr must be strictly increasing");
            (*pp)[p] = grid[p];
        }
    } else {
        return fail(HEC_ERR_ARG, "unknown partition kind");
    }
    return HEC_OK;
}

static inline int32_t owner_of(const std::vector<int32_t>& pp, int32_t j) {
    return (int32_t)(std::upper_bound(pp.begin(), pp.end(), j) - pp.begin()) - 1;
}

hec_status build_plan(const CsrView& A, int32_t P, int32_t kind, const int32_t* grid,
                      hec_plan_s* plan) {
    plan->n_parts = P;
    plan->n_rows = A.n_rows;
    plan->nnz = A.nnz;
    plan->row_ptr.assign(A.row_ptr, A.row_ptr + A.n_rows + 1);
    hec_status st = make_part_ptr(A, P, kind, grid, &plan->part_ptr);
    if (st != HEC_OK) return st;
    const std::vector<int32_t>& pp = plan->part_ptr;
    plan->parts.assign(P, PartPlan());
    // recv sets, interior / boundary rows
    for (int32_t p = 0; p < P; ++p) {
        PartPlan& pt = plan->parts[p];
        pt.r0 = pp[p];
        pt.r1 = pp[p + 1];
        std::vector<int32_t> cand;
        for (int32_t i = pt.r0; i < pt.r1; ++i) {
            bool outside = false;
            for (int32_t k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) {
                const int32_t j = A.col[k];
                if (j < pt.r0 || j >= pt.r1) { cand.push_back(j); outside = true; }
            }
            (outside ? pt.boundary : pt.interior).push_back(i - pt.r0);
        }
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        pt.recv.swap(cand);
        // recv grouped by owner (ascending columns => ascending owners), A10
        pt.recv_off.assign((size_t)P + 1, 0);
        for (int32_t j : pt.recv) pt.recv_off[owner_of(pp, j) + 1]++;
        for (int32_t q = 0; q < P; ++q) pt.recv_off[q + 1] += pt.recv_off[q];
    }
    // send lists: send_{p->q} = recv_q restricted to part p, minus r0_p (sorted)
    for (int32_t p = 0; p < P; ++p) {
        PartPlan& pt = plan->parts[p];
        pt.send_off.assign((size_t)P + 1, 0);
        pt.send_idx.clear();
        for (int32_t q = 0; q < P; ++q) {
            if (q != p) {
                const PartPlan& pq = plan->parts[q];
                for (int32_t t = pq.recv_off[p]; t < pq.recv_off[p + 1]; ++t)
                    pt.send_idx.push_back(pq.recv[t] - pt.r0);
            }
            pt.send_off[q + 1] = (int32_t)pt.send_idx.size();
        }
    }
    return HEC_OK;
}

// Local sub-matrix: owned column c -> c - r0; halo column g -> n_loc + pos(g)
// (A10).  Local order within a row: owned columns (ascending), then halo
// columns below r0, then halo columns at/above r1 -- which is ascending local id.
hec_status build_local_csr(const hec_plan_s& P, const CsrView& A, int32_t part, int32_t which,
                           CsrOwned* out) {
    const PartPlan& pt = P.parts[part];
    const int32_t n_loc = pt.r1 - pt.r0;
    std::vector<int32_t> all;
    const std::vector<int32_t>* rows;
    if (which == HEC_SUB_INTERIOR) rows = &pt.interior;
    else if (which == HEC_SUB_BOUNDARY) rows = &pt.boundary;
    else if (which == HEC_SUB_ALL) {
        all.resize(n_loc);
        for (int32_t i = 0; i < n_loc; ++i) all[i] = i;
        rows = &all;
    } else {
        return fail(HEC_ERR_ARG, "unknown sub-matrix kind");
    }
    out->n_rows = (int32_t)rows->size();
    out->n_cols = n_loc + (int32_t)pt.recv.size();
    out->row_ptr.assign((size_t)out->n_rows + 1, 0);
    int64_t nnz = 0;
    for (size_t r = 0; r < rows->size(); ++r) {
        const int32_t i = pt.r0 + (*rows)[r];
        nnz += A.row_ptr[i + 1] - A.row_ptr[i];
    }
    out->col.resize((size_t)nnz);
    out->val.resize((size_t)nnz);
    int64_t p = 0;
    for (size_t r = 0; r < rows->size(); ++r) {
        const int32_t i = pt.r0 + (*rows)[r];
        const int32_t b = A.row_ptr[i], e = A.row_ptr[i + 1];
        // columns ascending: [b, lo) below r0, [lo, hi) owned, [hi, e) above
        int32_t lo = b, hi;
        while (lo < e && A.col[lo] < pt.r0) ++lo;
        hi = lo;
        while (hi < e && A.col[hi] < pt.r1) ++hi;
        for (int32_t k = lo; k < hi; ++k) { out->col[p] = A.col[k] - pt.r0; out->val[p++] = A.val[k]; }
        auto halo = [&](int32_t k) {
            const int32_t g = A.col[k];
            const int32_t pos = (int32_t)(std::lower_bound(pt.recv.begin(), pt.recv.end(), g) - pt.recv.begin());
            out->col[p] = n_loc + pos;
            out->val[p++] = A.val[k];
        };
        for (int32_t k = b; k < lo; ++k) halo(k);
        for (int32_t k = hi; k < e; ++k) halo(k);
        out->row_ptr[r + 1] = (int32_t)p;
    }
    return HEC_OK;
}

// Reading A12: the partition width comes from all its local rows (a local row
// has the same length as the global row).
int32_t part_width(const hec_plan_s& P, int32_t part, const hec_opts& o) {
    const PartPlan& pt = P.parts[part];
    CsrView v;
    v.n_rows = pt.r1 - pt.r0;
    v.n_cols = P.n_rows;
    std::vector<int32_t> rp((size_t)v.n_rows + 1);
    for (int32_t i = 0; i <= v.n_rows; ++i) rp[i] = P.row_ptr[pt.r0 + i] - P.row_ptr[pt.r0];
    v.row_ptr = rp.data();
    v.nnz = rp[v.n_rows];
    return choose_width(v, o);
}

}  // namespace hec

using namespace hec;

extern "C" {

hec_status hec_partition(const hec_csr* A, int32_t n_parts, int32_t kind, const int32_t* grid,
                         hec_plan* out) {
    if (!out) return fail(HEC_ERR_ARG, "NULL out");
    *out = nullptr;
    CsrView v;
    hec_status st = validate_csr(A, &v);
    if (st != HEC_OK) return st;
    if (v.n_rows != v.n_cols) return fail(HEC_ERR_DIM, "partitioning needs a square matrix (A14)");
    if (n_parts < 1 || n_parts > v.n_rows) return fail(HEC_ERR_PARTS, "n_parts out of [1, n_rows]");
    std::unique_ptr<hec_plan_s> plan;
    try {
        plan.reset(new hec_plan_s());
        st = build_plan(v, n_parts, kind, grid, plan.get());
    } catch (...) {
        return fail(HEC_ERR_NOMEM, "host allocation failed in hec_partition");
    }
    if (st != HEC_OK) return st;
    *out = plan.release();
    return HEC_OK;
}

hec_status hec_plan_n_parts(hec_plan P, int32_t* n) {
    if (!P || !n) return fail(HEC_ERR_ARG, "NULL argument");
    *n = P->n_parts;
    return HEC_OK;
}

hec_status hec_plan_part_ptr(hec_plan P, int32_t* pp) {
    if (!P || !pp) return fail(HEC_ERR_ARG, "NULL argument");
    std::memcpy(pp, P->part_ptr.data(), sizeof(int32_t) * P->part_ptr.size());
    return HEC_OK;
}

static void fill_info(const PartPlan& pt, int32_t P, hec_part_info* o) {
    o->r0 = pt.r0;
    o->r1 = pt.r1;
    o->n_halo = (int32_t)pt.recv.size();
    o->n_send = (int32_t)pt.send_idx.size();
    o->n_interior = (int32_t)pt.interior.size();
    o->n_boundary = (int32_t)pt.boundary.size();
    o->n_recv_peers = 0;
    o->n_send_peers = 0;
    for (int32_t q = 0; q < P; ++q) {
        o->n_recv_peers += pt.recv_off[q + 1] > pt.recv_off[q];
        o->n_send_peers += pt.send_off[q + 1] > pt.send_off[q];
    }
    o->width = -1;
    o->reserved = 0;
}

hec_status hec_plan_part_info(hec_plan P, int32_t part, hec_part_info* out) {
    if (!P || !out) return fail(HEC_ERR_ARG, "NULL argument");
    if (part < 0 || part >= P->n_parts) return fail(HEC_ERR_PARTS, "part out of range");
    return hec_plan_part_info_opts(P, part, nullptr, out);
}

hec_status hec_plan_part_info_opts(hec_plan P, int32_t part, const hec_opts* o, hec_part_info* out) {
    if (!P || !out) return fail(HEC_ERR_ARG, "NULL argument");
    if (part < 0 || part >= P->n_parts) return fail(HEC_ERR_PARTS, "part out of range");
    const hec_opts op = normalise_opts(o);
    hec_status st = check_opts(op);
    if (st != HEC_OK) return st;
    fill_info(P->parts[part], P->n_parts, out);
    out->width = part_width(*P, part, op);
    return HEC_OK;
}

hec_status hec_plan_export(hec_plan P, int32_t part, hec_plan_arrays* out) {
    if (!P || !out) return fail(HEC_ERR_ARG, "NULL argument");
    if (part < 0 || part >= P->n_parts) return fail(HEC_ERR_PARTS, "part out of range");
    const PartPlan& pt = P->parts[part];
    auto cp = [](int32_t* dst, const std::vector<int32_t>& src) {
        if (dst && !src.empty()) std::memcpy(dst, src.data(), sizeof(int32_t) * src.size());
    };
    cp(out->recv_cols, pt.recv);
    cp(out->recv_off, pt.recv_off);
    cp(out->send_idx, pt.send_idx);
    cp(out->send_off, pt.send_off);
    cp(out->interior, pt.interior);
    cp(out->boundary, pt.boundary);
    return HEC_OK;
}

void hec_plan_free(hec_plan P) { delete P; }

}  // extern "C"
