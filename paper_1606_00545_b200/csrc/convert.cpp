// convert.cpp -- error state, CSR validation and the host CSR -> HEC converter.
//
// HEC = ELL part stored column by column + the irregular remainder in CSR
// (§2.1; P:73 for the column-major layout, the stride "a
// multiple of 32 ... we set it as 256" and the ELL/CSR boundary "a
// recommended value 20").  Readings A1-A4, A7, A15 are stated in DESIGN.md §3.
#include <algorithm>
#include <cstring>
#include <string>

#include "hec_internal.h"

namespace hec {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

hec_status fail(hec_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

hec_status cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? HEC_ERR_NOMEM : HEC_ERR_CUDA;
}

// Reading A7: canonical CSR or HEC_ERR_FORMAT.
hec_status validate_csr(const hec_csr* A, CsrView* out) {
    if (!A) return fail(HEC_ERR_ARG, "NULL csr");
    if (A->n_rows < 0 || A->n_cols < 0 || A->nnz < 0)
        return fail(HEC_ERR_ARG, "negative csr dimension");
    if (!A->row_ptr) return fail(HEC_ERR_ARG, "NULL row_ptr");
    if (A->nnz > 0 && (!A->col_idx || !A->val)) return fail(HEC_ERR_ARG, "NULL col_idx/val");
    if (A->nnz > INT32_MAX) return fail(HEC_ERR_ARG, "nnz exceeds int32 index range");
    const int32_t* rp = A->row_ptr;
    if (rp[0] != 0) return fail(HEC_ERR_FORMAT, "row_ptr[0] != 0");
    if ((int64_t)rp[A->n_rows] != A->nnz) return fail(HEC_ERR_FORMAT, "row_ptr[n_rows] != nnz");
    for (int32_t i = 0; i < A->n_rows; ++i) {
        const int32_t b = rp[i], e = rp[i + 1];
        if (e < b) return fail(HEC_ERR_FORMAT, "row_ptr decreases at row " + std::to_string(i));
        int32_t prev = -1;
        for (int32_t k = b; k < e; ++k) {
            const int32_t c = A->col_idx[k];
            if (c < 0 || c >= A->n_cols)
                return fail(HEC_ERR_FORMAT, "column out of range in row " + std::to_string(i));
            if (c <= prev)
                return fail(HEC_ERR_FORMAT, "unsorted or duplicate column in row " + std::to_string(i));
            prev = c;
        }
    }
    out->n_rows = A->n_rows;
    out->n_cols = A->n_cols;
    out->nnz = A->nnz;
    out->row_ptr = A->row_ptr;
    out->col = A->col_idx;
    out->val = A->val;
    return HEC_OK;
}

hec_opts normalise_opts(const hec_opts* o) {
    hec_opts d;
    hec_opts_default(&d);
    return o ? *o : d;
}

hec_status check_opts(const hec_opts& o) {
    if (o.width_policy < HEC_WIDTH_BG3 || o.width_policy > HEC_WIDTH_FIXED)
        return fail(HEC_ERR_ARG, "unknown width_policy");
    if (o.cap < 0) return fail(HEC_ERR_ARG, "negative cap");
    if (o.width_policy == HEC_WIDTH_FIXED && o.fixed_width < 0)
        return fail(HEC_ERR_ARG, "negative fixed_width");
    if (o.stride_unit <= 0 || o.stride_unit % 32 != 0)
        return fail(HEC_ERR_ARG, "stride_unit must be a positive multiple of 32 (P:73)");
    return HEC_OK;
}

// Reading A1.  BG3: k* = smallest k >= 0 with 3 #{rows: len > k} < n,
// computed from the row-length histogram; w = min(cap, k*).
int32_t choose_width(const CsrView& A, const hec_opts& o) {
    if (o.width_policy == HEC_WIDTH_FIXED) return o.fixed_width;
    const int32_t n = A.n_rows;
    if (n == 0) return 0;
    int32_t max_len = 0;
    for (int32_t i = 0; i < n; ++i) max_len = std::max(max_len, A.row_ptr[i + 1] - A.row_ptr[i]);
    if (o.width_policy == HEC_WIDTH_CAP) return std::min(o.cap, max_len);
    std::vector<int64_t> hist((size_t)max_len + 2, 0);
    for (int32_t i = 0; i < n; ++i) hist[A.row_ptr[i + 1] - A.row_ptr[i]]++;
    int64_t longer = n - hist[0];  // #{len > 0}
    int32_t k = 0;
    while (3 * longer >= (int64_t)n) {  // k is not yet below the one-third threshold
        ++k;
        longer -= hist[k];              // #{len > k}
    }
    return std::min(o.cap, k);
}

// Readings A2-A4, A15: s = roundup(n, unit); slot j of row i at j*s + i holds
// the row's j-th entry (j < min(len, w)) or (-1, +0.0); spilled entries go,
// in order, to a compact CSR tail of the rows with len > w.
hec_status convert(const CsrView& A, int32_t width, int32_t stride_unit, HostHec* out) {
    const int32_t n = A.n_rows;
    const int64_t s64 = ((int64_t)n + stride_unit - 1) / stride_unit * stride_unit;
    if (s64 > INT32_MAX) return fail(HEC_ERR_ARG, "stride exceeds int32");
    const int32_t s = (int32_t)s64;
    out->n_rows = n;
    out->n_cols = A.n_cols;
    out->width = width;
    out->stride = s;
    out->nnz = A.nnz;
    const size_t slots = (size_t)width * (size_t)s;
    try {
        out->ell_col.assign(slots, -1);
        out->ell_val.assign(slots, 0.0);
        out->tail_rows.clear();
        out->tail_ptr.assign(1, 0);
        out->tail_col.clear();
        out->tail_val.clear();
    } catch (...) {
        return fail(HEC_ERR_NOMEM, "host allocation for HEC arrays failed");
    }
    int64_t ell_nnz = 0, tail_nnz = 0;
    int32_t tail_rows = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t len = A.row_ptr[i + 1] - A.row_ptr[i];
        if (len > width) { ++tail_rows; tail_nnz += len - width; }
    }
    try {
        out->tail_rows.reserve(tail_rows);
        out->tail_ptr.reserve((size_t)tail_rows + 1);
        out->tail_col.reserve((size_t)tail_nnz);
        out->tail_val.reserve((size_t)tail_nnz);
    } catch (...) {
        return fail(HEC_ERR_NOMEM, "host allocation for HEC tail failed");
    }
    int32_t* ec = out->ell_col.data();
    double* ev = out->ell_val.data();
    for (int32_t i = 0; i < n; ++i) {
        const int32_t b = A.row_ptr[i], e = A.row_ptr[i + 1];
        const int32_t m = std::min(e - b, width);
        for (int32_t j = 0; j < m; ++j) {
            ec[(size_t)j * s + i] = A.col[b + j];
            ev[(size_t)j * s + i] = A.val[b + j];
        }
        ell_nnz += m;
        if (e - b > width) {
            out->tail_rows.push_back(i);
            out->tail_col.insert(out->tail_col.end(), A.col + b + width, A.col + e);
            out->tail_val.insert(out->tail_val.end(), A.val + b + width, A.val + e);
            out->tail_ptr.push_back((int32_t)out->tail_col.size());
        }
    }
    out->ell_nnz = ell_nnz;
    return HEC_OK;
}

}  // namespace hec

extern "C" {

void hec_opts_default(hec_opts* o) {
    if (!o) return;
    o->width_policy = HEC_WIDTH_BG3;
    o->cap = 20;         // P:73 "a recommended value 20"
    o->fixed_width = 0;
    o->stride_unit = 256;  // P:73 "we set it as 256"
}

const char* hec_last_error(void) { return hec::g_err.c_str(); }

const char* hec_version(void) { return "hec-b200 0.1 (sm_100a)"; }

}  // extern "C"
