// api.cpp -- the single-GPU C ABI: hec_from_csr / hec_info / hec_export /
// hec_spmv / hec_spmv_host / hec_free and hec_plan_part_hec.
//
// hec_spmv is Alg. 1 of PAPER.md: the ELL part "is performed
// firstly" by ell_kernel, then the CSR part by tail_kernel, both on the
// caller's stream (stream order gives the ELL -> CSR ordering).
#include <cstring>
#include <memory>

#include "hec_internal.h"

namespace hec {

template <typename T>
static hec_status dmalloc_copy(T** dst, const T* src, size_t n, cudaStream_t s, int64_t* bytes) {
    *dst = nullptr;
    if (n == 0) return HEC_OK;
    HEC_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(dst), n * sizeof(T)));
    *bytes += (int64_t)(n * sizeof(T));
    if (src) HEC_CUDA_TRY(cudaMemcpyAsync(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
    return HEC_OK;
}

static void release(hec_matrix_s* m) {
    if (!m) return;
    if (m->device >= 0) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(m->device);
        void* ptrs[] = {m->d_ell_col, m->d_ell_val, m->d_tail_out, m->d_tail_order, m->d_tail_ptr, m->d_tail_col,
                        m->d_tail_val, m->d_rowmap, m->d_stage_x, m->d_stage_y};
        for (void* p : ptrs)
            if (p) cudaFree(p);
        cudaSetDevice(cur);
    }
    delete m;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (dev >= 0 && dev != prev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

hec_status make_matrix(HostHec&& h, int32_t device, cudaStream_t s, const int32_t* rowmap,
                       int32_t n_rowmap, int32_t row_off, int32_t n_loc, hec_matrix* out) {
    std::unique_ptr<hec_matrix_s, void (*)(hec_matrix_s*)> m(new (std::nothrow) hec_matrix_s(),
                                                             release);
    if (!m) return fail(HEC_ERR_NOMEM, "host allocation failed");
    m->device = device;
    m->n_rows = h.n_rows;
    m->n_cols = h.n_cols;
    m->width = h.width;
    m->stride = h.stride;
    m->nnz = h.nnz;
    m->ell_nnz = h.ell_nnz;
    m->tail_rows = (int32_t)h.tail_rows.size();
    m->tail_nnz = (int64_t)h.tail_col.size();
    // bin the tail rows by spilled length (tail kernel lanes per row)
    std::vector<int32_t> order(h.tail_rows.size());
    {
        int64_t cnt[kTailBins] = {0};
        for (size_t t = 0; t < order.size(); ++t) cnt[tail_bin_of(h.tail_ptr[t + 1] - h.tail_ptr[t])]++;
        m->tail_bin_off[0] = 0;
        for (int b = 0; b < kTailBins; ++b) m->tail_bin_off[b + 1] = m->tail_bin_off[b] + cnt[b];
        int64_t pos[kTailBins];
        for (int b = 0; b < kTailBins; ++b) pos[b] = m->tail_bin_off[b];
        for (size_t t = 0; t < order.size(); ++t)
            order[pos[tail_bin_of(h.tail_ptr[t + 1] - h.tail_ptr[t])]++] = (int32_t)t;
        int best = 0;
        for (int b = 1; b < kTailBins; ++b) if (cnt[b] > cnt[best]) best = b;
        m->tail_group = 1 << best;
    }
    m->h_tail_rows = h.tail_rows;
    m->row_off = row_off;
    m->n_loc = n_loc;
    if (device < 0) {
        m->host = std::move(h);
        *out = m.release();
        return HEC_OK;
    }
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0)
        return fail(HEC_ERR_NODEV, "no CUDA device available");
    if (device >= n_dev) return fail(HEC_ERR_ARG, "device ordinal out of range");
    DeviceGuard g(device);
    int64_t bytes = 0;
    hec_status st;
    if ((st = dmalloc_copy(&m->d_ell_col, h.ell_col.data(), h.ell_col.size(), s, &bytes))) return st;
    if ((st = dmalloc_copy(&m->d_ell_val, h.ell_val.data(), h.ell_val.size(), s, &bytes))) return st;
    std::vector<int32_t> tail_out(h.tail_rows.size());
    for (size_t t = 0; t < tail_out.size(); ++t)
        tail_out[t] = rowmap ? rowmap[h.tail_rows[t]] : row_off + h.tail_rows[t];
    if ((st = dmalloc_copy(&m->d_tail_out, tail_out.data(), tail_out.size(), s, &bytes))) return st;
    if ((st = dmalloc_copy(&m->d_tail_order, order.data(), order.size(), s, &bytes))) return st;
    if (!h.tail_rows.empty())
        if ((st = dmalloc_copy(&m->d_tail_ptr, h.tail_ptr.data(), h.tail_ptr.size(), s, &bytes))) return st;
    if ((st = dmalloc_copy(&m->d_tail_col, h.tail_col.data(), h.tail_col.size(), s, &bytes))) return st;
    if ((st = dmalloc_copy(&m->d_tail_val, h.tail_val.data(), h.tail_val.size(), s, &bytes))) return st;
    if (rowmap)
        if ((st = dmalloc_copy(&m->d_rowmap, rowmap, (size_t)n_rowmap, s, &bytes))) return st;
    HEC_CUDA_TRY(cudaStreamSynchronize(s));  // host vectors die after return
    m->device_bytes = bytes;
    *out = m.release();
    return HEC_OK;
}

hec_status launch_spmv(const hec_matrix_s* A, const double* x, const double* x_halo, double* y,
                       cudaStream_t s) {
    EllArgs e;
    e.col = A->d_ell_col;
    e.val = A->d_ell_val;
    e.stride = A->stride;
    e.n_rows = A->n_rows;
    e.width = A->width;
    e.x = x;
    e.x_halo = x_halo;
    e.n_loc = A->n_loc >= 0 ? A->n_loc : A->n_cols;
    e.y = y;
    e.rowmap = A->d_rowmap;
    e.row_off = A->row_off;
    cudaError_t err = launch_ell(e, s);  // Alg. 1 lines 1-3: ELL first
    if (err != cudaSuccess) return cuda_fail(err, "ell_kernel launch");
    if (A->tail_rows > 0) {              // Alg. 1 lines 5-7: then the CSR part
        TailArgs t;
        t.n_tail = A->tail_rows;
        t.order = A->d_tail_order;
        for (int b = 0; b <= kTailBins; ++b) t.bin_off[b] = A->tail_bin_off[b];
        t.out_rows = A->d_tail_out;
        t.ptr = A->d_tail_ptr;
        t.col = A->d_tail_col;
        t.val = A->d_tail_val;
        t.x = x;
        t.x_halo = x_halo;
        t.n_loc = e.n_loc;
        t.y = y;
        err = launch_tail(t, s);
        if (err != cudaSuccess) return cuda_fail(err, "tail_kernel launch");
    }
    return HEC_OK;
}

}  // namespace hec

using namespace hec;

extern "C" {

hec_status hec_from_csr(const hec_csr* A, const hec_opts* o, int32_t device, void* stream,
                        hec_matrix* out) {
    if (!out) return fail(HEC_ERR_ARG, "NULL out");
    *out = nullptr;
    if (device < -1) return fail(HEC_ERR_ARG, "device must be >= -1");
    CsrView v;
    hec_status st = validate_csr(A, &v);
    if (st != HEC_OK) return st;
    const hec_opts op = normalise_opts(o);
    if ((st = check_opts(op)) != HEC_OK) return st;
    HostHec h;
    try {
        st = convert(v, choose_width(v, op), op.stride_unit, &h);
    } catch (...) {
        return fail(HEC_ERR_NOMEM, "host allocation failed in hec_from_csr");
    }
    if (st != HEC_OK) return st;
    return make_matrix(std::move(h), device, (cudaStream_t)stream, nullptr, 0, 0, -1, out);
}

hec_status hec_info(hec_matrix A, hec_matrix_info* o) {
    if (!A || !o) return fail(HEC_ERR_ARG, "NULL argument");
    o->n_rows = A->n_rows;
    o->n_cols = A->n_cols;
    o->ell_width = A->width;
    o->ell_stride = A->stride;
    o->nnz = A->nnz;
    o->ell_nnz = A->ell_nnz;
    o->tail_rows = A->tail_rows;
    o->tail_group = A->tail_group;
    o->tail_nnz = A->tail_nnz;
    o->device_bytes = A->device_bytes;
    o->device = A->device;
    o->reserved = 0;
    return HEC_OK;
}

hec_status hec_export(hec_matrix A, hec_host_arrays* o) {
    if (!A || !o) return fail(HEC_ERR_ARG, "NULL argument");
    const size_t slots = (size_t)A->width * (size_t)A->stride;
    if (o->tail_rows && A->tail_rows)
        std::memcpy(o->tail_rows, A->h_tail_rows.data(), sizeof(int32_t) * A->tail_rows);
    if (A->device < 0) {
        const HostHec& h = A->host;
        if (o->ell_col && slots) std::memcpy(o->ell_col, h.ell_col.data(), slots * sizeof(int32_t));
        if (o->ell_val && slots) std::memcpy(o->ell_val, h.ell_val.data(), slots * sizeof(double));
        if (o->tail_ptr) std::memcpy(o->tail_ptr, h.tail_ptr.data(), h.tail_ptr.size() * sizeof(int32_t));
        if (o->tail_col && A->tail_nnz) std::memcpy(o->tail_col, h.tail_col.data(), A->tail_nnz * sizeof(int32_t));
        if (o->tail_val && A->tail_nnz) std::memcpy(o->tail_val, h.tail_val.data(), A->tail_nnz * sizeof(double));
        return HEC_OK;
    }
    DeviceGuard g(A->device);
    if (o->ell_col && slots) HEC_CUDA_TRY(cudaMemcpy(o->ell_col, A->d_ell_col, slots * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (o->ell_val && slots) HEC_CUDA_TRY(cudaMemcpy(o->ell_val, A->d_ell_val, slots * sizeof(double), cudaMemcpyDeviceToHost));
    if (o->tail_ptr) {
        if (A->tail_rows)
            HEC_CUDA_TRY(cudaMemcpy(o->tail_ptr, A->d_tail_ptr, ((size_t)A->tail_rows + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
        else
            o->tail_ptr[0] = 0;
    }
    if (o->tail_col && A->tail_nnz) HEC_CUDA_TRY(cudaMemcpy(o->tail_col, A->d_tail_col, A->tail_nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (o->tail_val && A->tail_nnz) HEC_CUDA_TRY(cudaMemcpy(o->tail_val, A->d_tail_val, A->tail_nnz * sizeof(double), cudaMemcpyDeviceToHost));
    return HEC_OK;
}

static hec_status check_xy(hec_matrix A, const double* x, double* y) {
    if (!A) return fail(HEC_ERR_ARG, "NULL matrix");
    if (A->device < 0) return fail(HEC_ERR_NODEV, "host-only matrix handle (device = -1); no CPU fallback");
    if (A->n_rows > 0 && !y) return fail(HEC_ERR_ARG, "NULL y");
    if (A->n_cols > 0 && !x && A->nnz > 0) return fail(HEC_ERR_ARG, "NULL x");
    if (x && y) {
        const char* xb = reinterpret_cast<const char*>(x);
        const char* xe = xb + sizeof(double) * (size_t)A->n_cols;
        const char* yb = reinterpret_cast<const char*>(y);
        const char* ye = yb + sizeof(double) * (size_t)A->n_rows;
        if (xb < ye && yb < xe && A->n_rows > 0 && A->n_cols > 0)
            return fail(HEC_ERR_ARG, "x and y overlap");
    }
    return HEC_OK;
}

hec_status hec_spmv(hec_matrix A, const double* x, double* y, void* stream) {
    hec_status st = check_xy(A, x, y);
    if (st != HEC_OK) return st;
    if (A->n_rows == 0) return HEC_OK;
    DeviceGuard g(A->device);
    return launch_spmv(A, x, nullptr, y, (cudaStream_t)stream);
}

hec_status hec_spmv_host(hec_matrix A, const double* x_host, double* y_host, void* stream) {
    if (!A) return fail(HEC_ERR_ARG, "NULL matrix");
    if (A->device < 0) return fail(HEC_ERR_NODEV, "host-only matrix handle (device = -1); no CPU fallback");
    if ((A->n_cols > 0 && !x_host) || (A->n_rows > 0 && !y_host)) return fail(HEC_ERR_ARG, "NULL host vector");
    if (A->n_rows == 0) return HEC_OK;
    DeviceGuard g(A->device);
    cudaStream_t s = (cudaStream_t)stream;
    if (!A->d_stage_x && A->n_cols > 0) {
        HEC_CUDA_TRY(cudaMalloc(&A->d_stage_x, sizeof(double) * (size_t)A->n_cols));
        A->device_bytes += sizeof(double) * (int64_t)A->n_cols;
    }
    if (!A->d_stage_y) {
        HEC_CUDA_TRY(cudaMalloc(&A->d_stage_y, sizeof(double) * (size_t)A->n_rows));
        A->device_bytes += sizeof(double) * (int64_t)A->n_rows;
    }
    if (A->n_cols > 0)
        HEC_CUDA_TRY(cudaMemcpyAsync(A->d_stage_x, x_host, sizeof(double) * (size_t)A->n_cols,
                                     cudaMemcpyHostToDevice, s));
    hec_status st = launch_spmv(A, A->d_stage_x, nullptr, A->d_stage_y, s);
    if (st != HEC_OK) return st;
    HEC_CUDA_TRY(cudaMemcpyAsync(y_host, A->d_stage_y, sizeof(double) * (size_t)A->n_rows,
                                 cudaMemcpyDeviceToHost, s));
    HEC_CUDA_TRY(cudaStreamSynchronize(s));
    return HEC_OK;
}

int32_t hec_spmv_launches(hec_matrix A) {
    if (!A || A->n_rows == 0) return 0;
    return 1 + (A->tail_rows > 0 ? 1 : 0);
}

void hec_free(hec_matrix A) { release(A); }

hec_status hec_plan_part_hec(hec_plan P, const hec_csr* A, int32_t part, int32_t which,
                             const hec_opts* o, int32_t device, void* stream, hec_matrix* out) {
    if (!P || !out) return fail(HEC_ERR_ARG, "NULL argument");
    *out = nullptr;
    if (part < 0 || part >= P->n_parts) return fail(HEC_ERR_PARTS, "part out of range");
    CsrView v;
    hec_status st = validate_csr(A, &v);
    if (st != HEC_OK) return st;
    if (v.n_rows != P->n_rows || v.nnz != P->nnz) return fail(HEC_ERR_STATE, "matrix does not match the plan");
    const hec_opts op = normalise_opts(o);
    if ((st = check_opts(op)) != HEC_OK) return st;
    CsrOwned L;
    HostHec h;
    try {
        if ((st = build_local_csr(*P, v, part, which, &L)) != HEC_OK) return st;
        if ((st = convert(L.view(), part_width(*P, part, op), op.stride_unit, &h)) != HEC_OK) return st;
    } catch (...) {
        return fail(HEC_ERR_NOMEM, "host allocation failed in hec_plan_part_hec");
    }
    const int32_t n_loc = P->parts[part].r1 - P->parts[part].r0;
    return make_matrix(std::move(h), device, (cudaStream_t)stream, nullptr, 0, 0, n_loc, out);
}

}  // extern "C"
