// dist.cpp -- row-partitioned HEC SpMV with halo exchange (one process per GPU).
//
// PAPER.md §2.2: each GPU holds one (partition matrix, segment
// vector) pair; the x entries a segment "can not provide" are exchanged -- in
// the paper through a host-resident shared cache.  Here (reading A13) the
// exchange is device to device: a pack kernel gathers x_local[send_idx] into a
// contiguous send buffer and grouped NCCL send/recv over NVLink deliver each
// peer's slice into this rank's x_halo (ordered by peer, reading A10).  The
// rows are split into interior (x_local only) and boundary (reading A11): the
// interior SpMV runs on the caller's stream while the pack + exchange run on a
// high-priority communication stream; the boundary SpMV waits for the halo.
#include <cstring>
#include <memory>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: host ranges around each phase's enqueue (nsys)

#include "hec_internal.h"

struct LocalGroup;

struct hec_dist_s {
    int32_t rank = 0, n_parts = 1, device = 0;
    int32_t r0 = 0, r1 = 0, n_halo = 0, n_send = 0;
    int32_t n_interior = 0, n_boundary = 0, width = 0;
    int64_t nnz_local = 0;
    hec_matrix interior = nullptr, boundary = nullptr;
    int32_t* d_send_idx = nullptr;
    double* d_sendbuf = nullptr;
    double* d_x_halo = nullptr;
    std::vector<int32_t> send_off, recv_off;
    ncclComm_t comm = nullptr;
    bool local = false;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_start = nullptr, ev_halo = nullptr;
    int64_t device_bytes = 0;
    // ---- peer-memory transport ----
    bool p2p = false;
    void* d_win = nullptr;              // [flags: n_parts u64, 256 B aligned][halo buf 0][halo buf 1]
    std::vector<void*> opened;          // peer windows mapped with cudaIpcOpenMemHandle
    std::vector<int32_t> nbr;           // neighbour ranks (send or receive side), ascending
    std::vector<int4> push_chunks;      // {destination rank, first send entry, end, halo position there}
    std::vector<int64_t> all_nhalo;     // every rank's halo length (from the plan)
    int4* d_push_chunks = nullptr;
    int32_t* d_nbr = nullptr;
    void* d_peer_tab = nullptr;         // [buf0 ptrs | flag ptrs | n_halo] per rank
    unsigned int* d_done = nullptr;
    int32_t* d_err = nullptr;
    uint64_t epoch = 0;
    void* ws = nullptr;                 // Krylov workspace (krylov.cu), freed through ws_free
    void (*ws_free)(void*) = nullptr;
    double* d_stage_x = nullptr;        // hec_spmv_dist_host staging (first call)
    double* d_stage_y = nullptr;
    // phase timing (hec_dist_set_timing): events at the call's start and at the
    // end of the interior rows (caller's stream) and of exchange + boundary rows
    // (communication stream)
    bool timing = false;
    cudaEvent_t tm_start = nullptr, tm_interior = nullptr, tm_comm = nullptr;
    bool tm_valid = false, tm_comm_valid = false;
};

namespace hec {

static hec_status nccl_fail(ncclResult_t r, const char* what) {
    return fail(HEC_ERR_NCCL, std::string("NCCL error in ") + what + ": " + ncclGetErrorString(r));
}

#define HEC_NCCL_TRY(expr)                                          \
    do {                                                            \
        ncclResult_t _r = (expr);                                   \
        if (_r != ncclSuccess) return ::hec::nccl_fail(_r, #expr);  \
    } while (0)

static void dist_release(hec_dist_s* d) {
    if (!d) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(d->device);
    if (d->ws && d->ws_free) d->ws_free(d->ws);
    if (d->comm) ncclCommDestroy(d->comm);
    for (void* p : d->opened) cudaIpcCloseMemHandle(p);
    if (d->d_win) cudaFree(d->d_win);
    if (d->d_push_chunks) cudaFree(d->d_push_chunks);
    if (d->d_nbr) cudaFree(d->d_nbr);
    if (d->d_peer_tab) cudaFree(d->d_peer_tab);
    if (d->d_done) cudaFree(d->d_done);
    if (d->d_err) cudaFree(d->d_err);
    if (d->ev_start) cudaEventDestroy(d->ev_start);
    for (cudaEvent_t e : {d->tm_start, d->tm_interior, d->tm_comm})
        if (e) cudaEventDestroy(e);
    if (d->ev_halo) cudaEventDestroy(d->ev_halo);
    if (d->comm_stream) cudaStreamDestroy(d->comm_stream);
    if (d->d_send_idx) cudaFree(d->d_send_idx);
    if (d->d_sendbuf) cudaFree(d->d_sendbuf);
    if (d->d_x_halo) cudaFree(d->d_x_halo);
    if (d->d_stage_x) cudaFree(d->d_stage_x);
    if (d->d_stage_y) cudaFree(d->d_stage_y);
    hec_free(d->interior);
    hec_free(d->boundary);
    cudaSetDevice(cur);
    delete d;
}

// A sub-HEC (interior or boundary rows) whose output rows are either one
// contiguous range (row_off) or an explicit row map.
static hec_status make_sub(const hec_plan_s& P, const CsrView& A, int32_t part, int32_t which,
                           const hec_opts& op, int32_t width, int32_t device, cudaStream_t s,
                           hec_matrix* out) {
    const PartPlan& pt = P.parts[part];
    const std::vector<int32_t>& rows = which == HEC_SUB_INTERIOR ? pt.interior : pt.boundary;
    CsrOwned L;
    HostHec h;
    hec_status st = build_local_csr(P, A, part, which, &L);
    if (st != HEC_OK) return st;
    if ((st = convert(L.view(), width, op.stride_unit, &h)) != HEC_OK) return st;
    bool contiguous = true;
    for (size_t k = 1; k < rows.size() && contiguous; ++k) contiguous = rows[k] == rows[0] + (int32_t)k;
    const int32_t n_loc = pt.r1 - pt.r0;
    if (contiguous)
        return make_matrix(std::move(h), device, s, nullptr, 0, rows.empty() ? 0 : rows[0], n_loc, out);
    return make_matrix(std::move(h), device, s, rows.data(), (int32_t)rows.size(), 0, n_loc, out);
}

static hec_status dist_build(const hec_csr* A, hec_plan P, const hec_opts* o, int32_t rank,
                             int32_t device, bool local, hec_dist_s** out) {
    CsrView v;
    hec_status st = validate_csr(A, &v);
    if (st != HEC_OK) return st;
    if (v.n_rows != P->n_rows || v.nnz != P->nnz) return fail(HEC_ERR_STATE, "matrix does not match the plan");
    if (rank < 0 || rank >= P->n_parts) return fail(HEC_ERR_PARTS, "rank out of range");
    const hec_opts op = normalise_opts(o);
    if ((st = check_opts(op)) != HEC_OK) return st;
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0)
        return fail(HEC_ERR_NODEV, "no CUDA device available");
    if (device < 0 || device >= n_dev) return fail(HEC_ERR_ARG, "device ordinal out of range");
    int prev = 0;
    cudaGetDevice(&prev);
    HEC_CUDA_TRY(cudaSetDevice(device));
    std::unique_ptr<hec_dist_s, void (*)(hec_dist_s*)> d(new hec_dist_s(), dist_release);
    const PartPlan& pt = P->parts[rank];
    d->rank = rank;
    d->n_parts = P->n_parts;
    d->device = device;
    d->r0 = pt.r0;
    d->r1 = pt.r1;
    d->n_halo = (int32_t)pt.recv.size();
    d->n_send = (int32_t)pt.send_idx.size();
    d->n_interior = (int32_t)pt.interior.size();
    d->n_boundary = (int32_t)pt.boundary.size();
    d->nnz_local = (int64_t)P->row_ptr[pt.r1] - P->row_ptr[pt.r0];
    d->send_off = pt.send_off;
    d->recv_off = pt.recv_off;
    d->local = local;
    // peer-memory transport metadata: where each send entry lands in its
    // destination's halo (q's receive segment from this rank starts at
    // q.recv_off[rank], reading A10), and the neighbour set
    d->all_nhalo.resize(P->n_parts);
    for (int32_t q = 0; q < P->n_parts; ++q) d->all_nhalo[q] = (int64_t)P->parts[q].recv.size();
    for (int32_t q = 0; q < P->n_parts; ++q) {
        const int32_t sc = pt.send_off[q + 1] - pt.send_off[q];
        const int32_t rc = pt.recv_off[q + 1] - pt.recv_off[q];
        if (q != rank && (sc > 0 || rc > 0)) d->nbr.push_back(q);
        // one push CTA per kPushChunk entries of one destination: the
        // destination's buffer pointer is loaded once per CTA and the stores
        // of a CTA are contiguous there
        for (int32_t k = pt.send_off[q]; k < pt.send_off[q + 1]; k += kPushChunk)
            d->push_chunks.push_back(make_int4(q, k, std::min(pt.send_off[q + 1], k + kPushChunk),
                                               P->parts[q].recv_off[rank] + (k - pt.send_off[q])));
    }
    d->width = part_width(*P, rank, op);
    cudaStream_t s = nullptr;
    HEC_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    try {
        st = make_sub(*P, v, rank, HEC_SUB_INTERIOR, op, d->width, device, s, &d->interior);
        if (st == HEC_OK) st = make_sub(*P, v, rank, HEC_SUB_BOUNDARY, op, d->width, device, s, &d->boundary);
    } catch (...) {
        st = fail(HEC_ERR_NOMEM, "host allocation failed in hec_dist_create");
    }
    if (st != HEC_OK) { cudaStreamDestroy(s); cudaSetDevice(prev); return st; }
    int64_t bytes = d->interior->device_bytes + d->boundary->device_bytes;
    cudaError_t e = cudaSuccess;
    if (d->n_send > 0) {
        e = cudaMalloc(&d->d_send_idx, sizeof(int32_t) * d->n_send);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d->d_send_idx, pt.send_idx.data(), sizeof(int32_t) * d->n_send, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaMalloc(&d->d_sendbuf, sizeof(double) * d->n_send);
        bytes += (int64_t)d->n_send * 12;
    }
    if (e == cudaSuccess && d->n_halo > 0) {
        e = cudaMalloc(&d->d_x_halo, sizeof(double) * d->n_halo);
        bytes += (int64_t)d->n_halo * 8;
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (e != cudaSuccess) { cudaSetDevice(prev); return cuda_fail(e, "dist buffers"); }
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);  // hi = greatest priority
    e = cudaStreamCreateWithPriority(&d->comm_stream, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_start, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_halo, cudaEventDisableTiming);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "dist streams/events");
    d->device_bytes = bytes;
    *out = d.release();
    return HEC_OK;
}

static bool has_exchange(const hec_dist_s* d) { return d->n_halo > 0 || d->n_send > 0; }

static size_t flag_bytes(int32_t n_parts) { return ((size_t)n_parts * 8 + 255) / 256 * 256; }

// This rank's receive window: arrival flags (zeroed) and two halo buffers.
static hec_status p2p_alloc_window(hec_dist_s* d) {
    if (d->d_win) return HEC_OK;
    const size_t fb = flag_bytes(d->n_parts), bytes = fb + 2 * sizeof(double) * (size_t)d->n_halo;
    HEC_CUDA_TRY(cudaMalloc(&d->d_win, bytes));  // cudaMalloc: exportable through CUDA IPC
    HEC_CUDA_TRY(cudaMemset(d->d_win, 0, bytes));
    HEC_CUDA_TRY(cudaMalloc(&d->d_done, sizeof(unsigned int)));
    HEC_CUDA_TRY(cudaMemset(d->d_done, 0, sizeof(unsigned int)));
    HEC_CUDA_TRY(cudaMalloc(&d->d_err, sizeof(int32_t)));
    HEC_CUDA_TRY(cudaMemset(d->d_err, 0, sizeof(int32_t)));
    HEC_CUDA_TRY(cudaDeviceSynchronize());
    d->device_bytes += (int64_t)bytes;
    return HEC_OK;
}

static uint64_t* win_flags(void* win) { return static_cast<uint64_t*>(win); }
static double* win_buf0(void* win, int32_t n_parts) {
    return reinterpret_cast<double*>(static_cast<char*>(win) + flag_bytes(n_parts));
}

// Upload the sender tables once every neighbour's window is mapped (wins[q]).
static hec_status p2p_finish(hec_dist_s* d, const std::vector<void*>& wins) {
    const int32_t P = d->n_parts;
    std::vector<uint64_t> tab(3 * (size_t)P, 0);  // buf0 ptrs, flag ptrs, n_halo
    for (int32_t q : d->nbr) {
        if (!wins[q]) return fail(HEC_ERR_STATE, "missing peer window");
        tab[q] = reinterpret_cast<uint64_t>(win_buf0(wins[q], P));
        tab[P + q] = reinterpret_cast<uint64_t>(win_flags(wins[q]));
    }
    for (int32_t q = 0; q < P; ++q) tab[2 * P + q] = (uint64_t)d->all_nhalo[q];
    HEC_CUDA_TRY(cudaMalloc(&d->d_peer_tab, tab.size() * 8));
    HEC_CUDA_TRY(cudaMemcpy(d->d_peer_tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));
    if (!d->nbr.empty()) {
        HEC_CUDA_TRY(cudaMalloc(&d->d_nbr, d->nbr.size() * sizeof(int32_t)));
        HEC_CUDA_TRY(cudaMemcpy(d->d_nbr, d->nbr.data(), d->nbr.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    if (!d->push_chunks.empty()) {
        const size_t nb = d->push_chunks.size() * sizeof(int4);
        HEC_CUDA_TRY(cudaMalloc(&d->d_push_chunks, nb));
        HEC_CUDA_TRY(cudaMemcpy(d->d_push_chunks, d->push_chunks.data(), nb, cudaMemcpyHostToDevice));
    }
    d->p2p = true;
    return HEC_OK;
}

static PushArgs push_args(const hec_dist_s* d, const double* x_local, uint64_t ep) {
    const int32_t P = d->n_parts;
    PushArgs a;
    a.x = x_local;
    a.idx = d->d_send_idx;
    a.chunks = d->d_push_chunks;
    a.n_chunks = (int32_t)d->push_chunks.size();
    a.peer_buf0 = static_cast<double* const*>(d->d_peer_tab);
    a.peer_flags = reinterpret_cast<uint64_t* const*>(static_cast<uint64_t*>(d->d_peer_tab) + P);
    a.peer_nhalo = reinterpret_cast<const int64_t*>(static_cast<uint64_t*>(d->d_peer_tab) + 2 * P);
    a.nbr = d->d_nbr;
    a.n_nbr = (int32_t)d->nbr.size();
    a.rank = d->rank;
    a.epoch = ep;
    a.done = d->d_done;
    return a;
}

static PeerWait wait_args(const hec_dist_s* d, uint64_t ep) {
    PeerWait w;
    w.flags = win_flags(d->d_win);
    w.peers = d->d_nbr;
    w.n = (int32_t)d->nbr.size();
    w.epoch = ep;
    w.err = d->d_err;
    return w;
}

// The peer-memory wait's error word (set when a neighbour's flag did not
// arrive within ~10 s); the caller has synchronised the stream that ran it.
hec_status dist_err(hec_dist_s* D) {
    if (!D->d_err) return HEC_OK;
    HEC_CUDA_TRY(cudaStreamSynchronize(D->comm_stream));
    int32_t err = 0;
    HEC_CUDA_TRY(cudaMemcpy(&err, D->d_err, sizeof(err), cudaMemcpyDeviceToHost));
    if (err) return fail(HEC_ERR_STATE, "peer-memory halo: a neighbour's data did not arrive within 10 s");
    return HEC_OK;
}

static double* p2p_halo(const hec_dist_s* d, uint64_t ep) {
    return d->n_halo ? win_buf0(d->d_win, d->n_parts) + (ep & 1) * (uint64_t)d->n_halo : nullptr;
}

}  // namespace hec

using namespace hec;

extern "C" {

hec_status hec_nccl_unique_id(uint8_t id[HEC_NCCL_ID_BYTES]) {
    if (!id) return fail(HEC_ERR_ARG, "NULL id");
    static_assert(sizeof(ncclUniqueId) == HEC_NCCL_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    HEC_NCCL_TRY(ncclGetUniqueId(&u));
    std::memcpy(id, &u, HEC_NCCL_ID_BYTES);
    return HEC_OK;
}

hec_status hec_dist_create(const hec_csr* A, hec_plan P, const hec_opts* o, int32_t rank,
                           const uint8_t id[HEC_NCCL_ID_BYTES], int32_t device, hec_dist* out) {
    if (!out || !P) return fail(HEC_ERR_ARG, "NULL argument");
    *out = nullptr;
    hec_dist_s* d = nullptr;
    hec_status st = dist_build(A, P, o, rank, device, false, &d);
    if (st != HEC_OK) return st;
    if (P->n_parts > 1) {
        if (!id) { dist_release(d); return fail(HEC_ERR_ARG, "NULL NCCL id"); }
        ncclUniqueId u;
        std::memcpy(&u, id, HEC_NCCL_ID_BYTES);
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        ncclResult_t r = ncclCommInitRank(&d->comm, P->n_parts, u, rank);
        cudaSetDevice(prev);
        if (r != ncclSuccess) { dist_release(d); return nccl_fail(r, "ncclCommInitRank"); }
    }
    *out = d;
    return HEC_OK;
}

hec_status hec_dist_create_p2p(const hec_csr* A, hec_plan P, const hec_opts* o, int32_t rank, int32_t device,
                               hec_dist* out, uint8_t handle_out[HEC_IPC_BYTES]) {
    if (!out || !P || !handle_out) return fail(HEC_ERR_ARG, "NULL argument");
    *out = nullptr;
    static_assert(sizeof(cudaIpcMemHandle_t) == HEC_IPC_BYTES, "cudaIpcMemHandle_t size");
    hec_dist_s* d = nullptr;
    hec_status st = dist_build(A, P, o, rank, device, false, &d);
    if (st != HEC_OK) return st;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    st = p2p_alloc_window(d);
    cudaIpcMemHandle_t h;
    if (st == HEC_OK) {
        cudaError_t e = cudaIpcGetMemHandle(&h, d->d_win);
        if (e != cudaSuccess) st = cuda_fail(e, "cudaIpcGetMemHandle");
    }
    cudaSetDevice(prev);
    if (st != HEC_OK) { dist_release(d); return st; }
    std::memcpy(handle_out, &h, HEC_IPC_BYTES);
    *out = d;
    return HEC_OK;
}

// Map every neighbour's window from its IPC handle (handles: n_parts x
// HEC_IPC_BYTES in rank order; this rank's own entry is ignored).
static hec_status p2p_connect_ipc(hec_dist_s* d, const uint8_t* handles) {
    std::vector<void*> wins(d->n_parts, nullptr);
    for (int32_t q : d->nbr) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + (size_t)q * HEC_IPC_BYTES, HEC_IPC_BYTES);
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle (peer window)");
        d->opened.push_back(p);
        wins[q] = p;
    }
    return p2p_finish(d, wins);
}

hec_status hec_dist_p2p_connect(hec_dist D, const uint8_t* handles) {
    if (!D || !handles) return fail(HEC_ERR_ARG, "NULL argument");
    if (D->p2p || D->local) return fail(HEC_ERR_STATE, "handle already connected or local");
    if (!D->d_win) return fail(HEC_ERR_STATE, "no window: create the handle with hec_dist_create_p2p");
    DeviceGuard g(D->device);
    return p2p_connect_ipc(D, handles);
}

hec_status hec_dist_enable_p2p(hec_dist D) {
    if (!D) return fail(HEC_ERR_ARG, "NULL handle");
    if (D->p2p || D->local) return fail(HEC_ERR_STATE, "handle already connected or local");
    if (D->n_parts == 1) return HEC_OK;
    if (!D->comm) return fail(HEC_ERR_STATE, "no NCCL communicator to exchange the window handles");
    DeviceGuard g(D->device);
    hec_status st = p2p_alloc_window(D);
    if (st != HEC_OK) return st;
    cudaIpcMemHandle_t h;
    HEC_CUDA_TRY(cudaIpcGetMemHandle(&h, D->d_win));
    uint8_t* dbuf = nullptr;
    const size_t nb = (size_t)D->n_parts * HEC_IPC_BYTES;
    HEC_CUDA_TRY(cudaMalloc(&dbuf, nb + HEC_IPC_BYTES));
    std::vector<uint8_t> all(nb);
    cudaError_t e = cudaMemcpy(dbuf + nb, &h, HEC_IPC_BYTES, cudaMemcpyHostToDevice);
    ncclResult_t r = ncclSuccess;
    if (e == cudaSuccess) r = ncclAllGather(dbuf + nb, dbuf, HEC_IPC_BYTES, ncclUint8, D->comm, D->comm_stream);
    if (e == cudaSuccess && r == ncclSuccess) e = cudaStreamSynchronize(D->comm_stream);
    if (e == cudaSuccess && r == ncclSuccess) e = cudaMemcpy(all.data(), dbuf, nb, cudaMemcpyDeviceToHost);
    cudaFree(dbuf);
    if (r != ncclSuccess) return nccl_fail(r, "window handle all-gather");
    if (e != cudaSuccess) return cuda_fail(e, "window handle all-gather");
    return p2p_connect_ipc(D, all.data());
}

hec_status hec_dist_p2p_connect_local(hec_dist* D, int32_t n) {
    if (!D || n < 1) return fail(HEC_ERR_ARG, "NULL argument");
    for (int32_t p = 0; p < n; ++p)
        if (!D[p] || !D[p]->local || D[p]->rank != p || D[p]->n_parts != n || D[p]->p2p)
            return fail(HEC_ERR_STATE, "handles must be the n unconnected ranks from hec_dist_create_local");
    DeviceGuard g(D[0]->device);
    std::vector<void*> wins(n);
    for (int32_t p = 0; p < n; ++p) {
        hec_status st = p2p_alloc_window(D[p]);
        if (st != HEC_OK) return st;
        wins[p] = D[p]->d_win;
    }
    for (int32_t p = 0; p < n; ++p) {
        hec_status st = p2p_finish(D[p], wins);
        if (st != HEC_OK) return st;
    }
    return HEC_OK;
}

hec_status hec_dist_check(hec_dist D) {
    if (!D) return fail(HEC_ERR_ARG, "NULL handle");
    DeviceGuard g(D->device);
    HEC_CUDA_TRY(cudaStreamSynchronize(D->comm_stream));
    return dist_err(D);
}

hec_status hec_dist_create_local(const hec_csr* A, hec_plan P, const hec_opts* o, int32_t device,
                                 hec_dist* out) {
    if (!out || !P) return fail(HEC_ERR_ARG, "NULL argument");
    for (int32_t p = 0; p < P->n_parts; ++p) out[p] = nullptr;
    for (int32_t p = 0; p < P->n_parts; ++p) {
        hec_dist_s* d = nullptr;
        hec_status st = dist_build(A, P, o, p, device, true, &d);
        if (st != HEC_OK) {
            for (int32_t q = 0; q < p; ++q) { dist_release(out[q]); out[q] = nullptr; }
            return st;
        }
        out[p] = d;
    }
    return HEC_OK;
}

}  // extern "C"

namespace hec {

// The distributed product on `s` (device already current).  The caller's
// stream waits for the exchange before the boundary rows AND before returning
// control of `s`, so every later NCCL call issued on `s` (e.g. the Krylov
// all-reduces) is ordered after this exchange on every rank.
// Host-side NVTX range for the scope (one phase of hec_spmv_dist's enqueue);
// an nsys timeline lines the ranges up with the kernels they launch.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

hec_status dist_spmv_launch(hec_dist_s* D, const double* x_local, double* y_local, cudaStream_t s) {
    NvtxRange all("hec_spmv_dist");
    if (D->p2p && !D->nbr.empty()) {
        // peer-memory transport: fused pack + NVLink stores + flag release on
        // the comm stream, then wait for the neighbours' flags and run the
        // boundary rows behind it; the interior overlaps on the caller's stream
        const uint64_t ep = ++D->epoch;
        if (D->timing) HEC_CUDA_TRY(cudaEventRecord(D->tm_start, s));
        HEC_CUDA_TRY(cudaEventRecord(D->ev_start, s));
        HEC_CUDA_TRY(cudaStreamWaitEvent(D->comm_stream, D->ev_start, 0));
        {
            NvtxRange r("hec.push (pack + NVLink stores + release)");
            HEC_CUDA_TRY(launch_push(push_args(D, x_local, ep), D->comm_stream));
        }
        const PeerWait w = wait_args(D, ep);
        {
            NvtxRange r("hec.wait + boundary");
            if (D->n_boundary > 0) {
                hec_status st = launch_spmv_peer(D->boundary, x_local, p2p_halo(D, ep), y_local, D->comm_stream, w);
                if (st != HEC_OK) return st;
            } else {
                HEC_CUDA_TRY(launch_peer_wait(w, D->comm_stream));
            }
        }
        HEC_CUDA_TRY(cudaEventRecord(D->ev_halo, D->comm_stream));
        if (D->timing) HEC_CUDA_TRY(cudaEventRecord(D->tm_comm, D->comm_stream));
        NvtxRange r("hec.interior");
        hec_status st = launch_spmv(D->interior, x_local, nullptr, y_local, s);
        if (st != HEC_OK) return st;
        if (D->timing) HEC_CUDA_TRY(cudaEventRecord(D->tm_interior, s));
        D->tm_valid = D->timing;
        D->tm_comm_valid = D->timing;
        HEC_CUDA_TRY(cudaStreamWaitEvent(s, D->ev_halo, 0));
        return HEC_OK;
    }
    if (has_exchange(D) && !D->comm && !D->local)
        return fail(HEC_ERR_STATE, "no halo transport: connect the peer-memory windows (hec_dist_p2p_connect)");
    const bool ex = has_exchange(D) && D->comm;
    if (D->timing) HEC_CUDA_TRY(cudaEventRecord(D->tm_start, s));
    if (ex) {
        // comm stream: pack + grouped send/recv, overlapped with the interior SpMV
        HEC_CUDA_TRY(cudaEventRecord(D->ev_start, s));
        HEC_CUDA_TRY(cudaStreamWaitEvent(D->comm_stream, D->ev_start, 0));
        NvtxRange rx("hec.pack + ncclSend/ncclRecv + boundary");
        HEC_CUDA_TRY(launch_pack(D->d_send_idx, D->n_send, x_local, D->d_sendbuf, D->comm_stream));
        ncclResult_t r = ncclGroupStart();
        for (int32_t q = 0; q < D->n_parts && r == ncclSuccess; ++q) {
            const int32_t sc = D->send_off[q + 1] - D->send_off[q];
            const int32_t rc = D->recv_off[q + 1] - D->recv_off[q];
            if (sc > 0) r = ncclSend(D->d_sendbuf + D->send_off[q], sc, ncclDouble, q, D->comm, D->comm_stream);
            if (r == ncclSuccess && rc > 0)
                r = ncclRecv(D->d_x_halo + D->recv_off[q], rc, ncclDouble, q, D->comm, D->comm_stream);
        }
        ncclResult_t r2 = ncclGroupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess) return nccl_fail(r != ncclSuccess ? r : r2, "halo send/recv");
        // boundary rows right behind the halo on the (high-priority) comm
        // stream: they write rows of y disjoint from the interior's, so they
        // need not wait for the interior kernel -- critical path
        // max(interior, pack + exchange + boundary)
        if (D->n_boundary > 0) {
            hec_status st = launch_spmv(D->boundary, x_local, D->d_x_halo, y_local, D->comm_stream);
            if (st != HEC_OK) return st;
        }
        HEC_CUDA_TRY(cudaEventRecord(D->ev_halo, D->comm_stream));
        if (D->timing) HEC_CUDA_TRY(cudaEventRecord(D->tm_comm, D->comm_stream));
    }
    NvtxRange ri("hec.interior");
    hec_status st = launch_spmv(D->interior, x_local, nullptr, y_local, s);  // interior rows
    if (st != HEC_OK) return st;
    if (D->timing) HEC_CUDA_TRY(cudaEventRecord(D->tm_interior, s));
    D->tm_valid = D->timing;
    D->tm_comm_valid = D->timing && ex;
    if (ex) HEC_CUDA_TRY(cudaStreamWaitEvent(s, D->ev_halo, 0));
    else if (D->n_boundary > 0) st = launch_spmv(D->boundary, x_local, D->d_x_halo, y_local, s);
    return st;
}

// Local emulation of one distributed product over all n ranks on one device
// and one stream (device current, handles validated by the caller).
hec_status dist_local_spmv_launch(hec_dist_s** D, int32_t n, const double* const* x_locals,
                                  double* const* y_locals, cudaStream_t s) {
    if (D[0]->p2p) {
        // peer-memory transport emulated on one device and one stream: every
        // rank's push kernel (stores into the other ranks' windows + flag
        // release), then every rank's interior rows and flag wait + boundary
        // rows (the flags are already set, so no wait ever spins)
        for (int32_t p = 0; p < n; ++p) {
            const uint64_t ep = ++D[p]->epoch;
            cudaError_t e = D[p]->nbr.empty() ? cudaSuccess : launch_push(push_args(D[p], x_locals[p], ep), s);
            if (e != cudaSuccess) return cuda_fail(e, "push kernel");
        }
        for (int32_t p = 0; p < n; ++p) {
            const uint64_t ep = D[p]->epoch;
            hec_status st = launch_spmv(D[p]->interior, x_locals[p], nullptr, y_locals[p], s);
            if (st == HEC_OK && D[p]->n_boundary > 0) {
                st = D[p]->nbr.empty()
                         ? launch_spmv(D[p]->boundary, x_locals[p], p2p_halo(D[p], ep), y_locals[p], s)
                         : launch_spmv_peer(D[p]->boundary, x_locals[p], p2p_halo(D[p], ep), y_locals[p], s,
                                            wait_args(D[p], ep));
            }
            if (st != HEC_OK) return st;
        }
        return HEC_OK;
    }
    for (int32_t p = 0; p < n; ++p) {
        cudaError_t e = launch_pack(D[p]->d_send_idx, D[p]->n_send, x_locals[p], D[p]->d_sendbuf, s);
        if (e != cudaSuccess) return cuda_fail(e, "halo pack");
    }
    for (int32_t p = 0; p < n; ++p)          // the "exchange": sender p -> receiver q
        for (int32_t q = 0; q < n; ++q) {
            const int32_t sc = D[p]->send_off[q + 1] - D[p]->send_off[q];
            if (sc <= 0) continue;
            const int32_t rc = D[q]->recv_off[p + 1] - D[q]->recv_off[p];
            if (rc != sc) return fail(HEC_ERR_STATE, "send/recv count mismatch");
            cudaError_t e = cudaMemcpyAsync(D[q]->d_x_halo + D[q]->recv_off[p], D[p]->d_sendbuf + D[p]->send_off[q],
                                            sizeof(double) * sc, cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return cuda_fail(e, "local exchange");
        }
    for (int32_t p = 0; p < n; ++p) {
        hec_status st = launch_spmv(D[p]->interior, x_locals[p], nullptr, y_locals[p], s);
        if (st == HEC_OK && D[p]->n_boundary > 0)
            st = launch_spmv(D[p]->boundary, x_locals[p], D[p]->d_x_halo, y_locals[p], s);
        if (st != HEC_OK) return st;
    }
    return HEC_OK;
}

int64_t dist_n_local(hec_dist_s* D) { return (int64_t)D->r1 - D->r0; }

bool dist_is_local(hec_dist_s* D) { return D->local; }

int32_t dist_rank(hec_dist_s* D) { return D->rank; }

ncclComm_t dist_comm(hec_dist_s* D) { return D->comm; }

int32_t dist_parts(hec_dist_s* D) { return D->n_parts; }

int32_t dist_device(hec_dist_s* D) { return D->device; }


void** dist_ws_slot(hec_dist_s* D, void (***free_fn)(void*)) {
    *free_fn = &D->ws_free;
    return &D->ws;
}

}  // namespace hec

extern "C" {

hec_status hec_spmv_dist(hec_dist D, const double* x_local, double* y_local, void* stream) {
    if (!D) return fail(HEC_ERR_ARG, "NULL handle");
    if (D->local) return fail(HEC_ERR_STATE, "local-emulation handle: use hec_spmv_dist_local");
    const int32_t n_loc = D->r1 - D->r0;
    if (n_loc > 0 && (!x_local || !y_local)) return fail(HEC_ERR_ARG, "NULL x_local/y_local");
    if (x_local && y_local && x_local < y_local + n_loc && y_local < x_local + n_loc)
        return fail(HEC_ERR_ARG, "x_local and y_local overlap");
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != D->device) cudaSetDevice(D->device);
    hec_status st = dist_spmv_launch(D, x_local, y_local, (cudaStream_t)stream);
    if (prev != D->device) cudaSetDevice(prev);
    return st;
}

hec_status hec_spmv_dist_host(hec_dist D, const double* x_host_local, double* y_host_local, void* stream) {
    if (!D) return fail(HEC_ERR_ARG, "NULL handle");
    if (D->local) return fail(HEC_ERR_STATE, "local-emulation handle: use hec_spmv_dist_local");
    const int32_t n_loc = D->r1 - D->r0;
    if (n_loc > 0 && (!x_host_local || !y_host_local)) return fail(HEC_ERR_ARG, "NULL host vector");
    DeviceGuard g(D->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t nb = sizeof(double) * (size_t)(n_loc > 0 ? n_loc : 1);
    if (!D->d_stage_x) {
        HEC_CUDA_TRY(cudaMalloc(&D->d_stage_x, nb));
        HEC_CUDA_TRY(cudaMalloc(&D->d_stage_y, nb));
        D->device_bytes += 2 * (int64_t)nb;
    }
    if (n_loc > 0)
        HEC_CUDA_TRY(cudaMemcpyAsync(D->d_stage_x, x_host_local, sizeof(double) * n_loc, cudaMemcpyHostToDevice, s));
    hec_status st = dist_spmv_launch(D, D->d_stage_x, D->d_stage_y, s);
    if (st != HEC_OK) return st;
    if (n_loc > 0)
        HEC_CUDA_TRY(cudaMemcpyAsync(y_host_local, D->d_stage_y, sizeof(double) * n_loc, cudaMemcpyDeviceToHost, s));
    HEC_CUDA_TRY(cudaStreamSynchronize(s));
    return HEC_OK;
}

hec_status hec_dist_set_timing(hec_dist D, int32_t enable) {
    if (!D) return fail(HEC_ERR_ARG, "NULL handle");
    DeviceGuard g(D->device);
    if (enable && !D->tm_start) {
        HEC_CUDA_TRY(cudaEventCreate(&D->tm_start));
        HEC_CUDA_TRY(cudaEventCreate(&D->tm_interior));
        HEC_CUDA_TRY(cudaEventCreate(&D->tm_comm));
    }
    D->timing = enable != 0;
    D->tm_valid = D->tm_comm_valid = false;
    return HEC_OK;
}

hec_status hec_dist_phase_times(hec_dist D, float* interior_ms, float* comm_ms) {
    if (!D || !interior_ms || !comm_ms) return fail(HEC_ERR_ARG, "NULL argument");
    if (!D->tm_valid) return fail(HEC_ERR_STATE, "no timed hec_spmv_dist call (hec_dist_set_timing first)");
    DeviceGuard g(D->device);
    HEC_CUDA_TRY(cudaEventSynchronize(D->tm_interior));
    HEC_CUDA_TRY(cudaEventElapsedTime(interior_ms, D->tm_start, D->tm_interior));
    *comm_ms = -1.0f;
    if (D->tm_comm_valid) {
        HEC_CUDA_TRY(cudaEventSynchronize(D->tm_comm));
        HEC_CUDA_TRY(cudaEventElapsedTime(comm_ms, D->tm_start, D->tm_comm));
    }
    return HEC_OK;
}

hec_status hec_dist_comm_size(hec_dist D, int32_t* nranks, int32_t* version) {
    if (!D || !nranks || !version) return fail(HEC_ERR_ARG, "NULL argument");
    int v = 0, c = 0;
    ncclGetVersion(&v);
    if (D->comm) {
        ncclResult_t r = ncclCommCount(D->comm, &c);
        if (r != ncclSuccess) return nccl_fail(r, "ncclCommCount");
    }
    *nranks = c;
    *version = v;
    return HEC_OK;
}

hec_status hec_spmv_dist_local(hec_dist* D, int32_t n, const double* const* x_locals,
                               double* const* y_locals, void* stream) {
    if (!D || n < 1 || !x_locals || !y_locals) return fail(HEC_ERR_ARG, "NULL argument");
    for (int32_t p = 0; p < n; ++p)
        if (!D[p] || !D[p]->local || D[p]->rank != p || D[p]->n_parts != n)
            return fail(HEC_ERR_STATE, "handles must be the n ranks from hec_dist_create_local");
    DeviceGuard g(D[0]->device);
    return dist_local_spmv_launch(D, n, x_locals, y_locals, (cudaStream_t)stream);
}

hec_status hec_dist_get_info(hec_dist D, hec_dist_info* o) {
    if (!D || !o) return fail(HEC_ERR_ARG, "NULL argument");
    o->rank = D->rank;
    o->n_parts = D->n_parts;
    o->r0 = D->r0;
    o->r1 = D->r1;
    o->n_halo = D->n_halo;
    o->n_send = D->n_send;
    o->n_interior = D->n_interior;
    o->n_boundary = D->n_boundary;
    o->width = D->width;
    o->launches = hec_spmv_launches(D->interior) + hec_spmv_launches(D->boundary) +
                  (D->p2p ? (D->nbr.empty() ? 0 : 2) : (has_exchange(D) && D->n_send > 0 ? 1 : 0));
    o->device_bytes = D->device_bytes;
    const int64_t n_loc = D->r1 - D->r0;
    o->algorithmic_bytes = 12 * D->nnz_local + 8 * (n_loc + D->n_halo) + 8 * n_loc;
    o->nnz_local = D->nnz_local;
    return HEC_OK;
}

void hec_dist_free(hec_dist D) { dist_release(D); }

}  // extern "C"
