// hec_internal.h -- internal declarations shared by the libhec.so sources.
// Not part of the ABI (that is include/hec.h).
#pragma once

#include <cstdint>
#include <string>
#include <vector>
#include <cstdlib>
#include <algorithm>

#include <cuda_runtime.h>

#include "hec.h"

namespace hec {

// ----------------------------------------------------------------- errors --
void set_error(const std::string& msg);
hec_status fail(hec_status st, const std::string& msg);
hec_status cuda_fail(cudaError_t e, const char* what);

#define HEC_CUDA_TRY(expr)                                              \
    do {                                                                \
        cudaError_t _e = (expr);                                        \
        if (_e != cudaSuccess) return ::hec::cuda_fail(_e, #expr);      \
    } while (0)

// --------------------------------------------------------------- host HEC --
// A CSR view with int64 offsets (the public struct uses int32 row_ptr).
struct CsrView {
    int32_t n_rows = 0, n_cols = 0;
    int64_t nnz = 0;
    const int32_t* row_ptr = nullptr;
    const int32_t* col = nullptr;
    const double* val = nullptr;
};

// Host-side local CSR (owned storage) used for partition sub-matrices.
struct CsrOwned {
    int32_t n_rows = 0, n_cols = 0;
    std::vector<int32_t> row_ptr, col;
    std::vector<double> val;
    CsrView view() const {
        CsrView v;
        v.n_rows = n_rows; v.n_cols = n_cols; v.nnz = (int64_t)col.size();
        v.row_ptr = row_ptr.data(); v.col = col.data(); v.val = val.data();
        return v;
    }
};

struct HostHec {
    int32_t n_rows = 0, n_cols = 0, width = 0, stride = 0;
    int64_t nnz = 0, ell_nnz = 0;
    std::vector<int32_t> ell_col;   // [width*stride], column-major, -1 = padding
    std::vector<double> ell_val;    // [width*stride], +0.0 padding
    std::vector<int32_t> tail_rows, tail_ptr, tail_col;
    std::vector<double> tail_val;
};

hec_status validate_csr(const hec_csr* A, CsrView* out);
hec_opts normalise_opts(const hec_opts* o);
hec_status check_opts(const hec_opts& o);
// Width from a row-length histogram (reading A1).
int32_t choose_width(const CsrView& A, const hec_opts& o);
// CSR -> HEC fill with a given width (readings A2-A4, A15).
hec_status convert(const CsrView& A, int32_t width, int32_t stride_unit, HostHec* out);
// Device layout of the CSR tail ("warp chunks", plan_chunks in api.cpp): the
// tail rows are cut into super-blocks of consecutive tail rows; inside one
// they are sorted by (lanes per row G = 2^lg, spilled length) and every CUDA
// block descriptor takes 256/G rows of one G.  Lane l of warp w of a
// descriptor reads, in iteration i, the entry pair at base_w + 64 i + 2 l:
// every warp-wide load is one aligned 256-byte (index) and 512-byte (value)
// segment, whatever the row lengths.  Padding entries are (-1, +0.0)
// (reading A4).  A lane's pairs are its row's entries 2(iG + lr), +1 in
// order, lr = its lane within the row.
constexpr int kTailChunk = 64;         // entries per warp per iteration (32 lanes x a pair)
constexpr int kTailSuperRows = 2048;   // tail rows regrouped by length within blocks of this many (sweep: 256 340 us, 512 282, 1024 251, 2048 249, 4096 262, 16384 300 on the power-law tail)

// Lanes per tail row: the smallest power of two >= ceil(L / epl), capped at
// 2^kTailMaxLg, where epl = target entries per lane.  Up to 32 lanes a row
// lives in one warp (shuffle reduction); 64-256 lanes span 2-8 warps of one
// CTA (shuffle, then the warps' partials combined through shared memory).
// Warps per tail descriptor (one CUDA block of 32 kTailWarps threads takes
// one descriptor); rows span at most all of them: G <= 32 kTailWarps lanes.
#ifndef HEC_TAIL_WARPS
#define HEC_TAIL_WARPS 8
#endif
constexpr int kTailWarps = HEC_TAIL_WARPS;
constexpr int kTailThreads = 32 * kTailWarps;
static_assert(kTailWarps == 2 || kTailWarps == 4 || kTailWarps == 8, "tail descriptor warps: 2, 4 or 8");
constexpr int kTailMaxLg = kTailWarps == 8 ? 8 : kTailWarps == 4 ? 7 : 6;
// x ring (tail_ring_kernel): columns per CTA ring (a power of two; 128 KiB of
// fp64) and tail rows per super-block when the ring schedule is used
constexpr int kRingCols = 16384;
#ifndef HEC_RING_DEPTH
#define HEC_RING_DEPTH 3
#endif
constexpr int kRingDepth = HEC_RING_DEPTH;  // stages in flight per ring CTA (its windows share the ring)
constexpr int kRingSuperRows = 1024;
#ifndef HEC_TAIL_EPL_BIG
#define HEC_TAIL_EPL_BIG 48  // measured with the batched tail loop: 8 -> 316/335 us, 16 -> 274, 32 -> 262; final tree: 24 / 32 / 48 -> step 0.4264 / 0.4211 / 0.4184 ms
#endif
constexpr int kTailEplBig = HEC_TAIL_EPL_BIG;  // entries per lane for tails of >= 2^22 entries
inline int tail_max_lg() {             // HEC_TAIL_MAXLG (tuning): 5..8
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("HEC_TAIL_MAXLG");
        v = e ? std::max(5, std::min(kTailMaxLg, std::atoi(e))) : kTailMaxLg;
    }
    return v;
}
// Target entries per lane of the tail kernels for a tail of this many entries
// (plan_chunks and the fused small-tail map must agree; HEC_TAIL_EPL tunes).
inline int tail_epl(size_t tail_nnz) {
    int epl = tail_nnz >= ((size_t)1 << 22) ? kTailEplBig : 2;
    if (const char* e = std::getenv("HEC_TAIL_EPL")) epl = std::max(1, std::min(64, std::atoi(e)));
    return epl;
}
inline int tail_lg_for(int32_t L, int epl) {
    int lg = 0;
    const int cap = tail_max_lg();
    while (lg < cap && (epl << lg) < L) ++lg;
    return lg;
}

// ------------------------------------------------------------------ plans --
struct PartPlan {
    int32_t r0 = 0, r1 = 0;
    std::vector<int32_t> recv;       // global columns, ascending
    std::vector<int32_t> recv_off;   // [P+1]
    std::vector<int32_t> send_idx;   // local indices, concatenated over peers
    std::vector<int32_t> send_off;   // [P+1]
    std::vector<int32_t> interior, boundary;
};

}  // namespace hec

struct hec_plan_s {
    int32_t n_parts = 0;
    int32_t n_rows = 0;
    int64_t nnz = 0;
    std::vector<int32_t> part_ptr;
    std::vector<int32_t> row_ptr;    // copy of the global row_ptr (row lengths, A12)
    std::vector<hec::PartPlan> parts;
};

namespace hec {
// Local sub-matrix of a part (which = HEC_SUB_*), local column numbering.
hec_status build_local_csr(const hec_plan_s& P, const CsrView& A, int32_t part, int32_t which,
                           CsrOwned* out);
int32_t part_width(const hec_plan_s& P, int32_t part, const hec_opts& o);
hec_status build_plan(const CsrView& A, int32_t P, int32_t kind, const int32_t* grid,
                      hec_plan_s* plan);
}  // namespace hec

// ------------------------------------------------------------ device HEC --
struct hec_matrix_s {
    // Krylov workspace cached by the first solve on this handle (krylov.cu);
    // freed with the handle through ws_free
    void* ws = nullptr;
    void (*ws_free)(void*) = nullptr;
    int32_t device = -1;
    int32_t n_rows = 0, n_cols = 0, width = 0, stride = 0;
    int64_t nnz = 0, ell_nnz = 0, tail_nnz = 0;
    int32_t tail_rows = 0;
    bool tail_coo = false;             // HYB comparison variant: the remainder in COO
    int32_t* d_coo_row = nullptr;      // HYB: output row of every remainder entry
    std::vector<int32_t> h_tail_ptr;   // tail_ptr kept on the host for hec_export (both layouts)
    hec::HostHec host;                 // full copy only for host-only handles
    std::vector<int32_t> h_tail_rows;  // local tail row ids (always kept; small)
    // device arrays
    int32_t* d_ell_col = nullptr;
    double* d_ell_val = nullptr;
    int32_t* d_tail_out = nullptr;     // output row of each tail row (after row map)
    std::vector<int32_t> h_tail_order; // device tail row position p holds tail row h_tail_order[p]
    std::vector<int4> h_tail_blk;      // descriptors {first row position, count, lg, first warp}
    std::vector<int4> h_tail_warp;     // 8 per descriptor: {first entry, iterations, first row, count << 8 | lg}
    int4* d_tail_warp = nullptr;
    int64_t* d_tail_region = nullptr;  // SM-local tail schedule: [n_regions + 1] unit boundaries
    int4* d_tail_units = nullptr;      // SM-local tail schedule: each warp unit's first warp meta
    int32_t* d_tail_uwidx = nullptr;   // ... and its index in the warp-meta array
    unsigned int* d_tail_ctr = nullptr;  // [n_regions] claim counters + 1 done counter
    int32_t tail_regions = 0;
    bool tail_reverse = false;         // tail launch walks its descriptors last to first (api.cpp)
    // x-ring schedule (TailArgs::ring_*): one allocation holding
    // the stages, the per-CTA stage prefix and the units
    void* d_ring = nullptr;
    const int4 *d_ring_stage = nullptr, *d_ring_unit = nullptr;
    const int32_t* d_ring_cta = nullptr;
    int32_t ring_ctas = 0;
    double ring_cover = 0.0;
    // rows grouped by ELL length inside windows of kGroupRows (device position
    // p holds row h_ell_perm[p]; d_ell_perm[p] = that row's output row, the
    // ELL launch's row map)
    int32_t* d_ell_perm = nullptr;
    std::vector<int32_t> h_ell_perm;
    // second-phase slot skipping (EllArgs::tile_w): longest ELL row per 64-row tile
    uint8_t* d_tile_w = nullptr;
    double tile_skip = 0.0;            // fraction of the ELL slots the kernel does not read
    // ELL index compression (EllArgs::d16): int16 deltas beside d_ell_col
    int16_t* d_ell_d16 = nullptr;
    int32_t idx16_base[16] = {};
    double idx16_esc = -1.0;           // escaped fraction of the ELL slots (-1: not evaluated)           // fraction of the tail's stored entries inside their stage's window
    // concurrent tail (big tails, whole plain launches): the tail kernel on its
    // own stream beside the ELL kernel, sums into tsum, then one combine pass
    bool tail_conc = false;
    double* d_tsum = nullptr;
    cudaStream_t s_tail = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int64_t tail_entries = 0;          // device tail positions (stored entries + padding)
    int4* d_tail_blk = nullptr;        // per CUDA block: {first position, count, lg, 0}
    int32_t* d_tail_col = nullptr;
    double* d_tail_val = nullptr;
    int32_t* d_rowmap = nullptr;       // output row of each row, or null (then row_off + i)
    int32_t row_off = 0;
    int32_t n_loc = -1;                // >= 0: columns >= n_loc read x_halo[c - n_loc]
    double* d_stage_x = nullptr;       // hec_spmv_host staging
    double* d_stage_y = nullptr;
    // hec_spmv_host pipeline: row chunks whose ELL+tail run as soon as the x
    // prefix they read has arrived, and whose y goes back while later chunks
    // compute (H2D, compute and D2H overlap; PCIe is full duplex).
    int32_t n_chunks = 1;
    std::vector<int32_t> chunk_row;    // [n_chunks+1], multiples of 512
    std::vector<int32_t> chunk_xend;   // [n_chunks]: x[0 : xend) needed by rows < chunk_row[c+1]
    std::vector<int64_t> chunk_blk;    // [n_chunks+1]: tail-kernel blocks of each chunk
    // small tails, tail first (plain hec_spmv only): per ELL CTA tile, its tail
    // rows (the tail kernel stores their sums, the ELL kernel adds them)
    int32_t* d_fuse = nullptr;         // one allocation: cta ptr [n_cta + 1] | tail rows ascending
    const int32_t *d_fuse_cta = nullptr, *d_fuse_row = nullptr;
    int32_t fuse_tile = 0;             // rows per ELL CTA the map was built for (0: not fused)
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    std::vector<cudaEvent_t> ev_x, ev_y;
    cudaEvent_t ev_start = nullptr;
    int64_t device_bytes = 0;
};

namespace hec {
// Build a device (or host-only) matrix handle from a host HEC.
hec_status make_matrix(HostHec&& h, int32_t device, cudaStream_t s, const int32_t* rowmap,
                       int32_t n_rowmap, int32_t row_off, int32_t n_loc, hec_matrix* out,
                       bool coo_tail = false);
// Makes `dev` current for the scope, restoring the caller's device after.
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

// Launch the HEC product (ELL kernel then tail kernel) for one handle.
hec_status launch_spmv(const hec_matrix_s* A, const double* x, const double* x_halo, double* y,
                       cudaStream_t s);
hec_status launch_spmv_axpby(const hec_matrix_s* A, double alpha, const double* x, double beta, double* y,
                             cudaStream_t s);
struct PeerWait;
// The boundary product of the peer-memory transport: peer_wait_kernel, then the
// ELL kernel as its programmatic dependent, then the tail.
hec_status launch_spmv_peer(const hec_matrix_s* A, const double* x, const double* x_halo, double* y,
                            cudaStream_t s, const PeerWait& w);
}  // namespace hec

// ---------------------------------------------------------------- kernels --
namespace hec {
// Peer-memory halo transport (dist.cpp): peer_wait_kernel waits
// until every neighbour rank has released this call's epoch into flags[q]
// (ld.acquire.sys), with a ~10 s timeout that sets *err instead of hanging.
struct PeerWait {
    const uint64_t* flags = nullptr;  // this rank's arrival flags, one per source rank
    const int32_t* peers = nullptr;   // neighbour ranks to wait for
    int32_t n = 0;                    // 0: no wait
    uint64_t epoch = 0;
    int32_t* err = nullptr;
};
constexpr int32_t kPushChunk = 512;  // send entries per push CTA (2 per thread; 256-2048 measured alike)
struct PushArgs {                     // fused pack + NVLink store + release
    const double* x;                  // x_local
    const int32_t* idx;               // send_idx (grouped by destination rank)
    const int4* chunks;               // per CTA: {destination rank, first entry, end, halo position}
    int32_t n_chunks;
    double* const* peer_buf0;         // [n_parts] peer q's halo buffer 0 (buffer 1 follows it)
    const int64_t* peer_nhalo;        // [n_parts] peer q's halo length
    uint64_t* const* peer_flags;      // [n_parts] peer q's arrival flags
    const int32_t* nbr;               // neighbour ranks (send or receive side)
    int32_t n_nbr;
    int32_t rank;
    uint64_t epoch;
    unsigned int* done;               // CTA completion counter (self-resetting)
};

#ifndef HEC_ELL_PHASE
#define HEC_ELL_PHASE 8  // ELL widths above this load their slots in two phases (measured: 8 > 16 > 6)
#endif
// slots of a two-phase width loaded in the first phase: one before the
// middle (w = 9: 4 + 5), so warps whose rows all have <= 4 ELL entries skip
// the whole second phase (power-law step 0.4347 -> 0.4210 ms; 5 + 4 and 6 + 3
// measured, degree-sorted within +-1.3%: profiles/round2/phase/).
// HEC_ELL_P1_DELTA (tuning) shifts the split.
#ifndef HEC_ELL_P1_DELTA
#define HEC_ELL_P1_DELTA (-1)
#endif
__host__ __device__ constexpr int ell_first_phase(int w) { return (w + 1) / 2 + HEC_ELL_P1_DELTA; }
constexpr int kIdx16MaxW = 16;  // widths with compiled-in slot loops (compressed indices and slot skipping need one)
#ifndef HEC_GROUP_ROWS
#define HEC_GROUP_ROWS 1024  // measured 512 / 1024 / 4096: -0.1% / -1.0% / -0.6% on the power-law step
#endif
constexpr int32_t kGroupRows = HEC_GROUP_ROWS;  // windows in which rows are grouped by ELL length (a multiple of 512)
constexpr int16_t kIdxEsc = INT16_MIN;      // the int32 column must be read
constexpr int16_t kIdxPad = INT16_MIN + 1;  // padding slot (column -1)
struct EllArgs {
    const int32_t* col;
    const double* val;
    int64_t stride;
    int64_t avail;     // slot-column entries readable from `col`/`val` (stride - row offset)
    int32_t n_rows;
    int32_t width;
    const double* x;
    const double* x_halo;
    int32_t n_loc;
    double* y;
    const int32_t* rowmap;
    int32_t row_off;
    double alpha = 1.0, beta = 0.0;  // Eq. (2): y = alpha A x + beta y
    // damped-Jacobi epilogue (A22), when diag != null: y = x + omega ((b - A x) / diag),
    // with x, b, diag indexed by the output row (square, single matrix)
    const double* diag = nullptr;
    const double* b = nullptr;
    double omega = 0.0;
    bool pdl = false;  // launch as a programmatic dependent (peer-memory boundary rows)
    // per 64-row tile (one warp's rows): the tile's longest ELL row, when the
    // tiles' second-phase slots are worth skipping (rows grouped by length);
    // slots >= tile_w[i >> 6] are padding for every row of the tile and are not read
    const uint8_t* tile_w = nullptr;
    // small tails, tail first (plain y = A x of a whole matrix): the tail kernel
    // stored the tail rows' sums into y just before; CTA b adds them to its
    // rows fuse_row[fuse_cta[b] .. fuse_cta[b+1]) (ascending)
    const int32_t* fuse_cta = nullptr;
    const int32_t* fuse_row = nullptr;
    // 16-bit column deltas ("ELL index compression"): when d16 !=
    // null, slot j of row i stores d = col - (row0 + i) - base[j] as an int16
    // (same column-major position as col), kIdxPad for a padding slot and
    // kIdxEsc where the delta does not fit -- then the int32 column is read
    const int16_t* d16 = nullptr;
    int32_t row0 = 0;                 // row index of this launch's first row
    int32_t base[kIdx16MaxW] = {};   // per-slot delta base
};
struct TailArgs {
    const int4* blk;            // block descriptors {first row position, count, lg, first warp} (diag)
    const int4* warp;           // 8 per descriptor: {first entry, iterations, first row, count << 8 | lg}
    int64_t blk_begin, blk_end;
    const int32_t* out_rows;
    const int32_t* col;
    const double* val;
    const double* x;
    const double* x_halo;
    int32_t n_loc;
    double* y;
    double alpha = 1.0;  // the tail adds alpha * (its part of A x)
    bool reverse = false;     // CTA b takes descriptor blk_end - 1 - b (the ELL kernel's last rows first)
    bool store_only = false;  // store the row sums instead of adding them: into y (small tails first,
                              // the ELL kernel adds them) or into tsum (concurrent tail, combined after)
    double* tsum = nullptr;   // [tail rows], indexed by device row position
    // SM-local persistent schedule (tail_warp_kernel; whole launches only): warp
    // units [region[r], region[r+1]) are SM r's, claimed through region_ctr[r];
    // units[u] = {first warp-meta index, warp metas of the unit}
    const int64_t* region = nullptr;
    const int4* units = nullptr;        // per unit: its first warp meta (carried inline)
    const int32_t* unit_widx = nullptr; // per unit: that meta's index in `warp`
    int32_t n_regions = 0;
    unsigned int* region_ctr = nullptr;  // [n_regions], zero between launches
    unsigned int* region_done = nullptr; // CTA completion counter (self-resetting)
    const double* diag = nullptr;  // Jacobi (A22): the tail adds -omega * (its part / diag[row])
    double omega = 0.0;
    // x-ring schedule (tail_ring_kernel; whole launches of big banded tails):
    // CTA b walks stages [ring_cta[b], ring_cta[b+1]); a stage {lo, hi, u0, u1}
    // is a run of warp units of one super-block whose x columns [lo, hi) sit in
    // the CTA's shared-memory ring; ring_unit[u] = {warp meta, metas, warp index
    // in its descriptor, 0}
    const int4* ring_stage = nullptr;
    const int32_t* ring_cta = nullptr;
    const int4* ring_unit = nullptr;
    int32_t ring_ctas = 0;
};
struct CooArgs {               // HYB remainder: row-sorted (row, col, val) triplets
    int64_t nnz;
    const int32_t* row;        // output rows
    const int32_t* col;
    const double* val;
    const double* x;
    double* y;
    double alpha;
    const double* diag = nullptr;  // Jacobi (A22): adds -omega * (part / diag[row])
    double omega = 0.0;
};
cudaError_t launch_coo(const CooArgs& a, cudaStream_t s);
cudaError_t launch_ell(const EllArgs& a, cudaStream_t s);
// Threads per ELL CTA for a width (each thread owns a row pair), and the grid
// cap beyond which the ELL kernel strides (fused tails need one tile per CTA).
int ell_block_threads(int32_t width);
int64_t ell_grid_cap();
cudaError_t launch_tail(const TailArgs& a, cudaStream_t s);
cudaError_t launch_ell_tma(const EllArgs& a, cudaStream_t s, int num_sms);
cudaError_t launch_pack(const int32_t* idx, int32_t n, const double* x, double* out,
                        cudaStream_t s);
cudaError_t launch_tail_combine(const int32_t* out_rows, const double* tsum, int32_t n, double* y, cudaStream_t s);
// d[i] = A_ii of a square single-device handle: ELL scan, then the tail (warp
// chunks or COO)
cudaError_t launch_diag(const hec_matrix_s* A, double* d, cudaStream_t s);
cudaError_t launch_push(const PushArgs& a, cudaStream_t s);
cudaError_t launch_peer_wait(const PeerWait& w, cudaStream_t s);
}  // namespace hec
