/*
 * hec.h -- C ABI of libhec.so: fp64 sparse matrix-vector multiplication
 * y = A x in the HEC (hybrid ELL + CSR) format on NVIDIA B200 (sm_100a), on one
 * GPU and row-partitioned across GPUs with a halo exchange of off-partition x.
 *
 * Source of the operations: Yang, Liu, Chen, "Development of Krylov and AMG
 * linear solvers for large-scale sparse matrices on GPUs" (arXiv 1606.00545),
 * cited as PAPER.md line numbers (P:n):
 *   - HEC format: §2.1 "Matrix Format", P:50 (ELL part + CSR remainder with
 *     arrays Ap/Aj/Ax), P:73 (column-by-column ELL storage, stride a multiple
 *     of 32 set to 256, ELL/CSR boundary "a recommended value 20").
 *   - SpMV: §2.2 Alg. 1, P:126-140 (ELL part first, then the CSR part, one
 *     CUDA core per row); Eq. (1), P:73-122 (y = sum_k x_k A[:,k]).
 *   - Distribution: §2.2 P:149-158 (row partition -- "sequence partition" for
 *     FDM/FVM matrices; vector segments; off-segment x entries exchanged
 *     through a shared cache, here replaced by device-to-device transfers).
 * Readings of silent/ambiguous passages (A1..A16) are listed in DESIGN.md §3.
 *
 * Conventions (all functions):
 *   - Every call returns hec_status; no C++ exception crosses the ABI.  On
 *     failure hec_last_error() returns a thread-local message for the last
 *     failing call on the calling thread.
 *   - Host input arrays are BORROWED for the duration of the call (copied).
 *   - Handles are owned by the caller and released with the matching *_free.
 *   - Device pointers (x, y) are caller-owned, fp64, contiguous; `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream).  Compute
 *     calls are asynchronous with respect to the host; asynchronous CUDA/NCCL
 *     faults surface at the next synchronising call.
 *   - Indices are int32 and values fp64, as the paper's CSR (reading A8:
 *     Table 2's Mb(CSR) = round((12 nnz + 4(n+1))/2^20) for all 12 matrices).
 *   - There is no CPU fallback: a compute call on a handle without a device,
 *     or on a host without a CUDA device, fails with HEC_ERR_NODEV / _CUDA.
 */
#ifndef HEC_H
#define HEC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HEC_OK = 0,
    HEC_ERR_ARG = 1,     /* NULL handle/pointer, negative size, unknown enum, aliasing x/y */
    HEC_ERR_FORMAT = 2,  /* non-canonical CSR (reading A7): row_ptr[0] != 0,
                            decreasing row_ptr, row_ptr[n] != nnz, unsorted or duplicate
                            columns within a row, column out of [0, n_cols) */
    HEC_ERR_DIM = 3,     /* length mismatch (e.g. distributed mode on a non-square A) */
    HEC_ERR_PARTS = 4,   /* n_parts < 1 or > n_rows, grid dims inconsistent with n,
                            more parts than grid planes, part index out of range */
    HEC_ERR_CUDA = 5,    /* a CUDA runtime call failed (message in hec_last_error) */
    HEC_ERR_NCCL = 6,    /* an NCCL call failed */
    HEC_ERR_NOMEM = 7,   /* host or device allocation failed */
    HEC_ERR_STATE = 8,   /* handle used in the wrong mode (rank/plan mismatch, ...) */
    HEC_ERR_NODEV = 9    /* compute requested on a host-only handle (device = -1) */
} hec_status;

const char* hec_last_error(void);
const char* hec_version(void);

/* ------------------------------------------------------------ matrices ---- */

/* Canonical CSR (Ap = row_ptr, Aj = col_idx, Ax = val).
 * row_ptr[n_rows+1], col_idx[nnz], val[nnz]; host memory, borrowed. */
typedef struct {
    int32_t n_rows, n_cols;
    int64_t nnz;
    const int32_t* row_ptr;
    const int32_t* col_idx;
    const double* val;
} hec_csr;

enum { HEC_WIDTH_BG3 = 0, HEC_WIDTH_CAP = 1, HEC_WIDTH_FIXED = 2 };

/* Conversion options (NULL -> defaults: BG3, cap 20, stride_unit 256).
 *   width_policy  HEC_WIDTH_BG3 (reading A1): w = min(cap, k*), k* = smallest
 *                 k >= 0 with 3 * #{rows: len > k} < n_rows;
 *                 HEC_WIDTH_CAP: w = min(cap, max row length);
 *                 HEC_WIDTH_FIXED: w = fixed_width.
 *   cap           ELL/CSR boundary, default 20 ("a recommended value 20").
 *   stride_unit   ELL stride s = roundup(n_rows, stride_unit); a positive
 *                 multiple of 32, default 256 (reading A2). */
typedef struct {
    int32_t width_policy;
    int32_t cap;
    int32_t fixed_width;
    int32_t stride_unit;
} hec_opts;

void hec_opts_default(hec_opts* o);

typedef struct hec_matrix_s* hec_matrix;

typedef struct {
    int32_t n_rows, n_cols;
    int32_t ell_width;     /* w */
    int32_t ell_stride;    /* s */
    int64_t nnz;           /* nnz(A) = ell_nnz + tail_nnz */
    int64_t ell_nnz;       /* non-padding ELL slots */
    int32_t tail_rows;     /* rows that spill into the CSR part */
    int32_t tail_group;    /* maximum lanes per tail row used by the tail kernel (rows take 1..256) */
    int64_t tail_nnz;
    int64_t device_bytes;  /* bytes of device arrays owned by the handle */
    int32_t device;        /* CUDA device ordinal, or -1 for a host-only handle */
    int32_t tail_fused;    /* 1: hec_spmv runs a small CSR tail FIRST (its row sums stored into y)
                              and the ELL kernel, launched as its programmatic dependent, adds
                              them -- the tail's latency hides under the ELL stream */
    int32_t tail_ring;     /* 1: hec_spmv runs a big CSR tail with the x-ring schedule (one CTA
                              per SM; each stage's x window staged in shared memory) */
    int32_t ell_idx16;     /* 1: the device ELL part also holds 16-bit column deltas and the ELL
                              kernel streams those (10 instead of 12 bytes per slot; opt-in with
                              HEC_IDX16=1 at hec_from_csr, measured no faster: DESIGN §5) */
    double tail_ring_cover; /* fraction of the stored tail entries whose column lies in their
                               stage's x window (computed for ring candidates, else 0) */
    double ell_idx16_escaped; /* fraction of ELL slots whose delta does not fit 16 bits and are
                                 read as int32 (-1: not evaluated) */
    double ell_tile_skip;  /* fraction of the ELL slots the kernel skips: second-phase slots past the
                              longest row of a warp's 64 rows (two-phase widths) */
    int32_t ell_tile_w;    /* 1: the skipping is on for this handle */
    int32_t ell_grouped;   /* 1: the device ELL rows are grouped by length inside windows of 1024
                              rows (y is written through the permutation; hec_export returns row order) */
} hec_matrix_info;

/* Caller-allocated export buffers, sized from hec_matrix_info:
 * ell_col/ell_val [w*s] column-major (slot j of row i at j*s + i; padding
 * slots are (-1, +0.0), reading A4); tail_rows [tail_rows] ascending;
 * tail_ptr [tail_rows+1]; tail_col/tail_val [tail_nnz] (reading A15: the CSR
 * part is compact, only rows with a spill).  Any pointer may be NULL to skip. */
typedef struct {
    int32_t* ell_col;
    double* ell_val;
    int32_t* tail_rows;
    int32_t* tail_ptr;
    int32_t* tail_col;
    double* tail_val;
} hec_host_arrays;

/* CSR -> HEC conversion (readings A1-A4, A15).  Validates A
 * (HEC_ERR_FORMAT), chooses w, fills the column-major ELL part with each row's
 * first min(len, w) entries in column order and the compact CSR tail with the
 * rest.  device >= 0: uploads to that CUDA device on `stream` (synchronised
 * before return).  device == -1: host-only handle, usable with hec_info and
 * hec_export (conversion checks without a GPU) but not for compute. */
hec_status hec_from_csr(const hec_csr* A, const hec_opts* o, int32_t device, void* stream,
                        hec_matrix* out);
/* Comparison variant (the paper's Table 3 formats): the
 * same ELL part, but the remainder kept in COO as in Bell & Garland's HYB
 * ("HYB (Hybrid of ELL and COO)") and added with fp64 atomics.  The
 * product is correct within the usual tolerance but the addition order of a
 * row's COO pieces is not fixed.  hec_spmv / hec_spmv_axpby / hec_spmv_host
 * accept the handle; hec_export returns the remainder as CSR.  device >= 0. */
hec_status hec_from_csr_hyb(const hec_csr* A, const hec_opts* o, int32_t device, void* stream,
                            hec_matrix* out);
hec_status hec_info(hec_matrix A, hec_matrix_info* out);
hec_status hec_export(hec_matrix A, hec_host_arrays* out);

/* y = A x (Alg. 1): the ELL kernel writes every row of y, then the
 * CSR-tail kernel adds the spilled entries of the tail rows (a small tail --
 * one wave of tail CTAs -- runs first instead, storing its row sums, and the
 * ELL kernel adds them: the same y bit for bit).  x: device, n_cols doubles;
 * y: device, n_rows doubles, fully overwritten; x and y must not overlap
 * (HEC_ERR_ARG).  Asynchronous on `stream`.  Calls on ONE handle must be
 * ordered (one stream, or synchronised): a big tail's SM-local schedule keeps
 * its claim counters in the handle. */
hec_status hec_spmv(hec_matrix A, const double* x, double* y, void* stream);

/* Same product with HOST x and y (n_cols / n_rows doubles; pinned memory is
 * fastest).  Copies x host->device, runs hec_spmv on library-owned device
 * buffers, copies y device->host and synchronises `stream` before returning. */
hec_status hec_spmv_host(hec_matrix A, const double* x_host, double* y_host, void* stream);

/* Number of kernels one hec_spmv launches on this matrix (1 or 2). */
int32_t hec_spmv_launches(hec_matrix A);

/* Eq. (2) (PAPER §2.3): y = alpha A x + beta y, fused into the
 * SpMV epilogue (the ELL kernel writes alpha*ell + beta*y_old, the CSR-tail
 * kernel adds alpha*tail).  beta == 0: y is not read (may hold NaN/garbage).
 * x, y: device, must not overlap.  Asynchronous on `stream`. */
hec_status hec_spmv_axpby(hec_matrix A, double alpha, const double* x, double beta, double* y,
                          void* stream);

/* d[i] = A_ii: the stored diagonal entry of row i, +0.0 when the row stores
 * none (A22).  A must be a square whole-matrix device handle
 * (HEC_ERR_DIM otherwise; HEC_ERR_NODEV for a host-only handle).  d: device,
 * n_rows doubles, fully overwritten.  Asynchronous on `stream`; setup-time. */
hec_status hec_diag(hec_matrix A, double* d, void* stream);

/* One damped-Jacobi sweep, the SpMV-based smoother of the paper's AMG ("damped
 * Jacobi"; "developed based on the SpMV and vector operations", P:542;
 * formula: DESIGN.md A22):
 *     x_out = x + omega * D^{-1} (b - A x),   D = diag(d)
 * fused into the SpMV epilogue (the ELL kernel writes x + omega((b - s_ell)/d),
 * the CSR-tail kernel subtracts omega(s_tail/d)); no FMA contraction in the
 * update.  A: square whole-matrix device handle (HEC_ERR_DIM).  d, b, x, x_out:
 * device, n_rows doubles; x_out is fully overwritten and must not overlap x, b
 * or d (HEC_ERR_ARG); rows with d_i = 0 give IEEE Inf/NaN.  Asynchronous on
 * `stream`. */
hec_status hec_jacobi(hec_matrix A, const double* d, const double* b, const double* x, double* x_out,
                      double omega, void* stream);

/* ------------------------------------------------------ vector operations ---- */
/* PAPER §2.3 Eqs. (3)-(6), on device vectors of length n
 * (asynchronous on `stream` unless stated):
 *   hec_axpby : y = alpha x + beta y   (Eq. 3)
 *   hec_axpbyz: z = alpha x + beta y   (Eq. 4; z may alias x or y)
 *   hec_dot   : *result = <x, y>       (Eq. 5; host result, synchronises)
 *   hec_norm2 : *result = ||x||_2      (Eq. 6; host result, synchronises)
 * Reductions use a fixed grid and a fixed summation order: deterministic. */
hec_status hec_axpby(int64_t n, double alpha, const double* x, double beta, double* y, void* stream);
hec_status hec_axpbyz(int64_t n, double alpha, const double* x, double beta, const double* y, double* z,
                      void* stream);
hec_status hec_dot(int64_t n, const double* x, const double* y, double* result, void* stream);
hec_status hec_norm2(int64_t n, const double* x, double* result, void* stream);

/* ------------------------------------------------------- Krylov solvers ---- */
/* The consumers of the SpMV in the paper (§2.8): BiCGSTAB exactly as
 * Alg. 4 with M = I (unpreconditioned; preconditioners are out of scope) and
 * shadow residual r0 = b - A x0, and CG ("implemented") for SPD A.
 * b: device rhs; x: device, initial guess on entry, iterate on return.
 * Stops when ||s||_2 or ||r||_2 <= tol ||r0||_2 (Alg. 4's two tests; CG: ||r||),
 * after max_it iterations, or on breakdown (rho = 0 -> breakdown = 1;
 * omega = 0 -> breakdown = 2; (r0, v) = 0, where Alg. 4's alpha is undefined
 * -> breakdown = 3, reading A20; (t, t) = 0 or a non-finite omega in BiCGSTAB,
 * (p, A p) = 0 or a non-finite alpha in CG -> breakdown = 4: x keeps the last
 * finite iterate).  Scalars, tests and breakdown checks stay on
 * the device (a done flag turns later passes into no-ops); the host reads the
 * state once per batch of iterations.  The first solve on a handle caches a
 * workspace of 6 n-vectors in it (freed with the handle); concurrent solves
 * on one handle from several host threads are safe (the second one allocates
 * its own).  Synchronises `stream` before returning. */
typedef struct {
    int32_t iterations;
    int32_t converged;
    int32_t breakdown;
    int32_t reserved;
    double rel_residual;  /* recurrence ||r_k||_2 / ||r_0||_2 at exit */
} hec_solve_info;

hec_status hec_bicgstab(hec_matrix A, const double* b, double* x, double tol, int32_t max_it, void* stream,
                        hec_solve_info* info);
hec_status hec_cg(hec_matrix A, const double* b, double* x, double tol, int32_t max_it, void* stream,
                  hec_solve_info* info);

void hec_free(hec_matrix A);

/* ---------------------------------------------------------- partitions ---- */

enum { HEC_PART_CONTIG_NNZ = 0, HEC_PART_CONTIG_ROWS = 1, HEC_PART_GRID = 2, HEC_PART_CONTIG_COST = 3,
       HEC_PART_EXPLICIT = 4 };

typedef struct hec_plan_s* hec_plan;

/* Row partition + halo plan ("sequence partition", P:158 vector
 * segments and the exchange of entries "a segment vector can not provide";
 * readings A9-A12).  A must be square (the row partition is also the vector
 * partition).  kind:
 *   HEC_PART_GRID: grid = {nx, ny, nz} with nx*ny*nz = n; part p owns planes
 *     [floor(p*E/P), floor((p+1)*E/P)) of the slowest axis with extent E > 1.
 *   HEC_PART_CONTIG_ROWS: part_ptr[p] = floor(p*n/P).
 *   HEC_PART_CONTIG_NNZ: part_ptr[p] = lower_bound(row_ptr, ceil(p*nnz/P)),
 *     then max(., part_ptr[p-1]+1), then min(., n-(P-p)).
 *   HEC_PART_CONTIG_COST (not in the paper): start from
 *     CONTIG_NNZ; then 4 times (stopping early at a fixed point): with w_p =
 *     the BG3 width (default options) of part p's rows, row i of part p costs
 *     3 w_p + 4 max(len_i - w_p, 0) (padded ELL slots + tail entries, weights
 *     from measured part times); part_ptr[p] = lower_bound(prefix cost,
 *     ceil(p C / P)), clamped as for CONTIG_NNZ.
 * For every part: recv = sorted global columns referenced outside the part;
 * sends to peer q = sorted local indices of recv_q inside the part; boundary
 * rows = rows with any off-part column; interior = the rest.  Host-only,
 * deterministic, immutable. */
/*   HEC_PART_EXPLICIT: grid = part_ptr[n_parts + 1] given by the caller
 *     (0 = part_ptr[0] < part_ptr[1] < ... < part_ptr[n_parts] = n), e.g. from
 *     hec_partition_order after B = P A P^T. */
hec_status hec_partition(const hec_csr* A, int32_t n_parts, int32_t kind, const int32_t* grid,
                         hec_plan* out);

typedef struct {
    int32_t r0, r1;          /* owned global rows [r0, r1) */
    int32_t n_halo;          /* |recv| */
    int32_t n_send;          /* total entries sent to all peers */
    int32_t n_interior, n_boundary;
    int32_t n_recv_peers, n_send_peers;
    int32_t width;           /* partition ELL width (reading A12) under the opts given to
                                hec_plan_part_info_opts; BG3/20 for hec_plan_part_info */
    int32_t reserved;
} hec_part_info;

/* Caller-allocated: recv_cols[n_halo] (global, ascending), recv_off[P+1],
 * send_idx[n_send] (local), send_off[P+1], interior[n_interior] and
 * boundary[n_boundary] (local row ids, ascending).  NULL entries are skipped. */
typedef struct {
    int32_t* recv_cols;
    int32_t* recv_off;
    int32_t* send_idx;
    int32_t* send_off;
    int32_t* interior;
    int32_t* boundary;
} hec_plan_arrays;

hec_status hec_plan_n_parts(hec_plan P, int32_t* n_parts);
hec_status hec_plan_part_ptr(hec_plan P, int32_t* part_ptr /* [n_parts+1] */);
hec_status hec_plan_part_info(hec_plan P, int32_t part, hec_part_info* out);
hec_status hec_plan_part_info_opts(hec_plan P, int32_t part, const hec_opts* o, hec_part_info* out);
hec_status hec_plan_export(hec_plan P, int32_t part, hec_plan_arrays* out);

enum { HEC_SUB_INTERIOR = 0, HEC_SUB_BOUNDARY = 1, HEC_SUB_ALL = 2 };

/* HEC of one part's local rows (which = interior, boundary, or all), with local
 * columns (owned -> [0, n_loc), halo entry g -> n_loc + position of g in recv),
 * each row in ascending local-column order, and the partition's width
 * (reading A12).  A must be the matrix the plan was built from. */
hec_status hec_plan_part_hec(hec_plan P, const hec_csr* A, int32_t part, int32_t which,
                             const hec_opts* o, int32_t device, void* stream, hec_matrix* out);
void hec_plan_free(hec_plan P);

/* Reordering for irregular matrices ("the rows of the matrix are
 * switched first and all the nonzero entries are put along the diagonal as
 * close as possible"; METIS is not available offline -- reading A21):
 *   hec_reorder_rcm: deterministic reverse Cuthill-McKee ordering of the
 *     pattern of A + A^T; perm[new] = old (caller-allocated, n entries).
 *   hec_permute: B = P A P^T, i.e. B[i][j] = A[perm[i]][perm[j]], canonical
 *     (rows re-sorted); caller allocates row_ptr_out[n+1], col_out[nnz],
 *     val_out[nnz].  Vectors follow with x_new[i] = x[perm[i]].
 * Square A only (HEC_ERR_DIM); perm must be a permutation (HEC_ERR_ARG). */
hec_status hec_reorder_rcm(const hec_csr* A, int32_t* perm);

/* Partitioning orders for irregular matrices (NEXT-4; the contract of SPEC's
 * partition_rows, implementation per S:188 -- METIS is out of
 * reach offline, reading A21).  Graph = pattern of A + A^T without the
 * diagonal, edge weight = stored entries it stands for (1 or 2).
 *   HEC_ORDER_BISECT: recursive bisection by BFS level sets from a
 *     pseudo-peripheral vertex (George-Liu), lowest index first; parts
 *     balanced by rows (sizes within 1 when n_parts | n on connected graphs).
 *   HEC_ORDER_MULTILEVEL: multilevel k-way (heavy-edge matching, spectral
 *     order of the coarsest graph cut into equal-nonzero pieces, greedy
 *     boundary refinement at every level; the best edge cut of 3 matching
 *     orders); parts balanced by nonzeros within 3%.
 * Outputs (caller-allocated): perm[n] with perm[new] = old, the parts
 * contiguous in the new order, and part_ptr[n_parts + 1].  Partition B =
 * P A P^T (hec_permute) with HEC_PART_EXPLICIT and part_ptr.  Deterministic.
 * Square A only (HEC_ERR_DIM); 1 <= n_parts <= n (HEC_ERR_PARTS). */
enum { HEC_ORDER_BISECT = 0, HEC_ORDER_MULTILEVEL = 1 };
hec_status hec_partition_order(const hec_csr* A, int32_t n_parts, int32_t method, int32_t* perm, int32_t* part_ptr);
hec_status hec_permute(const hec_csr* A, const int32_t* perm, int32_t* row_ptr_out, int32_t* col_out,
                       double* val_out);

/* -------------------------------------------------------- distributed ---- */

typedef struct hec_dist_s* hec_dist;

#define HEC_NCCL_ID_BYTES 128

/* Rank 0 creates the NCCL unique id and broadcasts it (e.g. torch.distributed). */
hec_status hec_nccl_unique_id(uint8_t id[HEC_NCCL_ID_BYTES]);

/* COLLECTIVE over the n_parts ranks (ncclCommInitRank).  Builds this rank's
 * interior and boundary sub-HECs on `device`, the halo send list, the send and
 * x_halo buffers, a high-priority communication stream and events. */
hec_status hec_dist_create(const hec_csr* A, hec_plan P, const hec_opts* o, int32_t rank,
                           const uint8_t id[HEC_NCCL_ID_BYTES], int32_t device, hec_dist* out);

/* Single-process emulation of all n_parts ranks on ONE device (for testing the
 * distributed kernels on one GPU): out[n_parts] handles whose exchange is a
 * device-to-device copy instead of NCCL.  Free each with hec_dist_free. */
hec_status hec_dist_create_local(const hec_csr* A, hec_plan P, const hec_opts* o, int32_t device,
                                 hec_dist* out);

/* COLLECTIVE: y_local = (A x)[r0:r1] for this rank (every rank calls it in the
 * same order).  x_local/y_local: device, n_loc doubles, must not overlap.
 * On `stream`: the interior SpMV (x_local only) runs while a high-priority
 * stream exchanges the halo with the peers -- the peer-memory push kernel once
 * the handle is connected (hec_dist_enable_p2p / hec_dist_p2p_connect, below),
 * else a pack kernel and NCCL grouped send/recv -- and then runs the boundary
 * SpMV.  HEC_ERR_STATE for a multi-rank handle with neither transport.
 * Asynchronous; ordered after prior work on `stream` and before later work on it. */
hec_status hec_spmv_dist(hec_dist D, const double* x_local, double* y_local, void* stream);

/* COLLECTIVE, end to end with HOST buffers (the distributed analogue of
 * hec_spmv_host): copies x_host_local (n_loc doubles, pageable or pinned) to a
 * device staging buffer on `stream`, runs hec_spmv_dist, copies y back into
 * y_host_local (n_loc doubles) and synchronises `stream`.  Staging buffers are
 * allocated by the first call and kept in the handle (calls on one handle must
 * therefore not overlap). */
hec_status hec_spmv_dist_host(hec_dist D, const double* x_host_local, double* y_host_local, void* stream);

/* Phase timing of hec_spmv_dist (the overlap evidence of SURVEY §8(a) a10):
 * with timing on, every call records CUDA events at its start (caller's
 * stream), at the end of the interior rows (caller's stream) and at the end
 * of the exchange + boundary rows (communication stream).
 * hec_dist_phase_times (synchronises them) gives, for the LAST call, both ends
 * in ms from the call's start: interior_ms, and comm_ms (-1 when the call had
 * no exchange).  comm_ms <= interior_ms means the exchange and the boundary
 * rows were entirely hidden behind the interior rows.  HEC_ERR_STATE without
 * a timed call. */
hec_status hec_dist_set_timing(hec_dist D, int32_t enable);
hec_status hec_dist_phase_times(hec_dist D, float* interior_ms, float* comm_ms);

/* The handle's NCCL communicator: *nranks = ncclCommCount (0 when the handle
 * has none: P = 1 or a peer-memory-only handle), *version = ncclGetVersion. */
hec_status hec_dist_comm_size(hec_dist D, int32_t* nranks, int32_t* version);

/* ---- peer-memory halo transport ----
 * The export of P:158 without NCCL: every rank exposes a receive window (its
 * arrival flags and two halo buffers, alternating by call parity) through CUDA
 * IPC; per hec_spmv_dist one push kernel gathers x_local[send_idx] and stores
 * each entry straight into the destination rank's window over NVLink, fences
 * at system scope and releases the call's epoch into every neighbour's flag;
 * a one-CTA kernel acquires the neighbours' flags and the boundary SpMV runs
 * as its programmatic dependent.  Neighbours always exchange flags (even with
 * no data), which is what makes the double-buffered window safe to reuse.
 * A missing peer times out after ~10 s instead of hanging (hec_dist_check). */
#define HEC_IPC_BYTES 64

/* Like hec_dist_create but with no NCCL communicator: builds this rank's
 * state, allocates its window and writes its CUDA IPC handle to handle_out.
 * The caller all-gathers the n_parts handles (any transport, e.g.
 * torch.distributed) and passes them to hec_dist_p2p_connect. */
hec_status hec_dist_create_p2p(const hec_csr* A, hec_plan P, const hec_opts* o, int32_t rank, int32_t device,
                               hec_dist* out, uint8_t handle_out[HEC_IPC_BYTES]);

/* handles: n_parts x HEC_IPC_BYTES in rank order (own entry ignored).  Maps
 * every neighbour's window (cudaIpcOpenMemHandle) and switches D to the
 * peer-memory transport.  Every rank must have created its window first. */
hec_status hec_dist_p2p_connect(hec_dist D, const uint8_t* handles);

/* COLLECTIVE, for handles from hec_dist_create: allocates the window,
 * all-gathers the IPC handles over the handle's NCCL communicator and
 * connects, so hec_spmv_dist uses the peer-memory transport while the
 * distributed solvers keep NCCL for their all-reduces. */
hec_status hec_dist_enable_p2p(hec_dist D);

/* The local-emulation handles (hec_dist_create_local) switched to the
 * peer-memory transport: the windows are plain device pointers of this
 * process; hec_spmv_dist_local then runs every push before any wait. */
hec_status hec_dist_p2p_connect_local(hec_dist* D, int32_t n);

/* Synchronises the handle's communication stream and reports HEC_ERR_STATE
 * if a peer-memory wait timed out (the affected results are garbage). */
hec_status hec_dist_check(hec_dist D);

/* Local emulation: one call performs the exchange and both SpMV phases for
 * all n handles created by hec_dist_create_local, in rank order, on `stream`. */
hec_status hec_spmv_dist_local(hec_dist* D, int32_t n, const double* const* x_locals,
                               double* const* y_locals, void* stream);

typedef struct {
    int32_t rank, n_parts, r0, r1, n_halo, n_send;
    int32_t n_interior, n_boundary;
    int32_t width;
    int32_t launches;        /* kernels this rank launches per hec_spmv_dist (excl. NCCL's own) */
    int64_t device_bytes;
    int64_t algorithmic_bytes;  /* 12 nnz_loc + 8 (n_loc + n_halo) + 8 n_loc */
    int64_t nnz_local;
} hec_dist_info;

hec_status hec_dist_get_info(hec_dist D, hec_dist_info* out);

/* COLLECTIVE distributed solvers: every rank passes its segments of b and x
 * (n_loc each); SpMVs are hec_spmv_dist and the dot products are all-reduced
 * with ncclAllReduce over this rank set (replacing the paper's CPU summation
 * of per-GPU partial results).  Not available on local-emulation handles. */
hec_status hec_bicgstab_dist(hec_dist D, const double* b_local, double* x_local, double tol, int32_t max_it,
                             void* stream, hec_solve_info* info);
hec_status hec_cg_dist(hec_dist D, const double* b_local, double* x_local, double tol, int32_t max_it,
                       void* stream, hec_solve_info* info);
/* The same two solvers over ALL n ranks of a local emulation
 * (hec_dist_create_local, handles in rank order) on one device and one
 * stream: SpMVs are hec_spmv_dist_local; each rank's dot partials are reduced
 * in its fixed order and the per-rank results summed in rank order (a
 * stand-in for ncclAllReduce -- one valid order of the same sum), so the
 * distributed solvers' P > 1 logic runs without P GPUs.  b_locals[p] /
 * x_locals[p]: rank p's device segments (n_loc(p) doubles); x holds x0 on
 * entry.  Synchronises `stream`. */
hec_status hec_bicgstab_dist_local(hec_dist* D, int32_t n, const double* const* b_locals, double* const* x_locals,
                                   double tol, int32_t max_it, void* stream, hec_solve_info* info);
hec_status hec_cg_dist_local(hec_dist* D, int32_t n, const double* const* b_locals, double* const* x_locals,
                             double tol, int32_t max_it, void* stream, hec_solve_info* info);
void hec_dist_free(hec_dist D);

#ifdef __cplusplus
}
#endif
#endif /* HEC_H */
