// krylov.cu -- the consumers of the SpMV hot path:
// the vector operations of PAPER.md §2.3 (Eqs. (3)-(6)), the
// unpreconditioned BiCGSTAB of Alg. 4 (M = I) and CG ("implemented",
// P:294), on one GPU (hec_matrix) or row-partitioned (hec_dist).
//
// Design (B200): the whole iteration stays on the device and on one stream.
//  - Fused vector passes, one specialised kernel per update (4 independent
//    elements per thread per trip), write per-block partial dot products from a FIXED grid; a
//    one-block kernel sums them in a fixed order (deterministic) into a small
//    device scalar array.  In distributed mode an ncclAllReduce over those few
//    doubles replaces the paper's "sub results are sent back to CPU".
//  - A one-thread "step" kernel derives alpha / beta / omega and evaluates
//    Alg. 4's tests (||s||, ||r||, rho = 0, omega = 0) ON THE DEVICE, setting
//    a done flag and the iteration count; every later vector pass sees the
//    flag and does nothing, so x and r freeze exactly at the stopping point.
//  - The host enqueues batches of iterations and reads the scalars once per
//    batch (no per-iteration host round trip).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "hec_internal.h"

struct hec_dist_s;  // dist.cpp

namespace hec {

// scalar slots
enum {
    SC_RHO = 0, SC_RHO_PREV, SC_ALPHA, SC_OMEGA, SC_BETA,
    SC_D0, SC_D1,          // reduced dot products of the last pass
    SC_R0NORM, SC_THR,     // ||r0||, tol ||r0||
    SC_DONE,               // 0 running; 1 converged; 2 breakdown / stop
    SC_CONV, SC_BREAK, SC_ITER, SC_RES,  // converged flag, breakdown code, iterations, ||r||/||r0||
    SC_FINAL_S,            // BiCGSTAB stopped on ||s||: x += alpha p still to apply
    SC_N
};

enum VecOp {
    OP_DOT1,      // d0 = (a, b)
    OP_DOT2,      // d0 = (a, b), d1 = (c, d)
    OP_RESID,     // r = b - v ; r0 = r ; d0 = (r, r)
    OP_COPY,      // p = r
    OP_BICG_P,    // p = r + beta (p - omega v)
    OP_BICG_S,    // s = r - alpha v ; d0 = (s, s)
    OP_BICG_XR,   // x = x + alpha p + omega s ; r = s - omega t ; d0 = (r, r) ; d1 = (r0, r)
    OP_X_ALPHA_P, // x = x + alpha p   (only when SC_FINAL_S is set)
    OP_CG_XR,     // x = x + alpha p ; r = r - alpha q ; d0 = (r, r)
    OP_CG_P,      // p = r + beta p
    OP_AXPBY,     // y = ca x + cb y            (Eq. 3)
    OP_AXPBYZ,    // z = ca x + cb y            (Eq. 4)
};

struct VecArgs {
    int64_t n;
    double* sc;         // device scalars; null for the stand-alone Eq. (3)-(6) calls
    double* part;       // [2][kRedBlocks] partial dots (null: no dots)
    unsigned int* ctr;  // non-null: the last CTA reduces the partials and runs the step (fused)
    int n_dots;         // dots this pass produces (fused reduce)
    int step_mode;      // step to run after the reduce (-1: none)
    int first;
    double tol;
    bool vec2;          // every vector 16-byte aligned: 128-bit loads/stores of element pairs
    double ca, cb;      // coefficients of OP_AXPBY / OP_AXPBYZ
    double *x, *r, *r0, *p, *v, *s, *t, *b;
    const double *a1, *b1, *c1, *d1;
};

constexpr int kRedBlocks = 1184;   // 8 x 148: fixed grid => fixed summation order
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    if (w == 0)
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    return v;  // valid in thread 0
}

// Element pairs: the same expressions on two adjacent elements through one
// 128-bit access per vector.
struct D2 { double x, y; };
__device__ __forceinline__ D2 operator+(D2 a, D2 b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ D2 operator-(D2 a, D2 b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ D2 operator*(double c, D2 a) { return {c * a.x, c * a.y}; }

template <typename T> __device__ __forceinline__ T LD(const double* p, int64_t i);
template <> __device__ __forceinline__ double LD<double>(const double* p, int64_t i) { return p[i]; }
template <> __device__ __forceinline__ D2 LD<D2>(const double* p, int64_t i) {
    const double2 v = reinterpret_cast<const double2*>(p)[i];
    return {v.x, v.y};
}
__device__ __forceinline__ void ST(double* p, int64_t i, double v) { p[i] = v; }
__device__ __forceinline__ void ST(double* p, int64_t i, D2 v) {
    reinterpret_cast<double2*>(p)[i] = make_double2(v.x, v.y);
}
__device__ __forceinline__ void ACC(double& d, double a, double b) { d += a * b; }
__device__ __forceinline__ void ACC(double& d, D2 a, D2 b) { d += a.x * b.x; d += a.y * b.y; }

// One unit (an element, or a pair when T = D2) of each op; d0/d1 accumulate
// the pass's dot products.
template <int OP, typename T>
__device__ __forceinline__ void vec_elem(const VecArgs& a, int64_t i, double alpha, double omega, double beta,
                                         double& d0, double& d1) {
    if (OP == OP_DOT1) { ACC(d0, LD<T>(a.a1, i), LD<T>(a.b1, i)); }
    if (OP == OP_DOT2) { ACC(d0, LD<T>(a.a1, i), LD<T>(a.b1, i)); ACC(d1, LD<T>(a.c1, i), LD<T>(a.d1, i)); }
    if (OP == OP_RESID) { const T ri = LD<T>(a.b, i) - LD<T>(a.v, i); ST(a.r, i, ri); ST(a.r0, i, ri); ACC(d0, ri, ri); }
    if (OP == OP_COPY) { ST(a.p, i, LD<T>(a.r, i)); }
    if (OP == OP_BICG_P) { ST(a.p, i, LD<T>(a.r, i) + beta * (LD<T>(a.p, i) - omega * LD<T>(a.v, i))); }
    if (OP == OP_BICG_S) { const T si = LD<T>(a.r, i) - alpha * LD<T>(a.v, i); ST(a.s, i, si); ACC(d0, si, si); }
    if (OP == OP_BICG_XR) {
        const T si = LD<T>(a.s, i);
        ST(a.x, i, LD<T>(a.x, i) + alpha * LD<T>(a.p, i) + omega * si);
        const T ri = si - omega * LD<T>(a.t, i);
        ST(a.r, i, ri); ACC(d0, ri, ri); ACC(d1, LD<T>(a.r0, i), ri);
    }
    if (OP == OP_X_ALPHA_P) { ST(a.x, i, LD<T>(a.x, i) + alpha * LD<T>(a.p, i)); }
    if (OP == OP_CG_XR) {
        ST(a.x, i, LD<T>(a.x, i) + alpha * LD<T>(a.p, i));
        const T ri = LD<T>(a.r, i) - alpha * LD<T>(a.v, i);
        ST(a.r, i, ri); ACC(d0, ri, ri);
    }
    if (OP == OP_CG_P) { ST(a.p, i, LD<T>(a.r, i) + beta * LD<T>(a.p, i)); }
    if (OP == OP_AXPBY) { ST(a.r, i, a.ca * LD<T>(a.a1, i) + a.cb * LD<T>(a.r, i)); }
    if (OP == OP_AXPBYZ) { ST(a.r, i, a.ca * LD<T>(a.a1, i) + a.cb * LD<T>(a.b1, i)); }
}

__device__ void step_body(double* sc, int mode, double tol, int first);

template <int OP, typename T>
__device__ __forceinline__ void vec_loop(const VecArgs& a, int64_t n_units, double alpha, double omega,
                                         double beta, double& d0, double& d1) {
    // 4 independent units per thread per trip (memory-level parallelism)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n_units; i += 4 * stride) {
#pragma unroll
        for (int u = 0; u < 4; ++u) vec_elem<OP, T>(a, i + u * stride, alpha, omega, beta, d0, d1);
    }
    for (; i < n_units; i += stride) vec_elem<OP, T>(a, i, alpha, omega, beta, d0, d1);
}

template <int OP>
__global__ void __launch_bounds__(kRedThreads) vec_kernel(VecArgs a) {
    __shared__ double sh[2][32];
    __shared__ bool last;
    double alpha = 0.0, omega = 0.0, beta = 0.0;
    bool skip = false;
    if (a.sc) {
        skip = a.sc[SC_DONE] != 0.0;
        if (OP == OP_X_ALPHA_P) skip = a.sc[SC_FINAL_S] != 1.0;
        alpha = a.sc[SC_ALPHA];
        omega = a.sc[SC_OMEGA];
        beta = a.sc[SC_BETA];
    }
    double d0 = 0.0, d1 = 0.0;
    if (!skip) {
        if (a.vec2) {
            vec_loop<OP, D2>(a, a.n >> 1, alpha, omega, beta, d0, d1);
            if ((a.n & 1) && blockIdx.x == 0 && threadIdx.x == 0)  // odd length: the last element
                vec_elem<OP, double>(a, a.n - 1, alpha, omega, beta, d0, d1);
        } else {
            vec_loop<OP, double>(a, a.n, alpha, omega, beta, d0, d1);
        }
    }
    if (a.part) {
        d0 = block_sum(d0, sh[0]);
        d1 = block_sum(d1, sh[1]);
        if (threadIdx.x == 0) {
            a.part[blockIdx.x] = d0;
            a.part[kRedBlocks + blockIdx.x] = d1;
        }
    }
    if (a.ctr) {
        // fused reduce + step: the last CTA to finish sums the partials in the
        // fixed order of reduce_kernel and runs the scalar step (one launch
        // instead of three; the summation order, hence every bit, is unchanged)
        if (threadIdx.x == 0) {
            __threadfence();
            last = atomicAdd(a.ctr, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (last) {
            __threadfence();
            for (int k = 0; k < a.n_dots; ++k) {
                double v = 0.0;
                for (int b = threadIdx.x; b < kRedBlocks; b += blockDim.x) v += __ldcg(a.part + k * kRedBlocks + b);
                v = block_sum(v, sh[0]);
                if (threadIdx.x == 0) a.sc[SC_D0 + k] = v;
            }
            if (threadIdx.x == 0) {
                if (a.step_mode >= 0) step_body(a.sc, a.step_mode, a.tol, a.first);
                *a.ctr = 0;
            }
        }
    }
}

// Sum the per-block partials in a fixed order: sc[SC_D0 + k] = sum_b part[k][b].
__global__ void __launch_bounds__(kRedThreads) reduce_kernel(const double* part, int n_parts, double* sc) {
    __shared__ double sh[32];
    for (int k = 0; k < n_parts; ++k) {
        double v = 0.0;
        for (int b = threadIdx.x; b < kRedBlocks; b += blockDim.x) v += part[k * kRedBlocks + b];
        v = block_sum(v, sh);
        if (threadIdx.x == 0) sc[SC_D0 + k] = v;
    }
}

enum Step {
    ST_INIT,          // after r0: rho = ||r0||^2, thresholds; done if r0 = 0
    ST_BICG_BEGIN,    // top of iteration k: count it; rho = 0 -> "Fails"; beta (k > 1)
    ST_BICG_ALPHA,    // alpha = rho / (r0, v); (r0, v) = 0 -> breakdown 3
    ST_BICG_S,        // ||s|| <= thr -> converged (x += alpha p pending)
    ST_BICG_OMEGA,    // omega = (t, s) / (t, t); (t, t) = 0 or omega not finite -> breakdown 4
    ST_BICG_R,        // ||r|| <= thr -> converged; omega = 0 -> breakdown 2; rho = (r0, r)
    ST_CG_ALPHA,      // count the iteration; alpha = rho / (p, q); (p, q) = 0 -> breakdown 4
    ST_CG_R,          // rho_new = (r, r): converged?; beta = rho_new / rho
    ST_FINAL_DONE,    // clear the pending x += alpha p
};

__device__ void step_body(double* sc, int mode, double tol, int first) {
    if (mode == ST_FINAL_DONE) { if (sc[SC_FINAL_S] == 1.0) sc[SC_FINAL_S] = 2.0; return; }
    if (sc[SC_DONE] != 0.0) return;
    switch (mode) {
        case ST_INIT: {
            const double r0n = sqrt(sc[SC_D0]);
            sc[SC_RHO] = sc[SC_D0];
            sc[SC_R0NORM] = r0n;
            sc[SC_THR] = tol * r0n;
            sc[SC_ITER] = 0.0;
            sc[SC_RES] = r0n > 0.0 ? 1.0 : 0.0;
            if (r0n == 0.0) { sc[SC_DONE] = 1.0; sc[SC_CONV] = 1.0; }
            break;
        }
        case ST_BICG_BEGIN:
            sc[SC_ITER] += 1.0;
            if (sc[SC_RHO] == 0.0) { sc[SC_DONE] = 2.0; sc[SC_BREAK] = 1.0; break; }          // "Fails"
            if (!first) sc[SC_BETA] = (sc[SC_RHO] / sc[SC_RHO_PREV]) * (sc[SC_ALPHA] / sc[SC_OMEGA]);
            break;
        case ST_BICG_ALPHA:
            if (sc[SC_D0] == 0.0) { sc[SC_DONE] = 2.0; sc[SC_BREAK] = 3.0; break; }           // reading A20
            sc[SC_ALPHA] = sc[SC_RHO] / sc[SC_D0];
            break;
        case ST_BICG_S:
            if (sqrt(sc[SC_D0]) <= sc[SC_THR]) {                                              // ||s|| satisfied
                sc[SC_DONE] = 1.0; sc[SC_CONV] = 1.0; sc[SC_FINAL_S] = 1.0;
                sc[SC_RES] = sqrt(sc[SC_D0]) / sc[SC_R0NORM];
            }
            break;
        case ST_BICG_OMEGA:
            // (t, t) = 0 (t = A s = 0 with s != 0: A singular) or a non-finite
            // omega: omega_k is undefined -> breakdown 4 (reading A20); x, r freeze
            if (sc[SC_D1] == 0.0 || !isfinite(sc[SC_D0] / sc[SC_D1])) { sc[SC_DONE] = 2.0; sc[SC_BREAK] = 4.0; break; }
            sc[SC_OMEGA] = sc[SC_D0] / sc[SC_D1];
            break;
        case ST_BICG_R:
            sc[SC_RES] = sqrt(sc[SC_D0]) / sc[SC_R0NORM];
            if (sqrt(sc[SC_D0]) <= sc[SC_THR]) { sc[SC_DONE] = 1.0; sc[SC_CONV] = 1.0; break; }   // ||r|| satisfied
            if (sc[SC_OMEGA] == 0.0) { sc[SC_DONE] = 2.0; sc[SC_BREAK] = 2.0; break; }
            sc[SC_RHO_PREV] = sc[SC_RHO];
            sc[SC_RHO] = sc[SC_D1];                                                          // rho_k = (r0, r)
            break;
        case ST_CG_ALPHA:  // counts the iteration (nothing between its start and here can stop it)
            sc[SC_ITER] += 1.0;
            // (p, q) = 0: alpha undefined (A not SPD) -> breakdown 4 (reading A20)
            if (sc[SC_D0] == 0.0 || !isfinite(sc[SC_RHO] / sc[SC_D0])) { sc[SC_DONE] = 2.0; sc[SC_BREAK] = 4.0; break; }
            sc[SC_ALPHA] = sc[SC_RHO] / sc[SC_D0];
            break;
        case ST_CG_R:
            sc[SC_RES] = sqrt(sc[SC_D0]) / sc[SC_R0NORM];
            if (sqrt(sc[SC_D0]) <= sc[SC_THR]) { sc[SC_DONE] = 1.0; sc[SC_CONV] = 1.0; break; }
            sc[SC_BETA] = sc[SC_D0] / sc[SC_RHO];
            sc[SC_RHO_PREV] = sc[SC_RHO];
            sc[SC_RHO] = sc[SC_D0];
            break;
    }
}

__global__ void step_kernel(double* sc, int mode, double tol, int first) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    step_body(sc, mode, tol, first);
}

// Local emulation of the all-reduce (hec_*_dist_local): every rank's reduced
// dots summed in rank order and written back to every rank's scalars -- one
// valid order of the sum ncclAllReduce computes across the ranks.
__global__ void local_allreduce_kernel(double* const* scs, int R, int n_dots) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int k = 0; k < n_dots; ++k) {
        double v = 0.0;
        for (int r = 0; r < R; ++r) v += scs[r][SC_D0 + k];
        for (int r = 0; r < R; ++r) scs[r][SC_D0 + k] = v;
    }
}

// The scalar step on every rank's scalars (identical inputs, identical results).
__global__ void step_all_kernel(double* const* scs, int R, int mode, double tol, int first) {
    const int r = threadIdx.x;
    if (blockIdx.x == 0 && r < R) step_body(scs[r], mode, tol, first);
}

// ------------------------------------------------------------------ host --
// The operator a solve runs on: one matrix, or this rank of a distributed one.
struct Op {
    hec_matrix_s* A = nullptr;
    hec_dist_s* D = nullptr;
    int64_t n = 0;
    ncclComm_t comm = nullptr;  // non-null: dots are all-reduced across ranks
    // local emulation (hec_*_dist_local): all R ranks on one device, this Op
    // is rank 0's; the others are solved alongside (Solver::sub)
    hec_dist_s** Dl = nullptr;
    int32_t R = 1;
};

hec_status dist_spmv_launch(hec_dist_s* D, const double* x, double* y, cudaStream_t s);   // dist.cpp
hec_status dist_local_spmv_launch(hec_dist_s** D, int32_t n, const double* const* xs, double* const* ys,
                                  cudaStream_t s);
bool dist_is_local(hec_dist_s* D);
int32_t dist_rank(hec_dist_s* D);
int64_t dist_n_local(hec_dist_s* D);
ncclComm_t dist_comm(hec_dist_s* D);
int32_t dist_parts(hec_dist_s* D);
int32_t dist_device(hec_dist_s* D);
hec_status dist_err(hec_dist_s* D);  // HEC_ERR_STATE if a peer-memory halo wait timed out
void** dist_ws_slot(hec_dist_s* D, void (***free_fn)(void*));

#define HEC_TRY(expr)                         \
    do {                                      \
        hec_status _st = (expr);              \
        if (_st != HEC_OK) return _st;        \
    } while (0)

// 128-bit element pairs need every vector the pass touches 16-byte aligned.
static bool aligned16(const VecArgs& a) {
    const void* ps[] = {a.x, a.r, a.r0, a.p, a.v, a.s, a.t, a.b, a.a1, a.b1, a.c1, a.d1};
    for (const void* p : ps)
        if (p && (reinterpret_cast<uintptr_t>(p) & 15)) return false;
    return true;
}

template <int OP>
static cudaError_t launch_vec(const VecArgs& a, cudaStream_t s) {
    vec_kernel<OP><<<kRedBlocks, kRedThreads, 0, s>>>(a);
    return cudaGetLastError();
}

static cudaError_t launch_vec_op(int op, const VecArgs& a, cudaStream_t s) {
    switch (op) {
        case OP_DOT1: return launch_vec<OP_DOT1>(a, s);
        case OP_DOT2: return launch_vec<OP_DOT2>(a, s);
        case OP_RESID: return launch_vec<OP_RESID>(a, s);
        case OP_COPY: return launch_vec<OP_COPY>(a, s);
        case OP_BICG_P: return launch_vec<OP_BICG_P>(a, s);
        case OP_BICG_S: return launch_vec<OP_BICG_S>(a, s);
        case OP_BICG_XR: return launch_vec<OP_BICG_XR>(a, s);
        case OP_X_ALPHA_P: return launch_vec<OP_X_ALPHA_P>(a, s);
        case OP_CG_XR: return launch_vec<OP_CG_XR>(a, s);
        case OP_CG_P: return launch_vec<OP_CG_P>(a, s);
        case OP_AXPBY: return launch_vec<OP_AXPBY>(a, s);
        case OP_AXPBYZ: return launch_vec<OP_AXPBYZ>(a, s);
    }
    return cudaErrorInvalidValue;
}

// Device workspace of a solve: scalars, block partials, the fused-pass
// counter, a pinned scalar mirror and 6 vectors (BiCGSTAB's r, r0, p, v, s, t;
// CG uses 4).  Cached in the matrix / dist handle by the first solve and
// reused (allocation and the implicit synchronisation of cudaFree cost ~10 ms
// per solve otherwise); a second host thread solving on the same handle at the
// same time gets a private one.
struct SolverWs {
    int64_t n = 0;
    std::mutex busy;
    double* sc = nullptr;
    double* part = nullptr;
    unsigned int* ctr = nullptr;
    double* h_sc = nullptr;
    std::vector<double*> vecs;
    hec_status alloc(int64_t n_) {
        n = n_;
        HEC_CUDA_TRY(cudaMalloc(&sc, SC_N * sizeof(double)));
        HEC_CUDA_TRY(cudaMalloc(&part, 2 * kRedBlocks * sizeof(double)));
        HEC_CUDA_TRY(cudaMalloc(&ctr, sizeof(unsigned int)));
        HEC_CUDA_TRY(cudaMallocHost(&h_sc, SC_N * sizeof(double)));
        for (int k = 0; k < 6; ++k) {
            double* v = nullptr;
            HEC_CUDA_TRY(cudaMalloc(&v, sizeof(double) * (size_t)(n > 0 ? n : 1)));
            vecs.push_back(v);
        }
        return HEC_OK;
    }
    ~SolverWs() {
        if (sc) cudaFree(sc);
        if (part) cudaFree(part);
        if (ctr) cudaFree(ctr);
        if (h_sc) cudaFreeHost(h_sc);
        for (double* v : vecs) cudaFree(v);
    }
};

static void ws_delete(void* p) { delete static_cast<SolverWs*>(p); }

struct Solver {
    Op op;
    cudaStream_t s;
    double tol = 0.0;
    double* sc = nullptr;
    double* part = nullptr;
    double* h_sc = nullptr;  // pinned mirror
    unsigned int* ctr = nullptr;  // last-CTA counter of the fused passes (self-resetting)
    std::vector<double*> vecs;
    SolverWs* ws = nullptr;
    std::unique_ptr<SolverWs> own;        // private workspace (cached one busy)
    std::unique_lock<std::mutex> lock;
    // local emulation: one sub-solver (workspace) per rank r >= 1; tab[r] maps
    // rank 0's vectors {b, x, workspace...} to rank r's, so the algorithm
    // below is written once against rank 0's pointers
    std::vector<std::unique_ptr<Solver>> sub;
    std::vector<std::vector<const double*>> tab;
    std::vector<int64_t> n_r;
    double** d_scs = nullptr;
    ~Solver() { if (d_scs) cudaFree(d_scs); }

    // rank 0 pointer -> rank r pointer (null stays null)
    const double* tr(const double* p, int r) const {
        if (!p || r == 0) return p;
        for (size_t i = 0; i < tab[0].size(); ++i)
            if (tab[0][i] == p) return tab[r][i];
        return nullptr;  // not a solver vector: a bug; the launch fails on null
    }
    hec_status init_group(const double* const* bs, double* const* xs) {
        const int R = op.R;
        tab.assign(R, {});
        n_r.assign(R, 0);
        std::vector<double*> scs(R);
        for (int r = 0; r < R; ++r) {
            Solver* S = this;
            if (r > 0) {
                sub.emplace_back(new Solver());
                S = sub.back().get();
                S->op.D = op.Dl[r];
                S->op.n = dist_n_local(op.Dl[r]);
                S->s = s;
                S->tol = tol;
                HEC_TRY(S->init());
            }
            n_r[r] = r == 0 ? op.n : S->op.n;
            tab[r].push_back(bs[r]);
            tab[r].push_back(xs[r]);
            for (double* v : S->vecs) tab[r].push_back(v);
            scs[r] = S->sc;
        }
        HEC_CUDA_TRY(cudaMalloc(&d_scs, R * sizeof(double*)));
        HEC_CUDA_TRY(cudaMemcpyAsync(d_scs, scs.data(), R * sizeof(double*), cudaMemcpyHostToDevice, s));
        return HEC_OK;
    }
    Solver* rank(int r) { return r == 0 ? this : sub[r - 1].get(); }

    hec_status init() {
        void** slot;
        void (**free_fn)(void*);
        if (op.A) { slot = &op.A->ws; free_fn = &op.A->ws_free; }
        else slot = dist_ws_slot(op.D, &free_fn);
        {
            static std::mutex create;  // first solve on a handle creates its cached workspace
            std::lock_guard<std::mutex> g(create);
            if (!*slot) {
                std::unique_ptr<SolverWs> w(new SolverWs());
                HEC_TRY(w->alloc(op.n));
                *slot = w.release();
                *free_fn = ws_delete;
            }
        }
        ws = static_cast<SolverWs*>(*slot);
        lock = std::unique_lock<std::mutex>(ws->busy, std::try_to_lock);
        if (!lock.owns_lock()) {
            own.reset(new SolverWs());
            HEC_TRY(own->alloc(op.n));
            ws = own.get();
        }
        sc = ws->sc; part = ws->part; ctr = ws->ctr; h_sc = ws->h_sc; vecs = ws->vecs;
        HEC_CUDA_TRY(cudaMemsetAsync(sc, 0, SC_N * sizeof(double), s));
        HEC_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned int), s));
        return HEC_OK;
    }
    hec_status spmv(const double* x, double* y) {
        if (op.A) return launch_spmv(op.A, x, nullptr, y, s);
        if (op.R > 1) {
            std::vector<const double*> xs(op.R);
            std::vector<double*> ys(op.R);
            for (int r = 0; r < op.R; ++r) {
                xs[r] = tr(x, r);
                ys[r] = const_cast<double*>(tr(y, r));
            }
            return dist_local_spmv_launch(op.Dl, op.R, xs.data(), ys.data(), s);
        }
        if (dist_is_local(op.D)) return dist_local_spmv_launch(&op.D, 1, &x, &y, s);
        return dist_spmv_launch(op.D, x, y, s);
    }
    // local emulation: the pass on every rank, per-rank reduce, the rank-order
    // all-reduce stand-in, then the step on every rank's scalars
    hec_status pass_group(int vop, const VecArgs& a0, int n_dots, int mode, int first) {
        for (int r = 0; r < op.R; ++r) {
            Solver* S = rank(r);
            VecArgs a = a0;
            a.x = const_cast<double*>(tr(a0.x, r)); a.r = const_cast<double*>(tr(a0.r, r));
            a.r0 = const_cast<double*>(tr(a0.r0, r)); a.p = const_cast<double*>(tr(a0.p, r));
            a.v = const_cast<double*>(tr(a0.v, r)); a.s = const_cast<double*>(tr(a0.s, r));
            a.t = const_cast<double*>(tr(a0.t, r)); a.b = const_cast<double*>(tr(a0.b, r));
            a.a1 = tr(a0.a1, r); a.b1 = tr(a0.b1, r); a.c1 = tr(a0.c1, r); a.d1 = tr(a0.d1, r);
            a.n = n_r[r];
            a.sc = S->sc;
            a.part = n_dots > 0 ? S->part : nullptr;
            a.ctr = nullptr;
            a.vec2 = aligned16(a);
            HEC_CUDA_TRY(launch_vec_op(vop, a, s));
            if (n_dots > 0) {
                reduce_kernel<<<1, kRedThreads, 0, s>>>(S->part, n_dots, S->sc);
                HEC_CUDA_TRY(cudaGetLastError());
            }
        }
        if (n_dots > 0) {
            local_allreduce_kernel<<<1, 32, 0, s>>>(d_scs, op.R, n_dots);
            HEC_CUDA_TRY(cudaGetLastError());
        }
        if (mode >= 0) HEC_TRY(step(mode, first));
        return HEC_OK;
    }
    // One vector pass; n_dots > 0: its dots land in SC_D0.. (all-reduced across
    // ranks); then the scalar step `mode` (-1: none).  One GPU: a single launch
    // (the pass's last CTA reduces and steps).  Distributed: pass, reduce,
    // ncclAllReduce, step kernel.
    hec_status pass(int vop, VecArgs a, int n_dots, int mode = -1, int first = 0) {
        if (op.R > 1) return pass_group(vop, a, n_dots, mode, first);
        a.n = op.n;
        a.sc = sc;
        a.part = n_dots > 0 ? part : nullptr;
        a.vec2 = aligned16(a);
        if (!op.comm) {
            a.ctr = (n_dots > 0 || mode >= 0) ? ctr : nullptr;
            a.n_dots = n_dots;
            a.step_mode = mode;
            a.first = first;
            a.tol = tol;
            HEC_CUDA_TRY(launch_vec_op(vop, a, s));
            return HEC_OK;
        }
        HEC_CUDA_TRY(launch_vec_op(vop, a, s));
        if (n_dots > 0) {
            reduce_kernel<<<1, kRedThreads, 0, s>>>(part, n_dots, sc);
            HEC_CUDA_TRY(cudaGetLastError());
            ncclResult_t r = ncclAllReduce(sc + SC_D0, sc + SC_D0, n_dots, ncclDouble, ncclSum, op.comm, s);
            if (r != ncclSuccess) return fail(HEC_ERR_NCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
        }
        if (mode >= 0) HEC_TRY(step(mode, first));
        return HEC_OK;
    }
    hec_status step(int mode, int first = 0) {
        if (op.R > 1) {
            step_all_kernel<<<1, 32 * ((op.R + 31) / 32), 0, s>>>(d_scs, op.R, mode, tol, first);
            HEC_CUDA_TRY(cudaGetLastError());
            return HEC_OK;
        }
        step_kernel<<<1, 32, 0, s>>>(sc, mode, tol, first);
        HEC_CUDA_TRY(cudaGetLastError());
        return HEC_OK;
    }
    hec_status read_scalars() {
        HEC_CUDA_TRY(cudaMemcpyAsync(h_sc, sc, SC_N * sizeof(double), cudaMemcpyDeviceToHost, s));
        HEC_CUDA_TRY(cudaStreamSynchronize(s));
        return HEC_OK;
    }
};

// Host loop: enqueue iterations in batches, read the device state once per batch.
template <typename Iter>
static hec_status run_batches(Solver& S, int32_t max_it, Iter enqueue_iteration, hec_solve_info* info) {
    int32_t enq = 0, batch = 4;
    HEC_TRY(S.read_scalars());
    while (S.h_sc[SC_DONE] == 0.0 && enq < max_it) {
        const int32_t nb = std::min(batch, max_it - enq);
        for (int32_t j = 0; j < nb; ++j) HEC_TRY(enqueue_iteration(enq + j + 1));
        enq += nb;
        HEC_TRY(S.read_scalars());
        batch = std::min(batch * 2, 32);
    }
    info->iterations = (int32_t)S.h_sc[SC_ITER];
    info->converged = S.h_sc[SC_CONV] != 0.0;
    info->breakdown = (int32_t)S.h_sc[SC_BREAK];
    info->rel_residual = S.h_sc[SC_RES];
    return HEC_OK;
}

// Alg. 4 with M = I: p* = p, s* = s.
static hec_status bicgstab(Solver& S, const double* b, double* x, int32_t max_it, hec_solve_info* info) {
    double *r = S.vecs[0], *r0 = S.vecs[1], *p = S.vecs[2], *v = S.vecs[3], *s = S.vecs[4], *t = S.vecs[5];
    // r0 = b - A x0 (SpMV; vector update); rho_0 = (r0, r) = ||r0||^2
    HEC_TRY(S.spmv(x, v));
    VecArgs a = {};
    a.b = const_cast<double*>(b); a.v = v; a.r = r; a.r0 = r0;
    HEC_TRY(S.pass(OP_RESID, a, 1, ST_INIT));
    auto iteration = [&](int32_t k) -> hec_status {
        HEC_TRY(S.step(ST_BICG_BEGIN, k == 1));               // rho_{k-1} = 0 -> Fails; beta_{k-1}
        VecArgs q = {};
        q.r = r; q.p = p; q.v = v;
        HEC_TRY(S.pass(k == 1 ? OP_COPY : OP_BICG_P, q, 0));  // p = r | p = r + beta (p - omega v)
        HEC_TRY(S.spmv(p, v));                                // v = A p*
        q = {}; q.a1 = r0; q.b1 = v;
        HEC_TRY(S.pass(OP_DOT1, q, 1, ST_BICG_ALPHA));        // (r0, v); alpha_k = rho_{k-1} / (r0, v)
        q = {}; q.r = r; q.v = v; q.s = s;
        HEC_TRY(S.pass(OP_BICG_S, q, 1, ST_BICG_S));          // s = r - alpha v ; ||s|| is satisfied?
        q = {}; q.x = x; q.p = p;
        HEC_TRY(S.pass(OP_X_ALPHA_P, q, 0, ST_FINAL_DONE));   //   then x = x + alpha p* ; stop
        HEC_TRY(S.spmv(s, t));                                // t = A s*
        q = {}; q.a1 = t; q.b1 = s; q.c1 = t; q.d1 = t;
        HEC_TRY(S.pass(OP_DOT2, q, 2, ST_BICG_OMEGA));        // (t, s), (t, t); omega_k = (t, s) / ||t||^2
        q = {}; q.x = x; q.p = p; q.s = s; q.t = t; q.r = r; q.r0 = r0;
        // x, r updates; ||r||^2, (r0, r); ||r|| satisfied? omega = 0? rho_k
        return S.pass(OP_BICG_XR, q, 2, ST_BICG_R);
    };
    return run_batches(S, max_it, iteration, info);
}

// Conjugate gradients ("CG ... implemented"; Saad Alg. 6.18), SPD A.
static hec_status cg(Solver& S, const double* b, double* x, int32_t max_it, hec_solve_info* info) {
    double *r = S.vecs[0], *r0 = S.vecs[1], *p = S.vecs[2], *q = S.vecs[3];
    HEC_TRY(S.spmv(x, q));
    VecArgs a = {};
    a.b = const_cast<double*>(b); a.v = q; a.r = r; a.r0 = r0;   // r = b - A x ; rho = (r, r)
    HEC_TRY(S.pass(OP_RESID, a, 1, ST_INIT));
    a = {}; a.r = r; a.p = p;                                     // p = r
    HEC_TRY(S.pass(OP_COPY, a, 0));
    auto iteration = [&](int32_t) -> hec_status {
        HEC_TRY(S.spmv(p, q));                                    // q = A p
        VecArgs c = {};
        c.a1 = p; c.b1 = q;
        HEC_TRY(S.pass(OP_DOT1, c, 1, ST_CG_ALPHA));              // (p, q); count; alpha = rho / (p, q)
        c = {}; c.x = x; c.p = p; c.r = r; c.v = q;
        HEC_TRY(S.pass(OP_CG_XR, c, 1, ST_CG_R));                 // x += alpha p; r -= alpha q; (r, r); beta
        c = {}; c.r = r; c.p = p;
        return S.pass(OP_CG_P, c, 0);                             // p = r + beta p
    };
    return run_batches(S, max_it, iteration, info);
}

static hec_status solve(Op op, int method, const double* b, double* x, double tol, int32_t max_it, void* stream,
                        hec_solve_info* info, const double* const* bs = nullptr, double* const* xs = nullptr) {
    if (!info || (op.n > 0 && (!b || !x))) return fail(HEC_ERR_ARG, "NULL argument");
    if (!(tol >= 0) || max_it < 0) return fail(HEC_ERR_ARG, "negative tol or max_it");
    std::memset(info, 0, sizeof(*info));
    DeviceGuard g(op.A ? op.A->device : dist_device(op.D));  // workspace + launches on the handle's device
    Solver S;
    S.op = op;
    S.s = (cudaStream_t)stream;
    S.tol = tol;
    HEC_TRY(S.init());
    if (op.R > 1) HEC_TRY(S.init_group(bs, xs));
    hec_status st = method == 0 ? bicgstab(S, b, x, max_it, info) : cg(S, b, x, max_it, info);
    if (st == HEC_OK) HEC_CUDA_TRY(cudaStreamSynchronize(S.s));
    // peer-memory transport: a halo wait that timed out leaves boundary rows
    // computed from stale data -- report it instead of a converged solve
    if (st == HEC_OK && op.D) st = dist_err(op.D);
    for (int r = 1; r < op.R && st == HEC_OK; ++r) st = dist_err(op.Dl[r]);
    return st;
}

static hec_status vec_op(int op, int64_t n, double ca, const double* xa, double cb, const double* xb, double* out,
                         void* stream) {
    if (n < 0) return fail(HEC_ERR_ARG, "negative length");
    if (n == 0) return HEC_OK;
    VecArgs a = {};
    a.n = n; a.ca = ca; a.cb = cb; a.a1 = xa; a.b1 = xb; a.r = out;
    a.vec2 = aligned16(a);
    HEC_CUDA_TRY(launch_vec_op(op, a, (cudaStream_t)stream));
    return HEC_OK;
}

static hec_status dot_op(int64_t n, const double* xa, const double* xb, double* result, void* stream) {
    if (n < 0 || !result) return fail(HEC_ERR_ARG, "bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    double *part = nullptr, *d = nullptr;
    HEC_CUDA_TRY(cudaMalloc(&part, 2 * kRedBlocks * sizeof(double)));
    HEC_CUDA_TRY(cudaMalloc(&d, SC_N * sizeof(double)));
    VecArgs a = {};
    a.n = n; a.a1 = xa; a.b1 = xb; a.part = part;
    a.vec2 = aligned16(a);
    cudaError_t e = launch_vec_op(OP_DOT1, a, s);
    if (e == cudaSuccess) {
        reduce_kernel<<<1, kRedThreads, 0, s>>>(part, 1, d);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(result, d + SC_D0, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(part);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "dot");
    return HEC_OK;
}

}  // namespace hec

using namespace hec;

extern "C" {

hec_status hec_axpby(int64_t n, double alpha, const double* x, double beta, double* y, void* stream) {
    if (n > 0 && (!x || !y)) return fail(HEC_ERR_ARG, "NULL vector");
    return vec_op(OP_AXPBY, n, alpha, x, beta, nullptr, y, stream);
}

hec_status hec_axpbyz(int64_t n, double alpha, const double* x, double beta, const double* y, double* z,
                      void* stream) {
    if (n > 0 && (!x || !y || !z)) return fail(HEC_ERR_ARG, "NULL vector");
    return vec_op(OP_AXPBYZ, n, alpha, x, beta, y, z, stream);
}

hec_status hec_dot(int64_t n, const double* x, const double* y, double* result, void* stream) {
    if (n > 0 && (!x || !y)) return fail(HEC_ERR_ARG, "NULL vector");
    return dot_op(n, x, y, result, stream);
}

hec_status hec_norm2(int64_t n, const double* x, double* result, void* stream) {
    if (n > 0 && !x) return fail(HEC_ERR_ARG, "NULL vector");
    hec_status st = dot_op(n, x, x, result, stream);
    if (st == HEC_OK) *result = std::sqrt(*result);
    return st;
}

hec_status hec_bicgstab(hec_matrix A, const double* b, double* x, double tol, int32_t max_it, void* stream,
                        hec_solve_info* info) {
    if (!A) return fail(HEC_ERR_ARG, "NULL matrix");
    if (A->device < 0) return fail(HEC_ERR_NODEV, "host-only matrix handle; no CPU fallback");
    if (A->n_rows != A->n_cols) return fail(HEC_ERR_DIM, "Krylov solvers need a square matrix");
    Op op;
    op.A = A;
    op.n = A->n_rows;
    return solve(op, 0, b, x, tol, max_it, stream, info);
}

hec_status hec_cg(hec_matrix A, const double* b, double* x, double tol, int32_t max_it, void* stream,
                  hec_solve_info* info) {
    if (!A) return fail(HEC_ERR_ARG, "NULL matrix");
    if (A->device < 0) return fail(HEC_ERR_NODEV, "host-only matrix handle; no CPU fallback");
    if (A->n_rows != A->n_cols) return fail(HEC_ERR_DIM, "Krylov solvers need a square matrix");
    Op op;
    op.A = A;
    op.n = A->n_rows;
    return solve(op, 1, b, x, tol, max_it, stream, info);
}

hec_status hec_bicgstab_dist(hec_dist D, const double* b_local, double* x_local, double tol, int32_t max_it,
                             void* stream, hec_solve_info* info) {
    if (!D) return fail(HEC_ERR_ARG, "NULL handle");
    Op op;
    op.D = D;
    op.n = dist_n_local(D);
    op.comm = dist_comm(D);
    if (dist_parts(D) > 1 && !op.comm)
        return fail(HEC_ERR_STATE, "distributed solvers need the NCCL communicator of hec_dist_create");
    return solve(op, 0, b_local, x_local, tol, max_it, stream, info);
}

static hec_status dist_local_solve(int method, hec_dist* D, int32_t n, const double* const* b_locals,
                                   double* const* x_locals, double tol, int32_t max_it, void* stream,
                                   hec_solve_info* info) {
    if (!D || n < 1 || !b_locals || !x_locals) return fail(HEC_ERR_ARG, "NULL argument");
    for (int32_t p = 0; p < n; ++p) {
        if (!D[p] || !dist_is_local(D[p]) || dist_parts(D[p]) != n || dist_rank(D[p]) != p)
            return fail(HEC_ERR_STATE, "handles must be the n ranks from hec_dist_create_local, in rank order");
        if (dist_n_local(D[p]) > 0 && (!b_locals[p] || !x_locals[p])) return fail(HEC_ERR_ARG, "NULL segment");
    }
    Op op;
    op.D = D[0];
    op.n = dist_n_local(D[0]);
    op.Dl = D;
    op.R = n;
    return solve(op, method, b_locals[0], x_locals[0], tol, max_it, stream, info, b_locals, x_locals);
}

hec_status hec_bicgstab_dist_local(hec_dist* D, int32_t n, const double* const* b_locals, double* const* x_locals,
                                   double tol, int32_t max_it, void* stream, hec_solve_info* info) {
    return dist_local_solve(0, D, n, b_locals, x_locals, tol, max_it, stream, info);
}

hec_status hec_cg_dist_local(hec_dist* D, int32_t n, const double* const* b_locals, double* const* x_locals,
                             double tol, int32_t max_it, void* stream, hec_solve_info* info) {
    return dist_local_solve(1, D, n, b_locals, x_locals, tol, max_it, stream, info);
}

hec_status hec_cg_dist(hec_dist D, const double* b_local, double* x_local, double tol, int32_t max_it,
                       void* stream, hec_solve_info* info) {
    if (!D) return fail(HEC_ERR_ARG, "NULL handle");
    Op op;
    op.D = D;
    op.n = dist_n_local(D);
    op.comm = dist_comm(D);
    if (dist_parts(D) > 1 && !op.comm)
        return fail(HEC_ERR_STATE, "distributed solvers need the NCCL communicator of hec_dist_create");
    return solve(op, 1, b_local, x_local, tol, max_it, stream, info);
}

}  // extern "C"
