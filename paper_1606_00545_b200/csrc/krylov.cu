// krylov.cu -- the consumers of the SpMV hot path:
// the vector operations of PAPER.md §2.3 (Eqs. (2)-(6)), the
// unpreconditioned BiCGSTAB of Alg. 4 (M = I) and CG ("implemented",
// P:294), on one GPU (hec_matrix) or row-partitioned (hec_dist).
//
// Design: one stream, no host round trip for the scalars.  Fused vector passes
// (grid-stride, fixed grid) write per-block partial dot products; a one-block
// kernel sums them in a fixed order (deterministic) into a small device scalar
// array; in distributed mode an ncclAllReduce over those few doubles replaces
// the paper's "sub results are sent back to CPU"; a one-thread kernel
// derives alpha / beta / omega.  The host reads two norms per iteration for the
// stopping tests of Alg. 4 (lines "||s|| is satisfied", "||r|| is satisfied").
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "hec_internal.h"

struct hec_dist_s;  // dist.cpp

namespace hec {

// scalar slots
enum {
    SC_RHO = 0, SC_RHO_PREV, SC_ALPHA, SC_OMEGA, SC_BETA,
    SC_D0, SC_D1, SC_D2,  // reduced dot products of the last pass
    SC_R0NORM2, SC_N
};

enum VecOp {
    OP_DOT1,      // d0 = (a, b)
    OP_DOT2,      // d0 = (a, b), d1 = (c, d)
    OP_RESID,     // r = b - v ; r0 = r ; d0 = (r, r)
    OP_COPY,      // p = r
    OP_BICG_P,    // p = r + beta (p - omega v)
    OP_BICG_S,    // s = r - alpha v ; d0 = (s, s)
    OP_BICG_XR,   // x = x + alpha p + omega s ; r = s - omega t ; d0 = (r, r) ; d1 = (r0, r)
    OP_X_ALPHA_P, // x = x + alpha p
    OP_CG_XR,     // x = x + alpha p ; r = r - alpha q ; d0 = (r, r)
    OP_CG_P,      // p = r + beta p
    OP_AXPBY,     // y = alpha_in x + beta_in y            (Eq. 3)
    OP_AXPBYZ,    // z = alpha_in x + beta_in y            (Eq. 4)
};

struct VecArgs {
    int op;
    int64_t n;
    const double* sc;   // device scalars (alpha, beta, omega read from here)
    double* part;       // [3][kRedBlocks] partial dots
    double ca, cb;      // host-given coefficients (OP_AXPBY / OP_AXPBYZ)
    // operands (meaning per op, see VecOp)
    double *x, *r, *r0, *p, *v, *s, *t, *b;
    const double *a1, *b1, *c1, *d1;
};

constexpr int kRedBlocks = 592;   // 4 x 148: fixed grid => fixed summation order
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

__global__ void __launch_bounds__(kRedThreads) vec_kernel(VecArgs a) {
    __shared__ double sh[3][32];
    double d0 = 0.0, d1 = 0.0;
    const double alpha = a.sc ? a.sc[SC_ALPHA] : 0.0;
    const double omega = a.sc ? a.sc[SC_OMEGA] : 0.0;
    const double beta = a.sc ? a.sc[SC_BETA] : 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
        switch (a.op) {
            case OP_DOT1: d0 += a.a1[i] * a.b1[i]; break;
            case OP_DOT2: d0 += a.a1[i] * a.b1[i]; d1 += a.c1[i] * a.d1[i]; break;
            case OP_RESID: {
                const double ri = a.b[i] - a.v[i];
                a.r[i] = ri; a.r0[i] = ri; d0 += ri * ri; break;
            }
            case OP_COPY: a.p[i] = a.r[i]; break;
            case OP_BICG_P: a.p[i] = a.r[i] + beta * (a.p[i] - omega * a.v[i]); break;
            case OP_BICG_S: {
                const double si = a.r[i] - alpha * a.v[i];
                a.s[i] = si; d0 += si * si; break;
            }
            case OP_BICG_XR: {
                const double si = a.s[i];
                a.x[i] = a.x[i] + alpha * a.p[i] + omega * si;
                const double ri = si - omega * a.t[i];
                a.r[i] = ri; d0 += ri * ri; d1 += a.r0[i] * ri; break;
            }
            case OP_X_ALPHA_P: a.x[i] = a.x[i] + alpha * a.p[i]; break;
            case OP_CG_XR: {
                a.x[i] = a.x[i] + alpha * a.p[i];
                const double ri = a.r[i] - alpha * a.v[i];
                a.r[i] = ri; d0 += ri * ri; break;
            }
            case OP_CG_P: a.p[i] = a.r[i] + beta * a.p[i]; break;
            case OP_AXPBY: a.r[i] = a.ca * a.a1[i] + a.cb * a.r[i]; break;
            case OP_AXPBYZ: a.r[i] = a.ca * a.a1[i] + a.cb * a.b1[i]; break;
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
}

// Sum the per-block partials in a fixed order: sc[dst + k] = sum_b part[k][b].
__global__ void __launch_bounds__(kRedThreads) reduce_kernel(const double* part, int n_parts, double* sc, int dst) {
    __shared__ double sh[32];
    for (int k = 0; k < n_parts; ++k) {
        double v = 0.0;
        for (int b = threadIdx.x; b < kRedBlocks; b += blockDim.x) v += part[k * kRedBlocks + b];
        v = block_sum(v, sh);
        if (threadIdx.x == 0) sc[dst + k] = v;
    }
}

enum Derive { DV_ALPHA_BICG, DV_OMEGA, DV_BETA_BICG, DV_ALPHA_CG, DV_BETA_CG, DV_RHO_FROM_D1, DV_SET_RHO_D0 };

__global__ void derive_kernel(double* sc, int mode) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    switch (mode) {
        case DV_ALPHA_BICG: sc[SC_ALPHA] = sc[SC_RHO] / sc[SC_D0]; break;          // alpha = rho/(r0, v)
        case DV_OMEGA: sc[SC_OMEGA] = sc[SC_D0] / sc[SC_D1]; break;                 // omega = (t,s)/(t,t)
        case DV_BETA_BICG:                                                          // beta = (rho/rho_prev)(alpha/omega)
            sc[SC_BETA] = (sc[SC_RHO] / sc[SC_RHO_PREV]) * (sc[SC_ALPHA] / sc[SC_OMEGA]); break;
        case DV_ALPHA_CG: sc[SC_ALPHA] = sc[SC_RHO] / sc[SC_D0]; break;            // alpha = (r,r)/(p,q)
        case DV_BETA_CG: sc[SC_BETA] = sc[SC_D0] / sc[SC_RHO]; sc[SC_RHO_PREV] = sc[SC_RHO]; sc[SC_RHO] = sc[SC_D0]; break;
        case DV_RHO_FROM_D1: sc[SC_RHO_PREV] = sc[SC_RHO]; sc[SC_RHO] = sc[SC_D1]; break;
        case DV_SET_RHO_D0: sc[SC_RHO] = sc[SC_D0]; sc[SC_R0NORM2] = sc[SC_D0]; break;
    }
}

// ------------------------------------------------------------------ host --
// The operator a solve runs on: one matrix, or this rank of a distributed one.
struct Op {
    hec_matrix_s* A = nullptr;
    hec_dist_s* D = nullptr;
    int64_t n = 0;
    ncclComm_t comm = nullptr;  // non-null: dots are all-reduced across ranks
};

hec_status dist_spmv_launch(hec_dist_s* D, const double* x, double* y, cudaStream_t s);   // dist.cpp
int64_t dist_n_local(hec_dist_s* D);
ncclComm_t dist_comm(hec_dist_s* D);

struct Solver {
    Op op;
    cudaStream_t s;
    double* sc = nullptr;
    double* part = nullptr;
    double* h_sc = nullptr;  // pinned mirror
    std::vector<double*> vecs;

    hec_status init(int n_vecs) {
        HEC_CUDA_TRY(cudaMalloc(&sc, SC_N * sizeof(double)));
        HEC_CUDA_TRY(cudaMemsetAsync(sc, 0, SC_N * sizeof(double), s));
        HEC_CUDA_TRY(cudaMalloc(&part, 3 * kRedBlocks * sizeof(double)));
        HEC_CUDA_TRY(cudaMallocHost(&h_sc, SC_N * sizeof(double)));
        for (int k = 0; k < n_vecs; ++k) {
            double* v = nullptr;
            HEC_CUDA_TRY(cudaMalloc(&v, sizeof(double) * (size_t)(op.n > 0 ? op.n : 1)));
            vecs.push_back(v);
        }
        return HEC_OK;
    }
    ~Solver() {
        if (sc) cudaFree(sc);
        if (part) cudaFree(part);
        if (h_sc) cudaFreeHost(h_sc);
        for (double* v : vecs) cudaFree(v);
    }
    hec_status spmv(const double* x, double* y) {
        if (op.A) return launch_spmv(op.A, x, nullptr, y, s);
        return dist_spmv_launch(op.D, x, y, s);
    }
    // run a fused vector pass; n_dots > 0: reduce its dots into SC_D0.. (all-reduced across ranks)
    hec_status pass(VecArgs a, int n_dots) {
        a.n = op.n;
        a.sc = sc;
        a.part = n_dots > 0 ? part : nullptr;
        vec_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(a);
        HEC_CUDA_TRY(cudaGetLastError());
        if (n_dots > 0) {
            reduce_kernel<<<1, kRedThreads, 0, s>>>(part, n_dots, sc, SC_D0);
            HEC_CUDA_TRY(cudaGetLastError());
            if (op.comm) {
                ncclResult_t r = ncclAllReduce(sc + SC_D0, sc + SC_D0, n_dots, ncclDouble, ncclSum, op.comm, s);
                if (r != ncclSuccess) return fail(HEC_ERR_NCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
            }
        }
        return HEC_OK;
    }
    hec_status derive(int mode) {
        derive_kernel<<<1, 32, 0, s>>>(sc, mode);
        HEC_CUDA_TRY(cudaGetLastError());
        return HEC_OK;
    }
    hec_status read_scalars() {
        HEC_CUDA_TRY(cudaMemcpyAsync(h_sc, sc, SC_N * sizeof(double), cudaMemcpyDeviceToHost, s));
        HEC_CUDA_TRY(cudaStreamSynchronize(s));
        return HEC_OK;
    }
};

#define HEC_TRY(expr)                         \
    do {                                      \
        hec_status _st = (expr);              \
        if (_st != HEC_OK) return _st;        \
    } while (0)

// Alg. 4 with M = I: p* = p, s* = s.
static hec_status bicgstab(Solver& S, const double* b, double* x, double tol, int32_t max_it,
                           hec_solve_info* info) {
    double *r = S.vecs[0], *r0 = S.vecs[1], *p = S.vecs[2], *v = S.vecs[3], *s = S.vecs[4], *t = S.vecs[5];
    info->iterations = 0;
    info->converged = 0;
    info->breakdown = 0;
    // r0 = b - A x0 (SpMV; vector update); rho_0 = (r0, r) = ||r0||^2
    HEC_TRY(S.spmv(x, v));
    VecArgs a = {};
    a.op = OP_RESID; a.b = const_cast<double*>(b); a.v = v; a.r = r; a.r0 = r0;
    HEC_TRY(S.pass(a, 1));
    HEC_TRY(S.derive(DV_SET_RHO_D0));
    HEC_TRY(S.read_scalars());
    const double r0n = std::sqrt(S.h_sc[SC_R0NORM2]);
    const double thr = tol * r0n;
    info->rel_residual = r0n > 0 ? 1.0 : 0.0;
    if (r0n == 0.0) { info->converged = 1; return HEC_OK; }
    for (int32_t k = 1; k <= max_it; ++k) {
        info->iterations = k;
        // rho_{k-1} = (r0, r) is in SC_RHO (from the previous pass)
        if (S.h_sc[SC_RHO] == 0.0) { info->breakdown = 1; return HEC_OK; }         // "Fails"
        if (k == 1) {
            a = {}; a.op = OP_COPY; a.r = r; a.p = p;                               // p = r
            HEC_TRY(S.pass(a, 0));
        } else {
            HEC_TRY(S.derive(DV_BETA_BICG));                                        // beta_{k-1}
            a = {}; a.op = OP_BICG_P; a.r = r; a.p = p; a.v = v;                    // p = r + beta (p - omega v)
            HEC_TRY(S.pass(a, 0));
        }
        HEC_TRY(S.spmv(p, v));                                                      // v = A p
        a = {}; a.op = OP_DOT1; a.a1 = r0; a.b1 = v;                                // (r0, v)
        HEC_TRY(S.pass(a, 1));
        HEC_TRY(S.derive(DV_ALPHA_BICG));                                           // alpha = rho / (r0, v)
        a = {}; a.op = OP_BICG_S; a.r = r; a.v = v; a.s = s;                        // s = r - alpha v ; ||s||^2
        HEC_TRY(S.pass(a, 1));
        HEC_TRY(S.read_scalars());
        if (S.h_sc[SC_D0 + 0] != S.h_sc[SC_D0 + 0] || !std::isfinite(S.h_sc[SC_ALPHA])) {
            info->breakdown = 3;                                                    // (r0, v) = 0 (reading A20)
            return HEC_OK;
        }
        if (std::sqrt(S.h_sc[SC_D0]) <= thr) {                                     // ||s|| is satisfied
            a = {}; a.op = OP_X_ALPHA_P; a.x = x; a.p = p;                          // x = x + alpha p
            HEC_TRY(S.pass(a, 0));
            HEC_CUDA_TRY(cudaStreamSynchronize(S.s));
            info->converged = 1;
            info->rel_residual = std::sqrt(S.h_sc[SC_D0]) / r0n;
            return HEC_OK;
        }
        HEC_TRY(S.spmv(s, t));                                                      // t = A s
        a = {}; a.op = OP_DOT2; a.a1 = t; a.b1 = s; a.c1 = t; a.d1 = t;             // (t, s), (t, t)
        HEC_TRY(S.pass(a, 2));
        HEC_TRY(S.derive(DV_OMEGA));                                                // omega = (t,s)/||t||^2
        a = {}; a.op = OP_BICG_XR; a.x = x; a.p = p; a.s = s; a.t = t; a.r = r; a.r0 = r0;
        HEC_TRY(S.pass(a, 2));                                                      // x, r updates; ||r||^2, (r0, r)
        HEC_TRY(S.derive(DV_RHO_FROM_D1));                                          // rho_k = (r0, r) for the next k
        HEC_TRY(S.read_scalars());
        info->rel_residual = std::sqrt(S.h_sc[SC_D0]) / r0n;
        if (std::sqrt(S.h_sc[SC_D0]) <= thr) { info->converged = 1; return HEC_OK; }   // ||r|| satisfied
        if (S.h_sc[SC_OMEGA] == 0.0) { info->breakdown = 2; return HEC_OK; }           // omega_k = 0
    }
    return HEC_OK;
}

// Conjugate gradients ("CG ... implemented"; Saad Alg. 6.18), SPD A.
static hec_status cg(Solver& S, const double* b, double* x, double tol, int32_t max_it, hec_solve_info* info) {
    double *r = S.vecs[0], *r0 = S.vecs[1], *p = S.vecs[2], *q = S.vecs[3];
    info->iterations = 0;
    info->converged = 0;
    info->breakdown = 0;
    HEC_TRY(S.spmv(x, q));
    VecArgs a = {};
    a.op = OP_RESID; a.b = const_cast<double*>(b); a.v = q; a.r = r; a.r0 = r0;  // r = b - A x ; rho = (r, r)
    HEC_TRY(S.pass(a, 1));
    HEC_TRY(S.derive(DV_SET_RHO_D0));
    a = {}; a.op = OP_COPY; a.r = r; a.p = p;                                     // p = r
    HEC_TRY(S.pass(a, 0));
    HEC_TRY(S.read_scalars());
    const double r0n = std::sqrt(S.h_sc[SC_R0NORM2]);
    const double thr = tol * r0n;
    info->rel_residual = r0n > 0 ? 1.0 : 0.0;
    if (r0n == 0.0) { info->converged = 1; return HEC_OK; }
    for (int32_t k = 1; k <= max_it; ++k) {
        info->iterations = k;
        HEC_TRY(S.spmv(p, q));                                                    // q = A p
        a = {}; a.op = OP_DOT1; a.a1 = p; a.b1 = q;                               // (p, q)
        HEC_TRY(S.pass(a, 1));
        HEC_TRY(S.derive(DV_ALPHA_CG));                                           // alpha = rho / (p, q)
        a = {}; a.op = OP_CG_XR; a.x = x; a.p = p; a.r = r; a.v = q;              // x += alpha p; r -= alpha q; (r,r)
        HEC_TRY(S.pass(a, 1));
        HEC_TRY(S.derive(DV_BETA_CG));                                            // beta = (r,r)_new / rho; rho = new
        HEC_TRY(S.read_scalars());
        info->rel_residual = std::sqrt(S.h_sc[SC_RHO]) / r0n;
        if (std::sqrt(S.h_sc[SC_RHO]) <= thr) { info->converged = 1; return HEC_OK; }
        a = {}; a.op = OP_CG_P; a.r = r; a.p = p;                                 // p = r + beta p
        HEC_TRY(S.pass(a, 0));
    }
    return HEC_OK;
}

static hec_status solve(Op op, int method, const double* b, double* x, double tol, int32_t max_it, void* stream,
                        hec_solve_info* info) {
    if (!info || (op.n > 0 && (!b || !x))) return fail(HEC_ERR_ARG, "NULL argument");
    if (tol < 0 || max_it < 0) return fail(HEC_ERR_ARG, "negative tol or max_it");
    Solver S;
    S.op = op;
    S.s = (cudaStream_t)stream;
    HEC_TRY(S.init(method == 0 ? 6 : 4));
    if (method == 0) return bicgstab(S, b, x, tol, max_it, info);
    return cg(S, b, x, tol, max_it, info);
}

static hec_status vec_op(int op, int64_t n, double ca, const double* xa, double cb, const double* xb, double* out,
                         void* stream) {
    if (n < 0) return fail(HEC_ERR_ARG, "negative length");
    if (n == 0) return HEC_OK;
    VecArgs a = {};
    a.op = op; a.n = n; a.ca = ca; a.cb = cb; a.a1 = xa; a.b1 = xb; a.r = out;
    vec_kernel<<<kRedBlocks, kRedThreads, 0, (cudaStream_t)stream>>>(a);
    HEC_CUDA_TRY(cudaGetLastError());
    return HEC_OK;
}

static hec_status dot_op(int64_t n, const double* xa, const double* xb, double* result, void* stream) {
    if (n < 0 || !result) return fail(HEC_ERR_ARG, "bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    double *part = nullptr, *d = nullptr;
    HEC_CUDA_TRY(cudaMalloc(&part, 2 * kRedBlocks * sizeof(double)));
    HEC_CUDA_TRY(cudaMalloc(&d, sizeof(double)));
    VecArgs a = {};
    a.op = OP_DOT1; a.n = n; a.a1 = xa; a.b1 = xb; a.part = part;
    vec_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(a);
    reduce_kernel<<<1, kRedThreads, 0, s>>>(part, 1, d, 0);
    cudaError_t e = cudaMemcpyAsync(result, d, sizeof(double), cudaMemcpyDeviceToHost, s);
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
    return solve(op, 0, b_local, x_local, tol, max_it, stream, info);
}

hec_status hec_cg_dist(hec_dist D, const double* b_local, double* x_local, double tol, int32_t max_it,
                       void* stream, hec_solve_info* info) {
    if (!D) return fail(HEC_ERR_ARG, "NULL handle");
    Op op;
    op.D = D;
    op.n = dist_n_local(D);
    op.comm = dist_comm(D);
    return solve(op, 1, b_local, x_local, tol, max_it, stream, info);
}

}  // extern "C"
