// kernels.cu -- sm_100a kernels of the HEC SpMV hot path.
//
//   ell_kernel   Alg. 1 lines 1-3: every row's ELL part,
//                y_i = sum_{j<w, col != -1} ELLval[j*s+i] * x[ELLcol[j*s+i]].
//                Column-major slots make a warp's slot-j loads one
//                contiguous segment; each thread owns 2 adjacent rows so values
//                arrive as 128-bit (double2) and indices as 64-bit (int2)
//                loads.  The matrix streams are read once with L1::no_allocate
//                and an L2 evict_first policy so x stays cached for the gathers.
//   tail_kernel  Alg. 1 lines 5-7: the CSR remainder of the rows
//                that spill, G = 1..256 lanes per row, reduced with
//                __shfl_xor_sync (and shared memory across warps) and added
//                into the ELL result (ordered after ell_kernel).
//   coo_kernel   HYB comparison variant: the remainder as COO with atomics.
//   pack_kernel  the halo export of P:158 for the NCCL transport:
//                sendbuf[k] = x_local[send_idx[k]].
//   push_kernel / peer_wait_kernel  the peer-memory transport (export + NVLink
//                stores + epoch flags).
//   diag kernels  A_ii for the damped-Jacobi sweep (EPI_JACOBI epilogue).
//
// No tensor cores: SpMV is not a dense contraction (BASELINE.json north_star);
// the roofline is HBM bandwidth.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "hec_internal.h"

namespace hec {

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ int2 ld_stream_i2(const int32_t* ptr, uint64_t pol) {
    int2 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ double2 ld_stream_d2(const double* ptr, uint64_t pol) {
    double2 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(ptr), "l"(pol));
    return r;
}

// volatile variants: issue order pinned so every slot load of a row pair is in
// flight before the first x gather (ptxas otherwise sinks them to their use).
__device__ __forceinline__ int2 ld_stream_i2v(const int32_t* ptr, uint64_t pol) {
    int2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ double2 ld_stream_d2v(const double* ptr, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ int32_t ld_stream_i1(const int32_t* ptr, uint64_t pol) {
    int32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
                 : "=r"(r)
                 : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ double ld_stream_d1(const double* ptr, uint64_t pol) {
    double r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(r)
                 : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ int32_t ld_l1_i1(const int32_t* ptr, uint64_t pol) {
    int32_t r;
    asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ int2 ld_l1_i2(const int32_t* ptr, uint64_t pol) {
    int2 r;
    asm("ld.global.nc.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;" : "=r"(r.x), "=r"(r.y) : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ int4 ld_l1_i4(const int32_t* ptr, uint64_t pol) {
    int4 r;
    asm("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ double2 ld_l1_d2(const double* ptr, uint64_t pol) {
    double2 r;
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ double ld_l1_d1(const double* ptr, uint64_t pol) {
    double r;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ void st_stream_d2(double* ptr, double a, double b) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(ptr), "d"(a), "d"(b) : "memory");
}

__device__ __forceinline__ void st_stream_d1(double* ptr, double a) {
    asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(ptr), "d"(a) : "memory");
}

// ------------------------------------------------ peer-memory sync (PTX) --
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t global_timer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// One thread polls the arrival flags of every neighbour until they reach this
// call's epoch (ld.acquire.sys).  Runs as its own one-CTA kernel on the
// communication stream; the boundary kernel is its programmatic dependent, so
// the acquire is ordered before every halo read by griddepcontrol.wait.
// Gives up after ~10 s (sets *err; the result is then garbage and
// hec_dist_check reports it) so a missing peer cannot hang the GPU.
__device__ __forceinline__ void peer_wait(const uint64_t* flags, const int32_t* peers, int32_t n,
                                          uint64_t epoch, int32_t* err) {
    if (threadIdx.x == 0) {
        const uint64_t t0 = global_timer_ns();
        for (int32_t i = 0; i < n; ++i) {
            const uint64_t* f = flags + peers[i];
            while (ld_acquire_sys(f) < epoch) {
                if (global_timer_ns() - t0 > 10000000000ull) {
                    atomicExch(err, 1);
                    break;
                }
                __nanosleep(64);
            }
        }
    }
    __syncthreads();
}

// x gather: columns >= n_loc live in the halo buffer (distributed boundary).
// (An L2 evict_last hint on the gathers was measured: no gain, r06.)
template <bool HALO>
__device__ __forceinline__ double gather_x(const double* __restrict__ x,
                                           const double* __restrict__ xh, int32_t n_loc,
                                           int32_t c) {
    if (HALO && c >= n_loc) return __ldg(xh + (c - n_loc));
    return __ldg(x + c);
}


// ------------------------------------------------------------- ELL kernel --
// W > 0: width known at compile time (fully unrolled); W == 0: runtime width.
// EPI: the epilogue, compiled in only where it is used (keeping it out of the
// plain kernel keeps the load schedule of the hot path intact):
//   EPI_NONE    y = A x                         (hec_spmv)
//   EPI_AXPBY   y = alpha A x + beta y          (Eq. (2), hec_spmv_axpby)
//   EPI_JACOBI  y = x + omega ((b - A x) / d)   (damped Jacobi, A22, hec_jacobi)
enum { EPI_NONE = 0, EPI_AXPBY = 1, EPI_JACOBI = 2 };
#ifndef HEC_JAC_MINB
#define HEC_JAC_MINB 0  // min CTAs/SM for the Jacobi variant: 0 = compiler default (5 spills and
                        // is slower; 4 spills for w >= 12; profiles/round1/jacobi/minb_sweep.jsonl)
#endif

// One damped-Jacobi row update, each operation rounded on its own (no FMA
// contraction), in the oracle's order: r = b - s, q = r / d, x + omega q.
__device__ __forceinline__ double jacobi_row(double x, double b, double d, double omega, double s) {
    return __dadd_rn(x, __dmul_rn(omega, __ddiv_rn(__dsub_rn(b, s), d)));
}

#ifndef HEC_TAIL_UNROLL
#define HEC_TAIL_UNROLL 2  // entry-pair iterations per lane unrolled
#endif
constexpr int kTailUnroll = HEC_TAIL_UNROLL;

__device__ __forceinline__ uint32_t ld_stream_u32v(const void* ptr, uint64_t pol) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
    return r;
}

// c = *p when d is the escape code (a predicated load in straight-line PTX)
__device__ __forceinline__ void ld_if_esc(int32_t& c, int32_t d, const int32_t* p) {
    asm volatile("{\n.reg .pred e;\nsetp.eq.s32 e, %1, -32768;\n@e ld.global.nc.s32 %0, [%2];\n}"
                 : "+r"(c) : "r"(d), "l"(p));
}

// Slots [J0, J1) of a row pair: loads, then gathers, then FMAs in slot order.
// C16: the column indices come as the pair's two int16 deltas in one 32-bit
// load (EllArgs::d16); an escaped delta reads the slot's int32 column.
template <int J0, int J1, bool HALO, bool C16 = false>
__device__ __forceinline__ void ell_phase(const EllArgs& a, const int32_t* cp, const double* vp, int64_t s,
                                          uint64_t pol, double& acc0, double& acc1, int64_t i0 = 0) {
    constexpr int N = J1 - J0;
    int2 c[N];
    double2 v[N];
    if constexpr (C16) {
        uint32_t p[N];
        const int16_t* dp = a.d16 + i0;
#pragma unroll
        for (int j = 0; j < N; ++j) p[j] = ld_stream_u32v(dp + (J0 + j) * s, pol);
#pragma unroll
        for (int j = 0; j < N; ++j) v[j] = ld_stream_d2v(vp + (J0 + j) * s, pol);
        // decode; an escaped slot (a few % of a stencil's row pairs have one)
        // reads its int32 column with a predicated load -- straight-line code,
        // so the stream loads above stay ahead of every wait
        const int32_t r = a.row0 + (int32_t)i0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const int32_t d0 = (int32_t)(int16_t)(p[j] & 0xffffu), d1 = (int32_t)(int16_t)(p[j] >> 16);
            c[j].x = d0 == kIdxPad ? -1 : r + a.base[J0 + j] + d0;
            c[j].y = d1 == kIdxPad ? -1 : r + 1 + a.base[J0 + j] + d1;
            ld_if_esc(c[j].x, d0, cp + (J0 + j) * s);
            ld_if_esc(c[j].y, d1, cp + (J0 + j) * s + 1);
        }
    } else {
#pragma unroll
        for (int j = 0; j < N; ++j) c[j] = ld_stream_i2v(cp + (J0 + j) * s, pol);
#pragma unroll
        for (int j = 0; j < N; ++j) v[j] = ld_stream_d2v(vp + (J0 + j) * s, pol);
    }
    double x0[N], x1[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        x0[j] = c[j].x >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[j].x) : 0.0;
        x1[j] = c[j].y >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[j].y) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
        acc0 = fma(v[j].x, x0[j], acc0);
        acc1 = fma(v[j].y, x1[j], acc1);
    }
}

// ell_phase for slots [J0, J1) of which only [J0, wt) can hold entries (wt
// warp-uniform): the rest are neither loaded nor gathered.  A skipped slot
// adds nothing, exactly as a padding slot (col -1, +0.0) would.
template <int J0, int J1, bool HALO>
__device__ __forceinline__ void ell_phase_upto(const EllArgs& a, const int32_t* cp, const double* vp, int64_t s,
                                               uint64_t pol, double& acc0, double& acc1, int wt) {
    constexpr int N = J1 - J0;
    int2 c[N];
    double2 v[N];
#pragma unroll
    for (int j = 0; j < N; ++j) c[j] = J0 + j < wt ? ld_stream_i2v(cp + (J0 + j) * s, pol) : make_int2(-1, -1);
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = J0 + j < wt ? ld_stream_d2v(vp + (J0 + j) * s, pol) : make_double2(0.0, 0.0);
    double x0[N], x1[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        x0[j] = c[j].x >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[j].x) : 0.0;
        x1[j] = c[j].y >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[j].y) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {  // a skipped slot adds +0.0 x 0.0, as padding does
        acc0 = fma(v[j].x, x0[j], acc0);
        acc1 = fma(v[j].y, x1[j], acc1);
    }
}

// FUSE (small tails, "tail first"): the tail kernel ran just before this
// launch and stored each tail row's sum into y; this kernel is its
// programmatic dependent, so its CTAs stream their ELL rows while the tail
// finishes, and only a CTA that owns tail rows waits for it (at its very end)
// before adding the stored sum: y_i = ell_i + tail_i, the one rounding of the
// red.add path.  The CTA's tail rows: fuse_row[fuse_cta[b] .. fuse_cta[b+1]).
__device__ __forceinline__ bool fuse_has(const EllArgs& a, int32_t q0, int32_t q1, int64_t row) {
    while (q0 < q1) {  // binary search of the CTA's (ascending) tail rows
        const int32_t m = (q0 + q1) >> 1;
        const int32_t r = __ldg(a.fuse_row + m);
        if (r == row) return true;
        if (r < row) q0 = m + 1; else q1 = m;
    }
    return false;
}

template <int W, bool HALO, bool ROWMAP, int EPI, bool FUSE = false, bool C16 = false>
__global__ void __launch_bounds__(256, EPI == EPI_JACOBI ? HEC_JAC_MINB : 0) ell_kernel(EllArgs a) {
    constexpr bool AXPBY = EPI == EPI_AXPBY;
    int32_t q0 = 0, q1 = 0;
    if constexpr (FUSE) {  // loaded now, used after the ELL rows (nothing waits for it)
        q0 = __ldg(a.fuse_cta + blockIdx.x);
        q1 = __ldg(a.fuse_cta + blockIdx.x + 1);
    }
    // Programmatic dependent launch: the tail kernel may be scheduled once every
    // CTA of this grid has started (it griddepcontrol.waits for this grid's
    // completion before it touches y).  No memory clobber: nothing is ordered
    // by it, and a clobber costs the hot loop 14 registers.
    // Boundary rows under the peer-memory transport are launched as dependents
    // of peer_wait_kernel: wait for it (x_halo has landed) before letting the
    // tail kernel start or touching x_halo.  A no-op when launched normally.
    if (HALO) asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    const uint64_t pol = policy_evict_first();
    const int32_t width = W > 0 ? W : a.width;
    const int64_t s = a.stride;
    const int64_t n_pairs = ((int64_t)a.n_rows + 1) >> 1;
    for (int64_t pr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pr < n_pairs;
         pr += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = pr << 1;  // rows i0, i0+1 (i0+1 < s because s is even)
        const int32_t* cp = a.col + i0;
        const double* vp = a.val + i0;
        double acc0 = 0.0, acc1 = 0.0;
        if (W > 0) {
            // All slot loads of the row pair first (2W independent 64/128-bit
            // streams in flight), then the x gathers, then the FMAs in slot order.
            // Widths above HEC_ELL_PHASE run in two such phases (fewer live
            // registers, more resident warps).
            constexpr int WW = W > 0 ? W : 1;
            constexpr int P1 = WW > HEC_ELL_PHASE ? ell_first_phase(WW) : WW;
            // rows grouped by length: the warp's longest row (one byte per 64
            // rows, loaded beside the first phase) bounds the second phase
            const int wt = (P1 < WW && a.tile_w) ? (int)__ldg(a.tile_w + (i0 >> 6)) : WW;
            ell_phase<0, P1, HALO, C16>(a, cp, vp, s, pol, acc0, acc1, i0);
            if constexpr (P1 < WW) {
                if (wt >= WW) ell_phase<P1, WW, HALO, C16>(a, cp, vp, s, pol, acc0, acc1, i0);
                else if (wt > P1) ell_phase_upto<P1, WW, HALO>(a, cp, vp, s, pol, acc0, acc1, wt);
            }
        } else {
#pragma unroll 4
            for (int j = 0; j < width; ++j) {
                const int2 c = ld_stream_i2(cp + j * s, pol);
                const double2 v = ld_stream_d2(vp + j * s, pol);
                const double x0 = c.x >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c.x) : 0.0;
                const double x1 = c.y >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c.y) : 0.0;
                acc0 = fma(v.x, x0, acc0);
                acc1 = fma(v.y, x1, acc1);
            }
        }
        // Eq. (2) epilogue y = alpha A x + beta y (alpha = 1, beta = 0 for hec_spmv:
        // exact, and y is then never read)
        const bool two = i0 + 1 < a.n_rows;
        if (ROWMAP) {
            const int32_t g0 = __ldg(a.rowmap + i0), g1 = two ? __ldg(a.rowmap + i0 + 1) : 0;
            double* y0 = a.y + g0;
            double* y1 = two ? a.y + g1 : nullptr;
            if (EPI == EPI_JACOBI) {  // grouped rows of a square matrix: x, b, d indexed by the output row
                acc0 = jacobi_row(__ldg(a.x + g0), __ldg(a.b + g0), __ldg(a.diag + g0), a.omega, acc0);
                if (two) acc1 = jacobi_row(__ldg(a.x + g1), __ldg(a.b + g1), __ldg(a.diag + g1), a.omega, acc1);
            }
            if (AXPBY && a.beta != 0.0) {
                acc0 = a.alpha * acc0 + a.beta * *y0;
                if (two) acc1 = a.alpha * acc1 + a.beta * *y1;
            } else if (AXPBY) {
                acc0 *= a.alpha;
                acc1 *= a.alpha;
            }
            st_stream_d1(y0, acc0);
            if (two) st_stream_d1(y1, acc1);
        } else {
            double* yp = a.y + a.row_off + i0;
            if (EPI == EPI_JACOBI) {  // square single matrix: x, b, d indexed like y
                const int64_t g = a.row_off + i0;
                const double *xg = a.x + g, *bg = a.b + g, *dg = a.diag + g;
                if (two && (((uintptr_t)xg | (uintptr_t)bg | (uintptr_t)dg) & 15) == 0) {
                    // b and d are streamed once (evict-first); x_i was just gathered (L1/L2)
                    const double2 bb = ld_stream_d2v(bg, pol), dd = ld_stream_d2v(dg, pol);
                    const double2 xx = __ldg(reinterpret_cast<const double2*>(xg));
                    acc0 = jacobi_row(xx.x, bb.x, dd.x, a.omega, acc0);
                    acc1 = jacobi_row(xx.y, bb.y, dd.y, a.omega, acc1);
                } else {
                    acc0 = jacobi_row(__ldg(xg), __ldg(bg), __ldg(dg), a.omega, acc0);
                    if (two) acc1 = jacobi_row(__ldg(xg + 1), __ldg(bg + 1), __ldg(dg + 1), a.omega, acc1);
                }
            }
            if (AXPBY && a.beta != 0.0) {
                acc0 = a.alpha * acc0 + a.beta * yp[0];
                if (two) acc1 = a.alpha * acc1 + a.beta * yp[1];
            } else if (AXPBY) {
                acc0 *= a.alpha;
                acc1 *= a.alpha;
            }
            if constexpr (FUSE) {
                if (q1 > q0) {
                    const bool t0 = fuse_has(a, q0, q1, i0), t1 = two && fuse_has(a, q0, q1, i0 + 1);
                    if (t0 || t1) {
                        asm volatile("griddepcontrol.wait;" ::: "memory");  // the tail kernel's stores
                        if (t0) acc0 = acc0 + __ldcg(yp);
                        if (t1) acc1 = acc1 + __ldcg(yp + 1);
                    }
                }
            }
            if (two && ((reinterpret_cast<uintptr_t>(yp) & 15) == 0)) {
                st_stream_d2(yp, acc0, acc1);
            } else {
                st_stream_d1(yp, acc0);
                if (two) st_stream_d1(yp + 1, acc1);
            }
        }
    }
}

// ------------------------------------------------------------ tail kernel --
// The CSR part (Alg. 1 lines 5-7) for the rows that spill.  Rows
// are regrouped by length inside super-blocks of consecutive tail rows
// (plan_chunks, api.cpp): a CUDA block takes 256/G rows that all use G = 2^lg
// lanes (G ~ spilled length / entries-per-lane target, 8 for big tails and 2
// for small ones, capped at 256; longer rows loop).  The G lanes of a row read its contiguous entries, gather
// x, reduce with __shfl_xor_sync and the first lane adds the row sum into the
// ELL result (this kernel runs after ell_kernel on the same stream).
// Blocks of one super-block run back to back, so its entries and the x window
// they touch are reused in L2.  Fixed reduction order: deterministic.
// One block descriptor's work for the 256 threads tid = 0..255 of the CTA.

// Tail loop variants (measured on power-law 2^23, profiles/round2/tailvar/): 0 = one pair per
// iteration, unroll 2 (323 us at 8 entries per lane); 3 = value loads predicated on a real index
// (fewer bytes, slower: 344 us); 4 = each lane issues the index + value loads of HEC_TAIL_BATCH
// iterations before any gather (batch 8 at 6 CTAs/SM and 32 entries per lane: 262 us)
#ifndef HEC_TAIL_V
#define HEC_TAIL_V 4
#endif
#ifndef HEC_TAIL_BATCH
#define HEC_TAIL_BATCH 8  // HEC_TAIL_V 4: iterations whose loads are issued together
#endif
#ifndef HEC_TAIL_NOVAL
#define HEC_TAIL_NOVAL 0
#endif

// ---- value stream through the bulk-copy engine (HEC_TAIL_V 5) ----
// The tail is bound by the L1 sector throughput of its loads (ncu: ~82% of
// peak; dropping the value stream cuts the sectors 112 M -> 90 M and the time
// 249 -> 202 us, profiles/round2/l1probe): so each warp copies its batch of
// values (B iterations x 64 entries, contiguous in the warp-chunk layout) into
// its own shared-memory buffer with one cp.async.bulk completing on the
// warp's mbarrier, while the lanes load the indices and gather x through the
// LSU as before; the values are read from shared memory after the wait.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_val(double* dst, const double* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the lanes' reads of the last batch came first
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra.uni W_%=;\n}\n" ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}

// One warp's pairs in the warp-chunk layout (hec_internal.h): wm = {first
// entry, iterations, ...}; lane l reads the pair at base + 64 i + 2 l.  Returns
// the lane's partial sum (its row's entries 2 (i G + lr), +1 in order).
template <bool HALO>
__device__ __forceinline__ double warp_chunk_sum(const TailArgs& a, int4 wm, int l, uint64_t pol) {
    double acc = 0.0;
    const int tid = l;  // only tid & 31 is used below
    {
        // every warp-wide load is one whole 256-byte (index) / 512-byte (value)
        // segment, read once: streamed past L1 with the L2 evict-first policy,
        // so L1 and L2 keep the x gathers.  Padding (-1, +0.0) reads no x and
        // adds nothing (also for lanes of absent rows: all their pairs pad).
        const int32_t k0 = wm.x + 2 * (tid & 31), k1 = k0 + kTailChunk * wm.y;
#if HEC_TAIL_V == 4
        // all of the lane's index and value loads first (<= HEC_TAIL_BATCH
        // iterations per batch), then the gathers, then the FMAs in order
        constexpr int B = HALO ? (HEC_TAIL_BATCH + 1) / 2 : HEC_TAIL_BATCH;  // the halo select costs registers
        for (int32_t kb = k0; kb < k1; kb += B * kTailChunk) {
            int2 c[B];
            double2 v[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int32_t k = kb + u * kTailChunk;
                c[u] = k < k1 ? ld_stream_i2(a.col + k, pol) : make_int2(-1, -1);
#if HEC_TAIL_NOVAL  // EXPERIMENT ONLY (wrong results): no value stream, to size the L1 sector cost
                v[u] = make_double2(1.0, 1.0);
#else
                v[u] = k < k1 ? ld_stream_d2(a.val + k, pol) : make_double2(0.0, 0.0);
#endif
            }
            double xs[2 * B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                xs[2 * u] = c[u].x >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[u].x) : 0.0;
                xs[2 * u + 1] = c[u].y >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[u].y) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
                if (c[u].x >= 0) acc = fma(v[u].x, xs[2 * u], acc);
                if (c[u].y >= 0) acc = fma(v[u].y, xs[2 * u + 1], acc);
            }
        }
#else
#pragma unroll kTailUnroll
        for (int32_t k = k0; k < k1; k += kTailChunk) {
            const int2 c = ld_stream_i2(a.col + k, pol);
#if HEC_TAIL_V == 3
            // padding pairs (c.x < 0) read no value bytes
            const double2 v = c.x >= 0 ? ld_stream_d2(a.val + k, pol) : make_double2(0.0, 0.0);
#else
            const double2 v = ld_stream_d2(a.val + k, pol);
#endif
            const double x0 = c.x >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c.x) : 0.0;
            const double x1 = c.y >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c.y) : 0.0;
            if (c.x >= 0) acc = fma(v.x, x0, acc);
            if (c.y >= 0) acc = fma(v.y, x1, acc);
        }
#endif
    }
    return acc;
}

// HEC_TAIL_V 5: warp_chunk_sum with the values staged by the bulk-copy engine
// into sv (B x 64 doubles, this warp's) on mbarrier bar; phase counts the
// warp's batches so far (the mbarrier's parity).
template <bool HALO>
__device__ __forceinline__ double warp_chunk_sum_tma(const TailArgs& a, int4 wm, int l, uint64_t pol, double* sv,
                                                     uint64_t* bar, uint32_t& phase) {
    constexpr int B = HALO ? (HEC_TAIL_BATCH + 1) / 2 : HEC_TAIL_BATCH;
    double acc = 0.0;
    const int32_t w0 = wm.x, w1 = wm.x + kTailChunk * wm.y;  // the warp's entries
    for (int32_t kw = w0; kw < w1; kw += B * kTailChunk) {
        const int32_t nb = min(B * kTailChunk, w1 - kw);      // entries in this batch (a multiple of 64)
        __syncwarp();                                          // every lane is done with sv
        if (l == 0) bulk_val(sv, a.val + kw, (uint32_t)nb * 8u, bar, pol);
        int2 c[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int32_t k = kw + u * kTailChunk + 2 * l;
            c[u] = u * kTailChunk < nb ? ld_stream_i2(a.col + k, pol) : make_int2(-1, -1);
        }
        double xs[2 * B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            xs[2 * u] = c[u].x >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[u].x) : 0.0;
            xs[2 * u + 1] = c[u].y >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[u].y) : 0.0;
        }
        mbar_wait_parity(bar, phase & 1u);
        ++phase;
        // a padding entry has x = 0 (no gather) and value +0.0: its FMA adds
        // +0.0 to a sum that is never -0.0 (it starts at +0.0), i.e. nothing --
        // so no predicate (and no live indices) is needed here
#pragma unroll
        for (int u = 0; u < B; ++u) {
            if (u * kTailChunk < nb) {
                const double2 v = *reinterpret_cast<const double2*>(sv + u * kTailChunk + 2 * l);
                acc = fma(v.x, xs[2 * u], acc);
                acc = fma(v.y, xs[2 * u + 1], acc);
            }
        }
    }
    return acc;
}

template <bool HALO, bool JACOBI>
__device__ __forceinline__ void tail_desc(const TailArgs& a, int64_t desc, int tid, uint64_t pol, double* wsum,
                                          double* sv = nullptr, uint64_t* bar = nullptr) {
    // one load per warp: {first entry, iterations, first row, count << 8 | lg}
    // (warp-chunk layout, hec_internal.h) -- no dependent metadata loads
    // before the stream starts
    const int4 wm = __ldg(a.warp + desc * kTailWarps + (tid >> 5));
    const int lg = wm.w & 255;
    const int G = 1 << lg;
    const int lane = tid & (G - 1);
    const int grp = tid >> lg;
    double* yp = nullptr;
    int32_t orow = 0;
    const bool active = grp < (wm.w >> 8);
    if (active && lane == 0) {
        orow = __ldg(a.out_rows + wm.z + grp);
        yp = a.y + orow;
    }
    double acc;
    if (sv) {
        uint32_t phase = 0;
        acc = warp_chunk_sum_tma<HALO>(a, wm, tid & 31, pol, sv, bar, phase);
    } else {
        acc = warp_chunk_sum<HALO>(a, wm, tid & 31, pol);
    }
    if (lg <= 5) {
        for (int off = G >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off, G);
    } else {
        // a row spans G / 32 warps: full-warp shuffle, then the row's first
        // warp adds the warps' partials in warp order (deterministic)
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if ((tid & 31) == 0) wsum[tid >> 5] = acc;
        __syncthreads();
        if (lane == 0) {
            const int w0 = tid >> 5, nw = G >> 5;
            acc = wsum[w0];
            for (int w = 1; w < nw; ++w) acc += wsum[w0 + w];
        }
    }
    // The row's one addition into the ELL result, y_i = ell_i + tail_i, as a
    // fire-and-forget reduction at L2 (red.global.add.f64): no load of y, so
    // the CTA retires without another memory round trip.  Each row has exactly
    // one tail sum and the ELL kernel has finished, so the result is the same
    // single rounded addition as a load-add-store (y - q == y + (-q) in IEEE).
    double q = 0.0;
    if (lane == 0 && active)  // the ELL kernel wrote x + omega ((b - s_ell) / d): add -omega (s_tail / d)
        q = JACOBI ? -__dmul_rn(a.omega, __ddiv_rn(acc, __ldg(a.diag + orow))) : __dmul_rn(a.alpha, acc);
    // y holds the ELL result: with programmatic dependent launch this kernel may
    // have started before ell_kernel finished, so wait for it here (a no-op
    // when launched normally or once it has returned)
    if (a.store_only) {  // small tails first (the ELL kernel adds it) / concurrent tail (combined later)
        if (lane == 0 && active) {
            if (a.tsum) a.tsum[wm.z + grp] = q;
            else *yp = q;
        }
        return;
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (lane == 0 && active) asm volatile("red.global.add.f64 [%0], %1;" ::"l"(yp), "d"(q) : "memory");
}

#ifndef HEC_TAIL_MINB
#define HEC_TAIL_MINB (48 / kTailWarps)  // CTAs per SM: 48 warps leave the batched loads 40 registers (64 warps: 32 regs, 275 us; 32 warps: 277 us)
#endif

template <bool HALO, bool JACOBI>
__global__ void __launch_bounds__(kTailThreads, HEC_TAIL_MINB) tail_kernel(TailArgs a) {
    __shared__ double wsum[kTailWarps];  // per-warp partials of rows wider than a warp
    // store_only: the ELL kernel is this grid's programmatic dependent -- let
    // it start streaming right away (it waits for these stores where it needs them)
    if (a.store_only) asm volatile("griddepcontrol.launch_dependents;");
    const uint64_t pol = policy_evict_first();
#if HEC_TAIL_V == 5
    constexpr int B = HALO ? (HEC_TAIL_BATCH + 1) / 2 : HEC_TAIL_BATCH;
    __shared__ __align__(128) double sval[kTailWarps][B * kTailChunk];  // per warp: one batch of values
    __shared__ __align__(8) uint64_t sbar[kTailWarps];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) mbar_init1(&sbar[w]);
    __syncwarp();
    tail_desc<HALO, JACOBI>(a, a.reverse ? a.blk_end - 1 - blockIdx.x : a.blk_begin + blockIdx.x, threadIdx.x, pol,
                            wsum, sval[w], &sbar[w]);
#else
    // reverse: the descriptors from the last to the first, so the first CTAs
    // gather the x band (and red.add into the y lines) the ELL kernel's last
    // CTAs just left in L2
    tail_desc<HALO, JACOBI>(a, a.reverse ? a.blk_end - 1 - blockIdx.x : a.blk_begin + blockIdx.x, threadIdx.x, pol,
                            wsum);
#endif
}

// SM-local persistent schedule, warp by warp (whole-matrix launches of big
// tails; opt-in HEC_TAIL_WARP=1): the tail's WARP UNITS (one warp-chunk warp
// of rows with G <= 32 lanes; or all G/32 warps of one row with G > 32, which
// the warp then walks one after the other) are cut into one contiguous region
// per SM, and each resident warp claims the next unit of its SM's region
// through a counter (the next claim issued before the current unit's work) --
// so the warps sharing an SM's L1 gather from neighbouring rows' x window, with
// no barrier between units.  A warp that runs out of its SM's work steals from
// the next regions: every unit is claimed exactly once whatever the placement;
// the last warp to finish resets the counters.  Same lanes, partial sums,
// reduction order and one red.add per row as tail_kernel: bitwise equal.
__device__ __forceinline__ uint32_t sm_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

// One warp unit: wm0 = the unit's first warp meta (carried in the unit list,
// so no dependent metadata load); its index in the warp-meta array is read
// for the row-in-descriptor and, for rows over several warps, the next metas.
template <bool HALO, bool JACOBI>
__device__ __forceinline__ void tail_unit(const TailArgs& a, int4 wm0, int64_t u, int l, uint64_t pol) {
    const int lg = wm0.w & 255, G = 1 << lg;
    const int32_t widx = __ldg(a.unit_widx + u);
    const int grp = (((widx & (kTailWarps - 1)) << 5) + l) >> lg;  // the lane's row within its descriptor
    double acc;
    if (G <= 32) {
        acc = warp_chunk_sum<HALO>(a, wm0, l, pol);
        for (int off = G >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off, G);
    } else {  // one row over G / 32 warps: each a full-warp tree, added in warp order
        acc = 0.0;
        for (int j = 0; j < (G >> 5); ++j) {
            double p = warp_chunk_sum<HALO>(a, j == 0 ? wm0 : __ldg(a.warp + widx + j), l, pol);
            for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
            acc = j == 0 ? p : acc + p;
        }
    }
    const bool lead = (l & (G - 1)) == 0 && grp < (wm0.w >> 8);
    if (lead) {
        const int32_t orow = __ldg(a.out_rows + wm0.z + grp);
        const double q = JACOBI ? -__dmul_rn(a.omega, __ddiv_rn(acc, __ldg(a.diag + orow))) : __dmul_rn(a.alpha, acc);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(a.y + orow), "d"(q) : "memory");
    }
}

// A region's units, claimed two ahead: while unit i runs, the claim for i + 2
// is in flight and unit i + 1's meta (claimed an iteration ago) is loading.
template <bool HALO, bool JACOBI>
__device__ __forceinline__ void tail_region(const TailArgs& a, int r, int l, uint64_t pol) {
    const int64_t r0 = __ldg(a.region + r), r1 = __ldg(a.region + r + 1);
    unsigned int c0 = 0, c1 = 0;
    if (l == 0) {
        c0 = atomicAdd(a.region_ctr + r, 1u);
        c1 = atomicAdd(a.region_ctr + r, 1u);
    }
    int64_t u = r0 + __shfl_sync(0xffffffffu, c0, 0);
    if (u >= r1) return;
    int4 wm = __ldg(a.units + u);
    int64_t un = r0 + __shfl_sync(0xffffffffu, c1, 0);
    while (true) {
        unsigned int c2 = 0;
        if (l == 0 && un < r1) c2 = atomicAdd(a.region_ctr + r, 1u);
        const int4 wn = un < r1 ? __ldg(a.units + un) : make_int4(0, 0, 0, 0);
        tail_unit<HALO, JACOBI>(a, wm, u, l, pol);
        if (un >= r1) break;
        u = un;
        wm = wn;
        un = r0 + __shfl_sync(0xffffffffu, c2, 0);
    }
}

template <bool HALO, bool JACOBI>
__global__ void __launch_bounds__(kTailThreads, HEC_TAIL_MINB) tail_warp_kernel(TailArgs a) {
    const uint64_t pol = policy_evict_first();
    const int l = threadIdx.x & 31;
    const int R = a.n_regions;
    const int home = (int)(sm_id() % (uint32_t)R);
    tail_region<HALO, JACOBI>(a, home, l, pol);
    // then steal: the lanes read every region's counter at once (one round
    // trip per 32 regions, starting after home) and the warp joins the first
    // region with work left; done when none has any
    while (true) {
        int found = -1;
        for (int base = 1; base < R && found < 0; base += 32) {
            const int k = base + l;
            const int r = home + k < R ? home + k : home + k - R;
            bool has = false;
            if (k < R)
                has = __ldg(a.region + r) + (int64_t)*(volatile const unsigned int*)(a.region_ctr + r) <
                      __ldg(a.region + r + 1);
            const unsigned int m = __ballot_sync(0xffffffffu, has);
            if (m) {
                const int kk = base + __ffs(m) - 1;
                found = home + kk < R ? home + kk : home + kk - R;
            }
        }
        if (found < 0) break;
        tail_region<HALO, JACOBI>(a, found, l, pol);
    }
    if (l == 0) {
        __threadfence();
        if (atomicAdd(a.region_done, 1u) == gridDim.x * (blockDim.x >> 5) - 1) {
            for (int r = 0; r < R; ++r) a.region_ctr[r] = 0;
            __threadfence();
            *a.region_done = 0;
        }
    }
}

// ------------------------------------------------------ x-ring tail kernel --
// The tail is bound by the L1 wavefronts of its x gathers (one 128-byte line
// per lane: ncu ~82% of the L1 throughput), and most of its columns
// sit in a band around the row (power-law: 90% within +-4,096).  So one CTA
// per SM walks a contiguous run of warp units (plan_ring, api.cpp) stage by
// stage, and the x columns a stage mostly reads, [lo, hi), are staged into a
// shared-memory ring of kRingCols columns by the bulk-copy engine: a
// producer warp copies only each stage's NEW columns (the windows slide
// along the rows), two stages ahead of their use (full/empty mbarriers, no
// CTA-wide barrier), and the consumer warps gather in-window columns from
// shared memory, the rest from global memory.  Same lanes, partial sums,
// reduction order and one red.add per row as tail_kernel: bitwise equal.
#ifndef HEC_RING_BATCH
#define HEC_RING_BATCH 4  // iterations whose loads a lane issues together (8 spills at 31 warps)
#endif
template <bool HALO>
__device__ __forceinline__ double warp_chunk_sum_ring(const TailArgs& a, int4 wm, int l, uint64_t pol,
                                                      const double* ring, int32_t lo, uint32_t span) {
    double acc = 0.0;
    constexpr int B = HALO ? (HEC_RING_BATCH + 1) / 2 : HEC_RING_BATCH;
    const int32_t k0 = wm.x + 2 * l, k1 = k0 + kTailChunk * wm.y;
    for (int32_t kb = k0; kb < k1; kb += B * kTailChunk) {
        int2 c[B];
        double2 v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int32_t k = kb + u * kTailChunk;
            c[u] = k < k1 ? ld_stream_i2(a.col + k, pol) : make_int2(-1, -1);
            v[u] = k < k1 ? ld_stream_d2(a.val + k, pol) : make_double2(0.0, 0.0);
        }
        double xs[2 * B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            // in the window: the ring slot (the window lies inside [0, n_loc));
            // padding (-1) reads nothing
            xs[2 * u] = (uint32_t)(c[u].x - lo) < span ? ring[c[u].x & (kRingCols - 1)]
                        : c[u].x >= 0                ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[u].x)
                                                     : 0.0;
            xs[2 * u + 1] = (uint32_t)(c[u].y - lo) < span ? ring[c[u].y & (kRingCols - 1)]
                            : c[u].y >= 0                ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[u].y)
                                                         : 0.0;
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            if (c[u].x >= 0) acc = fma(v[u].x, xs[2 * u], acc);
            if (c[u].y >= 0) acc = fma(v[u].y, xs[2 * u + 1], acc);
        }
    }
    return acc;
}

template <bool HALO, bool JACOBI>
__device__ __forceinline__ void tail_ring_unit(const TailArgs& a, int4 un, int l, uint64_t pol, const double* ring,
                                               int32_t lo, uint32_t span) {
    const int4 wm0 = __ldg(a.warp + un.x);
    const int lg = wm0.w & 255, G = 1 << lg;
    const int grp = ((un.z << 5) + l) >> lg;  // the lane's row within its descriptor
    double acc;
    if (G <= 32) {
        acc = warp_chunk_sum_ring<HALO>(a, wm0, l, pol, ring, lo, span);
        for (int off = G >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off, G);
    } else {  // one row over G / 32 warps: each a full-warp tree, added in warp order
        acc = 0.0;
        for (int j = 0; j < un.y; ++j) {
            double p = warp_chunk_sum_ring<HALO>(a, j == 0 ? wm0 : __ldg(a.warp + un.x + j), l, pol, ring, lo, span);
            for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
            acc = j == 0 ? p : acc + p;
        }
    }
    if ((l & (G - 1)) == 0 && grp < (wm0.w >> 8)) {
        const int32_t orow = __ldg(a.out_rows + wm0.z + grp);
        const double q = JACOBI ? -__dmul_rn(a.omega, __ddiv_rn(acc, __ldg(a.diag + orow))) : __dmul_rn(a.alpha, acc);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(a.y + orow), "d"(q) : "memory");
    }
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

#ifndef HEC_RING_NW
#define HEC_RING_NW 31  // consumer warps per ring CTA (one CTA per SM; measured 16/24/31: 380/447/269 us)
#endif

template <bool HALO, bool JACOBI>
__global__ void __launch_bounds__((HEC_RING_NW + 1) * 32, 1) tail_ring_kernel(TailArgs a) {
    extern __shared__ __align__(128) double ring[];  // kRingCols columns
    constexpr int NW = HEC_RING_NW, D = kRingDepth;
    __shared__ __align__(8) uint64_t full[D], empty[D];
    __shared__ uint32_t claim[D];  // per stage slot: the next unit to claim
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int32_t s0 = __ldg(a.ring_cta + blockIdx.x), s1 = __ldg(a.ring_cta + blockIdx.x + 1);
    if (threadIdx.x == 0) {
        for (int d = 0; d < D; ++d) {
            mbar_init(&full[d], 1);
            mbar_init(&empty[d], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (w == NW) {  // producer: lane 0 copies each stage's new columns
        if (l != 0) return;
        int32_t loaded = INT32_MIN;
        for (int32_t s = s0; s < s1; ++s) {
            const int k = s - s0, d = k % D;
            const int4 st = __ldg(a.ring_stage + s);
            // stage s's new columns overwrite only columns of stages <= s - D
            // (plan_ring: hi_s - lo_(s-D+1) <= kRingCols), and slot d's claim
            // counter is free once stage s - D is done
            if (k >= D) mbar_wait_parity(&empty[d], ((k - D) / D) & 1);
            claim[d] = 0;
            const int32_t c0 = max(loaded, st.x), c1 = st.y;
            if (c1 > c0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // consumers' reads came first
                asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                             ::"r"(smem_addr(&full[d])), "r"((uint32_t)(c1 - c0) * 8u) : "memory");
                const int32_t p0 = c0 & (kRingCols - 1);
                const int32_t n0 = min(c1 - c0, kRingCols - p0);
                bulk_g2s(ring + p0, a.x + c0, (uint32_t)n0 * 8u, &full[d]);
                if (c1 - c0 > n0) bulk_g2s(ring, a.x + c0 + n0, (uint32_t)(c1 - c0 - n0) * 8u, &full[d]);
                loaded = c1;
            } else {
                mbar_arrive(&full[d]);
            }
        }
        return;
    }
    const uint64_t pol = policy_evict_first();
    for (int32_t s = s0; s < s1; ++s) {
        const int k = s - s0, d = k % D;
        const int4 st = __ldg(a.ring_stage + s);
        mbar_wait_parity(&full[d], (k / D) & 1);
        const uint32_t span = (uint32_t)(st.y - st.x);
        // units claimed one at a time, the biggest first (a super-block's
        // units are sorted by ascending row length), so the stage's last
        // units are small ones and the warps finish together
        while (true) {
            uint32_t c = 0;
            if (l == 0) c = atomicAdd(&claim[d], 1u);
            c = __shfl_sync(0xffffffffu, c, 0);
            if ((int32_t)c >= st.w - st.z) break;
            tail_ring_unit<HALO, JACOBI>(a, __ldg(a.ring_unit + st.w - 1 - (int32_t)c), l, pol, ring, st.x, span);
        }
        __syncwarp();
        if (l == 0) mbar_arrive(&empty[d]);
    }
}

// ------------------------------------------------------- HYB: COO kernel --
// Comparison variant: the Bell-Garland HYB remainder in
// COO instead of CSR.  Lane l of a warp owns 8 consecutive row-sorted
// entries (vector loads), sums each run of equal rows, and adds every run into
// y with an fp64 atomic (rows may span lanes and warps; the addition order of
// those partial sums is not fixed -- parity is within tolerance, exact only in
// the integer regime).
__device__ __forceinline__ double coo_part(const CooArgs& a, int32_t row, double acc) {
    return a.diag ? -__dmul_rn(a.omega, __ddiv_rn(acc, __ldg(a.diag + row))) : a.alpha * acc;
}

__global__ void __launch_bounds__(256) coo_kernel(CooArgs a) {
    const int64_t k0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (k0 >= a.nnz) return;
    const int n = a.nnz - k0 < 8 ? (int)(a.nnz - k0) : 8;
    int32_t row[8], col[8];
    double val[8];
    if (n == 8) {  // k0 is a multiple of 8: 32-byte aligned int4 / double2 loads
        const int4 r0 = __ldg(reinterpret_cast<const int4*>(a.row + k0));
        const int4 r1 = __ldg(reinterpret_cast<const int4*>(a.row + k0) + 1);
        const int4 c0 = __ldg(reinterpret_cast<const int4*>(a.col + k0));
        const int4 c1 = __ldg(reinterpret_cast<const int4*>(a.col + k0) + 1);
        row[0] = r0.x; row[1] = r0.y; row[2] = r0.z; row[3] = r0.w;
        row[4] = r1.x; row[5] = r1.y; row[6] = r1.z; row[7] = r1.w;
        col[0] = c0.x; col[1] = c0.y; col[2] = c0.z; col[3] = c0.w;
        col[4] = c1.x; col[5] = c1.y; col[6] = c1.z; col[7] = c1.w;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(a.val + k0) + j);
            val[2 * j] = v.x;
            val[2 * j + 1] = v.y;
        }
    } else {
        for (int j = 0; j < 8; ++j) {
            row[j] = j < n ? __ldg(a.row + k0 + j) : -1;
            col[j] = j < n ? __ldg(a.col + k0 + j) : 0;
            val[j] = j < n ? __ldg(a.val + k0 + j) : 0.0;
        }
    }
    double xg[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) xg[j] = j < n ? __ldg(a.x + col[j]) : 0.0;
    double acc = 0.0;
    int32_t cur = row[0];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (j < n) {
            if (row[j] != cur) {
                atomicAdd(a.y + cur, coo_part(a, cur, acc));
                acc = 0.0;
                cur = row[j];
            }
            acc = fma(val[j], xg[j], acc);
        }
    }
    atomicAdd(a.y + cur, coo_part(a, cur, acc));
}

cudaError_t launch_coo(const CooArgs& a, cudaStream_t s) {
    if (a.nnz <= 0) return cudaSuccess;
    const int64_t threads = (a.nnz + 7) / 8;
    const int64_t blocks = (threads + 255) / 256;
    coo_kernel<<<(unsigned)blocks, 256, 0, s>>>(a);
    return cudaGetLastError();
}

// ------------------------------------------------------------ pack kernel --
__global__ void __launch_bounds__(256) pack_kernel(const int32_t* __restrict__ idx, int32_t n,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ out) {
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        out[k] = __ldg(x + __ldg(idx + k));
}

// --------------------------------------------------------------- launchers --
static int g_num_sms = 0;

static int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

// Kernel launch through cudaLaunchKernelEx.  (An L2 persisting access-policy
// window on x was measured, r09: slower for every config; not used.)
// pdl = programmatic dependent launch: the kernel may start while the previous
// kernel on the stream drains (it must griddepcontrol.wait before consuming).
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kernel)(KArgs...), dim3 g, dim3 b, cudaStream_t s, bool pdl, size_t smem,
                            Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

static bool tail_pdl() {
    static int v = -1;
    if (v < 0) {
        // default on (measured q3: SPE10 0.0279 -> 0.0237 ms, no change elsewhere);
        // HEC_PDL=0 launches the tail kernel plainly
        const char* e = std::getenv("HEC_PDL");
        v = (e && std::atoi(e) == 0) ? 0 : 1;
    }
    return v == 1;
}

// ELL CTA size: 128 threads for single-phase widths (w <= HEC_ELL_PHASE), 256
// for the two-phase ones (measured, profiles/round1/ell_block/: 256^3 0.2467 ->
// 0.2448 ms, 128^3 0.0349 -> 0.0346, SPE10 0.0223 -> 0.0219 with 128; power-law
// w = 9 0.503 -> 0.519 ms with 128, so it keeps 256).  HEC_ELL_BLOCK (tuning)
// forces 64/128/192/256 for every width.
static int ell_block(int32_t width) {
    static int forced = -1;
    if (forced < 0) {
        const char* e = std::getenv("HEC_ELL_BLOCK");
        const int b = e ? std::atoi(e) : 0;
        forced = (b == 64 || b == 128 || b == 192 || b == 256) ? b : 0;
    }
    if (forced) return forced;
    return (width > 0 && width <= HEC_ELL_PHASE) ? 128 : 256;
}

int ell_block_threads(int32_t width) { return ell_block(width); }
int64_t ell_grid_cap() { return (int64_t)num_sms() * 8 * 64; }

template <bool HALO, bool ROWMAP, int EPI, bool FUSE, bool C16>
static cudaError_t launch_ell_t2(const EllArgs& a, cudaStream_t s) {
    const int64_t n_pairs = ((int64_t)a.n_rows + 1) >> 1;
    const int threads = ell_block(a.width);
    int64_t blocks = (n_pairs + threads - 1) / threads;
    // one row pair per thread, grid-stride only beyond 64 full waves (a
    // persistent grid of 5-40 blocks/SM was measured slower, r15; forcing
    // >= 6 CTAs/SM by a 40-register cap too, pdl run)
    int64_t cap = ell_grid_cap();
    if (FUSE && (blocks > cap || 2 * threads * blocks < a.n_rows)) return cudaErrorInvalidValue;  // planned per tile
    static int per_sm = -1;  // HEC_ELL_CAP (tuning): at most this many CTAs per SM, grid-stride beyond
    if (per_sm < 0) {
        const char* e = std::getenv("HEC_ELL_CAP");
        per_sm = e ? std::max(0, std::atoi(e)) : 0;
    }
    if (per_sm > 0 && !FUSE) cap = std::min<int64_t>(cap, (int64_t)num_sms() * per_sm);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const dim3 g((unsigned)blocks), b(threads);
    switch (a.width) {
#define HEC_W(w) \
    case w: return launch_k(ell_kernel<w, HALO, ROWMAP, EPI, FUSE, C16>, g, b, s, a.pdl, 0, a);
        HEC_W(1) HEC_W(2) HEC_W(3) HEC_W(4) HEC_W(5) HEC_W(6) HEC_W(7) HEC_W(8)
        HEC_W(9) HEC_W(10) HEC_W(11) HEC_W(12) HEC_W(13) HEC_W(14) HEC_W(15) HEC_W(16)
#undef HEC_W
        default:
            if constexpr (C16) return cudaErrorInvalidValue;  // compressed indices need a compiled width
            else return launch_k(ell_kernel<0, HALO, ROWMAP, EPI, FUSE>, g, b, s, a.pdl, 0, a);
    }
}

template <bool HALO, bool ROWMAP, int EPI, bool FUSE = false>
static cudaError_t launch_ell_t(const EllArgs& a, cudaStream_t s) {
    if (a.d16 && a.width >= 1 && a.width <= kIdx16MaxW) return launch_ell_t2<HALO, ROWMAP, EPI, FUSE, true>(a, s);
    return launch_ell_t2<HALO, ROWMAP, EPI, FUSE, false>(a, s);
}

// ELL kernel choice: "reg" (register-streaming ell_kernel) or "tma" (bulk-copy
// pipeline, ell_tma.cu).  HEC_ELL_KERNEL overrides the default (tuning only).
static int ell_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("HEC_ELL_KERNEL");
        v = (e && std::strcmp(e, "tma") == 0) ? 1 : 0;
    }
    return v;
}

cudaError_t launch_ell(const EllArgs& a, cudaStream_t s) {
    if (a.n_rows <= 0) return cudaSuccess;
    if (ell_variant() == 1 && a.alpha == 1.0 && a.beta == 0.0 && !a.diag && !a.fuse_cta) {
        cudaError_t e = launch_ell_tma(a, s, num_sms());
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();  // clear the sticky-free "not supported" status
    }
    const bool halo = a.x_halo != nullptr;
    const bool rowmap = a.rowmap != nullptr;
    // (single square matrices: no halo; a row map only for rows grouped by length)
    if (a.diag) {  // hec_jacobi
        if (halo) return cudaErrorInvalidValue;
        return rowmap ? launch_ell_t<false, true, EPI_JACOBI>(a, s) : launch_ell_t<false, false, EPI_JACOBI>(a, s);
    }
    if (a.alpha != 1.0 || a.beta != 0.0) {  // hec_spmv_axpby
        if (halo) return cudaErrorInvalidValue;
        return rowmap ? launch_ell_t<false, true, EPI_AXPBY>(a, s) : launch_ell_t<false, false, EPI_AXPBY>(a, s);
    }
    if (a.fuse_cta) {  // plain whole-matrix product with its small tail fused in
        if (halo || rowmap) return cudaErrorInvalidValue;
        return launch_ell_t<false, false, EPI_NONE, true>(a, s);
    }
    if (halo) return rowmap ? launch_ell_t<true, true, EPI_NONE>(a, s) : launch_ell_t<true, false, EPI_NONE>(a, s);
    return rowmap ? launch_ell_t<false, true, EPI_NONE>(a, s) : launch_ell_t<false, false, EPI_NONE>(a, s);
}

cudaError_t launch_tail(const TailArgs& a, cudaStream_t s) {
    const int64_t blocks = a.blk_end - a.blk_begin;
    if (blocks <= 0) return cudaSuccess;
    if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
    const bool pdl = tail_pdl() && !a.store_only;  // store_only runs first: an ordinary launch
    if (a.diag && a.x_halo) return cudaErrorInvalidValue;
    if (a.store_only && (a.diag || a.x_halo || a.alpha != 1.0)) return cudaErrorInvalidValue;
    if (a.ring_stage && !a.store_only && a.ring_ctas > 0 && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0) {
        // x-ring schedule: one CTA per SM, the ring in dynamic shared memory
        const size_t smem = sizeof(double) * kRingCols;
        static bool attr[3] = {false, false, false};
        auto go = [&](auto kern, int which) {
            if (!attr[which]) {
                cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess) return e;
                attr[which] = true;
            }
            return launch_k(kern, dim3((unsigned)a.ring_ctas), dim3((HEC_RING_NW + 1) * 32), s, pdl, smem, a);
        };
        if (a.diag) return go(tail_ring_kernel<false, true>, 0);
        if (a.x_halo) return go(tail_ring_kernel<true, false>, 1);
        return go(tail_ring_kernel<false, false>, 2);
    }
    if (a.region && !a.store_only) {  // SM-local persistent schedule, warp by warp: 6 CTAs per SM
        const int64_t g = std::min<int64_t>(blocks, (int64_t)num_sms() * HEC_TAIL_MINB);
        if (a.diag) return launch_k(tail_warp_kernel<false, true>, dim3((unsigned)g), dim3(kTailThreads), s, pdl, 0, a);
        if (a.x_halo) return launch_k(tail_warp_kernel<true, false>, dim3((unsigned)g), dim3(kTailThreads), s, pdl, 0, a);
        return launch_k(tail_warp_kernel<false, false>, dim3((unsigned)g), dim3(kTailThreads), s, pdl, 0, a);
    }
    if (a.diag) return launch_k(tail_kernel<false, true>, dim3((unsigned)blocks), dim3(kTailThreads), s, pdl, 0, a);
    if (a.x_halo) return launch_k(tail_kernel<true, false>, dim3((unsigned)blocks), dim3(kTailThreads), s, pdl, 0, a);
    return launch_k(tail_kernel<false, false>, dim3((unsigned)blocks), dim3(kTailThreads), s, pdl, 0, a);
}

// Concurrent tail: y[out_rows[p]] += tsum[p] once the ELL kernel and the
// store-only tail kernel (on a second stream) have both finished -- the single
// rounded addition y_i = ell_i + tail_i of the red.add path, bitwise.
__global__ void __launch_bounds__(256) tail_combine_kernel(const int32_t* __restrict__ out_rows,
                                                           const double* __restrict__ tsum, int32_t n,
                                                           double* __restrict__ y) {
    for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        double* yr = y + __ldg(out_rows + p);
        *yr = *yr + __ldg(tsum + p);
    }
}

cudaError_t launch_tail_combine(const int32_t* out_rows, const double* tsum, int32_t n, double* y, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int blocks = (n + 255) / 256;
    if (blocks > num_sms() * 8) blocks = num_sms() * 8;
    tail_combine_kernel<<<blocks, 256, 0, s>>>(out_rows, tsum, n, y);
    return cudaGetLastError();
}

cudaError_t launch_pack(const int32_t* idx, int32_t n, const double* x, double* out,
                        cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int blocks = (n + 255) / 256;
    if (blocks > num_sms() * 8) blocks = num_sms() * 8;
    pack_kernel<<<blocks, 256, 0, s>>>(idx, n, x, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------ diagonal --
// d[i] = A_ii (A22), setup-time: the ELL slots of row i, then (stream order)
// the tail rows, which overwrite only where the diagonal spilled.
__global__ void __launch_bounds__(256) diag_ell_kernel(const int32_t* __restrict__ col,
                                                       const double* __restrict__ val, int64_t stride,
                                                       int32_t width, int32_t n, const int32_t* __restrict__ perm,
                                                       double* __restrict__ d) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = perm ? perm[i] : (int32_t)i;  // the row stored at position i
        double v = 0.0;
        for (int32_t j = 0; j < width; ++j)
            if (col[j * stride + i] == r) v = val[j * stride + i];
        d[r] = v;
    }
}

// The tail's diagonal entries in the warp-chunk layout: one CTA per
// descriptor, each lane scans its pairs; at most one entry per row matches,
// so every d[row] has a single writer (after diag_ell_kernel, stream order).
__global__ void __launch_bounds__(kTailThreads) diag_tail_kernel(TailArgs a, double* __restrict__ d) {
    const int tid = threadIdx.x;
    const int4 wm = __ldg(a.warp + (int64_t)blockIdx.x * kTailWarps + (tid >> 5));
    const int grp = tid >> (wm.w & 255);
    if (grp >= (wm.w >> 8)) return;
    const int32_t r = __ldg(a.out_rows + wm.z + grp);
    for (int32_t i = 0; i < wm.y; ++i) {
        const int64_t k = wm.x + (int64_t)kTailChunk * i + 2 * (tid & 31);
        if (a.col[k] == r) d[r] = a.val[k];
        if (a.col[k + 1] == r) d[r] = a.val[k + 1];
    }
}

__global__ void __launch_bounds__(256) diag_coo_kernel(const int32_t* __restrict__ row,
                                                       const int32_t* __restrict__ col,
                                                       const double* __restrict__ val, int64_t nnz,
                                                       double* __restrict__ d) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        if (row[k] == col[k]) d[row[k]] = val[k];
}

// ------------------------------------------------ peer-memory halo push --
// The export of P:158 fused with the transfer: each CTA takes kPushChunk send
// entries of one destination rank, gathers x_local[send_idx[k]] and stores
// them straight into that rank's halo buffer (this call's parity) through its
// IPC mapping over NVLink -- no staging buffer, no copy engine, no NCCL
// kernel.  Each CTA then fences at system scope and counts itself done; the
// last CTA releases this call's epoch into every neighbour's arrival flag
// (st.release.sys).  Neighbours
// with nothing to receive still get the flag: it tells them this rank has
// finished reading its own halo buffer of the previous call.
__global__ void __launch_bounds__(256) push_kernel(PushArgs a) {
    if ((int32_t)blockIdx.x < a.n_chunks) {
        const int4 c = __ldg(a.chunks + blockIdx.x);  // {q, k0, k1, halo position of k0 at q}
        double* dst = a.peer_buf0[c.x] + ((a.epoch & 1) ? a.peer_nhalo[c.x] : 0) + c.w - c.y;
#pragma unroll 8
        for (int32_t k = c.y + threadIdx.x; k < c.z; k += blockDim.x) dst[k] = __ldg(a.x + __ldg(a.idx + k));
    }
    // every CTA's stores, then one system-scope fence per CTA (after the
    // barrier, as in a grid-wide sync); the last CTA releases the epoch
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned int prev = atomicAdd(a.done, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence_system();
            for (int32_t i = 0; i < a.n_nbr; ++i) {
                const int32_t q = a.nbr[i];
                st_release_sys(a.peer_flags[q] + a.rank, a.epoch);
            }
            *a.done = 0;  // the next call's push is stream-ordered after this one
        }
    }
}

__global__ void peer_wait_kernel(PeerWait w) { peer_wait(w.flags, w.peers, w.n, w.epoch, w.err); }

cudaError_t launch_push(const PushArgs& a, cudaStream_t s) {
    if (a.n_nbr <= 0) return cudaSuccess;
    const int blocks = a.n_chunks > 0 ? a.n_chunks : 1;  // >= 1: the flags go out even with no data
    push_kernel<<<blocks, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_peer_wait(const PeerWait& w, cudaStream_t s) {
    if (w.n <= 0) return cudaSuccess;
    peer_wait_kernel<<<1, 32, 0, s>>>(w);
    return cudaGetLastError();
}

cudaError_t launch_diag(const hec_matrix_s* A, double* d, cudaStream_t s) {
    if (A->n_rows <= 0) return cudaSuccess;
    const int cap = num_sms() * 8;
    auto grid = [cap](int64_t n) { int64_t g = (n + 255) / 256; return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g)); };
    diag_ell_kernel<<<grid(A->n_rows), 256, 0, s>>>(A->d_ell_col, A->d_ell_val, A->stride,
                                                    A->d_ell_col ? A->width : 0, A->n_rows, A->d_ell_perm, d);
    if (A->tail_rows > 0 && A->tail_coo)
        diag_coo_kernel<<<grid(A->tail_nnz), 256, 0, s>>>(A->d_coo_row, A->d_tail_col, A->d_tail_val, A->tail_nnz, d);
    else if (A->tail_rows > 0 && !A->h_tail_blk.empty()) {
        TailArgs t = {};
        t.blk = A->d_tail_blk;
        t.warp = A->d_tail_warp;
        t.out_rows = A->d_tail_out;
        t.col = A->d_tail_col;
        t.val = A->d_tail_val;
        diag_tail_kernel<<<(unsigned)A->h_tail_blk.size(), kTailThreads, 0, s>>>(t, d);
    }
    return cudaGetLastError();
}

}  // namespace hec
