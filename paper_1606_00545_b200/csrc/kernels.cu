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
//                that spill, G lanes per row, reduced with __shfl_xor_sync and
//                added into the ELL result (ordered after ell_kernel).
//   pack_kernel  the halo export of P:158: sendbuf[k] = x_local[send_idx[k]].
//
// No tensor cores: SpMV is not a dense contraction (BASELINE.json north_star);
// the roofline is HBM bandwidth.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

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

__device__ __forceinline__ void st_stream_d2(double* ptr, double a, double b) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(ptr), "d"(a), "d"(b) : "memory");
}

__device__ __forceinline__ void st_stream_d1(double* ptr, double a) {
    asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(ptr), "d"(a) : "memory");
}

// x gather: columns >= n_loc live in the halo buffer (distributed boundary).
__device__ __forceinline__ double ld_keep_d1(const double* ptr, uint64_t pol) {
    double r;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// x gather: columns >= n_loc live in the halo buffer (distributed boundary).
// __constant__ flag (tuning experiment): 1 = gathers carry an L2 evict_last hint.
__constant__ int c_x_keep = 0;

template <bool HALO>
__device__ __forceinline__ double gather_x(const double* __restrict__ x,
                                           const double* __restrict__ xh, int32_t n_loc,
                                           int32_t c) {
    const double* p = (HALO && c >= n_loc) ? xh + (c - n_loc) : x + c;
    if (c_x_keep) return ld_keep_d1(p, policy_evict_last());
    return __ldg(p);
}

// ------------------------------------------------------------- ELL kernel --
// W > 0: width known at compile time (fully unrolled); W == 0: runtime width.
template <int W, bool HALO, bool ROWMAP>
__global__ void __launch_bounds__(256) ell_kernel(EllArgs a) {
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
            constexpr int WW = W > 0 ? W : 1;
            int2 c[WW];
            double2 v[WW];
#pragma unroll
            for (int j = 0; j < WW; ++j) c[j] = ld_stream_i2v(cp + j * s, pol);
#pragma unroll
            for (int j = 0; j < WW; ++j) v[j] = ld_stream_d2v(vp + j * s, pol);
            double x0[WW], x1[WW];
#pragma unroll
            for (int j = 0; j < WW; ++j) {
                x0[j] = c[j].x >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[j].x) : 0.0;
                x1[j] = c[j].y >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[j].y) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < WW; ++j) {
                acc0 = fma(v[j].x, x0[j], acc0);
                acc1 = fma(v[j].y, x1[j], acc1);
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
        if (ROWMAP) {
            st_stream_d1(a.y + a.rowmap[i0], acc0);
            if (i0 + 1 < a.n_rows) st_stream_d1(a.y + a.rowmap[i0 + 1], acc1);
        } else {
            double* yp = a.y + a.row_off + i0;
            if (i0 + 1 < a.n_rows && ((reinterpret_cast<uintptr_t>(yp) & 15) == 0)) {
                st_stream_d2(yp, acc0, acc1);
            } else {
                st_stream_d1(yp, acc0);
                if (i0 + 1 < a.n_rows) st_stream_d1(yp + 1, acc1);
            }
        }
    }
}

// ------------------------------------------------------------ tail kernel --
// One warp per work unit: the tail rows whose first spilled entry falls in a
// slice of <= 256 entries (plan_chunks, api.cpp), processed in row order as
// the contiguous entry range [ptr[rb], ptr[re]) in batches of 256 entries.
//   1. the unit's <= 257 row pointers are staged in shared memory once;
//   2. per batch, 8 coalesced col/val loads and 8 x gathers per lane are in
//      flight together; the products are transposed through shared memory
//      (padded, conflict-free) so lane l owns entries kb + 8l .. kb + 8l + 7;
//   3. each lane finds the row of its first entry (binary search in shared
//      memory) and walks its 8 entries: rows that start and end inside the
//      lane are added into y directly; the partial of the lane's last open
//      row is its carry-out;
//   4. a segmented inclusive scan of the carry-outs (__shfl_up_sync, keyed by
//      row) gives each lane the carry-in of its first row, which completes
//      rows spanning lanes; a warp carry joins rows spanning batches.
// Every row is summed in one place in a fixed order: deterministic, no atomics.
// The CSR part runs after the ELL kernel on the same stream.
// kTailRun = entries per lane per batch (template RUN); the product buffer is
// padded one slot per RUN so both the row-major write and the lane-run read
// are bank-conflict free.
template <int RUN>
__device__ __forceinline__ int tail_pad(int i) { return i + i / RUN; }

template <bool HALO, int RUN>
__global__ void __launch_bounds__(128) tail_kernel(TailArgs a) {
    constexpr int kTailRun = RUN;
    __shared__ int32_t s_ptr[4][kTailWarpEntries + 1];
    __shared__ double s_p[4][32 * RUN + 32];
    __shared__ double s_sum[4][kTailWarpEntries];
    const uint64_t pol = policy_evict_first();
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t w = a.warp_begin + (int64_t)blockIdx.x * 4 + wib;
    if (w >= a.warp_end) return;  // warp-uniform
    const int32_t rb = __ldg(a.warp_row + w), re = __ldg(a.warp_row + w + 1);
    if (rb >= re) return;
    const int32_t R = re - rb;  // <= kTailWarpEntries rows
    int32_t* sp = s_ptr[wib];
    double* pp = s_p[wib];
    double* ss = s_sum[wib];   // completed row sums, written once per row
    const int32_t k_first = __ldg(a.ptr + rb), ke = __ldg(a.ptr + re);
    int32_t rw = 0;       // (relative) row containing the batch's first entry
    double carry = 0.0;   // partial sum of row rw from earlier batches
    for (int32_t kb = k_first; kb < ke; kb += 32 * kTailRun) {
        int32_t c[kTailRun];
        double v[kTailRun];
#pragma unroll
        for (int i = 0; i < kTailRun; ++i) {
            const int32_t k = kb + 32 * i + lane;
            c[i] = k < ke ? ld_stream_i1(a.col + k, pol) : -1;
            v[i] = k < ke ? ld_stream_d1(a.val + k, pol) : 0.0;
        }
        if (kb == k_first)  // stage the row pointers while the first batch is in flight
            for (int32_t i = lane; i <= R; i += 32) sp[i] = __ldg(a.ptr + rb + i);
#pragma unroll
        for (int i = 0; i < kTailRun; ++i) {
            const double xg = c[i] >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[i]) : 0.0;
            pp[tail_pad<RUN>(32 * i + lane)] = v[i] * xg;
        }
        __syncwarp();
        const int32_t kl = kb + kTailRun * lane;
        int32_t rr = R - 1, first_row = -1;
        double acc = 0.0, head = 0.0;
        bool head_done = false;
        if (kl < ke) {
            int32_t lo = rw, hi = R - 1;  // first row whose end exceeds kl
            while (lo < hi) {
                const int32_t mid = (lo + hi) >> 1;
                if (sp[mid + 1] > kl) hi = mid; else lo = mid + 1;
            }
            rr = lo;
            first_row = lo;
            int32_t rend = sp[rr + 1];
            bool first = true;
#pragma unroll
            for (int j = 0; j < kTailRun; ++j) {
                const int32_t k = kl + j;
                if (k < ke) {
                    acc += pp[tail_pad<RUN>(kTailRun * lane + j)];
                    if (k + 1 == rend) {  // row rr ends at entry k
                        if (first) { head = acc; head_done = true; first = false; }
                        else { ss[rr] = acc; }
                        acc = 0.0;
                        ++rr;
                        rend = rr < R ? sp[rr + 1] : ke;
                    }
                }
            }
        }
        __syncwarp();  // pp is rewritten by the next batch
        const int32_t row_out = kl < ke ? rr : 0x7fffffff;
        double cs = acc;
        if (lane == 0 && row_out == rw) cs += carry;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double cu = __shfl_up_sync(FULL, cs, d);
            const int32_t ru = __shfl_up_sync(FULL, row_out, d);
            if (lane >= d && ru == row_out) cs += cu;
        }
        const double prev_cs = __shfl_up_sync(FULL, cs, 1);
        const int32_t prev_row = __shfl_up_sync(FULL, row_out, 1);
        if (head_done) {
            const double cin = lane == 0 ? carry : (prev_row == first_row ? prev_cs : 0.0);
            ss[first_row] = head + cin;
        }
        const double cs31 = __shfl_sync(FULL, cs, 31);
        const int32_t row31 = __shfl_sync(FULL, row_out, 31);
        if (kb + 32 * kTailRun < ke) { carry = cs31; rw = row31; }
    }
    __syncwarp();
    // add the unit's row sums into y: independent, coalesced out_rows loads
    for (int32_t r = lane; r < R; r += 32) {
        double* yp = a.y + __ldg(a.out_rows + rb + r);
        *yp += ss[r];
    }
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
        if (const char* e = std::getenv("HEC_X_KEEP")) {
            const int one = std::atoi(e) != 0;
            cudaMemcpyToSymbol(c_x_keep, &one, sizeof(int));
        }
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

template <bool HALO, bool ROWMAP>
static cudaError_t launch_ell_t(const EllArgs& a, cudaStream_t s) {
    const int64_t n_pairs = ((int64_t)a.n_rows + 1) >> 1;
    const int threads = 256;
    int64_t blocks = (n_pairs + threads - 1) / threads;
    const int64_t cap = (int64_t)num_sms() * 8 * 64;  // grid-stride beyond 64 waves
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const dim3 g((unsigned)blocks), b(threads);
    switch (a.width) {
#define HEC_W(w) \
    case w: ell_kernel<w, HALO, ROWMAP><<<g, b, 0, s>>>(a); break;
        HEC_W(1) HEC_W(2) HEC_W(3) HEC_W(4) HEC_W(5) HEC_W(6) HEC_W(7) HEC_W(8)
        HEC_W(9) HEC_W(10) HEC_W(11) HEC_W(12) HEC_W(13) HEC_W(14) HEC_W(15) HEC_W(16)
#undef HEC_W
        default: ell_kernel<0, HALO, ROWMAP><<<g, b, 0, s>>>(a); break;
    }
    return cudaGetLastError();
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
    if (ell_variant() == 1) {
        cudaError_t e = launch_ell_tma(a, s, num_sms());
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();  // clear the sticky-free "not supported" status
    }
    const bool halo = a.x_halo != nullptr;
    const bool rowmap = a.rowmap != nullptr;
    if (halo) return rowmap ? launch_ell_t<true, true>(a, s) : launch_ell_t<true, false>(a, s);
    return rowmap ? launch_ell_t<false, true>(a, s) : launch_ell_t<false, false>(a, s);
}

cudaError_t launch_tail(const TailArgs& a, cudaStream_t s) {
    const int64_t warps = a.warp_end - a.warp_begin;
    if (warps <= 0) return cudaSuccess;
    const int64_t blocks = (warps + 3) / 4;
    if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
    static int run = -1;
    if (run < 0) {
        const char* e = std::getenv("HEC_TAIL_RUN");
        run = (e && std::atoi(e) == 16) ? 16 : 8;
    }
    if (run == 16) {
        if (a.x_halo) tail_kernel<true, 16><<<(unsigned)blocks, 128, 0, s>>>(a);
        else tail_kernel<false, 16><<<(unsigned)blocks, 128, 0, s>>>(a);
    } else {
        if (a.x_halo) tail_kernel<true, 8><<<(unsigned)blocks, 128, 0, s>>>(a);
        else tail_kernel<false, 8><<<(unsigned)blocks, 128, 0, s>>>(a);
    }
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

}  // namespace hec
