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
template <bool HALO>
__device__ __forceinline__ double gather_x(const double* __restrict__ x,
                                           const double* __restrict__ xh, int32_t n_loc,
                                           int32_t c) {
    if (HALO && c >= n_loc) return __ldg(xh + (c - n_loc));
    return __ldg(x + c);
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
// the contiguous entry range [ptr[rb], ptr[re]).  The unit's <= 257 row
// pointers are staged in shared memory once; entries are handled in batches
// of 8 windows of 32: all 16 coalesced col/val loads of a batch, then its 8 x
// gathers, are in flight before any is used.  Per window, every lane finds
// its row by a 5-step shuffle search over the ends of the next 32 rows, a
// segmented inclusive scan (__shfl_up_sync) sums each row's products, a carry
// joins rows that cross windows, and the lane holding a row's last entry adds
// the row sum into y (after the ELL kernel).  All lanes do useful work
// whatever the row lengths; the order of additions is fixed (deterministic).
constexpr int kTailBatch = 8;

template <bool HALO>
__global__ void __launch_bounds__(256) tail_kernel(TailArgs a) {
    __shared__ int32_t s_ptr[8][kTailWarpEntries + 1];
    const uint64_t pol = policy_evict_first();
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t w = a.warp_begin + (int64_t)blockIdx.x * 8 + wib;
    if (w >= a.warp_end) return;  // warp-uniform
    const int32_t rb = __ldg(a.warp_row + w), re = __ldg(a.warp_row + w + 1);
    if (rb >= re) return;
    const int32_t R = re - rb;  // <= 256 rows
    int32_t* sp = s_ptr[wib];
    for (int32_t i = lane; i <= R; i += 32) sp[i] = __ldg(a.ptr + rb + i);
    __syncwarp();
    const int32_t ke = sp[R];
    int32_t rw = rb;      // row of the current window's first entry
    double carry = 0.0;   // partial sum of row rw from earlier windows
    for (int32_t kb = sp[0]; kb < ke; kb += 32 * kTailBatch) {
        int32_t c[kTailBatch];
        double v[kTailBatch], xg[kTailBatch];
#pragma unroll
        for (int i = 0; i < kTailBatch; ++i) {
            const int32_t k = kb + 32 * i + lane;
            c[i] = k < ke ? ld_stream_i1(a.col + k, pol) : -1;
            v[i] = k < ke ? ld_stream_d1(a.val + k, pol) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < kTailBatch; ++i)
            xg[i] = c[i] >= 0 ? gather_x<HALO>(a.x, a.x_halo, a.n_loc, c[i]) : 0.0;
#pragma unroll
        for (int i = 0; i < kTailBatch; ++i) {
            const int32_t k0 = kb + 32 * i;
            if (k0 >= ke) break;  // warp-uniform
            const int32_t k = k0 + lane;
            const bool valid = k < ke;
            const double p = v[i] * xg[i];
            // end (one past the last entry) of row rw + lane; rows past re end at ke
            const int32_t rl = rw - rb + 1 + lane;
            const int32_t end_l = rl <= R ? sp[rl] : ke;
            // lo = #{j : end_j <= k}: a window holds <= 32 rows, so lo <= 31
            int lo = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int32_t e = __shfl_sync(FULL, end_l, lo + step - 1);
                if (e <= k) lo += step;
            }
            const int32_t my_end = __shfl_sync(FULL, end_l, lo);
            const int32_t row = valid ? rw + lo : 0x7fffffff;
            double sum = (lane == 0) ? p + carry : p;  // entry k0 always belongs to row rw
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double su = __shfl_up_sync(FULL, sum, d);
                const int32_t ru = __shfl_up_sync(FULL, row, d);
                if (lane >= d && ru == row) sum += su;
            }
            if (valid && k + 1 == my_end) {  // last entry of its row: the row is complete
                double* yp = a.y + __ldg(a.out_rows + row);
                *yp += sum;
            }
            const double s31 = __shfl_sync(FULL, sum, 31);
            const int32_t row31 = __shfl_sync(FULL, row, 31);
            const int32_t end31 = __shfl_sync(FULL, my_end, 31);
            if (k0 + 32 < ke) {  // next window exists (lane 31 was valid)
                if (k0 + 32 < end31) { carry = s31; rw = row31; }
                else { carry = 0.0; rw = row31 + 1; }
            }
        }
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
    const int64_t blocks = (warps + 7) / 8;
    if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
    if (a.x_halo) tail_kernel<true><<<(unsigned)blocks, 256, 0, s>>>(a);
    else tail_kernel<false><<<(unsigned)blocks, 256, 0, s>>>(a);
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
