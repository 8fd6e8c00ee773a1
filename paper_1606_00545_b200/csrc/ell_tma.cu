// ell_tma.cu -- the ELL part of Alg. 1 with the matrix
// streams staged through shared memory by the bulk-copy engine (TMA,
// cp.async.bulk) in a persistent, warp-specialised kernel.
//
// One CTA per SM (or two), a ring of S stages.  Stage k holds one tile of
// R = 512 rows: for every slot j < W the contiguous slot-column segments
// ELLcol[j*s + tile*R : +R] (int32) and ELLval[j*s + tile*R : +R] (fp64) --
// the column-major layout of P:73 makes each a single 2 KiB / 4 KiB bulk copy.
//   producer warp : waits `empty[k]`, arms `full[k]` with the tile's bytes and
//                   issues 2W bulk copies (L2 evict_first) that complete on it.
//   consumer warps: wait `full[k]`, read their 2 rows x W slots into
//                   registers (int2 / double2, conflict-free), release the
//                   stage, then gather x (L1/L2), FMA in slot order and stream
//                   y out.  The gathers of tile k overlap the copies of k+1..k+S-1.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "hec_internal.h"

namespace hec {

namespace {

constexpr int kRows = 512;             // rows per tile
constexpr int kConsumerWarps = 8;      // 256 consumer threads, 2 rows each
constexpr int kThreads = (kConsumerWarps + 1) * 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra.uni WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

template <int W, bool ROWMAP>
__global__ void __launch_bounds__(kThreads, 1) ell_tma_kernel(EllArgs a, int stages) {
    extern __shared__ __align__(128) unsigned char smem[];
    // layout: [stages][W][kRows] int32 | [stages][W][kRows] double | full[stages] | empty[stages]
    const size_t col_bytes = (size_t)stages * W * kRows * 4;
    const size_t val_bytes = (size_t)stages * W * kRows * 8;
    int32_t* s_col = reinterpret_cast<int32_t*>(smem);
    double* s_val = reinterpret_cast<double*>(smem + col_bytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + col_bytes + val_bytes);
    uint64_t* empty = full + stages;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int k = 0; k < stages; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int64_t s = a.stride;
    const int64_t n_tiles = (a.n_rows + kRows - 1) / kRows;

    if (warp == kConsumerWarps) {  // ---------------- producer warp
        if (lane == 0) {
            const uint64_t pol = pol_evict_first();
            int k = 0;
            for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
                const int st = k % stages;
                const int round = k / stages;
                if (round > 0) mbar_wait(&empty[st], (round - 1) & 1);
                const int64_t r0 = tile * kRows;
                const int64_t rows = (a.avail - r0) < kRows ? (a.avail - r0) : kRows;  // within the stride
                const uint32_t cb = (uint32_t)(rows * 4), vb = (uint32_t)(rows * 8);
                mbar_arrive_expect_tx(&full[st], (uint32_t)W * (cb + vb));
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    bulk_g2s(s_col + ((size_t)st * W + j) * kRows, a.col + j * s + r0, cb, &full[st], pol);
                    bulk_g2s(s_val + ((size_t)st * W + j) * kRows, a.val + j * s + r0, vb, &full[st], pol);
                }
            }
        }
        return;
    }

    // ---------------------------------------------- consumer warps
    const int t = threadIdx.x;  // 0..255: rows 2t, 2t+1 of the tile
    int k = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
        const int st = k % stages;
        const int round = k / stages;
        mbar_wait(&full[st], round & 1);
        int2 c[W];
        double2 v[W];
        const int32_t* sc = s_col + (size_t)st * W * kRows;
        const double* sv = s_val + (size_t)st * W * kRows;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            c[j] = reinterpret_cast<const int2*>(sc + j * kRows)[t];
            v[j] = reinterpret_cast<const double2*>(sv + j * kRows)[t];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);  // stage free: the rest runs from registers
        const int64_t i0 = tile * kRows + 2 * t;
        if (i0 < a.n_rows) {
            double x0[W], x1[W];
#pragma unroll
            for (int j = 0; j < W; ++j) {
                x0[j] = c[j].x >= 0 ? __ldg(a.x + c[j].x) : 0.0;
                x1[j] = c[j].y >= 0 ? __ldg(a.x + c[j].y) : 0.0;
            }
            double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
            for (int j = 0; j < W; ++j) {
                acc0 = fma(v[j].x, x0[j], acc0);
                acc1 = fma(v[j].y, x1[j], acc1);
            }
            if (ROWMAP) {
                __stcs(a.y + a.rowmap[i0], acc0);
                if (i0 + 1 < a.n_rows) __stcs(a.y + a.rowmap[i0 + 1], acc1);
            } else {
                double* yp = a.y + a.row_off + i0;
                if (i0 + 1 < a.n_rows && ((reinterpret_cast<uintptr_t>(yp) & 15) == 0)) {
                    __stcs(reinterpret_cast<double2*>(yp), make_double2(acc0, acc1));
                } else {
                    __stcs(yp, acc0);
                    if (i0 + 1 < a.n_rows) __stcs(yp + 1, acc1);
                }
            }
        }
    }
}

template <int W, bool ROWMAP>
cudaError_t launch_w(const EllArgs& a, cudaStream_t s, int num_sms) {
    const int stage_bytes = W * kRows * 12;
    int stages = (200 * 1024) / stage_bytes;
    if (const char* e = std::getenv("HEC_TMA_STAGES")) stages = std::atoi(e);
    if (stages > 8) stages = 8;
    if (stages < 2) return cudaErrorNotSupported;
    const size_t smem = (size_t)stages * stage_bytes + 2 * stages * sizeof(uint64_t);
    cudaError_t e = cudaFuncSetAttribute(ell_tma_kernel<W, ROWMAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t n_tiles = (a.n_rows + kRows - 1) / kRows;
    int blocks_per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, ell_tma_kernel<W, ROWMAP>, kThreads, smem);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
    int64_t grid = (int64_t)num_sms * blocks_per_sm;
    if (grid > n_tiles) grid = n_tiles;
    ell_tma_kernel<W, ROWMAP><<<(unsigned)grid, kThreads, smem, s>>>(a, stages);
    return cudaGetLastError();
}

}  // namespace

// Returns cudaErrorNotSupported when this variant does not apply (halo
// columns, width outside 1..16); the caller then uses the register kernel.
cudaError_t launch_ell_tma(const EllArgs& a, cudaStream_t s, int num_sms) {
    if (a.x_halo != nullptr) return cudaErrorNotSupported;
    const bool rm = a.rowmap != nullptr;
    switch (a.width) {
#define HEC_TW(w) \
    case w: return rm ? launch_w<w, true>(a, s, num_sms) : launch_w<w, false>(a, s, num_sms);
        HEC_TW(1) HEC_TW(2) HEC_TW(3) HEC_TW(4) HEC_TW(5) HEC_TW(6) HEC_TW(7) HEC_TW(8)
        HEC_TW(9) HEC_TW(10) HEC_TW(11) HEC_TW(12) HEC_TW(13) HEC_TW(14) HEC_TW(15) HEC_TW(16)
#undef HEC_TW
        default: return cudaErrorNotSupported;
    }
}

}  // namespace hec
