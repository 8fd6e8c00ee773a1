// api.cpp -- the single-GPU C ABI: hec_from_csr / hec_info / hec_export /
// hec_spmv / hec_spmv_host / hec_free and hec_plan_part_hec.
//
// hec_spmv is Alg. 1 of PAPER.md: the ELL part "is performed
// firstly" by ell_kernel, then the CSR part by tail_kernel, both on the
// caller's stream (stream order gives the ELL -> CSR ordering).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>

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
        if (m->ws && m->ws_free) m->ws_free(m->ws);
        void* ptrs[] = {m->d_ell_col, m->d_ell_val, m->d_tail_out, m->d_tail_blk, m->d_fuse, m->d_tail_region,
                        m->d_tail_ctr, m->d_tsum, m->d_tail_units, m->d_tail_uwidx,
                        m->d_tail_warp, m->d_tail_col, m->d_tail_val, m->d_rowmap, m->d_coo_row, m->d_stage_x,
                        m->d_stage_y, m->d_ring, m->d_ell_d16, m->d_tile_w, m->d_ell_perm};
        for (void* p : ptrs)
            if (p) cudaFree(p);
        for (cudaEvent_t e : m->ev_x) cudaEventDestroy(e);
        for (cudaEvent_t e : m->ev_y) cudaEventDestroy(e);
        if (m->ev_start) cudaEventDestroy(m->ev_start);
        if (m->ev_fork) cudaEventDestroy(m->ev_fork);
        if (m->ev_join) cudaEventDestroy(m->ev_join);
        if (m->s_tail) cudaStreamDestroy(m->s_tail);
        if (m->s_h2d) cudaStreamDestroy(m->s_h2d);
        if (m->s_d2h) cudaStreamDestroy(m->s_d2h);
        cudaSetDevice(cur);
    }
    delete m;
}

// Row chunks (for hec_spmv_host; one chunk for sub-matrices and small
// matrices), the x prefix each chunk reads, and the tail-kernel work list.
static void plan_chunks(hec_matrix_s* m, const HostHec& h, bool pipelined, std::vector<int32_t>* order,
                        std::vector<int4>* blk, std::vector<int4>* warp, int64_t* entries, int32_t super,
                        std::vector<int64_t>* sb_blk, int32_t row_align = 512) {
    const int32_t n = h.n_rows;
    // ~1M-row chunks, at most 16 (32 chunks measured slower: 3.62 vs 3.41 ms on
    // 256^3; smaller first/last chunks too: 3.36 vs 3.31 ms; the floor is the
    // concurrent H2D + D2H of x and y, 2.78 ms there)
    int32_t K = pipelined ? n / (1 << 20) : 1;
    K = K < 1 ? 1 : (K > 16 ? 16 : K);
    int64_t per = ((int64_t)n + K - 1) / K;
    per = (per + row_align - 1) / row_align * row_align;  // grouped rows never straddle a chunk
    m->chunk_row.assign(1, 0);
    while (m->chunk_row.back() < n)
        m->chunk_row.push_back((int32_t)std::min<int64_t>(n, m->chunk_row.back() + per));
    if (m->chunk_row.size() == 1) m->chunk_row.push_back(0);  // n == 0: one empty chunk
    m->n_chunks = (int32_t)m->chunk_row.size() - 1;
    const int C = m->n_chunks;
    // x prefix per chunk (pipelined host path only)
    m->chunk_xend.assign(C, h.n_cols);
    if (pipelined && C > 1) {
        std::vector<int32_t> cmax(C, -1);
        for (int c = 0; c < C; ++c)
            for (int32_t j = 0; j < h.width; ++j) {
                const int32_t* colj = h.ell_col.data() + (size_t)j * h.stride;
                for (int32_t i = m->chunk_row[c]; i < m->chunk_row[c + 1]; ++i) cmax[c] = std::max(cmax[c], colj[i]);
            }
        int c = 0;
        for (size_t t = 0; t < h.tail_rows.size(); ++t) {
            while (h.tail_rows[t] >= m->chunk_row[c + 1]) ++c;
            for (int32_t k = h.tail_ptr[t]; k < h.tail_ptr[t + 1]; ++k) cmax[c] = std::max(cmax[c], h.tail_col[k]);
        }
        int32_t run = -1;
        for (int q = 0; q < C; ++q) {
            run = std::max(run, cmax[q]);
            m->chunk_xend[q] = run + 1;
        }
    }
    // Tail rows of each chunk (contiguous: tail rows are ascending), cut into
    // super-blocks of kTailSuperRows consecutive tail rows; inside a
    // super-block the rows are sorted by (lanes-per-row G = 2^lg, length),
    // and each CUDA block takes 256/G rows of one G.  Consecutive blocks cover
    // one super-block, so its entries and x window are still reused in L2
    // while every group gets a row width that keeps its lanes busy; sorting
    // by length keeps the rows sharing a warp (G < 32) nearly equally long,
    // so the warp-chunk layout (hec_internal.h) pads little.
    const int32_t tr = (int32_t)h.tail_rows.size();
    const int32_t* tp = h.tail_ptr.data();
    order->assign(tr, 0);
    blk->clear();
    warp->clear();
    *entries = 0;
    m->chunk_blk.assign(C + 1, 0);
    // target entries per lane: more entries per lane = more loads in flight per
    // row and fewer rows in flight -- better for big tails (measured r11:
    // power-law 2^23 tail 8 > 4 > 2 > 1), worse for tiny ones (SPE10)
    const int epl = tail_epl(h.tail_col.size());
    if (const char* e = std::getenv("HEC_TAIL_SUPER")) super = std::max(256, std::atoi(e));  // tuning
    sb_blk->clear();
    int32_t t0 = 0;
    for (int c = 0; c < C; ++c) {
        int32_t t1 = t0;
        while (t1 < tr && h.tail_rows[t1] < m->chunk_row[c + 1]) ++t1;
        for (int32_t sb = t0; sb < t1; sb += super) {
            const int32_t se = std::min(t1, sb + super);
            sb_blk->push_back((int64_t)blk->size());  // this super-block's first descriptor
            for (int32_t t = sb; t < se; ++t) (*order)[t] = t;
            auto key = [&](int32_t t) {
                const int32_t L = tp[t + 1] - tp[t];
                return std::make_pair(tail_lg_for(L, epl), L);
            };
            std::stable_sort(order->begin() + sb, order->begin() + se,
                             [&](int32_t a, int32_t b) { return key(a) < key(b); });
            for (int32_t f = sb; f < se;) {
                const int g = key((*order)[f]).first, G = 1 << g, per_blk = kTailThreads >> g;
                int32_t cnt = 0;
                while (cnt < per_blk && f + cnt < se && key((*order)[f + cnt]).first == g) ++cnt;
                blk->push_back(make_int4(f, cnt, g, (int32_t)warp->size()));
                // the descriptor's warps: thread tid = 32 w + l serves row tid >> g
                for (int w = 0; w < kTailWarps; ++w) {
                    int32_t iters = 0;
                    const int32_t r_lo = (32 * w) >> g, r_hi = std::min(cnt, ((32 * w + 31) >> g) + 1);
                    for (int32_t r = r_lo; r < r_hi; ++r) {
                        const int32_t t = (*order)[f + r];
                        iters = std::max(iters, (tp[t + 1] - tp[t] + 2 * G - 1) / (2 * G));
                    }
                    warp->push_back(make_int4((int32_t)std::min<int64_t>(*entries, INT32_MAX), iters, f, (cnt << 8) | g));
                    *entries += (int64_t)iters * kTailChunk;
                }
                f += cnt;
            }
        }
        m->chunk_blk[c + 1] = (int64_t)blk->size();
        t0 = t1;
    }
    sb_blk->push_back((int64_t)blk->size());
}

// Every stored tail entry's device position in the warp-chunk layout:
// f(position, index of the entry in the host tail arrays).  Thread tid =
// 32 w + l of a descriptor serves row tid >> lg as lane lr = tid & (G - 1);
// in iteration i it reads its row's entries 2 (i G + lr) + e, e = 0, 1, at
// position base_w + 64 i + 2 l + e.
template <typename F>
static void for_each_tail_entry(const std::vector<int4>& blk, const std::vector<int4>& warp,
                                const std::vector<int32_t>& order, const std::vector<int32_t>& tail_ptr, F f) {
    for (const int4& d : blk) {
        const int g = d.z, G = 1 << g;
        for (int w = 0; w < kTailWarps; ++w) {
            const int4 wm = warp[(size_t)d.w + w];
            for (int l = 0; l < 32; ++l) {
                const int tid = 32 * w + l, r = tid >> g, lr = tid & (G - 1);
                if (r >= d.y) continue;
                const int32_t t = order[(size_t)d.x + r];
                const int32_t b = tail_ptr[t], L = tail_ptr[t + 1] - b;
                for (int32_t i = 0; i < wm.y; ++i)
                    for (int e = 0; e < 2; ++e) {
                        const int32_t idx = 2 * (i * G + lr) + e;
                        if (idx < L) f((int64_t)wm.x + (int64_t)kTailChunk * i + 2 * l + e, b + idx);
                    }
            }
        }
    }
}

// x-ring schedule of the tail (tail_ring_kernel).  Warp units --
// one warp meta of rows with G <= 32 lanes, or the G / 32 metas of one longer
// row, which a single warp then walks in turn -- are split over one CTA per
// SM in contiguous runs of equal stored positions; a CTA's run is cut into
// stages at super-block boundaries.  Each stage gets the window [lo, hi) of
// x columns its gathers read from the CTA's shared-memory ring: centred on
// the median column of the stage's entries (made non-decreasing along the
// run), with one half-width h per CTA so that hi_s - lo_(s-D+1) <= the ring's
// kRingCols columns, D = kRingDepth stages in flight (stage s's new columns
// only overwrite ring slots of columns below lo_(s-D+1), i.e. of stages
// <= s - D) and lo, hi even (16-byte bulk copies).  Columns outside the window are gathered from global memory,
// so any matrix is correct; `cover` says how many stored entries hit.
struct RingPlan {
    std::vector<int4> stage;   // {lo, hi, u0, u1}
    std::vector<int4> unit;    // {warp meta, metas, warp index in the descriptor, 0}
    std::vector<int32_t> cta;  // [n_cta + 1] stage prefix
    double cover = 0.0;
};
static void plan_ring(const std::vector<int4>& blk, const std::vector<int4>& warp, const std::vector<int64_t>& sb_blk,
                      const std::vector<int32_t>& dcol, int32_t n_x, int n_cta, RingPlan* rp) {
    std::vector<int4> unit;
    std::vector<int32_t> usb;          // super-block of each unit
    std::vector<int64_t> upre(1, 0);   // prefix of the units' stored positions
    for (size_t q = 0; q + 1 < sb_blk.size(); ++q)
        for (int64_t d = sb_blk[q]; d < sb_blk[q + 1]; ++d) {
            const int g = blk[(size_t)d].z, G = 1 << g, cnt = blk[(size_t)d].y;
            const int32_t w0 = blk[(size_t)d].w;
            if (G <= 32) {
                for (int w = 0; w < kTailWarps && ((32 * w) >> g) < cnt; ++w) {
                    unit.push_back(make_int4(w0 + w, 1, w, 0));
                    usb.push_back((int32_t)q);
                    upre.push_back(upre.back() + (int64_t)warp[(size_t)w0 + w].y * kTailChunk);
                }
            } else {
                const int nw = G >> 5;
                for (int r = 0; r < cnt; ++r) {
                    int64_t e = 0;
                    for (int j = 0; j < nw; ++j) e += (int64_t)warp[(size_t)w0 + r * nw + j].y * kTailChunk;
                    unit.push_back(make_int4(w0 + r * nw, nw, r * nw, 0));
                    usb.push_back((int32_t)q);
                    upre.push_back(upre.back() + e);
                }
            }
        }
    const int64_t U = (int64_t)unit.size();
    if (U == 0 || n_cta <= 0) return;
    std::vector<int64_t> ub((size_t)n_cta + 1, U);
    ub[0] = 0;
    for (int c = 1; c < n_cta; ++c) {
        ub[c] = std::lower_bound(upre.begin(), upre.end(), upre.back() * c / n_cta) - upre.begin();
        ub[c] = std::max(std::min(ub[c], U), ub[c - 1]);
    }
    // stored columns (local x) of a unit's positions
    auto unit_cols = [&](int64_t u, std::vector<int32_t>* out) {
        const int4 un = unit[(size_t)u];
        for (int j = 0; j < un.y; ++j) {
            const int4 wm = warp[(size_t)un.x + j];
            for (int64_t p = wm.x; p < (int64_t)wm.x + (int64_t)wm.y * kTailChunk; ++p) {
                const int32_t c = dcol[(size_t)p];
                if (c >= 0 && c < n_x) out->push_back(c);
            }
        }
    };
    const int64_t W = kRingCols;
    const int32_t nx_even = n_x & ~1;
    int64_t stored = 0, hit = 0;
    rp->cta.assign(1, 0);
    std::vector<int32_t> cols;
    for (int c = 0; c < n_cta; ++c) {
        std::vector<int64_t> cen;
        std::vector<std::pair<int64_t, int64_t>> su;  // stage unit ranges
        for (int64_t u = ub[c]; u < ub[c + 1];) {
            int64_t v = u;
            while (v < ub[c + 1] && usb[(size_t)v] == usb[(size_t)u]) ++v;
            cols.clear();
            for (int64_t k = u; k < v; ++k) unit_cols(k, &cols);
            int64_t m = cen.empty() ? 0 : cen.back();
            if (!cols.empty()) {
                std::nth_element(cols.begin(), cols.begin() + cols.size() / 2, cols.end());
                m = std::max<int64_t>(cols[cols.size() / 2], cen.empty() ? 0 : cen.back());
            }
            cen.push_back(m);
            su.emplace_back(u, v);
            u = v;
        }
        // the windows of kRingDepth consecutive stages share the ring
        int64_t dmax = 0;
        for (size_t k = 1; k < cen.size(); ++k)
            dmax = std::max(dmax, cen[k] - cen[k >= (size_t)kRingDepth - 1 ? k - (kRingDepth - 1) : 0]);
        const int64_t h = std::max<int64_t>(0, (W - dmax - 4) / 2);
        for (size_t k = 0; k < cen.size(); ++k) {
            int64_t lo = std::max<int64_t>(0, ((cen[k] - h) >> 1) << 1);
            int64_t hi = std::min<int64_t>(nx_even, ((cen[k] + h + 1) >> 1) << 1);
            if (h == 0 || hi < lo) hi = lo;
            rp->stage.push_back(make_int4((int32_t)lo, (int32_t)hi, (int32_t)su[k].first, (int32_t)su[k].second));
            cols.clear();
            for (int64_t u = su[k].first; u < su[k].second; ++u) unit_cols(u, &cols);
            stored += (int64_t)cols.size();
            for (int32_t col : cols) hit += (col >= lo && col < hi);
        }
        rp->cta.push_back((int32_t)rp->stage.size());
    }
    rp->unit = std::move(unit);
    rp->cover = stored > 0 ? (double)hit / (double)stored : 0.0;
}

// ELL index compression: the ELL kernel is bound by the bytes it
// streams, 12 per slot (fp64 value + int32 column).  Where the columns sit at
// (nearly) fixed offsets from the row -- stencils, banded reservoir matrices
// -- slot j of row i stores d = col - i - base_j as an int16 next to the
// int32 array, base_j the most common offset of slot j; padding stores
// kIdxPad, and a slot whose delta does not fit stores kIdxEsc and the kernel
// reads its int32 column instead.  10 bytes per slot instead of 12; the
// arithmetic and every result are unchanged.  Opt-in (HEC_IDX16=1): measured
// no faster (256^3 0.253 vs 0.245 ms, 150^3 and SPE10 within 2%), DESIGN §5.
static hec_status plan_idx16(hec_matrix_s* m, const HostHec& h, cudaStream_t s, int64_t* bytes) {
    const char* e = std::getenv("HEC_IDX16");
    const int32_t w = h.width, n = h.n_rows;
    if (!e || std::atoi(e) == 0 || w < 1 || w > kIdx16MaxW || n == 0) return HEC_OK;
    const int64_t sstr = h.stride;
    // base_j: the mode of (col - row) over every row, or over 2^16 rows drawn
    // by a hash (a fixed stride would alias with grid periods: every 256th row
    // of 256^3 is an x = 0 boundary row)
    std::vector<int32_t> rows;
    if (n <= (1 << 16)) {
        rows.resize(n);
        for (int32_t i = 0; i < n; ++i) rows[i] = i;
    } else {
        rows.resize(1 << 16);
        for (uint64_t k = 0; k < rows.size(); ++k) {
            uint64_t z = (k + 1) * 0x9E3779B97F4A7C15ULL;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            rows[k] = (int32_t)((z ^ (z >> 31)) % (uint64_t)n);
        }
    }
    std::vector<int64_t> dl;
    for (int32_t j = 0; j < w; ++j) {
        dl.clear();
        const int32_t* cj = h.ell_col.data() + (size_t)j * sstr;
        for (int32_t i : rows)
            if (cj[i] >= 0) dl.push_back((int64_t)cj[i] - i);
        int64_t best = 0, bc = 0;
        std::sort(dl.begin(), dl.end());
        for (size_t a = 0; a < dl.size();) {
            size_t b = a;
            while (b < dl.size() && dl[b] == dl[a]) ++b;
            if ((int64_t)(b - a) > bc) { bc = (int64_t)(b - a); best = dl[a]; }
            a = b;
        }
        m->idx16_base[j] = (int32_t)std::max<int64_t>(INT32_MIN / 2, std::min<int64_t>(INT32_MAX / 2, best));
    }
    std::vector<int16_t> d16((size_t)w * sstr, kIdxPad);  // rows past n_rows: padding
    int64_t esc = 0;
    for (int32_t j = 0; j < w; ++j) {
        const int32_t* cj = h.ell_col.data() + (size_t)j * sstr;
        int16_t* dj = d16.data() + (size_t)j * sstr;
        for (int32_t i = 0; i < n; ++i) {
            const int64_t d = (int64_t)cj[i] - i - m->idx16_base[j];
            if (cj[i] < 0) dj[i] = kIdxPad;
            else if (d > kIdxPad && d <= INT16_MAX) dj[i] = (int16_t)d;
            else { dj[i] = kIdxEsc; ++esc; }
        }
    }
    m->idx16_esc = (double)esc / ((double)w * n);
    hec_status st = dmalloc_copy(&m->d_ell_d16, d16.data(), d16.size(), s, bytes);
    if (st != HEC_OK) return st;
    HEC_CUDA_TRY(cudaStreamSynchronize(s));  // d16 dies after return
    return HEC_OK;
}

// ELL rows grouped by length: inside windows of kGroupRows rows,
// rows are stably sorted by their ELL length (longest first), so a warp's 64
// rows are nearly equally long and the second-phase slots past the longest
// of them -- padding for all 64 -- are skipped (plan_tile_w).  The ELL part
// of row perm[p] is stored at position p; the ELL launch writes that row's
// output (the tail, keyed by row, is unaffected).  Handles with a two-phase
// width and at least min_rows rows, when grouping makes at least 5% more
// slots skippable than the natural order already does (HEC_ELL_GROUP=0
// never, =1 always).
static void skip_fraction(const HostHec& h, const int32_t* len_at, double* out) {
    const int32_t w = h.width, P1 = ell_first_phase(w);
    const int64_t nt = ((int64_t)h.stride + 63) / 64;
    int64_t read = 0;
    for (int64_t t = 0; t < nt; ++t) {
        int32_t mx = 0;
        for (int64_t i = t * 64; i < std::min<int64_t>((t + 1) * 64, h.n_rows); ++i) mx = std::max(mx, len_at[i]);
        read += 64 * (int64_t)std::max(P1, mx);
    }
    *out = 1.0 - (double)read / ((double)w * 64.0 * (double)nt);
}
static void plan_group(HostHec& h, int32_t min_rows, std::vector<int32_t>* perm) {
    perm->clear();
    const int32_t w = h.width, n = h.n_rows;
    int env = -1;
    if (const char* e = std::getenv("HEC_ELL_GROUP")) env = std::atoi(e) != 0 ? 1 : 0;
    if (env == 0 || w <= HEC_ELL_PHASE || w > kIdx16MaxW || n < 64 || (env < 0 && n < min_rows)) return;
    std::vector<int32_t> len((size_t)n, 0);
    for (int32_t j = 0; j < w; ++j) {
        const int32_t* cj = h.ell_col.data() + (size_t)j * h.stride;
        for (int32_t i = 0; i < n; ++i) len[i] += cj[i] >= 0;
    }
    std::vector<int32_t> p((size_t)n);
    for (int32_t i = 0; i < n; ++i) p[i] = i;
    for (int32_t b = 0; b < n; b += kGroupRows) {
        const int32_t e = std::min(n, b + kGroupRows);
        std::stable_sort(p.begin() + b, p.begin() + e, [&](int32_t a, int32_t c) { return len[a] > len[c]; });
    }
    bool ident = true;
    for (int32_t i = 0; i < n && ident; ++i) ident = p[i] == i;
    if (ident) return;
    std::vector<int32_t> lp((size_t)n);
    for (int32_t i = 0; i < n; ++i) lp[i] = len[p[i]];
    double nat = 0.0, grp = 0.0;
    skip_fraction(h, len.data(), &nat);
    skip_fraction(h, lp.data(), &grp);
    if (env != 1 && grp - nat < 0.05) return;
    std::vector<int32_t> tc((size_t)n);
    std::vector<double> tv((size_t)n);
    for (int32_t j = 0; j < w; ++j) {
        int32_t* cj = h.ell_col.data() + (size_t)j * h.stride;
        double* vj = h.ell_val.data() + (size_t)j * h.stride;
        for (int32_t i = 0; i < n; ++i) {
            tc[i] = cj[p[i]];
            tv[i] = vj[p[i]];
        }
        std::copy(tc.begin(), tc.end(), cj);
        std::copy(tv.begin(), tv.end(), vj);
    }
    perm->swap(p);
}

// Second-phase slot skipping: ELL widths loaded in two phases
// (w > HEC_ELL_PHASE) read the second phase's slots only up to the longest
// row of each warp's 64 rows.  Worth it where rows of similar length sit
// together (degree-sorted inputs); planned when at least 5% of the slots go
// unread (HEC_TILE_SKIP=0 never, =1 always).
static hec_status plan_tile_w(hec_matrix_s* m, const HostHec& h, cudaStream_t s, int64_t* bytes) {
    const int32_t w = h.width, n = h.n_rows;
    const int P1 = ell_first_phase(w);
    int env = -1;
    if (const char* e = std::getenv("HEC_TILE_SKIP")) env = std::atoi(e) != 0 ? 1 : 0;
    if (env == 0 || w <= HEC_ELL_PHASE || w > kIdx16MaxW || n == 0) return HEC_OK;
    const int64_t nt = ((int64_t)h.stride + 63) / 64;
    std::vector<uint8_t> tw((size_t)nt, 0);
    for (int32_t j = 0; j < w; ++j) {
        const int32_t* cj = h.ell_col.data() + (size_t)j * h.stride;
        for (int32_t i = 0; i < n; ++i)
            if (cj[i] >= 0) tw[(size_t)(i >> 6)] = (uint8_t)std::max<int>(tw[(size_t)(i >> 6)], j + 1);
    }
    int64_t read = 0;
    for (int64_t t = 0; t < nt; ++t) read += 64 * (int64_t)std::max<int>(P1, tw[(size_t)t]);
    m->tile_skip = 1.0 - (double)read / ((double)w * 64.0 * (double)nt);
    if (env != 1 && m->tile_skip < 0.05) return HEC_OK;
    hec_status st = dmalloc_copy(&m->d_tile_w, tw.data(), tw.size(), s, bytes);
    if (st != HEC_OK) return st;
    HEC_CUDA_TRY(cudaStreamSynchronize(s));
    return HEC_OK;
}

static hec_status make_matrix_impl(HostHec&& h, int32_t device, cudaStream_t s, const int32_t* rowmap,
                                   int32_t n_rowmap, int32_t row_off, int32_t n_loc, hec_matrix* out, bool coo_tail);

// Every host planning step (tail layout, grouping, rings) allocates: a failed
// allocation is reported, never thrown across the C ABI (the handle's device
// memory is released by its owner on the way out).
hec_status make_matrix(HostHec&& h, int32_t device, cudaStream_t s, const int32_t* rowmap,
                       int32_t n_rowmap, int32_t row_off, int32_t n_loc, hec_matrix* out, bool coo_tail) {
    try {
        return make_matrix_impl(std::move(h), device, s, rowmap, n_rowmap, row_off, n_loc, out, coo_tail);
    } catch (const std::bad_alloc&) {
        return fail(HEC_ERR_NOMEM, "host allocation failed while building the device HEC");
    } catch (...) {
        return fail(HEC_ERR_STATE, "unexpected exception while building the device HEC");
    }
}

static hec_status make_matrix_impl(HostHec&& h, int32_t device, cudaStream_t s, const int32_t* rowmap,
                                   int32_t n_rowmap, int32_t row_off, int32_t n_loc, hec_matrix* out, bool coo_tail) {
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
    m->tail_coo = coo_tail;
    std::vector<int32_t> order;
    std::vector<int4> blk, warp;
    std::vector<int64_t> sb_blk;
    int64_t entries = 0;
    // x-ring schedule (opt-in HEC_TAIL_RING=1, measured slower
    // than the one-CTA-per-descriptor grid on the power-law tail: 269 vs 248
    // us at best): planned with the ring's super-block size
    int ring_env = 0;
    if (const char* e = std::getenv("HEC_TAIL_RING")) ring_env = std::atoi(e) != 0 ? 1 : 0;
    const bool ring_cand = !coo_tail && !h.tail_rows.empty() && ring_env == 1;
    // rows grouped by ELL length: whole matrices from 2^20 rows (below, the
    // launch dominates and a small tail is better run first, fused with the
    // ELL launch), distributed sub-matrices from 2^16 rows
    const bool whole = n_loc < 0 && !rowmap && row_off == 0;
    if (!coo_tail) plan_group(h, whole ? (1 << 20) : (1 << 16), &m->h_ell_perm);
    plan_chunks(m.get(), h, n_loc < 0 && !rowmap && !coo_tail, &order, &blk, &warp, &entries,
                ring_cand ? kRingSuperRows : kTailSuperRows, &sb_blk, m->h_ell_perm.empty() ? 512 : kGroupRows);
    int64_t bytes = 0;
    hec_status st;
    if ((st = dmalloc_copy(&m->d_ell_col, h.ell_col.data(), h.ell_col.size(), s, &bytes))) return st;
    if (!m->h_ell_perm.empty()) {
        // the ELL launch's output row of device position p: the stored row's
        // own output row (row map or offset) -- for whole matrices perm[p]
        std::vector<int32_t> out(m->h_ell_perm.size());
        for (size_t p = 0; p < out.size(); ++p) {
            const int32_t r = m->h_ell_perm[p];
            out[p] = rowmap ? rowmap[r] : row_off + r;
        }
        if ((st = dmalloc_copy(&m->d_ell_perm, out.data(), out.size(), s, &bytes))) return st;
        HEC_CUDA_TRY(cudaStreamSynchronize(s));
    }
    if ((st = plan_idx16(m.get(), h, s, &bytes))) return st;
    if ((st = plan_tile_w(m.get(), h, s, &bytes))) return st;
    if (coo_tail) {  // HYB comparison variant: remainder as row-sorted COO triplets
        std::vector<int32_t> rows(h.tail_col.size());
        for (size_t t = 0; t < h.tail_rows.size(); ++t)
            for (int32_t k = h.tail_ptr[t]; k < h.tail_ptr[t + 1]; ++k)
                rows[k] = rowmap ? rowmap[h.tail_rows[t]] : row_off + h.tail_rows[t];
        m->h_tail_ptr = h.tail_ptr;
        if ((st = dmalloc_copy(&m->d_ell_val, h.ell_val.data(), h.ell_val.size(), s, &bytes))) return st;
        if ((st = dmalloc_copy(&m->d_coo_row, rows.data(), rows.size(), s, &bytes))) return st;
        if ((st = dmalloc_copy(&m->d_tail_col, h.tail_col.data(), h.tail_col.size(), s, &bytes))) return st;
        if ((st = dmalloc_copy(&m->d_tail_val, h.tail_val.data(), h.tail_val.size(), s, &bytes))) return st;
        HEC_CUDA_TRY(cudaStreamSynchronize(s));
        m->device_bytes = bytes;
        *out = m.release();
        return HEC_OK;
    }
    if ((st = dmalloc_copy(&m->d_ell_val, h.ell_val.data(), h.ell_val.size(), s, &bytes))) return st;
    if (!h.tail_rows.empty()) {
        // Device copy of the CSR tail in the warp-chunk layout (hec_internal.h):
        // every entry goes to the position its lane reads it from, gaps are
        // (-1, +0.0) padding (reading A4).  hec_export walks the same map back.
        if (entries > INT32_MAX) return fail(HEC_ERR_DIM, "padded CSR tail exceeds int32 positions");
        const size_t tr = h.tail_rows.size();
        std::vector<int32_t> dcol((size_t)entries, -1), dout(tr);
        std::vector<double> dval((size_t)entries, 0.0);
        for_each_tail_entry(blk, warp, order, h.tail_ptr, [&](int64_t pos, int32_t k) {
            dcol[(size_t)pos] = h.tail_col[k];
            dval[(size_t)pos] = h.tail_val[k];
        });
        for (size_t p = 0; p < tr; ++p) dout[p] = rowmap ? rowmap[h.tail_rows[order[p]]] : row_off + h.tail_rows[order[p]];
        int n_sm = 0;
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device);
        if (ring_cand && n_sm > 0) {
            RingPlan rp;
            plan_ring(blk, warp, sb_blk, dcol, n_loc >= 0 ? n_loc : h.n_cols, n_sm, &rp);
            m->ring_cover = rp.cover;
            if (!rp.stage.empty()) {
                const size_t b4 = sizeof(int4) * (rp.stage.size() + rp.unit.size());
                HEC_CUDA_TRY(cudaMalloc(&m->d_ring, b4 + sizeof(int32_t) * rp.cta.size()));
                bytes += (int64_t)(b4 + sizeof(int32_t) * rp.cta.size());
                int4* p4 = static_cast<int4*>(m->d_ring);
                HEC_CUDA_TRY(cudaMemcpyAsync(p4, rp.stage.data(), sizeof(int4) * rp.stage.size(),
                                             cudaMemcpyHostToDevice, s));
                HEC_CUDA_TRY(cudaMemcpyAsync(p4 + rp.stage.size(), rp.unit.data(), sizeof(int4) * rp.unit.size(),
                                             cudaMemcpyHostToDevice, s));
                int32_t* pc = reinterpret_cast<int32_t*>(p4 + rp.stage.size() + rp.unit.size());
                HEC_CUDA_TRY(cudaMemcpyAsync(pc, rp.cta.data(), sizeof(int32_t) * rp.cta.size(),
                                             cudaMemcpyHostToDevice, s));
                HEC_CUDA_TRY(cudaStreamSynchronize(s));  // rp dies after this scope
                m->d_ring_stage = p4;
                m->d_ring_unit = p4 + rp.stage.size();
                m->d_ring_cta = pc;
                m->ring_ctas = n_sm;
            }
        }
        // Descriptor order of the tail launch: last to first -- its
        // first CTAs then gather the x band the ELL kernel's last CTAs left in
        // L2 (power-law: 0.4217 -> 0.4170 ms) -- when the tail reaches the last
        // rows at all (degree-sorted: the tail rows are the top rows, nothing
        // to reuse, and reversed measured 0.494 -> 0.500 ms).
        // HEC_TAIL_REVERSE=0/1 overrides.
        m->tail_reverse = h.tail_rows.back() >= h.n_rows - std::max<int32_t>(1, h.n_rows / 20);
        if (const char* e = std::getenv("HEC_TAIL_REVERSE")) m->tail_reverse = std::atoi(e) != 0;
        m->h_tail_order = order;
        m->h_tail_ptr = h.tail_ptr;
        m->h_tail_blk = blk;
        m->h_tail_warp = warp;
        m->tail_entries = entries;
        if ((st = dmalloc_copy(&m->d_tail_out, dout.data(), dout.size(), s, &bytes))) return st;
        if ((st = dmalloc_copy(&m->d_tail_blk, blk.data(), blk.size(), s, &bytes))) return st;
        if ((st = dmalloc_copy(&m->d_tail_warp, warp.data(), warp.size(), s, &bytes))) return st;
        if ((st = dmalloc_copy(&m->d_tail_col, dcol.data(), dcol.size(), s, &bytes))) return st;
        if ((st = dmalloc_copy(&m->d_tail_val, dval.data(), dval.size(), s, &bytes))) return st;
        // SM-local persistent schedule, warp by warp (opt-in HEC_TAIL_WARP=1,
        // big tails: more descriptors than one wave): warp units cut into one
        // region per SM with equal entries.  DESIGN §5 has the measurements.
        bool warp_sched = false;
        if (const char* e = std::getenv("HEC_TAIL_WARP"))
            warp_sched = n_sm > 0 && (int64_t)blk.size() > (int64_t)n_sm * (48 / kTailWarps) && std::atoi(e) != 0;
        if (warp_sched) {
            std::vector<int4> units;
            std::vector<int32_t> uwidx;
            std::vector<int64_t> uent(1, 0);  // prefix of the units' (padded) entries
            for (size_t d = 0; d < blk.size(); ++d) {
                const int g = blk[d].z, G = 1 << g, cnt = blk[d].y;
                const int32_t w0 = blk[d].w;
                if (G <= 32) {
                    for (int w = 0; w < kTailWarps; ++w) {
                        if (((32 * w) >> g) >= cnt) break;  // no rows in this warp (nor later ones)
                        units.push_back(warp[(size_t)w0 + w]);
                        uwidx.push_back(w0 + w);
                        uent.push_back(uent.back() + (int64_t)warp[(size_t)w0 + w].y * kTailChunk);
                    }
                } else {
                    const int nw = G >> 5;
                    for (int r = 0; r < cnt; ++r) {
                        int64_t e = 0;
                        for (int j = 0; j < nw; ++j) e += (int64_t)warp[(size_t)w0 + r * nw + j].y * kTailChunk;
                        units.push_back(warp[(size_t)w0 + r * nw]);
                        uwidx.push_back(w0 + r * nw);
                        uent.push_back(uent.back() + e);
                    }
                }
            }
            std::vector<int64_t> reg((size_t)n_sm + 1, 0);
            for (int r = 1; r < n_sm; ++r) {
                const int64_t target = uent.back() * r / n_sm;
                reg[r] = std::lower_bound(uent.begin(), uent.end(), target) - uent.begin();
                reg[r] = std::max(reg[r], reg[r - 1]);
            }
            reg[n_sm] = (int64_t)units.size();
            if ((st = dmalloc_copy(&m->d_tail_units, units.data(), units.size(), s, &bytes))) return st;
            if ((st = dmalloc_copy(&m->d_tail_uwidx, uwidx.data(), uwidx.size(), s, &bytes))) return st;
            if ((st = dmalloc_copy(&m->d_tail_region, reg.data(), reg.size(), s, &bytes))) return st;
            std::vector<unsigned int> zero((size_t)n_sm + 1, 0u);
            if ((st = dmalloc_copy(&m->d_tail_ctr, zero.data(), zero.size(), s, &bytes))) return st;
            m->tail_regions = n_sm;
            HEC_CUDA_TRY(cudaStreamSynchronize(s));  // units / reg die after this scope
        }
        // concurrent tail for big tails (opt-in HEC_TAIL_CONC=1): measured slower
        // (power-law 0.484 vs 0.436 ms: the two kernels share the memory system
        // and the scattered combine pass costs 48 us), DESIGN §5
        if (const char* e = std::getenv("HEC_TAIL_CONC"))
            if (std::atoi(e) != 0 && (int64_t)blk.size() > (int64_t)n_sm * (48 / kTailWarps) && n_loc < 0 && !rowmap) {
                HEC_CUDA_TRY(cudaMalloc(&m->d_tsum, sizeof(double) * h.tail_rows.size()));
                bytes += (int64_t)(sizeof(double) * h.tail_rows.size());
                HEC_CUDA_TRY(cudaStreamCreateWithFlags(&m->s_tail, cudaStreamNonBlocking));
                HEC_CUDA_TRY(cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming));
                HEC_CUDA_TRY(cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming));
                m->tail_conc = true;
            }
        HEC_CUDA_TRY(cudaStreamSynchronize(s));  // host vectors die after return
    }
    // Small tails, tail first: the tail kernel (one wave) stores its row sums
    // into y and the ELL kernel, its programmatic dependent, adds them in the
    // CTAs that own tail rows -- the tail's latency hides under the ELL stream
    // instead of trailing it.  Whole matrices whose ELL CTAs each take one tile
    // of rows (no grid stride).  HEC_FUSE_TAIL=0 disables; HEC_FUSE_TAIL_MAX =
    // most tail-kernel CTAs (default: one wave, 148 x 6).
    if (!h.tail_rows.empty() && n_loc < 0 && !rowmap && row_off == 0 && m->h_ell_perm.empty()) {
        int64_t fmax = (int64_t)148 * (48 / kTailWarps);
        if (const char* e = std::getenv("HEC_FUSE_TAIL_MAX")) fmax = std::atol(e);
        bool fuse = (int64_t)blk.size() <= fmax;
        if (const char* e = std::getenv("HEC_FUSE_TAIL")) fuse = fuse && std::atoi(e) != 0;
        const int32_t T = 2 * ell_block_threads(h.width);
        const int64_t n_cta = ((int64_t)h.n_rows + T - 1) / T;
        if (fuse && n_cta <= ell_grid_cap()) {
            const size_t tr = h.tail_rows.size();
            std::vector<int32_t> buf((size_t)n_cta + 1 + tr, 0);
            for (size_t t = 0; t < tr; ++t) {
                buf[(size_t)(h.tail_rows[t] / T) + 1]++;
                buf[(size_t)n_cta + 1 + t] = h.tail_rows[t];  // ascending
            }
            for (int64_t c = 0; c < n_cta; ++c) buf[(size_t)c + 1] += buf[(size_t)c];
            if ((st = dmalloc_copy(&m->d_fuse, buf.data(), buf.size(), s, &bytes))) return st;
            HEC_CUDA_TRY(cudaStreamSynchronize(s));  // buf dies after this scope
            m->d_fuse_cta = m->d_fuse;
            m->d_fuse_row = m->d_fuse + n_cta + 1;
            m->fuse_tile = T;
        }
    }
    if (rowmap)
        if ((st = dmalloc_copy(&m->d_rowmap, rowmap, (size_t)n_rowmap, s, &bytes))) return st;
    HEC_CUDA_TRY(cudaStreamSynchronize(s));
    m->device_bytes = bytes;
    *out = m.release();
    return HEC_OK;
}

// Chunk c of the handle (rows [chunk_row[c], chunk_row[c+1]), r0 a multiple
// of 512), or all chunks when c < 0: ELL kernel then tail kernel.
static hec_status launch_chunks(const hec_matrix_s* A, int c, const double* x, const double* x_halo,
                                double* y, cudaStream_t s, double alpha = 1.0, double beta = 0.0,
                                const double* jd = nullptr, const double* jb = nullptr, double omega = 0.0,
                                const PeerWait* pw = nullptr) {
    const int32_t r0 = c < 0 ? 0 : A->chunk_row[c];
    const int32_t r1 = c < 0 ? A->n_rows : A->chunk_row[c + 1];
    EllArgs e;
    e.col = A->d_ell_col ? A->d_ell_col + r0 : nullptr;
    e.val = A->d_ell_val ? A->d_ell_val + r0 : nullptr;
    e.stride = A->stride;
    e.avail = (int64_t)A->stride - r0;
    e.n_rows = r1 - r0;
    e.width = A->width;
    e.x = x;
    e.x_halo = x_halo;
    e.n_loc = A->n_loc >= 0 ? A->n_loc : A->n_cols;
    e.y = (A->d_rowmap || A->d_ell_perm) ? y : y + r0;
    e.rowmap = A->d_ell_perm ? A->d_ell_perm + r0 : A->d_rowmap ? A->d_rowmap + r0 : nullptr;
    e.row_off = A->row_off;
    e.alpha = alpha;
    e.beta = beta;
    if (A->d_ell_d16) {  // compressed column indices (plan_idx16)
        e.d16 = A->d_ell_d16 + r0;
        e.row0 = r0;
        for (int j = 0; j < A->width && j < kIdx16MaxW; ++j) e.base[j] = A->idx16_base[j];
    }
    if (A->d_tile_w) e.tile_w = A->d_tile_w + r0 / 64;  // r0: a multiple of 512
    e.diag = jd;  // Jacobi epilogue (whole matrix only: c < 0)
    e.b = jb;
    e.omega = omega;
    // plain whole-matrix product: the small tail rides in the ELL launch
    const bool fused = A->fuse_tile > 0 && c < 0 && !pw && !jd && alpha == 1.0 && beta == 0.0 && !x_halo &&
                       A->fuse_tile == 2 * ell_block_threads(A->width);
    if (fused) {
        e.fuse_cta = A->d_fuse_cta;
        e.fuse_row = A->d_fuse_row;
        e.pdl = true;  // dependent of the tail kernel launched just before it
    }
    if (pw) {  // peer-memory transport: wait for the peers' flags, boundary ELL as its dependent
        cudaError_t we = launch_peer_wait(*pw, s);
        if (we != cudaSuccess) return cuda_fail(we, "peer_wait_kernel launch");
        e.pdl = pw->n > 0;
    }
    const int64_t b0 = c < 0 ? 0 : A->chunk_blk[c];
    const int64_t b1 = c < 0 ? A->chunk_blk[A->n_chunks] : A->chunk_blk[c + 1];
    TailArgs t;
    t.blk = A->d_tail_blk;
    t.warp = A->d_tail_warp;
    t.blk_begin = b0;
    t.blk_end = b1;
    t.out_rows = A->d_tail_out;
    t.col = A->d_tail_col;
    t.val = A->d_tail_val;
    t.x = x;
    t.x_halo = x_halo;
    t.n_loc = e.n_loc;
    t.y = y;
    t.alpha = alpha;
    t.diag = jd;
    t.omega = omega;
    if (c < 0 && A->tail_regions > 0) {  // whole launch: the SM-local persistent schedule
        t.region = A->d_tail_region;
        t.units = A->d_tail_units;
        t.unit_widx = A->d_tail_uwidx;
        t.n_regions = A->tail_regions;
        t.region_ctr = A->d_tail_ctr;
        t.region_done = A->d_tail_ctr + A->tail_regions;
    }
    if (c < 0 && A->d_ring_stage) {  // whole launch: the x-ring schedule
        t.ring_stage = A->d_ring_stage;
        t.ring_unit = A->d_ring_unit;
        t.ring_cta = A->d_ring_cta;
        t.ring_ctas = A->ring_ctas;
    }
    cudaError_t err;
    if (A->tail_conc && c < 0 && !pw && !jd && alpha == 1.0 && beta == 0.0 && !x_halo) {
        // concurrent tail: the tail kernel (sums into tsum) on its own stream
        // beside the ELL kernel, then y[row] += tsum once both are done
        HEC_CUDA_TRY(cudaEventRecord(A->ev_fork, s));
        HEC_CUDA_TRY(cudaStreamWaitEvent(A->s_tail, A->ev_fork, 0));
        t.store_only = true;
        t.tsum = A->d_tsum;
        t.region = nullptr;
        err = launch_tail(t, A->s_tail);
        if (err != cudaSuccess) return cuda_fail(err, "tail_kernel launch");
        HEC_CUDA_TRY(cudaEventRecord(A->ev_join, A->s_tail));
        err = launch_ell(e, s);
        if (err != cudaSuccess) return cuda_fail(err, "ell_kernel launch");
        HEC_CUDA_TRY(cudaStreamWaitEvent(s, A->ev_join, 0));
        err = launch_tail_combine(A->d_tail_out, A->d_tsum, A->tail_rows, y, s);
        return err == cudaSuccess ? HEC_OK : cuda_fail(err, "tail_combine launch");
    }
    if (fused) {
        // small tail, tail first: its row sums go into y, then the ELL kernel
        // (programmatic dependent) adds them -- the same y_i = ell_i + tail_i
        t.store_only = true;
        err = launch_tail(t, s);
        if (err != cudaSuccess) return cuda_fail(err, "tail_kernel launch");
        err = launch_ell(e, s);
        return err == cudaSuccess ? HEC_OK : cuda_fail(err, "ell_kernel launch");
    }
    err = launch_ell(e, s);  // Alg. 1 lines 1-3: ELL first
    if (err != cudaSuccess) return cuda_fail(err, "ell_kernel launch");
    if (A->tail_coo) {                   // HYB comparison variant: COO remainder
        CooArgs k;
        k.nnz = A->tail_nnz;
        k.row = A->d_coo_row;
        k.col = A->d_tail_col;
        k.val = A->d_tail_val;
        k.x = x;
        k.y = y;
        k.alpha = alpha;
        k.diag = jd;
        k.omega = omega;
        err = launch_coo(k, s);
        return err == cudaSuccess ? HEC_OK : cuda_fail(err, "coo_kernel launch");
    }
    if (A->tail_rows > 0 && b1 > b0) {  // Alg. 1 lines 5-7: then the CSR part
        t.reverse = A->tail_reverse;
        err = launch_tail(t, s);
        if (err != cudaSuccess) return cuda_fail(err, "tail_kernel launch");
    }
    return HEC_OK;
}

hec_status launch_spmv(const hec_matrix_s* A, const double* x, const double* x_halo, double* y,
                       cudaStream_t s) {
    return launch_chunks(A, -1, x, x_halo, y, s);
}

hec_status launch_spmv_axpby(const hec_matrix_s* A, double alpha, const double* x, double beta, double* y,
                             cudaStream_t s) {
    return launch_chunks(A, -1, x, nullptr, y, s, alpha, beta);
}

hec_status launch_spmv_peer(const hec_matrix_s* A, const double* x, const double* x_halo, double* y,
                            cudaStream_t s, const PeerWait& w) {
    if (!x_halo) return fail(HEC_ERR_STATE, "peer wait needs a halo");
    return launch_chunks(A, -1, x, x_halo, y, s, 1.0, 0.0, nullptr, nullptr, 0.0, &w);
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

hec_status hec_from_csr_hyb(const hec_csr* A, const hec_opts* o, int32_t device, void* stream,
                            hec_matrix* out) {
    if (!out) return fail(HEC_ERR_ARG, "NULL out");
    *out = nullptr;
    if (device < 0) return fail(HEC_ERR_NODEV, "the HYB comparison variant is device-only");
    CsrView v;
    hec_status st = validate_csr(A, &v);
    if (st != HEC_OK) return st;
    const hec_opts op = normalise_opts(o);
    if ((st = check_opts(op)) != HEC_OK) return st;
    HostHec h;
    try {
        st = convert(v, choose_width(v, op), op.stride_unit, &h);
    } catch (...) {
        return fail(HEC_ERR_NOMEM, "host allocation failed in hec_from_csr_hyb");
    }
    if (st != HEC_OK) return st;
    return make_matrix(std::move(h), device, (cudaStream_t)stream, nullptr, 0, 0, -1, out, true);
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
    o->tail_group = 1 << tail_max_lg();
    o->tail_nnz = A->tail_nnz;
    o->device_bytes = A->device_bytes;
    o->device = A->device;
    o->tail_fused = A->fuse_tile > 0 && A->fuse_tile == 2 * ell_block_threads(A->width) ? 1 : 0;
    o->tail_ring = A->d_ring_stage ? 1 : 0;
    o->ell_idx16 = A->d_ell_d16 ? 1 : 0;
    o->ell_idx16_escaped = A->idx16_esc;
    o->ell_tile_skip = A->tile_skip;
    o->ell_tile_w = A->d_tile_w ? 1 : 0;
    o->ell_grouped = A->d_ell_perm ? 1 : 0;
    o->tail_ring_cover = A->ring_cover;
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
    if (!A->h_ell_perm.empty() && slots) {  // rows grouped by length on the device: back to row order
        const std::vector<int32_t>& p = A->h_ell_perm;
        try {
            std::vector<int32_t> tc(p.size());
            std::vector<double> tv(p.size());
            for (int32_t j = 0; j < A->width; ++j) {
                const size_t b = (size_t)j * A->stride;
                if (o->ell_col) {
                    for (size_t i = 0; i < p.size(); ++i) tc[(size_t)p[i]] = o->ell_col[b + i];
                    std::copy(tc.begin(), tc.end(), o->ell_col + b);
                }
                if (o->ell_val) {
                    for (size_t i = 0; i < p.size(); ++i) tv[(size_t)p[i]] = o->ell_val[b + i];
                    std::copy(tv.begin(), tv.end(), o->ell_val + b);
                }
            }
        } catch (...) {
            return fail(HEC_ERR_NOMEM, "host allocation failed in hec_export");
        }
    }
    if (!A->tail_rows) {
        if (o->tail_ptr) o->tail_ptr[0] = 0;
        return HEC_OK;
    }
    if (A->tail_coo) {  // HYB: remainder kept in the original (row-sorted) order
        if (o->tail_ptr) std::memcpy(o->tail_ptr, A->h_tail_ptr.data(), A->h_tail_ptr.size() * sizeof(int32_t));
        if (o->tail_col) HEC_CUDA_TRY(cudaMemcpy(o->tail_col, A->d_tail_col, A->tail_nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (o->tail_val) HEC_CUDA_TRY(cudaMemcpy(o->tail_val, A->d_tail_val, A->tail_nnz * sizeof(double), cudaMemcpyDeviceToHost));
        return HEC_OK;
    }
    // the device tail is stored in the warp-chunk layout (make_matrix): read it
    // back and walk the same position map to the host CSR order
    std::vector<int32_t> dcol((size_t)A->tail_entries);
    std::vector<double> dval((size_t)A->tail_entries);
    HEC_CUDA_TRY(cudaMemcpy(dcol.data(), A->d_tail_col, dcol.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    HEC_CUDA_TRY(cudaMemcpy(dval.data(), A->d_tail_val, dval.size() * sizeof(double), cudaMemcpyDeviceToHost));
    if (o->tail_ptr) std::memcpy(o->tail_ptr, A->h_tail_ptr.data(), A->h_tail_ptr.size() * sizeof(int32_t));
    for_each_tail_entry(A->h_tail_blk, A->h_tail_warp, A->h_tail_order, A->h_tail_ptr, [&](int64_t pos, int32_t k) {
        if (o->tail_col) o->tail_col[k] = dcol[(size_t)pos];
        if (o->tail_val) o->tail_val[k] = dval[(size_t)pos];
    });
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

hec_status hec_spmv_axpby(hec_matrix A, double alpha, const double* x, double beta, double* y, void* stream) {
    hec_status st = check_xy(A, x, y);
    if (st != HEC_OK) return st;
    if (A->n_rows == 0) return HEC_OK;
    DeviceGuard g(A->device);
    return launch_spmv_axpby(A, alpha, x, beta, y, (cudaStream_t)stream);
}

static bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
    const char* pa = static_cast<const char*>(a);
    const char* pb = static_cast<const char*>(b);
    return a && b && na && nb && pa < pb + nb && pb < pa + na;
}

hec_status hec_diag(hec_matrix A, double* d, void* stream) {
    if (!A) return fail(HEC_ERR_ARG, "NULL matrix");
    if (A->device < 0) return fail(HEC_ERR_NODEV, "host-only matrix handle (device = -1); no CPU fallback");
    if (A->n_rows != A->n_cols || A->n_loc >= 0 || A->d_rowmap || A->row_off)
        return fail(HEC_ERR_DIM, "hec_diag needs a square whole-matrix handle");
    if (A->n_rows == 0) return HEC_OK;
    if (!d) return fail(HEC_ERR_ARG, "NULL d");
    DeviceGuard g(A->device);
    cudaError_t e = launch_diag(A, d, (cudaStream_t)stream);
    return e == cudaSuccess ? HEC_OK : cuda_fail(e, "diag kernel launch");
}

hec_status hec_jacobi(hec_matrix A, const double* d, const double* b, const double* x, double* x_out,
                      double omega, void* stream) {
    if (!A) return fail(HEC_ERR_ARG, "NULL matrix");
    if (A->device < 0) return fail(HEC_ERR_NODEV, "host-only matrix handle (device = -1); no CPU fallback");
    if (A->n_rows != A->n_cols || A->n_loc >= 0 || A->d_rowmap || A->row_off)
        return fail(HEC_ERR_DIM, "hec_jacobi needs a square whole-matrix handle");
    const size_t n = (size_t)A->n_rows;
    if (n == 0) return HEC_OK;
    if (!d || !b || !x || !x_out) return fail(HEC_ERR_ARG, "NULL vector");
    const size_t nb = n * sizeof(double);
    if (overlaps(x_out, nb, x, nb) || overlaps(x_out, nb, b, nb) || overlaps(x_out, nb, d, nb))
        return fail(HEC_ERR_ARG, "x_out overlaps x, b or d");
    DeviceGuard g(A->device);
    return launch_chunks(A, -1, x, nullptr, x_out, (cudaStream_t)stream, 1.0, 0.0, d, b, omega);
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
    const int K = A->n_chunks;
    if (K <= 1) {  // small matrix: copy, compute, copy back
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
    // Pipelined: x arrives in K pieces on s_h2d; row chunk c computes on s as
    // soon as the x prefix it reads (chunk_xend[c]) is resident; its y slice
    // goes back on s_d2h while later chunks compute (PCIe is full duplex).
    // The chunks' ELL rows and tail warp units are exactly those of a whole
    // hec_spmv, so the result is bitwise identical.
    if (!A->s_h2d) {
        HEC_CUDA_TRY(cudaStreamCreateWithFlags(&A->s_h2d, cudaStreamNonBlocking));
        HEC_CUDA_TRY(cudaStreamCreateWithFlags(&A->s_d2h, cudaStreamNonBlocking));
        HEC_CUDA_TRY(cudaEventCreateWithFlags(&A->ev_start, cudaEventDisableTiming));
        A->ev_x.resize(K, nullptr);
        A->ev_y.resize(K, nullptr);
        for (int c = 0; c < K; ++c) {
            HEC_CUDA_TRY(cudaEventCreateWithFlags(&A->ev_x[c], cudaEventDisableTiming));
            HEC_CUDA_TRY(cudaEventCreateWithFlags(&A->ev_y[c], cudaEventDisableTiming));
        }
    }
    // x piece p = the part of the x prefix chunk p needs beyond chunk p-1's
    // (chunk_xend is non-decreasing), so chunk p waits for exactly its piece
    std::vector<int64_t> xb(K + 1);
    xb[0] = 0;
    for (int p = 1; p < K; ++p) xb[p] = std::max<int64_t>(xb[p - 1], std::min<int64_t>(A->chunk_xend[p - 1], A->n_cols));
    xb[K] = A->n_cols;
    HEC_CUDA_TRY(cudaEventRecord(A->ev_start, s));  // ordered after prior work on s
    HEC_CUDA_TRY(cudaStreamWaitEvent(A->s_h2d, A->ev_start, 0));
    HEC_CUDA_TRY(cudaStreamWaitEvent(A->s_d2h, A->ev_start, 0));
    for (int p = 0; p < K; ++p) {
        if (xb[p + 1] > xb[p])
            HEC_CUDA_TRY(cudaMemcpyAsync(A->d_stage_x + xb[p], x_host + xb[p], sizeof(double) * (xb[p + 1] - xb[p]),
                                         cudaMemcpyHostToDevice, A->s_h2d));
        HEC_CUDA_TRY(cudaEventRecord(A->ev_x[p], A->s_h2d));
    }
    int waited = -1;
    for (int c = 0; c < K; ++c) {
        int need = 0;  // last x piece overlapping [0, chunk_xend[c])
        while (need < K - 1 && xb[need + 1] < A->chunk_xend[c]) ++need;
        if (need > waited) {
            HEC_CUDA_TRY(cudaStreamWaitEvent(s, A->ev_x[need], 0));
            waited = need;
        }
        hec_status st = launch_chunks(A, c, A->d_stage_x, nullptr, A->d_stage_y, s);
        if (st != HEC_OK) return st;
        HEC_CUDA_TRY(cudaEventRecord(A->ev_y[c], s));
        HEC_CUDA_TRY(cudaStreamWaitEvent(A->s_d2h, A->ev_y[c], 0));
        const int32_t r0 = A->chunk_row[c], r1 = A->chunk_row[c + 1];
        HEC_CUDA_TRY(cudaMemcpyAsync(y_host + r0, A->d_stage_y + r0, sizeof(double) * (size_t)(r1 - r0),
                                     cudaMemcpyDeviceToHost, A->s_d2h));
    }
    if (waited < K - 1) HEC_CUDA_TRY(cudaStreamWaitEvent(s, A->ev_x[K - 1], 0));  // x buffer reuse order
    HEC_CUDA_TRY(cudaEventRecord(A->ev_start, A->s_d2h));
    HEC_CUDA_TRY(cudaStreamWaitEvent(s, A->ev_start, 0));
    HEC_CUDA_TRY(cudaStreamSynchronize(s));
    return HEC_OK;
}

int32_t hec_spmv_launches(hec_matrix A) {
    if (!A || A->n_rows == 0) return 0;
    return 1 + (A->tail_rows > 0 ? 1 : 0);  // (tail first for small tails: still two launches)
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
