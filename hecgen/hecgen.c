/*
 * hecgen.c -- seeded synthetic input generators shared by the oracle and the
 * product path.  This module holds NONE of the method's arithmetic (no SpMV,
 * no HEC conversion, no partitioning): it only manufactures CSR matrices and
 * x vectors with the shapes of the paper's workloads.
 *
 * Randomness is a counter-based splitmix64 keyed by (seed, stream, index), so
 * every row can be produced independently and the result does not depend on
 * library versions (SURVEY.md §8(d) "Synthetic inputs").
 *
 * Every generated matrix is canonical CSR: row_ptr[0]=0, non-decreasing,
 * strictly increasing columns per row (§2.1, the Ap/Aj/Ax arrays;
 * int32 indices + fp64 values as pinned by Table 2's Mb(CSR) column).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ---------------------------------------------------------------- RNG ---- */
static inline uint64_t fin64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* ctr(seed, stream, index) = fin(fin(fin(seed) ^ stream) ^ index) */
uint64_t hecgen_ctr(uint64_t seed, uint64_t stream, uint64_t index) {
    return fin64(fin64(fin64(seed) ^ stream) ^ index);
}

/* uniform [0,1) with 53 random bits */
double hecgen_u01(uint64_t seed, uint64_t stream, uint64_t index) {
    return (double)(hecgen_ctr(seed, stream, index) >> 11) * 0x1.0p-53;
}

/* stream identifiers (small constants, documented in DESIGN.md) */
enum {
    ST_X = 0, ST_INACT = 1, ST_PERM = 2, ST_LEN = 3, ST_COL = 4, ST_VAL = 5,
    ST_XINT = 6, ST_RAND = 7
};

/* ------------------------------------------------------------ vectors ---- */
/* kind 0: U[-1,1): x_j = 2*(ctr(seed,0,j)>>11)*2^-53 - 1 (SURVEY §8(d) default)
 * kind 1: ones
 * kind 2: integers uniform in [-2^20, 2^20] (integer-exact regime, pin P3)   */
int hecgen_vector(int64_t n, int kind, uint64_t seed, double* x) {
    if (n < 0 || (n > 0 && !x)) return 1;
    for (int64_t j = 0; j < n; ++j) {
        if (kind == 0) {
            x[j] = 2.0 * hecgen_u01(seed, ST_X, (uint64_t)j) - 1.0;
        } else if (kind == 1) {
            x[j] = 1.0;
        } else if (kind == 2) {
            uint64_t r = hecgen_ctr(seed, ST_XINT, (uint64_t)j) % ((1ULL << 21) + 1ULL);
            x[j] = (double)((int64_t)r - (int64_t)(1LL << 20));
        } else {
            return 1;
        }
    }
    return 0;
}

/* ------------------------------------------------------- 2D / 3D grids ---- */
/* nnz of the 7-point stencil with Dirichlet truncation:
 * 7n - 2(ny*nz + nx*nz + nx*ny) (matches PAPER P:406) -- but
 * here computed by counting, the closed form is a test pin. */
int64_t hecgen_poisson3d_nnz(int32_t nx, int32_t ny, int32_t nz) {
    if (nx < 1 || ny < 1 || nz < 1) return -1;
    int64_t nnz = 0;
    for (int32_t k = 0; k < nz; ++k)
        for (int32_t j = 0; j < ny; ++j)
            for (int32_t i = 0; i < nx; ++i)
                nnz += 1 + (k > 0) + (j > 0) + (i > 0) + (i < nx - 1) + (j < ny - 1) + (k < nz - 1);
    return nnz;
}

/* 3D 7-point Laplacian, natural order r = i + nx*(j + ny*k), diagonal 6,
 * off-diagonals -1, Dirichlet truncation (PAPER §3.1 3D_Poisson). */
int hecgen_poisson3d(int32_t nx, int32_t ny, int32_t nz,
                     int32_t* row_ptr, int32_t* col, double* val) {
    if (nx < 1 || ny < 1 || nz < 1) return 1;
    const int64_t pxy = (int64_t)nx * ny;
    int64_t p = 0, r = 0;
    row_ptr[0] = 0;
    for (int32_t k = 0; k < nz; ++k)
        for (int32_t j = 0; j < ny; ++j)
            for (int32_t i = 0; i < nx; ++i, ++r) {
                if (k > 0)      { col[p] = (int32_t)(r - pxy); val[p++] = -1.0; }
                if (j > 0)      { col[p] = (int32_t)(r - nx);  val[p++] = -1.0; }
                if (i > 0)      { col[p] = (int32_t)(r - 1);   val[p++] = -1.0; }
                col[p] = (int32_t)r; val[p++] = 6.0;
                if (i < nx - 1) { col[p] = (int32_t)(r + 1);   val[p++] = -1.0; }
                if (j < ny - 1) { col[p] = (int32_t)(r + nx);  val[p++] = -1.0; }
                if (k < nz - 1) { col[p] = (int32_t)(r + pxy); val[p++] = -1.0; }
                row_ptr[r + 1] = (int32_t)p;
            }
    return 0;
}

int64_t hecgen_poisson2d_nnz(int32_t nx, int32_t ny) {
    if (nx < 1 || ny < 1) return -1;
    int64_t nnz = 0;
    for (int32_t j = 0; j < ny; ++j)
        for (int32_t i = 0; i < nx; ++i)
            nnz += 1 + (j > 0) + (i > 0) + (i < nx - 1) + (j < ny - 1);
    return nnz;
}

/* 2D 5-point Laplacian, natural order r = i + nx*j, diagonal 4, off -1. */
int hecgen_poisson2d(int32_t nx, int32_t ny, int32_t* row_ptr, int32_t* col, double* val) {
    if (nx < 1 || ny < 1) return 1;
    int64_t p = 0, r = 0;
    row_ptr[0] = 0;
    for (int32_t j = 0; j < ny; ++j)
        for (int32_t i = 0; i < nx; ++i, ++r) {
            if (j > 0)      { col[p] = (int32_t)(r - nx); val[p++] = -1.0; }
            if (i > 0)      { col[p] = (int32_t)(r - 1);  val[p++] = -1.0; }
            col[p] = (int32_t)r; val[p++] = 4.0;
            if (i < nx - 1) { col[p] = (int32_t)(r + 1);  val[p++] = -1.0; }
            if (j < ny - 1) { col[p] = (int32_t)(r + nx); val[p++] = -1.0; }
            row_ptr[r + 1] = (int32_t)p;
        }
    return 0;
}

/* --------------------------------------------------------- power law ---- */
/* Row length L_i: truncated discrete power law on [lmin, lmax] with exponent
 * alpha, by inverse CDF on U(seed, ST_LEN, i).  Lengths are clamped to n. */
typedef struct { int32_t lmin, lmax; double* cdf; } pl_table;

static int pl_make(pl_table* t, int32_t lmin, int32_t lmax, double alpha) {
    t->lmin = lmin; t->lmax = lmax;
    int32_t m = lmax - lmin + 1;
    t->cdf = (double*)malloc(sizeof(double) * (size_t)m);
    if (!t->cdf) return 1;
    double s = 0.0;
    for (int32_t k = 0; k < m; ++k) { s += pow((double)(lmin + k), -alpha); t->cdf[k] = s; }
    for (int32_t k = 0; k < m; ++k) t->cdf[k] /= s;
    t->cdf[m - 1] = 1.0;
    return 0;
}

static int32_t pl_draw(const pl_table* t, double u) {
    int32_t lo = 0, hi = t->lmax - t->lmin;       /* smallest k with cdf[k] > u */
    while (lo < hi) { int32_t mid = (lo + hi) / 2; if (t->cdf[mid] > u) hi = mid; else lo = mid + 1; }
    return t->lmin + lo;
}

/* Pass 1: row_ptr only. Returns nnz (or -1). */
int64_t hecgen_powerlaw_rowptr(int32_t n, int32_t lmin, int32_t lmax, double alpha,
                               uint64_t seed, int32_t* row_ptr) {
    if (n < 1 || lmin < 1 || lmax < lmin) return -1;
    pl_table t;
    if (pl_make(&t, lmin, lmax, alpha)) return -1;
    int64_t p = 0;
    row_ptr[0] = 0;
    for (int32_t i = 0; i < n; ++i) {
        int32_t L = pl_draw(&t, hecgen_u01(seed, ST_LEN, (uint64_t)i));
        if (L > n) L = n;
        p += L;
        if (p > INT32_MAX) { free(t.cdf); return -1; }
        row_ptr[i + 1] = (int32_t)p;
    }
    free(t.cdf);
    return p;
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* Pass 2: columns and values given row_ptr from pass 1.
 * Row i holds the diagonal plus L_i-1 distinct columns; each draw is local
 * (p_local) at i+delta, delta uniform in +-[1, band], clipped to [0,n), else
 * global uniform on [0,n).  Collisions are redrawn; the row is then sorted.
 * Values: off-diagonal U[-1,1), diagonal 1 + sum|off| (diagonally dominant);
 * integer option: off-diagonal uniform in [-8,8]\{0}, diagonal 1. */
int hecgen_powerlaw_fill(int32_t n, int32_t band, double p_local, int integer_values,
                         uint64_t seed, const int32_t* row_ptr, int32_t* col, double* val) {
    if (n < 1 || band < 1) return 1;
    for (int32_t i = 0; i < n; ++i) {
        const int64_t b = row_ptr[i];
        const int32_t L = row_ptr[i + 1] - row_ptr[i];
        int32_t* c = col + b;
        int32_t have = 0;
        uint64_t attempt = 0;
        if (L == 0) continue;
        c[have++] = i;
        while (have < L) {
            int32_t need = L - have;
            for (int32_t d = 0; d < need; ++d, ++attempt) {
                uint64_t key = ((uint64_t)(uint32_t)i << 24) ^ attempt;  /* attempt < 2^24 */
                double u = hecgen_u01(seed, ST_COL, 2 * key);
                uint64_t r = hecgen_ctr(seed, ST_COL, 2 * key + 1);
                int64_t j;
                /* after 16 L attempts the band is exhausted (p_local = 1 and L >
                 * 2 band + 1): draw globally so the row always completes */
                if (u < p_local && attempt < 16 * (uint64_t)L) {
                    int64_t delta = 1 + (int64_t)(r % (uint64_t)band);
                    if ((r >> 32) & 1) delta = -delta;
                    j = (int64_t)i + delta;
                    if (j < 0) j = 0;
                    if (j >= n) j = n - 1;
                } else {
                    j = (int64_t)(r % (uint64_t)n);
                }
                c[have + d] = (int32_t)j;
            }
            have = L;
            qsort(c, (size_t)have, sizeof(int32_t), cmp_i32);
            int32_t u = 0;
            for (int32_t k = 0; k < have; ++k)
                if (u == 0 || c[k] != c[u - 1]) c[u++] = c[k];
            have = u;
        }
        /* values */
        double s = 0.0;
        int32_t diag = -1;
        for (int32_t k = 0; k < L; ++k) {
            if (c[k] == i) { diag = k; continue; }
            double v;
            uint64_t vk = (uint64_t)(b + k);
            if (integer_values) {
                int64_t q = (int64_t)(hecgen_ctr(seed, ST_VAL, vk) % 16ULL) - 8;  /* -8..7 */
                if (q >= 0) q += 1;                                                 /* -8..-1,1..8 */
                v = (double)q;
            } else {
                v = 2.0 * hecgen_u01(seed, ST_VAL, vk) - 1.0;
            }
            val[b + k] = v;
            s += fabs(v);
        }
        val[b + diag] = integer_values ? 1.0 : 1.0 + s;
    }
    return 0;
}

/* Degree-sorted stress variant (SURVEY §8(d) power-law recipe): B = P A P^T
 * with rows in descending length order, ties by ascending original row
 * (stable), i.e. perm[r] = the original row placed at r, and every column
 * renamed j -> inv[j] then re-sorted within its row (values move with their
 * columns).  Square A only.  Output arrays sized like A's. */
typedef struct { int32_t c; int32_t k; } hg_ck;
static int cmp_ck(const void* a, const void* b) {
    int32_t x = ((const hg_ck*)a)->c, y = ((const hg_ck*)b)->c;
    return (x > y) - (x < y);
}

int hecgen_degree_sort(int32_t n, const int32_t* row_ptr, const int32_t* col, const double* val,
                       int32_t* perm, int32_t* out_rp, int32_t* out_col, double* out_val) {
    if (n < 1) return 1;
    int32_t lmax = 0;
    for (int32_t i = 0; i < n; ++i) {
        int32_t L = row_ptr[i + 1] - row_ptr[i];
        if (L > lmax) lmax = L;
    }
    /* counting sort by descending length, stable */
    int64_t* start = calloc((size_t)lmax + 2, sizeof(int64_t));
    int32_t* inv = malloc(sizeof(int32_t) * (size_t)n);
    hg_ck* buf = malloc(sizeof(hg_ck) * ((size_t)lmax + 1));
    if (!start || !inv || !buf) { free(start); free(inv); free(buf); return 2; }
    for (int32_t i = 0; i < n; ++i) start[lmax - (row_ptr[i + 1] - row_ptr[i]) + 1]++;
    for (int32_t l = 1; l <= lmax + 1; ++l) start[l] += start[l - 1];
    for (int32_t i = 0; i < n; ++i) {
        int64_t r = start[lmax - (row_ptr[i + 1] - row_ptr[i])]++;
        perm[r] = i;
        inv[i] = (int32_t)r;
    }
    out_rp[0] = 0;
    for (int32_t r = 0; r < n; ++r) {
        const int32_t i = perm[r];
        const int32_t b = row_ptr[i], L = row_ptr[i + 1] - b;
        for (int32_t k = 0; k < L; ++k) { buf[k].c = inv[col[b + k]]; buf[k].k = b + k; }
        qsort(buf, (size_t)L, sizeof(hg_ck), cmp_ck);
        const int32_t o = out_rp[r];
        for (int32_t k = 0; k < L; ++k) { out_col[o + k] = buf[k].c; out_val[o + k] = val[buf[k].k]; }
        out_rp[r + 1] = o + L;
    }
    free(start); free(inv); free(buf);
    return 0;
}

/* ------------------------------------------------------ SPE10-shaped ---- */
/* 60 x 220 x 85 grid (SURVEY §8(d) "SPE10 recipe"), cells inactive with
 * probability p_inact, log-permeability from seeded smooth fields (Tarbert-like
 * layers k < nz_top, channelised Upper-Ness-like below), TPFA transmissibility
 * T = 2/(1/k_a + 1/k_b) * (A/Delta) between active face neighbours, a small
 * accumulation term on the diagonal, and 5 fully perforated wells appended as
 * extra unknowns coupled symmetrically with WI = wi_scale * k_cell. */
typedef struct {
    int32_t nx, ny, nz, nz_top, n_wells;
    double p_inact;
    uint64_t seed;
    int32_t wx[5], wy[5];
} spe_params;

static void spe_default(spe_params* p, int32_t nx, int32_t ny, int32_t nz, uint64_t seed) {
    p->nx = nx; p->ny = ny; p->nz = nz;
    p->nz_top = (nz * 35) / 85;
    p->p_inact = 0.02; p->seed = seed; p->n_wells = 5;
    p->wx[0] = nx / 2 - 1 < 0 ? 0 : nx / 2 - 1; p->wy[0] = ny / 2 - 1 < 0 ? 0 : ny / 2 - 1;  /* injector (29,109) at 60x220 */
    p->wx[1] = 0;      p->wy[1] = 0;
    p->wx[2] = nx - 1; p->wy[2] = 0;
    p->wx[3] = 0;      p->wy[3] = ny - 1;
    p->wx[4] = nx - 1; p->wy[4] = ny - 1;
}

static double spe_logk(const spe_params* p, int32_t i, int32_t j, int32_t k) {
    const double PI = 3.14159265358979323846;
    double g = 0.0;
    int layer_group = (k < p->nz_top) ? 0 : 1;
    for (int m = 0; m < 8; ++m) {
        uint64_t base = (uint64_t)(layer_group * 64 + m * 8);
        double fx = 0.5 + 3.5 * hecgen_u01(p->seed, ST_PERM, base + 0);
        double fy = 0.5 + 6.0 * hecgen_u01(p->seed, ST_PERM, base + 1);
        double fz = 0.5 + 2.0 * hecgen_u01(p->seed, ST_PERM, base + 2);
        double ph = 2.0 * PI * hecgen_u01(p->seed, ST_PERM, base + 3);
        g += cos(2.0 * PI * (fx * i / p->nx + fy * j / p->ny + fz * k / p->nz) + ph);
    }
    g *= 0.5;   /* sum of 8 unit cosines has std 2; scale to ~1 */
    if (layer_group == 0) return log(100.0) + 1.5 * g;
    /* channelised: sinuous bands along y */
    double amp = 4.0 + 4.0 * hecgen_u01(p->seed, ST_PERM, 1000 + (uint64_t)k);
    double lam = 40.0 + 60.0 * hecgen_u01(p->seed, ST_PERM, 2000 + (uint64_t)k);
    double ph = 2.0 * PI * hecgen_u01(p->seed, ST_PERM, 3000 + (uint64_t)k);
    double c0 = p->nx * (0.2 + 0.6 * hecgen_u01(p->seed, ST_PERM, 4000 + (uint64_t)k));
    double centre = c0 + amp * sin(2.0 * PI * j / lam + ph);
    int channel = fabs((double)i - centre) < 4.0;
    return channel ? log(2000.0) + 1.0 * g : log(0.01) + 2.5 * g;
}

/* Builds the whole matrix into malloc'ed arrays (caller frees with hecgen_free). */
int hecgen_spe10(int32_t nx, int32_t ny, int32_t nz, uint64_t seed,
                 int32_t* n_out, int64_t* nnz_out,
                 int32_t** row_ptr_out, int32_t** col_out, double** val_out) {
    if (nx < 2 || ny < 2 || nz < 1) return 1;
    spe_params P; spe_default(&P, nx, ny, nz, seed);
    const int64_t nc = (int64_t)nx * ny * nz;
    int32_t* id = (int32_t*)malloc(sizeof(int32_t) * (size_t)nc);
    double* kk = (double*)malloc(sizeof(double) * (size_t)nc);
    if (!id || !kk) { free(id); free(kk); return 2; }
    int32_t na = 0;
    for (int64_t c = 0; c < nc; ++c) {
        int32_t i = (int32_t)(c % nx), j = (int32_t)((c / nx) % ny), k = (int32_t)(c / ((int64_t)nx * ny));
        int inactive = hecgen_u01(seed, ST_INACT, (uint64_t)c) < P.p_inact;
        for (int w = 0; w < P.n_wells; ++w)   /* perforated cells stay active */
            if (i == P.wx[w] && j == P.wy[w]) inactive = 0;
        id[c] = inactive ? -1 : na++;
        kk[c] = exp(spe_logk(&P, i, j, k));
    }
    const int32_t n = na + P.n_wells;
    /* neighbours: -z, -y, -x, +x, +y, +z in that (ascending column) order;
     * face factors A/Delta: x 20*... with dx=20, dy=10, dz=2 */
    const double fac[3] = { (10.0 * 2.0) / 20.0, (20.0 * 2.0) / 10.0, (20.0 * 10.0) / 2.0 };
    const double wi_scale = 0.05;
    /* count + transmissibility mean */
    int64_t nnz = 0; double tsum = 0.0; int64_t tcnt = 0;
    int32_t* rp = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    if (!rp) { free(id); free(kk); return 2; }
    rp[0] = 0;
    int32_t r = 0;
    int32_t wcount[5] = {0, 0, 0, 0, 0};
    for (int64_t c = 0; c < nc; ++c) {
        if (id[c] < 0) continue;
        int32_t i = (int32_t)(c % nx), j = (int32_t)((c / nx) % ny), k = (int32_t)(c / ((int64_t)nx * ny));
        int64_t nb[6] = { k > 0 ? c - (int64_t)nx * ny : -1, j > 0 ? c - nx : -1, i > 0 ? c - 1 : -1,
                          i < nx - 1 ? c + 1 : -1, j < ny - 1 ? c + nx : -1, k < nz - 1 ? c + (int64_t)nx * ny : -1 };
        int32_t cnt = 1;
        for (int d = 0; d < 6; ++d) {
            if (nb[d] < 0 || id[nb[d]] < 0) continue;
            ++cnt;
            double t = 2.0 / (1.0 / kk[c] + 1.0 / kk[nb[d]]) * fac[d < 3 ? 2 - d : d - 3];
            tsum += t; ++tcnt;
        }
        for (int w = 0; w < P.n_wells; ++w)
            if (i == P.wx[w] && j == P.wy[w]) { ++cnt; ++wcount[w]; }
        nnz += cnt;
        rp[++r] = (int32_t)nnz;
    }
    for (int w = 0; w < P.n_wells; ++w) { nnz += 1 + wcount[w]; rp[++r] = (int32_t)nnz; }
    const double acc = 1e-3 * (tcnt ? tsum / (double)tcnt : 1.0);
    int32_t* col = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
    double* val = (double*)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
    double* wdiag = (double*)calloc((size_t)P.n_wells, sizeof(double));
    if (!col || !val || !wdiag) { free(id); free(kk); free(rp); free(col); free(val); free(wdiag); return 2; }
    /* well rows: collect (cell id, WI) in cell order (ascending column) */
    int32_t** wcol = (int32_t**)calloc((size_t)P.n_wells, sizeof(int32_t*));
    double** wval = (double**)calloc((size_t)P.n_wells, sizeof(double*));
    for (int w = 0; w < P.n_wells; ++w) {
        wcol[w] = (int32_t*)malloc(sizeof(int32_t) * (size_t)(wcount[w] + 1));
        wval[w] = (double*)malloc(sizeof(double) * (size_t)(wcount[w] + 1));
        wcount[w] = 0;
    }
    int64_t p = 0;
    for (int64_t c = 0; c < nc; ++c) {
        if (id[c] < 0) continue;
        int32_t i = (int32_t)(c % nx), j = (int32_t)((c / nx) % ny), k = (int32_t)(c / ((int64_t)nx * ny));
        int64_t nb[6] = { k > 0 ? c - (int64_t)nx * ny : -1, j > 0 ? c - nx : -1, i > 0 ? c - 1 : -1,
                          i < nx - 1 ? c + 1 : -1, j < ny - 1 ? c + nx : -1, k < nz - 1 ? c + (int64_t)nx * ny : -1 };
        double diag = acc;
        int64_t pdiag = -1;
        for (int d = 0; d < 6; ++d) {
            if (d == 3) { pdiag = p; col[p] = id[c]; val[p++] = 0.0; }
            if (nb[d] < 0 || id[nb[d]] < 0) continue;
            double t = 2.0 / (1.0 / kk[c] + 1.0 / kk[nb[d]]) * fac[d < 3 ? 2 - d : d - 3];
            col[p] = id[nb[d]]; val[p++] = -t; diag += t;
        }
        for (int w = 0; w < P.n_wells; ++w)
            if (i == P.wx[w] && j == P.wy[w]) {
                double wi = wi_scale * kk[c];
                col[p] = na + w; val[p++] = -wi; diag += wi;
                wcol[w][wcount[w]] = id[c]; wval[w][wcount[w]] = -wi; wcount[w]++;
                wdiag[w] += wi;
            }
        val[pdiag] = diag;
    }
    for (int w = 0; w < P.n_wells; ++w) {
        for (int32_t q = 0; q < wcount[w]; ++q) { col[p] = wcol[w][q]; val[p++] = wval[w][q]; }
        col[p] = na + w; val[p++] = wdiag[w] + acc;
        free(wcol[w]); free(wval[w]);
    }
    free(wcol); free(wval); free(wdiag); free(id); free(kk);
    *n_out = n; *nnz_out = nnz; *row_ptr_out = rp; *col_out = col; *val_out = val;
    return 0;
}

/* -------------------------------------------------- small random CSR ---- */
/* Random sparse matrix for brute-force tests: each (i,j) present with
 * probability density; values integer in [-8,8] (integer_values) or U[-1,1). */
int64_t hecgen_random_rowptr(int32_t n_rows, int32_t n_cols, double density, uint64_t seed, int32_t* row_ptr) {
    int64_t p = 0;
    row_ptr[0] = 0;
    for (int32_t i = 0; i < n_rows; ++i) {
        for (int32_t j = 0; j < n_cols; ++j)
            if (hecgen_u01(seed, ST_RAND, (uint64_t)i * (uint64_t)n_cols + (uint64_t)j) < density) ++p;
        row_ptr[i + 1] = (int32_t)p;
    }
    return p;
}

int hecgen_random_fill(int32_t n_rows, int32_t n_cols, double density, int integer_values,
                       uint64_t seed, const int32_t* row_ptr, int32_t* col, double* val) {
    for (int32_t i = 0; i < n_rows; ++i) {
        int64_t p = row_ptr[i];
        for (int32_t j = 0; j < n_cols; ++j) {
            uint64_t key = (uint64_t)i * (uint64_t)n_cols + (uint64_t)j;
            if (hecgen_u01(seed, ST_RAND, key) < density) {
                col[p] = j;
                if (integer_values) val[p] = (double)((int64_t)(hecgen_ctr(seed, ST_VAL, key) % 17ULL) - 8);
                else val[p] = 2.0 * hecgen_u01(seed, ST_VAL, key) - 1.0;
                ++p;
            }
        }
    }
    return 0;
}

void hecgen_free(void* p) { free(p); }

/* FNV-1a 64 over raw bytes, for logging input identity. */
uint64_t hecgen_fnv1a(const void* data, int64_t nbytes, uint64_t h) {
    const unsigned char* b = (const unsigned char*)data;
    if (h == 0) h = 0xcbf29ce484222325ULL;
    for (int64_t i = 0; i < nbytes; ++i) { h ^= b[i]; h *= 0x100000001b3ULL; }
    return h;
}
