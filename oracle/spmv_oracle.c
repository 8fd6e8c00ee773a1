/*
 * spmv_oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain serial CPU definition
 * of y = A x for a CSR matrix.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library; the
 * product path (paper_1606_00545_b200) never does.
 *
 * It shares no code with the CUDA path.  Built with
 *   gcc -O2 -ffp-contract=off -fno-fast-math
 * so that every product is rounded and then added (no FMA contraction).
 *
 * O1:  for i in [r0,r1): s = +0.0;
 *        for k in [row_ptr[i], row_ptr[i+1]): s = s + val[k]*x[col[k]];  y[i] = s
 *     This is the plain definition of the matrix-vector product the paper
 *     computes (Eq. (1); Alg. 1 is a re-organised evaluation
 *     of the same sums), taken row by row in column order.
 * O1' r_i = sum_k |val[k]| * |x[col[k]]|, the scale of the parity tolerance
 *     tau_i = 1e-12 * r_i (BASELINE.json north_star).
 * O1p the same O1 loop with its rows split over host threads (OpenMP static
 *     schedule; SURVEY.md §8(d) CPU timing (ii)).  Each row is still summed by
 *     one thread in column order, so the result is bit-identical to O1; it is
 *     used only to time a parallel CPU baseline.
 */
#include <stdint.h>
#include <math.h>
#include <omp.h>

void oracle_csr_spmv(int32_t r0, int32_t r1, const int32_t* row_ptr, const int32_t* col,
                     const double* val, const double* x, double* y) {
    for (int32_t i = r0; i < r1; ++i) {
        double s = 0.0;
        for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            double prod = val[k] * x[col[k]];
            s = s + prod;
        }
        y[i - r0] = s;
    }
}

void oracle_csr_absmv(int32_t r0, int32_t r1, const int32_t* row_ptr, const int32_t* col,
                      const double* val, const double* x, double* r) {
    for (int32_t i = r0; i < r1; ++i) {
        double s = 0.0;
        for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            double prod = fabs(val[k]) * fabs(x[col[k]]);
            s = s + prod;
        }
        r[i - r0] = s;
    }
}

int oracle_csr_spmv_omp(int32_t r0, int32_t r1, const int32_t* row_ptr, const int32_t* col,
                        const double* val, const double* x, double* y) {
    int threads = 1;
#pragma omp parallel
    {
#pragma omp single
        threads = omp_get_num_threads();
#pragma omp for schedule(static)
        for (int32_t i = r0; i < r1; ++i) {
            double s = 0.0;
            for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
                double prod = val[k] * x[col[k]];
                s = s + prod;
            }
            y[i - r0] = s;
        }
    }
    return threads;
}
