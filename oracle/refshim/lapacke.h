/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Minimal <lapacke.h> for compiling the reference's unmodified
 * proj/src/lapack.cpp (which includes it at lapack.cpp:3-7 after defining
 * LAPACK_COMPLEX_CUSTOM / lapack_complex_double).  No lapacke.h ships in this
 * image; the LAPACKE *_work drivers the reference calls are exported (with a
 * `scipy_` prefix, LP64) by scipy's OpenBLAS 0.3.31, so each name is mapped
 * onto that symbol and declared with the standard LAPACKE prototype.
 */
#pragma once

#include <complex>

#ifndef lapack_int
#define lapack_int int
#endif
#ifndef lapack_complex_double
#define lapack_complex_double std::complex<double>
#endif

#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102

#define LAPACKE_dgesdd_work scipy_LAPACKE_dgesdd_work
#define LAPACKE_dgesvd_work scipy_LAPACKE_dgesvd_work
#define LAPACKE_dgeqrf_work scipy_LAPACKE_dgeqrf_work
#define LAPACKE_dorgqr_work scipy_LAPACKE_dorgqr_work
#define LAPACKE_zgesdd_work scipy_LAPACKE_zgesdd_work
#define LAPACKE_zgesvd_work scipy_LAPACKE_zgesvd_work
#define LAPACKE_zgeqrf_work scipy_LAPACKE_zgeqrf_work
#define LAPACKE_zungqr_work scipy_LAPACKE_zungqr_work

extern "C" {
lapack_int LAPACKE_dgesdd_work(int matrix_layout, char jobz, lapack_int m, lapack_int n, double* a,
                               lapack_int lda, double* s, double* u, lapack_int ldu, double* vt,
                               lapack_int ldvt, double* work, lapack_int lwork, lapack_int* iwork);
lapack_int LAPACKE_dgesvd_work(int matrix_layout, char jobu, char jobvt, lapack_int m,
                               lapack_int n, double* a, lapack_int lda, double* s, double* u,
                               lapack_int ldu, double* vt, lapack_int ldvt, double* work,
                               lapack_int lwork);
lapack_int LAPACKE_dgeqrf_work(int matrix_layout, lapack_int m, lapack_int n, double* a,
                               lapack_int lda, double* tau, double* work, lapack_int lwork);
lapack_int LAPACKE_dorgqr_work(int matrix_layout, lapack_int m, lapack_int n, lapack_int k,
                               double* a, lapack_int lda, const double* tau, double* work,
                               lapack_int lwork);
lapack_int LAPACKE_zgesdd_work(int matrix_layout, char jobz, lapack_int m, lapack_int n,
                               lapack_complex_double* a, lapack_int lda, double* s,
                               lapack_complex_double* u, lapack_int ldu,
                               lapack_complex_double* vt, lapack_int ldvt,
                               lapack_complex_double* work, lapack_int lwork, double* rwork,
                               lapack_int* iwork);
lapack_int LAPACKE_zgesvd_work(int matrix_layout, char jobu, char jobvt, lapack_int m,
                               lapack_int n, lapack_complex_double* a, lapack_int lda, double* s,
                               lapack_complex_double* u, lapack_int ldu,
                               lapack_complex_double* vt, lapack_int ldvt,
                               lapack_complex_double* work, lapack_int lwork, double* rwork);
lapack_int LAPACKE_zgeqrf_work(int matrix_layout, lapack_int m, lapack_int n,
                               lapack_complex_double* a, lapack_int lda, lapack_complex_double* tau,
                               lapack_complex_double* work, lapack_int lwork);
lapack_int LAPACKE_zungqr_work(int matrix_layout, lapack_int m, lapack_int n, lapack_int k,
                               lapack_complex_double* a, lapack_int lda,
                               const lapack_complex_double* tau, lapack_complex_double* work,
                               lapack_int lwork);
}
