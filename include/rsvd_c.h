/*
 * rsvd_c.h — C ABI of the B200-native randomized truncated SVD engine
 * (librsvd_b200.so, built from paper_1710_01463_b200/csrc/).
 *
 * This is the drop-in boundary for the reference's factorization path
 * (rlftn, /root/reference/proj).  Every entry point names the reference
 * interface it replaces.  Plain pointers and sizes only: no torch or Eigen
 * types cross this boundary.  Matrices are column-major with an explicit
 * leading dimension, the layout of Eigen's default storage that the reference
 * hands to LAPACK (types.hpp:12-13, lapack.cpp:122).
 *
 * Pointers are host or device memory as selected by `flags`
 * (RSVD_PTR_HOST / RSVD_PTR_DEVICE).  With host pointers the call copies in,
 * computes on the handle's stream and copies out before returning.  With
 * device pointers the call is stream-ordered on the handle's stream; scalar
 * outputs (rank, discarded weight) are still returned synchronously.
 *
 * Return codes mirror the reference's exception classes:
 *   RSVD_OK            0
 *   RSVD_ERR_INVALID   1  std::invalid_argument (factorize.cpp:44-45,56-59,79-83)
 *   RSVD_ERR_NUMERICAL 2  std::runtime_error("lapack: ... failed", lapack.cpp:52-55)
 *   RSVD_ERR_CUDA      3  device / driver failure (no reference analogue)
 * rsvd_last_error() returns the message of the handle's last failure, using
 * the reference's wording for the argument errors.
 */
#ifndef RSVD_C_H_
#define RSVD_C_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSVD_OK 0
#define RSVD_ERR_INVALID 1
#define RSVD_ERR_NUMERICAL 2
#define RSVD_ERR_CUDA 3

#define RSVD_PTR_HOST 0
#define RSVD_PTR_DEVICE 1

typedef struct rsvd_context* rsvd_handle;

/* Library / handle lifecycle.  A handle owns the device workspace (grow-only,
 * like the reference's thread_local LAPACK Workspace, lapack.cpp:23-50), a
 * stream and its last-error string.  One handle per host thread (the
 * reference's functions are re-entrant). */
int rsvd_create(rsvd_handle* handle, int device);
int rsvd_destroy(rsvd_handle handle);
const char* rsvd_last_error(rsvd_handle handle);
/* Use a caller-owned cudaStream_t (e.g. torch's current stream); NULL = the
 * handle's own (non-blocking) stream.  Pass cudaStreamLegacy ((void*)1) for
 * the legacy default stream, which torch reports as stream 0. */
int rsvd_set_stream(rsvd_handle handle, void* cuda_stream);
/* Release the cached workspace. */
int rsvd_trim(rsvd_handle handle);
/* Library version string. */
const char* rsvd_version(void);

/* rlftn::mix64 / derive_seed (rng.hpp:11-22). */
uint64_t rsvd_mix64(uint64_t z);
uint64_t rsvd_derive_seed(uint64_t seed, uint64_t tag);

/* rlftn::CounterRng(seed).fill_gaussian(out, count) (rng.hpp:62-64), computed
 * on the device.  64-bit words are bit-exact; normals use the device libm
 * (see DESIGN.md for the measured ulp distance to glibc). */
int rsvd_fill_gaussian_f64(rsvd_handle handle, uint64_t seed, double* out, int64_t count,
                           int flags);

/* rlftn::rsvd<double>(a, RsvdParams{rank, oversample, power, seed})
 * (factorize.hpp:62-63, factorize.cpp:76-95).
 *   oversample is the total sample width l (0 -> min(2*rank, min(m,n)));
 *   U: m x rank (ldu >= m), S: rank, Vt: rank x n (ldvt >= rank).
 *   Only the leading *out_rank columns / values / rows are meaningful; the
 *   rest of the caller's buffers is zeroed.  *discarded_weight is the sum of
 *   squares of the sampled but dropped values (discarded_exact = false). */
int rsvd_f64(rsvd_handle handle, const double* A, int64_t m, int64_t n, int64_t lda,
             int64_t rank, int64_t oversample, int power, uint64_t seed, double* U, int64_t ldu,
             double* S, double* Vt, int64_t ldvt, int64_t* out_rank, double* discarded_weight,
             int flags);

/* Batched rsvd over `batch` independent matrices of one shape (a TEBD layer's
 * disjoint bonds, mps.cpp:448-457; the sector loop of block_factorize,
 * blocks.cpp:60-84).  Matrix b starts at A + b*strideA, U + b*strideU,
 * S + b*strideS, Vt + b*strideVt and uses seeds[b] (host array).
 * out_rank / discarded_weight are host arrays of length batch. */
int rsvd_f64_batched(rsvd_handle handle, int64_t batch, const double* A, int64_t m, int64_t n,
                     int64_t lda, int64_t strideA, int64_t rank, int64_t oversample, int power,
                     const uint64_t* seeds, double* U, int64_t ldu, int64_t strideU, double* S,
                     int64_t strideS, double* Vt, int64_t ldvt, int64_t strideVt,
                     int64_t* out_rank, double* discarded_weight, int flags);

/* Row-sharded rsvd of ONE large matrix over P ranks (C3/C5): this
 * rank holds rows [row_offset, row_offset + m_local) of the m_global x n matrix
 * A (A_local, ld lda) and receives the matching rows of U (U_local, ldu);
 * S and Vt (replicated) and out_rank / discarded_weight are identical on every
 * rank.  The only exchanges are sum all-reduces of the m-side l x l Grams and
 * of the n x l panels A^T Q, through the communicator attached to the handle:
 *   rsvd_attach_nccl   one process per GPU, ncclAllReduce on the handle stream;
 *   rsvd_attach_group  in-process ranks (one host thread + handle each), host
 *                      barriers only — P ranks may share one GPU.
 * Validation follows rsvd with m = m_global. */
typedef struct rsvd_group_s* rsvd_group;
int rsvd_group_create(rsvd_group* group, int nranks);
int rsvd_group_destroy(rsvd_group group);
int rsvd_attach_group(rsvd_handle handle, rsvd_group group, int rank);
int rsvd_nccl_unique_id(unsigned char* id128);
int rsvd_attach_nccl(rsvd_handle handle, int nranks, int rank, const unsigned char* id128);
int rsvd_detach(rsvd_handle handle);
int rsvd_f64_rowsharded(rsvd_handle handle, const double* A_local, int64_t m_local, int64_t n,
                        int64_t lda, int64_t m_global, int64_t row_offset, int64_t rank,
                        int64_t oversample, int power, uint64_t seed, double* U_local,
                        int64_t ldu, double* S, double* Vt, int64_t ldvt, int64_t* out_rank,
                        double* discarded_weight, int flags);

/* rlftn::tsvd<double>(a, chi) (factorize.hpp:49-50, factorize.cpp:42-50): full
 * thin SVD then truncation to r = min(chi, numerical rank) with the EXACT
 * discarded weight (discarded_exact = true).  U: m x min(chi, min(m,n)),
 * S, Vt: min(chi, min(m,n)) x n.  GPU path for min(m, n) <= 1600 (the TEBD
 * sector blocks below rsvd_min_dim and the block_factorize exact route,
 * blocks.cpp:82); larger -> RSVD_ERR_INVALID. */
int rsvd_tsvd_f64(rsvd_handle handle, const double* A, int64_t m, int64_t n, int64_t lda,
                  int64_t chi, double* U, int64_t ldu, double* S, double* Vt, int64_t ldvt,
                  int64_t* out_rank, double* discarded_weight, int flags);
int rsvd_tsvd_f64_batched(rsvd_handle handle, int64_t batch, const double* A, int64_t m,
                          int64_t n, int64_t lda, int64_t strideA, int64_t chi, double* U,
                          int64_t ldu, int64_t strideU, double* S, int64_t strideS, double* Vt,
                          int64_t ldvt, int64_t strideVt, int64_t* out_rank,
                          double* discarded_weight, int flags);

/* rlftn::randomized_range<double>(a, ell, power, seed) (factorize.hpp:56-57,
 * factorize.cpp:52-74): Q (m x ell, ldq >= m) with orthonormal columns
 * spanning the sampled dominant range. */
int rsvd_randomized_range_f64(rsvd_handle handle, const double* A, int64_t m, int64_t n,
                              int64_t lda, int64_t ell, int power, uint64_t seed, double* Q,
                              int64_t ldq, int flags);

/* rlftn::reconstruction_error(a, f, ErrorNorm::frobenius) (factorize.cpp:97-104):
 * ||A - U diag(S) Vt||_F for a rank-r factorization. */
int rsvd_reconstruction_error_f64(rsvd_handle handle, const double* A, int64_t m, int64_t n,
                                  int64_t lda, const double* U, int64_t ldu, const double* S,
                                  const double* Vt, int64_t ldvt, int64_t r, double* out,
                                  int flags);

/* ---- Complex instantiation: Scalar = std::complex<double> ------------------
 * The reference instantiates the same path for Complex (factorize.cpp:106-118:
 * rsvd, tsvd, randomized_range, reconstruction_error over zgemm, zgeqrf+zungqr
 * and zgesdd/zgesvd, lapack.cpp:73-110, 154-177), used by complex TEBD runs
 * (mps.cpp:549-569, cli.cpp:164).  Matrices are std::complex<double> /
 * complex128 column-major, passed as double* to the interleaved (re, im)
 * storage; leading dimensions and strides count COMPLEX elements; S (singular
 * values) and discarded_weight stay real.  Arguments, defaults, errors and
 * messages are those of the double entry points above; Vt is V^H (right_adj).
 * Omega is the reference's complex CounterRng fill (rng.hpp:66-71). */
int rsvd_z128(rsvd_handle handle, const double* A, int64_t m, int64_t n, int64_t lda,
              int64_t rank, int64_t oversample, int power, uint64_t seed, double* U, int64_t ldu,
              double* S, double* Vt, int64_t ldvt, int64_t* out_rank, double* discarded_weight,
              int flags);
int rsvd_z128_batched(rsvd_handle handle, int64_t batch, const double* A, int64_t m, int64_t n,
                      int64_t lda, int64_t strideA, int64_t rank, int64_t oversample, int power,
                      const uint64_t* seeds, double* U, int64_t ldu, int64_t strideU, double* S,
                      int64_t strideS, double* Vt, int64_t ldvt, int64_t strideVt,
                      int64_t* out_rank, double* discarded_weight, int flags);
/* rlftn::tsvd<Complex> (factorize.cpp:42-50); GPU path for min(m, n) <= 1600. */
int rsvd_tsvd_z128(rsvd_handle handle, const double* A, int64_t m, int64_t n, int64_t lda,
                   int64_t chi, double* U, int64_t ldu, double* S, double* Vt, int64_t ldvt,
                   int64_t* out_rank, double* discarded_weight, int flags);
int rsvd_tsvd_z128_batched(rsvd_handle handle, int64_t batch, const double* A, int64_t m,
                           int64_t n, int64_t lda, int64_t strideA, int64_t chi, double* U,
                           int64_t ldu, int64_t strideU, double* S, int64_t strideS, double* Vt,
                           int64_t ldvt, int64_t strideVt, int64_t* out_rank,
                           double* discarded_weight, int flags);
int rsvd_randomized_range_z128(rsvd_handle handle, const double* A, int64_t m, int64_t n,
                               int64_t lda, int64_t ell, int power, uint64_t seed, double* Q,
                               int64_t ldq, int flags);
int rsvd_reconstruction_error_z128(rsvd_handle handle, const double* A, int64_t m, int64_t n,
                                   int64_t lda, const double* U, int64_t ldu, const double* S,
                                   const double* Vt, int64_t ldvt, int64_t r, double* out,
                                   int flags);
/* CounterRng(seed).fill_gaussian(complex<double>*, count) (rng.hpp:66-71):
 * out receives 2 * count doubles. */
int rsvd_fill_gaussian_z128(rsvd_handle handle, uint64_t seed, double* out, int64_t count,
                            int flags);

/* Argument validation of rlftn::rsvd + randomized_range with the reference's
 * order and messages (factorize.cpp:79-83, 56-59); host-only, usable without a
 * GPU.  On success *ell_out is the resolved sample width. */
int rsvd_validate_params(int64_t m, int64_t n, int64_t rank, int64_t oversample, int power,
                         int64_t* ell_out, char* msg, int64_t msg_len);

/* Diagnostics (no reference analogue; the reference only brackets the
 * factorization with steady_clock, mps.cpp:275-277).
 *   rsvd_kernel_launches: engine kernels launched by this process so far.
 *   rsvd_profile_enable:  per-stage CUDA-event timing of subsequent calls.
 *   rsvd_profile_read:    accumulated ms / call counts per stage; returns the
 *                         number of stages (names via rsvd_profile_stage_name).
 *   rsvd_last_jacobi_sweeps: max one-sided Jacobi sweeps of the last rsvd. */
uint64_t rsvd_kernel_launches(void);
int rsvd_profile_enable(rsvd_handle handle, int on);
int rsvd_profile_read(rsvd_handle handle, double* ms, int64_t* calls, int n);
const char* rsvd_profile_stage_name(int i);
int rsvd_last_jacobi_sweeps(rsvd_handle handle);
/* Which FP64 GEMM ran the last rsvd's A-passes: 0 the DMMA (mma.sync .f64)
 * GEMM, 1 the emulated-FP64 GEMM on the INT8 tensor cores (ozaki.cu). */
int rsvd_last_gemm_path(rsvd_handle handle);

/* rlftn::block_factorize<double>(a, chi, request, method) (blocks.cpp:38-118):
 * truncated factorization of a block-diagonal matrix with one dense block per
 * symmetry sector.  Sector s: charge charges[s] (unique), block rows[s] x
 * cols[s] at blocks[s] (column-major, leading dimension ld[s]).
 * Request (SectorRankRequest, blocks.hpp:31-35): policy 0 per_sector_estimate
 * (slack < 0 -> default), 1 maximal.  Method (BlockMethod, blocks.hpp:49-63):
 * kind 0 tsvd / 1 rsvd with oversample (l), power, seed (per-sector seeds
 * derive_seed(seed, charge), blocks.cpp:78) and rsvd_min_dim.  Equal-shape
 * sectors of a route are factorized by one batched engine call.
 * Outputs per sector: out_rank[s] = kept rank after the global top-chi
 * selection; U[s] (ldu[s] >= rows[s]) and Vt[s] (ldvt[s] >= its rank) need
 * room for min(rows[s], cols[s], chi) columns / rows, S[s] for as many values;
 * sector_dw[s] and *total_dw the discarded weights, *exact = discarded_exact.
 * Errors: the reference's messages (blocks.cpp:42-46, 19-24). */
int rsvd_block_factorize_f64(rsvd_handle handle, int64_t nsectors, const int64_t* charges,
                             const double* const* blocks, const int64_t* rows, const int64_t* cols,
                             const int64_t* ld, int64_t chi, int policy, int64_t slack, int kind,
                             int64_t oversample, int power, uint64_t seed, int64_t rsvd_min_dim,
                             double* const* U, const int64_t* ldu, double* const* S,
                             double* const* Vt, const int64_t* ldvt, int64_t* out_rank,
                             double* sector_dw, double* total_dw, int* exact, int flags);

/* ---- TEBD two-site bond update (rlftn::apply_gate, mps.cpp:111-323) ----
 * Table-driven device operations that let a caller assemble theta', measure
 * it and apply the gauge update for a whole layer of disjoint bonds
 * (mps.cpp:448-457) in a few launches.  The tables are HOST arrays (copied
 * by the call); every pointer inside them is DEVICE memory.  Element (i, j)
 * of an operand lives at base[i * rs + j * cs] (strides in elements; a
 * complex element is two interleaved doubles).  `complex_` selects double2
 * elements (the SymmetricMPS<Complex> instantiation, mps.cpp:551-555).
 * Stream-ordered on the handle's stream; nothing is synchronized. */
typedef struct {
  const void* src;
  int64_t rs, cs;
  const double* row_scale; /* optional, NULL = 1: src row i scaled by row_scale[i] */
  const double* col_scale; /* optional, NULL = 1 */
  double coef_re, coef_im; /* coefficient (coef_im ignored for real data) */
} rsvd_block_term;

typedef struct {
  void* dst;
  int64_t rs, cs;
  int64_t rows, cols;
  int64_t term_begin, term_count; /* terms[term_begin .. +term_count) */
} rsvd_block_job;

typedef struct {
  const void* A; int64_t a_rs, a_cs; /* M x K */
  const void* B; int64_t b_rs, b_cs; /* K x N */
  void* C; int64_t c_rs, c_cs;       /* M x N */
  int64_t M, N, K;
} rsvd_gemm_job;

/* dst(i, j) = sum_t coef_t * row_scale_t[i] * col_scale_t[j] * src_t(i, j) for
 * every job (zero when term_count = 0): the lambda-weighted site blocks
 * (mps.cpp:130-137), gate mixing of the (m1, m2) blocks (mps.cpp:205-222),
 * the product form's Kronecker sums x / y (mps.cpp:223-255) and the gauge
 * update (mps.cpp:307-316).  Jobs must not write overlapping elements. */
int rsvd_combine_blocks(rsvd_handle handle, int complex_, int64_t njobs,
                        const rsvd_block_job* jobs, int64_t nterms, const rsvd_block_term* terms);
/* C = A B for every job (independent shapes): theta_mu = Astack Bstack
 * (mps.cpp:164-204), the product form's core r * y (mps.cpp:265) and the
 * lift qfac * left (mps.cpp:301-303). */
int rsvd_grouped_gemm(rsvd_handle handle, int complex_, int64_t njobs, const rsvd_gemm_job* jobs);
/* out[s] (device) = sum of |x|^2 over blocks[slot_begin[s] .. slot_begin[s+1])
 * in table order, bitwise reproducible: ||theta'||^2 per bond (mps.cpp:268).
 * Only dst/rs/cs/rows/cols of the blocks are read. */
int rsvd_block_sqnorms(rsvd_handle handle, int complex_, int64_t nslots, const int64_t* slot_begin,
                       const rsvd_block_job* blocks, double* out);
/* Thin QR, A = Q R for a batch of m x n (m >= n >= 1) matrices: the
 * product-form factor lapack::qr(x, q, r) (mps.cpp:265 -> lapack.cpp:180-201),
 * computed by the engine's CholeskyQR2 (shifted / completed when A is
 * ill-conditioned or rank-deficient, so Q always has n orthonormal columns
 * and A = Q R to working precision).  R is n x n: upper triangular when A
 * has full numerical rank, a column-permuted triangle otherwise. */
int rsvd_qr_f64(rsvd_handle handle, int64_t batch, const double* A, int64_t m, int64_t n,
                int64_t lda, int64_t strideA, double* Q, int64_t ldq, int64_t strideQ, double* R,
                int64_t ldr, int64_t strideR, int flags);

/* Testing hook (not part of the reference surface): the engine's batched FP64
 * GEMM, C = op(A) B, on device pointers; trans_a selects A^T (A stored K x M). */
int rsvd_testing_dgemm(rsvd_handle handle, int trans_a, int64_t M, int64_t N, int64_t K,
                       const double* A, int64_t lda, int64_t strideA, const double* B,
                       int64_t ldb, int64_t strideB, double* C, int64_t ldc, int64_t strideC,
                       int64_t batch);

/* Testing hook: the emulated-FP64 GEMM of the A-passes (Ozaki slices on the
 * INT8 tensor cores), same arguments as rsvd_testing_dgemm.  Needs M, N, K
 * multiples of 16 and K <= 65536 (RSVD_ERR_INVALID otherwise). */
int rsvd_testing_ozaki_gemm(rsvd_handle handle, int trans_a, int64_t M, int64_t N, int64_t K,
                            const double* A, int64_t lda, int64_t strideA, const double* B,
                            int64_t ldb, int64_t strideB, double* C, int64_t ldc, int64_t strideC,
                            int64_t batch);

#ifdef __cplusplus
}
#endif

#endif /* RSVD_C_H_ */
