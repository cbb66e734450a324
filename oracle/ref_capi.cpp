// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// C entry points over the REFERENCE's own compiled hot path.  oracle/Makefile
// (target `ref`) compiles the unmodified /root/reference/proj/src/
// factorize.cpp, lapack.cpp and blocks.cpp against the committed minimal
// Eigen / LAPACKE shims (oracle/refshim/) and links them, together with this
// file, into oracle/_ref/librlftn_ref.so (scipy's OpenBLAS 0.3.31).  Python
// front-end: oracle/ref.py.  Only tests/, smoke() and bench.py's CPU legs may
// load it; the product never does.
//
// Besides marshalling, this file restates the reference test helpers that
// build inputs (tests/helpers.hpp:47-88: std::mt19937_64 +
// std::normal_distribution Gaussian draws, Householder-QR isometries,
// A = U diag(sigma) V^H) so acceptance A1/A2 (acceptance.cpp:194-280) can be
// rerun on the very same inputs.  helpers.hpp takes the isometry from Eigen's
// HouseholderQR; here it is the reference's own lapack::orthonormal_columns
// (dgeqrf+dorgqr) -- the same reflector convention (beta = -sign(alpha)|x|),
// so the two agree to rounding.

#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "rlftn/blocks.hpp"
#include "rlftn/factorize.hpp"
#include "rlftn/lapack.hpp"
#include "rlftn/rng.hpp"

extern "C" void scipy_openblas_set_num_threads(int);
extern "C" int scipy_openblas_get_num_threads(void);

// lapack.cpp:15 declares this unprefixed (OpenBLAS' own name); scipy's build
// prefixes it, so forward.
extern "C" void openblas_set_num_threads(int n) { scipy_openblas_set_num_threads(n); }

namespace {

using rlftn::Complex;
using rlftn::Index;
template <class S>
using Mat = rlftn::Matrix<S>;

thread_local std::string g_err;
thread_local rlftn::BlockFactorization<double> g_bf;
thread_local rlftn::BlockFactorization<Complex> g_zbf;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

template <class S>
Mat<S> from_colmajor(const S* a, Index m, Index n, Index lda) {
  Mat<S> out(m, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i) out(i, j) = a[i + j * lda];
  return out;
}

template <class S>
void to_colmajor(const Mat<S>& a, S* dst, Index ld) {
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) dst[i + j * ld] = a(i, j);
}

// Factors written with U m x r (ld m), S r, Vt r x n (ld = ldvt >= r).
template <class S>
void emit(const rlftn::TruncatedFactorization<S>& f, S* U, double* Sg, S* Vt, Index ldvt,
          int64_t* rank, double* dw) {
  const Index r = f.rank();
  if (r > ldvt) throw std::logic_error("ref: output buffers too small");
  to_colmajor(f.left, U, f.left.rows());
  for (Index i = 0; i < r; ++i) Sg[i] = f.sigma[i];
  to_colmajor(f.right_adj, Vt, ldvt);
  *rank = r;
  *dw = f.discarded_weight;
}

template <class S>
int rsvd_t(const S* A, int64_t m, int64_t n, int64_t lda, int64_t k, int64_t ell, int q,
           uint64_t seed, S* U, double* Sg, S* Vt, int64_t ldvt, int64_t* rank, double* dw) {
  return guarded([&] {
    const Mat<S> a = from_colmajor(A, m, n, lda);
    rlftn::RsvdParams p;
    p.rank = k;
    p.oversample = ell;
    p.power = q;
    p.seed = seed;
    emit(rlftn::rsvd(a, p), U, Sg, Vt, ldvt, rank, dw);
  });
}

template <class S>
int tsvd_t(const S* A, int64_t m, int64_t n, int64_t lda, int64_t chi, S* U, double* Sg, S* Vt,
           int64_t ldvt, int64_t* rank, double* dw) {
  return guarded([&] {
    const Mat<S> a = from_colmajor(A, m, n, lda);
    emit(rlftn::tsvd(a, chi), U, Sg, Vt, ldvt, rank, dw);
  });
}

template <class S>
int range_t(const S* A, int64_t m, int64_t n, int64_t lda, int64_t ell, int q, uint64_t seed,
            S* Q) {
  return guarded([&] {
    const Mat<S> a = from_colmajor(A, m, n, lda);
    to_colmajor(rlftn::randomized_range(a, ell, q, seed), Q, m);
  });
}

template <class S>
int recon_t(const S* A, int64_t m, int64_t n, const S* U, const double* Sg, const S* Vt,
            int64_t ldvt, int64_t r, int spectral, double* out) {
  return guarded([&] {
    rlftn::TruncatedFactorization<S> f;
    f.left = from_colmajor(U, m, r, m);
    f.sigma = rlftn::VectorR(r);
    for (Index i = 0; i < r; ++i) f.sigma[i] = Sg[i];
    f.right_adj = from_colmajor(Vt, r, n, ldvt);
    *out = rlftn::reconstruction_error(from_colmajor(A, m, n, m), f,
                                       spectral ? rlftn::ErrorNorm::spectral
                                                : rlftn::ErrorNorm::frobenius);
  });
}

template <class S>
int block_t(rlftn::BlockFactorization<S>& out, int64_t ns, int64_t nc, const int64_t* charges,
            const S* const* blocks, const int64_t* rows, const int64_t* cols, int64_t chi,
            int maximal, int64_t slack, int kind, int64_t oversample, int power, uint64_t seed,
            int64_t min_dim, double* total_dw, int* exact) {
  return guarded([&] {
    rlftn::BlockDiagMatrix<S> a;
    for (int64_t s = 0; s < nc; ++s) a.charges.push_back(static_cast<rlftn::SectorId>(charges[s]));
    for (int64_t s = 0; s < ns; ++s)
      a.blocks.push_back(from_colmajor(blocks[s], rows[s], cols[s], rows[s]));
    rlftn::SectorRankRequest req;
    req.policy = maximal ? rlftn::RankPolicy::maximal : rlftn::RankPolicy::per_sector_estimate;
    req.slack = slack;
    rlftn::BlockMethod method;
    method.kind = kind ? rlftn::BlockMethod::Kind::rsvd : rlftn::BlockMethod::Kind::tsvd;
    method.rsvd.oversample = oversample;
    method.rsvd.power = power;
    method.rsvd.seed = seed;
    method.rsvd_min_dim = min_dim;
    out = rlftn::block_factorize(a, chi, req, method);
    *total_dw = out.discarded_weight;
    *exact = out.discarded_exact ? 1 : 0;
  });
}

template <class S>
int block_sector_t(const rlftn::BlockFactorization<S>& bf, int64_t s, S* U, double* Sg, S* Vt,
                   int64_t* rank, double* dw) {
  return guarded([&] {
    if (s < 0 || s >= static_cast<int64_t>(bf.factors.size()))
      throw std::invalid_argument("ref: sector index out of range");
    const auto& f = bf.factors[static_cast<std::size_t>(s)];
    *rank = f.rank();
    *dw = f.discarded_weight;
    if (U) to_colmajor(f.left, U, f.left.rows());
    if (Sg)
      for (Index i = 0; i < f.rank(); ++i) Sg[i] = f.sigma[i];
    if (Vt) to_colmajor(f.right_adj, Vt, f.rank());
  });
}

// ---- restated reference test helpers (tests/helpers.hpp:47-88) -----------

template <class S>
S random_normal(std::mt19937_64& rng) {  // helpers.hpp:47-56
  std::normal_distribution<double> nd;
  if constexpr (rlftn::is_complex_v<S>) {
    const double re = nd(rng), im = nd(rng);
    return S(re, im) / std::sqrt(2.0);
  } else {
    return nd(rng);
  }
}

template <class S>
Mat<S> gaussian(Index rows, Index cols, std::mt19937_64& rng) {  // helpers.hpp:58-64 (row order)
  Mat<S> a(rows, cols);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j) a(i, j) = random_normal<S>(rng);
  return a;
}

template <class S>
int with_spectrum_t(int64_t rows, int64_t cols, const double* sigma, int64_t k, uint64_t gen_seed,
                    S* out) {
  return guarded([&] {
    if (k > std::min(rows, cols))
      throw std::invalid_argument("matrix_with_spectrum: too many values");
    std::mt19937_64 gen(gen_seed);
    // random_isometry(rows, k) then random_isometry(cols, k) from the same
    // generator (helpers.hpp:79-80); Q of the Householder QR (66-73).
    const Mat<S> u = rlftn::lapack::orthonormal_columns(gaussian<S>(rows, k, gen));
    const Mat<S> v = rlftn::lapack::orthonormal_columns(gaussian<S>(cols, k, gen));
    rlftn::VectorR s(k);
    for (Index i = 0; i < k; ++i) s[i] = sigma[i];
    to_colmajor(Mat<S>((u * s.asDiagonal()) * v.adjoint()), out, rows);
  });
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { scipy_openblas_set_num_threads(n); }
int ref_get_threads() { return scipy_openblas_get_num_threads(); }
void ref_use_single_thread() { rlftn::lapack::use_single_thread(); }  // lapack.cpp:225

uint64_t ref_mix64(uint64_t z) { return rlftn::mix64(z); }
uint64_t ref_derive_seed(uint64_t s, uint64_t t) { return rlftn::derive_seed(s, t); }
void ref_fill_gaussian(uint64_t seed, double* dst, int64_t n) {
  rlftn::CounterRng(seed).fill_gaussian(dst, static_cast<std::size_t>(n));
}
void ref_zfill_gaussian(uint64_t seed, Complex* dst, int64_t n) {
  rlftn::CounterRng(seed).fill_gaussian(dst, static_cast<std::size_t>(n));
}

int ref_rsvd_d(const double* A, int64_t m, int64_t n, int64_t lda, int64_t k, int64_t ell, int q,
               uint64_t seed, double* U, double* S, double* Vt, int64_t ldvt, int64_t* rank,
               double* dw) {
  return rsvd_t(A, m, n, lda, k, ell, q, seed, U, S, Vt, ldvt, rank, dw);
}
int ref_rsvd_z(const Complex* A, int64_t m, int64_t n, int64_t lda, int64_t k, int64_t ell, int q,
               uint64_t seed, Complex* U, double* S, Complex* Vt, int64_t ldvt, int64_t* rank,
               double* dw) {
  return rsvd_t(A, m, n, lda, k, ell, q, seed, U, S, Vt, ldvt, rank, dw);
}
int ref_tsvd_d(const double* A, int64_t m, int64_t n, int64_t lda, int64_t chi, double* U,
               double* S, double* Vt, int64_t ldvt, int64_t* rank, double* dw) {
  return tsvd_t(A, m, n, lda, chi, U, S, Vt, ldvt, rank, dw);
}
int ref_tsvd_z(const Complex* A, int64_t m, int64_t n, int64_t lda, int64_t chi, Complex* U,
               double* S, Complex* Vt, int64_t ldvt, int64_t* rank, double* dw) {
  return tsvd_t(A, m, n, lda, chi, U, S, Vt, ldvt, rank, dw);
}
int ref_randomized_range_d(const double* A, int64_t m, int64_t n, int64_t lda, int64_t ell, int q,
                           uint64_t seed, double* Q) {
  return range_t(A, m, n, lda, ell, q, seed, Q);
}
int ref_randomized_range_z(const Complex* A, int64_t m, int64_t n, int64_t lda, int64_t ell,
                           int q, uint64_t seed, Complex* Q) {
  return range_t(A, m, n, lda, ell, q, seed, Q);
}
int ref_reconstruction_error_d(const double* A, int64_t m, int64_t n, const double* U,
                               const double* S, const double* Vt, int64_t ldvt, int64_t r,
                               int spectral, double* out) {
  return recon_t(A, m, n, U, S, Vt, ldvt, r, spectral, out);
}
int ref_reconstruction_error_z(const Complex* A, int64_t m, int64_t n, const Complex* U,
                               const double* S, const Complex* Vt, int64_t ldvt, int64_t r,
                               int spectral, double* out) {
  return recon_t(A, m, n, U, S, Vt, ldvt, r, spectral, out);
}
int ref_orthonormal_columns_d(const double* A, int64_t m, int64_t n, double* Q) {
  return guarded([&] {
    to_colmajor(rlftn::lapack::orthonormal_columns(from_colmajor(A, m, n, m)), Q, m);
  });
}
int ref_singular_values_d(const double* A, int64_t m, int64_t n, double* s) {
  return guarded([&] {
    const rlftn::VectorR v = rlftn::lapack::singular_values(from_colmajor(A, m, n, m));
    for (Index i = 0; i < v.size(); ++i) s[i] = v[i];
  });
}
int ref_sector_request(int maximal, int64_t chi, int64_t slack, const int64_t* dims, int64_t nd,
                       int64_t* out) {
  return guarded([&] {
    rlftn::SectorRankRequest req;
    req.policy = maximal ? rlftn::RankPolicy::maximal : rlftn::RankPolicy::per_sector_estimate;
    req.chi = chi;
    req.slack = slack;
    std::vector<Index> d(dims, dims + nd);
    const std::vector<Index> r = rlftn::sector_request(req, d);
    for (std::size_t i = 0; i < r.size(); ++i) out[i] = r[i];
  });
}
int ref_block_factorize_d(int64_t ns, int64_t nc, const int64_t* charges, const double* const* blocks,
                          const int64_t* rows, const int64_t* cols, int64_t chi, int maximal,
                          int64_t slack, int kind, int64_t oversample, int power, uint64_t seed,
                          int64_t min_dim, double* total_dw, int* exact) {
  return block_t(g_bf, ns, nc, charges, blocks, rows, cols, chi, maximal, slack, kind, oversample,
                 power, seed, min_dim, total_dw, exact);
}
int ref_block_sector_d(int64_t s, double* U, double* S, double* Vt, int64_t* rank, double* dw) {
  return block_sector_t(g_bf, s, U, S, Vt, rank, dw);
}
int ref_block_factorize_z(int64_t ns, int64_t nc, const int64_t* charges, const Complex* const* blocks,
                          const int64_t* rows, const int64_t* cols, int64_t chi, int maximal,
                          int64_t slack, int kind, int64_t oversample, int power, uint64_t seed,
                          int64_t min_dim, double* total_dw, int* exact) {
  return block_t(g_zbf, ns, nc, charges, blocks, rows, cols, chi, maximal, slack, kind, oversample,
                 power, seed, min_dim, total_dw, exact);
}
int ref_block_sector_z(int64_t s, Complex* U, double* S, Complex* Vt, int64_t* rank, double* dw) {
  return block_sector_t(g_zbf, s, U, S, Vt, rank, dw);
}
int ref_matrix_with_spectrum_d(int64_t rows, int64_t cols, const double* sigma, int64_t k,
                               uint64_t gen_seed, double* out) {
  return with_spectrum_t(rows, cols, sigma, k, gen_seed, out);
}
int ref_matrix_with_spectrum_z(int64_t rows, int64_t cols, const double* sigma, int64_t k,
                               uint64_t gen_seed, Complex* out) {
  return with_spectrum_t(rows, cols, sigma, k, gen_seed, out);
}

}  // extern "C"
