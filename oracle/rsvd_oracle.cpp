// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference randomized truncated SVD path
// (rlftn::rsvd and everything it calls).  Only tests/, __graft_entry__.smoke()
// and bench.py's CPU-baseline / reference arm may load this library, and only
// as the checker or the timed CPU baseline; the product path
// (paper_1710_01463_b200, librsvd_b200.so) never links or calls it.
//
// Why a restatement: the reference (/root/reference/proj) needs Eigen 3.4 and
// vendored doctest/CLI11 (CMakeLists.txt:18, README.md:27-29), none of which
// exist in this image, so its factorize.cpp/lapack.cpp cannot be compiled
// here.  Its rng.hpp is header-only and IS compiled directly from the
// reference tree by oracle/Makefile (oracle/_ref/rng_kat), which pins the
// CounterRng restatement below bit-for-bit.
//
// The arithmetic boundary is the same as the reference's: OpenBLAS
// cblas_dgemm (Eigen operator* with EIGEN_USE_BLAS, CMakeLists.txt:37-38) and
// LAPACKE dgeqrf/dorgqr/dgesdd/dgesvd *_work drivers with workspace queries
// (lapack.cpp:60-201).  The reference pins no BLAS version; we link the
// OpenBLAS 0.3.31 shipped in scipy's wheel (symbols carry a `scipy_` prefix).
//
// Every function cites the reference file:line it follows.

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numbers>
#include <stdexcept>
#include <string>
#include <vector>

#define BLASFN(x) scipy_##x

extern "C" {
// cblas / lapacke prototypes (LP64).  No lapacke.h in the image.
enum { CblasColMajor = 102 };
enum { CblasNoTrans = 111, CblasTrans = 112 };
void BLASFN(cblas_dgemm)(int layout, int ta, int tb, int m, int n, int k, double alpha,
                         const double* a, int lda, const double* b, int ldb, double beta, double* c,
                         int ldc);
int BLASFN(LAPACKE_dgesdd_work)(int layout, char jobz, int m, int n, double* a, int lda, double* s,
                                double* u, int ldu, double* vt, int ldvt, double* work, int lwork,
                                int* iwork);
int BLASFN(LAPACKE_dgesvd_work)(int layout, char jobu, char jobvt, int m, int n, double* a,
                                int lda, double* s, double* u, int ldu, double* vt, int ldvt,
                                double* work, int lwork);
int BLASFN(LAPACKE_dgeqrf_work)(int layout, int m, int n, double* a, int lda, double* tau,
                                double* work, int lwork);
int BLASFN(LAPACKE_dorgqr_work)(int layout, int m, int n, int k, double* a, int lda,
                                const double* tau, double* work, int lwork);
// Complex instantiation (lapack.cpp:73-87, 100-110, 154-177; Eigen complex
// operator* -> zgemm).  std::complex<double> is layout-compatible with
// lapack_complex_double (lapack.cpp:4-6).
enum { CblasConjTrans = 113 };
void BLASFN(cblas_zgemm)(int layout, int ta, int tb, int m, int n, int k, const void* alpha,
                         const void* a, int lda, const void* b, int ldb, const void* beta, void* c,
                         int ldc);
int BLASFN(LAPACKE_zgesdd_work)(int layout, char jobz, int m, int n, void* a, int lda, double* s,
                                void* u, int ldu, void* vt, int ldvt, void* work, int lwork,
                                double* rwork, int* iwork);
int BLASFN(LAPACKE_zgesvd_work)(int layout, char jobu, char jobvt, int m, int n, void* a, int lda,
                                double* s, void* u, int ldu, void* vt, int ldvt, void* work,
                                int lwork, double* rwork);
int BLASFN(LAPACKE_zgeqrf_work)(int layout, int m, int n, void* a, int lda, void* tau, void* work,
                                int lwork);
int BLASFN(LAPACKE_zungqr_work)(int layout, int m, int n, int k, void* a, int lda, const void* tau,
                                void* work, int lwork);
void BLASFN(openblas_set_num_threads)(int);
int BLASFN(openblas_get_num_threads)(void);
}

namespace oracle {

constexpr int kColMajor = 102;  // LAPACK_COL_MAJOR

// ------------------------------------------------------------------ rng ---

// rng.hpp:11-15
inline std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// rng.hpp:20-22
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag) { return seed ^ mix64(tag); }

// rng.hpp:34-78.  Word j (j = 1, 2, ...) is mix64(seed + j * golden); normals
// come in Box-Muller pairs (cos first, cached sin second).
class CounterRng {
 public:
  explicit CounterRng(std::uint64_t seed) : key_(seed) {}
  std::uint64_t next() { return mix64(key_ + (++counter_) * 0x9e3779b97f4a7c15ull); }
  double uniform() { return static_cast<double>((next() >> 11) + 1) * 0x1.0p-53; }  // rng.hpp:46
  double normal() {                                                                // rng.hpp:50-60
    if (have_cached_) {
      have_cached_ = false;
      return cached_;
    }
    const double r = std::sqrt(-2.0 * std::log(uniform()));
    const double t = 2.0 * std::numbers::pi * uniform();
    cached_ = r * std::sin(t);
    have_cached_ = true;
    return r * std::cos(t);
  }
  void fill_gaussian(double* dst, std::size_t n) {  // rng.hpp:62-64
    for (std::size_t i = 0; i < n; ++i) dst[i] = normal();
  }
  // rng.hpp:66-71: std::complex<double>(normal() * inv_sqrt2, normal() * inv_sqrt2).
  // The two calls are unsequenced; g++ (the reference's Linux build) evaluates
  // the imaginary argument first, so the Box-Muller cosine lands in im and the
  // sine in re -- pinned by the reference-built KAT (tests/golden/rng_kat.json
  // "complex").
  void fill_gaussian(std::complex<double>* dst, std::size_t n) {
    constexpr double inv_sqrt2 = 0.70710678118654752440;
    for (std::size_t i = 0; i < n; ++i) {
      const double first = normal();
      const double second = normal();
      dst[i] = std::complex<double>(second * inv_sqrt2, first * inv_sqrt2);
    }
  }

 private:
  std::uint64_t key_;
  std::uint64_t counter_ = 0;
  double cached_ = 0.0;
  bool have_cached_ = false;
};

// --------------------------------------------------------------- matrix ---

// Owning column-major matrix, lda == rows (types.hpp:12-13; lapack.cpp:122).
struct Mat {
  std::int64_t rows = 0, cols = 0;
  std::vector<double> d;
  Mat() = default;
  Mat(std::int64_t r, std::int64_t c) : rows(r), cols(c), d(static_cast<std::size_t>(r * c), 0.0) {}
  double* data() { return d.data(); }
  const double* data() const { return d.data(); }
  double& operator()(std::int64_t i, std::int64_t j) { return d[static_cast<std::size_t>(i + j * rows)]; }
  double operator()(std::int64_t i, std::int64_t j) const {
    return d[static_cast<std::size_t>(i + j * rows)];
  }
  std::int64_t size() const { return rows * cols; }
};

[[noreturn]] void fail(const char* driver, int info) {  // lapack.cpp:52-55
  throw std::runtime_error(std::string("lapack: ") + driver + " failed with info=" +
                           std::to_string(info));
}

// C = op(A) * op(B) through dgemm, the Eigen operator* route (CMakeLists.txt:37-38).
Mat gemm(const Mat& a, bool ta, const Mat& b, bool tb) {
  const std::int64_t m = ta ? a.cols : a.rows;
  const std::int64_t k = ta ? a.rows : a.cols;
  const std::int64_t n = tb ? b.rows : b.cols;
  Mat c(m, n);
  if (m == 0 || n == 0) return c;
  if (k == 0) return c;
  BLASFN(cblas_dgemm)(CblasColMajor, ta ? CblasTrans : CblasNoTrans, tb ? CblasTrans : CblasNoTrans,
                      static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), 1.0, a.data(),
                      static_cast<int>(std::max<std::int64_t>(1, a.rows)), b.data(),
                      static_cast<int>(std::max<std::int64_t>(1, b.rows)), 0.0, c.data(),
                      static_cast<int>(std::max<std::int64_t>(1, m)));
  return c;
}

// Grow-only workspace (lapack.cpp:23-50).
struct Workspace {
  std::vector<double> dwork;
  std::vector<int> iwork;
  double* dd(std::size_t n) {
    if (dwork.size() < n) dwork.resize(n);
    return dwork.data();
  }
  int* ii(std::size_t n) {
    if (iwork.size() < n) iwork.resize(n);
    return iwork.data();
  }
};
Workspace& ws() {
  thread_local Workspace w;
  return w;
}

// lapack.cpp:60-71
int gesdd(char jobz, int m, int n, double* a, int lda, double* s, double* u, int ldu, double* vt,
          int ldvt) {
  const int k = std::min(m, n);
  double query = 0;
  int info = BLASFN(LAPACKE_dgesdd_work)(kColMajor, jobz, m, n, a, lda, s, u, ldu, vt, ldvt, &query,
                                         -1, ws().ii(8 * static_cast<std::size_t>(k)));
  if (info != 0) return info;
  const int lwork = static_cast<int>(query);
  return BLASFN(LAPACKE_dgesdd_work)(kColMajor, jobz, m, n, a, lda, s, u, ldu, vt, ldvt,
                                     ws().dd(static_cast<std::size_t>(lwork)), lwork,
                                     ws().ii(8 * static_cast<std::size_t>(k)));
}
// lapack.cpp:89-98
int gesvd(char jobu, char jobvt, int m, int n, double* a, int lda, double* s, double* u, int ldu,
          double* vt, int ldvt) {
  double query = 0;
  int info = BLASFN(LAPACKE_dgesvd_work)(kColMajor, jobu, jobvt, m, n, a, lda, s, u, ldu, vt, ldvt,
                                         &query, -1);
  if (info != 0) return info;
  const int lwork = static_cast<int>(query);
  return BLASFN(LAPACKE_dgesvd_work)(kColMajor, jobu, jobvt, m, n, a, lda, s, u, ldu, vt, ldvt,
                                     ws().dd(static_cast<std::size_t>(lwork)), lwork);
}

// lapack.cpp:112-128: thin SVD of a copy, gesdd('S') then gesvd('S','S').
void svd(const Mat& a, Mat& u, std::vector<double>& s, Mat& vt) {
  const int m = static_cast<int>(a.rows), n = static_cast<int>(a.cols);
  if (m == 0 || n == 0) throw std::invalid_argument("lapack::svd: empty matrix");
  const int k = std::min(m, n);
  u = Mat(m, k);
  s.assign(static_cast<std::size_t>(k), 0.0);
  vt = Mat(k, n);
  Mat work = a;
  int info = gesdd('S', m, n, work.data(), m, s.data(), u.data(), m, vt.data(), k);
  if (info != 0) {
    work = a;
    info = gesvd('S', 'S', m, n, work.data(), m, s.data(), u.data(), m, vt.data(), k);
    if (info != 0) fail("gesdd/gesvd", info);
  }
}

// lapack.cpp:130-144 (singular values only)
std::vector<double> singular_values(const Mat& a) {
  const int m = static_cast<int>(a.rows), n = static_cast<int>(a.cols);
  if (m == 0 || n == 0) return {};
  std::vector<double> s(static_cast<std::size_t>(std::min(m, n)));
  Mat work = a;
  int info = gesdd('N', m, n, work.data(), m, s.data(), nullptr, m, nullptr, 1);
  if (info != 0) {
    work = a;
    info = gesvd('N', 'N', m, n, work.data(), m, s.data(), nullptr, m, nullptr, 1);
    if (info != 0) fail("gesdd/gesvd", info);
  }
  return s;
}

// lapack.cpp:146-153, 163-170, 180-201, 211-215: thin Householder QR,
// explicit Q with min(m,n) orthonormal columns.
Mat orthonormal_columns(Mat a) {
  const int m = static_cast<int>(a.rows), n = static_cast<int>(a.cols);
  if (m == 0 || n == 0) throw std::invalid_argument("lapack::qr: empty matrix");
  const int k = std::min(m, n);
  std::vector<double> tau(static_cast<std::size_t>(k));
  double query = 0;
  int info = BLASFN(LAPACKE_dgeqrf_work)(kColMajor, m, n, a.data(), m, tau.data(), &query, -1);
  if (info == 0) {
    const int lwork = static_cast<int>(query);
    info = BLASFN(LAPACKE_dgeqrf_work)(kColMajor, m, n, a.data(), m, tau.data(),
                                       ws().dd(static_cast<std::size_t>(lwork)), lwork);
  }
  if (info != 0) fail("geqrf", info);
  a.cols = k;  // conservativeResize(m, k): leading m*k entries are kept
  a.d.resize(static_cast<std::size_t>(m) * static_cast<std::size_t>(k));
  info = BLASFN(LAPACKE_dorgqr_work)(kColMajor, m, k, k, a.data(), m, tau.data(), &query, -1);
  if (info == 0) {
    const int lwork = static_cast<int>(query);
    info = BLASFN(LAPACKE_dorgqr_work)(kColMajor, m, k, k, a.data(), m, tau.data(),
                                       ws().dd(static_cast<std::size_t>(lwork)), lwork);
  }
  if (info != 0) fail("orgqr", info);
  return a;
}

// ------------------------------------------------------------ factorize ---

struct Factorization {
  Mat left;                   // m x r
  std::vector<double> sigma;  // r
  Mat right_adj;              // r x n
  double discarded_weight = 0.0;
  bool discarded_exact = true;
};

// factorize.cpp:17-24
std::int64_t numerical_rank(const std::vector<double>& sigma, std::int64_t m, std::int64_t n) {
  if (sigma.empty() || sigma[0] <= 0.0) return 0;
  const double cut =
      static_cast<double>(std::max(m, n)) * std::numeric_limits<double>::epsilon() * sigma[0];
  std::int64_t r = static_cast<std::int64_t>(sigma.size());
  while (r > 0 && sigma[static_cast<std::size_t>(r - 1)] <= cut) --r;
  return r;
}

// factorize.cpp:26-38
Factorization truncate_full(const Mat& u, const std::vector<double>& s, const Mat& vt,
                            std::int64_t chi, std::int64_t m, std::int64_t n) {
  Factorization f;
  const std::int64_t r = std::min(chi, numerical_rank(s, m, n));
  f.discarded_weight = 0.0;
  for (std::size_t k = static_cast<std::size_t>(r); k < s.size(); ++k) f.discarded_weight += s[k] * s[k];
  f.left = Mat(u.rows, r);
  std::copy(u.d.begin(), u.d.begin() + static_cast<std::ptrdiff_t>(u.rows * r), f.left.d.begin());
  f.sigma.assign(s.begin(), s.begin() + r);
  f.right_adj = Mat(r, vt.cols);
  for (std::int64_t j = 0; j < vt.cols; ++j)
    for (std::int64_t i = 0; i < r; ++i) f.right_adj(i, j) = vt(i, j);
  f.discarded_exact = true;
  return f;
}

// factorize.cpp:42-50
Factorization tsvd(const Mat& a, std::int64_t chi) {
  if (a.rows == 0 || a.cols == 0) throw std::invalid_argument("tsvd: empty matrix");
  if (chi < 1) throw std::invalid_argument("tsvd: rank must be >= 1");
  Mat u, vt;
  std::vector<double> s;
  svd(a, u, s, vt);
  return truncate_full(u, s, vt, chi, a.rows, a.cols);
}

// factorize.cpp:52-74.  `omega` (optional) replaces the CounterRng draw so a
// device-generated sketch can be fed to the oracle for same-input parity.
Mat randomized_range(const Mat& a, std::int64_t ell, int power, std::uint64_t seed,
                     const double* omega = nullptr) {
  const std::int64_t m = a.rows, n = a.cols;
  if (m == 0 || n == 0) throw std::invalid_argument("randomized_range: empty matrix");
  if (ell < 1 || ell > std::min(m, n))
    throw std::invalid_argument("randomized_range: need 1 <= ell <= min(m, n)");
  if (power < 0) throw std::invalid_argument("randomized_range: power must be >= 0");
  Mat om(n, ell);
  if (omega) {
    std::memcpy(om.data(), omega, sizeof(double) * static_cast<std::size_t>(n * ell));
  } else {
    CounterRng rng(seed);
    rng.fill_gaussian(om.data(), static_cast<std::size_t>(om.size()));
  }
  Mat q = orthonormal_columns(gemm(a, false, om, false));
  for (int t = 0; t < power; ++t) {
    q = orthonormal_columns(gemm(a, true, q, false));
    q = orthonormal_columns(gemm(a, false, q, false));
  }
  return q;
}

// factorize.cpp:76-95
Factorization rsvd(const Mat& a, std::int64_t rank, std::int64_t oversample, int power,
                   std::uint64_t seed, const double* omega = nullptr) {
  const std::int64_t m = a.rows, n = a.cols;
  if (m == 0 || n == 0) throw std::invalid_argument("rsvd: empty matrix");
  if (rank < 1) throw std::invalid_argument("rsvd: rank must be >= 1");
  std::int64_t ell = oversample;
  if (ell == 0) ell = std::min(2 * rank, std::min(m, n));
  if (ell < rank) throw std::invalid_argument("rsvd: oversample must be >= rank");
  const Mat q = randomized_range(a, ell, power, seed, omega);
  const Mat b = gemm(q, true, a, false);  // ell x n
  Mat ub, vtb;
  std::vector<double> sb;
  svd(b, ub, sb, vtb);
  Factorization f = truncate_full(ub, sb, vtb, rank, m, n);
  f.left = gemm(q, false, f.left, false);
  f.discarded_exact = false;
  return f;
}

// factorize.cpp:97-104
double reconstruction_error(const Mat& a, const Factorization& f, bool spectral) {
  Mat us = f.left;
  for (std::int64_t j = 0; j < us.cols; ++j)
    for (std::int64_t i = 0; i < us.rows; ++i) us(i, j) *= f.sigma[static_cast<std::size_t>(j)];
  Mat rec = gemm(us, false, f.right_adj, false);
  if (rec.rows != a.rows || rec.cols != a.cols) rec = Mat(a.rows, a.cols);
  Mat resid(a.rows, a.cols);
  for (std::size_t i = 0; i < resid.d.size(); ++i) resid.d[i] = a.d[i] - rec.d[i];
  if (!spectral) {
    double s = 0.0;  // Eigen's norm(): sqrt of the sum of squares
    for (double v : resid.d) s += v * v;
    return std::sqrt(s);
  }
  const std::vector<double> s = singular_values(resid);
  return s.empty() ? 0.0 : s[0];
}

// ---------------------------------------------------------------- blocks ---

// blocks.cpp:19-36
std::vector<std::int64_t> sector_request(int maximal, std::int64_t chi, std::int64_t slack,
                                         const std::vector<std::int64_t>& dims) {
  if (chi < 1) throw std::invalid_argument("sector_request: chi must be >= 1");
  const std::int64_t n = static_cast<std::int64_t>(dims.size());
  if (n < 1) throw std::invalid_argument("sector_request: need at least one sector");
  std::vector<std::int64_t> out(dims.size());
  if (maximal) {
    for (std::size_t s = 0; s < dims.size(); ++s) out[s] = std::min(chi, dims[s]);
    return out;
  }
  const std::int64_t base = (chi + n - 1) / n;
  const std::int64_t sl = slack >= 0 ? slack : std::max<std::int64_t>(2, (base + 19) / 20);
  for (std::size_t s = 0; s < dims.size(); ++s) out[s] = std::min(base + sl, dims[s]);
  return out;
}

struct BlockResult {
  std::vector<Factorization> factors;
  double discarded_weight = 0.0;
  bool discarded_exact = true;
};

// blocks.cpp:38-118: per-sector rsvd (kind == 1 and min dim >= min_dim) or
// tsvd, then the global top-chi selection, ties by charge then position.
BlockResult block_factorize(const std::vector<Mat>& blocks, const std::vector<std::int64_t>& charges,
                            std::int64_t chi, int maximal, std::int64_t slack, int kind,
                            std::int64_t oversample, int power, std::uint64_t seed,
                            std::int64_t min_dim) {
  if (blocks.size() != charges.size())
    throw std::invalid_argument("block_factorize: charges/blocks size mismatch");
  if (blocks.empty()) throw std::invalid_argument("block_factorize: no sectors");
  {
    std::vector<std::int64_t> c = charges;
    std::sort(c.begin(), c.end());
    if (std::adjacent_find(c.begin(), c.end()) != c.end())
      throw std::invalid_argument("block_factorize: duplicate sector charge");
  }
  std::vector<std::int64_t> dims(blocks.size());
  for (std::size_t s = 0; s < blocks.size(); ++s) dims[s] = std::min(blocks[s].rows, blocks[s].cols);
  const std::vector<std::int64_t> want = sector_request(maximal, chi, slack, dims);

  BlockResult out;
  out.factors.resize(blocks.size());
  for (std::size_t s = 0; s < blocks.size(); ++s) {
    Factorization& f = out.factors[s];
    if (want[s] == 0 || dims[s] == 0) {
      f.left = Mat(blocks[s].rows, 0);
      f.sigma.clear();
      f.right_adj = Mat(0, blocks[s].cols);
      double sq = 0.0;
      for (double v : blocks[s].d) sq += v * v;
      f.discarded_weight = sq;
      continue;
    }
    if (kind == 1 && dims[s] >= min_dim) {
      const std::int64_t ell = oversample > 0 ? std::min(std::max(oversample, want[s]), dims[s])
                                              : std::min(2 * want[s], dims[s]);
      f = rsvd(blocks[s], want[s], ell, power,
               derive_seed(seed, static_cast<std::uint64_t>(charges[s])));
      out.discarded_exact = false;
    } else {
      f = tsvd(blocks[s], want[s]);
    }
  }
  struct Cand {
    double sigma;
    std::int64_t charge, pos;
    std::size_t sector;
  };
  std::vector<Cand> cand;
  for (std::size_t s = 0; s < out.factors.size(); ++s)
    for (std::size_t k = 0; k < out.factors[s].sigma.size(); ++k)
      cand.push_back({out.factors[s].sigma[k], charges[s], static_cast<std::int64_t>(k), s});
  std::sort(cand.begin(), cand.end(), [](const Cand& x, const Cand& y) {
    if (x.sigma != y.sigma) return x.sigma > y.sigma;
    if (x.charge != y.charge) return x.charge < y.charge;
    return x.pos < y.pos;
  });
  std::vector<std::int64_t> keep(out.factors.size(), 0);
  for (std::size_t i = 0; i < cand.size() && static_cast<std::int64_t>(i) < chi; ++i)
    ++keep[cand[i].sector];
  for (std::size_t s = 0; s < out.factors.size(); ++s) {
    Factorization& f = out.factors[s];
    const std::int64_t r = keep[s];
    for (std::size_t k = static_cast<std::size_t>(r); k < f.sigma.size(); ++k)
      f.discarded_weight += f.sigma[k] * f.sigma[k];
    Mat l(f.left.rows, r), ra(r, f.right_adj.cols);
    for (std::int64_t j = 0; j < r; ++j)
      for (std::int64_t i = 0; i < l.rows; ++i) l(i, j) = f.left(i, j);
    for (std::int64_t j = 0; j < ra.cols; ++j)
      for (std::int64_t i = 0; i < r; ++i) ra(i, j) = f.right_adj(i, j);
    f.left = l;
    f.right_adj = ra;
    f.sigma.resize(static_cast<std::size_t>(r));
    out.discarded_weight += f.discarded_weight;
  }
  return out;
}


// ============================================================ complex ===
// The reference instantiates the same path for std::complex<double>
// (factorize.cpp:106-118; lapack.cpp:73-110, 154-177, 206-223).  Same
// operation order; A^H where the real path has A^T (factorize.cpp:70, 86).
namespace z {

using C = std::complex<double>;

struct Mat {
  std::int64_t rows = 0, cols = 0;
  std::vector<C> d;
  Mat() = default;
  Mat(std::int64_t r, std::int64_t c) : rows(r), cols(c), d(static_cast<std::size_t>(r * c), C(0)) {}
  C* data() { return d.data(); }
  const C* data() const { return d.data(); }
  C& operator()(std::int64_t i, std::int64_t j) { return d[static_cast<std::size_t>(i + j * rows)]; }
  C operator()(std::int64_t i, std::int64_t j) const { return d[static_cast<std::size_t>(i + j * rows)]; }
  std::int64_t size() const { return rows * cols; }
};

struct Workspace {
  std::vector<C> zwork;
  std::vector<double> rwork;
  std::vector<int> iwork;
  C* zz(std::size_t n) {
    if (zwork.size() < n) zwork.resize(n);
    return zwork.data();
  }
  double* rr(std::size_t n) {
    if (rwork.size() < n) rwork.resize(n);
    return rwork.data();
  }
  int* ii(std::size_t n) {
    if (iwork.size() < n) iwork.resize(n);
    return iwork.data();
  }
};
Workspace& ws() {
  thread_local Workspace w;
  return w;
}

// C = op(A) op(B), op in {N, H} (Eigen operator* / adjoint() -> zgemm).
Mat gemm(const Mat& a, bool ha, const Mat& b, bool hb) {
  const std::int64_t m = ha ? a.cols : a.rows;
  const std::int64_t k = ha ? a.rows : a.cols;
  const std::int64_t n = hb ? b.rows : b.cols;
  Mat c(m, n);
  if (m == 0 || n == 0 || k == 0) return c;
  const C one(1.0), zero(0.0);
  BLASFN(cblas_zgemm)(CblasColMajor, ha ? int(CblasConjTrans) : int(CblasNoTrans),
                      hb ? int(CblasConjTrans) : int(CblasNoTrans), static_cast<int>(m), static_cast<int>(n),
                      static_cast<int>(k), &one, a.data(),
                      static_cast<int>(std::max<std::int64_t>(1, a.rows)), b.data(),
                      static_cast<int>(std::max<std::int64_t>(1, b.rows)), &zero, c.data(),
                      static_cast<int>(std::max<std::int64_t>(1, m)));
  return c;
}

// lapack.cpp:73-87 (rwork sizing as there)
int gesdd(char jobz, int m, int n, C* a, int lda, double* s, C* u, int ldu, C* vt, int ldvt) {
  const auto k = static_cast<std::size_t>(std::min(m, n));
  const auto mx = static_cast<std::size_t>(std::max(m, n));
  const std::size_t lrwork =
      jobz == 'N' ? 7 * k : std::max<std::size_t>(1, 5 * k * k + 7 * k) + 2 * k * mx;
  C query = 0;
  int info = BLASFN(LAPACKE_zgesdd_work)(kColMajor, jobz, m, n, a, lda, s, u, ldu, vt, ldvt, &query,
                                         -1, ws().rr(lrwork), ws().ii(8 * k));
  if (info != 0) return info;
  const int lwork = static_cast<int>(query.real());
  return BLASFN(LAPACKE_zgesdd_work)(kColMajor, jobz, m, n, a, lda, s, u, ldu, vt, ldvt,
                                     ws().zz(static_cast<std::size_t>(lwork)), lwork,
                                     ws().rr(lrwork), ws().ii(8 * k));
}
// lapack.cpp:100-110
int gesvd(char jobu, char jobvt, int m, int n, C* a, int lda, double* s, C* u, int ldu, C* vt,
          int ldvt) {
  const auto k = static_cast<std::size_t>(std::min(m, n));
  C query = 0;
  int info = BLASFN(LAPACKE_zgesvd_work)(kColMajor, jobu, jobvt, m, n, a, lda, s, u, ldu, vt, ldvt,
                                         &query, -1, ws().rr(5 * k));
  if (info != 0) return info;
  const int lwork = static_cast<int>(query.real());
  return BLASFN(LAPACKE_zgesvd_work)(kColMajor, jobu, jobvt, m, n, a, lda, s, u, ldu, vt, ldvt,
                                     ws().zz(static_cast<std::size_t>(lwork)), lwork,
                                     ws().rr(5 * k));
}

// lapack.cpp:112-128
void svd(const Mat& a, Mat& u, std::vector<double>& s, Mat& vt) {
  const int m = static_cast<int>(a.rows), n = static_cast<int>(a.cols);
  if (m == 0 || n == 0) throw std::invalid_argument("lapack::svd: empty matrix");
  const int k = std::min(m, n);
  u = Mat(m, k);
  s.assign(static_cast<std::size_t>(k), 0.0);
  vt = Mat(k, n);
  Mat work = a;
  int info = gesdd('S', m, n, work.data(), m, s.data(), u.data(), m, vt.data(), k);
  if (info != 0) {
    work = a;
    info = gesvd('S', 'S', m, n, work.data(), m, s.data(), u.data(), m, vt.data(), k);
    if (info != 0) fail("gesdd/gesvd", info);
  }
}

// lapack.cpp:130-144
std::vector<double> singular_values(const Mat& a) {
  const int m = static_cast<int>(a.rows), n = static_cast<int>(a.cols);
  if (m == 0 || n == 0) return {};
  std::vector<double> s(static_cast<std::size_t>(std::min(m, n)));
  Mat work = a;
  int info = gesdd('N', m, n, work.data(), m, s.data(), nullptr, m, nullptr, 1);
  if (info != 0) {
    work = a;
    info = gesvd('N', 'N', m, n, work.data(), m, s.data(), nullptr, m, nullptr, 1);
    if (info != 0) fail("gesdd/gesvd", info);
  }
  return s;
}

// lapack.cpp:154-162, 171-177, 180-201, 216-219 (zgeqrf + zungqr)
Mat orthonormal_columns(Mat a) {
  const int m = static_cast<int>(a.rows), n = static_cast<int>(a.cols);
  if (m == 0 || n == 0) throw std::invalid_argument("lapack::qr: empty matrix");
  const int k = std::min(m, n);
  std::vector<C> tau(static_cast<std::size_t>(k));
  C query = 0;
  int info = BLASFN(LAPACKE_zgeqrf_work)(kColMajor, m, n, a.data(), m, tau.data(), &query, -1);
  if (info == 0) {
    const int lwork = static_cast<int>(query.real());
    info = BLASFN(LAPACKE_zgeqrf_work)(kColMajor, m, n, a.data(), m, tau.data(),
                                       ws().zz(static_cast<std::size_t>(lwork)), lwork);
  }
  if (info != 0) fail("geqrf", info);
  a.cols = k;
  a.d.resize(static_cast<std::size_t>(m) * static_cast<std::size_t>(k));
  info = BLASFN(LAPACKE_zungqr_work)(kColMajor, m, k, k, a.data(), m, tau.data(), &query, -1);
  if (info == 0) {
    const int lwork = static_cast<int>(query.real());
    info = BLASFN(LAPACKE_zungqr_work)(kColMajor, m, k, k, a.data(), m, tau.data(),
                                       ws().zz(static_cast<std::size_t>(lwork)), lwork);
  }
  if (info != 0) fail("orgqr", info);
  return a;
}

struct Factorization {
  Mat left;
  std::vector<double> sigma;
  Mat right_adj;
  double discarded_weight = 0.0;
  bool discarded_exact = true;
};

// factorize.cpp:26-38 (numerical_rank is scalar-independent, :17-24)
Factorization truncate_full(const Mat& u, const std::vector<double>& s, const Mat& vt,
                            std::int64_t chi, std::int64_t m, std::int64_t n) {
  Factorization f;
  const std::int64_t r = std::min(chi, numerical_rank(s, m, n));
  for (std::size_t k = static_cast<std::size_t>(r); k < s.size(); ++k) f.discarded_weight += s[k] * s[k];
  f.left = Mat(u.rows, r);
  std::copy(u.d.begin(), u.d.begin() + static_cast<std::ptrdiff_t>(u.rows * r), f.left.d.begin());
  f.sigma.assign(s.begin(), s.begin() + r);
  f.right_adj = Mat(r, vt.cols);
  for (std::int64_t j = 0; j < vt.cols; ++j)
    for (std::int64_t i = 0; i < r; ++i) f.right_adj(i, j) = vt(i, j);
  f.discarded_exact = true;
  return f;
}

// factorize.cpp:42-50
Factorization tsvd(const Mat& a, std::int64_t chi) {
  if (a.rows == 0 || a.cols == 0) throw std::invalid_argument("tsvd: empty matrix");
  if (chi < 1) throw std::invalid_argument("tsvd: rank must be >= 1");
  Mat u, vt;
  std::vector<double> s;
  svd(a, u, s, vt);
  return truncate_full(u, s, vt, chi, a.rows, a.cols);
}

// factorize.cpp:52-74 with Scalar = complex: Omega from the complex fill,
// A^H on the power step.
Mat randomized_range(const Mat& a, std::int64_t ell, int power, std::uint64_t seed,
                     const C* omega = nullptr) {
  const std::int64_t m = a.rows, n = a.cols;
  if (m == 0 || n == 0) throw std::invalid_argument("randomized_range: empty matrix");
  if (ell < 1 || ell > std::min(m, n))
    throw std::invalid_argument("randomized_range: need 1 <= ell <= min(m, n)");
  if (power < 0) throw std::invalid_argument("randomized_range: power must be >= 0");
  Mat om(n, ell);
  if (omega) {
    std::copy(omega, omega + n * ell, om.d.begin());
  } else {
    CounterRng rng(seed);
    rng.fill_gaussian(om.data(), static_cast<std::size_t>(om.size()));
  }
  Mat q = orthonormal_columns(gemm(a, false, om, false));
  for (int t = 0; t < power; ++t) {
    q = orthonormal_columns(gemm(a, true, q, false));
    q = orthonormal_columns(gemm(a, false, q, false));
  }
  return q;
}

// factorize.cpp:76-95 (B = Q^H A)
Factorization rsvd(const Mat& a, std::int64_t rank, std::int64_t oversample, int power,
                   std::uint64_t seed, const C* omega = nullptr) {
  const std::int64_t m = a.rows, n = a.cols;
  if (m == 0 || n == 0) throw std::invalid_argument("rsvd: empty matrix");
  if (rank < 1) throw std::invalid_argument("rsvd: rank must be >= 1");
  std::int64_t ell = oversample;
  if (ell == 0) ell = std::min(2 * rank, std::min(m, n));
  if (ell < rank) throw std::invalid_argument("rsvd: oversample must be >= rank");
  const Mat q = randomized_range(a, ell, power, seed, omega);
  const Mat b = gemm(q, true, a, false);
  Mat ub, vtb;
  std::vector<double> sb;
  svd(b, ub, sb, vtb);
  Factorization f = truncate_full(ub, sb, vtb, rank, m, n);
  f.left = gemm(q, false, f.left, false);
  f.discarded_exact = false;
  return f;
}

// factorize.cpp:97-104
double reconstruction_error(const Mat& a, const Factorization& f, bool spectral) {
  Mat us = f.left;
  for (std::int64_t j = 0; j < us.cols; ++j)
    for (std::int64_t i = 0; i < us.rows; ++i) us(i, j) *= f.sigma[static_cast<std::size_t>(j)];
  Mat rec = gemm(us, false, f.right_adj, false);
  if (rec.rows != a.rows || rec.cols != a.cols) rec = Mat(a.rows, a.cols);
  Mat resid(a.rows, a.cols);
  for (std::size_t i = 0; i < resid.d.size(); ++i) resid.d[i] = a.d[i] - rec.d[i];
  if (!spectral) {
    double s = 0.0;
    for (const C& v : resid.d) s += std::norm(v);
    return std::sqrt(s);
  }
  const std::vector<double> s = singular_values(resid);
  return s.empty() ? 0.0 : s[0];
}

}  // namespace z

}  // namespace oracle

// ------------------------------------------------------------- C ABI ---
//
// Error convention shared with include/rsvd_c.h: 0 ok, 1 invalid argument,
// 2 numerical (LAPACK) failure.  The message of the last failure is kept per
// thread and returned by oracle_last_error().

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

oracle::Mat wrap(const double* a, std::int64_t m, std::int64_t n, std::int64_t lda) {
  oracle::Mat x(m, n);
  for (std::int64_t j = 0; j < n; ++j)
    std::memcpy(x.data() + j * m, a + j * lda, sizeof(double) * static_cast<std::size_t>(m));
  return x;
}

void emit(const oracle::Factorization& f, double* u, double* s, double* vt, std::int64_t ldvt,
          std::int64_t* rank, double* dw) {
  const std::int64_t r = static_cast<std::int64_t>(f.sigma.size());
  *rank = r;
  *dw = f.discarded_weight;
  if (u) std::memcpy(u, f.left.data(), sizeof(double) * static_cast<std::size_t>(f.left.size()));
  if (s) std::memcpy(s, f.sigma.data(), sizeof(double) * static_cast<std::size_t>(r));
  if (vt)
    for (std::int64_t j = 0; j < f.right_adj.cols; ++j)
      for (std::int64_t i = 0; i < r; ++i) vt[i + j * ldvt] = f.right_adj(i, j);
}
}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }
void oracle_set_threads(int n) { BLASFN(openblas_set_num_threads)(n); }
int oracle_get_threads(void) { return BLASFN(openblas_get_num_threads)(); }

std::uint64_t oracle_mix64(std::uint64_t z) { return oracle::mix64(z); }
std::uint64_t oracle_derive_seed(std::uint64_t s, std::uint64_t t) { return oracle::derive_seed(s, t); }

void oracle_rng_words(std::uint64_t seed, std::uint64_t* out, std::int64_t n) {
  oracle::CounterRng rng(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = rng.next();
}
void oracle_fill_gaussian(std::uint64_t seed, double* out, std::int64_t n) {
  oracle::CounterRng rng(seed);
  rng.fill_gaussian(out, static_cast<std::size_t>(n));
}

// rsvd(A, {k, ell, q, seed}).  U is m x k (ld m), S k, Vt k x n (ld ldvt);
// only the leading *rank columns/values/rows are written.  omega may be null.
int oracle_rsvd(const double* a, std::int64_t m, std::int64_t n, std::int64_t lda, std::int64_t k,
                std::int64_t ell, int q, std::uint64_t seed, const double* omega, double* u,
                double* s, double* vt, std::int64_t ldvt, std::int64_t* rank, double* dw) {
  return guarded([&] {
    const oracle::Mat am = wrap(a, m, n, lda);
    emit(oracle::rsvd(am, k, ell, q, seed, omega), u, s, vt, ldvt, rank, dw);
  });
}

int oracle_tsvd(const double* a, std::int64_t m, std::int64_t n, std::int64_t lda, std::int64_t chi,
                double* u, double* s, double* vt, std::int64_t ldvt, std::int64_t* rank, double* dw) {
  return guarded([&] {
    const oracle::Mat am = wrap(a, m, n, lda);
    emit(oracle::tsvd(am, chi), u, s, vt, ldvt, rank, dw);
  });
}

// Q (m x ell, ld m) of randomized_range.
int oracle_randomized_range(const double* a, std::int64_t m, std::int64_t n, std::int64_t lda,
                            std::int64_t ell, int q, std::uint64_t seed, const double* omega,
                            double* qout) {
  return guarded([&] {
    const oracle::Mat am = wrap(a, m, n, lda);
    const oracle::Mat qm = oracle::randomized_range(am, ell, q, seed, omega);
    std::memcpy(qout, qm.data(), sizeof(double) * static_cast<std::size_t>(qm.size()));
  });
}

// ||A - U diag(S) Vt|| (frobenius: spectral == 0).
int oracle_reconstruction_error(const double* a, std::int64_t m, std::int64_t n, std::int64_t lda,
                                const double* u, const double* s, const double* vt,
                                std::int64_t ldvt, std::int64_t r, int spectral, double* out) {
  return guarded([&] {
    oracle::Factorization f;
    f.left = wrap(u, m, r, m);
    f.sigma.assign(s, s + r);
    f.right_adj = wrap(vt, r, n, ldvt);
    *out = oracle::reconstruction_error(wrap(a, m, n, lda), f, spectral != 0);
  });
}

// Thin Householder Q (geqrf + orgqr) — also used by the test-input generator
// to build Haar factors.
int oracle_orthonormal_columns(const double* a, std::int64_t m, std::int64_t n, double* qout) {
  return guarded([&] {
    const oracle::Mat qm = oracle::orthonormal_columns(wrap(a, m, n, m));
    std::memcpy(qout, qm.data(), sizeof(double) * static_cast<std::size_t>(qm.size()));
  });
}

// Full thin SVD (gesdd/gesvd) — used by tests for singular-value references.
int oracle_singular_values(const double* a, std::int64_t m, std::int64_t n, double* s) {
  return guarded([&] {
    const std::vector<double> v = oracle::singular_values(wrap(a, m, n, m));
    std::memcpy(s, v.data(), sizeof(double) * v.size());
  });
}

int oracle_sector_request(int maximal, std::int64_t chi, std::int64_t slack, const std::int64_t* dims,
                          std::int64_t ns, std::int64_t* out) {
  return guarded([&] {
    const std::vector<std::int64_t> d(dims, dims + ns);
    const auto r = oracle::sector_request(maximal, chi, slack, d);
    std::memcpy(out, r.data(), sizeof(std::int64_t) * r.size());
  });
}

// block_factorize over ns sectors; block s is rows[s] x cols[s] column-major at
// blocks[s].  Outputs per sector: ranks[s], dws[s]; sigma values concatenated
// in sector order into sigma_out (capacity sum of min dims); u_out[s] /
// vt_out[s] (optional, may be null) receive rows[s] x rank and rank x cols[s]
// column-major factors (ld rows[s] and rank).
int oracle_block_factorize(std::int64_t ns, const std::int64_t* charges, const double* const* blocks,
                           const std::int64_t* rows, const std::int64_t* cols, std::int64_t chi,
                           int maximal, std::int64_t slack, int kind, std::int64_t oversample,
                           int power, std::uint64_t seed, std::int64_t min_dim,
                           std::int64_t* ranks, double* dws, double* sigma_out,
                           double* const* u_out, double* const* vt_out, double* total_dw,
                           int* exact) {
  return guarded([&] {
    std::vector<oracle::Mat> bl;
    for (std::int64_t s = 0; s < ns; ++s) bl.push_back(wrap(blocks[s], rows[s], cols[s], rows[s]));
    const std::vector<std::int64_t> ch(charges, charges + ns);
    const oracle::BlockResult r = oracle::block_factorize(bl, ch, chi, maximal, slack, kind,
                                                          oversample, power, seed, min_dim);
    std::int64_t off = 0;
    for (std::int64_t s = 0; s < ns; ++s) {
      const oracle::Factorization& f = r.factors[static_cast<std::size_t>(s)];
      const std::int64_t k = static_cast<std::int64_t>(f.sigma.size());
      ranks[s] = k;
      dws[s] = f.discarded_weight;
      std::memcpy(sigma_out + off, f.sigma.data(), sizeof(double) * static_cast<std::size_t>(k));
      off += k;
      if (u_out && u_out[s])
        std::memcpy(u_out[s], f.left.data(), sizeof(double) * static_cast<std::size_t>(f.left.size()));
      if (vt_out && vt_out[s])
        std::memcpy(vt_out[s], f.right_adj.data(),
                    sizeof(double) * static_cast<std::size_t>(f.right_adj.size()));
    }
    *total_dw = r.discarded_weight;
    *exact = r.discarded_exact ? 1 : 0;
  });
}

}  // extern "C"

// ---- complex instantiation (interleaved re/im, column-major) ----
namespace {
using ZC = std::complex<double>;
oracle::z::Mat zwrap(const ZC* a, std::int64_t m, std::int64_t n, std::int64_t lda) {
  oracle::z::Mat x(m, n);
  for (std::int64_t j = 0; j < n; ++j) std::copy(a + j * lda, a + j * lda + m, x.data() + j * m);
  return x;
}
void zemit(const oracle::z::Factorization& f, ZC* u, double* s, ZC* vt, std::int64_t ldvt,
           std::int64_t* rank, double* dw) {
  const std::int64_t r = static_cast<std::int64_t>(f.sigma.size());
  *rank = r;
  *dw = f.discarded_weight;
  if (u) std::copy(f.left.d.begin(), f.left.d.end(), u);
  if (s) std::copy(f.sigma.begin(), f.sigma.end(), s);
  if (vt)
    for (std::int64_t j = 0; j < f.right_adj.cols; ++j)
      for (std::int64_t i = 0; i < r; ++i) vt[i + j * ldvt] = f.right_adj(i, j);
}
}  // namespace

extern "C" {
void oracle_zfill_gaussian(std::uint64_t seed, void* out, std::int64_t n) {
  oracle::CounterRng rng(seed);
  rng.fill_gaussian(static_cast<ZC*>(out), static_cast<std::size_t>(n));
}
int oracle_zrsvd(const void* a, std::int64_t m, std::int64_t n, std::int64_t lda, std::int64_t k,
                 std::int64_t ell, int q, std::uint64_t seed, const void* omega, void* u, double* s,
                 void* vt, std::int64_t ldvt, std::int64_t* rank, double* dw) {
  return guarded([&] {
    const auto am = zwrap(static_cast<const ZC*>(a), m, n, lda);
    zemit(oracle::z::rsvd(am, k, ell, q, seed, static_cast<const ZC*>(omega)), static_cast<ZC*>(u),
          s, static_cast<ZC*>(vt), ldvt, rank, dw);
  });
}
int oracle_ztsvd(const void* a, std::int64_t m, std::int64_t n, std::int64_t lda, std::int64_t chi,
                 void* u, double* s, void* vt, std::int64_t ldvt, std::int64_t* rank, double* dw) {
  return guarded([&] {
    const auto am = zwrap(static_cast<const ZC*>(a), m, n, lda);
    zemit(oracle::z::tsvd(am, chi), static_cast<ZC*>(u), s, static_cast<ZC*>(vt), ldvt, rank, dw);
  });
}
int oracle_zrandomized_range(const void* a, std::int64_t m, std::int64_t n, std::int64_t lda,
                             std::int64_t ell, int q, std::uint64_t seed, const void* omega,
                             void* qout) {
  return guarded([&] {
    const auto qm = oracle::z::randomized_range(zwrap(static_cast<const ZC*>(a), m, n, lda), ell, q,
                                                seed, static_cast<const ZC*>(omega));
    std::copy(qm.d.begin(), qm.d.end(), static_cast<ZC*>(qout));
  });
}
int oracle_zreconstruction_error(const void* a, std::int64_t m, std::int64_t n, std::int64_t lda,
                                 const void* u, const double* s, const void* vt, std::int64_t ldvt,
                                 std::int64_t r, int spectral, double* out) {
  return guarded([&] {
    oracle::z::Factorization f;
    f.left = zwrap(static_cast<const ZC*>(u), m, r, m);
    f.sigma.assign(s, s + r);
    f.right_adj = zwrap(static_cast<const ZC*>(vt), r, n, ldvt);
    *out = oracle::z::reconstruction_error(zwrap(static_cast<const ZC*>(a), m, n, lda), f,
                                           spectral != 0);
  });
}
int oracle_zorthonormal_columns(const void* a, std::int64_t m, std::int64_t n, void* qout) {
  return guarded([&] {
    const auto qm = oracle::z::orthonormal_columns(zwrap(static_cast<const ZC*>(a), m, n, m));
    std::copy(qm.d.begin(), qm.d.end(), static_cast<ZC*>(qout));
  });
}
int oracle_zsingular_values(const void* a, std::int64_t m, std::int64_t n, double* s) {
  return guarded([&] {
    const auto v = oracle::z::singular_values(zwrap(static_cast<const ZC*>(a), m, n, m));
    std::copy(v.begin(), v.end(), s);
  });
}
}  // extern "C"
