// rsvd_b200.hpp — header-only C++ drop-in for rlftn's factorization API over
// the C ABI of include/rsvd_c.h.
//
// Mirrors proj/include/rlftn/factorize.hpp: RsvdParams (hpp:40-45),
// TruncatedFactorization<Scalar> (hpp:15-31), rsvd (hpp:62-63), tsvd
// (hpp:49-50), randomized_range (hpp:56-57), reconstruction_error
// (hpp:68-70), each for Scalar = double and std::complex<double> as the
// reference instantiates them (factorize.cpp:106-118), and rng.hpp's mix64 /
// derive_seed / seed_tag.  Errors are rethrown as the reference's exception
// types with the reference's messages (std::invalid_argument for argument
// errors, std::runtime_error otherwise).  The matrix type is an owning
// column-major buffer with lda == rows, i.e. exactly the storage Eigen hands
// to LAPACK (types.hpp:12-13), so an Eigen caller passes a.data()/a.rows()/
// a.cols().
#pragma once

#include <algorithm>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "rsvd_c.h"

namespace rlftn_b200 {

using Index = std::int64_t;
using Complex = std::complex<double>;

template <class Scalar>
struct Matrix {
  Index r = 0, c = 0;
  std::vector<Scalar> v;
  using value_type = Scalar;
  Matrix() = default;
  Matrix(Index rows, Index cols) : r(rows), c(cols), v(static_cast<size_t>(rows * cols), Scalar(0)) {}
  Index rows() const { return r; }
  Index cols() const { return c; }
  Scalar* data() { return v.data(); }
  const Scalar* data() const { return v.data(); }
  Scalar& operator()(Index i, Index j) { return v[static_cast<size_t>(i + j * r)]; }
  Scalar operator()(Index i, Index j) const { return v[static_cast<size_t>(i + j * r)]; }
};
using MatrixR = Matrix<double>;
using MatrixC = Matrix<Complex>;

struct RsvdParams {
  Index rank = 0;
  Index oversample = 0;  // total sample width l; 0 -> min(2*rank, min(m, n))
  int power = 4;
  std::uint64_t seed = 0;
};

template <class Scalar>
struct TruncatedFactorization {
  Matrix<Scalar> left;         // m x r
  std::vector<double> sigma;   // r
  Matrix<Scalar> right_adj;    // r x n
  double discarded_weight = 0.0;
  bool discarded_exact = true;
  Index rank() const { return static_cast<Index>(sigma.size()); }
};

namespace seed_tag {
inline constexpr std::uint64_t initial_state = 1;
inline constexpr std::uint64_t rsvd_stream = 2;
inline constexpr std::uint64_t bench_matrix = 3;
}  // namespace seed_tag

inline std::uint64_t mix64(std::uint64_t z) { return rsvd_mix64(z); }
inline std::uint64_t derive_seed(std::uint64_t s, std::uint64_t t) { return rsvd_derive_seed(s, t); }

// One engine handle per thread (the reference is re-entrant).
class Engine {
 public:
  explicit Engine(int device = 0) {
    const int rc = rsvd_create(&h_, device);
    if (rc != RSVD_OK) {
      const std::string msg = h_ ? rsvd_last_error(h_) : "rsvd_create failed";
      if (h_) rsvd_destroy(h_);
      h_ = nullptr;
      throw std::runtime_error(msg);
    }
  }
  ~Engine() {
    if (h_) rsvd_destroy(h_);
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  rsvd_handle raw() const { return h_; }

  void check(int rc) const {
    if (rc == RSVD_OK) return;
    const std::string msg = rsvd_last_error(h_);
    if (rc == RSVD_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }

 private:
  rsvd_handle h_ = nullptr;
};

inline Engine& default_engine() {
  thread_local Engine e(0);
  return e;
}

namespace detail {
template <class Scalar>
const double* dp(const Scalar* p) {
  return reinterpret_cast<const double*>(p);
}
template <class Scalar>
double* dp(Scalar* p) {
  return reinterpret_cast<double*>(p);
}
template <class Scalar>
constexpr bool is_complex() {
  return std::is_same_v<Scalar, Complex>;
}
// Copy the leading r columns / rows of the engine's k-wide outputs.
template <class Scalar>
TruncatedFactorization<Scalar> trim(const Matrix<Scalar>& u, const std::vector<double>& s,
                                    const Matrix<Scalar>& vt, Index r, double dw, bool exact) {
  TruncatedFactorization<Scalar> f;
  f.left = Matrix<Scalar>(u.rows(), r);
  for (Index j = 0; j < r; ++j)
    for (Index i = 0; i < u.rows(); ++i) f.left(i, j) = u(i, j);
  f.sigma.assign(s.begin(), s.begin() + r);
  f.right_adj = Matrix<Scalar>(r, vt.cols());
  for (Index j = 0; j < vt.cols(); ++j)
    for (Index i = 0; i < r; ++i) f.right_adj(i, j) = vt(i, j);
  f.discarded_weight = dw;
  f.discarded_exact = exact;
  return f;
}
}  // namespace detail

// rlftn::rsvd<Scalar> (factorize.cpp:76-95) on the GPU.
template <class Scalar>
TruncatedFactorization<Scalar> rsvd(const Matrix<Scalar>& a, const RsvdParams& p,
                                    Engine& e = default_engine()) {
  static_assert(std::is_same_v<Scalar, double> || detail::is_complex<Scalar>());
  const Index m = a.rows(), n = a.cols();
  const Index k = p.rank > 0 ? p.rank : 1;
  Matrix<Scalar> u(m, k), vt(k, n);
  std::vector<double> s(static_cast<size_t>(k));
  std::int64_t r = 0;
  double dw = 0.0;
  auto fn = detail::is_complex<Scalar>() ? rsvd_z128 : rsvd_f64;
  e.check(fn(e.raw(), detail::dp(a.data()), m, n, m > 0 ? m : 1, p.rank, p.oversample, p.power,
             p.seed, detail::dp(u.data()), m > 0 ? m : 1, s.data(), detail::dp(vt.data()), k, &r,
             &dw, RSVD_PTR_HOST));
  return detail::trim(u, s, vt, r, dw, false);
}

// rlftn::tsvd<Scalar> (factorize.cpp:42-50): full thin SVD truncated to chi.
template <class Scalar>
TruncatedFactorization<Scalar> tsvd(const Matrix<Scalar>& a, Index chi,
                                    Engine& e = default_engine()) {
  static_assert(std::is_same_v<Scalar, double> || detail::is_complex<Scalar>());
  const Index m = a.rows(), n = a.cols();
  Index k = chi < (m < n ? m : n) ? chi : (m < n ? m : n);
  if (k < 1) k = 1;
  Matrix<Scalar> u(m, k), vt(k, n);
  std::vector<double> s(static_cast<size_t>(k));
  std::int64_t r = 0;
  double dw = 0.0;
  auto fn = detail::is_complex<Scalar>() ? rsvd_tsvd_z128 : rsvd_tsvd_f64;
  e.check(fn(e.raw(), detail::dp(a.data()), m, n, m > 0 ? m : 1, chi, detail::dp(u.data()),
             m > 0 ? m : 1, s.data(), detail::dp(vt.data()), k, &r, &dw, RSVD_PTR_HOST));
  return detail::trim(u, s, vt, r, dw, true);
}

// rlftn::randomized_range<Scalar> (factorize.cpp:52-74).
template <class Scalar>
Matrix<Scalar> randomized_range(const Matrix<Scalar>& a, Index ell, int power, std::uint64_t seed,
                                Engine& e = default_engine()) {
  Matrix<Scalar> q(a.rows(), ell > 0 ? ell : 0);
  auto fn = detail::is_complex<Scalar>() ? rsvd_randomized_range_z128 : rsvd_randomized_range_f64;
  e.check(fn(e.raw(), detail::dp(a.data()), a.rows(), a.cols(), a.rows() > 0 ? a.rows() : 1, ell,
             power, seed, detail::dp(q.data()), a.rows() > 0 ? a.rows() : 1, RSVD_PTR_HOST));
  return q;
}

// rlftn::reconstruction_error(a, f, ErrorNorm::frobenius) (factorize.cpp:97-104).
template <class Scalar>
double reconstruction_error(const Matrix<Scalar>& a, const TruncatedFactorization<Scalar>& f,
                            Engine& e = default_engine()) {
  double out = 0.0;
  const Index r = f.rank();
  auto fn = detail::is_complex<Scalar>() ? rsvd_reconstruction_error_z128
                                         : rsvd_reconstruction_error_f64;
  e.check(fn(e.raw(), detail::dp(a.data()), a.rows(), a.cols(), a.rows(),
             r ? detail::dp(f.left.data()) : nullptr, a.rows(), r ? f.sigma.data() : nullptr,
             r ? detail::dp(f.right_adj.data()) : nullptr, r > 0 ? r : 1, r, &out,
             RSVD_PTR_HOST));
  return out;
}

// ---- blocks.hpp: block-diagonal (symmetry-sector) factorization ---------
using SectorId = int;  // blocks.hpp:14

// blocks.hpp:16-27
template <class Scalar>
struct BlockDiagMatrix {
  std::vector<SectorId> charges;
  std::vector<Matrix<Scalar>> blocks;
  Index sector_count() const { return static_cast<Index>(blocks.size()); }
};

enum class RankPolicy { per_sector_estimate, maximal };  // blocks.hpp:29-32

struct SectorRankRequest {  // blocks.hpp:36-41
  RankPolicy policy = RankPolicy::per_sector_estimate;
  Index chi = 0;
  Index slack = -1;
};

struct BlockMethod {  // blocks.hpp:49-63
  enum class Kind { tsvd, rsvd };
  Kind kind = Kind::tsvd;
  RsvdParams rsvd;
  Index rsvd_min_dim = 32;
  static BlockMethod deterministic() { return {}; }
  static BlockMethod randomized(int power = 4, std::uint64_t seed = 0) {
    BlockMethod m;
    m.kind = Kind::rsvd;
    m.rsvd.power = power;
    m.rsvd.seed = seed;
    return m;
  }
};

template <class Scalar>
struct BlockFactorization {  // blocks.hpp:68-81
  std::vector<SectorId> charges;
  std::vector<TruncatedFactorization<Scalar>> factors;
  double discarded_weight = 0.0;
  bool discarded_exact = true;
  Index total_rank() const {
    Index r = 0;
    for (const auto& f : factors) r += f.rank();
    return r;
  }
};

// rlftn::block_factorize<double> (blocks.cpp:38-118) through
// rsvd_block_factorize_f64: equal-shape sectors share one batched engine call,
// then the reference's global top-chi selection and tie-breaks.
inline BlockFactorization<double> block_factorize(const BlockDiagMatrix<double>& a, Index chi,
                                                  const SectorRankRequest& request,
                                                  const BlockMethod& method,
                                                  Engine& e = default_engine()) {
  if (a.blocks.size() != a.charges.size())  // blocks.cpp:42 (the ABI takes one count)
    throw std::invalid_argument("block_factorize: charges/blocks size mismatch");
  const Index ns = static_cast<Index>(a.blocks.size());
  std::vector<std::int64_t> ch(a.charges.begin(), a.charges.end()), rows(ns), cols(ns), ld(ns),
      ldu(ns), ldvt(ns), rank(ns);
  std::vector<const double*> in(ns);
  std::vector<Matrix<double>> u(ns), vt(ns);
  std::vector<std::vector<double>> s(ns);
  std::vector<double*> up(ns), sp(ns), vp(ns);
  std::vector<double> sdw(ns);
  for (Index i = 0; i < ns; ++i) {
    const Matrix<double>& b = a.blocks[static_cast<size_t>(i)];
    rows[i] = b.rows(), cols[i] = b.cols(), ld[i] = b.rows() > 0 ? b.rows() : 1;
    in[i] = b.data();
    const Index cap = std::max<Index>(1, std::min(std::min(b.rows(), b.cols()), chi));
    u[i] = Matrix<double>(b.rows() > 0 ? b.rows() : 1, cap);
    vt[i] = Matrix<double>(cap, b.cols() > 0 ? b.cols() : 1);
    s[i].assign(static_cast<size_t>(cap), 0.0);
    up[i] = u[i].data(), sp[i] = s[i].data(), vp[i] = vt[i].data();
    ldu[i] = u[i].rows(), ldvt[i] = cap;
  }
  double tot = 0.0;
  int exact = 1;
  e.check(rsvd_block_factorize_f64(
      e.raw(), ns, ch.data(), in.data(), rows.data(), cols.data(), ld.data(), chi,
      request.policy == RankPolicy::maximal ? 1 : 0, request.slack,
      method.kind == BlockMethod::Kind::rsvd ? 1 : 0, method.rsvd.oversample, method.rsvd.power,
      method.rsvd.seed, method.rsvd_min_dim, up.data(), ldu.data(), sp.data(), vp.data(),
      ldvt.data(), rank.data(), sdw.data(), &tot, &exact, RSVD_PTR_HOST));
  BlockFactorization<double> out;
  out.charges = a.charges;
  out.discarded_weight = tot;
  out.discarded_exact = exact != 0;
  for (Index i = 0; i < ns; ++i) {
    Matrix<double> left(rows[i], rank[i]), right(rank[i], cols[i]);
    for (Index j = 0; j < rank[i]; ++j)
      for (Index r = 0; r < rows[i]; ++r) left(r, j) = u[i](r, j);
    for (Index j = 0; j < cols[i]; ++j)
      for (Index r = 0; r < rank[i]; ++r) right(r, j) = vt[i](r, j);
    TruncatedFactorization<double> f;
    f.left = std::move(left);
    f.sigma.assign(s[i].begin(), s[i].begin() + rank[i]);
    f.right_adj = std::move(right);
    f.discarded_weight = sdw[i];
    f.discarded_exact = method.kind == BlockMethod::Kind::tsvd ||
                        std::min(rows[i], cols[i]) < method.rsvd_min_dim;
    out.factors.push_back(std::move(f));
  }
  return out;
}

}  // namespace rlftn_b200
