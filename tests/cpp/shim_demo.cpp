// Drop-in demo / test of include/rsvd_b200.hpp: the reference's
// "tsvd keeps the leading values" and "rsvd matches tsvd" checks written
// against the C++ shim exactly as a reference caller would (test_factorize.cpp).
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "rsvd_b200.hpp"

using namespace rlftn_b200;

int main() {
  // Rank-3 diagonal-ish test: A = diag(3, 2, 1) padded into 40 x 30 with an
  // orthogonal mix would need a QR; keep it simple: a scaled diagonal.
  MatrixR a(40, 30);
  for (Index i = 0; i < 30; ++i) a(i, i) = std::pow(0.5, static_cast<double>(i));
  const auto f = rsvd(a, RsvdParams{5, 12, 2, 7});
  if (f.rank() != 5) { std::printf("FAIL rank %lld\n", (long long)f.rank()); return 1; }
  for (Index k = 0; k < 5; ++k) {
    const double want = std::pow(0.5, static_cast<double>(k));
    if (std::abs(f.sigma[k] - want) > 1e-12 * want) { std::printf("FAIL sigma %lld\n", (long long)k); return 1; }
  }
  double tail = 0.0;
  for (Index k = 5; k < 30; ++k) tail += std::pow(0.25, static_cast<double>(k));
  const double err = reconstruction_error(a, f);
  if (std::abs(err * err - tail) > 1e-10 * tail) { std::printf("FAIL err %.17g vs %.17g\n", err * err, tail); return 1; }
  try {
    (void)rsvd(a, RsvdParams{3, 2, 4, 1});
    std::printf("FAIL no throw\n");
    return 1;
  } catch (const std::invalid_argument& e) {
    if (std::string(e.what()) != "rsvd: oversample must be >= rank") { std::printf("FAIL msg %s\n", e.what()); return 1; }
  }
  // tsvd keeps the leading values exactly (test_factorize.cpp:33-55).
  MatrixR d(3, 3);
  d(0, 0) = 3.0, d(1, 1) = 2.0, d(2, 2) = 1.0;
  const auto t = tsvd(d, 2);
  if (t.rank() != 2 || std::abs(t.sigma[0] - 3.0) > 1e-14 || std::abs(t.sigma[1] - 2.0) > 1e-14 ||
      std::abs(t.discarded_weight - 1.0) > 1e-14 || !t.discarded_exact) {
    std::printf("FAIL tsvd\n");
    return 1;
  }
  // Complex instantiation (factorize.cpp:106-118): a phase-twisted diagonal.
  MatrixC z(24, 20);
  for (Index i = 0; i < 20; ++i)
    z(i, i) = std::polar(std::pow(0.5, static_cast<double>(i)), 0.3 * static_cast<double>(i));
  const auto fz = rsvd(z, RsvdParams{6, 12, 2, 3});
  const auto tz = tsvd(z, 6);
  for (Index k = 0; k < 6; ++k) {
    const double want = std::pow(0.5, static_cast<double>(k));
    if (std::abs(fz.sigma[k] - want) > 1e-12 * want || std::abs(tz.sigma[k] - want) > 1e-12 * want) {
      std::printf("FAIL complex sigma %lld\n", (long long)k);
      return 1;
    }
  }
  double ztail = 0.0;
  for (Index k = 6; k < 20; ++k) ztail += std::pow(0.25, static_cast<double>(k));
  const double zerr = reconstruction_error(z, tz);
  if (std::abs(zerr * zerr - ztail) > 1e-10 * ztail) { std::printf("FAIL complex err\n"); return 1; }
  const auto q = randomized_range(z, 8, 1, 5);
  if (q.rows() != 24 || q.cols() != 8) { std::printf("FAIL range shape\n"); return 1; }
  // block_factorize (test_blocks.cpp:82-95, 114-140): global selection of the
  // chi largest values across sectors, exact ties to the lower charge.
  BlockDiagMatrix<double> bd;
  bd.charges = {7, 3};
  bd.blocks.resize(2, MatrixR(2, 2));
  for (auto& b : bd.blocks) b(0, 0) = 2.0, b(1, 1) = 1.0;
  SectorRankRequest req;
  req.policy = RankPolicy::maximal;
  const auto bf = block_factorize(bd, 3, req, BlockMethod::deterministic());
  if (bf.factors[0].rank() != 1 || bf.factors[1].rank() != 2 ||
      std::abs(bf.discarded_weight - 1.0) > 1e-14 || !bf.discarded_exact) {
    std::printf("FAIL block_factorize ties\n");
    return 1;
  }
  // randomized sectors of equal shape share one batched engine call
  BlockDiagMatrix<double> big;
  big.charges = {0, 1, 2};
  for (int s = 0; s < 3; ++s) {
    MatrixR b(48, 40);
    for (Index i = 0; i < 40; ++i) b(i, i) = std::pow(0.7, static_cast<double>(i)) * (1.0 + s);
    big.blocks.push_back(b);
  }
  const auto rb = block_factorize(big, 12, SectorRankRequest{}, BlockMethod::randomized(2, 9));
  if (rb.total_rank() != 12 || rb.discarded_exact || std::abs(rb.factors[2].sigma[0] - 3.0) > 1e-12) {
    std::printf("FAIL block_factorize rsvd (rank %lld)\n", (long long)rb.total_rank());
    return 1;
  }
  try {
    BlockDiagMatrix<double> dup;
    dup.charges = {1, 1};
    dup.blocks.resize(2, MatrixR(2, 2));
    (void)block_factorize(dup, 2, SectorRankRequest{}, BlockMethod::deterministic());
    std::printf("FAIL no throw (duplicate)\n");
    return 1;
  } catch (const std::invalid_argument& ex) {
    if (std::string(ex.what()) != "block_factorize: duplicate sector charge") {
      std::printf("FAIL msg %s\n", ex.what());
      return 1;
    }
  }
  std::printf("shim ok: sigma0=%.3f rank=%lld err^2=%.6e complex err^2=%.6e\n", f.sigma[0],
              (long long)f.rank(), err * err, zerr * zerr);
  return 0;
}
