// ORACLE — TEST INFRASTRUCTURE ONLY.
// Known-answer dump of the REFERENCE CounterRng, compiled directly against
// /root/reference/proj/include/rlftn/rng.hpp (header-only, no Eigen) by
// oracle/Makefile into oracle/_ref/rng_kat.  Prints, per seed, the first
// words and normals as exact hex so tests can pin the oracle restatement and
// the device generator bit-for-bit against the reference's own code.
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "rlftn/rng.hpp"

int main(int argc, char** argv) {
  const int nwords = argc > 1 ? std::atoi(argv[1]) : 16;
  const int nnormal = argc > 2 ? std::atoi(argv[2]) : 33;
  const std::uint64_t seeds[] = {0ull, 1ull, 42ull, 0xdeadbeefcafef00dull,
                                 rlftn::derive_seed(1, rlftn::seed_tag::rsvd_stream),
                                 rlftn::derive_seed(5, rlftn::seed_tag::rsvd_stream)};
  std::printf("{\n \"mix64\": [");
  for (std::uint64_t t = 0; t < 8; ++t)
    std::printf("%s\"%016" PRIx64 "\"", t ? ", " : "", rlftn::mix64(t));
  std::printf("],\n \"streams\": [\n");
  for (std::size_t s = 0; s < sizeof(seeds) / sizeof(seeds[0]); ++s) {
    rlftn::CounterRng w(seeds[s]);
    std::printf("  {\"seed\": \"%016" PRIx64 "\", \"words\": [", seeds[s]);
    for (int i = 0; i < nwords; ++i) std::printf("%s\"%016" PRIx64 "\"", i ? ", " : "", w.next());
    rlftn::CounterRng g(seeds[s]);
    std::printf("], \"normals\": [");
    for (int i = 0; i < nnormal; ++i) {
      const double v = g.normal();
      std::uint64_t bits;
      std::memcpy(&bits, &v, 8);
      std::printf("%s\"%016" PRIx64 "\"", i ? ", " : "", bits);
    }
    // Complex fill (rng.hpp:66-71): which Box-Muller value lands in re / im
    // depends on the compiler's argument evaluation order, so it is dumped
    // from the reference's own header as built here (g++).
    rlftn::CounterRng c(seeds[s]);
    std::vector<std::complex<double>> z(static_cast<std::size_t>(nnormal));
    c.fill_gaussian(z.data(), z.size());
    std::printf("], \"complex\": [");
    for (int i = 0; i < nnormal; ++i) {
      std::uint64_t br, bi;
      const double re = z[static_cast<std::size_t>(i)].real(), im = z[static_cast<std::size_t>(i)].imag();
      std::memcpy(&br, &re, 8);
      std::memcpy(&bi, &im, 8);
      std::printf("%s\"%016" PRIx64 "\", \"%016" PRIx64 "\"", i ? ", " : "", br, bi);
    }
    std::printf("]}%s\n", s + 1 < sizeof(seeds) / sizeof(seeds[0]) ? "," : "");
  }
  std::printf(" ]\n}\n");
  return 0;
}
