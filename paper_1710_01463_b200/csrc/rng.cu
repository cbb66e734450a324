// Counter-based Gaussian sketch Omega on the device.
//
// Reproduces rlftn::CounterRng (rng.hpp:34-71) as used by randomized_range
// (factorize.cpp:61-63): Omega (n x l) is filled in column-major linear order
// e = i + j*n with CounterRng(seed).normal().  Element e belongs to
// Box-Muller pair p = e/2, which consumes SplitMix64 words 2p+1 (u1, radius)
// and 2p+2 (u2, angle); even e takes r*cos(t), odd e the cached r*sin(t)
// (rng.hpp:50-60).  Being counter-based, every pair is independent, so one
// thread produces one pair: no sequential state, one read-free HBM write
// stream.  The 64-bit words are bit-exact; log/sin/cos come from the device
// libm (<= 1-2 ulp from glibc's), see DESIGN.md §RNG for the measured match.
#include "common.cuh"

namespace rsvd {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform_from(uint64_t w) {
  return static_cast<double>((w >> 11) + 1) * 0x1.0p-53;  // (0, 1], rng.hpp:46
}

// Box-Muller pair p of the stream `seed`: (r cos t, r sin t).
__device__ __forceinline__ void normal_pair(uint64_t seed, uint64_t p, double& c, double& s) {
  const uint64_t kGolden = 0x9e3779b97f4a7c15ull;
  const double u1 = uniform_from(mix64(seed + (2 * p + 1) * kGolden));
  const double u2 = uniform_from(mix64(seed + (2 * p + 2) * kGolden));
  const double r = sqrt(-2.0 * log(u1));
  const double t = (2.0 * 3.141592653589793) * u2;
  double sn, cs;
  sincos(t, &sn, &cs);
  c = __dmul_rn(r, cs);
  s = __dmul_rn(r, sn);
}

__global__ void fill_gaussian_kernel(double* __restrict__ out, int64_t ld, int64_t stride,
                                     int64_t rows, int64_t cols, int64_t valid_cols,
                                     const uint64_t* __restrict__ seeds, int64_t batch) {
  const int64_t valid = rows * valid_cols;
  const int64_t pairs = (valid + 1) / 2;
  const int64_t zero_elems = rows * (cols - valid_cols);
  const int64_t work = pairs + zero_elems;
  const int64_t total = work * batch;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = w / work;
    const int64_t x = w - b * work;
    double* o = out + b * stride;
    if (x < pairs) {
      double c, s;
      normal_pair(seeds[b], static_cast<uint64_t>(x), c, s);
      const int64_t e0 = 2 * x, e1 = e0 + 1;
      {
        const int64_t j = e0 / rows, i = e0 - j * rows;
        o[i + j * ld] = c;
      }
      if (e1 < valid) {
        const int64_t j = e1 / rows, i = e1 - j * rows;
        o[i + j * ld] = s;
      }
    } else {
      const int64_t z = x - pairs;
      const int64_t j = valid_cols + z / rows, i = z % rows;
      o[i + j * ld] = 0.0;
    }
  }
}

__global__ void fill_flat_kernel(double* __restrict__ out, int64_t count, uint64_t seed) {
  const int64_t pairs = (count + 1) / 2;
  for (int64_t x = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < pairs;
       x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double c, s;
    normal_pair(seed, static_cast<uint64_t>(x), c, s);
    out[2 * x] = c;
    if (2 * x + 1 < count) out[2 * x + 1] = s;
  }
}

}  // namespace

void launch_fill_gaussian(MatRef out, int64_t rows, int64_t cols, int64_t valid_cols,
                          const uint64_t* seeds_dev, int64_t batch, cudaStream_t st) {
  if (rows <= 0 || cols <= 0 || batch <= 0) return;
  const int64_t work = ((rows * valid_cols + 1) / 2 + rows * (cols - valid_cols)) * batch;
  const int threads = 256;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(work, threads), 16 * num_sms()));
  fill_gaussian_kernel<<<blocks, threads, 0, st>>>(out.base, out.ld, out.stride, rows, cols,
                                                   valid_cols, seeds_dev, batch);
  RSVD_LAUNCH("fill_gaussian_kernel");
}

void launch_fill_gaussian_flat(double* out, int64_t count, uint64_t seed, cudaStream_t st) {
  if (count <= 0) return;
  const int threads = 256;
  const int blocks =
      static_cast<int>(std::min<int64_t>(ceil_div((count + 1) / 2, threads), 16 * num_sms()));
  fill_flat_kernel<<<blocks, threads, 0, st>>>(out, count, seed);
  RSVD_LAUNCH("fill_flat_kernel");
}

}  // namespace rsvd
