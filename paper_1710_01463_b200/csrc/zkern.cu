// Complex (std::complex<double>) instantiation of the RSVD path: the device
// kernels that are specific to complex arithmetic.  The reference instantiates
// rsvd / tsvd / randomized_range for Complex (factorize.cpp:106-118) on top of
// zgemm, zgeqrf+zungqr and zgesdd (lapack.cpp:73-110, 154-177).
//
// Layouts (see zpath.inc for the pipeline):
//   I-layout  the caller's complex128 column-major matrix; viewed as a real
//             (2 rows) x cols matrix with interleaved (re, im) rows ("A-hat").
//   P-layout  a complex rows x l basis stored as a real rows x 2lp matrix:
//             column 2j = Re x_j, column 2j+1 = Im x_j.  Every small complex
//             product is then a real GEMM against a realified right factor
//             M~ (M~[2a,2c] = Re M, M~[2a+1,2c] = -Im M, M~[2a,2c+1] = Im M,
//             M~[2a+1,2c+1] = Re M), so (X M)_P = X_P M~, and the CholeskyQR
//             Gram of X is read off the real Gram X_P^T X_P.
//   PAIR      the real 2 rows x 2lp matrix [x^_j, (-i x_j)^] (interleaved):
//             A-hat^T PAIR(Q) = (A^H Q)_P, the TN A-pass, lands in P-layout.
#include <cfloat>

#include <cooperative_groups.h>

#include "common.cuh"

namespace rsvd {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform_from(uint64_t w) {
  return static_cast<double>((w >> 11) + 1) * 0x1.0p-53;
}

unsigned grid_for(int64_t work, int threads, int cap_per_sm = 8) {
  return static_cast<unsigned>(
      std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, threads), cap_per_sm * num_sms())));
}

// ---------------------------------------------------------------- Omega
// Complex CounterRng fill (rng.hpp:66-71) of Omega (n x l) in column-major
// linear order: entry t = i + j n takes Box-Muller pair t, i.e. words 2t+1
// (radius) and 2t+2 (angle).  g++ evaluates the imaginary constructor
// argument first, so re = (r sin) / sqrt 2 and im = (r cos) / sqrt 2 (pinned by
// the reference-built KAT, tests/golden/rng_kat.json "complex").
// Written to P-layout; columns j >= l are zero.
// tan of the Jacobi angle, t = sign(d) 2g / (|d| + sqrt(d^2 + 4g^2)), with
// a hardware reciprocal refined by two Newton steps instead of the IEEE
// division (~1e-15 relative instead of 0.5 ulp): t only decides how well the
// pair is annihilated, while c = (1 + t^2)^-1/2 and s = c t stay orthonormal
// to working precision whatever t is.  Saves ~60 cycles of the rotation
// chain per step.
__device__ __forceinline__ double zjacobi_tan(double d, double g2) {
  const double den = fabs(d) + sqrt(fma(d, d, g2 * g2));
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
  r = r * fma(-den, r, 2.0);
  r = r * fma(-den, r, 2.0);
  return copysign(1.0, d) * g2 * r;
}

__global__ void zfill_kernel(double* __restrict__ out, int64_t ld, int64_t stride, int64_t rows,
                             int64_t lp, int64_t ell, const uint64_t* __restrict__ seeds,
                             int64_t batch) {
  const int64_t per = rows * lp;
  const int64_t total = per * batch;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = w / per, x = w - b * per;
    const int64_t j = x / rows, i = x - j * rows;
    double re = 0.0, im = 0.0;
    if (j < ell) {
      const uint64_t t = static_cast<uint64_t>(i + j * rows);
      const uint64_t kGolden = 0x9e3779b97f4a7c15ull;
      const double u1 = uniform_from(mix64(seeds[b] + (2 * t + 1) * kGolden));
      const double u2 = uniform_from(mix64(seeds[b] + (2 * t + 2) * kGolden));
      const double r = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincos((2.0 * 3.141592653589793) * u2, &sn, &cs);
      constexpr double inv_sqrt2 = 0.70710678118654752440;
      re = __dmul_rn(__dmul_rn(r, sn), inv_sqrt2);
      im = __dmul_rn(__dmul_rn(r, cs), inv_sqrt2);
    }
    double* o = out + b * stride;
    o[i + (2 * j) * ld] = re;
    o[i + (2 * j + 1) * ld] = im;
  }
}

__global__ void zfill_flat_kernel(double2* __restrict__ out, int64_t count, uint64_t seed) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < count;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t kGolden = 0x9e3779b97f4a7c15ull;
    const double u1 = uniform_from(mix64(seed + (2 * t + 1) * kGolden));
    const double u2 = uniform_from(mix64(seed + (2 * t + 2) * kGolden));
    const double r = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincos((2.0 * 3.141592653589793) * u2, &sn, &cs);
    constexpr double inv_sqrt2 = 0.70710678118654752440;
    out[t] = make_double2(__dmul_rn(__dmul_rn(r, sn), inv_sqrt2),
                          __dmul_rn(__dmul_rn(r, cs), inv_sqrt2));
  }
}

// -------------------------------------------------------- layout glue
// NN A-pass combine: Pm = A-hat X_P (2m x 2lp; column 2j = (A Re x_j)^,
// 2j+1 = (A Im x_j)^) -> Y = A x_j in P-layout:
//   Re y = Re(P_2j) - Im(P_2j+1),  Im y = Im(P_2j) + Re(P_2j+1).
__global__ void zcombine_nn_kernel(const double* __restrict__ P, int64_t ldp, int64_t sp,
                                   double* __restrict__ Y, int64_t ldy, int64_t sy, int64_t m,
                                   int64_t lp, int64_t batch) {
  const int64_t per = m * lp, total = per * batch;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = w / per, x = w - b * per;
    const int64_t j = x / m, i = x - j * m;
    const double* pb = P + b * sp;
    const double2 p0 = *reinterpret_cast<const double2*>(pb + 2 * i + (2 * j) * ldp);
    const double2 p1 = *reinterpret_cast<const double2*>(pb + 2 * i + (2 * j + 1) * ldp);
    double* yb = Y + b * sy;
    yb[i + (2 * j) * ldy] = p0.x - p1.y;
    yb[i + (2 * j + 1) * ldy] = p0.y + p1.x;
  }
}

// PAIR(Q): P-layout Q (m x 2lp) -> real 2m x 2lp with column 2j = q^_j and
// column 2j+1 = (-i q_j)^ = (Im q, -Re q) interleaved.
__global__ void zpair_kernel(const double* __restrict__ Q, int64_t ldq, int64_t sq,
                             double* __restrict__ out, int64_t ldo, int64_t so, int64_t m,
                             int64_t lp, int64_t batch) {
  const int64_t per = m * lp, total = per * batch;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = w / per, x = w - b * per;
    const int64_t j = x / m, i = x - j * m;
    const double re = Q[b * sq + i + (2 * j) * ldq], im = Q[b * sq + i + (2 * j + 1) * ldq];
    double* ob = out + b * so;
    *reinterpret_cast<double2*>(ob + 2 * i + (2 * j) * ldo) = make_double2(re, im);
    *reinterpret_cast<double2*>(ob + 2 * i + (2 * j + 1) * ldo) = make_double2(im, -re);
  }
}

// P-layout -> I-layout (rows x cols complex): out[i, c] = X[i, 2c] + i X[i, 2c+1].
__global__ void zp2i_kernel(const double* __restrict__ X, int64_t ldx, int64_t sx,
                            double* __restrict__ out, int64_t ldo, int64_t so, int64_t rows,
                            int64_t cols, int64_t batch) {
  const int64_t per = rows * cols, total = per * batch;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = w / per, x = w - b * per;
    const int64_t c = x / rows, i = x - c * rows;
    const double re = X[b * sx + i + (2 * c) * ldx], im = X[b * sx + i + (2 * c + 1) * ldx];
    *reinterpret_cast<double2*>(out + b * so + 2 * i + c * ldo) = make_double2(re, im);
  }
}

// I-layout -> P-layout (rows x cols complex).
__global__ void zi2p_kernel(const double* __restrict__ X, int64_t ldx, int64_t sx,
                            double* __restrict__ out, int64_t ldo, int64_t so, int64_t rows,
                            int64_t cols, int64_t batch) {
  const int64_t per = rows * cols, total = per * batch;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = w / per, x = w - b * per;
    const int64_t c = x / rows, i = x - c * rows;
    const double2 v = *reinterpret_cast<const double2*>(X + b * sx + 2 * i + c * ldx);
    out[b * so + i + (2 * c) * ldo] = v.x;
    out[b * so + i + (2 * c + 1) * ldo] = v.y;
  }
}

// Conjugate transpose, P-layout in (rows x cols complex) -> I-layout out
// (cols x rows complex): out[c, i] = conj(X[i, c]).  32 x 32 complex tiles.
__global__ void zadj_p2i_kernel(const double* __restrict__ X, int64_t ldx, int64_t sx,
                                double* __restrict__ out, int64_t ldo, int64_t so, int64_t rows,
                                int64_t cols) {
  __shared__ double2 tile[32][33];
  const int64_t b = blockIdx.z;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32, c0 = static_cast<int64_t>(blockIdx.y) * 32;
  const double* src = X + b * sx;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + threadIdx.x, c = c0 + y;
    double2 v = make_double2(0.0, 0.0);
    if (r < rows && c < cols) v = make_double2(src[r + (2 * c) * ldx], -src[r + (2 * c + 1) * ldx]);
    tile[y][threadIdx.x] = v;
  }
  __syncthreads();
  double* dst = out + b * so;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + threadIdx.x, r = r0 + y;  // out(c, r) = conj(X(r, c))
    if (c < cols && r < rows) *reinterpret_cast<double2*>(dst + 2 * c + r * ldo) = tile[threadIdx.x][y];
  }
}

// Conjugate transpose in I-layout (rows x cols -> cols x rows).
__global__ void zadj_i2i_kernel(const double* __restrict__ X, int64_t ldx, int64_t sx,
                                double* __restrict__ out, int64_t ldo, int64_t so, int64_t rows,
                                int64_t cols) {
  __shared__ double2 tile[32][33];
  const int64_t b = blockIdx.z;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32, c0 = static_cast<int64_t>(blockIdx.y) * 32;
  const double* src = X + b * sx;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + threadIdx.x, c = c0 + y;
    double2 v = make_double2(0.0, 0.0);
    if (r < rows && c < cols) {
      v = *reinterpret_cast<const double2*>(src + 2 * r + c * ldx);
      v.y = -v.y;
    }
    tile[y][threadIdx.x] = v;
  }
  __syncthreads();
  double* dst = out + b * so;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + threadIdx.x, r = r0 + y;
    if (c < cols && r < rows) *reinterpret_cast<double2*>(dst + 2 * c + r * ldo) = tile[threadIdx.x][y];
  }
}

// Identity in P-layout (rows x l complex, l <= rows): X[i, 2i] = 1.
__global__ void zidentity_p_kernel(double* __restrict__ X, int64_t ld, int64_t stride, int64_t rows,
                                   int64_t lp, int64_t ell, int64_t batch) {
  const int64_t per = rows * 2 * lp, total = per * batch;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = w / per, x = w - b * per;
    const int64_t c = x / rows, i = x - c * rows;
    X[b * stride + i + c * ld] = (c % 2 == 0 && c / 2 == i && i < ell) ? 1.0 : 0.0;
  }
}

// Realified Hermitian Gram, in place.  In: Gt = X_P^T X_P (2lp x 2lp real,
// symmetric).  Out: the realification of G = X^H X in the M~ convention,
//   G_ac = Gt[2a,2c] + Gt[2a+1,2c+1] + i (Gt[2a,2c+1] - Gt[2a+1,2c]),
// whose real Cholesky factor is exactly the realified complex factor R~
// (realification is a *-homomorphism and R~ is upper triangular with
// diagonal blocks r I), so the real CholeskyQR machinery orthonormalises the
// complex basis X_P (engine.cu orth(..., cplx = true)).
__global__ void hermitize_kernel(double* __restrict__ G, int64_t lp, const int* __restrict__ mask) {
  const int64_t b = blockIdx.y;
  if (mask && !mask[b]) return;
  const int64_t L = 2 * lp;
  double* g = G + b * L * L;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < lp * lp;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = e % lp, c = e / lp;
    double* p0 = g + 2 * a + (2 * c) * L;  // column 2c, rows 2a, 2a+1
    double* p1 = g + 2 * a + (2 * c + 1) * L;
    const double2 c0 = *reinterpret_cast<const double2*>(p0);
    const double2 c1 = *reinterpret_cast<const double2*>(p1);
    const double gr = c0.x + c1.y;
    const double gi = a == c ? 0.0 : c1.x - c0.y;
    *reinterpret_cast<double2*>(p0) = make_double2(gr, -gi);
    *reinterpret_cast<double2*>(p1) = make_double2(gi, gr);
  }
}

// ------------------------------------------------------ complex Jacobi
// One-sided (Hestenes) Jacobi on the complex l x l factor H (factorize.cpp:88
// -> lapack::svd of B, here of Rt^H): columns p, q with alpha = |h_p|^2,
// beta = |h_q|^2, gamma = h_p^H h_q = |gamma| e: the real rotation of
// (h_p, conj(e) h_q) (zeta = (beta - alpha) / 2|gamma|, t = sign(zeta) /
// (|zeta| + sqrt(1 + zeta^2))) gives h_p' = c h_p - s conj(e) h_q,
// h_q' = s e h_p + c h_q; J accumulates the same unitary 2 x 2.  Rotation test
// |gamma| > sqrt(l) eps sqrt(alpha beta) (dgesvj's); round-robin ordering,
// every pair once per sweep; stops after a sweep with no rotation or whose
// largest rotated ratio was below 1e-7 (quadratic convergence).
// Each item is owned by a thread-block cluster of S CTAs (S = 1 for large
// batches): the l/2 disjoint pairs of a round-robin step are spread over the
// S x 16 warps, one cluster barrier per step; H and J live in global scratch
// (L2), read with ld.global.cg so no CTA sees a stale L1 line.  RPL > 0 keeps
// each warp's two columns in registers (RPL complex rows per lane) between
// the dot products and the rotation; RPL = 0 streams them twice.
//   src_mode 0: H = Rt^H from the realified R~t (2lp x 2lp);
//   src_mode 1: H from a P-layout l x 2lp matrix (tsvd: H = A_e Qb).
__device__ __forceinline__ double2 ldcg2(const double2* p) { return __ldcg(p); }

template <int RPL>
__global__ void __launch_bounds__(512) zjacobi_kernel(const double* __restrict__ src,
                                                      int64_t src_ld, int64_t src_stride,
                                                      int src_mode, double2* __restrict__ H,
                                                      double2* __restrict__ J, int ell,
                                                      int64_t lp, int max_sweeps,
                                                      int* __restrict__ sweeps_out, int S) {
  namespace cg = cooperative_groups;
  const int crank = S > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
  const int64_t b = blockIdx.x / S;
  double2* Hb = H + b * lp * lp;
  double2* Jb = J + b * lp * lp;
  const double* Sb = src + b * src_stride;
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  auto sync_all = [&] {
    if (S > 1)
      cg::this_cluster().sync();
    else
      __syncthreads();
  };
  for (int64_t e = static_cast<int64_t>(crank) * nt + tid; e < lp * lp;
       e += static_cast<int64_t>(S) * nt) {
    const int a = static_cast<int>(e % lp), c = static_cast<int>(e / lp);
    double2 h = make_double2(0.0, 0.0);
    if (a < ell && c < ell) {
      if (src_mode == 0)  // H[a, c] = conj(Rt[c, a]) = Rt~[2c, 2a] + i Rt~[2c+1, 2a]
        h = make_double2(Sb[2 * c + (2 * a) * src_ld], Sb[2 * c + 1 + (2 * a) * src_ld]);
      else
        h = make_double2(Sb[a + (2 * c) * src_ld], Sb[a + (2 * c + 1) * src_ld]);
    }
    Hb[e] = h;
    Jb[e] = make_double2(a == c ? 1.0 : 0.0, 0.0);
  }
  __shared__ unsigned long long s_max;  // largest rotated ratio of the sweep (bits of a double >= 0)
  __shared__ int s_rot;
  const int le = ell + (ell & 1);
  const double tol = sqrt(static_cast<double>(ell)) * DBL_EPSILON;
  const int gw = crank * nw + warp, tw = S * nw;
  int sweep = 0;
  if (tid == 0) s_max = 0ull, s_rot = 0;
  sync_all();
  for (; sweep < max_sweeps && ell > 1; ++sweep) {
    for (int step = 0; step < le - 1; ++step) {
      for (int k = gw; k < le / 2; k += tw) {
        const int pp = k == 0 ? 0 : ((k - 1 + step) % (le - 1)) + 1;
        const int qq = ((le - 2 - k + step) % (le - 1)) + 1;
        if (pp >= ell || qq >= ell) continue;
        const int pc = min(pp, qq), qc = max(pp, qq);
        double2* hp = Hb + pc * lp;
        double2* hq = Hb + qc * lp;
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
        double2 xr[RPL > 0 ? RPL : 1], yr[RPL > 0 ? RPL : 1];
        if (RPL > 0) {
#pragma unroll
          for (int r = 0; r < (RPL > 0 ? RPL : 1); ++r) {
            const int i = lane + 32 * r;
            xr[r] = i < ell ? ldcg2(hp + i) : make_double2(0.0, 0.0);
            yr[r] = i < ell ? ldcg2(hq + i) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int r = 0; r < (RPL > 0 ? RPL : 1); ++r) {
            const double2 x = xr[r], y = yr[r];
            al = fma(x.x, x.x, fma(x.y, x.y, al));
            be = fma(y.x, y.x, fma(y.y, y.y, be));
            gr = fma(x.x, y.x, fma(x.y, y.y, gr));
            gi = fma(x.x, y.y, fma(-x.y, y.x, gi));
          }
        } else {
          for (int i = lane; i < ell; i += 32) {
            const double2 x = ldcg2(hp + i), y = ldcg2(hq + i);
            al = fma(x.x, x.x, fma(x.y, x.y, al));
            be = fma(y.x, y.x, fma(y.y, y.y, be));
            gr = fma(x.x, y.x, fma(x.y, y.y, gr));
            gi = fma(x.x, y.y, fma(-x.y, y.x, gi));
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          gr += __shfl_xor_sync(0xffffffffu, gr, o);
          gi += __shfl_xor_sync(0xffffffffu, gi, o);
        }
        const double g = hypot(gr, gi);
        const double nrm = sqrt(al) * sqrt(be);
        if (!(g > tol * nrm) || g == 0.0) continue;
        if (lane == 0) {
          atomicMax(&s_max, static_cast<unsigned long long>(__double_as_longlong(g / nrm)));
          s_rot = 1;
        }
        const double zeta = (be - al) / (2.0 * g);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        const double er = gr / g, ei = gi / g;  // e = gamma / |gamma|
        // h_p' = c h_p - s conj(e) h_q ; h_q' = s e h_p + c h_q
        auto rot = [&](double2 x, double2 y, double2& xo, double2& yo) {
          const double2 ey = make_double2(er * y.x + ei * y.y, er * y.y - ei * y.x);  // conj(e) y
          const double2 ex = make_double2(er * x.x - ei * x.y, er * x.y + ei * x.x);  // e x
          xo = make_double2(c * x.x - sn * ey.x, c * x.y - sn * ey.y);
          yo = make_double2(sn * ex.x + c * y.x, sn * ex.y + c * y.y);
        };
        if (RPL > 0) {
#pragma unroll
          for (int r = 0; r < (RPL > 0 ? RPL : 1); ++r) {
            const int i = lane + 32 * r;
            if (i < ell) {
              double2 xo, yo;
              rot(xr[r], yr[r], xo, yo);
              hp[i] = xo;
              hq[i] = yo;
            }
          }
        } else {
          for (int i = lane; i < ell; i += 32) {
            double2 xo, yo;
            rot(ldcg2(hp + i), ldcg2(hq + i), xo, yo);
            hp[i] = xo;
            hq[i] = yo;
          }
        }
        double2* jp = Jb + pc * lp;
        double2* jq = Jb + qc * lp;
        for (int i = lane; i < ell; i += 32) {
          double2 xo, yo;
          rot(ldcg2(jp + i), ldcg2(jq + i), xo, yo);
          jp[i] = xo;
          jq[i] = yo;
        }
      }
      sync_all();
    }
    // Cluster-wide decision: every CTA reads every CTA's flags (identical result).
    bool any = false;
    double mx = 0.0;
    if (S > 1) {
      cg::cluster_group cl = cg::this_cluster();
      for (int r = 0; r < S; ++r) {
        any = any || (*cl.map_shared_rank(&s_rot, r) != 0);
        mx = fmax(mx, __longlong_as_double(static_cast<long long>(*cl.map_shared_rank(&s_max, r))));
      }
    } else {
      any = s_rot != 0;
      mx = __longlong_as_double(static_cast<long long>(s_max));
    }
    sync_all();
    if (tid == 0) s_max = 0ull, s_rot = 0;
    sync_all();
    if (!any || mx < 1e-7) {
      ++sweep;
      break;
    }
  }
  if (crank == 0 && tid == 0 && sweeps_out) sweeps_out[b] = sweep;
}

// sigma_c = ||W e_c|| (complex columns), descending with ties by index,
// numerical rank cut (factorize.cpp:17-24) r = min(k, rank), discarded weight
// over the sampled tail (factorize.cpp:30-31).
__global__ void zfinalize_kernel(const double2* __restrict__ W, int64_t lp, int ell, int64_t k,
                                 int64_t m, int64_t n, double* __restrict__ sigma_out,
                                 int* __restrict__ perm, int* __restrict__ rank_out,
                                 double* __restrict__ dw_out) {
  extern __shared__ double s_sig[];
  int* s_pos = reinterpret_cast<int*>(s_sig + lp);
  const int64_t b = blockIdx.x;
  const double2* Wb = W + b * lp * lp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = warp; c < ell; c += nw) {
    double s = 0.0;
    for (int r = lane; r < ell; r += 32) {
      const double2 x = Wb[r + c * lp];
      s = fma(x.x, x.x, fma(x.y, x.y, s));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) s_sig[c] = sqrt(s);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ell; c += blockDim.x) {
    const double v = s_sig[c];
    int pos = 0;
    for (int d = 0; d < ell; ++d) {
      const double w = s_sig[d];
      pos += (w > v) || (w == v && d < c);
    }
    s_pos[c] = pos;
    perm[b * lp + pos] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // perm (global, written above by this block) maps positions to columns
    const int* pb = perm + b * lp;
    const double smax = ell > 0 ? s_sig[pb[0]] : 0.0;
    int nr = 0;
    if (smax > 0.0) {
      const double cut = static_cast<double>(m > n ? m : n) * DBL_EPSILON * smax;
      for (int c = 0; c < ell; ++c) nr += s_sig[c] > cut;
    }
    const int r = static_cast<int>(nr < k ? nr : k);
    rank_out[b] = r;
    double dw = 0.0;
    for (int pos = r; pos < ell; ++pos) {
      const double v = s_sig[pb[pos]];
      dw += v * v;
    }
    dw_out[b] = dw;
  }
  __syncthreads();
  const int r = rank_out[b];
  for (int c = threadIdx.x; c < ell; c += blockDim.x) {
    const int pos = s_pos[c];
    if (pos < k) sigma_out[b * k + pos] = pos < r ? s_sig[c] : 0.0;
  }
  for (int pos = ell + threadIdx.x; pos < k; pos += blockDim.x) sigma_out[b * k + pos] = 0.0;
}

// Right factors of the lift, from the complex l x l W (or J) with the sorted
// column order perm and 1/sigma (sigma may be null):
//   half == 1: M (2lp x k) with M[2a, c] = Re w, M[2a+1, c] = -Im w, so that
//              PAIR(Q) M = (Q w)^ lands in I-layout;
//   half == 0: realified M~ (2lp x 2k) for a P-layout product.
// Columns c >= rank[b] are zero.
__global__ void zlift_operand_kernel(const double2* __restrict__ W, int64_t lp, const int* __restrict__ perm,
                                     const double* __restrict__ sigma, int64_t k,
                                     const int* __restrict__ rank, int ell, int half,
                                     double* __restrict__ M, int64_t ldm, int64_t sm) {
  const int64_t b = blockIdx.y;
  const int r = rank[b];
  const int64_t L = 2 * lp;
  const int64_t cols = half ? k : 2 * k;
  const int64_t total = L * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t R2 = e % L, C = e / L;
    const int a = static_cast<int>(R2 >> 1), ra = static_cast<int>(R2 & 1);
    const int c = static_cast<int>(half ? C : C >> 1), rc = static_cast<int>(half ? 0 : C & 1);
    double v = 0.0;
    if (c < r && a < ell) {
      double2 w = W[b * lp * lp + a + static_cast<int64_t>(perm[b * lp + c]) * lp];
      if (sigma) {
        const double is = 1.0 / sigma[b * k + c];
        w.x *= is;
        w.y *= is;
      }
      v = (ra == rc) ? w.x : (ra ? -w.y : w.y);
    }
    M[b * sm + R2 + C * ldm] = v;
  }
}

}  // namespace

// ------------------------------------------------------------- launchers
void launch_zfill_gaussian_p(MatRef out, int64_t rows, int64_t lp, int64_t ell,
                             const uint64_t* seeds_dev, int64_t batch, cudaStream_t st) {
  if (rows <= 0 || lp <= 0 || batch <= 0) return;
  zfill_kernel<<<grid_for(rows * lp * batch, 256), 256, 0, st>>>(out.base, out.ld, out.stride, rows,
                                                                  lp, ell, seeds_dev, batch);
  RSVD_LAUNCH("zfill_kernel");
}

void launch_zfill_gaussian_flat(double* out, int64_t count, uint64_t seed, cudaStream_t st) {
  if (count <= 0) return;
  zfill_flat_kernel<<<grid_for(count, 256, 16), 256, 0, st>>>(reinterpret_cast<double2*>(out),
                                                              count, seed);
  RSVD_LAUNCH("zfill_flat_kernel");
}

void launch_zcombine_nn(CMatRef P, MatRef Y, int64_t m, int64_t lp, int64_t batch,
                        cudaStream_t st) {
  if (m <= 0 || batch <= 0) return;
  zcombine_nn_kernel<<<grid_for(m * lp * batch, 256), 256, 0, st>>>(P.base, P.ld, P.stride, Y.base,
                                                                     Y.ld, Y.stride, m, lp, batch);
  RSVD_LAUNCH("zcombine_nn_kernel");
}

void launch_zpair(CMatRef Q, MatRef out, int64_t m, int64_t lp, int64_t batch, cudaStream_t st) {
  if (m <= 0 || batch <= 0) return;
  zpair_kernel<<<grid_for(m * lp * batch, 256), 256, 0, st>>>(Q.base, Q.ld, Q.stride, out.base,
                                                               out.ld, out.stride, m, lp, batch);
  RSVD_LAUNCH("zpair_kernel");
}

void launch_zp2i(CMatRef X, MatRef out, int64_t rows, int64_t cols, int64_t batch,
                 cudaStream_t st) {
  if (rows <= 0 || cols <= 0 || batch <= 0) return;
  zp2i_kernel<<<grid_for(rows * cols * batch, 256), 256, 0, st>>>(X.base, X.ld, X.stride, out.base,
                                                                   out.ld, out.stride, rows, cols,
                                                                   batch);
  RSVD_LAUNCH("zp2i_kernel");
}

void launch_zi2p(CMatRef X, MatRef out, int64_t rows, int64_t cols, int64_t batch,
                 cudaStream_t st) {
  if (rows <= 0 || cols <= 0 || batch <= 0) return;
  zi2p_kernel<<<grid_for(rows * cols * batch, 256), 256, 0, st>>>(X.base, X.ld, X.stride, out.base,
                                                                   out.ld, out.stride, rows, cols,
                                                                   batch);
  RSVD_LAUNCH("zi2p_kernel");
}

void launch_zadjoint(CMatRef X, bool from_p, MatRef out, int64_t rows, int64_t cols,
                     int64_t batch, cudaStream_t st) {
  if (rows <= 0 || cols <= 0 || batch <= 0) return;
  dim3 grid(static_cast<unsigned>(ceil_div(rows, 32)), static_cast<unsigned>(ceil_div(cols, 32)),
            static_cast<unsigned>(batch));
  if (from_p)
    zadj_p2i_kernel<<<grid, dim3(32, 8), 0, st>>>(X.base, X.ld, X.stride, out.base, out.ld,
                                                  out.stride, rows, cols);
  else
    zadj_i2i_kernel<<<grid, dim3(32, 8), 0, st>>>(X.base, X.ld, X.stride, out.base, out.ld,
                                                  out.stride, rows, cols);
  RSVD_LAUNCH("zadj_kernel");
}

void launch_zidentity_p(MatRef X, int64_t rows, int64_t lp, int64_t ell, int64_t batch,
                        cudaStream_t st) {
  if (rows <= 0 || batch <= 0) return;
  zidentity_p_kernel<<<grid_for(rows * 2 * lp * batch, 256), 256, 0, st>>>(X.base, X.ld, X.stride,
                                                                            rows, lp, ell, batch);
  RSVD_LAUNCH("zidentity_p_kernel");
}

void launch_hermitize(double* G, int64_t lp, const int* mask, int64_t batch, cudaStream_t st) {
  if (batch <= 0 || lp <= 0) return;
  dim3 grid(grid_for(lp * lp, 256, 2), static_cast<unsigned>(batch));
  hermitize_kernel<<<grid, 256, 0, st>>>(G, lp, mask);
  RSVD_LAUNCH("hermitize_kernel");
}


// ------------------------------------------- complex Gram-accelerated Jacobi
// Block-cyclic complex one-sided Jacobi for many items (the complex analogue
// of jacobi.cu's jacobi_gram_kernel): columns in blocks of 16; a sweep is a
// diagonal phase (every block rotates its 120 intra pairs) plus nb - 1
// round-robin block-pair phases (256 inter pairs each), so every pair is
// rotated once per sweep.  Per task (item, block pair) the 32 complex columns
// are staged in shared memory in P-layout (64 real columns), the complex Gram
// G = X^H X is formed on DMMA (Re: Re^T Re + Im^T Im, Im: Re^T Im - Im^T Re),
// the 15-16 rotation steps run on G and on the accumulated unitary V (a warp
// per pair, same complex rotation as zjacobi_kernel, exact 2 x 2 block), and
// X <- X V, J <- J V run on DMMA as the real products X_P V~ with the
// realified V.  Same rotation test and sweep stop rule as the scalar kernel;
// one cooperative grid, a grid barrier per phase.
__device__ __forceinline__ void zdmma(double (&c)[4], double a0, double a1, double b0) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}
__device__ __forceinline__ int zrr(int slot, int s, int nn) {
  return slot == 0 ? 0 : 1 + (slot - 1 + s) % (nn - 1);
}

// CLU: few tasks (single matrices) -- each task is owned by a thread-block
// cluster of S CTAs that split its rows (32 R per CTA): every CTA forms the
// partial Gram of its row slice, the S partials are summed through DSMEM in
// rank order (bit-identical G in every CTA), the rotations run redundantly and
// each CTA applies V~ to its own rows of H and J (jacobi.cu's clug scheme).
template <int R, bool CLU, int MINB>
__global__ void __launch_bounds__(512, MINB)
    zjacobi_gram_kernel(const double* __restrict__ src, int64_t src_ld, int64_t src_stride,
                        int src_mode, double2* __restrict__ H, double2* __restrict__ J, int ell,
                        int lp, int nb, int64_t batch, int max_sweeps,
                        unsigned* __restrict__ flags, int* __restrict__ sweeps_out) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int W = 16, NC = 32, RC = 64, GP = NC + 1;
  // Rows staged per CTA: the 32 R slice of a cluster, else l rounded up to
  // 16 (C2-shaped l = 138 -> 144: 108 KB of staging, two CTAs per SM).
  const int rows = CLU ? 32 * R : min(32 * R, (ell + 15) & ~15);
  const int PITCH = rows + 2;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_rot;
  __shared__ unsigned long long s_mx;
  double* Xs = sm;                                          // RC x PITCH (P-layout)
  double2* Vs = reinterpret_cast<double2*>(Xs + RC * PITCH);  // V[k + c * GP]
  double2* Gs = Vs + NC * GP;                               // G[row + col * GP]
  double2* Gp = Gs + NC * GP;                               // CLU: this CTA's partial Gram
  int* conv = reinterpret_cast<int*>(Gp + (CLU ? NC * GP : 0));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t sq = static_cast<int64_t>(lp) * lp;
  const double tol2 = static_cast<double>(ell) * DBL_EPSILON * DBL_EPSILON;
  const int S = CLU ? static_cast<int>(cg::this_cluster().num_blocks()) : 1;
  const int crank = CLU ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
  const int row0 = crank * rows;                         // this CTA's slice of the rows
  const int lrows = max(0, min(rows, ell - row0));
  const int64_t nclu = gridDim.x / S, clu = blockIdx.x / S;

  const int64_t gtid = blockIdx.x * static_cast<int64_t>(blockDim.x) + tid;
  const int64_t gstride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = gtid; e < sq * batch; e += gstride) {
    const int64_t b = e / sq, rem = e - b * sq;
    const int a = static_cast<int>(rem % lp), c = static_cast<int>(rem / lp);
    const double* S = src + b * src_stride;
    double2 h = make_double2(0.0, 0.0);
    if (a < ell && c < ell) {
      if (src_mode == 0)
        h = make_double2(S[2 * c + (2 * a) * src_ld], S[2 * c + 1 + (2 * a) * src_ld]);
      else
        h = make_double2(S[a + (2 * c) * src_ld], S[a + (2 * c + 1) * src_ld]);
    }
    H[e] = h;
    J[e] = make_double2(a == c ? 1.0 : 0.0, 0.0);
  }
  unsigned long long* mxr =
      reinterpret_cast<unsigned long long*>(flags + ((3 * batch + 1) & ~int64_t(1)));
  for (int64_t e = gtid; e < 3 * batch; e += gstride) {
    flags[e] = 0u;
    mxr[e] = 0ull;
  }
  for (int64_t i = tid; i < batch; i += blockDim.x) conv[i] = 0;
  grid.sync();

  const int half = nb / 2;
  const int64_t tasks = batch * half;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    unsigned* fl = flags + (sweep % 3) * batch;
    unsigned long long* mxs = mxr + (sweep % 3) * batch;
    if (blockIdx.x == 0)
      for (int64_t i = tid; i < batch; i += blockDim.x) {
        flags[((sweep + 1) % 3) * batch + i] = 0u;
        mxr[((sweep + 1) % 3) * batch + i] = 0ull;
      }
    for (int phase = 0; phase < nb; ++phase) {
      const bool diag = phase == 0;
      for (int64_t task = clu; task < tasks; task += nclu) {
        const int64_t item = task / half;
        if (conv[item]) continue;
        const int k = static_cast<int>(task % half);
        int bp, bq;
        if (diag) {
          bp = 2 * k, bq = 2 * k + 1;
        } else {
          const int p = zrr(k, phase - 1, nb), q = zrr(nb - 1 - k, phase - 1, nb);
          bp = min(p, q), bq = max(p, q);
        }
        // a block-pair task whose second block is all padding has no pair
        // that can rotate (intra-block pairs belong to the diagonal phase)
        if (bp * W >= ell || (!diag && bq * W >= ell)) continue;
        double2* Hg = H + item * sq;
        double2* Jg = J + item * sq;
        auto gcol = [&](int c) { return c < W ? bp * W + c : bq * W + (c - W); };
        auto stage = [&](const double2* M) {  // I-layout global -> P-layout smem
          for (int e = tid; e < NC * rows; e += blockDim.x) {
            const int c = e / rows, r = e - c * rows;
            const int gc = gcol(c);
            double2 v = make_double2(0.0, 0.0);
            if (gc < ell && r < lrows) v = __ldcg(M + row0 + r + static_cast<int64_t>(gc) * lp);
            Xs[(2 * c) * PITCH + r] = v.x;
            Xs[(2 * c + 1) * PITCH + r] = v.y;
          }
        };
        stage(Hg);
        for (int e = tid; e < NC * GP; e += blockDim.x) {
          const int c = e / GP, r = e - c * GP;
          Vs[e] = make_double2(r == c ? 1.0 : 0.0, 0.0);
        }
        if (tid == 0) {
          s_rot = 0;
          s_mx = 0ull;
        }
        __syncthreads();
        // G = X^H X on DMMA: warps 0-7 the real part, 8-15 the imaginary part,
        // one 16 x 8 tile each (K runs over the rows twice).
        {
          const int part = warp >> 3, tw = warp & 7;
          const int tm = tw >> 2, tn = tw & 3;
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          const int a_0 = 16 * tm + g, a_1 = a_0 + 8, b_0 = 8 * tn + g;
          // pass 1: Re(a)^T Re(b) (real part) / Re(a)^T Im(b) (imaginary part)
          {
            const double* ap0 = Xs + (2 * a_0) * PITCH;
            const double* ap1 = Xs + (2 * a_1) * PITCH;
            const double* bp0 = Xs + (2 * b_0 + part) * PITCH;
#pragma unroll 4
            for (int k0 = 0; k0 < rows; k0 += 4) zdmma(acc, ap0[k0 + t4], ap1[k0 + t4], bp0[k0 + t4]);
          }
          // pass 2: Im(a)^T Im(b) (real part) / -Im(a)^T Re(b) (imaginary part)
          {
            const double* ap0 = Xs + (2 * a_0 + 1) * PITCH;
            const double* ap1 = Xs + (2 * a_1 + 1) * PITCH;
            const double* bp0 = Xs + (2 * b_0 + 1 - part) * PITCH;
            const double sg = part ? -1.0 : 1.0;
#pragma unroll 4
            for (int k0 = 0; k0 < rows; k0 += 4)
              zdmma(acc, ap0[k0 + t4], ap1[k0 + t4], sg * bp0[k0 + t4]);
          }
          const int r0 = 16 * tm + g, c0 = 8 * tn + 2 * t4;
          double* gd = reinterpret_cast<double*>(CLU ? Gp : Gs);
          gd[2 * (r0 + c0 * GP) + part] = acc[0];
          gd[2 * (r0 + (c0 + 1) * GP) + part] = acc[1];
          gd[2 * (r0 + 8 + c0 * GP) + part] = acc[2];
          gd[2 * (r0 + 8 + (c0 + 1) * GP) + part] = acc[3];
        }
        if (CLU) {  // G = sum of the S partials, in rank order
          cg::cluster_group cl = cg::this_cluster();
          cl.sync();
          for (int e = tid; e < NC * NC; e += blockDim.x) {
            const int c = e / NC, r = e - c * NC;
            double2 v = make_double2(0.0, 0.0);
            for (int rr = 0; rr < S; ++rr) {
              const double2 w = *cl.map_shared_rank(&Gp[r + c * GP], rr);
              v.x += w.x;
              v.y += w.y;
            }
            Gs[r + c * GP] = v;
          }
          cl.sync();  // every CTA has read every partial
        } else {
          __syncthreads();
        }
        int rotated = 0, big = 0;
        const int steps = diag ? 15 : 16;
        for (int s2 = 0; s2 < steps; ++s2) {
          int i, jx;
          if (diag) {
            const int blk = warp >> 3, pi = warp & 7;
            const int a0 = zrr(pi, s2, 16), b0 = zrr(15 - pi, s2, 16);
            i = blk * 16 + min(a0, b0);
            jx = blk * 16 + max(a0, b0);
          } else {
            i = warp;
            jx = 16 + ((warp + s2) & 15);
          }
          const double al = Gs[i + i * GP].x, be = Gs[jx + jx * GP].x;
          const double2 ga = Gs[i + jx * GP];
          const double gg = ga.x * ga.x + ga.y * ga.y, ab = al * be;
          const bool rot = al > 0.0 && be > 0.0 && gg > tol2 * ab;
          double c = 1.0, sn = 0.0, tt = 0.0, gm = 0.0, er = 1.0, ei = 0.0;
          if (rot) {
            big |= gg >= 1e-14 * ab;
            gm = sqrt(gg);
            er = ga.x / gm, ei = ga.y / gm;
            const double d = be - al, g2 = 2.0 * gm;
            const double mag = fmax(fabs(d), g2);
            if (mag > 1e-140 && mag < 1e140) {
              tt = zjacobi_tan(d, g2);
            } else {
              const double zeta = d / g2;
              tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
            }
            c = rsqrt(fma(tt, tt, 1.0));
            sn = c * tt;
            rotated = 1;
            // columns of G and V (lane = row): x' = c x - s conj(e) y, y' = s e x + c y
            auto colrot = [&](double2* M, int ld) {
              const double2 x = M[lane + i * ld], y = M[lane + jx * ld];
              const double2 ey = make_double2(er * y.x + ei * y.y, er * y.y - ei * y.x);
              const double2 ex = make_double2(er * x.x - ei * x.y, er * x.y + ei * x.x);
              M[lane + i * ld] = make_double2(c * x.x - sn * ey.x, c * x.y - sn * ey.y);
              M[lane + jx * ld] = make_double2(sn * ex.x + c * y.x, sn * ex.y + c * y.y);
            };
            colrot(Gs, GP);
            colrot(Vs, GP);
          }
          __syncthreads();
          if (rot) {  // rows (lane = column): row_i' = c row_i - s e row_j, row_j' = s conj(e) row_i + c row_j
            const double2 x = Gs[i + lane * GP], y = Gs[jx + lane * GP];
            const double2 ey = make_double2(er * y.x - ei * y.y, er * y.y + ei * y.x);  // e y
            const double2 ex = make_double2(er * x.x + ei * x.y, er * x.y - ei * x.x);  // conj(e) x
            Gs[i + lane * GP] = make_double2(c * x.x - sn * ey.x, c * x.y - sn * ey.y);
            Gs[jx + lane * GP] = make_double2(sn * ex.x + c * y.x, sn * ex.y + c * y.y);
            __syncwarp();
            if (lane == 0) {
              Gs[i + i * GP] = make_double2(al - tt * gm, 0.0);
              Gs[jx + jx * GP] = make_double2(be + tt * gm, 0.0);
              Gs[i + jx * GP] = make_double2(0.0, 0.0);
              Gs[jx + i * GP] = make_double2(0.0, 0.0);
            }
          }
          __syncthreads();
        }
        if (rotated && lane == 0) {
          atomicOr(&s_rot, 1);
          if (big) atomicMax(&s_mx, 1ull);
        }
        __syncthreads();
        if (s_rot) {
          // (X V)_P = X_P V~ (64 x 64 realified V), warp per 16-row slab, in two
          // halves of 32 output columns (register budget), written straight to
          // the global I-layout matrix; Xs (the staged pair) is only read.
          auto apply_v = [&](double2* Mg) {
            const int slabs = rows / 16;
            for (int sl = warp; sl < slabs; sl += W) {
              const int r0 = sl * 16;
              // two CTAs per SM (MINB 2): two passes of 32 columns in 64
              // registers; one CTA per SM: one pass of 64 columns
              constexpr int NH = MINB == 1 ? 1 : 2, NT = 8 / NH;
#pragma unroll 1
              for (int hf = 0; hf < NH; ++hf) {
                double acc[NT][4];
#pragma unroll
                for (int n = 0; n < NT; ++n)
#pragma unroll
                  for (int qq = 0; qq < 4; ++qq) acc[n][qq] = 0.0;
#pragma unroll 4
                for (int kq = 0; kq < RC / 4; ++kq) {
                  const int kc = kq * 4 + t4;  // real row of V~
                  const double a0 = Xs[kc * PITCH + r0 + g], a1 = Xs[kc * PITCH + r0 + g + 8];
                  const int ka = kc >> 1, kr = kc & 1;
#pragma unroll
                  for (int n = 0; n < NT; ++n) {
                    const int cc = 8 * NT * hf + n * 8 + g, ca = cc >> 1, cr = cc & 1;
                    const double2 v = Vs[ka + ca * GP];
                    // V~[2a+ra][2c+rc]: (0,0),(1,1) Re; (0,1) Im; (1,0) -Im
                    const double b0 = (kr == cr) ? v.x : (kr ? -v.y : v.y);
                    zdmma(acc[n], a0, a1, b0);
                  }
                }
                if (Mg == nullptr) {  // in place (one pass only: all of X_P was read)
                  __syncwarp();
#pragma unroll
                  for (int n = 0; n < NT; ++n)
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                      const int r = r0 + g + ((qq & 2) ? 8 : 0);
                      const int cc = 8 * NT * hf + n * 8 + 2 * t4 + (qq & 1);
                      Xs[cc * PITCH + r] = acc[n][qq];
                    }
                  continue;
                }
                // (Re, Im) of one complex column are the (qq, qq + 1) pairs
#pragma unroll
                for (int n = 0; n < NT; ++n)
#pragma unroll
                  for (int h2 = 0; h2 < 2; ++h2) {
                    const int r = r0 + g + h2 * 8;
                    const int ccx = (8 * NT * hf + n * 8 + 2 * t4) >> 1;  // complex column in the pair
                    const int gc = gcol(ccx);
                    if (r < lrows && gc < ell)
                      Mg[row0 + r + static_cast<int64_t>(gc) * lp] =
                          make_double2(acc[n][2 * h2], acc[n][2 * h2 + 1]);
                  }
              }
            }
          };
          if constexpr (MINB == 1) {
            // one pass: update the staged pair in place, then write H back
            // with coalesced column stores
            apply_v(nullptr);
            __syncthreads();
            for (int e = tid; e < NC * rows; e += blockDim.x) {
              const int cc = e / rows, r = e - cc * rows;
              const int gc = gcol(cc);
              if (gc < ell && r < lrows)
                Hg[row0 + r + static_cast<int64_t>(gc) * lp] =
                    make_double2(Xs[(2 * cc) * PITCH + r], Xs[(2 * cc + 1) * PITCH + r]);
            }
          } else {
            apply_v(Hg);
          }
          __syncthreads();  // H written: Xs is free for the J pair
          stage(Jg);
          __syncthreads();
          apply_v(Jg);
        }
        __syncthreads();
        if (tid == 0 && s_rot) {
          atomicOr(fl + item, 1u);
          atomicMax(mxs + item, s_mx);
        }
      }
      grid.sync();
    }
    auto done = [&](int64_t i) { return __ldcg(fl + i) == 0u || __ldcg(mxs + i) == 0ull; };
    int all = 1;
    for (int64_t i = 0; i < batch; ++i) {
      const bool d = done(i);
      if (tid == 0 && !conv[i] && d && blockIdx.x == 0) sweeps_out[i] = sweep + 1;
      all &= (conv[i] || d);
    }
    __syncthreads();
    for (int64_t i = tid; i < batch; i += blockDim.x)
      if (done(i)) conv[i] = 1;
    __syncthreads();
    if (all) break;
  }
  if (blockIdx.x == 0)
    for (int64_t i = tid; i < batch; i += blockDim.x)
      if (!conv[i]) sweeps_out[i] = max_sweeps;
}

template <int R, bool CLU, int MINB>
bool launch_zgram_t(const double* src, int64_t src_ld, int64_t src_stride, int src_mode, double* H,
                    double* J, int64_t ell, int64_t lp, int max_sweeps, int* sweeps,
                    unsigned* flags, int64_t batch, int S, cudaStream_t st) {
  const int rows = CLU ? 32 * R : static_cast<int>(std::min<int64_t>(32 * R, (ell + 15) & ~int64_t(15)));
  const size_t bytes = static_cast<size_t>(64) * (rows + 2) * sizeof(double) +
                       (CLU ? 3 : 2) * 32 * 33 * sizeof(double2) + batch * sizeof(int) + 16;
  if (bytes > 227 * 1024) return false;
  auto kern = zjacobi_gram_kernel<R, CLU, MINB>;
  RSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
  int nb = static_cast<int>((ell + 15) / 16);
  nb += nb & 1;
  const int64_t tasks = batch * (nb / 2);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = static_cast<unsigned>(CLU ? S : 1);
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = CLU ? 2 : 1;
  int64_t grid = 0;
  if (CLU) {
    cfg.gridDim = dim3(static_cast<unsigned>(S));
    int max_clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1) {
      cudaGetLastError();
      return false;
    }
    grid = std::max<int64_t>(1, std::min<int64_t>(tasks, max_clusters)) * S;
  } else {
    int per_sm = 0;
    RSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 512, bytes));
    if (per_sm < 1) return false;
    grid = std::max<int64_t>(1, std::min<int64_t>(tasks, per_sm * num_sms()));
  }
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  int ell_i = static_cast<int>(ell), lp_i = static_cast<int>(lp);
  double2* Hc = reinterpret_cast<double2*>(H);
  double2* Jc = reinterpret_cast<double2*>(J);
  RSVD_CUDA(cudaLaunchKernelEx(&cfg, kern, src, src_ld, src_stride, src_mode, Hc, Jc, ell_i, lp_i,
                               nb, batch, max_sweeps, flags, sweeps));
  RSVD_LAUNCH("zjacobi_gram_kernel");
  return true;
}

bool launch_zjacobi_gram(const double* src, int64_t src_ld, int64_t src_stride, int src_mode,
                         double* H, double* J, int64_t ell, int64_t lp, int max_sweeps,
                         int* sweeps, unsigned* flags, int64_t batch, cudaStream_t st) {
  if (!flags || ell < 2) return false;
  int nb = static_cast<int>((ell + 15) / 16);
  nb += nb & 1;
  const int64_t tasks = batch * (nb / 2);
  const int R = static_cast<int>((ell + 31) / 32);
  if (tasks * 4 <= num_sms() && R >= 2) {
    // Few tasks: split each task's rows over a cluster of S <= 6 CTAs.
    const int smax = static_cast<int>(std::min<int64_t>(6, num_sms() / std::max<int64_t>(tasks, 1)));
    if (smax >= 2) {
      int rl = (R + smax - 1) / smax;
      rl = rl <= 1 ? 1 : (rl <= 2 ? 2 : (rl <= 3 ? 3 : 5));
      const int S = (R + rl - 1) / rl;
      bool ok = false;
      if (S >= 2) {
        if (rl == 1) ok = launch_zgram_t<1, true, 1>(src, src_ld, src_stride, src_mode, H, J, ell, lp, max_sweeps, sweeps, flags, batch, S, st);
        else if (rl == 2) ok = launch_zgram_t<2, true, 1>(src, src_ld, src_stride, src_mode, H, J, ell, lp, max_sweeps, sweeps, flags, batch, S, st);
        else if (rl == 3) ok = launch_zgram_t<3, true, 1>(src, src_ld, src_stride, src_mode, H, J, ell, lp, max_sweeps, sweeps, flags, batch, S, st);
        else ok = launch_zgram_t<5, true, 1>(src, src_ld, src_stride, src_mode, H, J, ell, lp, max_sweeps, sweeps, flags, batch, S, st);
      }
      if (ok) return true;
    }
  }
  // The 64-register (MINB = 2) instantiations only pay off when two CTAs
  // really fit an SM's shared memory; otherwise they just spill.
  auto two_fit = [&] {
    const int64_t rows = std::min<int64_t>(32 * R, (ell + 15) & ~int64_t(15));
    const int64_t bytes = 64 * (rows + 2) * 8 + 2 * 32 * 33 * 16 + batch * 4 + 16;
    int per_sm_smem = 0;
    cudaDeviceGetAttribute(&per_sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, current_device());
    return 2 * (bytes + 1024) <= per_sm_smem;
  };
  const bool minb2 = two_fit();
  if (R <= 3 && minb2) return launch_zgram_t<3, false, 2>(src, src_ld, src_stride, src_mode, H, J, ell, lp, max_sweeps, sweeps, flags, batch, 1, st);
  if (R <= 5 && minb2) return launch_zgram_t<5, false, 2>(src, src_ld, src_stride, src_mode, H, J, ell, lp, max_sweeps, sweeps, flags, batch, 1, st);
  if (R <= 5) return launch_zgram_t<5, false, 1>(src, src_ld, src_stride, src_mode, H, J, ell, lp, max_sweeps, sweeps, flags, batch, 1, st);
  if (R <= 9) return launch_zgram_t<9, false, 1>(src, src_ld, src_stride, src_mode, H, J, ell, lp, max_sweeps, sweeps, flags, batch, 1, st);
  return false;
}

template <int RPL>
void launch_zjacobi_t(const double* src, int64_t src_ld, int64_t src_stride, int src_mode,
                      double* H, double* J, int ell, int64_t lp, int max_sweeps, int* sweeps,
                      int64_t batch, int S, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(S);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(512);
  cfg.gridDim = dim3(static_cast<unsigned>(batch * S));
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = S > 1 ? 1 : 0;
  RSVD_CUDA(cudaLaunchKernelEx(&cfg, zjacobi_kernel<RPL>, src, src_ld, src_stride, src_mode,
                               reinterpret_cast<double2*>(H), reinterpret_cast<double2*>(J), ell,
                               lp, max_sweeps, sweeps, S));
  RSVD_LAUNCH("zjacobi_kernel");
}

void launch_zjacobi(const double* src, int64_t src_ld, int64_t src_stride, int src_mode,
                    double* H, double* J, int64_t ell, int64_t lp, int max_sweeps, int* sweeps,
                    int64_t batch, cudaStream_t st, unsigned* flags) {
  if (batch <= 0) return;
  if (launch_zjacobi_gram(src, src_ld, src_stride, src_mode, H, J, ell, lp, max_sweeps, sweeps,
                          flags, batch, st))
    return;
  // Cluster size: fill the SMs (S CTAs per item, at most 8, portable) but
  // never more warps than the l/2 pairs of a step.
  const int64_t pairs = (ell + 1) / 2;
  int S = static_cast<int>(std::min<int64_t>(8, std::max<int64_t>(1, num_sms() / batch)));
  S = static_cast<int>(std::min<int64_t>(S, std::max<int64_t>(1, ceil_div(pairs, 16))));
  const int e = static_cast<int>(ell);
  const int rpl = static_cast<int>(ceil_div(ell, 32));
  if (rpl <= 1)
    launch_zjacobi_t<1>(src, src_ld, src_stride, src_mode, H, J, e, lp, max_sweeps, sweeps, batch, S, st);
  else if (rpl <= 2)
    launch_zjacobi_t<2>(src, src_ld, src_stride, src_mode, H, J, e, lp, max_sweeps, sweeps, batch, S, st);
  else if (rpl <= 3)
    launch_zjacobi_t<3>(src, src_ld, src_stride, src_mode, H, J, e, lp, max_sweeps, sweeps, batch, S, st);
  else if (rpl <= 5)
    launch_zjacobi_t<5>(src, src_ld, src_stride, src_mode, H, J, e, lp, max_sweeps, sweeps, batch, S, st);
  else if (rpl <= 9)
    launch_zjacobi_t<9>(src, src_ld, src_stride, src_mode, H, J, e, lp, max_sweeps, sweeps, batch, S, st);
  else
    launch_zjacobi_t<0>(src, src_ld, src_stride, src_mode, H, J, e, lp, max_sweeps, sweeps, batch, S, st);
}

void launch_zfinalize(const double* W, int64_t lp, int64_t ell, int64_t k, int64_t m, int64_t n,
                      double* sigma_out, int* perm, int* rank, double* dw, int64_t batch,
                      cudaStream_t st) {
  if (batch <= 0) return;
  const size_t smem = lp * (sizeof(double) + sizeof(int));
  zfinalize_kernel<<<static_cast<unsigned>(batch), 512, smem, st>>>(
      reinterpret_cast<const double2*>(W), lp, static_cast<int>(ell), k, m, n, sigma_out, perm,
      rank, dw);
  RSVD_LAUNCH("zfinalize_kernel");
}

void launch_zlift_operand(const double* W, int64_t lp, const int* perm, const double* sigma,
                          int64_t k, const int* rank, int64_t ell, bool half, MatRef M,
                          int64_t batch, cudaStream_t st) {
  if (batch <= 0 || k <= 0) return;
  const int64_t total = 2 * lp * (half ? k : 2 * k);
  dim3 grid(grid_for(total, 256, 2), static_cast<unsigned>(batch));
  zlift_operand_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const double2*>(W), lp, perm, sigma, k,
                                             rank, static_cast<int>(ell), half ? 1 : 0, M.base,
                                             M.ld, M.stride);
  RSVD_LAUNCH("zlift_operand_kernel");
}

}  // namespace rsvd
