// One-sided (Hestenes) Jacobi SVD of the small l x l factor H.
//
// Replaces the LAPACK dgesdd('S') / dgesvd fallback call on the projected
// matrix B = Q^T A (factorize.cpp:86-90 -> lapack.cpp:112-128).  The engine
// never forms B: it computes B^T = A^T Q (n x l), CholeskyQR2 gives
// B^T = Qb * Rt, and H = Rt^T is the l x l matrix whose SVD is B's up to the
// orthonormal Qb.  Rotations from the right, H J -> W with orthogonal
// columns, give sigma_i = ||W e_i|| (computed from the vectors themselves,
// hence relatively accurate), U~ = W Sigma^{-1} and V~ = Qb J.
//
// Parallel cyclic ordering (round-robin tournament): each of the l-1 steps of
// a sweep rotates l/2 disjoint column pairs, one warp per pair; a sweep with
// no rotation above tol = sqrt(l) * eps (dgesvj's convergence test) ends the
// iteration.  One CTA per batch item; H and J live in shared memory when both
// fit, otherwise in global memory (L2-resident).
#include <cfloat>

#include "common.cuh"

namespace rsvd {
namespace {

constexpr int kJacThreads = 1024;
constexpr int kJacWarps = kJacThreads / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Round-robin pairing for `nn` (even) players at step s: slot 0 fixed, the
// others rotate.  Pair k couples slot k with slot nn-1-k.
__device__ __forceinline__ int rr_player(int slot, int s, int nn) {
  if (slot == 0) return 0;
  return 1 + (slot - 1 + s) % (nn - 1);
}

template <bool IN_SMEM>
__global__ void __launch_bounds__(kJacThreads)
    jacobi_kernel(double* __restrict__ H, double* __restrict__ J, int ell, int ellp,
                  int max_sweeps, int* __restrict__ sweeps_out) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_rot;
  const int64_t b = blockIdx.x;
  const int64_t sq = static_cast<int64_t>(ellp) * ellp;
  double* Hg = H + b * sq;
  double* Jg = J + b * sq;
  double* Hs = IN_SMEM ? sm : Hg;
  double* Js = IN_SMEM ? sm + sq : Jg;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (IN_SMEM) {
    for (int64_t e = tid; e < sq; e += blockDim.x) Hs[e] = Hg[e];
  }
  for (int64_t e = tid; e < sq; e += blockDim.x) {
    const int64_t j = e / ellp, i = e - j * ellp;
    Js[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();

  const double tol = sqrt(static_cast<double>(ell)) * DBL_EPSILON;
  const int nn = ell + (ell & 1);
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    int rotated = 0;
    for (int s = 0; s < nn - 1; ++s) {
      for (int k = warp; k < nn / 2; k += kJacWarps) {
        const int p = rr_player(k, s, nn), q = rr_player(nn - 1 - k, s, nn);
        const int i = min(p, q), j = max(p, q);
        if (j >= ell) continue;  // dummy player for odd l
        double* hi = Hs + static_cast<int64_t>(i) * ellp;
        double* hj = Hs + static_cast<int64_t>(j) * ellp;
        double a = 0.0, bb = 0.0, g = 0.0;
        for (int r = lane; r < ell; r += 32) {
          const double x = hi[r], y = hj[r];
          a = fma(x, x, a);
          bb = fma(y, y, bb);
          g = fma(x, y, g);
        }
        a = warp_sum(a);
        bb = warp_sum(bb);
        g = warp_sum(g);
        if (!(a > 0.0) || !(bb > 0.0)) continue;
        if (!(fabs(g) > tol * sqrt(a) * sqrt(bb))) continue;
        const double zeta = (bb - a) / (2.0 * g);
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + tt * tt);
        const double sn = c * tt;
        for (int r = lane; r < ell; r += 32) {
          const double x = hi[r], y = hj[r];
          hi[r] = c * x - sn * y;
          hj[r] = sn * x + c * y;
        }
        double* ji = Js + static_cast<int64_t>(i) * ellp;
        double* jj = Js + static_cast<int64_t>(j) * ellp;
        for (int r = lane; r < ell; r += 32) {
          const double x = ji[r], y = jj[r];
          ji[r] = c * x - sn * y;
          jj[r] = sn * x + c * y;
        }
        rotated = 1;
      }
      __syncthreads();
    }
    if (rotated && lane == 0) atomicOr(&s_rot, 1);
    __syncthreads();
    const int any = s_rot;
    __syncthreads();
    if (!any) break;
  }
  if (IN_SMEM) {
    for (int64_t e = tid; e < sq; e += blockDim.x) {
      Hg[e] = Hs[e];
      Jg[e] = Js[e];
    }
  }
  if (tid == 0 && sweeps_out) sweeps_out[b] = sweep + 1;
}

}  // namespace

void launch_jacobi(double* H, double* J, int64_t ell, int64_t ellp, int max_sweeps, int* sweeps,
                   int64_t batch, cudaStream_t st) {
  const int64_t bytes = 2 * ellp * ellp * static_cast<int64_t>(sizeof(double));
  if (bytes <= 220 * 1024) {
    RSVD_CUDA(cudaFuncSetAttribute(jacobi_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(bytes)));
    jacobi_kernel<true><<<static_cast<unsigned>(batch), kJacThreads, bytes, st>>>(
        H, J, static_cast<int>(ell), static_cast<int>(ellp), max_sweeps, sweeps);
  } else {
    jacobi_kernel<false><<<static_cast<unsigned>(batch), kJacThreads, 0, st>>>(
        H, J, static_cast<int>(ell), static_cast<int>(ellp), max_sweeps, sweeps);
  }
  RSVD_LAUNCH("jacobi_kernel");
}

}  // namespace rsvd
