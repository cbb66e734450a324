// Diagonally pivoted Cholesky of the l x l Gram G = Y^T Y, the small dense
// step of CholeskyQR that replaces Householder geqrf+orgqr
// (lapack.cpp:146-201, orthonormal_columns lapack.cpp:211-215).
//
// For each batch item (one CTA of 1024 threads):
//   P^T G P ~= R^T R with R (r x l) upper trapezoidal in pivoted order,
//   stopping at the first pivot <= tau * max(diag G): the numerical rank r of
//   Y (LAPACK dpstf2 semantics).  Outputs
//     T     (l x l): Q1 = Y * T has the r orthonormal-ish leading columns
//                    (T = P[:, :r] R11^{-1}); columns >= r are zero and get
//                    filled by the basis completion (aux.cu), which is how
//                    the reference's "always l orthonormal columns, arbitrary
//                    completion when rank deficient" contract
//                    (lapack.hpp:18-20) is honoured without Householder;
//     Rfull (l x l): [R11 R12; 0] P^T, so that Y ~= Q1 * Rfull;
//     rank, perm.
// The matrix lives in shared memory when it fits (l <= 156), otherwise it is
// factored in place in global memory (L2-resident for l <= ~600).
#include <algorithm>

#include "common.cuh"

namespace rsvd {
namespace {

constexpr int kCholThreads = 1024;
constexpr int kCholWarps = kCholThreads / 32;

// Block-wide argmax of d[i] over i in [lo, hi) with ties to the smallest i.
__device__ void block_argmax(const double* W, int ld, int lo, int hi, double* s_val, int* s_idx,
                             double& best_val, int& best_idx) {
  double v = -1.0;
  int ix = 0x7fffffff;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double d = W[i + static_cast<int64_t>(i) * ld];
    if (d > v || (d == v && i < ix)) v = d, ix = i;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, off);
    const int oi = __shfl_xor_sync(0xffffffffu, ix, off);
    if (ov > v || (ov == v && oi < ix)) v = ov, ix = oi;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s_val[warp] = v, s_idx[warp] = ix;
  __syncthreads();
  if (warp == 0) {
    v = lane < kCholWarps ? s_val[lane] : -1.0;
    ix = lane < kCholWarps ? s_idx[lane] : 0x7fffffff;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, off);
      const int oi = __shfl_xor_sync(0xffffffffu, ix, off);
      if (ov > v || (ov == v && oi < ix)) v = ov, ix = oi;
    }
    if (lane == 0) s_val[32] = v, s_idx[32] = ix;
  }
  __syncthreads();
  best_val = s_val[32];
  best_idx = s_idx[32];
  __syncthreads();
}

template <bool IN_SMEM>
__global__ void __launch_bounds__(kCholThreads)
    pchol_kernel(double* __restrict__ G, double* __restrict__ T, double* __restrict__ Rfull,
                 int* __restrict__ rank_out, int* __restrict__ perm_out, int ell, int ellp,
                 double tau) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double s_val[33];
  __shared__ int s_idx[33];
  const int64_t b = blockIdx.x;
  const int64_t sq = static_cast<int64_t>(ellp) * ellp;
  double* Gb = G + b * sq;
  double* W = IN_SMEM ? sm : Gb;
  double* colbuf = IN_SMEM ? sm + sq : sm;  // kCholWarps x ellp scratch for the inverse
  double* rrow = colbuf + static_cast<int64_t>(kCholWarps) * ellp;  // current row of R
  int* perm = reinterpret_cast<int*>(rrow + ellp);
  const int tid = threadIdx.x;
  const int ld = ellp;

  if (IN_SMEM)
    for (int64_t e = tid; e < sq; e += blockDim.x) W[e] = Gb[e];
  for (int i = tid; i < ellp; i += blockDim.x) perm[i] = i;
  __syncthreads();

  double dmax0;
  int p;
  block_argmax(W, ld, 0, ell, s_val, s_idx, dmax0, p);
  int r = ell;
  if (!(dmax0 > 0.0)) r = 0;
  for (int j = 0; j < r; ++j) {
    double piv;
    block_argmax(W, ld, j, ell, s_val, s_idx, piv, p);
    if (!(piv > tau * dmax0)) {
      r = j;
      break;
    }
    if (p != j) {  // symmetric swap of rows and columns j <-> p
      for (int i = tid; i < ell; i += blockDim.x) {
        const double x = W[j + static_cast<int64_t>(i) * ld];
        W[j + static_cast<int64_t>(i) * ld] = W[p + static_cast<int64_t>(i) * ld];
        W[p + static_cast<int64_t>(i) * ld] = x;
      }
      __syncthreads();
      for (int i = tid; i < ell; i += blockDim.x) {
        const double x = W[i + static_cast<int64_t>(j) * ld];
        W[i + static_cast<int64_t>(j) * ld] = W[i + static_cast<int64_t>(p) * ld];
        W[i + static_cast<int64_t>(p) * ld] = x;
      }
      if (tid == 0) {
        const int x = perm[j];
        perm[j] = perm[p];
        perm[p] = x;
      }
      __syncthreads();
    }
    const double rjj = sqrt(piv);
    const double inv = 1.0 / rjj;
    // Row j of R: W[j][c] / rjj for c > j.  Column j below the diagonal is
    // updated to match so the trailing block stays symmetric.
    for (int c = j + 1 + tid; c < ell; c += blockDim.x) {
      const double v = W[j + static_cast<int64_t>(c) * ld] * inv;
      W[j + static_cast<int64_t>(c) * ld] = v;
      rrow[c] = v;
    }
    if (tid == 0) W[j + static_cast<int64_t>(j) * ld] = rjj;
    __syncthreads();
    // Trailing update W[a][c] -= R[j][a] R[j][c], a, c > j: one warp per
    // column, lanes along the contiguous rows.
    {
      const int warp = tid >> 5, lane = tid & 31;
      for (int c = j + 1 + warp; c < ell; c += kCholWarps) {
        const double rc = rrow[c];
        double* col = W + static_cast<int64_t>(c) * ld;
        for (int a = j + 1 + lane; a < ell; a += 32) col[a] -= rrow[a] * rc;
      }
    }
    __syncthreads();
  }

  // Outputs: Rfull[i][perm[c]] = R[i][c] (i < r, c >= i), zero elsewhere.
  double* Tb = T + b * sq;
  double* Rb = Rfull ? Rfull + b * sq : nullptr;
  for (int64_t e = tid; e < sq; e += blockDim.x) {
    Tb[e] = 0.0;
    if (Rb) Rb[e] = 0.0;
  }
  __syncthreads();
  if (Rb) {
    for (int64_t e = tid; e < static_cast<int64_t>(r) * ell; e += blockDim.x) {
      const int c = static_cast<int>(e / r), i = static_cast<int>(e - static_cast<int64_t>(c) * r);
      if (c >= i) Rb[i + static_cast<int64_t>(perm[c]) * ld] = W[i + static_cast<int64_t>(c) * ld];
    }
  }
  // T = P[:, :r] R11^{-1}: column c of R11^{-1} by backward substitution on
  // x = e_c (one warp per column, axpy form so lanes work in parallel).
  const int warp = tid >> 5, lane = tid & 31;
  double* x = colbuf + static_cast<int64_t>(warp) * ellp;
  for (int c = warp; c < r; c += kCholWarps) {
    for (int i = lane; i <= c; i += 32) x[i] = (i == c) ? 1.0 : 0.0;
    __syncwarp();
    for (int k = c; k >= 0; --k) {
      const double xk = x[k] / W[k + static_cast<int64_t>(k) * ld];
      __syncwarp();
      if (lane == 0) x[k] = xk;
      for (int i = lane; i < k; i += 32) x[i] -= W[i + static_cast<int64_t>(k) * ld] * xk;
      __syncwarp();
    }
    for (int i = lane; i <= c; i += 32) Tb[perm[i] + static_cast<int64_t>(c) * ld] = x[i];
    __syncwarp();
  }
  if (tid < ellp && perm_out) perm_out[b * ellp + tid] = perm[tid];
  if (tid == 0) rank_out[b] = r;
}

}  // namespace

void launch_pchol(const double* G, double* T, double* Rfull, int* rank, int* perm, int64_t ell,
                  int64_t ellp, double tau, int64_t batch, cudaStream_t st) {
  const int64_t sq_bytes = ellp * ellp * static_cast<int64_t>(sizeof(double));
  const int64_t scratch =
      (kCholWarps + 1) * ellp * static_cast<int64_t>(sizeof(double)) + ellp * 4 + 16;
  const bool in_smem = sq_bytes + scratch <= 220 * 1024;
  double* Gm = const_cast<double*>(G);  // factored in place when not in shared memory
  if (in_smem) {
    const int bytes = static_cast<int>(sq_bytes + scratch);
    RSVD_CUDA(cudaFuncSetAttribute(pchol_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   bytes));
    pchol_kernel<true><<<static_cast<unsigned>(batch), kCholThreads, bytes, st>>>(
        Gm, T, Rfull, rank, perm, static_cast<int>(ell), static_cast<int>(ellp), tau);
  } else {
    const int bytes = static_cast<int>(scratch);
    RSVD_CUDA(cudaFuncSetAttribute(pchol_kernel<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    pchol_kernel<false><<<static_cast<unsigned>(batch), kCholThreads, bytes, st>>>(
        Gm, T, Rfull, rank, perm, static_cast<int>(ell), static_cast<int>(ellp), tau);
  }
  RSVD_LAUNCH("pchol_kernel");
}

}  // namespace rsvd
