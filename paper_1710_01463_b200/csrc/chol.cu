// Diagonally pivoted Cholesky of the l x l Gram G = Y^T Y, the small dense
// step of CholeskyQR that replaces Householder geqrf+orgqr
// (lapack.cpp:146-201, orthonormal_columns lapack.cpp:211-215).
//
// For each batch item (one CTA):
//   P^T G P ~= R^T R with R (r x l) upper trapezoidal in pivoted order,
//   stopping at the first pivot <= tau * max(diag G): the numerical rank r of
//   Y (LAPACK dpstrf semantics).  Outputs
//     T     (l x l): R11^{-1} in pivot order, upper triangular; Q1 = (Y P) T
//                    (Y's columns gathered through perm) has the r leading
//                    columns; columns >= r are zero and get
//                    filled by the basis completion (aux.cu), which is how
//                    the reference's "always l orthonormal columns, arbitrary
//                    completion when rank deficient" contract
//                    (lapack.hpp:18-20) is honoured without Householder;
//     Rfull (l x l): [R11 R12; 0] P^T, so that Y ~= Q1 * Rfull;
//     rank, perm.
//
// Algorithm (blocked, swap-free, dpstrf-like):
//   * panels of PB = 32 pivots; inside a panel the pivot search runs on the
//     lazily updated diagonal d - work (one warp), pivots are swapped
//     *logically* through a position -> storage map, and row j of R is formed
//     from the panel-start Schur column minus the in-panel rank-jj correction
//     (shared-memory panel buffer);
//   * at the end of a panel the trailing Schur complement is rebuilt in a
//     second buffer in the new pivot order with a rank-32 DMMA update
//     (mma.sync m16n8k4 f64), so no row/column swap ever touches global memory;
//   * R rows are written in original column order, which is Rfull directly;
//   * R11^{-1} by a blocked DMMA inverse (blocked_upper_inverse below).
#include <cooperative_groups.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace rsvd {
namespace {

constexpr int kCholThreads = 512;
constexpr int kCholWarps = kCholThreads / 32;
constexpr int PB = 32;  // panel width (pivots per panel)

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

constexpr int kInvWarps = 8;      // warps active in the blocked inverse
constexpr int kInvPitch = 36;     // 32 x 36 per-warp tile: 4 mod 16 words, conflict free
constexpr int kInvSmem = kInvWarps * 32 * kInvPitch;  // doubles of shared scratch needed

// X = R^{-1} for an upper-triangular R of order nbk*32 (column-major, ld),
// by the whole CTA.  Stage A: each diagonal block inverted by one warp, lane
// c owning column c (fully unrolled backward substitution, R_II broadcast
// from shared memory).  Stage B: block diagonals d = 1..nbk-1 in order;
// X_IJ = -X_II (sum_{K=I+1..J} R_IK X_KJ), one warp per block, both
// products on DMMA (mma.sync m16n8k4 f64).
__device__ void blocked_upper_inverse(const double* __restrict__ R, double* __restrict__ X, int ld,
                                      int nbk, double* smem, int warp, int lane) {
  const int g = lane >> 2, t = lane & 3;
  double* S = smem + warp * 32 * kInvPitch;
  if (warp < kInvWarps) {
    for (int I = warp; I < nbk; I += kInvWarps) {
      const int o = I * 32;
      for (int e = lane; e < 1024; e += 32) {
        const int c = e >> 5, i = e & 31;
        S[i * kInvPitch + c] = R[(o + i) + static_cast<int64_t>(o + c) * ld];
      }
      __syncwarp();
      const int c = lane;
      double x[32];
#pragma unroll
      for (int i = 31; i >= 0; --i) {
        double s = 0.0;
#pragma unroll
        for (int k = i + 1; k < 32; ++k) s = fma(S[i * kInvPitch + k], x[k], s);
        const double rii = S[i * kInvPitch + i];
        x[i] = (i == c) ? 1.0 / rii : ((i < c) ? -s / rii : 0.0);
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) X[(o + i) + static_cast<int64_t>(o + c) * ld] = x[i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int dg = 1; dg < nbk; ++dg) {
    if (warp < kInvWarps) {
      for (int I = warp; I + dg < nbk; I += kInvWarps) {
        const int J = I + dg;
        const int oI = I * 32, oJ = J * 32;
        double acc[2][4][4];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[a][n][q] = 0.0;
        // K runs over whole 32-blocks; operands are fetched 16 k at a time
        // (all loads issued before the MMAs) to overlap the L2 latency.
        for (int kc = oI + 32; kc < oJ + 32; kc += 16) {
          double af[4][4], bf[4][4];
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) {
            const int k0 = kc + s4 * 4;
            const double* rc = R + static_cast<int64_t>(k0 + t) * ld + oI + g;
            af[s4][0] = rc[0], af[s4][1] = rc[8], af[s4][2] = rc[16], af[s4][3] = rc[24];
#pragma unroll
            for (int n = 0; n < 4; ++n)
              bf[s4][n] = X[(k0 + t) + static_cast<int64_t>(oJ + n * 8 + g) * ld];
          }
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
            for (int n = 0; n < 4; ++n) {
              dmma_16x8x4(acc[0][n], af[s4][0], af[s4][1], bf[s4][n]);
              dmma_16x8x4(acc[1][n], af[s4][2], af[s4][3], bf[s4][n]);
            }
        }
        // S (row k, col c) = acc
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int i = a * 16 + g + ((q & 2) ? 8 : 0), c = n * 8 + 2 * t + (q & 1);
              S[i * kInvPitch + c] = acc[a][n][q];
              acc[a][n][q] = 0.0;
            }
        __syncwarp();
        // X_IJ = -X_II * S
#pragma unroll
        for (int k0 = 0; k0 < 32; k0 += 4) {
          const double* xc = X + static_cast<int64_t>(oI + k0 + t) * ld + oI + g;
          const double a00 = xc[0], a01 = xc[8], a10 = xc[16], a11 = xc[24];
#pragma unroll
          for (int n = 0; n < 4; ++n) {
            const double b0 = S[(k0 + t) * kInvPitch + n * 8 + g];
            dmma_16x8x4(acc[0][n], a00, a01, b0);
            dmma_16x8x4(acc[1][n], a10, a11, b0);
          }
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int i = a * 16 + g + ((q & 2) ? 8 : 0), c = n * 8 + 2 * t + (q & 1);
              X[(oI + i) + static_cast<int64_t>(oJ + c) * ld] = -acc[a][n][q];
            }
        __syncwarp();
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kCholThreads)
    pchol_kernel(double* __restrict__ G, double* __restrict__ T, double* __restrict__ Rfull,
                 double* __restrict__ scratch, int* __restrict__ rank_out,
                 int* __restrict__ perm_out, int ell, int ellp, double tau, int pivot,
                 const int* __restrict__ mask, int rp_global) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double s_piv;
  __shared__ int s_stop;
  const int64_t b = blockIdx.x;
  if (mask && !mask[b]) return;  // whole CTA: item not selected
  const int64_t sq = static_cast<int64_t>(ellp) * ellp;
  const int ld = ellp;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // Shared layout.  The panel pitch is 4 or 12 mod 16 words (ellp is a
  // multiple of 8), which makes the DMMA fragment loads conflict free, and
  // >= ellp + 16 so 16-wide tiles never read past zeroed storage.
  const int rp_pitch = ellp + 20;
  // Large l (realified complex Grams): the panel does not fit next to the
  // inverse workspace; it then lives in the scratch tail (rp_global).
  const int64_t big = rp_global ? static_cast<int64_t>(kInvSmem)
                                : max(static_cast<int64_t>(PB) * rp_pitch, static_cast<int64_t>(kInvSmem));
  double* Rp = rp_global ? scratch + 2 * sq * static_cast<int64_t>(gridDim.x) + b * PB * rp_pitch
                         : sm;                     // PB x rp_pitch (panel rows of R)
  double* d = sm + big;                            // panel-start Schur diagonal (by position)
  double* work = d + ellp;                         // in-panel sum of R[k][x]^2
  double* diag = work + ellp;                      // diagonal of R11 (by position)
  int* loc = reinterpret_cast<int*>(diag + ellp);  // position -> storage row/col (this panel)
  int* pos2orig = loc + ellp;                      // position -> original index

  double* Wcur = G + b * sq;
  double* Wnext = scratch + b * 2 * sq;
  double* Rorig = Rfull ? Rfull + b * sq : scratch + b * 2 * sq + sq;  // row j: R[j][orig]

  for (int i = tid; i < ellp; i += blockDim.x) {
    d[i] = i < ell ? Wcur[i + static_cast<int64_t>(i) * ld] : 0.0;
    pos2orig[i] = i;
  }
  for (int64_t e = tid; e < sq; e += blockDim.x) Rorig[e] = 0.0;
  __syncthreads();

  if (warp == 0) {  // max diagonal
    double v = 0.0;
    for (int i = lane; i < ell; i += 32) v = fmax(v, d[i]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) {
      s_piv = v;
      s_stop = !(v > 0.0);
    }
  }
  __syncthreads();
  const double thresh = tau * s_piv;
  int r = s_stop ? 0 : ell;

  for (int j0 = 0; j0 < r; j0 += PB) {
    const int jb = min(PB, ell - j0);
    for (int i = tid; i < ellp; i += blockDim.x) {
      work[i] = 0.0;
      loc[i] = i;
    }
    for (int e = tid; e < PB * rp_pitch; e += blockDim.x) Rp[e] = 0.0;
    __syncthreads();
    int jdone = jb;
    for (int jj = 0; jj < jb; ++jj) {
      const int j = j0 + jj;
      if (warp == 0) {
        // pivot: argmax over positions >= j of d - work (ties -> lowest position)
        double v = -DBL_MAX;
        int ix = 0x7fffffff;
        for (int x = j + lane; x < ell; x += 32) {
          const double dv = d[x] - work[x];
          if (dv > v || (dv == v && x < ix)) v = dv, ix = x;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, v, off);
          const int oi = __shfl_xor_sync(0xffffffffu, ix, off);
          if (ov > v || (ov == v && oi < ix)) v = ov, ix = oi;
        }
        if (!pivot) {  // plain Cholesky: keep the order, still test the pivot floor
          ix = j;
          v = d[j] - work[j];
        } else if (pivot == 2) {
          // Pair pivoting (realified complex Gram, columns 2a / 2a+1 = Re / Im
          // of complex column a): even positions take the best even original
          // column, odd positions its partner, so P is the realification of a
          // complex permutation and R stays the realified complex factor.
          int want = -1;
          if (j & 1) want = pos2orig[j - 1] ^ 1;
          v = -DBL_MAX;
          ix = 0x7fffffff;
          for (int x = j + lane; x < ell; x += 32) {
            const int o = pos2orig[x];
            const bool ok = (j & 1) ? (o == want) : ((o & 1) == 0);
            if (!ok) continue;
            const double dv = d[x] - work[x];
            if (dv > v || (dv == v && x < ix)) v = dv, ix = x;
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, off);
            const int oi = __shfl_xor_sync(0xffffffffu, ix, off);
            if (ov > v || (ov == v && oi < ix)) v = ov, ix = oi;
          }
          if (ix == 0x7fffffff) ix = j, v = -DBL_MAX;  // no candidate: stop
        }
        const bool stop = !(v > thresh);
        if (!stop && ix != j) {  // logical swap of positions j and ix
          for (int k = lane; k < jj; k += 32) {
            const double t0 = Rp[k * rp_pitch + j];
            Rp[k * rp_pitch + j] = Rp[k * rp_pitch + ix];
            Rp[k * rp_pitch + ix] = t0;
          }
          if (lane == 0) {
            double t = d[j];
            d[j] = d[ix];
            d[ix] = t;
            t = work[j];
            work[j] = work[ix];
            work[ix] = t;
            int u = loc[j];
            loc[j] = loc[ix];
            loc[ix] = u;
            u = pos2orig[j];
            pos2orig[j] = pos2orig[ix];
            pos2orig[ix] = u;
          }
        }
        if (lane == 0) {
          s_piv = v;
          s_stop = stop;
        }
      }
      __syncthreads();
      if (s_stop) {
        jdone = jj;
        r = j;
        if (pivot == 2 && (j & 1)) {  // drop the unpaired half: rank stays even
          jdone = jj - 1;
          r = j - 1;
          for (int e = tid; e < ellp; e += blockDim.x) Rorig[(j - 1) + static_cast<int64_t>(e) * ld] = 0.0;
          __syncthreads();
        }
        break;
      }
      const double rjj = sqrt(s_piv);
      const double inv = 1.0 / rjj;
      const double* wcol = Wcur + static_cast<int64_t>(loc[j]) * ld;
      for (int x = j + 1 + tid; x < ell; x += blockDim.x) {
        double s = wcol[loc[x]];
        for (int k = 0; k < jj; ++k) s -= Rp[k * rp_pitch + j] * Rp[k * rp_pitch + x];
        const double v = s * inv;
        Rp[jj * rp_pitch + x] = v;
        work[x] += v * v;
        Rorig[j + static_cast<int64_t>(pos2orig[x]) * ld] = v;
      }
      if (tid == 0) {
        Rp[jj * rp_pitch + j] = rjj;
        diag[j] = rjj;
        Rorig[j + static_cast<int64_t>(pos2orig[j]) * ld] = rjj;
      }
      __syncthreads();
    }
    const int j1 = j0 + jdone;
    if (jdone < jb || j1 >= ell) break;  // rank found, or finished
    // Trailing rebuild: Wnext[x][y] = Wcur[loc x][loc y] - sum_k Rp[k][x] Rp[k][y]
    // for positions x, y in [j1, ell): 16 x 16 DMMA tiles, one per warp.
    const int nt = ell - j1;
    const int tiles = (nt + 15) / 16;
    const int g = lane >> 2, t = lane & 3;
    for (int tile = warp; tile < tiles * tiles; tile += kCholWarps) {
      const int tx = tile % tiles, ty = tile / tiles;
      const int x0 = j1 + tx * 16, y0 = j1 + ty * 16;
      double acc[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[h][q] = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < PB; k0 += 4) {
        const double a0 = Rp[(k0 + t) * rp_pitch + x0 + g];
        const double a1 = Rp[(k0 + t) * rp_pitch + x0 + g + 8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double b0 = Rp[(k0 + t) * rp_pitch + y0 + h * 8 + g];
          dmma_16x8x4(acc[h], a0, a1, b0);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int x = x0 + g + ((q & 2) ? 8 : 0);
          const int y = y0 + h * 8 + 2 * t + (q & 1);
          if (x < ell && y < ell) {
            const double w = Wcur[loc[x] + static_cast<int64_t>(loc[y]) * ld];
            Wnext[x + static_cast<int64_t>(y) * ld] = w - acc[h][q];
          }
        }
    }
    __syncthreads();
    for (int x = j1 + tid; x < ell; x += blockDim.x)
      d[x] = Wnext[x + static_cast<int64_t>(x) * ld];
    double* tmp = Wcur;
    Wcur = Wnext;
    Wnext = tmp;
    __syncthreads();
  }
  __syncthreads();

  // ---- T = R11^{-1} (pivot order; the apply GEMM gathers Y's columns) ----
  // R11 in position order, column-contiguous, padded to whole 32-blocks with
  // an identity tail: C11[i + c*ld] = Rorig[i][pos2orig[c]] (i <= c < r).
  double* C11 = Wnext;  // both trailing buffers are free now
  double* X = Wcur;     // R11^{-1}, position order
  const int nbk = (r + 31) / 32;
  const int rp = nbk * 32;  // <= ellp (ellp is a multiple of 32)
  for (int64_t e = tid; e < static_cast<int64_t>(rp) * rp; e += blockDim.x) {
    const int c = static_cast<int>(e / rp), i = static_cast<int>(e - static_cast<int64_t>(c) * rp);
    double v = 0.0;
    if (c < r) v = i <= c ? Rorig[i + static_cast<int64_t>(pos2orig[c]) * ld] : 0.0;
    else if (i == c) v = 1.0;
    C11[i + static_cast<int64_t>(c) * ld] = v;
  }
  __syncthreads();
  blocked_upper_inverse(C11, X, ld, nbk, sm, warp, lane);
  double* Tb = T + b * sq;
  for (int64_t e = tid; e < sq; e += blockDim.x) Tb[e] = 0.0;
  __syncthreads();
  for (int64_t e = tid; e < static_cast<int64_t>(r) * r; e += blockDim.x) {
    const int c = static_cast<int>(e / r), i = static_cast<int>(e - static_cast<int64_t>(c) * r);
    if (i <= c) Tb[i + static_cast<int64_t>(c) * ld] = X[i + static_cast<int64_t>(c) * ld];
  }
  if (perm_out)
    for (int i = tid; i < ellp; i += blockDim.x) perm_out[b * ellp + i] = pos2orig[i];
  if (tid == 0) rank_out[b] = r;
}

// One warp factors the 32 x 32 diagonal block whose current values lane c
// holds in a[0..31] (column c), writes R_JJ (upper) to W and Rd and its
// inverse to Dt; returns the in-block breakdown index (32 = none).  Columns
// at or beyond `ell` arrive as identity columns.
__device__ __forceinline__ int factor_diag_block(double (&a)[32], double* __restrict__ W, int ld, int ell, int o,
                                 double thresh, double* Rd, double* Dt, int lane) {
  // Cholesky of the 32 x 32 block (lane = column, a[i] = row i) and, in the
  // same sweep, Z = R^{-T} by forward substitution (lane j holds column j of
  // Z, i.e. row j of R^{-1}).  Row k of R is broadcast through shared memory
  // (Rd, read as double2) for the rank-1 update, column k through Dt (which
  // holds R^T until the end); pivots use a warp-uniform rsqrt.  ~11k cycles
  // (tools/probe/diag_probe4.cu) against ~29k for shuffles + a separate
  // backward substitution.
  int brk = 32;
  double z[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double akk = __shfl_sync(0xffffffffu, a[k], k);
    if (brk == 32 && o + k < ell && !(akk > thresh)) brk = k;
    double rk, inv = 1.0;
    if (brk == 32) {
      inv = rsqrt(akk);
      rk = (lane == k) ? akk * inv : (lane > k ? a[k] * inv : 0.0);
    } else {
      rk = (lane == k) ? 1.0 : 0.0;  // beyond the breakdown: keep R_JJ invertible
    }
    a[k] = rk;
    // Lookahead: the next pivot (lane k + 1's a[k + 1]) is updated first
    // from the lane's own r_k,k+1, so the pivot chain shfl -> rsqrt -> fma
    // does not wait for the row broadcast below.
    if (k + 1 < 32 && lane == k + 1) a[k + 1] = fma(-rk, rk, a[k + 1]);
    Rd[k * kInvPitch + lane] = rk;
    Dt[lane * kInvPitch + k] = rk;
    __syncwarp();
    const double rkm = lane > k ? rk : 0.0;
    const double rkn = lane > k + 1 ? rk : 0.0;  // element k + 1: lane k + 1 already done
    const double2* row = reinterpret_cast<const double2*>(Rd + k * kInvPitch);
#pragma unroll
    for (int i2 = (k + 1) / 2; i2 < 16; ++i2) {
      const double2 v = row[i2];
      if (2 * i2 > k) a[2 * i2] = fma(-v.x, 2 * i2 == k + 1 ? rkn : rkm, a[2 * i2]);
      if (2 * i2 + 1 > k) a[2 * i2 + 1] = fma(-v.y, 2 * i2 + 1 == k + 1 ? rkn : rkm, a[2 * i2 + 1]);
    }
    const double2* col = reinterpret_cast<const double2*>(Dt + k * kInvPitch);
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int i2 = 0; 2 * i2 < k; ++i2) {
      const double2 v = col[i2];
      s0 = fma(v.x, z[2 * i2], s0);
      if (2 * i2 + 1 < k) s1 = fma(v.y, z[2 * i2 + 1], s1);
    }
    z[k] = ((lane == k ? 1.0 : 0.0) - (s0 + s1)) * inv;
  }
  const bool colok = o + lane < ell;
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (colok && o + k < ell && k <= lane) W[(o + k) + static_cast<int64_t>(o + lane) * ld] = a[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) Dt[lane * kInvPitch + k] = z[k];  // (R^{-1})[lane][k] = Z[k][lane]
  __syncwarp();
  return brk;
}

// Unpivoted blocked Cholesky with breakdown detection (same outputs as
// pchol_kernel with the identity permutation).  Right-looking over 32-column
// blocks: one warp factors the 32 x 32 diagonal block in registers (lane =
// column, row k broadcast by shuffles) and inverts it; the block row of R
// right of it is R_JJ^{-T} A_J,right on DMMA; the trailing matrix takes a
// rank-32 DMMA update in place.  A pivot <= tau * max(diag G) stops the
// factorization at the numerical rank r (the remaining columns are completed
// by the caller), which for the generic bases of the power iteration (Gaussian
// mixing) coincides with the pivoted rank.  Used wherever the pivot order is
// not consumed: every CholeskyQR pass except the first pass on B^T.
__global__ void __launch_bounds__(kCholThreads)
    uchol_kernel(double* __restrict__ G, double* __restrict__ T, double* __restrict__ Rfull,
                 double* __restrict__ scratch, int* __restrict__ rank_out,
                 int* __restrict__ perm_out, int ell, int ellp, double tau, const CholOpts o,
                 int rp_global) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double s_thresh;
  __shared__ int s_r;
  __shared__ int s_go;
  const int64_t b = blockIdx.x;
  const int64_t sq = static_cast<int64_t>(ellp) * ellp;
  const int ld = ellp;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rp_pitch = ellp + 20;
  const int64_t big = rp_global ? static_cast<int64_t>(kInvSmem)
                                : max(static_cast<int64_t>(PB) * rp_pitch, static_cast<int64_t>(kInvSmem));
  double* Rp = rp_global ? scratch + 2 * sq * static_cast<int64_t>(gridDim.x) + b * PB * rp_pitch
                         : sm;      // 32 x rp_pitch: row block J of R, columns >= o + 32
  double* Rd = sm + big;            // R_JJ,        Rd[i * 36 + c]
  double* Dt = Rd + 32 * kInvPitch;  // R_JJ^{-1},  Dt[i * 36 + c]
  double* W = G + b * sq;
  double* C11 = scratch + b * 2 * sq;
  double* X = C11 + sq;

  // Gating (CholOpts): the shifted retry runs only for items whose first
  // factorization stopped short of full rank, and records them in ill_out.
  if (tid == 0) {
    int go = 1;
    if (o.gate_rank) {
      go = o.gate_rank[b] < ell;
      if (o.ill_out) o.ill_out[b] = go;
    }
    if (o.mask && !o.mask[b]) go = 0;
    s_go = go;
  }
  __syncthreads();
  if (!s_go) return;
  if (o.Gsrc) {
    const double* src = o.Gsrc + b * sq;
    for (int64_t e = tid; e < sq; e += blockDim.x) W[e] = src[e];
    __syncthreads();
  }
  if (o.shift_coef > 0.0) {  // G += s I, s = coef * tr(G) (shifted CholeskyQR)
    if (warp == 0) {
      double tr = 0.0;
      for (int i = lane; i < ell; i += 32) tr += W[i + static_cast<int64_t>(i) * ld];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, off);
      const double sh = o.shift_coef * tr;
      for (int i = lane; i < ell; i += 32) W[i + static_cast<int64_t>(i) * ld] += sh;
    }
    __syncthreads();
  }

  if (warp == 0) {
    double v = 0.0;
    for (int i = lane; i < ell; i += 32) v = fmax(v, W[i + static_cast<int64_t>(i) * ld]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) {
      s_thresh = tau * v;
      s_r = (v > 0.0) ? ell : 0;
    }
  }
  __syncthreads();
  const double thresh = s_thresh;
  int r = s_r;
  const int nbk_all = (ell + 31) / 32;
  for (int e = tid; e < PB * rp_pitch; e += blockDim.x) Rp[e] = 0.0;
  __syncthreads();
  // Prologue: the first diagonal block.
  if (warp == 0 && r == ell) {
    double a[32];
    const bool colok = lane < ell;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      a[i] = (colok && i < ell) ? W[i + static_cast<int64_t>(lane) * ld] : (i == lane ? 1.0 : 0.0);
    const int brk = factor_diag_block(a, W, ld, ell, 0, thresh, Rd, Dt, lane);
    if (lane == 0 && brk < 32) s_r = brk;
  }
  __syncthreads();
  r = s_r;
  // Iteration J: panel J (all warps); then, with lookahead, warp 0 updates and
  // factors diagonal block J+1 while warps 1.. apply the rest of the rank-32
  // trailing update.
  for (int J = 0; J < nbk_all; ++J) {
    const int o = J * 32;
    // Block row J of R right of the diagonal: X = R_JJ^{-T} A_J,chunk (DMMA).
    const int nchunk = (ell - o - 32 + 31) / 32;
    for (int ch = warp; ch < nchunk; ch += kCholWarps) {
      const int cs = o + 32 + ch * 32;
      double acc[2][4][4];
#pragma unroll
      for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[a2][n][q] = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < 32; k0 += 4) {
        // A operand (R_JJ^{-T})[i][k] = Rinv[k][i]
        const double a00 = Dt[(k0 + t) * kInvPitch + g], a01 = Dt[(k0 + t) * kInvPitch + g + 8];
        const double a10 = Dt[(k0 + t) * kInvPitch + g + 16],
                     a11 = Dt[(k0 + t) * kInvPitch + g + 24];
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          const int c = cs + n * 8 + g;
          const double bv = (c < ell) ? W[(o + k0 + t) + static_cast<int64_t>(c) * ld] : 0.0;
          dmma_16x8x4(acc[0][n], a00, a01, bv);
          dmma_16x8x4(acc[1][n], a10, a11, bv);
        }
      }
#pragma unroll
      for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = a2 * 16 + g + ((q & 2) ? 8 : 0);
            const int c = cs + n * 8 + 2 * t + (q & 1);
            if (c < ell) {
              Rp[i * rp_pitch + c] = acc[a2][n][q];
              W[(o + i) + static_cast<int64_t>(c) * ld] = acc[a2][n][q];
            }
          }
    }
    __syncthreads();
    if (r < ell) break;  // rank found: the trailing matrix is not needed
    const int j1 = o + 32;
    if (j1 >= ell) break;
    if (warp == 0) {
      // Lookahead: A_{J+1,J+1} -= R_{J,J+1}^T R_{J,J+1}, then factor it.
      double a[32];
      const bool colok = j1 + lane < ell;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        double v = (colok && j1 + i < ell) ? W[(j1 + i) + static_cast<int64_t>(j1 + lane) * ld]
                                           : (i == lane ? 1.0 : 0.0);
        if (colok && j1 + i < ell) {
          double s = 0.0;
#pragma unroll 8
          for (int k = 0; k < PB; ++k) s = fma(Rp[k * rp_pitch + j1 + i], Rp[k * rp_pitch + j1 + lane], s);
          v -= s;
        }
        a[i] = v;
      }
      const int brk = factor_diag_block(a, W, ld, ell, j1, thresh, Rd, Dt, lane);
      if (lane == 0 && brk < 32) s_r = j1 + brk;
    }
    // Trailing update W[x][y] -= sum_k Rp[k][x] Rp[k][y], x, y in [j1, ell),
    // minus the diagonal block J+1 (warp 0 owns it), on warps 1..
    {
      const int nt = ell - j1;
      const int tiles = (nt + 15) / 16;
      for (int tile = warp - 1; warp > 0 && tile < tiles * tiles; tile += kCholWarps - 1) {
        const int tx = tile % tiles, ty = tile / tiles;
        const int x0 = j1 + tx * 16, y0 = j1 + ty * 16;
        if (x0 < j1 + 32 && y0 < j1 + 32) continue;
        double acc[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[h][q] = 0.0;
#pragma unroll
        for (int k0 = 0; k0 < PB; k0 += 4) {
          const double a0 = Rp[(k0 + t) * rp_pitch + x0 + g];
          const double a1 = Rp[(k0 + t) * rp_pitch + x0 + g + 8];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double b0 = Rp[(k0 + t) * rp_pitch + y0 + h * 8 + g];
            dmma_16x8x4(acc[h], a0, a1, b0);
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int xx = x0 + g + ((q & 2) ? 8 : 0);
            const int yy = y0 + h * 8 + 2 * t + (q & 1);
            if (xx < ell && yy < ell) W[xx + static_cast<int64_t>(yy) * ld] -= acc[h][q];
          }
      }
    }
    __syncthreads();
    r = s_r;
  }
  // Rfull (rows < r of R in original order) and T = R11^{-1}.
  double* Rb = Rfull ? Rfull + b * sq : nullptr;
  if (Rb)
    for (int64_t e = tid; e < sq; e += blockDim.x) {
      const int c = static_cast<int>(e / ld), i = static_cast<int>(e - static_cast<int64_t>(c) * ld);
      Rb[e] = (i < r && i <= c && c < ell) ? W[e] : 0.0;
    }
  const int nbk = (r + 31) / 32;
  const int rpad = nbk * 32;
  for (int64_t e = tid; e < static_cast<int64_t>(rpad) * rpad; e += blockDim.x) {
    const int c = static_cast<int>(e / rpad), i = static_cast<int>(e - static_cast<int64_t>(c) * rpad);
    double v = 0.0;
    if (c < r) v = i <= c ? W[i + static_cast<int64_t>(c) * ld] : 0.0;
    else if (i == c) v = 1.0;
    C11[i + static_cast<int64_t>(c) * ld] = v;
  }
  __syncthreads();
  blocked_upper_inverse(C11, X, ld, nbk, sm, warp, lane);
  double* Tb = T + b * sq;
  for (int64_t e = tid; e < sq; e += blockDim.x) {
    const int c = static_cast<int>(e / ld), i = static_cast<int>(e - static_cast<int64_t>(c) * ld);
    Tb[e] = (c < r && i <= c) ? X[e] : 0.0;
  }
  if (perm_out)
    for (int i = tid; i < ellp; i += blockDim.x) perm_out[b * ellp + i] = i;
  if (tid == 0) rank_out[b] = r;
}


// ---------------------------------------------------------------------------
// Grid-parallel unpivoted Cholesky + inverse (gchol).  The single-CTA kernels
// above keep one item's whole factorization on one SM, which is latency bound
// (~0.7 ms for l = 288, one CTA per item, the trailing matrix in L2).  gchol is
// one persistent cooperative grid over all SMs; per 32-column block J:
//   A  one warp per item factors the updated diagonal block (factor_diag_block:
//      R_JJ and D_J = R_JJ^{-1}, breakdown -> numerical rank);
//   B  warp tasks over (item, 32-column chunk): the block row
//      R_J,right = D_J^T G_J,right, and the block column of the inverse
//      T_I,J = -(sum_{K=I..J-1} T_I,K R_K,J) D_J  (T = R^{-1} built as R is);
//   C  warp tasks over (item, upper 32 x 32 tile): the rank-32 trailing update
//      G_right -= R_J,right^T R_J,right,
// all products on DMMA (mma.sync m16n8k4 f64), operands from L2, with grid-wide
// barriers between the phases.  Same outputs and breakdown rule as uchol_kernel.

// Repeat CholeskyQR passes (the second pass of CholeskyQR2 / 3) factor a Gram
// G = I + E of an already orthonormal-to-O(u kappa^2) basis.  With F = triu(E)
// (diagonal halved), R' = I + F has R'^T R' = G + F^T F and Q = Y (I - F) has
// ||Q^T Q - I|| = O(||F||^2): for ||F||_F^2 <= 1e-16 ~ u that is the exact
// factor's own orthogonality, without the latency-bound factorization.  Items
// with a larger F (ill-conditioned first passes) take the exact path.
// (gchol: CholOpts::lin; fcqr: FcqrArgs::lin.)
constexpr double kLinTol2 = 1e-16;

constexpr int kGcThreads = 256;  // 8 warps: <= 255 registers, so the diagonal factor stays in registers
constexpr int kGcWarps = kGcThreads / 32;
constexpr int kGcDiagWarps = 2;  // warps per CTA with diagonal-factor smem

struct GcholArgs {
  double* G;
  double* T;
  double* Rfull;
  double* scratch;
  int* rank;
  int* perm;
  int ell, ellp;
  double tau;
  int64_t batch;
  CholOpts o;
};

// acc (32 x 32, fragment layout) += A (32 x 32) * B (32 x 32), operands read
// through the accessors; loads of 4 k-steps are issued before their DMMAs so
// each group costs one memory round trip.
template <class FA, class FB>
__device__ __forceinline__ void warp_mma32(double (&acc)[2][4][4], FA&& Aat, FB&& Bat, int g,
                                           int t) {
#pragma unroll
  for (int k1 = 0; k1 < 32; k1 += 16) {
    double av[4][2][2], bv[4][4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int k = k1 + kk * 4 + t;
#pragma unroll
      for (int a2 = 0; a2 < 2; ++a2) {
        av[kk][a2][0] = Aat(a2 * 16 + g, k);
        av[kk][a2][1] = Aat(a2 * 16 + g + 8, k);
      }
#pragma unroll
      for (int n = 0; n < 4; ++n) bv[kk][n] = Bat(k, n * 8 + g);
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        dmma_16x8x4(acc[0][n], av[kk][0][0], av[kk][0][1], bv[kk][n]);
        dmma_16x8x4(acc[1][n], av[kk][1][0], av[kk][1][1], bv[kk][n]);
      }
  }
}

__device__ __forceinline__ void zero_acc(double (&acc)[2][4][4]) {
#pragma unroll
  for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[a2][n][q] = 0.0;
}

// Store the fragment: f(i, c, value) for the 32 x 32 tile.
template <class F>
__device__ __forceinline__ void store_acc(const double (&acc)[2][4][4], F&& f, int g, int t) {
#pragma unroll
  for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        f(a2 * 16 + g + ((q & 2) ? 8 : 0), n * 8 + 2 * t + (q & 1), acc[a2][n][q]);
}

__device__ __forceinline__ double* gc_item_scratch(const GcholArgs& a, int64_t b) {
  return a.scratch + b * 2 * static_cast<int64_t>(a.ellp) * a.ellp;
}

// Phase A for one item by one warp: factor the (updated) diagonal block J,
// publish D_J (scratch) and T_JJ, lower the rank on breakdown.
__device__ void gc_factor_diag(const GcholArgs& a, int64_t b, int J, double* Rd, double* Dt,
                               int lane) {
  const int ell = a.ell, ld = a.ellp, o = J * 32;
  const int64_t sq = static_cast<int64_t>(ld) * ld;
  double* W = a.G + b * sq;
  double* S = gc_item_scratch(a, b);
  double av[32];
  const bool colok = o + lane < ell;
#pragma unroll
  for (int i = 0; i < 32; ++i)
    av[i] = (colok && o + i < ell) ? __ldcg(W + (o + i) + static_cast<int64_t>(o + lane) * ld)
                                   : (i == lane ? 1.0 : 0.0);
  const int brk = factor_diag_block(av, W, ld, ell, o, S[2 * sq - 1], Rd, Dt, lane);
  int r = a.rank[b];
  if (brk < 32 && o + brk < r) r = o + brk;
  double* Tb = a.T + b * sq;
#pragma unroll 4
  for (int i = 0; i < 32; ++i) {
    const double x = Dt[i * kInvPitch + lane];
    S[i * 32 + lane] = x;  // D_J, row-major
    if (o + i < ell && o + lane < ell)
      Tb[(o + i) + static_cast<int64_t>(o + lane) * ld] = (o + lane < r && i <= lane) ? x : 0.0;
  }
  __syncwarp();
  if (lane == 0) a.rank[b] = r;
}

// Grid-parallel unpivoted Cholesky + inverse.  Per 32-column block J
// (right-looking, D_J = R_JJ^{-1}):
//   B  R_J,c = D_J^T G_J,c (c > J) and T_I,J = -Acc_I,J D_J (I < J);
//   C  G_x,y -= R_J,x^T R_J,y (upper tiles), Acc_I,J' (+)= T_I,J R_J,J'
//      (I <= J < J'): the inverse is built right-looking too, so no task
//      carries a chain longer than one 32 x 32 x 32 product; the diagonal block
//      J+1 is updated first and factored by the same warp (lookahead).
// Two grid barriers per block; a launch whose items are all gated off exits
// before the first barrier.
// CLU: the whole (small) grid is one thread-block cluster and the grid
// barriers become cluster barriers (hardware, ~1 us cheaper each); used for
// single matrices / small batches whose widest step fits 16 CTAs.  Cross-CTA
// data is read with ld.global.cg in both modes.
// MODE 0: persistent cooperative grid over all items; MODE 1: the same as
// one thread-block cluster; MODE 2: one independent CTA per item (blockIdx.x
// = item, block barriers only, no co-residency needed) -- for small l_p,
// where an item's whole factorization is a few dozen warp tasks and the
// grid / cluster barriers would dominate.
#ifdef RSVD_GCHOL_TRACE
// %globaltimer stamps of CTA 0, thread 0: [0] start, [1] before block 0's
// factor, [2 + 2 J] phase B of block J starts, [3 + 2 J] phase C starts
// (tools/probe/gchol_trace.cu).
__device__ unsigned long long g_gc_trace[160];
#define GC_TRACE(i)                                                                        \
  do {                                                                                     \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (i) < 160) {                               \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      g_gc_trace[i] = t_;                                                                  \
    }                                                                                      \
  } while (0)
#else
#define GC_TRACE(i) do {} while (0)
#endif

template <int MODE>
__global__ void __launch_bounds__(kGcThreads, 1) gchol_kernel(const GcholArgs a_in) {
  namespace cg = cooperative_groups;
  struct Sync {
    __device__ void sync() {
      if constexpr (MODE == 1)
        cg::this_cluster().sync();
      else if constexpr (MODE == 2)
        __syncthreads();
      else
        cg::this_grid().sync();
    }
  } grid;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_any;
  GcholArgs a = a_in;
  int cta = blockIdx.x, ncta = gridDim.x;
  if constexpr (MODE == 2) {  // this CTA's item as a batch of one
    const int64_t b0 = blockIdx.x, q = static_cast<int64_t>(a.ellp) * a.ellp;
    a.G += b0 * q;
    a.T += b0 * q;
    if (a.Rfull) a.Rfull += b0 * q;
    a.scratch += b0 * 2 * q;
    a.rank += b0;
    if (a.perm) a.perm += b0 * a.ellp;
    if (a.o.gate_rank) a.o.gate_rank += b0;
    if (a.o.mask) a.o.mask += b0;
    if (a.o.ill_out) a.o.ill_out += b0;
    if (a.o.Gsrc) a.o.Gsrc += b0 * q;
    a.batch = 1;
    cta = 0;
    ncta = 1;
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ell = a.ell, ld = a.ellp;
  const int64_t sq = static_cast<int64_t>(ld) * ld;
  const int64_t batch = a.batch;
  const int nb = (ell + 31) / 32;
  GC_TRACE(0);
  const int64_t gw = static_cast<int64_t>(cta) * kGcWarps + warp;
  const int64_t nw = static_cast<int64_t>(ncta) * kGcWarps;
  const int64_t gtid = static_cast<int64_t>(cta) * blockDim.x + tid;
  const int64_t gstride = static_cast<int64_t>(ncta) * blockDim.x;
  // scratch per item: [0, 1024) D_J; [sq, 2 sq) Acc (strictly upper blocks);
  // [2 sq - 3] ||F||_F^2 (lin), [2 sq - 2] go flag, [2 sq - 1] pivot floor
  // (a diagonal block of Acc).
  auto go_of = [&](int64_t b) -> double* { return gc_item_scratch(a, b) + 2 * sq - 2; };
  const bool lin = a.o.lin;
  auto gate = [&](int64_t b) {
    int go = 1;
    if (a.o.gate_rank) go = a.o.gate_rank[b] < ell;
    if (a.o.mask && !a.o.mask[b]) go = 0;
    return go;
  };
  // Every CTA evaluates the same predicate: all exit together or none does.
  if (tid == 0) s_any = 0;
  __syncthreads();
  for (int64_t b = tid; b < batch; b += blockDim.x)
    if (gate(b)) s_any = 1;
  __syncthreads();
  if (!s_any) {
    if (a.o.ill_out)
      for (int64_t b = gtid; b < batch; b += gstride) a.o.ill_out[b] = 0;
    return;
  }
  for (int64_t b = gtid; b < batch; b += gstride) {
    const int go = gate(b);
    if (a.o.ill_out) a.o.ill_out[b] = (a.o.gate_rank && a.o.gate_rank[b] < ell) ? 1 : 0;
    go_of(b)[0] = go ? 1.0 : 0.0;
    if (lin) go_of(b)[-1] = 0.0;
  }
  grid.sync();
  // Per item (flag read once), 16-byte stores (sq is a multiple of 1024),
  // spread over the whole grid: one CTA per item left single matrices with
  // ~40 us of zeroing on one SM (l_p = 544).
  for (int64_t b = 0; b < batch; ++b) {
    if (go_of(b)[0] == 0.0) continue;
    double2* t2 = reinterpret_cast<double2*>(a.T + b * sq);
    const double2 z = make_double2(0.0, 0.0);
    for (int64_t e = gtid; e < sq / 2; e += gstride) t2[e] = z;
    if (lin) {  // ||F||_F^2 over the upper triangle, grid-wide
      __shared__ double s_f;
      if (tid == 0) s_f = 0.0;
      __syncthreads();
      const double* W = a.G + b * sq;
      double f2 = 0.0;
      for (int64_t e = gtid; e < sq; e += gstride) {
        const int i = static_cast<int>(e % ld), j = static_cast<int>(e / ld);
        if (i <= j && j < ell) {
          const double v = __ldcg(W + e);
          const double f = i == j ? 0.5 * (v - 1.0) : v;
          f2 = fma(f, f, f2);
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) f2 += __shfl_xor_sync(0xffffffffu, f2, off);
      if (lane == 0) atomicAdd(&s_f, f2);
      __syncthreads();
      if (tid == 0) atomicAdd(go_of(b) - 1, s_f);
    }
    if (a.o.Gsrc) {
      const double2* s2 = reinterpret_cast<const double2*>(a.o.Gsrc + b * sq);
      double2* g2 = reinterpret_cast<double2*>(a.G + b * sq);
      for (int64_t e = gtid; e < sq / 2; e += gstride) g2[e] = s2[e];
    }
  }
  grid.sync();
  if (lin) {
    // Items with ||F||_F^2 <= kLinTol2: T = I - F, Rfull = I + F, rank = ell,
    // written grid-wide; their go flag is cleared below (gate() and the sum
    // are stable in this phase, the flag is not).
    for (int64_t b = 0; b < batch; ++b) {
      if (!gate(b) || !(__ldcg(go_of(b) - 1) <= kLinTol2)) continue;
      const double* W = a.G + b * sq;
      double* Tb = a.T + b * sq;
      for (int64_t e = gtid; e < sq; e += gstride) {
        const int i = static_cast<int>(e % ld), j = static_cast<int>(e / ld);
        const bool up = i <= j && j < ell;
        const double v = up ? __ldcg(W + e) : 0.0;
        if (up) Tb[e] = i == j ? fma(-0.5, v, 1.5) : -v;
        if (a.Rfull) a.Rfull[b * sq + e] = up ? (i == j ? fma(0.5, v, 0.5) : v) : 0.0;
      }
      if (a.perm)
        for (int64_t e = gtid; e < ld; e += gstride) a.perm[b * ld + e] = static_cast<int>(e);
    }
  }
  for (int64_t b = gw; b < batch; b += nw) {  // shift, pivot floor, initial rank
    if (go_of(b)[0] == 0.0) continue;
    if (lin && __ldcg(go_of(b) - 1) <= kLinTol2) {
      __syncwarp();
      if (lane == 0) {
        a.rank[b] = ell;
        go_of(b)[0] = 0.0;
      }
      continue;
    }
    double* W = a.G + b * sq;
    double tr = 0.0, mx = 0.0;
    for (int i = lane; i < ell; i += 32) {
      const double d = W[i + static_cast<int64_t>(i) * ld];
      tr += d;
      mx = fmax(mx, d);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      tr += __shfl_xor_sync(0xffffffffu, tr, off);
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    }
    if (a.o.shift_coef > 0.0) {
      const double sh = a.o.shift_coef * tr;
      for (int i = lane; i < ell; i += 32) W[i + static_cast<int64_t>(i) * ld] += sh;
      mx += sh;
    }
    __syncwarp();
    if (lane == 0) {
      go_of(b)[1] = a.tau * mx;
      a.rank[b] = (mx > 0.0) ? ell : 0;
    }
  }
  grid.sync();
  if (lin) {  // every item took the first-order factor: all CTAs leave together
    if (tid == 0) s_any = 0;
    __syncthreads();
    for (int64_t b = tid; b < batch; b += blockDim.x)
      if (__ldcg(go_of(b)) != 0.0) s_any = 1;
    __syncthreads();
    if (!s_any) return;
  }

  const bool diag_warp = warp < kGcDiagWarps;
  double* Rd = sm + (diag_warp ? warp : 0) * 2 * 32 * kInvPitch;
  double* Dt = Rd + 32 * kInvPitch;
  // Items whose diagonal factorizations this warp owns.
  const int64_t d0 = static_cast<int64_t>(cta) + static_cast<int64_t>(warp) * ncta;
  const int64_t dstep = static_cast<int64_t>(ncta) * kGcDiagWarps;
  GC_TRACE(1);
  if (diag_warp)
    for (int64_t b = d0; b < batch; b += dstep)
      if (go_of(b)[0] != 0.0 && a.rank[b] > 0) gc_factor_diag(a, b, 0, Rd, Dt, lane);
  grid.sync();

  const int64_t pw = static_cast<int64_t>(cta) * (kGcWarps - kGcDiagWarps) + (warp - kGcDiagWarps);
  const int64_t npw = static_cast<int64_t>(ncta) * (kGcWarps - kGcDiagWarps);
  for (int J = 0; J < nb; ++J) {
    const int o = J * 32;
    const int nr = nb - J - 1;  // blocks right of J
    GC_TRACE(2 + 2 * J);
    // ---- Phase B ----------------------------------------------------------
    {
      const int per = nr + J;
      for (int64_t task = gw; task < batch * per; task += nw) {
        const int64_t b = task / per;
        const int idx = static_cast<int>(task - b * per);
        if (go_of(b)[0] == 0.0) continue;
        const int r = a.rank[b];
        if (r <= o) continue;
        double* W = a.G + b * sq;
        const double* D = gc_item_scratch(a, b);
        double acc[2][4][4];
        zero_acc(acc);
        if (idx < nr) {
          if (r < o + 32) continue;  // broke down inside block J
          const int cs = o + 32 + idx * 32;
          warp_mma32(acc, [&](int i, int k) { return D[k * 32 + i]; },
                     [&](int k, int c) {
                       return cs + c < ell ? __ldcg(W + (o + k) + static_cast<int64_t>(cs + c) * ld)
                                           : 0.0;
                     },
                     g, t);
          store_acc(acc, [&](int i, int c, double v) {
            if (cs + c < ell) W[(o + i) + static_cast<int64_t>(cs + c) * ld] = v;
          }, g, t);
        } else {
          const int I = idx - nr;
          const double* Acc = gc_item_scratch(a, b) + sq;
          warp_mma32(acc,
                     [&](int i, int k) {
                       return __ldcg(Acc + (32 * I + i) + static_cast<int64_t>(o + k) * ld);
                     },
                     [&](int k, int c) { return D[k * 32 + c]; }, g, t);
          double* Tb = a.T + b * sq;
          store_acc(acc, [&](int i, int c, double v) {
            if (o + c < ell) Tb[(32 * I + i) + static_cast<int64_t>(o + c) * ld] = (o + c < r) ? -v : 0.0;
          }, g, t);
        }
      }
    }
    grid.sync();
    GC_TRACE(3 + 2 * J);
    if (nr == 0) break;
    // ---- Phase C (+ lookahead factor of block J+1) -----------------------
    if (diag_warp) {
      for (int64_t b = d0; b < batch; b += dstep) {
        if (go_of(b)[0] == 0.0 || a.rank[b] < o + 32) continue;
        double* W = a.G + b * sq;
        const int x0 = o + 32;
        double acc[2][4][4];
        zero_acc(acc);
        warp_mma32(acc,
                   [&](int i, int k) {
                     return x0 + i < ell ? __ldcg(W + (o + k) + static_cast<int64_t>(x0 + i) * ld) : 0.0;
                   },
                   [&](int k, int c) {
                     return x0 + c < ell ? __ldcg(W + (o + k) + static_cast<int64_t>(x0 + c) * ld) : 0.0;
                   },
                   g, t);
        store_acc(acc, [&](int i, int c, double v) {
          if (x0 + i < ell && x0 + c < ell) W[(x0 + i) + static_cast<int64_t>(x0 + c) * ld] -= v;
        }, g, t);
        __syncwarp();
        gc_factor_diag(a, b, J + 1, Rd, Dt, lane);
      }
    } else {
      // Tile tasks per item: nr (nr + 1) / 2 - 1 trailing tiles (tx <= ty,
      // without (0, 0)) then (J + 1) * nr inverse-accumulation tiles.
      const int ntr = nr * (nr + 1) / 2 - 1;
      const int per = ntr + (J + 1) * nr;
      for (int64_t task = pw; task < batch * per; task += npw) {
        const int64_t b = task / per;
        int idx = static_cast<int>(task - b * per);
        if (go_of(b)[0] == 0.0 || a.rank[b] < o + 32) continue;
        double* W = a.G + b * sq;
        double acc[2][4][4];
        zero_acc(acc);
        if (idx < ntr) {
          idx += 1;
          int ty = 0;
          while (idx > ty) idx -= ++ty;
          const int x0 = o + 32 + 32 * idx, y0 = o + 32 + 32 * ty;
          warp_mma32(acc,
                     [&](int i, int k) {
                       return x0 + i < ell ? __ldcg(W + (o + k) + static_cast<int64_t>(x0 + i) * ld) : 0.0;
                     },
                     [&](int k, int c) {
                       return y0 + c < ell ? __ldcg(W + (o + k) + static_cast<int64_t>(y0 + c) * ld) : 0.0;
                     },
                     g, t);
          store_acc(acc, [&](int i, int c, double v) {
            if (x0 + i < ell && y0 + c < ell) W[(x0 + i) + static_cast<int64_t>(y0 + c) * ld] -= v;
          }, g, t);
        } else {
          idx -= ntr;
          const int I = idx / nr, Jp = J + 1 + idx % nr;  // Acc_I,J' (+)= T_I,J R_J,J'
          const double* Tb = a.T + b * sq;
          double* Acc = gc_item_scratch(a, b) + sq;
          warp_mma32(acc,
                     [&](int i, int k) {
                       return __ldcg(Tb + (32 * I + i) + static_cast<int64_t>(o + k) * ld);
                     },
                     [&](int k, int c) {
                       return 32 * Jp + c < ell
                                  ? __ldcg(W + (o + k) + static_cast<int64_t>(32 * Jp + c) * ld)
                                  : 0.0;
                     },
                     g, t);
          const bool first = I == J;
          store_acc(acc, [&](int i, int c, double v) {
            double* p = Acc + (32 * I + i) + static_cast<int64_t>(32 * Jp + c) * ld;
            *p = first ? v : *p + v;
          }, g, t);
        }
      }
    }
    grid.sync();
  }
  // Epilogue: Rfull (rows < r, upper), identity permutation.
  for (int64_t b = cta; b < batch; b += ncta) {
    if (go_of(b)[0] == 0.0) continue;
    if (a.perm)
      for (int i = tid; i < ld; i += blockDim.x) a.perm[b * ld + i] = i;
    if (!a.Rfull) continue;
    const int r = a.rank[b];
    for (int c = warp; c < ld; c += kGcWarps)
      for (int i = lane; i < ld; i += 32) {
        const int64_t e = b * sq + i + static_cast<int64_t>(c) * ld;
        a.Rfull[e] = (i < r && i <= c && c < ell) ? a.G[e] : 0.0;
      }
  }
}

// ---------------------------------------------------------------------------
// Fused CholeskyQR pass for small bases (fcqr_kernel), l_p <= 160: one CTA per
// item does the whole pass -- Gram, Cholesky, inverse factors and Q = Y R^-1 --
// with the Gram / R kept in shared memory as upper 32 x 32 blocks, so the
// latency-bound small factorization never goes through L2 or a grid barrier
// and the three launches (+ split-K reduce and mirror) of the unfused pass
// become one.  Same outputs and breakdown rule as gchol_kernel:
//   1. G = Y^T Y, upper blocks, Y streamed in CR-row chunks (cp.async double
//      buffer, DMMA); the full symmetric G is also written to G0 (global) for
//      the shifted-CholeskyQR retry of ill-conditioned items;
//   2. per 32-column block J: one warp factors the diagonal block
//      (factor_diag_block: R_JJ, D_J = R_JJ^-1, breakdown at pivot <= tau *
//      max diag G -> rank r), R_J,c = D_J^T G_J,c, trailing update
//      G_c,c' -= R_J,c^T R_J,c' (warp tasks, DMMA, shared memory);
//   3. Rf = R (rows < r) when requested; W_IJ = R_IJ D_J in place of R_IJ;
//   4. Q_J = Y_J D_J - sum_{I<J} Q_I W_IJ: each warp owns 16-row slabs and runs
//      the block columns J in order (no CTA barrier; columns >= r are zero, the
//      caller's completion fills them).
// 16-byte global -> shared async copy; bytes < 16 zero-fills the rest.
__device__ __forceinline__ void cpa16(void* dst, const void* src, int bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes)
               : "memory");
}

constexpr int kFqThreads = 256;  // 8 warps: <= 255 registers, the diagonal factor stays in registers
constexpr int kFqWarps = kFqThreads / 32;
constexpr int kFqBlk = 32 * kInvPitch;  // doubles per stored 32 x 32 block (pitch 36)

struct FcqrArgs {
  const double* Y;
  int64_t ldy, sY;
  double* Q;
  int64_t ldq, sQ;
  double* G0;  // full symmetric Gram (l_p x l_p, ld l_p) per item, or null
  double* Rf;  // R (l_p x l_p, ld l_p, upper, zero below / beyond rank), or null
  double* xs;  // CLU: per item (nub + nbk) blocks of kFqBlk doubles (D_J / W_IJ exchange)
  int* rank;
  int rows, ell, ellp, cr;  // cr: staged rows per chunk (multiple of 16)
  double tau;
  int lin;  // repeat pass: first-order factor when ||triu(G - I)||_F^2 <= kLinTol2
};

__device__ __forceinline__ int fq_ub(int I, int J) { return J * (J + 1) / 2 + I; }  // I <= J

// CLU: the item is owned by a thread-block cluster of S CTAs that split its
// rows; the partial Grams are summed through DSMEM in rank order (each CTA
// reduces every S-th block into CTA 0), CTA 0 factors, and every CTA copies
// D_J / W_IJ back from CTA 0 and applies them to its own rows -- for single
// or few items, whose Gram and apply would otherwise run on one SM.
#ifdef RSVD_FCQR_TRACE
__device__ unsigned long long g_fq_trace[64];
#define FQ_TRACE(i)                                                                        \
  do {                                                                                     \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                             \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      g_fq_trace[i] = t_;                                                                  \
    }                                                                                      \
  } while (0)
#else
#define FQ_TRACE(i) do {} while (0)
#endif
template <bool CLU>
__global__ void __launch_bounds__(kFqThreads, 1) fcqr_kernel(const FcqrArgs a) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double sm[];
  __shared__ double s_red[kFqWarps];
  __shared__ int s_rank;
  __shared__ double s_thresh;
  int S = 1, q = 0;
  int64_t b = blockIdx.x;
  if constexpr (CLU) {
    S = static_cast<int>(cg::this_cluster().num_blocks());
    q = static_cast<int>(cg::this_cluster().block_rank());
    b = blockIdx.x / S;
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int ell = a.ell, ellp = a.ellp, rows = a.rows, CR = a.cr, CRP = a.cr + 4;
  const int nbk = ellp / 32, nub = nbk * (nbk + 1) / 2;
  double* Gb = sm;                   // upper blocks, element (i, j) at i + j * kInvPitch
  double* U = sm + nub * kFqBlk;     // union: Y chunk buffers | D_J blocks + diag scratch
  double* Dst = U;                   // D_J (row-major, pitch kInvPitch), J < nbk
  double* Rd = U + nbk * kFqBlk;     // factor_diag_block scratch
  double* Dt = Rd + kFqBlk;
  const double* Y = a.Y + b * a.sY;
  double* Q = a.Q + b * a.sQ;
  auto blk = [&](int I, int J) { return Gb + fq_ub(I, J) * kFqBlk; };
  // this CTA's rows [row0, row0 + nrow)
  const int rpc = ((rows + S - 1) / S + 15) & ~15;  // multiple of 16: aligned 16-byte row pairs
  const int row0 = q * rpc, nrow = max(0, min(rows, row0 + rpc) - row0);
  FQ_TRACE(0);

  // ---- 1. Gram (upper blocks) ------------------------------------------------
  // 16-byte copies need 16-byte aligned columns (even ld, aligned base);
  // otherwise (odd row counts) 8-byte copies.
  const bool vec16 = (a.ldy % 2 == 0) && (a.sY % 2 == 0) &&
                     ((reinterpret_cast<uintptr_t>(a.Y) & 15u) == 0);
  double* const Sbuf = sm;  // the Gram phase stages Y over the whole shared memory
  auto stage = [&](int c, int buf) {
    const int r0 = row0 + c * CR;
    double* dst = Sbuf + buf * ellp * CRP;
    if (vec16) {
      const int per = CR / 2;
      for (int e = tid; e < ellp * per; e += kFqThreads) {
        const int col = e / per, r = 2 * (e - col * per);
        const int gr = r0 + r;
        int bytes = 0;
        const double* src = Y;
        if (col < ell && gr < row0 + nrow) {
          bytes = min(16, (row0 + nrow - gr) * 8);
          src = Y + gr + static_cast<int64_t>(col) * a.ldy;
        }
        cpa16(dst + r + col * CRP, src, bytes);
      }
    } else {
      for (int e = tid; e < ellp * CR; e += kFqThreads) {
        const int col = e / CR, r = e - col * CR;
        const int gr = r0 + r;
        const bool ok = col < ell && gr < row0 + nrow;
        const double* src = ok ? Y + gr + static_cast<int64_t>(col) * a.ldy : Y;
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst + r + col * CRP));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
                     "r"(ok ? 8 : 0)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  const int nch = (nrow + CR - 1) / CR;
  // Whole upper 32 x 32 blocks per warp (block ub = warp, warp + 8: at most 2
  // for l_p <= 160), register-blocked like warp_mma32: per k-step 8 fragment
  // loads feed 8 independent DMMAs (per-tile operands would need 3 loads per
  // DMMA and leave the Gram shared-memory bound).
  constexpr int kGB = 2;
  int bI[kGB], bJ[kGB];
#pragma unroll
  for (int v = 0; v < kGB; ++v) {
    const int ub = warp + kFqWarps * v;
    int J = 0;
    while ((J + 1) * (J + 2) / 2 <= ub) ++J;
    bJ[v] = J;
    bI[v] = ub - J * (J + 1) / 2;
  }
  double acc[kGB][2][4][4];
#pragma unroll
  for (int v = 0; v < kGB; ++v) zero_acc(acc[v]);
  if (nch > 0) stage(0, 0);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      stage(c + 1, (c + 1) & 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    if (c == 0) FQ_TRACE(14);
    const double* Yc = Sbuf + (c & 1) * ellp * CRP;
#pragma unroll
    for (int v = 0; v < kGB; ++v) {
      if (warp + kFqWarps * v < nub) {
        const double* Ab = Yc + (32 * bI[v] + g) * CRP + t;
        const double* Bb = Yc + (32 * bJ[v] + g) * CRP + t;
#pragma unroll 2
        for (int k0 = 0; k0 < CR; k0 += 4) {
          double av[2][2], bv[4];
#pragma unroll
          for (int a2 = 0; a2 < 2; ++a2) {
            av[a2][0] = Ab[(16 * a2) * CRP + k0];
            av[a2][1] = Ab[(16 * a2 + 8) * CRP + k0];
          }
#pragma unroll
          for (int n = 0; n < 4; ++n) bv[n] = Bb[(8 * n) * CRP + k0];
#pragma unroll
          for (int n = 0; n < 4; ++n) {
            dmma_16x8x4(acc[v][0][n], av[0][0], av[0][1], bv[n]);
            dmma_16x8x4(acc[v][1][n], av[1][0], av[1][1], bv[n]);
          }
        }
      }
    }
    __syncthreads();  // buffer c & 1 is restaged at c + 2; the last one frees the G blocks
    if (c == 0) FQ_TRACE(15);
  }
#pragma unroll
  for (int v = 0; v < kGB; ++v) {
    const int ub = warp + kFqWarps * v;
    if (ub < nub) {
      double* W = Gb + ub * kFqBlk;
      double* G0 = (!CLU && a.G0) ? a.G0 + b * static_cast<int64_t>(ellp) * ellp : nullptr;
      const int I = bI[v], J = bJ[v];
      store_acc(acc[v], [&](int i, int j, double x) {
        W[i + j * kInvPitch] = x;
        if (G0) {
          const int64_t gi = 32 * I + i, gj = 32 * J + j;
          G0[gi + gj * ellp] = x;
          G0[gj + gi * ellp] = x;
        }
      }, g, t);
    }
  }
  __syncthreads();
  if constexpr (CLU) {
    // Sum the S partial Grams into CTA 0, block ub by CTA ub mod S, ranks in
    // order (bit-identical to any schedule).
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    double* G0 = a.G0 ? a.G0 + b * static_cast<int64_t>(ellp) * ellp : nullptr;
    double* dst0 = cl.map_shared_rank(Gb, 0);
    for (int ub = q; ub < nub; ub += S) {
      int J = 0;
      while ((J + 1) * (J + 2) / 2 <= ub) ++J;
      const int I = ub - J * (J + 1) / 2;
      for (int e = tid; e < 1024; e += kFqThreads) {
        const int i = e & 31, j = e >> 5;
        const int off = ub * kFqBlk + i + j * kInvPitch;
        double v = 0.0;
        for (int r = 0; r < S; ++r) v += cl.map_shared_rank(Gb, r)[off];
        dst0[off] = v;
        if (G0) {
          const int64_t gi = 32 * I + i, gj = 32 * J + j;
          G0[gi + gj * ellp] = v;
          G0[gj + gi * ellp] = v;
        }
      }
    }
    cl.sync();
  }
  FQ_TRACE(2);

  // ---- 1b. repeat pass: first-order factor when G = I + small E -------------
  __shared__ int s_lin;
  __shared__ double s_ef[kFqWarps];
  if (q == 0) {
    if (a.lin) {
      double ef = 0.0;  // ||F||_F^2, F = triu(E) with diag(E) / 2
      for (int ub = warp; ub < nub; ub += kFqWarps) {
        int J = 0;
        while ((J + 1) * (J + 2) / 2 <= ub) ++J;
        const int I = ub - J * (J + 1) / 2;
        const double* Wb = blk(I, J);
        for (int e = lane; e < 1024; e += 32) {
          const int i = e & 31, j = e >> 5, gi = 32 * I + i, gj = 32 * J + j;
          if (gi <= gj && gj < ell) {
            const double v = Wb[i + j * kInvPitch];
            const double f = gi == gj ? 0.5 * (v - 1.0) : v;
            ef = fma(f, f, ef);
          }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ef += __shfl_xor_sync(0xffffffffu, ef, off);
      if (lane == 0) s_ef[warp] = ef;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kFqWarps; ++w) t += s_ef[w];
        s_lin = t <= kLinTol2 ? 1 : 0;  // NaN fails
      }
    } else if (tid == 0) {
      s_lin = 0;
    }
    __syncthreads();
  }
  // ---- 2. pivot floor, rank; blocked Cholesky in shared memory ---------------
  if (q == 0 && s_lin) {
    // R = I + F: W_IJ = R_IJ D_J = F_IJ + O(E^2) = G_IJ (already in place),
    // D_J = I - F_JJ, rank = ell; Rf = I + F when requested.
    for (int J = 0; J < nbk; ++J) {
      const double* Gj = blk(J, J);
      double* D = Dst + J * kFqBlk;
      for (int e = tid; e < 1024; e += kFqThreads) {
        const int i = e >> 5, j = e & 31, gi = 32 * J + i, gj = 32 * J + j;
        double v = (i == j) ? 1.0 : 0.0;
        if (gi < ell && gj < ell) {
          if (i < j) v = -Gj[i + j * kInvPitch];
          else if (i == j) v = fma(-0.5, Gj[i + j * kInvPitch], 1.5);
        }
        D[i * kInvPitch + j] = v;  // row-major, as the apply reads it
      }
    }
    if (tid == 0) {
      s_rank = ell;
      a.rank[b] = ell;
    }
    if (a.Rf) {
      double* Rf = a.Rf + b * static_cast<int64_t>(ellp) * ellp;
      for (int e = tid; e < ellp * ellp; e += kFqThreads) {
        const int i = e % ellp, j = e / ellp;
        double v = 0.0;
        if (i <= j && j < ell) {
          const double gv = blk(i >> 5, j >> 5)[(i & 31) + (j & 31) * kInvPitch];
          v = (i < j) ? gv : fma(0.5, gv, 0.5);
        }
        Rf[e] = v;
      }
    }
    __syncthreads();
  } else if (q == 0) {
  if (warp == 0) {
    double mx = 0.0;
    for (int i = lane; i < ell; i += 32) mx = fmax(mx, blk(i >> 5, i >> 5)[(i & 31) * (kInvPitch + 1)]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if (lane == 0) {
      s_thresh = a.tau * mx;
      s_rank = mx > 0.0 ? ell : 0;
    }
  }
  __syncthreads();
  const double thresh = s_thresh;
  // Factor the diagonal block J by warp 0 (R_JJ in place, D_J = R_JJ^-1,
  // breakdown -> rank).
  auto factor = [&](int J) {
    double* W = blk(J, J);
    double av[32];
    const bool colok = 32 * J + lane < ell;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      av[i] = (colok && 32 * J + i < ell) ? W[i + lane * kInvPitch] : (i == lane ? 1.0 : 0.0);
    const int brk = factor_diag_block(av, W, kInvPitch, ell - 32 * J, 0, thresh, Rd, Dt, lane);
    double* D = Dst + J * kFqBlk;
#pragma unroll 4
    for (int k = 0; k < 32; ++k) D[lane * kInvPitch + k] = Dt[lane * kInvPitch + k];
    if (lane == 0 && brk < 32 && 32 * J + brk < s_rank) s_rank = 32 * J + brk;
  };
  if (warp == 0 && s_rank > 0) factor(0);
  __syncthreads();
  FQ_TRACE(3);
  for (int J = 0; J < nbk; ++J) {
    if (s_rank < 32 * (J + 1)) break;  // broke down in or before block J
    const int nr = nbk - J - 1;
    if (nr == 0) break;
    const double* D = Dst + J * kFqBlk;
    for (int c = J + 1 + warp; c < nbk; c += kFqWarps) {  // R_J,c = D_J^T G_J,c
      double* W = blk(J, c);
      double ac[2][4][4];
      zero_acc(ac);
      warp_mma32(ac, [&](int i, int k) { return D[k * kInvPitch + i]; },
                 [&](int k, int cc) { return W[k + cc * kInvPitch]; }, g, t);
      __syncwarp();
      store_acc(ac, [&](int i, int cc, double v) { W[i + cc * kInvPitch] = v; }, g, t);
    }
    __syncthreads();
    // G_c,c' -= R_J,c^T R_J,c' (J < c <= c'); warp 0 takes (J+1, J+1) and then
    // factors block J+1 while the other warps finish the trailing tiles.
    auto trail = [&](int c, int c2) {
      const double* Rc = blk(J, c);
      const double* Rc2 = blk(J, c2);
      double* W = blk(c, c2);
      double ac[2][4][4];
      zero_acc(ac);
      warp_mma32(ac, [&](int i, int k) { return Rc[k + i * kInvPitch]; },
                 [&](int k, int cc) { return Rc2[k + cc * kInvPitch]; }, g, t);
      store_acc(ac, [&](int i, int cc, double v) { W[i + cc * kInvPitch] -= v; }, g, t);
    };
    if (warp == 0) {
      trail(J + 1, J + 1);
      __syncwarp();
      if (32 * (J + 1) < s_rank) factor(J + 1);
    } else {
      const int ntr = nr * (nr + 1) / 2;
      for (int task = 1 + (warp - 1); task < ntr; task += kFqWarps - 1) {
        int idx = task, cp = 0;
        while (idx > cp) idx -= ++cp;
        trail(J + 1 + idx, J + 1 + cp);
      }
    }
    __syncthreads();
    FQ_TRACE(4 + J);
  }
  FQ_TRACE(10);
  const int r = s_rank;
  const int nbr = (r + 31) / 32;  // block columns with live R / D

  // ---- 3. outputs: rank, Rf; W_IJ = R_IJ D_J in place ---------------------------
  if (tid == 0) a.rank[b] = r;
  if (a.Rf) {
    double* Rf = a.Rf + b * static_cast<int64_t>(ellp) * ellp;
    for (int e = tid; e < ellp * ellp; e += kFqThreads) {
      const int i = e % ellp, j = e / ellp;
      double v = 0.0;
      if (i < r && i <= j && j < ell) v = blk(i >> 5, j >> 5)[(i & 31) + (j & 31) * kInvPitch];
      Rf[e] = v;
    }
    __syncthreads();
  }
  {
    const int nw = nbr * (nbr - 1) / 2;
    for (int task = warp; task < nw; task += kFqWarps) {
      int I = task, J = 1;
      while (I >= J) I -= J++;
      double* W = blk(I, J);
      const double* D = Dst + J * kFqBlk;
      double ac[2][4][4];
      zero_acc(ac);
      warp_mma32(ac, [&](int i, int k) { return W[i + k * kInvPitch]; },
                 [&](int k, int cc) { return D[k * kInvPitch + cc]; }, g, t);
      __syncwarp();
      store_acc(ac, [&](int i, int cc, double v) { W[i + cc * kInvPitch] = v; }, g, t);
    }
  }
  __syncthreads();
  FQ_TRACE(11);
  }  // q == 0
  if constexpr (CLU) {
    // Every CTA takes D_J, W_IJ (I < J) and the rank from CTA 0 through L2:
    // CTA 0 writes them to xs, the others stage them back with 16-byte
    // cp.async (reading them through DSMEM serialises on CTA 0's SM).
    cg::cluster_group cl = cg::this_cluster();
    constexpr int per = kFqBlk / 2;
    const int nw = nbk * (nbk - 1) / 2, nblk = nw + nbk;
    auto off = [&](int e) {  // e-th double2 of the exchange -> its shared-memory index
      const int bi = e / per, w = e - bi * per;
      if (bi < nw) {
        int I = bi, J = 1;
        while (I >= J) I -= J++;
        return fq_ub(I, J) * per + w;
      }
      return (nub + bi - nw) * per + w;
    };
    double2* xg = reinterpret_cast<double2*>(a.xs + b * static_cast<int64_t>(nub + nbk) * kFqBlk);
    if (q == 0) {
      const double2* s2 = reinterpret_cast<const double2*>(sm);
      for (int e = tid; e < nblk * per; e += kFqThreads) __stcg(xg + e, s2[off(e)]);
      __threadfence();
    }
    cl.sync();
    if (q != 0) {
      for (int e = tid; e < nblk * per; e += kFqThreads) cpa16(sm + 2 * off(e), xg + e, 16);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      if (tid == 0) s_rank = *cl.map_shared_rank(&s_rank, 0);
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    cl.sync();  // CTA 0's s_rank stays alive until every CTA has read it
  }
  const int r = s_rank;
  const int nbr = (r + 31) / 32;

  // ---- 4. Q = Y R^-1, 16-row slabs per warp, block columns in order -----------
  const int rend = row0 + nrow;
  for (int r0 = row0 + 16 * warp; r0 < rend; r0 += 16 * kFqWarps) {
    const int ra = r0 + g, rb = r0 + g + 8;
    for (int J = 0; J < nbk; ++J) {
      double ac[4][4];
#pragma unroll
      for (int n = 0; n < 4; ++n)
#pragma unroll
        for (int q = 0; q < 4; ++q) ac[n][q] = 0.0;
      if (J < nbr) {
        // All 8 k-steps' fragments of a 32-column block are loaded before
        // their DMMAs: one L2 round trip per block instead of four.
        const double* D = Dst + J * kFqBlk;
        const double* Yj = Y + static_cast<int64_t>(32 * J) * a.ldy;
        double a0v[8], a1v[8];
#pragma unroll
        for (int kq = 0; kq < 8; ++kq) {
          const int k = 4 * kq + t;
          const bool okc = 32 * J + k < ell;
          a0v[kq] = (okc && ra < rend) ? __ldcg(Yj + ra + static_cast<int64_t>(k) * a.ldy) : 0.0;
          a1v[kq] = (okc && rb < rend) ? __ldcg(Yj + rb + static_cast<int64_t>(k) * a.ldy) : 0.0;
        }
#pragma unroll
        for (int kq = 0; kq < 8; ++kq)
#pragma unroll
          for (int n = 0; n < 4; ++n)
            dmma_16x8x4(ac[n], a0v[kq], a1v[kq], D[(4 * kq + t) * kInvPitch + n * 8 + g]);
        for (int I = 0; I < J; ++I) {
          const double* W = blk(I, J);
          const double* Qi = Q + static_cast<int64_t>(32 * I) * a.ldq;
#pragma unroll
          for (int kq = 0; kq < 8; ++kq) {
            const int k = 4 * kq + t;
            a0v[kq] = ra < rend ? __ldcg(Qi + ra + static_cast<int64_t>(k) * a.ldq) : 0.0;
            a1v[kq] = rb < rend ? __ldcg(Qi + rb + static_cast<int64_t>(k) * a.ldq) : 0.0;
          }
#pragma unroll
          for (int kq = 0; kq < 8; ++kq)
#pragma unroll
            for (int n = 0; n < 4; ++n)
              dmma_16x8x4(ac[n], a0v[kq], a1v[kq], -W[(4 * kq + t) + (n * 8 + g) * kInvPitch]);
        }
      }
      double* Qj = Q + static_cast<int64_t>(32 * J) * a.ldq;
#pragma unroll
      for (int n = 0; n < 4; ++n)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int row = (q & 2) ? rb : ra, col = n * 8 + 2 * t + (q & 1);
          if (row < rend) Qj[row + static_cast<int64_t>(col) * a.ldq] = (32 * J + col < r) ? ac[n][q] : 0.0;
        }
      __syncwarp();
      __threadfence_block();
    }
  }
  FQ_TRACE(13);
}

}  // namespace

// Per item 2 l_p^2 (trailing buffers / inverse), plus a tail of PB x (l_p + 20)
// per item for the single-CTA kernels' panel when it does not fit in shared
// memory next to the inverse workspace (l_p > ~840).
constexpr int64_t kSmemCap = 227 * 1024;
bool panel_in_global(int64_t ellp) {
  const int64_t big = std::max<int64_t>(PB * (ellp + 20), kInvSmem);
  return big * 8 + 3 * ellp * 8 + 2 * ellp * 4 + 64 > kSmemCap ||
         big * 8 + 2 * 32 * kInvPitch * 8 + 64 > kSmemCap;
}
int64_t fcqr_xscratch_elems(int64_t ellp, int64_t batch) {
  const int64_t nbk = ellp / 32;
  return (nbk * (nbk + 1) / 2 + nbk) * kFqBlk * batch;
}
int64_t pchol_scratch_elems(int64_t ellp, int64_t batch) {
  return 2 * ellp * ellp * batch + (panel_in_global(ellp) ? batch * PB * (ellp + 20) : 0);
}

void launch_pchol(double* G, double* T, double* Rfull, double* scratch, int* rank, int* perm,
                  int64_t ell, int64_t ellp, double tau, bool pivot, int64_t batch,
                  cudaStream_t st, const CholOpts* opts) {
  if (batch <= 0) return;
  if (ellp % 32 != 0) throw CudaError("launch_pchol: ellp must be a multiple of 32");
  const int64_t pitch = ellp + 20;
  const int rpg = panel_in_global(ellp) ? 1 : 0;
  const int64_t big = rpg ? static_cast<int64_t>(kInvSmem) : std::max<int64_t>(PB * pitch, kInvSmem);
  // gchol for the plain factorizations; the gated / masked calls of the
  // ill-conditioned fallback (usually no item active) use the one-CTA-per-item
  // kernel: cooperative launches replayed from a CUDA graph cost ~1 ms each
  // even when every CTA exits at once (C2: 44.6 -> 24.3 ms per step).
  if (!pivot && (!opts || opts->lin)) {
    GcholArgs ga{G, T, Rfull, scratch, rank, perm, static_cast<int>(ell), static_cast<int>(ellp),
                 tau, batch, opts ? *opts : CholOpts{}};
    const int bytes = kGcDiagWarps * 2 * 32 * kInvPitch * 8;
    // per device: the smem opt-in is per context, the co-resident grid per SKU
    static std::atomic<int> grid_dev[kMaxDevices];
    int grid = grid_dev[current_device()].load(std::memory_order_acquire);
    if (grid == 0) {
      RSVD_CUDA(cudaFuncSetAttribute(gchol_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     bytes));
      int per_sm = 0;
      RSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gchol_kernel<0>, kGcThreads,
                                                              bytes));
      if (per_sm < 1) throw CudaError("gchol_kernel: does not fit on an SM");
      grid = per_sm * num_sms();
      grid_dev[current_device()].store(grid, std::memory_order_release);
    }
    // l_p <= 96 (single small matrices, narrow TEBD sectors): one CTA per
    // item, block barriers only (C1 Cholesky 0.60 -> 0.52 ms per call chain;
    // from l_p = 160 up the grid / cluster modes are as fast or faster).
    if (ceil_div(ellp, 32) <= 3) {
      static std::atomic<uint64_t> attr2{0};
      once_per_device(attr2, [&] {
        RSVD_CUDA(cudaFuncSetAttribute(gchol_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       bytes));
      });
      gchol_kernel<2><<<static_cast<unsigned>(batch), kGcThreads, bytes, st>>>(ga);
      RSVD_LAUNCH("gchol_kernel");
      return;
    }
    // Size the persistent grid to the work: the widest step has one warp task
    // per (item, upper 32 x 32 tile); a full-GPU grid for a small batch (a
    // chunk of the host pipeline) only spins in grid barriers while occupying
    // the SMs the other chunk's GEMMs could use.
    const int64_t nbk = ceil_div(ellp, 32);
    const int64_t want = ceil_div(batch * nbk * (nbk + 1) / 2, kGcWarps);
    int g = static_cast<int>(std::min<int64_t>(grid, std::max<int64_t>(want, 32)));
    // Small work: one cluster of 8-16 CTAs with cluster barriers.
    // 16-CTA (non-portable) clusters available on this device: 0 unknown, 1 no, 2 yes
    static std::atomic<int> clu_dev[kMaxDevices];
    if (want <= 16) {
      int clu_ok = clu_dev[current_device()].load(std::memory_order_acquire) - 1;
      if (clu_ok < 0) {
        clu_ok = 0;
        if (cudaFuncSetAttribute(gchol_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 bytes) == cudaSuccess &&
            cudaFuncSetAttribute(gchol_kernel<1>,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
          cudaLaunchConfig_t probe{};
          cudaLaunchAttribute pa[1];
          pa[0].id = cudaLaunchAttributeClusterDimension;
          pa[0].val.clusterDim.x = 16;
          pa[0].val.clusterDim.y = 1;
          pa[0].val.clusterDim.z = 1;
          probe.gridDim = dim3(16);
          probe.blockDim = dim3(kGcThreads);
          probe.dynamicSmemBytes = bytes;
          probe.attrs = pa;
          probe.numAttrs = 1;
          int ncl = 0;
          if (cudaOccupancyMaxActiveClusters(&ncl, gchol_kernel<1>, &probe) == cudaSuccess &&
              ncl >= 1)
            clu_ok = 1;
        }
        cudaGetLastError();
        clu_dev[current_device()].store(clu_ok + 1, std::memory_order_release);
      }
      if (clu_ok == 1) {
        const int S = static_cast<int>(std::max<int64_t>(8, std::min<int64_t>(16, want)));
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = static_cast<unsigned>(S);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(static_cast<unsigned>(S));
        cfg.blockDim = dim3(kGcThreads);
        cfg.dynamicSmemBytes = bytes;
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        RSVD_CUDA(cudaLaunchKernelEx(&cfg, gchol_kernel<1>, ga));
        RSVD_LAUNCH("gchol_kernel");
        return;
      }
    }
    void* args[] = {&ga};
    RSVD_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(gchol_kernel<0>), dim3(g),
                                          dim3(kGcThreads), args, bytes, st));
    RSVD_LAUNCH("gchol_kernel");
    return;
  }
  if (!pivot) {
    const CholOpts o = opts ? *opts : CholOpts{};
    const int64_t ub = big * 8 + 2 * 32 * kInvPitch * 8 + 64;
    RSVD_CUDA(cudaFuncSetAttribute(uchol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(ub)));
    uchol_kernel<<<static_cast<unsigned>(batch), kCholThreads, ub, st>>>(
        G, T, Rfull, scratch, rank, perm, static_cast<int>(ell), static_cast<int>(ellp), tau, o, rpg);
    RSVD_LAUNCH("uchol_kernel");
    return;
  }
  const int64_t bytes = big * 8 + 3 * ellp * 8 + 2 * ellp * 4 + 64;
  RSVD_CUDA(cudaFuncSetAttribute(pchol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
  pchol_kernel<<<static_cast<unsigned>(batch), kCholThreads, bytes, st>>>(
      G, T, Rfull, scratch, rank, perm, static_cast<int>(ell), static_cast<int>(ellp), tau,
      pivot ? (opts && opts->pairs ? 2 : 1) : 0, opts ? opts->mask : nullptr, rpg);
  RSVD_LAUNCH("pchol_kernel");
}


// Fused CholeskyQR pass (fcqr_kernel) for l_p <= 160; false when it does not
// apply (the caller runs the unfused Gram / gchol / apply sequence).
bool launch_fused_cqr(const double* Y, int64_t ldy, int64_t strideY, double* Q, int64_t ldq,
                      int64_t strideQ, double* G0, double* Rf, double* xscratch, int* rank,
                      int64_t rows, int64_t ell, int64_t ellp, double tau, int64_t batch,
                      cudaStream_t st, bool lin) {
  if (batch <= 0) return true;
  if (ellp % 32 != 0 || ellp > 160 || rows < 1 || rows > (1 << 30)) return false;
  const int64_t nbk = ellp / 32, nub = nbk * (nbk + 1) / 2;
  const int64_t gbytes = nub * kFqBlk * 8, dbytes = (nbk + 2) * kFqBlk * 8;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, current_device());
  const int64_t cap = std::max(0, optin - 256);  // room for the kernel's static shared memory
  // The Gram phase stages Y over the whole allocation (the G blocks are
  // written only after its last chunk): CR rows x l_p, double buffered.
  int cr = 64;
  while (cr > 16 && 2 * ellp * (cr + 4) * 8 > std::max<int64_t>(gbytes + dbytes, cap / 2)) cr -= 16;
  const int64_t bytes = std::max<int64_t>(gbytes + dbytes, 2 * ellp * (cr + 4) * 8);
  if (bytes > cap) return false;
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    RSVD_CUDA(cudaFuncSetAttribute(fcqr_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(cap)));
  });
  FcqrArgs fa{Y, ldy, strideY, Q, ldq, strideQ, G0, Rf, xscratch, rank, static_cast<int>(rows),
              static_cast<int>(ell), static_cast<int>(ellp), cr, tau, lin ? 1 : 0};
  // Few items: split each item's rows over a cluster (up to 8 CTAs, >= 64 rows each).
  int S = 1;
  while (xscratch && S < 8 && batch * S * 2 <= num_sms() && rows >= 64 * S * 2) S *= 2;
  if (S > 1) {
    static std::atomic<uint64_t> attr2{0};
    once_per_device(attr2, [&] {
      RSVD_CUDA(cudaFuncSetAttribute(fcqr_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(cap)));
    });
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(S);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(static_cast<unsigned>(batch * S));
    cfg.blockDim = dim3(kFqThreads);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    RSVD_CUDA(cudaLaunchKernelEx(&cfg, fcqr_kernel<true>, fa));
  } else {
    fcqr_kernel<false><<<static_cast<unsigned>(batch), kFqThreads, bytes, st>>>(fa);
  }
  RSVD_LAUNCH("fcqr_kernel");
  return true;
}

}  // namespace rsvd
