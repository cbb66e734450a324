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
// Block-cyclic ordering: columns in blocks of 16, one sweep = a diagonal
// phase (each block pair (2k, 2k+1) rotates its intra pairs) plus nb - 1
// round-robin block-pair phases (every inter-block pair once).  A task =
// (item, block pair): G = X^T X of its 32 columns on DMMA, 15-16 rotation
// steps on G and a 32 x 32 V (dgesvj's threshold |g| <= sqrt(l) eps
// sqrt(alpha beta), exact 2 x 2 updates), then X <- X V and J <- J V on DMMA.
// An item stops after a sweep whose largest rotated ratio was below 1e-7
// (quadratic convergence leaves ~1e-14 behind: the sweep that only confirms
// convergence at the 1e-9 level is no longer run).
//
// Two kernels:
//   * jacobi_df_kernel  -- many tasks (batches: C2, C4, TEBD layers) and any
//     l: dataflow over (sweep, phase, item, pair) with per-item dependencies,
//     no grid barrier, no l-dependent shared memory;
//   * jacobi_clug_kernel -- few tasks (single matrices: C1, C3, C5): every
//     task is owned by a thread-block cluster whose CTAs split its rows.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include <cfloat>

#include "common.cuh"

namespace rsvd {
namespace {

// Sweep stop rule: an item is done after a sweep whose largest rotated
// g^2 / (alpha beta) stayed below (1e-7)^2.
__constant__ double c_stop_ratio2 = 1e-14;

// Round-robin pairing for `nn` (even) players at step s: slot 0 fixed, the
// others rotate.  Pair k couples slot k with slot nn-1-k.
__device__ __forceinline__ int rr_player(int slot, int s, int nn) {
  if (slot == 0) return 0;
  return 1 + (slot - 1 + s) % (nn - 1);
}

// tan of the Jacobi angle, t = sign(d) 2g / (|d| + sqrt(d^2 + 4g^2)), with
// a hardware reciprocal refined by two Newton steps instead of the IEEE
// division (~1e-15 relative instead of 0.5 ulp): t only decides how well the
// pair is annihilated, while c = (1 + t^2)^-1/2 and s = c t stay orthonormal
// to working precision whatever t is.  Saves ~60 cycles of the rotation
// chain per step.
__device__ __forceinline__ double jacobi_tan(double d, double g2) {
  const double den = fabs(d) + sqrt(fma(d, d, g2 * g2));
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
  r = r * fma(-den, r, 2.0);
  r = r * fma(-den, r, 2.0);
  return copysign(1.0, d) * g2 * r;
}

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// 16-byte global -> shared async copy; bytes < 16 zero-fills the rest.
__device__ __forceinline__ void cpa16(void* dst, const void* src, int bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cpa_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// Stage the 32 columns gcol(c) (rows [0, rows), zero past ell / for padding
// columns) of a column-major ellp x ellp matrix into S (column pitch PITCH).
template <int PITCH, class GC>
__device__ __forceinline__ void stage_pair(double* S, const double* G, int ell, int ellp, int rows,
                                           GC&& gcol, int tid, int nthreads) {
  const int half_rows = rows / 2;
  for (int e = tid; e < 32 * half_rows; e += nthreads) {
    const int c = e / half_rows, r = 2 * (e - c * half_rows);
    const int gc = gcol(c);
    int bytes = 0;
    const double* src = G;
    if (gc < ell && r < ell) {
      bytes = min(16, (ell - r) * 8);
      src = G + r + static_cast<int64_t>(gc) * ellp;
    }
    cpa16(S + c * PITCH + r, src, bytes);
  }
  cpa_wait_all();
}

// Row-split cluster variant (jacobi_clug_kernel) for few tasks: every
// (item, block pair) task is owned by a thread-block CLUSTER of S CTAs, CTA q
// holding a slice of the rows of the 32 columns and of J; each task's
// rotations are done on the block pair's 32 x 32 Gram: every CTA forms the Gram of its row slice on DMMA, the S
// partials are summed through DSMEM in rank order (bit-identical G in every
// CTA), the 16 steps run redundantly on G and V in each CTA, and each CTA
// applies X <- X V, J <- J V to its rows.  Two cluster barriers per task
// instead of one per rotation step.
template <int RL>
__global__ void __launch_bounds__(512, 1)
    jacobi_clug_kernel(double* __restrict__ H, double* __restrict__ J, int ell, int ellp, int nb,
                       int64_t batch, int max_sweeps, unsigned* __restrict__ flags,
                       int* __restrict__ sweeps_out) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int W = 16, NC = 32, VP = NC + 4, GP = NC + 1, PITCH = 32 * RL + 4, ROWS = 32 * RL;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_rot;
  __shared__ unsigned long long s_mx;
  double* Hs = sm;                 // NC x PITCH (local rows)
  double* Vs = Hs + NC * PITCH;    // NC x VP
  double* Gs = Vs + NC * VP;       // NC x GP: the summed Gram
  double* Gp = Gs + NC * GP;       // NC x GP: this CTA's partial Gram (read remotely)
  int* conv = reinterpret_cast<int*>(Gp + NC * GP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int S = static_cast<int>(cluster.num_blocks());
  const int q = static_cast<int>(cluster.block_rank());
  const int row0 = q * ROWS;
  const int64_t sq = static_cast<int64_t>(ellp) * ellp;
  const double tol2 = static_cast<double>(ell) * DBL_EPSILON * DBL_EPSILON;
  const int64_t nclu = gridDim.x / S;
  const int64_t clu = blockIdx.x / S;

  const int64_t gtid = blockIdx.x * static_cast<int64_t>(blockDim.x) + tid;
  const int64_t gstride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = gtid; e < sq * batch; e += gstride) {
    const int64_t rem = e % sq;
    J[e] = (rem % ellp == rem / ellp) ? 1.0 : 0.0;
  }
  unsigned long long* mxr = reinterpret_cast<unsigned long long*>(flags + ((3 * batch + 1) & ~int64_t(1)));
  for (int64_t e = gtid; e < 3 * batch; e += gstride) {
    flags[e] = 0u;
    mxr[e] = 0ull;
  }
  for (int64_t i = tid; i < batch; i += blockDim.x) conv[i] = 0;
  grid.sync();

  const int half = nb / 2;
  const int64_t tasks = batch * half;
  // local slice [row0, row0 + ROWS) of the ellp rows, clipped to ell
  const int lrows = max(0, min(ROWS, ell - row0));
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
          const int p = rr_player(k, phase - 1, nb), qq = rr_player(nb - 1 - k, phase - 1, nb);
          bp = min(p, qq), bq = max(p, qq);
        }
        // a block-pair task whose second block is all padding has no pair
        // that can rotate (and intra-block pairs belong to the diagonal phase)
        if (bp * W >= ell || (!diag && bq * W >= ell)) continue;
        double* Hg = H + item * sq;
        double* Jg = J + item * sq;
        auto gcol = [&](int c) { return c < W ? bp * W + c : bq * W + (c - W); };
        // local rows: global row = row0 + r; stage_pair works on rows [0, ROWS)
        // of a shifted matrix view whose "ell" is the local row count.
        const double* Hl = Hg + row0;
        {
          const int half_rows = ROWS / 2;
          for (int e = tid; e < 32 * half_rows; e += blockDim.x) {
            const int c = e / half_rows, r = 2 * (e - c * half_rows);
            const int gc = gcol(c);
            int bytes = 0;
            const double* src = Hg;
            if (gc < ell && r < lrows) {
              bytes = min(16, (lrows - r) * 8);
              src = Hl + r + static_cast<int64_t>(gc) * ellp;
            }
            cpa16(Hs + c * PITCH + r, src, bytes);
          }
          cpa_wait_all();
        }
        for (int e = tid; e < NC * VP; e += blockDim.x) {
          const int c = e / VP, r = e - c * VP;
          Vs[e] = (r == c) ? 1.0 : 0.0;
        }
        if (tid == 0) {
          s_rot = 0;
          s_mx = 0ull;
        }
        __syncthreads();
        if (warp < 8) {  // partial Gram of the local rows (DMMA)
          const int tm = warp >> 2, tn = warp & 3;
          double acc[4] = {0.0, 0.0, 0.0, 0.0}, acc2[4] = {0.0, 0.0, 0.0, 0.0};
          const double* a0p = Hs + (16 * tm + g) * PITCH;
          const double* a1p = Hs + (16 * tm + g + 8) * PITCH;
          const double* b0p = Hs + (8 * tn + g) * PITCH;
#pragma unroll 4
          for (int k0 = 0; k0 < ROWS; k0 += 8) {  // two accumulators: half the DMMA chain
            dmma_16x8x4(acc, a0p[k0 + t4], a1p[k0 + t4], b0p[k0 + t4]);
            dmma_16x8x4(acc2, a0p[k0 + 4 + t4], a1p[k0 + 4 + t4], b0p[k0 + 4 + t4]);
          }
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) acc[qq] += acc2[qq];
          const int r0 = 16 * tm + g, c0 = 8 * tn + 2 * t4;
          Gp[r0 + c0 * GP] = acc[0];
          Gp[r0 + (c0 + 1) * GP] = acc[1];
          Gp[r0 + 8 + c0 * GP] = acc[2];
          Gp[r0 + 8 + (c0 + 1) * GP] = acc[3];
        }
        cluster.sync();
        for (int e = tid; e < NC * NC; e += blockDim.x) {
          const int c = e / NC, r = e - c * NC;
          double v = 0.0;
          for (int rr = 0; rr < S; ++rr) v += *cluster.map_shared_rank(&Gp[r + c * GP], rr);
          Gs[r + c * GP] = v;
        }
        cluster.sync();  // every CTA has read every partial
        int rotated = 0, big = 0;
        const int steps = diag ? 15 : 16;
        for (int s2 = 0; s2 < steps; ++s2) {
          int i, jx;
          if (diag) {
            const int blk = warp >> 3, pi = warp & 7;
            const int a0 = rr_player(pi, s2, 16), b0 = rr_player(15 - pi, s2, 16);
            i = blk * 16 + min(a0, b0);
            jx = blk * 16 + max(a0, b0);
          } else {
            i = warp;
            jx = 16 + ((warp + s2) & 15);
          }
          const double al = Gs[i + i * GP], be = Gs[jx + jx * GP], ga = Gs[i + jx * GP];
          const double gg = ga * ga, ab = al * be;
          const bool rot = al > 0.0 && be > 0.0 && gg > tol2 * ab;
          double c = 1.0, sn = 0.0, tt = 0.0;
          if (rot) {
            big |= gg >= c_stop_ratio2 * ab;
            const double d = be - al, g2 = 2.0 * ga;
            const double mag = fmax(fabs(d), fabs(g2));
            if (mag > 1e-140 && mag < 1e140) {
              tt = jacobi_tan(d, g2);
            } else {
              const double zeta = d / g2;
              tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
            }
            c = rsqrt(fma(tt, tt, 1.0));
            sn = c * tt;
            rotated = 1;
            const double gi = Gs[lane + i * GP], gj = Gs[lane + jx * GP];
            Gs[lane + i * GP] = c * gi - sn * gj;
            Gs[lane + jx * GP] = sn * gi + c * gj;
            const double vi = Vs[i * VP + lane], vj = Vs[jx * VP + lane];
            Vs[i * VP + lane] = c * vi - sn * vj;
            Vs[jx * VP + lane] = sn * vi + c * vj;
          }
          __syncthreads();
          if (rot) {
            const double gi = Gs[i + lane * GP], gj = Gs[jx + lane * GP];
            Gs[i + lane * GP] = c * gi - sn * gj;
            Gs[jx + lane * GP] = sn * gi + c * gj;
            __syncwarp();
            if (lane == 0) {
              Gs[i + i * GP] = al - tt * ga;
              Gs[jx + jx * GP] = be + tt * ga;
              Gs[i + jx * GP] = 0.0;
              Gs[jx + i * GP] = 0.0;
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
          constexpr int slabs = ROWS / 16;
          for (int pass = 0; pass < 2; ++pass) {  // 0: X <- X V, 1: J <- J V
            if (pass == 1) {
              __syncthreads();
              const int half_rows = ROWS / 2;
              const double* Jl = Jg + row0;
              for (int e = tid; e < 32 * half_rows; e += blockDim.x) {
                const int c = e / half_rows, r = 2 * (e - c * half_rows);
                const int gc = gcol(c);
                int bytes = 0;
                const double* src = Jg;
                if (gc < ell && r < lrows) {
                  bytes = min(16, (lrows - r) * 8);
                  src = Jl + r + static_cast<int64_t>(gc) * ellp;
                }
                cpa16(Hs + c * PITCH + r, src, bytes);
              }
              cpa_wait_all();
              __syncthreads();
            }
            double* dst = pass == 0 ? Hg : Jg;
            for (int sl = warp; sl < slabs; sl += W) {
              const int r0 = sl * 16;
              double acc[NC / 8][4];
#pragma unroll
              for (int n = 0; n < NC / 8; ++n)
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) acc[n][qq] = 0.0;
#pragma unroll
              for (int kq = 0; kq < 8; ++kq) {
                const int kc = kq * 4 + t4;
                const double a0 = Hs[kc * PITCH + r0 + g], a1 = Hs[kc * PITCH + r0 + g + 8];
#pragma unroll
                for (int n = 0; n < NC / 8; ++n)
                  dmma_16x8x4(acc[n], a0, a1, Vs[(n * 8 + g) * VP + kc]);
              }
#pragma unroll
              for (int n = 0; n < NC / 8; ++n)
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                  const int r = r0 + g + ((qq & 2) ? 8 : 0);
                  const int cc = n * 8 + 2 * t4 + (qq & 1);
                  const int gc = gcol(cc);
                  if (r < lrows && gc < ell) dst[row0 + r + static_cast<int64_t>(gc) * ellp] = acc[n][qq];
                }
            }
          }
        }
        __syncthreads();
        if (tid == 0 && q == 0 && s_rot) {
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

template <int RL>
bool launch_clu_t(double* H, double* J, int64_t ell, int64_t ellp, int max_sweeps, int* sweeps,
                  unsigned* flags, int64_t batch, int S, cudaStream_t st) {
  const size_t bytes = (static_cast<size_t>(32) * (32 * RL + 4) + 32 * 36 + 2 * 32 * 33) * sizeof(double) +
                       batch * sizeof(int) + 16;
  auto kern = jacobi_clug_kernel<RL>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(bytes)) != cudaSuccess ||
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  int nb = static_cast<int>((ell + 15) / 16);
  nb += nb & 1;
  const int64_t tasks = batch * (nb / 2);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(S);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cfg.gridDim = dim3(static_cast<unsigned>(S));
  int max_clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1) {
    cudaGetLastError();
    return false;
  }
  const int64_t ncl = std::max<int64_t>(1, std::min<int64_t>(tasks, max_clusters));
  cfg.gridDim = dim3(static_cast<unsigned>(ncl * S));
  int ell_i = static_cast<int>(ell), ellp_i = static_cast<int>(ellp);
  if (cudaLaunchKernelEx(&cfg, kern, H, J, ell_i, ellp_i, nb, batch, max_sweeps, flags, sweeps) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  RSVD_LAUNCH("jacobi_clug_kernel");
  return true;
}

// Cluster size and rows per lane for the row-split kernel (S <= 6 and the
// clusters of all tasks co-resident), rounded so the S slices cover l.
bool launch_clu(double* H, double* J, int64_t ell, int64_t ellp, int max_sweeps, int* sweeps,
                unsigned* flags, int64_t batch, cudaStream_t st) {
  int nb = static_cast<int>((ell + 15) / 16);
  nb += nb & 1;
  const int64_t tasks = batch * (nb / 2);
  const int R = static_cast<int>((ell + 31) / 32);
  // Per step the cluster barrier competes with the per-CTA rotation work:
  // 5-6 CTAs per task measured best (C3: S 3/5/9 -> 4.6/4.4/4.8 ms, C5:
  // S 3/5/9 -> 11.1/9.7/18.7 ms -- at 9 the clusters no longer fit at once).
  int smax = static_cast<int>(std::min<int64_t>(6, num_sms() / std::max<int64_t>(tasks, 1)));
  if (smax < 2) return false;
  int rl = (R + smax - 1) / smax;
  static const int kRL[] = {1, 2, 3, 4, 6, 8, 12};  // 8, 12: wide factors (tsvd up to l = 1600)
  int pick = 0;
  while (pick < 6 && kRL[pick] < rl) ++pick;
  if (kRL[pick] < rl) return false;
  rl = kRL[pick];
  const int S = (R + rl - 1) / rl;
  if (S < 2) return false;
  switch (rl) {
    case 1: return launch_clu_t<1>(H, J, ell, ellp, max_sweeps, sweeps, flags, batch, S, st);
    case 2: return launch_clu_t<2>(H, J, ell, ellp, max_sweeps, sweeps, flags, batch, S, st);
    case 3: return launch_clu_t<3>(H, J, ell, ellp, max_sweeps, sweeps, flags, batch, S, st);
    case 4: return launch_clu_t<4>(H, J, ell, ellp, max_sweeps, sweeps, flags, batch, S, st);
    case 6: return launch_clu_t<6>(H, J, ell, ellp, max_sweeps, sweeps, flags, batch, S, st);
    case 8: return launch_clu_t<8>(H, J, ell, ellp, max_sweeps, sweeps, flags, batch, S, st);
    default: return launch_clu_t<12>(H, J, ell, ellp, max_sweeps, sweeps, flags, batch, S, st);
  }
}


// ---------------------------------------------------------------------------
// Dataflow row-streamed Gram-accelerated block-cyclic Jacobi (jacobi_df_kernel).
// Same sweep order, rotation formula, thresholds and convergence rule as
// jacobi_gram_kernel, but
//   * no grid-wide barrier: tasks (sweep, phase, item, block pair) are pulled
//     in that order from one atomic counter by a persistent grid, and a
//     block-pair task waits only for the two previous-phase tasks of its OWN
//     item that held its blocks (per item-block phase counters), a phase-0 task
//     for the item's previous sweep (release/acquire) -- items, and the pairs
//     of a phase, never wait for each other, so uneven task times and
//     converged items cost nothing;
//   * the convergence decision for sweep s of an item is taken by its phase-0
//     tasks of sweep s + 1 from that sweep's final flags;
//   * nothing scales with l in shared memory: G = X^T X of the task's 32
//     columns is accumulated over RC-row chunks staged by cp.async (double
//     buffer), the 16 rotation steps run on G / V in shared memory (8 warps,
//     two column pairs each per step), and X <- X V, J <- J V read their
//     16-row slabs from global memory (L2) into DMMA fragments and write the
//     products back in place -- any l (tsvd of 4096^2 and beyond).
// Dependencies point only to earlier tasks, which were pulled by running
// CTAs, so the launch needs no co-residency guarantee (plain launch, graph
// friendly).  Workspace (jacobi_flag_elems): per item 3 rotating "rotated"
// flags, 3 rotating "big rotation" flags, a completion counter and a
// converged flag; then the task counter and the converged-item count.
#ifdef RSVD_JDF_TRACE
// Phase sums of CTA 0 (ns): pull + dependency wait, Gram, rotation steps,
// X/J update, bookkeeping; task count (tools/probe/jdf_trace.cu).
__device__ unsigned long long g_jdf_trace[8];
__device__ __forceinline__ unsigned long long jdf_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define JDF_MARK(slot)                                         \
  do {                                                         \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                 \
      const unsigned long long n_ = jdf_now();                 \
      jdf_acc[slot] += n_ - jdf_last;                          \
      jdf_last = n_;                                           \
    }                                                          \
  } while (0)
#else
#define JDF_MARK(slot) do {} while (0)
#endif

template <int RC, int MINB>
__global__ void __launch_bounds__(256, MINB)
    jacobi_df_kernel(double* __restrict__ H, double* __restrict__ J, int ell, int ellp, int nb,
                     int64_t batch, int max_sweeps, unsigned* __restrict__ flags,
                     int* __restrict__ sweeps_out) {
  constexpr int W = 16, NC = 32, VP = NC + 4, GP = NC + 1, NW = 8;
  constexpr int PITCH = RC + 4;  // = 4 mod 16 doubles: conflict-free DMMA fragment loads
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_rot;
  __shared__ unsigned long long s_mx;
  __shared__ long long s_task;
  __shared__ int s_work;
  const int nch = (ell + RC - 1) / RC;
  double* Xs = sm;                                   // (1 or 2) x (NC x PITCH) row chunks
  double* Vs = sm + (nch > 1 ? 2 : 1) * NC * PITCH;  // NC x VP, column-major V[c*VP + k]
  double* Gs = Vs + NC * VP;                         // NC x GP, G[row + col*GP]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t sq = static_cast<int64_t>(ellp) * ellp;
  const double tol2 = static_cast<double>(ell) * DBL_EPSILON * DBL_EPSILON;

  const int64_t fpad = (3 * batch + 1) & ~int64_t(1);
  unsigned* fl3 = flags;
  unsigned long long* mx3 = reinterpret_cast<unsigned long long*>(flags + fpad);
  unsigned* cnt = flags + fpad + 6 * batch;
  unsigned* convg = cnt + batch;
  unsigned long long* next = reinterpret_cast<unsigned long long*>(convg + batch);
  unsigned* nconv = reinterpret_cast<unsigned*>(next + 1);
  unsigned* bdone = nconv + 2;  // [item][block]: phases the block has completed

  const int half = nb / 2;
  const int64_t per_phase = batch * half;
  const int64_t total = static_cast<int64_t>(max_sweeps) * nb * per_phase;
  const int slabs = (ell + 15) / 16;
#ifdef RSVD_JDF_TRACE
  unsigned long long jdf_acc[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long jdf_last = jdf_now();
#endif
  for (;;) {
    if (tid == 0) {
      long long t = -1;
      if (*reinterpret_cast<volatile unsigned*>(nconv) < batch) {
        t = static_cast<long long>(atomicAdd(next, 1ull));
        if (t >= total) t = -1;
      }
      s_task = t;
    }
    __syncthreads();
    const long long t = s_task;
    if (t < 0) break;
    const int sweep = static_cast<int>(t / (nb * per_phase));
    const int64_t rem = t - static_cast<int64_t>(sweep) * nb * per_phase;
    const int phase = static_cast<int>(rem / per_phase);
    const int64_t r2 = rem - phase * per_phase;
    const int64_t item = r2 / half;
    const int k = static_cast<int>(r2 - item * half);
    const bool diag = phase == 0;
    int bp, bq;
    if (diag) {
      bp = 2 * k, bq = 2 * k + 1;
    } else {
      const int p = rr_player(k, phase - 1, nb), q = rr_player(nb - 1 - k, phase - 1, nb);
      bp = min(p, q), bq = max(p, q);
    }
    const unsigned gph = static_cast<unsigned>(static_cast<int64_t>(sweep) * nb + phase);
    unsigned* bd = bdone + item * nb;
    if (tid == 0) {
      // 1: do the task; 0: count it without work; -1: item converged, skip
      int work = 1;
      volatile unsigned* vc = convg + item;
      if (diag) {
        // the item's whole previous sweep (its flags decide convergence)
        const unsigned need = static_cast<unsigned>(static_cast<int64_t>(sweep) * nb * half);
        while (ld_acquire(cnt + item) < need && *vc == 0u) __nanosleep(100);
      } else {
        // only the two tasks of the previous phase that held blocks bp, bq
        while ((ld_acquire(bd + bp) < gph || ld_acquire(bd + bq) < gph) && *vc == 0u) __nanosleep(100);
      }
      if (*vc != 0u) {
        work = -1;
      } else if (diag && sweep > 0) {
        const int slot = (sweep - 1) % 3;
        if (__ldcg(fl3 + slot * batch + item) == 0u || __ldcg(mx3 + slot * batch + item) == 0ull) {
          work = -1;
          // every phase-0 task of this sweep reaches the same verdict; the
          // first one to flag the item records it
          if (atomicCAS(convg + item, 0u, 1u) == 0u) {
            sweeps_out[item] = sweep;
            atomicAdd(nconv, 1u);
          }
        }
      }
      if (work == 1 && diag && k == 0) {  // this sweep's successor slot starts clean
        const int slot = (sweep + 1) % 3;
        fl3[slot * batch + item] = 0u;
        mx3[slot * batch + item] = 0ull;
      }
      // a block-pair task whose second block is all padding has no pair that
      // can rotate (intra-block pairs belong to the diagonal phase)
      if (work == 1 && (bp * W >= ell || (!diag && bq * W >= ell))) work = 0;
      s_work = work;
      s_rot = 0;
      s_mx = 0ull;
    }
    __syncthreads();
    JDF_MARK(0);
    const int work = s_work;
    if (work == 1) {
#ifdef RSVD_JDF_TRACE
      if (blockIdx.x == 0 && threadIdx.x == 0) jdf_acc[5] += 1;
#endif
      double* Hg = H + item * sq;
      double* Jg = J + item * sq;
      auto gcol = [&](int c) { return c < W ? bp * W + c : bq * W + (c - W); };
      auto stage = [&](int c, int buf) {
        const int r0 = c * RC;
        double* dst = Xs + buf * NC * PITCH;
        for (int e = tid; e < NC * (RC / 2); e += NW * 32) {
          const int cc = e / (RC / 2), r = 2 * (e - cc * (RC / 2));
          const int gc = gcol(cc), gr = r0 + r;
          int bytes = 0;
          const double* src = Hg;
          if (gc < ell && gr < ell) {
            bytes = min(16, (ell - gr) * 8);
            src = Hg + gr + static_cast<int64_t>(gc) * ellp;
          }
          cpa16(dst + cc * PITCH + r, src, bytes);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      };
      for (int e = tid; e < NC * VP; e += NW * 32) {
        const int c = e / VP, r = e - c * VP;
        Vs[e] = (r == c) ? 1.0 : 0.0;
      }
      // ---- G = X^T X over row chunks (cp.async double buffer, DMMA) ----
      const int tm = warp >> 2, tn = warp & 3;
      // two accumulators (even / odd k-steps): half the dependent DMMA chain
      double acc[4] = {0.0, 0.0, 0.0, 0.0}, acc2[4] = {0.0, 0.0, 0.0, 0.0};
      stage(0, 0);
      for (int c = 0; c < nch; ++c) {
        if (c + 1 < nch) {
          stage(c + 1, (c + 1) & 1);
          asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const double* Xb = Xs + (c & 1) * NC * PITCH;
        const double* a0p = Xb + (16 * tm + g) * PITCH;
        const double* a1p = Xb + (16 * tm + g + 8) * PITCH;
        const double* b0p = Xb + (8 * tn + g) * PITCH;
#pragma unroll 4
        for (int k0 = 0; k0 < RC; k0 += 8) {
          dmma_16x8x4(acc, a0p[k0 + t4], a1p[k0 + t4], b0p[k0 + t4]);
          dmma_16x8x4(acc2, a0p[k0 + 4 + t4], a1p[k0 + 4 + t4], b0p[k0 + 4 + t4]);
        }
        __syncthreads();  // buffer c & 1 is restaged at c + 2
      }
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) acc[qq] += acc2[qq];
      {
        const int r0 = 16 * tm + g, c0 = 8 * tn + 2 * t4;
        Gs[r0 + c0 * GP] = acc[0];
        Gs[r0 + (c0 + 1) * GP] = acc[1];
        Gs[r0 + 8 + c0 * GP] = acc[2];
        Gs[r0 + 8 + (c0 + 1) * GP] = acc[3];
      }
      __syncthreads();
      JDF_MARK(1);
      // ---- rotation steps on G and V ----
      // A step's 16 disjoint pairs act on G as G <- R^T G R with R a
      // permuted direct sum of 2 x 2 rotations, so every 2 x 2 block
      // (pair p rows, pair q cols) transforms independently:
      // G_pq <- R_p^T G_pq R_q.  Phase A: thread p < 16 derives pair p's
      // rotation from the current G; phase B: one thread per upper block
      // (p <= q, mirrored) and two V rows per thread apply them.
      double* Rc = Gs + NC * GP;  // c, s, t per pair; flag per pair after
      int* Rf = reinterpret_cast<int*>(Rc + 3 * 16);
      int rotated = 0, big = 0;
      const int steps = diag ? 15 : 16;
      auto pair_of = [&](int pr, int s2, int& i, int& jx) {
        if (diag) {
          const int blk = pr >> 3, pk = pr & 7;
          const int a0 = rr_player(pk, s2, 16), b0 = rr_player(15 - pk, s2, 16);
          i = blk * 16 + min(a0, b0);
          jx = blk * 16 + max(a0, b0);
        } else {
          i = pr;
          jx = 16 + ((pr + s2) & 15);
        }
      };
      const int bpp = tid >> 4, bqq = tid & 15;  // phase-B block of this thread
      const int vp = tid >> 4, vr = (tid & 15) * 2;  // phase-B V rows of this thread
      for (int s2 = 0; s2 < steps; ++s2) {
        if (tid < 16) {
          int i, jx;
          pair_of(tid, s2, i, jx);
          const double al = Gs[i + i * GP], be = Gs[jx + jx * GP], ga = Gs[i + jx * GP];
          const double gg = ga * ga, ab = al * be;
          const bool rot = al > 0.0 && be > 0.0 && gg > tol2 * ab;
          double c = 1.0, sn = 0.0, tt = 0.0;
          if (rot) {
            big |= gg >= c_stop_ratio2 * ab;
            const double d = be - al, g2 = 2.0 * ga;
            const double mag = fmax(fabs(d), fabs(g2));
            if (mag > 1e-140 && mag < 1e140) {
              tt = jacobi_tan(d, g2);
            } else {
              const double zeta = d / g2;
              tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
            }
            c = rsqrt(fma(tt, tt, 1.0));
            sn = c * tt;
            rotated = 1;
          }
          Rc[tid] = c;
          Rc[16 + tid] = sn;
          Rc[32 + tid] = tt;
          Rf[tid] = rot;
        }
        __syncthreads();
        if (bpp <= bqq) {
          int ip, jp, iq, jq;
          pair_of(bpp, s2, ip, jp);
          pair_of(bqq, s2, iq, jq);
          if (bpp == bqq) {
            if (Rf[bpp]) {
              const double ga = Gs[ip + jp * GP], tt = Rc[32 + bpp];
              Gs[ip + ip * GP] -= tt * ga;
              Gs[jp + jp * GP] += tt * ga;
              Gs[ip + jp * GP] = 0.0;
              Gs[jp + ip * GP] = 0.0;
            }
          } else if (Rf[bpp] | Rf[bqq]) {
            const double cp = Rc[bpp], sp = Rc[16 + bpp], cq = Rc[bqq], sq2 = Rc[16 + bqq];
            const double a = Gs[ip + iq * GP], b = Gs[ip + jq * GP];
            const double c0 = Gs[jp + iq * GP], d = Gs[jp + jq * GP];
            // right: columns (iq, jq) by R_q; left: rows (ip, jp) by R_p
            const double a1 = cq * a - sq2 * b, b1 = sq2 * a + cq * b;
            const double c1 = cq * c0 - sq2 * d, d1 = sq2 * c0 + cq * d;
            const double a2 = cp * a1 - sp * c1, c2 = sp * a1 + cp * c1;
            const double b2 = cp * b1 - sp * d1, d2 = sp * b1 + cp * d1;
            Gs[ip + iq * GP] = a2;
            Gs[ip + jq * GP] = b2;
            Gs[jp + iq * GP] = c2;
            Gs[jp + jq * GP] = d2;
            Gs[iq + ip * GP] = a2;
            Gs[jq + ip * GP] = b2;
            Gs[iq + jp * GP] = c2;
            Gs[jq + jp * GP] = d2;
          }
        }
        if (Rf[vp]) {
          int i, jx;
          pair_of(vp, s2, i, jx);
          const double c = Rc[vp], sn = Rc[16 + vp];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const double vi = Vs[i * VP + vr + u], vj = Vs[jx * VP + vr + u];
            Vs[i * VP + vr + u] = c * vi - sn * vj;
            Vs[jx * VP + vr + u] = sn * vi + c * vj;
          }
        }
        __syncthreads();
      }
      if (rotated) {
        atomicOr(&s_rot, 1);
        if (big) atomicMax(&s_mx, 1ull);
      }
      __syncthreads();
      JDF_MARK(2);
      if (s_rot) {
        // ---- X <- X V and J <- J V, in place, 16-row slab per warp ----
        for (int job = warp; job < 2 * slabs; job += NW) {
          double* M = job < slabs ? Hg : Jg;
          const int r0 = (job < slabs ? job : job - slabs) * 16;
          const int ra = r0 + g, rb = r0 + g + 8;
          double accv[NC / 8][4];
#pragma unroll
          for (int n = 0; n < NC / 8; ++n)
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) accv[n][qq] = 0.0;
#pragma unroll
          for (int kq = 0; kq < 8; ++kq) {
            const int kc = kq * 4 + t4;
            const int gc = gcol(kc);
            const double* col = M + static_cast<int64_t>(gc) * ellp;
            const bool okc = gc < ell;
            const double a0 = (okc && ra < ell) ? __ldcg(col + ra) : 0.0;
            const double a1 = (okc && rb < ell) ? __ldcg(col + rb) : 0.0;
#pragma unroll
            for (int n = 0; n < NC / 8; ++n)
              dmma_16x8x4(accv[n], a0, a1, Vs[(n * 8 + g) * VP + kc]);
          }
#pragma unroll
          for (int n = 0; n < NC / 8; ++n)
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              const int r = (qq & 2) ? rb : ra;
              const int gc = gcol(n * 8 + 2 * t4 + (qq & 1));
              if (r < ell && gc < ell) __stcg(M + r + static_cast<int64_t>(gc) * ellp, accv[n][qq]);
            }
        }
      }
      __syncthreads();
      JDF_MARK(3);
      if (tid == 0 && s_rot) {
        const int slot = sweep % 3;
        atomicOr(fl3 + slot * batch + item, 1u);
        atomicMax(mx3 + slot * batch + item, s_mx);
      }
    }
    if (tid == 0 && work >= 0) {
      __threadfence();
      atomicMax(bd + bp, gph + 1);
      atomicMax(bd + bq, gph + 1);
      atomicAdd(cnt + item, 1u);
    }
    JDF_MARK(4);
  }
#ifdef RSVD_JDF_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int i = 0; i < 6; ++i) g_jdf_trace[i] = jdf_acc[i];
#endif
}

// J = I per item, sweeps = max_sweeps (overwritten on convergence), flags,
// counters and the task queue zeroed.
__global__ void jacobi_df_init_kernel(double* __restrict__ J, int ellp, int64_t batch,
                                      int max_sweeps, unsigned* __restrict__ flags,
                                      int64_t nflags, int* __restrict__ sweeps_out) {
  const int64_t sq = static_cast<int64_t>(ellp) * ellp;
  const int64_t gtid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t gstride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = gtid; e < sq * batch; e += gstride) {
    const int64_t rem = e % sq;
    J[e] = (rem % ellp == rem / ellp) ? 1.0 : 0.0;
  }
  for (int64_t e = gtid; e < nflags; e += gstride) flags[e] = 0u;
  for (int64_t e = gtid; e < batch; e += gstride) sweeps_out[e] = max_sweeps;
}

template <int RC, int MINB>
void launch_df_t(double* H, double* J, int64_t ell, int64_t ellp, int max_sweeps, int* sweeps,
                 unsigned* flags, int64_t batch, cudaStream_t st) {
  const int nbuf = ell > RC ? 2 : 1;
  const size_t bytes = (static_cast<size_t>(nbuf * 32) * (RC + 4) + 32 * 36 + 32 * 33 + 3 * 16 + 8) *
                       sizeof(double);
  auto kern = jacobi_df_kernel<RC, MINB>;
  RSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
  int per_sm = 0;
  RSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, bytes));
  if (per_sm < 1) throw CudaError("jacobi_df_kernel: does not fit on an SM");
  int nb = static_cast<int>((ell + 15) / 16);
  nb += nb & 1;
  const int64_t per_phase = batch * (nb / 2);
  // One CTA per task of a phase at most: extra CTAs would only spin on the
  // next phase's dependencies (C4: 5.2 -> 6.1 ms with twice the grid).
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(per_phase, per_sm * num_sms())));
  const int64_t nflags = jacobi_flag_elems(batch, ellp);
  const int64_t init_work = std::max<int64_t>(ellp * ellp * batch, nflags);
  jacobi_df_init_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(init_work, 256), 8 * num_sms())),
                          256, 0, st>>>(J, static_cast<int>(ellp), batch, max_sweeps, flags, nflags,
                                        sweeps);
  RSVD_LAUNCH("jacobi_df_init_kernel");
  kern<<<grid, 256, bytes, st>>>(H, J, static_cast<int>(ell), static_cast<int>(ellp), nb, batch,
                                 max_sweeps, flags, sweeps);
  RSVD_LAUNCH("jacobi_df_kernel");
}

}  // namespace

// Per item: 3 rotating "rotated" flags, then (8-byte aligned) 3 rotating
// "a rotation with g^2 >= c_stop_ratio2 alpha beta" flags.

int64_t jacobi_flag_elems(int64_t batch, int64_t ellp) {
  // + per-item completion counter and converged flag, task counter (8 B) and
  // converged-item count for jacobi_df_kernel, then its per (item, 16-column
  // block) phase counters
  const int64_t nbk = (ellp + 15) / 16 + 2;
  return ((3 * batch + 1) & ~int64_t(1)) + 6 * batch + 2 * batch + 4 + batch * nbk;
}

void launch_jacobi(double* H, double* J, int64_t ell, int64_t ellp, int max_sweeps, int* sweeps,
                   unsigned* flags, int64_t batch, cudaStream_t st) {
  int nbt = static_cast<int>((ell + 15) / 16);
  nbt += nbt & 1;
  // Fewer tasks than SMs / 4 (single matrices): split every task's rows over
  // a cluster; with more tasks the dataflow kernel keeps all SMs busy.
  if (batch * (nbt / 2) * 4 <= num_sms() &&
      launch_clu(H, J, ell, ellp, max_sweeps, sweeps, flags, batch, st))
    return;
  if (ell <= 144 && ell > 64) return launch_df_t<144, 4>(H, J, ell, ellp, max_sweeps, sweeps, flags, batch, st);
  // Wider factors: 96-row chunks (C4's 276 rows in 3 chunks: 5.19 -> 5.00 ms).
  launch_df_t<96, 3>(H, J, ell, ellp, max_sweeps, sweeps, flags, batch, st);
}

}  // namespace rsvd
