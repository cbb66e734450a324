// Table-driven kernels of the TEBD two-site bond update (SURVEY §8f row 3,
// rlftn::apply_gate, mps.cpp:111-323), so that a whole layer of disjoint
// bonds (mps.cpp:448-457) is assembled, measured and gauge-updated in a
// handful of launches instead of tens of small library calls per bond:
//
//   combine_blocks  out(i, j) = sum_t coef_t * rs_t[i] * cs_t[j] * src_t(i, j)
//                   -- the lambda-weighted site blocks alm / br (mps.cpp:130-137)
//                   written straight into the stacked operands of theta, the
//                   gate mixing of the (m1, m2) blocks (mps.cpp:205-222), the
//                   product form's x / y sums of Kronecker terms
//                   (mps.cpp:223-255) and the gauge update
//                   g1 = linv * U rows, g2 = Vt cols * rinv (mps.cpp:307-316);
//   grouped_gemm    C = A B for a table of independently shaped products --
//                   theta_mu = Astack_mu Bstack_mu (mps.cpp:164-204), the
//                   product form's core r * y (mps.cpp:265) and the lift
//                   qfac * left (mps.cpp:301-303);
//   block_sqnorms   ||theta'||^2 per bond, fixed summation order
//                   (mps.cpp:268).
// Every operand is addressed with explicit (row, column) element strides, so
// strided device views are consumed in place.  Scalars are double or
// double2 (interleaved complex, the SymmetricMPS<Complex> instantiation).
#include "common.cuh"

namespace rsvd {
namespace {

struct Real {
  using T = double;
  __device__ static T zero() { return 0.0; }
  __device__ static T load(const void* p, int64_t e) { return __ldg(static_cast<const double*>(p) + e); }
  __device__ static void store(void* p, int64_t e, T v) { static_cast<double*>(p)[e] = v; }
  __device__ static T scale(T v, double s) { return v * s; }
  __device__ static T fma_c(double cre, double, T v, T acc) { return ::fma(cre, v, acc); }
  __device__ static T fma(T a, T b, T acc) { return ::fma(a, b, acc); }
  __device__ static double sq(T v) { return v * v; }
};

struct Cplx {
  using T = double2;
  __device__ static T zero() { return make_double2(0.0, 0.0); }
  __device__ static T load(const void* p, int64_t e) { return __ldg(static_cast<const double2*>(p) + e); }
  __device__ static void store(void* p, int64_t e, T v) { static_cast<double2*>(p)[e] = v; }
  __device__ static T scale(T v, double s) { return make_double2(v.x * s, v.y * s); }
  __device__ static T fma_c(double cre, double cim, T v, T acc) {
    return make_double2(::fma(cre, v.x, ::fma(-cim, v.y, acc.x)), ::fma(cre, v.y, ::fma(cim, v.x, acc.y)));
  }
  __device__ static T fma(T a, T b, T acc) {
    return make_double2(::fma(a.x, b.x, ::fma(-a.y, b.y, acc.x)), ::fma(a.x, b.y, ::fma(a.y, b.x, acc.y)));
  }
  __device__ static double sq(T v) { return v.x * v.x + v.y * v.y; }
};

// One thread per output element; the job of element e is found by binary
// search in the prefix sums of the job sizes (column-major walk inside a job,
// so consecutive threads touch consecutive rows).
template <class O>
__global__ void combine_blocks_kernel(const rsvd_block_job* __restrict__ jobs,
                                      const rsvd_block_term* __restrict__ terms,
                                      const int64_t* __restrict__ start, int64_t njobs,
                                      int64_t total) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += stride) {
    int64_t lo = 0, hi = njobs - 1;
    while (lo < hi) {  // last job with start <= e
      const int64_t mid = (lo + hi + 1) >> 1;
      if (start[mid] <= e) lo = mid; else hi = mid - 1;
    }
    const rsvd_block_job& jb = jobs[lo];
    const int64_t local = e - start[lo];
    const int64_t i = local % jb.rows, j = local / jb.rows;
    typename O::T acc = O::zero();
    for (int64_t t = jb.term_begin; t < jb.term_begin + jb.term_count; ++t) {
      const rsvd_block_term& tm = terms[t];
      typename O::T v = O::load(tm.src, i * tm.rs + j * tm.cs);
      double s = 1.0;
      if (tm.row_scale) s *= tm.row_scale[i];
      if (tm.col_scale) s *= tm.col_scale[j];
      acc = O::fma_c(tm.coef_re * s, tm.coef_im * s, v, acc);
    }
    O::store(jb.dst, i * jb.rs + j * jb.cs, acc);
  }
}

// C = A B per job, one 64 x 64 output tile per CTA (tile table built on the
// host), 256 threads with a 4 x 4 register micro-tile, K staged through shared
// memory in slabs of 16.
constexpr int kGT = 64, kGK = 16;
template <class O>
__global__ void __launch_bounds__(256)
    grouped_gemm_kernel(const rsvd_gemm_job* __restrict__ jobs, const int4* __restrict__ tiles) {
  using T = typename O::T;
  __shared__ T As[kGK][kGT + 1];
  __shared__ T Bs[kGK][kGT + 1];
  const int4 tl = tiles[blockIdx.x];  // (job, tile row, tile col, -)
  const rsvd_gemm_job& jb = jobs[tl.x];
  const int64_t m0 = static_cast<int64_t>(tl.y) * kGT, n0 = static_cast<int64_t>(tl.z) * kGT;
  const int tid = threadIdx.x, tr = tid / 16, tc = tid % 16;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = O::zero();
  for (int64_t k0 = 0; k0 < jb.K; k0 += kGK) {
    for (int e = tid; e < kGK * kGT; e += 256) {
      const int kk = e / kGT, mm = e % kGT;  // A: consecutive threads -> consecutive rows
      const int64_t gi = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gi < jb.M && gk < jb.K) ? O::load(jb.A, gi * jb.a_rs + gk * jb.a_cs) : O::zero();
      const int nn = e / kGK, kb = e % kGK;  // B: consecutive threads -> consecutive k
      const int64_t gj = n0 + nn, gk2 = k0 + kb;
      Bs[kb][nn] = (gj < jb.N && gk2 < jb.K) ? O::load(jb.B, gk2 * jb.b_rs + gj * jb.b_cs) : O::zero();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGK; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[kk][tr + 16 * u];
        b[u] = Bs[kk][tc + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = O::fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t gi = m0 + tr + 16 * u, gj = n0 + tc + 16 * v;
      if (gi < jb.M && gj < jb.N) O::store(jb.C, gi * jb.c_rs + gj * jb.c_cs, acc[u][v]);
    }
}

// out[slot] = sum over the slot's blocks of |x|^2, one CTA per slot, blocks in
// table order, fixed-shape tree reduction (bitwise reproducible).
template <class O>
__global__ void __launch_bounds__(256)
    block_sqnorm_kernel(const rsvd_block_job* __restrict__ blocks, const int64_t* __restrict__ begin,
                        double* __restrict__ out) {
  __shared__ double red[256];
  const int64_t s = blockIdx.x;
  double acc = 0.0;
  for (int64_t b = begin[s]; b < begin[s + 1]; ++b) {
    const rsvd_block_job& jb = blocks[b];
    const int64_t n = jb.rows * jb.cols;
    for (int64_t e = threadIdx.x; e < n; e += 256) {
      const int64_t i = e % jb.rows, j = e / jb.rows;
      acc += O::sq(O::load(jb.dst, i * jb.rs + j * jb.cs));
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[s] = red[0];
}

}  // namespace

void launch_combine_blocks(bool cplx, const rsvd_block_job* jobs_dev, const rsvd_block_term* terms_dev,
                           const int64_t* start_dev, int64_t njobs, int64_t total, cudaStream_t st) {
  if (total <= 0 || njobs <= 0) return;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 16 * num_sms()));
  if (cplx)
    combine_blocks_kernel<Cplx><<<blocks, 256, 0, st>>>(jobs_dev, terms_dev, start_dev, njobs, total);
  else
    combine_blocks_kernel<Real><<<blocks, 256, 0, st>>>(jobs_dev, terms_dev, start_dev, njobs, total);
  RSVD_LAUNCH("combine_blocks_kernel");
}

void launch_grouped_gemm(bool cplx, const rsvd_gemm_job* jobs_dev, const int4* tiles_dev,
                         int64_t ntiles, cudaStream_t st) {
  if (ntiles <= 0) return;
  if (ntiles > 0x7fffffff) throw CudaError("grouped_gemm: too many tiles");
  if (cplx)
    grouped_gemm_kernel<Cplx><<<static_cast<unsigned>(ntiles), 256, 0, st>>>(jobs_dev, tiles_dev);
  else
    grouped_gemm_kernel<Real><<<static_cast<unsigned>(ntiles), 256, 0, st>>>(jobs_dev, tiles_dev);
  RSVD_LAUNCH("grouped_gemm_kernel");
}

int64_t grouped_gemm_tile(int64_t extent) { return ceil_div(extent, kGT); }

void launch_block_sqnorms(bool cplx, const rsvd_block_job* blocks_dev, const int64_t* begin_dev,
                          int64_t nslots, double* out_dev, cudaStream_t st) {
  if (nslots <= 0) return;
  if (cplx)
    block_sqnorm_kernel<Cplx><<<static_cast<unsigned>(nslots), 256, 0, st>>>(blocks_dev, begin_dev, out_dev);
  else
    block_sqnorm_kernel<Real><<<static_cast<unsigned>(nslots), 256, 0, st>>>(blocks_dev, begin_dev, out_dev);
  RSVD_LAUNCH("block_sqnorm_kernel");
}

}  // namespace rsvd
