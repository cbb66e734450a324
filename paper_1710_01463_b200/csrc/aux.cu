// Small glue kernels of the RSVD pipeline: basis completion, transposes,
// spectrum finalisation (numerical rank + truncation + discarded weight) and
// the residual reduction used by reconstruction_error.
#include <cfloat>

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

// Completion of a rank-deficient basis: columns [rank, ell) of Q are replaced
// by independent Gaussian columns (scaled to unit expected norm) drawn from
// the item's seed split by `tag`; the following CholeskyQR pass
// orthonormalises them against the retained span.  The reference's Householder
// Q completes such bases "arbitrarily" (lapack.hpp:18-20); this completion is
// arbitrary too, but deterministic per seed.
// Rows are indexed globally (row_offset + i of rows_global) so a row-sharded
// basis gets the same completion as the unsharded one.
__global__ void complete_basis_kernel(double* __restrict__ Q, int64_t ld, int64_t stride,
                                      int64_t rows, int64_t ell, const int* __restrict__ rank,
                                      const uint64_t* __restrict__ seeds, uint64_t tag,
                                      int64_t row_offset, int64_t rows_global,
                                      const int* __restrict__ mask) {
  const int64_t b = blockIdx.y;
  if (mask && !mask[b]) return;
  const int r = rank[b];
  if (r >= ell) return;
  const uint64_t key = seeds[b] ^ mix64(tag);
  const double scale = 1.0 / sqrt(static_cast<double>(rows_global));
  const int64_t total = rows * (ell - r);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = r + e / rows, i = e % rows;
    const uint64_t idx = static_cast<uint64_t>(row_offset + i + j * rows_global);
    const double u1 = uniform_from(mix64(key + (2 * idx + 1) * 0x9e3779b97f4a7c15ull));
    const double u2 = uniform_from(mix64(key + (2 * idx + 2) * 0x9e3779b97f4a7c15ull));
    const double z = sqrt(-2.0 * log(u1)) * cos((2.0 * 3.141592653589793) * u2);
    Q[b * stride + i + j * ld] = z * scale;
  }
}

__global__ void transpose_kernel(const double* __restrict__ in, int64_t ldi, int64_t stri,
                                 int64_t rows, int64_t cols, double* __restrict__ out,
                                 int64_t ldo, int64_t stro) {
  __shared__ double tile[32][33];
  const int64_t b = blockIdx.z;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32, c0 = static_cast<int64_t>(blockIdx.y) * 32;
  const double* src = in + b * stri;
  double* dst = out + b * stro;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + threadIdx.x, c = c0 + y;
    tile[y][threadIdx.x] = (r < rows && c < cols) ? src[r + c * ldi] : 0.0;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + threadIdx.x, r = r0 + y;  // out(c, r) = in(r, c)
    if (c < cols && r < rows) dst[c + r * ldo] = tile[threadIdx.x][y];
  }
}

__global__ void set_identity_kernel(double* __restrict__ out, int64_t ld, int64_t stride,
                                    int64_t n, int64_t batch) {
  const int64_t total = n * n * batch;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = e / (n * n), rem = e % (n * n);
    const int64_t j = rem / n, i = rem % n;
    out[b * stride + i + j * ld] = (i == j) ? 1.0 : 0.0;
  }
}

// sigma_i = ||HJ e_i||, sorted descending (ties by column index), numerical
// rank cut and discarded weight of the sampled tail:
//   numerical_rank (factorize.cpp:17-24): values <= max(m,n)*eps*sigma_0 are
//   zero; r = min(k, that rank) (truncate_full, factorize.cpp:26-38);
//   discarded = sum_{i >= r} sigma_i^2 over the l sampled values.
__global__ void finalize_spectrum_kernel(const double* __restrict__ HJ, int64_t ellp, int ell,
                                         int64_t k, int64_t m, int64_t n,
                                         double* __restrict__ sigma_out, int* __restrict__ perm,
                                         int* __restrict__ rank_out, double* __restrict__ dw_out) {
  extern __shared__ double s_sig[];
  int* s_pos = reinterpret_cast<int*>(s_sig + ellp);
  const int64_t b = blockIdx.x;
  const double* Hb = HJ + b * ellp * ellp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = warp; c < ell; c += nw) {
    double s = 0.0;
    for (int r = lane; r < ell; r += 32) {
      const double x = Hb[r + c * ellp];
      s = fma(x, x, s);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) s_sig[c] = sqrt(s);
  }
  __syncthreads();
  // Rank sort: position of column c in the descending order.
  for (int c = threadIdx.x; c < ell; c += blockDim.x) {
    const double v = s_sig[c];
    int pos = 0;
    for (int d = 0; d < ell; ++d) {
      const double w = s_sig[d];
      pos += (w > v) || (w == v && d < c);
    }
    s_pos[c] = pos;
    perm[b * ellp + pos] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // sorted values, in order
    // perm (global, written above by this block) maps positions to columns
    const int* pb = perm + b * ellp;
    const double smax = ell > 0 ? s_sig[pb[0]] : 0.0;
    int nr = 0;
    if (smax > 0.0) {
      const double cut = static_cast<double>(m > n ? m : n) * DBL_EPSILON * smax;
      for (int c = 0; c < ell; ++c) nr += s_sig[c] > cut;
    }
    const int r = static_cast<int>(nr < k ? nr : k);
    rank_out[b] = r;
    // discarded weight in descending order of the tail (as the reference's loop)
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

// dst[:, c] = src[:, perm[c]] / sigma[c] (sigma may be null: no scaling) for
// c < rank[b]; zero for rank[b] <= c < k.
__global__ void gather_scale_kernel(const double* __restrict__ src, int64_t ld_src,
                                    int64_t stride_src, const int* __restrict__ perm,
                                    int64_t ellp_perm, const double* __restrict__ sigma,
                                    int64_t sigma_stride, const int* __restrict__ rank,
                                    int64_t rows, int64_t k, double* __restrict__ dst,
                                    int64_t ld_dst, int64_t stride_dst) {
  const int64_t b = blockIdx.y;
  const int r = rank[b];
  const int64_t total = rows * k;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / rows, i = e % rows;
    double v = 0.0;
    if (c < r) {
      const int pc = perm[b * ellp_perm + c];
      v = src[b * stride_src + i + pc * ld_src];
      if (sigma) v /= sigma[b * sigma_stride + c];
    }
    dst[b * stride_dst + i + c * ld_dst] = v;
  }
}

__global__ void zero_cols_kernel(double* __restrict__ X, int64_t ld, int64_t stride, int64_t rows,
                                 int64_t cols, const int* __restrict__ rank) {
  const int64_t b = blockIdx.y;
  const int64_t r = rank[b];
  const int64_t total = rows * (cols - r);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = r + e / rows, i = e % rows;
    X[b * stride + i + c * ld] = 0.0;
  }
}

__global__ void zero_rows_kernel(double* __restrict__ X, int64_t ld, int64_t stride, int64_t rows,
                                 int64_t cols, const int* __restrict__ rank) {
  const int64_t b = blockIdx.y;
  const int64_t r = rank[b];
  const int64_t nr = rows - r;
  const int64_t total = nr * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / nr, i = r + e % nr;
    X[b * stride + i + c * ld] = 0.0;
  }
}

__global__ void copy_kernel(const double* __restrict__ in, int64_t ldi, int64_t stri, int64_t rows,
                            int64_t cols, double* __restrict__ out, int64_t ldo, int64_t stro) {
  const int64_t b = blockIdx.y;
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / rows, i = e % rows;
    out[b * stro + i + c * ldo] = in[b * stri + i + c * ldi];
  }
}

// Fixed-shape two-level sum of squares of (A - R): block partials.
__global__ void residual_sumsq_kernel(const double* __restrict__ A, int64_t lda,
                                      const double* __restrict__ R, int64_t ldr, int64_t rows,
                                      int64_t cols, double* __restrict__ partial) {
  __shared__ double red[32];
  const int64_t total = rows * cols;
  double s = 0.0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / rows, i = e % rows;
    const double d = A[i + c * lda] - R[i + c * ldr];
    s = fma(d, d, s);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
  }
}

__global__ void scale_columns_kernel(double* __restrict__ X, int64_t ld, int64_t rows,
                                     int64_t cols, const double* __restrict__ sc) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / rows, i = e % rows;
    X[i + c * ld] *= sc[c];
  }
}

__global__ void identity_rect_kernel(double* __restrict__ X, int64_t ld, int64_t stride,
                                     int64_t rows, int64_t cols) {
  const int64_t b = blockIdx.y;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < rows * cols;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / rows, i = e % rows;
    X[b * stride + i + c * ld] = (i == c) ? 1.0 : 0.0;
  }
}

__global__ void masked_copy_kernel(const int* __restrict__ mask, const double* __restrict__ src,
                                   int64_t lds, int64_t ss, double* __restrict__ dst, int64_t ldd,
                                   int64_t sd, int64_t rows, int64_t cols) {
  const int64_t b = blockIdx.y;
  if (!mask[b]) return;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < rows * cols;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / rows, i = e - c * rows;
    dst[b * sd + i + c * ldd] = src[b * ss + i + c * lds];
  }
}

// Exact power-of-two range scaling (extreme-magnitude inputs).  Per item:
// the largest |x| over rows x cols; outside [2^-200, 2^200] the item gets the
// factor c = 2^-e (max |x| c in [0.5, 1)), else c = 1.  Scaling by a power of
// two is exact, so in-range inputs are untouched bit for bit.
__global__ void maxabs_kernel(const double* __restrict__ X, int64_t ld, int64_t stride,
                              int64_t rows, int64_t cols, unsigned long long* __restrict__ bits) {
  __shared__ double red[32];
  const int64_t b = blockIdx.y;
  const double* x = X + b * stride;
  double mx = 0.0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < rows * cols;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / rows, r = e - c * rows;
    mx = fmax(mx, fabs(x[r + c * ld]));
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    // non-negative doubles order like their bit patterns: an integer max is exact
    atomicMax(bits + b, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

__global__ void choose_scale_kernel(unsigned long long* __restrict__ bits,
                                    double* __restrict__ scale, int64_t batch) {
  const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const double m = __longlong_as_double(static_cast<long long>(bits[b]));
  double c = 1.0;
  if (m > 0.0 && isfinite(m) && (m < 0x1p-200 || m > 0x1p200)) {
    int e = 0;
    frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
    c = ldexp(1.0, -e);
  }
  scale[b] = c;
}

// X[b] *= c[b] (pow2 == true) or X[b] *= 1 / c[b]^pw for the spectrum (sigma,
// pw = 1) and the discarded weight (pw = 2); items with c == 1 are skipped.
__global__ void apply_scale_kernel(double* __restrict__ X, int64_t ld, int64_t stride,
                                   int64_t rows, int64_t cols, const double* __restrict__ scale,
                                   int inverse_power) {
  const int64_t b = blockIdx.y;
  const double c = scale[b];
  if (c == 1.0) return;
  double f = c;
  if (inverse_power == 1) f = 1.0 / c;
  if (inverse_power == 2) f = 1.0 / (c * c);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < rows * cols;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t cc = e / rows, r = e - cc * rows;
    X[b * stride + r + cc * ld] *= f;
  }
}

unsigned grid1(int64_t work, int threads, int cap_per_sm = 8) {
  return static_cast<unsigned>(
      std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, threads), cap_per_sm * num_sms())));
}

// x-extent of a (x, batch) grid whose items usually exit at once (completion
// of full-rank bases, masked copies, unit scales): about two CTAs per SM in
// total instead of one per 256 elements, so the no-op case launches a few
// hundred CTAs rather than tens of thousands.
unsigned grid_items(int64_t work, int threads, int64_t batch, int per_sm = 2) {
  return static_cast<unsigned>(std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(work, threads),
                           ceil_div(static_cast<int64_t>(per_sm) * num_sms(), std::max<int64_t>(batch, 1)))));
}

}  // namespace

void launch_complete_basis(MatRef Q, int64_t rows, int64_t ell, const int* rank,
                           const uint64_t* seeds_dev, uint64_t tag, int64_t batch,
                           int64_t row_offset, int64_t rows_global, cudaStream_t st,
                           const int* mask) {
  if (batch <= 0 || rows <= 0) return;
  dim3 grid(grid_items(rows * ell, 256, batch), static_cast<unsigned>(batch));
  complete_basis_kernel<<<grid, 256, 0, st>>>(Q.base, Q.ld, Q.stride, rows, ell, rank, seeds_dev,
                                              tag, row_offset, rows_global, mask);
  RSVD_LAUNCH("complete_basis_kernel");
}

void launch_transpose(CMatRef in, int64_t rows, int64_t cols, MatRef out, int64_t batch,
                      cudaStream_t st) {
  if (batch <= 0 || rows <= 0 || cols <= 0) return;
  dim3 grid(static_cast<unsigned>(ceil_div(rows, 32)), static_cast<unsigned>(ceil_div(cols, 32)),
            static_cast<unsigned>(batch));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in.base, in.ld, in.stride, rows, cols, out.base,
                                                 out.ld, out.stride);
  RSVD_LAUNCH("transpose_kernel");
}

void launch_set_identity_rect(MatRef out, int64_t rows, int64_t cols, int64_t batch,
                              cudaStream_t st) {
  if (batch <= 0 || rows <= 0 || cols <= 0) return;
  dim3 grid(grid1(rows * cols, 256, 2), static_cast<unsigned>(batch));
  identity_rect_kernel<<<grid, 256, 0, st>>>(out.base, out.ld, out.stride, rows, cols);
  RSVD_LAUNCH("identity_rect_kernel");
}

void launch_masked_copy(const int* mask, CMatRef src, MatRef dst, int64_t rows, int64_t cols,
                        int64_t batch, cudaStream_t st) {
  if (batch <= 0 || rows <= 0 || cols <= 0) return;
  dim3 grid(grid_items(rows * cols, 256, batch), static_cast<unsigned>(batch));
  masked_copy_kernel<<<grid, 256, 0, st>>>(mask, src.base, src.ld, src.stride, dst.base, dst.ld,
                                           dst.stride, rows, cols);
  RSVD_LAUNCH("masked_copy_kernel");
}

void launch_choose_scale(CMatRef X, int64_t rows, int64_t cols, double* scale, int64_t batch,
                         cudaStream_t st) {
  if (batch <= 0) return;
  // scale[] doubles as the max-bits accumulator (same 8 bytes per item).
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(scale);
  RSVD_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned long long) * batch, st));
  dim3 grid(grid1(rows * cols, 256, 4), static_cast<unsigned>(batch));
  if (batch > 1) grid.x = std::max(1u, std::min(grid.x, static_cast<unsigned>(4 * num_sms() / batch + 1)));
  maxabs_kernel<<<grid, 256, 0, st>>>(X.base, X.ld, X.stride, rows, cols, bits);
  RSVD_LAUNCH("maxabs_kernel");
  choose_scale_kernel<<<static_cast<unsigned>(ceil_div(batch, 256)), 256, 0, st>>>(bits, scale,
                                                                                   batch);
  RSVD_LAUNCH("choose_scale_kernel");
}

void launch_apply_scale(MatRef X, int64_t rows, int64_t cols, const double* scale,
                        int inverse_power, int64_t batch, cudaStream_t st) {
  if (batch <= 0 || rows <= 0 || cols <= 0) return;
  dim3 grid(grid_items(rows * cols, 256, batch, 8), static_cast<unsigned>(batch));
  apply_scale_kernel<<<grid, 256, 0, st>>>(X.base, X.ld, X.stride, rows, cols, scale,
                                           inverse_power);
  RSVD_LAUNCH("apply_scale_kernel");
}

void launch_set_identity(MatRef out, int64_t n, int64_t batch, cudaStream_t st) {
  if (batch <= 0 || n <= 0) return;
  set_identity_kernel<<<grid1(n * n * batch, 256), 256, 0, st>>>(out.base, out.ld, out.stride, n,
                                                                  batch);
  RSVD_LAUNCH("set_identity_kernel");
}

void launch_finalize_spectrum(const double* HJ, int64_t ellp, int64_t ell, int64_t k, int64_t m,
                              int64_t n, double* sigma_out, int* perm, int* rank,
                              double* discarded, int64_t batch, cudaStream_t st) {
  if (batch <= 0) return;
  const size_t smem = ellp * (sizeof(double) + sizeof(int));
  finalize_spectrum_kernel<<<static_cast<unsigned>(batch), 512, smem, st>>>(
      HJ, ellp, static_cast<int>(ell), k, m, n, sigma_out, perm, rank, discarded);
  RSVD_LAUNCH("finalize_spectrum_kernel");
}

void launch_gather_scale_columns(const double* src, int64_t ld_src, int64_t stride_src,
                                 const int* perm, int64_t ellp_perm, const double* sigma,
                                 int64_t sigma_stride, const int* rank, int64_t rows, int64_t k,
                                 double* dst, int64_t ld_dst, int64_t stride_dst, int64_t batch,
                                 cudaStream_t st) {
  if (batch <= 0 || rows <= 0 || k <= 0) return;
  dim3 grid(grid1(rows * k, 256, 2), static_cast<unsigned>(batch));
  gather_scale_kernel<<<grid, 256, 0, st>>>(src, ld_src, stride_src, perm, ellp_perm, sigma,
                                            sigma_stride, rank, rows, k, dst, ld_dst, stride_dst);
  RSVD_LAUNCH("gather_scale_kernel");
}

void launch_zero_columns_from_rank(MatRef X, int64_t rows, int64_t cols, const int* rank,
                                   int64_t batch, cudaStream_t st) {
  if (batch <= 0 || rows <= 0 || cols <= 0) return;
  dim3 grid(grid_items(rows * cols, 256, batch, 4), static_cast<unsigned>(batch));
  zero_cols_kernel<<<grid, 256, 0, st>>>(X.base, X.ld, X.stride, rows, cols, rank);
  RSVD_LAUNCH("zero_cols_kernel");
}

void launch_zero_rows_from_rank(MatRef X, int64_t rows, int64_t cols, const int* rank,
                                int64_t batch, cudaStream_t st) {
  if (batch <= 0 || rows <= 0 || cols <= 0) return;
  dim3 grid(grid_items(rows * cols, 256, batch, 4), static_cast<unsigned>(batch));
  zero_rows_kernel<<<grid, 256, 0, st>>>(X.base, X.ld, X.stride, rows, cols, rank);
  RSVD_LAUNCH("zero_rows_kernel");
}

void launch_copy_matrix(CMatRef in, int64_t rows, int64_t cols, MatRef out, int64_t batch,
                        cudaStream_t st) {
  if (batch <= 0 || rows <= 0 || cols <= 0) return;
  dim3 grid(grid1(rows * cols, 256, 2), static_cast<unsigned>(batch));
  copy_kernel<<<grid, 256, 0, st>>>(in.base, in.ld, in.stride, rows, cols, out.base, out.ld,
                                    out.stride);
  RSVD_LAUNCH("copy_kernel");
}

void launch_scale_columns(MatRef X, int64_t rows, int64_t cols, const double* sc, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  scale_columns_kernel<<<grid1(rows * cols, 256), 256, 0, st>>>(X.base, X.ld, rows, cols, sc);
  RSVD_LAUNCH("scale_columns_kernel");
}

void launch_residual_sumsq(CMatRef A, CMatRef R, int64_t rows, int64_t cols, double* partial,
                           int64_t nparts, cudaStream_t st) {
  residual_sumsq_kernel<<<static_cast<unsigned>(nparts), 256, 0, st>>>(A.base, A.ld, R.base, R.ld,
                                                                       rows, cols, partial);
  RSVD_LAUNCH("residual_sumsq_kernel");
}

}  // namespace rsvd
