// Shared device/host helpers for the B200 RSVD engine (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include "../../include/rsvd_c.h"

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>

namespace rsvd {

// Strided batch of column-major matrices: element (i, j) of item b lives at
// base[b * stride + i + j * ld].
struct MatRef {
  double* base;
  int64_t ld;
  int64_t stride;
  __host__ __device__ double* item(int64_t b) const { return base + b * stride; }
};
struct CMatRef {
  const double* base;
  int64_t ld;
  int64_t stride;
  __host__ __device__ const double* item(int64_t b) const { return base + b * stride; }
  CMatRef() = default;
  __host__ __device__ CMatRef(const double* p, int64_t l, int64_t s) : base(p), ld(l), stride(s) {}
  __host__ __device__ CMatRef(const MatRef& m) : base(m.base), ld(m.ld), stride(m.stride) {}
};

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
// Number of engine kernels launched by this process (reported by bench.py as
// gpu_launches; every launch site goes through RSVD_LAUNCH).
extern std::atomic<uint64_t> g_kernel_launches;
#define RSVD_CUDA(call) ::rsvd::check_cuda((call), #call)
#define RSVD_LAUNCH(what)                                                  \
  do {                                                                     \
    ::rsvd::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);     \
    ::rsvd::check_cuda(cudaGetLastError(), what);                          \
  } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Per-device facts, cached per device ordinal (thread-safe: the in-process
// rank threads of sharding.GroupReducer and multi-device callers share them).
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d & (kMaxDevices - 1);
}
// SM count of the current device (148 on a full B200; fewer under MIG / MPS
// limits), used for grid sizing and co-residency of cooperative launches.
inline int num_sms() {
  static std::atomic<int> cache[kMaxDevices];
  const int d = current_device();
  int v = cache[d].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0)
      v = 148;
    cache[d].store(v, std::memory_order_relaxed);
  }
  return v;
}
// Total memory of the current device in bytes (cached per device ordinal).
inline int64_t device_total_memory() {
  static std::atomic<int64_t> cache[kMaxDevices];
  const int d = current_device();
  int64_t v = cache[d].load(std::memory_order_relaxed);
  if (v <= 0) {
    size_t fr = 0, tot = 0;
    v = cudaMemGetInfo(&fr, &tot) == cudaSuccess ? static_cast<int64_t>(tot) : (int64_t{180} << 30);
    cache[d].store(v, std::memory_order_relaxed);
  }
  return v;
}
// Function attributes (e.g. the dynamic shared-memory opt-in) are per device
// context: `mask` (one per kernel instantiation) records the devices on which
// `apply` already ran.  apply() is idempotent, so a race only repeats it.
template <class F>
inline void once_per_device(std::atomic<uint64_t>& mask, F&& apply) {
  const uint64_t bit = 1ull << current_device();
  if (mask.load(std::memory_order_acquire) & bit) return;
  apply();
  mask.fetch_or(bit, std::memory_order_acq_rel);
}

// ---------------------------------------------------------------- kernels
// Launch wrappers (defined in the .cu files).  All are batched and
// stream-ordered; none synchronizes.

// rng.cu — CounterRng Gaussian fill of `rows x cols` (column-major, ld) per
// item, seeds[b] per item (device array); columns >= valid_cols are zeroed.
void launch_fill_gaussian(MatRef out, int64_t rows, int64_t cols, int64_t valid_cols,
                          const uint64_t* seeds_dev, int64_t batch, cudaStream_t st);
void launch_fill_gaussian_flat(double* out, int64_t count, uint64_t seed, cudaStream_t st);

// gemm_f64.cu — C = op(A) * B with op(A) = A (NN) or A^T (TN, A stored K x M).
// When splits > 1 the partial products go to `partial` (splits*batch items
// of M x N, ld M) and are reduced in fixed order into C (deterministic).
void dgemm(bool trans_a, int64_t M, int64_t N, int64_t K, CMatRef A, CMatRef B, MatRef C,
           int64_t batch, double* partial, int64_t partial_capacity, cudaStream_t st);
// Structured variants: NN with a per-item column map on A (A(:, k) =
// A_stored(:, colmapA[item*colmap_stride + k])), upper-triangular B (skips the
// zero K-range per output tile), and symmetric C (upper tiles only, mirrored).
struct GemmOpts {
  const int* colmapA = nullptr;
  int64_t colmap_stride = 0;
  bool b_upper = false;
  bool c_upper = false;
  // item_mask[b] == 0 skips item b entirely (C untouched): the masked passes
  // of the ill-conditioned CholeskyQR fallback (engine.cu orth).
  const int* item_mask = nullptr;
};
void dgemm_ex(bool trans_a, int64_t M, int64_t N, int64_t K, CMatRef A, CMatRef B, MatRef C,
              int64_t batch, double* partial, int64_t partial_capacity, const GemmOpts& opt,
              cudaStream_t st);
// gemm_tma.cu — TMA/mbarrier-fed variant of the 128 x 96 tile (no column map);
// returns false (nothing launched) when the operands do not qualify.
// ozaki.cu — FP64 GEMM emulated on the tcgen05 INT8 tensor cores.
// oz_prepare_a slices A (rows x cols, column-major) once: sR row-major with
// per-row exponents eRow (operand of C = A B), sC column-major with per-column
// exponents eCol (operand of C = A^T B); each oz_slice_bytes(rows, cols, batch).
// oz_slice_b slices the right operand B (K x N column-major) into sB / eB
// (oz_slice_bytes(K, N, batch) bytes, N * batch ints); oz_gemm: C (M x N) =
// op(A) B from the slices of op(A) (sA / eA, M x K, K-major) and of B.
bool oz_supported(int64_t rows, int64_t cols, int64_t K);
double oz_grid_efficiency(int64_t M, int64_t N, int64_t batch);
#ifdef RSVD_OZ_TRACE
void oz_trace_read(unsigned long long* out, int64_t n);  // tools/probe/oz_trace.py
#endif
int64_t oz_slice_bytes(int64_t rows, int64_t cols, int64_t batch);
void oz_prepare_a(CMatRef A, int64_t rows, int64_t cols, int64_t batch, int8_t* sR, int8_t* sC,
                  int* eRow, int* eCol, cudaStream_t st);
void oz_slice_b(CMatRef B, int64_t K, int64_t N, int64_t batch, int8_t* sB, int* eB,
                cudaStream_t st);
void oz_gemm(int64_t M, int64_t N, int64_t K, const int8_t* sA, const int* eA, const int8_t* sB,
             const int* eB, MatRef C, int64_t batch, cudaStream_t st);
bool dgemm_tma(bool trans_a, int64_t M, int64_t N, int64_t K, CMatRef A, CMatRef B, double* C,
               int64_t ldc, int64_t strideC, int64_t batch, int splits, int64_t kps, bool c_upper,
               const int* item_mask,
               bool b_upper, cudaStream_t st, int tile = 0);
int64_t dgemm_partial_elems(bool trans_a, int64_t M, int64_t N, int64_t K, int64_t batch);

// chol.cu — pivoted / plain Cholesky of SPD Grams (ell x ell, ld ell).
// G is consumed (used as factorization storage); scratch holds
// pchol_scratch_elems(ellp, batch) doubles.
int64_t pchol_scratch_elems(int64_t ellp, int64_t batch);
// Options of the unpivoted kernel (any CholOpts forces it):
//   mask       item b runs only if mask[b] != 0;
//   gate_rank  item b runs only if gate_rank[b] < ell; ill_out[b] records it;
//   Gsrc       factor a copy of Gsrc[b] (G[b] is overwritten);
//   shift_coef factor G + coef * tr(G) * I (shifted CholeskyQR).
struct CholOpts {
  const int* mask = nullptr;
  const int* gate_rank = nullptr;
  int* ill_out = nullptr;
  const double* Gsrc = nullptr;
  double shift_coef = 0.0;
  bool pairs = false;  // pivoted kernel: pivot complex columns (2a, 2a+1) together
  // Repeat CholeskyQR pass (unpivoted, alone): items whose Gram is I + E with
  // ||triu(E)||_F^2 <= 1e-16 (diagonal halved) get the first-order factor
  // R = I + F, T = I - F, rank = ell; the rest are factored exactly.
  bool lin = false;
};
void launch_pchol(double* G, double* T, double* Rfull, double* scratch, int* rank, int* perm,
                  int64_t ell, int64_t ellp, double tau, bool pivot, int64_t batch,
                  cudaStream_t st, const CholOpts* opts = nullptr);

// chol.cu -- one fused CholeskyQR pass for l_p <= 160 (Gram, Cholesky with
// breakdown -> rank, Q = Y R^-1): Q columns >= rank are zero (completion is the
// caller's); G0 (full symmetric Gram) and Rf (R, zero below / beyond rank) are
// written when non-null.  Returns false when the shape does not qualify.
// xscratch: fcqr_xscratch_elems(ellp, batch) doubles (row-split cluster mode;
// null disables it).  lin (repeat passes): items whose Gram is within 1e-8 of I
// take the first-order factor R = I + triu(G - I) / (1 + [diag]) instead of the
// exact Cholesky (rank = ell); the others are factored exactly.
bool launch_fused_cqr(const double* Y, int64_t ldy, int64_t strideY, double* Q, int64_t ldq,
                      int64_t strideQ, double* G0, double* Rf, double* xscratch, int* rank,
                      int64_t rows, int64_t ell, int64_t ellp, double tau, int64_t batch,
                      cudaStream_t st, bool lin = false);
int64_t fcqr_xscratch_elems(int64_t ellp, int64_t batch);

// jacobi.cu — one-sided Jacobi on H (ellp x ellp per item; first `ell`
// columns live), accumulating J; sweeps until converged.
// flags: jacobi_flag_elems(batch) unsigned ints of workspace.
int64_t jacobi_flag_elems(int64_t batch, int64_t ellp);
void launch_jacobi(double* H, double* J, int64_t ell, int64_t ellp, int max_sweeps, int* sweeps,
                   unsigned* flags, int64_t batch, cudaStream_t st);

// tebd.cu -- table-driven TEBD bond-update kernels (tables in device memory).
void launch_combine_blocks(bool cplx, const rsvd_block_job* jobs_dev, const rsvd_block_term* terms_dev,
                           const int64_t* start_dev, int64_t njobs, int64_t total, cudaStream_t st);
void launch_grouped_gemm(bool cplx, const rsvd_gemm_job* jobs_dev, const int4* tiles_dev,
                         int64_t ntiles, cudaStream_t st);
int64_t grouped_gemm_tile(int64_t extent);  // tiles along one extent
void launch_block_sqnorms(bool cplx, const rsvd_block_job* blocks_dev, const int64_t* begin_dev,
                          int64_t nslots, double* out_dev, cudaStream_t st);

// aux.cu
void launch_complete_basis(MatRef Q, int64_t rows, int64_t ell, const int* rank,
                           const uint64_t* seeds_dev, uint64_t tag, int64_t batch,
                           int64_t row_offset, int64_t rows_global, cudaStream_t st,
                           const int* mask = nullptr);

// Sum all-reduce across the ranks of a row-sharded factorization (NCCL or an
// in-process group); stream-ordered on `st`.
struct Reducer {
  virtual ~Reducer() = default;
  virtual void allreduce_sum(double* buf, int64_t count, cudaStream_t st) = 0;
  virtual bool capturable() const = 0;  // safe inside CUDA-graph capture
};
// shard.cu
struct Group;
Group* group_create(int nranks);
void group_destroy(Group* g);
std::unique_ptr<Reducer> make_group_reducer(Group* g, int rank);
std::unique_ptr<Reducer> make_nccl_reducer(int nranks, int rank, const unsigned char* id);
void nccl_unique_id(unsigned char* out);
void launch_transpose(CMatRef in, int64_t rows, int64_t cols, MatRef out, int64_t batch,
                      cudaStream_t st);
// Exact power-of-two range scaling of extreme-magnitude items (aux.cu):
// scale[b] = 2^-e when max|X[b]| is outside [2^-200, 2^200], else 1;
// apply: X[b] *= scale[b] (inverse_power 0), / scale[b] (1), / scale[b]^2 (2).
void launch_choose_scale(CMatRef X, int64_t rows, int64_t cols, double* scale, int64_t batch,
                         cudaStream_t st);
void launch_apply_scale(MatRef X, int64_t rows, int64_t cols, const double* scale,
                        int inverse_power, int64_t batch, cudaStream_t st);
// dst[b] = src[b] (rows x cols) for the items with mask[b] != 0.
void launch_masked_copy(const int* mask, CMatRef src, MatRef dst, int64_t rows, int64_t cols,
                        int64_t batch, cudaStream_t st);
void launch_set_identity(MatRef out, int64_t n, int64_t batch, cudaStream_t st);
void launch_set_identity_rect(MatRef out, int64_t rows, int64_t cols, int64_t batch,
                              cudaStream_t st);
void launch_finalize_spectrum(const double* HJ, int64_t ellp, int64_t ell, int64_t k,
                              int64_t m, int64_t n, double* sigma_out, int* perm, int* rank,
                              double* discarded, int64_t batch, cudaStream_t st);
void launch_gather_scale_columns(const double* src, int64_t ld_src, int64_t stride_src,
                                 const int* perm, int64_t ellp_perm, const double* sigma,
                                 int64_t sigma_stride, const int* rank, int64_t rows, int64_t k,
                                 double* dst,
                                 int64_t ld_dst, int64_t stride_dst, int64_t batch,
                                 cudaStream_t st);
void launch_zero_columns_from_rank(MatRef X, int64_t rows, int64_t cols, const int* rank,
                                   int64_t batch, cudaStream_t st);
void launch_zero_rows_from_rank(MatRef X, int64_t rows, int64_t cols, const int* rank,
                                int64_t batch, cudaStream_t st);
void launch_copy_matrix(CMatRef in, int64_t rows, int64_t cols, MatRef out, int64_t batch,
                        cudaStream_t st);
void launch_scale_columns(MatRef X, int64_t rows, int64_t cols, const double* sc, cudaStream_t st);
void launch_residual_sumsq(CMatRef A, CMatRef R, int64_t rows, int64_t cols, double* partial,
                           int64_t nparts, cudaStream_t st);

// zkern.cu — complex instantiation (see the layout notes there).
void launch_zfill_gaussian_p(MatRef out, int64_t rows, int64_t lp, int64_t ell,
                             const uint64_t* seeds_dev, int64_t batch, cudaStream_t st);
void launch_zfill_gaussian_flat(double* out, int64_t count, uint64_t seed, cudaStream_t st);
void launch_zcombine_nn(CMatRef P, MatRef Y, int64_t m, int64_t lp, int64_t batch,
                        cudaStream_t st);
void launch_zpair(CMatRef Q, MatRef out, int64_t m, int64_t lp, int64_t batch, cudaStream_t st);
void launch_zp2i(CMatRef X, MatRef out, int64_t rows, int64_t cols, int64_t batch,
                 cudaStream_t st);
void launch_zi2p(CMatRef X, MatRef out, int64_t rows, int64_t cols, int64_t batch,
                 cudaStream_t st);
void launch_zadjoint(CMatRef X, bool from_p, MatRef out, int64_t rows, int64_t cols,
                     int64_t batch, cudaStream_t st);
void launch_zidentity_p(MatRef X, int64_t rows, int64_t lp, int64_t ell, int64_t batch,
                        cudaStream_t st);
void launch_hermitize(double* G, int64_t lp, const int* mask, int64_t batch, cudaStream_t st);
// flags (jacobi_flag_elems(batch), optional): enables the block-cyclic
// Gram-accelerated kernel for batches with many tasks.
void launch_zjacobi(const double* src, int64_t src_ld, int64_t src_stride, int src_mode,
                    double* H, double* J, int64_t ell, int64_t lp, int max_sweeps, int* sweeps,
                    int64_t batch, cudaStream_t st, unsigned* flags = nullptr);
void launch_zfinalize(const double* W, int64_t lp, int64_t ell, int64_t k, int64_t m, int64_t n,
                      double* sigma_out, int* perm, int* rank, double* dw, int64_t batch,
                      cudaStream_t st);
void launch_zlift_operand(const double* W, int64_t lp, const int* perm, const double* sigma,
                          int64_t k, const int* rank, int64_t ell, bool half, MatRef M,
                          int64_t batch, cudaStream_t st);

}  // namespace rsvd
