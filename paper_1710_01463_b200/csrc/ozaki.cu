// FP64 GEMM emulated on the tcgen05 INT8 tensor cores (Ozaki scheme, split
// into signed 8-bit slices), for the RSVD A-passes Y = A X and Z = A^T Y
// (factorize.cpp:68, 70, 71, 86).
//
// B200 has no tcgen05 f64 kind: the warp-level DMMA path (gemm_tma.cu) tops
// out at ~37 TFLOP/s.  The INT8 tensor cores run ~4.5 POPS dense, so an FP64
// product rebuilt from exact integer products of short slices is faster even
// after paying for the slice products:
//   x = 2^e * sum_{p<S} s_p 2^(-6-8p),   s_0 in [-65, 65], s_p in [-128, 127]
//       (balanced base-256 digits of rint(x 2^(54-e)); e per row of op(A) /
//       per column of B; S = 7 slices = 54 bits below 2^e)
//   (A B)_ij = 2^(eA_i + eB_j - 12) * sum_{d<S} 2^(-8d) * sum_{p+q=d} (A_p B_q)_ij
// Every slice product is exact in INT32 (|s| <= 128, <= 7 terms per diagonal,
// K chunks of <= 16384 per launch); the terms with p + q >= S are below 2^-54
// of the row/column maxima and are dropped, which leaves a normwise error of
// the order of an FP64 GEMM's.
//
// Layout.  A is sliced ONCE per rsvd call into both K-major layouts:
//   R: slices of A with per-row exponents, row-major  [item][p][row][col]
//      (the K-major operand of the NN pass  Y = A X)
//   C: slices of A with per-column exponents, col-major [item][p][col][row]
//      (the K-major operand of the TN pass  Z = A^T Y)
// The small right operand (X or Y, K x N column-major = K-major) is sliced per
// pass.  A CTA owns a 128 x BN output tile and keeps the S diagonal sums in
// TMEM (S * BN = 448 columns); per 32-byte K step one TMA box brings the S
// slices of each operand (32B swizzle), and one thread issues the S(S+1)/2 =
// 28 slice products of that step as 10 stacked tcgen05.mma.kind::i8.  The
// epilogue folds the diagonals in FP64 (Horner in 2^-8) and writes (or adds
// to, for the later K chunks) C column-major.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <mutex>

#include "common.cuh"

namespace rsvd {
namespace {

constexpr int kOzS = 7;       // slices per operand
constexpr int kOzBM = 128;    // UMMA M
constexpr int kOzBN = 64;     // UMMA N of the wide tile (S * BN = 448 of the 512 TMEM columns)
constexpr int kOzBNs = 32;    // narrow tile for grids of one or two thin waves (C3: 288 tiles)
constexpr int kOzKC = 32;     // K bytes per stage = one MMA K step = one 32B swizzle row
constexpr int kOzStages = 5;  // 5 x 42 KB ring
constexpr int kOzKChunk = 16384;  // K per launch: 7 * 16384 * 128^2 < 2^31
constexpr int kExpNone = static_cast<int>(0x80808080u);  // cudaMemset(0x80): below any frexp exponent

__device__ __forceinline__ uint32_t sm_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mb_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "OZW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra OZW_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                       int c3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5}], [%6];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_c, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_c),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// K-major operand tile of `rows` x 32 bytes in the canonical no-swizzle
// ("interleaved") layout: 8 x 16-byte core matrices of 128 contiguous bytes,
// the two of one K step 128 bytes apart (LBO), 8-row groups 256 bytes apart
// (SBO), descriptor version 1.  This is also the layout of the slices in
// global memory (tile_off), so a TMA box row is 256 contiguous bytes.
__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(128 >> 4) << 16) |
         (static_cast<uint64_t>(256 >> 4) << 32) | (static_cast<uint64_t>(1) << 46);
}

// Byte offset of the 16-byte chunk (row r, K bytes 16c .. 16c+15) inside one
// slice plane of `R` rows x `K` bytes: [r / 8][c][r % 8][16].
__device__ __forceinline__ int64_t tile_off(int r, int c, int K) {
  return (static_cast<int64_t>(r >> 3) * (K >> 4) + c) * 128 + (r & 7) * 16;
}

// Exact int32 -> double on the FP64 pipe (I2F.F64 runs on the conversion unit
// at a few per clock per SM: 448 per thread made the TMEM drain ~10% of a
// tile): 2^52 + 2^31 + v has the low word v ^ 0x80000000.
__device__ __forceinline__ double i32_to_f64(uint32_t v) {
  return __hiloint2double(0x43300000, static_cast<int>(v ^ 0x80000000u)) - 4503601774854144.0;
}

// x 2^e for |x| < 2^35 and any e the exponents of two doubles can add up to:
// two multiplies by normal powers of two built from their exponent bits
// (branch-free and a handful of instructions: an inlined ldexp per element made
// the TMEM drain ~70 KB of straight-line code that ran from L2 at every tile,
// 9 us of an 88 us tile).  Below 2^-2040 the product underflows to 0 either way.
__device__ __forceinline__ double scale_pow2(double x, int e) {
  e = max(e, -2040);
  const int e1 = e >> 1, e2 = e - e1;
  return (x * __hiloint2double((1023 + e1) << 20, 0)) * __hiloint2double((1023 + e2) << 20, 0);
}

__device__ __forceinline__ int usable_exp(int e) { return e == kExpNone ? 0 : e; }  // all-zero line

// Signed 8-bit slices of x (|x| < 2^e): V = rint(x 2^(54-e)), |V| <= 2^54, as
// 7 balanced base-256 digits d_0 (most significant, |d_0| <= 65) .. d_6 (in
// [-128, 127]), V = sum_p d_p 256^(6-p): x = 2^e sum_p d_p 2^(-6-8p) up to the
// rounding of V (<= 2^(e-55)).  No FP64 <-> integer conversion instruction
// (they run at a few per clock per SM) and no 64-bit integer shifts: V is
// split into hi = rint(v 2^-24) and lo = rint(v - hi 2^24) with the 1.5 * 2^52
// trick, which leaves both integers in the low words of two doubles.  Adding
// the bias 128 * (256^k - 1) / 255 turns balanced digits into plain bytes
// (d + 128 in [0, 255]): the returned words hold d_6, d_5, d_4 (+128 each) in
// bytes 0-2 of .x (byte 3 is the carry, unused) and d_3 .. d_0 (+128) in .y;
// pack16 flips the top bits after the byte transpose.
__device__ __forceinline__ uint2 digit_bytes(double x, double sc_lo, double sc_hi) {
  constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  const double v = (x * sc_lo) * sc_hi;           // exact: powers of two
  const double th = fma(v, 0x1p-24, kMagic);
  const double hd = th - kMagic;                  // rint(v 2^-24), |hd| <= 2^30
  const double tl = fma(hd, -0x1p24, v) + kMagic;  // v - hd 2^24 is exact, |.| <= 2^23
  const uint32_t lo = static_cast<uint32_t>(__double2loint(tl)) + 0x808080u;
  const uint32_t hi = static_cast<uint32_t>(__double2loint(th)) + 0x80808080u + (lo >> 24);
  return make_uint2(lo, hi);
}

// 2^(54 - e) as two finite powers of two (e is a frexp exponent: any int in
// [-1073, 1024]).
struct SliceScale {
  double lo, hi;
  __device__ explicit SliceScale(int e) {
    const int t = 54 - e, a = t / 2;
    lo = __hiloint2double((1023 + a) << 20, 0);
    hi = __hiloint2double((1023 + t - a) << 20, 0);
  }
};

// Slices of 16 consecutive values (get(u), u < 16) packed per slice into 16
// bytes: a byte transpose of the 16 digit words, 14 PRMT per 4 values (one
// PRMT gathers two digit positions of two values, one more joins two pairs).
template <class Get>
__device__ __forceinline__ void pack16(Get get, const SliceScale& sc, uint4 (&out)[kOzS]) {
  uint32_t w[kOzS][4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint2 d = digit_bytes(get(4 * g + u), sc.lo, sc.hi);
      lo[u] = d.x;  // d_6, d_5, d_4, carry
      hi[u] = d.y;  // d_3, d_2, d_1, d_0
    }
    const uint32_t l01a = __byte_perm(lo[0], lo[1], 0x5140), l01c = __byte_perm(lo[2], lo[3], 0x5140);
    const uint32_t l2a = __byte_perm(lo[0], lo[1], 0x7362), l2c = __byte_perm(lo[2], lo[3], 0x7362);
    const uint32_t h01a = __byte_perm(hi[0], hi[1], 0x5140), h01c = __byte_perm(hi[2], hi[3], 0x5140);
    const uint32_t h23a = __byte_perm(hi[0], hi[1], 0x7362), h23c = __byte_perm(hi[2], hi[3], 0x7362);
    w[6][g] = __byte_perm(l01a, l01c, 0x5410) ^ 0x80808080u;
    w[5][g] = __byte_perm(l01a, l01c, 0x7632) ^ 0x80808080u;
    w[4][g] = __byte_perm(l2a, l2c, 0x5410) ^ 0x80808080u;
    w[3][g] = __byte_perm(h01a, h01c, 0x5410) ^ 0x80808080u;
    w[2][g] = __byte_perm(h01a, h01c, 0x7632) ^ 0x80808080u;
    w[1][g] = __byte_perm(h23a, h23c, 0x5410) ^ 0x80808080u;
    w[0][g] = __byte_perm(h23a, h23c, 0x7632) ^ 0x80808080u;
  }
#pragma unroll
  for (int p = 0; p < kOzS; ++p) out[p] = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
}

__device__ __forceinline__ int exp_of_max(double amax) {
  int e;
  frexp(amax, &e);
  return e;  // amax < 2^e
}

// 64 x 64 staging tile [col][row] with pitch 72 and 2 doubles of padding after
// every 16 rows: 16-byte reads of (column, 16-row chunk) by thread pairs and
// row reads by 32 consecutive rows are both bank-conflict free.
constexpr int kOzTP = 72;
__device__ __forceinline__ int oz_tile_idx(int c, int r) { return c * kOzTP + r + 2 * (r >> 4); }

// Per-row and per-column exponents of A (rows x cols, column-major): 64 x 64
// tiles, atomicMax into eRow / eCol (pre-set to kExpNone).  Rows reduce in
// registers (16 columns per thread) and shared memory; columns from a shared
// copy of |A| (16 rows per thread, then 4 lanes).
__global__ void __launch_bounds__(256) oz_exp_kernel(const double* __restrict__ A, int64_t lda,
                                                     int64_t sA, int rows, int cols, int* eRow,
                                                     int* eCol) {
  __shared__ double rmax[4][64];
  __shared__ __align__(16) double tile[64 * kOzTP];  // [col][row] of |A|
  const int item = blockIdx.z;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const double* Ab = A + item * sA;
  const int i = i0 + tx;
  double rm = 0.0;
#pragma unroll 4
  for (int c = ty; c < 64; c += 4) {
    const int j = j0 + c;
    double v = 0.0;
    if (i < rows && j < cols) v = fabs(Ab[i + static_cast<int64_t>(j) * lda]);
    rm = fmax(rm, v);
    tile[oz_tile_idx(c, tx)] = v;
  }
  rmax[ty][tx] = rm;
  __syncthreads();
  const int c = threadIdx.x >> 2, part = (threadIdx.x & 3) * 16;
  const double2* colp = reinterpret_cast<const double2*>(&tile[oz_tile_idx(c, part)]);
  double cm = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const double2 q = colp[u];
    cm = fmax(cm, fmax(q.x, q.y));
  }
  cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, 1));
  cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, 2));
  const int j = j0 + c;
  if ((threadIdx.x & 3) == 0 && j < cols && cm > 0.0)
    atomicMax(&eCol[static_cast<int64_t>(item) * cols + j], exp_of_max(cm));
  if (threadIdx.x < 64) {
    const double r = fmax(fmax(rmax[0][tx], rmax[1][tx]), fmax(rmax[2][tx], rmax[3][tx]));
    if (i < rows && r > 0.0) atomicMax(&eRow[static_cast<int64_t>(item) * rows + i], exp_of_max(r));
  }
}

// Slices of A in both K-major layouts (rows, cols multiples of 16):
//   sR[item][p] (tile_off with row i, K = cols) with eRow[i]   and
//   sC[item][p] (tile_off with row j, K = rows) with eCol[j].
// 64 x 64 tiles through shared memory, [col][row] with pitch 72 and 2 doubles
// of padding after every 16 rows: the column pass (thread = column, 16-row
// chunk; 16-byte reads) and the row pass (a warp = 32 consecutive rows of one
// 16-column chunk) are both bank-conflict free, and every warp stores whole
// 128-byte lines of the tiled layout.

__global__ void __launch_bounds__(256) oz_slice_a_kernel(const double* __restrict__ A, int64_t lda,
                                                         int64_t sA, int rows, int cols,
                                                         const int* __restrict__ eRow,
                                                         const int* __restrict__ eCol,
                                                         int8_t* __restrict__ sR,
                                                         int8_t* __restrict__ sC) {
  __shared__ __align__(16) double tile[64 * kOzTP];
  const int item = blockIdx.z;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const double* Ab = A + item * sA;
  {
    // all 16 loads of the thread in flight before the first shared-memory store
    const int r = threadIdx.x & 63, c0 = threadIdx.x >> 6;
    const double* src = Ab + (i0 + r) + static_cast<int64_t>(j0 + c0) * lda;
    const bool rok = i0 + r < rows;
    double v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      v[k] = (rok && j0 + c0 + 4 * k < cols) ? __ldg(src + static_cast<int64_t>(4 * k) * lda) : 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[oz_tile_idx(c0 + 4 * k, r)] = v[k];
  }
  __syncthreads();
  const int64_t plane = static_cast<int64_t>(rows) * cols;
  // column-major slices: column j0 + a, rows i0 + part .. +15
  {
    const int a = threadIdx.x >> 2, part = (threadIdx.x & 3) * 16;
    const int j = j0 + a;
    if (j < cols && i0 + part < rows) {
      const SliceScale sc(usable_exp(eCol[static_cast<int64_t>(item) * cols + j]));
      const double2* src = reinterpret_cast<const double2*>(&tile[oz_tile_idx(a, part)]);
      double v[16];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double2 q = src[u];
        v[2 * u] = q.x;
        v[2 * u + 1] = q.y;
      }
      uint4 out[kOzS];
      pack16([&](int u) { return v[u]; }, sc, out);
      int8_t* dst = sC + item * kOzS * plane + tile_off(j, (i0 + part) >> 4, rows);
#pragma unroll
      for (int p = 0; p < kOzS; ++p) *reinterpret_cast<uint4*>(dst + p * plane) = out[p];
    }
  }
  // row-major slices: row i0 + a, columns j0 + part .. +15
  {
    const int a = threadIdx.x & 63, part = (threadIdx.x >> 6) * 16;
    const int i = i0 + a;
    if (i < rows && j0 + part < cols) {
      const SliceScale sc(usable_exp(eRow[static_cast<int64_t>(item) * rows + i]));
      uint4 out[kOzS];
      pack16([&](int u) { return tile[oz_tile_idx(part + u, a)]; }, sc, out);
      int8_t* dst = sR + item * kOzS * plane + tile_off(i, (j0 + part) >> 4, cols);
#pragma unroll
      for (int p = 0; p < kOzS; ++p) *reinterpret_cast<uint4*>(dst + p * plane) = out[p];
    }
  }
}

// Exponents of the right operand B (K x N column-major): eB[item][j] (pre-set
// to kExpNone) by atomicMax over K ranges of kOzBK; one warp per column, one
// CTA per 8 columns and K range.
constexpr int kOzBK = 512;  // K per CTA of the B kernels (32 chunks of 16 x 8 columns = 256 threads)

__global__ void __launch_bounds__(256) oz_exp_b_kernel(const double* __restrict__ B, int64_t ldb,
                                                       int64_t sBst, int K, int N, int* eB) {
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5), item = blockIdx.z, lane = threadIdx.x & 31;
  const int k0 = blockIdx.y * kOzBK, k1 = min(K, k0 + kOzBK);
  const double* col = B + item * sBst + static_cast<int64_t>(j) * ldb;
  double m = 0.0;
  for (int k = k0 + lane; k < k1; k += 32) m = fmax(m, fabs(col[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0 && m > 0.0) atomicMax(&eB[static_cast<int64_t>(item) * N + j], exp_of_max(m));
}

// Slices of the right operand B (K % 16 == 0, N % 8 == 0) with eB's exponent
// per column: sB[item][p] in the tiled layout (tile_off with row = column j of
// B).  One CTA per 8 columns (one row group) and K range: the 8 x 512 block
// is staged through shared memory (coalesced loads along K; pitch 578 with 2
// doubles of padding per 16 keeps the 16-byte reads conflict free), then
// thread (r, c) packs the 16-byte chunk (column r, K chunk c), so a warp
// stores whole 128-byte lines.
constexpr int kOzBP = kOzBK + 2 * (kOzBK / 16) + 2;

__global__ void __launch_bounds__(256) oz_slice_b_kernel(const double* __restrict__ B, int64_t ldb,
                                                         int64_t sBst, int K, int N,
                                                         int8_t* __restrict__ sB,
                                                         const int* __restrict__ eB) {
  __shared__ __align__(16) double tile[8 * kOzBP];
  const int j0 = blockIdx.x * 8, k0 = blockIdx.y * kOzBK, item = blockIdx.z;
  const double* Bb = B + item * sBst + static_cast<int64_t>(j0) * ldb + k0;
  {
    double v[16];  // all 16 loads in flight
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int r = t >> 1, kk = (t & 1) * 256 + static_cast<int>(threadIdx.x);
      v[t] = (k0 + kk < K) ? __ldg(Bb + static_cast<int64_t>(r) * ldb + kk) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int r = t >> 1, kk = (t & 1) * 256 + static_cast<int>(threadIdx.x);
      tile[r * kOzBP + kk + 2 * (kk >> 4)] = v[t];
    }
  }
  __syncthreads();
  const int r = threadIdx.x & 7, cl = threadIdx.x >> 3;
  const int j = j0 + r, c = blockIdx.y * (kOzBK / 16) + cl;
  if (c >= (K >> 4)) return;
  const SliceScale sc(usable_exp(eB[static_cast<int64_t>(item) * N + j]));
  const double2* src = reinterpret_cast<const double2*>(&tile[r * kOzBP + 18 * cl]);
  double v[16];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const double2 q = src[u];
    v[2 * u] = q.x;
    v[2 * u + 1] = q.y;
  }
  const int64_t plane = static_cast<int64_t>(N) * K;
  uint4 out[kOzS];
  pack16([&](int u) { return v[u]; }, sc, out);
  int8_t* d = sB + item * kOzS * plane + tile_off(j, c, K);
#pragma unroll
  for (int p = 0; p < kOzS; ++p) *reinterpret_cast<uint4*>(d + p * plane) = out[p];
}

#ifdef RSVD_OZ_TRACE
// Per-CTA %globaltimer stamps (ns): entry, setup done, first stage landed,
// accumulators complete, exit.  Read by tools/probe/oz_trace.py.
constexpr int kOzTraceCtas = 8192;
__device__ unsigned long long g_oz_trace[kOzTraceCtas * 8];
__device__ __forceinline__ unsigned long long oz_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
  return t;
}
#define OZ_STAMP(i)                                                                       \
  do {                                                                                    \
    const unsigned lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);  \
    if (lin < kOzTraceCtas) g_oz_trace[lin * 8 + (i)] = oz_now();                         \
  } while (0)
#else
#define OZ_STAMP(i) \
  do {              \
  } while (0)
#endif

struct OzArgs {
  int M, N, K;
  int k_begin;     // this launch's K range: [k_begin, k_begin + K)
  int accumulate;  // C += (later K chunks) instead of C =
  double* C;
  int64_t ldc, strideC;
  const int* eA;  // per row of op(A): eA[item * M + i]
  const int* eB;  // per column of B:  eB[item * N + j]
};

constexpr int kOzBytesA = kOzS * kOzBM * kOzKC;
template <int BN>
struct OzTile {
  static constexpr int kBytesB = kOzS * BN * kOzKC;
  static constexpr int kStage = kOzBytesA + kBytesB;
  static constexpr int kSmem = kOzStages * kStage + 1024 + 512;
  static constexpr int kTmemCols = kOzS * BN > 256 ? 512 : 256;
};

// One 128 x BN tile of C per CTA.  Warp 0 lane 0: TMA producer; warp 1 lane 0:
// MMA issuer; warp 2 owns the TMEM allocation; all four warps drain TMEM
// (warp w reads lanes 32w..32w+31 = tile rows).
template <int BN>
__device__ __forceinline__ void oz_tile(const CUtensorMap& tmA, const CUtensorMap& tmB,
                                        const OzArgs& p, const int n0) {
  constexpr int kStage = OzTile<BN>::kStage, kTmemCols = OzTile<BN>::kTmemCols;
  extern __shared__ __align__(1024) unsigned char oz_smem[];
  const uint32_t raw = sm_addr(oz_smem);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  unsigned char* sgen = oz_smem + (sbase - raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sgen + kOzStages * kStage);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kOzStages + 1);
  int* seb = reinterpret_cast<int*>(bars + 2 * kOzStages + 2);  // eB - 12 of the tile's columns
  const uint32_t bar0 = sm_addr(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (kOzStages + s); };
  const uint32_t done_bar = bar0 + 8u * (2 * kOzStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * kOzBM, item = blockIdx.z;
  if (threadIdx.x == 0) OZ_STAMP(0);
  if (threadIdx.x >= 64) {
    const int col = n0 + static_cast<int>(threadIdx.x) - 64;
    seb[threadIdx.x - 64] =
        (col < p.N ? usable_exp(p.eB[static_cast<int64_t>(item) * p.N + col]) : 0) - 12;
  }
  const int nk = (p.K + kOzKC - 1) / kOzKC;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kOzStages; ++s) {
      mb_init(full_bar(s), 1);
      mb_init(empty_bar(s), 1);
    }
    mb_init(done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     sm_addr(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) OZ_STAMP(1);

  if (warp == 0 && lane == 0) {
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % kOzStages;
      if (kc >= kOzStages) mb_wait(empty_bar(s), ((kc / kOzStages) - 1) & 1);
      const uint32_t dA = sbase + s * kStage, dB = dA + kOzBytesA;
      mb_expect_tx(full_bar(s), kStage);
      tma_4d(dA, &tmA, 8 * (p.k_begin + kc * kOzKC), m0 >> 3, 0, item, full_bar(s));
      tma_4d(dB, &tmB, 8 * (p.k_begin + kc * kOzKC), n0 >> 3, 0, item, full_bar(s));
    }
  } else if (warp == 1 && lane == 0) {
    // kind::i8: D s32 (bits 4-5 = 2), A/B signed (bits 7, 10), K-major, N >> 3 at 17, M >> 4 at 24.
    // The S slices of B sit back to back in shared memory (slice q = rows
    // q*BN .. q*BN+BN-1 of one K-major tile) and diagonal d's accumulator at
    // TMEM columns d*BN, so A_p times slices q0 .. q0+nq-1 is ONE MMA of
    // N = nq*BN into columns (p+q0)*BN onward: up to 256-wide MMAs, which keep
    // the tensor core's shared-memory operand reads under the SM's bandwidth
    // (a 128 x 64 x 32 MMA is smem-bound at 48 cycles, 256-wide runs at N/2).
    constexpr uint32_t idesc0 = (2u << 4) | (1u << 7) | (1u << 10) |
                                (static_cast<uint32_t>(kOzBM >> 4) << 24);
    constexpr int kQ = 256 / BN;  // B slices per MMA
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % kOzStages;
      mb_wait(full_bar(s), (kc / kOzStages) & 1);
      if (kc == 0) OZ_STAMP(2);
      tc_fence_after();
      const uint32_t dA = sbase + s * kStage, dB = dA + kOzBytesA;
#pragma unroll
      for (int pa = 0; pa < kOzS; ++pa) {
        const uint64_t da = umma_desc_kmajor(dA + pa * (kOzBM * kOzKC));
#pragma unroll
        for (int q0 = 0; q0 < kOzS - pa; q0 += kQ) {
          const int nq = (kOzS - pa - q0) < kQ ? (kOzS - pa - q0) : kQ;
          const uint64_t db = umma_desc_kmajor(dB + q0 * (BN * kOzKC));
          const uint32_t idesc = idesc0 | (static_cast<uint32_t>((nq * BN) >> 3) << 17);
          tc_mma_i8(tmem + static_cast<uint32_t>((pa + q0) * BN), da, db, idesc,
                    (kc > 0 || pa > 0) ? 1u : 0u);
        }
      }
      tc_commit(empty_bar(s));
    }
    tc_commit(done_bar);
  }
  __syncwarp();
  mb_wait(done_bar, 0);
  __syncwarp();
  tc_fence_after();
  if (threadIdx.x == 0) OZ_STAMP(3);

  const int row = m0 + warp * 32 + lane;
  const bool row_ok = row < p.M;
  const int ea = row_ok ? usable_exp(p.eA[static_cast<int64_t>(item) * p.M + row]) : 0;
  double* Crow = p.C + item * p.strideC + row;
  const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  // Two halves of 32 columns: 7 TMEM loads each (x32), Horner over the
  // diagonals, one scaling by 2^(eA + eB - 12) built from its exponent bits
  // (ldexp only outside the normal range), then the stores (the values of a
  // later K chunk's C are read up front, 32 independent loads).
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    if (n0 + c0 >= p.N) break;
    double t[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) t[j] = 0.0;
#pragma unroll 1
    for (int d = kOzS - 1; d >= 0; --d) {
      uint32_t r[32];
      tc_ld32(lane_base + static_cast<uint32_t>(d * BN + c0), r);
#pragma unroll
      for (int j = 0; j < 32; ++j) t[j] = fma(t[j], 0.00390625, i32_to_f64(r[j]));
    }
    if (threadIdx.x == 0) OZ_STAMP(c0 ? 6 : 4);
    if (row_ok) {
      double* cp = Crow + static_cast<int64_t>(n0 + c0) * p.ldc;
      const int nc = min(min(32, BN - c0), p.N - n0 - c0);
      if (p.accumulate) {
        double cv[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) cv[j] = j < nc ? cp[j * p.ldc] : 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) t[j] = cv[j] + scale_pow2(t[j], ea + seb[c0 + j]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) t[j] = scale_pow2(t[j], ea + seb[c0 + j]);
      }
#pragma unroll
      for (int j = 0; j < 32; ++j, cp += p.ldc)
        if (j < nc) *cp = t[j];
    }
    if (threadIdx.x == 0 && c0 == 0) OZ_STAMP(5);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(kTmemCols)
                 : "memory");
  }
  if (threadIdx.x == 0) OZ_STAMP(7);
}

template <int BN>
__global__ void __launch_bounds__(128, 1) oz_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB,
                                                         const OzArgs p) {
  oz_tile<BN>(tmA, tmB, p, static_cast<int>(blockIdx.x) * BN);
}

// `wide` 64-column tiles and one 32-column tile for a remainder of N of at
// most 32 columns (l_p = 288 = 4 x 64 + 32: a fifth wide tile would be half
// padding, 10% of the launch).
__global__ void __launch_bounds__(128, 1) oz_gemm_mixed_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBw,
    const __grid_constant__ CUtensorMap tmBn, const OzArgs p, const int wide) {
  if (static_cast<int>(blockIdx.x) < wide)
    oz_tile<kOzBN>(tmA, tmBw, p, static_cast<int>(blockIdx.x) * kOzBN);
  else
    oz_tile<kOzBNs>(tmA, tmBn, p, wide * kOzBN);
}

PFN_cuTensorMapEncodeTiled_v12000 oz_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r{};
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &q, 12000, cudaEnableDefault,
                                         &r) == cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(q);
    cudaGetLastError();
  });
  return fn;
}

// Slices in the tiled layout [item][p][rows / 8][K / 16][8][16 bytes]: as a
// tensor of bytes {8 K (one row group, contiguous), rows / 8, S, batch}; a box
// {256 bytes = the two core matrices of one K step, box_rows / 8, S, 1} lands
// in shared memory exactly as umma_desc_kmajor expects.  No swizzle: every box
// row is 256 contiguous bytes of global memory (two full lines per request).
bool oz_map(CUtensorMap* map, const int8_t* base, int64_t K, int64_t rows, int64_t batch,
            int box_rows) {
  auto fn = oz_encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(8 * K), static_cast<cuuint64_t>(rows / 8),
                              static_cast<cuuint64_t>(kOzS), static_cast<cuuint64_t>(batch)};
  const cuuint64_t str[3] = {static_cast<cuuint64_t>(8 * K), static_cast<cuuint64_t>(K * rows),
                             static_cast<cuuint64_t>(K * rows * kOzS)};
  const cuuint32_t box[4] = {8 * kOzKC, static_cast<cuuint32_t>(box_rows / 8), kOzS, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(base), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

#ifdef RSVD_OZ_TRACE
void oz_trace_read(unsigned long long* out, int64_t n) {
  RSVD_CUDA(cudaMemcpyFromSymbol(out, g_oz_trace, sizeof(unsigned long long) * n));
}
#endif

bool oz_supported(int64_t rows, int64_t cols, int64_t K) {
  return rows % 16 == 0 && cols % 16 == 0 && K % 16 == 0 && rows < (1ll << 31) &&
         cols < (1ll << 31);
}

int64_t oz_slice_bytes(int64_t rows, int64_t cols, int64_t batch) {
  return kOzS * rows * cols * batch;
}

void oz_prepare_a(CMatRef A, int64_t rows, int64_t cols, int64_t batch, int8_t* sR, int8_t* sC,
                  int* eRow, int* eCol, cudaStream_t st) {
  RSVD_CUDA(cudaMemsetAsync(eRow, 0x80, sizeof(int) * rows * batch, st));
  RSVD_CUDA(cudaMemsetAsync(eCol, 0x80, sizeof(int) * cols * batch, st));
  dim3 grid(static_cast<unsigned>(ceil_div(cols, 64)), static_cast<unsigned>(ceil_div(rows, 64)),
            static_cast<unsigned>(batch));
  oz_exp_kernel<<<grid, 256, 0, st>>>(A.base, A.ld, A.stride, static_cast<int>(rows),
                                      static_cast<int>(cols), eRow, eCol);
  RSVD_LAUNCH("oz_exp_kernel");
  oz_slice_a_kernel<<<grid, 256, 0, st>>>(A.base, A.ld, A.stride, static_cast<int>(rows),
                                          static_cast<int>(cols), eRow, eCol, sR, sC);
  RSVD_LAUNCH("oz_slice_a_kernel");
}

void oz_slice_b(CMatRef B, int64_t K, int64_t N, int64_t batch, int8_t* sB, int* eB,
                cudaStream_t st) {
  RSVD_CUDA(cudaMemsetAsync(eB, 0x80, sizeof(int) * N * batch, st));
  dim3 grid(static_cast<unsigned>(N / 8), static_cast<unsigned>(ceil_div(K, kOzBK)),
            static_cast<unsigned>(batch));
  oz_exp_b_kernel<<<grid, 256, 0, st>>>(B.base, B.ld, B.stride, static_cast<int>(K),
                                        static_cast<int>(N), eB);
  RSVD_LAUNCH("oz_exp_b_kernel");
  oz_slice_b_kernel<<<grid, 256, 0, st>>>(B.base, B.ld, B.stride, static_cast<int>(K),
                                          static_cast<int>(N), sB, eB);
  RSVD_LAUNCH("oz_slice_b_kernel");
}

namespace {

template <int BN>
void oz_gemm_launch(int64_t M, int64_t N, int64_t K, const int8_t* sA, const int* eA,
                    const int8_t* sB, const int* eB, MatRef C, int64_t batch, cudaStream_t st) {
  CUtensorMap ma, mb;
  if (!oz_map(&ma, sA, K, M, batch, kOzBM) || !oz_map(&mb, sB, K, N, batch, BN))
    throw CudaError("oz_gemm: cuTensorMapEncodeTiled failed");
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    RSVD_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   OzTile<BN>::kSmem));
  });
  dim3 grid(static_cast<unsigned>(ceil_div(N, BN)), static_cast<unsigned>(ceil_div(M, kOzBM)),
            static_cast<unsigned>(batch));
  for (int64_t k0 = 0; k0 < K; k0 += kOzKChunk) {
    OzArgs a{static_cast<int>(M), static_cast<int>(N), static_cast<int>(std::min<int64_t>(kOzKChunk, K - k0)),
             static_cast<int>(k0), k0 > 0 ? 1 : 0, C.base, C.ld, C.stride, eA, eB};
    oz_gemm_kernel<BN><<<grid, 128, OzTile<BN>::kSmem, st>>>(ma, mb, a);
    RSVD_LAUNCH("oz_gemm_kernel");
  }
}

// Fraction of the SM-waves a grid of `tiles` one-CTA-per-SM tiles keeps busy.
double oz_fill(int64_t tiles) {
  const int64_t sm = num_sms();
  return static_cast<double>(tiles) / static_cast<double>(ceil_div(tiles, sm) * sm);
}

}  // namespace

// Output tile width for an M x N product over `batch` items: 64 columns (the
// most work per byte of A) unless the grid is a few thin waves that 32-wide
// tiles fill better (a 32-wide tile costs ~7% more tensor time per column).
int oz_tile_n(int64_t M, int64_t N, int64_t batch) {
  const int64_t mt = ceil_div(M, kOzBM) * batch;
  const double f64 = oz_fill(mt * ceil_div(N, kOzBN)), f32 = 0.93 * oz_fill(mt * ceil_div(N, kOzBNs));
  return f32 > f64 ? kOzBNs : kOzBN;
}

// Tensor-time efficiency of the grid oz_gemm would launch (1 = full waves of wide tiles).
double oz_grid_efficiency(int64_t M, int64_t N, int64_t batch) {
  const int64_t mt = ceil_div(M, kOzBM) * batch;
  return std::max(oz_fill(mt * ceil_div(N, kOzBN)), 0.93 * oz_fill(mt * ceil_div(N, kOzBNs)));
}

void oz_gemm(int64_t M, int64_t N, int64_t K, const int8_t* sA, const int* eA, const int8_t* sB,
             const int* eB, MatRef C, int64_t batch, cudaStream_t st) {
  if (oz_tile_n(M, N, batch) == kOzBNs) {
    oz_gemm_launch<kOzBNs>(M, N, K, sA, eA, sB, eB, C, batch, st);
    return;
  }
  const int64_t wide = N / kOzBN, rem = N - wide * kOzBN;
  if (wide == 0 || rem == 0 || rem > kOzBNs) {
    oz_gemm_launch<kOzBN>(M, N, K, sA, eA, sB, eB, C, batch, st);
    return;
  }
  CUtensorMap ma, mbw, mbn;
  if (!oz_map(&ma, sA, K, M, batch, kOzBM) || !oz_map(&mbw, sB, K, N, batch, kOzBN) ||
      !oz_map(&mbn, sB, K, N, batch, kOzBNs))
    throw CudaError("oz_gemm: cuTensorMapEncodeTiled failed");
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    RSVD_CUDA(cudaFuncSetAttribute(oz_gemm_mixed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   OzTile<kOzBN>::kSmem));
  });
  dim3 grid(static_cast<unsigned>(wide + 1), static_cast<unsigned>(ceil_div(M, kOzBM)),
            static_cast<unsigned>(batch));
  for (int64_t k0 = 0; k0 < K; k0 += kOzKChunk) {
    OzArgs a{static_cast<int>(M), static_cast<int>(N), static_cast<int>(std::min<int64_t>(kOzKChunk, K - k0)),
             static_cast<int>(k0), k0 > 0 ? 1 : 0, C.base, C.ld, C.stride, eA, eB};
    oz_gemm_mixed_kernel<<<grid, 128, OzTile<kOzBN>::kSmem, st>>>(ma, mbw, mbn, a,
                                                                  static_cast<int>(wide));
    RSVD_LAUNCH("oz_gemm_mixed_kernel");
  }
}

}  // namespace rsvd
