// FP64 tensor-core GEMM for the RSVD A-passes, Grams and small products.
//
// B200 has no tcgen05 f64 kind (ptxas rejects .kind::f64), so the FP64 tensor
// path is the warp-level DMMA `mma.sync.aligned.m16n8k4.row.col.f64`.  The
// probe in profiles/r01_fp64_peak.txt measured every DMMA shape at the same
// 37.1 TFLOP/s ceiling; m16n8k4 has the simplest fragments.
//
// Call sites replaced (reference): Eigen operator* -> OpenBLAS dgemm at
// factorize.cpp:68 (A*Omega), :70 (A^H*Q), :71 (A*Q), :86 (Q^H*A, computed
// here as its transpose A^T*Q), :92 (Q*U~), and the Gram/TRSM parts of the
// QR that replaces geqrf+orgqr (lapack.cpp:180-201).
//
//   NN: C(MxN) = A(MxK, col-major, lda) * B(KxN, col-major, ldb)
//   TN: C(MxN) = A^T * B, A stored K x M (col-major, lda)
//
// Tiling: CTA tile BM x BN over a K-slab BK, WARPS_M x WARPS_N warps, each
// warp owning (MT*16) x (NT*8) of C in registers.  Operands are staged
// global->shared with cp.async (16 B when every column start is 16 B aligned,
// 8 B otherwise) through a STAGES-deep ring.  Shared tiles are padded by 4
// doubles per column so the m16n8k4 fragment loads are bank-conflict free
// (pitch = 4 mod 16 words of 8 B).  Split-K writes per-split partials that a
// second kernel sums in fixed order: no atomics, bitwise reproducible.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace rsvd {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src, bool valid) {
  const int sz = valid ? BYTES : 0;  // src-size 0 => zero fill
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(sz));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(sz));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

struct GemmArgs {
  int64_t M, N, K;
  const double* A;
  int64_t lda, strideA;
  const double* B;
  int64_t ldb, strideB;
  double* C;
  int64_t ldc, strideC;
  int64_t batch;
  int splits;
  int64_t k_per_split;  // multiple of BK
  // Optional structure flags:
  //   colmapA (NN only): A(i, k) = A_stored(i, colmapA[item*colmap_stride + k])
  //   b_upper: B is upper triangular, output tile [n0, n0+BN) needs k < n0+BN
  //   c_upper: only tiles touching the upper triangle of C are computed
  const int* colmapA;
  int64_t colmap_stride;
  int b_upper;
  int c_upper;
  const int* item_mask;  // item_mask[b] == 0: skip item b
};

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool TRANS_A, int VEC>
struct GemmCfg {
  static constexpr int kThreads = WARPS_M * WARPS_N * 32;
  static constexpr int MT = BM / (WARPS_M * 16);
  static constexpr int NT = BN / (WARPS_N * 8);
  static_assert(MT * WARPS_M * 16 == BM, "BM");
  static_assert(NT * WARPS_N * 8 == BN, "BN");
  static_assert(BK % 4 == 0, "BK");
  // NN: A tile stored [k][i] (i contiguous), pitch BM+4.
  // TN: A tile stored [i][k] (k contiguous), pitch BK+4.
  static constexpr int kPitchA = TRANS_A ? (BK + 4) : (BM + 4);
  static constexpr int kTileA = TRANS_A ? BM * kPitchA : BK * kPitchA;
  // B tile stored [j][k] (k contiguous), pitch BK+4.
  static constexpr int kPitchB = BK + 4;
  static constexpr int kTileB = BN * kPitchB;
  static constexpr int kStageElems = kTileA + kTileB;
  static constexpr size_t kSmemBytes = sizeof(double) * kStageElems * STAGES;
};

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool TRANS_A, int VEC,
          int MINB>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32, MINB)
    dgemm_kernel(const GemmArgs p) {
  using Cfg = GemmCfg<BM, BN, BK, WARPS_M, WARPS_N, STAGES, TRANS_A, VEC>;
  constexpr int MT = Cfg::MT, NT = Cfg::NT;
  extern __shared__ __align__(16) double smem[];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % WARPS_M) * (MT * 16);
  const int wn = (warp / WARPS_M) * (NT * 8);

  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
  const int64_t bz = blockIdx.z;
  const int64_t item = bz / p.splits;
  const int split = static_cast<int>(bz % p.splits);
  if (p.c_upper && m0 >= n0 + BN) return;  // tile strictly below the diagonal
  if (p.item_mask && !p.item_mask[item]) return;
  const int64_t k_begin = split * p.k_per_split;
  int64_t k_end = min(p.K, k_begin + p.k_per_split);
  if (p.b_upper) k_end = min(k_end, n0 + BN);  // rows >= n0+BN of an upper B are zero
  const int64_t num_k_tiles = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;

  const double* __restrict__ Ab = p.A + item * p.strideA;
  const double* __restrict__ Bb = p.B + item * p.strideB;
  const int* __restrict__ cmap = p.colmapA ? p.colmapA + item * p.colmap_stride : nullptr;

  // ---- global -> shared staging of one K-slab --------------------------
  auto load_stage = [&](int stage, int64_t k0) {
    double* sA = smem + stage * Cfg::kStageElems;
    double* sB = sA + Cfg::kTileA;
    if constexpr (!TRANS_A) {
      // A(i, k) at Ab[i + k*lda]; tile BK columns of BM contiguous rows.
      constexpr int kChunksPerCol = BM / VEC;
      constexpr int kChunks = kChunksPerCol * BK;
#pragma unroll 4
      for (int c = tid; c < kChunks; c += Cfg::kThreads) {
        const int kk = c / kChunksPerCol;
        const int ii = (c % kChunksPerCol) * VEC;
        const int64_t gi = m0 + ii, gk = k0 + kk;
        const bool ok = (gi < p.M) && (gk < k_end);
        const int64_t col = (ok && cmap) ? cmap[gk] : gk;
        const double* src = ok ? Ab + gi + col * p.lda : Ab;
        cp_async<VEC * 8>(sA + kk * Cfg::kPitchA + ii, src, ok);
      }
    } else {
      // A_s(k, i) at Ab[k + i*lda]; tile BM columns of BK contiguous rows.
      constexpr int kChunksPerCol = BK / VEC;
      constexpr int kChunks = kChunksPerCol * BM;
#pragma unroll 4
      for (int c = tid; c < kChunks; c += Cfg::kThreads) {
        const int ii = c / kChunksPerCol;
        const int kk = (c % kChunksPerCol) * VEC;
        const int64_t gi = m0 + ii, gk = k0 + kk;
        const bool ok = (gi < p.M) && (gk < k_end);
        const double* src = ok ? Ab + gk + gi * p.lda : Ab;
        cp_async<VEC * 8>(sA + ii * Cfg::kPitchA + kk, src, ok);
      }
    }
    {
      // B(k, j) at Bb[k + j*ldb]; tile BN columns of BK contiguous rows.
      constexpr int kChunksPerCol = BK / VEC;
      constexpr int kChunks = kChunksPerCol * BN;
#pragma unroll 4
      for (int c = tid; c < kChunks; c += Cfg::kThreads) {
        const int jj = c / kChunksPerCol;
        const int kk = (c % kChunksPerCol) * VEC;
        const int64_t gj = n0 + jj, gk = k0 + kk;
        const bool ok = (gj < p.N) && (gk < k_end);
        const double* src = ok ? Bb + gk + gj * p.ldb : Bb;
        cp_async<VEC * 8>(sB + jj * Cfg::kPitchB + kk, src, ok);
      }
    }
  };

  double acc[MT][NT][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

  // Prologue: fill STAGES-1 slabs.
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < num_k_tiles) load_stage(s, k_begin + static_cast<int64_t>(s) * BK);
    cp_async_commit();
  }

  for (int64_t kt = 0; kt < num_k_tiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    // Prefetch slab kt + STAGES - 1 into the slot freed at iteration kt-1.
    {
      const int64_t nk = kt + STAGES - 1;
      if (nk < num_k_tiles) load_stage(static_cast<int>(nk % STAGES), k_begin + nk * BK);
      cp_async_commit();
    }
    const double* sA = smem + static_cast<int>(kt % STAGES) * Cfg::kStageElems;
    const double* sB = sA + Cfg::kTileA;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[MT][2], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int r = wm + i * 16 + g;
        if constexpr (!TRANS_A) {
          a[i][0] = sA[(kk + t) * Cfg::kPitchA + r];
          a[i][1] = sA[(kk + t) * Cfg::kPitchA + r + 8];
        } else {
          a[i][0] = sA[r * Cfg::kPitchA + kk + t];
          a[i][1] = sA[(r + 8) * Cfg::kPitchA + kk + t];
        }
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = sB[(wn + j * 8 + g) * Cfg::kPitchB + kk + t];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma_16x8x4(acc[i][j], a[i][0], a[i][1], b[j]);
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: C[row + col*ldc] ---------------------------------------
  // Split partials are laid out [split][item], each M x N.
  double* Cb = p.splits > 1 ? p.C + (static_cast<int64_t>(split) * p.batch + item) * p.strideC
                            : p.C + item * p.strideC;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int64_t r0 = m0 + wm + i * 16 + g;
      const int64_t c0 = n0 + wn + j * 8 + 2 * t;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = r0 + h * 8;
        if (r < p.M) {
          if (c0 < p.N) Cb[r + c0 * p.ldc] = acc[i][j][2 * h];
          if (c0 + 1 < p.N) Cb[r + (c0 + 1) * p.ldc] = acc[i][j][2 * h + 1];
        }
      }
    }
  }
}

// Fixed-order split reduction: C[item](i,j) = sum_s partial[s][item](i,j).
__global__ void splitk_reduce_kernel(const double* __restrict__ partial, int64_t M, int64_t N,
                                     int splits, int64_t batch, double* __restrict__ C,
                                     int64_t ldc, int64_t strideC, const int* __restrict__ mask) {
  const int64_t per = M * N;
  const int64_t total = per * batch;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t item = e / per;
    const int64_t rem = e - item * per;
    if (mask && !mask[item]) continue;
    const int64_t j = rem / M, i = rem - j * M;
    double s = 0.0;
    for (int sp = 0; sp < splits; ++sp) s += partial[(sp * batch + item) * per + rem];
    C[item * strideC + i + j * ldc] = s;
  }
}

// C(r, c) = C(c, r) for r > c (square items).
__global__ void mirror_upper_kernel(double* __restrict__ C, int64_t n, int64_t ldc,
                                    int64_t strideC, int64_t batch, const int* __restrict__ mask) {
  const int64_t per = n * n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < per * batch;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t item = e / per, rem = e - item * per;
    if (mask && !mask[item]) continue;
    const int64_t c = rem / n, r = rem - c * n;
    if (r > c) C[item * strideC + r + c * ldc] = C[item * strideC + c + r * ldc];
  }
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool TRANS_A, int VEC,
          int MINB = 1>
void launch_cfg(const GemmArgs& a, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, BK, WARPS_M, WARPS_N, STAGES, TRANS_A, VEC>;
  auto kern = dgemm_kernel<BM, BN, BK, WARPS_M, WARPS_N, STAGES, TRANS_A, VEC, MINB>;
  static std::atomic<uint64_t> attr_set{0};
  once_per_device(attr_set, [&] {
    RSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(Cfg::kSmemBytes)));
  });
  dim3 grid(static_cast<unsigned>(ceil_div(a.N, BN)), static_cast<unsigned>(ceil_div(a.M, BM)),
            static_cast<unsigned>(a.batch * a.splits));
  kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes, st>>>(a);
  RSVD_LAUNCH("dgemm_kernel");
}

// Tile configurations: BK = 16, 3-stage cp.async ring (<= 108 KB of shared memory).
constexpr int kBK = 16;
constexpr int kStages = 3;

struct Choice {
  int bm, bn;
  int splits;
  int64_t kps;
};

Choice choose(int64_t M, int64_t N, int64_t K, int64_t batch, bool allow80 = true) {
  Choice c{128, 64, 1, 0};
  // Prefer a BN that covers N with little padding waste.
  // The 128 x 96 tile (TMA path) is the efficient one: take it unless 64-wide
  // tiles cover N with strictly less padding.
  const int64_t w64 = round_up(N, 64), w96 = round_up(N, 96);
  if (N <= 32) c.bn = 32;
  else if (N <= 64) c.bn = 64;
  // 96-wide tiles take the TMA kernel (~25% faster per flop): worth up to
  // 12.5% padding (N = 256: lift 1.97 -> 1.70 ms on C4).
  else c.bn = (8 * w96 <= 9 * w64) ? 96 : 64;
  c.bm = (M <= 64) ? 64 : 128;
  // 128 x 80 TMA tiles where they cut the padding by more than 12.5%
  // (l_p = 160, C2 / TEBD sectors: 160 columns instead of 192).
  const int64_t w80 = round_up(N, 80);
  if (allow80 && N > 64 && c.bm == 128 && 9 * w80 < 8 * std::min(w96, w64)) c.bn = 80;
  const int64_t tiles = ceil_div(M, c.bm) * ceil_div(N, c.bn) * batch;
  const int64_t slots = 2 * num_sms();  // two resident CTAs per SM
  int64_t splits = 1;
  // Fewer than ~4 waves of output tiles: split K so that the last wave is as
  // full as possible (fewer splits among nearly equal), each split keeping
  // >= 256 of K -- or 64 for very few tiles (single small matrices, C1) --
  // and >= 512 once the tiles alone fill a wave.  (C3 / C5's A^T Q: 96 tiles
  // -> 3 splits, 0.97 of a wave instead of 4 splits, 1.3 waves; a 4-item C4
  // batch, 384 tiles -> 3 splits.)
  if (tiles < 4 * slots) {
    const int64_t kmin = (tiles * 8 <= num_sms() && K >= 1024) ? 64 : (tiles < slots ? 256 : 512);
    const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(64, K / kmin));
    double best_eff = -1.0;
    for (int64_t sp = 1; sp <= smax; ++sp) {
      const int64_t ctas = tiles * sp;
      const double eff = static_cast<double>(ctas) / static_cast<double>(ceil_div(ctas, slots) * slots);
      if (eff > best_eff * 1.02) best_eff = eff, splits = sp;
      if (ctas >= 4 * slots) break;
    }
  }
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, 64));
  int64_t kps = round_up(ceil_div(K, splits), kBK);
  splits = ceil_div(K, kps);
  c.splits = static_cast<int>(std::max<int64_t>(1, splits));
  c.kps = kps;
  return c;
}

template <bool TRANS_A, int VEC>
void dispatch(const Choice& c, const GemmArgs& a, cudaStream_t st) {
  if (c.bm == 128 && c.bn == 96)  // 128 registers: two CTAs per SM (profiles/r01_gemm_tune.txt)
    launch_cfg<128, 96, kBK, 4, 2, kStages, TRANS_A, VEC, 2>(a, st);
  else if (c.bm == 128 && c.bn == 64)
    launch_cfg<128, 64, kBK, 4, 2, kStages, TRANS_A, VEC>(a, st);
  else if (c.bm == 128 && c.bn == 32)
    launch_cfg<128, 32, kBK, 4, 2, kStages, TRANS_A, VEC>(a, st);
  else if (c.bm == 64 && c.bn == 96)
    launch_cfg<64, 96, kBK, 2, 4, kStages, TRANS_A, VEC>(a, st);
  else if (c.bm == 64 && c.bn == 64)
    launch_cfg<64, 64, kBK, 2, 4, kStages, TRANS_A, VEC>(a, st);
  else
    launch_cfg<64, 32, kBK, 2, 4, kStages, TRANS_A, VEC>(a, st);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

// Split-K count of the symmetric 96 x 96 Gram tiling: the upper tiles times
// the splits should fill whole waves of the 2 x SMs resident CTAs (C4: 192
// tiles -> 3 splits = 1.95 waves instead of 2 splits = 1.3 waves), each split
// keeping >= 256 of K.
int64_t sq96_splits(int64_t M, int64_t K, int64_t batch) {
  const int64_t t = M / 96, tiles = t * (t + 1) / 2 * batch;
  const int64_t slots = 2 * num_sms();
  const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(64, K / 256));
  if (tiles >= 4 * slots) return 1;
  int64_t best = 1;
  double best_eff = -1.0;
  for (int64_t sp = 1; sp <= smax; ++sp) {
    const int64_t ctas = tiles * sp;
    const double eff = static_cast<double>(ctas) / static_cast<double>(ceil_div(ctas, slots) * slots);
    // prefer fuller waves; among (nearly) equal, fewer splits (less partial traffic)
    if (eff > best_eff * 1.02) best_eff = eff, best = sp;
    if (ctas >= 3 * slots) break;
  }
  return best;
}

int64_t dgemm_partial_elems(bool trans_a, int64_t M, int64_t N, int64_t K, int64_t batch) {
  const Choice c = choose(M, N, K, batch);
  int64_t splits = c.splits;
  if (trans_a && M == N && M % 96 == 0) {  // the 96 x 96 Gram tiling of dgemm_ex
    const int64_t sp = sq96_splits(M, K, batch);
    splits = std::max(splits, ceil_div(K, round_up(ceil_div(K, sp), kBK)));
  }
  return splits > 1 ? splits * batch * M * N : 0;
}

void dgemm(bool trans_a, int64_t M, int64_t N, int64_t K, CMatRef A, CMatRef B, MatRef C,
           int64_t batch, double* partial, int64_t partial_capacity, cudaStream_t st) {
  dgemm_ex(trans_a, M, N, K, A, B, C, batch, partial, partial_capacity, GemmOpts{}, st);
}

void dgemm_ex(bool trans_a, int64_t M, int64_t N, int64_t K, CMatRef A, CMatRef B, MatRef C,
              int64_t batch, double* partial, int64_t partial_capacity, const GemmOpts& opt,
              cudaStream_t st) {
  if (M <= 0 || N <= 0 || batch <= 0) return;
  // 16-byte aligned operands with even strides: the TMA tiles can take them.
  const bool tma_ok = aligned16(A.base) && aligned16(B.base) && A.ld % 2 == 0 && B.ld % 2 == 0 &&
                      (batch == 1 || (A.stride % 2 == 0 && B.stride % 2 == 0)) && !opt.colmapA &&
                      (trans_a || M % 16 == 0);
  Choice c = choose(M, N, K, batch, tma_ok);
  // Symmetric Gram of a 96-multiple width: 96 x 96 TMA tiles (the 128 x 96
  // tile leaves a partial row tile and computes ~40% more than the upper half).
  // (Only when the TMA path can take the operands: an odd row count, e.g. a
  // tsvd of a 37 x 53 block, has an odd leading dimension.)
  const bool tma_operands = aligned16(A.base) && aligned16(B.base) && A.ld % 2 == 0 &&
                            B.ld % 2 == 0 && (batch == 1 || (A.stride % 2 == 0 && B.stride % 2 == 0));
  const bool sq96 = opt.c_upper && trans_a && M == N && M % 96 == 0 && !opt.colmapA &&
                    tma_operands;
  if (sq96) {
    int64_t splits = sq96_splits(M, K, batch);
    int64_t kps = round_up(ceil_div(K, splits), kBK);
    splits = ceil_div(K, kps);
    c.bm = 96, c.bn = 96, c.splits = static_cast<int>(splits), c.kps = kps;
  }
  if (K <= 0) c.splits = 1, c.kps = kBK;
  const int64_t need = c.splits > 1 ? static_cast<int64_t>(c.splits) * batch * M * N : 0;
  if (need > partial_capacity) {
    c.splits = 1;
    c.kps = round_up(std::max<int64_t>(K, 1), kBK);
  }
  GemmArgs a{};
  a.M = M, a.N = N, a.K = K;
  a.A = A.base, a.lda = A.ld, a.strideA = A.stride;
  a.B = B.base, a.ldb = B.ld, a.strideB = B.stride;
  a.batch = batch;
  a.splits = c.splits;
  a.k_per_split = c.kps;
  a.colmapA = trans_a ? nullptr : opt.colmapA;
  a.colmap_stride = opt.colmap_stride;
  a.b_upper = opt.b_upper ? 1 : 0;
  a.c_upper = (opt.c_upper && M == N) ? 1 : 0;
  a.item_mask = opt.item_mask;
  if (c.splits > 1) {
    a.C = partial, a.ldc = M, a.strideC = M * N;
  } else {
    a.C = C.base, a.ldc = C.ld, a.strideC = C.stride;
  }
  // 16-byte cp.async needs every staged column start 16 B aligned.
  const bool vec2 = aligned16(A.base) && aligned16(B.base) && (A.ld % 2 == 0) &&
                    (B.ld % 2 == 0) && (A.stride % 2 == 0) && (B.stride % 2 == 0) &&
                    (trans_a ? true : (M % 2 == 0)) && (K % 2 == 0) && (c.kps % 2 == 0);
  const bool tma_done =
      !a.colmapA && ((c.bm == 128 && (c.bn == 96 || c.bn == 80)) || sq96) &&
      dgemm_tma(trans_a, M, N, K, A, B, a.C, a.ldc, a.strideC, batch, c.splits, c.kps,
                a.c_upper != 0, opt.item_mask, a.b_upper != 0, st, sq96 ? 1 : (c.bn == 80 ? 2 : 0));
  if (sq96 && !tma_done) throw CudaError("dgemm: 96x96 Gram tile needs the TMA path");
  if (c.bn == 80 && !tma_done) throw CudaError("dgemm: 128x80 tile needs the TMA path");
  if (tma_done) {
  } else if (trans_a) {
    if (vec2) dispatch<true, 2>(c, a, st);
    else dispatch<true, 1>(c, a, st);
  } else {
    if (vec2) dispatch<false, 2>(c, a, st);
    else dispatch<false, 1>(c, a, st);
  }
  if (c.splits > 1) {
    const int64_t total = M * N * batch;
    const int threads = 256;
    const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, threads), 8 * num_sms()));
    splitk_reduce_kernel<<<blocks, threads, 0, st>>>(partial, M, N, c.splits, batch, C.base, C.ld,
                                                     C.stride, opt.item_mask);
    RSVD_LAUNCH("splitk_reduce_kernel");
  }
  if (a.c_upper) {  // symmetric result: mirror the upper triangle
    const int64_t total = M * M * batch;
    const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 8 * num_sms()));
    mirror_upper_kernel<<<blocks, 256, 0, st>>>(C.base, M, C.ld, C.stride, batch, opt.item_mask);
    RSVD_LAUNCH("mirror_upper_kernel");
  }
}

}  // namespace rsvd
