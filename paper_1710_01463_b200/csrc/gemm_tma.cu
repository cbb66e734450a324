// TMA-fed FP64 DMMA GEMM for the RSVD A-passes and Grams (sm_100a).
//
// Same math and tiling as gemm_f64.cu (C tile 128 x 96, eight warps of
// 32 x 48, mma.sync m16n8k4 .f64), but the operand tiles are moved by the
// Tensor Memory Accelerator:
//   * one elected thread issues cp.async.bulk.tensor loads of whole K-slabs
//     (BK = 16 doubles = one 128-byte swizzle span) into a STAGES-deep ring;
//   * full[s] mbarriers carry the transaction bytes, empty[s] mbarriers collect
//     one arrival per consumer warp, so the main loop has no __syncthreads and
//     no per-thread address arithmetic for the copies;
//   * tiles land with the 128B swizzle (16-byte chunk ^= row mod 8), which makes
//     the m16n8k4 fragment loads bank-conflict free without padding.
// Box layouts (innermost first):
//   B   (K x N, K contiguous):          box {16 k, BN j}        -> row j
//   A^T (TN, stored K x M, K contiguous): box {16 k, BM i}      -> row i
//   A   (NN, stored M x K, M contiguous): viewed as 4-D {16 i_lo, K, M/16, batch},
//                                        box {16, 16 k, BM/16}  -> row i_hi*16 + k
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"

namespace rsvd {
namespace {

constexpr int kTBK = 16;  // doubles per 128-byte swizzle row

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5}], [%6];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

struct TmaArgs {
  int64_t M, N, K;
  double* C;
  int64_t ldc, strideC;
  int64_t batch;
  int splits;
  int64_t k_per_split;
  int c_upper, b_upper;
  const int* item_mask;
};

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool TRANS_A>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32, 2)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB, const TmaArgs p) {
  constexpr int kWarps = WARPS_M * WARPS_N;
  constexpr int MT = BM / (WARPS_M * 16);
  constexpr int NT = BN / (WARPS_N * 8);
  constexpr uint32_t kBytesA = BM * kTBK * 8, kBytesB = BN * kTBK * 8;
  constexpr uint32_t kStage = kBytesA + kBytesB;  // multiple of 1024
  static_assert(kBytesA % 1024 == 0 && kBytesB % 1024 == 0, "1024-byte aligned tiles");
  extern __shared__ unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  const uint32_t sbase = (smem_addr(smem_raw) + 1023u) & ~1023u;
  const unsigned char* sgen = smem_raw + (sbase - smem_addr(smem_raw));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % WARPS_M) * (MT * 16);
  const int wn = (warp / WARPS_M) * (NT * 8);
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
  const int64_t bz = blockIdx.z;
  const int64_t item = bz / p.splits;
  const int split = static_cast<int>(bz % p.splits);
  if (p.c_upper && m0 >= n0 + BN) return;
  if (p.item_mask && !p.item_mask[item]) return;
  const int64_t k_begin = split * p.k_per_split;
  int64_t k_end = min(p.K, k_begin + p.k_per_split);
  if (p.b_upper) k_end = min(k_end, n0 + BN);
  const int num_k_tiles = k_end > k_begin ? static_cast<int>((k_end - k_begin + kTBK - 1) / kTBK) : 0;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_addr(&full_bar[s]), 1);
      mbar_init(smem_addr(&empty_bar[s]), kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  __syncthreads();

  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    const uint32_t fb = smem_addr(&full_bar[s]);
    const uint32_t dA = sbase + s * kStage, dB = dA + kBytesA;
    const int k0 = static_cast<int>(k_begin + static_cast<int64_t>(kt) * kTBK);
    mbar_expect_tx(fb, kStage);
    if constexpr (TRANS_A)
      tma_load_3d(dA, &tmA, k0, static_cast<int>(m0), static_cast<int>(item), fb);
    else
      tma_load_4d(dA, &tmA, 0, k0, static_cast<int>(m0 / 16), static_cast<int>(item), fb);
    tma_load_3d(dB, &tmB, k0, static_cast<int>(n0), static_cast<int>(item), fb);
  };
  if (tid == 0)
    for (int kt = 0; kt < STAGES - 1 && kt < num_k_tiles; ++kt) issue(kt);

  double acc[MT][NT][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

  // Fragment rows are (multiple of 8) + g, so the swizzle XOR of a K-contiguous
  // tile row is the per-thread constant g << 4.
  const uint32_t xg = static_cast<uint32_t>(g) << 4;
  const uint32_t baseA = TRANS_A ? static_cast<uint32_t>(wm + g) * 128u
                                 : static_cast<uint32_t>(wm >> 4) * 2048u + g * 8u;
  const uint32_t baseB = static_cast<uint32_t>(wn + g) * 128u;

  for (int kt = 0; kt < num_k_tiles; ++kt) {
    if (tid == 0) {
      const int nk = kt + STAGES - 1;
      if (nk < num_k_tiles) {
        if (nk >= STAGES)
          mbar_wait(smem_addr(&empty_bar[nk % STAGES]), ((nk / STAGES) - 1) & 1);
        issue(nk);
      }
    }
    const int s = kt % STAGES;
    mbar_wait(smem_addr(&full_bar[s]), (kt / STAGES) & 1);
    const unsigned char* tA = sgen + s * kStage;
    const unsigned char* tB = tA + kBytesA;
#pragma unroll
    for (int kk = 0; kk < kTBK; kk += 4) {
      const int k = kk + t;
      double a[MT][2], b[NT];
      const uint32_t kx = (static_cast<uint32_t>(k) * 8u) ^ xg;  // K-contiguous tiles
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t off;
          if constexpr (TRANS_A) {
            off = baseA + (i * 16 + h * 8) * 128 + kx;
          } else {  // row i_hi*16 + k, 16-byte chunk (i_lo/2) ^ (k & 7)
            off = (baseA + i * 2048 + h * 64 + k * 128) ^ ((static_cast<uint32_t>(k) & 7u) << 4);
          }
          a[i][h] = *reinterpret_cast<const double*>(tA + off);
        }
#pragma unroll
      for (int j = 0; j < NT; ++j)
        b[j] = *reinterpret_cast<const double*>(tB + baseB + j * 1024 + kx);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma_16x8x4(acc[i][j], a[i][0], a[i][1], b[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_addr(&empty_bar[s]));
  }

  double* Cb = p.splits > 1 ? p.C + (static_cast<int64_t>(split) * p.batch + item) * p.strideC
                            : p.C + item * p.strideC;
#pragma unroll
  for (int i = 0; i < MT; ++i)
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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
  });
  return fn;
}

bool make_map(CUtensorMap* map, const double* base, int rank, const cuuint64_t* dims,
              const cuuint64_t* strides_bytes, const cuuint32_t* box) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUresult r =
      fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), dims,
         strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

constexpr int kBM = 128, kBN = 96, kWM = 4, kWN = 2;

// 3 stages (86 KB) keep two CTAs per SM; measured faster than 4 (one CTA).
constexpr int kTmaStages = 3;

template <int STAGES, bool TRANS_A, int BM = kBM, int BN = kBN, int WM = kWM, int WN = kWN>
void launch(const CUtensorMap& ma, const CUtensorMap& mb, const TmaArgs& a, cudaStream_t st) {
  auto kern = dgemm_tma_kernel<BM, BN, WM, WN, STAGES, TRANS_A>;
  const size_t bytes = static_cast<size_t>(STAGES) * (BM + BN) * kTBK * 8 + 1024;
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    RSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(bytes)));
  });
  dim3 grid(static_cast<unsigned>(ceil_div(a.N, BN)), static_cast<unsigned>(ceil_div(a.M, BM)),
            static_cast<unsigned>(a.batch * a.splits));
  kern<<<grid, WM * WN * 32, bytes, st>>>(ma, mb, a);
  RSVD_LAUNCH("dgemm_tma_kernel");
}

}  // namespace

bool dgemm_tma(bool trans_a, int64_t M, int64_t N, int64_t K, CMatRef A, CMatRef B, double* C,
               int64_t ldc, int64_t strideC, int64_t batch, int splits, int64_t kps, bool c_upper,
               const int* item_mask, bool b_upper, cudaStream_t st, int tile) {
  // tile 0: 128 x 96 (8 warps as 4 x 2); tile 1: 96 x 96 (2 x 4 warps) for the
  // symmetric Gram of a 96-multiple l_p (no partial 128-row tiles); tile 2:
  // 128 x 80 (4 x 2 warps of 32 x 40) for 160-wide operands.
  const int bm = tile == 1 ? 96 : kBM, bn = tile == 1 ? 96 : (tile == 2 ? 80 : kBN);
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  if (!al16(A.base) || !al16(B.base)) return false;
  if (A.ld % 2 || B.ld % 2 || A.stride % 2 || B.stride % 2) return false;
  if (kps % kTBK) return false;
  if (!trans_a && M % 16) return false;
  if (batch > 65535 || M > (1ll << 31) || N > (1ll << 31) || K > (1ll << 31)) return false;
  const int64_t sA = batch > 1 ? A.stride : M * K, sB = batch > 1 ? B.stride : N * K;
  if (batch > 1 && (A.stride <= 0 || B.stride <= 0)) return false;
  CUtensorMap ma, mb;
  {
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(N),
                                static_cast<cuuint64_t>(batch)};
    const cuuint64_t str[2] = {static_cast<cuuint64_t>(B.ld) * 8, static_cast<cuuint64_t>(sB) * 8};
    const cuuint32_t box[3] = {kTBK, static_cast<cuuint32_t>(bn), 1};
    if (!make_map(&mb, B.base, 3, dims, str, box)) return false;
  }
  if (trans_a) {
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M),
                                static_cast<cuuint64_t>(batch)};
    const cuuint64_t str[2] = {static_cast<cuuint64_t>(A.ld) * 8, static_cast<cuuint64_t>(sA) * 8};
    const cuuint32_t box[3] = {kTBK, static_cast<cuuint32_t>(bm), 1};
    if (!make_map(&ma, A.base, 3, dims, str, box)) return false;
  } else {
    const cuuint64_t dims[4] = {16, static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M / 16),
                                static_cast<cuuint64_t>(batch)};
    const cuuint64_t str[3] = {static_cast<cuuint64_t>(A.ld) * 8, 128,
                               static_cast<cuuint64_t>(sA) * 8};
    const cuuint32_t box[4] = {16, kTBK, static_cast<cuuint32_t>(bm / 16), 1};
    if (!make_map(&ma, A.base, 4, dims, str, box)) return false;
  }
  TmaArgs a{M, N, K, C, ldc, strideC, batch, splits, kps, c_upper ? 1 : 0, b_upper ? 1 : 0,
            item_mask};
  if (tile == 1) {
    if (trans_a) launch<3, true, 96, 96, 2, 4>(ma, mb, a, st);
    else launch<3, false, 96, 96, 2, 4>(ma, mb, a, st);
    return true;
  }
  if (tile == 2) {
    if (trans_a) launch<kTmaStages, true, 128, 80, 4, 2>(ma, mb, a, st);
    else launch<kTmaStages, false, 128, 80, 4, 2>(ma, mb, a, st);
    return true;
  }
  if (trans_a) launch<kTmaStages, true>(ma, mb, a, st);
  else launch<kTmaStages, false>(ma, mb, a, st);
  return true;
}

}  // namespace rsvd
