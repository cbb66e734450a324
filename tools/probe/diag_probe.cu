// Cycle count of the one-warp 32 x 32 diagonal-block Cholesky + inverse
// (chol.cu factor_diag_block) and of alternative formulations.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
//     -o tools/probe/diag_probe tools/probe/diag_probe.cu
#include "../../paper_1710_01463_b200/csrc/chol.cu"

#include <cstdio>
#include <random>
#include <vector>

namespace rsvd {
std::atomic<uint64_t> g_kernel_launches{0};

// Cholesky only (no inverse), same broadcast scheme.
__device__ __forceinline__ int chol_only(double (&a)[32], double* Rd, int lane, double thresh) {
  int brk = 32;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double akk = __shfl_sync(0xffffffffu, a[k], k);
    if (brk == 32 && !(akk > thresh)) brk = k;
    const double inv = rsqrt(akk);
    const double rk = (lane == k) ? akk * inv : (lane > k ? a[k] * inv : 0.0);
    a[k] = rk;
    Rd[k * kInvPitch + lane] = rk;
    __syncwarp();
    const double rkm = lane > k ? rk : 0.0;
    const double2* row = reinterpret_cast<const double2*>(Rd + k * kInvPitch);
#pragma unroll
    for (int i2 = (k + 1) / 2; i2 < 16; ++i2) {
      const double2 v = row[i2];
      if (2 * i2 > k) a[2 * i2] = fma(-v.x, rkm, a[2 * i2]);
      if (2 * i2 + 1 > k) a[2 * i2 + 1] = fma(-v.y, rkm, a[2 * i2 + 1]);
    }
  }
  return brk;
}
}  // namespace rsvd

using namespace rsvd;

__global__ void kdiag(const double* G, double* out, long long* cyc, int mode, int reps) {
  __shared__ double W[32 * kInvPitch], Rd[32 * kInvPitch], Dt[32 * kInvPitch];
  const int lane = threadIdx.x;
  double acc = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double a[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = G[i + lane * 32] + r * 1e-300;
    int brk;
    if (mode == 0)
      brk = factor_diag_block(a, W, kInvPitch, 32, 0, 1e-300, Rd, Dt, lane);
    else
      brk = chol_only(a, Rd, lane, 1e-300);
    acc += a[lane & 31] + Dt[lane] + brk;
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) *cyc = (t1 - t0) / reps;
  out[lane] = acc;
}

__global__ void kcheck(const double* G, double* Rout, double* Dout) {
  __shared__ double W[32 * kInvPitch], Rd[32 * kInvPitch], Dt[32 * kInvPitch];
  const int lane = threadIdx.x;
  double a[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = G[i + lane * 32];
  factor_diag_block(a, W, kInvPitch, 32, 0, 1e-300, Rd, Dt, lane);
  __syncwarp();
  for (int i = 0; i < 32; ++i) {
    Rout[i + lane * 32] = i <= lane ? W[i + lane * kInvPitch] : 0.0;
    Dout[i + lane * 32] = Dt[i * kInvPitch + lane];  // D(i, lane)
  }
}

__global__ void klat(double x0, double* out, long long* cyc) {
  __shared__ double sh[64];
  const int lane = threadIdx.x;
  double x = x0 + lane * 1e-3;
  long long t[8];
  t[0] = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; ++i) x = fma(x, 0.999999, 1e-7);
  t[1] = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; ++i) x = rsqrt(x) + 0.5;
  t[2] = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; ++i) x = sqrt(x) + 0.5;
  t[3] = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; ++i) x = 1.5 / x + 0.5;
  t[4] = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) * 1.0000001;
  t[5] = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; ++i) {
    sh[lane] = x;
    __syncwarp();
    x = sh[(lane + 3) & 31] * 1.0000001;
    __syncwarp();
  }
  t[6] = clock64();
  if (lane == 0)
    for (int i = 0; i < 6; ++i) cyc[i] = (t[i + 1] - t[i]) / 100;
  out[lane] = x;
}

int main() {
  {
    double* o;
    long long* c;
    cudaMalloc(&o, 64 * 8);
    cudaMalloc(&c, 8 * 8);
    klat<<<1, 32>>>(1.3, o, c);
    klat<<<1, 32>>>(1.3, o, c);
    cudaDeviceSynchronize();
    long long h[6];
    cudaMemcpy(h, c, 6 * 8, cudaMemcpyDeviceToHost);
    printf("latency (cycles per dependent op incl. loop): dfma %lld rsqrt %lld sqrt %lld div %lld shfl+mul %lld sts-sync-lds+mul %lld\n",
           h[0], h[1], h[2], h[3], h[4], h[5]);
  }
  std::mt19937_64 g(5);
  std::normal_distribution<double> nd;
  std::vector<double> y(64 * 32), G(32 * 32, 0.0);
  for (auto& v : y) v = nd(g);
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j)
      for (int k = 0; k < 64; ++k) G[i + j * 32] += y[k + i * 64] * y[k + j * 64];
  double *dG, *dout;
  long long* dc;
  cudaMalloc(&dG, 32 * 32 * 8);
  cudaMalloc(&dout, 32 * 8);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dG, G.data(), 32 * 32 * 8, cudaMemcpyHostToDevice);
  {  // check: R^T R = G and R D = I for the factor_diag_block outputs
    double *dW, *dD;
    cudaMalloc(&dW, 32 * 32 * 8);
    cudaMalloc(&dD, 32 * 32 * 8);
    kcheck<<<1, 32>>>(dG, dW, dD);
    cudaDeviceSynchronize();
    std::vector<double> R(1024), D(1024);
    cudaMemcpy(R.data(), dW, 1024 * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(D.data(), dD, 1024 * 8, cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0, gmax = 0;
    for (int i = 0; i < 32; ++i)
      for (int j = 0; j < 32; ++j) {
        double s1 = 0, s2 = 0;
        for (int k = 0; k < 32; ++k) {
          s1 += (k <= i ? R[k + i * 32] : 0) * (k <= j ? R[k + j * 32] : 0);
          s2 += (k >= i ? R[i + k * 32] : 0) * D[k + j * 32];
        }
        gmax = std::max(gmax, std::fabs(G[i + j * 32]));
        e1 = std::max(e1, std::fabs(s1 - G[i + j * 32]));
        e2 = std::max(e2, std::fabs(s2 - (i == j ? 1.0 : 0.0)));
      }
    printf("maxerr |R^T R - G|/max|G| %.2e, |R D - I| %.2e\n", e1 / gmax, e2);
  }
  for (int mode = 0; mode < 2; ++mode) {
    kdiag<<<1, 32>>>(dG, dout, dc, mode, 20);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("mode %d: %lld cycles per 32x32 factor (%s)\n", mode, c, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
