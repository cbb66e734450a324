// Probe: one-warp 32 x 32 Cholesky (registers, smem row broadcast) + R^{-1}
// by per-lane backward substitution from shared memory.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int P = 36;
__device__ long long g_mid;

__device__ __forceinline__ int fdb4(double (&a)[32], double* Rd, double* Dt, int lane) {
  // Rd: rows of R (Rd[k*P + j] = R[k][j]); Dt first holds R^T rows
  // (Dt[j*P + i] = R[i][j]) for the forward substitution Z = R^{-T}, then
  // (after the sweep) X = R^{-1} = Z^T row-major.
  int brk = 32;
  double z[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double akk = __shfl_sync(0xffffffffu, a[k], k);
    if (brk == 32 && !(akk > 1e-300)) brk = k;
    double rk, inv = 1.0;
    if (brk == 32) {
      inv = rsqrt(akk);
      rk = (lane == k) ? akk * inv : (lane > k ? a[k] * inv : 0.0);
    } else {
      rk = (lane == k) ? 1.0 : 0.0;
    }
    a[k] = rk;
    Rd[k * P + lane] = rk;
    Dt[lane * P + k] = rk;
    __syncwarp();
    const double rkm = lane > k ? rk : 0.0;
    const double2* row = reinterpret_cast<const double2*>(Rd + k * P);
#pragma unroll
    for (int i2 = (k + 1) / 2; i2 < 16; ++i2) {
      const double2 v = row[i2];
      if (2 * i2 > k) a[2 * i2] = fma(-v.x, rkm, a[2 * i2]);
      if (2 * i2 + 1 > k) a[2 * i2 + 1] = fma(-v.y, rkm, a[2 * i2 + 1]);
    }
    // z[k] = (delta_k,lane - sum_{i<k} R[i][k] z[i]) / R[k][k]
    const double2* col = reinterpret_cast<const double2*>(Dt + k * P);
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int i2 = 0; 2 * i2 < k; ++i2) {
      const double2 v = col[i2];
      s0 = fma(v.x, z[2 * i2], s0);
      if (2 * i2 + 1 < k) s1 = fma(v.y, z[2 * i2 + 1], s1);
    }
    z[k] = ((lane == k ? 1.0 : 0.0) - (s0 + s1)) * inv;
  }
  if (lane == 0) g_mid = clock64();
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) Dt[lane * P + k] = z[k];  // X[lane][k] = Z[k][lane]
  __syncwarp();
  return brk;
}

__global__ void probe(const double* W, int ld, double* out, long long* cyc) {
  __shared__ __align__(16) double Rd[32 * P], Dt[32 * P];
  const int lane = threadIdx.x;
  double a[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = __ldcg(W + i + lane * ld);
  double dummy = 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) dummy += a[i];
  if (dummy == 12345.0) out[0] = 1.0;
  long long t1 = clock64();
  const int brk = fdb4(a, Rd, Dt, lane);
  long long t2 = clock64();
  double err = 0.0;  // (R X)[lane][c] = sum_k R[lane][k] X[k][c]
  for (int c = 0; c < 32; ++c) {
    double s = 0.0;
    for (int k = 0; k < 32; ++k) s += (k >= lane ? Rd[lane * P + k] : 0.0) * Dt[k * P + c];
    err = fmax(err, fabs(s - (lane == c ? 1.0 : 0.0)));
  }
  // and R^T R = G
  double err2 = 0.0;
  for (int c = 0; c < 32; ++c) {
    double s = 0.0;
    for (int k = 0; k < 32; ++k) s += (k <= lane ? Rd[k * P + lane] : 0.0) * (k <= c ? Rd[k * P + c] : 0.0);
    err2 = fmax(err2, fabs(s - W[lane + c * ld]));
  }
  out[lane] = fmax(err, err2) + 100 * brk;
  if (lane == 0) { cyc[0] = t2 - t1; cyc[1] = g_mid - t1; }
}

int main() {
  const int ld = 288;
  static double h[288 * 32];
  for (int j = 0; j < 32; ++j)
    for (int i = 0; i < 288; ++i) h[i + j * ld] = (i < 32) ? (i == j ? 40.0 : 1.0 / (1 + i + j)) : 0.0;
  double *W, *out;
  long long* cyc;
  cudaMalloc(&W, sizeof(h));
  cudaMalloc(&out, 256);
  cudaMalloc(&cyc, 64);
  cudaMemcpy(W, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    probe<<<1, 32>>>(W, ld, out, cyc);
    long long c;
    double o[32];
    long long cc[2];
    cudaMemcpy(cc, cyc, 16, cudaMemcpyDeviceToHost);
    c = cc[0];
    printf("  cholesky part %lld\n", cc[1]);
    cudaMemcpy(o, out, 256, cudaMemcpyDeviceToHost);
    double e = 0;
    for (int i = 0; i < 32; ++i) e = e > o[i] ? e : o[i];
    printf("chol(smem bcast) + inverse %lld cycles, max err %.3e (brk*100 added)\n", c, e);
  }
  return 0;
}
