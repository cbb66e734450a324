// Probe: which part of the one-warp 32 x 32 Cholesky dominates.
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void probe(const double* W, int ld, double* out, long long* cyc) {
  const int lane = threadIdx.x;
  double a[32], z[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = __ldcg(W + i + lane * ld);
  long long t1 = clock64();
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double akk = __shfl_sync(0xffffffffu, a[k], k);
    double inv = 1.0;
    if (V & 1) {
      inv = rsqrt(akk);
      const double rkk = akk * inv;
      const double rk = (lane == k) ? rkk : (lane > k ? a[k] * inv : 0.0);
      a[k] = rk;
#pragma unroll
      for (int i = k + 1; i < 32; ++i) {
        const double rki = __shfl_sync(0xffffffffu, rk, i);
        if (lane > k) a[i] -= rki * rk;
      }
    }
    if (V & 2) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int i = 0; i < k; ++i) {
        const double p = __shfl_sync(0xffffffffu, a[i], k) * z[i];
        switch (i & 3) {
          case 0: s0 += p; break;
          case 1: s1 += p; break;
          case 2: s2 += p; break;
          default: s3 += p; break;
        }
      }
      z[k] = ((lane == k ? 1.0 : 0.0) - ((s0 + s1) + (s2 + s3))) * inv;
    } else {
      z[k] = inv;
    }
  }
  long long t2 = clock64();
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) acc += a[i] + z[i];
  out[lane] = acc;
  if (lane == 0) cyc[0] = t2 - t1;
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
  long long c;
  for (int rep = 0; rep < 2; ++rep) {
    probe<1><<<1, 32>>>(W, ld, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("chol only     %lld\n", c);
    probe<2><<<1, 32>>>(W, ld, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("z only        %lld\n", c);
    probe<3><<<1, 32>>>(W, ld, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("chol + z      %lld\n", c);
  }
  return 0;
}
