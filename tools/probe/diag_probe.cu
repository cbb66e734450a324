// Probe: cycle cost of the 32 x 32 diagonal Cholesky + inverse (one warp),
// split into its parts.  nvcc -arch=sm_100a -O3 -o diag_probe diag_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kInvPitch = 36;
#include "fdb.inc"

__global__ void probe(double* W, int ld, double* out, long long* cyc, int variant) {
  __shared__ double Rd[32 * kInvPitch], Dt[32 * kInvPitch];
  const int lane = threadIdx.x;
  double a[32];
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = __ldcg(W + i + lane * ld);
  long long t1 = clock64();
  int brk = 0;
  if (variant == 0) brk = factor_diag_block(a, W, ld, 32, 0, 1e-300, Rd, Dt, lane);
  long long t2 = clock64();
  out[lane] = Dt[lane * kInvPitch + lane] + brk;
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}

int main() {
  const int n = 32, ld = 288;
  double h[288 * 32];
  for (int j = 0; j < 32; ++j)
    for (int i = 0; i < 288; ++i) h[i + j * ld] = (i < 32) ? (i == j ? 40.0 : 1.0 / (1 + i + j)) : 0.0;
  double *W, *out;
  long long* cyc;
  cudaMalloc(&W, sizeof(h));
  cudaMalloc(&out, 256);
  cudaMalloc(&cyc, 64);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(W, h, sizeof(h), cudaMemcpyHostToDevice);
    probe<<<1, 32>>>(W, ld, out, cyc, 0);
    long long c[2];
    cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
    printf("loads %lld cycles, factor+inverse %lld cycles\n", c[0], c[1]);
  }
  (void)n;
  return 0;
}
