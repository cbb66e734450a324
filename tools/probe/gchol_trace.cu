// Per-block phase timing of the grid / cluster Cholesky (chol.cu gchol_kernel,
// built with RSVD_GCHOL_TRACE) through launch_pchol, plus the time per call.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -DRSVD_GCHOL_TRACE \
//     --expt-relaxed-constexpr -o tools/probe/gchol_trace tools/probe/gchol_trace.cu
#include "../../paper_1710_01463_b200/csrc/chol.cu"

#include <cstdio>
#include <random>
#include <vector>

namespace rsvd {
std::atomic<uint64_t> g_kernel_launches{0};
}

static void run(int ell, int ellp, int batch, int reps) {
  using namespace rsvd;
  const size_t sq = static_cast<size_t>(ellp) * ellp;
  // G = Y^T Y + I-ish, SPD
  std::vector<double> h(sq * batch, 0.0);
  std::mt19937_64 g(ell);
  std::normal_distribution<double> nd;
  const int rows = ell + 8;
  std::vector<double> y(static_cast<size_t>(rows) * ell);
  for (auto& v : y) v = nd(g);
  for (int i = 0; i < ell; ++i)
    for (int j = 0; j < ell; ++j) {
      double s = 0;
      for (int k = 0; k < rows; ++k) s += y[k + i * rows] * y[k + j * rows];
      for (int b = 0; b < batch; ++b) h[b * sq + i + j * ellp] = s;
    }
  double *G0, *G, *T, *scr;
  int *rank, *perm;
  cudaMalloc(&G0, sq * batch * 8);
  cudaMalloc(&G, sq * batch * 8);
  cudaMalloc(&T, sq * batch * 8);
  cudaMalloc(&scr, pchol_scratch_elems(ellp, batch) * 8);
  cudaMalloc(&rank, batch * 4);
  cudaMalloc(&perm, batch * ellp * 4);
  cudaMemcpy(G0, h.data(), sq * batch * 8, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float tot = 0;
  for (int r = 0; r < reps + 2; ++r) {
    cudaMemcpyAsync(G, G0, sq * batch * 8, cudaMemcpyDeviceToDevice, st);
    cudaEventRecord(e0, st);
    launch_pchol(G, T, nullptr, scr, rank, perm, ell, ellp, 1e-13, false, batch, st);
    cudaEventRecord(e1, st);
    cudaStreamSynchronize(st);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2) tot += ms;
  }
  {  // item `batch - 1`: R^T R = G0 and R T = I (upper parts)
    const size_t off = sq * (batch - 1);
    std::vector<double> R(sq), Tm(sq);
    cudaMemcpy(R.data(), G + off, sq * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(Tm.data(), T + off, sq * 8, cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0, gm = 0;
    for (int i = 0; i < ell; ++i)
      for (int j = i; j < ell; ++j) {
        double s1 = 0, s2 = 0;
        for (int k = 0; k <= i; ++k) s1 += R[k + i * ellp] * R[k + j * ellp];
        for (int k = i; k <= j; ++k) s2 += R[i + k * ellp] * Tm[k + j * ellp];
        gm = std::max(gm, std::fabs(h[off + i + j * ellp]));
        e1 = std::max(e1, std::fabs(s1 - h[off + i + j * ellp]));
        e2 = std::max(e2, std::fabs(s2 - (i == j ? 1.0 : 0.0)));
      }
    printf("   check: |R^T R - G|/max|G| %.2e, |R T - I| %.2e\n", e1 / gm, e2);
  }
  unsigned long long tr[160];
  cudaMemcpyFromSymbol(tr, g_gc_trace, sizeof(tr));
  int rk = 0;
  cudaMemcpy(&rk, rank, 4, cudaMemcpyDeviceToHost);
  printf("ell %d ellp %d batch %d: %.1f us/call, rank %d; %s\n", ell, ellp, batch, 1000.0 * tot / reps, rk,
         cudaGetErrorString(cudaGetLastError()));
  const int nb = (ell + 31) / 32;
  printf("   setup %.2f us; factor0 %.2f us\n", (tr[1] - tr[0]) / 1e3, (tr[2] - tr[1]) / 1e3);
  double sb = 0, sc = 0;
  for (int J = 0; J < nb; ++J) {
    const double b = (tr[3 + 2 * J] - tr[2 + 2 * J]) / 1e3;
    const double c = J + 1 < nb ? (tr[4 + 2 * J] - tr[3 + 2 * J]) / 1e3 : 0.0;
    sb += b;
    sc += c;
    if (J < 3 || J + 2 >= nb) printf("   J %2d: B %.2f us, C %.2f us\n", J, b, c);
  }
  printf("   sum B %.1f us, sum C %.1f us\n", sb, sc);
  cudaFree(G0);
  cudaFree(G);
  cudaFree(T);
  cudaFree(scr);
  cudaFree(rank);
  cudaFree(perm);
  cudaStreamDestroy(st);
}

int main() {
  run(272, 288, 1, 5);   // C3
  run(544, 544, 1, 5);   // C5
  run(276, 288, 32, 5);  // C4
  run(276, 288, 5, 5);   // C4 host chunk
  run(90, 96, 3, 5);     // one CTA per item (MODE 2)
  return 0;
}
