// Phase timing of the fused CholeskyQR kernel (chol.cu fcqr_kernel) from
// %globaltimer stamps of CTA 0 (built with RSVD_FCQR_TRACE), plus the event
// time per launch.  Build + run:
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -DRSVD_FCQR_TRACE \
//     --expt-relaxed-constexpr -o /tmp/fcqr_trace tools/probe/fcqr_trace.cu && /tmp/fcqr_trace
#include "../../paper_1710_01463_b200/csrc/chol.cu"

#include <cstdio>
#include <random>
#include <vector>

namespace rsvd {
std::atomic<uint64_t> g_kernel_launches{0};
}

static void run(int rows, int ell, int ellp, int batch, int reps) {
  using namespace rsvd;
  const size_t n = static_cast<size_t>(rows) * ellp * batch;
  std::vector<double> h(n);
  std::mt19937_64 g(rows * 131 + ell);
  std::normal_distribution<double> nd;
  for (auto& x : h) x = nd(g);
  double *Y, *Q, *G0, *XS;
  int* rank;
  cudaMalloc(&Y, n * 8);
  cudaMalloc(&Q, n * 8);
  cudaMalloc(&G0, static_cast<size_t>(ellp) * ellp * batch * 8);
  cudaMalloc(&rank, batch * 4);
  cudaMalloc(&XS, fcqr_xscratch_elems(ellp, batch) * 8);
  cudaMemcpy(Y, h.data(), n * 8, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w)
    launch_fused_cqr(Y, rows, (int64_t)rows * ellp, Q, rows, (int64_t)rows * ellp, G0, nullptr, XS, rank,
                     rows, ell, ellp, 1e-13, batch, st);
  cudaEventRecord(e0, st);
  for (int r = 0; r < reps; ++r)
    launch_fused_cqr(Y, rows, (int64_t)rows * ellp, Q, rows, (int64_t)rows * ellp, G0, nullptr, XS, rank,
                     rows, ell, ellp, 1e-13, batch, st);
  cudaEventRecord(e1, st);
  cudaStreamSynchronize(st);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long tr[64];
  cudaMemcpyFromSymbol(tr, g_fq_trace, sizeof(tr));
  int rk = 0;
  cudaMemcpy(&rk, rank, 4, cudaMemcpyDeviceToHost);
  printf("rows %d ell %d ellp %d batch %d: %.2f us/launch, rank %d; %s\n", rows, ell, ellp, batch,
         1000.0 * ms / reps, rk, cudaGetErrorString(cudaGetLastError()));
  printf("   first chunk staged +%.2f us, first chunk computed +%.2f us\n", (tr[14] - tr[0]) / 1000.0,
         (tr[15] - tr[0]) / 1000.0);
  const char* names[14] = {"start", "gram", "clu-reduce", "pivfloor+f0", "J0", "J1", "J2", "J3", "J4", "-",
                           "chol-done", "W-prod", "clu-copy", "apply"};
  unsigned long long prev = tr[0];
  for (int i = 1; i < 14; ++i) {
    if (tr[i] == 0 || tr[i] < tr[0] || tr[i] - tr[0] > 100000000ull) continue;
    printf("   %-12s +%7.2f us (at %7.2f)\n", names[i], (tr[i] - prev) / 1000.0, (tr[i] - tr[0]) / 1000.0);
    prev = tr[i];
  }
  cudaMemset(Y, 0, 0);
  unsigned long long z[64] = {0};
  cudaMemcpyToSymbol(g_fq_trace, z, sizeof(z));
  cudaFree(Y);
  cudaFree(Q);
  cudaFree(G0);
  cudaFree(rank);
  cudaStreamDestroy(st);
}

int main() {
  run(1024, 74, 96, 1, 50);   // C1
  run(1024, 74, 96, 1, 50);
  run(256, 138, 160, 256, 20);  // C2
  run(256, 138, 160, 1, 20);
  run(1024, 138, 160, 1, 20);
  run(4096, 138, 160, 1, 20);
  run(300, 90, 96, 1, 20);
  return 0;
}
