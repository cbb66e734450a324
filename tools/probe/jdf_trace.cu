// Phase sums of CTA 0 of the dataflow Jacobi (jacobi.cu jacobi_df_kernel,
// built with RSVD_JDF_TRACE) and the time per launch_jacobi call.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -DRSVD_JDF_TRACE \
//     --expt-relaxed-constexpr -o tools/probe/jdf_trace tools/probe/jdf_trace.cu
#ifdef JSRC
#include JSRC
#else
#include "../../paper_1710_01463_b200/csrc/jacobi.cu"
#endif

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

namespace rsvd {
std::atomic<uint64_t> g_kernel_launches{0};
}

static void run(int ell, int ellp, int batch, int reps, int which = 0) {
  using namespace rsvd;
  const size_t sq = static_cast<size_t>(ellp) * ellp, n = sq * batch;
  std::vector<double> h(n, 0.0);
  std::mt19937_64 g(ell * 7 + batch);
  std::normal_distribution<double> nd;
  // upper-triangular H with a graded diagonal, like R^T of a CholeskyQR
  for (int b = 0; b < batch; ++b)
    for (int j = 0; j < ell; ++j)
      for (int i = 0; i < ell; ++i) h[b * sq + i + j * ellp] = nd(g) * std::pow(j + 1.0, -1.5);
  double *H0, *H, *J;
  unsigned* flags;
  int* sweeps;
  cudaMalloc(&H0, n * 8);
  cudaMalloc(&H, n * 8);
  cudaMalloc(&J, n * 8);
  cudaMalloc(&flags, jacobi_flag_elems(batch, ellp) * 4);
  cudaMalloc(&sweeps, batch * 4);
  cudaMemcpy(H0, h.data(), n * 8, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float tot = 0;
  for (int r = 0; r < reps + 2; ++r) {
    cudaMemcpyAsync(H, H0, n * 8, cudaMemcpyDeviceToDevice, st);
    cudaEventRecord(e0, st);
    if (which == 0 || which == 3) launch_jacobi(H, J, ell, ellp, 30, sweeps, flags, batch, st);
#ifndef JSRC
    else if (which == 1) launch_df_t<144, 4>(H, J, ell, ellp, 30, sweeps, flags, batch, st);
    else launch_df_t<96, 3>(H, J, ell, ellp, 30, sweeps, flags, batch, st);
#endif
    cudaEventRecord(e1, st);
    cudaStreamSynchronize(st);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2) tot += ms;
  }
  unsigned long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#ifdef RSVD_JDF_TRACE
  cudaMemcpyFromSymbol(tr, g_jdf_trace, sizeof(tr));
#endif
#ifdef RSVD_JCLU_TRACE
  if (which == 3) {
    cudaMemcpyFromSymbol(tr, g_jclu_trace, sizeof(tr));
    const double nt = tr[5] ? double(tr[5]) : 1.0;
    printf("   clug CTA0: %llu tasks; per task us: stage %.2f gram+reduce %.2f rot %.2f apply %.2f grid-barrier %.2f\n",
           tr[5], tr[0] / nt / 1e3, tr[1] / nt / 1e3, tr[2] / nt / 1e3, tr[3] / nt / 1e3, tr[4] / nt / 1e3);
  }
#endif
  int sw = 0;
  cudaMemcpy(&sw, sweeps, 4, cudaMemcpyDeviceToHost);
  {  // item 0: W = H0 J (columns orthogonal), J orthogonal
    std::vector<double> w(sq), jj(sq);
    cudaMemcpy(w.data(), H, sq * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(jj.data(), J, sq * 8, cudaMemcpyDeviceToHost);
    double ow = 0, oj = 0, rec = 0, nrm = 0;
    for (int a = 0; a < ell; ++a)
      for (int b2 = 0; b2 < ell; ++b2) {
        double sw2 = 0, sj = 0, na = 0, nb = 0, hj = 0;
        for (int i = 0; i < ell; ++i) {
          sw2 += w[i + a * ellp] * w[i + b2 * ellp];
          na += w[i + a * ellp] * w[i + a * ellp];
          nb += w[i + b2 * ellp] * w[i + b2 * ellp];
          sj += jj[i + a * ellp] * jj[i + b2 * ellp];
          hj += h[i + b2 * ellp] * jj[b2 + a * ellp] * 0;  // (unused)
        }
        if (a != b2) ow = std::max(ow, std::fabs(sw2) / std::sqrt(na * nb));
        oj = std::max(oj, std::fabs(sj - (a == b2 ? 1.0 : 0.0)));
      }
    for (int a = 0; a < ell; ++a)
      for (int i = 0; i < ell; ++i) {
        double v = 0;
        for (int k = 0; k < ell; ++k) v += h[i + k * ellp] * jj[k + a * ellp];
        rec = std::max(rec, std::fabs(v - w[i + a * ellp]));
        nrm = std::max(nrm, std::fabs(w[i + a * ellp]));
      }
    printf("   item0: max |cos(w_a, w_b)| %.2e, |J^T J - I| %.2e, |H0 J - W| / max|W| %.2e\n", ow, oj, rec / nrm);
  }
  printf("[%d] ell %d ellp %d batch %d: %.3f ms/call, sweeps(item0) %d; %s\n", which, ell, ellp, batch, tot / reps, sw,
         cudaGetErrorString(cudaGetLastError()));
  const double nt = tr[5] ? double(tr[5]) : 1.0;
  printf("   CTA0: %llu tasks; per task us: wait %.2f gram %.2f rot %.2f apply %.2f fin %.2f\n", tr[5],
         tr[0] / nt / 1e3, tr[1] / nt / 1e3, tr[2] / nt / 1e3, tr[3] / nt / 1e3, tr[4] / nt / 1e3);
  cudaFree(H0);
  cudaFree(H);
  cudaFree(J);
  cudaFree(flags);
  cudaFree(sweeps);
  cudaStreamDestroy(st);
}

int main() {
  if (getenv("JDF_SMALL")) {
    run(74, 96, 1, 5, 0);    // C1 (shared-memory kernel)
    run(74, 96, 1, 5, 3);
    run(40, 64, 512, 5, 0);
    run(96, 96, 64, 5, 0);
    run(20, 32, 1000, 5, 0);
    run(5, 32, 3, 5, 0);
    return 0;
  }
  if (getenv("JDF_ONLY_CLU")) {
    run(272, 288, 1, 5, 3);  // C3 (cluster kernel)
    run(544, 544, 1, 3, 3);  // C5
    run(74, 96, 1, 5, 3);    // C1
    run(74, 96, 1, 5, 2);    // C1 through the dataflow kernel
    run(74, 96, 1, 5, 1);
    run(272, 288, 1, 5, 2);  // C3 through the dataflow kernel
    return 0;
  }
  run(138, 160, 256, 5, 0);  // C2
  run(276, 288, 32, 5, 0);   // C4
  run(138, 160, 64, 5, 0);
  run(40, 64, 512, 5, 0);
  return 0;
}
