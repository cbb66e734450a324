// FP64 throughput probe for sm_100a: DMMA shapes vs DFMA.  Used once to pick
// the GEMM micro-kernel; results recorded under profiles/.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void dmma_loop(double* out, int iters) {
  double acc[8][4];
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; i++) { a[i] = 1.0 + threadIdx.x * 1e-9 + i; }
#pragma unroll
  for (int i = 0; i < 4; i++) { b[i] = 0.5 + i * 1e-9; }
#pragma unroll
  for (int c = 0; c < 8; c++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[c][j] = 0.0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int c = 0; c < 8; c++) {
      if (SHAPE == 0) {  // m8n8k4: A 1, B 1, C 2
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a[c]), "d"(b[0]));
      } else if (SHAPE == 1) {  // m16n8k4: A 2, B 1, C 4
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[c]), "d"(a[(c + 1) & 7]), "d"(b[0]));
      } else if (SHAPE == 2) {  // m16n8k8: A 4, B 2, C 4
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[c]), "d"(a[(c + 1) & 7]), "d"(a[(c + 2) & 7]), "d"(a[(c + 3) & 7]), "d"(b[0]), "d"(b[1]));
      } else if (SHAPE == 3) {  // m16n8k16: A 8, B 4, C 4
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      } else {  // DFMA: 4 independent fma per chain
#pragma unroll
        for (int j = 0; j < 4; j++) acc[c][j] = fma(a[c], b[j], acc[c][j]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; c++)
#pragma unroll
    for (int j = 0; j < 4; j++) s += acc[c][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int SHAPE>
void run(const char* name, double flops_per_warp_instr, int blocks, int threads) {
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  int iters = 4096;
  dmma_loop<SHAPE><<<blocks, threads>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  dmma_loop<SHAPE><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double warps = (double)blocks * threads / 32;
  double flops = warps * iters * 8 * flops_per_warp_instr;
  printf("%-10s blocks=%d threads=%d  %.3f ms  %.2f TFLOP/s  err=%s\n", name, blocks, threads, ms,
         flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clock=%d kHz\n", sms, clk);
  for (int tpb : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps;
      run<0>("m8n8k4", 2.0 * 8 * 8 * 4, blocks, tpb);
      run<1>("m16n8k4", 2.0 * 16 * 8 * 4, blocks, tpb);
      run<2>("m16n8k8", 2.0 * 16 * 8 * 8, blocks, tpb);
      run<3>("m16n8k16", 2.0 * 16 * 8 * 16, blocks, tpb);
      run<4>("dfma", 2.0 * 32 * 4, blocks, tpb);
    }
  }
  return 0;
}
