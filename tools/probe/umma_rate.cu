// Probe: tcgen05.mma issue rate on one SM per CTA (148 CTAs), operands from
// shared memory (SS) with various N, swizzles and kinds.  Prints cycles per
// MMA and MAC/cycle/SM.  nvcc -gencode arch=compute_100a,code=sm_100a -o umma_rate umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sm_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, int sbo, int layout) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) |
         (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46) | (static_cast<uint64_t>(layout) << 61);
}

template <int KIND, int N, int LAYOUT>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sm_addr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(sm_addr(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const int sbo = LAYOUT == 6 ? 256 : (LAYOUT == 2 ? 1024 : 512);
    const uint32_t a = sm_addr(smem), b = a + 32 * 1024;
    const uint64_t da = desc(a, sbo, LAYOUT), db = desc(b, sbo, LAYOUT);
    uint32_t idesc;
    if (KIND == 0) idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24);
    else idesc = (1u << 4) | ((N >> 3) << 17) | ((128 >> 4) << 24);  // f8f6f4 e4m3, f32 accum
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t col = (it & 1) ? 256u : 0u;
      if (KIND == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem + col), "l"(da), "l"(db), "r"(idesc), "r"(1u) : "memory");
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem + col), "l"(da), "l"(db), "r"(idesc), "r"(1u) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(sm_addr(&bar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(sm_addr(&bar)) : "memory");
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}

template <int KIND, int N, int LAYOUT>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  auto k = rate_kernel<KIND, N, LAYOUT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 4096;
  k<<<148, 128, 64 * 1024>>>(iters, d);
  k<<<148, 128, 64 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double cyc = avg / iters;
  printf("%-28s N=%3d cycles/mma=%7.2f  MAC/cyc/SM=%7.0f  %s\n", name, N, cyc, 128.0 * N * 32 / cyc,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 64, 6>("i8 SW32");
  run<0, 128, 6>("i8 SW32");
  run<0, 256, 6>("i8 SW32");
  run<0, 64, 2>("i8 SW128");
  run<0, 128, 2>("i8 SW128");
  run<0, 256, 2>("i8 SW128");
  run<0, 64, 4>("i8 SW64");
  run<1, 64, 6>("f8 SW32");
  run<1, 128, 6>("f8 SW32");
  run<1, 256, 6>("f8 SW32");
  run<1, 256, 2>("f8 SW128");
  return 0;
}
