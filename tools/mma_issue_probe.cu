// Is the ~50-cycle per-MMA issue cost the compiler's waterfall loop (ELECT +
// R2UR.BROADCAST per tcgen05.mma) or the instruction itself?  Variant with all
// operands uniform (TMEM base assumed 0: the only allocation of the CTA).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ inline uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
template <bool TS, int N, int MODE>
__global__ void rate(int reps, long long* out, uint32_t* tm_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) *tm_out = slot;
  if (warp == 0) {
    const uint32_t a = su32(smem), b = su32(smem + 32768);
    const uint64_t ad = sdesc(a, 128, 256), bd = sdesc(b, 128, 256);
    long long t0 = clock64();
    if (MODE == 0) {
      // whole warp runs the loop; elect inside each iteration, operands uniform
      for (int r = 0; r < reps; ++r) {
        const uint32_t d = 128u + (uint32_t)((r & 3) * N);
        const uint32_t ta = (uint32_t)(r & 7) * 8u;
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, 1, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
            "r"(ta), "l"(bd), "n"(idesc(N))
            : "memory");
      }
    } else {
      // one elected thread runs the loop, operands uniform-derived
      uint32_t pred;
      asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
      if (pred) {
        for (int r = 0; r < reps; ++r) {
          const uint32_t d = 128u + (uint32_t)((r & 3) * N);
          const uint32_t ta = (uint32_t)(r & 7) * 8u;
          if (TS)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                         "r"(ta), "l"(bd), "n"(idesc(N)) : "memory");
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                         "l"(ad), "l"(bd), "n"(idesc(N)) : "memory");
        }
      }
      __syncwarp();
    }
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
      asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)));
      out[0] = clock64() - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
template <bool TS, int N, int MODE>
void run(long long* d, uint32_t* t) {
  cudaFuncSetAttribute(rate<TS, N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int reps = 4096;
  rate<TS, N, MODE><<<1, 128, 70 * 1024>>>(reps, d, t);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0; uint32_t ht = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&ht, t, 4, cudaMemcpyDeviceToHost);
  printf("%s N=%3d mode %d: %6.2f cycles/instr  (tmem base %u, %s)\n", TS ? "TS" : "SS", N, MODE, (double)h / reps, ht,
         cudaGetErrorString(e));
}
int main() {
  long long* d; uint32_t* t;
  cudaMalloc(&d, 64); cudaMalloc(&t, 64);
  run<true, 32, 0>(d, t); run<true, 32, 1>(d, t); run<false, 32, 1>(d, t);
  run<true, 64, 1>(d, t); run<false, 64, 1>(d, t); run<true, 16, 1>(d, t);
  return 0;
}
