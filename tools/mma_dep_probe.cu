// Microbenchmark: is the ~46-50 cycle floor of narrow tcgen05.mma a throughput
// limit or the accumulate dependency on one D?  Issues `reps` MMAs round-robin
// over NACC independent accumulators (TMEM columns 256 + a*N).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_dep_probe mma_dep_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// PAIR: cta_group::2 over a 2-CTA cluster (M=256); else cta_group::1 (M=128).
template <int N, bool TS, int NACC, bool PAIR>
__global__ void __cluster_dims__(2, 1, 1) probe(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cta_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  const bool issuer = PAIR ? rank == 0 : true;
  if (issuer && threadIdx.x == 0) {
    const uint32_t a = su32(smem), b = su32(smem + 32768);
    const uint64_t ad = sdesc(a, 128, 256), bd = sdesc(b, 128, 256);
    const uint32_t id = idesc(PAIR ? 256 : 128, N);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t d = tm + 256 + (uint32_t)((r % NACC) * N);
      if (PAIR) {
        if (TS)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                       "r"(tm + (r & 7) * 8), "l"(bd), "r"(id), "r"(1));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(ad), "l"(bd), "r"(id), "r"(1));
      } else {
        if (TS)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                       "r"(tm + (r & 7) * 8), "l"(bd), "r"(id), "r"(1));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(ad), "l"(bd), "r"(id), "r"(1));
      }
    }
    if (PAIR)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(su32(&bar)), "h"((uint16_t)3));
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)));
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  if (PAIR && rank == 1 && threadIdx.x == 0)
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)));
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

template <int N, bool TS, int NACC, bool PAIR>
void run(long long* d) {
  cudaFuncSetAttribute(probe<N, TS, NACC, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int reps = 4096;
  probe<N, TS, NACC, PAIR><<<2, 128, 70 * 1024>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%s N=%3d %s acc=%d : %7.2f cycles/instr (%s)\n", PAIR ? "pair M=256" : "1cta M=128", N,
         TS ? "TS" : "SS", NACC, (double)h / reps, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<32, true, 1, false>(d); run<32, true, 2, false>(d); run<32, true, 4, false>(d);
  run<64, true, 1, false>(d); run<64, true, 2, false>(d); run<64, true, 3, false>(d);
  run<32, false, 1, false>(d); run<32, false, 4, false>(d);
  run<64, false, 1, false>(d); run<64, false, 3, false>(d);
  run<32, true, 1, true>(d); run<32, true, 2, true>(d); run<32, true, 4, true>(d);
  run<64, true, 1, true>(d); run<64, true, 2, true>(d); run<64, true, 3, true>(d);
  run<128, true, 1, true>(d); run<128, true, 2, true>(d);
  return 0;
}
