// Issue-side cost of K1's per-step MMA sequence on a CTA pair (cta_group::2),
// with NW warps of the leader CTA issuing concurrently (each its own
// accumulator).  Per step and warp: [mbarrier wait on a completed barrier]
// + 16 TS MMAs (8 x N=64, 8 x N=32) + [fence::after_thread_sync] + 2 SS MMAs
// (N=128) + [multicast commit].  Reports cycles per step per warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o issue_probe issue_probe.cu
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
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void wait_done(uint64_t* b) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 1, %2;\n\t"
                 "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(0x989680u) : "memory");
}

// FLAGS: 1 = wait per step, 2 = fence before GEMM1, 4 = commit per step,
//        8 = whole warp + elect_one (else lane 0 only), 16 = skip GEMM1,
//        32 = K1's real operand layout (B3 region for the lo MMAs, 9 rotating V slots of
//             12 KB, 6 rotating XB slots)
template <int NW, int FLAGS>
__global__ void __cluster_dims__(2, 1, 1) probe(int steps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];  // 200 KB: A 8K | XB 6x4K | V 9x12K
  __shared__ uint64_t bar[4], idle;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&idle)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) {
    const uint32_t h = (uint32_t)i * 2654435761u;
    ((uint32_t*)smem)[i] = (h & 0x03ff03ffu) | 0x38003800u;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  const bool active = rank == 0 && warp < NW && ((FLAGS & 8) || lane == 0);
  if (active) {
    const uint32_t a = su32(smem), b = su32(smem + 40960);
    const uint64_t ad = sdesc(a, 128, 512), bd0 = sdesc(b, 128, 2048);
    const uint64_t xb0 = sdesc(a + 8192, 128, 512);
    const uint32_t id2 = idesc(256, 64), id2h = idesc(256, 32), id1 = idesc(256, 128);
    const uint32_t O = tm + 384 + (uint32_t)(warp * 64);
    const long long t0 = clock64();
    for (int t = 0; t < steps; ++t) {
      const uint32_t S = tm + (uint32_t)((t % 3) * 128);
      const uint64_t bd = (FLAGS & 32) ? bd0 + (uint64_t)((t % 9) * (12288 >> 4)) : bd0;
      const uint64_t b3 = (FLAGS & 32) ? bd + (8192 >> 4) : bd;
      const uint64_t xb = (FLAGS & 32) ? xb0 + (uint64_t)((t % 6) * (4096 >> 4)) : ad + 2048 / 16;
      if (FLAGS & 1) wait_done(&idle);
      if (!(FLAGS & 8) || elect_one()) {
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const uint32_t ahi = S + 32 * (m >> 1) + 8 * (m & 1);
          ts(O, ahi, bd + 16 * m, id2);
          ts(O, ahi + 16, b3 + 16 * m, id2h);
        }
      }
      if (FLAGS & 8) __syncwarp();
      if (FLAGS & 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (!(FLAGS & 8) || elect_one()) {
        if (!(FLAGS & 16))
          for (int k = 0; k < 2; ++k) ss(S, ad + 16 * k, xb + 16 * k, id1, k);
        if (FLAGS & 4)
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                       ::"r"(su32(&bar[warp])), "h"((uint16_t)3));
      }
      if (FLAGS & 8) __syncwarp();
    }
    const long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) out[warp] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int NW, int FLAGS>
void run(long long* d, const char* name) {
  cudaFuncSetAttribute(probe<NW, FLAGS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int steps = 1000;
  cudaMemset(d, 0, 64);
  probe<NW, FLAGS><<<148, 128, 160 * 1024>>>(steps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("NW=%d %-34s:", NW, name);
  for (int w = 0; w < NW; ++w) printf(" %7.1f", (double)h[w] / steps);
  printf("  cycles/step/warp (%s)\n", cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<1, 0>(d, "16+2 MMAs");
  run<1, 16>(d, "16 MMAs (no GEMM1)");
  run<1, 4>(d, "+commit");
  run<1, 6>(d, "+commit +fence");
  run<1, 7>(d, "+commit +fence +wait");
  run<1, 15>(d, "+commit +fence +wait, whole warp");
  run<2, 0>(d, "16+2 MMAs");
  run<2, 4>(d, "+commit");
  run<2, 7>(d, "+commit +fence +wait");
  run<2, 15>(d, "+commit +fence +wait, whole warp");
  run<1, 15 | 32>(d, "... whole warp, K1 operand layout");
  run<1, 8 | 32>(d, "MMAs only, whole warp, K1 layout");
  return 0;
}
