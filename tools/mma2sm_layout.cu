// Layout check for tcgen05.mma.cta_group::2: which CTA supplies which rows of
// B (N dimension), and D placement.  A = 1 everywhere (K=16), B row n of CTA r
// holds 1 + 100 r + (row index within that CTA's block).
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
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

template <int N, bool TS>
__global__ void __cluster_dims__(2, 1, 1) lay(float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  // A: 128 rows x 16 k of 1.0 (K-major canonical, SBO = 256 B) at smem[0, 4K)
  __half* A = (__half*)smem;
  for (int i = threadIdx.x; i < 128 * 16; i += blockDim.x) A[i] = __float2half(1.f);
  // B: up to 128 rows x 16 k at smem[32K...): row r of this CTA -> 1 + 100*rank + r
  __half* B = (__half*)(smem + 32768);
  for (int e = threadIdx.x; e < 128 * 16; e += blockDim.x) {
    const int g = e / 128, rem = e % 128;        // 8-row group, within group: chunk, row, k
    const int q = rem / 64, r = (rem % 64) / 8;  // k-chunk (0/1), row in group
    (void)q;
    const int row = g * 8 + r;
    B[e] = __float2half((float)(1 + 100 * rank + row));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (TS) {
    // copy A into TMEM columns [0, 8) (f16 pairs) of this CTA: each thread its lane
    if (warp < 4) {
      uint32_t v[8];
      for (int i = 0; i < 8; ++i) v[i] = 0x3c003c00u;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                       tm + ((uint32_t)(32 * warp) << 16)),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  if (rank == 0 && threadIdx.x == 0) {
    const uint64_t ad = sdesc(su32(A), 128, 256), bd = sdesc(su32(B), 128, 256);
    if (TS)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 256),
                   "r"(tm), "l"(bd), "r"(idesc(256, N)), "r"(0));
    else
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + 256),
                   "l"(ad), "l"(bd), "r"(idesc(256, N)), "r"(0));
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(su32(&bar)), "h"((uint16_t)3));
  }
  if (threadIdx.x == 0)
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)));
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    uint32_t v[16];
    for (int c0 = 0; c0 < N; c0 += 16) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(tm + 256 + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      if (lane == 0)
        for (int i = 0; i < 16; ++i) out[rank * 256 + c0 + i] = __uint_as_float(v[i]) / 16.f;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, bool TS>
void run(float* d) {
  cudaFuncSetAttribute(lay<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  cudaMemset(d, 0, 512 * 4);
  lay<N, TS><<<2, 128, 70 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  float h[512];
  cudaMemcpy(h, d, 512 * 4, cudaMemcpyDeviceToHost);
  printf("N=%d %s (%s)\n", N, TS ? "TS" : "SS", cudaGetErrorString(e));
  for (int r = 0; r < 2; ++r) {
    printf("  CTA%d row0 D[0:%d]:", r, N);
    for (int i = 0; i < N; ++i) printf(" %g", h[r * 256 + i]);
    printf("\n");
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 512 * 4);
  run<32, false>(d);
  run<64, false>(d);
  run<32, true>(d);
  run<64, true>(d);
  return 0;
}
