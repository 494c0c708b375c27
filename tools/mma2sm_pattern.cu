// Per-tile tensor-pipe cost of K1's MMA pattern on a CTA pair (cta_group::2,
// M=256), 74 clusters (all 148 SMs) in parallel.  Patterns per 128-column tile:
//   0: f16  8 x [TS N=2W, TS N=W]         + 2 x SS N=128 (GEMM1) + 1 commit
//   1: f16  8 x TS N=2W ; f8f6f4 4 x TS N=W (K=32)  + GEMM1 + 1 commit
//   2: f16  8 x TS N=2W only              + GEMM1 + 1 commit   (lower bound)
//   3: f8f6f4 4 x TS N=2W (K=32) + f8f6f4 4 x TS N=W + GEMM1 + 1 commit
//   4/5: pattern 0 + 3 waits (try_wait / test_wait) on already-complete barriers
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma2sm_pattern mma2sm_pattern.cu
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
__device__ __forceinline__ void ts_f16(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void ts_f8(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void ss_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void done_wait(uint64_t* b, bool test) {
  uint32_t ok = 0;
  while (!ok) {
    if (test)
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], 1;\n\t"
                   "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(su32(b)) : "memory");
    else
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 1, %2;\n\t"
                   "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(0x989680u) : "memory");
  }
}

template <int W, int PAT>
__global__ void __cluster_dims__(2, 1, 1) pat(int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, idle[3];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cta_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&idle[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) {
    const uint32_t h = (uint32_t)i * 2654435761u;
    ((uint32_t*)smem)[i] = (h & 0x03ff03ffu) | 0x38003800u;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t a = su32(smem), b = su32(smem + 32768);
    const uint64_t ad = sdesc(a, 128, 512), bd = sdesc(b, 128, 2048);
    const uint32_t id2 = idesc(256, 2 * W), id2h = idesc(256, W), id1 = idesc(256, 128);
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t S = tm + (t % 3) * 128, O = tm + 384;
      if (PAT >= 4) {
        done_wait(&idle[0], PAT == 5);
        done_wait(&idle[1], PAT == 5);
      }
      if (PAT == 0 || PAT >= 4) {
        for (int m = 0; m < 8; ++m) {
          const uint32_t ahi = S + 32 * (m >> 1) + 8 * (m & 1);
          ts_f16(O, ahi, bd + 16 * m, id2);
          ts_f16(O, ahi + 16, bd + 16 * m, id2h);
        }
      } else if (PAT == 1) {
        for (int m = 0; m < 8; ++m) ts_f16(O, S + 32 * (m >> 1) + 8 * (m & 1), bd + 16 * m, id2);
        for (int m = 0; m < 4; ++m) ts_f8(O + 2 * W, S + 64 + 8 * m, bd + 16 * m, id2h);
      } else if (PAT == 2) {
        for (int m = 0; m < 8; ++m) ts_f16(O, S + 32 * (m >> 1) + 8 * (m & 1), bd + 16 * m, id2);
      } else {
        for (int m = 0; m < 4; ++m) ts_f8(O, S + 8 * m, bd + 16 * m, id2);
        for (int m = 0; m < 4; ++m) ts_f8(O + 2 * W, S + 64 + 8 * m, bd + 16 * m, id2h);
      }
      if (PAT >= 4) done_wait(&idle[2], PAT == 5);
      const uint32_t S3 = tm + ((t + 3) % 3) * 128;
      for (int k = 0; k < 2; ++k) ss_f16(S3, ad + 16 * k, ad + 16 * k + 2048, id1, k);
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(su32(&bar)), "h"((uint16_t)3));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(su32(&bar)), "h"((uint16_t)3));
    // wait for the final arrival (tiles + 1 arrivals on a count-1 barrier: parity of the last phase)
    const uint32_t par = (uint32_t)(tiles & 1);
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)), "r"(par));
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int W, int PAT>
void run(long long* d) {
  cudaFuncSetAttribute(pat<W, PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int tiles = 2000;
  pat<W, PAT><<<148, 128, 70 * 1024>>>(tiles, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("W=%d pattern %d : %7.1f cycles per tile pair (%s)\n", W, PAT, (double)h / tiles,
         cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<32, 0>(d); run<32, 1>(d); run<32, 2>(d); run<32, 3>(d); run<32, 4>(d); run<32, 5>(d);
  run<16, 0>(d); run<16, 1>(d); run<16, 2>(d); run<16, 3>(d);
  return 0;
}
