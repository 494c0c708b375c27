// Tensor-pipe issue queue depth: timestamps after each MMA issue.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
template <int N>
__global__ void q(long long* out) {
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
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    long long ts[33];
    const uint64_t bd = sdesc(su32(smem + 32768), 128, 256);
    const uint32_t id = idesc(128, N);
    ts[0] = clock64();
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 256),
                   "r"(tm + (r & 7) * 8), "l"(bd), "r"(id));
      ts[r + 1] = clock64();
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)));
    long long te = clock64();
    for (int r = 0; r <= 32; ++r) out[r] = ts[r] - ts[0];
    out[33] = te - ts[0];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
// NW warps (lane 0 each) issue 32 MMAs concurrently into separate accumulators.
template <int N, int NW>
__global__ void q2(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
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
  const uint32_t tm = slot;
  if (warp < NW && lane == 0) {
    const uint64_t bd = sdesc(su32(smem + 32768), 128, 256);
    const uint32_t id = idesc(128, N);
    const uint32_t D = tm + 256 + (uint32_t)(warp * N);
    const long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < 32; ++r)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(D),
                   "r"(tm + (r & 7) * 8), "l"(bd), "r"(id));
    const long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp])));
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar[warp])));
    const long long t2 = clock64();
    out[2 * warp] = t1 - t0;
    out[2 * warp + 1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
template <int N, int NW> void run2(long long* d) {
  cudaFuncSetAttribute(q2<N, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  q2<N, NW><<<1, 128, 70 * 1024>>>(d);
  cudaDeviceSynchronize();
  long long h[8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("N=%d %d issuing warps x 32 MMAs:", N, NW);
  for (int w = 0; w < NW; ++w) printf("  w%d issue %lld done %lld", w, h[2 * w], h[2 * w + 1]);
  printf("\n");
}
template <int N> void run(long long* d) {
  cudaFuncSetAttribute(q<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  q<N><<<1, 128, 70 * 1024>>>(d);
  cudaDeviceSynchronize();
  long long h[34];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("N=%d issue times:", N);
  for (int r = 1; r <= 32; ++r) printf(" %lld", h[r]);
  printf(" | done %lld\n", h[33]);
}
int main() { long long* d; cudaMalloc(&d, 64 * 8); run<64>(d); run<256>(d);
  run2<64, 1>(d); run2<64, 2>(d); run2<64, 4>(d); run2<32, 2>(d); run2<32, 4>(d); return 0; }
