// Check of the transposed-product building block for a symmetric K(X,X)
// kernel: tcgen05.mma.cta_group::2 with A = P^T read from shared memory in the
// MN-major no-swizzle layout (P stored row i, 8 consecutive j per 16 B, the
// same bytes the K-major layout of P uses), B split along N between the two
// CTAs.  Exact small-integer operands; prints max |D - D_ref| per variant.
//   variant 0: SBO = MN-group stride, LBO = K-group stride
//   variant 1: swapped
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mn_major_probe mn_major_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
// kind::f16, F32 accumulate, A major bit 15 (1 = MN-major), B K-major
__host__ __device__ constexpr uint32_t idesc(int m, int n, int a_mn) {
  return (1u << 4) | ((uint32_t)a_mn << 15) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int NI = 128, NJ = 128, NH = 32, N = 2 * NH;  // K = i, M = j (per CTA), N split
constexpr uint32_t XS = 2048;                           // i-group stride of P (16 j-groups x 128 B)

__global__ void __cluster_dims__(2, 1, 1) probe(const float* P, const float* B, float* D, int variant) {
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
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  // P_rank (i, j) -> (i/8)*XS + (j/8)*128 + (i%8)*16 + (j%8)*2
  __half* sP = (__half*)smem;
  for (int e = threadIdx.x; e < NI * NJ; e += blockDim.x) {
    const int i = e / NJ, j = e % NJ;
    const uint32_t off = (i / 8) * XS + (j / 8) * 128 + (i % 8) * 16 + (j % 8) * 2;
    sP[off / 2] = __float2half(P[(rank * NI + i) * NJ + j]);
  }
  // B_rank (n, i), K-major: (n/8)*2048 + (i/8)*128 + (n%8)*16 + (i%8)*2
  __half* sB = (__half*)(smem + 32768);
  for (int e = threadIdx.x; e < NH * NI; e += blockDim.x) {
    const int n = e / NI, i = e % NI;
    const uint32_t off = (n / 8) * 2048 + (i / 8) * 128 + (n % 8) * 16 + (i % 8) * 2;
    sB[off / 2] = __float2half(B[(rank * NH + n) * NI + i]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (rank == 0 && threadIdx.x == 0) {
    for (int s = 0; s < NI / 16; ++s) {
      const uint32_t pa = su32(sP) + s * 2 * XS;  // next 16 i = two i-groups
      const uint64_t ad = variant == 0 ? sdesc(pa, XS, 128) : sdesc(pa, 128, XS);
      const uint64_t bd = sdesc(su32(sB) + s * 256, 128, 2048);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                   "l"(ad), "l"(bd), "r"(idesc(256, N, 1)), "r"(s));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(su32(&bar)), "h"((uint16_t)3));
  }
  if (threadIdx.x == 0)
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)));
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  {  // thread t = TMEM lane t = row m (= j) of this CTA's half of D
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(tm + ((uint32_t)(32 * warp) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int q = 0; q < 16; ++q) D[(rank * NJ + threadIdx.x) * N + c0 + q] = __uint_as_float(v[q]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  const int nP = 2 * NI * NJ, nB = 2 * NH * NI, nD = 2 * NJ * N;
  float *hP = new float[nP], *hB = new float[nB], *hD = new float[nD];
  srand(1);
  for (int e = 0; e < nP; ++e) hP[e] = (float)(rand() % 5 - 2);
  for (int e = 0; e < nB; ++e) hB[e] = (float)(rand() % 5 - 2);
  float *dP, *dB, *dD;
  cudaMalloc(&dP, nP * 4);
  cudaMalloc(&dB, nB * 4);
  cudaMalloc(&dD, nD * 4);
  cudaMemcpy(dP, hP, nP * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, nB * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(dD, 0, nD * 4);
    probe<<<2, 128, 64 * 1024>>>(dP, dB, dD, variant);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, nD * 4, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int r = 0; r < 2; ++r)
      for (int j = 0; j < NJ; ++j)
        for (int n = 0; n < N; ++n) {
          const int src = n / NH, nn = n % NH;  // B columns [0,32) from CTA0, [32,64) from CTA1
          double ref = 0;
          for (int i = 0; i < NI; ++i) ref += (double)hP[(r * NI + i) * NJ + j] * hB[(src * NH + nn) * NI + i];
          const double d = hD[(r * NJ + j) * N + n] - ref;
          if (d * d > worst * worst) worst = d < 0 ? -d : d;
        }
    printf("variant %d (%s): max |D - ref| = %g\n", variant, cudaGetErrorString(e), worst);
  }
  return 0;
}
