// tcgen05.mma rate and layout probe for the blocked symmetric kernel (K1-sym2).
//  1. cycles per instruction, cta_group::1, M = 128, for narrow N (f16 SS / TS,
//     f8f6f4 SS with A MN-major), one issuing thread, 1 or 4 accumulators;
//  2. the same with TWO warps issuing concurrently (separate accumulators):
//     is the ~46-cycle floor per issuer or per tensor pipe?
//  3. correctness of kind::f8f6f4 (E4M3) with A MN-major in shared memory
//     (core matrix 8 K-rows x 16 MN-bytes) for both LBO/SBO assignments.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate_probe mma_rate_probe.cu
#include <cuda_fp8.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ inline uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
// kind::f16: a/b format 0 = F16; kind::f8f6f4: 0 = E4M3.  bit 15: A MN-major.
__host__ __device__ constexpr uint32_t idesc(int n, bool a_mn) {
  return (1u << 4) | (a_mn ? (1u << 15) : 0u) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

enum { K_F16_SS = 0, K_F16_TS = 1, K_F8_SS = 2 };

template <int KIND>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint32_t ta, uint64_t b, uint32_t id, uint32_t acc) {
  if (KIND == K_F16_SS)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
  else if (KIND == K_F16_TS)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(ta), "l"(b), "r"(id), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}

// NW warps (lane 0 each) issue `reps` MMAs round-robin over NACC accumulators
// of their own; out[w] = cycles of warp w (issue of the first to completion).
template <int KIND, int N, int NACC, int NW>
__global__ void rate(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x38383838u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (warp < NW && (threadIdx.x & 31) == 0) {
    const uint32_t a = su32(smem) + warp * 16384, b = su32(smem + 65536);
    const uint64_t ad = KIND == K_F8_SS ? sdesc(a, 1024, 128) : sdesc(a, 128, 256);
    const uint64_t bd = sdesc(b, 128, 256);
    const uint32_t id = idesc(N, KIND == K_F8_SS);
    const uint32_t base = tm + 128 + (uint32_t)warp * (384 / NW);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t d = base + (uint32_t)((r % NACC) * N);
      mma<KIND>(d, ad, tm + (uint32_t)(r & 7) * 8, bd, id, 1u);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp])));
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
        su32(&bar[warp])));
    out[warp] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int KIND, int N, int NACC, int NW>
void run_rate(const char* name, long long* d) {
  cudaFuncSetAttribute(rate<KIND, N, NACC, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int reps = 4096;
  rate<KIND, N, NACC, NW><<<1, 128, 100 * 1024>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[4] = {0, 0, 0, 0};
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int w = 0; w < NW; ++w) mx = h[w] > mx ? h[w] : mx;
  printf("%-10s N=%3d acc=%d warps=%d : %7.2f cycles/instr/warp, %7.2f cycles/instr total (%s)\n", name, N,
         NACC, NW, (double)mx / reps, (double)mx / reps / NW, cudaGetErrorString(e));
}

// Layout check: D[128 x 32] = A[128 x 32] B[32 x 32]^T with A (M x K) E4M3
// MN-major in smem, B (N x K) E4M3 K-major (core matrix 8 rows x 16 B,
// K-chunks at 128 B, 8-row groups at 256 B).  mode 0: LBO = K-direction
// stride (1024), SBO = MN-direction stride (128); mode 1: swapped.
__global__ void f8_check(const uint8_t* A, const uint8_t* B, float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // A: byte of (m, k) at (k>>3)*1024 + (m>>4)*128 + (k&7)*16 + (m&15)  (mode 0)
  //                    or (k>>3)*128 + (m>>4)*256 ... (mode 1: K-groups at 128, M-groups at 256)
  for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
    const int m = e / 32, k = e % 32;
    uint32_t off = mode == 0 ? (k >> 3) * 1024 + (m >> 4) * 128 + (k & 7) * 16 + (m & 15)
                             : (m >> 4) * 512 + (k >> 3) * 128 + (k & 7) * 16 + (m & 15);
    smem[off] = A[e];
  }
  for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
    const int n = e / 32, k = e % 32;
    const uint32_t off = 4096 + (n >> 3) * 256 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15);
    smem[off] = B[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint64_t ad = mode == 0 ? sdesc(su32(smem), 1024, 128) : sdesc(su32(smem), 128, 512);
    const uint64_t bd = sdesc(su32(smem + 4096), 128, 256);
    mma<K_F8_SS>(tm, ad, 0, bd, idesc(32, true), 0u);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
      su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(tm + ((uint32_t)(32 * warp) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int c = 0; c < 32; ++c) D[(32 * warp + lane) * 32 + c] = __uint_as_float(r[c]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run_rate<K_F16_SS, 32, 1, 1>("f16 SS", d);
  run_rate<K_F16_SS, 32, 4, 1>("f16 SS", d);
  run_rate<K_F16_SS, 64, 1, 1>("f16 SS", d);
  run_rate<K_F16_SS, 64, 4, 1>("f16 SS", d);
  run_rate<K_F16_TS, 32, 1, 1>("f16 TS", d);
  run_rate<K_F16_TS, 32, 4, 1>("f16 TS", d);
  run_rate<K_F16_TS, 64, 1, 1>("f16 TS", d);
  run_rate<K_F8_SS, 32, 1, 1>("f8 SS mn", d);
  run_rate<K_F8_SS, 32, 4, 1>("f8 SS mn", d);
  run_rate<K_F16_SS, 32, 2, 2>("f16 SS", d);
  run_rate<K_F16_SS, 64, 2, 2>("f16 SS", d);
  run_rate<K_F16_TS, 32, 2, 2>("f16 TS", d);
  run_rate<K_F16_TS, 32, 1, 3>("f16 TS", d);
  run_rate<K_F16_SS, 32, 1, 3>("f16 SS", d);
  run_rate<K_F16_SS, 128, 1, 1>("f16 SS", d);
  run_rate<K_F16_SS, 128, 1, 2>("f16 SS", d);
  run_rate<K_F16_SS, 256, 1, 1>("f16 SS", d);
  // layout check
  const int M = 128, N = 32, K = 32;
  uint8_t hA[M * K], hB[N * K];
  float fa[M * K], fb[N * K];
  srand(1);
  for (int i = 0; i < M * K; ++i) {
    __nv_fp8_e4m3 v((float)((rand() % 15) - 7) * 0.25f);
    hA[i] = v.__x;
    fa[i] = (float)v;
  }
  for (int i = 0; i < N * K; ++i) {
    __nv_fp8_e4m3 v((float)((rand() % 9) - 4) * 0.5f);
    hB[i] = v.__x;
    fb[i] = (float)v;
  }
  uint8_t *dA, *dB;
  float* dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(f8_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 1024);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dD, 0, M * N * 4);
    f8_check<<<1, 128, 16 * 1024>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    float hD[M * N];
    cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
    double err = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)fa[m * K + k] * fb[n * K + k];
        err = fmax(err, fabs(s - hD[m * N + n]));
      }
    printf("f8 MN-major A layout mode %d: max abs err %.3g (%s)\n", mode, err, cudaGetErrorString(e));
  }
  return 0;
}
