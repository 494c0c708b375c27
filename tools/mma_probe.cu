// Microbenchmark: cycles per tcgen05.mma (kind::f16, M=128) for A from SMEM
// (SS) or TMEM (TS) at several N; tcgen05.ld throughput; MUFU ex2 rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cstdio>
#include <cstdint>
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

template <int N, bool TS>
__global__ void probe(int reps, long long* out) {
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
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = su32(smem), b = su32(smem + 32768);
    const uint64_t ad = sdesc(a, 128, 256), bd = sdesc(b, 128, 256);
    const uint32_t id = idesc(128, N);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (TS)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 256),
                     "r"(tm + (r & 7) * 8), "l"(bd), "r"(id), "r"(1));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + 256),
                     "l"(ad), "l"(bd), "r"(id), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)));
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// tcgen05.ld 32x32b.x32 throughput with `warps` warps (each reads its lane quarter)
__global__ void ldprobe(int reps, long long* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint32_t v[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(tm + (r & 7) * 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int i = 0; i < 32; ++i) acc ^= v[i];
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[warp] = t1 - t0;
  if (acc == 0x12345) out[100] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

__global__ void mufuprobe(int reps, float* sink, long long* out) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = -(threadIdx.x + i) * 1e-3f;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  sink[threadIdx.x] = s;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}


// the kernel's per-tile pattern: 8 x (TS N=2W, TS N=W) + 2 x SS N=128, rotating S buffers
template <int W, int MODE>
__global__ void patprobe(int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[3];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 100000;" ::"r"(su32(&bar2[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    ((uint32_t*)smem)[i] = (MODE >= 5) ? ((h & 0x03ff03ffu) | 0x38003800u) : 0x3c003c00u;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = su32(smem), b = su32(smem + 32768);
    const uint64_t ad = sdesc(a, 128, 512), bd = sdesc(b, 128, 2048);
    const uint32_t id2 = idesc(128, 2 * W), id2h = idesc(128, W), id1 = idesc(128, 128);
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t S = tm + (t % 3) * 128, O = tm + 384;
      if (MODE == 6 || MODE == 7) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (MODE == 7) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (MODE != 2)
        for (int m = 0; m < 8; ++m) {
          const uint32_t ahi = S + 32 * (m >> 1) + 8 * (m & 1);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(O),
                       "r"(ahi), "l"(bd + 16 * m), "r"(id2), "r"(1));
          if (MODE != 1)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(O),
                         "r"(ahi + 16), "l"(bd + 16 * m), "r"(id2h), "r"(1));
        }
      if (MODE == 3 || MODE == 4)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[0])));
      const uint32_t S3 = tm + ((t + 3) % 3) * 128;
      if (MODE == 7) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (MODE == 8) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      for (int k = 0; k < 2; ++k)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(S3),
                     "l"(ad + 16 * k), "l"(ad + 16 * k + 2048), "r"(id1), "r"(k));
      if (MODE == 3) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[1])));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[2])));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)));
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int W, int MODE>
void runpat(long long* d, const char* name, int grid = 1) {
  cudaFuncSetAttribute(patprobe<W, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  patprobe<W, MODE><<<grid, 128, 70 * 1024>>>(2000, d);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("pattern W=%d %-34s: %7.1f cycles/tile\n", W, name, (double)h / 2000);
}

template <int N, bool TS>
void run(long long* d) {
  cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int reps = 4096;
  probe<N, TS><<<1, 128, 70 * 1024>>>(reps, d);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("M=128 N=%3d %s : %7.2f cycles/instr  (ideal N/2 = %d)\n", N, TS ? "TS(A tmem)" : "SS(A smem)",
         (double)h / reps, N / 2);
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  run<16, false>(d); run<32, false>(d); run<64, false>(d); run<128, false>(d); run<256, false>(d);
  run<16, true>(d);  run<32, true>(d);  run<64, true>(d);  run<128, true>(d);  run<256, true>(d);
  for (int warps : {4, 8, 16}) {
    ldprobe<<<1, 32 * warps>>>(4096, d);
    long long h[16];
    cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < warps; ++i) mx = h[i] > mx ? h[i] : mx;
    double bytes = 4096.0 * warps * 32 * 32 * 4;
    printf("tcgen05.ld x32 with %2d warps: %.1f B/clk per SM\n", warps, bytes / mx);
  }
  runpat<32, 0>(d, "8x(TS 64 + TS 32) + 2x SS128");
  runpat<32, 1>(d, "8x(TS 64) + 2x SS128");
  runpat<32, 2>(d, "2x SS128 only");
  runpat<16, 0>(d, "8x(TS 32 + TS 16) + 2x SS128");
  runpat<32, 3>(d, "pattern + 3 commits per tile");
  runpat<32, 4>(d, "pattern + 1 commit per tile");
  runpat<32, 6>(d, "pattern + 1 fence::after per tile");
  runpat<32, 7>(d, "pattern + 3 fence::after per tile");
  runpat<32, 8>(d, "pattern + 1 fence::before per tile");
  runpat<32, 0>(d, "pattern, 148 CTAs, ones", 148);
  runpat<32, 5>(d, "pattern, 1 CTA, random data", 1);
  runpat<32, 5>(d, "pattern, 148 CTAs, random data", 148);
  float* sink;
  cudaMalloc(&sink, 4096 * 4);
  for (int th : {128, 256, 512, 1024}) {
    mufuprobe<<<1, th>>>(4096, sink, d);
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("MUFU.EX2 with %4d threads: %.2f ex2/clk per SM\n", th, 4096.0 * 8 * th / h);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
