// Synchronisation latency probes (one B200): mbarrier ping-pong between two
// warps of one CTA and between the two CTAs of a cluster, with the three wait
// flavours K1 can use, plus tcgen05.commit -> mbarrier wake latency.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_probe sync_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <int MODE>
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    if (MODE == 0)
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
                   "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(su32(bar)), "r"(parity), "r"(0x989680u) : "memory");
    else if (MODE == 1)
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                   "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(su32(bar)), "r"(parity) : "memory");
    else
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                   "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(su32(bar)), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void arrive_remote(uint64_t* bar, uint32_t target) {
  uint32_t addr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(su32(bar)), "r"(target));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}

// CROSS = 0: warps 0 and 1 of CTA 0 ping-pong; CROSS = 1: warp 0 of CTA 0 and CTA 1.
template <int MODE, int CROSS>
__global__ void __cluster_dims__(2, 1, 1) pingpong(int reps, long long* out) {
  __shared__ uint64_t bar[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  cluster_sync();
  const bool ping = CROSS ? (rank == 0 && warp == 0) : (rank == 0 && warp == 0);
  const bool pong = CROSS ? (rank == 1 && warp == 0) : (rank == 0 && warp == 1);
  if (lane == 0 && (ping || pong)) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t par = (uint32_t)(r & 1);
      if (ping) {
        if (CROSS) arrive_remote(&bar[1], 1); else arrive_local(&bar[1]);
        wait<MODE>(&bar[0], par);
      } else {
        wait<MODE>(&bar[1], par);
        if (CROSS) arrive_remote(&bar[0], 0); else arrive_local(&bar[0]);
      }
    }
    long long t1 = clock64();
    if (ping && blockIdx.x == 0) out[0] = t1 - t0;
  }
  __syncwarp();
  cluster_sync();
}

// tcgen05.commit (no MMA in flight) -> mbarrier observed by the same thread,
// and observed by a different warp (it records clock64 when it wakes).
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) commit_lat(int reps, long long* out) {
  __shared__ uint64_t bar, ack;
  __shared__ uint32_t slot;
  __shared__ long long tw;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&ack)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  cluster_sync();
  long long acc_self = 0, acc_other = 0;
  if (lane == 0 && warp < 2) {
    for (int r = 0; r < reps; ++r) {
      const uint32_t par = (uint32_t)(r & 1);
      if (warp == 0) {
        const long long t0 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        wait<MODE>(&bar, par);
        const long long t1 = clock64();
        acc_self += t1 - t0;
        wait<MODE>(&ack, par);  // other warp has recorded its wake time
        acc_other += tw - t0;
      } else {
        wait<MODE>(&bar, par);
        tw = clock64();
        arrive_local(&ack);
      }
    }
    if (warp == 0 && blockIdx.x == 0) {
      out[0] = acc_self;
      out[1] = acc_other;
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
  cluster_sync();
}

template <int MODE, int CROSS>
void run_pp(long long* d, int grid) {
  const int reps = 10000;
  pingpong<MODE, CROSS><<<grid, 64>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("pingpong %s wait=%d grid=%3d: %6.1f cycles one-way (%s)\n", CROSS ? "cross-CTA " : "same-CTA  ",
         MODE, grid, (double)h / reps / 2, cudaGetErrorString(e));
}
template <int MODE>
void run_commit(long long* d) {
  const int reps = 10000;
  commit_lat<MODE><<<2, 64>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2] = {0, 0};
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("commit->wake wait=%d: issuing thread %6.1f, other warp %6.1f cycles (%s)\n", MODE,
         (double)h[0] / reps, (double)h[1] / reps, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run_pp<0, 0>(d, 2); run_pp<1, 0>(d, 2); run_pp<2, 0>(d, 2);
  run_pp<0, 1>(d, 2); run_pp<1, 1>(d, 2); run_pp<2, 1>(d, 2);
  run_pp<0, 1>(d, 148); run_pp<1, 1>(d, 148);
  run_commit<0>(d); run_commit<1>(d); run_commit<2>(d);
  return 0;
}
