// L2 reduction throughput for the symmetric kernels' accumulation:
//   red.global.add.u64 from registers, 32 lanes x 8 B contiguous per instruction
//   vs cp.reduce.async.bulk .add.u64 of 2 KB blocks from shared memory
// and the TMEM row layout of a cta_group::1 M = 64 tcgen05.mma.
// usage: red_probe
#include <cstdint>
#include <cstdio>

__global__ void red_regs(unsigned long long* acc, int64_t words, int iters) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x >> 5);
  int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  for (int it = 0; it < iters; ++it) {
    const int64_t base = ((w + (int64_t)it * stride) * 32) % words;
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(acc + base + lane), "l"(1ull) : "memory");
  }
}

__global__ void red_bulk(unsigned long long* acc, int64_t words, int iters) {
  __shared__ __align__(128) unsigned long long st[4][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 256; i += 32) st[warp & 3][i] = 1;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x >> 5);
  int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int64_t base = ((w + (int64_t)it * stride) * 256) % words;
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], 2048;\n\t"
                   "cp.async.bulk.commit_group;" ::"l"(acc + base),
                   "r"((unsigned)__cvta_generic_to_shared(st[warp & 3])) : "memory");
      if ((it & 7) == 7) asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const int64_t words = (64ll << 20) / 8;  // 64 MB region (L2 resident)
  unsigned long long* acc;
  cudaMalloc(&acc, words * 8);
  cudaMemset(acc, 0, words * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    const int iters = 4096;
    cudaEventRecord(a);
    red_regs<<<148 * 4, 256>>>(acc, words, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 148.0 * 4 * 8 * iters * 256;
    printf("red.global.add.u64 (256 B / warp-instr): %.2f TB/s\n", bytes / ms / 1e9);
    cudaEventRecord(a);
    red_bulk<<<148 * 4, 256>>>(acc, words, iters / 8);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double bytes2 = 148.0 * 4 * 8 * (iters / 8) * 2048;
    printf("cp.reduce.async.bulk .add.u64 (2 KB): %.2f TB/s\n", bytes2 / ms / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
