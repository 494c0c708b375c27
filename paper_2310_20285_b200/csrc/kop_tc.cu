// K1 on tcgen05/TMEM: fused kernel-matmul  out = K(Xr, Xc) V  with K never
// materialised (replaces the tile body of prior_matvec, gp.py:162-171).
//
// One CTA pair (cluster of 2, cta_group::2 MMAs with M = 256) per two SMs;
// each CTA owns a 128-row tile and both sweep the same column tiles.
// Roles per CTA (24 warps; registers rebalanced per warpgroup with setmaxnreg):
//   warp 0 lane 0 producer: the CTA's row tile + its half of each XB column
//                 tile (1-D bulk copies, cp.async.bulk -> UBLKCP).
//   warp 3 lane 0 producer: the CTA's half of each V column tile.
//   warps 0/3 lane 1  relays: forward this CTA's copy completions to the
//                 leader CTA's barriers (the MMAs need both halves).
//   warp 1        (leader only) GEMM2 issuer, whole warp, elect.sync issues:
//                   O[256x2WP] += P_hi . [Vhi|Vlo],  O[:, :WP] += P_lo . Vhi
//                   (kind::f16, A = P in TMEM); one wait per step on rdy[g]
//                   (P(g) written, V(g) and XB(g+3) landed).
//   warp 2        TMEM allocation, then (leader only) GEMM1 issuer:
//                   S[256x128] = XA . XB^T  (kind::f16, SS) for tile t after
//                   GEMM2(t-3) completed (it overwrites that S/P buffer).
//                 Two issuing warps because one thread issues a tcgen05.mma
//                 only every ~46 cycles (tools/mma_queue_probe.cu).
//   warps 4-19    four epilogue warpgroups in two groups of 8 warps that
//                 alternate column tiles (each warp: one TMEM lane quarter,
//                 one 64-column half): TMEM -> regs, kernel transform (ex2 for
//                 RBF, sqrt + ex2 for Matern), fp16 hi/lo split, regs -> TMEM
//                 over S (P aliases S).  96 registers each.
//   warps 20-23   correction warpgroup: drains O every CH column tiles into
//                 fp64 shared-memory accumulators, scales, writes rows (to
//                 every destination of a fused-gather launch).
// cta_group::2 splits B by rows: CTA0 supplies B rows [0, N/2), CTA1 rows
// [N/2, N), each at the same shared-memory offset (tools/mma2sm_layout.cu),
// so CTA0 holds [XB rows 0-63 | Vhi | Vhi rows 0..WP/2) and CTA1
// [XB rows 64-127 | Vlo | Vhi rows WP/2..WP).  A pair instruction costs the
// same cycles as a single-CTA one (tools/mma2sm_probe.cu), halving the
// tensor time per SM.
//
// Precision (hard part 2): the distance GEMM uses a 3-term fp16
// split packed along K,  [u_hi u_lo u_hi a_hi a_lo 1 1] . [x_hi x_hi x_lo 1 1 b_hi b_lo],
// which returns the exponent argument  L - |x~_i - x~_j|^2  (RBF) or
// |x~_i - x~_j|^2 (Matern) directly, with x~ = (x - mean) * scale, so no
// per-pair FMAs are needed before the MUFU op.  The contraction uses the
// 3-term fp16 split  P_hi V_hi + P_lo V_hi + P_hi V_lo  with kernel values
// pre-scaled by 2^s and RHS columns by 2^e_c into fp16 range; fp32 tensor
// accumulation is flushed to fp64 every CH*128 columns at fixed global
// column boundaries (reduction order independent of row sharding).
#include <cuda_fp16.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "kop.cuh"

namespace {

constexpr int BM = 128;          // rows per CTA tile (a pair covers 256)
constexpr int BN = 128;          // columns per tile (GEMM1 N, GEMM2 K)
constexpr int CH = 16;           // column tiles per fp32 accumulation chunk
// Epilogue: two groups (tile parity) of two warpgroups each; the two warps
// of a group that share a TMEM lane quarter split the tile's columns, so four
// warps per SMSP feed the MUFU (tools/epi_probe.cu: one warp per SMSP reaches
// 56 % of the MUFU rate, two 83 %) and a group waiting on s_full leaves two.
// Registers are rebalanced with setmaxnreg: 40 for the producer / MMA and the
// correction warpgroups, 96 for the four epilogue warpgroups.
constexpr int EPI_WARPS = 16;
constexpr int NTHREADS = 32 * (4 + EPI_WARPS + 4);
constexpr int SMEM_BUDGET = 225 * 1024;
constexpr int TMEM_COLS = 512;
constexpr int NS_MAX = 3;        // S/P buffers in TMEM (3 x 128 columns; symmetric kernel 2)
constexpr int NR = 12;           // s_full / rdy rings: >= max wait lag (XB depth, V depth, 4)
constexpr int TRACE_TILES = 256, TRACE_EV = 16;
constexpr uint32_t PBUF = 2u * BM * BN * 2u;  // symmetric kernel: one [P_hi | P_lo] buffer (64 KB)

// ------------------------------------------------------------------ PTX

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef NCGP_SYM1_PT
// K1-sym1: GEMM2 reads P from TMEM (TS MMA, no shared-memory A reads) and the
// three split terms accumulate into one set of WP columns, which frees TMEM
// for a third S buffer (build-time A/B: 0 = the round-1 layout, P only in
// shared memory, [hi Vhi + lo Vhi | hi Vlo] accumulators, two S buffers at WP = 32)
#define NCGP_SYM1_PT 1
#endif
// (2: as 1, but the transposed product keeps the two-instruction form --
// P_hi^T [Vhi | Vlo] (N = 2 WP) + P_lo^T Vhi -- so P^T is read from shared
// memory once per k-step instead of twice, into a single-buffered D_T of
// 2 WP columns)
#ifndef NCGP_PAIR_PT
// symmetric pair kernel: GEMM2 reads P from TMEM (written over S, as in the
// plain kernel) instead of from shared memory; shared memory then only holds
// P for the transposed product (build-time A/B)
#define NCGP_PAIR_PT 0
#endif
#ifndef NCGP_PAIR_F8
// symmetric pair kernel: the split term P_lo Vhi of both products in E4M3
// (as K1-sym2): P buffers of 48 instead of 64 KB -- three of them where
// shared memory allows -- and half the transposed product's P_lo MMAs
#define NCGP_PAIR_F8 0
#endif
#ifndef NCGP_PAIR_RED
#define NCGP_PAIR_RED 0  // the pair kernel's flushes by RED (build-time A/B)
#endif
#ifndef NCGP_SYM1_RED
// K1-sym1 flushes with coalesced red.global.add.u64 into a column-major
// accumulator (as K1-sym2) instead of staging + TMA bulk reductions (build-time A/B)
#define NCGP_SYM1_RED 1
#endif
#ifndef NCGP_SYM1_PT2NS
#define NCGP_SYM1_PT2NS 0  // build-time A/B: PT = 2 at WP = 32 with two S buffers and two D_T buffers
#endif
#ifndef NCGP_SYM1_PT16
#define NCGP_SYM1_PT16 2  // the same at WP = 16
#endif
#ifndef NCGP_SYM1_NS16
#define NCGP_SYM1_NS16 3  // K1-sym1 S buffers at WP = 16 (build-time A/B: 2 or 3)
#endif
#ifndef NCGP_FX_CVT
#define NCGP_FX_CVT 0  // fixed-point conversion: 0 cvt.rni.s64.f32 (XU), 1 two-limb FMA (build-time A/B)
#endif
#ifndef NCGP_WAIT_MODE
#define NCGP_WAIT_MODE 0  // 0: try_wait + suspend hint, 1: try_wait (default limit), 2: test_wait spin
#endif
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
#if NCGP_WAIT_MODE == 0
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
      : "memory");
#elif NCGP_WAIT_MODE == 1
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}
// Bounded wait: a pipeline bug traps (kernel error, ~17 s) instead of hanging the GPU.
#ifndef NCGP_WAIT_NS
#define NCGP_WAIT_NS 0  // back-off between polls of every wait (build-time A/B: 20 / 60 / 150 ns +1 % slower at cfg3)
#endif
#ifndef NCGP_WAIT_CHEAP
#define NCGP_WAIT_CHEAP 0  // poll loop reads the clock every 256th try only (build-time A/B:
                           // cfg3 285.4 vs 281.6 ms -- the tighter loop polls more often and is slower)
#endif
#ifndef NCGP_WAIT_RELAX_NS
#define NCGP_WAIT_RELAX_NS 0  // mbar_wait_relaxed sleeps this long between tries (0: same as mbar_wait;
                              // 100 / 400 ns on K1-sym2's producer and drain waits: +-0)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
#if NCGP_WAIT_CHEAP
  // the polling warps share issue slots with the epilogue: keep the loop to
  // the try, a counter and the branch, and check the time-out rarely
  uint32_t spins = 0;
  while (!mbar_try(bar, parity)) {
    if ((++spins & 255u) == 0u && clock64() - t0 > (1ll << 35)) __trap();
  }
#else
  while (!mbar_try(bar, parity)) {
#if NCGP_WAIT_NS > 0
    __nanosleep(NCGP_WAIT_NS);
#endif
    if (clock64() - t0 > (1ll << 35)) __trap();
  }
#endif
}
// For waits off the critical path (a producer waiting for a free slot, a
// drain warp waiting for its accumulator): back off between tries.
__device__ __forceinline__ void mbar_wait_relaxed(uint64_t* bar, uint32_t parity) {
#if NCGP_WAIT_RELAX_NS > 0
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  uint32_t spins = 0;
  while (!mbar_try(bar, parity)) {
    __nanosleep(NCGP_WAIT_RELAX_NS);
    if ((++spins & 255u) == 0u && clock64() - t0 > (1ll << 35)) __trap();
  }
#else
  mbar_wait(bar, parity);
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Arrive (once) on the barrier at this smem offset in BOTH CTAs of the pair
// when all previously issued tcgen05 ops of this thread have completed.
__device__ __forceinline__ void tc_commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// Same, but arriving only on the leader CTA's barrier.
__device__ __forceinline__ void tc_commit2_leader(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)1)
      : "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` in the leader CTA (rank 0)
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T  (both K-major)
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]^T
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// the same, kind::f8f6f4 (E4M3 x E4M3); A MN-major via the idesc bit
__device__ __forceinline__ void mma_f8_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]));
}
// hi (16 columns) then lo (16 columns): one 32-column store
__device__ __forceinline__ void tmem_st_hilo(uint32_t taddr, const uint32_t (&h)[16],
                                             const uint32_t (&l)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]),
      "r"(h[8]), "r"(h[9]), "r"(h[10]), "r"(h[11]), "r"(h[12]), "r"(h[13]), "r"(h[14]),
      "r"(h[15]), "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]), "r"(l[4]), "r"(l[5]), "r"(l[6]),
      "r"(l[7]), "r"(l[8]), "r"(l[9]), "r"(l[10]), "r"(l[11]), "r"(l[12]), "r"(l[13]),
      "r"(l[14]), "r"(l[15]));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// wait::ld that also "defines" the destination registers of an in-flight
// tcgen05.ld, so the compiler cannot copy them (e.g. across a loop back-edge)
// before the data has landed.
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.wait::ld.sync.aligned;"
      : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
        "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
        "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]),
        "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]),
        "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
      :
      : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// TMA bulk reduction shared -> global (fp32 add), one bulk group per call
__device__ __forceinline__ void bulk_reduce_add_f32(float* gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile(
      "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;\n\t"
      "cp.async.bulk.commit_group;" ::"l"(gdst),
      "r"(ssrc), "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// all but the most recent bulk group have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
// TMA bulk reduction shared -> global (u64 add: two's-complement int64 sums)
__device__ __forceinline__ void bulk_reduce_add_u64(unsigned long long* gdst, uint32_t ssrc,
                                                    uint32_t bytes) {
  asm volatile(
      "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;\n\t"
      "cp.async.bulk.commit_group;" ::"l"(gdst),
      "r"(ssrc), "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// pack (lo element, hi element) -> f16x2 with lo in the low half
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// Shared-memory matrix descriptor, K-major, no swizzle (canonical layout
// ((8,m),(8,2)) : ((16B, SBO), (2B, LBO)) in bytes).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
// Instruction descriptor: kind::f16, A/B = F16 (K-major), D = F32,
// M = 256 (a CTA pair, 128 rows per CTA).
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}


struct TcParams {
  const uint8_t* xa_pack;
  const uint8_t* col_pack;
  int64_t tile_stride;   // bytes between column-tile records
  uint32_t rec_bytes;    // one CTA's half record (offset of CTA1's half)
  uint32_t a_bytes;      // one packed 128-row tile
  uint32_t xbh_bytes;    // half an XB tile (64 rows)
  uint32_t v2_bytes;     // WP rows x 128 columns fp16 (GEMM2 B half, N = 2 WP)
  uint32_t v3_bytes;     // WP/2 rows (GEMM2 B half, N = WP)
  int ka;                // K of GEMM1 (multiple of 16)
  int w;                 // real RHS width
  int64_t rt0;           // first global row tile of this launch (even)
  int64_t pairs;         // local row-tile pairs
  int64_t nloc;          // local rows
  int64_t col_tiles;
  int splits;
  int64_t tiles_per_split;
  float L;               // log2(s2 * 2^s): Matern exponent offset
  const int* col_exp;    // per RHS column exponent e_c
  int s_exp;             // kernel prescale exponent s
  void* outs[NCGP_MAX_OUTS];  // destinations, offset to this launch's first row
  int n_out;
  int64_t ldo;
  int out_f64;
  double* partial;       // [splits][nloc][w] when splits > 1
  int na;                // row-tile buffers in shared memory (1 or 2)
  int sx, sv;            // XB ring depth (3 or 6), V ring depth (6 or 9)
  long long* trace;      // debug: per-tile timestamps of cluster 0 (nullptr in production)
  int n_items;           // work items: pairs * splits, or the symmetric item table's length
  const int4* item_tab;  // symmetric kernel: (row-tile pair, c0, c1, -) per item
  // symmetric kernel: int64 fixed-point accumulator [WP/8][acc_rows][8] (zeroed), the
  // 8-column groups of 32 rows contiguous (2 KB, one bulk reduction each); an fp32
  // partial x (kernel's scaled domain) adds round(x * fx), fx = 2^F
  unsigned long long* acc;
  int64_t acc_rows;
  float fx, fxi;
  int sym_dbg;           // symmetric kernel variant bits (correct results): 64 = flip whether
                         // T(g) is held back behind GEMM1(g + NS); 128 (single-CTA kernel) =
                         // GEMM2 reads P from TMEM (TS), as measured slower.  Debug
                         // instantiations only (timing / diagnosis, wrong results): 1 = drop
                         // D_T reductions, 2 = drop O reductions, 4 = no transposed MMAs,
                         // 8 = no D_T loads, 16 = no P stores to shared memory
  EpiDev epi;            // plain kernel, splits == 1: the apply's epilogue at the row store
  float* sym_dump;       // symmetric kernel debug: raw D_T per (pair, tile, rank) when set
  int npb;               // symmetric kernel: P buffers in shared memory (2, or 1 for large D)
  const uint8_t* v8_pack;  // blocked symmetric kernel: per column tile, Vhi in E4M3 (x 2^-LO8_SHIFT)
  uint32_t v8_bytes;       // WP x 128 bytes (K-major, 8-row groups at 1024 B)
  int nblk;                // blocked symmetric kernel: 2 KB staging blocks per drain warp
  int debug_mode;        // debug (timing only, wrong results): 1 = epilogue skips TMEM traffic,
                         // 2 = no GEMM2, 3 = no GEMM1, 4 = no column copies (8: XB only, 9: V only)
};

template <bool DBG>
__device__ __forceinline__ void trace_ev(const TcParams& p, uint32_t tile, int ev) {
  if (DBG && p.trace != nullptr && blockIdx.x == 0 && tile < (uint32_t)TRACE_TILES)
    p.trace[tile * TRACE_EV + ev] = clock64();
}

struct Item {
  int pp, c0, c1;  // row-tile pair, column-tile range
};

__device__ __forceinline__ Item item_of(const TcParams& p, int it) {
  Item r;
  if (p.item_tab != nullptr) {
    const int4 t = p.item_tab[it];
    r.pp = t.x;
    r.c0 = t.y;
    r.c1 = t.z;
    return r;
  }
  r.pp = it / p.splits;
  const int sp = it - r.pp * p.splits;
  r.c0 = sp * (int)p.tiles_per_split;
  r.c1 = min((int)p.col_tiles, r.c0 + (int)p.tiles_per_split);
  return r;
}

// Iterates the cluster's global column-tile sequence across its items.
struct TileIter {
  int it, ct;
  Item cur;
  bool valid;
  __device__ __forceinline__ void start(const TcParams& p, int items) {
    it = (int)(blockIdx.x >> 1);
    valid = it < items;
    if (valid) {
      cur = item_of(p, it);
      ct = cur.c0;
    }
  }
  __device__ __forceinline__ void next(const TcParams& p, int items) {
    if (++ct >= cur.c1) {
      it += (int)(gridDim.x >> 1);
      valid = it < items;
      if (valid) {
        cur = item_of(p, it);
        ct = cur.c0;
      }
    }
  }
  __device__ __forceinline__ bool first_in_item() const { return ct == cur.c0; }
  // symmetric kernel: this tile's P also serves the transposed product
  // (column tiles right of the pair's 256 x 256 diagonal block)
  __device__ __forceinline__ bool transposed() const { return ct >= 2 * cur.pp + 2; }
  __device__ __forceinline__ bool last_in_item() const { return ct == cur.c1 - 1; }
  __device__ __forceinline__ bool first_in_chunk() const {
    return ct == cur.c0 || (ct & (CH - 1)) == 0;
  }
  __device__ __forceinline__ bool last_in_chunk() const {
    return ct == cur.c1 - 1 || (ct & (CH - 1)) == CH - 1;
  }
};

// Position in a ring of mbarrier-guarded slots (no divisions on the hot path).
struct Ring {
  uint32_t idx, phase, size;
  __device__ __forceinline__ void init(uint32_t n) {
    idx = 0;
    phase = 0;
    size = n;
  }
  __device__ __forceinline__ void adv() {
    if (++idx == size) {
      idx = 0;
      phase ^= 1u;
    }
  }
};

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// Kernel transform of one 32-column chunk: S (fp32 exponent argument) ->
// P_hi / P_lo packed fp16 pairs.
template <int FAM>
__device__ __forceinline__ void transform_chunk(const uint32_t (&r)[32], float L,
                                                uint32_t (&hi)[16], uint32_t (&lo)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    float k0, k1;
    const float g0 = __uint_as_float(r[2 * i]);
    const float g1 = __uint_as_float(r[2 * i + 1]);
    if (FAM == NCGP_RBF) {
      k0 = ex2(g0);  // g <= L up to the rounding of the d^2 expansion
      k1 = ex2(g1);
    } else {
      const float a0 = sqrt_approx(fmaxf(g0, 0.f));
      const float a1 = sqrt_approx(fmaxf(g1, 0.f));
      const float e0 = ex2(fmaf(a0, -1.4426950408889634f, L));
      const float e1 = ex2(fmaf(a1, -1.4426950408889634f, L));
      k0 = fmaf(a0, e0, e0);
      k1 = fmaf(a1, e1, e1);
    }
    const float h0 = __uint_as_float(__float_as_uint(k0) & 0xFFFFE000u);
    const float h1 = __uint_as_float(__float_as_uint(k1) & 0xFFFFE000u);
    hi[i] = pack_h2(h0, h1);
    lo[i] = pack_h2(k0 - h0, k1 - h1);
  }
}

// Deterministic accumulation of the symmetric kernels.  Every flushed fp32
// partial (O chunk or transposed tile, in the kernel's scaled domain) is
// rounded to an int64 multiple of 2^-F and added to the global accumulator
// with an integer bulk reduction.  Integer addition is associative and
// commutative, so the sums do not depend on the order in which CTAs flush,
// on the number of CTAs, or on how the work list is split across processes:
// the product is bitwise reproducible (hard part 5) and 1-GPU
// and N-GPU results are identical.  |P V| < 2^28 per pair after the fp16
// prescaling, so a flush (<= 2048 columns) is below 2^39 and the sum below
// n 2^28: F = min(3, 33 - ceil(log2 n)) keeps every flush below 2^42 (the
// conversion's range) and the sum below 2^62, at a resolution of 2^-31 of
// the largest entry scale.
// fp32 -> int64 round-to-nearest for |v| < 2^43 on the FMA / ALU pipes: two
// 21-bit limbs, each rounded with the 1.5 * 2^23 magic constant
// (cvt.rni.s64.f32 executes on the XU pipe at the MUFU's 16 per clock and
// would compete with the epilogue's ex2; tools/cvt_probe.cu).  s is the
// unscaled partial, fx = 2^F, fxi = 2^(21 - F).
__device__ __forceinline__ long long fx_round(float s, float fx, float fxi) {
  const float M = 12582912.0f;
  const float th = fmaf(s, fx * 0x1p-21f, M);   // rint(s 2^F / 2^21) + M
  const float hf = th - M;
  const float rs = fmaf(hf, -fxi, s);           // s - h 2^(21 - F), exact
  const float tl = fmaf(rs, fx, M);             // rint(rs 2^F) + M, |rs 2^F| <= 2^20
  const long long h = (long long)(__float_as_int(th) - 0x4B400000);
  return (h << 21) + (long long)(__float_as_int(tl) - 0x4B400000);
}
// One call adds 8 columns (group h) of the warp's 32 rows (one per lane)
// through a 2 KB staging block (row r at 64 r, 16-byte chunk k at
// k ^ ((r >> 1) & 3): conflict-free stores); NBLK blocks per warp rotate.
template <uint32_t NBLK>
__device__ __forceinline__ void fx_flush8(const TcParams& p, uint32_t stg_warp, uint32_t& nst,
                                          int lane, int h, const float (&v)[8], int64_t row0,
                                          bool skip) {
  if (lane == 0) {
    if (NBLK == 2)
      bulk_wait_read1();  // the block written two flushes ago has been read
    else
      bulk_wait_read();
  }
  __syncwarp();
  const uint32_t blk = stg_warp + (nst & (NBLK - 1u)) * 2048u;
  ++nst;
  const uint32_t rowa = blk + (uint32_t)lane * 64u;
  const uint32_t swz = (uint32_t)((lane >> 1) & 3);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
#if NCGP_FX_CVT == 0
    const long long q0 = __float2ll_rn(v[2 * k] * p.fx);
    const long long q1 = __float2ll_rn(v[2 * k + 1] * p.fx);
#else
    const long long q0 = fx_round(v[2 * k], p.fx, p.fxi);
    const long long q1 = fx_round(v[2 * k + 1], p.fx, p.fxi);
#endif
    st_shared_v4(rowa + 16u * ((uint32_t)k ^ swz), (uint32_t)q0, (uint32_t)((unsigned long long)q0 >> 32),
                 (uint32_t)q1, (uint32_t)((unsigned long long)q1 >> 32));
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0 && !skip) bulk_reduce_add_u64(p.acc + ((int64_t)h * p.acc_rows + row0) * 8, blk, 2048u);
}

// ---- shared by the blocked symmetric kernel (K1-sym2) and the pair kernel's
// E4M3 split term (NCGP_PAIR_F8); see the K1-sym2 section below
#ifndef NCGP_SYM2_RB
#define NCGP_SYM2_RB 4  // row tiles per block (build-time A/B: 4 or 2)
#endif
#ifndef NCGP_SYM2_NS
#define NCGP_SYM2_NS 1  // S buffers in TMEM (build-time A/B: 1 or 2)
#endif
#ifndef NCGP_SYM2_NP
#define NCGP_SYM2_NP 2  // P regions in TMEM (build-time A/B: 2 or 1)
#endif
constexpr int RB = NCGP_SYM2_RB;            // row tiles per block
constexpr int LO8_SHIFT = 6;                // P_lo * 2^6, Vhi * 2^-6 in E4M3
constexpr uint32_t PH2 = BM * BN * 2;       // P_hi (fp16, MN-major for T)
constexpr uint32_t P2BUF = PH2 + BM * BN;   // [P_hi | P_lo E4M3]: 48 KB
constexpr int NR2 = 16;                     // per-tile barrier rings (power of two)
constexpr uint32_t TP2 = 96;                // TMEM columns of one P region (hi 64 | lo8 32)
#ifndef NCGP_SYM2_HOLD
#define NCGP_SYM2_HOLD 0  // build-time A/B: T(g) issued only after GEMM1(g + HOLD)
#endif
#ifndef NCGP_SYM2_HOLDG2
#define NCGP_SYM2_HOLDG2 0  // build-time A/B: GEMM2(g) issued only after GEMM1(g + HOLDG2)
#endif
#ifndef NCGP_SYM2_LATE
#define NCGP_SYM2_LATE 0  // epilogue: both chunks transformed before the P-buffer waits and stores
                          // (build-time A/B; measured slower: cfg3 293.1 vs 280.9 ms, n = 2e5 10.48 vs 9.75 ms)
#endif
#ifndef NCGP_SYM2_REG_LO
#define NCGP_SYM2_REG_LO 40  // registers of the producer / MMA-issuing warps (build-time A/B)
#endif
#ifndef NCGP_SYM2_REG_DR
#define NCGP_SYM2_REG_DR 56  // registers of the drain warps; LO * 4 + DR * 4 + 96 * 16 <= 80 * 24
                             // (32 / 64: drain spills 220 -> 136 B, cfg3 282.3 vs 282.2 ms: +-0)
#endif
#ifndef NCGP_SYM2_ABL
#define NCGP_SYM2_ABL 0  // timing ablations (wrong results): 1 no T MMAs, 2 no P stores for T,
                         // 4 no GEMM2 f16 MMAs, 8 no accumulator flushes, 16 no E4M3 conversion
#endif

__device__ __forceinline__ void mma1_f8_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma1_f8_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// kind::f8f6f4, A/B E4M3, D F32, M = 128; bit 15: A MN-major
__host__ __device__ constexpr uint32_t idesc1_f8(int n, bool a_mn) {
  return (1u << 4) | (a_mn ? (1u << 15) : 0u) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
// two floats -> E4M3x2 (a in the low byte)
__device__ __forceinline__ uint32_t e4m3x2(float a, float b) {
  uint16_t d;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(d) : "f"(b), "f"(a));
  return (uint32_t)d;
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}

// One 32-column chunk: S -> P_hi (fp16, rounded to nearest) and P_lo * 2^6 (E4M3).
template <int FAM>
__device__ __forceinline__ void transform_chunk2(const uint32_t (&r)[32], float L,
                                                 uint32_t (&hi)[16], uint32_t (&l8)[8]) {
  constexpr float S8 = (float)(1 << LO8_SHIFT);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    float k0, k1;
    const float g0 = __uint_as_float(r[2 * i]);
    const float g1 = __uint_as_float(r[2 * i + 1]);
    if (FAM == NCGP_RBF) {
      k0 = ex2(g0);
      k1 = ex2(g1);
    } else {
      const float a0 = sqrt_approx(fmaxf(g0, 0.f));
      const float a1 = sqrt_approx(fmaxf(g1, 0.f));
      const float e0 = ex2(fmaf(a0, -1.4426950408889634f, L));
      const float e1 = ex2(fmaf(a1, -1.4426950408889634f, L));
      k0 = fmaf(a0, e0, e0);
      k1 = fmaf(a1, e1, e1);
    }
    // round to the nearest value with 11 significant bits (fp16-exact)
    const float h0 = __uint_as_float((__float_as_uint(k0) + 0x1000u) & 0xFFFFE000u);
    const float h1 = __uint_as_float((__float_as_uint(k1) + 0x1000u) & 0xFFFFE000u);
    hi[i] = pack_h2(h0, h1);
    const uint32_t q = (NCGP_SYM2_ABL & 16) ? __float_as_uint(k0 - h0) & 0xFFFFu
                                            : e4m3x2((k0 - h0) * S8, (k1 - h1) * S8);
    if (i & 1)
      l8[i >> 1] |= q << 16;
    else
      l8[i >> 1] = q;
  }
}

// The same 8 columns of the warp's 32 rows straight from registers: one
// coalesced red.global.add.u64 per column into the column-major [WP][rows]
// accumulator -- no shared-memory staging, no TMA queueing behind the
// producers' loads (K1-sym2 and, with NCGP_SYM1_RED / NCGP_PAIR_RED, the
// other symmetric kernels; sym_finalize_kernel(colmajor = 1) reads it).
__device__ __forceinline__ void fx_red8(const TcParams& p, int lane, int h, const float (&v)[8],
                                        int64_t row0, bool skip) {
  if (skip) return;
  unsigned long long* dst = p.acc + row0 + lane;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    atomicAdd(dst + (int64_t)(8 * h + c) * p.acc_rows, (unsigned long long)__float2ll_rn(v[c] * p.fx));
}

// ATM (symmetric kernel, WP = 16, large D): the row tile lives in TMEM (the
// drain warps load it per item; GEMM1 becomes a TS MMA), which frees its
// shared memory for the two P buffers.
template <int FAM, int WP, bool DBG, bool SYM, bool ATM = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    kop_tc_kernel(const TcParams p) {
  static_assert(!ATM || (SYM && WP == 16), "row tile in TMEM: symmetric kernel, WP = 16");
  // WP = 128: the wide-RHS kernel (K2, posterior variance and products with
  // 32 < w <= 128).  The three split terms P_hi Vhi + P_hi Vlo + P_lo Vhi
  // accumulate into one set of 128 TMEM columns (N = 128 MMAs on the
  // CTA-split B blocks [Vhi half | Vlo half]), so O is double-buffered next
  // to two S buffers; every item (row-tile pair x <= 16 column tiles, K1's
  // fp32 accumulation span) leaves an fp32 partial row block in HBM, summed
  // in fp64 by the reduce pass.
  constexpr bool WIDE = WP == 128;
  static_assert(!WIDE || !SYM, "the wide kernel is the plain kernel");
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const int items = p.n_items;
  // S/P buffers in TMEM.  The symmetric kernel double-buffers its O and D_T
  // accumulators (2 x 2 WP columns each): with WP = 32 that leaves room for
  // two S/P buffers only, with WP = 16 for three.
  constexpr int NS = (WIDE || (SYM && (WP == 32 || ATM))) ? 2 : NS_MAX;
  // NCGP_PAIR_F8: P_lo in E4M3 ([P_hi | P_lo8] buffers of 48 KB, up to three),
  // Vhi in E4M3 next to each V slot (this CTA's half) and the own V block (full)
  constexpr bool PF8 = SYM && NCGP_PAIR_F8;
  constexpr uint32_t PB = PF8 ? P2BUF : PBUF;

  // ---- shared-memory carve-up (identical offsets in both CTAs)
  // this CTA's V half: [B2 | B3] (wide kernel: [B3 | B4], the CTA-split Vhi and Vlo)
  const uint32_t vslot0 = WIDE ? 2u * p.v3_bytes : p.v2_bytes + p.v3_bytes;
  const uint32_t v8h = PF8 ? p.v8_bytes / 2u : 0u;  // this CTA's half of the column tile's Vhi8
  const uint32_t vslot = vslot0 + v8h;
  uint8_t* sA = smem;                                   // na x a_bytes (own row tile)
  uint8_t* sXB = sA + (size_t)p.na * p.a_bytes;         // sx x xbh_bytes
  uint8_t* sV = sXB + (size_t)p.sx * p.xbh_bytes;       // sv x vslot
  // symmetric kernel: this CTA's own V block [Vhi | Vlo] (the transposed
  // product's B) and two P buffers [P_hi | P_lo] (its MN-major A)
  uint8_t* sVI = sV + (size_t)p.sv * vslot;
  uint8_t* sP = sVI + (SYM ? 2 * (size_t)p.v2_bytes + (PF8 ? p.v8_bytes : 0u) : 0);
  // symmetric kernel: fp32 staging rows [128][WP] for the bulk reductions
  float* sStage = reinterpret_cast<float*>(sP + (SYM ? (size_t)p.npb * PB : 0));
  // symmetric kernel: P buffer of tile g (two alternate by tile parity; one
  // when shared memory is short).  GEMM2(g) and T(g) always commit to
  // pt_free[g & 1], whose phases then advance once per two tiles; the
  // epilogue of tile g waits for tile g - npb's phase, which with one buffer
  // is the other group's barrier.  A single barrier would let a group, which
  // only sees every other phase, alias a phase two behind as complete.
  auto pbuf = [&](uint32_t g) -> uint32_t {
    return PF8 ? g % (uint32_t)p.npb : (p.npb == 2 ? (g & 1u) : 0u);
  };
  // pt_free barrier of tile g and its phase: two alternating (a group sees
  // every other phase), or with PF8 a ring of 6 (no waiter lags 6 tiles)
  auto ptb = [&](uint32_t g) -> uint32_t { return PF8 ? g % 6u : (g & 1u); };
  auto ptph = [&](uint32_t g) -> uint32_t { return PF8 ? (g / 6u) & 1u : (g >> 1) & 1u; };
  double* sAcc = reinterpret_cast<double*>(sStage + (SYM ? BM * WP : 0));  // [WP][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sAcc + ((SYM || WIDE) ? 0 : WP * BM));
  uint64_t* xb_land = bars;               // [6]   local copy completion
  uint64_t* v_land = xb_land + 6;         // [9]   local copy completion
  uint64_t* a_land = v_land + 9;          // [2]   local copy completion
  uint64_t* xb_pro = a_land + 2;          // [NS]  leader: XB of tiles 0..NS-1 landed (2 halves)
  // rdy[g mod NR] (leader): everything step g of the MMA warp needs -- P(g)
  // written (8 epilogue warps), V(g) landed (2 halves), XB(g + NS) landed (2
  // halves) -- so the MMA warp waits once per step.  A wait issued behind
  // in-flight tcgen05 ops stalls the tensor pipe ~130 cycles
  // (tools/mma2sm_pattern.cu), so waits in the MMA warp are kept to a minimum.
  uint64_t* rdy = xb_pro + NS;            // [NR]
  uint64_t* a_full = rdy + NR;            // [2]   leader: both row tiles landed
  uint64_t* a_empty = a_full + 2;         // [2]   both: row tile free (multicast commit)
  uint64_t* s_full = a_empty + 2;         // [NR]  both: GEMM1 of a tile done (multicast)
  uint64_t* o_full = s_full + NR;         // [2]   both: O chunk complete (multicast)
  uint64_t* o_empty = o_full + 2;         // [2]   leader: O drained (8 warp arrivals)
  uint64_t* g2done = o_empty + 2;         // [NR]  leader: GEMM2 of a step done (commit)
  uint64_t* vi_land = g2done + NR;        // [1]   SYM: local V block landed
  uint64_t* vi_full = vi_land + 1;        // [1]   SYM leader: both V blocks landed
  uint64_t* vi_empty = vi_full + 1;       // [1]   SYM both: V block free (multicast commit)
  uint64_t* pt_free = vi_empty + 1;       // [2 / 6] SYM both: P buffer free (multicast commit)
  uint64_t* dt_full = pt_free + (PF8 ? 6 : 2);  // [2] SYM both: transposed product done
  uint64_t* dt_empty = dt_full + 2;       // [2]   SYM leader: D_T drained (8 warp arrivals)
  uint64_t* s_free = dt_empty + 2;        // [NR]  SYM leader: S(g) loaded by the epilogue (16 warps)
  uint64_t* xb_full = s_free + NR;        // [NR]  SYM leader: XB(g) landed (2 halves)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xb_full + NR);
  // SYM leader: GEMM1 tiles issued so far (the transposed issuer queues T(g)
  // behind GEMM1(g + NS) in the in-order tensor pipe)
  volatile uint32_t* g1_cnt = tmem_slot + 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 6; ++s) mbar_init(&xb_land[s], 1);
    for (int s = 0; s < 9; ++s) mbar_init(&v_land[s], 1);
    for (int s = 0; s < NS; ++s) mbar_init(&xb_pro[s], 2);
    for (int s = 0; s < NR; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&g2done[s], 1);
      // epilogue group (8 warps x 2 CTAs), V, XB (symmetric kernel: XB has its own ring)
      mbar_init(&rdy[s], SYM ? 16 + 2 : 16 + 2 + 2);
      mbar_init(&s_free[s], 16);
      mbar_init(&xb_full[s], 2);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&a_land[b], 1);
      mbar_init(&a_full[b], ATM ? 8 : 2);  // ATM: 4 drain warps x 2 CTAs
      mbar_init(&a_empty[b], 1);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 8);
      mbar_init(&pt_free[b], (SYM && !NCGP_PAIR_PT) ? 2 : 1);  // SYM: GEMM2(g) and T(g) both read P(g)
      if (PF8) {
        mbar_init(&pt_free[2 + 2 * b], (SYM && !NCGP_PAIR_PT) ? 2 : 1);
        mbar_init(&pt_free[3 + 2 * b], (SYM && !NCGP_PAIR_PT) ? 2 : 1);
      }
      mbar_init(&dt_full[b], 1);
      mbar_init(&dt_empty[b], 8);
    }
    mbar_init(vi_land, 1);
    mbar_init(vi_full, 2);
    mbar_init(vi_empty, 1);
    *g1_cnt = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive
  if (DBG && p.trace != nullptr && threadIdx.x == 0) {  // per-CTA span (global timer, ns)
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[TRACE_TILES * TRACE_EV + 4 * blockIdx.x] = (long long)t;
  }
  tc_fence_after();
  // warp-uniform (see kop_sym2_kernel): MMA operands derived from it stay in
  // uniform registers instead of a per-MMA ELECT / R2UR waterfall loop
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  // TMEM columns: S/P buffers [0, 384), O double buffer [384, 384 + 4 WP);
  // symmetric kernel: S/P [0, 256), O double buffer [256, 256 + 4 WP),
  // D_T double buffer [256 + 4 WP, 256 + 8 WP)
  auto tS = [&](int b) -> uint32_t { return tmem + (uint32_t)(b * BN); };
  constexpr uint32_t AW = WIDE ? WP : 2 * WP;  // TMEM columns of one O accumulator
  auto tO = [&](int b) -> uint32_t { return tmem + (uint32_t)(NS * BN) + (uint32_t)b * AW; };
  auto tDT = [&](uint32_t b) -> uint32_t { return tmem + (uint32_t)(NS * BN + 4 * WP) + b * 2u * WP; };
  const uint32_t tA = tmem + (uint32_t)(NS * BN + 8 * WP);  // ATM: row tile, ka / 2 columns
  constexpr uint32_t NO = 2u;  // O buffers
  const int64_t half_off = (int64_t)rank * p.rec_bytes;   // this CTA's half of a record

  // setmaxnreg sits at the top of each warpgroup's branch so that ptxas sees
  // one register budget per region (a shared prologue would cap all at 40).
  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
  if (warp == 0 || (!SYM && warp == 3)) {
    // ================= producers (lane 0) and relays (lane 1) =================
    // (symmetric kernel: all four in warp 0 -- lanes 0/1 XB, lanes 2/3 V --
    // so warp 3 can issue the transposed product)
    // Slot reuse is signalled by GEMM1 completions (s_full, one multicast commit
    // per tile): XB slot g mod sx is free once GEMM1(g - sx) completed; V slot
    // g mod sv once GEMM2(g - sv) did, which the in-order tensor pipe finishes
    // before GEMM1(g - sv + NS).  s_full has NR >= max(sx, sv) entries so no
    // waiter can lag two phases.  Relays forward this CTA's copy completions
    // to the leader CTA's barriers (the MMA consumes both CTAs' halves).
    const bool is_x = SYM ? (lane < 2) : (warp == 0);
    const int role = SYM ? (lane < 4 ? (lane & 1) : lane - 2) : lane;  // 0/1 producer/relay
    // (symmetric kernel: lane 4 loads this CTA's own V block per item, lane 5
    // relays it; separate loops, because vi_empty depends on rdy, which
    // depends on the XB stream running ahead)
    const uint32_t depth = is_x ? (uint32_t)p.sx : (uint32_t)p.sv;
    // symmetric kernel: GEMM1 no longer waits for GEMM2, so V slots are
    // released by GEMM2's own completion (g2done, multicast)
    const uint32_t lagt = is_x ? (uint32_t)p.sx : (SYM ? depth : (uint32_t)(p.sv - NS));  // tile g - lagt
    uint64_t* rel = (SYM && !is_x) ? g2done : s_full;
    uint64_t* land = is_x ? xb_land : v_land;
    if (role == 0) {
      TileIter ti;
      ti.start(p, items);
      Ring r, sr;
      r.init(depth);
      sr.init(NR);
      uint32_t nitem = 0, g = 0;
      while (ti.valid) {
        if (!ATM && is_x && ti.first_in_item()) {
          const uint32_t ab = p.na == 2 ? (nitem & 1u) : 0u;
          const uint32_t aph = p.na == 2 ? ((nitem >> 1) & 1u) : (nitem & 1u);
          mbar_wait(&a_empty[ab], aph ^ 1u);
          mbar_expect_tx(&a_land[ab], p.a_bytes);
          const int64_t rt = p.rt0 + 2 * (int64_t)ti.cur.pp + rank;
          bulk_g2s(sA + ab * p.a_bytes, p.xa_pack + rt * (int64_t)p.a_bytes, p.a_bytes,
                   &a_land[ab]);
          ++nitem;
        }
        if (g >= depth) mbar_wait(&rel[sr.idx], sr.phase);
        const int64_t src = (int64_t)ti.ct * p.tile_stride + half_off;
        if (DBG && (p.debug_mode == 4 || p.debug_mode == 5 || p.debug_mode == (is_x ? 8 : 9))) {
          mbar_expect_tx(&land[r.idx], 0);  // timing only: no copy
        } else if (is_x) {
          mbar_expect_tx(&land[r.idx], p.xbh_bytes);
          bulk_g2s(sXB + (size_t)r.idx * p.xbh_bytes, p.col_pack + src, p.xbh_bytes,
                   &land[r.idx]);
        } else {
          mbar_expect_tx(&land[r.idx], vslot);
          bulk_g2s(sV + (size_t)r.idx * vslot, p.col_pack + src + p.xbh_bytes, vslot0,
                   &land[r.idx]);
          if (PF8)  // this CTA's half (rows) of the column tile's Vhi8
            bulk_g2s(sV + (size_t)r.idx * vslot + vslot0,
                     p.v8_pack + (int64_t)ti.ct * p.v8_bytes + (int64_t)rank * v8h, v8h, &land[r.idx]);
        }
        r.adv();
        if (g >= lagt) sr.adv();
        ++g;
        ti.next(p, items);
      }
    } else if (SYM && role == 2) {
      uint32_t nitem = 0;
      for (int it = (int)(blockIdx.x >> 1); it < items; it += (int)(gridDim.x >> 1), ++nitem) {
        const Item cur = item_of(p, it);
        mbar_wait(vi_empty, (nitem & 1u) ^ 1u);
        mbar_expect_tx(vi_land, 2 * p.v2_bytes + (PF8 ? p.v8_bytes : 0u));
        // Vhi of column tile rt sits in the record's CTA0 half, Vlo in its CTA1 half
        const int64_t rt = p.rt0 + 2 * (int64_t)cur.pp + rank;
        const int64_t vb = rt * p.tile_stride + p.xbh_bytes;
        bulk_g2s(sVI, p.col_pack + vb, p.v2_bytes, vi_land);
        bulk_g2s(sVI + p.v2_bytes, p.col_pack + vb + p.rec_bytes, p.v2_bytes, vi_land);
        if (PF8) bulk_g2s(sVI + 2 * p.v2_bytes, p.v8_pack + rt * p.v8_bytes, p.v8_bytes, vi_land);
      }
    } else if (SYM && role == 3) {
      uint32_t nitem = 0;
      for (int it = (int)(blockIdx.x >> 1); it < items; it += (int)(gridDim.x >> 1), ++nitem) {
        mbar_wait(vi_land, nitem & 1u);
        mbar_arrive_cluster(leader_addr(vi_full));
      }
    } else if (role == 1) {
      TileIter ti;
      ti.start(p, items);
      Ring r, rr;
      r.init(depth);
      rr.init(NR);
      uint32_t nitem = 0, g = 0;
      while (ti.valid) {
        if (!ATM && is_x && ti.first_in_item()) {
          const uint32_t ab = p.na == 2 ? (nitem & 1u) : 0u;
          const uint32_t aph = p.na == 2 ? ((nitem >> 1) & 1u) : (nitem & 1u);
          mbar_wait(&a_land[ab], aph);
          mbar_arrive_cluster(leader_addr(&a_full[ab]));
          ++nitem;
        }
        mbar_wait(&land[r.idx], r.phase);
        // V(g) -> rdy[g]; XB(t) -> rdy[t - NS] (prologue tiles: xb_pro[t])
        if (!is_x)
          mbar_arrive_cluster(leader_addr(&rdy[rr.idx]));
        else if (SYM)
          mbar_arrive_cluster(leader_addr(&xb_full[rr.idx]));
        else if (g < (uint32_t)NS)
          mbar_arrive_cluster(leader_addr(&xb_pro[g]));
        else
          mbar_arrive_cluster(leader_addr(&rdy[rr.idx]));
        if (!is_x || SYM || g >= (uint32_t)NS) rr.adv();
        r.adv();
        ++g;
        ti.next(p, items);
      }
      // the last NS steps have no XB(g + NS): stand in for those arrivals
      if (is_x && !SYM)
        for (uint32_t t = g < (uint32_t)NS ? (uint32_t)NS : g; t < g + (uint32_t)NS; ++t) {
          mbar_arrive_cluster(leader_addr(&rdy[rr.idx]));
          rr.adv();
        }
    }
  } else if (warp == 1 || warp == 2 || (SYM && warp == 3)) {
    // ================= MMA issuers (leader CTA; whole warp, elected lane issues) =====
    // One thread issues a tcgen05.mma only every ~46 cycles and blocks once
    // the ~7-deep tensor queue is full (tools/mma_queue_probe.cu), so the two
    // GEMMs get their own issuing warps: warp 1 issues GEMM2 (16 MMAs per
    // step), warp 2 issues GEMM1.  GEMM1(t) overwrites the S buffer GEMM2(t -
    // NS) reads, so warp 2 waits for GEMM2(t - NS)'s completion (g2done) first.
    if (rank == 0) {
      const uint32_t id1 = idesc_f16(BN), id2 = idesc_f16(2 * WP), id2h = idesc_f16(WP);
      if (warp == 2) {
        // ---------------- GEMM1 issuer
        const uint32_t sbo_x = (uint32_t)(p.ka / 8) * 128u;
        const int ksteps1 = p.ka / 16;
        const uint64_t dA0 = sdesc(smem_u32(sA), 128u, sbo_x);
        const uint64_t dX0 = sdesc(smem_u32(sXB), 128u, sbo_x);
        const uint64_t astep = p.a_bytes >> 4, xstep = p.xbh_bytes >> 4;
        const uint64_t xend = dX0 + (uint64_t)p.sx * xstep;
        TileIter look;
        look.start(p, items);
        uint64_t dx = dX0;
        uint32_t s1 = 0, c1 = 0, item1 = 0, g1n = 0, gd = 0, gdph = 0;
        while (look.valid) {
          const bool li = look.last_in_item();
          if (look.first_in_item()) {
            if (p.na == 2)
              mbar_wait(&a_full[item1 & 1u], (item1 >> 1) & 1u);
            else
              mbar_wait(&a_full[0], item1 & 1u);
            ++item1;
          }
          if (SYM) {  // XB(t) landed; S buffer free once the epilogue loaded S(t - NS)
            // (NCGP_PAIR_PT: once GEMM2(t - NS) has read P over it)
            mbar_wait(&xb_full[c1], (g1n / (uint32_t)NR) & 1u);
            if (g1n >= (uint32_t)NS) {
              mbar_wait(NCGP_PAIR_PT ? &g2done[gd] : &s_free[gd], gdph);
              if (++gd == (uint32_t)NR) {
                gd = 0;
                gdph ^= 1u;
              }
            }
          } else if (g1n < (uint32_t)NS) {
            mbar_wait(&xb_pro[g1n], 0);
          } else {  // S buffer free; XB(t) landed (it is part of rdy(t - NS))
            mbar_wait(&g2done[gd], gdph);
            if (++gd == (uint32_t)NR) {
              gd = 0;
              gdph ^= 1u;
            }
          }
          tc_fence_after();
          if (lane == 0) trace_ev<DBG>(p, g1n, 9);
          const uint32_t ab = p.na == 2 ? ((item1 - 1u) & 1u) : 0u;
          const uint64_t da = dA0 + ab * astep;
          const uint32_t d = tmem + s1 * (uint32_t)BN;
          const uint32_t liu = __shfl_sync(0xffffffffu, li ? 1u : 0u, 0);
          if (elect_one()) {
            if (ATM)  // A = this CTA's row tile in TMEM (8 columns per K step of 16)
              for (int k = 0; k < ksteps1; ++k)
                mma_ts(d, tA + 8u * k, dx + (uint64_t)(16 * k), id1, k > 0);
            else if (!(DBG && (p.debug_mode == 3 || p.debug_mode == 6)))
              for (int k = 0; k < ksteps1; ++k)
                mma_ss(d, da + (uint64_t)(16 * k), dx + (uint64_t)(16 * k), id1, k > 0);
            tc_commit2(&s_full[c1]);  // also releases XB / V slots (see producers)
            if (liu) tc_commit2(&a_empty[ab]);
          }
          __syncwarp();
          if (lane == 0) trace_ev<DBG>(p, g1n, 2);
          if (SYM && lane == 0) *g1_cnt = g1n + 1u;
          ++g1n;
          c1 = (c1 + 1u == (uint32_t)NR) ? 0u : c1 + 1u;
          s1 = (s1 + 1u == (uint32_t)NS) ? 0u : s1 + 1u;
          dx += xstep;
          if (dx == xend) dx = dX0;
          look.next(p, items);
        }
        if (SYM && lane == 0) *g1_cnt = 0xFFFFFFFFu;
      } else if (warp == 1) {
        // ---------------- GEMM2 issuer
        const uint64_t dV0 = sdesc(smem_u32(sV), 128u, (uint32_t)(BN * 16));
        const uint64_t vstep = vslot >> 4, vend = dV0 + (uint64_t)p.sv * vstep;
        const uint64_t v3off = p.v2_bytes >> 4;
        TileIter cur;
        cur.start(p, items);
        uint64_t dv = dV0;
        uint32_t s2 = 0, r = 0, rph = 0, q = 0, gt = 0;
        while (cur.valid) {
          // (wide kernel: one O accumulation per item)
          const bool fresh = WIDE ? cur.first_in_item() : cur.first_in_chunk();
          const bool last = WIDE ? cur.last_in_item() : cur.last_in_chunk();
          if (lane == 0) trace_ev<DBG>(p, gt, 11);
          mbar_wait(&rdy[r], rph);  // P(g), V(g) (and XB(g + NS)) present
          const uint32_t ob = NO == 2u ? (q & 1u) : 0u;
          if (fresh) mbar_wait(&o_empty[ob], ((q / NO) & 1u) ^ 1u);
          tc_fence_after();
          if (lane == 0) trace_ev<DBG>(p, gt, 0);
          // GEMM2: P_hi x [Vhi | Vlo] (N = 2 WP: CTA0 supplies Vhi, CTA1 Vlo), then
          // P_lo x Vhi (N = WP: each CTA supplies half of Vhi's rows).
          const uint32_t a0 = tmem + s2 * (uint32_t)BN;
          const uint32_t obu = __shfl_sync(0xffffffffu, ob, 0);
          const uint32_t fu = __shfl_sync(0xffffffffu, fresh ? 1u : 0u, 0);
          const uint32_t lu = __shfl_sync(0xffffffffu, last ? 1u : 0u, 0);
          const uint32_t dO = tO((int)obu);
          if (elect_one()) {
            if (SYM && NCGP_PAIR_PT) {
              // symmetric kernel, P in TMEM over S(g) (the plain kernel's TS MMAs);
              // the shared-memory copy is the transposed product's only
#pragma unroll
              for (int m = 0; m < BN / 16; ++m) {
                const uint32_t ahi = a0 + 32u * (m >> 1) + 8u * (m & 1);
                mma_ts(dO, ahi, dv + (uint64_t)(16 * m), id2, (fu && m == 0) ? 0u : 1u);
                mma_ts(dO, ahi + 16u, dv + v3off + (uint64_t)(16 * m), id2h, 1u);
              }
              tc_commit2(&g2done[r]);  // V slot g and S buffer g free (both CTAs)
            } else if (SYM) {
              // symmetric kernel: P(g) from shared-memory buffer g mod 2 (K-major
              // canonical layout, the same bytes the transposed product reads)
              const uint64_t ph = sdesc(smem_u32(sP) + pbuf(gt) * PB, 128u, 2048u);
              if (PF8) {  // P_hi [Vhi | Vlo] (f16) + P_lo8 Vhi8 (E4M3, K = 32, A K-major rows i)
                const uint64_t p8 = sdesc(smem_u32(sP) + pbuf(gt) * PB + PH2, 128u, 1024u);
                // this CTA's Vhi8 half behind the V slot: K-major, 8-row groups at 1024 B
                const uint64_t b8 = sdesc(0u, 128u, 1024u) | (((dv & 0x3FFFull) + (vslot0 >> 4)) & 0x3FFFull);
                constexpr uint32_t id28 = idesc1_f8(WP, false) + ((uint32_t)((256 - 128) >> 4) << 24);
#pragma unroll
                for (int m = 0; m < BN / 16; ++m)
                  mma_ss(dO, ph + (uint64_t)(16 * m), dv + (uint64_t)(16 * m), id2, (fu && m == 0) ? 0u : 1u);
#pragma unroll
                for (int q2 = 0; q2 < BN / 32; ++q2)
                  mma_f8_ss(dO, p8 + (uint64_t)(16 * q2), b8 + (uint64_t)(16 * q2), id28, 1u);
              } else {
                const uint64_t pl = ph + ((PBUF / 2) >> 4);
#pragma unroll
                for (int m = 0; m < BN / 16; ++m) {
                  mma_ss(dO, ph + (uint64_t)(16 * m), dv + (uint64_t)(16 * m), id2, (fu && m == 0) ? 0u : 1u);
                  mma_ss(dO, pl + (uint64_t)(16 * m), dv + v3off + (uint64_t)(16 * m), id2h, 1u);
                }
              }
              tc_commit2(&g2done[r]);           // V slot g free (both CTAs)
              tc_commit2(&pt_free[ptb(gt)]);    // with T(g): P(g)'s buffer free
            } else {
              if (WIDE) {  // P_hi Vhi, P_hi Vlo, P_lo Vhi into the same 128 columns
                const uint64_t b4 = (uint64_t)(p.v3_bytes >> 4);
#pragma unroll
                for (int m = 0; m < BN / 16; ++m) {
                  const uint32_t ahi = a0 + 32u * (m >> 1) + 8u * (m & 1);
                  const uint64_t b = dv + (uint64_t)(16 * m);
                  mma_ts(dO, ahi, b, id2h, (fu && m == 0) ? 0u : 1u);
                  mma_ts(dO, ahi, b + b4, id2h, 1u);
                  mma_ts(dO, ahi + 16u, b, id2h, 1u);
                }
              } else if (!(DBG && (p.debug_mode == 2 || p.debug_mode == 6))) {
#pragma unroll
                for (int m = 0; m < BN / 16; ++m) {
                  const uint32_t ahi = a0 + 32u * (m >> 1) + 8u * (m & 1);
                  mma_ts(dO, ahi, dv + (uint64_t)(16 * m), id2, (fu && m == 0) ? 0u : 1u);
                  mma_ts(dO, ahi + 16u, dv + v3off + (uint64_t)(16 * m), id2h, 1u);
                }
              }
              tc_commit2_leader(&g2done[r]);  // frees S buffer g for GEMM1(g + NS)
            }
            if (lu) tc_commit2(&o_full[obu]);
          }
          __syncwarp();
          if (lane == 0) trace_ev<DBG>(p, gt, 1);
          q += last ? 1u : 0u;
          s2 = (s2 + 1u == (uint32_t)NS) ? 0u : s2 + 1u;
          dv += vstep;
          if (dv == vend) dv = dV0;
          if (++r == (uint32_t)NR) {
            r = 0;
            rph ^= 1u;
          }
          ++gt;
          cur.next(p, items);
        }
      } else if (SYM) {
        // ---------------- transposed-product issuer (symmetric kernel)
        // D_T[j, :] += P(t)^T [V_I0 | V_I1]: A = P^T from each CTA's shared
        // memory (MN-major: the K-major bytes of P read transposed), B split
        // along N so each CTA supplies its own V block; CTA c's lanes keep
        // columns [c WP, (c + 1) WP) -- its rows' contribution to out_J.
        const uint32_t idT = idesc_f16(2 * WP) | (1u << 15);
        const uint64_t dP0 = sdesc(smem_u32(sP), 2048u, 128u);
        const uint64_t dVh = sdesc(smem_u32(sVI), 128u, (uint32_t)(BN * 16));
        const uint64_t dVl = dVh + (p.v2_bytes >> 4);
        TileIter cur;
        cur.start(p, items);
        uint32_t r = 0, rph = 0, gt = 0, nitem = 0, dtq = 0;
        while (cur.valid) {
          if (cur.first_in_item()) {
            mbar_wait(vi_full, nitem & 1u);
            ++nitem;
          }
          mbar_wait(&rdy[r], rph);  // P(g) stored in both CTAs' shared memory
          if (lane == 0) trace_ev<DBG>(p, gt, 12);
          const bool tp = cur.transposed();
          if (tp) mbar_wait(&dt_empty[dtq & 1u], ((dtq >> 1) & 1u) ^ 1u);
          // With two S buffers, T(g) enters the tensor pipe after GEMM1(g + 2):
          // the GEMM2 -> GEMM1 -> epilogue chain must not queue behind the
          // transposed product (three buffers leave enough slack without it)
          // (not with the row tile in TMEM: GEMM1 of an item's first tile
          // waits for the drain warps' A load, which comes after they drained
          // this tile's D_T -- holding T(g) for it would close a cycle)
          if (!ATM && (NS == 2) != ((p.sym_dbg & 64) != 0))
            while (*g1_cnt < gt + (uint32_t)NS + 1u) {
            }
          tc_fence_after();
          if (lane == 0) trace_ev<DBG>(p, gt, 13);
          const uint32_t tpu = __shfl_sync(0xffffffffu, tp ? 1u : 0u, 0);
          const uint32_t dtb = __shfl_sync(0xffffffffu, dtq & 1u, 0);
          const uint32_t liu = __shfl_sync(0xffffffffu, cur.last_in_item() ? 1u : 0u, 0);
          if (elect_one()) {
            if (tpu && !(DBG && (p.sym_dbg & 4))) {
              const uint64_t pa = dP0 + (uint64_t)pbuf(gt) * (PB >> 4);
              if (PF8) {
                // P_hi^T Vhi + P_hi^T Vlo (f16), then P_lo8^T Vhi8 (E4M3, K = 32, A MN-major,
                // core matrix 8 K-rows x 16 MN-bytes) with B = this CTA's own Vhi8 block
                const uint32_t dt = tDT(dtb);
                const uint64_t p8 = sdesc(smem_u32(sP) + pbuf(gt) * PB + PH2, 1024u, 128u);
                const uint64_t b8 = sdesc(smem_u32(sVI) + 2u * p.v2_bytes, 128u, 1024u);
                constexpr uint32_t idT8 = idesc1_f8(2 * WP, true) + ((uint32_t)((256 - 128) >> 4) << 24);
#pragma unroll 1
                for (int m = 0; m < BN / 16; ++m) {
                  const uint64_t ah = pa + (uint64_t)m * (4096 >> 4);
                  mma_ss(dt, ah, dVh + (uint64_t)(16 * m), idT, m > 0 ? 1u : 0u);
                  mma_ss(dt, ah, dVl + (uint64_t)(16 * m), idT, 1u);
                }
#pragma unroll
                for (int q2 = 0; q2 < BN / 32; ++q2)
                  mma_f8_ss(dt, p8 + (uint64_t)q2 * (4096 >> 4), b8 + (uint64_t)(16 * q2), idT8, 1u);
              } else {
#pragma unroll 1
                for (int m = 0; m < BN / 16; ++m) {
                  const uint64_t ah = pa + (uint64_t)m * (4096 >> 4), al = ah + ((PBUF / 2) >> 4);
                  const uint64_t bh = dVh + (uint64_t)(16 * m), bl = dVl + (uint64_t)(16 * m);
                  const uint32_t dt = tDT(dtb);
                  mma_ss(dt, ah, bh, idT, m > 0 ? 1u : 0u);
                  mma_ss(dt, ah, bl, idT, 1u);
                  mma_ss(dt, al, bh, idT, 1u);
                }
              }
            }
            if (tpu) tc_commit2(&dt_full[dtb]);
            tc_commit2(&pt_free[ptb(gt)]);
            if (liu) tc_commit2(vi_empty);
          }
          __syncwarp();
          if (lane == 0) trace_ev<DBG>(p, gt, 14);
          dtq += tp ? 1u : 0u;
          ++gt;
          if (++r == (uint32_t)NR) {
            r = 0;
            rph ^= 1u;
          }
          cur.next(p, items);
        }
      }
    }
  }
  } else if (warp < 4 + EPI_WARPS) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 96;");
    // ================= epilogue: two groups of 8 warps =================
    // group e transforms tiles g = e (mod 2); within a group, the warp with
    // TMEM lane quarter wq and column half hc does chunks 2hc, 2hc + 1.
    const int e = (warp - 4) / 8;            // 0 or 1
    const int hc = ((warp - 4) % 8) / 4;     // column half
    const int wq = warp & 3;                 // TMEM lane quarter
    const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
    const uint32_t col0 = (uint32_t)(hc * (BN / 2));
    TileIter ti;
    ti.start(p, items);
    Ring er;  // s_full ring (NR)
    er.init(NR);
    uint32_t bb = 0;  // S buffer of the current tile (g mod NS)
    const float L = p.L;
    uint32_t gt = 0;
    const bool tr = (wq == 0 && hc == 0 && lane == 0);
    while (ti.valid) {
      if ((int)(gt & 1u) == e) {
        const int b = (int)bb;
        if (tr) trace_ev<DBG>(p, gt, 3 + 2 * e);
        // symmetric kernel: P buffer e is free once GEMM2(gt - 2) and T(gt - 2)
        // completed.  Waited on every tile (both commit pt_free for every
        // tile), just before the first shared-memory store, so the first
        // chunk's TMEM load and transform overlap them.
        bool pt_wait = SYM && gt >= (uint32_t)p.npb;
        mbar_wait(&s_full[er.idx], er.phase);
        tc_fence_after();
        if (tr) trace_ev<DBG>(p, gt, 4 + 2 * e);
        if (!(DBG && (p.debug_mode == 1 || p.debug_mode == 5))) {
          const uint32_t base = tS(b) + lane_off + col0;
          uint32_t ra[32], hi[16], lo[16];
          if constexpr (SYM) {
            // P goes to shared memory only (row i = TMEM lane, 8 consecutive j
            // per 16 B): the K-major A of GEMM2 and the MN-major A of T.  S(g)
            // is released to GEMM1(g + NS) as soon as it is loaded.
            const int i = 32 * wq + lane;
            const uint32_t rowb0 = smem_u32(sP) + pbuf(gt) * PB + (uint32_t)(i >> 3) * 2048u +
                                   (uint32_t)(i & 7) * 16u + (col0 >> 3) * 128u;
            // PF8: P_lo8 at + PH2, row i, 16 consecutive j per 16 B (as K1-sym2)
            const uint32_t row8b = smem_u32(sP) + pbuf(gt) * PB + PH2 + (uint32_t)(i >> 3) * 1024u +
                                   (uint32_t)(i & 7) * 16u + (col0 >> 4) * 128u;
            uint32_t l8[8];
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) {
              tmem_ld32(base + 32 * c, ra);
              tmem_wait_ld(ra);
              if (!NCGP_PAIR_PT && c == BN / 64 - 1) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(leader_addr(&s_free[er.idx]));
              }
              if (PF8)
                transform_chunk2<FAM>(ra, L, hi, l8);
              else
                transform_chunk<FAM>(ra, L, hi, lo);
              if (NCGP_PAIR_PT) {  // P over S(g) for GEMM2's TS MMAs
                if (FAM == NCGP_RBF) {
                  tmem_st_hilo(base + 32 * c, hi, lo);
                } else {
                  tmem_st16(base + 32 * c, hi);
                  tmem_st16(base + 32 * c + 16, lo);
                }
              }
              if (pt_wait) {
                const uint32_t t = gt - (uint32_t)p.npb;
                mbar_wait(&pt_free[ptb(t)], ptph(t));
                pt_wait = false;
                if (tr) trace_ev<DBG>(p, gt, 8);
              }
              if (!(DBG && (p.sym_dbg & 16))) {
                const uint32_t rowb = rowb0 + 512u * c;
#pragma unroll
                for (int g = 0; g < 4; ++g)
                  st_shared_v4(rowb + 128u * g, hi[4 * g], hi[4 * g + 1], hi[4 * g + 2], hi[4 * g + 3]);
                if (PF8) {
                  st_shared_v4(row8b + 256u * c, l8[0], l8[1], l8[2], l8[3]);
                  st_shared_v4(row8b + 256u * c + 128u, l8[4], l8[5], l8[6], l8[7]);
                } else {
#pragma unroll
                  for (int g = 0; g < 4; ++g)
                    st_shared_v4(rowb + PBUF / 2 + 128u * g, lo[4 * g], lo[4 * g + 1], lo[4 * g + 2],
                                 lo[4 * g + 3]);
                }
              }
            }
            if (NCGP_PAIR_PT) tmem_wait_st();
            fence_proxy_async_smem();
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) {
              tmem_ld32(base + 32 * c, ra);
              tmem_wait_ld(ra);
              transform_chunk<FAM>(ra, L, hi, lo);
              if (FAM == NCGP_RBF) {
                tmem_st_hilo(base + 32 * c, hi, lo);
              } else {
                tmem_st16(base + 32 * c, hi);
                tmem_st16(base + 32 * c + 16, lo);
              }
            }
            tmem_wait_st();
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_addr(&rdy[er.idx]));
        if (tr) trace_ev<DBG>(p, gt, e == 0 ? 7 : 10);
      }
      ++gt;
      er.adv();
      bb = (bb + 1u == (uint32_t)NS) ? 0u : bb + 1u;
      ti.next(p, items);
    }
  } else {
    // (symmetric kernel: 56 -- 4 x 32 x 40 + 16 x 32 x 96 + 4 x 32 x 56 = the 61,440 pool)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(SYM ? 56 : 40));
    // ================= correction warpgroup =================
    const int wq = warp & 3;
    const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
    const int row = 32 * wq + lane;
    if (SYM) {
      // O chunks and each transposed tile's D_T go into the int64 fixed-point
      // accumulator (fx_flush8: one 2 KB bulk reduction per 8 columns of the
      // warp's 32 rows); rows past n are padding
      TileIter ti;
      ti.start(p, items);
      uint32_t q = 0, dtq = 0, nst = 0;
      constexpr uint32_t NBLK = WP == 32 ? 2u : 1u;  // staging blocks per warp (BM x WP x 4 bytes)
      const uint32_t stg_warp = smem_u32(sStage) + (uint32_t)wq * NBLK * 2048u;
      uint32_t aitem = 0;
      while (ti.valid) {
        if (ATM && ti.first_in_item()) {
          // this CTA's row tile into TMEM: row = lane, 16-byte K chunk q of the
          // canonical K-major pack -> columns 4q .. 4q + 3; once GEMM1 of the
          // previous item is done with it (a_empty), then a_full on the leader
          mbar_wait(&a_empty[0], (aitem & 1u) ^ 1u);
          tc_fence_after();
          const int64_t rt = p.rt0 + 2 * (int64_t)ti.cur.pp + rank;
          const int r = 32 * wq + lane;
          const uint8_t* src = p.xa_pack + rt * (int64_t)p.a_bytes + (size_t)(r >> 3) * (p.ka / 8) * 128 +
                               (size_t)(r & 7) * 16;
          for (int q = 0; q < p.ka / 8; ++q) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + (size_t)q * 128));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                             tA + lane_off + 4u * q),
                         "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
          }
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(leader_addr(&a_full[0]));
          ++aitem;
        }
        if (ti.transposed()) {
          mbar_wait(&dt_full[dtq & 1u], (dtq >> 1) & 1u);
          tc_fence_after();
          const int64_t j0 = (int64_t)ti.ct * BM + 32 * wq;  // output rows of the transposed product
          const bool ld = !(DBG && (p.sym_dbg & 8));
#pragma unroll
          for (int h = 0; h < WP / 8; ++h) {
            uint32_t x[8];
            if (ld) {
              tmem_ld8(tDT(dtq & 1u) + lane_off + (uint32_t)(rank * WP + 8 * h), x);
              tmem_wait_ld();
            } else {
#pragma unroll
              for (int c = 0; c < 8; ++c) x[c] = 0u;
            }
            float v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = __uint_as_float(x[c]);
            if (DBG && p.sym_dump != nullptr) {
              float* dd = p.sym_dump + ((((int64_t)ti.cur.pp * p.col_tiles + ti.ct) * 2 + rank) * BM + row) * WP + 8 * h;
#pragma unroll
              for (int c = 0; c < 8; ++c) dd[c] = v[c];
            }
            if (NCGP_PAIR_RED)
              fx_red8(p, lane, h, v, j0, DBG && (p.sym_dbg & 1));
            else
              fx_flush8<NBLK>(p, stg_warp, nst, lane, h, v, j0, DBG && (p.sym_dbg & 1));
          }
          tc_fence_before();
          if (lane == 0) mbar_arrive_cluster(leader_addr(&dt_empty[dtq & 1u]));
          if (lane == 0 && wq == 0 && ti.it == (int)(blockIdx.x >> 1)) trace_ev<DBG>(p, ti.ct - ti.cur.c0, 15);
          ++dtq;
        }
        if (ti.last_in_chunk()) {
          mbar_wait(&o_full[q & 1u], (q >> 1) & 1u);
          tc_fence_after();
          const int64_t i0 = (2 * (int64_t)ti.cur.pp + rank) * BM + 32 * wq;
#pragma unroll
          for (int h = 0; h < WP / 8; ++h) {
            uint32_t x[8], y[8];
            tmem_ld8(tO(q & 1u) + lane_off + 8 * h, x);       // P_hi Vhi + P_lo Vhi
            tmem_ld8(tO(q & 1u) + lane_off + WP + 8 * h, y);  // P_hi Vlo
            tmem_wait_ld();
            float v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = __uint_as_float(x[c]) + __uint_as_float(y[c]);
            if (NCGP_PAIR_RED)
              fx_red8(p, lane, h, v, i0, DBG && (p.sym_dbg & 2));
            else
              fx_flush8<NBLK>(p, stg_warp, nst, lane, h, v, i0, DBG && (p.sym_dbg & 2));
          }
          tc_fence_before();
          if (lane == 0) mbar_arrive_cluster(leader_addr(&o_empty[q & 1u]));
          ++q;
        }
        ti.next(p, items);
      }
      if (lane == 0 && !NCGP_PAIR_RED) bulk_wait_all();
    } else if constexpr (WIDE) {
      // wide kernel: each item's O (fp32, accumulated in TMEM over <= 64
      // column tiles) -> the fp32 partial [split][local row][WP] in HBM
      TileIter ti;
      ti.start(p, items);
      uint32_t q = 0;
      float* const part = reinterpret_cast<float*>(p.partial);
      while (ti.valid) {
        if (ti.last_in_item()) {
          const uint32_t ob = q & 1u;
          mbar_wait(&o_full[ob], (q >> 1) & 1u);
          tc_fence_after();
          const int64_t i = (2 * (int64_t)ti.cur.pp + rank) * BM + row;  // local row
          const int64_t sp = ti.it % p.splits;
          float4* dst = reinterpret_cast<float4*>(part + (sp * p.nloc + i) * WP);
#pragma unroll 1
          for (int h = 0; h < WP / 8; ++h) {
            uint32_t x[8];
            tmem_ld8(tO((int)ob) + lane_off + 8 * h, x);  // all three split terms
            tmem_wait_ld();
            if (i < p.nloc) {
              dst[2 * h] = make_float4(__uint_as_float(x[0]), __uint_as_float(x[1]),
                                       __uint_as_float(x[2]), __uint_as_float(x[3]));
              dst[2 * h + 1] = make_float4(__uint_as_float(x[4]), __uint_as_float(x[5]),
                                           __uint_as_float(x[6]), __uint_as_float(x[7]));
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(leader_addr(&o_empty[ob]));
          ++q;
        }
        ti.next(p, items);
      }
    } else {
    double* acc = sAcc + row;  // acc[c * BM], conflict-free across the warp
#pragma unroll
    for (int c = 0; c < WP; ++c) acc[c * BM] = 0.0;
    TileIter ti;
    ti.start(p, items);
    uint32_t q = 0;
    while (ti.valid) {
      if (ti.last_in_chunk()) {
        const int ob = (int)(q & 1u);
        mbar_wait(&o_full[ob], (q >> 1) & 1u);
        tc_fence_after();
#pragma unroll 1
        for (int h = 0; h < WP / 8; ++h) {  // 8 columns at a time (40-register budget)
          uint32_t r[8], t[8];
          tmem_ld8(tO(ob) + lane_off + 8 * h, r);       // P_hi Vhi + P_lo Vhi
          tmem_ld8(tO(ob) + lane_off + WP + 8 * h, t);  // P_hi Vlo
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 8; ++c)
            acc[(8 * h + c) * BM] += (double)__uint_as_float(r[c]) + (double)__uint_as_float(t[c]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_addr(&o_empty[ob]));
        ++q;
        if (ti.last_in_item()) {
          const int64_t i = (2 * (int64_t)ti.cur.pp + rank) * BM + row;  // local row
          if (i < p.nloc) {
            const int64_t sp = ti.it % p.splits;  // once per item
            auto kv = [&](int c) -> double {
              return ldexp(acc[c * BM], -(p.s_exp + __ldg(&p.col_exp[c])));
            };
            if (p.splits > 1) {
              for (int c = 0; c < p.w; ++c) p.partial[(sp * p.nloc + i) * p.w + c] = kv(c);
            } else if (p.out_f64) {  // own output, then the peers', through the epilogue
              ncgp::epi_row<double, NCGP_MAX_OUTS>(p.epi, i, p.w, kv,
                                                   reinterpret_cast<double* const*>(p.outs), p.n_out, p.ldo);
            } else {
              ncgp::epi_row<float, NCGP_MAX_OUTS>(p.epi, i, p.w, kv,
                                                  reinterpret_cast<float* const*>(p.outs), p.n_out, p.ldo);
            }
          }
#pragma unroll
          for (int c = 0; c < WP; ++c) acc[c * BM] = 0.0;
        }
      }
      ti.next(p, items);
    }
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (DBG && p.trace != nullptr && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[TRACE_TILES * TRACE_EV + 4 * blockIdx.x + 1] = (long long)t;
  }
  cluster_sync();  // both CTAs done with TMEM / remote barriers
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ single-CTA symmetric kernel
// K1-sym1: the symmetric K(X, X) kernel with cta_group::1 MMAs.  One CTA per
// SM owns a 128-row tile I and sweeps column tiles J >= I; each P(I, J) tile
// serves O_I += P V_J (GEMM2, A = P K-major) and D_T = P^T V_I (T, A = P
// MN-major), both read from the same shared-memory copy of P.  Against the
// pair kernel: the transposed product has no wasted half (B = [Vhi_I | Vlo_I]
// is this CTA's own block), at the price of one MMA issue per SM instead of
// per pair and full (not half) column records per CTA.
// Roles (24 warps): warp 0 lane 0 producer (row tile per item, XB and V per
// column tile); warp 1 GEMM2; warp 2 TMEM allocation + GEMM1; warp 3 the
// transposed product (and this row tile's V block per item); warps 4-19 the
// epilogue (as in the pair kernel's symmetric mode); warps 20-23 the O / D_T
// drains into the fp32 accumulator.
__device__ __forceinline__ void mma1_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma1_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit1(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// kind::f16, A/B F16, D F32, M = 128; bit 15: A MN-major (transposed)
__host__ __device__ constexpr uint32_t idesc1_f16(int n, bool a_mn = false) {
  return (1u << 4) | (a_mn ? (1u << 15) : 0u) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}

struct Tile1 {  // the CTA's global column-tile sequence across its items
  int it, ct, r, c0, c1;
  bool valid;
  __device__ __forceinline__ void load(const TcParams& p) {
    const int4 t = p.item_tab[it];
    r = t.x;
    c0 = t.y;
    c1 = t.z;
    ct = c0;
  }
  __device__ __forceinline__ void start(const TcParams& p) {
    it = (int)blockIdx.x;
    valid = it < p.n_items;
    if (valid) load(p);
  }
  __device__ __forceinline__ void next(const TcParams& p) {
    if (++ct >= c1) {
      it += (int)gridDim.x;
      valid = it < p.n_items;
      if (valid) load(p);
    }
  }
  __device__ __forceinline__ bool first_in_item() const { return ct == c0; }
  __device__ __forceinline__ bool last_in_item() const { return ct == c1 - 1; }
  __device__ __forceinline__ bool transposed() const { return ct > r; }
  __device__ __forceinline__ bool first_in_chunk() const { return ct == c0 || (ct & (CH - 1)) == 0; }
  __device__ __forceinline__ bool last_in_chunk() const {
    return ct == c1 - 1 || (ct & (CH - 1)) == CH - 1;
  }
};

template <int FAM, int WP, bool DBG>
__global__ void __launch_bounds__(NTHREADS, 1) kop_sym1_kernel(const TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // S buffers next to double-buffered O and D_T (2 x 2 WP columns each):
  // two at WP = 32, three at WP = 16
  // P-in-TMEM mode: 1 (merged D_T) at WP = 32, 2 (two-instruction T into a
  // 2 WP-column D_T, double-buffered) at WP = 16, where TMEM has the room
  // (RBF w = 10, n = 2e5: 8.8 -> 8.0 ms; cfg4 shape 3.41 -> 3.36 ms)
  constexpr int PTM = WP == 16 ? NCGP_SYM1_PT16 : NCGP_SYM1_PT;
  constexpr bool PT = PTM != 0;
  constexpr bool TM = PTM == 1;     // D_T merged into WP columns (double-buffered)
  constexpr int NS1 = (PTM == 2 && WP == 32 && NCGP_SYM1_PT2NS) ? 2 : (PT ? 3 : (WP == 16 ? NCGP_SYM1_NS16 : 2));
  constexpr uint32_t AW = PT ? WP : 2 * WP;  // TMEM columns of one O accumulator
  constexpr uint32_t DW = TM ? WP : 2 * WP;  // TMEM columns of one D_T accumulator
  constexpr uint32_t NDT = (PT && !TM && WP == 32 && !NCGP_SYM1_PT2NS) ? 1u : 2u;  // D_T buffers (PT = 2: two fit at WP = 16)
  const uint32_t xb_bytes = 2u * p.xbh_bytes;  // 128 XB rows
  const uint32_t vb_bytes = 2u * p.v2_bytes;   // [Vhi | Vlo]: 2 WP rows
  uint8_t* sA = smem;
  uint8_t* sXB = sA + p.a_bytes;
  uint8_t* sV = sXB + (size_t)p.sx * xb_bytes;
  uint8_t* sVI = sV + (size_t)p.sv * vb_bytes;
  uint8_t* sP = sVI + vb_bytes;
  float* sStage = reinterpret_cast<float*>(sP + (size_t)p.npb * PBUF);
  // P buffer of tile g: two alternating, or one when shared memory is short
  auto pbuf = [&](uint32_t g) -> uint32_t { return p.npb == 2 ? (g & 1u) : 0u; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + BM * WP);
  uint64_t* xb_full = bars;            // [6]
  uint64_t* v_full = xb_full + 6;      // [9]
  uint64_t* a_full = v_full + 9;       // [1]
  uint64_t* a_empty = a_full + 1;      // [1]
  uint64_t* vi_full = a_empty + 1;     // [1]
  uint64_t* vi_empty = vi_full + 1;    // [1]
  uint64_t* s_full = vi_empty + 1;     // [NR] GEMM1(g) done
  uint64_t* s_free = s_full + NR;      // [NR] S(g) loaded by the epilogue group (8 warps)
  uint64_t* rdy = s_free + NR;         // [NR] P(g) stored (8 warps)
  uint64_t* g2done = rdy + NR;         // [NR] GEMM2(g) done
  uint64_t* pt_free = g2done + NR;     // [2]  GEMM2(g) and T(g) done with P buffer g & 1
  uint64_t* o_full = pt_free + 2;      // [2]
  uint64_t* o_empty = o_full + 2;      // [2]  4 drain warps
  uint64_t* dt_full = o_empty + 2;     // [2]
  uint64_t* dt_empty = dt_full + 2;    // [2]  4 drain warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dt_empty + 2);
  volatile uint32_t* g1_cnt = tmem_slot + 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 6; ++s) mbar_init(&xb_full[s], 1);
    for (int s = 0; s < 9; ++s) mbar_init(&v_full[s], 1);
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    mbar_init(vi_full, 1);
    mbar_init(vi_empty, 1);
    for (int s = 0; s < NR; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], 8);
      mbar_init(&rdy[s], 8);
      mbar_init(&g2done[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&pt_free[b], 2);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 4);
      mbar_init(&dt_full[b], 1);
      mbar_init(&dt_empty[b], 4);
    }
    *g1_cnt = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (DBG && p.trace != nullptr && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[TRACE_TILES * TRACE_EV + 4 * blockIdx.x] = (long long)t;
  }
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform MMA operands
  auto tS = [&](uint32_t b) -> uint32_t { return tmem + b * (uint32_t)BN; };
  auto tO = [&](uint32_t b) -> uint32_t { return tmem + (uint32_t)(NS1 * BN) + b * AW; };
  auto tDT = [&](uint32_t b) -> uint32_t { return tmem + (uint32_t)(NS1 * BN) + 2u * AW + b * DW; };
  const bool p_tmem = PT || (p.sym_dbg & 128) != 0;  // P also in TMEM (over S) for GEMM2

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == 0) {
      // ================= producer (lane 0) =================
      if (lane == 0) {
        Tile1 ti;
        ti.start(p);
        Ring xr, vr, xs, vs;  // slot rings; release rings (s_full for XB, g2done for V)
        xr.init((uint32_t)p.sx);
        vr.init((uint32_t)p.sv);
        xs.init(NR);
        vs.init(NR);
        uint32_t g = 0, nitem = 0;
        while (ti.valid) {
          if (ti.first_in_item()) {
            mbar_wait(a_empty, (nitem & 1u) ^ 1u);
            mbar_expect_tx(a_full, p.a_bytes);
            bulk_g2s(sA, p.xa_pack + (int64_t)ti.r * p.a_bytes, p.a_bytes, a_full);
            ++nitem;
          }
          const uint8_t* rec = p.col_pack + (int64_t)ti.ct * p.tile_stride;
          if (g >= (uint32_t)p.sx) {
            mbar_wait(&s_full[xs.idx], xs.phase);
            xs.adv();
          }
          mbar_expect_tx(&xb_full[xr.idx], xb_bytes);
          uint8_t* dx = sXB + (size_t)xr.idx * xb_bytes;
          bulk_g2s(dx, rec, p.xbh_bytes, &xb_full[xr.idx]);
          bulk_g2s(dx + p.xbh_bytes, rec + p.rec_bytes, p.xbh_bytes, &xb_full[xr.idx]);
          xr.adv();
          if (g >= (uint32_t)p.sv) {
            mbar_wait(&g2done[vs.idx], vs.phase);
            vs.adv();
          }
          mbar_expect_tx(&v_full[vr.idx], vb_bytes);
          uint8_t* dv = sV + (size_t)vr.idx * vb_bytes;
          bulk_g2s(dv, rec + p.xbh_bytes, p.v2_bytes, &v_full[vr.idx]);                    // Vhi
          bulk_g2s(dv + p.v2_bytes, rec + p.rec_bytes + p.xbh_bytes, p.v2_bytes, &v_full[vr.idx]);  // Vlo
          vr.adv();
          ++g;
          ti.next(p);
        }
      }
    } else if (warp == 2) {
      // ================= GEMM1: S(g) = XA . XB(g)^T =================
      const uint32_t sbo_x = (uint32_t)(p.ka / 8) * 128u;
      const int ksteps1 = p.ka / 16;
      const uint64_t dA = sdesc(smem_u32(sA), 128u, sbo_x);
      const uint64_t dX0 = sdesc(smem_u32(sXB), 128u, sbo_x);
      const uint32_t id1 = idesc1_f16(BN);
      Tile1 ti;
      ti.start(p);
      Ring xr, sf;
      xr.init((uint32_t)p.sx);
      sf.init(NR);
      uint32_t g = 0, c1 = 0, nitem = 0, sb = 0;
      while (ti.valid) {
        const bool li = ti.last_in_item();
        if (ti.first_in_item()) {
          mbar_wait(a_full, nitem & 1u);
          ++nitem;
        }
        mbar_wait(&xb_full[xr.idx], xr.phase);
        if (g >= (uint32_t)NS1) {  // S buffer free once the epilogue loaded S(g - NS1)
          // (P in TMEM, sym_dbg 128: once GEMM2(g - NS1) has read it)
          mbar_wait(p_tmem ? &g2done[sf.idx] : &s_free[sf.idx], sf.phase);
          sf.adv();
        }
        tc_fence_after();
        if (lane == 0) trace_ev<DBG>(p, g, 9);
        const uint64_t dx = dX0 + (uint64_t)xr.idx * (xb_bytes >> 4);
        const uint32_t d = tS(sb);
        const uint32_t liu = __shfl_sync(0xffffffffu, li ? 1u : 0u, 0);
        if (elect_one()) {
          for (int k = 0; k < ksteps1; ++k)
            mma1_ss(d, dA + (uint64_t)(16 * k), dx + (uint64_t)(16 * k), id1, k > 0);
          tc_commit1(&s_full[c1]);  // also frees XB slot g (producer)
          if (liu) tc_commit1(a_empty);
        }
        __syncwarp();
        if (lane == 0) trace_ev<DBG>(p, g, 2);
        if (lane == 0) *g1_cnt = g + 1u;
        sb = sb + 1u == (uint32_t)NS1 ? 0u : sb + 1u;
        xr.adv();
        c1 = (c1 + 1u == (uint32_t)NR) ? 0u : c1 + 1u;
        ++g;
        ti.next(p);
      }
      if (lane == 0) *g1_cnt = 0xFFFFFFFFu;
    } else if (warp == 1) {
      // ================= GEMM2: O_I += P(g) [Vhi | Vlo] + P_lo Vhi =================
      const uint32_t id2 = idesc1_f16(2 * WP), id2h = idesc1_f16(WP);
      const uint64_t dV0 = sdesc(smem_u32(sV), 128u, (uint32_t)(BN * 16));
      Tile1 ti;
      ti.start(p);
      Ring vr, rr;
      vr.init((uint32_t)p.sv);
      rr.init(NR);
      uint32_t g = 0, q = 0, sb = 0;
      while (ti.valid) {
        const bool fresh = ti.first_in_chunk(), last = ti.last_in_chunk();
        if (lane == 0) trace_ev<DBG>(p, g, 11);
        mbar_wait(&rdy[rr.idx], rr.phase);
        mbar_wait(&v_full[vr.idx], vr.phase);
        const uint32_t ob = q & 1u;
        if (fresh) mbar_wait(&o_empty[ob], ((q >> 1) & 1u) ^ 1u);
        tc_fence_after();
        if (lane == 0) trace_ev<DBG>(p, g, 0);
        const uint64_t dv = dV0 + (uint64_t)vr.idx * (vb_bytes >> 4);
        const uint64_t ph = sdesc(smem_u32(sP) + pbuf(g) * PBUF, 128u, 2048u);
        const uint64_t pl = ph + ((PBUF / 2) >> 4);
        const uint32_t obu = __shfl_sync(0xffffffffu, ob, 0);
        const bool fu = __shfl_sync(0xffffffffu, fresh ? 1u : 0u, 0) != 0u;
        const bool lu = __shfl_sync(0xffffffffu, last ? 1u : 0u, 0) != 0u;
        const uint32_t dO = tO(obu);
        if (elect_one()) {
          if (PT) {  // A = P from TMEM; P_hi Vhi, P_hi Vlo, P_lo Vhi into the same WP columns
            const uint32_t a0 = tS(sb);
            const uint64_t vlo = (uint64_t)(p.v2_bytes >> 4);
#pragma unroll
            for (int m = 0; m < BN / 16; ++m) {
              const uint32_t ahi = a0 + 32u * (m >> 1) + 8u * (m & 1);
              const uint64_t b = dv + (uint64_t)(16 * m);
              mma1_ts(dO, ahi, b, id2h, (fu && m == 0) ? 0u : 1u);
              mma1_ts(dO, ahi, b + vlo, id2h, 1u);
              mma1_ts(dO, ahi + 16u, b, id2h, 1u);
            }
          } else if (p.sym_dbg & 128) {  // A = P from TMEM (the epilogue's copy over S(g))
            const uint32_t a0 = tS(sb);
#pragma unroll
            for (int m = 0; m < BN / 16; ++m) {
              const uint32_t ahi = a0 + 32u * (m >> 1) + 8u * (m & 1);
              mma1_ts(dO, ahi, dv + (uint64_t)(16 * m), id2, (fu && m == 0) ? 0u : 1u);
              mma1_ts(dO, ahi + 16u, dv + (uint64_t)(16 * m), id2h, 1u);
            }
          } else {
#pragma unroll
            for (int m = 0; m < BN / 16; ++m) {
              mma1_ss(dO, ph + (uint64_t)(16 * m), dv + (uint64_t)(16 * m), id2, (fu && m == 0) ? 0u : 1u);
              mma1_ss(dO, pl + (uint64_t)(16 * m), dv + (uint64_t)(16 * m), id2h, 1u);
            }
          }
          tc_commit1(&g2done[rr.idx]);  // V slot g free
          tc_commit1(&pt_free[g & 1u]);
          if (lu) tc_commit1(&o_full[obu]);
        }
        __syncwarp();
        if (lane == 0) trace_ev<DBG>(p, g, 1);
        q += last ? 1u : 0u;
        sb = sb + 1u == (uint32_t)NS1 ? 0u : sb + 1u;
        vr.adv();
        rr.adv();
        ++g;
        ti.next(p);
      }
    } else {
      // ================= T: D_T(J) = P(g)^T [Vhi_I | Vlo_I] + P_lo^T Vhi_I =================
      const uint32_t idT = idesc1_f16(2 * WP, true), idTh = idesc1_f16(WP, true);
      const uint64_t dP0 = sdesc(smem_u32(sP), 2048u, 128u);
      const uint64_t dVI = sdesc(smem_u32(sVI), 128u, (uint32_t)(BN * 16));
      Tile1 ti;
      ti.start(p);
      Ring rr;
      rr.init(NR);
      uint32_t g = 0, nitem = 0, dtq = 0;
      // Holding T(g) behind GEMM1(g + 2) (as the pair kernel does at WP = 32)
      // costs 5 % at cfg3 here (one box, interleaved: 316 vs 300 ms) and is
      // neutral for Matern and at WP = 16: off unless sym_dbg bit 64.
      const bool hold = (p.sym_dbg & 64) != 0;
      while (ti.valid) {
        if (ti.first_in_item()) {  // this row tile's V block (the transposed product's B)
          mbar_wait(vi_empty, (nitem & 1u) ^ 1u);
          if (elect_one()) {
            mbar_expect_tx(vi_full, vb_bytes);
            const uint8_t* rec = p.col_pack + (int64_t)ti.r * p.tile_stride;
            bulk_g2s(sVI, rec + p.xbh_bytes, p.v2_bytes, vi_full);
            bulk_g2s(sVI + p.v2_bytes, rec + p.rec_bytes + p.xbh_bytes, p.v2_bytes, vi_full);
          }
          __syncwarp();
          mbar_wait(vi_full, nitem & 1u);
          ++nitem;
        }
        mbar_wait(&rdy[rr.idx], rr.phase);
        if (lane == 0) trace_ev<DBG>(p, g, 12);
        const bool tp = ti.transposed();
        if (tp) mbar_wait(&dt_empty[dtq % NDT], ((dtq / NDT) & 1u) ^ 1u);
        if (hold)  // T(g) behind GEMM1(g + NS1) in the in-order tensor pipe
          while (*g1_cnt < g + (uint32_t)NS1 + 1u) {
          }
        tc_fence_after();
        if (lane == 0) trace_ev<DBG>(p, g, 13);
        const bool tpu = __shfl_sync(0xffffffffu, tp ? 1u : 0u, 0) != 0u;
        const uint32_t dtb = __shfl_sync(0xffffffffu, dtq % NDT, 0);
        const bool liu = __shfl_sync(0xffffffffu, ti.last_in_item() ? 1u : 0u, 0) != 0u;
        if (elect_one()) {
          if (tpu && !(DBG && (p.sym_dbg & 4))) {
            const uint64_t pa = dP0 + (uint64_t)pbuf(g) * (PBUF >> 4);
            const uint32_t dt = tDT(dtb);
            const uint64_t vlo = (uint64_t)(p.v2_bytes >> 4);
#pragma unroll 1
            for (int m = 0; m < BN / 16; ++m) {
              const uint64_t ah = pa + (uint64_t)m * (4096 >> 4), al = ah + ((PBUF / 2) >> 4);
              const uint64_t b = dVI + (uint64_t)(16 * m);
              if (TM) {  // P_hi^T Vhi, P_hi^T Vlo, P_lo^T Vhi into the same WP columns
                mma1_ss(dt, ah, b, idTh, m > 0 ? 1u : 0u);
                mma1_ss(dt, ah, b + vlo, idTh, 1u);
                mma1_ss(dt, al, b, idTh, 1u);
              } else {
                mma1_ss(dt, ah, b, idT, m > 0 ? 1u : 0u);
                mma1_ss(dt, al, b, idTh, 1u);
              }
            }
          }
          if (tpu) tc_commit1(&dt_full[dtb]);
          tc_commit1(&pt_free[g & 1u]);
          if (liu) tc_commit1(vi_empty);
        }
        __syncwarp();
        if (lane == 0) trace_ev<DBG>(p, g, 14);
        dtq += tp ? 1u : 0u;
        rr.adv();
        ++g;
        ti.next(p);
      }
    }
  } else if (warp < 4 + EPI_WARPS) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 96;");
    // ================= epilogue: two groups of 8 warps alternate tiles =================
    const int e = (warp - 4) / 8;
    const int hc = ((warp - 4) % 8) / 4;
    const int wq = warp & 3;
    const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
    const uint32_t col0 = (uint32_t)(hc * (BN / 2));
    const int i = 32 * wq + lane;
    const uint32_t rowb_base = (uint32_t)(i >> 3) * 2048u + (uint32_t)(i & 7) * 16u + (col0 >> 3) * 128u;
    Tile1 ti;
    ti.start(p);
    Ring er;
    er.init(NR);
    const float L = p.L;
    uint32_t g = 0, sb = 0;
    const bool tr = (wq == 0 && hc == 0 && lane == 0);
    while (ti.valid) {
      if ((int)(g & 1u) == e) {
        if (tr) trace_ev<DBG>(p, g, 3 + 2 * e);
        bool pt_wait = g >= (uint32_t)p.npb;
        mbar_wait(&s_full[er.idx], er.phase);
        tc_fence_after();
        if (tr) trace_ev<DBG>(p, g, 4 + 2 * e);
        const uint32_t base = tS(sb) + lane_off + col0;
        const uint32_t rowb0 = smem_u32(sP) + pbuf(g) * PBUF + rowb_base;
        uint32_t ra[32], hi[16], lo[16];
#pragma unroll
        for (int c = 0; c < BN / 64; ++c) {
          tmem_ld32(base + 32 * c, ra);
          tmem_wait_ld(ra);
          if (c == BN / 64 - 1 && !p_tmem) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_free[er.idx]);
          }
          transform_chunk<FAM>(ra, L, hi, lo);
          if (p_tmem) {
            if (FAM == NCGP_RBF) {
              tmem_st_hilo(base + 32 * c, hi, lo);
            } else {
              tmem_st16(base + 32 * c, hi);
              tmem_st16(base + 32 * c + 16, lo);
            }
          }
          if (pt_wait) {  // tile g - npb's GEMM2 and T are done with the buffer
            const uint32_t t = g - (uint32_t)p.npb;
            mbar_wait(&pt_free[t & 1u], (t >> 1) & 1u);
            pt_wait = false;
            if (tr) trace_ev<DBG>(p, g, 8);
          }
          const uint32_t rowb = rowb0 + 512u * c;
          if (!(DBG && (p.sym_dbg & 16))) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              st_shared_v4(rowb + 128u * k, hi[4 * k], hi[4 * k + 1], hi[4 * k + 2], hi[4 * k + 3]);
              st_shared_v4(rowb + PBUF / 2 + 128u * k, lo[4 * k], lo[4 * k + 1], lo[4 * k + 2], lo[4 * k + 3]);
            }
          }
        }
        if (p_tmem) {
          tmem_wait_st();
          tc_fence_before();
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&rdy[er.idx]);
        if (tr) trace_ev<DBG>(p, g, e == 0 ? 7 : 10);
      }
      ++g;
      sb = sb + 1u == (uint32_t)NS1 ? 0u : sb + 1u;
      er.adv();
      ti.next(p);
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    // ================= drains: O every CH tiles, D_T every transposed tile =================
    // into the int64 fixed-point accumulator (fx_flush8, deterministic)
    const int wq = warp & 3;
    const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
    constexpr uint32_t NBLK = WP == 32 ? 2u : 1u;  // staging blocks per warp (BM x WP x 4 bytes)
    const uint32_t stg_warp = smem_u32(sStage) + (uint32_t)wq * NBLK * 2048u;
    uint32_t nst = 0;
    auto drain = [&](uint32_t tacc, int64_t row0, bool skip, bool two) {
#pragma unroll
      for (int h = 0; h < WP / 8; ++h) {
        uint32_t x[8], y[8];
        tmem_ld8(tacc + lane_off + 8 * h, x);       // merged: all three terms; else hi Vhi + lo Vhi
        if (two) tmem_ld8(tacc + lane_off + WP + 8 * h, y);  // [WP, 2 WP): hi Vlo
        tmem_wait_ld();
        float v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = two ? __uint_as_float(x[c]) + __uint_as_float(y[c]) : __uint_as_float(x[c]);
        if (NCGP_SYM1_RED) {
          fx_red8(p, lane, h, v, row0, skip);
        } else {
          fx_flush8<NBLK>(p, stg_warp, nst, lane, h, v, row0, skip);
        }
      }
      tc_fence_before();
    };
    Tile1 ti;
    ti.start(p);
    uint32_t q = 0, dtq = 0;
    while (ti.valid) {
      if (ti.transposed()) {
        mbar_wait(&dt_full[dtq % NDT], (dtq / NDT) & 1u);
        tc_fence_after();
        if (!(DBG && (p.sym_dbg & 8))) drain(tDT(dtq % NDT), (int64_t)ti.ct * BM + 32 * wq, DBG && (p.sym_dbg & 1), !TM);
        else tc_fence_before();
        if (lane == 0) mbar_arrive(&dt_empty[dtq % NDT]);
        ++dtq;
      }
      if (ti.last_in_chunk()) {
        mbar_wait(&o_full[q & 1u], (q >> 1) & 1u);
        tc_fence_after();
        drain(tO(q & 1u), (int64_t)ti.r * BM + 32 * wq, DBG && (p.sym_dbg & 2), !PT);
        if (lane == 0) mbar_arrive(&o_empty[q & 1u]);
        ++q;
      }
      ti.next(p);
    }
    if (lane == 0 && !NCGP_SYM1_RED) bulk_wait_all();
  }

  if (DBG && p.trace != nullptr && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[TRACE_TILES * TRACE_EV + 4 * blockIdx.x + 1] = (long long)t;
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ blocked symmetric kernel
// K1-sym2: the symmetric K(X, X) product on blocks of RB = 4 row tiles.
// Work item = (row block b, column tiles [c0, c1), 16 of them by default);
// tiles run column-major inside the item: for each column tile J the row
// tiles I = 4b .. min(4b+3, J) of the block.  So
//   * the 4 row accumulators O_I stay in TMEM for the whole item (flushed
//     once per item, i.e. every 2048 columns as in the other flavours), and
//   * the transposed accumulator D_T(J) collects the block's row tiles before
//     it is drained: one int64 staging + bulk reduction per 4 tiles instead of
//     per tile (the shared-memory traffic that bound K1-sym1, ncu r02b).
// The column tile's data (XB_J, V_J) stays in shared memory for its tiles;
// the row data (XA_I, V_I) is streamed per tile.
// Pipelining (tools/trace_sym2.py): S (GEMM1's output) is single-buffered and
// released as soon as the epilogue has loaded it; P, which GEMM2 reads from
// TMEM, has its own double-buffered region -- so neither GEMM2 nor the
// epilogue's transcendentals sit on the S round trip.  That needs P in 96
// TMEM columns per tile: P_hi in fp16 (64) and the split term P_lo in E4M3
// (32).  P_hi is rounded to nearest, so |P_lo| <= 2^-12 |P|; P_lo * 2^6 and
// Vhi * 2^-6 are E4M3 (kind::f8f6f4, K = 32): the term is 2^-12 of the
// product and its 2^-4 relative rounding adds ~1e-5 relative error
// (measured against fp64 in tests/test_gpu_symmetric.py).
// Both products take the same split:
//   GEMM2  O_I  += P_hi [Vhi_J ; Vlo_J] (two N = WP MMAs per k-step, A = P_hi
//                  in TMEM) + P_lo8 Vhi8_J (A in TMEM)
//   T      D_T(J) += P_hi^T [Vhi_I | Vlo_I] (N = 2 WP, A MN-major in shared
//                  memory) + P_lo8^T Vhi8_I
// Every tcgen05.mma operand is warp-uniform (see `uni` below).
// Roles (24 warps): warp 0 lane 0 producer; warp 1 GEMM2; warp 2 TMEM
// allocation + GEMM1; warp 3 the transposed product T; warps 4-19 the
// epilogue (two groups alternating tiles); warps 20-23 the drains (D_T per
// column tile, the 4 O accumulators at each item's end) into the int64
// fixed-point accumulator (deterministic, as K1-sym1).
// The CTA's tile sequence: items (row block, column range), column-major inside.
struct Tile2 {
  int it, c0, c1, ct, r, rlo, rend;
  bool valid;
  __device__ __forceinline__ void load(const TcParams& p) {
    const int4 t = p.item_tab[it];
    rlo = RB * t.x;
    rend = min(rlo + RB, (int)p.col_tiles);
    c0 = t.y;
    c1 = t.z;
    ct = c0;
    r = rlo;
  }
  __device__ __forceinline__ void start(const TcParams& p) {
    it = (int)blockIdx.x;
    valid = it < p.n_items;
    if (valid) load(p);
  }
  __device__ __forceinline__ int rhi() const { return min(rend, ct + 1); }
  __device__ __forceinline__ void next(const TcParams& p) {
    if (++r >= rhi()) {
      r = rlo;
      if (++ct >= c1) {
        it += (int)gridDim.x;
        valid = it < p.n_items;
        if (valid) load(p);
      }
    }
  }
  __device__ __forceinline__ bool first_r() const { return r == rlo; }   // new column tile
  __device__ __forceinline__ bool last_r() const { return r + 1 == rhi(); }
  __device__ __forceinline__ bool tp() const { return r < ct; }          // off-diagonal
  __device__ __forceinline__ bool tp_first() const { return r < ct && r == rlo; }
  __device__ __forceinline__ bool tp_last() const { return r < ct && r + 1 == min(rend, ct); }
  __device__ __forceinline__ int k() const { return r - rlo; }
  __device__ __forceinline__ bool o_fresh() const { return ct == max(c0, r); }
  __device__ __forceinline__ bool o_last() const { return ct == c1 - 1; }
};

// DBG: per-tile clock64 trace of CTA 0 (tools/trace_sym2.py): 0/1/2 GEMM1 wait/go/issued,
// 3/4/5/6 epilogue wait/s_full/S released/done, 7/8/9 GEMM2 wait/go/issued,
// 10/11/12 T wait/go/issued, 13/14 drain of D_T start/done
template <int FAM, int WP, bool DBG>
__global__ void __launch_bounds__(NTHREADS, 1) kop_sym2_kernel(const TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // TMEM: S (NS x 128) | P (NP x 96) | O_0..O_{RB-1} (WP each) | D_T (2 WP, NDT buffers)
  constexpr uint32_t NS = NCGP_SYM2_NS, NP = NCGP_SYM2_NP;
  constexpr uint32_t TBASE = NS * BN + NP * TP2 + RB * WP;
  constexpr uint32_t NDT = TBASE + 4 * WP <= TMEM_COLS ? 2u : 1u;
  static_assert(TBASE + NDT * 2 * WP <= TMEM_COLS, "TMEM budget");
  const uint32_t vb_bytes = 2u * p.v2_bytes;        // [Vhi | Vlo]: 2 WP rows x 128
  const uint32_t vi_bytes = vb_bytes + p.v8_bytes;  // + Vhi in E4M3
  uint8_t* sXA = smem;                                   // [sx] row tiles
  uint8_t* sVI = sXA + (size_t)p.sx * p.a_bytes;         // [sv] row tiles' V (T's B)
  uint8_t* sXB = sVI + (size_t)p.sv * vi_bytes;          // [2] column tile XB
  uint8_t* sVJ = sXB + 2 * (size_t)p.a_bytes;            // [2] column tile V (GEMM2's B)
  uint8_t* sP = sVJ + 2 * (size_t)vi_bytes;              // [2] P for T
  uint8_t* sStage = sP + 2 * (size_t)P2BUF;              // [4 warps][nblk] 2 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + 4 * p.nblk * 2048);
  uint64_t* xa_full = bars;              // [4]
  uint64_t* vi_full = xa_full + 4;       // [4]
  uint64_t* xb_full = vi_full + 4;       // [2]
  uint64_t* xb_empty = xb_full + 2;      // [2]  GEMM1 done with the slot
  uint64_t* vj_full = xb_empty + 2;      // [2]
  uint64_t* vj_empty = vj_full + 2;      // [2]  GEMM2 done with the slot
  uint64_t* s_full = vj_empty + 2;       // [NR2] GEMM1(g) done
  uint64_t* s_free = s_full + NR2;       // [NR2] S(g) loaded by the epilogue (8 warps)
  uint64_t* rdy = s_free + NR2;          // [NR2] P(g) in TMEM and shared memory (8 warps)
  uint64_t* g2done = rdy + NR2;          // [NR2] GEMM2(g) done (P region g & 1 free)
  uint64_t* tdone = g2done + NR2;        // [NR2] T(g) done (P smem buffer and V_I slot free)
  uint64_t* o_full = tdone + NR2;        // [RB]
  uint64_t* o_empty = o_full + RB;       // [RB] 4 drain warps (after loading O)
  uint64_t* dt_full = o_empty + RB;      // [2]
  uint64_t* dt_empty = dt_full + 2;      // [2]  4 drain warps (after loading D_T)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dt_empty + 2);
  volatile uint32_t* g1_cnt = tmem_slot + 1;  // GEMM1 tiles issued (NCGP_SYM2_HOLD)

  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) {
      mbar_init(&xa_full[s], 1);
      mbar_init(&vi_full[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&xb_full[s], 1);
      mbar_init(&xb_empty[s], 1);
      mbar_init(&vj_full[s], 1);
      mbar_init(&vj_empty[s], 1);
      mbar_init(&dt_full[s], 1);
      mbar_init(&dt_empty[s], 4);
    }
    for (int s = 0; s < NR2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], 8);
      mbar_init(&rdy[s], 8);
      mbar_init(&g2done[s], 1);
      mbar_init(&tdone[s], 1);
    }
    for (int k = 0; k < RB; ++k) {
      mbar_init(&o_full[k], 1);
      mbar_init(&o_empty[k], 4);
    }
    *g1_cnt = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // Every operand of a tcgen05.mma must be warp-uniform in the compiler's
  // analysis, or ptxas wraps each MMA in an ELECT / R2UR.BROADCAST waterfall
  // loop that costs ~50 cycles per instruction (tools/mma_issue_probe.cu:
  // 16.9 cycles per TS N = 32 MMA with uniform operands).  Values that derive
  // from loads (the TMEM base, the work-item fields) are broadcast from lane 0
  // with __shfl_sync, which the compiler treats as uniform.
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  auto uni = [](uint32_t v) -> uint32_t { return __shfl_sync(0xffffffffu, v, 0); };
  auto tS = [&](uint32_t b) -> uint32_t { return tmem + b * (uint32_t)BN; };
  auto tP = [&](uint32_t b) -> uint32_t { return tmem + NS * (uint32_t)BN + b * TP2; };
  auto tO = [&](uint32_t k) -> uint32_t { return tmem + NS * (uint32_t)BN + NP * TP2 + k * (uint32_t)WP; };
  auto tDT = [&](uint32_t b) -> uint32_t { return tmem + TBASE + b * (uint32_t)(2 * WP); };
  auto par = [](uint32_t t) -> uint32_t { return (t / NR2) & 1u; };

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(NCGP_SYM2_REG_LO));
    if (warp == 0) {
      // ================= producers =================
      // lane 0: GEMM1's operands (XA per tile, XB per column tile); lane 1:
      // the V blocks (V_I per tile for T, V_J per column tile for GEMM2).  Two
      // threads, so that waiting for T to free a V_I slot never delays the
      // next row tile's XA (GEMM1 is on the single S buffer's round trip).
      if (lane < 2) {
        Tile2 ti;
        ti.start(p);
        Ring r;
        r.init((uint32_t)(lane == 0 ? p.sx : p.sv));
        uint32_t g = 0, jq = 0;
        while (ti.valid) {
          const uint32_t s = jq & 1u;
          if (lane == 0) {
            if (ti.first_r()) {  // this column tile's XB, for its <= 4 tiles
              const uint8_t* rec = p.col_pack + (int64_t)ti.ct * p.tile_stride;
              if (jq >= 2) mbar_wait_relaxed(&xb_empty[s], ((jq >> 1) & 1u) ^ 1u);
              mbar_expect_tx(&xb_full[s], p.a_bytes);
              uint8_t* dx = sXB + (size_t)s * p.a_bytes;
              bulk_g2s(dx, rec, p.xbh_bytes, &xb_full[s]);
              bulk_g2s(dx + p.xbh_bytes, rec + p.rec_bytes, p.xbh_bytes, &xb_full[s]);
            }
            if (g >= (uint32_t)p.sx) {  // XA slot freed by GEMM1(g - sx)
              const uint32_t t = g - (uint32_t)p.sx;
              mbar_wait_relaxed(&s_full[t % NR2], par(t));
            }
            mbar_expect_tx(&xa_full[r.idx], p.a_bytes);
            bulk_g2s(sXA + (size_t)r.idx * p.a_bytes, p.xa_pack + (int64_t)ti.r * p.a_bytes, p.a_bytes,
                     &xa_full[r.idx]);
          } else {
            auto load_v = [&](uint8_t* dst, int64_t tile, uint64_t* bar) {  // [Vhi | Vlo | Vhi8]
              const uint8_t* rec = p.col_pack + tile * p.tile_stride;
              bulk_g2s(dst, rec + p.xbh_bytes, p.v2_bytes, bar);
              bulk_g2s(dst + p.v2_bytes, rec + p.rec_bytes + p.xbh_bytes, p.v2_bytes, bar);
              bulk_g2s(dst + vb_bytes, p.v8_pack + tile * p.v8_bytes, p.v8_bytes, bar);
            };
            if (ti.first_r()) {  // V_J for GEMM2
              if (jq >= 2) mbar_wait_relaxed(&vj_empty[s], ((jq >> 1) & 1u) ^ 1u);
              mbar_expect_tx(&vj_full[s], vi_bytes);
              load_v(sVJ + (size_t)s * vi_bytes, ti.ct, &vj_full[s]);
            }
            if (g >= (uint32_t)p.sv) {  // V_I slot freed by T(g - sv)
              const uint32_t t = g - (uint32_t)p.sv;
              mbar_wait_relaxed(&tdone[t % NR2], par(t));
            }
            mbar_expect_tx(&vi_full[r.idx], vi_bytes);
            load_v(sVI + (size_t)r.idx * vi_bytes, ti.r, &vi_full[r.idx]);
          }
          jq += ti.first_r() ? 1u : 0u;
          r.adv();
          ++g;
          ti.next(p);
        }
      }
    } else if (warp == 2) {
      // ================= GEMM1: S(g) = XA_I . XB_J^T =================
      const uint32_t sbo_x = (uint32_t)(p.ka / 8) * 128u;
      const int ksteps1 = p.ka / 16;
      const uint64_t dA0 = sdesc(smem_u32(sXA), 128u, sbo_x);
      const uint64_t dX0 = sdesc(smem_u32(sXB), 128u, sbo_x);
      const uint32_t id1 = idesc1_f16(BN);
      Tile2 ti;
      ti.start(p);
      Ring xr;
      xr.init((uint32_t)p.sx);
      uint32_t g = 0, jq = 0;
      while (ti.valid) {
        const uint32_t s = jq & 1u;
        if (lane == 0) trace_ev<DBG>(p, g, 0);
        if (ti.first_r()) mbar_wait(&xb_full[s], (jq >> 1) & 1u);
        mbar_wait(&xa_full[xr.idx], xr.phase);
        if (g >= NS) mbar_wait(&s_free[(g - NS) % NR2], par(g - NS));  // S(g - NS) loaded
        tc_fence_after();
        if (lane == 0) trace_ev<DBG>(p, g, 1);
        const uint64_t da = dA0 + (uint64_t)xr.idx * (p.a_bytes >> 4);
        const uint32_t su = uni(s), lr = uni(ti.last_r() ? 1u : 0u);
        const uint64_t dx = dX0 + (uint64_t)su * (p.a_bytes >> 4);
        if (elect_one()) {
          for (int k = 0; k < ksteps1; ++k)
            mma1_ss(tS(g % NS), da + (uint64_t)(16 * k), dx + (uint64_t)(16 * k), id1, k > 0);
          tc_commit1(&s_full[g % NR2]);  // also frees the XA slot (producer)
          if (lr) tc_commit1(&xb_empty[su]);
        }
        __syncwarp();
        if (lane == 0) trace_ev<DBG>(p, g, 2);
        if ((NCGP_SYM2_HOLD || NCGP_SYM2_HOLDG2) && lane == 0) *g1_cnt = g + 1u;
        jq += ti.last_r() ? 1u : 0u;
        xr.adv();
        ++g;
        ti.next(p);
      }
      if (lane == 0) *g1_cnt = 0xFFFFFFFFu;
    } else if (warp == 1) {
      // ================= GEMM2: O_I += P_hi [Vhi_J ; Vlo_J] + P_lo8 Vhi8_J (A = P in TMEM) =================
      const uint32_t id2h = idesc1_f16(WP), id28 = idesc1_f8(WP, false);
      const uint64_t dV0 = sdesc(smem_u32(sVJ), 128u, (uint32_t)(BN * 16));
      const uint64_t dV80 = sdesc(smem_u32(sVJ) + vb_bytes, 128u, 1024u);
      const uint64_t vlo = (uint64_t)(p.v2_bytes >> 4);
      Tile2 ti;
      ti.start(p);
      uint32_t g = 0, jq = 0, ouse = 0;  // ouse bit k: parity of O_k's uses
      while (ti.valid) {
        const uint32_t s = jq & 1u;
        const int k = ti.k();
        const bool fresh = ti.o_fresh();
        if (lane == 0) trace_ev<DBG>(p, g, 7);
        mbar_wait(&rdy[g % NR2], par(g));
        if (ti.first_r()) mbar_wait(&vj_full[s], (jq >> 1) & 1u);
        if (fresh) {
          mbar_wait(&o_empty[k], ((ouse >> k) & 1u) ^ 1u);
          ouse ^= 1u << k;
        }
        if (NCGP_SYM2_HOLDG2)  // GEMM2(g) behind GEMM1(g + HOLDG2) in the in-order tensor pipe
          while (*g1_cnt < g + 1u + (uint32_t)NCGP_SYM2_HOLDG2 && *g1_cnt != 0xFFFFFFFFu) {
          }
        tc_fence_after();
        if (lane == 0) trace_ev<DBG>(p, g, 8);
        const uint32_t su = uni(s), ku = uni((uint32_t)k), fu = uni(fresh ? 1u : 0u);
        const uint32_t ol = uni(ti.o_last() ? 1u : 0u), lr = uni(ti.last_r() ? 1u : 0u);
        const uint64_t vo = (uint64_t)su * (vi_bytes >> 4);
        const uint32_t dO = tO(ku), a0 = tP(g % NP);
        if (elect_one()) {
#pragma unroll
          for (int m = 0; m < ((NCGP_SYM2_ABL & 4) ? 0 : BN / 16); ++m) {
            const uint64_t b = dV0 + vo + (uint64_t)(16 * m);
            mma1_ts(dO, a0 + 8u * m, b, id2h, (fu != 0u && m == 0) ? 0u : 1u);
            mma1_ts(dO, a0 + 8u * m, b + vlo, id2h, 1u);
          }
#ifndef NCGP_SYM2_G2F8
#define NCGP_SYM2_G2F8 1
#endif
#pragma unroll
          for (int q = 0; q < (NCGP_SYM2_G2F8 ? BN / 32 : 0); ++q)
            mma1_f8_ts(dO, a0 + 64u + 8u * q, dV80 + vo + (uint64_t)(16 * q), id28, 1u);
          tc_commit1(&g2done[g % NR2]);
          if (ol) tc_commit1(&o_full[ku]);
          if (lr) tc_commit1(&vj_empty[su]);
        }
        __syncwarp();
        if (lane == 0) trace_ev<DBG>(p, g, 9);
        jq += ti.last_r() ? 1u : 0u;
        ++g;
        ti.next(p);
      }
    } else {
      // ================= T: D_T(J) += P_hi^T [Vhi_I | Vlo_I] + P_lo8^T Vhi8_I =================
      const uint32_t idT = idesc1_f16(2 * WP, true), idT8 = idesc1_f8(WP, true);
      const uint64_t dPH0 = sdesc(smem_u32(sP), 2048u, 128u);        // MN-major fp16
      const uint64_t dP80 = sdesc(smem_u32(sP) + PH2, 1024u, 128u);  // MN-major E4M3
      const uint64_t dVI0 = sdesc(smem_u32(sVI), 128u, (uint32_t)(BN * 16));
      const uint64_t dV80 = sdesc(smem_u32(sVI) + vb_bytes, 128u, 1024u);
      Tile2 ti;
      ti.start(p);
      Ring vr;
      vr.init((uint32_t)p.sv);
      uint32_t g = 0, dq = 0;
      while (ti.valid) {
        if (lane == 0) trace_ev<DBG>(p, g, 10);
        mbar_wait(&rdy[g % NR2], par(g));
        mbar_wait(&vi_full[vr.idx], vr.phase);
        const bool tp = ti.tp();
        if (ti.tp_first()) mbar_wait(&dt_empty[dq % NDT], ((dq / NDT) & 1u) ^ 1u);
        if (NCGP_SYM2_HOLD)  // T(g) behind GEMM1(g + HOLD) in the in-order tensor pipe
          while (*g1_cnt < g + 1u + (uint32_t)NCGP_SYM2_HOLD && *g1_cnt != 0xFFFFFFFFu) {
          }
        tc_fence_after();
        if (lane == 0) trace_ev<DBG>(p, g, 11);
        const uint32_t tpu = uni(tp ? 1u : 0u), fu = uni(ti.tp_first() ? 1u : 0u);
        const uint32_t tlu = uni(ti.tp_last() ? 1u : 0u), dqb = uni(dq % NDT);
        if (elect_one()) {
          if (tpu) {
            const uint64_t pb = (uint64_t)(g & 1u) * (P2BUF >> 4);
            const uint64_t vo = (uint64_t)vr.idx * (vi_bytes >> 4);
            const uint32_t dt = tDT(dqb);
#pragma unroll
            for (int m = 0; m < ((NCGP_SYM2_ABL & 1) ? 0 : BN / 16); ++m)
              mma1_ss(dt, dPH0 + pb + (uint64_t)m * (4096 >> 4), dVI0 + vo + (uint64_t)(16 * m), idT,
                      (fu != 0u && m == 0) ? 0u : 1u);
#pragma unroll
            for (int q = 0; q < ((NCGP_SYM2_ABL & 1) ? 0 : BN / 32); ++q)
              mma1_f8_ss(dt, dP80 + pb + (uint64_t)q * (4096 >> 4), dV80 + vo + (uint64_t)(16 * q), idT8, 1u);
            if (tlu) tc_commit1(&dt_full[dqb]);
          }
          tc_commit1(&tdone[g % NR2]);
        }
        __syncwarp();
        if (lane == 0) trace_ev<DBG>(p, g, 12);
        dq += ti.tp_last() ? 1u : 0u;
        vr.adv();
        ++g;
        ti.next(p);
      }
    }
  } else if (warp < 4 + EPI_WARPS) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 96;");  // the CTA pool: 8192 released by the decs
    // ================= epilogue: two groups of 8 warps alternate tiles =================
    const int e = (warp - 4) / 8;
    const int hc = ((warp - 4) % 8) / 4;
    const int wq = warp & 3;
    const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
    const uint32_t col0 = (uint32_t)(hc * (BN / 2));
    const int i = 32 * wq + lane;
    const uint32_t rowh = (uint32_t)(i >> 3) * 2048u + (uint32_t)(i & 7) * 16u + (col0 >> 3) * 128u;
    const uint32_t row8 = PH2 + (uint32_t)(i >> 3) * 1024u + (uint32_t)(i & 7) * 16u + (col0 >> 4) * 128u;
    Tile2 ti;
    ti.start(p);
    const float L = p.L;
    uint32_t g = 0;
    const bool tr = wq == 0 && hc == 0 && lane == 0;
    while (ti.valid) {
      if ((int)(g & 1u) == e) {
        const bool tp = ti.tp();
        if (tr) trace_ev<DBG>(p, g, 3);
        mbar_wait(&s_full[g % NR2], par(g));
        tc_fence_after();
        if (tr) trace_ev<DBG>(p, g, 4);
        // load both chunks of S, then release the (single) S buffer to GEMM1
        uint32_t ra[32], rb[32], hi[16], l8[8];
        tmem_ld32(tS(g % NS) + lane_off + col0, ra);
        tmem_ld32(tS(g % NS) + lane_off + col0 + 32, rb);
        tmem_wait_ld(ra);
        tmem_wait_ld(rb);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[g % NR2]);
        if (tr) trace_ev<DBG>(p, g, 5);
        const uint32_t pr = tP(g % NP) + lane_off;
        const uint32_t pbase = smem_u32(sP) + (g & 1u) * P2BUF;
#if NCGP_SYM2_LATE
        // Transform both chunks into registers first, and only then wait for
        // this group's P region (GEMM2(g - NP)) and P buffer (T(g - 2)): those
        // were issued when this group finished its previous tile, so waiting
        // before the first store would idle the group for most of their run.
        uint32_t hi1[16], l81[8];
        transform_chunk2<FAM>(ra, L, hi, l8);
        transform_chunk2<FAM>(rb, L, hi1, l81);
        if (g >= NP) {  // GEMM2(g - NP) has read this P region
          mbar_wait(&g2done[(g - NP) % NR2], par(g - NP));
          tc_fence_after();
        }
        {
          const uint32_t cc = col0 >> 5;  // first chunk of the tile (0 or 2)
          tmem_st16(pr + 16u * cc, hi);
          tmem_st8(pr + 64u + 8u * cc, l8);
          tmem_st16(pr + 16u * (cc + 1u), hi1);
          tmem_st8(pr + 64u + 8u * (cc + 1u), l81);
        }
        if (tp && !(NCGP_SYM2_ABL & 2)) {
          if (g >= 2u)  // T(g - 2) is done with this P smem buffer
            mbar_wait(&tdone[(g - 2u) % NR2], par(g - 2u));
          const uint32_t rh = pbase + rowh;
          const uint32_t r8 = pbase + row8;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            st_shared_v4(rh + 128u * k, hi[4 * k], hi[4 * k + 1], hi[4 * k + 2], hi[4 * k + 3]);
          st_shared_v4(r8, l8[0], l8[1], l8[2], l8[3]);
          st_shared_v4(r8 + 128u, l8[4], l8[5], l8[6], l8[7]);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            st_shared_v4(rh + 512u + 128u * k, hi1[4 * k], hi1[4 * k + 1], hi1[4 * k + 2], hi1[4 * k + 3]);
          st_shared_v4(r8 + 256u, l81[0], l81[1], l81[2], l81[3]);
          st_shared_v4(r8 + 256u + 128u, l81[4], l81[5], l81[6], l81[7]);
        }
#else
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c == 0)
            transform_chunk2<FAM>(ra, L, hi, l8);
          else
            transform_chunk2<FAM>(rb, L, hi, l8);
          if (c == 0 && g >= NP) {  // GEMM2(g - NP) has read this P region
            mbar_wait(&g2done[(g - NP) % NR2], par(g - NP));
            tc_fence_after();
          }
          const uint32_t cc = (col0 >> 5) + (uint32_t)c;  // chunk of the tile (0..3)
          tmem_st16(pr + 16u * cc, hi);
          tmem_st8(pr + 64u + 8u * cc, l8);
          if (tp && !(NCGP_SYM2_ABL & 2)) {
            if (c == 0 && g >= 2u)  // T(g - 2) is done with this P smem buffer
              mbar_wait(&tdone[(g - 2u) % NR2], par(g - 2u));
            const uint32_t rh = pbase + rowh + 512u * c;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              st_shared_v4(rh + 128u * k, hi[4 * k], hi[4 * k + 1], hi[4 * k + 2], hi[4 * k + 3]);
            const uint32_t r8 = pbase + row8 + 256u * c;
            st_shared_v4(r8, l8[0], l8[1], l8[2], l8[3]);
            st_shared_v4(r8 + 128u, l8[4], l8[5], l8[6], l8[7]);
          }
        }
#endif
        tmem_wait_st();
        tc_fence_before();
        if (tp) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&rdy[g % NR2]);
        if (tr) trace_ev<DBG>(p, g, 6);
      }
      ++g;
      ti.next(p);
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(NCGP_SYM2_REG_DR));
    // ================= drains: D_T per column tile, O_I at each item's end =================
    // Each accumulator is loaded into registers and released at once (D_T is
    // single-buffered at WP = 32), then rounded to int64 and bulk-reduced.
    const int wq = warp & 3;
    const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
    // int64 fixed point straight from registers: one coalesced red.global.add.u64
    // per column (the accumulator is column-major here, [WP][acc_rows]) -- no
    // shared-memory staging and no TMA queueing behind the producers' loads
    // (bulk reductions through 2 KB staging blocks cost 14 % at n = 2e5).
    auto flush = [&](const float (&v)[WP], int64_t row0) {
      if (NCGP_SYM2_ABL & 8) return;
      unsigned long long* dst = p.acc + row0 + lane;
#pragma unroll
      for (int c = 0; c < WP; ++c) {
        const long long q = __float2ll_rn(v[c] * p.fx);
        atomicAdd(dst + (int64_t)c * p.acc_rows, (unsigned long long)q);
      }
    };
    Tile2 ti;
    ti.start(p);
    uint32_t dq = 0, ouse = 0, g = 0;
    while (ti.valid) {
      if (ti.tp_last()) {
        if (wq == 0 && lane == 0) trace_ev<DBG>(p, g, 13);
        mbar_wait_relaxed(&dt_full[dq % NDT], (dq / NDT) & 1u);
        tc_fence_after();
        float v[WP];
        const uint32_t ta = tDT(dq % NDT) + lane_off;
#pragma unroll
        for (int h = 0; h < WP / 8; ++h) {
          uint32_t x[8], y[8];
          tmem_ld8(ta + 8 * h, x);
          tmem_ld8(ta + WP + 8 * h, y);  // [WP, 2 WP): P_hi^T Vlo
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 8; ++c) v[8 * h + c] = __uint_as_float(x[c]) + __uint_as_float(y[c]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dt_empty[dq % NDT]);
        flush(v, (int64_t)ti.ct * BM + 32 * wq);
        if (wq == 0 && lane == 0) trace_ev<DBG>(p, g, 14);
        ++dq;
      }
      if (ti.o_last()) {
        const int k = ti.k();
        mbar_wait_relaxed(&o_full[k], (ouse >> k) & 1u);
        ouse ^= 1u << k;
        tc_fence_after();
        float v[WP];
        const uint32_t ta = tO((uint32_t)k) + lane_off;
#pragma unroll
        for (int h = 0; h < WP / 8; ++h) {
          uint32_t x[8];
          tmem_ld8(ta + 8 * h, x);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 8; ++c) v[8 * h + c] = __uint_as_float(x[c]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_empty[k]);
        flush(v, (int64_t)ti.r * BM + 32 * wq);
      }
      ++g;
      ti.next(p);
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ packing

// column means of Xc in fp64 (single block, fixed order)
template <typename T>
__global__ void col_mean_kernel(const T* __restrict__ X, int64_t n, int d, double* __restrict__ mu) {
  __shared__ double sm[32];
  for (int f = 0; f < d; ++f) {
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += (double)X[i * d + f];
    double s = ncgp::block_sum(acc, sm);
    if (threadIdx.x == 0) mu[f] = n > 0 ? s / (double)n : 0.0;
    __syncthreads();
  }
}

__device__ __forceinline__ __half h_of(double v) { return __double2half(v); }

// Writes the augmented rows of one operand into the canonical K-major
// no-swizzle layout: tile | row-group g | k-chunk q | row r | k.
// role 0 = row operand (A), role 1 = column operand (B).
// Column operand tiles are split in two 64-row halves, one per CTA of a pair:
// rows 0-63 at the record start, rows 64-127 at +half (CTA1's half record).
template <typename T>
__global__ void pack_x_kernel(const T* __restrict__ X, int64_t n, int d, int ka,
                              const double* __restrict__ mu, double alpha, double sign,
                              double L, int role, uint8_t* __restrict__ pack, int64_t stride,
                              int64_t half, int64_t n_tiles) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int qn = ka / 8;
  const int64_t rows = n_tiles * BM;
  if (e >= rows * qn) return;
  const int64_t row = e / qn;
  const int q = (int)(e % qn);
  const int64_t tile = row / BM;
  const int r = (int)(row % BM);
  uint16_t out[8];
  if (row >= n) {
#pragma unroll
    for (int k = 0; k < 8; ++k) out[k] = 0;
  } else {
    double nrm = 0.0;
    for (int f = 0; f < d; ++f) {
      const double x = ((double)X[row * d + f] - mu[f]) * alpha;
      nrm += x * x;
    }
    // a/b term: RBF  a = -|x|^2 (+L on the column side), Matern  a = +|x|^2
    const double ab = (sign > 0 ? -nrm : nrm) + (role == 1 ? L : 0.0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = q * 8 + k;
      double v = 0.0;
      if (idx < 3 * d) {
        const int f = idx % d;
        const int part = idx / d;  // 0,1,2
        const double x = ((double)X[row * d + f] - mu[f]) * alpha;
        const double xs = role == 0 ? 2.0 * sign * x : x;
        const double hi = (double)__half2float(h_of(xs));
        const double lo = (double)__half2float(h_of(xs - hi));
        if (role == 0)
          v = (part == 1) ? lo : hi;  // [u_hi, u_lo, u_hi]
        else
          v = (part == 2) ? lo : hi;  // [x_hi, x_hi, x_lo]
      } else if (idx < 3 * d + 4) {
        const int t = idx - 3 * d;
        const double hi = (double)__half2float(h_of(ab));
        const double lo = (double)__half2float(h_of(ab - hi));
        if (role == 0)
          v = (t == 0) ? hi : (t == 1 ? lo : 1.0);       // [a_hi, a_lo, 1, 1]
        else
          v = (t == 2) ? hi : (t == 3 ? lo : 1.0);       // [1, 1, b_hi, b_lo]
      }
      out[k] = __half_as_ushort(h_of(v));
    }
  }
  const int g = r / 8, rr = r % 8;
  uint8_t* dst;
  if (role == 0)
    dst = pack + tile * stride + ((int64_t)(g * qn + q) * 8 + rr) * 16;
  else
    dst = pack + tile * stride + (g >= 8 ? half : 0) + ((int64_t)((g & 7) * qn + q) * 8 + rr) * 16;
  uint4 val;
  val.x = out[0] | ((uint32_t)out[1] << 16);
  val.y = out[2] | ((uint32_t)out[3] << 16);
  val.z = out[4] | ((uint32_t)out[5] << 16);
  val.w = out[6] | ((uint32_t)out[7] << 16);
  *reinterpret_cast<uint4*>(dst) = val;
}

// max |x~|^2 over rows (precision guard), atomicMax on the float bit pattern
template <typename T>
__global__ void max_norm_kernel(const T* __restrict__ X, int64_t n, int d,
                                const double* __restrict__ mu, double alpha,
                                unsigned int* __restrict__ out_bits) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float v = 0.f;
  if (i < n) {
    double nrm = 0.0;
    for (int f = 0; f < d; ++f) {
      const double x = ((double)X[i * d + f] - mu[f]) * alpha;
      nrm += x * x;
    }
    v = (float)nrm;
  }
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  if ((threadIdx.x & 31) == 0) atomicMax(out_bits, __float_as_uint(v));
}

// per RHS column: exponent e_c with max|v_c| * 2^e_c < 2^14  (max is order-free)
template <typename T>
__global__ void col_absmax_kernel(const T* __restrict__ V, int64_t ldv, int64_t n, int w,
                                  unsigned int* __restrict__ bits) {
  const int c = threadIdx.x % 32 + 32 * blockIdx.y;
  if (c >= w) return;
  float m = 0.f;
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; j < n;
       j += (int64_t)gridDim.x * (blockDim.x / 32))
    m = fmaxf(m, fabsf((float)V[j * ldv + c]));
  atomicMax(&bits[c], __float_as_uint(m));
}

__global__ void col_exp_kernel(const unsigned int* __restrict__ bits, int w, int wp,
                               int* __restrict__ col_exp) {
  const int c = threadIdx.x;
  if (c >= wp) return;
  int e = 0;
  if (c < w) {
    const float m = __uint_as_float(bits[c]);
    if (m > 0.f && isfinite(m)) {
      int p;
      frexpf(m, &p);  // m < 2^p
      e = 14 - p;
    }
  }
  col_exp[c] = e;
}

// V (n x w, row stride ldv) -> per column tile and CTA half: B2 (GEMM2 B rows
// for N = 2 WP: CTA0 = Vhi, CTA1 = Vlo) then B3 (N = WP: CTA0 = Vhi rows
// [0, WP/2), CTA1 = Vhi rows [WP/2, WP)).  Each block is K-major no-swizzle:
// c-group g | j-chunk q | row c%8 | j%8 (SBO = 2048 B).
template <typename T>
__global__ void pack_v_kernel(const T* __restrict__ V, int64_t ldv, int64_t n, int w, int wp,
                              const int* __restrict__ col_exp, uint8_t* __restrict__ col_pack,
                              int64_t tile_stride, int64_t half, uint32_t xbh_bytes,
                              uint32_t v2_bytes, int64_t col_tiles, int wide = 0) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t chunks = col_tiles * (BN / 8);
  if (e >= chunks * wp) return;
  const int c = (int)(e % wp);
  const int64_t qg = e / wp;
  const int64_t tile = qg / (BN / 8);
  const int q = (int)(qg % (BN / 8));
  const int64_t j0 = qg * 8;
  const float sc = ldexpf(1.f, col_exp[c]);
  uint16_t hi[8], lo[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int64_t j = j0 + k;
    float v = (j < n && c < w) ? (float)V[j * ldv + c] * sc : 0.f;
    const __half h = __float2half_rn(v);
    hi[k] = __half_as_ushort(h);
    lo[k] = __half_as_ushort(__float2half_rn(v - __half2float(h)));
  }
  const int g = c / 8, rr = c % 8;
  uint8_t* rec = col_pack + tile * tile_stride + xbh_bytes;
  const int64_t in_blk = ((int64_t)q * 8 + rr) * 16;
  uint4 a, b;
  a.x = hi[0] | ((uint32_t)hi[1] << 16); a.y = hi[2] | ((uint32_t)hi[3] << 16);
  a.z = hi[4] | ((uint32_t)hi[5] << 16); a.w = hi[6] | ((uint32_t)hi[7] << 16);
  b.x = lo[0] | ((uint32_t)lo[1] << 16); b.y = lo[2] | ((uint32_t)lo[3] << 16);
  b.z = lo[4] | ((uint32_t)lo[5] << 16); b.w = lo[6] | ((uint32_t)lo[7] << 16);
  const int gh = wp / 16;  // c-groups per CTA in B3 / B4
  const int cta = g / gh;
  if (wide) {
    // wide kernel: B3 (Vhi) then B4 (Vlo), each split between the CTAs
    uint8_t* r = rec + (cta ? half : 0) + (int64_t)(g - cta * gh) * 2048 + in_blk;
    *reinterpret_cast<uint4*>(r) = a;
    *reinterpret_cast<uint4*>(r + v2_bytes / 2) = b;
    return;
  }
  // B2: CTA0 <- Vhi, CTA1 <- Vlo, c-group g at g * 2048
  *reinterpret_cast<uint4*>(rec + (int64_t)g * 2048 + in_blk) = a;
  *reinterpret_cast<uint4*>(rec + half + (int64_t)g * 2048 + in_blk) = b;
  // B3: Vhi c-groups split between the CTAs
  *reinterpret_cast<uint4*>(rec + (cta ? half : 0) + v2_bytes + (int64_t)(g - cta * gh) * 2048 +
                            in_blk) = a;
}

// K1-sym2: Vhi of each column tile in E4M3 (x 2^-LO8_SHIFT), the B operand
// of the transposed product's small split term: K-major, element (c, j) at
// (c / 8) * 1024 + (j / 16) * 128 + (c % 8) * 16 + j % 16.  Vhi is the same
// fp16 value pack_v_kernel stores (|Vhi| < 2^14, so |Vhi 2^-6| < 448).
template <typename T>
__global__ void pack_v8_kernel(const T* __restrict__ V, int64_t ldv, int64_t n, int w, int wp,
                               const int* __restrict__ col_exp, uint8_t* __restrict__ v8,
                               int64_t col_tiles) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t chunks = col_tiles * (BN / 16);
  if (e >= chunks * wp) return;
  const int c = (int)(e % wp);
  const int64_t qg = e / wp;
  const int64_t tile = qg / (BN / 16);
  const int q = (int)(qg % (BN / 16));
  const float sc = ldexpf(1.f, col_exp[c]);
  constexpr float S8 = 1.f / (float)(1 << LO8_SHIFT);
  uint32_t b[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float x[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int64_t j = qg * 16 + 4 * k + t;
      const float v = (j < n && c < w) ? (float)V[j * ldv + c] * sc : 0.f;
      x[t] = __half2float(__float2half_rn(v)) * S8;
    }
    b[k] = e4m3x2(x[0], x[1]) | (e4m3x2(x[2], x[3]) << 16);
  }
  uint4 val;
  val.x = b[0];
  val.y = b[1];
  val.z = b[2];
  val.w = b[3];
  *reinterpret_cast<uint4*>(v8 + tile * ((int64_t)wp * BN) + (c / 8) * 1024 + q * 128 + (c % 8) * 16) = val;
}

template <typename T>
__global__ void reduce_partial_kernel(const double* __restrict__ partial, int splits,
                                      int64_t nloc, int w, const ncgp::OutPtrs<T> out,
                                      int64_t ldo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nloc * w) return;
  double s = 0.0;
  for (int p = 0; p < splits; ++p) s += partial[(int64_t)p * nloc * w + e];
#pragma unroll
  for (int k = 0; k < NCGP_MAX_OUTS; ++k)
    if (k < out.n) out.p[k][(e / w) * ldo + (e % w)] = (T)s;
}

// wide kernel: fixed-order fp64 sum of the fp32 partials [split][row][128],
// scaled back by 2^-(s + e_c), to every destination (coalesced over columns)
template <typename T>
__global__ void wide_reduce_kernel(const float* __restrict__ part, int splits, int64_t nloc,
                                   int w, int s_exp, const int* __restrict__ col_exp,
                                   const ncgp::OutPtrs<T> out, int64_t ldo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nloc * w) return;
  const int64_t i = e / w;
  const int c = (int)(e % w);
  double acc = 0.0;
  for (int sp = 0; sp < splits; ++sp) acc += (double)part[((int64_t)sp * nloc + i) * 128 + c];
  const T v = (T)ldexp(acc, -(s_exp + __ldg(&col_exp[c])));
#pragma unroll
  for (int k = 0; k < NCGP_MAX_OUTS; ++k)
    if (k < out.n) out.p[k][i * ldo + c] = v;
}

// K2 square-reduce (posterior.py:67-84): the pass's columns g0 + c (c < w) of
// A = K(X*, X) [Q_0 | ... | Q_{C-1}] (class-major, R columns per class) are
// summed over splits in fp64 (fixed order), squared, and added to
// sq[row][class] in column order by one thread per row -- A never reaches HBM
// as a whole and the sums are deterministic.  One block of 128 threads per row.
__global__ void wide_sqsum_kernel(const float* __restrict__ part, int splits, int64_t nloc,
                                  int w, int s_exp, const int* __restrict__ col_exp, int g0,
                                  int R, int C, double* __restrict__ sq) {
  __shared__ double a2[128];
  const int64_t i = blockIdx.x;
  const int c = threadIdx.x;
  double a = 0.0;
  if (c < w) {
    for (int sp = 0; sp < splits; ++sp) a += (double)part[((int64_t)sp * nloc + i) * 128 + c];
    a = ldexp(a, -(s_exp + __ldg(&col_exp[c])));
  }
  a2[c] = a * a;
  __syncthreads();
  if (c == 0) {
    int cls = g0 / R;
    double run = 0.0;
    for (int k = 0; k < w; ++k) {
      const int ck = (g0 + k) / R;
      if (ck != cls) {
        sq[i * C + cls] += run;
        run = 0.0;
        cls = ck;
      }
      run += a2[k];
    }
    if (cls < C) sq[i * C + cls] += run;
  }
}

// var[t, c] = max(s2[c] - sq[t, c], 0)  (posterior.py:80-84)
template <typename T>
__global__ void var_finalize_kernel(const double* __restrict__ sq, int64_t n, int C,
                                    const double* __restrict__ s2, T* __restrict__ var,
                                    int64_t ldv) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * C) return;
  const int64_t i = e / C;
  const int c = (int)(e % C);
  const double v = s2[c] - sq[e];
  var[i * ldv + c] = (T)(v > 0.0 ? v : 0.0);
}

// split columns: the fixed-order fp64 sum of the partial rows, one thread per
// row, through the apply's epilogue
template <typename T>
__global__ void reduce_partial_epi_kernel(const double* __restrict__ partial, int splits,
                                          int64_t nloc, int w, const EpiDev e,
                                          const ncgp::OutPtrs<T> out, int64_t ldo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nloc) return;
  auto kv = [&](int c) -> double {
    double s = 0.0;
    for (int p = 0; p < splits; ++p) s += partial[((int64_t)p * nloc + i) * w + c];
    return s;
  };
  ncgp::epi_row<T, NCGP_MAX_OUTS>(e, i, w, kv, out.p, out.n, ldo);
}

// symmetric kernel: rows of the int64 fixed-point accumulator (layout of
// fx_flush8) scaled back by 2^-(F + s + e_c) in fp64, through the epilogue,
// to every destination; one thread per row
__global__ void sym_finalize_kernel(const unsigned long long* __restrict__ acc, int64_t acc_rows,
                                    int64_t row_begin, int64_t n, int w, int fx_exp, int s_exp,
                                    const int* __restrict__ col_exp, const EpiDev e,
                                    const ncgp::OutPtrs<float> out, int64_t ldo, int colmajor) {
  // rows [row_begin, n): every pointer (out, base, out2, V, noise state) is
  // indexed by the operator's global rows
  const int64_t i = row_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int swz = (int)((i >> 1) & 3);
  auto kv = [&](int c) -> double {
    const int h = c >> 3, cc = c & 7;
    const int64_t idx = colmajor ? (int64_t)c * acc_rows + i
                                 : ((int64_t)h * acc_rows + i) * 8 + (((cc >> 1) ^ swz) << 1) + (cc & 1);
    return ldexp((double)(long long)acc[idx], -(fx_exp + s_exp + __ldg(&col_exp[c])));
  };
  ncgp::epi_row<float, NCGP_MAX_OUTS>(e, i, w, kv, out.p, out.n, ldo);
}

// ------------------------------------------------------------------ host

long long* g_trace = nullptr;  // debug hook (ncgp_debug_set_trace)
float* g_sym_dump = nullptr;   // debug hook (ncgp_debug_set_sym_dump)
// Symmetric K(X, X) kernel policy.  Evaluating only the tiles on and right
// of the diagonal halves the transcendental work (the bound of the plain
// kernel) but adds the transposed product and an fp32 reduction of every
// transposed tile.  Two flavours:
//   K1-sym1 (cta_group::1, default where its shared memory fits, D <= ~24):
//     one B200, CUDA events: cfg3 RBF 316 -> 296 ms, cfg3 Matern 542 -> 356
//     ms, RBF w = 10 at n = 1e6 281 -> 209 ms; it loses below ~300 column
//     tiles (the triangular list balances poorly over 148 CTAs);
//   K1-sym (the pair kernel): larger D; wins for Matern-3/2 at any width and
//     for RBF at WP = 16 from ~512 column tiles.
// NCGP_SYM=1 forces it on, NCGP_SYM=0 off (the plain kernel's results are
// bitwise reproducible across row shardings; the symmetric kernels' fp32
// reductions are not).
bool sym_enabled(const ncgp_kop* op, int family, int wp, int64_t col_tiles, int cg) {
  if (op->knob_sym == 0) return false;
  if (op->knob_sym == 1) return true;
  // thresholds from tools/sym_threshold.py (one B200, size-dependent item length):
  // Matern-3/2 (two MUFU ops per pair, so the halving pays early) from ~15k
  // points on every flavour (n = 16k: 0.75-0.82 of the plain kernel's time,
  // 38k: 0.62-0.67); RBF from ~38k on the single-CTA kernels (0.93) and from
  // ~65k at WP = 16 on the pair kernel (D = 50: 0.99-1.10 below that)
  if (family == NCGP_MATERN32) return col_tiles >= 90;   // n = 12k: 0.90-0.92
  // RBF on K1-sym1 at WP = 16 (the fits' C <= 16 operators): 0.87 of the plain
  // kernel's time at n = 16k, 0.73-0.81 from 20k to 38k
  if (cg == 1 && wp == 16) return col_tiles >= 120;
  if (cg == 1 || cg == 3) return col_tiles >= 300;
  return col_tiles >= 512 && wp == 16;
}
int g_debug_mode = 0;          // debug hook (ncgp_debug_set_mode)

int ka_of(int d) { return ((3 * d + 4) + 15) / 16 * 16; }
// padded RHS width of a launch: 16 / 32 (the plain and symmetric kernels) or
// 128 (the wide kernel, 32 < w <= 128)
int wp_of(int w) { return w <= 16 ? 16 : (w <= 32 ? 32 : 128); }
constexpr int WIDE_WP = 128;
#ifndef NCGP_WIDE_ITEM
#define NCGP_WIDE_ITEM 16
#endif
constexpr int WIDE_ITEM = NCGP_WIDE_ITEM;  // column tiles per wide item (fp32 TMEM accumulation span)
constexpr int64_t WIDE_ROWS = 4096;  // rows per wide launch (bounds the fp32 partials)

struct Layout {
  size_t mu, guard, colexp, bits, xa, col, partial, symacc, symtab, varacc, v8, total;
  uint32_t a_bytes, xbh_bytes, rec_bytes;
  int64_t tile_stride, row_tiles, col_tiles;
};

// Column splits per row-tile pair.  Items (pair, column range) are dealt
// round-robin to the persistent clusters, so the slowest cluster runs
// ceil(items / clusters) of them; each item also restarts the pipeline (about
// one tile).  Pick the split count that minimises that critical path: at
// N = 1e5 one item per pair leaves the last wave 28 % full.  Depends only on
// the operator's full shape, so every row shard reduces in the same order.
int splits_for(int64_t pairs, int64_t col_tiles, int clusters) {
  auto cost = [&](int64_t s) {  // < 0: this s yields the same split as a smaller one
    const int64_t tps = (col_tiles + s - 1) / s;
    if ((col_tiles + tps - 1) / tps != s) return -1.0;
    return (double)((pairs * s + clusters - 1) / clusters) * (double)(tps + 1);
  };
  const int64_t smax = std::min<int64_t>(col_tiles, 64);
  double best = 1e300;
  for (int64_t s = 1; s <= smax; ++s) {
    const double c = cost(s);
    if (c >= 0 && c < best) best = c;
  }
  // the fewest splits within 1 % of the best (fewer partial rows to reduce)
  for (int64_t s = 1; s <= smax; ++s) {
    const double c = cost(s);
    if (c >= 0 && c <= best * 1.01) return (int)s;
  }
  return 1;
}

// Symmetric kernel work list: row-tile pair a covers column tiles [2a, nb)
// (the diagonal 256 x 256 block plus everything right of it); the transposed
// products of tiles c >= 2a + 2 cover the blocks left of the diagonal.  The
// columns are cut into global blocks of SYM_ITEM tiles, and the list is
// block-major: (block 0: pairs 0, 1, ...), (block 1: ...), ...  The clusters
// running at the same time then share one block's column records and the
// fp32 accumulator rows its transposed products reduce into, both L2-sized
// (at N = 1e6 a pair-major list streamed all 192 MB of records and 128 MB of
// accumulator rows through L2 at once).
// (The item length is a creation-time knob, NCGP_SYM_ITEM, default 128; the
// workspace's item table is sized for the shortest allowed length, 16, and
// longer items only shorten the list.)
constexpr int SYM_ITEM_MIN = 16;
template <typename F>
void sym_walk(int64_t pairs, int64_t nb, F&& f, int item = SYM_ITEM_MIN, bool pair_order = false) {
  const int64_t L = std::max(item, SYM_ITEM_MIN);
  if (pair_order) {  // NCGP_SYM_ORDER=pair: the pair-major list (experiments)
    for (int64_t a = 0; a < pairs; ++a)
      for (int64_t c0 = 2 * a; c0 < nb; c0 += L) f(a, c0, std::min<int64_t>(nb, c0 + L));
    return;
  }
  for (int64_t b0 = 0; b0 < nb; b0 += L) {
    const int64_t b1 = std::min<int64_t>(nb, b0 + L);
    for (int64_t a = 0; a < pairs && 2 * a < b1; ++a) f(a, std::max<int64_t>(b0, 2 * a), b1);
  }
}
int64_t sym_item_count(int64_t pairs, int64_t nb) {
  int64_t n = 0;
  sym_walk(pairs, nb, [&](int64_t, int64_t, int64_t) { ++n; });
  return n;
}
std::vector<int4> sym_items(int64_t pairs, int64_t nb, int item, bool pair_order) {
  std::vector<int4> t;
  t.reserve((size_t)sym_item_count(pairs, nb));
  sym_walk(pairs, nb, [&](int64_t a, int64_t c0, int64_t c1) {
    t.push_back(make_int4((int)a, (int)c0, (int)c1, 0));
  }, item, pair_order);
  return t;
}

// Single-CTA symmetric kernel (K1-sym1): row tile r covers column tiles
// [r, nb); same block-major order.
constexpr size_t SMEM_MAX = 232448;  // sm_100 opt-in maximum per block
size_t smem1_bytes(uint32_t a_bytes, int wp, int sx, int sv, int npb = 2);
size_t smem2_bytes(uint32_t a_bytes, int wp, int sx, int sv, int nblk);
// Flavour of the symmetric kernel an operator's work list is built for: the
// single-CTA kernel where its shared memory fits the widest RHS (full column
// records plus two P buffers), else the pair kernel.  NCGP_SYM_CG=1 / 2 forces.
int sym_cg(const ncgp_kop* op, int d, int w_max) {
  if (op->knob_sym_cg >= 1 && op->knob_sym_cg <= 3) return op->knob_sym_cg;
  const uint32_t a = (uint32_t)(BM * ka_of(d) * 2);
  // the blocked kernel (K1-sym2, flavour 3) for RBF at WP = 32 wherever its
  // rings fit (one B200: cfg3 283 ms against K1-sym1's 328; K1-sym1 stays ahead
  // at WP = 16 -- n = 2e5 RBF w = 10: 8.7 against 9.3 ms -- and for Matern-3/2,
  // whose two MUFU ops per pair outweigh the shared-memory savings: cfg3-matern
  // 372 against 389 ms; tools/flavours.py)
  if (op->family == NCGP_RBF && wp_of(w_max) == 32 && smem2_bytes(a, 32, 2, 2, 0) <= SMEM_MAX) return 3;
  // rings no shallower than (XB 2, V 4) or (XB 3, V 2): D = 24 at WP = 16
  // only fits (2, 3), which ran slower than the plain kernel; the pair kernel
  // keeps 3-deep rings there
  const int wpm = wp_of(w_max);
  if (smem1_bytes(a, wpm, 2, 4, 2) <= SMEM_MAX || smem1_bytes(a, wpm, 3, 2, 2) <= SMEM_MAX) return 1;
  // Matern-3/2 at WP = 32 beyond D = 8 (tools/flavours.py, one B200, n = 1e5 / 4e5):
  // the blocked kernel where its rings fit (D <= ~12: 4.05 / 63.8 ms against
  // K1-sym1's 4.39 / 70.4 and the pair kernel's 5.15 / 80.0), then K1-sym1 on
  // its shallowest rings with one P buffer (D = 20: 4.42 / 71.0 against 5.16 / 82.0;
  // D = 32: 5.02 / 81.7 against 5.18 / 84.7) -- the epilogue's two MUFU ops
  // per pair hide the shallower rings
  if (op->family == NCGP_MATERN32 && wpm == 32) {
    if (smem2_bytes(a, 32, 2, 2, 0) <= SMEM_MAX) return 3;
    if (smem1_bytes(a, 32, 2, 2, 1) <= SMEM_MAX) return 1;  // one P buffer from D ~ 12 up
  }
  // experiments (NCGP_SYM1_NPB=1): one-P-buffer single-CTA kernel
  if (op->knob_npb1 && smem1_bytes(a, wp_of(w_max), 2, 2, 1) <= SMEM_MAX) return 1;
  return 2;
}
template <typename F>
void sym1_walk(int64_t nb, F&& f, int item = SYM_ITEM_MIN) {
  const int64_t L = std::max(item, SYM_ITEM_MIN);
  for (int64_t b0 = 0; b0 < nb; b0 += L) {
    const int64_t b1 = std::min<int64_t>(nb, b0 + L);
    for (int64_t r = 0; r < b1; ++r) f(r, std::max<int64_t>(b0, r), b1);
  }
}
int64_t sym1_item_count(int64_t nb) {
  int64_t n = 0;
  sym1_walk(nb, [&](int64_t, int64_t, int64_t) { ++n; });
  return n;
}
// K1-sym2 work list: row blocks of RB tiles, block b covering column tiles
// [RB b, nb); the columns cut at global blocks of L tiles (L a multiple of
// RB, so every row of an item's block meets the item's last column), and the
// list block-major like the other flavours.
template <typename F>
void sym2_walk(int64_t nb, F&& f, int item = SYM_ITEM_MIN) {
  const int64_t L = (std::max(item, SYM_ITEM_MIN) + RB - 1) / RB * RB;
  const int64_t nrb = (nb + RB - 1) / RB;
  for (int64_t b0 = 0; b0 < nb; b0 += L) {
    const int64_t b1 = std::min<int64_t>(nb, b0 + L);
    for (int64_t b = 0; b < nrb && RB * b < b1; ++b) f(b, std::max<int64_t>(b0, RB * b), b1);
  }
}
// tiles of a K1-sym2 item: per column tile c, the block's rows r <= c
int64_t sym2_item_tiles(int64_t b, int64_t c0, int64_t c1, int64_t nb) {
  const int64_t rlo = RB * b, rend = std::min<int64_t>(rlo + RB, nb);
  int64_t t = 0;
  for (int64_t c = c0; c < c1; ++c) t += std::min<int64_t>(rend, c + 1) - rlo;
  return t;
}
size_t smem2_bytes(uint32_t a_bytes, int wp, int sx, int sv, int nblk) {
  const size_t vb = (size_t)wp * BN * 4, v8 = (size_t)wp * BN;
  return (size_t)sx * a_bytes + (size_t)sv * (vb + v8) + 2 * (size_t)a_bytes + 2 * (vb + v8) +
         2 * (size_t)P2BUF + (size_t)4 * nblk * 2048 + (4 + 4 + 2 * 6 + 5 * NR2 + 2 * RB) * sizeof(uint64_t) +
         16 + 1024;
}
size_t smem1_bytes(uint32_t a_bytes, int wp, int sx, int sv, int npb) {
  const size_t v2 = (size_t)wp * BN * 2;
  return (size_t)a_bytes + (size_t)sx * a_bytes + (size_t)sv * 2 * v2 + 2 * v2 + npb * (size_t)PBUF +
         (size_t)BM * wp * 4 + (6 + 9 + 4 + 4 * NR + 10) * sizeof(uint64_t) + 16 + 1024;
}

Layout layout_of(int64_t n_rows, int64_t n_cols, int d, int w_max, int sms) {
  Layout L{};
  const int ka = ka_of(d);
  const int wpm = wp_of(w_max);
  L.a_bytes = (uint32_t)(BM * ka * 2);
  L.xbh_bytes = L.a_bytes / 2;
  const uint32_t v2 = (uint32_t)(wpm * BN * 2), v3 = v2 / 2;
  L.rec_bytes = L.xbh_bytes + v2 + v3;
  L.row_tiles = ((n_rows + BM - 1) / BM + 1) / 2 * 2;  // whole pairs
  L.col_tiles = (n_cols + BN - 1) / BN;
  L.tile_stride = 2 * (int64_t)L.rec_bytes;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = ncgp::align_up(off + bytes, 256);
    return o;
  };
  L.mu = take(64 * sizeof(double));
  L.guard = take(16);
  L.colexp = take(WIDE_WP * sizeof(int));
  L.bits = take(WIDE_WP * sizeof(unsigned));
  L.xa = take((size_t)L.row_tiles * L.a_bytes);
  // square operators get one zero record past the last column tile: the
  // symmetric kernel reads the padding row tile's V block from it
  L.col = take((size_t)(L.col_tiles + (n_rows == n_cols ? 1 : 0)) * L.tile_stride);
  // fp64 partial rows [splits][rows][w] when a pair's columns are split; the
  // wide kernel's fp32 partials [splits][WIDE_ROWS][128] share the region
  const int sp = splits_for(L.row_tiles / 2, L.col_tiles, std::max(1, sms / 2));
  size_t part = (size_t)(sp > 1 ? sp : 0) * (size_t)(L.row_tiles * BM) * std::min(w_max, 32) *
                sizeof(double);
  if (wpm == WIDE_WP) {
    const int64_t spw = (L.col_tiles + WIDE_ITEM - 1) / WIDE_ITEM;
    const size_t wide = (size_t)spw * std::min<int64_t>(WIDE_ROWS, L.row_tiles * BM) * WIDE_WP *
                        sizeof(float);
    part = std::max(part, wide);
    // posterior variance: fp64 sum of squares per (row, output) (ncgp_kop_posterior_var)
    L.varacc = take((size_t)L.row_tiles * BM * 64 * sizeof(double));
  }
  L.partial = take(part + 256);
  // symmetric kernel (square operators): int64 accumulator and item table
  const bool sq = n_rows == n_cols;
  L.symacc = take(sq ? (size_t)L.row_tiles * BM * std::min(wpm, 32) * sizeof(unsigned long long) : 0);
  L.symtab = take(sq ? (size_t)std::max(sym_item_count(L.row_tiles / 2, L.col_tiles),
                                         sym1_item_count(L.col_tiles)) * 16
                     : 0);
  // blocked symmetric kernel: Vhi in E4M3 per column tile (WP x 128 bytes)
  L.v8 = take(sq && wpm <= 32 ? (size_t)(L.col_tiles + 1) * wpm * BN : 0);
  L.total = off;
  return L;
}

// the wide kernel (WP = 128): no fp64 accumulator rows in shared memory
size_t smem_wide(uint32_t a_bytes, int sx, int sv) {
  const size_t v2 = (size_t)WIDE_WP * BN * 2;  // a CTA's [B3 | B4] V slot
  return (size_t)a_bytes + (size_t)sx * (a_bytes / 2) + (size_t)sv * v2 +
         (6 + 9 + 2 + NS_MAX + 5 * NR + 8 + 12) * sizeof(uint64_t) + 16 + 1024;
}

size_t smem_bytes(uint32_t a_bytes, int wp, int na, int sx, int sv, int sym_npb = 0) {
  const size_t v2 = (size_t)wp * BN * 2, v3 = v2 / 2;
  // NCGP_PAIR_F8 (symmetric pair kernel): [P_hi | P_lo8] buffers, Vhi8 halves
  // behind the V slots and a full Vhi8 block behind the own V block
  const bool f8 = NCGP_PAIR_F8 && sym_npb > 0;
  const size_t v8 = (size_t)wp * BN;
  return (size_t)na * a_bytes + (size_t)sx * (a_bytes / 2) + (size_t)sv * (v2 + v3 + (f8 ? v8 / 2 : 0)) +
         (sym_npb ? 2 * v2 + (f8 ? v8 : 0) + sym_npb * (size_t)(f8 ? P2BUF : PBUF) + (size_t)BM * wp * 4
                  : (size_t)wp * BM * 8) +
         (6 + 9 + 2 + NS_MAX + 5 * NR + 8 + 12 + (f8 ? 8 : 0)) * sizeof(uint64_t) + 16 + 1024;
}

// The pair kernel with its row tile in TMEM (large D, WP = 16).  NCGP_SYM_ATM=0
// disables it.
bool atm_allowed(const ncgp_kop* op) { return op->knob_atm; }

// Which symmetric kernel a full-range apply of width w runs: 0 none (the
// plain kernel), 1 the pair kernel, 2 the single-CTA kernel.
int sym_variant(const ncgp_kop* op, int w) {
  if (op->sym_items <= 0 || g_debug_mode != 0) return 0;
  const int wp = wp_of(w);
  if (wp > 32) return 0;
  if (!sym_enabled(op, op->family, wp, op->col_tiles, op->sym_cg)) return 0;
  const uint32_t a_bytes = (uint32_t)(BM * op->ka * 2);
  if (op->sym_cg == 1) return smem1_bytes(a_bytes, wp, 2, 2, 1) <= SMEM_MAX ? 2 : 0;
  if (op->sym_cg == 3) return smem2_bytes(a_bytes, wp, 2, 2, 0) <= SMEM_MAX ? 4 : 0;
  if (smem_bytes(a_bytes, wp, 1, 3, 3, 2) <= (size_t)SMEM_BUDGET) return 1;
  if (wp == 16 && atm_allowed(op) && op->ka <= 2 * 128 &&
      smem_bytes(a_bytes, wp, 0, 3, 3, 2) <= (size_t)SMEM_BUDGET)
    return 1;
  if (op->family == NCGP_MATERN32 && smem_bytes(a_bytes, wp, 1, 3, 3, 1) <= (size_t)SMEM_BUDGET) return 1;
  if (op->knob_npb == 1 && smem_bytes(a_bytes, wp, 1, 3, 3, 1) <= (size_t)SMEM_BUDGET) return 1;
  return 0;
}

}  // namespace

namespace ncgp {

struct VarPass {
  int g0, R, C;
  double* sq;  // [n_rows][C] fp64 sums of squares
};
int tc_wide(ncgp_kop* op, const void* V, int64_t ldv, int w, const OutSet* out, int64_t ldo,
            int64_t r0, int64_t r1, cudaStream_t st, const VarPass* var);
int tc_posterior_var(ncgp_kop* op, const void* W, int64_t ldw, int C, int R, const double* s2,
                     void* var, int64_t ldvar, cudaStream_t st) {
  NCGP_CHECK_ARG(C >= 1 && C <= 64 && R >= 1, NCGP_DIMENSION_MISMATCH, "C = %d, R = %d", C, R);
  NCGP_CHECK_ARG(ldw >= (int64_t)C * R && ldvar >= C, NCGP_DIMENSION_MISMATCH, "leading dimension");
  const Layout L = layout_of(op->n_rows, op->n_cols, op->d, op->w_max, op->sms);
  double* sq = reinterpret_cast<double*>(op->ws + L.varacc);
  NCGP_CUDA(cudaMemsetAsync(sq, 0, (size_t)op->n_rows * C * sizeof(double), st));
  const int total = C * R;
  for (int g0 = 0; g0 < total; g0 += WIDE_WP) {
    const int w = std::min(WIDE_WP, total - g0);
    const VarPass vp{g0, R, C, sq};
    const int rc = tc_wide(op, static_cast<const float*>(W) + g0, ldw, w, nullptr, 0, 0,
                           op->n_rows, st, &vp);
    if (rc != NCGP_OK) return rc;
  }
  const int64_t tot = op->n_rows * C;
  var_finalize_kernel<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
      sq, op->n_rows, C, s2, static_cast<float*>(var), ldvar);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

int64_t tc_sym_acc_elems(const ncgp_kop* op, int w) {
  return sym_variant(op, w) ? op->row_tiles * BM * wp_of(w) : 0;
}

int tc_sym_finalize(ncgp_kop* op, const unsigned long long* acc, int w, const OutSet& out,
                    int64_t ldo, cudaStream_t st, const EpiDev& epi, int64_t row_begin,
                    int64_t row_end) {
  if (row_end < 0) row_end = op->n_rows;
  if (row_end <= row_begin) return NCGP_OK;
  const Layout L = layout_of(op->n_rows, op->n_cols, op->d, op->w_max, op->sms);
  const int* col_exp = reinterpret_cast<const int*>(op->ws + L.colexp);
  const int s_exp = (int)lround(log2(op->k_scale));
  sym_finalize_kernel<<<(unsigned)((row_end - row_begin + 127) / 128), 128, 0, st>>>(
      acc, op->row_tiles * BM, row_begin, row_end, w, op->sym_fx, s_exp, col_exp, epi,
      ncgp::out_ptrs<float>(out, 0, ldo), ldo,
      (op->sym_cg == 3 || (op->sym_cg == 1 && NCGP_SYM1_RED) || (op->sym_cg == 2 && NCGP_PAIR_RED)) ? 1 : 0);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

bool tc_supported(int dtype, int d, int w_max) {
  if (dtype != NCGP_F32) return false;
  if (d < 1 || d > 64 || w_max < 1 || w_max > WIDE_WP) return false;
  const uint32_t a = (uint32_t)(BM * ka_of(d) * 2);
  if (smem_bytes(a, wp_of(std::min(w_max, 32)), 1, 3, 6) > (size_t)SMEM_BUDGET) return false;
  // wide RHS (w_max > 32): the WP = 128 kernel with (XB 2, V 3) rings, D <= ~50
  return w_max <= 32 || smem_wide(a, 3, 3) <= SMEM_MAX;
}

// The wide kernel over rows [r0, r1) in blocks of WIDE_ROWS: products with
// 32 < w <= 128 (out != nullptr) or, with `var`, one 128-column pass of K2's
// square-reduce (posterior variance).
int tc_wide(ncgp_kop* op, const void* V, int64_t ldv, int w, const OutSet* out, int64_t ldo,
            int64_t r0, int64_t r1, cudaStream_t st, const VarPass* var) {
  NCGP_CHECK_ARG(op->w_max > 32, NCGP_UNSUPPORTED,
                 "w = %d needs an operator created with w_max > 32 (the wide kernel)", w);
  NCGP_CHECK_ARG(w >= 1 && w <= WIDE_WP, NCGP_DIMENSION_MISMATCH, "wide width %d", w);
  NCGP_CHECK_ARG(r0 % (2 * BM) == 0, NCGP_DIMENSION_MISMATCH,
                 "row_begin must be a multiple of %d for the tcgen05 operator", 2 * BM);
  const Layout L = layout_of(op->n_rows, op->n_cols, op->d, op->w_max, op->sms);
  int* col_exp = reinterpret_cast<int*>(op->ws + L.colexp);
  unsigned int* bits = reinterpret_cast<unsigned int*>(op->ws + L.bits);
  const float* Vf = static_cast<const float*>(V);
  const int wp = WIDE_WP;
  NCGP_CUDA(cudaMemsetAsync(bits, 0, WIDE_WP * sizeof(unsigned), st));
  {
    dim3 grid((unsigned)std::min<int64_t>(1024, (op->n_cols + 7) / 8), (unsigned)((w + 31) / 32));
    col_absmax_kernel<float><<<grid, 256, 0, st>>>(Vf, ldv, op->n_cols, w, bits);
    NCGP_LAUNCHED();
    col_exp_kernel<<<1, WIDE_WP, 0, st>>>(bits, w, wp, col_exp);
    NCGP_LAUNCHED();
  }
  const uint32_t v2 = (uint32_t)(wp * BN * 2);
  {
    const int64_t tot = op->col_tiles * (BN / 8) * wp;
    pack_v_kernel<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        Vf, ldv, op->n_cols, w, wp, col_exp, op->col_pack, L.tile_stride, L.rec_bytes,
        L.xbh_bytes, v2, op->col_tiles, 1);
    NCGP_LAUNCHED();
  }
  TcParams p{};
  p.xa_pack = op->xa_pack;
  p.col_pack = op->col_pack;
  p.tile_stride = L.tile_stride;
  p.rec_bytes = L.rec_bytes;
  p.a_bytes = L.a_bytes;
  p.xbh_bytes = L.xbh_bytes;
  p.v2_bytes = v2;
  p.v3_bytes = v2 / 2;
  p.ka = op->ka;
  p.w = w;
  p.col_tiles = op->col_tiles;
  // items of <= WIDE_ITEM column tiles: each accumulates in fp32 TMEM over
  // at most 2048 columns (K1's chunk); the splits are summed in fp64 in a
  // fixed order
  p.splits = (int)((op->col_tiles + WIDE_ITEM - 1) / WIDE_ITEM);
  p.tiles_per_split = (p.col_tiles + p.splits - 1) / p.splits;
  p.splits = (int)((p.col_tiles + p.tiles_per_split - 1) / p.tiles_per_split);
  const int s_exp = (int)lround(log2(op->k_scale));
  p.s_exp = s_exp;
  p.L = (float)(log2(op->s2) + s_exp);
  p.col_exp = col_exp;
  p.out_f64 = 0;
  p.n_out = 0;
  p.ldo = ldo;
  p.partial = op->partial;
  p.na = 1;
  p.sx = 3;
  p.sv = smem_wide(p.a_bytes, 3, 4) <= SMEM_MAX ? 4 : 3;
  p.epi.alpha = 1.0;
  const size_t smem = smem_wide(p.a_bytes, p.sx, p.sv);
  NCGP_CHECK_ARG(smem <= SMEM_MAX, NCGP_UNSUPPORTED, "wide kernel: shared memory for d=%d", op->d);
  const int clusters = std::max(1, op->sms / 2);
  auto kern = op->family == NCGP_RBF ? kop_tc_kernel<NCGP_RBF, WIDE_WP, false, false>
                                     : kop_tc_kernel<NCGP_MATERN32, WIDE_WP, false, false>;
  NCGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  op->last_variant = 3;
  const float* part = reinterpret_cast<const float*>(op->partial);
  for (int64_t rb = r0; rb < r1; rb += WIDE_ROWS) {
    const int64_t re = std::min(r1, rb + WIDE_ROWS);
    p.rt0 = rb / BM;
    p.nloc = re - rb;
    p.pairs = (p.nloc + 2 * BM - 1) / (2 * BM);
    p.n_items = (int)(p.pairs * p.splits);
    const unsigned grid = 2u * (unsigned)std::min<int64_t>(p.n_items, clusters);
    kern<<<grid, NTHREADS, smem, st>>>(p);
    NCGP_LAUNCHED();
    if (var != nullptr) {
      wide_sqsum_kernel<<<(unsigned)p.nloc, 128, 0, st>>>(part, p.splits, p.nloc, w, s_exp, col_exp,
                                                          var->g0, var->R, var->C,
                                                          var->sq + rb * var->C);
    } else {
      const int64_t tot = p.nloc * w;
      wide_reduce_kernel<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
          part, p.splits, p.nloc, w, s_exp, col_exp, ncgp::out_ptrs<float>(*out, rb, ldo), ldo);
    }
    NCGP_LAUNCHED();
  }
  return NCGP_OK;
}

size_t tc_workspace_bytes(int64_t n_rows, int64_t n_cols, int d, int w_max) {
  return layout_of(n_rows, n_cols, d, w_max, sm_count()).total;
}

int tc_prepare(ncgp_kop* op, cudaStream_t st) {
  const Layout L = layout_of(op->n_rows, op->n_cols, op->d, op->w_max, op->sms);
  NCGP_CHECK_ARG(op->ws_bytes >= L.total, NCGP_INVALID_INPUT, "tcgen05 workspace too small");
  op->ka = ka_of(op->d);
  op->wpad = wp_of(op->w_max);
  op->row_tiles = L.row_tiles;
  op->col_tiles = L.col_tiles;
  op->xa_pack = op->ws + L.xa;
  op->col_pack = op->ws + L.col;
  op->col_tile_bytes = (size_t)L.tile_stride;
  op->partial = reinterpret_cast<double*>(op->ws + L.partial);
  op->sym_items = 0;
  op->sym_acc = reinterpret_cast<unsigned long long*>(op->ws + L.symacc);
  // fixed-point fraction bits of the symmetric accumulator (fx_round):
  // flushes below 2^42, |sum| < n 2^28 2^F < 2^62
  op->sym_fx = std::min(3, 33 - (int)ceil(log2((double)std::max<int64_t>(op->n_cols, 2))));
  op->sym_tab = reinterpret_cast<int4*>(op->ws + L.symtab);
  op->v8_pack = op->ws + L.v8;
  std::vector<int4> tab;
  if (op->n_rows == op->n_cols)
    NCGP_CUDA(cudaMemsetAsync(op->col_pack + (size_t)L.col_tiles * L.tile_stride, 0,
                              (size_t)L.tile_stride, st));
  if (op->Xr == op->Xc && op->n_rows == op->n_cols) {
    op->sym_cg = sym_cg(op, op->d, op->w_max);
    // Column tiles per work item of K1-sym1 / the pair kernel.  Long items
    // flush O less often; short ones balance the triangular list over the CTAs
    // (each CTA walks items round-robin, so the slowest one runs
    // ceil(items / CTAs) of them).  128 from ~64-128 rounds per CTA up, halved
    // down to 16 below that (tools/item_sweep.py: pair kernel, Matern D = 20
    // w = 10: n = 1e5 3.43 -> 3.28 ms, n = 1.5e5 7.67 -> 7.25 ms with 16;
    // K1-sym1 n = 45k 0.96 -> 0.81 ms; from n = 2e5 up 64 / 128 are ahead).
    // The length depends on the operator alone, never on how many processes
    // split the list: the N-GPU product stays bitwise the one-GPU product.
    auto auto_item = [&](double tiles, double rounds) {
      int it = 128;
      while (it > SYM_ITEM_MIN && tiles / ((double)op->sms * it) < rounds) it >>= 1;
      return it;
    };
    const double nbt = (double)L.col_tiles;
    // K1-sym1 restarts an item cheaply: ~128 rounds (n = 1e5: 16 tiles, 3.19 against
    // 3.36 ms with 128); the pair kernel reloads its row tile into TMEM per item: ~64
    const int item1 = op->knob_item > 0 ? op->knob_item : auto_item(0.5 * nbt * nbt, 128.0);
    const int itemp = op->knob_item > 0 ? op->knob_item : auto_item(0.25 * nbt * nbt, 64.0);  // 256-row pairs
    if (op->sym_cg == 1)
      sym1_walk(L.col_tiles, [&](int64_t r, int64_t c0, int64_t c1) {
        tab.push_back(make_int4((int)r, (int)c0, (int)c1, 0));
      }, item1);
    else if (op->sym_cg == 3)  // items of 16 column tiles: O is flushed every 2048 columns
      sym2_walk(L.col_tiles, [&](int64_t b, int64_t c0, int64_t c1) {
        tab.push_back(make_int4((int)b, (int)c0, (int)c1, 0));
      }, op->knob_item2);
    else
      tab = sym_items(L.row_tiles / 2, L.col_tiles, itemp, op->knob_pair_order);
    NCGP_CUDA(cudaMemcpyAsync(op->sym_tab, tab.data(), tab.size() * sizeof(int4),
                              cudaMemcpyHostToDevice, st));
    op->sym_items = (int64_t)tab.size();  // the stream sync below keeps `tab` alive long enough
    op->sym_cum.assign(tab.size() + 1, 0);
    for (size_t k = 0; k < tab.size(); ++k)
      op->sym_cum[k + 1] = op->sym_cum[k] + (op->sym_cg == 3 ? sym2_item_tiles(tab[k].x, tab[k].y, tab[k].z, L.col_tiles)
                                                               : (int64_t)(tab[k].z - tab[k].y));
  }
  // prescale kernel values into fp16 range: s2 * 2^s in (2^13, 2^14]
  const int s_exp = 14 - (int)ceil(log2(op->s2));
  op->k_scale = ldexp(1.0, s_exp);
  const double log2e = 1.4426950408889634;
  double alpha, sign, Lc;
  if (op->family == NCGP_RBF) {
    alpha = sqrt(log2e / (2.0 * op->ell * op->ell));  // -|x~|^2 = -d^2 log2e / (2 l^2)
    sign = 1.0;
    Lc = log2(op->s2) + s_exp;
  } else {
    alpha = sqrt(3.0) / op->ell;                     // |x~| = sqrt(3) d / l
    sign = -1.0;
    Lc = 0.0;
  }
  double* mu = reinterpret_cast<double*>(op->ws + L.mu);
  const float* Xr = static_cast<const float*>(op->Xr);
  const float* Xc = static_cast<const float*>(op->Xc);
  col_mean_kernel<float><<<1, 1024, 0, st>>>(Xc, op->n_cols, op->d, mu);
  NCGP_LAUNCHED();
  const int qn = op->ka / 8;
  {
    const int64_t tot = L.row_tiles * BM * qn;
    pack_x_kernel<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        Xr, op->n_rows, op->d, op->ka, mu, alpha, sign, Lc, 0, op->xa_pack, L.a_bytes, 0,
        L.row_tiles);
    NCGP_LAUNCHED();
  }
  {
    const int64_t tot = L.col_tiles * BN * qn;
    pack_x_kernel<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        Xc, op->n_cols, op->d, op->ka, mu, alpha, sign, Lc, 1, op->col_pack, L.tile_stride,
        L.rec_bytes, L.col_tiles);
    NCGP_LAUNCHED();
  }
  // precision guard: the expanded distance loses ~2^-22 |x~|^2 absolute
  unsigned int* gbits = reinterpret_cast<unsigned int*>(op->ws + L.guard);
  NCGP_CUDA(cudaMemsetAsync(gbits, 0, 8, st));
  max_norm_kernel<float><<<(unsigned)((op->n_rows + 255) / 256), 256, 0, st>>>(
      Xr, op->n_rows, op->d, mu, alpha, gbits);
  NCGP_LAUNCHED();
  max_norm_kernel<float><<<(unsigned)((op->n_cols + 255) / 256), 256, 0, st>>>(
      Xc, op->n_cols, op->d, mu, alpha, gbits);
  NCGP_LAUNCHED();
  unsigned int hb = 0;
  NCGP_CUDA(cudaMemcpyAsync(&hb, gbits, 4, cudaMemcpyDeviceToHost, st));
  NCGP_CUDA(cudaStreamSynchronize(st));
  float mx;
  memcpy(&mx, &hb, 4);
  NCGP_CHECK_ARG(mx <= 256.f, NCGP_UNSUPPORTED,
                 "inputs span %.3g squared (scaled) lengthscales from their mean: beyond the "
                 "tcgen05 operator's precision range, use the CUDA-core operator",
                 (double)mx);
  return NCGP_OK;
}

int tc_apply(ncgp_kop* op, const void* V, int64_t ldv, int w, const OutSet& out, int64_t ldo,
             int64_t r0, int64_t r1, cudaStream_t st, const EpiDev& epi, const SymPart* part) {
  if (wp_of(w) == WIDE_WP) {
    NCGP_CHECK_ARG(part == nullptr, NCGP_UNSUPPORTED, "no symmetric kernel for w = %d", w);
    NCGP_CHECK_ARG(!epi.active, NCGP_UNSUPPORTED, "fused epilogues need w <= 32 (got %d)", w);
    return tc_wide(op, V, ldv, w, &out, ldo, r0, r1, st, nullptr);
  }
  if (part != nullptr) {
    NCGP_CHECK_ARG(sym_variant(op, w) != 0, NCGP_UNSUPPORTED,
                   "no symmetric kernel for this operator and width");
    NCGP_CHECK_ARG(part->nparts >= 1 && part->part >= 0 && part->part < part->nparts,
                   NCGP_INVALID_INPUT, "bad part %d of %d", part->part, part->nparts);
    r0 = 0;
    r1 = op->n_rows;
  }
  NCGP_CHECK_ARG(r0 % (2 * BM) == 0, NCGP_DIMENSION_MISMATCH,
                 "row_begin must be a multiple of %d for the tcgen05 operator", 2 * BM);
  const Layout L = layout_of(op->n_rows, op->n_cols, op->d, op->w_max, op->sms);
  const int wp = wp_of(w);
  int* col_exp = reinterpret_cast<int*>(op->ws + L.colexp);
  unsigned int* bits = reinterpret_cast<unsigned int*>(op->ws + L.bits);
  const float* Vf = static_cast<const float*>(V);
  NCGP_CUDA(cudaMemsetAsync(bits, 0, WIDE_WP * sizeof(unsigned), st));
  {
    dim3 grid((unsigned)std::min<int64_t>(1024, (op->n_cols + 7) / 8), (unsigned)((w + 31) / 32));
    col_absmax_kernel<float><<<grid, 256, 0, st>>>(Vf, ldv, op->n_cols, w, bits);
    NCGP_LAUNCHED();
    col_exp_kernel<<<1, WIDE_WP, 0, st>>>(bits, w, wp, col_exp);
    NCGP_LAUNCHED();
  }
  const uint32_t v2 = (uint32_t)(wp * BN * 2);
  {
    const int64_t tot = op->col_tiles * (BN / 8) * wp;
    pack_v_kernel<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        Vf, ldv, op->n_cols, w, wp, col_exp, op->col_pack, L.tile_stride, L.rec_bytes,
        L.xbh_bytes, v2, op->col_tiles);
    NCGP_LAUNCHED();
  }
  TcParams p{};
  p.xa_pack = op->xa_pack;
  p.col_pack = op->col_pack;
  p.tile_stride = L.tile_stride;
  p.rec_bytes = L.rec_bytes;
  p.a_bytes = L.a_bytes;
  p.xbh_bytes = L.xbh_bytes;
  p.v2_bytes = v2;
  p.v3_bytes = v2 / 2;
  p.ka = op->ka;
  p.w = w;
  p.rt0 = r0 / BM;
  p.nloc = r1 - r0;
  p.pairs = (p.nloc + 2 * BM - 1) / (2 * BM);
  p.col_tiles = op->col_tiles;
  // splits depend on the operator's full row count only, so every row is
  // reduced in the same order whichever row range (shard) is launched
  const int clusters = std::max(1, op->sms / 2);
  p.splits = splits_for(op->row_tiles / 2, p.col_tiles, clusters);
  p.tiles_per_split = (p.col_tiles + p.splits - 1) / p.splits;
  p.splits = (int)((p.col_tiles + p.tiles_per_split - 1) / p.tiles_per_split);
  const int s_exp = (int)lround(log2(op->k_scale));
  p.s_exp = s_exp;
  p.L = (float)(log2(op->s2) + s_exp);  // RBF clamp / Matern exponent offset
  p.col_exp = col_exp;
  p.out_f64 = op->dtype == NCGP_F64;
  p.n_out = out.n;
  for (int k = 0; k < out.n; ++k)
    p.outs[k] = static_cast<uint8_t*>(out.p[k]) + r0 * ldo * (p.out_f64 ? 8 : 4);
  p.ldo = ldo;
  p.partial = op->partial;
  p.trace = g_trace;
  p.debug_mode = g_debug_mode;
  p.n_items = (int)(p.pairs * p.splits);
  p.item_tab = nullptr;
  p.acc = nullptr;
  p.acc_rows = op->row_tiles * BM;
  p.fx = ldexpf(1.f, op->sym_fx);
  p.fxi = ldexpf(1.f, 21 - op->sym_fx);
  p.epi = epi;
  // symmetric kernel: K(X, X) with the whole row range in one launch
  const bool dbg = (g_trace != nullptr) || (g_debug_mode != 0);
  bool sym = r0 == 0 && r1 == op->n_rows && sym_variant(op, w) != 0;
  // items of this launch: all, or part `part` of `nparts` slices of equal
  // tile count (contiguous in the block-major list)
  int64_t it_lo = 0, it_hi = op->sym_items;
  if (part != nullptr) {
    const int64_t tot = op->sym_cum.back();
    auto cut = [&](int k) {
      const int64_t target = tot * k / part->nparts;
      return (int64_t)(std::lower_bound(op->sym_cum.begin(), op->sym_cum.end(), target) -
                       op->sym_cum.begin());
    };
    it_lo = std::min<int64_t>(cut(part->part), op->sym_items);
    it_hi = std::min<int64_t>(cut(part->part + 1), op->sym_items);
  }
  unsigned long long* const sym_acc = part != nullptr ? part->acc : op->sym_acc;
  const size_t acc_bytes = (size_t)op->row_tiles * BM * wp * sizeof(unsigned long long);
  // variant bits always; the result-changing debug bits only with a debug hook set
  const int sym_dbg = op->knob_sym_var | (dbg ? [] {
    const char* e = getenv("NCGP_SYM_DBG");
    return e != nullptr ? atoi(e) : 0;
  }() : 0);
  const bool sym_fin = part == nullptr;
  if (sym && op->sym_cg == 3) {
    // deepest rings that fit: (sx, sv, staging blocks per drain warp)
    // (the drains reduce straight from registers: no staging blocks)
    const int cand[][3] = {{3, 3, 0}, {3, 2, 0}, {2, 2, 0}};
    bool fit = false;
    for (auto& c : cand)
      if (smem2_bytes(p.a_bytes, wp, c[0], c[1], c[2]) <= SMEM_MAX) {
        p.sx = c[0];
        p.sv = c[1];
        p.nblk = c[2];
        fit = true;
        break;
      }
    NCGP_CHECK_ARG(fit, NCGP_UNSUPPORTED, "blocked symmetric kernel: shared memory for d=%d", op->d);
    p.na = 1;
    p.splits = 1;
    p.tiles_per_split = p.col_tiles;
    p.n_items = (int)(it_hi - it_lo);
    p.item_tab = op->sym_tab + it_lo;
    p.acc = sym_acc;
    p.v8_pack = op->v8_pack;
    p.v8_bytes = (uint32_t)(wp * BN);
    NCGP_CUDA(cudaMemsetAsync(p.acc, 0, acc_bytes, st));
    op->last_variant = 4;
    if (p.n_items == 0) return NCGP_OK;  // an empty part
    {
      const int64_t tot = op->col_tiles * (BN / 16) * wp;
      pack_v8_kernel<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
          Vf, ldv, op->n_cols, w, wp, col_exp, op->v8_pack, op->col_tiles);
      NCGP_LAUNCHED();
    }
    const size_t smem = smem2_bytes(p.a_bytes, wp, p.sx, p.sv, p.nblk);
    const unsigned grid = (unsigned)std::min<int64_t>(p.n_items, op->sms);
    auto launch = [&](auto kern) -> int {
      NCGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<grid, NTHREADS, smem, st>>>(p);
      NCGP_LAUNCHED();
      return NCGP_OK;
    };
    p.trace = g_trace;
    int rc;
    if (op->family == NCGP_RBF)
      rc = g_trace != nullptr ? (wp == 16 ? launch(kop_sym2_kernel<NCGP_RBF, 16, true>)
                                          : launch(kop_sym2_kernel<NCGP_RBF, 32, true>))
                              : (wp == 16 ? launch(kop_sym2_kernel<NCGP_RBF, 16, false>)
                                          : launch(kop_sym2_kernel<NCGP_RBF, 32, false>));
    else
      rc = wp == 16 ? launch(kop_sym2_kernel<NCGP_MATERN32, 16, false>)
                    : launch(kop_sym2_kernel<NCGP_MATERN32, 32, false>);
    if (rc != NCGP_OK) return rc;
    return sym_fin ? tc_sym_finalize(op, p.acc, w, out, ldo, st, epi) : NCGP_OK;
  }
  if (sym && op->sym_cg == 1) {
    const int cand[][2] = {{3, 6}, {3, 4}, {3, 3}, {2, 4}, {3, 2}, {2, 3}, {2, 2}};
    bool fit = false;
    for (int npb = 2; npb >= 1 && !fit; --npb)
      for (auto& c : cand)
        if (smem1_bytes(p.a_bytes, wp, c[0], c[1], npb) <= SMEM_MAX) {
          p.sx = c[0];
          p.sv = c[1];
          p.npb = npb;
          fit = true;
          break;
        }
    if (fit) {
      p.na = 1;
      p.splits = 1;
      p.tiles_per_split = p.col_tiles;
      p.n_items = (int)(it_hi - it_lo);
      p.item_tab = op->sym_tab + it_lo;
      p.acc = sym_acc;
      p.sym_dbg = sym_dbg;
      NCGP_CUDA(cudaMemsetAsync(p.acc, 0, acc_bytes, st));
      op->last_variant = 2;
      if (p.n_items == 0) return NCGP_OK;  // an empty part
      const size_t smem = smem1_bytes(p.a_bytes, wp, p.sx, p.sv, p.npb);
      const unsigned grid = (unsigned)std::min<int64_t>(p.n_items, op->sms);
      auto launch = [&](auto kern) -> int {
        NCGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, NTHREADS, smem, st>>>(p);
        NCGP_LAUNCHED();
        return NCGP_OK;
      };
      int rc;
      if (op->family == NCGP_RBF)
        rc = dbg ? (wp == 16 ? launch(kop_sym1_kernel<NCGP_RBF, 16, true>) : launch(kop_sym1_kernel<NCGP_RBF, 32, true>))
                 : (wp == 16 ? launch(kop_sym1_kernel<NCGP_RBF, 16, false>) : launch(kop_sym1_kernel<NCGP_RBF, 32, false>));
      else
        rc = dbg ? (wp == 16 ? launch(kop_sym1_kernel<NCGP_MATERN32, 16, true>)
                             : launch(kop_sym1_kernel<NCGP_MATERN32, 32, true>))
                 : (wp == 16 ? launch(kop_sym1_kernel<NCGP_MATERN32, 16, false>)
                             : launch(kop_sym1_kernel<NCGP_MATERN32, 32, false>));
      if (rc != NCGP_OK) return rc;
      return sym_fin ? tc_sym_finalize(op, p.acc, w, out, ldo, st, epi) : NCGP_OK;
    }
    sym = false;
  }
  if (sym) {
    // two P buffers with the deepest rings that fit, else one P buffer
    // (large D: the row tile and XB ring outgrow the 227 KB)
    // (npb, na, sx, sv); na = 0: the row tile lives in TMEM (ATM, WP = 16)
    // (NCGP_PAIR_F8: three 48 KB P buffers first, where they fit)
    const int cand[][4] = {{3, 1, 3, 3}, {3, 0, 3, 3}, {3, 1, 2, 3}, {3, 0, 2, 3},
                           {2, 1, 6, 6}, {2, 1, 3, 6}, {2, 1, 3, 5}, {2, 1, 3, 4}, {2, 1, 3, 3},
                           {2, 0, 3, 6}, {2, 0, 3, 4}, {2, 0, 3, 3},
                           {1, 1, 3, 6}, {1, 1, 3, 4}, {1, 1, 3, 3}};
    const int force = op->knob_npb;  // NCGP_SYM_NPB experiments: force 1 or 2 P buffers
    sym = false;
    for (auto& c : cand)
      // one P buffer serialises the two epilogue groups on it: a 1.15x gain
      // for Matern-3/2 at D = 50 but a loss for RBF (tools/sym_exp.py)
      if ((c[0] < 3 || NCGP_PAIR_F8) &&
          (force == c[0] || (force == 0 && (c[0] >= 2 || op->family == NCGP_MATERN32))) &&
          (c[1] > 0 || (wp == 16 && atm_allowed(op))) &&
          smem_bytes(p.a_bytes, wp, c[1], c[2], c[3], c[0]) <= (size_t)SMEM_BUDGET) {
        p.npb = c[0];
        p.na = c[1];
        p.sx = c[2];
        p.sv = c[3];
        sym = true;
        break;
      }
  }
  if (sym) {
    p.splits = 1;
    p.tiles_per_split = p.col_tiles;
    p.n_items = (int)(it_hi - it_lo);
    p.item_tab = op->sym_tab + it_lo;
    p.acc = sym_acc;
    p.sym_dbg = sym_dbg;
    p.sym_dump = g_sym_dump;
    NCGP_CUDA(cudaMemsetAsync(p.acc, 0, acc_bytes, st));
    op->last_variant = 1;
    if (p.n_items == 0) return NCGP_OK;
    if (NCGP_PAIR_F8) {  // Vhi in E4M3 per column tile (the split term's B)
      p.v8_pack = op->v8_pack;
      p.v8_bytes = (uint32_t)(wp * BN);
      const int64_t tot = op->col_tiles * (BN / 16) * wp;
      pack_v8_kernel<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
          Vf, ldv, op->n_cols, w, wp, col_exp, op->v8_pack, op->col_tiles);
      NCGP_LAUNCHED();
    }
    const size_t smem = smem_bytes(p.a_bytes, wp, p.na, p.sx, p.sv, p.npb);
    const unsigned grid = 2u * (unsigned)std::min<int64_t>(p.n_items, clusters);
    auto launch = [&](auto kern) -> int {
      NCGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
      kern<<<grid, NTHREADS, smem, st>>>(p);
      NCGP_LAUNCHED();
      return NCGP_OK;
    };
    int rc;
    if (p.na == 0)  // row tile in TMEM (DBG trace: RBF only)
      rc = op->family == NCGP_RBF ? (dbg ? launch(kop_tc_kernel<NCGP_RBF, 16, true, true, true>)
                                         : launch(kop_tc_kernel<NCGP_RBF, 16, false, true, true>))
                                  : launch(kop_tc_kernel<NCGP_MATERN32, 16, false, true, true>);
    else if (dbg)  // per-tile trace of cluster 0 (tools/trace_sym.py)
      rc = op->family == NCGP_RBF
               ? (wp == 16 ? launch(kop_tc_kernel<NCGP_RBF, 16, true, true>)
                           : launch(kop_tc_kernel<NCGP_RBF, 32, true, true>))
               : (wp == 16 ? launch(kop_tc_kernel<NCGP_MATERN32, 16, true, true>)
                           : launch(kop_tc_kernel<NCGP_MATERN32, 32, true, true>));
    else if (op->family == NCGP_RBF)
      rc = wp == 16 ? launch(kop_tc_kernel<NCGP_RBF, 16, false, true>)
                    : launch(kop_tc_kernel<NCGP_RBF, 32, false, true>);
    else
      rc = wp == 16 ? launch(kop_tc_kernel<NCGP_MATERN32, 16, false, true>)
                    : launch(kop_tc_kernel<NCGP_MATERN32, 32, false, true>);
    if (rc != NCGP_OK) return rc;
    return sym_fin ? tc_sym_finalize(op, p.acc, w, out, ldo, st, epi) : NCGP_OK;
  }
  NCGP_CHECK_ARG(part == nullptr, NCGP_UNSUPPORTED, "no symmetric kernel for this operator");
  // deepest rings that fit: (na, sx, sv) from (2, 6, 9) down to (1, 3, 6)
  {
    const int cand[][3] = {{2, 6, 9}, {2, 6, 6}, {2, 3, 9}, {2, 3, 6}, {1, 6, 6}, {1, 3, 6}};
    bool ok = false;
    for (auto& c : cand)
      if (smem_bytes(p.a_bytes, wp, c[0], c[1], c[2]) <= (size_t)SMEM_BUDGET) {
        p.na = c[0];
        p.sx = c[1];
        p.sv = c[2];
        ok = true;
        break;
      }
    NCGP_CHECK_ARG(ok, NCGP_UNSUPPORTED, "shared memory too small for d=%d", op->d);
    // timing experiments: NCGP_RINGS "na,sx,sv"
    const int na = op->knob_rings[0], sx = op->knob_rings[1], sv = op->knob_rings[2];
    if (na > 0 && smem_bytes(p.a_bytes, wp, na, sx, sv) <= (size_t)SMEM_BUDGET) {
      p.na = na;
      p.sx = sx;
      p.sv = sv;
    }
  }
  NCGP_CHECK_ARG((int64_t)p.splits * p.nloc * w * 8 <= (int64_t)(L.total - L.partial) ||
                     p.splits == 1,
                 NCGP_INVALID_INPUT, "partial workspace too small");
  const size_t smem = smem_bytes(p.a_bytes, wp, p.na, p.sx, p.sv);
  const int64_t items = p.pairs * p.splits;
  op->last_variant = 0;
  const unsigned grid = 2u * (unsigned)std::min<int64_t>(items, clusters);
  auto launch = [&](auto kern) -> int {
    NCGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    kern<<<grid, NTHREADS, smem, st>>>(p);
    NCGP_LAUNCHED();
    return NCGP_OK;
  };
  int rc;
  if (op->family == NCGP_RBF) {
    if (dbg)
      rc = wp == 16 ? launch(kop_tc_kernel<NCGP_RBF, 16, true, false>)
                    : launch(kop_tc_kernel<NCGP_RBF, 32, true, false>);
    else
      rc = wp == 16 ? launch(kop_tc_kernel<NCGP_RBF, 16, false, false>)
                    : launch(kop_tc_kernel<NCGP_RBF, 32, false, false>);
  } else {
    if (dbg)
      rc = wp == 16 ? launch(kop_tc_kernel<NCGP_MATERN32, 16, true, false>)
                    : launch(kop_tc_kernel<NCGP_MATERN32, 32, true, false>);
    else
      rc = wp == 16 ? launch(kop_tc_kernel<NCGP_MATERN32, 16, false, false>)
                    : launch(kop_tc_kernel<NCGP_MATERN32, 32, false, false>);
  }
  if (rc != NCGP_OK) return rc;
  if (p.splits > 1) {
    const int64_t tot = p.nloc * w;
    const unsigned rb = (unsigned)((p.nloc + 127) / 128);
    if (epi.active && p.out_f64)
      reduce_partial_epi_kernel<double><<<rb, 128, 0, st>>>(
          p.partial, p.splits, p.nloc, w, epi, ncgp::out_ptrs<double>(out, r0, ldo), ldo);
    else if (epi.active)
      reduce_partial_epi_kernel<float><<<rb, 128, 0, st>>>(
          p.partial, p.splits, p.nloc, w, epi, ncgp::out_ptrs<float>(out, r0, ldo), ldo);
    else if (p.out_f64)
      reduce_partial_kernel<double><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
          p.partial, p.splits, p.nloc, w, ncgp::out_ptrs<double>(out, r0, ldo), ldo);
    else
      reduce_partial_kernel<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
          p.partial, p.splits, p.nloc, w, ncgp::out_ptrs<float>(out, r0, ldo), ldo);
    NCGP_LAUNCHED();
  }
  return NCGP_OK;
}

}  // namespace ncgp

// Debug / test hook (host only, no GPU): the symmetric kernels' work list for
// nb column tiles -- flavour 1 (K1-sym1: row tile, c0, c1), 2 (CTA pairs:
// row-tile pair, c0, c1) or 3 (K1-sym2: row block of 4, c0, c1) -- as int32
// triples into out (capacity cap triples); returns the item count (or -1).
// tests/test_sym_worklist.py checks that the tiles they cover are exactly the
// on-or-above-diagonal tiles, each once.
extern "C" int64_t ncgp_debug_sym_items(int flavour, int64_t nb, int item, int32_t* out, int64_t cap) {
  if (nb < 1 || item < 1) return -1;
  int64_t k = 0;
  auto put = [&](int64_t a, int64_t c0, int64_t c1) {
    if (out != nullptr && k < cap) {
      out[3 * k] = (int32_t)a;
      out[3 * k + 1] = (int32_t)c0;
      out[3 * k + 2] = (int32_t)c1;
    }
    ++k;
  };
  if (flavour == 1)
    sym1_walk(nb, put, item);
  else if (flavour == 2)
    sym_walk((nb + 1) / 2, nb, put, item);
  else if (flavour == 3)
    sym2_walk(nb, put, item);
  else
    return -1;
  return k;
}

extern "C" int ncgp_debug_set_sym_dump(void* dev_buf) {
  g_sym_dump = static_cast<float*>(dev_buf);
  return 0;
}

extern "C" int ncgp_debug_set_trace(void* dev_buf) {
  g_trace = static_cast<long long*>(dev_buf);
  return NCGP_OK;
}

extern "C" int ncgp_debug_set_mode(int mode) {
  g_debug_mode = mode;
  return NCGP_OK;
}
