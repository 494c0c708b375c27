// K6: deterministic reductions and tall-skinny products for the inner
// solver (solver.py:203-331) and the low-rank root (linalg.py:51-62).
//
// Every long reduction is two-pass with a fixed block partition and fp64
// partials summed in index order, so results are bit-reproducible for a
// given (n, SM count) and never use atomics.
#include <type_traits>

#include "common.cuh"

namespace {

constexpr int RB = 256;  // reduction block size

int64_t reduce_blocks(int64_t n, int sms) {
  int64_t g = (n + 8191) / 8192;  // >= 8192 elements per block
  const int64_t cap = (int64_t)sms * 4;
  if (g > cap) g = cap;
  return g < 1 ? 1 : g;
}

template <typename T>
__global__ void dots_partial_kernel(int64_t n, int npairs, const T* x0, const T* y0, const T* x1,
                                    const T* y1, const T* x2, const T* y2, const T* x3,
                                    const T* y3, int64_t chunk, double* __restrict__ partial) {
  __shared__ double sm[32];
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = min(n, lo + chunk);
  const T* xs[4] = {x0, x1, x2, x3};
  const T* ys[4] = {y0, y1, y2, y3};
  // one sweep for all pairs: every iteration issues the loads of all pairs
  // (independent accumulators, fixed order), then one block reduction each
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = lo + threadIdx.x; i < hi; i += RB) {
#pragma unroll
    for (int p = 0; p < 4; ++p)
      if (p < npairs) acc[p] += (double)xs[p][i] * (double)ys[p][i];
  }
  for (int p = 0; p < npairs; ++p) {
    double s = ncgp::block_sum(acc[p], sm);
    if (threadIdx.x == 0) partial[(int64_t)p * gridDim.x + blockIdx.x] = s;
  }
}

// fp32, 16-byte aligned operands: float4 loads, chunk a multiple of 4 * RB
__global__ void dots_partial_v4_kernel(int64_t n, int npairs, const float* x0, const float* y0,
                                       const float* x1, const float* y1, const float* x2,
                                       const float* y2, const float* x3, const float* y3,
                                       int64_t chunk, double* __restrict__ partial) {
  __shared__ double sm[32];
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = min(n, lo + chunk);
  const int64_t hi4 = lo + (hi - lo) / 4 * 4;
  const float* xs[4] = {x0, x1, x2, x3};
  const float* ys[4] = {y0, y1, y2, y3};
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = lo + 4 * (int64_t)threadIdx.x; i < hi4; i += 4 * RB) {
#pragma unroll
    for (int p = 0; p < 4; ++p)
      if (p < npairs) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(xs[p] + i));
        const float4 b = __ldg(reinterpret_cast<const float4*>(ys[p] + i));
        acc[p] += (double)a.x * (double)b.x + (double)a.y * (double)b.y + (double)a.z * (double)b.z +
                  (double)a.w * (double)b.w;
      }
  }
  for (int64_t i = hi4 + threadIdx.x; i < hi; i += RB) {
#pragma unroll
    for (int p = 0; p < 4; ++p)
      if (p < npairs) acc[p] += (double)xs[p][i] * (double)ys[p][i];
  }
  for (int p = 0; p < npairs; ++p) {
    const double t = ncgp::block_sum(acc[p], sm);
    if (threadIdx.x == 0) partial[(int64_t)p * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ partial, int64_t nblk, int nvec,
                                    double* __restrict__ out) {
  // one warp per output vector entry; lanes stride then a fixed-order warp tree
  const int v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (v >= nvec) return;
  double acc = 0.0;
  for (int64_t b = lane; b < nblk; b += 32) acc += partial[(int64_t)v * nblk + b];
  acc = ncgp::warp_sum(acc);
  if (lane == 0) out[v] = acc;
}

// partial[r * G + blk] = sum_{i in chunk blk} Q_r[i] z[i]
template <typename T>
__global__ void gemv_t_partial_kernel(const T* __restrict__ Q, int64_t ldq, int k,
                                      const T* __restrict__ z, int64_t n, int64_t chunk,
                                      double* __restrict__ partial) {
  __shared__ double sm[32];
  const int r = blockIdx.y;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = min(n, lo + chunk);
  const T* q = Q + (int64_t)r * ldq;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += RB) acc += (double)q[i] * (double)z[i];
  double s = ncgp::block_sum(acc, sm);
  if (threadIdx.x == 0) partial[(int64_t)r * gridDim.x + blockIdx.x] = s;
}

// fp32 with 16-byte alignment: RPB rows of Q per block share each float4 of
// z, so z is read from L2 once per RPB rows and every thread keeps RPB * 4
// independent loads in flight.  chunk is a multiple of 4 * RB.
template <int RPB>
__global__ void gemv_t_partial_v4_kernel(const float* __restrict__ Q, int64_t ldq, int k,
                                         const float* __restrict__ z, int64_t n, int64_t chunk,
                                         double* __restrict__ partial) {
  __shared__ double sm[32];
  const int r0 = blockIdx.y * RPB;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = min(n, lo + chunk);
  const int64_t hi4 = lo + (hi - lo) / 4 * 4;
  double acc[RPB];
#pragma unroll
  for (int rr = 0; rr < RPB; ++rr) acc[rr] = 0.0;
  for (int64_t i = lo + 4 * (int64_t)threadIdx.x; i < hi4; i += 4 * RB) {
    const float4 zv = __ldg(reinterpret_cast<const float4*>(z + i));
#pragma unroll
    for (int rr = 0; rr < RPB; ++rr) {
      if (r0 + rr < k) {
        const float4 qv = __ldcs(reinterpret_cast<const float4*>(Q + (int64_t)(r0 + rr) * ldq + i));
        acc[rr] += (double)qv.x * (double)zv.x + (double)qv.y * (double)zv.y +
                   (double)qv.z * (double)zv.z + (double)qv.w * (double)zv.w;
      }
    }
  }
  for (int64_t i = hi4 + threadIdx.x; i < hi; i += RB) {  // ragged tail of the last chunk
#pragma unroll
    for (int rr = 0; rr < RPB; ++rr)
      if (r0 + rr < k) acc[rr] += (double)Q[(int64_t)(r0 + rr) * ldq + i] * (double)z[i];
  }
#pragma unroll
  for (int rr = 0; rr < RPB; ++rr) {
    const double t = ncgp::block_sum(acc[rr], sm);
    if (threadIdx.x == 0 && r0 + rr < k) partial[(int64_t)(r0 + rr) * gridDim.x + blockIdx.x] = t;
  }
}

template <typename T>
__global__ void gemv_n_kernel(const T* __restrict__ Q, int64_t ldq, int k,
                              const double* __restrict__ y, const T* __restrict__ s, double alpha,
                              T* __restrict__ out, int64_t n) {
  extern __shared__ double ys[];
  for (int r = threadIdx.x; r < k; r += blockDim.x) ys[r] = y[r];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int r = 0; r < k; ++r) acc += (double)Q[(int64_t)r * ldq + i] * ys[r];
  out[i] = (T)((s ? (double)s[i] : 0.0) + alpha * acc);
}

// 4 elements per thread through 16-byte (fp32) / 2 x 16-byte (fp64) accesses
template <typename T>
__global__ void lincomb4_kernel(int64_t n4, double a, const T* __restrict__ x, double b,
                                const T* __restrict__ y, double c, const T* __restrict__ z,
                                T* __restrict__ out) {
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int PER = sizeof(T) == 4 ? 1 : 2;  // vectors per 4 elements
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n4) return;
#pragma unroll
  for (int h = 0; h < PER; ++h) {
    const int64_t o = q * PER + h;
    const V xv = reinterpret_cast<const V*>(x)[o];
    const V yv = y ? reinterpret_cast<const V*>(y)[o] : V{};
    const V zv = z ? reinterpret_cast<const V*>(z)[o] : V{};
    const T* xe = reinterpret_cast<const T*>(&xv);
    const T* ye = reinterpret_cast<const T*>(&yv);
    const T* ze = reinterpret_cast<const T*>(&zv);
    V rv;
    T* re = reinterpret_cast<T*>(&rv);
#pragma unroll
    for (int e = 0; e < (int)(sizeof(V) / sizeof(T)); ++e) {
      double r = a * (double)xe[e];
      if (y) r += b * (double)ye[e];
      if (z) r += c * (double)ze[e];
      re[e] = (T)r;
    }
    reinterpret_cast<V*>(out)[o] = rv;
  }
}

template <typename T>
__global__ void lincomb_kernel(int64_t n, double a, const T* __restrict__ x, double b,
                               const T* __restrict__ y, double c, const T* __restrict__ z,
                               T* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double r = a * (double)x[i];
  if (y) r += b * (double)y[i];
  if (z) r += c * (double)z[i];
  out[i] = (T)r;
}

// Gram partials: partial[split][a][b] = sum_{i in split} S_a[i] Y_b[i]
constexpr int GT = 32;   // output tile
constexpr int GK = 64;   // i per shared-memory step
template <typename T>
__global__ void __launch_bounds__(256)
gram_partial_kernel(const T* __restrict__ S, int64_t lds, int ka, const T* __restrict__ Y,
                    int64_t ldy, int kb, int64_t n, int64_t chunk, double* __restrict__ partial) {
  __shared__ T sa[GT][GK + 1];
  __shared__ T sb[GT][GK + 1];
  const int a0 = blockIdx.x * GT, b0 = blockIdx.y * GT;
  const int64_t lo = (int64_t)blockIdx.z * chunk;
  const int64_t hi = min(n, lo + chunk);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 2x2 outputs each
  double acc[2][2] = {{0, 0}, {0, 0}};
  for (int64_t i0 = lo; i0 < hi; i0 += GK) {
    __syncthreads();
    for (int e = threadIdx.x; e < GT * GK; e += 256) {
      const int r = e / GK, c = e % GK;
      const int64_t i = i0 + c;
      sa[r][c] = (a0 + r < ka && i < hi) ? S[(int64_t)(a0 + r) * lds + i] : T(0);
      sb[r][c] = (b0 + r < kb && i < hi) ? Y[(int64_t)(b0 + r) * ldy + i] : T(0);
    }
    __syncthreads();
    T t[2][2] = {{0, 0}, {0, 0}};
#pragma unroll 8
    for (int c = 0; c < GK; ++c) {
      const T x0 = sa[ty][c], x1 = sa[ty + 16][c];
      const T y0 = sb[tx][c], y1 = sb[tx + 16][c];
      t[0][0] += x0 * y0; t[0][1] += x0 * y1;
      t[1][0] += x1 * y0; t[1][1] += x1 * y1;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) acc[u][v] += (double)t[u][v];
  }
  double* P = partial + (int64_t)blockIdx.z * ka * kb;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int a = a0 + ty + 16 * u, b = b0 + tx + 16 * v;
      if (a < ka && b < kb) P[(int64_t)a * kb + b] = acc[u][v];
    }
}

__global__ void gram_reduce_kernel(const double* __restrict__ partial, int splits, int ka, int kb,
                                   double* __restrict__ M, int64_t ldm) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ka * kb) return;
  double s = 0.0;
  for (int p = 0; p < splits; ++p) s += partial[(int64_t)p * ka * kb + e];
  M[(e / kb) * ldm + (e % kb)] = s;
}

// out_c[i] = sum_b S_b[i] U[b][c]; block = 256 rows x RC outputs
constexpr int RC = 16;
constexpr int RBK = 128;  // U rows staged per step
template <typename T>
__global__ void __launch_bounds__(256)
rotate_kernel(const T* __restrict__ S, int64_t lds, int kb, const double* __restrict__ U,
              int64_t ldu, int kc, T* __restrict__ out, int64_t ldo, int64_t n) {
  __shared__ T us[RBK][RC];
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int c0 = blockIdx.y * RC;
  T acc[RC];
#pragma unroll
  for (int c = 0; c < RC; ++c) acc[c] = T(0);
  for (int b0 = 0; b0 < kb; b0 += RBK) {
    const int nb = min(RBK, kb - b0);
    __syncthreads();
    for (int e = threadIdx.x; e < RBK * RC; e += 256) {
      const int r = e / RC, c = e % RC;
      us[r][c] = (r < nb && c0 + c < kc) ? (T)U[(int64_t)(b0 + r) * ldu + c0 + c] : T(0);
    }
    __syncthreads();
    if (i < n) {
      for (int r = 0; r < nb; ++r) {
        const T s = S[(int64_t)(b0 + r) * lds + i];
#pragma unroll
        for (int c = 0; c < RC; ++c) acc[c] += s * us[r][c];
      }
    }
  }
  if (i < n) {
#pragma unroll
    for (int c = 0; c < RC; ++c)
      if (c0 + c < kc) out[(int64_t)(c0 + c) * ldo + i] = acc[c];
  }
}

template <typename T>
__global__ void marginal_var_kernel(const T* __restrict__ A, int64_t lda, int64_t nt, int C, int R,
                                    double s2_0, double s2_1, const double* __restrict__ s2v,
                                    T* __restrict__ var) {
  const int64_t wv = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wv >= nt * C) return;
  const int64_t t = wv / C;
  const int c = (int)(wv % C);
  const T* a = A + t * lda + (int64_t)c * R;
  double acc = 0.0;
  for (int r = lane; r < R; r += 32) acc += (double)a[r] * (double)a[r];
  acc = ncgp::warp_sum(acc);
  if (lane == 0) {
    const double v = s2v[c] - acc;
    var[wv] = (T)(v > 0.0 ? v : 0.0);
  }
}

}  // namespace

extern "C" {

size_t ncgp_reduce_workspace_bytes(int64_t n, int k) {
  const int64_t g = reduce_blocks(n, ncgp::sm_count());
  return ncgp::align_up((size_t)g * (k < 4 ? 4 : k) * sizeof(double), 256);
}

int ncgp_dots(int dtype, int64_t n, int npairs, const void* const* xs, const void* const* ys,
              double* out, void* workspace, size_t ws_bytes, void* stream) {
  NCGP_CHECK_ARG(npairs >= 1 && npairs <= 4, NCGP_INVALID_INPUT, "1 <= npairs <= 4");
  cudaStream_t st = ncgp::as_stream(stream);
  if (n == 0) {
    NCGP_CUDA(cudaMemsetAsync(out, 0, npairs * sizeof(double), st));
    return NCGP_OK;
  }
  const int64_t G = reduce_blocks(n, ncgp::sm_count());
  NCGP_CHECK_ARG(ws_bytes >= (size_t)G * npairs * sizeof(double), NCGP_INVALID_INPUT,
                 "reduce workspace too small");
  const int64_t chunk = (n + G - 1) / G;
  double* part = static_cast<double*>(workspace);
  const void* x[4] = {xs[0], npairs > 1 ? xs[1] : xs[0], npairs > 2 ? xs[2] : xs[0],
                      npairs > 3 ? xs[3] : xs[0]};
  const void* y[4] = {ys[0], npairs > 1 ? ys[1] : ys[0], npairs > 2 ? ys[2] : ys[0],
                      npairs > 3 ? ys[3] : ys[0]};
  bool aligned = true;
  for (int p = 0; p < 4; ++p)
    aligned = aligned && (((uintptr_t)x[p] | (uintptr_t)y[p]) & 15) == 0;
  if (dtype == NCGP_F32 && aligned) {
    const int64_t chunk4 = (chunk + 4 * RB - 1) / (4 * RB) * (4 * RB);
    const int64_t G4 = (n + chunk4 - 1) / chunk4;  // <= G
    dots_partial_v4_kernel<<<(unsigned)G4, RB, 0, st>>>(
        n, npairs, (const float*)x[0], (const float*)y[0], (const float*)x[1], (const float*)y[1],
        (const float*)x[2], (const float*)y[2], (const float*)x[3], (const float*)y[3], chunk4, part);
    NCGP_LAUNCHED();
    sum_partials_kernel<<<(npairs + 7) / 8, 256, 0, st>>>(part, G4, npairs, out);
    NCGP_LAUNCHED();
    return NCGP_OK;
  }
  if (dtype == NCGP_F64)
    dots_partial_kernel<double><<<(unsigned)G, RB, 0, st>>>(
        n, npairs, (const double*)x[0], (const double*)y[0], (const double*)x[1],
        (const double*)y[1], (const double*)x[2], (const double*)y[2], (const double*)x[3],
        (const double*)y[3], chunk, part);
  else
    dots_partial_kernel<float><<<(unsigned)G, RB, 0, st>>>(
        n, npairs, (const float*)x[0], (const float*)y[0], (const float*)x[1],
        (const float*)y[1], (const float*)x[2], (const float*)y[2], (const float*)x[3],
        (const float*)y[3], chunk, part);
  NCGP_LAUNCHED();
  sum_partials_kernel<<<(npairs + 7) / 8, 256, 0, st>>>(part, G, npairs, out);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

int ncgp_gemv_t(int dtype, const void* Q, int64_t ldq, int k, const void* z, int64_t n,
                double* out, void* workspace, size_t ws_bytes, void* stream) {
  NCGP_CHECK_ARG(k >= 0 && k <= 65535, NCGP_DIMENSION_MISMATCH, "bad k");
  cudaStream_t st = ncgp::as_stream(stream);
  if (k == 0) return NCGP_OK;
  if (n == 0) {
    NCGP_CUDA(cudaMemsetAsync(out, 0, k * sizeof(double), st));
    return NCGP_OK;
  }
  const int sms = ncgp::sm_count();
  int64_t G = reduce_blocks(n, sms);
  int64_t per = ((int64_t)sms * 4 + k - 1) / k;  // blocks per row so k*G ~ 4 waves
  if (G > per) G = per < 1 ? 1 : per;
  NCGP_CHECK_ARG(ws_bytes >= (size_t)G * k * sizeof(double), NCGP_INVALID_INPUT,
                 "reduce workspace too small");
  double* part = static_cast<double*>(workspace);
  constexpr int RPB = 8;
  if (dtype == NCGP_F32 && ldq % 4 == 0 && ((uintptr_t)Q & 15) == 0 && ((uintptr_t)z & 15) == 0) {
    // vector path: Gv blocks per group of RPB rows, ~16 blocks per SM in
    // total (a few resident blocks per SM would leave the SMs that got one
    // more block finishing last)
    const int groups = (k + RPB - 1) / RPB;
    int64_t Gv = (n + 4 * RB * 8 - 1) / (4 * RB * 8);  // >= 8 vector sweeps per thread
    const int64_t perv = ((int64_t)sms * 16 + groups - 1) / groups;
    if (Gv > perv) Gv = perv < 1 ? 1 : perv;
    const int64_t gws = (int64_t)(ws_bytes / ((size_t)k * sizeof(double)));
    if (Gv > gws) Gv = gws;  // the workspace holds gws * k partials
    const int64_t chunk = ((n + Gv - 1) / Gv + 4 * RB - 1) / (4 * RB) * (4 * RB);
    Gv = (n + chunk - 1) / chunk;
    gemv_t_partial_v4_kernel<RPB><<<dim3((unsigned)Gv, (unsigned)groups), RB, 0, st>>>(
        (const float*)Q, ldq, k, (const float*)z, n, chunk, part);
    NCGP_LAUNCHED();
    sum_partials_kernel<<<(k + 7) / 8, 256, 0, st>>>(part, Gv, k, out);
    NCGP_LAUNCHED();
    return NCGP_OK;
  }
  const int64_t chunk = (n + G - 1) / G;
  dim3 grid((unsigned)G, (unsigned)k);
  if (dtype == NCGP_F64)
    gemv_t_partial_kernel<double><<<grid, RB, 0, st>>>((const double*)Q, ldq, k,
                                                       (const double*)z, n, chunk, part);
  else
    gemv_t_partial_kernel<float><<<grid, RB, 0, st>>>((const float*)Q, ldq, k, (const float*)z,
                                                      n, chunk, part);
  NCGP_LAUNCHED();
  sum_partials_kernel<<<(k + 7) / 8, 256, 0, st>>>(part, G, k, out);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

int ncgp_gemv_n(int dtype, const void* Q, int64_t ldq, int k, const double* y, const void* s,
                double alpha, void* out, int64_t n, void* stream) {
  NCGP_CHECK_ARG(k >= 0 && k <= 6000, NCGP_DIMENSION_MISMATCH, "gemv_n supports k <= 6000");
  if (n == 0) return NCGP_OK;
  cudaStream_t st = ncgp::as_stream(stream);
  const unsigned g = (unsigned)((n + 255) / 256);
  const size_t smem = (size_t)(k > 0 ? k : 1) * sizeof(double);
  if (dtype == NCGP_F64)
    gemv_n_kernel<double><<<g, 256, smem, st>>>((const double*)Q, ldq, k, y, (const double*)s,
                                                 alpha, (double*)out, n);
  else
    gemv_n_kernel<float><<<g, 256, smem, st>>>((const float*)Q, ldq, k, y, (const float*)s,
                                                alpha, (float*)out, n);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

int ncgp_lincomb(int dtype, int64_t n, double a, const void* x, double b, const void* y, double c,
                 const void* z, void* out, void* stream) {
  if (n == 0) return NCGP_OK;
  cudaStream_t st = ncgp::as_stream(stream);
  auto al16 = [](const void* p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; };
  if (n % 4 == 0 && al16(x) && al16(y) && al16(z) && al16(out)) {
    const int64_t n4 = n / 4;
    const unsigned g4 = (unsigned)((n4 + 255) / 256);
    if (dtype == NCGP_F64)
      lincomb4_kernel<double><<<g4, 256, 0, st>>>(n4, a, (const double*)x, b, (const double*)y,
                                                  c, (const double*)z, (double*)out);
    else
      lincomb4_kernel<float><<<g4, 256, 0, st>>>(n4, a, (const float*)x, b, (const float*)y, c,
                                                 (const float*)z, (float*)out);
    NCGP_LAUNCHED();
    return NCGP_OK;
  }
  const unsigned g = (unsigned)((n + 255) / 256);
  if (dtype == NCGP_F64)
    lincomb_kernel<double><<<g, 256, 0, st>>>(n, a, (const double*)x, b, (const double*)y, c,
                                              (const double*)z, (double*)out);
  else
    lincomb_kernel<float><<<g, 256, 0, st>>>(n, a, (const float*)x, b, (const float*)y, c,
                                             (const float*)z, (float*)out);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

static int gram_splits(int64_t n, int ka, int kb) {
  const int64_t tiles = (int64_t)((ka + GT - 1) / GT) * ((kb + GT - 1) / GT);
  int64_t s = ((int64_t)ncgp::sm_count() * 8 + tiles - 1) / tiles;
  const int64_t maxs = (n + 4095) / 4096;
  if (s > maxs) s = maxs;
  if (s > 512) s = 512;
  return (int)(s < 1 ? 1 : s);
}

size_t ncgp_gram_workspace_bytes(int64_t n, int ka, int kb) {
  return ncgp::align_up((size_t)gram_splits(n, ka, kb) * ka * kb * sizeof(double), 256);
}

int ncgp_gram(int dtype, const void* S, int64_t lds, int ka, const void* Y, int64_t ldy, int kb,
              int64_t n, double* M, int64_t ldm, void* workspace, size_t ws_bytes, void* stream) {
  NCGP_CHECK_ARG(ka >= 0 && kb >= 0 && ka <= 65535 * GT && kb <= 65535 * GT,
                 NCGP_DIMENSION_MISMATCH, "bad gram shape");
  if (ka == 0 || kb == 0) return NCGP_OK;
  cudaStream_t st = ncgp::as_stream(stream);
  const int splits = gram_splits(n, ka, kb);
  NCGP_CHECK_ARG(ws_bytes >= (size_t)splits * ka * kb * sizeof(double), NCGP_INVALID_INPUT,
                 "gram workspace too small");
  int64_t chunk = (n + splits - 1) / splits;
  chunk = (chunk + GK - 1) / GK * GK;
  double* part = static_cast<double*>(workspace);
  dim3 grid((ka + GT - 1) / GT, (kb + GT - 1) / GT, splits);
  if (dtype == NCGP_F64)
    gram_partial_kernel<double><<<grid, 256, 0, st>>>((const double*)S, lds, ka,
                                                      (const double*)Y, ldy, kb, n, chunk, part);
  else
    gram_partial_kernel<float><<<grid, 256, 0, st>>>((const float*)S, lds, ka, (const float*)Y,
                                                     ldy, kb, n, chunk, part);
  NCGP_LAUNCHED();
  const int64_t tot = (int64_t)ka * kb;
  gram_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(part, splits, ka, kb, M, ldm);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

int ncgp_rotate(int dtype, const void* S, int64_t lds, int kb, const double* U, int64_t ldu,
                int kc, void* out, int64_t ldo, int64_t n, void* stream) {
  NCGP_CHECK_ARG(kb >= 0 && kc >= 0 && kc <= 65535 * RC, NCGP_DIMENSION_MISMATCH, "bad shape");
  if (n == 0 || kc == 0) return NCGP_OK;
  cudaStream_t st = ncgp::as_stream(stream);
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)((kc + RC - 1) / RC));
  if (dtype == NCGP_F64)
    rotate_kernel<double><<<grid, 256, 0, st>>>((const double*)S, lds, kb, U, ldu, kc,
                                                (double*)out, ldo, n);
  else
    rotate_kernel<float><<<grid, 256, 0, st>>>((const float*)S, lds, kb, U, ldu, kc,
                                               (float*)out, ldo, n);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

int ncgp_marginal_var(int dtype, const void* A, int64_t lda, int64_t nt, int C, int R,
                      const double* s2_dev, void* var, void* stream) {
  NCGP_CHECK_ARG(C >= 1 && R >= 0, NCGP_DIMENSION_MISMATCH, "bad shape");
  if (nt == 0) return NCGP_OK;
  cudaStream_t st = ncgp::as_stream(stream);
  const int64_t warps = nt * C;
  const unsigned g = (unsigned)((warps * 32 + 255) / 256);
  if (dtype == NCGP_F64)
    marginal_var_kernel<double><<<g, 256, 0, st>>>((const double*)A, lda, nt, C, R, 0, 0, s2_dev,
                                                   (double*)var);
  else
    marginal_var_kernel<float><<<g, 256, 0, st>>>((const float*)A, lda, nt, C, R, 0, 0, s2_dev,
                                                  (float*)var);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

}  // extern "C"
