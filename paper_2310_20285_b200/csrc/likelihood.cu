// K3/K4/K5: per-point likelihood kernels (softmax and Bernoulli-logit).
//
// All are HBM-bound elementwise passes over CN-layout data: one thread owns
// one data point (its C contiguous latent entries) so each thread's loads are
// a contiguous C-element segment and a warp covers 32*C contiguous elements.
#include <math.h>

#include "common.cuh"

namespace {

constexpr double kProbFloor = 1e-12;  // likelihoods.py:22

template <typename T>
__device__ __forceinline__ T dev_exp(T x);
template <>
__device__ __forceinline__ double dev_exp<double>(double x) { return exp(x); }
template <>
__device__ __forceinline__ float dev_exp<float>(float x) { return expf(x); }

// softmax_rows (likelihoods.py:285-288) + grad_log_lik (:247-250) +
// pseudo_targets (outer.py:129-131) for one point.
template <typename T, int CMAX>
__global__ void softmax_stats_kernel(const T* __restrict__ f, const int64_t* __restrict__ y,
                                     int64_t n, int C, T* __restrict__ pi_out,
                                     T* __restrict__ grad_out, T* __restrict__ yhat_out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  T e[CMAX];
  const T* fp = f + p * C;
  T mx = fp[0];
  for (int c = 1; c < C; ++c) mx = fp[c] > mx ? fp[c] : mx;
  T sum = 0;
#pragma unroll
  for (int c = 0; c < CMAX; ++c)
    if (c < C) { e[c] = dev_exp<T>(fp[c] - mx); sum += e[c]; }
  const int64_t lab = y ? y[p] : -1;
#pragma unroll
  for (int c = 0; c < CMAX; ++c)
    if (c < C) {
      e[c] = e[c] / sum;  // pi
      if (pi_out) pi_out[p * C + c] = e[c];
    }
  if (!grad_out && !yhat_out) return;
  T g[CMAX];
  T gm = 0;
#pragma unroll
  for (int c = 0; c < CMAX; ++c)
    if (c < C) {
      g[c] = (c == lab ? T(1) : T(0)) - e[c];
      if (grad_out) grad_out[p * C + c] = g[c];
      gm += g[c];
    }
  if (!yhat_out) return;
  // W^+ g = P diag(1/max(pi, floor)) P g  (likelihoods.py:302-305)
  gm /= T(C);
  T um = 0;
#pragma unroll
  for (int c = 0; c < CMAX; ++c)
    if (c < C) {
      const T pc = e[c] > T(kProbFloor) ? e[c] : T(kProbFloor);
      g[c] = (g[c] - gm) * (T(1) / pc);
      um += g[c];
    }
  um /= T(C);
#pragma unroll
  for (int c = 0; c < CMAX; ++c)
    if (c < C) yhat_out[p * C + c] = fp[c] + (g[c] - um);
}

// The same per point, with the block's 128 points x C values moved through
// shared memory: the (n, C) row-major rows of a block are one contiguous
// range, so every global load and store is a coalesced sweep instead of a
// C-strided access per thread.
template <typename T, int CMAX>
__global__ void softmax_stats_tiled_kernel(const T* __restrict__ f, const int64_t* __restrict__ y,
                                           int64_t n, int C, T* __restrict__ pi_out,
                                           T* __restrict__ grad_out, T* __restrict__ yhat_out) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* tile = reinterpret_cast<T*>(smraw);  // [128][C]
  const int64_t p0 = (int64_t)blockIdx.x * 128;
  const int np = n - p0 < 128 ? (int)(n - p0) : 128;
  const int m = np * C;
  const T* src = f + p0 * C;
  for (int j = threadIdx.x; j < m; j += blockDim.x) tile[j] = src[j];
  __syncthreads();
  const int t = threadIdx.x;
  const bool live = t < np;
  T fv[CMAX], e[CMAX], g[CMAX];
  T sum = 0, gm = 0;
  if (live) {
    T mx = tile[t * C];
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < C) {
        fv[c] = tile[t * C + c];
        mx = fv[c] > mx ? fv[c] : mx;
      }
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < C) { e[c] = dev_exp<T>(fv[c] - mx); sum += e[c]; }
    const int64_t lab = y ? y[p0 + t] : -1;
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < C) {
        e[c] = e[c] / sum;  // pi
        g[c] = (c == lab ? T(1) : T(0)) - e[c];
        gm += g[c];
      }
  }
  // one coalesced store sweep per requested output, staged through the tile
  auto store = [&](T* dst, int which) {
    __syncthreads();
    if (live) {
      if (which == 0) {
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < C) tile[t * C + c] = e[c];
      } else if (which == 1) {
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < C) tile[t * C + c] = g[c];
      } else {
        // W^+ g = P diag(1/max(pi, floor)) P g  (likelihoods.py:302-305)
        const T gmean = gm / T(C);
        T u[CMAX];
        T um = 0;
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < C) {
            const T pc = e[c] > T(kProbFloor) ? e[c] : T(kProbFloor);
            u[c] = (g[c] - gmean) * (T(1) / pc);
            um += u[c];
          }
        um /= T(C);
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < C) tile[t * C + c] = fv[c] + (u[c] - um);
      }
    }
    __syncthreads();
    T* d = dst + p0 * C;
    for (int j = threadIdx.x; j < m; j += blockDim.x) d[j] = tile[j];
  };
  if (pi_out) store(pi_out, 0);
  if (grad_out) store(grad_out, 1);
  if (yhat_out) store(yhat_out, 2);
}

// out = beta*base + alpha*W^+ V, column blocks (likelihoods.py:291-310)
template <typename T, int CMAX>
__global__ void softmax_winv_kernel(const T* __restrict__ pi, int64_t n, int C,
                                    const T* __restrict__ V, int64_t ldv, int k,
                                    const T* __restrict__ base, int64_t ldb, T alpha, T beta,
                                    T* __restrict__ out, int64_t ldo) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (p >= n || b >= k) return;
  const T* v = V + b * ldv + p * C;
  const T* pp = pi + p * C;
  T u[CMAX];
  T m = 0;
#pragma unroll
  for (int c = 0; c < CMAX; ++c)
    if (c < C) { u[c] = v[c]; m += u[c]; }
  m /= T(C);
  T m2 = 0;
#pragma unroll
  for (int c = 0; c < CMAX; ++c)
    if (c < C) {
      const T pc = pp[c] > T(kProbFloor) ? pp[c] : T(kProbFloor);
      u[c] = (u[c] - m) * (T(1) / pc);
      m2 += u[c];
    }
  m2 /= T(C);
  T* o = out + b * ldo + p * C;
  const T* bs = base ? base + b * ldb + p * C : nullptr;
#pragma unroll
  for (int c = 0; c < CMAX; ++c)
    if (c < C) {
      T r = alpha * (u[c] - m2);
      if (bs) r += beta * bs[c];
      o[c] = r;
    }
}

// (diag(pi) - pi pi') v per point (likelihoods.py:252-256)
template <typename T, int CMAX>
__global__ void softmax_w_kernel(const T* __restrict__ pi, int64_t n, int C,
                                 const T* __restrict__ V, int64_t ldv, int k,
                                 T* __restrict__ out, int64_t ldo) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (p >= n || b >= k) return;
  const T* v = V + b * ldv + p * C;
  const T* pp = pi + p * C;
  T dot = 0;
  for (int c = 0; c < C; ++c) dot += pp[c] * v[c];
  T* o = out + b * ldo + p * C;
  for (int c = 0; c < C; ++c) o[c] = pp[c] * v[c] - pp[c] * dot;
}

template <typename T>
__device__ __forceinline__ T expit(T x) {
  if (x >= T(0)) return T(1) / (T(1) + dev_exp<T>(-x));
  const T e = dev_exp<T>(x);
  return e / (T(1) + e);
}

// likelihoods.py:202-212 and pseudo_targets outer.py:129-131
template <typename T>
__global__ void bernoulli_stats_kernel(const T* __restrict__ f, const int64_t* __restrict__ y,
                                       int64_t n, T* __restrict__ winv, T* __restrict__ w,
                                       T* __restrict__ grad, T* __restrict__ yhat) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T fi = f[i];
  const T s = expit<T>(fi);
  T wi, wv;
  if (sizeof(T) == 8) {
    // reference clamp verbatim: s in [1e-12, 1 - 1e-12]
    const T sc = fmin(fmax((double)s, kProbFloor), 1.0 - kProbFloor);
    wi = T(1) / (sc * (T(1) - sc));
    wv = s * (T(1) - s);
  } else {
    // fp32: 1 - 1e-12 rounds to 1, so use s * sigma(-f) with the same floor
    // (W^-1 <= ~1e12), see SURVEY.md 8(a) a12.
    const T prod = s * expit<T>(-fi);
    wv = prod;
    wi = T(1) / (prod > T(1e-12) ? prod : T(1e-12));
  }
  const T g = (y ? (T)y[i] : T(0)) - s;
  if (winv) winv[i] = wi;
  if (w) w[i] = wv;
  if (grad) grad[i] = g;
  if (yhat) yhat[i] = fi + wi * g;
}

// Poisson, log link (likelihoods.py:174-182, outer.py:129-131): w = e^f,
// winv = e^-f, grad = y - e^f, yhat = f + winv * grad
template <typename T>
__global__ void poisson_stats_kernel(const T* __restrict__ f, const T* __restrict__ y, int64_t n,
                                     T* __restrict__ winv, T* __restrict__ w, T* __restrict__ grad,
                                     T* __restrict__ yhat) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T fi = f[i];
  const T wv = dev_exp<T>(fi);
  const T wi = dev_exp<T>(-fi);
  const T g = (y ? y[i] : T(0)) - wv;
  if (winv) winv[i] = wi;
  if (w) w[i] = wv;
  if (grad) grad[i] = g;
  if (yhat) yhat[i] = fi + wi * g;
}

template <typename T>
__global__ void diag_apply_kernel(const T* __restrict__ d, int64_t n, const T* __restrict__ V,
                                  int64_t ldv, int k, const T* __restrict__ base, int64_t ldb,
                                  T alpha, T beta, T* __restrict__ out, int64_t ldo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= n || b >= k) return;
  T r = alpha * d[i] * V[b * ldv + i];
  if (base) r += beta * base[b * ldb + i];
  out[b * ldo + i] = r;
}

template <int CMAX, typename T>
int launch_stats(const T* f, const int64_t* y, int64_t n, int C, T* pi, T* g, T* yh,
                 cudaStream_t st) {
  if constexpr (CMAX <= 16)  // tiles of <= 16 KB; wider C keeps the per-thread kernel (registers)
    softmax_stats_tiled_kernel<T, CMAX><<<(unsigned)((n + 127) / 128), 128,
                                         (size_t)128 * C * sizeof(T), st>>>(f, y, n, C, pi, g, yh);
  else
    softmax_stats_kernel<T, CMAX><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(f, y, n, C, pi, g,
                                                                                 yh);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

template <typename T>
int stats_t(const void* f, const int64_t* y, int64_t n, int C, void* pi, void* g, void* yh,
            cudaStream_t st) {
  auto F = static_cast<const T*>(f);
  auto P = static_cast<T*>(pi);
  auto G = static_cast<T*>(g);
  auto Y = static_cast<T*>(yh);
  if (C <= 4) return launch_stats<4>(F, y, n, C, P, G, Y, st);
  if (C <= 16) return launch_stats<16>(F, y, n, C, P, G, Y, st);
  return launch_stats<64>(F, y, n, C, P, G, Y, st);
}

template <int CMAX, typename T>
int launch_winv(const T* pi, int64_t n, int C, const T* V, int64_t ldv, int k, const T* base,
                int64_t ldb, T a, T b, T* out, int64_t ldo, cudaStream_t st) {
  dim3 grid((unsigned)((n + 127) / 128), (unsigned)k);
  softmax_winv_kernel<T, CMAX><<<grid, 128, 0, st>>>(pi, n, C, V, ldv, k, base, ldb, a, b, out,
                                                     ldo);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

template <typename T>
int winv_t(const void* pi, int64_t n, int C, const void* V, int64_t ldv, int k, const void* base,
           int64_t ldb, double a, double b, void* out, int64_t ldo, cudaStream_t st) {
  auto P = static_cast<const T*>(pi);
  auto Vv = static_cast<const T*>(V);
  auto B = static_cast<const T*>(base);
  auto O = static_cast<T*>(out);
  if (C <= 4) return launch_winv<4>(P, n, C, Vv, ldv, k, B, ldb, (T)a, (T)b, O, ldo, st);
  if (C <= 16) return launch_winv<16>(P, n, C, Vv, ldv, k, B, ldb, (T)a, (T)b, O, ldo, st);
  return launch_winv<64>(P, n, C, Vv, ldv, k, B, ldb, (T)a, (T)b, O, ldo, st);
}

}  // namespace

extern "C" {

int ncgp_softmax_stats(int dtype, const void* f, const int64_t* labels, int64_t n, int C,
                       void* pi, void* grad, void* yhat, void* stream) {
  NCGP_CHECK_ARG(C >= 2 && C <= 64, NCGP_UNSUPPORTED, "softmax supports 2 <= C <= 64 (got %d)", C);
  NCGP_CHECK_ARG(n >= 0, NCGP_DIMENSION_MISMATCH, "negative n");
  if (n == 0) return NCGP_OK;
  NCGP_CHECK_ARG(f && pi, NCGP_INVALID_INPUT, "null operand");
  NCGP_CHECK_ARG(!(grad || yhat) || labels, NCGP_INVALID_INPUT, "labels required");
  cudaStream_t st = ncgp::as_stream(stream);
  if (dtype == NCGP_F64) return stats_t<double>(f, labels, n, C, pi, grad, yhat, st);
  if (dtype == NCGP_F32) return stats_t<float>(f, labels, n, C, pi, grad, yhat, st);
  NCGP_CHECK_ARG(false, NCGP_UNSUPPORTED, "dtype %d", dtype);
}

int ncgp_softmax_winv(int dtype, const void* pi, int64_t n, int C, const void* V, int64_t ldv,
                      int k, const void* base, int64_t ldb, double alpha, double beta, void* out,
                      int64_t ldo, void* stream) {
  NCGP_CHECK_ARG(C >= 2 && C <= 64, NCGP_UNSUPPORTED, "softmax supports 2 <= C <= 64 (got %d)", C);
  NCGP_CHECK_ARG(k >= 0 && k <= 65535 && n >= 0, NCGP_DIMENSION_MISMATCH, "bad shape");
  if (n == 0 || k == 0) return NCGP_OK;
  NCGP_CHECK_ARG(ldv >= n * C && ldo >= n * C && (!base || ldb >= n * C),
                 NCGP_DIMENSION_MISMATCH, "leading dimension < n*C");
  cudaStream_t st = ncgp::as_stream(stream);
  if (dtype == NCGP_F64)
    return winv_t<double>(pi, n, C, V, ldv, k, base, ldb, alpha, beta, out, ldo, st);
  if (dtype == NCGP_F32)
    return winv_t<float>(pi, n, C, V, ldv, k, base, ldb, alpha, beta, out, ldo, st);
  NCGP_CHECK_ARG(false, NCGP_UNSUPPORTED, "dtype %d", dtype);
}

int ncgp_softmax_w(int dtype, const void* pi, int64_t n, int C, const void* V, int64_t ldv, int k,
                   void* out, int64_t ldo, void* stream) {
  NCGP_CHECK_ARG(C >= 2, NCGP_UNSUPPORTED, "softmax needs C >= 2");
  NCGP_CHECK_ARG(k >= 0 && k <= 65535 && n >= 0, NCGP_DIMENSION_MISMATCH, "bad shape");
  if (n == 0 || k == 0) return NCGP_OK;
  cudaStream_t st = ncgp::as_stream(stream);
  dim3 grid((unsigned)((n + 127) / 128), (unsigned)k);
  if (dtype == NCGP_F64)
    softmax_w_kernel<double, 64><<<grid, 128, 0, st>>>(
        (const double*)pi, n, C, (const double*)V, ldv, k, (double*)out, ldo);
  else
    softmax_w_kernel<float, 64><<<grid, 128, 0, st>>>((const float*)pi, n, C, (const float*)V,
                                                       ldv, k, (float*)out, ldo);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

int ncgp_bernoulli_stats(int dtype, const void* f, const int64_t* labels, int64_t n, void* winv,
                         void* w, void* grad, void* yhat, void* stream) {
  NCGP_CHECK_ARG(n >= 0, NCGP_DIMENSION_MISMATCH, "negative n");
  if (n == 0) return NCGP_OK;
  NCGP_CHECK_ARG(!(grad || yhat) || labels, NCGP_INVALID_INPUT, "labels required");
  cudaStream_t st = ncgp::as_stream(stream);
  const unsigned g = (unsigned)((n + 255) / 256);
  if (dtype == NCGP_F64)
    bernoulli_stats_kernel<double><<<g, 256, 0, st>>>((const double*)f, labels, n,
                                                      (double*)winv, (double*)w, (double*)grad,
                                                      (double*)yhat);
  else
    bernoulli_stats_kernel<float><<<g, 256, 0, st>>>((const float*)f, labels, n, (float*)winv,
                                                     (float*)w, (float*)grad, (float*)yhat);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

int ncgp_poisson_stats(int dtype, const void* f, const void* counts, int64_t n, void* winv,
                       void* w, void* grad, void* yhat, void* stream) {
  NCGP_CHECK_ARG(n >= 0, NCGP_DIMENSION_MISMATCH, "negative n");
  if (n == 0) return NCGP_OK;
  NCGP_CHECK_ARG(f != nullptr, NCGP_INVALID_INPUT, "null latent");
  NCGP_CHECK_ARG(!(grad || yhat) || counts, NCGP_INVALID_INPUT, "counts required");
  cudaStream_t st = ncgp::as_stream(stream);
  const unsigned g = (unsigned)((n + 255) / 256);
  if (dtype == NCGP_F64)
    poisson_stats_kernel<double><<<g, 256, 0, st>>>((const double*)f, (const double*)counts, n,
                                                    (double*)winv, (double*)w, (double*)grad,
                                                    (double*)yhat);
  else
    poisson_stats_kernel<float><<<g, 256, 0, st>>>((const float*)f, (const float*)counts, n,
                                                   (float*)winv, (float*)w, (float*)grad,
                                                   (float*)yhat);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

int ncgp_diag_apply(int dtype, const void* dvec, int64_t n, const void* V, int64_t ldv, int k,
                    const void* base, int64_t ldb, double alpha, double beta, void* out,
                    int64_t ldo, void* stream) {
  NCGP_CHECK_ARG(k >= 0 && k <= 65535 && n >= 0, NCGP_DIMENSION_MISMATCH, "bad shape");
  if (n == 0 || k == 0) return NCGP_OK;
  cudaStream_t st = ncgp::as_stream(stream);
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)k);
  if (dtype == NCGP_F64)
    diag_apply_kernel<double><<<grid, 256, 0, st>>>((const double*)dvec, n, (const double*)V, ldv,
                                                    k, (const double*)base, ldb, alpha, beta,
                                                    (double*)out, ldo);
  else
    diag_apply_kernel<float><<<grid, 256, 0, st>>>((const float*)dvec, n, (const float*)V, ldv,
                                                   k, (const float*)base, ldb, (float)alpha,
                                                   (float)beta, (float*)out, ldo);
  NCGP_LAUNCHED();
  return NCGP_OK;
}

}  // extern "C"
