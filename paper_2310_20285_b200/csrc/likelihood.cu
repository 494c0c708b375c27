// K3/K4/K5: per-point likelihood kernels (softmax and Bernoulli-logit).
//
// All are HBM-bound elementwise passes over CN-layout data: one thread owns
// one data point (its C contiguous latent entries) so each thread's loads are
// a contiguous C-element segment and a warp covers 32*C contiguous elements.
#include <math.h>

#include <algorithm>

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

// ---- staged per-point kernels (round 2): a block owns PTS = 256 points, i.e.
// a contiguous 256 C-element segment of every CN-layout operand.  Operands are
// swept between HBM and shared memory with 16-byte vector accesses (every
// segment starts at a multiple of 1024 C bytes), each thread then works on its
// point from shared memory, and the results are swept back the same way.  So
// global traffic is fully coalesced and vectorised, and the per-point values
// live in shared memory instead of CMAX-sized register arrays (the per-thread
// kernels ran at 37 % occupancy with 77 registers; ncu, r02d).
constexpr int PTS = 256;
constexpr size_t kStagedSmem = 96 * 1024;  // the staged kernels' largest tile set (2 blocks per SM)

// m elements from global to shared memory: 16-byte cp.async (LDGSTS) copies
// where the global segment is 16-byte aligned -- all of a thread's copies are
// in flight at once, no register round trip -- element-wise otherwise.  The
// caller waits with async_wait_all() + __syncthreads().
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <typename T>
__device__ __forceinline__ void sweep_in(T* __restrict__ dst, const T* __restrict__ src, int m) {
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    constexpr int E = 16 / sizeof(T);
    const int mv = m / E;
    for (int j = threadIdx.x; j < mv; j += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst + j * E)),
                   "l"(src + j * E)
                   : "memory");
    for (int j = mv * E + threadIdx.x; j < m; j += blockDim.x) dst[j] = src[j];
  } else {
    for (int j = threadIdx.x; j < m; j += blockDim.x) dst[j] = src[j];
  }
}
__device__ __forceinline__ void async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
template <typename T>
__device__ __forceinline__ void sweep_out(T* __restrict__ dst, const T* __restrict__ src, int m) {
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    constexpr int E = 16 / sizeof(T);
    const int mv = m / E;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int j = threadIdx.x; j < mv; j += blockDim.x) __stcs(d4 + j, s4[j]);
    for (int j = mv * E + threadIdx.x; j < m; j += blockDim.x) dst[j] = src[j];
  } else {
    for (int j = threadIdx.x; j < m; j += blockDim.x) dst[j] = src[j];
  }
}

// softmax_rows + grad_log_lik + pseudo_targets, staged.  smem: f tile, then
// one output tile per requested output.  Per point only pi (CMAX registers)
// is kept; grad and the W^+ g terms are recomputed from it.
template <typename T, int CMAX>
__global__ void __launch_bounds__(PTS) softmax_stats_staged_kernel(
    const T* __restrict__ f, const int64_t* __restrict__ y, int64_t n, int C, T* __restrict__ pi_out,
    T* __restrict__ grad_out, T* __restrict__ yhat_out) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* fin = reinterpret_cast<T*>(smraw);
  const int64_t p0 = (int64_t)blockIdx.x * PTS;
  const int np = n - p0 < PTS ? (int)(n - p0) : PTS;
  const int m = np * C;
  T* outs[3] = {pi_out, grad_out, yhat_out};
  T* tiles[3];
  int no = 0;
  for (int k = 0; k < 3; ++k) tiles[k] = outs[k] ? fin + (size_t)PTS * C * (++no) : nullptr;
  sweep_in(fin, f + p0 * C, m);
  async_wait_all();
  __syncthreads();
  const int t = threadIdx.x;
  if (t < np) {
    const T* fv = fin + t * C;
    T e[CMAX];
    T mx = fv[0];
#pragma unroll
    for (int c = 1; c < CMAX; ++c)
      if (c < C) mx = fv[c] > mx ? fv[c] : mx;
    T sum = 0;
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < C) { e[c] = dev_exp<T>(fv[c] - mx); sum += e[c]; }
    const T rs = T(1) / sum;  // one division per point: e * (1 / sum) is within an ulp of e / sum
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < C) e[c] = e[c] * rs;  // pi (likelihoods.py:285-288)
    const int64_t lab = (grad_out || yhat_out) ? y[p0 + t] : -1;
    if (tiles[0]) {
#pragma unroll
      for (int c = 0; c < CMAX; ++c)
        if (c < C) tiles[0][t * C + c] = e[c];
    }
    T gm = 0;
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < C) {
        const T g = (c == lab ? T(1) : T(0)) - e[c];
        gm += g;
        if (tiles[1]) tiles[1][t * C + c] = g;
      }
    if (tiles[2]) {
      // yhat = f + W^+ g,  W^+ g = P diag(1/max(pi, floor)) P g  (likelihoods.py:302-305)
      const T gmean = gm / T(C);
      T um = 0;
#pragma unroll
      for (int c = 0; c < CMAX; ++c)
        if (c < C) {
          const T pc = e[c] > T(kProbFloor) ? e[c] : T(kProbFloor);
          const T u = (((c == lab ? T(1) : T(0)) - e[c]) - gmean) * (T(1) / pc);
          tiles[2][t * C + c] = u;  // u kept in the output tile, no second division
          um += u;
        }
      um /= T(C);
#pragma unroll
      for (int c = 0; c < CMAX; ++c)
        if (c < C) tiles[2][t * C + c] = fv[c] + (tiles[2][t * C + c] - um);
    }
  }
  __syncthreads();
  for (int k = 0; k < 3; ++k)
    if (tiles[k]) sweep_out(outs[k] + p0 * C, tiles[k], m);
}

// out = beta base + alpha W^+ V (likelihoods.py:291-310), staged.  The pi
// tile is loaded once per block and turned into 1 / max(pi, floor) in place
// (one division per entry), then the block's kb column blocks of V
// (grid.y slices the k columns so that wide W+ applies -- the virtual
// solver run's S blocks, k ~ 800 -- still fill the GPU) are swept through in
// turn (pi is not re-read per column block).
template <typename T>
__global__ void __launch_bounds__(PTS) softmax_winv_staged_kernel(
    const T* __restrict__ pi, int64_t n, int C, const T* __restrict__ V, int64_t ldv, int k,
    const T* __restrict__ base, int64_t ldb, T alpha, T beta, T* __restrict__ out, int64_t ldo,
    int kb) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* tp = reinterpret_cast<T*>(smraw);
  T* tv = tp + PTS * C;
  T* tb = tv + PTS * C;
  const int64_t p0 = (int64_t)blockIdx.x * PTS;
  const int np = n - p0 < PTS ? (int)(n - p0) : PTS;
  const int m = np * C;
  const int t = threadIdx.x;
  const int b0 = blockIdx.y * kb, b1 = min(k, b0 + kb);
  sweep_in(tp, pi + p0 * C, m);
  sweep_in(tv, V + b0 * ldv + p0 * C, m);
  if (base) sweep_in(tb, base + b0 * ldb + p0 * C, m);
  async_wait_all();
  __syncthreads();
  if (t < np)
    for (int c = 0; c < C; ++c) {
      const T pc = tp[t * C + c] > T(kProbFloor) ? tp[t * C + c] : T(kProbFloor);
      tp[t * C + c] = T(1) / pc;
    }
  for (int b = b0; b < b1; ++b) {
    if (b > b0) {
      sweep_in(tv, V + b * ldv + p0 * C, m);
      if (base) sweep_in(tb, base + b * ldb + p0 * C, m);
      async_wait_all();
      __syncthreads();
    }
    if (t < np) {
      const T* rp = tp + t * C;
      T* v = tv + t * C;
      T mean = 0;
      for (int c = 0; c < C; ++c) mean += v[c];
      mean /= T(C);
      // u_c = (v_c - mean) / max(pi_c, floor), in place over the V tile
      T m2 = 0;
      for (int c = 0; c < C; ++c) {
        const T u = (v[c] - mean) * rp[c];
        v[c] = u;
        m2 += u;
      }
      m2 /= T(C);
      for (int c = 0; c < C; ++c) {
        T r = alpha * (v[c] - m2);
        if (base) r += beta * tb[t * C + c];
        v[c] = r;
      }
    }
    __syncthreads();
    sweep_out(out + b * ldo + p0 * C, tv, m);
    __syncthreads();
  }
}

// (diag(pi) - pi pi') v per point (likelihoods.py:252-256), staged
template <typename T>
__global__ void __launch_bounds__(PTS) softmax_w_staged_kernel(
    const T* __restrict__ pi, int64_t n, int C, const T* __restrict__ V, int64_t ldv,
    T* __restrict__ out, int64_t ldo) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* tp = reinterpret_cast<T*>(smraw);
  T* tv = tp + PTS * C;
  const int64_t p0 = (int64_t)blockIdx.x * PTS;
  const int b = blockIdx.y;
  const int np = n - p0 < PTS ? (int)(n - p0) : PTS;
  const int m = np * C;
  sweep_in(tp, pi + p0 * C, m);
  sweep_in(tv, V + b * ldv + p0 * C, m);
  async_wait_all();
  __syncthreads();
  const int t = threadIdx.x;
  if (t < np) {
    const T* pp = tp + t * C;
    T* v = tv + t * C;
    T dot = 0;
    for (int c = 0; c < C; ++c) dot += pp[c] * v[c];
    for (int c = 0; c < C; ++c) v[c] = pp[c] * v[c] - pp[c] * dot;
  }
  __syncthreads();
  sweep_out(out + b * ldo + p0 * C, tv, m);
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

// Elementwise kernels: each thread owns EW = 4 elements, blockDim apart (every
// access stays coalesced), with all loads issued before any use -- four
// independent loads in flight per thread instead of one.
constexpr int EW = 4;

// likelihoods.py:202-212 and pseudo_targets outer.py:129-131
template <typename T>
__global__ void bernoulli_stats_kernel(const T* __restrict__ f, const int64_t* __restrict__ y,
                                       int64_t n, T* __restrict__ winv, T* __restrict__ w,
                                       T* __restrict__ grad, T* __restrict__ yhat) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x * EW + threadIdx.x;
  T fv[EW], yv[EW];
#pragma unroll
  for (int u = 0; u < EW; ++u) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    fv[u] = i < n ? __ldcs(f + i) : T(0);
    yv[u] = (y && i < n) ? (T)__ldcs(y + i) : T(0);
  }
#pragma unroll
  for (int u = 0; u < EW; ++u) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    if (i >= n) break;
    const T fi = fv[u];
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
    const T g = yv[u] - s;
    if (winv) __stcs(winv + i, wi);
    if (w) __stcs(w + i, wv);
    if (grad) __stcs(grad + i, g);
    if (yhat) __stcs(yhat + i, fi + wi * g);
  }
}

// Poisson, log link (likelihoods.py:174-182, outer.py:129-131): w = e^f,
// winv = e^-f, grad = y - e^f, yhat = f + winv * grad
template <typename T>
__global__ void poisson_stats_kernel(const T* __restrict__ f, const T* __restrict__ y, int64_t n,
                                     T* __restrict__ winv, T* __restrict__ w, T* __restrict__ grad,
                                     T* __restrict__ yhat) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x * EW + threadIdx.x;
  T fv[EW], yv[EW];
#pragma unroll
  for (int u = 0; u < EW; ++u) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    fv[u] = i < n ? __ldcs(f + i) : T(0);
    yv[u] = (y && i < n) ? __ldcs(y + i) : T(0);
  }
#pragma unroll
  for (int u = 0; u < EW; ++u) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    if (i >= n) break;
    const T fi = fv[u];
    const T wv = dev_exp<T>(fi);
    const T wi = dev_exp<T>(-fi);
    const T g = yv[u] - wv;
    if (winv) __stcs(winv + i, wi);
    if (w) __stcs(w + i, wv);
    if (grad) __stcs(grad + i, g);
    if (yhat) __stcs(yhat + i, fi + wi * g);
  }
}

template <typename T>
__global__ void diag_apply_kernel(const T* __restrict__ d, int64_t n, const T* __restrict__ V,
                                  int64_t ldv, int k, const T* __restrict__ base, int64_t ldb,
                                  T alpha, T beta, T* __restrict__ out, int64_t ldo) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x * EW + threadIdx.x;
  const int b = blockIdx.y;
  if (b >= k) return;
  T dv[EW], vv[EW], bv[EW];
#pragma unroll
  for (int u = 0; u < EW; ++u) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    const bool in = i < n;
    dv[u] = in ? d[i] : T(0);
    vv[u] = in ? __ldcs(V + b * ldv + i) : T(0);
    bv[u] = (in && base) ? __ldcs(base + b * ldb + i) : T(0);
  }
#pragma unroll
  for (int u = 0; u < EW; ++u) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    if (i >= n) break;
    T r = alpha * dv[u] * vv[u];
    if (base) r += beta * bv[u];
    __stcs(out + b * ldo + i, r);
  }
}

template <int CMAX, typename T>
int launch_stats(const T* f, const int64_t* y, int64_t n, int C, T* pi, T* g, T* yh,
                 cudaStream_t st) {
  const int nout = (pi ? 1 : 0) + (g ? 1 : 0) + (yh ? 1 : 0);
  const size_t sm = (size_t)(1 + nout) * PTS * C * sizeof(T);
  if (CMAX <= 16 && sm <= kStagedSmem) {  // staged: vectorised sweeps, values in shared memory
    auto kern = softmax_stats_staged_kernel<T, CMAX>;
    NCGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStagedSmem));
    kern<<<(unsigned)((n + PTS - 1) / PTS), PTS, sm, st>>>(f, y, n, C, pi, g, yh);
  } else if constexpr (CMAX <= 16)  // tiles of <= 16 KB; wider C keeps the per-thread kernel (registers)
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
  const size_t sm = (size_t)(base ? 3 : 2) * PTS * C * sizeof(T);
  if (sm <= kStagedSmem) {
    auto kern = softmax_winv_staged_kernel<T>;
    NCGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStagedSmem));
    // column blocks per CTA: enough CTAs (~2048) to fill the GPU, pi loaded once per CTA
    const int64_t nbx = (n + PTS - 1) / PTS;
    const int slices = (int)std::max<int64_t>(1, std::min<int64_t>(k, 2048 / std::max<int64_t>(1, nbx)));
    const int kb = (k + slices - 1) / slices;
    kern<<<dim3((unsigned)nbx, (unsigned)((k + kb - 1) / kb)), PTS, sm, st>>>(pi, n, C, V, ldv, k, base,
                                                                            ldb, a, b, out, ldo, kb);
    NCGP_LAUNCHED();
    return NCGP_OK;
  }
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
  const size_t es = dtype == NCGP_F64 ? 8 : 4;
  const size_t sm = 2 * (size_t)PTS * C * es;
  if (sm <= kStagedSmem) {
    const dim3 sg((unsigned)((n + PTS - 1) / PTS), (unsigned)k);
    if (dtype == NCGP_F64) {
      auto kern = softmax_w_staged_kernel<double>;
      NCGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStagedSmem));
      kern<<<sg, PTS, sm, st>>>((const double*)pi, n, C, (const double*)V, ldv, (double*)out, ldo);
    } else {
      auto kern = softmax_w_staged_kernel<float>;
      NCGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStagedSmem));
      kern<<<sg, PTS, sm, st>>>((const float*)pi, n, C, (const float*)V, ldv, (float*)out, ldo);
    }
    NCGP_LAUNCHED();
    return NCGP_OK;
  }
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
  const unsigned g = (unsigned)((n + 256 * EW - 1) / (256 * EW));
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
  const unsigned g = (unsigned)((n + 256 * EW - 1) / (256 * EW));
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
  dim3 grid((unsigned)((n + 256 * EW - 1) / (256 * EW)), (unsigned)k);
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
