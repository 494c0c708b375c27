// CUDA-core kernel-matmul: the fp64 path (conformance / cfg1) and the
// exact-distance fp32 path used when the tcgen05 operator's precision guard
// rejects an input.  Same contract as the tcgen05 kernel:
//
//   out[i, c] = sum_j k(Xr[i], Xc[j]) V[j, c]
//
// fp64 arithmetic replays the reference's operation order per entry:
// _sqdist accumulates (x_i - x_j)^2 feature by feature (gp.py:108-113) and
// kernel_from_sqdist applies clamp / divide / exp / scale in the same order
// (gp.py:84-98); explicit _rn intrinsics stop the compiler from fusing
// those into FMAs.  Only the long j-sum differs from numpy's pairwise sum
// (it is a fixed-order split sum here), i.e. results agree to ~1e-15.
#include <math.h>

#include "kop.cuh"

namespace {

constexpr int BR = 128;      // rows per block, one per thread
template <typename T>
constexpr int jt_of() { return sizeof(T) == 8 ? 32 : 64; }  // columns staged per step
constexpr int CHUNK = 2048;  // fp32 accumulators flushed to fp64 this often

template <typename T, int FAM>
struct KernelFn;

template <int FAM>
struct KernelFn<double, FAM> {
  double ell, s2, neg2l2;
  template <int DMAX>
  __device__ __forceinline__ double sqd(const double* xi, const double* xj, int D) const {
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
      if (d < D) {
        double t = __dsub_rn(xi[d], xj[d]);
        acc = __dadd_rn(acc, __dmul_rn(t, t));
      }
    }
    return acc;
  }
  __device__ __forceinline__ double operator()(double d2) const {
    d2 = fmax(d2, 0.0);
    if (FAM == NCGP_RBF) {
      return __dmul_rn(exp(__ddiv_rn(d2, neg2l2)), s2);
    } else {
      double a = __ddiv_rn(__dsqrt_rn(__dmul_rn(d2, 3.0)), ell);
      double e = exp(-a);
      return __dmul_rn(__dmul_rn(e, __dadd_rn(a, 1.0)), s2);
    }
  }
};

template <int FAM>
struct KernelFn<float, FAM> {
  float c, s2, sq3l;
  template <int DMAX>
  __device__ __forceinline__ float sqd(const float* xi, const float* xj, int D) const {
    // padded features are zero on both sides, so no predicate is needed
    float acc = 0.f;
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
      float t = xi[d] - xj[d];
      acc = fmaf(t, t, acc);
    }
    return acc;
  }
  __device__ __forceinline__ float operator()(float d2) const {
    d2 = fmaxf(d2, 0.f);
    if (FAM == NCGP_RBF) {
      return s2 * exp2f(d2 * c);  // c = -log2(e) / (2 l^2)
    } else {
      float a = sqrtf(d2) * sq3l;  // sqrt(3) d / l
      return s2 * (1.f + a) * exp2f(-1.4426950408889634f * a);
    }
  }
};

template <typename T, int FAM, int DMAX, int WT>
__global__ void __launch_bounds__(BR)
kop_simt_kernel(const T* __restrict__ Xr, int64_t nloc, const T* __restrict__ Xc,
                int64_t nc, int D, const T* __restrict__ V, int64_t ldv, int w,
                int64_t cols_per_split, double* __restrict__ partial, KernelFn<T, FAM> kf) {
  constexpr int JT = jt_of<T>();
  __shared__ T xs[JT][DMAX + 1];
  __shared__ T vs[JT][WT];
  const int64_t i = (int64_t)blockIdx.x * BR + threadIdx.x;
  const bool live = i < nloc;
  const int split = blockIdx.y;
  const int c0 = blockIdx.z * WT;
  const int64_t j0 = (int64_t)split * cols_per_split;
  const int64_t j1 = min(nc, j0 + cols_per_split);

  T xi[DMAX];
#pragma unroll
  for (int d = 0; d < DMAX; ++d) xi[d] = (live && d < D) ? Xr[i * D + d] : T(0);

  double acc64[WT];
  T acc[WT];
#pragma unroll
  for (int c = 0; c < WT; ++c) { acc64[c] = 0.0; acc[c] = T(0); }

  int since_flush = 0;
  for (int64_t jt = j0; jt < j1; jt += JT) {
    const int nj = (int)min((int64_t)JT, j1 - jt);
    __syncthreads();
    for (int e = threadIdx.x; e < JT * DMAX; e += BR) {
      int jj = e / DMAX, d = e % DMAX;
      xs[jj][d] = (jj < nj && d < D) ? Xc[(jt + jj) * D + d] : T(0);
    }
    for (int e = threadIdx.x; e < JT * WT; e += BR) {
      int jj = e / WT, c = e % WT;
      vs[jj][c] = (jj < nj && c0 + c < w) ? V[(jt + jj) * ldv + c0 + c] : T(0);
    }
    __syncthreads();
    for (int jj = 0; jj < nj; ++jj) {
      const T kv = kf(kf.template sqd<DMAX>(xi, xs[jj], D));
#pragma unroll
      for (int c = 0; c < WT; ++c) acc[c] += kv * vs[jj][c];
    }
    if (sizeof(T) == 4) {
      since_flush += nj;
      if (since_flush >= CHUNK) {
#pragma unroll
        for (int c = 0; c < WT; ++c) { acc64[c] += (double)acc[c]; acc[c] = T(0); }
        since_flush = 0;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < WT; ++c) acc64[c] += (double)acc[c];
  if (live) {
    double* dst = partial + ((int64_t)split * nloc + i) * w;
#pragma unroll
    for (int c = 0; c < WT; ++c)
      if (c0 + c < w) dst[c0 + c] = acc64[c];
  }
}

template <typename T>
__global__ void reduce_splits_kernel(const double* __restrict__ partial, int splits,
                                     int64_t nloc, int w, const ncgp::OutPtrs<T> out, int64_t ldo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nloc * w) return;
  const int64_t i = e / w;
  const int c = (int)(e % w);
  double s = 0.0;
  for (int p = 0; p < splits; ++p) s += partial[(int64_t)p * nloc * w + e];
#pragma unroll
  for (int k = 0; k < NCGP_MAX_OUTS; ++k)
    if (k < out.n) out.p[k][i * ldo + c] = (T)s;
}

// the same fixed-order split sum, one thread per row, through the epilogue
template <typename T>
__global__ void reduce_splits_epi_kernel(const double* __restrict__ partial, int splits,
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

int pick_wt(int w) { return w <= 1 ? 1 : (w <= 4 ? 4 : (w <= 16 ? 16 : 32)); }
int pick_dmax(int d) { return d <= 8 ? 8 : (d <= 16 ? 16 : (d <= 32 ? 32 : 64)); }

constexpr int JT = 64;  // split granularity (multiple of both staging widths)

int plan_splits(int64_t nloc, int64_t nc, int zs, int sms) {
  const int64_t row_blocks = (nloc + BR - 1) / BR;
  const int64_t target = (int64_t)sms * 16;
  int64_t splits = (target + row_blocks * zs - 1) / (row_blocks * zs);
  const int64_t max_splits = (nc + JT - 1) / JT;
  if (splits > max_splits) splits = max_splits;
  if (splits > 64) splits = 64;
  return (int)(splits < 1 ? 1 : splits);
}

template <typename T, int FAM, int DMAX, int WT>
int launch_t(ncgp_kop* op, const T* Xr, int64_t nloc, const T* V, int64_t ldv, int w,
             const ncgp::OutPtrs<T>& out, int64_t ldo, cudaStream_t st, const EpiDev& epi) {
  const int zs = (w + WT - 1) / WT;
  // planned on the full row count: row shards reduce in the same order
  const int splits = plan_splits(op->n_rows, op->n_cols, zs, op->sms);
  int64_t cps = (op->n_cols + splits - 1) / splits;
  cps = (cps + JT - 1) / JT * JT;
  const size_t need = (size_t)splits * nloc * w * sizeof(double);
  NCGP_CHECK_ARG(need <= op->ws_bytes, NCGP_INVALID_INPUT,
                 "kop workspace too small (%zu < %zu)", op->ws_bytes, need);
  double* partial = reinterpret_cast<double*>(op->ws);
  KernelFn<T, FAM> kf;
  if constexpr (sizeof(T) == 8) {
    kf.ell = op->ell; kf.s2 = op->s2; kf.neg2l2 = -2.0 * op->ell * op->ell;
  } else {
    kf.c = (float)(-1.4426950408889634 / (2.0 * op->ell * op->ell));
    kf.s2 = (float)op->s2;
    kf.sq3l = (float)(1.7320508075688772 / op->ell);
  }
  dim3 grid((unsigned)((nloc + BR - 1) / BR), (unsigned)splits, (unsigned)zs);
  kop_simt_kernel<T, FAM, DMAX, WT><<<grid, BR, 0, st>>>(
      Xr, nloc, static_cast<const T*>(op->Xc), op->n_cols, op->d, V, ldv, w, cps, partial, kf);
  NCGP_LAUNCHED();
  if (epi.active) {
    reduce_splits_epi_kernel<T><<<(unsigned)((nloc + 127) / 128), 128, 0, st>>>(
        partial, splits, nloc, w, epi, out, ldo);
  } else {
    const int64_t tot = nloc * w;
    reduce_splits_kernel<T><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(partial, splits,
                                                                             nloc, w, out, ldo);
  }
  NCGP_LAUNCHED();
  return NCGP_OK;
}

template <typename T, int FAM, int DMAX>
int dispatch_wt(ncgp_kop* op, const T* Xr, int64_t nloc, const T* V, int64_t ldv, int w,
                const ncgp::OutPtrs<T>& out, int64_t ldo, cudaStream_t st, const EpiDev& e) {
  switch (pick_wt(w)) {
    case 1: return launch_t<T, FAM, DMAX, 1>(op, Xr, nloc, V, ldv, w, out, ldo, st, e);
    case 4: return launch_t<T, FAM, DMAX, 4>(op, Xr, nloc, V, ldv, w, out, ldo, st, e);
    case 16: return launch_t<T, FAM, DMAX, 16>(op, Xr, nloc, V, ldv, w, out, ldo, st, e);
    default: return launch_t<T, FAM, DMAX, 32>(op, Xr, nloc, V, ldv, w, out, ldo, st, e);
  }
}

template <typename T, int FAM>
int dispatch_d(ncgp_kop* op, const T* Xr, int64_t nloc, const T* V, int64_t ldv, int w,
               const ncgp::OutPtrs<T>& out, int64_t ldo, cudaStream_t st, const EpiDev& e) {
  switch (pick_dmax(op->d)) {
    case 8: return dispatch_wt<T, FAM, 8>(op, Xr, nloc, V, ldv, w, out, ldo, st, e);
    case 16: return dispatch_wt<T, FAM, 16>(op, Xr, nloc, V, ldv, w, out, ldo, st, e);
    case 32: return dispatch_wt<T, FAM, 32>(op, Xr, nloc, V, ldv, w, out, ldo, st, e);
    default: return dispatch_wt<T, FAM, 64>(op, Xr, nloc, V, ldv, w, out, ldo, st, e);
  }
}

template <typename T>
int dispatch_fam(ncgp_kop* op, const T* Xr, int64_t nloc, const T* V, int64_t ldv, int w,
                 const ncgp::OutPtrs<T>& out, int64_t ldo, cudaStream_t st, const EpiDev& e) {
  if (op->family == NCGP_RBF)
    return dispatch_d<T, NCGP_RBF>(op, Xr, nloc, V, ldv, w, out, ldo, st, e);
  return dispatch_d<T, NCGP_MATERN32>(op, Xr, nloc, V, ldv, w, out, ldo, st, e);
}

}  // namespace

namespace ncgp {

size_t simt_workspace_bytes(int dtype, int64_t n_rows, int64_t n_cols, int d, int w_max) {
  (void)dtype; (void)d;
  // worst case over w <= w_max: splits * n_rows * w doubles, splits <= 64
  size_t best = 0;
  for (int w = 1; w <= w_max; ++w) {
    const int wt = pick_wt(w);
    const int zs = (w + wt - 1) / wt;
    const int splits = plan_splits(n_rows, n_cols, zs, sm_count());
    size_t b = (size_t)splits * n_rows * w * sizeof(double);
    if (b > best) best = b;
  }
  return align_up(best, 256);
}

int simt_apply(ncgp_kop* op, const void* V, int64_t ldv, int w, const OutSet& out, int64_t ldo,
               int64_t r0, int64_t r1, cudaStream_t st, const EpiDev& epi) {
  NCGP_CHECK_ARG(op->d <= 64, NCGP_UNSUPPORTED, "CUDA-core operator supports d <= 64 (got %d)",
                 op->d);
  const int64_t nloc = r1 - r0;
  if (nloc <= 0 || w <= 0) return NCGP_OK;
  if (op->dtype == NCGP_F64) {
    const double* Xr = static_cast<const double*>(op->Xr) + r0 * op->d;
    return dispatch_fam<double>(op, Xr, nloc, static_cast<const double*>(V), ldv, w,
                                out_ptrs<double>(out, r0, ldo), ldo, st, epi);
  }
  const float* Xr = static_cast<const float*>(op->Xr) + r0 * op->d;
  return dispatch_fam<float>(op, Xr, nloc, static_cast<const float*>(V), ldv, w,
                             out_ptrs<float>(out, r0, ldo), ldo, st, epi);
}

}  // namespace ncgp
