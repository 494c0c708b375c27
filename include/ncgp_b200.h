/*
 * ncgp_b200.h -- C ABI of the B200-native IterNCGP hot path (libncgp_b200.so).
 *
 * The reference package ``ncgp`` is pure Python; the seam this library
 * replaces is its operator plug-in boundary:
 *
 *   RegressionSystem(apply_kernel, apply_noise, rhs)      solver.py:42-57
 *   apply_kernel = prior_matvec(prior, X, ., tile)          outer.py:180-181, gp.py:144-172
 *   apply_noise  = likelihood.w_inv_matvec(f, .)           outer.py:186, likelihoods.py:258-262
 *
 * Every entry point below names the reference function it replaces.
 *
 * Conventions
 *  - Every function returns an int status: NCGP_OK (0) or one of
 *    NCGP_DIMENSION_MISMATCH (1, -> ncgp.DimensionMismatch), NCGP_INVALID_INPUT
 *    (2, -> ncgp.InvalidInput), NCGP_CUDA_ERROR (3), NCGP_UNSUPPORTED (4).
 *    ncgp_last_error() returns a thread-local message for the last failure.
 *  - All array arguments are caller-owned DEVICE pointers; the library does
 *    no device allocation on the hot path.  Scratch space is passed in as a
 *    ``workspace`` sized by the matching *_workspace_bytes query.
 *  - All work is enqueued on the caller's ``stream`` (a cudaStream_t passed
 *    as void*; NULL = legacy default stream).  Nothing synchronises except
 *    functions documented as blocking.
 *  - ``dtype`` selects NCGP_F32 (float) or NCGP_F64 (double) for every
 *    floating-point array of the call.  Reductions accumulate in fp64 with
 *    a fixed order, so results are deterministic run to run.
 *  - Vectors over (point, output) pairs use the reference's CN layout
 *    (gp.py:4-8): entry n*C + c, i.e. an N x C row-major matrix.
 *  - Column blocks (solver buffers S, T, Q) are stored column-contiguous:
 *    column b starts at ptr + b * ld.
 *  - Operators are bound to the device current at creation; an operator
 *    must not be used by two host threads at once.
 */
#ifndef NCGP_B200_H
#define NCGP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  NCGP_OK = 0,
  NCGP_DIMENSION_MISMATCH = 1,
  NCGP_INVALID_INPUT = 2,
  NCGP_CUDA_ERROR = 3,
  NCGP_UNSUPPORTED = 4
};

enum { NCGP_F32 = 0, NCGP_F64 = 1 };
enum { NCGP_RBF = 0, NCGP_MATERN32 = 1 };

/* Kernel-operator implementation selector (NCGP_KOP_AUTO picks the tcgen05
 * path for fp32 and the fp64 CUDA-core path for fp64). */
enum { NCGP_KOP_AUTO = 0, NCGP_KOP_TCGEN05 = 1, NCGP_KOP_SIMT = 2 };

const char* ncgp_last_error(void);
int ncgp_version(void);
/* Blocking: queries the current device. */
int ncgp_device_info(int* sm_count, int* cc_major, int* cc_minor);
/* Number of kernels this library has launched in this process. */
int64_t ncgp_launch_count(void);

/* ---------------------------------------------------------------------
 * K1 fused kernel-matmul (replaces prior_matvec gp.py:144-172 with the
 * tile body gp.py:162-171, _sqdist gp.py:101-113, kernel_from_sqdist
 * gp.py:78-98; newton_update outer.py:134-137; and, with X_rows =
 * X_test, the dense cross_covariance products of posterior.py:52-84).
 *
 *   out[i, c] = sum_j k(Xr[i], Xc[j]) * V[j, c]      0 <= i < n_rows, c < w
 *
 * for one stationary kernel (family, lengthscale, outputscale).  K is never
 * materialised.  Xr: (n_rows, d) row-major, Xc: (n_cols, d) row-major,
 * V: (n_cols, w) with row stride ldv, out: (n_rows, w) with row stride ldo.
 * ------------------------------------------------------------------- */
typedef struct ncgp_kop ncgp_kop;

size_t ncgp_kop_workspace_bytes(int impl, int dtype, int64_t n_rows,
                                int64_t n_cols, int d, int w_max);

/* Packs Xr / Xc into the operator's tiled layout (enqueued on stream). */
int ncgp_kop_create(ncgp_kop** op, int impl, int family, double lengthscale,
                    double outputscale, int dtype, const void* Xr,
                    int64_t n_rows, const void* Xc, int64_t n_cols, int d,
                    int w_max, void* workspace, size_t workspace_bytes,
                    void* stream);

/* out[row_begin:row_end, :w] = K(Xr[row_begin:row_end], Xc) V.
 * row_begin must be a multiple of 256 (a row-tile pair) for row sharding. */
int ncgp_kop_apply(ncgp_kop* op, const void* V, int64_t ldv, int w,
                   void* out, int64_t ldo, int64_t row_begin,
                   int64_t row_end, void* stream);

/* Row-sharded apply with the all-gather fused into the store (SURVEY.md
 * 8(e); replaces ncgp_kop_apply + an all-gather of the output rows).  Rows
 * [row_begin, row_end) of K V are stored, at their global row offsets, into
 * every buffer outs[0..n_out): this rank's own (n_rows, w) output and the
 * gather buffers of its peers mapped into this process (CUDA IPC / symmetric
 * memory over NVLink), so the exchange overlaps the kernel instead of
 * following it.  `outs` is a host array of device pointers; all buffers
 * share the row stride ldo.  The caller orders the peers' reads after this
 * stream (a cross-rank barrier).  1 <= n_out <= NCGP_MAX_OUTS. */
#define NCGP_MAX_OUTS 8
int ncgp_kop_apply_multi(ncgp_kop* op, const void* V, int64_t ldv, int w,
                         void* const* outs, int n_out, int64_t ldo,
                         int64_t row_begin, int64_t row_end, void* stream);

/* Fused epilogue of an apply (SURVEY.md 2.3, K1 "optional epilogues"):
 *
 *   out  = alpha * (K V) + beta * base + gamma * (W^-1 V)
 *   out2 = K V                                   (optional raw product)
 *
 * evaluated per output row inside K1's reduction pass, so the Newton-step
 * operator K^ = K + W^-1 (W^+ for softmax) is applied without a second pass
 * over K V.  It replaces, in one call,
 *   - t = apply_kernel(s); z = t + apply_noise(s)          solver.py:262,265
 *     (alpha 1, gamma 1, out2 = t),
 *   - r = rhs - apply_kernel(v) - apply_noise(v)            solver.py:249
 *     (alpha -1, beta 1, base = rhs, gamma -1),
 *   - f = prior_matvec(w) + m                               outer.py:134-137
 *     (alpha 1, beta 1, base = m, out2 = g = K w).
 * noise = NCGP_NOISE_SOFTMAX: W^+ from the cached probabilities pi (n_rows,
 * w) row-major (softmax_pinv_apply, likelihoods.py:291-310; w = C);
 * NCGP_NOISE_DIAG: diagonal W^-1 d (n_rows * w, CN), e.g. Bernoulli
 * (likelihoods.py:210-212) or Gaussian noise variances (likelihoods.py:109).
 * The noise term needs V's row i next to output row i, so it is only valid
 * for square operators (K(X, X)).  base / out2 / noise_state are indexed by
 * the apply's global rows with strides ldb / ld2 (noise_state dense).
 * A NULL epilogue is the plain product (alpha 1, nothing else). */
enum { NCGP_NOISE_NONE = 0, NCGP_NOISE_SOFTMAX = 1, NCGP_NOISE_DIAG = 2 };
typedef struct ncgp_kop_epilogue {
  double alpha, beta, gamma;
  const void* base;        /* NULL: beta ignored */
  int64_t ldb;
  int noise;               /* NCGP_NOISE_*; NONE: gamma ignored */
  const void* noise_state; /* pi (softmax) or d (diagonal) */
  void* out2;              /* NULL: no raw copy */
  int64_t ld2;
} ncgp_kop_epilogue;

int ncgp_kop_apply_ex(ncgp_kop* op, const void* V, int64_t ldv, int w,
                      void* out, int64_t ldo, int64_t row_begin,
                      int64_t row_end, const ncgp_kop_epilogue* epi,
                      void* stream);

/* The symmetric K(X, X) kernel split across `nparts` processes (SURVEY.md
 * 8(e); no reference counterpart: the reference has no multi-GPU path).
 *
 * The symmetric kernels accumulate in int64 fixed point (2^-F resolution in
 * the kernel's scaled domain, F fixed by n): integer addition is associative,
 * so the product is bitwise identical run to run, for any CTA schedule and
 * for any number of parts -- the property the reference pins with its
 * tile-size invariance (gp.py:144-172 "bit-identical for any tile size",
 * test_gp.py:106-110).
 *
 * ncgp_kop_sym_acc_elems: int64 elements of the per-process accumulator for
 * RHS width w, or 0 when a full apply of width w would not use a symmetric
 * kernel (rectangular operator, too small, or the shape does not fit); the
 * caller then row-shards with row_begin / row_end.
 * ncgp_kop_sym_partial: part `part` of `nparts` slices of the triangular work
 * list (equal tile counts) into `acc` (acc_elems >= ncgp_kop_sym_acc_elems;
 * zeroed first, on `stream`).  The integer sum of all parts' acc (an
 * all-reduce with int64 SUM) is the full product in a padded, swizzled
 * layout; ncgp_kop_sym_finalize writes the (n_rows, w) product with row
 * stride ldo through the epilogue (V: the operand, needed only for a noise
 * term; epi may be NULL).  Errors: NCGP_UNSUPPORTED when
 * ncgp_kop_sym_acc_elems is 0, NCGP_DIMENSION_MISMATCH when acc_elems is
 * too small. */
int64_t ncgp_kop_sym_acc_elems(const ncgp_kop* op, int w);
int ncgp_kop_sym_partial(ncgp_kop* op, const void* V, int64_t ldv, int w, int part,
                         int nparts, int64_t* acc, int64_t acc_elems, void* stream);
int ncgp_kop_sym_finalize(ncgp_kop* op, const int64_t* acc, int64_t acc_elems,
                          const void* V, int64_t ldv, int w, void* out, int64_t ldo,
                          const ncgp_kop_epilogue* epi, void* stream);
/* The same for rows [row_begin, row_end) only: the finalize of a process that
 * keeps a row shard of the solver state.  out, V and the
 * epilogue's base / out2 / noise_state stay indexed by the operator's global
 * rows, as in ncgp_kop_apply_ex; only rows of the range are read or written,
 * so a caller holding just its shard passes (shard pointer - row_begin * ld). */
int ncgp_kop_sym_finalize_rows(ncgp_kop* op, const int64_t* acc, int64_t acc_elems,
                               const void* V, int64_t ldv, int w, void* out, int64_t ldo,
                               const ncgp_kop_epilogue* epi, int64_t row_begin,
                               int64_t row_end, void* stream);

/* Symmetric-kernel policy of an operator (no reference counterpart): -1 the
 * default size policy, 0 always the plain tiled kernel, 1 a symmetric kernel
 * whenever one fits (K(X, X) launches over all rows).  Both give correct
 * products; the plain kernel's fp64-flushed rows and the symmetric kernels'
 * int64 sums are each bitwise reproducible, but they differ from each other
 * in the last bits.  The initial mode comes from NCGP_SYM (read at creation). */
int ncgp_kop_set_sym(ncgp_kop* op, int mode);

/* K2 fused cross-kernel posterior variance (replaces posterior_marginal_var,
 * posterior.py:67-84, and its dense cross_covariance, gp.py:175-196):
 *
 *   var[t, c] = max(s2[c] - sum_{r<R} (sum_j k(Xr[t], Xc[j]) W[j, c*R + r])^2, 0)
 *
 * for the operator's rows t (test points) and C outputs sharing its kernel
 * spec.  W is (n_cols, C*R) with row stride ldw: the class-major root
 * [Q_0 | ... | Q_{C-1}], Q_c[j, r] = Q[j*C + c, r].  Each kernel tile is
 * evaluated once per 128 root columns (not per 32), its product with the
 * root accumulates in TMEM over <= 2048 training points, and the fp32
 * partials are summed in fp64 in a fixed order and squared per row -- A is
 * never materialised.  s2: device fp64 [C]; var: (n_rows, C) row stride
 * ldvar, in the operator's dtype.  Needs a tcgen05 operator created with
 * w_max > 32 (else NCGP_UNSUPPORTED; callers then use the product path). */
int ncgp_kop_posterior_var(ncgp_kop* op, const void* W, int64_t ldw, int C,
                           int R, const double* s2, void* var, int64_t ldvar,
                           void* stream);

/* Actual implementation chosen (NCGP_KOP_TCGEN05 or NCGP_KOP_SIMT). */
int ncgp_kop_impl(const ncgp_kop* op);
/* Kernel variant of the last apply (telemetry, no reference counterpart):
 * 0 = plain tiled product, 1 = symmetric K(X, X) kernel on CTA pairs, 2 =
 * symmetric K(X, X) kernel on single CTAs (each off-diagonal tile evaluated
 * once, serving both K V and K^T V), 3 = wide-RHS kernel (32 < w <= 128,
 * K2), -1 = none yet. */
int ncgp_kop_last_variant(const ncgp_kop* op);
int ncgp_kop_destroy(ncgp_kop* op);

/* ---------------------------------------------------------------------
 * K3/K4/K5 likelihood kernels.
 * ------------------------------------------------------------------- */

/* Softmax per-point statistics (likelihoods.py:235-238 probabilities,
 * :285-288 softmax_rows, :247-250 grad_log_lik, outer.py:129-131
 * pseudo_targets).  f, grad, yhat: CN (n*C); pi: (n, C).  grad / yhat may
 * be NULL. */
int ncgp_softmax_stats(int dtype, const void* f, const int64_t* labels,
                       int64_t n, int C, void* pi, void* grad, void* yhat,
                       void* stream);

/* out[:, b] = beta * base[:, b] + alpha * (W(f)^+ V[:, b])  for b < k
 * with W^+ the blockwise softmax pseudo-inverse (likelihoods.py:291-310,
 * via w_inv_matvec :258-262).  V, base, out: column blocks of length n*C.
 * base may be NULL (then beta is ignored). */
int ncgp_softmax_winv(int dtype, const void* pi, int64_t n, int C,
                      const void* V, int64_t ldv, int k, const void* base,
                      int64_t ldb, double alpha, double beta, void* out,
                      int64_t ldo, void* stream);

/* W_n products (diag(pi_n) - pi_n pi_n') v_n (likelihoods.py:252-256). */
int ncgp_softmax_w(int dtype, const void* pi, int64_t n, int C,
                   const void* V, int64_t ldv, int k, void* out, int64_t ldo,
                   void* stream);

/* Bernoulli-logit statistics (likelihoods.py:202-212, outer.py:129-131):
 * winv = 1/(s(1-s)) with the reference's clamp, w = s(1-s),
 * grad = y - s, yhat = f + winv * grad.  Any output may be NULL. */
int ncgp_bernoulli_stats(int dtype, const void* f, const int64_t* labels,
                         int64_t n, void* winv, void* w, void* grad,
                         void* yhat, void* stream);

/* Poisson log-link statistics (likelihoods.py:174-182, outer.py:129-131):
 * w = exp(f), winv = exp(-f), grad = y - exp(f), yhat = f + winv * grad;
 * counts in the working dtype.  Any output may be NULL. */
int ncgp_poisson_stats(int dtype, const void* f, const void* counts, int64_t n,
                       void* winv, void* w, void* grad, void* yhat,
                       void* stream);

/* out[:, b] = beta * base[:, b] + alpha * diag(dvec) V[:, b]
 * (_apply_diag likelihoods.py:149-153). */
int ncgp_diag_apply(int dtype, const void* dvec, int64_t n, const void* V,
                    int64_t ldv, int k, const void* base, int64_t ldb,
                    double alpha, double beta, void* out, int64_t ldo,
                    void* stream);

/* ---------------------------------------------------------------------
 * K6 vector / tall-skinny kernels for the inner solver (solver.py:203-331,
 * linalg.py:51-62).  Reductions write fp64 results to DEVICE memory.
 * ------------------------------------------------------------------- */

size_t ncgp_reduce_workspace_bytes(int64_t n, int k);

/* out[p] = sum_i x_p[i] * y_p[i] for p < npairs (npairs <= 4); xs / ys are
 * HOST arrays of device pointers. */
int ncgp_dots(int dtype, int64_t n, int npairs, const void* const* xs,
              const void* const* ys, double* out, void* workspace,
              size_t workspace_bytes, void* stream);

/* out[r] = sum_i Q[r*ldq + i] * z[i]  for r < k   (Q' z, linalg.py:62). */
int ncgp_gemv_t(int dtype, const void* Q, int64_t ldq, int k, const void* z,
                int64_t n, double* out, void* workspace,
                size_t workspace_bytes, void* stream);

/* out[i] = s[i] + alpha * sum_r Q[r*ldq + i] * y[r]   (y: device fp64). */
int ncgp_gemv_n(int dtype, const void* Q, int64_t ldq, int k,
                const double* y, const void* s, double alpha, void* out,
                int64_t n, void* stream);

/* out = a*x + b*y + c*z (any of y, z may be NULL). */
int ncgp_lincomb(int dtype, int64_t n, double a, const void* x, double b,
                 const void* y, double c, const void* z, void* out,
                 void* stream);

/* M[a*ldm + b] = sum_i S[a*lds + i] * Y[b*ldy + i] for a < ka, b < kb,
 * fp64 result (the recycled Gram S'(T + W^+ S), solver.py:311). */
size_t ncgp_gram_workspace_bytes(int64_t n, int ka, int kb);
int ncgp_gram(int dtype, const void* S, int64_t lds, int ka, const void* Y,
              int64_t ldy, int kb, int64_t n, double* M, int64_t ldm,
              void* workspace, size_t workspace_bytes, void* stream);

/* out[c*ldo + i] = sum_b S[b*lds + i] * U[b*ldu + c]  for c < kc
 * (buffer rotation S U, T U, S diag(l)^-1/2: solver.py:325-330).  U is a
 * device fp64 (kb x kc) matrix with row stride ldu. */
int ncgp_rotate(int dtype, const void* S, int64_t lds, int kb,
                const double* U, int64_t ldu, int kc, void* out, int64_t ldo,
                int64_t n, void* stream);

/* ---------------------------------------------------------------------
 * K2 posterior helpers (posterior.py:52-84).
 * ------------------------------------------------------------------- */

/* var[t*C + c] = max(s2[c] - sum_{r<R} A[t*lda + c*R + r]^2, 0);
 * s2: device fp64 array of C prior variances. */
int ncgp_marginal_var(int dtype, const void* A, int64_t lda, int64_t nt,
                      int C, int R, const double* s2, void* var,
                      void* stream);

#ifdef __cplusplus
}
#endif

#endif /* NCGP_B200_H */
