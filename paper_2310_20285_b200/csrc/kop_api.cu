// C ABI of the K1 kernel operator (see include/ncgp_b200.h).
#include <stdio.h>
#include <stdlib.h>

#include <new>

#include "kop.cuh"

namespace ncgp {

EpiDev make_epi(const ncgp_kop_epilogue* e, const void* V, int64_t ldv, int w, int dtype,
                int64_t r0) {
  EpiDev d{};
  d.alpha = 1.0;
  if (e == nullptr) return d;
  const size_t es = dtype == NCGP_F64 ? 8 : 4;
  auto row = [&](const void* p, int64_t ld) -> const void* {
    return p ? static_cast<const uint8_t*>(p) + (size_t)(r0 * ld) * es : nullptr;
  };
  d.alpha = e->alpha;
  d.beta = e->beta;
  d.gamma = e->gamma;
  d.base = row(e->base, e->ldb);
  d.ldb = e->ldb;
  d.noise = e->noise;
  d.ns = e->noise != NCGP_NOISE_NONE ? row(e->noise_state, w) : nullptr;
  d.V = e->noise != NCGP_NOISE_NONE ? row(V, ldv) : nullptr;
  d.ldv = ldv;
  d.out2 = e->out2 ? static_cast<uint8_t*>(e->out2) + (size_t)(r0 * e->ld2) * es : nullptr;
  d.ld2 = e->ld2;
  d.active = 1;
  return d;
}

}  // namespace ncgp

namespace {

// Tuning / experiment knobs (NCGP_* environment variables), read once when
// an operator is created so that an apply never consults the environment.
void read_knobs(ncgp_kop* op) {
  auto env = [](const char* k) -> const char* { return getenv(k); };
  if (const char* e = env("NCGP_SYM")) op->knob_sym = e[0] == '0' ? 0 : (e[0] == '1' ? 1 : -1);
  if (const char* e = env("NCGP_SYM_CG")) op->knob_sym_cg = (e[0] >= '1' && e[0] <= '3') ? e[0] - '0' : 0;
  if (const char* e = env("NCGP_SYM_ITEM")) op->knob_item = atoi(e) > 0 ? atoi(e) : 0;
  if (const char* e = env("NCGP_SYM2_ITEM")) op->knob_item2 = atoi(e) > 0 ? atoi(e) : 16;
  if (const char* e = env("NCGP_SYM_ORDER")) op->knob_pair_order = e[0] == 'p';
  if (const char* e = env("NCGP_SYM_ATM")) op->knob_atm = e[0] != '0';
  if (const char* e = env("NCGP_SYM_NPB")) op->knob_npb = atoi(e);
  if (const char* e = env("NCGP_SYM1_NPB")) op->knob_npb1 = e[0] == '1';
  // only the bits that keep results correct (variants); the timing-only
  // debug bits are honoured by the debug instantiations alone
  if (const char* e = env("NCGP_SYM_DBG")) op->knob_sym_var = atoi(e) & (64 | 128);
  if (const char* e = env("NCGP_RINGS")) {
    int a, b, c;
    if (sscanf(e, "%d,%d,%d", &a, &b, &c) == 3) {
      op->knob_rings[0] = a;
      op->knob_rings[1] = b;
      op->knob_rings[2] = c;
    }
  }
}

int resolve_impl(int impl, int dtype, int d, int w_max) {
  if (impl == NCGP_KOP_AUTO)
    return (dtype == NCGP_F32 && ncgp::tc_supported(dtype, d, w_max)) ? NCGP_KOP_TCGEN05
                                                                       : NCGP_KOP_SIMT;
  return impl;
}

}  // namespace

extern "C" {

size_t ncgp_kop_workspace_bytes(int impl, int dtype, int64_t n_rows, int64_t n_cols, int d,
                                int w_max) {
  const int res = resolve_impl(impl, dtype, d, w_max);
  const size_t simt = ncgp::simt_workspace_bytes(dtype, n_rows, n_cols, d, w_max);
  if (res != NCGP_KOP_TCGEN05) return simt;
  const size_t tc = ncgp::tc_workspace_bytes(n_rows, n_cols, d, w_max);
  // AUTO may fall back to the CUDA-core operator when the inputs fail the
  // tcgen05 precision guard (see ncgp_kop_create): room for either
  return impl == NCGP_KOP_AUTO && simt > tc ? simt : tc;
}

int ncgp_kop_create(ncgp_kop** out, int impl, int family, double lengthscale, double outputscale,
                    int dtype, const void* Xr, int64_t n_rows, const void* Xc, int64_t n_cols,
                    int d, int w_max, void* workspace, size_t workspace_bytes, void* stream) {
  NCGP_CHECK_ARG(out != nullptr, NCGP_INVALID_INPUT, "null output handle");
  *out = nullptr;
  NCGP_CHECK_ARG(family == NCGP_RBF || family == NCGP_MATERN32, NCGP_INVALID_INPUT,
                 "unknown kernel family %d", family);
  NCGP_CHECK_ARG(lengthscale > 0 && lengthscale < 1e300, NCGP_INVALID_INPUT,
                 "lengthscale must be a positive finite real");
  NCGP_CHECK_ARG(outputscale > 0 && outputscale < 1e300, NCGP_INVALID_INPUT,
                 "outputscale must be a positive finite real");
  NCGP_CHECK_ARG(dtype == NCGP_F32 || dtype == NCGP_F64, NCGP_UNSUPPORTED, "dtype %d", dtype);
  NCGP_CHECK_ARG(n_rows >= 0 && n_cols >= 0 && d >= 1 && w_max >= 1, NCGP_DIMENSION_MISMATCH,
                 "bad operator shape rows=%lld cols=%lld d=%d w_max=%d", (long long)n_rows,
                 (long long)n_cols, d, w_max);
  NCGP_CHECK_ARG(Xr != nullptr && Xc != nullptr, NCGP_INVALID_INPUT, "null input matrix");
  const int res = resolve_impl(impl, dtype, d, w_max);
  if (res == NCGP_KOP_TCGEN05)
    NCGP_CHECK_ARG(ncgp::tc_supported(dtype, d, w_max), NCGP_UNSUPPORTED,
                   "tcgen05 operator needs fp32, d <= 64, w_max <= 64 (d=%d w_max=%d)", d, w_max);
  const size_t need = ncgp_kop_workspace_bytes(res, dtype, n_rows, n_cols, d, w_max);
  NCGP_CHECK_ARG(workspace_bytes >= need, NCGP_INVALID_INPUT,
                 "workspace too small: %zu < %zu bytes", workspace_bytes, need);
  ncgp_kop* op = new (std::nothrow) ncgp_kop();
  NCGP_CHECK_ARG(op != nullptr, NCGP_INVALID_INPUT, "host allocation failed");
  op->impl = res;
  op->family = family;
  op->dtype = dtype;
  op->d = d;
  op->ell = lengthscale;
  op->s2 = outputscale;
  op->n_rows = n_rows;
  op->n_cols = n_cols;
  op->w_max = w_max;
  op->sms = ncgp::sm_count();
  op->Xr = Xr;
  op->Xc = Xc;
  op->ws = static_cast<uint8_t*>(workspace);
  op->ws_bytes = workspace_bytes;
  read_knobs(op);
  if (res == NCGP_KOP_TCGEN05) {
    int rc = ncgp::tc_prepare(op, ncgp::as_stream(stream));
    if (rc == NCGP_UNSUPPORTED && impl == NCGP_KOP_AUTO &&
        workspace_bytes >= ncgp::simt_workspace_bytes(dtype, n_rows, n_cols, d, w_max)) {
      // the inputs fail the tcgen05 precision guard: AUTO uses the CUDA-core
      // operator instead (still on the GPU)
      op->impl = NCGP_KOP_SIMT;
      rc = NCGP_OK;
    }
    if (rc != NCGP_OK) {
      delete op;
      return rc;
    }
  }
  *out = op;
  return NCGP_OK;
}

static int kop_apply_outs(ncgp_kop* op, const void* V, int64_t ldv, int w,
                          const ncgp::OutSet& outs, int64_t ldo, int64_t row_begin,
                          int64_t row_end, void* stream,
                          const ncgp_kop_epilogue* epi = nullptr) {
  NCGP_CHECK_ARG(op != nullptr, NCGP_INVALID_INPUT, "null operator");
  NCGP_CHECK_ARG(w >= 0 && w <= op->w_max, NCGP_DIMENSION_MISMATCH,
                 "rhs width %d outside [0, %d]", w, op->w_max);
  NCGP_CHECK_ARG(ldv >= w && ldo >= w, NCGP_DIMENSION_MISMATCH, "leading dimension < width");
  NCGP_CHECK_ARG(0 <= row_begin && row_begin <= row_end && row_end <= op->n_rows,
                 NCGP_DIMENSION_MISMATCH, "row range [%lld, %lld) outside [0, %lld)",
                 (long long)row_begin, (long long)row_end, (long long)op->n_rows);
  NCGP_CHECK_ARG(outs.n >= 1 && outs.n <= NCGP_MAX_OUTS, NCGP_INVALID_INPUT,
                 "%d output buffers (1..%d)", outs.n, NCGP_MAX_OUTS);
  if (w == 0 || row_end == row_begin) return NCGP_OK;
  NCGP_CHECK_ARG(V != nullptr, NCGP_INVALID_INPUT, "null operand");
  for (int k = 0; k < outs.n; ++k)
    NCGP_CHECK_ARG(outs.p[k] != nullptr, NCGP_INVALID_INPUT, "null output %d", k);
  if (epi != nullptr) {
    NCGP_CHECK_ARG(epi->noise >= NCGP_NOISE_NONE && epi->noise <= NCGP_NOISE_DIAG,
                   NCGP_INVALID_INPUT, "unknown noise kind %d", epi->noise);
    NCGP_CHECK_ARG(epi->noise == NCGP_NOISE_NONE || op->n_rows == op->n_cols, NCGP_DIMENSION_MISMATCH,
                   "a noise term needs a square operator (K(X, X)), got %lld x %lld",
                   (long long)op->n_rows, (long long)op->n_cols);
    NCGP_CHECK_ARG(epi->noise == NCGP_NOISE_NONE || epi->noise_state != nullptr, NCGP_INVALID_INPUT,
                   "null noise state");
    NCGP_CHECK_ARG(epi->base == nullptr || epi->ldb >= w, NCGP_DIMENSION_MISMATCH, "ldb < width");
    NCGP_CHECK_ARG(epi->out2 == nullptr || epi->ld2 >= w, NCGP_DIMENSION_MISMATCH, "ld2 < width");
  }
  const EpiDev ed = ncgp::make_epi(epi, V, ldv, w, op->dtype, row_begin);
  if (op->n_cols == 0) {
    NCGP_CHECK_ARG(epi == nullptr, NCGP_UNSUPPORTED, "epilogue of an empty operator");
    // empty sum: zero output rows
    const size_t es = op->dtype == NCGP_F64 ? 8 : 4;
    for (int k = 0; k < outs.n; ++k)
      NCGP_CUDA(cudaMemset2DAsync(static_cast<uint8_t*>(outs.p[k]) + row_begin * ldo * es,
                                  ldo * es, 0, w * es, row_end - row_begin,
                                  ncgp::as_stream(stream)));
    return NCGP_OK;
  }
  if (op->impl == NCGP_KOP_TCGEN05)
    return ncgp::tc_apply(op, V, ldv, w, outs, ldo, row_begin, row_end, ncgp::as_stream(stream), ed);
  op->last_variant = 0;
  return ncgp::simt_apply(op, V, ldv, w, outs, ldo, row_begin, row_end, ncgp::as_stream(stream), ed);
}

int ncgp_kop_apply_ex(ncgp_kop* op, const void* V, int64_t ldv, int w, void* out, int64_t ldo,
                      int64_t row_begin, int64_t row_end, const ncgp_kop_epilogue* epi,
                      void* stream) {
  ncgp::OutSet o{};
  o.p[0] = out;
  o.n = 1;
  return kop_apply_outs(op, V, ldv, w, o, ldo, row_begin, row_end, stream, epi);
}

int ncgp_kop_apply(ncgp_kop* op, const void* V, int64_t ldv, int w, void* out, int64_t ldo,
                   int64_t row_begin, int64_t row_end, void* stream) {
  ncgp::OutSet o{};
  o.p[0] = out;
  o.n = 1;
  return kop_apply_outs(op, V, ldv, w, o, ldo, row_begin, row_end, stream);
}

int ncgp_kop_apply_multi(ncgp_kop* op, const void* V, int64_t ldv, int w, void* const* outs,
                         int n_out, int64_t ldo, int64_t row_begin, int64_t row_end,
                         void* stream) {
  NCGP_CHECK_ARG(outs != nullptr, NCGP_INVALID_INPUT, "null output list");
  NCGP_CHECK_ARG(n_out >= 1 && n_out <= NCGP_MAX_OUTS, NCGP_INVALID_INPUT,
                 "%d output buffers (1..%d)", n_out, NCGP_MAX_OUTS);
  ncgp::OutSet o{};
  for (int k = 0; k < n_out; ++k) o.p[k] = outs[k];
  o.n = n_out;
  return kop_apply_outs(op, V, ldv, w, o, ldo, row_begin, row_end, stream);
}

int ncgp_kop_impl(const ncgp_kop* op) { return op ? op->impl : -1; }

int ncgp_kop_set_sym(ncgp_kop* op, int mode) {
  NCGP_CHECK_ARG(op != nullptr, NCGP_INVALID_INPUT, "null operator");
  NCGP_CHECK_ARG(mode >= -1 && mode <= 1, NCGP_INVALID_INPUT, "symmetric mode %d not in {-1, 0, 1}", mode);
  op->knob_sym = mode;
  return NCGP_OK;
}

int64_t ncgp_kop_sym_acc_elems(const ncgp_kop* op, int w) {
  if (op == nullptr || op->impl != NCGP_KOP_TCGEN05 || w < 1 || w > op->w_max) return 0;
  return ncgp::tc_sym_acc_elems(op, w);
}

int ncgp_kop_sym_partial(ncgp_kop* op, const void* V, int64_t ldv, int w, int part, int nparts,
                         int64_t* acc, int64_t acc_elems, void* stream) {
  NCGP_CHECK_ARG(op != nullptr && V != nullptr && acc != nullptr, NCGP_INVALID_INPUT,
                 "null argument");
  NCGP_CHECK_ARG(ldv >= w, NCGP_DIMENSION_MISMATCH, "leading dimension < width");
  const int64_t need = ncgp_kop_sym_acc_elems(op, w);
  NCGP_CHECK_ARG(need > 0, NCGP_UNSUPPORTED, "no symmetric kernel for this operator and width %d", w);
  NCGP_CHECK_ARG(acc_elems >= need, NCGP_DIMENSION_MISMATCH, "accumulator has %lld elements, need %lld",
                 (long long)acc_elems, (long long)need);
  ncgp::OutSet none{};
  none.n = 0;
  const ncgp::SymPart sp{part, nparts, reinterpret_cast<unsigned long long*>(acc)};
  const EpiDev ed = ncgp::make_epi(nullptr, V, ldv, w, op->dtype, 0);
  return ncgp::tc_apply(op, V, ldv, w, none, w, 0, op->n_rows, ncgp::as_stream(stream), ed, &sp);
}

int ncgp_kop_sym_finalize_rows(ncgp_kop* op, const int64_t* acc, int64_t acc_elems, const void* V,
                               int64_t ldv, int w, void* out, int64_t ldo,
                               const ncgp_kop_epilogue* epi, int64_t row_begin, int64_t row_end,
                               void* stream) {
  NCGP_CHECK_ARG(op != nullptr && acc != nullptr && out != nullptr, NCGP_INVALID_INPUT,
                 "null argument");
  NCGP_CHECK_ARG(ldo >= w, NCGP_DIMENSION_MISMATCH, "leading dimension < width");
  NCGP_CHECK_ARG(row_begin >= 0 && row_begin <= row_end && row_end <= op->n_rows,
                 NCGP_DIMENSION_MISMATCH, "row range [%lld, %lld) outside [0, %lld]",
                 (long long)row_begin, (long long)row_end, (long long)op->n_rows);
  const int64_t need = ncgp_kop_sym_acc_elems(op, w);
  NCGP_CHECK_ARG(need > 0, NCGP_UNSUPPORTED, "no symmetric kernel for this operator and width %d", w);
  NCGP_CHECK_ARG(acc_elems >= need, NCGP_DIMENSION_MISMATCH, "accumulator has %lld elements, need %lld",
                 (long long)acc_elems, (long long)need);
  if (epi != nullptr) {
    NCGP_CHECK_ARG(epi->noise == NCGP_NOISE_NONE || (V != nullptr && ldv >= w && epi->noise_state),
                   NCGP_INVALID_INPUT, "a noise term needs the operand V and its noise state");
    NCGP_CHECK_ARG(epi->noise >= NCGP_NOISE_NONE && epi->noise <= NCGP_NOISE_DIAG,
                   NCGP_INVALID_INPUT, "unknown noise kind %d", epi->noise);
  }
  ncgp::OutSet o{};
  o.p[0] = out;
  o.n = 1;
  const EpiDev ed = ncgp::make_epi(epi, V, ldv, w, op->dtype, 0);
  return ncgp::tc_sym_finalize(op, reinterpret_cast<const unsigned long long*>(acc), w, o, ldo,
                               ncgp::as_stream(stream), ed, row_begin, row_end);
}

int ncgp_kop_sym_finalize(ncgp_kop* op, const int64_t* acc, int64_t acc_elems, const void* V,
                          int64_t ldv, int w, void* out, int64_t ldo,
                          const ncgp_kop_epilogue* epi, void* stream) {
  NCGP_CHECK_ARG(op != nullptr, NCGP_INVALID_INPUT, "null argument");
  return ncgp_kop_sym_finalize_rows(op, acc, acc_elems, V, ldv, w, out, ldo, epi, 0, op->n_rows,
                                    stream);
}

int ncgp_kop_posterior_var(ncgp_kop* op, const void* W, int64_t ldw, int C, int R,
                           const double* s2, void* var, int64_t ldvar, void* stream) {
  NCGP_CHECK_ARG(op != nullptr && W != nullptr && s2 != nullptr && var != nullptr,
                 NCGP_INVALID_INPUT, "null argument");
  NCGP_CHECK_ARG(op->impl == NCGP_KOP_TCGEN05 && op->w_max > 32, NCGP_UNSUPPORTED,
                 "the posterior kernel needs a tcgen05 operator created with w_max > 32");
  if (op->n_rows == 0) return NCGP_OK;
  NCGP_CHECK_ARG(op->n_cols > 0, NCGP_UNSUPPORTED, "empty training set");
  return ncgp::tc_posterior_var(op, W, ldw, C, R, s2, var, ldvar, ncgp::as_stream(stream));
}

int ncgp_kop_last_variant(const ncgp_kop* op) { return op ? op->last_variant : -1; }

int ncgp_kop_destroy(ncgp_kop* op) {
  delete op;
  return NCGP_OK;
}

}  // extern "C"
