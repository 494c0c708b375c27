// Kernel-operator plan shared by the tcgen05 and CUDA-core implementations.
#pragma once

#include "common.cuh"

#include <vector>

struct ncgp_kop {
  int impl;      // NCGP_KOP_TCGEN05 | NCGP_KOP_SIMT
  int family;    // NCGP_RBF | NCGP_MATERN32
  int dtype;     // NCGP_F32 | NCGP_F64
  int d;
  double ell, s2;
  int64_t n_rows, n_cols;
  int w_max;
  int sms;
  const void* Xr;  // caller-owned (SIMT path reads it on every apply)
  const void* Xc;
  uint8_t* ws;     // caller-owned workspace
  size_t ws_bytes;
  // ---- tcgen05 path state (see kop_tc.cu) ----
  int ka;               // packed K of the distance GEMM (multiple of 16)
  int wpad;             // padded RHS width of the contraction GEMM
  int64_t row_tiles, col_tiles;
  uint8_t* xa_pack;     // row operand tiles
  uint8_t* col_pack;    // per column tile: [XB | Vhi | Vlo]
  size_t col_tile_bytes;
  double* col_scale;    // per RHS column power-of-two scale (wpad)
  double* partial;      // fp64 partial sums
  double k_scale;       // 2^s prescale of kernel values
  // symmetric kernel (Xr == Xc): work list and int64 fixed-point accumulator (kop_tc.cu)
  int64_t sym_items;
  int4* sym_tab;
  unsigned long long* sym_acc;
  int sym_fx = 0;         // fixed-point fraction bits F of the accumulator (2^-F resolution)
  // tuning / experiment knobs, read once at creation (NCGP_* environment variables)
  int knob_sym = -1;      // NCGP_SYM: -1 policy, 0 off, 1 forced on
  int knob_sym_cg = 0;    // NCGP_SYM_CG: 0 policy, 1, 2 or 3 forced flavour
  int knob_item = 0;      // NCGP_SYM_ITEM: column tiles per work item (0: by problem size, sym_auto_item)
  int knob_item2 = 16;    // NCGP_SYM2_ITEM: the same for the blocked kernel (its O accumulates
                          // in fp32 TMEM over a whole item)
  bool knob_pair_order = false;  // NCGP_SYM_ORDER=pair
  bool knob_atm = true;   // NCGP_SYM_ATM
  int knob_npb = 0;       // NCGP_SYM_NPB (pair kernel), 0 policy
  bool knob_npb1 = false; // NCGP_SYM1_NPB=1 (single-CTA kernel with one P buffer)
  int knob_sym_var = 0;   // NCGP_SYM_DBG bits that keep results correct (64: hold T, 128: TS GEMM2)
  int knob_rings[3] = {0, 0, 0};  // NCGP_RINGS "na,sx,sv" (plain kernel)
  std::vector<int64_t> sym_cum;  // host: tiles before each work item (partition of the list)
  uint8_t* v8_pack = nullptr;  // blocked symmetric kernel: per column tile Vhi in E4M3
  int sym_cg = 2;         // symmetric kernel flavour the work list was built for: 1 single-CTA
                          // (K1-sym1), 2 CTA pairs (K1-sym), 3 blocked single-CTA (K1-sym2)
  int last_variant = -1;  // 0 plain, 1 symmetric pair kernel, 2 symmetric single-CTA kernel,
                          // 3 wide-RHS kernel (K2), 4 blocked symmetric kernel (K1-sym2)
};

// Epilogue of an apply (ncgp_kop_epilogue, include/ncgp_b200.h), with every
// row-indexed pointer already offset to the launch's first row.
struct EpiDev {
  double alpha, beta, gamma;
  const void* base;
  int64_t ldb;
  int noise;         // NCGP_NOISE_*
  const void* ns;    // softmax: pi (rows, w); diag: d (rows * w)
  const void* V;     // the operand's rows i (W^-1 V needs V[i, :]); square operators only
  int64_t ldv;
  void* out2;        // raw K V copy (may be null)
  int64_t ld2;
  int active;        // 0: plain store of K V
};

namespace ncgp {

constexpr double kEpiProbFloor = 1e-12;  // likelihoods.py:22

// One output row of an apply through its epilogue:
//   out = alpha * K V + beta * base + gamma * W^-1 V,  out2 = K V
// kv(c) returns the fp64 product entry (i, c).  The softmax pseudo-inverse
// replays softmax_pinv_apply (likelihoods.py:291-310) in the output dtype.
template <typename T, int NMAX, typename KV>
__device__ __forceinline__ void epi_row(const EpiDev& e, int64_t i, int w, KV kv, T* const* outs,
                                        int n_out, int64_t ldo) {
  if (!e.active) {
    for (int c = 0; c < w; ++c) {
      const T v = (T)kv(c);
#pragma unroll
      for (int k = 0; k < NMAX; ++k)
        if (k < n_out) outs[k][i * ldo + c] = v;
    }
    return;
  }
  const T* Vr = e.V ? static_cast<const T*>(e.V) + i * e.ldv : nullptr;
  const T* pr = e.noise == NCGP_NOISE_SOFTMAX ? static_cast<const T*>(e.ns) + i * w : nullptr;
  T m = 0, m2 = 0;
  if (pr) {
    for (int c = 0; c < w; ++c) m += Vr[c];
    m /= T(w);
    for (int c = 0; c < w; ++c) {
      const T pc = pr[c] > T(kEpiProbFloor) ? pr[c] : T(kEpiProbFloor);
      m2 += (Vr[c] - m) * (T(1) / pc);
    }
    m2 /= T(w);
  }
  for (int c = 0; c < w; ++c) {
    const double k = kv(c);
    if (e.out2) static_cast<T*>(e.out2)[i * e.ld2 + c] = (T)k;
    double r = e.alpha * k;
    if (e.base) r += e.beta * (double)static_cast<const T*>(e.base)[i * e.ldb + c];
    if (pr) {
      const T pc = pr[c] > T(kEpiProbFloor) ? pr[c] : T(kEpiProbFloor);
      r += e.gamma * (double)((Vr[c] - m) * (T(1) / pc) - m2);
    } else if (e.noise == NCGP_NOISE_DIAG) {
      r += e.gamma * (double)(static_cast<const T*>(e.ns)[i * w + c] * Vr[c]);
    }
    const T v = (T)r;
#pragma unroll
    for (int k = 0; k < NMAX; ++k)
      if (k < n_out) outs[k][i * ldo + c] = v;
  }
}

// Destinations of an apply: the caller's output plus, for a row-sharded
// product with the all-gather fused into the store, every peer's (n_rows, w)
// gather buffer mapped into this process (CUDA IPC / symmetric memory).
// Row i of the product is stored to p[k] + i * ldo for every k.
struct OutSet {
  void* p[NCGP_MAX_OUTS];
  int n;
};
template <typename T>
struct OutPtrs {  // typed, already offset to this launch's first row
  T* p[NCGP_MAX_OUTS];
  int n;
};
template <typename T>
inline OutPtrs<T> out_ptrs(const OutSet& o, int64_t r0, int64_t ldo) {
  OutPtrs<T> r{};
  r.n = o.n;
  for (int k = 0; k < o.n; ++k) r.p[k] = static_cast<T*>(o.p[k]) + r0 * ldo;
  return r;
}

// CUDA-core implementation (kop_simt.cu)
size_t simt_workspace_bytes(int dtype, int64_t n_rows, int64_t n_cols, int d, int w_max);
int simt_apply(ncgp_kop* op, const void* V, int64_t ldv, int w, const OutSet& out, int64_t ldo,
               int64_t r0, int64_t r1, cudaStream_t st, const EpiDev& epi);

// Host: the device epilogue of an apply over rows [r0, r1) (pointers offset to r0).
EpiDev make_epi(const ncgp_kop_epilogue* e, const void* V, int64_t ldv, int w, int dtype, int64_t r0);

// tcgen05 implementation (kop_tc.cu)
bool tc_supported(int dtype, int d, int w_max);
size_t tc_workspace_bytes(int64_t n_rows, int64_t n_cols, int d, int w_max);
int tc_prepare(ncgp_kop* op, cudaStream_t st);
// symmetric kernel split over processes: this part's items, contributions left in acc
struct SymPart {
  int part, nparts;
  unsigned long long* acc;
};
int tc_apply(ncgp_kop* op, const void* V, int64_t ldv, int w, const OutSet& out, int64_t ldo,
             int64_t r0, int64_t r1, cudaStream_t st, const EpiDev& epi,
             const SymPart* part = nullptr);
int64_t tc_sym_acc_elems(const ncgp_kop* op, int w);
// K2: posterior marginal variance through the wide kernel's square-reduce
int tc_posterior_var(ncgp_kop* op, const void* W, int64_t ldw, int C, int R, const double* s2,
                     void* var, int64_t ldvar, cudaStream_t st);
int tc_sym_finalize(ncgp_kop* op, const unsigned long long* acc, int w, const OutSet& out,
                    int64_t ldo, cudaStream_t st, const EpiDev& epi, int64_t row_begin = 0,
                    int64_t row_end = -1);

}  // namespace ncgp
