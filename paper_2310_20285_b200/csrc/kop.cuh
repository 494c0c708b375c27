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
  // symmetric kernel (Xr == Xc): work list and fp32 accumulator (kop_tc.cu)
  int64_t sym_items;
  int4* sym_tab;
  float* sym_acc;
  std::vector<int64_t> sym_cum;  // host: tiles before each work item (partition of the list)
  int sym_cg = 2;         // symmetric kernel flavour the work list was built for (1 or 2)
  int last_variant = -1;  // 0 plain, 1 symmetric pair kernel, 2 symmetric single-CTA kernel
};

namespace ncgp {

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
               int64_t r0, int64_t r1, cudaStream_t st);

// tcgen05 implementation (kop_tc.cu)
bool tc_supported(int dtype, int d, int w_max);
size_t tc_workspace_bytes(int64_t n_rows, int64_t n_cols, int d, int w_max);
int tc_prepare(ncgp_kop* op, cudaStream_t st);
// symmetric kernel split over processes: this part's items, contributions left in acc
struct SymPart {
  int part, nparts;
  float* acc;
};
int tc_apply(ncgp_kop* op, const void* V, int64_t ldv, int w, const OutSet& out, int64_t ldo,
             int64_t r0, int64_t r1, cudaStream_t st, const SymPart* part = nullptr);
int64_t tc_sym_acc_elems(const ncgp_kop* op, int w);
int tc_sym_finalize(ncgp_kop* op, const float* acc, int w, const OutSet& out, int64_t ldo,
                    cudaStream_t st);

}  // namespace ncgp
