// tcgen05 / TMEM fused kernel-matmul -- placeholder until the kernel lands.
#include "kop.cuh"

namespace ncgp {

bool tc_supported(int, int, int) { return false; }
size_t tc_workspace_bytes(int64_t, int64_t, int, int) { return 0; }
int tc_prepare(ncgp_kop*, cudaStream_t) {
  set_error("tcgen05 operator not built");
  return NCGP_UNSUPPORTED;
}
int tc_apply(ncgp_kop*, const void*, int64_t, int, void*, int64_t, int64_t, int64_t,
             cudaStream_t) {
  set_error("tcgen05 operator not built");
  return NCGP_UNSUPPORTED;
}

}  // namespace ncgp
