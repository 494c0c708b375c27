// Error plumbing, launch counting and device queries for libncgp_b200.
#include <stdarg.h>

#include "common.cuh"

namespace ncgp {

static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

std::atomic<int64_t>& launch_counter() { return g_launches; }

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

}  // namespace ncgp

extern "C" {

const char* ncgp_last_error(void) { return ncgp::g_err; }

int ncgp_version(void) { return 1; }

int64_t ncgp_launch_count(void) { return ncgp::g_launches.load(); }

int ncgp_device_info(int* sms, int* major, int* minor) {
  int dev = 0;
  NCGP_CUDA(cudaGetDevice(&dev));
  if (sms) NCGP_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
  if (major) NCGP_CUDA(cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev));
  if (minor) NCGP_CUDA(cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev));
  return NCGP_OK;
}

}  // extern "C"
