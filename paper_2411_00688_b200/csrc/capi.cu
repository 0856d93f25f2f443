// Library-level C ABI: version, thread-local error message, device query.
#include "common.cuh"

namespace psb {

namespace {
thread_local std::string g_err;
}

void set_error(const std::string& msg) { g_err = msg; }

int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}

int sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      cached = n;
    else
      cached = 148;
  }
  return cached;
}

}  // namespace psb

extern "C" {

int psb_abi_version(void) { return PSB_ABI_VERSION; }

const char* psb_last_error(void) { return psb::g_err.c_str(); }

int psb_device_sm_count(int* out) {
  int dev = 0;
  PSB_CUDA(cudaGetDevice(&dev));
  PSB_CUDA(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev));
  return PSB_OK;
}

}  // extern "C"
