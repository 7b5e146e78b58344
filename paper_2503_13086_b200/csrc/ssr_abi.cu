// C-ABI utilities: per-thread error string, version, device query.
#include <cstdio>
#include <string>

#include "ssr_common.cuh"

namespace ssr {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SSR_OK;
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return SSR_ERR_CUDA;
}

int check_launch(const char* what) { return check_cuda(cudaGetLastError(), what); }

}  // namespace ssr

extern "C" const char* ssr_last_error(void) { return ssr::g_err.c_str(); }

extern "C" int ssr_version(void) { return 1; }

extern "C" int ssr_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
  int dev = 0;
  SSR_TRY(ssr::check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
  cudaDeviceProp p;
  SSR_TRY(ssr::check_cuda(cudaGetDeviceProperties(&p, dev), "cudaGetDeviceProperties"));
  *sm_count = p.multiProcessorCount;
  *cc_major = p.major;
  *cc_minor = p.minor;
  return SSR_OK;
}
