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

// ------------------------------------------------------------------ peer buffers (CUDA IPC)
// ssr_exchange_adam reads and writes other ranks' buffers directly.  A rank
// exports (handle of the buffer's allocation, offset inside it); every other
// rank opens the handle on its own device with lazy peer access, so its
// kernels address the exporter's memory over NVLink / NVSwitch.  Opened
// allocations are reference-counted per handle: two buffers of one allocation
// share one mapping.
#include <cstring>
#include <map>
#include <mutex>

namespace {
typedef int (*AddrRangeFn)(unsigned long long*, size_t*, unsigned long long);  // cuMemGetAddressRange_v2

struct Opened {
  void* base;
  int refs;
};
std::mutex g_ipc_mu;
std::map<std::string, Opened> g_ipc;  // handle bytes -> mapping
}  // namespace

extern "C" int ssr_ipc_export(const void* ptr, uint8_t* handle, int64_t* offset) {
  if (!ptr || !handle || !offset) {
    ssr::set_error("ssr_ipc_export: invalid argument");
    return SSR_ERR_INVALID;
  }
  static AddrRangeFn range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    SSR_TRY(ssr::check_cuda(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q),
                            "cuMemGetAddressRange entry point"));
    if (!fn || q != cudaDriverEntryPointSuccess) {
      ssr::set_error("ssr_ipc_export: cuMemGetAddressRange unavailable");
      return SSR_ERR_CUDA;
    }
    range = (AddrRangeFn)fn;
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, (unsigned long long)ptr) != 0) {
    ssr::set_error("ssr_ipc_export: cuMemGetAddressRange failed (not a device allocation)");
    return SSR_ERR_CUDA;
  }
  cudaIpcMemHandle_t h;
  SSR_TRY(ssr::check_cuda(cudaIpcGetMemHandle(&h, (void*)base), "cudaIpcGetMemHandle"));
  static_assert(sizeof(h) == SSR_IPC_HANDLE_BYTES, "cudaIpcMemHandle_t size");
  std::memcpy(handle, &h, sizeof h);
  *offset = (int64_t)((unsigned long long)ptr - base);
  return SSR_OK;
}

extern "C" int ssr_ipc_open(const uint8_t* handle, int64_t offset, void** ptr) {
  if (!handle || !ptr || offset < 0) {
    ssr::set_error("ssr_ipc_open: invalid argument");
    return SSR_ERR_INVALID;
  }
  const std::string key((const char*)handle, SSR_IPC_HANDLE_BYTES);
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto it = g_ipc.find(key);
  if (it == g_ipc.end()) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void* base = nullptr;
    SSR_TRY(ssr::check_cuda(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess),
                            "cudaIpcOpenMemHandle"));
    it = g_ipc.emplace(key, Opened{base, 0}).first;
  }
  it->second.refs++;
  *ptr = (char*)it->second.base + offset;
  return SSR_OK;
}

extern "C" int ssr_ipc_close(const uint8_t* handle) {
  if (!handle) {
    ssr::set_error("ssr_ipc_close: invalid argument");
    return SSR_ERR_INVALID;
  }
  const std::string key((const char*)handle, SSR_IPC_HANDLE_BYTES);
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto it = g_ipc.find(key);
  if (it == g_ipc.end()) return SSR_OK;
  if (--it->second.refs == 0) {
    // the exporter may already have released the allocation: not an error here
    cudaIpcCloseMemHandle(it->second.base);
    cudaGetLastError();
    g_ipc.erase(it);
  }
  return SSR_OK;
}
