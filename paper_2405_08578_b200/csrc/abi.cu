// Library-wide C-ABI entry points: version, errors, launch accounting.
#include <atomic>
#include <cstring>

#include "ps_common.cuh"

namespace ps {
namespace {
thread_local char g_err[512] = {0};
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace ps

extern "C" int ps_abi_version(void) { return PS_ABI_VERSION; }

extern "C" const char* ps_last_error(void) { return ps::g_err; }

extern "C" uint64_t ps_kernel_launches(void) { return ps::g_launches.load(std::memory_order_relaxed); }

extern "C" int ps_device_sync(void* stream) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) {
    ps::set_error("cudaStreamSynchronize: %s", cudaGetErrorString(e));
    return PS_ERR_CUDA;
  }
  return ps::check_cuda("ps_device_sync");
}
