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

// ---- roofline probe: the float64 FMA pipe ------------------------------------
// Each thread runs 8 independent DFMA chains for `iters` steps; the result is
// stored so nothing is dead code.  FLOPs = 2 * 8 * iters * threads.
namespace {
__global__ void __launch_bounds__(256) fp64_fma_probe(int64_t iters, double seed, double* __restrict__ sink) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed + (threadIdx.x + k) * 1e-9;
  const double b = 0.999999999, c = 1e-12;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) sink[blockIdx.x] = s;  // never true; keeps the chains live
}
}  // namespace

extern "C" int ps_probe_fp64_fma(int64_t iters, int32_t blocks, double* sink, double* out_flops, void* stream) {
  PS_REQUIRE(iters > 0 && blocks > 0 && sink && out_flops, PS_ERR_ARGUMENT, "bad probe arguments");
  fp64_fma_probe<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, 1.0, sink);
  PS_LAUNCHED("fp64_fma_probe");
  *out_flops = 2.0 * 8.0 * (double)iters * 256.0 * (double)blocks;
  return ps::check_cuda("fp64_fma_probe");
}
