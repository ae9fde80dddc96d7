// Shared device/host helpers of the peakstitch_b200 library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>

#include "../../include/peakstitch_b200.h"

namespace ps {

// ---------------------------------------------------------------------------
// error reporting / launch accounting (host side)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
void count_launch(uint64_t n = 1);

inline int check_cuda(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return PS_ERR_CUDA;
  }
  return PS_OK;
}

#define PS_LAUNCHED(name)                      \
  do {                                         \
    ::ps::count_launch();                      \
    int _st = ::ps::check_cuda(name);          \
    if (_st != PS_OK) return _st;              \
  } while (0)

#define PS_REQUIRE(cond, code, ...)            \
  do {                                         \
    if (!(cond)) {                             \
      ::ps::set_error(__VA_ARGS__);            \
      return (code);                           \
    }                                          \
  } while (0)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Arena {
  char* base;
  size_t size;
  size_t used;
  template <class T>
  T* take(size_t n) {
    used = align_up(used, 256);
    T* p = base ? reinterpret_cast<T*>(base + used) : nullptr;
    used += n * sizeof(T);
    return p;
  }
};

// ---------------------------------------------------------------------------
// ramped-pixel access.  P[r,c] exactly as apply_linear_ramp computes it
// (reference imaging.py:146-149): fl(I + fl(k * alpha)), k = r*nc + c + 1.
// Explicit _rn intrinsics keep nvcc from contracting into an FMA.
// ---------------------------------------------------------------------------
struct RampU8 {
  const uint8_t* p;
  int64_t pitch;
  int32_t nr, nc;
  double alpha;
  __device__ __forceinline__ double at(int r, int c) const {
    double k = (double)((int64_t)r * nc + c + 1);
    return __dadd_rn((double)p[(int64_t)r * pitch + c], __dmul_rn(k, alpha));
  }
};

struct RampF64 {
  const double* p;
  int64_t pitch;
  int32_t nr, nc;
  __device__ __forceinline__ double at(int r, int c) const {
    return p[(int64_t)r * pitch + c];
  }
};

struct RampF64Raw {
  const double* p;
  int64_t pitch;
  int32_t nr, nc;
  double alpha;
  __device__ __forceinline__ double at(int r, int c) const {
    double k = (double)((int64_t)r * nc + c + 1);
    return __dadd_rn(p[(int64_t)r * pitch + c], __dmul_rn(k, alpha));
  }
};

// numpy's float64 pairwise summation (add.reduce over a contiguous axis):
// n < 8 sequential from 0.0; n <= 128 eight interleaved accumulators then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the tail; else split at
// n/2 rounded down to a multiple of 8.  Elements are pulled in index order
// from `next()`, so the evaluation can stream a filtered sequence.
template <class Next>
__device__ double np_pairwise_stream(Next& next, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, next());
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) r[t] = next();
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int t = 0; t < 8; ++t) r[t] = __dadd_rn(r[t], next());
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, next());
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  double a = np_pairwise_stream(next, n2);
  double b = np_pairwise_stream(next, n - n2);
  return __dadd_rn(a, b);
}

// numpy float mod (npy_divmod): fmod, then + b when the signs differ; a zero
// result is +0.0.  Used as np.mod(x, 2*pi) in descriptor.py:138, 215.
__device__ __forceinline__ double np_mod_pos(double a, double b) {
  double m = fmod(a, b);
  if (m != 0.0) {
    if (m < 0.0) m = __dadd_rn(m, b);
  } else {
    m = 0.0;
  }
  return m;
}

__device__ __forceinline__ int warp_lane() { return threadIdx.x & 31; }

}  // namespace ps
