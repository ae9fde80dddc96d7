// Shared device/host helpers of the peakstitch_b200 library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <cmath>

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
// (reference imaging.py:129-132): fl(I + fl(k * alpha)), k = r*nc + c + 1.
// Explicit _rn intrinsics keep nvcc from contracting into an FMA.
// ---------------------------------------------------------------------------
// exact int -> double for 0 <= x < 2^32 on the FP64 pipe (no I2F):
// the bits 0x43300000:x are 2^52 + x, and subtracting 2^52 is exact.
__device__ __forceinline__ double u32_to_f64(unsigned x) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)x), 4503599627370496.0);
}

// (callers guarantee nr * nc < 2^31 and nr * pitch < 2^31: 32-bit offsets)
struct RampU8 {
  static constexpr int kElem = 1;  // elements of *p per pixel
  const uint8_t* p;
  int64_t pitch;
  int32_t nr, nc;
  double alpha;
  __device__ __forceinline__ double at(int r, int c) const {
    const double k = u32_to_f64((unsigned)(r * nc + c + 1));
    return __dadd_rn(u32_to_f64(p[r * (int)pitch + c]), __dmul_rn(k, alpha));
  }
  __device__ __forceinline__ unsigned key(int r, int c) const { return p[r * (int)pitch + c]; }
};

// BT.601 grey in the evaluation order of the x86-64 OpenBLAS dgemv kernel
// behind numpy's `rgb @ LUMA` (two FMAs around the green product; measured
// on all 2^24 triples -- the host check `ps_gray_table_check` decides at run
// time whether this formula reproduces the run host's own bits).
__host__ __device__ __forceinline__ double bt601_fma(unsigned r, unsigned g, unsigned b) {
#ifdef __CUDA_ARCH__
  return __fma_rn((double)b, 0.114, __fma_rn((double)r, 0.299, __dmul_rn((double)g, 0.587)));
#else
  return std::fma((double)b, 0.114, std::fma((double)r, 0.299, (double)g * 0.587));
#endif
}

// Interleaved RGB8: the grey is the host's own BT.601 bits -- from
// a 2^24-entry table, or (lut == nullptr) from bt601_fma once the table has
// been checked equal to it; key() is the exact integer luma 299R + 587G +
// 114B, whose order equals the grey order (distinct greys differ by >= 0.001).
struct RampRGB8 {
  static constexpr int kElem = 3;
  const uint8_t* p;
  int64_t pitch;  // pixels
  int32_t nr, nc;
  double alpha;
  const double* lut;
  __device__ __forceinline__ unsigned rgb(int r, int c) const {
    const uint8_t* q = p + 3 * (r * (int)pitch + c);
    return ((unsigned)q[0] << 16) | ((unsigned)q[1] << 8) | (unsigned)q[2];
  }
  __device__ __forceinline__ unsigned key(int r, int c) const {
    const uint8_t* q = p + 3 * (r * (int)pitch + c);
    return 299u * q[0] + 587u * q[1] + 114u * q[2];
  }
  __device__ __forceinline__ double gray(int r, int c) const {
    const uint8_t* q = p + 3 * (r * (int)pitch + c);
    if (lut) return __ldg(lut + (((unsigned)q[0] << 16) | ((unsigned)q[1] << 8) | (unsigned)q[2]));
    return bt601_fma(q[0], q[1], q[2]);
  }
  __device__ __forceinline__ double at(int r, int c) const {
    const double k = u32_to_f64((unsigned)(r * nc + c + 1));
    return __dadd_rn(gray(r, c), __dmul_rn(k, alpha));
  }
};

struct RampF64 {
  static constexpr int kElem = 1;
  const double* p;
  int64_t pitch;
  int32_t nr, nc;
  __device__ __forceinline__ double at(int r, int c) const {
    return p[(int64_t)r * pitch + c];
  }
};

// round-to-nearest add that nvcc may not contract (host: plain IEEE add)
__host__ __device__ __forceinline__ double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}

struct RampF64Raw {
  static constexpr int kElem = 1;
  const double* p;
  int64_t pitch;
  int32_t nr, nc;
  double alpha;
  __device__ __forceinline__ double at(int r, int c) const {
    const double k = u32_to_f64((unsigned)(r * nc + c + 1));
    return __dadd_rn(p[(int64_t)r * pitch + c], __dmul_rn(k, alpha));
  }
};

// Leaf of the pairwise sum: n <= 128 elements.
template <class Next>
__host__ __device__ inline double np_pairwise_leaf(Next& next, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = dadd(res, next());
    return res;
  }
  double r[8];
  for (int t = 0; t < 8; ++t) r[t] = next();
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int t = 0; t < 8; ++t) r[t] = dadd(r[t], next());
  double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
  for (; i < n; ++i) res = dadd(res, next());
  return res;
}

// numpy's float64 pairwise summation (add.reduce over a contiguous axis):
// n < 8 sequential from 0.0; n <= 128 eight interleaved accumulators then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the tail; else split at
// n/2 rounded down to a multiple of 8 and add the halves.  Elements are
// pulled in index order from `next()`, so a filtered sequence can be
// streamed.  Iterative (explicit stack): no device recursion.
template <class Next>
__host__ __device__ inline double np_pairwise_stream(Next& next, int64_t n) {
  int64_t right[64];
  double left[64];
  bool has_left[64];
  int sp = 0;
  int64_t len = n;
  double result = 0.0;
  for (;;) {
    while (len > 128) {  // descend into the left half
      int64_t n2 = len / 2;
      n2 -= n2 % 8;
      right[sp] = len - n2;
      has_left[sp] = false;
      ++sp;
      len = n2;
    }
    result = np_pairwise_leaf(next, len);
    for (;;) {  // ascend
      if (sp == 0) return result;
      if (!has_left[sp - 1]) {
        left[sp - 1] = result;
        has_left[sp - 1] = true;
        len = right[sp - 1];
        break;  // now sum the right half
      }
      result = dadd(left[sp - 1], result);
      --sp;
    }
  }
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
