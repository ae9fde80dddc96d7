// Shared pieces of the K2 describe kernels (reference descriptor.py:82-269;
// SURVEY.md §8(a) A5-A9): the per-call parameter block, the reference's
// float64 bin arithmetic (mod 2 pi, trunc) and the float32 screens that
// decide most bins before any float64 work.  Included by describe.cu (the
// float64 kernels) and describe_f32.cu (the float32 throughput kernel).
#pragma once

#include "ps_common.cuh"

namespace ps {

constexpr int kMaxDescScales = 16;

struct DescParams {
  int n_scales;
  int scale[kMaxDescScales];
  int w[kMaxDescScales];       // region side after region_size + _fit_region cap
  double fx[kMaxDescScales];   // fixed-point scale 2^e of the histogram accumulators
  int lb[kMaxDescScales];      // bits per accumulator limb (3 limbs per bin)
  int d, D, orient;
  double k36, k8, two_pi;  // PEAK_BINS / TWO_PI, ORIENTATION_BINS / TWO_PI, TWO_PI
  double theta[36], cos_t[36], sin_t[36];  // theta0_k and cos/sin(-theta0_k)
  double cb36[37], sb36[37];                // cos/sin of the 36-bin edges m*2pi/36
  double c8[9], s8[9];                      // cos/sin of m*pi/4 (8-bin edges relative to theta0)
  int n_w8, w8_scale[kMaxDescScales];       // scales whose region side is 8 (fast path, d = 4)
  int default_w8;                           // the default scale is one of them
  int n_w16, w16_scale[kMaxDescScales];     // ... region side 16
  int default_w16;
};

// numpy mod(x, 2*pi) for -4*pi < x < 2*pi (descriptor.py:138, 215): fmod is
// x + 2*pi exactly below -2*pi (Sterbenz), then + 2*pi when negative, and a
// zero result is +0.0 -- identical to npy_divmod on this range.
__device__ __forceinline__ double mod_two_pi(double x, double two_pi) {
  if (x <= -two_pi) x = __dadd_rn(x, two_pi);
  if (x < 0.0) {
    x = __dadd_rn(x, two_pi);
  } else if (x == 0.0) {
    x = 0.0;
  }
  return x;
}

// ---- float32 screening of the discrete decisions -------------------------------
// On 8-bit rasters the gradients (exact float64 differences of the ramped
// raster) are bounded and well scaled, so the orientation bin of a sample is
// first taken from float32 atan2 and accepted only when the float32 bin
// coordinate lies at least kBinMargin from a bin edge (its error is < 2e-5
// bins: f32 rounding of the inputs, atan2f, the theta0 shift, the scaling);
// otherwise the float64 path decides.  Magnitudes stay float64 (a float32
// magnitude merges near-identical flat-region descriptors); in the
// general kernel the 36-bin argmax is accepted only when the top bin leads the
// next by more than the screening error, else that histogram is rebuilt in
// float64 (the fast kernels queue such keypoints for the general kernel).
constexpr float kBinMargin = 1e-4f;

__device__ __forceinline__ bool certified_bin(float x, int nbins, int& bin) {
  const float f = floorf(x);
  const float fr = x - f;
  bin = min(max((int)f, 0), nbins - 1);
  return fr > kBinMargin && fr < 1.0f - kBinMargin && x > 0.0f && x < (float)nbins;
}

// 8-bin octant of phi = atan2(v, u) in [0, 2 pi) from signs and |u| vs |v|,
// certified when phi is more than kBinMargin bins (7.85e-5 rad) from an edge:
// min(|u|, |v|) and ||u| - |v|| / sqrt(2) bound the distance to the axes and to
// the diagonals (relative to |u| + |v| >= r).  float32 error is ~3e-7 rad.
__device__ __forceinline__ bool octant_bin(float u, float v, int& bin) {
  const float au = fabsf(u), av = fabsf(v), sum = au + av;
  const bool upper = v >= 0.0f;
  const bool q_odd = upper ? !(u > 0.0f) : !(u < 0.0f);  // quadrants 1 and 3
  const int q = upper ? (q_odd ? 1 : 0) : (q_odd ? 3 : 2);
  const bool second = q_odd ? av < au : av > au;
  bin = 2 * q + (second ? 1 : 0);
  const float d = 7.854e-5f * sum;
  return fminf(au, av) > d && fabsf(au - av) > 1.4143f * d;
}

// Bin of a float64 gradient (a, b) whose float32 bin coordinate fell within
// kBinMargin of edge m (angle of the edge: cos ce, sin se).  The exact angle
// lies more than 1e-12 rad from the edge unless |b ce - a se| is tiny, and
// then the reference's float64 atan2 / mod / trunc cannot straddle the edge,
// so the side of the edge decides the bin; -1 asks for the full float64 path.
__device__ __forceinline__ int side_bin(double a, double b, double ce, double se, int m, int nbins) {
  const double sd = __dsub_rn(__dmul_rn(b, ce), __dmul_rn(a, se));
  const double thr = 1e-12 * (fabs(a) + fabs(b));
  if (sd > thr) return m == nbins ? 0 : m;
  if (sd < -thr) return m == 0 ? nbins - 1 : m - 1;
  return -1;
}

__device__ __forceinline__ float wrap_two_pi_f(float x) {
  const float tp = 6.283185307179586f;
  if (x < 0.0f) x += tp;
  if (x < 0.0f) x += tp;
  return x;
}

// float32 atan2 for the screen: octant reduction + degree-8 (in t^2) fit of
// atan on [0, 1]; max error 1.4e-7 rad in float32 evaluation (plus ~2e-7 from
// the reduction), far inside the 1.7e-5 rad (1e-4 bin) screen margin.
__device__ __forceinline__ float fast_atan2f(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mn = fminf(ax, ay), mx = fmaxf(ax, ay);
  const float t = mx > 0.0f ? __fdividef(mn, mx) : 0.0f;
  const float z = t * t;
  float p = -0.00405279453843832f;
  p = __fmaf_rn(p, z, 0.021855242550373077f);
  p = __fmaf_rn(p, z, -0.05589873343706131f);
  p = __fmaf_rn(p, z, 0.09640958160161972f);
  p = __fmaf_rn(p, z, -0.13908010721206665f);
  p = __fmaf_rn(p, z, 0.19946402311325073f);
  p = __fmaf_rn(p, z, -0.3332984149456024f);
  p = __fmaf_rn(p, z, 0.9999993443489075f);
  float r = p * t;
  if (ay > ax) r = 1.5707963267948966f - r;
  if (x < 0.0f) r = 3.141592653589793f - r;
  return y < 0.0f ? -r : r;
}

// Exact bin of a sample whose float32 screen fell near an edge (rare): the
// side of edge m, else the float64 atan2 path.
// (ce, se) is the edge direction rotated by theta0 (c0, s0).
__device__ __forceinline__ int exact_bin(double a, double b, double c0, double s0, double cm, double sm, int m,
                                      int nbins, double shift, double k, double two_pi) {
  const double ce = __dsub_rn(__dmul_rn(c0, cm), __dmul_rn(s0, sm));
  const double se = __dadd_rn(__dmul_rn(s0, cm), __dmul_rn(c0, sm));
  int bin = side_bin(a, b, ce, se, m, nbins);
  if (bin < 0) {
    const double ori = mod_two_pi(__dsub_rn(atan2(b, a), shift), two_pi);
    bin = min((int)__dmul_rn(ori, k), nbins - 1);
  }
  return bin;
}

// Float32 throughput path (describe_f32.cu): every w = 8, d = 4 keypoint at
// least 6 pixels inside an 8-bit (grey or RGB) image; everything else is
// appended to `work` for the float64 general kernel.  Writes float32 rows
// only.  window_slots: the caller vouches for the window layout of the
// default scale (PS_DESCRIBE_WINDOW_SLOTS); with L = 8 the tile kernel runs.
template <class Img>
int launch_describe_f32(const Img& im, const ps_image_batch* img, const ps_keypoints* kp, int32_t default_scale,
                        const DescParams& prm, float* out_desc32, bool window_slots, int64_t* work,
                        unsigned long long* n_work, cudaStream_t s);

}  // namespace ps
