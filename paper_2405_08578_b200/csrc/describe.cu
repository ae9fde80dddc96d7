// K2 -- orientation-normalised gradient-histogram descriptor
// (reference descriptor.py:82-269).
//
// One warp per keypoint.  All geometry, gradients, interpolation and bin
// decisions are float64 with the reference's exact operation order (explicit
// _rn intrinsics, no FMA contraction) on the ramped raster P, recomputed from
// the 8-bit image and alpha (the ramp is never materialised).  The two
// magnitude histograms are accumulated per bin in raster (sample) order,
// like np.bincount, so equal inputs give bit-identical descriptors (F6).
// atan2 / hypot are CUDA's float64 versions (numpy's own differ from libm by
// ~1 ulp), hence the 1e-4 relative parity bar of contract P2.
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "describe_common.cuh"

namespace ps {
namespace {

constexpr int kWarps = 8;



// Histogram accumulation is exact fixed point: q = rint(mag * 2^e) split into
// three limbs of `lb` bits, each summed with a native 32-bit shared atomic
// (limb sums cannot overflow: nsamp * 2^lb < 2^32).  Integer sums are
// order-independent, so the histograms are bit-reproducible (F6) without
// serial chains; the scale keeps the quantum ~1e-15 of the largest sum.
struct FxHist {
  unsigned* h;  // [3][nbins]
  int nbins, lb;
  __device__ __forceinline__ void add(int bin, double mag, double fx) const {
    if (mag == 0.0) return;
    const unsigned long long q = __double2ull_rn(__dmul_rn(mag, fx));
    const unsigned m = (1u << lb) - 1u;
    atomicAdd(h + bin, (unsigned)(q & m));
    atomicAdd(h + nbins + bin, (unsigned)((q >> lb) & m));
    atomicAdd(h + 2 * nbins + bin, (unsigned)(q >> (2 * lb)));
  }
  __device__ __forceinline__ unsigned long long get(int bin) const {
    return (unsigned long long)h[bin] + ((unsigned long long)h[nbins + bin] << lb) +
           ((unsigned long long)h[2 * nbins + bin] << (2 * lb));
  }
  __device__ __forceinline__ void zero(int lane) const {
    for (int q = lane; q < 3 * nbins; q += 32) h[q] = 0u;
  }
};

// Stage P over rows [r0, r0+PR) x cols [c0, c0+PC) into stage[y * SP + x]:
// lane (sx, sy) owns column sx and rows sy, sy + 2, ...
template <class Img>
__device__ __forceinline__ void stage_box(const Img& im, double* stage, int SP, int r0, int c0, int PR, int PC, int sx,
                                          int sy) {
  if (sx >= PC) return;
  for (int y = sy; y < PR; y += 2) stage[y * SP + sx] = im.at(r0 + y, c0 + sx);
}
// 8-bit raster, at most 2*MAXR rows: all pixel loads are issued before any is
// consumed (one memory latency per box), then the ramp is applied.
template <int MAXR>
__device__ __forceinline__ void stage_box_u8(const RampU8& im, double* stage, int SP, int r0, int c0, int PR, int PC,
                                             int sx, int sy) {
  if (sx >= PC) return;
  const int pitch = (int)im.pitch;
  const uint8_t* p = im.p + (r0 + sy) * pitch + (c0 + sx);
  unsigned v[MAXR];
#pragma unroll
  for (int i = 0; i < MAXR; ++i) v[i] = (sy + 2 * i < PR) ? (unsigned)__ldg(p + 2 * i * pitch) : 0u;
  double k = u32_to_f64((unsigned)((r0 + sy) * im.nc + c0 + sx + 1));  // ramp index, exact in float64
  const double kstep = u32_to_f64(2u * (unsigned)im.nc);
#pragma unroll
  for (int i = 0; i < MAXR; ++i) {
    if (sy + 2 * i < PR) stage[(sy + 2 * i) * SP + sx] = __dadd_rn(u32_to_f64(v[i]), __dmul_rn(k, im.alpha));
    k = __dadd_rn(k, kstep);
  }
}

// RGB8 raster: the three channel bytes of every pixel, then the table greys,
// are all requested before any is consumed.
template <int MAXR>
__device__ __forceinline__ void stage_box_rgb8(const RampRGB8& im, double* stage, int SP, int r0, int c0, int PR,
                                               int PC, int sx, int sy) {
  if (sx >= PC) return;
  unsigned key[MAXR];
#pragma unroll
  for (int i = 0; i < MAXR; ++i) key[i] = (sy + 2 * i < PR) ? im.rgb(r0 + sy + 2 * i, c0 + sx) : 0u;
  double g[MAXR];
  if (im.lut) {
#pragma unroll
    for (int i = 0; i < MAXR; ++i) g[i] = __ldg(im.lut + key[i]);
  } else {
#pragma unroll
    for (int i = 0; i < MAXR; ++i) g[i] = bt601_fma(key[i] >> 16, (key[i] >> 8) & 255u, key[i] & 255u);
  }
  double k = u32_to_f64((unsigned)((r0 + sy) * im.nc + c0 + sx + 1));
  const double kstep = u32_to_f64(2u * (unsigned)im.nc);
#pragma unroll
  for (int i = 0; i < MAXR; ++i) {
    if (sy + 2 * i < PR) stage[(sy + 2 * i) * SP + sx] = __dadd_rn(g[i], __dmul_rn(k, im.alpha));
    k = __dadd_rn(k, kstep);
  }
}

template <class Img>
__device__ __forceinline__ void axis_sample(const Img& im, int r, int c, double& a, double& b) {
  // descriptor.py:135-136 (gradient_at convention, :98-115)
  a = __dsub_rn(im.at(r + 1, c), im.at(r - 1, c));
  b = __dsub_rn(im.at(r, c + 1), im.at(r, c - 1));
}

// One keypoint, one warp.  W / DD > 0 fix the region side / grid at compile
// time (the common w in {8, 16, 32}, d = 4); 0 means runtime values.
// Staging capacity (doubles per warp) for compile-time W: the P box of the
// rotated patch plus its two gradient fields.  The rotated grid spans at most
// (W-1)*sqrt(2) in x and y, so pr1 - pr0 <= ceil((W-1)*sqrt(2)) + 1.
template <int W>
struct Stage {
  static constexpr int kSpan = W > 0 ? (int)((W - 1) * 1.41422) + 3 : 0;  // >= pr1 - pr0 + 1
  static constexpr int kStride = kSpan + 2 > 16 ? kSpan + 2 : 16;           // row stride (>= kSpan + 2)
  static constexpr int kP = (kSpan + 2) * kStride;
  static constexpr int kF = kSpan * kStride;
  static constexpr int kTotal = W > 0 ? kP + 2 * kF : 0;  // doubles per warp
  static_assert(W <= 0 || W + 2 <= kStride, "stage stride too small");
};
constexpr int kStageW = 8;  // region side served from shared memory
constexpr int kStageDoubles = Stage<kStageW>::kTotal;

// Fast-path (w = 8) layout: one 16 x 16 box of P (rows at a stride of 24
// doubles: axis reads of a half-warp hit 16 distinct 8-byte banks) that holds
// both the axis region and every rotated patch; the rotated samples form
// their gradient-field corners from it directly.
template <int W>
struct FastBox;
template <>
struct FastBox<8> {
  static constexpr int kBox = 16;        // staged P box side
  static constexpr int kOff = 7;         // box starts at floor(cy) - kOff (clamped)
  static constexpr int SPP = 24;
  static constexpr int kTotal = kBox * SPP;  // doubles per keypoint
};
// w = 16 (the reference's default 32..128 windows): the axis region spans
// 18 rows and a rotated patch lies within cy -/+ (7.5 sqrt(2) + 2).
template <>
struct FastBox<16> {
  static constexpr int kBox = 26;
  static constexpr int kOff = 12;
  static constexpr int SPP = 26;
  static constexpr int kTotal = kBox * SPP;
};
using FastStage = FastBox<8>;


template <int W, int DD, bool FAST, class Img>
__device__ __forceinline__ void describe_keypoint(const Img& im, int row, int col, int w_rt, int d_rt, double fx,
                                                  int lb, const DescParams& prm, unsigned* hbase, double* stage,
                                                  float* __restrict__ o32, double* __restrict__ o64) {
  constexpr bool kStaged = W == kStageW;
  constexpr int SP = Stage<W>::kStride;
  const int lane = threadIdx.x & 31;
  const int w = W > 0 ? W : w_rt;
  const int d = DD > 0 ? DD : d_rt;
  const int D = d * d * 8;
  const int ws = w / d, nsamp = w * w;
  const int nr = im.nr, nc = im.nc;
  const double two_pi = prm.two_pi;
  // _fit_region (descriptor.py:129-130)
  const int r0 = min(max(row - w / 2, 1), nr - 1 - w);
  const int c0 = min(max(col - w / 2, 1), nc - 1 - w);
  const FxHist h128{hbase, D, lb};
  const FxHist h36{hbase + 3 * D, 36, lb};
  h128.zero(lane);
  h36.zero(lane);
  const int sx_ = lane & 15, sy_ = lane >> 4;  // staging: 2 rows x 16 columns per step
  if (kStaged) {  // P over rows r0-1..r0+w, cols c0-1..c0+w
    stage_box(im, stage, SP, r0 - 1, c0 - 1, W + 2, W + 2, sx_, sy_);
  }
  __syncwarp();
  auto axis_ab = [&](int iv, int iu, double& a, double& b) {
    if (kStaged) {
      a = __dsub_rn(stage[(iv + 2) * SP + iu + 1], stage[iv * SP + iu + 1]);
      b = __dsub_rn(stage[(iv + 1) * SP + iu + 2], stage[(iv + 1) * SP + iu]);
    } else {
      axis_sample(im, r0 + iv, c0 + iu, a, b);
    }
  };
  // bin of a float64 gradient (reference arithmetic), optionally shifted by -theta0
  auto bin64 = [&](double a, double b, double shift, double k, int nbins) {
    const double ori = mod_two_pi(__dsub_rn(atan2(b, a), shift), two_pi);
    return min((int)__dmul_rn(ori, k), nbins - 1);
  };
  // 36-bin orientation of an axis sample: float32 screen, edge side test, float64
  auto bin36 = [&](double a, double b, float af, float bf) {
    const float x = wrap_two_pi_f(atan2f(bf, af)) * 5.729577951308232f;
    int bin;
    if (certified_bin(x, 36, bin)) return bin;
    const int m = min(max(__float2int_rn(x), 0), 36);
    bin = side_bin(a, b, prm.cb36[m], prm.sb36[m], m, 36);
    return bin >= 0 ? bin : bin64(a, b, 0.0, prm.k36, 36);
  };
  if (prm.orient) {
    // --- dominant orientation: 36-bin histogram of the axis region (:142-146)
    bool exact = !FAST;
    int hk = -1;
    for (;;) {
#pragma unroll 4
      for (int s = lane; s < nsamp; s += 32) {
        double a, b;
        axis_ab(s / w, s % w, a, b);
        if (exact) {
          h36.add(bin64(a, b, 0.0, prm.k36, 36), hypot(a, b), fx);
        } else {
          const float af = (float)a, bf = (float)b;
          h36.add(bin36(a, b, af, bf), __dsqrt_rn(__fma_rn(a, a, __dmul_rn(b, b))), fx);
        }
      }
      __syncwarp();
      if (exact) break;
      // float32 magnitudes: accept the argmax only with a clear lead.  Keys are
      // the float32 bin sums with the low 6 mantissa bits replaced by 63 - bin.
      const float f1 = (float)h36.get(lane), f2 = lane < 4 ? (float)h36.get(lane + 32) : 0.0f;
      const unsigned k1 = (__float_as_uint(f1) & ~63u) | (63u - lane);
      const unsigned k2 = lane < 4 ? ((__float_as_uint(f2) & ~63u) | (31u - lane)) : 0u;
      const unsigned top = __reduce_max_sync(0xffffffffu, max(k1, k2));
      const unsigned sec = __reduce_max_sync(0xffffffffu, max(k1 == top ? 0u : k1, k2 == top ? 0u : k2));
      const float tv = __uint_as_float(top & ~63u), sv = __uint_as_float(sec & ~63u);
      if (sv < tv * 0.99994f) {  // lead > 6e-5 relative: float64 sums agree
        hk = 63 - (int)(top & 63u);
        break;
      }
      exact = true;  // near-tie: rebuild this histogram in float64 (warp-uniform)
      h36.zero(lane);
      __syncwarp();
    }
    if (hk < 0) {  // first argmax over the 36 bins (exact integer sums)
      unsigned long long hv = h36.get(lane);
      hk = lane;
      if (lane < 4 && h36.get(lane + 32) > hv) { hv = h36.get(lane + 32); hk = lane + 32; }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long v2 = __shfl_xor_sync(0xffffffffu, hv, o);
        const int k2 = __shfl_xor_sync(0xffffffffu, hk, o);
        if (v2 > hv || (v2 == hv && k2 < hk)) { hv = v2; hk = k2; }
      }
    }
    const double theta0 = prm.theta[hk], ct = prm.cos_t[hk], st = prm.sin_t[hk];
    const float theta0f = (float)theta0;
    // --- rotated grid centred on the (clamped) feature pixel (:237-240, 164-216)
    const double half = (double)(w - 1) / 2.0;
    const double cy = fmin(fmax((double)row, 1.0 + half), __dsub_rn((double)nr - 2.0, half));
    const double cx = fmin(fmax((double)col, 1.0 + half), __dsub_rn((double)nc - 2.0, half));
    // Rounded positions are coordinate-wise monotone in u and in v, so each
    // extreme of x / y over the grid sits at the corner picked by the signs.
    const double xmin = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, ct >= 0.0 ? -half : half)), __dmul_rn(st, st >= 0.0 ? half : -half));
    const double xmax = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, ct >= 0.0 ? half : -half)), __dmul_rn(st, st >= 0.0 ? -half : half));
    const double ymin = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, st >= 0.0 ? -half : half)), __dmul_rn(ct, ct >= 0.0 ? -half : half));
    const double ymax = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, st >= 0.0 ? half : -half)), __dmul_rn(ct, ct >= 0.0 ? half : -half));
    const int pr0 = max((int)floor(ymin), 1), pr1 = min((int)ceil(ymax), nr - 2);
    const int pc0 = max((int)floor(xmin), 1), pc1 = min((int)ceil(xmax), nc - 2);
    const int xcap = max(pc1 - pc0 - 1, 0), ycap = max(pr1 - pr0 - 1, 0);
    const double xhi = (double)(nc - 2), yhi = (double)(nr - 2);
    const int FR = pr1 - pr0 + 1, FC = pc1 - pc0 + 1;  // field patch (descriptor.py:192-193)
    double* fa = stage + Stage<W>::kP;
    double* fb = fa + Stage<W>::kF;
    if (kStaged) {
      __syncwarp();
      const int PC = FC + 2, PR = FR + 2;
      stage_box(im, stage, SP, pr0 - 1, pc0 - 1, PR, PC, sx_, sy_);
      __syncwarp();
      for (int y = sy_; y < FR; y += 2)
        if (sx_ < FC) {
          fa[y * SP + sx_] = __dsub_rn(stage[(y + 2) * SP + sx_ + 1], stage[y * SP + sx_ + 1]);
          fb[y * SP + sx_] = __dsub_rn(stage[(y + 1) * SP + sx_ + 2], stage[(y + 1) * SP + sx_]);
        }
      __syncwarp();
    }
    // 8-bin edges m*pi/4 + theta0 as (cos, sin) for the side test
    const double c0t = ct, s0t = -st;  // cos(theta0), sin(theta0)
#pragma unroll 2
    for (int s = lane; s < nsamp; s += 32) {
      const int iv = s / w, iu = s % w;
      const double u = __dsub_rn((double)iu, half), v = __dsub_rn((double)iv, half);
      const double x = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, u)), __dmul_rn(st, v));
      const double y = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, u)), __dmul_rn(ct, v));
      const bool inside = x >= 1.0 && x <= xhi && y >= 1.0 && y <= yhi;
      if (!inside) continue;  // mag = hypot * valid = +0.0 adds nothing
      const double lx = __dsub_rn(fmin(fmax(x, (double)pc0), (double)pc1), (double)pc0);
      const double ly = __dsub_rn(fmin(fmax(y, (double)pr0), (double)pr1), (double)pr0);
      const int x0 = min((int)floor(lx), xcap), y0 = min((int)floor(ly), ycap);
      const double fxx = __dsub_rn(lx, (double)x0), fyy = __dsub_rn(ly, (double)y0);
      const int x1 = min(x0 + 1, pc1 - pc0), y1 = min(y0 + 1, pr1 - pr0);
      double a00, b00, a01, b01, a10, b10, a11, b11;
      if (kStaged) {
        a00 = fa[y0 * SP + x0]; b00 = fb[y0 * SP + x0];
        a01 = fa[y0 * SP + x1]; b01 = fb[y0 * SP + x1];
        a10 = fa[y1 * SP + x0]; b10 = fb[y1 * SP + x0];
        a11 = fa[y1 * SP + x1]; b11 = fb[y1 * SP + x1];
      } else {
        const int gy0 = pr0 + y0, gy1 = pr0 + y1, gx0 = pc0 + x0, gx1 = pc0 + x1;
        axis_sample(im, gy0, gx0, a00, b00);
        axis_sample(im, gy0, gx1, a01, b01);
        axis_sample(im, gy1, gx0, a10, b10);
        axis_sample(im, gy1, gx1, a11, b11);
      }
      const double sy = __dsub_rn(1.0, fyy), sx = __dsub_rn(1.0, fxx);
      // left-to-right: f00*(1-fy)*(1-fx) + f01*(1-fy)*fx + f10*fy*(1-fx) + f11*fy*fx
      const double as = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(a00, sy), sx), __dmul_rn(__dmul_rn(a01, sy), fxx)),
                                            __dmul_rn(__dmul_rn(a10, fyy), sx)),
                                  __dmul_rn(__dmul_rn(a11, fyy), fxx));
      const double bs = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(b00, sy), sx), __dmul_rn(__dmul_rn(b01, sy), fxx)),
                                            __dmul_rn(__dmul_rn(b10, fyy), sx)),
                                  __dmul_rn(__dmul_rn(b11, fyy), fxx));
      const int cell = ((iv / ws) * d + iu / ws) * 8;
      if (FAST) {
        const float af = (float)as, bf = (float)bs;
        const float xb = wrap_two_pi_f(atan2f(bf, af) - theta0f) * 1.2732395447351628f;
        int ob;
        if (!certified_bin(xb, 8, ob)) {
          const int m = min(max(__float2int_rn(xb), 0), 8);
          const double ce = __dsub_rn(__dmul_rn(c0t, prm.c8[m]), __dmul_rn(s0t, prm.s8[m]));
          const double se = __dadd_rn(__dmul_rn(s0t, prm.c8[m]), __dmul_rn(c0t, prm.s8[m]));
          ob = side_bin(as, bs, ce, se, m, 8);
          if (ob < 0) ob = bin64(as, bs, theta0, prm.k8, 8);
        }
        h128.add(cell + ob, __dsqrt_rn(__fma_rn(as, as, __dmul_rn(bs, bs))), fx);
      } else {
        h128.add(cell + bin64(as, bs, theta0, prm.k8, 8), hypot(as, bs), fx);
      }
    }
  } else {
#pragma unroll 4
    for (int s = lane; s < nsamp; s += 32) {
      const int iv = s / w, iu = s % w;
      double a, b;
      axis_ab(iv, iu, a, b);
      const int cell = ((iv / ws) * d + iu / ws) * 8;
      if (FAST) {
        const float af = (float)a, bf = (float)b;
        const float xb = wrap_two_pi_f(atan2f(bf, af)) * 1.2732395447351628f;
        int ob;
        if (!certified_bin(xb, 8, ob)) {
          const int m = min(max(__float2int_rn(xb), 0), 8);
          ob = side_bin(a, b, prm.c8[m], prm.s8[m], m, 8);
          if (ob < 0) ob = bin64(a, b, 0.0, prm.k8, 8);
        }
        h128.add(cell + ob, __dsqrt_rn(__fma_rn(a, a, __dmul_rn(b, b))), fx);
      } else {
        h128.add(cell + bin64(a, b, 0.0, prm.k8, 8), hypot(a, b), fx);
      }
    }
  }
  __syncwarp();
  // --- L2 normalise, clamp at 0.2, renormalise (descriptor.py:250-255)
  constexpr int kPer = DD > 0 ? (DD * DD * 8 + 31) / 32 : 16;
  const double inv_fx = 1.0 / fx;  // exact: fx is a power of two
  double vals[kPer];
  double ss = 0.0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int q = lane + 32 * j;
    vals[j] = q < D ? __dmul_rn((double)h128.get(q), inv_fx) : 0.0;
    ss = __dadd_rn(ss, __dmul_rn(vals[j], vals[j]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
  const double n1 = __dsqrt_rn(ss);
  double n2 = 0.0;
  if (n1 > 0.0) {
    const double r1 = __drcp_rn(n1);
    double ss2 = 0.0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      vals[j] = fmin(__dmul_rn(vals[j], r1), 0.2);
      ss2 = __dadd_rn(ss2, __dmul_rn(vals[j], vals[j]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss2 = __dadd_rn(ss2, __shfl_xor_sync(0xffffffffu, ss2, o));
    n2 = __drcp_rn(__dsqrt_rn(ss2));
  }
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int q = lane + 32 * j;
    if (q < D) {
      const double v = n1 > 0.0 ? __dmul_rn(vals[j], n2) : 0.0;
      if (o32) o32[q] = __double2float_rn(v);
      if (o64) o64[q] = v;
    }
  }
  __syncwarp();
}


// ---- 8-bit fast path, w = 8 (C1/C2/C4/C5 L_min) -----------------------------------

// Returns false (nothing written) when the 36-bin argmax has no clear lead;
// the caller then queues the keypoint for the float64 kernel.
// Fast-path histograms: exact fixed point, two 26-bit limbs per bin (two
// native 32-bit shared atomics per sample; 64 samples x 2^26 < 2^32), scale
// 2^e chosen per keypoint from the largest magnitude so a bin sum stays
// below 2^52: quantum ~2^-46 of the largest bin -- far below float32
// resolution, so near-identical regions keep distinct descriptors (F6).
constexpr int kLimb = 26;  // w = 8: 64 samples; w = 16 (256 samples) uses 24-bit limbs
template <int L = kLimb>
__device__ __forceinline__ void h2_add(unsigned* h, int nb, int bin, double mag, double fx) {
  if (!(mag > 0.0)) return;
  const unsigned long long q = __double2ull_rn(__dmul_rn(mag, fx));
  atomicAdd(h + bin, (unsigned)(q & ((1u << L) - 1u)));
  atomicAdd(h + nb + bin, (unsigned)(q >> L));
}
template <int L = kLimb>
__device__ __forceinline__ unsigned long long h2_get(const unsigned* h, int nb, int bin) {
  return ((unsigned long long)h[nb + bin] << L) + (unsigned long long)h[bin];
}
// Warp-uniform fixed-point scale from the lanes' largest magnitudes: the max
// of the (non-negative) doubles' high words (one REDUX) bounds the exponent eb,
// every magnitude is < 2^(eb - 1022) and a bin sum of NS = 64 of them is
// < 2^(eb - 1016), so 2^(1068 - eb) keeps every sum below 2^52.
template <int LOG = 6>  // log2(samples per keypoint)
__device__ __forceinline__ double fx_scale52_warp(double mx) {
  const unsigned eb = __reduce_max_sync(0xffffffffu, (unsigned)__double2hiint(mx)) >> 20;
  if (eb == 0u) return 1.0;  // all magnitudes zero (or subnormal)
  const int be = min(2097 - LOG - (int)eb, 2046);  // 2^(52 - (eb - 1022 + LOG)), biased
  return __hiloint2double(be << 20, 0);
}

template <int W, class Img>
__device__ __forceinline__ bool describe_keypoint_w8u8(const Img& im, int row, int col, const DescParams& prm,
                                                       unsigned* hbase, double* stage, float* __restrict__ o32,
                                                       double* __restrict__ o64) {
  static_assert(W == 8 || W == 16, "fast path: w = 8 or 16");
  constexpr int NS = W * W, SPL = NS / 32, D = 128, SP = FastBox<W>::SPP;
  constexpr int LOG = W == 8 ? 6 : 8, LIMB = 32 - LOG;  // limb sums of NS samples stay below 2^32
  constexpr int WS = W / 4;
  const int lane = threadIdx.x & 31;
  const int nr = im.nr, nc = im.nc;
  constexpr int BX = FastBox<W>::kBox;
  const int r0 = min(max(row - W / 2, 1), nr - 1 - W);
  const int c0 = min(max(col - W / 2, 1), nc - 1 - W);
  constexpr double half = (double)(W - 1) / 2.0;
  // centre clamp min(max(row, 1 + half), nr - 2 - half) on half-integers, in
  // integers (2 cy is an integer; exact)
  const int cy2 = min(max(2 * row, 2 + (W - 1)), 2 * (nr - 2) - (W - 1));
  const int cx2 = min(max(2 * col, 2 + (W - 1)), 2 * (nc - 2) - (W - 1));
  const double cy = 0.5 * (double)cy2, cx = 0.5 * (double)cx2;
  // One staged box for both phases: the axis region spans rows r0-1..r0+W and
  // any rotated patch pr0-1..pr1+1 lies within cy -/+ ((W-1)/2 sqrt(2) + 2), so
  // rows floor(cy)-kOff .. floor(cy)-kOff+BX-1 (clamped to the image) hold both.
  constexpr int OFF = FastBox<W>::kOff;
  const int BR = max(0, min((cy2 >> 1) - OFF, nr - BX)), BC = max(0, min((cx2 >> 1) - OFF, nc - BX));
  unsigned* h128 = hbase;         // [2][128]
  unsigned* h36 = hbase + 2 * D;  // [2][36]
  static_assert((2 * (D + 36)) % 4 == 0, "vector zeroing");
  for (int q = lane; q < 2 * (D + 36) / 4; q += 32) reinterpret_cast<uint4*>(hbase)[q] = make_uint4(0u, 0u, 0u, 0u);
  if constexpr (W == 8) {  // 16 columns: half-warps take alternate rows
    const int sx_ = lane & 15, sy_ = lane >> 4;
    if constexpr (std::is_same<Img, RampRGB8>::value)
      stage_box_rgb8<BX / 2>(im, stage, SP, BR, BC, BX, BX, sx_, sy_);
    else
      stage_box_u8<BX / 2>(im, stage, SP, BR, BC, BX, BX, sx_, sy_);
  } else {  // 26 columns: lane = column, even rows then odd rows
#pragma unroll
    for (int sy = 0; sy < 2; ++sy) {
      if constexpr (std::is_same<Img, RampRGB8>::value)
        stage_box_rgb8<BX / 2>(im, stage, SP, BR, BC, BX, BX, lane, sy);
      else
        stage_box_u8<BX / 2>(im, stage, SP, BR, BC, BX, BX, lane, sy);
    }
  }
  __syncwarp();
  const double* pa = stage + (r0 - 1 - BR) * SP + (c0 - 1 - BC);  // axis region origin
  auto axis_ab = [&](int iv, int iu, double& a, double& b) {
    a = __dsub_rn(pa[(iv + 2) * SP + iu + 1], pa[iv * SP + iu + 1]);
    b = __dsub_rn(pa[(iv + 1) * SP + iu + 2], pa[(iv + 1) * SP + iu]);
  };
  auto bin64 = [&](double a, double b, double shift, double k, int nbins) {
    const double ori = mod_two_pi(__dsub_rn(atan2(b, a), shift), prm.two_pi);
    return min((int)__dmul_rn(ori, k), nbins - 1);
  };
  double mg[SPL];  // float64 magnitudes (~1 ulp): descriptors stay ~1e-15 accurate
  float mgf[SPL];  // orientation-histogram magnitudes
  int bn[SPL];
  if (!prm.orient) {
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      const int s = lane + 32 * j, iv = s / W, iu = s % W;
      double a, b;
      axis_ab(iv, iu, a, b);
      const float af = (float)a, bf = (float)b;
      const float xb = wrap_two_pi_f(fast_atan2f(bf, af)) * 1.2732395447351628f;
      int ob;
      if (!certified_bin(xb, 8, ob)) {
        const int m = min(max(__float2int_rn(xb), 0), 8);
        ob = side_bin(a, b, prm.c8[m], prm.s8[m], m, 8);
        if (ob < 0) ob = bin64(a, b, 0.0, prm.k8, 8);
      }
      mg[j] = __dsqrt_rn(__fma_rn(a, a, __dmul_rn(b, b)));
      bn[j] = ((iv / WS) * 4 + iu / WS) * 8 + ob;
    }
  } else {
    // --- 36-bin dominant orientation over the axis region (descriptor.py:142-146)
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      const int s = lane + 32 * j;
      double a, b;
      axis_ab(s / W, s % W, a, b);
      const float af = (float)a, bf = (float)b;
      const float x = wrap_two_pi_f(fast_atan2f(bf, af)) * 5.729577951308232f;
      int bin;
      if (!certified_bin(x, 36, bin)) {
        const int m = min(max(__float2int_rn(x), 0), 36);
        bin = side_bin(a, b, prm.cb36[m], prm.sb36[m], m, 36);
        if (bin < 0) bin = bin64(a, b, 0.0, prm.k36, 36);
      }
      // float32 magnitudes: this histogram only decides a certified argmax
      const float s2 = __fmaf_rn(af, af, __fmul_rn(bf, bf));
      mgf[j] = s2 > 0.0f ? __fmul_rn(s2, rsqrtf(s2)) : 0.0f;
      bn[j] = bin;
    }
    {
      // NS sums stay below 2^31: scale 2^(157 - LOG - e) for a largest magnitude < 2^(e - 126)
      float mx = mgf[0];
#pragma unroll
      for (int j = 1; j < SPL; ++j) mx = fmaxf(mx, mgf[j]);
      const unsigned eb = __reduce_max_sync(0xffffffffu, __float_as_uint(mx)) >> 23;
      const float f36 = eb == 0u ? 1.0f : __uint_as_float((unsigned)min(max(284 - LOG - (int)eb, 1), 254) << 23);
#pragma unroll
      for (int j = 0; j < SPL; ++j) atomicAdd(h36 + bn[j], __float2uint_rn(__fmul_rn(mgf[j], f36)));
    }
    __syncwarp();
    // argmax with a clear lead (else the whole keypoint is redone in float64)
    const unsigned v1 = h36[lane], v2 = lane < 4 ? h36[lane + 32] : 0u;
    const unsigned k1 = (__float_as_uint((float)v1) & ~63u) | (63u - lane);
    const unsigned k2 = lane < 4 ? ((__float_as_uint((float)v2) & ~63u) | (31u - lane)) : 0u;
    const unsigned top = __reduce_max_sync(0xffffffffu, max(k1, k2));
    const unsigned sec = __reduce_max_sync(0xffffffffu, max(k1 == top ? 0u : k1, k2 == top ? 0u : k2));
    const float tv = __uint_as_float(top & ~63u), sv = __uint_as_float(sec & ~63u);
    if (!(sv < tv * 0.99994f)) {  // warp-uniform
      __syncwarp();
      return false;
    }
    const int hk = 63 - (int)(top & 63u);
    const double theta0 = prm.theta[hk], ct = prm.cos_t[hk], st = prm.sin_t[hk];
    const float theta0f = (float)theta0;
    // --- rotated grid (descriptor.py:164-216, 237-240)
    const double xmin = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, ct >= 0.0 ? -half : half)), __dmul_rn(st, st >= 0.0 ? half : -half));
    const double xmax = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, ct >= 0.0 ? half : -half)), __dmul_rn(st, st >= 0.0 ? -half : half));
    const double ymin = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, st >= 0.0 ? -half : half)), __dmul_rn(ct, ct >= 0.0 ? -half : half));
    const double ymax = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, st >= 0.0 ? half : -half)), __dmul_rn(ct, ct >= 0.0 ? half : -half));
    const int pr0 = max((int)floor(ymin), 1), pr1 = min((int)ceil(ymax), nr - 2);
    const int pc0 = max((int)floor(xmin), 1), pc1 = min((int)ceil(xmax), nc - 2);
    const int xcap = max(pc1 - pc0 - 1, 0), ycap = max(pr1 - pr0 - 1, 0);
    const double xhi = (double)(nc - 2), yhi = (double)(nr - 2);
    const double dpc0 = (double)pc0, dpr0 = (double)pr0;
    // the patch lies in the staged box and is at least 2 x 2 (cannot fail for
    // images >= 16 x 16; be safe)
    if (pr0 - 1 < BR || pr1 + 1 >= BR + BX || pc0 - 1 < BC || pc1 + 1 >= BC + BX || pr1 <= pr0 || pc1 <= pc0) {
      __syncwarp();
      return false;
    }
    // gradient fields fa(y, x) = P(y+1, x) - P(y-1, x), fb(y, x) = P(y, x+1) -
    // P(y, x-1) of the patch (descriptor.py:192-193), formed at the four
    // corners of each sample straight from the staged raster
    const double* pb = stage + (pr0 - 1 - BR) * SP + (pc0 - 1 - BC);  // P(pr0 - 1, pc0 - 1)
    const double c0t = ct, s0t = -st;  // cos / sin of theta0
    const bool all_valid = xmin >= 1.0 && xmax <= xhi && ymin >= 1.0 && ymax <= yhi;  // corner extent inside
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      const int s = lane + 32 * j, iv = s / W, iu = s % W;
      const double u = (double)iu - half, v = (double)iv - half;  // exact
      const double x = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, u)), __dmul_rn(st, v));
      const double y = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, u)), __dmul_rn(ct, v));
      mg[j] = 0.0;
      bn[j] = 0;
      if (!all_valid && !(x >= 1.0 && x <= xhi && y >= 1.0 && y <= yhi)) continue;  // hypot * valid = 0
      // The reference clips x to [pc0, pc1] first; for a valid sample that is
      // the identity: x >= xmin and x <= xmax hold exactly (same rounded
      // expressions, monotone in u and v), and the image clamps of pc0 / pc1
      // are the validity bounds themselves.
      const double lx = __dsub_rn(x, dpc0), ly = __dsub_rn(y, dpr0);
      const int x0 = max(min((int)floor(lx), xcap), 0), y0 = max(min((int)floor(ly), ycap), 0);
      const double fxx = __dsub_rn(lx, (double)x0), fyy = __dsub_rn(ly, (double)y0);
      // corners (y0, x0) .. (y0 + 1, x0 + 1): x0 <= pc1 - pc0 - 1 since pc1 > pc0
      const double* q = pb + y0 * SP + x0;  // P(pr0 + y0 - 1, pc0 + x0 - 1)
      const double p01 = q[1], p02 = q[2];
      const double p10 = q[SP], p11 = q[SP + 1], p12 = q[SP + 2], p13 = q[SP + 3];
      const double p20 = q[2 * SP], p21 = q[2 * SP + 1], p22 = q[2 * SP + 2], p23 = q[2 * SP + 3];
      const double p31 = q[3 * SP + 1], p32 = q[3 * SP + 2];
      const double a00 = __dsub_rn(p21, p01), a01 = __dsub_rn(p22, p02);
      const double a10 = __dsub_rn(p31, p11), a11 = __dsub_rn(p32, p12);
      const double b00 = __dsub_rn(p12, p10), b01 = __dsub_rn(p13, p11);
      const double b10 = __dsub_rn(p22, p20), b11 = __dsub_rn(p23, p21);
      const double sy = __dsub_rn(1.0, fyy), sx = __dsub_rn(1.0, fxx);
      // bilinear blend with shared corner weights and FMAs (differs from the
      // reference's left-to-right products by ~1 ulp; the bar is 1e-4)
      const double w00 = __dmul_rn(sy, sx), w01 = __dmul_rn(sy, fxx), w10 = __dmul_rn(fyy, sx), w11 = __dmul_rn(fyy, fxx);
      const double as = __fma_rn(a11, w11, __fma_rn(a10, w10, __fma_rn(a01, w01, __dmul_rn(a00, w00))));
      const double bs = __fma_rn(b11, w11, __fma_rn(b10, w10, __fma_rn(b01, w01, __dmul_rn(b00, w00))));
      const float af = (float)as, bf = (float)bs;
      int ob;  // octant of the theta0-rotated gradient (ct = cos theta0, st = -sin theta0)
      if (!octant_bin(__fmaf_rn(af, (float)ct, -__fmul_rn(bf, (float)st)),
                      __fmaf_rn(bf, (float)ct, __fmul_rn(af, (float)st)), ob)) {
        const float xb = wrap_two_pi_f(fast_atan2f(bf, af) - theta0f) * 1.2732395447351628f;
        const int m = min(max(__float2int_rn(xb), 0), 8);
        const double ce = __dsub_rn(__dmul_rn(c0t, prm.c8[m]), __dmul_rn(s0t, prm.s8[m]));
        const double se = __dadd_rn(__dmul_rn(s0t, prm.c8[m]), __dmul_rn(c0t, prm.s8[m]));
        ob = side_bin(as, bs, ce, se, m, 8);
        if (ob < 0) ob = bin64(as, bs, theta0, prm.k8, 8);
      }
      mg[j] = __dsqrt_rn(__fma_rn(as, as, __dmul_rn(bs, bs)));
      bn[j] = ((iv / WS) * 4 + iu / WS) * 8 + ob;
    }
  }
  double mx = mg[0];
#pragma unroll
  for (int j = 1; j < SPL; ++j) mx = fmax(mx, mg[j]);
  const double fx = fx_scale52_warp<LOG>(mx);
#pragma unroll
  for (int j = 0; j < SPL; ++j) h2_add<LIMB>(h128, D, bn[j], mg[j], fx);
  __syncwarp();
  // --- L2 normalise, clamp at 0.2, renormalise (descriptor.py:250-255).
  // Lane l owns bins 4l..4l+3 (one 16-byte shared load per limb array, one
  // 16-byte store of the float32 row); 1/||v|| comes from rsqrt (~1 ulp).
  static_assert(D == 128, "four bins per lane");
  {
    const double inv = 1.0 / fx;  // exact (power of two)
    const uint4 lo = *reinterpret_cast<const uint4*>(h128 + 4 * lane);
    const uint4 hi = *reinterpret_cast<const uint4*>(h128 + D + 4 * lane);
    double v0 = __dmul_rn((double)(((unsigned long long)hi.x << LIMB) + lo.x), inv);
    double v1 = __dmul_rn((double)(((unsigned long long)hi.y << LIMB) + lo.y), inv);
    double v2 = __dmul_rn((double)(((unsigned long long)hi.z << LIMB) + lo.z), inv);
    double v3 = __dmul_rn((double)(((unsigned long long)hi.w << LIMB) + lo.w), inv);
    double ss = __dadd_rn(__dadd_rn(__dmul_rn(v0, v0), __dmul_rn(v1, v1)), __dadd_rn(__dmul_rn(v2, v2), __dmul_rn(v3, v3)));
#pragma unroll
    for (int o = 16; o; o >>= 1) ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    if (ss > 0.0) {
      const double r1 = rsqrt(ss);
      v0 = __dmul_rn(v0, r1);
      v1 = __dmul_rn(v1, r1);
      v2 = __dmul_rn(v2, r1);
      v3 = __dmul_rn(v3, r1);
      v0 = v0 < 0.2 ? v0 : 0.2;  // non-negative values: no NaN handling needed
      v1 = v1 < 0.2 ? v1 : 0.2;
      v2 = v2 < 0.2 ? v2 : 0.2;
      v3 = v3 < 0.2 ? v3 : 0.2;
      double s2 =
          __dadd_rn(__dadd_rn(__dmul_rn(v0, v0), __dmul_rn(v1, v1)), __dadd_rn(__dmul_rn(v2, v2), __dmul_rn(v3, v3)));
#pragma unroll
      for (int o = 16; o; o >>= 1) s2 = __dadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, o));
      const double r2 = rsqrt(s2);
      v0 = __dmul_rn(v0, r2);
      v1 = __dmul_rn(v1, r2);
      v2 = __dmul_rn(v2, r2);
      v3 = __dmul_rn(v3, r2);
    } else {
      v0 = v1 = v2 = v3 = 0.0;
    }
    if (o32)
      reinterpret_cast<float4*>(o32)[lane] =
          make_float4(__double2float_rn(v0), __double2float_rn(v1), __double2float_rn(v2), __double2float_rn(v3));
    if (o64) {
      reinterpret_cast<double2*>(o64)[2 * lane] = make_double2(v0, v1);
      reinterpret_cast<double2*>(o64)[2 * lane + 1] = make_double2(v2, v3);
    }
  }
  __syncwarp();
  return true;
}

template <class Img>
__global__ void __launch_bounds__(kWarps * 32, 3) describe_kernel(Img img, int64_t img_stride, int B,
                                                                  const int32_t* __restrict__ kp_row,
                                                                  const int32_t* __restrict__ kp_col,
                                                                  const int32_t* __restrict__ kp_scale,
                                                                  int32_t default_scale,
                                                                  const int32_t* __restrict__ counts, int64_t cap,
                                                                  DescParams prm, float* __restrict__ out32,
                                                                  double* __restrict__ out64,
                                                                  const int64_t* __restrict__ work,
                                                                  const unsigned long long* __restrict__ n_work) {
  extern __shared__ double dsm[];
  const int wid = threadIdx.x >> 5;
  const int D = prm.D;
  double* stage = dsm + wid * kStageDoubles;
  unsigned* hw = reinterpret_cast<unsigned*>(dsm + kWarps * kStageDoubles) + wid * 3 * (D + 36);
  const int64_t total = work ? (int64_t)*n_work : (int64_t)B * cap;
  const bool small = total < (1ll << 31);
  int w_def = -1, lb_def = 0;
  double fx_def = 0.0;
  for (int s = 0; s < prm.n_scales; ++s)
    if (prm.scale[s] == default_scale) { w_def = prm.w[s]; fx_def = prm.fx[s]; lb_def = prm.lb[s]; }
  for (int64_t gi = (int64_t)blockIdx.x * kWarps + wid; gi < total; gi += (int64_t)gridDim.x * kWarps) {
    const int64_t g = work ? work[gi] : gi;
    const int b = small ? (int)((unsigned)g / (unsigned)cap) : (int)(g / cap);
    const int64_t i = g - (int64_t)b * cap;
    if (counts && i >= counts[b]) continue;
    Img im = img;
    im.p = img.p + (int64_t)b * img_stride * decltype(img)::kElem;
    const int row = kp_row[g], col = kp_col[g];
    int w = w_def, lb = lb_def;
    double fx = fx_def;
    if (kp_scale) {
      const int scale = kp_scale[g];
      w = -1;
      for (int s = 0; s < prm.n_scales; ++s)
        if (prm.scale[s] == scale) { w = prm.w[s]; fx = prm.fx[s]; lb = prm.lb[s]; }
    }
    if (w < 0) continue;  // scale outside the set (unwritten); any position is fine (_fit_region clamps)
    float* o32 = out32 ? out32 + g * D : nullptr;
    double* o64 = out64 ? out64 + g * D : nullptr;
    constexpr bool kFast = std::is_same<Img, RampU8>::value;
    if (prm.d == 4 && w == 8) {
      describe_keypoint<8, 4, kFast>(im, row, col, w, 4, fx, lb, prm, hw, stage, o32, o64);
    } else if (prm.d == 4 && w == 16) {
      describe_keypoint<16, 4, kFast>(im, row, col, w, 4, fx, lb, prm, hw, stage, o32, o64);
    } else if (prm.d == 4 && w == 32) {
      describe_keypoint<32, 4, kFast>(im, row, col, w, 4, fx, lb, prm, hw, stage, o32, o64);
    } else {
      describe_keypoint<0, 0, kFast>(im, row, col, w, prm.d, fx, lb, prm, hw, stage, o32, o64);
    }
  }
}

// (image, slot) walk of a grid-stride loop: slot += qstep * cap + rstep
__device__ __forceinline__ void advance_slot(int& b, int64_t& i, int qstep, int64_t rstep, int64_t cap) {
  b += qstep;
  i += rstep;
  if (i >= cap) {
    i -= cap;
    ++b;
  }
}

// 8-bit rasters: w = 8 keypoints through the lean fast path (more resident
// warps); everything else -- other region sides and 36-bin near-ties -- is
// queued for describe_kernel.
constexpr int kFastWarps = 8;
#ifndef PS_FAST_MINB
#define PS_FAST_MINB 4
#endif
constexpr int kFastHist = 2 * (128 + 36);

template <int W, class Img>
__global__ void __launch_bounds__(kFastWarps * 32, W == 8 ? PS_FAST_MINB : 3) describe_fast_u8(Img img, int64_t img_stride, int B,
                                                                       const int32_t* __restrict__ kp_row,
                                                                       const int32_t* __restrict__ kp_col,
                                                                       const int32_t* __restrict__ kp_scale,
                                                                       int32_t default_scale,
                                                                       const int32_t* __restrict__ counts, int64_t cap,
                                                                       DescParams prm, float* __restrict__ out32,
                                                                       double* __restrict__ out64,
                                                                       int64_t* __restrict__ work,
                                                                       unsigned long long* __restrict__ n_work) {
  extern __shared__ double dsm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int BX = FastBox<W>::kBox;
  double* stage = dsm + wid * FastBox<W>::kTotal;
  unsigned* hw = reinterpret_cast<unsigned*>(dsm + kFastWarps * FastBox<W>::kTotal) + wid * kFastHist;
  const int n_fast = W == 8 ? prm.n_w8 : prm.n_w16;
  const int* fast_scale = W == 8 ? prm.w8_scale : prm.w16_scale;
  const int64_t total = (int64_t)B * cap;
  const int64_t S = (int64_t)gridDim.x * kFastWarps;
  // grid-stride over (image b, slot i); (b, i) advance without a division
  int64_t g = (int64_t)blockIdx.x * kFastWarps + wid;
  int b = (int)(g / cap);
  int64_t i = g - (int64_t)b * cap;
  const int qstep = (int)(S / cap);
  const int64_t rstep = S - (int64_t)qstep * cap;
  for (; g < total; g += S, advance_slot(b, i, qstep, rstep, cap)) {
    if (counts && i >= counts[b]) continue;
    Img im = img;
    im.p = img.p + (int64_t)b * img_stride * decltype(img)::kElem;
    const int row = kp_row[g], col = kp_col[g];
    if (row < 0 || row >= im.nr || col < 0 || col >= im.nc) {  // outside the image: general kernel (it clamps)
      if (lane == 0) work[atomicAdd(n_work, 1ull)] = g;
      continue;
    }
    bool fast = (W == 8 ? prm.default_w8 : prm.default_w16) && im.nr >= BX && im.nc >= BX;
    if (kp_scale) {
      const int scale = kp_scale[g];
      fast = false;
      for (int k = 0; k < n_fast; ++k) fast |= fast_scale[k] == scale;
      fast &= im.nr >= BX && im.nc >= BX;
    }
    bool ok = false;
    if (fast)
      ok = describe_keypoint_w8u8<W>(im, row, col, prm, hw, stage, out32 ? out32 + g * 128 : nullptr,
                                     out64 ? out64 + g * 128 : nullptr);
    if (!ok && lane == 0) work[atomicAdd(n_work, 1ull)] = g;  // other sides and near-ties: general kernel
  }
}

__global__ void max_abs_kernel(const double* __restrict__ p, int B, int nr, int nc, int64_t pitch, int64_t stride,
                               unsigned long long* __restrict__ out) {
  double m = 0.0;
  const int64_t total = (int64_t)B * nr * nc;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / ((int64_t)nr * nc), rem = t % ((int64_t)nr * nc);
    const double v = fabs(p[b * stride + (rem / nc) * pitch + rem % nc]);
    m = v > m ? v : m;  // NaN ignored
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// region_size + _fit_region width on the host, with the host libm exactly as
// the reference computes it (descriptor.py:82-95, 118-128).
int region_width(int scale, double beta0, int d, int l_max, int nr, int nc, int* w_out) {
  PS_REQUIRE(scale <= l_max, PS_ERR_CONFIG, "scale %d exceeds configured l_max %d", scale, l_max);
  const double beta = beta0 * std::pow((double)scale / (double)l_max, -0.5);
  int w = (int)std::floor(beta * scale * d + 0.5);
  w = std::min(w, scale);
  w -= w % d;
  w = std::max(w, d);
  const int capw = std::min(nr, nc) - 2;
  PS_REQUIRE(capw >= d, PS_ERR_VALUE, "%dx%d image too small for a %dx%d subregion grid", nr, nc, d, d);
  if (w > capw) w = capw - capw % d;
  *w_out = w;
  return PS_OK;
}

}  // namespace
}  // namespace ps

using namespace ps;

// ---- two keypoints per warp (half-warp each) --------------------------------
// The same arithmetic as describe_keypoint_w8u8 with 16 lanes per keypoint
// (4 samples per lane per phase, 8 descriptor bins per lane): the
// per-keypoint scalar work -- centre, extents, argmax, reductions -- is issued
// once for two keypoints.  Half-warp reductions: butterflies with xor < 16 and
// full-warp REDUX over values masked to one half.
__device__ __forceinline__ unsigned half_max_u32(unsigned v, int hsel) {
  const unsigned a = __reduce_max_sync(0xffffffffu, hsel == 0 ? v : 0u);
  const unsigned b = __reduce_max_sync(0xffffffffu, hsel == 1 ? v : 0u);
  return hsel ? b : a;
}
// fixed-point scale from the half's largest magnitude (64 samples per keypoint)
__device__ __forceinline__ double fx_scale52_half(double mx, int hsel) {
  const unsigned eb = half_max_u32((unsigned)__double2hiint(mx), hsel) >> 20;
  if (eb == 0u) return 1.0;
  const int be = min(2091 - (int)eb, 2046);
  return __hiloint2double(be << 20, 0);
}


template <bool ORIENT, class Img>
__device__ __forceinline__ bool describe_pair_w8(const Img& im, int row, int col, bool act, const DescParams& prm,
                                                 unsigned* hbase, double* stage, float* __restrict__ o32,
                                                 double* __restrict__ o64) {
  constexpr int W = 8, SPL = 4, D = 128, SP = FastStage::SPP, WS = W / 4, BX = FastStage::kBox;
  const int lane = threadIdx.x & 31, hl = lane & 15, hsel = lane >> 4;
  const int nr = im.nr, nc = im.nc;
  const int r0 = min(max(row - W / 2, 1), nr - 1 - W);
  const int c0 = min(max(col - W / 2, 1), nc - 1 - W);
  constexpr double half = (double)(W - 1) / 2.0;
  const int cy2 = min(max(2 * row, 2 + (W - 1)), 2 * (nr - 2) - (W - 1));
  const int cx2 = min(max(2 * col, 2 + (W - 1)), 2 * (nc - 2) - (W - 1));
  const double cy = 0.5 * (double)cy2, cx = 0.5 * (double)cx2;
  const int BR = max(0, min((cy2 >> 1) - 7, nr - BX)), BC = max(0, min((cx2 >> 1) - 7, nc - BX));
  unsigned* h128 = hbase;
  unsigned* h36 = hbase + 2 * D;
#pragma unroll
  for (int q = hl; q < 2 * (D + 36) / 4; q += 16) reinterpret_cast<uint4*>(hbase)[q] = make_uint4(0u, 0u, 0u, 0u);
  if constexpr (std::is_same<Img, RampRGB8>::value) {
    stage_box_rgb8<BX / 2>(im, stage, SP, BR, BC, BX, BX, hl, 0);
    stage_box_rgb8<BX / 2>(im, stage, SP, BR, BC, BX, BX, hl, 1);
  } else {
    stage_box_u8<BX / 2>(im, stage, SP, BR, BC, BX, BX, hl, 0);
    stage_box_u8<BX / 2>(im, stage, SP, BR, BC, BX, BX, hl, 1);
  }
  __syncwarp();
  const double* pa = stage + (r0 - 1 - BR) * SP + (c0 - 1 - BC);
  auto axis_ab = [&](int iv, int iu, double& a, double& b) {
    a = __dsub_rn(pa[(iv + 2) * SP + iu + 1], pa[iv * SP + iu + 1]);
    b = __dsub_rn(pa[(iv + 1) * SP + iu + 2], pa[(iv + 1) * SP + iu]);
  };
  double mg[SPL];
  int bn[SPL];
  bool ok = act;
  if constexpr (!ORIENT) {
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      const int s = hl + 16 * j, iv = s / W, iu = s % W;
      double a, b;
      axis_ab(iv, iu, a, b);
      const float xb = wrap_two_pi_f(fast_atan2f((float)b, (float)a)) * 1.2732395447351628f;
      int ob;
      if (!certified_bin(xb, 8, ob)) {
        const int m = min(max(__float2int_rn(xb), 0), 8);
        ob = exact_bin(a, b, 1.0, 0.0, prm.c8[m], prm.s8[m], m, 8, 0.0, prm.k8, prm.two_pi);
      }
      mg[j] = __dsqrt_rn(__fma_rn(a, a, __dmul_rn(b, b)));
      bn[j] = ((iv / WS) * 4 + iu / WS) * 8 + ob;
    }
  } else {
    // The 36-bin histogram only decides the dominant orientation, and only
    // with a clear lead (6e-5 relative), so float32 magnitudes (~2^-22) and
    // one 32-bit fixed-point limb suffice; the descriptor's own magnitudes
    // (the rotated phase) stay float64.
    float mgf[SPL];
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      const int s = hl + 16 * j;
      double a, b;
      axis_ab(s / W, s % W, a, b);
      const float af = (float)a, bf = (float)b;
      const float x = wrap_two_pi_f(fast_atan2f(bf, af)) * 5.729577951308232f;
      int bin;
      if (!certified_bin(x, 36, bin)) {
        const int m = min(max(__float2int_rn(x), 0), 36);
        bin = exact_bin(a, b, 1.0, 0.0, prm.cb36[m], prm.sb36[m], m, 36, 0.0, prm.k36, prm.two_pi);
      }
      const float s2 = __fmaf_rn(af, af, __fmul_rn(bf, bf));
      mgf[j] = s2 > 0.0f ? __fmul_rn(s2, rsqrtf(s2)) : 0.0f;
      bn[j] = bin;
    }
    {
      // 64 sums stay below 2^31: scale 2^(151 - e) for a largest magnitude < 2^(e - 126)
      const float mx = fmaxf(fmaxf(mgf[0], mgf[1]), fmaxf(mgf[2], mgf[3]));
      const unsigned eb = half_max_u32(__float_as_uint(mx), hsel) >> 23;
      const float f36 = eb == 0u ? 1.0f : __uint_as_float((unsigned)min(max(278 - (int)eb, 1), 254) << 23);
#pragma unroll
      for (int j = 0; j < SPL; ++j) atomicAdd(h36 + bn[j], __float2uint_rn(__fmul_rn(mgf[j], f36)));
    }
    __syncwarp();
    // argmax with a clear lead over the half's 36 bins (3 per lane)
    unsigned k1 = 0u, k2 = 0u;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int bin = hl + 16 * t;
      const unsigned k = bin < 36 ? ((__float_as_uint((float)h36[bin]) & ~63u) | (63u - bin)) : 0u;
      if (k > k1) { k2 = k1; k1 = k; } else if (k > k2) { k2 = k; }
    }
    const unsigned top = half_max_u32(k1, hsel);
    const unsigned sec = half_max_u32(k1 == top ? k2 : k1, hsel);
    const float tv = __uint_as_float(top & ~63u), sv = __uint_as_float(sec & ~63u);
    ok = ok && (sv < tv * 0.99994f);
    const int hk = 63 - (int)(top & 63u);
    const double theta0 = prm.theta[hk], ct = prm.cos_t[hk], st = prm.sin_t[hk];
    const float theta0f = (float)theta0, ctf = (float)ct, stf = (float)st;
    const double xmin = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, ct >= 0.0 ? -half : half)), __dmul_rn(st, st >= 0.0 ? half : -half));
    const double xmax = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, ct >= 0.0 ? half : -half)), __dmul_rn(st, st >= 0.0 ? -half : half));
    const double ymin = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, st >= 0.0 ? -half : half)), __dmul_rn(ct, ct >= 0.0 ? -half : half));
    const double ymax = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, st >= 0.0 ? half : -half)), __dmul_rn(ct, ct >= 0.0 ? half : -half));
    int pr0 = max((int)floor(ymin), 1), pr1 = min((int)ceil(ymax), nr - 2);
    int pc0 = max((int)floor(xmin), 1), pc1 = min((int)ceil(xmax), nc - 2);
    if (pr0 - 1 < BR || pr1 + 1 >= BR + BX || pc0 - 1 < BC || pc1 + 1 >= BC + BX || pr1 <= pr0 || pc1 <= pc0) {
      ok = false;  // cannot happen for images >= 16 x 16; keep the addresses inside the box
      pr0 = BR + 1; pr1 = BR + 2; pc0 = BC + 1; pc1 = BC + 2;
    }
    if (!__any_sync(0xffffffffu, ok)) return false;
    const int xcap = max(pc1 - pc0 - 1, 0), ycap = max(pr1 - pr0 - 1, 0);
    const double xhi = (double)(nc - 2), yhi = (double)(nr - 2);
    const double dpc0 = (double)pc0, dpr0 = (double)pr0;
    const double* pb = stage + (pr0 - 1 - BR) * SP + (pc0 - 1 - BC);
    const double c0t = ct, s0t = -st;
    // x and y are monotone in u and v under round-to-nearest, so the grid's
    // corner extent bounds every sample: one test per keypoint when it is inside
    const bool all_valid = xmin >= 1.0 && xmax <= xhi && ymin >= 1.0 && ymax <= yhi;
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      const int s = hl + 16 * j, iv = s / W, iu = s % W;
      const double u = (double)iu - half, v = (double)iv - half;
      const double x = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, u)), __dmul_rn(st, v));
      const double y = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, u)), __dmul_rn(ct, v));
      mg[j] = 0.0;
      bn[j] = 0;
      if (!all_valid && !(x >= 1.0 && x <= xhi && y >= 1.0 && y <= yhi)) continue;
      const double lx = __dsub_rn(x, dpc0), ly = __dsub_rn(y, dpr0);
      const int x0 = max(min((int)floor(lx), xcap), 0), y0 = max(min((int)floor(ly), ycap), 0);
      const double fxx = __dsub_rn(lx, (double)x0), fyy = __dsub_rn(ly, (double)y0);
      const double* q = pb + y0 * SP + x0;
      const double p01 = q[1], p02 = q[2];
      const double p10 = q[SP], p11 = q[SP + 1], p12 = q[SP + 2], p13 = q[SP + 3];
      const double p20 = q[2 * SP], p21 = q[2 * SP + 1], p22 = q[2 * SP + 2], p23 = q[2 * SP + 3];
      const double p31 = q[3 * SP + 1], p32 = q[3 * SP + 2];
      const double a00 = __dsub_rn(p21, p01), a01 = __dsub_rn(p22, p02);
      const double a10 = __dsub_rn(p31, p11), a11 = __dsub_rn(p32, p12);
      const double b00 = __dsub_rn(p12, p10), b01 = __dsub_rn(p13, p11);
      const double b10 = __dsub_rn(p22, p20), b11 = __dsub_rn(p23, p21);
      const double sy = __dsub_rn(1.0, fyy), sx = __dsub_rn(1.0, fxx);
      const double w00 = __dmul_rn(sy, sx), w01 = __dmul_rn(sy, fxx), w10 = __dmul_rn(fyy, sx), w11 = __dmul_rn(fyy, fxx);
      const double as = __fma_rn(a11, w11, __fma_rn(a10, w10, __fma_rn(a01, w01, __dmul_rn(a00, w00))));
      const double bs = __fma_rn(b11, w11, __fma_rn(b10, w10, __fma_rn(b01, w01, __dmul_rn(b00, w00))));
      // orientation relative to theta0: rotate by -theta0 (ct = cos theta0, st = -sin theta0), octant test
      const float af = (float)as, bf = (float)bs;
      int ob;
      if (!octant_bin(__fmaf_rn(af, ctf, -__fmul_rn(bf, stf)), __fmaf_rn(bf, ctf, __fmul_rn(af, stf)), ob)) {
        const float xb = wrap_two_pi_f(fast_atan2f(bf, af) - theta0f) * 1.2732395447351628f;
        const int m = min(max(__float2int_rn(xb), 0), 8);
        ob = exact_bin(as, bs, c0t, s0t, prm.c8[m], prm.s8[m], m, 8, theta0, prm.k8, prm.two_pi);
      }
      mg[j] = __dsqrt_rn(__fma_rn(as, as, __dmul_rn(bs, bs)));
      bn[j] = ((iv / WS) * 4 + iu / WS) * 8 + ob;
    }
  }
  const double fx = fx_scale52_half(fmax(fmax(mg[0], mg[1]), fmax(mg[2], mg[3])), hsel);
#pragma unroll
  for (int j = 0; j < SPL; ++j) h2_add(h128, D, bn[j], mg[j], fx);
  __syncwarp();
  // L2 normalise, clamp at 0.2, renormalise: lane owns bins 8 hl .. 8 hl + 7
  const double inv = 1.0 / fx;
  double v[8];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const uint4 lo = *reinterpret_cast<const uint4*>(h128 + 8 * hl + 4 * t);
    const uint4 hi = *reinterpret_cast<const uint4*>(h128 + D + 8 * hl + 4 * t);
    v[4 * t + 0] = __dmul_rn((double)(((unsigned long long)hi.x << kLimb) + lo.x), inv);
    v[4 * t + 1] = __dmul_rn((double)(((unsigned long long)hi.y << kLimb) + lo.y), inv);
    v[4 * t + 2] = __dmul_rn((double)(((unsigned long long)hi.z << kLimb) + lo.z), inv);
    v[4 * t + 3] = __dmul_rn((double)(((unsigned long long)hi.w << kLimb) + lo.w), inv);
  }
  // two interleaved partial sums halve the dependent FMA chains (the order
  // is immaterial at the 1e-4 bar: the reference's own norm is a BLAS ddot)
  double sa = __dmul_rn(v[0], v[0]), sb = __dmul_rn(v[1], v[1]);
#pragma unroll
  for (int t = 2; t < 8; t += 2) {
    sa = __fma_rn(v[t], v[t], sa);
    sb = __fma_rn(v[t + 1], v[t + 1], sb);
  }
  double ss = __dadd_rn(sa, sb);
#pragma unroll
  for (int o = 8; o; o >>= 1) ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
  if (ss > 0.0) {
    const double r1 = rsqrt(ss);
    double s2a = 0.0, s2b = 0.0;
#pragma unroll
    for (int t = 0; t < 8; t += 2) {
      const double w0 = __dmul_rn(v[t], r1), w1 = __dmul_rn(v[t + 1], r1);
      v[t] = fmin(w0, 0.2);
      v[t + 1] = fmin(w1, 0.2);
      s2a = __fma_rn(v[t], v[t], s2a);
      s2b = __fma_rn(v[t + 1], v[t + 1], s2b);
    }
    double s2 = __dadd_rn(s2a, s2b);
#pragma unroll
    for (int o = 8; o; o >>= 1) s2 = __dadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, o));
    const double r2 = rsqrt(s2);
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] = __dmul_rn(v[t], r2);
  } else {
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] = 0.0;
  }
  if (ok) {
    if (o32) {
      float4* d = reinterpret_cast<float4*>(o32) + 2 * hl;
      d[0] = make_float4(__double2float_rn(v[0]), __double2float_rn(v[1]), __double2float_rn(v[2]), __double2float_rn(v[3]));
      d[1] = make_float4(__double2float_rn(v[4]), __double2float_rn(v[5]), __double2float_rn(v[6]), __double2float_rn(v[7]));
    }
    if (o64) {
      double2* d = reinterpret_cast<double2*>(o64) + 4 * hl;
#pragma unroll
      for (int t = 0; t < 4; ++t) d[t] = make_double2(v[2 * t], v[2 * t + 1]);
    }
  }
  __syncwarp();
  return ok;
}

constexpr int kPairWarps = 8;
#ifndef PS_PAIR_BLOCKS_PER_SM
// Grid cap of the pair kernel in blocks per SM (3 are resident).  The grid
// stride decides which keypoints are in flight together: with many short
// grid-stride sweeps the resident blocks work on consecutive slots (their
// 16x16 boxes overlap and the descriptor rows are written in order), with
// one block per 8 pairs the block set-up dominates.  A/B on C2 (64 images):
// 12 -> 9.79 ms, 48 -> 9.47, 100 -> 9.33, 200 -> 9.25, 400 -> 9.29,
// 1200 -> 9.71, uncapped -> 9.84.
#define PS_PAIR_BLOCKS_PER_SM 200
#endif
#ifndef PS_W16_BLOCKS_PER_SM
#define PS_W16_BLOCKS_PER_SM 100  // grid cap of the w = 16 kernel (A/B: 16 -> 0.707 ms, 100 -> 0.685 per 16 images)
#endif
template <bool ORIENT, class Img>
__global__ void __launch_bounds__(kPairWarps * 32, 3) describe_pair_kernel(Img img, int64_t img_stride, int B,
                                                                           const int32_t* __restrict__ kp_row,
                                                                           const int32_t* __restrict__ kp_col,
                                                                           const int32_t* __restrict__ kp_scale,
                                                                           const int32_t* __restrict__ counts,
                                                                           int64_t cap, DescParams prm,
                                                                           float* __restrict__ out32,
                                                                           double* __restrict__ out64,
                                                                           int64_t* __restrict__ work,
                                                                           unsigned long long* __restrict__ n_work,
                                                                           const int64_t* __restrict__ in_work,
                                                                           const unsigned long long* __restrict__ in_n) {
  extern __shared__ double dsm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, hsel = lane >> 4, hl = lane & 15;
  double* stage = dsm + (2 * wid + hsel) * FastStage::kTotal;
  unsigned* hw = reinterpret_cast<unsigned*>(dsm + 2 * kPairWarps * FastStage::kTotal) + (2 * wid + hsel) * kFastHist;
  if (in_work) {  // the slots a previous kernel queued (float32 kernel: border keypoints, other sides)
    const int64_t nin = (int64_t)*in_n;
    for (int64_t pi = (int64_t)blockIdx.x * kPairWarps + wid; 2 * pi < nin; pi += (int64_t)gridDim.x * kPairWarps) {
      const bool live = 2 * pi + hsel < nin;
      const int64_t g = live ? in_work[2 * pi + hsel] : 0;
      const int b = (int)(g / cap);
      int row = live ? kp_row[g] : 8, col = live ? kp_col[g] : 8;
      bool fast = live && img.nr >= FastStage::kBox && img.nc >= FastStage::kBox && row >= 0 && row < img.nr &&
                  col >= 0 && col < img.nc;
      if (fast) {
        if (kp_scale) {
          const int scale = kp_scale[g];
          bool f = false;
          for (int k = 0; k < prm.n_w8; ++k) f |= prm.w8_scale[k] == scale;
          fast = f;
        } else {
          fast = prm.default_w8;
        }
      }
      if (!__any_sync(0xffffffffu, fast)) {
        if (live && hl == 0) work[atomicAdd(n_work, 1ull)] = g;
        continue;
      }
      Img im = img;
      im.p = img.p + (int64_t)(fast ? b : 0) * img_stride * decltype(img)::kElem;
      if (!fast) { row = 8; col = 8; }
      const bool ok = describe_pair_w8<ORIENT>(im, row, col, fast, prm, hw, stage,
                                               out32 ? out32 + g * 128 : nullptr, out64 ? out64 + g * 128 : nullptr);
      if (live && !ok && hl == 0) work[atomicAdd(n_work, 1ull)] = g;
    }
    return;
  }
  const int64_t total = (int64_t)B * cap;
  const int64_t npairs = (total + 1) / 2;
  const bool box_ok = img.nr >= FastStage::kBox && img.nc >= FastStage::kBox;
  // (image b, slot i) of this half's slot g advance without a division
  const int64_t gstep = 2 * (int64_t)gridDim.x * kPairWarps;
  int64_t gi0 = 2 * ((int64_t)blockIdx.x * kPairWarps + wid) + hsel;
  int bcur = (int)(gi0 / cap);
  int64_t icur = gi0 - (int64_t)bcur * cap;
  const int qstep = (int)(gstep / cap);  // gstep = qstep * cap + rstep: O(1) per step for any cap
  const int64_t rstep = gstep - (int64_t)qstep * cap;
  for (int64_t pi = (int64_t)blockIdx.x * kPairWarps + wid; pi < npairs;
       pi += (int64_t)gridDim.x * kPairWarps, advance_slot(bcur, icur, qstep, rstep, cap)) {
    const int64_t g = 2 * pi + hsel;  // this half's slot
    bool live = g < total;
    int b = 0;
    if (live) {
      b = bcur;
      live = !counts || icur < counts[b];
    }
    int row = live ? kp_row[g] : 8, col = live ? kp_col[g] : 8;
    // keypoints outside the image (the reference translates their region
    // inward, descriptor.py:118-131) go to the general kernel
    bool fast = live && box_ok && row >= 0 && row < img.nr && col >= 0 && col < img.nc;
    if (fast) {
      if (kp_scale) {
        const int scale = kp_scale[g];
        bool f = false;
        for (int k = 0; k < prm.n_w8; ++k) f |= prm.w8_scale[k] == scale;
        fast = f;
      } else {
        fast = prm.default_w8;
      }
    }
    if (!__any_sync(0xffffffffu, fast)) {  // neither keypoint takes the fast path
      if (live && hl == 0) work[atomicAdd(n_work, 1ull)] = g;
      continue;
    }
    if (!fast) { row = 8; col = 8; b = 0; }
    Img im = img;
    im.p = img.p + (int64_t)b * img_stride * decltype(img)::kElem;
    const bool ok = describe_pair_w8<ORIENT>(im, row, col, fast, prm, hw, stage, out32 ? out32 + g * 128 : nullptr,
                                     out64 ? out64 + g * 128 : nullptr);
    if (live && !ok && hl == 0) work[atomicAdd(n_work, 1ull)] = g;  // other sides and near-ties: general kernel
  }
}

// 8-bit rasters (grey or RGB): w = 8 keypoints through the fast kernel, the
// rest (other sides, 36-bin near-ties) queued for the general kernel.
template <class Img>
int launch_fast(const Img& im, const ps_image_batch* img, const ps_keypoints* kp, int32_t default_scale,
                const DescParams& prm, float* out_desc32, double* out_desc64, int64_t total, size_t shmem,
                int policy, bool window_slots, cudaStream_t s) {
  if (policy == PS_DESCRIBE_GENERAL) {  // the general kernel for every keypoint
    int64_t blocks = (total + kWarps - 1) / kWarps;
    if (blocks > 148 * 8) blocks = 148 * 8;
    describe_kernel<Img><<<(unsigned)blocks, kWarps * 32, shmem, s>>>(im, img->image_stride, img->batch, kp->row,
                                                                      kp->col, kp->scale, default_scale, kp->count,
                                                                      kp->cap, prm, out_desc32, out_desc64, nullptr,
                                                                      nullptr);
    PS_LAUNCHED("describe_kernel");
    return check_cuda("describe_kernel");
  }
  int64_t* work = nullptr;
  static std::atomic<unsigned long long> pool_set{0};  // per device: keep freed queue memory in the pool
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(pool_set.load() & bit)) {  // idempotent: racing threads set the same attribute
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_set.fetch_or(bit);
  }
  cudaMallocAsync(&work, (size_t)total * sizeof(int64_t) + 16, s);
  int st = check_cuda("cudaMallocAsync(describe work list)");
  if (st) return st;
  unsigned long long* n_work = reinterpret_cast<unsigned long long*>(work + total);
  cudaMemsetAsync(n_work, 0, sizeof(unsigned long long), s);
  const bool pair = policy != PS_DESCRIBE_SINGLE;
  // float32-only output: the float32 throughput kernel (describe_f32.cu) for
  // w = 8 keypoints; float64 output or PS_DESCRIBE_PRECISE: the float64 kernels
  const bool f32 = policy == PS_DESCRIBE_AUTO && out_desc64 == nullptr && out_desc32 != nullptr && prm.d == 4 &&
                   prm.n_w8 > 0;
  if (f32) {
    // float32 kernel -> its queue (border keypoints, other sides) through the
    // float64 pair kernel -> what that queues through the general kernel
    int st2 = launch_describe_f32(im, img, kp, default_scale, prm, out_desc32, window_slots, work, n_work, s);
    if (st2) return st2;
    int64_t* work2 = nullptr;
    cudaMallocAsync(&work2, (size_t)total * sizeof(int64_t) + 16, s);
    st2 = check_cuda("cudaMallocAsync(describe work list 2)");
    if (st2) return st2;
    unsigned long long* n_work2 = reinterpret_cast<unsigned long long*>(work2 + total);
    cudaMemsetAsync(n_work2, 0, sizeof(unsigned long long), s);
    const size_t pshmem =
        (size_t)2 * kPairWarps * (FastStage::kTotal * sizeof(double) + kFastHist * sizeof(unsigned));
    auto kern = prm.orient ? describe_pair_kernel<true, Img> : describe_pair_kernel<false, Img>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pshmem);
    kern<<<148 * 3, kPairWarps * 32, pshmem, s>>>(im, img->image_stride, img->batch, kp->row, kp->col, kp->scale,
                                                  kp->count, kp->cap, prm, out_desc32, out_desc64, work2, n_work2,
                                                  work, n_work);
    PS_LAUNCHED("describe_pair_kernel(queued)");
    describe_kernel<Img><<<148 * 2, kWarps * 32, shmem, s>>>(im, img->image_stride, img->batch, kp->row, kp->col,
                                                             kp->scale, default_scale, kp->count, kp->cap, prm,
                                                             out_desc32, out_desc64, work2, n_work2);
    PS_LAUNCHED("describe_kernel(queued)");
    cudaFreeAsync(work2, s);
    cudaFreeAsync(work, s);
    return check_cuda("cudaFreeAsync");
  } else if (prm.n_w8 == 0 && prm.n_w16 > 0) {  // w = 16 scales only (e.g. the default 32..128 windows)
    const size_t fshmem = (size_t)kFastWarps * (FastBox<16>::kTotal * sizeof(double) + kFastHist * sizeof(unsigned));
    cudaFuncSetAttribute(describe_fast_u8<16, Img>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fshmem);
    int64_t fblocks = (total + kFastWarps - 1) / kFastWarps;
    if (fblocks > 148 * PS_W16_BLOCKS_PER_SM) fblocks = 148 * PS_W16_BLOCKS_PER_SM;
    describe_fast_u8<16, Img><<<(unsigned)fblocks, kFastWarps * 32, fshmem, s>>>(
        im, img->image_stride, img->batch, kp->row, kp->col, kp->scale, default_scale, kp->count, kp->cap, prm,
        out_desc32, out_desc64, work, n_work);
    PS_LAUNCHED("describe_fast_u8<16>");
  } else if (pair) {
    const size_t pshmem =
        (size_t)2 * kPairWarps * (FastStage::kTotal * sizeof(double) + kFastHist * sizeof(unsigned));
    auto kern = prm.orient ? describe_pair_kernel<true, Img> : describe_pair_kernel<false, Img>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pshmem);
    int64_t pblocks = ((total + 1) / 2 + kPairWarps - 1) / kPairWarps;
    if (pblocks > 148 * PS_PAIR_BLOCKS_PER_SM) pblocks = 148 * PS_PAIR_BLOCKS_PER_SM;
    kern<<<(unsigned)pblocks, kPairWarps * 32, pshmem, s>>>(im, img->image_stride, img->batch, kp->row, kp->col,
                                                             kp->scale, kp->count, kp->cap, prm, out_desc32,
                                                             out_desc64, work, n_work, nullptr, nullptr);
    PS_LAUNCHED("describe_pair_kernel");
  } else {
    const size_t fshmem = (size_t)kFastWarps * (FastStage::kTotal * sizeof(double) + kFastHist * sizeof(unsigned));
    cudaFuncSetAttribute(describe_fast_u8<8, Img>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fshmem);
    int64_t fblocks = (total + kFastWarps - 1) / kFastWarps;
    if (fblocks > 148 * 16) fblocks = 148 * 16;
    describe_fast_u8<8, Img><<<(unsigned)fblocks, kFastWarps * 32, fshmem, s>>>(
        im, img->image_stride, img->batch, kp->row, kp->col, kp->scale, default_scale, kp->count, kp->cap, prm,
        out_desc32, out_desc64, work, n_work);
    PS_LAUNCHED("describe_fast_u8");
  }
  describe_kernel<Img><<<148 * 2, kWarps * 32, shmem, s>>>(im, img->image_stride, img->batch, kp->row, kp->col,
                                                           kp->scale, default_scale, kp->count, kp->cap, prm,
                                                           out_desc32, out_desc64, work, n_work);
  PS_LAUNCHED("describe_kernel(queued)");
  cudaFreeAsync(work, s);
  return check_cuda("cudaFreeAsync");
}

extern "C" int ps_describe(const ps_image_batch* img, const ps_keypoints* kp, int32_t default_scale,
                           const int32_t* host_scale_set, int32_t n_scale_set, double beta0, int32_t d, int32_t l_max,
                           int32_t orientation_normalize, float* out_desc32, double* out_desc64, void* stream) {
  return ps_describe_ex(img, kp, default_scale, host_scale_set, n_scale_set, beta0, d, l_max, orientation_normalize,
                        out_desc32, out_desc64, PS_DESCRIBE_AUTO, stream);
}

extern "C" int ps_describe_ex(const ps_image_batch* img, const ps_keypoints* kp, int32_t default_scale,
                              const int32_t* host_scale_set, int32_t n_scale_set, double beta0, int32_t d,
                              int32_t l_max, int32_t orientation_normalize, float* out_desc32, double* out_desc64,
                              int32_t policy, void* stream) {
  PS_REQUIRE(img && kp && img->data && kp->row && kp->col && host_scale_set, PS_ERR_ARGUMENT,
             "null argument to ps_describe");
  const bool window_slots = (policy & PS_DESCRIBE_WINDOW_SLOTS) != 0;
  policy &= ~PS_DESCRIBE_WINDOW_SLOTS;
  PS_REQUIRE(policy == PS_DESCRIBE_AUTO || policy == PS_DESCRIBE_GENERAL || policy == PS_DESCRIBE_SINGLE ||
                 policy == PS_DESCRIBE_PRECISE,
             PS_ERR_ARGUMENT, "unknown describe policy %d", policy);
  PS_REQUIRE(beta0 > 0, PS_ERR_CONFIG, "beta0 must be positive, got %g", beta0);
  PS_REQUIRE(d >= 1, PS_ERR_CONFIG, "subregion grid count must be >= 1, got %d", d);
  PS_REQUIRE(l_max >= 1, PS_ERR_CONFIG, "l_max must be >= 1, got %d", l_max);
  PS_REQUIRE(d <= 8, PS_ERR_ARGUMENT, "d <= 8 supported (descriptor length <= 512)");
  PS_REQUIRE(n_scale_set >= 1 && n_scale_set <= kMaxDescScales, PS_ERR_ARGUMENT, "1..%d scales supported",
             kMaxDescScales);
  PS_REQUIRE(img->nr >= 3 && img->nc >= 3, PS_ERR_VALUE, "image too small");
  PS_REQUIRE((int64_t)img->nr * img->nc < (int64_t)INT32_MAX && (int64_t)img->nr * img->row_pitch < (int64_t)INT32_MAX,
             PS_ERR_ARGUMENT, "image too large (nr*pitch >= 2^31)");
  cudaStream_t s = (cudaStream_t)stream;
  // bound on |P| for the fixed-point histogram scale
  double pmax = 255.0 + 0.05 * 255.0;
  if (img->pixel_type != PS_PIXELS_U8 && img->pixel_type != PS_PIXELS_RGB8) {  // greys of RGB8 are <= 255 too
    unsigned long long* dmax = nullptr;
    cudaMallocAsync(&dmax, sizeof(unsigned long long), s);
    cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), s);
    max_abs_kernel<<<148 * 4, 256, 0, s>>>((const double*)img->data, img->batch, img->nr, img->nc, img->row_pitch,
                                           img->batch > 1 ? img->image_stride : 0, dmax);
    PS_LAUNCHED("max_abs_kernel");
    unsigned long long hbits = 0;
    cudaMemcpyAsync(&hbits, dmax, sizeof(hbits), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(dmax, s);
    cudaStreamSynchronize(s);
    int st = check_cuda("max_abs");
    if (st) return st;
    double m;
    memcpy(&m, &hbits, sizeof(m));
    pmax = m + (img->pixel_type == PS_PIXELS_F64_RAW ? 0.05 * 255.0 : 0.0);
    PS_REQUIRE(std::isfinite(pmax), PS_ERR_VALUE, "pixel values must be finite");
    if (pmax < 1e-300) pmax = 1e-300;
  }
  DescParams prm{};
  prm.n_scales = n_scale_set;
  for (int si = 0; si < n_scale_set; ++si) {
    prm.scale[si] = host_scale_set[si];
    int st = region_width(host_scale_set[si], beta0, d, l_max, img->nr, img->nc, &prm.w[si]);
    if (st) return st;
    // limb width: nsamp * 2^lb < 2^32; scale: every bin sum (<= nsamp *
    // 2*sqrt(2)*pmax) stays below 2^(3*lb), i.e. fits the three limbs
    const double nsamp = (double)prm.w[si] * prm.w[si];
    const int lb = std::min(21, 32 - (int)std::ceil(std::log2(nsamp + 1.0)));
    PS_REQUIRE(lb >= 8, PS_ERR_ARGUMENT, "descriptor region %d too large", prm.w[si]);
    prm.lb[si] = lb;
    prm.fx[si] = std::ldexp(1.0, (int)std::floor(3.0 * lb - std::log2(nsamp * 2.9 * pmax)));
  }
  for (int si = 0; si < n_scale_set; ++si) {
    if (d == 4 && prm.w[si] == 8) {
      prm.w8_scale[prm.n_w8++] = prm.scale[si];
      if (prm.scale[si] == default_scale) prm.default_w8 = 1;
    }
    if (d == 4 && prm.w[si] == 16) {
      prm.w16_scale[prm.n_w16++] = prm.scale[si];
      if (prm.scale[si] == default_scale) prm.default_w16 = 1;
    }
  }
  const double two_pi = 2.0 * M_PI;  // descriptor.py:31
  prm.d = d;
  prm.D = d * d * 8;
  prm.orient = orientation_normalize ? 1 : 0;
  prm.k36 = 36 / two_pi;
  prm.k8 = 8 / two_pi;
  prm.two_pi = two_pi;
  for (int m = 0; m <= 36; ++m) {
    prm.cb36[m] = std::cos(m * (two_pi / 36));
    prm.sb36[m] = std::sin(m * (two_pi / 36));
  }
  for (int m = 0; m <= 8; ++m) {
    prm.c8[m] = std::cos(m * (two_pi / 8));
    prm.s8[m] = std::sin(m * (two_pi / 8));
  }
  for (int k = 0; k < 36; ++k) {  // descriptor.py:146 and :180 (host libm, as Python's math)
    const double th = ((double)k + 0.5) * (two_pi / 36);
    prm.theta[k] = th;
    prm.cos_t[k] = std::cos(-th);
    prm.sin_t[k] = std::sin(-th);
  }
  const int64_t total = (int64_t)img->batch * kp->cap;
  if (total == 0) return PS_OK;
  const size_t shmem = (size_t)kWarps * (kStageDoubles * sizeof(double) + 3 * (prm.D + 36) * sizeof(unsigned));
  int64_t blocks = (total + kWarps - 1) / kWarps;
  if (blocks > 148 * 8) blocks = 148 * 8;
  cudaFuncSetAttribute(describe_kernel<RampU8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
  cudaFuncSetAttribute(describe_kernel<RampF64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
  cudaFuncSetAttribute(describe_kernel<RampF64Raw>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
  if (img->pixel_type == PS_PIXELS_U8) {
    RampU8 im{(const uint8_t*)img->data, img->row_pitch, img->nr, img->nc, img->alpha};
    return launch_fast(im, img, kp, default_scale, prm, out_desc32, out_desc64, total, shmem, policy, window_slots,
                       s);
  } else if (img->pixel_type == PS_PIXELS_RGB8) {
    RampRGB8 im{(const uint8_t*)img->data, img->row_pitch, img->nr, img->nc, img->alpha, img->gray_lut};
    cudaFuncSetAttribute(describe_kernel<RampRGB8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
    return launch_fast(im, img, kp, default_scale, prm, out_desc32, out_desc64, total, shmem, policy, window_slots,
                       s);
  } else if (img->pixel_type == PS_PIXELS_F64_RAW) {
    RampF64Raw im{(const double*)img->data, img->row_pitch, img->nr, img->nc, img->alpha};
    describe_kernel<<<(unsigned)blocks, kWarps * 32, shmem, s>>>(im, img->image_stride, img->batch, kp->row, kp->col,
                                                                  kp->scale, default_scale, kp->count, kp->cap, prm,
                                                                  out_desc32, out_desc64, nullptr, nullptr);
  } else {
    PS_REQUIRE(img->pixel_type == PS_PIXELS_F64, PS_ERR_ARGUMENT, "unknown pixel type");
    RampF64 im{(const double*)img->data, img->row_pitch, img->nr, img->nc};
    describe_kernel<<<(unsigned)blocks, kWarps * 32, shmem, s>>>(im, img->image_stride, img->batch, kp->row, kp->col,
                                                                  kp->scale, default_scale, kp->count, kp->cap, prm,
                                                                  out_desc32, out_desc64, nullptr, nullptr);
  }
  PS_LAUNCHED("describe_kernel");
  return PS_OK;
}
