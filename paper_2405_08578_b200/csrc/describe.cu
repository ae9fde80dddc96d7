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
#include <cmath>
#include <vector>

#include "ps_common.cuh"

namespace ps {
namespace {

constexpr int kMaxDescScales = 16;
constexpr int kWarps = 4;

struct DescParams {
  int n_scales;
  int scale[kMaxDescScales];
  int w[kMaxDescScales];  // region side after region_size + _fit_region cap
  int d, D, orient;
  double k36, k8, two_pi;  // PEAK_BINS / TWO_PI, ORIENTATION_BINS / TWO_PI, TWO_PI
  double theta[36], cos_t[36], sin_t[36];  // theta0_k and cos/sin(-theta0_k)
};

// Add `mag` to hist[bin] for the 32 samples of a chunk, per bin in lane
// (= raster) order.  Lanes with the same bin form a group; its lowest lane
// folds the members' magnitudes in sequentially.
__device__ __forceinline__ void ordered_add(double* hist, double* stage, int bin, double mag, bool on) {
  const int lane = threadIdx.x & 31;
  on = on && mag != 0.0;  // +0.0 leaves a non-negative sum bit-identical
  stage[lane] = mag;
  const unsigned peers = __match_any_sync(0xffffffffu, on ? bin : (0x40000000 | lane));
  __syncwarp();
  if (on && (__ffs(peers) - 1) == lane) {
    double h = hist[bin];
    unsigned m = peers;
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      h = __dadd_rn(h, stage[j]);
    }
    hist[bin] = h;
  }
  __syncwarp();
}

template <class Img>
__device__ __forceinline__ void axis_sample(const Img& im, int r, int c, double& a, double& b) {
  // descriptor.py:135-136 (gradient_at convention, :98-115)
  a = __dsub_rn(im.at(r + 1, c), im.at(r - 1, c));
  b = __dsub_rn(im.at(r, c + 1), im.at(r, c - 1));
}

template <class Img>
__global__ void __launch_bounds__(kWarps * 32) describe_kernel(Img img, int64_t img_stride, int B,
                                                               const int32_t* __restrict__ kp_row,
                                                               const int32_t* __restrict__ kp_col,
                                                               const int32_t* __restrict__ kp_scale,
                                                               int32_t default_scale,
                                                               const int32_t* __restrict__ counts, int64_t cap,
                                                               DescParams prm, float* __restrict__ out32,
                                                               double* __restrict__ out64) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int D = prm.D;
  double* hist = smem + wid * (D + 36 + 32);
  double* hist36 = hist + D;
  double* stage = hist36 + 36;
  const int nr = img.nr, nc = img.nc;
  const double two_pi = prm.two_pi;
  const int64_t total = (int64_t)B * cap;
  for (int64_t g = (int64_t)blockIdx.x * kWarps + wid; g < total; g += (int64_t)gridDim.x * kWarps) {
    const int b = (int)(g / cap);
    const int64_t i = g % cap;
    if (counts && i >= counts[b]) continue;
    Img im = img;
    im.p = img.p + (int64_t)b * img_stride;
    const int row = kp_row[g], col = kp_col[g];
    const int scale = kp_scale ? kp_scale[g] : default_scale;
    int w = -1;
    for (int s = 0; s < prm.n_scales; ++s)
      if (prm.scale[s] == scale) w = prm.w[s];
    if (w < 0 || row < 0 || row >= nr || col < 0 || col >= nc) continue;  // validated by the caller
    const int d = prm.d, ws = w / d, nsamp = w * w;
    // _fit_region (descriptor.py:129-130)
    const int r0 = min(max(row - w / 2, 1), nr - 1 - w);
    const int c0 = min(max(col - w / 2, 1), nc - 1 - w);
    for (int q = lane; q < D; q += 32) hist[q] = 0.0;
    if (prm.orient) {
      // --- dominant orientation: 36-bin histogram over the axis region (:142-146)
      for (int q = lane; q < 36; q += 32) hist36[q] = 0.0;
      __syncwarp();
      for (int base = 0; base < nsamp; base += 32) {
        const int s = base + lane;
        const bool on = s < nsamp;
        double mag = 0.0;
        int bin = 0;
        if (on) {
          double a, bb;
          axis_sample(im, r0 + s / w, c0 + s % w, a, bb);
          mag = hypot(a, bb);
          const double ori = np_mod_pos(atan2(bb, a), two_pi);
          bin = min((int)__dmul_rn(ori, prm.k36), 35);
        }
        ordered_add(hist36, stage, bin, mag, on);
      }
      // first argmax over 36 bins
      double hv = hist36[lane];
      int hk = lane;
      if (lane < 4 && hist36[lane + 32] > hv) { hv = hist36[lane + 32]; hk = lane + 32; }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, hv, o);
        const int k2 = __shfl_xor_sync(0xffffffffu, hk, o);
        if (v2 > hv || (v2 == hv && k2 < hk)) { hv = v2; hk = k2; }
      }
      const double theta0 = prm.theta[hk], ct = prm.cos_t[hk], st = prm.sin_t[hk];
      // --- rotated grid centred on the (clamped) feature pixel (:237-240, 164-216)
      const double half = (double)(w - 1) / 2.0;
      const double cy = fmin(fmax((double)row, 1.0 + half), __dsub_rn((double)nr - 2.0, half));
      const double cx = fmin(fmax((double)col, 1.0 + half), __dsub_rn((double)nc - 2.0, half));
      // sample positions are coordinate-wise monotone in (u, v), so the grid's
      // extreme x / y lie at its corners
      double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
#pragma unroll
      for (int cv = 0; cv < 2; ++cv)
#pragma unroll
        for (int cu = 0; cu < 2; ++cu) {
          const double u = __dsub_rn((double)(cu * (w - 1)), half);
          const double v = __dsub_rn((double)(cv * (w - 1)), half);
          const double x = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, u)), __dmul_rn(st, v));
          const double y = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, u)), __dmul_rn(ct, v));
          xmin = fmin(xmin, x); xmax = fmax(xmax, x);
          ymin = fmin(ymin, y); ymax = fmax(ymax, y);
        }
      const int pr0 = max((int)floor(ymin), 1), pr1 = min((int)ceil(ymax), nr - 2);
      const int pc0 = max((int)floor(xmin), 1), pc1 = min((int)ceil(xmax), nc - 2);
      const int xcap = max(pc1 - pc0 - 1, 0), ycap = max(pr1 - pr0 - 1, 0);
      for (int base = 0; base < nsamp; base += 32) {
        const int s = base + lane;
        const bool on = s < nsamp;
        double mag = 0.0;
        int cell = 0;
        if (on) {
          const int iv = s / w, iu = s % w;
          const double u = __dsub_rn((double)iu, half), v = __dsub_rn((double)iv, half);
          const double x = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, u)), __dmul_rn(st, v));
          const double y = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, u)), __dmul_rn(ct, v));
          const bool inside = x >= 1.0 && x <= (double)(nc - 2) && y >= 1.0 && y <= (double)(nr - 2);
          const double lx = __dsub_rn(fmin(fmax(x, (double)pc0), (double)pc1), (double)pc0);
          const double ly = __dsub_rn(fmin(fmax(y, (double)pr0), (double)pr1), (double)pr0);
          const int x0 = min((int)floor(lx), xcap), y0 = min((int)floor(ly), ycap);
          const double fx = __dsub_rn(lx, (double)x0), fy = __dsub_rn(ly, (double)y0);
          const int x1 = min(x0 + 1, pc1 - pc0), y1 = min(y0 + 1, pr1 - pr0);
          const int gy0 = pr0 + y0, gy1 = pr0 + y1, gx0 = pc0 + x0, gx1 = pc0 + x1;
          double a00, b00, a01, b01, a10, b10, a11, b11;
          axis_sample(im, gy0, gx0, a00, b00);
          axis_sample(im, gy0, gx1, a01, b01);
          axis_sample(im, gy1, gx0, a10, b10);
          axis_sample(im, gy1, gx1, a11, b11);
          const double sy = __dsub_rn(1.0, fy), sx = __dsub_rn(1.0, fx);
          // left-to-right: f00*(1-fy)*(1-fx) + f01*(1-fy)*fx + f10*fy*(1-fx) + f11*fy*fx
          const double as = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(a00, sy), sx), __dmul_rn(__dmul_rn(a01, sy), fx)),
                                                __dmul_rn(__dmul_rn(a10, fy), sx)),
                                      __dmul_rn(__dmul_rn(a11, fy), fx));
          const double bs = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(b00, sy), sx), __dmul_rn(__dmul_rn(b01, sy), fx)),
                                                __dmul_rn(__dmul_rn(b10, fy), sx)),
                                      __dmul_rn(__dmul_rn(b11, fy), fx));
          mag = __dmul_rn(hypot(as, bs), inside ? 1.0 : 0.0);
          const double ori = np_mod_pos(__dsub_rn(atan2(bs, as), theta0), two_pi);
          const int ob = min((int)__dmul_rn(ori, prm.k8), 7);
          cell = ((iv / ws) * d + iu / ws) * 8 + ob;
        }
        ordered_add(hist, stage, cell, mag, on);
      }
    } else {
      __syncwarp();
      for (int base = 0; base < nsamp; base += 32) {
        const int s = base + lane;
        const bool on = s < nsamp;
        double mag = 0.0;
        int cell = 0;
        if (on) {
          const int iv = s / w, iu = s % w;
          double a, bb;
          axis_sample(im, r0 + iv, c0 + iu, a, bb);
          mag = hypot(a, bb);
          const double ori = np_mod_pos(atan2(bb, a), two_pi);
          const int ob = min((int)__dmul_rn(ori, prm.k8), 7);
          cell = ((iv / ws) * d + iu / ws) * 8 + ob;
        }
        ordered_add(hist, stage, cell, mag, on);
      }
    }
    // --- L2 normalise, clamp at 0.2, renormalise (descriptor.py:250-255)
    double ss = 0.0;
    for (int q = lane; q < D; q += 32) ss = __dadd_rn(ss, __dmul_rn(hist[q], hist[q]));
#pragma unroll
    for (int o = 16; o; o >>= 1) ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    const double n1 = __dsqrt_rn(ss);
    double scale1 = 0.0;
    if (n1 > 0.0) {
      double ss2 = 0.0;
      for (int q = lane; q < D; q += 32) {
        const double v = fmin(__ddiv_rn(hist[q], n1), 0.2);
        hist[q] = v;
        ss2 = __dadd_rn(ss2, __dmul_rn(v, v));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) ss2 = __dadd_rn(ss2, __shfl_xor_sync(0xffffffffu, ss2, o));
      scale1 = __dsqrt_rn(ss2);
    }
    for (int q = lane; q < D; q += 32) {
      const double v = n1 > 0.0 ? __ddiv_rn(hist[q], scale1) : 0.0;
      if (out32) out32[g * D + q] = __double2float_rn(v);
      if (out64) out64[g * D + q] = v;
    }
    __syncwarp();
  }
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

extern "C" int ps_describe(const ps_image_batch* img, const ps_keypoints* kp, int32_t default_scale,
                           const int32_t* host_scale_set, int32_t n_scale_set, double beta0, int32_t d, int32_t l_max,
                           int32_t orientation_normalize, float* out_desc32, double* out_desc64, void* stream) {
  PS_REQUIRE(img && kp && img->data && kp->row && kp->col && host_scale_set, PS_ERR_ARGUMENT,
             "null argument to ps_describe");
  PS_REQUIRE(beta0 > 0, PS_ERR_CONFIG, "beta0 must be positive, got %g", beta0);
  PS_REQUIRE(d >= 1, PS_ERR_CONFIG, "subregion grid count must be >= 1, got %d", d);
  PS_REQUIRE(l_max >= 1, PS_ERR_CONFIG, "l_max must be >= 1, got %d", l_max);
  PS_REQUIRE(d <= 8, PS_ERR_ARGUMENT, "d <= 8 supported (descriptor length <= 512)");
  PS_REQUIRE(n_scale_set >= 1 && n_scale_set <= kMaxDescScales, PS_ERR_ARGUMENT, "1..%d scales supported",
             kMaxDescScales);
  PS_REQUIRE(img->nr >= 3 && img->nc >= 3, PS_ERR_VALUE, "image too small");
  DescParams prm{};
  prm.n_scales = n_scale_set;
  for (int s = 0; s < n_scale_set; ++s) {
    prm.scale[s] = host_scale_set[s];
    int st = region_width(host_scale_set[s], beta0, d, l_max, img->nr, img->nc, &prm.w[s]);
    if (st) return st;
  }
  const double two_pi = 2.0 * M_PI;  // descriptor.py:31
  prm.d = d;
  prm.D = d * d * 8;
  prm.orient = orientation_normalize ? 1 : 0;
  prm.k36 = 36 / two_pi;
  prm.k8 = 8 / two_pi;
  prm.two_pi = two_pi;
  for (int k = 0; k < 36; ++k) {  // descriptor.py:146 and :180 (host libm, as Python's math)
    const double th = ((double)k + 0.5) * (two_pi / 36);
    prm.theta[k] = th;
    prm.cos_t[k] = std::cos(-th);
    prm.sin_t[k] = std::sin(-th);
  }
  const int64_t total = (int64_t)img->batch * kp->cap;
  if (total == 0) return PS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t shmem = (size_t)kWarps * (prm.D + 36 + 32) * sizeof(double);
  int64_t blocks = (total + kWarps - 1) / kWarps;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (img->pixel_type == PS_PIXELS_U8) {
    RampU8 im{(const uint8_t*)img->data, img->row_pitch, img->nr, img->nc, img->alpha};
    describe_kernel<<<(unsigned)blocks, kWarps * 32, shmem, s>>>(im, img->image_stride, img->batch, kp->row, kp->col,
                                                                  kp->scale, default_scale, kp->count, kp->cap, prm,
                                                                  out_desc32, out_desc64);
  } else if (img->pixel_type == PS_PIXELS_F64_RAW) {
    RampF64Raw im{(const double*)img->data, img->row_pitch, img->nr, img->nc, img->alpha};
    describe_kernel<<<(unsigned)blocks, kWarps * 32, shmem, s>>>(im, img->image_stride, img->batch, kp->row, kp->col,
                                                                  kp->scale, default_scale, kp->count, kp->cap, prm,
                                                                  out_desc32, out_desc64);
  } else {
    PS_REQUIRE(img->pixel_type == PS_PIXELS_F64, PS_ERR_ARGUMENT, "unknown pixel type");
    RampF64 im{(const double*)img->data, img->row_pitch, img->nr, img->nc};
    describe_kernel<<<(unsigned)blocks, kWarps * 32, shmem, s>>>(im, img->image_stride, img->batch, kp->row, kp->col,
                                                                  kp->scale, default_scale, kp->count, kp->cap, prm,
                                                                  out_desc32, out_desc64);
  }
  PS_LAUNCHED("describe_kernel");
  return PS_OK;
}
