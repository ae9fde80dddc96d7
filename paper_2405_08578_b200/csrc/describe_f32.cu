// K2 float32 throughput kernel: the descriptor of every w = 8, d = 4 keypoint
// of an 8-bit raster (grey or RGB) that lies at least 6 pixels inside the
// image -- all of C1, C2, C4 and C5's keypoints but a border fringe.
// Reference: descriptor.py:219-256 (region :118-131, dominant orientation
// :142-161, rotated bilinear gradients :164-216, histogram and
// normalisation :243-255); SURVEY.md §8(a) A5-A9.
//
// Layout: a half-warp per keypoint (two per warp).  The half-warp first
// stages the keypoint's gradient fields a(y, x) = I(y+1, x) - I(y-1, x),
// b(y, x) = I(y, x+1) - I(y, x-1) over rows / columns -5..+5 about the
// keypoint as float2 in shared memory (exact: integer differences of the
// 8-bit key).  The linear ramp of apply_linear_ramp (imaging.py:113-132) adds
// the same constant (2 nc alpha, 2 alpha) to every field value, and the
// bilinear weights sum to one, so it is added once per sample.  Lane l owns
// subregion l (descriptor.py:247-248): its four samples in both phases and
// its 8 descriptor bins, so the descriptor histogram needs no atomics.  The
// rotated sample positions relative to the keypoint depend only on theta0:
// a per-device table (built in float64 as the reference computes them, then
// rounded) gives each sample's corner offset and bilinear fractions.
//
// Arithmetic is float32 (packed FFMA2 / FADD2): the descriptor is ~1e-7
// relative from the reference's float64 one (the P2 bar is 1e-4).  Every
// DISCRETE decision is certified against a rigorous error bound that includes
// the reference's own ramp-rounding noise, and is otherwise taken exactly:
//   * 36-bin orientation bin of an axis sample: accepted >= 1e-4 bins from an
//     edge; at the four axis edges the sign of one component decides; else
//     the float32 side test of the edge, else the reference's float64
//     arithmetic (exact_axis_bin);
//   * dominant orientation: the top bin's exact fixed-point sum must lead the
//     next by 6.1e-5 relative, else the keypoint goes to the float64 kernel;
//   * 8-bin octant of a descriptor sample: accepted when the rotated gradient
//     is farther from the four bin lines than the sample's own error bound;
//     else the float32 side test of the nearest line, else float64
//     (exact_rot_bin).
// The float64 kernels of describe.cu serve every other keypoint and every
// call that asks for float64 output.
#include <atomic>

#include "describe_common.cuh"

namespace ps {
namespace {

constexpr int kF32Warps = 8;
constexpr int kFS = 12;              // field row stride (float2)
constexpr int kFR = 11;              // field rows / columns: offsets -5 .. +5 about the keypoint
constexpr int kFieldF2 = kFR * kFS;  // float2 per keypoint
constexpr int kHStride = 12;         // lane-private 8-bin histogram stride (floats)
constexpr int kH36 = 40;             // 36-bin histogram, padded
constexpr int kPerKpF = 2 * kFieldF2 + 16 * kHStride + kH36;  // floats per keypoint (half-warp)
static_assert(kPerKpF % 4 == 0 && (2 * kFieldF2) % 4 == 0, "16-byte aligned histograms");
#ifndef PS_F32_MINB
#define PS_F32_MINB 4  // resident blocks per SM the register budget targets
#endif
#ifndef PS_F32_BLOCKS_PER_SM
#define PS_F32_BLOCKS_PER_SM 200  // grid cap: resident blocks work on consecutive slots (as the pair kernel)
#endif

// Error-model constants (per component, against the reference's float64 values):
constexpr float kRefNoise = 6e-14f;  // reference ramp rounding: P = fl(I + fl(k alpha)), |dP| <= 2^-45 per pixel
constexpr float kRelF32 = 4e-7f;     // float32 rounding of ks * blend + ramp and of the theta0 rotation
constexpr float kPosF32 = 6e-7f;     // weights (fractions rounded to float32) and blend rounding, x sum |corner|
constexpr float kBand = 2e-14f;      // the reference's own float64 rounding of atan2 / mod / trunc near an edge

struct F32Params {
  float cA, cB;                  // ramp part of a / b: 2 nc alpha, 2 alpha
  float ks;                      // key -> grey scale: 1 (8-bit grey), 0.001 (RGB luma key 299 R + 587 G + 114 B)
  float ct[36], st[36];          // cos(-theta0_k), sin(-theta0_k) (descriptor.py:180)
  float ce36[37], se36[37];      // cos / sin of the 36-bin edges m 2 pi / 36 (descriptor.py:144)
  float ce8[36][9], se8[36][9];  // cos / sin of theta0_k + m pi / 4: 8-bin edges as absolute angles (:215, 244)
};

// Rotated-grid geometry per (theta0 bin k, sample j of lane l):
// {fx, fy, corner offset (int bits), 0}; x - cx = cos_t u - sin_t v,
// y - cy = sin_t u + cos_t v in float64 (descriptor.py:179-184), floor and
// fraction (:197-200), fractions rounded to float32.  Per device, built once.
__device__ float4 g_geom8[36 * 4 * 16];

__global__ void init_geom8_kernel(DescParams prm) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 36 * 64) return;
  const int k = t >> 6, j = (t >> 4) & 3, l = t & 15;
  const int iv = 2 * (l >> 2) + (j >> 1), iu = 2 * (l & 3) + (j & 1);
  const double u = (double)iu - 3.5, v = (double)iv - 3.5;
  const double x = __dsub_rn(__dmul_rn(prm.cos_t[k], u), __dmul_rn(prm.sin_t[k], v));
  const double y = __dadd_rn(__dmul_rn(prm.sin_t[k], u), __dmul_rn(prm.cos_t[k], v));
  const double x0 = floor(x), y0 = floor(y);
  g_geom8[t] = make_float4(__double2float_rn(x - x0), __double2float_rn(y - y0),
                           __int_as_float((int)y0 * kFS + (int)x0), 0.0f);
}

__device__ __forceinline__ float u_to_f(unsigned v) {  // exact for v < 2^23, no I2F
  return __uint_as_float(0x4B000000u | v) - 8388608.0f;
}
__device__ __forceinline__ float key_f(const RampU8& im, int r, int c) {
  return u_to_f(__ldg(im.p + r * (int)im.pitch + c));
}
__device__ __forceinline__ float key_f(const RampRGB8& im, int r, int c) {
  const uint8_t* q = im.p + 3 * (r * (int)im.pitch + c);
  return u_to_f(299u * __ldg(q) + 587u * __ldg(q + 1) + 114u * __ldg(q + 2));
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// fast_atan2f (describe_common.cuh) with an approximate reciprocal (2^-23
// relative: < 1.2e-7 rad more); x or y nonzero (the ramp keeps a != 0).
__device__ __forceinline__ float atan2_f32(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float t = fminf(ax, ay) * rcp_approx(fmaxf(fmaxf(ax, ay), 1e-30f));
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
__device__ __forceinline__ unsigned half_max(unsigned v, int hsel) {
  const unsigned a = __reduce_max_sync(0xffffffffu, hsel == 0 ? v : 0u);
  const unsigned b = __reduce_max_sync(0xffffffffu, hsel == 1 ? v : 0u);
  return hsel ? b : a;
}
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: fadd_rd(x, kMagic) holds floor(x) in its low bits
constexpr int kMagicBits = 0x4B400000;
// floor / fraction of a bin coordinate 0 <= x < 2^22 without a conversion
// instruction; certified when >= kBinMargin from both edges and inside [0, n)
__device__ __forceinline__ bool cert_bin(float x, int nbins, int& bin) {
  const float t = __fadd_rd(x, kMagic);
  bin = __float_as_int(t) - kMagicBits;
  const float fr = x - (t - kMagic);
  return fr > kBinMargin && fr < 1.0f - kBinMargin && x > 0.0f && bin < nbins;
}

// Side of the bin edge (cos e, sin e) of a float32 gradient (a, b) whose
// components are within (ea, eb) of the reference's float64 gradient: +1
// above, -1 below, 0 undecided.  sd = b cos e - a sin e = |g| sin(phi - e);
// the bound adds the rounding of the float32 table entries and of sd (4 ulp
// of its two terms) and the band inside which the reference's own float64
// atan2 / mod / trunc could fall on either side (side_bin,
// describe_common.cuh).  Exactly axis-aligned integer gradients, whose side
// only the tiny ramp term decides, are decided here.
__device__ __forceinline__ int side_f32(float a, float b, float ce, float se, float ea, float eb) {
  const float p = a * se;
  const float sd = fmaf(b, ce, -p);
  const float bound =
      fmaf(2.5e-7f, fabsf(b * ce) + fabsf(p), fmaf(kBand, fabsf(a) + fabsf(b), fabsf(ce) * eb + fabsf(se) * ea));
  return sd > bound ? 1 : (sd < -bound ? -1 : 0);
}
__device__ __forceinline__ int side_to_bin(int side, int m, int nbins) {
  return side > 0 ? (m == nbins ? 0 : m) : (m == 0 ? nbins - 1 : m - 1);
}

// ---- exact (reference float64) decisions for the rare undecided samples ----
// bin of the axis sample at (r, c) (descriptor.py:135-138, 144 / 243-246)
template <class Img>
__device__ __noinline__ int exact_axis_bin(Img im, int r, int c, double cm, double sm, int m, int nbins, double k,
                                           double two_pi) {
  const double a = __dsub_rn(im.at(r + 1, c), im.at(r - 1, c));
  const double b = __dsub_rn(im.at(r, c + 1), im.at(r, c - 1));
  return exact_bin(a, b, 1.0, 0.0, cm, sm, m, nbins, 0.0, k, two_pi);
}

// 8-bin of rotated sample (iv, iu) of the interior keypoint (row, col) whose
// grid centre is the keypoint itself (descriptor.py:237-240 clamp inactive):
// descriptor.py:179-215 in the reference's float64 operation order.
template <class Img>
__device__ __noinline__ int exact_rot_bin(Img im, int row, int col, int iv, int iu, double ct, double st,
                                          double theta0, double cm, double sm, int m, double k8, double two_pi) {
  const int nr = im.nr, nc = im.nc;
  const double half = 3.5, cx = (double)col, cy = (double)row;
  const double xmin = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, ct >= 0.0 ? -half : half)), __dmul_rn(st, st >= 0.0 ? half : -half));
  const double xmax = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, ct >= 0.0 ? half : -half)), __dmul_rn(st, st >= 0.0 ? -half : half));
  const double ymin = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, st >= 0.0 ? -half : half)), __dmul_rn(ct, ct >= 0.0 ? -half : half));
  const double ymax = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, st >= 0.0 ? half : -half)), __dmul_rn(ct, ct >= 0.0 ? half : -half));
  const int pr0 = max((int)floor(ymin), 1), pr1 = min((int)ceil(ymax), nr - 2);
  const int pc0 = max((int)floor(xmin), 1), pc1 = min((int)ceil(xmax), nc - 2);
  const double u = (double)iu - half, v = (double)iv - half;
  const double x = __dsub_rn(__dadd_rn(cx, __dmul_rn(ct, u)), __dmul_rn(st, v));
  const double y = __dadd_rn(__dadd_rn(cy, __dmul_rn(st, u)), __dmul_rn(ct, v));
  const double lx = __dsub_rn(fmin(fmax(x, (double)pc0), (double)pc1), (double)pc0);
  const double ly = __dsub_rn(fmin(fmax(y, (double)pr0), (double)pr1), (double)pr0);
  const int x0 = min((int)floor(lx), max(pc1 - pc0 - 1, 0)), y0 = min((int)floor(ly), max(pr1 - pr0 - 1, 0));
  const double fxx = __dsub_rn(lx, (double)x0), fyy = __dsub_rn(ly, (double)y0);
  const int x1 = min(x0 + 1, pc1 - pc0), y1 = min(y0 + 1, pr1 - pr0);
  const int gx0 = pc0 + x0, gx1 = pc0 + x1, gy0 = pr0 + y0, gy1 = pr0 + y1;
  auto fa = [&](int r, int c) { return __dsub_rn(im.at(r + 1, c), im.at(r - 1, c)); };
  auto fb = [&](int r, int c) { return __dsub_rn(im.at(r, c + 1), im.at(r, c - 1)); };
  const double sy = __dsub_rn(1.0, fyy), sx = __dsub_rn(1.0, fxx);
  // f00*(1-fy)*(1-fx) + f01*(1-fy)*fx + f10*fy*(1-fx) + f11*fy*fx, left to right (descriptor.py:204-210)
  auto interp = [&](double f00, double f01, double f10, double f11) {
    return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(f00, sy), sx), __dmul_rn(__dmul_rn(f01, sy), fxx)),
                               __dmul_rn(__dmul_rn(f10, fyy), sx)),
                     __dmul_rn(__dmul_rn(f11, fyy), fxx));
  };
  const double as = interp(fa(gy0, gx0), fa(gy0, gx1), fa(gy1, gx0), fa(gy1, gx1));
  const double bs = interp(fb(gy0, gx0), fb(gy0, gx1), fb(gy1, gx0), fb(gy1, gx1));
  return exact_bin(as, bs, ct, -st, cm, sm, m, 8, theta0, k8, two_pi);
}

// Blended gradient (a, b) of sample j of lane l (theta0 bin k) over the
// staged fields (descriptor.py:195-213), ramp constant added once (weights
// sum to one), plus its per-component error bound (ea, eb): kPosF32 x the
// corners' absolute sum, kRelF32 x |value|, kRefNoise.  The axis sample of
// the region when orientation normalisation is off.
template <bool ORIENT>
__device__ __forceinline__ float2 blend_sample(const float2* Fc, const float4* __restrict__ geom, int k, int j, int l,
                                               int aoff, float ks, float cA, float cB, float2& err) {
  float2 s, sabs;
  if constexpr (ORIENT) {
    const float4 gm = geom[(k * 4 + j) * 16 + l];
    const float fx = gm.x, fy = gm.y;
    const float2* q = Fc + __float_as_int(gm.z);
    const float2 f00 = q[0], f01 = q[1], f10 = q[kFS], f11 = q[kFS + 1];
    const float gx = 1.0f - fx, gy = 1.0f - fy;
    s = __fmul2_rn(f00, make_float2(gy * gx, gy * gx));
    s = __ffma2_rn(f01, make_float2(gy * fx, gy * fx), s);
    s = __ffma2_rn(f10, make_float2(fy * gx, fy * gx), s);
    s = __ffma2_rn(f11, make_float2(fy * fx, fy * fx), s);
    sabs = __fadd2_rn(make_float2(fabsf(f00.x), fabsf(f00.y)), make_float2(fabsf(f01.x), fabsf(f01.y)));
    sabs = __fadd2_rn(sabs, make_float2(fabsf(f10.x), fabsf(f10.y)));
    sabs = __fadd2_rn(sabs, make_float2(fabsf(f11.x), fabsf(f11.y)));
  } else {
    s = Fc[aoff];
    sabs = make_float2(0.0f, 0.0f);
  }
  const float2 g = __ffma2_rn(s, make_float2(ks, ks), make_float2(cA, cB));
  err = __ffma2_rn(sabs, make_float2(kPosF32 * ks, kPosF32 * ks),
                   __ffma2_rn(make_float2(fabsf(g.x), fabsf(g.y)), make_float2(kRelF32, kRelF32),
                              make_float2(kRefNoise, kRefNoise)));
  return g;
}

// Rare paths, out of line: 36-bin bins (8 bits per sample in `bins`) of the
// axis samples flagged in `unc` -- the float32 side test of the nearest edge,
// else the reference's float64 arithmetic.
template <class Img>
__device__ __noinline__ unsigned fb_bin36(Img im, const float2* Fc, int row, int col, int sr, int sc, unsigned unc,
                                          unsigned bins, const F32Params* fp, const DescParams* prm) {
  for (int j = 0; j < 4; ++j) {
    if (!((unc >> j) & 1u)) continue;
    const int iv = 2 * sr + (j >> 1), iu = 2 * sc + (j & 1);
    const float2 f = Fc[(iv - 4) * kFS + (iu - 4)];
    const float a = fmaf(f.x, fp->ks, fp->cA), bb = fmaf(f.y, fp->ks, fp->cB);
    const float x = wrap_two_pi_f(atan2_f32(bb, a)) * 5.729577951308232f;
    const int m = min(max(__float2int_rn(x), 0), 36);
    const int side = side_f32(a, bb, fp->ce36[m], fp->se36[m], fmaf(kRelF32, fabsf(a), kRefNoise),
                              fmaf(kRelF32, fabsf(bb), kRefNoise));
    const int bin = side ? side_to_bin(side, m, 36)
                         : exact_axis_bin(im, row - 4 + iv, col - 4 + iu, prm->cb36[m], prm->sb36[m], m, 36, prm->k36,
                                          prm->two_pi);
    bins = (bins & ~(255u << (8 * j))) | ((unsigned)bin << (8 * j));
  }
  return bins;
}

// 8-bin octants of the descriptor samples flagged in `unc`: the float32 side
// test of the nearest bin line, else the reference's float64 arithmetic.
template <bool ORIENT, class Img>
__device__ __noinline__ unsigned fb_bin8(Img im, const float2* Fc, const float4* geom, int row, int col, int l,
                                         unsigned unc, unsigned obs, int hk, const F32Params* fp,
                                         const DescParams* prm) {
  const float theta0f = ORIENT ? (float)prm->theta[hk] : 0.0f;
  const int sr = l >> 2, sc = l & 3;
  for (int j = 0; j < 4; ++j) {
    if (!((unc >> j) & 1u)) continue;
    const int iv = 2 * sr + (j >> 1), iu = 2 * sc + (j & 1);
    float2 err;
    const float2 g = blend_sample<ORIENT>(Fc, geom, hk, j, l, (iv - 4) * kFS + (iu - 4), fp->ks, fp->cA, fp->cB, err);
    const float xb = wrap_two_pi_f(atan2_f32(g.y, g.x) - theta0f) * 1.2732395447351628f;
    const int m = min(max(__float2int_rn(xb), 0), 8);
    const int side = side_f32(g.x, g.y, fp->ce8[hk][m], fp->se8[hk][m], err.x, err.y);
    int ob;
    if (side) {
      ob = side_to_bin(side, m, 8);
    } else if constexpr (ORIENT) {
      ob = exact_rot_bin(im, row, col, iv, iu, prm->cos_t[hk], prm->sin_t[hk], prm->theta[hk], prm->c8[m], prm->s8[m],
                         m, prm->k8, prm->two_pi);
    } else {
      ob = exact_axis_bin(im, row - 4 + iv, col - 4 + iu, prm->c8[m], prm->s8[m], m, 8, prm->k8, prm->two_pi);
    }
    obs = (obs & ~(255u << (8 * j))) | ((unsigned)ob << (8 * j));
  }
  return obs;
}

template <bool ORIENT, class Img>
__global__ void __launch_bounds__(kF32Warps * 32, PS_F32_MINB)
    describe_f32_kernel(Img img, int64_t img_stride, int B, const int32_t* __restrict__ kp_row,
                        const int32_t* __restrict__ kp_col, const int32_t* __restrict__ kp_scale,
                        const int32_t* __restrict__ counts, int64_t cap, const __grid_constant__ DescParams prm,
                        const __grid_constant__ F32Params fp, float* __restrict__ out32,
                        int64_t* __restrict__ work, unsigned long long* __restrict__ n_work) {
  extern __shared__ float4 smf4[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, hsel = lane >> 4, hl = lane & 15;
  float* kb = reinterpret_cast<float*>(smf4) + (2 * wid + hsel) * kPerKpF;
  float2* F = reinterpret_cast<float2*>(kb);
  float* h8 = kb + 2 * kFieldF2 + kHStride * hl;
  unsigned* h36 = reinterpret_cast<unsigned*>(kb + 2 * kFieldF2 + 16 * kHStride);
  const float2* Fc = F + 5 * kFS + 5;  // field at offset (0, 0) from the keypoint
  const float4* __restrict__ geom = g_geom8;
  // this lane's subregion: samples (iv, iu) = (2 sr + j / 2, 2 sc + j % 2), cell 8 hl (descriptor.py:247-248)
  const int sr = hl >> 2, sc = hl & 3;
  const float cA = fp.cA, cB = fp.cB, ks = fp.ks;
  const int64_t total = (int64_t)B * cap;
  const int64_t npairs = (total + 1) / 2;
  const bool img_ok = img.nr >= 13 && img.nc >= 13;
  const int64_t gstep = 2 * (int64_t)gridDim.x * kF32Warps;
  int64_t gi0 = 2 * ((int64_t)blockIdx.x * kF32Warps + wid) + hsel;
  int bcur = (int)(gi0 / cap);
  int64_t icur = gi0 - (int64_t)bcur * cap;
  const int qstep = (int)(gstep / cap);
  const int64_t rstep = gstep - (int64_t)qstep * cap;
  // axis region r0 = row - 4, c0 = col - 4 (descriptor.py:129-130): field offset of sample j
  auto axis_off = [&](int j) { return (2 * sr + (j >> 1) - 4) * kFS + (2 * sc + (j & 1) - 4); };
  for (int64_t pi = (int64_t)blockIdx.x * kF32Warps + wid; pi < npairs; pi += (int64_t)gridDim.x * kF32Warps) {
    const int64_t g = 2 * pi + hsel;
    bool live = g < total;
    int b = 0;
    if (live) {
      b = bcur;
      live = !counts || icur < counts[b];
    }
    bcur += qstep;  // (image, slot) of the next step, without a division
    icur += rstep;
    if (icur >= cap) {
      icur -= cap;
      ++bcur;
    }
    int row = live ? kp_row[g] : 6, col = live ? kp_col[g] : 6;
    bool fast = live && img_ok && row >= 6 && row <= img.nr - 7 && col >= 6 && col <= img.nc - 7;
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
    if (!fast) {  // a dummy interior keypoint keeps the half-warp in step; nothing is written
      row = 6;
      col = 6;
      b = 0;
    }
    Img im = img;
    im.p = img.p + (int64_t)b * img_stride * decltype(img)::kElem;

    // ---- gradient fields of rows row-5..row+5, columns col-5..col+5 (descriptor.py:135-136, 192-193)
    {
      const int xs = col - 6 + min(hl, 12);  // lane = pixel column col-6 .. col+6
      float p[13];
#pragma unroll
      for (int y = 0; y < 13; ++y) p[y] = key_f(im, row - 6 + y, xs);
#pragma unroll
      for (int y = 1; y < 12; ++y) {
        const float pr = __shfl_down_sync(0xffffffffu, p[y], 1, 16);
        const float pl = __shfl_up_sync(0xffffffffu, p[y], 1, 16);
        if (hl >= 1 && hl <= 11) F[(y - 1) * kFS + hl - 1] = make_float2(p[y + 1] - p[y - 1], pr - pl);
      }
    }
    reinterpret_cast<float4*>(h8)[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    reinterpret_cast<float4*>(h8)[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (hl < kH36 / 4) reinterpret_cast<uint4*>(h36)[hl] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();

    bool ok = fast;
    float ct = 1.0f, st = 0.0f;
    int hk = 0;
    if constexpr (ORIENT) {
      // ---- dominant orientation: 36-bin histogram of the axis region (descriptor.py:142-146)
      float mg[4];
      unsigned bins = 0u, unc = 0u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = Fc[axis_off(j)];
        const float a = fmaf(f.x, ks, cA), bb = fmaf(f.y, ks, cB);
        const float x = wrap_two_pi_f(atan2_f32(bb, a)) * 5.729577951308232f;
        int bin;
        if (!cert_bin(x, 36, bin)) {
          // at the axis edges 0, 90, 180, 270 degrees one component's sign decides
          // exactly (sd = b cos e - a sin e with cos, sin in {0, +-1})
          const int m = min(max(__float2int_rn(x), 0), 36);
          const int q = m == 36 ? 0 : m / 9;
          const float c = q == 0 ? bb : (q == 1 ? -a : (q == 2 ? -bb : a));
          const bool axis =
              m % 9 == 0 && fabsf(c) > fmaf(kRelF32, fabsf(c), fmaf(kBand, fabsf(a) + fabsf(bb), kRefNoise));
          if (axis)
            bin = side_to_bin(c > 0.0f ? 1 : -1, m, 36);
          else
            unc |= 1u << j;
        }
        bins |= (unsigned)(bin & 255) << (8 * j);
        mg[j] = sqrt_approx(fmaf(a, a, bb * bb));
      }
      if (__any_sync(0xffffffffu, unc)) {  // near another edge: float32 side test, else float64
        if (unc) bins = fb_bin36(im, Fc, row, col, sr, sc, unc, bins, &fp, &prm);
      }
      // exact fixed-point sums (native shared atomics, order-independent):
      // q = rint(mag 2^(22 - e)) <= 2^23 for the half's largest magnitude < 2^(e + 1)
      const unsigned eb = half_max(__float_as_uint(fmaxf(fmaxf(mg[0], mg[1]), fmaxf(mg[2], mg[3]))), hsel) >> 23;
      const float s36 = eb == 0u ? 1.0f : __uint_as_float((unsigned)min(max(276 - (int)eb, 1), 254) << 23);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        atomicAdd(h36 + ((bins >> (8 * j)) & 255u), __float_as_uint(fmaf(mg[j], s36, 8388608.0f)) - 0x4B000000u);
      __syncwarp();
      // argmax with a clear lead (the sums are < 1e-5 relative from the
      // reference's; keys: the sum with its low 6 bits replaced by 63 - bin)
      unsigned k1 = 0u, k2 = 0u;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int bin = hl + 16 * t;
        const unsigned k = bin < 36 ? ((h36[bin] & ~63u) | (63u - bin)) : 0u;
        if (k > k1) {
          k2 = k1;
          k1 = k;
        } else if (k > k2) {
          k2 = k;
        }
      }
      const unsigned top = half_max(k1, hsel);
      const unsigned sec = half_max(k1 == top ? k2 : k1, hsel);
      const unsigned tv = top & ~63u, sv = sec & ~63u;
      ok = ok && sv < tv - (tv >> 14);  // lead > 6.1e-5 relative
      hk = 63 - (int)(top & 63u);
      ct = fp.ct[hk];
      st = fp.st[hk];
    }
    // ---- descriptor samples (rotated grid, descriptor.py:164-216; or the axis region, :241-242)
    float mg2[4];
    unsigned obs = 0u, unc2 = 0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 err;
      const float2 g = blend_sample<ORIENT>(Fc, geom, hk, j, hl, axis_off(j), ks, cA, cB, err);
      const float a = g.x, bb = g.y;
      // theta0 frame: phi = atan2(b, a) - theta0 (cos theta0 = ct, sin theta0 = -st); 8 octants
      const float ar = fmaf(a, ct, -bb * st), br = fmaf(bb, ct, a * st);
      const float aa = fabsf(ar), ab = fabsf(br);
      const bool upper = br >= 0.0f;
      const bool q_odd = upper ? !(ar > 0.0f) : !(ar < 0.0f);
      const int q = upper ? (q_odd ? 1 : 0) : (q_odd ? 3 : 2);
      const bool second = q_odd ? ab < aa : ab > aa;
      obs |= (unsigned)(2 * q + (second ? 1 : 0)) << (8 * j);
      const float ec = err.x + err.y;  // bound on either rotated component's error
      unc2 |= (fminf(aa, ab) > ec && fabsf(aa - ab) > 2.0f * ec) ? 0u : 1u << j;
      mg2[j] = sqrt_approx(fmaf(a, a, bb * bb));
    }
    if (__any_sync(0xffffffffu, unc2)) {  // near an octant line: float32 side test, else float64
      if (unc2) obs = fb_bin8<ORIENT>(im, Fc, geom, row, col, hl, unc2, obs, hk, &fp, &prm);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) h8[(obs >> (8 * j)) & 255u] += mg2[j];
    // ---- L2 normalise, clamp at 0.2, renormalise (descriptor.py:250-255); lane = bins 8 hl .. 8 hl + 7
    const float4 lo = reinterpret_cast<const float4*>(h8)[0], hi = reinterpret_cast<const float4*>(h8)[1];
    float v[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    float sa = v[0] * v[0], sb = v[1] * v[1];
#pragma unroll
    for (int t = 2; t < 8; t += 2) {
      sa = fmaf(v[t], v[t], sa);
      sb = fmaf(v[t + 1], v[t + 1], sb);
    }
    float ss = sa + sb;
#pragma unroll
    for (int o = 8; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (ss > 0.0f) {
      const float r1 = rsqrtf(ss);
      float s2a = 0.0f, s2b = 0.0f;
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        v[t] = fminf(v[t] * r1, 0.2f);
        v[t + 1] = fminf(v[t + 1] * r1, 0.2f);
        s2a = fmaf(v[t], v[t], s2a);
        s2b = fmaf(v[t + 1], v[t + 1], s2b);
      }
      float s2 = s2a + s2b;
#pragma unroll
      for (int o = 8; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      const float r2 = rsqrtf(s2);
#pragma unroll
      for (int t = 0; t < 8; ++t) v[t] *= r2;
    } else {
#pragma unroll
      for (int t = 0; t < 8; ++t) v[t] = 0.0f;
    }
    if (ok) {
      float4* d = reinterpret_cast<float4*>(out32 + g * 128) + 2 * hl;
      d[0] = make_float4(v[0], v[1], v[2], v[3]);
      d[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
    if (live && !ok && hl == 0) work[atomicAdd(n_work, 1ull)] = g;  // border, other sides, 36-bin near-ties
    __syncwarp();
  }
}

// The geometry table, once per device (stream-ordered before the describe
// launch; under graph capture the build is recorded into the graph and the
// device is not marked ready, so the next eager call builds it for good).
std::atomic<unsigned long long> g_geom_ready{0};
int ensure_geom8(const DescParams& prm, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (g_geom_ready.load() & bit) return PS_OK;
  init_geom8_kernel<<<(36 * 64 + 255) / 256, 256, 0, s>>>(prm);
  PS_LAUNCHED("init_geom8_kernel");
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusNone) g_geom_ready.fetch_or(bit);
  return PS_OK;
}

}  // namespace

template <class Img>
int launch_describe_f32(const Img& im, const ps_image_batch* img, const ps_keypoints* kp, const DescParams& prm,
                        float* out_desc32, int64_t* work, unsigned long long* n_work, cudaStream_t s) {
  F32Params fp{};
  fp.cA = (float)(2.0 * (double)img->nc * img->alpha);
  fp.cB = (float)(2.0 * img->alpha);
  fp.ks = img->pixel_type == PS_PIXELS_RGB8 ? 0.001f : 1.0f;
  for (int k = 0; k < 36; ++k) {
    fp.ct[k] = (float)prm.cos_t[k];
    fp.st[k] = (float)prm.sin_t[k];
    for (int m = 0; m <= 8; ++m) {  // theta0 = 0 when orientation normalisation is off
      const double e = (prm.orient ? prm.theta[k] : 0.0) + m * (prm.two_pi / 8);
      fp.ce8[k][m] = (float)std::cos(e);
      fp.se8[k][m] = (float)std::sin(e);
    }
  }
  for (int m = 0; m <= 36; ++m) {
    fp.ce36[m] = (float)prm.cb36[m];
    fp.se36[m] = (float)prm.sb36[m];
  }
  int st = ensure_geom8(prm, s);
  if (st) return st;
  const int64_t total = (int64_t)img->batch * kp->cap;
  const size_t shm = (size_t)2 * kF32Warps * kPerKpF * sizeof(float);
  auto kern = prm.orient ? describe_f32_kernel<true, Img> : describe_f32_kernel<false, Img>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  int64_t blocks = ((total + 1) / 2 + kF32Warps - 1) / kF32Warps;
  if (blocks > 148 * PS_F32_BLOCKS_PER_SM) blocks = 148 * PS_F32_BLOCKS_PER_SM;
  kern<<<(unsigned)blocks, kF32Warps * 32, shm, s>>>(im, img->image_stride, img->batch, kp->row, kp->col, kp->scale,
                                                      kp->count, kp->cap, prm, fp, out_desc32, work, n_work);
  PS_LAUNCHED("describe_f32_kernel");
  return PS_OK;
}

template int launch_describe_f32<RampU8>(const RampU8&, const ps_image_batch*, const ps_keypoints*, const DescParams&,
                                         float*, int64_t*, unsigned long long*, cudaStream_t);
template int launch_describe_f32<RampRGB8>(const RampRGB8&, const ps_image_batch*, const ps_keypoints*,
                                           const DescParams&, float*, int64_t*, unsigned long long*, cudaStream_t);

}  // namespace ps
