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
#include <type_traits>

#include "describe_common.cuh"

namespace ps {
namespace {

constexpr int kF32Warps = 8;
constexpr int kFS = 12;              // field row stride (float2)
constexpr int kFR = 11;              // field rows / columns: offsets -5 .. +5 about the keypoint
constexpr int kFieldF2 = kFR * kFS;  // float2 per keypoint
constexpr int kH8W = 8 * 32;         // a warp's descriptor bins, transposed: bin k of lane l at k * 32 + l
constexpr int kH36 = 40;             // 36-bin histogram of a half-warp's keypoint, padded
constexpr int kHistWarpF = kH8W + 2 * kH36;                          // per-warp histogram floats
constexpr int kBoxF = 16 * 2 * kFieldF2 + kF32Warps * kHistWarpF;  // box kernel: 16 fields, 8 warp histograms
static_assert((2 * kFieldF2) % 4 == 0 && kHistWarpF % 4 == 0, "16-byte aligned blocks");
// Tile kernel (window layout of L = 8, C2): a block stages the fields of a
// tile of kTR x kTC windows (32 x 64 pixels, 64 keypoints) once.
constexpr int kTR = 4, kTC = 8;
constexpr int kTFR = kTR * 8 + 10;  // field rows: image rows R0-5 .. R0+36
constexpr int kTFC = kTC * 8 + 10;  // field columns: C0-5 .. C0+68
constexpr int kTFS = 76;            // field row stride (float2)
constexpr int kTPR = kTFR + 2;      // staged pixel rows: R0-6 .. R0+37
constexpr int kTPC = kTC * 8 + 16;  // staged pixel columns: C0-8 .. C0+71 (8-byte chunks)
constexpr int kTileFieldF = 2 * kTFR * kTFS;
constexpr int kTileUnionF = kTPR * kTPC > kF32Warps * kHistWarpF ? kTPR * kTPC : kF32Warps * kHistWarpF;  // pixels, then histograms
constexpr int kTileF = kTileFieldF + kTileUnionF;
static_assert(kTFC <= kTFS && kTileFieldF % 4 == 0, "tile layout");
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
  int tab36;                     // 8-bit grey with a small ramp: axis-sample 36-bins from g_bin36 (exact)
  float ct[36], st[36];          // cos(-theta0_k), sin(-theta0_k) (descriptor.py:180)
  float ce36[37], se36[37];      // cos / sin of the 36-bin edges m 2 pi / 36 (descriptor.py:144)
  float ce8[36][9], se8[36][9];  // cos / sin of theta0_k + m pi / 4: 8-bin edges as absolute angles (:215, 244)
};

// Rotated-grid geometry per (theta0 bin k, sample j of lane l):
// {fx, fy, corner offset (int bits), 0}; x - cx = cos_t u - sin_t v,
// y - cy = sin_t u + cos_t v in float64 (descriptor.py:179-184), floor and
// fraction (:197-200), fractions rounded to float32.  Per device, built once.
__device__ float4 g_geom8[2][36 * 4 * 16];  // [0]: field stride kFS (per-keypoint box), [1]: kTFS (tile)
#ifdef PS_F32_DEBUG
__device__ unsigned g_dbg_n;
__device__ unsigned long long g_dbg_cnt[8];  // fb8 samples, fb8 special lines, fb8 exact, fb36 samples, fb36 exact, lead failures
#define DBG_COUNT(i) atomicAdd(&g_dbg_cnt[i], 1ull)
#else
#define DBG_COUNT(i) ((void)0)
#endif

// 36-bin of an axis sample of an 8-bit grey raster within the quadrant:
// g_bin36[|da| * 256 + |db|] = floor(atan2(|db|, |da|) / 10 degrees), da, db
// the integer differences of a = da + 2 nc alpha, b = db + 2 alpha
// (descriptor.py:135-138, 144).  The bin is exact, not a screen: no integer
// pair with |da|, |db| <= 255 comes within 1.27e-3 (in gradient units) of a
// non-axis 10-degree edge line (tests/test_host_logic.py checks all 2^16),
// while the ramp moves a gradient by |(2 nc alpha, 2 alpha)| < 1e-3
// (tab36's host condition) and the reference's rounding by ~1e-13; on the
// axes the positive ramp decides (da = 0 < db: just below 90 degrees, bin 8;
// db = 0: just above 0, bin 0).  Quadrants by the signs of a, b mirror it.
__device__ uint8_t g_bin36[256 * 256];

__global__ void init_geom8_kernel(DescParams prm) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int e = t; e < 256 * 256; e += gridDim.x * blockDim.x) {
    const int da = e >> 8, db = e & 255;
    int bin = 0;
    if (da == 0 && db > 0) bin = 8;
    else if (db > 0) bin = (int)floor(atan2((double)db, (double)da) * (36.0 / (2.0 * M_PI)));
    g_bin36[e] = (uint8_t)bin;
  }
  if (t >= 36 * 64) return;
  const int k = t >> 6, j = (t >> 4) & 3, l = t & 15;
  const int iv = 2 * (l >> 2) + (j >> 1), iu = 2 * (l & 3) + (j & 1);
  const double u = (double)iu - 3.5, v = (double)iv - 3.5;
  const double x = __dsub_rn(__dmul_rn(prm.cos_t[k], u), __dmul_rn(prm.sin_t[k], v));
  const double y = __dadd_rn(__dmul_rn(prm.sin_t[k], u), __dmul_rn(prm.cos_t[k], v));
  const double x0 = floor(x), y0 = floor(y);
  const float fx = __double2float_rn(x - x0), fy = __double2float_rn(y - y0);
  g_geom8[0][t] = make_float4(fx, fy, __int_as_float((int)y0 * kFS + (int)x0), 0.0f);
  g_geom8[1][t] = make_float4(fx, fy, __int_as_float((int)y0 * kTFS + (int)x0), 0.0f);
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


// Blended gradient (a, b) of sample j of lane l (theta0 bin k) over fields of
// row stride FS (descriptor.py:195-213), ramp constant added once (weights
// sum to one), plus a per-component error bound (ea, eb): kPosF32 x the
// corners' absolute sum, kRelF32 x |value|, kRefNoise.  The axis sample of
// the region when orientation normalisation is off.
template <bool ORIENT, int FS>
__device__ __forceinline__ float2 blend_sample(const float2* Fc, const float4* __restrict__ geom, int k, int j, int l,
                                               int aoff, float ks, float cA, float cB, float2& err) {
  float2 s, sabs;
  if constexpr (ORIENT) {
    const float4 gm = geom[(k * 4 + j) * 16 + l];
    const float fx = gm.x, fy = gm.y;
    const float2* q = Fc + __float_as_int(gm.z);
    const float2 f00 = q[0], f01 = q[1], f10 = q[FS], f11 = q[FS + 1];
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
template <int FS, class Img>
__device__ __noinline__ unsigned fb_bin36(Img im, const float2* Fc, int row, int col, int sr, int sc, unsigned unc,
                                          unsigned bins, const F32Params* fp, const DescParams* prm) {
  for (int j = 0; j < 4; ++j) {
    if (!((unc >> j) & 1u)) continue;
    const int iv = 2 * sr + (j >> 1), iu = 2 * sc + (j & 1);
    const float2 f = Fc[(iv - 4) * FS + (iu - 4)];
    const float a = fmaf(f.x, fp->ks, fp->cA), bb = fmaf(f.y, fp->ks, fp->cB);
    const float x = wrap_two_pi_f(atan2_f32(bb, a)) * 5.729577951308232f;
    const int m = min(max(__float2int_rn(x), 0), 36);
    const int side = side_f32(a, bb, fp->ce36[m], fp->se36[m], fmaf(kRelF32, fabsf(a), kRefNoise),
                              fmaf(kRelF32, fabsf(bb), kRefNoise));
    DBG_COUNT(3);
    if (!side) DBG_COUNT(4);
    const int bin = side ? side_to_bin(side, m, 36)
                         : exact_axis_bin(im, row - 4 + iv, col - 4 + iu, prm->cb36[m], prm->sb36[m], m, 36, prm->k36,
                                          prm->two_pi);
    bins = (bins & ~(255u << (8 * j))) | ((unsigned)bin << (8 * j));
  }
  return bins;
}

// 8-bin octants of the descriptor samples flagged in `unc` (rare): the
// float32 side test of the nearest bin line with a per-corner error bound,
// else the reference's float64 arithmetic.
//
// Per-corner bound: the reference blends with weights from its float64
// fractions, ours come from fractions rounded to float32 (|dfx| <= 2^-24 fx
// + 8e-12, the reference's own position rounding for images < 32768 wide),
// 1 - fx rounded (<= min(fx, 2^-25)), weight products and the four-term FMA
// chain rounded (5 ulp of the weight).  So |our blend - reference blend| <=
// sum_ij c_ij |f_ij| with c_00 = 3e-7 w00 + gy dgx + gx dgy, etc.: a corner
// with a (near) zero weight contributes (almost) nothing, which decides the
// samples that sit on a pixel row or column.
//
// Axis and diagonal bin lines (theta0 + m pi/4 a multiple of pi/4, i.e.
// theta0 in {45, 135, 225, 315} degrees, or no orientation normalisation):
// sd = b cos e - a sin e is then, up to a positive factor, an exact integer
// combination of the corner fields plus the ramp constants, blended once --
// so gradients that are exactly axis-aligned or diagonal in the integer
// image, whose side only the ramp term (2 nc alpha, 2 alpha) decides, are
// decided here; the true line differs from the exact axis or diagonal by
// float64 rounding (~1e-16 rad), inside kBand.
template <bool ORIENT, int FS, class Img>
__device__ __noinline__ unsigned fb_bin8(Img im, const float2* Fc, const float4* geom, int row, int col, int l,
                                         unsigned unc, unsigned obs, int hk, const F32Params* fp,
                                         const DescParams* prm) {
  const float theta0f = ORIENT ? (float)prm->theta[hk] : 0.0f;
  const float ks = fp->ks;
  const int sr = l >> 2, sc = l & 3;
  for (int j = 0; j < 4; ++j) {
    if (!((unc >> j) & 1u)) continue;
    const int iv = 2 * sr + (j >> 1), iu = 2 * sc + (j & 1);
    float2 f00, f01, f10, f11;
    float w00, w01, w10, w11, c00, c01, c10, c11;
    if constexpr (ORIENT) {
      const float4 gm = geom[(hk * 4 + j) * 16 + l];
      const float fx = gm.x, fy = gm.y;
      const float2* q = Fc + __float_as_int(gm.z);
      f00 = q[0];
      f01 = q[1];
      f10 = q[FS];
      f11 = q[FS + 1];
      const float gx = 1.0f - fx, gy = 1.0f - fy;
      w00 = gy * gx;
      w01 = gy * fx;
      w10 = fy * gx;
      w11 = fy * fx;
      const float dfx = fmaf(6e-8f, fx, 8e-12f), dfy = fmaf(6e-8f, fy, 8e-12f);
      const float dgx = dfx + fminf(fx, 3e-8f), dgy = dfy + fminf(fy, 3e-8f);
      c00 = 1.25f * fmaf(3e-7f, w00, fmaf(gy, dgx, gx * dgy));
      c01 = 1.25f * fmaf(3e-7f, w01, fmaf(gy, dfx, fx * dgy));
      c10 = 1.25f * fmaf(3e-7f, w10, fmaf(fy, dgx, gx * dfy));
      c11 = 1.25f * fmaf(3e-7f, w11, fmaf(fy, dfx, fx * dfy));
    } else {
      f00 = Fc[(iv - 4) * FS + (iu - 4)];
      f01 = f10 = f11 = make_float2(0.0f, 0.0f);
      w00 = 1.0f;
      w01 = w10 = w11 = 0.0f;
      c00 = c01 = c10 = c11 = 0.0f;
    }
    auto blend = [&](float v00, float v01, float v10, float v11) {
      return fmaf(v11, w11, fmaf(v10, w10, fmaf(v01, w01, v00 * w00)));
    };
    auto bound = [&](float v00, float v01, float v10, float v11) {
      return ks * fmaf(c11, fabsf(v11), fmaf(c10, fabsf(v10), fmaf(c01, fabsf(v01), c00 * fabsf(v00))));
    };
    const float a = fmaf(blend(f00.x, f01.x, f10.x, f11.x), ks, fp->cA);
    const float bb = fmaf(blend(f00.y, f01.y, f10.y, f11.y), ks, fp->cB);
    const float xb = wrap_two_pi_f(atan2_f32(bb, a) - theta0f) * 1.2732395447351628f;
    const int m = min(max(__float2int_rn(xb), 0), 8);
    const float ce = fp->ce8[hk][m], se = fp->se8[hk][m];
    int side = 0;
    const float ace = fabsf(ce), ase = fabsf(se);
    if (ace < 1e-6f || ase < 1e-6f || fabsf(ace - ase) < 1e-6f) {
      // axis or diagonal line: sd / k = sy * b - sx * a with sx, sy in {0, +-1}
      DBG_COUNT(1);
      const float sx = ase < 1e-6f ? 0.0f : copysignf(1.0f, se), sy = ace < 1e-6f ? 0.0f : copysignf(1.0f, ce);
      const float h00 = fmaf(sy, f00.y, -sx * f00.x), h01 = fmaf(sy, f01.y, -sx * f01.x);
      const float h10 = fmaf(sy, f10.y, -sx * f10.x), h11 = fmaf(sy, f11.y, -sx * f11.x);
      const float sd = fmaf(blend(h00, h01, h10, h11), ks, fmaf(sy, fp->cB, -sx * fp->cA));
      const float bd = bound(h00, h01, h10, h11) + fmaf(kRelF32, fabsf(sd), 2.0f * kRefNoise) +
                       kBand * (fabsf(a) + fabsf(bb));
      side = sd > bd ? 1 : (sd < -bd ? -1 : 0);
    } else {
      const float ea = bound(f00.x, f01.x, f10.x, f11.x) + fmaf(kRelF32, fabsf(a), kRefNoise);
      const float eb = bound(f00.y, f01.y, f10.y, f11.y) + fmaf(kRelF32, fabsf(bb), kRefNoise);
      side = side_f32(a, bb, ce, se, ea, eb);
    }
    DBG_COUNT(0);
    if (!side) DBG_COUNT(2);
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

// Dominant orientation of a keypoint whose float32 36-bin sums have no clear
// lead (rare): float64 magnitudes hypot(a, b) of the reference's ramped
// differences (descriptor.py:135-137), summed in exact fixed point (46-bit
// samples in two 26-bit limbs, native shared atomics, order-independent) into
// the bins already decided, first argmax (:146).  Called by the whole warp;
// each half-warp resolves its own keypoint in `scr` (72 words, re-zeroed by
// the caller).
template <class Img>
__device__ __noinline__ int orient_exact36(Img im, int row, int col, int hl, int hsel, unsigned bins, unsigned* scr) {
  for (int q = hl; q < 72; q += 16) scr[q] = 0u;
  __syncwarp();
  const int sr = hl >> 2, sc = hl & 3;
  double mg[4];
  double mx = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = row - 4 + 2 * sr + (j >> 1), c = col - 4 + 2 * sc + (j & 1);
    const double a = __dsub_rn(im.at(r + 1, c), im.at(r - 1, c));
    const double b = __dsub_rn(im.at(r, c + 1), im.at(r, c - 1));
    mg[j] = hypot(a, b);
    mx = fmax(mx, mg[j]);
  }
  // every magnitude < 2^(eb - 1022): scale 2^(1068 - eb) keeps it below 2^46, a bin sum of 64 below 2^52
  const unsigned eb = half_max((unsigned)__double2hiint(mx), hsel) >> 20;
  const double fxs = eb == 0u ? 1.0 : __hiloint2double(min(2091 - (int)eb, 2046) << 20, 0);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const unsigned long long q = __double2ull_rn(__dmul_rn(mg[j], fxs));
    const int bin = (bins >> (8 * j)) & 255;
    atomicAdd(scr + bin, (unsigned)(q & 0x3FFFFFFull));
    atomicAdd(scr + 36 + bin, (unsigned)(q >> 26));
  }
  __syncwarp();
  unsigned long long best = 0ull;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const int bin = hl + 16 * t;
    if (bin < 36) {
      const unsigned long long v = (unsigned long long)scr[bin] + ((unsigned long long)scr[36 + bin] << 26);
      const unsigned long long key = (v << 6) | (unsigned long long)(63 - bin);
      best = key > best ? key : best;
    }
  }
#pragma unroll
  for (int o = 8; o; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
    best = other > best ? other : best;
  }
  __syncwarp();
  return 63 - (int)(best & 63ull);
}

// The descriptor of one keypoint per half-warp from its staged fields (Fc =
// the field at the keypoint, row stride FS): dominant orientation, rotated
// samples, histogram, normalisation, float32 row (descriptor.py:219-256).
// Keypoints that are not `fast` are appended to `work` for the float64
// kernel.  h8: this lane's 8 bins, h8[k * 32] (zeroed; conflict-free: lane
// l always hits bank l), h36: the half's 36-bin sums (zeroed), scr: 72 words
// of scratch for this half (inside the warp's bins; re-zeroed after use).
template <bool ORIENT, int FS, class Img>
__device__ __forceinline__ void describe_kp(const Img& im, const float2* Fc, const float4* __restrict__ geom, int row,
                                            int col, bool fast, bool live, int64_t g, float* h8, unsigned* h36,
                                            unsigned* scr, int hl, int hsel, const F32Params& fp,
                                            const DescParams& prm, float* __restrict__ out32,
                                            int64_t* __restrict__ work, unsigned long long* __restrict__ n_work) {
  const int sr = hl >> 2, sc = hl & 3;  // this lane's subregion (descriptor.py:247-248)
  const float cA = fp.cA, cB = fp.cB, ks = fp.ks;
  // axis region r0 = row - 4, c0 = col - 4 (descriptor.py:129-130): field offset of sample j
  auto axis_off = [&](int j) { return (2 * sr + (j >> 1) - 4) * FS + (2 * sc + (j & 1) - 4); };
  bool ok = fast;
  float ct = 1.0f, st = 0.0f;
  int hk = 0;
  if constexpr (ORIENT) {
    // ---- dominant orientation: 36-bin histogram of the axis region (descriptor.py:142-146)
    float mg[4];
    unsigned bins = 0u, unc = 0u;
    constexpr bool kU8 = std::is_same<Img, RampU8>::value;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = Fc[axis_off(j)];
      const float a = fmaf(f.x, ks, cA), bb = fmaf(f.y, ks, cB);
      int bin;
      if (kU8 && fp.tab36) {
        // exact table bin: |da|, |db| from the float bits (|d| + 2^23), quadrant from the signs of a, b
        const unsigned ia = __float_as_uint(fabsf(f.x) + 8388608.0f), ib = __float_as_uint(fabsf(f.y) + 8388608.0f);
        const int t = __ldg(g_bin36 + __byte_perm(ib, ia, 0x2240));  // |da| << 8 | |db|
        const bool na = a < 0.0f, nb = bb < 0.0f;
        bin = nb ? (na ? 18 + t : 35 - t) : (na ? 17 - t : t);
        bins |= (unsigned)bin << (8 * j);
        mg[j] = sqrt_approx(fmaf(a, a, bb * bb));
        continue;
      }
      const float x = wrap_two_pi_f(atan2_f32(bb, a)) * 5.729577951308232f;
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
      if (unc) bins = fb_bin36<FS>(im, Fc, row, col, sr, sc, unc, bins, &fp, &prm);
    }
    // exact fixed-point sums (native shared atomics, order-independent):
    // q = rint(mag 2^(22 - e)) <= 2^23 for the half's largest magnitude < 2^(e + 1)
    const unsigned eb = half_max(__float_as_uint(fmaxf(fmaxf(mg[0], mg[1]), fmaxf(mg[2], mg[3]))), hsel) >> 23;
    const float s36 = eb == 0u ? 1.0f : __uint_as_float((unsigned)min(max(276 - (int)eb, 1), 254) << 23);
    // A lane's four samples (one subregion) usually share a bin in smooth
    // regions: then one atomic, else four.
    unsigned q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = __float_as_uint(fmaf(mg[j], s36, 8388608.0f)) - 0x4B000000u;
    const unsigned b0 = bins & 255u;
    if (bins == b0 * 0x01010101u) {
      atomicAdd(h36 + b0, (q[0] + q[1]) + (q[2] + q[3]));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) atomicAdd(h36 + ((bins >> (8 * j)) & 255u), q[j]);
    }
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
    hk = 63 - (int)(top & 63u);
    const bool lead = sv < tv - (tv >> 14);  // lead > 6.1e-5 relative: the float64 sums agree
    if (__any_sync(0xffffffffu, fast && !lead)) {  // near-tie: float64 magnitudes, exact sums
      DBG_COUNT(5);
      const int hx = orient_exact36(im, row, col, hl, hsel, bins, scr);
      if (!lead) hk = hx;
#pragma unroll
      for (int k = 0; k < 8; ++k) h8[32 * k] = 0.0f;
      __syncwarp();
    }
    ct = fp.ct[hk];
    st = fp.st[hk];
  }
  // ---- descriptor samples (rotated grid, descriptor.py:164-216; or the axis region, :241-242)
  float mg2[4];
  unsigned obs = 0u, unc2 = 0u;
#pragma unroll 2
  for (int j = 0; j < 4; ++j) {
    float2 err;
    const float2 gv = blend_sample<ORIENT, FS>(Fc, geom, hk, j, hl, axis_off(j), ks, cA, cB, err);
    const float a = gv.x, bb = gv.y;
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
    if (unc2) obs = fb_bin8<ORIENT, FS>(im, Fc, geom, row, col, hl, unc2, obs, hk, &fp, &prm);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) h8[32 * ((obs >> (8 * j)) & 255u)] += mg2[j];
  // ---- L2 normalise, clamp at 0.2, renormalise (descriptor.py:250-255); lane = bins 8 hl .. 8 hl + 7
  float2 p[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) p[k] = make_float2(h8[64 * k], h8[64 * k + 32]);
  float2 q2 = __fmul2_rn(p[0], p[0]);
#pragma unroll
  for (int k = 1; k < 4; ++k) q2 = __ffma2_rn(p[k], p[k], q2);
  float ss = q2.x + q2.y;
#pragma unroll
  for (int o = 8; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float r1 = ss > 0.0f ? rsqrtf(ss) : 0.0f;  // a flat (all-zero) histogram stays zero
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    p[k] = __fmul2_rn(p[k], make_float2(r1, r1));
    p[k] = make_float2(fminf(p[k].x, 0.2f), fminf(p[k].y, 0.2f));
  }
  q2 = __fmul2_rn(p[0], p[0]);
#pragma unroll
  for (int k = 1; k < 4; ++k) q2 = __ffma2_rn(p[k], p[k], q2);
  float s2 = q2.x + q2.y;
#pragma unroll
  for (int o = 8; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  const float r2 = ss > 0.0f ? rsqrtf(s2) : 0.0f;
#pragma unroll
  for (int k = 0; k < 4; ++k) p[k] = __fmul2_rn(p[k], make_float2(r2, r2));
  if (ok) {
    float4* d = reinterpret_cast<float4*>(out32 + g * 128) + 2 * hl;
    d[0] = make_float4(p[0].x, p[0].y, p[1].x, p[1].y);
    d[1] = make_float4(p[2].x, p[2].y, p[3].x, p[3].y);
  }
  if (live && !ok && hl == 0) work[atomicAdd(n_work, 1ull)] = g;  // border keypoints, other region sides
}

// Any keypoint list: a half-warp per keypoint stages its own 11 x 11 fields.
template <bool ORIENT, class Img>
__global__ void __launch_bounds__(kF32Warps * 32, PS_F32_MINB)
    describe_f32_kernel(Img img, int64_t img_stride, int B, const int32_t* __restrict__ kp_row,
                        const int32_t* __restrict__ kp_col, const int32_t* __restrict__ kp_scale,
                        const int32_t* __restrict__ counts, int64_t cap, const __grid_constant__ DescParams prm,
                        const __grid_constant__ F32Params fp, float* __restrict__ out32,
                        int64_t* __restrict__ work, unsigned long long* __restrict__ n_work) {
  extern __shared__ float4 smf4[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, hsel = lane >> 4, hl = lane & 15;
  float2* F = reinterpret_cast<float2*>(reinterpret_cast<float*>(smf4) + (2 * wid + hsel) * 2 * kFieldF2);
  float* hw = reinterpret_cast<float*>(smf4) + 16 * 2 * kFieldF2 + wid * kHistWarpF;  // this warp's histograms
  float* h8 = hw + lane;
  unsigned* h36 = reinterpret_cast<unsigned*>(hw + kH8W + hsel * kH36);
  unsigned* scr = reinterpret_cast<unsigned*>(hw + hsel * (kH8W / 2));
  const float2* Fc = F + 5 * kFS + 5;  // field at offset (0, 0) from the keypoint
  const float4* __restrict__ geom = g_geom8[0];
  const int64_t total = (int64_t)B * cap;
  const int64_t npairs = (total + 1) / 2;
  const bool img_ok = img.nr >= 13 && img.nc >= 13;
  const int64_t gstep = 2 * (int64_t)gridDim.x * kF32Warps;
  int64_t gi0 = 2 * ((int64_t)blockIdx.x * kF32Warps + wid) + hsel;
  int bcur = (int)(gi0 / cap);
  int64_t icur = gi0 - (int64_t)bcur * cap;
  const int qstep = (int)(gstep / cap);
  const int64_t rstep = gstep - (int64_t)qstep * cap;
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
#pragma unroll
    for (int k = 0; k < 8; ++k) h8[32 * k] = 0.0f;
    if (hl < kH36 / 4) reinterpret_cast<uint4*>(h36)[hl] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    describe_kp<ORIENT, kFS>(im, Fc, geom, row, col, fast, live, g, h8, h36, scr, hl, hsel, fp, prm, out32, work,
                             n_work);
    __syncwarp();
  }
}

constexpr int kChunksPerThread = (kTPR * (kTPC / 8) + kF32Warps * 32 - 1) / (kF32Warps * 32);
// The 8-byte pixel chunks of tile task `task` this thread stages: chunk q =
// row q / (kTPC / 8) (image row R0 - 6 + r), 8 columns from C0 - 8 + 8 k;
// pixels outside the image read as 0 (no interior keypoint's fields use them).
__device__ __forceinline__ void load_tile_chunks(const RampU8& img, int64_t img_stride, int nr, int nc, int pitch,
                                                 int64_t task, int tiles, int tcn, int tid,
                                                 uint2 (&pre)[kChunksPerThread]) {
  const int b = (int)(task / tiles), t = (int)(task - (int64_t)b * tiles);
  const int tr = t / tcn, tc = t - tr * tcn;
  const int R0 = tr * kTR * 8, C0 = tc * kTC * 8;
  const uint8_t* ip = img.p + (int64_t)b * img_stride;
#pragma unroll
  for (int u = 0; u < kChunksPerThread; ++u) {
    const int q = tid + u * kF32Warps * 32;
    const int r = q / (kTPC / 8), k = q - r * (kTPC / 8);
    const int gr = R0 - 6 + r, gc = C0 - 8 + 8 * k;
    uint2 w = make_uint2(0u, 0u);
    if (q < kTPR * (kTPC / 8) && gr >= 0 && gr < nr) {
      if (gc >= 0 && gc + 8 <= nc) {
        w = __ldg(reinterpret_cast<const uint2*>(ip + gr * pitch + gc));
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (gc + i >= 0 && gc + i < nc) {
            const unsigned by = __ldg(ip + gr * pitch + gc + i);
            if (i < 4) w.x |= by << (8 * i);
            else w.y |= by << (8 * (i - 4));
          }
      }
    }
    pre[u] = w;
  }
}

// The window layout of L = 8 (ps_detect of a nested scale set with dedupe:
// slots 2w, 2w+1 = max, min of window w, row-major): a block stages the
// fields of a tile of kTR x kTC windows with coalesced 8-byte loads, then
// its 16 half-warps describe the tile's 64 keypoints.  Keypoints outside
// their window (any other layout) or near the border go to `work`.
template <bool ORIENT>
__global__ void __launch_bounds__(kF32Warps * 32, PS_F32_MINB)
    describe_f32_tile_kernel(RampU8 img, int64_t img_stride, int B, const int32_t* __restrict__ kp_row,
                             const int32_t* __restrict__ kp_col, const int32_t* __restrict__ counts, int64_t cap,
                             const __grid_constant__ DescParams prm, const __grid_constant__ F32Params fp,
                             float* __restrict__ out32, int64_t* __restrict__ work,
                             unsigned long long* __restrict__ n_work) {
  extern __shared__ float4 smf4[];
  float* sm = reinterpret_cast<float*>(smf4);
  float2* F = reinterpret_cast<float2*>(sm);           // [kTFR][kTFS]: image rows R0-5.., columns C0-5..
  float* px = sm + kTileFieldF;                         // [kTPR][kTPC]: image rows R0-6.., columns C0-8..
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31, hsel = lane >> 4, hl = lane & 15;
  float* hw = sm + kTileFieldF + wid * kHistWarpF;  // this warp's histograms: alias px once the fields are built
  float* h8 = hw + lane;
  unsigned* h36 = reinterpret_cast<unsigned*>(hw + kH8W + hsel * kH36);
  unsigned* scr = reinterpret_cast<unsigned*>(hw + hsel * (kH8W / 2));
  int* kpr = reinterpret_cast<int*>(sm + kTileF);  // the tile's keypoints: row, column, slot / flags
  int* kpc = kpr + 2 * kTR * kTC;
  int* kpf = kpc + 2 * kTR * kTC;
  int* kctr = kpf + 2 * kTR * kTC;  // next window of the tile to describe
  const float4* __restrict__ geom = g_geom8[1];
  const int nr = img.nr, nc = img.nc, pitch = (int)img.pitch;
  const int nwr = (nr + 7) >> 3, ncw = (nc + 7) >> 3;
  const int trn = (nwr + kTR - 1) / kTR, tcn = (ncw + kTC - 1) / kTC;
  const int tiles = trn * tcn;
  const int64_t ntask = (int64_t)B * tiles;
  uint2 pre[kChunksPerThread];
  for (int64_t task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int b = (int)(task / tiles), t = (int)(task - (int64_t)b * tiles);
    const int tr = t / tcn, tc = t - tr * tcn;
    const int R0 = tr * kTR * 8, C0 = tc * kTC * 8;
    const uint8_t* ip = img.p + (int64_t)b * img_stride;
    const int64_t gb = (int64_t)b * cap;
    // ---- the tile's 64 keypoints, once: keypoint k (round k / 16, warp k / 2 % 8, half k % 2) is
    //      window (tr * kTR + k / 16, tc * kTC + k / 2 % 8)'s max (k even) / min; slot << 2 | live << 1 | fast
    if (tid == 0) *kctr = 0;
    if (tid < 2 * kTR * kTC) {
      const int wr = tr * kTR + (tid >> 4), wc = tc * kTC + ((tid >> 1) & 7);
      const int slot = 2 * (wr * ncw + wc) + (tid & 1);
      const bool live = wr < nwr && wc < ncw && (!counts || slot < counts[b]);
      const int row = live ? kp_row[gb + slot] : 0, col = live ? kp_col[gb + slot] : 0;
      const bool fast = live && row >= wr * 8 && row < wr * 8 + 8 && col >= wc * 8 && col < wc * 8 + 8 &&
                        row >= 6 && row <= nr - 7 && col >= 6 && col <= nc - 7 && prm.default_w8;
      if (live && !fast) work[atomicAdd(n_work, 1ull)] = gb + slot;  // border keypoints, other layouts
      kpr[tid] = row;
      kpc[tid] = col;
      kpf[tid] = slot << 2 | (live ? 2 : 0) | (fast ? 1 : 0);
    }
    // ---- pixels -> float keys (exact)
    load_tile_chunks(img, img_stride, nr, nc, pitch, task, tiles, tcn, tid, pre);
#pragma unroll
    for (int u = 0; u < kChunksPerThread; ++u) {
      const int q = tid + u * kF32Warps * 32;
      if (q < kTPR * (kTPC / 8)) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          v[i] = __uint_as_float(__byte_perm(pre[u].x, 0x4Bu, 0x4550u + i)) - 8388608.0f;
          v[4 + i] = __uint_as_float(__byte_perm(pre[u].y, 0x4Bu, 0x4550u + i)) - 8388608.0f;
        }
        float4* d = reinterpret_cast<float4*>(px + q * 8);
        d[0] = make_float4(v[0], v[1], v[2], v[3]);
        d[1] = make_float4(v[4], v[5], v[6], v[7]);
      }
    }
    __syncthreads();
    // ---- fields: a(fr, fc) = px[fr+2][fc+3] - px[fr][fc+3], b = px[fr+1][fc+4] - px[fr+1][fc+2]
    //      (descriptor.py:135-136); thread = a column run of 14 rows
    if (tid < 3 * kTFC) {
      const int fc = tid % kTFC, fr0 = (tid / kTFC) * 14;
      const float* pc = px + fr0 * kTPC + fc + 3;
      float up = pc[0], mid = pc[kTPC];
#pragma unroll
      for (int i = 0; i < 14; ++i) {
        const float dn = pc[(i + 2) * kTPC];
        const float* prow = pc + (i + 1) * kTPC;
        F[(fr0 + i) * kTFS + fc] = make_float2(dn - up, prow[1] - prow[-1]);
        up = mid;
        mid = dn;
      }
    }
    __syncthreads();
    // the next task's pixel chunks: their global latency overlaps this task's keypoints

    // ---- the tile's 64 keypoints, 16 per round; the two halves of a warp take window w's max and min
#pragma unroll
    for (int k = 0; k < 8; ++k) h8[32 * k] = 0.0f;
    if (hl < kH36 / 4) reinterpret_cast<uint4*>(h36)[hl] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    // windows are claimed dynamically (a warp whose keypoints take a rare path
    // does not hold the block's next barrier while the others idle)
#pragma unroll 1
    for (;;) {
      int wl = 0;
      if (lane == 0) wl = atomicAdd(kctr, 1);
      wl = __shfl_sync(0xffffffffu, wl, 0);
      if (wl >= kTR * kTC) break;
      const int k = 2 * wl + hsel;
      const int f = kpf[k];
      const bool fast = f & 1;
      if (!__any_sync(0xffffffffu, fast)) continue;
      int row = kpr[k], col = kpc[k];
      // a half without a fast keypoint shadows its partner's (same window): in the image and the tile
      const int prow = __shfl_xor_sync(0xffffffffu, row, 16), pcol = __shfl_xor_sync(0xffffffffu, col, 16);
      if (!fast) {
        row = prow;
        col = pcol;
      }
      const int64_t g = gb + (f >> 2);
      RampU8 im = img;
      im.p = ip;
      const float2* Fc = F + (row - (R0 - 5)) * kTFS + (col - (C0 - 5));
      describe_kp<ORIENT, kTFS>(im, Fc, geom, row, col, fast, fast, g, h8, h36, scr, hl, hsel, fp, prm, out32,
                                work, n_work);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 8; ++k) h8[32 * k] = 0.0f;
      if (hl < kH36 / 4) reinterpret_cast<uint4*>(h36)[hl] = make_uint4(0u, 0u, 0u, 0u);
      __syncwarp();
    }
    __syncthreads();
  }
}

// The geometry tables, once per device (stream-ordered before the describe
// launch; under graph capture the build is recorded into the graph and the
// device is not marked ready, so the next eager call builds it for good).
std::atomic<unsigned long long> g_geom_ready{0};
int ensure_geom8(const DescParams& prm, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (g_geom_ready.load() & bit) return PS_OK;
  init_geom8_kernel<<<64, 256, 0, s>>>(prm);
  PS_LAUNCHED("init_geom8_kernel");
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusNone) g_geom_ready.fetch_or(bit);
  return PS_OK;
}

template <class Img>
void fill_f32_params(F32Params& fp, const ps_image_batch* img, const DescParams& prm) {
  fp.cA = (float)(2.0 * (double)img->nc * img->alpha);
  fp.cB = (float)(2.0 * img->alpha);
  fp.ks = img->pixel_type == PS_PIXELS_RGB8 ? 0.001f : 1.0f;
  fp.tab36 = img->pixel_type == PS_PIXELS_U8 && std::hypot(2.0 * (double)img->nc * img->alpha, 2.0 * img->alpha) < 1e-3;
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
}

}  // namespace

#ifdef PS_F32_DEBUG
extern "C" __attribute__((visibility("default"))) int ps_f32_debug_counts(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_dbg_cnt, sizeof(g_dbg_cnt));
  unsigned long long z[8] = {};
  cudaMemcpyToSymbol(g_dbg_cnt, z, sizeof(z));
  return 0;
}
#endif

template <class Img>
int launch_describe_f32(const Img& im, const ps_image_batch* img, const ps_keypoints* kp, int32_t default_scale,
                        const DescParams& prm, float* out_desc32, bool window_slots, int64_t* work,
                        unsigned long long* n_work, cudaStream_t s) {
  F32Params fp{};
  fill_f32_params<Img>(fp, img, prm);
  int st = ensure_geom8(prm, s);
  if (st) return st;
  const int64_t total = (int64_t)img->batch * kp->cap;
  // tile kernel: the window layout of L = 8 (default scale) of an 8-bit grey batch with 8-byte aligned rows
  const bool tile = window_slots && std::is_same<Img, RampU8>::value && kp->scale == nullptr && prm.default_w8 &&
                    default_scale == 8 && ((uintptr_t)img->data) % 8 == 0 && img->row_pitch % 8 == 0 &&
                    (img->batch == 1 || img->image_stride % 8 == 0);
  if constexpr (std::is_same<Img, RampU8>::value) {
    if (tile) {
      const size_t shm = (size_t)kTileF * sizeof(float) + (3 * 2 * kTR * kTC + 4) * sizeof(int);
      auto kern = prm.orient ? describe_f32_tile_kernel<true> : describe_f32_tile_kernel<false>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
      const int nwr = (img->nr + 7) / 8, ncw = (img->nc + 7) / 8;
      const int64_t tasks = (int64_t)img->batch * ((nwr + kTR - 1) / kTR) * ((ncw + kTC - 1) / kTC);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kF32Warps * 32, shm);
      int64_t blocks = (int64_t)148 * std::max(per_sm, 1);
      if (blocks > tasks) blocks = tasks;
      kern<<<(unsigned)blocks, kF32Warps * 32, shm, s>>>(im, img->image_stride, img->batch, kp->row, kp->col,
                                                          kp->count, kp->cap, prm, fp, out_desc32, work, n_work);
      PS_LAUNCHED("describe_f32_tile_kernel");
      return PS_OK;
    }
  }
  const size_t shm = (size_t)kBoxF * sizeof(float);
  auto kern = prm.orient ? describe_f32_kernel<true, Img> : describe_f32_kernel<false, Img>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  int64_t blocks = ((total + 1) / 2 + kF32Warps - 1) / kF32Warps;
  if (blocks > 148 * PS_F32_BLOCKS_PER_SM) blocks = 148 * PS_F32_BLOCKS_PER_SM;
  kern<<<(unsigned)blocks, kF32Warps * 32, shm, s>>>(im, img->image_stride, img->batch, kp->row, kp->col, kp->scale,
                                                      kp->count, kp->cap, prm, fp, out_desc32, work, n_work);
  PS_LAUNCHED("describe_f32_kernel");
  return PS_OK;
}

template int launch_describe_f32<RampU8>(const RampU8&, const ps_image_batch*, const ps_keypoints*, int32_t,
                                         const DescParams&, float*, bool, int64_t*, unsigned long long*,
                                         cudaStream_t);
template int launch_describe_f32<RampRGB8>(const RampRGB8&, const ps_image_batch*, const ps_keypoints*, int32_t,
                                           const DescParams&, float*, bool, int64_t*, unsigned long long*,
                                           cudaStream_t);

}  // namespace ps
