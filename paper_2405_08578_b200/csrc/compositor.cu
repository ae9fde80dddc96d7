// Compositor: inverse-mapped resampling of every placed
// image into the canvas and feather / overwrite blending
// (reference compositor.py:84-160).
//
// One thread per canvas pixel.  Each pixel walks the placements in order, so
// its accumulators see exactly the reference's per-pixel operation sequence
// (accum += where(valid, w * sample, 0), weights += where(valid, w, 0),
// counts += valid, solo = sample); all float64 arithmetic uses explicit _rn
// intrinsics in numpy's evaluation order, so the composite is bit-identical.
// Blocks of up to kBatch placements travel as a kernel parameter; longer
// lists carry the per-pixel state through global memory between launches.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "ps_common.cuh"

namespace ps {
namespace {

constexpr int kBatch = 64;

struct PlaceBatch {
  ps_placement p[kBatch];
  int n;
};

template <class Pix>
__device__ __forceinline__ double px(const ps_placement& P, int r, int c) {
  return (double)reinterpret_cast<const Pix*>(P.data)[(int64_t)r * P.row_pitch + c];
}

// _sample_bilinear (compositor.py:61-74) on clipped coordinates
template <class Pix>
__device__ __forceinline__ double sample_bilinear(const ps_placement& P, double xs, double ys) {
  const int x0 = min(max((int)floor(xs), 0), max(P.nc - 2, 0));
  const int y0 = min(max((int)floor(ys), 0), max(P.nr - 2, 0));
  const double fx = __dsub_rn(xs, (double)x0), fy = __dsub_rn(ys, (double)y0);
  const int x1 = min(x0 + 1, P.nc - 1), y1 = min(y0 + 1, P.nr - 1);
  const double gy = __dsub_rn(1.0, fy), gx = __dsub_rn(1.0, fx);
  double v = __dmul_rn(__dmul_rn(px<Pix>(P, y0, x0), gy), gx);
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(px<Pix>(P, y0, x1), gy), fx));
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(px<Pix>(P, y1, x0), fy), gx));
  return __dadd_rn(v, __dmul_rn(__dmul_rn(px<Pix>(P, y1, x1), fy), fx));
}

// _sample_nearest (compositor.py:77-81): rint is round-half-even, as np.rint
template <class Pix>
__device__ __forceinline__ double sample_nearest(const ps_placement& P, double xs, double ys) {
  const int x = min(max((int)rint(xs), 0), P.nc - 1);
  const int y = min(max((int)rint(ys), 0), P.nr - 1);
  return px<Pix>(P, y, x);
}

template <int RESAMPLE, int BLEND>
__global__ void __launch_bounds__(256) composite_kernel(PlaceBatch pb, int height, int width, int dx, int dy,
                                                        int first, int last, double* __restrict__ out,
                                                        double* __restrict__ weightmap, double* __restrict__ acc_g,
                                                        int* __restrict__ cnt_g, double* __restrict__ solo_g) {
  // placements whose canvas block meets this CTA's tile, in placement order
  __shared__ int list[kBatch];
  __shared__ int n_list;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  if (tid < 32) {
    const int tc0 = blockIdx.x * blockDim.x, tc1 = tc0 + blockDim.x;
    const int tr0 = blockIdx.y * blockDim.y, tr1 = tr0 + blockDim.y;
    int base = 0;
    for (int k0 = 0; k0 < pb.n; k0 += 32) {
      const int k = k0 + tid;
      bool hit = false;
      if (k < pb.n) {
        const ps_placement& P = pb.p[k];
        hit = P.r_lo < tr1 && P.r_hi > tr0 && P.c_lo < tc1 && P.c_hi > tc0;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (hit) list[base + __popc(bal & ((1u << tid) - 1u))] = k;
      base += __popc(bal);
    }
    if (tid == 0) n_list = base;
  }
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (c >= width || r >= height) return;
  const int64_t o = (int64_t)r * width + c;
  double acc = 0.0, wsum = 0.0, solo = 0.0;
  int cnt = 0;
  if (!first) {
    acc = acc_g[o];
    wsum = weightmap[o];
    cnt = cnt_g[o];
    solo = solo_g[o];
  }
  const double X = (double)c + (double)dx, Y = (double)r + (double)dy;  // np.arange(...) + dx
  const int nl = n_list;
  for (int q = 0; q < nl; ++q) {
    const ps_placement& P = pb.p[list[q]];
    if (r < P.r_lo || r >= P.r_hi || c < P.c_lo || c >= P.c_hi) continue;  // outside this image's block
    // inverse.transform_points (registration.py:66-73)
    const double sx = __dadd_rn(__dsub_rn(__dmul_rn(P.cos_t, X), __dmul_rn(P.sin_t, Y)), P.t_x);
    const double sy = __dadd_rn(__dadd_rn(__dmul_rn(P.sin_t, X), __dmul_rn(P.cos_t, Y)), P.t_y);
    const double xmax = (double)(P.nc - 1), ymax = (double)(P.nr - 1);
    const bool valid = sx >= 0.0 && sx <= xmax && sy >= 0.0 && sy <= ymax;
    // an invalid sample adds +0.0 to the (non-negative) accumulators: a no-op
    if (!valid) continue;
    // the reference clips (sx, sy) to the image first: the identity for a valid sample
    double v;
    if (RESAMPLE == PS_RESAMPLE_BILINEAR)
      v = P.pixel_type == PS_PIXELS_U8 ? sample_bilinear<uint8_t>(P, sx, sy) : sample_bilinear<double>(P, sx, sy);
    else
      v = P.pixel_type == PS_PIXELS_U8 ? sample_nearest<uint8_t>(P, sx, sy) : sample_nearest<double>(P, sx, sy);
    if (BLEND == PS_BLEND_OVERWRITE) {
      acc = v;
      wsum = 1.0;
      cnt = 1;
      solo = v;
    } else {
      // feather weight 1 + distance to the nearest source border (compositor.py:146-148);
      // all four distances are >= 0 here, so plain compares pick the minimum
      const double ex = __dsub_rn(xmax, sx), ey = __dsub_rn(ymax, sy);
      const double mx = sx < ex ? sx : ex, my = sy < ey ? sy : ey;
      const double w = __dadd_rn(1.0, mx < my ? mx : my);
      acc = __dadd_rn(acc, __dmul_rn(w, v));
      wsum = __dadd_rn(wsum, w);
      cnt += 1;
      solo = v;
    }
  }
  if (last) {
    // single cover: the sample verbatim (compositor.py:155-157); else accum / weights
    const double res = cnt == 1 ? solo : (wsum > 0.0 ? __ddiv_rn(acc, wsum) : 0.0);
    out[o] = res;
    weightmap[o] = wsum;
  } else {
    acc_g[o] = acc;
    weightmap[o] = wsum;
    cnt_g[o] = cnt;
    solo_g[o] = solo;
  }
}

template <int RESAMPLE, int BLEND>
void launch(const PlaceBatch& pb, int height, int width, int dx, int dy, int first, int last, double* out,
            double* wm, double* acc, int* cnt, double* solo, cudaStream_t st) {
  const dim3 block(32, 8);
  const dim3 grid((width + 31) / 32, (height + 7) / 8);
  composite_kernel<RESAMPLE, BLEND><<<grid, block, 0, st>>>(pb, height, width, dx, dy, first, last, out, wm, acc,
                                                            cnt, solo);
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" int ps_warp_and_blend(const ps_placement* host_placements, int32_t n, int32_t height, int32_t width,
                                 int32_t dx, int32_t dy, int32_t blend, int32_t resample, double* out,
                                 double* weightmap, void* stream) {
  PS_REQUIRE(blend == PS_BLEND_FEATHER || blend == PS_BLEND_OVERWRITE, PS_ERR_VALUE, "unknown blend mode %d", blend);
  PS_REQUIRE(resample == PS_RESAMPLE_BILINEAR || resample == PS_RESAMPLE_NEAREST, PS_ERR_VALUE,
             "unknown resample mode %d", resample);
  PS_REQUIRE(n >= 0 && height >= 0 && width >= 0, PS_ERR_ARGUMENT, "bad sizes");
  if ((int64_t)height * width == 0) return PS_OK;
  PS_REQUIRE(out && weightmap && (n == 0 || host_placements), PS_ERR_ARGUMENT, "null pointer");
  for (int k = 0; k < n; ++k) {
    const ps_placement& P = host_placements[k];
    PS_REQUIRE(P.data && P.nr > 0 && P.nc > 0 && P.row_pitch >= P.nc, PS_ERR_ARGUMENT, "placement %d: bad image", k);
    PS_REQUIRE(P.pixel_type == PS_PIXELS_U8 || P.pixel_type == PS_PIXELS_F64, PS_ERR_ARGUMENT,
               "placement %d: pixel type must be u8 or f64", k);
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* acc = nullptr;
  double* solo = nullptr;
  int* cnt = nullptr;
  const int64_t npx = (int64_t)height * width;
  if (n > kBatch) {  // state carried between launches
    cudaMallocAsync(&acc, npx * sizeof(double), st);
    cudaMallocAsync(&solo, npx * sizeof(double), st);
    cudaMallocAsync(&cnt, npx * sizeof(int), st);
    int s = check_cuda("cudaMallocAsync(compositor state)");
    if (s) return s;
  }
  int k0 = 0;
  do {
    PlaceBatch pb;
    memset(&pb, 0, sizeof(pb));
    pb.n = std::min(kBatch, n - k0);
    if (pb.n > 0) memcpy(pb.p, host_placements + k0, pb.n * sizeof(ps_placement));
    const int first = k0 == 0, last = k0 + pb.n >= n;
    if (resample == PS_RESAMPLE_BILINEAR) {
      if (blend == PS_BLEND_FEATHER)
        launch<PS_RESAMPLE_BILINEAR, PS_BLEND_FEATHER>(pb, height, width, dx, dy, first, last, out, weightmap, acc,
                                                       cnt, solo, st);
      else
        launch<PS_RESAMPLE_BILINEAR, PS_BLEND_OVERWRITE>(pb, height, width, dx, dy, first, last, out, weightmap, acc,
                                                         cnt, solo, st);
    } else {
      if (blend == PS_BLEND_FEATHER)
        launch<PS_RESAMPLE_NEAREST, PS_BLEND_FEATHER>(pb, height, width, dx, dy, first, last, out, weightmap, acc,
                                                      cnt, solo, st);
      else
        launch<PS_RESAMPLE_NEAREST, PS_BLEND_OVERWRITE>(pb, height, width, dx, dy, first, last, out, weightmap, acc,
                                                        cnt, solo, st);
    }
    PS_LAUNCHED("composite_kernel");
    k0 += pb.n;
  } while (k0 < n);
  if (acc) {
    cudaFreeAsync(acc, st);
    cudaFreeAsync(solo, st);
    cudaFreeAsync(cnt, st);
  }
  return check_cuda("compositor");
}
