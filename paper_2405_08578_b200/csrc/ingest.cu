// RGB ingest helpers: the BT.601 grey the reference
// computes with numpy (`rgb @ LUMA`, imaging.py:66-68) on the device.
#include "ps_common.cuh"

namespace ps {
namespace {

// mismatches between the run host's grey table and bt601_fma over all 2^24 triples
__global__ void gray_table_check(const double* __restrict__ lut, unsigned long long* __restrict__ bad) {
  unsigned long long cnt = 0;
  for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < (1u << 24); k += gridDim.x * blockDim.x)
    cnt += __double_as_longlong(lut[k]) != __double_as_longlong(bt601_fma(k >> 16, (k >> 8) & 255u, k & 255u));
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(bad, cnt);
}

__global__ void rgb_to_gray(RampRGB8 im, int64_t img_stride, int B, double* __restrict__ out) {
  const int64_t per = (int64_t)im.nr * im.nc;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)B * per;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(t / per);
    const int r = (int)((t % per) / im.nc), c = (int)(t % im.nc);
    RampRGB8 q = im;
    q.p = im.p + (int64_t)b * img_stride * RampRGB8::kElem;
    out[t] = q.gray(r, c);
  }
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" int ps_gray_table_check(const double* lut, unsigned long long* out_mismatches, void* stream) {
  PS_REQUIRE(lut && out_mismatches, PS_ERR_ARGUMENT, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(out_mismatches, 0, sizeof(unsigned long long), st);
  gray_table_check<<<148 * 8, 256, 0, st>>>(lut, out_mismatches);
  PS_LAUNCHED("gray_table_check");
  return PS_OK;
}

extern "C" int ps_rgb_to_gray(const ps_image_batch* img, double* out, void* stream) {
  PS_REQUIRE(img && img->data && out, PS_ERR_ARGUMENT, "null argument");
  PS_REQUIRE(img->pixel_type == PS_PIXELS_RGB8, PS_ERR_ARGUMENT, "ps_rgb_to_gray needs RGB8 pixels");
  PS_REQUIRE((int64_t)img->nr * img->row_pitch * 3 < (int64_t)INT32_MAX, PS_ERR_ARGUMENT, "image too large");
  RampRGB8 im{(const uint8_t*)img->data, img->row_pitch, img->nr, img->nc, 0.0, img->gray_lut};
  const int64_t total = (int64_t)img->batch * img->nr * img->nc;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  rgb_to_gray<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, (cudaStream_t)stream>>>(
      im, img->batch > 1 ? img->image_stride : 0, img->batch, out);
  PS_LAUNCHED("rgb_to_gray");
  return PS_OK;
}
