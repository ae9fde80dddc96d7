// K1 -- multiscale window-extremum detector (reference detector.py:154-172).
//
// Semantics reproduced:
//  * windows of side L tile the image row-major, trailing ones shrunk
//    (detector.py:87-103); window_index = (row0/L)*ceil(nc/L) + col0/L;
//  * per window the FIRST argmax / argmin of the ramped float64 raster
//    (detector.py:114-119).  For 8-bit input with a valid ramp (alpha >= 2^-40
//    and alpha*nr*nc <= 0.5) the ramp makes every pixel distinct and the rule
//    is the integer key (v, k): max -> largest v then HIGHEST flat index,
//    min -> smallest v then LOWEST flat index.  Otherwise the float64 values
//    P[r,c] are recomputed bit-exactly and compared with first-occurrence ties;
//  * dedupe keeps the first (smallest-scale) feature per (row, col, polarity)
//    (detector.py:139-151) and the output is ordered (scale, window, polarity).
//    A scale L whose every window is a union of windows of a smaller scale L'
//    (L % L' == 0) can only contribute duplicates, so with dedupe it is not
//    evaluated at all; for the usual doubling scale sets only L_min remains.
#include <cub/cub.cuh>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "ps_common.cuh"

namespace ps {
namespace {

constexpr int kMaxScales = 16;

struct ScalePlan {
  int n;                    // evaluated scales (ascending)
  int L[kMaxScales];        // window side
  int wc[kMaxScales];       // windows per row
  int nwin[kMaxScales];     // windows per image
  int64_t raw_off[kMaxScales + 1];  // raw feature offset of scale i (2 per window)
};

struct KpOut {
  int32_t* row;
  int32_t* col;
  double* value;
  int32_t* scale;
  int8_t* pol;
  int32_t* window;
  int64_t cap;
};

// The ramped value of pixel (r, c) whose 8-bit sample v the caller already holds in its key: the
// same two operations as RampU8::at without the dependent pixel load (RGB8 needs the grey: at()).
template <class Img>
__device__ __forceinline__ double value_from_key(const Img& im, unsigned, int r, int c) { return im.at(r, c); }
template <>
__device__ __forceinline__ double value_from_key<RampU8>(const RampU8& im, unsigned v, int r, int c) {
  const double k = u32_to_f64((unsigned)(r * im.nc + c + 1));
  return __dadd_rn(u32_to_f64(v), __dmul_rn(k, im.alpha));
}

// ---- comparison helpers -----------------------------------------------------

struct BestF64 {
  double v;
  int32_t k;
};
// max: larger value wins, equal value -> lower flat index (first occurrence)
__device__ __forceinline__ bool better_max(double v, int32_t k, double bv, int32_t bk) {
  return v > bv || (v == bv && k < bk);
}
__device__ __forceinline__ bool better_min(double v, int32_t k, double bv, int32_t bk) {
  return v < bv || (v == bv && k < bk);
}

// ---- generic kernel: one warp per window -----------------------------------
// MODE 0: integer key (u8 value or RGB luma, valid ramp); MODE 1: float64
// compare on P[r,c].
template <int MODE, class Img>
__global__ void __launch_bounds__(256) window_extrema_warp(
    Img img, int64_t img_stride, int B, int L, int wc, int nwin, int32_t* __restrict__ tmax,
    int32_t* __restrict__ tmin, KpOut out, int32_t scale_tag) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int nr = img.nr, nc = img.nc;
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < (int64_t)B * nwin;
       g += warps) {
    const int b = (int)(g / nwin);
    const int w = (int)(g % nwin);
    Img im = img;
    im.p = img.p + (int64_t)b * img_stride * decltype(img)::kElem;
    const int r0 = (w / wc) * L, c0 = (w % wc) * L;
    const int h = min(L, nr - r0), wd = min(L, nc - c0);
    int32_t kmax, kmin;
    if constexpr (MODE == 0) {
      uint64_t best_hi = 0, best_lo = ~0ull;
      for (int r = 0; r < h; ++r) {
        const int64_t rowbase = (int64_t)(r0 + r) * nc;
        for (int c = lane; c < wd; c += 32) {
          const uint64_t v = im.key(r0 + r, c0 + c);
          const uint64_t key = (v << 32) | (uint64_t)(rowbase + c0 + c);
          best_hi = key > best_hi ? key : best_hi;
          best_lo = key < best_lo ? key : best_lo;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        uint64_t a = __shfl_xor_sync(0xffffffffu, best_hi, o);
        uint64_t c = __shfl_xor_sync(0xffffffffu, best_lo, o);
        best_hi = a > best_hi ? a : best_hi;
        best_lo = c < best_lo ? c : best_lo;
      }
      kmax = (int32_t)(best_hi & 0xffffffffu);
      kmin = (int32_t)(best_lo & 0xffffffffu);
    } else {
      double vh = 0, vl = 0;
      int32_t kh = INT32_MAX, kl = INT32_MAX;
      bool any = false;
      for (int r = 0; r < h; ++r) {
        for (int c = lane; c < wd; c += 32) {
          const double v = im.at(r0 + r, c0 + c);
          const int32_t k = (r0 + r) * nc + c0 + c;
          if (!any) {
            vh = vl = v;
            kh = kl = k;
            any = true;
          } else {
            if (better_max(v, k, vh, kh)) { vh = v; kh = k; }
            if (better_min(v, k, vl, kl)) { vl = v; kl = k; }
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, vh, o);
        int32_t k2 = __shfl_xor_sync(0xffffffffu, kh, o);
        double v3 = __shfl_xor_sync(0xffffffffu, vl, o);
        int32_t k3 = __shfl_xor_sync(0xffffffffu, kl, o);
        if (k2 != INT32_MAX && (kh == INT32_MAX || better_max(v2, k2, vh, kh))) { vh = v2; kh = k2; }
        if (k3 != INT32_MAX && (kl == INT32_MAX || better_min(v3, k3, vl, kl))) { vl = v3; kl = k3; }
      }
      kmax = kh;
      kmin = kl;
    }
    if (lane == 0) {
      if (tmax) {
        tmax[(int64_t)b * nwin + w] = kmax;
        tmin[(int64_t)b * nwin + w] = kmin;
      }
      if (out.row) {  // direct emission: slot 2w (max), 2w+1 (min)
        const int64_t s = (int64_t)b * out.cap + 2 * (int64_t)w;
        const int32_t ks[2] = {kmax, kmin};
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int rr = ks[q] / nc, cc = ks[q] % nc;
          out.row[s + q] = rr;
          out.col[s + q] = cc;
          out.value[s + q] = im.at(rr, cc);
          if (out.scale) out.scale[s + q] = scale_tag;
          if (out.pol) out.pol[s + q] = (int8_t)q;
          if (out.window) out.window[s + q] = w;
        }
      }
    }
  }
}

// ---- fast path: u8, L = 8, valid ramp, 16-byte aligned rows ---------------
// One thread owns two horizontally adjacent 8x8 windows (a 16-byte column
// strip over 8 rows, eight 16-byte loads; a warp reads 8 rows x 512 B).
// Keys are 16-bit (v << 8 | 8*lr + lc) packed two per register with PRMT and
// reduced with the 3-input packed-u16 max/min (VIMNMX3).
__device__ __forceinline__ void keys_of_word(uint32_t word, uint32_t idxbytes, uint32_t& k01,
                                             uint32_t& k23) {
  k01 = __byte_perm(word, idxbytes, 0x1504);  // [idx0, v0, idx1, v1]
  k23 = __byte_perm(word, idxbytes, 0x3726);  // [idx2, v2, idx3, v3]
}

__device__ __forceinline__ void emit_pair(const KpOut& out, int64_t slot, int32_t kmax, int32_t kmin,
                                          int nc, const RampU8& im, int32_t scale_tag, int w) {
  const int r0 = kmax / nc, c0 = kmax % nc, r1 = kmin / nc, c1 = kmin % nc;
  *reinterpret_cast<int2*>(out.row + slot) = make_int2(r0, r1);
  *reinterpret_cast<int2*>(out.col + slot) = make_int2(c0, c1);
  *reinterpret_cast<double2*>(out.value + slot) = make_double2(im.at(r0, c0), im.at(r1, c1));
  if (out.scale) { out.scale[slot] = scale_tag; out.scale[slot + 1] = scale_tag; }
  if (out.pol) { out.pol[slot] = 0; out.pol[slot + 1] = 1; }
  if (out.window) { out.window[slot] = w; out.window[slot + 1] = w; }
}

__global__ void __launch_bounds__(256) detect_u8_w8(RampU8 img, int64_t img_stride, int B, int wr_n,
                                                    int wc_n, int pairs_per_row, KpOut out,
                                                    int32_t* __restrict__ tmax, int32_t* __restrict__ tmin) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per_img = (int64_t)wr_n * pairs_per_row;
  if (t >= (int64_t)B * per_img) return;
  const int b = (int)(t / per_img);
  const int rem = (int)(t % per_img);
  const int wr = rem / pairs_per_row, q = rem % pairs_per_row;
  const int nr = img.nr, nc = img.nc;
  RampU8 im = img;
  im.p = img.p + (int64_t)b * img_stride * decltype(img)::kElem;
  const int r0 = wr * 8, cbase = q * 16;
  const int w0 = wr * wc_n + 2 * q;
  const bool second = (2 * q + 1) < wc_n;
  int32_t kmax[2], kmin[2];
  if (r0 + 8 <= nr && cbase + 16 <= nc) {
    uint32_t mx[2] = {0u, 0u}, mn[2] = {0xffffffffu, 0xffffffffu};
    const uint8_t* base = im.p + (int64_t)r0 * im.pitch + cbase;
    uint4 rows[8];
#pragma unroll
    for (int lr = 0; lr < 8; ++lr) rows[lr] = __ldg(reinterpret_cast<const uint4*>(base + lr * im.pitch));
#pragma unroll
    for (int lr = 0; lr < 8; ++lr) {
      const uint32_t ib = (uint32_t)(lr * 8) * 0x01010101u;
      uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
      keys_of_word(rows[lr].x, ib + 0x03020100u, a0, a1);
      keys_of_word(rows[lr].y, ib + 0x07060504u, a2, a3);
      keys_of_word(rows[lr].z, ib + 0x03020100u, b0, b1);
      keys_of_word(rows[lr].w, ib + 0x07060504u, b2, b3);
      mx[0] = __vimax3_u16x2(mx[0], __vimax3_u16x2(a0, a1, a2), a3);
      mn[0] = __vimin3_u16x2(mn[0], __vimin3_u16x2(a0, a1, a2), a3);
      mx[1] = __vimax3_u16x2(mx[1], __vimax3_u16x2(b0, b1, b2), b3);
      mn[1] = __vimin3_u16x2(mn[1], __vimin3_u16x2(b0, b1, b2), b3);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t hi = max(mx[h] & 0xffffu, mx[h] >> 16);
      const uint32_t lo = min(mn[h] & 0xffffu, mn[h] >> 16);
      const int cw = cbase + 8 * h;
      kmax[h] = (r0 + (int)((hi & 0xff) >> 3)) * nc + cw + (int)(hi & 7);
      kmin[h] = (r0 + (int)((lo & 0xff) >> 3)) * nc + cw + (int)(lo & 7);
    }
  } else {
    // edge strip: scalar keys over the clipped windows (same order)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t hi = 0, lo = 0xffffffffu;
      const int cw = cbase + 8 * h;
      for (int lr = 0; lr < 8 && r0 + lr < nr; ++lr)
        for (int lc = 0; lc < 8 && cw + lc < nc; ++lc) {
          const uint32_t key = ((uint32_t)im.p[(int64_t)(r0 + lr) * im.pitch + cw + lc] << 8) | (lr * 8 + lc);
          hi = max(hi, key);
          lo = min(lo, key);
        }
      kmax[h] = (r0 + (int)((hi & 0xff) >> 3)) * nc + cw + (int)(hi & 7);
      kmin[h] = (r0 + (int)((lo & 0xff) >> 3)) * nc + cw + (int)(lo & 7);
    }
  }
  const int64_t nwin = (int64_t)wr_n * wc_n;
  if (out.row) {
    emit_pair(out, (int64_t)b * out.cap + 2 * (int64_t)w0, kmax[0], kmin[0], nc, im, 8, w0);
    if (second) emit_pair(out, (int64_t)b * out.cap + 2 * (int64_t)(w0 + 1), kmax[1], kmin[1], nc, im, 8, w0 + 1);
  }
  if (tmax) {
    tmax[b * nwin + w0] = kmax[0];
    tmin[b * nwin + w0] = kmin[0];
    if (second) {
      tmax[b * nwin + w0 + 1] = kmax[1];
      tmin[b * nwin + w0 + 1] = kmin[1];
    }
  }
}

// ---- vectorised strip kernel: any window side (integer-key mode) ----------
// One CTA per (image, window row); thread t owns the 16-pixel column chunk
// [16t, 16t + 16) over the window row's rows (one 16-byte load per row for
// u8, three for RGB8).  Per pixel column it keeps the max and min of the key
// (v << 8 | r), r = row within the window: the largest v with the HIGHEST
// row and the smallest v with the LOWEST row -- the integer-key rule of
// detector.py:114-119 restricted to one column.  The column keys go to
// shared memory and one thread per window folds its columns left to right
// (max: >= so the highest column wins a tie, min: < so the lowest does),
// which completes the rule: highest / lowest flat index among equal values.
// Reads every image byte once (HBM-bound).
template <class Img>
struct StripKeys;

template <>
struct StripKeys<RampU8> {
  // accumulators: 16-bit keys (v << 8 | r), two per register (columns 2i, 2i+1),
  // reduced with the packed u16 max / min
  using K = uint32_t;
  using Raw = uint4;
  static constexpr int kBatch = 8;  // rows whose loads are in flight together
  static constexpr int kBatch16 = 8;  // the same for detect_strip16 (row pairs: fold2; single-buffered)
  static constexpr int kStage16 = 8;  // rows staged through shared memory besides (8 + 8 = C1 / C5's 16-row windows)
  static constexpr int kMinBlocks16 = 3;  // its resident 256-thread CTAs per SM
  static constexpr int kMaxThreads = 256;
  static constexpr int kAcc = 8;    // registers per accumulator set
  static constexpr int kMaxRows = 256;  // the row index must fit its 8 bits
  __device__ __forceinline__ static Raw load(const RampU8& im, int rr, int chunk) {
    return __ldg(reinterpret_cast<const uint4*>(im.p + (int64_t)rr * im.pitch) + chunk);
  }
  __device__ __forceinline__ static void init(uint32_t (&mx)[kAcc], uint32_t (&mn)[kAcc]) {
#pragma unroll
    for (int j = 0; j < kAcc; ++j) { mx[j] = 0u; mn[j] = 0xffffffffu; }
  }
  __device__ __forceinline__ static void fold(const Raw& q, uint32_t r, uint32_t (&mx)[kAcc], uint32_t (&mn)[kAcc]) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t k01 = __byte_perm(w[i], r, 0x1404u);  // [r, v0, r, v1]
      const uint32_t k23 = __byte_perm(w[i], r, 0x3424u);  // [r, v2, r, v3]
      mx[2 * i] = __vmaxu2(mx[2 * i], k01);
      mn[2 * i] = __vminu2(mn[2 * i], k01);
      mx[2 * i + 1] = __vmaxu2(mx[2 * i + 1], k23);
      mn[2 * i + 1] = __vminu2(mn[2 * i + 1], k23);
    }
  }
  // two rows at once: 3-input packed max / min
  __device__ __forceinline__ static void fold2(const Raw& q0, const Raw& q1, uint32_t r, uint32_t (&mx)[kAcc],
                                               uint32_t (&mn)[kAcc]) {
    const uint32_t w0[4] = {q0.x, q0.y, q0.z, q0.w}, w1[4] = {q1.x, q1.y, q1.z, q1.w};
    const uint32_t r1 = r + 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t a01 = __byte_perm(w0[i], r, 0x1404u), a23 = __byte_perm(w0[i], r, 0x3424u);
      const uint32_t b01 = __byte_perm(w1[i], r1, 0x1404u), b23 = __byte_perm(w1[i], r1, 0x3424u);
      mx[2 * i] = __vimax3_u16x2(mx[2 * i], a01, b01);
      mn[2 * i] = __vimin3_u16x2(mn[2 * i], a01, b01);
      mx[2 * i + 1] = __vimax3_u16x2(mx[2 * i + 1], a23, b23);
      mn[2 * i + 1] = __vimin3_u16x2(mn[2 * i + 1], a23, b23);
    }
  }
  __device__ __forceinline__ static K key(const uint32_t (&acc)[kAcc], int j) {  // column j: (v << 8 | r)
    return (acc[j >> 1] >> (16 * (j & 1))) & 0xffffu;
  }
};

template <>
struct StripKeys<RampRGB8> {
  // accumulators: 32-bit keys (k << 8 | r), k = 299R + 587G + 114B < 2^18
  using K = uint32_t;
  struct Raw {
    uint4 a, b, c;
  };
  static constexpr int kBatch = 4;
  static constexpr int kBatch16 = 4;  // detect_strip16: rows in flight per lane (single-buffered)
  static constexpr int kMinBlocks16 = 3;
  static constexpr int kMaxThreads = 256;
  static constexpr int kAcc = 16;
  static constexpr int kMaxRows = 256;  // the row index must fit its 8 bits
  __device__ __forceinline__ static void init(K (&mx)[kAcc], K (&mn)[kAcc]) {
#pragma unroll
    for (int j = 0; j < kAcc; ++j) { mx[j] = 0u; mn[j] = 0xffffffffu; }
  }
  __device__ __forceinline__ static K key(const K (&acc)[kAcc], int j) { return acc[j]; }  // (v << 8 | r)
  __device__ __forceinline__ static Raw load(const RampRGB8& im, int rr, int chunk) {
    const uint4* src = reinterpret_cast<const uint4*>(im.p + 3 * (int64_t)rr * im.pitch) + 3 * chunk;
    return Raw{__ldg(src), __ldg(src + 1), __ldg(src + 2)};
  }
  // detect_strip16: a lane reduces its whole chunk to ONE key per polarity, (k << 12 | r << 4 | j)
  // (k < 2^18, r < 2^8, j = column within the chunk): 2 accumulator registers instead of 32, which
  // is what lets a third CTA reside per SM.  PARTIAL: only the first `nvalid` columns exist.
  template <bool PARTIAL>
  __device__ __forceinline__ static void fold_one(const Raw& q, uint32_t r, int nvalid, K& mx, K& mn) {
    const uint32_t w[13] = {q.a.x, q.a.y, q.a.z, q.a.w, q.b.x, q.b.y, q.b.z, q.b.w, q.c.x, q.c.y, q.c.z, q.c.w, 0u};
    const uint32_t r4 = r << 4;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int o = 3 * j;
      const uint32_t px = __byte_perm(w[o >> 2], w[(o >> 2) + 1], (uint32_t)(o & 3) * 0x111u + 0x210u);
      const uint32_t hi = __dp4a(px, 0x00000201u, 0u);
      const uint32_t lo = __dp4a(px, 0x00724b2bu, 0u);
      const K key = (hi << 20) + (lo << 12) + (r4 + (uint32_t)j);
      if (!PARTIAL || j < nvalid) {
        mx = max(mx, key);
        mn = min(mn, key);
      }
    }
  }
  __device__ __forceinline__ static void fold(const Raw& q, uint32_t r, K (&mx)[kAcc], K (&mn)[kAcc]) {
    const uint32_t w[13] = {q.a.x, q.a.y, q.a.z, q.a.w, q.b.x, q.b.y, q.b.z, q.b.w, q.c.x, q.c.y, q.c.z, q.c.w, 0u};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int o = 3 * j;  // byte offset of pixel j's R
      // [R, G, B, x] of pixel j from the two words it spans
      const uint32_t px = __byte_perm(w[o >> 2], w[(o >> 2) + 1], (uint32_t)(o & 3) * 0x111u + 0x210u);
      // 299R + 587G + 114B = 256 (R + 2G) + (43R + 75G + 114B): two byte dot products
      const uint32_t hi = __dp4a(px, 0x00000201u, 0u);
      const uint32_t lo = __dp4a(px, 0x00724b2bu, 0u);
      const K key = (hi << 16) + (lo << 8) + r;  // (k << 8 | r)
      mx[j] = max(mx[j], key);
      mn[j] = min(mn[j], key);
    }
  }
};


// A task is (image, window row, segment of SW windows, at most 256 column
// chunks); thread t owns the segment's column chunk t over all the window
// row's rows.  Loads are software pipelined: the next kBatch rows are
// requested before the current ones are folded.
template <class Img>
__global__ void __launch_bounds__(StripKeys<Img>::kMaxThreads) detect_strip(
    Img img, int64_t img_stride, int B, int L, int wr_n, int wc, int nwin, int SW, int nseg,
    int32_t* __restrict__ tmax, int32_t* __restrict__ tmin, KpOut out, int32_t scale_tag) {
  using SK = StripKeys<Img>;
  using K = typename SK::K;
  using A = typename std::conditional<std::is_same<Img, RampU8>::value, uint32_t, K>::type;
  constexpr int NB = SK::kBatch;
  extern __shared__ unsigned char strip_smem[];
  const int nr = img.nr, nc = img.nc;
  K* cmax = reinterpret_cast<K*>(strip_smem);
  K* cmin = cmax + (size_t)SW * L;
  for (int64_t task = blockIdx.x; task < (int64_t)B * wr_n * nseg; task += gridDim.x) {
    const int seg = (int)(task % nseg);
    const int64_t bw = task / nseg;
    const int b = (int)(bw / wr_n), wr = (int)(bw % wr_n);
    Img im = img;
    im.p = img.p + (int64_t)b * img_stride * decltype(img)::kElem;
    const int r0 = wr * L, h = min(L, nr - r0);
    const int cs = seg * SW * L, ce = min(cs + SW * L, nc);  // cs is a multiple of 16 (SW is)
    const int chunks = (ce - cs + 15) >> 4, chunk0 = cs >> 4;
    __syncthreads();  // the previous task's folds are done with the column keys
    for (int t = threadIdx.x; t < chunks; t += blockDim.x) {
      A mx[SK::kAcc], mn[SK::kAcc];
      SK::init(mx, mn);
      typename SK::Raw cur[NB], nxt[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) cur[i] = SK::load(im, r0 + min(i, h - 1), chunk0 + t);
      for (int r = 0; r < h; r += NB) {
#pragma unroll
        for (int i = 0; i < NB; ++i) nxt[i] = SK::load(im, r0 + min(r + NB + i, h - 1), chunk0 + t);  // clamped
#pragma unroll
        for (int i = 0; i < NB; ++i)
          if (r + i < h) SK::fold(cur[i], (uint32_t)(r + i), mx, mn);
#pragma unroll
        for (int i = 0; i < NB; ++i) cur[i] = nxt[i];
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        cmax[16 * t + j] = SK::key(mx, j);
        cmin[16 * t + j] = SK::key(mn, j);
      }
    }
    __syncthreads();
    const int w0 = seg * SW, w1 = min(w0 + SW, wc);
    for (int wcol = w0 + (int)threadIdx.x; wcol < w1; wcol += blockDim.x) {
      const int c0 = wcol * L, c1 = min(c0 + L, nc);
      K bx = cmax[c0 - cs], bn = cmin[c0 - cs];
      int cx = c0, cn = c0;
      for (int c = c0 + 1; c < c1; ++c) {
        const K kx = cmax[c - cs], kn = cmin[c - cs];
        if (kx >= bx) { bx = kx; cx = c; }
        if (kn < bn) { bn = kn; cn = c; }
      }
      const int32_t kmax = (r0 + (int)(bx & 0xffu)) * nc + cx;
      const int32_t kmin = (r0 + (int)(bn & 0xffu)) * nc + cn;
      const int w = wr * wc + wcol;
      if (tmax) {
        tmax[(int64_t)b * nwin + w] = kmax;
        tmin[(int64_t)b * nwin + w] = kmin;
      }
      if (out.row) {  // direct emission: slot 2w (max), 2w+1 (min)
        const int64_t sl = (int64_t)b * out.cap + 2 * (int64_t)w;
        const int32_t ks[2] = {kmax, kmin};
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int rr = ks[q] / nc, cc = ks[q] % nc;
          out.row[sl + q] = rr;
          out.col[sl + q] = cc;
          out.value[sl + q] = im.at(rr, cc);
          if (out.scale) out.scale[sl + q] = scale_tag;
          if (out.pol) out.pol[sl + q] = (int8_t)q;
          if (out.window) out.window[sl + q] = w;
        }
      }
    }
  }
}

// Any window side up to kStripWMaxL, without block barriers: a task is
// (image, window row, run of W windows) and belongs to ONE warp -- lane l owns
// the 16-pixel chunk chunk0 + l of the run's columns (W * L + misalignment
// <= 32 chunks) over the window row's rows, the column keys go to the warp's
// own shared-memory slice, and after a __syncwarp the run's windows are folded
// by one lane each exactly as in detect_strip.  Warps are independent, so the
// loads of one overlap the folds of the others (detect_strip's CTAs idle at
// two barriers per task, and a window row split into 256-chunk segments
// leaves a ragged last segment); the chunks shared by neighbouring runs (at
// most one per side) are read twice, from L2.
constexpr int kStripWMaxL = 160;
constexpr int kStripWCols = 512;  // column keys per warp and polarity
template <class Img>
struct StripW;
// u8: a lane keeps kBatch rows in flight in registers AND kStage rows in flight into its own
// shared-memory slots (cp.async, 16 bytes per row): bytes in flight are what bounds the kernel, and
// registers alone hold too few of them (8 rows x 1024 threads = 131 KB per SM -> 0.46 of HBM).
template <>
struct StripW<RampU8> {
#ifndef PS_STRIPW_STAGE
#define PS_STRIPW_STAGE 10  // 8 + 10 rows: two rounds cover C4's 36-row windows exactly (A/B 8..18: 16.7 us vs 18.7)
#endif
#ifndef PS_STRIPW_WARPS
#define PS_STRIPW_WARPS 8
#endif
#ifndef PS_STRIPW_BLOCKS
#define PS_STRIPW_BLOCKS 3
#endif
  static constexpr int kBatch = 8, kStage = PS_STRIPW_STAGE, kMinBlocks = PS_STRIPW_BLOCKS, kWarps = PS_STRIPW_WARPS;
  using KS = uint16_t;  // stored column key (v << 8 | r)
};
template <>
struct StripW<RampRGB8> {
  static constexpr int kBatch = 2, kStage = 0, kMinBlocks = 3, kWarps = 8;
  using KS = uint32_t;
};
template <class Img>
constexpr size_t stripw_smem() {
  // per warp: the staging slots, reused for the run's column keys once its rows are folded
  return StripW<Img>::kWarps * std::max<size_t>(2 * kStripWCols * sizeof(typename StripW<Img>::KS), (size_t)StripW<Img>::kStage * 512);
}
__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_smem), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
inline int stripw_windows(int L) { return (kStripWCols - 30) / L; }  // 15 + W L + 15 <= 512

template <class Img>
__global__ void __launch_bounds__(32 * StripW<Img>::kWarps, StripW<Img>::kMinBlocks) detect_stripw(
    Img img, int64_t img_stride, int B, int L, int wr_n, int wc, int nwin, int W, int nrun,
    int32_t* __restrict__ tmax, int32_t* __restrict__ tmin, KpOut out, int32_t scale_tag) {
  using SK = StripKeys<Img>;
  using K = typename SK::K;
  using A = typename std::conditional<std::is_same<Img, RampU8>::value, uint32_t, K>::type;
  using KS = typename StripW<Img>::KS;
  constexpr int NB = StripW<Img>::kBatch, NS = StripW<Img>::kStage;
  extern __shared__ __align__(16) unsigned char stripw_raw[];
  const int nr = img.nr, nc = img.nc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int WPB = StripW<Img>::kWarps;
  unsigned char* warp_area = stripw_raw + (size_t)warp * (stripw_smem<Img>() / WPB);
  KS* cmax = reinterpret_cast<KS*>(warp_area);  // the column keys alias the staging slots
  KS* cmin = cmax + kStripWCols;
  // this lane's staging slots: row i of a staged batch at stage + 512 i (conflict-free 16-byte reads)
  unsigned char* stage = warp_area + lane * 16;
  const int64_t ntask = (int64_t)B * wr_n * nrun, wstride = (int64_t)gridDim.x * WPB;
  for (int64_t task = (int64_t)blockIdx.x * WPB + warp; task < ntask; task += wstride) {
    const int run = (int)(task % nrun);
    const int64_t bw = task / nrun;
    const int b = (int)(bw / wr_n), wr = (int)(bw % wr_n);
    Img im = img;
    im.p = img.p + (int64_t)b * img_stride * decltype(img)::kElem;
    const int r0 = wr * L, h = min(L, nr - r0);
    const int w0 = run * W, w1 = min(w0 + W, wc);
    const int cb = w0 * L, ce = min(w1 * L, nc);
    const int chunk0 = cb >> 4, nch = ((ce + 15) >> 4) - chunk0;  // <= 32
    A mx[SK::kAcc], mn[SK::kAcc];
    SK::init(mx, mn);
    __syncwarp();  // the previous run's window folds are done with the keys (they alias the staging slots)
    if constexpr (NS > 0) {
      if (lane < nch) {
        // rows [r, r + NB) travel through registers, rows [r + NB, r + NB + NS) through the lane's
        // staging slots, alternately: both kinds are in flight while the other is folded
        const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
        const unsigned char* colp = reinterpret_cast<const unsigned char*>(im.p) + 16 * (int64_t)(chunk0 + lane);
        auto stage_rows = [&](int ra) {  // rows ra .. ra + NS - 1 (those below h) -> the slots
#pragma unroll
          for (int i = 0; i < NS; ++i)
            if (ra + i < h) cp_async16(stage_s + 512u * i, colp + (int64_t)(r0 + ra + i) * im.pitch);
          cp_async_commit();
        };
        typename SK::Raw cur[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) cur[i] = SK::load(im, r0 + min(i, h - 1), chunk0 + lane);  // clamped
        stage_rows(NB);
        for (int r = 0; r < h; r += NB + NS) {
          if (r + NB <= h) {
#pragma unroll
            for (int i = 0; i < NB; i += 2) SK::fold2(cur[i], cur[i + 1], (uint32_t)(r + i), mx, mn);
          } else {
#pragma unroll
            for (int i = 0; i < NB; ++i)
              if (r + i < h) SK::fold(cur[i], (uint32_t)(r + i), mx, mn);
          }
          if (r + NB + NS < h) {
#pragma unroll
            for (int i = 0; i < NB; ++i) cur[i] = SK::load(im, r0 + min(r + NB + NS + i, h - 1), chunk0 + lane);
          }
          cp_async_wait_all();
          const int rs = r + NB;
          if (rs + NS <= h) {
#pragma unroll
            for (int i = 0; i < NS; i += 2)
              SK::fold2(*reinterpret_cast<const uint4*>(stage + 512 * i),
                        *reinterpret_cast<const uint4*>(stage + 512 * (i + 1)), (uint32_t)(rs + i), mx, mn);
          } else {
#pragma unroll
            for (int i = 0; i < NS; ++i)
              if (rs + i < h) SK::fold(*reinterpret_cast<const uint4*>(stage + 512 * i), (uint32_t)(rs + i), mx, mn);
          }
          if (r + 2 * NB + NS < h) stage_rows(r + 2 * NB + NS);  // after the slots' last reads were consumed
        }
      }
    } else if (lane < nch) {
      typename SK::Raw cur[NB];
      for (int r = 0; r < h; r += NB) {
        // one batch of rows in flight per warp (no second buffer): the registers saved double the
        // resident warps, which is what keeps enough bytes in flight per SM
#pragma unroll
        for (int i = 0; i < NB; ++i) cur[i] = SK::load(im, r0 + min(r + i, h - 1), chunk0 + lane);  // clamped
        if constexpr (std::is_same<Img, RampU8>::value) {
          if (r + NB <= h) {
#pragma unroll
            for (int i = 0; i < NB; i += 2) SK::fold2(cur[i], cur[i + 1], (uint32_t)(r + i), mx, mn);
          } else {
#pragma unroll
            for (int i = 0; i < NB; ++i)
              if (r + i < h) SK::fold(cur[i], (uint32_t)(r + i), mx, mn);
          }
        } else {
#pragma unroll
          for (int i = 0; i < NB; ++i)
            if (r + i < h) SK::fold(cur[i], (uint32_t)(r + i), mx, mn);
        }
      }
    }
    __syncwarp();  // every lane has folded its staged rows
    if (lane < nch) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        cmax[16 * lane + j] = (KS)SK::key(mx, j);
        cmin[16 * lane + j] = (KS)SK::key(mn, j);
      }
    }
    __syncwarp();
    const int cs = chunk0 << 4;
    for (int wcol = w0 + lane; wcol < w1; wcol += 32) {
      const int c0 = wcol * L, c1 = min(c0 + L, nc);
      K bx = cmax[c0 - cs], bn = cmin[c0 - cs];
      int cx = c0, cn = c0;
      for (int c = c0 + 1; c < c1; ++c) {
        const K kx = cmax[c - cs], kn = cmin[c - cs];
        if (kx >= bx) { bx = kx; cx = c; }
        if (kn < bn) { bn = kn; cn = c; }
      }
      const int32_t kmax = (r0 + (int)(bx & 0xffu)) * nc + cx;
      const int32_t kmin = (r0 + (int)(bn & 0xffu)) * nc + cn;
      const int w = wr * wc + wcol;
      if (tmax) {
        tmax[(int64_t)b * nwin + w] = kmax;
        tmin[(int64_t)b * nwin + w] = kmin;
      }
      if (out.row) {  // direct emission: slot 2w (max), 2w+1 (min)
        const int64_t sl = (int64_t)b * out.cap + 2 * (int64_t)w;
        const int32_t ks[2] = {kmax, kmin};
        const unsigned vs[2] = {(unsigned)(bx >> 8), (unsigned)(bn >> 8)};
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int rr = ks[q] / nc, cc = ks[q] % nc;
          out.row[sl + q] = rr;
          out.col[sl + q] = cc;
          out.value[sl + q] = value_from_key(im, vs[q], rr, cc);
          if (out.scale) out.scale[sl + q] = scale_tag;
          if (out.pol) out.pol[sl + q] = (int8_t)q;
          if (out.window) out.window[sl + q] = w;
        }
      }
    }
  }
}

// Window sides that are multiples of 16 (every scale of C1, C3 and C5): a
// window is G = L / 16 whole 16-pixel chunks and its rows are split into R
// groups, so G * R lanes (a power of two <= 32) own one window and each lane
// folds one chunk over L / R rows (8 when L <= 64: all loads in flight at
// once).  Lane = (row group, window of the warp, chunk), chunk fastest, so a
// row group's lanes read contiguous columns.  Each lane reduces its 16
// columns to one (v, r, c) key per polarity and the window's lanes combine
// with xor shuffles -- no shared memory, no block barrier.  Max: largest
// (v, r, c), i.e. the highest flat index among equal values; min: smallest
// (v, r, c), the lowest.
template <class Img>
__global__ void __launch_bounds__(256, StripKeys<Img>::kMinBlocks16) detect_strip16(
    Img img, int64_t img_stride, int B, int L, int G, int R, int wr_n, int wc, int nwin, int32_t* __restrict__ tmax,
    int32_t* __restrict__ tmin, KpOut out, int32_t scale_tag) {
  using SK = StripKeys<Img>;
  using A = typename std::conditional<std::is_same<Img, RampU8>::value, uint32_t, typename SK::K>::type;
  constexpr int NB = SK::kBatch16;
  const int nr = img.nr, nc = img.nc;
  const int lane = threadIdx.x & 31;
  const int W = 32 / (G * R);                 // windows per warp
  const int wblocks = (wc + W - 1) / W;       // warps per window row
  const int c = lane % G, wl = (lane / G) % W, rg = lane / (G * W);
  const int rpt = L / R;                      // rows per lane
  const int64_t nwarps = (int64_t)B * wr_n * wblocks;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gw < nwarps; gw += wstride) {
    const int wb = (int)(gw % wblocks);
    const int64_t bw = gw / wblocks;
    const int b = (int)(bw / wr_n), wr = (int)(bw % wr_n);
    const int wcol = wb * W + wl;
    const int chunk = wcol * G + c;
    Img im = img;
    im.p = img.p + (int64_t)b * img_stride * decltype(img)::kElem;
    const int r0 = wr * L, h = min(L, nr - r0);
    const int ra = rg * rpt, rb = min(ra + rpt, h);
    const bool has = wcol < wc && 16 * chunk < nc && ra < rb;
    const int cw = 16 * c;  // column offset of the chunk within its window
    unsigned long long bx = 0ull, bn = ~0ull;
    // one batch of rows in flight per lane and no second buffer: the registers saved let another
    // CTA reside per SM, which keeps more bytes in flight than two batches would
    if constexpr (std::is_same<Img, RampU8>::value) {
      A mx[SK::kAcc], mn[SK::kAcc];
      SK::init(mx, mn);
      // as detect_stripw: NB rows in flight in registers and NS more into the lane's own staging
      // slots (cp.async), alternately
      constexpr int NS = SK::kStage16;
      __shared__ __align__(16) unsigned char stage16[8][NS * 512];
      if (has) {
        unsigned char* stage = stage16[threadIdx.x >> 5] + lane * 16;
        const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
        const unsigned char* colp = reinterpret_cast<const unsigned char*>(im.p) + 16 * (int64_t)chunk;
        auto stage_rows = [&](int r) {  // rows r .. r + NS - 1 (those below rb) -> the slots
#pragma unroll
          for (int i = 0; i < NS; ++i)
            if (r + i < rb) cp_async16(stage_s + 512u * i, colp + (int64_t)(r0 + r + i) * im.pitch);
          cp_async_commit();
        };
        typename SK::Raw cur[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) cur[i] = SK::load(im, r0 + min(ra + i, rb - 1), chunk);  // clamped
        stage_rows(ra + NB);
        for (int r = ra; r < rb; r += NB + NS) {
          if (r + NB <= rb) {
#pragma unroll
            for (int i = 0; i < NB; i += 2) SK::fold2(cur[i], cur[i + 1], (uint32_t)(r + i), mx, mn);
          } else {
#pragma unroll
            for (int i = 0; i < NB; ++i)
              if (r + i < rb) SK::fold(cur[i], (uint32_t)(r + i), mx, mn);
          }
          if (r + NB + NS < rb) {
#pragma unroll
            for (int i = 0; i < NB; ++i) cur[i] = SK::load(im, r0 + min(r + NB + NS + i, rb - 1), chunk);
          }
          cp_async_wait_all();
          const int rs = r + NB;
          if (rs + NS <= rb) {
#pragma unroll
            for (int i = 0; i < NS; i += 2)
              SK::fold2(*reinterpret_cast<const uint4*>(stage + 512 * i),
                        *reinterpret_cast<const uint4*>(stage + 512 * (i + 1)), (uint32_t)(rs + i), mx, mn);
          } else {
#pragma unroll
            for (int i = 0; i < NS; ++i)
              if (rs + i < rb) SK::fold(*reinterpret_cast<const uint4*>(stage + 512 * i), (uint32_t)(rs + i), mx, mn);
          }
          if (r + 2 * NB + NS < rb) stage_rows(r + 2 * NB + NS);  // after the slots' last reads were consumed
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (16 * chunk + j >= nc) continue;
          const unsigned long long col = (unsigned long long)(cw + j);
          const unsigned long long fx = ((unsigned long long)SK::key(mx, j) << 8) | col;  // (v, r, c)
          const unsigned long long fn = ((unsigned long long)SK::key(mn, j) << 8) | col;
          bx = fx > bx ? fx : bx;
          bn = fn < bn ? fn : bn;
        }
      }
    } else {  // RGB8: the chunk's single (k, r, j) key per polarity
      typename SK::K kx = 0u, kn = 0xffffffffu;
      if (has) {
        const int nvalid = min(16, nc - 16 * chunk);
        typename SK::Raw cur[NB];
        for (int r = ra; r < rb; r += NB) {
#pragma unroll
          for (int i = 0; i < NB; ++i) cur[i] = SK::load(im, r0 + min(r + i, rb - 1), chunk);  // clamped
          if (nvalid == 16) {
#pragma unroll
            for (int i = 0; i < NB; ++i)
              if (r + i < rb) SK::template fold_one<false>(cur[i], (uint32_t)(r + i), 16, kx, kn);
          } else {
#pragma unroll
            for (int i = 0; i < NB; ++i)
              if (r + i < rb) SK::template fold_one<true>(cur[i], (uint32_t)(r + i), nvalid, kx, kn);
          }
        }
        bx = ((unsigned long long)(kx >> 4) << 8) | (unsigned long long)(cw + (int)(kx & 15u));  // (v, r, c)
        bn = ((unsigned long long)(kn >> 4) << 8) | (unsigned long long)(cw + (int)(kn & 15u));
      }
    }
    for (int o = 1; o < G; o <<= 1) {  // chunks of the window
      const unsigned long long ox = __shfl_xor_sync(0xffffffffu, bx, o);
      const unsigned long long on = __shfl_xor_sync(0xffffffffu, bn, o);
      bx = ox > bx ? ox : bx;
      bn = on < bn ? on : bn;
    }
    for (int o = G * W; o < 32; o <<= 1) {  // row groups of the window
      const unsigned long long ox = __shfl_xor_sync(0xffffffffu, bx, o);
      const unsigned long long on = __shfl_xor_sync(0xffffffffu, bn, o);
      bx = ox > bx ? ox : bx;
      bn = on < bn ? on : bn;
    }
    if (wcol < wc && c == 0 && rg == 0) {
      const int c0 = wcol * L;
      const int32_t kmax = (r0 + (int)((bx >> 8) & 0xffull)) * nc + c0 + (int)(bx & 0xffull);
      const int32_t kmin = (r0 + (int)((bn >> 8) & 0xffull)) * nc + c0 + (int)(bn & 0xffull);
      const int w = wr * wc + wcol;
      if (tmax) {
        tmax[(int64_t)b * nwin + w] = kmax;
        tmin[(int64_t)b * nwin + w] = kmin;
      }
      if (out.row) {  // direct emission: slot 2w (max), 2w+1 (min)
        const int64_t sl = (int64_t)b * out.cap + 2 * (int64_t)w;
        const int32_t ks[2] = {kmax, kmin};
        const unsigned vs[2] = {(unsigned)(bx >> 16) & 0xffu, (unsigned)(bn >> 16) & 0xffu};  // u8: (v, r, c) keys
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int rr = ks[q] / nc, cc = ks[q] % nc;
          out.row[sl + q] = rr;
          out.col[sl + q] = cc;
          out.value[sl + q] = value_from_key(im, vs[q], rr, cc);
          if (out.scale) out.scale[sl + q] = scale_tag;
          if (out.pol) out.pol[sl + q] = (int8_t)q;
          if (out.window) out.window[sl + q] = w;
        }
      }
    }
  }
}

// windows per task: at most 256 chunks of 16 columns, a multiple of 16 windows
// (16-byte aligned chunk starts); a window row narrower than that is one task
int strip_windows(int L, int wc) {
  const int sw = std::max(16, (4096 / L) / 16 * 16);
  return std::min(sw, (wc + 15) / 16 * 16);
}

template <class Img>
int launch_strip(const Img& img, const ps_image_batch* ib, int B, int L, int wc, int nwin, const KpOut& ko,
                 int32_t* tmax, int32_t* tmin, cudaStream_t st) {
  using K = typename StripKeys<Img>::K;
  if (L % 16 == 0 && L <= 256 && (L & (L - 1)) == 0) {  // whole-chunk windows (G a power of two): the shuffle kernel
    const int wr_n = (img.nr + L - 1) / L;
    const int G = L / 16, R = std::max(1, std::min(L / 16, 32 / G));  // G * R lanes per window, 16 rows each up to L = 64
    const int W = 32 / (G * R);
    const int64_t warps = (int64_t)B * wr_n * ((wc + W - 1) / W);
    const int grid = (int)std::min<int64_t>((warps + 7) / 8, 148 * 24);
    detect_strip16<Img><<<grid, 256, 0, st>>>(img, ib->image_stride, B, L, G, R, wr_n, wc, nwin, tmax, tmin, ko,
                                              L);
    PS_LAUNCHED("detect_strip16");
    return PS_OK;
  }
  const int wr_n = (img.nr + L - 1) / L;
  if (L <= kStripWMaxL) {  // warp-owned runs of windows: no block barriers
    const int nrun = (wc + stripw_windows(L) - 1) / stripw_windows(L);
    const int W = (wc + nrun - 1) / nrun;  // balanced runs
    const int64_t tasks = (int64_t)B * wr_n * nrun;
    constexpr int WPB = StripW<Img>::kWarps;
    const int grid = (int)std::min<int64_t>((tasks + WPB - 1) / WPB, 148 * StripW<Img>::kMinBlocks * 4);
    cudaFuncSetAttribute(detect_stripw<Img>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stripw_smem<Img>());
    detect_stripw<Img><<<grid, 32 * WPB, stripw_smem<Img>(), st>>>(img, ib->image_stride, B, L, wr_n, wc, nwin, W, nrun,
                                                              tmax, tmin, ko, L);
    PS_LAUNCHED("detect_stripw");
    return PS_OK;
  }
  const int SW = strip_windows(L, wc), nseg = (wc + SW - 1) / SW;
  const size_t smem = 2 * (size_t)SW * L * sizeof(K);
  const int chunks = std::min((SW * L + 15) / 16, (img.nc + 15) / 16);
  const int threads = std::min(StripKeys<Img>::kMaxThreads, (chunks + 31) / 32 * 32);
  cudaFuncSetAttribute(detect_strip<Img>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t tasks = (int64_t)B * wr_n * nseg;
  const int grid = (int)std::min<int64_t>(tasks, 148 * 32);
  detect_strip<Img><<<grid, threads, smem, st>>>(img, ib->image_stride, B, L, wr_n, wc, nwin, SW, nseg, tmax, tmin,
                                                 ko, L);
  PS_LAUNCHED("detect_strip");
  return PS_OK;
}

// strip kernel preconditions: 16-byte aligned rows and images, rows of at
// most 2^16 (row index in the key), column keys within the shared memory
bool strip_ok(const ps_image_batch* ib, int L, int key_bytes, int max_rows) {
  const int64_t bpp = ib->pixel_type == PS_PIXELS_RGB8 ? 3 : 1;
  const bool aligned = ((uintptr_t)ib->data) % 16 == 0 && (ib->row_pitch * bpp) % 16 == 0 &&
                       (ib->image_stride * bpp) % 16 == 0;
  const int wc = (ib->nc + L - 1) / L;
  const size_t smem = 2 * (size_t)strip_windows(L, wc) * L * key_bytes;
  return aligned && L <= max_rows && smem <= 200 * 1024;
}

// ---- general emission (several scales and/or dedupe) ------------------------
struct Tables {
  int32_t* tmax[kMaxScales];
  int32_t* tmin[kMaxScales];
};

__global__ void dedupe_flags(ScalePlan sp, Tables tb, int B, int nc, int dedupe, int32_t* __restrict__ flags) {
  const int64_t raw = sp.raw_off[sp.n];
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < (int64_t)B * raw;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(g / raw);
    const int64_t f = g % raw;
    int si = 0;
    while (f >= sp.raw_off[si + 1]) ++si;
    const int64_t loc = f - sp.raw_off[si];
    const int w = (int)(loc >> 1), pol = (int)(loc & 1);
    int keep = 1;
    if (dedupe) {
      const int32_t k = pol ? tb.tmin[si][(int64_t)b * sp.nwin[si] + w] : tb.tmax[si][(int64_t)b * sp.nwin[si] + w];
      const int r = k / nc, c = k % nc;
      for (int sj = 0; sj < si; ++sj) {
        const int wj = (r / sp.L[sj]) * sp.wc[sj] + c / sp.L[sj];
        const int32_t kj = pol ? tb.tmin[sj][(int64_t)b * sp.nwin[sj] + wj] : tb.tmax[sj][(int64_t)b * sp.nwin[sj] + wj];
        if (kj == k) { keep = 0; break; }
      }
    }
    flags[g] = keep;
  }
}

template <class Img>
__global__ void scatter_kept(ScalePlan sp, Tables tb, Img img, int64_t img_stride, int B,
                             const int32_t* __restrict__ flags, const int32_t* __restrict__ pos, KpOut out,
                             int32_t* __restrict__ counts) {
  const int64_t raw = sp.raw_off[sp.n];
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < (int64_t)B * raw;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(g / raw);
    const int64_t f = g % raw;
    const int64_t base = pos[(int64_t)b * raw];
    if (f == raw - 1) counts[b] = (int32_t)(pos[g] + flags[g] - base);
    if (!flags[g]) continue;
    int si = 0;
    while (f >= sp.raw_off[si + 1]) ++si;
    const int64_t loc = f - sp.raw_off[si];
    const int w = (int)(loc >> 1), pol = (int)(loc & 1);
    const int32_t k = pol ? tb.tmin[si][(int64_t)b * sp.nwin[si] + w] : tb.tmax[si][(int64_t)b * sp.nwin[si] + w];
    Img im = img;
    im.p = img.p + (int64_t)b * img_stride * decltype(img)::kElem;
    const int r = k / img.nc, c = k % img.nc;
    const int64_t s = (int64_t)b * out.cap + (pos[g] - base);
    out.row[s] = r;
    out.col[s] = c;
    out.value[s] = im.at(r, c);
    if (out.scale) out.scale[s] = sp.L[si];
    if (out.pol) out.pol[s] = (int8_t)pol;
    if (out.window) out.window[s] = w;
  }
}

__global__ void fill_counts(int32_t* counts, int B, int32_t v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B) counts[i] = v;
}

// ---- host planning -----------------------------------------------------------

int validate_scales(int nr, int nc, const int32_t* s, int n) {
  // ScaleSet.__post_init__ / validate_for (detector.py:33-68)
  PS_REQUIRE(n >= 1, PS_ERR_CONFIG, "scale set must contain at least one size");
  PS_REQUIRE(n <= kMaxScales, PS_ERR_ARGUMENT, "at most %d scales supported", kMaxScales);
  for (int i = 0; i < n; ++i) PS_REQUIRE(s[i] >= 8, PS_ERR_CONFIG, "window sizes must be integers >= 8");
  for (int i = 1; i < n; ++i) PS_REQUIRE(s[i] > s[i - 1], PS_ERR_CONFIG, "window sizes must be strictly increasing");
  PS_REQUIRE(s[n - 1] <= std::min(nr, nc), PS_ERR_CONFIG, "largest window %d exceeds image side %d", s[n - 1],
             std::min(nr, nc));
  PS_REQUIRE((int64_t)nr * nc < (int64_t)INT32_MAX, PS_ERR_ARGUMENT, "image too large (nr*nc >= 2^31)");
  return PS_OK;
}

ScalePlan make_plan(int nr, int nc, const int32_t* s, int n, int dedupe) {
  ScalePlan sp{};
  sp.n = 0;
  for (int i = 0; i < n; ++i) {
    bool shadowed = false;
    if (dedupe)
      for (int j = 0; j < i; ++j)
        if (s[i] % s[j] == 0) shadowed = true;
    if (shadowed) continue;
    const int L = s[i];
    sp.L[sp.n] = L;
    sp.wc[sp.n] = (nc + L - 1) / L;
    sp.nwin[sp.n] = ((nr + L - 1) / L) * sp.wc[sp.n];
    sp.n++;
  }
  sp.raw_off[0] = 0;
  for (int i = 0; i < sp.n; ++i) sp.raw_off[i + 1] = sp.raw_off[i] + 2 * (int64_t)sp.nwin[i];
  return sp;
}

// The ramp must separate equal keys (alpha >= 2^-40, far above the grey's
// rounding noise) and stay below half the smallest grey step: 1 for u8,
// 0.001 (integer luma / 1000) for RGB8.
bool key_rule_valid(int nr, int nc, double alpha, double step = 1.0) {
  return alpha >= 9.094947017729282e-13 /* 2^-40 */ && alpha * (double)nr * (double)nc <= 0.5 * step;
}

size_t scan_temp_bytes(int64_t n) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return t;
}

size_t workspace_need(int B, const ScalePlan& sp, bool direct) {
  if (direct) return 0;
  Arena a{nullptr, 0, 0};
  for (int i = 0; i < sp.n; ++i) {
    a.take<int32_t>((size_t)B * sp.nwin[i]);
    a.take<int32_t>((size_t)B * sp.nwin[i]);
  }
  const int64_t raw = (int64_t)B * sp.raw_off[sp.n];
  a.take<int32_t>(raw);
  a.take<int32_t>(raw);
  a.take<char>(scan_temp_bytes(raw));
  return a.used + 256;
}

int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g > 148 * 64) g = 148 * 64;
  return (int)std::max<int64_t>(g, 1);
}

template <class Img>
int launch_key(const Img&, const ps_image_batch*, int, int, int, int, bool, const KpOut&, int32_t*, int32_t*,
               cudaStream_t) {
  set_error("integer-key detection requires 8-bit pixels");
  return PS_ERR_ARGUMENT;
}

// RGB8 with a valid ramp: integer luma key; the vectorised strip kernel when
// the rows are 16-byte aligned, else the generic warp-per-window kernel.
int launch_key(const RampRGB8& img, const ps_image_batch* ib, int B, int L, int wc, int nwin, bool,
               const KpOut& ko, int32_t* tmax, int32_t* tmin, cudaStream_t st) {
  if (strip_ok(ib, L, 4, StripKeys<RampRGB8>::kMaxRows)) return launch_strip(img, ib, B, L, wc, nwin, ko, tmax, tmin, st);
  window_extrema_warp<0><<<grid_for((int64_t)B * nwin, 8), 256, 0, st>>>(img, ib->image_stride, B, L, wc, nwin,
                                                                           tmax, tmin, ko, L);
  PS_LAUNCHED("window_extrema_warp<rgb key>");
  return PS_OK;
}

// u8 pixels with a valid ramp: integer-key kernels (L == 8 vectorised path).
int launch_key(const RampU8& img, const ps_image_batch* ib, int B, int L, int wc, int nwin, bool aligned,
               const KpOut& ko, int32_t* tmax, int32_t* tmin, cudaStream_t st) {
  if (L == 8 && aligned) {
    const int wr_n = (img.nr + 7) / 8, wc_n = (img.nc + 7) / 8, ppr = (wc_n + 1) / 2;
    const int64_t th = (int64_t)B * wr_n * ppr;
    detect_u8_w8<<<(unsigned)((th + 255) / 256), 256, 0, st>>>(img, ib->image_stride, B, wr_n, wc_n, ppr, ko, tmax,
                                                                tmin);
    PS_LAUNCHED("detect_u8_w8");
  } else if (strip_ok(ib, L, 4, StripKeys<RampU8>::kMaxRows)) {
    return launch_strip(img, ib, B, L, wc, nwin, ko, tmax, tmin, st);
  } else {
    window_extrema_warp<0><<<grid_for((int64_t)B * nwin, 8), 256, 0, st>>>(img, ib->image_stride, B, L, wc, nwin,
                                                                             tmax, tmin, ko, L);
    PS_LAUNCHED("window_extrema_warp<key>");
  }
  return PS_OK;
}

template <class Img>
int run_detect(const ps_image_batch* ib, Img img, bool u8, const int32_t* s, int n, int dedupe, ps_keypoints* out,
               void* ws, size_t ws_bytes, cudaStream_t st) {
  const int B = ib->batch, nr = ib->nr, nc = ib->nc;
  ScalePlan sp = make_plan(nr, nc, s, n, dedupe);
  const bool rgb = ib->pixel_type == PS_PIXELS_RGB8;
  const bool keymode = (u8 || rgb) && key_rule_valid(nr, nc, ib->alpha, rgb ? 0.001 : 1.0);
  const bool direct = sp.n == 1;  // one evaluated scale: no cross-scale dedupe needed
  PS_REQUIRE(out->cap >= sp.raw_off[sp.n], PS_ERR_CAPACITY, "keypoint capacity %lld < %lld",
             (long long)out->cap, (long long)sp.raw_off[sp.n]);
  KpOut ko{out->row, out->col, out->value, out->scale, out->polarity, out->window, out->cap};
  if (direct) {
    const int L = sp.L[0];
    const bool aligned = (((uintptr_t)ib->data) % 16 == 0) && ib->row_pitch % 16 == 0 && ib->image_stride % 16 == 0;
    if (keymode) {
      int rc = launch_key(img, ib, B, L, sp.wc[0], sp.nwin[0], aligned, ko, nullptr, nullptr, st);
      if (rc) return rc;
    } else {
      window_extrema_warp<1><<<grid_for((int64_t)B * sp.nwin[0], 8), 256, 0, st>>>(
          img, ib->image_stride, B, L, sp.wc[0], sp.nwin[0], nullptr, nullptr, ko, L);
      PS_LAUNCHED("window_extrema_warp<f64>");
    }
    fill_counts<<<(B + 255) / 256, 256, 0, st>>>(out->count, B, (int32_t)sp.raw_off[1]);
    PS_LAUNCHED("fill_counts");
    return PS_OK;
  }
  const size_t need = workspace_need(B, sp, false);
  PS_REQUIRE(ws != nullptr && ws_bytes >= need, PS_ERR_ARGUMENT, "detect workspace %zu < %zu", ws_bytes, need);
  Arena a{(char*)ws, ws_bytes, 0};
  Tables tb{};
  for (int i = 0; i < sp.n; ++i) {
    tb.tmax[i] = a.take<int32_t>((size_t)B * sp.nwin[i]);
    tb.tmin[i] = a.take<int32_t>((size_t)B * sp.nwin[i]);
  }
  const int64_t raw = (int64_t)B * sp.raw_off[sp.n];
  int32_t* flags = a.take<int32_t>(raw);
  int32_t* pos = a.take<int32_t>(raw);
  size_t tb_bytes = scan_temp_bytes(raw);
  void* tmp = a.take<char>(tb_bytes);
  KpOut none{};
  for (int i = 0; i < sp.n; ++i) {
    const int L = sp.L[i];
    const bool aligned = (((uintptr_t)ib->data) % 16 == 0) && ib->row_pitch % 16 == 0 && ib->image_stride % 16 == 0;
    if (keymode) {
      int rc = launch_key(img, ib, B, L, sp.wc[i], sp.nwin[i], aligned, none, tb.tmax[i], tb.tmin[i], st);
      if (rc) return rc;
    } else {
      window_extrema_warp<1><<<grid_for((int64_t)B * sp.nwin[i], 8), 256, 0, st>>>(
          img, ib->image_stride, B, L, sp.wc[i], sp.nwin[i], tb.tmax[i], tb.tmin[i], none, L);
      PS_LAUNCHED("window_extrema_warp<f64>");
    }
  }
  dedupe_flags<<<grid_for(raw, 256), 256, 0, st>>>(sp, tb, B, nc, dedupe, flags);
  PS_LAUNCHED("dedupe_flags");
  cub::DeviceScan::ExclusiveSum(tmp, tb_bytes, flags, pos, (int)raw, st);
  PS_LAUNCHED("cub_exclusive_scan");
  scatter_kept<<<grid_for(raw, 256), 256, 0, st>>>(sp, tb, img, ib->image_stride, B, flags, pos, ko, out->count);
  PS_LAUNCHED("scatter_kept");
  return PS_OK;
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" int ps_detect_plan(int32_t batch, int32_t nr, int32_t nc, const int32_t* host_scales, int32_t n_scales,
                              int32_t dedupe, int64_t* cap_out, size_t* workspace_bytes_out) {
  PS_REQUIRE(batch >= 1 && nr >= 1 && nc >= 1 && host_scales, PS_ERR_ARGUMENT, "bad detect plan arguments");
  int st = validate_scales(nr, nc, host_scales, n_scales);
  if (st) return st;
  ScalePlan sp = make_plan(nr, nc, host_scales, n_scales, dedupe);
  if (cap_out) *cap_out = sp.raw_off[sp.n];
  if (workspace_bytes_out) *workspace_bytes_out = workspace_need(batch, sp, sp.n == 1);
  return PS_OK;
}

extern "C" int ps_detect(const ps_image_batch* img, const int32_t* host_scales, int32_t n_scales, int32_t dedupe,
                         ps_keypoints* out, void* workspace, size_t workspace_bytes, void* stream) {
  PS_REQUIRE(img && out && host_scales && img->data && out->row && out->col && out->value && out->count,
             PS_ERR_ARGUMENT, "null argument to ps_detect");
  PS_REQUIRE((int64_t)img->nr * img->row_pitch < (int64_t)INT32_MAX, PS_ERR_ARGUMENT,
             "image too large (nr*pitch >= 2^31)");
  PS_REQUIRE(img->batch >= 1 && img->nr >= 1 && img->nc >= 1 && img->row_pitch >= img->nc &&
                 (img->batch == 1 || img->image_stride >= img->row_pitch * img->nr),
             PS_ERR_ARGUMENT, "bad image geometry");
  int st = validate_scales(img->nr, img->nc, host_scales, n_scales);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (img->pixel_type == PS_PIXELS_U8) {
    PS_REQUIRE(img->alpha > 0 && img->alpha * img->nr * img->nc <= 0.05 * 255.0, PS_ERR_CONFIG,
               "alpha=%g outside the ramp limits (imaging.py:121-128)", img->alpha);
    RampU8 im{(const uint8_t*)img->data, img->row_pitch, img->nr, img->nc, img->alpha};
    return run_detect(img, im, true, host_scales, n_scales, dedupe, out, workspace, workspace_bytes, s);
  }
  if (img->pixel_type == PS_PIXELS_F64_RAW) {
    PS_REQUIRE(img->alpha > 0 && img->alpha * img->nr * img->nc <= 0.05 * 255.0, PS_ERR_CONFIG,
               "alpha=%g outside the ramp limits (imaging.py:121-128)", img->alpha);
    RampF64Raw im{(const double*)img->data, img->row_pitch, img->nr, img->nc, img->alpha};
    return run_detect(img, im, false, host_scales, n_scales, dedupe, out, workspace, workspace_bytes, s);
  }
  if (img->pixel_type == PS_PIXELS_RGB8) {
    PS_REQUIRE(img->alpha > 0 && img->alpha * img->nr * img->nc <= 0.05 * 255.0, PS_ERR_CONFIG,
               "alpha=%g outside the ramp limits (imaging.py:121-128)", img->alpha);
    PS_REQUIRE((int64_t)img->nr * img->row_pitch * 3 < (int64_t)INT32_MAX, PS_ERR_ARGUMENT,
               "image too large (3*nr*pitch >= 2^31)");
    RampRGB8 im{(const uint8_t*)img->data, img->row_pitch, img->nr, img->nc, img->alpha, img->gray_lut};
    return run_detect(img, im, false, host_scales, n_scales, dedupe, out, workspace, workspace_bytes, s);
  }
  PS_REQUIRE(img->pixel_type == PS_PIXELS_F64, PS_ERR_ARGUMENT, "unknown pixel type %d", img->pixel_type);
  RampF64 im{(const double*)img->data, img->row_pitch, img->nr, img->nc};
  return run_detect(img, im, false, host_scales, n_scales, dedupe, out, workspace, workspace_bytes, s);
}
