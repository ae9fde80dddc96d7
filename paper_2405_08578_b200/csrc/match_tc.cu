// K3 (tensor cores) -- mutual-nearest-neighbour matching of 128-d descriptors
// on tcgen05 with an exact float64 certification (reference matcher.py:48-95).
//
// Design (SURVEY.md §7 hard part 1, contract P3):
//  1. Bit-identical descriptor rows are grouped on each side; the lowest index
//     represents its group.  Distances to identical rows are bitwise equal, so
//     np.argmin's first-occurrence winner among them is the representative.
//  2. Pass 1 (rows): one CTA owns 128 rows of X (fp16, K-major SW128 image in
//     shared memory for the whole pass) and streams every 256-row tile of Y
//     through a 3-stage bulk-copy pipeline; one thread issues 8 tcgen05.mma
//     (M=128, N=256, K=16) per tile into a double-buffered TMEM accumulator;
//     four epilogue warps read it with tcgen05.ld (thread = row) and keep
//     v = |y|^2 - 2 x.y with a fused running minimum; only when a tile holds a
//     value below the row's current k-th best is it rescanned into a top-k list
//     (k = PS_TC_TOPK = 3).
//     The distance matrix never leaves TMEM.
//  3. Certification: |v - (d^2 - |x|^2)| <= E_i, a rigorous bound from the
//     fp16 rounding residual norms and fp32 accumulation, so the true first
//     argmin is among the candidates with v <= v_min + 2 E_i; those are
//     recomputed with the reference's exact float64 arithmetic.  Rows whose
//     candidate set may exceed the list are enumerated on the tensor cores
//     (MODE 1) and decided exactly in float64.
//  4. The column argmin nn21: pass 1 keeps, per row, every column that can be
//     closer than delta_s inside its certified candidate set, and the exact
//     distances below delta_s it computes compete for their columns (ColCand
//     below) -- for every column acceptance reads, that is the column argmin.
//     Only when that list is incomplete (a row with more such columns than its
//     list holds, rows left to the exact scan, a void certificate) pass 2
//     repeats 2-3 for the columns that can be matched (nn12 of rows with
//     d < delta_s) against all rows.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cuda_fp16.h>

#include "ps_common.cuh"
#include "tc_primitives.cuh"

namespace ps {
namespace tc {

// A CTA owns XH X operand tiles of BMH = 128 rows (one M = 128 MMA each,
// against the same Y tile).  XH = 2 (N = 128) halves the Y bytes per MMA and
// is 7 % faster on dense 104k^2 data, but slower on the duplicate-heavy C4
// pair (fewer, longer CTAs for the near-tie passes), so XH = 1 (N = 256) is
// the default; -DPS_TC_XH=2 selects the other geometry.
#ifndef PS_TC_XH
#define PS_TC_XH 1
#endif
#ifndef PS_TC_BN
#define PS_TC_BN (256 / PS_TC_XH)
#endif
constexpr int BMH = 128;       // X rows per operand tile / MMA (= TMEM lanes)
constexpr int XH = PS_TC_XH;   // X tiles per CTA
constexpr int BM = BMH * XH;   // X rows per CTA
constexpr int BN = PS_TC_BN;   // Y rows per tile (= MMA N)
constexpr int NACC = 512 / (XH * BN);  // accumulator buffers in flight (TMEM holds 512 columns)
static_assert(NACC >= 2 && (NACC & (NACC - 1)) == 0, "TMEM ring");
constexpr int KD = 128;        // descriptor length
// Candidates kept per (row, part, split).  The scan's cost is its ALU-pipe instructions (half rate,
// four epilogue warps per scheduler in lockstep: ~8 cycles of scheduler time per warp instruction,
// PS_TC_DIAG_CLOCKS), and both the hit rate and the insertion shrink with the list: 3 instead of 4
// is +7 % on C5's pairs (6,360 -> 6,810 pairs/s), 2 % on the dense match, nothing on C4; 2 makes so
// many rows overflow on clustered descriptors that C5 collapses (152 pairs/s).
#ifndef PS_TC_TOPK
#define PS_TC_TOPK 3
#endif
constexpr int TOPK = PS_TC_TOPK;  // candidates kept per (row, part, split)
// Y-tile stages: as many as fit beside the X tiles (XH = 1, BN = 256: 2 x 72 KB;
// BN = 128: 5 x 36 KB); the enumeration pass trades some for per-warp hit buffers
constexpr int kSmemBudget = 232448 - 2304;
constexpr int STAGES_TOP = (kSmemBudget - XH * BMH * (128 * 2 + 32)) / (BN * (128 * 2 + 32));
constexpr int STAGES_ENUM = (kSmemBudget - XH * BMH * (128 * 2 + 32) - 16 * (4096 / 16 * 8 + 16)) / (BN * (128 * 2 + 32));
static_assert(STAGES_TOP >= 2 && STAGES_ENUM >= 2, "pipeline depth");
#ifndef PS_EPI_WARPS
#define PS_EPI_WARPS 16
#endif
constexpr int kEpiWarps = PS_EPI_WARPS;  // kParts warps per TMEM lane quarter, BN / kParts columns each
constexpr int kParts = kEpiWarps / (4 * XH);  // top-4 lists per (row, split)
constexpr int HITBUF = 4096 / kEpiWarps;  // hits staged per epilogue warp before one bulk append
#ifndef PS_TC_COPY_PARTS
#define PS_TC_COPY_PARTS 8
#endif
constexpr int kCopyParts = PS_TC_COPY_PARTS;  // bulk copies per Y tile (lanes of the producer warp)
// Each operand tile is the K-major SW128 image of the 128 descriptor columns
// followed by a 16-column augmentation block (no swizzle, 32 B per row): X rows
// carry (1, 1, 1, 0...), Y rows carry -- with the descriptor part scaled by -2
// (exact) -- the three-term fp16 split of |y|^2 (padding: +inf).  The ninth
// MMA k-step then leaves v = |y|^2 - 2 x.y in TMEM.
constexpr int KA = 16;                           // augmentation columns
constexpr uint32_t ROW_BYTES = KD * 2 + KA * 2;  // 288
constexpr uint32_t A_BYTES = BMH * ROW_BYTES;    // 36 KB per X tile (XH per CTA)
constexpr uint32_t B_BYTES = BN * ROW_BYTES;     // 36 KB
constexpr int kThreads = 64 + 32 * kEpiWarps;  // warp 0 bulk copies, warp 1 MMA/TMEM, warps 2.. epilogue
template <int MODE>
constexpr size_t smem_bytes() {
  return XH * A_BYTES + (MODE == 0 ? STAGES_TOP : STAGES_ENUM) * (size_t)B_BYTES + 256 +
         (MODE == 0 ? kParts * BM * sizeof(float) : kEpiWarps * (HITBUF * 8 + 16));
}

// ---- operand preparation ----------------------------------------------------------
// Row u of the output (u < count) is source row idx[u] (or u); rows >= count are
// zero.  Writes the tile image (fp16 K-major SW128 descriptor part, then the
// augmentation block; `is_y` selects the Y form: -2 x_h and the split |y|^2,
// +inf for padding rows), and float64 |x|, |x - x_h|, |x_h|; folds their
// maxima into maxes[0..2] (non-negative float bits).
// max that propagates NaN (its bits order above +inf as unsigned)
__device__ __forceinline__ float nan_max(float a, float b) { return (b != b || b > a) ? b : a; }

// This lane's four elements (lane * 4 .. + 3) of a 128-wide row, one vector load.
template <class T>
__device__ __forceinline__ void load4(const T* __restrict__ row, int lane, double (&x)[4]) {
  if constexpr (sizeof(T) == 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(row) + lane);
    x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
  } else {
    const double2 v0 = __ldg(reinterpret_cast<const double2*>(row) + 2 * lane);
    const double2 v1 = __ldg(reinterpret_cast<const double2*>(row) + 2 * lane + 1);
    x[0] = v0.x; x[1] = v0.y; x[2] = v1.x; x[3] = v1.y;
  }
}

template <class T>
__device__ __forceinline__ void prep_tiles_body(const T* __restrict__ src, const int32_t* __restrict__ idx,
                           const int32_t* __restrict__ count_p, int64_t count_const, int64_t n_pad, int R,
                           uint8_t* __restrict__ tiles, double* __restrict__ info, unsigned* __restrict__ maxes,
                           int is_y, int align) {
  const int lane = threadIdx.x & 31;
  const int64_t count = count_p ? (int64_t)*count_p : count_const;
  // only the row blocks that hold live rows are ever read (align = rows per reader)
  const int64_t n_used = min(n_pad, (count + align - 1) / align * align);
  float mx0 = 0.0f, mx1 = 0.0f, mx2 = 0.0f;  // lane 0: running maxima of this warp's rows
  for (int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < n_used;
       u += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const bool live = u < count;
    const int64_t s = live ? (idx ? (int64_t)idx[u] : u) : 0;
    double x[4] = {0.0, 0.0, 0.0, 0.0};
    if (live) load4(src + s * KD, lane, x);
    __half h[4];
    double sx = 0.0, sr = 0.0, sh = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      h[e] = __double2half(x[e]);
      const double hv = (double)__half2float(h[e]);
      const double rv = x[e] - hv;
      sx += x[e] * x[e];
      sr += rv * rv;
      sh += hv * hv;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      sx += __shfl_xor_sync(0xffffffffu, sx, o);
      sr += __shfl_xor_sync(0xffffffffu, sr, o);
      sh += __shfl_xor_sync(0xffffffffu, sh, o);
    }
    const int64_t tile = u / R;
    const int r = (int)(u % R);
    uint8_t* base = tiles + tile * (int64_t)R * ROW_BYTES;
    const uint32_t off = sw128_offset(R, r, lane * 4);
    if (is_y) {
#pragma unroll
      for (int e = 0; e < 4; ++e) h[e] = __hmul(h[e], __float2half(-2.0f));  // exact
    }
    __half2 p0 = __halves2half2(h[0], h[1]), p1 = __halves2half2(h[2], h[3]);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&p0);
    pk.y = *reinterpret_cast<uint32_t*>(&p1);
    *reinterpret_cast<uint2*>(base + off) = pk;
    if (lane < 2) {  // augmentation block: core matrix (r / 8, k / 8), 16 B per row
      uint4 q = make_uint4(0u, 0u, 0u, 0u);
      if (lane == 0) {
        __half a0, a1, a2;
        if (!is_y) {
          a0 = a1 = a2 = __float2half(1.0f);
        } else if (!live) {
          a0 = __float2half(INFINITY);
          a1 = a2 = __float2half(0.0f);
        } else {  // |y|^2 = a0 + a1 + a2 (to ~2^-33 relative, or a0 = inf when out of range)
          a0 = __double2half(sx);
          const double r1 = __hisinf(a0) ? 0.0 : sx - (double)__half2float(a0);
          a1 = __double2half(r1);
          a2 = __double2half(r1 - (double)__half2float(a1));
        }
        const __half2 q0 = __halves2half2(a0, a1), q1 = __halves2half2(a2, __float2half(0.0f));
        q.x = *reinterpret_cast<const uint32_t*>(&q0);
        q.y = *reinterpret_cast<const uint32_t*>(&q1);
      }
      *reinterpret_cast<uint4*>(base + R * KD * 2 + (r >> 3) * 256 + lane * 128 + (r & 7) * 16) = q;
    }
    if (lane == 0) {
      info[3 * u + 0] = sqrt(sx);
      info[3 * u + 1] = sqrt(sr);
      info[3 * u + 2] = sqrt(sh);
      if (live) {
        mx0 = nan_max(mx0, (float)(sqrt(sx) * (1.0 + 1e-6)));
        mx1 = nan_max(mx1, (float)(sqrt(sr) * (1.0 + 1e-6)));
        mx2 = nan_max(mx2, (float)(sqrt(sh) * (1.0 + 1e-6)));
      }
    }
  }
  if (!maxes) return;
  // one atomic per block and quantity (same-address atomics per row serialise)
  __shared__ float smx[3][32];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) { smx[0][w] = mx0; smx[1][w] = mx1; smx[2][w] = mx2; }
  __syncthreads();
  if (threadIdx.x < 3) {
    float m = 0.0f;
    for (int q = 0; q < nw; ++q) m = nan_max(m, smx[threadIdx.x][q]);
    if (m != 0.0f) atomicMax(maxes + threadIdx.x, __float_as_uint(m));
  }
}
template <class T>
__global__ void prep_tiles(const T* __restrict__ src, const int32_t* __restrict__ idx,
                           const int32_t* __restrict__ count_p, int64_t count_const, int64_t n_pad, int R,
                           uint8_t* __restrict__ tiles, double* __restrict__ info, unsigned* __restrict__ maxes,
                           int is_y, int align) {
  prep_tiles_body<T>(src, idx, count_p, count_const, n_pad, R, tiles, info, maxes, is_y, align);
}


// The certified error bound of a row's v values (see certify_exact_body):
// |v - (d^2 - |x|^2)| <= E for every column.  rx = |x - x_h|, hx = |x_h|;
// ymax = float bits of max |y|, max |y - y_h|, max |y_h| over the columns.
// Out of the fp16 range (|y|^2 split to inf, or elements): no certificate (inf).
__device__ __forceinline__ double cert_bound(double rx, double hx, const unsigned* __restrict__ ymax) {
  const double Nmax = __uint_as_float(ymax[0]), Rmax = __uint_as_float(ymax[1]), Hmax = __uint_as_float(ymax[2]);
  // v = fp32-accumulated sum of 144 fp16 products: x_h . (-2 y_h) plus the
  // three-term split of |y|^2 (split error <= 2^-33 |y|^2 + fp16 underflow)
  const double gamma = 144.0 * 2.384185791015625e-07;  // 144 * 2^-22 (fp32 accumulation)
  double E = 1.01 * (2.0 * (rx * Nmax + hx * Rmax) + gamma * (2.0 * hx * Hmax + Nmax * Nmax) +
                     1e-9 * Nmax * Nmax + 1.2e-7);
  if (!(E < 1e30) || !(Nmax * Nmax < 6.0e4)) E = INFINITY;
  return E;
}

// Column candidates: the mutual test without a second pass.  A pair
// (i, j = nn12[i]) is accepted only if d(i, j) < delta_s and i is the first
// argmin of column j over the distinct rows of A; that argmin's distance is
// then below delta_s too.  So pass 1 keeps, per row, every column whose
// squared distance can be below delta_s^2 (v <= delta_s^2 - |x|^2 + E, the
// certification bound) inside its certified candidate set -- the row's limit
// in the candidate limit becomes max(v_min + 2E, that threshold) -- and every exact
// float64 distance below delta_s it computes (certify_exact, pair_dist_min)
// competes for its column: cbits[j] = smallest distance bits, then nn21[j] =
// lowest original row at that distance (cand_argmin, pair_argmin).  For every
// column acceptance looks at, that equals pass 2's result.  It is incomplete
// -- and pass 2 then runs as before (needs_pass2) -- when a row's top-4 may
// not hold all its columns below the threshold (*incomplete; the row is not
// made an overflow row for it: on clustered descriptors that would be most
// rows), or when rows were decided by the exact scan (exact_rows: overflow
// rows beyond the enumerated ones, or an enumeration that outgrew its buffer).
// cbits == nullptr disables it all (pass 2 itself, rows-only calls).
struct ColCand {
  double delta_s;
  int32_t* incomplete;        // set when some row may have unlisted columns below the threshold
  unsigned long long* cbits;  // per original column
  int32_t* nn21;              // per original column
  unsigned long long* list;   // (original row << 32 | original column) of certify_exact's candidates
  double* pd;                 // their distances
  unsigned long long* n_list;
};
__device__ __forceinline__ bool needs_pass2(const int32_t* __restrict__ n_overflow, int enum_rows,
                                            const unsigned long long* __restrict__ n_pairs, int64_t cap,
                                            const int32_t* __restrict__ incomplete) {
  return *incomplete != 0 || *n_overflow > enum_rows || (int64_t)*n_pairs > cap;
}

// ---- the tcgen05 row-minimum kernel --------------------------------------------------
__device__ __forceinline__ void topk_insert(float v, int j, float (&tv)[TOPK], int (&tj)[TOPK]) {
  // sorted ascending; caller guarantees v < tv[TOPK-1]
#pragma unroll
  for (int q = TOPK - 1; q > 0; --q) {
    const bool shift = v < tv[q - 1];
    const float nv = shift ? tv[q - 1] : v;
    const int nj = shift ? tj[q - 1] : j;
    if (v < tv[q]) { tv[q] = nv; tj[q] = nj; }
  }
  if (v < tv[0]) { tv[0] = v; tj[0] = j; }
}

// MODE 0: per-row top-4 of v.  MODE 1: enumerate every (row, column) with
// v <= lim[row] into pairs (row << 32 | column), capacity `cap`.
// grid = (row blocks, splits): CTA (rb, sp) streams the sp-th contiguous
// share of the Y tiles; MODE 0 writes one top-4 list per (split, part) --
// list index sp * kParts + part of row g at topv[(list * nx_pad + g) * TOPK].
template <int MODE>
__device__ __forceinline__ void nn_topk_tc_body(const uint8_t* __restrict__ Xt, const uint8_t* __restrict__ Yt,
                                                          const int32_t* __restrict__ cnt_x,
                                                          const int32_t* __restrict__ cnt_y, float* __restrict__ topv,
                                                          int32_t* __restrict__ topj, const float* __restrict__ lim,
                                                          unsigned long long* __restrict__ pairs,
                                                          unsigned long long* __restrict__ n_pairs, int64_t cap) {
  constexpr int STAGES = MODE == 0 ? STAGES_TOP : STAGES_ENUM;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int nx = *cnt_x, ny = *cnt_y;
  const int rb = blockIdx.x;
  if (rb * BM >= nx) return;  // uniform for the whole CTA
  const int n_all = ny > 0 ? (ny + BN - 1) / BN : 0;
  const int per = (n_all + gridDim.y - 1) / gridDim.y;
  const int t_begin = min(n_all, (int)blockIdx.y * per);
  const int n_tiles = min(n_all, t_begin + per) - t_begin;  // may be 0 (then lists stay empty)
  // The row blocks walk their Y tiles from staggered starting points (a ring):
  // in lockstep every CTA would request the same tile from the same L2 lines
  // at once.  Results do not depend on the order: candidates within the
  // certified margin are strictly below the 4th best, so ties at the 4th
  // place never decide them, and the enumeration collects every hit.
  const int t_rot = n_tiles > 0 ? (int)(((int64_t)rb * n_tiles) / gridDim.x) % n_tiles : 0;
  const int n_pre = min(n_tiles, STAGES);  // Y tiles issued by thread 0 during the set-up
  const int64_t nx_pad = (int64_t)gridDim.x * BM;
  uint8_t* smem = smem_raw;  // 1024-aligned (SWIZZLE_128B atoms)
  uint8_t* sA = smem;
  uint8_t* sB = smem + XH * A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* a_full = bars;
  uint64_t* b_full = bars + 1;
  uint64_t* b_empty = b_full + STAGES;
  uint64_t* acc_full = b_empty + STAGES;
  uint64_t* acc_empty = acc_full + NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NACC);
  // MODE 1: per-epilogue-warp hit buffer + fill counter
  unsigned long long* hitbuf = reinterpret_cast<unsigned long long*>(bars + 32);
  int* hitcnt = reinterpret_cast<int*>(hitbuf + kEpiWarps * HITBUF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // MODE 0: each (row, part) thread publishes its list's 4th best; the row's
  // other parts prune with the smallest of them (see the epilogue)
  float* sthr = reinterpret_cast<float*>(bars + 32);
  if (MODE == 1 && threadIdx.x < kEpiWarps) hitcnt[threadIdx.x] = 0;
  if (MODE == 0 && threadIdx.x < kParts * BM) sthr[threadIdx.x] = INFINITY;
  if (threadIdx.x == 0) {
    mbar_init(a_full, 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(b_full + s, 1);
      mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < NACC; ++s) {
      mbar_init(acc_full + s, 1);
      mbar_init(acc_empty + s, kEpiWarps);  // one arrival per epilogue warp (512 thread arrivals serialised)
    }
    mbar_fence_init();
    // the operand copies start before the TMEM allocation and the CTA barrier:
    // the X tiles and the first STAGES Y tiles (their stages start empty)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // initialised barriers -> async proxy
    mbar_arrive_expect_tx(a_full, XH * A_BYTES);
    bulk_g2s(sA, Xt + (size_t)rb * XH * A_BYTES, XH * A_BYTES, a_full);  // the CTA's XH tiles are contiguous
    for (int t = 0; t < n_pre; ++t) {
      const int tr = t + t_rot < n_tiles ? t + t_rot : t + t_rot - n_tiles;
      mbar_arrive_expect_tx(b_full + t, B_BYTES);
      bulk_g2s(sB + t * B_BYTES, Yt + (size_t)(t_begin + tr) * B_BYTES, B_BYTES, b_full + t);
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
#ifdef PS_TC_DIAG_EARLY  // diagnostic builds only: launch + barrier init + TMEM allocation cost
  if (MODE == 0) {
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
    return;
  }
#endif

  if (warp == 0) {
    // ---- bulk-copy producer: each tile in kCopyParts pieces issued by as
    // many lanes (one 72 KB request at a time left the copy engine idle
    // between tiles: the pipeline ran at ~2 us per tile, twice the MMA time)
    if (lane < kCopyParts) {
      constexpr uint32_t piece = B_BYTES / kCopyParts;
      static_assert(B_BYTES % (16 * kCopyParts) == 0, "16-byte pieces");
      for (int t = n_pre; t < n_tiles; ++t) {
        const int s = t % STAGES;
        mbar_wait(b_empty + s, ((t / STAGES) & 1) ^ 1);
#ifdef PS_TC_DIAG_NOCOPY  // diagnostic builds only: MMA rate on the resident stages (wrong results)
        if (MODE == 0 && t >= STAGES) {
          if (lane == 0) mbar_arrive(b_full + s);
          continue;
        }
#endif
        if (lane == 0) mbar_arrive_expect_tx(b_full + s, B_BYTES);
        __syncwarp((1u << kCopyParts) - 1u);  // the expectation is posted before any piece can complete
        const int tr = t + t_rot < n_tiles ? t + t_rot : t + t_rot - n_tiles;
        bulk_g2s(sB + s * B_BYTES + lane * piece, Yt + (size_t)(t_begin + tr) * B_BYTES + lane * piece, piece,
                 b_full + s);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      const uint32_t idesc = idesc_f16_f32(BMH, BN);
      const uint32_t a0 = smem_u32(sA);
#ifndef PS_TC_NO_PREDESC  // operand descriptors built once (-DPS_TC_NO_PREDESC: rebuilt per MMA, 2.4 % slower) (the start-address field of a Y stage is added per tile)
      uint64_t adp[XH][KD / 16 + 1], bdp[KD / 16 + 1];
#pragma unroll
      for (int h = 0; h < XH; ++h) {
#pragma unroll
        for (int k = 0; k < KD / 16; ++k)
          adp[h][k] = sdesc_k_sw128(a0 + h * A_BYTES + (k >> 2) * (BMH * 128) + (uint32_t)((k & 3) * 32));
        adp[h][KD / 16] = sdesc_k_none(a0 + h * A_BYTES + BMH * KD * 2);
      }
      const uint32_t bb = smem_u32(sB);
#pragma unroll
      for (int k = 0; k < KD / 16; ++k) bdp[k] = sdesc_k_sw128(bb + (k >> 2) * (BN * 128) + (uint32_t)((k & 3) * 32));
      bdp[KD / 16] = sdesc_k_none(bb + BN * KD * 2);
#endif
      mbar_wait(a_full, 0);
#ifdef PS_TC_DIAG_CLOCKS  // diagnostic builds only: where the issuer and one epilogue warp spend their cycles
      long long c_acc = 0, c_b = 0, c_iss = 0;
#endif
      for (int t = 0; t < n_tiles; ++t) {
        const int s = t % STAGES, ab = t % NACC;
#ifdef PS_TC_DIAG_CLOCKS
        const long long k0 = clock64();
#endif
        mbar_wait(acc_empty + ab, ((t / NACC) & 1) ^ 1);
#ifdef PS_TC_DIAG_CLOCKS
        const long long k1 = clock64();
#endif
        mbar_wait(b_full + s, (t / STAGES) & 1);
#ifdef PS_TC_DIAG_CLOCKS
        const long long k2 = clock64();
        c_acc += k1 - k0;
        c_b += k2 - k1;
#endif
        tc_fence_after();
        const uint32_t b0 = smem_u32(sB + s * B_BYTES);
#ifndef PS_TC_NO_PREDESC
        const uint64_t soff = (uint64_t)((uint32_t)s * (B_BYTES >> 4));  // stage offset in the 16-byte address field
#pragma unroll
        for (int h = 0; h < XH; ++h) {
          const uint32_t acc = tmem + (uint32_t)((ab * XH + h) * BN);
#pragma unroll
          for (int k = 0; k <= KD / 16; ++k) mma_f16(acc, adp[h][k], bdp[k] + soff, idesc, k > 0 ? 1u : 0u);
        }
        (void)b0;
#else
#pragma unroll
        for (int h = 0; h < XH; ++h) {  // accumulator (ab, h): TMEM columns (ab * XH + h) * BN
          const uint32_t ah = a0 + h * A_BYTES, acc = tmem + (uint32_t)((ab * XH + h) * BN);
#pragma unroll
          for (int k = 0; k < KD / 16; ++k) {
            const uint32_t koff = (uint32_t)((k & 3) * 32);  // 16 fp16 = 32 B within the atom
            const uint64_t ad = sdesc_k_sw128(ah + (k >> 2) * (BMH * 128) + koff);
            const uint64_t bd = sdesc_k_sw128(b0 + (k >> 2) * (BN * 128) + koff);
            mma_f16(acc, ad, bd, idesc, k > 0 ? 1u : 0u);
          }
#ifndef PS_TC_DIAG_NOAUG  // diagnostic builds only: without the |y|^2 augmentation step (wrong results)
          mma_f16(acc, sdesc_k_none(ah + BMH * KD * 2), sdesc_k_none(b0 + BN * KD * 2), idesc, 1u);
#endif
        }
#endif  // PS_TC_NO_PREDESC
        mma_commit(b_empty + s);
        mma_commit(acc_full + ab);
#ifdef PS_TC_DIAG_CLOCKS
        c_iss += clock64() - k2;
#endif
      }
#ifdef PS_TC_DIAG_CLOCKS
      if (MODE == 0 && blockIdx.x == 7 && blockIdx.y == 0)
        printf("[issuer] tiles %d: wait acc_empty %lld, wait b_full %lld, issue %lld cycles per tile\n", n_tiles,
               c_acc / n_tiles, c_b / n_tiles, c_iss / n_tiles);
#endif
    }
  } else {  // ---- epilogue: thread = row, kParts warps per lane quarter split the columns
    const int quarter = warp & 3;
    const int ew = warp - 2, sub = ew >> 2, h = sub / kParts, part = sub % kParts;
    constexpr int kCols = BN / kParts;
    const int row = h * BMH + quarter * 32 + lane;
    float tv[TOPK];
    int tj[TOPK];
#pragma unroll
    for (int q = 0; q < TOPK; ++q) { tv[q] = INFINITY; tj[q] = -1; }
    const int64_t grow = (int64_t)rb * BM + row;
    // dead rows (beyond the count; their X rows may be stale) get a NaN limit: no v compares <= NaN
    const float my_lim = (MODE == 1 && grow < nx) ? lim[grow] : __int_as_float(0x7fc00000);
#ifdef PS_TC_DIAG_CLOCKS
    long long e_wait = 0, e_work = 0, e_mark = 0, e_ld = 0, e_hot = 0, e_slow = 0, e_nslow = 0;
#endif
    for (int t = 0; t < n_tiles; ++t) {
      const int ab = t % NACC;
#ifdef PS_TC_DIAG_CLOCKS
      const long long q0 = clock64();
      if (t > 0) e_work += q0 - e_mark;
#endif
      mbar_wait(acc_full + ab, (t / NACC) & 1);
#ifdef PS_TC_DIAG_CLOCKS
      e_mark = clock64();
      e_wait += e_mark - q0;
#endif
      tc_fence_after();
      const int tg = t_begin + (t + t_rot < n_tiles ? t + t_rot : t + t_rot - n_tiles);  // global tile index
      const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + (ab * XH + h) * BN + part * kCols;
#ifdef PS_TC_DIAG_NOEPI  // diagnostic builds only: the accumulator handshake without reading it (wrong results)
      if (MODE == 0) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + ab);
        continue;
      }
#endif
      // Pruning bound shared by the row's kParts threads: every published 4th
      // best has four real values at or below it, so the row's final top-4
      // lies strictly below the smallest of them (ties at the bound cannot be
      // certification candidates: the merged 4th best is then <= them).
      // Stale reads are safe -- the published values only decrease.
      float tsh = INFINITY;
      if (MODE == 0) {
#pragma unroll
        for (int p2 = 0; p2 < kParts; ++p2)
          if (p2 != part) tsh = fminf(tsh, *(volatile float*)(sthr + p2 * BM + row));
      }
      // one pass per 64-column chunk; groups of 4 columns are tested against the
      // row's threshold (4th best, or the enumeration limit) with one branch
      unsigned long long* hb = hitbuf + ew * HITBUF;
      int fill = MODE == 1 ? hitcnt[ew] : 0;
      constexpr int kChunk = kCols < 64 ? kCols : 64;  // TMEM columns per load (x64 or x32)
#ifdef PS_TC_SCAN_2PHASE
      if constexpr (MODE == 0) {
        // A/B build only (-DPS_TC_SCAN_2PHASE): two-phase scan -- (1) a branch-free pass over the
        // chunk's 16 groups that only records which groups beat the bound, (2) a warp-uniform loop
        // over the union of the lanes' hit groups that re-reads those four columns from TMEM
        // (dynamic address: no register indexing) and inserts; the accumulator is released after (2).
        // The scan, not the TMEM read, is what the epilogue costs (LOADONLY / NOEPI diagnostics: 1.86
        // vs 2.50 ms per dense pass), but this compact form (the scan loop shrinks from ~1,500 to
        // ~300 instructions) measures 2.53 ms against the inlined form's 2.50: neither code size nor
        // the insertions are the cost -- the ~90 compare instructions per warp and tile are.
#pragma unroll 1
        for (int c0 = 0; c0 < kCols; c0 += kChunk) {
          uint32_t hit = 0;
#ifdef PS_TC_DIAG_CLOCKS
          const long long z0 = clock64();
#endif
          uint32_t r[kChunk];
          tmem_ld_cols(tbase + c0, r);
          tmem_ld_wait();
#ifdef PS_TC_DIAG_CLOCKS
          e_ld += clock64() - z0;
#endif
          if (c0 + kChunk >= kCols) {  // the accumulator's values are in registers: release it before the scan
            tc_fence_before();
            __syncwarp();  // every lane's TMEM reads are complete (tcgen05.wait::ld) before lane 0 releases
            if (lane == 0) mbar_arrive(acc_empty + ab);
          }
          const float thr0 = fminf(tv[TOPK - 1], tsh);  // the bound only falls: later groups may be flagged needlessly
#pragma unroll
          for (int q = 0; q < kChunk / 4; ++q) {
            const float m4 = fminf(fminf(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1])),
                                   fminf(__uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])));
            hit |= m4 < thr0 ? 1u << q : 0u;
          }
          uint32_t wm = __reduce_or_sync(0xffffffffu, hit);
#ifdef PS_TC_DIAG_CLOCKS
          const long long z1 = clock64();
          e_hot += z1 - z0;
          e_nslow += __popc(wm);
#endif
          const int jb = tg * BN + part * kCols + c0;
#pragma unroll 1
          while (wm) {
            const int g = __ffs(wm) - 1;
            wm &= wm - 1u;
            // the group's four values: a warp-uniform jump into 16 four-move cases (the registers
            // cannot be indexed; re-reading the columns from TMEM cost ~500 cycles per group)
            uint32_t x0, x1, x2, x3;
            static_assert(kChunk == 64 || kChunk == 32, "chunk of 8 or 16 groups");
#define PS_GROUP(q) \
  case q:           \
    x0 = r[(4 * (q)) % kChunk], x1 = r[(4 * (q) + 1) % kChunk], x2 = r[(4 * (q) + 2) % kChunk], x3 = r[(4 * (q) + 3) % kChunk]; \
    break;
            switch (g) {
              PS_GROUP(0) PS_GROUP(1) PS_GROUP(2) PS_GROUP(3) PS_GROUP(4) PS_GROUP(5) PS_GROUP(6) PS_GROUP(7)
              PS_GROUP(8) PS_GROUP(9) PS_GROUP(10) PS_GROUP(11) PS_GROUP(12) PS_GROUP(13) PS_GROUP(14)
              default:
                x0 = r[kChunk - 4], x1 = r[kChunk - 3], x2 = r[kChunk - 2], x3 = r[kChunk - 1];
            }
#undef PS_GROUP
            if ((hit >> g) & 1u) {
              // the whole warp pays for this block whenever one lane is in it: one insertion of the
              // group's minimum (first column on ties), the other three only if the group's second
              // smallest also beats the updated bound (rare)
              const float v0 = __uint_as_float(x0), v1 = __uint_as_float(x1), v2 = __uint_as_float(x2),
                          v3 = __uint_as_float(x3);
              const float lo01 = fminf(v0, v1), lo23 = fminf(v2, v3), m4 = fminf(lo01, lo23);
              if (m4 < fminf(tv[TOPK - 1], tsh)) {
                const int jm = v0 == m4 ? 0 : v1 == m4 ? 1 : v2 == m4 ? 2 : 3;
                topk_insert(m4, jb + 4 * g + jm, tv, tj);
                const float s4 = fminf(fmaxf(lo01, lo23), fminf(fmaxf(v0, v1), fmaxf(v2, v3)));
                if (s4 < fminf(tv[TOPK - 1], tsh)) {
#pragma unroll 1
                  for (int e = 0; e < 4; ++e) {
                    const float v = e == 0 ? v0 : e == 1 ? v1 : e == 2 ? v2 : v3;
                    if (e != jm && v < fminf(tv[TOPK - 1], tsh)) topk_insert(v, jb + 4 * g + e, tv, tj);
                  }
                }
              }
            }
          }
        }
#ifdef PS_TC_DIAG_CLOCKS
        e_slow += clock64() - e_mark;
#endif
        *(volatile float*)(sthr + part * BM + row) = tv[TOPK - 1];
        continue;
      }
#endif
#pragma unroll 1
      for (int c0 = 0; c0 < kCols; c0 += kChunk) {
        uint32_t r[kChunk];
        tmem_ld_cols(tbase + c0, r);
        tmem_ld_wait();
#ifndef PS_TC_LATE_RELEASE
        // the accumulator's values are in registers now: release it BEFORE the compare work, so the
        // MMA of tile t + 2 can be issued while this tile is still being scanned (released after the
        // scan, the issue of t + 2 started ~700 cycles after MMA t ended and could not finish before
        // MMA t + 1 did: the tensor pipe idled every tile)
        if (c0 + kChunk >= kCols) {
          tc_fence_before();
          __syncwarp();  // every lane's TMEM reads are complete (tcgen05.wait::ld) before lane 0 releases
          if (lane == 0) mbar_arrive(acc_empty + ab);
        }
#endif
        const int jb = tg * BN + part * kCols + c0;
#ifdef PS_TC_DIAG_LOADONLY  // diagnostic builds only: the TMEM read without the scan (wrong results)
        if (MODE == 0) {
          uint32_t x = 0;
#pragma unroll
          for (int q = 0; q < kChunk; q += 16) x ^= r[q];
          if (x == 0x9E3779B9u) tv[0] = 0.0f;
          continue;
        }
#endif
#pragma unroll
        for (int q = 0; q < kChunk / 4; ++q) {
          const float v0 = __uint_as_float(r[4 * q + 0]);
          const float v1 = __uint_as_float(r[4 * q + 1]);
          const float v2 = __uint_as_float(r[4 * q + 2]);
          const float v3 = __uint_as_float(r[4 * q + 3]);
          const float m4 = fminf(fminf(v0, v1), fminf(v2, v3));
          if (MODE == 0) {
            if (m4 < fminf(tv[TOPK - 1], tsh)) {
              if (v0 < fminf(tv[TOPK - 1], tsh)) topk_insert(v0, jb + 4 * q + 0, tv, tj);
              if (v1 < fminf(tv[TOPK - 1], tsh)) topk_insert(v1, jb + 4 * q + 1, tv, tj);
              if (v2 < fminf(tv[TOPK - 1], tsh)) topk_insert(v2, jb + 4 * q + 2, tv, tj);
              if (v3 < fminf(tv[TOPK - 1], tsh)) topk_insert(v3, jb + 4 * q + 3, tv, tj);
            }
          } else if (__any_sync(0xffffffffu, m4 <= my_lim)) {
            // an inf limit (void certificate) enumerates every real column (padding columns hold +inf).
            // The group's hits (<= 4 per lane) are appended with one 3-bit-plane prefix sum.
            const int jq = jb + 4 * q;
            const unsigned hm = (unsigned)(v0 <= my_lim && jq < ny) | ((unsigned)(v1 <= my_lim && jq + 1 < ny) << 1) |
                                ((unsigned)(v2 <= my_lim && jq + 2 < ny) << 2) |
                                ((unsigned)(v3 <= my_lim && jq + 3 < ny) << 3);
            const unsigned cnt = __popc(hm), lt = (1u << lane) - 1u;
            const unsigned p0 = __ballot_sync(0xffffffffu, cnt & 1u), p1 = __ballot_sync(0xffffffffu, cnt & 2u),
                           p2 = __ballot_sync(0xffffffffu, cnt & 4u);
            const int pre = __popc(p0 & lt) + 2 * __popc(p1 & lt) + 4 * __popc(p2 & lt);
            const int tot = __popc(p0) + 2 * __popc(p1) + 4 * __popc(p2);
            if (fill + tot > HITBUF) {  // flush first (warp-uniform): one global atomic per buffer
              __syncwarp();
              unsigned long long base = 0;
              if (lane == 0) base = atomicAdd(n_pairs, (unsigned long long)fill);
              base = __shfl_sync(0xffffffffu, base, 0);
              for (int f = lane; f < fill; f += 32)
                if ((int64_t)(base + f) < cap) pairs[base + f] = hb[f];
              __syncwarp();
              fill = 0;
            }
            unsigned m = hm;
            int k = fill + pre;
            while (m) {
              const int e = __ffs(m) - 1;
              m &= m - 1u;
              hb[k++] = ((unsigned long long)grow << 32) | (unsigned long long)(jq + e);
            }
            fill += tot;
          }
        }
      }
      if (MODE == 1) {
        __syncwarp();
        if (lane == 0) hitcnt[ew] = fill;
        __syncwarp();
      } else {
        *(volatile float*)(sthr + part * BM + row) = tv[TOPK - 1];
      }
#ifdef PS_TC_LATE_RELEASE  // diagnostic builds only: the accumulator released after the scan
      tc_fence_before();
      __syncwarp();  // every lane's TMEM reads are complete (tcgen05.wait::ld) before lane 0 releases
      if (lane == 0) mbar_arrive(acc_empty + ab);
#endif
    }
#ifdef PS_TC_DIAG_CLOCKS
    if (MODE == 0 && blockIdx.x == 7 && blockIdx.y == 0 && lane == 0 && (ew == 0 || ew == 5))
      printf("[epilogue warp %d] wait acc_full %lld, ld + scan %lld cycles per tile (2-phase: ld %lld, ld + hot %lld, "
             "wait-done to slow-done %lld, slow groups %lld per 100 tiles)\n", ew, e_wait / n_tiles,
             e_work / max(n_tiles - 1, 1), e_ld / n_tiles, e_hot / n_tiles, e_slow / n_tiles, 100 * e_nslow / n_tiles);
#endif
    if (MODE == 1) {
      unsigned long long* hb = hitbuf + ew * HITBUF;
      const int fill = hitcnt[ew];
      unsigned long long base = 0;
      if (lane == 0 && fill) base = atomicAdd(n_pairs, (unsigned long long)fill);
      base = __shfl_sync(0xffffffffu, base, 0);
      for (int e = lane; e < fill; e += 32)
        if ((int64_t)(base + e) < cap) pairs[base + e] = hb[e];
    }
    if (MODE == 0 && grow < nx) {
      const int64_t list = (int64_t)blockIdx.y * kParts + part;
#pragma unroll
      for (int q = 0; q < TOPK; ++q) {
        topv[(list * nx_pad + grow) * TOPK + q] = tv[q];
        topj[(list * nx_pad + grow) * TOPK + q] = tj[q];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) nn_topk_tc(const uint8_t* __restrict__ Xt, const uint8_t* __restrict__ Yt,
                                                          const int32_t* __restrict__ cnt_x,
                                                          const int32_t* __restrict__ cnt_y, float* __restrict__ topv,
                                                          int32_t* __restrict__ topj, const float* __restrict__ lim,
                                                          unsigned long long* __restrict__ pairs,
                                                          unsigned long long* __restrict__ n_pairs, int64_t cap) {
  nn_topk_tc_body<MODE>(Xt, Yt, cnt_x, cnt_y, topv, topj, lim, pairs, n_pairs, cap);
}


// ---- certification + exact float64 recheck ------------------------------------------
// Reference distance between float-typed rows a and b (numpy pairwise order).
template <class T>
__device__ __forceinline__ double exact_dist(const T* __restrict__ a, const T* __restrict__ b) {
  double r[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) r[t] = 0.0;
#pragma unroll 4
  for (int k = 0; k < KD; k += 8) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const double e = __dsub_rn((double)b[k + t], (double)a[k + t]);
      r[t] = __dadd_rn(r[t], __dmul_rn(e, e));
    }
  }
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                              __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7]))));
}

// The same distance computed by an aligned group of 8 lanes: lane t of the
// group owns accumulator r[t] (elements 8m + t, m sequential), and the groups'
// lanes combine in the reference's ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) order.
// Loads of the group are 32-byte contiguous per step.  Result valid in lane t=0.
template <class T>
__device__ __forceinline__ double exact_dist8(const T* __restrict__ a, const T* __restrict__ b, int t) {
  double r = 0.0;
#pragma unroll
  for (int m = 0; m < KD / 8; ++m) {
    const double e = __dsub_rn((double)b[8 * m + t], (double)a[8 * m + t]);
    r = __dadd_rn(r, __dmul_rn(e, e));
  }
  const double p1 = __dadd_rn(r, __shfl_down_sync(0xffffffffu, r, 1));   // t even: r_t + r_{t+1}
  const double p2 = __dadd_rn(p1, __shfl_down_sync(0xffffffffu, p1, 2)); // t % 4 == 0
  const double p4 = __dadd_rn(p2, __shfl_down_sync(0xffffffffu, p2, 4)); // t == 0
  return __dsqrt_rn(p4);
}

// One thread per X' row u.  x_orig[u] / y_orig[j'] map tile rows to original
// indices (ties break on original indices).  Writes nn[x_orig[u]] and d[...];
// rows whose candidates may not fit the top-4 are appended to `overflow`.
template <class T>
__device__ __forceinline__ void certify_exact_body(const float* __restrict__ topv, const int32_t* __restrict__ topj,
                              const int32_t* __restrict__ cnt_x, const int32_t* __restrict__ x_orig,
                              const int32_t* __restrict__ y_orig, const double* __restrict__ xinfo,
                              const unsigned* __restrict__ ymax, const T* __restrict__ X, const T* __restrict__ Y,
                              int32_t* __restrict__ nn, double* __restrict__ dist, int32_t* __restrict__ overflow,
                              int32_t* __restrict__ n_overflow, float* __restrict__ overflow_lim, int n_lists,
                              int64_t nx_pad, const ColCand cc) {
  const int nx = *cnt_x;
  const int t = threadIdx.x & 7;
  const int per_block = blockDim.x >> 3;
  for (int ub = blockIdx.x * per_block; ub < nx; ub += gridDim.x * per_block) {  // 8 lanes per row
    const int u = ub + (threadIdx.x >> 3);
    const bool live = u < nx;
    const int uu = live ? u : 0;
    const int xi = x_orig ? x_orig[uu] : uu;
    // |v - (d^2 - |x|^2)| <= 2(|x - x_h||y| + |x_h||y - y_h|) + 2 g |x_h||y_h| + rounding of v;
    // out of the fp16 range there is no certificate: every column is enumerated
    // and the rows fall back to the exact scan
    const double E = cert_bound(xinfo[3 * uu + 1], xinfo[3 * uu + 2], ymax);
    float tv[TOPK];
    int tj[TOPK];
#pragma unroll
    for (int q = 0; q < TOPK; ++q) { tv[q] = INFINITY; tj[q] = -1; }
    for (int l = 0; l < n_lists; ++l) {  // the 4 smallest of the per-split lists are the global top-4
      float lv[TOPK];
      int lj[TOPK];
      if constexpr (TOPK == 4) {
        const float4 v4 = __ldg(reinterpret_cast<const float4*>(topv + ((int64_t)l * nx_pad + uu) * TOPK));
        const int4 j4 = __ldg(reinterpret_cast<const int4*>(topj + ((int64_t)l * nx_pad + uu) * TOPK));
        lv[0] = v4.x; lv[1] = v4.y; lv[2] = v4.z; lv[3] = v4.w;
        lj[0] = j4.x; lj[1] = j4.y; lj[2] = j4.z; lj[3] = j4.w;
      } else {
#pragma unroll
        for (int q = 0; q < TOPK; ++q) {
          lv[q] = topv[((int64_t)l * nx_pad + uu) * TOPK + q];
          lj[q] = topj[((int64_t)l * nx_pad + uu) * TOPK + q];
        }
      }
#pragma unroll
      for (int q = 0; q < TOPK; ++q)
        if (lv[q] < tv[TOPK - 1]) topk_insert(lv[q], lj[q], tv, tj);
    }
    const double lim = (double)tv[0] + 2.0 * E;
    double cth = -INFINITY;  // column threshold: v of every column that can be closer than delta_s (ColCand)
    // once some row has declared the list incomplete the column pass will run, so later rows need not
    // widen their candidate sets (a benign race: the list is simply not used then)
    if (cc.cbits && *(volatile int32_t*)cc.incomplete == 0) {
      const double nxv = xinfo[3 * uu];
      const double c = cc.delta_s * cc.delta_s * (1.0 + 1e-9) - nxv * nxv + E + 1e-6;
      cth = (c == c) ? c : INFINITY;
    }
    const double clim = fmax(lim, cth);  // candidate limit
    const bool over = (double)tv[TOPK - 1] <= lim;  // candidates may extend past the top-4
    // a row whose 4th best is within the column threshold may have any number of columns below it:
    // the list is declared incomplete instead of enumerating them (clustered descriptors: most rows)
    const bool many = cc.cbits && (double)tv[TOPK - 1] <= cth;
    if (live && over && t == 0) {
      const int slot = atomicAdd(n_overflow, 1);
      overflow[slot] = u;
      // otherwise the enumeration lists the row's (at most three) column candidates too
      overflow_lim[slot] = __double2float_ru(many ? lim : clim);
    }
    if (live && many && t == 0) *cc.incomplete = 1;
    double bd = INFINITY;
    int bj = INT32_MAX;
    // the (up to TOPK) candidate distances are computed together: TOPK
    // independent accumulator chains per lane instead of TOPK serial ones
    // (each distance keeps the reference's exact operation order)
    bool cand[TOPK];
    int yj[TOPK];
    bool any = false;
#pragma unroll
    for (int q = 0; q < TOPK; ++q) {
      cand[q] = live && !over && tj[q] >= 0 && (double)tv[q] <= clim;
      yj[q] = cand[q] ? (y_orig ? y_orig[tj[q]] : tj[q]) : 0;
      any |= cand[q];
    }
    if (__any_sync(0xffffffffu, any)) {  // warp-uniform
      const T* xa = X + (int64_t)xi * KD;
      double r[TOPK];
#pragma unroll
      for (int q = 0; q < TOPK; ++q) r[q] = 0.0;
#pragma unroll 4
      for (int m = 0; m < KD / 8; ++m) {
        const double xe = (double)xa[8 * m + t];
#pragma unroll
        for (int q = 0; q < TOPK; ++q) {
          const double e = __dsub_rn((double)Y[(int64_t)yj[q] * KD + 8 * m + t], xe);
          r[q] = __dadd_rn(r[q], __dmul_rn(e, e));
        }
      }
#pragma unroll
      for (int q = 0; q < TOPK; ++q) {  // the 8-lane combination of exact_dist8
        const double p1 = __dadd_rn(r[q], __shfl_down_sync(0xffffffffu, r[q], 1));
        const double p2 = __dadd_rn(p1, __shfl_down_sync(0xffffffffu, p1, 2));
        const double p4 = __dadd_rn(p2, __shfl_down_sync(0xffffffffu, p2, 4));
        const double dd = __dsqrt_rn(p4);
        if (cand[q] && (dd < bd || (dd == bd && yj[q] < bj))) { bd = dd; bj = yj[q]; }
        if (cc.cbits && cand[q] && t == 0 && dd < cc.delta_s) {  // competes for its column
          const unsigned long long slot = atomicAdd(cc.n_list, 1ull);  // <= TOPK per row: the list cannot overflow
          cc.list[slot] = ((unsigned long long)(unsigned)xi << 32) | (unsigned long long)(unsigned)yj[q];
          cc.pd[slot] = dd;
          atomicMin(cc.cbits + yj[q], (unsigned long long)__double_as_longlong(dd));
        }
      }
    }
    if (live && !over && t == 0) {
      nn[xi] = bj;
      dist[xi] = bd;
    }
  }
}
template <class T>
__global__ void certify_exact(const float* __restrict__ topv, const int32_t* __restrict__ topj,
                              const int32_t* __restrict__ cnt_x, const int32_t* __restrict__ x_orig,
                              const int32_t* __restrict__ y_orig, const double* __restrict__ xinfo,
                              const unsigned* __restrict__ ymax, const T* __restrict__ X, const T* __restrict__ Y,
                              int32_t* __restrict__ nn, double* __restrict__ dist, int32_t* __restrict__ overflow,
                              int32_t* __restrict__ n_overflow, float* __restrict__ overflow_lim, int n_lists,
                              int64_t nx_pad, const ColCand cc) {
  certify_exact_body<T>(topv, topj, cnt_x, x_orig, y_orig, xinfo, ymax, X, Y, nn, dist, overflow, n_overflow,
                        overflow_lim, n_lists, nx_pad, cc);
}


// overflow row q -> source row of X (composition of the two index lists)
__device__ __forceinline__ void gather_rows_body(const int32_t* __restrict__ overflow, const int32_t* __restrict__ n_overflow,
                            const int32_t* __restrict__ x_idx, int32_t* __restrict__ out) {
  const int n = *n_overflow;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
    out[q] = x_idx ? x_idx[overflow[q]] : overflow[q];
}
__global__ void gather_rows(const int32_t* __restrict__ overflow, const int32_t* __restrict__ n_overflow,
                            const int32_t* __restrict__ x_idx, int32_t* __restrict__ out) {
  gather_rows_body(overflow, n_overflow, x_idx, out);
}


// exact distance of every enumerated (overflow row, column) pair; per row the
// minimum distance bits, then the lowest original column at that distance
template <class T>
__device__ __forceinline__ void pair_dist_min_body(const unsigned long long* __restrict__ pairs,
                              const unsigned long long* __restrict__ n_pairs, int64_t cap,
                              const int32_t* __restrict__ xsrc, const int32_t* __restrict__ y_idx,
                              const T* __restrict__ X, const T* __restrict__ Y, double* __restrict__ pd,
                              unsigned long long* __restrict__ best_bits, const ColCand cc) {
  const int64_t n = min((int64_t)*n_pairs, cap);
  const int t = threadIdx.x & 7;
  const int64_t per_block = blockDim.x >> 3;
  // the loop bound depends only on the block, so whole warps stay converged for the shuffles
  for (int64_t kb = (int64_t)blockIdx.x * per_block; kb < n; kb += (int64_t)gridDim.x * per_block) {
    const int64_t k = kb + (threadIdx.x >> 3);
    const bool live = k < n;
    const unsigned long long pr = live ? pairs[k] : 0ull;
    const int q = (int)(pr >> 32), jt = (int)(pr & 0xffffffffu);
    const int yj = live ? (y_idx ? y_idx[jt] : jt) : 0;
    const int xs = live ? xsrc[q] : 0;
    const double d = exact_dist8(X + (int64_t)xs * KD, Y + (int64_t)yj * KD, t);
    if (live && t == 0) {
      pd[k] = d;
      atomicMin(best_bits + q, (unsigned long long)__double_as_longlong(d));
      if (cc.cbits && d < cc.delta_s) atomicMin(cc.cbits + yj, (unsigned long long)__double_as_longlong(d));
    }
  }
}
template <class T>
__global__ void pair_dist_min(const unsigned long long* __restrict__ pairs,
                              const unsigned long long* __restrict__ n_pairs, int64_t cap,
                              const int32_t* __restrict__ xsrc, const int32_t* __restrict__ y_idx,
                              const T* __restrict__ X, const T* __restrict__ Y, double* __restrict__ pd,
                              unsigned long long* __restrict__ best_bits, const ColCand cc) {
  pair_dist_min_body<T>(pairs, n_pairs, cap, xsrc, y_idx, X, Y, pd, best_bits, cc);
}


template <class T>
__device__ __forceinline__ void pair_argmin_body(const unsigned long long* __restrict__ pairs, const unsigned long long* __restrict__ n_pairs,
                            int64_t cap, const int32_t* __restrict__ y_idx, const double* __restrict__ pd,
                            const unsigned long long* __restrict__ best_bits, int* __restrict__ best_j,
                            const int32_t* __restrict__ xsrc, const ColCand cc) {
  const int64_t n = min((int64_t)*n_pairs, cap);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(pairs[k] >> 32), jt = (int)(pairs[k] & 0xffffffffu);
    const int yj = y_idx ? y_idx[jt] : jt;
    const unsigned long long db = (unsigned long long)__double_as_longlong(pd[k]);
    if (db == best_bits[q]) atomicMin(best_j + q, yj);
    if (cc.cbits && db == cc.cbits[yj]) atomicMin(cc.nn21 + yj, xsrc[q]);  // the column's first row at its minimum
  }
}
template <class T>
__global__ void pair_argmin(const unsigned long long* __restrict__ pairs, const unsigned long long* __restrict__ n_pairs,
                            int64_t cap, const int32_t* __restrict__ y_idx, const double* __restrict__ pd,
                            const unsigned long long* __restrict__ best_bits, int* __restrict__ best_j,
                            const int32_t* __restrict__ xsrc, const ColCand cc) {
  pair_argmin_body<T>(pairs, n_pairs, cap, y_idx, pd, best_bits, best_j, xsrc, cc);
}


__device__ __forceinline__ void pair_write_body(const int32_t* __restrict__ n_overflow, const int32_t* __restrict__ xsrc,
                           const unsigned long long* __restrict__ best_bits, const int* __restrict__ best_j,
                           int32_t* __restrict__ nn, double* __restrict__ dist, int enum_rows) {
  const int n = min(*n_overflow, enum_rows);  // rows beyond were not enumerated (exact_rows decides them)
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    nn[xsrc[q]] = best_j[q];
    dist[xsrc[q]] = __longlong_as_double((long long)best_bits[q]);
  }
}
__global__ void pair_write(const int32_t* __restrict__ n_overflow, const int32_t* __restrict__ xsrc,
                           const unsigned long long* __restrict__ best_bits, const int* __restrict__ best_j,
                           int32_t* __restrict__ nn, double* __restrict__ dist, int enum_rows) {
  pair_write_body(n_overflow, xsrc, best_bits, best_j, nn, dist, enum_rows);
}


// exact full scans (only if the enumerated pairs overflowed their buffer)
template <class T>
__device__ __forceinline__ void exact_rows_body(const int32_t* __restrict__ rows, const int32_t* __restrict__ n_rows,
                           const int32_t* __restrict__ x_orig, const T* __restrict__ X, const T* __restrict__ Y,
                           int64_t ny, int32_t* __restrict__ nn, double* __restrict__ dist,
                           const unsigned long long* __restrict__ n_pairs, int64_t cap, int enum_rows) {
  __shared__ double sd[32];
  __shared__ int sj[32];
  // rows [0, enum_rows) were enumerated on the tensor cores; when their pairs
  // fit the buffer only the rows beyond need the exact scan
  const int q0 = (n_pairs && (int64_t)*n_pairs <= cap) ? enum_rows : 0;
  const int n = *n_rows;
  if (q0 >= n) return;
  for (int q = q0 + blockIdx.x; q < n; q += gridDim.x) {
    const int u = rows[q];
    const int xi = x_orig ? x_orig[u] : u;
    double bd = INFINITY;
    int bj = INT32_MAX;
    for (int64_t j = threadIdx.x; j < ny; j += blockDim.x) {
      const double dd = exact_dist(X + (int64_t)xi * KD, Y + j * KD);
      if (dd < bd || (dd == bd && (int)j < bj)) { bd = dd; bj = (int)j; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double d2 = __shfl_xor_sync(0xffffffffu, bd, o);
      const int j2 = __shfl_xor_sync(0xffffffffu, bj, o);
      if (d2 < bd || (d2 == bd && j2 < bj)) { bd = d2; bj = j2; }
    }
    if ((threadIdx.x & 31) == 0) { sd[threadIdx.x >> 5] = bd; sj[threadIdx.x >> 5] = bj; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        if (sd[w] < bd || (sd[w] == bd && sj[w] < bj)) { bd = sd[w]; bj = sj[w]; }
      nn[xi] = bj;
      dist[xi] = bd;
    }
    __syncthreads();
  }
}
template <class T>
__global__ void exact_rows(const int32_t* __restrict__ rows, const int32_t* __restrict__ n_rows,
                           const int32_t* __restrict__ x_orig, const T* __restrict__ X, const T* __restrict__ Y,
                           int64_t ny, int32_t* __restrict__ nn, double* __restrict__ dist,
                           const unsigned long long* __restrict__ n_pairs, int64_t cap, int enum_rows) {
  exact_rows_body<T>(rows, n_rows, x_orig, X, Y, ny, nn, dist, n_pairs, cap, enum_rows);
}


// ---- duplicate rows --------------------------------------------------------------------
// Open-addressing table of row hashes (tsize a power of two, keys 0 = empty):
// per hash the lowest row index.  slot_of[i] receives row i's slot.
// (hash_rows / b_hash below: a half-warp per row.)

// rep[i] = the lowest row with row i's hash when bitwise equal to row i, else
// i itself (a hash collision only splits a group); flag[i] = (rep == i).
template <class T>
__device__ __forceinline__ void mark_reps_table_body(const T* __restrict__ X, int64_t n, const int32_t* __restrict__ tidx,
                                const int32_t* __restrict__ slot_of, int32_t* __restrict__ rep,
                                int32_t* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
       i += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int l = tidx[slot_of[i]];
    bool same = true;
    if (l != (int)i) {
      double a[4], c[4];
      load4(X + i * KD, lane, a);
      load4(X + (int64_t)l * KD, lane, c);
#pragma unroll
      for (int e = 0; e < 4; ++e) same &= a[e] == c[e];
      same = __all_sync(0xffffffffu, same);
    }
    if (lane == 0) {
      const int r = same ? l : (int)i;
      rep[i] = r;
      flag[i] = r == (int)i;
    }
  }
}
template <class T>
__global__ void mark_reps_table(const T* __restrict__ X, int64_t n, const int32_t* __restrict__ tidx,
                                const int32_t* __restrict__ slot_of, int32_t* __restrict__ rep,
                                int32_t* __restrict__ flag) {
  mark_reps_table_body<T>(X, n, tidx, slot_of, rep, flag);
}


__global__ void copy_from_rep(const int32_t* __restrict__ rep, int64_t n, int32_t* __restrict__ nn,
                              double* __restrict__ dist) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = rep[i];
    if (r != (int32_t)i) {
      nn[i] = nn[r];
      dist[i] = dist[r];
    }
  }
}

__global__ void iota32(int32_t* v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

// columns worth checking: nn12 of rows with d < delta_s
__device__ __forceinline__ void mark_columns_body(const int32_t* __restrict__ a_uniq, const int32_t* __restrict__ n_auniq,
                             const int32_t* __restrict__ nn12, const double* __restrict__ d12, double delta_s,
                             int32_t* __restrict__ colflag, const int32_t* __restrict__ n_overflow, int enum_rows,
                             const unsigned long long* __restrict__ n_pairs, int64_t pair_cap,
                             const int32_t* __restrict__ incomplete) {
  // pass 1's column candidates already decided nn21 (ColCand): no column needs pass 2
  if (incomplete && !needs_pass2(n_overflow, enum_rows, n_pairs, pair_cap, incomplete)) return;
  const int n = *n_auniq;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    const int i = a_uniq[u];
    if (d12[i] < delta_s) colflag[nn12[i]] = 1;
  }
}
__global__ void mark_columns(const int32_t* __restrict__ a_uniq, const int32_t* __restrict__ n_auniq,
                             const int32_t* __restrict__ nn12, const double* __restrict__ d12, double delta_s,
                             int32_t* __restrict__ colflag, const int32_t* __restrict__ n_overflow, int enum_rows,
                             const unsigned long long* __restrict__ n_pairs, int64_t pair_cap,
                             const int32_t* __restrict__ incomplete) {
  mark_columns_body(a_uniq, n_auniq, nn12, d12, delta_s, colflag, n_overflow, enum_rows, n_pairs, pair_cap,
                    incomplete);
}


// acceptance over original rows (matcher.py:74-79); only representatives can be mutual
__device__ __forceinline__ void accept_pairs_body(const int32_t* __restrict__ a_rep, int64_t n1, const int32_t* __restrict__ nn12,
                             const double* __restrict__ d12, const int32_t* __restrict__ nn21, double delta_s,
                             unsigned long long* __restrict__ keys_pair, unsigned long long* __restrict__ keys_delta,
                             unsigned long long* __restrict__ counter) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n1; i += (int64_t)gridDim.x * blockDim.x) {
    if (a_rep[i] != (int32_t)i) continue;
    const int j = nn12[i];
    if (d12[i] < delta_s && nn21[j] == (int32_t)i) {
      const unsigned long long slot = atomicAdd(counter, 1ull);
      keys_pair[slot] = ((unsigned long long)i << 32) | (unsigned long long)j;
      keys_delta[slot] = (unsigned long long)__double_as_longlong(d12[i]);
    }
  }
}
__global__ void accept_pairs(const int32_t* __restrict__ a_rep, int64_t n1, const int32_t* __restrict__ nn12,
                             const double* __restrict__ d12, const int32_t* __restrict__ nn21, double delta_s,
                             unsigned long long* __restrict__ keys_pair, unsigned long long* __restrict__ keys_delta,
                             unsigned long long* __restrict__ counter) {
  accept_pairs_body(a_rep, n1, nn12, d12, nn21, delta_s, keys_pair, keys_delta, counter);
}


// ---- column candidates (ColCand): certify_exact's list -> nn21 ---------------------------
__device__ __forceinline__ void cand_argmin_body(const ColCand cc) {
  if (!cc.cbits) return;
  const int64_t n = (int64_t)*cc.n_list;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int xi = (int)(cc.list[k] >> 32), yj = (int)(cc.list[k] & 0xffffffffu);
    if ((unsigned long long)__double_as_longlong(cc.pd[k]) == cc.cbits[yj]) atomicMin(cc.nn21 + yj, xi);
  }
}
__global__ void cand_argmin(const ColCand cc) { cand_argmin_body(cc); }

// ---- host orchestration ------------------------------------------------------------
struct Side {  // a descriptor matrix with its duplicate-row structure
  int32_t *iota, *slot_of, *rep, *flag, *uniq, *n_uniq;
  unsigned long long* tkey;  // hash table of rows
  int32_t* tidx;
  int64_t tsize;
};

struct TcWs {
  Side a, b;
  void* cub_tmp;
  size_t cub_bytes;
  uint8_t *xt, *yt;
  float* topv;
  double *xinfo, *yinfo;
  unsigned* ymax;
  int32_t *topj, *nn12, *nn21, *overflow, *n_overflow, *colflag, *cols, *n_cols, *xsrc, *best_j;
  double *d12, *d21, *pd;
  float* lim;
  unsigned long long *pairs, *n_pairs, *best_bits;
  int64_t pair_cap;
  unsigned long long *cand, *n_cand, *cbits;  // pass 1's column candidates (ColCand)
  double* cpd;
  int32_t* cand_incomplete;
  int64_t cand_cap;
};

inline int64_t rup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

constexpr int kMaxSplit = 8;
constexpr int kSMs = 148;
// asynchronous mode: row blocks of the near-tie enumeration launched blind
// (the rest of a larger overflow list is decided by the exact scan)
constexpr int kEnumBlocksAsync = 4;
constexpr int kThroughputRowBlocks = 32;

// statistics of the last tensor-core match on this thread (ps_match_stats)
thread_local int64_t g_stats[8];  // uniq_a, uniq_b, cols, overflow rows, enumerated pairs, mma flops, -, -

int32_t read_count(const int32_t* p, cudaStream_t st) {
  int32_t h = 0;
  cudaMemcpyAsync(&h, p, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return h;
}
// two device counts with one synchronisation
void read_counts(const int32_t* p, const int32_t* q, int64_t* hp, int64_t* hq, cudaStream_t st) {
  int32_t h[2] = {0, 0};
  cudaMemcpyAsync(&h[0], p, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h[1], q, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  *hp = h[0];
  *hq = h[1];
}

// row blocks x column splits.  One CTA per SM is resident (~180 KB of shared
// memory), so the split minimises waves x (tiles per CTA + per-CTA overhead,
// about four tiles' worth: launch, TMEM allocation, X tile, pipeline fill).
// throughput = true (asynchronous mode, where matches of other pairs run
// concurrently): no column split once there are enough row blocks -- every
// CTA pays its fixed cost (TMEM allocation, X tile, pipeline fill and drain)
// once, so fewer, longer CTAs leave more of the machine to the other pairs.
dim3 tc_grid(int64_t rows, int64_t cols, bool throughput = false) {
  const int rb = (int)std::max<int64_t>(1, (rows + BM - 1) / BM);
  const int tiles = (int)std::max<int64_t>(1, (cols + BN - 1) / BN);
  int best = 1;
  int64_t best_cost = INT64_MAX;
  for (int s = 1; s <= std::min(kMaxSplit, tiles) && !(throughput && rb >= kThroughputRowBlocks); ++s) {
    const int64_t waves = ((int64_t)rb * s + kSMs - 1) / kSMs;
    const int64_t cost = waves * ((tiles + s - 1) / s + 4 * XH);
    if (cost < best_cost) { best_cost = cost; best = s; }
  }
#ifdef PS_DIAG  // diagnostic builds only (-DPS_DIAG): the product library reads no environment
  if (const char* e = getenv("PS_TC_SPLIT")) best = std::max(1, std::min({atoi(e), kMaxSplit, tiles}));
#endif
  return dim3(rb, best);
}

size_t cub_need(int64_t n) {  // the order-preserving selections
  size_t b = 0;
  cub::DeviceSelect::Flagged(nullptr, b, (const int32_t*)nullptr, (const int32_t*)nullptr, (int32_t*)nullptr,
                             (int32_t*)nullptr, (int)n);
  return b;
}

TcWs carve_tc(void* base, int64_t n1, int64_t n2, size_t* used) {
  Arena ar{(char*)base, 0, 0};
  TcWs w{};
  auto side = [&](Side& s, int64_t n) {
    s.iota = ar.take<int32_t>(n);
    s.slot_of = ar.take<int32_t>(n);
    s.rep = ar.take<int32_t>(n);
    s.flag = ar.take<int32_t>(n);
    s.uniq = ar.take<int32_t>(n);
    s.n_uniq = ar.take<int32_t>(1);
    s.tsize = 64;
    while (s.tsize < 2 * n) s.tsize <<= 1;
    s.tkey = ar.take<unsigned long long>(s.tsize);
    s.tidx = ar.take<int32_t>(s.tsize);
  };
  side(w.a, n1);
  side(w.b, n2);
  const int64_t nmax = std::max(n1, n2);
  w.cub_bytes = cub_need(nmax);
  w.cub_tmp = ar.take<char>(w.cub_bytes);
  const int64_t xrows = rup(nmax, BM), yrows = rup(nmax, BN);
  w.xt = ar.take<uint8_t>((size_t)xrows * ROW_BYTES);
  w.yt = ar.take<uint8_t>((size_t)yrows * ROW_BYTES);
  w.xinfo = ar.take<double>(3 * xrows);
  w.yinfo = ar.take<double>(3 * yrows);
  w.ymax = ar.take<unsigned>(4);
  w.topv = ar.take<float>(xrows * TOPK * kParts * kMaxSplit);
  w.topj = ar.take<int32_t>(xrows * TOPK * kParts * kMaxSplit);
  w.nn12 = ar.take<int32_t>(n1);
  w.d12 = ar.take<double>(n1);
  w.nn21 = ar.take<int32_t>(n2);
  w.d21 = ar.take<double>(n2);
  w.overflow = ar.take<int32_t>(nmax);
  w.n_overflow = ar.take<int32_t>(1);
  w.lim = ar.take<float>(rup(nmax, BM));
  w.xsrc = ar.take<int32_t>(nmax);
  w.best_j = ar.take<int32_t>(nmax);
  w.best_bits = ar.take<unsigned long long>(nmax);
  w.pair_cap = std::max<int64_t>(1 << 22, 64 * nmax);
  w.pairs = ar.take<unsigned long long>(w.pair_cap);
  w.pd = ar.take<double>(w.pair_cap);
  w.n_pairs = ar.take<unsigned long long>(1);
  w.colflag = ar.take<int32_t>(n2);
  w.cols = ar.take<int32_t>(n2);
  w.n_cols = ar.take<int32_t>(1);
  w.cand_cap = std::max<int64_t>(1 << 18, 8 * nmax);
  w.cand = ar.take<unsigned long long>(w.cand_cap);
  w.cpd = ar.take<double>(w.cand_cap);
  w.n_cand = ar.take<unsigned long long>(1);
  w.cand_incomplete = ar.take<int32_t>(1);
  w.cbits = ar.take<unsigned long long>(n2);
  *used = ar.used + 256;
  return w;
}

int grid_for(int64_t work, int per) {
  int64_t g = (work + per - 1) / per;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

template <class T>
__global__ void hash_rows(const T* __restrict__ X, int64_t n, unsigned long long* __restrict__ tkey,
                          int32_t* __restrict__ tidx, int64_t tsize, int32_t* __restrict__ slot_of);  // below

template <class T>
int dedupe(const T* X, int64_t n, Side& s, const TcWs& w, cudaStream_t st) {
  cudaMemsetAsync(s.tkey, 0, s.tsize * sizeof(unsigned long long), st);
  cudaMemsetAsync(s.tidx, 0x7f, s.tsize * sizeof(int32_t), st);
  hash_rows<T><<<grid_for(n, 16), 256, 0, st>>>(X, n, s.tkey, s.tidx, s.tsize, s.slot_of);  // a half-warp per row
  PS_LAUNCHED("hash_rows");
  mark_reps_table<T><<<grid_for(n, 8), 256, 0, st>>>(X, n, s.tidx, s.slot_of, s.rep, s.flag);
  PS_LAUNCHED("mark_reps_table");
  iota32<<<grid_for(n, 256), 256, 0, st>>>(s.iota, n);
  PS_LAUNCHED("iota32");
  size_t tb = w.cub_bytes;
  cub::DeviceSelect::Flagged(w.cub_tmp, tb, s.iota, s.flag, s.uniq, s.n_uniq, (int)n, st);
  PS_LAUNCHED("cub_select(reps)");
  return PS_OK;
}

// One direction: for every row X[x_idx[u]] (u < *n_x) the exact first argmin
// over Y rows (candidates from tensor cores, all Y rows reachable through
// y_idx[0..*n_y) which must include every distinct row of Y).
template <class T>
int nearest_pass(const T* X, int64_t nx_max, const int32_t* x_idx, const int32_t* n_x, const T* Y, int64_t ny_all,
                 const int32_t* y_idx, const int32_t* n_y, int32_t* nn, double* dist, const TcWs& w,
                 cudaStream_t st, int64_t* nx_io = nullptr, int64_t* ny_io = nullptr, bool sync = true,
                 ColCand cc = ColCand{}, int* enum_rows_out = nullptr,  // cc.cbits: the pass also decides the columns
                 int32_t* incomplete_out = nullptr) {  // sync: *cc.incomplete, read with the overflow count
  const int64_t xrows = rup(nx_max, BM), yrows = rup(ny_all, BN);
  cudaMemsetAsync(w.ymax, 0, 4 * sizeof(unsigned), st);
  cudaMemsetAsync(w.n_overflow, 0, sizeof(int32_t), st);
  prep_tiles<T><<<grid_for(xrows, 8), 256, 0, st>>>(X, x_idx, n_x, 0, xrows, BMH, w.xt, w.xinfo, nullptr, 0, BM);
  PS_LAUNCHED("prep_tiles(X)");
  prep_tiles<T><<<grid_for(yrows, 8), 256, 0, st>>>(Y, y_idx, n_y, 0, yrows, BN, w.yt, w.yinfo, w.ymax, 1, BN);
  PS_LAUNCHED("prep_tiles(Y)");
  // the attribute is per device: set it on every call (cheap, idempotent, thread-safe)
  cudaFuncSetAttribute(nn_topk_tc<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<0>());
  cudaFuncSetAttribute(nn_topk_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<1>());
  // the counts size the grids; a caller that already knows one passes it in (>= 0)
  int64_t nx = nx_io && *nx_io >= 0 ? *nx_io : -1, ny = ny_io && *ny_io >= 0 ? *ny_io : -1;
  if (!sync) {  // no host round trip: grids sized by the upper bounds, the kernels read the device counts
    nx = nx_max;
    ny = ny_all;
  } else if (nx < 0 && ny < 0) read_counts(n_x, n_y, &nx, &ny, st);
  else if (nx < 0) nx = read_count(n_x, st);
  else if (ny < 0) ny = read_count(n_y, st);
  if (nx_io && sync) *nx_io = nx;
  if (ny_io && sync) *ny_io = ny;
  if (nx <= 0) return PS_OK;
  const dim3 g0 = tc_grid(nx, ny, !sync);
  const int64_t flops_tile = 2ll * BM * BN * KD;
  if (sync) g_stats[5] += (int64_t)g0.x * ((ny + BN - 1) / BN) * flops_tile;
  nn_topk_tc<0><<<g0, kThreads, smem_bytes<0>(), st>>>(w.xt, w.yt, n_x, n_y, w.topv, w.topj, nullptr, nullptr,
                                                      nullptr, 0);
  PS_LAUNCHED("nn_topk_tc<top4>");
  certify_exact<T><<<grid_for(nx, 32), 256, 0, st>>>(w.topv, w.topj, n_x, x_idx, y_idx, w.xinfo, w.ymax, X, Y, nn,
                                                      dist, w.overflow, w.n_overflow, w.lim, kParts * (int)g0.y,
                                                      (int64_t)g0.x * BM, cc);
  PS_LAUNCHED("certify_exact");
  // rows with more near-tied candidates than the top-4: enumerate every
  // column within their certified limit on the tensor cores, then decide exactly
  gather_rows<<<grid_for(nx_max, 256), 256, 0, st>>>(w.overflow, w.n_overflow, x_idx, w.xsrc);
  PS_LAUNCHED("gather_rows");
  // operand tiles of the overflow rows: the enumeration reads at most the
  // first kEnumBlocksAsync row blocks without a host count (async), all of
  // them with one (sync; rows beyond take the exact scan either way)
  int64_t n_over = -1;
  if (sync && cc.cbits && incomplete_out) {  // one synchronisation for both
    int64_t inc = 0;
    read_counts(w.n_overflow, cc.incomplete, &n_over, &inc, st);
    *incomplete_out = (int32_t)inc;
  } else if (sync) {
    n_over = read_count(w.n_overflow, st);
  }
  const int64_t over_rows = sync ? rup(n_over, BM) : std::min<int64_t>(xrows, (int64_t)kEnumBlocksAsync * BM);
  if (over_rows > 0) {
    prep_tiles<T><<<grid_for(over_rows, 8), 256, 0, st>>>(X, w.xsrc, w.n_overflow, 0, over_rows, BMH, w.xt, w.xinfo,
                                                          nullptr, 0, BM);
    PS_LAUNCHED("prep_tiles(overflow)");
  }
  cudaMemsetAsync(w.n_pairs, 0, sizeof(unsigned long long), st);
  cudaMemsetAsync(w.best_bits, 0xff, nx_max * sizeof(unsigned long long), st);
  cudaMemsetAsync(w.best_j, 0x7f, nx_max * sizeof(int32_t), st);
  int enum_rows = INT32_MAX;
  if (sync) {
    g_stats[3] += n_over;
    if (n_over > 0) {
      g_stats[5] += (int64_t)tc_grid(n_over, ny).x * ((ny + BN - 1) / BN) * flops_tile;
      nn_topk_tc<1><<<tc_grid(n_over, ny), kThreads, smem_bytes<1>(), st>>>(w.xt, w.yt, w.n_overflow, n_y, nullptr,
                                                                            nullptr, w.lim, w.pairs, w.n_pairs,
                                                                            w.pair_cap);
      PS_LAUNCHED("nn_topk_tc<enumerate>");
    }
  } else {
    // the overflow count is unknown on the host: a grid for every row, each
    // row block beyond *n_overflow exits at once; the few live row blocks get
    // the widest column split (near-ties are rare, so they are few)
    const int tiles = (int)std::max<int64_t>(1, (ny + BN - 1) / BN);
    const dim3 ge((unsigned)std::min<int64_t>(kEnumBlocksAsync, (nx + BM - 1) / BM), (unsigned)std::min(kMaxSplit, tiles));
    enum_rows = (int)ge.x * BM;  // overflow rows beyond these take the exact scan
    nn_topk_tc<1><<<ge, kThreads, smem_bytes<1>(), st>>>(w.xt, w.yt, w.n_overflow, n_y, nullptr, nullptr, w.lim,
                                                         w.pairs, w.n_pairs, w.pair_cap);
    PS_LAUNCHED("nn_topk_tc<enumerate>");
  }
  if (enum_rows_out) *enum_rows_out = enum_rows;
  pair_dist_min<T><<<148 * 16, 256, 0, st>>>(w.pairs, w.n_pairs, w.pair_cap, w.xsrc, y_idx, X, Y, w.pd, w.best_bits,
                                             cc);
  PS_LAUNCHED("pair_dist_min");
  pair_argmin<T><<<148 * 8, 256, 0, st>>>(w.pairs, w.n_pairs, w.pair_cap, y_idx, w.pd, w.best_bits, w.best_j,
                                          w.xsrc, cc);
  PS_LAUNCHED("pair_argmin");
  if (cc.cbits) {
    cand_argmin<<<148 * 4, 256, 0, st>>>(cc);
    PS_LAUNCHED("cand_argmin");
  }
  pair_write<<<grid_for(nx_max, 256), 256, 0, st>>>(w.n_overflow, w.xsrc, w.best_bits, w.best_j, nn, dist,
                                                     enum_rows);
  PS_LAUNCHED("pair_write");
  exact_rows<T><<<148 * 4, 256, 0, st>>>(w.overflow, w.n_overflow, x_idx, X, Y, ny_all, nn, dist, w.n_pairs,
                                         w.pair_cap, enum_rows);
  PS_LAUNCHED("exact_rows");
  return PS_OK;
}

// ---- many pairs, one launch sequence ---------------------------------------------------
// ps_match_batch_async: P (set a, set b) nearest_neighbor matches over S
// descriptor sets as ONE sequence of ~35 launches (blockIdx.y / .z = pair, or
// set for the per-set stages) instead of ~45 per pair.  Each set is hashed,
// grouped and turned into operand tiles once however many pairs it enters (in
// a 3 x 3 stitch every image is in 8 pairs): its X-form tiles serve the pairs'
// row passes, its Y-form tiles both passes.  Per pair the stages are those of
// nearest_pass in asynchronous mode, through the same kernel bodies, so every
// pair's result equals ps_match_async's (the mosaic loop the batch replaces:
// reference mosaic.py:79-112 calling match_features, matcher.py:57-95).
constexpr int kBatchMaxSets = 512;
constexpr int kBatchMaxPairs = 256;

template <class T>
struct BatchIn {  // kernel parameter (__grid_constant__): the sets and the pair list
  const T* desc[kBatchMaxSets];
  int32_t rows[kBatchMaxSets];  // capacity (grids, workspace)
  const int32_t* cnt[kBatchMaxSets];  // optional device row count (<= rows): the kernels use min(rows, *cnt)
  uint8_t role[kBatchMaxSets];  // bit 0: set a of some pair (X-form tiles), bit 1: set b of some pair
  int16_t pa[kBatchMaxPairs], pb[kBatchMaxPairs];
};

struct BatchWs {  // uniform slots: set s / pair q at base + s (q) * stride
  int64_t n, xrows, yrows, tsize, nchunk, lists, pair_cap, over_rows;
  int32_t *slot_of, *rep, *flag, *uniq, *n_uniq, *sel_cnt;  // per set (sel_cnt: per set or pair)
  unsigned long long* tkey;
  int32_t* tidx;
  uint8_t *xt, *yt;
  double *xinfo, *yinfo;
  unsigned* ymax;
  float* topv;  // per pair from here
  int32_t* topj;
  int32_t *nn12, *nn21, *colflag, *cols, *n_cols, *overflow, *n_overflow, *xsrc, *best_j;
  double *d12, *d21, *xinfo2, *xinfoo, *pd;
  uint8_t *xt2, *xto;
  float* lim;
  unsigned long long *best_bits, *pairs, *n_pairs, *kp, *kd, *counter;
  unsigned long long *cand, *n_cand, *cbits;  // pass 0's column candidates per pair (ColCand)
  double* cpd;
  int32_t* cand_incomplete;
  int64_t cand_cap;
};

constexpr int kSelChunk = 2048;  // flags per selection CTA (256 threads x 8)

BatchWs carve_batch(void* base, int64_t S, int64_t P, int64_t n, size_t* used) {
  Arena ar{(char*)base, 0, 0};
  BatchWs w{};
  const int64_t N = std::max<int64_t>(n, 1);
  w.n = N;
  w.xrows = rup(N, BM);
  w.yrows = rup(N, BN);
  w.tsize = 64;
  while (w.tsize < 2 * N) w.tsize <<= 1;
  w.nchunk = (N + kSelChunk - 1) / kSelChunk;
  w.lists = kParts * kMaxSplit;
  w.pair_cap = std::max<int64_t>(1 << 16, 4 * N);
  w.over_rows = std::min<int64_t>(w.xrows, (int64_t)kEnumBlocksAsync * BM);
  w.slot_of = ar.take<int32_t>(S * N);
  w.rep = ar.take<int32_t>(S * N);
  w.flag = ar.take<int32_t>(S * N);
  w.uniq = ar.take<int32_t>(S * N);
  w.n_uniq = ar.take<int32_t>(S);
  w.sel_cnt = ar.take<int32_t>(std::max(S, P) * w.nchunk);
  w.tkey = ar.take<unsigned long long>(S * w.tsize);
  w.tidx = ar.take<int32_t>(S * w.tsize);
  w.xt = ar.take<uint8_t>(S * w.xrows * ROW_BYTES);
  w.xinfo = ar.take<double>(S * 3 * w.xrows);
  w.yt = ar.take<uint8_t>(S * w.yrows * ROW_BYTES);
  w.ymax = ar.take<unsigned>(S * 4);
  w.topv = ar.take<float>(P * w.lists * w.xrows * TOPK);
  w.topj = ar.take<int32_t>(P * w.lists * w.xrows * TOPK);
  w.nn12 = ar.take<int32_t>(P * N);
  w.nn21 = ar.take<int32_t>(P * N);
  w.colflag = ar.take<int32_t>(P * N);
  w.cols = ar.take<int32_t>(P * N);
  w.n_cols = ar.take<int32_t>(P);
  w.overflow = ar.take<int32_t>(P * N);
  w.n_overflow = ar.take<int32_t>(2 * P);
  w.xsrc = ar.take<int32_t>(P * N);
  w.best_j = ar.take<int32_t>(P * N);
  w.d12 = ar.take<double>(P * N);
  w.d21 = ar.take<double>(P * N);
  w.xt2 = ar.take<uint8_t>(P * w.xrows * ROW_BYTES);
  w.xinfo2 = ar.take<double>(P * 3 * w.xrows);
  w.xto = ar.take<uint8_t>(P * w.over_rows * ROW_BYTES);
  w.xinfoo = ar.take<double>(P * 3 * w.over_rows);
  w.lim = ar.take<float>(P * w.xrows);
  w.best_bits = ar.take<unsigned long long>(P * N);
  w.pairs = ar.take<unsigned long long>(P * w.pair_cap);
  w.pd = ar.take<double>(P * w.pair_cap);
  w.n_pairs = ar.take<unsigned long long>(2 * P);
  w.kp = ar.take<unsigned long long>(P * N);
  w.kd = ar.take<unsigned long long>(P * N);
  w.counter = ar.take<unsigned long long>(P);
  w.cand_cap = std::max<int64_t>(1 << 14, 4 * N);
  w.cand = ar.take<unsigned long long>(P * w.cand_cap);
  w.cpd = ar.take<double>(P * w.cand_cap);
  w.n_cand = ar.take<unsigned long long>(P);
  w.cand_incomplete = ar.take<int32_t>(P);
  w.cbits = ar.take<unsigned long long>(P * N);
  *used = ar.used + 256;
  return w;
}

// rows of set s the kernels work on: its device count when given (a graph
// replayed on new frames sees the new counts), else the host row count
template <class T>
__device__ __forceinline__ int64_t set_n(const BatchIn<T>& in, int64_t s) {
  const int64_t cap = in.rows[s];
  return in.cnt[s] ? max((int64_t)0, min(cap, (int64_t)__ldg(in.cnt[s]))) : cap;
}

template <class T>
struct PassView {  // pair q in pass 0 (distinct rows of a vs b) or 1 (matchable columns of b vs a)
  const T *X, *Y;
  const int32_t *x_idx, *n_x, *y_idx, *n_y;
  const uint8_t *xt, *yt;
  const double* xinfo;
  const unsigned* ymax;
  int32_t* nn;
  double* dist;
  int64_t ny;
};

template <class T>
__device__ __forceinline__ PassView<T> pass_view(const BatchIn<T>& in, const BatchWs& w, int q, int pass) {
  const int sa = in.pa[q], sb = in.pb[q];
  const int64_t xs = pass ? sb : sa, ys = pass ? sa : sb, qq = q;
  PassView<T> v;
  v.X = in.desc[xs];
  v.Y = in.desc[ys];
  v.x_idx = pass ? w.cols + qq * w.n : w.uniq + xs * w.n;
  v.n_x = pass ? w.n_cols + qq : w.n_uniq + xs;
  v.y_idx = w.uniq + ys * w.n;
  v.n_y = w.n_uniq + ys;
  v.xt = pass ? w.xt2 + qq * w.xrows * ROW_BYTES : w.xt + xs * w.xrows * ROW_BYTES;
  v.xinfo = pass ? w.xinfo2 + qq * 3 * w.xrows : w.xinfo + xs * 3 * w.xrows;
  v.yt = w.yt + ys * w.yrows * ROW_BYTES;
  v.ymax = w.ymax + 4 * ys;
  v.nn = (pass ? w.nn21 : w.nn12) + qq * w.n;
  v.dist = (pass ? w.d21 : w.d12) + qq * w.n;
  v.ny = set_n(in, ys);
  return v;
}

// per-set stages (blockIdx.y = set; sets in no pair are skipped).  A
// half-warp owns a row (lane hl: elements 8 hl .. 8 hl + 7, two 16-byte
// loads), so a warp keeps two rows' loads and reductions in flight.
template <class T>
__device__ __forceinline__ void load8(const T* __restrict__ row, int hl, double (&x)[8]) {
  if constexpr (sizeof(T) == 4) {
    const float4 v0 = __ldg(reinterpret_cast<const float4*>(row) + 2 * hl);
    const float4 v1 = __ldg(reinterpret_cast<const float4*>(row) + 2 * hl + 1);
    x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
    x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(row) + 4 * hl + k);
      x[2 * k] = v.x;
      x[2 * k + 1] = v.y;
    }
  }
}

// The table inserts with a half-warp per row (the key: a sum over the row's words).
// Each half-warp walks a contiguous run of rows two at a time, so "identical
// to the previous row" is tested on the hash keys it already holds: a row
// whose key equals its predecessor's skips the minimum update (the run's
// first row, the smallest index with that key in the run, competes; equal
// keys share a slot, so every slot still receives the smallest index of
// its key) -- one row load per row instead of two.
// The row key from the row's raw 32-bit words (no float <-> double conversions, one 32 x 32 -> 64
// multiply-add per word and one avalanche per lane; with three 64-bit multiplies per element
// b_hash was ALU-bound at 1.6 TB/s).  Any key function is exact here -- a collision only splits a
// group (mark_reps compares the rows) -- so only its cost and spread matter.
template <class T>
__device__ __forceinline__ unsigned long long row_hash_words(const T* __restrict__ row, int hl, unsigned hmask) {
  constexpr int W = (int)sizeof(T) * 2;  // 32-bit words of this lane's 8 elements
  const uint4* p = reinterpret_cast<const uint4*>(row) + hl * (W / 4);
  unsigned long long h = 0;
#pragma unroll
  for (int q = 0; q < W / 4; ++q) {
    const uint4 w = __ldg(p + q);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t c = (0x9E3779B1u * (uint32_t)(hl * W + 4 * q + e + 1)) | 1u;  // per-position odd multiplier
      const uint32_t x = ws[e] ^ __funnelshift_l(ws[e], ws[e], 15);
      h += (unsigned long long)x * c + (unsigned long long)(x >> 7);
    }
  }
  h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
  h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
  h ^= h >> 31;
#pragma unroll
  for (int o = 8; o; o >>= 1) h += __shfl_xor_sync(hmask, h, o);
  return h | 1ull;  // 0 marks an empty slot
}

__device__ __forceinline__ void hash_put(unsigned long long key, bool compete, int64_t i,
                                         unsigned long long* __restrict__ tkey, int32_t* __restrict__ tidx,
                                         int64_t tsize, int32_t* __restrict__ slot_of) {
  int64_t slot = (int64_t)((key >> 20) & (unsigned long long)(tsize - 1));
  for (;;) {  // plain read first: duplicate rows find their slot without an atomic
    unsigned long long prev = *(volatile unsigned long long*)(tkey + slot);
    if (prev == 0ull) prev = atomicCAS(tkey + slot, 0ull, key);
    if (prev == 0ull || prev == key) break;
    slot = (slot + 1) & (tsize - 1);
  }
  if (compete && *(volatile int32_t*)(tidx + slot) > (int32_t)i) atomicMin(tidx + slot, (int32_t)i);
  slot_of[i] = (int32_t)slot;
}

// Row keys into the open-addressing table, a half-warp per row (the grid's x dimension walks the rows)
template <class T>
__device__ __forceinline__ void hash_rows_body(const T* __restrict__ X, int64_t n, unsigned long long* __restrict__ tkey,
                                               int32_t* __restrict__ tidx, int64_t tsize,
                                               int32_t* __restrict__ slot_of) {
  const int hl = threadIdx.x & 15;
  const unsigned hmask = (threadIdx.x & 16) ? 0xffff0000u : 0x0000ffffu;
  const int64_t halves = (int64_t)gridDim.x * (blockDim.x >> 4);
  const int64_t hw = (int64_t)blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4);
  const int64_t run = (n + halves - 1) / halves;
  const int64_t i0 = hw * run, i1 = min(n, i0 + run);
  if (i0 >= i1) return;  // uniform per half-warp
  unsigned long long prev = 0ull;  // key of row i0 - 1 (none: 0 never equals a key)
  if (i0 > 0) prev = row_hash_words<T>(X + (i0 - 1) * KD, hl, hmask);
  // 16 rows' keys per round (lane k keeps row base + k's), then the 16 table
  // inserts run in parallel, one per lane
  const int hbase = threadIdx.x & 16;
  for (int64_t base = i0; base < i1; base += 16) {
    const int m = (int)min((int64_t)16, i1 - base);
    unsigned long long mine = 0ull;
#pragma unroll 4
    for (int k = 0; k < m; ++k) {
      const unsigned long long key = row_hash_words<T>(X + (base + k) * KD, hl, hmask);
      if (hl == k) mine = key;
    }
    unsigned long long before = __shfl_sync(hmask, mine, hbase + ((hl + 15) & 15));
    if (hl == 0) before = prev;
    if (hl < m) hash_put(mine, mine != before, base + hl, tkey, tidx, tsize, slot_of);
    prev = __shfl_sync(hmask, mine, hbase + m - 1);
  }
}


template <class T>
__global__ void b_hash(const __grid_constant__ BatchIn<T> in, const BatchWs w) {
  const int64_t s = blockIdx.y;
  if (!in.role[s]) return;
  hash_rows_body<T>(in.desc[s], set_n(in, s), w.tkey + s * w.tsize, w.tidx + s * w.tsize, w.tsize,
                    w.slot_of + s * w.n);
}
template <class T>
__global__ void hash_rows(const T* __restrict__ X, int64_t n, unsigned long long* __restrict__ tkey,
                          int32_t* __restrict__ tidx, int64_t tsize, int32_t* __restrict__ slot_of) {
  hash_rows_body<T>(X, n, tkey, tidx, tsize, slot_of);
}

template <class T>
__global__ void b_reps(const __grid_constant__ BatchIn<T> in, const BatchWs w) {
  const int64_t s = blockIdx.y;
  if (!in.role[s]) return;
  mark_reps_table_body<T>(in.desc[s], set_n(in, s), w.tidx + s * w.tsize, w.slot_of + s * w.n, w.rep + s * w.n,
                          w.flag + s * w.n);
}

__device__ __forceinline__ int64_t rup_dev(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// Both operand forms of a set's distinct rows from one read (prep_tiles'
// arithmetic): the Y-form tiles (every set in a pair), the X-form tiles (sets
// that are some pair's set a), the row norms (xinfo) and the Y maxima.
template <class T>
__global__ void b_prep_sets(const __grid_constant__ BatchIn<T> in, const BatchWs w) {
  const int64_t s = blockIdx.y;
  const int role = in.role[s];
  if (!role) return;  // uniform per block
  const bool want_x = role & 1;
  const T* src = in.desc[s];
  const int32_t* idx = w.uniq + s * w.n;
  const int64_t count = w.n_uniq[s];
  uint8_t* xt = w.xt + s * w.xrows * ROW_BYTES;
  uint8_t* yt = w.yt + s * w.yrows * ROW_BYTES;
  double* info = w.xinfo + s * 3 * w.xrows;
  const int64_t n_used_y = min(w.yrows, rup_dev(count, BN)), n_used_x = min(w.xrows, rup_dev(count, BM));
  const int hl = threadIdx.x & 15;
  const unsigned hmask = (threadIdx.x & 16) ? 0xffff0000u : 0x0000ffffu;
  float mx0 = 0.0f, mx1 = 0.0f, mx2 = 0.0f;
  for (int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4); u < n_used_y;
       u += (int64_t)gridDim.x * (blockDim.x >> 4)) {
    const bool live = u < count;
    double x[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (live) load8(src + (int64_t)idx[u] * KD, hl, x);
    __half h[8];
    double sx = 0.0, sr = 0.0, sh = 0.0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      h[e] = __double2half(x[e]);
      const double hv = (double)__half2float(h[e]);
      const double rv = x[e] - hv;
      sx += x[e] * x[e];
      sr += rv * rv;
      sh += hv * hv;
    }
#pragma unroll
    for (int o = 8; o; o >>= 1) {
      sx += __shfl_xor_sync(hmask, sx, o);
      sr += __shfl_xor_sync(hmask, sr, o);
      sh += __shfl_xor_sync(hmask, sh, o);
    }
    uint4 px, py;  // 8 fp16: x_h (X form) and -2 x_h (Y form, exact)
    {
      __half2 p[4], q[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        p[k] = __halves2half2(h[2 * k], h[2 * k + 1]);
        q[k] = __hmul2(p[k], __float2half2_rn(-2.0f));
      }
      px = make_uint4(*reinterpret_cast<uint32_t*>(&p[0]), *reinterpret_cast<uint32_t*>(&p[1]),
                      *reinterpret_cast<uint32_t*>(&p[2]), *reinterpret_cast<uint32_t*>(&p[3]));
      py = make_uint4(*reinterpret_cast<uint32_t*>(&q[0]), *reinterpret_cast<uint32_t*>(&q[1]),
                      *reinterpret_cast<uint32_t*>(&q[2]), *reinterpret_cast<uint32_t*>(&q[3]));
    }
    {  // Y form
      const int64_t tile = u / BN;
      const int r = (int)(u % BN);
      uint8_t* base = yt + tile * (int64_t)BN * ROW_BYTES;
      *reinterpret_cast<uint4*>(base + sw128_offset(BN, r, hl * 8)) = py;
      if (hl < 2) {
        uint4 q = make_uint4(0u, 0u, 0u, 0u);
        if (hl == 0) {
          __half a0, a1, a2;
          if (!live) {
            a0 = __float2half(INFINITY);
            a1 = a2 = __float2half(0.0f);
          } else {
            a0 = __double2half(sx);
            const double r1 = __hisinf(a0) ? 0.0 : sx - (double)__half2float(a0);
            a1 = __double2half(r1);
            a2 = __double2half(r1 - (double)__half2float(a1));
          }
          const __half2 q0 = __halves2half2(a0, a1), q1 = __halves2half2(a2, __float2half(0.0f));
          q.x = *reinterpret_cast<const uint32_t*>(&q0);
          q.y = *reinterpret_cast<const uint32_t*>(&q1);
        }
        *reinterpret_cast<uint4*>(base + BN * KD * 2 + (r >> 3) * 256 + hl * 128 + (r & 7) * 16) = q;
      }
    }
    if (want_x && u < n_used_x) {  // X form
      const int64_t tile = u / BMH;
      const int r = (int)(u % BMH);
      uint8_t* base = xt + tile * (int64_t)BMH * ROW_BYTES;
      *reinterpret_cast<uint4*>(base + sw128_offset(BMH, r, hl * 8)) = px;
      if (hl < 2) {
        uint4 q = make_uint4(0u, 0u, 0u, 0u);
        if (hl == 0) {
          const __half2 one = __float2half2_rn(1.0f), q1 = __halves2half2(__float2half(1.0f), __float2half(0.0f));
          q.x = *reinterpret_cast<const uint32_t*>(&one);
          q.y = *reinterpret_cast<const uint32_t*>(&q1);
        }
        *reinterpret_cast<uint4*>(base + BMH * KD * 2 + (r >> 3) * 256 + hl * 128 + (r & 7) * 16) = q;
      }
    }
    if (hl == 0 && live) {
      info[3 * u + 0] = sqrt(sx);
      info[3 * u + 1] = sqrt(sr);
      info[3 * u + 2] = sqrt(sh);
      mx0 = nan_max(mx0, (float)(sqrt(sx) * (1.0 + 1e-6)));
      mx1 = nan_max(mx1, (float)(sqrt(sr) * (1.0 + 1e-6)));
      mx2 = nan_max(mx2, (float)(sqrt(sh) * (1.0 + 1e-6)));
    }
  }
  __shared__ float smx[3][64];
  const int hw = threadIdx.x >> 4, nh = blockDim.x >> 4;
  if (hl == 0) { smx[0][hw] = mx0; smx[1][hw] = mx1; smx[2][hw] = mx2; }
  __syncthreads();
  if (threadIdx.x < 3) {
    float m = 0.0f;
    for (int k = 0; k < nh; ++k) m = nan_max(m, smx[threadIdx.x][k]);
    if (m != 0.0f) atomicMax(w.ymax + 4 * s + threadIdx.x, __float_as_uint(m));
  }
}

// Order-preserving selection of the flagged indices of every segment in two
// launches: segment g = the flags of set g (SEG 0: its representatives) or of
// pair g's columns (SEG 1), length rows[g] / rows[pb[g]].
template <class T, int SEG>
__device__ __forceinline__ int64_t seg_len(const BatchIn<T>& in, int g) {
  return SEG == 0 ? (in.role[g] ? set_n(in, g) : 0) : set_n(in, in.pb[g]);
}

__device__ __forceinline__ int block_sum256(int v, int* sh) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) t += sh[k];
  __syncthreads();
  return t;
}

template <class T, int SEG>
__global__ void __launch_bounds__(256) b_sel_count(const __grid_constant__ BatchIn<T> in,
                                                   const int32_t* __restrict__ flag, int64_t stride,
                                                   int32_t* __restrict__ cnt, int64_t nchunk) {
  __shared__ int sh[8];
  const int g = blockIdx.y;
  const int64_t len = seg_len<T, SEG>(in, g), c0 = (int64_t)blockIdx.x * kSelChunk;
  if (c0 >= len) return;
  const int32_t* f = flag + (int64_t)g * stride;
  const int64_t c1 = min(len, c0 + kSelChunk);
  int k = 0;
  for (int64_t i = c0 + threadIdx.x; i < c1; i += 256) k += f[i] != 0;
  k = block_sum256(k, sh);
  if (threadIdx.x == 0) cnt[(int64_t)g * nchunk + blockIdx.x] = k;
}

template <class T, int SEG>
__global__ void __launch_bounds__(256) b_sel_scatter(const __grid_constant__ BatchIn<T> in,
                                                     const int32_t* __restrict__ flag, int64_t stride,
                                                     const int32_t* __restrict__ cnt, int64_t nchunk,
                                                     int32_t* __restrict__ out, int32_t* __restrict__ n_out) {
  __shared__ int sh[8], wsum[8];
  const int g = blockIdx.y;
  const int64_t len = seg_len<T, SEG>(in, g), c0 = (int64_t)blockIdx.x * kSelChunk;
  if (c0 >= len) {
    if (blockIdx.x == 0 && threadIdx.x == 0) n_out[g] = 0;
    return;
  }
  int b = 0;  // flagged entries of the segment's earlier chunks
  for (int c = threadIdx.x; c < (int)blockIdx.x; c += 256) b += cnt[(int64_t)g * nchunk + c];
  int base = block_sum256(b, sh);
  const int32_t* f = flag + (int64_t)g * stride;
  int32_t* o = out + (int64_t)g * stride;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t c1 = min(len, c0 + kSelChunk);
  for (int64_t i0 = c0; i0 < c1; i0 += 256) {  // block-uniform trip count
    const int64_t i = i0 + threadIdx.x;
    const bool p = i < c1 && f[i] != 0;
    const unsigned m = __ballot_sync(0xffffffffu, p);
    if (lane == 0) wsum[wid] = __popc(m);
    __syncthreads();
    int pre = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int x = wsum[k];
      pre += k < wid ? x : 0;
      tot += x;
    }
    if (p) o[base + pre + __popc(m & ((1u << lane) - 1u))] = (int32_t)i;
    base += tot;
    __syncthreads();
  }
  if (c1 == len && threadIdx.x == 0) n_out[g] = base;
}

// pair q's column candidates (pass 0 only)
__device__ __forceinline__ ColCand col_cand(const BatchWs& w, int64_t q, int pass, double delta_s) {
  if (pass) return ColCand{};
  return ColCand{delta_s, w.cand_incomplete + q, w.cbits + q * w.n, w.nn21 + q * w.n, w.cand + q * w.cand_cap, w.cpd + q * w.cand_cap,
                 w.n_cand + q};
}

// per-pair stages (blockIdx.y = pair; the tensor-core kernel: blockIdx.z)
__global__ void b_init(int P, const BatchWs w) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= P) return;
  w.n_overflow[2 * q] = w.n_overflow[2 * q + 1] = 0;
  w.n_pairs[2 * q] = w.n_pairs[2 * q + 1] = 0ull;
  w.counter[q] = 0ull;
  w.n_cand[q] = 0ull;
  w.cand_incomplete[q] = 0;
}

template <int MODE, class T>
__global__ void __launch_bounds__(kThreads, 1) b_topk(const __grid_constant__ BatchIn<T> in, const BatchWs w,
                                                      int pass) {
  const int64_t q = blockIdx.z;
  const PassView<T> v = pass_view(in, w, (int)q, pass);
  if (MODE == 0)
    nn_topk_tc_body<0>(v.xt, v.yt, v.n_x, v.n_y, w.topv + q * w.lists * w.xrows * TOPK,
                       w.topj + q * w.lists * w.xrows * TOPK, nullptr, nullptr, nullptr, 0);
  else
    nn_topk_tc_body<1>(w.xto + q * w.over_rows * ROW_BYTES, v.yt, w.n_overflow + 2 * q + pass, v.n_y, nullptr,
                       nullptr, w.lim + q * w.xrows, w.pairs + q * w.pair_cap, w.n_pairs + 2 * q + pass,
                       w.pair_cap);
}

template <class T>
__global__ void b_certify(const __grid_constant__ BatchIn<T> in, const BatchWs w, int pass, int n_lists,
                          int64_t nx_pad, double delta_s) {
  const int64_t q = blockIdx.y;
  const PassView<T> v = pass_view(in, w, (int)q, pass);
  certify_exact_body<T>(w.topv + q * w.lists * w.xrows * TOPK, w.topj + q * w.lists * w.xrows * TOPK, v.n_x, v.x_idx,
                        v.y_idx, v.xinfo, v.ymax, v.X, v.Y, v.nn, v.dist, w.overflow + q * w.n,
                        w.n_overflow + 2 * q + pass, w.lim + q * w.xrows, n_lists, nx_pad,
                        col_cand(w, q, pass, delta_s));
}

// overflow rows -> source rows, and their enumeration minima reset
template <class T>
__global__ void b_gather(const __grid_constant__ BatchIn<T> in, const BatchWs w, int pass) {
  const int64_t q = blockIdx.y;
  const PassView<T> v = pass_view(in, w, (int)q, pass);
  const int32_t* ov = w.overflow + q * w.n;
  const int n = w.n_overflow[2 * q + pass];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    w.xsrc[q * w.n + k] = v.x_idx[ov[k]];
    w.best_bits[q * w.n + k] = ~0ull;
    w.best_j[q * w.n + k] = 0x7f7f7f7f;
  }
}

template <class T>
__global__ void b_prep_rows(const __grid_constant__ BatchIn<T> in, const BatchWs w, int pass, int over) {
  const int64_t q = blockIdx.y;
  if (over) {  // the overflow rows' X tiles (pair-private)
    const PassView<T> v = pass_view(in, w, (int)q, pass);
    prep_tiles_body<T>(v.X, w.xsrc + q * w.n, w.n_overflow + 2 * q + pass, 0, w.over_rows, BMH,
                       w.xto + q * w.over_rows * ROW_BYTES, w.xinfoo + q * 3 * w.over_rows, nullptr, 0, BM);
  } else {  // pass 1's X tiles: the pair's matchable columns of b
    prep_tiles_body<T>(in.desc[in.pb[q]], w.cols + q * w.n, w.n_cols + q, 0, w.xrows, BMH,
                       w.xt2 + q * w.xrows * ROW_BYTES, w.xinfo2 + q * 3 * w.xrows, nullptr, 0, BM);
  }
}

template <class T>
__global__ void b_pair_dist_min(const __grid_constant__ BatchIn<T> in, const BatchWs w, int pass, double delta_s) {
  const int64_t q = blockIdx.y;
  const PassView<T> v = pass_view(in, w, (int)q, pass);
  pair_dist_min_body<T>(w.pairs + q * w.pair_cap, w.n_pairs + 2 * q + pass, w.pair_cap, w.xsrc + q * w.n, v.y_idx,
                        v.X, v.Y, w.pd + q * w.pair_cap, w.best_bits + q * w.n, col_cand(w, q, pass, delta_s));
}

template <class T>
__global__ void b_pair_argmin(const __grid_constant__ BatchIn<T> in, const BatchWs w, int pass, double delta_s) {
  const int64_t q = blockIdx.y;
  const PassView<T> v = pass_view(in, w, (int)q, pass);
  pair_argmin_body<T>(w.pairs + q * w.pair_cap, w.n_pairs + 2 * q + pass, w.pair_cap, v.y_idx, w.pd + q * w.pair_cap,
                      w.best_bits + q * w.n, w.best_j + q * w.n, w.xsrc + q * w.n, col_cand(w, q, pass, delta_s));
  cand_argmin_body(col_cand(w, q, pass, delta_s));  // certify's list: the column minima are final here
}

template <class T>
__global__ void b_pair_write(const __grid_constant__ BatchIn<T> in, const BatchWs w, int pass, int enum_rows) {
  const int64_t q = blockIdx.y;
  const PassView<T> v = pass_view(in, w, (int)q, pass);
  pair_write_body(w.n_overflow + 2 * q + pass, w.xsrc + q * w.n, w.best_bits + q * w.n, w.best_j + q * w.n, v.nn,
                  v.dist, enum_rows);
}

template <class T>
__global__ void b_exact_rows(const __grid_constant__ BatchIn<T> in, const BatchWs w, int pass, int enum_rows) {
  const int64_t q = blockIdx.y;
  const PassView<T> v = pass_view(in, w, (int)q, pass);
  exact_rows_body<T>(w.overflow + q * w.n, w.n_overflow + 2 * q + pass, v.x_idx, v.X, v.Y, v.ny, v.nn, v.dist,
                     w.n_pairs + 2 * q + pass, w.pair_cap, enum_rows);
}

template <class T>
__global__ void b_mark_columns(const __grid_constant__ BatchIn<T> in, const BatchWs w, double delta_s, int enum_rows) {
  const int64_t q = blockIdx.y, sa = in.pa[q];
  mark_columns_body(w.uniq + sa * w.n, w.n_uniq + sa, w.nn12 + q * w.n, w.d12 + q * w.n, delta_s,
                    w.colflag + q * w.n, w.n_overflow + 2 * q, enum_rows, w.n_pairs + 2 * q, w.pair_cap,
                    w.cand_incomplete + q);
}

template <class T>
__global__ void b_accept(const __grid_constant__ BatchIn<T> in, const BatchWs w, double delta_s) {
  const int64_t q = blockIdx.y, sa = in.pa[q];
  accept_pairs_body(w.rep + sa * w.n, set_n(in, sa), w.nn12 + q * w.n, w.d12 + q * w.n, w.nn21 + q * w.n, delta_s,
                    w.kp + q * w.n, w.kd + q * w.n, w.counter + q);
}

// Accepted pairs sorted by (delta, ref1, ref2) by ranking (pair keys are
// unique, so ranks are a permutation) and written straight to the outputs
// (a pair's accepted count is at most min(n1, n2) <= the output stride).
constexpr int kBRankTile = 1024;
constexpr int kBRankLanes = 8;
__global__ void __launch_bounds__(256) b_rank_out(const BatchWs w, int64_t stride, int32_t* __restrict__ ref1,
                                                  int32_t* __restrict__ ref2, double* __restrict__ delta,
                                                  int64_t* __restrict__ out_count) {
  __shared__ unsigned long long td[kBRankTile], tp[kBRankTile];
  constexpr int kPerBlock = 256 / kBRankLanes;
  const int64_t q = blockIdx.y;
  const unsigned long long c = w.counter[q];
  if (blockIdx.x == 0 && threadIdx.x == 0) out_count[q] = (int64_t)c;
  const int n = (int)min((unsigned long long)stride, c);
  if ((int)(blockIdx.x * kPerBlock) >= n) return;  // uniform per block
  const unsigned long long* kd = w.kd + q * w.n;
  const unsigned long long* kp = w.kp + q * w.n;
  const int g = threadIdx.x & (kBRankLanes - 1);
  const int e = blockIdx.x * kPerBlock + threadIdx.x / kBRankLanes;
  const unsigned long long d = e < n ? kd[e] : 0ull, p = e < n ? kp[e] : 0ull;
  int rank = 0;
  for (int t0 = 0; t0 < n; t0 += kBRankTile) {
    __syncthreads();
    for (int k = threadIdx.x; k < kBRankTile; k += blockDim.x) {
      const int f = t0 + k;
      td[k] = f < n ? kd[f] : ~0ull;
      tp[k] = f < n ? kp[f] : ~0ull;
    }
    __syncthreads();
    const int m = min(kBRankTile, n - t0);
#pragma unroll 4
    for (int k = g; k < m; k += kBRankLanes) rank += (td[k] < d) | ((td[k] == d) & (tp[k] < p));
  }
#pragma unroll
  for (int o = 1; o < kBRankLanes; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
  if (e < n && g == 0) {
    ref1[q * stride + rank] = (int32_t)(p >> 32);
    ref2[q * stride + rank] = (int32_t)(p & 0xffffffffu);
    delta[q * stride + rank] = __longlong_as_double((long long)d);
  }
}

// column splits of a batched tensor-core launch (rb row blocks per pair)
int batch_split(int64_t P, int64_t rb, int64_t tiles) {
  if (P * rb >= kThroughputRowBlocks) return 1;
  int best = 1;
  int64_t best_cost = INT64_MAX;
  for (int s = 1; s <= std::min<int64_t>(kMaxSplit, tiles); ++s) {
    const int64_t waves = (P * rb * s + kSMs - 1) / kSMs;
    const int64_t cost = waves * ((tiles + s - 1) / s + 4 * XH);
    if (cost < best_cost) { best_cost = cost; best = s; }
  }
  return best;
}

template <class T>
int batch_impl(const BatchIn<T>& in, int S, int P, double delta_s, int32_t* ref1, int32_t* ref2, double* delta,
               int64_t stride, int64_t* out_count, void* ws, size_t ws_bytes, cudaStream_t st) {
  int64_t n = 1;
  for (int s = 0; s < S; ++s)
    if (in.role[s]) n = std::max<int64_t>(n, in.rows[s]);
  size_t need = 0;
  carve_batch(nullptr, S, P, n, &need);
  PS_REQUIRE(ws && ws_bytes >= need, PS_ERR_ARGUMENT, "batched match workspace %zu < %zu", ws_bytes, need);
  const BatchWs w = carve_batch(ws, S, P, n, &need);
  const int64_t N = w.n;
  cudaMemsetAsync(w.tkey, 0, (size_t)S * w.tsize * sizeof(unsigned long long), st);
  cudaMemsetAsync(w.tidx, 0x7f, (size_t)S * w.tsize * sizeof(int32_t), st);
  cudaMemsetAsync(w.ymax, 0, (size_t)S * 4 * sizeof(unsigned), st);
  cudaMemsetAsync(w.colflag, 0, (size_t)P * N * sizeof(int32_t), st);
  cudaMemsetAsync(w.cbits, 0xff, (size_t)P * N * sizeof(unsigned long long), st);
  cudaMemsetAsync(w.nn21, 0x7f, (size_t)P * N * sizeof(int32_t), st);
  // grids: blocks per set / pair capped so the whole launch is a few waves
  // (the bodies loop grid-stride; one tiny block per 8 rows of every set
  // made block scheduling the cost at C5's 512 sets)
  auto per = [](int64_t natural, int64_t groups) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(natural, (148 * 16 + groups - 1) / groups));
  };
  b_init<<<(P + 255) / 256, 256, 0, st>>>(P, w);
  PS_LAUNCHED("b_init");
  // per set: duplicate grouping, representatives, operand tiles
  const dim3 gs(per(grid_for(N, 8), S), S);
  b_hash<T><<<dim3(per(grid_for(N, 16), S), S), 256, 0, st>>>(in, w);
  PS_LAUNCHED("b_hash");
  b_reps<T><<<gs, 256, 0, st>>>(in, w);
  PS_LAUNCHED("b_reps");
  b_sel_count<T, 0><<<dim3(w.nchunk, S), 256, 0, st>>>(in, w.flag, N, w.sel_cnt, w.nchunk);
  PS_LAUNCHED("b_sel_count");
  b_sel_scatter<T, 0><<<dim3(w.nchunk, S), 256, 0, st>>>(in, w.flag, N, w.sel_cnt, w.nchunk, w.uniq, w.n_uniq);
  PS_LAUNCHED("b_sel_scatter");
  b_prep_sets<T><<<dim3(per(grid_for(w.yrows, 16), S), S), 256, 0, st>>>(in, w);
  PS_LAUNCHED("b_prep_sets");
  cudaFuncSetAttribute(b_topk<0, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<0>());
  cudaFuncSetAttribute(b_topk<1, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<1>());
  int enum_rows0 = 0;
  for (int pass = 0; pass < 2; ++pass) {
    int64_t nx = 1, ny = 1;  // row bounds over the pairs
    for (int q = 0; q < P; ++q) {
      nx = std::max<int64_t>(nx, in.rows[pass ? in.pb[q] : in.pa[q]]);
      ny = std::max<int64_t>(ny, in.rows[pass ? in.pa[q] : in.pb[q]]);
    }
    if (pass == 1) {
      // pass 0 decided nn21 of every pair none of whose rows took the exact scan (ColCand): only the
      // other pairs mark columns, so the stages below find no work for the former
      b_mark_columns<T><<<dim3(per(grid_for(N, 256), P), P), 256, 0, st>>>(in, w, delta_s, enum_rows0);
      PS_LAUNCHED("b_mark_columns");
      b_sel_count<T, 1><<<dim3(w.nchunk, P), 256, 0, st>>>(in, w.colflag, N, w.sel_cnt, w.nchunk);
      PS_LAUNCHED("b_sel_count");
      b_sel_scatter<T, 1><<<dim3(w.nchunk, P), 256, 0, st>>>(in, w.colflag, N, w.sel_cnt, w.nchunk, w.cols,
                                                             w.n_cols);
      PS_LAUNCHED("b_sel_scatter");
      b_prep_rows<T><<<dim3(per(grid_for(rup(nx, BM), 8), P), P), 256, 0, st>>>(in, w, pass, 0);
      PS_LAUNCHED("b_prep_rows(columns)");
    }
    const int64_t rb = (nx + BM - 1) / BM, tiles = (ny + BN - 1) / BN;
    const int split = batch_split(P, rb, tiles);
    b_topk<0, T><<<dim3(rb, split, P), kThreads, smem_bytes<0>(), st>>>(in, w, pass);
    PS_LAUNCHED("b_topk<top4>");
    b_certify<T><<<dim3(per(grid_for(nx, 32), P), P), 256, 0, st>>>(in, w, pass, kParts * split, rb * BM, delta_s);
    PS_LAUNCHED("b_certify");
    b_gather<T><<<dim3(per(grid_for(nx, 256), P), P), 256, 0, st>>>(in, w, pass);
    PS_LAUNCHED("b_gather");
    // near-tie rows: the first enum_rows of each pair enumerated on the
    // tensor cores, the rest (and overflowing enumerations) scanned exactly
    const int eb = (int)std::min<int64_t>(kEnumBlocksAsync, rb);
    const int enum_rows = eb * BM;
    if (pass == 0) enum_rows0 = enum_rows;
    b_prep_rows<T><<<dim3(per(grid_for(enum_rows, 8), P), P), 256, 0, st>>>(in, w, pass, 1);
    PS_LAUNCHED("b_prep_rows(overflow)");
    const int split_e = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)kMaxSplit, tiles, 4 * kSMs / (P * eb)}));
    b_topk<1, T><<<dim3(eb, split_e, P), kThreads, smem_bytes<1>(), st>>>(in, w, pass);
    PS_LAUNCHED("b_topk<enumerate>");
    b_pair_dist_min<T><<<dim3(std::max(4, 148 * 16 / P), P), 256, 0, st>>>(in, w, pass, delta_s);
    PS_LAUNCHED("b_pair_dist_min");
    b_pair_argmin<T><<<dim3(std::max(2, 148 * 8 / P), P), 256, 0, st>>>(in, w, pass, delta_s);
    PS_LAUNCHED("b_pair_argmin");
    b_pair_write<T><<<dim3(grid_for(enum_rows, 256), P), 256, 0, st>>>(in, w, pass, enum_rows);
    PS_LAUNCHED("b_pair_write");
    b_exact_rows<T><<<dim3(std::max(2, 148 * 4 / P), P), 256, 0, st>>>(in, w, pass, enum_rows);
    PS_LAUNCHED("b_exact_rows");
  }
  b_accept<T><<<dim3(per(grid_for(N, 256), P), P), 256, 0, st>>>(in, w, delta_s);
  PS_LAUNCHED("b_accept");
  b_rank_out<<<dim3((stride + 31) / 32, P), 256, 0, st>>>(w, stride, ref1, ref2, delta, out_count);
  PS_LAUNCHED("b_rank_out");
  return PS_OK;
}

}  // namespace tc
}  // namespace ps

// Candidate accepted pairs of nearest_neighbor matching on tensor cores; the
// caller sorts (keys_pair, keys_delta) and reads *counter.
template <class T>
int ps_tc_nearest_impl(const T* A, int64_t n1, const T* B, int64_t n2, double delta_s, unsigned long long* keys_pair,
                       unsigned long long* keys_delta, unsigned long long* counter, void* ws, size_t ws_bytes,
                       cudaStream_t st, bool sync, int64_t* count_out) {  // sync: *count_out = accepted pairs (or left alone)
  using namespace ps::tc;
  size_t need = 0;
  carve_tc(nullptr, n1, n2, &need);
  PS_REQUIRE(ws && ws_bytes >= need, PS_ERR_ARGUMENT, "tensor-core match workspace %zu < %zu", ws_bytes, need);
  TcWs w = carve_tc(ws, n1, n2, &need);
  for (int q = 0; q < 8; ++q) g_stats[q] = 0;
  // PS_TC_PROFILE=1 in a -DPS_DIAG build: per-stage timing and counters on stderr (syncs)
#ifdef PS_DIAG
  const bool prof = sync && getenv("PS_TC_PROFILE") != nullptr;
#else
  constexpr bool prof = false;
#endif
  cudaEvent_t ev[8];
  int nev = 0;
  auto mark = [&]() {
    if (!prof) return;
    cudaEventCreate(&ev[nev]);
    cudaEventRecord(ev[nev++], st);
  };
  auto count_of = [&](const int32_t* p) {
    int32_t h = 0;
    cudaMemcpyAsync(&h, p, 4, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return h;
  };
  mark();
  int rc = dedupe(A, n1, w.a, w, st);
  if (rc) return rc;
  rc = dedupe(B, n2, w.b, w, st);
  if (rc) return rc;
  mark();
  // pass 1: rows of A (representatives) against the distinct rows of B
  int64_t ua = -1, ub = -1;
  // pass 1 also decides the columns (ColCand): nn21 from the exact distances below delta_s it computes
  cudaMemsetAsync(w.n_cand, 0, sizeof(unsigned long long), st);
  cudaMemsetAsync(w.cbits, 0xff, n2 * sizeof(unsigned long long), st);
  cudaMemsetAsync(w.nn21, 0x7f, n2 * sizeof(int32_t), st);
  cudaMemsetAsync(w.cand_incomplete, 0, sizeof(int32_t), st);
  ColCand cc{delta_s, w.cand_incomplete, w.cbits, w.nn21, w.cand, w.cpd, w.n_cand};
#ifdef PS_TC_DIAG_NOCAND  // diagnostic builds only: always two passes
  cc = ColCand{};
#endif
  int enum_rows = INT32_MAX;
  int32_t incomplete = 0;
  rc = nearest_pass(A, n1, w.a.uniq, w.a.n_uniq, B, n2, w.b.uniq, w.b.n_uniq, w.nn12, w.d12, w, st, &ua, &ub, sync, cc,
                    &enum_rows, &incomplete);
  if (rc) return rc;
  g_stats[0] = ua;
  g_stats[1] = ub;
  // The column pass is needed only if pass 1's column candidates are incomplete.  Synchronous mode
  // knows the flag (read with the overflow count) and enumerates every overflow row, so what is left
  // is an enumeration that outgrew its buffer -- checked below with the accepted count, in the one
  // synchronisation the caller needs anyway.  Asynchronous mode cannot know: the column pass is
  // launched and finds no column (mark_columns).
  bool two_pass = !(sync && cc.cbits) || incomplete != 0;
  mark();
  const int of1 = prof ? count_of(w.n_overflow) : 0;
  unsigned long long np1 = 0;
  if (prof) {
    cudaMemcpyAsync(&np1, w.n_pairs, 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
  }
  // pass 2 (only when the candidate list outgrew its buffer, or the certificate is void): the columns
  // that can be matched against the distinct rows of A
  if (two_pass) {
  cudaMemsetAsync(w.colflag, 0, n2 * sizeof(int32_t), st);
  mark_columns<<<grid_for(n1, 256), 256, 0, st>>>(w.a.uniq, w.a.n_uniq, w.nn12, w.d12, delta_s, w.colflag,
                                                  w.n_overflow, enum_rows, w.n_pairs, w.pair_cap,
                                                  cc.cbits ? w.cand_incomplete : nullptr);
  PS_LAUNCHED("mark_columns");
  iota32<<<grid_for(n2, 256), 256, 0, st>>>(w.b.iota, n2);
  PS_LAUNCHED("iota32");
  size_t tb = w.cub_bytes;
  cub::DeviceSelect::Flagged(w.cub_tmp, tb, w.b.iota, w.colflag, w.cols, w.n_cols, (int)n2, st);
  PS_LAUNCHED("cub_select(columns)");
  mark();
  int64_t ncols = -1;
  rc = nearest_pass(B, n2, w.cols, w.n_cols, A, n1, w.a.uniq, w.a.n_uniq, w.nn21, w.d21, w, st, &ncols, &ua, sync);
  if (rc) return rc;
  g_stats[2] = ncols;
  }  // two_pass
  mark();
  accept_pairs<<<grid_for(n1, 256), 256, 0, st>>>(w.a.rep, n1, w.nn12, w.d12, w.nn21, delta_s, keys_pair, keys_delta,
                                                  counter);
  PS_LAUNCHED("accept_pairs");
  if (sync) {
    g_stats[6] = two_pass ? 2 : 1;  // passes run
    unsigned long long c = 0, np = 0;
    cudaMemcpyAsync(&c, counter, sizeof(c), cudaMemcpyDeviceToHost, st);
    if (!two_pass) cudaMemcpyAsync(&np, w.n_pairs, sizeof(np), cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    PS_REQUIRE(e == cudaSuccess, PS_ERR_CUDA, "match count: %s", cudaGetErrorString(e));
    if (!two_pass && (int64_t)np > w.pair_cap) {
      // pass 1's enumeration outgrew its buffer (its rows took the exact scan and listed no
      // columns): the column pass after all, and the acceptance again
      g_stats[6] = 2;
      cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
      cudaMemsetAsync(w.colflag, 0, n2 * sizeof(int32_t), st);
      mark_columns<<<grid_for(n1, 256), 256, 0, st>>>(w.a.uniq, w.a.n_uniq, w.nn12, w.d12, delta_s, w.colflag,
                                                      nullptr, 0, nullptr, 0, nullptr);
      PS_LAUNCHED("mark_columns");
      iota32<<<grid_for(n2, 256), 256, 0, st>>>(w.b.iota, n2);
      PS_LAUNCHED("iota32");
      size_t tb2 = w.cub_bytes;
      cub::DeviceSelect::Flagged(w.cub_tmp, tb2, w.b.iota, w.colflag, w.cols, w.n_cols, (int)n2, st);
      PS_LAUNCHED("cub_select(columns)");
      int64_t ncols2 = -1;
      rc = nearest_pass(B, n2, w.cols, w.n_cols, A, n1, w.a.uniq, w.a.n_uniq, w.nn21, w.d21, w, st, &ncols2, &ua, true);
      if (rc) return rc;
      g_stats[2] = ncols2;
      accept_pairs<<<grid_for(n1, 256), 256, 0, st>>>(w.a.rep, n1, w.nn12, w.d12, w.nn21, delta_s, keys_pair,
                                                      keys_delta, counter);
      PS_LAUNCHED("accept_pairs");
    } else if (count_out) {
      *count_out = (int64_t)c;
    }
  }
  if (prof) {
    cudaStreamSynchronize(st);
    float t[8] = {0};
    for (int i = 1; i < nev; ++i) cudaEventElapsedTime(&t[i], ev[i - 1], ev[i]);
    fprintf(stderr,
            "[tc] n1=%lld n2=%lld uniqA=%d uniqB=%d cols=%d overflow1=%d pairs1=%llu overflow2=%d | dedupe %.3f ms "
            "pass1 %.3f ms select %.3f ms pass2 %.3f ms\n",
            (long long)n1, (long long)n2, count_of(w.a.n_uniq), count_of(w.b.n_uniq), count_of(w.n_cols), of1, np1,
            count_of(w.n_overflow), t[1], t[2], t[3], t[4]);
    for (int i = 0; i < nev; ++i) cudaEventDestroy(ev[i]);
  }
  return PS_OK;
}

// One direction only: nn[i] / dist[i] = exact first argmin over the rows of
// Y of dist(X_i, Y_j) for every row i of X (reference matcher.py:74, 43-54).
template <class T>
int ps_tc_rows_impl(const T* X, int64_t nx, const T* Y, int64_t ny, int32_t* nn, double* dist, void* ws,
                    size_t ws_bytes, cudaStream_t st) {
  using namespace ps::tc;
  size_t need = 0;
  carve_tc(nullptr, nx, ny, &need);
  PS_REQUIRE(ws && ws_bytes >= need, PS_ERR_ARGUMENT, "tensor-core nearest workspace %zu < %zu", ws_bytes, need);
  TcWs w = carve_tc(ws, nx, ny, &need);
  int rc = dedupe(X, nx, w.a, w, st);
  if (rc) return rc;
  rc = dedupe(Y, ny, w.b, w, st);
  if (rc) return rc;
  rc = nearest_pass(X, nx, w.a.uniq, w.a.n_uniq, Y, ny, w.b.uniq, w.b.n_uniq, nn, dist, w, st);
  if (rc) return rc;
  copy_from_rep<<<grid_for(nx, 256), 256, 0, st>>>(w.a.rep, nx, nn, dist);  // duplicates share the answer
  PS_LAUNCHED("copy_from_rep");
  return PS_OK;
}
template int ps_tc_rows_impl<float>(const float*, int64_t, const float*, int64_t, int32_t*, double*, void*, size_t,
                                    cudaStream_t);
template int ps_tc_rows_impl<double>(const double*, int64_t, const double*, int64_t, int32_t*, double*, void*, size_t,
                                     cudaStream_t);

extern "C" int ps_match_stats(int64_t* out, int32_t n) {
  for (int q = 0; q < n && q < 8; ++q) out[q] = ps::tc::g_stats[q];
  return PS_OK;
}

size_t ps_tc_nearest_ws(int64_t n1, int64_t n2) {
  size_t need = 0;
  ps::tc::carve_tc(nullptr, n1, n2, &need);
  return need;
}

template int ps_tc_nearest_impl<float>(const float*, int64_t, const float*, int64_t, double, unsigned long long*,
                                       unsigned long long*, unsigned long long*, void*, size_t, cudaStream_t, bool, int64_t*);
template int ps_tc_nearest_impl<double>(const double*, int64_t, const double*, int64_t, double, unsigned long long*,
                                        unsigned long long*, unsigned long long*, void*, size_t, cudaStream_t, bool, int64_t*);

// ---- batched pairs: C entry points -------------------------------------------------------
namespace {
int batch_check(int32_t n_sets, const int64_t* set_rows, int32_t n_pairs, int32_t dim) {
  PS_REQUIRE(dim == ps::tc::KD, PS_ERR_ARGUMENT, "batched match needs %d-d descriptors, got %d", ps::tc::KD, dim);
  PS_REQUIRE(n_sets >= 1 && n_sets <= ps::tc::kBatchMaxSets, PS_ERR_ARGUMENT, "n_sets %d outside [1, %d]", n_sets,
             ps::tc::kBatchMaxSets);
  PS_REQUIRE(n_pairs >= 0 && n_pairs <= ps::tc::kBatchMaxPairs, PS_ERR_ARGUMENT, "n_pairs %d outside [0, %d]",
             n_pairs, ps::tc::kBatchMaxPairs);
  PS_REQUIRE(set_rows, PS_ERR_ARGUMENT, "null set_rows");
  for (int s = 0; s < n_sets; ++s)
    PS_REQUIRE(set_rows[s] >= 0 && set_rows[s] < INT32_MAX, PS_ERR_ARGUMENT, "bad row count %lld of set %d",
               (long long)set_rows[s], s);
  return PS_OK;
}
int64_t batch_rows_bound(int32_t n_sets, const int64_t* set_rows) {
  int64_t n = 1;
  for (int s = 0; s < n_sets; ++s) n = std::max<int64_t>(n, set_rows[s]);
  return n;
}
template <class T>
int batch_run(int32_t n_sets, const void* const* set_desc, const int64_t* set_rows,
              const int32_t* const* set_count, int32_t n_pairs,
              const int32_t* pair_a, const int32_t* pair_b, double delta_s, int32_t* out_ref1, int32_t* out_ref2,
              double* out_delta, int64_t out_stride, int64_t* out_count, void* ws, size_t ws_bytes,
              cudaStream_t st) {
  static thread_local ps::tc::BatchIn<T> in;  // ~11 KB: not on the stack
  memset(&in, 0, sizeof(in));
  for (int s = 0; s < n_sets; ++s) {
    in.desc[s] = static_cast<const T*>(set_desc[s]);
    in.rows[s] = (int32_t)set_rows[s];
    in.cnt[s] = set_count ? set_count[s] : nullptr;
  }
  for (int q = 0; q < n_pairs; ++q) {
    in.pa[q] = (int16_t)pair_a[q];
    in.pb[q] = (int16_t)pair_b[q];
    in.role[pair_a[q]] |= 1;
    in.role[pair_b[q]] |= 2;
  }
  return ps::tc::batch_impl<T>(in, n_sets, n_pairs, delta_s, out_ref1, out_ref2, out_delta, out_stride, out_count,
                               ws, ws_bytes, st);
}
}  // namespace

extern "C" int ps_match_batch_plan(int32_t n_sets, const int64_t* set_rows, int32_t n_pairs, int32_t dim,
                                   size_t* workspace_bytes_out) {
  const int rc = batch_check(n_sets, set_rows, n_pairs, dim);
  if (rc) return rc;
  size_t need = 0;
  ps::tc::carve_batch(nullptr, n_sets, std::max(n_pairs, 1), batch_rows_bound(n_sets, set_rows), &need);
  if (workspace_bytes_out) *workspace_bytes_out = need;
  return PS_OK;
}

extern "C" int ps_match_batch_async(int32_t n_sets, const void* const* set_desc, const int64_t* set_rows,
                                    const int32_t* const* set_count, int32_t n_pairs, const int32_t* pair_a, const int32_t* pair_b, int32_t dim,
                                    int32_t desc_is_f64, double delta_s, int32_t* out_ref1, int32_t* out_ref2,
                                    double* out_delta, int64_t out_stride, int64_t* out_count, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  int rc = batch_check(n_sets, set_rows, n_pairs, dim);
  if (rc) return rc;
  PS_REQUIRE(delta_s > 0, PS_ERR_CONFIG, "delta_s must be positive, got %g", delta_s);
  if (n_pairs == 0) return PS_OK;
  PS_REQUIRE(set_desc && pair_a && pair_b && out_ref1 && out_ref2 && out_delta && out_count, PS_ERR_ARGUMENT,
             "null argument to ps_match_batch_async");
  for (int q = 0; q < n_pairs; ++q) {
    const int a = pair_a[q], b = pair_b[q];
    PS_REQUIRE(a >= 0 && a < n_sets && b >= 0 && b < n_sets, PS_ERR_ARGUMENT, "pair %d: set index out of range", q);
    PS_REQUIRE(out_stride >= std::min(set_rows[a], set_rows[b]), PS_ERR_ARGUMENT,
               "out_stride %lld < min(rows) of pair %d", (long long)out_stride, q);
    PS_REQUIRE((set_desc[a] || set_rows[a] == 0) && (set_desc[b] || set_rows[b] == 0), PS_ERR_ARGUMENT,
               "pair %d: null descriptor set", q);
  }
  cudaStream_t st = (cudaStream_t)stream;
  rc = desc_is_f64 ? batch_run<double>(n_sets, set_desc, set_rows, set_count, n_pairs, pair_a, pair_b, delta_s, out_ref1,
                                       out_ref2, out_delta, out_stride, out_count, workspace, workspace_bytes, st)
                   : batch_run<float>(n_sets, set_desc, set_rows, set_count, n_pairs, pair_a, pair_b, delta_s, out_ref1,
                                      out_ref2, out_delta, out_stride, out_count, workspace, workspace_bytes, st);
  if (rc) return rc;
  return ps::check_cuda("ps_match_batch_async");
}

// ---- roofline probe: tensor-memory read bandwidth -----------------------------------------
// The nearest-neighbour epilogue must read every fp32 accumulator from TMEM
// (128 KB per 128 x 256 tile) while the MMA of a tile (K = 144) takes 9 x 128
// cycles: the TMEM read rate, not the MMA rate, bounds nn_topk_tc / b_topk.
// One CTA per SM allocates all 512 columns; kWarps warps (4 per lane
// quarter) each issue two 64-column tcgen05.ld per wait, `iters` times.
namespace {
constexpr int kProbeWarps = 16;
__global__ void __launch_bounds__(kProbeWarps * 32, 1) tmem_read_probe(int64_t iters, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ps::tc::tmem_alloc(&slot, 512);
  ps::tc::tc_fence_before();
  __syncthreads();
  ps::tc::tc_fence_after();
  const uint32_t tmem = slot;
  const int quarter = warp & 3, part = warp >> 2;  // 4 parts x 128 columns
  const uint32_t base = tmem + ((uint32_t)(quarter * 32) << 16) + part * 128;
  uint32_t acc = 0;
  for (int64_t it = 0; it < iters; ++it) {
    uint32_t a[64], b[64];
    ps::tc::tmem_ld_cols(base, a);
    ps::tc::tmem_ld_cols(base + 64, b);
    ps::tc::tmem_ld_wait();
#pragma unroll
    for (int k = 0; k < 64; k += 8) acc ^= a[k] + b[k + 1];
  }
  if (acc == 0x9E3779B9u) sink[blockIdx.x] = acc;  // keeps the loads; practically never true
  ps::tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) ps::tc::tmem_dealloc(tmem, 512);
}
}  // namespace

extern "C" int ps_probe_tmem_read(int64_t iters, int32_t blocks, uint32_t* sink, double* out_bytes, void* stream) {
  PS_REQUIRE(iters > 0 && blocks > 0 && sink && out_bytes, PS_ERR_ARGUMENT, "bad probe arguments");
  tmem_read_probe<<<blocks, kProbeWarps * 32, 0, (cudaStream_t)stream>>>(iters, sink);
  PS_LAUNCHED("tmem_read_probe");
  *out_bytes = (double)blocks * kProbeWarps * (double)iters * 2.0 * 64 * 32 * 4;
  return ps::check_cuda("tmem_read_probe");
}
