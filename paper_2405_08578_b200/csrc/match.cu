// K3 -- brute-force descriptor matching (reference matcher.py:57-95).
//
// Exact float64 semantics (contract P3): the reference's
// distance is np.linalg.norm(b - a[i], axis=1), i.e. per pair
//   x_t = (b_t - a_t)^2 (float64), numpy pairwise sum (eight interleaved
//   accumulators r[t] += x[8k+t], then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))),
//   sqrt.
// fl(b - a) = -fl(a - b) under round-to-nearest, so dist(i, j) is bitwise
// symmetric and the column pass is the row pass with the operands swapped.
// Ties go to the lowest index on both passes (np.argmin first occurrence).
// Accepted pairs are sorted by (delta, ref1, ref2) with stable radix sorts.
#include <cub/cub.cuh>

#include <algorithm>

#include "ps_common.cuh"

template <class T>
int ps_tc_nearest_impl(const T* A, int64_t n1, const T* B, int64_t n2, double delta_s, unsigned long long* keys_pair,
                       unsigned long long* keys_delta, unsigned long long* counter, void* ws, size_t ws_bytes,
                       cudaStream_t st, bool sync, int64_t* count_out);
size_t ps_tc_nearest_ws(int64_t n1, int64_t n2);
template <class T>
int ps_tc_rows_impl(const T* X, int64_t nx, const T* Y, int64_t ny, int32_t* nn, double* dist, void* ws,
                    size_t ws_bytes, cudaStream_t st);

namespace ps {
namespace {

// tensor-core path: 128-d nearest_neighbor problems large enough to pay off,
// unless the caller's per-call flags (OR-ed into `strategy`, see
// ps_match_strategy) force one path.  No environment switches.
constexpr int64_t kTcMinPairs = (int64_t)1 << 20;
int base_strategy(int32_t strategy) { return strategy & 0xff; }
bool use_tc(int64_t n1, int64_t n2, int dim, int32_t strategy) {
  if (base_strategy(strategy) != PS_MATCH_NEAREST || dim != 128 || (strategy & PS_MATCH_FORCE_EXACT)) return false;
  return (strategy & PS_MATCH_FORCE_TC) || n1 * n2 >= kTcMinPairs;
}
bool valid_strategy(int32_t strategy) {
  const int b = base_strategy(strategy);
  return (b == PS_MATCH_NEAREST || b == PS_MATCH_THRESHOLD_ALL || b == PS_MATCH_RATIO) &&
         (strategy & ~(0xff | PS_MATCH_FORCE_EXACT | PS_MATCH_FORCE_TC)) == 0 &&
         !((strategy & PS_MATCH_FORCE_EXACT) && (strategy & PS_MATCH_FORCE_TC));
}

constexpr int TILE = 32;     // rows x cols per tile
constexpr int SPAD = 129;    // padded smem row stride (doubles) for D <= 128
constexpr int kMaxDim = 128;

// exact reference distance from 8 interleaved accumulators
__device__ __forceinline__ double finish8(const double* r) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                              __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7]))));
}

__device__ __forceinline__ bool lex_less(double d, int j, double bd, int bj) {
  return d < bd || (d == bd && j < bj);
}

// Loads a TILE x dim tile (rows >= n zero-filled) into padded f64 smem.
template <class T>
__device__ __forceinline__ void load_tile(double* s, const T* __restrict__ X, int64_t n, int64_t r0, int dim) {
  for (int e = threadIdx.x; e < TILE * dim; e += blockDim.x) {
    const int r = e / dim, c = e % dim;
    s[r * SPAD + c] = (r0 + r < n) ? (double)X[(r0 + r) * dim + c] : 0.0;
  }
}

// For each row of X: first argmin over Y of the exact distance.
// 256 threads as 16x16, each owning a 2x2 micro-tile of (row, col) pairs.
// TOP2 also keeps the second-smallest distance of the row (a tie with the
// best counts: then second == best), for the ratio test.
template <class T, bool TOP2 = false>
__global__ void __launch_bounds__(256) nn_pass(const T* __restrict__ X, int64_t nx, const T* __restrict__ Y,
                                               int64_t ny, int dim, int32_t* __restrict__ best_j,
                                               double* __restrict__ best_d, double* __restrict__ second_d = nullptr) {
  extern __shared__ double sm[];
  double* Xs = sm;
  double* Ys = sm + TILE * SPAD;
  __shared__ double red_d[TILE][16];
  __shared__ double red_d2[TOP2 ? TILE : 1][16];
  __shared__ int red_j[TILE][16];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int nk = dim / 8;
  for (int64_t i0 = (int64_t)blockIdx.x * TILE; i0 < nx; i0 += (int64_t)gridDim.x * TILE) {
    __syncthreads();
    load_tile(Xs, X, nx, i0, dim);
    double bd[2] = {INFINITY, INFINITY};
    double b2[2] = {INFINITY, INFINITY};
    int bj[2] = {INT32_MAX, INT32_MAX};
    for (int64_t j0 = 0; j0 < ny; j0 += TILE) {
      __syncthreads();
      load_tile(Ys, Y, ny, j0, dim);
      __syncthreads();
      double acc[2][2][8];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int t = 0; t < 8; ++t) acc[a][b][t] = 0.0;
      for (int k = 0; k < nk; ++k) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int c = 8 * k + t;
          const double x0 = Xs[ty * SPAD + c], x1 = Xs[(ty + 16) * SPAD + c];
          const double y0 = Ys[tx * SPAD + c], y1 = Ys[(tx + 16) * SPAD + c];
          double e;
          e = __dsub_rn(y0, x0); acc[0][0][t] = __dadd_rn(acc[0][0][t], __dmul_rn(e, e));
          e = __dsub_rn(y1, x0); acc[0][1][t] = __dadd_rn(acc[0][1][t], __dmul_rn(e, e));
          e = __dsub_rn(y0, x1); acc[1][0][t] = __dadd_rn(acc[1][0][t], __dmul_rn(e, e));
          e = __dsub_rn(y1, x1); acc[1][1][t] = __dadd_rn(acc[1][1][t], __dmul_rn(e, e));
        }
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int64_t j = j0 + tx + 16 * b;
          if (j < ny) {
            const double dd = finish8(acc[a][b]);
            if (lex_less(dd, (int)j, bd[a], bj[a])) {
              if (TOP2) b2[a] = bd[a];
              bd[a] = dd;
              bj[a] = (int)j;
            } else if (TOP2) {
              b2[a] = fmin(b2[a], dd);
            }
          }
        }
    }
    // reduce the 16 column-owners of each row
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      red_d[ty + 16 * a][tx] = bd[a];
      red_j[ty + 16 * a][tx] = bj[a];
      if (TOP2) red_d2[ty + 16 * a][tx] = b2[a];
    }
    __syncthreads();
    if (threadIdx.x < TILE) {
      const int r = threadIdx.x;
      double d = red_d[r][0], d2 = TOP2 ? red_d2[r][0] : 0.0;
      int j = red_j[r][0];
      for (int q = 1; q < 16; ++q) {
        if (lex_less(red_d[r][q], red_j[r][q], d, j)) {
          if (TOP2) d2 = fmin(d, red_d2[r][q]);
          d = red_d[r][q];
          j = red_j[r][q];
        } else if (TOP2) {
          d2 = fmin(d2, red_d[r][q]);
        }
      }
      if (i0 + r < nx) {
        best_j[i0 + r] = j;
        best_d[i0 + r] = d;
        if (TOP2) second_d[i0 + r] = d2;
      }
    }
  }
}

// threshold_all: every pair with dist < delta_s (unordered; sorted afterwards).
template <class T>
__global__ void __launch_bounds__(256) threshold_pass(const T* __restrict__ X, int64_t nx,
                                                      const T* __restrict__ Y, int64_t ny, int dim, double delta_s,
                                                      unsigned long long* __restrict__ keys_pair,
                                                      unsigned long long* __restrict__ keys_delta,
                                                      unsigned long long* __restrict__ counter, int64_t cap) {
  extern __shared__ double sm[];
  double* Xs = sm;
  double* Ys = sm + TILE * SPAD;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int nk = dim / 8;
  const int64_t tiles_j = (ny + TILE - 1) / TILE;
  const int64_t ntiles = ((nx + TILE - 1) / TILE) * tiles_j;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = (tile / tiles_j) * TILE, j0 = (tile % tiles_j) * TILE;
    __syncthreads();
    load_tile(Xs, X, nx, i0, dim);
    load_tile(Ys, Y, ny, j0, dim);
    __syncthreads();
    double acc[2][2][8];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[a][b][t] = 0.0;
    for (int k = 0; k < nk; ++k) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int c = 8 * k + t;
        const double x0 = Xs[ty * SPAD + c], x1 = Xs[(ty + 16) * SPAD + c];
        const double y0 = Ys[tx * SPAD + c], y1 = Ys[(tx + 16) * SPAD + c];
        double e;
        e = __dsub_rn(y0, x0); acc[0][0][t] = __dadd_rn(acc[0][0][t], __dmul_rn(e, e));
        e = __dsub_rn(y1, x0); acc[0][1][t] = __dadd_rn(acc[0][1][t], __dmul_rn(e, e));
        e = __dsub_rn(y0, x1); acc[1][0][t] = __dadd_rn(acc[1][0][t], __dmul_rn(e, e));
        e = __dsub_rn(y1, x1); acc[1][1][t] = __dadd_rn(acc[1][1][t], __dmul_rn(e, e));
      }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int64_t i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
        if (i < nx && j < ny) {
          const double dd = finish8(acc[a][b]);
          if (dd < delta_s) {
            const unsigned long long slot = atomicAdd(counter, 1ull);
            if ((int64_t)slot < cap) {
              keys_pair[slot] = ((unsigned long long)i << 32) | (unsigned long long)j;
              keys_delta[slot] = (unsigned long long)__double_as_longlong(dd);
            }
          }
        }
      }
  }
}

// nearest_neighbor acceptance (matcher.py:74-79): mutual and dist < delta_s.
__global__ void mnn_select(const int32_t* __restrict__ nn12, const double* __restrict__ d12,
                           const int32_t* __restrict__ nn21, int64_t n1, double delta_s,
                           unsigned long long* __restrict__ keys_pair, unsigned long long* __restrict__ keys_delta,
                           unsigned long long* __restrict__ counter) {
  // order of emission is irrelevant: the result is sorted by (delta, ref1)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n1; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = nn12[i];
    if (nn21[j] == (int32_t)i && d12[i] < delta_s) {
      const unsigned long long slot = atomicAdd(counter, 1ull);
      keys_pair[slot] = ((unsigned long long)i << 32) | (unsigned long long)j;
      keys_delta[slot] = (unsigned long long)__double_as_longlong(d12[i]);
    }
  }
}

// ratio test (extra strategy, not in the reference; SURVEY.md F2 / north
// star "Lowe ratio"): row i keeps its first nearest neighbour when
// best < ratio * second, float64 as the oracle computes it.
__global__ void ratio_select(const int32_t* __restrict__ nn12, const double* __restrict__ d12,
                             const double* __restrict__ d12b, int64_t n1, double ratio,
                             unsigned long long* __restrict__ keys_pair, unsigned long long* __restrict__ keys_delta,
                             unsigned long long* __restrict__ counter) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n1; i += (int64_t)gridDim.x * blockDim.x) {
    if (d12[i] < __dmul_rn(ratio, d12b[i])) {
      const unsigned long long slot = atomicAdd(counter, 1ull);
      keys_pair[slot] = ((unsigned long long)i << 32) | (unsigned long long)nn12[i];
      keys_delta[slot] = (unsigned long long)__double_as_longlong(d12[i]);
    }
  }
}

__global__ void pad_unused(unsigned long long* __restrict__ kp, unsigned long long* __restrict__ kd,
                           const unsigned long long* __restrict__ counter, int64_t n) {
  const int64_t c = (int64_t)*counter;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    if (k >= c) {
      kp[k] = ~0ull;
      kd[k] = ~0ull;
    }
}

// Sort of up to kSmallSort (delta bits, pair key) entries by (delta, ref1,
// ref2) by ranking: entry e goes to slot #{f : (kd_f, kp_f) < (kd_e, kp_e)}
// (pair keys are unique, so the ranks are a permutation).  n^2 comparisons
// spread over the whole GPU beat a one-CTA sort at these sizes.
constexpr int kSmallSort = 16384;
constexpr int kRankTile = 1024;
constexpr int kRankLanes = 8;  // lanes per ranked entry (each compares against every 8th key)
__global__ void __launch_bounds__(256) rank_scatter(const unsigned long long* __restrict__ kd,
                                                    const unsigned long long* __restrict__ kp,
                                                    const unsigned long long* __restrict__ counter, int n_max,
                                                    unsigned long long* __restrict__ kd_out,
                                                    unsigned long long* __restrict__ kp_out) {
  __shared__ unsigned long long td[kRankTile], tp[kRankTile];
  constexpr int kPerBlock = 256 / kRankLanes;
  const int n = (int)min((unsigned long long)n_max, *counter);
  if ((int)(blockIdx.x * kPerBlock) >= n) return;  // uniform per block
  const int g = threadIdx.x & (kRankLanes - 1);
  const int e = blockIdx.x * kPerBlock + threadIdx.x / kRankLanes;
  const unsigned long long d = e < n ? kd[e] : 0ull, p = e < n ? kp[e] : 0ull;
  int rank = 0;
  for (int t0 = 0; t0 < n; t0 += kRankTile) {
    __syncthreads();
    for (int q = threadIdx.x; q < kRankTile; q += blockDim.x) {
      const int f = t0 + q;
      td[q] = f < n ? kd[f] : ~0ull;
      tp[q] = f < n ? kp[f] : ~0ull;
    }
    __syncthreads();
    const int m = min(kRankTile, n - t0);
#pragma unroll 4
    for (int q = g; q < m; q += kRankLanes) rank += (td[q] < d) | ((td[q] == d) & (tp[q] < p));
  }
#pragma unroll
  for (int o = 1; o < kRankLanes; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
  if (e < n && g == 0) {
    kd_out[rank] = d;
    kp_out[rank] = p;
  }
}

__global__ void unpack_pairs(const unsigned long long* __restrict__ keys_delta,
                             const unsigned long long* __restrict__ vals_pair, const unsigned long long* __restrict__ counter,
                             int64_t cap, int32_t* __restrict__ ref1, int32_t* __restrict__ ref2,
                             double* __restrict__ delta, int64_t* __restrict__ out_count) {
  const int64_t n = (int64_t)*counter;
  const int64_t m = n < cap ? n : cap;
  if (blockIdx.x == 0 && threadIdx.x == 0) *out_count = n;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    ref1[k] = (int32_t)(vals_pair[k] >> 32);
    ref2[k] = (int32_t)(vals_pair[k] & 0xffffffffu);
    delta[k] = __longlong_as_double((long long)keys_delta[k]);
  }
}

__global__ void pair_points_kernel(const int32_t* __restrict__ ref1, const int32_t* __restrict__ ref2,
                                   const int64_t* __restrict__ count, const int32_t* __restrict__ row1,
                                   const int32_t* __restrict__ col1, const int32_t* __restrict__ row2,
                                   const int32_t* __restrict__ col2, double* __restrict__ src,
                                   double* __restrict__ dst, int64_t cap) {
  const int64_t n = min(*count, cap);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int a = ref1[k], b = ref2[k];
    src[2 * k] = (double)col1[a];
    src[2 * k + 1] = (double)row1[a];
    dst[2 * k] = (double)col2[b];
    dst[2 * k + 1] = (double)row2[b];
  }
}

struct MatchWs {
  int32_t* nn12;
  double* d12;
  int32_t* nn21;
  double* d21;
  unsigned long long *kp, *kd, *kp2, *kd2, *counter;
  void* tmp;
  size_t tmp_bytes;
  void* extra;  // tensor-core path workspace
  size_t extra_bytes;
};

size_t sort_temp_bytes(int64_t n) {
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (const unsigned long long*)nullptr, (unsigned long long*)nullptr, (int)n);
  return t;
}

MatchWs carve(void* base, int64_t n1, int64_t n2, int64_t cand, size_t* used, size_t extra = 0) {
  Arena a{(char*)base, 0, 0};
  MatchWs w{};
  w.nn12 = a.take<int32_t>(n1);
  w.d12 = a.take<double>(n1);
  w.nn21 = a.take<int32_t>(n2);
  w.d21 = a.take<double>(n1 > n2 ? n1 : n2);  // column distances, or the rows' second-best (ratio test)
  w.kp = a.take<unsigned long long>(cand);
  w.kd = a.take<unsigned long long>(cand);
  w.kp2 = a.take<unsigned long long>(cand);
  w.kd2 = a.take<unsigned long long>(cand);
  w.counter = a.take<unsigned long long>(1);
  w.tmp_bytes = sort_temp_bytes(cand > 0 ? cand : 1);
  w.tmp = a.take<char>(w.tmp_bytes);
  w.extra = extra ? a.take<char>(extra) : nullptr;
  w.extra_bytes = extra;
  *used = a.used + 256;
  return w;
}

int64_t candidate_cap(int64_t n1, int64_t n2, int strategy, int64_t cap) {
  strategy = base_strategy(strategy);
  return strategy == PS_MATCH_NEAREST ? (n1 < n2 ? n1 : n2) : strategy == PS_MATCH_RATIO ? n1 : cap;
}

int grid_blocks(int64_t work, int per) {
  int64_t g = (work + per - 1) / per;
  if (g > 148 * 8) g = 148 * 8;
  return (int)(g < 1 ? 1 : g);
}

template <class T>
int launch_match(const T* desc1, int64_t n1, const T* desc2, int64_t n2, int dim, double delta_s, int strategy,
                 const MatchWs& w, int64_t cand, cudaStream_t st) {
  const size_t shmem = 2 * TILE * SPAD * sizeof(double);
  cudaFuncSetAttribute(nn_pass<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
  cudaFuncSetAttribute(threshold_pass<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
  strategy = base_strategy(strategy);
  if (strategy == PS_MATCH_RATIO) {
    cudaFuncSetAttribute(nn_pass<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
    // d21 holds the rows' second-best distances (no column pass)
    nn_pass<T, true><<<grid_blocks(n1, TILE), 256, shmem, st>>>(desc1, n1, desc2, n2, dim, w.nn12, w.d12, w.d21);
    PS_LAUNCHED("nn_pass(rows,top2)");
    ratio_select<<<grid_blocks(n1, 256), 256, 0, st>>>(w.nn12, w.d12, w.d21, n1, delta_s, w.kp, w.kd, w.counter);
    PS_LAUNCHED("ratio_select");
  } else if (strategy == PS_MATCH_NEAREST) {
    nn_pass<T><<<grid_blocks(n1, TILE), 256, shmem, st>>>(desc1, n1, desc2, n2, dim, w.nn12, w.d12);
    PS_LAUNCHED("nn_pass(rows)");
    nn_pass<T><<<grid_blocks(n2, TILE), 256, shmem, st>>>(desc2, n2, desc1, n1, dim, w.nn21, w.d21);
    PS_LAUNCHED("nn_pass(cols)");
    mnn_select<<<grid_blocks(n1, 256), 256, 0, st>>>(w.nn12, w.d12, w.nn21, n1, delta_s, w.kp, w.kd, w.counter);
    PS_LAUNCHED("mnn_select");
  } else {
    const int64_t ntiles = ((n1 + TILE - 1) / TILE) * ((n2 + TILE - 1) / TILE);
    threshold_pass<T><<<grid_blocks(ntiles, 1), 256, shmem, st>>>(desc1, n1, desc2, n2, dim, delta_s, w.kp, w.kd,
                                                                  w.counter, cand);
    PS_LAUNCHED("threshold_pass");
  }
  return PS_OK;
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" int ps_match_plan(int64_t n1, int64_t n2, int32_t dim, int32_t strategy, int64_t cap,
                             size_t* workspace_bytes_out) {
  PS_REQUIRE(n1 >= 0 && n2 >= 0 && cap >= 0, PS_ERR_ARGUMENT, "bad sizes");
  PS_REQUIRE(valid_strategy(strategy), PS_ERR_CONFIG, "unknown match strategy %d", strategy);
  size_t used = 0;
  carve(nullptr, n1, n2, candidate_cap(n1, n2, strategy, cap), &used,
        use_tc(n1, n2, dim, strategy) ? ps_tc_nearest_ws(n1, n2) : 0);
  if (workspace_bytes_out) *workspace_bytes_out = used;
  return PS_OK;
}

namespace {
int match_impl(const void* desc1, int64_t n1, const void* desc2, int64_t n2, int32_t dim, int32_t desc_is_f64,
               double delta_s, int32_t strategy, int32_t* out_ref1, int32_t* out_ref2, double* out_delta,
               int64_t* out_count, int64_t cap, void* workspace, size_t workspace_bytes, void* stream, bool sync) {
  PS_REQUIRE(delta_s > 0, PS_ERR_CONFIG, "delta_s must be positive, got %g", delta_s);
  PS_REQUIRE(valid_strategy(strategy), PS_ERR_CONFIG, "unknown match strategy %d", strategy);
  PS_REQUIRE(base_strategy(strategy) != PS_MATCH_RATIO || delta_s <= 1.0, PS_ERR_CONFIG,
             "ratio must be in (0, 1], got %g", delta_s);
  PS_REQUIRE(dim >= 8 && dim % 8 == 0 && dim <= kMaxDim, PS_ERR_ARGUMENT,
             "descriptor length %d unsupported (multiple of 8, <= %d)", dim, kMaxDim);
  PS_REQUIRE(out_count, PS_ERR_ARGUMENT, "null out_count");
  PS_REQUIRE(n1 < INT32_MAX && n2 < INT32_MAX, PS_ERR_ARGUMENT, "too many descriptors");
  cudaStream_t st = (cudaStream_t)stream;
  if (n1 == 0 || n2 == 0) {  // matcher.py:66-67
    cudaMemsetAsync(out_count, 0, sizeof(int64_t), st);
    return check_cuda("memset");
  }
  PS_REQUIRE(desc1 && desc2, PS_ERR_ARGUMENT, "null descriptors");
  const int64_t cand = candidate_cap(n1, n2, strategy, cap);
  const bool tc = use_tc(n1, n2, dim, strategy);
  const size_t extra = tc ? ps_tc_nearest_ws(n1, n2) : 0;
  size_t used = 0;
  carve(nullptr, n1, n2, cand, &used, extra);
  PS_REQUIRE(workspace && workspace_bytes >= used, PS_ERR_ARGUMENT, "match workspace %zu < %zu", workspace_bytes,
             used);
  MatchWs w = carve(workspace, n1, n2, cand, &used, extra);
  cudaMemsetAsync(w.counter, 0, sizeof(unsigned long long), st);
  int rc;
  int64_t tc_count = -1;  // the tensor-core path's accepted count when it has read it already
  if (tc) {
    rc = desc_is_f64 ? ps_tc_nearest_impl((const double*)desc1, n1, (const double*)desc2, n2, delta_s, w.kp, w.kd,
                                          w.counter, w.extra, w.extra_bytes, st, sync, &tc_count)
                     : ps_tc_nearest_impl((const float*)desc1, n1, (const float*)desc2, n2, delta_s, w.kp, w.kd,
                                          w.counter, w.extra, w.extra_bytes, st, sync, &tc_count);
  } else {
    rc = desc_is_f64
             ? launch_match((const double*)desc1, n1, (const double*)desc2, n2, dim, delta_s, strategy, w, cand, st)
             : launch_match((const float*)desc1, n1, (const float*)desc2, n2, dim, delta_s, strategy, w, cand, st);
  }
  if (rc) return rc;
  // Sort by (delta, ref1, ref2): two stable radix passes, pair key first,
  // then delta bits (non-negative doubles order like their bit patterns).
  // cub needs a host-side length: the tensor-core path has synchronised with
  // the host already, so its accepted count is read back and only those keys
  // are sorted; the asynchronous CUDA-core path sorts the whole candidate
  // capacity with unused slots padded by all-ones keys (they sort last), and
  // so does the tensor-core path in asynchronous mode.
  int n = (int)(cand > 0 ? cand : 1);
  if (tc && sync) {
    unsigned long long c = (unsigned long long)std::max<int64_t>(tc_count, 0);
    if (tc_count < 0) {
      cudaMemcpyAsync(&c, w.counter, sizeof(c), cudaMemcpyDeviceToHost, st);
      const cudaError_t e = cudaStreamSynchronize(st);
      PS_REQUIRE(e == cudaSuccess, PS_ERR_CUDA, "match count: %s", cudaGetErrorString(e));
    }
    n = (int)std::max<unsigned long long>(1ull, std::min<unsigned long long>(c, (unsigned long long)n));
  }
  if (n <= kSmallSort) {
    rank_scatter<<<(n + 256 / kRankLanes - 1) / (256 / kRankLanes), 256, 0, st>>>(w.kd, w.kp, w.counter, n, w.kd2,
                                                                                w.kp2);
    PS_LAUNCHED("rank_scatter");
    unpack_pairs<<<grid_blocks(n, 256), 256, 0, st>>>(w.kd2, w.kp2, w.counter, cap, out_ref1, out_ref2, out_delta,
                                                      out_count);
    PS_LAUNCHED("unpack_pairs");
    return PS_OK;
  }
  pad_unused<<<grid_blocks(n, 256), 256, 0, st>>>(w.kp, w.kd, w.counter, n);
  PS_LAUNCHED("pad_unused");
  size_t tb = w.tmp_bytes;
  // pair keys are (row << 32 | column): only the bits that can differ are sorted.  The rows of
  // nearest_neighbor / ratio_test matches are unique, so their row bits alone order the pairs
  // (padding keys are placed last by the delta sort whatever this one does with them)
  int row_bits = 1;
  while (row_bits < 32 && (1ll << row_bits) < n1) ++row_bits;
  const int base = strategy & 0xff;
  const int bit0 = (base == PS_MATCH_NEAREST || base == PS_MATCH_RATIO) ? 32 : 0;
  cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.kp, w.kp2, w.kd, w.kd2, n, bit0, 32 + row_bits, st);
  PS_LAUNCHED("cub_sort(pair)");
  tb = w.tmp_bytes;
  cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.kd2, w.kd, w.kp2, w.kp, n, 0, 64, st);
  PS_LAUNCHED("cub_sort(delta)");
  unpack_pairs<<<grid_blocks(n, 256), 256, 0, st>>>(w.kd, w.kp, w.counter, cap, out_ref1, out_ref2, out_delta,
                                                    out_count);
  PS_LAUNCHED("unpack_pairs");
  return PS_OK;
}
}  // namespace

extern "C" int ps_match(const void* desc1, int64_t n1, const void* desc2, int64_t n2, int32_t dim,
                        int32_t desc_is_f64, double delta_s, int32_t strategy, int32_t* out_ref1, int32_t* out_ref2,
                        double* out_delta, int64_t* out_count, int64_t cap, void* workspace, size_t workspace_bytes,
                        void* stream) {
  return match_impl(desc1, n1, desc2, n2, dim, desc_is_f64, delta_s, strategy, out_ref1, out_ref2, out_delta,
                    out_count, cap, workspace, workspace_bytes, stream, true);
}

extern "C" int ps_match_async(const void* desc1, int64_t n1, const void* desc2, int64_t n2, int32_t dim,
                              int32_t desc_is_f64, double delta_s, int32_t strategy, int32_t* out_ref1,
                              int32_t* out_ref2, double* out_delta, int64_t* out_count, int64_t cap, void* workspace,
                              size_t workspace_bytes, void* stream) {
  return match_impl(desc1, n1, desc2, n2, dim, desc_is_f64, delta_s, strategy, out_ref1, out_ref2, out_delta,
                    out_count, cap, workspace, workspace_bytes, stream, false);
}

extern "C" int ps_pair_points(const int32_t* ref1, const int32_t* ref2, const int64_t* count, const int32_t* row1,
                              const int32_t* col1, const int32_t* row2, const int32_t* col2, double* src_xy,
                              double* dst_xy, int64_t cap, void* stream) {
  PS_REQUIRE(ref1 && ref2 && count && row1 && col1 && row2 && col2 && src_xy && dst_xy, PS_ERR_ARGUMENT,
             "null argument to ps_pair_points");
  if (cap <= 0) return PS_OK;
  pair_points_kernel<<<grid_blocks(cap, 256), 256, 0, (cudaStream_t)stream>>>(ref1, ref2, count, row1, col1, row2,
                                                                              col2, src_xy, dst_xy, cap);
  PS_LAUNCHED("pair_points");
  return PS_OK;
}

extern "C" int ps_nearest_plan(int64_t nx, int64_t ny, int32_t dim, int32_t flags, size_t* workspace_bytes_out) {
  PS_REQUIRE(nx >= 0 && ny >= 0, PS_ERR_ARGUMENT, "bad sizes");
  PS_REQUIRE(dim >= 8 && dim % 8 == 0 && dim <= kMaxDim, PS_ERR_ARGUMENT, "descriptor length %d unsupported", dim);
  PS_REQUIRE(valid_strategy(PS_MATCH_NEAREST | flags), PS_ERR_ARGUMENT, "bad flags %d", flags);
  if (workspace_bytes_out)
    *workspace_bytes_out = use_tc(nx, ny, dim, PS_MATCH_NEAREST | flags) ? ps_tc_nearest_ws(nx, ny) : 256;
  return PS_OK;
}

extern "C" int ps_nearest(const void* X, int64_t nx, const void* Y, int64_t ny, int32_t dim, int32_t desc_is_f64,
                          int32_t flags, int32_t* out_index, double* out_dist, void* workspace, size_t workspace_bytes,
                          void* stream) {
  PS_REQUIRE(dim >= 8 && dim % 8 == 0 && dim <= kMaxDim, PS_ERR_ARGUMENT, "descriptor length %d unsupported", dim);
  PS_REQUIRE(valid_strategy(PS_MATCH_NEAREST | flags), PS_ERR_ARGUMENT, "bad flags %d", flags);
  PS_REQUIRE(nx < INT32_MAX && ny < INT32_MAX, PS_ERR_ARGUMENT, "too many descriptors");
  if (nx == 0) return PS_OK;
  PS_REQUIRE(X && Y && out_index && out_dist && ny > 0, PS_ERR_ARGUMENT, "null argument / empty Y in ps_nearest");
  cudaStream_t st = (cudaStream_t)stream;
  if (use_tc(nx, ny, dim, PS_MATCH_NEAREST | flags)) {
    return desc_is_f64 ? ps_tc_rows_impl((const double*)X, nx, (const double*)Y, ny, out_index, out_dist, workspace,
                                         workspace_bytes, st)
                       : ps_tc_rows_impl((const float*)X, nx, (const float*)Y, ny, out_index, out_dist, workspace,
                                         workspace_bytes, st);
  }
  const size_t shmem = 2 * TILE * SPAD * sizeof(double);
  if (desc_is_f64) {
    cudaFuncSetAttribute(nn_pass<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
    nn_pass<double><<<grid_blocks(nx, TILE), 256, shmem, st>>>((const double*)X, nx, (const double*)Y, ny, dim,
                                                               out_index, out_dist);
  } else {
    cudaFuncSetAttribute(nn_pass<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
    nn_pass<float><<<grid_blocks(nx, TILE), 256, shmem, st>>>((const float*)X, nx, (const float*)Y, ny, dim, out_index,
                                                              out_dist);
  }
  PS_LAUNCHED("nn_pass");
  return PS_OK;
}
