// tree.cu — device-resident best-first tree growth:
// grow_tree (tree.cpp:186-261) with partition_leaf (tree.cpp:114-128), the
// children's gather_leaf_statistics (tree.cpp:244-246), the histogram of the
// smaller child only and the larger child by subtraction (row a10).
//
// Device state per tree: two ping-pong "ordered" buffers of (row id, g, h),
// SoA. Every open leaf owns a contiguous range [begin, begin+count) of one of
// them, so its histogram reads ids and g/h contiguously (HBG_GH_LEAF_ALIGNED,
// the algorithmic-bytes layout of SURVEY §8d) however deep the leaf is. A
// split partitions the parent's range stably into the other buffer (left rows
// first, in leaf order — the reference's order), computing both children's
// fp64 totals on the way in a fixed order.
#include <algorithm>
#include <vector>

#include "hbg_internal.h"

namespace hbg {

namespace {

constexpr int kPartThreads = 512;
constexpr int kPartItems = 8;
constexpr int kPartTile = kPartThreads * kPartItems;  // positions per block

template <typename T>
struct PartArgs {
  const int32_t* rows;
  const T* g;  // float (bits32) or double (bits64) leaf-aligned g/h
  const T* h;
  int64_t n;
  const uint8_t* packed;
  int64_t row_stride;
  int byte_off;
  int shift;
  uint32_t mask;
  int thr;
  uint8_t* flags;
  int32_t* block_left;
  double* block_sums;  // [nblocks][4] = gl, hl, gr, hr
};

// Deterministic block reduction of 4 doubles + one int (warp shuffle tree, then warps in order).
__device__ void block_reduce_4d1i(double v[4], int& c, double (*sd)[kPartThreads / 32], int* sc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] += __shfl_down_sync(0xffffffffu, v[j], off);
    c += __shfl_down_sync(0xffffffffu, c, off);
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) sd[j][w] = v[j];
    sc[w] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 0; j < 4; ++j) {
      double s = 0.0;
      for (int i = 0; i < kPartThreads / 32; ++i) s += sd[j][i];
      v[j] = s;
    }
    int s = 0;
    for (int i = 0; i < kPartThreads / 32; ++i) s += sc[i];
    c = s;
  }
}

// Per-iteration block ranks: each warp's ballot counts -> exclusive warp
// offsets (computed by warp 0 with shuffles) + iteration totals.
struct RankScratch {
  int wl[kPartThreads / 32], wn[kPartThreads / 32];
  int ol[kPartThreads / 32], on[kPartThreads / 32];
  int tl, tn;
};

__device__ __forceinline__ void block_ranks(unsigned lm, unsigned vm, RankScratch& rs) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    rs.wl[w] = __popc(lm);
    rs.wn[w] = __popc(vm);
  }
  __syncthreads();
  if (w == 0) {
    constexpr int W = kPartThreads / 32;
    int l = lane < W ? rs.wl[lane] : 0, nn = lane < W ? rs.wn[lane] : 0;
    int il = l, in = nn;  // inclusive scans
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, il, off), b = __shfl_up_sync(0xffffffffu, in, off);
      if (lane >= off) {
        il += a;
        in += b;
      }
    }
    if (lane < W) {
      rs.ol[lane] = il - l;
      rs.on[lane] = in - nn;
    }
    if (lane == W - 1) {
      rs.tl = il;
      rs.tn = in;
    }
  }
  __syncthreads();
}

// Pass 1: side flag per position (bin <= thr goes left, tree.cpp:117-123),
// per-block left count and fp64 per-side g/h sums.
template <typename T>
__global__ void __launch_bounds__(kPartThreads) partition_count_kernel(PartArgs<T> a) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kPartTile;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  int c = 0;
#pragma unroll
  for (int i = 0; i < kPartItems; ++i) {
    const int64_t pos = base + i * kPartThreads + threadIdx.x;
    if (pos < a.n) {
      const int32_t row = __ldg(a.rows + pos);
      const uint32_t byte = __ldg(a.packed + static_cast<int64_t>(row) * a.row_stride + a.byte_off);
      const bool left = ((byte >> a.shift) & a.mask) <= static_cast<uint32_t>(a.thr);
      a.flags[pos] = left ? 1 : 0;
      const double gv = __ldg(a.g + pos), hv = __ldg(a.h + pos);
      if (left) {
        ++c;
        v[0] += gv;
        v[1] += hv;
      } else {
        v[2] += gv;
        v[3] += hv;
      }
    }
  }
  __shared__ double sd[4][kPartThreads / 32];
  __shared__ int sc[kPartThreads / 32];
  block_reduce_4d1i(v, c, sd, sc);
  if (threadIdx.x == 0) {
    a.block_left[blockIdx.x] = c;
#pragma unroll
    for (int j = 0; j < 4; ++j) a.block_sums[4 * blockIdx.x + j] = v[j];
  }
}

// Pass 2 (one CTA): exclusive scan of the block left counts and fixed-order
// fp64 child totals. out_totals = {gl, hl, gr, hr}, *left_total = rows left.
// Thread t owns a contiguous run of blocks; runs are combined by a pairwise
// tree in thread order, so the totals do not depend on timing.
constexpr int kScanT = 256;

__global__ void __launch_bounds__(kScanT) partition_scan_kernel(const int32_t* block_left,
                                                                const double* block_sums, int nb,
                                                                int64_t* block_off, double* out_totals,
                                                                int64_t* left_total) {
  const int t = threadIdx.x;
  const int chunk = (nb + kScanT - 1) / kScanT;
  const int b0 = min(nb, t * chunk), b1 = min(nb, b0 + chunk);
  int64_t local = 0;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int b = b0; b < b1; ++b) {
    local += block_left[b];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] += block_sums[4 * b + j];
  }
  __shared__ int64_t ss[kScanT];
  __shared__ double sv[4][kScanT];
  ss[t] = local;
#pragma unroll
  for (int j = 0; j < 4; ++j) sv[j][t] = v[j];
  __syncthreads();
  for (int off = 1; off < kScanT; off <<= 1) {  // inclusive Hillis-Steele scan of counts
    const int64_t x = t >= off ? ss[t - off] : 0;
    __syncthreads();
    ss[t] += x;
    __syncthreads();
  }
  int64_t run = ss[t] - local;  // exclusive prefix of this thread's run
  for (int b = b0; b < b1; ++b) {
    block_off[b] = run;
    run += block_left[b];
  }
  for (int st = kScanT / 2; st > 0; st >>= 1) {  // pairwise tree, fixed shape
    if (t < st) {
#pragma unroll
      for (int j = 0; j < 4; ++j) sv[j][t] += sv[j][t + st];
    }
    __syncthreads();
  }
  if (t == 0) {
    *left_total = ss[kScanT - 1];
#pragma unroll
    for (int j = 0; j < 4; ++j) out_totals[j] = sv[j][0];
  }
}

// Pass 3: stable scatter of (row, g, h) into the other buffer, left side first.
template <typename T>
__global__ void __launch_bounds__(kPartThreads) partition_scatter_kernel(
    const int32_t* __restrict__ rows, const T* __restrict__ g, const T* __restrict__ h,
    const uint8_t* __restrict__ flags, int64_t n, const int64_t* __restrict__ block_off,
    const int64_t* __restrict__ left_total, int32_t* __restrict__ orow, T* __restrict__ og,
    T* __restrict__ oh) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kPartTile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ RankScratch rs;
  const int64_t L = *left_total;
  const int64_t left_before = block_off[blockIdx.x];
  int64_t lrun = left_before;         // left rows before this item, in leaf order
  int64_t rrun = base - left_before;  // right rows before this item
  const int64_t rem = (n - base + kPartThreads - 1) / kPartThreads;
  const int iters = static_cast<int>(rem < kPartItems ? rem : kPartItems);
  for (int i = 0; i < iters; ++i) {
    const int64_t pos = base + i * kPartThreads + threadIdx.x;
    const bool valid = pos < n;
    const bool left = valid && flags[pos];
    const unsigned lm = __ballot_sync(0xffffffffu, left);
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    block_ranks(lm, vm, rs);
    const unsigned below = (1u << lane) - 1u;
    if (valid) {
      const int lrank = rs.ol[w] + __popc(lm & below);
      const int prank = rs.on[w] + __popc(vm & below);  // position rank within this iteration
      const int64_t dst = left ? lrun + lrank : L + rrun + (prank - lrank);
      orow[dst] = rows[pos];
      og[dst] = g[pos];
      oh[dst] = h[pos];
    }
    lrun += rs.tl;
    rrun += rs.tn - rs.tl;
    __syncthreads();
  }
}

// Leaves of at most one tile: flags, totals, ranks and the stable scatter in a
// single CTA (one launch instead of three).
template <typename T>
__global__ void __launch_bounds__(kPartThreads) partition_small_kernel(PartArgs<T> a, int32_t* __restrict__ orow,
                                                                       T* __restrict__ og, T* __restrict__ oh,
                                                                       double* out_totals, int64_t* left_total) {
  __shared__ uint8_t flag[kPartTile];
  __shared__ double sd[4][kPartThreads / 32];
  __shared__ int sc[kPartThreads / 32];
  __shared__ RankScratch rs;
  __shared__ int64_t L_sh;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  int c = 0;
#pragma unroll
  for (int i = 0; i < kPartItems; ++i) {
    const int pos = i * kPartThreads + threadIdx.x;
    if (pos < a.n) {
      const int32_t row = __ldg(a.rows + pos);
      const uint32_t byte = __ldg(a.packed + static_cast<int64_t>(row) * a.row_stride + a.byte_off);
      const bool left = ((byte >> a.shift) & a.mask) <= static_cast<uint32_t>(a.thr);
      flag[pos] = left ? 1 : 0;
      const double gv = __ldg(a.g + pos), hv = __ldg(a.h + pos);
      if (left) {
        ++c;
        v[0] += gv;
        v[1] += hv;
      } else {
        v[2] += gv;
        v[3] += hv;
      }
    }
  }
  block_reduce_4d1i(v, c, sd, sc);  // thread 0 holds the totals
  if (threadIdx.x == 0) {
    L_sh = c;
    *left_total = c;
#pragma unroll
    for (int j = 0; j < 4; ++j) out_totals[j] = v[j];
  }
  __syncthreads();
  const int64_t L = L_sh;
  int64_t lrun = 0, rrun = 0;
  const int iters = static_cast<int>((a.n + kPartThreads - 1) / kPartThreads);
  for (int i = 0; i < iters; ++i) {
    const int pos = i * kPartThreads + threadIdx.x;
    const bool valid = pos < a.n;
    const bool left = valid && flag[pos];
    const unsigned lm = __ballot_sync(0xffffffffu, left);
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    block_ranks(lm, vm, rs);
    const unsigned below = (1u << lane) - 1u;
    if (valid) {
      const int lrank = rs.ol[w] + __popc(lm & below);
      const int prank = rs.on[w] + __popc(vm & below);
      const int64_t dst = left ? lrun + lrank : L + rrun + (prank - lrank);
      orow[dst] = a.rows[pos];
      og[dst] = a.g[pos];
      oh[dst] = a.h[pos];
    }
    lrun += rs.tl;
    rrun += rs.tn - rs.tl;
    __syncthreads();
  }
}

// ---- small leaves: deterministic fixed-point histogram through L2 atomics ----
// For a leaf of a few thousand rows the shared-memory kernel's fixed cost
// (clearing and folding per-warp cells) dominates. Here every (row, feature)
// adds int64 fixed-point g and h (scale 2^S per LEAF from the leaf's own max
// |g|, |h|, |q| <= 2^39 per element, so any leaf of < 2^23 rows sums without
// overflow and a leaf of tiny values keeps their precision) and a u32 count straight
// into an L2-resident accumulator with native 64-bit reductions (REDG.E.ADD.64)
// from all SMs. Integer addition commutes, so the result is bitwise
// deterministic and more precise than fp32 accumulation (2^-40 of max|g| per
// element).

// Per-leaf scales for a leaf of n <= kAtomicHistRows rows, one block: max
// |g|, |h| over the leaf's own rows (order-free integer max of the
// non-negative floats' bits) -> exps. A per-tree scale would quantise a leaf
// of values far below the tree's max (converged logistic hessians, residuals
// next to an outlier) to a few bits.
__global__ void fixed_leaf_scale_kernel(const float* __restrict__ g, const float* __restrict__ h, int64_t n,
                                        int* __restrict__ exps) {
  __shared__ unsigned int m[2];
  if (threadIdx.x == 0) m[0] = m[1] = 0u;
  __syncthreads();
  unsigned int mg = 0u, mh = 0u;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    mg = max(mg, __float_as_uint(fabsf(g[i])));
    mh = max(mh, __float_as_uint(fabsf(h[i])));
  }
  mg = __reduce_max_sync(0xffffffffu, mg);
  mh = __reduce_max_sync(0xffffffffu, mh);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&m[0], mg);
    atomicMax(&m[1], mh);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int eg = 0, eh = 0;
    frexpf(__uint_as_float(m[0]), &eg);
    frexpf(__uint_as_float(m[1]), &eh);
    exps[0] = 39 - eg;
    exps[1] = 39 - eh;
  }
}

// Thread = (row, 32-bit word of the packed row): the word's features.
__global__ void small_hist_atomic_kernel(const int32_t* __restrict__ rows, const float* __restrict__ g,
                                         const float* __restrict__ h, int64_t n,
                                         const uint32_t* __restrict__ packed, int64_t gs_words,
                                         int words_per_row, int bits, int d, int k,
                                         const int* __restrict__ exps, unsigned long long* __restrict__ acc) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * words_per_row) return;
  const int64_t pos = t / words_per_row;
  const int w = static_cast<int>(t - pos * words_per_row);
  const int32_t row = rows[pos];
  // group-planar layout: word w of a row sits in slice group w / wps
  const int wps = bits == 8 ? 8 : 4;  // words per 32-feature slice
  const uint32_t word = __ldg(packed + (w / wps) * gs_words + static_cast<int64_t>(row) * wps + w % wps);
  const int64_t qg = __double2ll_rn(ldexp(static_cast<double>(g[pos]), exps[0]));
  const int64_t qh = __double2ll_rn(ldexp(static_cast<double>(h[pos]), exps[1]));
  const int fpw = 32 / bits;
  const uint32_t mask = (1u << bits) - 1u;
  const size_t D = static_cast<size_t>(d) * k;
  unsigned int* cnt = reinterpret_cast<unsigned int*>(acc + 2 * D);
  for (int p = 0; p < fpw; ++p) {
    // slice-major word index -> feature id (32 features per slice)
    const int f = (w * fpw) + p;
    if (f >= d) break;
    const uint32_t b = (word >> (bits * p)) & mask;
    const size_t o = static_cast<size_t>(f) * k + b;
    atomicAdd(acc + o, static_cast<unsigned long long>(qg));
    atomicAdd(acc + D + o, static_cast<unsigned long long>(qh));
    atomicAdd(cnt + o, 1u);
  }
}

// Fixed point -> SoA fp64 histogram (+ sibling = parent - hist when given),
// and clear the accumulator for the next leaf.
__global__ void small_hist_finish_kernel(unsigned long long* __restrict__ acc, const int* __restrict__ exps,
                                         int64_t cells, double* __restrict__ out, const double* parent,
                                         double* sibling) {
  const double sg = ldexp(1.0, -exps[0]), sh = ldexp(1.0, -exps[1]);
  unsigned int* cnt = reinterpret_cast<unsigned int*>(acc + 2 * cells);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cells;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double vg = static_cast<double>(static_cast<long long>(acc[i])) * sg;
    const double vh = static_cast<double>(static_cast<long long>(acc[cells + i])) * sh;
    const double vc = static_cast<double>(cnt[i]);
    acc[i] = 0ull;
    acc[cells + i] = 0ull;
    cnt[i] = 0u;
    out[i] = vg;
    out[cells + i] = vh;
    out[2 * cells + i] = vc;
    if (parent) {
      const double pg = parent[i], ph = parent[cells + i], pc = parent[2 * cells + i];
      sibling[i] = pg - vg;
      sibling[cells + i] = ph - vh;
      sibling[2 * cells + i] = pc - vc;
    }
  }
}

}  // namespace

size_t small_hist_acc_bytes(int d, int k) {
  const size_t D = static_cast<size_t>(d) * k;
  return D * 8 * 2 + D * 4 + 16;
}

void launch_fixed_leaf_scale(const float* g, const float* h, int64_t n, int* exps, cudaStream_t s) {
  fixed_leaf_scale_kernel<<<1, 1024, 0, s>>>(g, h, n, exps);
  HBG_LAUNCH_CHECK();
}

void launch_small_hist_atomic(const int32_t* rows, const float* g, const float* h, int64_t n,
                              const uint32_t* packed, int64_t gs_words, int words_per_row, int bits, int d,
                              int k, const int* exps, void* acc, cudaStream_t s) {
  const int64_t items = n * words_per_row;
  if (items == 0) return;
  small_hist_atomic_kernel<<<static_cast<unsigned>((items + 255) / 256), 256, 0, s>>>(
      rows, g, h, n, packed, gs_words, words_per_row, bits, d, k, exps,
      static_cast<unsigned long long*>(acc));
  HBG_LAUNCH_CHECK();
}

void launch_small_hist(const int32_t* rows, const float* g, const float* h, int64_t n,
                       const uint32_t* packed, int64_t gs_words, int words_per_row, int bits, int d, int k,
                       const int* exps, void* acc, double* out, const double* parent, double* sibling,
                       cudaStream_t s) {
  unsigned long long* a = static_cast<unsigned long long*>(acc);
  const int64_t items = n * words_per_row;
  if (items > 0) {
    small_hist_atomic_kernel<<<static_cast<unsigned>((items + 255) / 256), 256, 0, s>>>(
        rows, g, h, n, packed, gs_words, words_per_row, bits, d, k, exps, a);
    HBG_LAUNCH_CHECK();
  }
  const int64_t cells = static_cast<int64_t>(d) * k;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((cells + 255) / 256, 296));
  small_hist_finish_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(a, exps, cells, out, parent, sibling);
  HBG_LAUNCH_CHECK();
}

void configure_tree_kernels() {
  set_max_shared_carveout(reinterpret_cast<const void*>(fixed_leaf_scale_kernel));
  set_max_shared_carveout(reinterpret_cast<const void*>(small_hist_atomic_kernel));
  set_max_shared_carveout(reinterpret_cast<const void*>(small_hist_finish_kernel));
  set_max_shared_carveout(reinterpret_cast<const void*>(partition_small_kernel<float>));
  set_max_shared_carveout(reinterpret_cast<const void*>(partition_count_kernel<float>));
  set_max_shared_carveout(reinterpret_cast<const void*>(partition_scan_kernel));
  set_max_shared_carveout(reinterpret_cast<const void*>(partition_scatter_kernel<float>));
  set_max_shared_carveout(reinterpret_cast<const void*>(partition_small_kernel<double>));
  set_max_shared_carveout(reinterpret_cast<const void*>(partition_count_kernel<double>));
  set_max_shared_carveout(reinterpret_cast<const void*>(partition_scatter_kernel<double>));
}

// One split of a leaf's range: flags/counts/totals, scan, scatter. `scratch`
// must hold n bytes of flags + per-block arrays (see partition_scratch_bytes).
size_t partition_scratch_bytes(int64_t n) {
  const int64_t nb = std::max<int64_t>(1, (n + kPartTile - 1) / kPartTile);
  return static_cast<size_t>(n) + 16 + static_cast<size_t>(nb) * (4 + 32 + 8) + 64;
}

namespace {

template <typename T>
void launch_partition_t(const int32_t* rows, const T* g, const T* h, int64_t n, const uint8_t* packed,
                        int64_t row_stride, int feature, int bits, int thr, int32_t* orow, T* og, T* oh,
                        void* scratch, double* d_totals, int64_t* d_left, cudaStream_t s) {
  const int64_t nb = std::max<int64_t>(1, (n + kPartTile - 1) / kPartTile);
  uint8_t* p = static_cast<uint8_t*>(scratch);
  uint8_t* flags = p;
  p += (static_cast<size_t>(n) + 15) / 16 * 16;
  double* block_sums = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(nb) * 32;
  int64_t* block_off = reinterpret_cast<int64_t*>(p);
  p += static_cast<size_t>(nb) * 8;
  int32_t* block_left = reinterpret_cast<int32_t*>(p);
  PartArgs<T> a{};
  a.rows = rows;
  a.g = g;
  a.h = h;
  a.n = n;
  a.packed = packed;
  a.row_stride = row_stride;
  const int slice = feature / 32, fl = feature % 32;
  if (bits == 8) {
    a.byte_off = slice * 32 + fl;
    a.shift = 0;
    a.mask = 0xFF;
  } else {
    a.byte_off = slice * 16 + (fl / 8) * 4 + (fl % 8) / 2;
    a.shift = 4 * (fl % 2);
    a.mask = 0xF;
  }
  a.thr = thr;
  a.flags = flags;
  a.block_left = block_left;
  a.block_sums = block_sums;
  if (n <= kPartTile) {
    partition_small_kernel<T><<<1, kPartThreads, 0, s>>>(a, orow, og, oh, d_totals, d_left);
    HBG_LAUNCH_CHECK();
    return;
  }
  partition_count_kernel<T><<<static_cast<unsigned>(nb), kPartThreads, 0, s>>>(a);
  HBG_LAUNCH_CHECK();
  partition_scan_kernel<<<1, kScanT, 0, s>>>(block_left, block_sums, static_cast<int>(nb), block_off,
                                           d_totals, d_left);
  HBG_LAUNCH_CHECK();
  partition_scatter_kernel<T><<<static_cast<unsigned>(nb), kPartThreads, 0, s>>>(
      rows, g, h, flags, n, block_off, d_left, orow, og, oh);
  HBG_LAUNCH_CHECK();
}

}  // namespace

void launch_partition(const int32_t* rows, const float* g, const float* h, int64_t n,
                      const uint8_t* packed, int64_t row_stride, int feature, int bits, int thr,
                      int32_t* orow, float* og, float* oh, void* scratch, double* d_totals,
                      int64_t* d_left, cudaStream_t s) {
  launch_partition_t<float>(rows, g, h, n, packed, row_stride, feature, bits, thr, orow, og, oh, scratch,
                            d_totals, d_left, s);
}

void launch_partition_f64(const int32_t* rows, const double* g, const double* h, int64_t n,
                          const uint8_t* packed, int64_t row_stride, int feature, int bits, int thr,
                          int32_t* orow, double* og, double* oh, void* scratch, double* d_totals,
                          int64_t* d_left, cudaStream_t s) {
  launch_partition_t<double>(rows, g, h, n, packed, row_stride, feature, bits, thr, orow, og, oh, scratch,
                             d_totals, d_left, s);
}

}  // namespace hbg
