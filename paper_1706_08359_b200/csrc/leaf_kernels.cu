// leaf_kernels.cu — sm_100a kernels around the histogram build:
//   (2) leaf-indexed gather of g/h            (tree.cpp:11-25)
//   (4) histogram subtraction                 (row a10; absent in the reference)
//   (5) best-split scan over bins, fp64       (row a11, tree.cpp:59-112,163-182)
// plus the SoA -> HistogramBin conversion used by the host drop-in.
#include <algorithm>

#include "hbg_internal.h"

namespace hbg {

namespace {

constexpr int kGatherThreads = 256;
constexpr int kGatherMaxBlocks = 1184;  // 8 x 148 SMs

// leaf_g[i] = g[idx[i]] (fp32) and a per-block fp64 partial of the totals.
// Each block owns a contiguous chunk; the in-block reduction order is fixed,
// so totals are deterministic for a given count.
__global__ void gather_kernel(const int32_t* __restrict__ idx, int64_t n, const float* __restrict__ g,
                              const float* __restrict__ h, float* __restrict__ lg,
                              float* __restrict__ lh, int64_t chunk, double* __restrict__ partial) {
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t b1 = min(b0 + chunk, n);
  double sg = 0.0, sh = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const int32_t r = __ldg(idx + i);
    const float gv = __ldg(g + r);
    const float hv = __ldg(h + r);
    if (lg) lg[i] = gv;
    if (lh) lh[i] = hv;
    sg += gv;
    sh += hv;
  }
  __shared__ double red[2][kGatherThreads];
  red[0][threadIdx.x] = sg;
  red[1][threadIdx.x] = sh;
  __syncthreads();
  for (int s = kGatherThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      red[0][threadIdx.x] += red[0][threadIdx.x + s];
      red[1][threadIdx.x] += red[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = red[0][0];
    partial[2 * blockIdx.x + 1] = red[1][0];
  }
}

__global__ void gather_finalize_kernel(const double* partial, int blocks, double* totals) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double sg = 0.0, sh = 0.0;
    for (int b = 0; b < blocks; ++b) {
      sg += partial[2 * b];
      sh += partial[2 * b + 1];
    }
    totals[0] = sg;
    totals[1] = sh;
  }
}

__global__ void subtract_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                double* __restrict__ out, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = a[i] - b[i];
}

__global__ void hist_to_bins_kernel(const double* __restrict__ hist, int64_t cells,
                                    hbg_bin* __restrict__ bins) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cells;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    hbg_bin b;
    b.grad_sum = hist[i];
    b.hess_sum = hist[cells + i];
    b.count = static_cast<int64_t>(hist[2 * cells + i]);
    bins[i] = b;
  }
}

// tree.cpp:59-64
__device__ __forceinline__ double leaf_value(double g, double h, double lambda) {
  const double denom = h + lambda;
  return denom <= 0.0 ? 0.0 : -g / denom;
}

// tree.cpp:66-74
__device__ __forceinline__ double gain_of(double lg, double lh, double rg, double rh, double lambda) {
  const double dl = lh + lambda;
  const double dr = rh + lambda;
  const double dp = lh + rh + lambda;
  if (dl <= 0.0 || dr <= 0.0 || dp <= 0.0) return 0.0;
  const double g = __dadd_rn(lg, rg);
  // explicit rounding intrinsics: no FMA contraction, so gains are bit-identical
  // to the reference's double arithmetic on the same histogram
  return __dsub_rn(__dadd_rn(__ddiv_rn(__dmul_rn(lg, lg), dl), __ddiv_rn(__dmul_rn(rg, rg), dr)),
                   __ddiv_rn(__dmul_rn(g, g), dp));
}

struct Cand {
  double gain;
  int f, b;
  double lg, lh;
  int64_t lc;
};

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  if (a.f < 0) return false;
  if (b.f < 0) return true;
  return a.gain > b.gain || (a.gain == b.gain && a.f < b.f);
}

constexpr int kScanThreads = 1024;

// One CTA. Thread t scans features t, t+T, ... sequentially over bins in the
// reference order (find_best_threshold, tree.cpp:76-112: fp64 prefix sums,
// min_data skip/break, strict > so the smallest bin wins); the CTA then takes
// the max gain with the lowest feature id on ties (find_best_split :172).
__global__ void __launch_bounds__(kScanThreads) best_split_kernel(
    const double* __restrict__ hist, int d, int k, const double* d_totals, const int64_t* d_count,
    double gt, double ht, int64_t count, int64_t min_data, double lambda, hbg_split* out) {
  if (d_totals) {
    gt = d_totals[0];
    ht = d_totals[1];
  }
  if (d_count) count = *d_count;
  Cand best{0.0, -1, -1, 0.0, 0.0, 0};
  if (!(count < 2 * min_data || count < 2)) {  // early exit, tree.cpp:165
    const size_t D = static_cast<size_t>(d) * k;
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double* hg = hist + static_cast<size_t>(f) * k;
      const double* hh = hg + D;
      const double* hc = hg + 2 * D;
      double lg = 0.0, lh = 0.0;
      int64_t lc = 0;
      for (int b = 0; b < k - 1; ++b) {
        lg += hg[b];
        lh += hh[b];
        lc += static_cast<int64_t>(hc[b]);
        if (lc < min_data) continue;
        const int64_t rc = count - lc;
        if (rc < min_data) break;
        const double gain = gain_of(lg, lh, gt - lg, ht - lh, lambda);
        if (gain <= 0.0) continue;
        if (best.f < 0 || gain > best.gain || (gain == best.gain && f < best.f)) {
          best = Cand{gain, f, b, lg, lh, lc};
        }
      }
    }
  }
  __shared__ Cand red[kScanThreads];
  red[threadIdx.x] = best;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s && better(red[threadIdx.x + s], red[threadIdx.x]))
      red[threadIdx.x] = red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const Cand c = red[0];
    hbg_split o;
    o.feature = c.f;
    o.threshold_bin = c.b;
    o.gain = c.gain;
    o.left_grad = c.lg;
    o.left_hess = c.lh;
    o.left_count = c.lc;
    o.right_grad = gt - c.lg;
    o.right_hess = ht - c.lh;
    o.right_count = count - c.lc;
    o.left_value = leaf_value(c.lg, c.lh, lambda);
    o.right_value = leaf_value(gt - c.lg, ht - c.lh, lambda);
    if (c.f < 0) {
      o.threshold_bin = -1;
      o.gain = 0.0;
    }
    *out = o;
  }
}

__global__ void iota_kernel(int32_t* out, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<int32_t>(i);
}

}  // namespace

void launch_iota(int32_t* out, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 4736);
  iota_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(out, n);
  HBG_LAUNCH_CHECK();
}

size_t gather_scratch_doubles(int64_t n) {
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(kGatherMaxBlocks, (n + 2047) / 2048));
  return static_cast<size_t>(2 * blocks);
}

void launch_gather(const int32_t* idx, int64_t n, const float* g, const float* h, float* lg,
                   float* lh, double* totals, double* scratch, cudaStream_t s) {
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(kGatherMaxBlocks, (n + 2047) / 2048));
  const int64_t chunk = (n + blocks - 1) / blocks;
  gather_kernel<<<static_cast<unsigned>(blocks), kGatherThreads, 0, s>>>(idx, n, g, h, lg, lh,
                                                                         std::max<int64_t>(chunk, 1), scratch);
  HBG_LAUNCH_CHECK();
  gather_finalize_kernel<<<1, 32, 0, s>>>(scratch, static_cast<int>(blocks), totals);
  HBG_LAUNCH_CHECK();
}

void launch_subtract(const double* a, const double* b, double* out, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 2368);
  subtract_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(a, b, out, n);
  HBG_LAUNCH_CHECK();
}

void launch_hist_to_bins(const double* d_hist, int64_t cells, hbg_bin* d_bins, cudaStream_t s) {
  if (cells == 0) return;
  const int64_t blocks = std::min<int64_t>((cells + 255) / 256, 2368);
  hist_to_bins_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(d_hist, cells, d_bins);
  HBG_LAUNCH_CHECK();
}

void launch_best_split(const double* d_hist, int d, int k, const double* d_totals,
                       const int64_t* d_count, double gt, double ht, int64_t count,
                       int64_t min_data, double lambda, hbg_split* out, cudaStream_t s) {
  int threads = std::min(kScanThreads, std::max(32, (d + 31) / 32 * 32));
  // power of two for the tree reduction
  int p2 = 32;
  while (p2 < threads) p2 <<= 1;
  best_split_kernel<<<1, p2, 0, s>>>(d_hist, d, k, d_totals, d_count, gt, ht, count, min_data,
                                     lambda, out);
  HBG_LAUNCH_CHECK();
}

}  // namespace hbg
