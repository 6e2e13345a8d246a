// leaf_kernels.cu — sm_100a kernels around the histogram build:
//   (2) leaf-indexed gather of g/h            (tree.cpp:11-25)
//   (4) histogram subtraction                 (row a10; absent in the reference)
//   (5) best-split scan over bins, fp64       (row a11, tree.cpp:59-112,163-182)
// plus the SoA -> HistogramBin conversion used by the host drop-in.
#include <algorithm>
#include <mutex>

#include "hbg_internal.h"
#include "scan_device.cuh"

namespace hbg {

namespace {

using namespace dev;

constexpr int kGatherThreads = 256;
constexpr int kGatherMaxBlocks = 1184;  // 8 x 148 SMs

// leaf_g[i] = g[idx[i]] (fp32) and a per-block fp64 partial of the totals.
// Each block owns a contiguous chunk; the in-block reduction order is fixed,
// so totals are deterministic for a given count.
template <typename T>
__global__ void gather_kernel(const int32_t* __restrict__ idx, int64_t n, const T* __restrict__ g,
                              const T* __restrict__ h, T* __restrict__ lg,
                              T* __restrict__ lh, int64_t chunk, double* __restrict__ partial) {
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t b1 = min(b0 + chunk, n);
  double sg = 0.0, sh = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const int32_t r = __ldg(idx + i);
    const T gv = __ldg(g + r);
    const T hv = __ldg(h + r);
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

// Fixed-order combine of the per-block partials: thread t sums a contiguous
// run of blocks, then a pairwise tree in thread order.
__global__ void gather_finalize_kernel(const double* partial, int blocks, double* totals) {
  __shared__ double r[2][256];
  const int t = threadIdx.x;
  const int chunk = (blocks + 255) / 256;
  double sg = 0.0, sh = 0.0;
  for (int b = t * chunk; b < min(blocks, (t + 1) * chunk); ++b) {
    sg += partial[2 * b];
    sh += partial[2 * b + 1];
  }
  r[0][t] = sg;
  r[1][t] = sh;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (t < st) {
      r[0][t] += r[0][t + st];
      r[1][t] += r[1][t + st];
    }
    __syncthreads();
  }
  if (t == 0) {
    totals[0] = r[0][0];
    totals[1] = r[1][0];
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

// One CTA per leaf histogram (blockIdx.x selects the leaf of a batch). The
// scan reproduces find_best_threshold (tree.cpp:76-112) exactly: per feature
// the prefix sums run sequentially in bin order in fp64 (one thread per
// feature over a shared-memory copy of the chunk), then every candidate bin's
// gain is evaluated in parallel with the reference's expression, and the
// winner is the max gain, lowest feature, lowest bin — the outcome of the
// reference's strict `>` loops (the `break` when the right side gets too
// small only removes bins whose right count is already below min_data).
struct FinishScanArgs {
  unsigned long long* acc;
  const int* exps;
  int d, k;
  double* small_out;
  double* large_io;
  int small_is_left;
  const double* totals;
  int64_t nl, nr;
  int lsplit, rsplit;
  int64_t min_data;
  double lambda;
  hbg_split* out;
  Cand* partial;
  int fchunk;
};

struct ScanArgs {
  const double* hist_base;
  int64_t hist_stride;
  int d, k;
  const double* d_totals;
  int64_t totals_stride;
  const int64_t* counts_dev;
  int64_t count0, count1;
  double gt, ht;
  int64_t min_data;
  double lambda;
  hbg_split* out_base;
  Cand* partial;  // [leaf][chunk] when gridDim.x > 1
  int fchunk;     // features per CTA
};

__device__ __forceinline__ void leaf_scalars(const ScanArgs& a, int leaf, double& gt, double& ht,
                                             int64_t& count) {
  gt = a.gt;
  ht = a.ht;
  if (a.d_totals) {
    gt = a.d_totals[leaf * a.totals_stride];
    ht = a.d_totals[leaf * a.totals_stride + 1];
  }
  count = a.counts_dev ? a.counts_dev[leaf] : (leaf == 0 ? a.count0 : a.count1);
}

// grid = (feature chunks, leaves). Each CTA scans fchunk features of one leaf;
// with several chunks the per-chunk winners go to `partial` and
// split_final_kernel picks among them. `better` is a strict total order on
// (gain, feature, bin), so the winner does not depend on the chunking.
__global__ void __launch_bounds__(kScanThreads) best_split_kernel(ScanArgs a) {
  const int leaf = blockIdx.y;
  const double* hist = a.hist_base + leaf * a.hist_stride;
  const int d = a.d, k = a.k;
  double gt, ht;
  int64_t count;
  leaf_scalars(a, leaf, gt, ht, count);
  extern __shared__ __align__(16) unsigned char scan_smem[];
  const int chunk_cells = a.fchunk * k;
  double* pg = reinterpret_cast<double*>(scan_smem);
  double* ph = pg + chunk_cells;
  double* pc = ph + chunk_cells;  // counts as exact doubles (< 2^53)
  __shared__ Cand warp_best[kScanThreads / 32];
  const bool splittable = !(count < 2 * a.min_data || count < 2);  // tree.cpp:165
  const size_t D = static_cast<size_t>(d) * k;
  const int f0 = blockIdx.x * a.fchunk;
  const int nf = splittable ? max(0, min(a.fchunk, d - f0)) : 0;
  const int cells = nf * k;
  // stage transposed, [bin][feature]: the prefix threads read consecutive addresses
#pragma unroll 6
  for (int i = threadIdx.x; i < cells; i += blockDim.x) {
    const size_t o = static_cast<size_t>(f0) * k + i;
    const int f = i / k, b = i - f * k;
    pg[b * nf + f] = hist[o];
    ph[b * nf + f] = hist[D + o];
    pc[b * nf + f] = hist[2 * D + o];
  }
  __syncthreads();
  Cand best = scan_staged(pg, ph, pc, nf, k, f0, gt, ht, static_cast<double>(count),
                          static_cast<double>(a.min_data), a.lambda);
  best = block_best(best, warp_best);
  if (threadIdx.x == 0) {
    if (gridDim.x == 1) {
      write_split(best, gt, ht, count, a.lambda, a.out_base + leaf);
    } else {
      a.partial[leaf * gridDim.x + blockIdx.x] = best;
    }
  }
}

// Small-leaf split tail, fused: fixed-point accumulator (small child) ->
// fp64 small histogram, larger child = parent - small in the parent's slot,
// accumulator cleared, and both children's split scans — one launch.
// grid = feature chunks; a CTA handles its chunk for both children.
__global__ void __launch_bounds__(kScanThreads) finish_scan_kernel(FinishScanArgs a) {
  const int d = a.d, k = a.k;
  const size_t D = static_cast<size_t>(d) * k;
  extern __shared__ __align__(16) unsigned char scan_smem[];
  const int chunk_cells = a.fchunk * k;
  double* st = reinterpret_cast<double*>(scan_smem);  // [child][stat][cells]
  __shared__ Cand warp_best[kScanThreads / 32];
  const int f0 = blockIdx.x * a.fchunk;
  const int nf = max(0, min(a.fchunk, d - f0));
  const int cells = nf * k;
  const double sg = ldexp(1.0, -a.exps[0]), sh = ldexp(1.0, -a.exps[1]);
  unsigned int* cnt = reinterpret_cast<unsigned int*>(a.acc + 2 * D);
  double* sm = st + (a.small_is_left ? 0 : 3 * chunk_cells);
  double* lg = st + (a.small_is_left ? 3 * chunk_cells : 0);
#pragma unroll 4
  for (int i = threadIdx.x; i < cells; i += blockDim.x) {
    const size_t o = static_cast<size_t>(f0) * k + i;
    const double vg = static_cast<double>(static_cast<long long>(a.acc[o])) * sg;
    const double vh = static_cast<double>(static_cast<long long>(a.acc[D + o])) * sh;
    const double vc = static_cast<double>(cnt[o]);
    a.acc[o] = 0ull;
    a.acc[D + o] = 0ull;
    cnt[o] = 0u;
    const double pg = a.large_io[o], ph = a.large_io[D + o], pc = a.large_io[2 * D + o];
    a.small_out[o] = vg;
    a.small_out[D + o] = vh;
    a.small_out[2 * D + o] = vc;
    a.large_io[o] = pg - vg;
    a.large_io[D + o] = ph - vh;
    a.large_io[2 * D + o] = pc - vc;
    const int f = i / k, b = i - f * k;
    const int t = b * nf + f;
    sm[t] = vg;
    sm[chunk_cells + t] = vh;
    sm[2 * chunk_cells + t] = vc;
    lg[t] = pg - vg;
    lg[chunk_cells + t] = ph - vh;
    lg[2 * chunk_cells + t] = pc - vc;
  }
  __syncthreads();
  for (int child = 0; child < 2; ++child) {
    const bool want = child == 0 ? a.lsplit : a.rsplit;
    if (!want) continue;  // uniform across the CTA
    double* base = st + child * 3 * chunk_cells;
    const double gt = a.totals[2 * child], ht = a.totals[2 * child + 1];
    const int64_t count = child == 0 ? a.nl : a.nr;
    Cand best = scan_staged(base, base + chunk_cells, base + 2 * chunk_cells, nf, k, f0, gt, ht,
                            static_cast<double>(count), static_cast<double>(a.min_data), a.lambda);
    best = block_best(best, warp_best);
    if (threadIdx.x == 0) {
      if (gridDim.x == 1) {
        write_split(best, gt, ht, count, a.lambda, a.out + child);
      } else {
        a.partial[child * gridDim.x + blockIdx.x] = best;
      }
    }
    __syncthreads();
  }
}

__global__ void split_final_kernel(ScanArgs a, int nchunks) {
  const int leaf = blockIdx.x;
  __shared__ Cand warp_best[kScanThreads / 32];
  Cand best{0.0, -1, -1, 0.0, 0.0, 0};
  for (int i = threadIdx.x; i < nchunks; i += blockDim.x) {
    const Cand c = a.partial[leaf * nchunks + i];
    if (better(c, best)) best = c;
  }
  best = block_best(best, warp_best);
  if (threadIdx.x == 0) {
    double gt, ht;
    int64_t count;
    leaf_scalars(a, leaf, gt, ht, count);
    write_split(best, gt, ht, count, a.lambda, a.out_base + leaf);
  }
}

// losses.cpp:24-26 (squared) and :57-60 (logistic), in fp64, stored fp32 (the
// bits32 per-element cast, histogram.cpp:97-98).
__global__ void grad_hess_kernel(int loss, const double* __restrict__ scores,
                                 const double* __restrict__ targets, int64_t n, float* __restrict__ g,
                                 float* __restrict__ h) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double s = scores[i], t = targets[i];
    if (loss == HBG_LOSS_SQUARED) {
      g[i] = static_cast<float>(s - t);
      h[i] = 1.0f;
    } else {
      const double p = 1.0 / (1.0 + exp(-s));
      const double hh = p * (1.0 - p);
      g[i] = static_cast<float>(p - t);
      h[i] = static_cast<float>(hh > 1e-16 ? hh : 1e-16);
    }
  }
}

// scores[row] += lr * value for every row of every final leaf (boosting.cpp:48-50).
__global__ void score_update_kernel(const LeafRange* __restrict__ leaves, const int32_t* __restrict__ rows0,
                                    const int32_t* __restrict__ rows1, double lr, double* __restrict__ scores) {
  const LeafRange L = leaves[blockIdx.y];
  const int32_t* rows = L.buf == 0 ? rows0 : rows1;
  const double add = lr * L.value;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L.count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    scores[rows[L.begin + i]] += add;
}

struct Parts8 {
  const double* p[8];
};

// out[i] = ((p0[i] + p1[i]) + p2[i]) + ... in part order (reduce_impl, histogram.cpp:108-127)
__global__ void reduce_parts_kernel(Parts8 parts, int nparts, int64_t n, double* out, int accumulate) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = accumulate ? out[i] : parts.p[0][i];
    for (int j = accumulate ? 0 : 1; j < nparts; ++j) v += parts.p[j][i];
    out[i] = v;
  }
}

__global__ void iota_kernel(int32_t* out, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<int32_t>(i);
}

}  // namespace

void configure_leaf_kernels() {
  for (const void* f : {reinterpret_cast<const void*>(gather_kernel<float>), reinterpret_cast<const void*>(gather_kernel<double>),
                        reinterpret_cast<const void*>(gather_finalize_kernel),
                        reinterpret_cast<const void*>(subtract_kernel),
                        reinterpret_cast<const void*>(hist_to_bins_kernel),
                        reinterpret_cast<const void*>(best_split_kernel),
                        reinterpret_cast<const void*>(split_final_kernel),
                        reinterpret_cast<const void*>(finish_scan_kernel),
                        reinterpret_cast<const void*>(reduce_parts_kernel),
                        reinterpret_cast<const void*>(iota_kernel),
                        reinterpret_cast<const void*>(grad_hess_kernel),
                        reinterpret_cast<const void*>(score_update_kernel)})
    set_max_shared_carveout(f);
}

void launch_grad_hess(int loss, const double* scores, const double* targets, int64_t n, float* g,
                      float* h, cudaStream_t s) {
  if (n == 0) return;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 4736);
  grad_hess_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(loss, scores, targets, n, g, h);
  HBG_LAUNCH_CHECK();
}

void launch_score_update(const LeafRange* leaves, int nleaves, const int32_t* rows0,
                         const int32_t* rows1, double lr, double* scores, cudaStream_t s) {
  if (nleaves == 0) return;
  score_update_kernel<<<dim3(32, nleaves), 256, 0, s>>>(leaves, rows0, rows1, lr, scores);
  HBG_LAUNCH_CHECK();
}

void launch_reduce_parts(const std::vector<const double*>& parts, int64_t n, double* out,
                         cudaStream_t s) {
  if (n == 0) return;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 2368);
  for (size_t j0 = 0; j0 < parts.size(); j0 += 8) {
    Parts8 p{};
    const int m = static_cast<int>(std::min<size_t>(8, parts.size() - j0));
    for (int j = 0; j < m; ++j) p.p[j] = parts[j0 + j];
    reduce_parts_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(p, m, n, out, j0 > 0 ? 1 : 0);
    HBG_LAUNCH_CHECK();
  }
}

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

template <typename T>
void launch_gather_t(const int32_t* idx, int64_t n, const T* g, const T* h, T* lg, T* lh, double* totals,
                     double* scratch, cudaStream_t s) {
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(kGatherMaxBlocks, (n + 2047) / 2048));
  const int64_t chunk = (n + blocks - 1) / blocks;
  gather_kernel<T><<<static_cast<unsigned>(blocks), kGatherThreads, 0, s>>>(idx, n, g, h, lg, lh,
                                                                            std::max<int64_t>(chunk, 1), scratch);
  HBG_LAUNCH_CHECK();
  gather_finalize_kernel<<<1, 256, 0, s>>>(scratch, static_cast<int>(blocks), totals);
  HBG_LAUNCH_CHECK();
}

void launch_gather(const int32_t* idx, int64_t n, const float* g, const float* h, float* lg,
                   float* lh, double* totals, double* scratch, cudaStream_t s) {
  launch_gather_t<float>(idx, n, g, h, lg, lh, totals, scratch, s);
}

void launch_gather_f64(const int32_t* idx, int64_t n, const double* g, const double* h, double* lg,
                       double* lh, double* totals, double* scratch, cudaStream_t s) {
  launch_gather_t<double>(idx, n, g, h, lg, lh, totals, scratch, s);
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

void* scan_scratch(size_t bytes);

void launch_finish_scan(const FinishScanArgsHost& h, cudaStream_t s) {
  static std::once_flag once[64];
  int dev = 0;
  HBG_CUDA(cudaGetDevice(&dev));
  std::call_once(once[dev & 63], [] {
    HBG_CUDA(cudaFuncSetAttribute(finish_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  2 * 3 * 2048 * 8));
  });
  FinishScanArgs a{};
  a.acc = static_cast<unsigned long long*>(h.acc);
  a.exps = h.exps;
  a.d = h.d;
  a.k = h.k;
  a.small_out = h.small_out;
  a.large_io = h.large_io;
  a.small_is_left = h.small_is_left;
  a.totals = h.totals;
  a.nl = h.nl;
  a.nr = h.nr;
  a.lsplit = h.lsplit;
  a.rsplit = h.rsplit;
  a.min_data = h.min_data;
  a.lambda = h.lambda;
  a.out = h.out;
  const int64_t cells = static_cast<int64_t>(h.d) * h.k;
  const int64_t per_cta = std::min<int64_t>(2048, std::max<int64_t>(2048, (cells + 147) / 148));
  a.fchunk = static_cast<int>(std::max<int64_t>(1, per_cta / h.k));
  const int nchunks = std::max(1, (h.d + a.fchunk - 1) / a.fchunk);
  if (nchunks > 1) a.partial = static_cast<Cand*>(scan_scratch(2 * static_cast<size_t>(nchunks) * sizeof(Cand)));
  finish_scan_kernel<<<nchunks, kScanThreads, static_cast<size_t>(a.fchunk) * h.k * 48, s>>>(a);
  HBG_LAUNCH_CHECK();
  if (nchunks > 1) {
    ScanArgs f{};
    f.d = h.d;
    f.k = h.k;
    f.d_totals = h.totals;
    f.totals_stride = 2;
    f.count0 = h.nl;
    f.count1 = h.nr;
    f.min_data = h.min_data;
    f.lambda = h.lambda;
    f.out_base = h.out;
    f.partial = a.partial;
    split_final_kernel<<<2, kScanThreads, 0, s>>>(f, nchunks);
    HBG_LAUNCH_CHECK();
  }
}

// Per-device grow-only scratch for the split scan's per-chunk winners. Calls
// on one device must be stream-ordered (documented: not re-entrant).
void* scan_scratch(size_t bytes) {
  static std::mutex mu;
  static void* buf[64] = {nullptr};
  static size_t cap[64] = {0};
  int dev = 0;
  HBG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (cap[dev & 63] < bytes) {
    if (buf[dev & 63]) HBG_CUDA(cudaFree(buf[dev & 63]));
    buf[dev & 63] = nullptr;
    cap[dev & 63] = 0;
    HBG_CUDA(cudaMalloc(&buf[dev & 63], bytes));
    cap[dev & 63] = bytes;
  }
  return buf[dev & 63];
}

void launch_best_split(const double* d_hist, int d, int k, const double* d_totals,
                       const int64_t* d_count, double gt, double ht, int64_t count,
                       int64_t min_data, double lambda, hbg_split* out, cudaStream_t s) {
  launch_best_split_batch(d_hist, 0, 1, d, k, d_totals, 0, d_count, count, 0, gt, ht, min_data,
                          lambda, out, s);
}

void launch_best_split_batch(const double* d_hist, int64_t hist_stride, int leaves, int d, int k,
                             const double* d_totals, int64_t totals_stride, const int64_t* d_counts,
                             int64_t count0, int64_t count1, double gt, double ht, int64_t min_data,
                             double lambda, hbg_split* out, cudaStream_t s) {
  require(k <= kScanMaxChunkCells, "max_bin too large for the split scan");
  require(leaves >= 1 && leaves <= 2, "split-scan batches hold one or two leaves");
  static std::once_flag once[64];
  int dev = 0;
  HBG_CUDA(cudaGetDevice(&dev));
  std::call_once(once[dev & 63], [] {
    HBG_CUDA(cudaFuncSetAttribute(best_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kScanMaxChunkCells * 24));
  });
  ScanArgs a{};
  a.hist_base = d_hist;
  a.hist_stride = hist_stride;
  a.d = d;
  a.k = k;
  a.d_totals = d_totals;
  a.totals_stride = totals_stride;
  a.counts_dev = d_counts;
  a.count0 = count0;
  a.count1 = count1;
  a.gt = gt;
  a.ht = ht;
  a.min_data = min_data;
  a.lambda = lambda;
  a.out_base = out;
  // Spread wide histograms over ~one wave of CTAs; narrow ones stay in one CTA.
  const int64_t cells = static_cast<int64_t>(d) * k;
  const int64_t per_cta = std::min<int64_t>(kScanMaxChunkCells, std::max<int64_t>(2048, (cells + 147) / 148));
  a.fchunk = static_cast<int>(std::max<int64_t>(1, per_cta / k));
  const int nchunks = std::max(1, (d + a.fchunk - 1) / a.fchunk);
  if (nchunks > 1) a.partial = static_cast<Cand*>(scan_scratch(static_cast<size_t>(leaves) * nchunks * sizeof(Cand)));
  const size_t smem = static_cast<size_t>(a.fchunk) * k * 24;
  best_split_kernel<<<dim3(nchunks, leaves), kScanThreads, smem, s>>>(a);
  HBG_LAUNCH_CHECK();
  if (nchunks > 1) {
    split_final_kernel<<<leaves, kScanThreads, 0, s>>>(a, nchunks);
    HBG_LAUNCH_CHECK();
  }
}

}  // namespace hbg
