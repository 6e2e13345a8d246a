// scan_device.cuh — the best-split scan over bins on the device (row a11:
// find_best_threshold / split_gain / optimal_leaf_value, tree.cpp:59-112),
// shared by the per-leaf scan kernels (leaf_kernels.cu) and the persistent
// tree grower (grow_persistent.cu). Not a public header.
#pragma once

#include <cstdint>

#include "hbg.h"

namespace hbg {
namespace dev {

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
  double lg, lh;  // the winner's left sums (prefix in bin order)
  int64_t lc;
};

// max gain; ties -> lowest feature, then lowest bin (tree.cpp:95,172)
__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  if (a.f < 0) return false;
  if (b.f < 0) return true;
  if (a.gain != b.gain) return a.gain > b.gain;
  return a.f < b.f || (a.f == b.f && a.b < b.b);
}

constexpr int kScanThreads = 256;

__device__ __forceinline__ Cand shfl_cand(const Cand& c, int src) {
  Cand o;
  o.gain = __shfl_sync(0xffffffffu, c.gain, src);
  o.f = __shfl_sync(0xffffffffu, c.f, src);
  o.b = __shfl_sync(0xffffffffu, c.b, src);
  o.lg = __shfl_sync(0xffffffffu, c.lg, src);
  o.lh = __shfl_sync(0xffffffffu, c.lh, src);
  o.lc = __shfl_sync(0xffffffffu, c.lc, src);
  return o;
}

// Best candidate of the CTA (strict total order `better`), in thread 0.
// Warp butterfly with shuffles, then one warp over the warp winners.
__device__ inline Cand block_best(Cand c, Cand* warp_best) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const Cand o = shfl_cand(c, lane ^ off);
    if (better(o, c)) c = o;
  }
  if (lane == 0) warp_best[w] = c;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    c = lane < nw ? warp_best[lane] : Cand{0.0, -1, -1, 0.0, 0.0, 0};
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const Cand o = shfl_cand(c, lane ^ off);
      if (better(o, c)) c = o;
    }
  }
  return c;
}
constexpr int kScanMaxChunkCells = 6144;  // features*bins staged per CTA (24 B each, dynamic smem)

__device__ inline void write_split(const Cand& c, double gt, double ht, int64_t count, double lambda,
                            hbg_split* out) {
  hbg_split o{};
  o.feature = c.f;
  o.threshold_bin = c.b;
  if (c.f >= 0) {
    o.gain = c.gain;
    o.left_grad = c.lg;
    o.left_hess = c.lh;
    o.left_count = c.lc;
    o.right_grad = gt - c.lg;
    o.right_hess = ht - c.lh;
    o.right_count = count - c.lc;
    o.left_value = leaf_value(c.lg, c.lh, lambda);
    o.right_value = leaf_value(gt - c.lg, ht - c.lh, lambda);
  } else {
    o.threshold_bin = -1;
  }
  *out = o;
}

// Scan of one staged chunk ([bin][feature] fp64 g/h/count, nf features from
// feature f0) -> this thread's best candidate. Staging must be complete
// (caller syncs); the prefix runs in place.
// Threads [tid of nth] of the CTA scan one staged histogram; every thread of
// the CTA must call (the prefix and the gains are separated by __syncthreads).
__device__ inline Cand scan_staged_t(double* pg, double* ph, double* pc, int nf, int k, int f0, double gt,
                                     double ht, double cnt, double md, double lambda, int tid, int nth) {
  // sequential prefix in bin order (the reference's order, tree.cpp:80-83),
  // one thread per (feature, statistic); loads batched ahead of the adds
  for (int t = tid; t < 3 * nf; t += nth) {
    const int f = t % nf, stat = t / nf;
    double* arr = stat == 0 ? pg : (stat == 1 ? ph : pc);
    double run = 0.0;  // integer-valued for counts: exact
    for (int b0 = 0; b0 < k; b0 += 8) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = b0 + j < k ? arr[(b0 + j) * nf + f] : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        run += v[j];
        if (b0 + j < k) arr[(b0 + j) * nf + f] = run;
      }
    }
  }
  __syncthreads();
  // every candidate bin's gain, branch-free in batches of 4 so the fp64
  // divisions of independent cells overlap
  Cand best{0.0, -1, -1, 0.0, 0.0, 0};
  const int cells = nf * k;
  for (int i0 = tid; i0 < cells; i0 += 4 * nth) {
    double gain[4];
    bool ok[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = min(i0 + j * nth, cells - 1);
      const int b = i / nf;
      const double lc = pc[i], lg = pg[i], lh = ph[i];
      ok[j] = i0 + j * nth < cells && b < k - 1 && lc >= md && cnt - lc >= md;
      gain[j] = gain_of(lg, lh, gt - lg, ht - lh, lambda);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + j * nth;
      if (!ok[j] || !(gain[j] > 0.0)) continue;
      const int b = i / nf, f = i - b * nf;
      const Cand c{gain[j], f0 + f, b, pg[i], ph[i], static_cast<int64_t>(pc[i])};
      if (better(c, best)) best = c;
    }
  }
  return best;
}

__device__ inline Cand scan_staged(double* pg, double* ph, double* pc, int nf, int k, int f0, double gt,
                                   double ht, double cnt, double md, double lambda) {
  return scan_staged_t(pg, ph, pc, nf, k, f0, gt, ht, cnt, md, lambda, static_cast<int>(threadIdx.x),
                       static_cast<int>(blockDim.x));
}

}  // namespace dev
}  // namespace hbg
