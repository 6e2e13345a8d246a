// hist_kernels.cu — sm_100a kernels for subsystems (1) packed layout and
// (3) the feature-histogram build.
//
// Histogram kernel design (DESIGN.md §3 has the measurements behind it):
//  * Rows in lanes. A warp takes a 32-row tile of the leaf; lane l owns leaf
//    position t+l and loads that row's 32-feature slice (32 B at 8-bit, 16 B
//    at 4-bit) with 128-bit loads, plus its fp32 g/h.
//  * Feature rotation (the paper's Alg. 2 "rotated" schedule, reference
//    lockstep.cpp:98-105): at step p lane l updates feature (l + p) mod 32, so
//    the 32 lanes of every shared-memory instruction hit 32 distinct feature
//    columns. With the [bin][feature] cell layout the bank is the feature,
//    so every LDS/STS/ATOMS is bank-conflict-free whatever the bins are.
//  * Per-warp private fp32 {g,h} cells (plain LDS.64/FADD/STS.64 — sm_100a has
//    no native shared fp32 atomic; atomicAdd(float) is a CAS loop measured 5x
//    slower) and CTA-shared u32 counts via the native ATOMS.POPC.INC. The
//    RMW steps stay in program order (volatile asm), which keeps lane A's
//    step-p store ahead of lane B's step-(p+1) load of the same cell.
//  * Each CTA folds its warps' cells in a fixed order and writes one fp32/u32
//    partial; reduce_partials_kernel sums partials over row segments in a
//    fixed order in fp64. Results are therefore deterministic for a given
//    (leaf size, feature count, GPU), like the reference's fixed 64 Ki-chunk
//    reduction (histogram.cpp:159-215).
#include <algorithm>
#include <mutex>
#include <type_traits>
#include <vector>

#include <cooperative_groups.h>

#include "hbg_internal.h"
#include "hist_device.cuh"

namespace hbg {

namespace {

using namespace dev;

template <typename T>
struct TileIn {
  int32_t row;  // raw int32 row id (row_index_t): widening it right after the
                // load would make the load's consumer immediate and stall on it
  T g, h;
};

// Distributed shared memory: this CTA's address of `p`, in cluster rank q's
// shared memory (mapa + ld.shared::cluster — not a generic load).
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, int q) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(dev::smem_addr(p)), "r"(q));
  return r;
}
__device__ __forceinline__ float ld_dsmem(const float* p, int q) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(dsmem_addr(p, q)));
  return v;
}
__device__ __forceinline__ double ld_dsmem(const double* p, int q) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(dsmem_addr(p, q)));
  return v;
}
__device__ __forceinline__ uint4 ld_dsmem_v4(const void* p, int q) {  // 16-byte aligned
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(dsmem_addr(p, q)));
  return v;
}
__device__ __forceinline__ uint32_t ld_dsmem(const uint32_t* p, int q) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(dsmem_addr(p, q)));
  return v;
}

__device__ __forceinline__ void hist_stamp(const HistArgs& a, int slot) {
  if (a.prof != nullptr && blockIdx.x == static_cast<unsigned>(a.prof_cta) && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.prof[slot] = t;
  }
}

// T = float: bits32 (the reference's per-element fp32 cast, histogram.cpp:97-98);
// T = double: bits64 (reference_impl<double>, histogram.cpp:131-145) — fp64
// inputs, fp64 per-warp cells, fp64 partials.
template <int BITS, int K, bool kRowIndexed, typename T>
__global__ void __launch_bounds__(K >= 256 ? 128 : 512, BITS == 4 ? 2 : 1) hist_kernel(HistArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int kCells = K * 32;
  constexpr int kCellBytes = 2 * sizeof(T);
  using T2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  // warps [0, gb * wpg) own {g,h} cells and process rows; a fused launch may
  // add warps that only help clear, fold and reduce
  const int cw = a.gb * a.wpg;
  T2* gh = reinterpret_cast<T2*>(smem);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + static_cast<size_t>(cw) * kCells * kCellBytes);
  const T* __restrict__ ag = static_cast<const T*>(a.g);
  const T* __restrict__ ah = static_cast<const T*>(a.h);
  // Programmatic dependent launch: the next kernel in the stream may start
  // launching now (its CTAs become resident as ours exit); everything before
  // griddepcontrol.wait touches only this CTA's shared memory, so the clear
  // overlaps the previous kernel's tail. (Both are no-ops without PDL.)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  {
    const int n16 = (cw * kCells * kCellBytes + a.gb * kCells * 4) / 16;
    uint4* z = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // inputs and outputs of earlier kernels settled
  hist_stamp(a, 0);

  // a cluster's CTAs are consecutive: there, nclusters clusters per group block
  const int clu = a.cluster > 1 ? static_cast<int>(blockIdx.x) / a.cluster : 0;
  const int bi = a.cluster > 1 ? clu / a.nclusters : blockIdx.x % a.nblocks;
  const int seg = a.cluster > 1 ? (clu % a.nclusters) * a.cluster + static_cast<int>(blockIdx.x) % a.cluster
                                : blockIdx.x / a.nblocks;
  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int gl = w % a.gb;
  const int sub = w / a.gb;
  const int group = bi * a.gb + gl;
  const bool row_warp = sub < a.wpg && group < a.num_groups;
  {
    const int64_t s0 = static_cast<int64_t>(seg) * a.seg_len;
    const int64_t s1 = min(s0 + a.seg_len, a.n);
    const uint32_t gh_base = smem_addr(gh + static_cast<size_t>(w) * kCells);
    uint32_t* cnt_g = cnt + static_cast<size_t>(gl) * kCells;
    const unsigned char* base = a.packed + static_cast<int64_t>(group) * a.group_stride;
    constexpr int R = rows_per_lane<K, T>();
    const int64_t step = static_cast<int64_t>(a.wpg) * 32 * R;

    // Two-stage software pipeline, so no load waits on another load in the
    // same iteration (issue is in order): stage A fetches the leaf entries
    // (row id, g, h) of tile t+2s, stage B fetches the packed slices of tile
    // t+s using the row ids stage A delivered one iteration earlier, and the
    // update loop consumes tile t. A tile is 32*R rows; lane l owns rows
    // t + 32r + l.
    auto fetch_entry = [&](int64_t t, TileIn<T> (&in)[R]) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t pos = t + 32 * r + lane;
        if (pos < s1) {
          in[r].row = __ldg(a.idx + pos);  // never null: the identity leaf uses an iota array
          if constexpr (!kRowIndexed) {
            in[r].g = __ldg(ag + pos);
            in[r].h = __ldg(ah + pos);
          }
        } else {
          in[r].row = -1;
          in[r].g = T(0);
          in[r].h = T(0);
        }
      }
    };
    auto fetch_slice = [&](TileIn<T> (&in)[R], Slice<BITS> (&sl)[R]) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (in[r].row >= 0) {
          if constexpr (kRowIndexed) {
            in[r].g = __ldg(ag + in[r].row);
            in[r].h = __ldg(ah + in[r].row);
          }
          load_slice<BITS>(base + static_cast<int64_t>(in[r].row) * a.row_stride, sl[r]);
        } else {
#pragma unroll
          for (int j = 0; j < Slice<BITS>::kWords; ++j) sl[r].w[j] = 0;
        }
      }
    };

    int64_t t = s0 + static_cast<int64_t>(sub) * 32 * R;
    TileIn<T> e0[R], e1[R];
    Slice<BITS> cur[R];
    // the pipeline's first loads are in flight while the cells are cleared
    if (row_warp) {
      fetch_entry(t, e0);
      fetch_entry(t + step, e1);
      fetch_slice(e0, cur);
    }
    __syncthreads();  // cells cleared
    hist_stamp(a, 1);
    for (; row_warp && t < s1; t += step) {
      TileIn<T> e2[R];
      Slice<BITS> nxt[R];
      fetch_entry(t + 2 * step, e2);  // stage A (t + 2s)
      fetch_slice(e1, nxt);           // stage B (t + s)
#pragma unroll
      for (int r = 0; r < R; ++r) rotate_slice<BITS>(cur[r], lane);
      if (t + 32 * R <= s1) {
        T g[R], h[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          g[r] = e0[r].g;
          h[r] = e0[r].h;
        }
#pragma unroll
        for (int p = 0; p < 32; ++p) update_step_rows<BITS, K, R, T>(cur, p, lane, gh_base, cnt_g, g, h);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool valid = e0[r].row >= 0;
#pragma unroll
          for (int p = 0; p < 32; ++p)
            update_step<BITS, K, true, T>(cur[r], p, lane, gh_base, cnt_g, e0[r].g, e0[r].h, valid);
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        e0[r] = e1[r];
        e1[r] = e2[r];
        cur[r] = nxt[r];
      }
    }
  }
  __syncthreads();
  hist_stamp(a, 2);

  // Fold the warps of each group in a fixed order.
  auto fold = [&](int g2, int c, T& sg, T& sh) {
    sg = T(0);
    sh = T(0);
#pragma unroll 4
    for (int s = 0; s < a.wpg; ++s) {
      const T2 v = gh[static_cast<size_t>(s * a.gb + g2) * kCells + c];
      sg += v.x;
      sh += v.y;
    }
  };
  if (a.cluster > 1) {
    // Cluster mode: this CTA folds its warps into its own sub-histogram in
    // shared memory; after a cluster barrier, CTA r sums cells [r*per, ...)
    // over the cluster's C sub-histograms through distributed shared memory
    // (ranks in order: deterministic). One cluster per group block writes the
    // fp64 histogram directly; with several, each writes its fp64 sums to HBM
    // and the last cluster to arrive (device-scope counter) adds the clusters'
    // sums in cluster order and writes the histogram.
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int ncell = a.gb * kCells;
    T* sub_g = reinterpret_cast<T*>(smem + static_cast<size_t>(cw) * kCells * kCellBytes +
                                    static_cast<size_t>(a.gb) * kCells * 4);
    T* sub_h = sub_g + ncell;
    uint32_t* sub_c = reinterpret_cast<uint32_t*>(sub_h + ncell);
    int& last_flag = *reinterpret_cast<int*>(sub_c + ncell);  // (dynamic: the limit is for all shared memory)
    for (int i = threadIdx.x; i < ncell; i += blockDim.x) {
      const int g2 = i / kCells, c = i - g2 * kCells;
      T sg, sh;
      fold(g2, c, sg, sh);
      sub_g[i] = sg;
      sub_h[i] = sh;
      sub_c[i] = cnt[i];
    }
    hist_stamp(a, 3);
    cl.sync();
    hist_stamp(a, 4);
    const int C = static_cast<int>(cl.num_blocks()), r = static_cast<int>(cl.block_rank());
    const int per = (ncell + C - 1) / C;
    const int i0 = r * per, i1 = min(ncell, (r + 1) * per);
    const size_t D = static_cast<size_t>(a.d) * a.max_bin;
    const int nk = a.nclusters, kk = clu % nk;
    double* cg_ = static_cast<double*>(a.part_g);
    double* ch_ = static_cast<double*>(a.part_h);
    auto emit = [&](int i, double vg, double vh, unsigned long long vc) {
      const int g2 = i / kCells, c = i - g2 * kCells;
      const int bin = c >> 5, f = (bi * a.gb + g2) * 32 + (c & 31);
      if (f >= a.d || bin >= a.max_bin) return;
      const size_t o = static_cast<size_t>(f) * a.max_bin + bin;
      a.out[o] = vg;
      a.out[D + o] = vh;
      a.out[2 * D + o] = static_cast<double>(vc);
      if (a.parent) {
        const double pg = a.parent[o], ph = a.parent[D + o], pc = a.parent[2 * D + o];
        a.sibling[o] = pg - vg;
        a.sibling[D + o] = ph - vh;
        a.sibling[2 * D + o] = pc - static_cast<double>(vc);
      }
    };
    // Gather cells [i0, i1) of the C sub-histograms into local staging (the
    // per-warp cells and the count cells are free once folded) as 16-byte
    // remote loads, all of a thread's loads in flight at once; the CTAs start
    // at different ranks so they do not all read the same CTA's shared memory
    // at the same time. Then the sums, in rank order (deterministic).
    {
      T* st_g = reinterpret_cast<T*>(smem);  // [C][per]: C * per == ncell <= cw * kCells
      T* st_h = st_g + static_cast<size_t>(C) * per;
      uint32_t* st_c = cnt;                  // [C][per]: the count cells
      const int nloc = max(0, i1 - i0);
      const int vgh = nloc * static_cast<int>(sizeof(T)) / 16, vc = nloc / 4;  // 16-B vectors per array
      const int per_rank = 2 * vgh + vc;
      const int items = C * per_rank;
      constexpr int kBatch = 8;
      for (int base = 0; base < items; base += kBatch * static_cast<int>(blockDim.x)) {
        uint4 v[kBatch];
        uint4* dst[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
          const int it = base + b * static_cast<int>(blockDim.x) + static_cast<int>(threadIdx.x);
          dst[b] = nullptr;
          if (it < items) {
            const int qq = it / per_rank, k = it - qq * per_rank;
            const int q = qq + r < C ? qq + r : qq + r - C;
            const void* src;
            if (k < vgh) {
              src = reinterpret_cast<const uint4*>(sub_g + i0) + k;
              dst[b] = reinterpret_cast<uint4*>(st_g + static_cast<size_t>(q) * per) + k;
            } else if (k < 2 * vgh) {
              src = reinterpret_cast<const uint4*>(sub_h + i0) + (k - vgh);
              dst[b] = reinterpret_cast<uint4*>(st_h + static_cast<size_t>(q) * per) + (k - vgh);
            } else {
              src = reinterpret_cast<const uint4*>(sub_c + i0) + (k - 2 * vgh);
              dst[b] = reinterpret_cast<uint4*>(st_c + static_cast<size_t>(q) * per) + (k - 2 * vgh);
            }
            v[b] = ld_dsmem_v4(src, q);
          }
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b)
          if (dst[b] != nullptr) *dst[b] = v[b];
      }
      __syncthreads();
    }
    for (int i = i0 + static_cast<int>(threadIdx.x); i < i1; i += blockDim.x) {
      const T* st_g = reinterpret_cast<const T*>(smem);
      const T* st_h = st_g + static_cast<size_t>(C) * per;
      double vg = 0.0, vh = 0.0;
      unsigned long long vc = 0;
      for (int q = 0; q < C; ++q) {
        vg += static_cast<double>(st_g[q * per + (i - i0)]);
        vh += static_cast<double>(st_h[q * per + (i - i0)]);
        vc += cnt[q * per + (i - i0)];
      }
      if (nk == 1) {
        emit(i, vg, vh, vc);
      } else {
        const size_t o = (static_cast<size_t>(bi) * nk + kk) * ncell + i;
        cg_[o] = vg;
        ch_[o] = vh;
        a.part_c[o] = static_cast<uint32_t>(vc);
      }
    }
    hist_stamp(a, 6);  // this CTA's share reduced
    if (nk > 1) {
      __threadfence();  // this cluster's sums are visible before it is counted
      cl.sync();
      if (r == 0 && threadIdx.x == 0) {
        const unsigned old = atomicAdd(a.bar + bi, 1u);
        last_flag = old == static_cast<unsigned>(nk - 1);
        if (last_flag) a.bar[bi] = 0u;  // every cluster has arrived: reset for the next launch
      }
      cl.sync();
      if (*cl.map_shared_rank(&last_flag, 0)) {
        __threadfence();
        for (int i = i0 + static_cast<int>(threadIdx.x); i < i1; i += blockDim.x) {
          double vg = 0.0, vh = 0.0;
          unsigned long long vc = 0;
#pragma unroll 4
          for (int q = 0; q < nk; ++q) {
            const size_t o = (static_cast<size_t>(bi) * nk + q) * ncell + i;
            vg += __ldcg(cg_ + o);
            vh += __ldcg(ch_ + o);
            vc += __ldcg(a.part_c + o);
          }
          emit(i, vg, vh, vc);
        }
      }
    }
    cl.sync();  // no CTA leaves while another still reads its shared memory
    hist_stamp(a, 5);
    return;
  }
  if (a.direct) {
    // Single row segment: write the final fp64 histogram (and the fused
    // sibling = parent - this) in output order, so global accesses coalesce;
    // a batch of parent loads is issued before any store (sibling may alias
    // parent element-wise).
    const int f0 = bi * a.gb * 32;
    const int nf = max(0, min(a.gb * 32, a.d - f0));
    const int total = nf * a.max_bin;
    const size_t D = static_cast<size_t>(a.d) * a.max_bin;
    const size_t base = static_cast<size_t>(f0) * a.max_bin;
    constexpr int B = 4;
    for (int i0 = threadIdx.x; i0 < total; i0 += B * blockDim.x) {
      double vg[B], vh[B], vc[B], pg[B], ph[B], pc[B];
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int i = i0 + j * blockDim.x;
        if (i < total) {
          const int fl = i / a.max_bin, bin = i - fl * a.max_bin;
          const int g2 = fl >> 5;
          const int c = (bin << 5) | (fl & 31);
          T sg, sh;
          fold(g2, c, sg, sh);
          vg[j] = sg;
          vh[j] = sh;
          vc[j] = cnt[static_cast<size_t>(g2) * kCells + c];
          if (a.parent) {
            pg[j] = a.parent[base + i];
            ph[j] = a.parent[D + base + i];
            pc[j] = a.parent[2 * D + base + i];
          }
        }
      }
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int i = i0 + j * blockDim.x;
        if (i < total) {
          a.out[base + i] = vg[j];
          a.out[D + base + i] = vh[j];
          a.out[2 * D + base + i] = vc[j];
          if (a.parent) {
            a.sibling[base + i] = pg[j] - vg[j];
            a.sibling[D + base + i] = ph[j] - vh[j];
            a.sibling[2 * D + base + i] = pc[j] - vc[j];
          }
        }
      }
    }
    hist_stamp(a, 5);
    return;
  }
  // One partial per CTA (T sums, u32 counts).
  T* part_g = static_cast<T*>(a.part_g);
  T* part_h = static_cast<T*>(a.part_h);
  for (int i = threadIdx.x; i < a.gb * kCells; i += blockDim.x) {
    const int g2 = i / kCells;
    const int c = i - g2 * kCells;
    T sg, sh;
    fold(g2, c, sg, sh);
    const size_t o = (static_cast<size_t>(blockIdx.x) * a.gb + g2) * kCells + c;
    part_g[o] = sg;
    part_h[o] = sh;
    a.part_c[o] = cnt[static_cast<size_t>(g2) * kCells + c];
  }
  hist_stamp(a, 3);
}

// out (SoA fp64 [3][d][max_bin]) = fixed-order fp64 sum of the CTA partials
// over row segments. Block = one bin row of one slice group (32 cells, lane =
// feature) x kReduceWarps warps; warp w sums segments w, w+W, ... in order,
// then the warps' sums are combined in warp order: deterministic, and the
// partial reads are 128-byte coalesced with W independent streams per cell.
constexpr int kReduceWarps = 32;

template <typename T>
__global__ void __launch_bounds__(kReduceWarps * 32) reduce_partials_kernel(
    HistArgs a, int nseg, int k_alloc, int d, int max_bin, double* out, const double* parent,
    double* sibling) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the histogram kernel's partials (PDL launch)
  const T* part_g = static_cast<const T*>(a.part_g);
  const T* part_h = static_cast<const T*>(a.part_h);
  const int cells = k_alloc * 32;
  const int group = blockIdx.y;
  const int bin = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int c = bin * 32 + lane;
  const int bi = group / a.gb;
  const int gl = group - bi * a.gb;
  double sg = 0.0, sh = 0.0;
  uint64_t sc = 0;
#pragma unroll 8
  for (int s = w; s < nseg; s += kReduceWarps) {
    const size_t cta = static_cast<size_t>(s) * a.nblocks + bi;
    const size_t o = (cta * a.gb + gl) * cells + c;
    sg += static_cast<double>(part_g[o]);
    sh += static_cast<double>(part_h[o]);
    sc += a.part_c[o];
  }
  __shared__ double rg[kReduceWarps][32], rh[kReduceWarps][32];
  __shared__ uint64_t rc[kReduceWarps][32];
  rg[w][lane] = sg;
  rh[w][lane] = sh;
  rc[w][lane] = sc;
  __syncthreads();
  if (w != 0) return;
  for (int i = 1; i < kReduceWarps; ++i) {
    sg += rg[i][lane];
    sh += rh[i][lane];
    sc += rc[i][lane];
  }
  const int f = group * 32 + lane;
  if (f >= d || bin >= max_bin) return;
  const size_t D = static_cast<size_t>(d) * max_bin;
  const size_t o = static_cast<size_t>(f) * max_bin + bin;
  out[o] = sg;
  out[D + o] = sh;
  out[2 * D + o] = static_cast<double>(sc);
  if (parent) {  // histogram subtraction (row a10), fused
    const double pg = parent[o], ph = parent[D + o], pc = parent[2 * D + o];
    sibling[o] = pg - sg;
    sibling[D + o] = ph - sh;
    sibling[2 * D + o] = pc - static_cast<double>(sc);
  }
}

// Row-sharded histogram with the allreduce FUSED into the
// reduction: block (bin, group) reduces its bin row of this rank's partials
// (as reduce_partials_kernel), publishes the row in this rank's exchange area
// (data, fence.sys, flag = tag with release semantics), then reads every
// rank's row over peer memory (NVLink) and sums them in rank order — every
// rank ends with the bit-identical global histogram, with no separate
// collective launch. Rows alternate between two parities per call; a rank
// starts call c only after its call c-1 read every peer's c-1 rows, which the
// peers published after finishing their c-2 reads (same parity).
constexpr int kXRow = 16 + 3 * 32;  // doubles per exchanged row: flag + pad, 32 x (g, h, count)

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const double* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys_u64(double* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Block b handles bin rows b, b + gridDim.x, ... (a small grid: blocks that
// wait for peers must not keep other kernels off the SMs when ranks share a
// GPU). Phase 1 publishes all its rows, phase 2 sums every rank's rows.
constexpr int kXBlocks = 32;

template <typename T>
__global__ void __launch_bounds__(kReduceWarps * 32) reduce_exchange_kernel(
    HistArgs a, int nseg, int k_alloc, int d, int max_bin, int nbins, double* out, PeerHistArgs x) {
  const T* part_g = static_cast<const T*>(a.part_g);
  const T* part_h = static_cast<const T*>(a.part_h);
  const int cells = k_alloc * 32;
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int nrows = nbins * a.num_groups;
  __shared__ double rg[kReduceWarps][32], rh[kReduceWarps][32];
  __shared__ uint64_t rc[kReduceWarps][32];
  for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
    const int group = row / nbins, bin = row - group * nbins;
    const int c = bin * 32 + lane;
    const int bi = group / a.gb;
    const int gl = group - bi * a.gb;
    double sg = 0.0, sh = 0.0;
    uint64_t sc = 0;
#pragma unroll 4
    for (int s = w; s < nseg; s += kReduceWarps) {
      const size_t cta = static_cast<size_t>(s) * a.nblocks + bi;
      const size_t o = (cta * a.gb + gl) * cells + c;
      sg += static_cast<double>(part_g[o]);
      sh += static_cast<double>(part_h[o]);
      sc += a.part_c[o];
    }
    rg[w][lane] = sg;
    rh[w][lane] = sh;
    rc[w][lane] = sc;
    __syncthreads();
    if (w == 0) {
      for (int i = 1; i < kReduceWarps; ++i) {
        sg += rg[i][lane];
        sh += rh[i][lane];
        sc += rc[i][lane];
      }
      double* mine = x.xown + (static_cast<size_t>(x.parity) * nrows + row) * kXRow;
      mine[16 + lane] = sg;
      mine[48 + lane] = sh;
      mine[80 + lane] = static_cast<double>(sc);
      __syncwarp();
      if (lane == 0) {
        __threadfence_system();
        st_release_sys_u64(mine, x.tag);
      }
    }
    __syncthreads();
  }
  if (w != 0) return;
  for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
    const int group = row / nbins, bin = row - group * nbins;
    double tg = 0.0, th = 0.0, tc = 0.0;
    for (int r = 0; r < x.nranks; ++r) {
      const double* blk = x.xpeer[r] + (static_cast<size_t>(x.parity) * nrows + row) * kXRow;
      if (lane == 0) {
        const long long t0 = clock64();
        while (ld_acquire_sys_u64(blk) != x.tag) {
          if (clock64() - t0 > x.timeout_cycles) {
            atomicCAS(x.error, 0, 1);
            break;
          }
        }
      }
      __syncwarp();
      const double g = __ldcv(blk + 16 + lane), h = __ldcv(blk + 48 + lane), n = __ldcv(blk + 80 + lane);
      tg = r == 0 ? g : tg + g;
      th = r == 0 ? h : th + h;
      tc = r == 0 ? n : tc + n;
    }
    const int f = group * 32 + lane;
    if (f >= d || bin >= max_bin) continue;
    const size_t D = static_cast<size_t>(d) * max_bin;
    const size_t o = static_cast<size_t>(f) * max_bin + bin;
    out[o] = tg;
    out[D + o] = th;
    out[2 * D + o] = tc;
  }
}

// Column-major uint8 bins -> row-major packed words at pack_feature_tuples
// bit positions (binning.cpp:141-156): word w of a row holds features
// w*fpw .. w*fpw+fpw-1 at bits*p. One launch covers one 32-feature slice
// group (its words_per_slice words); pad slots are 0.
__global__ void pack_kernel(const uint8_t* cols, int f0, int nf, int64_t n, int max_bin, int bits,
                            int64_t gs_words, uint32_t* packed, int* bad) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int fpw = 32 / bits;
  const int w = f0 / fpw + blockIdx.y;
  uint32_t word = 0;
  for (int p = 0; p < fpw; ++p) {
    const int fl = blockIdx.y * fpw + p;  // feature within the group
    if (fl >= nf) break;
    const uint32_t b = cols[static_cast<size_t>(fl) * n + r];
    if (b >= static_cast<uint32_t>(max_bin)) atomicOr(bad, 1);
    word |= b << (bits * p);
  }
  const int wps = 32 / fpw;  // words per 32-feature slice (group-planar layout)
  packed[static_cast<size_t>(w / wps) * gs_words + static_cast<size_t>(r) * wps + w % wps] = word;
}

__global__ void f64_to_f32_kernel(const double* in, float* out, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<float>(in[i]);
}

}  // namespace

// Every kernel of the library asks for the maximum shared-memory carveout, so
// back-to-back launches of kernels with different shared-memory footprints
// (the per-split sequence of the tree grower) never force the SM to
// reconfigure its L1/shared split between launches.
void set_max_shared_carveout(const void* func) {
  HBG_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout,
                                cudaSharedmemCarveoutMaxShared));
}

namespace {

template <int BITS, int K, typename T>
void set_smem_attr_t(int device) {
  static std::once_flag once[64];
  std::call_once(once[device & 63], [] {
    HBG_CUDA(cudaFuncSetAttribute(hist_kernel<BITS, K, false, T>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    HBG_CUDA(cudaFuncSetAttribute(hist_kernel<BITS, K, true, T>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    set_max_shared_carveout(reinterpret_cast<const void*>(hist_kernel<BITS, K, false, T>));
    set_max_shared_carveout(reinterpret_cast<const void*>(hist_kernel<BITS, K, true, T>));
    HBG_CUDA(cudaFuncSetAttribute(hist_kernel<BITS, K, false, T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    HBG_CUDA(cudaFuncSetAttribute(hist_kernel<BITS, K, true, T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
}

template <int BITS, int K>
void set_smem_attr(int device) {
  set_smem_attr_t<BITS, K, float>(device);
  set_smem_attr_t<BITS, K, double>(device);
}

template <int BITS, int K, typename T>
int occupancy(int threads, size_t smem, int device) {
  set_smem_attr<BITS, K>(device);
  int blocks = 0;
  HBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, hist_kernel<BITS, K, false, T>, threads,
                                                         smem));
  return std::max(blocks, 1);
}

// Occupancy queries are cached per (device, variant, block, smem): the plan
// is recomputed for every leaf of the per-leaf drop-in, where a driver query
// per call was a measurable part of a deep leaf's few microseconds.
int occupancy_for(int bits, int k_alloc, int threads, size_t smem, int device, int acc_bytes) {
  struct Key {
    int device, bits, k, threads, acc;
    size_t smem;
    int occ;
  };
  static std::mutex m;
  static std::vector<Key> cache;
  {
    std::lock_guard<std::mutex> lk(m);
    for (const Key& c : cache)
      if (c.device == device && c.bits == bits && c.k == k_alloc && c.threads == threads && c.acc == acc_bytes &&
          c.smem == smem)
        return c.occ;
  }
  int occ;
  const bool f64 = acc_bytes == 8;
  if (bits == 4) occ = f64 ? occupancy<4, 16, double>(threads, smem, device) : occupancy<4, 16, float>(threads, smem, device);
  else if (k_alloc == 64) occ = f64 ? occupancy<8, 64, double>(threads, smem, device) : occupancy<8, 64, float>(threads, smem, device);
  else if (k_alloc == 128) occ = f64 ? occupancy<8, 128, double>(threads, smem, device) : occupancy<8, 128, float>(threads, smem, device);
  else occ = f64 ? occupancy<8, 256, double>(threads, smem, device) : occupancy<8, 256, float>(threads, smem, device);
  std::lock_guard<std::mutex> lk(m);
  cache.push_back(Key{device, bits, k_alloc, threads, acc_bytes, smem, occ});
  return occ;
}

using HistKernel = void (*)(HistArgs);

template <typename T>
HistKernel hist_kernel_ptr_t(int bits, int k_alloc, bool ri) {
  if (bits == 4) return ri ? hist_kernel<4, 16, true, T> : hist_kernel<4, 16, false, T>;
  if (k_alloc == 64) return ri ? hist_kernel<8, 64, true, T> : hist_kernel<8, 64, false, T>;
  if (k_alloc == 128) return ri ? hist_kernel<8, 128, true, T> : hist_kernel<8, 128, false, T>;
  return ri ? hist_kernel<8, 256, true, T> : hist_kernel<8, 256, false, T>;
}

HistKernel hist_kernel_ptr(int bits, int k_alloc, bool ri, int acc_bytes) {
  return acc_bytes == 8 ? hist_kernel_ptr_t<double>(bits, k_alloc, ri) : hist_kernel_ptr_t<float>(bits, k_alloc, ri);
}

// How many clusters of C CTAs (block `threads`, `smem` bytes each) can be
// resident at once on `device` (0: none). Cached.
int max_active_clusters(int bits, int k_alloc, int threads, size_t smem, int device, int acc_bytes, int C) {
  struct Key {
    int device, bits, k, threads, acc, C;
    size_t smem;
    int n;
  };
  static std::mutex m;
  static std::vector<Key> cache;
  {
    std::lock_guard<std::mutex> lk(m);
    for (const Key& c : cache)
      if (c.device == device && c.bits == bits && c.k == k_alloc && c.threads == threads && c.acc == acc_bytes &&
          c.smem == smem && c.C == C)
        return c.n;
  }
  set_smem_attr<8, 64>(device);
  set_smem_attr<4, 16>(device);
  set_smem_attr<8, 128>(device);
  set_smem_attr<8, 256>(device);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, reinterpret_cast<const void*>(hist_kernel_ptr(bits, k_alloc, false, acc_bytes)),
                                     &cfg) != cudaSuccess) {
    n = 0;
    (void)cudaGetLastError();
  }
  std::lock_guard<std::mutex> lk(m);
  cache.push_back(Key{device, bits, k_alloc, threads, acc_bytes, C, smem, n});
  return n;
}

}  // namespace

void configure_hist_kernels(int device) {
  // every shared-memory histogram variant may be launched without a prior
  // occupancy query (direct small-leaf plans): set their limits up front
  set_smem_attr<4, 16>(device);
  set_smem_attr<8, 64>(device);
  set_smem_attr<8, 128>(device);
  set_smem_attr<8, 256>(device);
  set_max_shared_carveout(reinterpret_cast<const void*>(reduce_partials_kernel<float>));
  set_max_shared_carveout(reinterpret_cast<const void*>(reduce_partials_kernel<double>));
  set_max_shared_carveout(reinterpret_cast<const void*>(pack_kernel));
  set_max_shared_carveout(reinterpret_cast<const void*>(f64_to_f32_kernel));
}

void configure_kernels(int device) {
  static std::once_flag once[64];
  std::call_once(once[device & 63], [device] {
    configure_hist_kernels(device);
    configure_leaf_kernels();
    configure_tree_kernels();
    configure_grow_kernels();
  });
}

int sm_count(int device) {
  static int cache[64] = {0};
  int& c = cache[device & 63];
  if (c == 0) HBG_CUDA(cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, device));
  return c;
}

// Leaves up to this many rows take the single-segment direct path.
constexpr int64_t kDirectRows = 1024;

HistPlan plan_histogram(int bits, int max_bin, int num_groups, int64_t n, int device, bool allow_direct,
                        int acc_bytes, bool allow_fused) {
  HistPlan p{};
  p.bits = bits;
  p.acc_bytes = acc_bytes;
  p.k_alloc = bits == 4 ? 16 : (max_bin <= 64 ? 64 : (max_bin <= 128 ? 128 : 256));
  const size_t cells = static_cast<size_t>(p.k_alloc) * 32;
  const size_t ghw = cells * 2 * static_cast<size_t>(acc_bytes);  // per-warp private {g,h}
  const size_t cntw = cells * 4;  // per-group shared counts
  const size_t smem_max = 232448;
  const int max_warps = 16;
  // The group block (slice groups per CTA) that maximises warps per CTA (the
  // latency hiding of the ordered read-modify-write chains); ties -> more
  // groups per CTA (fewer re-reads of the leaf entries).
  int gb = 0, warps = 0;
  for (int cand = 1; cand <= std::min(num_groups, max_warps); ++cand) {
    if (cand * cntw >= smem_max) break;
    const int w_per_group = static_cast<int>(std::min<size_t>(max_warps, (smem_max - cand * cntw) / ghw)) / cand;
    if (w_per_group < 1) break;
    if (cand * w_per_group >= warps) {
      gb = cand;
      warps = cand * w_per_group;
    }
  }
  require(gb >= 1 && warps >= 1, "histogram footprint exceeds shared memory");
  const int warps_full = warps;
  // Small leaves: shrink the CTA (less shared memory to clear and fold) so the
  // grid still spreads over the SMs with >= 4 tiles per warp.
  const int rpl = rows_per_lane_of(p.k_alloc, acc_bytes);
  {
    const int64_t tile_rows = static_cast<int64_t>(32) * rpl;
    const int64_t warps_needed =
        std::max<int64_t>(1, (n + 4 * tile_rows - 1) / (4 * tile_rows)) * num_groups;
    const int64_t per_cta = (warps_needed + sm_count(device) - 1) / sm_count(device);
    const int64_t want = std::max<int64_t>(gb, (per_cta + gb - 1) / gb * gb);
    if (want < warps) warps = static_cast<int>(want);
  }
  p.gb = gb;
  p.wpg = warps / gb;
  p.warps = gb * p.wpg;
  p.smem = p.warps * ghw + gb * cntw;
  p.nblocks = (num_groups + gb - 1) / gb;
  if (allow_direct && !allow_fused && n <= kDirectRows) {
    // one row segment: each CTA folds and writes the final histogram itself;
    // as many warps as there are 32-row tiles (the fold runs on all of them)
    const int max_wpg = std::max(1, warps_full / gb);
    const int64_t w = std::min<int64_t>(max_wpg, std::max<int64_t>(4 / gb + 1, (n + 31) / 32));
    p.wpg = static_cast<int>(std::max<int64_t>(1, w));
    p.warps = gb * p.wpg;
    p.smem = p.warps * ghw + gb * cntw;
    p.nseg = 1;
    p.seg_len = std::max<int64_t>(32, (n + 31) / 32 * 32);
    p.ctas = p.nblocks;
    p.part_values = 0;
    return p;
  }
  if (allow_fused) {
    const int64_t tiles = (n + 32 * rpl - 1) / (32 * rpl);
    const int max_wpg = std::max(1, warps_full / gb);
    // Up to ~2 tiles per row warp on the clusters that fit (measured: beyond
    // that the two-launch plan with PDL is as fast or faster — D6 12.6 vs
    // 16.2 us; below ~12K rows one cluster wins, D12 8.5 vs 12.9 us): clusters of C
    // CTAs, one row segment per CTA, the segments' sub-histograms summed over
    // distributed shared memory (hist_kernel's cluster mode) — no grid
    // barrier, no cooperative launch (so PDL overlaps consecutive calls).
    {
      const size_t subw = cells * (2 * static_cast<size_t>(acc_bytes) + 4);  // a CTA's sub-histogram, per group
      const size_t fixed = gb * (cntw + subw) + 16;
      const int max_wpg_c = fixed >= smem_max ? 0 : static_cast<int>(std::min<size_t>(
          max_wpg, (smem_max - fixed) / (static_cast<size_t>(gb) * ghw)));
      const int cta_cap = p.k_alloc >= 256 ? 4 : 16;
      if (max_wpg_c >= 1 && gb * max_wpg_c <= cta_cap) {
        const size_t smem_full = static_cast<size_t>(gb * max_wpg_c) * ghw + gb * (cntw + subw) + 16;
        const int warps_full_c = std::min(cta_cap, std::max(gb * max_wpg_c, 8));
        int C = 0, kmax = 0;
        for (int c : {16, 8}) {
          const int m = max_active_clusters(bits, p.k_alloc, warps_full_c * 32, smem_full, device, acc_bytes, c);
          if (m / p.nblocks >= 1) {
            C = c;
            kmax = m / p.nblocks;
            break;
          }
        }
        const int64_t slots = static_cast<int64_t>(C) * max_wpg_c;  // row warps per cluster
        static const int tpw = std::getenv("HBG_CLUSTER_TPW") ? std::atoi(std::getenv("HBG_CLUSTER_TPW")) : 2;
        if (C > 0 && tiles <= tpw * slots * kmax) {
          const int K = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kmax, (tiles + 2 * slots - 1) / (2 * slots))));
          // the fewest row warps that keep every warp at <= 2 tiles (or all of them)
          const int64_t want = (tiles + 2 * static_cast<int64_t>(K) * C - 1) / (2 * static_cast<int64_t>(K) * C);
          const int wpg_c = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_wpg_c, want)));
          const int cta_warps = std::min(cta_cap, std::max(gb * wpg_c, 8));
          int64_t seg_len = (n + static_cast<int64_t>(K) * C - 1) / (static_cast<int64_t>(K) * C);
          seg_len = std::max<int64_t>(32, (seg_len + 31) / 32 * 32);
          p.wpg = wpg_c;
          p.warps = std::max(cta_warps, gb * wpg_c);
          p.smem = static_cast<size_t>(gb * wpg_c) * ghw + gb * (cntw + subw) + 16;
          p.seg_len = seg_len;
          p.nseg = K * C;
          p.cluster = C;
          p.nclusters = K;
          p.ctas = p.nblocks * K * C;
          p.part_values = K > 1 ? static_cast<size_t>(p.nblocks) * K * gb * cells : 0;
          return p;
        }
      }
    }
  }
  const int occ = occupancy_for(bits, p.k_alloc, p.warps * 32, p.smem, device, acc_bytes);
  const int64_t slots = static_cast<int64_t>(sm_count(device)) * occ;  // CTAs per wave
  // Row segments: fill whole waves (1..4) as evenly as possible.
  int64_t nseg = 1;
  {
    double best_eff = -1.0;
    for (int64_t waves = 1; waves <= 4; ++waves) {
      const int64_t ns = std::max<int64_t>(1, slots * waves / p.nblocks);
      const double eff = static_cast<double>(p.nblocks * ns) /
                         static_cast<double>(slots * ((p.nblocks * ns + slots - 1) / slots));
      if (eff > best_eff + 0.02) {
        best_eff = eff;
        nseg = ns;
      }
    }
  }
  const int64_t min_rows = static_cast<int64_t>(p.wpg) * 32 * rpl * 2;  // >= 2 tiles per warp
  nseg = std::max<int64_t>(1, std::min<int64_t>(nseg, (n + min_rows - 1) / min_rows));
  int64_t seg_len = (n + nseg - 1) / nseg;
  seg_len = std::max<int64_t>(32, (seg_len + 31) / 32 * 32);
  p.seg_len = seg_len;
  p.nseg = static_cast<int>(std::max<int64_t>(1, (n + seg_len - 1) / seg_len));
  p.ctas = p.nblocks * p.nseg;
  p.part_values = static_cast<size_t>(p.ctas) * gb * cells;
  return p;
}

void launch_histogram(const HistPlan& plan, const HistArgs& args, cudaStream_t s) {
  const dim3 grid(plan.ctas), block(plan.warps * 32);
  const HistKernel kern = hist_kernel_ptr(plan.bits, plan.k_alloc, args.gh_indexed != 0, plan.acc_bytes);
  // Every variant is launched with programmatic stream serialization (PDL):
  // its launch and shared-memory clear overlap the previous kernel's tail
  // (the kernel waits in griddepcontrol.wait before touching global memory).
  static const bool pdl = std::getenv("HBG_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = plan.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[3];
  int na = 0;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (plan.cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = plan.cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  HBG_CUDA(cudaLaunchKernelEx(&cfg, kern, args));
}

size_t hist_exchange_doubles(int k_alloc, int max_bin, int num_groups) {
  return static_cast<size_t>(2) * std::min(k_alloc, max_bin) * num_groups * kXRow;
}

void launch_reduce_exchange(const HistPlan& plan, const HistArgs& args, int num_features, int max_bin,
                            double* d_hist, const PeerHistArgs& x, cudaStream_t s) {
  const int nbins = std::min(plan.k_alloc, max_bin);
  const int blocks = std::min(kXBlocks, nbins * args.num_groups);
  (plan.acc_bytes == 8 ? reduce_exchange_kernel<double> : reduce_exchange_kernel<float>)<<<blocks, kReduceWarps * 32, 0, s>>>(
      args, plan.nseg, plan.k_alloc, num_features, max_bin, nbins, d_hist, x);
  HBG_LAUNCH_CHECK();
}

void launch_reduce_partials(const HistPlan& plan, const HistArgs& args, int num_features,
                            int max_bin, double* d_hist, cudaStream_t s, const double* parent,
                            double* sibling) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min(plan.k_alloc, max_bin), args.num_groups);
  cfg.blockDim = dim3(kReduceWarps * 32);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // launch overlaps the histogram's tail
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = std::getenv("HBG_NO_PDL") == nullptr ? 1 : 0;
  HBG_CUDA(cudaLaunchKernelEx(&cfg, plan.acc_bytes == 8 ? reduce_partials_kernel<double> : reduce_partials_kernel<float>,
                              args, plan.nseg, plan.k_alloc, num_features, max_bin, d_hist, parent, sibling));
}

void launch_pack(const uint8_t* d_cols, int f0, int nf, int num_features, int64_t num_rows,
                 int max_bin, int bits, int64_t group_stride_words, uint32_t* d_packed, int* d_bad,
                 cudaStream_t s) {
  (void)num_features;
  if (num_rows == 0) return;
  const int words_per_slice = bits == 4 ? 4 : 8;  // 32 features per slice
  const dim3 block(256), grid(static_cast<unsigned>((num_rows + 255) / 256), words_per_slice);
  pack_kernel<<<grid, block, 0, s>>>(d_cols, f0, nf, num_rows, max_bin, bits, group_stride_words,
                                     d_packed, d_bad);
  HBG_LAUNCH_CHECK();
}

void launch_f64_to_f32(const double* in, float* out, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 4096);
  f64_to_f32_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(in, out, n);
  HBG_LAUNCH_CHECK();
}

}  // namespace hbg
