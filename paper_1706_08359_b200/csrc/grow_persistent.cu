// grow_persistent.cu — best-first tree growth (grow_tree, tree.cpp:186-261) as
// ONE persistent cooperative kernel: one CTA per SM, all splits of a tree run
// without returning to the host.
//
// The host loop (capi.cu grow_tree_impl) pays a launch sequence and a
// device->host round trip per split (~50 us/split measured) against a few us
// of device work for the typical small leaf. Here the per-split decisions are
// recomputed REDUNDANTLY by every CTA from the same data in the same order
// (so every CTA reaches bit-identical results without a leader/broadcast
// round trip); CTA 0 alone writes the persistent outputs. A typical split
// (parent <= one tile of rows) costs ONE grid barrier:
//
//   pick        the open leaf with the largest gain, lowest node id on ties
//               (the reference's pool order, strict > at tree.cpp:212-218)
//   partition   partition_leaf (tree.cpp:114-128): stable, left rows first,
//               into the other ordered buffer. Small parents: the scan CTAs
//               each rank the whole parent (registers) and write a share of
//               the output; fp64 child totals (gather_leaf_statistics,
//               tree.cpp:244-246) in a fixed order. Large parents: per-CTA
//               chunks in pipelined tiles + one barrier.
//   histogram   of the SMALLER child only (row a10). Small enough: each scan
//               CTA accumulates its feature chunk directly (int64 fixed point
//               in shared memory: deterministic); larger: the shared-memory
//               rows-in-lanes schedule of hist_kernel over (segment,
//               slice-group) items + a fixed-order fp64 reduction
//   exchange    row-sharded (nranks > 1): each scan CTA publishes its chunk of
//               this rank's smaller-child histogram + totals in peer memory and
//               sums every rank's, in rank order (see "peer exchange" below)
//   finish      per feature chunk: larger child = parent - small (every node
//               owns a slot, no aliasing), both children's split scans
//               (scan_device.cuh: the reference's fp64 operation order)
//   barrier     then every CTA reduces the per-chunk winners and picks again
//
// Cross-CTA data written inside the kernel is read through L2 (__ldcg); only
// the packed and column-major datasets use the read-only path.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "hbg_internal.h"
#include "hist_device.cuh"
#include "scan_device.cuh"

namespace hbg {

namespace {

using namespace dev;

constexpr int kItems = 8;               // parent rows per thread in the small-parent path
constexpr int kPartItems = 8;           // positions per thread per tile, large-parent partition
constexpr int kMaxRanks = 8;            // row shards exchanging through peer memory
// Data every CTA reads right after a barrier (the per-chunk winners, the node
// gains and pick stamps) is written kRep times and CTA b reads copy b % kRep:
// 148 SMs requesting the same L2 line serialise in its slice (a 2 KB
// broadcast read measured ~700 cycles vs 286 for one reader,
// microbench/latency.cu).
constexpr int kRep = 8;
constexpr int kXHeader = 16;            // doubles before the exchange blocks (done flag)
constexpr int kXBlockHeader = 16;       // doubles per block before the histogram: flag, totals
constexpr int64_t kDirectRows = 8192;   // smaller child: direct per-chunk histogram up to this size
constexpr int64_t kDirectBudget = 16384;  // ... and up to this many (row, feature) updates per scan CTA

template <int K>
__host__ __device__ constexpr int grow_threads() {
  return K >= 256 ? 256 : 512;
}

struct NodeDev {
  int64_t begin, count;  // this rank's rows [begin, begin+count) of ordered buffer `buf`
  int64_t gcount;        // rows of the node over all ranks
  double grad, hess;     // fp64 totals over all ranks (gather_leaf_statistics)
  hbg_split best;        // valid when has_best
  int32_t buf, has_best;
};

enum Path { kNoHist = 0, kDirect = 1, kSmem = 2 };

// The split being executed (every CTA holds its own copy in shared memory).
struct Desc {
  int32_t done, iter;
  int32_t parent, left_id, right_id;
  int32_t buf_in, buf_out;
  int32_t feature, thr;
  int32_t lsplit, rsplit, small_is_left, path;
  int32_t nseg, items;
  int32_t mslot;         // partition scratch slot (wave member; 0 for grow_kernel)
  int32_t pbase;         // first shared-memory histogram item of this split in part_g/h/c
  int64_t begin, count;  // parent range
  int64_t nl, nr;        // rows left / right over all ranks (the split's left_count)
  int64_t seg_len;
  int64_t nl_loc;        // this rank's rows sent left (partition)
  double tot_loc[4];     // this rank's gl, hl, gr, hr (partition)
  double tot[4];         // gl, hl, gr, hr over all ranks
};

struct GrowArgs {
  const uint8_t* packed;
  const uint8_t* colbins;  // [d][N] uint8: one byte per (feature, row)
  int64_t nrows;
  int64_t row_stride, group_stride;  // group-planar packed layout
  int words_per_row, bits, d, k, num_groups;
  int32_t* rows[2];
  float* g[2];
  float* h[2];
  double* slots;  // node id -> 3*D doubles (SoA grad|hess|count)
  NodeDev* nodes;
  double* node_gain;  // [kRep][max_nodes] gain of a node's best split, -1 without one
  int* picked;        // [kRep][max_nodes] split index + 1 at which the node was split, 0 = open
  int max_nodes;
  hbg_split* split_log;
  hbg_tree_node* tree;
  int* counts;    // [0] num_splits, [1] num_nodes, [2] error
  unsigned* bar;  // grid barrier word
  uint8_t* flags;
  int64_t* cta_left;
  int* warp_left;  // per (member, CTA, warp): left rows of the warp's run (large-parent partition)
  double* cta_sums;
  float* part_g;
  float* part_h;
  uint32_t* part_c;
  Cand* cand;  // [kRep][2][nchunks]
  const double* root_tot;  // {G, H}
  int64_t root_count;
  int num_leaves;
  int64_t min_data;
  double lambda;
  // launch geometry
  int gb, wpg, nblocks;  // histogram: slice groups per CTA item, warps per group
  int rpl;               // rows per lane of the histogram schedule
  int fchunk, nchunks;   // finish/scan: features per chunk
  int cchunk;            // features per chunk the shared-memory layout holds (>= fchunk)
  long long timeout_cycles;
  unsigned long long* prof;  // optional: [iter][kProfSlots] globaltimer stamps of CTA 0
  // row sharding (nranks > 1): per-split exchange of the smaller child's
  // histogram chunks and the partition totals through peer memory
  int nranks, rank;
  double* xown;                    // this rank's exchange area
  const double* xpeer[kMaxRanks];  // every rank's exchange area (xpeer[rank] == xown), mapped
  size_t xblock;                   // doubles per (parity, chunk) block
  unsigned long long gen;          // tree generation (tags are monotonic across trees)
  int debug;                       // HBG_GROW_DEBUG: CTA 0 prints every pick
  // wave grower (single rank; see "wave grower" below)
  Cand* wcand;            // [member][child][wcstride] chunk winners of the current wave
  size_t wcstride;        // chunks per member and child in wcand
  double* wtot;           // [wmax][4] the members' children totals (gl, hl, gr, hr), from their item CTAs
  unsigned char* wstate;  // per-CTA commit log, wstate_stride bytes each
  size_t wstate_stride;
  LeafRange* ranges;      // [max_nodes] rows of every unexpanded node -> its final leaf's value (score update)
  int wmax;               // members per wave
  int wlarge;             // speculative large members allowed (HBG_WAVE_LARGE)
  int64_t spec_rows;      // ... up to this many rows (HBG_WAVE_SPEC_ROWS)
  int wcap;               // features per wave chunk the shared-memory layout holds
  int ecap;               // speculative expansions allowed up to this total
  int64_t small_max;      // parents up to this many rows join waves (kItems * NT)
};

constexpr int kProfSlots = 20;

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// CTA 0 stamps phase boundaries of iteration `iter` when profiling is on.
__device__ __forceinline__ void stamp(const GrowArgs& a, int iter, int slot) {
  if (a.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
    a.prof[static_cast<size_t>(iter) * kProfSlots + slot] = global_ns();
}

enum GrowError { kErrNone = 0, kErrBarrierTimeout = 1, kErrPartition = 2, kErrEmptySide = 3, kErrPeerTimeout = 4 };

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ int error_of(const GrowArgs& a) {
  return *reinterpret_cast<volatile int*>(a.counts + 2);
}

__device__ __forceinline__ void set_error(const GrowArgs& a, int e) { atomicCAS(a.counts + 2, 0, e); }

// Grid barrier with one atomic per CTA: CTA 0 adds 2^31 - (G-1), the others
// 1, so the word's top bit flips exactly when the last CTA arrives (no reset,
// no second round trip). Writes before the barrier are visible after it.
__device__ __forceinline__ void grid_sync(const GrowArgs& a) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // The arrival is a release and the poll an acquire at gpu scope, both
    // cumulative over the CTA's writes ordered before them by __syncthreads:
    // no separate fences.
    const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    const unsigned old = atom_add_acq_rel(a.bar, inc);
    const long long t0 = clock64();
    while (((old ^ ld_acquire(a.bar)) & 0x80000000u) == 0) {
      if (clock64() - t0 > a.timeout_cycles) {
        set_error(a, kErrBarrierTimeout);
        break;
      }
    }
  }
  __syncthreads();
}

// ---- peer exchange (row sharding) -------------------------------------------
// Rank r's exchange area: a header (done flag) + blocks [parity][chunk], each
// = {flag, this rank's totals: gl, hl, gr, hr, rows left, rows; the chunk's
// smaller-child histogram [stat][cell] fp64}. Writer: data, fence.sys, flag =
// tag (release.sys). Reader: poll the flag (acquire.sys), read. Every rank
// sums all ranks' blocks in rank order, so every rank holds bit-identical
// global histograms and totals and takes the identical decisions. Parities
// alternate per split: a rank publishes split i only after it read every
// peer's split i-1, which every peer published only after finishing its reads
// of split i-2 (the same parity). Tags carry the tree generation, so flags
// never need resetting; a done handshake ends every tree.
__device__ __forceinline__ unsigned long long ld_acquire_sys(const double* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(double* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ const double* xblock(const GrowArgs& a, const double* base, int parity, int c) {
  return base + kXHeader + (static_cast<size_t>(parity) * a.nchunks + c) * a.xblock;
}

__device__ __forceinline__ unsigned long long xtag(const GrowArgs& a, int iter) {
  return (a.gen << 24) | static_cast<unsigned long long>(iter + 2);  // root: iter = -1
}

// Thread 0: wait until `p` carries `tag` (bounded: a dead peer is an error).
__device__ __forceinline__ bool wait_flag(const GrowArgs& a, const double* p, unsigned long long tag) {
  const long long t0 = clock64();
  unsigned long long v;
  while ((v = ld_acquire_sys(p)) != tag) {
    if (clock64() - t0 > a.timeout_cycles) {
      if (atomicCAS(a.counts + 2, 0, kErrPeerTimeout) == 0) {  // where: the awaited tag and the value seen
        a.counts[3] = static_cast<int>(tag & 0xFFFFFF);
        a.counts[4] = static_cast<int>(v & 0xFFFFFF);
        a.counts[5] = static_cast<int>(blockIdx.x);
      }
      return false;
    }
  }
  return true;
}

// Publish this rank's chunk (vals: 3 stats x `stride` doubles in shared
// memory, `cells` used) and totals tot[0..5] into block (parity, c); then
// replace vals and tot by the rank-order sums over all ranks. Whole CTA.
template <int NT>
__device__ void exchange_chunk(const GrowArgs& a, int parity, int c, unsigned long long tag, double* vals,
                               int stride, int cells, double* tot /* smem, 6 */) {
  double* mine = const_cast<double*>(xblock(a, a.xown, parity, c));
  for (int i = threadIdx.x; i < cells; i += NT) {
    mine[kXBlockHeader + i] = vals[i];
    mine[kXBlockHeader + cells + i] = vals[stride + i];
    mine[kXBlockHeader + 2 * cells + i] = vals[2 * stride + i];
  }
  if (threadIdx.x == 0)
    for (int j = 0; j < 6; ++j) mine[1 + j] = tot[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(mine, tag);
  }
  __shared__ double s_tot[6];
  for (int r = 0; r < a.nranks; ++r) {
    const double* blk = xblock(a, a.xpeer[r], parity, c);
    if (threadIdx.x == 0) wait_flag(a, blk, tag);
    __syncthreads();
    for (int i = threadIdx.x; i < cells; i += NT) {
      const double g = __ldcv(blk + kXBlockHeader + i), h = __ldcv(blk + kXBlockHeader + cells + i),
                   n = __ldcv(blk + kXBlockHeader + 2 * cells + i);
      vals[i] = r == 0 ? g : vals[i] + g;
      vals[stride + i] = r == 0 ? h : vals[stride + i] + h;
      vals[2 * stride + i] = r == 0 ? n : vals[2 * stride + i] + n;
    }
    if (threadIdx.x == 0)
      for (int j = 0; j < 6; ++j) s_tot[j] = r == 0 ? __ldcv(blk + 1 + j) : s_tot[j] + __ldcv(blk + 1 + j);
  }
  __syncthreads();
  if (threadIdx.x < 6) tot[threadIdx.x] = s_tot[threadIdx.x];
  __syncthreads();
}

// Thread 0 only: publish totals into block (parity, c) (when `publish`), then
// the rank-order sum of every rank's block totals.
__device__ void exchange_totals(const GrowArgs& a, int parity, int c, unsigned long long tag, bool publish,
                                double* tot /* 6 */) {
  if (publish) {
    double* mine = const_cast<double*>(xblock(a, a.xown, parity, c));
    for (int j = 0; j < 6; ++j) mine[1 + j] = tot[j];
    __threadfence_system();
    st_release_sys(mine, tag);
  }
  double sum[6];
  for (int r = 0; r < a.nranks; ++r) {
    const double* blk = xblock(a, a.xpeer[r], parity, c);
    wait_flag(a, blk, tag);
    for (int j = 0; j < 6; ++j) sum[j] = r == 0 ? __ldcv(blk + 1 + j) : sum[j] + __ldcv(blk + 1 + j);
  }
  for (int j = 0; j < 6; ++j) tot[j] = sum[j];
}

template <int NT>
struct PartShared {
  double sd[4][NT / 32];
  long long sc[NT / 32];
  double tot[4];
  long long cnt;
  long long scan[NT / 32];
};

// Fixed-order block sum of 4 doubles + a count: warp shuffle tree, then the
// warps in order (thread 0). Result in ps.tot / ps.cnt for every thread.
template <int NT>
__device__ void block_sum_4d1(double v[4], long long c, PartShared<NT>& ps) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] += __shfl_down_sync(0xffffffffu, v[j], off);
    c += __shfl_down_sync(0xffffffffu, c, off);
  }
  __syncthreads();  // ps reuse
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) ps.sd[j][w] = v[j];
    ps.sc[w] = c;
  }
  __syncthreads();
  if (threadIdx.x < 4) {  // one thread per statistic, warps in order
    const int j = threadIdx.x;
    double s = 0.0;
    for (int i = 0; i < NT / 32; ++i) s += ps.sd[j][i];
    ps.tot[j] = s;
  } else if (threadIdx.x == 32) {
    long long s = 0;
    for (int i = 0; i < NT / 32; ++i) s += ps.sc[i];
    ps.cnt = s;
  }
  __syncthreads();
}

// Exclusive block scan of one count per thread (thread order).
template <int NT>
__device__ long long block_excl_scan(long long x, PartShared<NT>& ps) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long inc = x;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += y;
  }
  __syncthreads();
  if (lane == 31) ps.scan[w] = inc;
  __syncthreads();
  long long base = 0;
  for (int i = 0; i < w; ++i) base += ps.scan[i];
  return base + inc - x;
}

struct SplitFeat {
  int feature, thr;
};

__device__ __forceinline__ SplitFeat split_feat(int feature, int /*bits*/, int thr) { return SplitFeat{feature, thr}; }

// Bin of (row, feature) from the resident column-major copy: one byte.
__device__ __forceinline__ uint32_t col_bin(const GrowArgs& a, int32_t row, int feature) {
  return __ldg(a.colbins + static_cast<size_t>(feature) * a.nrows + row);
}

__device__ __forceinline__ bool goes_left(const GrowArgs& a, int32_t row, const SplitFeat& sf) {
  return col_bin(a, row, sf.feature) <= static_cast<uint32_t>(sf.thr);  // tree.cpp:117-123
}

__device__ __forceinline__ bool splittable(int64_t n, int64_t min_data) { return !(n < 2 * min_data || n < 2); }

__device__ __forceinline__ double* slot_of(const GrowArgs& a, int node) {
  return a.slots + static_cast<size_t>(node) * 3 * static_cast<size_t>(a.d) * a.k;
}

__device__ __forceinline__ hbg_split load_split(const hbg_split* p) {
  hbg_split s;
  const double* src = reinterpret_cast<const double*>(p);
  double* dst = reinterpret_cast<double*>(&s);
#pragma unroll
  for (int j = 0; j < static_cast<int>(sizeof(hbg_split) / 8); ++j) dst[j] = __ldcg(src + j);
  return s;
}

// Branch-free warp argmax on a 96-bit key (hi, lo), max wins; every lane
// ends with the winning key. For a candidate split: hi = the bits of its gain
// (a positive double orders like its bit pattern; no candidate = 0), lo =
// ~((f << 12) | b) so the lowest feature, then the lowest bin wins ties —
// the reference's strict `>` scans (tree.cpp:95,172).
__device__ __forceinline__ void warp_argmax_key(unsigned long long& hi, unsigned& lo, int width = 32) {
  if (width == 32) {  // three single-instruction integer reductions (redux.sync), lexicographic
    const unsigned h1 = static_cast<unsigned>(hi >> 32), h0 = static_cast<unsigned>(hi);
    const unsigned m1 = __reduce_max_sync(0xffffffffu, h1);
    const unsigned m0 = __reduce_max_sync(0xffffffffu, h1 == m1 ? h0 : 0u);
    lo = __reduce_max_sync(0xffffffffu, h1 == m1 && h0 == m0 ? lo : 0u);
    hi = (static_cast<unsigned long long>(m1) << 32) | m0;
    return;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    if (off >= width) continue;
    const unsigned long long oh = __shfl_xor_sync(0xffffffffu, hi, off);
    const unsigned ol = __shfl_xor_sync(0xffffffffu, lo, off);
    const bool take = oh > hi || (oh == hi && ol > lo);
    hi = take ? oh : hi;
    lo = take ? ol : lo;
  }
}

__device__ __forceinline__ unsigned long long gain_key(double gain) {
  return gain > 0.0 ? static_cast<unsigned long long>(__double_as_longlong(gain)) : 0ull;
}

// ---------------------------------------------------------------------- pick

// Children of the split just executed, as every CTA computed them.
struct Kid {
  int64_t begin, count, gcount;
  double grad, hess;
  hbg_split best;
  int32_t buf, has_best;
};

// Every CTA (warp 0): choose the parent of split `i` and fill `D` (identical
// in every CTA: same data, same order). kid_l/kid_l+1: the newest nodes,
// whose state comes from the CTA's own `kid` copies (CTA 0's global writes
// of them are not yet visible). CTA 0 records the split.
// The open leaves with a split, kept by every CTA in shared memory (trees of
// up to kPickPool leaves): the pick is an argmax over them, no L2 round trip.
constexpr int kPickPool = 256;
struct PickPool {
  unsigned long long key[kPickPool];  // gain key
  short node[kPickPool];
  int n;
};

template <int NT>
__device__ void pick(const GrowArgs& a, int i, int kid_l, const Kid* kid, Desc& D, PickPool* pool) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int nnodes = 1 + 2 * i;
    const int rep = blockIdx.x % kRep;
    int err = lane == 0 ? error_of(a) : 0;
    err = __shfl_sync(0xffffffffu, err, 0);
    unsigned long long hk = 0ull;
    unsigned lk = 0u;
    if (pool != nullptr) {
      // the newest nodes join the pool (the root at i == 0); the best leaves it
      if (lane == 0) {
        if (i == 0) pool->n = 0;
        for (int c = 0; c < (i == 0 ? 1 : 2); ++c) {
          const Kid& q = kid[c];
          const unsigned long long k = q.has_best ? gain_key(q.best.gain) : 0ull;
          if (k == 0ull) continue;
          pool->key[pool->n] = k;
          pool->node[pool->n] = static_cast<short>(kid_l + c);
          ++pool->n;
        }
      }
      __syncwarp();
      const int n = pool->n;
      int idx = -1;
      if (i < a.num_leaves - 1 && err == kErrNone) {
#pragma unroll
        for (int u = 0; u < kPickPool / 32; ++u) {
          const int e = u * 32 + lane;
          const unsigned long long h = e < n ? pool->key[e] : 0ull;
          const unsigned l = e < n ? 0xFFFFFFFFu - static_cast<unsigned>(pool->node[e]) : 0u;  // lowest id on ties
          const bool take = h > hk || (h == hk && l > lk);
          hk = take ? h : hk;
          lk = take ? l : lk;
          idx = take ? e : idx;
        }
      }
      const unsigned long long h0 = hk;
      const unsigned l0 = lk;
      warp_argmax_key(hk, lk);
      const unsigned bal = __ballot_sync(0xffffffffu, hk != 0ull && h0 == hk && l0 == lk);
      const int e = bal ? __shfl_sync(0xffffffffu, idx, __ffs(bal) - 1) : -1;
      __syncwarp();  // every lane's pool reads before lane 0 rewrites it
      if (lane == 0 && e >= 0) {  // remove it: the last entry fills the hole
        pool->key[e] = pool->key[n - 1];
        pool->node[e] = pool->node[n - 1];
        pool->n = n - 1;
      }
      __syncwarp();
    } else if (i < a.num_leaves - 1 && err == kErrNone) {
      constexpr int kU = 16;  // 16 x 32 lanes >= 509 nodes: one round of loads
      for (int n0 = 0; n0 < nnodes; n0 += kU * 32) {
        double gain[kU];
        int pk[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {  // loads first, then the compares
          const int n = n0 + u * 32 + lane;
          gain[u] = n < nnodes ? __ldcg(a.node_gain + rep * a.max_nodes + n) : -1.0;
          pk[u] = n < nnodes ? __ldcg(a.picked + rep * a.max_nodes + n) : 1;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int n = n0 + u * 32 + lane;
          double g = gain[u];
          if (kid_l >= 0 && (n == kid_l || n == kid_l + 1)) {
            const Kid& q = kid[n - kid_l];
            g = q.has_best ? q.best.gain : -1.0;
          } else if (pk[u] != 0 && pk[u] != i + 1) {
            g = -1.0;  // split earlier (i+1: CTA 0 already recorded this very pick)
          }
          const unsigned long long h = n < nnodes ? gain_key(g) : 0ull;
          const unsigned l = 0xFFFFFFFFu - static_cast<unsigned>(n);  // lowest node id wins ties
          const bool take = h > hk || (h == hk && l > lk);
          hk = take ? h : hk;
          lk = take ? l : lk;
        }
      }
    }
    warp_argmax_key(hk, lk);
    const int p = hk == 0ull ? -1 : static_cast<int>(0xFFFFFFFFu - lk);
    if (lane == 0) {
      if (p < 0) {
        D.done = 1;
        if (blockIdx.x == 0) {
          a.counts[0] = i;
          a.counts[1] = nnodes;
        }
      } else {
        int64_t begin, count, gcount;
        int buf;
        hbg_split bs;
        if (kid_l >= 0 && (p == kid_l || p == kid_l + 1)) {
          const Kid& q = kid[p - kid_l];
          begin = q.begin;
          count = q.count;
          gcount = q.gcount;
          buf = q.buf;
          bs = q.best;
        } else {
          const NodeDev* P = a.nodes + rep * a.max_nodes + p;
          begin = __ldcg(&P->begin);
          count = __ldcg(&P->count);
          gcount = __ldcg(&P->gcount);
          buf = __ldcg(&P->buf);
          bs = load_split(&P->best);
        }
        const int left = 1 + 2 * i, right = 2 + 2 * i;
        if (blockIdx.x == 0) {
          for (int q = 0; q < kRep; ++q) a.picked[q * a.max_nodes + p] = i + 1;
          a.split_log[i] = bs;
          a.tree[p] = hbg_tree_node{bs.feature, bs.threshold_bin, left, right, 0.0};
        }
        const int64_t nl = bs.left_count, nr = gcount - nl;  // over all ranks
        D.done = 0;
        D.iter = i;
        D.mslot = 0;
        D.pbase = 0;
        D.parent = p;
        D.left_id = left;
        D.right_id = right;
        D.buf_in = buf;
        D.buf_out = 1 - buf;
        D.begin = begin;
        D.count = count;
        D.feature = bs.feature;
        D.thr = bs.threshold_bin;
        D.nl = nl;
        D.nr = nr;
        if (a.debug && (blockIdx.x == 0 || nl <= 0 || nr <= 0))
          printf("CTA %d ", blockIdx.x), printf("rank %d split %d: parent %d local %lld global %lld feat %d thr %d nl %lld nr %lld gain %g\n", a.rank, i,
                 p, static_cast<long long>(count), static_cast<long long>(gcount), bs.feature, bs.threshold_bin,
                 static_cast<long long>(nl), static_cast<long long>(nr), bs.gain);
        if (nl <= 0 || nr <= 0) {  // tree.cpp:124-126 (logic_error)
          set_error(a, kErrEmptySide);
          D.done = 1;
        }
        const bool scan = i + 2 < a.num_leaves;  // leaves after this split < num_leaves
        D.lsplit = scan && splittable(nl, a.min_data);
        D.rsplit = scan && splittable(nr, a.min_data);
        D.small_is_left = nl <= nr;
        const int64_t ns = nl <= nr ? nl : nr;
        // direct per-chunk accumulation costs ns * fchunk shared-memory
        // updates per scan CTA; beyond the budget the whole grid shares the
        // work through the shared-memory histogram
        const bool direct = ns <= kDirectRows && ns * a.fchunk <= kDirectBudget;
        D.path = !(D.lsplit || D.rsplit) ? kNoHist : (direct ? kDirect : kSmem);
        if (D.path == kSmem) {
          // row segments x slice-group blocks ~ one item per CTA, >= 2 tiles per warp
          const int64_t min_rows = static_cast<int64_t>(a.wpg) * 32 * 2 * a.rpl;
          int64_t nseg = gridDim.x / a.nblocks;
          if (nseg < 1) nseg = 1;
          const int64_t cap = (ns + min_rows - 1) / min_rows;
          if (nseg > cap) nseg = cap;
          int64_t seg_len = (ns + nseg - 1) / nseg;
          seg_len = (seg_len + 31) / 32 * 32;
          nseg = (ns + seg_len - 1) / seg_len;
          D.seg_len = seg_len;
          D.nseg = static_cast<int32_t>(nseg);
          D.items = static_cast<int32_t>(nseg * a.nblocks);
        }
      }
    }
  }
  __syncthreads();
}

// After the partition (all CTAs): the children's records (this rank's row
// ranges, global sizes; totals local until the exchange).
__device__ void set_children(const GrowArgs& a, const Desc& D, Kid* kid) {
  if (threadIdx.x == 0) {
    kid[0] = Kid{D.begin, D.nl_loc, D.nl, D.tot[0], D.tot[1], hbg_split{}, D.buf_out, 0};
    kid[1] = Kid{D.begin + D.nl_loc, D.count - D.nl_loc, D.nr, D.tot[2], D.tot[3], hbg_split{}, D.buf_out, 0};
    kid[0].best.feature = kid[1].best.feature = -1;
  }
  __syncthreads();
}

// CTA 0: the children's leaf values and persistent records (read by later
// picks, after at least one more barrier), from the global totals.
__device__ void store_children(const GrowArgs& a, const Desc& D, Kid* kid) {
  if (blockIdx.x != 0) return;  // uniform per CTA
  __shared__ NodeDev rec[2];
  __shared__ int ids[2];
  if (threadIdx.x == 0) {
    for (int c = 0; c < 2; ++c) {
      const int id = c == 0 ? D.left_id : D.right_id;
      Kid& q = kid[c];
      q.grad = D.tot[2 * c];
      q.hess = D.tot[2 * c + 1];
      a.tree[id] = hbg_tree_node{-1, -1, -1, -1, leaf_value(q.grad, q.hess, a.lambda)};
      rec[c] = NodeDev{q.begin, q.count, q.gcount, q.grad, q.hess, q.best, q.buf, q.has_best};
      ids[c] = id;
    }
  }
  __syncthreads();
  // every replica, written by the whole CTA (one thread would serialise
  // 2 x kRep x 128 B of stores on CTA 0's critical path)
  constexpr int W = static_cast<int>(sizeof(NodeDev) / 8);
  static_assert(sizeof(NodeDev) % 8 == 0, "NodeDev is copied in 8-byte words");
  for (int t = threadIdx.x; t < 2 * kRep * W; t += blockDim.x) {
    const int c = t / (kRep * W), r = (t / W) % kRep, w = t % W;
    reinterpret_cast<double*>(a.nodes + static_cast<size_t>(r) * a.max_nodes + ids[c])[w] =
        reinterpret_cast<const double*>(&rec[c])[w];
  }
  if (threadIdx.x < 2 * kRep) {
    const int c = threadIdx.x / kRep, r = threadIdx.x % kRep;
    a.node_gain[static_cast<size_t>(r) * a.max_nodes + ids[c]] = rec[c].has_best ? rec[c].best.gain : -1.0;
  }
}

// ------------------------------------------------------------------ partition

// Small parent (<= kItems*NT rows): EVERY CTA reads and ranks the whole parent
// (thread t holds positions [t*kItems, t*kItems+kItems) in registers), so the
// fp64 totals and the left count are known everywhere without a barrier; each
// CTA writes only its share of the output positions. Returns the rows kept in
// registers for the direct histogram.
struct RegRows {
  int32_t row[kItems];
  float g[kItems], h[kItems];
  uint32_t left;  // bit j: item j goes left
  int nvalid;
};

template <int NT>
__device__ void partition_redundant(const GrowArgs& a, Desc& D, RegRows& rr, PartShared<NT>& ps, int parts, int part,
                                    unsigned char* stage /* smem, kItems*NT*12 B */) {
  const int64_t n = D.count;
  const int32_t* rin = a.rows[D.buf_in] + D.begin;
  const float* gin = a.g[D.buf_in] + D.begin;
  const float* hin = a.h[D.buf_in] + D.begin;
  const SplitFeat sf = split_feat(D.feature, a.bits, D.thr);
  // coalesced loads into shared memory, then each thread takes its blocked
  // run of positions [t*kItems, t*kItems+kItems) (ranks by one block scan)
  int32_t* srow = reinterpret_cast<int32_t*>(stage);
  float* sg = reinterpret_cast<float*>(srow + kItems * NT);
  float* sh = sg + kItems * NT;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int q = j * NT + threadIdx.x;
    if (q < n) {
      srow[q] = __ldcg(rin + q);
      sg[q] = __ldcg(gin + q);
      sh[q] = __ldcg(hin + q);
    }
  }
  __syncthreads();
  const int64_t p0 = static_cast<int64_t>(threadIdx.x) * kItems;
  {
    int64_t nv = n - p0;
    nv = nv < 0 ? 0 : (nv > kItems ? kItems : nv);
    rr.nvalid = static_cast<int>(nv);
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int q = static_cast<int>(p0) + j;
    rr.row[j] = j < rr.nvalid ? srow[q] : 0;
    rr.g[j] = j < rr.nvalid ? sg[q] : 0.f;
    rr.h[j] = j < rr.nvalid ? sh[q] : 0.f;
  }
  bool lf[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) lf[j] = j < rr.nvalid && goes_left(a, rr.row[j], sf);
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  long long c = 0;
  rr.left = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if (j >= rr.nvalid) continue;
    if (lf[j]) {
      rr.left |= 1u << j;
      ++c;
      v[0] += rr.g[j];
      v[1] += rr.h[j];
    } else {
      v[2] += rr.g[j];
      v[3] += rr.h[j];
    }
  }
  const long long lbase = block_excl_scan<NT>(c, ps);  // left rows before this thread's positions
  block_sum_4d1<NT>(v, c, ps);
  const int64_t L = ps.cnt;
  if (threadIdx.x == 0) {
    for (int j = 0; j < 4; ++j) D.tot_loc[j] = D.tot[j] = ps.tot[j];
    D.nl_loc = L;
    if (a.nranks == 1 && L != D.nl) set_error(a, kErrPartition);
  }
  // share `part` of the output positions (`parts` CTAs write one share each)
  const int64_t share = (n + parts - 1) / parts;
  const int64_t s0 = static_cast<int64_t>(part) * share, s1 = min(n, s0 + share);
  int32_t* rout = a.rows[D.buf_out] + D.begin;
  float* gout = a.g[D.buf_out] + D.begin;
  float* hout = a.h[D.buf_out] + D.begin;
  long long lr = lbase;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if (j >= rr.nvalid) continue;
    const int64_t pos = p0 + j;
    const bool left = (rr.left >> j) & 1u;
    const int64_t dst = left ? lr : L + (pos - lr);
    if (pos >= s0 && pos < s1) {
      rout[dst] = rr.row[j];
      gout[dst] = rr.g[j];
      hout[dst] = rr.h[j];
    }
    lr += left ? 1 : 0;
  }
  __syncthreads();
}

// Large parents: CTA b owns the positions [b*chunk, (b+1)*chunk) of the
// parent, and warp w of it the contiguous run [b*chunk + w*wchunk, ...)
// (wchunk a multiple of 32). Both passes stream a warp's run 32 positions at a
// time — every load and store coalesced — with kPartItems steps in flight;
// pass 1 also records each warp's left count, so pass 2 knows where every
// warp's rows go and places them by warp ballots: no shared-memory staging,
// no block-wide scan inside the loop.
template <int NT>
__device__ __forceinline__ int64_t part_chunk(int64_t n) {
  constexpr int64_t kRun = 32 * (NT / 32);  // one 32-position step per warp
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  return (per + kRun - 1) / kRun * kRun;
}

// Pass 1 (every CTA, its chunk): side flags, fp64 side sums (each lane in its
// fixed position order, then a fixed-order block sum), the CTA's and each
// warp's left counts.
template <int NT>
__device__ void partition_count(const GrowArgs& a, const Desc& D, PartShared<NT>& ps) {
  constexpr int W = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t n = D.count, chunk = part_chunk<NT>(n), wchunk = chunk / W;
  const int64_t ws = static_cast<int64_t>(blockIdx.x) * chunk + w * wchunk;
  const int64_t we = min(n, ws + wchunk);
  const int32_t* rin = a.rows[D.buf_in] + D.begin;
  const float* gin = a.g[D.buf_in] + D.begin;
  const float* hin = a.h[D.buf_in] + D.begin;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  long long c = 0;
  // software pipeline: the next steps' (row, g, h) loads are in flight while
  // this batch's bins (dependent on its rows) are gathered and its flags written
  auto load = [&](int64_t p0, int32_t(&r)[kPartItems], float(&gv)[kPartItems], float(&hv)[kPartItems]) {
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) {
      const int64_t pos = p0 + 32 * j + lane;
      const bool ok = pos < we;
      r[j] = ok ? __ldcg(rin + pos) : 0;
      gv[j] = ok ? __ldcg(gin + pos) : 0.f;
      hv[j] = ok ? __ldcg(hin + pos) : 0.f;
    }
  };
  int32_t r[kPartItems];
  float gv[kPartItems], hv[kPartItems];
  load(ws, r, gv, hv);
  for (int64_t p0 = ws; p0 < we; p0 += 32 * kPartItems) {
    uint32_t bin[kPartItems];
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) bin[j] = p0 + 32 * j + lane < we ? col_bin(a, r[j], D.feature) : 0u;
    int32_t r2[kPartItems];
    float g2[kPartItems], h2[kPartItems];
    load(p0 + 32 * kPartItems, r2, g2, h2);
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) {
      const int64_t pos = p0 + 32 * j + lane;
      if (pos >= we) continue;
      const bool left = bin[j] <= static_cast<uint32_t>(D.thr);  // tree.cpp:117-123
      a.flags[D.begin + pos] = left ? 1 : 0;
      if (left) {
        ++c;
        v[0] += gv[j];
        v[1] += hv[j];
      } else {
        v[2] += gv[j];
        v[3] += hv[j];
      }
    }
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) {
      r[j] = r2[j];
      gv[j] = g2[j];
      hv[j] = h2[j];
    }
  }
  const int wl = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(c));
  if (lane == 0) a.warp_left[(static_cast<size_t>(D.mslot) * gridDim.x + blockIdx.x) * W + w] = wl;
  block_sum_4d1<NT>(v, c, ps);
  if (threadIdx.x == 0) {
    const size_t slot = static_cast<size_t>(D.mslot) * gridDim.x + blockIdx.x;
    a.cta_left[slot] = ps.cnt;
    for (int j = 0; j < 4; ++j) a.cta_sums[4 * slot + j] = ps.tot[j];
  }
}

// Pass 2 (every CTA, its chunk): the parent's totals and left count L, this
// CTA's and warp's left rows before them, then each warp moves its run: per
// 32-position step a ballot of the left flags gives every lane its slot —
// left rows to [lb, ...), right rows to [L + (position - lefts before), ...).
template <int NT>
__device__ void partition_scatter(const GrowArgs& a, Desc& D, PartShared<NT>& ps, unsigned char* /*smem*/) {
  constexpr int W = NT / 32;
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  long long c = 0;
  for (int b = threadIdx.x; b < G; b += NT) {  // G <= NT: one CTA record per thread
    const size_t slot = static_cast<size_t>(D.mslot) * G + b;
    c = __ldcg(a.cta_left + slot);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldcg(a.cta_sums + 4 * slot + j);
  }
  const long long before_t = block_excl_scan<NT>(c, ps);
  __shared__ long long s_before;
  if (static_cast<int>(threadIdx.x) == static_cast<int>(blockIdx.x)) s_before = before_t;
  block_sum_4d1<NT>(v, c, ps);
  const int64_t L = ps.cnt;
  if (threadIdx.x == 0) {
    for (int j = 0; j < 4; ++j) D.tot_loc[j] = D.tot[j] = ps.tot[j];
    D.nl_loc = L;
    if (a.nranks == 1 && L != D.nl) set_error(a, kErrPartition);
  }
  __syncthreads();
  const int64_t n = D.count, chunk = part_chunk<NT>(n), wchunk = chunk / W;
  const int64_t ws = static_cast<int64_t>(blockIdx.x) * chunk + w * wchunk;
  const int64_t we = min(n, ws + wchunk);
  if (ws >= we) return;
  // left rows before this warp: the CTA's prefix + the warps before it in the CTA
  const int* wl = a.warp_left + (static_cast<size_t>(D.mslot) * G + blockIdx.x) * W;
  const int mine = lane < w ? __ldcg(wl + lane) : 0;
  int64_t lb = s_before + static_cast<int64_t>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(mine)));
  const int32_t* rin = a.rows[D.buf_in] + D.begin;
  const float* gin = a.g[D.buf_in] + D.begin;
  const float* hin = a.h[D.buf_in] + D.begin;
  const uint8_t* fin = a.flags + D.begin;
  int32_t* rout = a.rows[D.buf_out] + D.begin;
  float* gout = a.g[D.buf_out] + D.begin;
  float* hout = a.h[D.buf_out] + D.begin;
  const unsigned below = (1u << lane) - 1u;
  auto load = [&](int64_t p0, int32_t(&r)[kPartItems], float(&gv)[kPartItems], float(&hv)[kPartItems],
                  uint8_t(&f)[kPartItems]) {
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) {
      const int64_t pos = p0 + 32 * j + lane;
      const bool ok = pos < we;
      r[j] = ok ? __ldcg(rin + pos) : 0;
      gv[j] = ok ? __ldcg(gin + pos) : 0.f;
      hv[j] = ok ? __ldcg(hin + pos) : 0.f;
      f[j] = ok ? __ldcg(fin + pos) : 0;
    }
  };
  int32_t r[kPartItems];
  float gv[kPartItems], hv[kPartItems];
  uint8_t f[kPartItems];
  load(ws, r, gv, hv, f);
  for (int64_t p0 = ws; p0 < we; p0 += 32 * kPartItems) {
    int32_t r2[kPartItems];
    float g2[kPartItems], h2[kPartItems];
    uint8_t f2[kPartItems];
    load(p0 + 32 * kPartItems, r2, g2, h2, f2);  // the next batch in flight while this one is placed
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) {
      const int64_t pos = p0 + 32 * j + lane;
      const bool ok = pos < we;
      const unsigned bl = __ballot_sync(0xffffffffu, ok && f[j]);
      const int lp = __popc(bl & below);
      if (ok) {
        const int64_t dst = f[j] ? lb + lp : L + (pos - lb - lp);
        rout[dst] = r[j];
        gout[dst] = gv[j];
        hout[dst] = hv[j];
      }
      lb += __popc(bl);
    }
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) {
      r[j] = r2[j];
      gv[j] = g2[j];
      hv[j] = h2[j];
      f[j] = f2[j];
    }
  }
}

// ------------------------------------------------------------------ histogram

__device__ __forceinline__ void small_child(const GrowArgs& a, const Desc& D, const int32_t*& rows,
                                            const float*& g, const float*& h, int64_t& n) {
  const int64_t off = D.small_is_left ? 0 : D.nl_loc;  // this rank's rows of the (globally) smaller child
  n = D.small_is_left ? D.nl_loc : D.count - D.nl_loc;
  rows = a.rows[D.buf_out] + D.begin + off;
  g = a.g[D.buf_out] + D.begin + off;
  h = a.h[D.buf_out] + D.begin + off;
}

// int64 fixed-point accumulation in shared memory from native 32-bit atomics:
// the low word's returned old value gives the carry into the high word.
// Integer addition commutes: the sum is exact and order-independent.
__device__ __forceinline__ void smem_add_i64(unsigned* lohi, long long q) {
  const unsigned lo = static_cast<unsigned>(q);
  const unsigned hi = static_cast<unsigned>(static_cast<unsigned long long>(q) >> 32);
  const unsigned old = atomicAdd(lohi, lo);
  const unsigned carry = old + lo < old ? 1u : 0u;
  if (hi + carry) atomicAdd(lohi + 1, hi + carry);
}

// Direct histogram of up to kItems (row, g, h) (bit u of `mask` set) into the
// chunk's fixed-point cells [f][bin]: acc holds 2 words per cell for g, then
// h, then a u32 count. sg, sh: exact powers of two, so the products equal
// ldexp(v, e). All loads of a feature are issued before its atomics.
__device__ __forceinline__ void direct_accumulate(const GrowArgs& a, unsigned* acc, int cells, int f0, int nf,
                                                  const int32_t (&row)[kItems], const float (&g)[kItems],
                                                  const float (&h)[kItems], uint32_t mask, double sg, double sh) {
  long long qg[kItems], qh[kItems];
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    qg[u] = __double2ll_rn(static_cast<double>(g[u]) * sg);
    qh[u] = __double2ll_rn(static_cast<double>(h[u]) * sh);
  }
  for (int f = 0; f < nf; ++f) {
    uint32_t b[kItems];
#pragma unroll
    for (int u = 0; u < kItems; ++u) b[u] = ((mask >> u) & 1u) ? col_bin(a, row[u], f0 + f) : 0u;
#pragma unroll
    for (int u = 0; u < kItems; ++u) {
      if (!((mask >> u) & 1u)) continue;
      const int cell = f * a.k + static_cast<int>(b[u]);
      smem_add_i64(acc + 2 * cell, qg[u]);
      smem_add_i64(acc + 2 * (cells + cell), qh[u]);
      atomicAdd(acc + 4 * cells + cell, 1u);
    }
  }
}

// ------------------------------------------------------------ finish and scan

// Smem layout of the finish phase: staging [child][stat][bin][feature] fp64
// (6 * cchunk * k doubles), then the direct accumulator (20 B per cell).
__device__ __forceinline__ unsigned* direct_acc(const GrowArgs& a, unsigned char* smem) {
  return reinterpret_cast<unsigned*>(smem + static_cast<size_t>(6) * a.cchunk * a.k * sizeof(double));
}

// Small-parent partition staging: after the finish phase's staging and the
// direct accumulator (both live while the partition runs).
__device__ __forceinline__ unsigned char* part_stage(const GrowArgs& a, unsigned char* smem) {
  const size_t off = static_cast<size_t>(a.cchunk) * a.k * (6 * sizeof(double) + 20);
  return smem + (off + 15) / 16 * 16;
}

// The direct accumulator's fixed-point scales are per CHILD: max |g|, |h|
// over the rows being accumulated (the bit patterns of non-negative floats
// order like the floats), so |q| <= 2^39 at the child's own largest value. A
// per-tree scale would quantise a leaf of values far below the tree's max
// (converged logistic hessians, residuals next to an outlier) to a few bits.
// Every chunk CTA of a child reduces the same rows, so all agree; the finish
// reads the maxima back.
__device__ __forceinline__ unsigned* direct_max() {
  __shared__ unsigned m[2];
  return m;
}

__device__ __forceinline__ void zero_direct(const GrowArgs& a, unsigned char* smem, int cells, int NT) {
  unsigned* acc = direct_acc(a, smem);
  for (int i = threadIdx.x; i < 5 * cells; i += NT) acc[i] = 0u;
  if (threadIdx.x == 0) direct_max()[0] = direct_max()[1] = 0u;
}

__device__ __forceinline__ unsigned abs_bits(float v) { return __float_as_uint(fabsf(v)); }

// Whole block: fold this thread's maxima in; after the barrier every thread
// holds the child's scales q = v * eg (resp. eh), exact powers of two.
__device__ __forceinline__ void direct_scales(unsigned mg, unsigned mh, double& eg, double& eh) {
  unsigned* m = direct_max();
  mg = __reduce_max_sync(0xffffffffu, mg);
  mh = __reduce_max_sync(0xffffffffu, mh);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(m, mg);
    atomicMax(m + 1, mh);
  }
  __syncthreads();
  int e0 = 0, e1 = 0;
  frexpf(__uint_as_float(m[0]), &e0);
  frexpf(__uint_as_float(m[1]), &e1);
  eg = ldexp(1.0, 39 - e0);
  eh = ldexp(1.0, 39 - e1);
}

// Scales of the rows of `mask` held in registers.
__device__ __forceinline__ void direct_scales_regs(const float (&g)[kItems], const float (&h)[kItems], uint32_t mask,
                                                   double& eg, double& eh) {
  unsigned mg = 0u, mh = 0u;
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    if ((mask >> u) & 1u) {
      mg = max(mg, abs_bits(g[u]));
      mh = max(mh, abs_bits(h[u]));
    }
  }
  direct_scales(mg, mh, eg, eh);
}

// Scales of n leaf-aligned rows in global memory (the smaller child of a
// large parent, <= kDirectRows rows).
template <int NT>
__device__ __forceinline__ void direct_scales_range(const float* g, const float* h, int64_t n, double& eg, double& eh) {
  unsigned mg = 0u, mh = 0u;
  for (int64_t q = threadIdx.x; q < n; q += NT) {
    mg = max(mg, abs_bits(__ldcg(g + q)));
    mh = max(mh, abs_bits(__ldcg(h + q)));
  }
  direct_scales(mg, mh, eg, eh);
}

// Where a chunk's per-child winners go: p[r * rep_stride + child * child_stride]
// for the `reps` replicas.
struct CandOut {
  Cand* p;
  int reps;
  size_t rep_stride, child_stride;
};

__device__ __forceinline__ CandOut legacy_out(const GrowArgs& a, int c) {
  return CandOut{a.cand + c, kRep, static_cast<size_t>(2) * a.nchunks, static_cast<size_t>(a.nchunks)};
}

// Both children's scans of one staged feature chunk at once: threads
// [0, NT/2) child 0 (staging st[0..3*stride)), the rest child 1; per-child
// chunk winner -> out. Whole CTA.
template <int NT>
__device__ void scan_chunk(const GrowArgs& a, double* st, int chunk_cells, int nf, int f0, const CandOut& out,
                           bool want0, bool want1, const double* tot, int64_t n0, int64_t n1) {
  const int k = a.k;
  constexpr int half = NT / 2, W = NT / 32;
  const int child = static_cast<int>(threadIdx.x) < half ? 0 : 1;
  const int tid = static_cast<int>(threadIdx.x) - child * half;
  const bool want = child == 0 ? want0 : want1;
  double* base = st + child * 3 * chunk_cells;
  const double gt = tot[2 * child], ht = tot[2 * child + 1];
  const int64_t count = child == 0 ? n0 : n1;
  const Cand best = scan_staged_t(base, base + chunk_cells, base + 2 * chunk_cells, want ? nf : 0, k, f0, gt, ht,
                                  static_cast<double>(count), static_cast<double>(a.min_data), a.lambda, tid, half);
  // argmax on (gain bits, ~(f,b)) keys, then the winner's left sums from
  // the staged prefix sums
  unsigned long long hk = best.f >= 0 ? gain_key(best.gain) : 0ull;
  unsigned lk = best.f >= 0 ? 0xFFFFFFFFu - ((static_cast<unsigned>(best.f) << 12) | static_cast<unsigned>(best.b)) : 0u;
  warp_argmax_key(hk, lk);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ unsigned long long s_hk[W];
  __shared__ unsigned s_lk[W];
  if (lane == 0) {
    s_hk[w] = hk;
    s_lk[w] = lk;
  }
  __syncthreads();
  if (w == 0 || w == W / 2) {
    hk = lane < W / 2 ? s_hk[w + lane] : 0ull;
    lk = lane < W / 2 ? s_lk[w + lane] : 0u;
    warp_argmax_key(hk, lk);
    if (lane == 0 && want) {
      Cand c{0.0, -1, -1, 0.0, 0.0, 0};
      if (hk != 0ull) {
        const unsigned fb = 0xFFFFFFFFu - lk;
        const int f = static_cast<int>(fb >> 12), b = static_cast<int>(fb & 0xFFFu);
        const int t = b * nf + (f - f0);
        c = Cand{__longlong_as_double(static_cast<long long>(hk)), f, b, base[t], base[chunk_cells + t],
                 static_cast<int64_t>(base[2 * chunk_cells + t])};
      }
      for (int r = 0; r < out.reps; ++r) out.p[r * out.rep_stride + child * out.child_stride] = c;
    }
  }
  __syncthreads();
}

// Row sharding, a split without a histogram: the scan CTAs still exchange
// (totals only), so every chunk's blocks advance in lockstep every split.
template <int NT>
__device__ void exchange_totals_chunk(const GrowArgs& a, Desc& D, int c) {
  __shared__ double s_tot[6];
  if (threadIdx.x == 0) {
    for (int j = 0; j < 4; ++j) s_tot[j] = D.tot_loc[j];
    s_tot[4] = static_cast<double>(D.nl_loc);
    s_tot[5] = 0.0;
  }
  __syncthreads();
  exchange_chunk<NT>(a, D.iter & 1, c, xtag(a, D.iter), nullptr, 0, 0, s_tot);
  if (threadIdx.x == 0) {
    for (int j = 0; j < 4; ++j) D.tot[j] = s_tot[j];
    if (static_cast<int64_t>(s_tot[4]) != D.nl) set_error(a, kErrPartition);
  }
  __syncthreads();
}

// Per feature chunk c: the smaller child's fp64 histogram (from the direct
// accumulator, or the fixed-order fp64 sum of the item partials), the larger
// child = parent - small, both written to their node slots and staged for
// the two scans; per-chunk winners -> a.cand.
template <int K, int NT>
__device__ __forceinline__ void finish_range(const GrowArgs& a, const Desc& D, int f0, int nf, int c, unsigned char* smem,
                             const CandOut& out) {
  constexpr int kCells = K * 32;
  const int d = a.d, k = a.k;
  const size_t Dc = static_cast<size_t>(d) * k;
  const int small_id = D.small_is_left ? D.left_id : D.right_id;
  const int large_id = D.small_is_left ? D.right_id : D.left_id;
  const double* par = slot_of(a, D.parent);
  double* so = slot_of(a, small_id);
  double* lo = slot_of(a, large_id);
  double* st = reinterpret_cast<double*>(smem);
  const int chunk_cells = a.cchunk * k;
  double* sm = st + (D.small_is_left ? 0 : 3 * chunk_cells);
  double* lg = st + (D.small_is_left ? 3 * chunk_cells : 0);
  const int cells = nf * k;
  if (D.path == kDirect) {
    int e0 = 0, e1 = 0;  // the child's scales (direct_scales)
    frexpf(__uint_as_float(direct_max()[0]), &e0);
    frexpf(__uint_as_float(direct_max()[1]), &e1);
    const double sg = ldexp(1.0, e0 - 39), sh = ldexp(1.0, e1 - 39);
    const unsigned* acc = direct_acc(a, smem);
    for (int i = threadIdx.x; i < cells; i += NT) {  // i = f * k + b
      const auto rd = [&](int w) {
        return static_cast<long long>((static_cast<unsigned long long>(acc[2 * w + 1]) << 32) | acc[2 * w]);
      };
      const int f = i / k, b = i - f * k;
      const int t = b * nf + f;
      sm[t] = static_cast<double>(rd(i)) * sg;
      sm[chunk_cells + t] = static_cast<double>(rd(cells + i)) * sh;
      sm[2 * chunk_cells + t] = static_cast<double>(acc[4 * cells + i]);
    }
  } else {
    // Thread t takes cell i = t mod cells (i = f * k + b: lanes are consecutive
    // bins, one line per warp-load of the feature-major partials) and segment
    // stream t / cells; the streams (NT / cells of them when the CTA has more
    // threads than cells) are combined in order through shared memory: a
    // fixed shape, so the sums are deterministic.
    const int streams = cells >= NT ? 1 : NT / cells;
    double* red = reinterpret_cast<double*>(part_stage(a, smem));  // streams x cells x 3
    for (int i0 = 0; i0 < cells; i0 += NT) {
      const int t = static_cast<int>(threadIdx.x);
      const int i = i0 + (streams > 1 ? t % cells : t), j = streams > 1 ? t / cells : 0;
      double vg = 0.0, vh = 0.0;
      unsigned long long vc = 0;
      const bool mine = i < cells && j < streams;
      if (mine) {
        const int f = f0 + i / k, b = i % k;
        const int gr = f >> 5, bi = gr / a.gb, gl = gr - bi * a.gb;
        const int cl = (f & 31) * K + b;
#pragma unroll 4
        for (int s = j; s < D.nseg; s += streams) {
          const size_t o = ((static_cast<size_t>(D.pbase) + static_cast<size_t>(s) * a.nblocks + bi) * a.gb + gl) * kCells + cl;
          vg += static_cast<double>(__ldcg(a.part_g + o));
          vh += static_cast<double>(__ldcg(a.part_h + o));
          vc += __ldcg(a.part_c + o);
        }
      }
      if (streams > 1) {
        if (mine) {
          double* r = red + (static_cast<size_t>(j) * cells + i) * 3;
          r[0] = vg;
          r[1] = vh;
          r[2] = static_cast<double>(vc);
        }
        __syncthreads();
        if (mine && j == 0) {
          for (int q = 1; q < streams; ++q) {
            const double* r = red + (static_cast<size_t>(q) * cells + i) * 3;
            vg += r[0];
            vh += r[1];
            vc += static_cast<unsigned long long>(r[2]);
          }
        }
      }
      if (mine && j == 0) {
        const int f = i / k, b = i - f * k;
        const int tt = b * nf + f;
        sm[tt] = vg;
        sm[chunk_cells + tt] = vh;
        sm[2 * chunk_cells + tt] = static_cast<double>(vc);
      }
      if (streams > 1) __syncthreads();
    }
  }
  __syncthreads();
  if (a.nranks > 1) {  // this rank's chunk + totals -> every rank's, summed in rank order
    __shared__ double s_tot[6];
    if (threadIdx.x == 0) {
      for (int j = 0; j < 4; ++j) s_tot[j] = D.tot_loc[j];
      s_tot[4] = static_cast<double>(D.nl_loc);
      s_tot[5] = 0.0;
    }
    __syncthreads();
    exchange_chunk<NT>(a, D.iter & 1, c, xtag(a, D.iter), sm, chunk_cells, cells, s_tot);
    if (threadIdx.x == 0) {
      for (int j = 0; j < 4; ++j) const_cast<Desc&>(D).tot[j] = s_tot[j];
      if (static_cast<int64_t>(s_tot[4]) != D.nl) set_error(a, kErrPartition);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < cells; i += NT) {
    const size_t o = static_cast<size_t>(f0) * k + i;
    const int f = i / k, b = i - f * k;
    const int t = b * nf + f;
    const double pg = __ldcg(par + o), ph = __ldcg(par + Dc + o), pc = __ldcg(par + 2 * Dc + o);
    const double vg = sm[t], vh = sm[chunk_cells + t], vc = sm[2 * chunk_cells + t];
    so[o] = vg;
    so[Dc + o] = vh;
    so[2 * Dc + o] = vc;
    const double xg = pg - vg, xh = ph - vh, xc = pc - vc;
    lo[o] = xg;
    lo[Dc + o] = xh;
    lo[2 * Dc + o] = xc;
    lg[t] = xg;
    lg[chunk_cells + t] = xh;
    lg[2 * chunk_cells + t] = xc;
  }
  __syncthreads();
  scan_chunk<NT>(a, st, chunk_cells, nf, f0, out, D.lsplit, D.rsplit, D.tot, D.nl, D.nr);
}

// Feature chunk c of the one-split-at-a-time grower (winners -> a.cand).
// (force-inlined: a call would put the kernel's GrowArgs in local memory —
// measured on the 4-bit instantiation, where the inliner declined: 576 B stack
// frame, every `a.` access a local load, the whole tree 13% slower)
template <int K, int NT>
__device__ __forceinline__ void finish_chunk(const GrowArgs& a, const Desc& D, int c, unsigned char* smem,
                                             Cand* /*wb*/) {
  const int f0 = c * a.fchunk;
  finish_range<K, NT>(a, D, f0, min(a.fchunk, a.d - f0), c, smem, legacy_out(a, c));
}

// Every CTA (warp 0): per-child winner over the chunks (bit-identical in every
// CTA); lanes 0-15 child 0, lanes 16-31 child 1.
template <int NT>
__device__ void winners(const GrowArgs& a, const Desc& D, Kid* kid) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x, child = lane >> 4, sub = lane & 15;
    const bool want = child == 0 ? D.lsplit : D.rsplit;
    Cand c{0.0, -1, -1, 0.0, 0.0, 0};
    unsigned long long hk = 0ull;
    unsigned lk = 0u;
    if (want) {
      for (int i0 = 0; i0 < a.nchunks; i0 += 4 * 16) {
        Cand o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // loads first
          const int i = i0 + u * 16 + sub;
          const Cand* q = a.cand + ((blockIdx.x % kRep) * 2 + child) * a.nchunks + (i < a.nchunks ? i : 0);
          o[u].gain = i < a.nchunks ? __ldcg(&q->gain) : 0.0;
          o[u].f = __ldcg(&q->f);
          o[u].b = __ldcg(&q->b);
          o[u].lg = __ldcg(&q->lg);
          o[u].lh = __ldcg(&q->lh);
          o[u].lc = __ldcg(&q->lc);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned long long h = o[u].f >= 0 ? gain_key(o[u].gain) : 0ull;
          const unsigned l = 0xFFFFFFFFu - ((static_cast<unsigned>(o[u].f) << 12) | static_cast<unsigned>(o[u].b));
          const bool take = h > hk || (h == hk && l > lk);
          hk = take ? h : hk;
          lk = take ? l : lk;
          if (take) c = o[u];
        }
      }
    }
    warp_argmax_key(hk, lk, 16);  // within each half-warp (xor offsets < 16)
    {
      // the lane holding the winner hands over its left sums
      const unsigned mine = (hk != 0ull && c.f >= 0 && gain_key(c.gain) == hk &&
                             0xFFFFFFFFu - ((static_cast<unsigned>(c.f) << 12) | static_cast<unsigned>(c.b)) == lk)
                                ? 1u : 0u;
      const unsigned bal = __ballot_sync(0xffffffffu, mine) & (child == 0 ? 0x0000FFFFu : 0xFFFF0000u);
      const int src = bal ? __ffs(bal) - 1 : lane;
      const Cand w = shfl_cand(c, src);
      c = hk == 0ull ? Cand{0.0, -1, -1, 0.0, 0.0, 0} : w;
    }
    if (sub == 0 && want) {
      const double gt = D.tot[2 * child], ht = D.tot[2 * child + 1];
      const int64_t count = child == 0 ? D.nl : D.nr;
      write_split(c, gt, ht, count, a.lambda, &kid[child].best);
      kid[child].has_best = c.f >= 0 ? 1 : 0;
    }
  }
  __syncthreads();
}

struct TileIn {
  int32_t row;
  float g, h;
};

// The rows-in-lanes, feature-rotated accumulation of hist_kernel
// (hist_kernels.cu) over positions [s0, s1) of one slice group, for one warp
// of `wpg` row-interleaved warps. idx/g/h were written by this kernel's
// partition, so they are read through L2.
template <int BITS, int K>
__device__ __forceinline__ void accumulate_rows(const GrowArgs& a, const int32_t* idx, const float* gp,
                                                const float* hp, int64_t s0, int64_t s1, int sub,
                                                const unsigned char* base, uint32_t gh_base, uint32_t* cnt_g) {
  constexpr int R = rows_per_lane<K>();
  const int lane = threadIdx.x & 31;
  const int64_t step = static_cast<int64_t>(a.wpg) * 32 * R;
  auto fetch_entry = [&](int64_t t, TileIn(&in)[R]) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t pos = t + 32 * r + lane;
      if (pos < s1) {
        in[r].row = __ldcg(idx + pos);
        in[r].g = __ldcg(gp + pos);
        in[r].h = __ldcg(hp + pos);
      } else {
        in[r].row = -1;
        in[r].g = 0.f;
        in[r].h = 0.f;
      }
    }
  };
  auto fetch_slice = [&](TileIn(&in)[R], Slice<BITS>(&sl)[R]) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (in[r].row >= 0) {
        load_slice<BITS>(base + static_cast<int64_t>(in[r].row) * a.row_stride, sl[r]);
      } else {
#pragma unroll
        for (int j = 0; j < Slice<BITS>::kWords; ++j) sl[r].w[j] = 0;
      }
    }
  };
  int64_t t = s0 + static_cast<int64_t>(sub) * 32 * R;
  TileIn e0[R], e1[R];
  Slice<BITS> cur[R];
  fetch_entry(t, e0);
  fetch_entry(t + step, e1);
  fetch_slice(e0, cur);
  for (; t < s1; t += step) {
    TileIn e2[R];
    Slice<BITS> nxt[R];
    fetch_entry(t + 2 * step, e2);
    fetch_slice(e1, nxt);
#pragma unroll
    for (int r = 0; r < R; ++r) rotate_slice<BITS>(cur[r], lane);
    if (t + 32 * R <= s1) {
      float g[R], h[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        g[r] = e0[r].g;
        h[r] = e0[r].h;
      }
#pragma unroll
      for (int p = 0; p < 32; ++p) update_step_rows<BITS, K, R>(cur, p, lane, gh_base, cnt_g, g, h);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool valid = e0[r].row >= 0;
#pragma unroll
        for (int p = 0; p < 32; ++p)
          update_step<BITS, K, true>(cur[r], p, lane, gh_base, cnt_g, e0[r].g, e0[r].h, valid);
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

// Shared-memory histogram of the smaller child: items = (row segment, slice
// group block); each item -> one fp32/u32 partial per group of the block
// (part_g/h/c item D.pbase + item).
template <int BITS, int K, int NT>
__device__ void hist_smem_item(const GrowArgs& a, const Desc& D, int item, unsigned char* smem) {
  constexpr int kCells = K * 32;
  const int32_t* rows;
  const float* g;
  const float* h;
  int64_t n;
  small_child(a, D, rows, g, h, n);
  const int warps = a.gb * a.wpg;
  float2* gh = reinterpret_cast<float2*>(smem);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + static_cast<size_t>(warps) * kCells * 8);
  const int w = threadIdx.x >> 5;
  const int bi = item % a.nblocks, seg = item / a.nblocks;
  {
    const int n16 = (warps * kCells * 8 + a.gb * kCells * 4) / 16;
    uint4* z = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < n16; i += NT) z[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  if (w < warps) {
    const int gl = w % a.gb, sub = w / a.gb;
    const int group = bi * a.gb + gl;
    if (group < a.num_groups) {
      const int64_t s0 = static_cast<int64_t>(seg) * D.seg_len;
      const int64_t s1 = min(s0 + D.seg_len, n);
      const uint32_t gh_base = smem_addr(gh + static_cast<size_t>(w) * kCells);
      const unsigned char* base = a.packed + static_cast<int64_t>(group) * a.group_stride;
      accumulate_rows<BITS, K>(a, rows, g, h, s0, s1, sub, base, gh_base, cnt + static_cast<size_t>(gl) * kCells);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < a.gb * kCells; i += NT) {
    const int g2 = i / kCells, c = i - g2 * kCells;
    float sg = 0.f, sh = 0.f;
    for (int s = 0; s < a.wpg; ++s) {  // warps of the group in a fixed order
      const float2 v = gh[static_cast<size_t>(s * a.gb + g2) * kCells + c];
      sg += v.x;
      sh += v.y;
    }
    // feature-major partial ([feature][bin]): the finish's warp-loads of
    // consecutive bins are one line each
    const size_t o = ((static_cast<size_t>(D.pbase) + item) * a.gb + g2) * kCells + (c & 31) * K + (c >> 5);
    a.part_g[o] = sg;
    a.part_h[o] = sh;
    a.part_c[o] = cnt[static_cast<size_t>(g2) * kCells + c];
  }
  __syncthreads();
}

template <int BITS, int K, int NT>
__device__ void hist_smem(const GrowArgs& a, const Desc& D, unsigned char* smem) {
  for (int item = blockIdx.x; item < D.items; item += gridDim.x) hist_smem_item<BITS, K, NT>(a, D, item, smem);
}

template <int BITS, int K>
__global__ void __launch_bounds__(grow_threads<K>(), 1) grow_kernel(GrowArgs a) {
  constexpr int NT = grow_threads<K>();
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Cand wb[NT / 32];
  __shared__ PartShared<NT> ps;
  __shared__ Desc D;
  __shared__ Kid kid[2];
  // the pick's shared-memory pool (not at 256 bins: its 3 KB would cost the
  // histogram one of its three 64 KB warps)
  __shared__ __align__(8) unsigned char pool_raw[K >= 256 ? 8 : sizeof(PickPool)];
  PickPool* pool = nullptr;
  if constexpr (K < 256) pool = a.num_leaves <= kPickPool ? reinterpret_cast<PickPool*>(pool_raw) : nullptr;
  if (a.nranks == 1) {
    // root: histogram, totals and best split were computed by the
    // host-launched kernels; every CTA builds the root record
    if (threadIdx.x == 0) {
      const double G = __ldcg(a.root_tot), H = __ldcg(a.root_tot + 1);
      kid[0] = Kid{0, a.root_count, a.root_count, G, H, load_split(&a.nodes[0].best), 0, 0};
      kid[0].has_best = kid[0].best.feature >= 0 ? 1 : 0;
    }
  } else {
    // row-sharded root: this rank's histogram (slot 0) and totals -> the
    // rank-order sums over all ranks; the scan CTAs scan their chunk of the
    // global root histogram
    const bool chunk_cta = static_cast<int>(blockIdx.x) < a.nchunks;
    __shared__ double rt[6];
    if (threadIdx.x == 0) {
      rt[0] = __ldcg(a.root_tot);
      rt[1] = __ldcg(a.root_tot + 1);
      rt[2] = rt[3] = rt[4] = 0.0;
      rt[5] = static_cast<double>(a.root_count);
      if (!chunk_cta) exchange_totals(a, 1, 0, xtag(a, -1), false, rt);
    }
    __syncthreads();
    if (chunk_cta) {
      const int d = a.d, k = a.k, c = blockIdx.x;
      const size_t Dc = static_cast<size_t>(d) * k;
      const int f0 = c * a.fchunk, nf = min(a.fchunk, d - f0), cells = nf * k, cc = a.fchunk * k;
      double* st = reinterpret_cast<double*>(smem);
      double* root = a.slots;  // node 0's slot
      for (int i = threadIdx.x; i < cells; i += NT) {
        const size_t o = static_cast<size_t>(f0) * k + i;
        const int f = i / k, b = i - f * k, t = b * nf + f;
        st[t] = __ldcg(root + o);
        st[cc + t] = __ldcg(root + Dc + o);
        st[2 * cc + t] = __ldcg(root + 2 * Dc + o);
      }
      __syncthreads();
      exchange_chunk<NT>(a, 1, c, xtag(a, -1), st, cc, cells, rt);
      for (int i = threadIdx.x; i < cells; i += NT) {  // the global root histogram in slot 0
        const size_t o = static_cast<size_t>(f0) * k + i;
        const int f = i / k, b = i - f * k, t = b * nf + f;
        root[o] = st[t];
        root[Dc + o] = st[cc + t];
        root[2 * Dc + o] = st[2 * cc + t];
      }
      __syncthreads();
      const int64_t N = static_cast<int64_t>(rt[5]);
      const bool ok = a.num_leaves >= 2 && splittable(N, a.min_data);  // tree.cpp:165
      scan_chunk<NT>(a, st, cc, nf, f0, legacy_out(a, c), ok, false, rt, N, 0);
    }
    grid_sync(a);
    if (threadIdx.x == 0) {  // the root "split" descriptor for winners(): child 0 = the root
      const int64_t N = static_cast<int64_t>(rt[5]);
      D.lsplit = a.num_leaves >= 2 && splittable(N, a.min_data);
      D.rsplit = 0;
      D.tot[0] = rt[0];
      D.tot[1] = rt[1];
      D.nl = N;
      kid[0] = Kid{0, a.root_count, N, rt[0], rt[1], hbg_split{}, 0, 0};
      kid[0].best.feature = -1;
    }
    __syncthreads();
    winners<NT>(a, D, kid);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const Kid& r = kid[0];
    a.tree[0] = hbg_tree_node{-1, -1, -1, -1, leaf_value(r.grad, r.hess, a.lambda)};
    const NodeDev rec{0, r.count, r.gcount, r.grad, r.hess, r.best, 0, r.has_best};
    for (int q = 0; q < kRep; ++q) a.nodes[q * a.max_nodes] = rec;
    for (int q = 0; q < kRep; ++q) a.node_gain[q * a.max_nodes] = r.has_best ? r.best.gain : -1.0;
  }
  __syncthreads();
  pick<NT>(a, 0, 0, kid, D, pool);  // node 0 is "kid_l" (kid[1] is never consulted: nnodes = 1)
  while (!D.done) {
    const int it = D.iter;
    stamp(a, it, 0);
    // (with row sharding a rank's part of a parent can be small while the
    // globally smaller child needs the shared-memory histogram)
    const bool small_parent = D.count <= static_cast<int64_t>(kItems) * NT && D.path != kSmem;
    if (a.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {  // class and sizes of this split
      a.prof[static_cast<size_t>(it) * kProfSlots + 7] = (small_parent ? 0 : 4) + D.path;
      a.prof[static_cast<size_t>(it) * kProfSlots + 10] = static_cast<unsigned long long>(D.count);
      a.prof[static_cast<size_t>(it) * kProfSlots + 11] = static_cast<unsigned long long>(D.nl < D.nr ? D.nl : D.nr);
    }
    const bool chunk_cta = static_cast<int>(blockIdx.x) < a.nchunks;
    const int f0 = blockIdx.x * a.fchunk;
    const int nf = chunk_cta ? min(a.fchunk, a.d - f0) : 0;
    if (small_parent) {
      // the scan CTAs (one feature chunk each) rank the whole parent and share
      // the scatter; the others only wait at the barrier
      if (chunk_cta) {
        RegRows rr;
        if (D.path == kDirect) zero_direct(a, smem, nf * a.k, NT);
        partition_redundant<NT>(a, D, rr, ps, a.nchunks, blockIdx.x, part_stage(a, smem));
        set_children(a, D, kid);
        stamp(a, it, 1);
        if (D.path == kDirect) {
          // the smaller child's rows are in registers already: accumulate this
          // CTA's feature chunk, then finish and scan it
          const uint32_t valid = rr.nvalid >= 32 ? ~0u : ((1u << rr.nvalid) - 1u);
          const uint32_t want = (D.small_is_left ? rr.left : ~rr.left) & valid;
          double eg, eh;
          direct_scales_regs(rr.g, rr.h, want, eg, eh);
          direct_accumulate(a, direct_acc(a, smem), nf * a.k, f0, nf, rr.row, rr.g, rr.h, want, eg, eh);
          __syncthreads();
          stamp(a, it, 2);
          finish_chunk<K, NT>(a, D, blockIdx.x, smem, wb);
        } else if (a.nranks > 1 && D.path == kNoHist) {
          exchange_totals_chunk<NT>(a, D, blockIdx.x);
        }
        // (kSmem cannot occur: the smaller child of a small parent is <= kDirectRows)
      } else if (a.nranks > 1) {
        // this rank's left count is needed for the children's row ranges:
        // rank the parent like the scan CTAs (no share of the scatter)
        RegRows rr;
        partition_redundant<NT>(a, D, rr, ps, a.nchunks, blockIdx.x, part_stage(a, smem));
        set_children(a, D, kid);
      } else {
        if (threadIdx.x == 0) {
          D.nl_loc = D.nl;  // one rank: the split's counts are this rank's
          D.tot[0] = D.tot[1] = D.tot[2] = D.tot[3] = 0.0;  // not used here
        }
        __syncthreads();
        set_children(a, D, kid);
      }
      stamp(a, it, 3);
      grid_sync(a);
    } else {
      partition_count<NT>(a, D, ps);
      grid_sync(a);
      partition_scatter<NT>(a, D, ps, smem);
      grid_sync(a);
      set_children(a, D, kid);
      stamp(a, it, 1);
      if (D.path == kDirect) {
        if (chunk_cta) {
          zero_direct(a, smem, nf * a.k, NT);
          __syncthreads();
          const int32_t* rows;
          const float* g;
          const float* h;
          int64_t n;
          small_child(a, D, rows, g, h, n);
          double eg, eh;
          direct_scales_range<NT>(g, h, n, eg, eh);
          for (int64_t j0 = 0; j0 < n; j0 += static_cast<int64_t>(NT) * kItems) {
            int32_t r[kItems];
            float gg[kItems], hh[kItems];
            uint32_t mask = 0;
#pragma unroll
            for (int u = 0; u < kItems; ++u) {
              const int64_t j = j0 + static_cast<int64_t>(u) * NT + threadIdx.x;
              const bool ok = j < n;
              r[u] = ok ? __ldcg(rows + j) : 0;
              gg[u] = ok ? __ldcg(g + j) : 0.f;
              hh[u] = ok ? __ldcg(h + j) : 0.f;
              mask |= ok ? 1u << u : 0u;
            }
            direct_accumulate(a, direct_acc(a, smem), nf * a.k, f0, nf, r, gg, hh, mask, eg, eh);
          }
          __syncthreads();
          stamp(a, it, 2);
          finish_chunk<K, NT>(a, D, blockIdx.x, smem, wb);
        }
        stamp(a, it, 3);
        grid_sync(a);
      } else if (D.path == kNoHist) {
        if (a.nranks > 1)
          for (int c = blockIdx.x; c < a.nchunks; c += gridDim.x) exchange_totals_chunk<NT>(a, D, c);
      } else if (D.path == kSmem) {
        hist_smem<BITS, K, NT>(a, D, smem);
        stamp(a, it, 2);
        grid_sync(a);
        for (int c = blockIdx.x; c < a.nchunks; c += gridDim.x) finish_chunk<K, NT>(a, D, c, smem, wb);
        stamp(a, it, 3);
        grid_sync(a);
      }
    }
    stamp(a, it, 4);
    if (D.path != kNoHist) winners<NT>(a, D, kid);
    stamp(a, it, 8);
    store_children(a, D, kid);
    stamp(a, it, 6);
    // every warp has read this split's D (the D.path test above) before
    // warp 0 rewrites it for the next one (without a histogram there is no
    // barrier in between on CTAs other than 0; racecheck)
    __syncthreads();
    pick<NT>(a, it + 1, D.left_id, kid, D, pool);
    stamp(a, it, 5);
  }
  if (a.nranks > 1 && blockIdx.x == 0 && threadIdx.x == 0) {
    // done handshake: no rank starts the next tree (and overwrites a block)
    // before every rank has finished reading this tree's blocks
    __threadfence_system();
    st_release_sys(a.xown, a.gen);
    for (int r = 0; r < a.nranks; ++r) wait_flag(a, a.xpeer[r], a.gen);
  }
}

// ---------------------------------------------------------------- wave grower
//
// Best-first growth expands ONE leaf per step (tree.cpp:210-258), and
// grow_kernel above pays one split's latency chain (partition, histogram,
// scans, barrier, pick: ~15 us) 254 times per 255-leaf tree while most splits
// touch a few thousand rows. The wave grower (single rank) expands SEVERAL
// leaves per wave and replays the reference's pick order over the results:
//
//  * A leaf's children (rows, histograms, best splits) depend only on the
//    leaf, never on when it is split: the partitions are stable, the
//    direct-path histograms exact fixed point, the shared-memory histograms a
//    fixed-order sum over the same segments, the scans per feature. So the
//    tree is bit-identical to grow_kernel's (tested).
//  * Every CTA replays the reference loop on its own copy of the open-leaf
//    pool: while the best open leaf (max gain, lowest output id on ties: the
//    pool order, strict > at tree.cpp:212-218) is already expanded, COMMIT it
//    — its children join the pool with output ids 2i+1, 2i+2 as
//    tree.cpp:224-236 numbers them. The first best open leaf that is not
//    expanded yet is the reference's next split, for certain.
//  * The next wave expands that leaf plus up to wmax-1 speculative ones: the
//    expandable nodes of the speculative tree (children of expanded nodes,
//    committed or not) with the largest min-gain along their path
//    (best-first expands in that order up to ties). Speculation is bounded in
//    total by `ecap`; an expansion the replay never commits is not emitted,
//    and its children never enter the pool. Rows stay partitioned among the
//    unexpanded nodes of the speculative tree (an unexpanded node's range is
//    never rewritten after its creation), so the score update walks those
//    with the value of the final leaf above each (wave_emit).
//
// A wave runs its small members (parent <= small_max rows) as (member,
// feature chunk) items in one phase — each CTA ranks its member's parent in
// registers, accumulates its chunk exactly, subtracts and scans — and its
// large members through grow_kernel's paths, every CTA taking a chunk of
// every large member: two-pass partition, direct or shared-memory histogram
// of the smaller child, chunk finishes. The last CTA to finish a member's
// chunks (atomic count) reduces the chunk winners and publishes the
// children's records. Barriers per wave: 1 (small members only) to 4. The
// output (split log, tree, score-update ranges) is written once at the end
// from the replayed commit log.

constexpr int kWN = 1536;  // node ids per tree (shared-memory state): 254 speculative expansions beyond 255 leaves
static_assert(kWN <= 2048, "node ids are packed in 11 bits");

// Speculation order: prio buckets of 1/32 octave (a positive float's top 13 bits).
__device__ __forceinline__ int prio_bucket(float p) { return static_cast<int>(__float_as_uint(p) >> 18); }
constexpr int kWL = 256;   // open leaves: num_leaves <= kWL
constexpr int kWMax = 16;  // members per wave

struct WaveSmem {
  unsigned long long gkey[kWN];  // gain key of node n's best split (0: none)
  float prio[kWN];               // min gain along the path from the root
  short kid[kWN];                // left child once expanded, -1 before
  unsigned char large[kWN];      // 0: small; runs the large-parent paths: 1 (<= spec_rows rows), 2
  unsigned avail[kWN];           // expandable (discovered, gain > 0, not expanded): av_pack(), sorted descending
  unsigned long long fkey[kWL];  // the replay's open leaves with a split: gain key, node, output id
  short fnode[kWL], fout[kWL];
  short wave[kWMax];             // members: small ones first
  unsigned char later[kWL];      // commit i: bit c = child c was split later
  short cnode[kWL], ckid[kWL], cout[kWL];  // commit i: node, left child node, output id
  unsigned fresh[32];            // the last wave's new expandable entries, sorted (wave_integrate)
  NodeDev wrec[2 * kWMax];       // the last wave's children records (wave_publish), member-major
  int nav, nfr, committed, next, expanded, done, W, nsmall, nwc, wc, nwaves, hitems, ditems, err, nfresh;
};

// An expandable-list entry, ordered as the speculation ranks nodes: prio
// bucket (descending), then the lowest node id; the size class rides along.
// 13 + 11 + 2 bits.
__device__ __forceinline__ unsigned av_pack(int node, int cls, int bucket) {
  return (static_cast<unsigned>(bucket) << 13) | (static_cast<unsigned>(2047 - node) << 2) |
         static_cast<unsigned>(cls);
}
__device__ __forceinline__ int av_node(unsigned v) { return 2047 - static_cast<int>((v >> 2) & 0x7FFu); }
__device__ __forceinline__ int av_class(unsigned v) { return static_cast<int>(v & 3u); }
__device__ __forceinline__ int av_bucket(unsigned v) { return static_cast<int>(v >> 13); }

// Per-CTA state in global memory (written by the CTA's warp 0 when it forms
// a wave, read back by the same CTA at the end): the parent of each child pair.
__host__ __device__ inline size_t wave_state_bytes(int /*num_leaves*/, int max_nodes) {
  return (2 * static_cast<size_t>(max_nodes / 2 + 1) + 255) / 256 * 256;
}

__device__ __forceinline__ short* wave_ppar(const GrowArgs& a) {
  return reinterpret_cast<short*>(a.wstate + static_cast<size_t>(blockIdx.x) * a.wstate_stride);
}

// Would the split of a node with these sizes run the shared-memory histogram
// (grow_kernel's choice at pick time: kept, so the trees stay bit-identical)?
__device__ __forceinline__ bool runs_large(const GrowArgs& a, int64_t count, int64_t nl) {
  const int64_t nr = count - nl;
  if (count > a.small_max) return true;
  const bool ls = splittable(nl, a.min_data), rs = splittable(nr, a.min_data);
  const int64_t ns = nl <= nr ? nl : nr;
  return (ls || rs) && !(ns <= kDirectRows && ns * a.fchunk <= kDirectBudget);
}

// Warp 0 after a wave's barrier: the members' children (records built by
// wave_publish) join the speculative tree.
__device__ void wave_integrate(const GrowArgs& a, WaveSmem& w) {
  const int lane = threadIdx.x;
  const int W = w.W;
  bool add = false;
  int id = 0;
  if (lane < 2 * W) {
    const int x = w.wave[lane >> 1];
    id = w.kid[x] + (lane & 1);
    const NodeDev& P = w.wrec[lane];  // wave_publish: member lane >> 1, child lane & 1
    const double g = P.has_best ? P.best.gain : -1.0;
    const int64_t n = P.count;
    const int64_t nl = P.best.left_count;
    const unsigned long long key = gain_key(g);
    w.gkey[id] = key;
    w.kid[id] = -1;
    const int cls = runs_large(a, n, nl) ? (n <= a.spec_rows ? 1 : 2) : 0;
    const float pr = fminf(w.prio[x], static_cast<float>(g));
    w.large[id] = static_cast<unsigned char>(cls);
    w.prio[id] = pr;
    add = key != 0ull;
    id = static_cast<int>(av_pack(id, cls, prio_bucket(pr)));
  }
  const int err = lane == 31 ? error_of(a) : 0;  // (one L2 round trip with the loads above)
  // the new entries, sorted descending across the lanes (bitonic), merged into
  // the sorted list from its end (every entry moves right by the number of new
  // entries above it; a round's reads precede its writes, which land at or
  // above the rows still to be read)
  unsigned key = add ? static_cast<unsigned>(id) : 0u;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const unsigned o = __shfl_xor_sync(0xffffffffu, key, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      key = (lower == up ? o > key : o < key) ? o : key;
    }
  }
  w.fresh[lane] = key;
  if (lane == 0) w.nfresh = __popc(__ballot_sync(0xffffffffu, add));
  else __ballot_sync(0xffffffffu, add);
  if (lane == 31) w.err = err;
  __syncwarp();
}

// Warp 1, while warp 0 replays: merge the sorted new entries (w.fresh) into
// the sorted expandable list from its end — every entry moves right by the
// number of new entries above it; a round's reads precede its writes, which
// land at or above the rows still to be read; entries above the largest new
// one stay put (the loop stops there).
__device__ void wave_merge(WaveSmem& w) {
  const int lane = threadIdx.x & 31;
  const int m = w.nfresh, n = w.nav;
  if (m == 0) return;
  const unsigned key = w.fresh[lane];
  int above = 0;  // new entry `lane`'s position: lane + the old entries above it
  if (lane < m) {
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (w.avail[mid] > key) lo = mid + 1; else hi = mid;
    }
    above = lo;
  }
  const unsigned top = w.fresh[0];
  for (int i0 = n - 1; i0 >= 0; i0 -= 32) {
    const int i = i0 - lane;
    const unsigned v = i >= 0 ? w.avail[i] : 0xFFFFFFFFu;
    int s_new = 0;  // new entries above v
    if (v < top) {
      int lo = 0, hi = m;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (w.fresh[mid] > v) lo = mid + 1; else hi = mid;
      }
      s_new = lo;
    }
    __syncwarp();
    if (i >= 0 && s_new > 0) w.avail[i + s_new] = v;
    if (!__any_sync(0xffffffffu, s_new > 0)) break;  // every earlier entry ranks above all new ones
  }
  __syncwarp();
  if (lane < m) w.avail[lane + above] = key;
  if (lane == 0) w.nav = n + m;
  __syncwarp();
}

// Every CTA (identical everywhere): warp 0 replays the reference's picks over
// the expanded leaves (commit) while warp 1 merges the last wave's new
// expandable entries (wave_merge); then warp 0 forms the next wave: the certain pick plus
// the first entries of the sorted expandable list — small nodes, and large
// ones of <= spec_rows rows ranked within the R best (R = the commits still to
// come) when HBG_WAVE_LARGE allows: a speculative large expansion costs a
// partition and histogram pass over its rows. Whole CTA.
template <int NT>
__device__ void wave_select(const GrowArgs& a, WaveSmem& w) {
  __shared__ int s_best, s_committed, s_nfr;
  const int L1 = a.num_leaves - 1;
  __syncthreads();  // warp 0's integrate is complete for warp 1's merge
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int nfr = w.nfr, committed = w.committed;
    const int err = w.err;  // read with the integrate loads
    int best = -1;
    const long long rc0 = clock64();
    while (err == kErrNone && committed < L1) {
      unsigned long long hk = 0ull;
      unsigned lk = 0u;
      int idx = -1;
#pragma unroll
      for (int u = 0; u < kWL / 32; ++u) {
        const int i = u * 32 + lane;
        const unsigned long long h = i < nfr ? w.fkey[i] : 0ull;
        const unsigned l = i < nfr ? 0xFFFFFFFFu - static_cast<unsigned>(w.fout[i]) : 0u;
        const bool take = h > hk || (h == hk && l > lk);
        hk = take ? h : hk;
        lk = take ? l : lk;
        idx = take ? i : idx;
      }
      unsigned long long H = hk;
      unsigned Lk = lk;
      warp_argmax_key(H, Lk);
      if (H == 0ull) break;
      const unsigned bal = __ballot_sync(0xffffffffu, hk == H && lk == Lk);
      const int e = __shfl_sync(0xffffffffu, idx, __ffs(bal) - 1);
      const int x = w.fnode[e];
      const int kd = w.kid[x];
      if (kd < 0) {
        best = e;
        break;
      }
      // commit: the reference splits x now (tree.cpp:220-256). Every lane's
      // reads of this pass are done before lane 0 rewrites the list (the
      // shuffles above order them only by data dependence; racecheck).
      __syncwarp();
      if (lane == 0) {
        const int o = w.fout[e];
        w.cnode[committed] = static_cast<short>(x);
        w.ckid[committed] = static_cast<short>(kd);
        w.cout[committed] = static_cast<short>(o);
        w.later[committed] = 0;
        if (o > 0) w.later[(o - 1) >> 1] |= static_cast<unsigned char>(1 << ((o - 1) & 1));
        const int t = nfr - 1;  // the last entry fills the hole
        w.fkey[e] = w.fkey[t];
        w.fnode[e] = w.fnode[t];
        w.fout[e] = w.fout[t];
        int m = t;
        for (int c = 0; c < 2; ++c) {
          if (w.gkey[kd + c] == 0ull) continue;
          w.fkey[m] = w.gkey[kd + c];
          w.fnode[m] = static_cast<short>(kd + c);
          w.fout[m] = static_cast<short>(2 * committed + 1 + c);
          ++m;
        }
      }
      __syncwarp();
      nfr += (w.gkey[kd] != 0ull ? 1 : 0) + (w.gkey[kd + 1] != 0ull ? 1 : 0) - 1;
      ++committed;
    }
    if (lane == 0) {
      s_best = best >= 0 && committed < L1 && err == kErrNone ? best : -1;
      s_committed = committed;
      s_nfr = nfr;
      if (w.nwaves > 0) {
        stamp(a, w.nwaves - 1, 8);  // (the merge ran alongside)
        if (a.prof != nullptr && blockIdx.x == 0) {
          unsigned long long* t = a.prof + static_cast<size_t>(w.nwaves - 1) * kProfSlots;
          t[12] = static_cast<unsigned long long>(committed - w.committed);
          t[11] = static_cast<unsigned long long>(clock64() - rc0);  // replay cycles (overrides slot 11)
          t[14] = static_cast<unsigned long long>(w.nav);
          t[15] = static_cast<unsigned long long>(nfr);
        }
      }
    }
  } else if (threadIdx.x < 64) {
    wave_merge(w);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    short* ppar = wave_ppar(a);
    const int best = s_best, committed = s_committed;
    int W = 0, nsmall = 0;
    if (best >= 0) {
      const int ps = w.fnode[best];
      int m = min(L1 - committed, a.wmax);
      m = max(1, min(m, a.ecap - w.expanded));
      const int nav = w.nav;
      const long long c0 = clock64();
      // large entries qualify down to the R-th entry's key
      const int r = L1 - committed - 1;
      const unsigned tr = a.wlarge > 0 && r > 0 ? (nav > r ? w.avail[r] : 0u) : 0xFFFFFFFFu;
      if (lane == 0) w.wave[0] = static_cast<short>(ps);
      W = 1;
      for (int i0 = 0; i0 < nav && W < m; i0 += 32) {
        const int i = i0 + lane;
        const unsigned v = i < nav ? w.avail[i] : 0u;
        const int cls = av_class(v);
        const bool el = i < nav && av_node(v) != ps && (cls == 0 || (cls == 1 && v >= tr));
        const unsigned bal = __ballot_sync(0xffffffffu, el);
        const int r2 = W + __popc(bal & ((1u << lane) - 1u));
        if (el && r2 < m) w.wave[r2] = static_cast<short>(av_node(v));
        W = min(m, W + __popc(bal));
      }
      __syncwarp();
      if (lane == 0 && a.prof != nullptr && blockIdx.x == 0 && w.nwaves > 0)
        a.prof[static_cast<size_t>(w.nwaves - 1) * kProfSlots + 13] = static_cast<unsigned long long>(clock64() - c0);
      if (lane == 0 && w.nwaves > 0) stamp(a, w.nwaves - 1, 9);
      // members leave the expandable list; small members first
      for (int j = lane; j < W; j += 32) w.kid[w.wave[j]] = -2;  // mark
      __syncwarp();
      int nav2 = 0;  // compaction in place: a round's reads precede its writes, which land below them
      for (int i0 = 0; i0 < nav; i0 += 32) {
        const int i = i0 + lane;
        const unsigned n = i < nav ? w.avail[i] : 0u;
        const bool keep = i < nav && w.kid[av_node(n)] != -2;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) w.avail[nav2 + __popc(bal & ((1u << lane) - 1u))] = n;
        nav2 += __popc(bal);
        __syncwarp();
      }
      short mem = lane < W ? w.wave[lane] : 0;
      const bool sm = lane < W && !w.large[mem];
      const unsigned bs = __ballot_sync(0xffffffffu, sm), bl = __ballot_sync(0xffffffffu, lane < W && !sm);
      nsmall = __popc(bs);
      const int pos = sm ? __popc(bs & ((1u << lane) - 1u)) : nsmall + __popc(bl & ((1u << lane) - 1u));
      __syncwarp();
      if (lane < W) {
        w.wave[pos] = mem;
        w.kid[mem] = static_cast<short>(w.next + 2 * pos);
        ppar[(w.next + 2 * pos - 1) >> 1] = mem;
      }
      __syncwarp();
      if (lane == 0) w.nav = nav2;
    }
    if (lane == 0) {
      w.nfr = s_nfr;
      w.committed = committed;
      w.done = W == 0 ? 1 : 0;
      w.W = W;
      w.nsmall = nsmall;
      w.next += 2 * W;
      w.expanded += W;
      // small members' feature chunks: ~one (member, chunk) item per CTA
      const int target = nsmall > 0 ? max(1, static_cast<int>(gridDim.x) / nsmall) : 1;
      w.wc = min(a.wcap, max(1, (a.d + target - 1) / target));
      w.nwc = (a.d + w.wc - 1) / w.wc;
    }
  }
  __syncthreads();
}

// Warp 0 (lane j: member j): the members' splits as Descs (the parents'
// records were published before an earlier barrier); thread 0 then lays out
// the shared-memory histogram items. Whole CTA.
__device__ void load_members(const GrowArgs& a, WaveSmem& w, Desc* Dm) {
  const int lane = threadIdx.x;
  if (lane < w.W) {
    Desc& D = Dm[lane];
    const int x = w.wave[lane], kd = w.kid[x];
    const bool large = lane >= w.nsmall;
    const NodeDev* P = a.nodes + static_cast<size_t>(blockIdx.x % kRep) * a.max_nodes + x;
    const int64_t begin = __ldcg(&P->begin), count = __ldcg(&P->count), gcount = __ldcg(&P->gcount);
    const int buf = __ldcg(&P->buf);
    const int64_t nl = __ldcg(&P->best.left_count);
    D.done = 0;
    D.iter = w.nwaves;
    D.mslot = lane;
    D.pbase = 0;
    D.parent = x;
    D.left_id = kd;
    D.right_id = kd + 1;
    D.buf_in = buf;
    D.buf_out = 1 - buf;
    D.begin = begin;
    D.count = count;
    D.feature = __ldcg(&P->best.feature);
    D.thr = __ldcg(&P->best.threshold_bin);
    D.nl = nl;
    D.nr = gcount - nl;
    if (D.nl <= 0 || D.nr <= 0) set_error(a, kErrEmptySide);  // tree.cpp:124-126
    D.lsplit = splittable(D.nl, a.min_data);
    D.rsplit = splittable(D.nr, a.min_data);
    D.small_is_left = D.nl <= D.nr;
    const int64_t ns = D.nl <= D.nr ? D.nl : D.nr;
    D.items = 0;
    if (!(D.lsplit || D.rsplit)) {
      D.path = kNoHist;
    } else if (!large || (ns <= kDirectRows && ns * a.fchunk <= kDirectBudget)) {
      D.path = kDirect;
    } else {  // grow_kernel's segment plan (pick)
      D.path = kSmem;
      const int64_t min_rows = static_cast<int64_t>(a.wpg) * 32 * 2 * a.rpl;
      int64_t nseg = gridDim.x / a.nblocks;
      if (nseg < 1) nseg = 1;
      const int64_t cap = (ns + min_rows - 1) / min_rows;
      if (nseg > cap) nseg = cap;
      int64_t seg_len = (ns + nseg - 1) / nseg;
      seg_len = (seg_len + 31) / 32 * 32;
      nseg = (ns + seg_len - 1) / seg_len;
      D.seg_len = seg_len;
      D.nseg = static_cast<int32_t>(nseg);
      D.items = static_cast<int32_t>(nseg * a.nblocks);
    }
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    int h = 0, dd = 0;
    for (int j = w.nsmall; j < w.W; ++j) {
      Dm[j].pbase = h;
      h += Dm[j].items;
      dd += Dm[j].path == kDirect ? a.nchunks : 0;
    }
    w.hitems = h;
    w.ditems = dd;
  }
  __syncthreads();
}

// After the wave's last barrier, every CTA: warp j builds member j's
// children records — per child, the winner over its chunk winners (as
// winners()), the totals from the partition (large members: every CTA's own
// Desc; small members: a.wtot, written by their item CTAs) — into shared
// memory for wave_integrate, and writes them to the CTA's own replica of the
// node records (the copies any CTA reads later are then its own writes, or
// identical writes of another CTA with the same replica: no barrier needed
// before this CTA's next load_members). Replaces a last-arriver publish
// before the barrier (an atomic and a load round trip on the critical CTA).
template <int NT>
__device__ void wave_publish(const GrowArgs& a, WaveSmem& w, const Desc* Dm) {
  const int W = w.W, wp = static_cast<int>(threadIdx.x >> 5);
  if (wp < W) {
    const Desc& D = Dm[wp];
    const int lane = threadIdx.x & 31, child = lane >> 4, sub = lane & 15;
    const bool small = wp < w.nsmall;
    const int nwc = small ? w.nwc : a.nchunks;
    const bool want = D.path != kNoHist && (child == 0 ? D.lsplit : D.rsplit);
    Cand c{0.0, -1, -1, 0.0, 0.0, 0};
    unsigned long long hk = 0ull;
    unsigned lk = 0u;
    if (want) {
      const Cand* base = a.wcand + (static_cast<size_t>(D.mslot) * 2 + child) * a.wcstride;
      for (int i = sub; i < nwc; i += 16) {
        Cand o;
        o.gain = __ldcg(&base[i].gain);
        o.f = __ldcg(&base[i].f);
        o.b = __ldcg(&base[i].b);
        o.lg = __ldcg(&base[i].lg);
        o.lh = __ldcg(&base[i].lh);
        o.lc = __ldcg(&base[i].lc);
        const unsigned long long h = o.f >= 0 ? gain_key(o.gain) : 0ull;
        const unsigned l = 0xFFFFFFFFu - ((static_cast<unsigned>(o.f) << 12) | static_cast<unsigned>(o.b));
        const bool take = h > hk || (h == hk && l > lk);
        hk = take ? h : hk;
        lk = take ? l : lk;
        if (take) c = o;
      }
    }
    double tg = 0.0, th = 0.0;
    if (sub == 0) {
      tg = small ? __ldcg(a.wtot + 4 * D.mslot + 2 * child) : D.tot[2 * child];
      th = small ? __ldcg(a.wtot + 4 * D.mslot + 2 * child + 1) : D.tot[2 * child + 1];
    }
    warp_argmax_key(hk, lk, 16);
    {
      const unsigned mine = (hk != 0ull && c.f >= 0 && gain_key(c.gain) == hk &&
                             0xFFFFFFFFu - ((static_cast<unsigned>(c.f) << 12) | static_cast<unsigned>(c.b)) == lk)
                                ? 1u : 0u;
      const unsigned bal = __ballot_sync(0xffffffffu, mine) & (child == 0 ? 0x0000FFFFu : 0xFFFF0000u);
      const int src = bal ? __ffs(bal) - 1 : lane;
      const Cand wv = shfl_cand(c, src);
      c = hk == 0ull ? Cand{0.0, -1, -1, 0.0, 0.0, 0} : wv;
    }
    if (sub == 0) {
      NodeDev& r = w.wrec[2 * wp + child];
      // one rank (the wave grower's only case): this rank's rows are all rows
      r.begin = child == 0 ? D.begin : D.begin + D.nl;
      r.count = child == 0 ? D.nl : D.count - D.nl;
      r.gcount = child == 0 ? D.nl : D.nr;
      r.grad = tg;
      r.hess = th;
      r.buf = D.buf_out;
      if (want) {
        write_split(c, r.grad, r.hess, r.gcount, a.lambda, &r.best);
        r.has_best = c.f >= 0 ? 1 : 0;
      } else {
        r.best = hbg_split{};
        r.best.feature = -1;
        r.has_best = 0;
      }
    }
  }
  __syncthreads();
  const size_t rep = static_cast<size_t>(blockIdx.x % kRep);
  constexpr int Wd = static_cast<int>(sizeof(NodeDev) / 8);
  for (int t = threadIdx.x; t < 2 * W * Wd; t += NT) {
    const int m = t / (2 * Wd), ch = (t / Wd) % 2, q = t % Wd;
    reinterpret_cast<double*>(a.nodes + rep * a.max_nodes + Dm[m].left_id + ch)[q] =
        reinterpret_cast<const double*>(&w.wrec[2 * m + ch])[q];
  }
  for (int t = threadIdx.x; t < 2 * W; t += NT)
    a.node_gain[rep * a.max_nodes + Dm[t >> 1].left_id + (t & 1)] = w.wrec[t].has_best ? w.wrec[t].best.gain : -1.0;
  __syncthreads();
}

// A small member's item CTA: the children totals it ranked (wave_publish reads them).
__device__ __forceinline__ void member_totals(const GrowArgs& a, const Desc& D) {
  if (threadIdx.x == 0)
    for (int q = 0; q < 4; ++q) a.wtot[4 * D.mslot + q] = D.tot[q];
}

__device__ __forceinline__ CandOut wave_out(const GrowArgs& a, const Desc& D, int c) {
  return CandOut{a.wcand + static_cast<size_t>(D.mslot) * 2 * a.wcstride + c, 1, 0, a.wcstride};
}

// CTA owning (member, chunk) item x of I items over G CTAs (contiguous runs).
__device__ __forceinline__ int item_cta(int x, int I, int G) {
  return I <= G ? x : static_cast<int>((static_cast<int64_t>(x + 1) * G + I - 1) / I) - 1;
}

// Small members: items (member, feature chunk of wc features); every CTA of a
// member ranks its parent in registers and writes one share of the output.
template <int K, int NT>
__device__ void wave_small(const GrowArgs& a, const WaveSmem& w, Desc* Dm, PartShared<NT>& ps, unsigned char* smem) {
  const int G = gridDim.x, b = blockIdx.x;
  const int nwc = w.nwc, wc = w.wc, I = w.nsmall * nwc;
  int x0, x1;
  if (I <= G) {
    x0 = b < I ? b : I;
    x1 = b < I ? b + 1 : I;
  } else {
    x0 = static_cast<int>(static_cast<int64_t>(b) * I / G);
    x1 = static_cast<int>(static_cast<int64_t>(b + 1) * I / G);
  }
  int cur = -1;
  RegRows rr;
  for (int x = x0; x < x1; ++x) {
    const int j = x / nwc, c = x - j * nwc;
    Desc& D = Dm[j];
    if (j != cur) {
      const int bj0 = item_cta(j * nwc, I, G), bj1 = item_cta((j + 1) * nwc - 1, I, G);
      partition_redundant<NT>(a, D, rr, ps, bj1 - bj0 + 1, b - bj0, part_stage(a, smem));
      cur = j;
    }
    if (D.path == kDirect) {
      const int f0 = c * wc, nf = min(wc, a.d - f0);
      zero_direct(a, smem, nf * a.k, NT);
      __syncthreads();
      const uint32_t valid = rr.nvalid >= 32 ? ~0u : ((1u << rr.nvalid) - 1u);
      const uint32_t want = (D.small_is_left ? rr.left : ~rr.left) & valid;
      double eg, eh;
      direct_scales_regs(rr.g, rr.h, want, eg, eh);
      direct_accumulate(a, direct_acc(a, smem), nf * a.k, f0, nf, rr.row, rr.g, rr.h, want, eg, eh);
      __syncthreads();
      finish_range<K, NT>(a, D, f0, nf, 0, smem, wave_out(a, D, c));
    }
    member_totals(a, D);
  }
}

// Large members after their partition: direct-path items (member, chunk) and
// shared-memory histogram items (member, segment, slice block) over all CTAs;
// then (barrier) the shared-memory members' chunk finishes.
template <int BITS, int K, int NT>
__device__ void wave_large_hist(const GrowArgs& a, const WaveSmem& w, Desc* Dm, unsigned char* smem) {
  const int G = gridDim.x;
  const int hitems = w.hitems, total = w.hitems + w.ditems;
  for (int x = blockIdx.x; x < total; x += G) {
    if (x < hitems) {  // heavy items first
      int j = w.nsmall;
      while (Dm[j].path != kSmem || x >= Dm[j].pbase + Dm[j].items) ++j;
      hist_smem_item<BITS, K, NT>(a, Dm[j], x - Dm[j].pbase, smem);
      continue;
    }
    int r = x - hitems, j = w.nsmall;
    while (Dm[j].path != kDirect || r >= a.nchunks) {
      if (Dm[j].path == kDirect) r -= a.nchunks;
      ++j;
    }
    const Desc& D = Dm[j];
    const int c = r, f0 = c * a.fchunk, nf = min(a.fchunk, a.d - f0);
    zero_direct(a, smem, nf * a.k, NT);
    __syncthreads();
    const int32_t* rows;
    const float* g;
    const float* h;
    int64_t n;
    small_child(a, D, rows, g, h, n);
    double eg, eh;
    direct_scales_range<NT>(g, h, n, eg, eh);
    for (int64_t j0 = 0; j0 < n; j0 += static_cast<int64_t>(NT) * kItems) {
      int32_t rw[kItems];
      float gg[kItems], hh[kItems];
      uint32_t mask = 0;
#pragma unroll
      for (int u = 0; u < kItems; ++u) {
        const int64_t q = j0 + static_cast<int64_t>(u) * NT + threadIdx.x;
        const bool ok = q < n;
        rw[u] = ok ? __ldcg(rows + q) : 0;
        gg[u] = ok ? __ldcg(g + q) : 0.f;
        hh[u] = ok ? __ldcg(h + q) : 0.f;
        mask |= ok ? 1u << u : 0u;
      }
      direct_accumulate(a, direct_acc(a, smem), nf * a.k, f0, nf, rw, gg, hh, mask, eg, eh);
    }
    __syncthreads();
    finish_range<K, NT>(a, D, f0, nf, 0, smem, wave_out(a, D, c));
  }
  if (hitems == 0) return;
  stamp(a, w.nwaves, 17);  // CTA 0's items done
  if (a.prof != nullptr) {  // slot 18: the last CTA's arrival at the items' barrier
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(a.prof + static_cast<size_t>(w.nwaves) * kProfSlots + 18, global_ns());
  }
  grid_sync(a);
  stamp(a, w.nwaves, 19);
  int nsm = 0;
  for (int j = w.nsmall; j < w.W; ++j) nsm += Dm[j].path == kSmem ? 1 : 0;
  for (int x = blockIdx.x; x < nsm * a.nchunks; x += G) {
    int q = x / a.nchunks, j = w.nsmall;
    const int c = x - q * a.nchunks;
    while (Dm[j].path != kSmem || q > 0) {
      if (Dm[j].path == kSmem) --q;
      ++j;
    }
    const Desc& D = Dm[j];
    const int f0 = c * a.fchunk;
    finish_range<K, NT>(a, D, f0, min(a.fchunk, a.d - f0), 0, smem, wave_out(a, D, c));
  }
}

// The output from the replayed commit log (every CTA holds the same log):
// split i, the split node, its two children (tree.cpp:224-246). And for the
// score update: the rows of every unexpanded node (the leaves of the
// speculative tree partition the rows; an unexpanded node's range in its
// buffer is never written after its creation) with the value of the final
// leaf that contains it.
__device__ void wave_emit(const GrowArgs& a, const WaveSmem& w, unsigned char* smem) {
  const short* ppar = wave_ppar(a);
  const int committed = w.committed;
  const int stride = gridDim.x * blockDim.x;
  unsigned char* split = smem;  // node committed as a split (from the log)
  for (int u = threadIdx.x; u < w.next; u += blockDim.x) split[u] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < committed; i += blockDim.x) split[w.cnode[i]] = 1;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < committed; i += stride) {
    const int x = w.cnode[i], kd = w.ckid[i], o = w.cout[i], later = w.later[i];
    const hbg_split bs = load_split(&a.nodes[x].best);
    a.split_log[i] = bs;
    a.tree[o] = hbg_tree_node{bs.feature, bs.threshold_bin, 2 * i + 1, 2 * i + 2, 0.0};
    for (int c = 0; c < 2; ++c) {
      if ((later >> c) & 1) continue;  // a child split later is written by its own commit
      const NodeDev* q = a.nodes + kd + c;
      a.tree[2 * i + 1 + c] = hbg_tree_node{-1, -1, -1, -1, leaf_value(__ldcg(&q->grad), __ldcg(&q->hess), a.lambda)};
    }
  }
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < w.next; u += stride) {
    LeafRange r{0, 0, 0.0, 0, 0};
    if (w.kid[u] < 0) {
      int z = u;  // the final leaf above u: the first node whose parent was committed as a split
      while (z != 0 && !split[ppar[(z - 1) >> 1]]) z = ppar[(z - 1) >> 1];
      const NodeDev* q = a.nodes + u;
      const NodeDev* f = a.nodes + z;
      r = LeafRange{__ldcg(&q->begin), __ldcg(&q->count), leaf_value(__ldcg(&f->grad), __ldcg(&f->hess), a.lambda),
                    __ldcg(&q->buf), 0};
    }
    a.ranges[u] = r;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.counts[0] = committed;
    a.counts[1] = 1 + 2 * committed;
    a.counts[4] = w.next;
  }
}

template <int BITS, int K>
__global__ void __launch_bounds__(grow_threads<K>(), 1) grow_wave_kernel(GrowArgs a) {
  constexpr int NT = grow_threads<K>();
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ PartShared<NT> ps;
  __shared__ Desc Dm[kWMax];
  __shared__ WaveSmem w;
  // the root (histogram, totals, best split computed by host-launched kernels)
  if (threadIdx.x == 0) {
    const double G = __ldcg(a.root_tot), H = __ldcg(a.root_tot + 1);
    const hbg_split bs = load_split(&a.nodes[0].best);
    const int hb = bs.feature >= 0 ? 1 : 0;
    if (blockIdx.x == 0) {
      const NodeDev rec{0, a.root_count, a.root_count, G, H, bs, 0, hb};
      for (int q = 0; q < kRep; ++q) a.nodes[static_cast<size_t>(q) * a.max_nodes] = rec;
      for (int q = 0; q < kRep; ++q) a.node_gain[static_cast<size_t>(q) * a.max_nodes] = hb ? bs.gain : -1.0;
      a.tree[0] = hbg_tree_node{-1, -1, -1, -1, leaf_value(G, H, a.lambda)};
    }
    const unsigned long long k0 = hb ? gain_key(bs.gain) : 0ull;
    w.gkey[0] = k0;
    w.prio[0] = hb ? static_cast<float>(bs.gain) : 0.f;
    w.kid[0] = -1;
    w.large[0] = runs_large(a, a.root_count, hb ? bs.left_count : 0) ? (a.root_count <= a.spec_rows ? 1 : 2) : 0;
    w.nav = w.nfr = w.nfresh = 0;
    w.committed = w.expanded = w.done = w.W = w.nsmall = w.nwaves = w.err = 0;
    w.next = 1;
    if (k0 != 0ull && a.num_leaves >= 2) {
      w.fkey[0] = k0;
      w.fnode[0] = 0;
      w.fout[0] = 0;
      w.avail[0] = av_pack(0, w.large[0], prio_bucket(w.prio[0]));
      w.nfr = w.nav = 1;
    }
  }
  grid_sync(a);  // CTA 0's root records
  wave_select<NT>(a, w);
  while (!w.done) {
    if (a.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long* t = a.prof + static_cast<size_t>(w.nwaves) * kProfSlots;
      t[7] = static_cast<unsigned long long>(w.W - w.nsmall);
      t[10] = static_cast<unsigned long long>(w.W);
      t[11] = static_cast<unsigned long long>(w.committed);
    }
    stamp(a, w.nwaves, 0);
    load_members(a, w, Dm);
    for (int j = w.nsmall; j < w.W; ++j) partition_count<NT>(a, Dm[j], ps);
    if (w.nsmall > 0) wave_small<K, NT>(a, w, Dm, ps, smem);
    stamp(a, w.nwaves, 1);
    if (w.W > w.nsmall) {
      grid_sync(a);
      for (int j = w.nsmall; j < w.W; ++j) partition_scatter<NT>(a, Dm[j], ps, smem);
      grid_sync(a);
      stamp(a, w.nwaves, 2);
      wave_large_hist<BITS, K, NT>(a, w, Dm, smem);
    }
    stamp(a, w.nwaves, 3);
    if (a.prof != nullptr) {  // slot 16: the last CTA's arrival at the wave's final barrier
      __syncthreads();
      if (threadIdx.x == 0) atomicMax(a.prof + static_cast<size_t>(w.nwaves) * kProfSlots + 16, global_ns());
    }
    grid_sync(a);
    stamp(a, w.nwaves, 4);
    wave_publish<NT>(a, w, Dm);
    if (threadIdx.x < 32) wave_integrate(a, w);
    stamp(a, w.nwaves, 6);
    if (threadIdx.x == 0) ++w.nwaves;
    wave_select<NT>(a, w);
    stamp(a, w.nwaves - 1, 5);
  }
  wave_emit(a, w, smem);
  if (blockIdx.x == 0 && threadIdx.x == 0) a.counts[3] = w.nwaves;
}

// scores[row] += lr * value for every leaf node (tree[i].left < 0) of a grown
// tree (boosting.cpp:48-50); every leaf owns a contiguous ordered-buffer range.
__global__ void score_update_nodes_kernel(const NodeDev* __restrict__ nodes,
                                          const hbg_tree_node* __restrict__ tree,
                                          const int32_t* __restrict__ rows0, const int32_t* __restrict__ rows1,
                                          double lr, double* __restrict__ scores) {
  const int i = blockIdx.y;
  if (tree[i].left >= 0) return;
  const NodeDev L = nodes[i];
  const int32_t* rows = L.buf == 0 ? rows0 : rows1;
  const double add = lr * tree[i].value;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < L.count;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    scores[rows[L.begin + j]] += add;
}

template <int BITS, int K>
struct GrowKernel {
  static void* fn(bool wave) {
    return wave ? reinterpret_cast<void*>(grow_wave_kernel<BITS, K>) : reinterpret_cast<void*>(grow_kernel<BITS, K>);
  }
};

void* grow_fn(int bits, int k_alloc, bool wave) {
  if (bits == 4) return GrowKernel<4, 16>::fn(wave);
  if (k_alloc == 64) return GrowKernel<8, 64>::fn(wave);
  if (k_alloc == 128) return GrowKernel<8, 128>::fn(wave);
  return GrowKernel<8, 256>::fn(wave);
}

// The wave grower runs single-rank trees of the shapes where it pays (below;
// HBG_GROW=wave forces it, HBG_GROW=legacy disables it), and only while its
// node slots (speculative expansions included) fit kWaveSlotBudget.
constexpr size_t kWaveSlotBudget = size_t(4) << 30;

// Speculative expansions allowed beyond the num_leaves-1 the tree commits;
// -1: the wave grower does not apply (row shards, > kWL leaves, 256-bin
// slots — the shared-memory state would cost the histogram a third of its
// warps — or node slots beyond kWN / kWaveSlotBudget).
int wave_extra(const PersistentGrowArgs& h) {
  const char* e = std::getenv("HBG_GROW");
  if (h.nranks > 1 || (e != nullptr && std::strcmp(e, "legacy") == 0)) return -1;
  if (h.num_leaves > kWL || (h.bits != 4 && h.k > 128)) return -1;
  // waves pay where the per-split chain (partition, histogram, scans,
  // barrier, pick) dominates and a speculative expansion is cheap: 8-bit data
  // with <= 4096 feature x bin cells. Measured (255 leaves, min_data 1) against
  // one split per barrier: Higgs 28 x k64 at 1M rows 2.4 vs 4.6 ms, 3M 2.6 vs
  // 5.3, 10.5M 5.4 vs 6.0; but 200 features 7.3 vs 5.2 and the 4-bit k16
  // kernel 6.8 vs 6.0 (10.5M rows).
  const bool forced = e != nullptr && std::strcmp(e, "wave") == 0;  // HBG_GROW=wave: whenever it fits
  if (!forced && (h.bits == 4 || static_cast<long long>(h.d) * h.k > 4096)) return -1;
  const int L1 = std::max(0, h.num_leaves - 1);
  const size_t slot = static_cast<size_t>(3) * h.d * h.k * sizeof(double);
  const long long fit = std::min<long long>(kWN, static_cast<long long>(kWaveSlotBudget / std::max<size_t>(slot, 1)));
  const long long x = std::min<long long>(L1, (fit - 1) / 2 - 2LL * L1);
  return x < 0 ? -1 : static_cast<int>(x);
}

int wave_max_members() {
  const char* e = std::getenv("HBG_WAVE_MAX");
  const int m = e != nullptr ? std::atoi(e) : 16;
  return std::max(1, std::min(kWMax, m));
}

int grow_nt(int k_alloc) { return k_alloc >= 256 ? grow_threads<256>() : grow_threads<64>(); }

constexpr size_t kSmemMax = 232448;  // static + dynamic shared memory per CTA

size_t grow_static_smem(void* fn) {
  cudaFuncAttributes attr{};
  HBG_CUDA(cudaFuncGetAttributes(&attr, fn));
  return attr.sharedSizeBytes;
}

struct GrowGeom {
  int k_alloc, nt, gb, wpg, nblocks, fchunk, nchunks, ctas;
  int cchunk, wcap;  // chunk capacity of the shared-memory layout; wave chunk limit
  bool wave;
  int extra, ecap, wmax, max_nodes;
  size_t wcstride;
  size_t smem, part_values;
};

GrowGeom grow_geometry(const PersistentGrowArgs& h, int device) {
  GrowGeom g{};
  g.k_alloc = h.bits == 4 ? 16 : (h.k <= 64 ? 64 : (h.k <= 128 ? 128 : 256));
  g.nt = grow_nt(g.k_alloc);
  const size_t cells = static_cast<size_t>(g.k_alloc) * 32;
  const size_t ghw = cells * 8, cntw = cells * 4;
  g.extra = wave_extra(h);
  g.wave = g.extra >= 0;
  // both kernels lay out the shared-memory histogram for the same budget
  // when the wave kernel applies to this shape (the partials, hence the
  // trees, are then bit-identical between them)
  const bool wave_shape = h.num_leaves <= kWL && (h.bits == 4 || h.k <= 128);
  const size_t smem_max = kSmemMax - std::max(grow_static_smem(grow_fn(h.bits, g.k_alloc, false)),
                                              wave_shape ? grow_static_smem(grow_fn(h.bits, g.k_alloc, true)) : 0);
  const int max_warps = g.nt / 32;
  int gb = 0, warps = 0;
  for (int cand = 1; cand <= std::min(h.num_groups, max_warps); ++cand) {
    if (cand * cntw >= smem_max) break;
    const int wpg = static_cast<int>(std::min<size_t>(max_warps, (smem_max - cand * cntw) / ghw)) / cand;
    if (wpg < 1) break;
    if (cand * wpg >= warps) {
      gb = cand;
      warps = cand * wpg;
    }
  }
  require(gb >= 1, "histogram footprint exceeds shared memory");
  g.gb = gb;
  g.wpg = warps / gb;
  g.nblocks = (h.num_groups + gb - 1) / gb;
  g.ctas = h.ctas > 0 ? std::min(h.ctas, sm_count(device)) : sm_count(device);
  // scan chunks: one per CTA at most (the direct paths give CTA c chunk c), so
  // at least ceil(d / CTAs) features each; the staging must fit shared memory
  g.fchunk = std::max(1, (h.d + g.ctas - 1) / g.ctas);
  g.nchunks = std::max(1, (h.d + g.fchunk - 1) / g.fchunk);
  const size_t hist_smem = static_cast<size_t>(g.gb * g.wpg) * ghw + g.gb * cntw;
  // finish: fp64 staging of both children + the direct fixed-point accumulator
  // (+ the small-parent partition staging), per feature of a chunk
  const size_t per_feature = static_cast<size_t>(h.k) * (6 * sizeof(double) + 20);
  const size_t stage_smem = static_cast<size_t>(kItems) * g.nt * 12;
  auto part_smem_of = [&](int f) { return (f * per_feature + 15) / 16 * 16 + stage_smem; };
  // wave chunks: as many features as the shared memory holds (up to d)
  g.wcap = 1;
  while (g.wcap < h.d && part_smem_of(g.wcap + 1) <= smem_max) ++g.wcap;
  g.cchunk = std::max(g.fchunk, g.wave ? g.wcap : g.fchunk);
  const size_t part_smem = part_smem_of(g.cchunk);
  g.smem = std::max(hist_smem, part_smem);
  require(g.ctas <= g.nt, "more CTAs than threads per CTA (per-CTA records are scanned one per thread)");
  require(g.smem <= smem_max, "tree grower: features x bins per scan chunk exceed shared memory "
                              "(too many features for one grid)");
  const size_t items = static_cast<size_t>(std::max(g.ctas, g.nblocks));
  g.part_values = items * g.gb * cells;
  const int L1 = std::max(0, h.num_leaves - 1);
  g.wmax = wave_max_members();
  g.wcstride = static_cast<size_t>(std::max({g.ctas, g.nchunks, (h.d + g.wcap - 1) / g.wcap}));
  if (g.wave) g.part_values *= static_cast<size_t>(g.wmax);  // every large member of a wave
  g.ecap = L1 + std::max(0, g.extra);
  // node ids: the root + 2 per expansion; speculative expansions stop at
  // ecap, the certain ones (<= L1) may go past it
  g.max_nodes = g.wave ? 1 + 2 * (g.ecap + L1) : std::max(1, 2 * h.num_leaves - 1);
  return g;
}

}  // namespace

int grow_max_nodes(const PersistentGrowArgs& h, int device) { return grow_geometry(h, device).max_nodes; }

size_t grow_nodes_bytes(int max_nodes) {  // kRep replicas; replica 0 first
  return static_cast<size_t>(kRep) * std::max(1, max_nodes) * sizeof(NodeDev);
}

size_t grow_root_split_offset() { return offsetof(NodeDev, best); }

size_t grow_exchange_doubles(const PersistentGrowArgs& h, int device) {
  const GrowGeom g = grow_geometry(h, device);
  const size_t block = kXBlockHeader + static_cast<size_t>(3) * g.fchunk * h.k;
  return kXHeader + static_cast<size_t>(2) * g.nchunks * block;
}

size_t grow_scratch_bytes(const PersistentGrowArgs& h, int device) {
  const GrowGeom g = grow_geometry(h, device);
  const size_t max_nodes = static_cast<size_t>(g.max_nodes);
  size_t b = 0;
  auto add = [&](size_t n) { b += (n + 255) / 256 * 256; };
  add(sizeof(unsigned));                      // barrier
  add(kRep * max_nodes * sizeof(double));     // node_gain
  add(kRep * max_nodes * sizeof(int));        // picked
  add(static_cast<size_t>(h.num_rows) + 16);  // flags
  add(static_cast<size_t>(g.ctas) * 8 * (g.wave ? g.wmax : 1));   // cta_left
  add(static_cast<size_t>(g.ctas) * (g.nt / 32) * 4 * (g.wave ? g.wmax : 1));  // warp_left
  add(static_cast<size_t>(g.ctas) * 32 * (g.wave ? g.wmax : 1));  // cta_sums
  add(g.part_values * 4 * 3);                 // part_g/h/c
  add(static_cast<size_t>(kRep * 2 * g.nchunks) * sizeof(Cand));
  if (g.wave) {
    add(static_cast<size_t>(2 * g.wmax) * g.wcstride * sizeof(Cand));           // wcand
    add(static_cast<size_t>(g.wmax) * 4 * sizeof(double));                      // wtot
    add(static_cast<size_t>(g.ctas) * wave_state_bytes(h.num_leaves, g.max_nodes));  // wstate
    add(static_cast<size_t>(g.max_nodes) * sizeof(LeafRange));                       // ranges
  }
  return b;
}

void configure_grow_kernels() {
  for (int v = 0; v < 8; ++v) {
    const int bits = (v & 3) == 0 ? 4 : 8, k = (v & 3) == 0 ? 16 : ((v & 3) == 1 ? 64 : ((v & 3) == 2 ? 128 : 256));
    void* fn = grow_fn(bits, k, v >= 4);
    HBG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemMax - grow_static_smem(fn))));
    set_max_shared_carveout(fn);
  }
}

void launch_score_update_nodes(const void* nodes, const hbg_tree_node* tree, int num_nodes,
                               const int32_t* rows0, const int32_t* rows1, double lr, double* scores,
                               cudaStream_t s) {
  if (num_nodes <= 0) return;
  score_update_nodes_kernel<<<dim3(16, num_nodes), 256, 0, s>>>(static_cast<const NodeDev*>(nodes), tree, rows0,
                                                                rows1, lr, scores);
  HBG_LAUNCH_CHECK();
}

const void* launch_grow_persistent(const PersistentGrowArgs& h, int device, cudaStream_t s) {
  const GrowGeom g = grow_geometry(h, device);
  GrowArgs a{};
  a.packed = h.packed;
  a.colbins = h.colbins;
  a.nrows = h.num_rows;
  a.row_stride = h.row_stride;
  a.group_stride = h.group_stride;
  a.words_per_row = h.words_per_row;
  a.bits = h.bits;
  a.d = h.d;
  a.k = h.k;
  a.num_groups = h.num_groups;
  for (int b = 0; b < 2; ++b) {
    a.rows[b] = h.rows[b];
    a.g[b] = h.g[b];
    a.h[b] = h.h[b];
  }
  a.slots = h.slots;
  a.nodes = static_cast<NodeDev*>(h.nodes);
  a.split_log = h.split_log;
  a.tree = h.tree;
  a.counts = h.counts;
  a.root_tot = h.root_totals;
  a.root_count = h.num_rows;
  a.num_leaves = h.num_leaves;
  a.min_data = h.min_data;
  a.lambda = h.lambda;
  a.gb = g.gb;
  a.wpg = g.wpg;
  a.nblocks = g.nblocks;
  a.rpl = g.k_alloc >= 256 ? rows_per_lane<256>() : rows_per_lane<64>();
  a.fchunk = g.fchunk;
  a.nchunks = g.nchunks;
  a.cchunk = g.cchunk;
  a.wcap = g.wcap;
  a.wmax = g.wmax;
  a.wlarge = std::getenv("HBG_WAVE_LARGE") != nullptr ? std::atoi(std::getenv("HBG_WAVE_LARGE")) : 1;
  a.spec_rows = std::getenv("HBG_WAVE_SPEC_ROWS") != nullptr ? std::atoll(std::getenv("HBG_WAVE_SPEC_ROWS")) : 262144;
  a.wcstride = g.wcstride;
  a.ecap = g.ecap;
  a.small_max = static_cast<int64_t>(kItems) * g.nt;
  a.timeout_cycles = h.timeout_cycles;  // a hung barrier or exchange becomes an error, not a hang
  a.prof = h.prof;
  a.nranks = std::max(1, h.nranks);
  a.debug = std::getenv("HBG_GROW_DEBUG") != nullptr;
  a.rank = h.rank;
  require(a.nranks <= kMaxRanks, "at most 8 row shards exchange through peer memory");
  if (a.nranks > 1) {
    require(h.xown != nullptr, "row sharding needs the exchange areas");
    a.xown = h.xown;
    for (int r = 0; r < a.nranks; ++r) {
      require(h.xpeer[r] != nullptr, "exchange area of a rank not attached");
      a.xpeer[r] = h.xpeer[r];
    }
    a.xblock = kXBlockHeader + static_cast<size_t>(3) * g.fchunk * h.k;
    a.gen = h.gen;
  }
  unsigned char* p = static_cast<unsigned char*>(h.scratch);
  auto take = [&](size_t n) {
    unsigned char* q = p;
    p += (n + 255) / 256 * 256;
    return q;
  };
  const size_t max_nodes = static_cast<size_t>(g.max_nodes);
  a.bar = reinterpret_cast<unsigned*>(take(sizeof(unsigned)));
  a.max_nodes = static_cast<int>(max_nodes);
  a.node_gain = reinterpret_cast<double*>(take(kRep * max_nodes * sizeof(double)));
  a.picked = reinterpret_cast<int*>(take(kRep * max_nodes * sizeof(int)));
  a.flags = take(static_cast<size_t>(h.num_rows) + 16);
  a.cta_left = reinterpret_cast<int64_t*>(take(static_cast<size_t>(g.ctas) * 8 * (g.wave ? g.wmax : 1)));
  a.warp_left = reinterpret_cast<int*>(take(static_cast<size_t>(g.ctas) * (g.nt / 32) * 4 * (g.wave ? g.wmax : 1)));
  a.cta_sums = reinterpret_cast<double*>(take(static_cast<size_t>(g.ctas) * 32 * (g.wave ? g.wmax : 1)));
  float* part = reinterpret_cast<float*>(take(g.part_values * 12));
  a.part_g = part;
  a.part_h = part + g.part_values;
  a.part_c = reinterpret_cast<uint32_t*>(part + 2 * g.part_values);
  a.cand = reinterpret_cast<Cand*>(take(static_cast<size_t>(kRep * 2 * g.nchunks) * sizeof(Cand)));
  if (g.wave) {
    a.wcand = reinterpret_cast<Cand*>(take(static_cast<size_t>(2 * g.wmax) * g.wcstride * sizeof(Cand)));
    a.wtot = reinterpret_cast<double*>(take(static_cast<size_t>(g.wmax) * 4 * sizeof(double)));
    a.wstate_stride = wave_state_bytes(h.num_leaves, g.max_nodes);
    a.wstate = take(static_cast<size_t>(g.ctas) * a.wstate_stride);
    a.ranges = reinterpret_cast<LeafRange*>(take(static_cast<size_t>(g.max_nodes) * sizeof(LeafRange)));
  }

  require(static_cast<size_t>(p - static_cast<unsigned char*>(h.scratch)) <= h.scratch_bytes,
          "grow scratch smaller than its layout");
  HBG_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(unsigned), s));
  HBG_CUDA(cudaMemsetAsync(a.picked, 0, kRep * max_nodes * sizeof(int), s));
  HBG_CUDA(cudaMemsetAsync(a.counts, 0, 8 * sizeof(int), s));
  void* fn = grow_fn(h.bits, g.k_alloc, g.wave);
  int occ = 0;
  HBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, g.nt, g.smem));
  require(occ >= 1, "tree grower kernel cannot be resident");
  void* args[] = {&a};
  if (g.ctas == sm_count(device)) {
    HBG_CUDA(cudaLaunchCooperativeKernel(fn, dim3(g.ctas), dim3(g.nt), args, g.smem, s));
  } else {
    // a partial grid (several ranks sharing one GPU in tests): a plain launch
    // of one CTA per SM; every CTA of it is resident while the SMs suffice
    HBG_CUDA(cudaLaunchKernel(fn, dim3(g.ctas), dim3(g.nt), args, g.smem, s));
  }
  return g.wave ? static_cast<const void*>(a.ranges) : h.nodes;
}

}  // namespace hbg
