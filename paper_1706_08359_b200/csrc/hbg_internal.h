// hbg_internal.h — shared declarations between the C-ABI layer (capi.cu) and
// the kernels (hist_kernels.cu, leaf_kernels.cu). Not a public header.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "hbg.h"

namespace hbg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define HBG_CUDA(call)                                                    \
  do {                                                                    \
    cudaError_t hbg_e_ = (call);                                          \
    if (hbg_e_ != cudaSuccess) ::hbg::throw_cuda(hbg_e_, #call, __FILE__, __LINE__); \
  } while (0)
#define HBG_LAUNCH_CHECK() HBG_CUDA(cudaGetLastError())

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(HBG_ERR_INVALID_ARGUMENT, msg);
}

// Geometry of one histogram launch (chosen on the host by plan_histogram()).
struct HistPlan {
  int k_alloc;      // power-of-two bin slots per feature in shared memory (16/64/128/256)
  int bits;         // 4 or 8
  int warps;        // warps per CTA
  int gb;           // slice groups per CTA ("group block")
  int wpg;          // warps per group (row-interleaved over 32-row tiles)
  int nblocks;      // ceil(num_groups / gb)
  int nseg;         // row segments
  int64_t seg_len;  // leaf positions per segment (multiple of 32)
  int ctas;         // nblocks * nseg
  size_t smem;      // dynamic shared memory per CTA
  size_t part_values;  // entries in each partial array (ctas * gb * 32 * k_alloc)
  int acc_bytes;       // 4: fp32 g/h and cells (bits32); 8: fp64 (bits64)
  int cluster;         // > 1: ONE launch of clusters of this many CTAs (one per row segment);
                       //    the segments' sub-histograms are summed over distributed shared
                       //    memory inside each cluster (no grid barrier); with nclusters > 1
                       //    the clusters' fp64 sums meet in HBM and the last cluster to
                       //    finish adds them up
  int nclusters;       // clusters per group block (cluster mode)
};
// Bytes of one g/h partial element: the CTAs' own type, or fp64 for the
// cluster sums of the multi-cluster mode.
inline int part_elem_bytes(const HistPlan& p) { return p.cluster > 1 ? 8 : p.acc_bytes; }

struct HistArgs {
  const uint8_t* packed;
  int64_t row_stride;  // bytes between rows of one slice group (slice_bytes)
  int64_t group_stride;  // bytes between slice groups (group-planar layout)
  const int32_t* idx;  // nullptr: identity leaf
  int64_t n;
  const void* g;  // float (bits32) or double (bits64) per HistPlan::acc_bytes
  const void* h;
  int gh_indexed;
  int num_groups;
  int gb, wpg, nblocks;
  int64_t seg_len;
  void* part_g;  // per-CTA partials, same type as g/h
  void* part_h;
  uint32_t* part_c;
  // direct mode (a single row segment): the CTAs write the final fp64
  // histogram (and the fused sibling) themselves, no partials / reduce launch
  int direct;
  int d;
  int max_bin;
  double* out;
  const double* parent;
  double* sibling;
  // fused mode (HistPlan::fused): the grid barrier's counter (self-resetting,
  // one per dataset) and the segment count the reduction runs over
  int nseg;
  int cluster;  // HistPlan::cluster
  int nclusters;
  unsigned* bar;  // multi-cluster mode: one arrival counter per group block
  unsigned long long* prof;  // optional %globaltimer stamps of one CTA (HBG_HIST_PROFILE), 8 slots
  int prof_cta;              // the stamped CTA (HBG_HIST_PROFILE_CTA, default 0)
};

// allow_direct = false: always per-CTA partials + a reduction (the row-sharded
// path fuses its exchange into that reduction).
// acc_bytes: 4 = fp32 g/h inputs, cells and partials (PrecisionMode::bits32);
// 8 = fp64 throughout (PrecisionMode::bits64).
// allow_fused: leaves up to ~4 tiles per row warp on the resident clusters
// take the single-launch cluster mode (not where several ranks share a GPU
// and wait on each other inside kernels: clusters need whole GPCs free).
HistPlan plan_histogram(int bits, int max_bin, int num_groups, int64_t n, int device, bool allow_direct = true,
                        int acc_bytes = 4, bool allow_fused = false);
// Bytes of the partial buffers of a plan (g, h: acc_bytes each; count: 4).
inline size_t hist_part_bytes(const HistPlan& p) { return p.part_values * (2 * part_elem_bytes(p) + 4) + 16; }

void launch_histogram(const HistPlan& plan, const HistArgs& args, cudaStream_t s);
// d_hist = reduced histogram; when `parent` is non-null also writes
// sibling = parent - d_hist (histogram subtraction fused into the reduction;
// sibling may alias parent).
void launch_reduce_partials(const HistPlan& plan, const HistArgs& args, int num_features,
                            int max_bin, double* d_hist, cudaStream_t s,
                            const double* parent = nullptr, double* sibling = nullptr);
// Row-sharded histogram with the cross-rank sum fused into the reduction
// (reduce_exchange_kernel): every rank's exchange region is mapped.
struct PeerHistArgs {
  int nranks, rank;
  double* xown;
  const double* xpeer[8];
  unsigned long long tag;
  int parity;
  int* error;  // device flag: a peer never published (timeout)
  long long timeout_cycles;
};
size_t hist_exchange_doubles(int k_alloc, int max_bin, int num_groups);
void launch_reduce_exchange(const HistPlan& plan, const HistArgs& args, int num_features, int max_bin,
                            double* d_hist, const PeerHistArgs& x, cudaStream_t s);
// Packs features [f0, f0 + nf) (one 32-feature slice group; d_cols holds
// their column-major bins) into the group's words of every row.
void launch_pack(const uint8_t* d_cols, int f0, int nf, int num_features, int64_t num_rows,
                 int max_bin, int bits, int64_t group_stride_words, uint32_t* d_packed, int* d_bad,
                 cudaStream_t s);
void launch_iota(int32_t* out, int64_t n, cudaStream_t s);
void launch_f64_to_f32(const double* in, float* out, int64_t n, cudaStream_t s);
void launch_hist_to_bins(const double* d_hist, int64_t cells, hbg_bin* d_bins, cudaStream_t s);
void launch_subtract(const double* a, const double* b, double* out, int64_t n, cudaStream_t s);
void launch_gather(const int32_t* idx, int64_t n, const float* g, const float* h, float* lg,
                   float* lh, double* totals, double* scratch, cudaStream_t s);
// fp64 g/h (bits64): leaf-aligned copies (optional) and fixed-order totals.
void launch_gather_f64(const int32_t* idx, int64_t n, const double* g, const double* h, double* lg,
                       double* lh, double* totals, double* scratch, cudaStream_t s);
size_t gather_scratch_doubles(int64_t n);
// Split scans of 1-2 histograms in one launch (one CTA each): histogram i at
// d_hist + i*hist_stride, totals at d_totals + i*totals_stride, count
// d_counts[i] (or count0/count1 when d_counts is null), result out[i].
void launch_best_split_batch(const double* d_hist, int64_t hist_stride, int leaves, int d, int k,
                             const double* d_totals, int64_t totals_stride, const int64_t* d_counts,
                             int64_t count0, int64_t count1, double gt, double ht, int64_t min_data,
                             double lambda, hbg_split* out, cudaStream_t s);
void launch_best_split(const double* d_hist, int d, int k, const double* d_totals,
                       const int64_t* d_count, double gt, double ht, int64_t count,
                       int64_t min_data, double lambda, hbg_split* out, cudaStream_t s);

size_t partition_scratch_bytes(int64_t n);
// Stable split of one leaf's contiguous (row, g, h) range by bin(feature) <= thr
// into the other buffer (left rows first); d_totals = {gl, hl, gr, hr} (fp64),
// *d_left = rows sent left.
void launch_partition(const int32_t* rows, const float* g, const float* h, int64_t n,
                      const uint8_t* packed, int64_t row_stride, int feature, int bits, int thr,
                      int32_t* orow, float* og, float* oh, void* scratch, double* d_totals,
                      int64_t* d_left, cudaStream_t s);
// The same with fp64 g/h (PrecisionMode::bits64 trees).
void launch_partition_f64(const int32_t* rows, const double* g, const double* h, int64_t n,
                          const uint8_t* packed, int64_t row_stride, int feature, int bits, int thr,
                          int32_t* orow, double* og, double* oh, void* scratch, double* d_totals,
                          int64_t* d_left, cudaStream_t s);

// One final leaf of a grown tree: its rows' range in ordered buffer `buf`.
struct LeafRange {
  int64_t begin, count;
  double value;
  int32_t buf, pad;
};
void launch_grad_hess(int loss, const double* scores, const double* targets, int64_t n, float* g,
                      float* h, cudaStream_t s);
void launch_score_update(const LeafRange* leaves, int nleaves, const int32_t* rows0,
                         const int32_t* rows1, double lr, double* scores, cudaStream_t s);
void launch_reduce_parts(const std::vector<const double*>& parts, int64_t n, double* out,
                         cudaStream_t s);

void set_max_shared_carveout(const void* func);
void configure_hist_kernels(int device);
void configure_leaf_kernels();
void configure_tree_kernels();
void configure_kernels(int device);  // carveout for every non-histogram kernel, once per device

// Small leaves (tree grower): fixed-point histogram through L2 atomics.
constexpr int64_t kAtomicHistRows = 4096;
size_t small_hist_acc_bytes(int d, int k);
// fixed-point scales exps[0..1] from one leaf's rows (n <= kAtomicHistRows; one block)
void launch_fixed_leaf_scale(const float* g, const float* h, int64_t n, int* exps, cudaStream_t s);
void launch_small_hist(const int32_t* rows, const float* g, const float* h, int64_t n,
                       const uint32_t* packed, int64_t group_stride_words, int words_per_row, int bits, int d, int k,
                       const int* exps, void* acc, double* out, const double* parent, double* sibling,
                       cudaStream_t s);

// Small-leaf split tail fused: accumulator -> small/large histograms + both scans.
struct FinishScanArgsHost {
  void* acc;
  const int* exps;
  int d, k;
  double* small_out;
  double* large_io;
  int small_is_left;
  const double* totals;  // gl, hl, gr, hr
  int64_t nl, nr;
  int lsplit, rsplit;
  int64_t min_data;
  double lambda;
  hbg_split* out;  // [2]
};
void launch_finish_scan(const FinishScanArgsHost& a, cudaStream_t s);
void launch_small_hist_atomic(const int32_t* rows, const float* g, const float* h, int64_t n,
                              const uint32_t* packed, int64_t group_stride_words, int words_per_row, int bits, int d,
                              int k, const int* exps, void* acc, cudaStream_t s);

// Persistent tree grower (grow_persistent.cu): all splits of one tree in a
// single cooperative kernel, one CTA per SM.
struct PersistentGrowArgs {
  const uint8_t* packed;
  const uint8_t* colbins;  // [d][num_rows] uint8 bins
  int64_t row_stride;
  int64_t group_stride;  // group-planar packed layout
  int words_per_row, bits, d, k, num_groups;
  int64_t num_rows;
  int32_t* rows[2];
  float* g[2];
  float* h[2];
  double* slots;         // grow_max_nodes() node slots of 3*d*k doubles
  void* nodes;           // grow_nodes_bytes(num_leaves), nodes[0].best = root split
  hbg_split* split_log;  // device, num_leaves-1
  hbg_tree_node* tree;   // device, 2*num_leaves-1
  int* counts;           // device, 4 ints: num_splits, num_nodes, error
  void* scratch;         // grow_scratch_bytes()
  size_t scratch_bytes;  // allocated size of `scratch`
  const double* root_totals;  // device {G, H}
  int num_leaves;
  int64_t min_data;
  double lambda;
  unsigned long long* prof;  // optional phase stamps (HBG_GROW_PROFILE)
  int ctas;                  // 0: one CTA per SM (cooperative launch)
  // row sharding through peer memory (nranks > 1)
  int nranks, rank;
  double* xown;
  const double* xpeer[8];
  unsigned long long gen;
  long long timeout_cycles;  // bound of every in-kernel wait (wait_timeout_cycles)
};
// HBG_PEER_TIMEOUT_MS (default 60 s) in clock64 cycles of `device`
long long wait_timeout_cycles(int device);
size_t grow_exchange_doubles(const PersistentGrowArgs& a, int device);
int grow_max_nodes(const PersistentGrowArgs& a, int device);  // node-table entries of the kernel used
size_t grow_nodes_bytes(int max_nodes);
size_t grow_root_split_offset();
size_t grow_scratch_bytes(const PersistentGrowArgs& a, int device);
void configure_grow_kernels();
// Returns what the score update reads: the node records by output id
// (grow_kernel; launch_score_update_nodes) or, for the wave grower, counts[4]
// LeafRange entries (launch_score_update).
const void* launch_grow_persistent(const PersistentGrowArgs& a, int device, cudaStream_t s);
// scores[row] += lr * value for the rows of every leaf node of a persistent-grown tree
void launch_score_update_nodes(const void* nodes, const hbg_tree_node* tree, int num_nodes,
                               const int32_t* rows0, const int32_t* rows1, double lr, double* scores,
                               cudaStream_t s);

int sm_count(int device);

// Runs f, mapping exceptions to HBG_* status codes + the thread-local last error.
int guarded_call_impl(void (*fn)(void*), void* arg);
template <typename F>
int guarded_call(F&& f) {
  return guarded_call_impl([](void* p) { (*static_cast<F*>(p))(); }, &f);
}

}  // namespace hbg
