/*
 * hbg.h — C ABI of the B200-native feature-histogram path (arXiv 1706.08359 hot path).
 *
 * Plain C types only (no torch / CUDA types in the signatures; streams are
 * passed as `void*` holding a cudaStream_t, NULL = the legacy default stream).
 * Every entry point returns an HBG_* status; on failure hbg_last_error()
 * returns a message (thread-local), mirroring the reference's exceptions.
 *
 * Reference seam being replaced (paths under /root/reference/proj):
 *   HistogramSet build_histograms_partitioned(const BinnedDataset&, const LeafState&,
 *                                             PrecisionMode, int)   include/histoboost/histogram.hpp:133-134
 *   dispatched from build_leaf_histograms                           src/tree.cpp:138-161
 *   selected by enum class HistogramBackend {partitioned, lockstep} include/histoboost/tree.hpp:78
 * INTEGRATION.md shows the `HistogramBackend::cuda` arm a maintainer adds.
 */
#ifndef HBG_H
#define HBG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (error behaviour of the reference, histogram.cpp / tree.cpp) ---- */
#define HBG_OK 0
#define HBG_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument: shape / config (histogram.cpp:27-40,148-154) */
#define HBG_ERR_LOGIC 2            /* std::logic_error: empty split side (tree.cpp:124-126) */
#define HBG_ERR_CUDA 3             /* CUDA runtime failure (no CPU fallback exists) */
#define HBG_ERR_OUT_OF_MEMORY 4
#define HBG_ERR_NCCL 5

/* g/h addressing for the device builder (hbg_build_histograms_device). */
#define HBG_GH_LEAF_ALIGNED 0 /* g[i] belongs to leaf position i (LeafState::gradients, leaf.hpp:15-16) */
#define HBG_GH_ROW_INDEXED 1  /* g[indices[i]] — gather fused into the histogram kernel */

/* Accumulation precision: the values of histoboost::PrecisionMode
 * (histogram_set.hpp:11, enum class PrecisionMode { bits32, bits64 }).
 * BITS32: g/h cast to fp32 per element (histogram.cpp:97-98), fp32 per-warp
 *         sums reduced in fp64 — the fast path (stats_tolerance 1e-4).
 * BITS64: fp64 g/h in HBM, fp64 shared-memory cells and fp64 partials
 *         (reference_impl<double>, histogram.cpp:131-145) — meets the
 *         reference's stats_tolerance(bits64) = 1e-12. */
#define HBG_PRECISION_BITS32 0
#define HBG_PRECISION_BITS64 1

/* One histogram bin; identical layout to histoboost::HistogramBin (histogram_set.hpp:17-21). */
typedef struct hbg_bin {
  double grad_sum;
  double hess_sum;
  int64_t count;
} hbg_bin;

/* Best split of a leaf; the fields of histoboost::SplitInfo (tree.hpp:15-24) except
 * threshold_value, which the caller maps through its BinBoundaries (tree.cpp:174-180). */
typedef struct hbg_split {
  int32_t feature; /* -1: no positive-gain split (std::nullopt) */
  int32_t threshold_bin;
  double gain;
  double left_grad, left_hess, right_grad, right_hess;
  int64_t left_count, right_count;
  double left_value, right_value;
} hbg_split;

/* Device-resident packed dataset (subsystem 1). */
typedef struct hbg_dataset hbg_dataset;

/* How the dataset sits in HBM: row-major, one row = num_groups slices of
 * slice_bytes; a slice holds 32 features (8-bit: 4 per 32-bit word; 4-bit:
 * 8 per word), at the bit positions of pack_feature_tuples (binning.cpp:123-158). */
typedef struct hbg_layout {
  int64_t num_rows;
  int32_t num_features;
  int32_t max_bin;           /* k: 16, 64 or 256 (any 2..256 accepted) */
  int32_t bits_per_bin;      /* 4 iff max_bin <= 16 (prepare_packed, binning.cpp:230) else 8 */
  int32_t features_per_word; /* 8 or 4 */
  int32_t words_per_row;     /* ceil(num_features / features_per_word) */
  int32_t row_stride_bytes;  /* slice_bytes: rows of one slice group are contiguous */
  int32_t slice_bytes;       /* 16 (4-bit) or 32 (8-bit) */
  int32_t num_groups;        /* ceil(num_features / 32) */
  int32_t device;
  int64_t group_stride_bytes; /* slice group g of row r at packed + g*group_stride + r*row_stride
                                 (group-planar: a warp's 32 consecutive rows of one group are one
                                 contiguous 1 KB, whatever the number of groups) */
} hbg_layout;

const char* hbg_last_error(void);
int32_t hbg_version(void);

/* ---- dataset (rows a1 -> a2 of SURVEY §8) ----
 * columns[f] points at num_rows uint8 bins of feature f (BinnedColumn::bins,
 * dataset.hpp:21-26); every bin must be < max_bin (checked on device).
 * Multi-GPU row shards pass columns[f] + row_begin and the shard's row count. */
int hbg_dataset_create(const uint8_t* const* columns, int32_t num_features, int64_t num_rows,
                       int32_t max_bin, int32_t device, hbg_dataset** out);
int hbg_dataset_destroy(hbg_dataset* ds);
int hbg_dataset_layout(const hbg_dataset* ds, hbg_layout* out);
/* Copies the packed rows to host: num_rows * words_per_row uint32 (row-major, pad words dropped). */
int hbg_dataset_packed_words(const hbg_dataset* ds, uint32_t* host_words);

/* ---- histogram construction (rows a5-a7) ----
 * Host drop-in for build_histograms_partitioned: indices/gradients/hessians
 * are the LeafState arrays (leaf-aligned doubles, leaf.hpp:13-21); `out`
 * receives num_features * max_bin bins, feature-major (HistogramSet order).
 * Synchronous. count == 0 gives an all-zero histogram. The arrays go up in
 * chunks, each either converted to fp32 by a library thread pool into a
 * pinned stage and copied (8 B/row), or — for pinned host arrays
 * (cudaHostAlloc/cudaHostRegister), a share of the chunks — copied as fp64
 * (16 B/row) and converted on the device; row ids travel only for chunks that
 * are not one contiguous range. The same floats and sums on every route:
 * bit-identical results. A row id outside [0, num_rows) returns
 * HBG_ERR_INVALID_ARGUMENT (checked while the ids are staged). */
int hbg_build_histograms(hbg_dataset* ds, const int32_t* indices, int64_t count,
                         const double* gradients, const double* hessians, hbg_bin* out);
/* The same call with the reference's PrecisionMode argument
 * (build_histograms_partitioned(data, leaf, precision), histogram.hpp:133):
 * HBG_PRECISION_BITS32 is hbg_build_histograms; HBG_PRECISION_BITS64 uploads
 * the fp64 LeafState arrays as they are (16 B/row; pageable ones through the
 * library's pinned stage) and accumulates in fp64. */
int hbg_build_histograms_ex(hbg_dataset* ds, const int32_t* indices, int64_t count,
                            const double* gradients, const double* hessians, int32_t precision,
                            hbg_bin* out);

/* Development aid: with HBG_HIST_PROFILE set in the environment, every
 * histogram launch records %globaltimer stamps (ns) of its CTA 0 — start,
 * shared memory cleared, rows done, partials written, grid barrier passed,
 * reduced; [6] the reduction's first loads, [7] unused — and this copies the
 * last launch's eight to host `out`. */
int hbg_debug_hist_stamps(hbg_dataset* ds, unsigned long long* out);

/* Development aid: bytes the last host histogram call on `ds`
 * (hbg_build_histograms, _ex) copied host->device and device->host — each staged
 * chunk goes as fp32 (8 B/row) or fp64 (16 B/row), row ids only for chunks
 * that are not one contiguous range — written to out[0] and out[1]. */
int hbg_debug_host_copy_bytes(hbg_dataset* ds, int64_t* out);

/* Device builder (the performance path). d_indices may be NULL for the
 * identity leaf [0, count) (the root). d_grad/d_hess are fp32, addressed per
 * gh_mode. d_hist receives the device histogram: SoA fp64
 * [3][num_features][max_bin] = grad, hess, count (counts exact in fp64).
 * Asynchronous on `stream`; not re-entrant per handle. */
int hbg_build_histograms_device(hbg_dataset* ds, const int32_t* d_indices, int64_t count,
                                const float* d_grad, const float* d_hess, int32_t gh_mode,
                                double* d_hist, void* stream);

/* bits64 device builder: d_grad/d_hess are fp64 (addressed per gh_mode),
 * accumulated in fp64 shared-memory cells and reduced in fp64. */
int hbg_build_histograms_device_f64(hbg_dataset* ds, const int32_t* d_indices, int64_t count,
                                    const double* d_grad, const double* d_hess, int32_t gh_mode,
                                    double* d_hist, void* stream);

/* Device SoA histogram -> hbg_bin[num_features * max_bin] (device pointer). */
int hbg_hist_to_bins_device(const double* d_hist, int32_t num_features, int32_t max_bin,
                            hbg_bin* d_bins, void* stream);

/* ---- histogram subtraction (row a10): sibling = parent - child, elementwise over
 * n_values = 3 * num_features * max_bin doubles (counts stay exact). */
int hbg_subtract_device(const double* d_parent, const double* d_child, double* d_sibling,
                        int64_t n_values, void* stream);

/* ---- leaf gather (row a4): leaf_g[i] = g[idx[i]], leaf_h[i] = h[idx[i]] in fp32,
 * d_totals[0..1] = fp64 sums in a fixed order (grad_total, hess_total). */
int hbg_gather_leaf_device(const int32_t* d_indices, int64_t count, const float* d_grad,
                           const float* d_hess, float* d_leaf_grad, float* d_leaf_hess,
                           double* d_totals, void* stream);

/* gather_leaf_statistics (tree.cpp:11-25) for host callers: leaf_g[i] =
 * g[indices[i]], leaf_h[i] = h[indices[i]] (fp64, host arrays of count) and
 * totals[0..1] = fp64 grad/hess totals in a fixed order, computed on `device`
 * (g/h: host fp64 arrays of num_rows; every index must be < num_rows). */
int hbg_gather_leaf_statistics(const int32_t* indices, int64_t count, const double* gradients,
                               const double* hessians, int64_t num_rows, double* leaf_grad,
                               double* leaf_hess, double* totals, int32_t device);

/* ---- best-split scan (row a11): find_best_split (tree.cpp:163-182) over a device
 * SoA histogram, fp64, the reference's tie rules (smallest bin, then lowest
 * feature). Parent totals come from the caller (LeafState totals, tree.cpp:167).
 * d_out: device hbg_split; feature = -1 when no split. */
int hbg_best_split_device(const double* d_hist, int32_t num_features, int32_t max_bin,
                          double grad_total, double hess_total, int64_t count,
                          int64_t min_data_in_leaf, double lambda, hbg_split* d_out, void* stream);
/* Same, totals read from device memory (d_totals = {grad, hess}, d_count int64). */
int hbg_best_split_device_totals(const double* d_hist, int32_t num_features, int32_t max_bin,
                                 const double* d_totals, const int64_t* d_count,
                                 int64_t min_data_in_leaf, double lambda, hbg_split* d_out,
                                 void* stream);
/* Host convenience: hists are host hbg_bin[num_features * max_bin]; runs the same
 * device scan and returns 1 if a split was found (0 otherwise) in *found. */
int hbg_find_best_split(const hbg_bin* hists, int32_t num_features, int32_t max_bin,
                        double grad_total, double hess_total, int64_t count,
                        int64_t min_data_in_leaf, double lambda, hbg_split* out, int32_t* found);

/* ---- device-resident tree growth ----
 * grow_tree (tree.cpp:186-261) with the partitioned backend's semantics:
 * best-first over the pool of open leaves (strict >, the oldest leaf wins
 * ties), children numbered left then right, leaf values from the children's
 * regathered totals, both children's best splits computed while
 * leaves < num_leaves. On the device: stable partition_leaf (tree.cpp:114-128)
 * of a leaf's contiguous row range, fp64 child totals in a fixed order, the
 * histogram of the SMALLER child only and the larger one by subtraction. */
typedef struct hbg_grow_params {
  int32_t num_leaves;       /* GrowParams::num_leaves (tree.hpp:81) */
  int32_t precision;        /* GrowParams::precision (tree.hpp:84): HBG_PRECISION_BITS32 grows
                               with fp32 g/h in the persistent kernel; HBG_PRECISION_BITS64
                               grows with fp64 g/h and fp64 histograms at every leaf (host-
                               driven loop; hbg_grow_tree_host / hbg_grow_tree_f64 only) */
  int64_t min_data_in_leaf; /* GrowParams::min_data_in_leaf */
  double lambda;            /* GrowParams::lambda */
} hbg_grow_params;

/* TreeNode (tree.hpp:26-35) minus threshold_value (mapped by the caller). */
typedef struct hbg_tree_node {
  int32_t feature;       /* -1 on leaves */
  int32_t threshold_bin; /* -1 on leaves */
  int32_t left, right;   /* -1 on leaves */
  double value;
} hbg_tree_node;

/* d_grad/d_hess: fp32 per-row gradients/hessians (device, num_rows each).
 * split_log: host, num_leaves-1 entries (SplitInfo order of execution);
 * nodes: host, 2*num_leaves-1 entries. Synchronous on `stream`.
 * Not re-entrant per handle. The whole tree runs in one persistent kernel:
 * one split per grid barrier, or (8-bit data, <= 4096 feature x bin cells,
 * <= 256 leaves) several speculative expansions per barrier with the
 * reference's pick order replayed — bit-identical trees. Environment:
 * HBG_GROW=legacy | wave | host forces the one-split kernel, the wave kernel
 * (where it fits) or the per-split host loop. */
int hbg_grow_tree(hbg_dataset* ds, const float* d_grad, const float* d_hess,
                  const hbg_grow_params* params, hbg_split* split_log, int32_t* num_splits,
                  hbg_tree_node* nodes, int32_t* num_nodes, void* stream);

/* bits64 tree on fp64 device gradients/hessians (params->precision must be
 * HBG_PRECISION_BITS64). */
int hbg_grow_tree_f64(hbg_dataset* ds, const double* d_grad, const double* d_hess,
                      const hbg_grow_params* params, hbg_split* split_log, int32_t* num_splits,
                      hbg_tree_node* nodes, int32_t* num_nodes, void* stream);

/* Host-pointer drop-in for grow_tree (tree.cpp:186-261): fp64 per-row
 * gradients/hessians in host memory (the reference's std::span<const double>
 * arguments). params->precision BITS32: cast to fp32 (the bits32 per-element
 * cast, histogram.cpp:97-98; by the staging pool, or on the device for a
 * share of the chunks of pinned arrays), then grown as hbg_grow_tree; BITS64: uploaded as
 * fp64 and grown as hbg_grow_tree_f64. split_log: host,
 * num_leaves-1 entries; nodes: host, 2*num_leaves-1 entries. Synchronous. */
int hbg_grow_tree_host(hbg_dataset* ds, const double* gradients, const double* hessians,
                       const hbg_grow_params* params, hbg_split* split_log, int32_t* num_splits,
                       hbg_tree_node* nodes, int32_t* num_nodes);

/* ---- row-sharded growth ----
 * One process (or thread) per GPU; each rank's dataset and d_grad/d_hess hold
 * its own rows (hbg_dataset_create on columns + row_begin). The hook sums
 * n doubles in place across ranks on `stream` (the leaf histograms, SoA fp64
 * with exact counts, and leaf totals), so every rank scans identical
 * histograms and grows the identical tree. Returns HBG_OK or an error status.
 * hbg_comm_allreduce (below) is the NCCL implementation. */
typedef int (*hbg_allreduce_fn)(double* d_buf, int64_t n_values, void* stream, void* ctx);
int hbg_grow_tree_sharded(hbg_dataset* ds, const float* d_grad, const float* d_hess,
                          const hbg_grow_params* params, hbg_allreduce_fn allreduce, void* ctx,
                          hbg_split* split_log, int32_t* num_splits, hbg_tree_node* nodes,
                          int32_t* num_nodes, void* stream);

/* ---- row-sharded growth inside the persistent kernel ----
 * Each rank owns an exchange area on its GPU; every rank maps every rank's
 * area (CUDA IPC across processes: hbg_peer_handle + hbg_peer_open; same
 * process: hbg_peer_attach). hbg_grow_tree_peer then grows the tree with the
 * per-split exchange of the smaller child's histogram chunks and the
 * partition totals done INSIDE the one-kernel grower over NVLink peer memory
 * (every rank sums all ranks' contributions in rank order: identical
 * histograms, identical trees on every rank). d_grad/d_hess/dataset: this
 * rank's rows. All ranks call it for the same tree with the same params.
 * ctas: CTAs per rank (0 = one per SM; a partial grid lets several ranks
 * share one GPU, as the tests do). Trees grown through the peer must not
 * exceed params->num_leaves of hbg_peer_create (workspace reserved there). */
/* The dataset's own CUDA stream (created with the handle; the host drop-ins
 * run on it). Ranks sharing one GPU should each grow on their dataset's
 * stream: consecutively created streams land on distinct hardware queues
 * (with CUDA_DEVICE_MAX_CONNECTIONS >= the rank count), so the ranks'
 * persistent grids run concurrently. */
void* hbg_dataset_stream(const hbg_dataset* ds);

#define HBG_PEER_HANDLE_BYTES 64
typedef struct hbg_peer hbg_peer;
/* Every in-kernel wait on another rank (exchange flags, grid barriers) is
 * bounded by HBG_PEER_TIMEOUT_MS (environment, default 60000): ranks may reach
 * a peer call that far apart; an expired wait is an HBG_ERR_CUDA status with
 * hbg_last_error() naming it, never a hang. */
int hbg_peer_create(hbg_dataset* ds, int32_t nranks, int32_t rank, int32_t ctas,
                    const hbg_grow_params* params /* the largest tree: its workspace is reserved */,
                    hbg_peer** out);
int hbg_peer_handle(hbg_peer* p, uint8_t* out /* HBG_PEER_HANDLE_BYTES */);
int hbg_peer_open(hbg_peer* p, int32_t peer_rank, const uint8_t* handle);
int hbg_peer_attach(hbg_peer* p, int32_t peer_rank, const hbg_peer* q);
int hbg_peer_destroy(hbg_peer* p);
/* Row-sharded histogram of one leaf (this rank's rows, as
 * hbg_build_histograms_device) with the cross-rank sum FUSED into the
 * histogram's reduction kernel over peer memory: every rank's d_hist receives
 * the bit-identical global histogram (rank-order sum), no separate collective.
 * Every rank calls it for the same leaf (a rank without rows of it too).
 * Asynchronous on `stream`; hbg_peer_check (device-wide synchronisation)
 * reports a rank that never published. */
int hbg_build_histograms_peer(hbg_dataset* ds, const int32_t* d_indices, int64_t count, const float* d_grad,
                              const float* d_hess, int32_t gh_mode, double* d_hist, hbg_peer* peer, void* stream);
int hbg_peer_check(hbg_peer* p);
/* boost_one_iteration (as hbg_boost_one_iteration) with the tree grown through
 * hbg_grow_tree_peer: this rank's rows' targets/scores; every rank calls it. */
int hbg_boost_one_iteration_peer(hbg_dataset* ds, const double* d_targets, double* d_scores, int32_t loss,
                                 double learning_rate, const hbg_grow_params* params, hbg_peer* peer,
                                 hbg_split* split_log, int32_t* num_splits, hbg_tree_node* nodes, int32_t* num_nodes,
                                 void* stream);
int hbg_grow_tree_peer(hbg_dataset* ds, const float* d_grad, const float* d_hess, const hbg_grow_params* params,
                       hbg_peer* peer, hbg_split* split_log, int32_t* num_splits, hbg_tree_node* nodes,
                       int32_t* num_nodes, void* stream);

/* NCCL communicator implementing the hook: one process per GPU, the 128-byte
 * unique id produced by rank 0 is shared out of band. Pass the hbg_comm* as
 * `ctx` with hbg_comm_allreduce as `allreduce`. */
#define HBG_COMM_ID_BYTES 128
typedef struct hbg_comm hbg_comm;
int hbg_comm_get_unique_id(uint8_t* out /* HBG_COMM_ID_BYTES */);
int hbg_comm_init(hbg_comm** out, int32_t nranks, int32_t rank, const uint8_t* unique_id,
                  int32_t device);
int hbg_comm_destroy(hbg_comm* comm);
int hbg_comm_allreduce(double* d_buf, int64_t n_values, void* stream, void* ctx);

/* ---- one boosting iteration on the device ----
 * boost_one_iteration (boosting.cpp:26-51): g,h of the loss at the cached
 * scores (losses.cpp:24-26 squared, :57-60 logistic; fp64 math, fp32
 * storage), grow_tree as hbg_grow_tree, then d_scores[row] +=
 * learning_rate * value(row's leaf). d_targets/d_scores: fp64 device arrays of
 * num_rows. allreduce may be NULL (single rank) or the row-sharded hook. */
#define HBG_LOSS_SQUARED 0
#define HBG_LOSS_LOGISTIC 1
int hbg_boost_one_iteration(hbg_dataset* ds, const double* d_targets, double* d_scores, int32_t loss,
                            double learning_rate, const hbg_grow_params* params, hbg_allreduce_fn allreduce,
                            void* ctx, hbg_split* split_log, int32_t* num_splits, hbg_tree_node* nodes,
                            int32_t* num_nodes, void* stream);

/* reduce_private_histograms (histogram.cpp:147-157) on the device: d_out =
 * sum of nparts device buffers of n_values doubles, added in part order. */
int hbg_reduce_histograms_device(const double* const* d_parts, int32_t nparts, int64_t n_values,
                                 double* d_out, void* stream);

/* ---- measurement hooks (bench.py roofline) ----
 * When enabled, the handle records a CUDA event pair around every histogram
 * kernel launch (in-stream, no host sync). hbg_dataset_kernel_time waits for
 * the recorded launches, returns their summed duration and count, and clears
 * the record. */
int hbg_dataset_set_profiling(hbg_dataset* ds, int32_t enabled);
int hbg_dataset_kernel_time(hbg_dataset* ds, double* total_ms, int64_t* launches);

/* ---- stream helpers for callers without a CUDA runtime binding ---- */
int hbg_stream_synchronize(void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HBG_H */
