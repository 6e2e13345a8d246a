/*
 * hbg_oracle.h — CPU ORACLE for the hbg feature-histogram path.
 *
 * TEST INFRASTRUCTURE ONLY. This is a plain-C restatement of the reference
 * (histoboost, /root/reference/proj) algorithms on the histogram hot path. It
 * exists to CHECK the CUDA path: only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load it. The product library
 * (paper_1706_08359_b200/libhbg.so) never links or calls it.
 *
 * Parity pinning: every function here is checked against (a) the golden
 * vectors of the reference's own tests (tests/golden/known_answers.json) and
 * (b) the reference itself compiled from /root/reference by oracle/Makefile
 * into oracle/_ref/libhistoboost_ref.so (tests/test_oracle.py).
 */
#ifndef HBG_ORACLE_H
#define HBG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as histoboost::HistogramBin (histogram_set.hpp:17-21). */
typedef struct hbo_bin {
  double grad_sum;
  double hess_sum;
  int64_t count;
} hbo_bin;

/* Same fields as histoboost::SplitInfo (tree.hpp:15-24), minus threshold_value. */
typedef struct hbo_split {
  int32_t feature;
  int32_t threshold_bin;
  double gain;
  double left_grad, left_hess, right_grad, right_hess;
  int64_t left_count, right_count;
  double left_value, right_value;
} hbo_split;

/* std::mt19937_64 (the reference's only RNG engine, random.hpp). */
typedef struct hbo_mt64 {
  uint64_t mt[312];
  int mti;
} hbo_mt64;

void hbo_mt64_seed(hbo_mt64* r, uint64_t seed);
uint64_t hbo_mt64_next(hbo_mt64* r);
double hbo_uniform_double(hbo_mt64* r);                 /* random.hpp:14-17 */
uint64_t hbo_uniform_below(hbo_mt64* r, uint64_t bound); /* random.hpp:19-22 */
double hbo_normal_double(hbo_mt64* r);                  /* random.hpp:24-29 */

/* bench.cpp:17-38 — column-major bins, out[f * rows + i]. */
void hbo_gen_synthetic_bins(int64_t rows, int features, int max_bin, uint64_t seed,
                            uint8_t* out);
/* bench.cpp:69-73 — g = 2u-1 then h = u from mt19937_64(seed ^ 0xdeadbeefcafef00d). */
void hbo_gen_grad_hess(int64_t rows, uint64_t seed, double* g, double* h);
/* bench.cpp:40-57 — returns count (rows >> depth) or -1 on invalid depth.
 * `out` must hold `rows` entries (scratch for the permutation). */
int64_t hbo_leaf_index_sample(int64_t rows, int depth, uint64_t seed, int32_t* out);

/* binning.cpp:123-158 — tuple-major words[t * rows + i]; bits 8 or 4;
 * pad slots carry bin 0. Returns number of tuples, -1 if 4-bit and k > 16. */
int hbo_pack_feature_tuples(const uint8_t* cols, int d, int64_t rows, int bits, int max_bin,
                            uint32_t* words);
/* binning.cpp:160-182 (redistribute_bins) — returns expansion m; writes spread bins. */
int hbo_redistribute_bins(const uint8_t* col, int64_t rows, int bin_capacity, uint8_t* spread,
                          int* original_effective_bins);
/* binning.cpp:184-202 (fold_histogram). */
void hbo_fold_histogram(const hbo_bin* in, int k, int expansion, hbo_bin* out);

/* tree.cpp:11-25 — leaf-aligned g/h plus double totals in index order. */
void hbo_gather_leaf(const int32_t* idx, int64_t n, const double* g, const double* h,
                     double* leaf_g, double* leaf_h, double* grad_total, double* hess_total);

/* histogram.cpp:86-106 (reference_impl<Acc>) — one feature; precision 32 or 64. */
void hbo_build_histogram(const uint8_t* col, int k, const int32_t* idx, int64_t n,
                         const double* leaf_g, const double* leaf_h, int precision, hbo_bin* out);
/* histogram.cpp:159-215 (build_histograms_partitioned, dense features only):
 * 64Ki-row chunks reduced in chunk order — bit-identical to the reference for
 * any worker count. out[f * k + b]. */
void hbo_build_histograms_partitioned(const uint8_t* cols, int d, int64_t rows, int k,
                                      const int32_t* idx, int64_t n, const double* leaf_g,
                                      const double* leaf_h, int precision, hbo_bin* out);

/* tree.cpp:59-64 / :66-74 */
double hbo_optimal_leaf_value(double grad_sum, double hess_sum, double lambda);
double hbo_split_gain(double lg, double lh, double rg, double rh, double lambda);
/* tree.cpp:76-112 — returns 1 and fills *out when a positive-gain threshold exists. */
int hbo_find_best_threshold(const hbo_bin* hist, int k, int feature_id, double grad_total,
                            double hess_total, int64_t count, int64_t min_data_in_leaf,
                            double lambda, hbo_split* out);
/* tree.cpp:163-182 minus the boundary lookup; hists[f * k + b]. */
int hbo_find_best_split(const hbo_bin* hists, int d, int k, double grad_total, double hess_total,
                        int64_t count, int64_t min_data_in_leaf, double lambda, hbo_split* out);
/* tree.cpp:114-128 — stable split; returns left count or -1 on an empty side. */
int64_t hbo_partition_leaf(const int32_t* idx, int64_t n, const uint8_t* col, int threshold_bin,
                           int32_t* left, int32_t* right);

/* tree.cpp:186-261 — best-first growth with the partitioned builder at the
 * given precision. Writes up to num_leaves-1 executed splits to split_log and
 * returns how many; node arrays (2*num_leaves-1 entries) are optional. */
int hbo_grow_tree(const uint8_t* cols, int d, int64_t rows, int k, const double* g,
                  const double* h, int num_leaves, int64_t min_data_in_leaf, double lambda,
                  int precision, hbo_split* split_log, int32_t* node_feature,
                  int32_t* node_threshold_bin, int32_t* node_left, int32_t* node_right,
                  double* node_value, int* num_nodes);

/* losses.cpp:24-26 (loss 0 = squared: g = s - t, h = 1) and :57-60
 * (loss 1 = logistic: p = sigmoid(s), g = p - t, h = max(p(1-p), 1e-16)). */
void hbo_grad_hess(int loss, const double* scores, const double* targets, int64_t n, double* g,
                   double* h);
/* boost_one_iteration (boosting.cpp:26-51): gradients at the cached scores,
 * grow_tree, scores += learning_rate * tree(row) via binned routing. Writes the
 * executed splits (num_leaves-1 capacity) and returns how many. */
int hbo_boost_one_iteration(const uint8_t* cols, int d, int64_t rows, int k, const double* targets,
                            int loss, double learning_rate, int num_leaves, int64_t min_data_in_leaf,
                            double lambda, int precision, double* scores, hbo_split* split_log);

/* histogram.cpp:12-15 */
int hbo_stats_close(double a, double b, double tolerance);

#ifdef __cplusplus
}
#endif

#endif
