// ref_shim.cpp — TEST INFRASTRUCTURE: a C ABI over the UNMODIFIED reference
// (histoboost, /root/reference/proj), compiled together with the reference's
// own source files by oracle/Makefile into oracle/_ref/libhistoboost_ref.so.
//
// Nothing from the reference is copied here; this file only calls its public
// API. It serves two purposes:
//   * pins the C oracle (oracle/hbg_oracle.c) against the real reference
//     (tests/test_oracle.py) and generates golden fixtures (tests/golden/);
//   * is bench.py's CPU reference arm (`--impl reference`, cpu_baseline
//     kind "reference"): build_histograms_partitioned / grow_tree timed on all
//     host cores.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <vector>

#include "histoboost/bench.hpp"
#include "histoboost/boosting.hpp"
#include "histoboost/binning.hpp"
#include "histoboost/histogram.hpp"
#include "histoboost/parallel.hpp"
#include "histoboost/tree.hpp"

using namespace histoboost;

namespace {

struct SplitOut {  // == hbo_split (oracle/hbg_oracle.h)
  int32_t feature;
  int32_t threshold_bin;
  double gain;
  double left_grad, left_hess, right_grad, right_hess;
  int64_t left_count, right_count;
  double left_value, right_value;
};

void to_out(const SplitInfo& s, SplitOut* o) {
  o->feature = s.feature;
  o->threshold_bin = s.threshold_bin;
  o->gain = s.gain;
  o->left_grad = s.left_grad;
  o->left_hess = s.left_hess;
  o->right_grad = s.right_grad;
  o->right_hess = s.right_hess;
  o->left_count = s.left_count;
  o->right_count = s.right_count;
  o->left_value = s.left_value;
  o->right_value = s.right_value;
}

BinnedDataset make_dataset(const uint8_t* cols, int d, int64_t rows, int k) {
  BinnedDataset data;
  data.num_rows = rows;
  data.max_bin = k;
  data.columns.resize(static_cast<std::size_t>(d));
  data.boundaries.resize(static_cast<std::size_t>(d));
  for (int f = 0; f < d; ++f) {
    auto& c = data.columns[static_cast<std::size_t>(f)];
    c.bin_capacity = k;
    c.bins.assign(cols + static_cast<int64_t>(f) * rows, cols + static_cast<int64_t>(f + 1) * rows);
    for (int b = 1; b < k - 1; ++b) {
      data.boundaries[static_cast<std::size_t>(f)].upper_bounds.push_back(b + 0.5);
    }
    data.dense_features.push_back(f);
  }
  return data;
}

void copy_set(const HistogramSet& set, int k, void* out) {
  auto* o = static_cast<HistogramBin*>(out);
  for (std::size_t f = 0; f < set.size(); ++f) {
    std::memcpy(o + f * static_cast<std::size_t>(k), set[f].bins.data(),
                sizeof(HistogramBin) * static_cast<std::size_t>(k));
  }
}

thread_local char g_err[512];

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err; }

int ref_gen_synthetic_bins(int64_t rows, int d, int k, uint64_t seed, uint8_t* out) {
  BinnedDataset data = gen_synthetic_bins(rows, d, k, seed);
  for (int f = 0; f < d; ++f) {
    std::memcpy(out + static_cast<int64_t>(f) * rows, data.columns[static_cast<std::size_t>(f)].bins.data(),
                static_cast<std::size_t>(rows));
  }
  return 0;
}

int64_t ref_leaf_index_sample(int64_t rows, int depth, uint64_t seed, int32_t* out) {
  try {
    auto v = leaf_index_sample(rows, depth, seed);
    std::memcpy(out, v.data(), v.size() * sizeof(int32_t));
    return static_cast<int64_t>(v.size());
  } catch (const std::exception& e) {
    std::snprintf(g_err, sizeof g_err, "%s", e.what());
    return -1;
  }
}

int ref_pack_feature_tuples(const uint8_t* cols, int d, int64_t rows, int bits, int k,
                            uint32_t* words) {
  std::vector<BinnedColumn> columns(static_cast<std::size_t>(d));
  std::vector<int> ids(static_cast<std::size_t>(d));
  for (int f = 0; f < d; ++f) {
    columns[static_cast<std::size_t>(f)].bin_capacity = k;
    columns[static_cast<std::size_t>(f)].bins.assign(cols + static_cast<int64_t>(f) * rows,
                                                     cols + static_cast<int64_t>(f + 1) * rows);
    ids[static_cast<std::size_t>(f)] = f;
  }
  try {
    auto t = pack_feature_tuples(columns, ids, bits == 4 ? BinWidth::bits4 : BinWidth::bits8);
    for (std::size_t i = 0; i < t.size(); ++i) {
      std::memcpy(words + i * static_cast<std::size_t>(rows), t[i].words.data(),
                  static_cast<std::size_t>(rows) * sizeof(uint32_t));
    }
    return static_cast<int>(t.size());
  } catch (const std::exception& e) {
    std::snprintf(g_err, sizeof g_err, "%s", e.what());
    return -1;
  }
}

int ref_redistribute_bins(const uint8_t* col, int64_t rows, int k, uint8_t* spread, int* orig) {
  BinnedColumn c;
  c.bin_capacity = k;
  c.bins.assign(col, col + rows);
  auto [s, info] = redistribute_bins(c);
  std::memcpy(spread, s.bins.data(), static_cast<std::size_t>(rows));
  if (orig) *orig = info.original_effective_bins;
  return static_cast<int>(info.expansion);
}

// build_histograms_partitioned on leaf-aligned doubles (LeafState semantics).
int ref_build_histograms_partitioned(const uint8_t* cols, int d, int64_t rows, int k,
                                     const int32_t* idx, int64_t n, const double* leaf_g,
                                     const double* leaf_h, int precision, int workers,
                                     void* out) {
  BinnedDataset data = make_dataset(cols, d, rows, k);
  LeafState leaf;
  leaf.indices.assign(idx, idx + n);
  leaf.gradients.assign(leaf_g, leaf_g + n);
  leaf.hessians.assign(leaf_h, leaf_h + n);
  for (double v : leaf.gradients) leaf.grad_total += v;
  for (double v : leaf.hessians) leaf.hess_total += v;
  auto set = build_histograms_partitioned(
      data, leaf, precision == 64 ? PrecisionMode::bits64 : PrecisionMode::bits32, workers);
  copy_set(set, k, out);
  return 0;
}

int ref_find_best_threshold(const void* hist, int k, int feature_id, double gt, double ht,
                            int64_t count, int64_t min_data, double lambda, void* out) {
  HistogramEntry e;
  e.feature_id = feature_id;
  e.bins.assign(static_cast<const HistogramBin*>(hist), static_cast<const HistogramBin*>(hist) + k);
  auto best = find_best_threshold(e, LeafTotals{gt, ht, count}, min_data, lambda);
  if (!best) return 0;
  to_out(*best, static_cast<SplitOut*>(out));
  return 1;
}

// ---- persistent handles for timing the reference on the bench inputs ----
void* ref_dataset_new(const uint8_t* cols, int d, int64_t rows, int k) {
  return new BinnedDataset(make_dataset(cols, d, rows, k));
}
void ref_dataset_free(void* ds) { delete static_cast<BinnedDataset*>(ds); }

// gather_leaf_statistics (tree.cpp:11-25) from global double g/h.
void* ref_leaf_new(const int32_t* idx, int64_t n, const double* g, const double* h, int64_t rows) {
  std::vector<row_index_t> v(idx, idx + n);
  return new LeafState(gather_leaf_statistics(std::move(v), std::span<const double>(g, rows),
                                              std::span<const double>(h, rows)));
}
void ref_leaf_free(void* leaf) { delete static_cast<LeafState*>(leaf); }

// Times one build_histograms_partitioned call; returns seconds (out may be NULL).
double ref_build_timed(void* ds, void* leaf, int precision, int workers, void* out) {
  auto& data = *static_cast<BinnedDataset*>(ds);
  auto t0 = std::chrono::steady_clock::now();
  auto set = build_histograms_partitioned(
      data, *static_cast<LeafState*>(leaf),
      precision == 64 ? PrecisionMode::bits64 : PrecisionMode::bits32, workers);
  auto t1 = std::chrono::steady_clock::now();
  if (out) copy_set(set, data.max_bin, out);
  return std::chrono::duration<double>(t1 - t0).count();
}

// grow_tree (tree.cpp:186) with the partitioned backend; returns seconds and
// writes the split log (up to num_leaves - 1 entries) and its length.
double ref_grow_tree_timed(void* ds, const double* g, const double* h, int num_leaves,
                           int64_t min_data, double lambda, int precision, void* split_log,
                           int* logged) {
  auto& data = *static_cast<BinnedDataset*>(ds);
  GrowParams p;
  p.num_leaves = num_leaves;
  p.min_data_in_leaf = min_data;
  p.lambda = lambda;
  p.precision = precision == 64 ? PrecisionMode::bits64 : PrecisionMode::bits32;
  std::vector<SplitInfo> log;
  auto t0 = std::chrono::steady_clock::now();
  Tree tree = grow_tree(data, std::span<const double>(g, static_cast<std::size_t>(data.num_rows)),
                        std::span<const double>(h, static_cast<std::size_t>(data.num_rows)), p, &log);
  auto t1 = std::chrono::steady_clock::now();
  if (split_log) {
    for (std::size_t i = 0; i < log.size(); ++i) to_out(log[i], static_cast<SplitOut*>(split_log) + i);
  }
  if (logged) *logged = static_cast<int>(log.size());
  return std::chrono::duration<double>(t1 - t0).count();
}

int ref_worker_count() { return worker_count(); }

// boost_one_iteration (boosting.cpp:26-51) on the reference: scores in/out,
// returns seconds; writes the tree's split log.
double ref_boost_one_iteration(void* ds, const double* targets, int loss, double learning_rate,
                               int num_leaves, int64_t min_data, double lambda, int precision,
                               double* scores, void* split_log, int* logged) {
  auto& data = *static_cast<BinnedDataset*>(ds);
  Model model;
  model.loss = loss == 0 ? LossKind::squared : LossKind::logistic;
  model.learning_rate = learning_rate;
  BoosterParams p;
  p.learning_rate = learning_rate;
  p.num_leaves = num_leaves;
  p.min_data_in_leaf = min_data;
  p.lambda = lambda;
  p.precision = precision == 64 ? PrecisionMode::bits64 : PrecisionMode::bits32;
  std::vector<double> sc(scores, scores + data.num_rows);
  auto t0 = std::chrono::steady_clock::now();
  boost_one_iteration(model, data, std::span<const double>(targets, static_cast<std::size_t>(data.num_rows)),
                      p, sc);
  auto t1 = std::chrono::steady_clock::now();
  std::copy(sc.begin(), sc.end(), scores);
  (void)split_log;
  if (logged) *logged = model.trees.back().num_leaves() - 1;
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
