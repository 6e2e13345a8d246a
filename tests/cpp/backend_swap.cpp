// backend_swap.cpp — TEST: the reference's own types and predicates against the
// hbg drop-in (include/hbg_histoboost.hpp). The C++ analogue of
// test_tree.cpp:264-299 ("the lock-step backend grows the same tree as the
// partitioned one") for a `cuda` backend: histograms from
// build_histograms_cuda(precision) vs build_histograms_partitioned(bits64)
// under the reference's histograms_equivalent at stats_tolerance(precision) —
// 1e-4 for bits32 (the bar the reference applies to its own fp32 path,
// acceptance.cpp:204-223), 1e-12 for bits64 — with exact counts, the max
// deviation printed, and the same find_best_threshold winner per leaf; the
// same on a bin_dataset(sparse_threshold = 0.8) dataset whose sparse features
// the reference builds on its pair path (sparse.cpp); and grow_tree_cuda vs
// grow_tree under both precisions.
//
// Built here by oracle/Makefile against /root/reference (headers + objects)
// into oracle/_ref/backend_swap, which travels to the GPU box; run by
// tests/test_gpu_backend_swap.py.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <optional>
#include <random>

#include "hbg_histoboost.hpp"
#include "histoboost/bench.hpp"
#include "histoboost/binning.hpp"
#include "histoboost/random.hpp"

using namespace histoboost;

namespace {

// histograms_equivalent at the tolerance of the precision asked for, feature
// by feature, with the worst relative deviation printed
bool compare_sets(const HistogramSet& got, const HistogramSet& want, PrecisionMode pm, int& failures, int& checks,
                  const char* tag) {
  bool ok = got.size() == want.size();
  double worst = 0.0;
  for (std::size_t f = 0; ok && f < want.size(); ++f) {
    ok = got[f].feature_id == want[f].feature_id && got[f].precision == pm &&
         histograms_equivalent(got[f], want[f], stats_tolerance(pm));
    for (std::size_t b = 0; ok && b < want[f].bins.size(); ++b) {
      for (auto [x, y] : {std::pair{got[f].bins[b].grad_sum, want[f].bins[b].grad_sum},
                          std::pair{got[f].bins[b].hess_sum, want[f].bins[b].hess_sum}}) {
        double scale = std::max({1.0, std::fabs(x), std::fabs(y)});
        worst = std::max(worst, std::fabs(x - y) / scale);
      }
    }
  }
  ++checks;
  if (!ok) ++failures;
  std::printf("[%s] %shistograms %s vs reference bits64 at stats_tolerance(%s)=%.0e (max rel dev %.2e)\n",
              ok ? "PASS" : "FAIL", tag, precision_name(pm), precision_name(pm), stats_tolerance(pm), worst);
  return ok;
}

// the same find_best_threshold winner over all features
void compare_splits(const BinnedDataset& data, const LeafState& leaf, const HistogramSet& got,
                    const HistogramSet& want, int& failures, int& checks) {
  LeafTotals tot{leaf.grad_total, leaf.hess_total, leaf.count()};
  std::optional<SplitInfo> bw, bg;
  for (int f = 0; f < data.num_features(); ++f) {
    auto cw = find_best_threshold(want[static_cast<std::size_t>(f)], tot, 1, 0.0);
    auto cg = find_best_threshold(got[static_cast<std::size_t>(f)], tot, 1, 0.0);
    if (cw && (!bw || cw->gain > bw->gain)) bw = cw;
    if (cg && (!bg || cg->gain > bg->gain)) bg = cg;
  }
  const bool ok = bw.has_value() == bg.has_value() &&
                  (!bw || (bw->feature == bg->feature && bw->threshold_bin == bg->threshold_bin));
  ++checks;
  if (!ok) ++failures;
  std::printf("[%s]   best split %s (%d,%d)\n", ok ? "PASS" : "FAIL", ok ? "same" : "DIFF", bw ? bw->feature : -1,
              bw ? bw->threshold_bin : -1);
}

// grow_tree_cuda vs grow_tree(bits64) on inputs without near-ties: the same
// split sequence, node numbering and thresholds; leaf values within 1e-7
// relative under bits32 (the device keeps the per-row g/h as fp32 — the cast
// of histogram.cpp:97-98 — so its fp64 totals sum the rounded values: ~1e-9
// measured) and 1e-12 under bits64 (fp64 throughout; test_tree.cpp:264-299
// allows 1e-10 between the reference's own backends)
void compare_trees(const Tree& want, const Tree& got, const std::vector<SplitInfo>& want_log,
                   const std::vector<SplitInfo>& got_log, PrecisionMode pm, int& failures, int& checks,
                   const char* what) {
  const double tol = pm == PrecisionMode::bits64 ? 1e-12 : 1e-7;
  bool ok = want_log.size() == got_log.size() && want.nodes().size() == got.nodes().size();
  double worst = 0.0;
  for (std::size_t i = 0; ok && i < want_log.size(); ++i) {
    ok = want_log[i].feature == got_log[i].feature && want_log[i].threshold_bin == got_log[i].threshold_bin &&
         want_log[i].left_count == got_log[i].left_count && want_log[i].threshold_value == got_log[i].threshold_value;
  }
  for (std::size_t i = 0; ok && i < want.nodes().size(); ++i) {
    const TreeNode &a = want.nodes()[i], &b = got.nodes()[i];
    ok = a.feature == b.feature && a.threshold_bin == b.threshold_bin && a.left == b.left && a.right == b.right;
    const double dev_ = std::fabs(a.value - b.value) / std::max(1.0, std::fabs(a.value));
    worst = std::max(worst, dev_);
    ok = ok && dev_ <= tol;
  }
  ++checks;
  if (!ok) ++failures;
  std::printf("[%s] grow_tree_cuda(%s) %s: %zu splits %s (max value dev %.1e, tol %.0e)\n", ok ? "PASS" : "FAIL",
              precision_name(pm), what, want_log.size(), ok ? "identical" : "DIFFER", worst, tol);
}

}  // namespace

int main() {
  int failures = 0, checks = 0;
  std::mt19937_64 rng(2024);
  const int shapes[][3] = {{200000, 28, 64}, {150000, 28, 16}, {40000, 37, 256}, {60000, 70, 64}, {5000, 3, 100}};
  for (const auto& s : shapes) {
    BinnedDataset data = gen_synthetic_bins(s[0], s[1], s[2], 7 + s[1]);
    std::vector<double> g(static_cast<std::size_t>(s[0])), h(static_cast<std::size_t>(s[0]));
    for (auto& v : g) v = normal_double(rng);
    for (auto& v : h) v = 0.1 + uniform_double(rng);
    hbg::histoboost_backend::DeviceDataset dev(data);
    for (int depth : {0, 1, 4, 9}) {
      auto idx = leaf_index_sample(s[0], depth, 99 + depth);
      LeafState leaf = gather_leaf_statistics(std::move(idx), g, h);
      HistogramSet want = build_histograms_partitioned(data, leaf, PrecisionMode::bits64);
      for (PrecisionMode pm : {PrecisionMode::bits32, PrecisionMode::bits64}) {
        HistogramSet got = hbg::histoboost_backend::build_histograms_cuda(dev, leaf, pm);
        const bool ok_h = compare_sets(got, want, pm, failures, checks, "");
        (void)ok_h;
        compare_splits(data, leaf, got, want, failures, checks);
        std::printf("       rows=%d d=%d k=%d depth=%d leaf=%lld precision=%s\n", s[0], s[1], s[2], depth,
                    static_cast<long long>(leaf.count()), precision_name(pm));
      }
    }
  }
  // mixed dense/sparse dataset through bin_dataset(sparse_threshold = 0.8)
  // (the reference's default, boosting.hpp:21): the reference builds the
  // sparse features on its pair path (build_sparse_histogram, bin 0 = leaf
  // totals - matched pairs, sparse.cpp:40-43); the drop-in builds every
  // feature from the dense bins bin_dataset retains (binning.cpp:218-224)
  {
    const int rows = 120000, feats = 14;
    RawDataset raw;
    raw.columns.resize(feats);
    raw.targets.assign(rows, 0.0);
    for (int f = 0; f < feats; ++f) {
      const double zero_prob = f < 6 ? 0.0 : (f < 10 ? 0.85 : 0.97);
      auto& c = raw.columns[static_cast<std::size_t>(f)];
      c.resize(rows);
      for (auto& v : c) v = uniform_double(rng) < zero_prob ? 0.0 : normal_double(rng) + (f % 3);
    }
    BinnedDataset data = bin_dataset(raw, 64, 0.8, 5);
    std::vector<double> g(rows), h(rows);
    for (auto& v : g) v = normal_double(rng);
    for (auto& v : h) v = 0.1 + uniform_double(rng);
    hbg::histoboost_backend::DeviceDataset dev(data);
    std::printf("       sparse dataset: %zu dense + %zu sparse features\n", data.dense_features.size(),
                data.sparse_features.size());
    ++checks;
    if (data.sparse_features.size() < 4) ++failures, std::printf("[FAIL] expected sparse features\n");
    for (int depth : {0, 2, 6}) {
      auto idx = leaf_index_sample(rows, depth, 7 + depth);
      LeafState leaf = gather_leaf_statistics(std::move(idx), g, h);
      for (PrecisionMode pm : {PrecisionMode::bits32, PrecisionMode::bits64}) {
        HistogramSet want = build_histograms_partitioned(data, leaf, pm == PrecisionMode::bits64 ? pm : PrecisionMode::bits64);
        HistogramSet got = hbg::histoboost_backend::build_histograms_cuda(dev, leaf, pm);
        compare_sets(got, want, pm, failures, checks, "sparse-mix ");
        compare_splits(data, leaf, got, want, failures, checks);
      }
    }
    GrowParams gp;
    gp.num_leaves = 31;
    gp.min_data_in_leaf = 300;
    for (PrecisionMode pm : {PrecisionMode::bits32, PrecisionMode::bits64}) {
      gp.precision = pm;
      GrowParams ref = gp;
      ref.precision = PrecisionMode::bits64;
      std::vector<SplitInfo> want_log, got_log;
      Tree want = grow_tree(data, g, h, ref, &want_log);
      Tree got = hbg::histoboost_backend::grow_tree_cuda(dev, data, g, h, gp, &got_log);
      compare_trees(want, got, want_log, got_log, pm, failures, checks, "sparse-mix");
    }
  }
  // whole-tree drop-in: grow_tree_cuda vs the reference's grow_tree (bits64)
  // on inputs without near-ties (min_data_in_leaf large enough), both precisions
  for (const auto& s : {std::array<int, 4>{200000, 28, 64, 255}, std::array<int, 4>{100000, 40, 16, 63},
                        std::array<int, 4>{50000, 12, 256, 31}}) {
    BinnedDataset data = gen_synthetic_bins(s[0], s[1], s[2], 3 + s[1]);
    std::vector<double> g(static_cast<std::size_t>(s[0])), h(static_cast<std::size_t>(s[0]));
    for (auto& v : g) v = normal_double(rng);
    for (auto& v : h) v = 0.1 + uniform_double(rng);
    for (int r = 0; r < s[0]; ++r)  // some structure on feature 5
      g[static_cast<std::size_t>(r)] += 0.5 * (data.columns[5].bins[static_cast<std::size_t>(r)] > s[2] / 2);
    GrowParams gp;
    gp.num_leaves = s[3];
    gp.min_data_in_leaf = 400;
    gp.precision = PrecisionMode::bits64;
    std::vector<SplitInfo> want_log;
    Tree want = grow_tree(data, g, h, gp, &want_log);
    hbg::histoboost_backend::DeviceDataset dev(data);
    for (PrecisionMode pm : {PrecisionMode::bits32, PrecisionMode::bits64}) {
      GrowParams p2 = gp;
      p2.precision = pm;
      std::vector<SplitInfo> got_log;
      Tree got = hbg::histoboost_backend::grow_tree_cuda(dev, data, g, h, p2, &got_log);
      char what[96];
      std::snprintf(what, sizeof what, "rows=%d d=%d k=%d leaves=%d", s[0], s[1], s[2], s[3]);
      compare_trees(want, got, want_log, got_log, pm, failures, checks, what);
    }
  }
  // error behaviour: bins beyond the capacity are rejected like invalid_argument
  {
    BinnedDataset bad = gen_synthetic_bins(100, 2, 16, 1);
    bad.columns[1].bins[5] = 200;
    bool threw = false;
    try {
      hbg::histoboost_backend::DeviceDataset dev(bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    ++checks;
    if (!threw) ++failures;
    std::printf("[%s] out-of-range bin raises std::invalid_argument\n", threw ? "PASS" : "FAIL");
  }
  std::printf("%d/%d checks passed\n", checks - failures, checks);
  return failures;
}
