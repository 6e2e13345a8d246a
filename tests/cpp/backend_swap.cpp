// backend_swap.cpp — TEST: the reference's own types and predicates against the
// hbg drop-in (include/hbg_histoboost.hpp). The C++ analogue of
// test_tree.cpp:264-299 ("the lock-step backend grows the same tree as the
// partitioned one") for a `cuda` backend: histograms from
// build_histograms_cuda vs build_histograms_partitioned(bits64) under the
// reference's histograms_equivalent at stats_tolerance(bits32) = 1e-4 — the
// bar the reference applies to its own fp32 path (acceptance.cpp:204-223) —
// with exact counts, the max deviation printed, and the same
// find_best_threshold winner per leaf.
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
#include "histoboost/random.hpp"

using namespace histoboost;

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
      HistogramSet got = hbg::histoboost_backend::build_histograms_cuda(dev, leaf, PrecisionMode::bits32);
      bool ok = got.size() == want.size();
      double worst = 0.0;
      for (std::size_t f = 0; ok && f < want.size(); ++f) {
        ok = got[f].feature_id == want[f].feature_id &&
             histograms_equivalent(got[f], want[f], stats_tolerance(PrecisionMode::bits32));
        for (std::size_t b = 0; ok && b < want[f].bins.size(); ++b) {
          for (auto [x, y] : {std::pair{got[f].bins[b].grad_sum, want[f].bins[b].grad_sum},
                              std::pair{got[f].bins[b].hess_sum, want[f].bins[b].hess_sum}}) {
            double scale = std::max({1.0, std::fabs(x), std::fabs(y)});
            worst = std::max(worst, std::fabs(x - y) / scale);
          }
        }
      }
      LeafTotals tot{leaf.grad_total, leaf.hess_total, leaf.count()};
      std::optional<SplitInfo> bw, bg;
      for (int f = 0; f < data.num_features(); ++f) {
        auto cw = find_best_threshold(want[static_cast<std::size_t>(f)], tot, 1, 0.0);
        auto cg = find_best_threshold(got[static_cast<std::size_t>(f)], tot, 1, 0.0);
        if (cw && (!bw || cw->gain > bw->gain)) bw = cw;
        if (cg && (!bg || cg->gain > bg->gain)) bg = cg;
      }
      bool split_ok = bw.has_value() == bg.has_value() &&
                      (!bw || (bw->feature == bg->feature && bw->threshold_bin == bg->threshold_bin));
      ++checks;
      if (!ok || !split_ok) ++failures;
      std::printf("[%s] rows=%d d=%d k=%d depth=%d leaf=%lld hist=%s (max rel dev %.2e) split=%s (%d,%d)\n",
                  ok && split_ok ? "PASS" : "FAIL", s[0], s[1], s[2], depth,
                  static_cast<long long>(leaf.count()), ok ? "equivalent" : "DIFF", worst,
                  split_ok ? "same" : "DIFF", bw ? bw->feature : -1, bw ? bw->threshold_bin : -1);
    }
  }
  // whole-tree drop-in: grow_tree_cuda vs the reference's grow_tree (bits64)
  // on inputs without near-ties (min_data_in_leaf large enough): the same
  // split sequence, node numbering and thresholds; leaf values within 1e-7
  // relative (test_tree.cpp:264-299 allows 1e-10 between its own backends,
  // which share the fp64 inputs; the device keeps the per-row g/h as fp32 —
  // the bits32 cast of histogram.cpp:97-98 — so its fp64 totals sum the
  // rounded values: ~1e-9 measured)
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
    std::vector<SplitInfo> want_log, got_log;
    Tree want = grow_tree(data, g, h, gp, &want_log);
    hbg::histoboost_backend::DeviceDataset dev(data);
    Tree got = hbg::histoboost_backend::grow_tree_cuda(dev, data, g, h, gp, &got_log);
    bool ok = want_log.size() == got_log.size() && want.nodes().size() == got.nodes().size();
    double worst = 0.0;
    for (std::size_t i = 0; ok && i < want_log.size(); ++i) {
      ok = want_log[i].feature == got_log[i].feature && want_log[i].threshold_bin == got_log[i].threshold_bin &&
           want_log[i].left_count == got_log[i].left_count &&
           want_log[i].threshold_value == got_log[i].threshold_value;
    }
    for (std::size_t i = 0; ok && i < want.nodes().size(); ++i) {
      const TreeNode &a = want.nodes()[i], &b = got.nodes()[i];
      ok = a.feature == b.feature && a.threshold_bin == b.threshold_bin && a.left == b.left && a.right == b.right;
      const double dev_ = std::fabs(a.value - b.value) / std::max(1.0, std::fabs(a.value));
      worst = std::max(worst, dev_);
      ok = ok && dev_ <= 1e-7;
    }
    ++checks;
    if (!ok) ++failures;
    std::printf("[%s] grow_tree_cuda rows=%d d=%d k=%d leaves=%d: %zu splits %s (max value dev %.1e)\n",
                ok ? "PASS" : "FAIL", s[0], s[1], s[2], s[3], want_log.size(), ok ? "identical" : "DIFFER", worst);
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
