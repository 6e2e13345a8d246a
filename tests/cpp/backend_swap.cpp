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
