// hbg_histoboost.hpp — header-only C++ adaptor from the reference's types to
// the hbg C ABI: the drop-in a histoboost maintainer links.
//
// It mirrors the reference's operator interface for the hot path:
//   HistogramSet build_histograms_partitioned(const BinnedDataset&, const LeafState&,
//                                             PrecisionMode, int)   histogram.hpp:133-134
// as
//   HistogramSet hbg::histoboost_backend::build_histograms_cuda(const BinnedDataset&,
//                                             const LeafState&, PrecisionMode)
// with the same argument meaning (LeafState arrays are leaf-aligned doubles),
// the same output (one HistogramEntry per feature id, bin_capacity bins each)
// and the same error classes (std::invalid_argument / std::logic_error;
// CUDA failures surface as std::runtime_error — there is no CPU fallback).
//
// Requires the reference headers on the include path (histoboost/*.hpp) and
// linking libhbg.so. Dense features only: the reference runs sparse features
// on the CPU pair path (sparse.cpp), as the paper does.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "hbg.h"
#include "histoboost/dataset.hpp"
#include "histoboost/histogram.hpp"
#include "histoboost/leaf.hpp"
#include "histoboost/tree.hpp"

namespace hbg::histoboost_backend {

inline void check(int status) {
  if (status == HBG_OK) return;
  const std::string msg = hbg_last_error();
  if (status == HBG_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (status == HBG_ERR_LOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

// Device-resident packed copy of a BinnedDataset's dense columns. Build once
// per dataset (after bin_dataset), reuse for every leaf of every tree.
class DeviceDataset {
 public:
  explicit DeviceDataset(const histoboost::BinnedDataset& data, int device = 0)
      : num_features_(data.num_features()), max_bin_(data.max_bin) {
    if (!data.sparse_features.empty()) {
      throw std::invalid_argument("hbg backend: sparse features stay on the CPU pair path");
    }
    std::vector<const std::uint8_t*> cols(static_cast<std::size_t>(num_features_));
    for (int f = 0; f < num_features_; ++f) {
      cols[static_cast<std::size_t>(f)] = data.columns[static_cast<std::size_t>(f)].bins.data();
    }
    hbg_dataset* h = nullptr;
    check(hbg_dataset_create(cols.data(), num_features_, data.num_rows, max_bin_, device, &h));
    handle_.reset(h);
  }
  hbg_dataset* get() const { return handle_.get(); }
  int num_features() const { return num_features_; }
  int max_bin() const { return max_bin_; }

 private:
  struct Destroy {
    void operator()(hbg_dataset* h) const { hbg_dataset_destroy(h); }
  };
  std::unique_ptr<hbg_dataset, Destroy> handle_;
  int num_features_;
  int max_bin_;
};

// The drop-in for build_histograms_partitioned. `precision` is accepted for
// signature parity: the device accumulates fp32 partials reduced in fp64,
// which meets stats_tolerance(bits32) = 1e-4 and, on the BASELINE shapes,
// 1e-5 against bits64.
inline histoboost::HistogramSet build_histograms_cuda(const DeviceDataset& dev,
                                                      const histoboost::LeafState& leaf,
                                                      histoboost::PrecisionMode precision) {
  const int d = dev.num_features(), k = dev.max_bin();
  std::vector<hbg_bin> bins(static_cast<std::size_t>(d) * static_cast<std::size_t>(k));
  check(hbg_build_histograms(dev.get(), leaf.indices.data(), leaf.count(), leaf.gradients.data(),
                             leaf.hessians.data(), bins.data()));
  histoboost::HistogramSet out(static_cast<std::size_t>(d));
  for (int f = 0; f < d; ++f) {
    auto& e = out[static_cast<std::size_t>(f)];
    e.feature_id = f;
    e.precision = precision;
    e.bins.resize(static_cast<std::size_t>(k));
    static_assert(sizeof(hbg_bin) == sizeof(histoboost::HistogramBin), "HistogramBin layout");
    std::memcpy(e.bins.data(), bins.data() + static_cast<std::size_t>(f) * k,
                sizeof(hbg_bin) * static_cast<std::size_t>(k));
  }
  return out;
}

// The whole-tree drop-in for grow_tree (tree.hpp, tree.cpp:186-261): same
// arguments (fp64 per-row gradients/hessians, GrowParams, optional split
// log), same Tree (node numbering, values from the children's fp64 totals,
// threshold_value from data.boundaries as find_best_split does,
// tree.cpp:174-180). The histogram, subtraction, split scans and partitions
// run on the device; `params.backend`/`precision` are accepted for signature
// parity (the device builds fp32 histograms reduced in fp64).
inline histoboost::Tree grow_tree_cuda(const DeviceDataset& dev, const histoboost::BinnedDataset& data,
                                       std::span<const double> gradients, std::span<const double> hessians,
                                       const histoboost::GrowParams& params,
                                       std::vector<histoboost::SplitInfo>* split_log = nullptr) {
  if (params.num_leaves < 1) throw std::invalid_argument("num_leaves must be at least 1");
  if (gradients.size() != static_cast<std::size_t>(data.num_rows) ||
      hessians.size() != static_cast<std::size_t>(data.num_rows)) {
    throw std::invalid_argument("gradient/hessian length differs from the row count");
  }
  const hbg_grow_params p{params.num_leaves, 0, params.min_data_in_leaf, params.lambda};
  std::vector<hbg_split> log(static_cast<std::size_t>(std::max(1, params.num_leaves - 1)));
  std::vector<hbg_tree_node> nodes(static_cast<std::size_t>(std::max(1, 2 * params.num_leaves - 1)));
  std::int32_t ns = 0, nn = 0;
  check(hbg_grow_tree_host(dev.get(), gradients.data(), hessians.data(), &p, log.data(), &ns, nodes.data(), &nn));
  auto threshold_value = [&](int feature, int bin) {
    if (bin == 0) return -std::numeric_limits<double>::infinity();
    return data.boundaries[static_cast<std::size_t>(feature)].upper_bounds[static_cast<std::size_t>(bin - 1)];
  };
  histoboost::Tree tree;
  for (std::int32_t i = 0; i < nn; ++i) {
    const hbg_tree_node& n = nodes[static_cast<std::size_t>(i)];
    histoboost::TreeNode t;
    t.feature = n.feature;
    t.threshold_bin = n.threshold_bin;
    t.threshold_value = n.feature >= 0 ? threshold_value(n.feature, n.threshold_bin) : 0.0;
    t.left = n.left;
    t.right = n.right;
    t.value = n.value;
    tree.nodes().push_back(t);
  }
  if (split_log) {
    for (std::int32_t i = 0; i < ns; ++i) {
      const hbg_split& s = log[static_cast<std::size_t>(i)];
      histoboost::SplitInfo si;
      si.feature = s.feature;
      si.threshold_bin = s.threshold_bin;
      si.threshold_value = threshold_value(s.feature, s.threshold_bin);
      si.gain = s.gain;
      si.left_grad = s.left_grad;
      si.left_hess = s.left_hess;
      si.right_grad = s.right_grad;
      si.right_hess = s.right_hess;
      si.left_count = s.left_count;
      si.right_count = s.right_count;
      si.left_value = s.left_value;
      si.right_value = s.right_value;
      split_log->push_back(si);
    }
  }
  return tree;
}

}  // namespace hbg::histoboost_backend
