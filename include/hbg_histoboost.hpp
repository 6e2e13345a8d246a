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
// linking libhbg.so. Sparse features (BinnedDataset::sparse_features,
// classify_features, binning.cpp:98-109) are served from the dense bins that
// bin_dataset keeps for every column (binning.cpp:218-224: sparse_storage is
// added, columns[f].bins stays): the device histogram of such a feature is the
// same HistogramEntry the pair path (sparse.cpp:9-56) builds, within the
// reference's own sparse == dense tolerance (test_histogram.cpp:96-116).
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
      : num_features_(data.num_features()), max_bin_(data.max_bin), num_rows_(data.num_rows) {
    // every column, dense or sparse, by feature id: the HistogramSet index
    std::vector<const std::uint8_t*> cols(static_cast<std::size_t>(num_features_));
    for (int f = 0; f < num_features_; ++f) {
      const auto& bins = data.columns[static_cast<std::size_t>(f)].bins;
      if (static_cast<std::int64_t>(bins.size()) != data.num_rows) {
        throw std::invalid_argument("hbg backend: column " + std::to_string(f) + " has no dense bins");
      }
      cols[static_cast<std::size_t>(f)] = bins.data();
    }
    hbg_dataset* h = nullptr;
    check(hbg_dataset_create(cols.data(), num_features_, data.num_rows, max_bin_, device, &h));
    handle_.reset(h);
  }
  hbg_dataset* get() const { return handle_.get(); }
  int num_features() const { return num_features_; }
  int max_bin() const { return max_bin_; }
  std::int64_t num_rows() const { return num_rows_; }
  // The device copy is a snapshot: it must be rebuilt when the dataset is
  // re-binned or replaced. Cheap guard for callers that hold it next to a
  // BinnedDataset: the shape must still agree.
  void require_describes(const histoboost::BinnedDataset& data) const {
    if (data.num_rows != num_rows_ || data.num_features() != num_features_ || data.max_bin != max_bin_) {
      throw std::logic_error("hbg backend: DeviceDataset was built for a different dataset shape");
    }
  }

 private:
  struct Destroy {
    void operator()(hbg_dataset* h) const { hbg_dataset_destroy(h); }
  };
  std::unique_ptr<hbg_dataset, Destroy> handle_;
  int num_features_;
  int max_bin_;
  std::int64_t num_rows_;
};

inline std::int32_t to_hbg(histoboost::PrecisionMode p) {
  return p == histoboost::PrecisionMode::bits64 ? HBG_PRECISION_BITS64 : HBG_PRECISION_BITS32;
}

// The drop-in for build_histograms_partitioned, honouring PrecisionMode:
//  bits32 — fp32 inputs (the reference's per-element cast), fp32 per-warp
//           sums reduced in fp64. Against the reference's bits64 sums (tests,
//           DESIGN.md §5): <= 1e-5 up to 300K-row leaves; at the 10.5M-row
//           root 7.6e-5 (k64) / 2.1e-4 (k16), where the reference's own bits32
//           path is at 1.8e-4 / 7.5e-4 — fp32 inputs cannot do better there;
//  bits64 — fp64 inputs, fp64 accumulation: within stats_tolerance(bits64) =
//           1e-12 of the reference's bits64 (tests up to the 10.5M-row root).
inline histoboost::HistogramSet build_histograms_cuda(const DeviceDataset& dev,
                                                      const histoboost::LeafState& leaf,
                                                      histoboost::PrecisionMode precision) {
  const int d = dev.num_features(), k = dev.max_bin();
  std::vector<hbg_bin> bins(static_cast<std::size_t>(d) * static_cast<std::size_t>(k));
  check(hbg_build_histograms_ex(dev.get(), leaf.indices.data(), leaf.count(), leaf.gradients.data(),
                                leaf.hessians.data(), to_hbg(precision), bins.data()));
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
// run on the device with params.precision honoured (bits32: fp32 g/h in the
// persistent one-kernel grower; bits64: fp64 g/h and fp64 histograms at
// every leaf); `params.backend` selects nothing here (this IS the backend).
inline histoboost::Tree grow_tree_cuda(const DeviceDataset& dev, const histoboost::BinnedDataset& data,
                                       std::span<const double> gradients, std::span<const double> hessians,
                                       const histoboost::GrowParams& params,
                                       std::vector<histoboost::SplitInfo>* split_log = nullptr) {
  if (params.num_leaves < 1) throw std::invalid_argument("num_leaves must be at least 1");
  if (gradients.size() != static_cast<std::size_t>(data.num_rows) ||
      hessians.size() != static_cast<std::size_t>(data.num_rows)) {
    throw std::invalid_argument("gradient/hessian length differs from the row count");
  }
  const hbg_grow_params p{params.num_leaves, to_hbg(params.precision), params.min_data_in_leaf, params.lambda};
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
