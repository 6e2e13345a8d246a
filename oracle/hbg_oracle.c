/*
 * hbg_oracle.c — CPU ORACLE (test infrastructure; see hbg_oracle.h).
 *
 * A plain-C restatement of the histoboost reference algorithms on the
 * histogram hot path. Each function cites the reference file:line it follows
 * (paths relative to /root/reference/proj). Not part of the product: only the
 * tests, smoke() and bench.py's cpu_baseline leg load it.
 */
#include "hbg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- RNG */
/* std::mt19937_64 as fixed by the C++ standard ([rand.predef]); the
 * reference builds every deterministic input from it (random.hpp:10-12). */
#define MT_N 312
#define MT_M 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x7FFFFFFFULL

void hbo_mt64_seed(hbo_mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  r->mti = MT_N;
}

uint64_t hbo_mt64_next(hbo_mt64* r) {
  if (r->mti >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= MT_MATRIX_A;
      r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->mti = 0;
  }
  uint64_t y = r->mt[r->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* random.hpp:14-17 */
double hbo_uniform_double(hbo_mt64* r) { return (double)(hbo_mt64_next(r) >> 11) * 0x1.0p-53; }

/* random.hpp:19-22 */
uint64_t hbo_uniform_below(hbo_mt64* r, uint64_t bound) { return hbo_mt64_next(r) % bound; }

/* random.hpp:24-29 */
double hbo_normal_double(hbo_mt64* r) {
  double u1 = hbo_uniform_double(r);
  double u2 = hbo_uniform_double(r);
  if (u1 < 0x1.0p-60) u1 = 0x1.0p-60;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925287 * u2);
}

/* ------------------------------------------------------- bench inputs */
/* bench.cpp:17-38: per-feature engine seeded seed + f * 0x9e3779b97f4a7c15,
 * bins uniform in [1, max_bin - 1]. */
void hbo_gen_synthetic_bins(int64_t rows, int features, int max_bin, uint64_t seed,
                            uint8_t* out) {
  hbo_mt64 rng;
  for (int f = 0; f < features; ++f) {
    hbo_mt64_seed(&rng, seed + (uint64_t)f * 0x9e3779b97f4a7c15ULL);
    uint8_t* col = out + (int64_t)f * rows;
    for (int64_t i = 0; i < rows; ++i) {
      col[i] = (uint8_t)(1 + hbo_uniform_below(&rng, (uint64_t)(max_bin - 1)));
    }
  }
}

/* bench.cpp:69-73 */
void hbo_gen_grad_hess(int64_t rows, uint64_t seed, double* g, double* h) {
  hbo_mt64 rng;
  hbo_mt64_seed(&rng, seed ^ 0xdeadbeefcafef00dULL);
  for (int64_t i = 0; i < rows; ++i) g[i] = 2.0 * hbo_uniform_double(&rng) - 1.0;
  for (int64_t i = 0; i < rows; ++i) h[i] = hbo_uniform_double(&rng);
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* bench.cpp:40-57: identity at depth 0, else a partial Fisher-Yates prefix of
 * length rows >> depth, sorted. */
int64_t hbo_leaf_index_sample(int64_t rows, int depth, uint64_t seed, int32_t* out) {
  if (depth < 0 || depth > 62) return -1;
  int64_t take = rows >> depth;
  if (take < 1) return -1;
  for (int64_t i = 0; i < rows; ++i) out[i] = (int32_t)i;
  if (depth > 0) {
    hbo_mt64 rng;
    hbo_mt64_seed(&rng, seed);
    for (int64_t i = 0; i < take; ++i) {
      int64_t j = i + (int64_t)hbo_uniform_below(&rng, (uint64_t)(rows - i));
      int32_t t = out[i];
      out[i] = out[j];
      out[j] = t;
    }
    qsort(out, (size_t)take, sizeof(int32_t), cmp_i32);
  }
  return take;
}

/* ------------------------------------------------------------ packing */
/* binning.cpp:123-158: bits * p offset within each word, pad slots 0. */
int hbo_pack_feature_tuples(const uint8_t* cols, int d, int64_t rows, int bits, int max_bin,
                            uint32_t* words) {
  int per_word = 32 / bits;
  if (bits == 4 && max_bin > 16) return -1;
  int tuples = (d + per_word - 1) / per_word;
  memset(words, 0, sizeof(uint32_t) * (size_t)tuples * (size_t)rows);
  for (int t = 0; t < tuples; ++t) {
    for (int p = 0; p < per_word; ++p) {
      int f = t * per_word + p;
      if (f >= d) break;
      const uint8_t* col = cols + (int64_t)f * rows;
      uint32_t* w = words + (int64_t)t * rows;
      for (int64_t i = 0; i < rows; ++i) w[i] |= (uint32_t)col[i] << (bits * p);
    }
  }
  return tuples;
}

/* binning.cpp:160-182 */
int hbo_redistribute_bins(const uint8_t* col, int64_t rows, int bin_capacity, uint8_t* spread,
                          int* original_effective_bins) {
  int max_bin = -1;
  for (int64_t i = 0; i < rows; ++i)
    if ((int)col[i] > max_bin) max_bin = col[i];
  int spanned = max_bin + 1;
  if (original_effective_bins) *original_effective_bins = spanned > 1 ? spanned : 1;
  memcpy(spread, col, (size_t)rows);
  if (rows == 0 || spanned * 2 >= bin_capacity) return 1;
  int expansion = 1;
  while (expansion * 2 * spanned <= bin_capacity) expansion *= 2;
  uint32_t mask = (uint32_t)expansion - 1;
  for (int64_t i = 0; i < rows; ++i) {
    spread[i] = (uint8_t)((uint32_t)col[i] * (uint32_t)expansion + ((uint32_t)i & mask));
  }
  return expansion;
}

/* binning.cpp:184-202 */
void hbo_fold_histogram(const hbo_bin* in, int k, int expansion, hbo_bin* out) {
  if (expansion == 1) {
    memcpy(out, in, sizeof(hbo_bin) * (size_t)k);
    return;
  }
  memset(out, 0, sizeof(hbo_bin) * (size_t)k);
  for (int i = 0; i * expansion < k; ++i) {
    hbo_bin acc = {0.0, 0.0, 0};
    int end = (i + 1) * expansion < k ? (i + 1) * expansion : k;
    for (int j = i * expansion; j < end; ++j) {
      acc.grad_sum += in[j].grad_sum;
      acc.hess_sum += in[j].hess_sum;
      acc.count += in[j].count;
    }
    out[i] = acc;
  }
}

/* ---------------------------------------------------------- histogram */
/* tree.cpp:11-25 */
void hbo_gather_leaf(const int32_t* idx, int64_t n, const double* g, const double* h,
                     double* leaf_g, double* leaf_h, double* grad_total, double* hess_total) {
  double gt = 0.0, ht = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    leaf_g[i] = g[idx[i]];
    leaf_h[i] = h[idx[i]];
    gt += leaf_g[i];
    ht += leaf_h[i];
  }
  *grad_total = gt;
  *hess_total = ht;
}

/* histogram.cpp:86-106: Alg. 1 in leaf-index order, Acc = float | double. */
void hbo_build_histogram(const uint8_t* col, int k, const int32_t* idx, int64_t n,
                         const double* leaf_g, const double* leaf_h, int precision, hbo_bin* out) {
  memset(out, 0, sizeof(hbo_bin) * (size_t)k);
  if (precision == 32) {
    float* g = (float*)calloc((size_t)k, sizeof(float));
    float* h = (float*)calloc((size_t)k, sizeof(float));
    for (int64_t i = 0; i < n; ++i) {
      uint8_t b = col[idx[i]];
      g[b] += (float)leaf_g[i];
      h[b] += (float)leaf_h[i];
      out[b].count += 1;
    }
    for (int b = 0; b < k; ++b) {
      out[b].grad_sum = (double)g[b];
      out[b].hess_sum = (double)h[b];
    }
    free(g);
    free(h);
  } else {
    for (int64_t i = 0; i < n; ++i) {
      uint8_t b = col[idx[i]];
      out[b].grad_sum += leaf_g[i];
      out[b].hess_sum += leaf_h[i];
      out[b].count += 1;
    }
  }
}

/* histogram.cpp:159-215 for dense features: 64Ki-row chunks, partials
 * reduced in chunk order in Acc (reduce_impl, :108-127). */
void hbo_build_histograms_partitioned(const uint8_t* cols, int d, int64_t rows, int k,
                                      const int32_t* idx, int64_t n, const double* leaf_g,
                                      const double* leaf_h, int precision, hbo_bin* out) {
  const int64_t chunk = 65536;
  int64_t chunks = n == 0 ? 1 : (n + chunk - 1) / chunk;
  hbo_bin* part = (hbo_bin*)malloc(sizeof(hbo_bin) * (size_t)k);
  float* gf = (float*)malloc(sizeof(float) * (size_t)k);
  float* hf = (float*)malloc(sizeof(float) * (size_t)k);
  for (int f = 0; f < d; ++f) {
    const uint8_t* col = cols + (int64_t)f * rows;
    hbo_bin* o = out + (int64_t)f * k;
    if (chunks == 1) {
      hbo_build_histogram(col, k, idx, n, leaf_g, leaf_h, precision, o);
      continue;
    }
    memset(o, 0, sizeof(hbo_bin) * (size_t)k);
    for (int b = 0; b < k; ++b) gf[b] = hf[b] = 0.0f;
    for (int64_t c = 0; c < chunks; ++c) {
      int64_t begin = c * chunk;
      int64_t len = (begin + chunk < n ? begin + chunk : n) - begin;
      hbo_build_histogram(col, k, idx + begin, len, leaf_g + begin, leaf_h + begin, precision,
                          part);
      for (int b = 0; b < k; ++b) {
        if (precision == 32) {
          gf[b] += (float)part[b].grad_sum;
          hf[b] += (float)part[b].hess_sum;
        } else {
          o[b].grad_sum += part[b].grad_sum;
          o[b].hess_sum += part[b].hess_sum;
        }
        o[b].count += part[b].count;
      }
    }
    if (precision == 32) {
      for (int b = 0; b < k; ++b) {
        o[b].grad_sum = (double)gf[b];
        o[b].hess_sum = (double)hf[b];
      }
    }
  }
  free(part);
  free(gf);
  free(hf);
}

/* ------------------------------------------------------------- splits */
/* tree.cpp:59-64 */
double hbo_optimal_leaf_value(double grad_sum, double hess_sum, double lambda) {
  double denom = hess_sum + lambda;
  if (denom <= 0.0) return 0.0;
  return -grad_sum / denom;
}

/* tree.cpp:66-74 */
double hbo_split_gain(double lg, double lh, double rg, double rh, double lambda) {
  double dl = lh + lambda;
  double dr = rh + lambda;
  double dp = lh + rh + lambda;
  if (dl <= 0.0 || dr <= 0.0 || dp <= 0.0) return 0.0;
  double g = lg + rg;
  return lg * lg / dl + rg * rg / dr - g * g / dp;
}

/* tree.cpp:76-112: left = bins <= b for b in [0, k-2]; strict > keeps the
 * smallest bin on ties. */
int hbo_find_best_threshold(const hbo_bin* hist, int k, int feature_id, double grad_total,
                            double hess_total, int64_t count, int64_t min_data_in_leaf,
                            double lambda, hbo_split* out) {
  int found = 0;
  double lg = 0.0, lh = 0.0;
  int64_t lc = 0;
  for (int b = 0; b < k - 1; ++b) {
    lg += hist[b].grad_sum;
    lh += hist[b].hess_sum;
    lc += hist[b].count;
    if (lc < min_data_in_leaf) continue;
    int64_t rc = count - lc;
    if (rc < min_data_in_leaf) break;
    double rg = grad_total - lg;
    double rh = hess_total - lh;
    double gain = hbo_split_gain(lg, lh, rg, rh, lambda);
    if (gain <= 0.0) continue;
    if (!found || gain > out->gain) {
      found = 1;
      out->feature = feature_id;
      out->threshold_bin = b;
      out->gain = gain;
      out->left_grad = lg;
      out->left_hess = lh;
      out->left_count = lc;
      out->right_grad = rg;
      out->right_hess = rh;
      out->right_count = rc;
      out->left_value = hbo_optimal_leaf_value(lg, lh, lambda);
      out->right_value = hbo_optimal_leaf_value(rg, rh, lambda);
    }
  }
  return found;
}

/* tree.cpp:163-182 (early exit :165, lowest feature wins ties :172). */
int hbo_find_best_split(const hbo_bin* hists, int d, int k, double grad_total, double hess_total,
                        int64_t count, int64_t min_data_in_leaf, double lambda, hbo_split* out) {
  if (count < 2 * min_data_in_leaf || count < 2) return 0;
  int found = 0;
  for (int f = 0; f < d; ++f) {
    hbo_split cand;
    if (hbo_find_best_threshold(hists + (int64_t)f * k, k, f, grad_total, hess_total, count,
                                min_data_in_leaf, lambda, &cand)) {
      if (!found || cand.gain > out->gain) {
        *out = cand;
        found = 1;
      }
    }
  }
  return found;
}

/* tree.cpp:114-128 */
int64_t hbo_partition_leaf(const int32_t* idx, int64_t n, const uint8_t* col, int threshold_bin,
                           int32_t* left, int32_t* right) {
  int64_t nl = 0, nr = 0;
  for (int64_t i = 0; i < n; ++i) {
    if ((int)col[idx[i]] <= threshold_bin) {
      left[nl++] = idx[i];
    } else {
      right[nr++] = idx[i];
    }
  }
  if (nl == 0 || nr == 0) return -1;
  return nl;
}

/* ---------------------------------------------------------- grow tree */
typedef struct open_leaf {
  int node;
  int32_t* idx;
  int64_t n;
  double gt, ht;
  int has_best;
  hbo_split best;
} open_leaf;

static int leaf_best(const uint8_t* cols, int d, int64_t rows, int k, const double* g,
                     const double* h, open_leaf* L, int64_t min_data, double lambda,
                     int precision, hbo_bin* hist, double* lg, double* lh) {
  if (L->n < 2 * min_data || L->n < 2) return 0;
  double gt, ht;
  hbo_gather_leaf(L->idx, L->n, g, h, lg, lh, &gt, &ht);
  hbo_build_histograms_partitioned(cols, d, rows, k, L->idx, L->n, lg, lh, precision, hist);
  return hbo_find_best_split(hist, d, k, L->gt, L->ht, L->n, min_data, lambda, &L->best);
}

/* tree.cpp:186-261: strict > over the pool in insertion order (oldest leaf
 * wins ties), children appended left then right, both built from scratch. */
int hbo_grow_tree(const uint8_t* cols, int d, int64_t rows, int k, const double* g,
                  const double* h, int num_leaves, int64_t min_data_in_leaf, double lambda,
                  int precision, hbo_split* split_log, int32_t* node_feature,
                  int32_t* node_threshold_bin, int32_t* node_left, int32_t* node_right,
                  double* node_value, int* num_nodes) {
  if (num_leaves < 1) return -1;
  int max_nodes = 2 * num_leaves - 1;
  int nodes = 1;
  hbo_bin* hist = (hbo_bin*)malloc(sizeof(hbo_bin) * (size_t)d * (size_t)k);
  double* lg = (double*)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1));
  double* lh = (double*)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1));
  open_leaf* pool = (open_leaf*)calloc((size_t)num_leaves + 2, sizeof(open_leaf));
  int pool_n = 0, logged = 0;

  int32_t* all = (int32_t*)malloc(sizeof(int32_t) * (size_t)(rows > 0 ? rows : 1));
  for (int64_t i = 0; i < rows; ++i) all[i] = (int32_t)i;
  double gt, ht;
  hbo_gather_leaf(all, rows, g, h, lg, lh, &gt, &ht);
  if (node_feature) {
    for (int i = 0; i < max_nodes; ++i) {
      node_feature[i] = -1;
      node_threshold_bin[i] = -1;
      node_left[i] = node_right[i] = -1;
      node_value[i] = 0.0;
    }
    node_value[0] = hbo_optimal_leaf_value(gt, ht, lambda);
  }
  if (num_leaves >= 2) {
    open_leaf* r = &pool[pool_n++];
    r->node = 0;
    r->idx = all;
    r->n = rows;
    r->gt = gt;
    r->ht = ht;
    r->has_best = leaf_best(cols, d, rows, k, g, h, r, min_data_in_leaf, lambda, precision, hist,
                            lg, lh);
  } else {
    free(all);
  }

  int leaves = 1;
  while (leaves < num_leaves) {
    int pick = -1;
    for (int i = 0; i < pool_n; ++i) {
      if (!pool[i].has_best) continue;
      if (pick < 0 || pool[i].best.gain > pool[pick].best.gain) pick = i;
    }
    if (pick < 0) break;
    open_leaf chosen = pool[pick];
    memmove(&pool[pick], &pool[pick + 1], sizeof(open_leaf) * (size_t)(pool_n - pick - 1));
    --pool_n;
    if (split_log) split_log[logged] = chosen.best;
    ++logged;

    const uint8_t* col = cols + (int64_t)chosen.best.feature * rows;
    int32_t* left = (int32_t*)malloc(sizeof(int32_t) * (size_t)chosen.n);
    int32_t* right = (int32_t*)malloc(sizeof(int32_t) * (size_t)chosen.n);
    int64_t nl = hbo_partition_leaf(chosen.idx, chosen.n, col, chosen.best.threshold_bin, left,
                                    right);
    int64_t nr = chosen.n - nl;
    free(chosen.idx);

    int left_id = nodes, right_id = nodes + 1;
    nodes += 2;
    if (node_feature) {
      node_feature[chosen.node] = chosen.best.feature;
      node_threshold_bin[chosen.node] = chosen.best.threshold_bin;
      node_left[chosen.node] = left_id;
      node_right[chosen.node] = right_id;
      node_value[chosen.node] = 0.0;
    }
    ++leaves;

    open_leaf lo = {0}, ro = {0};
    lo.node = left_id;
    lo.idx = left;
    lo.n = nl;
    ro.node = right_id;
    ro.idx = right;
    ro.n = nr;
    hbo_gather_leaf(left, nl, g, h, lg, lh, &lo.gt, &lo.ht);
    hbo_gather_leaf(right, nr, g, h, lg, lh, &ro.gt, &ro.ht);
    if (node_feature) {
      node_value[left_id] = hbo_optimal_leaf_value(lo.gt, lo.ht, lambda);
      node_value[right_id] = hbo_optimal_leaf_value(ro.gt, ro.ht, lambda);
    }
    if (leaves < num_leaves) {
      lo.has_best = leaf_best(cols, d, rows, k, g, h, &lo, min_data_in_leaf, lambda, precision,
                              hist, lg, lh);
      ro.has_best = leaf_best(cols, d, rows, k, g, h, &ro, min_data_in_leaf, lambda, precision,
                              hist, lg, lh);
    }
    pool[pool_n++] = lo;
    pool[pool_n++] = ro;
  }
  for (int i = 0; i < pool_n; ++i) free(pool[i].idx);
  free(pool);
  free(hist);
  free(lg);
  free(lh);
  if (num_nodes) *num_nodes = nodes;
  return logged;
}

/* losses.cpp:14,24-26,57-60 */
void hbo_grad_hess(int loss, const double* scores, const double* targets, int64_t n, double* g,
                   double* h) {
  for (int64_t i = 0; i < n; ++i) {
    if (loss == 0) {
      g[i] = scores[i] - targets[i];
      h[i] = 1.0;
    } else {
      double p = 1.0 / (1.0 + exp(-scores[i]));
      g[i] = p - targets[i];
      double hh = p * (1.0 - p);
      h[i] = hh > 1e-16 ? hh : 1e-16;
    }
  }
}

/* boosting.cpp:26-51; the score update routes every row through the tree by
 * its bins (Tree::predict_binned, tree.cpp:47-57). */
int hbo_boost_one_iteration(const uint8_t* cols, int d, int64_t rows, int k, const double* targets,
                            int loss, double learning_rate, int num_leaves, int64_t min_data_in_leaf,
                            double lambda, int precision, double* scores, hbo_split* split_log) {
  double* g = (double*)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1));
  double* h = (double*)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1));
  int max_nodes = 2 * num_leaves - 1;
  int32_t* nf = (int32_t*)malloc(sizeof(int32_t) * (size_t)max_nodes);
  int32_t* nt = (int32_t*)malloc(sizeof(int32_t) * (size_t)max_nodes);
  int32_t* nl = (int32_t*)malloc(sizeof(int32_t) * (size_t)max_nodes);
  int32_t* nr = (int32_t*)malloc(sizeof(int32_t) * (size_t)max_nodes);
  double* nv = (double*)malloc(sizeof(double) * (size_t)max_nodes);
  int nn = 0;
  hbo_grad_hess(loss, scores, targets, rows, g, h);
  int logged = hbo_grow_tree(cols, d, rows, k, g, h, num_leaves, min_data_in_leaf, lambda, precision,
                             split_log, nf, nt, nl, nr, nv, &nn);
  for (int64_t i = 0; i < rows; ++i) {
    int at = 0;
    while (nf[at] >= 0) at = cols[(int64_t)nf[at] * rows + i] <= nt[at] ? nl[at] : nr[at];
    scores[i] += learning_rate * nv[at];
  }
  free(g);
  free(h);
  free(nf);
  free(nt);
  free(nl);
  free(nr);
  free(nv);
  return logged;
}

/* histogram.cpp:12-15 */
int hbo_stats_close(double a, double b, double tolerance) {
  double scale = 1.0;
  if (fabs(a) > scale) scale = fabs(a);
  if (fabs(b) > scale) scale = fabs(b);
  return fabs(a - b) <= tolerance * scale;
}
