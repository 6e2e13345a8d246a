// capi.cu — the extern "C" boundary declared in include/hbg.h.
//
// C++ host logic: argument validation with the reference's error classes
// (std::invalid_argument -> HBG_ERR_INVALID_ARGUMENT, std::logic_error ->
// HBG_ERR_LOGIC), device memory ownership, launch planning. There is no CPU
// fallback anywhere: a missing GPU or CUDA failure is an error status.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include "hbg_internal.h"

namespace hbg {

namespace {
thread_local std::string g_last_error;
}

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
                cudaGetErrorString(e), file, line, what);
  throw Error(e == cudaErrorMemoryAllocation ? HBG_ERR_OUT_OF_MEMORY : HBG_ERR_CUDA, buf);
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return HBG_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return HBG_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HBG_ERR_LOGIC;
  }
}

int guarded_call_impl(void (*fn)(void*), void* arg) {
  return guarded([&] { fn(arg); });
}

// A grow-only device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t need) {
    if (need > bytes) {
      if (p) HBG_CUDA(cudaFree(p));
      p = nullptr;
      bytes = 0;
      HBG_CUDA(cudaMalloc(&p, std::max<size_t>(need, 256)));
      bytes = std::max<size_t>(need, 256);
    }
    return p;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    HBG_CUDA(cudaGetDevice(&prev));
    if (prev != dev) HBG_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace hbg

struct hbg_dataset {
  hbg_layout layout{};
  uint32_t* packed = nullptr;  // num_rows * row_stride_bytes
  cudaStream_t stream = nullptr;
  // workspace (not re-entrant per handle)
  hbg::DevBuf colbins;  // column-major uint8 bins [feature][row] (the a1 layout), for partitions
  hbg::DevBuf host_parts;                 // host drop-in: per-chunk histograms
  cudaStream_t copy_stream = nullptr;     // host drop-in: H2D copies overlapped with the kernels
  cudaEvent_t chunk_ev[17] = {};  // per histogram chunk (<= 16) + [16]: the copy stream's start
  hbg::DevBuf part, iota, host_idx, host_gd, host_hd, host_gf, host_hf, host_hist, host_bins;
  int64_t iota_rows = 0;
  int64_t copy_h2d = 0, copy_d2h = 0;  // bytes of the last host drop-in call
  // tree growth workspace
  hbg::DevBuf ord[2][3];  // ping-pong (row, g, h) ordered buffers
  hbg::DevBuf slots, part_scratch, tree_small;  // leaf histograms, partition scratch, splits/totals
  hbg::DevBuf boost_g, boost_h, boost_leaves;   // boosting: fp32 gradients, final leaf ranges
  hbg::DevBuf small_acc, small_exps;            // fixed-point accumulator for small leaves
  hbg::DevBuf hist_bar;                         // multi-cluster arrival counters (zeroed once)
  hbg::DevBuf hist_prof;                        // HBG_HIST_PROFILE phase stamps of the last launch
  hbg::DevBuf grow_nodes, grow_log, grow_tree, grow_counts, grow_scratch, grow_root, grow_prof;  // persistent grower
  const void* grow_records = nullptr;  // the last grown tree's score-update input (launch_grow_persistent)
  bool grow_waves = false;             // ... LeafRange x grow_ranges (wave grower) or node records
  int grow_ranges = 0;
  void* pinned = nullptr;                      // host staging for per-split results
  void* stage = nullptr;                       // pinned staging of pageable host inputs (stage_bytes)
  size_t stage_bytes = 0;
  // measurement hooks
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;  // recorded, not yet read
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> spare;
  std::pair<cudaEvent_t, cudaEvent_t> event_pair() {
    if (!spare.empty()) {
      auto e = spare.back();
      spare.pop_back();
      return e;
    }
    std::pair<cudaEvent_t, cudaEvent_t> e;
    HBG_CUDA(cudaEventCreate(&e.first));
    HBG_CUDA(cudaEventCreate(&e.second));
    return e;
  }
  ~hbg_dataset() {
    if (pinned) cudaFreeHost(pinned);
    if (stage) {
      if (stream) cudaStreamSynchronize(stream);
      if (copy_stream) cudaStreamSynchronize(copy_stream);
      cudaFreeHost(stage);
    }
    for (auto& e : events) spare.push_back(e);
    for (auto& e : spare) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    if (stream) cudaStreamSynchronize(stream);
    if (copy_stream) cudaStreamSynchronize(copy_stream);
    for (auto& e : chunk_ev)
      if (e) cudaEventDestroy(e);
    if (packed) cudaFree(packed);
    if (stream) cudaStreamDestroy(stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
  }
};

// Row-sharding exchange area of one rank (grow_persistent.cu): allocated on
// the rank's device, exported as a CUDA IPC handle (other processes) or
// attached directly (same process); every rank maps every rank's area.
struct hbg_peer {
  int nranks = 1, rank = 0, device = 0, ctas = 0;
  double* xbuf = nullptr;
  size_t xdoubles = 0;          // tree-exchange region [0, xdoubles)
  size_t hoff = 0, hdoubles = 0;  // histogram-exchange region [hoff, hoff + hdoubles)
  unsigned long long hgen = 0;  // histogram-exchange generation
  int* error = nullptr;         // device flag: a peer never published
  const double* peers[8] = {nullptr};
  void* opened[8] = {nullptr};  // IPC mappings to close
  unsigned long long gen = 0;   // tree generation
  ~hbg_peer() {
    for (void* p : opened)
      if (p) cudaIpcCloseMemHandle(p);
    if (xbuf) cudaFree(xbuf);
    if (error) cudaFree(error);
  }
};

using namespace hbg;

// Bound of every in-kernel wait on another rank or on the grid (clock64
// cycles of `device`): HBG_PEER_TIMEOUT_MS, default 60 s — generous, because
// ranks reach a peer call at different times (data loading, GC, checkpoints)
// and there is no host handshake before the launch; a wait that expires is an
// HBG_ERR_CUDA status, never a hang.
long long hbg::wait_timeout_cycles(int device) {
  static std::once_flag once;
  static double ms = 60000.0;
  std::call_once(once, [] {
    if (const char* e = std::getenv("HBG_PEER_TIMEOUT_MS")) {
      const double v = std::atof(e);
      if (v > 0.0) ms = v;
    }
  });
  // the clock-rate query costs ~1 ms on this driver: once per device (a
  // racing first call just queries twice)
  static std::atomic<int> khz_of[64];
  int khz = khz_of[device & 63].load(std::memory_order_relaxed);
  if (khz <= 0) {
    if (cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device) != cudaSuccess || khz <= 0) khz = 2000000;
    khz_of[device & 63].store(khz, std::memory_order_relaxed);
  }
  return static_cast<long long>(ms * static_cast<double>(khz));
}


namespace {

void check_ds(const hbg_dataset* ds) { require(ds != nullptr, "null dataset handle"); }

// Device entry points run on the caller's stream; NULL is the CUDA legacy
// default stream (as everywhere in CUDA). The handle's own stream serves only
// the synchronous host drop-in.
cudaStream_t pick(hbg_dataset*, void* stream) { return static_cast<cudaStream_t>(stream); }


// ---- pageable host inputs -----------------------------------------------------
// The reference's LeafState arrays are std::vectors: pageable memory, which a
// cudaMemcpy moves through the driver's bounce buffers at ~11 GB/s (15-16 ms
// for the 168 MB of fp64 g/h of the 10.5M-row leaf vs 3.0 ms pinned,
// microbench/h2d_convert.cu). For such inputs the host pool converts fp64 ->
// fp32 (round to nearest: the same floats the device conversion makes) into a
// pinned stage chunk by chunk and the copy engine moves each finished chunk at
// once: 8 B/row over PCIe, the conversion (host-memory bound, ~4.3 G rows/s on
// 16 threads) the only exposed cost.
bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // (an unknown pointer is pageable; clear the sticky error)
    return false;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeManaged;
}

// A fixed pool of host workers (one per core up to 16), created on first use.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  int size() const { return static_cast<int>(th_.size()); }
  // One job at a time: callers on different threads (different handles, or
  // ctypes callers that released the GIL) hold job_mutex() from run() through
  // wait(), so a second job can never overwrite job_/pending_ while workers of
  // the first one are still picking it up.
  std::mutex& job_mutex() { return job_m_; }
  // fn(w) on every worker w; returns at once (wait() blocks until all finish)
  void run(std::function<void(int)> fn) {
    std::unique_lock<std::mutex> lk(m_);
    job_ = std::move(fn);
    pending_ = size();
    ++gen_;
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return pending_ == 0; });
  }
  ~HostPool() {
    {
      std::unique_lock<std::mutex> lk(m_);
      stop_ = true;
      cv_.notify_all();
    }
    for (auto& t : th_) t.join();
  }

 private:
  HostPool() {
    // one core stays with the calling thread, which issues the copies
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    int T = static_cast<int>(std::min<unsigned>(16, hw - 1));
    if (const char* e = std::getenv("HBG_HOST_THREADS")) T = std::max(1, std::min(64, std::atoi(e)));
    for (int w = 0; w < T; ++w) th_.emplace_back([this, w] { loop(w); });
  }
  void loop(int w) {
    uint64_t seen = 0;
    for (;;) {
      std::function<void(int)> fn;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        fn = job_;
      }
      fn(w);
      std::unique_lock<std::mutex> lk(m_);
      if (--pending_ == 0) done_.notify_all();
    }
  }
  std::mutex m_;
  std::mutex job_m_;
  std::condition_variable cv_, done_;
  std::function<void(int)> job_;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
  std::vector<std::thread> th_;
};

void* stage_buffer(hbg_dataset* ds, size_t bytes) {
  if (ds->stage_bytes < bytes) {
    if (ds->stage) {
      HBG_CUDA(cudaStreamSynchronize(ds->stream));
      if (ds->copy_stream) HBG_CUDA(cudaStreamSynchronize(ds->copy_stream));
      HBG_CUDA(cudaFreeHost(ds->stage));
      ds->stage = nullptr;
      ds->stage_bytes = 0;
    }
    HBG_CUDA(cudaHostAlloc(&ds->stage, bytes, cudaHostAllocDefault));
    ds->stage_bytes = bytes;
  }
  return ds->stage;
}

// Host staging stores (x86-64: SSE2 is baseline) — non-temporal, so the
// pinned stage lines are not read into the cache before being overwritten.
inline void convert_stream(const double* src, float* dst, int64_t n) {
  int64_t i = 0;
#if defined(__SSE2__)
  for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 15) != 0; ++i) dst[i] = static_cast<float>(src[i]);
  for (; i + 4 <= n; i += 4) {
    const __m128 lo = _mm_cvtpd_ps(_mm_loadu_pd(src + i));
    const __m128 hi = _mm_cvtpd_ps(_mm_loadu_pd(src + i + 2));
    _mm_stream_ps(dst + i, _mm_movelh_ps(lo, hi));
  }
#endif
  for (; i < n; ++i) dst[i] = static_cast<float>(src[i]);
}
inline void convert_stream(const double* src, double* dst, int64_t n) {  // bits64: a plain copy
  int64_t i = 0;
#if defined(__SSE2__)
  for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 15) != 0; ++i) dst[i] = src[i];
  for (; i + 2 <= n; i += 2) _mm_stream_pd(dst + i, _mm_loadu_pd(src + i));
#endif
  for (; i < n; ++i) dst[i] = src[i];
}
inline void copy_stream(const int32_t* src, int32_t* dst, int64_t n) {
  int64_t i = 0;
#if defined(__SSE2__)
  for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 15) != 0; ++i) dst[i] = src[i];
  for (; i + 4 <= n; i += 4)
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i)));
#endif
  for (; i < n; ++i) dst[i] = src[i];
}
inline void store_fence() {
#if defined(__SSE2__)
  _mm_sfence();
#endif
}

// Stage rows [0, n) of fp64 g/h (and, when idx != nullptr, the int32 row ids)
// into the pinned stage as Out (g | h | idx; float: the bits32 cast, double:
// a copy for bits64), in chunks of `chunk` rows
// converted by the host pool (chunks with direct[c] set are only checked:
// their g/h go up as fp64 straight from pinned caller memory); copy(c, b, e, gf, hf, id, contiguous) runs on
// the calling thread, in chunk order, as soon as chunk c is staged;
// `contiguous` says chunk c's ids are idx[0] + i (checked by the staging pass,
// which then stores no ids for it); a copy() that uploads ids of chunk c
// first calls fill_ids(c). Returns after the last copy was issued.
template <typename Out = float, typename Copy>
void stage_chunks(hbg_dataset* ds, const double* g, const double* h, const int32_t* idx, int64_t n, int64_t chunk,
                  const std::vector<char>& direct, Copy copy) {
  const size_t rows = static_cast<size_t>(n);
  char* st = static_cast<char*>(stage_buffer(ds, rows * (2 * sizeof(Out) + (idx ? 4 : 0)) + 64));
  Out* gf = reinterpret_cast<Out*>(st);
  Out* hf = gf + rows;
  int32_t* id = reinterpret_cast<int32_t*>(hf + rows);
  const int C = static_cast<int>((n + chunk - 1) / chunk);
  HostPool& pool = HostPool::get();
  std::lock_guard<std::mutex> job(pool.job_mutex());  // held until the last pool.wait()
  const int T = pool.size();
  const int64_t first = idx && n > 0 ? idx[0] : 0;
  // done[c]: workers finished with chunk c; broken[c]: some id of chunk c is
  // not first + i (the chunk is not a piece of one contiguous row range)
  std::unique_ptr<std::atomic<int>[]> done(new std::atomic<int>[static_cast<size_t>(3 * C)]);
  std::atomic<int>* broken = done.get() + C;
  std::atomic<int>* outside = done.get() + 2 * C;  // some id of chunk c is not a row of the dataset
  for (int c = 0; c < 3 * C; ++c) done[static_cast<size_t>(c)].store(0, std::memory_order_relaxed);
  const uint32_t limit = static_cast<uint32_t>(ds->layout.num_rows);
  static const bool prof = std::getenv("HBG_STAGE_PROFILE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto us = [&] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(); };
  // written[c*T + w]: worker w stored its slice of chunk c's ids (it does so
  // only when the slice is not first + i; copy() never needs a slice that
  // passed unless its chunk's histogram reads uploaded ids: fill_ids below)
  std::vector<char> written(static_cast<size_t>(C) * T, 0);
  pool.run([&, C, T](int w) {
    for (int c = 0; c < C; ++c) {
      const int64_t b = chunk * c, e = std::min<int64_t>(n, b + chunk);
      const int64_t s0 = b + (e - b) * w / T, s1 = b + (e - b) * (w + 1) / T;
      // the stage is read by the copy engine only: streaming stores (no
      // read-for-ownership of the destination lines)
      if (!direct[static_cast<size_t>(c)]) {
        convert_stream(g + s0, gf + s0, s1 - s0);
        convert_stream(h + s0, hf + s0, s1 - s0);
      }
      if (idx) {
        bool bad = false, oor = false;
        for (int64_t i = s0; i < s1; ++i) {
          bad |= static_cast<int64_t>(idx[i]) != first + i;
          oor |= static_cast<uint32_t>(idx[i]) >= limit;  // negative ids wrap above the limit
        }
        if (oor) outside[c].store(1, std::memory_order_relaxed);
        if (bad) {
          copy_stream(idx + s0, id + s0, s1 - s0);
          written[static_cast<size_t>(c) * T + w] = 1;
          broken[c].store(1, std::memory_order_relaxed);
        }
      }
      store_fence();
      done[static_cast<size_t>(c)].fetch_add(1, std::memory_order_release);
    }
  });
  // ids of chunk c in the stage, for a copy() that uploads them: the slices
  // the workers skipped are first + i
  auto fill_ids = [&](int c) {
    const int64_t b = chunk * c, e = std::min<int64_t>(n, b + chunk);
    for (int w = 0; w < T; ++w) {
      char& f = written[static_cast<size_t>(c) * T + w];
      if (f) continue;
      const int64_t s0 = b + (e - b) * w / T, s1 = b + (e - b) * (w + 1) / T;
      for (int64_t i = s0; i < s1; ++i) id[i] = static_cast<int32_t>(first + i);
      f = 1;
    }
  };
  double t_first = 0, t_last = 0;
  try {
    for (int c = 0; c < C; ++c) {
      while (done[static_cast<size_t>(c)].load(std::memory_order_acquire) < T) std::this_thread::yield();
      if (prof) (c == 0 ? t_first : t_last) = us();
      if (outside[c].load(std::memory_order_relaxed))
        throw Error(HBG_ERR_INVALID_ARGUMENT, "leaf row index out of range");
      const int64_t b = chunk * c, e = std::min<int64_t>(n, b + chunk);
      copy(c, b, e, gf, hf, id, idx != nullptr && broken[c].load(std::memory_order_relaxed) == 0, fill_ids);
    }
  } catch (...) {
    pool.wait();  // the workers still use `done` and the stage
    // copies already issued may still read the stage or the caller's pinned
    // arrays: let them finish before the caller gets control back
    if (ds->copy_stream) (void)cudaStreamSynchronize(ds->copy_stream);
    (void)cudaStreamSynchronize(ds->stream);
    (void)cudaGetLastError();
    throw;
  }
  const double t_issue = prof ? us() : 0;
  pool.wait();
  if (prof)
    std::fprintf(stderr, "[hbg stage] rows=%lld chunks=%d threads=%d: chunk0 %.0f us, last chunk %.0f us, issued %.0f us, joined %.0f us\n",
                 static_cast<long long>(n), C, T, t_first, t_last, t_issue, us());
}

constexpr int64_t kStageRows = int64_t(1) << 19;  // rows per staged chunk (4 MB of fp32 g/h)

// Histogram chunks of a host drop-in call: only the last chunk's conversion
// and histogram are exposed after the PCIe copies.
int host_chunks(int64_t count) {
  const char* e = std::getenv("HBG_HOST_CHUNKS");
  if (e != nullptr) return std::max(1, std::min(16, std::atoi(e)));
  return count >= (int64_t{1} << 21) ? 4 : 1;
}

// Staged chunks copied as fp64 straight from pinned caller memory (the rest
// are converted to fp32 by the host pool first): a fraction f of them,
// spread evenly, starting with chunk 0 so the copy engine starts at once.
// f balances host memory traffic (32 B/row converted, 16 B/row direct)
// against PCIe (8 vs 16 B/row); HBG_PINNED_DMA_FRAC overrides it.
std::vector<char> direct_chunks(int64_t n, int64_t chunk, bool pinned) {
  const int C = static_cast<int>((n + chunk - 1) / chunk);
  std::vector<char> d(static_cast<size_t>(C), 0);
  if (!pinned) return d;  // pageable memory crosses PCIe at a fraction of the pinned rate
  static const double f = [] {
    const char* e = std::getenv("HBG_PINNED_DMA_FRAC");
    return e ? std::max(0.0, std::min(1.0, std::atof(e))) : 0.25;
  }();
  for (int c = 0; c < C; ++c) d[static_cast<size_t>(c)] = std::ceil((c + 1) * f) > std::ceil(c * f);
  return d;
}

// Device row ids [first, first + n) of the dataset: the resident iota array.
const int32_t* identity_rows(hbg_dataset* ds, int64_t first, cudaStream_t s) {
  const int64_t N = ds->layout.num_rows;
  if (ds->iota_rows < N) {
    int32_t* io = static_cast<int32_t*>(ds->iota.get(static_cast<size_t>(N) * 4 + 4));
    launch_iota(io, N, s);
    ds->iota_rows = N;
  }
  return static_cast<const int32_t*>(ds->iota.p) + first;
}

// Device histogram of one leaf into d_hist; with `parent` also writes
// sibling = parent - d_hist in the same pass (sibling may alias parent).
// acc_bytes 4: d_g/d_h are fp32 (bits32); 8: fp64 with fp64 accumulation (bits64).
// allow_fused: the leaf may take the single-launch cluster mode (histogram +
// DSMEM reduction in one kernel). Off where ranks share a GPU and wait on each
// other inside kernels (a cluster could wait for SMs a waiting grid holds).
void build_device(hbg_dataset* ds, const int32_t* d_idx, int64_t count, const void* d_g,
                  const void* d_h, int gh_mode, double* d_hist, cudaStream_t s,
                  const double* parent = nullptr, double* sibling = nullptr, int acc_bytes = 4,
                  bool allow_fused = false) {
  const hbg_layout& L = ds->layout;
  require(count >= 0, "negative leaf size");
  require(count <= L.num_rows || d_idx != nullptr, "identity leaf larger than the dataset");
  require(gh_mode == HBG_GH_LEAF_ALIGNED || gh_mode == HBG_GH_ROW_INDEXED, "bad gh_mode");
  require(d_hist != nullptr, "null histogram output");
  const size_t D = static_cast<size_t>(L.num_features) * L.max_bin;
  if (count == 0 || L.num_features == 0) {
    HBG_CUDA(cudaMemsetAsync(d_hist, 0, 3 * D * sizeof(double), s));
    if (parent && sibling != parent)
      HBG_CUDA(cudaMemcpyAsync(sibling, parent, 3 * D * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return;
  }
  require(d_g != nullptr && d_h != nullptr, "null gradient/hessian pointer");
  if (d_idx == nullptr) d_idx = identity_rows(ds, 0, s);  // identity leaf [0, count)
  HistPlan plan = plan_histogram(L.bits_per_bin, L.max_bin, L.num_groups, count, L.device, true, acc_bytes,
                                 allow_fused);
  if (std::getenv("HBG_PLAN_DEBUG"))  // development aid
    std::fprintf(stderr, "[hbg plan] n=%lld ctas=%d warps=%d wpg=%d gb=%d nseg=%d seg_len=%lld cluster=%d x %d smem=%zu\n",
                 static_cast<long long>(count), plan.ctas, plan.warps, plan.wpg, plan.gb, plan.nseg,
                 static_cast<long long>(plan.seg_len), plan.cluster, plan.nclusters, plan.smem);
  char* part = static_cast<char*>(ds->part.get(hist_part_bytes(plan)));
  HistArgs a{};
  a.packed = reinterpret_cast<const uint8_t*>(ds->packed);
  a.row_stride = L.row_stride_bytes;
  a.group_stride = L.group_stride_bytes;
  a.idx = d_idx;
  a.n = count;
  a.g = d_g;
  a.h = d_h;
  a.gh_indexed = gh_mode == HBG_GH_ROW_INDEXED;
  a.num_groups = L.num_groups;
  a.gb = plan.gb;
  a.wpg = plan.wpg;
  a.nblocks = plan.nblocks;
  a.seg_len = plan.seg_len;
  a.part_g = part;
  a.part_h = part + plan.part_values * part_elem_bytes(plan);
  a.part_c = reinterpret_cast<uint32_t*>(part + 2 * plan.part_values * part_elem_bytes(plan));
  a.direct = plan.nseg == 1 ? 1 : 0;
  a.d = L.num_features;
  a.max_bin = L.max_bin;
  a.out = d_hist;
  a.parent = parent;
  a.sibling = sibling;
  a.nseg = plan.nseg;
  a.cluster = plan.cluster;
  a.nclusters = plan.nclusters;
  static const bool prof = std::getenv("HBG_HIST_PROFILE") != nullptr;  // development aid
  if (prof) {
    a.prof = static_cast<unsigned long long*>(ds->hist_prof.get(64));
    HBG_CUDA(cudaMemsetAsync(a.prof, 0, 64, s));
    static const int cta = std::getenv("HBG_HIST_PROFILE_CTA") ? std::atoi(std::getenv("HBG_HIST_PROFILE_CTA")) : 0;
    a.prof_cta = std::min(cta, plan.ctas - 1);
  }
  if (plan.nclusters > 1) {  // counters zeroed once; every launch leaves them 0
    const size_t need = static_cast<size_t>(std::max(plan.nblocks, 1)) * sizeof(unsigned) + 64;
    if (ds->hist_bar.bytes < need) {
      ds->hist_bar.get(need);
      HBG_CUDA(cudaMemsetAsync(ds->hist_bar.p, 0, ds->hist_bar.bytes, s));
    }
    a.bar = static_cast<unsigned*>(ds->hist_bar.p);
  }
  if (ds->profiling) {
    auto ev = ds->event_pair();
    HBG_CUDA(cudaEventRecord(ev.first, s));
    launch_histogram(plan, a, s);
    HBG_CUDA(cudaEventRecord(ev.second, s));
    ds->events.push_back(ev);
  } else {
    launch_histogram(plan, a, s);
  }
  if (!a.direct && a.cluster <= 1) launch_reduce_partials(plan, a, L.num_features, L.max_bin, d_hist, s, parent, sibling);
}

// Row-sharded histogram of one leaf: this rank's rows, the cross-rank sum
// fused into the reduction over peer memory (reduce_exchange_kernel); every
// rank must call it (a rank without rows of the leaf still exchanges).
void build_device_peer(hbg_dataset* ds, const int32_t* d_idx, int64_t count, const float* d_g, const float* d_h,
                       int gh_mode, double* d_hist, cudaStream_t s, hbg_peer* peer) {
  const hbg_layout& L = ds->layout;
  require(count >= 0, "negative leaf size");
  require(count <= L.num_rows || d_idx != nullptr, "identity leaf larger than the dataset");
  require(gh_mode == HBG_GH_LEAF_ALIGNED || gh_mode == HBG_GH_ROW_INDEXED, "bad gh_mode");
  require(d_hist != nullptr, "null histogram output");
  require(peer->device == L.device, "exchange area on another device");
  for (int r = 0; r < peer->nranks; ++r) require(peer->peers[r] != nullptr, "exchange area of a rank not attached");
  require(count == 0 || (d_g != nullptr && d_h != nullptr), "null gradient/hessian pointer");
  if (d_idx == nullptr && count > 0) d_idx = identity_rows(ds, 0, s);
  HistPlan plan = plan_histogram(L.bits_per_bin, L.max_bin, L.num_groups, std::max<int64_t>(count, 1), L.device,
                                 /*allow_direct=*/false);
  // No allocation on this path: a cudaMalloc/cudaFree here can wait for
  // another rank's reduction, which spins on this rank's rows (ranks sharing
  // a GPU). The partials were reserved by hbg_peer_create; a plan that would
  // need more takes fewer, longer row segments instead.
  if (hist_part_bytes(plan) > ds->part.bytes && ds->part.bytes > 0) {
    const size_t per_seg = static_cast<size_t>(plan.nblocks) * plan.gb * plan.k_alloc * 32;
    const size_t fit = std::max<size_t>(1, (ds->part.bytes - 16) / (per_seg * (2 * part_elem_bytes(plan) + 4)));
    const int64_t n = std::max<int64_t>(count, 1);
    int64_t seg_len = (n + static_cast<int64_t>(fit) - 1) / static_cast<int64_t>(fit);
    seg_len = (seg_len + 31) / 32 * 32;
    plan.seg_len = seg_len;
    plan.nseg = static_cast<int>((n + seg_len - 1) / seg_len);
    plan.ctas = plan.nblocks * plan.nseg;
    plan.part_values = static_cast<size_t>(plan.ctas) * plan.gb * plan.k_alloc * 32;
  }
  char* part = static_cast<char*>(ds->part.get(hist_part_bytes(plan)));
  HistArgs a{};
  a.packed = reinterpret_cast<const uint8_t*>(ds->packed);
  a.row_stride = L.row_stride_bytes;
  a.group_stride = L.group_stride_bytes;
  a.idx = d_idx;
  a.n = count;
  a.g = d_g;
  a.h = d_h;
  a.gh_indexed = gh_mode == HBG_GH_ROW_INDEXED;
  a.num_groups = L.num_groups;
  a.gb = plan.gb;
  a.wpg = plan.wpg;
  a.nblocks = plan.nblocks;
  a.seg_len = plan.seg_len;
  a.part_g = part;
  a.part_h = part + plan.part_values * plan.acc_bytes;
  a.part_c = reinterpret_cast<uint32_t*>(part + 2 * plan.part_values * plan.acc_bytes);
  a.d = L.num_features;
  a.max_bin = L.max_bin;
  if (count > 0) {
    if (ds->profiling) {  // the histogram kernel's own time (bench.py's roofline), as build_device
      auto ev = ds->event_pair();
      HBG_CUDA(cudaEventRecord(ev.first, s));
      launch_histogram(plan, a, s);
      HBG_CUDA(cudaEventRecord(ev.second, s));
      ds->events.push_back(ev);
    } else {
      launch_histogram(plan, a, s);
    }
  } else {
    plan.nseg = 0;  // nothing of this rank's; still publish zeros and sum
  }
  PeerHistArgs x{};
  x.nranks = peer->nranks;
  x.rank = peer->rank;
  x.xown = peer->xbuf + peer->hoff;
  for (int r = 0; r < peer->nranks; ++r) x.xpeer[r] = peer->peers[r] + peer->hoff;
  x.tag = ++peer->hgen;
  x.parity = static_cast<int>(x.tag & 1);
  x.error = peer->error;
  x.timeout_cycles = wait_timeout_cycles(L.device);
  launch_reduce_exchange(plan, a, L.num_features, L.max_bin, d_hist, x, s);
}

double leaf_value(double g, double h, double lambda) {  // tree.cpp:59-64
  const double denom = h + lambda;
  return denom <= 0.0 ? 0.0 : -g / denom;
}

struct OpenLeaf {  // tree.cpp:132-136
  int node;
  int buf;
  int64_t begin, count;  // this rank's rows of the leaf: [begin, begin+count) of buffer `buf`
  int64_t gcount;        // rows of the leaf over all ranks
  double grad, hess;     // global totals
  int slot;
  bool has_best;
  hbg_split best;
};

// Per-split device results copied back in one transfer.
struct SplitResults {
  hbg_split split[2];
  double totals[4];  // gl, hl, gr, hr (children of the split just executed; global)
  int64_t left;      // this rank's rows sent left
  double root[3];    // root grad, hess, rows (global)
};

// Row-sharded growth: every rank holds its own rows; the leaf
// histograms and totals are summed across ranks by `allreduce` (NCCL in
// production, hbg_comm_allreduce), so every rank scans identical histograms
// and takes identical decisions. allreduce == nullptr: single rank.
struct Reducer {
  hbg_allreduce_fn fn;
  void* ctx;
  void operator()(double* buf, int64_t n, cudaStream_t s) const {
    if (!fn) return;
    const int st = fn(buf, n, s, ctx);
    if (st != HBG_OK) throw Error(st, std::string("allreduce hook failed: ") + hbg_last_error());
  }
};

// d_grad/d_hess: fp32 (P.precision == HBG_PRECISION_BITS32) or fp64
// (HBG_PRECISION_BITS64: fp64 ordered buffers, partitions and fp64-accumulated
// histograms for every leaf — the reference's reference_impl<double>).
void grow_tree_impl(hbg_dataset* ds, const void* d_grad, const void* d_hess,
                    const hbg_grow_params& P, const Reducer& reduce, hbg_split* split_log,
                    int32_t* num_splits, hbg_tree_node* nodes_out, int32_t* num_nodes, cudaStream_t s,
                    std::vector<LeafRange>* final_leaves = nullptr) {
  const hbg_layout& L = ds->layout;
  require(P.num_leaves >= 1, "num_leaves must be at least 1");
  require(P.min_data_in_leaf >= 0, "min_data_in_leaf must be non-negative");
  require(P.precision == HBG_PRECISION_BITS32 || P.precision == HBG_PRECISION_BITS64, "unknown precision");
  const bool f64 = P.precision == HBG_PRECISION_BITS64;
  const size_t es = f64 ? 8 : 4;  // bytes per g/h element
  const bool sharded = reduce.fn != nullptr;
  const int64_t N = L.num_rows;
  const int d = L.num_features, k = L.max_bin;
  const size_t D3 = 3 * static_cast<size_t>(d) * k;
  const int max_slots = std::max(1, P.num_leaves);
  double* slots = static_cast<double*>(ds->slots.get(max_slots * D3 * sizeof(double) + 8));
  int32_t* rows[2];
  char* gb[2];
  char* hb[2];
  for (int b = 0; b < 2; ++b) {
    rows[b] = static_cast<int32_t*>(ds->ord[b][0].get(static_cast<size_t>(N) * 4 + 4));
    gb[b] = static_cast<char*>(ds->ord[b][1].get(static_cast<size_t>(N) * es + 8));
    hb[b] = static_cast<char*>(ds->ord[b][2].get(static_cast<size_t>(N) * es + 8));
  }
  auto G = [&](int b, int64_t i) { return gb[b] + static_cast<size_t>(i) * es; };
  auto H = [&](int b, int64_t i) { return hb[b] + static_cast<size_t>(i) * es; };
  void* scratch = ds->part_scratch.get(std::max(partition_scratch_bytes(N),
                                                gather_scratch_doubles(N) * sizeof(double)) + 64);
  SplitResults* dres = static_cast<SplitResults*>(ds->tree_small.get(sizeof(SplitResults)));
  if (!ds->pinned) HBG_CUDA(cudaMallocHost(&ds->pinned, sizeof(SplitResults)));
  SplitResults* hres = static_cast<SplitResults*>(ds->pinned);

  std::vector<hbg_tree_node> nodes;
  nodes.reserve(static_cast<size_t>(2 * P.num_leaves));
  std::vector<int> free_slots;
  for (int i = max_slots - 1; i >= 0; --i) free_slots.push_back(i);
  auto slot_ptr = [&](int i) { return slots + static_cast<size_t>(i) * D3; };
  auto splittable = [&](int64_t n) { return !(n < 2 * P.min_data_in_leaf || n < 2); };
  auto sync_results = [&] {
    HBG_CUDA(cudaMemcpyAsync(hres, dres, sizeof(SplitResults), cudaMemcpyDeviceToHost, s));
    HBG_CUDA(cudaStreamSynchronize(s));
  };

  // Root: ordered buffer 0 = (iota, g, h); totals in a fixed order; global
  // totals and row count (summed across ranks).
  launch_iota(rows[0], N, s);
  if (N > 0) {
    HBG_CUDA(cudaMemcpyAsync(gb[0], d_grad, static_cast<size_t>(N) * es, cudaMemcpyDeviceToDevice, s));
    HBG_CUDA(cudaMemcpyAsync(hb[0], d_hess, static_cast<size_t>(N) * es, cudaMemcpyDeviceToDevice, s));
  }
  if (f64)
    launch_gather_f64(rows[0], N, static_cast<const double*>(d_grad), static_cast<const double*>(d_hess), nullptr,
                      nullptr, dres->root, static_cast<double*>(scratch), s);
  else
    launch_gather(rows[0], N, static_cast<const float*>(d_grad), static_cast<const float*>(d_hess), nullptr,
                  nullptr, dres->root, static_cast<double*>(scratch), s);
  // bits32 small-leaf histogram path: accumulator cleared once (the finish
  // kernel clears it after every leaf), fixed-point scales per leaf (bits64
  // builds every leaf with fp64 accumulation instead)
  int* exps = static_cast<int*>(ds->small_exps.get(16));
  void* acc = ds->small_acc.get(small_hist_acc_bytes(d, k));
  if (!f64) HBG_CUDA(cudaMemsetAsync(acc, 0, small_hist_acc_bytes(d, k), s));
  const uint32_t* packed = ds->packed;
  const int64_t stride_words = L.group_stride_bytes / 4;  // group stride, in words
  const int acc_bytes = f64 ? 8 : 4;
  // histogram of one leaf range into `out` (+ sibling = parent - out)
  auto leaf_hist = [&](int buf, int64_t begin, int64_t count, double* out, const double* parent,
                       double* sibling) {
    if (!f64 && count <= kAtomicHistRows) {
      launch_fixed_leaf_scale(reinterpret_cast<const float*>(G(buf, begin)), reinterpret_cast<const float*>(H(buf, begin)),
                              count, exps, s);
      launch_small_hist(rows[buf] + begin, reinterpret_cast<const float*>(G(buf, begin)),
                        reinterpret_cast<const float*>(H(buf, begin)), count, packed, stride_words,
                        L.words_per_row, L.bits_per_bin, d, k, exps, acc, out, parent, sibling, s);
    } else {
      build_device(ds, rows[buf] + begin, count, G(buf, begin), H(buf, begin), HBG_GH_LEAF_ALIGNED, out, s, parent,
                   sibling, acc_bytes);
    }
  };
  hres->root[2] = static_cast<double>(N);  // pinned staging; the stream orders the copy
  HBG_CUDA(cudaMemcpyAsync(&dres->root[2], &hres->root[2], sizeof(double), cudaMemcpyHostToDevice, s));
  reduce(dres->root, 3, s);
  sync_results();
  const int64_t NG = static_cast<int64_t>(hres->root[2]);
  std::vector<OpenLeaf> pool;
  OpenLeaf root{0, 0, 0, N, NG, hres->root[0], hres->root[1], -1, false, {}};
  nodes.push_back(hbg_tree_node{-1, -1, -1, -1, leaf_value(root.grad, root.hess, P.lambda)});
  if (P.num_leaves >= 2) {
    if (splittable(NG)) {
      root.slot = free_slots.back();
      free_slots.pop_back();
      build_device(ds, rows[0], N, gb[0], hb[0], HBG_GH_LEAF_ALIGNED, slot_ptr(root.slot), s, nullptr, nullptr,
                   acc_bytes);
      reduce(slot_ptr(root.slot), static_cast<int64_t>(D3), s);
      launch_best_split(slot_ptr(root.slot), d, k, dres->root, nullptr, 0.0, 0.0, NG,
                        P.min_data_in_leaf, P.lambda, &dres->split[0], s);
      sync_results();
      root.has_best = hres->split[0].feature >= 0;
      root.best = hres->split[0];
    }
    pool.push_back(root);
  }

  int leaves = 1, logged = 0;
  while (leaves < P.num_leaves) {
    int pick = -1;
    for (size_t i = 0; i < pool.size(); ++i) {  // strict >: the oldest leaf wins ties (tree.cpp:212-218)
      if (!pool[i].has_best) continue;
      if (pick < 0 || pool[i].best.gain > pool[static_cast<size_t>(pick)].best.gain) pick = static_cast<int>(i);
    }
    if (pick < 0) break;
    OpenLeaf parent = pool[static_cast<size_t>(pick)];
    pool.erase(pool.begin() + pick);
    const hbg_split& sp = parent.best;
    split_log[logged++] = sp;

    const int out = 1 - parent.buf;
    const int64_t gl_n = sp.left_count, gr_n = parent.gcount - sp.left_count;  // global sizes
    if (gl_n <= 0 || gr_n <= 0) throw Error(HBG_ERR_LOGIC, "split produced an empty side");
    if (f64)
      launch_partition_f64(rows[parent.buf] + parent.begin, reinterpret_cast<const double*>(G(parent.buf, parent.begin)),
                           reinterpret_cast<const double*>(H(parent.buf, parent.begin)), parent.count,
                           reinterpret_cast<const uint8_t*>(ds->packed) + (sp.feature / 32) * L.group_stride_bytes,
                           L.row_stride_bytes, sp.feature % 32,
                           L.bits_per_bin, sp.threshold_bin, rows[out] + parent.begin,
                           reinterpret_cast<double*>(G(out, parent.begin)), reinterpret_cast<double*>(H(out, parent.begin)),
                           scratch, dres->totals, &dres->left, s);
    else
      launch_partition(rows[parent.buf] + parent.begin, reinterpret_cast<const float*>(G(parent.buf, parent.begin)),
                       reinterpret_cast<const float*>(H(parent.buf, parent.begin)), parent.count,
                       reinterpret_cast<const uint8_t*>(ds->packed) + (sp.feature / 32) * L.group_stride_bytes,
                       L.row_stride_bytes, sp.feature % 32,
                       L.bits_per_bin, sp.threshold_bin, rows[out] + parent.begin,
                       reinterpret_cast<float*>(G(out, parent.begin)), reinterpret_cast<float*>(H(out, parent.begin)),
                       scratch, dres->totals, &dres->left, s);
    reduce(dres->totals, 4, s);  // global child totals
    int64_t nl_local = gl_n;
    if (sharded) {  // this rank's left count is needed before the children can be addressed
      HBG_CUDA(cudaMemcpyAsync(&hres->left, &dres->left, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      HBG_CUDA(cudaStreamSynchronize(s));
      nl_local = hres->left;
    }

    const int left_id = static_cast<int>(nodes.size()), right_id = left_id + 1;
    hbg_tree_node& pn = nodes[static_cast<size_t>(parent.node)];
    pn.feature = sp.feature;
    pn.threshold_bin = sp.threshold_bin;
    pn.left = left_id;
    pn.right = right_id;
    pn.value = 0.0;
    nodes.push_back(hbg_tree_node{-1, -1, -1, -1, 0.0});
    nodes.push_back(hbg_tree_node{-1, -1, -1, -1, 0.0});
    ++leaves;

    OpenLeaf lo{left_id, out, parent.begin, nl_local, gl_n, 0.0, 0.0, -1, false, {}};
    OpenLeaf ro{right_id, out, parent.begin + nl_local, parent.count - nl_local, gr_n, 0.0, 0.0, -1,
                false, {}};
    const bool scan = leaves < P.num_leaves;
    const bool lsplit = scan && splittable(gl_n), rsplit = scan && splittable(gr_n);
    if (lsplit || rsplit) {
      // histogram of the globally smaller child; the larger = parent - smaller
      // in the parent's slot (ties build the left child)
      OpenLeaf& small = gl_n <= gr_n ? lo : ro;
      OpenLeaf& large = gl_n <= gr_n ? ro : lo;
      small.slot = free_slots.back();
      free_slots.pop_back();
      large.slot = parent.slot;
      parent.slot = -1;
      if (!f64 && !sharded && small.count <= kAtomicHistRows) {
        // small child: L2-atomic histogram, then one fused launch for the
        // conversion, the subtraction and both children's scans
        launch_fixed_leaf_scale(reinterpret_cast<const float*>(G(out, small.begin)),
                                reinterpret_cast<const float*>(H(out, small.begin)), small.count, exps, s);
        launch_small_hist_atomic(rows[out] + small.begin, reinterpret_cast<const float*>(G(out, small.begin)),
                                 reinterpret_cast<const float*>(H(out, small.begin)), small.count, packed,
                                 stride_words, L.words_per_row, L.bits_per_bin, d, k, exps, acc, s);
        FinishScanArgsHost fa{acc, exps, d, k, slot_ptr(small.slot), slot_ptr(large.slot),
                              &small == &lo ? 1 : 0, dres->totals, gl_n, gr_n, lsplit ? 1 : 0,
                              rsplit ? 1 : 0, P.min_data_in_leaf, P.lambda, &dres->split[0]};
        launch_finish_scan(fa, s);
        goto scanned;
      }
      if (!sharded) {
        leaf_hist(out, small.begin, small.count, slot_ptr(small.slot), slot_ptr(large.slot),
                  slot_ptr(large.slot));  // subtraction fused
      } else {
        leaf_hist(out, small.begin, small.count, slot_ptr(small.slot), nullptr, nullptr);
        reduce(slot_ptr(small.slot), static_cast<int64_t>(D3), s);  // global smaller child
        launch_subtract(slot_ptr(large.slot), slot_ptr(small.slot), slot_ptr(large.slot),
                        static_cast<int64_t>(D3), s);
      }
      if (lsplit && rsplit) {  // both children's scans in one launch
        launch_best_split_batch(slot_ptr(lo.slot), slot_ptr(ro.slot) - slot_ptr(lo.slot), 2, d, k,
                                dres->totals, 2, nullptr, gl_n, gr_n, 0.0, 0.0, P.min_data_in_leaf,
                                P.lambda, &dres->split[0], s);
      } else if (lsplit) {
        launch_best_split(slot_ptr(lo.slot), d, k, dres->totals, nullptr, 0.0, 0.0, gl_n,
                          P.min_data_in_leaf, P.lambda, &dres->split[0], s);
      } else {
        launch_best_split(slot_ptr(ro.slot), d, k, dres->totals + 2, nullptr, 0.0, 0.0, gr_n,
                          P.min_data_in_leaf, P.lambda, &dres->split[1], s);
      }
    scanned:;
    }
    if (parent.slot >= 0) free_slots.push_back(parent.slot);
    sync_results();
    if (!sharded && hres->left != gl_n)
      throw Error(HBG_ERR_LOGIC, "partition disagrees with the histogram counts");
    lo.grad = hres->totals[0];
    lo.hess = hres->totals[1];
    ro.grad = hres->totals[2];
    ro.hess = hres->totals[3];
    nodes[static_cast<size_t>(left_id)].value = leaf_value(lo.grad, lo.hess, P.lambda);
    nodes[static_cast<size_t>(right_id)].value = leaf_value(ro.grad, ro.hess, P.lambda);
    lo.has_best = lsplit && hres->split[0].feature >= 0;
    lo.best = hres->split[0];
    ro.has_best = rsplit && hres->split[1].feature >= 0;
    ro.best = hres->split[1];
    // a leaf that keeps no histogram cannot be split later
    if (!lo.has_best && lo.slot >= 0) free_slots.push_back(lo.slot), lo.slot = -1;
    if (!ro.has_best && ro.slot >= 0) free_slots.push_back(ro.slot), ro.slot = -1;
    pool.push_back(lo);
    pool.push_back(ro);
  }
  *num_splits = logged;
  *num_nodes = static_cast<int32_t>(nodes.size());
  if (nodes_out) std::copy(nodes.begin(), nodes.end(), nodes_out);
  if (final_leaves) {  // every row's leaf: the open leaves' row ranges
    final_leaves->clear();
    if (pool.empty()) pool.push_back(root);
    for (const OpenLeaf& l : pool) {
      const double v = nodes[static_cast<size_t>(l.node)].value;
      final_leaves->push_back(LeafRange{l.begin, l.count, v, l.buf});
    }
  }
}

// grow_tree on the device with ONE persistent kernel for all splits
// (grow_persistent.cu). The root (ordered buffers, totals, fixed-point scale,
// histogram, best split) uses the same kernels as the host loop; everything
// after it runs without host round trips. Single rank only: the row-sharded
// path exchanges histograms through the host-visible allreduce hook.
bool use_host_loop() {
  const char* e = std::getenv("HBG_GROW");
  return e != nullptr && std::strcmp(e, "host") == 0;
}

// Every device buffer of one persistent-grower call, acquired up front (and,
// for row-sharded ranks sharing a GPU, reserved at hbg_peer_create): a
// cudaMalloc/cudaFree while another rank's grid waits in an exchange would
// serialise behind it.
PersistentGrowArgs grow_workspace(hbg_dataset* ds, const hbg_grow_params& P, int ctas, int nranks) {
  const hbg_layout& L = ds->layout;
  const int64_t N = L.num_rows;
  const int d = L.num_features, k = L.max_bin;
  const size_t D3 = 3 * static_cast<size_t>(d) * k;
  const int max_out = std::max(1, 2 * P.num_leaves - 1);
  PersistentGrowArgs a{};
  a.nranks = nranks;
  a.packed = reinterpret_cast<const uint8_t*>(ds->packed);
  a.colbins = static_cast<const uint8_t*>(ds->colbins.p);
  a.row_stride = L.row_stride_bytes;
  a.group_stride = L.group_stride_bytes;
  a.words_per_row = L.words_per_row;
  a.bits = L.bits_per_bin;
  a.d = d;
  a.k = k;
  a.num_groups = L.num_groups;
  a.num_rows = N;
  a.ctas = ctas;
  a.num_leaves = P.num_leaves;
  const int max_nodes = grow_max_nodes(a, L.device);
  a.slots = static_cast<double*>(ds->slots.get(static_cast<size_t>(max_nodes) * D3 * sizeof(double) + 8));
  for (int b = 0; b < 2; ++b) {
    a.rows[b] = static_cast<int32_t*>(ds->ord[b][0].get(static_cast<size_t>(N) * 4 + 4));
    a.g[b] = static_cast<float*>(ds->ord[b][1].get(static_cast<size_t>(N) * 4 + 4));
    a.h[b] = static_cast<float*>(ds->ord[b][2].get(static_cast<size_t>(N) * 4 + 4));
  }
  a.nodes = ds->grow_nodes.get(grow_nodes_bytes(max_nodes));
  a.split_log = static_cast<hbg_split*>(ds->grow_log.get(static_cast<size_t>(max_out) * sizeof(hbg_split)));
  a.tree = static_cast<hbg_tree_node*>(ds->grow_tree.get(static_cast<size_t>(max_out) * sizeof(hbg_tree_node)));
  a.counts = static_cast<int*>(ds->grow_counts.get(8 * sizeof(int)));
  a.num_leaves = P.num_leaves;  // (sizes the scratch below)
  a.min_data = P.min_data_in_leaf;
  a.lambda = P.lambda;
  a.scratch_bytes = grow_scratch_bytes(a, L.device);
  a.scratch = ds->grow_scratch.get(a.scratch_bytes);
  a.scratch_bytes = ds->grow_scratch.bytes;
  a.root_totals = static_cast<double*>(ds->grow_root.get(4 * sizeof(double)));
  a.timeout_cycles = wait_timeout_cycles(L.device);
  ds->part_scratch.get(gather_scratch_doubles(N) * sizeof(double) + 64);
  if (N > 0 && d > 0) {  // the root histogram's partials (build_device)
    const HistPlan plan = plan_histogram(L.bits_per_bin, L.max_bin, L.num_groups, N, L.device);
    ds->part.get(hist_part_bytes(plan));
  }
  return a;
}

void grow_tree_persistent(hbg_dataset* ds, const float* d_grad, const float* d_hess, const hbg_grow_params& P,
                          hbg_split* split_log, int32_t* num_splits, hbg_tree_node* nodes_out,
                          int32_t* num_nodes, cudaStream_t s, hbg_peer* peer = nullptr) {
  const hbg_layout& L = ds->layout;
  require(P.num_leaves >= 1, "num_leaves must be at least 1");
  require(P.min_data_in_leaf >= 0, "min_data_in_leaf must be non-negative");
  require(P.precision == HBG_PRECISION_BITS32, "the persistent grower runs bits32 (fp32 g/h) trees");
  const int64_t N = L.num_rows;
  const int d = L.num_features, k = L.max_bin;
  const int max_nodes = std::max(1, 2 * P.num_leaves - 1);
  const bool sharded = peer != nullptr && peer->nranks > 1;
  PersistentGrowArgs a = grow_workspace(ds, P, sharded ? peer->ctas : 0, sharded ? peer->nranks : 1);
  double* slots = a.slots;
  double* root = const_cast<double*>(a.root_totals);
  void* gscratch = ds->part_scratch.p;

  // root: ordered buffer 0 = (iota, g, h), fp64 totals in a fixed order
  launch_iota(a.rows[0], N, s);
  if (N > 0) {
    HBG_CUDA(cudaMemcpyAsync(a.g[0], d_grad, static_cast<size_t>(N) * 4, cudaMemcpyDeviceToDevice, s));
    HBG_CUDA(cudaMemcpyAsync(a.h[0], d_hess, static_cast<size_t>(N) * 4, cudaMemcpyDeviceToDevice, s));
  }
  launch_gather(a.rows[0], N, d_grad, d_hess, nullptr, nullptr, root, static_cast<double*>(gscratch), s);
  if (sharded) {
    require(peer->device == L.device, "exchange area on another device");
    a.nranks = peer->nranks;
    a.rank = peer->rank;
    a.xown = peer->xbuf;
    for (int r = 0; r < peer->nranks; ++r) {
      require(peer->peers[r] != nullptr, "exchange area of a rank not attached");
      a.xpeer[r] = peer->peers[r];
    }
    require(grow_exchange_doubles(a, L.device) <= peer->xdoubles, "exchange area too small for this dataset");
    a.gen = ++peer->gen;
  }
  // root splittability over all ranks is decided in the kernel when sharded
  const bool root_splittable = sharded || (P.num_leaves >= 2 && !(N < 2 * P.min_data_in_leaf || N < 2));
  if (!root_splittable) {
    double tot[2] = {0.0, 0.0};
    HBG_CUDA(cudaMemcpyAsync(tot, root, sizeof tot, cudaMemcpyDeviceToHost, s));
    HBG_CUDA(cudaStreamSynchronize(s));
    if (nodes_out) nodes_out[0] = hbg_tree_node{-1, -1, -1, -1, leaf_value(tot[0], tot[1], P.lambda)};
    *num_splits = 0;
    *num_nodes = 1;
    return;
  }
  build_device(ds, a.rows[0], N, a.g[0], a.h[0], HBG_GH_LEAF_ALIGNED, slots, s, nullptr, nullptr, 4, !sharded);
  if (!sharded) {  // sharded: the kernel sums the ranks' root histograms first, then scans
    hbg_split* root_split = reinterpret_cast<hbg_split*>(static_cast<char*>(a.nodes) + grow_root_split_offset());
    launch_best_split(slots, d, k, root, nullptr, 0.0, 0.0, N, P.min_data_in_leaf, P.lambda, root_split, s);
  }
  const char* pe = std::getenv("HBG_GROW_PROFILE");
  std::vector<unsigned long long> prof;
  if (pe != nullptr) {  // phase stamps of CTA 0, printed to stderr (development aid)
    prof.assign(static_cast<size_t>(4 * max_nodes + 8) * 20, 0ull);
    a.prof = static_cast<unsigned long long*>(ds->grow_prof.get(prof.size() * 8));
    HBG_CUDA(cudaMemsetAsync(a.prof, 0, prof.size() * 8, s));
  }
  ds->grow_records = launch_grow_persistent(a, L.device, s);
  const bool waves = ds->grow_records != a.nodes;
  int counts[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  HBG_CUDA(cudaMemcpyAsync(counts, a.counts, sizeof counts, cudaMemcpyDeviceToHost, s));
  HBG_CUDA(cudaStreamSynchronize(s));
  if (counts[2] != 0) {
    static const char* what[] = {"", "grid barrier timed out", "partition disagrees with the histogram counts",
                                 "split produced an empty side", "peer exchange timed out"};
    char where[128] = "";
    if (counts[2] == 4)
      std::snprintf(where, sizeof where, " (rank %d CTA %d awaited tag %d, saw %d)", a.rank, counts[5], counts[3],
                    counts[4]);
    throw Error(counts[2] == 3 || counts[2] == 2 ? HBG_ERR_LOGIC : HBG_ERR_CUDA,
                std::string("persistent tree grower: ") + what[counts[2] % 5] + where);
  }
  *num_splits = counts[0];
  *num_nodes = counts[1];
  ds->grow_waves = waves;
  ds->grow_ranges = counts[4];
  if (a.prof != nullptr && waves) {
    HBG_CUDA(cudaMemcpy(prof.data(), a.prof, prof.size() * 8, cudaMemcpyDeviceToHost));
    // wave grower stamps: 0 start, 1 partitioned (large), 2 histogram (large), 3 chunks done,
    // 4 barrier, 5 next wave chosen; slot 7: large, 10: members, 11: splits committed before
    double tw[2][8] = {{0, 0, 0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 0, 0}};
    int nw[2] = {0, 0}, members[2] = {0, 0};
    for (int i = 0; i < counts[3]; ++i) {
      const unsigned long long* t = prof.data() + static_cast<size_t>(i) * 20;
      const int c = t[7] ? 1 : 0;
      ++nw[c];
      members[c] += static_cast<int>(t[10]);
      tw[c][0] += (t[3] - t[0]) * 1e-3;
      tw[c][1] += (t[4] - t[3]) * 1e-3;
      tw[c][2] += (t[5] - t[4]) * 1e-3;
      if (c) tw[c][3] += (t[1] - t[0]) * 1e-3, tw[c][4] += (t[2] - t[1]) * 1e-3;
      if (t[6] && t[8] && t[9]) {  // select: integrate, replay, speculation choice
        tw[c][5] += (t[6] - t[4]) * 1e-3;
        tw[c][6] += (t[8] - t[6]) * 1e-3;
        tw[c][7] += (t[9] - t[8]) * 1e-3;
      }
    }
    for (int c = 0; c < 2; ++c) {
      if (!nw[c]) continue;
      std::fprintf(stderr, "wave grower, %s: %d waves, %d expansions; avg us: work %.2f barrier %.2f select %.2f",
                   c ? "large parents" : "small-parent waves", nw[c], members[c], tw[c][0] / nw[c], tw[c][1] / nw[c],
                   tw[c][2] / nw[c]);
      if (c) std::fprintf(stderr, " (partition %.2f hist %.2f)", tw[c][3] / nw[c], tw[c][4] / nw[c]);
      std::fprintf(stderr, " [integrate %.2f replay %.2f choose %.2f]", tw[c][5] / nw[c], tw[c][6] / nw[c],
                   tw[c][7] / nw[c]);
      std::fprintf(stderr, "\n");
    }
    std::fprintf(stderr, "wave grower: %d splits committed, %d expansions\n", counts[0], members[0] + members[1]);
    if (std::atoi(pe) >= 2) {  // every wave with large members: count+small / scatter / hist / barrier
      for (int i = 0; i < counts[3]; ++i) {
        const unsigned long long* t = prof.data() + static_cast<size_t>(i) * 20;
        if (!t[7]) continue;
        std::fprintf(stderr, "  wave %3d: %2llu large of %2llu members: count+small %7.2f scatter %7.2f hist %7.2f "
                     "barrier %5.2f select %5.2f us",
                     i, t[7], t[10], (t[1] - t[0]) * 1e-3, (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3,
                     (t[4] - t[3]) * 1e-3, (t[5] - t[4]) * 1e-3);
        if (t[17] && t[19])  // inside hist: CTA 0's items, the last CTA's items, the finishes
          std::fprintf(stderr, "  [items cta0 %.2f last %.2f finish %.2f]", (t[17] - t[2]) * 1e-3,
                       (t[18] - t[2]) * 1e-3, (t[3] - t[19]) * 1e-3);
        std::fprintf(stderr, "\n");
      }
    }
    double cand = 0, commits = 0, nav = 0, nfr = 0, rep = 0, imb = 0, lat = 0;
    for (int i = 0; i < counts[3]; ++i) {
      const unsigned long long* t = prof.data() + static_cast<size_t>(i) * 20;
      commits += static_cast<double>(t[12]);
      cand += t[13] / 1965.0;  // SM cycles at 1965 MHz
      rep += t[11] / 1965.0;
      if (t[16] > t[3]) imb += (t[16] - t[3]) * 1e-3;  // last CTA's arrival after CTA 0's
      if (t[4] > t[16]) lat += (t[4] - t[16]) * 1e-3;  // release after the last arrival
      nav += static_cast<double>(t[14]);
      nfr += static_cast<double>(t[15]);
    }
    if (counts[3] > 0)
      std::fprintf(stderr, "wave grower: per wave %.2f commits replayed in %.2f us (clock64), choice %.2f us, "
                   "%.0f expandable, %.0f open leaves\n", commits / counts[3], rep / counts[3], cand / counts[3],
                   nav / counts[3], nfr / counts[3]);
    if (counts[3] > 0)
      std::fprintf(stderr, "wave grower: barrier phase = %.2f us waiting for the last CTA + %.2f us release\n",
                   imb / counts[3], lat / counts[3]);
  } else if (a.prof != nullptr) {
    HBG_CUDA(cudaMemcpy(prof.data(), a.prof, prof.size() * 8, cudaMemcpyDeviceToHost));
    // stamps: 0 start, 1 partitioned, 2 small-child histogram, 3 finish+scans, 4 barrier, 5 picked;
    // slot 7: class = (large parent ? 4 : 0) + path (0 none, 1 direct, 2 shared-memory histogram)
    static const char* nm[7] = {"partition", "child hist", "finish+scans", "barrier", "winners+pick", "loop",
                                "(winners)"};
    for (int cls = 0; cls < 8; ++cls) {
      double acc[7] = {0, 0, 0, 0, 0, 0, 0};
      int n[7] = {0, 0, 0, 0, 0, 0, 0}, splits = 0;
      for (int i = 0; i < counts[0]; ++i) {
        const unsigned long long* t = prof.data() + static_cast<size_t>(i) * 20;
        if (static_cast<int>(t[7]) != cls) continue;
        ++splits;
        for (int j = 0; j < 5; ++j)
          if (t[j] && t[j + 1]) acc[j] += (t[j + 1] - t[j]) * 1e-3, ++n[j];
        if (i + 1 < counts[0] && t[5] && t[20]) acc[5] += (t[20] - t[5]) * 1e-3, ++n[5];
        if (t[4] && t[8]) acc[6] += (t[8] - t[4]) * 1e-3, ++n[6];
      }
      if (splits == 0) continue;
      if (cls == 6)  // the shared-memory histogram splits one by one
        for (int i = 0; i < counts[0]; ++i) {
          const unsigned long long* t = prof.data() + static_cast<size_t>(i) * 20;
          if (static_cast<int>(t[7]) != cls) continue;
          std::fprintf(stderr, "   split %3d parent %9llu small %9llu: partition %7.1f hist %7.1f finish %7.1f us\n", i,
                       t[10], t[11], (t[1] - t[0]) * 1e-3, (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3);
        }
      std::fprintf(stderr, "grow class %s parent, path %d: %d splits\n", cls >= 4 ? "large" : "small", cls & 3, splits);
      for (int j = 0; j < 7; ++j)
        if (n[j]) std::fprintf(stderr, "   %-13s total %9.1f us avg %7.2f us\n", nm[j], acc[j], acc[j] / n[j]);
    }
  }
  if (counts[0] > 0)
    HBG_CUDA(cudaMemcpy(split_log, a.split_log, static_cast<size_t>(counts[0]) * sizeof(hbg_split),
                        cudaMemcpyDeviceToHost));
  if (nodes_out)
    HBG_CUDA(cudaMemcpy(nodes_out, a.tree, static_cast<size_t>(counts[1]) * sizeof(hbg_tree_node),
                        cudaMemcpyDeviceToHost));
}

// boost_one_iteration (boosting.cpp:26-51) on the device: gradients at the
// cached scores, grow_tree, and scores += learning_rate * value of each row's
// leaf — every final leaf owns a contiguous range of the ordered row buffer,
// so the update needs no tree traversal.
void boost_impl(hbg_dataset* ds, const double* d_targets, double* d_scores, int loss, double lr,
                const hbg_grow_params& P, const Reducer& reduce, hbg_split* split_log,
                int32_t* num_splits, hbg_tree_node* nodes, int32_t* num_nodes, cudaStream_t s,
                hbg_peer* peer = nullptr) {
  require(loss == HBG_LOSS_SQUARED || loss == HBG_LOSS_LOGISTIC, "unknown loss");
  require(P.precision == HBG_PRECISION_BITS32, "boosting iterations run bits32 (fp32 g/h) trees");
  const int64_t N = ds->layout.num_rows;
  float* g = static_cast<float*>(ds->boost_g.get(static_cast<size_t>(N) * 4 + 4));
  float* h = static_cast<float*>(ds->boost_h.get(static_cast<size_t>(N) * 4 + 4));
  launch_grad_hess(loss, d_scores, d_targets, N, g, h, s);
  if (reduce.fn == nullptr && (peer != nullptr || !use_host_loop())) {
    std::vector<hbg_tree_node> local;
    if (nodes == nullptr) {
      local.resize(static_cast<size_t>(std::max(1, 2 * P.num_leaves - 1)));
      nodes = local.data();
    }
    grow_tree_persistent(ds, g, h, P, split_log, num_splits, nodes, num_nodes, s, peer);
    if (*num_splits == 0) {  // a root-only tree: every row gets the root value
      LeafRange r{0, N, nodes[0].value, 0, 0};
      LeafRange* dl = static_cast<LeafRange*>(ds->boost_leaves.get(sizeof(LeafRange) + 8));
      HBG_CUDA(cudaMemcpyAsync(dl, &r, sizeof r, cudaMemcpyHostToDevice, s));
      launch_iota(static_cast<int32_t*>(ds->ord[0][0].get(static_cast<size_t>(N) * 4 + 4)), N, s);
      launch_score_update(dl, 1, static_cast<const int32_t*>(ds->ord[0][0].p), nullptr, lr, d_scores, s);
    } else if (ds->grow_waves) {
      launch_score_update(static_cast<const LeafRange*>(ds->grow_records), ds->grow_ranges,
                          static_cast<const int32_t*>(ds->ord[0][0].p), static_cast<const int32_t*>(ds->ord[1][0].p),
                          lr, d_scores, s);
    } else {
      launch_score_update_nodes(ds->grow_records, static_cast<const hbg_tree_node*>(ds->grow_tree.p), *num_nodes,
                                static_cast<const int32_t*>(ds->ord[0][0].p),
                                static_cast<const int32_t*>(ds->ord[1][0].p), lr, d_scores, s);
    }
    HBG_CUDA(cudaStreamSynchronize(s));
    return;
  }
  std::vector<LeafRange> leaves;
  grow_tree_impl(ds, g, h, P, reduce, split_log, num_splits, nodes, num_nodes, s, &leaves);
  LeafRange* dl = static_cast<LeafRange*>(ds->boost_leaves.get(leaves.size() * sizeof(LeafRange) + 8));
  HBG_CUDA(cudaMemcpyAsync(dl, leaves.data(), leaves.size() * sizeof(LeafRange), cudaMemcpyHostToDevice, s));
  const int32_t* rows[2] = {static_cast<const int32_t*>(ds->ord[0][0].p),
                            static_cast<const int32_t*>(ds->ord[1][0].p)};
  launch_score_update(dl, static_cast<int>(leaves.size()), rows[0], rows[1], lr, d_scores, s);
  HBG_CUDA(cudaStreamSynchronize(s));  // `leaves` (pageable) must outlive the copy
}

}  // namespace

extern "C" {

const char* hbg_last_error(void) { return g_last_error.c_str(); }

int32_t hbg_version(void) { return 1; }

int hbg_dataset_create(const uint8_t* const* columns, int32_t num_features, int64_t num_rows,
                       int32_t max_bin, int32_t device, hbg_dataset** out) {
  return guarded([&] {
    require(out != nullptr, "null output handle");
    *out = nullptr;
    require(num_features >= 0 && num_rows >= 0, "negative shape");
    require(max_bin >= 2 && max_bin <= 256, "max_bin out of range [2, 256]");
    require(num_rows <= INT32_MAX, "row ids are int32 (row_index_t, dataset.hpp:9)");
    require(num_features == 0 || columns != nullptr, "null columns");
    int ndev = 0;
    HBG_CUDA(cudaGetDeviceCount(&ndev));
    require(device >= 0 && device < ndev, "device ordinal out of range");
    DeviceGuard dg(device);
    configure_kernels(device);
    auto ds = std::make_unique<hbg_dataset>();
    hbg_layout& L = ds->layout;
    L.num_rows = num_rows;
    L.num_features = num_features;
    L.max_bin = max_bin;
    L.bits_per_bin = max_bin <= 16 ? 4 : 8;
    L.features_per_word = 32 / L.bits_per_bin;
    L.words_per_row = (num_features + L.features_per_word - 1) / L.features_per_word;
    L.slice_bytes = L.bits_per_bin == 4 ? 16 : 32;
    L.num_groups = (num_features + 31) / 32;
    // group-planar: slice group g of every row, then group g + 1 (each group
    // 256-B aligned), so a warp's tile of 32 consecutive rows of one group is
    // one contiguous run of 512 B / 1 KB — with row-major rows of G groups it
    // was 32 separate lines, which cost the LSU 4x the tag lookups of d <= 32
    // (measured: 0.32 vs 0.21 ms for the same updates at d >= 128)
    L.row_stride_bytes = L.slice_bytes;
    L.group_stride_bytes = (static_cast<int64_t>(num_rows) * L.slice_bytes + 255) / 256 * 256;
    L.device = device;
    HBG_CUDA(cudaStreamCreateWithFlags(&ds->stream, cudaStreamNonBlocking));
    const size_t packed_bytes = static_cast<size_t>(L.num_groups) * static_cast<size_t>(L.group_stride_bytes);
    HBG_CUDA(cudaMalloc(&ds->packed, std::max<size_t>(packed_bytes, 16)));
    if (packed_bytes > 0) {
      for (int f = 0; f < num_features; ++f) require(columns[f] != nullptr, "null column pointer");
      // Upload column-major bins (a1) and pack on device (a2), one 32-feature
      // slice group at a time. The column-major copy stays resident: the tree
      // grower's partition reads one byte per row of the split feature from
      // it (instead of a 32-byte sector of the packed row).
      DevBuf bad_buf;
      uint8_t* colbins = static_cast<uint8_t*>(ds->colbins.get(static_cast<size_t>(num_features) * num_rows));
      int* d_bad = static_cast<int*>(bad_buf.get(sizeof(int)));
      HBG_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), ds->stream));
      const int64_t gs_words = L.group_stride_bytes / 4;
      for (int f0 = 0; f0 < num_features; f0 += 32) {
        const int nf = std::min(32, num_features - f0);
        uint8_t* d_cols = colbins + static_cast<size_t>(f0) * num_rows;
        for (int f = 0; f < nf; ++f) {
          HBG_CUDA(cudaMemcpyAsync(d_cols + static_cast<size_t>(f) * num_rows, columns[f0 + f],
                                   static_cast<size_t>(num_rows), cudaMemcpyHostToDevice, ds->stream));
        }
        launch_pack(d_cols, f0, nf, num_features, num_rows, max_bin, L.bits_per_bin,
                    gs_words, ds->packed, d_bad, ds->stream);
      }
      int bad = 0;
      HBG_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, ds->stream));
      HBG_CUDA(cudaStreamSynchronize(ds->stream));
      require(bad == 0, "bin value >= max_bin in input columns");
    }
    *out = ds.release();
  });
}

int hbg_dataset_destroy(hbg_dataset* ds) {
  return guarded([&] {
    if (!ds) return;
    DeviceGuard dg(ds->layout.device);
    delete ds;
  });
}

int hbg_dataset_layout(const hbg_dataset* ds, hbg_layout* out) {
  return guarded([&] {
    check_ds(ds);
    require(out != nullptr, "null output");
    *out = ds->layout;
  });
}

int hbg_dataset_packed_words(const hbg_dataset* ds, uint32_t* host_words) {
  return guarded([&] {
    check_ds(ds);
    const hbg_layout& L = ds->layout;
    if (L.num_rows == 0 || L.words_per_row == 0) return;
    require(host_words != nullptr, "null output");
    DeviceGuard dg(L.device);
    // back to the reference's row-major tuple order (binning.cpp:141-156), one slice group at a time
    const int wps = L.slice_bytes / 4;
    for (int gidx = 0; gidx < L.num_groups; ++gidx) {
      const int w0 = gidx * wps, nw = std::min(wps, L.words_per_row - w0);
      HBG_CUDA(cudaMemcpy2D(host_words + w0, static_cast<size_t>(L.words_per_row) * 4,
                            reinterpret_cast<const char*>(ds->packed) + gidx * L.group_stride_bytes,
                            static_cast<size_t>(L.row_stride_bytes), static_cast<size_t>(nw) * 4,
                            static_cast<size_t>(L.num_rows), cudaMemcpyDeviceToHost));
    }
  });
}

int hbg_build_histograms(hbg_dataset* ds, const int32_t* indices, int64_t count,
                         const double* gradients, const double* hessians, hbg_bin* out) {
  return hbg_build_histograms_ex(ds, indices, count, gradients, hessians, HBG_PRECISION_BITS32, out);
}

int hbg_build_histograms_ex(hbg_dataset* ds, const int32_t* indices, int64_t count,
                            const double* gradients, const double* hessians, int32_t precision,
                            hbg_bin* out) {
  return guarded([&] {
    check_ds(ds);
    require(precision == HBG_PRECISION_BITS32 || precision == HBG_PRECISION_BITS64, "unknown precision");
    const hbg_layout& L = ds->layout;
    require(count >= 0, "negative leaf size");
    require(out != nullptr, "null output");
    require(count == 0 || (indices && gradients && hessians), "null leaf arrays");
    DeviceGuard dg(L.device);
    cudaStream_t s = ds->stream;
    const size_t D = static_cast<size_t>(L.num_features) * L.max_bin;
    double* d_hist = static_cast<double*>(ds->host_hist.get(3 * D * sizeof(double) + 8));
    hbg_bin* d_bins = static_cast<hbg_bin*>(ds->host_bins.get(D * sizeof(hbg_bin) + 8));
    int64_t& h2d = ds->copy_h2d;
    h2d = 0;
    ds->copy_d2h = static_cast<int64_t>(D * sizeof(hbg_bin));
    if (count > 0 && precision == HBG_PRECISION_BITS64) {
      // bits64: the fp64 LeafState arrays go up as they are (no per-element
      // cast): pinned ones straight from the caller's memory, pageable ones
      // copied chunk by chunk into the pinned stage by the host pool (the
      // driver's own pageable path runs at ~11 GB/s); the pool checks the
      // ids either way. One histogram launch accumulates in fp64.
      const size_t n = static_cast<size_t>(count);
      double* d_gd = static_cast<double*>(ds->host_gd.get(n * 8));
      double* d_hd = static_cast<double*>(ds->host_hd.get(n * 8));
      const int32_t* d_idx;
      const bool pinned = is_pinned(gradients) && is_pinned(hessians);
      if (!ds->copy_stream) HBG_CUDA(cudaStreamCreateWithFlags(&ds->copy_stream, cudaStreamNonBlocking));
      for (int c = 0; c < 17; ++c)
        if (!ds->chunk_ev[c]) HBG_CUDA(cudaEventCreateWithFlags(&ds->chunk_ev[c], cudaEventDisableTiming));
      HBG_CUDA(cudaEventRecord(ds->chunk_ev[16], s));
      HBG_CUDA(cudaStreamWaitEvent(ds->copy_stream, ds->chunk_ev[16], 0));
      int32_t* di = static_cast<int32_t*>(ds->host_idx.get(n * 4));
      // the ids travel unless every chunk is one range from idx[0]: chunks
      // that pass are held back until one fails (then all go). Pinned g/h
      // go straight from the caller's memory (every chunk `direct`: the pool
      // only checks the ids), pageable ones through the pinned stage.
      bool all_contig = true;
      int64_t sent = 0;
      const std::vector<char> direct(static_cast<size_t>((count + kStageRows - 1) / kStageRows), pinned ? 1 : 0);
      stage_chunks<double>(ds, gradients, hessians, indices, count, kStageRows, direct,
                           [&](int k, int64_t b, int64_t e, const double* gs, const double* hs, const int32_t* is,
                               bool contig, auto&& fill_ids) {
                             const size_t m = static_cast<size_t>(e - b);
                             const double* sg = pinned ? gradients : gs;
                             const double* sh = pinned ? hessians : hs;
                             HBG_CUDA(cudaMemcpyAsync(d_gd + b, sg + b, m * 8, cudaMemcpyHostToDevice, ds->copy_stream));
                             HBG_CUDA(cudaMemcpyAsync(d_hd + b, sh + b, m * 8, cudaMemcpyHostToDevice, ds->copy_stream));
                             h2d += static_cast<int64_t>(m) * 16;
                             all_contig = all_contig && contig;
                             if (!all_contig) {
                               for (int j = static_cast<int>(sent / kStageRows); j <= k; ++j) fill_ids(j);
                               HBG_CUDA(cudaMemcpyAsync(di + sent, is + sent, static_cast<size_t>(e - sent) * 4,
                                                        cudaMemcpyHostToDevice, ds->copy_stream));
                               h2d += (e - sent) * 4;
                               sent = e;
                             }
                           });
      HBG_CUDA(cudaEventRecord(ds->chunk_ev[0], ds->copy_stream));
      HBG_CUDA(cudaStreamWaitEvent(s, ds->chunk_ev[0], 0));
      if (all_contig) {
        require(indices[0] >= 0 && indices[0] + count <= L.num_rows, "leaf row index out of range");
        d_idx = identity_rows(ds, indices[0], s);
      } else {
        d_idx = di;
      }
      build_device(ds, d_idx, count, d_gd, d_hd, HBG_GH_LEAF_ALIGNED, d_hist, s, nullptr, nullptr, 8, true);
    } else if (count > 0) {
      // fp32 g/h in staged chunks of kStageRows rows. Each staged chunk is
      // either converted to fp32 by the host pool into the pinned stage and
      // copied as 8 B/row, or (pinned caller arrays only: `direct`) copied as
      // fp64 16 B/row straight from the caller's memory and converted on the
      // device — the split balances host memory bandwidth against PCIe. The
      // row ids are staged with g/h, each staged chunk checked for
      // idx[i] == idx[0] + i in the same pass: a histogram chunk whose rows
      // all pass reads the resident iota (the root, or any leaf of an ordered
      // layout, uploads no ids); the others upload the ids not yet sent.
      // Histogram chunk c runs as soon as its rows have landed; the C chunk
      // histograms are summed in chunk order — the same floats and sums
      // whichever route each row took (deterministic, bit-identical).
      const size_t n = static_cast<size_t>(count);
      const bool pinned = is_pinned(gradients) && is_pinned(hessians);
      float* d_gf = static_cast<float*>(ds->host_gf.get(n * 4));
      float* d_hf = static_cast<float*>(ds->host_hf.get(n * 4));
      double* d_gd = pinned ? static_cast<double*>(ds->host_gd.get(n * 8)) : nullptr;
      double* d_hd = pinned ? static_cast<double*>(ds->host_hd.get(n * 8)) : nullptr;
      const std::vector<char> direct = direct_chunks(count, kStageRows, pinned);
      const int C = host_chunks(count);
      if (!ds->copy_stream) HBG_CUDA(cudaStreamCreateWithFlags(&ds->copy_stream, cudaStreamNonBlocking));
      for (int c = 0; c < 17; ++c)
        if (!ds->chunk_ev[c]) HBG_CUDA(cudaEventCreateWithFlags(&ds->chunk_ev[c], cudaEventDisableTiming));
      HBG_CUDA(cudaEventRecord(ds->chunk_ev[16], s));  // the copy stream starts after prior work on s
      HBG_CUDA(cudaStreamWaitEvent(ds->copy_stream, ds->chunk_ev[16], 0));
      int32_t* di = static_cast<int32_t*>(ds->host_idx.get(n * 4));
      const int64_t first = indices[0];
      double* parts = C > 1 ? static_cast<double*>(ds->host_parts.get(static_cast<size_t>(C) * 3 * D * sizeof(double) + 8))
                            : d_hist;
      std::vector<const double*> part_ptrs;
      int next = 0;
      int64_t sent = 0;         // ids [0, sent) are on the device (or not needed)
      int64_t converted = 0;    // rows [0, converted) of d_gf/d_hf are final (or queued on s)
      bool run_contig = true;   // every staged chunk of histogram chunk `next` so far passed
      stage_chunks(ds, gradients, hessians, indices, count, kStageRows, direct,
                   [&](int k, int64_t b, int64_t e, const float* gs, const float* hs, const int32_t* is, bool contig,
                       auto&& fill_ids) {
                     const size_t m = static_cast<size_t>(e - b);
                     if (direct[static_cast<size_t>(k)]) {
                       HBG_CUDA(cudaMemcpyAsync(d_gd + b, gradients + b, m * 8, cudaMemcpyHostToDevice, ds->copy_stream));
                       HBG_CUDA(cudaMemcpyAsync(d_hd + b, hessians + b, m * 8, cudaMemcpyHostToDevice, ds->copy_stream));
                       h2d += static_cast<int64_t>(m) * 16;
                     } else {
                       HBG_CUDA(cudaMemcpyAsync(d_gf + b, gs + b, m * 4, cudaMemcpyHostToDevice, ds->copy_stream));
                       HBG_CUDA(cudaMemcpyAsync(d_hf + b, hs + b, m * 4, cudaMemcpyHostToDevice, ds->copy_stream));
                       h2d += static_cast<int64_t>(m) * 8;
                     }
                     run_contig = run_contig && contig;
                     for (; next < C && count * (next + 1) / C <= e; ++next) {
                       const int64_t cb = count * next / C, ce = count * (next + 1) / C;
                       const int32_t* rows_c;
                       if (run_contig && ce > cb) {
                         require(first + cb >= 0 && first + ce <= L.num_rows, "leaf row index out of range");
                         rows_c = identity_rows(ds, first + cb, s);
                       } else {
                         if (sent < ce) {
                           const int64_t from = std::max(sent, cb);
                           for (int64_t j = from / kStageRows; j <= (ce - 1) / kStageRows; ++j)
                             fill_ids(static_cast<int>(j));
                           HBG_CUDA(cudaMemcpyAsync(di + from, is + from, static_cast<size_t>(ce - from) * 4,
                                                    cudaMemcpyHostToDevice, ds->copy_stream));
                           h2d += (ce - from) * 4;
                           sent = ce;
                         }
                         rows_c = di + cb;
                       }
                       HBG_CUDA(cudaEventRecord(ds->chunk_ev[next], ds->copy_stream));
                       HBG_CUDA(cudaStreamWaitEvent(s, ds->chunk_ev[next], 0));
                       // device conversion of the direct rows up to ce
                       for (int64_t j = converted / kStageRows; converted < ce; ++j) {
                         const int64_t je = std::min<int64_t>(ce, (j + 1) * kStageRows);
                         if (direct[static_cast<size_t>(j)]) {
                           launch_f64_to_f32(d_gd + converted, d_gf + converted, je - converted, s);
                           launch_f64_to_f32(d_hd + converted, d_hf + converted, je - converted, s);
                         }
                         converted = je;
                       }
                       double* hc = parts + static_cast<size_t>(next) * (C > 1 ? 3 * D : 0);
                       build_device(ds, rows_c, ce - cb, d_gf + cb, d_hf + cb, HBG_GH_LEAF_ALIGNED, hc, s,
                                    nullptr, nullptr, 4, true);
                       part_ptrs.push_back(hc);
                       // a staged chunk straddling the boundary also holds
                       // rows of the next histogram chunk
                       run_contig = ce < e ? contig : true;
                     }
                   });
      if (C > 1) launch_reduce_parts(part_ptrs, static_cast<int64_t>(3 * D), d_hist, s);
    } else {
      build_device(ds, nullptr, 0, nullptr, nullptr, HBG_GH_LEAF_ALIGNED, d_hist, s);
    }
    launch_hist_to_bins(d_hist, static_cast<int64_t>(D), d_bins, s);
    if (D > 0) HBG_CUDA(cudaMemcpyAsync(out, d_bins, D * sizeof(hbg_bin), cudaMemcpyDeviceToHost, s));
    HBG_CUDA(cudaStreamSynchronize(s));
  });
}

// Development aid: the HBG_HIST_PROFILE %globaltimer stamps (ns) of the last
// histogram launch's CTA 0 (start, cleared, rows done, partials written,
// barrier passed, reduced), copied to host `out[6]`.
int hbg_debug_hist_stamps(hbg_dataset* ds, unsigned long long* out) {
  return guarded([&] {
    check_ds(ds);
    require(ds->hist_prof.p != nullptr, "no stamps: set HBG_HIST_PROFILE");
    HBG_CUDA(cudaMemcpy(out, ds->hist_prof.p, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  });
}

int hbg_debug_host_copy_bytes(hbg_dataset* ds, int64_t* out) {
  return guarded([&] {
    check_ds(ds);
    require(out != nullptr, "null argument");
    out[0] = ds->copy_h2d;
    out[1] = ds->copy_d2h;
  });
}

int hbg_build_histograms_device(hbg_dataset* ds, const int32_t* d_indices, int64_t count,
                                const float* d_grad, const float* d_hess, int32_t gh_mode,
                                double* d_hist, void* stream) {
  return guarded([&] {
    check_ds(ds);
    DeviceGuard dg(ds->layout.device);
    build_device(ds, d_indices, count, d_grad, d_hess, gh_mode, d_hist, pick(ds, stream), nullptr, nullptr, 4, true);
  });
}

int hbg_build_histograms_device_f64(hbg_dataset* ds, const int32_t* d_indices, int64_t count,
                                    const double* d_grad, const double* d_hess, int32_t gh_mode,
                                    double* d_hist, void* stream) {
  return guarded([&] {
    check_ds(ds);
    DeviceGuard dg(ds->layout.device);
    build_device(ds, d_indices, count, d_grad, d_hess, gh_mode, d_hist, pick(ds, stream), nullptr, nullptr, 8, true);
  });
}

int hbg_hist_to_bins_device(const double* d_hist, int32_t num_features, int32_t max_bin,
                            hbg_bin* d_bins, void* stream) {
  return guarded([&] {
    require(num_features >= 0 && max_bin >= 1, "bad shape");
    launch_hist_to_bins(d_hist, static_cast<int64_t>(num_features) * max_bin, d_bins,
                        static_cast<cudaStream_t>(stream));
  });
}

int hbg_subtract_device(const double* d_parent, const double* d_child, double* d_sibling,
                        int64_t n_values, void* stream) {
  return guarded([&] {
    require(n_values >= 0, "negative size");
    launch_subtract(d_parent, d_child, d_sibling, n_values, static_cast<cudaStream_t>(stream));
  });
}

int hbg_gather_leaf_device(const int32_t* d_indices, int64_t count, const float* d_grad,
                           const float* d_hess, float* d_leaf_grad, float* d_leaf_hess,
                           double* d_totals, void* stream) {
  return guarded([&] {
    require(count >= 0, "negative leaf size");
    require(d_totals != nullptr, "null totals");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // scratch per (thread, device): a buffer allocated on one device must not
    // serve a launch on another
    static thread_local DevBuf scratch[64];
    int dev = 0;
    HBG_CUDA(cudaGetDevice(&dev));
    double* sc = static_cast<double*>(scratch[dev & 63].get(gather_scratch_doubles(count) * sizeof(double)));
    launch_gather(d_indices, count, d_grad, d_hess, d_leaf_grad, d_leaf_hess, d_totals, sc, s);
  });
}

int hbg_gather_leaf_statistics(const int32_t* indices, int64_t count, const double* gradients,
                               const double* hessians, int64_t num_rows, double* leaf_grad,
                               double* leaf_hess, double* totals, int32_t device) {
  return guarded([&] {
    require(count >= 0 && num_rows >= 0, "negative size");
    require(totals != nullptr, "null totals");
    require(count == 0 || (indices && gradients && hessians && leaf_grad && leaf_hess), "null leaf arrays");
    for (int64_t i = 0; i < count; ++i)  // the reference leaves this UB (tree.cpp:19); here it is an error
      require(indices[i] >= 0 && indices[i] < num_rows, "leaf row index out of range");
    DeviceGuard dg(device);
    DevBuf di, dg_, dh, dlg, dlh, dt, sc;
    const size_t n = static_cast<size_t>(count), N = static_cast<size_t>(num_rows);
    int32_t* d_idx = static_cast<int32_t*>(di.get(n * 4 + 4));
    double* d_g = static_cast<double*>(dg_.get(N * 8 + 8));
    double* d_h = static_cast<double*>(dh.get(N * 8 + 8));
    double* d_lg = static_cast<double*>(dlg.get(n * 8 + 8));
    double* d_lh = static_cast<double*>(dlh.get(n * 8 + 8));
    double* d_t = static_cast<double*>(dt.get(2 * sizeof(double)));
    double* d_sc = static_cast<double*>(sc.get(gather_scratch_doubles(count) * sizeof(double)));
    if (count > 0) {
      HBG_CUDA(cudaMemcpy(d_idx, indices, n * 4, cudaMemcpyHostToDevice));
      HBG_CUDA(cudaMemcpy(d_g, gradients, N * 8, cudaMemcpyHostToDevice));
      HBG_CUDA(cudaMemcpy(d_h, hessians, N * 8, cudaMemcpyHostToDevice));
    }
    launch_gather_f64(d_idx, count, d_g, d_h, d_lg, d_lh, d_t, d_sc, nullptr);
    if (count > 0) {
      HBG_CUDA(cudaMemcpy(leaf_grad, d_lg, n * 8, cudaMemcpyDeviceToHost));
      HBG_CUDA(cudaMemcpy(leaf_hess, d_lh, n * 8, cudaMemcpyDeviceToHost));
    }
    HBG_CUDA(cudaMemcpy(totals, d_t, 2 * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int hbg_best_split_device(const double* d_hist, int32_t num_features, int32_t max_bin,
                          double grad_total, double hess_total, int64_t count,
                          int64_t min_data_in_leaf, double lambda, hbg_split* d_out, void* stream) {
  return guarded([&] {
    require(num_features >= 0 && max_bin >= 1, "bad shape");
    require(d_out != nullptr, "null output");
    launch_best_split(d_hist, num_features, max_bin, nullptr, nullptr, grad_total, hess_total,
                      count, min_data_in_leaf, lambda, d_out, static_cast<cudaStream_t>(stream));
  });
}

int hbg_best_split_device_totals(const double* d_hist, int32_t num_features, int32_t max_bin,
                                 const double* d_totals, const int64_t* d_count,
                                 int64_t min_data_in_leaf, double lambda, hbg_split* d_out,
                                 void* stream) {
  return guarded([&] {
    require(num_features >= 0 && max_bin >= 1, "bad shape");
    require(d_out != nullptr && d_totals != nullptr && d_count != nullptr, "null pointer");
    launch_best_split(d_hist, num_features, max_bin, d_totals, d_count, 0.0, 0.0, 0,
                      min_data_in_leaf, lambda, d_out, static_cast<cudaStream_t>(stream));
  });
}

int hbg_find_best_split(const hbg_bin* hists, int32_t num_features, int32_t max_bin,
                        double grad_total, double hess_total, int64_t count,
                        int64_t min_data_in_leaf, double lambda, hbg_split* out, int32_t* found) {
  return guarded([&] {
    require(num_features >= 0 && max_bin >= 1, "bad shape");
    require(out != nullptr && found != nullptr, "null output");
    require(num_features == 0 || hists != nullptr, "null histograms");
    const size_t D = static_cast<size_t>(num_features) * max_bin;
    std::vector<double> soa(3 * D);
    for (size_t i = 0; i < D; ++i) {
      soa[i] = hists[i].grad_sum;
      soa[D + i] = hists[i].hess_sum;
      soa[2 * D + i] = static_cast<double>(hists[i].count);
    }
    DevBuf dh, ds;
    double* d_hist = static_cast<double*>(dh.get(soa.size() * sizeof(double) + 8));
    hbg_split* d_out = static_cast<hbg_split*>(ds.get(sizeof(hbg_split)));
    if (D) HBG_CUDA(cudaMemcpy(d_hist, soa.data(), soa.size() * sizeof(double), cudaMemcpyHostToDevice));
    launch_best_split(d_hist, num_features, max_bin, nullptr, nullptr, grad_total, hess_total,
                      count, min_data_in_leaf, lambda, d_out, nullptr);
    HBG_CUDA(cudaMemcpy(out, d_out, sizeof(hbg_split), cudaMemcpyDeviceToHost));
    *found = out->feature >= 0 ? 1 : 0;
  });
}

int hbg_grow_tree(hbg_dataset* ds, const float* d_grad, const float* d_hess,
                  const hbg_grow_params* params, hbg_split* split_log, int32_t* num_splits,
                  hbg_tree_node* nodes, int32_t* num_nodes, void* stream) {
  return guarded([&] {
    check_ds(ds);
    require(params != nullptr && split_log != nullptr && num_splits != nullptr &&
                num_nodes != nullptr,
            "null argument");
    require(ds->layout.num_rows == 0 || (d_grad != nullptr && d_hess != nullptr),
            "null gradient/hessian pointer");
    require(params->precision == HBG_PRECISION_BITS32,
            "hbg_grow_tree takes fp32 gradients (bits32); bits64 trees: hbg_grow_tree_f64 / hbg_grow_tree_host");
    DeviceGuard dg(ds->layout.device);
    if (use_host_loop())
      grow_tree_impl(ds, d_grad, d_hess, *params, Reducer{nullptr, nullptr}, split_log, num_splits,
                     nodes, num_nodes, static_cast<cudaStream_t>(stream));
    else
      grow_tree_persistent(ds, d_grad, d_hess, *params, split_log, num_splits, nodes, num_nodes,
                           static_cast<cudaStream_t>(stream));
  });
}

int hbg_grow_tree_f64(hbg_dataset* ds, const double* d_grad, const double* d_hess,
                      const hbg_grow_params* params, hbg_split* split_log, int32_t* num_splits,
                      hbg_tree_node* nodes, int32_t* num_nodes, void* stream) {
  return guarded([&] {
    check_ds(ds);
    require(params != nullptr && split_log != nullptr && num_splits != nullptr && num_nodes != nullptr,
            "null argument");
    require(ds->layout.num_rows == 0 || (d_grad != nullptr && d_hess != nullptr),
            "null gradient/hessian pointer");
    require(params->precision == HBG_PRECISION_BITS64, "hbg_grow_tree_f64 grows bits64 trees");
    DeviceGuard dg(ds->layout.device);
    grow_tree_impl(ds, d_grad, d_hess, *params, Reducer{nullptr, nullptr}, split_log, num_splits, nodes,
                   num_nodes, static_cast<cudaStream_t>(stream));
  });
}

int hbg_grow_tree_host(hbg_dataset* ds, const double* gradients, const double* hessians,
                       const hbg_grow_params* params, hbg_split* split_log, int32_t* num_splits,
                       hbg_tree_node* nodes, int32_t* num_nodes) {
  return guarded([&] {
    check_ds(ds);
    require(params != nullptr && split_log != nullptr && num_splits != nullptr && num_nodes != nullptr,
            "null argument");
    const int64_t N = ds->layout.num_rows;
    require(N == 0 || (gradients != nullptr && hessians != nullptr), "null gradient/hessian pointer");
    require(params->precision == HBG_PRECISION_BITS32 || params->precision == HBG_PRECISION_BITS64,
            "unknown precision");
    DeviceGuard dg(ds->layout.device);
    cudaStream_t s = ds->stream;
    if (params->precision == HBG_PRECISION_BITS64) {  // fp64 g/h as they are, fp64 everywhere
      const size_t n = static_cast<size_t>(N);
      double* gd = static_cast<double*>(ds->host_gd.get(n * 8 + 8));
      double* hd = static_cast<double*>(ds->host_hd.get(n * 8 + 8));
      if (N > 0 && is_pinned(gradients) && is_pinned(hessians)) {
        HBG_CUDA(cudaMemcpyAsync(gd, gradients, n * 8, cudaMemcpyHostToDevice, s));
        HBG_CUDA(cudaMemcpyAsync(hd, hessians, n * 8, cudaMemcpyHostToDevice, s));
      } else if (N > 0) {  // pageable: copied into the pinned stage by the host pool, chunk by chunk
        stage_chunks<double>(ds, gradients, hessians, nullptr, N, kStageRows, direct_chunks(N, kStageRows, false),
                             [&](int, int64_t b, int64_t e, const double* gs, const double* hs, const int32_t*, bool,
                                 auto&&) {
                               const size_t m = static_cast<size_t>(e - b);
                               HBG_CUDA(cudaMemcpyAsync(gd + b, gs + b, m * 8, cudaMemcpyHostToDevice, s));
                               HBG_CUDA(cudaMemcpyAsync(hd + b, hs + b, m * 8, cudaMemcpyHostToDevice, s));
                             });
      }
      grow_tree_impl(ds, gd, hd, *params, Reducer{nullptr, nullptr}, split_log, num_splits, nodes, num_nodes, s);
      HBG_CUDA(cudaStreamSynchronize(s));
      return;
    }
    float *gf = nullptr, *hf = nullptr;
    if (N > 0) {  // fp32 g/h through stage_chunks (pinned arrays: a share of the chunks as fp64 directly)
      const size_t n = static_cast<size_t>(N);
      const bool pinned = is_pinned(gradients) && is_pinned(hessians);
      gf = static_cast<float*>(ds->boost_g.get(n * 4 + 4));
      hf = static_cast<float*>(ds->boost_h.get(n * 4 + 4));
      double* gd = pinned ? static_cast<double*>(ds->host_gd.get(n * 8)) : nullptr;
      double* hd = pinned ? static_cast<double*>(ds->host_hd.get(n * 8)) : nullptr;
      const std::vector<char> direct = direct_chunks(N, kStageRows, pinned);
      stage_chunks(ds, gradients, hessians, nullptr, N, kStageRows, direct,
                   [&](int k, int64_t b, int64_t e, const float* gs, const float* hs, const int32_t*, bool, auto&&) {
                     const size_t m = static_cast<size_t>(e - b);
                     if (direct[static_cast<size_t>(k)]) {
                       HBG_CUDA(cudaMemcpyAsync(gd + b, gradients + b, m * 8, cudaMemcpyHostToDevice, s));
                       HBG_CUDA(cudaMemcpyAsync(hd + b, hessians + b, m * 8, cudaMemcpyHostToDevice, s));
                       launch_f64_to_f32(gd + b, gf + b, e - b, s);
                       launch_f64_to_f32(hd + b, hf + b, e - b, s);
                     } else {
                       HBG_CUDA(cudaMemcpyAsync(gf + b, gs + b, m * 4, cudaMemcpyHostToDevice, s));
                       HBG_CUDA(cudaMemcpyAsync(hf + b, hs + b, m * 4, cudaMemcpyHostToDevice, s));
                     }
                   });
    }
    if (use_host_loop())
      grow_tree_impl(ds, gf, hf, *params, Reducer{nullptr, nullptr}, split_log, num_splits, nodes, num_nodes, s);
    else
      grow_tree_persistent(ds, gf, hf, *params, split_log, num_splits, nodes, num_nodes, s);
    HBG_CUDA(cudaStreamSynchronize(s));
  });
}

void* hbg_dataset_stream(const hbg_dataset* ds) { return ds ? static_cast<void*>(ds->stream) : nullptr; }

int hbg_peer_create(hbg_dataset* ds, int32_t nranks, int32_t rank, int32_t ctas, const hbg_grow_params* params,
                    hbg_peer** out) {
  return guarded([&] {
    check_ds(ds);
    require(out != nullptr && params != nullptr, "null argument");
    require(params->num_leaves >= 1, "num_leaves must be at least 1");
    *out = nullptr;
    require(nranks >= 1 && nranks <= 8 && rank >= 0 && rank < nranks, "bad rank / rank count (1..8)");
    require(ctas >= 0, "negative CTA count");
    const hbg_layout& L = ds->layout;
    DeviceGuard dg(L.device);
    configure_kernels(L.device);
    PersistentGrowArgs a{};
    a.bits = L.bits_per_bin;
    a.d = L.num_features;
    a.k = L.max_bin;
    a.num_groups = L.num_groups;
    a.num_rows = L.num_rows;
    a.ctas = ctas;
    a.nranks = nranks;
    auto p = std::make_unique<hbg_peer>();
    p->nranks = nranks;
    p->rank = rank;
    p->device = L.device;
    p->ctas = ctas;
    p->xdoubles = grow_exchange_doubles(a, L.device);
    const int k_alloc = L.bits_per_bin == 4 ? 16 : (L.max_bin <= 64 ? 64 : (L.max_bin <= 128 ? 128 : 256));
    p->hoff = (p->xdoubles + 31) / 32 * 32;
    p->hdoubles = hist_exchange_doubles(k_alloc, L.max_bin, L.num_groups);
    const size_t total = p->hoff + p->hdoubles;
    HBG_CUDA(cudaMalloc(&p->xbuf, total * sizeof(double)));
    HBG_CUDA(cudaMemset(p->xbuf, 0, total * sizeof(double)));
    HBG_CUDA(cudaMalloc(&p->error, sizeof(int)));
    HBG_CUDA(cudaMemset(p->error, 0, sizeof(int)));
    p->peers[rank] = p->xbuf;
    // reserve every buffer of the peer calls (trees, boosting): an allocation
    // while another rank's grid waits in an exchange serialises behind it
    grow_workspace(ds, *params, ctas, nranks);
    // ... and of hbg_build_histograms_peer: the partials of any leaf size
    // (a cudaMalloc/cudaFree while another rank's reduction spins on this
    // rank's rows can wait for that kernel: ranks sharing a GPU deadlock
    // until the exchange times out) and the identity rows
    {
      size_t part = 0;
      const int64_t top = std::max<int64_t>(L.num_rows, 1);
      for (int64_t n = 1;; n = std::min<int64_t>(top, n + std::max<int64_t>(1, n / 4))) {  // ~25% steps
        part = std::max(part, hist_part_bytes(plan_histogram(L.bits_per_bin, L.max_bin, L.num_groups, n, L.device,
                                                             /*allow_direct=*/false)));
        if (n == top) break;
      }
      ds->part.get(part);
      if (L.num_rows > 0) identity_rows(ds, 0, ds->stream);
    }
    ds->boost_g.get(static_cast<size_t>(L.num_rows) * 4 + 4);
    ds->boost_h.get(static_cast<size_t>(L.num_rows) * 4 + 4);
    ds->boost_leaves.get(sizeof(LeafRange) + 8);
    HBG_CUDA(cudaDeviceSynchronize());
    *out = p.release();
  });
}

int hbg_peer_handle(hbg_peer* p, uint8_t* out) {
  return guarded([&] {
    require(p != nullptr && out != nullptr, "null argument");
    DeviceGuard dg(p->device);
    cudaIpcMemHandle_t h;
    HBG_CUDA(cudaIpcGetMemHandle(&h, p->xbuf));
    static_assert(sizeof(h) <= HBG_PEER_HANDLE_BYTES, "IPC handle size");
    std::memset(out, 0, HBG_PEER_HANDLE_BYTES);
    std::memcpy(out, &h, sizeof h);
  });
}

int hbg_peer_open(hbg_peer* p, int32_t peer_rank, const uint8_t* handle) {
  return guarded([&] {
    require(p != nullptr && handle != nullptr, "null argument");
    require(peer_rank >= 0 && peer_rank < p->nranks && peer_rank != p->rank, "bad peer rank");
    DeviceGuard dg(p->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void* ptr = nullptr;
    HBG_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    if (p->opened[peer_rank]) cudaIpcCloseMemHandle(p->opened[peer_rank]);
    p->opened[peer_rank] = ptr;
    p->peers[peer_rank] = static_cast<const double*>(ptr);
  });
}

int hbg_peer_attach(hbg_peer* p, int32_t peer_rank, const hbg_peer* q) {
  return guarded([&] {
    require(p != nullptr && q != nullptr, "null argument");
    require(peer_rank >= 0 && peer_rank < p->nranks && peer_rank == q->rank && q->nranks == p->nranks,
            "bad peer rank");
    if (q->device != p->device) {  // same process, two GPUs: direct peer access over NVLink
      DeviceGuard dg(p->device);
      const cudaError_t e = cudaDeviceEnablePeerAccess(q->device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else HBG_CUDA(e);
    }
    p->peers[peer_rank] = q->xbuf;
  });
}

int hbg_build_histograms_peer(hbg_dataset* ds, const int32_t* d_indices, int64_t count, const float* d_grad,
                              const float* d_hess, int32_t gh_mode, double* d_hist, hbg_peer* peer, void* stream) {
  return guarded([&] {
    check_ds(ds);
    require(peer != nullptr, "null peer");
    DeviceGuard dg(ds->layout.device);
    build_device_peer(ds, d_indices, count, d_grad, d_hess, gh_mode, d_hist, pick(ds, stream), peer);
  });
}

int hbg_peer_check(hbg_peer* p) {
  return guarded([&] {
    require(p != nullptr, "null peer");
    DeviceGuard dg(p->device);
    HBG_CUDA(cudaDeviceSynchronize());  // every stream's exchanges have finished (or timed out)
    int e = 0;
    HBG_CUDA(cudaMemcpy(&e, p->error, sizeof e, cudaMemcpyDeviceToHost));
    if (e != 0) {
      HBG_CUDA(cudaMemset(p->error, 0, sizeof(int)));
      throw Error(HBG_ERR_CUDA, "peer histogram exchange timed out (a rank never published)");
    }
  });
}

int hbg_peer_destroy(hbg_peer* p) {
  return guarded([&] {
    if (!p) return;
    DeviceGuard dg(p->device);
    delete p;
  });
}

int hbg_grow_tree_peer(hbg_dataset* ds, const float* d_grad, const float* d_hess, const hbg_grow_params* params,
                       hbg_peer* peer, hbg_split* split_log, int32_t* num_splits, hbg_tree_node* nodes,
                       int32_t* num_nodes, void* stream) {
  return guarded([&] {
    check_ds(ds);
    require(params != nullptr && peer != nullptr && split_log != nullptr && num_splits != nullptr &&
                num_nodes != nullptr,
            "null argument");
    require(ds->layout.num_rows == 0 || (d_grad != nullptr && d_hess != nullptr),
            "null gradient/hessian pointer");
    DeviceGuard dg(ds->layout.device);
    grow_tree_persistent(ds, d_grad, d_hess, *params, split_log, num_splits, nodes, num_nodes,
                         static_cast<cudaStream_t>(stream), peer);
  });
}

int hbg_grow_tree_sharded(hbg_dataset* ds, const float* d_grad, const float* d_hess,
                          const hbg_grow_params* params, hbg_allreduce_fn allreduce, void* ctx,
                          hbg_split* split_log, int32_t* num_splits, hbg_tree_node* nodes,
                          int32_t* num_nodes, void* stream) {
  return guarded([&] {
    check_ds(ds);
    require(params != nullptr && split_log != nullptr && num_splits != nullptr &&
                num_nodes != nullptr && allreduce != nullptr,
            "null argument");
    require(ds->layout.num_rows == 0 || (d_grad != nullptr && d_hess != nullptr),
            "null gradient/hessian pointer");
    require(params->precision == HBG_PRECISION_BITS32, "hbg_grow_tree_sharded takes fp32 gradients (bits32)");
    DeviceGuard dg(ds->layout.device);
    grow_tree_impl(ds, d_grad, d_hess, *params, Reducer{allreduce, ctx}, split_log, num_splits,
                   nodes, num_nodes, static_cast<cudaStream_t>(stream));
  });
}

int hbg_boost_one_iteration(hbg_dataset* ds, const double* d_targets, double* d_scores, int32_t loss,
                            double learning_rate, const hbg_grow_params* params, hbg_allreduce_fn allreduce,
                            void* ctx, hbg_split* split_log, int32_t* num_splits, hbg_tree_node* nodes,
                            int32_t* num_nodes, void* stream) {
  return guarded([&] {
    check_ds(ds);
    require(params != nullptr && split_log != nullptr && num_splits != nullptr && num_nodes != nullptr,
            "null argument");
    require(ds->layout.num_rows == 0 || (d_targets != nullptr && d_scores != nullptr),
            "null targets/scores");
    DeviceGuard dg(ds->layout.device);
    boost_impl(ds, d_targets, d_scores, loss, learning_rate, *params, Reducer{allreduce, ctx}, split_log,
               num_splits, nodes, num_nodes, static_cast<cudaStream_t>(stream));
  });
}

int hbg_boost_one_iteration_peer(hbg_dataset* ds, const double* d_targets, double* d_scores, int32_t loss,
                                 double learning_rate, const hbg_grow_params* params, hbg_peer* peer,
                                 hbg_split* split_log, int32_t* num_splits, hbg_tree_node* nodes, int32_t* num_nodes,
                                 void* stream) {
  return guarded([&] {
    check_ds(ds);
    require(params != nullptr && peer != nullptr && split_log != nullptr && num_splits != nullptr &&
                num_nodes != nullptr,
            "null argument");
    require(ds->layout.num_rows == 0 || (d_targets != nullptr && d_scores != nullptr), "null targets/scores");
    DeviceGuard dg(ds->layout.device);
    boost_impl(ds, d_targets, d_scores, loss, learning_rate, *params, Reducer{nullptr, nullptr}, split_log,
               num_splits, nodes, num_nodes, static_cast<cudaStream_t>(stream), peer);
  });
}

int hbg_reduce_histograms_device(const double* const* d_parts, int32_t nparts, int64_t n_values,
                                 double* d_out, void* stream) {
  return guarded([&] {
    require(nparts >= 1 && d_parts != nullptr && d_out != nullptr && n_values >= 0, "bad arguments");
    std::vector<const double*> parts(d_parts, d_parts + nparts);
    launch_reduce_parts(parts, n_values, d_out, static_cast<cudaStream_t>(stream));
  });
}

int hbg_dataset_set_profiling(hbg_dataset* ds, int32_t enabled) {
  return guarded([&] {
    check_ds(ds);
    ds->profiling = enabled != 0;
  });
}

int hbg_dataset_kernel_time(hbg_dataset* ds, double* total_ms, int64_t* launches) {
  return guarded([&] {
    check_ds(ds);
    require(total_ms != nullptr && launches != nullptr, "null output");
    DeviceGuard dg(ds->layout.device);
    double t = 0.0;
    for (auto& e : ds->events) {
      HBG_CUDA(cudaEventSynchronize(e.second));
      float ms = 0.f;
      HBG_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
      t += ms;
      ds->spare.push_back(e);
    }
    *total_ms = t;
    *launches = static_cast<int64_t>(ds->events.size());
    ds->events.clear();
  });
}

int hbg_stream_synchronize(void* stream) {
  return guarded([&] { HBG_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream))); });
}

}  // extern "C"
