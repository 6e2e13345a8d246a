// Host-side input-path microbenchmark for the host drop-in (hbg_build_histograms):
// how fast can a leaf's fp64 g/h (LeafState, leaf.hpp:15-16) reach the device?
//   dma64   : cudaMemcpyAsync of the fp64 arrays from pinned memory (GPU converts)
//   cvtT    : T host threads convert fp64 -> fp32 into pinned staging (no DMA)
//   both    : T threads convert half the rows while the copy engine moves the
//             other half as fp64, then the fp32 half is copied
// Build: nvcc -O3 -o h2d_convert h2d_convert.cu -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t err_ = (x);                                                   \
    if (err_ != cudaSuccess) {                                              \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(err_), __FILE__, __LINE__); \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void convert(const double* g, const double* h, float* gf, float* hf, size_t b, size_t e, int T) {
  std::vector<std::thread> th;
  const size_t n = e - b;
  for (int t = 0; t < T; ++t) {
    th.emplace_back([=] {
      const size_t s = b + n * t / T, f = b + n * (t + 1) / T;
      for (size_t i = s; i < f; ++i) {
        gf[i] = static_cast<float>(g[i]);
        hf[i] = static_cast<float>(h[i]);
      }
    });
  }
  for (auto& x : th) x.join();
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? atol(argv[1]) : 10500000;
  double *g, *h;
  float *gf, *hf;
  CK(cudaMallocHost(&g, n * 8));
  CK(cudaMallocHost(&h, n * 8));
  CK(cudaMallocHost(&gf, n * 4));
  CK(cudaMallocHost(&hf, n * 4));
  std::vector<double> pg(n), ph(n);  // pageable copies
  for (size_t i = 0; i < n; ++i) g[i] = h[i] = pg[i] = ph[i] = 0.001 * (i % 997);
  void *dg, *dh;
  CK(cudaMalloc(&dg, n * 8));
  CK(cudaMalloc(&dh, n * 8));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const int hw = std::thread::hardware_concurrency();
  printf("rows %zu hw_threads %d\n", n, hw);
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now();
    CK(cudaMemcpyAsync(dg, g, n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dh, h, n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    double t1 = now();
    printf("dma64 pinned   %.3f ms  %.1f GB/s\n", (t1 - t0) * 1e3, 16.0 * n / (t1 - t0) / 1e9);
    t0 = now();
    CK(cudaMemcpyAsync(dg, pg.data(), n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dh, ph.data(), n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    t1 = now();
    printf("dma64 pageable %.3f ms  %.1f GB/s\n", (t1 - t0) * 1e3, 16.0 * n / (t1 - t0) / 1e9);
    t0 = now();
    CK(cudaMemcpyAsync(dg, gf, n * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dh, hf, n * 4, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    t1 = now();
    printf("dma32 pinned   %.3f ms  %.1f GB/s\n", (t1 - t0) * 1e3, 8.0 * n / (t1 - t0) / 1e9);
  }
  for (int T : {1, 2, 4, 8, 16, hw}) {
    double best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      double t0 = now();
      convert(g, h, gf, hf, 0, n, T);
      best = std::min(best, now() - t0);
    }
    printf("cvt T=%2d       %.3f ms  %.1f Grows/s\n", T, best * 1e3, n / best / 1e9);
  }
  for (double a : {0.2, 0.3, 0.4, 0.5}) {
    double best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      const size_t m = static_cast<size_t>(a * n);
      double t0 = now();
      CK(cudaMemcpyAsync(dg, g, m * 8, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(dh, h, m * 8, cudaMemcpyHostToDevice, s));
      // convert the rest in 4 chunks, each copied as soon as it is ready
      const int C = 4;
      for (int c = 0; c < C; ++c) {
        const size_t b = m + (n - m) * c / C, e = m + (n - m) * (c + 1) / C;
        convert(g, h, gf, hf, b, e, hw);
        CK(cudaMemcpyAsync(static_cast<float*>(dg) + b, gf + b, (e - b) * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(static_cast<float*>(dh) + b, hf + b, (e - b) * 4, cudaMemcpyHostToDevice, s));
      }
      CK(cudaStreamSynchronize(s));
      best = std::min(best, now() - t0);
    }
    printf("hybrid a=%.1f   %.3f ms\n", a, best * 1e3);
  }
  return 0;
}
