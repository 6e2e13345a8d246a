// Grid-barrier latency on sm_100a: one CTA per SM (cooperative launch), N
// back-to-back barriers, ns per barrier. Variants:
//   0 fence.sc + atomicAdd arrival, ld.acquire poll, fence after (the
//     persistent tree grower's first version)
//   1 atom.add.acq_rel.gpu arrival, ld.acquire poll, no extra fences
//   2 as 1 with __nanosleep(32) backoff in the poll
//   3 as 1 with the arrival counter striped: per-CTA flags, last-arriver found
//     through one counter but release through a per-generation flag
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o grid_barrier grid_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int V>
__device__ __forceinline__ void barrier(unsigned* bar) {
  __shared__ unsigned s_gen;
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    s_gen = ld_acquire(bar + 1);
    unsigned prev;
    if (V == 0) {
      __threadfence();
      prev = atomicAdd(bar, 1u);
    } else {
      prev = atom_add_acq_rel(bar, 1u);
    }
    s_last = prev == gridDim.x - 1;
    if (s_last) {
      bar[0] = 0;
      if (V == 0) {
        __threadfence();
        atomicAdd(bar + 1, 1u);
      } else {
        red_release(bar + 1, 1u);
      }
    } else {
      while (ld_acquire(bar + 1) == s_gen) {
        if (V == 2) __nanosleep(32);
      }
    }
    if (V == 0) __threadfence();
  }
  __syncthreads();
}

template <int V>
__global__ void kern(unsigned* bar, int iters, unsigned long long* out) {
  unsigned long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) barrier<V>(bar);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    *out = t1 - t0;
  }
}

__global__ void cg_kern(int iters, unsigned long long* out) {
  auto grid = cooperative_groups::this_grid();
  unsigned long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    *out = t1 - t0;
  }
}

template <int V>
void run(unsigned* bar, unsigned long long* out, int sms, int threads) {
  int iters = 2000;
  void* args[] = {&bar, &iters, &out};
  cudaMemset(bar, 0, 8);
  cudaLaunchCooperativeKernel((void*)kern<V>, sms, threads, args, 0, 0);
  cudaMemset(bar, 0, 8);
  cudaLaunchCooperativeKernel((void*)kern<V>, sms, threads, args, 0, 0);
  unsigned long long ns = 0;
  cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
  printf("variant %d threads %d: %.0f ns / barrier  (%s)\n", V, threads, double(ns) / iters,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* bar;
  unsigned long long* out;
  cudaMalloc(&bar, 8);
  cudaMalloc(&out, 8);
  for (int threads : {256, 512}) {
    run<0>(bar, out, sms, threads);
    run<1>(bar, out, sms, threads);
    run<2>(bar, out, sms, threads);
    int iters = 2000;
    void* args[] = {&iters, &out};
    cudaLaunchCooperativeKernel((void*)cg_kern, sms, threads, args, 0, 0);
    cudaLaunchCooperativeKernel((void*)cg_kern, sms, threads, args, 0, 0);
    unsigned long long ns = 0;
    cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
    printf("cg grid.sync threads %d: %.0f ns / barrier (%s)\n", threads, double(ns) / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
