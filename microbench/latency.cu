// Latency probes for the persistent tree grower's critical path (sm_100a):
// dependent ld.global.cg chains (L2 hits, data written by another SM vs the
// same SM), fence.sc, __syncthreads with 512 threads, a 16-warp fp64 block
// sum, a 32-lane 6-field shuffle argmax. One cooperative CTA per SM; CTA 1
// measures with clock64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency latency.cu
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(inc) : "memory");
    while (((old ^ ld_acquire(bar)) & 0x80000000u) == 0) {
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void probe(int* chain, int* chain2, unsigned* bar, long long* out, int n) {
  // CTA 0 writes a random-stride chain over `chain`; CTA 1 writes chain2
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) chain[i] = (int)((i * 7919LL + 4099) % n);
  }
  if (blockIdx.x == 1) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) chain2[i] = (int)((i * 7919LL + 4099) % n);
  }
  grid_sync(bar);
  // hot spot: every CTA's warp 0 reads the same 2 KB written by CTA 0 before
  // the barrier (like the per-chunk candidates) — 4 rounds of 16 independent
  // loads per lane
  for (int round = 0; round < 4; ++round) {
    if (blockIdx.x == 0) {
      for (int i = threadIdx.x; i < 512; i += blockDim.x) chain2[n - 512 + i] = i + round;
    }
    grid_sync(bar);
    if (threadIdx.x < 32) {
      long long a0 = clock64();
      int acc = 0;
      int v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldcg(chain2 + n - 512 + u * 32 + threadIdx.x);
#pragma unroll
      for (int u = 0; u < 16; ++u) acc += v[u];
      acc = __shfl_xor_sync(0xffffffffu, acc, 1);
      long long a1 = clock64();
      if (threadIdx.x == 0 && (blockIdx.x == 1 || blockIdx.x == 100)) out[8 + 2 * round + (blockIdx.x == 100)] = a1 - a0 + (acc == -5);
    }
    grid_sync(bar);
  }
  if (blockIdx.x != 1) return;
  long long t0, t1;
  int p = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int i = 0; i < 256; ++i) p = __ldcg(chain + p);
    t1 = clock64();
    out[0] = (t1 - t0) / 256;
    t0 = clock64();
    for (int i = 0; i < 256; ++i) p = __ldcg(chain2 + p);  // written by this SM
    t1 = clock64();
    out[1] = (t1 - t0) / 256 + (p == -7);
    t0 = clock64();
    for (int i = 0; i < 64; ++i) __threadfence();
    t1 = clock64();
    out[2] = (t1 - t0) / 64;
  }
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < 64; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / 64;
  // 16-warp fp64 block sum (shuffle tree + thread 0 over 16 warps), x64
  __shared__ double sd[32];
  double v = threadIdx.x * 0.5;
  t0 = clock64();
  for (int it = 0; it < 64; ++it) {
    double x = v + it;
    for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
    if ((threadIdx.x & 31) == 0) sd[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sd[i];
      sd[31] = s;
    }
    __syncthreads();
    v += sd[31] * 1e-30;
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = (t1 - t0) / 64 + (v == -1.0);
  // warp argmax over 6 fields (gain fp64, f, b, lg, lh fp64, lc int64), x64
  if (threadIdx.x < 32) {
    double g = threadIdx.x * 1.5, lg = 1, lh = 2;
    int f = threadIdx.x, b = 3;
    long long lc = 4;
    t0 = clock64();
    for (int it = 0; it < 64; ++it) {
      for (int off = 16; off > 0; off >>= 1) {
        const double og = __shfl_xor_sync(0xffffffffu, g, off);
        const int of = __shfl_xor_sync(0xffffffffu, f, off);
        const int ob = __shfl_xor_sync(0xffffffffu, b, off);
        const double olg = __shfl_xor_sync(0xffffffffu, lg, off);
        const double olh = __shfl_xor_sync(0xffffffffu, lh, off);
        const long long olc = __shfl_xor_sync(0xffffffffu, lc, off);
        if (og > g || (og == g && of < f)) {
          g = og; f = of; b = ob; lg = olg; lh = olh; lc = olc;
        }
      }
      g += it;
    }
    t1 = clock64();
    if (threadIdx.x == 0) out[5] = (t1 - t0) / 64 + (g == -1 && f == 0 && lc == 0);
  }
  // fp64 division latency chain
  if (threadIdx.x == 0) {
    double x = 1.7;
    t0 = clock64();
    for (int i = 0; i < 64; ++i) x = 3.0 / (x + 1.0);
    t1 = clock64();
    out[6] = (t1 - t0) / 64 + (x == 0);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int n = 1 << 20;
  int *chain, *chain2;
  unsigned* bar;
  long long* out;
  cudaMalloc(&chain, n * 4);
  cudaMalloc(&chain2, n * 4);
  cudaMalloc(&bar, 4);
  cudaMalloc(&out, 128);
  cudaMemset(bar, 0, 4);
  void* args[] = {&chain, &chain2, &bar, &out, &n};
  const int smem = getenv("SMEM") ? atoi(getenv("SMEM")) : 0;
  cudaFuncSetAttribute((void*)probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  if (smem) cudaFuncSetAttribute((void*)probe, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  printf("dynamic smem %d\n", smem);
  cudaLaunchCooperativeKernel((void*)probe, sms, 512, args, smem, 0);
  long long h[16];
  cudaMemcpy(h, out, 128, cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  printf("dependent ldcg, other SM's data : %lld cycles\n", h[0]);
  printf("dependent ldcg, own SM's data   : %lld cycles\n", h[1]);
  printf("__threadfence                   : %lld cycles\n", h[2]);
  printf("__syncthreads (512 thr)         : %lld cycles\n", h[3]);
  printf("fp64 block sum (16 warps)       : %lld cycles\n", h[4]);
  printf("6-field warp argmax             : %lld cycles\n", h[5]);
  printf("fp64 div chain                  : %lld cycles\n", h[6]);
  for (int r = 0; r < 4; ++r) printf("hot-spot 2 KB read by 148 CTAs, round %d: CTA1 %lld CTA100 %lld cycles\n", r, h[8 + 2 * r], h[9 + 2 * r]);
  return 0;
}
