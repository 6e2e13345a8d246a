// Distributed-shared-memory (thread-block-cluster) update-rate microbenchmark
// for the histogram inner loop on sm_100a — the "cluster DSMEM" option of
// BASELINE.json's north_star, measured against the local shared-memory RMW the
// histogram kernel uses (microbench/smem_update.cu has the local primitives).
//
// sm_100a has no native local shared fp32 atomic (atomicAdd(float) on
// __shared__ is an ATOMS.CAST.SPIN loop), but red.shared::cluster.add.f32 to a
// PARTNER CTA's shared memory compiles to a native ATOM.E.ADD.F32 (with a CAS
// fallback taken only when the address is the issuing CTA's own window).
// Question: does routing part of the {g,h,count} traffic through the cluster
// network raise the update rate beyond the local pipe's 5 wavefronts / 32
// updates?
//
// Modes (every CTA of a 2-CTA cluster runs the same mode; partner = rank ^ 1):
//   0 local    : per-warp LDS.64 {g,h} + FADD x2 + STS.64, ATOMS.POPC.INC count
//   1 dsm_gh   : red.shared::cluster.add.f32 g,h to the partner; local count
//   2 dsm_ghc  : g, h and count all remote
//   3 mix50    : alternate iterations between 0 and 1
//   4 mix25    : one in four iterations remote (mode 1), the rest local
//   5 dsm_i32  : red.shared::cluster.add.u32 x3 (fixed-point g,h + count)
//   6 dsm_gh_c4: as 1 with 4-CTA clusters, partner = rank ^ 1
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_update dsmem_update.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

constexpr int ITERS = 4096;

__device__ __forceinline__ uint32_t lcg(uint32_t& s) {
  s = s * 1664525u + 1013904223u;
  return s >> 26;
}

__device__ __forceinline__ void red_f32_cluster(uint32_t a, float v) {
  asm volatile("red.shared::cluster.add.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void red_u32_cluster(uint32_t a, uint32_t v) {
  asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

template <int MODE, int K, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) kern(float* out, unsigned long long* cycles) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int CELLS = K * 32;
  // layout: [shared remote-target gh: CELLS float2][shared cnt: CELLS u32][per-warp private gh]
  float2* shared_gh = reinterpret_cast<float2*>(smem);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + CELLS * 8);
  float2* priv = reinterpret_cast<float2*>(smem + CELLS * 12) + warp * CELLS;
  const int total16 = (CELLS * 12 + WARPS * CELLS * 8) / 16;
  for (int i = threadIdx.x; i < total16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  cluster.sync();
  const uint32_t partner = cluster.block_rank() ^ 1u;
  const uint32_t rgh = mapa(static_cast<uint32_t>(__cvta_generic_to_shared(shared_gh)), partner);
  const uint32_t rcnt = mapa(static_cast<uint32_t>(__cvta_generic_to_shared(cnt)), partner);
  const uint32_t lpriv = static_cast<uint32_t>(__cvta_generic_to_shared(priv));
  uint32_t s = blockIdx.x * 7919u + threadIdx.x * 104729u;
  const float g = 0.25f + lane, h = 0.5f;
  const uint32_t gi = lane + 1, hi = 3;
  unsigned long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
    const uint32_t b = lcg(s) & (K - 1);
    const uint32_t c = b * 32 + lane;
    bool remote;
    if (MODE == 0) remote = false;
    else if (MODE == 3) remote = it & 1;
    else if (MODE == 4) remote = (it & 3) == 0;
    else remote = true;
    if (!remote) {
      float x, y;
      asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(lpriv + c * 8));
      x += g;
      y += h;
      asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(lpriv + c * 8), "f"(x), "f"(y));
      atomicAdd(cnt + c, 1u);
    } else if (MODE == 5) {
      red_u32_cluster(rgh + c * 8, gi);
      red_u32_cluster(rgh + c * 8 + 4, hi);
      red_u32_cluster(rcnt + c * 4, 1u);
    } else {
      red_f32_cluster(rgh + c * 8, g);
      red_f32_cluster(rgh + c * 8 + 4, h);
      if (MODE == 2) red_u32_cluster(rcnt + c * 4, 1u);
      else atomicAdd(cnt + c, 1u);
    }
  }
  unsigned long long t1 = clock64();
  cluster.sync();
  float acc = 0.f;
  for (int i = threadIdx.x; i < CELLS; i += blockDim.x) acc += shared_gh[i].x + priv[i % CELLS].y + cnt[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE, int K = 64, int WARPS = 8, int CL = 2>
void run(const char* name, int sms) {
  const size_t smem = static_cast<size_t>(K) * 32 * 12 + static_cast<size_t>(WARPS) * K * 32 * 8;
  auto fn = kern<MODE, K, WARPS>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int grid = sms / CL * CL;
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, grid * WARPS * 32 * sizeof(float));
  cudaMalloc(&cyc, grid * sizeof(unsigned long long));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(WARPS * 32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, fn, out, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) cudaLaunchKernelEx(&cfg, fn, out, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  unsigned long long c[1024];
  cudaMemcpy(c, cyc, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += c[i];
  avg /= grid;
  const double upd = double(WARPS) * 32 * ITERS;
  cudaError_t err = cudaGetLastError();
  printf("K%-3d W%-2d CL%d %-9s upd/clk/SM %6.2f  (%.0f cyc/CTA, %.4f ms, chip %.1f Gupd/s) %s\n", K, WARPS, CL, name,
         upd / avg, avg, ms, upd * grid / (ms * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d, iters %d\n", sms, ITERS);
  run<0>("local", sms);
  run<1>("dsm_gh", sms);
  run<2>("dsm_ghc", sms);
  run<3>("mix50", sms);
  run<4>("mix25", sms);
  run<5>("dsm_i32", sms);
  run<1, 64, 8, 4>("dsm_gh", sms);
  run<0, 32, 16>("local", sms);
  run<1, 32, 16>("dsm_gh", sms);
  run<3, 32, 16>("mix50", sms);
  run<4, 32, 16>("mix25", sms);
  run<1, 32, 24>("dsm_gh", sms);
  run<0, 32, 24>("local", sms);
  run<4, 32, 24>("mix25", sms);
  return 0;
}
