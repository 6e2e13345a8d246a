// Shared-memory update-rate microbenchmark for the histogram inner loop on sm_100a.
//
// Each warp owns a private histogram region; lane l always touches column l, so
// every warp-instruction is bank-conflict-free by construction. Bins come from a
// register LCG (no global traffic) so the loop measures only the update path.
// Reports updates / clock / SM for each candidate update primitive:
//   rmw      : LDS.64 {g,h} + FADD x2 + STS.64, LDS/IADD/STS count       (plain RMW)
//   rmw_atc  : LDS.64/STS.64 {g,h} + atomicAdd(u32) count                (native ATOMS count)
//   atom_i32 : three native int32 atomicAdd (fixed-point g,h + count)
//   red_i32  : three red.shared.add.u32 (no return)
//   atom_f32 : atomicAdd(float) g,h (CAS loop on sm_100a) + atomicAdd(u32) count
//   lds_sts  : LDS.64 + STS.64 only (raw wavefront rate reference)
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_update smem_update.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ uint32_t lcg(uint32_t& s) {
  s = s * 1664525u + 1013904223u;
  return s >> 26;  // 6 bits; callers mask to K
}

template <int MODE, int K, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) kern(float* out, unsigned long long* cycles) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2* gh = reinterpret_cast<float2*>(smem) + warp * K * 32;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + WARPS * K * 32 * sizeof(float2)) + warp * K * 32;
  for (int i = threadIdx.x; i < WARPS * K * 32; i += blockDim.x) {
    reinterpret_cast<float2*>(smem)[i] = make_float2(0.f, 0.f);
    reinterpret_cast<uint32_t*>(smem + WARPS * K * 32 * sizeof(float2))[i] = 0;
  }
  __syncthreads();
  uint32_t s = blockIdx.x * 7919u + threadIdx.x * 104729u;
  float g = 0.25f + lane, h = 0.5f;
  int gi = lane + 1, hi = 3;
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    uint32_t b = lcg(s) & (K - 1);
    int a = b * 32 + lane;
    if (MODE == 0) {
      float2 v = gh[a];
      v.x += g; v.y += h;
      gh[a] = v;
      cnt[a] += 1;
    } else if (MODE == 1) {
      float2 v = gh[a];
      v.x += g; v.y += h;
      gh[a] = v;
      atomicAdd(&cnt[a], 1u);
    } else if (MODE == 2) {
      int* gi32 = reinterpret_cast<int*>(gh);
      atomicAdd(&gi32[2 * a], gi);
      atomicAdd(&gi32[2 * a + 1], hi);
      atomicAdd(&cnt[a], 1u);
    } else if (MODE == 3) {
      uint32_t* gi32 = reinterpret_cast<uint32_t*>(gh);
      uint32_t pa = static_cast<uint32_t>(__cvta_generic_to_shared(&gi32[2 * a]));
      uint32_t pc = static_cast<uint32_t>(__cvta_generic_to_shared(&cnt[a]));
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(pa), "r"(gi));
      asm volatile("red.shared.add.u32 [%0+4], %1;" ::"r"(pa), "r"(hi));
      asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(pc));
    } else if (MODE == 4) {
      float* f = reinterpret_cast<float*>(gh);
      atomicAdd(&f[2 * a], g);
      atomicAdd(&f[2 * a + 1], h);
      atomicAdd(&cnt[a], 1u);
    } else if (MODE == 5) {
      float2 v = gh[a];
      v.x += g; v.y += h;
      gh[a] = v;
    } else if (MODE == 6) {
      // packed {g,h} 64-bit RMW + count kept in the same 16B slot (LDS.128)
      float4* q = reinterpret_cast<float4*>(smem) + warp * K * 16;
      int a4 = (b * 32 + lane) >> 1;  // 16 lanes x 16B per bin row -> deliberately 2 lanes/slot? no: use own slot
      (void)a4;
      float4 v = q[(b & 31) * 32 + lane];
      v.x += g; v.y += h; v.z += 1.f;
      q[(b & 31) * 32 + lane] = v;
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  float acc = 0.f;
  for (int i = threadIdx.x; i < WARPS * K * 32; i += blockDim.x) {
    acc += reinterpret_cast<float2*>(smem)[i].x +
           reinterpret_cast<uint32_t*>(smem + WARPS * K * 32 * sizeof(float2))[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE, int K = 64, int WARPS = 8>
void run(const char* name, int sms) {
  size_t smem = WARPS * K * 32 * (sizeof(float2) + sizeof(uint32_t));
  cudaFuncSetAttribute(kern<MODE, K, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, sms * WARPS * 32 * sizeof(float));
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  kern<MODE, K, WARPS><<<sms, WARPS * 32, smem>>>(out, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<MODE, K, WARPS><<<sms, WARPS * 32, smem>>>(out, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c[1024];
  cudaMemcpy(c, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += c[i];
  avg /= sms;
  double updates_per_cta = double(WARPS) * 32 * ITERS;
  cudaError_t err = cudaGetLastError();
  printf("K%-3d W%-2d %-9s upd/clk/SM %6.2f  (%.0f cyc/CTA, %.3f ms, chip %.2f Gupd/s) %s\n", K, WARPS, name,
         updates_per_cta / avg, avg, ms, updates_per_cta * sms / (ms * 1e-3) / 1e9,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d, iters %d\n", sms, ITERS);
  run<5>("lds_sts", sms);
  run<0>("rmw", sms);
  run<1>("rmw_atc", sms);
  run<2>("atom_i32", sms);
  run<3>("red_i32", sms);
  run<4>("atom_f32", sms);
  run<6>("rmw_v4", sms);
  // more warps (TLP) with a smaller histogram
  run<0, 32, 16>("rmw", sms);
  run<1, 32, 16>("rmw_atc", sms);
  run<2, 32, 16>("atom_i32", sms);
  run<3, 32, 16>("red_i32", sms);
  run<5, 32, 16>("lds_sts", sms);
  run<0, 16, 32>("rmw", sms);
  run<2, 16, 32>("atom_i32", sms);
  return 0;
}
