// Shared-memory primitive costs on sm_100a for the histogram update, measured
// as cycles per warp-instruction (one instruction = 32 lanes on 32 distinct
// banks, so every figure is the conflict-free cost). Each mode issues N_OPS
// independent updates per iteration from a register LCG (no global traffic).
//
//   lds_sts64 : LDS.64 + STS.64 (the {g,h} fp32 read-modify-write)      -> 2 x 64-bit
//   lds_sts32 : LDS.32 + STS.32                                          -> 2 x 32-bit
//   popc_inc  : atomicAdd(u32, 1) -> ATOMS.POPC.INC (the count)
//   red_u32   : red.shared.add.u32 of a lane value (no return)
//   atom_u32  : atom.shared.add.u32 with the old value used
//   red_f32   : atomicAdd(float) on shared (CAS loop)
//   rmw5_p20  : the full update (LDS.64/FADD/STS.64 + POPC.INC) with each lane
//               active with probability 0.2 (bin-0 elision on Bosch-like data)
//   rmw5      : the same with every lane active
//   match_agg : __match_any_sync on (feature, bin) of one feature column, the
//               group leader adds the group's sum (the north_star's warp-
//               aggregation option); bins uniform over K
//
// All cells are CTA-shared except lds_sts (per-warp private, as the kernel).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_primitives smem_primitives.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

__device__ __forceinline__ uint32_t lcg(uint32_t& s) {
  s = s * 1664525u + 1013904223u;
  return s >> 20;
}

template <int MODE, int K>
__global__ void kern(float* out, unsigned long long* cycles, int warps_priv) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int CELLS = K * 32;
  uint32_t* shared_cells = reinterpret_cast<uint32_t*>(smem);  // CELLS x 4 B
  float2* priv = reinterpret_cast<float2*>(smem + CELLS * 4) + (warp % warps_priv) * CELLS;
  const int total16 = (CELLS * 4 + warps_priv * CELLS * 8) / 16;
  for (int i = threadIdx.x; i < total16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(shared_cells));
  const uint32_t pbase = static_cast<uint32_t>(__cvta_generic_to_shared(priv));
  uint32_t s = blockIdx.x * 7919u + threadIdx.x * 104729u;
  const float g = 0.25f + lane;
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
    const uint32_t b = lcg(s) & (K - 1);
    const uint32_t c = b * 32 + lane;
    if (MODE == 0) {
      float x, y;
      asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(pbase + c * 8));
      x += g;
      y += g;
      asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(pbase + c * 8), "f"(x), "f"(y));
    } else if (MODE == 1) {
      float x;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(pbase + c * 4));
      x += g;
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(pbase + c * 4), "f"(x));
    } else if (MODE == 2) {
      atomicAdd(shared_cells + c, 1u);
    } else if (MODE == 3) {
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(sbase + c * 4), "r"(s) : "memory");
    } else if (MODE == 4) {
      uint32_t old;
      asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(sbase + c * 4), "r"(s) : "memory");
      acc += old;
    } else if (MODE == 5) {
      atomicAdd(reinterpret_cast<float*>(shared_cells) + c, g);
    } else if (MODE == 7 || MODE == 8) {
      const bool on = MODE == 8 || ((lcg(s) & 1023u) < 205u);
      if (on) {
        float x, y;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(pbase + c * 8));
        x += g;
        y += g;
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(pbase + c * 8), "f"(x), "f"(y));
        atomicAdd(shared_cells + c, 1u);
      }
    } else if (MODE == 9) {  // red.shared.add.u32, 20% of the lanes active
      if ((lcg(s) & 1023u) < 205u) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(sbase + c * 4), "r"(s) : "memory");
    } else if (MODE == 10 || MODE == 11) {  // red.shared.add.u64 (all / 20% lanes)
      if (MODE == 10 || (lcg(s) & 1023u) < 205u)
        asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(sbase + c * 8), "l"(static_cast<unsigned long long>(s))
                     : "memory");
    } else if (MODE == 12 || MODE == 13) {
      // the CTA-shared fixed-point update: g and h as int64 (64-bit reds),
      // count (POPC.INC) — all lanes / 20% of the lanes (bin-0 elision)
      if (MODE == 12 || (lcg(s) & 1023u) < 205u) {
        const unsigned long long q = static_cast<unsigned long long>(s) * 2654435761ull;
        asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(sbase + c * 8), "l"(q) : "memory");
        asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(sbase + CELLS * 8 + c * 8), "l"(q >> 3) : "memory");
        atomicAdd(shared_cells + 4 * CELLS + c, 1u);
      }
    } else if (MODE == 6) {
      // all lanes on one feature column (f = it & 31): aggregate equal bins
      const uint32_t cell = b * 32 + (it & 31);
      const uint32_t peers = __match_any_sync(0xffffffffu, cell);
      const int leader = __ffs(peers) - 1;
      // segmented sum over the group: each lane adds the values of the group
      // members via a loop over the set bits (the group's members are known)
      float sum = 0.f;
      uint32_t m = peers;
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        sum += __shfl_sync(peers, g, src);
      }
      if (lane == leader) {
        float x;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(pbase + cell * 4));
        x += sum;
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(pbase + cell * 4), "f"(x));
      }
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  float a = static_cast<float>(acc);
  for (int i = threadIdx.x; i < CELLS; i += blockDim.x) a += shared_cells[i] + priv[i].x;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE, int K>
void run(const char* name, int sms, int warps, int warps_priv, double wf_per_op) {
  const size_t smem = static_cast<size_t>(K) * 32 * 4 * (MODE >= 10 ? 5 : 1) + static_cast<size_t>(warps_priv) * K * 32 * 8;
  auto fn = kern<MODE, K>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, sms * warps * 32 * sizeof(float));
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  fn<<<sms, warps * 32, smem>>>(out, cyc, warps_priv);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fn<<<sms, warps * 32, smem>>>(out, cyc, warps_priv);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c[1024];
  cudaMemcpy(c, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += c[i];
  avg /= sms;
  const double warp_ops = double(warps) * ITERS;  // warp-instructions (updates / 32) per SM
  cudaError_t err = cudaGetLastError();
  printf("%-10s K%-3d warps %2d  cycles/warp-op %6.3f  (ideal-wavefront model %.1f)  lane-updates/clk/SM %6.2f  %.3f ms %s\n",
         name, K, warps, avg / warp_ops, wf_per_op, 32.0 * warp_ops / avg, ms,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d, iters %d\n", sms, ITERS);
  for (int w : {8, 16, 32}) {
    const int wp = w <= 16 ? w : 16;
    run<0, 32>("lds_sts64", sms, w, wp, 4);
    run<1, 32>("lds_sts32", sms, w, wp, 2);
    run<2, 64>("popc_inc", sms, w, 1, 1);
    run<3, 64>("red_u32", sms, w, 1, 1);
    run<4, 64>("atom_u32", sms, w, 1, 1);
    run<5, 64>("red_f32", sms, w, 1, 1);
    run<6, 32>("match_agg", sms, w, wp, 0);
    run<8, 32>("rmw5", sms, w, wp, 5);
    run<7, 32>("rmw5_p20", sms, w, wp, 5);
    run<9, 64>("red_u32_p20", sms, w, 1, 1);
    run<10, 64>("red_u64", sms, w, 1, 2);
    run<11, 64>("red_u64_p20", sms, w, 1, 2);
    run<12, 64>("fx64_upd", sms, w, 1, 5);
    run<13, 64>("fx64_p20", sms, w, 1, 5);
  }
  return 0;
}
