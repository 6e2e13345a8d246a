// hist_device.cuh — device helpers of the histogram inner loop (the rows-in-
// lanes, feature-rotated schedule), shared by the standalone
// histogram kernel (hist_kernels.cu) and the persistent tree grower
// (grow_persistent.cu). Not a public header.
#pragma once

#include <cstdint>

namespace hbg {
namespace dev {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void lds_f2(uint32_t a, float& x, float& y) {
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
}

__device__ __forceinline__ void sts_f2(uint32_t a, float x, float y) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x), "f"(y));
}

// fp64 cells of the bits64 (PrecisionMode::bits64) kernels: one 16-byte
// {g,h} pair per cell, LDS.128 / STS.128.
__device__ __forceinline__ void lds_f2(uint32_t a, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}

__device__ __forceinline__ void sts_f2(uint32_t a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y));
}

template <int BITS>
struct Slice {
  static constexpr int kWords = BITS == 8 ? 8 : 4;  // 32 features per slice
  static constexpr int kFeatPerWord = 32 / BITS;
  uint32_t w[kWords];
};

// One lane fetches its row's whole slice: a 256-bit load (LDG.E.ENL2.256,
// sm_100) for the 32-byte 8-bit slice — one L1 request per gathered row
// instead of two — and a 128-bit load for the 16-byte 4-bit slice.
template <int BITS>
__device__ __forceinline__ void load_slice(const unsigned char* p, Slice<BITS>& s) {
  if constexpr (BITS == 8) {
    asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(s.w[0]), "=r"(s.w[1]), "=r"(s.w[2]), "=r"(s.w[3]), "=r"(s.w[4]), "=r"(s.w[5]),
                   "=r"(s.w[6]), "=r"(s.w[7])
                 : "l"(p));
  } else {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
    s.w[0] = a.x;
    s.w[1] = a.y;
    s.w[2] = a.z;
    s.w[3] = a.w;
  }
}

// Rotate the 32-feature slice so that feature (lane + p) mod 32 sits at
// position p: word rotation by a lane-dependent amount (select network),
// then a funnel shift for the sub-word part.
template <int BITS>
__device__ __forceinline__ void rotate_slice(Slice<BITS>& s, int lane) {
  constexpr int W = Slice<BITS>::kWords;
  const int fpw = Slice<BITS>::kFeatPerWord;
  const int q = lane / fpw;          // whole words
  const int r = (lane % fpw) * BITS;  // bits within a word
  uint32_t t[W];
#pragma unroll
  for (int step = W / 2; step >= 1; step >>= 1) {
    const bool on = (q & step) != 0;
#pragma unroll
    for (int j = 0; j < W; ++j) t[j] = on ? s.w[(j + step) % W] : s.w[j];
#pragma unroll
    for (int j = 0; j < W; ++j) s.w[j] = t[j];
  }
#pragma unroll
  for (int j = 0; j < W; ++j) t[j] = __funnelshift_r(s.w[j], s.w[(j + 1) % W], r);
#pragma unroll
  for (int j = 0; j < W; ++j) s.w[j] = t[j];
}

// T = float (bits32: the reference's per-element fp32 cast, histogram.cpp:97-98)
// or double (bits64); a cell is the {g,h} pair of T at gh_base + cell * 2 * sizeof(T).
template <int BITS, int K, bool kTail, typename T = float>
__device__ __forceinline__ void update_step(const Slice<BITS>& s, int p, int lane, uint32_t gh_base,
                                            uint32_t* cnt, T g, T h, bool active) {
  // Lane l's step-p cell and lane (l-1)'s step-(p+1) cell can coincide, so
  // consecutive steps must be ordered across lanes: __syncwarp is the
  // warp-scope memory-ordering point for that (all lanes execute it).
  asm volatile("bar.warp.sync -1;" ::: "memory");
  if (kTail && !active) return;
  constexpr int fpw = Slice<BITS>::kFeatPerWord;
  const uint32_t b = (s.w[p / fpw] >> (BITS * (p % fpw))) & (K - 1);
  const uint32_t cell = (b << 5) | ((lane + p) & 31);
  const uint32_t a = gh_base + cell * static_cast<uint32_t>(2 * sizeof(T));
  T x, y;
  lds_f2(a, x, y);
  x += g;
  y += h;
  sts_f2(a, x, y);
  atomicAdd(cnt + cell, 1u);  // ATOMS.POPC.INC
}

// Dual-row step: lane l updates the same feature (l+p) mod 32 for its R rows.
// The R read-modify-writes are issued together (R-fold more shared-memory work
// per ordered step, i.e. more independent MIO traffic per warp); when two of
// a lane's rows hit the same cell, the later one builds on the earlier sum so
// the last store carries both.
template <int BITS, int K, int R, typename T = float>
__device__ __forceinline__ void update_step_rows(const Slice<BITS> (&s)[R], int p, int lane,
                                                 uint32_t gh_base, uint32_t* cnt, const T (&g)[R],
                                                 const T (&h)[R]) {
  asm volatile("bar.warp.sync -1;" ::: "memory");
  constexpr int fpw = Slice<BITS>::kFeatPerWord;
  constexpr uint32_t kCellBytes = 2 * sizeof(T);
  uint32_t c[R];
  T x[R], y[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t b = (s[r].w[p / fpw] >> (BITS * (p % fpw))) & (K - 1);
    c[r] = (b << 5) | ((lane + p) & 31);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) lds_f2(gh_base + c[r] * kCellBytes, x[r], y[r]);
#pragma unroll
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int q = 0; q < r; ++q) {
      if (c[q] == c[r]) {
        x[r] = x[q];
        y[r] = y[q];
      }
    }
    x[r] += g[r];
    y[r] += h[r];
  }
#pragma unroll
  for (int r = 0; r < R; ++r) sts_f2(gh_base + c[r] * kCellBytes, x[r], y[r]);
#pragma unroll
  for (int r = 0; r < R; ++r) atomicAdd(cnt + c[r], 1u);  // ATOMS.POPC.INC
}

// Rows per lane per tile (see update_step_rows). One row keeps the 13-warp
// k<=128 kernels at their measured best (the shared-memory data pipe is ~85%
// busy either way); k=256 runs 3 warps/SM and needs the extra independent work
// (4 rows per lane = 12 independent chains per SM).
// fp64 cells (bits64) take twice the shared memory per warp, so half the
// warps fit: two rows per lane at k=64 and four from k=128 restore the
// independent read-modify-write chains per SM.
template <int K, typename T = float>
__host__ __device__ constexpr int rows_per_lane() {
  return sizeof(T) == 8 ? (K >= 128 ? 4 : (K >= 64 ? 2 : 1)) : (K >= 256 ? 4 : 1);
}
__host__ inline int rows_per_lane_of(int k_alloc, int acc_bytes = 4) {
  return acc_bytes == 8 ? (k_alloc >= 128 ? 4 : (k_alloc >= 64 ? 2 : 1)) : (k_alloc >= 256 ? 4 : 1);
}

}  // namespace dev
}  // namespace hbg
