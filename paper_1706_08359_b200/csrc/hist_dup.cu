// hist_dup.cu — the feature histogram for a dataset
// whose only slice group holds M < 32 features (Higgs: M = 28), without the
// 32 - M pad slots of the 32-step rotated schedule (hist_kernels.cu).
//
// The 32-step kernel gives every lane one row and rotates the row's 32-slot
// slice so that at step p the 32 lanes address 32 distinct feature columns
// (= 32 distinct banks): bank-conflict-free for any bins. With M = 28 real
// features, 4 of the 32 slots of every row are pads: 12.5% of the shared-
// memory read-modify-writes — the resource that bounds the kernel
// — do no work.
//
// Here a 32-row tile takes M steps. Lane l < M updates feature (l + p) mod M
// of its row at step p; lane M + j (j < U = 32 - M) updates feature (j + p)
// mod M of ITS row, i.e. the same feature as lane j. Every feature therefore
// has two cell homes per bin: home 1 in bank f, home 2 in bank f + U (a second
// [bin][32] array). Lane j (< U) uses home 1, lane M + j home 2, and every
// other lane uses home 2 exactly when its feature lies "after" the duplicated
// one of its residue class (f > d_c, d_c the step's duplicate with f = d_c mod
// U) — the shift chain d_c -> d_c + U -> ... ends in the free banks M..31. So
// every step addresses all 32 banks once (checked exhaustively for M = 28, 24,
// 16): 32 useful updates per conflict-free instruction instead of M.
//
// Cost: two homes double the per-warp cells (g and h as separate fp32 arrays,
// LDS.32/STS.32: the 32-bank rule, not the half-warp one of LDS.64), so fewer
// warps fit; R rows per lane restore the independent read-modify-write chains.
// The fold adds both homes per warp, warps in a fixed order: deterministic,
// and the per-CTA partials have the 32-step kernel's layout, so the same
// reduction (or direct output) follows.
#include <cstdint>
#include <mutex>

#include "hbg_internal.h"
#include "hist_device.cuh"

namespace hbg {

namespace {

using namespace dev;

// Rotate the first M/4 words of an 8-bit slice by r bytes (mod M): feature
// (r + p) mod M lands at byte p.
template <int M>
__device__ __forceinline__ void rotate_mod(Slice<8>& s, int r) {
  constexpr int W = M / 4;
  const int q = r >> 2;
  const int sh = (r & 3) * 8;
  uint32_t t[W];
#pragma unroll
  for (int step = 4; step >= 1; step >>= 1) {
    if (step >= W) continue;
    const bool on = (q & step) != 0;
#pragma unroll
    for (int j = 0; j < W; ++j) t[j] = on ? s.w[(j + step) % W] : s.w[j];
#pragma unroll
    for (int j = 0; j < W; ++j) s.w[j] = t[j];
  }
#pragma unroll
  for (int j = 0; j < W; ++j) t[j] = __funnelshift_r(s.w[j], s.w[(j + 1) % W], sh);
#pragma unroll
  for (int j = 0; j < W; ++j) s.w[j] = t[j];
}

__device__ __forceinline__ float lds_f(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v)); }
// Count increment (ATOMS.POPC.INC), predicated in the instruction itself: a
// branch around it would put the step under a convergence barrier.
__device__ __forceinline__ void atoms_inc(uint32_t a, uint32_t on) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %1, 0; @p red.shared.add.u32 [%0], 1; }" ::"r"(a), "r"(on) : "memory");
}

// Byte offset of lane `lane`'s step-p cell for bin b: home 1 at column f of
// the first [K][32] array, home 2 at column f + U of the second (kHome bytes
// further). p is a constant after unrolling, so the home rule folds to one or
// two compares per lane.
template <int M, uint32_t kHome>
__device__ __forceinline__ uint32_t cell_rel(int p, int lane, int rot, uint32_t b) {
  constexpr int U = 32 - M;
  int f = rot + p;
  f = f >= M ? f - M : f;
  bool h2;
  if (p + U <= M) {  // the step's duplicates p..p+U-1 do not wrap
    h2 = lane >= M || (lane >= U && lane + p < M);
  } else {  // they wrap: classes of the low duplicates shift
    h2 = lane >= M || (lane >= U && ((lane + p) & (U - 1)) < p + U - M);
  }
  return (b << 7) + (static_cast<uint32_t>(f) << 2) + (h2 ? kHome + (U << 2) : 0u);
}

template <int K, int M, int R, bool kRowIndexed>
__global__ void __launch_bounds__(256, 1) hist_dup_kernel(HistArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int U = 32 - M;
  constexpr uint32_t kHome = K * 32 * 4;  // one [K][32] 4-byte array
  const int warps = blockDim.x >> 5;
  {
    const int n16 = (warps * 4 + 2) * static_cast<int>(kHome) / 16;
    uint4* z = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const float* __restrict__ ag = static_cast<const float*>(a.g);
  const float* __restrict__ ah = static_cast<const float*>(a.h);
  const int seg = blockIdx.x;
  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rot = lane < M ? lane : lane - M;
  {
    const int64_t s0 = static_cast<int64_t>(seg) * a.seg_len;
    const int64_t s1 = min(s0 + a.seg_len, a.n);
    // per warp: g home 1 | g home 2 | h home 1 | h home 2; then the CTA's counts home 1 | home 2
    const uint32_t gbase = smem_addr(smem) + static_cast<uint32_t>(w) * 4 * kHome;
    const uint32_t cbase = smem_addr(smem) + static_cast<uint32_t>(warps) * 4 * kHome;
    const unsigned char* base = a.packed;
    const int64_t step = static_cast<int64_t>(warps) * 32 * R;

    auto fetch_entry = [&](int64_t t, int32_t (&row)[R], float (&g)[R], float (&h)[R]) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t pos = t + 32 * r + lane;
        if (pos < s1) {
          row[r] = __ldg(a.idx + pos);
          if constexpr (!kRowIndexed) {
            g[r] = __ldg(ag + pos);
            h[r] = __ldg(ah + pos);
          }
        } else {
          row[r] = -1;
          g[r] = 0.f;
          h[r] = 0.f;
        }
      }
    };
    auto fetch_slice = [&](const int32_t (&row)[R], float (&g)[R], float (&h)[R], Slice<8> (&sl)[R]) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (row[r] >= 0) {
          if constexpr (kRowIndexed) {
            g[r] = __ldg(ag + row[r]);
            h[r] = __ldg(ah + row[r]);
          }
          load_slice<8>(base + static_cast<int64_t>(row[r]) * a.row_stride, sl[r]);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) sl[r].w[j] = 0;
        }
      }
    };

    int64_t t = s0 + static_cast<int64_t>(w) * 32 * R;
    int32_t r0[R], r1[R];
    float g0[R], h0[R], g1[R], h1[R];
    Slice<8> cur[R];
    fetch_entry(t, r0, g0, h0);
    fetch_entry(t + step, r1, g1, h1);
    fetch_slice(r0, g0, h0, cur);
    for (; t < s1; t += step) {
      int32_t r2[R];
      float g2[R], h2[R];
      Slice<8> nxt[R];
      fetch_entry(t + 2 * step, r2, g2, h2);
      fetch_slice(r1, g1, h1, nxt);
#pragma unroll
      for (int r = 0; r < R; ++r) rotate_mod<M>(cur[r], rot);
      // Rows past the leaf's end (row -1) carry bin 0 and g = h = 0: their
      // read-modify-writes store the cell's value back unchanged (no other
      // lane touches that cell in the step), so only their count is masked —
      // no branch, no divergence inside the step sequence.
      uint32_t act[R];
#pragma unroll
      for (int r = 0; r < R; ++r) act[r] = r0[r] >= 0 ? 1u : 0u;
#pragma unroll
      for (int p = 0; p < M; ++p) {
        asm volatile("bar.warp.sync -1;" ::: "memory");
        uint32_t rel[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t b = (cur[r].w[p / 4] >> (8 * (p % 4))) & (K - 1);
          rel[r] = cell_rel<M, kHome>(p, lane, rot, b);
        }
        float x[R], y[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          x[r] = lds_f(gbase + rel[r]);
          y[r] = lds_f(gbase + 2 * kHome + rel[r]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
          for (int q = 0; q < r; ++q) {
            if (rel[q] == rel[r]) {  // the later row builds on the earlier sum
              x[r] = x[q];
              y[r] = y[q];
            }
          }
          x[r] += g0[r];
          y[r] += h0[r];
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          sts_f(gbase + rel[r], x[r]);
          sts_f(gbase + 2 * kHome + rel[r], y[r]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) atoms_inc(cbase + rel[r], act[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        r0[r] = r1[r];
        g0[r] = g1[r];
        h0[r] = h1[r];
        r1[r] = r2[r];
        g1[r] = g2[r];
        h1[r] = h2[r];
        cur[r] = nxt[r];
      }
    }
  }
  __syncthreads();

  // Fold: cell (bin, f < M) = sum over warps in order of home 1 + home 2.
  const float* cells = reinterpret_cast<const float*>(smem);
  const uint32_t* cnt = reinterpret_cast<const uint32_t*>(smem + static_cast<size_t>(warps) * 4 * kHome);
  constexpr int kWords = K * 32;  // words per [K][32] array
  auto fold = [&](int bin, int f, float& sg, float& sh, uint32_t& sc) {
    sg = 0.f;
    sh = 0.f;
    const int c1 = bin * 32 + f, c2 = c1 + U;
    for (int s = 0; s < warps; ++s) {
      const float* wc = cells + static_cast<size_t>(s) * 4 * kWords;
      sg += wc[c1];
      sg += wc[kWords + c2];
      sh += wc[2 * kWords + c1];
      sh += wc[3 * kWords + c2];
    }
    sc = cnt[c1] + cnt[kWords + c2];
  };
  if (a.direct) {
    const int total = M * a.max_bin;
    const size_t D = static_cast<size_t>(M) * a.max_bin;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int f = i / a.max_bin, bin = i - f * a.max_bin;
      float sg, sh;
      uint32_t sc;
      fold(bin, f, sg, sh, sc);
      const double vg = sg, vh = sh, vc = sc;
      a.out[i] = vg;
      a.out[D + i] = vh;
      a.out[2 * D + i] = vc;
      if (a.parent) {
        const double pg = a.parent[i], ph = a.parent[D + i], pc = a.parent[2 * D + i];
        a.sibling[i] = pg - vg;
        a.sibling[D + i] = ph - vh;
        a.sibling[2 * D + i] = pc - vc;
      }
    }
    return;
  }
  float* part_g = static_cast<float*>(a.part_g);
  float* part_h = static_cast<float*>(a.part_h);
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) {  // [bin][32], pad columns 0
    const int bin = i >> 5, f = i & 31;
    float sg = 0.f, sh = 0.f;
    uint32_t sc = 0;
    if (f < M) fold(bin, f, sg, sh, sc);
    const size_t o = static_cast<size_t>(blockIdx.x) * kWords + i;
    part_g[o] = sg;
    part_h[o] = sh;
    a.part_c[o] = sc;
  }
}

template <int K, int M, int R>
void set_attr_once(int device) {
  static std::once_flag once[64];
  std::call_once(once[device & 63], [] {
    for (const void* f : {reinterpret_cast<const void*>(hist_dup_kernel<K, M, R, false>),
                          reinterpret_cast<const void*>(hist_dup_kernel<K, M, R, true>)}) {
      HBG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
      set_max_shared_carveout(f);
    }
  });
}

template <int K, int M, int R>
void launch_t(const HistPlan& plan, const HistArgs& args, cudaStream_t s) {
  const dim3 grid(plan.ctas), block(plan.warps * 32);
  (args.gh_indexed ? hist_dup_kernel<K, M, R, true> : hist_dup_kernel<K, M, R, false>)<<<grid, block, plan.smem, s>>>(
      args);
  HBG_LAUNCH_CHECK();
}

}  // namespace

int hist_dup_rows_per_lane() {
  const char* e = std::getenv("HBG_DUP_R");
  const int r = e ? std::atoi(e) : 2;
  return r == 1 || r == 2 || r == 3 ? r : 2;
}

bool hist_dup_supported(int bits, int k_alloc, int num_groups, int d, int acc_bytes) {
  const char* e = std::getenv("HBG_HIST_DUP");
  if (e != nullptr && std::atoi(e) == 0) return false;
  return bits == 8 && k_alloc == 64 && num_groups == 1 && acc_bytes == 4 && (d == 28 || d == 24 || d == 16);
}

void configure_hist_dup(int device) {
  set_attr_once<64, 28, 1>(device);
  set_attr_once<64, 28, 2>(device);
  set_attr_once<64, 28, 3>(device);
  set_attr_once<64, 24, 2>(device);
  set_attr_once<64, 16, 2>(device);
}

void launch_histogram_dup(const HistPlan& plan, const HistArgs& args, cudaStream_t s) {
  if (plan.dup_m == 28) {
    if (plan.dup_r == 1) launch_t<64, 28, 1>(plan, args, s);
    else if (plan.dup_r == 3) launch_t<64, 28, 3>(plan, args, s);
    else launch_t<64, 28, 2>(plan, args, s);
  } else if (plan.dup_m == 24) {
    launch_t<64, 24, 2>(plan, args, s);
  } else {
    launch_t<64, 16, 2>(plan, args, s);
  }
}

}  // namespace hbg
