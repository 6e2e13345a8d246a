// Cost of the wave grower's replay loop in isolation (sm_100a): warp 0 of one
// CTA, an open-leaf pool of `nfr` entries in shared memory, `commits`
// iterations of {argmax over the pool (redux.sync keys), commit bookkeeping};
// cycles per commit by clock64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o replay replay.cu
#include <cstdio>

struct S {
  unsigned long long fkey[256], gkey[1280];
  short fnode[256], fout[256], kid[1280];
  unsigned char later[256];
  short cnode[256], ckid[256], cout[256];
};

__global__ void k(int nfr0, int commits, long long* out, int mode) {
  __shared__ S w;
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1280; i += blockDim.x) {
    w.gkey[i] = 1000000ull + (i * 7919u) % 100000u;
    w.kid[i] = static_cast<short>(i < 1000 ? 2 * i + 300 : -1);  // expanded nodes
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    w.fkey[i] = i < nfr0 ? w.gkey[i] : 0;
    w.fnode[i] = static_cast<short>(i);
    w.fout[i] = static_cast<short>(i);
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  int nfr = nfr0, committed = 0;
  const long long t0 = clock64();
  for (int it = 0; it < commits; ++it) {
    unsigned long long hk = 0;
    unsigned lk = 0;
    int idx = -1;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = u * 32 + lane + ((mode & 2) ? 1000 : 0);
      const unsigned long long h = i < nfr ? w.fkey[i] : 0ull;  // (mode 2: no loads)
      const unsigned l = i < nfr ? 0xFFFFFFFFu - static_cast<unsigned>(w.fout[i]) : 0u;
      const bool take = h > hk || (h == hk && l > lk);
      hk = take ? h : hk;
      lk = take ? l : lk;
      idx = take ? i : idx;
    }
    const unsigned h1 = static_cast<unsigned>(hk >> 32), h0 = static_cast<unsigned>(hk);
    const unsigned m1 = __reduce_max_sync(0xffffffffu, h1);
    const unsigned m0 = __reduce_max_sync(0xffffffffu, h1 == m1 ? h0 : 0u);
    const unsigned Lk = __reduce_max_sync(0xffffffffu, h1 == m1 && h0 == m0 ? lk : 0u);
    const unsigned long long H = (static_cast<unsigned long long>(m1) << 32) | m0;
    const unsigned bal = __ballot_sync(0xffffffffu, hk == H && lk == Lk);
    const int e = __shfl_sync(0xffffffffu, idx, __ffs(bal) - 1);
    const int x = w.fnode[e];
    const int kd = w.kid[x] & 1023;
    if (lane == 0 && !(mode & 1)) {
      const int o = w.fout[e];
      w.cnode[committed & 255] = static_cast<short>(x);
      w.ckid[committed & 255] = static_cast<short>(kd);
      w.cout[committed & 255] = static_cast<short>(o);
      w.later[committed & 255] = 0;
      if (o > 0) w.later[((o - 1) >> 1) & 255] |= static_cast<unsigned char>(1 << ((o - 1) & 1));
      const int t = nfr - 1;
      w.fkey[e] = w.fkey[t];
      w.fnode[e] = w.fnode[t];
      w.fout[e] = w.fout[t];
      int m = t;
      for (int c = 0; c < 2; ++c) {
        if (w.gkey[kd + c] == 0ull) continue;
        w.fkey[m] = w.gkey[kd + c] - 1000;
        w.fnode[m] = static_cast<short>(kd + c);
        w.fout[m] = static_cast<short>((2 * committed + 1 + c) & 511);
        ++m;
      }
    }
    __syncwarp();
    nfr += 1;
    if (nfr > 250) nfr = 200;
    ++committed;
  }
  const long long t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / commits + (nfr == -1);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int nfr : {16, 250}) {
    for (int mode : {0, 1, 2, 3}) {
      const int threads = 32;
      k<<<1, threads>>>(nfr, 200, d, mode);
      long long h = 0;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("pool %3d, mode %d (1: no commit block, 2: no pool loads): %lld cycles per commit (%s)\n", nfr, mode, h,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
