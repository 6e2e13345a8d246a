// The replay with the open-leaf pool kept SORTED (ascending by (gain key,
// -output id), the best last): a commit pops the last entry and inserts <= 2
// children at their ranks (warp-parallel rank count + shift). Compare with
// replay.cu (argmax over the unsorted pool per commit).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o replay_sorted replay_sorted.cu
#include <cstdio>

struct S {
  unsigned long long fkey[256], gkey[1280];
  unsigned short fout[256], fnode[256];
  short kid[1280];
  unsigned char later[256];
  short cnode[256], ckid[256], cout[256];
};

__device__ __forceinline__ bool less_entry(unsigned long long ka, unsigned oa, unsigned long long kb, unsigned ob) {
  return ka < kb || (ka == kb && oa > ob);  // lower output id ranks higher on ties
}

__global__ void k(int nfr0, int commits, long long* out) {
  __shared__ S w;
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1280; i += blockDim.x) {
    w.gkey[i] = 1000000ull + (i * 7919u) % 100000u;
    w.kid[i] = static_cast<short>(i < 1000 ? 2 * i + 300 : -1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // sorted initial pool
    for (int i = 0; i < nfr0; ++i) {
      unsigned long long kk = w.gkey[i];
      int p = i;
      while (p > 0 && less_entry(kk, i, w.fkey[p - 1], w.fout[p - 1])) {
        w.fkey[p] = w.fkey[p - 1], w.fout[p] = w.fout[p - 1], w.fnode[p] = w.fnode[p - 1];
        --p;
      }
      w.fkey[p] = kk, w.fout[p] = static_cast<unsigned short>(i), w.fnode[p] = static_cast<unsigned short>(i);
    }
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  int nfr = nfr0, committed = 0;
  const long long t0 = clock64();
  for (int it = 0; it < commits; ++it) {
    const int e = nfr - 1;  // the best
    const int x = w.fnode[e];
    const int kd = w.kid[x] & 1023;
    const unsigned o = w.fout[e];
    if (lane == 0) {
      w.cnode[committed & 255] = static_cast<short>(x);
      w.ckid[committed & 255] = static_cast<short>(kd);
      w.cout[committed & 255] = static_cast<short>(o);
      w.later[committed & 255] = 0;
      if (o > 0) w.later[((o - 1) >> 1) & 255] |= static_cast<unsigned char>(1 << ((o - 1) & 1));
    }
    nfr -= 1;  // pop
    for (int c = 0; c < 2; ++c) {
      const unsigned long long kc = w.gkey[kd + c] - 1000;
      const unsigned oc = (2 * committed + 1 + c) & 511;
      // rank = entries below the child
      int below = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = u * 32 + lane;
        below += i < nfr && less_entry(w.fkey[i], w.fout[i], kc, oc) ? 1 : 0;
      }
      const int p = __reduce_add_sync(0xffffffffu, below);
      // shift [p, nfr) up by one
      unsigned long long kk[8];
      unsigned short oo[8], nn[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = p + u * 32 + lane;
        if (i < nfr) kk[u] = w.fkey[i], oo[u] = w.fout[i], nn[u] = w.fnode[i];
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = p + u * 32 + lane;
        if (i < nfr) w.fkey[i + 1] = kk[u], w.fout[i + 1] = oo[u], w.fnode[i + 1] = nn[u];
      }
      __syncwarp();
      if (lane == 0) w.fkey[p] = kc, w.fout[p] = static_cast<unsigned short>(oc), w.fnode[p] = static_cast<unsigned short>(kd + c);
      __syncwarp();
      ++nfr;
    }
    if (nfr > 250) nfr = 200;
    ++committed;
  }
  const long long t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / commits + (nfr == -1);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int nfr : {16, 65, 128, 250}) {
    k<<<1, 32>>>(nfr, 200, d);
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("sorted pool %3d: %lld cycles per commit (%s)\n", nfr, h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
