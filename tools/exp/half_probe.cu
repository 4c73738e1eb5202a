// Experiment (not product code): does a warp running two independent latency chains in its two half-warps
// (divergent per iteration) beat one chain per warp?  Mimics K1's structure: a warp-min (REDUX) per
// iteration, then one of two handler bodies (shuffles + shared-memory loads + ALU) chosen per chain.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned body(unsigned x, const unsigned* sm, int lane, unsigned mask, int src0) {
#pragma unroll 1
  for (int k = 0; k < 6; ++k) {
    x = __shfl_sync(mask, x, src0 + (k & 7)) * 2654435761u + lane;
    x ^= sm[(x >> 7) & 255];
  }
  return x;
}
template <bool HALF>
__global__ void chain(unsigned* out, int iters) {
  __shared__ unsigned sm[256 * 16];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) sm[i] = i * 2654435761u;
  __syncthreads();
  const unsigned* s = sm + 256 * (w & 15);
  const unsigned hb = HALF ? (lane & 16) : 0, HM = HALF ? (0xFFFFu << hb) : 0xFFFFFFFFu;
  unsigned x = threadIdx.x + blockIdx.x * 977u, acc = 0;
  for (int it = 0; it < iters; ++it) {
    const unsigned d = __reduce_min_sync(HM, x & 0xFFFF);
    const bool which = ((d + it + (hb >> 4)) & 1) != 0;   // halves diverge about half the time
    if (which) x = body(x + d, s, lane, HM, hb);
    else x = body(x ^ d, s + 128, lane, HM, hb) + 7;
    acc += x;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  unsigned* o;
  cudaMalloc(&o, 148 * 8 * 256 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    float t1, t2;
    // one chain per warp: 16 warps/SM, `iters` iterations each
    cudaEventRecord(a);
    chain<false><<<148 * 2, 256>>>(o, 20000);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&t1, a, b);
    // two chains per warp (half-warps): same 16 warps/SM, same iterations -> twice the chains
    cudaEventRecord(a);
    chain<true><<<148 * 2, 256>>>(o, 20000);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&t2, a, b);
    printf("one chain/warp %.2f ms; two chains/warp %.2f ms -> chains per ms %.3fx\n", t1, t2, 2.0 * t1 / t2);
  }
  return 0;
}
