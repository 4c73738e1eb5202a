// Dependent-chain latency of the warp collectives and shared loads on K1's critical path (one warp,
// clock64 around 1024 dependent ops).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat lat_probe.cu
#include <cstdio>
#include <cstdint>
#define N 1024
struct Tab { uint32_t v[1024]; };
__global__ void k(uint32_t* out, uint32_t seed, long long* cyc, const __grid_constant__ Tab tab) {
  __shared__ uint32_t sm[1024];
  const int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) sm[i] = (i * 7 + 3) & 1023;
  __syncwarp();
  uint32_t v = seed + lane, acc = 0;
  long long t0, t1;
#define RUN(idx, body) \
  t0 = clock64(); \
  _Pragma("unroll 1") for (int i = 0; i < N; ++i) { body; } \
  t1 = clock64(); if (lane == 0) cyc[idx] = t1 - t0; acc += v;
  RUN(0, v = v * 3u + 1u)                                            // IMAD chain (loop overhead incl.)
  RUN(1, v = __shfl_sync(0xffffffffu, v, (v & 1u)) + 1u)             // SHFL.IDX
  RUN(2, v = __ballot_sync(0xffffffffu, (v & (1u << lane)) != 0) + v)  // VOTE.ANY (ballot)
  RUN(3, v = __reduce_min_sync(0xffffffffu, v) + (uint32_t)lane)      // REDUX.MIN (CREDUX)
  RUN(4, v = sm[v & 1023u] + 1u)                                      // LDS
  RUN(5, v = (v | 1u) / ((v >> 7) | 3u) + v)                          // u32 division by a variable
  RUN(6, v = __any_sync(0xffffffffu, (v & 3u) == 0u) + v * 5u)        // VOTE.ANY predicate
  RUN(7, v = __popc(__ballot_sync(0xffffffffu, v & 1u)) + v)          // ballot + popc
  RUN(8, if (v & 1u) v += 3u; else v ^= 5u; __syncwarp())             // uniform-ish branch + syncwarp
  RUN(9, if (lane == (int)(v & 31u)) v += 7u; v = __shfl_sync(0xffffffffu, v, 0))   // lane-0 block + shfl
  { uint32_t u = __shfl_sync(0xffffffffu, v, 0);                      // warp-uniform index chain
    RUN(10, u = tab.v[u & 1023u] + 1u)                                // LDC (param space, uniform index)
    RUN(11, u = sm[u & 1023u] + 1u)                                   // LDS (uniform address)
    v += u; }
  out[lane] = v + acc;
}
int main() {
  uint32_t* o; long long* c; cudaMalloc(&o, 128); cudaMalloc(&c, 8 * 16);
  static Tab tab; for (int i = 0; i < 1024; ++i) tab.v[i] = (i * 7 + 3) & 1023;
  k<<<1, 32>>>(o, 1, c, tab); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, 1, c, tab); cudaDeviceSynchronize();
  long long h[16]; cudaMemcpy(h, c, 8 * 16, cudaMemcpyDeviceToHost);
  const char* nm[] = {"IMAD+loop", "SHFL.IDX", "ballot", "REDUX.MIN", "LDS", "udiv", "any", "ballot+popc",
                      "branch+syncwarp", "lane-if+shfl", "LDC uniform", "LDS uniform"};
  for (int i = 0; i < 12; ++i) printf("%-16s %6.1f cyc/iter\n", nm[i], (double)h[i] / N);
  return 0;
}
