// sdas_kernels.cu -- sm_100a kernels of the SDAS strategy simulator (product path).
//
// K1 k1_simulate   : persistent, one replica per warp.  Integer-tick discrete-event simulation of
//                    the model of DESIGN.md §"Model" (M0-M20): warp-min next-event selection,
//                    lane-per-instance server state in registers, shared-memory rings (inbox,
//                    in-flight, decode-wait), lane-per-sequence continuous batching with
//                    ballot/popc emission and compaction, in-loop window metrics + controller
//                    (PAPER.md:18, 58-63, 196-220, 231-238, 278-280), and a finalize that builds
//                    log-bin histograms in shared memory, selects exact nearest-rank p50/p99 from
//                    the L2-resident records by radix select, writes the 176-B summary with
//                    vector stores and merges histograms/counters into cells with integer atomics.
// K3 k3_group_argmin: per group (all C candidates of one (i,k,s)) lexicographic argmin (M20).
// K4 k4_cell_pct    : pooled cell percentile (lower bin edge) for the row objective.
// K5 k5_row_argmin  : per row (i,k) argmin over candidates on pooled cells (M20).
//
// Nothing here is a dense contraction: no tensor cores (DESIGN.md §"Roofline").

#include <cuda_runtime.h>
#include <stdint.h>

#include "sdas_internal.h"

namespace sdas {

#define FULL 0xffffffffu

__constant__ uint64_t c_log2[257];

enum : uint32_t { IDLE = 0, RECV = 1, DECODE = 2 };
enum : uint32_t { TR_ARRIVE = 1, TR_RECV_START, TR_DECODE_START, TR_RECV_DONE, TR_DECODE_DONE, TR_EMIT,
                  TR_DELIVER, TR_REQ_DONE, TR_WINDOW, TR_CONTROL, TR_ITEM_WAIT, TR_OVERFLOW };
enum : uint32_t { F_OPENS = 1, F_CLOSES = 2 };

struct TraceRec { unsigned long long tick; uint32_t code, a, b, c; };
struct SeriesRec { unsigned long long qint; uint32_t busy; uint16_t maxq; uint8_t mode, B; };
static_assert(sizeof(TraceRec) == 24 && sizeof(SeriesRec) == 16, "record sizes");

struct WarpHdr {                        // per-replica counters owned by lane 0 (read by all after __syncwarp)
  unsigned long long sum_e2e, sum_ff, sum_e2e_int;
  uint32_t admitted, dropped, completed, max_e2e;
  uint32_t n_sat, good, w_n, w_good;
  uint32_t w_half, window_closes, mode_switches, batch_changes;
  uint32_t select_changes, completed_int, rejected, good_int;   // f2 (M28, M29)
  uint32_t gate_changes, ser_slot, cell, pad2;   // ser_slot: this replica's series slot, 0xFFFFFFFF = none;
                                                 // cell: (i*K + k)*C + c
  unsigned long long pace_free[8];               // f4 M30: per link, earliest tick of the next dispatch
  uint16_t gh[3][8];   // two-level rings: head of the inbox / in-flight / wait extension per instance
};
static_assert(sizeof(WarpHdr) <= 256, "WarpHdr");

// ------------------------------------------------------------------------------ primitives
// Philox4x32-10 (rule M2): ctr = (c0, c1, c2, c3), key = (k0, k1); returns words 0 and 1.
// The rounds stay rolled: K1 is instruction-fetch bound (its hot loop sits at the 32 KB L1.5 I-cache,
// DESIGN.md §5.2), and 4-5 inlined 10-round bodies cost ~70 I-cache lines for a ~1 % saving in issue.
__device__ __forceinline__ uint2 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                        uint32_t k1) {
#pragma unroll 1
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return make_uint2(c0, c1);
}
__device__ __forceinline__ uint4 philox4(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                         uint32_t k1) {
#pragma unroll 1
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

// EXP(M; x) = floor(-M ln((x+1)/2^32)) via Q32 log2 table + linear interpolation (rule M3).
__device__ __forceinline__ unsigned long long exp_sample(unsigned long long M, uint32_t x) {
  const unsigned long long y = (unsigned long long)x + 1ull;
  const int e = 63 - __clzll(y);
  const unsigned long long f = (y << (32 - e)) - (1ull << 32);
  const uint32_t i = (uint32_t)(f >> 24);
  const unsigned long long rho = f & 0xFFFFFFull;
  const unsigned long long Ti = c_log2[i], Tn = c_log2[i + 1];
  const unsigned long long lg = Ti + (((Tn - Ti) * rho) >> 24);
  const unsigned long long n = ((unsigned long long)(32 - e) << 32) - lg;
  return __umul64hi(M * 2977044472ull, n);
}

__device__ __forceinline__ uint32_t uni(uint32_t lo, uint32_t hi, uint32_t x) {
  return lo + (uint32_t)(((unsigned long long)x * ((unsigned long long)hi - lo + 1ull)) >> 32);
}

__device__ __forceinline__ uint32_t bin_of(uint32_t v) {    // rule M17
  if (v < 16u) return v;
  const uint32_t e = 31u - __clz(v);
  return 16u + 16u * (e - 4u) + ((v >> (e - 4u)) & 15u);
}
__device__ __forceinline__ uint32_t bin_lo(uint32_t b) {
  return b < 16u ? b : ((16u + ((b - 16u) & 15u)) << ((b - 16u) >> 4));
}

// floor(n / d) for d >= 1 from M = floor(2^32 / d) (0xFFFFFFFF for d = 1, DParams.rcp_*): umulhi(n, M) is
// the quotient or one less (n M > n 2^32 / d - n), so one remainder test corrects it.  Four dependent integer
// instructions instead of the ~125-cycle division sequence.
__device__ __forceinline__ uint32_t div_rcp(uint32_t n, uint32_t d, uint32_t M) {
  const uint32_t q = __umulhi(n, M);
  return n - q * d >= d ? q + 1u : q;
}

__device__ __forceinline__ uint32_t wrap_add(uint32_t a, uint32_t b, uint32_t cap) {
  const uint32_t x = a + b;
  return x >= cap ? x - cap : x;
}
__device__ __forceinline__ uint32_t sat32(unsigned long long v) {
  return v >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)v;
}
__device__ __forceinline__ unsigned long long make_body(uint32_t slot, uint32_t flags, uint32_t tokens,
                                                        uint32_t n_in) {
  return (unsigned long long)(slot | (flags << 16)) | ((unsigned long long)(tokens | (n_in << 16)) << 32);
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += y;
  }
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// MMPP-2 next arrival after A_prev (rule M4: restart at epoch edges; epoch k lasts max(1, EXP(D_{k mod 2}))).
// Out of line: K1's hot loop sits at the instruction-cache limit and Poisson grids never
// take this path.  mm_k / mm_end: the current epoch and its end (updated).
#ifdef K1_MMPP_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
unsigned long long mmpp_next(uint32_t j, uint32_t s_coord, unsigned long long A_prev, uint32_t& mm_k,
                                                unsigned long long& mm_end, const DArr& ad, uint32_t key0,
                                                uint32_t key1) {
  unsigned long long tt = A_prev;
  for (;;) {
    while (mm_end <= tt) {
      ++mm_k;
      const uint2 w = philox(mm_k, s_coord, 4u << 16, 0u, key0, key1);
      const unsigned long long d = exp_sample((mm_k & 1) ? ad.soj1 : ad.soj0, w.x);
      mm_end += d > 0 ? d : 1ull;
    }
    const uint2 w = philox(j, s_coord, 1u << 16, mm_k, key0, key1);
    const unsigned long long gg = exp_sample((mm_k & 1) ? ad.gap1 : ad.gap0, w.x);
    if (tt + gg < mm_end) return tt + gg;
    tt = mm_end;
  }
}

// ------------------------------------------------------------------------------ K1
template <typename T>
__device__ __forceinline__ T* at(uint8_t* base, uint32_t off) {
  return reinterpret_cast<T*>(base + off);
}

#include "sdas_k1.cuh"

// ------------------------------------------------------------------------------ argmin (M20)
struct Key {
  uint32_t bad, c;
  unsigned long long dropped, p, sum, completed, makespan, good, large;
};

__device__ __forceinline__ bool rate_gt(unsigned long long na, unsigned long long ma, unsigned long long nb,
                                        unsigned long long mb) {
  // na/ma > nb/mb  <=>  na*mb > nb*ma, compared as 128-bit products; a zero makespan is rate 0 (R-RATE0)
  if (ma == 0) { na = 0; ma = 1; }
  if (mb == 0) { nb = 0; mb = 1; }
  const unsigned long long h1 = __umul64hi(na, mb), l1 = na * mb;
  const unsigned long long h2 = __umul64hi(nb, ma), l2 = nb * ma;
  return h1 != h2 ? h1 > h2 : l1 > l2;
}

__device__ bool better(const Key& a, const Key& b, uint32_t obj, unsigned long long slo) {
  if (a.bad != b.bad) return a.bad < b.bad;
  if (obj == SDAS_MAX_THROUGHPUT || obj == SDAS_MAX_GOODPUT) {
    const unsigned long long na = obj == SDAS_MAX_GOODPUT ? a.good : a.completed;
    const unsigned long long nb = obj == SDAS_MAX_GOODPUT ? b.good : b.completed;
    if (rate_gt(na, a.makespan, nb, b.makespan)) return true;
    if (rate_gt(nb, b.makespan, na, a.makespan)) return false;
    if (a.p != b.p) return a.p < b.p;
  } else if (obj == SDAS_MAX_LARGE_FRAC_UNDER_SLO) {
    const bool fa = a.dropped == 0 && a.p <= slo, fb = b.dropped == 0 && b.p <= slo;
    if (fa != fb) return fa;
    if (fa) {
      if (a.large != b.large) return a.large > b.large;
    } else if (a.dropped != b.dropped) {
      return a.dropped < b.dropped;
    }
    if (a.p != b.p) return a.p < b.p;
  } else if (obj == SDAS_MIN_P99_E2E_INTERACTIVE) {   // M29: interactive latency only
    if (a.p != b.p) return a.p < b.p;
    if (a.sum != b.sum) return a.sum < b.sum;
  } else {
    if (a.dropped != b.dropped) return a.dropped < b.dropped;
    if (a.p != b.p) return a.p < b.p;
    if (a.sum != b.sum) return a.sum < b.sum;
  }
  return a.c < b.c;
}

__device__ __forceinline__ Key shfl_key(const Key& k, int src_xor) {
  Key o;
  o.bad = __shfl_xor_sync(FULL, k.bad, src_xor);
  o.c = __shfl_xor_sync(FULL, k.c, src_xor);
  o.dropped = __shfl_xor_sync(FULL, k.dropped, src_xor);
  o.p = __shfl_xor_sync(FULL, k.p, src_xor);
  o.sum = __shfl_xor_sync(FULL, k.sum, src_xor);
  o.completed = __shfl_xor_sync(FULL, k.completed, src_xor);
  o.makespan = __shfl_xor_sync(FULL, k.makespan, src_xor);
  o.good = __shfl_xor_sync(FULL, k.good, src_xor);
  o.large = __shfl_xor_sync(FULL, k.large, src_xor);
  return o;
}

__device__ __forceinline__ Key warp_best(Key mine, bool valid, uint32_t obj, unsigned long long slo) {
  if (!valid) mine.c = 0xFFFFFFFFu;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Key other = shfl_key(mine, o);
    const bool ov = other.c != 0xFFFFFFFFu, mv = mine.c != 0xFFFFFFFFu;
    if (ov && (!mv || better(other, mine, obj, slo))) mine = other;
  }
  return mine;
}

__global__ void k3_group_argmin(const uint8_t* __restrict__ blob, const uint8_t* __restrict__ summary,
                                int* __restrict__ best, uint32_t obj, unsigned long long slo) {
  const DParams& P = *reinterpret_cast<const DParams*>(blob);
  const unsigned long long lg = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (lg >= P.n_local_groups) return;
  Key bk{};
  bool have = false;
  for (uint32_t c = lane; c < P.C; c += 32) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(summary + (lg * P.C + c) * SDAS_SUMMARY_BYTES);
    Key k;
    k.bad = s[0] != SDAS_REPLICA_OK;
    k.c = c;
    k.dropped = s[2];
    k.completed = s[3];
    k.makespan = s[4] | ((unsigned long long)s[5] << 32);
    const bool ff = obj == SDAS_MIN_P99_FF, in = obj == SDAS_MIN_P99_E2E_INTERACTIVE;
    const int sw = ff ? 8 : in ? 34 : 6;
    k.sum = s[sw] | ((unsigned long long)s[sw + 1] << 32);
    k.p = obj == SDAS_MIN_P50_E2E ? s[12] : obj == SDAS_MIN_P90_E2E ? s[17] : ff ? s[15] : in ? s[37] : s[13];
    k.good = s[26];
    k.large = s[27];
    if (!have || better(k, bk, obj, slo)) { bk = k; have = true; }
  }
  const Key w = warp_best(bk, have, obj, slo);
  if (lane == 0) best[lg] = (int)w.c;
}

// pooled cell percentile (lower edge of the nearest-rank bin), one warp per cell
__global__ void k4_cell_pct(const uint8_t* __restrict__ blob, const int* __restrict__ cell_hist,
                            uint32_t* __restrict__ cell_p, unsigned long long n_cells, uint32_t obj) {
  const unsigned long long cell = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (cell >= n_cells) return;
  const int* h = cell_hist + cell * (SDAS_NHIST * SDAS_NBINS) +
                 (obj == SDAS_MIN_P99_FF ? SDAS_NBINS : obj == SDAS_MIN_P99_E2E_INTERACTIVE ? 2 * SDAS_NBINS : 0);
  const uint32_t lo_b = lane * 15u, hi_b = min(lo_b + 15u, (uint32_t)SDAS_NBINS);
  unsigned long long part = 0;
  for (uint32_t b = lo_b; b < hi_b; ++b) part += (uint32_t)h[b];
  const unsigned long long n = warp_sum64(part);
  uint32_t p = 0xFFFFFFFFu;
  if (n > 0) {
    const unsigned long long num = obj == SDAS_MIN_P50_E2E ? 50ull : obj == SDAS_MIN_P90_E2E ? 90ull : 99ull;
    const unsigned long long kq = (num * n + 99ull) / 100ull;
    unsigned long long incl = part;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned long long excl = incl - part;
    const int L = __ffs(__ballot_sync(FULL, incl >= kq && excl < kq)) - 1;
    unsigned long long cum = __shfl_sync(FULL, excl, L);
    uint32_t b = (uint32_t)L * 15u;
    for (;; ++b) {
      const unsigned long long cc = (uint32_t)h[b];
      if (cum + cc >= kq) break;
      cum += cc;
    }
    p = bin_lo(b);
  }
  if (lane == 0) cell_p[cell] = p;
}

__global__ void k5_row_argmin(const uint8_t* __restrict__ blob, const long long* __restrict__ cell_cnt,
                              const uint32_t* __restrict__ cell_p, int* __restrict__ best, unsigned long long n_rows,
                              uint32_t obj, unsigned long long slo) {
  const DParams& P = *reinterpret_cast<const DParams*>(blob);
  const unsigned long long row = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  Key bk{};
  bool have = false;
  for (uint32_t c = lane; c < P.C; c += 32) {
    const unsigned long long cell = row * P.C + c;
    const long long* q = cell_cnt + cell * SDAS_NCNT;
    Key k;
    k.bad = q[1] != q[0];
    k.c = c;
    k.dropped = (unsigned long long)q[5];
    k.p = cell_p[cell];
    k.sum = (unsigned long long)(obj == SDAS_MIN_P99_FF ? q[8] : obj == SDAS_MIN_P99_E2E_INTERACTIVE ? q[26] : q[7]);
    k.completed = (unsigned long long)q[6];
    k.makespan = (unsigned long long)q[9];
    k.good = (unsigned long long)q[11];
    k.large = (unsigned long long)q[12];
    if (!have || better(k, bk, obj, slo)) { bk = k; have = true; }
  }
  const Key w = warp_best(bk, have, obj, slo);
  if (lane == 0) best[row] = (int)w.c;
}

// ------------------------------------------------------------------------------ launchers
typedef void (*K1Fn)(const uint8_t*, Work*, uint8_t*, unsigned long long*, uint8_t*, long long*, int*, uint8_t*,
                     unsigned long long*, DParams);

static K1Fn k1_pick(bool trace, uint32_t maxout, bool cls, uint32_t lv, bool spill) {
#ifdef K1_EXP_LEAN_ONLY   // register / SASS experiments only: compile the config-2 instantiation alone
  return k1_simulate<false, 1, false, 2, false>;
#else
  if (!trace && !cls && lv == 2 && maxout == 1)
    return spill ? k1_simulate<false, 1, false, 2, true> : k1_simulate<false, 1, false, 2, false>;
  if (!trace && !cls && lv >= 1) {
    if (maxout > 1) return spill ? k1_simulate<false, 2, false, 1, true> : k1_simulate<false, 2, false, 1, false>;
    return spill ? k1_simulate<false, 1, false, 1, true> : k1_simulate<false, 1, false, 1, false>;
  }
  if (cls) {
    if (maxout > 1) return trace ? k1_simulate<true, 2, true, 0, false> : k1_simulate<false, 2, true, 0, false>;
    return trace ? k1_simulate<true, 1, true, 0, false> : k1_simulate<false, 1, true, 0, false>;
  }
  if (maxout > 1) return trace ? k1_simulate<true, 2, false, 0, false> : k1_simulate<false, 2, false, 0, false>;
  return trace ? k1_simulate<true, 1, false, 0, false> : k1_simulate<false, 1, false, 0, false>;
#endif
}

int launch_simulate(const uint8_t* params_dev, const DParams& hp, const sdas_buffers* bf, uint32_t blocks,
                    uint32_t warps_per_block, uint32_t smem_bytes, void* stream, const uint64_t* log2_table) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const K1Fn fn = k1_pick((hp.flags & SDAS_FLAG_TRACE) != 0, hp.max_out, hp.cls != 0, hp.lean,
                          hp.ring_s != 0xFFFFFFFFu);
  cudaError_t e = cudaMemcpyToSymbolAsync(c_log2, log2_table, sizeof(uint64_t) * 257, 0, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
  if (e != cudaSuccess) return (int)e;
  e = cudaMemsetAsync(bf->work, 0, sizeof(Work), s);
  if (e != cudaSuccess) return (int)e;
  if ((hp.flags & SDAS_FLAG_SERIES) && bf->series && hp.series_stride) {   // windows never reached read 0
    e = cudaMemsetAsync(bf->series, 0, (size_t)hp.series_slots * hp.series_windows * hp.n_inst * 16u, s);
    if (e != cudaSuccess) return (int)e;
  }
  if ((hp.flags & SDAS_FLAG_TRACE) && bf->trace) {
    e = cudaMemsetAsync(bf->trace, 0, 8, s);
    if (e != cudaSuccess) return (int)e;
  }
  if (hp.n_local_replicas == 0) return 0;
  fn<<<blocks, warps_per_block * 32, smem_bytes, s>>>(
      params_dev, reinterpret_cast<Work*>(bf->work), reinterpret_cast<uint8_t*>(bf->summary),
      reinterpret_cast<unsigned long long*>(bf->records), reinterpret_cast<uint8_t*>(bf->series),
      reinterpret_cast<long long*>(bf->cell_cnt), reinterpret_cast<int*>(bf->cell_hist),
      reinterpret_cast<uint8_t*>(bf->trace), reinterpret_cast<unsigned long long*>(bf->cell_series), hp);
  return (int)cudaGetLastError();
}

int launch_group_argmin(const uint8_t* params_dev, const DParams& hp, const sdas_buffers* bf, uint32_t objective,
                        uint64_t slo, void* stream) {
  if (hp.n_local_groups == 0) return 0;
  const uint32_t wpb = 8;
  const unsigned long long blocks = (hp.n_local_groups + wpb - 1) / wpb;
  k3_group_argmin<<<(unsigned)blocks, wpb * 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      params_dev, reinterpret_cast<const uint8_t*>(bf->summary), reinterpret_cast<int*>(bf->best_group), objective,
      slo);
  return (int)cudaGetLastError();
}

int launch_finalize(const uint8_t* params_dev, const DParams& hp, const sdas_buffers* bf, uint32_t objective,
                    uint64_t slo, uint64_t n_cells, uint64_t n_rows, void* stream) {
  (void)hp;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint32_t* cell_p = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(bf->work) + sizeof(Work));
  const uint32_t wpb = 8;
  if (n_cells) {
    k4_cell_pct<<<(unsigned)((n_cells + wpb - 1) / wpb), wpb * 32, 0, s>>>(
        params_dev, reinterpret_cast<const int*>(bf->cell_hist), cell_p, n_cells, objective);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
  }
  if (n_rows) {
    k5_row_argmin<<<(unsigned)((n_rows + wpb - 1) / wpb), wpb * 32, 0, s>>>(
        params_dev, reinterpret_cast<const long long*>(bf->cell_cnt), cell_p, reinterpret_cast<int*>(bf->best_row),
        n_rows, objective, slo);
  }
  return (int)cudaGetLastError();
}

int query_occupancy(uint32_t warps_per_block, uint32_t smem_bytes, uint32_t maxout, uint32_t cls, uint32_t lean,
                    uint32_t spill,
                    int* blocks_per_sm, int* n_sm) {
  {  // a block larger than the instantiation's launch bound cannot launch
    cudaFuncAttributes fa;
    const cudaError_t ea = cudaFuncGetAttributes(&fa, k1_pick(false, maxout, cls != 0, lean, spill != 0));
    if (ea != cudaSuccess) return (int)ea;
    if ((int)(warps_per_block * 32) > fa.maxThreadsPerBlock) {
      *blocks_per_sm = 0;
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(n_sm, cudaDevAttrMultiProcessorCount, dev);
      return 0;
    }
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  e = cudaDeviceGetAttribute(n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return (int)e;
  const K1Fn fn = k1_pick(false, maxout, cls != 0, lean, spill != 0);
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
  if (e != cudaSuccess) return (int)e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, (int)warps_per_block * 32, smem_bytes);
  return (int)e;
}

const char* cuda_error_string(int code) { return cudaGetErrorString((cudaError_t)code); }

}  // namespace sdas
