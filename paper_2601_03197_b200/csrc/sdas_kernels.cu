// sdas_kernels.cu -- sm_100a kernels of the SDAS strategy simulator (product path).
//
// K1 k1_simulate   : persistent, one replica per warp.  Integer-tick discrete-event simulation of
//                    the model of DESIGN.md §"Model" (M0-M20): warp-min next-event selection,
//                    lane-per-instance server state in registers, shared-memory rings (inbox,
//                    in-flight, decode-wait), lane-per-sequence continuous batching with
//                    ballot/popc emission and compaction, in-loop window metrics + controller
//                    (PAPER.md:18, 58-63, 196-220, 231-238, 278-280), and a finalize that builds
//                    log-bin histograms in shared memory, selects exact nearest-rank p50/p99 from
//                    the L2-resident records by radix select, writes the 128-B summary with
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

struct WarpHdr {                        // per-replica scalar state kept in shared memory
  unsigned long long sum_e2e, sum_ff, int_nsys, tokens;
  uint32_t admitted, dropped, arrivals, max_e2e;
  uint32_t n_sat, window_closes, mode_switches, good;
  uint32_t large_items, batch_changes, select_changes, w_n;
  uint32_t w_good, w_half, pad0, pad1;
  uint32_t cur_mode[SDAS_MAX_LINKS + 1];
  int32_t q_last_mode[SDAS_MAX_LINKS + 1];
  uint32_t rr[SDAS_MAX_ROLES];
  uint32_t sel[SDAS_MAX_ROLES];
  int32_t q_last_sel, pad2, pad3, pad4;
};
static_assert(sizeof(WarpHdr) <= 256, "WarpHdr");

// ------------------------------------------------------------------------------ primitives
// Philox4x32-10 (rule M2): ctr = (c0, c1, c2, c3), key = (k0, k1); returns words 0 and 1.
__device__ __forceinline__ uint2 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                        uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return make_uint2(c0, c1);
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

// ------------------------------------------------------------------------------ K1
template <typename T>
__device__ __forceinline__ T* at(uint8_t* base, uint32_t off) {
  return reinterpret_cast<T*>(base + off);
}

__global__ void __launch_bounds__(256, 2) k1_simulate(const uint8_t* __restrict__ blob, Work* __restrict__ work,
                                                   uint8_t* __restrict__ summary,
                                                   unsigned long long* __restrict__ records_out,
                                                   uint8_t* __restrict__ series, long long* __restrict__ cell_cnt,
                                                   int* __restrict__ cell_hist, uint8_t* __restrict__ trace_buf) {
  extern __shared__ __align__(16) uint8_t smem[];
  {
    const uint4* src = reinterpret_cast<const uint4*>(blob);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (uint32_t k = threadIdx.x; k < sizeof(DParams) / 16; k += blockDim.x) dst[k] = src[k];
  }
  __syncthreads();
  const DParams& P = *reinterpret_cast<const DParams*>(smem);
  const int lane = threadIdx.x & 31;
  const uint32_t wib = threadIdx.x >> 5;
  uint8_t* const Wr = smem + P.off_warps + wib * P.smem_per_warp;
  WarpHdr* const H = reinterpret_cast<WarpHdr*>(Wr);
  unsigned long long* const rA = at<unsigned long long>(Wr, P.off_reqA);
  uint32_t* const rFF = at<uint32_t>(Wr, P.off_reqFF);
  uint32_t* const rJ = at<uint32_t>(Wr, P.off_reqJ);
  uint16_t* const rO = at<uint16_t>(Wr, P.off_reqO);
  uint16_t* const rNit = at<uint16_t>(Wr, P.off_reqNit);
  uint16_t* const rOut = at<uint16_t>(Wr, P.off_reqOut);
  uint32_t* const bitmap = at<uint32_t>(Wr, P.off_bitmap);
  uint32_t* const scratch = at<uint32_t>(Wr, P.off_scratch);

  const uint32_t N = P.n_requests, C = P.C, n_inst = P.n_inst;
  const unsigned long long W = P.window;
  const uint32_t key0 = (uint32_t)P.master_seed, key1 = (uint32_t)(P.master_seed >> 32);
  const unsigned long long gwarp = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + wib;
  unsigned long long* const rec_scratch =
      reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(work) + sizeof(Work)) + gwarp * N;
  const DCand* const cands = reinterpret_cast<const DCand*>(blob + P.off_cand);
  const DArr* const arrs = reinterpret_cast<const DArr*>(blob + P.off_arr);

  // lane-resident per-instance constants
  const uint32_t my_role = lane < (int)n_inst ? P.inst[lane].role : 0u;

  for (;;) {
    unsigned long long x = 0;
    if (lane == 0) x = atomicAdd(&work->next_replica, 1ull);
    x = __shfl_sync(FULL, x, 0);
    if (x >= P.n_local_replicas) break;

    // ---------------------------------------------------------------- replica coordinates (M1)
    const uint32_t c = (uint32_t)(x % C);
    const unsigned long long g = P.first_group + (x / C) * P.world;
    const unsigned long long rid = g * C + c;
    const uint32_t s_coord = (uint32_t)(g % P.S) + P.seed_offset;
    const unsigned long long ik = g / P.S;
    const uint32_t kk = (uint32_t)(ik % P.K), ii = (uint32_t)(ik / P.K);
    const DCand& cd = cands[c];
    const DArr& ad = arrs[ii * P.K + kk];
    const bool trace_on = (P.flags & SDAS_FLAG_TRACE) && rid == P.trace_replica;
    unsigned long long* const rec =
        (P.flags & SDAS_FLAG_RECORDS) ? records_out + x * (unsigned long long)N : rec_scratch;
    SeriesRec* ser = nullptr;
    if ((P.flags & SDAS_FLAG_SERIES) && P.series_stride && rid % P.series_stride == 0 &&
        rid / P.series_stride < P.series_slots)
      ser = reinterpret_cast<SeriesRec*>(series) +
            (rid / P.series_stride) * (unsigned long long)P.series_windows * n_inst;

    // ---------------------------------------------------------------- init
    if (lane < 64 / 4) reinterpret_cast<uint4*>(H)[lane] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    for (uint32_t l = lane; l < P.n_links; l += 32) {
      H->cur_mode[l] = cd.mode[l] == 255 ? P.link[l].mode : cd.mode[l];
      H->q_last_mode[l] = -(1 << 30);
    }
    if (lane < (int)P.n_roles) {
      H->rr[lane] = 0;
      H->sel[lane] = P.role[lane].large_inst;
    }
    if (lane == 0) H->q_last_sel = -(1 << 30);
    for (uint32_t w = lane; w < P.bitmap_words; w += 32) {
      const uint32_t rem = P.request_cap - w * 32;
      bitmap[w] = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
    }
    __syncwarp();

    // lane-per-instance server state (rule M7)
    unsigned long long end = 0, cur = 0, acc_qint = 0, acc_lint = 0;
    uint32_t st = IDLE, ih = 0, in = 0, fh = 0, fn = 0, wh = 0, wn = 0, b = 0, fhead = 0;
    uint32_t Bk = lane < (int)n_inst ? P.inst[lane].B_default : 1u;
    int32_t qlB = -(1 << 30);
    uint32_t acc_busy = 0, acc_maxq = 0, cnt_deliv = 0, cnt_recv = 0, cnt_decode = 0;

    // uniform replica state
    unsigned long long t = 0, A_next = 0, nb = W;
    uint32_t jn = 0, P_next = 0, O_next = 0, nsys = 0, completed = 0, wk = 0;
    bool ovf = false;
    uint32_t status = SDAS_REPLICA_OK;
    uint32_t mm_k = 0;
    unsigned long long mm_end = 0;

    auto trace = [&](uint32_t code, uint32_t a, uint32_t bb, uint32_t cc) {
      if (trace_on && lane == 0) {
        const unsigned long long k = atomicAdd(reinterpret_cast<unsigned long long*>(trace_buf), 1ull);
        if (k < P.trace_cap) {
          TraceRec* r = reinterpret_cast<TraceRec*>(trace_buf + 8) + k;
          r->tick = t; r->code = code; r->a = a; r->b = bb; r->c = cc;
        }
      }
    };
    auto trace_lane = [&](uint32_t code, uint32_t a, uint32_t bb, uint32_t cc) {
      if (trace_on) {
        const unsigned long long k = atomicAdd(reinterpret_cast<unsigned long long*>(trace_buf), 1ull);
        if (k < P.trace_cap) {
          TraceRec* r = reinterpret_cast<TraceRec*>(trace_buf + 8) + k;
          r->tick = t; r->code = code; r->a = a; r->b = bb; r->c = cc;
        }
      }
    };

    // ---------------------------------------------------------------- arrivals (M4, M5)
    auto advance_epoch = [&]() {
      ++mm_k;
      const uint2 w = philox(mm_k, s_coord, 4u << 16, 0u, key0, key1);
      const unsigned long long d = exp_sample((mm_k & 1) ? ad.soj1 : ad.soj0, w.x);
      mm_end += d > 0 ? d : 1ull;
    };
    auto gen = [&](uint32_t j, unsigned long long A_prev) {
      if (ad.kind == SDAS_POISSON) {
        const uint2 w = philox(j, s_coord, 1u << 16, 0u, key0, key1);
        A_next = A_prev + exp_sample(ad.gap0, w.x);
      } else if (ad.kind == SDAS_DET) {
        A_next = (unsigned long long)j * ad.gap0;
      } else if (ad.kind == SDAS_LIST) {
        A_next = reinterpret_cast<const unsigned long long*>(blob + ad.list_off)[j];
      } else {  // MMPP2: restart at epoch edges
        unsigned long long tt = A_prev;
        while (mm_end <= tt) advance_epoch();
        for (;;) {
          const uint2 w = philox(j, s_coord, 1u << 16, mm_k, key0, key1);
          const unsigned long long gg = exp_sample((mm_k & 1) ? ad.gap1 : ad.gap0, w.x);
          if (tt + gg < mm_end) { A_next = tt + gg; break; }
          tt = mm_end;
          advance_epoch();
        }
      }
      const uint2 w = philox(j, s_coord, 2u << 16, 0u, key0, key1);
      P_next = uni(ad.p_lo, ad.p_hi, w.x);
      O_next = uni(ad.o_lo, ad.o_hi, w.y);
    };
    if (ad.kind == SDAS_MMPP2) {
      const uint2 w = philox(0u, s_coord, 4u << 16, 0u, key0, key1);
      const unsigned long long d = exp_sample(ad.soj0, w.x);
      mm_end = d > 0 ? d : 1ull;
    }
    if (N > 0) gen(0, 0);

    // ---------------------------------------------------------------- routing (M11)
    auto route = [&](uint32_t role) -> uint32_t {
      const DRole& R = P.role[role];
      if (R.n == 1) return R.first;
      uint32_t pol = R.route;
      if ((pol == SDAS_ROUTE_JSQ || pol == SDAS_ROUTE_RR) && cd.route_override != SDAS_ROUTE_NONE)
        pol = cd.route_override;
      if (pol == SDAS_ROUTE_RR) {
        const uint32_t k = H->rr[role];
        H->rr[role] = k + 1;
        return R.first + k % R.n;
      }
      if (pol == SDAS_ROUTE_FIXED) return R.first + R.route_fixed;
      if (pol == SDAS_ROUTE_SELECT) return H->sel[role];
      uint32_t key = 0xFFFFFFFFu;
      if (lane >= (int)R.first && lane < (int)(R.first + R.n)) {
        const uint32_t load = fn + in + (st == RECV ? 1u : 0u) + wn + b;
        key = (load << 4) | (uint32_t)(lane - R.first);
      }
      key = __reduce_min_sync(FULL, key);
      return R.first + (key & 15u);
    };

    // ---------------------------------------------------------------- emission (M9)
    auto emit = [&](uint32_t l, uint32_t slot, uint32_t tokens, uint32_t opens, uint32_t closes, uint32_t n_in,
                    uint32_t dest) -> uint32_t {
      const DLink& L = P.link[l];
      if (opens) {
        dest = route(L.dst);
        rO[slot] = (uint16_t)(rO[slot] + 1);                 // M13: +1 per opening message
      }
      trace(TR_EMIT, dest, rJ[slot], tokens | (opens << 16) | (closes << 17) | (l << 20));
      const DInst& D = P.inst[dest];
      const uint32_t fn_d = __shfl_sync(FULL, fn, dest);
      if (fn_d >= D.flight_cap) {
        trace(TR_OVERFLOW, 1, dest, 0);
        ovf = true;
        return dest;
      }
      const uint32_t idx = wrap_add(__shfl_sync(FULL, fh, dest), fn_d, D.flight_cap);
      const uint32_t tick = (uint32_t)(t + L.net);
      at<uint32_t>(Wr, D.off_ftick)[idx] = tick;
      at<unsigned long long>(Wr, D.off_fbody)[idx] = make_body(slot, opens | (closes << 1), tokens, n_in);
      if (lane == (int)dest) {
        if (fn == 0) fhead = tick;
        ++fn;
      }
      return dest;
    };

    // ---------------------------------------------------------------- completion (M13, M18)
    auto request_complete = [&](uint32_t slot) {
      --nsys;
      const unsigned long long e2e = t - rA[slot];
      const uint32_t f32 = rFF[slot];
      const uint32_t e32 = sat32(e2e);
      if (e2e >= 0xFFFFFFFFull || f32 == 0xFFFFFFFFu) H->n_sat += 1;
      if (lane == 0) rec[completed] = (unsigned long long)e32 | ((unsigned long long)f32 << 32);
      ++completed;
      H->sum_e2e += e2e;
      H->sum_ff += f32;
      if (e32 > H->max_e2e) H->max_e2e = e32;
      if (e2e <= P.slo) H->good += 1;
      H->w_n += 1;
      if (e2e <= cd.policy_slo) H->w_good += 1;
      if (2ull * e2e <= cd.policy_slo) H->w_half += 1;
      trace(TR_REQ_DONE, rJ[slot], e32, f32);
      bitmap[slot >> 5] |= 1u << (slot & 31);
    };
    auto item_complete = [&](uint32_t i, uint32_t slot) {
      if (P.inst[i].flags & 1u) H->large_items += 1;
      const uint32_t o = rO[slot] - 1u;
      rO[slot] = (uint16_t)o;
      if (o == 0) request_complete(slot);
    };
    auto feedback = [&](uint32_t role, uint32_t slot) {
      if (role == P.feedback_role && rFF[slot] == kUnsetFF) rFF[slot] = sat32(t - rA[slot]);
    };

    // ---------------------------------------------------------------- phase COMPLETE (M7-M10)
    auto complete = [&](uint32_t i) {
      const DInst& I = P.inst[i];
      const uint32_t role = I.role;
      const DRole& R = P.role[role];
      const uint32_t sti = __shfl_sync(FULL, st, i);
      if (sti == RECV) {
        const unsigned long long body = __shfl_sync(FULL, cur, i);
        if (lane == (int)i) { st = IDLE; ++cnt_recv; }
        const uint32_t slot = (uint32_t)(body & 0xFFFFu), flags = (uint32_t)(body >> 16) & 0xFFu;
        const uint32_t n_in = (uint32_t)(body >> 48);
        trace(TR_RECV_DONE, i, rJ[slot], flags);
        if (flags & F_CLOSES) {
          uint32_t out;
          if (role == 0) {
            out = rOut[slot];
          } else {
            const unsigned long long prod = (unsigned long long)n_in * R.out_num;
            const unsigned long long o64 =
                R.out_fixed + (R.out_den == 1 ? prod
                                              : (prod < 0xFFFFFFFFull ? (unsigned long long)((uint32_t)prod / R.out_den)
                                                                      : prod / R.out_den));
            out = o64 > 65535ull ? 65535u : (uint32_t)o64;
          }
          if (out > 0) {
            const uint32_t wn_i = __shfl_sync(FULL, wn, i);
            if (wn_i >= I.wait_cap) {
              trace(TR_OVERFLOW, 2, i, 0);
              ovf = true;
              return;
            }
            const uint32_t idx = wrap_add(__shfl_sync(FULL, wh, i), wn_i, I.wait_cap);
            at<uint32_t>(Wr, I.off_wait)[idx] = slot | (out << 16);
            if (lane == (int)i) ++wn;
            trace(TR_ITEM_WAIT, i, rJ[slot], out);
          } else {  // tool item: forward one 0-token message per out-link and complete now
            for (uint32_t q = 0; q < R.n_out; ++q) {
              emit(q ? R.out_link1 : R.out_link0, slot, 0u, 1u, 1u, 0u, 0u);
              if (ovf) return;
            }
            feedback(role, slot);
            item_complete(i, slot);
          }
        }
        return;
      }
      // DECODE: lane k = batch slot k
      const uint32_t bi = __shfl_sync(FULL, b, i);
      if (lane == (int)i) { st = IDLE; ++cnt_decode; }
      H->tokens += bi;
      trace(TR_DECODE_DONE, i, bi, 0);
      uint32_t* const bat = at<uint32_t>(Wr, I.off_batch);
      const bool act = lane < (int)bi;
      const uint32_t n_out = R.n_out;
      uint32_t w0 = 0, done = 0, a0 = 0, b0 = 0, a1 = 0, b1 = 0;
      if (act) {
        w0 = bat[lane];
        done = bat[32 + lane] + 1u;
        if (n_out > 0) { a0 = bat[64 + lane]; b0 = bat[96 + lane]; }
        if (n_out > 1) { a1 = bat[128 + lane]; b1 = bat[160 + lane]; }
      }
      const uint32_t slot = w0 & 0xFFFFu, out = w0 >> 16;
      uint32_t em = 0, tok0 = 0, fl0 = 0, nin0 = 0, tok1 = 0, fl1 = 0, nin1 = 0;
      auto decide = [&](uint32_t& a, uint32_t& bq, uint32_t link, uint32_t& tok, uint32_t& fl, uint32_t& nin) -> bool {
        const uint32_t prev = a & 0xFFFFu, next = a >> 16, mode = bq >> 24;
        if (done != next) return false;
        tok = next - prev;
        const bool tm = mode == SDAS_TOKEN;
        fl = (tm ? (prev == 0 ? 1u : 0u) : 1u) | ((tm ? (next == out ? 1u : 0u) : 1u) << 1);
        nin = tm ? out : tok;
        uint32_t nx = out;
        if (mode == SDAS_FUNCTION) {
          const uint32_t f = (bq & 0xFFFFu) + 1u;
          bq = (bq & 0xFFFF0000u) | f;
          const uint32_t Fp = min(R.n_functions, out);
          nx = (uint32_t)(((unsigned long long)(f + 1u) * out) / Fp);
        } else if (mode == SDAS_TOKEN) {
          nx = min(next + P.link[link].chunk, out);
        }
        a = next | (min(nx, 0xFFFFu) << 16);
        return true;
      };
      if (act && n_out > 0 && decide(a0, b0, R.out_link0, tok0, fl0, nin0)) em |= 1u;
      if (act && n_out > 1 && decide(a1, b1, R.out_link1, tok1, fl1, nin1)) em |= 2u;
      // messages in (batch order, out-link order), routed sequentially (M11)
      uint32_t emask = __ballot_sync(FULL, em != 0);
      while (emask) {
        const int k = __ffs(emask) - 1;
        emask &= emask - 1;
        const uint32_t emk = __shfl_sync(FULL, em, k);
        const uint32_t sk = __shfl_sync(FULL, slot, k);
        if (emk & 1u) {
          const uint32_t tk = __shfl_sync(FULL, tok0, k), fk = __shfl_sync(FULL, fl0, k),
                         nk = __shfl_sync(FULL, nin0, k), bk = __shfl_sync(FULL, b0, k);
          const uint32_t dest = emit(R.out_link0, sk, tk, fk & 1u, fk >> 1, nk, (bk >> 16) & 0xFFu);
          if (ovf) return;
          if ((fk & 1u) && lane == k) b0 = (b0 & 0xFF00FFFFu) | (dest << 16);
        }
        if (emk & 2u) {
          const uint32_t tk = __shfl_sync(FULL, tok1, k), fk = __shfl_sync(FULL, fl1, k),
                         nk = __shfl_sync(FULL, nin1, k), bk = __shfl_sync(FULL, b1, k);
          const uint32_t dest = emit(R.out_link1, sk, tk, fk & 1u, fk >> 1, nk, (bk >> 16) & 0xFFu);
          if (ovf) return;
          if ((fk & 1u) && lane == k) b1 = (b1 & 0xFF00FFFFu) | (dest << 16);
        }
      }
      if (role == P.feedback_role) {  // first output token at a feedback-role instance (M13)
        if (act && done == 1u && rFF[slot] == kUnsetFF) rFF[slot] = sat32(t - rA[slot]);
        __syncwarp();
      }
      const uint32_t fin = __ballot_sync(FULL, act && done == out);
      uint32_t fm = fin;
      while (fm) {
        const int k = __ffs(fm) - 1;
        fm &= fm - 1;
        item_complete(i, __shfl_sync(FULL, slot, k));
      }
      const uint32_t keep = __ballot_sync(FULL, act && done != out);
      __syncwarp();
      if (act && done != out) {  // stable compaction
        const uint32_t nk = __popc(keep & lanemask_lt());
        bat[nk] = w0;
        bat[32 + nk] = done;
        if (n_out > 0) { bat[64 + nk] = a0; bat[96 + nk] = b0; }
        if (n_out > 1) { bat[128 + nk] = a1; bat[160 + nk] = b1; }
      }
      __syncwarp();
      if (lane == (int)i) b = __popc(keep);
    };

    // ---------------------------------------------------------------- phase START (M7)
    auto start = [&](uint32_t i) {
      const DInst& I = P.inst[i];
      const uint32_t role = I.role;
      const DRole& R = P.role[role];
      const uint32_t in_i = __shfl_sync(FULL, in, i);
      if (in_i > 0) {  // RECV-first
        const uint32_t ih_i = __shfl_sync(FULL, ih, i);
        const unsigned long long body = at<unsigned long long>(Wr, I.off_inbox)[ih_i];
        const uint32_t slot = (uint32_t)(body & 0xFFFFu), flags = (uint32_t)(body >> 16) & 0xFFu;
        const uint32_t tokens = (uint32_t)(body >> 32) & 0xFFFFu;
        unsigned long long cost = (unsigned long long)I.h + (unsigned long long)I.beta * tokens;
        if (flags & F_OPENS) {
          const uint32_t ord = rNit[slot];
          rNit[slot] = (uint16_t)(ord + 1u);
          unsigned long long a = I.alpha;
          if (I.flags & 2u) {
            const uint2 w = philox(rJ[slot], s_coord, (3u << 16) | role, ord, key0, key1);
            a = exp_sample(I.alpha, w.x);
          }
          cost += a;
        }
        if (cost < 1) cost = 1;
        if (lane == (int)i) {
          st = RECV;
          end = t + cost;
          cur = body;
          ih = wrap_add(ih, 1u, I.inbox_cap);
          --in;
        }
        trace(TR_RECV_START, i, rJ[slot], (uint32_t)cost);
        return;
      }
      const uint32_t bi = __shfl_sync(FULL, b, i), Bi = __shfl_sync(FULL, Bk, i);
      const uint32_t wn_i = __shfl_sync(FULL, wn, i), wh_i = __shfl_sync(FULL, wh, i);
      const uint32_t nadm = Bi > bi ? min(Bi - bi, wn_i) : 0u;
      if (nadm) {  // FIFO admission, modes bound per (item, link) here (M9)
        uint32_t* const bat = at<uint32_t>(Wr, I.off_batch);
        if (lane >= (int)bi && lane < (int)(bi + nadm)) {
          const uint32_t e = at<uint32_t>(Wr, I.off_wait)[wrap_add(wh_i, lane - bi, I.wait_cap)];
          const uint32_t out = e >> 16;
          bat[lane] = e;
          bat[32 + lane] = 0;
          for (uint32_t q = 0; q < R.n_out; ++q) {
            const uint32_t l = q ? R.out_link1 : R.out_link0;
            const uint32_t mode = H->cur_mode[l];
            uint32_t next = out;
            if (mode == SDAS_FUNCTION) next = out / min(R.n_functions, out);
            else if (mode == SDAS_TOKEN) next = min(P.link[l].chunk, out);
            bat[64 + 64 * q + lane] = next << 16;
            bat[96 + 64 * q + lane] = (0xFFu << 16) | (mode << 24);
          }
        }
        __syncwarp();
      }
      const uint32_t nbat = bi + nadm;
      if (lane == (int)i) {
        wh = wrap_add(wh, nadm, I.wait_cap);
        wn -= nadm;
        b = nbat;
      }
      if (nbat > 0) {
        unsigned long long cost = (unsigned long long)I.tau0 + (unsigned long long)I.gamma * nbat;
        if (cost < 1) cost = 1;
        if (lane == (int)i) { st = DECODE; end = t + cost; }
        trace(TR_DECODE_START, i, nbat, (uint32_t)cost);
      }
    };

    // ---------------------------------------------------------------- phase ARRIVE (M14)
    auto arrive = [&]() {
      const uint32_t j = jn;
      H->arrivals += 1;
      if (nsys >= P.request_cap) {
        H->dropped += 1;
        trace(TR_ARRIVE, j, 0, 0xFFFFFFFFu);
      } else {
        H->admitted += 1;
        ++nsys;
        // lowest free request slot
        const uint32_t wv = lane < (int)P.bitmap_words ? bitmap[lane] : 0u;
        const uint32_t wm = __ballot_sync(FULL, wv != 0);
        const int wi = __ffs(wm) - 1;
        const uint32_t word = __shfl_sync(FULL, wv, wi);
        const uint32_t bit = __ffs(word) - 1;
        const uint32_t slot = (uint32_t)wi * 32u + bit;
        __syncwarp();
        bitmap[wi] = word & ~(1u << bit);
        rA[slot] = t;
        rFF[slot] = kUnsetFF;
        rJ[slot] = j;
        rO[slot] = 1;                  // M13: +1 on admission
        rNit[slot] = 0;
        rOut[slot] = (uint16_t)O_next;
        const uint32_t dest = route(0);
        trace(TR_ARRIVE, j, 1, dest);
        const DInst& D = P.inst[dest];
        const uint32_t in_d = __shfl_sync(FULL, in, dest);
        if (in_d >= D.inbox_cap) {
          trace(TR_OVERFLOW, 0, dest, 0);
          ovf = true;
        } else {
          const uint32_t idx = wrap_add(__shfl_sync(FULL, ih, dest), in_d, D.inbox_cap);
          at<unsigned long long>(Wr, D.off_inbox)[idx] = make_body(slot, F_OPENS | F_CLOSES, P_next, P_next);
          if (lane == (int)dest) ++in;
        }
      }
      ++jn;
      if (jn < N) gen(jn, t);
    };

    // ---------------------------------------------------------------- window close + control (M15, M16)
    auto control = [&](int32_t q) {
      for (uint32_t l = 0; l < P.n_links; ++l) {  // (i) three-band mode policy
        if (!((cd.ctl_links >> l) & 1u)) continue;
        const DRole& Rd = P.role[P.link[l].dst];
        const bool mine = lane >= (int)Rd.first && lane < (int)(Rd.first + Rd.n);
        const unsigned long long u =
            warp_sum64(mine ? (cd.metric_load ? acc_lint : (unsigned long long)acc_busy) : 0ull);
        const unsigned long long lhs = u * 1000ull;
        uint32_t band = 1;
        if (lhs >= (unsigned long long)cd.hi * W * Rd.n) band = 2;
        else if (lhs <= (unsigned long long)cd.lo * W * Rd.n) band = 0;
        const uint32_t want = cd.band[band], curm = H->cur_mode[l];
        if (want != curm && q - H->q_last_mode[l] >= (int32_t)cd.dwell) {
          H->cur_mode[l] = want;
          H->q_last_mode[l] = q;
          H->mode_switches += 1;
          trace(TR_CONTROL, 0, l, want);
        }
      }
      bool viol = false, calm = false;
      const uint32_t wnn = H->w_n;
      if (wnn >= 1) {
        const uint32_t k99 = (uint32_t)((99ull * wnn + 99ull) / 100ull);
        viol = H->w_good < k99;
        calm = H->w_half >= k99;
      }
      if (cd.batch_roles && wnn >= 1) {  // (ii) SLO-aware max_num_seqs, lane = instance
        bool changed = false;
        if (lane < (int)n_inst && ((cd.batch_roles >> my_role) & 1u)) {
          uint32_t nbB = Bk;
          if (viol) nbB = acc_qint > (unsigned long long)cd.q_hi * W ? min(32u, 2u * Bk) : max(1u, Bk / 2u);
          else if (calm) nbB = P.inst[lane].B_default;
          if (nbB != Bk && q - qlB >= (int32_t)cd.dwell) {
            Bk = nbB;
            qlB = q;
            changed = true;
          }
        }
        uint32_t chm = __ballot_sync(FULL, changed);
        H->batch_changes += __popc(chm);
        while (chm) {
          const int k = __ffs(chm) - 1;
          chm &= chm - 1;
          trace(TR_CONTROL, 1, k, __shfl_sync(FULL, Bk, k));
        }
      }
      if (cd.select_role >= 0) {  // (iii) model selection
        const DRole& Rs = P.role[cd.select_role];
        const uint32_t cs = H->sel[cd.select_role];
        const unsigned long long b1000 = (unsigned long long)__shfl_sync(FULL, acc_busy, cs) * 1000ull;
        uint32_t ns = cs;
        if (b1000 >= (unsigned long long)cd.hi * W || viol) ns = Rs.small_inst;
        else if (b1000 <= (unsigned long long)cd.lo * W && !viol) ns = Rs.large_inst;
        if (ns != cs && q - H->q_last_sel >= (int32_t)cd.dwell) {
          H->sel[cd.select_role] = ns;
          H->q_last_sel = q;
          H->select_changes += 1;
          trace(TR_CONTROL, 2, cd.select_role, ns);
        }
      }
    };
    auto close_window = [&](bool final_partial) {
      if (ser && wk < P.series_windows && lane < (int)n_inst) {
        const int32_t il = P.role[my_role].in_link;
        SeriesRec r;
        r.qint = acc_qint;
        r.busy = acc_busy;
        r.maxq = (uint16_t)min(acc_maxq, 65535u);
        r.mode = il < 0 ? 255 : (uint8_t)H->cur_mode[il];
        r.B = (uint8_t)Bk;
        ser[(unsigned long long)wk * n_inst + lane] = r;
      }
      if (!final_partial) {
        H->window_closes += 1;
        trace(TR_WINDOW, wk, 0, 0);
        if (cd.adaptive) control((int32_t)wk + 1);
      }
      acc_busy = 0; acc_qint = 0; acc_lint = 0; acc_maxq = 0;
      H->w_n = 0; H->w_good = 0; H->w_half = 0;
    };

    // ---------------------------------------------------------------- event loop (M12)
    unsigned long long int_nsys = 0;
    for (;;) {
      if (jn >= N && nsys == 0) break;
      uint32_t d = 0xFFFFFFFFu;
      if (lane < (int)n_inst) {
        if (st != IDLE) d = sat32(end - t);
        if (fn) d = min(d, fhead - (uint32_t)t);
      }
      if (lane == 0) {
        d = min(d, (uint32_t)(nb - t));
        if (jn < N) d = min(d, sat32(A_next - t));
      }
      d = __reduce_min_sync(FULL, d);
      const unsigned long long tn = t + d;
      if (P.max_ticks && tn > P.max_ticks) { status = SDAS_REPLICA_TRUNCATED; break; }
      if (d) {  // integrate the piecewise-constant state over [t, tn) (M15)
        if (lane < (int)n_inst) {
          const uint32_t Q = in + wn;
          if (st != IDLE) acc_busy += d;
          acc_qint += (unsigned long long)Q * d;
          acc_maxq = max(acc_maxq, Q);
          acc_lint += (unsigned long long)(fn + in + (st == RECV ? 1u : 0u) + wn + b) * d;
        }
        int_nsys += (unsigned long long)nsys * d;
      }
      t = tn;
      if (t == nb) {  // phase 0 WINDOW
        close_window(false);
        nb += W;
        ++wk;
      }
      // phase 1 COMPLETE (instance order)
      uint32_t cm = __ballot_sync(FULL, lane < (int)n_inst && st != IDLE && end == t);
      while (cm && !ovf) {
        const int i = __ffs(cm) - 1;
        cm &= cm - 1;
        complete((uint32_t)i);
      }
      if (ovf) break;
      // phase 2 DELIVER (per destination instance, FIFO; lane = instance)
      {
        bool lovf = false;
        if (lane < (int)n_inst && fn > 0 && fhead == (uint32_t)t) {
          const DInst& I = P.inst[lane];
          const uint32_t* ft = at<uint32_t>(Wr, I.off_ftick);
          const unsigned long long* fb = at<unsigned long long>(Wr, I.off_fbody);
          unsigned long long* ib = at<unsigned long long>(Wr, I.off_inbox);
          for (;;) {
            if (in >= I.inbox_cap) { lovf = true; break; }
            const unsigned long long body = fb[fh];
            ib[wrap_add(ih, in, I.inbox_cap)] = body;
            ++in;
            fh = wrap_add(fh, 1u, I.flight_cap);
            --fn;
            ++cnt_deliv;
            trace_lane(TR_DELIVER, lane, rJ[body & 0xFFFFu], (uint32_t)(body >> 32) & 0xFFFFu);
            if (fn == 0) break;
            fhead = ft[fh];
            if (fhead != (uint32_t)t) break;
          }
        }
        if (__ballot_sync(FULL, lovf)) {
          trace(TR_OVERFLOW, 0, 0, 0);
          ovf = true;
          break;
        }
        __syncwarp();
      }
      // phase 3 ARRIVE (increasing j)
      while (jn < N && A_next == t && !ovf) arrive();
      if (ovf) break;
      // phase 4 START (idle instances with work, increasing index)
      uint32_t sm = __ballot_sync(FULL, lane < (int)n_inst && st == IDLE && (in | wn | b) != 0u);
      while (sm) {
        const int i = __ffs(sm) - 1;
        sm &= sm - 1;
        start((uint32_t)i);
      }
    }

    // ---------------------------------------------------------------- finalize (M18, M19)
    uint8_t* const sum_out = summary + x * SDAS_SUMMARY_BYTES;
    const unsigned long long cell = ((unsigned long long)ii * P.K + kk) * C + c;
    uint32_t* const stg = scratch + 2 * SDAS_NBINS + 256;
    unsigned long long* const cst = reinterpret_cast<unsigned long long*>(stg + 32);
    __syncwarp();
    if (ovf) {
      if (lane < 32) stg[lane] = 0;
      __syncwarp();
      if (lane == 0) {
        stg[0] = SDAS_REPLICA_OVERFLOW;
        stg[4] = (uint32_t)t;
        stg[5] = (uint32_t)(t >> 32);
        stg[12] = stg[13] = stg[14] = stg[15] = 0xFFFFFFFFu;
        stg[16] = stg[17] = 0xFFFFFFFFu;
        stg[31] = (uint32_t)rid;
      }
      __syncwarp();
      if (lane < 8) reinterpret_cast<uint4*>(sum_out)[lane] = reinterpret_cast<const uint4*>(stg)[lane];
      if (lane == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(cell_cnt + cell * SDAS_NCNT + 0), 1ull);
        atomicAdd(reinterpret_cast<unsigned long long*>(cell_cnt + cell * SDAS_NCNT + 2), 1ull);
      }
      __syncwarp();
      continue;
    }
    close_window(true);  // final partial window: series only
    uint32_t* const he = scratch;
    uint32_t* const hf = scratch + SDAS_NBINS;
    uint32_t* const cnt = scratch + 2 * SDAS_NBINS;
    for (uint32_t k = lane; k < 2 * SDAS_NBINS; k += 32) he[k] = 0;
    __syncwarp();
    for (uint32_t k = lane; k < completed; k += 32) {  // log-bin histograms in shared memory (M17)
      const unsigned long long v = rec[k];
      atomicAdd(&he[bin_of((uint32_t)v)], 1u);
      atomicAdd(&hf[bin_of((uint32_t)(v >> 32))], 1u);
    }
    __syncwarp();
    // exact nearest-rank percentiles: histogram locates the bin, radix select inside it (M18)
    auto select = [&](const uint32_t* h, int field, uint32_t kq, uint32_t& val, uint32_t& binq) {
      const uint32_t lo_b = lane * 15u, hi_b = min(lo_b + 15u, (uint32_t)SDAS_NBINS);
      uint32_t part = 0;
      for (uint32_t bb = lo_b; bb < hi_b; ++bb) part += h[bb];
      uint32_t incl = warp_incl_scan(part, lane), excl = incl - part;
      int L = __ffs(__ballot_sync(FULL, incl >= kq && excl < kq)) - 1;
      uint32_t cum = __shfl_sync(FULL, excl, L);
      uint32_t bb = (uint32_t)L * 15u;
      for (;; ++bb) {
        const uint32_t cc = h[bb];
        if (cum + cc >= kq) break;
        cum += cc;
      }
      binq = bb;
      uint32_t r = kq - cum;
      if (bb < 16u) { val = bb; return; }
      const uint32_t lo = bin_lo(bb), nbits = (bb - 16u) >> 4;
      uint32_t prefix = 0;
      int left = (int)nbits;
      while (left > 0) {
        const int db = min(8, left), shift = left - db;
        for (uint32_t z = lane; z < 256u; z += 32) cnt[z] = 0;
        __syncwarp();
        for (uint32_t z = lane; z < completed; z += 32) {
          const unsigned long long v64 = rec[z];
          const uint32_t v = field ? (uint32_t)(v64 >> 32) : (uint32_t)v64;
          const uint32_t off = v - lo;
          if (v >= lo && (off >> nbits) == 0u && (off >> (shift + db)) == prefix)
            atomicAdd(&cnt[(off >> shift) & ((1u << db) - 1u)], 1u);
        }
        __syncwarp();
        uint32_t p2 = 0;
        for (uint32_t z = 8u * lane; z < 8u * lane + 8u; ++z) p2 += cnt[z];
        incl = warp_incl_scan(p2, lane);
        excl = incl - p2;
        L = __ffs(__ballot_sync(FULL, incl >= r && excl < r)) - 1;
        uint32_t cum2 = __shfl_sync(FULL, excl, L);
        uint32_t dd = 8u * (uint32_t)L;
        for (;; ++dd) {
          const uint32_t cc = cnt[dd];
          if (cum2 + cc >= r) break;
          cum2 += cc;
        }
        __syncwarp();
        r -= cum2;
        prefix = (prefix << db) | dd;
        left = shift;
      }
      val = lo + prefix;
    };
    uint32_t v50e = 0xFFFFFFFFu, v99e = 0xFFFFFFFFu, v50f = 0xFFFFFFFFu, v99f = 0xFFFFFFFFu;
    uint32_t b50e = 0xFFFFu, b99e = 0xFFFFu, b50f = 0xFFFFu, b99f = 0xFFFFu;
    if (completed > 0) {
      const uint32_t k50 = (uint32_t)((50ull * completed + 99ull) / 100ull);
      const uint32_t k99 = (uint32_t)((99ull * completed + 99ull) / 100ull);
      select(he, 0, k50, v50e, b50e);
      select(he, 0, k99, v99e, b99e);
      select(hf, 1, k50, v50f, b50f);
      select(hf, 1, k99, v99f, b99f);
    }
    const uint32_t deliv = __reduce_add_sync(FULL, lane < (int)n_inst ? cnt_deliv : 0u);
    const uint32_t recvs = __reduce_add_sync(FULL, lane < (int)n_inst ? cnt_recv : 0u);
    const uint32_t decs = __reduce_add_sync(FULL, lane < (int)n_inst ? cnt_decode : 0u);
    __syncwarp();
    if (lane == 0) {
      stg[0] = status; stg[1] = H->admitted; stg[2] = H->dropped; stg[3] = completed;
      stg[4] = (uint32_t)t; stg[5] = (uint32_t)(t >> 32);
      stg[6] = (uint32_t)H->sum_e2e; stg[7] = (uint32_t)(H->sum_e2e >> 32);
      stg[8] = (uint32_t)H->sum_ff; stg[9] = (uint32_t)(H->sum_ff >> 32);
      stg[10] = (uint32_t)int_nsys; stg[11] = (uint32_t)(int_nsys >> 32);
      stg[12] = v50e; stg[13] = v99e; stg[14] = v50f; stg[15] = v99f;
      stg[16] = b50e | (b99e << 16); stg[17] = b50f | (b99f << 16);
      stg[18] = H->max_e2e; stg[19] = H->n_sat;
      stg[20] = H->arrivals; stg[21] = deliv; stg[22] = recvs; stg[23] = decs;
      stg[24] = H->window_closes; stg[25] = H->mode_switches; stg[26] = H->good; stg[27] = H->large_items;
      stg[28] = (uint32_t)H->tokens; stg[29] = (uint32_t)(H->tokens >> 32);
      stg[30] = (H->batch_changes & 0xFFFFu) | (H->select_changes << 16);
      stg[31] = (uint32_t)rid;
      cst[0] = 1; cst[1] = status == SDAS_REPLICA_OK; cst[2] = 0; cst[3] = status == SDAS_REPLICA_TRUNCATED;
      cst[4] = H->admitted; cst[5] = H->dropped; cst[6] = completed; cst[7] = H->sum_e2e; cst[8] = H->sum_ff;
      cst[9] = t; cst[10] = int_nsys; cst[11] = H->good; cst[12] = H->large_items; cst[13] = H->arrivals;
      cst[14] = deliv; cst[15] = recvs; cst[16] = decs; cst[17] = H->window_closes; cst[18] = H->mode_switches;
      cst[19] = H->tokens; cst[20] = H->batch_changes; cst[21] = H->select_changes; cst[22] = H->n_sat;
      cst[23] = 0;
    }
    __syncwarp();
    if (lane < 8) reinterpret_cast<uint4*>(sum_out)[lane] = reinterpret_cast<const uint4*>(stg)[lane];
    int* const ch = cell_hist + cell * (2 * SDAS_NBINS);
    for (uint32_t k = lane; k < 2 * SDAS_NBINS; k += 32) {
      const uint32_t v = he[k];
      if (v) atomicAdd(ch + k, (int)v);
    }
    if (lane < SDAS_NCNT) {
      const unsigned long long v = cst[lane];
      if (v) atomicAdd(reinterpret_cast<unsigned long long*>(cell_cnt + cell * SDAS_NCNT + lane), v);
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------ argmin (M20)
struct Key {
  uint32_t bad, c;
  unsigned long long dropped, p, sum, completed, makespan, good, large;
};

__device__ __forceinline__ bool rate_gt(unsigned long long na, unsigned long long ma, unsigned long long nb,
                                        unsigned long long mb) {
  // na/ma > nb/mb  <=>  na*mb > nb*ma, compared as 128-bit products
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
    const bool ff = obj == SDAS_MIN_P99_FF;
    k.sum = ff ? (s[8] | ((unsigned long long)s[9] << 32)) : (s[6] | ((unsigned long long)s[7] << 32));
    k.p = obj == SDAS_MIN_P50_E2E ? s[12] : (ff ? s[15] : s[13]);
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
  const int* h = cell_hist + cell * (2 * SDAS_NBINS) + (obj == SDAS_MIN_P99_FF ? SDAS_NBINS : 0);
  const uint32_t lo_b = lane * 15u, hi_b = min(lo_b + 15u, (uint32_t)SDAS_NBINS);
  unsigned long long part = 0;
  for (uint32_t b = lo_b; b < hi_b; ++b) part += (uint32_t)h[b];
  const unsigned long long n = warp_sum64(part);
  uint32_t p = 0xFFFFFFFFu;
  if (n > 0) {
    const unsigned long long num = obj == SDAS_MIN_P50_E2E ? 50ull : 99ull;
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
    k.sum = (unsigned long long)(obj == SDAS_MIN_P99_FF ? q[8] : q[7]);
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
int launch_simulate(const uint8_t* params_dev, const DParams& hp, const sdas_buffers* bf, uint32_t blocks,
                    uint32_t warps_per_block, uint32_t smem_bytes, void* stream, const uint64_t* log2_table) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyToSymbolAsync(c_log2, log2_table, sizeof(uint64_t) * 257, 0, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k1_simulate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
  if (e != cudaSuccess) return (int)e;
  e = cudaMemsetAsync(bf->work, 0, sizeof(Work), s);
  if (e != cudaSuccess) return (int)e;
  if ((hp.flags & SDAS_FLAG_TRACE) && bf->trace) {
    e = cudaMemsetAsync(bf->trace, 0, 8, s);
    if (e != cudaSuccess) return (int)e;
  }
  if (hp.n_local_replicas == 0) return 0;
  k1_simulate<<<blocks, warps_per_block * 32, smem_bytes, s>>>(
      params_dev, reinterpret_cast<Work*>(bf->work), reinterpret_cast<uint8_t*>(bf->summary),
      reinterpret_cast<unsigned long long*>(bf->records), reinterpret_cast<uint8_t*>(bf->series),
      reinterpret_cast<long long*>(bf->cell_cnt), reinterpret_cast<int*>(bf->cell_hist),
      reinterpret_cast<uint8_t*>(bf->trace));
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

int query_occupancy(uint32_t warps_per_block, uint32_t smem_bytes, int* blocks_per_sm, int* n_sm) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  e = cudaDeviceGetAttribute(n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k1_simulate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
  if (e != cudaSuccess) return (int)e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k1_simulate, (int)warps_per_block * 32,
                                                    smem_bytes);
  return (int)e;
}

const char* cuda_error_string(int code) { return cudaGetErrorString((cudaError_t)code); }

}  // namespace sdas
