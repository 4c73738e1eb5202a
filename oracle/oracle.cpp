// oracle/oracle.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// A plain, slow, obviously-correct event-heap discrete-event simulation of the
// strategy-evaluation model of "Software-Defined Agentic Serving"
// (arXiv 2601.03197).  Every function cites the rule it follows; the rules are
// stated in DESIGN.md §"Model" (SURVEY.md §8(c) readings, PAPER.md passages):
//   M2 Philox keying, M3 integer samplers, M4/M5 arrivals and sizes,
//   M7 server (RECV-first, continuous batching), M8-M10 emission / receiver
//   items (PAPER.md:17 the three strategies), M11 routing,
//   M12 canonical tick order, M13 completion, M14 capacity, M15 windows
//   (PAPER.md:231-238 metrics plane), M16 control (PAPER.md:18, 196-220,
//   279-280), M17/M18 bins and nearest-rank percentiles, M19 summary, M20 argmin;
//   f1 M21-M24 KV home / routing / transfer penalty, f3 M25
//   constraint guard, f2 M26-M29 request classes, priority service,
//   admission gate, per-class metrics, f4 M30 pacing and M31
//   snapshot JSQ.
//
// Parity unpinned: the full model at scale (batching + RECV-first + modes +
// control) has no closed form; it is pinned compositionally by the hand traces, queueing
// closed forms, conservation laws and brute-force checks under tests/test_oracle_*.py.  Every
// decision rule configs 3-5 rank by (M16(ii)/(iii), M11 RR, LOAD metric, truncation, R-OVF,
// R-SAT, M20 argmins, M15 cell series) has its own hand-derived or brute-force pin
// (tests/test_oracle_control.py, test_oracle_argmin.py, test_oracle_cellseries.py).
//
// Deliberately naive: std::priority_queue of events, std::deque queues,
// std::vector<Item> batches, std::sort for percentiles.  No code is shared with
// the CUDA path.

#include "oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <deque>
#include <mutex>
#include <queue>
#include <thread>
#include <vector>

namespace {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------------------
// M2: Philox4x32-10 (Salmon et al., Random123), written from its definition.
// ---------------------------------------------------------------------------
void philox(const uint32_t in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c[4] = {in[0], in[1], in[2], in[3]};
  uint32_t k[2] = {key_in[0], key_in[1]};
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {  // key schedule: Weyl increments between rounds
      k[0] += 0x9E3779B9u;
      k[1] += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
  }
  out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

// Draw word `w` of Philox(ctr = (c0, s, kind<<16 | role, sub), key = master_seed)   (M2)
void draw(uint64_t master_seed, uint32_t c0, uint32_t s, uint32_t kind, uint32_t role, uint32_t sub,
          uint32_t out[4]) {
  uint32_t ctr[4] = {c0, s, (kind << 16) | role, sub};
  uint32_t key[2] = {(uint32_t)master_seed, (uint32_t)(master_seed >> 32)};
  philox(ctr, key, out);
}
enum { K_ARR = 1, K_ATTR = 2, K_SVC = 3, K_MMPP = 4 };

// ---------------------------------------------------------------------------
// M3: T[i] = round(2^32 * log2(1 + i/256)), computed here in long double.
// ---------------------------------------------------------------------------
struct Log2Table {
  uint64_t t[257];
  Log2Table() {
    for (int i = 0; i <= 256; ++i) {
      long double v = log2l(1.0L + (long double)i / 256.0L) * 4294967296.0L;
      t[i] = (uint64_t)llroundl(v);
    }
  }
};
const Log2Table& table() {
  static Log2Table T;
  return T;
}

// M3 EXP(M; x): floor(-M ln U), U = (x+1)/2^32, via a Q32 log2 with linear interpolation.
uint64_t exp_sample(uint64_t M, uint32_t x) {
  const uint64_t* T = table().t;
  uint64_t y = (uint64_t)x + 1;                       // 1 .. 2^32
  int e = 0;
  while ((y >> (e + 1)) != 0) ++e;                    // e = floor(log2 y)
  uint64_t f = (y << (32 - e)) - (1ull << 32);        // mantissa, Q32, in [0, 2^32)
  uint64_t i = f >> 24;
  uint64_t rho = f & 0xFFFFFFull;
  uint64_t lg = T[i] + (((T[i + 1] - T[i]) * rho) >> 24);  // ~ 2^32 log2(1 + f/2^32)
  uint64_t n = ((uint64_t)(32 - e) << 32) - lg;            // ~ 2^32 * (-log2 U)
  uint64_t a = M * 2977044472ull;                           // M * round(2^32 ln 2)
  return (uint64_t)(((u128)a * (u128)n) >> 64);
}

// M3 UNI(lo, hi; x) = lo + floor(x * (hi - lo + 1) / 2^32)
uint32_t uni(uint32_t lo, uint32_t hi, uint32_t x) {
  return lo + (uint32_t)(((uint64_t)x * ((uint64_t)hi - lo + 1)) >> 32);
}

// ---------------------------------------------------------------------------
// M17: log-linear bins, 16 sub-bins per octave above 16; 464 bins cover u32.
// ---------------------------------------------------------------------------
uint32_t bin_of(uint32_t v) {
  if (v < 16) return v;
  int e = 0;
  while (((uint64_t)v >> (e + 1)) != 0) ++e;  // floor(log2 v) >= 4 (64-bit: no shift by 32)
  return 16 + 16 * (uint32_t)(e - 4) + ((v >> (e - 4)) & 15u);
}
uint64_t bin_lo(uint32_t b) {
  if (b < 16) return b;
  return (uint64_t)(16 + (b - 16) % 16) << ((b - 16) / 16);
}

// M4/M5 arrivals and attributes for one seed coordinate.
int gen_arrivals(const orc_arrival& a, uint64_t ms, uint32_t s, uint32_t n, std::vector<uint64_t>& A,
                 std::vector<uint32_t>& P, std::vector<uint32_t>& O) {
  A.assign(n, 0); P.assign(n, 0); O.assign(n, 0);
  uint32_t w[4];
  if (a.kind == ORC_POISSON) {
    uint64_t t = 0;                                     // A_{-1} = 0
    for (uint32_t j = 0; j < n; ++j) {
      draw(ms, j, s, K_ARR, 0, 0, w);
      t += exp_sample(a.gap[0], w[0]);
      A[j] = t;
    }
  } else if (a.kind == ORC_DET) {
    for (uint32_t j = 0; j < n; ++j) A[j] = (uint64_t)j * a.gap[0];
  } else if (a.kind == ORC_LIST) {
    if (a.list_len < n || a.list == nullptr) return -1;
    for (uint32_t j = 0; j < n; ++j) {
      A[j] = a.list[j];
      if (j > 0 && A[j] < A[j - 1]) return -1;
    }
  } else if (a.kind == ORC_MMPP2) {
    // Epoch k: state k mod 2 (0 = low rate first), duration d_k = max(1, EXP(D_state; MMPP(k).w0)).
    std::vector<uint64_t> E(1, 0);                      // E_0 = 0
    auto epoch_end = [&](uint32_t k) -> uint64_t {      // E_{k+1}
      while (E.size() < (size_t)k + 2) {
        uint32_t kk = (uint32_t)E.size() - 1;
        uint32_t ww[4];
        draw(ms, kk, s, K_MMPP, 0, 0, ww);
        uint64_t d = std::max<uint64_t>(1, exp_sample(a.sojourn[kk % 2], ww[0]));
        E.push_back(E.back() + d);
      }
      return E[k + 1];
    };
    uint64_t t = 0;
    uint32_t k = 0;
    for (uint32_t j = 0; j < n; ++j) {
      while (epoch_end(k) <= t) ++k;                   // the epoch containing t
      for (;;) {
        draw(ms, j, s, K_ARR, 0, k, w);
        uint64_t g = exp_sample(a.gap[k % 2], w[0]);
        if (t + g < epoch_end(k)) { t = t + g; break; }
        t = epoch_end(k);                               // restart at the epoch edge
        ++k;
      }
      A[j] = t;
    }
  } else {
    return -1;
  }
  for (uint32_t j = 0; j < n; ++j) {
    draw(ms, j, s, K_ATTR, 0, 0, w);
    P[j] = uni(a.p_lo, a.p_hi, w[0]);
    O[j] = uni(a.o_lo, a.o_hi, w[1]);
  }
  return 0;
}

uint32_t band_of(uint64_t u, uint32_t lo, uint32_t hi, uint64_t W, uint32_t n) {
  u128 lhs = (u128)u * 1000u;
  if (lhs >= (u128)hi * W * n) return 2;
  if (lhs <= (u128)lo * W * n) return 0;
  return 1;
}

// M16(i): one window close of the three-band policy with dwell D and no-op suppression.
// Returns the mode in force from boundary q on; updates *q_last only when the mode changes.
uint32_t mode_step(uint64_t u, uint32_t lo, uint32_t hi, uint64_t W, uint32_t n, const uint32_t band[3],
                   uint32_t dwell, int64_t q, uint32_t cur, int64_t* q_last) {
  uint32_t want = band[band_of(u, lo, hi, W, n)];
  if (want == cur) return cur;                       // no-op: neither fires nor resets the timer
  if (q - *q_last < (int64_t)dwell) return cur;      // dwell suppression
  *q_last = q;
  return want;
}

uint32_t jsq(const uint32_t* loads, uint32_t n) {
  uint32_t best = 0;
  for (uint32_t i = 1; i < n; ++i)
    if (loads[i] < loads[best]) best = i;
  return best;
}

// ---------------------------------------------------------------------------
// One replica.
// ---------------------------------------------------------------------------
enum { IDLE = 0, RECV = 1, DECODE = 2 };
enum { PH_COMPLETE = 1, PH_DELIVER = 2 };
enum { TR_ARRIVE = 1, TR_RECV_START, TR_DECODE_START, TR_RECV_DONE, TR_DECODE_DONE, TR_EMIT,
       TR_DELIVER, TR_REQ_DONE, TR_WINDOW, TR_CONTROL, TR_ITEM_WAIT, TR_OVERFLOW };

struct Msg {
  uint32_t j, dest, link, opens, closes, tokens, n_in;
  uint32_t kv_kind;   // M23: 0 none, else the KV policy that charges this opening message
  uint64_t ready;     // M23 HINT: tick at which the hinted transfer completes
};

struct Event {
  uint64_t tick;
  uint32_t phase;
  uint64_t entity;  // instance index (COMPLETE) or emission seq (DELIVER)
  Msg msg;
  bool operator>(const Event& o) const {
    if (tick != o.tick) return tick > o.tick;
    if (phase != o.phase) return phase > o.phase;
    return entity > o.entity;
  }
};

struct Item {
  uint32_t j, out, done;
  uint32_t mode[ORC_MAX_LINKS], opened[ORC_MAX_LINKS], last[ORC_MAX_LINKS], fidx[ORC_MAX_LINKS],
      sticky[ORC_MAX_LINKS];
};

struct Inst {
  uint32_t role;
  orc_cost c;
  std::deque<Msg> inbox;
  uint32_t inflight = 0;
  std::deque<std::pair<uint32_t, uint32_t>> wait;  // (j, out)
  std::vector<Item> batch;
  uint32_t state = IDLE;
  uint64_t end = 0;
  Msg cur{};
  uint32_t B = 1, B_default = 1;
  int64_t q_last_B = INT64_MIN / 2;
  // window accumulators (M15)
  uint64_t w_busy = 0, w_qint = 0, w_lint = 0;
  uint32_t w_maxq = 0;
  uint32_t snap = 0;                 // M31: load polled at the last window close (state-store view)
  uint32_t Q() const { return (uint32_t)(inbox.size() + wait.size()); }
  uint32_t load() const {
    return inflight + (uint32_t)inbox.size() + (state == RECV ? 1u : 0u) + (uint32_t)wait.size() +
           (uint32_t)batch.size();
  }
};

struct Replica {
  const orc_pipeline& P;
  const orc_grid& G;
  const orc_candidate& cand;
  uint64_t rid;
  uint32_t s_coord;
  orc_summary& S;
  uint32_t* rec;        // [N][2] or null
  uint32_t* hist;       // [3][NBINS]: e2e, ff, interactive e2e (always provided internally)
  orc_series* series;   // this replica's [windows][n_inst] or null
  std::vector<uint64_t> cser;   // M15 cell-summed series: this replica's contribution [windows][n_inst][8]
  orc_trace* trace; uint64_t trace_cap; uint64_t* trace_n;

  std::vector<Inst> inst;
  std::vector<uint32_t> role_first, role_n;        // instances of each role
  std::vector<std::vector<uint32_t>> out_links;    // per role, links in index order
  std::vector<int32_t> in_link;                    // per role
  std::vector<uint32_t> cur_mode;                  // per link (controller state)
  std::vector<uint32_t> base_mode;                 // per link: the candidate's initial mode (M25 reset)
  std::vector<int64_t> q_last_mode;
  std::vector<uint32_t> rr;                        // per role
  std::vector<uint32_t> sel;                       // per role
  std::vector<uint64_t> pace_free;                 // M30: per link, earliest tick of the next dispatch
  int64_t q_last_sel = INT64_MIN / 2;

  std::vector<uint64_t> A;
  std::vector<uint32_t> Pj, Oj;
  std::vector<uint32_t> o, nitems;
  std::vector<uint64_t> ff;
  std::vector<uint32_t> home;      // M21: KV home instance (index within the KV role) of request j
  std::vector<uint8_t> cls;        // M26: 1 = interactive, 0 = background
  std::vector<uint32_t> ve_int;    // M29: interactive e2e values (saturated u32)
  bool gate_closed = false;        // M28: admission is interactive-only
  int64_t q_last_gate = INT64_MIN / 2;

  std::priority_queue<Event, std::vector<Event>, std::greater<Event>> heap;
  uint64_t seq = 0, t = 0;
  uint32_t nsys = 0, jn = 0;
  bool overflow = false;
  // per-window point counters
  uint32_t w_n = 0, w_good = 0, w_half = 0;

  Replica(const orc_pipeline& p, const orc_grid& g, const orc_candidate& c, uint64_t r, uint32_t s,
          orc_summary& out)
      : P(p), G(g), cand(c), rid(r), s_coord(s), S(out) {}

  void tr(uint32_t code, uint32_t a, uint32_t b, uint32_t c) {
    if (!trace) return;
    if (*trace_n < trace_cap) trace[*trace_n] = orc_trace{t, code, a, b, c};
    ++*trace_n;
  }

  uint32_t route(uint32_t role, uint32_t j) {  // M11 (+ M22 affinity)
    uint32_t n = role_n[role], f = role_first[role];
    if (n == 1) return f;
    if (P.kv_role && role == P.kv_role && cand.kv_policy == ORC_KV_AFFINITY) return f + home[j];
    const orc_role& R = P.roles[role];
    uint32_t pol = R.route;
    if ((pol == ORC_JSQ || pol == ORC_RR) && cand.route_override != ORC_ROUTE_NONE) pol = cand.route_override;
    if (pol == ORC_RR) return f + (rr[role]++ % n);
    if (pol == ORC_FIXED) return f + R.route_fixed;
    if (pol == ORC_SELECT) return sel[role];
    std::vector<uint32_t> loads(n);
    for (uint32_t i = 0; i < n; ++i) loads[i] = cand.stale_jsq ? inst[f + i].snap : inst[f + i].load();
    return f + jsq(loads.data(), n);
  }

  void set_overflow(uint32_t kind, uint32_t i) {
    if (!overflow) tr(TR_OVERFLOW, kind, i, 0);
    overflow = true;
  }

  // M9: push one message onto link l (emitted at tick t by an item of request j).
  void emit(uint32_t l, uint32_t j, uint32_t tokens, uint32_t opens, uint32_t closes, uint32_t n_in,
            uint32_t& sticky) {
    const orc_link& L = P.links[l];
    uint32_t dest;
    uint32_t kv_kind = 0;
    uint64_t ready = 0;
    if (opens) {
      dest = route(L.dst, j);
      sticky = dest;
      o[j] += 1;                                        // M13: +1 per opening message
      // M23: an opening message routed away from its KV home is charged by the KV policy
      if (P.kv_role && L.dst == P.kv_role && cand.kv_policy >= ORC_KV_RECOMPUTE &&
          dest != role_first[L.dst] + home[j]) {
        kv_kind = cand.kv_policy;
        ready = t + (uint64_t)P.kv_tau_xfer * P.kv_ctx_tokens;   // hinted transfer starts now
      }
    } else {
      dest = sticky;
    }
    tr(TR_EMIT, dest, j, tokens | (opens << 16) | (closes << 17) | (l << 20));
    if (inst[dest].inflight >= P.roles[L.dst].flight_cap) { set_overflow(1, dest); return; }
    inst[dest].inflight++;
    S.msgs_emitted++;
    S.tokens_emitted += tokens;
    // M30 pacing ("consecutive emissions on one link are >= pacing_gap apart"): the message
    // is dispatched at d = max(t, previous dispatch + gap) and arrives at d + net
    const uint64_t gap = cand.pacing_gap == 0xFFFFFFFFu ? L.pacing_gap : cand.pacing_gap;
    uint64_t d = t;
    if (gap) {
      d = std::max<uint64_t>(t, pace_free[l]);
      pace_free[l] = d + gap;
    }
    Event e{d + L.net, PH_DELIVER, ++seq, Msg{j, dest, l, opens, closes, tokens, n_in, kv_kind, ready}};
    heap.push(e);
  }

  void request_complete(uint32_t j) {  // M13, M18, M19
    nsys--;
    uint64_t e2e = t - A[j];
    uint64_t ffl = ff[j] - A[j];
    uint32_t e32 = e2e > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)e2e;
    uint32_t f32 = ffl > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)ffl;
    // a record field saturates at 2^32-1 (M18); a record holding the sentinel counts as saturated
    // (reading R-SAT).  The sums stay exact u64 (M19: "sum e2e, sum ff (u64)").
    if (e2e >= 0xFFFFFFFFull || ffl >= 0xFFFFFFFFull) S.n_saturated++;
    if (rec) { rec[2 * S.completed] = e32; rec[2 * S.completed + 1] = f32; }
    hist[bin_of(e32)]++;
    hist[ORC_NBINS + bin_of(f32)]++;
    if (cls[j]) {                    // M29 per-class metrics
      hist[2 * ORC_NBINS + bin_of(e32)]++;
      S.completed_int++;
      S.sum_e2e_int += e2e;
      if (e2e <= P.slo) S.good_int++;
      ve_int.push_back(e32);
    }
    S.completed++;
    S.sum_e2e += e2e;
    S.sum_ff += ffl;
    S.max_e2e = std::max(S.max_e2e, e32);
    if (e2e <= P.slo) S.good++;
    w_n++;
    if (e2e <= cand.policy_slo) w_good++;
    if (2 * (u128)e2e <= cand.policy_slo) w_half++;
    tr(TR_REQ_DONE, j, e32, f32);
  }

  void item_complete(uint32_t i, uint32_t j) {
    if (inst[i].c.large) S.large_items++;
    if (--o[j] == 0) request_complete(j);
  }

  void feedback(uint32_t role, uint32_t j) {  // M13 first feedback
    if (role == P.feedback_role && ff[j] == UINT64_MAX) ff[j] = t;
  }

  void complete(uint32_t i) {  // phase COMPLETE for instance i
    Inst& I = inst[i];
    const uint32_t role = I.role;
    const orc_role& R = P.roles[role];
    if (I.state == RECV) {
      Msg m = I.cur;
      I.state = IDLE;
      S.recv_steps++;
      tr(TR_RECV_DONE, i, m.j, m.opens | (m.closes << 1));
      if (m.closes) {  // M8: the item's input is complete
        uint64_t out;
        if (role == 0) out = Oj[m.j];
        else out = (uint64_t)R.out_fixed + ((uint64_t)m.n_in * R.out_num) / R.out_den;
        if (out > 65535) out = 65535;
        if (out > 0) {
          if (I.wait.size() >= R.wait_cap) { set_overflow(2, i); return; }
          I.wait.push_back({m.j, (uint32_t)out});
          tr(TR_ITEM_WAIT, i, m.j, (uint32_t)out);
        } else {  // tool item: forward one 0-token message per out-link, complete now (M9)
          for (uint32_t l : out_links[role]) {
            uint32_t st = 0;
            emit(l, m.j, 0, 1, 1, 0, st);
            if (overflow) return;
          }
          feedback(role, m.j);
          item_complete(i, m.j);
        }
      }
    } else if (I.state == DECODE) {
      I.state = IDLE;
      S.decode_steps++;
      tr(TR_DECODE_DONE, i, (uint32_t)I.batch.size(), 0);
      std::vector<Item> keep;
      for (Item& it : I.batch) {  // sequences in batch order
        it.done += 1;
        S.tokens += 1;
        uint32_t d = it.done;
        const std::vector<uint32_t>& ol = out_links[role];
        for (size_t q = 0; q < ol.size(); ++q) {  // out-links in index order
          uint32_t l = ol[q];
          if (it.mode[q] == ORC_BATCH) {
            if (d == it.out) emit(l, it.j, it.out, 1, 1, it.out, it.sticky[q]);
          } else if (it.mode[q] == ORC_FUNCTION) {
            uint32_t F = std::min(R.n_functions, it.out);
            uint32_t next = (uint32_t)(((uint64_t)(it.fidx[q] + 1) * it.out) / F);
            if (d == next) {
              uint32_t prev = (uint32_t)(((uint64_t)it.fidx[q] * it.out) / F);
              emit(l, it.j, next - prev, 1, 1, next - prev, it.sticky[q]);
              it.fidx[q]++;
            }
          } else {  // TOKEN(c)
            uint32_t c = P.links[l].chunk;
            if (d - it.last[q] == c || d == it.out) {
              emit(l, it.j, d - it.last[q], it.opened[q] ? 0 : 1, d == it.out ? 1 : 0, it.out,
                   it.sticky[q]);
              it.last[q] = d;
              it.opened[q] = 1;
            }
          }
          if (overflow) return;
        }
        if (d == 1) feedback(role, it.j);
        if (d == it.out) item_complete(i, it.j);
        else keep.push_back(it);
      }
      I.batch.swap(keep);
    }
  }

  void start(uint32_t i) {  // phase START for an idle instance (M7)
    Inst& I = inst[i];
    const orc_role& R = P.roles[I.role];
    if (!I.inbox.empty()) {  // RECV-first
      // M27: with priority service, the first interactive message, else the head (FIFO per class)
      size_t at = 0;
      if (cand.prio)
        for (size_t k = 0; k < I.inbox.size(); ++k)
          if (cls[I.inbox[k].j]) { at = k; break; }
      Msg m = I.inbox[at];
      I.inbox.erase(I.inbox.begin() + (long)at);
      uint64_t cost = (uint64_t)I.c.h + (uint64_t)I.c.beta * m.tokens;
      if (m.opens) {
        uint32_t ord = nitems[m.j]++;
        uint64_t a = I.c.alpha;
        if (R.svc_exp) {
          uint32_t w[4];
          draw(G.master_seed, m.j, s_coord, K_SVC, I.role, ord, w);
          a = exp_sample(I.c.alpha, w[0]);
        }
        cost += a;
      }
      if (m.opens && m.kv_kind) {  // M23: KV penalty of an opening RECV away from the KV home
        uint64_t pen;
        if (m.kv_kind == ORC_KV_RECOMPUTE) pen = (uint64_t)I.c.beta * P.kv_ctx_tokens;
        else if (m.kv_kind == ORC_KV_POSTHOC) pen = (uint64_t)P.kv_tau_xfer * P.kv_ctx_tokens;
        else pen = m.ready > t ? m.ready - t : 0;       // HINT: remaining hinted-transfer time
        cost += pen;
        S.kv_transfers++;
      }
      if (cost < 1) cost = 1;
      I.state = RECV;
      I.cur = m;
      I.end = t + cost;
      heap.push(Event{I.end, PH_COMPLETE, i, Msg{}});
      tr(TR_RECV_START, i, m.j, (uint32_t)cost);
      return;
    }
    while (I.batch.size() < I.B && !I.wait.empty()) {  // FIFO admission; modes bound here (M9)
      size_t at = 0;                                   // M27: interactive first with priority service
      if (cand.prio)
        for (size_t k = 0; k < I.wait.size(); ++k)
          if (cls[I.wait[k].first]) { at = k; break; }
      Item it{};
      it.j = I.wait[at].first;
      it.out = I.wait[at].second;
      I.wait.erase(I.wait.begin() + (long)at);
      const std::vector<uint32_t>& ol = out_links[I.role];
      for (size_t q = 0; q < ol.size(); ++q) it.mode[q] = cur_mode[ol[q]];
      I.batch.push_back(it);
    }
    if (!I.batch.empty()) {
      uint64_t cost = (uint64_t)I.c.tau0 + (uint64_t)I.c.gamma * I.batch.size();
      if (cost < 1) cost = 1;
      I.state = DECODE;
      I.end = t + cost;
      heap.push(Event{I.end, PH_COMPLETE, i, Msg{}});
      tr(TR_DECODE_START, i, (uint32_t)I.batch.size(), (uint32_t)cost);
    }
  }

  void arrive(uint32_t j) {  // phase ARRIVE (M14)
    S.arrivals++;
    if (gate_closed && !cls[j]) {   // M28: interactive-only admission rejects a background request
      S.dropped++;
      S.rejected++;
      tr(TR_ARRIVE, j, 2, 0xFFFFFFFFu);
      return;
    }
    if (nsys >= P.request_cap) {
      S.dropped++;
      tr(TR_ARRIVE, j, 0, 0xFFFFFFFFu);
      return;
    }
    S.admitted++;
    nsys++;
    o[j] = 1;                       // M13: +1 on admission (the source item)
    uint32_t dest = route(0, j);
    tr(TR_ARRIVE, j, 1, dest);
    if (inst[dest].inbox.size() >= P.roles[0].inbox_cap) { set_overflow(0, dest); return; }
    inst[dest].inbox.push_back(Msg{j, dest, 0xFFFFFFFFu, 1, 1, Pj[j], Pj[j], 0, 0});
  }

  void deliver(const Msg& m) {  // phase DELIVER
    Inst& I = inst[m.dest];
    I.inflight--;
    S.deliveries++;
    S.msgs_received++;
    S.tokens_received += m.tokens;
    tr(TR_DELIVER, m.dest, m.j, m.tokens);
    if (I.inbox.size() >= P.roles[I.role].inbox_cap) { set_overflow(0, m.dest); return; }
    I.inbox.push_back(m);
  }

  void advance(uint64_t t_next) {  // integrate piecewise-constant state over [t, t_next) (M15)
    uint64_t dt = t_next - t;
    for (Inst& I : inst) {
      if (I.state != IDLE) I.w_busy += dt;
      I.w_qint += (uint64_t)I.Q() * dt;
      I.w_maxq = std::max(I.w_maxq, I.Q());
      I.w_lint += (uint64_t)I.load() * dt;
    }
    S.int_nsys += (uint64_t)nsys * dt;
  }

  void write_series(uint64_t k) {
    if (!cser.empty() && k < G.series_windows) {      // M15 cell-summed series (reading R-CSER)
      for (size_t i = 0; i < inst.size(); ++i) {
        const Inst& I = inst[i];
        uint64_t* e = &cser[(k * inst.size() + i) * 8];
        int32_t il = in_link[I.role];
        e[0] += I.w_qint;
        e[1] += I.w_busy;
        e[2] += 1;                                       // replicas that closed window k
        e[3] += I.w_maxq;
        e[4] += I.B;
        if (il >= 0) e[5 + cur_mode[il]] += 1;           // replicas per in-link mode
      }
    }
    if (!series || k >= G.series_windows) return;
    for (size_t i = 0; i < inst.size(); ++i) {
      const Inst& I = inst[i];
      orc_series& e = series[k * inst.size() + i];
      e.qint = I.w_qint;
      e.busy = (uint32_t)I.w_busy;
      e.maxq = (uint16_t)std::min<uint32_t>(I.w_maxq, 65535u);
      int32_t il = in_link[I.role];
      e.mode = il < 0 ? 255 : (uint8_t)cur_mode[il];
      e.B = (uint8_t)I.B;
    }
  }

  void control(int64_t q) {  // M16, at the close of window q-1
    const uint64_t W = P.window;
    // (i) three-band mode policy per controlled link, and M25 (f3, compiled intents): a guarded link
    // is set to BATCH while fewer than ceil(guard_pct * n / 100) of the window's n >= 1 completions
    // met policy_slo (its guard_pct-quantile violates the bound), and otherwise reset to its initial
    // mode -- unless the band policy drives it, which then decides.  One decision per link per window,
    // with the same dwell / no-op suppression.
    bool gviol = false;
    if (cand.guard_links && w_n >= 1) gviol = w_good < (uint32_t)(((uint64_t)cand.guard_pct * w_n + 99) / 100);
    for (uint32_t l = 0; l < P.n_links; ++l) {
      const bool ctl = (cand.ctl_links >> l) & 1, grd = (cand.guard_links >> l) & 1;
      if (!ctl && !grd) continue;
      uint32_t nm;
      if (grd && gviol) {
        nm = cur_mode[l];
        if (nm != ORC_BATCH && q - q_last_mode[l] >= (int64_t)cand.dwell) { nm = ORC_BATCH; q_last_mode[l] = q; }
      } else if (ctl) {
        uint32_t d = P.links[l].dst;
        uint64_t u = 0;
        for (uint32_t x = 0; x < role_n[d]; ++x) {
          const Inst& I = inst[role_first[d] + x];
          u += cand.metric_load ? I.w_lint : I.w_busy;
        }
        nm = mode_step(u, cand.lo, cand.hi, W, role_n[d], cand.band, cand.dwell, q, cur_mode[l], &q_last_mode[l]);
      } else {
        nm = cur_mode[l];
        if (w_n >= 1 && nm != base_mode[l] && q - q_last_mode[l] >= (int64_t)cand.dwell) {
          nm = base_mode[l];
          q_last_mode[l] = q;
        }
      }
      if (nm != cur_mode[l]) {
        cur_mode[l] = nm;
        S.mode_switches++;
        tr(TR_CONTROL, 0, l, nm);
      }
    }
    bool viol = false, calm = false;
    if (w_n >= 1) {
      uint32_t k99 = (uint32_t)((99ull * w_n + 99) / 100);
      viol = w_good < k99;
      calm = w_half >= k99;
    }
    // (ii) SLO-aware batch size (set / reset of max_num_seqs)
    if (cand.batch_roles && w_n >= 1) {
      for (uint32_t r = 0; r < P.n_roles; ++r) {
        if (!((cand.batch_roles >> r) & 1)) continue;
        for (uint32_t x = 0; x < role_n[r]; ++x) {
          uint32_t i = role_first[r] + x;
          Inst& I = inst[i];
          uint32_t nb = I.B;
          if (viol) nb = (I.w_qint > (uint64_t)cand.q_hi * W) ? std::min(32u, 2 * I.B) : std::max(1u, I.B / 2);
          else if (calm) nb = I.B_default;
          if (nb != I.B && q - I.q_last_B >= (int64_t)cand.dwell) {
            I.B = nb;
            I.q_last_B = q;
            S.batch_changes++;
            tr(TR_CONTROL, 1, i, nb);
          }
        }
      }
    }
    // (iv) M28 admission gate on the source role's busy time, dwell and no-op as M16
    if (cand.admit) {
      uint64_t u = 0;
      for (uint32_t x = 0; x < role_n[0]; ++x) u += inst[role_first[0] + x].w_busy;
      bool want = gate_closed;
      if ((u128)u * 1000u >= (u128)cand.admit_hi * W * role_n[0]) want = true;
      else if ((u128)u * 1000u <= (u128)cand.admit_lo * W * role_n[0]) want = false;
      if (want != gate_closed && q - q_last_gate >= (int64_t)cand.dwell) {
        gate_closed = want;
        q_last_gate = q;
        S.gate_changes++;
        tr(TR_CONTROL, 3, 0, want ? 1u : 0u);
      }
    }
    // (iii) model selection (SELECT routing target)
    if (cand.select_role >= 0) {
      uint32_t r = (uint32_t)cand.select_role;
      uint32_t large_i = role_first[r], small_i = role_first[r] + role_n[r] - 1;
      for (uint32_t x = role_n[r]; x-- > 0;) if (inst[role_first[r] + x].c.large) large_i = role_first[r] + x;
      for (uint32_t x = role_n[r]; x-- > 0;) if (!inst[role_first[r] + x].c.large) small_i = role_first[r] + x;
      uint32_t cur = sel[r];
      u128 b1000 = (u128)inst[cur].w_busy * 1000u;
      uint32_t ns = cur;
      if (b1000 >= (u128)cand.hi * W || viol) ns = small_i;
      else if (b1000 <= (u128)cand.lo * W && !viol) ns = large_i;
      if (ns != cur && q - q_last_sel >= (int64_t)cand.dwell) {
        sel[r] = ns;
        q_last_sel = q;
        S.select_changes++;
        tr(TR_CONTROL, 2, r, ns);
      }
    }
  }

  void close_window(uint64_t k, bool final_partial) {
    write_series(k);
    if (!final_partial) {
      S.window_closes++;
      tr(TR_WINDOW, (uint32_t)k, 0, 0);
      if (cand.adaptive) control((int64_t)k + 1);
    }
    for (Inst& I : inst) { I.w_busy = I.w_qint = I.w_lint = 0; I.w_maxq = 0; }
    if (!final_partial)               // M31: the controller's poll of every instance's load
      for (Inst& I : inst) I.snap = I.load();
    w_n = w_good = w_half = 0;
  }

  int run() {
    const uint32_t N = G.n_requests;
    // topology
    uint32_t n_inst = 0;
    role_first.resize(P.n_roles); role_n.resize(P.n_roles);
    out_links.assign(P.n_roles, {}); in_link.assign(P.n_roles, -1);
    for (uint32_t r = 0; r < P.n_roles; ++r) {
      role_first[r] = n_inst;
      role_n[r] = P.roles[r].n_instances;
      for (uint32_t x = 0; x < role_n[r]; ++x) {
        Inst I;
        I.role = r;
        I.c = P.roles[r].inst_cost ? P.roles[r].inst_cost[x] : P.roles[r].cost;
        I.B = I.B_default = P.roles[r].max_num_seqs;
        inst.push_back(I);
      }
      n_inst += role_n[r];
    }
    for (uint32_t l = 0; l < P.n_links; ++l) {
      out_links[P.links[l].src].push_back(l);
      in_link[P.links[l].dst] = (int32_t)l;
    }
    cur_mode.resize(P.n_links);
    q_last_mode.assign(P.n_links, INT64_MIN / 2);
    for (uint32_t l = 0; l < P.n_links; ++l)
      cur_mode[l] = cand.mode[l] == 255 ? P.links[l].mode : cand.mode[l];
    base_mode = cur_mode;
    rr.assign(P.n_roles, 0);
    pace_free.assign(P.n_links, 0);
    sel.resize(P.n_roles);
    for (uint32_t r = 0; r < P.n_roles; ++r) {
      sel[r] = role_first[r];
      for (uint32_t x = role_n[r]; x-- > 0;) if (inst[role_first[r] + x].c.large) sel[r] = role_first[r] + x;
    }
    // workload (M4, M5)
    uint32_t r_i = 0, r_k = 0;
    {
      uint64_t g = rid / G.n_cand;
      uint64_t ik = g / G.n_seeds;
      r_k = (uint32_t)(ik % G.n_profiles);
      r_i = (uint32_t)(ik / G.n_profiles);
    }
    const orc_arrival& arr = G.arr[r_i * G.n_profiles + r_k];
    if (gen_arrivals(arr, G.master_seed, s_coord, N, A, Pj, Oj) != 0) return -1;
    o.assign(N, 0); nitems.assign(N, 0); ff.assign(N, UINT64_MAX);
    home.assign(N, 0);
    cls.assign(N, 0);
    if (arr.interactive_permille) {  // M26: class from ATTR draw sub-counter 1, word 0
      const uint64_t thr = ((uint64_t)arr.interactive_permille << 32) / 1000;
      for (uint32_t j = 0; j < N; ++j) {
        uint32_t w[4];
        draw(G.master_seed, j, s_coord, K_ATTR, 0, 1, w);
        cls[j] = (uint64_t)w[0] < thr ? 1 : 0;
      }
    }
    if (P.kv_role) {  // M21: KV home of every request, from ATTR words 2 and 3
      const uint64_t skew32 = ((uint64_t)P.kv_home_skew << 32) / 1000;
      for (uint32_t j = 0; j < N; ++j) {
        uint32_t w[4];
        draw(G.master_seed, j, s_coord, K_ATTR, 0, 0, w);
        home[j] = (uint64_t)w[2] < skew32 ? 0 : uni(0, role_n[P.kv_role] - 1, w[3]);
      }
    }

    const uint64_t W = P.window;
    uint64_t next_boundary = W;
    bool started = false;
    S.replica = rid;
    // event loop (M12)
    for (;;) {
      bool finished = (jn == N && nsys == 0);
      if (finished || overflow) break;
      uint64_t t_next = next_boundary;
      if (jn < N) t_next = std::min(t_next, A[jn]);
      if (!heap.empty()) t_next = std::min(t_next, heap.top().tick);
      if (G.max_ticks && t_next > G.max_ticks) { S.status = ORC_TRUNCATED; break; }
      if (started || t_next > 0) advance(t_next);
      started = true;
      t = t_next;
      // Phase 0: WINDOW
      if (t == next_boundary) {
        close_window(t / W - 1, false);
        next_boundary += W;
      }
      // collect heap events at t
      std::vector<Event> evs;
      while (!heap.empty() && heap.top().tick == t) { evs.push_back(heap.top()); heap.pop(); }
      // Phase 1: COMPLETE (instance order), Phase 2: DELIVER (emission-seq order)
      for (const Event& e : evs) {
        if (e.phase == PH_COMPLETE) complete((uint32_t)e.entity);
        if (overflow) break;
      }
      if (overflow) break;
      for (const Event& e : evs) {
        if (e.phase == PH_DELIVER) deliver(e.msg);
        if (overflow) break;
      }
      if (overflow) break;
      // Phase 3: ARRIVE (increasing j)
      while (jn < N && A[jn] == t) {
        arrive(jn++);
        if (overflow) break;
      }
      if (overflow) break;
      // Phase 4: START (increasing instance index)
      for (uint32_t i = 0; i < n_inst; ++i)
        if (inst[i].state == IDLE) start(i);
    }
    if (overflow) {
      uint64_t r = rid;
      uint64_t tk = t;
      std::memset(&S, 0, sizeof(S));
      S.status = ORC_OVERFLOW;
      S.stop_tick = tk;
      S.replica = r;
      std::memset(hist, 0, sizeof(uint32_t) * ORC_NHIST * ORC_NBINS);
      S.p50_e2e = S.p99_e2e = S.p50_ff = S.p99_ff = 0xFFFFFFFFu;
      S.p50_e2e_int = S.p99_e2e_int = 0xFFFFFFFFu;
      S.bin_p50_e2e = S.bin_p99_e2e = S.bin_p50_ff = S.bin_p99_ff = 0xFFFFu;
      S.p90_e2e = 0xFFFFFFFFu;
      return 0;
    }
    // final partial window: series only
    close_window(t / W, true);
    S.makespan = t;
    S.stop_tick = t;
    // M18 exact nearest-rank percentiles and their bins
    std::vector<uint32_t> ve, vf;
    if (rec) {
      for (uint32_t k = 0; k < S.completed; ++k) { ve.push_back(rec[2 * k]); vf.push_back(rec[2 * k + 1]); }
    }
    auto pct = [&](std::vector<uint32_t>& v, const uint32_t* h, uint32_t num, uint32_t& val, uint32_t& bin) {
      uint64_t n = S.completed;
      if (n == 0) { val = 0xFFFFFFFFu; bin = 0xFFFFu; return; }
      uint64_t k = (num * n + 99) / 100;
      std::sort(v.begin(), v.end());
      val = v[k - 1];
      uint64_t cum = 0;
      for (uint32_t b = 0; b < ORC_NBINS; ++b) {
        cum += h[b];
        if (cum >= k) { bin = b; break; }
      }
    };
    pct(ve, hist, 50, S.p50_e2e, S.bin_p50_e2e);
    pct(ve, hist, 99, S.p99_e2e, S.bin_p99_e2e);
    uint32_t bin90;
    pct(ve, hist, 90, S.p90_e2e, bin90);
    pct(vf, hist + ORC_NBINS, 50, S.p50_ff, S.bin_p50_ff);
    pct(vf, hist + ORC_NBINS, 99, S.p99_ff, S.bin_p99_ff);
    // M29: exact nearest-rank percentiles over the interactive completions alone
    S.p50_e2e_int = S.p99_e2e_int = 0xFFFFFFFFu;
    if (!ve_int.empty()) {
      std::sort(ve_int.begin(), ve_int.end());
      uint64_t n = ve_int.size();
      S.p50_e2e_int = ve_int[(50 * n + 99) / 100 - 1];
      S.p99_e2e_int = ve_int[(99 * n + 99) / 100 - 1];
    }
    return 0;
  }
};

int validate(const orc_pipeline* p, const orc_grid* g) {
  if (!p || !g || p->n_roles == 0 || g->n_cand == 0 || g->n_rates == 0 || g->n_profiles == 0 ||
      g->n_seeds == 0)
    return -1;
  if (p->n_links > ORC_MAX_LINKS || p->window == 0 || p->request_cap == 0 || p->feedback_role >= p->n_roles)
    return -1;
  std::vector<int> indeg(p->n_roles, 0);
  for (uint32_t l = 0; l < p->n_links; ++l) {
    const orc_link& L = p->links[l];
    if (L.src >= L.dst || L.dst >= p->n_roles || L.net < 1 || L.chunk < 1 || L.mode > 2) return -1;
    indeg[L.dst]++;
  }
  for (uint32_t r = 1; r < p->n_roles; ++r)
    if (indeg[r] != 1) return -1;  // M6: role 0 is the unique source; no joins
  if (p->kv_role >= p->n_roles || p->kv_home_skew > 1000) return -1;
  for (uint32_t r = 0; r < p->n_roles; ++r) {
    const orc_role& R = p->roles[r];
    if (R.n_instances < 1 || R.max_num_seqs < 1 || R.max_num_seqs > 32 || R.out_den < 1 || R.n_functions < 1)
      return -1;
  }
  return 0;
}

}  // namespace

extern "C" {

void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) { philox(ctr, key, out); }
uint64_t orc_log2_table(uint32_t i) { return i <= 256 ? table().t[i] : 0; }
uint64_t orc_exp_sample(uint64_t mean, uint32_t x) { return exp_sample(mean, x); }
uint32_t orc_uni(uint32_t lo, uint32_t hi, uint32_t x) { return uni(lo, hi, x); }
uint32_t orc_bin(uint32_t v) { return bin_of(v); }
uint64_t orc_bin_lo(uint32_t b) { return bin_lo(b); }
uint32_t orc_band(uint64_t u, uint32_t lo, uint32_t hi, uint64_t window, uint32_t n) {
  return band_of(u, lo, hi, window, n);
}
uint32_t orc_jsq(const uint32_t* loads, uint32_t n) { return jsq(loads, n); }
uint32_t orc_mode_step(uint64_t u, uint32_t lo, uint32_t hi, uint64_t window, uint32_t n, const uint32_t* band,
                       uint32_t dwell, int64_t q, uint32_t cur, int64_t* q_last) {
  return mode_step(u, lo, hi, window, n, band, dwell, q, cur, q_last);
}

int orc_arrivals(const orc_arrival* a, uint64_t master_seed, uint32_t s_coord, uint32_t n, uint64_t* ticks,
                 uint32_t* prompt, uint32_t* output) {
  std::vector<uint64_t> A;
  std::vector<uint32_t> P, O;
  int rc = gen_arrivals(*a, master_seed, s_coord, n, A, P, O);
  if (rc) return rc;
  for (uint32_t j = 0; j < n; ++j) {
    ticks[j] = A[j];
    if (prompt) prompt[j] = P[j];
    if (output) output[j] = O[j];
  }
  return 0;
}

int orc_simulate(const orc_pipeline* p, const orc_grid* g, const uint64_t* ids, uint64_t n, uint32_t threads,
                 orc_summary* out, uint32_t* records, uint32_t* hists, orc_series* series, uint64_t trace_id,
                 orc_trace* trace, uint64_t trace_cap, uint64_t* trace_n, uint64_t* cell_series) {
  if (validate(p, g)) return -1;
  uint32_t n_inst = 0;
  for (uint32_t r = 0; r < p->n_roles; ++r) n_inst += p->roles[r].n_instances;
  if (trace_n) *trace_n = 0;
  std::atomic<uint64_t> next(0);
  std::atomic<int> err(0);
  std::mutex cs_mu;
  const uint64_t cs_per_cell = (uint64_t)g->series_windows * n_inst * 8;
  auto worker = [&]() {
    std::vector<uint32_t> hbuf(ORC_NHIST * ORC_NBINS);
    std::vector<uint32_t> rbuf;
    for (;;) {
      uint64_t x = next.fetch_add(1);
      if (x >= n) break;
      uint64_t rid = ids[x];
      uint64_t g_idx = rid / g->n_cand;
      uint32_t s = (uint32_t)(g_idx % g->n_seeds) + g->seed_offset;
      const orc_candidate& c = g->cand[rid % g->n_cand];
      std::memset(&out[x], 0, sizeof(orc_summary));
      uint32_t* h = hists ? hists + x * ORC_NHIST * ORC_NBINS : hbuf.data();
      std::memset(h, 0, sizeof(uint32_t) * ORC_NHIST * ORC_NBINS);
      uint32_t* rec;
      if (records) rec = records + x * 2ull * g->n_requests;
      else { rbuf.assign(2ull * g->n_requests, 0); rec = rbuf.data(); }
      Replica R(*p, *g, c, rid, s, out[x]);
      R.rec = rec;
      R.hist = h;
      R.series = nullptr;
      if (series && g->series_stride && rid % g->series_stride == 0 && rid / g->series_stride < g->series_slots)
        R.series = series + (rid / g->series_stride) * (uint64_t)g->series_windows * n_inst;
      R.trace = (trace && rid == trace_id) ? trace : nullptr;
      R.trace_cap = trace_cap;
      R.trace_n = trace_n;
      if (cell_series && g->series_windows) R.cser.assign(cs_per_cell, 0);
      if (R.run() != 0) err = -1;
      if (cell_series && g->series_windows) {          // cell (i, k, c) of replica rid
        const uint64_t cell = (g_idx / g->n_seeds) * g->n_cand + rid % g->n_cand;
        std::lock_guard<std::mutex> lk(cs_mu);
        for (uint64_t q = 0; q < cs_per_cell; ++q) cell_series[cell * cs_per_cell + q] += R.cser[q];
      }
    }
  };
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  for (uint32_t t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  return err.load();
}

void orc_cells(const orc_grid* g, const orc_summary* sums, const uint32_t* hists, int64_t* cnt, int64_t* hist) {
  uint64_t C = g->n_cand, S = g->n_seeds, K = g->n_profiles, I = g->n_rates;
  uint64_t n_cells = I * K * C;
  std::memset(cnt, 0, sizeof(int64_t) * n_cells * ORC_NCNT);
  std::memset(hist, 0, sizeof(int64_t) * n_cells * ORC_NHIST * ORC_NBINS);
  for (uint64_t r = 0; r < I * K * S * C; ++r) {
    uint64_t c = r % C, gg = r / C, ik = gg / S;
    uint64_t cell = ik * C + c;
    const orc_summary& x = sums[r];
    int64_t* q = cnt + cell * ORC_NCNT;
    q[0] += 1;
    if (x.status == ORC_OVERFLOW) { q[2] += 1; continue; }
    if (x.status == ORC_OK) q[1] += 1;
    if (x.status == ORC_TRUNCATED) q[3] += 1;
    q[4] += x.admitted; q[5] += x.dropped; q[6] += x.completed; q[7] += x.sum_e2e; q[8] += x.sum_ff;
    q[9] += x.makespan; q[10] += x.int_nsys; q[11] += x.good; q[12] += x.large_items; q[13] += x.arrivals;
    q[14] += x.deliveries; q[15] += x.recv_steps; q[16] += x.decode_steps; q[17] += x.window_closes;
    q[18] += x.mode_switches; q[19] += x.tokens; q[20] += x.batch_changes; q[21] += x.select_changes;
    q[22] += x.n_saturated; q[23] += x.kv_transfers;
    q[24] += x.completed_int; q[25] += x.rejected; q[26] += x.sum_e2e_int; q[27] += x.good_int;
    for (int b = 0; b < ORC_NHIST * ORC_NBINS; ++b)
      hist[cell * ORC_NHIST * ORC_NBINS + b] += hists[r * ORC_NHIST * ORC_NBINS + b];
  }
}

}  // extern "C"

namespace {
// M20 comparison keys.  `better(a, b)` is a strict total order once c breaks ties.
struct Key {
  uint32_t bad;
  uint64_t dropped, p, sum, completed, makespan, good, large;
  uint32_t c;
};
// na/ma > nb/mb; a zero makespan is rate 0 (reading R-RATE0), which keeps the order total
bool rate_gt(uint64_t na, uint64_t ma, uint64_t nb, uint64_t mb) {
  if (ma == 0) { na = 0; ma = 1; }
  if (mb == 0) { nb = 0; mb = 1; }
  return (u128)na * mb > (u128)nb * ma;
}
bool better(const Key& a, const Key& b, uint32_t obj, uint64_t slo) {
  if (a.bad != b.bad) return a.bad < b.bad;
  switch (obj) {
    case ORC_OBJ_THROUGHPUT:
    case ORC_OBJ_GOODPUT: {
      uint64_t na = obj == ORC_OBJ_GOODPUT ? a.good : a.completed;
      uint64_t nb = obj == ORC_OBJ_GOODPUT ? b.good : b.completed;
      if (rate_gt(na, a.makespan, nb, b.makespan)) return true;
      if (rate_gt(nb, b.makespan, na, a.makespan)) return false;
      if (a.p != b.p) return a.p < b.p;
      break;
    }
    case ORC_OBJ_LARGE_UNDER_SLO: {
      bool fa = a.dropped == 0 && a.p <= slo, fb = b.dropped == 0 && b.p <= slo;
      if (fa != fb) return fa;
      if (fa) {
        if (a.large != b.large) return a.large > b.large;
      } else {
        if (a.dropped != b.dropped) return a.dropped < b.dropped;
      }
      if (a.p != b.p) return a.p < b.p;
      break;
    }
    case ORC_OBJ_P99_E2E_INT:   // interactive latency only: background drops are the gate's business
      if (a.p != b.p) return a.p < b.p;
      if (a.sum != b.sum) return a.sum < b.sum;
      break;
    default:
      if (a.dropped != b.dropped) return a.dropped < b.dropped;
      if (a.p != b.p) return a.p < b.p;
      if (a.sum != b.sum) return a.sum < b.sum;
      break;
  }
  return a.c < b.c;
}

// M18 on a pooled cell histogram: the lower edge of the bin holding the nearest-rank num-th percentile
// (the first bin whose cumulative count reaches ceil(num n / 100)); UINT32_MAX for an empty histogram.
uint64_t pooled_pct(const int64_t* h, uint32_t num) {
  uint64_t n = 0;
  for (int b = 0; b < ORC_NBINS; ++b) n += (uint64_t)h[b];
  if (n == 0) return 0xFFFFFFFFull;
  const uint64_t k = (num * n + 99) / 100;
  uint64_t cum = 0;
  for (uint32_t b = 0; b < ORC_NBINS; ++b) {
    cum += (uint64_t)h[b];
    if (cum >= k) return bin_lo(b);
  }
  return 0xFFFFFFFFull;
}
}  // namespace

extern "C" {

uint64_t orc_pooled_pct(const int64_t* hist, uint32_t num) { return pooled_pct(hist, num); }

void orc_argmin_groups(const orc_grid* g, const orc_summary* sums, uint32_t obj, uint64_t slo, int32_t* best) {
  uint64_t C = g->n_cand;
  uint64_t n_groups = (uint64_t)g->n_rates * g->n_profiles * g->n_seeds;
  for (uint64_t gg = 0; gg < n_groups; ++gg) {
    Key bk{};
    int32_t bc = -1;
    for (uint64_t c = 0; c < C; ++c) {
      const orc_summary& x = sums[gg * C + c];
      Key k{};
      k.bad = x.status != ORC_OK;
      k.dropped = x.dropped;
      k.p = obj == ORC_OBJ_P50_E2E ? x.p50_e2e : obj == ORC_OBJ_P99_FF ? x.p99_ff
          : obj == ORC_OBJ_P90_E2E ? x.p90_e2e : obj == ORC_OBJ_P99_E2E_INT ? x.p99_e2e_int : x.p99_e2e;
      k.sum = obj == ORC_OBJ_P99_FF ? x.sum_ff : obj == ORC_OBJ_P99_E2E_INT ? x.sum_e2e_int : x.sum_e2e;
      k.completed = x.completed; k.makespan = x.makespan; k.good = x.good; k.large = x.large_items;
      k.c = (uint32_t)c;
      if (bc < 0 || better(k, bk, obj, slo)) { bk = k; bc = (int32_t)c; }
    }
    best[gg] = bc;
  }
}

void orc_argmin_rows(const orc_grid* g, const int64_t* cnt, const int64_t* hist, uint32_t obj, uint64_t slo,
                     int32_t* best) {
  uint64_t C = g->n_cand;
  uint64_t n_rows = (uint64_t)g->n_rates * g->n_profiles;
  for (uint64_t row = 0; row < n_rows; ++row) {
    Key bk{};
    int32_t bc = -1;
    for (uint64_t c = 0; c < C; ++c) {
      uint64_t cell = row * C + c;
      const int64_t* q = cnt + cell * ORC_NCNT;
      const int64_t* h = hist + cell * ORC_NHIST * ORC_NBINS +
                         (obj == ORC_OBJ_P99_FF ? ORC_NBINS : obj == ORC_OBJ_P99_E2E_INT ? 2 * ORC_NBINS : 0);
      const uint64_t p = pooled_pct(h, obj == ORC_OBJ_P50_E2E ? 50 : obj == ORC_OBJ_P90_E2E ? 90 : 99);
      Key k{};
      k.bad = q[1] != q[0];
      k.dropped = (uint64_t)q[5];
      k.p = p;
      k.sum = (uint64_t)(obj == ORC_OBJ_P99_FF ? q[8] : obj == ORC_OBJ_P99_E2E_INT ? q[26] : q[7]);
      k.completed = (uint64_t)q[6]; k.makespan = (uint64_t)q[9]; k.good = (uint64_t)q[11];
      k.large = (uint64_t)q[12];
      k.c = (uint32_t)c;
      if (bc < 0 || better(k, bk, obj, slo)) { bk = k; bc = (int32_t)c; }
    }
    best[row] = bc;
  }
}

}  // extern "C"
