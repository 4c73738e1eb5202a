/* oracle/oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the SDAS strategy simulator
 * (rules M0-M20).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  It shares no code, header, table or constant generator with the
 * CUDA path (paper_2601_03197_b200/ and include/sdas.h): every struct below is
 * this file's own, and the Python wrapper (oracle/__init__.py) fills them from
 * the plain dicts of workloads/.
 *
 * Parity pins: see oracle/__init__.py header and DESIGN.md §"Parity pins".
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_BATCH = 0, ORC_FUNCTION = 1, ORC_TOKEN = 2 };
enum { ORC_JSQ = 0, ORC_RR = 1, ORC_FIXED = 2, ORC_SELECT = 3, ORC_ROUTE_NONE = 255 };
enum { ORC_POISSON = 0, ORC_MMPP2 = 1, ORC_DET = 2, ORC_LIST = 3 };
enum { ORC_OK = 0, ORC_OVERFLOW = 1, ORC_TRUNCATED = 2 };
enum { ORC_KV_OFF = 0, ORC_KV_AFFINITY = 1, ORC_KV_RECOMPUTE = 2, ORC_KV_POSTHOC = 3, ORC_KV_HINT = 4 };
enum { ORC_OBJ_P99_E2E = 0, ORC_OBJ_P50_E2E = 1, ORC_OBJ_P99_FF = 2, ORC_OBJ_THROUGHPUT = 3,
       ORC_OBJ_GOODPUT = 4, ORC_OBJ_LARGE_UNDER_SLO = 5, ORC_OBJ_P90_E2E = 6, ORC_OBJ_P99_E2E_INT = 7 };

#define ORC_NBINS 464
#define ORC_MAX_LINKS 8

typedef struct { uint32_t h, alpha, beta, tau0, gamma, large; } orc_cost;

typedef struct {
  uint32_t n_instances;
  orc_cost cost;
  const orc_cost* inst_cost;  /* NULL or [n_instances] */
  uint32_t max_num_seqs;
  uint32_t out_fixed, out_num, out_den;
  uint32_t n_functions;
  uint32_t svc_exp;
  uint32_t route, route_fixed;
  uint32_t inbox_cap, flight_cap, wait_cap;
} orc_role;

typedef struct { uint32_t src, dst, net, chunk, mode, pacing_gap; } orc_link;   /* pacing_gap: M30 (f4) */

typedef struct {
  uint32_t kind;
  uint64_t gap[2], sojourn[2];
  const uint64_t* list; uint32_t list_len;
  uint32_t p_lo, p_hi, o_lo, o_hi;
  uint32_t interactive_permille;  /* M26 (f2): share of interactive requests, 0..1000 */
} orc_arrival;

typedef struct {
  uint32_t adaptive;
  uint32_t mode[ORC_MAX_LINKS];   /* static mode / initial mode; 255 = pipeline default */
  uint32_t ctl_links;             /* bitmask */
  uint32_t metric_load;           /* 0 busy, 1 load */
  uint32_t lo, hi, dwell;
  uint32_t band[3];
  uint32_t route_override;        /* ORC_ROUTE_NONE or JSQ/RR */
  uint32_t batch_roles;           /* bitmask */
  uint32_t q_hi;
  int32_t select_role;            /* -1 none */
  uint64_t policy_slo;
  uint32_t kv_policy;             /* ORC_KV_* (rules M21-M24) */
  uint32_t guard_links;           /* M25 (f3): links flipped to BATCH while the window e2e quantile */
  uint32_t guard_pct;             /*   guard_pct (e.g. 90) exceeds policy_slo; else reset to base  */
  uint32_t prio;                  /* M27 (f2): serve interactive first at every inbox and wait queue */
  uint32_t admit;                 /* M28 (f2): admission gate on the source role's busy fraction */
  uint32_t admit_lo, admit_hi;    /*   reopen at <= lo, interactive-only at >= hi (permille) */
  uint32_t pacing_gap;            /* M30 (f4): 0xFFFFFFFF = each link's own gap, else this gap on every link */
  uint32_t stale_jsq;             /* M31 (f4): JSQ ranks the loads polled at the last window close */
} orc_candidate;

typedef struct {
  uint32_t n_roles; const orc_role* roles;
  uint32_t n_links; const orc_link* links;
  uint32_t feedback_role, request_cap;
  uint64_t window, slo;
  uint32_t kv_role;               /* 0 = no KV modelling; else the role holding per-request KV context */
  uint32_t kv_ctx_tokens, kv_tau_xfer, kv_home_skew;   /* context tokens, ticks/token, permille on inst 0 */
} orc_pipeline;

typedef struct {
  uint32_t n_cand; const orc_candidate* cand;
  uint32_t n_rates, n_profiles; const orc_arrival* arr;   /* [n_rates * n_profiles] */
  uint32_t n_seeds, seed_offset; uint64_t master_seed;
  uint32_t n_requests; uint64_t max_ticks;
  uint32_t series_stride, series_slots, series_windows;
} orc_grid;

typedef struct {
  uint32_t status, admitted, dropped, completed;
  uint64_t makespan, sum_e2e, sum_ff, int_nsys;
  uint32_t p50_e2e, p99_e2e, p50_ff, p99_ff;
  uint32_t bin_p50_e2e, bin_p99_e2e, bin_p50_ff, bin_p99_ff;
  uint32_t max_e2e, n_saturated;
  uint32_t arrivals, deliveries, recv_steps, decode_steps;
  uint32_t window_closes, mode_switches, good, large_items;
  uint64_t tokens;
  uint64_t stop_tick;
  uint64_t replica;
  uint32_t batch_changes, select_changes, kv_transfers, p90_e2e;   /* p90_e2e: exact nearest rank (f3) */
  uint32_t completed_int, rejected, good_int, gate_changes;   /* M29 (f2) per-class metrics */
  uint64_t sum_e2e_int;
  uint32_t p50_e2e_int, p99_e2e_int;
  uint64_t msgs_emitted, tokens_emitted;     /* conservation checks */
  uint64_t msgs_received, tokens_received;
} orc_summary;

typedef struct { uint64_t qint; uint32_t busy; uint16_t maxq; uint8_t mode; uint8_t B; } orc_series;

typedef struct { uint64_t tick; uint32_t code, a, b, c; } orc_trace;

/* --- primitives, exported for pin tests ---------------------------------------- */
void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t orc_log2_table(uint32_t i);
uint64_t orc_exp_sample(uint64_t mean, uint32_t x);
uint32_t orc_uni(uint32_t lo, uint32_t hi, uint32_t x);
uint32_t orc_bin(uint32_t v);
uint64_t orc_bin_lo(uint32_t b);
/* arrival ticks / attributes of requests 0..n-1 for seed coordinate s (rule M4/M5) */
int orc_arrivals(const orc_arrival* a, uint64_t master_seed, uint32_t s_coord, uint32_t n,
                 uint64_t* ticks, uint32_t* prompt, uint32_t* output);
/* controller band decision (rule M16(i)); returns 0 low / 1 mid / 2 high band */
uint32_t orc_band(uint64_t u, uint32_t lo, uint32_t hi, uint64_t window, uint32_t n);
/* JSQ over loads (rule M11) */
uint32_t orc_jsq(const uint32_t* loads, uint32_t n);
/* one window close of the M16(i) mode policy (dwell, no-op suppression); q_last in/out */
uint32_t orc_mode_step(uint64_t u, uint32_t lo, uint32_t hi, uint64_t window, uint32_t n, const uint32_t* band,
                       uint32_t dwell, int64_t q, uint32_t cur, int64_t* q_last);

/* --- the simulation ---------------------------------------------------------------- */
/* Runs replicas `ids[0..n)` (global ids r = g*C + c, g = (i*K + k)*S + s).
 * records: NULL or [n * n_requests] x {e2e u32, ff u32}
 * hists:   NULL or [n * ORC_NHIST * ORC_NBINS] u32 (e2e, ff, interactive e2e)
 * series:  NULL or [series_slots * series_windows * n_inst] (indexed by r / stride)
 * trace:   NULL or [trace_cap] for replica trace_id; *trace_n receives the count
 * cell_series: NULL or [n_cells * series_windows * n_inst * 8] u64, zeroed by the caller: per cell, window
 *   and instance {sum integral Q, sum busy, replicas that closed the window, sum max Q, sum B, replicas
 *   whose in-link was BATCH / FUNCTION / TOKEN} over the simulated replicas (M15 cell-summed series)
 * Returns 0 on success, <0 on invalid input. */
int orc_simulate(const orc_pipeline* p, const orc_grid* g, const uint64_t* ids, uint64_t n,
                 uint32_t threads, orc_summary* out, uint32_t* records, uint32_t* hists,
                 orc_series* series, uint64_t trace_id, orc_trace* trace, uint64_t trace_cap,
                 uint64_t* trace_n, uint64_t* cell_series);

/* Cell merge over a full grid (cells indexed (i*K + k)*C + c): cnt [n_cells * ORC_NCNT] i64,
 * hist [n_cells * ORC_NHIST * ORC_NBINS] i64.  summaries/hists indexed by global replica id. */
#define ORC_NCNT 28
#define ORC_NHIST 3
void orc_cells(const orc_grid* g, const orc_summary* sums, const uint32_t* hists, int64_t* cnt,
               int64_t* hist);
/* Per-group argmin (M20): best[g] = winning candidate c; per-row argmin over pooled cells. */
void orc_argmin_groups(const orc_grid* g, const orc_summary* sums, uint32_t objective,
                       uint64_t obj_slo, int32_t* best);
/* M18 on a pooled histogram [ORC_NBINS]: lower edge of the nearest-rank num-th percentile's bin */
uint64_t orc_pooled_pct(const int64_t* hist, uint32_t num);
void orc_argmin_rows(const orc_grid* g, const int64_t* cnt, const int64_t* hist,
                     uint32_t objective, uint64_t obj_slo, int32_t* best);

#ifdef __cplusplus
}
#endif
#endif
