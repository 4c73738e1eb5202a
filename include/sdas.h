/* include/sdas.h -- C-ABI of the B200-native SDAS strategy simulator.
 *
 * What it computes: a batched Monte-Carlo discrete-event simulation of agent
 * pipelines (e.g. developer -> tester, Fig. 1) whose inter-agent
 * message granularity is batching / function-by-function pipelining /
 * token-level streaming, optionally switched per window by a
 * metrics-driven controller, swept over
 * candidates x request rates x profiles x seeds, with exact per-replica
 * p50/p99 end-to-end and first-feedback latency, throughput, queue-length
 * series and an argmin over candidates.  The model rules M0-M20 are stated in
 * DESIGN.md §"Model" (SURVEY.md §8(c) readings).
 *
 * Conventions (all entry points):
 *  - Every quantity is an integer; 1 tick = 1 microsecond (rule M0).
 *  - Status codes are returned, never thrown; sdas_last_error() holds a
 *    thread-local message naming the offending field (valid until the next
 *    sdas_* call on the same thread).
 *  - The library NEVER allocates device memory.  The caller (PyTorch in the
 *    Python binding) allocates every buffer named in sdas_buffers with the byte
 *    sizes returned by sdas_results_layout(), 256-byte aligned.
 *  - Launches are asynchronous on `stream` (a cudaStream_t passed as void*).
 *  - Descriptors are deep-copied by sdas_pipeline_create; grid pointers are read
 *    only during the call.
 */
#ifndef SDAS_H
#define SDAS_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t sdas_status;
#define SDAS_OK 0
#define SDAS_E_INVALID_ARG -1   /* null pointer, bad enum, zero-length axis */
#define SDAS_E_INVALID_FIELD -2 /* descriptor invariant violated (SPEC.md:53 InvalidField); message names it */
#define SDAS_E_UNKNOWN_PARAM -3 /* set/reset on an unregistered knob (Table 1) */
#define SDAS_E_OUT_OF_RANGE -4  /* set value outside the knob's range (e.g. max_num_seqs 0) */
#define SDAS_E_BUFFER -5        /* a required buffer is NULL or misaligned */
#define SDAS_E_CUDA -6          /* CUDA launch / runtime error; message carries cudaGetErrorString */
#define SDAS_E_STATE -7         /* call order violated (e.g. sdas_metrics GROUP scope before control_sweep) */
#define SDAS_E_LIMIT -8         /* exceeds an implementation limit (shared-memory budget, instance count) */

const char* sdas_last_error(void);
const char* sdas_version(void);

/* ---- enums ---------------------------------------------------------------------- */
enum { SDAS_BATCH = 0, SDAS_FUNCTION = 1, SDAS_TOKEN = 2 };            /* PAPER.md:17 (a)(b)(c) */
enum { SDAS_ROUTE_JSQ = 0, SDAS_ROUTE_RR = 1, SDAS_ROUTE_FIXED = 2, SDAS_ROUTE_SELECT = 3,
       SDAS_ROUTE_NONE = 255 };
enum { SDAS_SVC_DET = 0, SDAS_SVC_EXP = 1 };
enum { SDAS_POISSON = 0, SDAS_MMPP2 = 1, SDAS_DET = 2, SDAS_LIST = 3 };  /* PAPER.md:38 "varying load" */
enum { SDAS_STATIC = 0, SDAS_ADAPTIVE = 1 };
enum { SDAS_KV_OFF = 0, SDAS_KV_AFFINITY = 1, SDAS_KV_RECOMPUTE = 2, SDAS_KV_POSTHOC = 3,
       SDAS_KV_HINT = 4 };                                              /* PAPER.md:284-290 (Fig. 6) */
enum { SDAS_METRIC_BUSY = 0, SDAS_METRIC_LOAD = 1 };
enum { SDAS_REPLICA_OK = 0, SDAS_REPLICA_OVERFLOW = 1, SDAS_REPLICA_TRUNCATED = 2 };
enum { SDAS_MIN_P99_E2E = 0, SDAS_MIN_P50_E2E = 1, SDAS_MIN_P99_FF = 2, SDAS_MAX_THROUGHPUT = 3,
       SDAS_MAX_GOODPUT = 4, SDAS_MAX_LARGE_FRAC_UNDER_SLO = 5,
       SDAS_MIN_P90_E2E = 6,                                                 /* f3: exact p90 */
       SDAS_MIN_P99_E2E_INTERACTIVE = 7 };                                   /* f2: M29 */
enum { SDAS_SCOPE_REPLICA = 0, SDAS_SCOPE_CELL = 1, SDAS_SCOPE_GROUP = 2, SDAS_SCOPE_ROW = 3 };

#define SDAS_FLAG_RECORDS 1u /* write per-request (e2e, ff) records to buffers.records */
#define SDAS_FLAG_SERIES 2u  /* write per-window queue-length series for sampled replicas */
#define SDAS_FLAG_TRACE 4u   /* write the event trace of grid.trace_replica (debug) */
#define SDAS_FLAG_STEPWISE 8u /* simulate every DECODE step as its own event (no silent-run coalescing,
                                 DESIGN.md §5); results are identical either way -- A/B and debugging */
#define SDAS_FLAG_GENERIC 16u /* never launch a specialised K1; results are identical
                                 either way -- A/B and parity tests */
#define SDAS_FLAG_MID 32u     /* at most the level-1 specialisation (A/B and parity tests) */
#define SDAS_FLAG_CELL_SERIES 128u /* accumulate the cell-summed window series (M15) into buffers.cell_series */
#define SDAS_FLAG_SPILL 64u   /* force the smallest shared-memory ring size (32 entries) on specialised
                                 K1 levels, so rings spill to their global extension;
                                 results are identical either way -- parity tests */

/* implementation limits (DESIGN.md §"Limits") */
#define SDAS_MAX_ROLES 8
#define SDAS_MAX_INSTANCES 8
#define SDAS_MAX_LINKS 7
#define SDAS_MAX_OUT 2       /* out-links per role (fan-out) */
#define SDAS_MAX_BATCH 32    /* max_num_seqs upper bound: one lane per sequence */
#define SDAS_MAX_REQUESTS 65535
#define SDAS_NBINS 464       /* rule M17: log-linear bins over u32 latencies */
#define SDAS_NCNT 28         /* int64 counters per cell */
#define SDAS_NHIST 3         /* histograms per cell: e2e, first feedback, interactive e2e (M29) */
#define SDAS_SUMMARY_BYTES 176

/* ---- pipeline description ---------- */
typedef struct {           /* per-message and per-token service model of one agent instance */
  uint32_t h_msg;          /* receive overhead per message (SPEC.md:203 h_rx, charged at the receiver) */
  uint32_t alpha, beta;    /* RECV(m) = h_msg + beta*m.tokens + alpha*[m opens an item]  (rule M7) */
  uint32_t tau0, gamma;    /* DECODE step = tau0 + gamma*b for batch size b            (rule M7) */
  uint32_t large;          /* 1 = LARGE model profile (model selection) */
} sdas_cost;

typedef struct {
  uint32_t n_instances;       /* 1..SDAS_MAX_INSTANCES in total over all roles */
  sdas_cost cost;             /* default cost of every instance */
  const sdas_cost* inst_cost; /* NULL, or [n_instances] per-instance overrides (copied) */
  uint32_t max_num_seqs;      /* default B, 1..32; knob "agent:<role>/max_num_seqs" */
  uint32_t out_fixed, out_num, out_den; /* non-source item output = out_fixed + n_in*out_num/out_den (M8) */
  uint32_t n_functions;       /* F: FUNCTION segments of this role's outputs (M8) */
  uint32_t svc;               /* SDAS_SVC_DET | SDAS_SVC_EXP (alpha ~ Exp(mean alpha) per item) */
  uint32_t route;             /* routing INTO this role when n_instances > 1 (M11) */
  uint32_t route_fixed;       /* instance for SDAS_ROUTE_FIXED */
  uint32_t inbox_cap;         /* delivered-not-started messages per instance (M14) */
  uint32_t flight_cap;        /* emitted-not-delivered messages addressed to an instance (M14) */
  uint32_t wait_cap;          /* items waiting for batch admission per instance (M14) */
} sdas_role_desc;

typedef struct {
  uint32_t src_role, dst_role; /* src < dst (DAG in topological order); role 0 is the only source */
  uint32_t net_delay;          /* >= 1 tick; delivery = emit + net_delay */
  uint32_t chunk_tokens;       /* >= 1; TOKEN(c) chunk; knob "link:<s>-><d>/chunk_tokens" */
  uint32_t mode;               /* default granularity; knob "link:<s>-><d>/comm_mode" */
  uint32_t pacing_gap;         /* M30 (f4): 0..2^18 ticks between consecutive dispatches on this link
                                  (PAPER.md:261); knob "link:<s>-><d>/pacing_gap";
                                  pacing_gap * the destination's flight_cap must stay below 2^30 */
} sdas_link_desc;

typedef struct {
  uint32_t n_roles; const sdas_role_desc* roles;   /* role 0 = the source */
  uint32_t n_links; const sdas_link_desc* links;   /* every non-source role has exactly one in-link */
  uint32_t feedback_role;                           /* first-feedback is measured here (M13) */
  uint32_t request_cap;                             /* R_cap: admitted-not-completed requests (M14) */
  uint64_t window_ticks;                            /* metrics/control window W (M15), 1..2^31-1 */
  uint64_t slo_ticks;                               /* "good" completions: e2e <= slo (M19) */
  /* f1 -- KV-cache transfer, controller hints and load balancing (rules M21-M24).
   * kv_role 0 disables KV modelling; otherwise every request's context (kv_ctx_tokens tokens) lives on
   * one instance of kv_role (its "home": instance 0 with probability kv_home_skew/1000, else uniform).
   * An opening message routed away from home pays, at its RECV, beta*ctx (RECOMPUTE), kv_tau_xfer*ctx
   * (POSTHOC transfer on arrival) or the part of a transfer started at routing time that is still
   * running (HINT), per the candidate's kv_policy. */
  uint32_t kv_role, kv_ctx_tokens, kv_tau_xfer, kv_home_skew;
} sdas_pipeline_desc;

typedef struct sdas_pipeline sdas_pipeline;

/* Deep-copies and validates `desc`.  Errors: SDAS_E_INVALID_ARG (NULL), SDAS_E_INVALID_FIELD
 * (message names the field), SDAS_E_LIMIT.  On success *out owns a pipeline (sdas_pipeline_destroy). */
sdas_status sdas_pipeline_create(const sdas_pipeline_desc* desc, sdas_pipeline** out);
void sdas_pipeline_destroy(sdas_pipeline* p); /* NULL-safe */

/* Table 1: set(parameter, value) / reset(parameter) on the pipeline's
 * knob registry ("each agent exposes ... knobs").  Knobs (SPEC.md:209, 498 addressing):
 *   "agent:<role>/max_num_seqs"      1..32      (default: desc value)
 *   "agent:<role>/n_functions"       1..255
 *   "link:<src>-><dst>/comm_mode"    0..2       (SDAS_BATCH/FUNCTION/TOKEN)
 *   "link:<src>-><dst>/chunk_tokens" 1..65535
 *   "link:<src>-><dst>/net_delay"    1..2^31-1
 *   "link:<src>-><dst>/pacing_gap"   0..2^18    (M30, f4)
 * Values set here are the initial knob values of every replica; reset restores the value given
 * at sdas_pipeline_create (idempotent).  Errors: SDAS_E_UNKNOWN_PARAM, SDAS_E_OUT_OF_RANGE. */
sdas_status sdas_set(sdas_pipeline* p, const char* knob, int64_t value);
sdas_status sdas_reset(sdas_pipeline* p, const char* knob);
sdas_status sdas_get(const sdas_pipeline* p, const char* knob, int64_t* value);

/* ---- sweep grid ------------------------------------------------------------------- */
typedef struct {
  uint32_t kind;              /* STATIC | ADAPTIVE workload policy (M16) */
  uint8_t mode[8];            /* per link: static mode / adaptive initial mode; 255 = pipeline knob */
  uint32_t ctl_links;         /* ADAPTIVE: bitmask of links whose comm_mode the controller drives */
  uint32_t metric;            /* SDAS_METRIC_BUSY | SDAS_METRIC_LOAD of the link's destination role */
  uint32_t lo_permille, hi_permille, dwell_windows; /* three-band thresholds and dwell D (M16(i)) */
  uint8_t band_mode[4];       /* modes for the low / mid / high band ([3] unused) */
  uint32_t route_override;    /* SDAS_ROUTE_NONE, or JSQ/RR for every JSQ/RR role (M11) */
  uint32_t batch_roles;       /* bitmask of roles with SLO-aware max_num_seqs control (M16(ii)) */
  uint32_t q_hi;              /* M16(ii): grow B when the window's integral Q > q_hi * W */
  int32_t select_role;        /* -1, or the SELECT role driven by model selection (M16(iii)) */
  uint32_t kv_policy;         /* SDAS_KV_*: routing / KV handling into kv_role (M21-M24) */
  uint32_t guard_links;       /* M25 constraint guard (f3): links set to BATCH while fewer than
                                 ceil(guard_pct * n / 100) of a window's n >= 1 completions met
                                 policy_slo_ticks, else reset to their initial mode (needs ADAPTIVE) */
  uint32_t guard_pct;         /* 0..100: the guarded end-to-end quantile (90 = p90) */
  uint32_t prio;              /* M27 (f2): 1 = every inbox and decode-wait queue serves interactive
                                 requests first (FIFO within a class); 0 = FIFO over both classes */
  uint32_t admit;             /* M28 (f2): 1 = admission gate (agent-level rule "admit only high-priority
                                 requests under load"), needs ADAPTIVE */
  uint32_t admit_lo_permille, admit_hi_permille; /* gate opens at <= lo, interactive-only at >= hi */
  uint32_t pacing_gap;        /* M30 (f4): 0xFFFFFFFF = every link's own pacing_gap knob; else this gap
                                 (0..2^18 ticks) on every link */
  uint32_t stale_jsq;         /* M31 (f4): 1 = JSQ routing ranks the per-instance loads polled at the last
                                 window close (the controller's state-store snapshot, SPEC.md:469 route()
                                 on the latest Snapshot) instead of the live loads; 0 = live JSQ (M11) */
  uint64_t policy_slo_ticks;  /* SLO used by the controller's window p99 test */
} sdas_candidate;

typedef struct {
  uint32_t kind;              /* SDAS_POISSON | MMPP2 | DET | LIST */
  uint64_t mean_gap[2];       /* ticks; [1] = high-rate state of MMPP2; gap*2977044472 < 2^64 */
  uint64_t mean_sojourn[2];   /* MMPP2 epoch means (low, high) */
  const uint64_t* list;       /* LIST: nondecreasing arrival ticks, list_len >= n_requests */
  uint32_t list_len;
  uint32_t prompt_lo, prompt_hi, out_lo, out_hi; /* P ~ U[lo,hi], O ~ U[lo,hi] (M5), <= 65535 */
  uint32_t interactive_permille; /* M26 (f2): share of interactive requests, 0..1000 (0 = one class) */
} sdas_arrival_desc;

typedef struct {
  uint32_t n_candidates; const sdas_candidate* cand;          /* axis c */
  uint32_t n_rates, n_profiles; const sdas_arrival_desc* arrivals; /* [n_rates * n_profiles], axes i, k */
  uint32_t n_seeds, seed_offset; uint64_t master_seed;         /* axis s; Philox key (M2) */
  uint32_t n_requests;                                         /* N per replica, 1..65535 */
  uint64_t max_ticks;                                          /* 0 = none; else TRUNCATED beyond */
  uint32_t flags;                                              /* SDAS_FLAG_* */
  uint32_t series_stride, series_slots, series_windows;        /* replicas r = m*stride, m < slots */
  uint64_t group_begin, group_end;   /* global group range [begin, end) of this call; end 0 = all */
  uint32_t rank, world;              /* group-interleaved partition: group g runs on rank g % world */
  uint64_t trace_replica; uint32_t trace_cap;                  /* SDAS_FLAG_TRACE */
} sdas_grid;
/* Replica id r = g*C + c with group g = (i*K + k)*S + s (rule M1).  The replicas of this call are
 * the groups g in [group_begin, group_end) with g % world == rank, all C candidates of each; local
 * replica x = lg*C + c for the lg-th such group. */

typedef struct {
  uint64_t params_bytes;     /* device: packed descriptors (written by the library) */
  uint64_t work_bytes;       /* device: scratch (replica counter + per-warp record scratch) */
  uint64_t summary_bytes;    /* device: n_local_replicas x 176-byte summary records, little-endian u32 words:
                                0 status, 1 admitted, 2 dropped, 3 completed, 4-5 makespan (or overflow tick),
                                6-7 sum e2e, 8-9 sum ff, 10-11 integral N_sys dt, 12-15 p50/p99 e2e, p50/p99 ff,
                                16 bins of p50/p99 e2e (u16 pair), 17 exact p90 e2e (f3), 18 max e2e, 19 saturated records, 20 arrivals,
                                21 deliveries, 22 RECV steps, 23 DECODE steps, 24 window closes, 25 mode
                                switches, 26 good, 27 large-model items, 28-29 output tokens, 30 max_num_seqs
                                changes (M16(ii)), 31 KV transfers (M24); f2 (M29): 32 interactive
                                completions, 33 rejected by the admission gate, 34-35 sum interactive e2e,
                                36-37 exact p50/p99 interactive e2e, 38 interactive good, 39 gate changes;
                                40 model-selection changes (M16(iii)), 41 bins of p50/p99 ff (u16 pair),
                                42-43 reserved (0).  Sums are exact u64; latencies saturate at 2^32-1 */
  uint64_t records_bytes;    /* device: n_local_replicas x n_requests x {u32 e2e, u32 ff} (FLAG_RECORDS) */
  uint64_t series_bytes;     /* device: series_slots x series_windows x n_instances x 16 B (FLAG_SERIES);
                                zeroed by sdas_simulate: windows a replica never reaches (it ended or
                                overflowed first) read as 0 */
  uint64_t cell_cnt_bytes;   /* device: n_cells x SDAS_NCNT int64 (zeroed by the caller; accumulated) */
  uint64_t cell_hist_bytes;  /* device: n_cells x SDAS_NHIST x SDAS_NBINS int32 (zeroed by the caller) */
  uint64_t best_group_bytes; /* device: n_local_groups int32 (control_sweep) */
  uint64_t best_row_bytes;   /* device: n_rows int32 (finalize) */
  uint64_t trace_bytes;      /* device: 8 + trace_cap x 24 B (FLAG_TRACE) */
  uint64_t n_local_replicas, n_local_groups, n_groups, n_cells, n_rows, n_replicas;
  uint32_t n_instances, smem_per_replica, warps_per_block, blocks_per_sm;
  uint64_t resident_replicas;
  uint32_t k1_variant;       /* K1 specialisation level running this grid: 0 generic,
                                1 no KV / pacing / classes / LOAD metric / max_ticks / STEPWISE,
                                2 LEAN (+ single instances, no fan-out) */
  uint32_t ring_s;           /* shared-memory ring size bound; 0xFFFFFFFF = rings whole */
  uint64_t cell_series_bytes; /* device: SDAS_FLAG_CELL_SERIES buffer (see sdas_buffers.cell_series) */
} sdas_layout;

typedef struct {
  void *params, *work, *summary, *records, *series, *cell_cnt, *cell_hist, *best_group, *best_row, *trace;
  void* cell_series;         /* SDAS_FLAG_CELL_SERIES: n_cells x series_windows x n_instances x 8 u64 (zeroed by
                                the caller; accumulated): per cell, window w < series_windows and instance
                                {sum integral Q dt, sum busy ticks, replicas that closed window w, sum max Q,
                                sum max_num_seqs, replicas whose in-link was BATCH, FUNCTION, TOKEN}
                                (M15 "plus cell-summed series", PAPER.md:231-238 aggregation); every window a
                                replica closed counts, also before a later overflow (DESIGN.md R-CSER) */
} sdas_buffers;

/* Sizes of every buffer for (p, grid) on the current device (queries the occupancy). */
sdas_status sdas_results_layout(const sdas_pipeline* p, const sdas_grid* grid, sdas_layout* out);

/* Simulate every local replica (K1, one replica per warp) and merge its histograms and counters
 * into the cell buffers (integer atomics).  Writes summaries (+ records / series / trace per
 * flags).  Required buffers: params, work, summary, cell_cnt, cell_hist.  Asynchronous. */
sdas_status sdas_simulate(const sdas_pipeline* p, const sdas_grid* grid, const sdas_buffers* dev, void* stream);

/* sdas_simulate + the per-group argmin over candidates (K3) for `objective` (rule M20).
 * Also requires best_group.  objective_slo is the SLO of SDAS_MAX_LARGE_FRAC_UNDER_SLO. */
sdas_status sdas_control_sweep(const sdas_pipeline* p, const sdas_grid* grid, uint32_t objective,
                               uint64_t objective_slo, const sdas_buffers* dev, void* stream);

/* K3 alone: per-group argmin for `objective` over summaries already written by sdas_simulate /
 * sdas_control_sweep with the same grid (re-rank candidates under another objective without
 * re-simulating).  Requires params, summary, best_group. */
sdas_status sdas_group_argmin(const sdas_pipeline* p, const sdas_grid* grid, uint32_t objective,
                              uint64_t objective_slo, const sdas_buffers* dev, void* stream);

/* Per-row (i, k) argmin over pooled cells (after the caller's all_reduce of the cell buffers). */
sdas_status sdas_finalize(const sdas_pipeline* p, const sdas_grid* grid, uint32_t objective,
                          uint64_t objective_slo, const sdas_buffers* dev, void* stream);

/* ---- metrics queries on HOST copies of the buffers (PAPER.md:231-238 metrics plane) ---- */
typedef struct {
  uint32_t status;
  uint64_t n_replicas, admitted, dropped, completed;
  uint32_t p50_e2e, p99_e2e, p50_ff, p99_ff;      /* exact (REPLICA) or bin lower edge (CELL/ROW) */
  uint32_t bin_p50_e2e, bin_p99_e2e, bin_p50_ff, bin_p99_ff;
  uint32_t p90_e2e, pad0;                         /* exact (REPLICA) or bin lower edge (CELL) p90 e2e */
  double mean_e2e, mean_ff;                       /* (double)sum / (double)n  (M19) */
  double throughput, goodput;                     /* completed*1e6/makespan, good*1e6/makespan (req/s) */
  uint64_t makespan, sum_e2e, sum_ff, int_nsys, good, large_items;
  uint64_t arrivals, deliveries, recv_steps, decode_steps, window_closes, mode_switches, tokens;
  uint64_t message_events, des_events;            /* arrivals + deliveries; + steps + window closes */
  uint64_t completed_int, rejected, sum_e2e_int, good_int;   /* f2 (M29) */
  uint32_t p50_e2e_int, p99_e2e_int;              /* exact (REPLICA) or bin lower edge (CELL) */
  int32_t best;                                   /* GROUP / ROW scope: winning candidate */
  const uint8_t* series;                          /* REPLICA scope with FLAG_SERIES: 16 B records */
  uint64_t series_len;                            /* windows x instances */
} sdas_metrics_out;

/* ---- f3: intent compilation ("declarative ... goals", 188 "compile these into concrete
 * policy rules", 220 intent-driven control; SPEC.md:432-436 Intent, 475-483 compile_intent) ----
 * An intent is an objective and/or explicit rules plus latency constraints.  It compiles, on the host,
 * into one M16/M25 policy vector (sdas_candidate) -- the unit the sweep evaluates -- and the M20
 * objective its sweep should rank by.  Templates (DESIGN.md §2 M25 and readings):
 *   MAX_THROUGHPUT : ADAPTIVE three-band comm_mode on every link, BUSY metric of the destination,
 *                    lo 400 / hi 800 permille, bands TOKEN / FUNCTION / BATCH, dwell = ceil(1 s / W)
 *                    windows; objective SDAS_MAX_THROUGHPUT.
 *   MIN_P90_LATENCY: TOKEN on every link (chunk = the link's chunk_tokens knob); objective
 *                    SDAS_MIN_P90_E2E.
 *   each constraint: a guard (M25) on its scope links with guard_pct = its quantile and
 *                    policy_slo_ticks = its bound; makes the policy ADAPTIVE.
 *   rules          : an explicit policy vector, passed through unchanged; an objective template then
 *                    overwrites only the mode fields (modes, kind, ctl_links, metric, lo/hi, bands,
 *                    dwell); with no objective the sweep objective is SDAS_MIN_P99_E2E.
 * Errors: SDAS_E_INVALID_ARG (NULL, bad enum, or InvalidIntent: no objective and no rules),
 * SDAS_E_LIMIT (constraints with different (metric, bound), or a bound that conflicts with the rules'
 * own policy_slo_ticks: one latency bound per compiled policy). */
enum { SDAS_INTENT_NONE = 0, SDAS_INTENT_MAX_THROUGHPUT = 1, SDAS_INTENT_MIN_P90_LATENCY = 2 };
enum { SDAS_CONSTRAINT_E2E_P90 = 0, SDAS_CONSTRAINT_E2E_P99 = 1 };
typedef struct {
  uint32_t metric;            /* SDAS_CONSTRAINT_*: a window quantile of end-to-end latency */
  uint32_t scope_links;       /* bitmask of links flipped to BATCH while violated; 0 = every link */
  uint64_t bound_ticks;       /* constraint: metric <= bound */
} sdas_constraint;
typedef struct {
  uint32_t objective;                         /* SDAS_INTENT_* */
  uint32_t n_constraints;
  const sdas_constraint* constraints;
  const sdas_candidate* rules;                /* optional explicit policy vector (NULL = none) */
} sdas_intent;
sdas_status sdas_compile_intent(const sdas_pipeline* p, const sdas_intent* intent, sdas_candidate* out,
                                uint32_t* objective_out);

/* host: host copies of the device buffers (only those the scope needs, same layout).
 * REPLICA: index = local replica; CELL: index = cell (i*K + k)*C + c; GROUP: local group;
 * ROW: index = (i*K + k).  Errors: SDAS_E_INVALID_ARG, SDAS_E_STATE (missing buffer). */
sdas_status sdas_metrics(const sdas_pipeline* p, const sdas_grid* grid, const sdas_buffers* host,
                         uint32_t scope, uint64_t index, sdas_metrics_out* out);

#ifdef __cplusplus
}
#endif
#endif /* SDAS_H */
