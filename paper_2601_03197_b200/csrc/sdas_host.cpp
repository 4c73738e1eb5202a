// sdas_host.cpp -- host side of libsdas: the C-ABI of include/sdas.h.
//
// Validation (SPEC.md:53 InvalidField conventions), the Table-1 knob registry (PAPER.md:196-217:
// set/reset, "each agent exposes ... knobs"), grid partitioning (group-interleaved over ranks,
// DESIGN.md §"Multi-GPU"), shared-memory layout planning for K1, packing of the device parameter
// block, launches on the caller's stream, and metric queries on host copies.
// No device memory is allocated here: the caller (PyTorch) owns every buffer.

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "sdas_internal.h"

using namespace sdas;

namespace {

thread_local std::string g_err;

sdas_status fail(sdas_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
sdas_status ok() {
  g_err.clear();
  return SDAS_OK;
}

// Q32 log2 table T[i] = round(2^32 log2(1 + i/256)) (rule M3), evaluated here through log1p.
struct Log2Tab {
  uint64_t t[257];
  Log2Tab() {
    const long double inv_ln2 = 1.0L / logl(2.0L);
    for (int i = 0; i <= 256; ++i) t[i] = (uint64_t)llroundl(ldexpl(log1pl((long double)i / 256.0L) * inv_ln2, 32));
  }
};
const Log2Tab& log2tab() {
  static Log2Tab T;
  return T;
}

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

}  // namespace

struct sdas_pipeline {
  std::vector<sdas_role_desc> roles;
  std::vector<std::vector<sdas_cost>> inst_cost;
  std::vector<sdas_link_desc> links;
  uint32_t feedback_role = 0, request_cap = 0;
  uint64_t window = 0, slo = 0;
  uint32_t kv_role = 0, kv_ctx = 0, kv_tau = 0, kv_skew = 0;   // f1 (M21-M24)
  // knob registry: current values and registered defaults (Table 1)
  std::vector<uint32_t> B_cur, B_def, F_cur, F_def;
  std::vector<uint32_t> mode_cur, mode_def, chunk_cur, chunk_def, net_cur, net_def, pace_cur, pace_def;
  uint32_t n_inst = 0;
};

namespace {

// Largest value EXP(M; x) can return (x = 0, rule M3): floor(M * round(2^32 ln 2) * 32 / 2^32) <= 22.19 M.
uint64_t exp_max(uint64_t M) { return (uint64_t)(((unsigned __int128)M * 2977044472ull * 32u) >> 32) + 1; }

sdas_status validate_desc(const sdas_pipeline_desc* d) {
  if (!d) return fail(SDAS_E_INVALID_ARG, "desc is NULL");
  if (d->n_roles == 0 || !d->roles) return fail(SDAS_E_INVALID_FIELD, "n_roles: at least one role required");
  if (d->n_roles > SDAS_MAX_ROLES) return fail(SDAS_E_LIMIT, "n_roles: at most %d", SDAS_MAX_ROLES);
  if (d->n_links > SDAS_MAX_LINKS) return fail(SDAS_E_LIMIT, "n_links: at most %d", SDAS_MAX_LINKS);
  if (d->n_links && !d->links) return fail(SDAS_E_INVALID_FIELD, "links: NULL with n_links > 0");
  if (d->feedback_role >= d->n_roles) return fail(SDAS_E_INVALID_FIELD, "feedback_role: out of range");
  if (d->request_cap < 1 || d->request_cap > 4096)
    return fail(SDAS_E_INVALID_FIELD, "request_cap: must be in 1..4096");
  if (d->kv_role >= d->n_roles) return fail(SDAS_E_INVALID_FIELD, "kv_role: must be 0 (off) or a non-source role");
  if (d->kv_home_skew > 1000) return fail(SDAS_E_INVALID_FIELD, "kv_home_skew: permille in 0..1000");
  if (d->kv_role && ((uint64_t)d->kv_ctx_tokens * d->kv_tau_xfer >= (1ull << 30) ||
                     (uint64_t)d->kv_ctx_tokens * (1u << 15) >= (1ull << 40)))
    return fail(SDAS_E_INVALID_FIELD, "kv_ctx_tokens/kv_tau_xfer: transfer must stay below 2^30 ticks");
  if (d->window_ticks < 1 || d->window_ticks >= (1ull << 31))
    return fail(SDAS_E_INVALID_FIELD, "window_ticks: must be in 1..2^31-1");
  uint32_t n_inst = 0;
  for (uint32_t r = 0; r < d->n_roles; ++r) {
    const sdas_role_desc& R = d->roles[r];
    if (R.n_instances < 1) return fail(SDAS_E_INVALID_FIELD, "roles[%u].n_instances: must be >= 1", r);
    n_inst += R.n_instances;
    if (R.max_num_seqs < 1 || R.max_num_seqs > SDAS_MAX_BATCH)
      return fail(SDAS_E_INVALID_FIELD, "roles[%u].max_num_seqs: must be in 1..32", r);
    if (R.out_den < 1) return fail(SDAS_E_INVALID_FIELD, "roles[%u].out_den: must be >= 1", r);
    if (R.n_functions < 1 || R.n_functions > 255)
      return fail(SDAS_E_INVALID_FIELD, "roles[%u].n_functions: must be in 1..255", r);
    if (R.svc > SDAS_SVC_EXP) return fail(SDAS_E_INVALID_FIELD, "roles[%u].svc: bad enum", r);
    if (R.route > SDAS_ROUTE_SELECT) return fail(SDAS_E_INVALID_FIELD, "roles[%u].route: bad enum", r);
    if (R.route == SDAS_ROUTE_FIXED && R.route_fixed >= R.n_instances)
      return fail(SDAS_E_INVALID_FIELD, "roles[%u].route_fixed: out of range", r);
    if (R.inbox_cap < 1 || R.inbox_cap > 65535 || R.wait_cap < 1 || R.wait_cap > 65535 || R.flight_cap > 65535 ||
        (r > 0 && R.flight_cap < 1))
      return fail(SDAS_E_INVALID_FIELD, "roles[%u].caps: inbox/wait in 1..65535, flight in 1..65535", r);
    const sdas_cost* cs = R.inst_cost;
    for (uint32_t x = 0; x < R.n_instances; ++x) {
      const sdas_cost& c = cs ? cs[x] : R.cost;
      if (c.h_msg >= (1u << 31) || c.alpha >= (1u << 31) || c.beta >= (1u << 15) || c.tau0 >= (1u << 31) ||
          c.gamma >= (1u << 25))
        return fail(SDAS_E_INVALID_FIELD, "roles[%u].cost: step costs must stay below 2^31 ticks", r);
      // worst-case step costs (K1 keeps every pending tick < 2^31 ahead): RECV of a 65535-token
      // message with the largest EXP draw (M3 tail) and the largest KV penalty (M23); DECODE of 32 sequences
      const uint64_t a_max = R.svc == SDAS_SVC_EXP ? exp_max(c.alpha) : c.alpha;
      uint64_t pen = 0;
      if (d->kv_role && r == d->kv_role)
        pen = std::max<uint64_t>((uint64_t)c.beta * d->kv_ctx_tokens, (uint64_t)d->kv_tau_xfer * d->kv_ctx_tokens);
      if ((uint64_t)c.h_msg + (uint64_t)c.beta * 65535u + a_max + pen >= (1ull << 31))
        return fail(SDAS_E_INVALID_FIELD, "roles[%u].cost: worst-case RECV (h + 65535 beta + max alpha draw + KV "
                                          "penalty) must stay below 2^31 ticks", r);
      if ((uint64_t)c.tau0 + (uint64_t)c.gamma * SDAS_MAX_BATCH >= (1ull << 31))
        return fail(SDAS_E_INVALID_FIELD, "roles[%u].cost: tau0 + 32 gamma must stay below 2^31 ticks", r);
    }
  }
  if (n_inst > SDAS_MAX_INSTANCES) return fail(SDAS_E_LIMIT, "instances: at most %d in total", SDAS_MAX_INSTANCES);
  std::vector<int> indeg(d->n_roles, 0), outdeg(d->n_roles, 0);
  for (uint32_t l = 0; l < d->n_links; ++l) {
    const sdas_link_desc& L = d->links[l];
    if (L.dst_role >= d->n_roles || L.src_role >= L.dst_role)
      return fail(SDAS_E_INVALID_FIELD, "links[%u]: need src_role < dst_role < n_roles", l);
    if (L.net_delay < 1 || L.net_delay >= (1u << 31))
      return fail(SDAS_E_INVALID_FIELD, "links[%u].net_delay: must be in 1..2^31-1", l);
    if (L.chunk_tokens < 1 || L.chunk_tokens > 65535)
      return fail(SDAS_E_INVALID_FIELD, "links[%u].chunk_tokens: must be in 1..65535", l);
    if (L.pacing_gap > (1u << 18)) return fail(SDAS_E_INVALID_FIELD, "links[%u].pacing_gap: must be in 0..2^18", l);
    if (L.mode > SDAS_TOKEN) return fail(SDAS_E_INVALID_FIELD, "links[%u].mode: bad enum", l);
    indeg[L.dst_role]++;
    outdeg[L.src_role]++;
  }
  for (uint32_t r = 1; r < d->n_roles; ++r)
    if (indeg[r] != 1) return fail(SDAS_E_INVALID_FIELD, "roles[%u]: needs exactly one in-link (role 0 is the only source, no joins)", r);
  for (uint32_t r = 0; r < d->n_roles; ++r)
    if (outdeg[r] > SDAS_MAX_OUT) return fail(SDAS_E_LIMIT, "roles[%u]: at most %d out-links", r, SDAS_MAX_OUT);
  return SDAS_OK;
}

int parse_knob(const sdas_pipeline* p, const char* knob, int* kind, uint32_t* idx) {
  // returns 0 ok; kinds: 0 max_num_seqs, 1 n_functions, 2 comm_mode, 3 chunk_tokens, 4 net_delay,
  // 5 pacing_gap
  if (!knob) return -1;
  unsigned a = 0, b = 0;
  char name[64] = {0};
  int n = 0;
  if (sscanf(knob, "agent:%u/%63s%n", &a, name, &n) == 2 && knob[n] == 0) {
    if (a >= p->roles.size()) return -1;
    *idx = a;
    if (!strcmp(name, "max_num_seqs")) { *kind = 0; return 0; }
    if (!strcmp(name, "n_functions")) { *kind = 1; return 0; }
    return -1;
  }
  n = 0;
  if (sscanf(knob, "link:%u->%u/%63s%n", &a, &b, name, &n) == 3 && knob[n] == 0) {
    for (uint32_t l = 0; l < p->links.size(); ++l) {
      if (p->links[l].src_role == a && p->links[l].dst_role == b) {
        *idx = l;
        if (!strcmp(name, "comm_mode")) { *kind = 2; return 0; }
        if (!strcmp(name, "chunk_tokens")) { *kind = 3; return 0; }
        if (!strcmp(name, "net_delay")) { *kind = 4; return 0; }
        if (!strcmp(name, "pacing_gap")) { *kind = 5; return 0; }
        return -1;
      }
    }
  }
  return -1;
}

struct Plan {
  DParams hp;
  uint64_t n_groups = 0, n_cells = 0, n_rows = 0, n_replicas = 0;
  uint32_t wpb = 1, blocks_per_sm = 1, n_sm = 148, smem_block = 0, blocks = 0;
  uint64_t total_warps = 0;
  uint64_t blob_bytes = 0;
};

sdas_status plan(const sdas_pipeline* p, const sdas_grid* g, Plan& pl) {
  if (!p || !g) return fail(SDAS_E_INVALID_ARG, "pipeline or grid is NULL");
  if (g->n_candidates == 0 || !g->cand) return fail(SDAS_E_INVALID_ARG, "grid.n_candidates: must be >= 1");
  if (g->n_rates == 0 || g->n_profiles == 0 || !g->arrivals)
    return fail(SDAS_E_INVALID_ARG, "grid.n_rates/n_profiles: must be >= 1");
  if (g->n_seeds == 0) return fail(SDAS_E_INVALID_ARG, "grid.n_seeds: must be >= 1");
  if (g->n_requests < 1 || g->n_requests > SDAS_MAX_REQUESTS)
    return fail(SDAS_E_INVALID_FIELD, "grid.n_requests: must be in 1..65535");
  if (g->world < 1 || g->rank >= g->world) return fail(SDAS_E_INVALID_ARG, "grid.rank/world: need rank < world");
  const uint32_t nl = (uint32_t)p->links.size();
  for (uint32_t c = 0; c < g->n_candidates; ++c) {
    const sdas_candidate& cd = g->cand[c];
    if (cd.kind > SDAS_ADAPTIVE) return fail(SDAS_E_INVALID_FIELD, "cand[%u].kind: bad enum", c);
    for (uint32_t l = 0; l < nl; ++l)
      if (cd.mode[l] != 255 && cd.mode[l] > SDAS_TOKEN) return fail(SDAS_E_INVALID_FIELD, "cand[%u].mode[%u]", c, l);
    for (int b = 0; b < 3; ++b)
      if (cd.band_mode[b] > SDAS_TOKEN) return fail(SDAS_E_INVALID_FIELD, "cand[%u].band_mode[%d]", c, b);
    if (cd.ctl_links >> nl) return fail(SDAS_E_INVALID_FIELD, "cand[%u].ctl_links: unknown link", c);
    if (cd.batch_roles >> p->roles.size()) return fail(SDAS_E_INVALID_FIELD, "cand[%u].batch_roles", c);
    if (cd.select_role >= (int32_t)p->roles.size()) return fail(SDAS_E_INVALID_FIELD, "cand[%u].select_role", c);
    if (cd.route_override != SDAS_ROUTE_NONE && cd.route_override > SDAS_ROUTE_RR)
      return fail(SDAS_E_INVALID_FIELD, "cand[%u].route_override: NONE, JSQ or RR", c);
    if (cd.metric > SDAS_METRIC_LOAD || cd.lo_permille > 1000000 || cd.hi_permille > 1000000 || cd.dwell_windows > (1u << 30))
      return fail(SDAS_E_INVALID_FIELD, "cand[%u]: metric/lo/hi/dwell out of range", c);
    if (cd.prio > 1 || cd.admit > 1) return fail(SDAS_E_INVALID_FIELD, "cand[%u].prio/admit: 0 or 1", c);
    if (cd.stale_jsq > 1) return fail(SDAS_E_INVALID_FIELD, "cand[%u].stale_jsq: 0 or 1", c);
    if (cd.admit && (cd.kind != SDAS_ADAPTIVE || cd.admit_lo_permille > cd.admit_hi_permille ||
                     cd.admit_hi_permille > 65535))
      return fail(SDAS_E_INVALID_FIELD, "cand[%u].admit: needs ADAPTIVE and admit_lo <= admit_hi <= 65535", c);
  }
  const uint64_t nIK = (uint64_t)g->n_rates * g->n_profiles;
  for (uint64_t a = 0; a < nIK; ++a) {
    const sdas_arrival_desc& A = g->arrivals[a];
    if (A.kind > SDAS_LIST) return fail(SDAS_E_INVALID_FIELD, "arrivals[%llu].kind: bad enum", (unsigned long long)a);
    if (A.interactive_permille > 1000)
      return fail(SDAS_E_INVALID_FIELD, "arrivals[%llu].interactive_permille: 0..1000", (unsigned long long)a);
    if (A.interactive_permille && p->kv_role)
      return fail(SDAS_E_LIMIT, "arrivals[%llu]: request classes with KV modelling are not supported",
                  (unsigned long long)a);
    if (A.prompt_lo > A.prompt_hi || A.prompt_hi > 65535 || A.out_lo > A.out_hi || A.out_hi > 65535)
      return fail(SDAS_E_INVALID_FIELD, "arrivals[%llu]: prompt/out ranges must be lo <= hi <= 65535",
                  (unsigned long long)a);
    const uint64_t lim = UINT64_MAX / 2977044472ull;
    if (A.kind == SDAS_POISSON || A.kind == SDAS_MMPP2) {
      for (int z = 0; z < (A.kind == SDAS_MMPP2 ? 2 : 1); ++z) {
        if (A.mean_gap[z] >= lim || A.mean_gap[z] > (1ull << 35))
          return fail(SDAS_E_INVALID_FIELD, "arrivals[%llu].mean_gap: too large", (unsigned long long)a);
        if (A.kind == SDAS_MMPP2 && A.mean_sojourn[z] >= lim)
          return fail(SDAS_E_INVALID_FIELD, "arrivals[%llu].mean_sojourn: too large", (unsigned long long)a);
      }
    }
    if (A.kind == SDAS_LIST) {
      if (!A.list || A.list_len < g->n_requests)
        return fail(SDAS_E_INVALID_FIELD, "arrivals[%llu].list: need list_len >= n_requests", (unsigned long long)a);
      for (uint32_t j = 1; j < g->n_requests; ++j)
        if (A.list[j] < A.list[j - 1])
          return fail(SDAS_E_INVALID_FIELD, "arrivals[%llu].list: must be nondecreasing", (unsigned long long)a);
    }
  }
  // requests per slot index must fit u16 slots; request_cap <= 4096 validated
  DParams& h = pl.hp;
  memset(&h, 0, sizeof(h));
  h.n_roles = (uint32_t)p->roles.size();
  h.n_links = nl;
  h.n_inst = p->n_inst;
  h.feedback_role = p->feedback_role;
  h.request_cap = p->request_cap;
  h.n_requests = g->n_requests;
  h.flags = g->flags;
  h.bitmap_words = (p->request_cap + 31) / 32;
  h.C = g->n_candidates; h.I = g->n_rates; h.K = g->n_profiles; h.S = g->n_seeds;
  h.seed_offset = g->seed_offset; h.rank = g->rank; h.world = g->world;
  h.series_stride = g->series_stride; h.series_slots = g->series_slots; h.series_windows = g->series_windows;
  h.trace_cap = g->trace_cap;
  h.window = p->window; h.slo = p->slo; h.max_ticks = g->max_ticks; h.master_seed = g->master_seed;
  h.trace_replica = g->trace_replica;
  pl.n_groups = nIK * g->n_seeds;
  pl.n_rows = nIK;
  pl.n_cells = nIK * g->n_candidates;
  pl.n_replicas = pl.n_groups * g->n_candidates;
  const uint64_t gb = g->group_begin, ge = g->group_end ? std::min<uint64_t>(g->group_end, pl.n_groups) : pl.n_groups;
  if (gb > ge) return fail(SDAS_E_INVALID_ARG, "grid.group_begin > group_end");
  const uint64_t first = gb + (uint64_t)((g->rank + g->world - (gb % g->world)) % g->world);
  h.first_group = first;
  h.n_local_groups = first < ge ? (ge - first + g->world - 1) / g->world : 0;
  h.n_local_replicas = h.n_local_groups * g->n_candidates;

  // --- topology
  uint32_t inst = 0;
  for (uint32_t r = 0; r < h.n_roles; ++r) {
    const sdas_role_desc& R = p->roles[r];
    DRole& D = h.role[r];
    D.first = inst; D.n = R.n_instances; D.route = R.route; D.route_fixed = R.route_fixed;
    D.out_fixed = R.out_fixed; D.out_num = R.out_num; D.out_den = R.out_den; D.n_functions = p->F_cur[r];
    D.in_link = -1;
    D.large_inst = inst;
    D.small_inst = inst + R.n_instances - 1;
    for (uint32_t x = R.n_instances; x-- > 0;) if (p->inst_cost[r][x].large) D.large_inst = inst + x;
    for (uint32_t x = R.n_instances; x-- > 0;) if (!p->inst_cost[r][x].large) D.small_inst = inst + x;
    for (uint32_t x = 0; x < R.n_instances; ++x) {
      DInst& I = h.inst[inst + x];
      const sdas_cost& c = p->inst_cost[r][x];
      I.role = r; I.h = c.h_msg; I.alpha = c.alpha; I.beta = c.beta; I.tau0 = c.tau0; I.gamma = c.gamma;
      I.B_default = p->B_cur[r];
      I.flags = (c.large ? 1u : 0u) | (R.svc == SDAS_SVC_EXP ? 2u : 0u);
      I.inbox_cap = R.inbox_cap; I.flight_cap = r > 0 ? R.flight_cap : 0; I.wait_cap = R.wait_cap;
    }
    inst += R.n_instances;
  }
  auto rcp32 = [](uint64_t d) -> uint32_t { return d <= 1 ? 0xFFFFFFFFu : (uint32_t)((1ull << 32) / d); };
  for (uint32_t i = 0; i < h.n_inst; ++i)
    for (uint32_t b = 0; b <= SDAS_MAX_BATCH; ++b)
      h.rcp_step[i][b] = rcp32(std::max<uint64_t>(1, (uint64_t)h.inst[i].tau0 + (uint64_t)h.inst[i].gamma * b));
  for (uint32_t f = 0; f < 256; ++f) h.rcp_fn[f] = rcp32(f);
  for (uint32_t l = 0; l < nl; ++l) {
    const sdas_link_desc& L = p->links[l];
    DLink& D = h.link[l];
    D.src = L.src_role; D.dst = L.dst_role; D.net = p->net_cur[l]; D.chunk = p->chunk_cur[l]; D.mode = p->mode_cur[l];
    D.gap = p->pace_cur[l];
    DRole& S = h.role[L.src_role];
    if (S.n_out == 0) S.out_link0 = l; else S.out_link1 = l;
    S.n_out++;
    h.role[L.dst_role].in_link = (int32_t)l;
  }
  h.kv_role = p->kv_role;
  h.need_pace = 0;
  for (uint32_t l = 0; l < nl; ++l) {
    if (p->pace_cur[l] && (uint64_t)p->pace_cur[l] * p->roles[p->links[l].dst_role].flight_cap >= (1ull << 30))
      return fail(SDAS_E_INVALID_FIELD, "links[%u]: pacing_gap x flight_cap must stay below 2^30", l);
    if (p->pace_cur[l]) h.need_pace = 1;
  }
  for (uint32_t cc = 0; cc < g->n_candidates; ++cc) {
    const uint32_t pg = g->cand[cc].pacing_gap;
    if (pg == 0xFFFFFFFFu) continue;
    if (pg > (1u << 18)) return fail(SDAS_E_INVALID_FIELD, "cand[%u].pacing_gap: 0..2^18 or 0xFFFFFFFF", cc);
    for (uint32_t l = 0; l < nl && pg; ++l)
      if ((uint64_t)pg * p->roles[p->links[l].dst_role].flight_cap >= (1ull << 30))
        return fail(SDAS_E_INVALID_FIELD, "cand[%u].pacing_gap x flight_cap must stay below 2^30", cc);
    if (pg) h.need_pace = 1;
  }
  h.cls = 0;   // the CLS instantiation runs request classes (M26-M29) and the admission gate (M28)
  for (uint64_t a = 0; a < (uint64_t)g->n_rates * g->n_profiles; ++a)
    if (g->arrivals[a].interactive_permille) h.cls = 1;
  for (uint32_t cc = 0; cc < g->n_candidates; ++cc)
    if (g->cand[cc].admit) h.cls = 1;   // a gate with one class rejects every arrival while closed
  h.kv_ctx = p->kv_ctx;
  h.kv_tau = p->kv_tau;
  h.kv_skew32 = ((uint64_t)p->kv_skew << 32) / 1000;
  for (uint32_t cc = 0; cc < g->n_candidates; ++cc)
  {
    if (g->cand[cc].kv_policy > SDAS_KV_HINT) return fail(SDAS_E_INVALID_FIELD, "cand[%u].kv_policy: bad enum", cc);
    if (g->cand[cc].guard_pct > 100) return fail(SDAS_E_INVALID_FIELD, "cand[%u].guard_pct > 100", cc);
    if (g->cand[cc].guard_links >> nl) return fail(SDAS_E_INVALID_FIELD, "cand[%u].guard_links: no such link", cc);
  }
  h.need_lint = 0;
  for (uint32_t cc = 0; cc < g->n_candidates; ++cc)
    if (g->cand[cc].kind == SDAS_ADAPTIVE && g->cand[cc].metric == SDAS_METRIC_LOAD) h.need_lint = 1;
  h.max_out = 1;
  for (uint32_t r = 0; r < h.n_roles; ++r) h.max_out = std::max(h.max_out, h.role[r].n_out);
  for (uint32_t r = 0; r < h.n_roles; ++r) h.role[r].batch_words = 1 + 2 * h.max_out;
  // K1 specialisation level: 1 = no KV modelling, no pacing, no request classes, no
  // LOAD-metric integral, no max_ticks truncation, no STEPWISE flag; 2 (LEAN) =
  // level 1 + one instance per role (routing and snapshot JSQ are identities) and no fan-out
  h.lean = (g->flags & SDAS_FLAG_GENERIC) == 0 && !h.kv_role && !h.need_pace && !h.need_lint && !h.cls &&
           (h.flags & SDAS_FLAG_TRACE) == 0 && (g->flags & SDAS_FLAG_STEPWISE) == 0 && g->max_ticks == 0 ? 1u : 0u;
  bool sel = false;                          // model selection needs two instances of a role: never LEAN
  for (uint32_t cc = 0; cc < g->n_candidates; ++cc) sel = sel || g->cand[cc].select_role >= 0;
  if (h.lean && !sel && h.n_inst == h.n_roles && h.max_out == 1 && !(g->flags & SDAS_FLAG_MID)) h.lean = 2;

  // --- shared-memory layout of one warp's replica, for a shared-memory ring size bound RS (two-level rings,
  // a ring of capacity > RS keeps its oldest RS entries in shared memory, the rest in the
  // warp's extension area of `work`; levels >= 1 only -- level 0 keeps every ring whole)
  auto layout_for = [&](uint32_t RS) -> uint64_t {
    uint64_t o = 256;  // WarpHdr
    const uint32_t R = p->request_cap;
    h.off_reqA = (uint32_t)o; o += 8ull * R;
    h.off_reqFF = (uint32_t)o; o += 8ull * R;              // exact u64 first-feedback latency (M13, M19)
    h.off_reqJ = (uint32_t)o; o += 4ull * R;
    h.off_reqO = (uint32_t)o; o += 4ull * R;
    h.off_reqNit = (uint32_t)o; o += 2ull * R;
    h.off_reqOut = (uint32_t)o; o += 2ull * R;
    h.off_reqHome = (uint32_t)o; o += R;                    // u8 KV home per request slot (M21)
    h.off_reqCls = (uint32_t)o; o += h.cls ? R : 0;         // u8 class per request slot (M26)
    o = align_up(o, 16);
    h.off_bitmap = (uint32_t)o; o += 4ull * h.bitmap_words;
    if (h.lean >= 1) {                                      // levels >= 1: arrival draw queue
      o = align_up(o, 16);
      h.off_arrq = (uint32_t)o; o += 32ull * 8 + 32ull * 4;
    }
    uint64_t gx = 0;
    for (uint32_t i = 0; i < h.n_inst; ++i) {
      DInst& I = h.inst[i];
      const uint64_t pin = std::min(I.inbox_cap, RS), pfl = std::min(I.flight_cap, RS), pwt = std::min(I.wait_cap, RS);
      o = align_up(o, 16);
      I.off_inbox = (uint32_t)o; o += 8ull * pin * (h.cls ? 2 : 1);   // class-1 ring follows (M27)
      if (h.kv_role && I.role == h.kv_role) o += 4ull * pin;         // hinted-transfer ready ticks (M23)
      o = align_up(o, 16);
      I.off_ftick = (uint32_t)o; o += 4ull * pfl;
      o = align_up(o, 16);
      I.off_fbody = (uint32_t)o; o += 8ull * pfl;
      if (h.kv_role && I.role == h.kv_role) o += 4ull * pfl;         // hinted-transfer ready ticks (M23)
      o = align_up(o, 16);
      I.off_wait = (uint32_t)o; o += 4ull * pwt * (h.cls ? 2 : 1);
      o = align_up(o, 16);
      I.off_batch = (uint32_t)o; o += 4ull * 32 * h.role[I.role].batch_words;
      I.gx_inbox = (uint32_t)gx; gx = align_up(gx + 8ull * (I.inbox_cap - pin), 16);
      I.gx_ftick = (uint32_t)gx; gx = align_up(gx + 4ull * (I.flight_cap - pfl), 16);
      I.gx_fbody = (uint32_t)gx; gx = align_up(gx + 8ull * (I.flight_cap - pfl), 16);
      I.gx_wait = (uint32_t)gx; gx = align_up(gx + 4ull * (I.wait_cap - pwt), 16);
    }
    h.gx_per_warp = align_up(gx, 256);
    o = align_up(o, 16);
    h.off_scratch = 256;
    return align_up(std::max<uint64_t>(o, 256 + (uint64_t)kScratchMin), 16);
  };
  h.off_warps = (uint32_t)align_up(sizeof(DParams), 128);
  const uint64_t smem_cap = 227 * 1024;
  int n_sm = 148;
  // occupancy: warps per block maximizing resident warps per SM for a given per-warp footprint
  auto occupancy = [&](uint64_t per_warp, uint32_t rs, uint32_t& bw, uint32_t& bb) -> uint64_t {
    uint64_t best_tot = 0;
    bw = 1; bb = 0;
    for (uint32_t wpb = 1; wpb <= 8; ++wpb) {
      const uint64_t sb = h.off_warps + (uint64_t)wpb * per_warp;
      if (sb > smem_cap) break;
      int bps = 0, nsm = 0;
      if (query_occupancy(wpb, (uint32_t)sb, h.max_out, h.cls, h.lean, rs != 0xFFFFFFFFu, &bps, &nsm) == 0) {
        n_sm = nsm;
        if (bps <= 0) continue;                 // block exceeds the instantiation's launch bound
      } else {
        bps = (int)std::min<uint64_t>(32, (228 * 1024) / (sb + 1024));
        bps = std::min(bps, (int)(64 / wpb));
      }
      const uint64_t tot = (uint64_t)bps * wpb;
      if (getenv("SDAS_PLAN_DEBUG"))                   // experiments: the occupancy the planner sees
        fprintf(stderr, "plan: ring_s %u per_warp %llu wpb %u block_smem %llu -> blocks/SM %d\n", rs,
                (unsigned long long)per_warp, wpb, (unsigned long long)sb, bps);
      if (tot >= best_tot) { best_tot = tot; bw = wpb; bb = (uint32_t)bps; }
    }
    return best_tot;
  };
  // ring size bound: the largest of (whole rings, 512, 256, ..., 32) that reaches the most resident warps
  // (level 0 and FLAG_SPILL = one choice each)
  uint32_t max_cap = 0;
  for (uint32_t i = 0; i < h.n_inst; ++i)
    max_cap = std::max(max_cap, std::max(h.inst[i].inbox_cap, std::max(h.inst[i].flight_cap, h.inst[i].wait_cap)));
  std::vector<uint32_t> cand_rs;
  if (!h.lean) cand_rs = {0xFFFFFFFFu};
  else if (g->flags & SDAS_FLAG_SPILL) cand_rs = {32u};
  else {
    cand_rs = {0xFFFFFFFFu};
    for (uint32_t rs = 512; rs >= 32; rs /= 2)
      if (rs < max_cap) cand_rs.push_back(rs);
  }
  uint32_t best_rs = cand_rs[0], best_w = 1, best_b = 0;
  uint64_t best_tot = 0;
  for (uint32_t rs : cand_rs) {
    const uint64_t per = layout_for(rs);
    uint32_t bw = 1, bb = 0;
    const uint64_t tot = per + h.off_warps <= smem_cap ? occupancy(per, rs, bw, bb) : 0;
    if (tot > best_tot) { best_tot = tot; best_rs = rs; best_w = bw; best_b = bb; }
  }
  h.ring_s = best_rs;
  h.smem_per_warp = (uint32_t)layout_for(best_rs);
  if (best_tot == 0 || h.off_warps + h.smem_per_warp > smem_cap)
    return fail(SDAS_E_LIMIT, "replica needs %u B of shared memory (max %llu): reduce caps or request_cap",
                h.smem_per_warp, (unsigned long long)(smem_cap - h.off_warps));
  pl.wpb = best_w;
  pl.blocks_per_sm = best_b;
  pl.n_sm = (uint32_t)n_sm;
  pl.smem_block = (uint32_t)(h.off_warps + (uint64_t)best_w * h.smem_per_warp);
  const uint64_t want_blocks = (h.n_local_replicas + best_w - 1) / best_w;
  pl.blocks = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)n_sm * best_b, want_blocks));
  pl.total_warps = (uint64_t)pl.blocks * best_w;
  h.off_rec_cls = sizeof(Work) + pl.total_warps * (uint64_t)g->n_requests * 8ull;
  h.off_gx = align_up(sizeof(Work) + pl.total_warps * (uint64_t)g->n_requests * 9ull, 256);

  // --- blob: DParams | candidates | arrivals | LIST ticks
  uint64_t b = align_up(sizeof(DParams), 64);
  h.off_cand = b; b += sizeof(DCand) * (uint64_t)g->n_candidates;
  h.off_arr = b; b += sizeof(DArr) * nIK;
  for (uint64_t a = 0; a < nIK; ++a)
    if (g->arrivals[a].kind == SDAS_LIST) b += 8ull * g->n_requests;
  pl.blob_bytes = align_up(b, 256);
  return SDAS_OK;
}

void pack_blob(const sdas_grid* g, const Plan& pl, std::vector<uint8_t>& blob) {
  blob.assign(pl.blob_bytes, 0);
  memcpy(blob.data(), &pl.hp, sizeof(DParams));
  DCand* dc = reinterpret_cast<DCand*>(blob.data() + pl.hp.off_cand);
  for (uint32_t c = 0; c < g->n_candidates; ++c) {
    const sdas_candidate& s = g->cand[c];
    DCand& d = dc[c];
    d.adaptive = s.kind == SDAS_ADAPTIVE;
    for (int l = 0; l < 8; ++l) d.mode[l] = s.mode[l];
    d.ctl_links = s.ctl_links; d.metric_load = s.metric == SDAS_METRIC_LOAD;
    d.lo = s.lo_permille; d.hi = s.hi_permille; d.dwell = s.dwell_windows;
    for (int k = 0; k < 4; ++k) d.band[k] = s.band_mode[k];
    d.route_override = s.route_override; d.batch_roles = s.batch_roles; d.q_hi = s.q_hi;
    d.select_role = s.select_role; d.policy_slo = s.policy_slo_ticks;
    d.kv_policy = (uint8_t)s.kv_policy;
    d.guard_links = (uint8_t)s.guard_links;
    d.guard_pct = (uint8_t)s.guard_pct;
    d.prio = s.prio ? 1u : 0u;
    d.admit = s.admit ? 1u : 0u;
    d.admit_lo = (uint16_t)s.admit_lo_permille;
    d.admit_hi = (uint16_t)s.admit_hi_permille;
    d.pace = s.pacing_gap;
    d.stale_jsq = s.stale_jsq ? 1u : 0u;
  }
  const uint64_t nIK = (uint64_t)g->n_rates * g->n_profiles;
  DArr* da = reinterpret_cast<DArr*>(blob.data() + pl.hp.off_arr);
  uint64_t lo = pl.hp.off_arr + sizeof(DArr) * nIK;
  for (uint64_t a = 0; a < nIK; ++a) {
    const sdas_arrival_desc& s = g->arrivals[a];
    DArr& d = da[a];
    d.kind = s.kind; d.list_len = s.list_len;
    d.gap0 = s.mean_gap[0]; d.gap1 = s.mean_gap[1]; d.soj0 = s.mean_sojourn[0]; d.soj1 = s.mean_sojourn[1];
    d.p_lo = s.prompt_lo; d.p_hi = s.prompt_hi; d.o_lo = s.out_lo; d.o_hi = s.out_hi;
    d.ithr = ((uint64_t)s.interactive_permille << 32) / 1000;
    if (s.kind == SDAS_LIST) {
      d.list_off = lo;
      memcpy(blob.data() + lo, s.list, 8ull * g->n_requests);
      lo += 8ull * g->n_requests;
    }
  }
}

sdas_status fill_layout(const Plan& pl, const sdas_grid* g, sdas_layout* L) {
  memset(L, 0, sizeof(*L));
  const DParams& h = pl.hp;
  L->params_bytes = pl.blob_bytes;
  const uint64_t scratch = pl.total_warps * (uint64_t)g->n_requests * 9ull;   // records + class bytes
  L->work_bytes = align_up(std::max<uint64_t>(h.off_gx + pl.total_warps * h.gx_per_warp,
                                              sizeof(Work) + pl.n_cells * 4ull), 256);
  (void)scratch;
  L->summary_bytes = align_up(std::max<uint64_t>(1, h.n_local_replicas) * SDAS_SUMMARY_BYTES, 256);
  L->records_bytes = (g->flags & SDAS_FLAG_RECORDS) ? align_up(h.n_local_replicas * g->n_requests * 8ull, 256) : 0;
  L->series_bytes = (g->flags & SDAS_FLAG_SERIES)
                        ? align_up((uint64_t)g->series_slots * g->series_windows * h.n_inst * 16ull, 256) : 0;
  L->cell_cnt_bytes = align_up(pl.n_cells * SDAS_NCNT * 8ull, 256);
  L->cell_hist_bytes = align_up(pl.n_cells * (uint64_t)SDAS_NHIST * SDAS_NBINS * 4ull, 256);
  L->best_group_bytes = align_up(std::max<uint64_t>(1, h.n_local_groups) * 4ull, 256);
  L->best_row_bytes = align_up(std::max<uint64_t>(1, pl.n_rows) * 4ull, 256);
  L->trace_bytes = (g->flags & SDAS_FLAG_TRACE) ? align_up(8ull + 24ull * g->trace_cap, 256) : 0;
  L->n_local_replicas = h.n_local_replicas;
  L->n_local_groups = h.n_local_groups;
  L->n_groups = pl.n_groups;
  L->n_cells = pl.n_cells;
  L->n_rows = pl.n_rows;
  L->n_replicas = pl.n_replicas;
  L->n_instances = h.n_inst;
  L->smem_per_replica = h.smem_per_warp;
  L->warps_per_block = pl.wpb;
  L->blocks_per_sm = pl.blocks_per_sm;
  L->resident_replicas = pl.total_warps;
  L->k1_variant = h.lean;
  L->ring_s = h.ring_s;
  L->cell_series_bytes = (g->flags & SDAS_FLAG_CELL_SERIES)
                             ? align_up(pl.n_cells * (uint64_t)g->series_windows * h.n_inst * 64ull, 256) : 0;
  return SDAS_OK;
}

bool aligned(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 255u) == 0; }

}  // namespace

extern "C" {

const char* sdas_last_error(void) { return g_err.c_str(); }
const char* sdas_version(void) { return "sdas-b200 0.1 (sm_100a)"; }

sdas_status sdas_pipeline_create(const sdas_pipeline_desc* desc, sdas_pipeline** out) {
  if (!out) return fail(SDAS_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  sdas_status s = validate_desc(desc);
  if (s != SDAS_OK) return s;
  sdas_pipeline* p = new sdas_pipeline();
  p->roles.assign(desc->roles, desc->roles + desc->n_roles);
  p->links.assign(desc->links, desc->links + desc->n_links);
  p->inst_cost.resize(desc->n_roles);
  for (uint32_t r = 0; r < desc->n_roles; ++r) {
    const sdas_role_desc& R = desc->roles[r];
    for (uint32_t x = 0; x < R.n_instances; ++x) p->inst_cost[r].push_back(R.inst_cost ? R.inst_cost[x] : R.cost);
    p->roles[r].inst_cost = nullptr;  // deep-copied above
    p->B_def.push_back(R.max_num_seqs);
    p->F_def.push_back(R.n_functions);
    p->n_inst += R.n_instances;
  }
  for (const sdas_link_desc& L : p->links) {
    p->mode_def.push_back(L.mode);
    p->chunk_def.push_back(L.chunk_tokens);
    p->net_def.push_back(L.net_delay);
    p->pace_def.push_back(L.pacing_gap);
  }
  p->B_cur = p->B_def; p->F_cur = p->F_def;
  p->mode_cur = p->mode_def; p->chunk_cur = p->chunk_def; p->net_cur = p->net_def; p->pace_cur = p->pace_def;
  p->feedback_role = desc->feedback_role;
  p->request_cap = desc->request_cap;
  p->window = desc->window_ticks;
  p->slo = desc->slo_ticks;
  p->kv_role = desc->kv_role;
  p->kv_ctx = desc->kv_ctx_tokens;
  p->kv_tau = desc->kv_tau_xfer;
  p->kv_skew = desc->kv_home_skew;
  *out = p;
  return ok();
}

void sdas_pipeline_destroy(sdas_pipeline* p) { delete p; }

sdas_status sdas_set(sdas_pipeline* p, const char* knob, int64_t value) {
  if (!p || !knob) return fail(SDAS_E_INVALID_ARG, "pipeline or knob is NULL");
  int kind;
  uint32_t idx;
  if (parse_knob(p, knob, &kind, &idx)) return fail(SDAS_E_UNKNOWN_PARAM, "unknown parameter '%s'", knob);
  static const int64_t lo[6] = {1, 1, 0, 1, 1, 0};
  static const int64_t hi[6] = {SDAS_MAX_BATCH, 255, SDAS_TOKEN, 65535, (1ll << 31) - 1, 1ll << 18};
  if (value < lo[kind] || value > hi[kind])
    return fail(SDAS_E_OUT_OF_RANGE, "value %lld out of range [%lld, %lld] for '%s'", (long long)value,
                (long long)lo[kind], (long long)hi[kind], knob);
  std::vector<uint32_t>* v[6] = {&p->B_cur, &p->F_cur, &p->mode_cur, &p->chunk_cur, &p->net_cur, &p->pace_cur};
  (*v[kind])[idx] = (uint32_t)value;
  return ok();
}

sdas_status sdas_reset(sdas_pipeline* p, const char* knob) {
  if (!p || !knob) return fail(SDAS_E_INVALID_ARG, "pipeline or knob is NULL");
  int kind;
  uint32_t idx;
  if (parse_knob(p, knob, &kind, &idx)) return fail(SDAS_E_UNKNOWN_PARAM, "unknown parameter '%s'", knob);
  std::vector<uint32_t>* cur[6] = {&p->B_cur, &p->F_cur, &p->mode_cur, &p->chunk_cur, &p->net_cur, &p->pace_cur};
  std::vector<uint32_t>* def[6] = {&p->B_def, &p->F_def, &p->mode_def, &p->chunk_def, &p->net_def, &p->pace_def};
  (*cur[kind])[idx] = (*def[kind])[idx];
  return ok();
}

sdas_status sdas_get(const sdas_pipeline* p, const char* knob, int64_t* value) {
  if (!p || !knob || !value) return fail(SDAS_E_INVALID_ARG, "NULL argument");
  int kind;
  uint32_t idx;
  if (parse_knob(p, knob, &kind, &idx)) return fail(SDAS_E_UNKNOWN_PARAM, "unknown parameter '%s'", knob);
  const std::vector<uint32_t>* cur[6] = {&p->B_cur, &p->F_cur, &p->mode_cur, &p->chunk_cur, &p->net_cur,
                                         &p->pace_cur};
  *value = (*cur[kind])[idx];
  return ok();
}

sdas_status sdas_results_layout(const sdas_pipeline* p, const sdas_grid* grid, sdas_layout* out) {
  if (!out) return fail(SDAS_E_INVALID_ARG, "out is NULL");
  Plan pl;
  sdas_status s = plan(p, grid, pl);
  if (s != SDAS_OK) return s;
  fill_layout(pl, grid, out);
  return ok();
}

static sdas_status run_sim(const sdas_pipeline* p, const sdas_grid* g, const sdas_buffers* d, void* stream,
                           Plan& pl) {
  if (!d) return fail(SDAS_E_INVALID_ARG, "buffers is NULL");
  sdas_status s = plan(p, g, pl);
  if (s != SDAS_OK) return s;
  if (!d->params || !d->work || !d->summary || !d->cell_cnt || !d->cell_hist)
    return fail(SDAS_E_BUFFER, "params, work, summary, cell_cnt and cell_hist are required");
  if (!aligned(d->params) || !aligned(d->work) || !aligned(d->summary) || !aligned(d->cell_cnt) ||
      !aligned(d->cell_hist))
    return fail(SDAS_E_BUFFER, "device buffers must be 256-byte aligned");
  if ((g->flags & SDAS_FLAG_RECORDS) && !d->records) return fail(SDAS_E_BUFFER, "FLAG_RECORDS needs records");
  if ((g->flags & SDAS_FLAG_SERIES) && !d->series) return fail(SDAS_E_BUFFER, "FLAG_SERIES needs series");
  if ((g->flags & SDAS_FLAG_TRACE) && !d->trace) return fail(SDAS_E_BUFFER, "FLAG_TRACE needs trace");
  if ((g->flags & SDAS_FLAG_CELL_SERIES) && g->series_windows && !d->cell_series)
    return fail(SDAS_E_BUFFER, "FLAG_CELL_SERIES needs cell_series");
  std::vector<uint8_t> blob;
  pack_blob(g, pl, blob);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(d->params, blob.data(), blob.size(), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return fail(SDAS_E_CUDA, "params upload: %s", cudaGetErrorString(e));
  int rc = launch_simulate(reinterpret_cast<const uint8_t*>(d->params), pl.hp, d, pl.blocks, pl.wpb, pl.smem_block,
                           stream, log2tab().t);
  if (rc) return fail(SDAS_E_CUDA, "K1 launch: %s", cuda_error_string(rc));
  // the pageable-memory async copy has been staged when cudaMemcpyAsync returned; `blob` may go
  return SDAS_OK;
}

sdas_status sdas_simulate(const sdas_pipeline* p, const sdas_grid* grid, const sdas_buffers* dev, void* stream) {
  Plan pl;
  sdas_status s = run_sim(p, grid, dev, stream, pl);
  return s == SDAS_OK ? ok() : s;
}

sdas_status sdas_control_sweep(const sdas_pipeline* p, const sdas_grid* grid, uint32_t objective,
                               uint64_t objective_slo, const sdas_buffers* dev, void* stream) {
  if (objective > SDAS_MIN_P99_E2E_INTERACTIVE) return fail(SDAS_E_INVALID_ARG, "objective: bad enum");
  if (dev && !dev->best_group) return fail(SDAS_E_BUFFER, "control_sweep needs best_group");
  Plan pl;
  sdas_status s = run_sim(p, grid, dev, stream, pl);
  if (s != SDAS_OK) return s;
  int rc = launch_group_argmin(reinterpret_cast<const uint8_t*>(dev->params), pl.hp, dev, objective, objective_slo,
                               stream);
  if (rc) return fail(SDAS_E_CUDA, "K3 launch: %s", cuda_error_string(rc));
  return ok();
}

sdas_status sdas_group_argmin(const sdas_pipeline* p, const sdas_grid* grid, uint32_t objective,
                              uint64_t objective_slo, const sdas_buffers* dev, void* stream) {
  if (objective > SDAS_MIN_P99_E2E_INTERACTIVE) return fail(SDAS_E_INVALID_ARG, "objective: bad enum");
  if (!dev || !dev->params || !dev->summary || !dev->best_group)
    return fail(SDAS_E_BUFFER, "group_argmin needs params, summary and best_group");
  Plan pl;
  sdas_status s = plan(p, grid, pl);
  if (s != SDAS_OK) return s;
  std::vector<uint8_t> blob;
  pack_blob(grid, pl, blob);
  cudaError_t e = cudaMemcpyAsync(dev->params, blob.data(), sizeof(DParams), cudaMemcpyHostToDevice,
                                  reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(SDAS_E_CUDA, "params upload: %s", cudaGetErrorString(e));
  int rc = launch_group_argmin(reinterpret_cast<const uint8_t*>(dev->params), pl.hp, dev, objective, objective_slo,
                               stream);
  if (rc) return fail(SDAS_E_CUDA, "K3 launch: %s", cuda_error_string(rc));
  return ok();
}

sdas_status sdas_finalize(const sdas_pipeline* p, const sdas_grid* grid, uint32_t objective, uint64_t objective_slo,
                          const sdas_buffers* dev, void* stream) {
  if (objective > SDAS_MIN_P99_E2E_INTERACTIVE) return fail(SDAS_E_INVALID_ARG, "objective: bad enum");
  if (!dev || !dev->params || !dev->work || !dev->cell_cnt || !dev->cell_hist || !dev->best_row)
    return fail(SDAS_E_BUFFER, "finalize needs params, work, cell_cnt, cell_hist and best_row");
  Plan pl;
  sdas_status s = plan(p, grid, pl);
  if (s != SDAS_OK) return s;
  std::vector<uint8_t> blob;
  pack_blob(grid, pl, blob);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(dev->params, blob.data(), sizeof(DParams), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return fail(SDAS_E_CUDA, "params upload: %s", cudaGetErrorString(e));
  int rc = launch_finalize(reinterpret_cast<const uint8_t*>(dev->params), pl.hp, dev, objective, objective_slo,
                           pl.n_cells, pl.n_rows, stream);
  if (rc) return fail(SDAS_E_CUDA, "K4/K5 launch: %s", cuda_error_string(rc));
  return ok();
}

sdas_status sdas_compile_intent(const sdas_pipeline* p, const sdas_intent* in, sdas_candidate* out,
                                uint32_t* objective_out) {
  if (!p || !in || !out || !objective_out) return fail(SDAS_E_INVALID_ARG, "NULL argument");
  if (in->objective > SDAS_INTENT_MIN_P90_LATENCY) return fail(SDAS_E_INVALID_ARG, "objective: bad enum");
  if (in->objective == SDAS_INTENT_NONE && !in->rules)
    return fail(SDAS_E_INVALID_ARG, "InvalidIntent: neither an objective nor explicit rules (SPEC.md:483)");
  if (in->n_constraints && !in->constraints) return fail(SDAS_E_INVALID_ARG, "constraints: NULL");
  const uint32_t nl = (uint32_t)p->links.size();
  const uint32_t all_links = nl ? (1u << nl) - 1u : 0u;
  sdas_candidate c;
  if (in->rules) {
    c = *in->rules;                                            // explicit rules pass through unchanged
  } else {
    memset(&c, 0, sizeof(c));
    c.kind = SDAS_STATIC;
    for (int l = 0; l < 8; ++l) c.mode[l] = 255;
    c.metric = SDAS_METRIC_BUSY;
    c.lo_permille = 400; c.hi_permille = 800; c.dwell_windows = 1;
    c.band_mode[0] = SDAS_TOKEN; c.band_mode[1] = SDAS_FUNCTION; c.band_mode[2] = SDAS_BATCH;
    c.band_mode[3] = SDAS_BATCH;
    c.route_override = SDAS_ROUTE_NONE; c.q_hi = 2; c.select_role = -1; c.kv_policy = SDAS_KV_OFF;
    c.guard_pct = 90;
    c.pacing_gap = 0xFFFFFFFFu;
  }
  uint32_t obj = SDAS_MIN_P99_E2E;
  const uint64_t W = p->window ? p->window : 1;
  if (in->objective == SDAS_INTENT_MAX_THROUGHPUT) {           // SPEC.md:478-479 three-band template
    c.kind = SDAS_ADAPTIVE;
    for (int l = 0; l < 8; ++l) c.mode[l] = 255;
    c.ctl_links = all_links;
    c.metric = SDAS_METRIC_BUSY;
    c.lo_permille = 400; c.hi_permille = 800;
    c.band_mode[0] = SDAS_TOKEN; c.band_mode[1] = SDAS_FUNCTION; c.band_mode[2] = SDAS_BATCH;
    c.dwell_windows = (uint32_t)std::max<uint64_t>(1, (1000000ull + W - 1) / W);   // 1000 ms dwell
    obj = SDAS_MAX_THROUGHPUT;
  } else if (in->objective == SDAS_INTENT_MIN_P90_LATENCY) {   // SPEC.md:480 token_stream everywhere
    c.kind = SDAS_STATIC;
    for (uint32_t l = 0; l < 8; ++l) c.mode[l] = l < nl ? (uint8_t)SDAS_TOKEN : 255;
    c.ctl_links = 0;
    c.dwell_windows = (uint32_t)std::max<uint64_t>(1, (1000000ull + W - 1) / W);
    obj = SDAS_MIN_P90_E2E;
  }
  for (uint32_t k = 0; k < in->n_constraints; ++k) {           // SPEC.md:480-481 constraint guards (M25)
    const sdas_constraint& q = in->constraints[k];
    if (q.metric > SDAS_CONSTRAINT_E2E_P99) return fail(SDAS_E_INVALID_ARG, "constraints[%u].metric: bad enum", k);
    if (q.scope_links & ~all_links) return fail(SDAS_E_INVALID_ARG, "constraints[%u].scope_links: no such link", k);
    const uint32_t pct = q.metric == SDAS_CONSTRAINT_E2E_P90 ? 90u : 99u;
    const bool first = k == 0;
    if (first && in->rules && (in->rules->batch_roles || in->rules->select_role >= 0) &&
        in->rules->policy_slo_ticks != q.bound_ticks)
      return fail(SDAS_E_LIMIT, "constraints[0].bound_ticks conflicts with the rules' policy_slo_ticks");
    if (!first && (pct != c.guard_pct || q.bound_ticks != c.policy_slo_ticks))
      return fail(SDAS_E_LIMIT, "constraints[%u]: one (metric, bound) per compiled policy", k);
    c.guard_pct = pct;
    c.policy_slo_ticks = q.bound_ticks;
    c.guard_links |= q.scope_links ? q.scope_links : all_links;
    c.kind = SDAS_ADAPTIVE;
  }
  *out = c;
  *objective_out = obj;
  return ok();
}

sdas_status sdas_metrics(const sdas_pipeline* p, const sdas_grid* grid, const sdas_buffers* host, uint32_t scope,
                         uint64_t index, sdas_metrics_out* out) {
  if (!p || !grid || !host || !out) return fail(SDAS_E_INVALID_ARG, "NULL argument");
  Plan pl;
  sdas_status s = plan(p, grid, pl);
  if (s != SDAS_OK) return s;
  memset(out, 0, sizeof(*out));
  out->best = -1;
  auto derive = [&]() {  // M19 fp64 derived values from integer sums
    out->mean_e2e = out->completed ? (double)out->sum_e2e / (double)out->completed : 0.0;
    out->mean_ff = out->completed ? (double)out->sum_ff / (double)out->completed : 0.0;
    out->throughput = out->makespan ? (double)(out->completed * 1000000ull) / (double)out->makespan : 0.0;
    out->goodput = out->makespan ? (double)(out->good * 1000000ull) / (double)out->makespan : 0.0;
    out->message_events = out->arrivals + out->deliveries;
    out->des_events = out->message_events + out->recv_steps + out->decode_steps + out->window_closes;
  };
  if (scope == SDAS_SCOPE_REPLICA) {
    if (!host->summary) return fail(SDAS_E_STATE, "REPLICA scope needs summary");
    if (index >= pl.hp.n_local_replicas) return fail(SDAS_E_INVALID_ARG, "index out of range");
    const uint32_t* w = reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(host->summary) +
                                                          index * SDAS_SUMMARY_BYTES);
    auto u64 = [&](int k) { return (uint64_t)w[k] | ((uint64_t)w[k + 1] << 32); };
    out->status = w[0]; out->n_replicas = 1; out->admitted = w[1]; out->dropped = w[2]; out->completed = w[3];
    out->makespan = u64(4); out->sum_e2e = u64(6); out->sum_ff = u64(8); out->int_nsys = u64(10);
    out->p50_e2e = w[12]; out->p99_e2e = w[13]; out->p50_ff = w[14]; out->p99_ff = w[15];
    out->bin_p50_e2e = w[16] & 0xFFFF; out->bin_p99_e2e = w[16] >> 16;
    out->bin_p50_ff = w[41] & 0xFFFF; out->bin_p99_ff = w[41] >> 16;
    out->p90_e2e = w[17];
    out->arrivals = w[20]; out->deliveries = w[21]; out->recv_steps = w[22]; out->decode_steps = w[23];
    out->window_closes = w[24]; out->mode_switches = w[25]; out->good = w[26]; out->large_items = w[27];
    out->tokens = u64(28);
    out->completed_int = w[32]; out->rejected = w[33]; out->sum_e2e_int = u64(34);
    out->p50_e2e_int = w[36]; out->p99_e2e_int = w[37]; out->good_int = w[38];
    derive();
    if (host->series && (grid->flags & SDAS_FLAG_SERIES) && grid->series_stride) {
      const uint64_t lg = index / pl.hp.C, c = index % pl.hp.C;
      const uint64_t rid = (pl.hp.first_group + lg * pl.hp.world) * pl.hp.C + c;
      if (rid % grid->series_stride == 0 && rid / grid->series_stride < grid->series_slots) {
        const uint64_t per = (uint64_t)grid->series_windows * pl.hp.n_inst;
        out->series = reinterpret_cast<const uint8_t*>(host->series) + (rid / grid->series_stride) * per * 16;
        out->series_len = std::min<uint64_t>(per, (uint64_t)(w[24] + 1) * pl.hp.n_inst);
      }
    }
    return ok();
  }
  if (scope == SDAS_SCOPE_CELL) {
    if (!host->cell_cnt || !host->cell_hist) return fail(SDAS_E_STATE, "CELL scope needs cell_cnt and cell_hist");
    if (index >= pl.n_cells) return fail(SDAS_E_INVALID_ARG, "index out of range");
    const int64_t* q = reinterpret_cast<const int64_t*>(host->cell_cnt) + index * SDAS_NCNT;
    const int32_t* h = reinterpret_cast<const int32_t*>(host->cell_hist) + index * SDAS_NHIST * SDAS_NBINS;
    out->status = q[2] ? SDAS_REPLICA_OVERFLOW : q[3] ? SDAS_REPLICA_TRUNCATED : SDAS_REPLICA_OK;
    out->n_replicas = q[0]; out->admitted = q[4]; out->dropped = q[5]; out->completed = q[6];
    out->sum_e2e = q[7]; out->sum_ff = q[8]; out->makespan = q[9]; out->int_nsys = q[10]; out->good = q[11];
    out->large_items = q[12]; out->arrivals = q[13]; out->deliveries = q[14]; out->recv_steps = q[15];
    out->decode_steps = q[16]; out->window_closes = q[17]; out->mode_switches = q[18]; out->tokens = q[19];
    auto pct = [&](const int32_t* hh, uint32_t num, uint32_t* val, uint32_t* bin) {
      uint64_t n = 0;
      for (int b = 0; b < SDAS_NBINS; ++b) n += (uint32_t)hh[b];
      *val = 0xFFFFFFFFu;
      *bin = 0xFFFFu;
      if (!n) return;
      const uint64_t k = (num * n + 99) / 100;
      uint64_t cum = 0;
      for (uint32_t b = 0; b < SDAS_NBINS; ++b) {
        cum += (uint32_t)hh[b];
        if (cum >= k) {
          *bin = b;
          *val = b < 16 ? b : (16u + ((b - 16u) & 15u)) << ((b - 16u) >> 4);
          return;
        }
      }
    };
    pct(h, 50, &out->p50_e2e, &out->bin_p50_e2e);
    pct(h, 99, &out->p99_e2e, &out->bin_p99_e2e);
    uint32_t bin90, binx;
    pct(h, 90, &out->p90_e2e, &bin90);
    pct(h + 2 * SDAS_NBINS, 50, &out->p50_e2e_int, &binx);
    pct(h + 2 * SDAS_NBINS, 99, &out->p99_e2e_int, &binx);
    out->completed_int = q[24]; out->rejected = q[25]; out->sum_e2e_int = q[26]; out->good_int = q[27];
    pct(h + SDAS_NBINS, 50, &out->p50_ff, &out->bin_p50_ff);
    pct(h + SDAS_NBINS, 99, &out->p99_ff, &out->bin_p99_ff);
    derive();
    return ok();
  }
  if (scope == SDAS_SCOPE_GROUP) {
    if (!host->best_group) return fail(SDAS_E_STATE, "GROUP scope needs best_group (run sdas_control_sweep)");
    if (index >= pl.hp.n_local_groups) return fail(SDAS_E_INVALID_ARG, "index out of range");
    out->best = reinterpret_cast<const int32_t*>(host->best_group)[index];
    return ok();
  }
  if (scope == SDAS_SCOPE_ROW) {
    if (!host->best_row) return fail(SDAS_E_STATE, "ROW scope needs best_row (run sdas_finalize)");
    if (index >= pl.n_rows) return fail(SDAS_E_INVALID_ARG, "index out of range");
    out->best = reinterpret_cast<const int32_t*>(host->best_row)[index];
    return ok();
  }
  return fail(SDAS_E_INVALID_ARG, "scope: bad enum");
}

}  // extern "C"
