// sdas_k1.cuh -- K1: persistent replica-per-warp simulation kernel (included by sdas_kernels.cu).
//
// One warp simulates one replica at a time (rules M0-M20); a warp claims the next local
// replica with one atomicAdd.  Layout of the work inside a warp:
//   * uniform replica state (time, arrival generator, counters) in registers, identical in all lanes;
//   * lane i = instance i: server state (step end, ring indices, batch size, max_num_seqs, window
//     accumulators) in registers, so the next-event search is one __reduce_min_sync over 32-bit
//     deltas and the window integration is lane-parallel;
//   * lane k = batch sequence k of the instance whose DECODE completes: token advance, emission test,
//     ballot/popc message placement, stable compaction;
//   * shared memory: request table, per-instance rings (inbox, in-flight, decode-wait), batch words,
//     controller state; the finalize scratch aliases the (dead) request table.
// TRACE adds the debug event trace (separate instantiation); MAXOUT is the largest fan-out (1 or 2);
// CLS (f2, M26-M29): two request classes -- per-class inbox / wait rings (class-1 ring right after the
// class-0 ring; used only under priority service, so FIFO across classes holds otherwise), the
// admission gate, per-class metrics.  Pipelines without interactive requests never pay for it.
// LV: 0 generic; 1 = no KV / pacing / classes / LOAD metric / truncation (compiled out);
// 2 (LEAN) = level 1 + one instance per role and no fan-out: routing is the identity.  Shrinks the
// I-cache-bound hot loop.  LEAN also skips events that change nothing observable: deliveries into busy
// instances, emission points of the source's runs, silent RECVs and the ends of RECVs that a held batch's
// run follows -- bit-identical to event-per-step execution.

#define K1_UNLIKELY(x) (x)   // marks cold branches (__builtin_expect layout measured +2 % slower)

#ifndef K1_LB_THREADS
#define K1_LB_THREADS 256   // 2 x 8 warps per SM at <= 128 registers
#define K1_LB_MAXREG 128
#endif
#ifndef K1_LEAN_THREADS     // the LEAN level's own bounds (A/B: -DK1_LEAN_THREADS=192 -DK1_LEAN_MAXREG=112)
#define K1_LEAN_THREADS K1_LB_THREADS
#define K1_LEAN_MAXREG K1_LB_MAXREG
#endif
template <bool TRACE, int MAXOUT, bool CLS, int LV, bool SPL>
__global__ void __launch_bounds__(LV == 2 ? K1_LEAN_THREADS : K1_LB_THREADS)
__maxnreg__(LV == 2 ? K1_LEAN_MAXREG : K1_LB_MAXREG)
k1_simulate(const uint8_t* __restrict__ blob, Work* __restrict__ work, uint8_t* __restrict__ summary,
            unsigned long long* __restrict__ records_out, uint8_t* __restrict__ series,
            long long* __restrict__ cell_cnt, int* __restrict__ cell_hist, uint8_t* __restrict__ trace_buf,
            unsigned long long* __restrict__ cell_series, const __grid_constant__ DParams Pk) {   // scalars from parameter space (uniform registers)
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
  uint8_t* const Wr = smem + Pk.off_warps + wib * Pk.smem_per_warp;
  WarpHdr* const H = reinterpret_cast<WarpHdr*>(Wr);
  unsigned long long* const rA = at<unsigned long long>(Wr, Pk.off_reqA);
  unsigned long long* const rFF = at<unsigned long long>(Wr, Pk.off_reqFF);
  uint32_t* const rJ = at<uint32_t>(Wr, Pk.off_reqJ);
  uint32_t* const rO = at<uint32_t>(Wr, Pk.off_reqO);
  uint16_t* const rNit = at<uint16_t>(Wr, Pk.off_reqNit);
  uint16_t* const rOut = at<uint16_t>(Wr, Pk.off_reqOut);
  uint32_t* const bitmap = at<uint32_t>(Wr, Pk.off_bitmap);
  uint32_t* const scratch = at<uint32_t>(Wr, Pk.off_scratch);

  // hoisted constants
  const uint32_t N = Pk.n_requests, C = Pk.C, n_inst = Pk.n_inst, fb_role = Pk.feedback_role;
  const uint32_t R_cap = Pk.request_cap, n_links = Pk.n_links;
  const uint32_t W32 = (uint32_t)Pk.window;
  constexpr bool LEAN = LV >= 2;
  const unsigned long long max_ticks = LV ? 0ull : Pk.max_ticks;   // specialised grids never truncate
  const bool need_lint = LV == 0 && Pk.need_lint != 0;
  const bool coalesce = LV || (Pk.flags & SDAS_FLAG_STEPWISE) == 0;   // silent DECODE runs
  const bool need_pace = LV == 0 && Pk.need_pace != 0;                     // f4 M30: some link is paced
  const uint32_t key0 = (uint32_t)Pk.master_seed, key1 = (uint32_t)(Pk.master_seed >> 32);
  const unsigned long long gwarp = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + wib;
  unsigned long long* const rec_scratch =
      reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(work) + sizeof(Work)) + gwarp * N;
  const DCand* const cands = reinterpret_cast<const DCand*>(blob + Pk.off_cand);
  const DArr* const arrs = reinterpret_cast<const DArr*>(blob + Pk.off_arr);

  // lane-resident constants of instance `lane`
  const bool is_inst = lane < (int)n_inst;
  const DInst& MI = P.inst[is_inst ? lane : 0];
  const uint32_t my_role = LEAN ? (uint32_t)lane : MI.role;
  // two-level rings (levels >= 1): a ring keeps its oldest RS entries in shared memory and
  // the rest in this warp's extension area of `work`; the my_*_cap registers hold the shared-memory sizes
  // min(capacity, RS) and the logical capacities (overflow, rule M14) are read from MI only past them
  // (LEAN only: on level 1 the extra code pushed the hot loop out of the instruction cache, +45 % at config 3)
  constexpr bool LAZY = LV == 2;   // deliveries into a busy instance are not events
  constexpr bool SILENT = LV == 2; // a RECV whose end changes nothing else is not an event
  constexpr bool CHAIN = LV == 2;  // a non-closing RECV while a batch is held flows into its next run (§5.8)
  constexpr bool SPILL = SPL;                          // a separate instantiation: grids whose rings fit whole
  static_assert(!SPL || LV >= 1, "two-level rings exist on the specialised levels only");   // never pay for it
  const uint32_t RS = SPILL ? Pk.ring_s : 0xFFFFFFFFu;
  const uint32_t my_inbox_cap = min(MI.inbox_cap, RS), my_flight_cap = min(MI.flight_cap, RS),
                 my_wait_cap = min(MI.wait_cap, RS);
  auto gxa = [&](uint32_t off) -> uint8_t* {           // extension area of this warp (cold paths only)
    return reinterpret_cast<uint8_t*>(work) + Pk.off_gx + gwarp * Pk.gx_per_warp + off;
  };
  uint8_t* const my_inbox = Wr + MI.off_inbox;
  uint8_t* const my_ftick = Wr + MI.off_ftick;
  uint8_t* const my_fbody = Wr + MI.off_fbody;
  const bool my_large = (MI.flags & 1u) != 0;
  // f1 (M21-M24): KV-role instances keep, per inbox entry, the tick a hinted transfer completes
  const uint32_t kv_role = LV ? 0u : Pk.kv_role;
  const bool my_kv = kv_role != 0 && is_inst && my_role == kv_role;
  uint32_t* const my_iready = reinterpret_cast<uint32_t*>(my_inbox + 8u * my_inbox_cap);
  // per in-flight entry of a KV-role instance: the tick its hinted transfer completes (emission + tau*ctx,
  // M23 HINT) -- kept beside the ring because pacing (M30) separates dispatch from emission
  uint32_t* const my_fready = reinterpret_cast<uint32_t*>(my_fbody + 8u * my_flight_cap);
  uint8_t* const rHome = Wr + Pk.off_reqHome;
  uint8_t* const rCls = Wr + Pk.off_reqCls;                        // f2: class per request slot
  uint8_t* const rec_cls = reinterpret_cast<uint8_t*>(work) + Pk.off_rec_cls + gwarp * N;

  for (;;) {
    unsigned long long x = 0;
    if (lane == 0) x = atomicAdd(&work->next_replica, 1ull);
    x = __shfl_sync(FULL, x, 0);
    if (x >= Pk.n_local_replicas) break;

    // ---------------------------------------------------------------- replica coordinates (M1)
    const uint32_t c = (uint32_t)(x % C);
    const unsigned long long g = Pk.first_group + (x / C) * Pk.world;
    const uint32_t s_coord = (uint32_t)(g % Pk.S) + Pk.seed_offset;
    const DCand& cd = cands[c];
    const DArr& ad = arrs[(g / Pk.S) % (Pk.I * (unsigned long long)Pk.K)];
    const bool trace_on = TRACE && g * C + c == Pk.trace_replica;
    unsigned long long* const rec =
        (Pk.flags & SDAS_FLAG_RECORDS) ? records_out + x * (unsigned long long)N : rec_scratch;

    // ---------------------------------------------------------------- init
    // Warp discipline (independent thread scheduling): warp-uniform scalars live in registers or are
    // lane-distributed; shared scalars are read-modify-written by lane 0 only and broadcast by shfl;
    // __syncwarp() orders cross-lane shared-memory traffic at phase boundaries.
    // current mode per link, 2 bits each (M16 state, bits 0-13); bits 28-30 cache the feedback role and
    // bit 31 cd.adaptive, so the hot paths test them from a register instead of a parameter / global load
    uint32_t modes = (cd.adaptive ? 0x80000000u : 0u) | (fb_role << 28);
    for (uint32_t l = 0; l < n_links; ++l)
      modes |= (uint32_t)(cd.mode[l] == 255 ? P.link[l].mode : cd.mode[l]) << (2 * l);
    int32_t qlm = -(1 << 30), q_last_sel = -(1 << 30);   // lane l: last change of link l's mode
    uint32_t rr_l = 0;                                    // lane r: round-robin counter of role r
    uint32_t sel_l = lane < (int)Pk.n_roles ? P.role[lane].large_inst : 0u;  // lane r: SELECT target
    if (lane == 0) {
      *H = WarpHdr{};
      uint32_t ss = 0xFFFFFFFFu;                          // series slot, computed once per replica (M15)
      if ((Pk.flags & SDAS_FLAG_SERIES) && Pk.series_stride) {
        const unsigned long long rid = g * C + c;
        if (rid % Pk.series_stride == 0 && rid / Pk.series_stride < Pk.series_slots)
          ss = (uint32_t)(rid / Pk.series_stride);
      }
      H->ser_slot = ss;
      H->cell = (uint32_t)(((g / Pk.S) % (Pk.I * (unsigned long long)Pk.K)) * C + c);
    }
    for (uint32_t w = lane; w < Pk.bitmap_words; w += 32) {
      const uint32_t rem = R_cap - w * 32;
      bitmap[w] = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
    }
    __syncwarp();

    // lane-per-instance server state (M7)
    unsigned long long cur = 0, acc_qint = 0, acc_lint = 0, tok = 0;
    uint32_t st = IDLE, end_lo = 0, ih = 0, in = 0, fh = 0, fn = 0, wh = 0, wn = 0, b = 0, fhead = 0;
    uint32_t Bk = is_inst ? MI.B_default : 1u;
    int32_t qlB = -(1 << 30);
    uint32_t acc_busy = 0, acc_maxq = 0, cnt_deliv = 0, cnt_recv = 0, cnt_decode = 0, n_large = 0, cnt_kv = 0;
    uint32_t H_next = 0;   // KV home (index within kv_role) of the next arriving request (M21)
    uint32_t snap = 0;     // M31: this instance's load polled at the last window close (stale JSQ)
    // A DECODE "run" is runm consecutive steps of one unchanged batch of which all but the last are
    // silent (no emission point, no finish, no first feedback, no admission, empty inbox): they change
    // nothing any other part of the model observes, so they complete as one event at end_lo with the
    // per-step bookkeeping applied in bulk.  A message or arrival entering the inbox mid-run cuts the run
    // at the first step boundary >= its tick (RECV-first START, M7); flushm > 0 = a cut landed exactly
    // on a boundary of this tick: that many silent steps end now (the instance is idle for START) and the
    // batch words still lack them -- the instance's next start_decode adds them (TRACE builds: the flush
    // loop before START applies them, with their trace records).
    uint32_t runm = 1, flushm = 0;
    // f2: class-1 (interactive) ring heads and counts; `in` / `wn` stay the totals over both rings
    uint32_t ih1 = 0, in1 = 0, wh1 = 0, wn1 = 0;
    const bool prio = CLS && cd.prio != 0;
    uint32_t C_next = 0;                                  // class of the next arriving request (M26)
    bool gate = false;                                    // M28: admission is interactive-only
    int32_t q_last_gate = -(1 << 30);

    // uniform replica state
    unsigned long long t = 0, A_next = 0, int_nsys_acc = 0;
    uint32_t t_lo = 0, nb_lo = W32, A_lo = 0, jn = 0, P_next = 0, O_next = 0, nsys = 0, wk = 0;
    bool arr_near = false, ovf = false, arr_more = N > 0;
    uint32_t status = SDAS_REPLICA_OK;
    uint32_t mm_k = 0;
    unsigned long long mm_end = 0;

    auto trace = [&](uint32_t code, uint32_t a, uint32_t bb, uint32_t cc) {
      if (TRACE && trace_on && lane == 0) {
        const unsigned long long k = atomicAdd(reinterpret_cast<unsigned long long*>(trace_buf), 1ull);
        if (k < Pk.trace_cap) {
          TraceRec* r = reinterpret_cast<TraceRec*>(trace_buf + 8) + k;
          r->tick = t; r->code = code; r->a = a; r->b = bb; r->c = cc;
        }
      }
    };
    auto trace_at = [&](unsigned long long tick, uint32_t code, uint32_t a, uint32_t bb, uint32_t cc) {
      if (TRACE && trace_on && lane == 0) {
        const unsigned long long k = atomicAdd(reinterpret_cast<unsigned long long*>(trace_buf), 1ull);
        if (k < Pk.trace_cap) {
          TraceRec* r = reinterpret_cast<TraceRec*>(trace_buf + 8) + k;
          r->tick = tick; r->code = code; r->a = a; r->b = bb; r->c = cc;
        }
      }
    };
    // trace records of the silent steps 1..n of a run that began at tick t_run (step length c);
    // with_last = false: the START of step n+1 is not a DECODE start
    auto trace_silent = [&](uint32_t i, uint32_t bi, uint32_t c, unsigned long long t_run, uint32_t n, bool last_start) {
      if (TRACE && trace_on)
        for (uint32_t j = 1; j <= n; ++j) {
          trace_at(t_run + (unsigned long long)j * c, TR_DECODE_DONE, i, bi, 0);
          if (j < n || last_start) trace_at(t_run + (unsigned long long)j * c, TR_DECODE_START, i, bi, c);
        }
    };
    auto trace_lane = [&](uint32_t code, uint32_t a, uint32_t bb, uint32_t cc) {
      if (TRACE && trace_on) {
        const unsigned long long k = atomicAdd(reinterpret_cast<unsigned long long*>(trace_buf), 1ull);
        if (k < Pk.trace_cap) {
          TraceRec* r = reinterpret_cast<TraceRec*>(trace_buf + 8) + k;
          r->tick = t; r->code = code; r->a = a; r->b = bb; r->c = cc;
        }
      }
    };

    // ---------------------------------------------------------------- arrivals (M4, M5)
    auto gen = [&](uint32_t j, unsigned long long A_prev) {
      const uint32_t kind = ad.kind;
      if (LV >= 1 && kind == SDAS_POISSON) {   // (levels >= 1: no KV home or class draws per arrival)
        // the draws of arrival j (M4 gap, M5 P and O) depend on j only: every 32nd arrival, lane k draws
        // those of arrival j + k in parallel into a per-warp queue, so 31 of 32 arrivals cost two loads
        // instead of two Philox chains on the event loop's critical path
        unsigned long long* const gq = reinterpret_cast<unsigned long long*>(Wr + Pk.off_arrq);
        uint32_t* const pq = reinterpret_cast<uint32_t*>(Wr + Pk.off_arrq + 256u);
        if ((j & 31u) == 0u) {
          const uint32_t jj = j + (uint32_t)lane;
          const uint2 w = philox(jj, s_coord, 1u << 16, 0u, key0, key1);
          const uint4 v = philox4(jj, s_coord, 2u << 16, 0u, key0, key1);
          __syncwarp();                                    // the previous block's last reads are done
          gq[lane] = exp_sample(ad.gap0, w.x);
          pq[lane] = uni(ad.p_lo, ad.p_hi, v.x) | (uni(ad.o_lo, ad.o_hi, v.y) << 16);   // both <= 65535
          __syncwarp();
        }
        A_next = A_prev + gq[j & 31u];
        const uint32_t po = pq[j & 31u];
        P_next = po & 0xFFFFu;
        O_next = po >> 16;
        arr_near = A_next - t < 0x80000000ull;
        A_lo = (uint32_t)A_next;
        return;
      }
      if (kind == SDAS_POISSON) {
        const uint2 w = philox(j, s_coord, 1u << 16, 0u, key0, key1);
        A_next = A_prev + exp_sample(ad.gap0, w.x);
      } else if (kind == SDAS_DET) {
        A_next = (unsigned long long)j * ad.gap0;
      } else if (kind == SDAS_LIST) {
        A_next = reinterpret_cast<const unsigned long long*>(blob + ad.list_off)[j];
      } else {  // MMPP2: restart at epoch edges
        A_next = mmpp_next(j, s_coord, A_prev, mm_k, mm_end, ad, key0, key1);
      }
      const uint4 w = philox4(j, s_coord, 2u << 16, 0u, key0, key1);
      P_next = uni(ad.p_lo, ad.p_hi, w.x);
      O_next = uni(ad.o_lo, ad.o_hi, w.y);
      if (kv_role) H_next = (unsigned long long)w.z < Pk.kv_skew32 ? 0u : uni(0u, P.role[kv_role].n - 1u, w.w);
      if (CLS) C_next = (unsigned long long)philox(j, s_coord, 2u << 16, 1u, key0, key1).x < ad.ithr ? 1u : 0u;
      arr_near = A_next - t < 0x80000000ull;
      A_lo = (uint32_t)A_next;
    };
    if (ad.kind == SDAS_MMPP2) {
      const uint2 w = philox(0u, s_coord, 4u << 16, 0u, key0, key1);
      const unsigned long long d = exp_sample(ad.soj0, w.x);
      mm_end = d > 0 ? d : 1ull;
    }
    if (N > 0) gen(0, 0);

    // ---------------------------------------------------------------- routing (M11)
    auto route = [&](uint32_t role, uint32_t slot) -> uint32_t {
      const DRole& R = P.role[role];
      if (LEAN || R.n == 1) return R.first;
      if (kv_role && role == kv_role && cd.kv_policy == SDAS_KV_AFFINITY) return R.first + rHome[slot];  // M22
      uint32_t pol = R.route;
      if ((pol == SDAS_ROUTE_JSQ || pol == SDAS_ROUTE_RR) && cd.route_override != SDAS_ROUTE_NONE)
        pol = cd.route_override;
      if (pol == SDAS_ROUTE_RR) {
        const uint32_t k = __shfl_sync(FULL, rr_l, role);
        if (lane == (int)role) rr_l = k + 1;
        return R.first + k % R.n;
      }
      if (pol == SDAS_ROUTE_FIXED) return R.first + R.route_fixed;
      if (pol == SDAS_ROUTE_SELECT) return __shfl_sync(FULL, sel_l, role);
      uint32_t key = 0xFFFFFFFFu;
      if (lane >= (int)R.first && lane < (int)(R.first + R.n)) {
        const uint32_t load = cd.stale_jsq ? snap : fn + in + (st == RECV ? 1u : 0u) + wn + b;
        key = (load << 4) | (uint32_t)(lane - R.first);
      }
      key = __reduce_min_sync(FULL, key);
      return R.first + (key & 15u);
    };
    // M23: the KV policy charged to an opening message on link l placed at `dest` (0 = none)
    auto kv_kind = [&](uint32_t l, uint32_t dest, uint32_t slot) -> uint32_t {
      if (!kv_role || P.link[l].dst != kv_role || cd.kv_policy < SDAS_KV_RECOMPUTE) return 0u;
      return dest != P.role[kv_role].first + rHome[slot] ? cd.kv_policy : 0u;
    };

    // lane-local: a message due at tick x will enter this instance's inbox while it may be mid-run: end the
    // run at the first step boundary >= x (the cut of M7's RECV-first START, applied when x becomes known)
    // (CHAIN, LEAN: a run may start after the current tick -- at the end of the RECV it follows; a message due
    // before that start cuts it to 0 steps: the instance is idle at the RECV end and RECV-first takes over)
    auto cut_at = [&](uint32_t x) {
      if (st != DECODE || runm <= (CHAIN ? 0u : 1u)) return;
      const uint32_t c = max(1u, MI.tau0 + MI.gamma * b);
      const uint32_t rs = end_lo - runm * c;
      const uint32_t mp = CHAIN && (int32_t)(x - rs) <= 0 ? 0u : div_rcp(x - rs + c - 1u, c, P.rcp_step[lane][b]);
      if (mp < runm) {
        runm = mp;
        end_lo = rs + mp * c;
      }
    };
    // M30 pacing gap of link l under this candidate (0 = unpaced)
    auto pace_gap = [&](uint32_t l) -> uint32_t { return cd.pace == 0xFFFFFFFFu ? P.link[l].gap : cd.pace; };
    // one message into destination `dest`'s in-flight ring (uniform; used by the serial paths)
    auto push_msg = [&](uint32_t l, uint32_t dest, uint32_t slot, uint32_t tokens, uint32_t flags, uint32_t n_in) {
      const uint32_t net = P.link[l].net;
      if (TRACE)
        trace(TR_EMIT, dest, rJ[slot], tokens | ((flags & 1u) << 16) | (((flags >> 1) & 1u) << 17) | (l << 20));
      const DInst& D = P.inst[dest];
      const uint32_t fn_d = __shfl_sync(FULL, fn, dest);
      if (K1_UNLIKELY(fn_d >= D.flight_cap)) {
        if (TRACE) trace(TR_OVERFLOW, 1, dest, 0);
        ovf = true;
        return;
      }
      const uint32_t pm_d = min(D.flight_cap, RS);
      const uint32_t idx = wrap_add(__shfl_sync(FULL, fh, dest), fn_d, pm_d);
      uint32_t tick = t_lo + net;
      if (need_pace) {                     // M30: dispatch at max(t, previous dispatch + gap)
        const uint32_t gp = pace_gap(l);
        if (gp) {
          uint32_t tk = 0;
          if (lane == 0) {
            const unsigned long long d = max(t, H->pace_free[l]);
            H->pace_free[l] = d + gp;
            tk = (uint32_t)d + net;
          }
          tick = __shfl_sync(FULL, tk, 0);
        }
      }
      if (lane == 0) {
        if (!SPILL || fn_d < pm_d) {
          at<uint32_t>(Wr, D.off_ftick)[idx] = tick;
          at<unsigned long long>(Wr, D.off_fbody)[idx] = make_body(slot, flags, tokens, n_in);
          if (kv_role && P.link[l].dst == kv_role)          // M23 HINT: the transfer starts at routing
            at<uint32_t>(Wr, D.off_fbody + 8u * D.flight_cap)[idx] = t_lo + Pk.kv_tau * Pk.kv_ctx;
        } else {                                            // past the shared-memory part: extension
          const uint32_t gi = wrap_add(H->gh[1][dest], fn_d - RS, D.flight_cap - RS);
          reinterpret_cast<uint32_t*>(gxa(D.gx_ftick))[gi] = tick;
          reinterpret_cast<unsigned long long*>(gxa(D.gx_fbody))[gi] = make_body(slot, flags, tokens, n_in);
        }
      }
      if (lane == (int)dest) {
        if (fn == 0) fhead = tick;
        ++fn;
        if (LAZY) cut_at(tick);                            // the delivery will not be an event of its own
        if (SILENT && st == RECV && (int32_t)(tick - end_lo) < 0) runm = 1u;
      }
    };

    // ---------------------------------------------------------------- completion (M13, M18)
    auto request_complete = [&](uint32_t slot) {
      --nsys;
      if (lane == 0) {                     // counters and the record: lane 0 owns them
        const unsigned long long e2e = t - rA[slot], ff = rFF[slot];
        const uint32_t f32 = sat32(ff), e32 = sat32(e2e);
        WarpHdr& h = *H;
        if (e2e >= 0xFFFFFFFFull || ff >= 0xFFFFFFFFull) ++h.n_sat;   // a field holds the sentinel (R-SAT)
        rec[h.completed] = (unsigned long long)e32 | ((unsigned long long)f32 << 32);
        if (CLS) {                         // M29 per-class metrics
          const uint32_t ci = rCls[slot];
          rec_cls[h.completed] = (uint8_t)ci;
          if (ci) {
            ++h.completed_int;
            h.sum_e2e_int += e2e;
            h.good_int += e2e <= Pk.slo ? 1u : 0u;
          }
        }
        ++h.completed;
        h.sum_e2e += e2e;
        h.sum_ff += ff;                    // exact (M19)
        h.max_e2e = max(h.max_e2e, e32);
        h.good += e2e <= Pk.slo ? 1u : 0u;
        ++h.w_n;
        const unsigned long long ps = cd.policy_slo;
        h.w_good += e2e <= ps ? 1u : 0u;
        h.w_half += 2ull * e2e <= ps ? 1u : 0u;
        if (TRACE) trace(TR_REQ_DONE, rJ[slot], e32, f32);
        bitmap[slot >> 5] |= 1u << (slot & 31);
      }
    };
    auto item_done = [&](uint32_t slot) {  // uniform: one item of request `slot` completes
      uint32_t o = 0;
      if (lane == 0) {
        o = rO[slot] - 1u;
        rO[slot] = o;
      }
      o = __shfl_sync(FULL, o, 0);
      if (o == 0) request_complete(slot);
    };

    // ---------------------------------------------------------------- phase COMPLETE: RECV (M8, M10)
    auto complete_recv = [&](uint32_t i) {
      const DInst& I = P.inst[i];
      const uint32_t role = LEAN ? i : I.role;      // LEAN: instance i is role i's only instance
      const DRole& R = P.role[role];
      const unsigned long long body = __shfl_sync(FULL, cur, i);
      // (the wait-ring position is read beside the message body, not behind the branches on it)
      const uint32_t wn_i = __shfl_sync(FULL, wn, i), wh_i = __shfl_sync(FULL, wh, i);
      const uint32_t slot = (uint32_t)(body & 0xFFFFu), flags = (uint32_t)(body >> 16) & 0xFFu;
      if (TRACE) trace(TR_RECV_DONE, i, rJ[slot], flags);
      uint32_t out = 0;
      if (flags & F_CLOSES) {
        if (role == 0) {
          out = rOut[slot];
        } else {
          const uint32_t n_in = (uint32_t)(body >> 48);
          const unsigned long long prod = (unsigned long long)n_in * R.out_num;
          const unsigned long long o64 =
              R.out_fixed + (R.out_den == 1 ? prod
                             : (prod < 0xFFFFFFFFull ? (unsigned long long)(R.out_den < 256u
                                                                                ? div_rcp((uint32_t)prod, R.out_den, P.rcp_fn[R.out_den])
                                                                                : (uint32_t)prod / R.out_den)
                                                     : prod / R.out_den));
          out = o64 > 65535ull ? 65535u : (uint32_t)o64;
        }
      }
      if (lane == (int)i) {
        st = IDLE;
        ++cnt_recv;
      }
      if (!(flags & F_CLOSES)) return;
      if (out > 0) {
        if (K1_UNLIKELY(wn_i >= I.wait_cap)) {
          if (TRACE) trace(TR_OVERFLOW, 2, i, 0);
          ovf = true;
          return;
        }
        if (CLS && prio && rCls[slot]) {   // M27: interactive items wait in the class-1 ring
          const uint32_t idx = wrap_add(__shfl_sync(FULL, wh1, i), __shfl_sync(FULL, wn1, i), I.wait_cap);
          if (lane == 0) at<uint32_t>(Wr, I.off_wait)[I.wait_cap + idx] = slot | (out << 16);
          if (lane == (int)i) ++wn1;
        } else {
          const uint32_t pmw = min(I.wait_cap, RS), k = wn_i - (CLS ? __shfl_sync(FULL, wn1, i) : 0u);
          const uint32_t idx = wrap_add(wh_i, k, pmw);
          if (lane == 0) {
            if (!SPILL || k < pmw) at<uint32_t>(Wr, I.off_wait)[idx] = slot | (out << 16);
            else reinterpret_cast<uint32_t*>(gxa(I.gx_wait))[wrap_add(H->gh[2][i], k - RS, I.wait_cap - RS)] =
                     slot | (out << 16);
          }
        }
        if (lane == (int)i) ++wn;
        if (TRACE) trace(TR_ITEM_WAIT, i, rJ[slot], out);
        return;
      }
      // tool item (out = 0): one 0-token message per out-link, then complete now (M9)
      for (uint32_t q = 0; q < R.n_out; ++q) {
        const uint32_t l = q ? R.out_link1 : R.out_link0;
        const uint32_t dest = route(P.link[l].dst, slot);
        if (lane == 0) rO[slot] += 1u;
        push_msg(l, dest, slot, 0u, F_OPENS | F_CLOSES | (kv_kind(l, dest, slot) << 2), 0u);
        if (K1_UNLIKELY(ovf)) return;
      }
      __syncwarp();                        // lane 0's ring writes precede the destinations' DELIVER reads
      // first feedback = the earliest first-output tick of the request's items (M13); a DECODE item may have
      // recorded a later one in advance (coalesced runs), so take the minimum
      if (lane == 0 && role == ((modes >> 28) & 7u)) rFF[slot] = min(rFF[slot], t - rA[slot]);
      if (P.inst[i].flags & 1u) { if (lane == (int)i) ++n_large; }
      item_done(slot);
    };


    // ---------------------------------------------------------------- phase COMPLETE: DECODE (M7, M9, M13)
    auto complete_decode = [&](uint32_t i) {
      const DInst& I = P.inst[i];
      const uint32_t role = LEAN ? i : I.role;      // LEAN: instance i is role i's only instance
      const DRole& R = P.role[role];
      const uint32_t bi = __shfl_sync(FULL, b, i);
      const uint32_t mi = __shfl_sync(FULL, runm, i);          // steps in this run (all but the last silent)
      const bool me = lane == (int)i;
      st = me ? IDLE : st;
      cnt_decode += me ? mi : 0u;
      tok += me ? (unsigned long long)mi * bi : 0ull;
      if (TRACE && mi > 1) {
        const uint32_t c = max(1u, I.tau0 + I.gamma * bi);
        trace_silent(i, bi, c, t - (unsigned long long)mi * c, mi - 1u, true);
      }
      if (TRACE) trace(TR_DECODE_DONE, i, bi, 0);
      uint32_t* const bat = at<uint32_t>(Wr, I.off_batch);
      const bool act = lane < (int)bi;
      const uint32_t n_out = R.n_out;
      // all 32 slots are loaded (slots >= bi hold stale words that are never observed)
      uint32_t wA = bat[lane], wB = bat[32 + lane], wD = 0;
      if (MAXOUT > 1) wD = bat[96 + lane];
      const uint32_t slot = wA & 0xFFFu, out = wA >> 16;
      const uint32_t done = (wB & 0xFFFFu) + mi;
      wB = (wB & 0xFFFF0000u) | done;
      // emission test (M9): link q emits when done reaches its next emission point
      const bool e0 = act && n_out > 0 && done == (wB >> 16);
      const bool e1 = MAXOUT > 1 && act && n_out > 1 && done == (wD & 0xFFFFu);
      const uint32_t m0 = __ballot_sync(FULL, e0);
      const uint32_t m1 = MAXOUT > 1 ? __ballot_sync(FULL, e1) : 0u;
      // (issued beside the emission votes: the emissions below change neither done nor out)
      const uint32_t fin = __ballot_sync(FULL, act && done == out);
      uint32_t wC = 0, wE = 0;
      if (m0 | m1) {
        wC = bat[64 + lane];
        if (MAXOUT > 1) wE = bat[128 + lane];
        for (int q = 0; q < MAXOUT; ++q) {
          const uint32_t mq = q ? m1 : m0;
          if (!mq) continue;
          const bool eq = q ? e1 : e0;
          const uint32_t l = q ? R.out_link1 : R.out_link0;
          const uint32_t mode = (wA >> (12 + 2 * q)) & 3u;
          uint32_t tokens = 0, flags = 0, n_in = 0, sticky = 0;
          if (eq) {
            const uint32_t prev = q ? (wD >> 16) : (wC & 0xFFFFu);
            const uint32_t next = q ? (wD & 0xFFFFu) : (wB >> 16);
            uint32_t fidx = q ? (wE & 0xFFu) : ((wC >> 16) & 0xFFu);
            sticky = q ? ((wE >> 8) & 0xFFu) : (wC >> 24);
            tokens = next - prev;
            const bool tm = mode == SDAS_TOKEN;
            flags = (tm ? (prev == 0 ? 1u : 0u) : 1u) | ((tm ? (next == out ? 1u : 0u) : 1u) << 1);
            n_in = tm ? out : tokens;
            uint32_t nx = out;
            if (mode == SDAS_FUNCTION) {
              ++fidx;
              const uint32_t Fp = min(R.n_functions, out);
              nx = div_rcp((fidx + 1u) * out, Fp, P.rcp_fn[Fp])   /* < 2^24: fidx < 256, out < 2^16 */;
            } else if (tm) {
              nx = min(next + P.link[l].chunk, out);
            }
            if (q == 0) {
              wB = (wB & 0xFFFFu) | (nx << 16);
              wC = next | (fidx << 16) | (wC & 0xFF000000u);
            } else {
              wD = nx | (next << 16);
              wE = fidx | (wE & 0xFF00u);
            }
          }
          const DRole& Rd = P.role[P.link[l].dst];
          const bool single = LEAN || Rd.n == 1;
          const uint32_t openers = LEAN ? 0u : __ballot_sync(FULL, eq && (flags & 1u));
          if (single || openers == 0) {
            // every message of this link goes to a known instance: place them in parallel
            // (per-destination order = batch order; M9/M11 sticky continuations)
            const uint32_t dest_single = LEAN ? P.link[l].dst : Rd.first;   // LEAN: role r = instance r
            uint32_t dest = (single || (flags & 1u)) ? dest_single : sticky;
            if (single && eq && (flags & 1u)) sticky = dest_single;
            // M30 pacing: the link's messages of this step leave in batch order, gp apart
            uint32_t gp = 0;
            unsigned long long d0 = t;
            if (need_pace) {
              gp = pace_gap(l);
              if (gp) d0 = max(t, H->pace_free[l]);
            }
            const uint32_t my_tick =
                t_lo + P.link[l].net + (gp ? (uint32_t)(d0 - t) + (uint32_t)__popc(mq & lanemask_lt()) * gp : 0u);
            // group lanes by destination (continuations may target different instances)
            uint32_t todo = mq;
            while (todo) {
              const uint32_t dk = __shfl_sync(FULL, dest, __ffs(todo) - 1);
              const uint32_t grp = __ballot_sync(FULL, eq && dest == dk) & todo;
              todo &= ~grp;
              const uint32_t fn_d = __shfl_sync(FULL, fn, dk), fh_d = __shfl_sync(FULL, fh, dk);
              const DInst& D = P.inst[dk];
              const uint32_t cnt = __popc(grp);
              if (K1_UNLIKELY(fn_d + cnt > D.flight_cap)) {
                if (TRACE) trace(TR_OVERFLOW, 1, dk, 0);
                ovf = true;
                return;
              }
              const uint32_t tick = __shfl_sync(FULL, my_tick, __ffs(grp) - 1);   // group's first message
              if ((grp >> lane) & 1u) {
                const uint32_t k = fn_d + __popc(grp & lanemask_lt()), pm_d = min(D.flight_cap, RS);
                if (!SPILL || k < pm_d) {
                  const uint32_t idx = wrap_add(fh_d, k, pm_d);
                  at<uint32_t>(Wr, D.off_ftick)[idx] = my_tick;
                  at<unsigned long long>(Wr, D.off_fbody)[idx] = make_body(slot, flags, tokens, n_in);
                } else {                                     // past the shared-memory part: extension
                  const uint32_t gi = wrap_add(H->gh[1][dk], k - RS, D.flight_cap - RS);
                  reinterpret_cast<uint32_t*>(gxa(D.gx_ftick))[gi] = my_tick;
                  reinterpret_cast<unsigned long long*>(gxa(D.gx_fbody))[gi] = make_body(slot, flags, tokens, n_in);
                }
                if (flags & 1u) atomicAdd(&rO[slot], 1u);          // M13: +1 per opening message
                if (TRACE) trace_lane(TR_EMIT, dk, rJ[slot], tokens | ((flags & 1u) << 16) | (((flags >> 1) & 1u) << 17) | (l << 20));
              }
              if (lane == (int)dk) {
                if (fn == 0) fhead = tick;
                fn += cnt;
                if (LAZY) cut_at(tick);                    // the delivery will not be an event of its own
                if (SILENT && st == RECV && (int32_t)(tick - end_lo) < 0) runm = 1u;   // re-arm a silent RECV
              }
            }
            __syncwarp();
            if (gp && lane == 0) H->pace_free[l] = d0 + (unsigned long long)__popc(mq) * gp;
          } else {
            // openings need sequential routing (JSQ sees every earlier placement, M11)
            uint32_t todo = mq;
            while (todo) {
              const int k = __ffs(todo) - 1;
              todo &= todo - 1;
              const uint32_t fk = __shfl_sync(FULL, flags, k), tk = __shfl_sync(FULL, tokens, k);
              const uint32_t nk = __shfl_sync(FULL, n_in, k), sk = __shfl_sync(FULL, slot, k);
              uint32_t dk = __shfl_sync(FULL, sticky, k);
              uint32_t fkv = fk;
              if (fk & 1u) {
                dk = route(P.link[l].dst, sk);
                if (lane == 0) rO[sk] += 1u;
                if (lane == k) sticky = dk;
                fkv |= kv_kind(l, dk, sk) << 2;
              }
              push_msg(l, dk, sk, tk, fkv, nk);
              if (K1_UNLIKELY(ovf)) return;
            }
            __syncwarp();                  // lane 0's ring writes precede the destinations' DELIVER reads
          }
          if (eq) {
            if (q == 0) wC = (wC & 0x00FFFFFFu) | (sticky << 24);
            else wE = (wE & 0xFFu) | (sticky << 8);
          }
        }
      }
      if (!coalesce && role == ((modes >> 28) & 7u)) {  // first output token at a feedback-role instance (M13)
        // (two items of one request may both reach done == 1 in this step: the CAS lets the first set it;
        // coalesced runs recorded it when the run started)
        if (act && done == 1u) atomicCAS(&rFF[slot], kUnsetFF, t - rA[slot]);
        __syncwarp();
      }
      if (!fin) {  // common case: write the advanced words back in place (stale slots included)
        bat[32 + lane] = wB;
        if (m0 | m1) {
          bat[64 + lane] = wC;
          if (MAXOUT > 1) { bat[96 + lane] = wD; bat[128 + lane] = wE; }
        }
        return;
      }
      n_large += (me && my_large) ? (uint32_t)__popc(fin) : 0u;
      uint32_t fm = fin;
      while (fm) {
        const int k = __ffs(fm) - 1;
        fm &= fm - 1;
        item_done(__shfl_sync(FULL, slot, k));
      }
      const bool keep = act && done != out;
      const uint32_t km = __ballot_sync(FULL, keep);
      if (!(m0 | m1)) {
        wC = bat[64 + lane];
        if (MAXOUT > 1) wE = bat[128 + lane];
      }
      __syncwarp();
      if (keep) {  // stable compaction
        const uint32_t nk = __popc(km & lanemask_lt());
        bat[nk] = wA;
        bat[32 + nk] = wB;
        bat[64 + nk] = wC;
        if (MAXOUT > 1) { bat[96 + nk] = wD; bat[128 + nk] = wE; }
      }
      __syncwarp();
      b = me ? (uint32_t)__popc(km) : b;
    };

    // ---------------------------------------------------------------- phase START (M7)
    auto start_recv = [&](uint32_t i) -> uint32_t {  // RECV-first: instance i pops its inbox head
      __syncwarp();                       // rNit / rJ written by other lanes earlier in this tick
      uint32_t cost32 = 0, slot = 0, toff = 0;
      if (lane == (int)i) {
        const bool from1 = CLS && in1 != 0u;                  // M27: interactive messages first
        const unsigned long long body =
            reinterpret_cast<unsigned long long*>(my_inbox)[from1 ? my_inbox_cap + ih1 : ih];
        slot = (uint32_t)(body & 0xFFFFu);
        const uint32_t flags = (uint32_t)(body >> 16) & 0xFFu;
        const uint32_t tokens = (uint32_t)(body >> 32) & 0xFFFFu;
        unsigned long long cost = (unsigned long long)MI.h + (unsigned long long)MI.beta * tokens;
        if (flags & F_OPENS) {
          const uint32_t ord = rNit[slot];
          rNit[slot] = (uint16_t)(ord + 1u);
          unsigned long long a = MI.alpha;
          if (MI.flags & 2u) {
            const uint2 w = philox(rJ[slot], s_coord, (3u << 16) | my_role, ord, key0, key1);
            a = exp_sample(MI.alpha, w.x);
          }
          cost += a;
          const uint32_t kvk = LV ? 0u : (flags >> 2) & 7u;   // levels >= 1 never model KV
          if (kvk) {  // M23: KV penalty of an opening RECV away from the request's KV home
            unsigned long long pen;
            if (kvk == SDAS_KV_RECOMPUTE) pen = (unsigned long long)MI.beta * Pk.kv_ctx;
            else if (kvk == SDAS_KV_POSTHOC) pen = (unsigned long long)Pk.kv_tau * Pk.kv_ctx;
            else pen = (uint32_t)max(0, (int32_t)(my_iready[ih] - t_lo));
            cost += pen;
            ++cnt_kv;
          }
        }
        if (cost < 1) cost = 1;
        cost32 = (uint32_t)cost;
        st = RECV;
        end_lo = t_lo + cost32;
        cur = body;
        if (from1) {
          ih1 = wrap_add(ih1, 1u, my_inbox_cap);
          --in1;
        } else {
          const uint32_t oih = ih;
          ih = wrap_add(ih, 1u, my_inbox_cap);
          if (SPILL && in > my_inbox_cap) {   // refill the vacated slot with the oldest extension entry
            const uint32_t g0 = H->gh[0][lane];
            reinterpret_cast<unsigned long long*>(my_inbox)[oih] =
                reinterpret_cast<const unsigned long long*>(gxa(MI.gx_inbox))[g0];
            H->gh[0][lane] = (uint16_t)wrap_add(g0, 1u, MI.inbox_cap - RS);
          }
        }
        --in;
        // SILENT (runm = 0 while in RECV): a non-closing message whose RECV end leaves nothing to start (no
        // inbox, wait or batch, no delivery due before it) only makes the instance idle: that happens at its
        // next event instead (busy is integrated up to end_lo, a delivery emitted for before end_lo re-arms it)
        const bool alone = SILENT && !((body >> 17) & 1u) && in == 0u;
        runm = (alone && wn == 0u && b == 0u && (fn == 0u || (int32_t)(fhead - end_lo) >= 0)) ? 0u : 1u;
        // CHAIN: the same message received while the instance holds a batch (RECV-first cut
        // the batch's run): with nothing due before the RECV ends and nothing to admit then (no waiting item,
        // or a full batch and no window close -- a possible B change -- up to the RECV end), the batch's next
        // run starts exactly then, so start_decode computes it now from that tick and the RECV end is no event
        // (a non-closing RECV completes with nothing but the count, M8)
#ifdef K1_COUNT_ITERS
        if (SILENT && !((body >> 17) & 1u) && b != 0u) {   // experiment: why a chain candidate fails
          atomicAdd(&work->pad[16], 1ull);
          if (in != 0u) atomicAdd(&work->pad[17], 1ull);
          if (!(wn == 0u || (b >= Bk && (int32_t)(nb_lo - end_lo) > 0))) atomicAdd(&work->pad[18], 1ull);
          if (!(fn == 0u || (int32_t)(fhead - end_lo) > 0)) atomicAdd(&work->pad[19], 1ull);
          if (wn != 0u) atomicAdd(&work->pad[20], 1ull);
        }
#endif
        if (CHAIN && alone && b != 0u && (wn == 0u || (b >= Bk && (int32_t)(nb_lo - end_lo) > 0)) &&
            (fn == 0u || (int32_t)(fhead - end_lo) > 0) && cost32 < (1u << 29)) {
          toff = cost32;
          ++cnt_recv;
        }
      }
      if (TRACE) trace(TR_RECV_START, i, rJ[__shfl_sync(FULL, slot, i)], __shfl_sync(FULL, cost32, i));
      return CHAIN ? __shfl_sync(FULL, toff, i) : 0u;
    };
    // AHEAD: emit now the messages of the emission points the source instance i passes at
    // steps 1 .. m-1 of its run (step k's messages carry emission tick t + k c, in batch order, M9); the
    // net delay is below one step, so at each emission tick the destination's in-flight ring holds exactly
    // that step's messages (M14); a step whose messages do not fit next to the ring's current content ends
    // the run there (its messages are then emitted by complete_decode, with the exact overflow test).
    // Returns the (possibly shorter) run length.  Lanes < nbat hold the batch words wA, wB.
    auto emit_ahead = [&](uint32_t i, const DRole& R, uint32_t nbat, uint32_t cost32, uint32_t m, uint32_t wA,
                          uint32_t wB) -> uint32_t {
      const uint32_t l = R.out_link0;                       // the destination role has one instance
      const uint32_t dk = LEAN ? P.link[l].dst : P.role[P.link[l].dst].first;
      const DInst& D = P.inst[dk];
      uint32_t* const bat = at<uint32_t>(Wr, P.inst[i].off_batch);
      const bool act = lane < (int)nbat;
      const uint32_t out = wA >> 16, mode = (wA >> 12) & 3u, slot = wA & 0xFFFu;
      const uint32_t done0 = wB & 0xFFFFu;
      uint32_t nxt = wB >> 16;
      uint32_t wC = act ? bat[64 + lane] : 0u;
      uint32_t prev = wC & 0xFFFFu, fidx = (wC >> 16) & 0xFFu;
      const uint32_t chunk = P.link[l].chunk, Fp = min(R.n_functions, out), net = P.link[l].net;
      uint32_t fn_d = __shfl_sync(FULL, fn, dk);
      const uint32_t fh_d = __shfl_sync(FULL, fh, dk), pm_d = min(D.flight_cap, RS);
      bool moved = false;
      for (;;) {
        const uint32_t s = (act && nxt < out) ? nxt - done0 : 0xFFFFFFFFu;   // step of the next emission
        const uint32_t k = __reduce_min_sync(FULL, s);
        if (k >= m) break;                                 // at the run end or beyond: complete_decode
        const uint32_t em = __ballot_sync(FULL, s == k);
        const uint32_t cnt = __popc(em);
        if (fn_d + cnt > D.flight_cap) { m = k; break; }   // no room next to the ring's content: end here
        const uint32_t tick = t_lo + k * cost32 + net;
        if (s == k) {
          const bool tm = mode == SDAS_TOKEN;
          const uint32_t tokens = nxt - prev;
          const uint32_t flags = (tm ? (prev == 0 ? 1u : 0u) : 1u) | ((tm ? (nxt == out ? 1u : 0u) : 1u) << 1);
          const uint32_t n_in = tm ? out : tokens;
          const uint32_t q = fn_d + __popc(em & lanemask_lt());
          const unsigned long long body = make_body(slot, flags, tokens, n_in);
          if (!SPILL || q < pm_d) {
            const uint32_t idx = wrap_add(fh_d, q, pm_d);
            at<uint32_t>(Wr, D.off_ftick)[idx] = tick;
            at<unsigned long long>(Wr, D.off_fbody)[idx] = body;
          } else {
            const uint32_t gi = wrap_add(H->gh[1][dk], q - RS, D.flight_cap - RS);
            reinterpret_cast<uint32_t*>(gxa(D.gx_ftick))[gi] = tick;
            reinterpret_cast<unsigned long long*>(gxa(D.gx_fbody))[gi] = body;
          }
          if (flags & 1u) atomicAdd(&rO[slot], 1u);       // M13: +1 per opening message
          prev = nxt;
          if (mode == SDAS_FUNCTION) {
            ++fidx;
            nxt = div_rcp((fidx + 1u) * out, Fp, P.rcp_fn[Fp])   /* < 2^24: fidx < 256, out < 2^16 */;
          } else {                                          // TOKEN (BATCH emits at the end only)
            nxt = min(nxt + chunk, out);
          }
        }
        if (lane == (int)dk) {
          if (fn == 0) fhead = tick;
          fn += cnt;
          cut_at(tick);
          if (SILENT && st == RECV && (int32_t)(tick - end_lo) < 0) runm = 1u;   // re-arm a silent RECV
        }
        fn_d += cnt;
        moved = true;
      }
      if (moved) {
        if (act) {
          bat[32 + lane] = done0 | (nxt << 16);
          bat[64 + lane] = prev | (fidx << 16) | (dk << 24);
        }
        __syncwarp();
      }
      return m;
    };
    // toff > 0 (CHAIN): the run starts toff ticks from now, when the RECV started this tick ends (no admission:
    // nothing waits)
    auto start_decode = [&](uint32_t i, uint32_t toff) {  // FIFO admission (modes bound here, M9) + DECODE step / run
      const uint32_t ts = t_lo + toff;                      // the run's start tick
      const DInst& I = P.inst[i];
      const uint32_t role = LEAN ? i : I.role;
      const DRole& R = P.role[role];
      const uint32_t bi = __shfl_sync(FULL, b, i), Bi = __shfl_sync(FULL, Bk, i);
      const uint32_t wn_i = __shfl_sync(FULL, wn, i);
      const uint32_t nadm = Bi > bi ? min(Bi - bi, wn_i) : 0u;
      const uint32_t n_out = R.n_out;
      uint32_t* const bat = at<uint32_t>(Wr, I.off_batch);
      uint32_t wA = 0, wB = 0, wD = 0;
      uint32_t n1 = 0;                                    // admitted from the class-1 ring (M27)
      if (nadm) {
        const uint32_t wh_i = __shfl_sync(FULL, wh, i);
        uint32_t wh1_i = 0;
        if (CLS) {
          n1 = min(nadm, __shfl_sync(FULL, wn1, i));
          wh1_i = __shfl_sync(FULL, wh1, i);
        }
        if (lane >= (int)bi && lane < (int)(bi + nadm)) {
          const uint32_t k = lane - bi;
          const uint32_t* const wr = at<uint32_t>(Wr, I.off_wait);
          const uint32_t e = (CLS && k < n1) ? wr[I.wait_cap + wrap_add(wh1_i, k, I.wait_cap)]
                                             : wr[wrap_add(wh_i, k - n1, min(I.wait_cap, RS))];
          const uint32_t out = e >> 16;
          wA = (e & 0xFFFu) | (out << 16);
          for (uint32_t q = 0; q < n_out; ++q) {
            const uint32_t l = q ? R.out_link1 : R.out_link0;
            const uint32_t mode = (modes >> (2 * l)) & 3u;
            uint32_t next = out;
            if (mode == SDAS_FUNCTION) {
              const uint32_t Fp = min(R.n_functions, out);   // >= 1: batch items have out >= 1
              next = div_rcp(out, Fp, P.rcp_fn[Fp]);
            }
            else if (mode == SDAS_TOKEN) next = min(P.link[l].chunk, out);
            wA |= mode << (12 + 2 * q);
            if (q == 0) wB = next << 16;
            else wD = next;
          }
          bat[lane] = wA;
          bat[32 + lane] = wB;
          bat[64 + lane] = 0xFF000000u;
          if (MAXOUT > 1) { bat[96 + lane] = wD; bat[128 + lane] = 0xFF00u; }
        }
        // every lane reads back only its own batch words; the two-level refill below rewrites wait slots
        // other lanes have just read
        if (SPILL) __syncwarp();
        const uint32_t pmw = min(I.wait_cap, RS);
        if (SPILL && wn_i > pmw) {   // refill the vacated slots with the oldest extension entries
          const uint32_t m = min(nadm, wn_i - pmw), g0 = H->gh[2][i], cx = I.wait_cap - RS;
          if (lane < (int)m)
            at<uint32_t>(Wr, I.off_wait)[wrap_add(wh_i, lane, pmw)] =
                reinterpret_cast<const uint32_t*>(gxa(I.gx_wait))[wrap_add(g0, lane, cx)];
          __syncwarp();
          if (lane == 0) H->gh[2][i] = (uint16_t)wrap_add(g0, m, cx);
        }
      }
      const uint32_t nbat = bi + nadm;
      // branch-free update of instance i (tau0 < 2^31 and gamma*32 < 2^30 are validated: no u32 overflow)
      const bool me = lane == (int)i;
      const uint32_t cost32 = max(1u, I.tau0 + I.gamma * nbat);
      const uint32_t rc = P.rcp_step[i][nbat];           // floor(2^32 / cost32), for the run-length divisions
      // run length: steps until the first sequence reaches an emission point / its end / first feedback.
      // AHEAD: the source role's inbox receives arrivals only, so its run is known up to the
      // next arrival; its emission points do not end the run -- their messages are emitted now, each with
      // its own emission tick, and the run ends at a finish / first feedback / arrival / window bound
      const uint32_t ahead_dst = LEAN ? P.link[R.out_link0].dst : P.role[P.link[R.out_link0].dst].first;
      const bool ahead = LAZY && role == 0 && n_out == 1 && nbat > 0 && P.link[R.out_link0].net < cost32 &&
                         (LEAN || P.role[P.link[R.out_link0].dst].n == 1) && nbat <= P.inst[ahead_dst].flight_cap;
      uint32_t m = 1;
      if (coalesce) {
        uint32_t sk = 0xFFFFFFFFu;
        if (lane < (int)bi) {
          wA = bat[lane];
          wB = bat[32 + lane];
          if (MAXOUT > 1) wD = bat[96 + lane];
        }
        if (!TRACE) {                      // silent steps of a run cut exactly at a boundary (cut_run)
          const uint32_t fl = __shfl_sync(FULL, flushm, i);
          if (fl) {
            if (lane < (int)bi) bat[32 + lane] = wB += fl;   // done += fl (stays below every stop point)
            flushm = lane == (int)i ? 0u : flushm;
          }
        }
        if (lane < (int)nbat) {
          const uint32_t done = wB & 0xFFFFu;
          uint32_t lim = wA >> 16;                                      // out
          if (n_out > 0 && !ahead) lim = min(lim, wB >> 16);
          if (MAXOUT > 1 && n_out > 1) lim = min(lim, wD & 0xFFFFu);
          // a sequence's first token lands at the end of this run's first step, known now, so the
          // first feedback (M13: the earliest such tick of the request) is recorded now and is no stop
          // point; rFF is read only when the request completes, after every one of its items finished
          const bool first = role == ((modes >> 28) & 7u) && done == 0u;
          if (first) atomicMin(&rFF[wA & 0xFFFu], t + toff + cost32 - rA[wA & 0xFFFu]);
          sk = lim - done;
        }
        if (LV) {
          // every run bound is a minimum, so they are computed beside the warp-min instead of one after the
          // other behind it: keep every pending tick < 2^31 ahead (min(m, max(1, 2^30 / c)) is the cap); end
          // at the first boundary >= a pending delivery (LAZY), >= the next window when the controller could
          // change B while items wait, >= the next arrival (AHEAD)
          uint32_t bnd = max(1u, div_rcp(1u << 30, cost32, rc));
          if (LAZY) {
            const uint32_t fn_i = __shfl_sync(FULL, fn, i), fh_i = __shfl_sync(FULL, fhead, i);
            if (fn_i) bnd = min(bnd, max(1u, div_rcp(fh_i - ts + cost32 - 1u, cost32, rc)));
          }
          if ((modes >> 31) && wn_i > nadm) bnd = min(bnd, div_rcp(nb_lo - ts + cost32 - 1u, cost32, rc));
          if (ahead && arr_near) bnd = min(bnd, max(1u, div_rcp(A_lo - ts + cost32 - 1u, cost32, rc)));
          m = __reduce_min_sync(FULL, sk);
          if (m > 1) m = min(m, bnd);
        } else {
        m = __reduce_min_sync(FULL, sk);
        if (m > 1) {
          // keep every pending tick < 2^31 ahead; end at the first boundary >= the next window when the
          // controller could change B while items wait; never step past max_ticks
          if ((unsigned long long)m * cost32 >= (1ull << 30)) m = max(1u, div_rcp(1u << 30, cost32, rc));
          if (LAZY) {                                      // end at the first boundary >= a pending delivery
            const uint32_t fn_i = __shfl_sync(FULL, fn, i), fh_i = __shfl_sync(FULL, fhead, i);
            if (fn_i) m = min(m, max(1u, div_rcp(fh_i - ts + cost32 - 1u, cost32, rc)));
          }
          const uint32_t span = m * cost32;
          if ((modes >> 31) && wn_i > nadm) {
            const uint32_t nbd = nb_lo - ts;
            if (span > nbd) m = div_rcp(nbd + cost32 - 1u, cost32, rc);
          }
          if (max_ticks && t + span > max_ticks)
            m = (uint32_t)max(1ull, (max_ticks - min(t, max_ticks)) / cost32);
          if (ahead && arr_near) m = min(m, max(1u, div_rcp(A_lo - ts + cost32 - 1u, cost32, rc)));   // next arrival
        }
        }
        if (ahead && m > 1) m = emit_ahead(i, R, nbat, cost32, m, wA, wB);
      }
      wh = me ? wrap_add(wh, nadm - n1, my_wait_cap) : wh;
      wn = me ? wn - nadm : wn;
      if (CLS) {
        wh1 = me ? wrap_add(wh1, n1, my_wait_cap) : wh1;
        wn1 = me ? wn1 - n1 : wn1;
      }
      b = me ? nbat : b;
      const bool go = me && nbat > 0;
      st = go ? (uint32_t)DECODE : st;
      end_lo = go ? ts + m * cost32 : end_lo;
      runm = go ? m : runm;
      if (TRACE && nbat > 0) trace(TR_DECODE_START, i, nbat, cost32);
    };
    // lane-local: a message / arrival enters this instance's inbox at tick t while it may be mid-run
    auto cut_run = [&]() {
      if (st != DECODE || runm <= (CHAIN ? 0u : 1u)) return;
      const uint32_t c = max(1u, MI.tau0 + MI.gamma * b);
      const uint32_t rs = end_lo - runm * c;                 // run start (>= 1 tick ago; CHAIN: maybe ahead)
      const uint32_t mp = CHAIN && (int32_t)(t_lo - rs) <= 0 ? 0u
                                                             : div_rcp(t_lo - rs + c - 1u, c, P.rcp_step[lane][b]);   // first boundary >= t
      if (mp >= runm) return;
      if (rs + mp * c != t_lo) {
        runm = mp;
        end_lo = rs + mp * c;
      } else if (TRACE) {                                    // boundary at this very tick: flush it
        flushm = mp;
        runm = mp;
        end_lo = t_lo;
      } else {                                               // boundary at this very tick: the run ends
        st = IDLE;
        cnt_decode += mp;
        tok += (unsigned long long)mp * b;
        flushm = mp;                                         // done += mp: at the next start_decode
      }
    };

    // ---------------------------------------------------------------- phase ARRIVE (M14)
    auto arrive = [&]() {
      const uint32_t j = jn;
      if (CLS && gate && !C_next) {       // M28: interactive-only admission rejects a background request
        if (lane == 0) {
          ++H->dropped;
          ++H->rejected;
        }
        if (TRACE) trace(TR_ARRIVE, j, 2, 0xFFFFFFFFu);
      } else if (nsys >= R_cap) {
        if (lane == 0) ++H->dropped;
        if (TRACE) trace(TR_ARRIVE, j, 0, 0xFFFFFFFFu);
      } else {
        if (lane == 0) ++H->admitted;
        ++nsys;
        __syncwarp();
        const uint32_t wv = lane < (int)Pk.bitmap_words ? bitmap[lane] : 0u;   // lowest free slot
        const uint32_t wm = __ballot_sync(FULL, wv != 0);
        const int wi = __ffs(wm) - 1;
        const uint32_t word = __shfl_sync(FULL, wv, wi);
        const uint32_t bit = __ffs(word) - 1;
        const uint32_t slot = (uint32_t)wi * 32u + bit;
        __syncwarp();                     // every lane's bitmap read precedes lane 0's update
        if (lane == 0) {
          bitmap[wi] = word & ~(1u << bit);
          rA[slot] = t;
          rFF[slot] = kUnsetFF;
          rJ[slot] = j;
          rO[slot] = 1u;                  // M13: +1 on admission
          rNit[slot] = 0;
          rOut[slot] = (uint16_t)O_next;
          rHome[slot] = (uint8_t)H_next;
          if (CLS) rCls[slot] = (uint8_t)C_next;
        }
        const uint32_t dest = route(0, slot);
        if (TRACE) trace(TR_ARRIVE, j, 1, dest);
        const bool bad = lane == (int)dest && in >= my_inbox_cap && (!SPILL || in >= MI.inbox_cap);
        if (lane == (int)dest && !bad) {
          unsigned long long* const ib = reinterpret_cast<unsigned long long*>(my_inbox);
          const unsigned long long body = make_body(slot, F_OPENS | F_CLOSES, P_next, P_next);
          if (CLS && prio && C_next) {      // M27: class-1 ring
            ib[my_inbox_cap + wrap_add(ih1, in1, my_inbox_cap)] = body;
            ++in1;
          } else {
            const uint32_t k = in - (CLS ? in1 : 0u);
            if (!SPILL || k < my_inbox_cap) ib[wrap_add(ih, k, my_inbox_cap)] = body;
            else reinterpret_cast<unsigned long long*>(gxa(MI.gx_inbox))[wrap_add(H->gh[0][lane], k - RS,
                                                                                 MI.inbox_cap - RS)] = body;
          }
          ++in;
          if (coalesce) cut_run();
        }
        if (K1_UNLIKELY(__any_sync(FULL, bad))) {
          if (TRACE) trace(TR_OVERFLOW, 0, dest, 0);
          ovf = true;
        }
      }
      ++jn;
      if (jn < N) {
        gen(jn, t);
      } else {
        arr_near = false;
        arr_more = false;
      }
    };

    // ---------------------------------------------------------------- window close + control (M15, M16)
    auto control = [&](int32_t q) {
      const uint32_t w_n = H->w_n;
      // M25 (f3): the guarded quantile of this window's completions violates policy_slo
      const bool gviol = cd.guard_links && w_n >= 1 &&
                         H->w_good < (uint32_t)(((unsigned long long)cd.guard_pct * w_n + 99ull) / 100ull);
      for (uint32_t l = 0; l < n_links; ++l) {  // (i) three-band mode policy / (M25) guard, one decision
        const bool ctl = (cd.ctl_links >> l) & 1u, grd = (cd.guard_links >> l) & 1u;
        if (!ctl && !grd) continue;
        uint32_t want;
        if (grd && gviol) {
          want = SDAS_BATCH;
        } else if (ctl) {
          const uint32_t dst = P.link[l].dst;
          const DRole& Rd = P.role[dst];
          const uint32_t rd_first = LEAN ? dst : Rd.first, rd_n = LEAN ? 1u : Rd.n;
          const bool mine = lane >= (int)rd_first && lane < (int)(rd_first + rd_n);
          const unsigned long long u =
              warp_sum64(mine ? (cd.metric_load ? acc_lint : (unsigned long long)acc_busy) : 0ull);
          const unsigned long long lhs = u * 1000ull;
          uint32_t band = 1;
          if (lhs >= (unsigned long long)cd.hi * Pk.window * rd_n) band = 2;
          else if (lhs <= (unsigned long long)cd.lo * Pk.window * rd_n) band = 0;
          want = cd.band[band];
        } else if (w_n >= 1) {
          want = cd.mode[l] == 255 ? P.link[l].mode : cd.mode[l];   // reset to the initial mode
        } else {
          continue;
        }
        const uint32_t curm = (modes >> (2 * l)) & 3u;
        const int32_t ql = __shfl_sync(FULL, qlm, l);
        if (want != curm && q - ql >= (int32_t)cd.dwell) {
          modes = (modes & ~(3u << (2 * l))) | (want << (2 * l));
          if (lane == (int)l) qlm = q;
          if (lane == 0) ++H->mode_switches;
          if (TRACE) trace(TR_CONTROL, 0, l, want);
        }
      }
      bool viol = false, calm = false;
      if (w_n >= 1) {
        const uint32_t k99 = (uint32_t)((99ull * w_n + 99ull) / 100ull);
        viol = H->w_good < k99;
        calm = H->w_half >= k99;
      }
      if (cd.batch_roles && w_n >= 1) {  // (ii) SLO-aware max_num_seqs, lane = instance
        bool changed = false;
        if (is_inst && ((cd.batch_roles >> my_role) & 1u)) {
          uint32_t nbB = Bk;
          if (viol) nbB = acc_qint > (unsigned long long)cd.q_hi * Pk.window ? min(32u, 2u * Bk) : max(1u, Bk / 2u);
          else if (calm) nbB = MI.B_default;
          if (nbB != Bk && q - qlB >= (int32_t)cd.dwell) {
            Bk = nbB;
            qlB = q;
            changed = true;
          }
        }
        uint32_t chm = __ballot_sync(FULL, changed);
        if (lane == 0) H->batch_changes += __popc(chm);
        if (TRACE) {
          while (chm) {
            const int k = __ffs(chm) - 1;
            chm &= chm - 1;
            trace(TR_CONTROL, 1, k, __shfl_sync(FULL, Bk, k));
          }
        }
      }
      if (CLS && cd.admit) {  // (iv) M28 admission gate on the source role's busy time
        const DRole& R0 = P.role[0];
        const bool mine = lane >= (int)R0.first && lane < (int)(R0.first + R0.n);
        const unsigned long long u1000 = warp_sum64(mine ? (unsigned long long)acc_busy : 0ull) * 1000ull;
        bool want = gate;
        if (u1000 >= (unsigned long long)cd.admit_hi * Pk.window * R0.n) want = true;
        else if (u1000 <= (unsigned long long)cd.admit_lo * Pk.window * R0.n) want = false;
        if (want != gate && q - q_last_gate >= (int32_t)cd.dwell) {
          gate = want;
          q_last_gate = q;
          if (lane == 0) ++H->gate_changes;
          if (TRACE) trace(TR_CONTROL, 3, 0, want ? 1u : 0u);
        }
      }
      if (!LEAN && cd.select_role >= 0) {  // (iii) model selection
        const DRole& Rs = P.role[cd.select_role];
        const uint32_t cs = __shfl_sync(FULL, sel_l, cd.select_role);
        const unsigned long long b1000 = (unsigned long long)__shfl_sync(FULL, acc_busy, cs) * 1000ull;
        uint32_t ns = cs;
        if (b1000 >= (unsigned long long)cd.hi * Pk.window || viol) ns = Rs.small_inst;
        else if (b1000 <= (unsigned long long)cd.lo * Pk.window && !viol) ns = Rs.large_inst;
        if (ns != cs && q - q_last_sel >= (int32_t)cd.dwell) {
          if (lane == cd.select_role) sel_l = ns;
          q_last_sel = q;
          if (lane == 0) ++H->select_changes;
          if (TRACE) trace(TR_CONTROL, 2, cd.select_role, ns);
        }
      }
    };
    auto close_window = [&](bool final_partial) {
      const uint32_t ss = H->ser_slot;
      if (ss != 0xFFFFFFFFu && wk < Pk.series_windows && is_inst) {
        SeriesRec* const ser = reinterpret_cast<SeriesRec*>(series) + (unsigned long long)ss * Pk.series_windows * n_inst;
        const int32_t il = P.role[my_role].in_link;
        SeriesRec r;
        r.qint = acc_qint;
        r.busy = acc_busy;
        r.maxq = (uint16_t)min(acc_maxq, 65535u);
        r.mode = il < 0 ? 255 : (uint8_t)((modes >> (2 * il)) & 3u);
        r.B = (uint8_t)Bk;
        ser[(unsigned long long)wk * n_inst + lane] = r;
      }
      if ((Pk.flags & SDAS_FLAG_CELL_SERIES) && wk < Pk.series_windows && is_inst) {   // M15 cell-summed series
        unsigned long long* const e =
            cell_series + (((unsigned long long)H->cell * Pk.series_windows + wk) * n_inst + lane) * 8u;
        const int32_t il = P.role[my_role].in_link;
        atomicAdd(e + 0, acc_qint);
        atomicAdd(e + 1, (unsigned long long)acc_busy);
        atomicAdd(e + 2, 1ull);
        atomicAdd(e + 3, (unsigned long long)acc_maxq);
        atomicAdd(e + 4, (unsigned long long)Bk);
        if (il >= 0) atomicAdd(e + 5 + ((modes >> (2 * il)) & 3u), 1ull);
      }
      if (!final_partial) {
        if (lane == 0) ++H->window_closes;
        if (TRACE) trace(TR_WINDOW, wk, 0, 0);
        if (cd.adaptive) control((int32_t)wk + 1);
      }
      acc_busy = 0; acc_qint = 0; acc_lint = 0; acc_maxq = 0;
      if (!final_partial) snap = fn + in + (st == RECV ? 1u : 0u) + wn + b;   // M31: the controller's poll
      __syncwarp();
      if (lane == 0) { H->w_n = 0; H->w_good = 0; H->w_half = 0; }
      __syncwarp();                        // the next window's control (same event) reads them
    };

    // lane-local DELIVER: move the in-flight head messages due by now (strict: due before now) into the
    // inbox; returns true on an inbox overflow (M14).  LAZY moves of messages due before now add the inbox
    // time they missed to the window integral and their step to max Q (the state after DELIVER at their
    // tick, which was not an event); messages due now enter the next integration step as in the model.
    auto deliver = [&](bool strict) -> bool {
      uint32_t* const ft = reinterpret_cast<uint32_t*>(my_ftick);
      unsigned long long* const fb = reinterpret_cast<unsigned long long*>(my_fbody);
      unsigned long long* ib = reinterpret_cast<unsigned long long*>(my_inbox);
      for (;;) {
        if (K1_UNLIKELY(in >= my_inbox_cap) && (!SPILL || in >= MI.inbox_cap)) return true;
        const unsigned long long body = fb[fh];
        if (CLS && prio && rCls[body & 0xFFFFu]) {        // M27: class-1 ring
          ib[my_inbox_cap + wrap_add(ih1, in1, my_inbox_cap)] = body;
          ++in1;
        } else {
          const uint32_t k = in - (CLS ? in1 : 0u);
          if (!SPILL || k < my_inbox_cap) {
            const uint32_t at_idx = wrap_add(ih, k, my_inbox_cap);
            ib[at_idx] = body;
            if (my_kv) my_iready[at_idx] = my_fready[fh];        // emission + tau*ctx (M23 HINT)
          } else {
            reinterpret_cast<unsigned long long*>(gxa(MI.gx_inbox))[wrap_add(H->gh[0][lane], k - RS,
                                                                             MI.inbox_cap - RS)] = body;
          }
        }
        ++in;
        if (LAZY && fhead != t_lo) {                       // due before now (window split: see close)
          acc_qint += t_lo - fhead;
          acc_maxq = max(acc_maxq, in + wn);
        }
        const uint32_t ofh = fh;
        fh = wrap_add(fh, 1u, my_flight_cap);
        if (SPILL && fn > my_flight_cap) {   // refill the vacated slot with the oldest extension entry
          const uint32_t g0 = H->gh[1][lane];
          ft[ofh] = reinterpret_cast<const uint32_t*>(gxa(MI.gx_ftick))[g0];
          fb[ofh] = reinterpret_cast<const unsigned long long*>(gxa(MI.gx_fbody))[g0];
          H->gh[1][lane] = (uint16_t)wrap_add(g0, 1u, MI.flight_cap - RS);
        }
        --fn;
        if (!LV) ++cnt_deliv;   // levels >= 1: derived at the finalize
        if (TRACE) trace_lane(TR_DELIVER, lane, rJ[body & 0xFFFFu], (uint32_t)(body >> 32) & 0xFFFFu);
        if (fn == 0) return false;
        fhead = ft[fh];
        if (LAZY ? (int32_t)(fhead - t_lo) > (strict ? -1 : 0) : fhead != t_lo) return false;
      }
    };

    // ---------------------------------------------------------------- event loop (M12)
#ifdef K1_COUNT_ITERS
    uint32_t n_iter = 0;   // experiment builds only (tools/iters.py): event-loop iterations -> summary word 42
#endif
    for (;;) {
#ifdef K1_COUNT_ITERS
      ++n_iter;
      uint32_t itype = 0;   // bit 0 WINDOW, 1 COMPLETE RECV, 2 COMPLETE DECODE, 3 DELIVER, 4 ARRIVE, 5/6 START RECV/DECODE
#endif
      __syncwarp();
      if (!arr_more && nsys == 0) break;   // (arr_more == jn < N, kept in a register)
      // next tick: warp-min over 32-bit deltas (every pending event lies < 2^31 ticks ahead)
      // (branch-free: lanes that are not instances hold IDLE / empty state and contribute nothing)
      const bool quiet = SILENT && st == RECV && runm == 0u;   // a silent RECV: idle from end_lo on
      uint32_t d = st != IDLE && !quiet ? end_lo - t_lo : 0xFFFFFFFFu;
      // LAZY: only idle instances (and any whose inbox could fill) wait for their deliveries as events
      d = fn && (!LAZY || st == IDLE || quiet || in + fn > my_inbox_cap) ? min(d, fhead - t_lo) : d;
      // a window boundary is an event of its own only while the next arrival is too far for 32-bit deltas
      // (or under max_ticks, whose truncation test must see every boundary before it, as M12 orders them)
      const uint32_t d0 = min(arr_near ? A_lo - t_lo : 0xFFFFFFFFu, (!arr_near || max_ticks) ? nb_lo - t_lo : 0xFFFFFFFFu);
      d = lane == 0 ? min(d, d0) : d;
      d = __reduce_min_sync(FULL, d);
      if (K1_UNLIKELY(max_ticks && t + d > max_ticks)) { status = SDAS_REPLICA_TRUNCATED; break; }
      // integrate the piecewise-constant state over [t, t + dd) (M15); a zero-length piece adds nothing
      auto integrate = [&](uint32_t dd) {
        const uint32_t Q = in + wn;
        acc_busy += st != IDLE ? (quiet ? min(dd, (uint32_t)max(0, (int32_t)(end_lo - t_lo))) : dd) : 0u;
        acc_qint += (unsigned long long)Q * dd;
        if (dd) acc_maxq = max(acc_maxq, Q);
        if (need_lint) acc_lint += (unsigned long long)(fn + Q + (st == RECV ? 1u : 0u) + b) * dd;
        if (!LV) int_nsys_acc += (unsigned long long)nsys * dd;   // levels >= 1: = sum_e2e at the end (finalize)
        t += dd;
        t_lo += dd;
      };
      // phase 0 WINDOW for every boundary on the way to t + d: nothing happens between two events, so a
      // window closes when the state is integrated up to its boundary, and its decisions apply from there on
      uint32_t rem = d;
      while (K1_UNLIKELY(rem >= nb_lo - t_lo)) {
        const uint32_t dd = nb_lo - t_lo;
        integrate(dd);
        rem -= dd;
        if (LAZY && fn && (int32_t)(fhead - t_lo) < 0) deliver(true);   // their inbox time before the boundary
#ifdef K1_COUNT_ITERS
        itype |= 1u;
#endif
        close_window(false);
        nb_lo += W32;
        ++wk;
        if (!arr_near && arr_more) arr_near = A_next - t < 0x80000000ull;
      }
      integrate(rem);
      // LAZY: messages delivered since the last event to a busy instance enter its inbox now -- before
      // COMPLETE's emissions test the in-flight rings (M14 counts undelivered only)
      if (LAZY && fn && (int32_t)(fhead - t_lo) < 0) deliver(true);
      if (quiet && (int32_t)(end_lo - t_lo) <= 0) {        // the silent RECV has ended: the instance is idle
        st = IDLE;
        ++cnt_recv;
      }
      // phase 1 COMPLETE (instance order)
      // (lanes >= n_inst stay IDLE with empty rings: no is_inst test needed in the phase votes)
      // the three phase votes are independent (COMPLETE's emissions are due after now and never change a
      // due in-flight head), so they are issued back to back instead of each behind the previous phase
      const bool done_here = st != IDLE && end_lo == t_lo;
      uint32_t cm = __ballot_sync(FULL, done_here);
      const uint32_t rm = __ballot_sync(FULL, done_here && st == RECV);
      const bool dv = fn > 0 && (LAZY ? (int32_t)(fhead - t_lo) <= 0 : fhead == t_lo);
      const uint32_t dvm = __ballot_sync(FULL, dv);
      if (cm) {
#ifdef K1_COUNT_ITERS
        itype |= (rm ? 2u : 0u) | ((cm & ~rm) ? 4u : 0u);
#endif
        do {
          const int i = __ffs(cm) - 1;
          cm &= cm - 1;
          if ((rm >> i) & 1u) complete_recv((uint32_t)i);
          else complete_decode((uint32_t)i);
          if (K1_UNLIKELY(ovf)) break;
        } while (cm);
        if (K1_UNLIKELY(ovf)) break;
      }
      // phase 2 DELIVER (per destination instance, FIFO; lane = instance).  LAZY: a busy destination's
      // deliveries are not events of their own; they are moved here at its next event, with
      // the inbox time they missed added to the window integral
      bool cut = false;                    // a DELIVER or ARRIVE may have cut a DECODE run
      if (dvm) {
#ifdef K1_COUNT_ITERS
        itype |= 8u;
#endif
        cut = true;
        bool lovf = false;
        if (dv) {
          if (coalesce) cut_run();
          lovf = deliver(false);
        }
        if (K1_UNLIKELY(__any_sync(FULL, lovf))) {
          if (TRACE) trace(TR_OVERFLOW, 0, 0, 0);
          ovf = true;
          break;
        }
        __syncwarp();
      }
      // phase 3 ARRIVE (increasing j)
      if (K1_UNLIKELY(arr_near && A_lo == t_lo)) {
#ifdef K1_COUNT_ITERS
        itype |= 16u;
#endif
        cut = true;
        do {
          arrive();
        } while (!ovf && arr_more && arr_near && A_lo == t_lo);
        if (K1_UNLIKELY(ovf)) break;
      }
      // runs cut exactly at this tick: apply their silent steps (they precede START, as in M12)
      if (TRACE && coalesce && cut) {
        uint32_t fm = __ballot_sync(FULL, flushm != 0u);
        while (fm) {
          const int i = __ffs(fm) - 1;
          fm &= fm - 1;
          const uint32_t n = __shfl_sync(FULL, flushm, i), bi = __shfl_sync(FULL, b, i);
          uint32_t* const bat = at<uint32_t>(Wr, P.inst[i].off_batch);
          if (lane < (int)bi) bat[32 + lane] += n;        // done += n (stays below every stop point)
          if (lane == i) {
            st = IDLE;
            cnt_decode += n;
            tok += (unsigned long long)n * b;
            flushm = 0;
          }
          if (TRACE) {
            const uint32_t c = max(1u, P.inst[i].tau0 + P.inst[i].gamma * bi);
            trace_silent(i, bi, c, t - (unsigned long long)n * c, n, false);
          }
        }
      }
      // phase 4 START (idle instances with work, increasing index)
      __syncwarp();                        // wait-ring / request-table writes of this tick are visible
      const bool can = st == IDLE && (in | wn | b) != 0u;
      uint32_t sm = __ballot_sync(FULL, can);
      const uint32_t recvm = __ballot_sync(FULL, can && in != 0u);
      if (sm) {
#ifdef K1_COUNT_ITERS
        itype |= (recvm ? 32u : 0u) | ((sm & ~recvm) ? 64u : 0u);
#endif
        do {
          const int i = __ffs(sm) - 1;
          sm &= sm - 1;
          const bool rv = (recvm >> i) & 1u;
          uint32_t toff = 0;
          if (rv) toff = start_recv((uint32_t)i);
          if (!rv || toff) start_decode((uint32_t)i, toff);   // (one call site: the chained run included)
        } while (sm);
      }
#ifdef K1_COUNT_ITERS
      if (lane == 0) {    // work->pad[1 + f]: iterations with flag f; pad[8 + f]: iterations whose only flag is f
        for (int f = 0; f < 7; ++f)
          if ((itype >> f) & 1u) atomicAdd(&work->pad[1 + f], 1ull);
        if (__popc(itype) == 1) atomicAdd(&work->pad[8 + __ffs(itype) - 1], 1ull);
      }
#endif
    }

    // ---------------------------------------------------------------- finalize (M18, M19)
    uint8_t* const sum_out = summary + x * SDAS_SUMMARY_BYTES;
    const unsigned long long cell = H->cell;                 // (i*K + k)*C + c, computed at the replica's start
    uint32_t* const stg = scratch + SDAS_NHIST * SDAS_NBINS + 256;   // 44 summary words, then counters
    unsigned long long* const cst = reinterpret_cast<unsigned long long*>(stg + SDAS_SUMMARY_BYTES / 4);
    __syncwarp();
    if (ovf) {
      stg[lane] = 0;
      if (lane < SDAS_SUMMARY_BYTES / 4 - 32) stg[32 + lane] = 0;
      __syncwarp();
      if (lane == 0) {
        stg[0] = SDAS_REPLICA_OVERFLOW;
        stg[4] = (uint32_t)t;
        stg[5] = (uint32_t)(t >> 32);
        stg[12] = stg[13] = stg[14] = stg[15] = 0xFFFFFFFFu;
        stg[16] = stg[17] = 0xFFFFFFFFu;
        stg[36] = stg[37] = 0xFFFFFFFFu;
        stg[41] = 0xFFFFFFFFu;
      }
      __syncwarp();
      if (lane < SDAS_SUMMARY_BYTES / 16)
        reinterpret_cast<uint4*>(sum_out)[lane] = reinterpret_cast<const uint4*>(stg)[lane];
      if (lane == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(cell_cnt + cell * SDAS_NCNT + 0), 1ull);
        atomicAdd(reinterpret_cast<unsigned long long*>(cell_cnt + cell * SDAS_NCNT + 2), 1ull);
      }
      __syncwarp();
      continue;
    }
    close_window(true);  // final partial window: series only
    __syncwarp();
    const uint32_t completed = H->completed;
    uint32_t* const he = scratch;
    uint32_t* const hf = scratch + SDAS_NBINS;
    uint32_t* const hi = scratch + 2 * SDAS_NBINS;       // interactive e2e (M29)
    uint32_t* const cnt = scratch + SDAS_NHIST * SDAS_NBINS;
    for (uint32_t k = lane; k < SDAS_NHIST * SDAS_NBINS; k += 32) he[k] = 0;
    __syncwarp();
    for (uint32_t k = lane; k < completed; k += 32) {  // log-bin histograms in shared memory (M17)
      const unsigned long long v = rec[k];
      atomicAdd(&he[bin_of((uint32_t)v)], 1u);
      atomicAdd(&hf[bin_of((uint32_t)(v >> 32))], 1u);
      if (CLS && rec_cls[k]) atomicAdd(&hi[bin_of((uint32_t)v)], 1u);
    }
    __syncwarp();
    // exact nearest-rank percentiles: the histogram locates the bin, a radix select inside it (M18)
    auto select = [&](const uint32_t* h, int field, uint32_t kq, uint32_t& val, uint32_t& binq, bool only_int) {
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
          if (v >= lo && (off >> nbits) == 0u && (off >> (shift + db)) == prefix && (!only_int || rec_cls[z]))
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
    // one select per quantile in a rolled loop: five (seven) inlined copies of the radix select evicted the
    // event loop from the instruction cache whenever a warp finalized.  q = 0..4: e2e p50,
    // p99, p90, first-feedback p50, p99; CLS q = 5, 6: interactive e2e p50, p99 (M29).  Each result goes
    // straight to its summary word (bins as u16 halves of words 16 and 41); empty sets keep the sentinels.
    const uint32_t n_int = CLS ? H->completed_int : 0u;
    if (lane == 0) {
      stg[12] = stg[13] = stg[14] = stg[15] = stg[16] = stg[17] = stg[41] = 0xFFFFFFFFu;
      stg[36] = stg[37] = 0xFFFFFFFFu;
    }
    __syncwarp();
    const uint32_t nq = completed == 0 ? 0u : (CLS && n_int > 0) ? 7u : 5u;
#pragma unroll 1
    for (uint32_t q = 0; q < nq; ++q) {
      const bool fq = q == 3 || q == 4, iq = q >= 5;
      const uint32_t pc = (q == 0 || q == 3 || q == 5) ? 50u : q == 2 ? 90u : 99u;
      const uint32_t kq = (uint32_t)((pc * (unsigned long long)(iq ? n_int : completed) + 99ull) / 100ull);
      uint32_t v = 0, bq = 0;
      select(iq ? hi : fq ? hf : he, fq ? 1 : 0, kq, v, bq, iq);
      if (lane == 0) {
        stg[q == 0 ? 12 : q == 1 ? 13 : q == 2 ? 17 : q == 3 ? 14 : q == 4 ? 15 : q == 5 ? 36 : 37] = v;
        if (q != 2 && q < 5) reinterpret_cast<uint16_t*>(stg)[q == 0 ? 32 : q == 1 ? 33 : q == 3 ? 82 : 83] = (uint16_t)bq;
      }
    }
    const uint32_t recvs = __reduce_add_sync(FULL, is_inst ? cnt_recv : 0u);
    // every delivered message is received before the last request completes and every other RECV is an
    // admitted arrival's (M7, M14): on levels >= 1 (no truncation; overflowed replicas report zeros)
    // deliveries = RECVs - admitted
    const uint32_t deliv = LV ? recvs - H->admitted : __reduce_add_sync(FULL, is_inst ? cnt_deliv : 0u);
    const uint32_t decs = __reduce_add_sync(FULL, is_inst ? cnt_decode : 0u);
    const uint32_t kvs = __reduce_add_sync(FULL, is_inst ? cnt_kv : 0u);
    const uint32_t larges = __reduce_add_sync(FULL, is_inst ? n_large : 0u);
    const unsigned long long tokens = warp_sum64(is_inst ? tok : 0ull);
    __syncwarp();
    if (lane == 0) {
      const WarpHdr& h = *H;
      const uint32_t admitted = h.admitted, dropped = h.dropped, good = h.good, n_sat = h.n_sat;
      const unsigned long long sum_e2e = h.sum_e2e, sum_ff = h.sum_ff;
      // integral of N(t) (M15) = sum over requests of (departure - arrival): on levels >= 1 a replica that
      // reaches the finalize has completed every admitted request (no truncation), so it is sum_e2e
      const unsigned long long int_nsys = LV ? sum_e2e : int_nsys_acc;
      const uint32_t window_closes = h.window_closes, mode_switches = h.mode_switches;
      const uint32_t batch_changes = h.batch_changes, select_changes = h.select_changes;
      const uint32_t arrivals = admitted + dropped;
      stg[0] = status; stg[1] = admitted; stg[2] = dropped; stg[3] = completed;
      stg[4] = (uint32_t)t; stg[5] = (uint32_t)(t >> 32);
      stg[6] = (uint32_t)sum_e2e; stg[7] = (uint32_t)(sum_e2e >> 32);
      stg[8] = (uint32_t)sum_ff; stg[9] = (uint32_t)(sum_ff >> 32);
      stg[10] = (uint32_t)int_nsys; stg[11] = (uint32_t)(int_nsys >> 32);
      stg[18] = h.max_e2e; stg[19] = n_sat;
      stg[20] = arrivals; stg[21] = deliv; stg[22] = recvs; stg[23] = decs;
      stg[24] = window_closes; stg[25] = mode_switches; stg[26] = good; stg[27] = larges;
      stg[28] = (uint32_t)tokens; stg[29] = (uint32_t)(tokens >> 32);
      stg[30] = batch_changes;
      stg[31] = kvs;
      stg[32] = h.completed_int; stg[33] = h.rejected;
      stg[34] = (uint32_t)h.sum_e2e_int; stg[35] = (uint32_t)(h.sum_e2e_int >> 32);
      stg[38] = h.good_int; stg[39] = h.gate_changes;
      stg[40] = select_changes; stg[42] = 0; stg[43] = 0;
#ifdef K1_COUNT_ITERS
      stg[42] = n_iter;
#endif
      cst[24] = h.completed_int; cst[25] = h.rejected; cst[26] = h.sum_e2e_int; cst[27] = h.good_int;
      cst[0] = 1; cst[1] = status == SDAS_REPLICA_OK; cst[2] = 0; cst[3] = status == SDAS_REPLICA_TRUNCATED;
      cst[4] = admitted; cst[5] = dropped; cst[6] = completed; cst[7] = sum_e2e; cst[8] = sum_ff;
      cst[9] = t; cst[10] = int_nsys; cst[11] = good; cst[12] = larges; cst[13] = arrivals;
      cst[14] = deliv; cst[15] = recvs; cst[16] = decs; cst[17] = window_closes; cst[18] = mode_switches;
      cst[19] = tokens; cst[20] = batch_changes; cst[21] = select_changes; cst[22] = n_sat;
      cst[23] = kvs;
    }
    __syncwarp();
    if (lane < SDAS_SUMMARY_BYTES / 16)
      reinterpret_cast<uint4*>(sum_out)[lane] = reinterpret_cast<const uint4*>(stg)[lane];
    int* const ch = cell_hist + cell * (SDAS_NHIST * SDAS_NBINS);
    for (uint32_t k = lane; k < (CLS ? SDAS_NHIST : 2) * SDAS_NBINS; k += 32) {
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
