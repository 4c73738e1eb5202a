// Internal device-side parameter block of libsdas (product path only; not shared with oracle/).
// The host library packs a DParams header followed by candidates, arrival descriptors and LIST
// tick arrays into the caller-provided `params` device buffer; K1 copies DParams into shared
// memory once per CTA.
#pragma once
#include <stdint.h>

#include "../../include/sdas.h"

namespace sdas {

constexpr unsigned long long kUnsetFF = ~0ull;   // first-feedback latency not yet observed (u64 slot)
constexpr uint32_t kNever = 0xFFFFFFFFu;
constexpr int kScratchMin = SDAS_NHIST * SDAS_NBINS * 4 + 256 * 4 + SDAS_SUMMARY_BYTES + SDAS_NCNT * 8;  // finalize scratch

struct DInst {          // one instance, 80 B
  uint32_t role, h, alpha, beta, tau0, gamma, B_default, flags;   // flags: bit0 large, bit1 svc_exp
  uint32_t inbox_cap, flight_cap, wait_cap;                       // logical capacities (M14)
  uint32_t off_inbox, off_ftick, off_fbody, off_wait, off_batch;  // byte offsets inside the warp region
  // two-level rings: a ring whose capacity exceeds DParams.ring_s keeps its oldest ring_s
  // entries in shared memory and the rest in this warp's extension area of `work` (byte offsets below)
  uint32_t gx_inbox, gx_ftick, gx_fbody, gx_wait;
};

struct DRole {          // one role, 64 B
  uint32_t first, n, route, route_fixed;
  uint32_t out_fixed, out_num, out_den, n_functions;
  int32_t in_link;
  uint32_t n_out, out_link0, out_link1;
  uint32_t large_inst, small_inst, batch_words, pad;      // batch_words = 2 + 2*n_out per slot
};

struct DLink {          // one link, 32 B
  uint32_t src, dst, net, chunk, mode, gap, pad1, pad2;   // gap: M30 pacing (pipeline knob)
};

struct DCand {          // one candidate, 80 B
  uint32_t adaptive;
  uint8_t mode[8];
  uint32_t ctl_links, metric_load, lo, hi, dwell;
  uint8_t band[4];
  uint32_t route_override, batch_roles, q_hi;
  int32_t select_role;
  uint8_t kv_policy, guard_links, guard_pct, stale_jsq;   // guard: M25 (f3); stale_jsq: M31 (f4)
  uint64_t policy_slo;
  uint32_t prio, admit;                              // f2: M27 priority service, M28 admission gate
  uint16_t admit_lo, admit_hi;
  uint32_t pace;                                     // f4 M30: 0xFFFFFFFF = link knobs, else every link
};

struct DArr {           // one arrival descriptor, 80 B
  uint32_t kind, list_len;
  uint64_t gap0, gap1, soj0, soj1;
  uint64_t list_off;    // byte offset of the LIST ticks inside the params blob
  uint32_t p_lo, p_hi, o_lo, o_hi;
  uint64_t ithr;        // M26: interactive iff ATTR(sub 1).w0 < ithr = floor(permille * 2^32 / 1000)
  uint64_t pad;
};

struct alignas(16) DParams {
  uint32_t n_roles, n_links, n_inst, feedback_role;
  uint32_t request_cap, n_requests, flags, bitmap_words;
  uint32_t C, I, K, S;
  uint32_t seed_offset, rank, world, series_stride;
  uint32_t series_slots, series_windows, trace_cap, smem_per_warp;
  uint32_t off_warps;        // byte offset of warp 0's region in the CTA's shared memory
  uint32_t off_reqA, off_reqFF, off_reqJ, off_reqO, off_reqNit, off_reqOut, off_bitmap, off_scratch;
  uint32_t max_out, need_lint, kv_role, kv_ctx, kv_tau, off_reqHome;
  uint32_t cls, off_reqCls;   // f2: two request classes (class-1 rings follow the class-0 rings)
  uint32_t need_pace, lean;   // f4: some link or candidate paces (M30); lean: K1 specialisation (§5.3)
  uint32_t ring_s;            // shared-memory ring size bound (levels >= 1; 0xFFFFFFFF = every ring whole)
  uint32_t off_arrq;          // LEAN: per-warp queue of the next 32 Poisson arrivals' draws (32 x u64 gap, 32 x u32 P|O)
  uint64_t off_gx, gx_per_warp;   // ring extension areas in `work`: warp w's at off_gx + w * gx_per_warp
  uint64_t off_rec_cls;       // f2: byte offset in `work` of the per-warp record-class arrays
  uint64_t kv_skew32;         // M21: home = instance 0 iff ATTR.w2 < kv_skew32 = floor(skew * 2^32 / 1000)
  uint64_t window, slo, max_ticks, master_seed;
  uint64_t first_group, n_local_groups, n_local_replicas, trace_replica;
  uint64_t off_cand, off_arr;
  DInst inst[SDAS_MAX_INSTANCES];
  DRole role[SDAS_MAX_ROLES];
  DLink link[SDAS_MAX_LINKS + 1];
  // reciprocals for K1's divisions (a u32 division by a variable is a ~125-cycle dependent chain on B200):
  // rcp_step[i][b] = floor(2^32 / c) for instance i's DECODE step cost c = max(1, tau0 + gamma b) (M7),
  // rcp_fn[f] = floor(2^32 / f) for FUNCTION emission-point divisors f = 1..255 (M9); 0xFFFFFFFF for 1
  uint32_t rcp_step[SDAS_MAX_INSTANCES][SDAS_MAX_BATCH + 1];
  uint32_t rcp_fn[256];
};

static_assert(sizeof(DInst) == 80, "DInst");
static_assert(sizeof(DRole) == 64, "DRole");
static_assert(sizeof(DCand) == 80, "DCand");
static_assert(sizeof(DArr) == 80, "DArr");
static_assert(sizeof(DParams) % 16 == 0, "DParams");

struct Work {              // head of the `work` buffer
  unsigned long long next_replica;
  unsigned long long pad[31];
  // followed by per-warp record scratch: total_warps x n_requests x u64
};

// Launch wrappers implemented in sdas_kernels.cu (host-callable).
int launch_simulate(const uint8_t* params_dev, const DParams& hp, const sdas_buffers* b, uint32_t blocks,
                    uint32_t warps_per_block, uint32_t smem_bytes, void* stream, const uint64_t* log2_table);
int launch_group_argmin(const uint8_t* params_dev, const DParams& hp, const sdas_buffers* b, uint32_t objective,
                        uint64_t slo, void* stream);
int launch_finalize(const uint8_t* params_dev, const DParams& hp, const sdas_buffers* b, uint32_t objective,
                    uint64_t slo, uint64_t n_cells, uint64_t n_rows, void* stream);
int query_occupancy(uint32_t warps_per_block, uint32_t smem_bytes, uint32_t maxout, uint32_t cls, uint32_t lean,
                    uint32_t spill, int* blocks_per_sm,
                    int* n_sm);
const char* cuda_error_string(int code);

}  // namespace sdas
