// engine.cuh — EconoServe's per-iteration scheduling step, B200-native.
//
// One warp owns one serving instance and runs its whole Engine::step() loop
// on-device (engine.hpp:104-116). All state lives in HBM as structure-of-
// arrays (layout: DESIGN.md §3); the per-instance scalar block `Inst` is
// staged in shared memory for the duration of a launch.
//
// The code is written warp-cooperatively against a tiny portability layer
// (W lanes, LANE, BALLOT, WSYNC...). nvcc builds it with W = 32 for sm_100a;
// the test-only host build (tests/hostsim) compiles the very same source with
// W = 1 so logic can be checked against the oracle on a CPU-only box. The
// product library is always the nvcc build — there is no CPU path in it.
//
// Reference data structures are replaced, not translated:
//   PtQueue sorted vector (queues.hpp:80-108)  -> ordered: per-(deadline bucket,
//       prompt) FIFO class lists + two-level bitmaps; FIFO: 32-ary min tree
//       over request ids. Greedy skip-fit (queues.hpp:279-299) becomes
//       O(takes) bitmap / tree queries instead of an O(|Q_P|) walk.
//   GtQueue vector of groups (queues.hpp:125-204) -> group pool + key-sorted
//       slot array + RL->group map + per-group cached demand sums.
//   KvcAllocator std::map free list (kvc.hpp:334-401) -> address-sorted array
//       of live regions; free gaps are its complement (always maximal in the
//       reference: give_back coalesces both sides, take leaves an adjacent
//       rest), so first-fit is a warp ballot over gaps and compact() a scan.
//   HostingSlot vector (kvc.hpp:17-24) -> per-hosted-request slot fields +
//       an insertion-ordered list of hosted ids.
#pragma once
#include <limits.h>
#include <math.h>
#include <stdint.h>

#include "econoserve_b200.h"
#include "glibc_libm.cuh"

#ifdef __CUDACC__
#define EDEV __device__ __forceinline__
// Every engine function inlines into k_engine_steps: measured 15% faster than
// separate device functions (no call/stack traffic, scheduling across calls).
#define EDEVNI __device__ __forceinline__
#define EHD __host__ __device__ __forceinline__
// Rare paths (compaction, the pipelining planner, preemption, overruns, idle
// stretches). Out of line (__noinline__) they left the hot code denser but
// measured 7% slower (call frames, generic pointers to the shared Inst,
// register allocation of the replay loop), so they stay inlined.
#define ECOLD __device__ __forceinline__
#define W 32
#define LANE ((int)(threadIdx.x & 31))
#define WSYNC() __syncwarp()
#define BALLOT(p) __ballot_sync(0xffffffffu, (p))
#define MATCH_ANY(v) __match_any_sync(0xffffffffu, (v))
#define FFS(m) (__ffs(m) - 1)
#define POPC(m) __popc(m)
#define LANEMASK_LT ((1u << LANE) - 1u)
#define SMEM_ADD(p, v) atomicAdd((p), (v))
#define CLZ64(x) __clzll((long long)(x))
#define CLZ32(x) __clz((int)(x))
template <class T> EDEV T shfl(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }
template <class T> EDEV T shfl_xor(T v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
EHD uint64_t umulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * (unsigned __int128)b) >> 64);
#endif
}
#else
#define EDEV static inline
#define EDEVNI static
#define EHD static inline
#define ECOLD static
#define W 1
#define LANE 0
#define WSYNC() ((void)0)
#define BALLOT(p) ((p) ? 1u : 0u)
#define MATCH_ANY(v) 1u
#define FFS(m) ((m) ? 0 : -1)
#define POPC(m) ((m) ? 1 : 0)
#define LANEMASK_LT 0u
#define SMEM_ADD(p, v) (*(p) += (v))
#define CLZ64(x) __builtin_clzll(x)
#define CLZ32(x) __builtin_clz(x)
template <class T> static inline T shfl(T v, int) { return v; }
template <class T> static inline T shfl_xor(T v, int) { return v; }
static inline uint64_t umulhi64(uint64_t a, uint64_t b) {
  return (uint64_t)(((__uint128_t)a * (__uint128_t)b) >> 64);
}
#endif

#ifdef __CUDACC__
#define PROF_NOW() ((int64_t)clock64())
#else
#define PROF_NOW() ((int64_t)0)
#endif
// Per-phase cycle counters (prof[3], [6..10], [13..15]) cost ~10 instructions
// each; they are compiled in only with -DECONO_PROF_PHASES (tools/probe_scale).
#ifdef ECONO_PROF_PHASES
#define PHASE_NOW() PROF_NOW()
#define PHASE_ADD(k, v) LANE0(I.prof[k] += (v))
#else
#define PHASE_NOW() ((int64_t)0)
#define PHASE_ADD(k, v) ((void)0)
#endif

// Event / sample recording switches. A translation unit compiled with
// ECONO_NOREC (csrc/kernel_fast.cu) gets a copy of the step loop with every
// recording path removed at compile time; the runtime launches it for
// batches that record nothing (the bench path), the generic copy otherwise.
#ifdef ECONO_NOREC
#define REC_EV(I) false
#define REC_SM(I) false
#else
#define REC_EV(I) ((I).record_events != 0)
#define REC_SM(I) ((I).record_samples != 0)
#endif
// The same translation unit is specialised for the ordered PT queue (class
// lists + bitmaps; econoserve-sdo/-full): the FIFO min-tree paths drop out.
// ECONO_SPEC_ORACLE_FULL: econoserve-full with the oracle predictor (the
// bench configuration): the noisy predictors' code and the non-pipelining
// branch drop out as well.
#ifdef ECONO_SPEC_ORACLE_FULL
#define PRED_ORACLE(I) true
#define FULL(I) true
#else
#define PRED_ORACLE(I) ((I).pred_model == ECONO_PRED_ORACLE)
#define FULL(I) ((I).full != 0)
#endif
// (ordered implies GT grouping: econoserve-sdo and -full both group.)
#ifdef ECONO_SPEC_ORDERED
#define ORD(I) true
#define GRP(I) true
#else
#define ORD(I) ((I).ordered != 0)
#define GRP(I) ((I).grouping != 0)
#endif

#define LANE0(stmt) \
  do {              \
    if (LANE == 0) { stmt; } \
    WSYNC();        \
  } while (0)
// A scalar update of warp-uniform state, executed by every lane on the same
// values (each lane loads the same words and stores the same result), so the
// warp never diverges around it: no BSSY/BSYNC pair, no branch, and no
// instruction-fetch stall at the reconvergence point — on this latency-bound
// path those stalls were the largest single cause (ncu: no_instructions, 38%
// of samples, a third of them at BSYNC). Only for statements whose operands
// are uniform and which contain no atomics or per-lane clocks; those keep
// LANE0.
#define UNI(stmt) \
  do {            \
    stmt;         \
  } while (0)

namespace econo {

typedef int64_t Tok;
static const int32_t INF32 = 0x7fffffff;

enum { ST_WAITING_PT = 0, ST_RUNNING = 1, ST_WAITING_GT = 2, ST_PREEMPTED = 3, ST_DONE = 4 };
enum { F_HOSTED = 1, F_WAS_PREEMPTED = 2, F_ALLOC_FAIL = 4, F_HAS_RESERVED = 8, F_HAS_SLOT = 16,
       F_PREFILL_FIN = 32, F_CAND = 64 };
enum {
  ERR_NONE = 0, ERR_ALLOC_FAIL, ERR_RESERVED_DRAW, ERR_SLOT_OUTSIDE, ERR_STUCK,
  ERR_RELEASE_UNKNOWN, ERR_TABLE_OVERFLOW, ERR_INFEASIBLE_KVC, ERR_INFEASIBLE_RESERVE,
  ERR_ARRIVAL_ORDER, ERR_FIRST_BLOCK, ERR_ADMIT_BLOCK, ERR_EXACT_ADMIT
};
enum { STATUS_RUN = 0, STATUS_DRAIN = 1 };

// Device pointer held in the shared-memory Inst. Every use carries
// __isGlobal, so accesses compile to global loads/stores (LDG/STG); generic
// ones could alias the shared-memory Inst, forcing its fields to be reloaded
// after every store.
#ifdef __CUDACC__
#define EMEM __host__ __device__ __forceinline__
#else
#define EMEM inline
#endif
template <class T>
struct GP {
  T* p;
  EMEM T* get() const {
#ifdef __CUDA_ARCH__
    T* q = p;
    __builtin_assume(__isGlobal(q));
    return q;
#else
    return p;
#endif
  }
  EMEM operator T*() const { return get(); }
  EMEM T& operator[](int64_t i) const { return get()[i]; }
  EMEM GP& operator=(T* q) {
    p = q;
    return *this;
  }
};

// Per-instance scalar block + SoA pointers. Kept in shared memory while a
// launch runs (one warp per instance), written back on exit.
struct Inst {
  // ---- configuration (immutable after create) ----
  int32_t n, policy, ordered, grouping, full, pred_model;
  int32_t nbd, nbk, record_events, record_samples, skip, _pad1;
  int32_t pmax, nbuckets, bm_words, bm_l2;    // PT class table (ordered mode)
  int32_t tree_levels, rl_cap;
  int32_t tr_pmin, tr_pmax, tr_rmin, tr_rmax;  // trace prompt / response length ranges (device init; burst-ingest class window)
  int32_t tree_off[8], tree_len[8];            // 32-ary min tree (FIFO mode)
  int32_t reg_cap, grp_cap, slot_cap, run_cap, ptiter_cap, adm_cap, scr_cap, hist_cap, sel_cap, _pad2;
  int64_t tfs, capacity, block, reserve_cap, general_cap, pred_quantum;
  double t_base, t_token, over_rate, reserve_penalty, pen_free, pen_offload, sched_cost;
  double pred_sigma, pred_accuracy, pred_tol, pred_pad, slo_scale, buffer_ratio;
  double dbounds[ECONO_MAX_BOUNDS];
  int64_t kbounds[ECONO_MAX_BOUNDS];
  // ---- dynamic scalars ----
  double clock, t_p, t_g;
  int64_t iter, completed, arrival_cursor, free_total, reserved_used, written_total, exam_count;
  int64_t hosted_total, hosted_overruns, alloc_failures, steps, executed, pt_dispatched, gt_scheduled;
  uint64_t next_group_id, gt_next_seq;
  int32_t pt_count, G, R, n_slots, n_regions, n_ptiter, n_adm, pts_admitted_iter, pt_admittable;
  int32_t reg_free_top, grp_free_top, n_sel, n_selg, n_hosts_members, sl_free_top, _pad4;
  int32_t error, err_id, status, mt_i, pmt_i, _pad0;
  int64_t err_val, ev_n, ev_cap, sm_n, sm_cap, ev_total;
  double wbuf[W];      // quiet-span replay: one chunk of per-step written fractions
  int64_t pt_min_lb;   // lower bound on the smallest queued prompt (only grows between arrivals)
  int64_t ovf_id, ovf_dem;  // first request whose prediction saturated (kRlSat) at init, its exact demand
  int32_t bcnt[ECONO_MAX_BOUNDS + 2];  // queued PTs per deadline bucket (ordered mode)
  int64_t quiet_steps, quiet_spans, bcast;
  // device cycle counters (econo_batch_debug): [0] quiet-span tests [1] quiet
  // replays [2] normal steps [4] spans [5] normal-step count; normal-step
  // phases [6] ingest [7] GT select+schedule [8] pipelining [9] PT batching
  // [10] execute_iteration; [11] launch total [12] launches; inside
  // execute_iteration [3] running-set pass + completions [13] prefill + sample
  // [14] prefill transitions [15] under-prediction, slot deadlines, tail.
  int64_t prof[16];
  double agg_written, agg_allocated;
  int64_t agg_fs, agg_tfs_hits, agg_pt_iters;
  // ---- baseline policies (engine.hpp:383-726; baselines.cuh) ----
  int32_t base, batch_cap, recompute, decode_pause, admission_open, n_admo, n_ongo, _pad3;
  int64_t chunk, max_out;
  double swap_stall, pending_stall;
  // ---- per-request SoA (n entries) ----
  GP<const double> arrival;
  GP<const int32_t> prompt;
  GP<const int32_t> true_rl;
  GP<int32_t> predicted, generated, occupied, allowance, gen_epoch, prefill_done;
  GP<int32_t> preempt_count, reserve_draws, held, reg_head, reserved, written;
  // pt_next and gt_next share storage: a request is never queued as a PT and
  // a GT at once, and each link is written when the request joins its queue
  GP<int32_t> sidx, pt_next, gt_next;  // sidx: a hosted request's slot-pool entry
  GP<uint8_t> state, flags;
  GP<double> waiting, preempt_t, exec_t, dispatch_t, first_tok, compl_clock, last_enq;
  GP<double> penalty, sched_share;
  // ---- KVC region pool (reg_cap) ----
  GP<int32_t> rg_start, rg_len, rg_owner, rg_next, reg_free, addr;
  // ---- PT queue ----
  GP<int32_t> cls_head, cls_tail, cls_cnt;
  GP<uint64_t> bm1, bm2;
  GP<int32_t> tree;
  // ---- GT groups (grp_cap) ----
  GP<uint64_t> gr_id, gr_seq;
  // gr_hd: the head member's demand, so the quiet-span test needs no
  // dependent load through the head id
  GP<int32_t> gr_rl, gr_head, gr_tail, gr_cnt, gr_db, gr_kb, gr_maxocc, grp_free, gq, rl_map, gr_hd;
  GP<double> gr_formed, gr_mindl;
  GP<int64_t> gr_dem;
  // ---- ordered lists ----
  GP<int32_t> run, slots, ptiter_id, ptiter_tok, adm;
  // ---- hosting-slot pool (slot_cap entries; I.slots lists entries in
  // insertion order): host, start offset (== deadline usage), length,
  // absolute start, hosted id; free entries on a stack ----
  GP<int32_t> sl_host, sl_off, sl_len, sl_abs, sl_hosted, sl_free;
  // ---- scratch ----
  GP<int32_t> sel_ids, selg_start, selg_rl;            // GT selection output
  GP<int32_t> wa_w, wa_b, wa_l, wa_u, wb_w, wb_b, wb_l, wb_u;  // planner regions
  GP<int32_t> cd_ri, cd_abs, cd_use, cd_len, assigned;   // planner candidates
  GP<int32_t> os_host, os_hosted, os_off, os_len, os_abs;  // planner output slots
  GP<int32_t> tmp_a, tmp_b, tmp_c;
  // ---- baseline policies: admit order (LIFO victims), ongoing chunked
  // prefills, per-request prefill target (recompute preemption) ----
  GP<int32_t> admo, ongo, ptarget;
  // ---- RNG (mt19937_64 x2) ----
  GP<uint64_t> mt, pmt;
  // ---- outputs ----
  GP<EconoEvent> ev;
  GP<EconoSample> sm;
  GP<int64_t> hist;
};

// ------------------------------------------------------------------------
// scalar helpers (common.hpp:26-35; std::min/max semantics kept for doubles)
// ------------------------------------------------------------------------
// block_round (common.hpp:26-29); power-of-two blocks (the usual case) take
// a mask instead of a 64-bit division.
EDEV Tok block_round(Tok t, Tok b) {
  if (t <= 0) return 0;
  if ((b & (b - 1)) == 0) return (t + b - 1) & ~(b - 1);
  return (t + b - 1) / b * b;
}
// a / b for nonnegative a, positive b: 32-bit division when both fit.
EDEV Tok udiv(Tok a, Tok b) {
  if (((uint64_t)a | (uint64_t)b) < (1ULL << 32)) return (Tok)((uint32_t)a / (uint32_t)b);
  return a / b;
}
EHD Tok ceil_tokens(double v) { return (Tok)ceil(v - 1e-9); }
EDEV double dmax(double a, double b) { return (a < b) ? b : a; }
EDEV double dmin(double a, double b) { return (b < a) ? b : a; }
EDEV Tok tmax(Tok a, Tok b) { return (a < b) ? b : a; }
EDEV Tok tmin(Tok a, Tok b) { return (b < a) ? b : a; }

EDEV double iteration_time(const Inst& I, Tok fs) {  // engine.hpp:46-51
  const Tok base = tmin(fs, I.tfs);
  const Tok over = tmax(0, fs - I.tfs);
  return I.t_base + I.t_token * (double)base + I.over_rate * (double)over;
}

template <class T>
EDEV T wmin(T v) {
  for (int o = W / 2; o > 0; o >>= 1) {
    T x = shfl_xor(v, o);
    v = x < v ? x : v;
  }
  return v;
}
template <class T>
EDEV T wsum(T v) {
  for (int o = W / 2; o > 0; o >>= 1) v += shfl_xor(v, o);
  return v;
}
// 32-bit reductions: one REDUX instruction instead of five shuffle rounds.
EDEV int32_t wmin32(int32_t v) {
#ifdef __CUDA_ARCH__
  return __reduce_min_sync(0xffffffffu, v);
#else
  return v;
#endif
}
EDEV int32_t wsum32(int32_t v) {
#ifdef __CUDA_ARCH__
  return __reduce_add_sync(0xffffffffu, v);
#else
  return v;
#endif
}

// Shift a[pos..n) right by one and store v at pos (room for n+1 required).
template <class T>
EDEV void arr_insert(T* a, int32_t n, int32_t pos, T v) {
  for (int32_t hi = n; hi > pos; hi -= W) {
    const int32_t i = hi - 1 - LANE;
    const bool ok = i >= pos;
    T x = T();
    if (ok) x = a[i];
    WSYNC();
    if (ok) a[i + 1] = x;
    WSYNC();
  }
  UNI(a[pos] = v);
}
// Remove a[pos..pos+k) from an n-element array.
template <class T>
EDEV void arr_erase(T* a, int32_t n, int32_t pos, int32_t k) {
  for (int32_t lo = pos; lo < n - k; lo += W) {
    const int32_t i = lo + LANE;
    const bool ok = i < n - k;
    T x = T();
    if (ok) x = a[i + k];
    WSYNC();
    if (ok) a[i] = x;
    WSYNC();
  }
}
template <class T>
EDEV void arr_insert(GP<T> a, int32_t n, int32_t pos, T v) {
  arr_insert(a.get(), n, pos, v);
}
template <class T>
EDEV void arr_erase(GP<T> a, int32_t n, int32_t pos, int32_t k) {
  arr_erase(a.get(), n, pos, k);
}
// Position of the first element equal to v (or -1), warp ballot scan.
EDEV int32_t arr_find(const int32_t* a, int32_t n, int32_t v) {
  for (int32_t base = 0; base < n; base += W) {
    const int32_t i = base + LANE;
    const unsigned m = BALLOT(i < n && a[i] == v);
    if (m) return base + FFS(m);
  }
  return -1;
}

// ------------------------------------------------------------------------
// events / errors
// ------------------------------------------------------------------------
// Called warp-uniformly with uniform arguments; every lane performs the same
// stores (see UNI), so the common no-recording case costs no divergence.
EDEV void logev(Inst& I, int kind, int32_t id, int64_t a, int64_t b) {  // engine.hpp:211-214
  {
    I.ev_total++;
    if (REC_EV(I)) {
      if (I.ev_n < I.ev_cap) {
        EconoEvent& e = I.ev[I.ev_n];
        e.iter = I.iter;
        e.clock = I.clock;
        e.kind = kind;
        e.id = id;
        e.a = a;
        e.b = b;
      }
      I.ev_n++;
    }
  }
}
EDEV void set_error(Inst& I, int code, int32_t id, int64_t val) {
  if (LANE == 0 && I.error == ERR_NONE) {
    I.error = code;
    I.err_id = id;
    I.err_val = val;
  }
  WSYNC();
}

// ------------------------------------------------------------------------
// RNG: std::mt19937_64 and the libstdc++ 13 distributions the path uses.
// Called by lane 0 only (one sequential stream per instance).
// ------------------------------------------------------------------------
EHD uint64_t mt_next(uint64_t* x, int32_t& idx) {
  if (idx >= 312) {
    const uint64_t up = 0xFFFFFFFF80000000ULL, lo = 0x7FFFFFFFULL;
    for (int k = 0; k < 312; ++k) {
      const int k1 = k + 1 == 312 ? 0 : k + 1;
      const int km = k + 156 >= 312 ? k + 156 - 312 : k + 156;
      const uint64_t y = (x[k] & up) | (x[k1] & lo);
      x[k] = x[km] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
    }
    idx = 0;
  }
  uint64_t z = x[idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= (z >> 43);
  return z;
}
EHD void mt_seed(uint64_t* x, int32_t& idx, uint64_t s) {
  x[0] = s;
  for (int i = 1; i < 312; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + (uint64_t)i;
  idx = 312;
}
// uniform_int_distribution::_S_nd (uniform_int_dist.h:257-282), Lemire with a
// 128-bit product split into umulhi/lo.
EHD uint64_t lemire(uint64_t* x, int32_t& idx, uint64_t range) {
  uint64_t r = mt_next(x, idx);
  uint64_t lo = r * range, hi = umulhi64(r, range);
  if (lo < range) {
    const uint64_t thr = (0 - range) % range;
    while (lo < thr) {
      r = mt_next(x, idx);
      lo = r * range;
      hi = umulhi64(r, range);
    }
  }
  return hi;
}
EHD uint64_t uniform_u64(uint64_t* x, int32_t& idx, uint64_t a, uint64_t b) {
  const uint64_t urange = b - a;
  if (urange < 0xFFFFFFFFFFFFFFFFULL) return lemire(x, idx, urange + 1) + a;
  return mt_next(x, idx) + a;
}
EHD double canonical(uint64_t* x, int32_t& idx) {  // random.tcc:3349-3380
  double r = (double)mt_next(x, idx) / 18446744073709551616.0;
  if (r >= 1.0) r = 0.99999999999999989;  // nextafter(1, 0)
  return r;
}
// A fresh normal_distribution per call (workload.hpp:233): polar method,
// random.tcc:1811-1844; the cached second variate is discarded.
EDEV double normal_fresh(uint64_t* x, int32_t& idx, double stddev) {
  double a, b, r2;
  do {
    a = 2.0 * canonical(x, idx) - 1.0;
    b = 2.0 * canonical(x, idx) - 1.0;
    r2 = a * a + b * b;
  } while (r2 > 1.0 || r2 == 0.0);
  const double mult = sqrt(-2 * econo_libm::log(r2) / r2);  // glibc's log, bit for bit
  double ret = b * mult;
  return ret * stddev + 0.0;
}
EDEV Tok quantize_up(Tok v, Tok q) { return q <= 1 ? v : block_round(v, q); }
// glibc's llround on x86-64: |v| >= 2^63 (or NaN) falls through to a plain
// (long long) conversion, i.e. cvttsd2si's "integer indefinite" LLONG_MIN
// (s_llround.c), where the device's conversion would saturate to LLONG_MAX.
EDEV Tok llround_glibc(double v) {
  if (!(v > -9223372036854775808.0 && v < 9223372036854775808.0)) return (Tok)LLONG_MIN;
  return (Tok)llround(v);
}
// predict_rl (workload.hpp:228-264)
EDEV Tok predict_rl(const Inst& I, Tok true_rl, uint64_t* x, int32_t& idx) {
  if (PRED_ORACLE(I)) return quantize_up(true_rl, I.pred_quantum);
  if (I.pred_model == ECONO_PRED_LOGNORMAL) {
    const double v = (double)true_rl * econo_libm::exp(normal_fresh(x, idx, I.pred_sigma));  // glibc's exp
    return quantize_up(tmax(1, llround_glibc(v)), I.pred_quantum);
  }
  const double t = (double)true_rl;
  const Tok lo_in = tmax(1, ceil_tokens(t * (1.0 - I.pred_tol)));
  const Tok hi_in = (Tok)floor(t * (1.0 + I.pred_tol) + 1e-9);
  if (canonical(x, idx) < I.pred_accuracy) {
    const Tok b = tmax(lo_in, hi_in);
    return quantize_up((Tok)uniform_u64(x, idx, (uint64_t)lo_in, (uint64_t)b), I.pred_quantum);
  }
  const double a = I.pred_tol, bb = 2.0 * I.pred_tol + 0.25;
  const double u = canonical(x, idx) * (bb - a) + a;
  Tok v;
  if (canonical(x, idx) < 0.5) {
    v = llround_glibc(t * (1.0 + u));
    if (v <= hi_in) v = hi_in + 1;
  } else {
    v = llround_glibc(t * (1.0 - u));
    if (v >= lo_in) v = lo_in - 1;
    if (v < 1) v = hi_in + 1;
  }
  return quantize_up(tmax(1, v), I.pred_quantum);
}
EHD Tok apply_padding(Tok p, double ratio) { return ceil_tokens((double)p * (1.0 + ratio)); }
// padded_rl (engine.hpp:188, 921): always apply_padding(predicted_rl), so it
// is recomputed instead of stored (4 bytes less per request).
// Predicted and padded RLs are stored in 32 bits, saturated at kRlSat =
// 2^30 tokens. Capacities are validated below 2^30, so a saturated request
// can never be scheduled — exactly like the reference's unsaturated int64
// value; init reports its exact int64 demand (Inst::ovf_*), never a wrapped one.
static const int32_t kRlSat = 1 << 30;
EHD int32_t sat_rl(Tok v) { return v >= (Tok)kRlSat ? kRlSat : (int32_t)v; }
EHD int32_t padded_of(const Inst& I, int64_t id) { return sat_rl(apply_padding(I.predicted[id], I.pred_pad)); }
// slo_deadline (engine.hpp:190-191), recomputed with the same operations
// from the trace (8 bytes less per request).
EHD double slo_of(const Inst& I, int64_t id) {
  return I.arrival[id] + I.slo_scale * (I.t_p + I.t_g * (double)I.true_rl[id]);
}

// ------------------------------------------------------------------------
// ordering keys (queues.hpp:30-69)
// ------------------------------------------------------------------------
EDEV int bucket_d(const Inst& I, double v) {
  int i = 0;
  while (i < I.nbd && !(v < I.dbounds[i])) ++i;
  return i;
}
EDEV int bucket_k(const Inst& I, Tok v) {
  int i = 0;
  while (i < I.nbk && !(v < I.kbounds[i])) ++i;
  return i;
}

// ------------------------------------------------------------------------
// PT queue — ordered mode: class (deadline bucket b, prompt p) FIFO lists.
// Queue order (queues.hpp:44-50 with kvc bucket 0 and seq == id) is
// b ascending, p descending, id ascending.
// ------------------------------------------------------------------------
EDEV int32_t cls_of(const Inst& I, int b, int p) { return b * (I.pmax + 1) + p; }
EDEV uint64_t mask_upto(int r) { return r >= 63 ? ~0ULL : ((1ULL << (r + 1)) - 1); }
EDEV void bm_set(Inst& I, int b, int p) {  // lane 0
  I.bm1[(int64_t)b * I.bm_words + (p >> 6)] |= 1ULL << (p & 63);
  I.bm2[(int64_t)b * I.bm_l2 + (p >> 12)] |= 1ULL << ((p >> 6) & 63);
}
EDEV void bm_clear(Inst& I, int b, int p) {  // lane 0
  uint64_t& w = I.bm1[(int64_t)b * I.bm_words + (p >> 6)];
  w &= ~(1ULL << (p & 63));
  if (w == 0) I.bm2[(int64_t)b * I.bm_l2 + (p >> 12)] &= ~(1ULL << ((p >> 6) & 63));
}
// bm_set from several lanes at once (words are shared between classes).
EDEV void bm_set_shared(Inst& I, int b, int p) {
#ifdef __CUDACC__
  atomicOr(reinterpret_cast<unsigned long long*>(&I.bm1[(int64_t)b * I.bm_words + (p >> 6)]),
           1ULL << (p & 63));
  atomicOr(reinterpret_cast<unsigned long long*>(&I.bm2[(int64_t)b * I.bm_l2 + (p >> 12)]),
           1ULL << ((p >> 6) & 63));
#else
  bm_set(I, b, p);
#endif
}
// Largest nonempty prompt class p <= x in bucket b, or -1.
EDEV int bm_prev(const Inst& I, int b, int64_t xx) {
  if (xx < 0 || I.bcnt[b] == 0) return -1;
  const int x = (int)(xx > I.pmax ? I.pmax : xx);
  const uint64_t* b1 = I.bm1 + (int64_t)b * I.bm_words;
  const uint64_t* b2 = I.bm2 + (int64_t)b * I.bm_l2;
  const int w = x >> 6;
  uint64_t word = b1[w] & mask_upto(x & 63);
  if (word) return (w << 6) + 63 - CLZ64(word);
  const int w2 = w - 1;
  if (w2 < 0) return -1;
  const int s = w2 >> 6;
  uint64_t sw = b2[s] & mask_upto(w2 & 63);
  if (!sw) {
    int found = -1;
    for (int hi = s - 1; hi >= 0 && found < 0; hi -= W) {
      const int j = hi - LANE;
      const unsigned m = BALLOT(j >= 0 && b2[j >= 0 ? j : 0] != 0);
      if (m) found = hi - FFS(m);
    }
    if (found < 0) return -1;
    sw = b2[found];
    const int ww = (found << 6) + 63 - CLZ64(sw);
    return (ww << 6) + 63 - CLZ64(b1[ww]);
  }
  const int ww = (s << 6) + 63 - CLZ64(sw);
  return (ww << 6) + 63 - CLZ64(b1[ww]);
}

// ------------------------------------------------------------------------
// PT queue — FIFO mode: 32-ary min tree over request ids (queue order ==
// arrival order == id order, seq == id). Leaves hold prompt_len or INF.
// ------------------------------------------------------------------------
EDEV int32_t tree_at(const Inst& I, int lvl, int64_t i) { return I.tree[I.tree_off[lvl] + i]; }
// First queued id >= pos whose prompt <= c, or -1.
EDEV int32_t tree_first(const Inst& I, int64_t pos, int64_t c) {
  if (c <= 0 || pos >= I.n) return -1;
  int lvl = 0;
  int64_t idx = pos, found = -1;
  for (;;) {
    const int64_t blk = idx >> 5;
    const int64_t len = I.tree_len[lvl];
    for (int j0 = 0; j0 < 32 && found < 0; j0 += W) {
      const int64_t node = blk * 32 + j0 + LANE;
      const bool ok = node >= idx && node < len && tree_at(I, lvl, node < len ? node : 0) <= c;
      const unsigned m = BALLOT(ok);
      if (m) found = blk * 32 + j0 + FFS(m);
    }
    if (found >= 0) break;
    if (lvl == I.tree_levels - 1) return -1;
    idx = blk + 1;
    ++lvl;
    if (idx >= I.tree_len[lvl]) return -1;
  }
  while (lvl > 0) {
    --lvl;
    const int64_t blk = found;
    const int64_t len = I.tree_len[lvl];
    int64_t f = -1;
    for (int j0 = 0; j0 < 32 && f < 0; j0 += W) {
      const int64_t node = blk * 32 + j0 + LANE;
      const bool ok = node < len && tree_at(I, lvl, node < len ? node : 0) <= c;
      const unsigned m = BALLOT(ok);
      if (m) f = blk * 32 + j0 + FFS(m);
    }
    found = f;
  }
  return (int32_t)found;
}
// Recompute ancestors of leaf range [lo, hi] (inclusive).
EDEV void tree_fix(Inst& I, int64_t lo, int64_t hi) {
  for (int lvl = 1; lvl < I.tree_levels; ++lvl) {
    lo >>= 5;
    hi >>= 5;
    const int64_t clen = I.tree_len[lvl - 1];
    if (hi - lo + 1 >= W) {  // many nodes: one lane per node
      for (int64_t nd = lo + LANE; nd <= hi; nd += W) {
        int32_t mn = INF32;
        for (int j = 0; j < 32; ++j) {
          const int64_t ch = nd * 32 + j;
          if (ch < clen) {
            const int32_t v = tree_at(I, lvl - 1, ch);
            mn = v < mn ? v : mn;
          }
        }
        I.tree[I.tree_off[lvl] + nd] = mn;
      }
    } else {  // few nodes: the warp reduces each node's children
      for (int64_t nd = lo; nd <= hi; ++nd) {
        int32_t mn = INF32;
        for (int j = LANE; j < 32; j += W) {
          const int64_t ch = nd * 32 + j;
          if (ch < clen) {
            const int32_t v = tree_at(I, lvl - 1, ch);
            mn = v < mn ? v : mn;
          }
        }
        mn = wmin(mn);
        LANE0(I.tree[I.tree_off[lvl] + nd] = mn);
      }
    }
    WSYNC();
  }
}
EDEV void tree_set(Inst& I, int64_t id, int32_t v) {
  LANE0(I.tree[id] = v);
  tree_fix(I, id, id);
}

// ------------------------------------------------------------------------
// KVC block manager (kvc.hpp:35-424) over the address-sorted region array.
// ------------------------------------------------------------------------
// First position p in [0, n) with pred(p) true for a monotone predicate
// (false...false true...true), n if none. One warp-wide round probes W
// evenly spaced positions in parallel, so a search costs ceil(log_W n)
// dependent round trips instead of log2 n (the host build bisects).
template <class F>
EDEV int32_t warp_search(int32_t n, F pred) {
  int32_t lo = 0, hi = n;  // answer in [lo, hi]; pred(hi) is true or hi == n
#ifdef __CUDACC__
  while (hi - lo > W) {
    const int32_t step = (hi - lo + W - 1) / W;
    const int32_t q = lo + (LANE + 1) * step - 1;  // last position of block LANE
    const bool t = q >= hi || pred(q);
    const unsigned m = BALLOT(t);
    if (!m) return hi;  // every block's last position (up to hi - 1) is false
    const int b = FFS(m);
    const int32_t qb = lo + (b + 1) * step - 1;
    lo += b * step;
    if (qb < hi) hi = qb;
  }
  const int32_t q = lo + LANE;
  const unsigned m = BALLOT(q < hi && pred(q));
  return m ? lo + FFS(m) : hi;
#else
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (pred(mid)) hi = mid; else lo = mid + 1;
  }
  return lo;
#endif
}
EDEV int32_t addr_lower(const Inst& I, Tok start) {  // first position with start >= start
  const int32_t* addr = I.addr;
  const int32_t* rs = I.rg_start;
  return warp_search(I.n_regions, [&](int32_t p) { return (Tok)rs[addr[p]] >= start; });
}
EDEV void addr_insert_region(Inst& I, int32_t r) {
  const int32_t pos = addr_lower(I, I.rg_start[r]);
  if (I.n_regions >= I.reg_cap) { set_error(I, ERR_TABLE_OVERFLOW, -1, 1); return; }
  arr_insert(I.addr, I.n_regions, pos, r);
  UNI(I.n_regions++);
}
EDEV void addr_remove_region(Inst& I, int32_t r) {
  const int32_t pos = addr_lower(I, I.rg_start[r]);
  arr_erase(I.addr, I.n_regions, pos, 1);
  UNI(I.n_regions--);
}
EDEV int32_t region_new(Inst& I, int32_t owner, Tok start, Tok len) {  // all lanes get the id
  if (I.reg_free_top <= 0) { set_error(I, ERR_TABLE_OVERFLOW, owner, 2); return -1; }
  // the free-list top and the owner's list fields load in one round; the
  // list tail is found by walking it (a holding has one region, or a few
  // after grow_exact), which saves a per-request tail pointer (4 B x n)
  const int32_t r = I.reg_free[I.reg_free_top - 1];
  const int32_t head = I.reg_head[owner], hd = I.held[owner];
  int32_t tail = head;
  if (tail >= 0)
    for (int32_t nx = I.rg_next[tail]; nx >= 0; nx = I.rg_next[tail]) tail = nx;
  WSYNC();
  {  // warp-uniform (every lane, same values)
    I.reg_free_top--;
    I.rg_start[r] = (int32_t)start;
    I.rg_len[r] = (int32_t)len;
    I.rg_owner[r] = owner;
    I.rg_next[r] = -1;
    if (tail < 0) I.reg_head[owner] = r; else I.rg_next[tail] = r;
    I.held[owner] = hd + (int32_t)len;
  }
  WSYNC();
  return r;
}

// owner_or_slot_host (kvc.hpp:405-410) for a slot whose host is h: walks up
// the chain of slots the hosts themselves occupy.
EDEV bool owner_or_slot_host(const Inst& I, int32_t h, int32_t owner) {
  for (int guard = 0; guard < 64; ++guard) {
    if (h == owner) return true;
    if (!(I.flags[h] & F_HAS_SLOT)) return false;
    h = I.sl_host[I.sidx[h]];
  }
  return false;
}

// compact() (kvc.hpp:372-401): slide every region down in address order.
ECOLD void kvc_compact(Inst& I) {
  const int32_t L = I.n_regions;
  int32_t* ns = I.tmp_a;  // new start per address position
  int32_t carry = 0;
  for (int32_t base = 0; base < L; base += W) {
    const int32_t j = base + LANE;
    int32_t len = j < L ? I.rg_len[I.addr[j]] : 0;
    int32_t incl = len;
    for (int o = 1; o < W; o <<= 1) {
      const int32_t y = shfl(incl, LANE - o >= 0 ? LANE - o : 0);
      if (LANE >= o) incl += y;
    }
    if (j < L) ns[j] = carry + incl - len;
    carry += shfl(incl, W - 1);
  }
  WSYNC();
  // slots move with the region holding their (pre-move) start
  for (int32_t base = 0; base < I.n_slots; base += W) {
    const int32_t si = base + LANE;
    if (si < I.n_slots) {
      const int32_t sp = I.slots[si];
      const int32_t abs = I.sl_abs[sp], sh = I.sl_host[sp];
      int32_t lo = 0, hi = L;  // last position with start <= abs
      while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (I.rg_start[I.addr[mid]] <= abs) lo = mid + 1; else hi = mid;
      }
      const int32_t pos = lo - 1;
      if (pos >= 0) {
        const int32_t r = I.addr[pos];
        const int32_t os = I.rg_start[r];
        if (abs < os + I.rg_len[r] && ns[pos] != os && owner_or_slot_host(I, sh, I.rg_owner[r]))
          I.tmp_b[si] = abs + (ns[pos] - os);
        else
          I.tmp_b[si] = abs;
      } else {
        I.tmp_b[si] = abs;
      }
    }
  }
  WSYNC();
  for (int32_t si = LANE; si < I.n_slots; si += W) I.sl_abs[I.slots[si]] = I.tmp_b[si];
  for (int32_t j = LANE; j < L; j += W) I.rg_start[I.addr[j]] = ns[j];
  WSYNC();
}

// take() (kvc.hpp:334-348): first fit over the complement of live regions.
// Returns the start or -1; *pos receives the address-array insert position.
EDEVNI Tok kvc_take(Inst& I, Tok need, int32_t* pos_out) {
  if (need > I.free_total) return -1;
  const int32_t L = I.n_regions;
  for (int32_t base = 0; base <= L; base += W) {
    const int32_t j = base + LANE;
    Tok gs = 0, gap = -1;
    if (j <= L) {
      if (j > 0) {
        const int32_t pr = I.addr[j - 1];
        gs = (Tok)I.rg_start[pr] + I.rg_len[pr];
      }
      const Tok ge = j < L ? (Tok)I.rg_start[I.addr[j]] : I.general_cap;
      gap = ge - gs;
    }
    const unsigned m = BALLOT(j <= L && gap >= need);
    if (m) {
      const int src = FFS(m);
      *pos_out = base + src;
      return shfl(gs, src);
    }
  }
  kvc_compact(I);
  *pos_out = L;
  return I.general_cap - I.free_total;
}

// allocate_exact / grow_exact (kvc.hpp:104-131): one new region at the fit.
EDEVNI bool kvc_alloc_region(Inst& I, int32_t id, Tok length) {
  const Tok need = block_round(length, I.block);
  int32_t pos = 0;
  const Tok s = kvc_take(I, need, &pos);
  if (s < 0) return false;
  const int32_t r = region_new(I, id, s, need);
  if (r < 0) return false;
  if (I.n_regions >= I.reg_cap) { set_error(I, ERR_TABLE_OVERFLOW, id, 3); return false; }
  arr_insert(I.addr, I.n_regions, pos, r);
  UNI(I.n_regions++; I.free_total -= need);
  return true;
}

EDEV bool kvc_draw_reserved(Inst& I, int32_t id, Tok tokens) {  // kvc.hpp:144-150
  if (I.reserved_used + tokens > I.reserve_cap) return false;
  UNI(I.reserved_used += tokens; I.reserved[id] += (int32_t)tokens; I.flags[id] |= F_HAS_RESERVED);
  return true;
}
EDEV void kvc_release_reserved(Inst& I, int32_t id) {  // kvc.hpp:152-159
  if (!(I.flags[id] & F_HAS_RESERVED)) return;
  UNI(I.reserved_used -= I.reserved[id]; I.reserved[id] = 0; I.flags[id] &= ~F_HAS_RESERVED);
}
EDEV void kvc_add_written(Inst& I, int32_t id, Tok d) {  // kvc.hpp:87-90 (lane 0 callers)
  I.written[id] += (int32_t)d;
  I.written_total += d;
}

// remove_slot (kvc.hpp:229-243)
EDEVNI void kvc_remove_slot(Inst& I, int32_t hosted) {
  if (!(I.flags[hosted] & F_HAS_SLOT)) return;
  const int32_t op = I.sidx[hosted];
  const int32_t oh = I.sl_host[op], oo = I.sl_off[op];
  const int32_t oa = I.sl_abs[op], ol = I.sl_len[op];
  int32_t mypos = -1;
  for (int32_t base = 0; base < I.n_slots; base += W) {
    const int32_t si = base + LANE;
    const int32_t sp = si < I.n_slots ? I.slots[si] : -1;
    if (sp >= 0 && sp != op && I.sl_host[sp] == hosted) {
      const int32_t a = I.sl_abs[sp];
      if (a >= oa && a + I.sl_len[sp] <= oa + ol) {
        I.sl_host[sp] = oh;
        I.sl_off[sp] += oo;
      }
    }
    const unsigned m = BALLOT(sp == op);
    if (m && mypos < 0) mypos = base + FFS(m);
  }
  WSYNC();
  if (mypos >= 0) {
    arr_erase(I.slots, I.n_slots, mypos, 1);
    UNI(I.n_slots--);
  }
  UNI(I.flags[hosted] &= ~F_HAS_SLOT; I.sl_free[I.sl_free_top++] = op);
}

// release (kvc.hpp:165-217)
// release (kvc.hpp:165-217). The request's own fields are loaded once up
// front; nothing below changes them except this function's final stores.
EDEVNI void kvc_release(Inst& I, int32_t id) {
  const int32_t head = I.reg_head[id], rsv = I.reserved[id], wr = I.written[id];
  const uint8_t f0 = I.flags[id];
  const bool had = head >= 0;
  if (!had && !(f0 & F_HAS_RESERVED) && !(f0 & F_HAS_SLOT)) {
    set_error(I, ERR_RELEASE_UNKNOWN, id, 0);
    return;
  }
  if (f0 & F_HAS_SLOT) kvc_remove_slot(I, id);
  if (had) {
    // promoted slots (host == id), in slot order
    int32_t np = 0;
    for (int32_t base = 0; base < I.n_slots; base += W) {
      const int32_t si = base + LANE;
      const bool hit = si < I.n_slots && I.sl_host[I.slots[si]] == id;
      const unsigned m = BALLOT(hit);
      if (hit) I.tmp_c[np + POPC(m & LANEMASK_LT)] = I.slots[si];
      np += POPC(m);
    }
    WSYNC();
    // drop the host's regions from the address order
    Tok freed = 0;
    for (int32_t r = head; r >= 0;) {
      const int32_t st = I.rg_start[r], ln = I.rg_len[r], nx = I.rg_next[r];
      const int32_t pos = addr_lower(I, st);
      arr_erase(I.addr, I.n_regions, pos, 1);
      UNI(I.n_regions--; I.reg_free[I.reg_free_top++] = r);
      freed += ln;
      r = nx;
    }
    UNI(I.reg_head[id] = -1; I.held[id] = 0);
    for (int32_t k = 0; k < np; ++k) {
      const int32_t sp = I.tmp_c[k];
      const int32_t h = I.sl_hosted[sp], sl = I.sl_len[sp];
      const int32_t r = region_new(I, h, I.sl_abs[sp], sl);
      if (r < 0) return;
      addr_insert_region(I, r);
      freed -= sl;
    }
    if (np > 0) {  // erase promoted slots (stable)
      int32_t w = 0;
      for (int32_t base = 0; base < I.n_slots; base += W) {
        const int32_t si = base + LANE;
        const int32_t sp = si < I.n_slots ? I.slots[si] : -1;
        const bool keep = sp >= 0 && I.sl_host[sp] != id;
        const bool drop = sp >= 0 && !keep;
        const unsigned m = BALLOT(keep), md = BALLOT(drop);
        WSYNC();
        if (keep) I.slots[w + POPC(m & LANEMASK_LT)] = sp;
        if (drop) {
          I.flags[I.sl_hosted[sp]] &= ~F_HAS_SLOT;
          I.sl_free[I.sl_free_top + POPC(md & LANEMASK_LT)] = sp;
        }
        w += POPC(m);
        WSYNC();
        UNI(I.sl_free_top += POPC(md));
      }
      UNI(I.n_slots = w);
    }
    UNI(I.free_total += freed);
  }
  // release_reserved (kvc.hpp:152-159) and the written count (kvc.hpp:92-101)
  UNI(if (f0 & F_HAS_RESERVED) { I.reserved_used -= rsv; I.reserved[id] = 0; }
        I.flags[id] = (uint8_t)(f0 & ~(F_HAS_RESERVED | F_HAS_SLOT));
        I.written_total -= wr; I.written[id] = 0);
}

// ------------------------------------------------------------------------
// GT queue (queues.hpp:125-204)
// ------------------------------------------------------------------------
EDEV uint64_t gkey_hi(const Inst& I, int32_t g) {
  if (!ORD(I)) return 0;
  return ((uint64_t)I.gr_db[g] << 56) | ((uint64_t)(255 - I.gr_kb[g]) << 48) |
         (0xFFFFFFFFFFFFULL - (uint64_t)I.gr_rl[g]);
}
EDEV bool gkey_less(const Inst& I, int32_t a, int32_t b) {
  const uint64_t ha = gkey_hi(I, a), hb = gkey_hi(I, b);
  if (ha != hb) return ha < hb;
  return I.gr_seq[a] < I.gr_seq[b];
}
EDEV int32_t gq_upper(const Inst& I, int32_t g) {  // upper_bound by key
  const uint64_t hg = gkey_hi(I, g), sg = I.gr_seq[g];
  const int32_t* gq = I.gq;
  return warp_search(I.G, [&](int32_t p) {
    const int32_t x = gq[p];
    const uint64_t hx = gkey_hi(I, x);
    return hg != hx ? hg < hx : sg < I.gr_seq[x];
  });
}
EDEV int32_t gq_pos(const Inst& I, int32_t g) {  // position of g (keys unique)
  const uint64_t hg = gkey_hi(I, g), sg = I.gr_seq[g];
  const int32_t* gq = I.gq;
  return warp_search(I.G, [&](int32_t p) {
    const int32_t x = gq[p];
    const uint64_t hx = gkey_hi(I, x);
    return !(hx != hg ? hx < hg : I.gr_seq[x] < sg);
  });
}
// place()'s re-insert at upper_bound (queues.hpp:187-197) and the removal of
// a group by its (unique) key.
EDEV void gq_insert(Inst& I, int32_t g) {
  const int32_t p2 = gq_upper(I, g);
  arr_insert(I.gq, I.G, p2, g);
  UNI(I.G++);
}
EDEV void gq_erase(Inst& I, int32_t g) {
  const int32_t pos = gq_pos(I, g);
  arr_erase(I.gq, I.G, pos, 1);
  UNI(I.G--);
}
EDEV void gq_rekey(Inst& I, int32_t g, double now) {  // place(): make_key (queues.hpp:187-193), lane 0
  if (ORD(I)) {
    I.gr_db[g] = bucket_d(I, dmax(0.0, I.gr_mindl[g] - now));
    I.gr_kb[g] = bucket_k(I, I.gr_maxocc[g]);
  }
}
EDEV int32_t rl_find(const Inst& I, int32_t rl) {
  if (rl >= 0 && rl < I.rl_cap) return I.rl_map[rl];
  for (int32_t base = 0; base < I.G; base += W) {  // rare: RL beyond the map
    const int32_t i = base + LANE;
    const unsigned m = BALLOT(i < I.G && I.gr_rl[I.gq[i < I.G ? i : 0]] == rl);
    if (m) return I.gq[base + FFS(m)];
  }
  return -1;
}
EDEV void rl_set(Inst& I, int32_t rl, int32_t g) {  // lane 0
  if (GRP(I) && rl >= 0 && rl < I.rl_cap) I.rl_map[rl] = g;
}
EDEV void gq_remove_at(Inst& I, int32_t pos) {  // drops the group from the queue and frees it
  const int32_t g = I.gq[pos];
  WSYNC();
  arr_erase(I.gq, I.G, pos, 1);
  UNI(I.G--; rl_set(I, I.gr_rl[g], -1); I.grp_free[I.grp_free_top++] = g);
}
EDEV Tok member_demand(const Inst& I, int32_t id) {  // gt_member_demand (engine.hpp:238-247)
  const Tok target = block_round((Tok)I.prompt[id] + I.generated[id] + padded_of(I, id), I.block);
  const Tok delta = target - I.held[id];
  return delta > 0 ? block_round(delta, I.block) : 0;
}
// group_insert_gt (queues.hpp:141-166). A waiting member's demand cannot
// change while it waits (its holdings and progress are frozen), so it is
// cached at join time and summed per group.
EDEVNI void group_insert_gt(Inst& I, int32_t id, int32_t padded, double deadline, int32_t occ, double now,
                            Tok d) {
  UNI(I.gt_next[id] = -1);
  if (GRP(I)) {
    const int32_t g = rl_find(I, padded);
    if (g >= 0) {
      // place() (queues.hpp:187-193) re-keys the group and re-inserts it at
      // upper_bound: keys are unique (the group's original seq), so when the
      // deadline and KVC buckets come out unchanged — always with ordering
      // off, where the key is the seq alone — the group stays where it is
      // and the queue is not touched.
      const int32_t cnt = I.gr_cnt[g], tail = I.gr_tail[g], mo = I.gr_maxocc[g];
      const int32_t odb = I.gr_db[g], okb = I.gr_kb[g];
      const int64_t gd = I.gr_dem[g];
      const double md = I.gr_mindl[g];
      const double nmd = dmin(md, deadline);
      const int32_t nmo = (int32_t)tmax(mo, occ);
      const int32_t ndb = ORD(I) ? bucket_d(I, dmax(0.0, nmd - now)) : odb;
      const int32_t nkb = ORD(I) ? bucket_k(I, nmo) : okb;
      const bool moved = ndb != odb || nkb != okb;
      if (moved) gq_erase(I, g);  // before the key fields change
      {  // warp-uniform (every lane, same values)
        if (cnt == 0) { I.gr_head[g] = id; I.gr_hd[g] = (int32_t)d; } else { I.gt_next[tail] = id; }
        I.gr_tail[g] = id;
        I.gr_cnt[g] = cnt + 1;
        I.gr_dem[g] = gd + d;
        I.gr_mindl[g] = nmd;
        I.gr_maxocc[g] = nmo;
        I.gr_db[g] = ndb;
        I.gr_kb[g] = nkb;
      }
      WSYNC();
      if (moved) gq_insert(I, g);
      return;
    }
  }
  if (I.grp_free_top <= 0 || I.G >= I.grp_cap) { set_error(I, ERR_TABLE_OVERFLOW, id, 4); return; }
  const int32_t g = I.grp_free[I.grp_free_top - 1];
  WSYNC();
  UNI(I.grp_free_top--;
        I.gr_id[g] = I.next_group_id++; I.gr_rl[g] = padded; I.gr_head[g] = id; I.gr_tail[g] = id;
        I.gr_hd[g] = (int32_t)d;
        I.gr_cnt[g] = 1; I.gr_dem[g] = d; I.gr_formed[g] = now; I.gr_mindl[g] = deadline;
        I.gr_maxocc[g] = occ; I.gr_seq[g] = I.gt_next_seq++;
        I.gr_db[g] = ORD(I) ? bucket_d(I, dmax(0.0, deadline - now)) : 0;
        I.gr_kb[g] = ORD(I) ? bucket_k(I, occ) : 0;
        rl_set(I, padded, g));
  gq_insert(I, g);
}
EDEV void group_insert_gt(Inst& I, int32_t id, int32_t padded, double deadline, int32_t occ, double now) {
  group_insert_gt(I, id, padded, deadline, occ, now, member_demand(I, id));
}

// ------------------------------------------------------------------------
// engine (engine.hpp:216-994), econoserve family
// ------------------------------------------------------------------------
// begin_gt_run (engine.hpp:350-363), lane 0. Every field is loaded before
// the first store: stores through the SoA pointers may alias later loads as
// far as the compiler knows, so interleaving them would serialise one
// memory round trip per field.
EDEV void begin_gt_run(Inst& I, int32_t id, bool hosted) {
  const uint8_t f = I.flags[id];
  const int32_t gen = I.generated[id], pad = padded_of(I, id);
  const double le = I.last_enq[id], wt = I.waiting[id], pt = I.preempt_t[id];
  const double wait = dmax(0.0, I.clock - le);
  uint8_t nf = hosted ? (uint8_t)(f | F_HOSTED) : (uint8_t)(f & ~F_HOSTED);
  I.flags[id] = (uint8_t)(nf & ~F_WAS_PREEMPTED);
  I.allowance[id] = gen + pad;
  I.gen_epoch[id] = gen;
  if (f & F_WAS_PREEMPTED) I.preempt_t[id] = pt + wait; else I.waiting[id] = wt + wait;
  I.state[id] = ST_RUNNING;
  I.run[I.R++] = id;
  I.adm[I.n_adm++] = id;
}

// ingest_arrivals (engine.hpp:216-235) for every arrival with t <= clock+1e-12.
// First index >= first whose arrival is > lim (arrivals are nondecreasing,
// so the due ones are a prefix): one warp probe of the next W arrivals
// answers the usual few-arrivals case in one load; a larger batch continues
// with a binary search.
EDEV int64_t due_end(const Inst& I, int64_t first, double lim) {
  const int64_t pos = first + LANE;
  const unsigned m = BALLOT(pos < I.n && I.arrival[pos < I.n ? pos : 0] <= lim);
  if (m != (W == 32 ? 0xffffffffu : 1u)) return first + POPC(m);  // prefix of due lanes
  int64_t lo = first + W, hi = I.n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (I.arrival[mid] <= lim) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <bool B>
EDEVNI void ingest(Inst& I) {
  const int64_t first = I.arrival_cursor;
  const double lim = I.clock + 1e-12;
  if (first >= I.n) return;
  const int64_t last = due_end(I, first, lim);
  if (last == first) return;
  const int64_t k = last - first;
  if (REC_EV(I)) {
    for (int64_t i = LANE; i < k; i += W) {
      const int64_t e = I.ev_n + i;
      if (e < I.ev_cap) {
        EconoEvent& ev = I.ev[e];
        ev.iter = I.iter; ev.clock = I.clock; ev.kind = ECONO_EV_ARRIVE; ev.id = (int32_t)(first + i);
        ev.a = 0; ev.b = 0;
      }
    }
  }
  if (B && I.policy == ECONO_POLICY_SYNC_COUPLED) {
    // sync-coupled: arrivals join the waiting groups (engine.hpp:226-228)
    for (int64_t id = first; id < last; ++id)
      group_insert_gt(I, (int32_t)id, padded_of(I, id), slo_of(I, id), 0, I.clock);
    UNI(I.arrival_cursor = last; I.ev_total += k; if (REC_EV(I)) I.ev_n += k);
    return;
  }
  if (!B) {
    int64_t pm = INT64_MAX;
    for (int64_t id = first + LANE; id < last; id += W) pm = I.prompt[id] < pm ? I.prompt[id] : pm;
    pm = wmin(pm);
    UNI(if (pm < I.pt_min_lb) I.pt_min_lb = pm);
  }
  if (!B && ORD(I)) {
    // class append in id order: peers of a class inside each warp chunk link
    // to each other; the lowest links to the class tail, the highest becomes it.
    for (int64_t base = first; base < last; base += W) {
      const int64_t id = base + LANE;
      const bool ok = id < last;
      int cls = -1 - LANE;
      int b = 0, p = 0;
      if (ok) {
        b = bucket_d(I, dmax(0.0, slo_of(I, id) - I.clock));
        p = I.prompt[id];
        cls = cls_of(I, b, p);
      }
      const unsigned grp = MATCH_ANY(cls);
      const unsigned bgrp = MATCH_ANY(ok ? b : -1 - LANE);
      if (ok && (bgrp & LANEMASK_LT) == 0) SMEM_ADD(&I.bcnt[b], (int32_t)POPC(bgrp));
      int32_t old_tail = -1;
      if (ok) old_tail = I.cls_tail[cls];
      WSYNC();
      if (ok) {
        const unsigned higher = grp & ~((2u << LANE) - 1u);
        I.pt_next[id] = higher ? (int32_t)(base + FFS(higher)) : -1;
        const bool lowest = (grp & LANEMASK_LT) == 0;
        const bool highest = higher == 0;
        if (lowest) {
          if (old_tail >= 0) I.pt_next[old_tail] = (int32_t)id; else I.cls_head[cls] = (int32_t)id;
          I.cls_cnt[cls] += POPC(grp);
        }
        if (highest) I.cls_tail[cls] = (int32_t)id;
      }
      WSYNC();
      if (ok) bm_set_shared(I, b, p);  // bitmap words are shared between classes
      WSYNC();
    }
  } else {
    // FIFO PT queue, or the baselines' wait_fifo_ (engine.hpp:229-230): a
    // sorted id set (arrivals append in id order, preemptions re-insert at
    // lower_bound), leaves hold the forward-size demand (the prompt).
    for (int64_t id = first + LANE; id < last; id += W) I.tree[id] = I.prompt[id];
    WSYNC();
    tree_fix(I, first, last - 1);
  }
  UNI(I.arrival_cursor = last; I.pt_count += (int32_t)k; I.ev_total += k;
        if (REC_EV(I)) I.ev_n += k);
}

// Takes up to k entries from the head of class (b,p); appends ids to out.
EDEV int32_t cls_take(Inst& I, int b, int p, int32_t k, int32_t* out, int32_t nout) {
  const int32_t c = cls_of(I, b, p);
  {  // warp-uniform (every lane, same values)
    int32_t h = I.cls_head[c];
    for (int32_t i = 0; i < k; ++i) {
      out[nout + i] = h;
      h = I.pt_next[h];
    }
    I.cls_head[c] = h;
    I.cls_cnt[c] -= k;
    I.bcnt[b] -= k;
    if (I.cls_cnt[c] == 0) {
      I.cls_tail[c] = -1;
      I.cls_head[c] = -1;
      bm_clear(I, b, p);
    }
    I.pt_count -= k;
  }
  WSYNC();
  return nout + k;
}

// dispatch_pt_reserved / _common (engine.hpp:365-381) for the npt selected
// PTs in I.tmp_a, lane-parallel: every lane loads its PT's fields at once,
// a prefix sum of the prompts replays draw_reserved's sequential capacity
// test (kvc.hpp:144-150) and the first failing draw is the error, exactly
// where the sequential loop would stop. Event slots, ptiter and adm
// positions are assigned in selection order.
EDEVNI void dispatch_pts(Inst& I, int32_t npt) {
  for (int32_t base = 0; base < npt; base += W) {
    const int32_t j = base + LANE;
    const bool on = j < npt;
    int32_t id = 0, p = 0, rsv = 0;
    uint8_t f = 0;
    double arr = 0.0, wt = 0.0;
    if (on) {
      id = I.tmp_a[j];
      p = I.prompt[id];
      rsv = I.reserved[id];
      f = I.flags[id];
      arr = I.arrival[id];
      wt = I.waiting[id];
    }
    Tok incl = on ? p : 0;  // inclusive prefix of prompt tokens within the chunk
    for (int o = 1; o < W; o <<= 1) {
      const Tok y = shfl(incl, LANE - o >= 0 ? LANE - o : 0);
      if (LANE >= o) incl += y;
    }
    const Tok used0 = I.reserved_used;
    const bool fits = !on || used0 + incl <= I.reserve_cap;
    const unsigned bad = BALLOT(!fits);
    const int32_t cnt = bad ? FFS(bad) : (npt - base < W ? npt - base : W);
    if (on && LANE < cnt) {
      I.reserved[id] = rsv + p;
      I.flags[id] = (uint8_t)(f | F_HAS_RESERVED);
      I.state[id] = ST_RUNNING;
      I.waiting[id] = wt + (I.clock - arr);
      I.ptiter_id[I.n_ptiter + LANE] = id;
      I.ptiter_tok[I.n_ptiter + LANE] = p;
      I.adm[I.n_adm + LANE] = id;
      if (REC_EV(I) && I.ev_n + LANE < I.ev_cap) {
        EconoEvent& e = I.ev[I.ev_n + LANE];
        e.iter = I.iter; e.clock = I.clock; e.kind = ECONO_EV_PT_DISPATCH; e.id = id; e.a = 0; e.b = 0;
      }
    }
    const Tok took = shfl(incl, cnt > 0 ? cnt - 1 : 0);
    const int32_t bad_id = shfl(id, cnt < W ? cnt : 0);
    WSYNC();
    UNI(I.reserved_used = used0 + (cnt > 0 ? took : 0); I.n_ptiter += cnt; I.n_adm += cnt;
          I.pts_admitted_iter += cnt; I.pt_dispatched += cnt; I.ev_total += cnt;
          if (REC_EV(I)) I.ev_n += cnt);
    if (bad) { set_error(I, ERR_RESERVED_DRAW, bad_id, 0); return; }
  }
}

// schedule_gt_member (engine.hpp:327-348): exact allocation, then the
// reserve release (kvc.hpp:152-159), written/occupied accounting and
// begin_gt_run in one lane-0 block whose loads all precede its stores.
EDEVNI void schedule_gt_member(Inst& I, int32_t id) {
  const Tok prompt = I.prompt[id], gen = I.generated[id], pad = padded_of(I, id);
  const Tok target = block_round(prompt + gen + pad, I.block);
  const Tok held = I.held[id];
  const Tok resident = prompt + gen;
  bool ok = true;
  if (held == 0) ok = kvc_alloc_region(I, id, prompt + gen + pad);
  else if (held < target) ok = kvc_alloc_region(I, id, target - held);
  if (I.error) return;
  if (!ok) { set_error(I, ERR_ALLOC_FAIL, id, 0); return; }
  {  // warp-uniform (every lane, same values)
    const uint8_t f = I.flags[id];
    const int32_t rsv = I.reserved[id], cur = I.written[id];
    const double le = I.last_enq[id], wt = I.waiting[id], pt = I.preempt_t[id];
    if (f & F_HAS_RESERVED) {
      I.reserved_used -= rsv;
      I.reserved[id] = 0;
    }
    if (cur < resident) {
      I.written[id] = (int32_t)resident;
      I.written_total += resident - cur;
    }
    I.occupied[id] = (int32_t)resident;
    const double wait = dmax(0.0, I.clock - le);
    I.flags[id] = (uint8_t)(f & ~(F_HAS_RESERVED | F_HOSTED | F_WAS_PREEMPTED));
    I.allowance[id] = (int32_t)(gen + pad);
    I.gen_epoch[id] = (int32_t)gen;
    if (f & F_WAS_PREEMPTED) I.preempt_t[id] = pt + wait; else I.waiting[id] = wt + wait;
    I.state[id] = ST_RUNNING;
    I.run[I.R++] = id;
    I.adm[I.n_adm++] = id;
    I.gt_scheduled++;
  }
  logev(I, ECONO_EV_GT_SCHEDULE, id, pad, 0);
  WSYNC();
}

// plan_pipeline (kvc_pipeline.hpp:29-136). Host group h's members are
// I.tmp_b[hs..he) (ids) with write bases I.tmp_c[hs..he). Appends planned
// slots to the os_* arrays; returns the new count.
ECOLD int32_t plan_host_group(Inst& I, int32_t l, int32_t hs, int32_t he, int32_t nout, int64_t* exams) {
  if (l < 2 || he <= hs) return nout;
  const Tok b = ceil_tokens(I.buffer_ratio * (double)l);
  int32_t nr = he - hs;
  int32_t *rw = I.wa_w, *rb = I.wa_b, *rlen = I.wa_l, *ru = I.wa_u;
  int32_t *nw = I.wb_w, *nb = I.wb_b, *nlen = I.wb_l, *nu = I.wb_u;
  for (int32_t i = LANE; i < nr; i += W) {
    rw[i] = I.tmp_b[hs + i];
    rb[i] = I.tmp_c[hs + i];
    rlen[i] = l;
    ru[i] = 0;
  }
  WSYNC();
  for (int level = 1;; ++level) {
    const Tok bound = (level >= 62 ? 0 : (Tok)l / ((Tok)1 << level)) - b;
    if (bound < 1) break;
    // candidates: second halves of regions with half >= 1, in region order
    int32_t nc = 0;
    for (int32_t base = 0; base < nr; base += W) {
      const int32_t ri = base + LANE;
      const int32_t half = ri < nr ? rlen[ri] / 2 : 0;
      const bool ok = ri < nr && half >= 1;
      const unsigned m = BALLOT(ok);
      if (ok) {
        const int32_t o = nc + POPC(m & LANEMASK_LT);
        I.cd_ri[o] = ri;
        I.cd_abs[o] = rb[ri] + (rlen[ri] - half);
        I.cd_use[o] = ru[ri] + (rlen[ri] - half);
        I.cd_len[o] = half;
      }
      nc += POPC(m);
    }
    WSYNC();
    if (nc == 0) break;
    if (LANE == 0) {  // std::shuffle (stl_algo.h:3719-3795) with the engine rng_
      const uint64_t n = (uint64_t)nc;
      auto swp = [&](uint64_t i, uint64_t j) {
        if (i == j) return;
        int32_t t;
        t = I.cd_ri[i]; I.cd_ri[i] = I.cd_ri[j]; I.cd_ri[j] = t;
        t = I.cd_abs[i]; I.cd_abs[i] = I.cd_abs[j]; I.cd_abs[j] = t;
        t = I.cd_use[i]; I.cd_use[i] = I.cd_use[j]; I.cd_use[j] = t;
        t = I.cd_len[i]; I.cd_len[i] = I.cd_len[j]; I.cd_len[j] = t;
      };
      uint64_t i = 1;
      if ((n % 2) == 0) { swp(i, uniform_u64(I.mt, I.mt_i, 0, 1)); ++i; }
      while (i != n) {
        const uint64_t sr = i + 1;
        const uint64_t x = uniform_u64(I.mt, I.mt_i, 0, sr * (sr + 1) - 1);
        const uint64_t p1 = x / (sr + 1), p2 = x % (sr + 1);
        swp(i, p1); ++i;
        swp(i, p2); ++i;
      }
    }
    for (int32_t i = LANE; i < nr; i += W) I.assigned[i] = -1;
    WSYNC();
    int32_t next_slot = 0;
    bool any = false;
    while (next_slot < nc) {
      // the group with RL <= bound closest to it; FCFS on ties (kvc_pipeline.hpp:77-86)
      *exams += I.G;
      int32_t best = -1, bpos = -1;
      for (int32_t base = 0; base < I.G; base += W) {
        const int32_t pi = base + LANE;
        if (pi < I.G) {
          const int32_t g = I.gq[pi];
          if (I.gr_cnt[g] > 0 && I.gr_rl[g] <= bound) {
            bool better = best < 0;
            if (!better) {
              better = I.gr_rl[g] > I.gr_rl[best] ||
                       (I.gr_rl[g] == I.gr_rl[best] &&
                        (I.gr_formed[g] < I.gr_formed[best] ||
                         (I.gr_formed[g] == I.gr_formed[best] && I.gr_id[g] < I.gr_id[best])));
            }
            if (better) { best = g; bpos = pi; }
          }
        }
      }
      for (int o = W / 2; o > 0; o >>= 1) {
        const int32_t ob = shfl_xor(best, o), op = shfl_xor(bpos, o);
        if (ob >= 0) {
          bool better = best < 0;
          if (!better) {
            better = I.gr_rl[ob] > I.gr_rl[best] ||
                     (I.gr_rl[ob] == I.gr_rl[best] &&
                      (I.gr_formed[ob] < I.gr_formed[best] ||
                       (I.gr_formed[ob] == I.gr_formed[best] && I.gr_id[ob] < I.gr_id[best])));
          }
          if (better) { best = ob; bpos = op; }
        }
      }
      best = shfl(best, 0);
      bpos = shfl(bpos, 0);
      if (best < 0) break;
      any = true;
      const int32_t take = I.gr_cnt[best] < nc - next_slot ? I.gr_cnt[best] : nc - next_slot;
      if (nout + take > 2 * I.scr_cap) { set_error(I, ERR_TABLE_OVERFLOW, -1, 7); return nout; }
      if (LANE == 0) {
        int32_t m = I.gr_head[best];
        Tok dsum = 0;
        for (int32_t i = 0; i < take; ++i) {
          const int32_t ci = next_slot + i;
          const int32_t ri = I.cd_ri[ci];
          I.os_host[nout + i] = rw[ri];
          I.os_hosted[nout + i] = m;
          I.os_off[nout + i] = I.cd_use[ci];
          I.os_len[nout + i] = I.cd_len[ci];
          I.os_abs[nout + i] = I.cd_abs[ci];
          I.assigned[ri] = m;
          dsum += member_demand(I, m);
          m = I.gt_next[m];
        }
        I.gr_head[best] = m;
        if (m >= 0) I.gr_hd[best] = (int32_t)member_demand(I, m);
        I.gr_cnt[best] -= take;
        I.gr_dem[best] -= dsum;
        if (I.gr_cnt[best] == 0) I.gr_tail[best] = -1;
      }
      WSYNC();
      nout += take;
      next_slot += take;
      if (I.gr_cnt[best] == 0) gq_remove_at(I, bpos);
    }
    if (!any) break;
    // halve every region (kvc_pipeline.hpp:540-556 in the reference order)
    int32_t nn = 0;
    for (int32_t base = 0; base < nr; base += W) {
      const int32_t ri = base + LANE;
      const bool ok = ri < nr;
      const int32_t half = ok ? rlen[ri] / 2 : 0;
      const int32_t cnt = ok ? (half < 1 ? 1 : 2) : 0;
      int32_t incl = cnt;
      for (int o = 1; o < W; o <<= 1) {
        const int32_t y = shfl(incl, LANE - o >= 0 ? LANE - o : 0);
        if (LANE >= o) incl += y;
      }
      if (ok) {
        const int32_t o = nn + incl - cnt;
        if (half < 1) {
          nw[o] = rw[ri]; nb[o] = rb[ri]; nlen[o] = rlen[ri]; nu[o] = ru[ri];
        } else {
          const int32_t kept = rlen[ri] - half;
          nw[o] = rw[ri]; nb[o] = rb[ri]; nlen[o] = kept; nu[o] = ru[ri];
          if (I.assigned[ri] >= 0) {
            nw[o + 1] = I.assigned[ri]; nb[o + 1] = rb[ri] + kept; nlen[o + 1] = half; nu[o + 1] = 0;
          } else {
            nw[o + 1] = rw[ri]; nb[o + 1] = rb[ri] + kept; nlen[o + 1] = half; nu[o + 1] = ru[ri] + kept;
          }
        }
      }
      nn += shfl(incl, W - 1);
    }
    WSYNC();
    if (nn > I.scr_cap) { set_error(I, ERR_TABLE_OVERFLOW, -1, 5); return nout; }
    int32_t* t;
    t = rw; rw = nw; nw = t;
    t = rb; rb = nb; nb = t;
    t = rlen; rlen = nlen; nlen = t;
    t = ru; ru = nu; nu = t;
    nr = nn;
  }
  return nout;
}

// add_slot containment (kvc.hpp:219-224, 318-332)
EDEV bool slot_fits(const Inst& I, int32_t host, int32_t abs, int32_t len) {
  for (int32_t r = I.reg_head[host]; r >= 0; r = I.rg_next[r])
    if (abs >= I.rg_start[r] && abs + len <= I.rg_start[r] + I.rg_len[r]) return true;
  if (I.flags[host] & F_HAS_SLOT) {
    const int32_t sp = I.sidx[host];
    if (abs >= I.sl_abs[sp] && abs + len <= I.sl_abs[sp] + I.sl_len[sp]) return true;
  }
  return false;
}

// select_gt_groups (queues.hpp:220-263) over the GT queue — econoserve's
// gt_queue_ or sync-coupled's waiting_groups_ (engine.hpp:712-713): takes
// whole groups in key order while their cached demand fits the free KVC,
// splits the first misfit member by member and stops. Selected ids go to
// I.sel_ids, group bounds to I.selg_start / I.selg_rl; returns the number of
// selected groups, *nsel_out the number of members.
EDEVNI int32_t select_gt(Inst& I, int32_t* nsel_out) {
  int32_t nsel = 0, nselg = 0, whole = 0;
  if (I.free_total > 0) {
    Tok remaining = I.free_total;
    int32_t gi = 0;
    while (gi < I.G) {
      const int32_t g = I.gq[gi];
      const Tok total = I.gr_dem[g];  // the group's fields load together
      const int32_t cnt = I.gr_cnt[g], head = I.gr_head[g], grl = I.gr_rl[g];
      UNI(I.exam_count++);
      if (nsel + cnt > I.sel_cap && total <= remaining) { set_error(I, ERR_TABLE_OVERFLOW, g, 8); return 0; }
      if (total <= remaining) {
        remaining -= total;
        {  // warp-uniform (every lane, same values)
          I.selg_start[nselg] = nsel;
          I.selg_rl[nselg] = grl;
          int32_t m = head;
          for (int32_t i = 0; i < cnt; ++i) { I.sel_ids[nsel + i] = m; m = I.gt_next[m]; }
          rl_set(I, grl, -1);  // the group leaves the queue (erased below, in one shift)
          I.grp_free[I.grp_free_top++] = g;
        }
        WSYNC();
        nsel += cnt;
        nselg++;
        whole++;
        gi++;
        continue;
      }
      int32_t taken = 0, m = head;
      Tok pd = 0, dm = 0;
      {  // warp-uniform (every lane, same values)
        Tok d = I.gr_hd[g];
        while (m >= 0) {
          const int32_t nx = I.gt_next[m];
          I.exam_count++;
          if (pd + d > remaining) { dm = d; break; }
          pd += d;
          I.sel_ids[nsel + taken] = m;
          taken++;
          m = nx;
          if (m >= 0) d = member_demand(I, m);
        }
      }
      dm = shfl(dm, 0);
      taken = shfl(taken, 0);
      m = shfl(m, 0);
      pd = shfl(pd, 0);
      if (taken > 0) {
        UNI(I.selg_start[nselg] = nsel; I.selg_rl[nselg] = I.gr_rl[g];
              I.gr_head[g] = m; I.gr_hd[g] = (int32_t)dm; I.gr_cnt[g] -= taken; I.gr_dem[g] -= pd);
        nsel += taken;
        nselg++;
        remaining -= pd;
      }
      break;
    }
    if (whole > 0) {
      WSYNC();
      arr_erase(I.gq, I.G, 0, whole);
      UNI(I.G -= whole);
    }
  }
  UNI(I.selg_start[nselg] = nsel);
  *nsel_out = nsel;
  return nselg;
}

EDEVNI void form_econoserve(Inst& I) {  // engine.hpp:263-325
  // ---- select_gt_groups (queues.hpp:220-263) ----
  [[maybe_unused]] const int64_t tp0 = PHASE_NOW();
  int32_t nsel = 0;
  const int32_t nselg = select_gt(I, &nsel);
  if (I.error) return;
  for (int32_t i = 0; i < nsel; ++i) {
    schedule_gt_member(I, I.sel_ids[i]);
    if (I.error) return;
  }

  [[maybe_unused]] const int64_t tp1 = PHASE_NOW();
  PHASE_ADD(7, tp1 - tp0);
  // ---- KVC pipelining (econoserve-full, engine.hpp:273-297) ----
  if (FULL(I) && nselg > 0) {
    int32_t nm = 0;  // host members flattened into tmp_b/tmp_c, group bounds in tmp_a
    for (int32_t gi = 0; gi < nselg; ++gi) {
      {  // warp-uniform (every lane, same values)
        I.tmp_a[gi] = nm;
        for (int32_t i = I.selg_start[gi]; i < I.selg_start[gi + 1]; ++i) {
          const int32_t id = I.sel_ids[i];
          const int32_t rh = I.reg_head[id];
          if (I.generated[id] == 0 && rh >= 0 && I.rg_next[rh] < 0) {  // exactly one region
            I.tmp_b[nm] = id;
            I.tmp_c[nm] = I.rg_start[rh] + I.prompt[id];
            nm++;
          }
        }
      }
      nm = shfl(nm, 0);
      WSYNC();
    }
    UNI(I.tmp_a[nselg] = nm);
    if (nm > 0 && I.G > 0) {
      int64_t exams = 0;
      int32_t nout = 0;
      for (int32_t gi = 0; gi < nselg; ++gi) {
        const int32_t hs = I.tmp_a[gi], he = I.tmp_a[gi + 1];
        nout = plan_host_group(I, I.selg_rl[gi], hs, he, nout, &exams);
        if (I.error) return;
      }
      UNI(I.exam_count += exams);
      for (int32_t i = 0; i < nout; ++i) {
        const int32_t host = I.os_host[i], hosted = I.os_hosted[i];
        const int32_t abs = I.os_abs[i], len = I.os_len[i];
        if (!slot_fits(I, host, abs, len)) { set_error(I, ERR_SLOT_OUTSIDE, hosted, 0); return; }
        if (I.n_slots >= I.slot_cap) { set_error(I, ERR_TABLE_OVERFLOW, hosted, 6); return; }
        {  // warp-uniform (every lane, same values)
          const int32_t sp = I.sl_free[--I.sl_free_top];
          I.sl_host[sp] = host;
          I.sl_off[sp] = I.os_off[i];
          I.sl_len[sp] = len;
          I.sl_abs[sp] = abs;
          I.sl_hosted[sp] = hosted;
          I.sidx[hosted] = sp;
          I.flags[hosted] |= F_HAS_SLOT;
          I.slots[I.n_slots++] = sp;
          I.hosted_total++;
          begin_gt_run(I, hosted, true);
          I.gt_scheduled++;
        }
        logev(I, ECONO_EV_HOSTED, hosted, host, I.os_off[i]);
        WSYNC();
      }
    }
  }

  [[maybe_unused]] const int64_t tp2 = PHASE_NOW();
  PHASE_ADD(8, tp2 - tp1);
  // ---- PT batching (engine.hpp:299-324, queues.hpp:279-299) ----
  const Tok tfs_rem = I.tfs - (Tok)I.R;
  const Tok rfree = I.reserve_cap - I.reserved_used;
  const Tok C0 = tmin(tfs_rem, rfree);
  int32_t npt = 0;
  if (I.pt_count > 0) {
    // pt_admittable (engine.hpp:301-307): some queued prompt fits both budgets
    bool adm = false;
    int adm_b = -1, adm_p = -1;  // the first bucket with a fitting class, and that class
    if (C0 >= 1 && C0 >= I.pt_min_lb) {
      if (ORD(I)) {
        for (int b = 0; b < I.nbuckets; ++b) {
          const int p = bm_prev(I, b, C0);
          if (p >= 1) { adm_b = b; adm_p = p; break; }
        }
        adm = adm_b >= 0;
      } else {
        adm = I.tree[I.tree_off[I.tree_levels - 1]] <= C0;
      }
      if (!adm) UNI(I.pt_min_lb = C0 + 1);
    }
    if (adm) UNI(I.pt_admittable = 1);
    if (tfs_rem > 0 && rfree > 0) {
      UNI(I.exam_count += I.pt_count);
      Tok C = C0;  // both budgets drop by p: take iff p <= min(budgets)
      if (!adm) {
        // nothing fits (the admittable probe above used the same bound)
      } else if (ORD(I)) {
        // buckets before adm_b hold nothing <= C0, and adm_b's first probe at
        // C0 is the admittable probe's answer; once the budget is below the
        // smallest queued prompt (pt_min_lb) nothing further can fit
        bool done = false;
        for (int b = adm_b; b < I.nbuckets && C > 0 && !done; ++b) {
          int p = b == adm_b ? adm_p : bm_prev(I, b, C);
          while (p >= 1) {
            const int32_t cnt = I.cls_cnt[cls_of(I, b, p)];
            const Tok fit = udiv(C, p);
            const int32_t k = (int32_t)(fit < cnt ? fit : cnt);
            npt = cls_take(I, b, p, k, I.tmp_a, npt);
            C -= (Tok)k * p;
            if (C < I.pt_min_lb) { done = true; break; }
            const Tok x = tmin((Tok)p - 1, C);
            if (x < 1) break;
            p = bm_prev(I, b, x);
          }
        }
      } else {
        int64_t pos = 0;
        while (C > 0) {
          const int32_t id = tree_first(I, pos, C);
          if (id < 0) break;
          UNI(I.tmp_a[npt] = id; I.pt_count--);
          npt++;
          C -= I.prompt[id];
          tree_set(I, id, INF32);
          pos = (int64_t)id + 1;
        }
      }
    }
    if (npt == 0 && I.pt_count > 0 && I.R == 0) {  // starvation guard (engine.hpp:314-323)
      if (ORD(I)) {
        for (int b = 0; b < I.nbuckets; ++b) {
          const int p = bm_prev(I, b, rfree);
          if (p >= 1) { npt = cls_take(I, b, p, 1, I.tmp_a, npt); break; }
        }
      } else {
        const int32_t id = tree_first(I, 0, rfree);
        if (id >= 0) {
          UNI(I.tmp_a[0] = id; I.pt_count--);
          npt = 1;
          tree_set(I, id, INF32);
        }
      }
    }
  }
  dispatch_pts(I, npt);
  PHASE_ADD(9, PHASE_NOW() - tp2);
}

#include "baselines.cuh"

ECOLD void vacate_slot(Inst& I, int32_t id, bool* rehomed) {  // engine.hpp:888-902
  const Tok in_slot = tmin((Tok)I.generated[id] - I.gen_epoch[id], (Tok)padded_of(I, id));
  bool rh = false;
  if (in_slot > 0 && kvc_draw_reserved(I, id, in_slot)) {
    rh = true;
  } else if (in_slot > 0) {
    UNI(const Tok w = I.written[id]; const Tok d = tmin(in_slot, w);
          I.written[id] -= (int32_t)d; I.written_total -= d; I.occupied[id] -= (int32_t)in_slot);
  }
  kvc_remove_slot(I, id);
  UNI(I.flags[id] &= ~F_HOSTED);
  *rehomed = rh;
}

template <bool B>
ECOLD void preempt_and_regroup(Inst& I, int32_t id, int why) {  // engine.hpp:904-928
  if (B) list_erase(I.admo, &I.n_admo, id);
  if (LANE == 0) {
    I.preempt_count[id]++;
    I.state[id] = ST_PREEMPTED;
    const Tok remaining = (Tok)I.true_rl[id] - I.generated[id];
    I.predicted[id] = sat_rl(predict_rl(I, remaining, I.pmt, I.pmt_i));
    I.flags[id] |= F_WAS_PREEMPTED;
    I.last_enq[id] = I.clock;
  }
  WSYNC();
  logev(I, ECONO_EV_PREEMPT, id, why, padded_of(I, id));
  UNI(I.state[id] = ST_WAITING_GT);
  if (B && I.policy != ECONO_POLICY_SYNC_COUPLED) {
    wait_insert(I, id);
    return;
  }
  group_insert_gt(I, id, padded_of(I, id), slo_of(I, id), I.occupied[id], I.clock);
}

template <bool B>
ECOLD void handle_underprediction(Inst& I, int32_t id) {  // engine.hpp:856-873
  if (!B && kvc_draw_reserved(I, id, I.block)) {
    UNI(I.allowance[id] += (int32_t)I.block; I.reserve_draws[id]++;
          I.penalty[id] += I.reserve_penalty);
    logev(I, ECONO_EV_RESERVE_TOPUP, id, 0, 0);
    WSYNC();
    return;
  }
  UNI(I.flags[id] |= F_ALLOC_FAIL; I.alloc_failures++);
  bool rehomed = true;
  if (I.flags[id] & F_HOSTED) vacate_slot(I, id, &rehomed);
  UNI(I.penalty[id] += rehomed ? I.pen_free : I.pen_offload);
  preempt_and_regroup<B>(I, id, 0);
}

ECOLD void handle_hosted_overrun(Inst& I, int32_t id) {  // engine.hpp:875-884
  UNI(I.hosted_overruns++);
  bool rehomed = false;
  vacate_slot(I, id, &rehomed);
  UNI(I.penalty[id] += rehomed ? I.pen_free : I.pen_offload; I.flags[id] |= F_ALLOC_FAIL;
        I.alloc_failures++);
  logev(I, ECONO_EV_HOSTED_OVERRUN, id, 0, 0);
  WSYNC();
  preempt_and_regroup<false>(I, id, 1);
}

// Stable compaction of the running list to RUNNING requests.
EDEV void run_compact(Inst& I) {
  int32_t w = 0;
  for (int32_t base = 0; base < I.R; base += W) {
    const int32_t i = base + LANE;
    const int32_t id = i < I.R ? I.run[i] : -1;
    const bool keep = id >= 0 && I.state[id] == ST_RUNNING;
    const unsigned m = BALLOT(keep);
    WSYNC();
    if (keep) I.run[w + POPC(m & LANEMASK_LT)] = id;
    w += POPC(m);
    WSYNC();
  }
  UNI(I.R = w);
}

template <bool B>
EDEVNI void execute_iteration(Inst& I, Tok fs) {  // engine.hpp:731-840
  [[maybe_unused]] const int64_t tx0 = PHASE_NOW();
  const double dt = iteration_time(I, fs) + (B ? I.pending_stall : 0.0);
  UNI(I.clock += dt; I.iter++; if (B) I.pending_stall = 0.0);
  const bool pause = B && I.decode_pause;
  const double sched = (double)I.exam_count * I.sched_cost;
  if (I.n_adm > 0 && sched > 0.0) {
    const double share = sched / (double)I.n_adm;
    for (int32_t i = LANE; i < I.n_adm; i += W) I.sched_share[I.adm[i]] += share;
  }
  // prefill + decode progress (per-request updates are independent)
  Tok wsum_pt = 0;
  for (int32_t i = LANE; i < I.n_ptiter; i += W) {
    const int32_t id = I.ptiter_id[i];
    const int32_t tk = I.ptiter_tok[i];
    const double e = I.exec_t[id];
    // econoserve prefills a prompt whole in its dispatch iteration, so its
    // prefill_done is 0 before and the prompt after: derived, not stored
    const int32_t pd = (B ? I.prefill_done[id] : 0) + tk, wr = I.written[id], oc = I.occupied[id];
    const int32_t pr = B ? I.ptarget[id] : I.prompt[id];
    const uint8_t f = I.flags[id];
    I.exec_t[id] = e + dt;
    if (B) I.prefill_done[id] = pd;
    I.written[id] = wr + tk;
    I.occupied[id] = oc + tk;
    wsum_pt += tk;
    if (pd >= pr) I.flags[id] = (uint8_t)(f | F_PREFILL_FIN);
  }
  wsum_pt = wsum32((int32_t)wsum_pt);  // prompt tokens of one iteration (< reserve capacity < 2^30)
  // every running GT writes exactly one token this iteration
  UNI(I.written_total += wsum_pt + (pause ? 0 : I.R));
  EconoSample s;
  s.iter = I.iter;
  s.clock = I.clock;
  s.dt = dt;
  s.forward_size = fs;
  s.kvc_written_frac = (double)I.written_total / (double)I.capacity;
  s.kvc_allocated_frac = (double)((I.general_cap - I.free_total) + I.reserved_used) / (double)I.capacity;
  s.completed = 0;
  s.pts_admitted = I.pts_admitted_iter;
  s.pt_admittable = I.pt_admittable;
  s._pad = 0;
  s.idle_repeat = 0;
  // One pass over the running set (engine.hpp:763-771, 784-791, 812-817):
  // decode progress, then completion and under-prediction tests on the new
  // counts. All fields of a request load in parallel; completions are
  // processed chunk by chunk in running order. Releasing a finished request
  // touches only its own counters, regions and the slots it hosts, never
  // another running request's progress, so it may precede the next chunk's
  // decode. Under-prediction candidates (generated >= allowance < true_rl)
  // are collected here in running order; completed requests never qualify.
  [[maybe_unused]] const int64_t tx1 = PHASE_NOW();
  PHASE_ADD(13, tx1 - tx0);
  int32_t completed_now = 0, npre = 0;
  const int32_t R0 = I.R;
  int32_t id_c0 = -1;   // the first chunk's ids and survivors: with R0 <= W the
  unsigned keep0 = 0;   // running list is compacted from the ballot, no re-read
  for (int32_t base = 0; base < R0; base += W) {
    const int32_t i = base + LANE;
    const int32_t id = i < R0 ? I.run[i] : -1;
    bool fin = false, under = false;
    if (pause && id >= 0) {  // vLLM prefill-only iteration: decodes stall (engine.hpp:744-749)
      const double wt = I.waiting[id];
      const int32_t g = I.generated[id], tr = I.true_rl[id], al = I.allowance[id];
      I.waiting[id] = wt + dt;
      fin = g >= tr;
      under = g >= al && g < tr;
    } else if (id >= 0) {
      const double e = I.exec_t[id];
      const int32_t g = I.generated[id] + 1;
      const int32_t oc = I.occupied[id], wr = I.written[id], tr = I.true_rl[id], al = I.allowance[id];
      const double ft = I.first_tok[id];
      I.exec_t[id] = e + dt;
      I.generated[id] = g;
      I.occupied[id] = oc + 1;
      I.written[id] = wr + 1;
      if (g == 1 && ft < 0.0) I.first_tok[id] = I.clock;
      fin = g >= tr;
      under = g >= al && g < tr;
    }
    const unsigned mu = BALLOT(under);
    if (under) I.tmp_a[npre + POPC(mu & LANEMASK_LT)] = id;
    npre += POPC(mu);
    unsigned m = BALLOT(fin);
    if (base == 0) {
      id_c0 = id;
      keep0 = BALLOT(id >= 0 && !fin);
    }
    WSYNC();
    while (m) {
      const int l = FFS(m);
      m &= m - 1;
      const int32_t cid = shfl(id, l);
      UNI(I.state[cid] = ST_DONE; I.compl_clock[cid] = I.clock);
      kvc_release(I, cid);
      if (I.error) return;
      UNI(I.occupied[cid] = 0; I.completed++);
      if (B) list_erase(I.admo, &I.n_admo, cid);
      logev(I, ECONO_EV_COMPLETE, cid, I.generated[cid], 0);
      WSYNC();
      completed_now++;
    }
  }
  if (completed_now) {
    if (R0 <= W) {  // releases never change another running request's state
      if ((keep0 >> LANE) & 1u) I.run[POPC(keep0 & LANEMASK_LT)] = id_c0;
      WSYNC();
      UNI(I.R = POPC(keep0));
    } else {
      run_compact(I);
    }
  }
  [[maybe_unused]] const int64_t tx2 = PHASE_NOW();
  PHASE_ADD(3, tx2 - tx1);
  // prefill transitions (engine.hpp:794-809)
  for (int32_t i = 0; i < I.n_ptiter; ++i) {
    const int32_t id = I.ptiter_id[i];
    const uint8_t f = I.flags[id];
    const uint8_t st = I.state[id];
    const int32_t pad = padded_of(I, id), oc = I.occupied[id], pr = I.prompt[id], gen = I.generated[id];
    const int32_t hd = I.held[id];
    const double slo = slo_of(I, id);
    if (!(f & F_PREFILL_FIN)) continue;
    WSYNC();
    UNI(I.flags[id] = (uint8_t)(f & ~F_PREFILL_FIN));
    if (st != ST_RUNNING) continue;
    if constexpr (B) {  // baselines keep decoding (engine.hpp:805-808)
      list_erase(I.ongo, &I.n_ongo, id);
      UNI(I.gen_epoch[id] = gen; I.run[I.R++] = id);
      logev(I, ECONO_EV_PREFILL_DONE, id, 1, 0);
      WSYNC();
      continue;
    }
    UNI(I.state[id] = ST_WAITING_GT; I.last_enq[id] = I.clock);
    // gt_member_demand (engine.hpp:238-247) from the fields loaded above
    const Tok tgt = block_round((Tok)pr + gen + pad, I.block);
    const Tok dl = tgt - hd;
    group_insert_gt(I, id, pad, slo, oc, I.clock, dl > 0 ? block_round(dl, I.block) : 0);
    logev(I, ECONO_EV_PREFILL_DONE, id, 0, 0);
    WSYNC();
    if (I.error) return;
  }
  [[maybe_unused]] const int64_t tx3 = PHASE_NOW();
  PHASE_ADD(14, tx3 - tx2);
  // under-prediction (engine.hpp:812-817): candidates fixed up front (above), handled in order
  for (int32_t k = 0; k < npre; ++k) {
    const int32_t id = I.tmp_a[k];
    if (I.state[id] != ST_RUNNING) continue;
    handle_underprediction<B>(I, id);
    if (I.error) return;
  }
  // hosted-slot deadlines over a copy of the slot list (engine.hpp:819-828)
  int32_t ncs = 0;
  for (int32_t base = 0; base < I.n_slots; base += W) {
    const int32_t si = base + LANE;
    bool c = false;
    int32_t h = -1;
    if (si < I.n_slots) {
      const int32_t sp = I.slots[si];
      const int32_t host = I.sl_host[sp], off = I.sl_off[sp];
      h = I.sl_hosted[sp];
      c = I.state[host] == ST_RUNNING && (I.generated[host] - I.gen_epoch[host]) >= off;
    }
    const unsigned m = BALLOT(c);
    if (c) {
      const int32_t o = ncs + POPC(m & LANEMASK_LT);
      I.tmp_b[o] = h;
      I.tmp_c[o] = I.sl_host[I.slots[si]];
      I.tmp_a[I.scr_cap + o] = I.sl_off[I.slots[si]];
    }
    ncs += POPC(m);
  }
  WSYNC();
  for (int32_t k = 0; k < ncs; ++k) {
    const int32_t hosted = I.tmp_b[k], host = I.tmp_c[k];
    if (I.state[host] != ST_RUNNING) continue;
    if ((Tok)I.generated[host] - I.gen_epoch[host] < I.tmp_a[I.scr_cap + k]) continue;
    if (I.state[hosted] == ST_DONE || !(I.flags[hosted] & F_HOSTED)) continue;
    handle_hosted_overrun(I, hosted);
    if (I.error) return;
  }
  if (npre || ncs) run_compact(I);
  {  // warp-uniform (every lane, same values)
    s.completed = completed_now;
    if (REC_SM(I)) {
      if (I.sm_n < I.sm_cap) I.sm[I.sm_n] = s;
      I.sm_n++;
    }
    I.executed++;
    I.agg_fs += fs;
    I.agg_written += s.kvc_written_frac;
    I.agg_allocated += s.kvc_allocated_frac;
    if ((double)fs >= 0.95 * (double)I.tfs) I.agg_tfs_hits++;
    if (s.pts_admitted > 0) I.agg_pt_iters++;
    I.hist[completed_now < I.hist_cap ? completed_now : I.hist_cap - 1]++;
    I.n_ptiter = 0;
    I.n_adm = 0;
    I.exam_count = 0;
    I.pts_admitted_iter = 0;
    I.pt_admittable = 0;
    if (B) {
      I.admission_open = I.admission_open || completed_now > 0;
      I.decode_pause = 0;
    }
#ifdef ECONO_PROF_PHASES
    if (LANE == 0) I.prof[15] += PROF_NOW() - tx3;
#endif
  }
  WSYNC();
}

ECOLD void handle_idle(Inst& I) {  // engine.hpp:930-961
  if (I.arrival_cursor < I.n) {
    const double next = I.arrival[I.arrival_cursor];
    {  // warp-uniform (every lane, same values)
      long long k = 1;
      if (next > I.clock) {
        const long long c = (long long)ceil((next - I.clock) / I.t_base);
        k = c > 1 ? c : 1;
      }
      const double dt = (double)k * I.t_base;
      I.clock += dt;
      I.iter += k;
      if (REC_SM(I)) {
        if (I.sm_n < I.sm_cap) {
          EconoSample& s = I.sm[I.sm_n];
          s.iter = I.iter;
          s.clock = I.clock;
          s.dt = dt;
          s.forward_size = 0;
          s.kvc_written_frac = (double)I.written_total / (double)I.capacity;
          s.kvc_allocated_frac =
              (double)((I.general_cap - I.free_total) + I.reserved_used) / (double)I.capacity;
          s.completed = 0;
          s.pts_admitted = 0;
          s.pt_admittable = 0;
          s._pad = 0;
          s.idle_repeat = k;
        }
        I.sm_n++;
      }
      I.err_val = k;
    }
    WSYNC();
    logev(I, ECONO_EV_IDLE, -1, I.err_val, 0);
    UNI(I.err_val = 0);
    return;
  }
  int32_t stuck = -1;  // first request not done (engine.hpp:951-960)
  for (int32_t base = 0; base < I.n && stuck < 0; base += W) {
    const int32_t i = base + LANE;
    const unsigned m = BALLOT(i < I.n && I.state[i] != ST_DONE);
    if (m) stuck = base + FFS(m);
  }
  set_error(I, ERR_STUCK, stuck, 0);
}

// Worst-case events one step can append (arrivals + every bounded list), so
// a launch stops and lets the host drain before a step could overflow.
EDEV int64_t step_event_bound(const Inst& I) {
  int64_t arrivals = 0;
  if (I.arrival_cursor < I.n) arrivals = due_end(I, I.arrival_cursor, I.clock + 1e-12) - I.arrival_cursor;
  if (I.base)  // every admitted or queued request: swap-in, dispatch, alloc_fail, preempt_swap, ...
    return arrivals + 2 * I.tfs + 8 * (I.arrival_cursor - I.completed) + 64;
  return arrivals + 2 * I.tfs + 4 * (I.arrival_cursor - I.completed - I.pt_count) + 2 * (int64_t)I.n_slots + 64;
}

// ------------------------------------------------------------------------
// Exact event-horizon skipping (SURVEY.md §7 hard part 7; the reference has
// no such thing). A step is "quiet" when ingest_arrivals admits nothing,
// select_gt_groups and select_pts select nothing (their inputs — free KVC,
// the GT queue head, tfs-|running|, the reserve and the PT queue — only
// change at events) and execute_iteration sees no completion, under-
// prediction or slot deadline. Quiet steps only advance clock/iter, the
// running requests' progress counters and the in-order sample aggregates, so
// a span of them is replayed with the same sequential FP adds (never k*dt).
// ------------------------------------------------------------------------
// *fuse: the event iteration that ends the span consists of completions only
// (no under-prediction, no slot deadline, nothing selectable), so the replay
// may run it too and finish it with complete_fused() instead of a normal step.
EDEVNI int64_t quiet_span(Inst& I, int64_t budget, bool* fuse) {
  *fuse = false;
  const int32_t R = I.R;
  if (R == 0 || I.n_ptiter != 0 || I.n_adm != 0 || budget <= 0) return 0;
  // The independent probes are issued together (three dependent levels in
  // all): the next arrival, the GT queue head, and the running requests.
  const bool has_arr = I.arrival_cursor < I.n;
  const Tok free_tok = I.free_total;
  const bool gt_check = free_tok > 0 && I.G > 0;
  const double ta = has_arr ? I.arrival[I.arrival_cursor] : 0.0;
  const int32_t g = gt_check ? I.gq[0] : 0;
  const int32_t id0 = LANE < R ? I.run[LANE] : -1;
  int64_t gd = 0;
  int32_t hd = 0;
  if (gt_check) {
    gd = I.gr_dem[g];
    hd = I.gr_hd[g];
  }
  // distance to the first completion (true_rl <= allowance) and to the first
  // under-prediction (allowance < true_rl, engine.hpp:812-817)
  int32_t kc = INT32_MAX, ku = INT32_MAX, ks = INT32_MAX;  // token counts < 2^30
  if (id0 >= 0) {
    const int32_t tr = I.true_rl[id0], al = I.allowance[id0], ge = I.generated[id0];
    if (tr <= al) kc = tr - ge; else ku = al - ge;
  }
  if (has_arr && ta <= I.clock + 1e-12) return 0;
  if (gt_check) {  // queues.hpp:220-263 would take >= 1 member
    if (gd <= free_tok || hd <= free_tok) return 0;
  }
  const Tok C0 = tmin(I.tfs - (Tok)R, I.reserve_cap - I.reserved_used);
  if (C0 >= 1 && I.pt_count > 0 && C0 >= I.pt_min_lb) {  // queues.hpp:279-299 would take a PT
    bool fit = false;
    if (ORD(I)) {
      for (int b = 0; b < I.nbuckets && !fit; ++b) fit = bm_prev(I, b, C0) >= 1;
    } else {
      fit = I.tree[I.tree_off[I.tree_levels - 1]] <= C0;
    }
    if (fit) return 0;
    UNI(I.pt_min_lb = C0 + 1);
  }
  // first decode-side event: completion / under-prediction / slot deadline
  for (int32_t i = W + LANE; i < R; i += W) {
    const int32_t id = I.run[i];
    const int32_t tr = I.true_rl[id], al = I.allowance[id], ge = I.generated[id];
    if (tr <= al) kc = kc < tr - ge ? kc : tr - ge; else ku = ku < al - ge ? ku : al - ge;
  }
  for (int32_t si = LANE; si < I.n_slots; si += W) {
    const int32_t sp = I.slots[si];
    const int32_t host = I.sl_host[sp];
    if (I.state[host] == ST_RUNNING) {
      const int32_t e = I.sl_off[sp] - (I.generated[host] - I.gen_epoch[host]);
      ks = e < ks ? e : ks;
    }
  }
  kc = wmin32(kc);
  ku = wmin32(ku);
  ks = wmin32(ks);
  const int64_t kev = kc == INT32_MAX && ku == INT32_MAX && ks == INT32_MAX ? INT64_MAX
                                                                          : (int64_t)(kc < ku ? (kc < ks ? kc : ks) : (ku < ks ? ku : ks));
  int64_t k = kev - 1;  // the event iteration itself runs as a normal step ...
  if (k > budget) k = budget;
  if (REC_SM(I) && k > I.sm_cap - I.sm_n) k = I.sm_cap - I.sm_n;
  // ... unless it only completes requests and fits the budget (bench path)
  // (running set within one warp: its completion scan and compaction are one
  // ballot; with more running requests a fused release measured slower)
  *fuse = !REC_EV(I) && !REC_SM(I) && R <= W && kev >= 1 && kev <= budget && kc == kev && ku > kev &&
          ks > kev;
  return k > 0 ? k : 0;
}

// Progress of one running request over a replayed span (execute_iteration's
// decode branch, engine.hpp:744-771, k times; exec_t by sequential adds).
EDEV void quiet_request(Inst& I, int32_t id, double e, int64_t k, double clk1) {
  I.exec_t[id] = e;
  if (I.generated[id] == 0 && I.first_tok[id] < 0.0) I.first_tok[id] = clk1;
  I.generated[id] += (int32_t)k;
  I.occupied[id] += (int32_t)k;
  I.written[id] += (int32_t)k;
}

// The replay without per-iteration samples (the bench path): every chain the
// reference advances once per iteration — clock, the in-order sample sums of
// metrics.hpp:153-162, and each running request's execution_time — advances
// in ONE loop, so the k-step span costs ~k dependent DADDs instead of one
// pass per chain. The per-iteration written fractions are computed W at a
// time across lanes and broadcast (shuffles are off the dependency chain).
EDEVNI int64_t quiet_steps_fused(Inst& I, int64_t k, Tok fs, double dt, double clk1, double af,
                                 int64_t wt0, double cap) {
  const bool has_arr = I.arrival_cursor < I.n;
  const double ta = has_arr ? I.arrival[I.arrival_cursor] : 0.0;
  const int32_t R = I.R;
  const int32_t my = LANE < R ? I.run[LANE] : -1;
  double e = my >= 0 ? I.exec_t[my] : 0.0;
  double clock = I.clock, aw = I.agg_written, aa = I.agg_allocated;
  int64_t j = 0;
  if (!has_arr) {
    // The fractions of a chunk go to shared memory; the unrolled chain then
    // reads them with loads the compiler can issue ahead of the adds (a
    // shuffle per step would put its latency on the aw chain).
    for (int64_t base = 0; base < k; base += W) {
      const int64_t jj = base + LANE;
      I.wbuf[LANE] = jj < k ? (double)(wt0 + (jj + 1) * fs) / cap : 0.0;
      WSYNC();
      const int lim = k - base < W ? (int)(k - base) : W;
      if (lim == W) {
#pragma unroll
        for (int l = 0; l < W; ++l) {
          clock += dt; aw += I.wbuf[l]; aa += af; e += dt;
        }
      } else {
        for (int l = 0; l < lim; ++l) {
          clock += dt; aw += I.wbuf[l]; aa += af; e += dt;
        }
      }
      WSYNC();
    }
    j = k;
  } else {  // the arrival cut-off is re-checked before every replayed step
    bool stop = false;
    for (int64_t base = 0; base < k && !stop; base += W) {
      const int64_t jj = base + LANE;
      const double wf = jj < k ? (double)(wt0 + (jj + 1) * fs) / cap : 0.0;
      const int lim = k - base < W ? (int)(k - base) : W;
      for (int l = 0; l < lim; ++l) {
        const double w = shfl(wf, l);
        if (j > 0 && ta <= clock + 1e-12) { stop = true; break; }
        clock += dt; aw += w; aa += af; e += dt;
        ++j;
      }
    }
  }
  k = j;
  if (my >= 0) quiet_request(I, my, e, k, clk1);
  for (int32_t i = W + LANE; i < R; i += W) {
    const int32_t id = I.run[i];
    double e2 = I.exec_t[id];
    for (int64_t t = 0; t < k; ++t) e2 += dt;
    quiet_request(I, id, e2, k, clk1);
  }
  WSYNC();
  UNI(I.clock = clock; I.written_total = wt0 + k * fs; I.agg_written = aw; I.agg_allocated = aa;
        I.iter += k; I.steps += k; I.executed += k; I.agg_fs += fs * k;
        if ((double)fs >= 0.95 * (double)I.tfs) I.agg_tfs_hits += k;
        I.hist[0] += k; I.quiet_steps += k; I.quiet_spans++);
  return k;
}

// The fused event iteration's completions (execute_iteration, engine.hpp:
// 784-791): the replay already ran its decode progress, clock and sample
// sums; the requests that reached true_rl complete in running order, exactly
// as in the running-set pass, and the iteration moves from hist[0] to its
// completion count. Under-predictions and slot deadlines cannot occur here
// (quiet_span's fuse test).
EDEVNI void complete_fused(Inst& I) {
  const int32_t R0 = I.R;
  int32_t completed_now = 0;
  int32_t id_c0 = -1;
  unsigned keep0 = 0;
  for (int32_t base = 0; base < R0; base += W) {
    const int32_t i = base + LANE;
    const int32_t id = i < R0 ? I.run[i] : -1;
    const bool fin = id >= 0 && I.generated[id] >= I.true_rl[id];
    if (base == 0) {
      id_c0 = id;
      keep0 = BALLOT(id >= 0 && !fin);
    }
    unsigned m = BALLOT(fin);
    WSYNC();
    while (m) {
      const int l = FFS(m);
      m &= m - 1;
      const int32_t cid = shfl(id, l);
      UNI(I.state[cid] = ST_DONE; I.compl_clock[cid] = I.clock);
      kvc_release(I, cid);
      if (I.error) return;
      UNI(I.occupied[cid] = 0; I.completed++);
      logev(I, ECONO_EV_COMPLETE, cid, I.generated[cid], 0);
      WSYNC();
      completed_now++;
    }
  }
  if (R0 <= W) {
    if ((keep0 >> LANE) & 1u) I.run[POPC(keep0 & LANEMASK_LT)] = id_c0;
    WSYNC();
    UNI(I.R = POPC(keep0));
  } else {
    run_compact(I);
  }
  UNI(I.hist[0]--; I.hist[completed_now < I.hist_cap ? completed_now : I.hist_cap - 1]++;
      I.quiet_steps--);
}

EDEVNI int64_t quiet_steps(Inst& I, int64_t k, bool fuse = false) {
  const Tok fs = I.R;
  const double dt = iteration_time(I, fs) + 0.0;
  const double clk1 = I.clock + dt;
  const double af = (double)((I.general_cap - I.free_total) + I.reserved_used) / (double)I.capacity;
  const int64_t wt0 = I.written_total;
  const double cap = (double)I.capacity;
  if (!REC_SM(I)) {  // one inlined replay serves both: k quiet iterations (+ the fused completing one)
    const int64_t kk = k + (fuse ? 1 : 0);
    const int64_t j = quiet_steps_fused(I, kk, fs, dt, clk1, af, wt0, cap);
    if (fuse && j == kk) complete_fused(I);  // an arrival cut-off leaves the event to a normal step
    return j;
  }
  // pass 1 (every lane, identical arithmetic): the sequential clock chain and
  // the arrival cut-off — ingest would admit an arrival at the next step.
  double clock = I.clock;
  {
    const bool has_arr = I.arrival_cursor < I.n;
    const double ta = has_arr ? I.arrival[I.arrival_cursor] : 0.0;
    int64_t j = 0;
    for (; j < k; ++j) {
      if (j > 0 && has_arr && ta <= clock + 1e-12) break;
      clock += dt;
    }
    k = j;
  }
  // pass 2: per-iteration written fractions computed lane-parallel, summed in
  // sample order (metrics.hpp:153-162) so the FP sums match the reference.
  double aw = I.agg_written, aa = I.agg_allocated;
  if (REC_SM(I)) {
    if (LANE == 0) {
      double c = I.clock;
      for (int64_t j = 0; j < k; ++j) {
        c += dt;
        const double wf = (double)(wt0 + (j + 1) * fs) / cap;
        aw += wf;
        aa += af;
        EconoSample& s = I.sm[I.sm_n + j];
        s.iter = I.iter + j + 1;
        s.clock = c;
        s.dt = dt;
        s.forward_size = fs;
        s.kvc_written_frac = wf;
        s.kvc_allocated_frac = af;
        s.completed = 0;
        s.pts_admitted = 0;
        s.pt_admittable = 0;
        s._pad = 0;
        s.idle_repeat = 0;
      }
    }
  } else {
    for (int64_t base = 0; base < k; base += W) {
      const int64_t jj = base + LANE;
      const double wf = jj < k ? (double)(wt0 + (jj + 1) * fs) / cap : 0.0;
      const int lim = k - base < W ? (int)(k - base) : W;
      for (int l = 0; l < lim; ++l) {
        aw += shfl(wf, l);
        aa += af;
      }
    }
  }
  WSYNC();
  // lane 0 alone holds the recorded path's sums (aw, aa)
  LANE0(I.clock = clock; I.written_total = wt0 + k * fs; I.agg_written = aw; I.agg_allocated = aa);
  for (int32_t i = LANE; i < I.R; i += W) {
    const int32_t id = I.run[i];
    double e = I.exec_t[id];
    for (int64_t j = 0; j < k; ++j) e += dt;
    I.exec_t[id] = e;
    if (I.generated[id] == 0 && I.first_tok[id] < 0.0) I.first_tok[id] = clk1;
    I.generated[id] += (int32_t)k;
    I.occupied[id] += (int32_t)k;
    I.written[id] += (int32_t)k;
  }
  UNI(I.iter += k; I.steps += k; I.executed += k; I.agg_fs += fs * k;
        if ((double)fs >= 0.95 * (double)I.tfs) I.agg_tfs_hits += k;
        I.hist[0] += k; if (REC_SM(I)) I.sm_n += k;
        I.quiet_steps += k; I.quiet_spans++);
  return k;
}

template <bool B>
EDEVNI void engine_step(Inst& I) {  // Engine::step (engine.hpp:104-116)
  [[maybe_unused]] const int64_t t0 = PHASE_NOW();
  ingest<B>(I);
  PHASE_ADD(6, PHASE_NOW() - t0);
  if (B) form_baseline(I); else form_econoserve(I);
  if (I.error) return;
  [[maybe_unused]] const int64_t t1 = PHASE_NOW();
  Tok fs = 0;
  for (int32_t i = LANE; i < I.n_ptiter; i += W) fs += I.ptiter_tok[i];
  fs = wsum32((int32_t)fs) + ((B && I.decode_pause) ? 0 : I.R);
  if (fs == 0) handle_idle(I); else execute_iteration<B>(I, fs);
  PHASE_ADD(10, PHASE_NOW() - t1);
  UNI(I.steps++);
}

}  // namespace econo
