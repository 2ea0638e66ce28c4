// runtime.cu — host runtime and C-ABI (include/econoserve_b200.h) around the
// on-device EconoServe engine (engine.cuh).
//
// Product build: nvcc -gencode arch=compute_100a,code=sm_100a (see
// __graft_entry__.build). Every instance is one warp (one CTA) of
// k_engine_steps; the host only sizes memory, launches, drains the optional
// event/sample logs, and formats errors. There is no CPU execution path: if
// the device is unavailable econo_create returns ECONO_ECUDA.
//
// ECONO_HOSTSIM (test-only, built by tests/hostsim.py with g++): the same
// engine source compiled for the host with one lane per "warp", used to check
// the engine logic against the oracle on machines without a GPU.
#include <limits.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <string>
#include <thread>
#include <vector>

#include "engine.cuh"
#include "steps.cuh"
#if !defined(ECONO_HOSTSIM)
#include <cuda_runtime.h>
// kernel_fast.cu: the step kernel specialised for non-recording, ordered-queue batches;
// kernel_fast_oracle.cu: the same for econoserve-full with the oracle predictor
void launch_engine_steps_fast(econo::Inst* insts, unsigned n_inst, int64_t max_steps, int64_t slice_ns,
                              cudaStream_t s);
void launch_engine_steps_fast_oracle(econo::Inst* insts, unsigned n_inst, int64_t max_steps, int64_t slice_ns,
                                     cudaStream_t s);
#endif

#ifndef ECONO_HOSTSIM
#include <cuda_runtime.h>
#endif

using namespace econo;

static_assert(sizeof(Inst) % 8 == 0, "Inst must be 8-byte granular");

// ---------------------------------------------------------------------------
// device entry points
// ---------------------------------------------------------------------------
namespace econo {

// init_requests (engine.hpp:165-209), split so the O(n) parts run grid-wide
// over every instance's requests and only the sequential pieces (the
// pred_rng_ stream for non-oracle predictors, scalar calibration) run per
// instance. Phase 1: trace AoS -> SoA, arrival-order check, prompt sum.
EDEV void init_soa_one(Inst& I, const EconoTraceRecord* tr, int64_t i, bool* order_bad, int64_t* prompt,
                       bool* len_bad) {
  double* arr = const_cast<double*>(I.arrival.get());
  int32_t* pr = const_cast<int32_t*>(I.prompt.get());
  int32_t* rl = const_cast<int32_t*>(I.true_rl.get());
  arr[i] = tr[i].arrival_time;
  pr[i] = (int32_t)tr[i].prompt_len;
  rl[i] = (int32_t)tr[i].true_rl;
  *order_bad = i > 0 && tr[i].arrival_time < tr[i - 1].arrival_time;
  *prompt = tr[i].prompt_len;
  *len_bad = tr[i].prompt_len < 1 || tr[i].prompt_len >= ((int64_t)1 << 30) || tr[i].true_rl < 1 ||
             tr[i].true_rl >= ((int64_t)1 << 30);
}
// Phase 1 for a trace uploaded as arrays (econo_batch_create_soa): the same
// checks on the instance's own SoA.
EDEV void init_check_one(const Inst& I, int64_t i, bool* order_bad, int64_t* prompt, bool* len_bad) {
  const int32_t p = I.prompt[i], r = I.true_rl[i];
  *order_bad = i > 0 && I.arrival[i] < I.arrival[i - 1];
  *prompt = p;
  *len_bad = p < 1 || p >= (1 << 30) || r < 1 || r >= (1 << 30);
}
// Phase 2 (per instance): calibration t_p / t_g (engine.hpp:171-176); the
// prompt sum is an exact integer, equal to the reference's sequential
// double sum of integers below 2^53.
EDEV void init_calibrate(Inst& I, int64_t prompt_sum) {
  const Tok mean_prompt = tmax(1, (Tok)llround((double)prompt_sum / (double)I.n));
  I.t_p = iteration_time(I, mean_prompt);
  I.t_g = iteration_time(I, I.tfs);
}
// Predictions consume pred_rng_ in id order (engine.hpp:187-188): sequential
// unless the predictor is the oracle.
EDEVNI void init_predict_sequential(Inst& I) {
  if (I.pred_model == ECONO_PRED_ORACLE) return;
  if (LANE == 0)
    for (int32_t i = 0; i < I.n; ++i) {
      const Tok p = predict_rl(I, I.true_rl[i], I.pmt, I.pmt_i);
      I.predicted[i] = sat_rl(p);
      const Tok pad = apply_padding(p, I.pred_pad);
      if (I.ovf_id >= I.n && (p >= kRlSat || pad >= kRlSat))  // engine.hpp:196-202 with int64 lengths
        I.ovf_id = i, I.ovf_dem = block_round((Tok)I.prompt[i] + tmax(I.true_rl[i], pad), I.block);
    }
  WSYNC();
}
// Worst-case KVC demand of request i (engine.hpp:193-197): Orca reserves the
// maximum output length, every other policy the larger of the true and
// padded lengths.
EDEV Tok worst_demand(const Inst& I, int64_t i) {
  const Tok out = I.policy == ECONO_POLICY_ORCA ? I.max_out : tmax(I.true_rl[i], padded_of(I, i));
  return block_round((Tok)I.prompt[i] + out, I.block);
}
// Phase 3: per-request fields + feasibility (engine.hpp:186-206).
EDEV bool init_req_one(Inst& I, int64_t i) {
  if (I.pred_model == ECONO_PRED_ORACLE) I.predicted[i] = sat_rl(quantize_up(I.true_rl[i], I.pred_quantum));
  I.state[i] = ST_WAITING_PT;
  if (I.base) I.dispatch_t[i] = -1.0;
  I.first_tok[i] = -1.0;
  I.compl_clock[i] = -1.0;
  I.reg_head[i] = -1;
  I.pt_next[i] = -1;  // also gt_next (shared storage)
  if (I.base) I.ptarget[i] = I.prompt[i];  // prefill_target = prompt_len (engine.hpp:189)
  return worst_demand(I, i) > I.general_cap || (!I.base && (Tok)I.prompt[i] > I.reserve_cap);
}
// Table initialisation for index i of every table.
EDEV void init_tables_one(Inst& I, int64_t i) {
  if (i < I.reg_cap) I.reg_free[i] = I.reg_cap - 1 - (int32_t)i;
  if (i < I.grp_cap) I.grp_free[i] = I.grp_cap - 1 - (int32_t)i;
  if (i < I.slot_cap) I.sl_free[i] = I.slot_cap - 1 - (int32_t)i;
  if (i < I.rl_cap) I.rl_map[i] = -1;
  if (I.ordered) {
    if (i < (int64_t)I.nbuckets * (I.pmax + 1)) { I.cls_head[i] = -1; I.cls_tail[i] = -1; }
  } else if (i <= I.tree_off[I.tree_levels - 1]) {
    I.tree[i] = INF32;
  }
}
EDEV int64_t init_table_extent(const Inst& I) {
  int64_t m = I.n;
  m = m > I.reg_cap ? m : I.reg_cap;
  m = m > I.grp_cap ? m : I.grp_cap;
  m = m > I.rl_cap ? m : I.rl_cap;
  const int64_t t = I.ordered ? (int64_t)I.nbuckets * (I.pmax + 1) : (int64_t)I.tree_off[I.tree_levels - 1] + 1;
  return m > t ? m : t;
}
// Phase 4 (per instance): report the first infeasible request like the
// reference (it throws at the first failing id), then open the tables.
EDEV void init_finish(Inst& I, int64_t first_bad) {
  if (first_bad < I.n) {
    const int32_t bad = (int32_t)first_bad;
    Tok worst = worst_demand(I, bad);
    if (I.policy != ECONO_POLICY_ORCA) {  // a saturated prediction: the exact int64 demand
      if (I.pred_model == ECONO_PRED_ORACLE)
        worst = block_round((Tok)I.prompt[bad] + tmax(I.true_rl[bad], apply_padding(quantize_up(I.true_rl[bad],
                            I.pred_quantum), I.pred_pad)), I.block);
      else if (bad == I.ovf_id)
        worst = I.ovf_dem;
    }
    I.error = worst > I.general_cap ? ERR_INFEASIBLE_KVC : ERR_INFEASIBLE_RESERVE;
    I.err_id = bad;
    I.err_val = worst > I.general_cap ? worst : I.reserve_cap;
    return;
  }
  I.reg_free_top = I.reg_cap;
  I.grp_free_top = I.grp_cap;
  I.sl_free_top = I.slot_cap;
  I.next_group_id = 1;
}

// finalize() per-request records (engine.hpp:963-984), one lane per request.
EDEV void engine_record(const Inst& I, int32_t i, EconoRecord& rc) {
  rc.id = i;
  rc.preempt_count = I.preempt_count[i];
  rc.arrival = I.arrival[i];
  const double extra = I.penalty[i] + I.sched_share[i];
  rc.completion_time = I.compl_clock[i] + extra;
  rc.first_token_time = I.first_tok[i];
  rc.waiting_time = I.waiting[i];
  rc.execution_time = I.exec_t[i];
  rc.preemption_time = I.preempt_t[i] + I.penalty[i];
  rc.scheduling_time_share = I.sched_share[i];
  rc.reserve_draws = I.reserve_draws[i];
  rc.met_slo = rc.completion_time <= slo_of(I, i);
  rc.prompt_len = I.prompt[i];
  rc.true_rl = I.true_rl[i];
  rc.slo_deadline = slo_of(I, i);
  rc.alloc_failure = (I.flags[i] & F_ALLOC_FAIL) ? 1 : 0;
  rc._pad = 0;
}

// Per-instance metric partial sums (metrics.hpp:110-173) for the cross-GPU
// reduction: [0]=n [1]=sum jct [2]=sum tbt [3]=tbt_n [4]=sum jct/true_rl
// [5]=met [6]=tokens [7]=preemptions [8]=reserve_draws [9]=alloc failures
// [10]=max completion [11..14]=sum waiting/execution/preemption/scheduling
// [15]=executed iters [16]=sum fs [17]=sum written frac [18]=sum allocated
// frac [19]=tfs hits [20]=pt iters [21]=hosted slots [22]=hosted overruns
// [23]=completed [24]=pt dispatched [25]=gt scheduled [26]=steps [27]=iter.
// acc[0..14] over requests lo, lo+stride, ... < I.n (one thread's share).
EDEV void partials_accumulate(const Inst& I, int64_t lo, int64_t stride, double* acc) {
  for (int64_t i = lo; i < I.n; i += stride) {
    EconoRecord rc;
    engine_record(I, (int32_t)i, rc);
    const double jct = rc.completion_time - rc.arrival;
    acc[0] += 1.0;
    acc[1] += jct;
    if (rc.true_rl >= 2 && rc.first_token_time >= 0.0) {
      acc[2] += (rc.completion_time - rc.first_token_time) / (double)(rc.true_rl - 1);
      acc[3] += 1.0;
    }
    acc[4] += jct / (double)rc.true_rl;
    acc[5] += rc.met_slo ? 1.0 : 0.0;
    acc[6] += (double)rc.true_rl;
    acc[7] += rc.preempt_count;
    acc[8] += rc.reserve_draws;
    acc[9] += rc.alloc_failure;
    acc[10] = rc.completion_time > acc[10] ? rc.completion_time : acc[10];
    acc[11] += rc.waiting_time;
    acc[12] += rc.execution_time;
    acc[13] += rc.preemption_time;
    acc[14] += rc.scheduling_time_share;
  }
}
EDEV void partials_combine(double* acc, const double* x) {
  for (int k = 0; k < 15; ++k) acc[k] = k == 10 ? (x[k] > acc[k] ? x[k] : acc[k]) : acc[k] + x[k];
}
// The per-request sums plus the instance's running aggregates.
EDEV void partials_finish(const Inst& I, const double* acc, double* out) {
  for (int k = 0; k < 15; ++k) out[k] = acc[k];
  out[15] = (double)I.executed;
  out[16] = (double)I.agg_fs;
  out[17] = I.agg_written;
  out[18] = I.agg_allocated;
  out[19] = (double)I.agg_tfs_hits;
  out[20] = (double)I.agg_pt_iters;
  out[21] = (double)I.hosted_total;
  out[22] = (double)I.hosted_overruns;
  out[23] = (double)I.completed;
  out[24] = (double)I.pt_dispatched;
  out[25] = (double)I.gt_scheduled;
  out[26] = (double)I.steps;
  out[27] = (double)I.iter;
  for (int k = 28; k < ECONO_PARTIAL_WORDS; ++k) out[k] = 0.0;
}
// Per-instance metric partial sums (metrics.hpp:110-173) for the cross-GPU
// reduction: [0]=n [1]=sum jct [2]=sum tbt [3]=tbt_n [4]=sum jct/true_rl
// [5]=met [6]=tokens [7]=preemptions [8]=reserve_draws [9]=alloc failures
// [10]=max completion [11..14]=sum waiting/execution/preemption/scheduling
// [15]=executed iters [16]=sum fs [17]=sum written frac [18]=sum allocated
// frac [19]=tfs hits [20]=pt iters [21]=hosted slots [22]=hosted overruns
// [23]=completed [24]=pt dispatched [25]=gt scheduled [26]=steps [27]=iter.
// Host build (tests): one pass in id order.
EDEV void engine_partials(const Inst& I, double* out) {
  double acc[15];
  for (int k = 0; k < 15; ++k) acc[k] = 0.0;
  partials_accumulate(I, 0, 1, acc);
  partials_finish(I, acc, out);
}

// ---- JCT order statistics (aggregate()'s percentile, metrics.hpp:81-89) ----
// JCT = completion_time - arrival with completion_time built exactly as
// finalize() does (engine.hpp:970-971), mapped to a uint64 whose unsigned
// order is the double order, so exact k-th smallest values come from an
// MSB-first radix select (11-bit digits, 6 passes) instead of a sort.
EDEV uint64_t jct_key(const Inst& I, int64_t i) {
  const double extra = I.penalty[i] + I.sched_share[i];
  const double ct = I.compl_clock[i] + extra;
  const double j = ct - I.arrival[i];
  uint64_t b;
  memcpy(&b, &j, sizeof(b));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
EHD double key_double(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
  double d;
  memcpy(&d, &b, sizeof(d));
  return d;
}
EHD bool key_matches(uint64_t k, uint64_t prefix, int consumed) {
  return consumed == 0 || (k >> (64 - consumed)) == prefix;
}
EHD uint32_t key_digit(uint64_t k, int consumed, int dbits) {
  return (uint32_t)((k >> (64 - consumed - dbits)) & ((1ULL << dbits) - 1));
}

}  // namespace econo

#ifndef ECONO_HOSTSIM
// Per-instance init scratch: [0] first out-of-order arrival, [1] prompt sum,
// [2] first infeasible request.
// SOA: the trace arrays were uploaded straight into the instance's SoA
// (econo_batch_create_soa): only the checks run.
template <bool SOA>
__global__ void __launch_bounds__(256) k_init_soa(Inst* insts, const EconoTraceRecord* const* traces,
                                                  unsigned long long* scr, int32_t inst0) {
  const int32_t ii = inst0 + (int32_t)blockIdx.y;
  Inst& I = insts[ii];
  const EconoTraceRecord* tr = traces[ii];
  unsigned long long* sc = scr + 4 * ii;
  int64_t psum = 0;
  long long bad = LLONG_MAX, lbad = LLONG_MAX;
  int32_t pmn = INT32_MAX, pmx = 0, rmn = INT32_MAX, rmx = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < I.n; i += (int64_t)gridDim.x * blockDim.x) {
    bool ob, lb;
    int64_t p;
    if (SOA) init_check_one(I, i, &ob, &p, &lb);
    else init_soa_one(I, tr, i, &ob, &p, &lb);
    psum += p;
    if (ob && i < bad) bad = i;
    if (lb && i < lbad) lbad = i;
    if (!lb) {
      const int32_t pp = (int32_t)p, rr = SOA ? I.true_rl[i] : (int32_t)tr[i].true_rl;
      pmn = pp < pmn ? pp : pmn;
      pmx = pp > pmx ? pp : pmx;
      rmn = rr < rmn ? rr : rmn;
      rmx = rr > rmx ? rr : rmx;
    }
  }
  pmn = __reduce_min_sync(0xffffffffu, pmn);
  pmx = __reduce_max_sync(0xffffffffu, pmx);
  rmn = __reduce_min_sync(0xffffffffu, rmn);
  rmx = __reduce_max_sync(0xffffffffu, rmx);
  if ((threadIdx.x & 31) == 0) {
    if (pmn < INT32_MAX) {
      atomicMin(&I.tr_pmin, pmn);
      atomicMax(&I.tr_pmax, pmx);
      atomicMin(&I.tr_rmin, rmn);
      atomicMax(&I.tr_rmax, rmx);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    psum += __shfl_xor_sync(0xffffffffu, psum, o);
    const long long b2 = __shfl_xor_sync(0xffffffffu, bad, o);
    bad = b2 < bad ? b2 : bad;
    const long long l2 = __shfl_xor_sync(0xffffffffu, lbad, o);
    lbad = l2 < lbad ? l2 : lbad;
  }
  if ((threadIdx.x & 31) == 0) {
    if (psum) atomicAdd(&sc[1], (unsigned long long)psum);
    if (bad != LLONG_MAX) atomicMin(&sc[0], (unsigned long long)bad);
    if (lbad != LLONG_MAX) atomicMin(&sc[3], (unsigned long long)lbad);
  }
}

__global__ void __launch_bounds__(32) k_init_scalar(Inst* insts, const uint64_t* seeds, const unsigned long long* scr) {
  __shared__ Inst I;
  inst_load(I, &insts[blockIdx.x]);
  const unsigned long long* sc = scr + 4 * blockIdx.x;
  if (sc[0] < (unsigned long long)I.n) {
    LANE0(I.error = ERR_ARRIVAL_ORDER; I.err_id = (int32_t)sc[0]);
  } else {
    if (threadIdx.x == 0) {
      mt_seed(I.mt, I.mt_i, seeds[2 * blockIdx.x]);
      mt_seed(I.pmt, I.pmt_i, seeds[2 * blockIdx.x + 1]);
      init_calibrate(I, (int64_t)sc[1]);
    }
    __syncwarp();
    init_predict_sequential(I);
  }
  inst_store(&insts[blockIdx.x], I);
}

__global__ void __launch_bounds__(256) k_init_req(Inst* insts, unsigned long long* scr) {
  Inst& I = insts[blockIdx.y];
  if (I.error) return;
  unsigned long long* sc = scr + 4 * blockIdx.y;
  const int64_t ext = init_table_extent(I);
  long long bad = LLONG_MAX;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ext; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < I.n && init_req_one(I, i) && i < bad) bad = i;
    init_tables_one(I, i);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const long long b2 = __shfl_xor_sync(0xffffffffu, bad, o);
    bad = b2 < bad ? b2 : bad;
  }
  if ((threadIdx.x & 31) == 0 && bad != LLONG_MAX) atomicMin(&sc[2], (unsigned long long)bad);
}

__global__ void __launch_bounds__(32) k_init_finish(Inst* insts, const unsigned long long* scr) {
  Inst& I = insts[blockIdx.x];
  const unsigned long long bad = scr[4 * blockIdx.x + 2];
  if (threadIdx.x == 0 && !I.error) init_finish(I, bad < (unsigned long long)I.n ? (int64_t)bad : I.n);
}

__global__ void __launch_bounds__(32) k_engine_steps(Inst* insts, int64_t max_steps, int64_t slice_ns) {
  if (insts[blockIdx.x].base) return;  // a baseline-policy instance (k_baseline_steps)
  const int64_t deadline = slice_ns > 0 ? now_ns() + slice_ns : 0;
  __shared__ Inst I;
  const int64_t t0 = PROF_NOW();
  inst_load(I, &insts[blockIdx.x]);
  engine_steps<false>(I, steps_for(I, max_steps), deadline);
  LANE0(I.prof[11] += PROF_NOW() - t0; I.prof[12]++);
  inst_store(&insts[blockIdx.x], I);
}

// The comparison policies (orca, vllm, sarathi, multires, sync-coupled) in
// their own kernel, so the econoserve kernel's code is not affected by them.
__global__ void __launch_bounds__(32) k_baseline_steps(Inst* insts, int64_t max_steps, int64_t slice_ns) {
  if (!insts[blockIdx.x].base) return;
  const int64_t deadline = slice_ns > 0 ? now_ns() + slice_ns : 0;
  __shared__ Inst I;
  inst_load(I, &insts[blockIdx.x]);
  engine_steps<true>(I, steps_for(I, max_steps), deadline);
  inst_store(&insts[blockIdx.x], I);
}

__global__ void k_engine_records(const Inst* inst, EconoRecord* out) {
  const Inst& I = *inst;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < I.n; i += gridDim.x * blockDim.x) {
    EconoRecord rc;
    // one thread per request: same arithmetic as engine_record
    rc.id = i;
    rc.preempt_count = I.preempt_count[i];
    rc.arrival = I.arrival[i];
    const double extra = I.penalty[i] + I.sched_share[i];
    rc.completion_time = I.compl_clock[i] + extra;
    rc.first_token_time = I.first_tok[i];
    rc.waiting_time = I.waiting[i];
    rc.execution_time = I.exec_t[i];
    rc.preemption_time = I.preempt_t[i] + I.penalty[i];
    rc.scheduling_time_share = I.sched_share[i];
    rc.reserve_draws = I.reserve_draws[i];
    rc.met_slo = rc.completion_time <= slo_of(I, i);
    rc.prompt_len = I.prompt[i];
    rc.true_rl = I.true_rl[i];
    rc.slo_deadline = slo_of(I, i);
    rc.alloc_failure = (I.flags[i] & F_ALLOC_FAIL) ? 1 : 0;
    rc._pad = 0;
    out[i] = rc;
  }
}

// ---------------------------------------------------------------------------
// Bulk ingest of a large arrival batch, grid-wide (econo_batch_ingest).
// ingest_arrivals (engine.hpp:216-235) appends every due arrival to its PT
// class (deadline bucket, prompt) in id order. For a burst that is a stable
// group-by over up to n arrivals: keys (class) are sorted by an LSD radix
// sort (8-bit digits, 4096-key tiles, stable in-tile ranks from warp
// match_any), then each class segment is spliced onto its class list.
// ---------------------------------------------------------------------------
struct BulkJob {
  int32_t inst, tiles;
  int64_t first, k, off, hoff;   // arrivals [first, first+k); key offset; histogram offset
  unsigned long long minp;       // min prompt of the batch
  unsigned long long bcnt[ECONO_MAX_BOUNDS + 2];
  int32_t wb0, wnb, wp0, wnp;    // k_ingest_ranges: class window buckets [wb0, wb0+wnb) x prompts [wp0, wp0+wnp)
  int32_t werr;                  // set when an arrival falls outside the window (k_ingest_stitch<true> reports it)
  int32_t sstride;               // segment slots per tile/range: a range holds at most one segment per class of its window
};
constexpr int kBulkTile = 4096;
constexpr int64_t kBulkBudget = (int64_t)128 << 20;  // keys per ingest group (4 x 4 B of temp each: 2 GB)
// ECONO_BULK_BUDGET (keys) lowers it: a test knob that forces the multi-group
// path of econo_batch_ingest on batches small enough for a parity test
inline int64_t bulk_budget() {
  const char* e = getenv("ECONO_BULK_BUDGET");
  const int64_t v = e ? atoll(e) : 0;
  return v > 0 && v < kBulkBudget ? v : kBulkBudget;
}

__global__ void __launch_bounds__(256) k_bulk_keys(const Inst* insts, BulkJob* jobs, uint32_t* key, uint32_t* val) {
  BulkJob& J = jobs[blockIdx.y];
  if ((int)blockIdx.x >= J.tiles) return;
  const Inst& I = insts[J.inst];
  __shared__ unsigned long long sb[ECONO_MAX_BOUNDS + 2];
  __shared__ unsigned long long smin;
  if (threadIdx.x < ECONO_MAX_BOUNDS + 2) sb[threadIdx.x] = 0;
  if (threadIdx.x == 0) smin = ~0ULL;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kBulkTile;
  const double now = I.clock;
  const int pm1 = I.pmax + 1;
  unsigned long long mn = ~0ULL;
  uint32_t cnt[ECONO_MAX_BOUNDS + 2];  // per-thread bucket counts (registers: unrolled compares)
#pragma unroll
  for (int bb = 0; bb < ECONO_MAX_BOUNDS + 2; ++bb) cnt[bb] = 0;
  for (int e = threadIdx.x; e < kBulkTile; e += blockDim.x) {
    const int64_t i = t0 + e;
    if (i >= J.k) break;
    const int64_t id = J.first + i;
    const int b = bucket_d(I, dmax(0.0, slo_of(I, id) - now));
    const int32_t p = I.prompt[id];
    key[J.off + i] = (uint32_t)(b * pm1 + p);
    val[J.off + i] = (uint32_t)id;
    mn = (unsigned long long)p < mn ? (unsigned long long)p : mn;
#pragma unroll
    for (int bb = 0; bb < ECONO_MAX_BOUNDS + 2; ++bb) cnt[bb] += b == bb;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, mn, o);
    mn = x < mn ? x : mn;
  }
#pragma unroll
  for (int bb = 0; bb < ECONO_MAX_BOUNDS + 2; ++bb) {
    uint32_t c = cnt[bb];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&sb[bb], (unsigned long long)c);
  }
  if ((threadIdx.x & 31) == 0) atomicMin(&smin, mn);
  __syncthreads();
  if (threadIdx.x == 0) atomicMin(&J.minp, smin);
  if (threadIdx.x < ECONO_MAX_BOUNDS + 2 && sb[threadIdx.x]) atomicAdd(&J.bcnt[threadIdx.x], sb[threadIdx.x]);
}

// Per-tile digit histograms, digit-major: hist[hoff + d * tiles + t].
__global__ void __launch_bounds__(256) k_radix_hist(const BulkJob* jobs, const uint32_t* key, int shift,
                                                    uint32_t* hist) {
  const BulkJob& J = jobs[blockIdx.y];
  if ((int)blockIdx.x >= J.tiles) return;
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kBulkTile;
  for (int e = threadIdx.x; e < kBulkTile && t0 + e < J.k; e += blockDim.x)
    atomicAdd(&h[(key[J.off + t0 + e] >> shift) & 255], 1u);
  __syncthreads();
  hist[J.hoff + (int64_t)threadIdx.x * J.tiles + blockIdx.x] = h[threadIdx.x];
}

// Exclusive scan of one job's 256 x tiles histogram (one CTA per job).
__global__ void __launch_bounds__(1024) k_radix_scan(const BulkJob* jobs, uint32_t* hist) {
  const BulkJob& J = jobs[blockIdx.x];
  const int64_t m = 256LL * J.tiles;
  uint32_t* h = hist + J.hoff;
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < m; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const uint32_t v = i < m ? h[i] : 0;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t w = ws[threadIdx.x];
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += y;
      }
      ws[threadIdx.x] = w;
    }
    __syncthreads();
    const uint32_t wpre = (threadIdx.x >> 5) ? ws[(threadIdx.x >> 5) - 1] : 0;
    if (i < m) h[i] = carry + wpre + x - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += wpre + x;
    __syncthreads();
  }
}

// Stable scatter of one tile: each warp ranks its 512 keys in order with
// match_any, warps are offset by the digit counts of the warps before them;
// the tile is first reordered by digit in shared memory so that every digit's
// run is written to global memory contiguously (coalesced), not key by key.
__global__ void __launch_bounds__(256) k_radix_scatter(const BulkJob* jobs, const uint32_t* kin, const uint32_t* vin,
                                                       uint32_t* kout, uint32_t* vout, int shift,
                                                       const uint32_t* hist) {
  const BulkJob& J = jobs[blockIdx.y];
  if ((int)blockIdx.x >= J.tiles) return;
  constexpr int PER = kBulkTile / 256;  // keys per thread
  __shared__ uint32_t sk[kBulkTile];
  __shared__ uint32_t sv[kBulkTile];
  __shared__ uint32_t cnt[8][256];
  __shared__ uint32_t tstart[256];
  const int64_t t0 = (int64_t)blockIdx.x * kBulkTile;
  const int n = (int)(J.k - t0 < kBulkTile ? J.k - t0 : kBulkTile);
  for (int d = threadIdx.x; d < 8 * 256; d += blockDim.x) (&cnt[0][0])[d] = 0;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t kr[PER], vr[PER], rank[PER];
#pragma unroll
  for (int r = 0; r < PER; ++r) {  // warp w owns keys [w*512, (w+1)*512) in order
    const int e = w * (kBulkTile / 8) + r * 32 + lane;
    kr[r] = e < n ? kin[J.off + t0 + e] : 0;
    vr[r] = e < n ? vin[J.off + t0 + e] : 0;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const int e = w * (kBulkTile / 8) + r * 32 + lane;
    const int d = e < n ? (int)((kr[r] >> shift) & 255) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    uint32_t base = 0;
    if (d >= 0) base = cnt[w][d];
    __syncwarp();
    if (d >= 0 && (peers & ((1u << lane) - 1u)) == 0) cnt[w][d] = base + __popc(peers);
    __syncwarp();
    rank[r] = base + __popc(peers & ((1u << lane) - 1u));
  }
  __syncthreads();
  {  // per digit: exclusive prefix over warps, and the digit's total in the tile
    const int d = threadIdx.x;
    uint32_t run = 0;
    for (int ww = 0; ww < 8; ++ww) {
      const uint32_t c = cnt[ww][d];
      cnt[ww][d] = run;
      run += c;
    }
    tstart[d] = run;
  }
  __syncthreads();
  {  // exclusive scan of the 256 digit totals -> start of each digit's run in the tile
    const uint32_t v = tstart[threadIdx.x];
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __shared__ uint32_t ws[8];
    if (lane == 31) ws[w] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int ww = 0; ww < w; ++ww) pre += ws[ww];
    __syncthreads();
    tstart[threadIdx.x] = pre + x - v;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const int e = w * (kBulkTile / 8) + r * 32 + lane;
    if (e < n) {
      const int d = (int)((kr[r] >> shift) & 255);
      const uint32_t lp = tstart[d] + cnt[w][d] + rank[r];
      sk[lp] = kr[r];
      sv[lp] = vr[r];
    }
  }
  __syncthreads();
  const uint32_t* hb = hist + J.hoff;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const uint32_t kv = sk[e];
    const int d = (int)((kv >> shift) & 255);
    const int64_t pos = (int64_t)hb[(int64_t)d * J.tiles + blockIdx.x] + (e - (int)tstart[d]);
    kout[J.off + pos] = kv;
    vout[J.off + pos] = sv[e];
  }
}

// Class segments of the sorted batch: heads splice onto the old class tail
// (or become the head) and set the class bitmaps.
__global__ void __launch_bounds__(256) k_bulk_heads(Inst* insts, const BulkJob* jobs, const uint32_t* key,
                                                    const uint32_t* val) {
  const BulkJob& J = jobs[blockIdx.y];
  if ((int)blockIdx.x >= J.tiles) return;
  Inst& I = insts[J.inst];
  const int64_t t0 = (int64_t)blockIdx.x * kBulkTile;
  for (int e = threadIdx.x; e < kBulkTile && t0 + e < J.k; e += blockDim.x) {
    const int64_t j = t0 + e;
    const uint32_t c = key[J.off + j];
    if (j > 0 && key[J.off + j - 1] == c) continue;
    const int32_t id = (int32_t)val[J.off + j];
    const int32_t old_tail = I.cls_tail[c];
    if (old_tail >= 0) I.pt_next[old_tail] = id; else I.cls_head[c] = id;
    const int b = (int)(c / (uint32_t)(I.pmax + 1)), p = (int)(c % (uint32_t)(I.pmax + 1));
    atomicOr(reinterpret_cast<unsigned long long*>(&I.bm1[(int64_t)b * I.bm_words + (p >> 6)]), 1ULL << (p & 63));
    atomicOr(reinterpret_cast<unsigned long long*>(&I.bm2[(int64_t)b * I.bm_l2 + (p >> 12)]),
             1ULL << ((p >> 6) & 63));
  }
}
// Links inside segments, new class tails, class counts (warp-aggregated).
__global__ void __launch_bounds__(256) k_bulk_tails(Inst* insts, const BulkJob* jobs, const uint32_t* key,
                                                    const uint32_t* val) {
  const BulkJob& J = jobs[blockIdx.y];
  if ((int)blockIdx.x >= J.tiles) return;
  Inst& I = insts[J.inst];
  const int64_t t0 = (int64_t)blockIdx.x * kBulkTile;
  for (int e = threadIdx.x; e < kBulkTile; e += blockDim.x) {
    const int64_t j = t0 + e;
    const bool in = j < J.k;
    const uint32_t c = in ? key[J.off + j] : 0xffffffffu;
    if (in) {
      const int32_t id = (int32_t)val[J.off + j];
      const bool tail = j + 1 == J.k || key[J.off + j + 1] != c;
      I.pt_next[id] = tail ? -1 : (int32_t)val[J.off + j + 1];
      if (tail) I.cls_tail[c] = id;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, c);
    if (in && (peers & ((1u << (threadIdx.x & 31)) - 1u)) == 0) atomicAdd(&I.cls_cnt[c], (int32_t)__popc(peers));
  }
}
// ---------------------------------------------------------------------------
// Burst ingest without a global sort (the default path): the class lists only
// need, for every arrival, the next arrival of the same class in id order.
//  k_ingest_tiles: per 4096-id tile, a stable two-pass radix sort of
//    (class, local index) in shared memory gives the in-tile successors,
//    written to pt_next in id order (coalesced), and one segment record per
//    class present in the tile (class, first, last, count: 8 bytes);
//  k_ingest_stitch: one CTA per instance walks its tiles from the last to the
//    first with a per-class table in shared memory (classes are distinct
//    within a tile, so a tile's segments are stitched in parallel), links each
//    segment's last id to the next tile's first of the class, then splices
//    every class onto its list (queues.hpp:85-92 order: id ascending within a
//    class) and updates counts, bitmaps and the ingest scalars.
// HBM traffic per arrival: 16 B read (arrival, true_rl, prompt) + 4 B written
// (pt_next) + the segments (<= 8 B, ~2 B at cfg3's class spread), against
// ~94 B for sort + scatter + splice.
// ---------------------------------------------------------------------------
constexpr int kTileI = 4096;
EDEV uint64_t seg_pack(uint32_t c, uint32_t f, uint32_t l, uint32_t n) {
  return ((uint64_t)c << 37) | ((uint64_t)f << 25) | ((uint64_t)l << 13) | (uint64_t)n;
}

// One stable pass of the tile by the 8-bit digit at `shift` (warp-ordered
// match_any ranks, exactly as k_radix_scatter's in-tile reorder).
EDEV void tile_radix_pass(const uint32_t* in, uint32_t* out, uint32_t (*cnt)[256], uint32_t* tstart, int shift) {
  constexpr int PER = kTileI / 256;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int d = threadIdx.x; d < 8 * 256; d += blockDim.x) (&cnt[0][0])[d] = 0;
  uint32_t kr[PER], rank[PER];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    kr[r] = in[w * (kTileI / 8) + r * 32 + lane];
    const int d = (int)((kr[r] >> shift) & 255);
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t base = cnt[w][d];
    __syncwarp();
    if ((peers & ((1u << lane) - 1u)) == 0) cnt[w][d] = base + __popc(peers);
    __syncwarp();
    rank[r] = base + __popc(peers & ((1u << lane) - 1u));
  }
  __syncthreads();
  {
    const int d = threadIdx.x;
    uint32_t run = 0;
    for (int ww = 0; ww < 8; ++ww) {
      const uint32_t c = cnt[ww][d];
      cnt[ww][d] = run;
      run += c;
    }
    tstart[d] = run;
  }
  __syncthreads();
  {
    const uint32_t v = tstart[threadIdx.x];
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __shared__ uint32_t ws[8];
    if (lane == 31) ws[w] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int ww = 0; ww < w; ++ww) pre += ws[ww];
    __syncthreads();
    tstart[threadIdx.x] = pre + x - v;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const int d = (int)((kr[r] >> shift) & 255);
    out[tstart[d] + cnt[w][d] + rank[r]] = kr[r];
  }
  __syncthreads();
}

// J.off: the job's first tile * kTileI in `segs`; J.hoff: its first tile in `nseg`.
__global__ void __launch_bounds__(256) k_ingest_tiles(Inst* insts, BulkJob* jobs, uint64_t* segs, int32_t* nseg) {
  BulkJob& J = jobs[blockIdx.y];
  if ((int)blockIdx.x >= J.tiles) return;
  Inst& I = insts[J.inst];
  __shared__ uint32_t ka[kTileI], kb[kTileI];
  __shared__ uint32_t cnt[8][256];
  __shared__ uint32_t tstart[256];
  __shared__ unsigned long long sb[ECONO_MAX_BOUNDS + 2];
  __shared__ unsigned long long smin;
  __shared__ uint32_t wsum[8];
  if (threadIdx.x < ECONO_MAX_BOUNDS + 2) sb[threadIdx.x] = 0;
  if (threadIdx.x == 0) smin = ~0ULL;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kTileI;
  const int n = (int)(J.k - t0 < kTileI ? J.k - t0 : kTileI);
  const double now = I.clock;
  const uint32_t pm1 = (uint32_t)I.pmax + 1;
  unsigned long long mn = ~0ULL;
  uint32_t bc[ECONO_MAX_BOUNDS + 2];
#pragma unroll
  for (int bb = 0; bb < ECONO_MAX_BOUNDS + 2; ++bb) bc[bb] = 0;
  for (int e = threadIdx.x; e < kTileI; e += blockDim.x) {
    uint32_t key = 0xFFFFFFFFu;  // padding sorts after every class (< 2^16)
    if (e < n) {
      const int64_t id = J.first + t0 + e;
      const int b = bucket_d(I, dmax(0.0, slo_of(I, id) - now));
      const int32_t p = I.prompt[id];
      key = (((uint32_t)b * pm1 + (uint32_t)p) << 12) | (uint32_t)e;
      mn = (unsigned long long)p < mn ? (unsigned long long)p : mn;
#pragma unroll
      for (int bb = 0; bb < ECONO_MAX_BOUNDS + 2; ++bb) bc[bb] += b == bb;
    }
    ka[e] = key;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, mn, o);
    mn = x < mn ? x : mn;
  }
#pragma unroll
  for (int bb = 0; bb < ECONO_MAX_BOUNDS + 2; ++bb) {
    uint32_t c = bc[bb];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&sb[bb], (unsigned long long)c);
  }
  if ((threadIdx.x & 31) == 0) atomicMin(&smin, mn);
  tile_radix_pass(ka, kb, cnt, tstart, 12);  // class bits 0..7
  tile_radix_pass(kb, ka, cnt, tstart, 20);  // class bits 8..15
  // sorted by (class, local index): successors, segment starts
  constexpr int PER = kTileI / 256;
  const int j0 = threadIdx.x * PER;
  uint32_t starts = 0;
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const int j = j0 + r;
    if (j < n) {
      const uint32_t k = ka[j], c = k >> 12;
      const bool last = j + 1 >= n || (ka[j + 1] >> 12) != c;
      // scattered within the tile's 16 KB of pt_next: merged in L2 before DRAM
      I.pt_next[J.first + t0 + (k & 4095)] = last ? -1 : (int32_t)(J.first + t0 + (ka[j + 1] & 4095));
      if (j == 0 || (ka[j - 1] >> 12) != c) starts |= 1u << r;
    }
  }
  // exclusive prefix of segment starts over the tile (thread order = sorted order)
  const uint32_t mine = __popc(starts);
  uint32_t x = mine;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  uint32_t pre = 0, total = 0;
  for (int ww = 0; ww < 8; ++ww) {
    if (ww < w) pre += wsum[ww];
    total += wsum[ww];
  }
  uint32_t s = pre + x - mine;
  // compacted segment starts (kb is free after the second pass), then one
  // record per segment: its end is the position before the next start
#pragma unroll
  for (int r = 0; r < PER; ++r)
    if (starts & (1u << r)) kb[s++] = (uint32_t)(j0 + r);
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < total; q += blockDim.x) {
    const uint32_t j = kb[q], e = (q + 1 < total ? kb[q + 1] : (uint32_t)n) - 1;
    segs[J.off + t0 + q] = seg_pack(ka[j] >> 12, ka[j] & 4095, ka[e] & 4095, e - j + 1);
  }
  if (threadIdx.x == 0) {
    nseg[J.hoff + blockIdx.x] = (int32_t)total;
    atomicMin(&J.minp, smin);
  }
  if (threadIdx.x < ECONO_MAX_BOUNDS + 2 && sb[threadIdx.x]) atomicAdd(&J.bcnt[threadIdx.x], sb[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// Burst ingest by range scans (the default when the class table fits shared
// memory): no sort at all. One warp owns a range of kRangeI ids and walks it
// from the last 32-id chunk to the first with a per-class table in shared
// memory, tab[c] = (arrivals of class c seen so far in the range) << 16 |
// (local index of the earliest of them). For each chunk:
//   succ(id) = the next lane of the same class (__match_any_sync peers), else
//              the class's earliest id in the later chunks (tab), else -1;
//   pt_next[id] = succ (one coalesced 128-byte store per chunk);
//   the chunk's lowest lane of each class becomes the class's earliest id.
// A class seen for the first time has its range-last id in that chunk: it
// gets a segment record (appended warp-aggregated) that the end of the range
// completes with the class's first id and count from tab. The stitch then
// links the ranges exactly as it links the tiles of k_ingest_tiles.
// The table covers only the job's class window (k_bulk_plan: the deadline
// buckets the batch's slack range can reach x the trace's prompt range; at
// cfg3 one bucket x 655 prompts = 2.6 KB), so shared memory does not bound
// the warps per SM, and a range holds at most one segment per window class.
// HBM traffic per arrival: 16 B read (arrival, true_rl, prompt) + 4 B written
// (pt_next) + the segment records (8 B written and re-read per class present
// in a range: < 1 B per arrival at cfg3's class spread).
// ---------------------------------------------------------------------------
constexpr int kRangeI = 32768;
constexpr int kRangeU = 8;   // chunks whose fields are loaded before they are scanned
EDEV uint64_t rseg_pack(uint32_t c, uint32_t f, uint32_t l, uint32_t n) {
  return ((uint64_t)c << 48) | ((uint64_t)f << 32) | ((uint64_t)l << 16) | (uint64_t)n;
}

// J.tiles: ranges; J.off: the job's first range * kRangeI in `segs`; J.hoff: its first range in `nseg`.
// Dynamic shared memory: 4 B x window classes. WB >= the bits of a window
// class index (the ballot count of the multisplit; compile-time: no branches).
template <int WB>
__global__ void __launch_bounds__(32) k_ingest_ranges(Inst* insts, BulkJob* jobs, uint64_t* segs, int32_t* nseg) {
  BulkJob& J = jobs[blockIdx.y];
  if ((int)blockIdx.x >= J.tiles) return;
  Inst& I = insts[J.inst];
  extern __shared__ uint32_t rtab[];
  const int lane = threadIdx.x;
  const uint32_t pm1 = (uint32_t)I.pmax + 1;
  // the table covers the job's class window only (k_bulk_plan): t = (b - wb0) * wnp + (p - wp0)
  const int wb0 = J.wb0, wp0 = J.wp0, wnp = J.wnp, wn = J.wnb * J.wnp;
  for (int c = lane; c < wn; c += 32) rtab[c] = 0;
  const int64_t r0 = (int64_t)blockIdx.x * kRangeI;
  const int n = (int)(J.k - r0 < kRangeI ? J.k - r0 : kRangeI);
  const int64_t gbase = J.first + r0;  // global id of local index 0
  const int32_t g32 = (int32_t)gbase;  // ids < 2^31
  // the bucket_d / slo_of operands in registers (same operations as engine.cuh)
  const double now = I.clock, scale = I.slo_scale, tp = I.t_p, tg = I.t_g;
  const int nbd = I.nbd;
  __shared__ double sdb[ECONO_MAX_BOUNDS];
  if (lane < ECONO_MAX_BOUNDS) sdb[lane] = I.dbounds[lane];
  __syncwarp();  // the zeroed table and the bounds, visible to every lane
  const double* A = I.arrival.p + gbase;
  const int32_t* P = I.prompt.p + gbase;
  const int32_t* RL = I.true_rl.p + gbase;
  int32_t* NX = I.pt_next.p + gbase;
  uint64_t* out = segs + J.off + (int64_t)blockIdx.x * J.sstride;
  const unsigned below = (1u << lane) - 1u, above = ~((2u << lane) - 1u);
  int ns = 0;  // segment records appended (warp-uniform)
  bool werr = false;
  // PT classes of a group of arrivals: (deadline bucket of max(0, slo - clock),
  // prompt). bucket_d's "first bound the slack is below" as a warp-uniform
  // loop over the bounds (highest first), every arrival of the group at once.
  auto classes = [&](const double* a, const int32_t* p, const int32_t* r, uint32_t* cc, const bool* val) {
    double sl[kRangeU];
    uint32_t b[kRangeU];
#pragma unroll
    for (int u = 0; u < kRangeU; ++u) {
      sl[u] = dmax(0.0, (a[u] + scale * (tp + tg * (double)r[u])) - now);
      b[u] = (uint32_t)nbd;
    }
#pragma unroll 1
    for (int q = nbd - 1; q >= 0; --q) {
      const double d = sdb[q];
#pragma unroll
      for (int u = 0; u < kRangeU; ++u) b[u] = sl[u] < d ? (uint32_t)q : b[u];
    }
#pragma unroll
    for (int u = 0; u < kRangeU; ++u) {
      const uint32_t t = (b[u] - (uint32_t)wb0) * (uint32_t)wnp + (uint32_t)(p[u] - wp0);
      // outside the window (impossible by k_bulk_plan's bound): flagged, kept inside the table
      if (val[u] && t >= (uint32_t)wn) werr = true;
      cc[u] = t < (uint32_t)wn ? t : 0u;
    }
  };
  // the lanes of a chunk holding the same window class c (v: the lane holds
  // an arrival). WB > 0: a warp multisplit, one ballot per class bit;
  // WB == 0: __match_any_sync (it serialises over the ~30 distinct classes
  // of a chunk). Computed for a whole group before its serial scan (ILP).
  auto peers_of = [&](uint32_t c, bool v) -> unsigned {
    if (WB == 0) return __match_any_sync(0xffffffffu, v ? c : 0xFFFFFFFFu);
    unsigned d = __ballot_sync(0xffffffffu, v);  // lanes whose validity or some class bit differs
    d = v ? ~d : d;
#pragma unroll
    for (int i = 0; i < (WB > 0 ? WB : 1); ++i) {
      unsigned bb;
      asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.u32 p, t, 0;\n\t"
          "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t}"
          : "=r"(bb) : "r"(c), "r"(1u << i));
      const unsigned m = (c & (1u << i)) ? 0xFFFFFFFFu : 0u;
      d |= bb ^ m;
    }
    return ~d;
  };
  // one 32-id chunk of the backward scan: chunk k, nx = &pt_next[this lane's id]
  auto scan = [&](int k, uint32_t c, bool v, int32_t* nx, unsigned peers) {
    const int e = k * 32 + lane;
    const uint32_t T = v ? rtab[c] : 0u;
    const unsigned up = peers & above;
    const int32_t succ = up ? g32 + (k * 32 + __ffs(up) - 1) : (T ? g32 + (int32_t)(T & 0xFFFFu) : -1);
    if (v) __stcs(nx, succ);
    __syncwarp();
    if (v && (peers & below) == 0u) rtab[c] = (((T >> 16) + (uint32_t)__popc(peers)) << 16) | (uint32_t)e;
    const bool fresh = v && T == 0u && up == 0u;  // the range's last id of a class seen for the first time
    const unsigned fb = __ballot_sync(0xffffffffu, fresh);
    if (fresh) out[ns + __popc(fb & below)] = rseg_pack(c, 0, (uint32_t)e, 0);
    ns += __popc(fb);
    __syncwarp();
  };
  const int nch = (n + 31) >> 5;
  const int g0 = nch % kRangeU ? nch % kRangeU : kRangeU;  // chunks in the top group
  {  // the top group: possibly fewer chunks, its top chunk possibly partial (checked path)
    double a[kRangeU];
    int32_t p[kRangeU], r[kRangeU];
    uint32_t cc[kRangeU];
    bool val[kRangeU];
#pragma unroll
    for (int u = 0; u < kRangeU; ++u) {
      const int e = (nch - 1 - u) * 32 + lane;
      const bool v = u < g0 && e < n;
      val[u] = v;
      a[u] = v ? __ldcs(A + e) : 0.0;
      p[u] = v ? __ldcs(P + e) : 0;
      r[u] = v ? __ldcs(RL + e) : 0;
    }
    classes(a, p, r, cc, val);
#pragma unroll
    for (int u = 0; u < kRangeU; ++u) {
      const int e = (nch - 1 - u) * 32 + lane;
      if (u < g0) scan(nch - 1 - u, e < n ? cc[u] : 0xFFFFFFFFu, e < n, NX + e, peers_of(cc[u], e < n));
    }
  }
  // full groups of kRangeU chunks below it, each loaded one group ahead of its
  // scan so that the HBM latency overlaps the scan; per-lane pointers with
  // constant per-chunk offsets (no 64-bit index arithmetic per access)
  int k0 = nch - 1 - g0;
  if (k0 >= 0) {
    double a[kRangeU], a2[kRangeU];
    int32_t p[kRangeU], r[kRangeU], p2[kRangeU], r2[kRangeU];
    auto load = [&](int kt, double* AA, int32_t* PP, int32_t* RR) {
      const int e = kt * 32 + lane;
      const double* pa = A + e;
      const int32_t* pp = P + e;
      const int32_t* pr = RL + e;
#pragma unroll
      for (int u = 0; u < kRangeU; ++u) {
        AA[u] = __ldcs(pa - 32 * u);
        PP[u] = __ldcs(pp - 32 * u);
        RR[u] = __ldcs(pr - 32 * u);
      }
    };
    auto group = [&](int kt, const double* AA, const int32_t* PP, const int32_t* RR) {
      uint32_t cc[kRangeU];
      bool val[kRangeU];
#pragma unroll
      for (int u = 0; u < kRangeU; ++u) val[u] = true;
      classes(AA, PP, RR, cc, val);
      int32_t* nx = NX + (kt * 32 + lane);
      unsigned pe[kRangeU];
#pragma unroll
      for (int u = 0; u < kRangeU; ++u) pe[u] = peers_of(cc[u], true);
#pragma unroll
      for (int u = 0; u < kRangeU; ++u) scan(kt - u, cc[u], true, nx - 32 * u, pe[u]);
    };
    load(k0, a, p, r);
    for (;;) {  // two groups per trip: the buffers swap roles without register moves
      if (k0 >= kRangeU) load(k0 - kRangeU, a2, p2, r2);
      group(k0, a, p, r);
      if ((k0 -= kRangeU) < 0) break;
      if (k0 >= kRangeU) load(k0 - kRangeU, a, p, r);
      group(k0, a2, p2, r2);
      if ((k0 -= kRangeU) < 0) break;
    }
  }
  __syncwarp();
  for (int q = lane; q < ns; q += 32) {  // complete the records: global class, first id and count
    const uint64_t s = out[q];
    const uint32_t t = (uint32_t)(s >> 48), T = rtab[t];
    const uint32_t c = ((uint32_t)wb0 + t / (uint32_t)wnp) * pm1 + (uint32_t)wp0 + t % (uint32_t)wnp;
    out[q] = rseg_pack(c, T & 0xFFFFu, (uint32_t)(s >> 16) & 0xFFFFu, T >> 16);
  }
  if (lane == 0) nseg[J.hoff + blockIdx.x] = ns;
  if (__any_sync(0xffffffffu, werr) && lane == 0) atomicExch(&J.werr, 1);
  // the batch's bucket counts and smallest prompt come from the class counts (k_ingest_stitch<true>)
}

// One CTA per job; dynamic shared memory: 3 x ncls int32 (+ bucket sums).
// RANGES: the segments of k_ingest_ranges (rseg_pack, kRangeI ids per range),
// else those of k_ingest_tiles (seg_pack, kTileI ids per tile).
template <bool RANGES>
__global__ void __launch_bounds__(512) k_ingest_stitch(Inst* insts, const BulkJob* jobs, const uint64_t* segs,
                                                       const int32_t* nseg) {
  const BulkJob& J = jobs[blockIdx.x];
  Inst& I = insts[J.inst];
  const int ncls = I.nbuckets * (I.pmax + 1);
  extern __shared__ int32_t tab[];
  int32_t* first = tab;
  int32_t* tail = tab + ncls;
  int32_t* cnt = tab + 2 * ncls;
  for (int c = threadIdx.x; c < ncls; c += blockDim.x) {
    first[c] = -1;
    cnt[c] = 0;
  }
  __syncthreads();
  constexpr int64_t span = RANGES ? kRangeI : kTileI;
  for (int t = J.tiles - 1; t >= 0; --t) {
    const int ns = nseg[J.hoff + t];
    const int64_t base = J.first + (int64_t)t * span;
    for (int q = threadIdx.x; q < ns; q += blockDim.x) {
      const uint64_t pk = segs[J.off + (int64_t)t * J.sstride + q];
      int c;
      int32_t gf, gl, m;
      if (RANGES) {
        c = (int)(pk >> 48);
        gf = (int32_t)(base + ((pk >> 32) & 0xFFFF));
        gl = (int32_t)(base + ((pk >> 16) & 0xFFFF));
        m = (int32_t)(pk & 0xFFFF);
      } else {
        c = (int)(pk >> 37);
        gf = (int32_t)(base + ((pk >> 25) & 4095));
        gl = (int32_t)(base + ((pk >> 13) & 4095));
        m = (int32_t)(pk & 8191);
      }
      const int32_t nx = first[c];
      if (nx >= 0) I.pt_next[gl] = nx; else tail[c] = gl;
      first[c] = gf;
      cnt[c] += m;
    }
    __syncthreads();
  }
  const int pm1 = I.pmax + 1;
  __shared__ int32_t sbc[ECONO_MAX_BOUNDS + 2];  // RANGES: bucket counts and the smallest prompt, from the class counts
  __shared__ int32_t smin;
  if (RANGES) {
    if (threadIdx.x < ECONO_MAX_BOUNDS + 2) sbc[threadIdx.x] = 0;
    if (threadIdx.x == 0) smin = INT32_MAX;
    __syncthreads();
  }
  for (int c = threadIdx.x; c < ncls; c += blockDim.x) {
    if (cnt[c] == 0) continue;
    if (RANGES) {
      atomicAdd(&sbc[c / pm1], cnt[c]);
      atomicMin(&smin, c % pm1);
    }
    const int32_t old_tail = I.cls_tail[c];
    if (old_tail >= 0) I.pt_next[old_tail] = first[c]; else I.cls_head[c] = first[c];
    I.cls_tail[c] = tail[c];
    I.cls_cnt[c] += cnt[c];
    const int b = c / pm1, p = c % pm1;
    atomicOr(reinterpret_cast<unsigned long long*>(&I.bm1[(int64_t)b * I.bm_words + (p >> 6)]), 1ULL << (p & 63));
    atomicOr(reinterpret_cast<unsigned long long*>(&I.bm2[(int64_t)b * I.bm_l2 + (p >> 12)]),
             1ULL << ((p >> 6) & 63));
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // the ingest scalars (k_bulk_finish)
    if (RANGES && J.werr && !I.error) {  // an arrival outside k_bulk_plan's class window
      I.error = ERR_TABLE_OVERFLOW;
      I.err_val = 99;
      I.err_id = (int32_t)J.first;
    }
    I.arrival_cursor = J.first + J.k;
    I.pt_count += (int32_t)J.k;
    I.ev_total += J.k;
    if (RANGES) {
      if ((int64_t)smin < I.pt_min_lb) I.pt_min_lb = (int64_t)smin;
      for (int b = 0; b < I.nbuckets; ++b) I.bcnt[b] += sbc[b];
    } else {
      if ((int64_t)J.minp < I.pt_min_lb) I.pt_min_lb = (int64_t)J.minp;
      for (int b = 0; b < I.nbuckets; ++b) I.bcnt[b] += (int32_t)J.bcnt[b];
    }
  }
}

// The instance scalars ingest() updates (engine.hpp:216-235).
__global__ void k_bulk_finish(Inst* insts, const BulkJob* jobs) {
  const BulkJob& J = jobs[blockIdx.x];
  if (threadIdx.x != 0) return;
  Inst& I = insts[J.inst];
  I.arrival_cursor = J.first + J.k;
  I.pt_count += (int32_t)J.k;
  I.ev_total += J.k;
  if ((int64_t)J.minp < I.pt_min_lb) I.pt_min_lb = (int64_t)J.minp;
  for (int b = 0; b < I.nbuckets; ++b) I.bcnt[b] += (int32_t)J.bcnt[b];
}
// Per instance: the arrivals ingest() would admit at the current clock.
// Per instance: the arrivals ingest() would admit at the current clock
// (plan[4i], plan[4i+1]) and the window of PT classes they can fall in
// (plan[4i+2]: buckets lo | hi << 32, plan[4i+3]: prompts lo | hi << 32).
// slack = max(0, arrival + slo_scale * (t_p + t_g * rl) - clock) is monotone
// in the arrival and in rl separately (IEEE operations round monotonically),
// and bucket_d is monotone in the slack, so the buckets at the four corners
// of [first arrival, last arrival] x [min rl, max rl] bound every arrival's
// bucket; the prompts lie in the trace's range. Anything non-finite: the
// whole class table.
__global__ void k_bulk_plan(const Inst* insts, int64_t* plan) {
  const Inst& I = insts[blockIdx.x];
  if (threadIdx.x != 0) return;
  int64_t first = I.arrival_cursor, k = 0;
  if (I.ordered && !I.record_events && !I.error && first < I.n) {
    const double lim = I.clock + 1e-12;
    if (I.arrival[first] <= lim) {
      int64_t lo = first + 1, hi = I.n;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (I.arrival[mid] <= lim) lo = mid + 1; else hi = mid;
      }
      k = lo - first;
    }
  }
  int64_t blo = 0, bhi = I.nbd, plo = 1, phi = I.pmax;
  if (k > 0 && I.tr_pmin <= I.tr_pmax && I.tr_rmin <= I.tr_rmax) {
    const double as[2] = {I.arrival[first], I.arrival[first + k - 1]};
    const int32_t rs[2] = {I.tr_rmin, I.tr_rmax};
    bool finite = true;
    int64_t mn = I.nbd, mx = 0;
    for (int x = 0; x < 2; ++x)
      for (int y = 0; y < 2; ++y) {
        const double v = (as[x] + I.slo_scale * (I.t_p + I.t_g * (double)rs[y])) - I.clock;
        finite = finite && isfinite(v);
        const int b = bucket_d(I, dmax(0.0, v));
        mn = b < mn ? b : mn;
        mx = b > mx ? b : mx;
      }
    if (finite) {
      blo = mn;
      bhi = mx;
    }
    plo = I.tr_pmin;
    phi = I.tr_pmax < I.pmax ? I.tr_pmax : I.pmax;
    if (plo > phi) plo = phi;
  }
  plan[4 * blockIdx.x] = first;
  plan[4 * blockIdx.x + 1] = k;
  plan[4 * blockIdx.x + 2] = blo | (bhi << 32);
  plan[4 * blockIdx.x + 3] = plo | (phi << 32);
}

// Partial sums, grid-wide: block (x, instance) reduces a strided slice of
// the instance's requests (one pass over ~89 B of SoA per request, HBM-bound)
// into scr[instance][x][16]; k_partials_finish then folds the slices in a
// fixed order, so results are deterministic run to run.
__global__ void __launch_bounds__(256) k_partials_slices(const Inst* insts, double* scr) {
  const Inst& I = insts[blockIdx.y];
  double acc[15];
  for (int k = 0; k < 15; ++k) acc[k] = 0.0;
  partials_accumulate(I, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x, acc);
  for (int k = 0; k < 15; ++k) {
    double v = acc[k];
    for (int o = 16; o > 0; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, v, o);
      v = k == 10 ? (x > v ? x : v) : v + x;
    }
    acc[k] = v;
  }
  __shared__ double ws[8][16];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 15; ++k) ws[w][k] = acc[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot[15];
    for (int k = 0; k < 15; ++k) tot[k] = ws[0][k];
    for (int j = 1; j < (int)(blockDim.x >> 5); ++j) partials_combine(tot, ws[j]);
    double* o = scr + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16;
    for (int k = 0; k < 15; ++k) o[k] = tot[k];
  }
}
__global__ void __launch_bounds__(32) k_partials_finish(const Inst* insts, const double* scr, int32_t slices,
                                                        double* out) {
  if (threadIdx.x != 0) return;
  const double* s0 = scr + (size_t)blockIdx.x * slices * 16;
  double acc[15];
  for (int k = 0; k < 15; ++k) acc[k] = s0[k];
  for (int j = 1; j < slices; ++j) partials_combine(acc, s0 + (size_t)j * 16);
  partials_finish(insts[blockIdx.x], acc, out + (size_t)blockIdx.x * ECONO_PARTIAL_WORDS);
}

// Materialises every instance's JCT keys (one pass over 32 B of SoA per
// request -> 8 B key): keys[off[inst] + i].
__global__ void __launch_bounds__(256) k_jct_keys(const Inst* insts, const int64_t* off, uint64_t* keys) {
  const Inst& I = insts[blockIdx.y];
  uint64_t* out = keys + off[blockIdx.y];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < I.n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = jct_key(I, i);
}
// One radix-select pass: for each of `nt` targets, a histogram of the next
// `dbits` bits of the keys whose top `consumed` bits equal the target's
// prefix. Per-instance mode (hist/prefixes indexed by instance) or global
// mode (one histogram over every instance). Shared-memory counters, flushed
// with one global atomic per non-empty bin.
__global__ void __launch_bounds__(256) k_jct_hist(const Inst* insts, const int64_t* off, const uint64_t* keys,
                                                  int32_t per_instance, int32_t nt, const uint64_t* prefixes,
                                                  int32_t consumed, int32_t dbits, unsigned long long* hist) {
  extern __shared__ uint32_t sh[];
  const int bins = 1 << dbits;
  for (int j = threadIdx.x; j < nt * bins; j += blockDim.x) sh[j] = 0;
  __syncthreads();
  const Inst& I = insts[blockIdx.y];
  const int64_t n = I.n;
  const uint64_t* kk = keys ? keys + off[blockIdx.y] : nullptr;
  const uint64_t* pf = prefixes + (per_instance ? (size_t)blockIdx.y * nt : 0);
  uint64_t p[8];
  for (int t = 0; t < nt; ++t) p[t] = pf[t];
  // JCTs cluster, so many lanes hit the same bin: lanes with equal (target,
  // digit) are merged with one match_any and their leader adds the count.
  // After the first pass almost no key matches a target's prefix, and a warp
  // with no match skips straight to its next load (a pure HBM stream).
  const int64_t n_pad = (n + 31) & ~(int64_t)31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += 2 * stride) {
    const bool in0 = i < n, in1 = i + stride < n;
    uint64_t k0 = 0, k1 = 0;
    if (kk) {
      k0 = in0 ? __ldcs(kk + i) : 0;
      k1 = in1 ? __ldcs(kk + i + stride) : 0;
    } else {  // keys derived on the fly (no key buffer)
      k0 = in0 ? jct_key(I, i) : 0;
      k1 = in1 ? jct_key(I, i + stride) : 0;
    }
#pragma unroll 2
    for (int h = 0; h < 2; ++h) {
      const uint64_t k = h ? k1 : k0;
      const bool in = h ? in1 : in0;
      for (int t = 0; t < nt; ++t) {
        const bool m = in && key_matches(k, p[t], consumed);
        if (!__any_sync(0xffffffffu, m)) continue;
        const int bin = m ? (int)(t * bins + key_digit(k, consumed, dbits)) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, bin);
        if (m && (peers & ((1u << (threadIdx.x & 31)) - 1u)) == 0) atomicAdd(&sh[bin], (uint32_t)__popc(peers));
      }
    }
  }
  __syncthreads();
  unsigned long long* h = hist + (per_instance ? (size_t)blockIdx.y * nt * bins : 0);
  for (int j = threadIdx.x; j < nt * bins; j += blockDim.x)
    if (sh[j]) atomicAdd(&h[j], (unsigned long long)sh[j]);
}
#endif

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

void set_err(char* err, size_t errlen, const char* fmt, ...) {
  if (!err || !errlen) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, errlen, fmt, ap);
  va_end(ap);
}

#ifdef ECONO_HOSTSIM
int dev_alloc(void** p, size_t sz) { *p = calloc(1, sz ? sz : 8); return *p ? 0 : 1; }
void dev_free(void* p) { free(p); }
int dev_h2d(void* d, const void* h, size_t sz) { memcpy(d, h, sz); return 0; }
int dev_d2h(void* h, const void* d, size_t sz) { memcpy(h, d, sz); return 0; }
#else
int dev_alloc(void** p, size_t sz) {
  const auto t0 = std::chrono::steady_clock::now();
  if (cudaMalloc(p, sz ? sz : 8) != cudaSuccess) return 1;
  const auto t1 = std::chrono::steady_clock::now();
  const int rc = cudaMemset(*p, 0, sz ? sz : 8) != cudaSuccess;
  if (sz > ((size_t)1 << 30) && getenv("ECONO_VERBOSE")) {
    cudaDeviceSynchronize();
    const auto t2 = std::chrono::steady_clock::now();
    fprintf(stderr, "[econo] dev_alloc %zu MB: malloc %.1f ms memset %.1f ms\n", sz >> 20,
            std::chrono::duration<double, std::milli>(t1 - t0).count(),
            std::chrono::duration<double, std::milli>(t2 - t1).count());
  }
  return rc;
}
void dev_free(void* p) { if (p) cudaFree(p); }
int dev_h2d(void* d, const void* h, size_t sz) { return cudaMemcpy(d, h, sz, cudaMemcpyHostToDevice) != cudaSuccess; }
int dev_d2h(void* h, const void* d, size_t sz) { return cudaMemcpy(h, d, sz, cudaMemcpyDeviceToHost) != cudaSuccess; }
#endif

struct Arena {  // bump allocator over one device allocation, 256-byte aligned
  size_t off = 0;
  char* base = nullptr;
  template <class T>
  T* take(int64_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += sizeof(T) * (size_t)(count > 0 ? count : 1);
    return p;
  }
};

int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

// Lays out every SoA array of one instance; with base == nullptr it only sizes.
void layout(Inst& I, char* base, size_t* bytes) {
  Arena a;
  a.base = base;
  const int64_t n = I.n;
  I.arrival = a.take<double>(n);
  I.prompt = a.take<int32_t>(n);
  I.true_rl = a.take<int32_t>(n);
  GP<int32_t>* i32s[] = {&I.predicted, &I.generated, &I.occupied, &I.allowance, &I.gen_epoch,
                      &I.preempt_count, &I.reserve_draws, &I.held, &I.reg_head,
                      &I.reserved, &I.written, &I.sidx, &I.pt_next};
  for (auto p : i32s) *p = a.take<int32_t>(n);
  // chunked prefills (baselines) only; econoserve derives it (engine.cuh)
  I.prefill_done = a.take<int32_t>(I.base ? n : 1);
  I.gt_next = I.pt_next.p;
  I.state = a.take<uint8_t>(n);
  I.flags = a.take<uint8_t>(n);
  GP<double>* f64s[] = {&I.waiting, &I.preempt_t, &I.exec_t, &I.first_tok,
                     &I.compl_clock, &I.last_enq, &I.penalty, &I.sched_share};
  for (auto p : f64s) *p = a.take<double>(n);
  // Request::dispatch_time is read only by the baselines (engine.hpp:527, 615)
  I.dispatch_t = a.take<double>(I.base ? n : 1);
  const int64_t rc = I.reg_cap;
  I.rg_start = a.take<int32_t>(rc);
  I.rg_len = a.take<int32_t>(rc);
  I.rg_owner = a.take<int32_t>(rc);
  I.rg_next = a.take<int32_t>(rc);
  I.reg_free = a.take<int32_t>(rc);
  I.addr = a.take<int32_t>(rc + W);
  if (I.ordered) {
    const int64_t nc = (int64_t)I.nbuckets * (I.pmax + 1);
    I.cls_head = a.take<int32_t>(nc);
    I.cls_tail = a.take<int32_t>(nc);
    I.cls_cnt = a.take<int32_t>(nc);
    I.bm1 = a.take<uint64_t>((int64_t)I.nbuckets * I.bm_words);
    I.bm2 = a.take<uint64_t>((int64_t)I.nbuckets * I.bm_l2);
  } else {
    I.tree = a.take<int32_t>(I.tree_off[I.tree_levels - 1] + 1);
  }
  const int64_t gc = I.grp_cap;
  I.gr_id = a.take<uint64_t>(gc);
  I.gr_seq = a.take<uint64_t>(gc);
  GP<int32_t>* g32[] = {&I.gr_rl, &I.gr_head, &I.gr_tail, &I.gr_cnt, &I.gr_db, &I.gr_kb, &I.gr_maxocc, &I.grp_free,
                        &I.gr_hd};
  for (auto p : g32) *p = a.take<int32_t>(gc);
  I.gq = a.take<int32_t>(gc + W);
  I.rl_map = a.take<int32_t>(I.rl_cap);
  I.gr_formed = a.take<double>(gc);
  I.gr_mindl = a.take<double>(gc);
  I.gr_dem = a.take<int64_t>(gc);
  I.run = a.take<int32_t>(I.run_cap + W);
  I.slots = a.take<int32_t>(I.slot_cap + W);
  GP<int32_t>* sl[] = {&I.sl_host, &I.sl_off, &I.sl_len, &I.sl_abs, &I.sl_hosted, &I.sl_free};
  for (auto p : sl) *p = a.take<int32_t>(I.slot_cap + W);
  I.ptiter_id = a.take<int32_t>(I.ptiter_cap);
  I.ptiter_tok = a.take<int32_t>(I.ptiter_cap);
  I.adm = a.take<int32_t>(I.adm_cap);
  I.sel_ids = a.take<int32_t>(I.sel_cap);
  I.selg_start = a.take<int32_t>(I.sel_cap + 1);
  I.selg_rl = a.take<int32_t>(I.sel_cap + 1);
  const int64_t pc = 2 * (int64_t)I.scr_cap + W;
  GP<int32_t>* pl[] = {&I.wa_w, &I.wa_b, &I.wa_l, &I.wa_u, &I.wb_w, &I.wb_b, &I.wb_l, &I.wb_u,
                    &I.cd_ri, &I.cd_abs, &I.cd_use, &I.cd_len, &I.assigned,
                    &I.os_host, &I.os_hosted, &I.os_off, &I.os_len, &I.os_abs, &I.tmp_a, &I.tmp_b, &I.tmp_c};
  for (auto p : pl) *p = a.take<int32_t>(pc);
  // baseline policies only (admit order <= running + this iteration's PTs)
  I.admo = a.take<int32_t>(I.base ? (int64_t)I.run_cap + I.ptiter_cap + W : 1);
  I.ongo = a.take<int32_t>(I.base ? (int64_t)I.run_cap + I.ptiter_cap + W : 1);
  I.ptarget = a.take<int32_t>(I.base ? n : 1);
  I.mt = a.take<uint64_t>(312);
  I.pmt = a.take<uint64_t>(312);
  I.hist = a.take<int64_t>(I.hist_cap);
  *bytes = a.off + 256;
}

// Rebases every pointer field of a copied Inst from one arena base to another.
void rebase(Inst& I, const char* from, char* to, size_t bytes) {
  char* fields = reinterpret_cast<char*>(&I.arrival);
  char* end = reinterpret_cast<char*>(&I.hist) + sizeof(I.hist);
  for (char* p = fields; p < end; p += sizeof(void*)) {
    uintptr_t v;
    memcpy(&v, p, sizeof(v));
    if (v >= (uintptr_t)from && v < (uintptr_t)from + bytes) {
      v = v - (uintptr_t)from + (uintptr_t)to;
      memcpy(p, &v, sizeof(v));
    }
  }
}

// Option validation in the reference constructor's order (engine.hpp:81-100).
int validate(const EconoOptions* o, int64_t n, char* err, size_t errlen) {
  const bool econo = o->policy >= ECONO_POLICY_ECONO_D && o->policy <= ECONO_POLICY_ECONO_FULL;
  if (o->kvc_capacity < 1) return set_err(err, errlen, "kvc capacity must be >= 1"), ECONO_ECONFIG;
  if (o->kvc_block_size < 1) return set_err(err, errlen, "kvc block_size must be >= 1"), ECONO_ECONFIG;
  const double rf = econo ? o->reserved_fraction : 0.0;
  if (rf < 0.0 || rf >= 1.0) return set_err(err, errlen, "reserved_fraction must be in [0, 1)"), ECONO_ECONFIG;
  if (o->n_deadline_bounds < 0 || o->n_deadline_bounds > ECONO_MAX_BOUNDS || o->n_kvc_bounds < 0 ||
      o->n_kvc_bounds > ECONO_MAX_BOUNDS || o->n_length_bounds < 0 || o->n_length_bounds > ECONO_MAX_BOUNDS)
    return set_err(err, errlen, "ordering: at most %d bucket boundaries", ECONO_MAX_BOUNDS), ECONO_ECONFIG;
  for (int i = 1; i < o->n_deadline_bounds; ++i)
    if (o->deadline_bounds[i] < o->deadline_bounds[i - 1]) goto unordered;
  for (int i = 1; i < o->n_kvc_bounds; ++i)
    if (o->kvc_bounds[i] < o->kvc_bounds[i - 1]) goto unordered;
  for (int i = 1; i < o->n_length_bounds; ++i)
    if (o->length_bounds[i] < o->length_bounds[i - 1]) goto unordered;
  if (o->tfs < 1) return set_err(err, errlen, "tfs must be >= 1"), ECONO_ECONFIG;
  if (o->chunk_size < 1) return set_err(err, errlen, "chunk_size must be >= 1"), ECONO_ECONFIG;
  if (o->batch_size_cap < 1) return set_err(err, errlen, "batch_size_cap must be >= 1"), ECONO_ECONFIG;
  if (o->padding_ratio < 0.0) return set_err(err, errlen, "padding_ratio must be >= 0"), ECONO_ECONFIG;
  if (o->reserved_fraction < 0.0 || o->reserved_fraction >= 1.0)
    return set_err(err, errlen, "reserved_fraction must be in [0, 1)"), ECONO_ECONFIG;
  if (o->buffer_ratio < 0.0) return set_err(err, errlen, "buffer_ratio must be >= 0"), ECONO_ECONFIG;
  if (!(o->t_base > 0.0)) return set_err(err, errlen, "cost model: t_base must be > 0"), ECONO_ECONFIG;
  if (!(o->t_token > 0.0)) return set_err(err, errlen, "cost model: t_token must be > 0"), ECONO_ECONFIG;
  if (o->cost_tfs < 1) return set_err(err, errlen, "cost model: tfs must be >= 1"), ECONO_ECONFIG;
  if (o->preempt_offload_penalty < 0.0 || o->preempt_free_penalty < 0.0 || o->reserve_penalty < 0.0 ||
      o->sched_cost_per_exam < 0.0 || o->swap_stall < 0.0)
    return set_err(err, errlen, "cost model: penalties must be >= 0"), ECONO_ECONFIG;
  if (o->pred_sigma < 0.0) return set_err(err, errlen, "predictor sigma must be >= 0"), ECONO_ECONFIG;
  if (o->pred_accuracy < 0.0 || o->pred_accuracy > 1.0)
    return set_err(err, errlen, "predictor accuracy must be in [0,1]"), ECONO_ECONFIG;
  if (o->pred_tolerance < 0.0) return set_err(err, errlen, "predictor tolerance must be >= 0"), ECONO_ECONFIG;
  if (o->pred_padding_ratio < 0.0) return set_err(err, errlen, "padding_ratio must be >= 0"), ECONO_ECONFIG;
  if (o->pred_quantum < 1) return set_err(err, errlen, "predictor quantum must be >= 1"), ECONO_ECONFIG;
  if (n <= 0) return set_err(err, errlen, "trace is empty"), ECONO_ECONFIG;
  if (o->policy < ECONO_POLICY_ORCA || o->policy > ECONO_POLICY_ECONO_FULL)
    return set_err(err, errlen, "unknown policy code %d", o->policy), ECONO_ECONFIG;
  if (o->kvc_capacity >= (int64_t)1 << 30)
    return set_err(err, errlen, "kvc capacity must be < 2^30 tokens on the device path"), ECONO_ECONFIG;
  return ECONO_OK;
unordered:
  return set_err(err, errlen, "ordering bucket boundaries must be increasing"), ECONO_ECONFIG;
}

// Fills configuration fields and capacities of an Inst from options + trace.
// scan = false (the device path): the per-record length checks run in
// k_init_soa instead of a host pass over every trace; only Orca's derived
// max_output_len still needs the host scan.
int configure(Inst& I, const EconoOptions* o, const EconoTraceRecord* t, int64_t n, char* err, size_t errlen,
              bool scan = true) {
  memset(&I, 0, sizeof(I));
  if (n >= (int64_t)1 << 31) return set_err(err, errlen, "trace longer than 2^31 requests"), ECONO_ECONFIG;
  int64_t pmax = 1, rmax = 0;
  const int64_t nscan = (scan || (o->policy == ECONO_POLICY_ORCA && o->max_output_len <= 0)) ? n : 0;
  for (int64_t i = 0; i < nscan; ++i) {
    if (t[i].prompt_len < 1 || t[i].prompt_len >= ((int64_t)1 << 30) || t[i].true_rl < 1 ||
        t[i].true_rl >= ((int64_t)1 << 30))
      return set_err(err, errlen, "request %lld: prompt_len and response_len must be in [1, 2^30)", (long long)i),
             ECONO_ECONFIG;
    pmax = imax(pmax, t[i].prompt_len);
    rmax = imax(rmax, t[i].true_rl);
  }
  I.n = (int32_t)n;
  I.policy = o->policy;
  I.ordered = o->policy == ECONO_POLICY_ECONO_SDO || o->policy == ECONO_POLICY_ECONO_FULL;
  I.grouping = o->policy != ECONO_POLICY_ECONO_D;
  I.base = o->policy < ECONO_POLICY_ECONO_D ? 1 : 0;
  I.batch_cap = o->batch_size_cap;
  I.recompute = o->vllm_recompute ? 1 : 0;
  I.chunk = o->chunk_size;
  I.swap_stall = o->swap_stall;
  I.admission_open = 1;
  // max_output_len <= 0 derives it from the trace (engine.hpp:178-180)
  I.max_out = o->max_output_len > 0 ? o->max_output_len : rmax;
  I.full = o->policy == ECONO_POLICY_ECONO_FULL;
  I.pred_model = o->pred_model;
  I.nbd = o->n_deadline_bounds;
  I.nbk = o->n_kvc_bounds;
  for (int i = 0; i < ECONO_MAX_BOUNDS; ++i) {
    I.dbounds[i] = o->deadline_bounds[i];
    I.kbounds[i] = o->kvc_bounds[i];
  }
  I.record_events = o->record_events ? 1 : 0;
  I.record_samples = o->record_samples ? 1 : 0;
  I.tfs = o->tfs;  // cost_.tfs = pol_.tfs (engine.hpp:98)
  I.capacity = o->kvc_capacity;
  I.block = o->kvc_block_size;
  // the reserved pool exists for the econoserve family only (engine.hpp:86-87)
  I.reserve_cap = I.base ? 0 : (int64_t)llround(o->reserved_fraction * (double)o->kvc_capacity);
  I.general_cap = I.capacity - I.reserve_cap;
  I.pred_quantum = o->pred_quantum;
  I.t_base = o->t_base;
  I.t_token = o->t_token;
  I.over_rate = o->t_token_over < 0.0 ? o->t_token : o->t_token_over;
  I.reserve_penalty = o->reserve_penalty;
  I.pen_free = o->preempt_free_penalty;
  I.pen_offload = o->preempt_offload_penalty;
  I.sched_cost = o->sched_cost_per_exam;
  I.pred_sigma = o->pred_sigma;
  I.pred_accuracy = o->pred_accuracy;
  I.pred_tol = o->pred_tolerance;
  I.pred_pad = o->pred_padding_ratio;
  I.slo_scale = o->slo_scale;
  I.buffer_ratio = o->buffer_ratio;
  I.free_total = I.general_cap;
  I.pt_min_lb = INT64_MAX;
  I.tr_pmin = I.tr_rmin = INT32_MAX;  // k_init_soa narrows them
  I.tr_pmax = I.tr_rmax = 0;
  I.ovf_id = INT64_MAX;  // no saturated prediction
  I.ovf_dem = 0;
  I.skip = (getenv("ECONO_NO_SKIP") || I.base) ? 0 : 1;
  // capacities
  // PT class tables span prompts 1..pmax. Ordered (econoserve) policies
  // reject any prompt above the reserved pool at init (engine.hpp:202-206),
  // so the pool size bounds the classes without scanning the trace.
  I.pmax = (int32_t)(I.ordered ? imax(1, I.reserve_cap) : pmax);
  I.nbuckets = I.nbd + 1;
  I.bm_words = (I.pmax >> 6) + 1;
  I.bm_l2 = (I.bm_words >> 6) + 1;
  {
    int64_t len = n, off = 0;
    int lv = 0;
    for (;;) {
      I.tree_off[lv] = (int32_t)off;
      I.tree_len[lv] = (int32_t)len;
      off += len;
      ++lv;
      if (len == 1) break;
      len = (len + 31) / 32;
    }
    I.tree_levels = lv;
  }
  const int64_t cap = I.capacity;
  I.reg_cap = (int32_t)(I.general_cap + 2);
  // Every waiting GT holds KVC (its prompt in the reserve after prefill,
  // engine.hpp:794-809 / SURVEY A.7, or its regions after an offload-free
  // preemption, engine.hpp:904-928), and every queued group is non-empty, so
  // at most `capacity` groups exist at once; freed groups are recycled.
  I.grp_cap = (int32_t)(imin(n, cap) + 1);
  I.slot_cap = (int32_t)(imin(n, cap) + 1);
  I.run_cap = (int32_t)(imin(n, cap) + 1);
  // Orca's PTs are bounded by its batch cap and the pool, not tfs
  I.ptiter_cap = (int32_t)(imin(n, I.base ? I.tfs + cap : I.tfs) + 2);
  I.adm_cap = (int32_t)(imin(n, cap + I.tfs) + 2);
  // Scratch bounds: selected GT members <= 2*general_cap (each
  // has a positive block demand or holds a region of >= 1 token); planner
  // regions/slots, compaction, promotion and deadline lists are bounded by
  // the general pool, the running set or tfs — never by the request count.
  I.sel_cap = (int32_t)(imin(n, 2 * I.general_cap) + 2);
  I.scr_cap = (int32_t)(imax(imax(I.general_cap, I.sel_cap), imax(imin(n, cap), I.tfs)) + 64);
  I.hist_cap = (int32_t)(imin(n, cap) + 2);
  I.rl_cap = (int32_t)(I.general_cap + 1);
  return ECONO_OK;
}

std::string format_error(const Inst& I, int* code) {
  char buf[512];
  *code = ECONO_ESIM;
  switch (I.error) {
    case ERR_ALLOC_FAIL:
      snprintf(buf, sizeof(buf), "exact allocation failed for scheduled request %d", I.err_id);
      break;
    case ERR_RESERVED_DRAW:
      snprintf(buf, sizeof(buf), "reserved pool draw failed for selected PT %d", I.err_id);
      break;
    case ERR_SLOT_OUTSIDE:
      snprintf(buf, sizeof(buf), "hosting slot outside the host's space");
      break;
    case ERR_STUCK:
      snprintf(buf, sizeof(buf),
               "simulation stuck: request %d can never be scheduled (demand exceeds what the "
               "configuration can free)", I.err_id);
      break;
    case ERR_RELEASE_UNKNOWN:
      snprintf(buf, sizeof(buf), "release: unknown id");
      break;
    case ERR_TABLE_OVERFLOW:
      snprintf(buf, sizeof(buf), "device table overflow (site %lld, request %d)", (long long)I.err_val, I.err_id);
      break;
    case ERR_INFEASIBLE_KVC:
      snprintf(buf, sizeof(buf), "request %d: KVC demand %lld exceeds usable capacity %lld", I.err_id,
               (long long)I.err_val, (long long)I.general_cap);
      break;
    case ERR_INFEASIBLE_RESERVE:
      snprintf(buf, sizeof(buf), "request %d: prompt does not fit the reserved pool (%lld tokens)", I.err_id,
               (long long)I.reserve_cap);
      break;
    case ERR_ARRIVAL_ORDER:
      *code = ECONO_ECONFIG;
      snprintf(buf, sizeof(buf), "trace arrival times must be nondecreasing");
      break;
    case ERR_FIRST_BLOCK:
      snprintf(buf, sizeof(buf), "first block grant failed unexpectedly");
      break;
    case ERR_ADMIT_BLOCK:
      snprintf(buf, sizeof(buf), "admission block grant failed unexpectedly");
      break;
    case ERR_EXACT_ADMIT:
      snprintf(buf, sizeof(buf), "exact allocation failed for admitted request %d", I.err_id);
      break;
    default:
      snprintf(buf, sizeof(buf), "unknown engine error %d", I.error);
  }
  return buf;
}

}  // namespace

// One instance's host-side bookkeeping.
struct HostInst {
  Inst desc;           // mirror of the device descriptor (device pointers)
  char* arena = nullptr;  // slice of econo_batch::block
  size_t arena_bytes = 0;
  EconoEvent* d_ev = nullptr;
  EconoSample* d_sm = nullptr;
  std::vector<EconoEvent> events;
  std::vector<EconoSample> samples;
  uint64_t seed = 1, pred_seed = 1;
  int32_t policy = 0;
  char* ckpt = nullptr;  // device copy of the arena (econo_batch_checkpoint)
  Inst ckpt_desc;
  std::vector<int64_t> ckpt_hist;
};

struct econo_batch {
  int device = 0;
  char* block = nullptr;  // every instance's arena, one allocation
  char* ckpt_block = nullptr;
  std::vector<HostInst> inst;
  Inst* d_insts = nullptr;
  // JCT keys for the percentile radix select (econo_batch_jct_prepare)
  uint64_t* d_keys = nullptr;
  int64_t* d_koff = nullptr;
  // bulk-ingest scratch (kept: a synchronous cudaFree of these GBs costs ~0.1 s)
  void* bulk_buf = nullptr;
  size_t bulk_bytes = 0;
  int64_t keys_total = 0;
  int64_t n_base = 0;  // baseline-policy instances (k_baseline_steps)
  bool fast = false;  // no recording and ordered PT queues in every econoserve instance: k_engine_steps_fast
  bool fast_oracle = false;  // ... and every one econoserve-full with the oracle predictor
  // trace staging buffers, kept until destroy: a cudaFree right after the
  // upload stalls for up to ~0.3 s next to a nearly full HBM (measured)
  void* stage[2] = {nullptr, nullptr};
  // small per-call device scratch (init descriptors, ingest plan, partial
  // sums, histogram passes), cached per slot and only ever grown: cudaFree /
  // cudaMalloc next to a nearly full HBM stall for tens to hundreds of ms
  void* scr[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t scr_bytes[6] = {0, 0, 0, 0, 0, 0};
  std::vector<uint64_t> h_keys;  // host build
#ifndef ECONO_HOSTSIM
  cudaStream_t stream = nullptr;
  // recorded after every launch on a caller stream; the handle's own stream
  // waits on it, so work the handle enqueues later (ingest plan, partial
  // sums, records) is ordered after the steps it reads
  cudaEvent_t launched = nullptr;
#endif
  std::vector<econo_engine*> views;
};

struct econo_engine {
  econo_batch* b;
  int32_t i;
  bool owns;
};

namespace {
enum { SCR_INIT = 0, SCR_PLAN, SCR_PART_OUT, SCR_PART_SLICES, SCR_HIST_PREFIX, SCR_HIST };
void dev_free(void* p);
int dev_alloc(void** p, size_t sz);
// Cached device scratch of at least `bytes` for one purpose (see econo_batch::scr).
void* batch_scratch(econo_batch* b, int slot, size_t bytes) {
  if (bytes > b->scr_bytes[slot]) {
    dev_free(b->scr[slot]);
    b->scr[slot] = nullptr;
    b->scr_bytes[slot] = 0;
    void* p;
    if (dev_alloc(&p, bytes)) return nullptr;
    b->scr[slot] = p;
    b->scr_bytes[slot] = bytes;
  }
  return b->scr[slot];
}
}  // namespace

namespace {

int cuda_check(char* err, size_t errlen, const char* what) {
#ifndef ECONO_HOSTSIM
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_err(err, errlen, "CUDA error in %s: %s", what, cudaGetErrorString(e));
    return ECONO_ECUDA;
  }
#else
  (void)err; (void)errlen; (void)what;
#endif
  return ECONO_OK;
}

int pull_descs(econo_batch* b) {
  std::vector<Inst> tmp(b->inst.size());
  if (dev_d2h(tmp.data(), b->d_insts, sizeof(Inst) * tmp.size())) return 1;
  for (size_t i = 0; i < tmp.size(); ++i) b->inst[i].desc = tmp[i];
  return 0;
}
int push_descs(econo_batch* b) {
  std::vector<Inst> tmp(b->inst.size());
  for (size_t i = 0; i < tmp.size(); ++i) tmp[i] = b->inst[i].desc;
  return dev_h2d(b->d_insts, tmp.data(), sizeof(Inst) * tmp.size());
}

int ensure_logs(HostInst& h, int64_t ev_cap, int64_t sm_cap) {
  Inst& I = h.desc;
  if (I.record_events && ev_cap > I.ev_cap) {
    dev_free(h.d_ev);
    void* p;
    if (dev_alloc(&p, sizeof(EconoEvent) * (size_t)ev_cap)) return 1;
    h.d_ev = (EconoEvent*)p;
    I.ev = h.d_ev;
    I.ev_cap = ev_cap;
  }
  if (I.record_samples && sm_cap > I.sm_cap) {
    dev_free(h.d_sm);
    void* p;
    if (dev_alloc(&p, sizeof(EconoSample) * (size_t)sm_cap)) return 1;
    h.d_sm = (EconoSample*)p;
    I.sm = h.d_sm;
    I.sm_cap = sm_cap;
  }
  return 0;
}

// Copies logged events/samples to the host vectors and empties the device logs.
int drain(HostInst& h) {
  Inst& I = h.desc;
  if (I.record_events && I.ev_n > 0) {
    const int64_t k = imin(I.ev_n, I.ev_cap);
    const size_t old = h.events.size();
    h.events.resize(old + (size_t)k);
    if (dev_d2h(h.events.data() + old, h.d_ev, sizeof(EconoEvent) * (size_t)k)) return 1;
    I.ev_n = 0;
  }
  if (I.record_samples && I.sm_n > 0) {
    const int64_t k = imin(I.sm_n, I.sm_cap);
    const size_t old = h.samples.size();
    h.samples.resize(old + (size_t)k);
    if (dev_d2h(h.samples.data() + old, h.d_sm, sizeof(EconoSample) * (size_t)k)) return 1;
    I.sm_n = 0;
  }
  return 0;
}

void launch_steps(econo_batch* b, int64_t max_steps, void* stream, int64_t slice_ns = 0) {
#ifdef ECONO_HOSTSIM
  (void)stream;
  (void)slice_ns;  // the host build has no device clock: max_steps only
  for (auto& h : b->inst) {
    if (h.desc.base) engine_steps<true>(h.desc, steps_for(h.desc, max_steps));
    else engine_steps<false>(h.desc, steps_for(h.desc, max_steps));
  }
  push_descs(b);
#else
  cudaStream_t s = stream ? (cudaStream_t)stream : b->stream;
  if (b->n_base < (int64_t)b->inst.size()) {
    if (b->fast_oracle) launch_engine_steps_fast_oracle(b->d_insts, (unsigned)b->inst.size(), max_steps, slice_ns, s);
    else if (b->fast) launch_engine_steps_fast(b->d_insts, (unsigned)b->inst.size(), max_steps, slice_ns, s);
    else k_engine_steps<<<(unsigned)b->inst.size(), 32, 0, s>>>(b->d_insts, max_steps, slice_ns);
  }
  if (b->n_base > 0) k_baseline_steps<<<(unsigned)b->inst.size(), 32, 0, s>>>(b->d_insts, max_steps, slice_ns);
  if (s != b->stream) {  // order the handle's stream after these launches
    cudaEventRecord(b->launched, s);
    cudaStreamWaitEvent(b->stream, b->launched, 0);
  }
#endif
}

int sync_batch(econo_batch* b, char* err, size_t errlen) {
#ifndef ECONO_HOSTSIM
  if (cudaStreamSynchronize(b->stream) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    set_err(err, errlen, "CUDA error: %s", cudaGetErrorString(cudaGetLastError()));
    return ECONO_ECUDA;
  }
#endif
  if (pull_descs(b)) return set_err(err, errlen, "device copy failed"), ECONO_ECUDA;
  return ECONO_OK;
}

// ---- JCT radix select (host driver; kernels k_jct_keys / k_jct_hist) ------
const int kDigitBits[6] = {11, 11, 11, 11, 11, 9};

int jct_prepare(econo_batch* b, char* err, size_t errlen) {
  int rc = sync_batch(b, err, errlen);
  if (rc) return rc;
  const int32_t ni = (int32_t)b->inst.size();
  std::vector<int64_t> off((size_t)ni + 1, 0);
  for (int32_t i = 0; i < ni; ++i) off[(size_t)i + 1] = off[(size_t)i] + b->inst[(size_t)i].desc.n;
  const int64_t total = off[(size_t)ni];
#ifdef ECONO_HOSTSIM
  b->h_keys.resize((size_t)total);
  for (int32_t i = 0; i < ni; ++i)
    for (int64_t k = 0; k < b->inst[(size_t)i].desc.n; ++k)
      b->h_keys[(size_t)(off[(size_t)i] + k)] = jct_key(b->inst[(size_t)i].desc, k);
#else
  if (total != b->keys_total) {
    // the burst-ingest scratch is not needed once the run reports: give its
    // HBM to the keys (a later ingest re-allocates it)
    dev_free(b->bulk_buf);
    b->bulk_buf = nullptr;
    b->bulk_bytes = 0;
    dev_free(b->d_keys);
    dev_free(b->d_koff);
    b->d_keys = nullptr;
    b->d_koff = nullptr;
    void *pk = nullptr, *po;
    if (dev_alloc(&po, sizeof(int64_t) * off.size())) return set_err(err, errlen, "key allocation failed"), ECONO_ECUDA;
    // 8 B per request when HBM allows; a batch that fills the GPU derives each
    // key from the request's fields in every histogram pass instead
    if (getenv("ECONO_JCT_NO_KEYS") || cudaMalloc(&pk, sizeof(uint64_t) * (size_t)total) != cudaSuccess) {
      (void)cudaGetLastError();
      pk = nullptr;
    }
    b->d_keys = (uint64_t*)pk;
    b->d_koff = (int64_t*)po;
    if (dev_h2d(b->d_koff, off.data(), sizeof(int64_t) * off.size())) return set_err(err, errlen, "copy failed"), ECONO_ECUDA;
  }
  int64_t nmax = 1;
  for (auto& h : b->inst) nmax = imax(nmax, h.desc.n);
  const unsigned gx = (unsigned)imax(1, imin((nmax + 255) / 256, (148 * 8 + ni - 1) / ni));
  if (b->d_keys) k_jct_keys<<<dim3(gx, (unsigned)ni), 256, 0, b->stream>>>(b->d_insts, b->d_koff, b->d_keys);
  rc = sync_batch(b, err, errlen);
  if (rc) return rc;
#endif
  b->keys_total = total;
  return cuda_check(err, errlen, "k_jct_keys");
}

// One pass: hist[g][t][2^dbits] for groups g (instances, or one global group).
int jct_hist(econo_batch* b, int per_instance, int nt, const uint64_t* prefixes, int consumed, int dbits,
             uint64_t* hist, char* err, size_t errlen) {
  const int32_t ni = (int32_t)b->inst.size();
  const int groups = per_instance ? ni : 1;
  const size_t bins = (size_t)1 << dbits;
  if (nt < 1 || nt > 8 || dbits < 1 || dbits > 11 || consumed < 0 || consumed + dbits > 64)
    return set_err(err, errlen, "jct_hist: bad arguments"), ECONO_ECONFIG;
  if (b->keys_total <= 0) return set_err(err, errlen, "jct keys not prepared"), ECONO_ECONFIG;
#ifdef ECONO_HOSTSIM
  std::fill(hist, hist + (size_t)groups * nt * bins, 0);
  int64_t o = 0;
  for (int32_t i = 0; i < ni; ++i) {
    const int64_t n = b->inst[(size_t)i].desc.n;
    const int g = per_instance ? i : 0;
    for (int64_t k = 0; k < n; ++k) {
      const uint64_t key = b->h_keys[(size_t)(o + k)];
      for (int t = 0; t < nt; ++t)
        if (key_matches(key, prefixes[(size_t)g * nt + t], consumed))
          hist[((size_t)g * nt + t) * bins + key_digit(key, consumed, dbits)]++;
    }
    o += n;
  }
  return ECONO_OK;
#else
  // identical prefixes (e.g. every target in the first pass) share one histogram
  std::vector<uint64_t> up;
  std::vector<int> map_t((size_t)groups * nt);
  int nu = 0;
  for (int g = 0; g < groups; ++g) {
    std::vector<uint64_t> u;
    for (int t = 0; t < nt; ++t) {
      const uint64_t pfx = prefixes[(size_t)g * nt + t];
      size_t j = 0;
      while (j < u.size() && u[j] != pfx) ++j;
      if (j == u.size()) u.push_back(pfx);
      map_t[(size_t)g * nt + t] = (int)j;
    }
    nu = std::max(nu, (int)u.size());
  }
  up.assign((size_t)groups * nu, 0);
  for (int g = 0; g < groups; ++g)
    for (int t = 0; t < nt; ++t) up[(size_t)g * nu + map_t[(size_t)g * nt + t]] = prefixes[(size_t)g * nt + t];
  static bool smem_set = false;
  if (!smem_set) {
    cudaFuncSetAttribute(k_jct_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2048 * 4);
    smem_set = true;
  }
  const size_t hbytes = sizeof(uint64_t) * (size_t)groups * nu * bins;
  void* dp = batch_scratch(b, SCR_HIST_PREFIX, sizeof(uint64_t) * (size_t)groups * nu);
  void* dh = batch_scratch(b, SCR_HIST, hbytes);
  if (!dp || !dh) return set_err(err, errlen, "allocation failed"), ECONO_ECUDA;
  cudaMemsetAsync(dh, 0, hbytes, b->stream);  // the passes accumulate with atomics
  dev_h2d(dp, up.data(), sizeof(uint64_t) * (size_t)groups * nu);
  int64_t nmax = 1;
  for (auto& h : b->inst) nmax = imax(nmax, h.desc.n);
  const unsigned gx = (unsigned)imax(1, imin((nmax + 511) / 512, (148 * 16 + ni - 1) / ni));
  k_jct_hist<<<dim3(gx, (unsigned)ni), 256, sizeof(uint32_t) * nu * bins, b->stream>>>(
      b->d_insts, b->d_koff, b->d_keys, per_instance, nu, (const uint64_t*)dp, consumed, dbits,
      (unsigned long long*)dh);
  int rc = sync_batch(b, err, errlen);
  if (!rc) rc = cuda_check(err, errlen, "k_jct_hist");
  std::vector<uint64_t> hu((size_t)groups * nu * bins);
  if (!rc && dev_d2h(hu.data(), dh, hbytes)) {
    set_err(err, errlen, "copy failed");
    rc = ECONO_ECUDA;
  }
  if (!rc)
    for (int g = 0; g < groups; ++g)
      for (int t = 0; t < nt; ++t)
        memcpy(hist + ((size_t)g * nt + t) * bins, hu.data() + ((size_t)g * nu + map_t[(size_t)g * nt + t]) * bins,
               sizeof(uint64_t) * bins);
  return rc;
#endif
}

// Exact k-th smallest keys: ranks[g][t] (0-based) -> keys[g][t].
int jct_select(econo_batch* b, int per_instance, int nt, const uint64_t* ranks, uint64_t* keys, char* err,
               size_t errlen) {
  const int groups = per_instance ? (int)b->inst.size() : 1;
  std::vector<uint64_t> pre((size_t)groups * nt, 0), rk(ranks, ranks + (size_t)groups * nt);
  int consumed = 0;
  for (int pass = 0; pass < 6; ++pass) {
    const int db = kDigitBits[pass];
    const size_t bins = (size_t)1 << db;
    std::vector<uint64_t> h((size_t)groups * nt * bins);
    int rc = jct_hist(b, per_instance, nt, pre.data(), consumed, db, h.data(), err, errlen);
    if (rc) return rc;
    for (size_t gt = 0; gt < (size_t)groups * nt; ++gt) {
      uint64_t cum = 0;
      size_t d = 0;
      for (; d < bins; ++d) {
        const uint64_t c = h[gt * bins + d];
        if (rk[gt] < cum + c) break;
        cum += c;
      }
      if (d == bins) return set_err(err, errlen, "radix select: rank beyond the key count"), ECONO_ESIM;
      rk[gt] -= cum;
      pre[gt] = (pre[gt] << db) | (uint64_t)d;
    }
    consumed += db;
  }
  std::copy(pre.begin(), pre.end(), keys);
  return ECONO_OK;
}

// percentile() (metrics.hpp:81-89) per instance from exact order statistics.
int jct_percentiles(econo_batch* b, const double* q, int nq, double* out, char* err, size_t errlen) {
  if (nq < 1 || nq > 4) return set_err(err, errlen, "1..4 quantiles per call"), ECONO_ECONFIG;
  int rc = jct_prepare(b, err, errlen);
  if (rc) return rc;
  const int32_t ni = (int32_t)b->inst.size();
  const int nt = 2 * nq;
  std::vector<uint64_t> ranks((size_t)ni * nt), keys((size_t)ni * nt);
  std::vector<double> frac((size_t)ni * nq);
  for (int32_t i = 0; i < ni; ++i) {
    const int64_t n = b->inst[(size_t)i].desc.n;
    for (int k = 0; k < nq; ++k) {
      const double rank = q[k] * (double)(n - 1);
      const uint64_t lo = (uint64_t)rank;
      const uint64_t hi = std::min<uint64_t>(lo + 1, (uint64_t)(n - 1));
      frac[(size_t)i * nq + k] = rank - (double)lo;
      ranks[(size_t)i * nt + 2 * k] = lo;
      ranks[(size_t)i * nt + 2 * k + 1] = hi;
    }
  }
  rc = jct_select(b, 1, nt, ranks.data(), keys.data(), err, errlen);
  if (rc) return rc;
  for (int32_t i = 0; i < ni; ++i)
    for (int k = 0; k < nq; ++k) {
      const double vlo = key_double(keys[(size_t)i * nt + 2 * k]), vhi = key_double(keys[(size_t)i * nt + 2 * k + 1]);
      const double f = frac[(size_t)i * nq + k];
      out[(size_t)i * nq + k] = vlo * (1.0 - f) + vhi * f;
    }
  return ECONO_OK;
}

}  // namespace

extern "C" {

void econo_default_options(EconoOptions* o) {
  memset(o, 0, sizeof(*o));
  o->policy = ECONO_POLICY_ECONO_FULL;
  o->batch_size_cap = 8;
  o->tfs = 2048;
  o->chunk_size = 512;
  o->padding_ratio = 0.10;
  o->reserved_fraction = 0.03;
  o->buffer_ratio = 0.15;
  o->t_base = 0.005;
  o->t_token = 1e-4;
  o->t_token_over = -1.0;
  o->cost_tfs = 2048;
  o->preempt_offload_penalty = 0.30;
  o->preempt_free_penalty = 0.06;
  o->reserve_penalty = 0.004;
  o->sched_cost_per_exam = 2e-5;
  o->swap_stall = 0.088;
  o->pred_model = ECONO_PRED_ORACLE;
  o->pred_accuracy = 1.0;
  o->pred_tolerance = 0.1;
  o->pred_quantum = 1;
  o->pred_seed = 1;
  o->n_deadline_bounds = 3;
  o->deadline_bounds[0] = 0.2;
  o->deadline_bounds[1] = 0.5;
  o->deadline_bounds[2] = 2.0;
  o->n_kvc_bounds = 4;
  o->n_length_bounds = 4;
  for (int i = 0; i < 4; ++i) o->kvc_bounds[i] = o->length_bounds[i] = 128 * (i + 1);
  o->kvc_capacity = 32768;
  o->kvc_block_size = 32;
  o->slo_scale = 2.0;
  o->seed = 1;
  o->record_events = 1;
  o->record_samples = 1;
}

void econo_batch_destroy(econo_batch* b) {
  if (!b) return;
  dev_free(b->block);
  dev_free(b->ckpt_block);
  for (auto& h : b->inst) {
    dev_free(h.d_ev);
    dev_free(h.d_sm);
  }
  dev_free(b->d_insts);
  dev_free(b->d_keys);
  dev_free(b->d_koff);
  dev_free(b->bulk_buf);
  dev_free(b->stage[0]);
  dev_free(b->stage[1]);
  for (auto* p : b->scr) dev_free(p);
  for (auto* v : b->views) delete v;
#ifndef ECONO_HOSTSIM
  if (b->launched) cudaEventDestroy(b->launched);
  if (b->stream) cudaStreamDestroy(b->stream);
#endif
  delete b;
}

int64_t econo_instance_bytes(const EconoTraceRecord* trace, int64_t n, const EconoOptions* opt, char* err,
                             size_t errlen) {
  int rc = validate(opt, n, err, errlen);
  if (rc) return -rc;
  Inst I;
  rc = configure(I, opt, trace, n, err, errlen);
  if (rc) return -rc;
  size_t bytes = 0;
  layout(I, nullptr, &bytes);
  return (int64_t)((bytes + 4095) & ~size_t(4095));
}

// traces (records) or soa (arrays): exactly one is non-null.
static int batch_create(const EconoTraceRecord* const* traces, const EconoTraceSoA* soa, const int64_t* ns,
                        int32_t n_inst, const EconoOptions* opts, int device, econo_batch** out, char* err,
                        size_t errlen) {
  *out = nullptr;
  if (n_inst < 1) return set_err(err, errlen, "n_inst must be >= 1"), ECONO_ECONFIG;
  for (int32_t i = 0; i < n_inst; ++i) {
    const int rc = validate(&opts[i], ns[i], err, errlen);
    if (rc) return rc;
  }
#ifndef ECONO_HOSTSIM
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device || device < 0)
    return set_err(err, errlen, "no CUDA device %d available (the EconoServe B200 path has no CPU fallback)", device),
           ECONO_ECUDA;
  if (cudaSetDevice(device) != cudaSuccess)
    return set_err(err, errlen, "cudaSetDevice(%d) failed", device), ECONO_ECUDA;
#endif
  econo_batch* b = new econo_batch();
  b->device = device;
  b->inst.resize((size_t)n_inst);
#ifndef ECONO_HOSTSIM
  cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&b->launched, cudaEventDisableTiming);
#endif
  std::vector<const EconoTraceRecord*> d_traces((size_t)n_inst);
  std::vector<uint64_t> seeds(2 * (size_t)n_inst);
  const auto t_alloc0 = std::chrono::steady_clock::now();
  {  // per-instance configuration scans its trace (lengths, max prompt): threads
    std::vector<int> rcs((size_t)n_inst, ECONO_OK);
    std::vector<std::string> msgs((size_t)n_inst);
    const int nt = (int)std::max<unsigned>(1, std::min<unsigned>(std::thread::hardware_concurrency(), 32));
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        char e2[512];
        for (int32_t i = t; i < n_inst; i += nt) {
#ifdef ECONO_HOSTSIM
          rcs[(size_t)i] = configure(b->inst[(size_t)i].desc, &opts[i], traces[i], ns[i], e2, sizeof(e2));
#else  // the record checks run on the device (k_init_soa)
          if (soa && opts[i].policy == ECONO_POLICY_ORCA && opts[i].max_output_len <= 0) {
            // Orca's derived max_output_len is the one host scan configure needs: records for it
            std::vector<EconoTraceRecord> rec((size_t)ns[i]);
            for (int64_t k = 0; k < ns[i]; ++k)
              rec[(size_t)k] = EconoTraceRecord{soa[i].arrival_time[k], soa[i].prompt_len[k], soa[i].true_rl[k]};
            rcs[(size_t)i] = configure(b->inst[(size_t)i].desc, &opts[i], rec.data(), ns[i], e2, sizeof(e2), false);
          } else {
            rcs[(size_t)i] = configure(b->inst[(size_t)i].desc, &opts[i], soa ? nullptr : traces[i], ns[i], e2,
                                       sizeof(e2), false);
          }
#endif
          if (rcs[(size_t)i]) msgs[(size_t)i] = e2;
        }
      });
    for (auto& x : th) x.join();
    for (int32_t i = 0; i < n_inst; ++i)
      if (rcs[(size_t)i]) {
        set_err(err, errlen, "%s", msgs[(size_t)i].c_str());
        econo_batch_destroy(b);
        return rcs[(size_t)i];
      }
  }
  b->fast = true;
  b->fast_oracle = true;
  for (int32_t i = 0; i < n_inst; ++i) {
    HostInst& h = b->inst[(size_t)i];
    h.seed = opts[i].seed;
    h.pred_seed = opts[i].pred_seed;
    h.policy = opts[i].policy;
    b->n_base += h.desc.base;
    if (!h.desc.base && (h.desc.record_events || h.desc.record_samples || !h.desc.ordered)) b->fast = false;
    if (!h.desc.base && (!h.desc.full || h.desc.pred_model != ECONO_PRED_ORACLE)) b->fast_oracle = false;
    size_t bytes = 0;
    layout(h.desc, nullptr, &bytes);
    h.arena_bytes = (bytes + 4095) & ~size_t(4095);
    seeds[2 * i] = opts[i].seed;
    seeds[2 * i + 1] = opts[i].pred_seed;
  }
  b->fast_oracle = b->fast_oracle && b->fast;
#ifndef ECONO_HOSTSIM
  {  // reserve the burst-ingest scratch now, before the arenas fill the GPU:
     // a late cudaMalloc next to a nearly full HBM is slow (~0.5 s measured)
    int64_t keys = 0, kmax = 0, jobs = 0;
    for (auto& h : b->inst)
      if (h.desc.ordered && !h.desc.record_events && h.desc.n >= 32768) {
        keys += h.desc.n;
        kmax = imax(kmax, h.desc.n);
        ++jobs;
      }
    if (jobs > 0) {
      const int64_t g = imin(keys, imax(bulk_budget(), kmax));  // keys in one group at most
      const size_t kb = (4 * (size_t)g + 255) & ~(size_t)255;
      const size_t hb = (4 * 256 * (size_t)(g / kBulkTile + jobs) + 255) & ~(size_t)255;
      const size_t need = 4 * kb + hb + sizeof(BulkJob) * (size_t)jobs;
      if (cudaMalloc(&b->bulk_buf, need) == cudaSuccess) b->bulk_bytes = need;
      else { (void)cudaGetLastError(); b->bulk_buf = nullptr; }
    }
  }
#endif
  {
    size_t total = 0;
    for (auto& h : b->inst) total += h.arena_bytes;
    void* blk;
    if (dev_alloc(&blk, total)) {
      econo_batch_destroy(b);
      return set_err(err, errlen, "device allocation of %zu bytes failed", total), ECONO_ECUDA;
    }
    b->block = (char*)blk;
    size_t off = 0;
    for (auto& h : b->inst) {
      h.arena = b->block + off;
      off += h.arena_bytes;
      size_t bytes = 0;
      layout(h.desc, h.arena, &bytes);
    }
  }
  for (int32_t i = 0; i < n_inst; ++i) {
    HostInst& h = b->inst[(size_t)i];
    const int64_t n = ns[i];
    if (ensure_logs(h, h.desc.record_events ? 4 * n + 4096 : 0, h.desc.record_samples ? 2 * n + 4096 : 0)) {
      econo_batch_destroy(b);
      return set_err(err, errlen, "device allocation of the event log failed"), ECONO_ECUDA;
    }
  }
  if (getenv("ECONO_VERBOSE"))
    fprintf(stderr, "[econo] create: arenas %.1f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_alloc0).count());
  void* di;
  if (dev_alloc(&di, sizeof(Inst) * (size_t)n_inst)) {
    econo_batch_destroy(b);
    return set_err(err, errlen, "device allocation failed"), ECONO_ECUDA;
  }
  b->d_insts = (Inst*)di;
  push_descs(b);
#ifdef ECONO_HOSTSIM
  for (int32_t i = 0; i < n_inst; ++i) {
    Inst& I = b->inst[(size_t)i].desc;
    double* arr = const_cast<double*>(I.arrival.get());
    int32_t* pr = const_cast<int32_t*>(I.prompt.get());
    int32_t* rl = const_cast<int32_t*>(I.true_rl.get());
    for (int64_t k = 0; k < I.n; ++k) {
      arr[k] = traces[i][k].arrival_time;
      pr[k] = (int32_t)traces[i][k].prompt_len;
      rl[k] = (int32_t)traces[i][k].true_rl;
    }
    mt_seed(I.mt, I.mt_i, seeds[2 * i]);
    mt_seed(I.pmt, I.pmt_i, seeds[2 * i + 1]);
    int64_t bad_order = I.n, psum = 0;
    for (int64_t k = 0; k < I.n; ++k) {
      bool ob, lb;
      int64_t p;
      init_soa_one(I, traces[i], k, &ob, &p, &lb);
      psum += p;
      if (ob && k < bad_order) bad_order = k;
    }
    if (bad_order < I.n) {
      I.error = ERR_ARRIVAL_ORDER;
      I.err_id = (int32_t)bad_order;
      continue;
    }
    init_calibrate(I, psum);
    init_predict_sequential(I);
    int64_t bad = I.n;
    const int64_t ext = init_table_extent(I);
    for (int64_t k = 0; k < ext; ++k) {
      if (k < I.n && init_req_one(I, k) && k < bad) bad = k;
      init_tables_one(I, k);
    }
    init_finish(I, bad);
  }
  push_descs(b);
#else
  {
    // Stage every trace in one device buffer (AoS; the init kernels convert
    // it to SoA). Host pages are pinned in place for the copy when possible.
    const bool verbose = getenv("ECONO_VERBOSE") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b2) { return std::chrono::duration<double, std::milli>(b2 - a).count(); };
    const auto t0 = now();
    // Traces are staged through two bounded device buffers (double-buffered:
    // the copy of one group of instances overlaps the AoS->SoA conversion of
    // the previous group), so staging never costs more than 2 x chunk bytes
    // of HBM however many instances the batch holds. Pinned host buffers copy
    // at full link speed; pageable ones go through the driver's bounce buffer.
    // Arrays (econo_batch_create_soa) are copied straight into each
    // instance's SoA: 16 B per request, no staging, checks only.
    const size_t rec = soa ? sizeof(double) + 2 * sizeof(int32_t) : sizeof(EconoTraceRecord);
    size_t largest = 0, total = 0;
    for (int32_t i = 0; i < n_inst; ++i) {
      largest = std::max(largest, rec * (size_t)ns[i]);
      total += rec * (size_t)ns[i];
    }
    // copy/check pipeline granularity: 256 MB staging chunks for records; 1 GB
    // instance groups for columns (no staging: fewer, larger check launches)
    const size_t chunk = std::min(total, std::max(largest, (size_t)(soa ? 1024 : 256) << 20));
    const int nbuf = soa ? 0 : (total > chunk ? 2 : 1);
    void* stage[2] = {nullptr, nullptr};
    for (int k = 0; k < nbuf; ++k)
      if (dev_alloc(&stage[k], chunk)) {
        for (int j = 0; j < k; ++j) dev_free(stage[j]);
        econo_batch_destroy(b);
        return set_err(err, errlen, "device trace staging allocation failed"), ECONO_ECUDA;
      }
    // instance groups [g0, g1) that fit one chunk
    std::vector<std::pair<int32_t, int32_t>> groups;
    for (int32_t i = 0; i < n_inst;) {
      int32_t j = i;
      size_t used = 0;
      while (j < n_inst && used + rec * (size_t)ns[j] <= chunk) used += rec * (size_t)ns[j++];
      groups.emplace_back(i, j);
      i = j;
    }
    for (size_t g = 0; g < groups.size() && !soa; ++g) {
      size_t o = 0;
      for (int32_t i = groups[g].first; i < groups[g].second; ++i) {
        d_traces[(size_t)i] = (const EconoTraceRecord*)((char*)stage[g % nbuf] + o);
        o += sizeof(EconoTraceRecord) * (size_t)ns[i];
      }
    }
    char* dinit = (char*)batch_scratch(b, SCR_INIT, 56 * (size_t)n_inst + 512);
    if (!dinit) {
      for (int k = 0; k < nbuf; ++k) dev_free(stage[k]);
      econo_batch_destroy(b);
      return set_err(err, errlen, "device allocation failed"), ECONO_ECUDA;
    }
    void* dt = dinit;
    void* ds = dinit + ((8 * (size_t)n_inst + 255) & ~(size_t)255);
    void* dsc = (char*)ds + ((16 * (size_t)n_inst + 255) & ~(size_t)255);
    dev_h2d(dt, d_traces.data(), sizeof(void*) * (size_t)n_inst);
    dev_h2d(ds, seeds.data(), sizeof(uint64_t) * 2 * (size_t)n_inst);
    std::vector<unsigned long long> sc0(4 * (size_t)n_inst, 0);
    for (int32_t i = 0; i < n_inst; ++i) sc0[4 * (size_t)i] = sc0[4 * (size_t)i + 2] = sc0[4 * (size_t)i + 3] = ~0ULL;
    dev_h2d(dsc, sc0.data(), sizeof(unsigned long long) * sc0.size());
    int64_t nmax = 0, emax = 0;
    for (auto& h : b->inst) {
      nmax = imax(nmax, h.desc.n);
      emax = imax(emax, h.desc.n + h.desc.general_cap + (int64_t)h.desc.nbuckets * (h.desc.pmax + 1) + 64);
    }
    cudaStream_t cs;
    cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    cudaEvent_t copied[2], converted[2];
    for (int k = 0; k < 2; ++k) {
      cudaEventCreateWithFlags(&copied[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&converted[k], cudaEventDisableTiming);
    }
    for (size_t g = 0; g < groups.size(); ++g) {
      const int k = (int)(g % 2);
      if (soa) {
        for (int32_t i = groups[g].first; i < groups[g].second; ++i) {
          const Inst& D = b->inst[(size_t)i].desc;
          const size_t m = (size_t)ns[i];
          cudaMemcpyAsync(const_cast<double*>(D.arrival.p), soa[i].arrival_time, sizeof(double) * m,
                          cudaMemcpyHostToDevice, cs);
          cudaMemcpyAsync(const_cast<int32_t*>(D.prompt.p), soa[i].prompt_len, sizeof(int32_t) * m,
                          cudaMemcpyHostToDevice, cs);
          cudaMemcpyAsync(const_cast<int32_t*>(D.true_rl.p), soa[i].true_rl, sizeof(int32_t) * m,
                          cudaMemcpyHostToDevice, cs);
        }
      } else {
        if (g >= (size_t)nbuf) cudaStreamWaitEvent(cs, converted[k % nbuf], 0);  // buffer free again
        for (int32_t i = groups[g].first; i < groups[g].second; ++i)
          cudaMemcpyAsync(const_cast<EconoTraceRecord*>(d_traces[(size_t)i]), traces[i],
                          sizeof(EconoTraceRecord) * (size_t)ns[i], cudaMemcpyHostToDevice, cs);
      }
      cudaEventRecord(copied[k], cs);
      cudaStreamWaitEvent(b->stream, copied[k], 0);
      const int32_t cnt = groups[g].second - groups[g].first;
      const unsigned gx = (unsigned)imin(imax(1, (nmax + 255) / 256), 1184 / imax(1, cnt / 8 + 1) + 1);
      if (soa)
        k_init_soa<true><<<dim3(gx, (unsigned)cnt), 256, 0, b->stream>>>(
            b->d_insts, (const EconoTraceRecord* const*)dt, (unsigned long long*)dsc, groups[g].first);
      else
        k_init_soa<false><<<dim3(gx, (unsigned)cnt), 256, 0, b->stream>>>(
            b->d_insts, (const EconoTraceRecord* const*)dt, (unsigned long long*)dsc, groups[g].first);
      cudaEventRecord(converted[k], b->stream);
    }
    cudaStreamSynchronize(b->stream);
    {  // per-record length checks from k_init_soa, in instance order
      std::vector<unsigned long long> sc1(sc0.size());
      dev_d2h(sc1.data(), dsc, sizeof(unsigned long long) * sc1.size());
      for (int32_t i = 0; i < n_inst; ++i)
        if (sc1[4 * (size_t)i + 3] < (unsigned long long)ns[i]) {
          set_err(err, errlen, "request %lld: prompt_len and response_len must be in [1, 2^30)",
                  (long long)sc1[4 * (size_t)i + 3]);
          for (int k = 0; k < 2; ++k) {
            cudaEventDestroy(copied[k]);
            cudaEventDestroy(converted[k]);
          }
          cudaStreamDestroy(cs);
          for (int k = 0; k < nbuf; ++k) dev_free(stage[k]);
          econo_batch_destroy(b);
          return ECONO_ECONFIG;
        }
    }
    const auto t1 = now();
    for (int k = 0; k < 2; ++k) {
      cudaEventDestroy(copied[k]);
      cudaEventDestroy(converted[k]);
    }
    cudaStreamDestroy(cs);
    b->stage[0] = stage[0];
    b->stage[1] = stage[1];
    const unsigned gx2 = (unsigned)imin(imax(1, (emax + 255) / 256), 1184 / imax(1, n_inst / 8 + 1) + 1);
    k_init_scalar<<<(unsigned)n_inst, 32, 0, b->stream>>>(b->d_insts, (const uint64_t*)ds,
                                                          (const unsigned long long*)dsc);
    k_init_req<<<dim3(gx2, (unsigned)n_inst), 256, 0, b->stream>>>(b->d_insts, (unsigned long long*)dsc);
    k_init_finish<<<(unsigned)n_inst, 32, 0, b->stream>>>(b->d_insts, (const unsigned long long*)dsc);
    const int rc = sync_batch(b, err, errlen);
    const auto t2 = now();
    if (verbose)
      fprintf(stderr, "[econo] create: trace upload + SoA conversion %.1f ms (%zu MB), init kernels %.1f ms\n", ms(t0, t1),
              total >> 20, ms(t1, t2));
    if (rc) { econo_batch_destroy(b); return rc; }
  }
#endif
  if (pull_descs(b)) { econo_batch_destroy(b); return set_err(err, errlen, "device copy failed"), ECONO_ECUDA; }
  for (auto& h : b->inst) {
    if (h.desc.error) {
      int code;
      std::string m = format_error(h.desc, &code);
      set_err(err, errlen, "%s", m.c_str());
      econo_batch_destroy(b);
      return code;
    }
  }
  *out = b;
  return ECONO_OK;
}

int econo_batch_create(const EconoTraceRecord* const* traces, const int64_t* ns, int32_t n_inst,
                       const EconoOptions* opts, int device, econo_batch** out, char* err, size_t errlen) {
  return batch_create(traces, nullptr, ns, n_inst, opts, device, out, err, errlen);
}

int econo_batch_create_soa(const EconoTraceSoA* traces, const int64_t* ns, int32_t n_inst, const EconoOptions* opts,
                           int device, econo_batch** out, char* err, size_t errlen) {
#ifdef ECONO_HOSTSIM  // the host build takes records: convert
  std::vector<std::vector<EconoTraceRecord>> recs((size_t)(n_inst > 0 ? n_inst : 0));
  std::vector<const EconoTraceRecord*> ptrs(recs.size());
  for (int32_t i = 0; i < n_inst; ++i) {
    recs[(size_t)i].resize((size_t)(ns[i] > 0 ? ns[i] : 0));
    for (int64_t k = 0; k < ns[i]; ++k)
      recs[(size_t)i][(size_t)k] = EconoTraceRecord{traces[i].arrival_time[k], traces[i].prompt_len[k],
                                                    traces[i].true_rl[k]};
    ptrs[(size_t)i] = recs[(size_t)i].data();
  }
  return batch_create(ptrs.data(), nullptr, ns, n_inst, opts, device, out, err, errlen);
#else
  return batch_create(nullptr, traces, ns, n_inst, opts, device, out, err, errlen);
#endif
}

int econo_batch_launch(econo_batch* b, int64_t max_steps, void* stream) {
  launch_steps(b, max_steps, stream);
  return ECONO_OK;
}

int econo_batch_launch_slice(econo_batch* b, int64_t max_steps, int64_t slice_ns, void* stream) {
  launch_steps(b, max_steps, stream, slice_ns > 0 ? slice_ns : 0);
  return ECONO_OK;
}

int econo_batch_launch_to(econo_batch* b, int64_t target_steps, int64_t slice_ns, void* stream) {
  if (target_steps < 0) return ECONO_ECONFIG;
  launch_steps(b, -target_steps, stream, slice_ns > 0 ? slice_ns : 0);
  return ECONO_OK;
}


int econo_batch_sync(econo_batch* b, char* err, size_t errlen) {
  int rc = sync_batch(b, err, errlen);
  if (rc) return rc;
  return cuda_check(err, errlen, "econo_batch_sync");
}

int econo_batch_scalars(econo_batch* b, EconoScalars* out) {
  for (size_t i = 0; i < b->inst.size(); ++i) {
    const Inst& I = b->inst[i].desc;
    EconoScalars& s = out[i];
    memset(&s, 0, sizeof(s));
    s.clock = I.clock;
    s.iter = I.iter;
    s.completed = I.completed;
    s.steps = I.steps;
    s.executed_iters = I.executed;
    s.hosted_slots_created = I.hosted_total;
    s.hosted_overruns = I.hosted_overruns;
    s.calibrated_prefill_time = I.t_p;
    s.calibrated_decode_time = I.t_g;
    s.pt_dispatched = I.pt_dispatched;
    s.gt_scheduled = I.gt_scheduled;
    s.pt_queue_len = I.pt_count;
    s.gt_queue_groups = I.G;
    s.running = I.R;
    s.arrived = I.arrival_cursor;
    s.done = I.completed >= I.n;
    s.error = I.error ? ECONO_ESIM : 0;
    s.quiet_steps = I.quiet_steps;
    s.quiet_spans = I.quiet_spans;
  }
  return ECONO_OK;
}

int econo_batch_engine(econo_batch* b, int32_t i, econo_engine** out) {
  if (i < 0 || i >= (int32_t)b->inst.size()) return ECONO_ECONFIG;
  econo_engine* e = new econo_engine{b, i, false};
  b->views.push_back(e);
  *out = e;
  return ECONO_OK;
}

int econo_batch_partials(econo_batch* b, double* out, char* err, size_t errlen) {
  const size_t bytes = sizeof(double) * ECONO_PARTIAL_WORDS * b->inst.size();
#ifdef ECONO_HOSTSIM
  for (size_t i = 0; i < b->inst.size(); ++i) engine_partials(b->inst[i].desc, out + i * ECONO_PARTIAL_WORDS);
  (void)bytes; (void)err; (void)errlen;
  return ECONO_OK;
#else
  const int32_t ni = (int32_t)b->inst.size();
  int64_t nmax = 1;
  for (auto& h : b->inst) nmax = imax(nmax, h.desc.n);
  // enough blocks to fill the machine a few times over, no more than the work
  const int32_t slices = (int32_t)imax(1, imin((nmax + 255) / 256, (148 * 8 + ni - 1) / ni));
  void* d = batch_scratch(b, SCR_PART_OUT, bytes);
  void* scr = batch_scratch(b, SCR_PART_SLICES, sizeof(double) * 16 * (size_t)slices * (size_t)ni);
  if (!d || !scr) return set_err(err, errlen, "device allocation failed"), ECONO_ECUDA;
  k_partials_slices<<<dim3((unsigned)slices, (unsigned)ni), 256, 0, b->stream>>>(b->d_insts, (double*)scr);
  k_partials_finish<<<(unsigned)ni, 32, 0, b->stream>>>(b->d_insts, (const double*)scr, slices, (double*)d);
  int rc = sync_batch(b, err, errlen);
  if (!rc && dev_d2h(out, d, bytes)) rc = ECONO_ECUDA;
  return rc;
#endif
}

int econo_batch_ingest(econo_batch* b, char* err, size_t errlen) {
#ifdef ECONO_HOSTSIM
  (void)b; (void)err; (void)errlen;
  return ECONO_OK;  // the host build ingests inside step()
#else
  const int32_t ni = (int32_t)b->inst.size();
  const bool verbose = getenv("ECONO_VERBOSE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b2) { return std::chrono::duration<double, std::milli>(b2 - a).count(); };
  const auto t0 = now();
  void* dplan = batch_scratch(b, SCR_PLAN, sizeof(int64_t) * 4 * (size_t)ni);
  if (!dplan) return set_err(err, errlen, "allocation failed"), ECONO_ECUDA;
  k_bulk_plan<<<(unsigned)ni, 32, 0, b->stream>>>(b->d_insts, (int64_t*)dplan);
  std::vector<int64_t> plan(4 * (size_t)ni);
  int rc = sync_batch(b, err, errlen);
  if (!rc && dev_d2h(plan.data(), dplan, sizeof(int64_t) * plan.size())) rc = ECONO_ECUDA;
  if (rc) return rc;
  const char* env = getenv("ECONO_BULK_INGEST_MIN");
  const int64_t thr = env ? atoll(env) : 32768;
  std::vector<BulkJob> jobs;
  int bits = 1;
  for (int32_t i = 0; i < ni; ++i) {
    const Inst& I = b->inst[(size_t)i].desc;
    const int64_t k = plan[4 * (size_t)i + 1];
    const uint64_t ncls = (uint64_t)I.nbuckets * (uint64_t)(I.pmax + 1);
    if (k < thr || k < 1 || ncls > 0xffffffffULL) continue;
    BulkJob J;
    memset(&J, 0, sizeof(J));
    J.inst = i;
    J.first = plan[4 * (size_t)i];
    {
      const int64_t bw = plan[4 * (size_t)i + 2], pw = plan[4 * (size_t)i + 3];
      J.wb0 = (int32_t)(bw & 0xffffffff);
      J.wnb = (int32_t)(bw >> 32) - J.wb0 + 1;
      J.wp0 = (int32_t)(pw & 0xffffffff);
      J.wnp = (int32_t)(pw >> 32) - J.wp0 + 1;
    }
    J.k = k;
    J.tiles = (int32_t)((k + kBulkTile - 1) / kBulkTile);
    J.minp = ~0ULL;
    jobs.push_back(J);
    while (bits < 32 && (ncls - 1) >> bits) ++bits;
  }
  if (jobs.empty()) return ECONO_OK;
  {  // the default path: tile-local sorts + a per-instance stitch (no global sort)
    int64_t max_ncls = 0;
    for (const BulkJob& J : jobs) {
      const Inst& I = b->inst[(size_t)J.inst].desc;
      max_ncls = imax(max_ncls, (int64_t)I.nbuckets * (I.pmax + 1));
    }
    const size_t smem = 12 * (size_t)max_ncls;
    // ranges (default) when the range scan's class table fits shared memory;
    // ECONO_INGEST_TILES forces the tile-sort path, ECONO_INGEST_RADIX the global sort
    size_t rsmem = 0;  // the largest class window
    for (const BulkJob& J : jobs) rsmem = std::max(rsmem, 4 * (size_t)J.wnb * (size_t)J.wnp);
    const bool ranges = !getenv("ECONO_INGEST_TILES") && rsmem <= 160 * 1024;
    const int64_t span = ranges ? kRangeI : kTileI;
    if (!getenv("ECONO_INGEST_RADIX") && max_ncls <= 65536 && smem <= 200 * 1024) {
      const int64_t budget = bulk_budget();
      std::vector<size_t> gs;
      int64_t max_off = 0, max_t = 0;
      for (BulkJob& J : jobs) {
        J.tiles = (int32_t)((J.k + span - 1) / span);
        J.sstride = ranges ? (int32_t)std::min<int64_t>(span, std::max<int64_t>(1, (int64_t)J.wnb * J.wnp)) : (int32_t)span;
      }
      for (size_t g0 = 0; g0 < jobs.size();) {  // groups of jobs within the scratch budget
        size_t g1 = g0;
        int64_t off = 0, tl = 0;
        while (g1 < jobs.size() && (g1 == g0 || off + (int64_t)jobs[g1].tiles * jobs[g1].sstride <= budget)) {
          jobs[g1].off = off;   // segment slots: sstride per tile/range
          jobs[g1].hoff = tl;   // per-tile/range segment counts
          off += (int64_t)jobs[g1].tiles * jobs[g1].sstride;
          tl += jobs[g1].tiles;
          ++g1;
        }
        gs.push_back(g0);
        max_off = imax(max_off, off);
        max_t = imax(max_t, tl);
        g0 = g1;
      }
      gs.push_back(jobs.size());
      const size_t sb = (8 * (size_t)max_off + 255) & ~(size_t)255, nb = (4 * (size_t)max_t + 255) & ~(size_t)255;
      const size_t need = sb + nb + sizeof(BulkJob) * jobs.size();
      if (need > b->bulk_bytes) {
        dev_free(b->bulk_buf);
        b->bulk_buf = nullptr;
        b->bulk_bytes = 0;
        if (cudaMalloc(&b->bulk_buf, need) == cudaSuccess) b->bulk_bytes = need;
      }
      if (!b->bulk_buf) return set_err(err, errlen, "bulk ingest allocation failed"), ECONO_ECUDA;
      char* base = (char*)b->bulk_buf;
      uint64_t* segs = (uint64_t*)base;
      int32_t* nseg = (int32_t*)(base + sb);
      void* dj = base + sb + nb;
      const auto t1 = now();
      dev_h2d(dj, jobs.data(), sizeof(BulkJob) * jobs.size());
      cudaFuncSetAttribute(k_ingest_stitch<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(k_ingest_stitch<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(k_ingest_ranges<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
      cudaFuncSetAttribute(k_ingest_ranges<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
      cudaFuncSetAttribute(k_ingest_ranges<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
      cudaFuncSetAttribute(k_ingest_ranges<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
      cudaFuncSetAttribute(k_ingest_ranges<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
      cudaFuncSetAttribute(k_ingest_ranges<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
      for (size_t g = 0; g + 1 < gs.size(); ++g) {
        const int32_t nj = (int32_t)(gs[g + 1] - gs[g]);
        int32_t tmax = 0;
        for (size_t q = gs[g]; q < gs[g + 1]; ++q) tmax = std::max(tmax, jobs[q].tiles);
        BulkJob* J = (BulkJob*)dj + gs[g];
        if (ranges) {
          int wb = 1;  // bits of the largest window class index
          for (size_t q = gs[g]; q < gs[g + 1]; ++q)
            while (wb < 16 && ((int64_t)1 << wb) < (int64_t)jobs[q].wnb * jobs[q].wnp) ++wb;
          const dim3 grid((unsigned)tmax, (unsigned)nj);
          if (getenv("ECONO_INGEST_MATCH")) k_ingest_ranges<0><<<grid, 32, rsmem, b->stream>>>(b->d_insts, J, segs, nseg);
          else if (wb <= 4) k_ingest_ranges<4><<<grid, 32, rsmem, b->stream>>>(b->d_insts, J, segs, nseg);
          else if (wb <= 8) k_ingest_ranges<8><<<grid, 32, rsmem, b->stream>>>(b->d_insts, J, segs, nseg);
          else if (wb <= 10) k_ingest_ranges<10><<<grid, 32, rsmem, b->stream>>>(b->d_insts, J, segs, nseg);
          else if (wb <= 12) k_ingest_ranges<12><<<grid, 32, rsmem, b->stream>>>(b->d_insts, J, segs, nseg);
          else k_ingest_ranges<16><<<grid, 32, rsmem, b->stream>>>(b->d_insts, J, segs, nseg);
          k_ingest_stitch<true><<<(unsigned)nj, 512, smem, b->stream>>>(b->d_insts, J, segs, nseg);
        } else {
          k_ingest_tiles<<<dim3((unsigned)tmax, (unsigned)nj), 256, 0, b->stream>>>(b->d_insts, J, segs, nseg);
          k_ingest_stitch<false><<<(unsigned)nj, 512, smem, b->stream>>>(b->d_insts, J, segs, nseg);
        }
      }
      rc = sync_batch(b, err, errlen);
      if (!rc) rc = cuda_check(err, errlen, "bulk ingest");
      if (verbose)
        fprintf(stderr, "[econo] bulk ingest (%s): plan+alloc %.1f ms, kernels %.1f ms (%zu jobs, %zu groups)\n",
                ranges ? "ranges" : "tiles", ms(t0, t1), ms(t1, now()), jobs.size(), gs.size() - 1);
      return rc;
    }
  }
  const int passes = (bits + 7) / 8;
  // groups of jobs whose keys fit the temp budget; offsets are per group
  const int64_t budget = bulk_budget();
  std::vector<size_t> gstart;
  int64_t max_off = 0, max_hoff = 0;
  for (size_t g0 = 0; g0 < jobs.size();) {
    size_t g1 = g0;
    int64_t off = 0, hoff = 0;
    while (g1 < jobs.size() && (g1 == g0 || off + jobs[g1].k <= budget)) {
      jobs[g1].off = off;
      jobs[g1].hoff = hoff;
      off += jobs[g1].k;
      hoff += 256LL * jobs[g1].tiles;
      ++g1;
    }
    gstart.push_back(g0);
    max_off = std::max(max_off, off);
    max_hoff = std::max(max_hoff, hoff);
    g0 = g1;
  }
  gstart.push_back(jobs.size());
  // one cached scratch block: keys, values (ping-pong), histograms, jobs
  const size_t kb = ((4 * (size_t)max_off + 255) & ~(size_t)255);
  const size_t hb = ((4 * (size_t)max_hoff + 255) & ~(size_t)255);
  const size_t need = 4 * kb + hb + sizeof(BulkJob) * jobs.size();
  if (need > b->bulk_bytes) {
    dev_free(b->bulk_buf);
    b->bulk_buf = nullptr;
    b->bulk_bytes = 0;
    if (cudaMalloc(&b->bulk_buf, need) == cudaSuccess) b->bulk_bytes = need;
  }
  char* base = (char*)b->bulk_buf;
  void *k0 = base, *k1 = base + kb, *v0 = base + 2 * kb, *v1 = base + 3 * kb, *dh = base + 4 * kb,
       *dj = base + 4 * kb + hb;
  if (!b->bulk_buf) {
    set_err(err, errlen, "bulk ingest allocation failed");
    rc = ECONO_ECUDA;
  } else {
    const auto t1 = now();
    dev_h2d(dj, jobs.data(), sizeof(BulkJob) * jobs.size());
    for (size_t g = 0; g + 1 < gstart.size(); ++g) {  // stream-ordered; one sync at the end
      const int32_t nj = (int32_t)(gstart[g + 1] - gstart[g]);
      int32_t tmax = 0;
      for (size_t q = gstart[g]; q < gstart[g + 1]; ++q) tmax = std::max(tmax, jobs[q].tiles);
      const dim3 grid((unsigned)tmax, (unsigned)nj);
      BulkJob* J = (BulkJob*)dj + gstart[g];
      uint32_t *kin = (uint32_t*)k0, *kout = (uint32_t*)k1, *vin = (uint32_t*)v0, *vout = (uint32_t*)v1;
      k_bulk_keys<<<grid, 256, 0, b->stream>>>(b->d_insts, J, kin, vin);
      for (int pass = 0; pass < passes; ++pass) {
        k_radix_hist<<<grid, 256, 0, b->stream>>>(J, kin, 8 * pass, (uint32_t*)dh);
        k_radix_scan<<<(unsigned)nj, 1024, 0, b->stream>>>(J, (uint32_t*)dh);
        k_radix_scatter<<<grid, 256, 0, b->stream>>>(J, kin, vin, kout, vout, 8 * pass, (const uint32_t*)dh);
        std::swap(kin, kout);
        std::swap(vin, vout);
      }
      k_bulk_heads<<<grid, 256, 0, b->stream>>>(b->d_insts, J, kin, vin);
      k_bulk_tails<<<grid, 256, 0, b->stream>>>(b->d_insts, J, kin, vin);
      k_bulk_finish<<<(unsigned)nj, 32, 0, b->stream>>>(b->d_insts, J);
    }
    rc = sync_batch(b, err, errlen);
    if (!rc) rc = cuda_check(err, errlen, "bulk ingest");
    if (verbose)
      fprintf(stderr, "[econo] bulk ingest: plan+alloc %.1f ms, kernels %.1f ms (%zu jobs, %zu groups)\n", ms(t0, t1),
              ms(t1, now()), jobs.size(), gstart.size() - 1);
  }
  if (verbose) fprintf(stderr, "[econo] bulk ingest: total %.1f ms\n", ms(t0, now()));
  return rc;
#endif
}

int econo_batch_jct_prepare(econo_batch* b, char* err, size_t errlen) { return jct_prepare(b, err, errlen); }

int econo_batch_jct_hist(econo_batch* b, int32_t n_targets, const uint64_t* prefixes, int32_t consumed_bits,
                         int32_t digit_bits, uint64_t* hist, char* err, size_t errlen) {
  return jct_hist(b, 0, n_targets, prefixes, consumed_bits, digit_bits, hist, err, errlen);
}

int econo_batch_jct_percentiles(econo_batch* b, const double* q, int32_t nq, double* out, char* err, size_t errlen) {
  return jct_percentiles(b, q, nq, out, err, errlen);
}

double econo_jct_key_to_double(uint64_t key) { return key_double(key); }

// aggregate() (metrics.hpp:96-175) for every instance at once: sums from the
// device partials (cross-request sums in a different order: the 1e-6 tier),
// p5/p95 exact from the radix select, counts and the completion histogram
// exact. trace_hash is left 0 (FNV-1a over the CSV bytes is inherently
// sequential; econo_report computes it for a single engine).
int econo_batch_reports(econo_batch* b, EconoReport* out, char* err, size_t errlen) {
  const int32_t ni = (int32_t)b->inst.size();
  std::vector<double> parts((size_t)ni * ECONO_PARTIAL_WORDS), pct((size_t)ni * 2);
  int rc = econo_batch_partials(b, parts.data(), err, errlen);
  if (rc) return rc;
  const double q[2] = {0.05, 0.95};
  rc = jct_percentiles(b, q, 2, pct.data(), err, errlen);
  if (rc) return rc;
  for (int32_t i = 0; i < ni; ++i) {
    const double* p = parts.data() + (size_t)i * ECONO_PARTIAL_WORDS;
    const Inst& I = b->inst[(size_t)i].desc;
    EconoReport& r = out[i];
    memset(&r, 0, sizeof(r));
    const double n = p[0];
    r.mean_jct = p[1] / n;
    r.p5_jct = pct[(size_t)i * 2];
    r.p95_jct = pct[(size_t)i * 2 + 1];
    r.mean_tbt = p[3] > 0 ? p[2] / p[3] : 0.0;
    r.ssr = p[5] / n;
    r.normalized_latency = p[4] / n;
    r.makespan = p[10];
    if (r.makespan > 0.0) {
      r.throughput_rps = n / r.makespan;
      r.throughput_tps = p[6] / r.makespan;
      r.goodput_rps = p[5] / r.makespan;
    }
    r.allocation_failure_pct = 100.0 * p[9] / n;
    r.preemptions = (int64_t)p[7];
    r.reserve_draws = (int64_t)p[8];
    r.mean_waiting = p[11] / n;
    r.mean_execution = p[12] / n;
    r.mean_preemption = p[13] / n;
    r.mean_scheduling = p[14] / n;
    const int64_t ex = I.executed;
    r.iterations = ex;
    if (ex > 0) {
      r.mean_forward_size = (double)I.agg_fs / (double)ex;
      r.mean_kvc_written = I.agg_written / (double)ex;
      r.mean_kvc_allocated = I.agg_allocated / (double)ex;
      r.tfs_hit_frac = (double)I.agg_tfs_hits / (double)ex;
      r.pt_admit_frac = (double)I.agg_pt_iters / (double)ex;
      std::vector<int64_t> hist((size_t)I.hist_cap);
      if (dev_d2h(hist.data(), I.hist, sizeof(int64_t) * hist.size()))
        return set_err(err, errlen, "device copy failed"), ECONO_ECUDA;
      int k = 0;
      for (int c = 0; c < I.hist_cap; ++c)
        if (hist[(size_t)c]) {
          if (k >= ECONO_MAX_HIST)  // the fixed-size report cannot hold it: say so, never truncate
            return set_err(err, errlen, "completion histogram has more than %d entries (ECONO_MAX_HIST)",
                           ECONO_MAX_HIST), ECONO_ESIM;
          r.hist_count[k] = c;
          r.hist_frac[k] = (double)hist[(size_t)c] / (double)ex;
          ++k;
        }
      r.n_hist = k;
    }
    r.hosted_slots = I.hosted_total;
    r.hosted_overruns = I.hosted_overruns;
    r.trace_hash = 0;
  }
  return ECONO_OK;
}

// Development counters: per instance ECONO_DEBUG_WORDS int64 (engine.cuh Inst::prof).
int econo_batch_debug(econo_batch* b, int64_t* out) {
  for (size_t i = 0; i < b->inst.size(); ++i)
    for (int k = 0; k < ECONO_DEBUG_WORDS; ++k) out[ECONO_DEBUG_WORDS * i + k] = b->inst[i].desc.prof[k];
  return ECONO_OK;
}

int econo_batch_checkpoint(econo_batch* b, char* err, size_t errlen) {
  int rc = sync_batch(b, err, errlen);
  if (rc) return rc;
  if (!b->ckpt_block) {
    size_t total = 0;
    for (auto& h : b->inst) total += h.arena_bytes;
    void* p;
    if (dev_alloc(&p, total)) return set_err(err, errlen, "checkpoint allocation failed"), ECONO_ECUDA;
    b->ckpt_block = (char*)p;
    size_t off = 0;
    for (auto& h : b->inst) {
      h.ckpt = b->ckpt_block + off;
      off += h.arena_bytes;
    }
  }
  for (auto& h : b->inst) {
#ifdef ECONO_HOSTSIM
    memcpy(h.ckpt, h.arena, h.arena_bytes);
#else
    if (cudaMemcpyAsync(h.ckpt, h.arena, h.arena_bytes, cudaMemcpyDeviceToDevice, b->stream) != cudaSuccess)
      return set_err(err, errlen, "checkpoint copy failed"), ECONO_ECUDA;
#endif
    h.ckpt_desc = h.desc;
  }
  return sync_batch(b, err, errlen);
}

int econo_batch_restore(econo_batch* b, char* err, size_t errlen) {
  int rc = sync_batch(b, err, errlen);
  if (rc) return rc;
  for (auto& h : b->inst) {
    if (!h.ckpt) return set_err(err, errlen, "no checkpoint to restore"), ECONO_ECONFIG;
#ifdef ECONO_HOSTSIM
    memcpy(h.arena, h.ckpt, h.arena_bytes);
#else
    if (cudaMemcpyAsync(h.arena, h.ckpt, h.arena_bytes, cudaMemcpyDeviceToDevice, b->stream) != cudaSuccess)
      return set_err(err, errlen, "restore copy failed"), ECONO_ECUDA;
#endif
    // logs are not part of the state: keep the current log buffers
    Inst d = h.ckpt_desc;
    d.ev = h.desc.ev; d.ev_cap = h.desc.ev_cap; d.ev_n = 0;
    d.sm = h.desc.sm; d.sm_cap = h.desc.sm_cap; d.sm_n = 0;
    h.desc = d;
  }
  if (push_descs(b)) return set_err(err, errlen, "device copy failed"), ECONO_ECUDA;
  return sync_batch(b, err, errlen);
}

// ---- single engine -------------------------------------------------------

int econo_create(const EconoTraceRecord* trace, int64_t n, const EconoOptions* opt, int device,
                 econo_engine** out, char* err, size_t errlen) {
  econo_batch* b = nullptr;
  const int rc = econo_batch_create(&trace, &n, 1, opt, device, &b, err, errlen);
  if (rc) return rc;
  *out = new econo_engine{b, 0, true};
  return ECONO_OK;
}

void econo_destroy(econo_engine* e) {
  if (!e) return;
  if (e->owns) {
    econo_batch_destroy(e->b);
    delete e;
  }
}

int econo_step(econo_engine* e, int64_t max_steps, int32_t* more, char* err, size_t errlen) {
  econo_batch* b = e->b;
  HostInst& h = b->inst[(size_t)e->i];
  if (b->inst.size() != 1) return set_err(err, errlen, "econo_step drives single-instance engines"), ECONO_ECONFIG;
  int64_t left = max_steps;
  for (;;) {
    Inst& I = h.desc;
    if (I.error) {
      int code;
      std::string m = format_error(I, &code);
      set_err(err, errlen, "%s", m.c_str());
      return code;
    }
    if (I.completed >= I.n || left <= 0) break;
    const int64_t before = I.steps;
    launch_steps(b, left, nullptr);
    int rc = sync_batch(b, err, errlen);
    if (rc) return rc;
    rc = cuda_check(err, errlen, "k_engine_steps");
    if (rc) return rc;
    left -= h.desc.steps - before;
    if (h.desc.status == STATUS_DRAIN) {
      const bool empty_logs = h.desc.ev_n == 0 && h.desc.sm_n == 0;
      if (drain(h)) return set_err(err, errlen, "device copy failed"), ECONO_ECUDA;
      if (empty_logs) {  // the next step needs a bigger log
        if (ensure_logs(h, 2 * h.desc.ev_cap + 4096, 2 * h.desc.sm_cap + 4096))
          return set_err(err, errlen, "device allocation of the event log failed"), ECONO_ECUDA;
      }
      push_descs(b);
    }
  }
  if (drain(h)) return set_err(err, errlen, "device copy failed"), ECONO_ECUDA;
  push_descs(b);
  *more = h.desc.completed < h.desc.n ? 1 : 0;
  return ECONO_OK;
}

int econo_run(econo_engine* e, char* err, size_t errlen) {
  int32_t more = 1;
  while (more) {
    const int rc = econo_step(e, (int64_t)1 << 40, &more, err, errlen);
    if (rc) return rc;
  }
  return ECONO_OK;
}

int64_t econo_events(econo_engine* e, EconoEvent* out, int64_t cap) {
  HostInst& h = e->b->inst[(size_t)e->i];
  const int64_t n = (int64_t)h.events.size();
  if (out) memcpy(out, h.events.data(), sizeof(EconoEvent) * (size_t)imin(n, cap));
  return n;
}

int64_t econo_samples(econo_engine* e, EconoSample* out, int64_t cap) {
  HostInst& h = e->b->inst[(size_t)e->i];
  const int64_t n = (int64_t)h.samples.size();
  if (out) memcpy(out, h.samples.data(), sizeof(EconoSample) * (size_t)imin(n, cap));
  return n;
}

int econo_scalars(econo_engine* e, EconoScalars* out) {
  std::vector<EconoScalars> all(e->b->inst.size());
  econo_batch_scalars(e->b, all.data());
  *out = all[(size_t)e->i];
  return ECONO_OK;
}

int econo_records(econo_engine* e, EconoRecord* out, int64_t cap, char* err, size_t errlen) {
  HostInst& h = e->b->inst[(size_t)e->i];
  const Inst& I = h.desc;
  if (I.error) {  // the engine's own SimulationError, not a generic message
    int code;
    const std::string m = format_error(I, &code);
    return set_err(err, errlen, "%s", m.c_str()), code;
  }
  if (I.completed < I.n)
    return set_err(err, errlen, "report requested before the run finished"), ECONO_ESIM;
  std::vector<EconoRecord> recs((size_t)I.n);
#ifdef ECONO_HOSTSIM
  for (int32_t i = 0; i < I.n; ++i) engine_record(I, i, recs[(size_t)i]);
#else
  void* d;
  if (dev_alloc(&d, sizeof(EconoRecord) * (size_t)I.n)) return set_err(err, errlen, "device allocation failed"), ECONO_ECUDA;
  k_engine_records<<<148, 256, 0, e->b->stream>>>(e->b->d_insts + e->i, (EconoRecord*)d);
  int rc = sync_batch(e->b, err, errlen);
  if (!rc && dev_d2h(recs.data(), d, sizeof(EconoRecord) * (size_t)I.n)) rc = ECONO_ECUDA;
  dev_free(d);
  if (rc) return rc;
#endif
  memcpy(out, recs.data(), sizeof(EconoRecord) * (size_t)imin(I.n, cap));
  return ECONO_OK;
}

// aggregate (metrics.hpp:96-175) + the report tail of finalize (engine.hpp:986-993).
int econo_report(econo_engine* e, EconoReport* out, char* err, size_t errlen) {
  HostInst& h = e->b->inst[(size_t)e->i];
  const Inst& I = h.desc;
  std::vector<EconoRecord> recs((size_t)I.n);
  int rc = econo_records(e, recs.data(), I.n, err, errlen);
  if (rc) return rc;
  EconoReport r;
  memset(&r, 0, sizeof(r));
  std::vector<double> jcts(recs.size());
  double tbt_sum = 0.0, norm_sum = 0.0;
  long tbt_n = 0, met = 0, failures = 0;
  int64_t tokens_total = 0;
  for (size_t i = 0; i < recs.size(); ++i) {
    const EconoRecord& rc2 = recs[i];
    const double jct = rc2.completion_time - rc2.arrival;
    jcts[i] = jct;
    if (rc2.true_rl >= 2 && rc2.first_token_time >= 0.0) {
      tbt_sum += (rc2.completion_time - rc2.first_token_time) / (double)(rc2.true_rl - 1);
      ++tbt_n;
    }
    norm_sum += jct / (double)rc2.true_rl;
    if (rc2.met_slo) ++met;
    tokens_total += rc2.true_rl;
    r.preemptions += rc2.preempt_count;
    r.reserve_draws += rc2.reserve_draws;
    if (rc2.alloc_failure) ++failures;
    r.makespan = r.makespan < rc2.completion_time ? rc2.completion_time : r.makespan;
    r.mean_waiting += rc2.waiting_time;
    r.mean_execution += rc2.execution_time;
    r.mean_preemption += rc2.preemption_time;
    r.mean_scheduling += rc2.scheduling_time_share;
  }
  const double n = (double)recs.size();
  for (double j : jcts) r.mean_jct += j;
  r.mean_jct /= n;
  std::sort(jcts.begin(), jcts.end());
  auto pct = [&](double q) {
    const double rank = q * (double)(jcts.size() - 1);
    const size_t lo = (size_t)rank;
    const size_t hi = std::min(lo + 1, jcts.size() - 1);
    const double frac = rank - (double)lo;
    return jcts[lo] * (1.0 - frac) + jcts[hi] * frac;
  };
  r.p5_jct = pct(0.05);
  r.p95_jct = pct(0.95);
  r.mean_tbt = tbt_n > 0 ? tbt_sum / (double)tbt_n : 0.0;
  r.ssr = (double)met / n;
  r.normalized_latency = norm_sum / n;
  r.mean_waiting /= n;
  r.mean_execution /= n;
  r.mean_preemption /= n;
  r.mean_scheduling /= n;
  if (r.makespan > 0.0) {
    r.throughput_rps = n / r.makespan;
    r.throughput_tps = (double)tokens_total / r.makespan;
    r.goodput_rps = (double)met / r.makespan;
  }
  r.allocation_failure_pct = 100.0 * (double)failures / n;
  // sample aggregates were accumulated on the device in sample order
  const long executed = (long)I.executed;
  r.iterations = executed;
  if (executed > 0) {
    r.mean_forward_size = (double)I.agg_fs / (double)executed;
    r.mean_kvc_written = I.agg_written / (double)executed;
    r.mean_kvc_allocated = I.agg_allocated / (double)executed;
    r.tfs_hit_frac = (double)I.agg_tfs_hits / (double)executed;
    r.pt_admit_frac = (double)I.agg_pt_iters / (double)executed;
    std::vector<int64_t> hist((size_t)I.hist_cap);
    if (dev_d2h(hist.data(), I.hist, sizeof(int64_t) * hist.size()))
      return set_err(err, errlen, "device copy failed"), ECONO_ECUDA;
    int k = 0;
    for (int c = 0; c < I.hist_cap; ++c)
      if (hist[(size_t)c]) {
        if (k >= ECONO_MAX_HIST)  // the fixed-size report cannot hold it: say so, never truncate
          return set_err(err, errlen, "completion histogram has more than %d entries (ECONO_MAX_HIST)",
                         ECONO_MAX_HIST), ECONO_ESIM;
        r.hist_count[k] = c;
        r.hist_frac[k] = (double)hist[(size_t)c] / (double)executed;
        ++k;
      }
    r.n_hist = k;
  }
  // trace hash: write_trace_csv + FNV-1a (workload.hpp:127-134, metrics.hpp:320-328)
  uint64_t hh = 1469598103934665603ULL;
  auto feed = [&](const char* s, int len) {
    for (int j = 0; j < len; ++j) {
      hh ^= (unsigned char)s[j];
      hh *= 1099511628211ULL;
    }
  };
  const char* hdr = "arrival_time,prompt_len,response_len\n";
  feed(hdr, (int)strlen(hdr));
  {  // the device holds the trace as SoA (lengths < 2^30, so int32 is exact)
    std::vector<double> arr((size_t)I.n);
    std::vector<int32_t> pr((size_t)I.n), rl((size_t)I.n);
    if (dev_d2h(arr.data(), I.arrival, sizeof(double) * arr.size()) ||
        dev_d2h(pr.data(), I.prompt, sizeof(int32_t) * pr.size()) ||
        dev_d2h(rl.data(), I.true_rl, sizeof(int32_t) * rl.size()))
      return set_err(err, errlen, "device copy failed"), ECONO_ECUDA;
    char buf[128];
    for (int32_t i = 0; i < I.n; ++i) {
      const int len = snprintf(buf, sizeof(buf), "%.17g,%lld,%lld\n", arr[(size_t)i], (long long)pr[(size_t)i],
                               (long long)rl[(size_t)i]);
      feed(buf, len);
    }
  }
  r.trace_hash = hh;
  r.hosted_slots = I.hosted_total;
  r.hosted_overruns = I.hosted_overruns;
  *out = r;
  return ECONO_OK;
}

// Canonical snapshot, assembled on the host from
// a copy of the instance's device arena.
int64_t econo_snapshot(econo_engine* e, int64_t* out, int64_t cap) {
  HostInst& h = e->b->inst[(size_t)e->i];
  std::vector<char> buf(h.arena_bytes);
  if (dev_d2h(buf.data(), h.arena, h.arena_bytes)) return -1;
  Inst I = h.desc;
  rebase(I, h.arena, buf.data(), h.arena_bytes);
  std::vector<int64_t> w;
  w.reserve(1024 + 24 * (size_t)I.n);
  auto bits = [](double d) {
    int64_t v;
    memcpy(&v, &d, 8);
    return v;
  };
  w.push_back(0x45434f4e);
  w.push_back(I.iter);
  w.push_back(bits(I.clock));
  w.push_back(I.completed);
  w.push_back(I.arrival_cursor);
  w.push_back(I.free_total);
  w.push_back(I.reserved_used);
  w.push_back(I.written_total);
  w.push_back(I.hosted_total);
  w.push_back(I.hosted_overruns);
  w.push_back(I.exam_count);
  w.push_back(I.n);
  // PT queue in order
  std::vector<int64_t> ptq;
  if (I.ordered) {
    for (int b = 0; b < I.nbuckets; ++b)
      for (int p = I.pmax; p >= 0; --p)
        for (int32_t id = I.cls_head[b * (I.pmax + 1) + p]; id >= 0; id = I.pt_next[id]) ptq.push_back(id);
  } else {  // FIFO PT queue / the baselines' wait_fifo_: present tree leaves in id order
    for (int64_t id = 0; id < I.n; ++id)
      if (I.tree[id] != INF32) ptq.push_back(id);
  }
  w.push_back((int64_t)ptq.size());
  w.insert(w.end(), ptq.begin(), ptq.end());
  // GT groups in key order
  w.push_back(I.G);
  for (int32_t k = 0; k < I.G; ++k) {
    const int32_t g = I.gq[k];
    w.push_back((int64_t)I.gr_id[g]);
    w.push_back(I.gr_rl[g]);
    w.push_back(bits(I.gr_formed[g]));
    w.push_back(bits(I.gr_mindl[g]));
    w.push_back(I.gr_maxocc[g]);
    w.push_back(I.ordered ? I.gr_db[g] : 0);
    w.push_back(I.ordered ? I.gr_kb[g] : 0);
    w.push_back(I.ordered ? I.gr_rl[g] : 0);
    w.push_back((int64_t)I.gr_seq[g]);
    w.push_back(I.gr_cnt[g]);
    int32_t m = I.gr_head[g];
    for (int32_t j = 0; j < I.gr_cnt[g]; ++j) {
      w.push_back(m);
      m = I.gt_next[m];
    }
  }
  // hosting slots in insertion order
  w.push_back(I.n_slots);
  for (int32_t k = 0; k < I.n_slots; ++k) {
    const int32_t sp = I.slots[k];
    w.push_back(I.sl_host[sp]);
    w.push_back(I.sl_hosted[sp]);
    w.push_back(I.sl_off[sp]);
    w.push_back(I.sl_len[sp]);
    w.push_back(I.sl_off[sp]);
    w.push_back(I.sl_abs[sp]);
  }
  // holdings by id
  int64_t nh = 0;
  for (int32_t id = 0; id < I.n; ++id) nh += I.reg_head[id] >= 0;
  w.push_back(nh);
  for (int32_t id = 0; id < I.n; ++id) {
    if (I.reg_head[id] < 0) continue;
    w.push_back(id);
    w.push_back(I.held[id]);
    int64_t nreg = 0;
    for (int32_t r = I.reg_head[id]; r >= 0; r = I.rg_next[r]) ++nreg;
    w.push_back(nreg);
    for (int32_t r = I.reg_head[id]; r >= 0; r = I.rg_next[r]) {
      w.push_back(I.rg_start[r]);
      w.push_back(I.rg_len[r]);
    }
  }
  // free gaps: the complement of the address-ordered regions
  std::vector<int64_t> gaps;
  int64_t cur = 0;
  for (int32_t k = 0; k <= I.n_regions; ++k) {
    const int64_t s = k < I.n_regions ? I.rg_start[I.addr[k]] : I.general_cap;
    if (s > cur) { gaps.push_back(cur); gaps.push_back(s - cur); }
    if (k < I.n_regions) cur = (int64_t)I.rg_start[I.addr[k]] + I.rg_len[I.addr[k]];
  }
  w.push_back((int64_t)gaps.size() / 2);
  w.insert(w.end(), gaps.begin(), gaps.end());
  int64_t nr = 0;
  for (int32_t id = 0; id < I.n; ++id) nr += (I.flags[id] & F_HAS_RESERVED) ? 1 : 0;
  w.push_back(nr);
  for (int32_t id = 0; id < I.n; ++id)
    if (I.flags[id] & F_HAS_RESERVED) { w.push_back(id); w.push_back(I.reserved[id]); }
  int64_t nw = 0;
  for (int32_t id = 0; id < I.n; ++id) nw += I.written[id] != 0;
  w.push_back(nw);
  for (int32_t id = 0; id < I.n; ++id)
    if (I.written[id] != 0) { w.push_back(id); w.push_back(I.written[id]); }
  w.push_back(I.R);
  for (int32_t k = 0; k < I.R; ++k) w.push_back(I.run[k]);
  for (int32_t i = 0; i < I.n; ++i) {
    w.push_back(I.state[i]);
    w.push_back(I.generated[i]);
    w.push_back(I.predicted[i]);
    w.push_back(padded_of(I, i));
    w.push_back(I.allowance[i]);
    w.push_back(I.gen_epoch[i]);
    w.push_back(I.occupied[i]);
    w.push_back((I.flags[i] & F_HOSTED) ? 1 : 0);
    w.push_back((I.flags[i] & F_WAS_PREEMPTED) ? 1 : 0);
    w.push_back(I.preempt_count[i]);
    w.push_back(I.reserve_draws[i]);
    w.push_back((I.flags[i] & F_ALLOC_FAIL) ? 1 : 0);
    w.push_back(I.base ? I.prefill_done[i] : (I.state[i] == ST_WAITING_PT ? 0 : I.prompt[i]));
    w.push_back(bits(I.waiting[i]));
    w.push_back(bits(I.preempt_t[i]));
    w.push_back(bits(I.exec_t[i]));
    w.push_back(I.base ? bits(I.dispatch_t[i]) : 0);  // dead state for econoserve: not kept
    w.push_back(bits(I.first_tok[i]));
    w.push_back(bits(I.compl_clock[i]));
    w.push_back(bits(I.last_enq[i]));
    w.push_back(bits(I.sched_share[i]));
    w.push_back(bits(I.penalty[i]));
    w.push_back(bits(slo_of(I, i)));
  }
  if (I.base) {  // baseline-policy tail
    w.push_back(0x42415345);
    w.push_back(I.decode_pause);
    w.push_back(I.admission_open);
    w.push_back(bits(I.pending_stall));
    w.push_back(I.n_admo);
    for (int32_t k = 0; k < I.n_admo; ++k) w.push_back(I.admo[k]);
    w.push_back(I.n_ongo);
    for (int32_t k = 0; k < I.n_ongo; ++k) w.push_back(I.ongo[k]);
    for (int32_t i = 0; i < I.n; ++i) w.push_back(I.ptarget[i]);
  }
  const int64_t nwords = (int64_t)w.size();
  if (out) memcpy(out, w.data(), sizeof(int64_t) * (size_t)imin(nwords, cap));
  return nwords;
}

// ---- host-side trace generation (input preparation) ----------------------
// generate_synthetic (workload.hpp:42-125) with libstdc++'s mt19937_64,
// generate_canonical, polar normal and exponential (random.tcc:1811-1844,
// 3349-3380; random.h:2358, 4904), glibc libm. Bit-identical to the reference.
namespace {
struct Mt64 {
  uint64_t x[312];
  int32_t i;
  explicit Mt64(uint64_t s) { mt_seed(x, i, s); }
  double canon() { return canonical(x, i); }
};
double cdf(double v) { return 0.5 * std::erfc(-v / std::sqrt(2.0)); }
double trunc_mean(double mu, double sg, double a, double b) {
  const double al = (std::log(a) - mu) / sg, be = (std::log(b) - mu) / sg;
  const double mass = cdf(be) - cdf(al);
  if (mass <= 0.0) return a;
  const double num = cdf(be - sg) - cdf(al - sg);
  return std::exp(mu + 0.5 * sg * sg) * num / mass;
}
double fit_mu(const EconoLengthDist& d) {
  const double a = (double)d.min_value, b = (double)d.max_value;
  double lo = std::log(a) - 10.0, hi = std::log(b) + 10.0;
  for (int k = 0; k < 200; ++k) {
    const double mid = 0.5 * (lo + hi);
    if (trunc_mean(mid, d.sigma, a, b) < d.mean) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}
struct Polar {  // normal_distribution with its cached second variate
  bool have = false;
  double saved = 0.0;
  double draw(Mt64& g) {
    if (have) { have = false; return saved; }
    double x, y, r2;
    do {
      x = 2.0 * g.canon() - 1.0;
      y = 2.0 * g.canon() - 1.0;
      r2 = x * x + y * y;
    } while (r2 > 1.0 || r2 == 0.0);
    const double mult = std::sqrt(-2 * std::log(r2) / r2);
    saved = x * mult;
    have = true;
    return y * mult;
  }
};
int64_t sample_len(const EconoLengthDist& d, double mu, Mt64& g) {
  if (d.min_value == d.max_value) return d.min_value;
  Polar nd;
  for (int attempt = 0; attempt < 10000; ++attempt) {
    const int64_t v = (int64_t)std::llround(std::exp(d.sigma * (nd.draw(g) * 1.0 + 0.0) + mu));
    if (v >= d.min_value && v <= d.max_value) return v;
  }
  return std::clamp<int64_t>((int64_t)std::llround(std::exp(mu)), d.min_value, d.max_value);
}
int check_dist(const EconoLengthDist& d, char* err, size_t errlen) {
  if (d.min_value < 1 || d.max_value < d.min_value)
    return set_err(err, errlen, "length distribution bounds invalid: min=%lld max=%lld", (long long)d.min_value,
                   (long long)d.max_value), ECONO_ECONFIG;
  if (d.sigma <= 0.0) return set_err(err, errlen, "length distribution sigma must be > 0"), ECONO_ECONFIG;
  if (d.mean < (double)d.min_value || d.mean > (double)d.max_value)
    return set_err(err, errlen, "length distribution mean outside [min, max]"), ECONO_ECONFIG;
  return ECONO_OK;
}
}  // namespace

int econo_generate_trace(int64_t n, double rate, const EconoLengthDist* p, const EconoLengthDist* r, uint64_t seed,
                         EconoTraceRecord* out, char* err, size_t errlen) {
  if (n < 1) return set_err(err, errlen, "n_requests must be >= 1"), ECONO_ECONFIG;
  if (!(rate > 0.0)) return set_err(err, errlen, "arrival_rate must be > 0"), ECONO_ECONFIG;
  int rc = check_dist(*p, err, errlen);
  if (!rc) rc = check_dist(*r, err, errlen);
  if (rc) return rc;
  const double mp = fit_mu(*p), mr = fit_mu(*r);
  Mt64 g(seed);
  double clock = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    clock += -std::log(1.0 - g.canon()) / rate;
    out[i].arrival_time = clock;
    out[i].prompt_len = sample_len(*p, mp, g);
    out[i].true_rl = sample_len(*r, mr, g);
  }
  return ECONO_OK;
}

}  // extern "C"

// ---- glibc exp/log port, evaluated on the device (glibc_libm.cuh) ---------
#ifndef ECONO_HOSTSIM
__global__ void k_libm_eval(int fn, const double* in, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = fn == 0 ? econo_libm::exp(in[i]) : econo_libm::log(in[i]);
}
#endif
int econo_libm_eval(int32_t fn, const double* in, double* out, int64_t n, int device, char* err, size_t errlen) {
  if (fn != 0 && fn != 1) return set_err(err, errlen, "fn must be 0 (exp) or 1 (log)"), ECONO_ECONFIG;
#ifdef ECONO_HOSTSIM
  (void)device;
  for (int64_t i = 0; i < n; ++i) out[i] = fn == 0 ? econo_libm::exp(in[i]) : econo_libm::log(in[i]);
  return ECONO_OK;
#else
  if (cudaSetDevice(device) != cudaSuccess) return set_err(err, errlen, "cudaSetDevice(%d) failed", device), ECONO_ECUDA;
  void *din = nullptr, *dout = nullptr;
  const size_t bytes = sizeof(double) * (size_t)(n > 0 ? n : 1);
  int rc = ECONO_OK;
  if (dev_alloc(&din, bytes) || dev_alloc(&dout, bytes) || dev_h2d(din, in, bytes)) rc = ECONO_ECUDA;
  if (!rc) {
    k_libm_eval<<<1184, 256>>>(fn, (const double*)din, (double*)dout, n);
    if (cudaDeviceSynchronize() != cudaSuccess || dev_d2h(out, dout, bytes)) rc = ECONO_ECUDA;
  }
  dev_free(din);
  dev_free(dout);
  if (rc) set_err(err, errlen, "CUDA error: %s", cudaGetErrorString(cudaGetLastError()));
  return rc;
#endif
}
