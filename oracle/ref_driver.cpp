// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI driver around the UNMODIFIED reference simulator headers
// (/root/reference/proj/include/econosim/*.hpp), compiled in place by
// oracle/Makefile into oracle/_ref/libecono_ref.so. It is the pin for the C
// restatement (oracle/econo_oracle.c) and the CPU baseline of bench.py
// (cpu_baseline.kind = "reference").
//
// Private engine state (running_gts_, exam_count_, KvcAllocator::free_/alloc_)
// is read through the test-only route SURVEY.md §7.1 describes: every std
// header and json.hpp first, then `#define private public`.
#include <algorithm>
#include <any>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <atomic>
#include <vector>

#include <json.hpp>

#define private public
#include "econosim/engine.hpp"
#include "econosim/sweep.hpp"
#undef private

#include "econoserve_b200.h"

using namespace econosim;

namespace {

void set_err(char* err, size_t errlen, const std::string& m) {
  if (err && errlen) {
    std::snprintf(err, errlen, "%s", m.c_str());
  }
}

EngineOptions to_options(const EconoOptions* o) {
  EngineOptions e;
  e.policy.kind = static_cast<PolicyKind>(o->policy);
  e.policy.tfs = o->tfs;
  e.policy.batch_size_cap = o->batch_size_cap;
  e.policy.chunk_size = o->chunk_size;
  e.policy.padding_ratio = o->padding_ratio;
  e.policy.reserved_fraction = o->reserved_fraction;
  e.policy.buffer_ratio = o->buffer_ratio;
  e.policy.max_output_len = o->max_output_len;
  e.policy.vllm_recompute = o->vllm_recompute != 0;
  e.cost.t_base = o->t_base;
  e.cost.t_token = o->t_token;
  e.cost.t_token_over = o->t_token_over;
  e.cost.tfs = o->cost_tfs;
  e.cost.preempt_offload_penalty = o->preempt_offload_penalty;
  e.cost.preempt_free_penalty = o->preempt_free_penalty;
  e.cost.reserve_penalty = o->reserve_penalty;
  e.cost.sched_cost_per_exam = o->sched_cost_per_exam;
  e.cost.swap_stall = o->swap_stall;
  e.predictor.model = static_cast<ErrorModel>(o->pred_model);
  e.predictor.sigma = o->pred_sigma;
  e.predictor.accuracy = o->pred_accuracy;
  e.predictor.tolerance = o->pred_tolerance;
  e.predictor.padding_ratio = o->pred_padding_ratio;
  e.predictor.quantum = o->pred_quantum;
  e.predictor.seed = o->pred_seed;
  e.ordering.deadline_bounds.assign(o->deadline_bounds, o->deadline_bounds + o->n_deadline_bounds);
  e.ordering.kvc_bounds.assign(o->kvc_bounds, o->kvc_bounds + o->n_kvc_bounds);
  e.ordering.length_bounds.assign(o->length_bounds, o->length_bounds + o->n_length_bounds);
  e.kvc.capacity = o->kvc_capacity;
  e.kvc.block_size = o->kvc_block_size;
  e.slo_scale = o->slo_scale;
  e.seed = o->seed;
  e.record_events = o->record_events != 0;
  return e;
}

Trace to_trace(const EconoTraceRecord* t, int64_t n) {
  Trace tr(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    tr[i].arrival_time = t[i].arrival_time;
    tr[i].prompt_len = t[i].prompt_len;
    tr[i].true_rl = t[i].true_rl;
  }
  return tr;
}

int64_t bits(double d) {
  int64_t v;
  std::memcpy(&v, &d, 8);
  return v;
}

int kind_code(const std::string& k) {
  static const std::map<std::string, int> m = {
      {"arrive", ECONO_EV_ARRIVE},           {"gt_schedule", ECONO_EV_GT_SCHEDULE},
      {"hosted", ECONO_EV_HOSTED},           {"pt_dispatch", ECONO_EV_PT_DISPATCH},
      {"prefill_done", ECONO_EV_PREFILL_DONE}, {"complete", ECONO_EV_COMPLETE},
      {"reserve_topup", ECONO_EV_RESERVE_TOPUP}, {"preempt", ECONO_EV_PREEMPT},
      {"hosted_overrun", ECONO_EV_HOSTED_OVERRUN}, {"idle", ECONO_EV_IDLE},
      {"alloc_fail", ECONO_EV_ALLOC_FAIL}, {"preempt_swap", ECONO_EV_PREEMPT_SWAP},
      {"swap_in", ECONO_EV_SWAP_IN}};
  auto it = m.find(k);
  return it == m.end() ? -1 : it->second;
}

// Parses the detail string back into the integer form of EconoEvent.
void parse_detail(const Event& ev, EconoEvent* out) {
  out->a = 0;
  out->b = 0;
  const std::string& d = ev.detail;
  long long a = 0, b = 0;
  switch (out->kind) {
    case ECONO_EV_GT_SCHEDULE:
    case ECONO_EV_COMPLETE:
      std::sscanf(d.c_str(), "rl=%lld", &a);
      out->a = a;
      break;
    case ECONO_EV_HOSTED:
      std::sscanf(d.c_str(), "host=%lld deadline=%lld", &a, &b);
      out->a = a;
      out->b = b;
      break;
    case ECONO_EV_PREEMPT: {
      out->a = d.rfind("overrun", 0) == 0 ? 1 : 0;
      auto p = d.find("l_new=");
      if (p != std::string::npos) out->b = std::atoll(d.c_str() + p + 6);
      break;
    }
    case ECONO_EV_IDLE:
      out->a = std::atoll(d.c_str());
      break;
    case ECONO_EV_PREFILL_DONE:
      out->a = d.empty() ? 1 : 0;  // "" = a baseline prefill that keeps decoding
      break;
    case ECONO_EV_PREEMPT_SWAP:
      std::sscanf(d.c_str(), "written=%lld", &a);
      out->a = a;
      break;
    default:
      break;
  }
}

struct RefEngine {
  std::unique_ptr<Engine> eng;
  long steps = 0;
};

}  // namespace

extern "C" {

int ref_create(const EconoTraceRecord* trace, int64_t n, const EconoOptions* opt, void** out,
               char* err, size_t errlen) {
  try {
    auto* h = new RefEngine();
    h->eng = std::make_unique<Engine>(to_trace(trace, n), to_options(opt));
    *out = h;
    return ECONO_OK;
  } catch (const ConfigError& e) {
    set_err(err, errlen, e.what());
    return ECONO_ECONFIG;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return ECONO_ESIM;
  }
}

void ref_destroy(void* h) { delete static_cast<RefEngine*>(h); }

// Deep copy of an engine (Engine is a value type): lets a benchmark warm up
// on the copy and time the original from the same state.
void* ref_clone(void* hv) {
  auto* h = static_cast<RefEngine*>(hv);
  auto* c = new RefEngine();
  c->eng = std::make_unique<Engine>(*h->eng);
  c->steps = h->steps;
  return c;
}

// Advances up to max_steps step() calls; *more = step()'s last return value.
int ref_step(void* hv, int64_t max_steps, int32_t* more, char* err, size_t errlen) {
  auto* h = static_cast<RefEngine*>(hv);
  try {
    bool m = h->eng->completed_ < static_cast<long>(h->eng->reqs_.size());
    for (int64_t i = 0; i < max_steps && m; ++i) {
      m = h->eng->step();
      ++h->steps;
    }
    *more = m ? 1 : 0;
    return ECONO_OK;
  } catch (const ConfigError& e) {
    set_err(err, errlen, e.what());
    return ECONO_ECONFIG;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return ECONO_ESIM;
  }
}

int64_t ref_events(void* hv, EconoEvent* out, int64_t cap) {
  auto* h = static_cast<RefEngine*>(hv);
  const auto& evs = h->eng->events();
  const int64_t n = static_cast<int64_t>(evs.size());
  for (int64_t i = 0; i < n && i < cap; ++i) {
    const Event& ev = evs[static_cast<size_t>(i)];
    out[i].iter = ev.iter;
    out[i].clock = ev.clock;
    out[i].kind = kind_code(ev.kind);
    out[i].id = ev.id;
    parse_detail(ev, &out[i]);
  }
  return n;
}

// Original detail string of event i (for byte-level checks of the formatter).
int ref_event_detail(void* hv, int64_t i, char* out, size_t cap) {
  auto* h = static_cast<RefEngine*>(hv);
  const auto& evs = h->eng->events();
  if (i < 0 || i >= static_cast<int64_t>(evs.size())) return -1;
  std::snprintf(out, cap, "%s|%s", evs[static_cast<size_t>(i)].kind.c_str(),
                evs[static_cast<size_t>(i)].detail.c_str());
  return 0;
}

int64_t ref_samples(void* hv, EconoSample* out, int64_t cap) {
  auto* h = static_cast<RefEngine*>(hv);
  const auto& ss = h->eng->samples();
  const int64_t n = static_cast<int64_t>(ss.size());
  for (int64_t i = 0; i < n && i < cap; ++i) {
    const IterationSample& s = ss[static_cast<size_t>(i)];
    std::memset(&out[i], 0, sizeof(EconoSample));
    out[i].iter = s.iter;
    out[i].clock = s.clock;
    out[i].dt = s.dt;
    out[i].forward_size = s.forward_size;
    out[i].kvc_written_frac = s.kvc_written_frac;
    out[i].kvc_allocated_frac = s.kvc_allocated_frac;
    out[i].completed = s.completed;
    out[i].pts_admitted = s.pts_admitted;
    out[i].pt_admittable = s.pt_admittable ? 1 : 0;
    out[i].idle_repeat = s.idle_repeat;
  }
  return n;
}

static void fill_report(const MetricsReport& rep, EconoReport* out) {
  std::memset(out, 0, sizeof(*out));
  out->mean_jct = rep.mean_jct;
  out->p5_jct = rep.p5_jct;
  out->p95_jct = rep.p95_jct;
  out->mean_tbt = rep.mean_tbt;
  out->ssr = rep.ssr;
  out->throughput_rps = rep.throughput_rps;
  out->throughput_tps = rep.throughput_tps;
  out->goodput_rps = rep.goodput_rps;
  out->normalized_latency = rep.normalized_latency;
  out->mean_kvc_written = rep.mean_kvc_written;
  out->mean_kvc_allocated = rep.mean_kvc_allocated;
  out->mean_forward_size = rep.mean_forward_size;
  out->allocation_failure_pct = rep.allocation_failure_pct;
  out->tfs_hit_frac = rep.tfs_hit_frac;
  out->pt_admit_frac = rep.pt_admit_frac;
  out->iterations = rep.iterations;
  out->makespan = rep.makespan;
  out->preemptions = rep.preemptions;
  out->reserve_draws = rep.reserve_draws;
  out->hosted_slots = rep.hosted_slots;
  out->hosted_overruns = rep.hosted_overruns;
  out->mean_waiting = rep.mean_waiting;
  out->mean_execution = rep.mean_execution;
  out->mean_preemption = rep.mean_preemption;
  out->mean_scheduling = rep.mean_scheduling;
  out->trace_hash = rep.trace_hash;
  int k = 0;
  for (const auto& [count, frac] : rep.iteration_completion_histogram) {
    if (k >= ECONO_MAX_HIST) break;
    out->hist_count[k] = count;
    out->hist_frac[k] = frac;
    ++k;
  }
  out->n_hist = k;
}

// finalize(): records + report. Valid only once the run finished.
int ref_finalize(void* hv, EconoRecord* recs, int64_t cap, EconoReport* rep_out, char* err,
                 size_t errlen) {
  auto* h = static_cast<RefEngine*>(hv);
  try {
    MetricsReport rep = h->eng->report();
    for (size_t i = 0; i < rep.records.size() && static_cast<int64_t>(i) < cap; ++i) {
      const RequestRecord& r = rep.records[i];
      EconoRecord& o = recs[i];
      std::memset(&o, 0, sizeof(o));
      o.id = r.id;
      o.preempt_count = r.preempt_count;
      o.arrival = r.arrival;
      o.first_token_time = r.first_token_time;
      o.completion_time = r.completion_time;
      o.waiting_time = r.waiting_time;
      o.execution_time = r.execution_time;
      o.preemption_time = r.preemption_time;
      o.scheduling_time_share = r.scheduling_time_share;
      o.reserve_draws = r.reserve_draws;
      o.met_slo = r.met_slo ? 1 : 0;
      o.prompt_len = r.prompt_len;
      o.true_rl = r.true_rl;
      o.slo_deadline = r.slo_deadline;
      o.alloc_failure = r.alloc_failure ? 1 : 0;
    }
    if (rep_out) fill_report(rep, rep_out);
    return ECONO_OK;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return ECONO_ESIM;
  }
}

// to_json(report).dump(indent) of the finished run (byte-level report schema).
int64_t ref_report_json(void* hv, char* out, int64_t cap, int with_records, int indent) {
  auto* h = static_cast<RefEngine*>(hv);
  try {
    MetricsReport rep = h->eng->report();
    std::string s = to_json(rep, with_records != 0).dump(indent);
    if (out && cap > 0) std::snprintf(out, static_cast<size_t>(cap), "%s", s.c_str());
    return static_cast<int64_t>(s.size());
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_scalars(void* hv, EconoScalars* o) {
  auto* h = static_cast<RefEngine*>(hv);
  const Engine& e = *h->eng;
  std::memset(o, 0, sizeof(*o));
  o->clock = e.clock_;
  o->iter = e.iter_;
  o->completed = e.completed_;
  o->steps = h->steps;
  long executed = 0;
  for (const auto& s : e.samples_)
    if (s.idle_repeat == 0) ++executed;
  o->executed_iters = executed;
  o->hosted_slots_created = e.hosted_total_;
  o->hosted_overruns = e.hosted_overruns_;
  o->calibrated_prefill_time = e.t_p_;
  o->calibrated_decode_time = e.t_g_;
  long pt = 0, gt = 0;
  for (const auto& ev : e.events_) {
    if (ev.kind == "pt_dispatch") ++pt;
    if (ev.kind == "gt_schedule" || ev.kind == "hosted") ++gt;
  }
  o->pt_dispatched = pt;
  o->gt_scheduled = gt;
  o->pt_queue_len = static_cast<int64_t>(e.pt_queue_.size());
  o->gt_queue_groups = static_cast<int64_t>(e.gt_queue_.size());
  o->running = static_cast<int64_t>(e.running_gts_.size());
  o->arrived = static_cast<int64_t>(e.arrival_cursor_);
  o->done = e.completed_ >= static_cast<long>(e.reqs_.size()) ? 1 : 0;
  return 0;
}

// Canonical state serialisation; see DESIGN.md "Snapshot format".
int64_t ref_snapshot(void* hv, int64_t* out, int64_t cap) {
  auto* h = static_cast<RefEngine*>(hv);
  const Engine& e = *h->eng;
  std::vector<int64_t> w;
  w.reserve(1024);
  const KvcAllocator& k = e.kvc_;
  w.push_back(0x45434f4e);
  w.push_back(e.iter_);
  w.push_back(bits(e.clock_));
  w.push_back(e.completed_);
  w.push_back(static_cast<int64_t>(e.arrival_cursor_));
  w.push_back(k.free_total_);
  w.push_back(k.reserved_used_);
  w.push_back(k.written_total_);
  w.push_back(e.hosted_total_);
  w.push_back(e.hosted_overruns_);
  w.push_back(e.exam_count_);
  w.push_back(static_cast<int64_t>(e.reqs_.size()));
  // PT queue (the baselines' wait_fifo_ in its place)
  const bool econo = is_econoserve(e.pol_.kind);
  if (econo) {
    w.push_back(static_cast<int64_t>(e.pt_queue_.entries().size()));
    for (const auto& pe : e.pt_queue_.entries()) w.push_back(pe.id);
  } else {
    w.push_back(static_cast<int64_t>(e.wait_fifo_.size()));
    for (RequestId id : e.wait_fifo_) w.push_back(id);
  }
  // GT queue (sync-coupled's waiting_groups_ in its place)
  const GtQueue& gq = econo ? e.gt_queue_ : e.waiting_groups_;
  w.push_back(static_cast<int64_t>(gq.groups().size()));
  for (const auto& g : gq.groups()) {
    w.push_back(static_cast<int64_t>(g.group_id));
    w.push_back(g.padded_rl);
    w.push_back(bits(g.formed_at));
    w.push_back(bits(g.min_deadline));
    w.push_back(g.max_occupied);
    w.push_back(g.key.deadline_bucket);
    w.push_back(g.key.kvc_bucket);
    w.push_back(g.key.length);
    w.push_back(static_cast<int64_t>(g.key.seq));
    w.push_back(static_cast<int64_t>(g.members.size()));
    for (RequestId id : g.members) w.push_back(id);
  }
  // slots
  w.push_back(static_cast<int64_t>(k.slots_.size()));
  for (const auto& s : k.slots_) {
    w.push_back(s.host_id);
    w.push_back(s.hosted_id);
    w.push_back(s.start_offset);
    w.push_back(s.length);
    w.push_back(s.deadline_usage);
    w.push_back(s.abs_start);
  }
  // holdings (ascending id)
  w.push_back(static_cast<int64_t>(k.alloc_.size()));
  for (const auto& [id, hld] : k.alloc_) {
    w.push_back(id);
    w.push_back(hld.total);
    w.push_back(static_cast<int64_t>(hld.regions.size()));
    for (const auto& r : hld.regions) {
      w.push_back(r.start);
      w.push_back(r.len);
    }
  }
  // free gaps
  w.push_back(static_cast<int64_t>(k.free_.size()));
  for (const auto& [s, l] : k.free_) {
    w.push_back(s);
    w.push_back(l);
  }
  // reserved draws
  w.push_back(static_cast<int64_t>(k.reserved_.size()));
  for (const auto& [id, t] : k.reserved_) {
    w.push_back(id);
    w.push_back(t);
  }
  // written (non-zero entries only)
  int64_t nw = 0;
  for (const auto& [id, t] : k.written_)
    if (t != 0) ++nw;
  w.push_back(nw);
  for (const auto& [id, t] : k.written_)
    if (t != 0) {
      w.push_back(id);
      w.push_back(t);
    }
  // running GTs in order
  w.push_back(static_cast<int64_t>(e.running_gts_.size()));
  for (RequestId id : e.running_gts_) w.push_back(id);
  // per-request state
  for (const Request& r : e.reqs_) {
    w.push_back(static_cast<int64_t>(r.state));
    w.push_back(r.generated);
    w.push_back(r.predicted_rl);
    w.push_back(r.padded_rl);
    w.push_back(r.allowance);
    w.push_back(r.generated_at_epoch);
    w.push_back(r.occupied_kvc);
    w.push_back(r.hosted ? 1 : 0);
    w.push_back(r.was_preempted ? 1 : 0);
    w.push_back(r.preempt_count);
    w.push_back(r.reserve_draws);
    w.push_back(r.alloc_failure_flag ? 1 : 0);
    w.push_back(r.prefill_done);
    w.push_back(bits(r.waiting_time));
    w.push_back(bits(r.preemption_time));
    w.push_back(bits(r.execution_time));
    // Request::dispatch_time is dead state for the econoserve policies (written at
    // engine.hpp:374, read only by the baselines, engine.hpp:527/615, in no record
    // or report): the device does not keep it for them, so it is not compared
    w.push_back(econo ? 0 : bits(r.dispatch_time));
    w.push_back(bits(r.first_token_time));
    w.push_back(bits(r.completion_clock));
    w.push_back(bits(r.last_enqueue_time));
    auto it = e.sched_share_.find(r.id);
    w.push_back(bits(it == e.sched_share_.end() ? 0.0 : it->second));
    auto pit = e.penalty_extra_.find(r.id);
    w.push_back(bits(pit == e.penalty_extra_.end() ? 0.0 : pit->second));
    w.push_back(bits(r.slo_deadline));
  }
  if (!econo) {  // baseline-policy tail
    w.push_back(0x42415345);
    w.push_back(e.decode_pause_ ? 1 : 0);
    w.push_back(e.admission_open_ ? 1 : 0);
    w.push_back(bits(e.pending_stall_));
    w.push_back(static_cast<int64_t>(e.admit_order_.size()));
    for (RequestId id : e.admit_order_) w.push_back(id);
    w.push_back(static_cast<int64_t>(e.ongoing_prefills_.size()));
    for (RequestId id : e.ongoing_prefills_) w.push_back(id);
    for (const Request& r : e.reqs_) w.push_back(r.prefill_target);
  }
  const int64_t n = static_cast<int64_t>(w.size());
  if (out) std::memcpy(out, w.data(), static_cast<size_t>(std::min(n, cap)) * 8);
  return n;
}

// generate_synthetic (workload.hpp:104-125) through the reference itself.
int ref_generate_trace(int64_t n, double rate, const EconoLengthDist* p, const EconoLengthDist* r,
                       uint64_t seed, EconoTraceRecord* out, char* err, size_t errlen) {
  try {
    SyntheticTraceSpec spec;
    spec.n_requests = static_cast<int>(n);
    spec.arrival_rate = rate;
    spec.prompt_dist = {p->mean, p->min_value, p->max_value, p->sigma};
    spec.rl_dist = {r->mean, r->min_value, r->max_value, r->sigma};
    spec.seed = seed;
    Trace t = generate_synthetic(spec);
    for (size_t i = 0; i < t.size(); ++i) {
      out[i].arrival_time = t[i].arrival_time;
      out[i].prompt_len = t[i].prompt_len;
      out[i].true_rl = t[i].true_rl;
    }
    return ECONO_OK;
  } catch (const ConfigError& e) {
    set_err(err, errlen, e.what());
    return ECONO_ECONFIG;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return ECONO_ESIM;
  }
}

// write_trace_csv + hash_trace_bytes (engine.hpp:988-990, metrics.hpp:320-328).
uint64_t ref_trace_hash(const EconoTraceRecord* t, int64_t n) {
  std::ostringstream oss;
  write_trace_csv(oss, to_trace(t, n));
  return hash_trace_bytes(oss.str());
}

// Burst ingest equivalent to ingest_arrivals() (engine.hpp:216-235) for the
// bench's CPU baseline: the reference's ordered insert is O(n^2) (672-773 s
// at 1M), so the post-ingest state is built with one stable sort
// (identical result: insert_ordered is an upper_bound insert, queues.hpp:85-92)
// and the measured window starts from it. Returns the number ingested.
int64_t ref_fast_ingest(void* hv) {
  auto* h = static_cast<RefEngine*>(hv);
  Engine& e = *h->eng;
  if (!is_econoserve(e.pol_.kind)) return -1;
  std::vector<PtEntry> add;
  while (e.arrival_cursor_ < e.trace_.size() &&
         e.trace_[e.arrival_cursor_].arrival_time <= e.clock_ + 1e-12) {
    const RequestId id = static_cast<RequestId>(e.arrival_cursor_++);
    Request& r = e.reqs_[id];
    e.log("arrive", id);
    TaskOrderInfo info;
    info.deadline_slack = r.slo_deadline - e.clock_;
    info.occupied_kvc = 0;
    info.length = r.record.prompt_len;
    add.push_back({id, make_key(info, e.pt_queue_.cfg_, e.pt_queue_.next_seq_++)});
  }
  auto& ent = e.pt_queue_.entries_;
  ent.insert(ent.end(), add.begin(), add.end());
  std::stable_sort(ent.begin(), ent.end(),
                   [](const PtEntry& a, const PtEntry& b) { return a.key < b.key; });
  return static_cast<int64_t>(add.size());
}

// Advances the idle stretch before the first arrival (engine.hpp:930-949) so
// that ref_fast_ingest sees the burst, i.e. exactly what step() does first.
int ref_idle_to_first_arrival(void* hv) {
  auto* h = static_cast<RefEngine*>(hv);
  Engine& e = *h->eng;
  e.ingest_arrivals();
  if (!e.pt_queue_.empty()) return 0;
  e.form_batch();
  e.handle_idle();
  ++h->steps;
  return 1;
}

// Times `steps` step() calls; returns wall seconds (CPU baseline timing).
double ref_time_steps(void* hv, int64_t steps, int64_t* pt_dispatched_delta) {
  auto* h = static_cast<RefEngine*>(hv);
  const size_t ev0 = h->eng->events_.size();
  const auto t0 = std::chrono::steady_clock::now();
  for (int64_t i = 0; i < steps; ++i) {
    if (!h->eng->step()) break;
    ++h->steps;
  }
  const auto t1 = std::chrono::steady_clock::now();
  int64_t pt = 0;
  for (size_t i = ev0; i < h->eng->events_.size(); ++i)
    if (h->eng->events_[i].kind == "pt_dispatch") ++pt;
  if (pt_dispatched_delta) *pt_dispatched_delta = pt;
  return std::chrono::duration<double>(t1 - t0).count();
}

// Multi-threaded CPU baseline: `n_eng` engines, one std::thread each, every
// engine stepped `steps` times (mirrors run_sweep's thread pool, sweep.hpp:112-149).
// Returns max wall seconds over threads; per-engine PT dispatch counts in out_pt.
double ref_time_steps_parallel(void** hv, int32_t n_eng, int64_t steps, int64_t* out_pt) {
  std::vector<std::thread> th;
  std::vector<double> secs(static_cast<size_t>(n_eng), 0.0);
  for (int32_t i = 0; i < n_eng; ++i)
    th.emplace_back([&, i] { secs[i] = ref_time_steps(hv[i], steps, out_pt ? &out_pt[i] : nullptr); });
  for (auto& t : th) t.join();
  double m = 0.0;
  for (double s : secs) m = std::max(m, s);
  return m;
}

// libstdc++ known-answer vectors for the restated RNG plumbing.
void ref_mt_draws(uint64_t seed, int64_t n, uint64_t* out) {
  Rng g(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = g();
}
void ref_shuffle_indices(uint64_t seed, int64_t n, int64_t* idx) {
  Rng g(seed);
  std::vector<int64_t> v(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) v[static_cast<size_t>(i)] = i;
  std::shuffle(v.begin(), v.end(), g);
  for (int64_t i = 0; i < n; ++i) idx[i] = v[static_cast<size_t>(i)];
}
// predict_rl + apply_padding over a sequence (workload.hpp:228-268).
int64_t ref_predict(const EconoOptions* o, uint64_t seed, const int64_t* true_rl, int64_t n, int64_t* out) {
  EngineOptions e = to_options(o);
  Rng g(seed);
  for (int64_t i = 0; i < n; ++i)
    out[i] = apply_padding(predict_rl(true_rl[i], e.predictor, g), e.predictor.padding_ratio);
  return n;
}

// nlohmann::ordered_json(v).dump(): the double printer the reports use.
int64_t ref_json_double(double v, char* out, int64_t cap) {
  const std::string s = Json(v).dump();
  if (out && cap > 0) std::snprintf(out, static_cast<size_t>(cap), "%s", s.c_str());
  return static_cast<int64_t>(s.size());
}

// load_trace_csv(istream, name) (workload.hpp:142-194) on an in-memory text.
int ref_parse_csv(const char* text, int64_t len, const char* name, EconoTraceRecord* out, int64_t cap,
                  int64_t* n, char* err, size_t errlen) {
  try {
    std::istringstream in(std::string(text, static_cast<size_t>(len)));
    Trace t = load_trace_csv(in, name);
    *n = static_cast<int64_t>(t.size());
    for (int64_t i = 0; i < *n && i < cap; ++i) {
      out[i].arrival_time = t[static_cast<size_t>(i)].arrival_time;
      out[i].prompt_len = t[static_cast<size_t>(i)].prompt_len;
      out[i].true_rl = t[static_cast<size_t>(i)].true_rl;
    }
    return ECONO_OK;
  } catch (const ConfigError& e) {
    set_err(err, errlen, e.what());
    return ECONO_ECONFIG;
  }
}

// write_trace_csv (workload.hpp:127-134).
int64_t ref_write_csv(const EconoTraceRecord* t, int64_t n, char* out, int64_t cap) {
  Trace tr(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    tr[static_cast<size_t>(i)].arrival_time = t[i].arrival_time;
    tr[static_cast<size_t>(i)].prompt_len = t[i].prompt_len;
    tr[static_cast<size_t>(i)].true_rl = t[i].true_rl;
  }
  std::ostringstream oss;
  write_trace_csv(oss, tr);
  const std::string s = oss.str();
  if (out && cap > 0) std::snprintf(out, static_cast<size_t>(cap), "%s", s.c_str());
  return static_cast<int64_t>(s.size());
}

// ---- experiment / sweep layer (config.hpp, sweep.hpp, metrics.hpp:243-318) ----
static int64_t put_str(const std::string& s, char* out, int64_t cap) {
  if (out && cap > 0) std::snprintf(out, static_cast<size_t>(cap), "%s", s.c_str());
  return static_cast<int64_t>(s.size());
}

// parse_config(json): 0, or 2 with the ConfigError message.
int ref_parse_config(const char* json, char* err, size_t errlen) {
  try {
    parse_config(Json::parse(json));
    return ECONO_OK;
  } catch (const ConfigError& e) {
    set_err(err, errlen, e.what());
    return ECONO_ECONFIG;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return 9;
  }
}

// to_json(run_experiment(parse_config(json))[policy]).dump(indent); -1 on error.
int64_t ref_experiment_report(const char* json, const char* policy, int with_records, int indent, char* out,
                              int64_t cap) {
  try {
    auto reports = run_experiment(parse_config(Json::parse(json)));
    return put_str(to_json(reports.at(policy), with_records != 0).dump(indent), out, cap);
  } catch (const std::exception&) {
    return -1;
  }
}

// render_table(compare(run_experiment(...), baseline)).
int64_t ref_render_table(const char* json, const char* baseline, char* out, int64_t cap) {
  try {
    auto reports = run_experiment(parse_config(Json::parse(json)));
    std::map<std::string, MetricsReport> by_name(reports.begin(), reports.end());
    return put_str(render_table(compare(by_name, baseline)), out, cap);
  } catch (const std::exception&) {
    return -1;
  }
}

// write_sweep_csv(run_sweep(parse_config(json), 1)).
int64_t ref_sweep_csv(const char* json, char* out, int64_t cap) {
  try {
    SweepResult r = run_sweep(parse_config(Json::parse(json)), 1);
    std::ostringstream oss;
    write_sweep_csv(oss, r);
    return put_str(oss.str(), out, cap);
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
