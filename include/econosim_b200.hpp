// econosim_b200.hpp — header-only C++ façade over the C-ABI
// (econoserve_b200.h) that mirrors the reference simulator's public surface
// for the EconoServe scheduling path, so existing callers switch with a
// namespace change:
//
//   econosim::Engine e(trace, opt);         ->  econosim_b200::Engine e(trace, opt);
//   econosim::run(trace, opt)               ->  econosim_b200::run(trace, opt)
//
// Type and member names follow /root/reference/proj/include/econosim/:
//   TraceRecord / Trace              workload.hpp:15-23
//   PolicyKind / PolicyConfig        policies.hpp:12-85
//   CostModel / iteration_time       engine.hpp:21-51
//   PredictorConfig / ErrorModel     workload.hpp:200-218
//   OrderingConfig                   queues.hpp:16-28
//   KvcConfig / EngineOptions        engine.hpp:63-77
//   Event                            engine.hpp:53-61
//   IterationSample / RequestRecord / MetricsReport   metrics.hpp:17-76
//   Engine::step/run/report/events/samples/clock/...  engine.hpp:79-145
//   ConfigError / SimulationError    common.hpp:17-24
// Every policy kind runs on the device: the econoserve-{d,sd,sdo,full} family
// and the five comparison baselines (k_baseline_steps).
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "econoserve_b200.h"

namespace econosim_b200 {

using Tokens = std::int64_t;
using Seconds = double;
using RequestId = std::int32_t;

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SimulationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct TraceRecord {
  Seconds arrival_time = 0.0;
  Tokens prompt_len = 1;
  Tokens true_rl = 1;
  bool operator==(const TraceRecord&) const = default;
};
static_assert(sizeof(TraceRecord) == sizeof(EconoTraceRecord), "TraceRecord layout");
using Trace = std::vector<TraceRecord>;

enum class PolicyKind { Orca, Vllm, Sarathi, MultiRes, SyncCoupled, EconoD, EconoSD, EconoSDO, EconoFull };
enum class ErrorModel { Oracle, Lognormal, BucketAccuracy };

struct PolicyConfig {
  PolicyKind kind = PolicyKind::EconoFull;
  Tokens tfs = 2048;
  int batch_size_cap = 8;
  Tokens chunk_size = 512;
  double padding_ratio = 0.10;
  double reserved_fraction = 0.03;
  double buffer_ratio = 0.15;
  Tokens max_output_len = 0;
  bool vllm_recompute = false;
};
struct CostModel {
  Seconds t_base = 0.005;
  Seconds t_token = 1e-4;
  Seconds t_token_over = -1.0;
  Tokens tfs = 2048;
  Seconds preempt_offload_penalty = 0.30;
  Seconds preempt_free_penalty = 0.06;
  Seconds reserve_penalty = 0.004;
  Seconds sched_cost_per_exam = 2e-5;
  Seconds swap_stall = 0.088;
  Seconds over_rate() const { return t_token_over < 0.0 ? t_token : t_token_over; }
};
inline Seconds iteration_time(Tokens fs, const CostModel& c) {
  const Tokens base = fs < c.tfs ? fs : c.tfs;
  const Tokens over = fs - c.tfs > 0 ? fs - c.tfs : 0;
  return c.t_base + c.t_token * static_cast<double>(base) + c.over_rate() * static_cast<double>(over);
}
struct PredictorConfig {
  ErrorModel model = ErrorModel::Oracle;
  double sigma = 0.0;
  double accuracy = 1.0;
  double tolerance = 0.1;
  double padding_ratio = 0.0;
  Tokens quantum = 1;
  std::uint64_t seed = 1;
};
struct OrderingConfig {
  bool enabled = true;  // derived from the policy, as in the reference
  std::vector<Seconds> deadline_bounds = {0.2, 0.5, 2.0};
  std::vector<Tokens> kvc_bounds = {128, 256, 384, 512};
  std::vector<Tokens> length_bounds = {128, 256, 384, 512};
};
struct KvcConfig {
  Tokens capacity = 32768;
  Tokens block_size = 32;
};
struct EngineOptions {
  PolicyConfig policy;
  CostModel cost;
  PredictorConfig predictor;
  OrderingConfig ordering;
  KvcConfig kvc;
  double slo_scale = 2.0;
  std::uint64_t seed = 1;
  bool record_events = true;
  int device = 0;  // extension: CUDA device ordinal
};

struct Event {
  long iter = 0;
  Seconds clock = 0.0;
  std::string kind;
  RequestId id = -1;
  std::string detail;
  bool operator==(const Event&) const = default;
};
struct IterationSample {
  long iter = 0;
  Seconds clock = 0.0;
  Seconds dt = 0.0;
  Tokens forward_size = 0;
  double kvc_written_frac = 0.0;
  double kvc_allocated_frac = 0.0;
  int completed = 0;
  int pts_admitted = 0;
  bool pt_admittable = false;
  long idle_repeat = 0;
};
struct RequestRecord {
  RequestId id = -1;
  Seconds arrival = 0.0;
  Seconds first_token_time = -1.0;
  Seconds completion_time = 0.0;
  Seconds waiting_time = 0.0;
  Seconds execution_time = 0.0;
  Seconds preemption_time = 0.0;
  Seconds scheduling_time_share = 0.0;
  int preempt_count = 0;
  int reserve_draws = 0;
  bool met_slo = false;
  Tokens prompt_len = 0;
  Tokens true_rl = 0;
  Seconds slo_deadline = 0.0;
  bool alloc_failure = false;
  Seconds jct() const { return completion_time - arrival; }
};
struct MetricsReport {
  std::string policy;
  std::uint64_t trace_hash = 0;
  double mean_jct = 0.0, p5_jct = 0.0, p95_jct = 0.0;
  double mean_tbt = 0.0;
  double ssr = 0.0;
  double throughput_rps = 0.0, throughput_tps = 0.0;
  double goodput_rps = 0.0;
  double normalized_latency = 0.0;
  double mean_kvc_written = 0.0, mean_kvc_allocated = 0.0;
  double mean_forward_size = 0.0;
  double allocation_failure_pct = 0.0;
  double tfs_hit_frac = 0.0;
  double pt_admit_frac = 0.0;
  std::map<int, double> iteration_completion_histogram;
  long iterations = 0;
  Seconds makespan = 0.0;
  long preemptions = 0;
  long reserve_draws = 0;
  long hosted_slots = 0;
  long hosted_overruns = 0;
  double mean_waiting = 0.0, mean_execution = 0.0, mean_preemption = 0.0, mean_scheduling = 0.0;
  std::vector<RequestRecord> records;
};

namespace detail {

[[noreturn]] inline void raise(int rc, const char* msg) {
  if (rc == ECONO_ECONFIG) throw ConfigError(msg);
  if (rc == ECONO_ESIM) throw SimulationError(msg);
  throw DeviceError(msg);
}

inline const char* policy_name(PolicyKind k) {
  static const char* n[] = {"orca", "vllm", "sarathi", "multires", "sync-coupled",
                            "econoserve-d", "econoserve-sd", "econoserve-sdo", "econoserve-full"};
  return n[static_cast<int>(k)];
}

inline EconoOptions to_c(const EngineOptions& o) {
  EconoOptions c;
  econo_default_options(&c);
  c.policy = static_cast<int32_t>(o.policy.kind);
  c.batch_size_cap = o.policy.batch_size_cap;
  c.tfs = o.policy.tfs;
  c.chunk_size = o.policy.chunk_size;
  c.padding_ratio = o.policy.padding_ratio;
  c.reserved_fraction = o.policy.reserved_fraction;
  c.buffer_ratio = o.policy.buffer_ratio;
  c.max_output_len = o.policy.max_output_len;
  c.vllm_recompute = o.policy.vllm_recompute ? 1 : 0;
  c.t_base = o.cost.t_base;
  c.t_token = o.cost.t_token;
  c.t_token_over = o.cost.t_token_over;
  c.cost_tfs = o.cost.tfs;
  c.preempt_offload_penalty = o.cost.preempt_offload_penalty;
  c.preempt_free_penalty = o.cost.preempt_free_penalty;
  c.reserve_penalty = o.cost.reserve_penalty;
  c.sched_cost_per_exam = o.cost.sched_cost_per_exam;
  c.swap_stall = o.cost.swap_stall;
  c.pred_model = static_cast<int32_t>(o.predictor.model);
  c.pred_sigma = o.predictor.sigma;
  c.pred_accuracy = o.predictor.accuracy;
  c.pred_tolerance = o.predictor.tolerance;
  c.pred_padding_ratio = o.predictor.padding_ratio;
  c.pred_quantum = o.predictor.quantum;
  c.pred_seed = o.predictor.seed;
  if (o.ordering.deadline_bounds.size() > ECONO_MAX_BOUNDS || o.ordering.kvc_bounds.size() > ECONO_MAX_BOUNDS ||
      o.ordering.length_bounds.size() > ECONO_MAX_BOUNDS)
    throw ConfigError("ordering: too many bucket boundaries");
  c.n_deadline_bounds = static_cast<int32_t>(o.ordering.deadline_bounds.size());
  c.n_kvc_bounds = static_cast<int32_t>(o.ordering.kvc_bounds.size());
  c.n_length_bounds = static_cast<int32_t>(o.ordering.length_bounds.size());
  for (size_t i = 0; i < o.ordering.deadline_bounds.size(); ++i) c.deadline_bounds[i] = o.ordering.deadline_bounds[i];
  for (size_t i = 0; i < o.ordering.kvc_bounds.size(); ++i) c.kvc_bounds[i] = o.ordering.kvc_bounds[i];
  for (size_t i = 0; i < o.ordering.length_bounds.size(); ++i) c.length_bounds[i] = o.ordering.length_bounds[i];
  c.kvc_capacity = o.kvc.capacity;
  c.kvc_block_size = o.kvc.block_size;
  c.slo_scale = o.slo_scale;
  c.seed = o.seed;
  c.record_events = o.record_events ? 1 : 0;
  c.record_samples = 1;
  return c;
}

// Event::kind / Event::detail exactly as Engine::log writes them (engine.hpp:211-214).
inline Event to_event(const EconoEvent& e) {
  static const char* kinds[] = {"arrive",  "gt_schedule",    "hosted", "pt_dispatch", "prefill_done",
                                "complete", "reserve_topup", "preempt", "hosted_overrun", "idle",
                                "alloc_fail", "preempt_swap", "swap_in"};
  Event out;
  out.iter = static_cast<long>(e.iter);
  out.clock = e.clock;
  out.kind = (e.kind >= 0 && e.kind < 13) ? kinds[e.kind] : "?";
  out.id = e.id;
  switch (e.kind) {
    case ECONO_EV_GT_SCHEDULE:
    case ECONO_EV_COMPLETE: out.detail = "rl=" + std::to_string(e.a); break;
    case ECONO_EV_HOSTED:
      out.detail = "host=" + std::to_string(e.a) + " deadline=" + std::to_string(e.b);
      break;
    case ECONO_EV_PREFILL_DONE: out.detail = e.a ? "" : "to-gt-queue"; break;
    case ECONO_EV_PREEMPT_SWAP: out.detail = "written=" + std::to_string(e.a); break;
    case ECONO_EV_PREEMPT:
      out.detail = std::string(e.a ? "overrun" : "underprediction") + " l_new=" + std::to_string(e.b);
      break;
    case ECONO_EV_IDLE: out.detail = std::to_string(e.a); break;
    default: break;
  }
  return out;
}

}  // namespace detail

class Engine {
 public:
  Engine(Trace trace, EngineOptions opt) : trace_(std::move(trace)), opt_(std::move(opt)) {
    const EconoOptions c = detail::to_c(opt_);
    char err[1024] = {0};
    econo_engine* h = nullptr;
    const int rc = econo_create(reinterpret_cast<const EconoTraceRecord*>(trace_.data()),
                                static_cast<int64_t>(trace_.size()), &c, opt_.device, &h, err, sizeof(err));
    if (rc) detail::raise(rc, err);
    h_.reset(h);
  }

  // Advances one engine cycle; returns false once every request is done.
  bool step() { return step_n(1); }
  // Extension: advances up to n cycles in one device launch.
  bool step_n(std::int64_t n) {
    char err[1024] = {0};
    int32_t more = 0;
    const int rc = econo_step(h_.get(), n, &more, err, sizeof(err));
    if (rc) detail::raise(rc, err);
    dirty_ = true;
    return more != 0;
  }
  MetricsReport run() {
    char err[1024] = {0};
    const int rc = econo_run(h_.get(), err, sizeof(err));
    if (rc) detail::raise(rc, err);
    dirty_ = true;
    return report();
  }
  MetricsReport report() {
    char err[1024] = {0};
    EconoReport r;
    int rc = econo_report(h_.get(), &r, err, sizeof(err));
    if (rc) detail::raise(rc, err);
    std::vector<EconoRecord> recs(trace_.size());
    rc = econo_records(h_.get(), recs.data(), static_cast<int64_t>(recs.size()), err, sizeof(err));
    if (rc) detail::raise(rc, err);
    MetricsReport m;
    m.policy = detail::policy_name(opt_.policy.kind);
    m.trace_hash = r.trace_hash;
    m.mean_jct = r.mean_jct; m.p5_jct = r.p5_jct; m.p95_jct = r.p95_jct; m.mean_tbt = r.mean_tbt;
    m.ssr = r.ssr; m.throughput_rps = r.throughput_rps; m.throughput_tps = r.throughput_tps;
    m.goodput_rps = r.goodput_rps; m.normalized_latency = r.normalized_latency;
    m.mean_kvc_written = r.mean_kvc_written; m.mean_kvc_allocated = r.mean_kvc_allocated;
    m.mean_forward_size = r.mean_forward_size; m.allocation_failure_pct = r.allocation_failure_pct;
    m.tfs_hit_frac = r.tfs_hit_frac; m.pt_admit_frac = r.pt_admit_frac;
    for (int i = 0; i < r.n_hist; ++i) m.iteration_completion_histogram[r.hist_count[i]] = r.hist_frac[i];
    m.iterations = static_cast<long>(r.iterations); m.makespan = r.makespan;
    m.preemptions = static_cast<long>(r.preemptions); m.reserve_draws = static_cast<long>(r.reserve_draws);
    m.hosted_slots = static_cast<long>(r.hosted_slots); m.hosted_overruns = static_cast<long>(r.hosted_overruns);
    m.mean_waiting = r.mean_waiting; m.mean_execution = r.mean_execution;
    m.mean_preemption = r.mean_preemption; m.mean_scheduling = r.mean_scheduling;
    m.records.reserve(recs.size());
    for (const auto& x : recs) {
      RequestRecord q;
      q.id = x.id; q.arrival = x.arrival; q.first_token_time = x.first_token_time;
      q.completion_time = x.completion_time; q.waiting_time = x.waiting_time;
      q.execution_time = x.execution_time; q.preemption_time = x.preemption_time;
      q.scheduling_time_share = x.scheduling_time_share; q.preempt_count = x.preempt_count;
      q.reserve_draws = x.reserve_draws; q.met_slo = x.met_slo != 0; q.prompt_len = x.prompt_len;
      q.true_rl = x.true_rl; q.slo_deadline = x.slo_deadline; q.alloc_failure = x.alloc_failure != 0;
      m.records.push_back(q);
    }
    return m;
  }

  const std::vector<Event>& events() {
    refresh();
    return events_;
  }
  const std::vector<IterationSample>& samples() {
    refresh();
    return samples_;
  }
  Seconds clock() const { return scalars().clock; }
  Seconds clock_from_samples() {
    Seconds s = 0.0;
    for (const auto& x : samples()) s += x.dt;
    return s;
  }
  long hosted_slots_created() const { return static_cast<long>(scalars().hosted_slots_created); }
  long hosted_overruns() const { return static_cast<long>(scalars().hosted_overruns); }
  Seconds calibrated_prefill_time() const { return scalars().calibrated_prefill_time; }
  Seconds calibrated_decode_time() const { return scalars().calibrated_decode_time; }
  // Extension: canonical state snapshot.
  std::vector<std::int64_t> snapshot() const {
    std::vector<std::int64_t> w(static_cast<size_t>(econo_snapshot(h_.get(), nullptr, 0)));
    econo_snapshot(h_.get(), w.data(), static_cast<int64_t>(w.size()));
    return w;
  }

 private:
  struct Deleter {
    void operator()(econo_engine* e) const { econo_destroy(e); }
  };
  EconoScalars scalars() const {
    EconoScalars s;
    econo_scalars(h_.get(), &s);
    return s;
  }
  void refresh() {
    if (!dirty_) return;
    std::vector<EconoEvent> ev(static_cast<size_t>(econo_events(h_.get(), nullptr, 0)));
    econo_events(h_.get(), ev.data(), static_cast<int64_t>(ev.size()));
    events_.clear();
    events_.reserve(ev.size());
    for (const auto& e : ev) events_.push_back(detail::to_event(e));
    std::vector<EconoSample> sm(static_cast<size_t>(econo_samples(h_.get(), nullptr, 0)));
    econo_samples(h_.get(), sm.data(), static_cast<int64_t>(sm.size()));
    samples_.clear();
    samples_.reserve(sm.size());
    for (const auto& s : sm) {
      IterationSample x;
      x.iter = static_cast<long>(s.iter); x.clock = s.clock; x.dt = s.dt; x.forward_size = s.forward_size;
      x.kvc_written_frac = s.kvc_written_frac; x.kvc_allocated_frac = s.kvc_allocated_frac;
      x.completed = s.completed; x.pts_admitted = s.pts_admitted; x.pt_admittable = s.pt_admittable != 0;
      x.idle_repeat = static_cast<long>(s.idle_repeat);
      samples_.push_back(x);
    }
    dirty_ = false;
  }

  Trace trace_;
  EngineOptions opt_;
  std::unique_ptr<econo_engine, Deleter> h_;
  std::vector<Event> events_;
  std::vector<IterationSample> samples_;
  bool dirty_ = true;
};

// One-call entry point (engine.hpp:1039-1042).
inline MetricsReport run(Trace trace, const EngineOptions& opt) {
  Engine engine(std::move(trace), opt);
  return engine.run();
}

// ---- wire formats (workload.hpp:127-194, metrics.hpp:181-240, 320-328) ----
// load_trace_csv / write_trace_csv with the reference's validation and bytes.
inline Trace load_trace_csv(const std::string& path) {
  char err[1024] = {0};
  int64_t n = 0;
  int rc = econo_load_trace_csv(path.c_str(), nullptr, 0, &n, err, sizeof(err));
  if (rc) detail::raise(rc, err);
  Trace t(static_cast<size_t>(n));
  rc = econo_load_trace_csv(path.c_str(), reinterpret_cast<EconoTraceRecord*>(t.data()), n, &n, err, sizeof(err));
  if (rc) detail::raise(rc, err);
  return t;
}
inline std::string write_trace_csv(const Trace& trace) {
  int64_t len = 0;
  const auto* p = reinterpret_cast<const EconoTraceRecord*>(trace.data());
  econo_write_trace_csv(p, static_cast<int64_t>(trace.size()), nullptr, 0, &len);
  std::string s(static_cast<size_t>(len) + 1, '\0');
  econo_write_trace_csv(p, static_cast<int64_t>(trace.size()), &s[0], len + 1, &len);
  s.resize(static_cast<size_t>(len));
  return s;
}
// to_json(report, with_records).dump(indent) as a string, byte-identical to the
// reference's nlohmann::ordered_json output (the CLI writes dump(2) + "\n").
inline std::string to_json_string(const MetricsReport& m, bool with_records = true, int indent = -1) {
  EconoReport r;
  std::memset(&r, 0, sizeof(r));
  r.trace_hash = m.trace_hash;
  r.mean_jct = m.mean_jct; r.p5_jct = m.p5_jct; r.p95_jct = m.p95_jct; r.mean_tbt = m.mean_tbt; r.ssr = m.ssr;
  r.throughput_rps = m.throughput_rps; r.throughput_tps = m.throughput_tps; r.goodput_rps = m.goodput_rps;
  r.normalized_latency = m.normalized_latency; r.mean_kvc_written = m.mean_kvc_written;
  r.mean_kvc_allocated = m.mean_kvc_allocated; r.mean_forward_size = m.mean_forward_size;
  r.allocation_failure_pct = m.allocation_failure_pct; r.tfs_hit_frac = m.tfs_hit_frac;
  r.pt_admit_frac = m.pt_admit_frac; r.iterations = m.iterations; r.makespan = m.makespan;
  r.preemptions = m.preemptions; r.reserve_draws = m.reserve_draws; r.hosted_slots = m.hosted_slots;
  r.hosted_overruns = m.hosted_overruns; r.mean_waiting = m.mean_waiting; r.mean_execution = m.mean_execution;
  r.mean_preemption = m.mean_preemption; r.mean_scheduling = m.mean_scheduling;
  for (const auto& kv : m.iteration_completion_histogram) {
    if (r.n_hist >= ECONO_MAX_HIST) break;
    r.hist_count[r.n_hist] = kv.first;
    r.hist_frac[r.n_hist] = kv.second;
    ++r.n_hist;
  }
  std::vector<EconoRecord> recs;
  if (with_records) {
    recs.reserve(m.records.size());
    for (const auto& q : m.records) {
      EconoRecord x;
      std::memset(&x, 0, sizeof(x));
      x.id = q.id; x.arrival = q.arrival; x.first_token_time = q.first_token_time;
      x.completion_time = q.completion_time; x.waiting_time = q.waiting_time; x.execution_time = q.execution_time;
      x.preemption_time = q.preemption_time; x.scheduling_time_share = q.scheduling_time_share;
      x.preempt_count = q.preempt_count; x.reserve_draws = q.reserve_draws; x.met_slo = q.met_slo ? 1 : 0;
      x.prompt_len = q.prompt_len; x.true_rl = q.true_rl; x.slo_deadline = q.slo_deadline;
      x.alloc_failure = q.alloc_failure ? 1 : 0;
      recs.push_back(x);
    }
  }
  const EconoRecord* rp = with_records ? recs.data() : nullptr;
  int64_t len = 0;
  econo_report_to_json(m.policy.c_str(), &r, rp, static_cast<int64_t>(recs.size()), nullptr, indent, nullptr, 0,
                       &len);
  std::string s(static_cast<size_t>(len) + 1, '\0');
  econo_report_to_json(m.policy.c_str(), &r, rp, static_cast<int64_t>(recs.size()), nullptr, indent, &s[0], len + 1,
                       &len);
  s.resize(static_cast<size_t>(len));
  return s;
}

}  // namespace econosim_b200
