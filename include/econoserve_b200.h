/*
 * econoserve_b200.h — C-ABI drop-in boundary for EconoServe's per-iteration
 * scheduling step (arXiv 2411.06364), B200-native (sm_100a).
 *
 * Every entry point replaces one piece of the reference simulator's public
 * surface (/root/reference/proj/include/econosim/...):
 *
 *   econo_create        <- econosim::Engine::Engine(Trace, EngineOptions)   engine.hpp:81-100
 *                          (validation: PolicyConfig::validate policies.hpp:76-84,
 *                           CostModel::validate engine.hpp:36-43,
 *                           PredictorConfig::validate workload.hpp:211-217,
 *                           OrderingConfig::validate queues.hpp:22-27,
 *                           KvcAllocator ctor kvc.hpp:37-47,
 *                           init_requests feasibility engine.hpp:165-209)
 *   econo_step          <- Engine::step()                                     engine.hpp:104-116
 *   econo_run           <- Engine::run() / econosim::run(trace, opt)          engine.hpp:118-122, 1039-1042
 *   econo_records       <- Engine::finalize() per-request records             engine.hpp:963-994
 *   econo_report        <- Engine::report() -> aggregate()                    engine.hpp:124-128, metrics.hpp:96-175
 *   econo_events        <- Engine::events()                                   engine.hpp:130
 *   econo_samples       <- Engine::samples()                                  engine.hpp:131
 *   econo_snapshot      <- requests()/gt_queue()/pt_queue()/kvc() accessors   engine.hpp:132-135
 *   econo_scalars       <- clock()/hosted_slots_created()/hosted_overruns()/
 *                          calibrated_prefill_time()/calibrated_decode_time() engine.hpp:136-145
 *   econo_batch_*       <- run_sweep's independent engines (sweep.hpp:112-149), as many
 *                          device-resident instances advanced by one kernel launch
 *
 * Errors: no exception crosses the ABI. Return codes mirror the CLI's exit
 * codes (tools/econosim.cpp:20-22, 183-192):
 *   ECONO_OK = 0, ECONO_ECONFIG = 2 (econosim::ConfigError),
 *   ECONO_ESIM = 3 (econosim::SimulationError / std::logic_error),
 *   ECONO_ECUDA = 4 (device unavailable / CUDA failure; the product never
 *                    falls back to a CPU path).
 * The message written to `err` names the request exactly as the reference
 * does ("request 0: KVC demand ... exceeds usable capacity ...").
 *
 * Threading: handles are independent; no global mutable state. One handle
 * must not be used from two threads at once (engine.hpp is single-threaded).
 */
#ifndef ECONOSERVE_B200_H
#define ECONOSERVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ECONO_OK 0
#define ECONO_ECONFIG 2
#define ECONO_ESIM 3
#define ECONO_ECUDA 4

/* econosim::PolicyKind (policies.hpp:12-22); only the EconoServe family runs here. */
#define ECONO_POLICY_ORCA 0
#define ECONO_POLICY_VLLM 1
#define ECONO_POLICY_SARATHI 2
#define ECONO_POLICY_MULTIRES 3
#define ECONO_POLICY_SYNC_COUPLED 4
#define ECONO_POLICY_ECONO_D 5
#define ECONO_POLICY_ECONO_SD 6
#define ECONO_POLICY_ECONO_SDO 7
#define ECONO_POLICY_ECONO_FULL 8

/* econosim::ErrorModel (workload.hpp:200) */
#define ECONO_PRED_ORACLE 0
#define ECONO_PRED_LOGNORMAL 1
#define ECONO_PRED_BUCKET 2

#define ECONO_MAX_BOUNDS 8
#define ECONO_MAX_HIST 256

/* econosim::TraceRecord (workload.hpp:15-21): identical layout (24 bytes), so a
 * reference caller can pass trace.data() directly. */
typedef struct EconoTraceRecord {
  double arrival_time;
  int64_t prompt_len;
  int64_t true_rl;
} EconoTraceRecord;

/* econosim::EngineOptions (engine.hpp:68-77) flattened into fixed-width fields. */
typedef struct EconoOptions {
  /* PolicyConfig (policies.hpp:65-85) */
  int32_t policy;
  int32_t batch_size_cap;
  int64_t tfs;
  int64_t chunk_size;
  double padding_ratio; /* PolicyConfig::padding_ratio: validated, unused by the engine */
  double reserved_fraction;
  double buffer_ratio;
  int64_t max_output_len;
  int32_t vllm_recompute;
  int32_t _pad0;
  /* CostModel (engine.hpp:21-44) */
  double t_base;
  double t_token;
  double t_token_over;
  int64_t cost_tfs; /* overwritten by policy.tfs in the ctor (engine.hpp:98) */
  double preempt_offload_penalty;
  double preempt_free_penalty;
  double reserve_penalty;
  double sched_cost_per_exam;
  double swap_stall;
  /* PredictorConfig (workload.hpp:202-218) */
  int32_t pred_model;
  int32_t _pad1;
  double pred_sigma;
  double pred_accuracy;
  double pred_tolerance;
  double pred_padding_ratio;
  int64_t pred_quantum;
  uint64_t pred_seed;
  /* OrderingConfig (queues.hpp:16-28); `enabled` is derived from the policy (engine.hpp:153-157) */
  int32_t n_deadline_bounds;
  int32_t n_kvc_bounds;
  int32_t n_length_bounds;
  int32_t _pad2;
  double deadline_bounds[ECONO_MAX_BOUNDS];
  int64_t kvc_bounds[ECONO_MAX_BOUNDS];
  int64_t length_bounds[ECONO_MAX_BOUNDS];
  /* KvcConfig (engine.hpp:63-66) */
  int64_t kvc_capacity;
  int64_t kvc_block_size;
  /* EngineOptions tail */
  double slo_scale;
  uint64_t seed;
  int32_t record_events;
  int32_t record_samples; /* extension: 0 keeps only the running sample aggregates */
} EconoOptions;

/* Event kinds: the `kind` strings logged by Engine::log (engine.hpp:211-214). */
#define ECONO_EV_ARRIVE 0         /* "arrive"                                  E:221 */
#define ECONO_EV_GT_SCHEDULE 1    /* "gt_schedule"  detail "rl=<a>"            E:347 */
#define ECONO_EV_HOSTED 2         /* "hosted"       "host=<a> deadline=<b>"    E:294 */
#define ECONO_EV_PT_DISPATCH 3    /* "pt_dispatch"                             E:380 */
#define ECONO_EV_PREFILL_DONE 4   /* "prefill_done" "to-gt-queue" (a=0), "" for baselines (a=1) E:803,807 */
#define ECONO_EV_COMPLETE 5       /* "complete"     "rl=<a>"                   E:851 */
#define ECONO_EV_RESERVE_TOPUP 6  /* "reserve_topup"                           E:862 */
#define ECONO_EV_PREEMPT 7        /* "preempt"  "<a?overrun:underprediction> l_new=<b>" E:915 */
#define ECONO_EV_HOSTED_OVERRUN 8 /* "hosted_overrun"                          E:882 */
#define ECONO_EV_IDLE 9           /* "idle"  id=-1  detail "<a>"               E:948 */
#define ECONO_EV_ALLOC_FAIL 10    /* "alloc_fail"                              E:437,641 */
#define ECONO_EV_PREEMPT_SWAP 11  /* "preempt_swap" "written=<a>"              E:474 */
#define ECONO_EV_SWAP_IN 12       /* "swap_in"                                 E:517,592,613 */

/* econosim::Event (engine.hpp:53-61) with the detail string kept as integers. */
typedef struct EconoEvent {
  int64_t iter;
  double clock;
  int32_t kind;
  int32_t id;
  int64_t a;
  int64_t b;
} EconoEvent;

/* econosim::IterationSample (metrics.hpp:37-48) */
typedef struct EconoSample {
  int64_t iter;
  double clock;
  double dt;
  int64_t forward_size;
  double kvc_written_frac;
  double kvc_allocated_frac;
  int32_t completed;
  int32_t pts_admitted;
  int32_t pt_admittable;
  int32_t _pad;
  int64_t idle_repeat;
} EconoSample;

/* econosim::RequestRecord (metrics.hpp:17-35) */
typedef struct EconoRecord {
  int32_t id;
  int32_t preempt_count;
  double arrival;
  double first_token_time;
  double completion_time;
  double waiting_time;
  double execution_time;
  double preemption_time;
  double scheduling_time_share;
  int32_t reserve_draws;
  int32_t met_slo;
  int64_t prompt_len;
  int64_t true_rl;
  double slo_deadline;
  int32_t alloc_failure;
  int32_t _pad;
} EconoRecord;

/* econosim::MetricsReport scalars (metrics.hpp:50-76); histogram returned separately. */
typedef struct EconoReport {
  double mean_jct, p5_jct, p95_jct, mean_tbt, ssr;
  double throughput_rps, throughput_tps, goodput_rps, normalized_latency;
  double mean_kvc_written, mean_kvc_allocated, mean_forward_size;
  double allocation_failure_pct, tfs_hit_frac, pt_admit_frac;
  int64_t iterations;
  double makespan;
  int64_t preemptions, reserve_draws, hosted_slots, hosted_overruns;
  double mean_waiting, mean_execution, mean_preemption, mean_scheduling;
  uint64_t trace_hash;
  int32_t n_hist;           /* entries in the completion histogram (<= ECONO_MAX_HIST; a report that would
                               need more fails with ECONO_ESIM instead of truncating) */
  int32_t _pad;
  int32_t hist_count[ECONO_MAX_HIST]; /* sorted ascending, like std::map<int,double> */
  double hist_frac[ECONO_MAX_HIST];
} EconoReport;

/* Engine scalars (engine.hpp:136-145) plus counters the bench reports. */
typedef struct EconoScalars {
  double clock;
  int64_t iter;           /* engine iteration counter (idle ticks included) */
  int64_t completed;
  int64_t steps;          /* Engine::step() calls so far */
  int64_t executed_iters; /* executed (non-idle) iterations */
  int64_t hosted_slots_created;
  int64_t hosted_overruns;
  double calibrated_prefill_time;
  double calibrated_decode_time;
  int64_t pt_dispatched;  /* pt_dispatch events so far (counted even when not recorded) */
  int64_t gt_scheduled;   /* gt_schedule + hosted events so far */
  int64_t pt_queue_len;
  int64_t gt_queue_groups;
  int64_t running;
  int64_t arrived;
  int32_t done;
  int32_t error;          /* ECONO_OK or ECONO_ESIM once the engine faulted */
  int64_t quiet_steps;    /* steps replayed by event-horizon skipping */
  int64_t quiet_spans;
} EconoScalars;

/* Default options, identical to a default-constructed econosim::EngineOptions
 * (engine.hpp:68-77) with policy econoserve-full. */
void econo_default_options(EconoOptions* opt);

/* ---- single-engine API (mirrors econosim::Engine) ---------------------- */
typedef struct econo_engine econo_engine;

int econo_create(const EconoTraceRecord* trace, int64_t n, const EconoOptions* opt, int device,
                 econo_engine** out, char* err, size_t errlen);
/* Advances up to max_steps Engine::step() calls in one device launch.
 * *more = 0 once every request is done (step() returned false). */
int econo_step(econo_engine* e, int64_t max_steps, int32_t* more, char* err, size_t errlen);
int econo_run(econo_engine* e, char* err, size_t errlen);
int econo_records(econo_engine* e, EconoRecord* out, int64_t cap, char* err, size_t errlen);
int econo_report(econo_engine* e, EconoReport* out, char* err, size_t errlen);
int64_t econo_events(econo_engine* e, EconoEvent* out, int64_t cap);
int64_t econo_samples(econo_engine* e, EconoSample* out, int64_t cap);
int econo_scalars(econo_engine* e, EconoScalars* out);
/* Canonical state serialisation (layout: DESIGN.md "Snapshot format"); returns
 * the number of int64 words needed (writes min(need, cap)). */
int64_t econo_snapshot(econo_engine* e, int64_t* out, int64_t cap);
void econo_destroy(econo_engine* e);

/* ---- multi-instance batch (one CTA per instance, on one device) --------- */
typedef struct econo_batch econo_batch;

/* Device bytes one instance of this trace + options occupies (its HBM arena,
 * sized exactly as econo_batch_create would): capacity planning, e.g. how
 * many instances fit on one GPU. Returns -code (2/3) on invalid input. */
int64_t econo_instance_bytes(const EconoTraceRecord* trace, int64_t n, const EconoOptions* opt, char* err,
                             size_t errlen);
int econo_batch_create(const EconoTraceRecord* const* traces, const int64_t* n, int32_t n_inst,
                       const EconoOptions* opts /* n_inst entries */, int device,
                       econo_batch** out, char* err, size_t errlen);
/* A trace as three arrays (the instance's own device layout): the same
 * content as EconoTraceRecord[n] (workload.hpp:20-24) with the lengths in
 * 32 bits (the device path requires them in [1, 2^30) anyway). */
typedef struct EconoTraceSoA {
  const double* arrival_time;
  const int32_t* prompt_len;
  const int32_t* true_rl;
} EconoTraceSoA;
/* econo_batch_create for traces given as arrays: each array is copied
 * straight into the instance's structure-of-arrays in HBM (16 B per request
 * over PCIe instead of the record's 24 B, no staging or conversion pass).
 * Same validation, messages and resulting state as econo_batch_create. */
int econo_batch_create_soa(const EconoTraceSoA* traces, const int64_t* n, int32_t n_inst,
                           const EconoOptions* opts /* n_inst entries */, int device,
                           econo_batch** out, char* err, size_t errlen);
/* Launches one device pass that advances every live instance by up to
 * max_steps steps on `stream` (a cudaStream_t, NULL = the handle's stream).
 * Asynchronous: no host synchronisation. */
int econo_batch_launch(econo_batch* b, int64_t max_steps, void* stream);
/* Time-sliced launch: every live instance advances by up to max_steps steps
 * but stops at the first step boundary after slice_ns of device time, so a
 * slow instance no longer holds every other SM idle until it finishes (the
 * host build ignores the slice). Asynchronous like econo_batch_launch. */
int econo_batch_launch_slice(econo_batch* b, int64_t max_steps, int64_t slice_ns, void* stream);
/* Advances every live instance until it has made target_steps Engine::step()
 * calls in total (instances already there do nothing), optionally
 * time-sliced like econo_batch_launch_slice (slice_ns <= 0: no slice). Brings
 * a batch whose instances drifted apart under time slices back to one common
 * step, e.g. to compare it with the reference at that step. Asynchronous. */
int econo_batch_launch_to(econo_batch* b, int64_t target_steps, int64_t slice_ns, void* stream);
/* Grid-wide ingest of the arrivals every instance would admit at the start of
 * its next step (ingest_arrivals, engine.hpp:216-235): the same class lists,
 * bitmaps and counters the in-kernel ingest builds, produced for large bursts
 * by a stable radix sort of the batch by PT class instead of one warp per
 * instance. Semantically a no-op reordering (it is the first part of the
 * next step, run early); applies to ordered-queue policies with event
 * recording off and batches of at least ECONO_BULK_INGEST_MIN (env, default
 * 32768) arrivals; other instances ingest in-kernel as usual. Synchronous. */
int econo_batch_ingest(econo_batch* b, char* err, size_t errlen);
int econo_batch_sync(econo_batch* b, char* err, size_t errlen);
int econo_batch_scalars(econo_batch* b, EconoScalars* out /* n_inst entries */);
int econo_batch_engine(econo_batch* b, int32_t i, econo_engine** out); /* borrowed view */
/* Device-side aggregation of the per-instance metric partial sums
 * (metrics.hpp:110-173) into `out` (ECONO_PARTIAL_WORDS doubles per instance). */
#define ECONO_PARTIAL_WORDS 32
int econo_batch_partials(econo_batch* b, double* out, char* err, size_t errlen);
/* aggregate() (metrics.hpp:96-175) for every instance, computed on the device:
 * per-request sums from the partials (reordered: 1e-6 relative), p5/p95 JCT
 * exact (radix select of the order statistics, then percentile()'s
 * interpolation, metrics.hpp:81-89), counts and the completion histogram
 * exact. trace_hash = 0 (econo_report computes it for one engine). */
int econo_batch_reports(econo_batch* b, EconoReport* out /* n_inst entries */, char* err, size_t errlen);
/* JCT order statistics. JCT keys are JCT doubles mapped to uint64 so that
 * unsigned order == double order (econo_jct_key_to_double inverts it).
 * econo_batch_jct_prepare materialises the keys of every instance (call it
 * after the last launch); econo_batch_jct_hist is one MSB-first radix-select
 * pass over ALL instances of the batch: for each of n_targets (<= 8) prefixes
 * (the top consumed_bits of the key), hist[t][d] counts keys with that prefix
 * whose next digit_bits (<= 11) bits equal d. Histograms from several
 * devices add up, so a cross-GPU select all-reduces them (metrics.py).
 * econo_batch_jct_percentiles: per-instance exact percentile() values for
 * nq <= 4 quantiles (out: n_inst x nq). */
int econo_batch_jct_prepare(econo_batch* b, char* err, size_t errlen);
int econo_batch_jct_hist(econo_batch* b, int32_t n_targets, const uint64_t* prefixes, int32_t consumed_bits,
                         int32_t digit_bits, uint64_t* hist, char* err, size_t errlen);
int econo_batch_jct_percentiles(econo_batch* b, const double* q, int32_t nq, double* out, char* err, size_t errlen);
double econo_jct_key_to_double(uint64_t key);
/* Device-side checkpoint / restore of every instance's complete state
 * (arena + descriptor), e.g. to rerun one scheduling window. */
int econo_batch_checkpoint(econo_batch* b, char* err, size_t errlen);
int econo_batch_restore(econo_batch* b, char* err, size_t errlen);
/* Development counters (ECONO_DEBUG_WORDS int64 per instance): device cycles
 * spent in the quiet-span test, quiet-span replay and normal steps (and its
 * phases), and their counts; layout documented at engine.cuh Inst::prof. */
#define ECONO_DEBUG_WORDS 16
int econo_batch_debug(econo_batch* b, int64_t* out);
void econo_batch_destroy(econo_batch* b);

/* ---- glibc 2.39 exp/log as the device computes them ---------------------- */
/* The lognormal predictor's exp and the polar method's log (workload.hpp:
 * 233-235, random.tcc:1811-1844) run on the device as a port of glibc's own
 * (x86-64 FMA variant), so predictions match the reference bit for bit.
 * Evaluates fn (0 = exp, 1 = log) over n inputs on `device`, for checking the
 * port against the host libm. */
int econo_libm_eval(int32_t fn, const double* in, double* out, int64_t n, int device, char* err, size_t errlen);

/* ---- host-side input preparation (out of the hot path) ------------------ */
/* econosim::generate_synthetic (workload.hpp:104-125), bit-identical to the
 * reference generator (same libstdc++/glibc algorithms). */
typedef struct EconoLengthDist {
  double mean;
  int64_t min_value;
  int64_t max_value;
  double sigma;
} EconoLengthDist;
int econo_generate_trace(int64_t n, double arrival_rate, const EconoLengthDist* prompt,
                         const EconoLengthDist* rl, uint64_t seed, EconoTraceRecord* out,
                         char* err, size_t errlen);

/* ---- wire formats either side of the path (host; wire.cpp) --------------- */
/* load_trace_csv (workload.hpp:142-194): same header check, validation order
 * and messages ("<name>: line N: ..."). Two-call pattern: out = NULL counts. */
int econo_parse_trace_csv(const char* text, int64_t len, const char* name, EconoTraceRecord* out, int64_t cap,
                          int64_t* n, char* err, size_t errlen);
int econo_load_trace_csv(const char* path, EconoTraceRecord* out, int64_t cap, int64_t* n, char* err,
                         size_t errlen);
/* write_trace_csv (workload.hpp:127-134), "%.17g" arrivals; *len = bytes
 * needed (out, when non-NULL, receives min(len, cap-1) bytes + NUL). */
int econo_write_trace_csv(const EconoTraceRecord* trace, int64_t n, char* out, int64_t cap, int64_t* len);
/* FNV-1a over write_trace_csv's bytes (metrics.hpp:320-328, the report's trace_hash). */
uint64_t econo_trace_hash(const EconoTraceRecord* trace, int64_t n);
/* to_json(report, with_records).dump(indent) (metrics.hpp:181-240), byte for
 * byte as nlohmann::ordered_json prints it; recs = NULL omits "records";
 * config_json (NULL: none) is the report's "config" echo (config.hpp:236-285)
 * already serialised for nesting depth 1; indent < 0 = compact. */
int econo_report_to_json(const char* policy, const EconoReport* report, const EconoRecord* recs, int64_t n_recs,
                         const char* config_json, int32_t indent, char* out, int64_t cap, int64_t* len);
/* nlohmann's double printer alone (Grisu2 digits + its layout rules). */
int econo_json_double(double v, char* out, int64_t cap, int64_t* len);

#ifdef __cplusplus
}
#endif

#endif /* ECONOSERVE_B200_H */
