"""ctypes mirror of include/econoserve_b200.h (the C-ABI drop-in boundary).

Field-for-field with the header; the header cites the reference structs each
one mirrors (econosim::TraceRecord workload.hpp:15-21, EngineOptions
engine.hpp:68-77, Event engine.hpp:53-61, IterationSample metrics.hpp:37-48,
RequestRecord metrics.hpp:17-35, MetricsReport metrics.hpp:50-76).
"""
import ctypes as C

import numpy as np

OK, ECONFIG, ESIM, ECUDA = 0, 2, 3, 4

POLICIES = {
    "orca": 0, "vllm": 1, "sarathi": 2, "multires": 3, "sync-coupled": 4,
    "econoserve-d": 5, "econoserve-sd": 6, "econoserve-sdo": 7, "econoserve-full": 8,
}
POLICY_NAMES = {v: k for k, v in POLICIES.items()}
PRED_MODELS = {"oracle": 0, "lognormal": 1, "bucket": 2}

EV_KINDS = ["arrive", "gt_schedule", "hosted", "pt_dispatch", "prefill_done", "complete",
            "reserve_topup", "preempt", "hosted_overrun", "idle", "alloc_fail", "preempt_swap", "swap_in"]
MAX_BOUNDS = 8
MAX_HIST = 256
PARTIAL_WORDS = 32
DEBUG_WORDS = 16  # ECONO_DEBUG_WORDS


class TraceRecord(C.Structure):
    _fields_ = [("arrival_time", C.c_double), ("prompt_len", C.c_int64), ("true_rl", C.c_int64)]


TRACE_DTYPE = np.dtype([("arrival_time", "<f8"), ("prompt_len", "<i8"), ("true_rl", "<i8")])


class Options(C.Structure):
    _fields_ = [
        ("policy", C.c_int32), ("batch_size_cap", C.c_int32), ("tfs", C.c_int64),
        ("chunk_size", C.c_int64), ("padding_ratio", C.c_double),
        ("reserved_fraction", C.c_double), ("buffer_ratio", C.c_double),
        ("max_output_len", C.c_int64), ("vllm_recompute", C.c_int32), ("_pad0", C.c_int32),
        ("t_base", C.c_double), ("t_token", C.c_double), ("t_token_over", C.c_double),
        ("cost_tfs", C.c_int64), ("preempt_offload_penalty", C.c_double),
        ("preempt_free_penalty", C.c_double), ("reserve_penalty", C.c_double),
        ("sched_cost_per_exam", C.c_double), ("swap_stall", C.c_double),
        ("pred_model", C.c_int32), ("_pad1", C.c_int32), ("pred_sigma", C.c_double),
        ("pred_accuracy", C.c_double), ("pred_tolerance", C.c_double),
        ("pred_padding_ratio", C.c_double), ("pred_quantum", C.c_int64),
        ("pred_seed", C.c_uint64),
        ("n_deadline_bounds", C.c_int32), ("n_kvc_bounds", C.c_int32),
        ("n_length_bounds", C.c_int32), ("_pad2", C.c_int32),
        ("deadline_bounds", C.c_double * MAX_BOUNDS), ("kvc_bounds", C.c_int64 * MAX_BOUNDS),
        ("length_bounds", C.c_int64 * MAX_BOUNDS),
        ("kvc_capacity", C.c_int64), ("kvc_block_size", C.c_int64),
        ("slo_scale", C.c_double), ("seed", C.c_uint64),
        ("record_events", C.c_int32), ("record_samples", C.c_int32),
    ]


class Event(C.Structure):
    _fields_ = [("iter", C.c_int64), ("clock", C.c_double), ("kind", C.c_int32),
                ("id", C.c_int32), ("a", C.c_int64), ("b", C.c_int64)]


EVENT_DTYPE = np.dtype([("iter", "<i8"), ("clock", "<f8"), ("kind", "<i4"), ("id", "<i4"),
                        ("a", "<i8"), ("b", "<i8")])


class Sample(C.Structure):
    _fields_ = [("iter", C.c_int64), ("clock", C.c_double), ("dt", C.c_double),
                ("forward_size", C.c_int64), ("kvc_written_frac", C.c_double),
                ("kvc_allocated_frac", C.c_double), ("completed", C.c_int32),
                ("pts_admitted", C.c_int32), ("pt_admittable", C.c_int32), ("_pad", C.c_int32),
                ("idle_repeat", C.c_int64)]


SAMPLE_DTYPE = np.dtype([("iter", "<i8"), ("clock", "<f8"), ("dt", "<f8"),
                         ("forward_size", "<i8"), ("kvc_written_frac", "<f8"),
                         ("kvc_allocated_frac", "<f8"), ("completed", "<i4"),
                         ("pts_admitted", "<i4"), ("pt_admittable", "<i4"), ("_pad", "<i4"),
                         ("idle_repeat", "<i8")])


class Record(C.Structure):
    _fields_ = [("id", C.c_int32), ("preempt_count", C.c_int32), ("arrival", C.c_double),
                ("first_token_time", C.c_double), ("completion_time", C.c_double),
                ("waiting_time", C.c_double), ("execution_time", C.c_double),
                ("preemption_time", C.c_double), ("scheduling_time_share", C.c_double),
                ("reserve_draws", C.c_int32), ("met_slo", C.c_int32),
                ("prompt_len", C.c_int64), ("true_rl", C.c_int64),
                ("slo_deadline", C.c_double), ("alloc_failure", C.c_int32), ("_pad", C.c_int32)]


RECORD_DTYPE = np.dtype([("id", "<i4"), ("preempt_count", "<i4"), ("arrival", "<f8"),
                         ("first_token_time", "<f8"), ("completion_time", "<f8"),
                         ("waiting_time", "<f8"), ("execution_time", "<f8"),
                         ("preemption_time", "<f8"), ("scheduling_time_share", "<f8"),
                         ("reserve_draws", "<i4"), ("met_slo", "<i4"), ("prompt_len", "<i8"),
                         ("true_rl", "<i8"), ("slo_deadline", "<f8"), ("alloc_failure", "<i4"),
                         ("_pad", "<i4")])

REPORT_DOUBLE_FIELDS = [
    "mean_jct", "p5_jct", "p95_jct", "mean_tbt", "ssr", "throughput_rps", "throughput_tps",
    "goodput_rps", "normalized_latency", "mean_kvc_written", "mean_kvc_allocated",
    "mean_forward_size", "allocation_failure_pct", "tfs_hit_frac", "pt_admit_frac"]


class Report(C.Structure):
    _fields_ = ([(f, C.c_double) for f in REPORT_DOUBLE_FIELDS] +
                [("iterations", C.c_int64), ("makespan", C.c_double),
                 ("preemptions", C.c_int64), ("reserve_draws", C.c_int64),
                 ("hosted_slots", C.c_int64), ("hosted_overruns", C.c_int64),
                 ("mean_waiting", C.c_double), ("mean_execution", C.c_double),
                 ("mean_preemption", C.c_double), ("mean_scheduling", C.c_double),
                 ("trace_hash", C.c_uint64), ("n_hist", C.c_int32), ("_pad", C.c_int32),
                 ("hist_count", C.c_int32 * MAX_HIST), ("hist_frac", C.c_double * MAX_HIST)])

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_
             if f not in ("_pad", "hist_count", "hist_frac", "n_hist")}
        d["iteration_completion_histogram"] = {
            int(self.hist_count[i]): float(self.hist_frac[i]) for i in range(self.n_hist)}
        return d


class Scalars(C.Structure):
    _fields_ = [("clock", C.c_double), ("iter", C.c_int64), ("completed", C.c_int64),
                ("steps", C.c_int64), ("executed_iters", C.c_int64),
                ("hosted_slots_created", C.c_int64), ("hosted_overruns", C.c_int64),
                ("calibrated_prefill_time", C.c_double), ("calibrated_decode_time", C.c_double),
                ("pt_dispatched", C.c_int64), ("gt_scheduled", C.c_int64),
                ("pt_queue_len", C.c_int64), ("gt_queue_groups", C.c_int64),
                ("running", C.c_int64), ("arrived", C.c_int64), ("done", C.c_int32),
                ("error", C.c_int32), ("quiet_steps", C.c_int64), ("quiet_spans", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class LengthDist(C.Structure):
    _fields_ = [("mean", C.c_double), ("min_value", C.c_int64), ("max_value", C.c_int64),
                ("sigma", C.c_double)]


def default_options(policy="econoserve-full", **kw):
    """A default-constructed econosim::EngineOptions (engine.hpp:68-77,
    policies.hpp:65-74, engine.hpp:21-33, workload.hpp:202-210, queues.hpp:16-20,
    engine.hpp:63-66) with keyword overrides."""
    o = Options()
    o.policy = POLICIES[policy] if isinstance(policy, str) else int(policy)
    o.batch_size_cap = 8
    o.tfs = 2048
    o.chunk_size = 512
    o.padding_ratio = 0.10
    o.reserved_fraction = 0.03
    o.buffer_ratio = 0.15
    o.max_output_len = 0
    o.vllm_recompute = 0
    o.t_base = 0.005
    o.t_token = 1e-4
    o.t_token_over = -1.0
    o.cost_tfs = 2048
    o.preempt_offload_penalty = 0.30
    o.preempt_free_penalty = 0.06
    o.reserve_penalty = 0.004
    o.sched_cost_per_exam = 2e-5
    o.swap_stall = 0.088
    o.pred_model = 0
    o.pred_sigma = 0.0
    o.pred_accuracy = 1.0
    o.pred_tolerance = 0.1
    o.pred_padding_ratio = 0.0
    o.pred_quantum = 1
    o.pred_seed = 1
    o.n_deadline_bounds = 3
    for i, v in enumerate((0.2, 0.5, 2.0)):
        o.deadline_bounds[i] = v
    o.n_kvc_bounds = 4
    o.n_length_bounds = 4
    for i, v in enumerate((128, 256, 384, 512)):
        o.kvc_bounds[i] = v
        o.length_bounds[i] = v
    o.kvc_capacity = 32768
    o.kvc_block_size = 32
    o.slo_scale = 2.0
    o.seed = 1
    o.record_events = 1
    o.record_samples = 1
    for k, v in kw.items():
        set_option(o, k, v)
    return o


def set_option(o, k, v):
    if k == "policy":
        o.policy = POLICIES[v] if isinstance(v, str) else int(v)
    elif k == "pred_model":
        o.pred_model = PRED_MODELS[v] if isinstance(v, str) else int(v)
    elif k in ("deadline_bounds", "kvc_bounds", "length_bounds"):
        arr = getattr(o, k)
        for i, x in enumerate(v):
            arr[i] = x
        setattr(o, "n_" + k, len(v))
    else:
        setattr(o, k, v)


def copy_options(o):
    c = Options()
    C.memmove(C.byref(c), C.byref(o), C.sizeof(Options))
    return c


class TraceSoA(C.Structure):
    """EconoTraceSoA: a trace as three arrays (include/econoserve_b200.h)."""
    _fields_ = [("arrival_time", C.c_void_p), ("prompt_len", C.c_void_p), ("true_rl", C.c_void_p)]


class SoaTrace:
    """A trace held as three contiguous columns — arrival_time f64, prompt_len
    i32, true_rl i32 — the instance's device layout (econo_batch_create_soa
    copies them into HBM as they are: 16 B per request). `out`: optional
    preallocated (e.g. page-locked) column buffers."""

    def __init__(self, arrival, prompt, true_rl):
        self.arrival = np.ascontiguousarray(arrival, dtype=np.float64)
        self.prompt = np.ascontiguousarray(prompt, dtype=np.int32)
        self.true_rl = np.ascontiguousarray(true_rl, dtype=np.int32)
        assert len(self.arrival) == len(self.prompt) == len(self.true_rl)

    @classmethod
    def from_records(cls, trace, out=None):
        t = trace_array(trace)
        if out is None:
            return cls(t["arrival_time"], t["prompt_len"].astype(np.int32), t["true_rl"].astype(np.int32))
        a, p, r = out
        a[:] = t["arrival_time"]
        p[:] = t["prompt_len"]
        r[:] = t["true_rl"]
        return cls(a, p, r)

    def records(self):
        t = np.zeros(len(self), dtype=TRACE_DTYPE)
        t["arrival_time"], t["prompt_len"], t["true_rl"] = self.arrival, self.prompt, self.true_rl
        return t

    def __len__(self):
        return len(self.arrival)

    def struct(self):
        return TraceSoA(self.arrival.ctypes.data, self.prompt.ctypes.data, self.true_rl.ctypes.data)


def trace_array(trace):
    """Accepts a structured numpy array, a list of (arrival, prompt, rl) tuples,
    or three columns; returns a contiguous TRACE_DTYPE array."""
    if isinstance(trace, np.ndarray) and trace.dtype == TRACE_DTYPE:
        return np.ascontiguousarray(trace)
    arr = np.zeros(len(trace), dtype=TRACE_DTYPE)
    for i, (a, p, r) in enumerate(trace):
        arr[i] = (a, p, r)
    return arr


def event_str(ev):
    """Renders an event row as the reference's (kind, detail) pair (engine.hpp:211-214)."""
    k = int(ev["kind"])
    name = EV_KINDS[k]
    a, b = int(ev["a"]), int(ev["b"])
    if k in (1, 5):
        d = f"rl={a}"
    elif k == 2:
        d = f"host={a} deadline={b}"
    elif k == 4:
        d = "" if a == 1 else "to-gt-queue"
    elif k == 7:
        d = ("overrun" if a == 1 else "underprediction") + f" l_new={b}"
    elif k == 9:
        d = str(a)
    elif k == 11:
        d = f"written={a}"
    else:
        d = ""
    return name, d
