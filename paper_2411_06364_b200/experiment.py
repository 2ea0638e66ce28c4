"""Experiment and sweep orchestration over the device engine (SURVEY.md §8(f)
row 4): the reference's JSON experiment config (config.hpp:20-330), its sweep
(sweep.hpp:15-168) and the report / comparison outputs (metrics.hpp:181-318),
with every (sweep cell, policy) pair run as one instance of a single device
batch instead of one engine per worker thread.

Scope: every policy of the reference — the EconoServe family and the five
baselines (orca, vllm, sarathi, multires, sync-coupled) — runs on the device.
Engine failures surface as the reference's SimulationError with the engine's
own message (e.g. "simulation stuck"), config problems as ConfigError.
"""
import copy
import ctypes as C
import json
import os

import numpy as np

from . import abi, wire
from .engine import ConfigError, Engine, _raise, generate_trace, load

POLICY_NAMES = ["orca", "vllm", "sarathi", "multires", "sync-coupled", "econoserve-d", "econoserve-sd",
                "econoserve-sdo", "econoserve-full"]
AXES = ["padding_ratio", "reserved_fraction", "buffer_ratio", "arrival_rate", "slo_scale"]  # sweep.hpp:22-23
SWEEP_METRICS = ["mean_jct", "p5_jct", "p95_jct", "mean_tbt", "ssr", "throughput_rps", "throughput_tps",
                 "goodput_rps", "normalized_latency", "mean_kvc_written", "mean_kvc_allocated",
                 "mean_forward_size", "allocation_failure_pct", "preemptions", "reserve_draws", "hosted_overruns",
                 "mean_waiting", "mean_execution", "mean_preemption", "mean_scheduling"]  # sweep.hpp:70-78
COMPARISON_METRICS = ["mean_jct", "p95_jct", "mean_tbt", "ssr", "throughput_rps", "throughput_tps", "goodput_rps",
                      "normalized_latency", "mean_kvc_written", "mean_forward_size",
                      "allocation_failure_pct"]  # metrics.hpp:243-258


def _dist(mean, lo, hi, sigma):
    return {"mean": float(mean), "min": int(lo), "max": int(hi), "sigma": float(sigma)}


def default_config():
    """default_config() (config.hpp:86-94) with its synthetic trace reset, as
    parse_config starts from (config.hpp:98-99)."""
    return {
        "trace_file": None, "synthetic": None, "policies": ["econoserve-full", "vllm"],
        "kvc": {"capacity": 32768, "block_size": 32},
        "cost": {"t_base": 0.005, "t_token": 1e-4, "t_token_over": -1.0, "preempt_offload_penalty": 0.30,
                 "preempt_free_penalty": 0.06, "reserve_penalty": 0.004, "sched_cost_per_exam": 2e-5,
                 "swap_stall": 0.088},
        "predictor": {"model": "oracle", "sigma": 0.0, "accuracy": 1.0, "tolerance": 0.1, "padding_ratio": 0.0,
                      "quantum": 1, "seed": 1},
        "policy_params": {"tfs": 2048, "batch_size_cap": 8, "chunk_size": 512, "reserved_fraction": 0.03,
                          "buffer_ratio": 0.15, "max_output_len": 0, "vllm_recompute": False},
        "ordering": {"deadline_bounds": [0.2, 0.5, 2.0], "kvc_bounds": [128, 256, 384, 512],
                     "length_bounds": [128, 256, 384, 512]},
        "slo_scale": 2.0, "seed": 1, "output_dir": "out", "jobs": 0, "sweep": {},
    }


def _check_keys(j, allowed, where):  # config.hpp:64-69
    if not isinstance(j, dict):
        raise ConfigError(f"{where} must be an object")
    for k in j:
        if k not in allowed:
            raise ConfigError(f"unknown key '{k}' in {where}")


def _get(j, key, default, kind):
    if key not in j:
        return default
    v = j[key]
    try:
        if kind is bool:
            if not isinstance(v, bool):
                raise TypeError
            return v
        if kind is str:
            if not isinstance(v, str):
                raise TypeError
            return v
        if isinstance(v, bool) or not isinstance(v, (int, float)):
            raise TypeError
        return kind(v)
    except (TypeError, ValueError):
        raise ConfigError(f"config value '{key}' has the wrong type") from None


def _length_dist(j, where, d):  # config.hpp:71-79
    _check_keys(j, {"mean", "min", "max", "sigma"}, where)
    return {"mean": _get(j, "mean", d["mean"], float), "min": _get(j, "min", d["min"], int),
            "max": _get(j, "max", d["max"], int), "sigma": _get(j, "sigma", d["sigma"], float)}


def parse_config(j):
    """parse_config (config.hpp:96-217): strict keys, the same defaults and
    the same validation order and messages (ExperimentConfig::validate,
    config.hpp:35-58)."""
    cfg = default_config()
    _check_keys(j, {"trace", "policies", "kvc", "cost", "predictor", "policy_params", "ordering", "slo_scale",
                    "seed", "output_dir", "jobs", "sweep"}, "config")
    cfg["seed"] = _get(j, "seed", cfg["seed"], int)
    cfg["slo_scale"] = _get(j, "slo_scale", cfg["slo_scale"], float)
    cfg["output_dir"] = _get(j, "output_dir", cfg["output_dir"], str)
    cfg["jobs"] = _get(j, "jobs", cfg["jobs"], int)
    if "policies" in j:
        if not isinstance(j["policies"], list) or not all(isinstance(p, str) for p in j["policies"]):
            raise ConfigError("config value 'policies' has the wrong type")
        cfg["policies"] = list(j["policies"])
    if "trace" in j:
        t = j["trace"]
        _check_keys(t, {"file", "synthetic"}, "trace")
        if "file" in t:
            cfg["trace_file"] = _get(t, "file", None, str)
        if "synthetic" in t:
            s = t["synthetic"]
            _check_keys(s, {"n_requests", "arrival_rate", "prompt", "response", "seed"}, "trace.synthetic")
            spec = {"n_requests": _get(s, "n_requests", 1000, int), "arrival_rate": _get(s, "arrival_rate", 1.0, float),
                    "seed": _get(s, "seed", cfg["seed"], int),
                    "prompt": _dist(19.31, 9, 2470, 0.8), "response": _dist(58.41, 13, 292, 0.8)}
            if "prompt" in s:
                spec["prompt"] = _length_dist(s["prompt"], "trace.synthetic.prompt", _dist(32.0, 1, 1024, 0.8))
            if "response" in s:
                spec["response"] = _length_dist(s["response"], "trace.synthetic.response", _dist(32.0, 1, 1024, 0.8))
            cfg["synthetic"] = spec
    if "kvc" in j:
        k = j["kvc"]
        _check_keys(k, {"capacity", "block_size"}, "kvc")
        cfg["kvc"] = {"capacity": _get(k, "capacity", cfg["kvc"]["capacity"], int),
                      "block_size": _get(k, "block_size", cfg["kvc"]["block_size"], int)}
    if "cost" in j:
        c = j["cost"]
        keys = list(cfg["cost"])
        _check_keys(c, set(keys), "cost")
        cfg["cost"] = {key: _get(c, key, cfg["cost"][key], float) for key in keys}
    if "predictor" in j:
        p = j["predictor"]
        _check_keys(p, {"model", "sigma", "accuracy", "tolerance", "padding_ratio", "quantum", "seed"}, "predictor")
        m = _get(p, "model", "oracle", str)
        if m not in ("oracle", "lognormal", "bucket"):
            raise ConfigError(f"unknown predictor model '{m}'; valid: oracle, lognormal, bucket")
        d = cfg["predictor"]
        cfg["predictor"] = {"model": m, "sigma": _get(p, "sigma", d["sigma"], float),
                            "accuracy": _get(p, "accuracy", d["accuracy"], float),
                            "tolerance": _get(p, "tolerance", d["tolerance"], float),
                            "padding_ratio": _get(p, "padding_ratio", d["padding_ratio"], float),
                            "quantum": _get(p, "quantum", d["quantum"], int), "seed": _get(p, "seed", cfg["seed"], int)}
    else:
        cfg["predictor"]["seed"] = cfg["seed"]
    if "policy_params" in j:
        p = j["policy_params"]
        d = cfg["policy_params"]
        _check_keys(p, set(d), "policy_params")
        cfg["policy_params"] = {"tfs": _get(p, "tfs", d["tfs"], int),
                                "batch_size_cap": _get(p, "batch_size_cap", d["batch_size_cap"], int),
                                "chunk_size": _get(p, "chunk_size", d["chunk_size"], int),
                                "reserved_fraction": _get(p, "reserved_fraction", d["reserved_fraction"], float),
                                "buffer_ratio": _get(p, "buffer_ratio", d["buffer_ratio"], float),
                                "max_output_len": _get(p, "max_output_len", d["max_output_len"], int),
                                "vllm_recompute": _get(p, "vllm_recompute", d["vllm_recompute"], bool)}
    if "ordering" in j:
        o = j["ordering"]
        _check_keys(o, {"deadline_bounds", "kvc_bounds", "length_bounds"}, "ordering")
        for key, kind in (("deadline_bounds", float), ("kvc_bounds", int), ("length_bounds", int)):
            if key in o:
                if not isinstance(o[key], list):
                    raise ConfigError(f"config value '{key}' has the wrong type")
                cfg["ordering"][key] = [kind(v) for v in o[key]]
    if "sweep" in j:
        for axis, values in j["sweep"].items():
            if not isinstance(values, list):
                raise ConfigError(f"config value '{axis}' has the wrong type")
            cfg["sweep"][axis] = [float(v) for v in values]
    validate(cfg)
    return cfg


def validate(cfg):
    """ExperimentConfig::validate (config.hpp:35-58) and the validators it calls."""
    if not cfg["policies"]:
        raise ConfigError("at least one policy is required")
    for p in cfg["policies"]:
        if p not in POLICY_NAMES:
            raise ConfigError(f"unknown policy '{p}'; valid policies: " + ", ".join(POLICY_NAMES))
    if cfg["trace_file"] is None and cfg["synthetic"] is None:
        raise ConfigError("a trace source is required: trace.file or trace.synthetic")
    if cfg["trace_file"] is not None and cfg["synthetic"] is not None:
        raise ConfigError("trace.file and trace.synthetic are mutually exclusive")
    if cfg["slo_scale"] <= 0.0:
        raise ConfigError("slo_scale must be > 0")
    pp = cfg["policy_params"]  # PolicyConfig::validate (policies.hpp:76-84); padding from the predictor
    if pp["tfs"] < 1:
        raise ConfigError("tfs must be >= 1")
    if pp["chunk_size"] < 1:
        raise ConfigError("chunk_size must be >= 1")
    if pp["batch_size_cap"] < 1:
        raise ConfigError("batch_size_cap must be >= 1")
    if pp["reserved_fraction"] < 0.0 or pp["reserved_fraction"] >= 1.0:
        raise ConfigError("reserved_fraction must be in [0, 1)")
    if pp["buffer_ratio"] < 0.0:
        raise ConfigError("buffer_ratio must be >= 0")
    c = cfg["cost"]  # CostModel::validate (engine.hpp:36-43)
    if not c["t_base"] > 0.0:
        raise ConfigError("cost model: t_base must be > 0")
    if not c["t_token"] > 0.0:
        raise ConfigError("cost model: t_token must be > 0")
    if min(c["preempt_offload_penalty"], c["preempt_free_penalty"], c["reserve_penalty"], c["sched_cost_per_exam"],
           c["swap_stall"]) < 0.0:
        raise ConfigError("cost model: penalties must be >= 0")
    p = cfg["predictor"]  # PredictorConfig::validate (workload.hpp:211-217)
    if p["sigma"] < 0.0:
        raise ConfigError("predictor sigma must be >= 0")
    if p["accuracy"] < 0.0 or p["accuracy"] > 1.0:
        raise ConfigError("predictor accuracy must be in [0,1]")
    if p["tolerance"] < 0.0:
        raise ConfigError("predictor tolerance must be >= 0")
    if p["padding_ratio"] < 0.0:
        raise ConfigError("padding_ratio must be >= 0")
    if p["quantum"] < 1:
        raise ConfigError("predictor quantum must be >= 1")
    o = cfg["ordering"]  # OrderingConfig::validate (queues.hpp:22-27)
    for key in ("deadline_bounds", "kvc_bounds", "length_bounds"):
        if any(b < a for a, b in zip(o[key], o[key][1:])):
            raise ConfigError("ordering bucket boundaries must be increasing")
    for axis, values in cfg["sweep"].items():
        if axis not in AXES:
            raise ConfigError(f"unknown sweep axis '{axis}'; valid axes: padding_ratio, reserved_fraction, "
                              "buffer_ratio, arrival_rate, slo_scale")
        if not values:
            raise ConfigError(f"sweep axis '{axis}' has an empty value list")
        if axis == "arrival_rate" and cfg["synthetic"] is None:
            raise ConfigError("sweep axis arrival_rate requires a synthetic trace")


def load_config(path):
    """load_config (config.hpp:219-229)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ConfigError(f"cannot open config file: {path}") from None
    try:
        j = json.loads(text)
    except ValueError as ex:
        raise ConfigError(f"config parse error in {path}: {ex}") from None
    return parse_config(j)


def apply_seed_override(cfg, env=None):
    """ECONOSIM_SEED (config.hpp:288-297)."""
    v = (os.environ if env is None else env).get("ECONOSIM_SEED")
    if not v:
        return cfg
    if not v.isdigit():
        raise ConfigError("ECONOSIM_SEED is not an integer")
    cfg = copy.deepcopy(cfg)
    cfg["seed"] = int(v)
    cfg["predictor"]["seed"] = int(v)
    if cfg["synthetic"] is not None:
        cfg["synthetic"]["seed"] = int(v)
    return cfg


def materialize_trace(cfg):
    """materialize_trace (config.hpp:299-302)."""
    if cfg["trace_file"] is not None:
        return wire.load_trace_csv(cfg["trace_file"])
    s = cfg["synthetic"]
    d = lambda x: (x["mean"], x["min"], x["max"], x["sigma"])  # noqa: E731
    return generate_trace(s["n_requests"], s["arrival_rate"], d(s["prompt"]), d(s["response"]), s["seed"])


def engine_options(cfg, policy):
    """engine_options (config.hpp:304-317) as EconoOptions; recording off
    (reports come from the running aggregates)."""
    pp, c, p, o = cfg["policy_params"], cfg["cost"], cfg["predictor"], cfg["ordering"]
    return abi.default_options(
        policy=policy, tfs=pp["tfs"], batch_size_cap=pp["batch_size_cap"], chunk_size=pp["chunk_size"],
        padding_ratio=p["padding_ratio"], reserved_fraction=pp["reserved_fraction"], buffer_ratio=pp["buffer_ratio"],
        max_output_len=pp["max_output_len"], vllm_recompute=int(pp["vllm_recompute"]),
        t_base=c["t_base"], t_token=c["t_token"], t_token_over=c["t_token_over"], cost_tfs=pp["tfs"],
        preempt_offload_penalty=c["preempt_offload_penalty"], preempt_free_penalty=c["preempt_free_penalty"],
        reserve_penalty=c["reserve_penalty"], sched_cost_per_exam=c["sched_cost_per_exam"],
        swap_stall=c["swap_stall"], pred_model=p["model"], pred_sigma=p["sigma"], pred_accuracy=p["accuracy"],
        pred_tolerance=p["tolerance"], pred_padding_ratio=p["padding_ratio"], pred_quantum=p["quantum"],
        pred_seed=p["seed"], deadline_bounds=o["deadline_bounds"], kvc_bounds=o["kvc_bounds"],
        length_bounds=o["length_bounds"], kvc_capacity=cfg["kvc"]["capacity"],
        kvc_block_size=cfg["kvc"]["block_size"], slo_scale=cfg["slo_scale"], seed=cfg["seed"],
        record_events=0, record_samples=0)


# ---- nlohmann::ordered_json-compatible serialisation of the config echo ----
def _dump(v, indent, depth):
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, int):
        return str(v)
    if isinstance(v, float):
        return wire.json_double(v)
    if isinstance(v, str):
        return json.dumps(v, ensure_ascii=False)
    nl = "" if indent < 0 else "\n"
    pad = lambda d: "" if indent < 0 else " " * (indent * d)  # noqa: E731
    if isinstance(v, list):
        if not v:
            return "[]"
        return ("[" + nl + ("," + nl).join(pad(depth + 1) + _dump(x, indent, depth + 1) for x in v) + nl +
                pad(depth) + "]")
    if not v:
        return "{}"
    sep = ":" if indent < 0 else ": "
    return ("{" + nl + ("," + nl).join(pad(depth + 1) + json.dumps(k) + sep + _dump(x, indent, depth + 1)
                                        for k, x in v.items()) + nl + pad(depth) + "}")


def config_echo(cfg):
    """to_json(ExperimentConfig) (config.hpp:236-285), in its key order and types."""
    j = {"seed": int(cfg["seed"]), "slo_scale": float(cfg["slo_scale"]), "output_dir": cfg["output_dir"],
         "jobs": int(cfg["jobs"]), "policies": list(cfg["policies"])}
    trace = {}
    if cfg["trace_file"] is not None:
        trace["file"] = cfg["trace_file"]
    if cfg["synthetic"] is not None:
        s = cfg["synthetic"]
        trace["synthetic"] = {"n_requests": s["n_requests"], "arrival_rate": float(s["arrival_rate"]), "seed": s["seed"],
                              "prompt": s["prompt"], "response": s["response"]}
    j["trace"] = trace
    j["kvc"] = {"capacity": cfg["kvc"]["capacity"], "block_size": cfg["kvc"]["block_size"]}
    j["cost"] = {k: float(v) for k, v in cfg["cost"].items()}
    p = cfg["predictor"]
    j["predictor"] = {"model": p["model"], "sigma": p["sigma"], "accuracy": p["accuracy"], "tolerance": p["tolerance"],
                      "padding_ratio": p["padding_ratio"], "quantum": p["quantum"], "seed": p["seed"]}
    j["policy_params"] = dict(cfg["policy_params"])
    j["ordering"] = {"deadline_bounds": [float(x) for x in cfg["ordering"]["deadline_bounds"]],
                     "kvc_bounds": [int(x) for x in cfg["ordering"]["kvc_bounds"]],
                     "length_bounds": [int(x) for x in cfg["ordering"]["length_bounds"]]}
    if cfg["sweep"]:
        j["sweep"] = {k: [float(x) for x in cfg["sweep"][k]] for k in sorted(cfg["sweep"])}
    return j


def config_json(cfg, indent=-1):
    """The echo serialised for nesting depth 1 of a report (metrics.hpp:220)."""
    return _dump(config_echo(cfg), indent, 1)


# ---- run_experiment / sweep -------------------------------------------------
class Result:
    """One policy's run: the device engine's records and report."""

    def __init__(self, policy, records, report):
        self.policy, self.records, self.report = policy, records, report

    def metric(self, name):
        return float(getattr(self.report, name))


def run_experiment(cfg, device=0, lib=None):
    """run_experiment (config.hpp:320-330): every configured policy on the
    shared trace; {policy: Result} in the reference's std::map order."""
    trace = materialize_trace(cfg)
    out = {}
    for name in cfg["policies"]:
        e = Engine(trace, engine_options(cfg, name), device=device, lib=lib)
        recs, rep = e.run()
        out[name] = Result(name, recs, rep)
    return dict(sorted(out.items()))


def report_json(cfg, result, with_records=True, indent=2, lib=None):
    """to_json(report).dump(indent) with the config echo, as `econosim run`
    writes report_<policy>.json (tools/econosim.cpp:38, plus its trailing newline)."""
    return wire.report_json(result.report, result.records if with_records else None, result.policy, indent,
                            lib=lib, config_json=config_json(cfg, indent))


def expand_sweep(cfg):
    """expand_sweep (sweep.hpp:30-50): cells in canonical axis order, last axis fastest."""
    axes = [a for a in AXES if a in cfg["sweep"]]
    if not axes:
        raise ConfigError("sweep requires at least one sweep axis")
    cells = [[]]
    for a in axes:
        cells = [c + [(a, v)] for c in cells for v in cfg["sweep"][a]]
    return axes, cells


def apply_cell(cfg, cell):
    """apply_cell (sweep.hpp:52-68)."""
    c = copy.deepcopy(cfg)
    c["sweep"] = {}
    for axis, v in cell:
        if axis == "padding_ratio":
            c["predictor"]["padding_ratio"] = v
        elif axis == "reserved_fraction":
            c["policy_params"]["reserved_fraction"] = v
        elif axis == "buffer_ratio":
            c["policy_params"]["buffer_ratio"] = v
        elif axis == "arrival_rate":
            c["synthetic"]["arrival_rate"] = v
        elif axis == "slo_scale":
            c["slo_scale"] = v
    return c


def run_sweep(cfg, device=0, lib=None):
    """run_sweep (sweep.hpp:112-149) as ONE device batch: every (cell, policy)
    pair is an instance, all advanced by the same launches, instead of one
    engine per worker thread. Returns (axes, [(cell, {policy: Result})]) in
    cell order; reports are exact (finalize + aggregate per instance)."""
    from .engine import Batch
    axes, cells = expand_sweep(cfg)
    cell_cfgs = [apply_cell(cfg, c) for c in cells]
    traces, opts, keys = [], [], []
    shared = None if "arrival_rate" in cfg["sweep"] else materialize_trace(cfg)
    for ci, cc in enumerate(cell_cfgs):
        tr = shared if shared is not None else materialize_trace(cc)
        for name in cc["policies"]:
            traces.append(tr)
            opts.append(engine_options(cc, name))
            keys.append((ci, name))
    b = Batch(traces, opts, device=device, lib=lib)
    b.launch(1 << 40)
    b.sync()
    L = b._L
    out = [(c, {}) for c in cells]
    for i, (ci, name) in enumerate(keys):
        v = C.c_void_p()
        L.econo_batch_engine(b.h, i, C.byref(v))
        n = len(traces[i])
        recs = np.zeros(n, dtype=abi.RECORD_DTYPE)
        rep = abi.Report()
        err = C.create_string_buffer(1024)
        rc = L.econo_records(v, recs.ctypes.data, n, err, 1024) or L.econo_report(v, C.byref(rep), err, 1024)
        if rc:  # the engine's own error (SimulationError for a stuck run), not a blanket ConfigError
            _raise(rc, err)
        out[ci][1][name] = Result(name, recs, rep)
    b.close()
    return axes, [(c, dict(sorted(r.items()))) for c, r in out]


def write_sweep_csv(axes, cells):
    """write_sweep_csv (sweep.hpp:152-168): one row per (cell, policy, metric)."""
    rows = ["".join(a + "," for a in axes) + "policy,metric,value\n"]
    for cell, reports in cells:
        prefix = "".join("%.17g," % v for _, v in cell)
        for policy, r in reports.items():
            for m in SWEEP_METRICS:
                rows.append(f"{prefix}{policy},{m},{'%.17g' % r.metric(m)}\n")
    return "".join(rows)


def render_table(results, baseline):
    """compare + render_table (metrics.hpp:268-318) over {policy: Result}."""
    if len(results) < 2:
        raise ConfigError("compare needs at least two reports")
    if baseline not in results:
        raise ConfigError(f"baseline policy '{baseline}' not present")
    h = results[baseline].report.trace_hash
    if any(r.report.trace_hash != h for r in results.values()):
        raise ConfigError("trace hash mismatch: reports were produced from different traces")
    pols = list(results)
    out = "%-24s" % "metric" + "".join(" %16s" % p for p in pols) + " %16s" % ("vs " + baseline) + "\n"
    for m in COMPARISON_METRICS:
        base = results[baseline].metric(m)
        last = results[pols[-1]].metric(m)
        out += "%-24s" % m + "".join(" %16.6g" % results[p].metric(m) for p in pols)
        out += " %15.3fx" % (last / base if base != 0.0 else 0.0) + "\n"
    return out


__all__ = ["parse_config", "load_config", "apply_seed_override", "materialize_trace", "engine_options",
           "run_experiment", "report_json", "config_json", "expand_sweep", "apply_cell", "run_sweep",
           "write_sweep_csv", "render_table"]
_ = load  # the product library is loaded by Engine/Batch
