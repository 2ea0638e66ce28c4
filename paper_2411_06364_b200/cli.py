"""`econosim`-style command line over the device engine (tools/econosim.cpp):
run / sweep / gen-trace / compare, exit codes 0 ok, 2 config error, 3
simulation error (econosim.cpp:20-22, 183-192). EconoServe policies only.

    python -m paper_2411_06364_b200 run -c cfg.json [-o outdir]
"""
import argparse
import json
import os
import sys

from . import experiment as X
from . import wire
from .engine import ConfigError, SimulationError, generate_trace

EXIT_OK, EXIT_CONFIG, EXIT_SIM = 0, 2, 3


def _write(path, text):  # write_file (econosim.cpp:24-29)
    d = os.path.dirname(path)
    if d:
        os.makedirs(d, exist_ok=True)
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError:
        raise ConfigError(f"cannot open output file: {path}") from None


def cmd_run(config, output=None):  # econosim.cpp:31-48
    cfg = X.apply_seed_override(X.load_config(config))
    if output:
        cfg["output_dir"] = output
    res = X.run_experiment(cfg)
    for pol, r in res.items():
        path = os.path.join(cfg["output_dir"], f"report_{pol}.json")
        _write(path, X.report_json(cfg, r, indent=2) + "\n")
        rep = r.report
        print(f"{pol}: mean_jct={rep.mean_jct:g}s ssr={rep.ssr:g} throughput={rep.throughput_rps:g} req/s -> {path}")
    if len(res) >= 2:
        print("\n" + X.render_table(res, cfg["policies"][0]), end="")
    return EXIT_OK


def cmd_sweep(config, out_csv=None):  # econosim.cpp:50-62
    cfg = X.apply_seed_override(X.load_config(config))
    axes, cells = X.run_sweep(cfg)
    path = out_csv or os.path.join(cfg["output_dir"], "sweep.csv")
    _write(path, X.write_sweep_csv(axes, cells))
    print(f"{len(cells)} cells x {len(cfg['policies'])} policies -> {path}")
    return EXIT_OK


def cmd_gen_trace(spec_path, out_path):  # econosim.cpp:64-96
    try:
        with open(spec_path) as f:
            j = json.load(f)
    except OSError:
        raise ConfigError(f"cannot open spec file: {spec_path}") from None
    except ValueError as ex:
        raise ConfigError(f"spec parse error: {ex}") from None
    if "trace" in j:
        cfg = X.apply_seed_override(X.parse_config(j))
        if cfg["synthetic"] is None:
            raise ConfigError("gen-trace config has no trace.synthetic block")
        s = cfg["synthetic"]
    else:
        X._check_keys(j, {"n_requests", "arrival_rate", "prompt", "response", "seed"}, "spec")
        s = {"n_requests": X._get(j, "n_requests", 1000, int), "arrival_rate": X._get(j, "arrival_rate", 1.0, float),
             "seed": X._get(j, "seed", 1, int), "prompt": X._dist(19.31, 9, 2470, 0.8),
             "response": X._dist(58.41, 13, 292, 0.8)}
        if "prompt" in j:
            s["prompt"] = X._length_dist(j["prompt"], "prompt", X._dist(32.0, 1, 1024, 0.8))
        if "response" in j:
            s["response"] = X._length_dist(j["response"], "response", X._dist(32.0, 1, 1024, 0.8))
        env = os.environ.get("ECONOSIM_SEED")
        if env:
            s["seed"] = int(env)
    d = lambda x: (x["mean"], x["min"], x["max"], x["sigma"])  # noqa: E731
    t = generate_trace(s["n_requests"], s["arrival_rate"], d(s["prompt"]), d(s["response"]), s["seed"])
    _write(out_path, wire.write_trace_csv(t))
    print(f"{len(t)} records -> {out_path}")
    return EXIT_OK


def main(argv=None):
    ap = argparse.ArgumentParser(prog="econosim-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("-c", "--config", required=True)
    r.add_argument("-o", "--output", default="")
    s = sub.add_parser("sweep")
    s.add_argument("-c", "--config", required=True)
    s.add_argument("-o", "--output", default="")
    g = sub.add_parser("gen-trace")
    g.add_argument("-s", "--spec", required=True)
    g.add_argument("-o", "--output", required=True)
    a = ap.parse_args(argv)
    try:
        if a.cmd == "run":
            return cmd_run(a.config, a.output or None)
        if a.cmd == "sweep":
            return cmd_sweep(a.config, a.output or None)
        return cmd_gen_trace(a.spec, a.output)
    except ConfigError as ex:
        print(f"config error: {ex}", file=sys.stderr)
        return EXIT_CONFIG
    except SimulationError as ex:
        print(f"simulation error: {ex}", file=sys.stderr)
        return EXIT_SIM
