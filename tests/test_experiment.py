"""Experiment/sweep orchestration against the
compiled reference: config parsing errors, run_experiment's JSON reports with
the config echo (byte for byte), the comparison table, and the sweep CSV — the
sweep run as ONE batch of (cell, policy) instances."""
import json
import re

import pytest

from conftest import HOSTSIM
from oracle import ref
from paper_2411_06364_b200 import experiment as X
from paper_2411_06364_b200.engine import ConfigError

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")

BASE = {
    "trace": {"synthetic": {"n_requests": 250, "arrival_rate": 60.0,
                            "prompt": {"mean": 40, "min": 8, "max": 200, "sigma": 0.6},
                            "response": {"mean": 50, "min": 8, "max": 160, "sigma": 0.6}}},
    "policies": ["econoserve-full", "econoserve-sd"],
    "kvc": {"capacity": 8192, "block_size": 16},
    "predictor": {"model": "lognormal", "sigma": 0.3, "padding_ratio": 0.1},
    "policy_params": {"tfs": 1024, "reserved_fraction": 0.05},
    "seed": 7,
}

BACK = ["hostsim", pytest.param("device", marks=pytest.mark.gpu)]


def stock_nlohmann(text):
    """The json.hpp in this image (cudnn_frontend's copy, the only one here:
    the reference does not vendor its own) is patched to print
    arrays of integers on one line even in pretty mode; stock nlohmann, which
    the product follows, breaks them over lines like every other array."""
    def expand(m):
        ind, key, body, comma = m.group(1), m.group(2), m.group(3), m.group(4)
        items = body.split(",")
        inner = ",\n".join(ind + "  " + x for x in items)
        return f'{ind}"{key}": [\n{inner}\n{ind}]{comma}'
    return re.sub(r'^( *)"(\w+)": \[(-?\d+(?:,-?\d+)*)\](,?)$', expand, text, flags=re.M)


def _lib(backend):
    return HOSTSIM if backend == "hostsim" else None


@pytest.mark.parametrize("backend", BACK)
def test_reports_and_table_match_reference(backend):
    text = json.dumps(BASE)
    cfg = X.parse_config(json.loads(text))
    res = X.run_experiment(cfg, lib=_lib(backend))
    assert list(res) == sorted(BASE["policies"])
    for pol, r in res.items():
        for rec, ind in ((True, 2), (False, -1)):
            want = ref.experiment_report(text, pol, rec, ind)
            assert X.report_json(cfg, r, with_records=rec, indent=ind, lib=_lib(backend)) == \
                (stock_nlohmann(want) if ind >= 0 else want), (pol, rec, ind)
    assert X.render_table(res, "econoserve-full") == ref.render_table(text, "econoserve-full")


@pytest.mark.parametrize("backend", BACK)
def test_sweep_csv_matches_reference(backend):
    j = dict(BASE, sweep={"slo_scale": [1.5, 3.0], "padding_ratio": [0.0, 0.2], "arrival_rate": [40.0, 90.0]})
    text = json.dumps(j)
    axes, cells = X.run_sweep(X.parse_config(json.loads(text)), lib=_lib(backend))
    assert axes == ["padding_ratio", "arrival_rate", "slo_scale"]
    assert len(cells) == 8
    assert X.write_sweep_csv(axes, cells) == ref.sweep_csv(text)


BAD = [
    {"bogus": 1},
    {"trace": {"synthetic": {"n_requests": 10, "nope": 1}}},
    {"trace": {"synthetic": {"prompt": {"mean": 5, "median": 3}}}},
    {"policies": []},
    {"policies": ["econoserve-full", "fifo"]},
    {"policies": ["econoserve-full"]},
    {"policies": ["econoserve-full"], "trace": {"file": "x.csv", "synthetic": {}}},
    {"policies": ["econoserve-full"], "trace": {"synthetic": {}}, "slo_scale": 0},
    {"policies": ["econoserve-full"], "trace": {"synthetic": {}}, "policy_params": {"tfs": 0}},
    {"policies": ["econoserve-full"], "trace": {"synthetic": {}}, "policy_params": {"reserved_fraction": 1.0}},
    {"policies": ["econoserve-full"], "trace": {"synthetic": {}}, "cost": {"t_base": 0}},
    {"policies": ["econoserve-full"], "trace": {"synthetic": {}}, "cost": {"swap_stall": -1}},
    {"policies": ["econoserve-full"], "trace": {"synthetic": {}}, "predictor": {"model": "perfect"}},
    {"policies": ["econoserve-full"], "trace": {"synthetic": {}}, "predictor": {"accuracy": 2}},
    {"policies": ["econoserve-full"], "trace": {"synthetic": {}}, "predictor": {"quantum": 0}},
    {"policies": ["econoserve-full"], "trace": {"synthetic": {}}, "ordering": {"kvc_bounds": [5, 3]}},
    {"policies": ["econoserve-full"], "trace": {"synthetic": {}}, "sweep": {"tfs": [1, 2]}},
    {"policies": ["econoserve-full"], "trace": {"synthetic": {}}, "sweep": {"slo_scale": []}},
    {"policies": ["econoserve-full"], "trace": {"file": "x.csv"}, "sweep": {"arrival_rate": [1.0]}},
]


@pytest.mark.parametrize("k", range(len(BAD)))
def test_config_errors_match_reference(k):
    text = json.dumps(BAD[k])
    want = ref.parse_config_error(text)
    assert want is not None and want[0] == 2, want
    with pytest.raises(ConfigError) as ex:
        X.parse_config(json.loads(text))
    assert str(ex.value) == want[1]


ALL = ["orca", "vllm", "sarathi", "multires", "sync-coupled", "econoserve-d", "econoserve-sd",
       "econoserve-sdo", "econoserve-full"]


@pytest.mark.parametrize("backend", BACK)
def test_every_policy_report_and_table_match_reference(backend):
    """All nine policies in one run (one batch: the baselines run in their own
    kernel), the per-policy JSON reports and the comparison table against
    vllm, the reference's usual baseline (tests/cli_tests.cpp:61-66)."""
    j = dict(BASE, policies=ALL)
    text = json.dumps(j)
    cfg = X.parse_config(json.loads(text))
    res = X.run_experiment(cfg, lib=_lib(backend))
    assert list(res) == sorted(ALL)
    for pol, r in res.items():
        want = ref.experiment_report(text, pol, True, 2)
        assert X.report_json(cfg, r, with_records=True, indent=2, lib=_lib(backend)) == stock_nlohmann(want), pol
    assert X.render_table(res, "vllm") == ref.render_table(text, "vllm")


@pytest.mark.parametrize("backend", BACK)
def test_sweep_with_baselines_matches_reference(backend):
    j = dict(BASE, policies=["vllm", "sarathi", "econoserve-full"],
             sweep={"padding_ratio": [0.0, 0.2], "arrival_rate": [40.0, 90.0]})
    text = json.dumps(j)
    axes, cells = X.run_sweep(X.parse_config(json.loads(text)), lib=_lib(backend))
    assert X.write_sweep_csv(axes, cells) == ref.sweep_csv(text)
