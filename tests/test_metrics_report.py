"""On-device aggregate() for many instances (econo_batch_reports) and exact
JCT percentiles by radix select (econo_batch_jct_percentiles, metrics.py
global_percentiles) against the oracle's report (metrics.hpp:96-175).
percentile() (metrics.hpp:81-89) is reproduced bit-exactly from exact order
statistics; reordered per-request sums are the 1e-6 tier."""
import numpy as np
import pytest

from conftest import HOSTSIM
from oracle import port
from paper_2411_06364_b200 import abi, metrics, workloads as W

FLOAT_KEYS = ["mean_jct", "mean_tbt", "ssr", "normalized_latency", "throughput_rps", "throughput_tps",
              "goodput_rps", "mean_kvc_written", "mean_kvc_allocated", "mean_forward_size",
              "tfs_hit_frac", "pt_admit_frac", "mean_waiting", "mean_execution", "mean_preemption",
              "mean_scheduling", "makespan", "allocation_failure_pct"]
INT_KEYS = ["iterations", "preemptions", "reserve_draws", "hosted_slots", "hosted_overruns"]


def _opts(pm="bucket"):
    c = W.CONFIGS["cfg1_alpaca_10k"]
    extra = dict(pred_accuracy=0.775, pred_tolerance=0.1) if pm == "bucket" else dict(pred_sigma=0.3)
    o = abi.default_options(**dict(c["opts"], pred_model=pm, **extra))
    o.record_events = 0
    o.record_samples = 0
    return o


def _traces(sizes, seed0):
    c = W.CONFIGS["cfg1_alpaca_10k"]
    return [port.generate_trace(n, 150.0, c["shape"]["prompt"], c["shape"]["rl"], seed0 + i)
            for i, n in enumerate(sizes)]


def ref_percentile(v, q):
    """detail::percentile (metrics.hpp:81-89)."""
    v = sorted(v)
    rank = q * float(len(v) - 1)
    lo = int(rank)
    hi = min(lo + 1, len(v) - 1)
    frac = rank - float(lo)
    return v[lo] * (1.0 - frac) + v[hi] * frac


def _batch(backend, traces, o):
    from paper_2411_06364_b200.engine import Batch
    b = Batch(traces, o, lib=HOSTSIM) if backend == "hostsim" else Batch(traces, o, device=0)
    b.launch(1 << 40)
    b.sync()
    return b


BACK = ["hostsim", pytest.param("device", marks=pytest.mark.gpu)]


@pytest.mark.parametrize("backend", BACK)
@pytest.mark.parametrize("pm", ["bucket", "lognormal"])
def test_batch_reports_match_oracle(backend, pm):
    traces = _traces([1, 2, 37, 600, 2500], 70)
    o = _opts(pm)
    b = _batch(backend, traces, o)
    reps = b.reports()
    pct = b.jct_percentiles([0.05, 0.95, 0.5])
    for i, t in enumerate(traces):
        recs, rep = port.OracleEngine(t, o).run()
        want = rep.as_dict()
        got = reps[i].as_dict()
        assert got["p5_jct"] == want["p5_jct"] and got["p95_jct"] == want["p95_jct"], i
        assert pct[i, 0] == want["p5_jct"] and pct[i, 1] == want["p95_jct"]
        jct = recs["completion_time"] - recs["arrival"]
        assert pct[i, 2] == ref_percentile(list(jct), 0.5)
        for k in FLOAT_KEYS:
            assert abs(got[k] - want[k]) <= 1e-6 * max(1.0, abs(want[k])), (i, k, got[k], want[k])
        for k in INT_KEYS:
            assert got[k] == want[k], (i, k)
        hg, hw = got["iteration_completion_histogram"], want["iteration_completion_histogram"]
        assert sorted(hg) == sorted(hw)
        for c in hw:
            assert abs(hg[c] - hw[c]) <= 1e-12, c


@pytest.mark.parametrize("backend", BACK)
def test_global_percentiles_exact(backend):
    traces = _traces([900, 1300, 250, 4000], 90)
    o = _opts()
    b = _batch(backend, traces, o)
    allj = []
    for t in traces:
        recs, _ = port.OracleEngine(t, o).run()
        allj += list(recs["completion_time"] - recs["arrival"])
    qs = [0.0, 0.05, 0.5, 0.95, 1.0]
    got = metrics.global_percentiles(b, qs)
    want = [ref_percentile(allj, q) for q in qs]
    assert got == want


@pytest.mark.gpu
def test_percentiles_without_key_buffer(monkeypatch):
    """A batch that fills the GPU has no room for the 8 B/request key buffer:
    the histogram passes then derive each key from the request's fields.
    Same exact order statistics either way."""
    traces = _traces([900, 1300, 250, 4000], 90)
    o = _opts()
    want_b = _batch("device", traces, o)
    want = metrics.global_percentiles(want_b, [0.0, 0.05, 0.5, 0.95, 1.0])
    want_i = want_b.jct_percentiles([0.05, 0.95])
    monkeypatch.setenv("ECONO_JCT_NO_KEYS", "1")
    b = _batch("device", traces, o)
    assert metrics.global_percentiles(b, [0.0, 0.05, 0.5, 0.95, 1.0]) == want
    assert np.array_equal(b.jct_percentiles([0.05, 0.95]), want_i)
