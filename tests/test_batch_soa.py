"""econo_batch_create_soa: a batch created from traces given as three arrays
(abi.SoaTrace: arrival f64, prompt i32, true_rl i32 — the device layout, 16 B
per request copied straight into HBM) is the batch econo_batch_create builds
from the same traces as records (workload.hpp:20-24): identical snapshots
after construction and after steps, identical errors for bad input. The host
build (tests/_hostsim) runs on CPU; the device build under -m gpu."""
import numpy as np
import pytest

from conftest import HOSTSIM
from oracle import port
from paper_2411_06364_b200 import abi, workloads as W
from paper_2411_06364_b200.engine import Batch, ConfigError

BACKENDS = ["hostsim", pytest.param("device", marks=pytest.mark.gpu)]


def _lib(backend):
    return HOSTSIM if backend == "hostsim" else None


def _opts(policy="econoserve-full", **kw):
    c = W.CONFIGS["cfg1_alpaca_10k"]
    o = abi.default_options(**dict(c["opts"], policy=policy, **kw))
    o.record_events = 0
    o.record_samples = 0
    return o


def _traces(k=3, n=1500):
    c = W.CONFIGS["cfg1_alpaca_10k"]
    return [port.generate_trace(n + 37 * i, 40.0, c["shape"]["prompt"], c["shape"]["rl"], 300 + i) for i in range(k)]


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("policy", ["econoserve-full", "econoserve-d", "orca", "vllm"])
def test_soa_batch_equals_record_batch(backend, policy):
    traces = _traces()
    o = _opts(policy, max_output_len=0) if policy == "orca" else _opts(policy)
    a = Batch(traces, o, device=0, lib=_lib(backend))
    b = Batch([abi.SoaTrace.from_records(t) for t in traces], o, device=0, lib=_lib(backend))
    for i in range(len(traces)):
        assert np.array_equal(a.snapshot(i), b.snapshot(i)), f"instance {i} after construction"
    for _ in range(3):
        a.launch(250)
        b.launch(250)
        a.sync()
        b.sync()
        for i in range(len(traces)):
            assert np.array_equal(a.snapshot(i), b.snapshot(i)), f"instance {i}"
    a.close()
    b.close()


@pytest.mark.parametrize("backend", BACKENDS)
def test_soa_batch_matches_oracle(backend):
    traces = _traces(2, 2000)
    o = _opts()
    b = Batch([abi.SoaTrace.from_records(t) for t in traces], o, device=0, lib=_lib(backend))
    oracles = [port.OracleEngine(t, o) for t in traces]
    for _ in range(4):
        b.launch(300)
        b.sync()
        for i, e in enumerate(oracles):
            e.step(300)
            assert np.array_equal(b.snapshot(i), e.snapshot()), f"instance {i}"
    b.close()


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("field,value", [("prompt", 0), ("true_rl", -3), ("prompt", 1 << 30)])
def test_soa_batch_rejects_bad_lengths_like_records(backend, field, value):
    traces = _traces(2, 800)
    traces[1][{"prompt": "prompt_len", "true_rl": "true_rl"}[field]][417] = value
    o = _opts()
    msgs = []
    for make in (lambda ts: ts, lambda ts: [abi.SoaTrace.from_records(t) for t in ts]):
        with pytest.raises(ConfigError) as ei:
            Batch(make(traces), o, device=0, lib=_lib(backend))
        msgs.append(str(ei.value))
    assert msgs[0] == msgs[1]
    assert "request 417" in msgs[0]


@pytest.mark.parametrize("backend", BACKENDS)
def test_soa_batch_rejects_unordered_arrivals_like_records(backend):
    traces = _traces(2, 800)
    traces[0]["arrival_time"][300] = traces[0]["arrival_time"][299] - 1.0
    o = _opts()
    msgs = []
    for make in (lambda ts: ts, lambda ts: [abi.SoaTrace.from_records(t) for t in ts]):
        with pytest.raises(ConfigError) as ei:
            Batch(make(traces), o, device=0, lib=_lib(backend))
        msgs.append(str(ei.value))
    assert msgs[0] == msgs[1]


def test_soa_trace_round_trips_records():
    t = _traces(1, 500)[0]
    s = abi.SoaTrace.from_records(t)
    assert s.prompt.dtype == np.int32 and s.true_rl.dtype == np.int32 and s.arrival.dtype == np.float64
    assert np.array_equal(s.records(), t)
