"""Device parity at BASELINE.json's stated sizes, on the bench's own path.

SURVEY.md §8(d): 1M-request instances are checked bit-exactly against the
reference over a prefix of >= 5,000 scheduler iterations (a full CPU run at
1M takes hours); configs[1] (100k) is checked over its whole run.

The device side runs exactly what bench.py runs: one Batch of several
instances (trace seeds 1000+i, the bench's instances 0..k-1; configs[2]'s
traces as page-locked-style columns through econo_batch_create_soa, like the
bench, configs[3]'s as records), the idle tick, the grid-wide burst ingest
(econo_batch_ingest: range scans) forced into several launch groups with
ECONO_BULK_BUDGET, then time-sliced launches (econo_batch_launch_slice /
launch_to) with recording off. The reference side is the unmodified reference compiled in place
(oracle/_ref, engine.hpp:104-116), one std::thread per engine, its burst
ingested by ref_fast_ingest (an order-identical stable sort in place of the
O(n^2) insert_ordered, queues.hpp:85-92).

At each checkpoint the canonical snapshot (block tables, free gaps, slots,
both queues in order, reserve/written maps, running order, 23 words per
request, FP fields as bit patterns: DESIGN.md §8) must be equal.
"""
import ctypes as C
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import ref
from paper_2411_06364_b200 import abi, metrics, workloads as W
from paper_2411_06364_b200.engine import Batch, generate_trace

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SLICE_NS = 100_000  # 100 us slices: instances drift apart, launch_to brings them back


def _opts(name, record):
    o = abi.default_options(**W.CONFIGS[name]["opts"])
    o.record_events = 1 if record else 0
    o.record_samples = 0
    return o


def _ref_step_all(engines, steps):
    hv = (C.c_void_p * len(engines))(*[e.h.value for e in engines])
    ref.lib().ref_time_steps_parallel(hv, len(engines), steps, None)


def _device_batch(name, traces, monkeypatch, budget):
    monkeypatch.setenv("ECONO_BULK_BUDGET", str(budget))
    b = Batch(traces, _opts(name, record=False), device=0)
    b.launch(1)      # idle tick up to the burst (engine.hpp:930-949)
    b.sync()
    b.ingest()       # the burst, grid-wide, several radix-sort groups
    b.launch(1)      # the rest of that step
    b.sync()
    return b


def _reference(name, traces):
    o = _opts(name, record=True)  # the reference's default options log events
    with ThreadPoolExecutor(len(traces)) as ex:
        engines = list(ex.map(lambda t: ref.RefEngine(t, o), traces))
    for e in engines:
        e.idle_to_first_arrival()
        e.fast_ingest()
        e.step(1)
    return engines


def _compare(b, engines, step):
    for i, e in enumerate(engines):
        s = b.scalars()[i]
        assert s.steps == step and not s.error, (i, s.steps, s.error)
        d, r = b.snapshot(i), e.snapshot()
        assert d.shape == r.shape and np.array_equal(d, r), f"instance {i} differs at step {step}"


def _run_prefix(name, k, monkeypatch, budget, checkpoints=(502, 5002), soa=False):
    c = W.CONFIGS[name]
    seeds = [1000 + i for i in range(k)]
    with ThreadPoolExecutor(k) as ex:
        traces = list(ex.map(lambda s: W.make_trace(name, generate_trace, seed=s), seeds))
    assert len(traces[0]) == c["n"]
    b = _device_batch(name, [abi.SoaTrace.from_records(t) for t in traces] if soa else traces, monkeypatch,
                      budget)
    engines = _reference(name, traces)
    _compare(b, engines, 2)
    at = 2
    for cp in checkpoints:
        b.advance_to(cp, slice_ns=SLICE_NS)
        _ref_step_all(engines, cp - at)
        at = cp
        _compare(b, engines, cp)
    adm = sum(s.pt_dispatched for s in b.scalars())
    assert adm > 0  # the window schedules work (PT admissions), it is not idle
    b.close()


def test_cfg3_1m_prefix_16_instances(monkeypatch):
    """configs[2] (BookCorpus 1M burst, econoserve-full): the bench's first 16
    instances from column traces, the burst ingest in several launch groups
    (a group holds ~60k segment slots; a 1M instance needs 31 ranges x its
    class window), 5,002 iterations."""
    _run_prefix("cfg3_bookcorpus_1m", 16, monkeypatch, budget=60_000, soa=True)


def test_cfg4_1m_prefix_8_instances(monkeypatch):
    """configs[3] (mixed 1M burst, lognormal sigma 0.3: preemptions, reserve
    top-ups, hosted slots) over 5,002 iterations, ingest in several groups."""
    _run_prefix("cfg4_mixed_1m", 8, monkeypatch, budget=400_000)


def test_cfg2_100k_full_run(monkeypatch):
    """configs[1] (ShareGPT 100k, Poisson 28 rps, pipelining): whole runs of
    two instances, final state, every request record and the report."""
    name = "cfg2_sharegpt_100k"
    traces = [W.make_trace(name, generate_trace, seed=1000 + i) for i in range(2)]
    b = Batch(traces, _opts(name, record=False), device=0)
    while True:
        b.launch(1 << 40, slice_ns=2_000_000)
        b.sync()
        if all(s.done or s.error for s in b.scalars()):
            break
    o = _opts(name, record=True)
    engines = [ref.RefEngine(t, o) for t in traces]
    _ref_step_all(engines, 1 << 40)
    reps = b.reports()
    for i, e in enumerate(engines):
        assert not b.scalars()[i].error
        assert np.array_equal(b.snapshot(i), e.snapshot()), f"instance {i} final state"
        rr, rp = e.finalize()
        assert np.array_equal(b.records(i), rr), f"instance {i} records"
        d = reps[i]
        for f in ("iterations", "preemptions", "reserve_draws", "hosted_slots", "hosted_overruns"):
            assert getattr(d, f) == getattr(rp, f), f
        assert d.hosted_slots > 0  # pipelining ran
        for f in ("mean_jct", "p5_jct", "p95_jct", "ssr", "makespan", "mean_tbt", "goodput_rps",
                  "mean_waiting", "mean_execution", "mean_scheduling", "mean_forward_size"):
            a, r = getattr(d, f), getattr(rp, f)
            assert abs(a - r) <= 1e-6 * max(1.0, abs(r)), (f, a, r)
    b.close()
