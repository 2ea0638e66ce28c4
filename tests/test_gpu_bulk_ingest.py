"""Grid-wide burst ingest (econo_batch_ingest: range scans + stitch by
default, k_ingest_ranges; tile sorts + stitch, k_ingest_tiles; or the global
radix sort by PT class, k_bulk_*) leaves exactly the state the reference's
ingest_arrivals (engine.hpp:216-235) does: snapshots after the ingest step
and after further steps equal the oracle's, bit for bit."""
import copy
import os

import numpy as np
import pytest

from oracle import port
from paper_2411_06364_b200 import abi, workloads as W
from paper_2411_06364_b200.engine import Batch

pytestmark = pytest.mark.gpu


def _opts(policy):
    b = W.CONFIGS["cfg3_bookcorpus_1m"]
    o = abi.default_options(**dict(b["opts"], policy=policy))
    o.record_events = 0
    o.record_samples = 0
    return o


@pytest.mark.parametrize("path", ["ranges", "tiles", "radix"])
@pytest.mark.parametrize("policy", ["econoserve-full", "econoserve-sdo"])
def test_bulk_ingest_matches_oracle(policy, path, monkeypatch):
    """Every device path: range scans + per-instance stitch (default),
    tile-local sorts + stitch (ECONO_INGEST_TILES) and the global LSD radix
    sort (ECONO_INGEST_RADIX). Sizes straddle the 4096-id tiles and the
    32768-id ranges."""
    monkeypatch.setenv("ECONO_BULK_INGEST_MIN", "1000")
    if path == "radix":
        monkeypatch.setenv("ECONO_INGEST_RADIX", "1")
    if path == "tiles":
        monkeypatch.setenv("ECONO_INGEST_TILES", "1")
    c = W.CONFIGS["cfg3_bookcorpus_1m"]
    traces = [port.generate_trace(n, 1e9, c["shape"]["prompt"], c["shape"]["rl"], 40 + i)
              for i, n in enumerate([20000, 500, 7000, 4096, 4097, 32768, 32769, 70001])]   # 500 stays below the threshold
    o = _opts(policy)
    b = Batch(traces, o, device=0)
    b.launch(1)          # idle tick to the burst
    b.sync()
    b.ingest()           # the burst, grid-wide (first part of step 2)
    b.launch(1)          # the rest of step 2
    b.sync()
    oracles = [port.OracleEngine(t, o) for t in traces]
    for i, e in enumerate(oracles):
        e.step(2)
        assert np.array_equal(b.snapshot(i), e.snapshot()), f"instance {i} after the ingest step"
    for _ in range(3):
        b.launch(300)
        b.sync()
        for i, e in enumerate(oracles):
            e.step(300)
            assert np.array_equal(b.snapshot(i), e.snapshot()), f"instance {i}"


@pytest.mark.parametrize("path", ["ranges", "tiles"])
def test_bulk_ingest_one_class_full_ranges(path, monkeypatch):
    """Every arrival in one PT class: a whole 32768-id range is one segment
    (count 32768, the largest the range records hold) and the class list
    runs through three ranges."""
    monkeypatch.setenv("ECONO_BULK_INGEST_MIN", "1000")
    if path == "tiles":
        monkeypatch.setenv("ECONO_INGEST_TILES", "1")
    c = W.CONFIGS["cfg3_bookcorpus_1m"]
    t = port.generate_trace(70000, 1e9, c["shape"]["prompt"], c["shape"]["rl"], 77)
    t["prompt_len"] = 1900
    t["true_rl"] = 600
    o = _opts("econoserve-full")
    b = Batch([t], o, device=0)
    b.launch(1)
    b.sync()
    b.ingest()
    b.launch(1)
    b.sync()
    e = port.OracleEngine(t, o)
    e.step(2)
    assert np.array_equal(b.snapshot(0), e.snapshot())
    b.launch(500)
    b.sync()
    e.step(500)
    assert np.array_equal(b.snapshot(0), e.snapshot())


@pytest.mark.parametrize("path", ["ranges", "tiles"])
def test_bulk_ingest_several_deadline_buckets(path, monkeypatch):
    """Deadline bounds inside the burst's slack range (cfg3's SLOs are ~27 s
    to ~900 s): the arrivals spread over four buckets, so the range scan's
    class window (k_bulk_plan's corner bound) spans several buckets; a mixed
    trace spreads the prompts too."""
    monkeypatch.setenv("ECONO_BULK_INGEST_MIN", "1000")
    if path == "tiles":
        monkeypatch.setenv("ECONO_INGEST_TILES", "1")
    c = W.CONFIGS["cfg3_bookcorpus_1m"]
    traces = [port.generate_trace(n, 1e9, c["shape"]["prompt"], c["shape"]["rl"], 90 + i)
              for i, n in enumerate([50000, 33000])]
    traces.append(W.mixed_trace(port.generate_trace, 40000, 1e9, 95))
    b0 = W.CONFIGS["cfg3_bookcorpus_1m"]
    o = abi.default_options(**dict(b0["opts"], policy="econoserve-full", reserved_fraction=0.2))  # mixed prompts fit
    o.record_events = 0
    o.record_samples = 0
    o.n_deadline_bounds = 3
    o.deadline_bounds[0], o.deadline_bounds[1], o.deadline_bounds[2] = 100.0, 250.0, 500.0
    b = Batch(traces, o, device=0)
    b.launch(1)
    b.sync()
    b.ingest()
    b.launch(1)
    b.sync()
    oracles = [port.OracleEngine(t, o) for t in traces]
    for i, e in enumerate(oracles):
        e.step(2)
        assert np.array_equal(b.snapshot(i), e.snapshot()), f"instance {i} after the ingest step"
    for _ in range(2):
        b.launch(400)
        b.sync()
        for i, e in enumerate(oracles):
            e.step(400)
            assert np.array_equal(b.snapshot(i), e.snapshot()), f"instance {i}"
