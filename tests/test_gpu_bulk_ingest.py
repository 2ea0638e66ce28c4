"""Grid-wide burst ingest (econo_batch_ingest: radix sort of the arrival batch
by PT class, k_bulk_*) leaves exactly the state the reference's
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


@pytest.mark.parametrize("path", ["tiles", "radix"])
@pytest.mark.parametrize("policy", ["econoserve-full", "econoserve-sdo"])
def test_bulk_ingest_matches_oracle(policy, path, monkeypatch):
    """Both device paths: tile-local sorts + per-instance stitch (default) and
    the global LSD radix sort (ECONO_INGEST_RADIX)."""
    monkeypatch.setenv("ECONO_BULK_INGEST_MIN", "1000")
    if path == "radix":
        monkeypatch.setenv("ECONO_INGEST_RADIX", "1")
    c = W.CONFIGS["cfg3_bookcorpus_1m"]
    traces = [port.generate_trace(n, 1e9, c["shape"]["prompt"], c["shape"]["rl"], 40 + i)
              for i, n in enumerate([20000, 500, 7000, 4096, 4097])]   # 500 stays below the threshold
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
