"""Time-sliced launches (econo_batch_launch_slice): where a launch stops
depends on device time, but every step is exact, so the final state of every
instance equals the fixed-launch run's, bit for bit."""
import numpy as np
import pytest

from oracle import port
from paper_2411_06364_b200 import abi, workloads as W
from paper_2411_06364_b200.engine import Batch

pytestmark = pytest.mark.gpu


def test_sliced_launches_match_fixed_launches():
    c = W.CONFIGS["cfg1_alpaca_10k"]
    traces = [port.generate_trace(n, 300.0, c["shape"]["prompt"], c["shape"]["rl"], 70 + i)
              for i, n in enumerate([400, 1500, 3000])]
    o = abi.default_options(**dict(c["opts"], pred_model="lognormal", pred_sigma=0.3))
    o.record_events = 0
    o.record_samples = 0
    a = Batch(traces, o, device=0)
    a.launch(1 << 40)
    a.sync()
    b = Batch(traces, o, device=0)
    launches = 0
    while not all(s.completed >= len(t) for s, t in zip(b.scalars(), traces)):
        b.launch(1 << 40, slice_ns=20_000)  # 20 us slices
        b.sync()
        launches += 1
        assert launches < 100000
    assert launches > 3  # the slices really cut the run
    assert np.array_equal(a.partials(), b.partials())
    for i in range(len(traces)):
        assert np.array_equal(a.snapshot(i), b.snapshot(i))
