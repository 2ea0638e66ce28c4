"""econo_batch_launch_to: every instance advances until it has made exactly
`target` step() calls (instances already there do nothing), so a batch whose
instances drifted apart comes back to one common step — the bench's parity
checkpoint and the scale-parity tests rely on it. Checked on the host build
(CPU) and on the device, against the oracle stepped to the same count."""
import numpy as np
import pytest

from oracle import port
from paper_2411_06364_b200 import abi, workloads as W
from paper_2411_06364_b200.engine import Batch

from conftest import HOSTSIM


@pytest.mark.parametrize("backend", ["hostsim", pytest.param("device", marks=pytest.mark.gpu)])
def test_launch_to_reaches_a_common_step(backend):
    c = W.CONFIGS["cfg1_alpaca_10k"]
    traces = [port.generate_trace(n, 200.0, c["shape"]["prompt"], c["shape"]["rl"], 90 + i)
              for i, n in enumerate([300, 800])]
    o = abi.default_options(**c["opts"])
    o.record_events = 0
    o.record_samples = 0
    lib = HOSTSIM if backend == "hostsim" else None
    b = Batch(traces, o, device=0, lib=lib)
    b.launch(37)          # both at 37
    b.sync()
    b.launch_to(20)       # already past: nothing happens
    b.sync()
    assert [s.steps for s in b.scalars()] == [37, 37]
    for target in (120, 121, 500):  # the 300-request instance finishes before step 500
        b.advance_to(target)
        assert all(s.steps == target or (s.done and s.steps < target) for s in b.scalars())
        for i, t in enumerate(traces):
            e = port.OracleEngine(t, o)
            e.step(target)
            assert np.array_equal(b.snapshot(i), e.snapshot()), (i, target)
    with pytest.raises(Exception):
        b.launch_to(-1)
