"""A launch on a caller's stream is ordered before the work the handle later
enqueues on its own stream (econo_batch_partials, _reports, econo_records):
the handle's stream waits on an event recorded after the launch. Calling
partials() right after an asynchronous launch, with no synchronisation,
gives the same sums as after an explicit sync."""
import numpy as np
import pytest

from oracle import port
from paper_2411_06364_b200 import abi, workloads as W
from paper_2411_06364_b200.engine import Batch

pytestmark = pytest.mark.gpu


def test_partials_right_after_a_caller_stream_launch():
    import torch
    c = W.CONFIGS["cfg1_alpaca_10k"]
    traces = [port.generate_trace(2000, 200.0, c["shape"]["prompt"], c["shape"]["rl"], 300 + i) for i in range(4)]
    o = abi.default_options(**c["opts"])
    o.record_events = 0
    o.record_samples = 0
    s = torch.cuda.Stream()
    a = Batch(traces, o, device=0)
    a.launch(1 << 40, s.cuda_stream)   # asynchronous, caller's stream
    got = a.partials()                  # no sync in between
    b = Batch(traces, o, device=0)
    b.launch(1 << 40, s.cuda_stream)
    s.synchronize()
    b.sync()
    want = b.partials()
    assert np.array_equal(got, want)
    assert all(x.done for x in a.scalars())
