"""Device-side metric partial sums (k_partials_slices + k_partials_finish,
runtime.cu) against the oracle's aggregate() (metrics.hpp:96-175): per
instance, within the 1e-6-relative contract for derived floating point;
integer counts exactly."""
import numpy as np
import pytest

from oracle import port
from paper_2411_06364_b200 import abi, metrics, workloads as W

pytestmark = pytest.mark.gpu

KEYS = ["mean_jct", "mean_tbt", "ssr", "normalized_latency", "throughput_rps", "throughput_tps",
        "goodput_rps", "mean_kvc_written", "mean_kvc_allocated", "mean_forward_size", "tfs_hit_frac",
        "pt_admit_frac", "mean_waiting", "mean_execution", "mean_preemption", "mean_scheduling",
        "makespan"]


def _opts():
    c = W.CONFIGS["cfg1_alpaca_10k"]
    o = abi.default_options(**dict(c["opts"], pred_model="bucket", pred_accuracy=0.775,
                                   pred_tolerance=0.1))
    o.record_events = 0
    o.record_samples = 0
    return o


def test_device_partials_match_oracle_reports():
    from paper_2411_06364_b200.engine import Batch
    c = W.CONFIGS["cfg1_alpaca_10k"]
    traces = [port.generate_trace(n, 150.0, c["shape"]["prompt"], c["shape"]["rl"], 50 + i)
              for i, n in enumerate([300, 1700, 5000])]
    o = _opts()
    b = Batch(traces, o, device=0)
    b.launch(1 << 40)
    b.sync()
    parts = b.partials()
    for i, t in enumerate(traces):
        _, rep = port.OracleEngine(t, o).run()
        want = rep.as_dict()
        s = metrics.summary(parts[i])
        for k in KEYS:
            assert abs(s[k] - want[k]) <= 1e-6 * max(1.0, abs(want[k])), (i, k, s[k], want[k])
        assert s["iterations"] == want["iterations"]
        assert s["preemptions"] == want["preemptions"]
        assert s["requests"] == len(t)
    # deterministic: the slice reduction runs in a fixed order
    assert np.array_equal(parts, b.partials())
