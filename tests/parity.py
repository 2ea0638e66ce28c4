"""Shared parity helpers: lock-step comparison of two engines (any pair of the
product Engine, the C oracle and the compiled reference) through the
canonical state snapshot after every step, then events, samples, records and
the aggregate report."""
import numpy as np

from paper_2411_06364_b200 import abi


def sat_trace(gen, n, rate, plo, phi, rlo, rhi, seed):
    """saturating_trace (tests/test_engine.cpp:28-37)."""
    return gen(n, rate, ((plo + phi) / 2, plo, phi, 0.4), ((rlo + rhi) / 2, rlo, rhi, 0.4), seed)


def base_options(kind, **kw):
    """base_options (tests/test_engine.cpp:11-26)."""
    d = dict(policy=kind, tfs=1024, reserved_fraction=0.05, buffer_ratio=0.0, t_base=0.005,
             t_token=1e-4, sched_cost_per_exam=0.0, pred_model="oracle", pred_padding_ratio=0.0,
             kvc_capacity=8192, kvc_block_size=32, seed=1)
    d.update(kw)
    return abi.default_options(**d)


def first_diff(sa, sb):
    n = min(len(sa), len(sb))
    d = np.nonzero(sa[:n] != sb[:n])[0]
    return int(d[0]) if len(d) else n


def lockstep(a, b, every=1, max_steps=None, check_snapshots=True, check_logs=True):
    """Steps engines a and b together; returns the number of steps.
    check_logs=False skips the event/sample logs (b may run with recording
    off: records and the aggregate report must still match exactly)."""
    steps = 0
    more = True
    while more and (max_steps is None or steps < max_steps):
        k = every if max_steps is None else min(every, max_steps - steps)
        more = a.step(k)
        mb = b.step(k)
        steps += k
        assert more == mb, f"step {steps}: more {more} vs {mb}"
        if check_snapshots:
            sa, sb = a.snapshot(), b.snapshot()
            if len(sa) != len(sb) or not np.array_equal(sa, sb):
                i = first_diff(sa, sb)
                raise AssertionError(
                    f"state diverged after step {steps} at word {i}: "
                    f"{sa[i:i + 6].tolist()} vs {sb[i:i + 6].tolist()}")
    if check_logs:
        ea, eb = a.events(), b.events()
        assert len(ea) == len(eb) and np.array_equal(ea, eb), "event logs differ"
        assert np.array_equal(a.samples(), b.samples()), "iteration samples differ"
    if not more:
        ra, pa = a.finalize()
        rb, pb = b.finalize()
        assert np.array_equal(ra, rb), "request records differ"
        da, db = pa.as_dict(), pb.as_dict()
        for k in da:
            assert da[k] == db[k], (k, da[k], db[k])
    return steps
