"""Device (sm_100a) engine vs the C oracle, bit-exact per step: state
snapshot (block tables, slots, queues, counters, per-request state), event
log, iteration samples, request records and the aggregate report."""
import numpy as np
import pytest

from oracle import port
from paper_2411_06364_b200 import abi, workloads as W
from paper_2411_06364_b200.engine import Engine

from cases import catalogue
from parity import lockstep

pytestmark = pytest.mark.gpu

CASES = catalogue(port.generate_trace)


@pytest.mark.parametrize("name,trace,opts", CASES, ids=[c[0] for c in CASES])
def test_lockstep_vs_oracle(name, trace, opts):
    """Snapshot after every single step."""
    lockstep(port.OracleEngine(trace, opts), Engine(trace, opts))


@pytest.mark.parametrize("name,trace,opts", CASES, ids=[c[0] for c in CASES])
def test_spans_vs_oracle(name, trace, opts):
    """Snapshots every 97 steps: exercises multi-step launches and the
    event-horizon skipping inside them."""
    lockstep(port.OracleEngine(trace, opts), Engine(trace, opts), every=97)


@pytest.mark.parametrize("name,trace,opts", CASES, ids=[c[0] for c in CASES])
def test_full_run_vs_oracle(name, trace, opts):
    """One launch for the whole run, then events / samples / records / report."""
    lockstep(port.OracleEngine(trace, opts), Engine(trace, opts), every=1 << 40)


@pytest.mark.parametrize("policy", ["econoserve-full", "econoserve-sd"])
def test_cfg1_full_run(policy):
    c = W.CONFIGS["cfg1_alpaca_10k"]
    t = port.generate_trace(c["n"], c["rate"], c["shape"]["prompt"], c["shape"]["rl"], c["seed"])
    opts = abi.default_options(**dict(c["opts"], policy=policy))
    lockstep(port.OracleEngine(t, opts), Engine(t, opts), every=1 << 40)
