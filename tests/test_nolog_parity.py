"""Parity with recording off (the bench / batch path): the engine keeps only
the running sample aggregates and takes the fused quiet-span replay
(engine.cuh quiet_steps_fused). State snapshots, request records and the
aggregate report must still equal the oracle's (which records everything)."""
import copy

import pytest

from conftest import BACKENDS, make_engine
from oracle import port
from parity import lockstep

from cases import catalogue

CASES = catalogue(port.generate_trace)


def _nolog(opts):
    o = copy.copy(opts)
    o.record_events = 0
    o.record_samples = 0
    return o


@pytest.mark.parametrize("backend", [b for b in BACKENDS if b != "oracle"])
@pytest.mark.parametrize("name,trace,opts", CASES, ids=[c[0] for c in CASES])
def test_nolog_spans_vs_oracle(backend, name, trace, opts):
    lockstep(port.OracleEngine(trace, opts), make_engine(backend, trace, _nolog(opts)), every=97,
             check_logs=False)


@pytest.mark.parametrize("backend", [b for b in BACKENDS if b != "oracle"])
@pytest.mark.parametrize("name,trace,opts", CASES[:8], ids=[c[0] for c in CASES[:8]])
def test_nolog_full_run_vs_oracle(backend, name, trace, opts):
    lockstep(port.OracleEngine(trace, opts), make_engine(backend, trace, _nolog(opts)),
             every=1 << 40, check_logs=False)
