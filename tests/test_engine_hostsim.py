"""The product engine SOURCE (engine.cuh + runtime.cu) compiled for the host
with one lane per warp (tests/_hostsim, test-only) against the oracle and the
reference fixtures. This checks the scheduling logic on a CPU-only box; the
device build is checked by tests/test_gpu_parity.py."""
import glob
import os

import pytest

from oracle import port
from paper_2411_06364_b200.engine import Engine

from cases import catalogue
from conftest import HOSTSIM
from parity import lockstep
from test_oracle_golden import FIXTURES, check_engine_against_fixture, load_fixture

CASES = catalogue(port.generate_trace)


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[:-4] for p in FIXTURES])
def test_hostsim_matches_reference_fixture(path):
    z, opts = load_fixture(path)
    check_engine_against_fixture(Engine(z["trace"], opts, lib=HOSTSIM), z)


@pytest.mark.parametrize("every", [1, 13, 1 << 40])
@pytest.mark.parametrize("name,trace,opts", CASES, ids=[c[0] for c in CASES])
def test_hostsim_lockstep_vs_oracle(name, trace, opts, every):
    if every == 1 and name.startswith(("sharegpt", "bookcorpus")):
        every = 61  # tens of thousands of steps: per-step snapshots cost minutes on CPU
    lockstep(port.OracleEngine(trace, opts), Engine(trace, opts, lib=HOSTSIM), every=every)
