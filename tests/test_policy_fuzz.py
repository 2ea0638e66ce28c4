"""Randomised configurations of every policy (capacity, block size, tfs,
chunk size, batch cap, recompute vs swap, swap stall, reserve, buffer ratio,
predictor), each run in lock-step against the compiled reference for up to
3,000 steps (vLLM recompute under a tight cache can livelock, in the
reference too); configurations the reference rejects must be rejected with
the same message."""
import numpy as np
import pytest

from oracle import port, ref
from paper_2411_06364_b200 import abi

from cases import BASELINES
from parity import base_options, sat_trace
from paper_2411_06364_b200.engine import ConfigError, SimulationError
from test_baselines import _engine, lockstep_or_same_error

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref (compiled reference) not built")


ECONO = ["econoserve-d", "econoserve-sd", "econoserve-sdo", "econoserve-full"]


def fuzz_case(seed, policies=BASELINES):
    rng = np.random.default_rng(seed)
    pol = policies[seed % len(policies)]
    n = int(rng.integers(40, 220))
    plo, rlo = int(rng.integers(4, 32)), int(rng.integers(4, 32))
    tr = sat_trace(port.generate_trace, n, float(rng.choice([20.0, 80.0, 400.0])), plo, plo + int(rng.integers(8, 120)),
                   rlo, rlo + int(rng.integers(8, 150)), int(rng.integers(1, 1000)))
    block = int(rng.choice([8, 16, 32]))
    cap = int(rng.choice([1024, 2048, 3072, 6144]))
    pm = str(rng.choice(["oracle", "lognormal", "bucket"]))
    kw = dict(kvc_capacity=cap, kvc_block_size=block, tfs=int(rng.choice([128, 512, 1024, 4096])),
              chunk_size=int(rng.choice([16, 64, 256, 512])), batch_size_cap=int(rng.integers(1, 17)),
              vllm_recompute=int(rng.integers(0, 2)), swap_stall=float(rng.choice([0.0, 0.002])),
              pred_model=pm, pred_sigma=0.4, pred_accuracy=0.7, pred_tolerance=0.15,
              pred_padding_ratio=float(rng.choice([0.0, 0.1, 0.3])), sched_cost_per_exam=float(rng.choice([0.0, 2e-5])),
              reserved_fraction=float(rng.choice([0.05, 0.1, 0.2])), buffer_ratio=float(rng.choice([0.0, 0.1, 0.25])))
    return pol, tr, base_options(pol, **kw)


SEEDS = list(range(120))


def run_case(seed, backend, policies=BASELINES):
    pol, tr, o = fuzz_case(seed, policies)
    try:
        ref.RefEngine(tr, o)
    except ref.EngineError as e:  # rejected at construction: the product must reject it the same way
        with pytest.raises((ConfigError, SimulationError)) as ex:
            _engine(backend, tr, o)
        assert str(ex.value) == str(e)
        return
    lockstep_or_same_error(tr, o, backend, every=1, max_steps=3000)


@pytest.mark.parametrize("seed", SEEDS)
def test_hostsim_fuzz(seed):
    run_case(seed, "hostsim")


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_device_fuzz(seed):
    run_case(seed, "device")


@pytest.mark.parametrize("seed", SEEDS)
def test_hostsim_fuzz_econoserve(seed):
    run_case(seed, "hostsim", ECONO)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_device_fuzz_econoserve(seed):
    run_case(seed, "device", ECONO)


def run_case_nolog(seed, backend):
    """The bench path: recording off (fused quiet-span replay, running
    aggregates only); snapshots, records and the report must still match."""
    from parity import lockstep
    pol, tr, o = fuzz_case(seed, ECONO)
    try:
        a = ref.RefEngine(tr, o)
    except ref.EngineError:
        return
    o2 = abi.default_options()
    C_fields = [f[0] for f in abi.Options._fields_]
    for f in C_fields:
        setattr(o2, f, getattr(o, f))
    o2.record_events = 0
    o2.record_samples = 0
    lockstep(a, _engine(backend, tr, o2), every=1, max_steps=3000, check_logs=False)


@pytest.mark.parametrize("seed", SEEDS[:60])
def test_hostsim_fuzz_nolog(seed):
    run_case_nolog(seed, "hostsim")


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS[:60])
def test_device_fuzz_nolog(seed):
    run_case_nolog(seed, "device")
