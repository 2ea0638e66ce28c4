"""The comparison policies — orca, vllm, sarathi, multires, sync-coupled
(engine.hpp:383-726) — against the compiled reference (oracle/_ref), bit-exact
per step: state snapshot (block tables, wait FIFO, waiting groups, admit
order, ongoing prefills, prefill targets), events, samples, records, report.
The host build (tests/_hostsim) runs on CPU; the device build under -m gpu.
Plus the reference's own property tests for these policies
(tests/test_engine.cpp:110-125, 243-283)."""
import numpy as np
import pytest

from oracle import port, ref
from paper_2411_06364_b200 import abi
from paper_2411_06364_b200.engine import ConfigError, Engine, SimulationError

from cases import BASELINES, baseline_catalogue
from conftest import HOSTSIM
from parity import base_options, lockstep, sat_trace
from snapshot import decode

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref (compiled reference) not built")

CASES = baseline_catalogue(port.generate_trace)
IDS = [c[0] for c in CASES]
BIG = ("alpaca", "mixed")


def _engine(backend, trace, opts):
    return Engine(trace, opts, lib=HOSTSIM) if backend == "hostsim" else Engine(trace, opts)


def lockstep_or_same_error(trace, opts, backend, every, max_steps=None):
    """lockstep(); when the reference itself fails (e.g. 'simulation stuck'),
    the product must fail with the same code and message at the same step."""
    a, b = ref.RefEngine(trace, opts), _engine(backend, trace, opts)
    try:
        return lockstep(a, b, every=every, max_steps=max_steps)
    except (ref.EngineError, ConfigError, SimulationError) as e:
        # replay both one step at a time to the failing step
        a, b = ref.RefEngine(trace, opts), _engine(backend, trace, opts)
        for _ in range(10 ** 7):
            ea = eb = None
            try:
                a.step(1)
            except ref.EngineError as x:
                ea = x
            try:
                b.step(1)
            except (ConfigError, SimulationError) as x:
                eb = x
            if ea or eb:
                assert ea is not None and eb is not None, (ea, eb, e)
                code = abi.ECONFIG if isinstance(eb, ConfigError) else abi.ESIM
                assert (ea.code, str(ea)) == (code, str(eb))
                return -1
        raise


@pytest.mark.parametrize("name,trace,opts", CASES, ids=IDS)
def test_hostsim_lockstep_vs_reference(name, trace, opts):
    lockstep_or_same_error(trace, opts, "hostsim", every=61 if name.startswith(BIG) else 1)


@pytest.mark.gpu
@pytest.mark.parametrize("name,trace,opts", CASES, ids=IDS)
def test_device_lockstep_vs_reference(name, trace, opts):
    lockstep_or_same_error(trace, opts, "device", every=1)


@pytest.mark.gpu
@pytest.mark.parametrize("name,trace,opts", CASES, ids=IDS)
def test_device_full_run_vs_reference(name, trace, opts):
    """One launch for the whole run, then events / samples / records / report."""
    lockstep_or_same_error(trace, opts, "device", every=1 << 40)


@pytest.mark.parametrize("backend", ["hostsim", pytest.param("device", marks=pytest.mark.gpu)])
def test_recompute_livelock_prefix(backend):
    """vLLM recompute preemption under a tight cache livelocks in the
    reference (no request ever finishes its recomputed prefill); the product
    reproduces the same endless schedule — checked over a prefix."""
    tr = sat_trace(port.generate_trace, 120, 200.0, 16, 64, 32, 128, 59)
    o = base_options("vllm", kvc_capacity=2048, vllm_recompute=1, swap_stall=0.002)
    assert lockstep_or_same_error(tr, o, backend, every=7, max_steps=3000) == 3000


@pytest.mark.parametrize("kind", BASELINES)
def test_runs_are_deterministic(kind):  # test_engine.cpp:110-125
    tr = sat_trace(port.generate_trace, 300, 40.0, 8, 64, 8, 96, 3)
    o = base_options(kind, pred_model="lognormal", pred_sigma=0.3, pred_padding_ratio=0.10)
    a, b = Engine(tr, o, lib=HOSTSIM), Engine(tr, o, lib=HOSTSIM)
    ra, pa = a.run()
    rb, pb = b.run()
    assert np.array_equal(ra, rb) and pa.as_dict() == pb.as_dict()
    assert np.array_equal(a.events(), b.events())


@pytest.mark.parametrize("kind", ["vllm", "sync-coupled"])
def test_token_conservation_and_clock_identity(kind):  # test_engine.cpp:127-145
    tr = sat_trace(port.generate_trace, 200, 30.0, 8, 80, 8, 64, 11)
    o = base_options(kind, pred_model="lognormal", pred_sigma=0.25, pred_padding_ratio=0.10)
    e = Engine(tr, o, lib=HOSTSIM)
    e.run()
    s = decode(e.snapshot())
    assert all(r["state"] == 4 for r in s["requests"])
    assert [r["generated"] for r in s["requests"]] == [int(x) for x in tr["true_rl"]]
    assert s["clock"] == pytest.approx(float(np.sum(e.samples()["dt"])), rel=1e-12)


def test_sync_coupled_tops_up_less_than_sd():  # test_engine.cpp:243-252
    tr = sat_trace(port.generate_trace, 300, 80.0, 8, 48, 16, 64, 47)
    _, sd = Engine(tr, base_options("econoserve-sd"), lib=HOSTSIM).run()
    _, sc = Engine(tr, base_options("sync-coupled"), lib=HOSTSIM).run()
    assert sd.pt_admit_frac > sc.pt_admit_frac


def test_orca_respects_its_batch_cap():  # test_engine.cpp:254-270
    tr = sat_trace(port.generate_trace, 40, 1000.0, 8, 32, 8, 32, 53)
    o = base_options("orca", batch_size_cap=8)
    e = Engine(tr, o, lib=HOSTSIM)
    _, rep = e.run()
    assert rep.allocation_failure_pct == 0.0
    assert max(e.samples()["completed"]) <= 8


def test_vllm_allocation_failures_under_pressure():  # test_engine.cpp:272-283
    tr = sat_trace(port.generate_trace, 120, 200.0, 16, 64, 32, 128, 59)
    e = Engine(tr, base_options("vllm", kvc_capacity=2048), lib=HOSTSIM)
    _, rep = e.run()
    assert rep.allocation_failure_pct > 0.0 and rep.preemptions > 0
    s = decode(e.snapshot())
    assert [r["generated"] for r in s["requests"]] == [int(x) for x in tr["true_rl"]]
    kinds = {abi.EV_KINDS[k] for k in e.events()["kind"]}
    assert {"alloc_fail", "preempt_swap", "swap_in"} <= kinds


def test_orca_infeasible_uses_max_output_len():  # engine.hpp:193-201
    o = base_options("orca", kvc_capacity=1024, max_output_len=2000)
    with pytest.raises(SimulationError, match="request 0: KVC demand"):
        Engine([(0.1, 10, 10)], o, lib=HOSTSIM)
