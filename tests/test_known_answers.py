"""The reference's own engine-level known answers and properties
(proj/tests/test_engine.cpp, test_queues.cpp, test_kvc.cpp, acceptance C1-C3)
re-asserted through the shared Engine API on every backend: the C oracle,
the host build of the product source, and the sm_100a device build (gpu)."""
import numpy as np
import pytest

from oracle import port
from paper_2411_06364_b200 import abi
from paper_2411_06364_b200.engine import ConfigError, SimulationError

from conftest import BACKENDS, make_engine
from parity import base_options, sat_trace
from snapshot import decode


def itime(fs, o):  # iteration_time (engine.hpp:46-51)
    base = min(fs, o.tfs)
    over = max(0, fs - o.tfs)
    rate = o.t_token if o.t_token_over < 0 else o.t_token_over
    return o.t_base + o.t_token * base + rate * over


def gen(*a):
    return port.generate_trace(*a)


def kinds(ev):
    return [abi.EV_KINDS[k] for k in ev["kind"]]


@pytest.mark.parametrize("backend", BACKENDS)
def test_single_request_closed_form_jct(backend):  # test_engine.cpp:66-80
    o = base_options("econoserve-full")
    e = make_engine(backend, [(0.005, 100, 20)], o)
    e.step(1 << 30)
    recs, rep = e.finalize()
    r = recs[0]
    expected = itime(100, o) + 20.0 * itime(1, o)
    jct = r["completion_time"] - r["arrival"]
    assert abs(jct - expected) <= 1e-9 * expected
    assert abs(r["waiting_time"]) <= 1e-12
    assert r["preemption_time"] == 0.0
    assert abs(r["execution_time"] - expected) <= 1e-9 * expected
    assert rep.preemptions == 0


@pytest.mark.parametrize("backend", BACKENDS)
def test_prefilled_prompt_enters_gt_queue_with_kv_resident(backend):  # test_engine.cpp:82-97
    o = base_options("econoserve-sd", kvc_capacity=8192)
    e = make_engine(backend, [(0.005, 100, 5), (50.0, 10, 5)], o)
    e.step(1)
    e.step(1)
    d = decode(e.snapshot())
    assert sum(len(g["members"]) for g in d["gt_groups"]) == 1
    r = d["requests"][0]
    assert r["state"] == 2  # WaitingGt
    assert r["occupied_kvc"] >= 100
    assert d["reserved"].get(0) == 100  # prompt staged in the reserve
    while e.step(1):
        pass
    assert decode(e.snapshot())["requests"][0]["state"] == 4


@pytest.mark.parametrize("backend", BACKENDS)
def test_empty_batch_advances_clock_by_idle_ticks(backend):  # test_engine.cpp:99-108
    e = make_engine(backend, [(1.0, 10, 5)], base_options("econoserve-full"))
    e.step(1)
    s = e.samples()
    assert len(s) == 1 and s[0]["idle_repeat"] > 0
    clk = decode(e.snapshot())["clock"]
    assert clk >= 1.0
    assert abs(clk - s[0]["dt"]) <= 1e-12


@pytest.mark.parametrize("backend", BACKENDS)
def test_deterministic_per_seed(backend):  # test_engine.cpp:110-125
    tr = sat_trace(gen, 300, 40.0, 8, 64, 8, 96, 3)
    o = base_options("econoserve-full", pred_model="lognormal", pred_sigma=0.3, pred_padding_ratio=0.10)
    a, b = make_engine(backend, tr, o), make_engine(backend, tr, o)
    a.step(1 << 30)
    b.step(1 << 30)
    assert np.array_equal(a.events(), b.events())
    ra, pa = a.finalize()
    rb, pb = b.finalize()
    assert np.array_equal(ra, rb) and pa.as_dict() == pb.as_dict()


@pytest.mark.parametrize("backend", BACKENDS)
def test_token_conservation_and_clock_identity(backend):  # test_engine.cpp:127-145
    tr = sat_trace(gen, 200, 30.0, 8, 80, 8, 64, 11)
    o = base_options("econoserve-full", pred_model="lognormal", pred_sigma=0.25, pred_padding_ratio=0.10)
    e = make_engine(backend, tr, o)
    e.step(1 << 30)
    d = decode(e.snapshot())
    for i, r in enumerate(d["requests"]):
        assert r["state"] == 4 and r["generated"] == tr[i]["true_rl"]
    s = e.samples()
    assert abs(d["clock"] - float(np.sum(s["dt"]))) <= 1e-12 * d["clock"]
    general = o.kvc_capacity - round(o.reserved_fraction * o.kvc_capacity)
    assert d["free_tokens"] == general and d["reserved_used"] == 0


@pytest.mark.parametrize("backend", BACKENDS)
def test_jct_identity(backend):  # test_engine.cpp:147-162
    tr = sat_trace(gen, 150, 25.0, 8, 60, 8, 64, 19)
    o = base_options("econoserve-full", sched_cost_per_exam=2e-5, pred_model="lognormal",
                     pred_sigma=0.3, pred_padding_ratio=0.05)
    e = make_engine(backend, tr, o)
    e.step(1 << 30)
    recs, _ = e.finalize()
    lhs = recs["completion_time"] - recs["arrival"]
    rhs = recs["waiting_time"] + recs["execution_time"] + recs["preemption_time"] + recs["scheduling_time_share"]
    assert np.all(np.abs(lhs - rhs) <= 1e-6)


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("padding", [0.0, 0.15])
def test_oracle_never_mispredicts(backend, padding):  # test_engine.cpp:164-179
    tr = sat_trace(gen, 400, 50.0, 8, 64, 8, 96, 23)
    e = make_engine(backend, tr, base_options("econoserve-full", pred_padding_ratio=padding))
    e.step(1 << 30)
    _, rep = e.finalize()
    assert rep.preemptions == 0 and rep.reserve_draws == 0
    assert rep.allocation_failure_pct == 0.0 and rep.hosted_overruns == 0
    k = kinds(e.events())
    assert "reserve_topup" not in k and "preempt" not in k


@pytest.mark.parametrize("backend", BACKENDS)
def test_underprediction_reserve_then_preempt(backend):  # test_engine.cpp:181-206
    tr = sat_trace(gen, 200, 40.0, 8, 40, 16, 120, 31)
    rich = make_engine(backend, tr, base_options("econoserve-sd", pred_model="lognormal",
                                                 pred_sigma=0.6, reserved_fraction=0.30))
    rich.step(1 << 30)
    assert rich.finalize()[1].reserve_draws > 0
    poor = make_engine(backend, tr, base_options("econoserve-sd", pred_model="lognormal",
                                                 pred_sigma=0.6, reserved_fraction=0.02))
    poor.step(1 << 30)
    assert poor.finalize()[1].preemptions > 0
    ev = poor.events()
    pre = ev[ev["kind"] == abi.EV_KINDS.index("preempt")]
    assert len(pre) > 0 and all(abi.event_str(x)[1].find("l_new") >= 0 for x in pre)
    d = decode(poor.snapshot())
    assert all(r["generated"] == tr[i]["true_rl"] for i, r in enumerate(d["requests"]))


@pytest.mark.parametrize("backend", BACKENDS)
def test_same_rl_groups_complete_together(backend):  # test_engine.cpp:208-231
    tr = sat_trace(gen, 400, 60.0, 8, 32, 8, 48, 41)
    e = make_engine(backend, tr, base_options("econoserve-sd"))
    e.step(1 << 30)
    ev = e.events()
    done = {int(x["id"]): int(x["iter"]) for x in ev if x["kind"] == 5}
    sched = {}
    for x in ev:
        if x["kind"] == 1:
            sched.setdefault((int(x["iter"]), int(x["a"])), []).append(int(x["id"]))
    checked = 0
    for members in sched.values():
        if len(members) < 2:
            continue
        checked += 1
        assert len({done[m] for m in members}) == 1
    assert checked > 0


@pytest.mark.parametrize("backend", BACKENDS)
def test_hosted_gts_meet_deadlines_under_oracle(backend):  # test_engine.cpp:233-241
    tr = sat_trace(gen, 500, 250.0, 8, 32, 8, 128, 43)
    e = make_engine(backend, tr, base_options("econoserve-full"))
    e.step(1 << 30)
    _, rep = e.finalize()
    assert rep.hosted_slots > 0 and rep.hosted_overruns == 0 and rep.preemptions == 0


@pytest.mark.parametrize("backend", BACKENDS)
def test_infeasible_request_named(backend):  # test_engine.cpp:284-294
    with pytest.raises(Exception) as ex:
        make_engine(backend, [(0.1, 2000, 10)], base_options("econoserve-full", kvc_capacity=1024))
    assert "request 0" in str(ex.value)
    if backend != "oracle":
        assert isinstance(ex.value, SimulationError)


@pytest.mark.parametrize("backend", BACKENDS)
def test_completion_histogram_matches_event_log(backend):  # test_engine.cpp:296-317
    tr = sat_trace(gen, 200, 40.0, 8, 48, 8, 64, 61)
    e = make_engine(backend, tr, base_options("econoserve-full"))
    e.step(1 << 30)
    _, rep = e.finalize()
    s = e.samples()
    executed = s[s["idle_repeat"] == 0]
    by_iter = {int(it): 0 for it in executed["iter"]}
    for x in e.events():
        if x["kind"] == 5:
            by_iter[int(x["iter"])] += 1
    hist = {}
    for c in by_iter.values():
        hist[c] = hist.get(c, 0.0) + 1.0 / len(executed)
    got = rep.as_dict()["iteration_completion_histogram"]
    assert set(hist) == set(got)
    for c, f in got.items():
        assert abs(hist[c] - f) <= 1e-12


@pytest.mark.parametrize("backend", ["hostsim", pytest.param("device", marks=pytest.mark.gpu)])
@pytest.mark.parametrize("field,value,msg", [
    ("tfs", 0, "tfs must be >= 1"),
    ("reserved_fraction", 1.0, "reserved_fraction must be in [0, 1)"),
    ("t_base", 0.0, "cost model: t_base must be > 0"),
    ("pred_quantum", 0, "predictor quantum must be >= 1"),
    ("pred_accuracy", 1.5, "predictor accuracy must be in [0,1]"),
    ("kvc_block_size", 0, "kvc block_size must be >= 1"),
    ("buffer_ratio", -1.0, "buffer_ratio must be >= 0"),
])
def test_config_errors(backend, field, value, msg):  # policies.hpp:76-84, engine.hpp:36-43, workload.hpp:211-217
    o = base_options("econoserve-full")
    setattr(o, field, value)
    with pytest.raises(ConfigError) as ex:
        make_engine(backend, [(0.1, 10, 10)], o)
    assert msg in str(ex.value)


@pytest.mark.parametrize("backend", ["hostsim", pytest.param("device", marks=pytest.mark.gpu)])
def test_arrival_order_and_empty_trace(backend):  # engine.hpp:97, 167-169
    o = base_options("econoserve-full")
    with pytest.raises(ConfigError, match="nondecreasing"):
        make_engine(backend, [(1.0, 10, 10), (0.5, 10, 10)], o)
    with pytest.raises(ConfigError, match="trace is empty"):
        make_engine(backend, np.zeros(0, dtype=abi.TRACE_DTYPE), o)


@pytest.mark.parametrize("backend", ["hostsim", pytest.param("device", marks=pytest.mark.gpu)])
def test_unknown_policy_code_rejected(backend):
    o = base_options("vllm")
    o.policy = 9
    with pytest.raises(ConfigError, match="unknown policy code 9"):
        make_engine(backend, [(0.1, 10, 10)], o)


@pytest.mark.parametrize("backend", BACKENDS)
def test_exact_allocation_and_pipelining_safety(backend):  # acceptance C1/C2 (oracle part)
    tr = gen(600, 120.0, (20.0, 8, 64, 0.6), (48.0, 8, 256, 0.8), 1)
    o = abi.default_options(policy="econoserve-full", tfs=512, reserved_fraction=0.05,
                            buffer_ratio=0.0, sched_cost_per_exam=0.0, kvc_capacity=8192,
                            kvc_block_size=32)
    e = make_engine(backend, tr, o)
    e.step(1 << 30)
    _, rep = e.finalize()
    assert rep.allocation_failure_pct == 0.0 and rep.preemptions == 0
    assert rep.hosted_slots > 0 and rep.hosted_overruns == 0


@pytest.mark.parametrize("backend", ["hostsim", pytest.param("device", marks=pytest.mark.gpu)])
def test_record_length_range_checked(backend):
    """The device path's per-record range check (k_init_soa on the device,
    the host scan in the host build): the first offending request is named."""
    o = base_options("econoserve-full")
    with pytest.raises(ConfigError, match=r"request 2: prompt_len and response_len must be in \[1, 2\^30\)"):
        make_engine(backend, [(0.1, 10, 10), (0.2, 10, 10), (0.3, 0, 10), (0.4, 10, 0)], o)


def test_instance_bytes_sizing():
    """econo_instance_bytes: the HBM an instance takes (capacity planning)."""
    from paper_2411_06364_b200.engine import instance_bytes
    from conftest import HOSTSIM
    o = base_options("econoserve-full")
    small = instance_bytes([(0.1 * i, 10, 10) for i in range(20000)], o, lib=HOSTSIM)
    big = instance_bytes([(0.1 * i, 10, 10) for i in range(40000)], o, lib=HOSTSIM)
    # beyond the KVC-capacity-sized tables, each request costs its SoA fields
    # (134 B for an econoserve instance)
    assert 0 < small < big and 125 < (big - small) / 20000 < 140
    o.tfs = 0
    with pytest.raises(ConfigError, match="tfs must be >= 1"):
        instance_bytes([(0.1, 10, 10)], o, lib=HOSTSIM)


@pytest.mark.parametrize("backend", ["hostsim", pytest.param("device", marks=pytest.mark.gpu)])
@pytest.mark.parametrize("sigma", [25.0, 60.0])
def test_extreme_lognormal_predictions_match_reference(backend, sigma):
    """Predictions far outside 32 bits: llround's x86 out-of-range value
    (LLONG_MIN -> max(1, .) = 1, s_llround.c) and predicted RLs >= 2^30,
    which the product saturates (engine.cuh kRlSat) and reports with the
    reference's exact int64 demand (engine.hpp:196-202), or which leave the
    run identical when no request is infeasible."""
    from oracle import port
    tr = sat_trace(gen, 300, 50.0, 8, 64, 8, 128, 71)
    opts = base_options("econoserve-full", pred_model="lognormal", pred_sigma=sigma, kvc_capacity=4096)
    try:
        o = port.OracleEngine(tr, opts)
        o.step(1 << 30)
        want = ("ok", o.snapshot())
    except Exception as ex:  # noqa: BLE001 — the reference's SimulationError
        want = ("error", str(ex))
    try:
        e = make_engine(backend, tr, opts)
        e.step(1 << 30)
        got = ("ok", e.snapshot())
    except Exception as ex:  # noqa: BLE001
        got = ("error", str(ex))
    assert got[0] == want[0], (got, want)
    if want[0] == "ok":
        assert np.array_equal(got[1], want[1])
    else:
        assert got[1] == want[1]
