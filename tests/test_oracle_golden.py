"""The C oracle (oracle/econo_oracle.c) pinned against golden vectors made by
the UNMODIFIED reference (tests/gen_golden.py -> tests/golden/) and, where the
compiled reference is present (oracle/_ref), against it directly."""
import glob
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import port, ref
from paper_2411_06364_b200 import abi, workloads as W

from cases import catalogue
from parity import lockstep

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIXTURES = sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.npz")) if not p.endswith("rng.npz"))


def digest(words):
    return np.frombuffer(hashlib.sha1(np.ascontiguousarray(words).tobytes()).digest()[:8], "<u8")[0]


def load_fixture(path):
    z = np.load(path)
    opts = abi.Options.from_buffer_copy(z["options"].tobytes())
    return z, opts


def check_engine_against_fixture(e, z):
    digs = z["step_digests"]
    assert digest(e.snapshot()) == digs[0]
    more, k = True, 0
    while more:
        more = e.step(1)
        k += 1
        assert digest(e.snapshot()) == digs[k], f"state digest differs after step {k}"
    assert k == len(digs) - 1
    assert np.array_equal(e.events(), z["events"])
    assert np.array_equal(e.samples(), z["samples"])
    recs, rep = e.finalize()
    assert np.array_equal(recs, z["records"])
    exp = json.loads(z["report"].tobytes().decode())
    got = rep.as_dict()
    for key, v in exp.items():
        if key == "iteration_completion_histogram":
            assert {int(a): b for a, b in v.items()} == got[key]
        else:
            assert got[key] == v, key
    assert np.array_equal(e.snapshot(), z["final_snapshot"])


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[:-4] for p in FIXTURES])
def test_oracle_matches_reference_fixture(path):
    z, opts = load_fixture(path)
    check_engine_against_fixture(port.OracleEngine(z["trace"], opts), z)


def test_fixtures_present():
    assert len(FIXTURES) >= 10


def test_mt19937_64_standard_known_answer():
    # C++ [rand.predef]: the 10000th invocation of a default-constructed
    # mt19937_64 produces 9981545732273789042.
    assert int(port.mt_draws(5489, 10000)[-1]) == 9981545732273789042


def test_rng_vectors():
    z = np.load(os.path.join(GOLDEN, "rng.npz"))
    for k in z.files:
        if k.startswith("mt_"):
            seed = int(k.split("_")[1])
            assert np.array_equal(port.mt_draws(seed, len(z[k])), z[k]), k
        elif k.startswith("shuffle_"):
            _, seed, n = k.split("_")
            assert np.array_equal(port.shuffle_indices(int(seed), int(n)), z[k]), k
    rl = np.arange(1, 2001, dtype=np.int64)
    for name, kw in [("lognormal_0.3", dict(pred_model="lognormal", pred_sigma=0.3, pred_padding_ratio=0.1)),
                     ("lognormal_0.6", dict(pred_model="lognormal", pred_sigma=0.6)),
                     ("bucket_0.775", dict(pred_model="bucket", pred_accuracy=0.775, pred_tolerance=0.10)),
                     ("bucket_0.732_q16", dict(pred_model="bucket", pred_accuracy=0.732,
                                               pred_tolerance=0.15, pred_quantum=16,
                                               pred_padding_ratio=0.15))]:
        got = port.predict(abi.default_options(**kw), 11, rl)
        assert np.array_equal(got, z["predict_" + name]), name


def test_trace_generator_vectors():
    z = np.load(os.path.join(GOLDEN, "rng.npz"))
    for cname in ("cfg1_alpaca_10k", "cfg2_sharegpt_100k", "cfg3_bookcorpus_1m"):
        c = W.CONFIGS[cname]
        t = port.generate_trace(2000, c["rate"], c["shape"]["prompt"], c["shape"]["rl"], 1)
        assert np.array_equal(t, z["trace_" + cname]), cname


needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
@pytest.mark.parametrize("name,trace,opts", catalogue(ref.generate_trace) if ref.available() else [],
                         ids=[c[0] for c in catalogue(ref.generate_trace)] if ref.available() else [])
def test_oracle_lockstep_vs_compiled_reference(name, trace, opts):
    lockstep(ref.RefEngine(trace, opts), port.OracleEngine(trace, opts), every=7)


@needs_ref
def test_oracle_cfg1_full_run_vs_reference():
    c = W.CONFIGS["cfg1_alpaca_10k"]
    t = ref.generate_trace(c["n"], c["rate"], c["shape"]["prompt"], c["shape"]["rl"], c["seed"])
    opts = abi.default_options(**c["opts"])
    lockstep(ref.RefEngine(t, opts), port.OracleEngine(t, opts), every=1 << 40)


@needs_ref
def test_fast_ingest_equals_ingest_arrivals():
    """The bench's CPU-baseline route (ref_fast_ingest) builds the same
    post-ingest state as the reference's own ingest_arrivals."""
    c = W.CONFIGS["cfg3_bookcorpus_1m"]
    t = ref.generate_trace(3000, c["rate"], c["shape"]["prompt"], c["shape"]["rl"], 4)
    for pol in ("econoserve-full", "econoserve-sd"):
        opts = abi.default_options(**dict(c["opts"], policy=pol))
        a, b = ref.RefEngine(t, opts), ref.RefEngine(t, opts)
        a.step(3)
        b.idle_to_first_arrival()
        b.fast_ingest()
        b.step(2)
        assert np.array_equal(a.snapshot(), b.snapshot())
        assert np.array_equal(a.events(), b.events())


@needs_ref
def test_event_detail_strings_match_reference():
    """The integer event encoding renders back to the reference's exact
    kind/detail strings (engine.hpp:221-948)."""
    from parity import base_options, sat_trace
    tr = sat_trace(ref.generate_trace, 200, 40.0, 8, 40, 16, 120, 31)
    o = base_options("econoserve-full", pred_model="lognormal", pred_sigma=0.6, reserved_fraction=0.02)
    e = ref.RefEngine(tr, o)
    e.run()
    ev = e.events()
    seen = set()
    for i in range(len(ev)):
        k, d = e.event_detail(i)
        assert abi.event_str(ev[i]) == (k, d)
        seen.add(k)
    assert {"preempt", "reserve_topup", "complete", "gt_schedule", "prefill_done", "idle"} <= seen
