"""Parity case catalogue: (name, trace factory, options) built from the
reference's own test fixtures (tests/test_engine.cpp, acceptance_main.cpp) and
the BASELINE.json config shapes at sizes the oracle finishes in seconds."""
from paper_2411_06364_b200 import abi, workloads as W

from parity import base_options, sat_trace


def catalogue(gen):
    """gen(n, rate, prompt_dist, rl_dist, seed) -> trace."""
    cases = []
    tr = sat_trace(gen, 300, 40.0, 8, 64, 8, 96, 3)  # test_engine.cpp:110-125
    for k in ["econoserve-full", "econoserve-sd", "econoserve-d", "econoserve-sdo"]:
        cases.append((f"determinism-{k}", tr, base_options(
            k, pred_model="lognormal", pred_sigma=0.3, pred_padding_ratio=0.1)))
    tr = sat_trace(gen, 200, 40.0, 8, 40, 16, 120, 31)  # test_engine.cpp:181-206
    for k, rf in [("econoserve-sd", 0.30), ("econoserve-sd", 0.02), ("econoserve-full", 0.02),
                  ("econoserve-d", 0.02)]:
        cases.append((f"underprediction-{k}-rf{rf}", tr, base_options(
            k, pred_model="lognormal", pred_sigma=0.6, reserved_fraction=rf)))
    tr = sat_trace(gen, 500, 250.0, 8, 32, 8, 128, 43)  # test_engine.cpp:233-241
    cases.append(("hosted-oracle-full", tr, base_options("econoserve-full")))
    for k in ["econoserve-full", "econoserve-sdo"]:
        cases.append((f"hosted-bucket-{k}", tr, base_options(
            k, pred_model="bucket", pred_accuracy=0.732, pred_tolerance=0.15,
            pred_padding_ratio=0.15, buffer_ratio=0.15, sched_cost_per_exam=2e-5)))
    tr = sat_trace(gen, 150, 25.0, 8, 60, 8, 64, 19)  # test_engine.cpp:147-162
    cases.append(("jct-identity", tr, base_options(
        "econoserve-full", sched_cost_per_exam=2e-5, pred_model="lognormal", pred_sigma=0.3,
        pred_padding_ratio=0.05)))
    tr = sat_trace(gen, 400, 60.0, 8, 32, 8, 48, 41)  # test_engine.cpp:208-231
    cases.append(("same-rl-groups", tr, base_options("econoserve-sd")))
    c = W.CONFIGS["cfg1_alpaca_10k"]
    a = gen(3000, 400.0, c["shape"]["prompt"], c["shape"]["rl"], 5)  # SURVEY §8a saturated Alpaca
    for pm, extra in [("bucket", dict(pred_accuracy=0.775, pred_tolerance=0.10)),
                      ("lognormal", dict(pred_sigma=0.3))]:
        for pol in ["econoserve-full", "econoserve-sd"]:
            cases.append((f"alpaca400-{pm}-{pol}", a, abi.default_options(
                **dict(c["opts"], policy=pol, pred_model=pm, **extra))))
    s = W.CONFIGS["cfg2_sharegpt_100k"]
    sg = gen(1500, 60.0, s["shape"]["prompt"], s["shape"]["rl"], 2)
    cases.append(("sharegpt-cfg2-shape", sg, abi.default_options(**s["opts"])))
    b = W.CONFIGS["cfg3_bookcorpus_1m"]
    bk = gen(300, 1e9, b["shape"]["prompt"], b["shape"]["rl"], 1)
    cases.append(("bookcorpus-cfg3-shape-burst", bk, abi.default_options(**b["opts"])))
    cases.append(("bookcorpus-cfg3-shape-burst-sd", bk, abi.default_options(
        **dict(b["opts"], policy="econoserve-sd"))))
    m = W.CONFIGS["cfg4_mixed_1m"]  # configs[3]: mixed trace, predictor error sweep (SURVEY §8(d) cfg 4)
    mx = W.make_trace("cfg4_mixed_1m", gen, n=600, seed=7)
    for tag, extra in [("lognormal0.1", dict(pred_sigma=0.1)),
                       ("lognormal0.6-pad0.25", dict(pred_sigma=0.6, pred_padding_ratio=0.25)),
                       ("bucket0.732-pad0.15", dict(pred_model="bucket", pred_accuracy=0.732, pred_tolerance=0.15,
                                                    pred_padding_ratio=0.15)),
                       ("sd-lognormal0.3", dict(policy="econoserve-sd", pred_sigma=0.3))]:
        cases.append((f"mixed-cfg4-{tag}", mx, abi.default_options(**dict(m["opts"], **extra))))
    return cases


BASELINES = ["orca", "vllm", "sarathi", "multires", "sync-coupled"]


def baseline_catalogue(gen):
    """The comparison policies (engine.hpp:383-726) on the reference's own
    test traces and the BASELINE config shapes; checked against the compiled
    reference (oracle/_ref)."""
    cases = []
    tr = sat_trace(gen, 300, 40.0, 8, 64, 8, 96, 3)  # test_engine.cpp:110-125
    for k in BASELINES:
        cases.append((f"determinism-{k}", tr, base_options(
            k, pred_model="lognormal", pred_sigma=0.3, pred_padding_ratio=0.1)))
    tr = sat_trace(gen, 120, 200.0, 16, 64, 32, 128, 59)  # test_engine.cpp:272-283 (tight cache)
    cases.append(("pressure-vllm", tr, base_options("vllm", kvc_capacity=2048)))
    cases.append(("pressure-vllm-stall", tr, base_options("vllm", kvc_capacity=2560, swap_stall=0.002)))
    cases.append(("pressure-sarathi-chunk48", tr, base_options(
        "sarathi", kvc_capacity=2048, chunk_size=48, swap_stall=0.001)))
    cases.append(("pressure-sarathi-recompute", tr, base_options(
        "sarathi", kvc_capacity=2048, chunk_size=40, vllm_recompute=1)))
    tr = sat_trace(gen, 40, 1000.0, 8, 32, 8, 32, 53)  # test_engine.cpp:254-270
    cases.append(("orca-cap8", tr, base_options("orca", batch_size_cap=8)))
    cases.append(("orca-cap3-maxout", tr, base_options("orca", batch_size_cap=3, max_output_len=40)))
    tr = sat_trace(gen, 200, 40.0, 8, 40, 16, 120, 31)  # test_engine.cpp:181-206 shape
    for k in ["multires", "sync-coupled", "orca"]:
        cases.append((f"underprediction-{k}", tr, base_options(
            k, pred_model="lognormal", pred_sigma=0.6, kvc_capacity=4096)))
    tr = sat_trace(gen, 300, 80.0, 8, 48, 16, 64, 47)  # test_engine.cpp:243-252
    cases.append(("gt-domination-sync-coupled", tr, base_options("sync-coupled")))
    c = W.CONFIGS["cfg1_alpaca_10k"]
    a = gen(3000, 400.0, c["shape"]["prompt"], c["shape"]["rl"], 5)
    for pol in ["vllm", "sarathi", "multires"]:
        cases.append((f"alpaca400-{pol}", a, abi.default_options(**dict(c["opts"], policy=pol))))
    m = W.CONFIGS["cfg4_mixed_1m"]
    mx = W.make_trace("cfg4_mixed_1m", gen, n=600, seed=7)
    for pol in BASELINES:
        cases.append((f"mixed-cfg4-{pol}", mx, abi.default_options(**dict(m["opts"], policy=pol, pred_sigma=0.3))))
    return cases
