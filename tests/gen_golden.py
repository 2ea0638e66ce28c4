"""Generates the committed golden fixtures in tests/golden/ by running the
UNMODIFIED reference simulator (oracle/_ref/libecono_ref.so, built from
/root/reference by oracle/Makefile). Run in a container that has
/root/reference:  python tests/gen_golden.py

Each engine fixture stores the trace, the EconoOptions bytes, the reference's
event log, iteration samples, request records, aggregate report, a per-step
digest of the canonical state snapshot and the final snapshot. rng.npz holds
libstdc++ known-answer vectors (mt19937_64 draws, std::shuffle permutations,
predict_rl sequences) that pin the restated RNG plumbing.
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from oracle import ref  # noqa: E402
from paper_2411_06364_b200 import abi  # noqa: E402

from parity import base_options, sat_trace  # noqa: E402

OUT = os.path.join(HERE, "golden")


def digest(words):
    return np.frombuffer(hashlib.sha1(np.ascontiguousarray(words).tobytes()).digest()[:8], "<u8")[0]


def engine_cases():
    g = ref.generate_trace
    cases = [
        ("single_request_full", [(0.005, 100, 20)], base_options("econoserve-full")),
        ("prefill_to_gt_sd", [(0.005, 100, 5), (50.0, 10, 5)], base_options("econoserve-sd")),
        ("idle_ticks_full", [(1.0, 10, 5)], base_options("econoserve-full")),
        ("determinism_full_lognormal", sat_trace(g, 300, 40.0, 8, 64, 8, 96, 3),
         base_options("econoserve-full", pred_model="lognormal", pred_sigma=0.3, pred_padding_ratio=0.1)),
        ("determinism_d_lognormal", sat_trace(g, 300, 40.0, 8, 64, 8, 96, 3),
         base_options("econoserve-d", pred_model="lognormal", pred_sigma=0.3, pred_padding_ratio=0.1)),
        ("underprediction_sd_rich", sat_trace(g, 200, 40.0, 8, 40, 16, 120, 31),
         base_options("econoserve-sd", pred_model="lognormal", pred_sigma=0.6, reserved_fraction=0.30)),
        ("underprediction_full_poor", sat_trace(g, 200, 40.0, 8, 40, 16, 120, 31),
         base_options("econoserve-full", pred_model="lognormal", pred_sigma=0.6, reserved_fraction=0.02)),
        ("hosted_full_oracle", sat_trace(g, 500, 250.0, 8, 32, 8, 128, 43), base_options("econoserve-full")),
        ("hosted_sdo_bucket", sat_trace(g, 500, 250.0, 8, 32, 8, 128, 43),
         base_options("econoserve-sdo", pred_model="bucket", pred_accuracy=0.732, pred_tolerance=0.15,
                      pred_padding_ratio=0.15, buffer_ratio=0.15, sched_cost_per_exam=2e-5)),
        ("jct_identity_full", sat_trace(g, 150, 25.0, 8, 60, 8, 64, 19),
         base_options("econoserve-full", sched_cost_per_exam=2e-5, pred_model="lognormal",
                      pred_sigma=0.3, pred_padding_ratio=0.05)),
        ("same_rl_groups_sd", sat_trace(g, 400, 60.0, 8, 32, 8, 48, 41), base_options("econoserve-sd")),
    ]
    return cases


def run_case(name, trace, opts):
    e = ref.RefEngine(trace, opts)
    digs = [digest(e.snapshot())]
    more = True
    while more:
        more = e.step(1)
        digs.append(digest(e.snapshot()))
    recs, rep = e.finalize()
    np.savez_compressed(
        os.path.join(OUT, name + ".npz"), trace=abi.trace_array(trace),
        options=np.frombuffer(bytes(opts), dtype=np.uint8), events=e.events(), samples=e.samples(),
        records=recs, step_digests=np.array(digs, dtype=np.uint64), final_snapshot=e.snapshot(),
        report=np.frombuffer(json.dumps(rep.as_dict()).encode(), dtype=np.uint8))
    print(f"{name}: {len(digs) - 1} steps, {len(e.events())} events")


def rng_vectors():
    from paper_2411_06364_b200 import workloads as W
    mt = {f"mt_{s}": ref.mt_draws(s, 10000) for s in (1, 5489, 1000)}
    sh = {f"shuffle_{s}_{n}": ref.shuffle_indices(s, n) for s in (1, 2, 7) for n in (1, 2, 3, 8, 33, 1000)}
    rl = np.arange(1, 2001, dtype=np.int64)
    pr = {}
    for name, kw in [("lognormal_0.3", dict(pred_model="lognormal", pred_sigma=0.3, pred_padding_ratio=0.1)),
                     ("lognormal_0.6", dict(pred_model="lognormal", pred_sigma=0.6)),
                     ("bucket_0.775", dict(pred_model="bucket", pred_accuracy=0.775, pred_tolerance=0.10)),
                     ("bucket_0.732_q16", dict(pred_model="bucket", pred_accuracy=0.732, pred_tolerance=0.15,
                                               pred_quantum=16, pred_padding_ratio=0.15))]:
        pr["predict_" + name] = ref.predict(abi.default_options(**kw), 11, rl)
    tr = {}
    for cname in ("cfg1_alpaca_10k", "cfg2_sharegpt_100k", "cfg3_bookcorpus_1m"):
        c = W.CONFIGS[cname]
        tr["trace_" + cname] = ref.generate_trace(2000, c["rate"], c["shape"]["prompt"], c["shape"]["rl"], 1)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **mt, **sh, **pr, **tr)
    print("rng vectors:", len(mt) + len(sh) + len(pr) + len(tr))


if __name__ == "__main__":
    assert ref.available(), "oracle/_ref/libecono_ref.so missing: make -C oracle (needs /root/reference)"
    os.makedirs(OUT, exist_ok=True)
    for name, trace, opts in engine_cases():
        run_case(name, trace, opts)
    rng_vectors()
