"""Sweep-style throughput of every policy on the device (dev tool): a batch of
`--instances` cfg-1 Alpaca instances (trace seeds 1000+i) run to completion
per policy, against the compiled reference running one instance per policy
on one host core."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2411_06364_b200 import abi, workloads as W  # noqa: E402
from paper_2411_06364_b200.engine import Batch, Engine, generate_trace  # noqa: E402

POLICIES = ["orca", "vllm", "sarathi", "multires", "sync-coupled", "econoserve-sd", "econoserve-full"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=148)
    ap.add_argument("--config", default="cfg1_alpaca_10k")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--policies", default=",".join(POLICIES))
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    c = W.CONFIGS[a.config]
    n = a.n or c["n"]
    Engine([(0.0, 10, 10)], abi.default_options()).run()  # context + module load
    traces = [generate_trace(n, c["rate"], c["shape"]["prompt"], c["shape"]["rl"], 1000 + i)
              for i in range(a.instances)]
    out = {}
    for pol in a.policies.split(","):
        o = abi.default_options(**dict(c["opts"], policy=pol, record_events=0, record_samples=0))
        t0 = time.perf_counter()
        b = Batch(traces, o, device=0)
        t1 = time.perf_counter()
        while True:
            b.launch(1 << 20)
            b.sync()
            sc = b.scalars()
            if all(s.completed >= n or s.error for s in sc):
                break
        t2 = time.perf_counter()
        errs = sum(1 for s in sc if s.error)
        steps = sum(s.steps for s in sc)
        b.close()
        r = dict(device_run_s=round(t2 - t1, 4), create_s=round(t1 - t0, 3), errors=errs,
                 steps_per_instance=steps // a.instances,
                 device_req_per_s=round(a.instances * n / (t2 - t1)))
        if not a.no_ref and ref.available():
            e = ref.RefEngine(traces[0], o)
            t3 = time.perf_counter()
            try:
                e.run()
            except ref.EngineError as x:
                r["ref_error"] = str(x)[:80]
            r["ref_one_instance_s"] = round(time.perf_counter() - t3, 4)
            r["ref_req_per_s_per_core"] = round(n / r["ref_one_instance_s"])
        out[pol] = r
        print(pol, json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
