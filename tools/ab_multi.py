"""A/B/C... of several builds of the product library in ONE process on the
same traces (dev tool). `--libs A,B,C` loads tools/_prof/lib_<X>.so (or a path).
Each build runs the bench's step (time-sliced k_engine_steps launches after
the burst ingest) and reports PT admissions/s; every build's state at a common
step (`--check-step`, reached with econo_batch_launch_to) is digested for the
first `--check` instances, and all builds must agree with the first one."""
import argparse
import hashlib
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_06364_b200.engine import Batch, generate_trace  # noqa: E402


def one(lib, traces, slice_us, launches, check, check_step, warm=3):
    b = Batch(traces, bench.options(), device=0, lib=lib)
    s = torch.cuda.Stream()
    b.launch(1, s.cuda_stream)
    s.synchronize()
    b.ingest()
    b.launch(1, s.cuda_stream)
    b.advance_to(check_step, s.cuda_stream, slice_ns=int(slice_us * 1000))
    dig = [hashlib.sha256(b.snapshot(i).tobytes()).hexdigest()[:16] for i in range(check)]
    for _ in range(warm):
        b.launch(1 << 40, s.cuda_stream, slice_ns=int(slice_us * 1000))
    s.synchronize()
    b.sync()
    sc0, d0 = b.scalars(), b.debug().copy()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(launches):
        b.launch(1 << 40, s.cuda_stream, slice_ns=int(slice_us * 1000))
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    b.sync()
    sc1, d = b.scalars(), b.debug() - d0
    adm = sum(x.pt_dispatched - y.pt_dispatched for x, y in zip(sc1, sc0))
    its = sum(x.steps - y.steps for x, y in zip(sc1, sc0))
    tot = d.sum(axis=0)
    b.close()
    return ms / launches, adm / ms * 1e3, its, tot, dig


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", default="base,uni")
    ap.add_argument("--instances", type=int, default=1184)
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--slice-us", type=float, default=250.0)
    ap.add_argument("--launches", type=int, default=10)
    ap.add_argument("--check", type=int, default=8)
    ap.add_argument("--check-step", type=int, default=3002)
    ap.add_argument("--workload", default=bench.WORKLOAD)
    ap.add_argument("--full-run", default="", help="also time one whole single-engine run of this config per lib")
    a = ap.parse_args()
    bench.WORKLOAD = a.workload
    traces = bench.make_traces(generate_trace, a.n, [1000 + i for i in range(a.instances)], pinned=True)
    ref_dig = None
    for r in range(a.rounds):
        for x in a.libs.split(","):
            lib = x if os.path.sep in x else os.path.join(ROOT, "tools", "_prof", f"lib_{x}.so")
            ms, rps, its, tot, dig = one(lib, traces, a.slice_us, a.launches, a.check, a.check_step)
            ref_dig = ref_dig or dig
            nsteps = max(1, tot[5])
            if a.full_run:
                import time
                from paper_2411_06364_b200 import abi, workloads as W
                from paper_2411_06364_b200.engine import Engine
                c = W.CONFIGS[a.full_run]
                o = abi.default_options(**c["opts"])
                o.record_events = 0
                o.record_samples = 0
                t = W.make_trace(a.full_run, generate_trace)
                t0 = time.perf_counter()
                Engine(t, o, device=0, lib=lib).run()
                print(f"   {x}: whole {a.full_run} run {time.perf_counter() - t0:.3f} s", flush=True)
            print(f"round {r} {x}: {1e3 * ms:.1f} us/launch {rps / 1e6:.2f}M req/s  iters {its}  "
                  f"normal steps {tot[5]} at {tot[2] / nsteps:.0f} cyc, spans {tot[4]} test {tot[0] / max(1, tot[4]):.0f} "
                  f"replay {tot[1] / max(1, its):.1f} cyc/iter  state@{a.check_step} "
                  f"{'SAME' if dig == ref_dig else 'DIFFERENT'}", flush=True)


if __name__ == "__main__":
    main()
