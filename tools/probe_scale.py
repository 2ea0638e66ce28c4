"""Instances-per-GPU / iterations-per-launch sweep of k_engine_steps with the
per-phase device cycle counters (development tool; run under gpurun)."""
import argparse
import os

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_06364_b200.engine import Batch, generate_trace  # noqa: E402

NAMES = ["test", "replay", "normal", "x_runpass", "spans", "nsteps", "ingest", "gtsel", "plan", "pt", "exec",
         "launch", "launches", "x_prefill", "x_transit", "x_tail"]


def run(traces, iters, launches, warm=3, lanes=0):
    t0 = time.time()
    b = Batch(traces, bench.options(), device=0)
    s = torch.cuda.Stream()
    b.launch(1, s.cuda_stream)
    s.synchronize()
    t_ing = time.time()
    b.ingest()
    t_ing = time.time() - t_ing
    b.launch(1, s.cuda_stream)
    s.synchronize()
    t_create = time.time() - t0
    for _ in range(warm):
        b.launch(iters, s.cuda_stream)
    s.synchronize()
    b.sync()
    sc0, d0 = b.scalars(), b.debug().copy()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(launches):
        b.launch(iters, s.cuda_stream)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    b.sync()
    sc1, d = b.scalars(), b.debug() - d0
    adm = sum(x.pt_dispatched - y.pt_dispatched for x, y in zip(sc1, sc0))
    I = len(traces)
    tot = d.sum(axis=0)
    per = {NAMES[k]: int(tot[k]) // I for k in range(len(NAMES)) if NAMES[k] != "-"}
    print(f"inst={I} iters={iters} launches={launches} lanes={lanes}: {ms:.3f} ms total, {1e3 * ms / launches:.1f} us/launch, "
          f"{1e3 * ms / (launches * iters):.3f} us/iter, adm={adm} -> {adm / ms * 1e3:.0f} req/s, "
          f"create+ingest {t_create:.2f}s (bulk ingest {1e3 * t_ing:.1f} ms), launch cycles max {int(d[:, 11].max())}", flush=True)
    print("   per-instance cycles:", per, flush=True)
    b.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--counts", default="148,296,444,592,740")
    ap.add_argument("--iters", default="100,1000")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--lanes", default="0")
    a = ap.parse_args()
    counts = [int(x) for x in a.counts.split(",")]
    t0 = time.time()
    traces = bench.make_traces(generate_trace, a.n, [1000 + i for i in range(max(counts))], pinned=True)
    print(f"tracegen {time.time() - t0:.1f}s", flush=True)
    for c in counts:
        for it in [int(x) for x in a.iters.split(",")]:
            for ln in [int(x) for x in a.lanes.split(",")]:
                run(traces[:c], it, max(1, 1000 // it) * 10 if it < 1000 else 10, lanes=ln)


if __name__ == "__main__":
    main()
