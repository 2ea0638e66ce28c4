"""Fixed-iteration launches vs time-sliced launches (econo_batch_launch_slice)
on the bench configuration (dev tool)."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_06364_b200.engine import Batch, generate_trace  # noqa: E402


def window(b, s, launches, iters, slice_ns):
    b.sync()
    sc0 = b.scalars()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(launches):
        b.launch(iters if not slice_ns else 1 << 40, s.cuda_stream, slice_ns=slice_ns)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    b.sync()
    sc1 = b.scalars()
    adm = sum(x.pt_dispatched - y.pt_dispatched for x, y in zip(sc1, sc0))
    st = [x.steps - y.steps for x, y in zip(sc1, sc0)]
    return ms, adm, sum(st) / len(st), min(st), max(st)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=1184)
    ap.add_argument("--slices", default="250,500,1000")
    a = ap.parse_args()
    traces = bench.make_traces(generate_trace, 1_000_000, [1000 + i for i in range(a.instances)], pinned=True)
    b = Batch(traces, bench.options(), device=0)
    s = torch.cuda.Stream()
    b.launch(1, s.cuda_stream)
    s.synchronize()
    b.ingest()
    b.launch(1, s.cuda_stream)
    for _ in range(3):
        b.launch(1000, s.cuda_stream)
    s.synchronize()
    for rep in range(2):
        ms, adm, avg, lo, hi = window(b, s, 10, 1000, 0)
        print(f"fixed 1000: {ms / 10 * 1e3:.1f} us/launch {adm / ms * 1e3 / 1e6:.2f}M req/s steps/inst avg {avg:.0f} [{lo},{hi}]", flush=True)
        for sl in [int(x) for x in a.slices.split(",")]:
            ms, adm, avg, lo, hi = window(b, s, 10, 1000, sl * 1000)
            print(f"slice {sl} us: {ms / 10 * 1e3:.1f} us/launch {adm / ms * 1e3 / 1e6:.2f}M req/s "
                  f"steps/inst avg {avg:.0f} [{lo},{hi}]", flush=True)


if __name__ == "__main__":
    main()
