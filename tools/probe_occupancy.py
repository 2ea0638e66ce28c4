"""Instances-per-SM sweep of the time-sliced bench step (dev tool): how PT
admissions/s scale with resident warps per SM. Uses --n requests per
instance so that the largest count fits in HBM (per-step work is O(takes),
not O(queue length), so the queue depth barely matters)."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_06364_b200.engine import Batch, generate_trace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--counts", default="1184,2368,3552,4736")
    ap.add_argument("--n", type=int, default=150_000)
    ap.add_argument("--slice-us", type=float, default=250.0)
    ap.add_argument("--launches", type=int, default=10)
    ap.add_argument("--lib", default=None)
    a = ap.parse_args()
    counts = [int(x) for x in a.counts.split(",")]
    traces = bench.make_traces(generate_trace, a.n, [1000 + i for i in range(max(counts))], pinned=True)
    sl = int(a.slice_us * 1000)
    for c in counts:
        b = Batch(traces[:c], bench.options(), device=0, lib=a.lib)
        s = torch.cuda.Stream()
        b.launch(1, s.cuda_stream)
        s.synchronize()
        b.ingest()
        b.launch(1, s.cuda_stream)
        for _ in range(3):
            b.launch(1 << 40, s.cuda_stream, slice_ns=sl)
        s.synchronize()
        b.sync()
        sc0 = b.scalars()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.launches):
            b.launch(1 << 40, s.cuda_stream, slice_ns=sl)
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        b.sync()
        sc1 = b.scalars()
        adm = sum(x.pt_dispatched - y.pt_dispatched for x, y in zip(sc1, sc0))
        its = sum(x.steps - y.steps for x, y in zip(sc1, sc0))
        print(f"instances {c} ({c / 148:.0f}/SM): {adm / ms * 1e3 / 1e6:.2f}M req/s, {its / ms * 1e3 / 1e9:.2f}G iter/s, "
              f"{ms / a.launches * 1e3:.0f} us/launch", flush=True)
        b.close()


if __name__ == "__main__":
    main()
