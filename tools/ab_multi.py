"""A/B/C... of several builds of the product library in ONE process on the
same traces (dev tool): `--libs A,B,C` loads
paper_2411_06364_b200/_lib/libeconoserve_b200_<X>.so each, alternating rounds."""
import argparse
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_06364_b200.engine import Batch, generate_trace  # noqa: E402


def one(lib, traces, iters=1000, launches=10, warm=3):
    b = Batch(traces, bench.options(), device=0, lib=lib)
    s = torch.cuda.Stream()
    b.launch(1, s.cuda_stream)
    s.synchronize()
    b.ingest()
    b.launch(1, s.cuda_stream)
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
    tot = d.sum(axis=0) // len(traces)
    b.close()
    return 1e3 * ms / launches, adm / ms * 1e3, tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", default="A,B")
    ap.add_argument("--instances", type=int, default=888)
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--rounds", type=int, default=2)
    a = ap.parse_args()
    traces = bench.make_traces(generate_trace, a.n, [1000 + i for i in range(a.instances)], pinned=True)
    for r in range(a.rounds):
        for x in a.libs.split(","):
            lib = os.path.join(ROOT, "paper_2411_06364_b200", "_lib", f"libeconoserve_b200_{x}.so")
            us, rps, tot = one(lib, traces)
            print(f"round {r} {x}: {us:.1f} us/launch {rps / 1e6:.2f}M req/s  test {tot[0]} replay {tot[1]} "
                  f"normal {tot[2]} launch {tot[11]}", flush=True)


if __name__ == "__main__":
    main()
