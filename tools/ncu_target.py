"""Short, ncu-friendly driver for the hot kernel (development tool).

Builds `--instances` cfg-3 instances exactly as bench.py does (trace seeds
1000+i, econoserve-full, 1M-request burst), runs the idle tick + burst ingest,
`--warmup` launches of `--iters` iterations, then `--launches` more. Profile the
last ones with e.g.

  ncu --set full --clock-control none --import-source on -k regex:k_engine_steps \
      -s <1 + warmup> -c 1 -o gpurun_out/prof python tools/ncu_target.py
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2411_06364_b200.engine import Batch, generate_trace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=32)
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--launches", type=int, default=2)
    ap.add_argument("--workload", default=bench.WORKLOAD)
    ap.add_argument("--slice-us", type=float, default=0.0, help="time-sliced launches (the bench's step)")
    a = ap.parse_args()
    bench.WORKLOAD = a.workload
    traces = bench.make_traces(generate_trace, a.n, [1000 + i for i in range(a.instances)])
    b = Batch(traces, bench.options(), device=0)
    b.launch(1)
    b.sync()
    b.ingest()
    b.launch(1)
    b.sync()
    for _ in range(a.warmup + a.launches):
        if a.slice_us > 0:
            b.launch(1 << 40, slice_ns=int(a.slice_us * 1000))
        else:
            b.launch(a.iters)
    b.sync()
    sc = b.scalars()
    print("errors:", sum(1 for s in sc if s.error), "pt_dispatched:", sum(s.pt_dispatched for s in sc),
          "steps:", sum(s.steps for s in sc))


if __name__ == "__main__":
    main()
