"""Times the end-of-run reduction kernels on the bench's 740 x 1M batch:
grid-wide partial sums, JCT key materialisation and the 6 radix-select
histogram passes (development tool; run under gpurun)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_06364_b200 import metrics  # noqa: E402
from paper_2411_06364_b200.engine import Batch, generate_trace  # noqa: E402

I = int(os.environ.get("INST", "740"))
traces = bench.make_traces(generate_trace, 1_000_000, [1000 + i for i in range(I)], pinned=True)
b = Batch(traces, bench.options(), device=0)
b.launch(1)
b.sync()
b.ingest()
b.launch(1)
b.launch(1000)
b.sync()
for rep in range(3):
    t0 = time.perf_counter(); p = b.partials(); t1 = time.perf_counter()
    b.jct_prepare(); torch.cuda.synchronize(); t2 = time.perf_counter()
    pct = metrics.global_percentiles(b, [0.05, 0.95]); t3 = time.perf_counter()
    print(f"partials {1e3*(t1-t0):.2f} ms, jct_prepare {1e3*(t2-t1):.2f} ms, global p5/p95 {1e3*(t3-t2):.2f} ms "
          f"(incl. a second prepare) -> {pct}", flush=True)
t0 = time.perf_counter(); reps = b.reports(); t1 = time.perf_counter()
print(f"batch reports {1e3*(t1-t0):.1f} ms; inst0 p5 {reps[0].p5_jct} p95 {reps[0].p95_jct}")
