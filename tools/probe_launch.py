import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import make_traces, options
from paper_2411_06364_b200.engine import Batch, generate_trace
I = int(sys.argv[1]) if len(sys.argv) > 1 else 64
trs = make_traces(generate_trace, 1_000_000, [1000 + i for i in range(I)])
b = Batch(trs, options()); b.launch(2); b.sync(); b.checkpoint()
s = torch.cuda.Stream()
for iters in (0, 1, 10, 100, 1000, 5000):
    b.restore()
    for _ in range(3): b.launch(max(iters, 1), s.cuda_stream)
    s.synchronize(); b.sync(); b.restore()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 10 if iters <= 1000 else 2
    d0 = b.debug().sum(axis=0)
    e0.record(s)
    for _ in range(reps): b.launch(iters, s.cuda_stream)
    e1.record(s); e1.synchronize(); b.sync()
    d = b.debug().sum(axis=0) - d0
    ms = e0.elapsed_time(e1) / reps
    print(f"I={I} iters/launch={iters}: {ms*1000:.1f} us/launch, {ms*1000/max(iters,1):.3f} us/iter; cycles/inst/launch: test {d[0]/I/reps:.0f} replay {d[1]/I/reps:.0f} normal {d[2]/I/reps:.0f} (n {d[5]/I/reps:.1f})", flush=True)
