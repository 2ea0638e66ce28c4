"""Quick device timing probe (development tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from concurrent.futures import ThreadPoolExecutor
import numpy as np
import torch
from paper_2411_06364_b200 import abi, workloads as W
from paper_2411_06364_b200.engine import Batch, Engine, generate_trace

def traces(cfg, n, k, seed0):
    c = W.CONFIGS[cfg]
    with ThreadPoolExecutor(16) as ex:
        return list(ex.map(lambda i: generate_trace(n, c["rate"], c["shape"]["prompt"], c["shape"]["rl"], seed0 + i), range(k)))

def probe(cfg, n, k, windows=5, K=1000):
    c = W.CONFIGS[cfg]
    t0 = time.time(); trs = traces(cfg, n, k, 1000); t1 = time.time()
    o = abi.default_options(**c["opts"]); o.record_events = 0; o.record_samples = 0
    b = Batch(trs, o); torch.cuda.synchronize(); t2 = time.time()
    print(f"{cfg} n={n} inst={k}: tracegen {t1-t0:.2f}s create+init {t2-t1:.2f}s", flush=True)
    s = torch.cuda.Stream()
    for w in range(windows + 2):
        st = 2 if w == 0 else K
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        sc0 = b.scalars() if w else None
        e0.record(s); b.launch(st, s.cuda_stream); e1.record(s); e1.synchronize(); b.sync()
        ms = e0.elapsed_time(e1); sc = b.scalars()
        it = np.mean([x.iter for x in sc]); pt = sum(x.pt_dispatched for x in sc); q = np.mean([x.pt_queue_len for x in sc])
        print(f"  launch {w}: steps {st} {ms:.3f} ms  ({1000*ms/st:.2f} us/step)  iter={it:.0f} pt_dispatched={pt} q={q:.0f} running={np.mean([x.running for x in sc]):.1f} err={[x.error for x in sc][:3]}", flush=True)

if __name__ == "__main__":
    probe("cfg3_bookcorpus_1m", 1_000_000, 1)
    probe("cfg3_bookcorpus_1m", 1_000_000, 64, windows=3)
    probe("cfg2_sharegpt_100k", 100_000, 1, windows=3)
