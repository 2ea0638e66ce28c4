mkdir -p gpurun_out
cat > /tmp/fr.py <<'PY'
import sys, time, os
sys.path.insert(0, os.getcwd())
from paper_2411_06364_b200 import abi, workloads as W
from paper_2411_06364_b200.engine import Engine, generate_trace
for lib in sys.argv[1:]:
    path = f"tools/_prof/lib_{lib}.so"
    c = W.CONFIGS["cfg1_alpaca_10k"]
    for rep in range(3):
        for rec in (1, 0):
            o = abi.default_options(**c["opts"]); o.record_events = rec; o.record_samples = rec
            t = W.make_trace("cfg1_alpaca_10k", generate_trace)
            t0 = time.perf_counter(); e = Engine(t, o, device=0, lib=path); t1 = time.perf_counter(); e.run(); t2 = time.perf_counter()
            print(f"{lib} rep {rep} record={rec}: create {t1-t0:.3f}s run {t2-t1:.3f}s", flush=True)
PY
timeout 900 python /tmp/fr.py nr2 fast fo2 > gpurun_out/r2t_fullruns.log 2>&1
