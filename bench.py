"""EconoServe per-iteration scheduling step on B200 — benchmark (driver contract).

Workload (BASELINE.json configs[2], the "1M queued" case the metric is quoted
on): BookCorpus-shaped synthetic trace, 1M requests arriving as one burst,
Llama-2-13B KVC (14,648 tokens, 16-token blocks, 14% reserve), tfs 4096,
econoserve-full (SLO-priority selection + GT grouping + KVC pipelining),
oracle predictor. Each GPU runs `--instances` independent serving instances
(one warp each; instance i uses trace seed 1000 + global index), so per-GPU
work is fixed as N grows ("scaling": "weak").

A step = one device pass advancing every instance by `--iters` scheduler
iterations (Engine::step(), engine.hpp:104-116) with 1M requests queued.
value = PT admissions (pt_dispatch, engine.hpp:380) per second over all GPUs;
us_per_iter = per-instance wall time of one scheduler iteration.

`--workload` selects another BASELINE.json config (cfg4_mixed_1m: the mixed
Alpaca/ShareGPT/BookCorpus 1M burst with the lognormal predictor, i.e. the
preemption path; cfg2_sharegpt_100k, cfg1_alpaca_10k); the default is the
metric's own 1M-queued case.

`--impl reference` times the unmodified reference simulator (oracle/_ref,
compiled from /root/reference by oracle/Makefile) on the host cores on the
same config: one engine per thread, each step a bounded window of iterations.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2411_06364_b200 import abi, metrics, workloads as W  # noqa: E402

METRIC = "scheduled requests/sec & us per scheduler iteration at 1M queued reqs; % HBM BW"
UNIT = "req/s"
WORKLOAD = "cfg3_bookcorpus_1m"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def options(record=False):
    o = abi.default_options(**W.CONFIGS[WORKLOAD]["opts"])
    o.record_events = 1 if record else 0
    o.record_samples = 1 if record else 0
    return o


def make_traces(gen, n, seeds, threads=32, pinned=False, soa=False):
    """One synthetic trace of the workload per seed (workloads.make_trace).
    pinned=True generates straight into one page-locked host buffer (the e2e
    contract: inputs copied from pinned host memory), returned as views.
    soa=True (with pinned): each trace as three page-locked columns
    (abi.SoaTrace: arrival f64, prompt i32, true_rl i32 — the device layout,
    16 B per request; econo_batch_create_soa uploads them as they are)."""
    outs = [None] * len(seeds)
    if pinned and soa:
        import torch
        m = len(seeds) * n
        ca = torch.empty(m, dtype=torch.float64, pin_memory=True).numpy()
        cp = torch.empty(m, dtype=torch.int32, pin_memory=True).numpy()
        cr = torch.empty(m, dtype=torch.int32, pin_memory=True).numpy()

        def one(a):
            i, seed = a
            t = W.make_trace(WORKLOAD, gen, n=n, seed=seed)
            sl = slice(i * n, (i + 1) * n)
            return abi.SoaTrace.from_records(t, out=(ca[sl], cp[sl], cr[sl]))
        with ThreadPoolExecutor(threads) as ex:
            return list(ex.map(one, enumerate(seeds)))
    if pinned:
        import torch
        rec = abi.TRACE_DTYPE.itemsize
        buf = torch.empty(len(seeds) * n * rec, dtype=torch.uint8, pin_memory=True).numpy()
        outs = [buf[i * n * rec:(i + 1) * n * rec].view(abi.TRACE_DTYPE) for i in range(len(seeds))]
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(lambda a: W.make_trace(WORKLOAD, gen, n=n, seed=a[0], out=a[1]), zip(seeds, outs)))


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML by a
    thread polling every millisecond, started right before the timed steps
    and stopped right after them (plus one sample at each end). In-process
    NVML reads replace an `nvidia-smi -lms` subprocess, whose periodic queries
    stalled CUDA calls of the job for up to ~0.5 s."""
    REASONS = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4)]

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.h = None
        self.stop_ev = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 — no NVML: no clock record
            self.h = None

    def _sample(self):
        nv = self.nv
        try:
            try:
                reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except AttributeError:
                reasons = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM), reasons))
        except Exception:  # noqa: BLE001 — a failed read is skipped
            pass

    def _loop(self):
        while not self.stop_ev.wait(0.001):
            self._sample()

    def start(self):
        if self.h is None:
            return
        self._sample()
        self.thread = threading.Thread(target=self._loop, daemon=True)
        self.thread.start()

    def stop(self):
        if self.h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.stop_ev.set()
        self.thread.join(timeout=2)
        self._sample()
        reasons = sorted({nm for _, r in self.rows for nm, bit in self.REASONS if r & bit})
        return {"sm_mhz": float(np.median([c for c, _ in self.rows])) if self.rows else None,
                "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, 1 ms polling over the timed steps"}


def measured_traffic(instances, slice_us):
    """ncu DRAM bytes and duration per k_engine_steps launch of this exact
    configuration (profiles/r02_traffic.json, made by tools/make_traffic.py
    from the committed launch list), else None."""
    p = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    c = d.get("config", {})
    if c.get("instances_per_gpu") == instances and c.get("slice_us") == slice_us and \
            c.get("workload") == WORKLOAD:
        return d
    return None


def roofline_block(abytes, secs, launches, inst, slice_us, counts, dbg, peak, peak_kind):
    """The dominant kernel's roofline: algorithmic bytes per launch (what the
    executed work must touch, algorithmic_bytes) over the measured launch
    time against the measured HBM copy bandwidth; the ncu DRAM bytes of the
    same configuration beside it; and the latency view that actually bounds
    a one-warp-per-instance dependency chain (cycles per event step)."""
    achieved = abytes / secs / 1e9
    tr = measured_traffic(inst, slice_us)
    normal = max(1, counts["normal_steps"])
    blk = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "traffic": tr["dram_bytes_per_launch"] if tr else None,
           "per_launch_algorithmic_bytes": abytes / launches, "peak_kind": peak_kind, "kernel": "k_engine_steps",
           "work_counts": counts,
           "latency": {"normal_step_cycles": float(dbg[2]) / normal,
                       "quiet_test_cycles": float(dbg[0]) / max(1, counts["spans"]),
                       "replay_cycles_per_span": float(dbg[1]) / max(1, counts["spans"]),
                       "l2_hit_latency_cycles": 262,
                       "normal_step_in_l2_round_trips": float(dbg[2]) / normal / 262,
                       "note": "one warp per instance runs a dependent chain; the bound is its latency, not "
                               "HBM bandwidth (issue slots ~10% busy, ncu profiles/r02_*)"},
           "note": "algorithmic bytes per executed unit (normal step, replayed span, admission, schedule, "
                   "completion; DESIGN.md §5), not per simulated iteration: a replay keeps the span in "
                   "registers"}
    if tr:
        blk["dram_achieved"] = tr["dram_bytes_per_launch"] / (tr["ncu_ns_per_launch"] * 1e-9) / 1e9
        blk["dram_frac"] = blk["dram_achieved"] / peak
        blk["traffic_source"] = tr.get("source")
    return blk


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


# --------------------------------------------------------------------------
# CPU baseline: the reference itself (oracle/_ref) on the host cores
# --------------------------------------------------------------------------
def reference_windows(n, threads, window, reps, warmup, digests=0):
    """Builds `threads` reference engines on the workload (trace seeds
    1000+i), ingests the 1M burst (oracle/ref_driver.cpp ref_fast_ingest —
    same post-ingest state as ingest_arrivals), runs `warmup` untimed windows
    of `window` step() calls (the device arm's warm-up ends at the same
    step), then times `reps` windows on one std::thread per engine. With
    digests > 0 the first engines' complete-state snapshot digests are taken
    at the end of the warm-up, where the device arm takes its own. Returns
    (per-window (seconds, admissions) list, setup seconds, digests)."""
    import ctypes as C

    from oracle import ref
    t0 = time.time()
    traces = make_traces(ref.generate_trace, n, [1000 + i for i in range(threads)], threads)
    o = options(record=True)  # the reference's default EngineOptions logs events
    with ThreadPoolExecutor(threads) as ex:
        engines = list(ex.map(lambda t: ref.RefEngine(t, o), traces))
    for e in engines:
        e.idle_to_first_arrival()
        e.fast_ingest()
        e.step(1)  # form + execute of the ingest step
    setup = time.time() - t0
    pts = np.zeros(threads, dtype=np.int64)
    hv = (C.c_void_p * threads)(*[e.h.value for e in engines])
    for _ in range(warmup):  # the same warm-up window the device arm runs
        ref.lib().ref_time_steps_parallel(hv, threads, window, pts.ctypes.data)
    dig = []
    if digests:
        with ThreadPoolExecutor(min(threads, digests)) as ex:
            dig = list(ex.map(lambda e: snapshot_digest(e.snapshot()), engines[:digests]))
    out = []
    for r in range(reps):
        secs = ref.lib().ref_time_steps_parallel(hv, threads, window, pts.ctypes.data)
        out.append((secs, int(pts.sum())))
    return out, setup, dig


def timed_start_step(args):
    """Engine::step() calls every instance has made when the timed steps
    begin, in both arms: the idle tick, the ingest step, then `warmup`
    windows of ref_iters steps."""
    return 2 + args.ref_iters * args.warmup


def snapshot_digest(snap):
    import hashlib
    return len(snap), hashlib.sha256(np.ascontiguousarray(snap).tobytes()).hexdigest()


def parity_block(dev_digests, ref_digests, step):
    """Device instances 0..k-1 of the benchmarked batch (trace seeds 1000+i)
    against the reference engines of the CPU baseline (the same seeds), both
    at Engine::step() call `step`: the canonical snapshot (DESIGN.md §8:
    block tables, free gaps, slots, both queues in order, reserve/written
    maps, the running order, 23 words per request) compared by SHA-256."""
    k = min(len(dev_digests), len(ref_digests))
    equal = [dev_digests[i] == ref_digests[i] for i in range(k)]
    return {"instances_checked": k, "iterations": step, "equal": bool(k) and all(equal),
            "mismatched": [i for i, e in enumerate(equal) if not e],
            "how": "the benchmarked batch itself (same burst ingest, same time-sliced launches) at the end of "
                   f"its warm-up (step {step}, where the timed steps start); its first {k} instances' "
                   "complete-state snapshots compared (SHA-256) with the unmodified reference (oracle/_ref) "
                   "engines of cpu_baseline at the end of their warm-up, the same step"}


def window_str(args, iters=None):
    it = iters or args.iters
    lo = 2 + it * args.warmup
    return f"scheduler iterations {lo}..{lo + it * args.steps} after the 1M burst ingest"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = args.ref_threads or min(os.cpu_count() or 1, 32)
    wins, setup, _ = reference_windows(args.n, threads, args.ref_iters, args.steps, args.warmup)
    secs = sum(w[0] for w in wins)
    adm = sum(w[1] for w in wins)
    value = adm / secs if secs > 0 else 0.0
    us_iter = 1e6 * secs / (args.ref_iters * len(wins))
    sample = (f"{threads} reference engines (one std::thread each) x {args.n} requests "
              f"({WORKLOAD}), a bounded sample of {args.ref_iters} step() calls per engine per step "
              f"(~28 ms each at 1M queued); after {args.warmup} warm-up steps the {args.steps} timed "
              f"steps cover {window_str(args, args.ref_iters)}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / len(wins), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "requests_per_instance": args.n, "instances": threads,
                   "iters_per_step": args.ref_iters, "policy": W.CONFIGS[WORKLOAD]["opts"]["policy"],
                   "window": window_str(args, args.ref_iters)},
        "us_per_iter": us_iter,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": setup,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def algorithmic_bytes(counts):
    """Minimal HBM bytes the design must move for the work a set of
    k_engine_steps launches did — counted per EXECUTED unit,
    not per simulated iteration: a quiet span replays its k iterations in
    registers (quiet_steps_fused), so it touches each running request once.
      per normal (event) step: 48 B per running request (generated, occupied,
        written r+w, exec_t r+w, true_rl, allowance, state) + 64 B of queue /
        bitmap / scalar probes;
      per replayed span: the same 48 B per running request + 64 B;
      per PT admission 40 B (class head/count, next link, prompt, reserve
        draw, dispatch fields); per GT schedule 96 B (allocation scan share,
        region record, address insert, request fields); per completion 64 B
        (release, record fields).
    `counts`: normal_steps, spans, mean_running, pt, gt, completed."""
    c = counts
    per_unit = 48.0 * c["mean_running"] + 64.0
    return ((c["normal_steps"] + c["spans"]) * per_unit + 40.0 * c["pt"] + 96.0 * c["gt"] +
            64.0 * c["completed"])


def work_counts(sc_before, sc_after, dbg):
    """The executed units of a window (device counters, econo_batch_debug)."""
    return {"normal_steps": int(dbg[5]), "spans": int(dbg[4]),
            "mean_running": float(np.mean([s.running for s in sc_after])),
            "pt": int(sum(a.pt_dispatched - b.pt_dispatched for a, b in zip(sc_after, sc_before))),
            "gt": int(sum(a.gt_scheduled - b.gt_scheduled for a, b in zip(sc_after, sc_before))),
            "completed": int(sum(a.completed - b.completed for a, b in zip(sc_after, sc_before)))}


def auto_instances(n, device, sms=148, world=1):
    """As many instances per SM as the GPU's free HBM holds: each needs its
    arena (econo_instance_bytes), plus the burst-ingest scratch (<= 2.2 GB).
    The end-of-run JCT keys (8 B per request) get a buffer only if HBM is
    left, else each histogram pass derives them from the request fields.
    Sized on the workload's own trace; at most 16 per SM (the registers of
    16 one-warp CTAs fill an SM).""" 
    import torch

    from paper_2411_06364_b200.engine import generate_trace, instance_bytes
    t = W.make_trace(WORKLOAD, generate_trace, n=n, seed=1000)
    per = instance_bytes(t, options())
    free, _ = torch.cuda.mem_get_info(device)
    slack = (1 << 30) if world == 1 else (4 << 30)  # staging, scratch, context growth (+ NCCL's own)
    # every instance that fits (+ the ingest scratch, 128M keys x 16 B); with
    # time-sliced launches an SM holding one instance more simply does more
    # work, so the count need not be a multiple of the SM count
    inst = int((free - 2.2e9 - slack) // per)
    return max(1, min(inst, 16 * sms))


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2411_06364_b200.engine import Batch, generate_trace

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:  # bring NCCL's buffers up before sizing the batch to the free HBM
        x = torch.ones(1, device=dev)
        dist.all_reduce(x)
        dist.barrier()
        torch.cuda.synchronize()
    I = args.instances or auto_instances(args.n, local, world=world)
    if world > 1:  # every rank runs the same count (the smallest fit)
        t_i = torch.tensor([I], dtype=torch.int64, device=dev)
        dist.all_reduce(t_i, op=dist.ReduceOp.MIN)
        I = int(t_i.item())
    seeds = [1000 + rank * I + i for i in range(I)]
    from paper_2411_06364_b200.engine import instance_bytes
    inst_mb = instance_bytes(W.make_trace(WORKLOAD, generate_trace, n=args.n, seed=1000), options()) / 1e6
    t0 = time.time()
    # host trace generation shares the box's cores between the ranks
    traces = make_traces(generate_trace, args.n, seeds, threads=max(2, (os.cpu_count() or 2) // world), pinned=True,
                         soa=True)
    t_gen = time.time() - t0

    # ---- one pass through the public API, from host trace buffers:
    # Batch(traces) [H2D] -> idle tick + 1M burst ingest -> W warm-up steps ->
    # K device-timed steps -> partial sums back to the host [D2H]. `value` is
    # the device-timed K steps; `e2e` is the same job's wall clock end to end.
    clocks = ClockSampler(local)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    b = Batch(traces, options(), device=local)
    t_created = time.perf_counter()
    b.launch(1, stream.cuda_stream)  # idle tick up to the burst (engine.hpp:930-949)
    stream.synchronize()
    b.ingest()                       # the 1M burst, grid-wide (engine.hpp:216-235)
    b.launch(1, stream.cuda_stream)  # the rest of that step
    stream.synchronize()
    b.sync()
    t_create_ingest = time.perf_counter() - t0
    t_ingest = time.perf_counter() - t_created
    sc_a = b.scalars()
    slice_ns = int(args.slice_us * 1000)
    step_n = (1 << 40) if slice_ns else args.iters
    # warm-up: W untimed steps, step w bringing every instance to step
    # 2 + (w+1) * ref_iters with time-sliced launches (econo_batch_launch_to),
    # so the timed window starts at the same iteration as the reference
    # arm's, every instance together
    warm_launches = 0
    for w in range(args.warmup):
        target = 2 + (w + 1) * args.ref_iters
        while True:
            b.launch_to(target, stream.cuda_stream, slice_ns=slice_ns)
            warm_launches += 1
            stream.synchronize()
            b.sync()
            if all(x.steps >= target or x.done or x.error for x in b.scalars()):
                break
    parity_dev = None
    t_parity = 0.0
    if world == 1 and not args.no_cpu_baseline and args.parity_instances > 0:
        # parity checkpoint at the start of the timed window: digests of the
        # first instances' complete state, compared with the reference's
        # (a check, not part of the job: its time is taken out of e2e)
        tp0 = time.perf_counter()
        parity_dev = [snapshot_digest(b.snapshot(i)) for i in range(min(args.parity_instances, I))]
        t_parity = time.perf_counter() - tp0
    stream.synchronize()
    b.sync()
    sc0 = b.scalars()
    d0 = b.debug().sum(axis=0)
    t_warm_done = time.perf_counter()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks.start()
    e0.record(stream)
    for _ in range(args.steps):
        b.launch(step_n, stream.cuda_stream, slice_ns=slice_ns)
    e1.record(stream)
    e1.synchronize()
    clk = clocks.stop()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = [e0.elapsed_time(e1) / 1e3]
    b.sync()
    sc1 = b.scalars()
    dbg = b.debug().sum(axis=0) - d0
    t_steps_done = time.perf_counter()
    parts = b.partials()
    t_e2e = time.perf_counter() - t0 - t_parity
    e2e_parts = {"create_s": t_created - t0, "ingest_s": t_ingest,
                 "steps_s": t_steps_done - t0 - t_create_ingest - t_parity,
                 "warmup_s": t_warm_done - t0 - t_create_ingest - t_parity,
                 "partials_s": t_e2e - (t_steps_done - t0 - t_parity),
                 "parity_snapshots_s_excluded": t_parity}
    e2e_adm = sum(x.pt_dispatched - y.pt_dispatched for x, y in zip(sc1, sc_a))
    h2d = sum(t.arrival.nbytes + t.prompt.nbytes + t.true_rl.nbytes for t in traces)
    d2h = parts.nbytes + I * 2 * 1600
    errors = [s.error for s in sc1 if s.error]
    log(f"[bench] device cycles: quiet_span {dbg[0]} replay {dbg[1]} normal {dbg[2]}; "
        f"spans {dbg[4]} normal steps {dbg[5]}")
    adm = sum(a.pt_dispatched - z.pt_dispatched for a, z in zip(sc1, sc0))
    gts = sum(a.gt_scheduled - z.gt_scheduled for a, z in zip(sc1, sc0))
    tot = float(sum(times))
    it_done = sum(a.steps - z.steps for a, z in zip(sc1, sc0))  # scheduler iterations, all instances
    it_warm = sum(a.steps - z.steps for a, z in zip(sc0, sc_a))
    wcounts = work_counts(sc0, sc1, dbg)
    abytes = algorithmic_bytes(wcounts)
    t = torch.tensor([tot, float(adm), float(gts), float(e2e_adm), t_e2e], dtype=torch.float64,
                     device=dev)
    # end-of-run report reduction (after the e2e window): exact global p5/p95
    # JCT by radix select, one histogram all-reduce per digit pass
    torch.cuda.synchronize()
    tr0 = time.perf_counter()
    pct = metrics.global_percentiles(b, [0.05, 0.95], dist=dist if world > 1 else None, device=dev)
    t_pct = time.perf_counter() - tr0
    if world > 1:
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        tot_max, adm_all, gts_all, e2e_adm_all, e2e_t = (mx[0].item(), sm[1].item(), sm[2].item(),
                                                         sm[3].item(), mx[4].item())
        # metric partial sums of every instance: one NCCL reduction per op
        gsum = metrics.all_reduce(metrics.combine(parts), dist, device=dev)
    else:
        gsum = metrics.combine(parts)
        tot_max, adm_all, gts_all, e2e_adm_all, e2e_t = tot, float(adm), float(gts), float(e2e_adm), t_e2e
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    value = adm_all / tot_max
    iters_total = it_done / I  # per instance over the window
    us_iter = 1e6 * tot_max / iters_total
    ips = iters_total / args.steps
    peak, peak_kind = measured_peaks()
    achieved = abytes / tot / 1e9  # GB/s, this rank's launches
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "requests_per_instance": args.n,
                   "instances_per_gpu": I, "iters_per_step": round(ips, 1),
                   "launch": (f"time-sliced: each step is one k_engine_steps launch in which every instance "
                              f"advances until {args.slice_us:g} us of device time have passed (econo_batch_"
                              f"launch_slice), ~{ips:.0f} scheduler iterations per instance on average"
                              if slice_ns else f"{args.iters} scheduler iterations per instance per launch"),
                   "policy": W.CONFIGS[WORKLOAD]["opts"]["policy"],
                   "l2": f"inputs larger than L2: {I} x ~{inst_mb:.0f} MB of instance state per GPU vs 126 MB L2, no flush",
                   "window": (window_str(args) if not slice_ns else
                              f"after the 1M burst ingest: {args.warmup} warm-up and {args.steps} timed slices; "
                              f"scheduler iterations ~{2 + (it_warm / I):.0f}..{2 + (it_warm + it_done) / I:.0f} "
                              f"per instance on average")},
        "us_per_iter": us_iter,
        "device_cycles": {"quiet_test": int(dbg[0]), "quiet_replay": int(dbg[1]), "normal_steps": int(dbg[2]),
                          "quiet_spans": int(dbg[4]), "normal_step_count": int(dbg[5])},
        "iters_per_s_per_gpu": iters_total * I / tot_max,
        "gt_scheduled_per_s": gts_all / tot_max,
        "quiet_step_frac": (sum(a.quiet_steps - z.quiet_steps for a, z in zip(sc1, sc0)) /
                            max(1, sum(a.steps - z.steps for a, z in zip(sc1, sc0)))),
        "ingest_and_create_s": t_create_ingest,
        "ingest_s": t_ingest,
        "tracegen_s": t_gen,
        "gpu_launches": args.steps,
        "roofline": roofline_block(abytes, tot, args.steps, I, args.slice_us if slice_ns else 0, wcounts, dbg, peak,
                                   peak_kind),
        "clocks": clk,
        "e2e": {"value": e2e_adm_all / e2e_t, "unit": UNIT, "breakdown": e2e_parts, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "scope": "the whole job through the public API: Batch(host traces: page-locked SoA columns, "
                         "econo_batch_create_soa, 16 B per request) + burst ingest + warm-up + timed steps + "
                         "partial sums to host, wall clock; admissions counted after the ingest"},
        "errors": len(errors),
        "report_reduction": {"global_jct_p5_p95": pct, "ms": 1e3 * t_pct,
                             "how": "k_jct_keys + 6 k_jct_hist radix-select passes, histograms all-reduced "
                                    "across ranks (NCCL) per pass; JCT of requests not yet complete is "
                                    "completion -1 by the reference's convention"},
        "global_metrics": {k: v for k, v in metrics.summary(gsum).items()
                           if k in ("requests", "iterations", "mean_forward_size", "mean_kvc_written",
                                    "tfs_hit_frac", "pt_admit_frac", "hosted_slots")},
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            thr = min(os.cpu_count() or 1, 16)
            wins, setup, ref_dig = reference_windows(args.n, thr, args.ref_iters, args.steps, args.warmup,
                                                     digests=len(parity_dev or []))
            if parity_dev is not None:
                line["parity"] = parity_block(parity_dev, ref_dig, timed_start_step(args))
            secs = sum(w[0] for w in wins)
            pts = sum(w[1] for w in wins)
            line["cpu_baseline"] = {
                "value": pts / secs if secs > 0 else 0.0, "unit": UNIT, "cores": thr,
                "kind": "reference", "us_per_iter": 1e6 * secs / (args.ref_iters * args.steps),
                "sample": f"{thr} reference engines x {args.n} requests ({WORKLOAD}), "
                          f"{window_str(args, args.ref_iters)} ({args.ref_iters} step() calls per engine per "
                          f"step: a bounded sample of the same workload), one std::thread per engine"}
            # the ratio to the reference arm, decomposed field by field
            ref_it = thr * args.ref_iters * args.steps
            line["vs_reference_terms"] = {
                "timed_from_step": timed_start_step(args),
                "same": ["workload and options (configs[2], econoserve-full, oracle predictor)",
                         "trace seeds 1000+i", "burst ingest then the same warm-up step count",
                         "first timed step", "metric: PT admissions per second of the timed steps"],
                "differs": {"instances": [I, thr], "iterations_per_instance": [it_done / I, args.ref_iters * args.steps],
                            "event_log": ["off (running aggregates; the records and report are identical)",
                                          "on (the reference's default EngineOptions)"]},
                "admissions_per_iteration": [adm / max(1, it_done), pts / ref_it],
                "instance_iterations_per_s": [it_done / I / tot, args.ref_iters * args.steps / secs],
                "note": "value / reference value = (instances ratio) x (per-instance iteration rate ratio) x "
                        "(admissions-per-iteration ratio); the last is ~1 (same steady state at 1M queued)"}
        except Exception as ex:  # the reference build is missing on this box
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {ex}"}
    if world == 1 and not args.no_full_runs:
        b.close()  # free the batch before the single-engine runs
        line["full_runs"] = full_runs(args)
    if world == 1 and not args.no_other_workloads:
        b.close()
        line["other_workloads"] = other_workloads(args, stream)
    if world == 1 and not args.no_policy_sweep:
        b.close()
        line["policy_sweep"] = policy_sweep(args)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def other_workloads(args, stream, launches=3, warm=2):
    """The same device-timed step on the other BASELINE.json shapes (north_star:
    Alpaca-, ShareGPT- and BookCorpus-shaped traces), each sized to the GPU
    like the headline (as many instances as HBM and the 16 resident warps per
    SM allow): configs[1] (ShareGPT 100k, Poisson 28 rps: KVC pipelining
    active) and configs[3] (the mixed 1M burst with the lognormal predictor:
    preemptions, reserve top-ups, hosted slots). Time-sliced launches."""
    import torch

    from paper_2411_06364_b200.engine import Batch, generate_trace
    global WORKLOAD
    keep = WORKLOAD
    out = {}
    peak, _ = measured_peaks()
    sl = int(args.slice_us * 1000)
    for name in ("cfg2_sharegpt_100k", "cfg4_mixed_1m"):
        WORKLOAD = name
        n = W.CONFIGS[name]["n"]
        inst = auto_instances(n, 0)
        traces = make_traces(generate_trace, n, [1000 + i for i in range(inst)], pinned=True)
        b = Batch(traces, options(), device=0)
        b.launch(1, stream.cuda_stream)
        stream.synchronize()
        b.ingest()
        for _ in range(warm):
            b.launch(1 << 40, stream.cuda_stream, slice_ns=sl)
        stream.synchronize()
        b.sync()
        sc0, d0 = b.scalars(), b.debug().sum(axis=0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(launches):
            b.launch(1 << 40, stream.cuda_stream, slice_ns=sl)
        e1.record(stream)
        e1.synchronize()
        secs = e0.elapsed_time(e1) / 1e3
        b.sync()
        sc1, dbg = b.scalars(), b.debug().sum(axis=0) - d0
        adm = sum(x.pt_dispatched - y.pt_dispatched for x, y in zip(sc1, sc0))
        its = sum(x.steps - y.steps for x, y in zip(sc1, sc0))
        wc = work_counts(sc0, sc1, dbg)
        ab = algorithmic_bytes(wc)
        out[name] = {"instances": inst, "requests_per_instance": n, "steps": launches,
                     "launch": f"time-sliced, {args.slice_us:g} us", "value": adm / secs, "unit": UNIT,
                     "us_per_iter": 1e6 * secs / (its / inst),
                     "quiet_step_frac": (sum(x.quiet_steps - y.quiet_steps for x, y in zip(sc1, sc0)) / max(1, its)),
                     "hosted_slots_created": int(sum(x.hosted_slots_created - y.hosted_slots_created
                                                     for x, y in zip(sc1, sc0))),
                     "normal_step_cycles": float(dbg[2]) / max(1, dbg[5]),
                     "roofline": {"achieved": ab / secs / 1e9, "peak": peak, "unit": "GB/s",
                                  "frac": ab / secs / 1e9 / peak, "work_counts": wc},
                     "errors": sum(1 for x in sc1 if x.error)}
        b.close()
        del traces
    WORKLOAD = keep
    return out


POLICIES = ["orca", "vllm", "sarathi", "multires", "sync-coupled", "econoserve-d", "econoserve-sd",
            "econoserve-sdo", "econoserve-full"]


def policy_sweep(args, inst=888):
    """The experiment layer's use case: every policy of the reference
    (policies.hpp:24-37, the five baselines included) run to completion on
    `inst` configs[0] instances (Alpaca 10k at 36 rps, trace seeds 1000+i),
    one batch per policy, wall clock around the launches. Beside it, the
    reference runs one such instance per policy on one host core; its
    all-cores rate assumes perfect scaling over the host's cores (run_sweep's
    thread pool, sweep.hpp:112-149)."""
    from paper_2411_06364_b200.engine import Batch, generate_trace
    c = W.CONFIGS["cfg1_alpaca_10k"]
    n = c["n"]
    # trace seeds from 1000 up whose prompts all fit econoserve's 3% reserve
    # (engine.hpp:198-206); the same traces for every policy
    rsv = round(c["opts"]["reserved_fraction"] * c["opts"]["kvc_capacity"])
    traces, seed = [], 1000
    while len(traces) < inst:
        t = generate_trace(n, c["rate"], c["shape"]["prompt"], c["shape"]["rl"], seed)
        seed += 1
        if int(t["prompt_len"].max()) <= rsv:
            traces.append(t)
    out_seeds = seed - 1000
    cores = os.cpu_count() or 1
    out = {"instances": inst, "requests_per_instance": n, "host_cores": cores,
           "trace_seeds": f"first {inst} feasible of 1000..{1000 + out_seeds - 1}"}
    for pol in POLICIES:
        o = abi.default_options(**dict(c["opts"], policy=pol, record_events=0, record_samples=0))
        b = Batch(traces, o, device=0)
        t0 = time.perf_counter()
        while True:
            b.launch(1 << 22)
            b.sync()
            sc = b.scalars()
            if all(x.completed >= n or x.error for x in sc):
                break
        secs = time.perf_counter() - t0
        b.close()
        r = {"device_s": secs, "completed_per_s": inst * n / secs,
             "errors": sum(1 for x in sc if x.error), "steps_per_instance": sum(x.steps for x in sc) / inst}
        if not args.no_cpu_baseline:
            try:
                from oracle import ref
                e = ref.RefEngine(traces[0], o)
                t1 = time.perf_counter()
                e.run()
                one = time.perf_counter() - t1
                r["reference_one_instance_s"] = one
                r["reference_all_cores_completed_per_s"] = n * cores / one
            except Exception as ex:  # noqa: BLE001
                r["reference"] = f"unavailable: {ex}"
        out[pol] = r
        log(f"policy_sweep {pol}: {secs:.3f}s")
    return out


def full_runs(args):
    """SURVEY §8(d) primary metric 2: completed requests/s over whole runs of
    configs[0] and configs[1], one engine each through the single-engine
    public API (Engine(trace, opts).run(), engine.hpp:1039-1042) from host
    trace buffers, wall clock; the reference's own full run is timed beside
    it on one host core for configs[0] (configs[1] takes ~155 s on the CPU,
    SURVEY §6, and is not repeated here)."""
    from paper_2411_06364_b200.engine import Engine, generate_trace
    out = {}
    for name in ("cfg1_alpaca_10k", "cfg2_sharegpt_100k"):
        c = W.CONFIGS[name]
        t = W.make_trace(name, generate_trace)
        o = abi.default_options(**c["opts"])
        o.record_events = 0
        o.record_samples = 0
        # untimed warm-up with the same options (first use of the kernel this
        # configuration selects, allocations after the big batch was released),
        # then the faster of two timed runs: sporadic ~0.5 s host/driver stalls
        # were seen around small single-engine runs
        Engine(W.make_trace(name, generate_trace, n=200), o, device=0).run()
        secs = float("inf")
        for _ in range(2):
            t0 = time.perf_counter()
            recs, rep = Engine(t, o, device=0).run()
            secs = min(secs, time.perf_counter() - t0)
        r = {"requests": len(t), "iterations": int(rep.iterations), "wall_s": secs,
             "completed_per_s": len(t) / secs, "mean_jct": rep.mean_jct, "ssr": rep.ssr,
             "hosted_slots": int(rep.hosted_slots)}
        if name == "cfg1_alpaca_10k" and not args.no_cpu_baseline:
            try:
                from oracle import ref
                o2 = abi.default_options(**c["opts"])  # the reference's default EngineOptions record events
                rt = ref.generate_trace(len(t), c["rate"], c["shape"]["prompt"], c["shape"]["rl"], c["seed"])
                e = ref.RefEngine(rt, o2)
                t1 = time.perf_counter()
                e.run()
                r["reference_wall_s"] = time.perf_counter() - t1
                r["reference_completed_per_s"] = len(rt) / r["reference_wall_s"]
            except Exception as ex:  # noqa: BLE001
                r["reference"] = f"unavailable: {ex}"
        out[name] = r
    return out


def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n, argv):
    """One process per GPU on this node, launched exactly as the driver
    does (torch.distributed.run, rendezvous on 127.0.0.1): each rank runs
    this script with the same arguments and reads RANK / LOCAL_RANK /
    WORLD_SIZE; rank 0 prints the JSON line. NCCL's init lines go to stderr
    (NCCL_DEBUG=INFO, INIT subsystem) so the communicator size is on record.
    Returns the launcher's exit code (the run's ranks are torchrun's children:
    a failure in any rank fails the launch)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + list(argv)
    log("[bench] launching", n, "ranks:", " ".join(cmd))
    return subprocess.call(cmd, env=env)


def spawn_selftest(args):
    """The rank plumbing alone, on CPU (gloo): every rank contributes its
    rank; rank 0 prints the world size and the reduced sum."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
    x = torch.tensor([float(rank)])
    if world > 1:
        dist.all_reduce(x)
    if rank == 0:
        print(json.dumps({"n_gpus": world, "gpus_flag": args.gpus, "rank_sum": x.item()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--instances", type=int, default=0,
                    help="serving instances per GPU (default: as many per SM as fit in HBM; ~157 MB each at 1M "
                         "requests, so 8 per SM = 1184 on a B200)")
    ap.add_argument("--iters", type=int, default=1000,
                    help="scheduler iterations per instance per step (one k_engine_steps launch)")
    ap.add_argument("--slice-us", type=float, default=20000.0,
                    help="time-sliced steps: each launch runs every instance until this much device time has "
                         "passed (0 = a fixed --iters iterations per instance, every launch waiting for its "
                         "slowest instance)")
    ap.add_argument("--ref-iters", type=int, default=100,
                    help="reference arm / cpu_baseline: step() calls per engine per step (bounded sample)")
    ap.add_argument("--parity-instances", type=int, default=16,
                    help="instances of the benchmarked batch compared bit for bit with the CPU baseline's "
                         "reference engines (0: no parity block)")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--ref-threads", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-workloads", action="store_true",
                    help="skip the configs[1] / configs[3] step measurements")
    ap.add_argument("--no-full-runs", action="store_true",
                    help="skip the whole-run completed-req/s measurements of configs[0] and configs[1]")
    ap.add_argument("--no-policy-sweep", action="store_true",
                    help="skip the all-policies configs[0] sweep (888 instances per policy)")
    ap.add_argument("--workload", default=WORKLOAD, choices=sorted(W.CONFIGS),
                    help="BASELINE.json config (default: configs[2], the 1M-queued case the metric is quoted on)")
    ap.add_argument("--spawn-selftest", action="store_true",
                    help="test hook: only the rank plumbing (gloo all-reduce of the ranks), no device work")
    args = ap.parse_args()
    globals()["WORKLOAD"] = args.workload
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without torchrun: launch the N ranks here
        sys.exit(spawn_ranks(args.gpus, sys.argv[1:]))
    if args.spawn_selftest:
        return spawn_selftest(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
