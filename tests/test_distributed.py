"""The multi-GPU path's only collective — the end-of-run metric reduction
 — on a world_size-2 gloo group on CPU. Each rank owns a
disjoint shard of instances (engine source built for the host); the reduced
result must equal the single-process reduction over all instances."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import port
from paper_2411_06364_b200 import abi, metrics, workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOSTSIM = os.path.join(ROOT, "tests", "_hostsim", "libeconoserve_hostsim.so")
N_INST = 4


def shard_traces(rank, world):
    c = W.CONFIGS["cfg1_alpaca_10k"]
    ids = [i for i in range(N_INST) if i % world == rank]
    return ids, [port.generate_trace(400, 200.0, c["shape"]["prompt"], c["shape"]["rl"], 1000 + i)
                 for i in ids]


def options():
    c = W.CONFIGS["cfg1_alpaca_10k"]
    o = abi.default_options(**dict(c["opts"], pred_model="bucket", pred_accuracy=0.775,
                                   pred_tolerance=0.1))
    o.record_events = 0
    o.record_samples = 0
    return o


def local_batch(rank, world):
    from paper_2411_06364_b200.engine import Batch
    _, trs = shard_traces(rank, world)
    b = Batch(trs, options(), lib=HOSTSIM)
    b.launch(1 << 40)
    b.sync()
    return b


def local_partials(rank, world):
    return local_batch(rank, world).partials()


QS = [0.05, 0.5, 0.95]


def _worker(rank, world, port_, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = local_batch(rank, world)
    p = metrics.combine(b.partials())
    red = metrics.all_reduce(p, dist)
    pct = metrics.global_percentiles(b, QS, dist=dist)  # 6 histogram all-reduces
    if rank == 0:
        out.put((red, pct))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_world2_metric_reduction_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port_ = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_, q)) for r in range(world)]
    for p in procs:
        p.start()
    red, pct = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    b1 = local_batch(0, 1)
    single = metrics.combine(b1.partials())
    assert np.allclose(red, single, rtol=1e-12, atol=0)
    assert pct == metrics.global_percentiles(b1, QS)  # exact order statistics
    s = metrics.summary(red)
    assert s["requests"] == N_INST * 400
    assert s["iterations"] > 0


def test_partials_summary_matches_per_instance_report():
    """For one instance the reduced partial sums reproduce aggregate()
    (metrics.hpp:96-175) within the 1e-6 contract for derived floating point."""
    from paper_2411_06364_b200.engine import Engine
    c = W.CONFIGS["cfg1_alpaca_10k"]
    t = port.generate_trace(500, 150.0, c["shape"]["prompt"], c["shape"]["rl"], 3)
    o = options()
    e = port.OracleEngine(t, o)
    _, rep = e.run()
    from paper_2411_06364_b200.engine import Batch
    b = Batch([t], o, lib=HOSTSIM)
    b.launch(1 << 40)
    b.sync()
    s = metrics.summary(metrics.combine(b.partials()))
    want = rep.as_dict()
    for k in ["mean_jct", "mean_tbt", "ssr", "normalized_latency", "throughput_rps",
              "throughput_tps", "goodput_rps", "mean_kvc_written", "mean_kvc_allocated",
              "mean_forward_size", "tfs_hit_frac", "pt_admit_frac", "mean_waiting",
              "mean_execution", "mean_preemption", "mean_scheduling", "makespan"]:
        assert abs(s[k] - want[k]) <= 1e-6 * max(1.0, abs(want[k])), k
    assert s["iterations"] == want["iterations"]
    assert s["preemptions"] == want["preemptions"]
