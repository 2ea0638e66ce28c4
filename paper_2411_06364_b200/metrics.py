"""Cross-instance metric reduction.

Each instance's metric partial sums are computed on the device
(k_engine_partials, runtime.cu; layout in include/econoserve_b200.h
ECONO_PARTIAL_WORDS) and reduced across instances and GPUs with ONE
collective per reduction op at end of run (NCCL over NVLink in bench.py,
gloo in the CPU tests). Field meanings follow aggregate()
(metrics.hpp:96-175); cross-instance sums may be reordered, so derived means
are the 1e-6-relative tier of the contract.
"""
import numpy as np

FIELDS = ["n", "sum_jct", "sum_tbt", "tbt_n", "sum_norm_latency", "met_slo", "tokens",
          "preemptions", "reserve_draws", "alloc_failures", "makespan", "sum_waiting",
          "sum_execution", "sum_preemption", "sum_scheduling", "executed_iters", "sum_forward_size",
          "sum_kvc_written", "sum_kvc_allocated", "tfs_hits", "pt_iters", "hosted_slots",
          "hosted_overruns", "completed", "pt_dispatched", "gt_scheduled", "steps", "iter"]
MAX_FIELDS = [FIELDS.index("makespan")]


def combine(partials):
    """Reduces an (instances, 32) array on the host: sums, max for makespan."""
    p = np.asarray(partials, dtype=np.float64).reshape(-1, partials.shape[-1])
    out = p.sum(axis=0)
    for k in MAX_FIELDS:
        out[k] = p[:, k].max() if len(p) else 0.0
    return out


def all_reduce(vec, dist, device=None):
    """One SUM and one MAX collective over the process group (torch.distributed)."""
    import torch
    t = torch.as_tensor(np.asarray(vec, dtype=np.float64), device=device)
    mx = t[MAX_FIELDS].clone()
    s = t.clone()
    s[MAX_FIELDS] = 0.0
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    s[MAX_FIELDS] = mx
    return s.cpu().numpy()


DIGIT_BITS = [11, 11, 11, 11, 11, 9]  # MSB-first digits of the 64-bit JCT key


def global_percentiles(batch, qs, n_local=None, dist=None, device=None):
    """Exact JCT percentiles over every request of every instance on every
    rank, with percentile()'s interpolation (metrics.hpp:81-89) applied to
    the global order statistics. Each of the 6 radix-select passes builds
    this device's digit histograms (econo_batch_jct_hist) and, across ranks,
    SUMs them with one all-reduce (NCCL over NVLink on GPUs, gloo in the CPU
    tests) — 2 x len(qs) x 2048 counters, not the 8 B/request JCT arrays."""
    import torch

    def allsum(a):
        if dist is None:
            return a
        t = torch.as_tensor(a.astype(np.int64), device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.cpu().numpy().astype(np.uint64)

    if n_local is None:
        n_local = int(sum(len(t) for t in batch.traces))
    n_total = int(allsum(np.array([n_local], dtype=np.uint64))[0])
    targets, fracs = [], []
    for q in qs:
        rank = q * float(n_total - 1)
        lo = int(rank)
        hi = min(lo + 1, n_total - 1)
        targets += [lo, hi]
        fracs.append(rank - float(lo))
    batch.jct_prepare()
    keys = []
    for c0 in range(0, len(targets), 8):  # <= 8 order statistics per histogram pass
        rk = np.array(targets[c0:c0 + 8], dtype=np.uint64)
        pre = np.zeros(len(rk), dtype=np.uint64)
        consumed = 0
        for db in DIGIT_BITS:
            h = allsum(batch.jct_hist(pre, consumed, db))
            for t in range(len(rk)):
                c = np.cumsum(h[t], dtype=np.uint64)
                d = int(np.searchsorted(c, rk[t], side="right"))
                below = int(c[d - 1]) if d > 0 else 0
                rk[t] -= np.uint64(below)
                pre[t] = (int(pre[t]) << db) | d
            consumed += db
        keys += list(pre)
    vals = [batch.key_to_double(k) for k in keys]
    return [vals[2 * i] * (1.0 - f) + vals[2 * i + 1] * f for i, f in enumerate(fracs)]


def summary(p):
    """Global report fields from reduced partial sums (aggregate, metrics.hpp:129-173)."""
    g = dict(zip(FIELDS, p))
    n = g["n"]
    ex = g["executed_iters"]
    mk = g["makespan"]
    return {
        "requests": n,
        "mean_jct": g["sum_jct"] / n if n else 0.0,
        "mean_tbt": g["sum_tbt"] / g["tbt_n"] if g["tbt_n"] else 0.0,
        "ssr": g["met_slo"] / n if n else 0.0,
        "normalized_latency": g["sum_norm_latency"] / n if n else 0.0,
        "throughput_rps": n / mk if mk > 0 else 0.0,
        "throughput_tps": g["tokens"] / mk if mk > 0 else 0.0,
        "goodput_rps": g["met_slo"] / mk if mk > 0 else 0.0,
        "allocation_failure_pct": 100.0 * g["alloc_failures"] / n if n else 0.0,
        "mean_waiting": g["sum_waiting"] / n if n else 0.0,
        "mean_execution": g["sum_execution"] / n if n else 0.0,
        "mean_preemption": g["sum_preemption"] / n if n else 0.0,
        "mean_scheduling": g["sum_scheduling"] / n if n else 0.0,
        "iterations": ex,
        "mean_forward_size": g["sum_forward_size"] / ex if ex else 0.0,
        "mean_kvc_written": g["sum_kvc_written"] / ex if ex else 0.0,
        "mean_kvc_allocated": g["sum_kvc_allocated"] / ex if ex else 0.0,
        "tfs_hit_frac": g["tfs_hits"] / ex if ex else 0.0,
        "pt_admit_frac": g["pt_iters"] / ex if ex else 0.0,
        "preemptions": g["preemptions"],
        "reserve_draws": g["reserve_draws"],
        "hosted_slots": g["hosted_slots"],
        "hosted_overruns": g["hosted_overruns"],
        "makespan": mk,
    }
