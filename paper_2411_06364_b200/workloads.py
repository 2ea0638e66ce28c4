"""Synthetic workload shapes of BASELINE.json `configs`.

Length distributions are the paper's Table 1 in the
reference's LengthDist form (workload.hpp:27-32); KVC token capacities come
from bytes/token = 2*2*layers*hidden.
"""
ALPACA = dict(prompt=(19.31, 9, 2470, 0.8), rl=(58.41, 13, 292, 0.8))
SHAREGPT = dict(prompt=(161.31, 16, 3200, 0.8), rl=(337.99, 19, 991, 0.8))
BOOKCORPUS = dict(prompt=(1952.11, 18, 2048, 0.1), rl=(681.2, 32, 1041, 0.8))

OPT13B_TOKENS = 14648     # 12 GB / 819,200 B per token
OPT175B_TOKENS = 55949    # 264 GB / 4,718,592 B per token
LLAMA2_13B_TOKENS = 14648

BURST_RATE = 1e9          # "1M queued": every arrival lands inside the first idle tick

MIXED_PARTS = (ALPACA, SHAREGPT, BOOKCORPUS)


def mixed_trace(gen, n, rate, seed, out=None):
    """configs[3]'s trace (SURVEY.md §8(d) cfg 4): three traces of the cfg 1-3
    shapes (seeds seed, seed+1, seed+2; n/3 each, the remainder to the last)
    merged by arrival time, stably, into one trace (load_trace_csv requires
    nondecreasing arrivals, workload.hpp:181-183). gen(n, rate, prompt, rl,
    seed) is generate_synthetic (workload.hpp:104-125)."""
    import numpy as np
    sizes = [n // 3, n // 3, n - 2 * (n // 3)]
    parts = [gen(m, rate, sh["prompt"], sh["rl"], seed + i) for i, (m, sh) in enumerate(zip(sizes, MIXED_PARTS)) if m]
    cat = np.concatenate(parts)
    order = np.argsort(cat["arrival_time"], kind="stable")
    if out is None:
        return cat[order]
    out[:] = cat[order]
    return out


def make_trace(name, gen, n=None, seed=None, out=None):
    """The synthetic trace of CONFIGS[name] (n and seed overridable)."""
    c = CONFIGS[name]
    n = c["n"] if n is None else n
    seed = c["seed"] if seed is None else seed
    if c["shape"] == "mixed":
        return mixed_trace(gen, n, c["rate"], seed, out=out)
    kw = {} if out is None else {"out": out}
    return gen(n, c["rate"], c["shape"]["prompt"], c["shape"]["rl"], seed, **kw)


# name -> (trace shape, n, arrival rate, trace seed, option overrides)
CONFIGS = {
    # configs[0]: the reference's own CPU-runnable case
    "cfg1_alpaca_10k": dict(shape=ALPACA, n=10_000, rate=36.0, seed=1, opts=dict(
        policy="econoserve-full", kvc_capacity=OPT13B_TOKENS, kvc_block_size=16,
        reserved_fraction=0.03, tfs=2048, pred_model="oracle", pred_padding_ratio=0.10,
        buffer_ratio=0.15)),
    # configs[1]: ShareGPT 100k, pipelining + reserved KVC
    "cfg2_sharegpt_100k": dict(shape=SHAREGPT, n=100_000, rate=28.0, seed=1, opts=dict(
        policy="econoserve-full", kvc_capacity=OPT175B_TOKENS, kvc_block_size=16,
        reserved_fraction=0.06, tfs=2048, pred_model="oracle", pred_padding_ratio=0.15,
        buffer_ratio=0.15)),
    # configs[2]: BookCorpus 1M burst ("1M queued"), SLO-priority selection
    "cfg3_bookcorpus_1m": dict(shape=BOOKCORPUS, n=1_000_000, rate=BURST_RATE, seed=1, opts=dict(
        policy="econoserve-full", kvc_capacity=LLAMA2_13B_TOKENS, kvc_block_size=16,
        reserved_fraction=0.14, tfs=4096, pred_model="oracle", pred_padding_ratio=0.20,
        buffer_ratio=0.10)),
    # configs[3]: mixed trace, predictor error sweep (preemption path)
    "cfg4_mixed_1m": dict(shape="mixed", n=1_000_000, rate=BURST_RATE, seed=1, opts=dict(
        policy="econoserve-full", kvc_capacity=OPT175B_TOKENS, kvc_block_size=16,
        reserved_fraction=0.06, tfs=4096, pred_model="lognormal", pred_sigma=0.3,
        pred_padding_ratio=0.10, buffer_ratio=0.15)),
}
