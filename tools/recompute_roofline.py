"""Recomputes the bench line's roofline from committed files alone (dev /
review tool): the work counts and timing of a bench JSON line (profiles/) and
the ncu launch list summary (profiles/r02_traffic.json).
Usage: python tools/recompute_roofline.py profiles/r02_bench.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main(path):
    line = json.load(open(path))
    r = line["roofline"]
    secs = line["ms_per_step"] * line["steps"] / 1e3
    ab = bench.algorithmic_bytes(r["work_counts"])
    frac = ab / secs / 1e9 / r["peak"]
    print(f"algorithmic bytes {ab:.4g} over {secs * 1e3:.3f} ms -> {ab / secs / 1e9:.1f} GB/s = {100 * frac:.2f}% of "
          f"{r['peak']} GB/s (line says {100 * r['frac']:.2f}%)")
    tr = json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json")))
    dram = tr["dram_bytes_per_launch"] / (tr["ncu_ns_per_launch"] * 1e-9) / 1e9
    print(f"ncu DRAM: {tr['dram_bytes_per_launch']:.4g} B per launch in {tr['ncu_ns_per_launch'] / 1e3:.1f} us -> "
          f"{dram:.1f} GB/s = {100 * dram / r['peak']:.2f}% (ncu per-launch time {tr['ncu_ns_per_launch'] / 1e6:.3f} ms vs "
          f"bench {line['ms_per_step']:.3f} ms)")


if __name__ == "__main__":
    main(*sys.argv[1:])
