"""Whole-run timings of configs[0] and configs[1] (bench.full_runs), dev tool.
Warms the CUDA context first so the first run does not pay for it."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_06364_b200 import abi  # noqa: E402
from paper_2411_06364_b200.engine import Engine  # noqa: E402

Engine([(0.0, 10, 10)], abi.default_options()).run()  # context + module load
a = argparse.Namespace(no_cpu_baseline=False)
for _ in range(2):
    print(json.dumps({k: (v["wall_s"], v.get("reference_wall_s")) for k, v in bench.full_runs(a).items()}))
