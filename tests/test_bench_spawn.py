"""`python bench.py --gpus N` launches its N ranks itself (torch.distributed.run
on 127.0.0.1, one process per GPU — the driver's own launch), so a bare
`--gpus 2` run reports n_gpus 2 instead of silently running one rank. The
rank plumbing is checked here on CPU with gloo (world 2)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus_flag_spawns_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--spawn-selftest"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["gpus_flag"] == 2 and d["rank_sum"] == 1.0
