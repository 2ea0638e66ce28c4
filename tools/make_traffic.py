"""profiles/r02_traffic.json from an ncu launch list of the bench (dev tool):
averages DRAM bytes and duration over the last `--launches` k_engine_steps
launches (the timed ones). Usage:
  python tools/make_traffic.py gpurun_out/r2_launches.csv --instances 1184 --slice-us 20000"""
import argparse
import csv
import json
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--instances", type=int, required=True)
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--launches", type=int, default=10)
    ap.add_argument("--slice-us", type=float, default=0)
    ap.add_argument("--out", default="profiles/r02_traffic.json")
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    K, M, V, I = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = defaultdict(dict)
    names = {}
    for r in rows[h + 1:]:
        if len(r) < len(hdr):
            continue
        per[int(r[I])][r[M]] = float(r[V].replace(",", ""))
        names[int(r[I])] = r[K].split("(")[0]
    ids = [i for i in sorted(per) if names[i].startswith("k_engine_steps")][-a.launches:]  # generic or specialised
    dram = [per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0) for i in ids]
    ns = [per[i]["gpu__time_duration.sum"] for i in ids]
    out = {"kernel": "k_engine_steps",
           "config": {"workload": "cfg3_bookcorpus_1m", "instances_per_gpu": a.instances, "slice_us": a.slice_us},
           "dram_bytes_per_launch": sum(dram) / len(dram), "ncu_ns_per_launch": sum(ns) / len(ns),
           "launches": len(ids), "source": a.source or a.csv}
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
