"""Summarises an ncu report (key raw metrics + hottest source lines) into a
text file for profiles/. Usage: python tools/ncu_summary.py rep.ncu-rep out.txt"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, out):
    lines = []
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    h, u = raw[0], raw[1]
    for row in raw[2:]:
        name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        lines.append(f"== kernel {name}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"  {k:70s} {row[i]:>16s} {u[i]}")
    src = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--print-source=cuda,sass"]))))
    cur_file, cur_line, text = None, None, {}
    samples, insts = defaultdict(int), defaultdict(int)
    hdr = None
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[0] != "":
            cur_line = (cur_file, int(r[0]))
            text[cur_line] = r[1]
            continue
        try:
            samples[cur_line] += int(r[4])
            insts[cur_line] += int(r[7]) if r[7] else 0
        except (ValueError, IndexError):
            pass
    tot = sum(samples.values()) or 1
    lines.append(f"== warp-stall samples by source line (total {tot}, instructions {sum(insts.values())})")
    for k, v in sorted(samples.items(), key=lambda x: -x[1])[:30]:
        lines.append(f"  {100 * v / tot:5.1f}%  inst {insts[k]:8d}  {k[0]}:{k[1]}  {text.get(k, '')[:90]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:25]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
