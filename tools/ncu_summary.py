"""Summarise ncu output for profiles/ (run in the build container).

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN_launches.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep > profiles/rNN_gemm_full.md

`launches`: per-kernel device time of one bench step (ncu --metrics
gpu__time_duration.sum, cold-cache/serialised: compare shares).  `full`: the
key roofline counters of a --set full capture (tensor pipe, DRAM bytes, L2,
registers).
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict


def _rows(text):
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if '"ID"' in l or l.startswith("ID,"))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def launches(path):
    rows = [r for r in _rows(open(path).read()) if r.get("Metric Name") == "gpu__time_duration.sum"]
    agg = OrderedDict()
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        if r.get("Metric Unit") == "ns":
            v /= 1e3
        elif r.get("Metric Unit") == "ms":
            v *= 1e3
        agg.setdefault(name, []).append(v)
    total = sum(sum(v) for v in agg.values())
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for name, vs in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{name}` | {len(vs)} | {sum(vs):.1f} | {100 * sum(vs) / total:.1f}% |")
    print(f"| **total** | {sum(len(v) for v in agg.values())} | {total:.1f} | 100% |")


FULL = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % (realtime)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_dim_x", "cluster x"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    hdr = next(csv.reader([lines[0]]))
    units = next(csv.reader([lines[1]]))
    data = [next(csv.reader([l])) for l in lines[2:] if l.strip()]
    cols = [(hdr.index(m), label) for m, label in FULL if m in hdr]
    print("| id | kernel | " + " | ".join(label for _, label in cols) + " |")
    print("|---|---|" + "---|" * len(cols))
    for r in data:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        vals = []
        for i, _ in cols:
            vals.append(f"{r[i]} {units[i]}".strip())
        print(f"| {r[hdr.index('ID')]} | `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
