"""Markdown table of ncu's NVLink byte counters for the exchange kernels next
to the bytes the plan says must cross NVLink (tools/nvlink_probe.py output).

  python tools/nvlink_summary.py gpurun_out/<run>_nvl_ncu.csv gpurun_out/<run>_nvprobe.log
"""
import csv
import json
import sys
from collections import OrderedDict


def main():
    csv_path, probe_path = sys.argv[1], sys.argv[2]
    probe = json.loads([ln for ln in open(probe_path) if ln.startswith("{")][-1])
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    idx = {h: i for i, h in enumerate(rows[0])}
    launches = OrderedDict()
    for r in rows[1:]:
        key = (int(r[idx["ID"]]), int(r[idx["Device"]]), r[idx["Kernel Name"]])
        launches.setdefault(key, {})[r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
    n = probe["gpus"]
    # every launch of both steps (warm-up and measured), per GPU in launch order
    step = sorted(launches, key=lambda k: (k[1], k[0]))
    assert all(0 <= k[1] < n for k in step)
    print(f"| launch | GPU | kernel | time (us) | NVLink tx user bytes | plan bytes | ratio | tx GB/s | tx incl. protocol |")
    print("|---|---|---|---|---|---|---|---|---|")
    for (i, dev, name) in step:
        m = launches[(i, dev, name)]
        tx = m.get("nvltx__bytes_data_user.sum", 0.0)
        if tx == 0:
            continue
        pr = probe["per_rank"][str(dev)]
        if "ep_dispatch" in name:
            kind = "push fwd (x + origin table)" if "<2, 0>" in name or ", 0>" in name else "push bwd (g*u)"
            plan = pr["push_bytes_remote"]
        else:
            kind = "GEMM scatter epilogue (y fwd / dx bwd)"
            plan = pr["scatter_bytes_remote"]
        us = m["gpu__time_duration.sum"] / 1e3
        print(f"| {i} | {dev} | {kind} | {us:.1f} | {tx:,.0f} | {plan:,} | {tx / plan:.4f} | "
              f"{tx / us / 1e3:.0f} | {m.get('nvltx__bytes.sum', 0):,.0f} |")


if __name__ == "__main__":
    main()
