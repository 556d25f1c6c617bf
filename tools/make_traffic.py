#!/usr/bin/env python3
"""Turn an ncu launch list of one bench step (csv with gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum per launch) into profiles/traffic.json (mean DRAM
bytes per fp8_block_gemm launch, read by bench.py as roofline.traffic) and a readable
profiles/<name>_launches.txt (per-kernel share of the step).
usage: make_traffic.py launches.csv out_name"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    src, name = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(open(src)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi, ui = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    idi = hdr.index("ID")
    launches = collections.OrderedDict()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr):
            continue
        d = launches.setdefault(r[idi], {"kernel": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    # the last complete bench step: 4 GEMM launches preceded by their quantizers
    lst = list(launches.values())
    gemm = [d for d in lst if "gemm" in d["kernel"]]
    last = gemm[-4:]
    tot = {k: sum(d.get(k, 0.0) for d in last) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum")}
    per_launch = (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / max(1, len(last))
    out = {"fp8_block_gemm_bytes_per_launch": round(per_launch),
           "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (--clock-control none) of bench.py; "
                     f"mean over the last step's {len(last)} fp8_block_gemm launches",
           "per_launch": [{"kernel": d["kernel"][:60], "dram_read": d.get("dram__bytes_read.sum"),
                           "dram_write": d.get("dram__bytes_write.sum"),
                           "us": round(d.get("gpu__time_duration.sum", 0) * 1e6, 2)} for d in last]}
    json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    # share of the step by kernel over the last step (from the 4th-last GEMM's quantizers on)
    first = lst.index(last[0])
    start = max(i for i in range(first) if "weight_blockwise" in lst[i]["kernel"]) if any(
        "weight_blockwise" in d["kernel"] for d in lst[:first]) else max(0, first - 5)
    step = lst[start:]
    t = sum(d.get("gpu__time_duration.sum", 0) for d in step)
    with open(os.path.join(ROOT, "profiles", f"{name}_launches.txt"), "w") as f:
        f.write(f"# ncu launch list of one bench.py step ({src}); cold-cache serialised per-launch times\n")
        f.write(f"# {'kernel':60s} {'us':>9s} {'share':>7s} {'DRAM rd MB':>11s} {'DRAM wr MB':>11s}\n")
        for d in step:
            us = d.get("gpu__time_duration.sum", 0) * 1e6
            f.write(f"  {d['kernel'][:60]:60s} {us:9.2f} {us / (t * 1e6) * 100:6.1f}% "
                    f"{d.get('dram__bytes_read.sum', 0) / 1e6:11.2f} {d.get('dram__bytes_write.sum', 0) / 1e6:11.2f}\n")
        f.write(f"# step total {t * 1e6:.1f} us\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
