#!/usr/bin/env python3
"""Summarise an ncu report (`ncu -i X.ncu-rep --page raw --csv`) into the metrics the
roofline discussion uses: duration, DRAM bytes, DRAM / L2 / tensor / FMA pipe utilisation,
issue activity, registers, top warp-stall reasons.  Usage: ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("Kernel Name", "kernel"),
    ("Grid Size", "grid"),
    ("Block Size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("dram__bytes.sum.per_second", "dram bandwidth"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu pipe inst %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__mem_tensor_reads_op_ldt.sum.pct_of_peak_sustained_elapsed", "TMEM ld (LDTM) %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem (LSU) wavefronts %"),
    ("sm__memory_throughput.avg.pct_of_peak_sustained_elapsed", "SM memory throughput %"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in data:
        print("-" * 100)
        for key, label in KEYS:
            if key in idx:
                v = r[idx[key]]
                u = units[idx[key]]
                if key == "Kernel Name":
                    v = v.split("(")[0][-90:]
                print(f"  {label:28s} {v} {u}")
        stalls = []
        for h, i in idx.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        top = sorted(stalls, reverse=True)[:6]
        print("  top stall samples          " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in top))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        main(p)
