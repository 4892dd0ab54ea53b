"""Summarise ncu reports / launch lists into profiles/ (text, committed).

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/x.txt
    python tools/ncu_summary.py report gpurun_out/prof.ncu-rep [more.ncu-rep ...] > profiles/y.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
    "smsp__inst_executed.sum", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    print(f"# launch list: {path}")
    print(f"{'id':>4} {'kernel':70s} {'us':>12}")
    tot = 0.0
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                us = v / 1000 if d["Metric Unit"] == "ns" else (v * 1000 if d["Metric Unit"] == "ms" else v)
                tot += us
                print(f"{d['ID']:>4} {d['Kernel Name'][:70]:70s} {us:12.1f}")
    print(f"total {tot:.1f} us")


def report(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(f"# {p}: no data")
            continue
        hdr, units = rows[0], rows[1]
        print(f"# ncu --set full: {p}")
        for vals in rows[2:]:
            name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
            print(f"## kernel {name[:110]}")
            for k in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    print(f"{k:90s} {vals[i]:>18s} {units[i]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2:])
