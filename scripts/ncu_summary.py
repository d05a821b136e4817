#!/usr/bin/env python3
"""Summarise ncu outputs for profiles/ (committed evidence).

  launches <launches.csv>            per-kernel count / mean / total of gpu__time_duration
  full <report.ncu-rep>              key metrics of a `--set full` capture
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Avg. Active Threads Per Warp", "Warp Cycles Per Issued Instruction",
        "Achieved Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate", "Branch Efficiency", "Eligible Warps Per Scheduler",
        "No Eligible"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "launch__registers_per_thread"]


def launches(path):
    txt = open(path).read().splitlines()
    i = [k for k, l in enumerate(txt) if l.startswith('"ID"')][0]
    agg = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO("\n".join(txt[i:]))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        agg.setdefault(r["Kernel Name"].split("(")[0][:70], []).append(float(r["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':70s} {'n':>5s} {'mean_us':>11s} {'total_ms':>10s} {'share':>6s}")
    for k, v in agg.items():
        print(f"{k:70s} {len(v):5d} {sum(v) / len(v) / 1e3:11.3f} {sum(v) / 1e6:10.3f} {sum(v) / tot:6.3f}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    cur = None
    for row in rows[1:]:
        d = dict(zip(h, row))
        k = d.get("Kernel Name", "")[:80]
        if k != cur:
            print(f"== {k}  (ID {d.get('ID')})")
            cur = k
        if d.get("Metric Name") in KEYS:
            print(f"   {d['Metric Name']:45s} {d['Metric Value']:>16s} {d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hdr, units = rr[0], dict(zip(rr[0], rr[1]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for row in rr[2:]:
            d = dict(zip(hdr, row))
            print("   raw:", {k: (d.get(k), units.get(k)) for k in RAW if k in d})
            try:
                rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale[units["dram__bytes_read.sum"]]
                wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale[units["dram__bytes_write.sum"]]
                print("   traffic_json:", json.dumps({"kernel": d.get("Kernel Name", "")[:60], "dram_read_bytes": rd,
                                                    "dram_write_bytes": wr, "traffic_bytes": rd + wr}))
            except (KeyError, ValueError):
                pass


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
