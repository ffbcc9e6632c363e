"""Summarise ncu outputs: launch list CSV (gpu__time_duration) and full reports.

    python tools/ncu_summary.py launches <csv>
    python tools/ncu_summary.py raw <ncu-rep> [kernel-regex]
    python tools/ncu_summary.py source <ncu-rep> <kernel-regex> [top]
"""
import csv
import io
import re
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
       "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
       "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
       "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                unit = d.get("Metric Unit", "")
                v = float(d["Metric Value"].replace(",", ""))
                scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
                         "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
                us = v * scale.get(unit, 1e-3)
                out.append((int(d["ID"]), d["Kernel Name"], us))
    tot = sum(x[2] for x in out)
    agg = {}
    for _, k, us in out:
        k = re.sub(r"\(.*", "", k)[:70]
        agg[k] = agg.get(k, 0) + us
    print(f"{len(out)} launches, total {tot/1e3:.3f} ms")
    for k, us in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"{us/1e3:10.3f} ms {us/tot*100:5.1f}%  {k}")


def raw(path, rx=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if rx and not re.search(rx, d.get("Kernel Name", "")):
            continue
        print(re.sub(r"\(.*", "", d.get("Kernel Name", "?")))
        for k in RAW:
            if k in d:
                print(f"   {k} = {d[k]} {units[hdr.index(k)]}")


def source(path, rx, top=40):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{rx}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[i0]
    data = [r for r in rows[i0 + 1:] if len(r) == len(hdr)]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iI = hdr.index("Instructions Executed")
    iT = hdr.index("Avg. Threads Executed")
    tot = sum(float(r[iS] or 0) for r in data) or 1
    toti = sum(float(r[iI] or 0) for r in data) or 1
    print(f"samples {tot:.0f} inst {toti:.3e}")
    sel = sorted(data, key=lambda r: -float(r[iS] or 0))[:top]
    for r in sorted(sel, key=lambda r: int(r[0], 16)):
        print(f"{r[0][-5:]} {float(r[iS] or 0)/tot*100:5.1f}% inst={float(r[iI] or 0)/toti*100:5.1f}%"
              f" thr={r[iT]:>5} {r[1][:80]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "raw":
        raw(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        source(sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
