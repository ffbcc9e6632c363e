"""Text summary of one kernel of an ncu --set full report (for profiles/).

    python tools/ncu_profile_txt.py REPORT.ncu-rep KERNEL_REGEX [LIB.so] > profiles/x.txt

Prints the headline raw metrics (tools/ncu_summary.py raw), the L1TEX data
pipe split, the stall-reason shares, the shared-memory wavefronts per
instruction kind (source page) and, with LIB.so (the profiled build), the
per-source-line attribution (tools/ncu_lines.py).
"""
import collections
import csv
import io
import re
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
rep, rx = sys.argv[1], sys.argv[2]
lib = sys.argv[3] if len(sys.argv) > 3 else None

print(subprocess.run([sys.executable, str(HERE / "ncu_summary.py"), "raw", rep, rx],
                     capture_output=True, text=True).stdout.rstrip())
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if not re.search(rx, d.get("Kernel Name", "")):
        continue
    print("# L1TEX data pipe (shared vs global), shared-memory wavefronts vs ideal")
    for k in ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
              "memory_l1_wavefronts_shared", "memory_l1_wavefronts_shared_ideal",
              "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum"):
        if k in d:
            print(f"   {k} = {d[k]}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(v)
          for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and v.isdigit()}
    tot = sum(st.values()) or 1
    print("   stalls: " + " ".join(f"{k}={v / tot * 100:.1f}%" for k, v in
                                   sorted(st.items(), key=lambda kv: -kv[1])[:10]))
    break

src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{rx}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
try:
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    ci = {c: i for i, c in enumerate(h)}
    wcol = next((c for c in h if c.startswith("L1 Wavefronts Shared") and "Ideal" not in c
                 and "Excessive" not in c), None)
    if wcol:
        agg = collections.defaultdict(lambda: [0, 0, 0])
        for r in rows[hi + 1:]:
            if len(r) != len(h):
                continue
            try:
                w = int(float(r[ci[wcol]] or 0))
                n = int(float(r[ci["Instructions Executed"]] or 0))
            except ValueError:  # a repeated header row (several kernels in the report)
                continue
            if not w or not n:
                continue
            op = r[ci["Source"]].split()
            op = next((t for t in op if not t.startswith("@")), "?").split(".")[0]
            key = (op, round(w / n * 2) / 2)
            agg[key][0] += w
            agg[key][1] += 1
        tw = sum(v[0] for v in agg.values()) or 1
        print("# shared-memory wavefronts by instruction kind (wavefronts per warp instruction)")
        for (op, deg), v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:8]:
            print(f"   {op:<10} {deg:4.1f} wf/inst {v[1]:5d} sites {v[0] / tw * 100:5.1f}% of {tw:.3e}")
except StopIteration:
    pass
if lib:
    print("# per-source-line attribution (tools/ncu_lines.py; line numbers of the profiled build)")
    print(subprocess.run([sys.executable, str(HERE / "ncu_lines.py"), rep, lib, rx.split("|")[0], "24"],
                         capture_output=True, text=True).stdout.rstrip())
