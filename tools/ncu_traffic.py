"""Per-launch DRAM bytes of the last launch of each kernel in an ncu launch
list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv), written into profiles/ncu_traffic.json under CONFIG (bench.py reads
k_isect_cta_dram_bytes as its roofline `traffic`).

    python tools/ncu_traffic.py LAUNCHES.csv CONFIG OUT.json "source note"
"""
import csv
import json
import re
import sys
from pathlib import Path

path, config, out = sys.argv[1], sys.argv[2], Path(sys.argv[3])
note = sys.argv[4] if len(sys.argv) > 4 else ""
rows = list(csv.reader(open(path)))
hdr = None
last = {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")
    name = re.sub(r"<.*", "", name)
    last.setdefault(name, {})
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(
        d.get("Metric Unit", "byte"), 1)
    last[name].setdefault(int(d["ID"]), {})[d["Metric Name"]] = (
        float(d["Metric Value"].replace(",", "")) * scale)
res = json.loads(out.read_text()) if out.exists() else {}
entry = {}
for name, launches in last.items():
    lid = max(launches)
    m = launches[lid]
    b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    entry[f"{name}_dram_bytes"] = int(b)
res[config] = entry
res["_source"] = note
out.write_text(json.dumps(res, indent=1, sort_keys=True) + "\n")
print(json.dumps(entry, indent=1, sort_keys=True))
