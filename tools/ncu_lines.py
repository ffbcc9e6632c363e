"""Per-source-line attribution of an ncu source-page capture.

    python tools/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_SUBSTR [TOP]

Maps each SASS address of the captured kernel (ncu --page source --print-source
sass) to its CUDA source line through nvdisasm --print-line-info of the same
library, and prints warp-instructions executed and stall samples per line.
The library must be the exact build that was profiled (built with -lineinfo).
"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def sass_lines(lib: str, kernel: str) -> dict:
    tmp = Path(tempfile.mkdtemp())
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, check=True,
                   capture_output=True)
    for cub in sorted(tmp.glob("*.cubin")):
        out = subprocess.run(["nvdisasm", "-c", "--print-line-info", str(cub)],
                             capture_output=True, text=True).stdout.split("\n")
        starts = [i for i, l in enumerate(out) if l.startswith(".text.") and kernel in l]
        if not starts:
            continue
        lm, cur = {}, None
        for l in out[starts[0] + 1:]:
            if l.startswith(".text."):
                break
            m = re.search(r'## File ".*?/([\w.]+)", line (\d+)', l)
            if m:
                cur = f"{m.group(1)}:{m.group(2)}"
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
            if m:
                lm[int(m.group(1), 16)] = cur
        return lm
    raise SystemExit(f"kernel {kernel} not found in {lib}")


def main():
    rep, lib, kernel = sys.argv[1], str(Path(sys.argv[2]).resolve()), sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                           "-k", f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[0], 16), int(r[ie] or 0), int(r[ws] or 0)) for r in rows[hi + 1:]
            if len(r) == len(h) and r[0].startswith("0x")]
    base = data[0][0]
    lm = sass_lines(lib, kernel)
    ins, st = collections.Counter(), collections.Counter()
    for a, n, s in data:
        k = lm.get(a - base, "?")
        ins[k] += n
        st[k] += s
    ti, ts = sum(ins.values()), max(1, sum(st.values()))
    print(f"{kernel}: {ti:.4g} warp-instructions, {ts} stall samples")
    for k, v in ins.most_common(top):
        print(f"  {k:>20} {v / ti * 100:5.1f}% instr {st[k] / ts * 100:5.1f}% stall")


if __name__ == "__main__":
    main()
