"""Stall-reason totals of source-line ranges of one kernel (ncu source view).

    python tools/ncu_stall_ranges.py REPORT KERNEL_REGEX FILE:L0-L1[=name] ...
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern, specs = sys.argv[1], sys.argv[2], sys.argv[3:]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}", "--launch-count",
                      "1", "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
ranges = []
for sp in specs:
    body, _, name = sp.partition("=")
    f, _, lr = body.partition(":")
    a, _, b = lr.partition("-")
    ranges.append((name or body, f, int(a), int(b)))
fname, hdr = None, None
tot = {r[0]: defaultdict(int) for r in ranges}
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    ln = int(r[0])
    for name, f, a, b in ranges:
        if f == fname and a <= ln <= b:
            for i, h in enumerate(hdr):
                if h.startswith("stall_") and "Not Issued" not in h and r[i].isdigit():
                    tot[name][h] += int(r[i])
            ie = hdr.index("Instructions Executed")
            if r[ie].isdigit():
                tot[name]["instr"] += int(r[ie])
for name, d in tot.items():
    s = sum(v for k, v in d.items() if k.startswith("stall_"))
    top = sorted(((k, v) for k, v in d.items() if k.startswith("stall_")), key=lambda kv: -kv[1])[:6]
    print(f"{name}: instr {d['instr']}  samples {s}  " + "  ".join(f"{k[6:]} {100 * v / max(s, 1):.0f}%" for k, v in top))
