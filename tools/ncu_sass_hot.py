"""Per-region SASS instruction counts of one kernel from an ncu report.
usage: python tools/ncu_sass_hot.py REPORT KERNEL_REGEX [launch_skip] [window]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
win = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-skip", str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
ie = h.index("Instructions Executed")
st = h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) == len(h) and r[ie].isdigit()]
# first kernel body only (the export can repeat)
seen, body = set(), []
for r in data:
    if r[0] in seen:
        break
    seen.add(r[0])
    body.append(r)
tot = sum(int(r[ie]) for r in body)
stalls = sum(int(r[st]) for r in body)
print(f"{rows[0][1][:90]}\n total warp-instr {tot}  sass {len(body)}  stall samples {stalls}")
w = defaultdict(lambda: [0, 0])
for i, r in enumerate(body):
    w[i // win][0] += int(r[ie])
    w[i // win][1] += int(r[st])
for k in sorted(w):
    if w[k][0] > tot * 0.01 or w[k][1] > stalls * 0.02:
        first = body[k * win][1].strip()[:50]
        print(f"{k * win:5d}-{k * win + win - 1:5d} {w[k][0]:10d} {100 * w[k][0] / tot:5.1f}%  stall {100 * w[k][1] / max(1, stalls):5.1f}%  {first}")
if "-v" in sys.argv:
    for i, r in enumerate(body):
        if int(r[ie]) > 0:
            print(f"{i:5d} {int(r[ie]):9d} {int(r[st]):6d} {r[1].strip()[:80]}")
