"""Per-CUDA-source-line instruction and stall totals of one kernel launch in an ncu report.

    python tools/ncu_src_lines.py REPORT KERNEL_REGEX [top_n] [--by-file]

Reads `ncu -i REPORT --page source --print-source sass,cuda --csv` (source lines
with their SASS underneath; the source-line row already holds the aggregate) and
prints the top lines by executed warp instructions and by stall samples, plus a
per-file total.  Needs a report captured with --import-source on and -lineinfo.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--launch-count", "1", "--print-source", "sass,cuda"], capture_output=True,
                         text=True).stdout
    fname, hdr = None, None
    lines = []
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name",):
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0]:
            continue
        ie = hdr.index("Instructions Executed")
        st = hdr.index("Warp Stall Sampling (All Samples)")
        if not r[ie].isdigit():
            continue
        lines.append((fname, int(r[0]), r[1].strip()[:90], int(r[ie]), int(r[st]) if r[st].isdigit() else 0))
    tot_i = sum(x[3] for x in lines)
    tot_s = sum(x[4] for x in lines)
    print(f"total warp-instr {tot_i}  stall samples {tot_s}")
    per_file = defaultdict(lambda: [0, 0])
    for f, _, _, i, s in lines:
        per_file[f][0] += i
        per_file[f][1] += s
    for f, (i, s) in sorted(per_file.items(), key=lambda kv: -kv[1][0]):
        print(f"  {f:<24} instr {i:>10} ({100 * i / max(tot_i, 1):5.1f}%)  stalls {s:>7} ({100 * s / max(tot_s, 1):5.1f}%)")
    print("\n-- top lines by instructions")
    for f, ln, src, i, s in sorted(lines, key=lambda x: -x[3])[:top]:
        print(f"{f}:{ln:<5} {i:>9} {100 * i / tot_i:5.1f}%  st {100 * s / max(tot_s, 1):5.1f}%  {src}")
    print("\n-- top lines by stall samples")
    for f, ln, src, i, s in sorted(lines, key=lambda x: -x[4])[:top]:
        print(f"{f}:{ln:<5} {i:>9} {100 * i / tot_i:5.1f}%  st {100 * s / max(tot_s, 1):5.1f}%  {src}")


if __name__ == "__main__":
    main()
