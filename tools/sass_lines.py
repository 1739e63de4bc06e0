"""Map SASS instructions of one kernel (nvdisasm -gi output) to source lines.

    nvdisasm -gi -c X.cubin > X.gi
    python tools/sass_lines.py X.gi KERNEL_SUBSTR PATTERN [PATTERN...]

For each instruction whose text matches any PATTERN (regex), prints the innermost
source file:line it comes from (plus the inlined-at chain head), aggregated."""
import re
import sys
from collections import Counter

path, kern, pats = sys.argv[1], sys.argv[2], [re.compile(p) for p in sys.argv[3:]]
inside = False
loc = None
cnt = Counter()
for line in open(path):
    if line.startswith("\t.text.") or line.startswith(".text."):
        inside = kern in line
        continue
    if not inside:
        continue
    m = re.search(r'## File "([^"]+)", line (\d+)(.*)', line)
    if m:
        loc = f'{m.group(1).split("/")[-1]}:{m.group(2)}'
        continue
    if "/*" in line and any(p.search(line) for p in pats):
        cnt[loc] += 1
for k, v in cnt.most_common(60):
    print(f"{v:5d}  {k}")
