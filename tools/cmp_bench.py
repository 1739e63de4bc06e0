"""Side-by-side of every numeric timing key of several bench.py JSON lines:
python tools/cmp_bench.py a.json b.json ..."""
import json
import sys


def flat(x, p="", out=None):
    out = {} if out is None else out
    if isinstance(x, dict):
        for k, v in x.items():
            flat(v, f"{p}.{k}" if p else k, out)
    elif isinstance(x, list):
        for i, v in enumerate(x):
            flat(v, f"{p}[{i}]", out)
    elif isinstance(x, (int, float)) and not isinstance(x, bool):
        out[p] = x
    return out


def timing(k):
    leaf = k.rsplit(".", 1)[-1]
    return leaf in ("ms", "ms_per_step", "p90") or leaf.endswith("_ms") or k.startswith("configs.c") and leaf == "value"


rows = [flat(json.loads(open(p).read().strip().splitlines()[-1])) for p in sys.argv[1:]]
names = [k for k in rows[0] if timing(k)]
print(f"{'key (ms)':44s}" + "".join(f"{p.split('/')[-1][:14]:>15s}" for p in sys.argv[1:]))
for k in names:
    print(f"{k[:44]:44s}" + "".join(f"{r.get(k, float('nan')):15.4f}" for r in rows))
