"""DRAM traffic per launch from an ncu --set full report -> profiles JSON.

    python tools/ncu_traffic.py gpurun_out/a.ncu-rep [b.ncu-rep ...] profiles/ncu_traffic.json

Groups launches by kernel family (smpc_kernel, edt = line table + Z+Y + X
passes, fuse_kernel, ...) and records dram__bytes_read.sum +
dram__bytes_write.sum per launch (mean over the captured launches).
bench.py reads the result into its roofline `traffic` field."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

FAMILIES = {"smpc_kernel": "smpc_kernel", "edt_line_lr_kernel": "edt", "edt_zy_kernel": "edt",
            "edt_x_kernel": "edt", "fuse_kernel": "fuse_kernel", "masked_pixels_kernel": "fuse_kernel",
            "rollout_kernel": "rollout_kernel", "sampler_kernel": "sampler_kernel"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    *reps, out = sys.argv[1:]
    res = {}
    for rep in reps:  # later reports override earlier ones per kernel family
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, units = rows[0], rows[1]
        ir, iw, ik = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("Kernel Name")
        per_kernel = defaultdict(list)
        for r in rows[2:]:
            name = r[ik].split("(")[0].split("<")[0].replace("void ", "").replace("vpb::", "").strip()
            b = float(r[ir]) * SCALE[units[ir]] + float(r[iw]) * SCALE[units[iw]]
            per_kernel[name].append(b)
        fam = defaultdict(float)
        for k, v in per_kernel.items():
            if k in FAMILIES:
                # smpc_kernel: the LAST captured launch (the fused-draw production variant)
                fam[FAMILIES[k]] += v[-1] if k == "smpc_kernel" else sum(v) / len(v)
        for k, v in fam.items():
            res[k] = {"bytes": v, "source": f"ncu --set full --clock-control none, {rep.split('/')[-1]}"}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
