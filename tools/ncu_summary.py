"""Per-launch summary of an ncu --set full report (details page) -> text.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep "header line" > profiles/rX_ncu_summary.txt
"""
import csv
import io
import subprocess
import sys

KEEP = ["DRAM Throughput", "Duration", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy"]


def main():
    rep, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.DictReader(io.StringIO(raw)))
    if header:
        print(header)
    seen = {}
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        seen.setdefault(key, {})
        name = r["Metric Name"]
        if name in KEEP and name not in seen[key]:
            seen[key][name] = f'{r["Metric Value"]} {r["Metric Unit"]}'.strip()
    for (lid, kname), metrics in seen.items():
        print(f"== [{lid}] {kname[:100]}")
        for k in KEEP:
            if k in metrics:
                print(f"   {k:<40} {metrics[k]}")


if __name__ == "__main__":
    main()
