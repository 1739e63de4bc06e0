"""One replan (masked fusion + EDT 256^3 + SMPC M=4096 x H=32) for ncu.

    ncu --set full -k regex:<kernel> python tools/profile_step.py
Runs `--warmup` untimed replans first (use ncu -s to skip their launches).
"""

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--samples", type=int, default=4096)
    ap.add_argument("--horizon", type=int, default=32)
    ap.add_argument("--grid", type=int, default=256)
    a = ap.parse_args()
    import bench

    args = argparse.Namespace(samples=a.samples, horizon=a.horizon, grid=a.grid, precision="fp32")
    S = bench.make_scene(args, torch.device("cuda", 0))
    from paper_2512_22575_b200 import distributed

    sh = distributed.ShardedSMPC(S["planner"])
    nominal = torch.zeros((a.horizon, 7), dtype=torch.float64, device="cuda")
    mask = (S["centers"], S["radii"])
    for k in range(a.warmup + a.iters):
        S["mapper"].update(S["depth"], mask=mask)
        f = S["mapper"].recompute_edt()
        sh.step_device(S["state"], S["goal"], f, nominal, k)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
