"""M=1 evaluation and the fused step for ncu (single-candidate latency)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import argparse  # noqa: E402

import torch  # noqa: E402


def main():
    import bench

    args = argparse.Namespace(samples=4096, horizon=32, grid=256, precision="fp32")
    S = bench.make_scene(args, torch.device("cuda", 0))
    pl, st, goal, field = S["planner"], S["state"], S["goal"], S["field"]
    nom = torch.zeros((32, 7), dtype=torch.float64, device="cuda")
    one = torch.zeros((1, 32, 7), dtype=torch.float64, device="cuda")
    eps = pl.sample_device(3)
    for k in range(3):
        pl.evaluate_device(st, goal, field, one)
        pl.smpc_step_device(st, goal, field, nom, eps)
        pl.smpc_generate_device(st, goal, field, nom, k)  # fused draws (the production step)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
