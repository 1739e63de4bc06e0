"""Fused SMPC step time vs M (C3 scene, H=32, L2 flushed before every launch):
separates the fixed per-launch cost (launch + merge tail) from the per-candidate
cost.  Prints one JSON object {M: mean us}."""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--ms", default="4,8,64,256,1024,2048,4096,8192,16384")
    ap.add_argument("--modes", default="generate", help="generate (fused draws), given (eps input), rollout")
    a = ap.parse_args()
    import bench

    args = argparse.Namespace(samples=4096, horizon=32, grid=256, precision="fp32")
    S = bench.make_scene(args, torch.device("cuda", 0))
    pl, st, goal, field = S["planner"], S["state"], S["goal"], S["field"]
    nom = torch.zeros((32, 7), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    res = {}
    for mode in a.modes.split(","):
        for M in [int(x) for x in a.ms.split(",")]:
            eps = pl.sample_device(7, samples=M)
            ts = []
            for it in range(a.iters + 5):
                flush.fill_(it & 255)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if mode == "generate":
                    pl.smpc_generate_device(st, goal, field, nom, 3 + it, samples=M)
                elif mode == "given":
                    pl.smpc_step_device(st, goal, field, nom, eps)
                else:
                    pl.evaluate_device(st, goal, field, eps, nom)
                e1.record()
                e1.synchronize()
                if it >= 5:
                    ts.append(e0.elapsed_time(e1) * 1e3)
            ts.sort()
            res[f"{mode}_{M}"] = {"mean_us": sum(ts) / len(ts), "p50_us": ts[len(ts) // 2]}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
