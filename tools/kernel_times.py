"""Warm per-stage device timings (CUDA events, median of N) for the C2/C3
scene: fusion, EDT, rollout (evaluate), fused SMPC step (partial only and
full), M=1 evaluate, sampler.  Prints one JSON object."""

import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def timeit(fn, n=30, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=4096)
    ap.add_argument("--horizon", type=int, default=32)
    ap.add_argument("--grid", type=int, default=256)
    a = ap.parse_args()
    import bench
    from paper_2512_22575_b200 import planner as PL

    args = argparse.Namespace(samples=a.samples, horizon=a.horizon, grid=a.grid, precision="fp32")
    S = bench.make_scene(args, torch.device("cuda", 0))
    pl, st, goal, field, mapper = S["planner"], S["state"], S["goal"], S["field"], S["mapper"]
    mask = (S["centers"], S["radii"])
    nom = torch.zeros((a.horizon, 7), dtype=torch.float64, device="cuda")
    eps = pl.sample_device(3)
    one = torch.zeros((1, a.horizon, 7), dtype=torch.float64, device="cuda")
    out = {}
    out["fusion_us"] = timeit(lambda: mapper.update(S["depth"], mask=mask))
    out["edt_us"] = timeit(lambda: mapper.recompute_edt())
    out["sampler_us"] = timeit(lambda: pl.sample_device(3, out=eps))
    out["rollout_eval_us"] = timeit(lambda: pl.evaluate_device(st, goal, field, eps, nom))
    out["smpc_partial_us"] = timeit(lambda: pl.smpc_partial_device(st, goal, field, nom, eps))
    out["smpc_step_us"] = timeit(lambda: pl.smpc_step_device(st, goal, field, nom, eps))
    out["eval_M1_us"] = timeit(lambda: pl.evaluate_device(st, goal, field, one))
    g = PL.SmpcGraph(pl, field)
    g.stage(st, goal, None, 0)
    out["graph_step_us"] = timeit(g.replay)
    print(json.dumps({k: round(v, 2) for k, v in out.items()}))


if __name__ == "__main__":
    main()
