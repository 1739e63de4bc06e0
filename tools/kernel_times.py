"""Warm per-kernel device durations (CUPTI via torch.profiler) for the C2/C3
scene: fusion, EDT, sampler, rollout, fused SMPC step, graph replay.
Host launch overhead is excluded (kernel durations only).  Prints JSON."""

import argparse
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402


def kernel_times(fn, n=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
    acc = defaultdict(float)
    cnt = defaultdict(int)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0:
            acc[e.name[:60]] += e.device_time_total
            cnt[e.name[:60]] += 1
    return {k: round(v / n, 2) for k, v in acc.items()}


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
    out = {
        "fusion": kernel_times(lambda: mapper.update(S["depth"], mask=mask)),
        "edt": kernel_times(lambda: mapper.recompute_edt()),
        "rollout_eval": kernel_times(lambda: pl.evaluate_device(st, goal, field, eps, nom)),
        "smpc_step": kernel_times(lambda: pl.smpc_step_device(st, goal, field, nom, eps)),
        "eval_M1": kernel_times(lambda: pl.evaluate_device(st, goal, field, one)),
    }
    g = PL.SmpcGraph(pl, field)
    g.stage(st, goal, None, 0)
    out["graph_replay"] = kernel_times(g.replay)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
