"""Per-stage time of the C1 closed loop through the public API (64^3 + 256 x H20):
host wall per call (perf_counter, no sync) and device+host per stage (synchronised)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    from paper_2512_22575_b200 import config, mapping, planner, robot, scene

    dev = torch.device("cuda", 0)
    dims, samples, horizon, frames = (64, 64, 64), 256, 20, 40
    chain, model = config.robot_7dof()
    grid, cam, _ = scene.bench_edt_scene(dims, device=dev)
    mapper = mapping.OccupancyMapper(grid, cam, outside_default=0.8)
    params = config.planner_params(7, {"samples": samples, "horizon": horizon})
    pl = planner.Planner(chain, model, params, device=dev)
    state = robot.JointState.resting(np.full(7, 0.05))
    goal = robot.forward_kinematics(chain, np.full(7, 0.35))[-1]
    nominal = np.zeros((horizon, 7))
    seq = scene.moving_obstacle_frames(cam, dims, frames, chain, model)
    depths = [mapping.DepthImage(d) for d, _ in seq]
    masks = [m for _, m in seq]
    rows = {"update": [], "edt": [], "snapshot": [], "step": [], "total": []}
    rows_sync = {k: [] for k in rows}
    for sync in (False, True):
        for f in range(frames):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            mapper.update(depths[f], mask=masks[f])
            if sync: torch.cuda.synchronize()
            t1 = time.perf_counter()
            mapper.recompute_edt()
            if sync: torch.cuda.synchronize()
            t2 = time.perf_counter()
            snap = mapper.snapshot()
            t3 = time.perf_counter()
            res = pl.smpc_step(state, goal, snap, nominal, f)
            t4 = time.perf_counter()
            state = pl.integrate(state, res.command)
            nominal = res.next_nominal
            if f >= 5:
                d = rows_sync if sync else rows
                d["update"].append(t1 - t0); d["edt"].append(t2 - t1); d["snapshot"].append(t3 - t2)
                d["step"].append(t4 - t3); d["total"].append(t4 - t0)
    for name, d in (("async", rows), ("sync", rows_sync)):
        print(name, {k: round(float(np.median(v)) * 1e6, 1) for k, v in d.items()})


if __name__ == "__main__":
    main()
