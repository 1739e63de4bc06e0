"""Per-phase device times of the C5 closed loop (bench.closed_loop): masked
fusion, EDT and the SMPC step, medians over the frames."""
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from paper_2512_22575_b200 import config, mapping, planner, robot, scene

    dims, samples, horizon, frames = (512, 512, 512), int(sys.argv[1]) if len(sys.argv) > 1 else 16384, 32, 30
    dev = torch.device("cuda", 0)
    chain, model = config.robot_7dof()
    grid, cam, _ = scene.bench_edt_scene(dims, device=dev)
    mapper = mapping.OccupancyMapper(grid, cam, outside_default=0.8)
    extent = np.array(dims) * grid.voxel_size
    params = config.planner_params(7, {"samples": samples, "horizon": horizon})
    pl = planner.Planner(chain, model, params, device=dev)
    state = robot.JointState.resting(np.full(7, 0.05))
    goal = robot.forward_kinematics(chain, np.full(7, 0.35))[-1]
    nominal = np.zeros((horizon, 7))
    half = np.maximum(extent * 0.25, grid.voxel_size * 2) / 2.0
    center = np.array([0.0, 0.0, extent[2] * 0.5])
    stream = torch.cuda.current_stream(dev)
    ph = {"fusion": [], "edt": [], "step": [], "step_host_us": []}
    import time
    for f in range(frames + 3):
        s_ = -1.0 + 2.0 * (f % 50) / 49.0
        cube_c = np.array([0.4 * s_, 0.25, 0.45])
        boxes = [(center - half, center + half), (cube_c - 0.05, cube_c + 0.05)]
        centers, radii = robot.sphere_positions(chain, np.full(7, 0.3) + 0.01 * f, model)
        depth = mapping.DepthImage(scene.render_boxes(cam, boxes, (centers, radii)))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(stream)
        mapper.update(depth, mask=(centers, radii))
        ev[1].record(stream)
        field = mapper.recompute_edt()
        ev[2].record(stream)
        t0 = time.perf_counter()
        res = pl.smpc_step(state, goal, field, nominal, f)
        t1 = time.perf_counter()
        ev[3].record(stream)
        ev[3].synchronize()
        if f >= 3:
            ph["fusion"].append(ev[0].elapsed_time(ev[1]))
            ph["edt"].append(ev[1].elapsed_time(ev[2]))
            ph["step"].append(ev[2].elapsed_time(ev[3]))
            ph["step_host_us"].append((t1 - t0) * 1e6)
        state = pl.integrate(state, res.command)
        nominal = res.next_nominal
    print(json.dumps({k: round(statistics.median(v), 4) for k, v in ph.items()}))
    # one traced fused step on the last frame's field and state (%globaltimer stamps)
    from paper_2512_22575_b200 import _device as D
    from paper_2512_22575_b200 import _lib
    lib = _lib.load()
    ctas = (samples + 3) // 4
    buf = torch.zeros(2 * ctas + 32, dtype=torch.int64, device=dev)
    nom_dev = torch.from_numpy(nominal).to(dev)
    costs = None
    lib.vpb_debug_smpc_trace(D.ptr(buf))
    out, eps = pl.smpc_generate_device(state, goal, field, nom_dev, 77)
    torch.cuda.synchronize()
    lib.vpb_debug_smpc_trace(None)
    t = buf.cpu().numpy().astype(np.float64)
    t0 = t[0:2 * ctas:2].min()
    done = t[1:2 * ctas:2] - t0
    c = torch.empty(samples, dtype=torch.float64, device=dev)
    pl.smpc_step_device(state, goal, field, nom_dev, eps, costs=c)
    w = planner.soft_weights(c, params.lam)
    print(json.dumps({"cta_done_us_p50_p100": [float(np.percentile(done, 50)) / 1e3, float(done.max()) / 1e3],
                      "merge_start_us": (t[2 * ctas] - t0) / 1e3, "merge_done_us": (t[2 * ctas + 1] - t0) / 1e3,
                      "step_done_us": (t[2 * ctas + 2] - t0) / 1e3,
                      "merge_stamps_us": {k: (t[2 * ctas + i] - t0) / 1e3 for k, i in
                                          (("heads", 14), ("min", 15), ("compacted", 16), ("expanded", 17),
                                           ("best_sums", 18), ("prologue", 19), ("n_start", 13))},
                      "nonzero_weights": int((w > 0).sum()), "cost_min": float(c.min()),
                      "cost_p50": float(c.median())}))


if __name__ == "__main__":
    main()
