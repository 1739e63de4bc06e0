"""Phase timeline of one fused SMPC step (C3 scene): per-CTA start / candidates
done (%globaltimer), merge and tail stamps.  Prints a JSON summary."""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def _pct(v, t0):
    v = v[v > 0]
    return [float(np.percentile(v - t0, p)) / 1e3 for p in (0, 50, 100)] if v.size else []


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=4096)
    ap.add_argument("--horizon", type=int, default=32)
    ap.add_argument("--flush", action="store_true", help="write 256 MiB before each traced launch (cold L2)")
    ap.add_argument("--converged", action="store_true",
                    help="bench.py's converged-regime C3 scene (reach_static after 30 replans: many nonzero weights)")
    ap.add_argument("--code-warm", action="store_true",
                    help="after the flush, run a 4-sample step first (pulls the kernel's code into L2, not the data)")
    a = ap.parse_args()
    import bench
    from paper_2512_22575_b200 import _device as D
    from paper_2512_22575_b200 import _lib

    args = argparse.Namespace(samples=a.samples, horizon=a.horizon, grid=256, precision="fp32")
    if a.converged:
        from paper_2512_22575_b200 import config, mapping, planner, robot, scene
        from paper_2512_22575_b200.geometry import RigidTransform

        dev = torch.device("cuda", 0)
        chain, model = config.robot_7dof()
        origin, voxel, occ = scene.reach_static_occupancy()
        grid = mapping.VoxelGrid(origin, voxel, occ.shape, device=dev)
        grid.set_log_odds(np.where(occ, 3.5, 0.0))
        field = mapping.edt_3d(grid, outside_default=0.8)
        params = config.planner_params(7, {"samples": a.samples, "horizon": a.horizon,
                                           "q_ref": scene.REACH_STATIC_QREF})
        pl = planner.Planner(chain, model, params, precision="fp32", device=dev)
        goal = RigidTransform.from_vec7(scene.REACH_STATIC_GOAL)
        st = robot.JointState.resting(scene.REACH_STATIC_START)
        nominal = np.zeros((a.horizon, 7))
        for f in range(30):
            res = pl.smpc_step(st, goal, field, nominal, 1000 + f)
            st = pl.integrate(st, res.command)
            nominal = res.next_nominal
        nom = torch.from_numpy(nominal).to(dev)
    else:
        S = bench.make_scene(args, torch.device("cuda", 0))
        pl, st, goal, field = S["planner"], S["state"], S["goal"], S["field"]
        nom = torch.zeros((a.horizon, 7), dtype=torch.float64, device="cuda")
    eps = pl.sample_device(3)
    ctas = (a.samples + 3) // 4  # fixed-topology path: 4 candidates per CTA
    buf = torch.zeros(2 * ctas + 32 + 3 * 128, dtype=torch.int64, device="cuda")
    for _ in range(5):
        pl.smpc_step_device(st, goal, field, nom, eps)
    torch.cuda.synchronize()
    lib = _lib.load()
    res = []
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda") if a.flush else None
    for it in range(11):
        buf.zero_()
        if flush is not None:
            flush.fill_(it)
        if a.code_warm:
            pl.smpc_generate_device(st, goal, field, nom, 7, samples=4)
        lib.vpb_debug_smpc_trace(D.ptr(buf))
        pl.smpc_generate_device(st, goal, field, nom, 3 + it)  # the production (fused-draw) step
        torch.cuda.synchronize()
        lib.vpb_debug_smpc_trace(None)
        t = buf.cpu().numpy().astype(np.float64)
        t0 = t[0:2 * ctas:2].min()
        start = t[0:2 * ctas:2] - t0
        done = t[1:2 * ctas:2] - t0
        res.append({
            "cta_start_us": [float(np.percentile(start, p)) / 1e3 for p in (0, 50, 90, 100)],
            "cta_eval_us_p50": float(np.median(done - start)) / 1e3,
            "cta_done_us": [float(np.percentile(done, p)) / 1e3 for p in (0, 50, 90, 100)],
            "group_merges_done_us": (t[2 * ctas] - t0) / 1e3,
            "global_merge_done_us": (t[2 * ctas + 1] - t0) / 1e3,
            "step_done_us": (t[2 * ctas + 2] - t0) / 1e3,
            "some_partials_written_us": [(x - t0) / 1e3 for x in t[2 * ctas + 3:2 * ctas + 7]],
            "u_star_done_us": (t[2 * ctas + 11] - t0) / 1e3,
            "reeval_done_us": (t[2 * ctas + 12] - t0) / 1e3,
            "global_merge_head_done_us": (t[2 * ctas + 13] - t0) / 1e3,
            "merge_heads_loaded_us": (t[2 * ctas + 14] - t0) / 1e3,
            "merge_min_known_us": (t[2 * ctas + 15] - t0) / 1e3,
            "merge_ctas_compacted_us": (t[2 * ctas + 16] - t0) / 1e3,
            "merge_expansion_done_us": (t[2 * ctas + 17] - t0) / 1e3,
            "merge_best_sums_fetched_us": (t[2 * ctas + 18] - t0) / 1e3,
            "merge_prologue_fetched_us": (t[2 * ctas + 19] - t0) / 1e3,
            "heavy_verdict_us": (t[2 * ctas + 20] - t0) / 1e3,
            "heavy_own_part_us": (t[2 * ctas + 21] - t0) / 1e3,
            "heavy_helpers_done_us": (t[2 * ctas + 22] - t0) / 1e3,
            "heavy_sums_done_us": (t[2 * ctas + 23] - t0) / 1e3,
            "slowest_ctas": [int(i) for i in np.argsort(done)[-6:]],
            # heavy merge, per helper that took part: woke (saw the verdict), first weights done, own part done
            "helper_woke_us": _pct(t[2 * ctas + 32::3], t0),
            "helper_weights_done_us": _pct(t[2 * ctas + 33::3], t0),
            "helper_part_done_us": _pct(t[2 * ctas + 34::3], t0),
            "helper_weights_dur_by_part_us": [round(float(b - a) / 1e3, 2) for a, b in
                                              zip(t[2 * ctas + 32::3], t[2 * ctas + 33::3]) if a > 0][:128],
            "helper_part_dur_by_part_us": [round(float(b - a) / 1e3, 2) for a, b in
                                           zip(t[2 * ctas + 32::3], t[2 * ctas + 34::3]) if a > 0][:128],
            "done_by_cta_decile_us": [float(np.median(d)) / 1e3 for d in np.array_split(done, 10)],
        })
    out = dict(res[-1])
    for k, v in out.items():  # scalar stamps: median over the traced steps
        if isinstance(v, float):
            out[k] = float(np.median([r[k] for r in res]))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
