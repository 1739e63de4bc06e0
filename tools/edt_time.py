"""EDT device times (CUDA events, L2 flushed between calls) on the bench
scene and on random occupancy at 256^3 / 512^3, plus a bit-exact spot check
against the oracle at 256^3.  Usage: python tools/edt_time.py [reps]"""

import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2512_22575_b200 import config, mapping, robot, scene  # noqa: E402


def time_edt(grid, reps, flush):
    mapping.edt_3d(grid)
    torch.cuda.synchronize()
    ts = []
    for k in range(reps):
        flush.fill_(k & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mapping.edt_3d(grid)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.mean(ts)


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {}
    chain, model = config.robot_7dof()
    centers, radii = robot.sphere_positions(chain, np.full(7, 0.3), model)
    for n in (256, 512):
        grid, cam, depth = scene.bench_edt_scene((n, n, n), robot_spheres=(centers, radii))
        mapper = mapping.OccupancyMapper(grid, cam)
        for _ in range(2):
            mapper.update(depth, mask=(centers, radii))
        out[f"bench{n}"] = time_edt(grid, reps, flush)
        for dens in (0.01, 0.1, 0.5):
            g = mapping.VoxelGrid((0, 0, 0), 0.02, (n, n, n))
            occ = torch.rand((n, n, n), device=dev, generator=torch.Generator(device=dev).manual_seed(7)) < dens
            g.set_log_odds(torch.where(occ, 3.5, 0.0).double())
            out[f"rand{n}_{dens}"] = time_edt(g, reps, flush)
            if n == 256 and dens == 0.1 and "--check" in sys.argv:
                import oracle
                oracle.set_threads(0)
                got = mapping.edt_3d(g).sq
                assert np.array_equal(got, oracle.edt3d_from_occupancy(occ.cpu().numpy())), "EDT mismatch"
                out["check"] = "bit-exact"
    out = {k: (round(v * 1000, 2) if isinstance(v, float) else v) for k, v in out.items()}
    print(json.dumps({"edt_us": out}))


if __name__ == "__main__":
    main()
