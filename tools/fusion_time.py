"""Masked fusion device times (CUDA events, L2 flushed between calls): the
256^3 bench scene, its full-coverage variant (backdrop) and the 512^3 bench
scene.  Usage: python tools/fusion_time.py [reps]"""

import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2512_22575_b200 import config, mapping, robot, scene  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    chain, model = config.robot_7dof()
    centers, radii = robot.sphere_positions(chain, np.full(7, 0.3), model)
    out = {}
    for name, n, backdrop in (("bench256", 256, False), ("full256", 256, True), ("bench512", 512, False)):
        grid, cam, depth = scene.bench_edt_scene((n, n, n), backdrop=backdrop, robot_spheres=(centers, radii))
        mapper = mapping.OccupancyMapper(grid, cam)
        depth.device_tensor(dev)
        mapper.update(depth, mask=(centers, radii))
        touched = int(grid.observed.sum().item())
        ts = []
        for k in range(reps):
            flush.fill_(k & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mapper.update(depth, mask=(centers, radii))
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name] = {"us": round(statistics.mean(ts) * 1000, 2), "touched": touched}
    print(json.dumps({"fusion": out}))


if __name__ == "__main__":
    main()
