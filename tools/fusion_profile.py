"""Masked fusion calls (256^3 bench scene) for ncu: python tools/fusion_profile.py [n]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_22575_b200 import config, mapping, robot, scene  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
chain, model = config.robot_7dof()
centers, radii = robot.sphere_positions(chain, np.full(7, 0.3), model)
grid, cam, depth = scene.bench_edt_scene((n, n, n), robot_spheres=(centers, radii))
mapper = mapping.OccupancyMapper(grid, cam)
depth.device_tensor(torch.device("cuda", 0))
for _ in range(4):
    mapper.update(depth, mask=(centers, radii))
torch.cuda.synchronize()
