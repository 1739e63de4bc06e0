"""EDT calls for ncu: the 256^3 bench scene (masked, 2 updates) and a random
grid (density argv[1], default 0.1; size argv[2], default 256)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_22575_b200 import config, mapping, robot, scene  # noqa: E402

dens = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
chain, model = config.robot_7dof()
centers, radii = robot.sphere_positions(chain, np.full(7, 0.3), model)
grid, cam, depth = scene.bench_edt_scene((n, n, n), robot_spheres=(centers, radii))
mapper = mapping.OccupancyMapper(grid, cam)
for _ in range(2):
    mapper.update(depth, mask=(centers, radii))
g = mapping.VoxelGrid((0, 0, 0), 0.02, (n, n, n))
occ = torch.rand((n, n, n), device="cuda", generator=torch.Generator(device="cuda").manual_seed(7)) < dens
g.set_log_odds(torch.where(occ, 3.5, 0.0).double())
mapping.edt_3d(g)
torch.cuda.synchronize()
for _ in range(2):
    mapping.edt_3d(grid)  # bench scene first
    mapping.edt_3d(g)
torch.cuda.synchronize()
