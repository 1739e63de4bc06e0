"""Synthetic inputs for benchmarks and smoke tests (host-side, untimed).

Restates the reference's bench and acceptance scenes as data generators:
the CLI EDT bench scene (vp/cli.py:153-179: 0.02 m voxels, origin
(-extent/2, -extent/2, 0), 160x120 camera at z = -1 looking +z, a box of 25%
of the extent centred at z = extent/2), the analytic box depth render
(vp/sim.py:218-258, slab test), the acceptance planner field
(t/test_acceptance.py:308-317) and the reach_static board scene
(vp/data/reach_static.yaml).  Nothing here is on the timed path.
"""

from __future__ import annotations

import numpy as np

from .geometry import RigidTransform
from .mapping import CameraModel, DepthImage, VoxelGrid


def bench_camera() -> CameraModel:
    return CameraModel(fx=120.0, fy=120.0, cx=79.5, cy=59.5, width=160, height=120, d_min=0.05, d_max=20.0,
                       pose=RigidTransform.from_translation((0.0, 0.0, -1.0)))


def render_boxes(cam: CameraModel, boxes, spheres=None) -> np.ndarray:
    """Per-pixel camera-z depth of the nearest axis-aligned box or sphere.

    boxes: iterable of (lo, hi) world corners; spheres: (centers, radii).
    Every pixel ray has unit z in the camera frame, so the ray parameter is
    the depth (vp/sim.py:228-233).  0 where nothing is hit in [d_min, d_max]."""
    us, vs = np.meshgrid(np.arange(cam.width), np.arange(cam.height))
    dirs_cam = np.stack([(us - cam.cx) / cam.fx, (vs - cam.cy) / cam.fy, np.ones_like(us, dtype=float)], axis=-1)
    dirs = dirs_cam @ cam.pose.rotation.matrix.T
    pos = cam.pose.translation
    best = np.full((cam.height, cam.width), np.inf)
    for lo, hi in boxes:
        lo, hi = np.asarray(lo, float), np.asarray(hi, float)
        with np.errstate(divide="ignore", invalid="ignore"):
            t1 = (lo - pos) / dirs
            t2 = (hi - pos) / dirs
        near, far = np.minimum(t1, t2), np.maximum(t1, t2)
        parallel = dirs == 0.0
        inside = (pos >= lo) & (pos <= hi)
        near = np.where(parallel, np.where(inside, -np.inf, np.inf), near)
        far = np.where(parallel, np.where(inside, np.inf, -np.inf), far)
        tmin, tmax = near.max(axis=-1), far.min(axis=-1)
        hit = (tmax >= tmin) & (tmax > 0.0)
        t = np.where(tmin > 0.0, tmin, tmax)
        best = np.where(hit & (t < best), t, best)
    if spheres is not None:
        for c, r in zip(*spheres):
            rel = pos - np.asarray(c, float)
            a = (dirs * dirs).sum(-1)
            b = 2.0 * (dirs * rel).sum(-1)
            cc = (rel * rel).sum() - r * r
            disc = b * b - 4 * a * cc
            ok = disc >= 0
            sd = np.sqrt(np.where(ok, disc, 0.0))
            tn, tf = (-b - sd) / (2 * a), (-b + sd) / (2 * a)
            t = np.where(tn > 0, tn, tf)
            best = np.where(ok & (t > 0) & (t < best), t, best)
    valid = (best >= cam.d_min) & (best <= cam.d_max)
    return np.where(valid, best, 0.0)


def bench_edt_scene(dims, backdrop: bool = False, robot_spheres=None, device=None):
    """(grid, camera, depth) of the CLI EDT bench (vp/cli.py:153-179).

    ``backdrop`` adds a wall behind the volume so every pixel returns (the
    full-coverage variant of SURVEY.md section 8d C2); ``robot_spheres``
    (centers, radii) are rendered into the image so body masking is
    exercised."""
    dims = tuple(int(d) for d in dims)
    voxel = 0.02
    extent = np.array(dims) * voxel
    origin = (-extent[0] / 2.0, -extent[1] / 2.0, 0.0)
    grid = VoxelGrid(origin, voxel, dims, device=device)
    cam = bench_camera()
    half = np.maximum(extent * 0.25, voxel * 2) / 2.0
    center = np.array([0.0, 0.0, extent[2] * 0.5])
    boxes = [(center - half, center + half)]
    if backdrop:
        boxes.append((np.array([-50.0, -50.0, extent[2] + 0.5]), np.array([50.0, 50.0, extent[2] + 0.6])))
    depth = DepthImage(render_boxes(cam, boxes, robot_spheres))
    return grid, cam, depth


def random_occupancy(dims, density: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.random(tuple(dims)) < density


def acceptance_planner_occupancy() -> tuple[tuple, float, np.ndarray]:
    """150x150x25 @ 0.02 m with the [60:80, 60:80, 5:20] block
    (t/test_acceptance.py:308-317).  Returns (origin, voxel, occupancy)."""
    occ = np.zeros((150, 150, 25), bool)
    occ[60:80, 60:80, 5:20] = True
    return (-1.5, -1.5, 0.0), 0.02, occ


def reach_static_occupancy() -> tuple[tuple, float, np.ndarray]:
    """Board + floor of vp/data/reach_static.yaml at 0.025 m (44x60x46)."""
    occ = np.zeros((44, 60, 46), bool)
    occ[29:31, 26:34, 28:40] = True
    occ[:, :, 0:6] = True
    return (-0.35, -0.75, 0.0), 0.025, occ


REACH_STATIC_START = np.array([0.6, 1.0, 0.0, -0.9, 0.0, 0.7, 0.0])
REACH_STATIC_GOAL = [0.3776841587, -0.2583876349, 0.8979771853, 0.8799231763, 0.1150809890, 0.3720255519,
                     -0.2721921353]
REACH_STATIC_QREF = [0.0, 0.95, 0.0, -0.85, 0.0, 0.72, 0.0]


def moving_obstacle_frames(cam: CameraModel, dims, frames: int, chain=None, model=None):
    """Depth frames + body masks of the closed-loop scene:
    the CLI bench box plus a 10 cm cube sweeping past it like the MotionScript
    of vp/data/two_goal_dynamic.yaml:33-41, the 7-DoF body rendered at a
    slowly moving configuration.  Host render (untimed input generation).
    Returns a list of (depth (H, W) f64, (centers, radii))."""
    from . import config, robot

    if chain is None:
        chain, model = config.robot_7dof()
    dims = tuple(int(d) for d in dims)
    voxel = 0.02
    extent = np.array(dims) * voxel
    half = np.maximum(extent * 0.25, voxel * 2) / 2.0
    center = np.array([0.0, 0.0, extent[2] * 0.5])
    out = []
    for f in range(frames):
        s_ = -1.0 + 2.0 * (f % 50) / 49.0
        cube_c = np.array([0.4 * s_, 0.25, 0.45])
        boxes = [(center - half, center + half), (cube_c - 0.05, cube_c + 0.05)]
        centers, radii = robot.sphere_positions(chain, np.full(7, 0.3) + 0.01 * f, model)
        out.append((render_boxes(cam, boxes, (centers, radii)), (centers, radii)))
    return out
