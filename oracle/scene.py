"""Host-only restatement of the benchmark scene for the reference arm.

TEST INFRASTRUCTURE (like the rest of oracle/): only tests/, bench.py's
cpu_baseline / --impl reference legs and __graft_entry__.smoke() use it.  It
imports numpy and the oracle's own C library, never the product package, so
`bench.py --impl reference` loads no product code (VERDICT r1 "bench
integrity").  tests/test_oracle_golden.py checks that it builds the same
problem as the product's host mirror.

What it restates (each from the reference file it follows):
  * the generic 7-DoF arm: vp/data/robot_7dof.yaml:9-77 (joints = pure z
    offsets, identity base, 11 spheres, 18 self pairs);
  * forward kinematics and sphere centres: vp/robot.py:172-200 (frame i+1 =
    frame i * offset_i * Rot(axis_i, q_i), Rodrigues vp/geometry.py);
  * the planner defaults: vp/data/planner_defaults.yaml:4-20 and
    tightened_limits vp/planner.py:291-306;
  * the CLI EDT bench scene: vp/cli.py:153-179 and the box depth render of
    vp/sim.py:218-258 (slab test; spheres rendered for the body mask).
"""

from __future__ import annotations

import numpy as np

from . import edt3d, fuse_voxels, masked_pixels

# vp/data/robot_7dof.yaml:9-77
JOINT_Z = np.array([0.15, 0.10, 0.25, 0.15, 0.25, 0.10, 0.12])
JOINT_AXES = np.array([[0, 0, 1], [0, 1, 0], [0, 0, 1], [0, 1, 0], [0, 0, 1], [0, 1, 0], [0, 0, 1]], float)
POS_LIMIT = np.array([2.9, 2.0, 2.9, 2.2, 2.9, 2.0, 2.9])
VEL_LIMIT = np.full(7, 2.5)
ACC_LIMIT = np.full(7, 10.0)
SPHERES = [(0, 0.08, 0.09), (1, 0.05, 0.08), (2, 0.08, 0.08), (2, 0.17, 0.08), (3, 0.05, 0.07),
           (3, 0.11, 0.07), (4, 0.08, 0.07), (4, 0.17, 0.07), (5, 0.05, 0.06), (6, 0.06, 0.06), (7, 0.02, 0.05)]
SELF_PAIRS = [[0, 6], [0, 7], [0, 8], [0, 9], [0, 10], [1, 6], [1, 7], [1, 9], [1, 10],
              [2, 6], [2, 7], [2, 10], [3, 8], [3, 9], [3, 10], [4, 9], [4, 10], [5, 10]]

# vp/data/planner_defaults.yaml:4-20
DEFAULTS = dict(dt=0.02, lam=0.05, sigma=1.0, noise_window=5, w_env=5e4, w_self=5e4, w_q=100.0, w_qd=100.0,
                w_qdd=100.0, w_s=0.01, w_ns=0.1, d_act=0.05, margin_frac=0.02)
POSE_W = np.diag([200.0, 200.0, 200.0, 80.0, 80.0, 80.0])
TERM_W = np.diag([2000.0, 2000.0, 2000.0, 800.0, 800.0, 800.0])


def rodrigues(axis, angle):
    """Rotation about a unit axis (vp/geometry.py Rotation3.from_axis_angle)."""
    x, y, z = axis
    k = np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])
    return np.eye(3) + np.sin(angle) * k + (1.0 - np.cos(angle)) * (k @ k)


def fk_frames(q):
    """[(R, t)] base first, flange last (vp/robot.py:172-189)."""
    r, t = np.eye(3), np.zeros(3)
    frames = [(r, t)]
    for i in range(7):
        t = t + r @ np.array([0.0, 0.0, JOINT_Z[i]])
        r = r @ rodrigues(JOINT_AXES[i], float(q[i]))
        frames.append((r, t))
    return frames


def sphere_positions(q):
    """World sphere centres and radii (vp/robot.py:192-200)."""
    frames = fk_frames(q)
    c = np.array([frames[link][1] + frames[link][0] @ np.array([0.0, 0.0, cz]) for link, cz, _ in SPHERES])
    return c, np.array([r for _, _, r in SPHERES])


def tightened_limits(margin_frac):
    """vp/planner.py:291-306."""
    eps_q = margin_frac * 2.0 * POS_LIMIT
    eps_v = margin_frac * 2.0 * VEL_LIMIT
    eps_a = margin_frac * 2.0 * ACC_LIMIT
    return (-POS_LIMIT + eps_q, POS_LIMIT - eps_q, -VEL_LIMIT + eps_v, VEL_LIMIT - eps_v,
            -ACC_LIMIT + eps_a, ACC_LIMIT - eps_a)


class Camera:
    """The CLI bench camera (vp/cli.py:160-170): 160x120, f = 120, at z = -1 looking +z."""

    fx = fy = 120.0
    cx, cy = 79.5, 59.5
    width, height = 160, 120
    d_min, d_max = 0.05, 20.0
    pose_r = np.eye(3)
    pose_t = np.array([0.0, 0.0, -1.0])

    def world_to_camera(self):
        return self.pose_r.T, -self.pose_r.T @ self.pose_t


def render_boxes(cam, boxes, spheres=None):
    """Camera-z depth of the nearest box / sphere per pixel (vp/sim.py:218-258)."""
    us, vs = np.meshgrid(np.arange(cam.width), np.arange(cam.height))
    dirs = np.stack([(us - cam.cx) / cam.fx, (vs - cam.cy) / cam.fy, np.ones_like(us, dtype=float)], -1)
    dirs = dirs @ cam.pose_r.T
    pos = cam.pose_t
    best = np.full((cam.height, cam.width), np.inf)
    for lo, hi in boxes:
        lo, hi = np.asarray(lo, float), np.asarray(hi, float)
        with np.errstate(divide="ignore", invalid="ignore"):
            t1, t2 = (lo - pos) / dirs, (hi - pos) / dirs
        near, far = np.minimum(t1, t2), np.maximum(t1, t2)
        par = dirs == 0.0
        inside = (pos >= lo) & (pos <= hi)
        near = np.where(par, np.where(inside, -np.inf, np.inf), near)
        far = np.where(par, np.where(inside, np.inf, -np.inf), far)
        tmin, tmax = near.max(-1), far.min(-1)
        hit = (tmax >= tmin) & (tmax > 0.0)
        t = np.where(tmin > 0.0, tmin, tmax)
        best = np.where(hit & (t < best), t, best)
    if spheres is not None:
        for c, r in zip(*spheres):
            rel = pos - np.asarray(c, float)
            a = (dirs * dirs).sum(-1)
            b = 2.0 * (dirs * rel).sum(-1)
            disc = b * b - 4 * a * ((rel * rel).sum() - r * r)
            ok = disc >= 0
            sd = np.sqrt(np.where(ok, disc, 0.0))
            tn, tf = (-b - sd) / (2 * a), (-b + sd) / (2 * a)
            t = np.where(tn > 0, tn, tf)
            best = np.where(ok & (t > 0) & (t < best), t, best)
    return np.where((best >= cam.d_min) & (best <= cam.d_max), best, 0.0)


def bench_map(n: int, updates: int = 2, q_mask=0.3):
    """The C2 map built on the host: CLI bench scene at n^3 (0.02 m voxels),
    7-DoF body mask at q = q_mask, `updates` masked fusions (serial oracle,
    like the reference) and the EDT.  Returns dict(log_odds, observed, sq,
    origin, voxel, depth, centers, radii, cam)."""
    voxel = 0.02
    dims = (n, n, n)
    extent = np.array(dims) * voxel
    origin = np.array([-extent[0] / 2.0, -extent[1] / 2.0, 0.0])
    cam = Camera()
    half = np.maximum(extent * 0.25, voxel * 2) / 2.0
    center = np.array([0.0, 0.0, extent[2] * 0.5])
    centers, radii = sphere_positions(np.full(7, q_mask))
    depth = render_boxes(cam, [(center - half, center + half)], (centers, radii))
    lo = np.zeros(dims)
    ob = np.zeros(dims, bool)
    pm = masked_pixels(depth, cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max, cam.pose_r, cam.pose_t,
                       centers, radii, 0.01)
    r, t = cam.world_to_camera()
    for _ in range(updates):
        fuse_voxels(lo, ob, (0, 0, 0), dims, origin, voxel, r, t, cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                    cam.height, cam.d_min, cam.d_max, depth, pm, centers, radii, 2.5 * voxel, 0.85, -0.4, -2.0, 3.5)
    return dict(log_odds=lo, observed=ob, sq=edt3d(lo), origin=origin, voxel=voxel, depth=depth, centers=centers,
                radii=radii, cam=cam, pixel_mask=pm)


def rollout_args(sq, origin, voxel, outside=0.8, q0=0.05, q_goal=0.35, q_ref=None, lo=(0, 0, 0)):
    """evaluate_batch's named inputs (vp/batch.py:162-212) for the bench
    problem: resting state at q0, goal = FK(q_goal) flange, planner defaults."""
    gr, gt = fk_frames(np.full(7, q_goal))[-1]
    sph = np.array([[0.0, 0.0, cz] for _, cz, _ in SPHERES])
    args = {
        "q0": np.full(7, q0), "qd0": np.zeros(7), "dt": DEFAULTS["dt"], "base_r": np.eye(3), "base_t": np.zeros(3),
        "off_r": np.tile(np.eye(3), (7, 1, 1)), "off_t": np.array([[0.0, 0.0, z] for z in JOINT_Z]),
        "axes": JOINT_AXES.copy(), "sph_link": np.array([s[0] for s in SPHERES]), "sph_loc": sph,
        "sph_r": np.array([s[2] for s in SPHERES]), "pairs": np.array(SELF_PAIRS), "goal_r": gr, "goal_t": gt,
        "pose_weight": POSE_W, "terminal_weight": TERM_W,
        "q_ref": np.zeros(7) if q_ref is None else np.asarray(q_ref, float),
        "field_sq": sq, "field_lo0": lo[0], "field_lo1": lo[1], "field_lo2": lo[2], "field_origin0": origin[0],
        "field_origin1": origin[1], "field_origin2": origin[2], "field_voxel": voxel, "field_outside": outside,
    }
    for k in ("w_env", "w_self", "w_q", "w_qd", "w_qdd", "w_s", "w_ns", "d_act"):
        args[k] = DEFAULTS[k]
    for k, v in zip(("pos_lo", "pos_hi", "vel_lo", "vel_hi", "acc_lo", "acc_hi"),
                    tightened_limits(DEFAULTS["margin_frac"])):
        args[k] = v
    return args


def moving_obstacle_frames(dims, frames: int):
    """Host copy of the closed-loop input sequence (the product's
    scene.moving_obstacle_frames): the bench box plus a
    10 cm cube sweeping along x, the body at q = 0.3 + 0.01 f.
    Returns [(depth, (centers, radii))]."""
    voxel = 0.02
    extent = np.array(dims) * voxel
    half = np.maximum(extent * 0.25, voxel * 2) / 2.0
    center = np.array([0.0, 0.0, extent[2] * 0.5])
    cam = Camera()
    out = []
    for f in range(frames):
        s_ = -1.0 + 2.0 * (f % 50) / 49.0
        cube_c = np.array([0.4 * s_, 0.25, 0.45])
        spheres = sphere_positions(np.full(7, 0.3) + 0.01 * f)
        out.append((render_boxes(cam, [(center - half, center + half), (cube_c - 0.05, cube_c + 0.05)], spheres),
                    spheres))
    return out
