"""Generate golden parity vectors by running the REFERENCE implementation.

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [name,name,...]

Every case below is built from the reference's own tests, CLI bench scenes and
acceptance scenes (file:line cited per case) and stores both the inputs and the
reference's outputs.  The oracle (oracle/vp_oracle.c) is pinned against these
files by tests/test_oracle_golden.py; the CUDA path is then checked against
the oracle (and these files) by the -m gpu tests.

Outputs (compressed npz, a few MB in total):
  edt.npz       fh_1d and edt_3d cases (vp/mapping.py:458-613)
  fusion.npz    _masked_pixels + _fuse_voxels sequences (vp/mapping.py:266-455)
  query.npz     _query_metric probes (vp/mapping.py:616-710)
  rollout.npz   evaluate_batch cases with all 49 packed args (vp/batch.py:161-336)
  softmin.npz   soft_weights / update_controls / smpc_step (vp/planner.py:373-630)
  edt_acceptance.npz  all 100 grids of acceptance criterion 1 (t/test_acceptance.py:57-81)
  integrate.npz Planner.integrate sequences (vp/planner.py:632-636)
"""

from __future__ import annotations

import math
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, "/root/reference/pkg/src")

from voxplan import config  # noqa: E402
from voxplan.cli import _bench_edt_scene  # noqa: E402
from voxplan.geometry import RigidTransform  # noqa: E402
from voxplan.mapping import (  # noqa: E402
    CameraModel,
    DepthImage,
    VoxelBox,
    VoxelGrid,
    _masked_pixels,
    edt_3d,
    fh_1d,
    query_distance,
    update_occupancy,
)
from voxplan.oracles import raycast_box_depth  # noqa: E402
from voxplan.planner import (  # noqa: E402
    Planner,
    _field_arguments,
    sample_perturbations,
    soft_weights,
    update_controls,
)
from voxplan.robot import JointState, forward_kinematics, load_robot, sphere_positions  # noqa: E402

OUT = Path(__file__).resolve().parent
INF = np.inf


def sq_to_i32(sq: np.ndarray) -> np.ndarray:
    """Exact integer squared distances; -1 encodes +inf."""
    out = np.where(np.isfinite(sq), sq, -1.0)
    assert np.all(out == np.round(out))
    return out.astype(np.int32)


# --------------------------------------------------------------------------
# EDT
# --------------------------------------------------------------------------
def make_edt() -> dict:
    d: dict[str, np.ndarray] = {}
    # fh_1d known answers, t/test_mapping.py:91-110
    lines = [
        np.array([INF, INF, 0.0, INF, INF]),
        np.zeros(7),
        np.full(6, INF),
    ]
    rng = np.random.default_rng(2)
    for _ in range(30):
        n = rng.integers(1, 40)
        line = rng.integers(0, 50, size=n).astype(float)
        line[rng.random(n) < 0.5] = INF
        lines.append(line)
    for i, line in enumerate(lines):
        d[f"fh_in_{i}"] = line
        d[f"fh_out_{i}"] = fh_1d(line)
    d["fh_count"] = np.array(len(lines))

    cases = []  # (name, occupancy bool array (grid), lo, hi)

    def add(name, occ, lo=None, hi=None):
        cases.append((name, occ.astype(bool), lo, hi))

    occ = np.zeros((3, 3, 3), bool)
    occ[1, 1, 1] = True
    add("center3", occ)  # t/test_mapping.py:121-127
    add("empty4", np.zeros((4, 4, 4), bool))  # :129-132
    add("full4", np.ones((4, 4, 4), bool))  # :134-138
    rng = np.random.default_rng(5)  # :140-150
    for i in range(10):
        density = rng.uniform(0.01, 0.5)
        add(f"rand12_{i}", rng.random((12, 12, 12)) < density)
    rng = np.random.default_rng(7)  # :152-161
    add("order_9x11x6", rng.random((9, 11, 6)) < 0.1)
    occ = np.zeros((6, 6, 6), bool)  # :176-182
    occ[1, 1, 1] = occ[5, 5, 5] = True
    add("subvol6", occ, (0, 0, 0), (3, 3, 3))
    add("subvol6_off", occ, (1, 2, 0), (6, 5, 4))
    rng = np.random.default_rng(20240817)  # t/test_acceptance.py:57-81 seeds
    for i in range(12):
        density = rng.uniform(0.01, 0.5)
        add(f"acc16_{i}", rng.random((16, 16, 16)) < density)
    # ragged / degenerate shapes and line lengths
    rng = np.random.default_rng(99)
    add("line_1x1x37", rng.random((1, 1, 37)) < 0.1)
    add("line_33x1x1", rng.random((33, 1, 1)) < 0.1)
    add("slab_5x40x1", rng.random((5, 40, 1)) < 0.05)
    add("single_voxel_occ", np.ones((1, 1, 1), bool))
    add("single_voxel_free", np.zeros((1, 1, 1), bool))
    occ = np.zeros((23, 17, 29), bool)
    occ[0, 0, 0] = True
    add("corner_source_23x17x29", occ)
    add("sparse_40x40x30", np.random.default_rng(17).random((40, 40, 30)) < 0.01)
    add("odd_65x33x70", np.random.default_rng(3).random((65, 33, 70)) < 0.002)
    # the acceptance planner field (t/test_acceptance.py:308-317)
    occ = np.zeros((150, 150, 25), bool)
    occ[60:80, 60:80, 5:20] = True
    add("acc_planner_150x150x25", occ)
    for i, (name, occ, lo, hi) in enumerate(cases):
        grid = VoxelGrid((0.0, 0.0, 0.0), 0.1, occ.shape)
        grid.log_odds[occ] = grid.params.l_max
        box = None if lo is None else VoxelBox(lo, hi)
        field = edt_3d(grid, box)
        b = box or grid.full_box()
        d[f"edt_name_{i}"] = np.array(name)
        d[f"edt_occ_{i}"] = np.packbits(occ.reshape(-1))
        d[f"edt_dims_{i}"] = np.array(occ.shape, np.int64)
        d[f"edt_lo_{i}"] = np.array(b.lo, np.int64)
        d[f"edt_hi_{i}"] = np.array(b.hi, np.int64)
        d[f"edt_sq_{i}"] = sq_to_i32(field.sq)
    d["edt_count"] = np.array(len(cases))
    # log-odds thresholding exactly at the boundary (l >= 1.0 is occupied)
    grid = VoxelGrid((0.0, 0.0, 0.0), 0.1, (6, 7, 8))
    rng = np.random.default_rng(123)
    vals = rng.choice(
        [1.0, np.nextafter(1.0, 0.0), 0.9999999999999999, 0.0, -2.0, 3.5, 0.85, 1.7], size=(6, 7, 8)
    )
    grid.log_odds[:] = vals
    d["thr_log_odds"] = vals
    d["thr_sq"] = sq_to_i32(edt_3d(grid).sq)
    return d


# --------------------------------------------------------------------------
# Fusion
# --------------------------------------------------------------------------
def classification_scene():
    """t/test_mapping.py:244-278 (copied parameters, not code)."""
    origin = np.array([-1.0, -1.0, 0.0])
    voxel = 0.05
    dims = (40, 40, 40)
    box_lo = np.array([-0.2, -0.3, 0.8])
    box_hi = np.array([0.2, 0.3, 1.2])
    pose = RigidTransform.from_translation((0.0, 0.0, -0.8))
    cam = CameraModel(70.0, 70.0, 40.0, 30.0, 80, 60, 0.1, 6.0, pose=pose)
    depth = raycast_box_depth(
        pose.translation, pose.rotation.matrix, cam.fx, cam.fy, cam.cx, cam.cy,
        cam.width, cam.height, cam.d_min, cam.d_max, [(box_lo, box_hi)],
    )
    return origin, voxel, dims, cam, DepthImage(depth)


def cam_dict(prefix, cam, d):
    d[prefix + "intr"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max])
    d[prefix + "wh"] = np.array([cam.width, cam.height], np.int64)
    d[prefix + "pose_r"] = cam.pose.rotation.matrix.copy()
    d[prefix + "pose_t"] = cam.pose.translation.copy()
    r, t = cam.world_to_camera()
    d[prefix + "w2c_r"] = np.ascontiguousarray(r)
    d[prefix + "w2c_t"] = np.ascontiguousarray(t)


def make_fusion() -> dict:
    d: dict[str, np.ndarray] = {}
    cases = []
    chain, model = load_robot(config.bundled_scenario_path("robot_7dof"))

    # (a) classification scene + mask sphere, 2 updates (t/test_mapping.py:227-241)
    origin, voxel, dims, cam, depth = classification_scene()
    mask = (np.array([[0.5, 0.5, 0.5]]), np.array([0.15]))
    cases.append(("classification", origin, voxel, dims, cam, [depth] * 2, [mask] * 2, None, 0.01))
    # (b) mask parked on the box surface, 4 updates (t/test_mapping.py:280-305)
    mask = (np.array([[0.0, 0.0, 0.8]]), np.array([0.12]))
    cases.append(("mask_on_surface", origin, voxel, dims, cam, [depth] * 4, [mask] * 4, None, 0.01))
    # (c) sub-volume update (VoxelBox) of the same scene
    cases.append(("subvolume", origin, voxel, dims, cam, [depth] * 3, [None] * 3, ((5, 3, 10), (33, 40, 37)), 0.01))
    # (d) CLI bench scene 64^3 (vp/cli.py:153-179) with the 7-DoF body mask at
    #     q = 0.3, 3 updates; robot spheres also
    #     rendered so masked pixels are exercised.
    grid, bcam, bdepth = _bench_edt_scene((64, 64, 64))
    q = np.full(7, 0.3)
    centers, radii = sphere_positions(chain, q, model)
    from voxplan.sim import BoxShape, MotionScript, Obstacle, advance_world, render_depth

    extent = np.array((64, 64, 64)) * 0.02
    box = Obstacle(
        BoxShape(tuple(np.maximum(extent * 0.25, 0.04))),
        MotionScript.fixed(RigidTransform.from_translation((0.0, 0.0, float(extent[2]) * 0.5))),
    )
    depth_robot = render_depth([box], advance_world([box], 0.0), bcam, extra_spheres=(centers, radii))
    cases.append(
        ("bench64_masked", grid.origin, grid.voxel_size, grid.dims, bcam,
         [bdepth, depth_robot, depth_robot], [(centers, radii)] * 3, None, 0.01)
    )
    # (e) single-voxel known answers (t/test_mapping.py:190-225)
    ucam = CameraModel(fx=1.0, fy=1.0, cx=0.0, cy=0.0, width=1, height=1, d_min=0.1, d_max=5.0)
    for cz in (1.0, 2.5, 2.0):
        cases.append(
            (f"single_z{cz}", np.array([-0.05, -0.05, cz - 0.05]), 0.1, (1, 1, 1), ucam,
             [DepthImage(np.array([[2.0]]))] * 20, [None] * 20, None, 0.01)
        )
    # (f) rational threshold sequence: 5 misses then h,h,h,h,m
    #     vs h,h,h,m,h on one voxel via depth switching.
    seq1 = [3.0] * 5 + [2.0, 2.0, 2.0, 2.0, 3.0]
    seq2 = [3.0] * 5 + [2.0, 2.0, 2.0, 3.0, 2.0]
    for name, seq in (("rational_a", seq1), ("rational_b", seq2)):
        cases.append(
            (name, np.array([-0.05, -0.05, 1.95]), 0.1, (1, 1, 1), ucam,
             [DepthImage(np.array([[s]])) for s in seq], [None] * len(seq), None, 0.01)
        )

    for i, (name, origin, voxel, dims, cam, depths, masks, box, pad) in enumerate(cases):
        grid = VoxelGrid(origin, voxel, dims)
        d[f"f_name_{i}"] = np.array(name)
        d[f"f_origin_{i}"] = np.asarray(origin, float)
        d[f"f_voxel_{i}"] = np.array(voxel, float)
        d[f"f_dims_{i}"] = np.array(dims, np.int64)
        d[f"f_pad_{i}"] = np.array(pad)
        if box is not None:
            d[f"f_box_{i}"] = np.array([box[0], box[1]], np.int64)
        cam_dict(f"f_cam{i}_", cam, d)
        d[f"f_nsteps_{i}"] = np.array(len(depths))
        vb = VoxelBox(*box) if box is not None else None
        for s, (dep, msk) in enumerate(zip(depths, masks)):
            d[f"f_depth_{i}_{s}"] = dep.data
            if msk is not None:
                d[f"f_mc_{i}_{s}"] = np.asarray(msk[0], float).reshape(-1, 3)
                d[f"f_mr_{i}_{s}"] = np.asarray(msk[1], float).reshape(-1)
                pm = _masked_pixels(dep, cam, d[f"f_mc_{i}_{s}"], d[f"f_mr_{i}_{s}"], pad)
            else:
                pm = np.zeros(dep.data.shape, bool)
            d[f"f_pm_{i}_{s}"] = pm
            update_occupancy(grid, dep, cam, mask=msk, volume=vb, mask_pad=pad)
            d[f"f_lo_{i}_{s}"] = grid.log_odds.copy()
            d[f"f_ob_{i}_{s}"] = grid.observed.copy()
    d["f_count"] = np.array(len(cases))
    return d


# --------------------------------------------------------------------------
# Query
# --------------------------------------------------------------------------
def make_query() -> dict:
    d: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(31)
    fields = []
    # lone source field (t/test_mapping.py:339-368)
    grid = VoxelGrid((0.0, 0.0, 0.0), 0.1, (5, 5, 5))
    grid.log_odds[2, 2, 2] = grid.params.l_max
    fields.append(("lone5", grid, None, 0.7))
    grid = VoxelGrid((0.0, 0.0, 0.0), 0.1, (3, 3, 3))
    fields.append(("empty3", grid, None, 1.0))
    grid = VoxelGrid((-1.0, -1.0, 0.0), 0.05, (40, 40, 30))
    grid.log_odds[np.random.default_rng(17).random((40, 40, 30)) < 0.01] = grid.params.l_max
    fields.append(("sparse40", grid, VoxelBox((3, 5, 2), (37, 31, 28)), 0.8))
    for i, (name, grid, box, outside) in enumerate(fields):
        field = edt_3d(grid, box, outside_default=outside)
        lo = np.asarray(grid.origin) - 0.1
        hi = np.asarray(grid.origin) + np.asarray(grid.dims) * grid.voxel_size + 0.1
        pts = rng.uniform(lo, hi, size=(600, 3))
        # exact voxel centres, faces and corners
        idx = rng.integers(0, np.asarray(grid.dims), size=(100, 3))
        pts = np.vstack([pts, grid.origin + (idx + 0.5) * grid.voxel_size,
                         grid.origin + idx * grid.voxel_size])
        vals = np.array([query_distance(field, p) for p in pts])
        b = field.volume
        d[f"q_name_{i}"] = np.array(name)
        d[f"q_sq_{i}"] = sq_to_i32(field.sq)
        d[f"q_lo_{i}"] = np.array(b.lo, np.int64)
        d[f"q_meta_{i}"] = np.array([*grid.origin, grid.voxel_size, outside])
        d[f"q_pts_{i}"] = pts
        d[f"q_val_{i}"] = vals
    d["q_count"] = np.array(len(fields))
    return d


# --------------------------------------------------------------------------
# Rollout
# --------------------------------------------------------------------------
ROLLOUT_KEYS = (
    "q0 qd0 dt base_r base_t off_r off_t axes sph_link sph_loc sph_r pairs goal_r goal_t "
    "pose_weight terminal_weight pos_lo pos_hi vel_lo vel_hi acc_lo acc_hi w_env w_self w_q "
    "w_qd w_qdd w_s w_ns d_act q_ref field_sq field_lo0 field_lo1 field_lo2 field_origin0 "
    "field_origin1 field_origin2 field_voxel field_outside"
).split()


def pack_args(planner: Planner, state, goal, snap) -> dict:
    p = planner.params
    vals = [
        np.ascontiguousarray(state.q, float), np.ascontiguousarray(state.qd, float), p.dt,
        planner._base_r, planner._base_t, planner._off_r, planner._off_t, planner._axes,
        planner._sph_link, planner._sph_loc, planner._sph_r, planner._pairs,
        np.ascontiguousarray(goal.rotation.matrix), np.ascontiguousarray(goal.translation),
        p.pose_weight, p.terminal_weight, planner._pos_lo, planner._pos_hi, planner._vel_lo,
        planner._vel_hi, planner._acc_lo, planner._acc_hi, p.w_env, p.w_self, p.w_q, p.w_qd,
        p.w_qdd, p.w_s, p.w_ns, p.d_act, p.q_ref, *_field_arguments(snap),
    ]
    return dict(zip(ROLLOUT_KEYS, vals))


def make_rollout() -> dict:
    d: dict[str, np.ndarray] = {}
    chain, model = load_robot(config.bundled_scenario_path("robot_7dof"))
    cases = []

    # (a) t/test_planner.py:304-335: 40x40x30 @1%, 5 samples, H=12, seed 17
    rng = np.random.default_rng(17)
    grid = VoxelGrid((-1.0, -1.0, 0.0), 0.05, (40, 40, 30))
    occ = rng.random((40, 40, 30)) < 0.01
    grid.log_odds[occ] = grid.params.l_max
    field = edt_3d(grid, outside_default=0.8)
    params = config.planner_params(7, {"samples": 5, "horizon": 12})
    goal = forward_kinematics(chain, np.full(7, 0.4))[-1]
    state = JointState(rng.normal(scale=0.3, size=7), rng.normal(scale=0.2, size=7), np.zeros(7))
    controls = rng.normal(scale=1.5, size=(5, 12, 7))
    cases.append(("kernel_vs_scalar", params, state, goal, field, controls, True, ("grid", (-1.0, -1.0, 0.0), 0.05, occ, None)))

    # (b) acceptance planner scene (t/test_acceptance.py:308-317), M=64, H=32,
    #     nominal 0.1, eps from the reference sampler (seed 3).  Robot starts
    #     in collision.
    grid = VoxelGrid((-1.5, -1.5, 0.0), 0.02, (150, 150, 25))
    occ = np.zeros((150, 150, 25), bool)
    occ[60:80, 60:80, 5:20] = True
    grid.log_odds[occ] = grid.params.l_max
    field = edt_3d(grid, outside_default=0.8)
    params = config.planner_params(7, {"samples": 64, "horizon": 32})
    goal = forward_kinematics(chain, np.full(7, 0.35))[-1]
    state = JointState.resting(np.full(7, 0.05))
    eps = sample_perturbations(params, 3)
    controls = np.full((32, 7), 0.1)[None] + eps
    cases.append(("acceptance_scene", params, state, goal, field, controls, False, ("grid", (-1.5, -1.5, 0.0), 0.02, occ, None)))

    # (c) reach_static board scene (vp/data/reach_static.yaml): collision-free
    #     start, board voxels, q_ref override, H=20 and H=32
    scen = config.load_scenario(config.bundled_scenario_path("reach_static"))
    gs = scen.grid_spec
    grid = VoxelGrid(gs.origin, gs.voxel_size, gs.dims)
    occ = np.zeros(gs.dims, bool)
    occ[29:31, 26:34, 28:40] = True  # board
    occ[:, :, 0:6] = True  # floor slab top
    grid.log_odds[occ] = grid.params.l_max
    field = edt_3d(grid, outside_default=0.8)
    for h in (20, 32):
        overrides = dict(scen.raw_config["planner"])
        overrides.update({"samples": 48, "horizon": h, "dt": 1.0 / scen.rate_hz})
        params = config.planner_params(7, overrides)
        state = JointState.resting(scen.start_q)
        eps = sample_perturbations(params, 11 + h)
        controls = eps + 0.2 * np.sin(np.arange(h))[None, :, None]
        cases.append((f"reach_static_H{h}", params, state, scen.goals[0], field, controls, h == 20,
                      ("grid", gs.origin, gs.voxel_size, occ, None)))

    # (d) no field (snap=None): far-away 1^3 inf field (vp/planner.py:429-441),
    #     H=64 (C4 shape, small M), moving state, random goal orientation
    params = config.planner_params(7, {"samples": 16, "horizon": 64})
    rng = np.random.default_rng(23)
    goal = forward_kinematics(chain, rng.uniform(-0.8, 0.8, size=7))[-1]
    state = JointState(rng.normal(scale=0.2, size=7), rng.normal(scale=0.5, size=7), np.zeros(7))
    controls = rng.normal(scale=3.0, size=(16, 64, 7))
    cases.append(("no_field_H64", params, state, goal, None, controls, False, None))

    # (e) degenerate rotation: goal at pi about x relative to the flange
    #     (t/test_planner.py:463-478), so flags must be raised.
    from voxplan.geometry import Rotation3

    ee = forward_kinematics(chain, np.zeros(7))[-1]
    goal = RigidTransform(ee.rotation @ Rotation3.rot_x(math.pi), ee.translation)
    params = config.planner_params(7, {"samples": 4, "horizon": 3, "sigma": 0.0})
    state = JointState.resting(np.zeros(7))
    controls = np.zeros((4, 3, 7))
    controls[1:] = rng.normal(scale=2.0, size=(3, 3, 7))
    cases.append(("degenerate_pi", params, state, goal, None, controls, False, None))

    for i, (name, params, state, goal, field, controls, store, gridspec) in enumerate(cases):
        planner = Planner(chain, model, params)
        args = pack_args(planner, state, goal, field)
        m, h, n = controls.shape
        costs = np.zeros(m)
        terms = np.zeros((m, 6))
        flags = np.zeros(m, np.uint8)
        tq = np.zeros((m, h + 1, n) if store else (1, 1, 1))
        tqd = np.zeros_like(tq)
        sp = np.zeros((m, h, model.count, 3) if store else (1, 1, 1, 3))
        from voxplan import batch

        vals = [args[k] for k in ROLLOUT_KEYS]
        batch.evaluate_batch(vals[0], vals[1], controls, *vals[2:], store, store, costs, terms, tq, tqd, sp, flags)
        d[f"r_name_{i}"] = np.array(name)
        for k in ROLLOUT_KEYS:
            if k == "field_sq":
                continue
            d[f"r_{k}_{i}"] = np.asarray(args[k])
        fsq = np.asarray(args["field_sq"])
        d[f"r_field_sq_{i}"] = sq_to_i32(fsq)
        d[f"r_field_shape_{i}"] = np.array(fsq.shape, np.int64)
        d[f"r_controls_{i}"] = controls
        d[f"r_costs_{i}"] = costs
        d[f"r_terms_{i}"] = terms
        d[f"r_flags_{i}"] = flags
        d[f"r_store_{i}"] = np.array(store)
        if store:
            d[f"r_trajq_{i}"] = tq
            d[f"r_trajqd_{i}"] = tqd
            d[f"r_sphpos_{i}"] = sp
        if gridspec is not None:
            d[f"r_grid_origin_{i}"] = np.asarray(gridspec[1], float)
            d[f"r_grid_voxel_{i}"] = np.array(gridspec[2])
            d[f"r_grid_occ_{i}"] = np.packbits(gridspec[3].reshape(-1))
            d[f"r_grid_dims_{i}"] = np.array(gridspec[3].shape, np.int64)
        # planner parameters for the host-side packing test
        d[f"r_params_{i}"] = np.array(
            [params.horizon, params.samples, params.dt, params.lam, params.noise_window,
             params.margin_frac]
        )
    d["r_count"] = np.array(len(cases))
    return d


# --------------------------------------------------------------------------
# Softmin / update / smpc_step
# --------------------------------------------------------------------------
def make_softmin() -> dict:
    d: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(5)
    cases = [
        (np.array([3.7]), 0.5),
        (np.full(8, 2.5), 0.5),
        (np.array([0.0, 0.8 * math.log(2.0)]), 0.8),
        (rng.uniform(0, 100, size=64), 0.5),
        (rng.integers(0, 2**16, size=32).astype(float) / 1024.0, 0.31),
        (rng.uniform(0.0, 64.0, size=512), 1e6),
        (rng.uniform(1e3, 1e5, size=4096), 0.05),
        (rng.uniform(10.0, 11.0, size=4096), 0.05),
        (rng.uniform(0.0, 3.0, size=1000), 0.05),
    ]
    for i, (c, lam) in enumerate(cases):
        d[f"s_costs_{i}"] = c
        d[f"s_lam_{i}"] = np.array(lam)
        w = soft_weights(c, lam)
        d[f"s_w_{i}"] = w
        h, n = (9, 3) if c.shape[0] <= 512 else (4, 2)
        nominal = rng.normal(size=(h, n))
        eps = rng.normal(size=(c.shape[0], h, n))
        d[f"s_nom_{i}"] = nominal
        d[f"s_eps_{i}"] = eps
        d[f"s_u_{i}"] = update_controls(nominal, eps, w)
    d["s_count"] = np.array(len(cases))

    # Full smpc_step on the acceptance scene with the reference eps
    chain, model = load_robot(config.bundled_scenario_path("robot_7dof"))
    grid = VoxelGrid((-1.0, -1.0, 0.0), 0.05, (30, 30, 30))
    grid.log_odds[12:16, 12:16, 10:14] = grid.params.l_max  # t/test_planner.py:432-451
    field = edt_3d(grid, outside_default=0.8)
    for j, (m, h, seed) in enumerate(((64, 12, 42), (256, 20, 0), (512, 32, 7))):
        params = config.planner_params(7, {"samples": m, "horizon": h})
        planner = Planner(chain, model, params)
        goal = forward_kinematics(chain, np.full(7, 0.35))[-1]
        state = JointState.resting(np.full(7, 0.1))
        nominal = np.zeros((h, 7)) if j != 2 else 0.3 * np.cos(np.arange(h * 7)).reshape(h, 7)
        res = planner.smpc_step(state, goal, field, nominal, rng_seed=seed)
        eps = sample_perturbations(params, seed)
        d[f"st_cfg_{j}"] = np.array([m, h, seed])
        d[f"st_nominal_{j}"] = nominal
        d[f"st_eps_{j}"] = eps
        d[f"st_command_{j}"] = res.command
        d[f"st_next_{j}"] = res.next_nominal
        dg = res.diagnostics
        d[f"st_diag_{j}"] = np.array([dg.best_cost, dg.weighted_cost, dg.e_pos, dg.e_ori,
                                      *[getattr(dg.breakdown, k) for k in
                                        ("pose", "collision", "limits", "smoothness", "nullspace", "terminal")]])
        args = pack_args(planner, state, goal, field)
        for k in ("q0", "qd0", "goal_r", "goal_t"):
            d[f"st_{k}_{j}"] = np.asarray(args[k])
    d["st_grid_occ"] = np.packbits(grid.occupied_mask().reshape(-1))
    d["st_count"] = np.array(3)
    return d


# --------------------------------------------------------------------------
# EDT acceptance criterion 1 (all 100 grids) and Planner.integrate
# --------------------------------------------------------------------------
def make_edt_acceptance() -> dict:
    """t/test_acceptance.py:57-81: 100 random 16^3 grids in the test's own RNG
    order (density ~ U(0.01, 0.5), then the occupancy draw)."""
    d: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(20240817)
    occs, sqs = [], []
    for _ in range(100):
        dims = (16, 16, 16)
        grid = VoxelGrid((0.0, 0.0, 0.0), 0.1, dims)
        density = rng.uniform(0.01, 0.5)
        occ = rng.random(dims) < density
        grid.log_odds[occ] = grid.params.l_max
        occs.append(np.packbits(occ.reshape(-1)))
        sqs.append(sq_to_i32(edt_3d(grid).sq))
    d["occ"] = np.stack(occs)
    d["sq"] = np.stack(sqs)
    return d


def make_integrate() -> dict:
    """Planner.integrate (vp/planner.py:632-636) on seeded states/commands."""
    chain, model = load_robot(config.bundled_scenario_path("robot_7dof"))
    rng = np.random.default_rng(632)
    d: dict[str, np.ndarray] = {}
    for j, dt_rate in enumerate((None, 100.0, 250.0)):
        over = {} if dt_rate is None else {"dt": 1.0 / dt_rate}
        params = config.planner_params(7, over)
        planner = Planner(chain, model, params)
        q, qd = rng.uniform(-1, 1, 7), rng.uniform(-0.5, 0.5, 7)
        state = JointState(q, qd, np.zeros(7))
        qs, qds, accs, cmds = [], [], [], []
        for _ in range(20):
            cmd = rng.uniform(-3, 3, 7)
            state = planner.integrate(state, cmd)
            cmds.append(cmd)
            qs.append(state.q)
            qds.append(state.qd)
            accs.append(state.qdd)
        d[f"i_dt_{j}"] = np.array(params.dt)
        d[f"i_q0_{j}"], d[f"i_qd0_{j}"] = q, qd
        d[f"i_cmd_{j}"], d[f"i_q_{j}"] = np.array(cmds), np.array(qs)
        d[f"i_qd_{j}"], d[f"i_qdd_{j}"] = np.array(qds), np.array(accs)
    d["i_count"] = np.array(3)
    return d


def main():
    only = set(sys.argv[1].split(",")) if len(sys.argv) > 1 else None
    for name, fn in (("edt", make_edt), ("fusion", make_fusion), ("query", make_query),
                     ("rollout", make_rollout), ("softmin", make_softmin),
                     ("edt_acceptance", make_edt_acceptance), ("integrate", make_integrate)):
        if only is not None and name not in only:
            continue
        data = fn()
        path = OUT / f"{name}.npz"
        np.savez_compressed(path, **data)
        print(f"wrote {path} ({path.stat().st_size / 1024:.0f} KiB, {len(data)} arrays)")


if __name__ == "__main__":
    main()
