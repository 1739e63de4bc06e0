"""GPU parity of the SMPC kernels (rollout/cost, softmin, update, smpc_step).

Bars (BASELINE.json north_star):
  * fp64 parity mode vs the reference golden vectors: rtol 1e-9 (the
    reference's own batch-vs-scalar bar, t/test_planner.py:304-335);
  * fp32 production mode: costs and the six terms within 1e-4 relative
    (absolute floor 1e-4 * (1 + total cost) per sample for terms that are
    tiny next to the total); weights |dw| <= 1e-4 * max w; U* within 1e-4
    relative (floor 1e-6).
The reference's own seeded noise (stored in the golden files) is fed to both
sides.
"""

import math

import numpy as np
import pytest

import oracle
from conftest import i32_to_sq, load_golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

KEYS = (
    "q0 qd0 dt base_r base_t off_r off_t axes sph_link sph_loc sph_r pairs goal_r goal_t "
    "pose_weight terminal_weight pos_lo pos_hi vel_lo vel_hi acc_lo acc_hi w_env w_self w_q "
    "w_qd w_qdd w_s w_ns d_act q_ref field_sq field_lo0 field_lo1 field_lo2 field_origin0 "
    "field_origin1 field_origin2 field_voxel field_outside"
).split()


@pytest.fixture(scope="module")
def pk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_22575_b200 as pkg
    from paper_2512_22575_b200 import config, mapping, planner, robot

    return pkg, config, mapping, planner, robot


def _setup(pk, g, i, precision):
    """Build Planner/state/goal/field for golden rollout case i from the
    stored packed arguments (same robot, same objective)."""
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200.geometry import RigidTransform, Rotation3

    chain, model = config.robot_7dof()
    prm = g[f"r_params_{i}"]
    h, m, dt, lam, win, margin = prm
    overrides = {"horizon": int(h), "samples": int(m), "dt": float(dt), "lam": float(lam),
                 "noise_window": int(win), "margin_frac": float(margin), "q_ref": g[f"r_q_ref_{i}"],
                 "pose_weight": g[f"r_pose_weight_{i}"], "terminal_weight": g[f"r_terminal_weight_{i}"]}
    params = config.planner_params(7, overrides)
    pl = planner.Planner(chain, model, params, precision=precision)
    P = planner.pack_problem(chain, model, params)
    for k in ("pos_lo", "pos_hi", "vel_lo", "vel_hi", "acc_lo", "acc_hi"):
        np.testing.assert_array_equal(np.array(getattr(P, k)[:7]), g[f"r_{k}_{i}"])
    state = robot.JointState(g[f"r_q0_{i}"], g[f"r_qd0_{i}"], np.zeros(7))
    goal = RigidTransform(Rotation3(g[f"r_goal_r_{i}"]), g[f"r_goal_t_{i}"])
    field = None
    if f"r_grid_occ_{i}" in g:
        sq = i32_to_sq(g[f"r_field_sq_{i}"])
        shape = tuple(int(v) for v in g[f"r_field_shape_{i}"])
        box = mapping.VoxelBox((0, 0, 0), shape)
        field = mapping.DistanceField(g[f"r_grid_origin_{i}"], float(g[f"r_grid_voxel_{i}"]), shape, box,
                                      torch.from_numpy(sq.astype(np.float32)).cuda(), float(g[f"r_field_outside_{i}"]))
    return pl, state, goal, field


def test_rollout_fp64_vs_golden(pk):
    g = load_golden("rollout")
    from paper_2512_22575_b200.errors import DegenerateRotation

    for i in range(int(g["r_count"])):
        name = str(g[f"r_name_{i}"])
        pl, state, goal, field = _setup(pk, g, i, "fp64")
        store = bool(g[f"r_store_{i}"])
        ctrl = g[f"r_controls_{i}"]
        flags = g[f"r_flags_{i}"]
        if flags.any():
            with pytest.raises(DegenerateRotation):
                pl.evaluate(state, goal, field, ctrl)
            costs, terms, fl, *_ = pl.evaluate_device(state, goal, field, torch.from_numpy(ctrl).cuda())
            np.testing.assert_array_equal(fl.cpu().numpy(), flags, err_msg=name)
            continue
        res = pl.evaluate(state, goal, field, ctrl, keep_trajectories=store, keep_spheres=store)
        np.testing.assert_allclose(res.costs, g[f"r_costs_{i}"], rtol=1e-9, err_msg=name)
        np.testing.assert_allclose(res.terms, g[f"r_terms_{i}"], rtol=1e-9, atol=1e-9, err_msg=name)
        if store:
            np.testing.assert_allclose(res.traj_q, g[f"r_trajq_{i}"], rtol=1e-12, atol=1e-12, err_msg=name)
            np.testing.assert_allclose(res.traj_qd, g[f"r_trajqd_{i}"], rtol=1e-12, atol=1e-12, err_msg=name)
            np.testing.assert_allclose(res.sphere_positions, g[f"r_sphpos_{i}"], rtol=1e-11, atol=1e-12)


def _fp32_close(got_costs, got_terms, want_costs, want_terms, name):
    """costs: rtol 1e-4; each term: 1e-4 relative or 1e-6 of (1 + the
    sample's total cost) absolute (terms that vanish next to the total)."""
    np.testing.assert_allclose(got_costs, want_costs, rtol=1e-4, err_msg=name)
    err = np.abs(got_terms - want_terms)
    bound = 1e-4 * np.abs(want_terms) + 1e-6 * (1.0 + np.abs(want_costs))[:, None]
    bad = err > bound
    assert not bad.any(), f"{name}: fp32 terms off at {np.argwhere(bad)[:5]}: {got_terms[bad][:5]} vs {want_terms[bad][:5]}"


def test_rollout_fp32_vs_golden(pk):
    g = load_golden("rollout")
    for i in range(int(g["r_count"])):
        name = str(g[f"r_name_{i}"])
        if g[f"r_flags_{i}"].any():
            continue
        pl, state, goal, field = _setup(pk, g, i, "fp32")
        res = pl.evaluate(state, goal, field, g[f"r_controls_{i}"])
        _fp32_close(res.costs, res.terms, g[f"r_costs_{i}"], g[f"r_terms_{i}"], name)


def test_rollout_fp32_large_batch_vs_oracle(pk):
    """C3 shape (M=4096, H=32) on the collision-free board scene against the
    oracle (fp64 C restatement) on the same inputs."""
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200 import scene
    from paper_2512_22575_b200.geometry import RigidTransform

    chain, model = config.robot_7dof()
    origin, voxel, occ = scene.reach_static_occupancy()
    grid = mapping.VoxelGrid(origin, voxel, occ.shape)
    grid.set_log_odds(np.where(occ, 3.5, 0.0))
    field = mapping.edt_3d(grid, outside_default=0.8)
    params = config.planner_params(7, {"samples": 4096, "horizon": 32, "q_ref": scene.REACH_STATIC_QREF})
    state = robot.JointState.resting(scene.REACH_STATIC_START)
    goal = RigidTransform.from_vec7(scene.REACH_STATIC_GOAL)
    rng = np.random.default_rng(77)
    ctrl = rng.normal(scale=1.5, size=(4096, 32, 7))
    res = planner.Planner(chain, model, params, "fp32").evaluate(state, goal, field, ctrl)
    args = _oracle_args(planner, chain, model, params, state, goal, field)
    want = oracle.evaluate_batch(args, ctrl)
    _fp32_close(res.costs, res.terms, want["costs"], want["terms"], "reach_static M=4096")
    res64 = planner.Planner(chain, model, params, "fp64").evaluate(state, goal, field, ctrl)
    np.testing.assert_allclose(res64.costs, want["costs"], rtol=1e-9)


def _oracle_args(planner, chain, model, params, state, goal, field):
    P = planner.pack_problem(chain, model, params)
    lims = planner.tightened_limits(chain, params.margin_frac)
    args = {
        "q0": state.q, "qd0": state.qd, "dt": params.dt, "base_r": chain.base_pose.rotation.matrix,
        "base_t": chain.base_pose.translation,
        "off_r": np.array([j.parent_offset.rotation.matrix for j in chain.joints]),
        "off_t": np.array([j.parent_offset.translation for j in chain.joints]),
        "axes": np.array([j.axis for j in chain.joints]),
        "sph_link": np.array([s.link for s in model.spheres]), "sph_loc": np.array([s.center for s in model.spheres]),
        "sph_r": model.radii(), "pairs": np.array(model.self_pairs), "goal_r": goal.rotation.matrix,
        "goal_t": goal.translation, "pose_weight": params.pose_weight, "terminal_weight": params.terminal_weight,
        "w_env": params.w_env, "w_self": params.w_self, "w_q": params.w_q, "w_qd": params.w_qd,
        "w_qdd": params.w_qdd, "w_s": params.w_s, "w_ns": params.w_ns, "d_act": params.d_act, "q_ref": params.q_ref,
    }
    for k, v in zip(("pos_lo", "pos_hi", "vel_lo", "vel_hi", "acc_lo", "acc_hi"), lims):
        args[k] = v
    del P
    if field is None:
        args.update(field_sq=np.full((1, 1, 1), np.inf), field_lo0=2**40, field_lo1=2**40, field_lo2=2**40,
                    field_origin0=0.0, field_origin1=0.0, field_origin2=0.0, field_voxel=1.0, field_outside=np.inf)
    else:
        args.update(field_sq=field.sq, field_lo0=field.volume.lo[0], field_lo1=field.volume.lo[1],
                    field_lo2=field.volume.lo[2], field_origin0=field.origin[0], field_origin1=field.origin[1],
                    field_origin2=field.origin[2], field_voxel=field.voxel_size, field_outside=field.outside_default)
    return args


def test_softmin_update_vs_golden(pk):
    pkg, config, mapping, planner, robot = pk
    g = load_golden("softmin")
    for i in range(int(g["s_count"])):
        w = planner.soft_weights(g[f"s_costs_{i}"], float(g[f"s_lam_{i}"]))
        np.testing.assert_allclose(w, g[f"s_w_{i}"], rtol=1e-12, atol=1e-300)
        u = planner.update_controls(g[f"s_nom_{i}"], g[f"s_eps_{i}"], g[f"s_w_{i}"])
        np.testing.assert_allclose(u, g[f"s_u_{i}"], rtol=1e-12, atol=1e-13)


def test_softmin_errors(pk):
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200.errors import WeightMismatch

    with pytest.raises(ValueError):
        planner.soft_weights(np.array([]), 0.5)
    with pytest.raises(ValueError):
        planner.soft_weights(np.array([1.0, np.inf]), 0.5)
    with pytest.raises(ValueError):
        planner.soft_weights(np.array([1.0]), 0.0)
    with pytest.raises(WeightMismatch):
        planner.update_controls(np.zeros((1, 1)), np.zeros((2, 1, 1)), np.array([0.6, 0.6]))
    # dyadic shift invariance holds bitwise (t/test_planner.py:369-377)
    rng = np.random.default_rng(7)
    costs = rng.integers(0, 2**16, size=32).astype(float) / 1024.0
    a = planner.soft_weights(costs, 0.31)
    for shift in (1.0, 64.0, -17.5):
        np.testing.assert_array_equal(planner.soft_weights(costs + shift, 0.31), a)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_smpc_step_vs_golden(pk, precision):
    """Full smpc_step with the reference's noise (golden st_*)."""
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200.geometry import RigidTransform, Rotation3
    from conftest import unpack_occ

    g = load_golden("softmin")
    chain, model = config.robot_7dof()
    occ = unpack_occ(g["st_grid_occ"], (30, 30, 30))
    grid = mapping.VoxelGrid((-1.0, -1.0, 0.0), 0.05, (30, 30, 30))
    grid.set_log_odds(np.where(occ, 3.5, 0.0))
    field = mapping.edt_3d(grid, outside_default=0.8)
    for j in range(int(g["st_count"])):
        m, h, seed = (int(v) for v in g[f"st_cfg_{j}"])
        params = config.planner_params(7, {"samples": m, "horizon": h})
        pl = planner.Planner(chain, model, params, precision=precision)
        state = robot.JointState(g[f"st_q0_{j}"], g[f"st_qd0_{j}"], np.zeros(7))
        goal = RigidTransform(Rotation3(g[f"st_goal_r_{j}"]), g[f"st_goal_t_{j}"])
        res = pl.smpc_step(state, goal, field, g[f"st_nominal_{j}"], seed, perturbations=g[f"st_eps_{j}"])
        diag = g[f"st_diag_{j}"]
        tol = 1e-9 if precision == "fp64" else 1e-4
        floor = 1e-12 if precision == "fp64" else 1e-6
        np.testing.assert_allclose(res.command, g[f"st_command_{j}"], rtol=tol, atol=floor)
        np.testing.assert_allclose(res.next_nominal, g[f"st_next_{j}"], rtol=tol, atol=floor)
        np.testing.assert_allclose(res.diagnostics.best_cost, diag[0], rtol=tol)
        np.testing.assert_allclose(res.diagnostics.weighted_cost, diag[1], rtol=tol)
        np.testing.assert_allclose(res.diagnostics.e_pos, diag[2], rtol=1e-12)
        np.testing.assert_allclose(res.diagnostics.e_ori, diag[3], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("samples,generic", [(4096, "0"), (16384, "0"), (3000, "1")])
def test_all_nonzero_weights_step_equals_explicit_update(pk, samples, generic, monkeypatch):
    """Every weight nonzero (lam = 1e4): the fused step's U* (helper-CTA N
    reduction) equals soft_weights + update_controls on the same costs, for
    the one-launch step and for repeated native-session steps (per-launch
    epochs of the helper protocol)."""
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200.geometry import RigidTransform

    # generic = "1": the runtime-topology kernel (8 candidates per CTA) takes the heavy merge too
    monkeypatch.setenv("VPB_GENERIC_ROLLOUT", generic)
    chain, model = config.robot_7dof()
    params = config.planner_params(7, {"samples": samples, "horizon": 32, "lam": 1e4})
    pl = planner.Planner(chain, model, params, "fp32")
    state = robot.JointState.resting(np.full(7, 0.1))
    goal = RigidTransform.from_vec7([0.3, -0.2, 0.7, 0.9, 0.1, 0.3, -0.2])
    nom = torch.from_numpy(0.1 * np.sin(np.arange(224)).reshape(32, 7)).cuda()
    for seed in (3, 4):
        out, eps = pl.smpc_generate_device(state, goal, None, nom, seed)
        costs = torch.empty(samples, dtype=torch.float64, device="cuda")
        pl.smpc_step_device(state, goal, None, nom, eps, costs=costs)
        w = planner.soft_weights(costs, params.lam)
        assert int((w > 0).sum()) == samples
        u = planner.update_controls(nom, eps.double(), w)
        np.testing.assert_allclose(out[:224].cpu().numpy(), u.cpu().numpy().reshape(-1), rtol=1e-10, atol=1e-12)
        res = pl.smpc_step(state, goal, None, nom.cpu().numpy(), seed)
        np.testing.assert_allclose(res.next_nominal.reshape(-1)[:217], out[231:448].cpu().numpy(), rtol=1e-10,
                                   atol=1e-12)


def test_finish_single_weight_shortcut_equals_reevaluation(pk):
    """With one nonzero softmin weight over all ranks (tiny lambda) the
    multi-device finish reuses that candidate's sums from its rank record
    instead of re-evaluating U*; clearing the record's nonzero count forces
    the re-evaluation, and both agree (vp/planner.py:373-400)."""
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200.geometry import RigidTransform

    chain, model = config.robot_7dof()
    params = config.planner_params(7, {"samples": 1024, "horizon": 20, "lam": 1e-6})
    pl = planner.Planner(chain, model, params, "fp32")
    state = robot.JointState.resting(np.full(7, 0.1))
    goal = RigidTransform.from_vec7([0.3, -0.2, 0.7, 0.9, 0.1, 0.3, -0.2])
    nom = torch.from_numpy(0.1 * np.sin(np.arange(140)).reshape(20, 7)).cuda()
    eps = pl.sample_device(5)
    hn = 140
    parts = []
    for r in range(4):
        p, _, _ = pl.smpc_partial_device(state, goal, None, nom, eps[r * 256:(r + 1) * 256].contiguous(),
                                          m_offset=r * 256)
        parts.append(p)
    parts = torch.stack(parts)
    assert int((parts[:, 4 + hn] == 1).sum()) >= 1
    fast = pl.smpc_finish_device(state, goal, None, nom, parts).cpu().numpy()
    slow_parts = parts.clone()
    slow_parts[:, 4 + hn] = -1.0
    slow = pl.smpc_finish_device(state, goal, None, nom, slow_parts).cpu().numpy()
    np.testing.assert_array_equal(fast[:2 * hn + 7], slow[:2 * hn + 7])
    np.testing.assert_allclose(fast, slow, rtol=1e-6, atol=1e-9, equal_nan=True)
    single = pl.smpc_step_device(state, goal, None, nom, eps).cpu().numpy()
    np.testing.assert_allclose(fast, single, rtol=1e-12, atol=1e-14, equal_nan=True)


@pytest.mark.parametrize("lam", [None, 1e4])
def test_smpc_shard_merge_equals_single(pk, lam):
    """Sharded partials (2 and 8 shards of one batch) merged in rank order
    equal the single-device step.  lam = 1e4 makes every
    weight nonzero: the N reduction then runs on the helper CTAs."""
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200.geometry import RigidTransform

    chain, model = config.robot_7dof()
    over = {"samples": 1024, "horizon": 20}
    if lam is not None:
        over["lam"] = lam
    params = config.planner_params(7, over)
    pl = planner.Planner(chain, model, params, "fp32")
    state = robot.JointState.resting(np.full(7, 0.1))
    goal = RigidTransform.from_vec7([0.3, -0.2, 0.7, 0.9, 0.1, 0.3, -0.2])
    nom = torch.zeros((20, 7), dtype=torch.float64, device="cuda")
    eps = pl.sample_device(123)
    part1, costs, _ = pl.smpc_partial_device(state, goal, None, nom, eps)
    single = pl.smpc_finish_device(state, goal, None, nom, part1.reshape(1, -1)).cpu().numpy()
    for shards in (2, 8):
        parts = []
        step = 1024 // shards
        for r in range(shards):
            p, c, _ = pl.smpc_partial_device(state, goal, None, nom, eps[r * step:(r + 1) * step].contiguous(),
                                              m_offset=r * step)
            torch.testing.assert_close(c, costs[r * step:(r + 1) * step], rtol=0, atol=0)
            parts.append(p)
        merged = pl.smpc_finish_device(state, goal, None, nom, torch.stack(parts)).cpu().numpy()
        np.testing.assert_allclose(merged, single, rtol=1e-12, atol=1e-14)
    # and the merged U* equals the explicit softmin + weighted mean on the same costs
    w = planner.soft_weights(costs, params.lam)
    u = planner.update_controls(nom, eps.double(), w)
    np.testing.assert_allclose(single[:140], u.cpu().numpy().reshape(-1), rtol=1e-10, atol=1e-12)


def test_degenerate_rotation_raises(pk):
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200.errors import DegenerateRotation
    from paper_2512_22575_b200.geometry import RigidTransform, Rotation3

    chain, model = config.robot_7dof()
    ee = robot.forward_kinematics(chain, np.zeros(7))[-1]
    goal = RigidTransform(ee.rotation @ Rotation3.rot_x(math.pi), ee.translation)
    params = config.planner_params(7, {"samples": 8, "horizon": 3, "sigma": 0.0})
    for prec in ("fp32", "fp64"):
        pl = planner.Planner(chain, model, params, prec)
        with pytest.raises(DegenerateRotation):
            pl.smpc_step(robot.JointState.resting(np.zeros(7)), goal, None, None, 0)


def test_sampler_statistics(pk):
    """Statistical parity with the reference sampler (t/test_planner.py:52-90)."""
    pkg, config, mapping, planner, robot = pk
    chain, model = config.robot_7dof()
    params = config.planner_params(7, {"samples": 32, "horizon": 10})
    eps = planner.sample_perturbations(params, 9).cpu().numpy()
    np.testing.assert_array_equal(eps[0], 0.0)
    assert np.abs(eps[1:]).max() > 0
    a = planner.sample_perturbations(params, 1).cpu().numpy()
    b = planner.sample_perturbations(params, 1).cpu().numpy()
    c = planner.sample_perturbations(params, 2).cpu().numpy()
    np.testing.assert_array_equal(a, b)
    assert np.abs(a - c).max() > 0
    # mean within 4 sigma / sqrt(M); smoothing preserves the variance (5%)
    p2 = config.planner_params(7, {"samples": 100_000, "horizon": 2, "sigma": 2.0})
    e2 = planner.sample_perturbations(p2, 123).cpu().numpy()
    assert np.abs(e2.mean(axis=0)).max() < 4.0 * 2.0 / math.sqrt(100_000)
    p3 = config.planner_params(7, {"samples": 20_000, "horizon": 12, "sigma": 1.5, "noise_window": 5})
    e3 = planner.sample_perturbations(p3, 7).cpu().numpy()
    np.testing.assert_allclose(e3[1:].std(axis=0), 1.5, rtol=0.05)
    p4 = config.planner_params(7, {"samples": 16, "horizon": 8, "sigma": 0.0})
    np.testing.assert_array_equal(planner.sample_perturbations(p4, 4).cpu().numpy(), 0.0)
    # shard offsets reproduce the same global stream
    pl = planner.Planner(chain, model, params, "fp64")
    full = pl.sample_device(5)
    half = pl.sample_device(5, m_offset=16, samples=16)
    torch.testing.assert_close(full[16:], half, rtol=0, atol=0)


def test_fixed_point_at_goal(pk):
    """t/test_planner.py:420-430 on the 7-DoF arm: zero noise at the goal
    keeps the command at zero."""
    pkg, config, mapping, planner, robot = pk
    chain, model = config.robot_7dof()
    q = np.full(7, 0.4)
    goal = robot.forward_kinematics(chain, q)[-1]
    params = config.planner_params(7, {"sigma": 0.0, "samples": 16, "horizon": 10, "q_ref": q})
    for prec in ("fp64", "fp32"):
        res = planner.Planner(chain, model, params, prec).smpc_step(robot.JointState.resting(q), goal, None, None, 0)
        np.testing.assert_allclose(res.command, 0.0, atol=1e-9)
        np.testing.assert_allclose(res.next_nominal, 0.0, atol=1e-9)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_fused_step_equals_partial_finish_and_graph(pk, precision):
    """The one-launch SMPC step, the partial + finish path and the CUDA-graph
    replay (per-call state from device memory) give the same step."""
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200.geometry import RigidTransform

    chain, model = config.robot_7dof()
    grid = mapping.VoxelGrid((-1.0, -1.0, 0.0), 0.05, (30, 30, 30))
    occ = np.zeros((30, 30, 30), bool)
    occ[12:16, 12:16, 10:14] = True
    grid.set_log_odds(np.where(occ, 3.5, 0.0))
    field = mapping.edt_3d(grid, outside_default=0.8)
    for m, h in ((1000, 20), (4096, 32), (300, 64)):
        params = config.planner_params(7, {"samples": m, "horizon": h})
        pl = planner.Planner(chain, model, params, precision)
        state = robot.JointState(np.full(7, 0.1), np.linspace(-0.2, 0.2, 7), np.zeros(7))
        goal = RigidTransform.from_vec7([0.3, -0.2, 0.7, 0.9, 0.1, 0.3, -0.2])
        nom = torch.from_numpy(0.2 * np.cos(np.arange(h * 7)).reshape(h, 7)).cuda()
        eps = pl.sample_device(99)
        fused = pl.smpc_step_device(state, goal, field, nom, eps).cpu().numpy()
        part, _, _ = pl.smpc_partial_device(state, goal, field, nom, eps)
        split = pl.smpc_finish_device(state, goal, field, nom, part.reshape(1, -1)).cpu().numpy()
        np.testing.assert_allclose(fused, split, rtol=1e-12, atol=1e-14)
        g = planner.SmpcGraph(pl, field)
        res = g.step(state, goal, nom.cpu().numpy(), 99)
        direct = pl.smpc_step(state, goal, field, nom.cpu().numpy(), 99)
        np.testing.assert_array_equal(res.command, direct.command)
        np.testing.assert_array_equal(res.next_nominal, direct.next_nominal)
        assert res.diagnostics.weighted_cost == direct.diagnostics.weighted_cost
        # a second replay with a new state/seed follows the staged inputs
        state2 = robot.JointState.resting(np.full(7, -0.2))
        res2 = g.step(state2, goal, None, 7)
        direct2 = pl.smpc_step(state2, goal, field, None, 7)
        np.testing.assert_array_equal(res2.command, direct2.command)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_fixed_topology_equals_generic(pk, precision, monkeypatch):
    """The compile-time-topology kernels (robot_7dof) and the runtime-topology
    kernels agree on costs, terms, flags and the fused SMPC step, on a field
    with obstacles near the arm (collision + self terms active) and on the
    collision-free board scene, H below, at and above one warp."""
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200 import scene
    from paper_2512_22575_b200.geometry import RigidTransform

    chain, model = config.robot_7dof()
    grid = mapping.VoxelGrid((-0.8, -0.8, 0.0), 0.04, (40, 40, 32))
    occ = np.zeros((40, 40, 32), bool)
    occ[22:26, 18:24, 8:20] = True
    occ[10:13, 25:28, 14:16] = True
    grid.set_log_odds(np.where(occ, 3.5, 0.0))
    near = mapping.edt_3d(grid, outside_default=0.8)
    origin, voxel, bocc = scene.reach_static_occupancy()
    g2 = mapping.VoxelGrid(origin, voxel, bocc.shape)
    g2.set_log_odds(np.where(bocc, 3.5, 0.0))
    board = mapping.edt_3d(g2, outside_default=0.8)
    rtol = 1e-4 if precision == "fp32" else 1e-11
    for field, (m, h) in ((near, (517, 20)), (board, (1024, 32)), (near, (300, 45)), (None, (64, 7))):
        params = config.planner_params(7, {"samples": m, "horizon": h})
        pl = planner.Planner(chain, model, params, precision)
        state = robot.JointState(np.linspace(-0.6, 0.8, 7), np.linspace(-0.3, 0.3, 7), np.zeros(7))
        goal = RigidTransform.from_vec7([0.35, -0.25, 0.6, 0.9, 0.1, 0.3, -0.2])
        nom = torch.from_numpy(0.3 * np.sin(np.arange(h * 7)).reshape(h, 7)).cuda()
        eps = pl.sample_device(5) * 3.0
        out = {}
        for mode in ("0", "1"):
            monkeypatch.setenv("VPB_GENERIC_ROLLOUT", mode)
            c, t, f, *_ = pl.evaluate_device(state, goal, field, eps, nom)
            step = pl.smpc_step_device(state, goal, field, nom, eps)
            out[mode] = (c.cpu().numpy(), t.cpu().numpy(), f.cpu().numpy(), step.cpu().numpy())
        (c0, t0, f0, s0), (c1, t1, f1, s1) = out["0"], out["1"]
        np.testing.assert_array_equal(f0, f1)
        ok = f1 == 0
        assert ok.sum() > m // 2
        if precision == "fp32":
            _fp32_close(c0[ok], t0[ok], c1[ok], t1[ok], f"fixed vs generic m={m} h={h}")
        else:
            np.testing.assert_allclose(c0[ok], c1[ok], rtol=rtol)
            np.testing.assert_allclose(t0[ok], t1[ok], rtol=rtol, atol=1e-12)
        if field is near:
            assert (t1[ok, 1] > 0).mean() > 0.05, "collision term inactive: the test would not cover it"
        hn = h * 7
        base = 2 * hn + 7
        assert s0[base + 10] == s1[base + 10]  # best sample index
        np.testing.assert_allclose(s0[base + 7], s1[base + 7], rtol=rtol)  # best cost
        if precision == "fp64":  # fp32 weights at lam = 0.05 amplify 1e-6 cost noise; fp64 compares U*
            np.testing.assert_allclose(s0[:base + 11], s1[:base + 11], rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("precision,horizon", [("fp32", 24), ("fp64", 24), ("fp32", 48)])
def test_native_session_equals_device_step(pk, precision, horizon):
    """vpb_smpc_session (one host call: staged block, captured graph of
    sampler + fused step, host diagnostics) returns exactly the device step
    on the same seed, follows a field rebuilt into a new buffer, and fills
    e_pos / e_ori like the reference (vp/planner.py:620-629).  H = 48 puts
    H n past the launch-parameter nominal (the session's staged-block path)."""
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200.geometry import RigidTransform, quaternion_angle

    chain, model = config.robot_7dof()
    grid = mapping.VoxelGrid((-1.0, -1.0, 0.0), 0.05, (30, 30, 30))
    occ = np.zeros((30, 30, 30), bool)
    occ[12:16, 12:16, 10:14] = True
    grid.set_log_odds(np.where(occ, 3.5, 0.0))
    f1 = mapping.edt_3d(grid, outside_default=0.8)
    occ[5:8, 20:24, 12:18] = True
    grid.set_log_odds(np.where(occ, 3.5, 0.0))
    f2 = mapping.edt_3d(grid, outside_default=0.8)
    assert f1.sq_device.data_ptr() != f2.sq_device.data_ptr()
    params = config.planner_params(7, {"samples": 700, "horizon": horizon})
    pl = planner.Planner(chain, model, params, precision)
    state = robot.JointState(np.full(7, 0.1), np.linspace(-0.2, 0.2, 7), np.zeros(7))
    goal = RigidTransform.from_vec7([0.3, -0.2, 0.7, 0.9, 0.1, 0.3, -0.2])
    nom = 0.2 * np.cos(np.arange(horizon * 7)).reshape(horizon, 7)
    for field, seed in ((f1, 5), (f2, 6), (f1, 7)):
        res = pl.smpc_step(state, goal, field, nom, seed)  # native session
        eps = pl.sample_device(seed)
        out = pl.smpc_step_device(state, goal, field, torch.from_numpy(nom).cuda(), eps).cpu().numpy()
        ref = pl.unpack_step(out, state, goal, horizon)
        np.testing.assert_array_equal(res.command, ref.command)
        np.testing.assert_array_equal(res.next_nominal, ref.next_nominal)
        assert res.diagnostics.weighted_cost == ref.diagnostics.weighted_cost
        assert res.diagnostics.best_cost == ref.diagnostics.best_cost
        ee = robot.forward_kinematics(chain, state.q)[-1]
        np.testing.assert_allclose(res.diagnostics.e_pos, np.linalg.norm(ee.translation - goal.translation),
                                   rtol=1e-12)
        np.testing.assert_allclose(res.diagnostics.e_ori, quaternion_angle(ee.rotation.to_quaternion(),
                                                                           goal.rotation.to_quaternion()),
                                   rtol=1e-9, atol=1e-12)
    assert len(pl._sessions) == 1  # one session serves both field buffers


@pytest.mark.parametrize("precision,window", [("fp32", 5), ("fp32", 7), ("fp64", 5)])
def test_generate_equals_sampler_plus_step(pk, precision, window):
    """vpb_smpc_generate (draws inside the fused step kernel for the compiled
    topology in fp32, window <= 5; sampler + step otherwise) gives the same
    perturbations as sample_device and the same step / shard partial."""
    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200.geometry import RigidTransform

    chain, model = config.robot_7dof()
    grid = mapping.VoxelGrid((-1.0, -1.0, 0.0), 0.05, (30, 30, 30))
    occ = np.zeros((30, 30, 30), bool)
    occ[12:16, 12:16, 10:14] = True
    grid.set_log_odds(np.where(occ, 3.5, 0.0))
    field = mapping.edt_3d(grid, outside_default=0.8)
    for m, h in ((1000, 20), (4096, 32), (300, 70)):
        params = config.planner_params(7, {"samples": m, "horizon": h, "noise_window": window})
        pl = planner.Planner(chain, model, params, precision)
        state = robot.JointState(np.full(7, 0.1), np.linspace(-0.2, 0.2, 7), np.zeros(7))
        goal = RigidTransform.from_vec7([0.3, -0.2, 0.7, 0.9, 0.1, 0.3, -0.2])
        nom = torch.from_numpy(0.2 * np.cos(np.arange(h * 7)).reshape(h, 7)).cuda()
        out, eps = pl.smpc_generate_device(state, goal, field, nom, 41)
        ref_eps = pl.sample_device(41)
        torch.testing.assert_close(eps, ref_eps, rtol=0, atol=0)
        ref = pl.smpc_step_device(state, goal, field, nom, ref_eps)
        torch.testing.assert_close(out, ref, rtol=0, atol=0, equal_nan=True)
        part, _ = pl.smpc_generate_device(state, goal, field, nom, 41, m_offset=64, partial=True)
        ref_part, _, _ = pl.smpc_partial_device(state, goal, field, nom, pl.sample_device(41, m_offset=64),
                                                m_offset=64)
        torch.testing.assert_close(part, ref_part, rtol=0, atol=0)


def test_sharded_graph_nccl_world1_equals_step(pk):
    """The per-rank CUDA graph of the sharded step (fused draw + shard partial,
    NCCL all-gather captured in the graph, rank-order merge + tail) on a
    one-rank NCCL group gives the single-device step."""
    import os
    import socket

    import torch.distributed as dist

    pkg, config, mapping, planner, robot = pk
    from paper_2512_22575_b200 import distributed
    from paper_2512_22575_b200.geometry import RigidTransform

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        chain, model = config.robot_7dof()
        grid = mapping.VoxelGrid((-1.0, -1.0, 0.0), 0.05, (30, 30, 30))
        occ = np.zeros((30, 30, 30), bool)
        occ[12:16, 12:16, 10:14] = True
        grid.set_log_odds(np.where(occ, 3.5, 0.0))
        field = mapping.edt_3d(grid, outside_default=0.8)
        params = config.planner_params(7, {"samples": 2048, "horizon": 32})
        pl = planner.Planner(chain, model, params, "fp32")
        sh = distributed.ShardedSMPC(pl, world=1, rank=0)
        g = distributed.ShardedGraph(sh, field)
        state = robot.JointState(np.full(7, 0.1), np.linspace(-0.2, 0.2, 7), np.zeros(7))
        goal = RigidTransform.from_vec7([0.3, -0.2, 0.7, 0.9, 0.1, 0.3, -0.2])
        nom = 0.2 * np.cos(np.arange(32 * 7)).reshape(32, 7)
        for seed in (3, 4):
            got = g.step(state, goal, nom, seed)
            want = pl.smpc_step(state, goal, field, nom, seed)
            np.testing.assert_allclose(got.command, want.command, rtol=1e-12, atol=1e-14)
            np.testing.assert_allclose(got.next_nominal, want.next_nominal, rtol=1e-12, atol=1e-14)
            np.testing.assert_allclose(got.diagnostics.best_cost, want.diagnostics.best_cost, rtol=1e-12)
            np.testing.assert_allclose(got.diagnostics.weighted_cost, want.diagnostics.weighted_cost, rtol=1e-12)
    finally:
        dist.destroy_process_group()


def test_integrate_matches_reference_golden(pk):
    """Planner.integrate (vp/planner.py:632-636) against the reference's own
    outputs (tests/golden/integrate.npz): bitwise, the same two fp64
    multiply-adds in the same order."""
    pkg, config, mapping, planner, robot = pk
    g = load_golden("integrate")
    chain, model = config.robot_7dof()
    for j in range(int(g["i_count"])):
        params = config.planner_params(7, {"dt": float(g[f"i_dt_{j}"])})
        pl = planner.Planner(chain, model, params)
        state = robot.JointState(g[f"i_q0_{j}"], g[f"i_qd0_{j}"], np.zeros(7))
        for k, cmd in enumerate(g[f"i_cmd_{j}"]):
            state = pl.integrate(state, cmd)
            np.testing.assert_array_equal(state.q, g[f"i_q_{j}"][k])
            np.testing.assert_array_equal(state.qd, g[f"i_qd_{j}"][k])
            np.testing.assert_array_equal(state.qdd, g[f"i_qdd_{j}"][k])
