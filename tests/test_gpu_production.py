"""Full SMPC step parity against the oracle at the production shapes.

SURVEY.md 8(c) tolerances for the fp32 production kernel (BASELINE.json
north_star: "rollout costs, weights and the updated mean control sequence
within 1e-4 relative in fp32"):
  * per-sample costs: rtol 1e-4;
  * softmin weights: |w_gpu - w_ref| <= 1e-4 * max w (the
    weights are near one-hot at lam = 0.05, so a relative bar on a 1e-30
    weight is meaningless; the floor is relative to the largest weight);
  * U*, command, next nominal: rtol 1e-4 with an absolute floor of 1e-4 *
    max |U*| (elements that cancel to ~0);
and rtol 1e-9 for the fp64 parity mode.  The reference's own seeded noise
(vp/planner.py:199-219, restated by oracle.sample_perturbations) is fed to
both sides.  The weights are the fused kernel's own (vpb_smpc_debug_weights),
not recomputed on the host.

Shapes: C3 (4096 x 32) on the C2 256^3 masked bench field and on the
acceptance planner scene (robot in collision, t/test_acceptance.py:308-317);
C5 (16384 x 32) in the converged regime (the state and warm start after 30
closed-loop frames, thousands of nonzero weights: the helper-CTA merge); the
C4 horizon (H = 64) with an active field.  Also counted: fp32 "face flips"
(SURVEY.md 7.3-6), samples whose collision term differs from the oracle's by
more than the tolerance.
"""

import numpy as np
import pytest

import oracle
from conftest import oracle_args

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_22575_b200 import config, mapping, planner, robot, scene

    oracle.build()
    oracle.set_threads(0)
    return config, mapping, planner, robot, scene


def _bench_field(pk, n):
    config, mapping, planner, robot, scene = pk
    chain, model = config.robot_7dof()
    centers, radii = robot.sphere_positions(chain, np.full(7, 0.3), model)
    grid, cam, depth = scene.bench_edt_scene((n, n, n), robot_spheres=(centers, radii))
    mapper = mapping.OccupancyMapper(grid, cam, outside_default=0.8)
    for _ in range(2):
        mapper.update(depth, mask=(centers, radii))
    return mapper.recompute_edt()


def _acceptance_field(pk):
    config, mapping, planner, robot, scene = pk
    origin, voxel, occ = scene.acceptance_planner_occupancy()
    grid = mapping.VoxelGrid(origin, voxel, occ.shape)
    grid.set_log_odds(np.where(occ, 3.5, 0.0))
    return mapping.edt_3d(grid, outside_default=0.8)


def _reach_field(pk):
    config, mapping, planner, robot, scene = pk
    origin, voxel, occ = scene.reach_static_occupancy()
    grid = mapping.VoxelGrid(origin, voxel, occ.shape)
    grid.set_log_odds(np.where(occ, 3.5, 0.0))
    return mapping.edt_3d(grid, outside_default=0.8)


def _step_parity(pk, pl, state, goal, field, nominal, eps, name, report):
    """One fused step on the GPU vs oracle.smpc_step on the same inputs."""
    config, mapping, planner, robot, scene = pk
    m, h, n = eps.shape
    fp32 = pl.precision == "fp32"
    nom_dev = torch.from_numpy(np.ascontiguousarray(nominal)).cuda()
    eps_dev = torch.from_numpy(eps).cuda().to(torch.float32 if fp32 else torch.float64)
    costs = torch.empty(m, dtype=torch.float64, device="cuda")
    out = pl.smpc_step_device(state, goal, field, nom_dev, eps_dev, costs=costs).cpu().numpy()
    w_gpu = pl.smpc_weights_device(m, h).cpu().numpy()
    c_gpu = costs.cpu().numpy()
    args = oracle_args(planner, pl.chain, pl.model, pl.params, state, goal, field)
    want = oracle.smpc_step(args, nominal, eps, pl.params.lam, pl.chain.acceleration_limits())
    w_ref = oracle.soft_weights(want["costs"], pl.params.lam)
    hn = h * n
    u_gpu = out[:hn].reshape(h, n)
    rtol = 1e-4 if fp32 else 1e-9
    # costs
    np.testing.assert_allclose(c_gpu, want["costs"], rtol=rtol, err_msg=f"{name}: costs")
    # weights (the kernel's own)
    dw = np.abs(w_gpu - w_ref).max()
    assert dw <= rtol * w_ref.max(), f"{name}: max |dw| = {dw:.3e} > {rtol} * max w = {w_ref.max():.3e}"
    np.testing.assert_allclose(w_gpu.sum(), 1.0, rtol=1e-12)
    # U*, command, next nominal
    floor = rtol * np.abs(want["u"]).max()
    np.testing.assert_allclose(u_gpu, want["u"], rtol=rtol, atol=floor, err_msg=f"{name}: U*")
    np.testing.assert_allclose(out[hn:hn + n], want["command"], rtol=rtol, atol=floor, err_msg=f"{name}: command")
    np.testing.assert_allclose(out[hn + n:2 * hn + n].reshape(h, n), want["next_nominal"], rtol=rtol, atol=floor,
                               err_msg=f"{name}: next nominal")
    base = 2 * hn + n
    np.testing.assert_allclose(out[base], want["weighted_cost"], rtol=rtol, err_msg=f"{name}: weighted cost")
    np.testing.assert_allclose(out[base + 7], want["best_cost"], rtol=rtol, err_msg=f"{name}: best cost")
    # fp32 face flips: the collision term of every sample (same code path, rollout kernel)
    flips = 0
    if fp32:
        got = pl.evaluate(state, goal, field, nominal[None] + eps.astype(np.float32).astype(np.float64))
        ref = oracle.evaluate_batch(args, nominal[None] + eps)
        err = np.abs(got.terms[:, 1] - ref["terms"][:, 1])
        flips = int((err > 1e-4 * np.abs(ref["terms"][:, 1]) + 1e-6 * (1.0 + np.abs(ref["costs"]))).sum())
    nnz = int((w_ref > 0).sum())
    report.append((name, pl.precision, m, h, nnz, float(dw / w_ref.max()),
                   float(np.max(np.abs(c_gpu - want["costs"]) / np.abs(want["costs"]))),
                   float(np.max(np.abs(u_gpu - want["u"])) / np.abs(want["u"]).max()), flips))
    assert flips == 0, f"{name}: {flips} fp32 face flips in the collision term"
    return nnz


@pytest.fixture(scope="module")
def report():
    rows = []
    yield rows
    print("\nname precision M H nonzero_w max|dw|/max_w max_rel_cost max|dU|/max|U| face_flips")
    for r in rows:
        print(" ".join(str(v) for v in r))


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_c3_step_bench_field(pk, report, precision):
    """C3: 4096 x 32 on the C2 256^3 masked bench map (the bench workload)."""
    config, mapping, planner, robot, scene = pk
    chain, model = config.robot_7dof()
    field = _bench_field(pk, 256)
    params = config.planner_params(7, {"samples": 4096, "horizon": 32})
    pl = planner.Planner(chain, model, params, precision)
    state = robot.JointState.resting(np.full(7, 0.05))
    goal = robot.forward_kinematics(chain, np.full(7, 0.35))[-1]
    for seed, nominal in ((11, np.zeros((32, 7))), (12, 0.3 * np.sin(np.arange(224.0)).reshape(32, 7))):
        eps = oracle.sample_perturbations(4096, 32, 7, params.sigma, params.noise_window, seed)
        _step_parity(pk, pl, state, goal, field, nominal, eps, f"C3 bench256 seed{seed}", report)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_c3_step_in_collision(pk, report, precision):
    """C3 on the acceptance planner scene: the start is in collision (costs
    ~1e5), so the collision term and the field query dominate."""
    config, mapping, planner, robot, scene = pk
    chain, model = config.robot_7dof()
    field = _acceptance_field(pk)
    params = config.planner_params(7, {"samples": 4096, "horizon": 32})
    pl = planner.Planner(chain, model, params, precision)
    state = robot.JointState.resting(np.full(7, 0.05))
    goal = robot.forward_kinematics(chain, np.full(7, 0.35))[-1]
    eps = oracle.sample_perturbations(4096, 32, 7, params.sigma, params.noise_window, 21)
    _step_parity(pk, pl, state, goal, field, np.zeros((32, 7)), eps, "C3 acceptance", report)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_c4_horizon_step_with_field(pk, report, precision):
    """The C4 horizon (H = 64) with an active field, 4096 samples (C4's
    per-rank shape at N = 16 and the merge at H n = 448)."""
    config, mapping, planner, robot, scene = pk
    chain, model = config.robot_7dof()
    field = _reach_field(pk)
    params = config.planner_params(7, {"samples": 4096, "horizon": 64, "q_ref": scene.REACH_STATIC_QREF})
    pl = planner.Planner(chain, model, params, precision)
    state = robot.JointState.resting(scene.REACH_STATIC_START)
    from paper_2512_22575_b200.geometry import RigidTransform

    goal = RigidTransform.from_vec7(scene.REACH_STATIC_GOAL)
    eps = oracle.sample_perturbations(4096, 64, 7, params.sigma, params.noise_window, 31)
    _step_parity(pk, pl, state, goal, field, np.zeros((64, 7)), eps, "C4-H64 reach_static", report)


def _converged_state(pk, pl, field, goal, start, frames):
    """Closed loop through the production path (native session, on-device
    noise): the state and warm start after `frames` replans."""
    config, mapping, planner, robot, scene = pk
    state = robot.JointState.resting(start)
    nominal = np.zeros((pl.params.horizon, 7))
    for f in range(frames):
        res = pl.smpc_step(state, goal, field, nominal, 1000 + f)
        state = pl.integrate(state, res.command)
        nominal = res.next_nominal
    return state, nominal


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_c5_converged_step(pk, report, precision):
    """C5 shape (16384 x 32) in the converged regime: the state after 30
    closed-loop frames on the reach_static board scene.  Thousands of weights
    are nonzero, so the merge runs the helper-CTA N reduction."""
    config, mapping, planner, robot, scene = pk
    from paper_2512_22575_b200.geometry import RigidTransform

    chain, model = config.robot_7dof()
    field = _reach_field(pk)
    params = config.planner_params(7, {"samples": 16384, "horizon": 32, "q_ref": scene.REACH_STATIC_QREF})
    goal = RigidTransform.from_vec7(scene.REACH_STATIC_GOAL)
    pl32 = planner.Planner(chain, model, params, "fp32")
    state, nominal = _converged_state(pk, pl32, field, goal, scene.REACH_STATIC_START, 30)
    pl = pl32 if precision == "fp32" else planner.Planner(chain, model, params, "fp64")
    eps = oracle.sample_perturbations(16384, 32, 7, params.sigma, params.noise_window, 41)
    nnz = _step_parity(pk, pl, state, goal, field, nominal, eps, "C5 converged", report)
    assert nnz > 32, f"expected the many-weights regime, got {nnz} nonzero weights"
