"""Pin the CPU oracle (oracle/vp_oracle.c) against golden vectors produced by
the reference itself (tests/golden/make_golden.py).  CPU only.

Bars: EDT / fh_1d / masked pixels / fusion bit-exact; query and rollout
within 1e-12 relative (libm transcendental ulps); softmin/update 1e-13.
"""

import numpy as np
import pytest

import oracle
from conftest import i32_to_sq, load_golden, unpack_occ

ROLLOUT_KEYS = (
    "q0 qd0 dt base_r base_t off_r off_t axes sph_link sph_loc sph_r pairs goal_r goal_t "
    "pose_weight terminal_weight pos_lo pos_hi vel_lo vel_hi acc_lo acc_hi w_env w_self w_q "
    "w_qd w_qdd w_s w_ns d_act q_ref field_sq field_lo0 field_lo1 field_lo2 field_origin0 "
    "field_origin1 field_origin2 field_voxel field_outside"
).split()


def rollout_args(g, i):
    args = {k: g[f"r_{k}_{i}"] for k in ROLLOUT_KEYS if k != "field_sq"}
    args["field_sq"] = i32_to_sq(g[f"r_field_sq_{i}"])
    return args


def test_fh_1d_golden():
    g = load_golden("edt")
    for i in range(int(g["fh_count"])):
        np.testing.assert_array_equal(oracle.fh_1d(g[f"fh_in_{i}"]), g[f"fh_out_{i}"])


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_edt_golden_bit_exact(threads):
    g = load_golden("edt")
    oracle.set_threads(threads)
    try:
        for i in range(int(g["edt_count"])):
            occ = unpack_occ(g[f"edt_occ_{i}"], g[f"edt_dims_{i}"])
            lo_odds = np.where(occ, 3.5, 0.0)
            got = oracle.edt3d(lo_odds, tuple(g[f"edt_lo_{i}"]), tuple(g[f"edt_hi_{i}"]))
            np.testing.assert_array_equal(got, i32_to_sq(g[f"edt_sq_{i}"]), err_msg=str(g[f"edt_name_{i}"]))
    finally:
        oracle.set_threads(0)


def test_edt_pass_order_independent():
    g = load_golden("edt")
    for i in range(int(g["edt_count"])):
        if str(g[f"edt_name_{i}"]) != "order_9x11x6":
            continue
        occ = unpack_occ(g[f"edt_occ_{i}"], g[f"edt_dims_{i}"])
        lo = np.where(occ, 3.5, 0.0)
        a = oracle.edt3d(lo, pass_order=("y", "x", "z"))
        for order in (("x", "y", "z"), ("z", "y", "x")):
            np.testing.assert_array_equal(a, oracle.edt3d(lo, pass_order=order))


def test_edt_threshold_boundary():
    g = load_golden("edt")
    np.testing.assert_array_equal(oracle.edt3d(g["thr_log_odds"]), i32_to_sq(g["thr_sq"]))


def _cam(g, i):
    fx, fy, cx, cy, dmin, dmax = g[f"f_cam{i}_intr"]
    w, h = (int(v) for v in g[f"f_cam{i}_wh"])
    return fx, fy, cx, cy, dmin, dmax, w, h


def test_masked_pixels_and_fusion_golden_bit_exact():
    g = load_golden("fusion")
    params = dict(l_hit=0.85, l_miss=-0.4, l_min=-2.0, l_max=3.5)
    for i in range(int(g["f_count"])):
        name = str(g[f"f_name_{i}"])
        dims = tuple(int(v) for v in g[f"f_dims_{i}"])
        voxel = float(g[f"f_voxel_{i}"])
        origin = g[f"f_origin_{i}"]
        fx, fy, cx, cy, dmin, dmax, w, h = _cam(g, i)
        if f"f_box_{i}" in g:
            lo, hi = g[f"f_box_{i}"]
        else:
            lo, hi = np.zeros(3, np.int64), np.array(dims)
        log_odds = np.zeros(dims)
        observed = np.zeros(dims, bool)
        for s in range(int(g[f"f_nsteps_{i}"])):
            depth = g[f"f_depth_{i}_{s}"]
            if f"f_mc_{i}_{s}" in g:
                mc, mr = g[f"f_mc_{i}_{s}"], g[f"f_mr_{i}_{s}"]
            else:
                mc, mr = np.zeros((0, 3)), np.zeros(0)
            pm = oracle.masked_pixels(depth, fx, fy, cx, cy, dmin, dmax, g[f"f_cam{i}_pose_r"],
                                      g[f"f_cam{i}_pose_t"], mc, mr, float(g[f"f_pad_{i}"]))
            np.testing.assert_array_equal(pm, g[f"f_pm_{i}_{s}"], err_msg=f"{name} step {s} mask")
            oracle.fuse_voxels(log_odds, observed, lo, hi - lo, origin, voxel, g[f"f_cam{i}_w2c_r"],
                               g[f"f_cam{i}_w2c_t"], fx, fy, cx, cy, w, h, dmin, dmax, depth, pm,
                               mc, mr, 2.5 * voxel, **params)
            np.testing.assert_array_equal(log_odds, g[f"f_lo_{i}_{s}"], err_msg=f"{name} step {s}")
            np.testing.assert_array_equal(observed, g[f"f_ob_{i}_{s}"], err_msg=f"{name} step {s}")


def test_fusion_rational_threshold_sequences():
    """h,h,h,h,m after 5 misses lands at 0.9999999999999999
    (not occupied), h,h,h,m,h lands exactly on 1.0 (occupied)."""
    g = load_golden("fusion")
    names = {str(g[f"f_name_{i}"]): i for i in range(int(g["f_count"]))}
    a = g[f"f_lo_{names['rational_a']}_9"][0, 0, 0]
    b = g[f"f_lo_{names['rational_b']}_9"][0, 0, 0]
    assert a == 0.9999999999999999 and b == 1.0


def test_query_golden():
    g = load_golden("query")
    for i in range(int(g["q_count"])):
        sq = i32_to_sq(g[f"q_sq_{i}"])
        ox, oy, oz, voxel, outside = g[f"q_meta_{i}"]
        lo = tuple(int(v) for v in g[f"q_lo_{i}"])
        got = np.array([oracle.query_metric(sq, lo, (ox, oy, oz), voxel, outside, p) for p in g[f"q_pts_{i}"]])
        np.testing.assert_array_equal(got, g[f"q_val_{i}"])


@pytest.mark.parametrize("threads", [1, 4])
def test_rollout_golden(threads):
    g = load_golden("rollout")
    oracle.set_threads(threads)
    try:
        for i in range(int(g["r_count"])):
            name = str(g[f"r_name_{i}"])
            store = bool(g[f"r_store_{i}"])
            out = oracle.evaluate_batch(rollout_args(g, i), g[f"r_controls_{i}"], store, store)
            np.testing.assert_array_equal(out["flags"], g[f"r_flags_{i}"], err_msg=name)
            ok = g[f"r_flags_{i}"] == 0
            np.testing.assert_allclose(out["costs"][ok], g[f"r_costs_{i}"][ok], rtol=1e-12, atol=0, err_msg=name)
            assert np.all(np.isinf(out["costs"][~ok]))
            np.testing.assert_allclose(out["terms"], g[f"r_terms_{i}"], rtol=1e-12, atol=1e-300, err_msg=name)
            if store:
                np.testing.assert_allclose(out["traj_q"], g[f"r_trajq_{i}"], rtol=1e-13, atol=1e-15)
                np.testing.assert_allclose(out["traj_qd"], g[f"r_trajqd_{i}"], rtol=1e-13, atol=1e-15)
                np.testing.assert_allclose(out["sphere_pos"], g[f"r_sphpos_{i}"], rtol=1e-12, atol=1e-15)
    finally:
        oracle.set_threads(0)


def test_softmin_update_golden():
    g = load_golden("softmin")
    for i in range(int(g["s_count"])):
        w = oracle.soft_weights(g[f"s_costs_{i}"], float(g[f"s_lam_{i}"]))
        np.testing.assert_allclose(w, g[f"s_w_{i}"], rtol=1e-13, atol=1e-300)
        u = oracle.update_controls(g[f"s_nom_{i}"], g[f"s_eps_{i}"], g[f"s_w_{i}"])
        np.testing.assert_allclose(u, g[f"s_u_{i}"], rtol=1e-12, atol=1e-14)


def test_softmin_validation_errors():
    with pytest.raises(ValueError):
        oracle.soft_weights(np.array([]), 0.5)
    with pytest.raises(ValueError):
        oracle.soft_weights(np.array([1.0, np.inf]), 0.5)
    with pytest.raises(ValueError):
        oracle.soft_weights(np.array([1.0]), 0.0)


def test_golden_fields_are_lipschitz_edts():
    """The fp32 rollout's far-cell exit (rollout_fixed.cuh, env_cost) assumes
    sqrt(field) is 1-Lipschitz between voxel centres, which holds for an
    exact EDT.  Pin it on every field the reference produced."""
    g = load_golden("rollout")
    i = 0
    checked = 0
    while f"r_field_sq_{i}" in g:
        d = np.sqrt(i32_to_sq(g[f"r_field_sq_{i}"]))
        if np.isfinite(d).all():
            for sh in [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, 0, 1), (0, 1, 1), (1, 1, 1)]:
                a = d[:d.shape[0] - sh[0], :d.shape[1] - sh[1], :d.shape[2] - sh[2]]
                b = d[sh[0]:, sh[1]:, sh[2]:]
                assert np.abs(a - b).max() <= np.sqrt(sum(sh)) + 1e-9
            checked += 1
        else:
            assert np.isinf(d).all()  # no source at all
        i += 1
    assert checked >= 1


def brute_force_sqdist(occ):
    """Independent O(N * sources) check, as vp/oracles.py:68-101 does for
    acceptance criterion 1 (t/test_acceptance.py:57-81)."""
    src = np.argwhere(occ)
    out = np.full(occ.shape, np.inf)
    if len(src):
        idx = np.indices(occ.shape).reshape(3, -1).T
        d = ((idx[:, None, :] - src[None, :, :]) ** 2).sum(-1).min(1)
        out = d.reshape(occ.shape).astype(float)
    return out


def test_edt_acceptance_100_grids_golden():
    """All 100 grids of acceptance criterion 1: oracle == reference == brute force."""
    g = load_golden("edt_acceptance")
    for i in range(g["occ"].shape[0]):
        occ = unpack_occ(g["occ"][i], (16, 16, 16))
        want = i32_to_sq(g["sq"][i])
        np.testing.assert_array_equal(want, brute_force_sqdist(occ), err_msg=f"grid {i}: golden vs brute force")
        np.testing.assert_array_equal(oracle.edt3d_from_occupancy(occ), want, err_msg=f"grid {i}")


def test_reference_arm_scene_matches_product_mirror():
    """oracle/scene.py (the reference arm's host-only scene, no product import)
    builds the same problem as the product's host mirror."""
    from oracle import scene as osc
    from paper_2512_22575_b200 import config, planner, robot
    from conftest import oracle_args

    chain, model = config.robot_7dof()
    params = config.planner_params(7, {"samples": 4096, "horizon": 32})
    state = robot.JointState.resting(np.full(7, 0.05))
    goal = robot.forward_kinematics(chain, np.full(7, 0.35))[-1]
    want = oracle_args(planner, chain, model, params, state, goal, None)
    got = osc.rollout_args(np.zeros((1, 1, 1)), np.zeros(3), 1.0)
    for k, v in want.items():
        if k.startswith("field_"):
            continue
        np.testing.assert_allclose(np.asarray(got[k], float), np.asarray(v, float), rtol=0, atol=1e-15, err_msg=k)
    c0, r0 = robot.sphere_positions(chain, np.full(7, 0.3), model)
    c1, r1 = osc.sphere_positions(np.full(7, 0.3))
    np.testing.assert_allclose(c1, c0, rtol=0, atol=1e-15)
    np.testing.assert_array_equal(r1, r0)
    assert params.lam == osc.DEFAULTS["lam"] and params.noise_window == osc.DEFAULTS["noise_window"]
