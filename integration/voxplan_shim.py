"""Reference-side binding: swap the voxplan numba seams for libvpb200.

A voxplan maintainer adds this module and calls ``install()`` once after
``import voxplan``.  The reference has no plugin registry: its
boundary is a set of module-level functions looked up at call time, so
rebinding the module attributes reroutes every internal caller.

    import voxplan, voxplan_shim
    voxplan_shim.install(voxplan)

Seams and the C entry point that replaces each one (include/vpb200.h):

    voxplan.mapping._fuse_voxels    (vp/mapping.py:266-354)  -> vpb_fuse_voxels
    voxplan.mapping.edt_3d          (vp/mapping.py:586-613)  -> vpb_edt3d
                                     (replaces the init + 3 _EDT_PASSES + inf mapping;
                                      the per-pass seam stays f64 in place)
    voxplan.batch.evaluate_batch    (vp/batch.py:161-336)    -> vpb_evaluate_batch (fp64 parity mode)
    voxplan.planner.soft_weights    (vp/planner.py:373-384)  -> vpb_soft_weights
    voxplan.planner.update_controls (vp/planner.py:387-400)  -> vpb_update_controls

The seams keep the reference's host-array contract: every call uploads its
numpy inputs, runs the kernel and writes the outputs back in place.  That is
the drop-in path.  The fast path keeps the state device-resident
(paper_2512_22575_b200.mapping / .planner).  Validation and exceptions stay in
the reference's Python callers, which run before each seam.
"""

from __future__ import annotations

import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2512_22575_b200 import _lib as L  # noqa: E402

MAX_J, MAX_S, MAX_P = L.MAX_JOINTS, L.MAX_SPHERES, L.MAX_PAIRS


def _fill(arr, values) -> None:
    L.fill(arr, values)


def problem_from_reference_args(q0, qd0, dt, base_r, base_t, off_r, off_t, axes, sph_link, sph_loc, sph_r, pairs,
                                 goal_r, goal_t, pose_weight, terminal_weight, pos_lo, pos_hi, vel_lo, vel_hi,
                                 acc_lo, acc_hi, w_env, w_self, w_q, w_qd, w_qdd, w_s, w_ns, d_act, q_ref,
                                 horizon) -> L.VpbProblem:
    """Pack evaluate_batch's flat arguments (vp/batch.py:162-195) into the
    vpb_problem block.  Spheres are stably sorted by link (the kernel emits
    sphere centres while it walks the chain); ``sph_orig`` keeps the caller's
    order for the outputs and self pairs are remapped to the sorted order."""
    n = int(np.asarray(q0).shape[0])
    sph_link = np.asarray(sph_link, dtype=np.int64).reshape(-1)
    ns = sph_link.shape[0]
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if n > MAX_J or ns > MAX_S or pairs.shape[0] > MAX_P:
        raise ValueError("robot exceeds the kernel limits (16 joints, 64 spheres, 256 pairs)")
    P = L.VpbProblem()
    P.n_joints, P.horizon, P.dt = n, int(horizon), float(dt)
    _fill(P.base_r, base_r)
    _fill(P.base_t, base_t)
    _fill(P.off_r, off_r)
    _fill(P.off_t, off_t)
    _fill(P.axes, axes)
    order = np.argsort(sph_link, kind="stable")
    pos = np.empty(ns, dtype=np.int64)
    pos[order] = np.arange(ns)
    sph_loc = np.asarray(sph_loc, dtype=float).reshape(-1, 3)
    sph_r = np.asarray(sph_r, dtype=float).reshape(-1)
    P.n_spheres = ns
    for k, s in enumerate(order):
        P.sph_link[k] = int(sph_link[s])
        P.sph_orig[k] = int(s)
        P.sph_loc[3 * k:3 * k + 3] = list(sph_loc[s])
        P.sph_r[k] = float(sph_r[s])
    P.n_pairs = pairs.shape[0]
    for q, (a, b) in enumerate(pairs):
        P.pairs[2 * q], P.pairs[2 * q + 1] = int(pos[a]), int(pos[b])
    _fill(P.goal_r, goal_r)
    _fill(P.goal_t, goal_t)
    _fill(P.pose_weight, pose_weight)
    _fill(P.terminal_weight, terminal_weight)
    for name, arr in zip(("pos_lo", "pos_hi", "vel_lo", "vel_hi", "acc_lo", "acc_hi", "q_ref", "q0", "qd0"),
                         (pos_lo, pos_hi, vel_lo, vel_hi, acc_lo, acc_hi, q_ref, q0, qd0)):
        _fill(getattr(P, name), arr)
    P.w_env, P.w_self, P.w_q, P.w_qd = float(w_env), float(w_self), float(w_q), float(w_qd)
    P.w_qdd, P.w_s, P.w_ns, P.d_act = float(w_qdd), float(w_s), float(w_ns), float(d_act)
    return P


def field_from_reference_args(sq_dev_ptr, shape, lo, origin, voxel, outside) -> L.VpbField:
    """_field_arguments' tuple (vp/planner.py:429-455) -> vpb_field."""
    f = L.VpbField()
    f.sq = sq_dev_ptr
    f.n = L.i64x3(shape)
    f.lo = L.i64x3(lo)
    _fill(f.origin, origin)
    f.voxel = float(voxel)
    f.outside_default = float(outside)
    return f


def install(voxplan) -> None:  # pragma: no cover - needs the reference and a GPU
    """Rebind the seams of an imported voxplan package."""
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    lib = L.load()

    def stream():
        return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)

    def to_dev(a, dtype=None):
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t.to(dev) if dtype is None else t.to(dev).to(dtype)

    def ptr(t):
        return ctypes.c_void_p(t.data_ptr())

    def check(rc, what):
        L.check(rc, what)

    # -- _fuse_voxels (29 positional args, vp/mapping.py:267-297) ------------------
    def fuse_voxels(log_odds, observed, lo0, lo1, lo2, n0, n1, n2, origin, voxel, cam_r, cam_t, fx, fy, cx, cy,
                    width, height, d_min, d_max, depth, pixel_masked, mask_centers, mask_radii, tau, l_hit,
                    l_miss, l_min, l_max):
        lo_d = to_dev(log_odds)
        ob_d = to_dev(observed.view(np.uint8))
        g = L.VpbGrid()
        g.log_odds, g.observed, g.occ_bits = ptr(lo_d), ptr(ob_d), None
        g.dims = L.i64x3(log_odds.shape)
        _fill(g.origin, origin)
        g.voxel = float(voxel)
        cam = L.VpbCamera()
        cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max = fx, fy, cx, cy, d_min, d_max
        cam.width, cam.height = int(width), int(height)
        _fill(cam.w2c_r, cam_r)
        _fill(cam.w2c_t, cam_t)
        prm = L.VpbMapParams()
        prm.l_hit, prm.l_miss, prm.l_min, prm.l_max, prm.tau = l_hit, l_miss, l_min, l_max, tau
        prm.l_occ_threshold = np.inf  # no packed mask on this path
        centers = np.ascontiguousarray(mask_centers, dtype=float).reshape(-1, 3)
        radii = np.ascontiguousarray(mask_radii, dtype=float).reshape(-1)
        depth_d = to_dev(np.asarray(depth, dtype=float))
        pm_d = to_dev(np.asarray(pixel_masked).view(np.uint8))
        check(lib.vpb_fuse_voxels(g, L.i64x3((lo0, lo1, lo2)), L.i64x3((n0, n1, n2)), cam, ptr(depth_d),
                                  ptr(pm_d), centers.ctypes.data_as(ctypes.c_void_p),
                                  radii.ctypes.data_as(ctypes.c_void_p), radii.shape[0], prm, stream()),
              "fuse_voxels")
        log_odds[...] = lo_d.cpu().numpy()
        observed[...] = ob_d.cpu().numpy().astype(bool)

    # -- edt_3d (vp/mapping.py:586-613) ---------------------------------------------
    ref_mapping = voxplan.mapping

    def edt_3d(grid, volume=None, outside_default=1.0, pass_order=("y", "x", "z")):
        box = volume or grid.full_box()
        grid.validate_box(box)
        if sorted(pass_order) != ["x", "y", "z"]:
            raise ValueError(f"pass_order must permute x, y, z; got {pass_order}")
        lo_d = to_dev(grid.log_odds)
        g = L.VpbGrid()
        g.log_odds, g.observed, g.occ_bits = ptr(lo_d), None, None
        g.dims = L.i64x3(grid.dims)
        n = L.i64x3(tuple(h - l for l, h in zip(box.lo, box.hi)))
        ws = torch.empty(int(lib.vpb_edt3d_workspace_bytes(n)), dtype=torch.uint8, device=dev)
        out = torch.empty(tuple(n), dtype=torch.float32, device=dev)
        check(lib.vpb_edt3d(g, L.i64x3(box.lo), n, float(grid.params.l_occ_threshold), 0, ptr(out), ptr(ws),
                            ws.numel(), stream()), "edt_3d")
        sq = out.to(torch.float64).cpu().numpy()  # +inf already where the box has no source
        return ref_mapping.DistanceField(origin=grid.origin, voxel_size=grid.voxel_size, dims=grid.dims,
                                         volume=box, sq=sq, outside_default=outside_default)

    # -- evaluate_batch (49 positional args, vp/batch.py:162-212) -------------------
    def evaluate_batch(q0, qd0, controls, dt, base_r, base_t, off_r, off_t, axes, sph_link, sph_loc, sph_r, pairs,
                       goal_r, goal_t, pose_weight, terminal_weight, pos_lo, pos_hi, vel_lo, vel_hi, acc_lo, acc_hi,
                       w_env, w_self, w_q, w_qd, w_qdd, w_s, w_ns, d_act, q_ref, field_sq, field_lo0, field_lo1,
                       field_lo2, field_origin0, field_origin1, field_origin2, field_voxel, field_outside,
                       store_traj, store_spheres, costs, terms, traj_q, traj_qd, sphere_pos, flags):
        m, h, _ = controls.shape
        P = problem_from_reference_args(q0, qd0, dt, base_r, base_t, off_r, off_t, axes, sph_link, sph_loc,
                                        sph_r, pairs, goal_r, goal_t, pose_weight, terminal_weight, pos_lo,
                                        pos_hi, vel_lo, vel_hi, acc_lo, acc_hi, w_env, w_self, w_q, w_qd, w_qdd,
                                        w_s, w_ns, d_act, q_ref, h)
        sq_d = to_dev(np.asarray(field_sq, dtype=np.float32))
        F = field_from_reference_args(ptr(sq_d), field_sq.shape, (field_lo0, field_lo1, field_lo2),
                                      (field_origin0, field_origin1, field_origin2), field_voxel, field_outside)
        c_d = to_dev(controls)
        outs = [torch.empty(a.shape, dtype=torch.float64, device=dev) for a in (costs, terms)]
        fl_d = torch.empty(flags.shape, dtype=torch.uint8, device=dev)
        tq = torch.empty(traj_q.shape, dtype=torch.float64, device=dev) if store_traj else None
        tqd = torch.empty(traj_qd.shape, dtype=torch.float64, device=dev) if store_traj else None
        sp = torch.empty(sphere_pos.shape, dtype=torch.float64, device=dev) if store_spheres else None
        nul = ctypes.c_void_p(None)
        check(lib.vpb_evaluate_batch(P, F, ptr(c_d), nul, L.DTYPE_F64, m, L.PREC_F64, ptr(outs[0]), ptr(outs[1]),
                                     ptr(fl_d), ptr(tq) if tq is not None else nul,
                                     ptr(tqd) if tqd is not None else nul, ptr(sp) if sp is not None else nul,
                                     stream()), "evaluate_batch")
        costs[...] = outs[0].cpu().numpy()
        terms[...] = outs[1].cpu().numpy()
        flags[...] = fl_d.cpu().numpy()
        if store_traj:
            traj_q[...] = tq.cpu().numpy()
            traj_qd[...] = tqd.cpu().numpy()
        if store_spheres:
            sphere_pos[...] = sp.cpu().numpy()

    # -- soft_weights / update_controls (vp/planner.py:373-400) ----------------------
    from paper_2512_22575_b200 import errors as our_errors
    from paper_2512_22575_b200 import planner as our_planner

    def soft_weights(costs, lam):
        return our_planner.soft_weights(np.asarray(costs, dtype=float), float(lam))

    def update_controls(nominal, eps, weights):
        try:
            return our_planner.update_controls(np.asarray(nominal, dtype=float), np.asarray(eps, dtype=float),
                                               np.asarray(weights, dtype=float))
        except our_errors.WeightMismatch as e:  # re-raise as the reference's own type
            raise voxplan.errors.WeightMismatch(str(e)) from None

    voxplan.mapping._fuse_voxels = fuse_voxels
    voxplan.mapping.edt_3d = edt_3d
    voxplan.batch.evaluate_batch = evaluate_batch
    voxplan.planner.soft_weights = soft_weights
    voxplan.planner.update_controls = update_controls
