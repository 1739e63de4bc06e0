"""CPU oracle for the ParaMaP hot path -- TEST INFRASTRUCTURE ONLY.

This package is the parity checker and the CPU baseline ("port").  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference`` arm) may import it.  The product package
``paper_2512_22575_b200`` never imports it and has no CPU fallback.

The arithmetic lives in ``oracle/vp_oracle.c`` (a float64 restatement of the
reference, compiled with ``-ffp-contract=off``); this module is a thin ctypes
wrapper that validates arguments the way the reference's Python layer does.
Parity of the restatement is pinned against golden vectors produced by the
reference itself (``tests/golden/*.npz``, see ``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libvp_oracle.so"
_lib = None

INF_SENTINEL = 1e20  # vp/mapping.py:32


def build() -> Path:
    """Compile the C restatement (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        _declare(_lib)
    return _lib


_d = ctypes.c_double
_i64 = ctypes.c_int64
_p = ctypes.c_void_p


def _declare(L):
    L.vpo_masked_pixels.argtypes = [_p, _i64, _i64, _d, _d, _d, _d, _d, _d, _p, _p, _p, _p, _i64, _d, _p]
    L.vpo_fuse_voxels.argtypes = (
        [_p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _p, _d, _p, _p, _d, _d, _d, _d]
        + [_i64, _i64, _d, _d, _p, _p, _p, _p, _i64, _d, _d, _d, _d, _d]
    )
    L.vpo_fh_1d.argtypes = [_p, _p, _i64]
    L.vpo_edt3d.argtypes = [_p, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _d, _p, _p]
    L.vpo_query_metric.argtypes = [_p, _i64, _i64, _i64, _i64, _i64, _i64, _d, _d, _d, _d, _d, _d, _d, _d]
    L.vpo_query_metric.restype = _d
    L.vpo_evaluate_batch.argtypes = [_p, _p, _i64, _i64, _p, _p, _p, _p, _p, _p]
    L.vpo_soft_weights.argtypes = [_p, _i64, _d, _p]
    L.vpo_update_controls.argtypes = [_p, _p, _p, _i64, _i64, _p]
    L.vpo_set_threads.argtypes = [ctypes.c_int]
    L.vpo_get_threads.restype = ctypes.c_int
    L.vpo_max_threads.restype = ctypes.c_int


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_p)


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def set_threads(n: int) -> None:
    lib().vpo_set_threads(int(n))


def get_threads() -> int:
    return int(lib().vpo_get_threads())


# ---------------------------------------------------------------------------
# mapping (vp/mapping.py)
# ---------------------------------------------------------------------------
def masked_pixels(depth, fx, fy, cx, cy, d_min, d_max, pose_r, pose_t, centers, radii, pad):
    """vp/mapping.py:357-380."""
    depth = _c(depth)
    pose_r, pose_t = _c(pose_r), _c(pose_t)
    centers = _c(centers).reshape(-1, 3)
    radii = _c(radii).reshape(-1)
    out = np.zeros(depth.shape, np.uint8)
    h, w = depth.shape
    lib().vpo_masked_pixels(
        _ptr(depth), h, w, fx, fy, cx, cy, d_min, d_max, _ptr(pose_r), _ptr(pose_t),
        _ptr(centers), _ptr(radii), centers.shape[0], pad, _ptr(out),
    )
    return out.astype(bool)


def fuse_voxels(log_odds, observed, lo, n, origin, voxel, cam_r, cam_t, fx, fy, cx, cy,
                width, height, d_min, d_max, depth, pixel_masked, centers, radii,
                tau, l_hit, l_miss, l_min, l_max):
    """vp/mapping.py:266-354, in place on (log_odds f64, observed bool) grids."""
    assert log_odds.dtype == np.float64 and log_odds.flags.c_contiguous
    assert observed.dtype == np.bool_ and observed.flags.c_contiguous
    obs_u8 = observed.view(np.uint8)
    origin, cam_r, cam_t, depth = _c(origin), _c(cam_r), _c(cam_t), _c(depth)
    pm = _c(pixel_masked, np.uint8)
    centers = _c(centers).reshape(-1, 3)
    radii = _c(radii).reshape(-1)
    gx, gy, gz = log_odds.shape
    lib().vpo_fuse_voxels(
        _ptr(log_odds), _ptr(obs_u8), gx, gy, gz, lo[0], lo[1], lo[2], n[0], n[1], n[2],
        _ptr(origin), voxel, _ptr(cam_r), _ptr(cam_t), fx, fy, cx, cy, width, height,
        d_min, d_max, _ptr(depth), _ptr(pm), _ptr(centers), _ptr(radii), centers.shape[0],
        tau, l_hit, l_miss, l_min, l_max,
    )


def fh_1d(line):
    """vp/mapping.py:486-499."""
    line = _c(line)
    out = np.empty_like(line)
    lib().vpo_fh_1d(_ptr(line), _ptr(out), line.shape[0])
    return out


_AXIS = {"x": 0, "y": 1, "z": 2}


def edt3d(log_odds, lo=(0, 0, 0), hi=None, threshold=1.0, pass_order=("y", "x", "z")):
    """edt_3d body (vp/mapping.py:586-613): float64 squared distances, inf = no source."""
    log_odds = _c(log_odds)
    hi = tuple(log_odds.shape) if hi is None else tuple(hi)
    n = tuple(int(h) - int(l) for l, h in zip(lo, hi))
    out = np.empty(n, np.float64)
    order = np.array([_AXIS[a] for a in pass_order], np.int32)
    gx, gy, gz = log_odds.shape
    lib().vpo_edt3d(_ptr(log_odds), gx, gy, gz, lo[0], lo[1], lo[2], n[0], n[1], n[2],
                    threshold, _ptr(order), _ptr(out))
    return out


def edt3d_from_occupancy(occ):
    lo = np.where(np.asarray(occ, bool), 3.5, 0.0)
    return edt3d(lo)


def query_metric(sq, lo, origin, voxel, outside_default, p):
    """vp/mapping.py:616-685."""
    sq = _c(sq)
    n0, n1, n2 = sq.shape
    return float(lib().vpo_query_metric(
        _ptr(sq), n0, n1, n2, lo[0], lo[1], lo[2], origin[0], origin[1], origin[2],
        voxel, outside_default, p[0], p[1], p[2]))


# ---------------------------------------------------------------------------
# planner (vp/batch.py, vp/planner.py)
# ---------------------------------------------------------------------------
class _RolloutArgs(ctypes.Structure):
    _fields_ = [
        ("n", _i64), ("n_spheres", _i64), ("n_pairs", _i64), ("dt", _d),
        ("q0", _p), ("qd0", _p), ("base_r", _p), ("base_t", _p), ("off_r", _p),
        ("off_t", _p), ("axes", _p), ("sph_link", _p), ("sph_loc", _p), ("sph_r", _p),
        ("pairs", _p), ("goal_r", _p), ("goal_t", _p), ("pose_weight", _p),
        ("terminal_weight", _p), ("pos_lo", _p), ("pos_hi", _p), ("vel_lo", _p),
        ("vel_hi", _p), ("acc_lo", _p), ("acc_hi", _p), ("w_env", _d), ("w_self", _d),
        ("w_q", _d), ("w_qd", _d), ("w_qdd", _d), ("w_s", _d), ("w_ns", _d), ("d_act", _d),
        ("q_ref", _p), ("field_sq", _p), ("field_n0", _i64), ("field_n1", _i64),
        ("field_n2", _i64), ("field_lo0", _i64), ("field_lo1", _i64), ("field_lo2", _i64),
        ("field_origin0", _d), ("field_origin1", _d), ("field_origin2", _d),
        ("field_voxel", _d), ("field_outside", _d),
    ]


_F64_KEYS = ("q0 qd0 base_r base_t off_r off_t axes sph_loc sph_r goal_r goal_t pose_weight "
             "terminal_weight pos_lo pos_hi vel_lo vel_hi acc_lo acc_hi q_ref field_sq").split()


def evaluate_batch(args: dict, controls, store_traj=False, store_spheres=False):
    """vp/batch.py:161-336.  `args` holds evaluate_batch's named inputs (the
    keys of tests/golden/make_golden.py:ROLLOUT_KEYS).  Returns a dict with
    costs, terms, flags (and traj_q/traj_qd/sphere_pos when requested)."""
    keep = {k: _c(args[k]) for k in _F64_KEYS}
    keep["sph_link"] = _c(args["sph_link"], np.int64)
    keep["pairs"] = _c(args["pairs"], np.int64).reshape(-1, 2)
    controls = _c(controls)
    m, h, n = controls.shape
    A = _RolloutArgs()
    A.n = n
    A.n_spheres = keep["sph_link"].shape[0]
    A.n_pairs = keep["pairs"].shape[0]
    A.dt = float(args["dt"])
    for k, v in keep.items():
        setattr(A, k, v.ctypes.data)
    for k in ("w_env", "w_self", "w_q", "w_qd", "w_qdd", "w_s", "w_ns", "d_act",
              "field_origin0", "field_origin1", "field_origin2", "field_voxel", "field_outside"):
        setattr(A, k, float(args[k]))
    fs = keep["field_sq"]
    A.field_n0, A.field_n1, A.field_n2 = fs.shape
    A.field_lo0, A.field_lo1, A.field_lo2 = (int(args["field_lo0"]), int(args["field_lo1"]),
                                             int(args["field_lo2"]))
    ns = A.n_spheres
    costs = np.zeros(m)
    terms = np.zeros((m, 6))
    flags = np.zeros(m, np.uint8)
    tq = np.zeros((m, h + 1, n)) if store_traj else None
    tqd = np.zeros((m, h + 1, n)) if store_traj else None
    sp = np.zeros((m, h, ns, 3)) if store_spheres else None
    lib().vpo_evaluate_batch(
        ctypes.byref(A), _ptr(controls), m, h, _ptr(costs), _ptr(terms), _ptr(flags),
        None if tq is None else _ptr(tq), None if tqd is None else _ptr(tqd),
        None if sp is None else _ptr(sp),
    )
    return {"costs": costs, "terms": terms, "flags": flags, "traj_q": tq, "traj_qd": tqd,
            "sphere_pos": sp}


def soft_weights(costs, lam):
    """vp/planner.py:373-384 (same validation errors)."""
    costs = _c(costs)
    if costs.size == 0:
        raise ValueError("cost batch is empty")
    if not np.isfinite(costs).all():
        raise ValueError("costs must be finite")
    if lam <= 0.0:
        raise ValueError(f"temperature must be positive, got {lam}")
    w = np.empty_like(costs)
    lib().vpo_soft_weights(_ptr(costs), costs.shape[0], float(lam), _ptr(w))
    return w


def update_controls(nominal, eps, w):
    """vp/planner.py:387-400 (weight-sum check raised by the caller's wrapper)."""
    nominal, eps, w = _c(nominal), _c(eps), _c(w)
    out = np.empty_like(nominal)
    m = eps.shape[0]
    lib().vpo_update_controls(_ptr(nominal), _ptr(eps), _ptr(w), m, nominal.size, _ptr(out))
    return out


def cpu_count() -> int:
    return int(lib().vpo_max_threads()) if _lib is not None or _LIB_PATH.exists() else (os.cpu_count() or 1)


# ---------------------------------------------------------------------------
# sampler + full step (vp/planner.py:182-219, :594-630) -- numpy restatement
# ---------------------------------------------------------------------------
def smoothing_matrix(horizon: int, window: int) -> np.ndarray:
    """vp/planner.py:182-196."""
    if window <= 1:
        return np.eye(horizon)
    back, fwd = (window - 1) // 2, window // 2
    a = np.zeros((horizon, horizon))
    for k in range(horizon):
        lo, hi = max(0, k - back), min(horizon, k + fwd + 1)
        a[k, lo:hi] = 1.0
        a[k] /= np.sqrt(hi - lo)
    return a


def sample_perturbations(samples: int, horizon: int, dof: int, sigma, window: int, rng_seed: int) -> np.ndarray:
    """vp/planner.py:199-219: per-sample Philox stream keyed by (seed, m),
    sample 0 = 0, moving-average smoothing, times sigma."""
    eps = np.empty((samples, horizon, dof))
    eps[0] = 0.0
    seed = int(rng_seed) & 0xFFFFFFFFFFFFFFFF
    for m in range(1, samples):
        gen = np.random.Generator(np.random.Philox(key=np.array([seed, m], dtype=np.uint64)))
        eps[m] = gen.standard_normal((horizon, dof))
    if window > 1 and samples > 1:
        eps = np.einsum("hk,mkn->mhn", smoothing_matrix(horizon, window), eps)
    eps *= np.broadcast_to(np.asarray(sigma, dtype=float), (dof,))
    return eps


def smpc_step(args: dict, nominal, eps, lam: float, acc_limits):
    """vp/planner.py:594-630 without the host FK diagnostics: evaluate ->
    soft_weights -> update_controls -> re-evaluate U* -> clip/shift."""
    nominal = _c(nominal)
    controls = nominal[None] + eps
    res = evaluate_batch(args, controls)
    if res["flags"].any():
        raise ValueError("degenerate rotation")
    w = soft_weights(res["costs"], lam)
    if abs(w.sum() - 1.0) > 1e-9:
        raise ValueError("weights do not sum to one")
    u = update_controls(nominal, eps, w)
    weighted = evaluate_batch(args, u[None])
    command = np.clip(u[0], -np.asarray(acc_limits), np.asarray(acc_limits))
    next_nominal = np.vstack([u[1:], np.zeros((1, u.shape[1]))])
    return {"u": u, "command": command, "next_nominal": next_nominal, "costs": res["costs"],
            "weighted_cost": float(weighted["costs"][0]), "weighted_terms": weighted["terms"][0],
            "best_cost": float(res["costs"].min())}


# ---------------------------------------------------------------------------
# sharded softmin protocol -- checker for the N-rank
# exchange: per-rank partial, then the fixed rank-order log-sum-exp merge.
# ---------------------------------------------------------------------------
def smpc_partial(costs, eps, lam: float, m_offset: int = 0) -> np.ndarray:
    """[m_r, Z_r, nonfinite_r, best_index_r, N_r (H n)] of one shard."""
    costs = _c(costs)
    eps = np.asarray(eps, dtype=np.float64)
    fin = np.isfinite(costs)
    m = costs[fin].min() if fin.any() else np.inf
    w = np.where(fin, np.exp(-(costs - m) / lam), 0.0) if np.isfinite(m) else np.zeros_like(costs)
    best = float(m_offset + int(np.argmin(np.where(fin, costs, np.inf)))) if fin.any() else -1.0
    n_r = np.einsum("m,mk->k", w, eps.reshape(eps.shape[0], -1))
    return np.concatenate([[m, w.sum(), float((~fin).sum()), best], n_r])


def merge_partials(parts, lam: float):
    """Merge rank partials in rank order -> (min, Z, nonfinite, best, N/Z)."""
    parts = np.asarray(parts, dtype=np.float64)
    m = parts[:, 0].min()
    scale = np.exp(-(parts[:, 0] - m) / lam)
    z = float((parts[:, 1] * scale).sum())
    n = (parts[:, 4:] * scale[:, None]).sum(axis=0)
    r_best = int(np.argmin(parts[:, 0]))
    return m, z, float(parts[:, 2].sum()), parts[r_best, 3], n / z
