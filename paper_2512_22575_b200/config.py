"""Planner defaults and the benchmark robot, as data.

The values are the ones the reference actually runs with: its packaged
planner defaults (vp/data/planner_defaults.yaml:4-20, which differ from the
SPEC.md table -- SURVEY.md section 5) and its generic 7-DoF arm
(vp/data/robot_7dof.yaml:9-77).  ``planner_params`` mirrors
vp/config.py:53-83 (defaults + overrides, diagonal or full weights).
"""

from __future__ import annotations

import copy

import numpy as np

PLANNER_DEFAULTS = {
    "horizon": 30,
    "samples": 512,
    "dt": 0.02,
    "lam": 0.05,
    "sigma": 1.0,
    "noise_window": 5,
    "pose_weight_diag": [200.0, 200.0, 200.0, 80.0, 80.0, 80.0],
    "terminal_weight_diag": [2000.0, 2000.0, 2000.0, 800.0, 800.0, 800.0],
    "w_env": 50000.0,
    "w_self": 50000.0,
    "w_q": 100.0,
    "w_qd": 100.0,
    "w_qdd": 100.0,
    "w_s": 0.01,
    "w_ns": 0.1,
    "d_act": 0.05,
    "margin_frac": 0.02,
}

_PLANNER_KEYS = set(PLANNER_DEFAULTS) | {"pose_weight", "terminal_weight", "q_ref"}


def _joint(z_offset: float, axis, limit: float) -> dict:
    return {
        "offset": [0.0, 0.0, z_offset, 1.0, 0.0, 0.0, 0.0],
        "axis": list(axis),
        "position_limits": [-limit, limit],
        "velocity_limit": 2.5,
        "acceleration_limit": 10.0,
    }


_Z, _Y = (0.0, 0.0, 1.0), (0.0, 1.0, 0.0)

ROBOT_7DOF = {
    "schema_version": 1,
    "name": "generic_7dof",
    "base_pose": [0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0],
    "joints": [
        _joint(0.15, _Z, 2.9), _joint(0.10, _Y, 2.0), _joint(0.25, _Z, 2.9), _joint(0.15, _Y, 2.2),
        _joint(0.25, _Z, 2.9), _joint(0.10, _Y, 2.0), _joint(0.12, _Z, 2.9),
    ],
    "spheres": [
        {"link": link, "center": [0.0, 0.0, cz], "radius": r}
        for link, cz, r in [
            (0, 0.08, 0.09), (1, 0.05, 0.08), (2, 0.08, 0.08), (2, 0.17, 0.08), (3, 0.05, 0.07),
            (3, 0.11, 0.07), (4, 0.08, 0.07), (4, 0.17, 0.07), (5, 0.05, 0.06), (6, 0.06, 0.06),
            (7, 0.02, 0.05),
        ]
    ],
    "self_pairs": [[0, 6], [0, 7], [0, 8], [0, 9], [0, 10], [1, 6], [1, 7], [1, 9], [1, 10],
                   [2, 6], [2, 7], [2, 10], [3, 8], [3, 9], [3, 10], [4, 9], [4, 10], [5, 10]],
}


def robot_7dof():
    """(chain, sphere model) of the benchmark arm."""
    from .robot import robot_from_dict

    return robot_from_dict(copy.deepcopy(ROBOT_7DOF))


def _weight_matrix(doc: dict, key: str) -> np.ndarray:
    full = doc.get(key)
    if full is not None:
        return np.asarray(full, dtype=float)
    return np.diag(np.asarray(doc[f"{key}_diag"], dtype=float))


def planner_params(dof: int, overrides: dict | None = None):
    """PlannerParams from the defaults plus overrides (vp/config.py:53-83)."""
    from .planner import PlannerParams

    doc = copy.deepcopy(PLANNER_DEFAULTS)
    overrides = dict(overrides or {})
    unknown = set(overrides) - _PLANNER_KEYS
    if unknown:
        raise ValueError(f"unknown planner keys: {sorted(unknown)}")
    doc.update(overrides)
    q_ref = np.asarray(doc.get("q_ref", np.zeros(dof)), dtype=float)
    if q_ref.shape != (dof,):
        raise ValueError(f"q_ref must have {dof} entries, got {q_ref.shape}")
    return PlannerParams(
        horizon=int(doc["horizon"]), samples=int(doc["samples"]), dt=float(doc["dt"]),
        lam=float(doc["lam"]), sigma=np.asarray(doc["sigma"], dtype=float),
        noise_window=int(doc["noise_window"]),
        pose_weight=_weight_matrix(doc, "pose_weight"),
        terminal_weight=_weight_matrix(doc, "terminal_weight"),
        w_env=float(doc["w_env"]), w_self=float(doc["w_self"]), w_q=float(doc["w_q"]),
        w_qd=float(doc["w_qd"]), w_qdd=float(doc["w_qdd"]), w_s=float(doc["w_s"]),
        w_ns=float(doc["w_ns"]), d_act=float(doc["d_act"]), margin_frac=float(doc["margin_frac"]),
        q_ref=q_ref,
    )
