"""Shared test configuration.

`-m gpu` tests need a B200 and the in-tree CUDA library; everything else runs
on the CPU build container (oracle vs golden vectors, host logic, C-ABI
exports, gloo world-size-2 sharding logic).
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")


def load_golden(name: str):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


def unpack_occ(bits, dims):
    n = int(np.prod(dims))
    return np.unpackbits(bits)[:n].astype(bool).reshape(tuple(int(d) for d in dims))


def i32_to_sq(a):
    a = np.asarray(a)
    return np.where(a < 0, np.inf, a.astype(np.float64))


@pytest.fixture(scope="session")
def golden():
    return load_golden


def oracle_args(planner, chain, model, params, state, goal, field):
    """evaluate_batch's named inputs (vp/batch.py:162-212) for the oracle, from
    the same robot, objective, state, goal and field the GPU planner gets."""
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
    if field is None:
        args.update(field_sq=np.full((1, 1, 1), np.inf), field_lo0=2**40, field_lo1=2**40, field_lo2=2**40,
                    field_origin0=0.0, field_origin1=0.0, field_origin2=0.0, field_voxel=1.0, field_outside=np.inf)
    else:
        args.update(field_sq=field.sq, field_lo0=field.volume.lo[0], field_lo1=field.volume.lo[1],
                    field_lo2=field.volume.lo[2], field_origin0=field.origin[0], field_origin1=field.origin[1],
                    field_origin2=field.origin[2], field_voxel=field.voxel_size, field_outside=field.outside_default)
    return args
