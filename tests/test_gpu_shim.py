"""The reference-side binding (integration/voxplan_shim.py) end to end.

1. `install()` on a stub namespace shaped like the voxplan package (the
   module attributes the shim rebinds), then every rebound seam
   is driven with the reference's golden inputs and checked against the
   reference's golden outputs -- the 29-argument `_fuse_voxels`, `edt_3d`,
   the 49-argument `evaluate_batch`, `soft_weights`, `update_controls`.
   Needs no reference on the box.
2. When the reference is installed in baseline/_ref (pip --target, untracked;
   see DESIGN.md), `install()` on the real package and a closed-loop episode
   of `run_episode` (vp/sim.py:420-548) with the seams rebound against the
   stock one: EpisodeLog records with timing stripped (`strip_timing_fields`,
   vp/sim.py:57-69), structurally equal and numerically within the stated
   tolerance.
"""

import dataclasses
import os
import sys
import types
from pathlib import Path

import numpy as np
import pytest

from conftest import i32_to_sq, load_golden, unpack_occ

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = Path(__file__).resolve().parents[1]
ROLLOUT_KEYS = (
    "q0 qd0 controls dt base_r base_t off_r off_t axes sph_link sph_loc sph_r pairs goal_r goal_t "
    "pose_weight terminal_weight pos_lo pos_hi vel_lo vel_hi acc_lo acc_hi w_env w_self w_q "
    "w_qd w_qdd w_s w_ns d_act q_ref field_sq field_lo0 field_lo1 field_lo2 field_origin0 "
    "field_origin1 field_origin2 field_voxel field_outside"
).split()


@pytest.fixture(scope="module")
def shim():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, str(ROOT / "integration"))
    import voxplan_shim

    return voxplan_shim


# ----------------------------------------------------------------------------- stub package
@dataclasses.dataclass(frozen=True)
class _Box:
    lo: tuple
    hi: tuple


@dataclasses.dataclass
class _Params:
    l_occ_threshold: float = 1.0


class _Grid:
    """The attributes edt_3d reads from a vp/mapping.py VoxelGrid."""

    def __init__(self, log_odds, origin=(0.0, 0.0, 0.0), voxel=0.1):
        self.log_odds = log_odds
        self.dims = log_odds.shape
        self.origin = np.asarray(origin, float)
        self.voxel_size = voxel
        self.params = _Params()

    def full_box(self):
        return _Box((0, 0, 0), self.dims)

    def validate_box(self, box):
        assert all(0 <= l < h <= d for l, h, d in zip(box.lo, box.hi, self.dims))


@dataclasses.dataclass(frozen=True)
class _DistanceField:
    origin: np.ndarray
    voxel_size: float
    dims: tuple
    volume: _Box
    sq: np.ndarray
    outside_default: float


class _WeightMismatch(Exception):
    pass


def _stub():
    return types.SimpleNamespace(
        mapping=types.SimpleNamespace(_fuse_voxels=None, edt_3d=None, DistanceField=_DistanceField),
        batch=types.SimpleNamespace(evaluate_batch=None),
        planner=types.SimpleNamespace(soft_weights=None, update_controls=None),
        errors=types.SimpleNamespace(WeightMismatch=_WeightMismatch),
    )


def test_install_rebinds_every_seam(shim):
    vp = _stub()
    shim.install(vp)
    for mod, name in (("mapping", "_fuse_voxels"), ("mapping", "edt_3d"), ("batch", "evaluate_batch"),
                      ("planner", "soft_weights"), ("planner", "update_controls")):
        assert callable(getattr(getattr(vp, mod), name)), f"{mod}.{name} not rebound"


def test_fuse_seam_golden(shim):
    """_fuse_voxels with the reference's 29 positional arguments (vp/mapping.py:267-297),
    in place, on the golden fusion sequences: bitwise log_odds / observed."""
    vp = _stub()
    shim.install(vp)
    g = load_golden("fusion")
    for i in range(int(g["f_count"])):
        name = str(g[f"f_name_{i}"])
        dims = tuple(int(v) for v in g[f"f_dims_{i}"])
        voxel = float(g[f"f_voxel_{i}"])
        origin = g[f"f_origin_{i}"]
        fx, fy, cx, cy, dmin, dmax = (float(v) for v in g[f"f_cam{i}_intr"])
        w, h = (int(v) for v in g[f"f_cam{i}_wh"])
        lo, hi = (g[f"f_box_{i}"] if f"f_box_{i}" in g else (np.zeros(3, np.int64), np.array(dims)))
        n = hi - lo
        log_odds = np.zeros(dims)
        observed = np.zeros(dims, bool)
        for s in range(int(g[f"f_nsteps_{i}"])):
            if f"f_mc_{i}_{s}" in g:
                mc, mr = g[f"f_mc_{i}_{s}"], g[f"f_mr_{i}_{s}"]
            else:
                mc, mr = np.zeros((0, 3)), np.zeros(0)
            vp.mapping._fuse_voxels(log_odds, observed, int(lo[0]), int(lo[1]), int(lo[2]), int(n[0]), int(n[1]),
                                    int(n[2]), origin, voxel, g[f"f_cam{i}_w2c_r"], g[f"f_cam{i}_w2c_t"], fx, fy, cx,
                                    cy, w, h, dmin, dmax, g[f"f_depth_{i}_{s}"], g[f"f_pm_{i}_{s}"], mc, mr,
                                    2.5 * voxel, 0.85, -0.4, -2.0, 3.5)
            np.testing.assert_array_equal(log_odds, g[f"f_lo_{i}_{s}"], err_msg=f"{name} step {s}")
            np.testing.assert_array_equal(observed, g[f"f_ob_{i}_{s}"], err_msg=f"{name} step {s}")


def test_edt_seam_golden(shim):
    """edt_3d(grid, volume) through the seam: the reference's DistanceField type, bit-exact sq."""
    vp = _stub()
    shim.install(vp)
    g = load_golden("edt")
    for i in range(int(g["edt_count"])):
        occ = unpack_occ(g[f"edt_occ_{i}"], g[f"edt_dims_{i}"])
        grid = _Grid(np.where(occ, 3.5, 0.0))
        box = _Box(tuple(int(v) for v in g[f"edt_lo_{i}"]), tuple(int(v) for v in g[f"edt_hi_{i}"]))
        field = vp.mapping.edt_3d(grid, box, outside_default=0.8)
        assert isinstance(field, _DistanceField) and field.volume == box and field.outside_default == 0.8
        np.testing.assert_array_equal(field.sq, i32_to_sq(g[f"edt_sq_{i}"]), err_msg=str(g[f"edt_name_{i}"]))


def test_evaluate_batch_seam_golden(shim):
    """evaluate_batch with the reference's 49 positional arguments (vp/batch.py:162-212),
    caller-allocated outputs written in place: fp64 parity mode, rtol 1e-9."""
    vp = _stub()
    shim.install(vp)
    g = load_golden("rollout")
    for i in range(int(g["r_count"])):
        name = str(g[f"r_name_{i}"])
        a = {k: g[f"r_{k}_{i}"] for k in ROLLOUT_KEYS}
        a["field_sq"] = i32_to_sq(a["field_sq"])
        store = bool(g[f"r_store_{i}"])
        m, hz, n = a["controls"].shape
        ns = a["sph_r"].shape[0]
        costs, terms = np.empty(m), np.empty((m, 6))
        flags = np.empty(m, np.uint8)
        tq = np.empty((m, hz + 1, n)) if store else np.empty((1, 1, 1))
        tqd = np.empty((m, hz + 1, n)) if store else np.empty((1, 1, 1))
        sp = np.empty((m, hz, ns, 3)) if store else np.empty((1, 1, 1, 1))
        vp.batch.evaluate_batch(*[a[k] for k in ROLLOUT_KEYS], store, store, costs, terms, tq, tqd, sp, flags)
        np.testing.assert_array_equal(flags, g[f"r_flags_{i}"], err_msg=name)
        ok = flags == 0
        np.testing.assert_allclose(costs[ok], g[f"r_costs_{i}"][ok], rtol=1e-9, err_msg=name)
        np.testing.assert_allclose(terms[ok], g[f"r_terms_{i}"][ok], rtol=1e-9, atol=1e-12, err_msg=name)
        if store:
            np.testing.assert_allclose(tq, g[f"r_trajq_{i}"], rtol=1e-11, atol=1e-13, err_msg=name)
            np.testing.assert_allclose(sp, g[f"r_sphpos_{i}"], rtol=1e-11, atol=1e-13, err_msg=name)


def test_softmin_update_seams_golden(shim):
    vp = _stub()
    shim.install(vp)
    g = load_golden("softmin")
    for i in range(int(g["s_count"])):
        w = vp.planner.soft_weights(g[f"s_costs_{i}"], float(g[f"s_lam_{i}"]))
        np.testing.assert_allclose(w, g[f"s_w_{i}"], rtol=1e-12, atol=1e-300)
        u = vp.planner.update_controls(g[f"s_nom_{i}"], g[f"s_eps_{i}"], g[f"s_w_{i}"])
        np.testing.assert_allclose(u, g[f"s_u_{i}"], rtol=1e-12, atol=1e-14)
    with pytest.raises(_WeightMismatch):  # re-raised as the reference's own type
        vp.planner.update_controls(np.zeros((2, 2)), np.zeros((3, 2, 2)), np.full(3, 0.5))


# ----------------------------------------------------------------------------- the real package
REF = ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def voxplan():
    if not (REF / "voxplan").is_dir():
        pytest.skip("reference not installed in baseline/_ref (see DESIGN.md: pip install --target)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
    sys.path.insert(0, str(REF))
    try:
        import voxplan  # noqa: F401
        import voxplan.sim  # noqa: F401
    except ImportError as exc:  # e.g. numba missing on the box
        pytest.skip(f"reference not importable: {exc}")
    import voxplan

    return voxplan


SEAMS = (("mapping", "_fuse_voxels"), ("mapping", "edt_3d"), ("batch", "evaluate_batch"),
         ("planner", "soft_weights"), ("planner", "update_controls"))


def _flat(doc, prefix=""):
    out = {}
    for k, v in doc.items():
        if isinstance(v, dict):
            out.update(_flat(v, f"{prefix}{k}."))
        else:
            out[prefix + k] = v
    return out


def test_episode_log_matches_reference(shim, voxplan, tmp_path):
    """run_episode on the reach_static scenario, stock vs seams rebound.
    Mapping is bit-exact and the planner runs the fp64 kernels (costs within
    a few ulp), but the closed loop feeds every command back into the next
    state and the softmin weights amplify cost differences by |S| / lam
    (SURVEY.md 7.3-5): a last-ulp difference grows ~1.6x per cycle
    (profiles/r2_episode_divergence.json, tools/episode_diff.py: 1e-16 at
    cycle 0, 1e-9 by cycle 60, 1e-4 by cycle 95 -- the episode is chaotic, not
    the kernels inexact).  So the comparison covers 60 cycles: every discrete
    field (cycle, goal index, goal cycles, success) exactly, every continuous
    field at rtol 1e-6 with an absolute floor of 1e-9."""
    import json

    from voxplan import parallel
    from voxplan.config import bundled_scenario_path, load_scenario
    from voxplan.sim import run_episode, strip_timing_fields, write_episode_log

    parallel.set_threads(8)
    scn = dataclasses.replace(load_scenario(bundled_scenario_path("reach_static")), timeout_cycles=60)
    ref_log = run_episode(scn)
    saved = {(m, n): getattr(getattr(voxplan, m), n) for m, n in SEAMS}
    try:
        shim.install(voxplan)
        gpu_log = run_episode(scn)
    finally:
        for (m, n), f in saved.items():
            setattr(getattr(voxplan, m), n, f)

    def docs(log, name):
        p = tmp_path / f"{name}.ndjson"
        write_episode_log(log, p)
        return [strip_timing_fields(json.loads(line)) for line in p.read_text().splitlines() if line.strip()]

    a, b = docs(ref_log, "ref"), docs(gpu_log, "gpu")
    assert len(a) == len(b)
    worst = {}
    for ra, rb in zip(a, b):
        fa, fb = _flat(ra), _flat(rb)
        assert fa.keys() == fb.keys()
        for k in fa:
            va, vb = fa[k], fb[k]
            if isinstance(va, (int, bool, str)) or va is None:
                assert va == vb, f"{k}: {va} != {vb}"
            else:
                x, y = np.asarray(va, float), np.asarray(vb, float)
                fin = np.isfinite(x)
                np.testing.assert_array_equal(np.isfinite(y), fin, err_msg=k)
                d = np.abs(x[fin] - y[fin]) / np.maximum(np.abs(x[fin]), 1e-3)
                worst[k] = max(worst.get(k, 0.0), float(np.max(d, initial=0.0)))
                np.testing.assert_allclose(y[fin], x[fin], rtol=1e-6, atol=1e-9, err_msg=k)
    print("\nEpisodeLog records:", len(a), "cycles; worst deviation |d| / max(|ref|, 1e-3) per field:",
          json.dumps(worst, sort_keys=True))
