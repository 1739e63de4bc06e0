"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU
and exports every entry point include/vpb200.h declares (no compute calls)."""

import ctypes
import re
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_2512_22575_b200 import _lib, build

    build.build()
    return _lib.load()


def header_functions():
    text = (ROOT / "include" / "vpb200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*[a-z_0-9 ]+?\*?\s*\b(vpb_[a-z0-9_]+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = header_functions()
    for want in ("vpb_fuse_voxels", "vpb_masked_pixels", "vpb_edt3d", "vpb_query_distance",
                 "vpb_evaluate_batch", "vpb_soft_weights", "vpb_update_controls", "vpb_smpc_partial",
                 "vpb_smpc_finish", "vpb_sample_perturbations"):
        assert want in names


def test_library_exports_every_header_symbol(lib):
    from paper_2512_22575_b200 import _lib

    for name in header_functions():
        assert hasattr(lib, name), f"{name} declared in vpb200.h but not exported"
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_library_is_sm100a(lib):
    from paper_2512_22575_b200 import _lib
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_pure_host_entry_points(lib):
    """Size queries are host-only and callable without a device."""
    from paper_2512_22575_b200._lib import i64x3

    assert lib.vpb_version() == 1
    assert lib.vpb_occ_words(i64x3((4, 5, 33))) == 4 * 5 * 2
    assert lib.vpb_edt3d_workspace_bytes(i64x3((8, 8, 8))) >= 8 * 8 * 8 * 6
    assert lib.vpb_smpc_partial_len(32, 7) == 4 + 224 + 7
    assert lib.vpb_smpc_out_len(32, 7) == 2 * 224 + 7 + 13
    # argument checks run before any CUDA call; a zero-byte upload is a no-op
    assert lib.vpb_stage_h2d(None, None, None, 16, None) == 1  # VPB_ERR_ARG
    assert b"vpb_stage_h2d" in lib.vpb_last_error()
    assert lib.vpb_stage_h2d(None, None, None, 0, None) == 0
    assert lib.vpb_pixel_scratch_bytes(160, 120) >= 160 * 120 * 5 + 64  # class byte + fp32 depth + rectangle slots


def test_struct_layout_matches_header(lib):
    """ctypes mirrors of the C structs have the C sizes (compiled probe)."""
    import subprocess, tempfile
    from paper_2512_22575_b200 import _lib

    src = '#include <stdio.h>\n#include "vpb200.h"\nint main(){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(vpb_camera), sizeof(vpb_map_params), sizeof(vpb_grid), sizeof(vpb_field), sizeof(vpb_problem), sizeof(vpb_journal));}'
    with tempfile.TemporaryDirectory() as d:
        c = Path(d) / "probe.c"
        c.write_text(src)
        exe = Path(d) / "probe"
        r = subprocess.run(["gcc", "-I", str(ROOT / "include"), str(c), "-o", str(exe)], capture_output=True, text=True)
        if r.returncode != 0:
            pytest.skip("no C compiler")
        sizes = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(t) for t in (_lib.VpbCamera, _lib.VpbMapParams, _lib.VpbGrid, _lib.VpbField, _lib.VpbProblem,
                                       _lib.VpbJournal)]
    assert sizes == want


def test_product_has_no_cpu_fallback():
    """Without CUDA the product path raises instead of computing on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2512_22575_b200 import mapping
    from paper_2512_22575_b200._lib import NativeError

    with pytest.raises(NativeError):
        mapping.VoxelGrid((0, 0, 0), 0.1, (4, 4, 4))


def test_product_never_imports_oracle():
    for path in (ROOT / "paper_2512_22575_b200").rglob("*.py"):
        text = path.read_text()
        assert "import oracle" not in text and "from oracle" not in text, path


def test_reference_shim_packs_like_planner():
    """integration/voxplan_shim.py packs evaluate_batch's flat arguments
    (vp/batch.py:162-195) into the same vpb_problem block as Planner."""
    import ctypes

    import numpy as np

    sys_path_root = str(ROOT / "integration")
    if sys_path_root not in sys.path:
        sys.path.insert(0, sys_path_root)
    import voxplan_shim
    from paper_2512_22575_b200 import config, planner

    chain, model = config.robot_7dof()
    params = config.planner_params(7, {"samples": 16, "horizon": 12})
    want = planner.pack_problem(chain, model, params)
    lims = planner.tightened_limits(chain, params.margin_frac)
    got = voxplan_shim.problem_from_reference_args(
        np.zeros(7), np.zeros(7), params.dt, chain.base_pose.rotation.matrix, chain.base_pose.translation,
        np.array([j.parent_offset.rotation.matrix for j in chain.joints]),
        np.array([j.parent_offset.translation for j in chain.joints]), np.array([j.axis for j in chain.joints]),
        np.array([s.link for s in model.spheres]), np.array([s.center for s in model.spheres]), model.radii(),
        np.array(model.self_pairs), np.eye(3), np.zeros(3), params.pose_weight, params.terminal_weight, *lims,
        params.w_env, params.w_self, params.w_q, params.w_qd, params.w_qdd, params.w_s, params.w_ns, params.d_act,
        params.q_ref, params.horizon)
    for name, _ in want._fields_:
        if name in ("acc_limit", "lam", "goal_r", "goal_t", "q0", "qd0", "dyn_state"):
            continue  # per-call / step-only fields the evaluate seam does not carry
        a, b = getattr(want, name), getattr(got, name)
        if isinstance(a, ctypes.Array):
            assert list(a) == list(b), name
        else:
            assert a == b, name


def test_host_ee_errors_vs_reference_golden():
    """vpb_ee_errors (host C, no GPU) reproduces the reference's smpc_step
    diagnostics e_pos / e_ori (vp/planner.py:620-629) from the golden steps."""
    import ctypes

    import numpy as np

    from conftest import load_golden
    from paper_2512_22575_b200 import _lib, config, planner

    lib = _lib.load()
    g = load_golden("softmin")
    chain, model = config.robot_7dof()
    P = planner.pack_problem(chain, model, config.planner_params(7))
    for j in range(int(g["st_count"])):
        q0 = np.ascontiguousarray(g[f"st_q0_{j}"], dtype=np.float64)
        gr = np.ascontiguousarray(g[f"st_goal_r_{j}"], dtype=np.float64)
        gt = np.ascontiguousarray(g[f"st_goal_t_{j}"], dtype=np.float64)
        ep, eo = ctypes.c_double(), ctypes.c_double()
        ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        assert lib.vpb_ee_errors(P, ptr(q0), ptr(gr), ptr(gt), ctypes.byref(ep), ctypes.byref(eo)) == 0
        diag = g[f"st_diag_{j}"]
        np.testing.assert_allclose(ep.value, diag[2], rtol=1e-12)
        np.testing.assert_allclose(eo.value, diag[3], rtol=1e-9, atol=1e-12)
