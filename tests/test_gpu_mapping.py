"""GPU parity of the mapping kernels (fusion, masked pixels, EDT, query).

Bars: log_odds / observed / pixel mask bitwise equal; EDT
squared distances bit-exact (inf positions equal); query fp64 values equal.
Every comparison runs the CUDA path through the package API (C ABI) and checks
it against the reference's golden vectors and/or the CPU oracle on the same
seeded inputs.
"""

import numpy as np
import pytest

import oracle
from conftest import i32_to_sq, load_golden, unpack_occ

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def M():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_22575_b200 import mapping

    return mapping


def grid_from_occ(M, occ, voxel=0.1, origin=(0.0, 0.0, 0.0)):
    g = M.VoxelGrid(origin, voxel, occ.shape)
    g.set_log_odds(np.where(occ, g.params.l_max, 0.0))
    return g


# ----------------------------------------------------------------------------- EDT
def test_edt_golden_bit_exact(M):
    g = load_golden("edt")
    for i in range(int(g["edt_count"])):
        occ = unpack_occ(g[f"edt_occ_{i}"], g[f"edt_dims_{i}"])
        grid = grid_from_occ(M, occ)
        box = M.VoxelBox(tuple(g[f"edt_lo_{i}"]), tuple(g[f"edt_hi_{i}"]))
        field = M.edt_3d(grid, box)
        np.testing.assert_array_equal(field.sq, i32_to_sq(g[f"edt_sq_{i}"]), err_msg=str(g[f"edt_name_{i}"]))


def test_edt_threshold_boundary(M):
    g = load_golden("edt")
    grid = M.VoxelGrid((0, 0, 0), 0.1, g["thr_log_odds"].shape)
    grid.set_log_odds(g["thr_log_odds"])
    np.testing.assert_array_equal(M.edt_3d(grid).sq, i32_to_sq(g["thr_sq"]))


@pytest.mark.parametrize("dims,density,seed", [
    ((64, 64, 64), 0.01, 1), ((64, 64, 64), 0.3, 2), ((37, 91, 45), 0.02, 3), ((128, 96, 80), 0.001, 4),
    ((200, 3, 150), 0.01, 5), ((1, 300, 7), 0.05, 6), ((70, 70, 33), 0.0, 7),
])
def test_edt_random_vs_oracle(M, dims, density, seed):
    occ = np.random.default_rng(seed).random(dims) < density
    grid = grid_from_occ(M, occ)
    got = M.edt_3d(grid).sq
    np.testing.assert_array_equal(got, oracle.edt3d_from_occupancy(occ))


def test_edt_subvolumes_vs_oracle(M):
    rng = np.random.default_rng(11)
    occ = rng.random((50, 61, 77)) < 0.01
    grid = grid_from_occ(M, occ)
    lo_odds = np.where(occ, 3.5, 0.0)
    for lo, hi in [((0, 0, 0), (50, 61, 77)), ((3, 5, 7), (40, 60, 70)), ((10, 0, 33), (11, 61, 65)),
                   ((0, 17, 31), (50, 18, 77)), ((7, 7, 1), (49, 60, 2))]:
        got = M.edt_3d(grid, M.VoxelBox(lo, hi)).sq
        np.testing.assert_array_equal(got, oracle.edt3d(lo_odds, lo, hi), err_msg=f"{lo} {hi}")


def test_edt_256_single_source_analytic(M):
    """Size-independent check at the C2 size: one source -> exact |d|^2."""
    n = 256
    occ = np.zeros((n, n, n), bool)
    src = (17, 200, 131)
    occ[src] = True
    got = M.edt_3d(grid_from_occ(M, occ)).sq_device
    idx = [torch.arange(n, device=got.device, dtype=torch.float32) - s for s in src]
    want = idx[0][:, None, None] ** 2 + idx[1][None, :, None] ** 2 + idx[2][None, None, :] ** 2
    assert torch.equal(got, want)


def test_edt_256_random_vs_oracle(M):
    """Full C2 size against the oracle (bit-exact)."""
    occ = np.random.default_rng(2024).random((256, 256, 256)) < 0.01
    got = M.edt_3d(grid_from_occ(M, occ)).sq
    oracle.set_threads(0)
    np.testing.assert_array_equal(got, oracle.edt3d_from_occupancy(occ))


def test_edt_512_properties(M):
    """C5 size: sources reproduce 0, growth is monotone, and the field is
    1-Lipschitz in distance between face neighbours (size-independent)."""
    n = 512
    rng = np.random.default_rng(9)
    pts = rng.integers(0, n, size=(40, 3))
    occ = torch.zeros((n, n, n), dtype=torch.bool, device="cuda")
    occ[pts[:, 0], pts[:, 1], pts[:, 2]] = True
    grid = M.VoxelGrid((0, 0, 0), 0.02, (n, n, n))
    grid.set_log_odds(torch.where(occ, 3.5, 0.0).double())
    a = M.edt_3d(grid).sq_device
    assert bool((a[occ] == 0).all())
    # exact value at a few voxels by brute force over the 40 sources
    probe = rng.integers(0, n, size=(200, 3))
    d2 = ((probe[:, None, :] - pts[None, :, :]) ** 2).sum(-1).min(1)
    got = a[probe[:, 0], probe[:, 1], probe[:, 2]].cpu().numpy()
    np.testing.assert_array_equal(got, d2.astype(np.float32))
    d = a.sqrt()
    for ax in range(3):
        diff = (d.narrow(ax, 1, n - 1) - d.narrow(ax, 0, n - 1)).abs()
        assert float(diff.max()) <= 1.0 + 1e-5
    grid.log_odds[5, 5, 5] = 3.5
    b = M.edt_3d(grid).sq_device
    assert bool((b <= a).all())


def test_edt_acceptance_100_grids(M):
    """All 100 grids of acceptance criterion 1 (t/test_acceptance.py:57-81),
    against the reference's own outputs (tests/golden/edt_acceptance.npz)."""
    g = load_golden("edt_acceptance")
    for i in range(g["occ"].shape[0]):
        occ = unpack_occ(g["occ"][i], (16, 16, 16))
        np.testing.assert_array_equal(M.edt_3d(grid_from_occ(M, occ)).sq, i32_to_sq(g["sq"][i]), err_msg=f"grid {i}")


@pytest.mark.parametrize("dims,density,seed", [
    ((600, 40, 32), 0.002, 21),   # x > 512: the 64-bit (WIDE) X pass
    ((40, 600, 32), 0.002, 22),   # y > 512: the 64-bit (WIDE) Z+Y pass
    ((24, 24, 1100), 0.001, 23),  # z > 1024: bit-scan Z pass + the generic FH passes
    ((1100, 8, 8), 0.002, 24),    # x > 1024: the generic (non-tiled) FH pass
    ((8, 1100, 8), 0.002, 25),    # y > 1024
    ((600, 40, 30), 0.003, 26),   # z % 4 != 0 with x > 512: the tile-per-line fallback
    ((1030, 3, 5), 0.0, 27),      # empty, long
])
def test_edt_long_lines_vs_oracle(M, dims, density, seed):
    occ = np.random.default_rng(seed).random(dims) < density
    if density > 0:
        occ[0, 0, 0] = occ[-1, -1, -1] = True  # sources at both ends of the longest lines
    got = M.edt_3d(grid_from_occ(M, occ)).sq
    oracle.set_threads(0)
    np.testing.assert_array_equal(got, oracle.edt3d_from_occupancy(occ))


@pytest.mark.parametrize("density", [0.001, 0.1, 0.5])
def test_edt_512_random_vs_oracle(M, density):
    """C5 size, bit-exact against the oracle over the whole 512^3 field."""
    occ = np.random.default_rng(512).random((512, 512, 512), dtype=np.float32) < density
    got = M.edt_3d(grid_from_occ(M, occ)).sq_device.cpu().numpy()
    oracle.set_threads(0)
    want = oracle.edt3d_from_occupancy(occ)
    assert np.array_equal(got.astype(np.float64), want)


@pytest.mark.parametrize("density", [0.1, 0.5])
def test_edt_256_densities_vs_oracle(M, density):
    occ = np.random.default_rng(256).random((256, 256, 256)) < density
    got = M.edt_3d(grid_from_occ(M, occ)).sq
    oracle.set_threads(0)
    np.testing.assert_array_equal(got, oracle.edt3d_from_occupancy(occ))


# ----------------------------------------------------------------------------- fusion
def _camera(M, g, i):
    from paper_2512_22575_b200.geometry import RigidTransform, Rotation3

    fx, fy, cx, cy, dmin, dmax = (float(v) for v in g[f"f_cam{i}_intr"])
    w, h = (int(v) for v in g[f"f_cam{i}_wh"])
    pose = RigidTransform(Rotation3(g[f"f_cam{i}_pose_r"]), g[f"f_cam{i}_pose_t"])
    return M.CameraModel(fx, fy, cx, cy, w, h, dmin, dmax, pose=pose)


def test_fusion_golden_bitwise(M):
    g = load_golden("fusion")
    for i in range(int(g["f_count"])):
        name = str(g[f"f_name_{i}"])
        dims = tuple(int(v) for v in g[f"f_dims_{i}"])
        grid = M.VoxelGrid(g[f"f_origin_{i}"], float(g[f"f_voxel_{i}"]), dims)
        cam = _camera(M, g, i)
        r, t = cam.world_to_camera()
        np.testing.assert_array_equal(r, g[f"f_cam{i}_w2c_r"])
        np.testing.assert_array_equal(t, g[f"f_cam{i}_w2c_t"])
        box = M.VoxelBox(*g[f"f_box_{i}"]) if f"f_box_{i}" in g else None
        for s in range(int(g[f"f_nsteps_{i}"])):
            depth = M.DepthImage(g[f"f_depth_{i}_{s}"])
            mask = (g[f"f_mc_{i}_{s}"], g[f"f_mr_{i}_{s}"]) if f"f_mc_{i}_{s}" in g else None
            if mask is not None:
                pm = M.masked_pixels(depth, cam, mask[0], mask[1], float(g[f"f_pad_{i}"]))
                np.testing.assert_array_equal(pm.cpu().numpy(), g[f"f_pm_{i}_{s}"], err_msg=f"{name} {s}")
            M.update_occupancy(grid, depth, cam, mask=mask, volume=box, mask_pad=float(g[f"f_pad_{i}"]))
            np.testing.assert_array_equal(grid.log_odds_host(), g[f"f_lo_{i}_{s}"], err_msg=f"{name} step {s}")
            np.testing.assert_array_equal(grid.observed_host(), g[f"f_ob_{i}_{s}"], err_msg=f"{name} step {s}")


def test_fusion_random_frames_vs_oracle(M):
    """Bench-style 72x80x96 grid, 7-DoF mask, moving cameras and boxes,
    8 frames: bitwise log_odds/observed and a consistent occupancy mask."""
    from paper_2512_22575_b200 import config, robot, scene
    from paper_2512_22575_b200.geometry import RigidTransform, Rotation3

    chain, model = config.robot_7dof()
    rng = np.random.default_rng(5)
    dims = (72, 80, 96)
    grid = M.VoxelGrid((-0.7, -0.8, 0.0), 0.02, dims)
    lo = np.zeros(dims)
    ob = np.zeros(dims, bool)
    box = M.VoxelBox((3, 0, 17), (70, 80, 90))
    for frame in range(8):
        q = rng.uniform(-1.0, 1.0, size=7)
        centers, radii = robot.sphere_positions(chain, q, model)
        yaw = rng.uniform(-0.3, 0.3)
        pose = RigidTransform(Rotation3.rot_y(yaw), (rng.uniform(-0.2, 0.2), rng.uniform(-0.2, 0.2), -1.0))
        cam = M.CameraModel(120.0, 118.0, 79.5, 59.5, 160, 120, 0.05, 20.0, pose=pose)
        c = rng.uniform([-0.3, -0.3, 0.6], [0.3, 0.3, 1.4])
        depth_np = scene.render_boxes(cam, [(c - 0.2, c + 0.2)], (centers, radii))
        depth = M.DepthImage(depth_np)
        M.update_occupancy(grid, depth, cam, mask=(centers, radii), volume=box)
        pm = oracle.masked_pixels(depth_np, cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max,
                                  cam.pose.rotation.matrix, cam.pose.translation, centers, radii, 0.01)
        r, t = cam.world_to_camera()
        oracle.fuse_voxels(lo, ob, box.lo, box.shape, grid.origin, grid.voxel_size, r, t, cam.fx, cam.fy, cam.cx,
                           cam.cy, cam.width, cam.height, cam.d_min, cam.d_max, depth_np, pm, centers, radii,
                           grid.tau, 0.85, -0.4, -2.0, 3.5)
        np.testing.assert_array_equal(grid.log_odds_host(), lo, err_msg=f"frame {frame}")
        np.testing.assert_array_equal(grid.observed_host(), ob, err_msg=f"frame {frame}")
    # occupancy mask maintained by the fusion kernel
    bits = grid._occ_bits.cpu().numpy().view(np.uint32)
    occ = lo >= 1.0
    wz = (dims[2] + 31) // 32
    want = np.zeros((dims[0], dims[1], wz), np.uint64)
    for z in range(dims[2]):
        want[:, :, z // 32] |= occ[:, :, z].astype(np.uint64) << np.uint64(z % 32)
    np.testing.assert_array_equal(bits.reshape(dims[0], dims[1], wz), want.astype(np.uint32))
    # EDT straight from the maintained mask equals the oracle on the log-odds
    mapper_field = M.edt_3d(grid)
    np.testing.assert_array_equal(mapper_field.sq, oracle.edt3d(lo))


def test_fusion_rectangle_slots_alternate(M):
    """The usable-pixel rectangle lives in two scratch slots that alternate per
    call (each call clears the other): frames whose rectangles shrink, vanish
    (no valid return) and grow again must each fuse exactly like the oracle."""
    from paper_2512_22575_b200 import config, robot, scene
    from paper_2512_22575_b200.geometry import RigidTransform, Rotation3

    chain, model = config.robot_7dof()
    dims = (64, 64, 80)
    grid = M.VoxelGrid((-0.64, -0.64, 0.0), 0.02, dims)
    lo = np.zeros(dims)
    ob = np.zeros(dims, bool)
    box = grid.full_box()
    centers, radii = robot.sphere_positions(chain, np.full(7, 0.2), model)
    pose = RigidTransform(Rotation3.rot_y(0.1), (0.0, 0.0, -1.0))
    cam = M.CameraModel(120.0, 118.0, 79.5, 59.5, 160, 120, 0.05, 20.0, pose=pose)
    boxes = [[((-0.1, -0.1, 0.7), (0.1, 0.1, 0.9))],           # small, near
             None,                                              # no valid return at all
             [((-0.6, -0.6, 1.2), (0.6, 0.6, 1.5))],           # wide, far
             [((0.2, 0.1, 0.8), (0.3, 0.25, 0.95))],           # small, off-centre
             None,
             None,
             [((-0.3, -0.5, 0.9), (0.5, 0.2, 1.3))]]
    for frame, bx in enumerate(boxes):
        if bx is None:
            depth_np = np.zeros((cam.height, cam.width))  # below d_min everywhere
        else:
            depth_np = scene.render_boxes(cam, [(np.array(a), np.array(b)) for a, b in bx], (centers, radii))
        M.update_occupancy(grid, M.DepthImage(depth_np), cam, mask=(centers, radii), volume=box)
        pm = oracle.masked_pixels(depth_np, cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max,
                                  cam.pose.rotation.matrix, cam.pose.translation, centers, radii, 0.01)
        r, t = cam.world_to_camera()
        oracle.fuse_voxels(lo, ob, box.lo, box.shape, grid.origin, grid.voxel_size, r, t, cam.fx, cam.fy, cam.cx,
                           cam.cy, cam.width, cam.height, cam.d_min, cam.d_max, depth_np, pm, centers, radii,
                           grid.tau, 0.85, -0.4, -2.0, 3.5)
        np.testing.assert_array_equal(grid.log_odds_host(), lo, err_msg=f"frame {frame}")
        np.testing.assert_array_equal(grid.observed_host(), ob, err_msg=f"frame {frame}")


def test_mapper_pipeline_256_masked(M):
    """C2 pipeline (bench scene 256^3 + 7-DoF mask): fusion + EDT from the
    maintained mask equal the oracle bit for bit."""
    from paper_2512_22575_b200 import config, robot, scene

    chain, model = config.robot_7dof()
    centers, radii = robot.sphere_positions(chain, np.full(7, 0.3), model)
    grid, cam, depth = scene.bench_edt_scene((256, 256, 256), robot_spheres=(centers, radii))
    mapper = M.OccupancyMapper(grid, cam, outside_default=0.8)
    lo = np.zeros(grid.dims)
    ob = np.zeros(grid.dims, bool)
    pm = oracle.masked_pixels(depth.data, cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max,
                              cam.pose.rotation.matrix, cam.pose.translation, centers, radii, 0.01)
    r, t = cam.world_to_camera()
    for _ in range(3):
        mapper.update(depth, mask=(centers, radii))
        oracle.fuse_voxels(lo, ob, (0, 0, 0), grid.dims, grid.origin, grid.voxel_size, r, t, cam.fx, cam.fy,
                           cam.cx, cam.cy, cam.width, cam.height, cam.d_min, cam.d_max, depth.data, pm, centers,
                           radii, grid.tau, 0.85, -0.4, -2.0, 3.5)
    np.testing.assert_array_equal(grid.log_odds_host(), lo)
    np.testing.assert_array_equal(grid.observed_host(), ob)
    field = mapper.recompute_edt()
    np.testing.assert_array_equal(field.sq, oracle.edt3d(lo))


def test_fusion_errors(M):
    from paper_2512_22575_b200.errors import FrameMismatch, VolumeOutOfBounds

    grid = M.VoxelGrid((0, 0, 0), 0.1, (4, 4, 4))
    cam = M.CameraModel(1.0, 1.0, 0.0, 0.0, 1, 1, 0.1, 5.0)
    with pytest.raises(FrameMismatch):
        M.update_occupancy(grid, M.DepthImage(np.zeros((2, 3))), cam)
    with pytest.raises(VolumeOutOfBounds):
        M.edt_3d(grid, M.VoxelBox((0, 0, 0), (5, 4, 4)))
    snap = M.snapshot(grid, M.edt_3d(grid))
    with pytest.raises(ValueError):
        M.update_occupancy(snap.grid, M.DepthImage(np.zeros((1, 1))), cam)


def test_snapshot_isolated_from_updates(M):
    grid = M.VoxelGrid((-0.05, -0.05, 1.95), 0.1, (1, 1, 1))
    cam = M.CameraModel(1.0, 1.0, 0.0, 0.0, 1, 1, 0.1, 5.0)
    snap = M.snapshot(grid, M.edt_3d(grid))
    before = snap.grid.log_odds_host().copy()
    M.update_occupancy(grid, M.DepthImage(np.array([[2.0]])), cam)
    np.testing.assert_array_equal(snap.grid.log_odds_host(), before)
    assert grid.log_odds_host()[0, 0, 0] == 0.85


# ----------------------------------------------------------------------------- query
def test_query_golden(M):
    g = load_golden("query")
    for i in range(int(g["q_count"])):
        sq = i32_to_sq(g[f"q_sq_{i}"])
        ox, oy, oz, voxel, outside = (float(v) for v in g[f"q_meta_{i}"])
        lo = tuple(int(v) for v in g[f"q_lo_{i}"])
        box = M.VoxelBox(lo, tuple(l + s for l, s in zip(lo, sq.shape)))
        field = M.DistanceField((ox, oy, oz), voxel, None, box,
                                torch.from_numpy(sq.astype(np.float32)).cuda(), outside)
        got = M.query_distances(field, g[f"q_pts_{i}"])
        np.testing.assert_array_equal(got, g[f"q_val_{i}"], err_msg=str(g[f"q_name_{i}"]))


def _random_rotation(rng):
    from paper_2512_22575_b200.geometry import Rotation3

    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    m = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                  [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                  [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
    u, _, vt = np.linalg.svd(m)
    return Rotation3(u @ vt)


def test_fusion_prefilter_stress_vs_oracle(M):
    """Arbitrary camera rotations/positions (inside and outside the grid),
    plus a camera whose projections land exactly on pixel boundaries, so the
    conservative fp32 prefilter's ambiguous branches are exercised."""
    from paper_2512_22575_b200 import scene
    from paper_2512_22575_b200.geometry import RigidTransform, Rotation3

    rng = np.random.default_rng(314)
    dims = (40, 33, 50)
    grid = M.VoxelGrid((-0.4, -0.33, 0.0), 0.02, dims)
    lo = np.zeros(dims)
    ob = np.zeros(dims, bool)
    cams = []
    for _ in range(10):
        pose = RigidTransform(_random_rotation(rng), rng.uniform(-1.5, 1.5, size=3))
        cams.append(M.CameraModel(rng.uniform(40, 200), rng.uniform(40, 200), rng.uniform(10, 60),
                                  rng.uniform(10, 50), 64, 48, 0.05, 20.0, pose=pose))
    # boundary camera: unit focal length, voxel centres at x = k*0.02 + 0.01 project to
    # u = x/z with z = 0.02 * odd -> exact half-integers appear
    pose = RigidTransform(Rotation3.identity(), (0.4 - 0.01, 0.33 - 0.01, -0.01))
    cams.append(M.CameraModel(1.0, 1.0, 0.0, 0.0, 64, 48, 0.001, 20.0, pose=pose))
    for i, cam in enumerate(cams):
        c = rng.uniform([-0.3, -0.3, 0.2], [0.3, 0.3, 0.9])
        spheres = (np.array([[0.05, -0.02, 0.5], [-0.1, 0.1, 0.3]]), np.array([0.11, 0.07]))
        d = scene.render_boxes(cam, [(c - 0.15, c + 0.15), ((-5, -5, 1.0), (5, 5, 1.1))], spheres)
        if i == len(cams) - 1:
            d = np.full((48, 64), 0.5)  # flat wall in front of the boundary camera
        M.update_occupancy(grid, M.DepthImage(d), cam, mask=spheres)
        pm = oracle.masked_pixels(d, cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max,
                                  cam.pose.rotation.matrix, cam.pose.translation, spheres[0], spheres[1], 0.01)
        r, t = cam.world_to_camera()
        oracle.fuse_voxels(lo, ob, (0, 0, 0), dims, grid.origin, grid.voxel_size, r, t, cam.fx, cam.fy, cam.cx,
                           cam.cy, cam.width, cam.height, cam.d_min, cam.d_max, d, pm, spheres[0], spheres[1],
                           grid.tau, 0.85, -0.4, -2.0, 3.5)
        np.testing.assert_array_equal(grid.log_odds_host(), lo, err_msg=f"camera {i}")
        np.testing.assert_array_equal(grid.observed_host(), ob, err_msg=f"camera {i}")
    assert ob.sum() > 1000


def test_mapper_pipeline_512_c5_frames(M):
    """C5 map path (512^3 bench grid, moving cube, 7-DoF body mask), 3
    frames: log_odds / observed bitwise and the EDT bit-exact against the
    oracle after every frame.  At 512^3 the coordinates are largest, which
    is where the fp32 prefilter's error bounds matter most."""
    from paper_2512_22575_b200 import scene

    grid, cam, _ = scene.bench_edt_scene((512, 512, 512))
    mapper = M.OccupancyMapper(grid, cam, outside_default=0.8)
    lo = np.zeros(grid.dims)
    ob = np.zeros(grid.dims, bool)
    r, t = cam.world_to_camera()
    oracle.set_threads(0)
    for f, (depth, (centers, radii)) in enumerate(scene.moving_obstacle_frames(cam, grid.dims, 3)):
        mapper.update(M.DepthImage(depth), mask=(centers, radii))
        pm = oracle.masked_pixels(depth, cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max,
                                  cam.pose.rotation.matrix, cam.pose.translation, centers, radii, 0.01)
        oracle.fuse_voxels(lo, ob, (0, 0, 0), grid.dims, grid.origin, grid.voxel_size, r, t, cam.fx, cam.fy,
                           cam.cx, cam.cy, cam.width, cam.height, cam.d_min, cam.d_max, depth, pm, centers,
                           radii, grid.tau, 0.85, -0.4, -2.0, 3.5)
        assert np.array_equal(grid.log_odds_host(), lo), f"frame {f}: log_odds"
        assert np.array_equal(grid.observed_host(), ob), f"frame {f}: observed"
        field = mapper.recompute_edt()
        assert np.array_equal(field.sq_device.cpu().numpy().astype(np.float64), oracle.edt3d(lo)), f"frame {f}: EDT"
    assert ob.sum() > 100000


def test_snapshot_copy_on_write(M):
    """O(1) snapshots (vp/mapping.py:125-133, 713-723 semantics): each snapshot
    keeps the state of the moment it was taken, bitwise, across later journaled
    fusions, an unjournaled in-place write and a dropped sibling snapshot; its
    EDT equals the oracle's on that state."""
    from paper_2512_22575_b200 import scene

    n = 96
    grid, cam, _ = scene.bench_edt_scene((n, n, n))
    mapper = M.OccupancyMapper(grid, cam, outside_default=0.8)
    frames = scene.moving_obstacle_frames(cam, (n, n, n), 8)
    want, snaps = [], []
    for f, (depth, mask) in enumerate(frames[:6]):
        mapper.update(M.DepthImage(depth), mask=mask)
        mapper.recompute_edt()
        if f in (1, 3, 4):
            snaps.append(mapper.snapshot())
            want.append((grid.log_odds_host().copy(), grid.observed_host().copy()))
    j = grid._journal
    assert j is not None and j.nseg >= 2  # the updates after the first snapshot were journaled
    del snaps[2], want[2]  # a dropped snapshot
    grid.mark_occupied(np.zeros(grid.dims, bool) | (np.arange(n)[:, None, None] == 3))  # unjournaled write
    for depth, mask in frames[6:]:
        mapper.update(M.DepthImage(depth), mask=mask)
    for s, (lo, ob) in zip(snaps, want):
        assert np.array_equal(s.grid.log_odds_host(), lo)
        assert np.array_equal(s.grid.observed_host(), ob)
        assert np.array_equal(M.edt_3d(s.grid).sq, oracle.edt3d(lo))
        with pytest.raises(ValueError):
            M.update_occupancy(s.grid, M.DepthImage(frames[0][0]), cam)
    assert not np.array_equal(grid.log_odds_host(), want[-1][0])


def test_snapshot_journal_stays_bounded(M):
    """The closed-loop pattern (snap = mapper.snapshot() every frame, the old
    one dropped): one journal segment at a time, never a materialisation."""
    from paper_2512_22575_b200 import scene

    n = 64
    grid, cam, _ = scene.bench_edt_scene((n, n, n))
    mapper = M.OccupancyMapper(grid, cam, outside_default=0.8)
    snap = None
    for depth, mask in scene.moving_obstacle_frames(cam, (n, n, n), 6):
        mapper.update(M.DepthImage(depth), mask=mask)
        mapper.recompute_edt()
        snap = mapper.snapshot()
        assert grid._journal is None or grid._journal.nseg <= 1
    assert snap.grid._state is None  # never read: never copied
    lo = grid.log_odds_host().copy()
    assert np.array_equal(snap.grid.log_odds_host(), lo)
