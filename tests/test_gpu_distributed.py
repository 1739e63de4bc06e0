"""Map replicas on the device: two ranks (gloo, sharing one
B200 -- the sandbox has one GPU) each run the product OccupancyMapper on its
own 256^3 grid; rank 0 alone renders the moving-obstacle frames and
ShardedMapper broadcasts them.  The replicas' fields and grids must be
bit-identical, and equal to the CPU oracle on the same frames."""

import hashlib
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

WORLD = 2
N = 256


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_2512_22575_b200 import distributed, mapping, scene

        torch.cuda.set_device(0)
        grid, cam, _ = scene.bench_edt_scene((N, N, N))
        mapper = mapping.OccupancyMapper(grid, cam, outside_default=0.8)
        sm = distributed.ShardedMapper(mapper, (cam.height, cam.width), world=WORLD, rank=rank,
                                       device=torch.device("cuda", 0))
        frames = scene.moving_obstacle_frames(cam, (N, N, N), 3) if rank == 0 else [(None, None)] * 3
        digests = []
        for depth, mask in frames:
            sm.update(depth, mask=mask)
            f = sm.recompute_edt()
            sq = f.sq_device.cpu().numpy()
            digests.append([hashlib.sha1(a.tobytes()).hexdigest()
                            for a in (sq, grid.log_odds_host(), grid.observed_host())])
        np.save(os.path.join(out_dir, f"digests{rank}.npy"), np.array(digests))
        if rank == 0:
            np.save(os.path.join(out_dir, "sq.npy"), sq)
    finally:
        dist.destroy_process_group()


def test_map_replicas_bitwise_two_ranks(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    mp.start_processes(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, start_method="spawn")
    d0, d1 = (np.load(tmp_path / f"digests{r}.npy") for r in range(WORLD))
    np.testing.assert_array_equal(d0, d1)
    import oracle
    from paper_2512_22575_b200 import scene

    cam = scene.bench_camera()
    lo = np.zeros((N, N, N))
    ob = np.zeros((N, N, N), bool)
    origin = np.array([-N * 0.01, -N * 0.01, 0.0])
    r, t = cam.world_to_camera()
    oracle.set_threads(0)
    for depth, (c, rad) in scene.moving_obstacle_frames(cam, (N, N, N), 3):  # the frames rank 0 sent
        pm = oracle.masked_pixels(depth, cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max,
                                  cam.pose.rotation.matrix, cam.pose.translation, c, rad, 0.01)
        oracle.fuse_voxels(lo, ob, (0, 0, 0), (N, N, N), origin, 0.02, r, t, cam.fx, cam.fy, cam.cx, cam.cy,
                           cam.width, cam.height, cam.d_min, cam.d_max, depth, pm, c, rad, 0.05, 0.85, -0.4, -2.0, 3.5)
    np.testing.assert_array_equal(np.load(tmp_path / "sq.npy").astype(np.float64), oracle.edt3d(lo))
