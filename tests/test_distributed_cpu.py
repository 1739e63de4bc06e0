"""World-size-2 host logic of the sharded SMPC step on CPU (gloo).

Each rank takes its slice of one candidate batch (ShardedSMPC.sample_range),
scores it with the oracle, reduces it to the softmin partial record of
SURVEY.md 8e, exchanges the records with the product's exchange_partials over
a real process group, and merges them in rank order.  The merged U* must equal
the unsharded soft_weights + update_controls of the whole batch
(vp/planner.py:373-400) on every rank, bit-identically across ranks.
"""

import hashlib
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from test_oracle_golden import rollout_args
from conftest import load_golden

WORLD = 2
M_LOCAL = 24


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    g = load_golden("rollout")
    args = rollout_args(g, 0)
    h = g["r_controls_0"].shape[1]
    n = g["r_controls_0"].shape[2]
    eps = oracle.sample_perturbations(WORLD * M_LOCAL, h, n, np.full(n, 0.5), 5, 11)
    nominal = np.linspace(-0.2, 0.2, h * n).reshape(h, n)
    costs = oracle.evaluate_batch(args, nominal[None] + eps)["costs"]
    return nominal, eps, costs, 0.05 * float(np.median(costs))


def _worker(rank, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_2512_22575_b200 import distributed

        nominal, eps, costs, lam = _problem()
        sh = distributed.ShardedSMPC(SimpleNamespace(params=SimpleNamespace(samples=M_LOCAL)), world=WORLD,
                                     rank=rank)
        lo, hi = sh.sample_range()
        part = torch.from_numpy(oracle.smpc_partial(costs[lo:hi], eps[lo:hi], lam, m_offset=lo))
        parts = distributed.exchange_partials(part, WORLD)
        m, z, nonfinite, best, delta = oracle.merge_partials(parts.numpy(), lam)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), u=nominal.reshape(-1) + delta, m=m, z=z, best=best,
                 nonfinite=nonfinite, lo=lo, hi=hi, parts=parts.numpy())
    finally:
        dist.destroy_process_group()


def test_sharded_merge_two_ranks_gloo(tmp_path):
    mp.start_processes(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, start_method="fork")
    nominal, eps, costs, lam = _problem()
    w = oracle.soft_weights(costs, lam)
    want = oracle.update_controls(nominal, eps, w).reshape(-1)
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(WORLD)]
    # disjoint, covering slices; sample 0 (the nominal) on rank 0
    assert [(int(r["lo"]), int(r["hi"])) for r in res] == [(0, M_LOCAL), (M_LOCAL, 2 * M_LOCAL)]
    # exchange returns the records in rank order on every rank
    np.testing.assert_array_equal(res[0]["parts"], res[1]["parts"])
    for r in res:
        np.testing.assert_allclose(r["u"], want, rtol=1e-12, atol=1e-15)
        assert float(r["m"]) == costs.min()
        assert int(r["best"]) == int(np.argmin(costs))
        assert float(r["nonfinite"]) == 0.0
        np.testing.assert_allclose(float(r["z"]), np.exp(-(costs - costs.min()) / lam).sum(), rtol=1e-13)
    # all ranks bit-identical (no broadcast needed)
    np.testing.assert_array_equal(res[0]["u"], res[1]["u"])


def test_merge_shift_invariance_and_order():
    """Merging is independent of how the batch is cut (1, 2, 3, 6 shards)."""
    nominal, eps, costs, lam = _problem()
    ref = None
    for shards in (1, 2, 3, 6):
        step = costs.shape[0] // shards
        parts = [oracle.smpc_partial(costs[k * step:(k + 1) * step], eps[k * step:(k + 1) * step], lam, k * step)
                 for k in range(shards)]
        m, z, _, best, delta = oracle.merge_partials(np.stack(parts), lam)
        assert int(best) == int(np.argmin(costs))
        if ref is None:
            ref = delta
        np.testing.assert_allclose(delta, ref, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("world,rank", [(1, 0), (4, 3), (8, 5)])
def test_sample_range_partition(world, rank):
    from paper_2512_22575_b200 import distributed

    sh = distributed.ShardedSMPC(SimpleNamespace(params=SimpleNamespace(samples=4096)), world=world, rank=rank)
    assert sh.global_samples == world * 4096
    assert sh.sample_range() == (rank * 4096, (rank + 1) * 4096)


# ----------------------------------------------------------------------------- map replicas
class _OracleMapper:
    """OccupancyMapper stand-in on the CPU oracle (the product mapper needs a
    GPU): masked pixels + fusion + EDT of the bench scene's grid."""

    def __init__(self, n):
        from oracle import scene as osc

        self.osc = osc
        self.cam = osc.Camera()
        self.dims = (n, n, n)
        extent = np.array(self.dims) * 0.02
        self.origin = np.array([-extent[0] / 2.0, -extent[1] / 2.0, 0.0])
        self.lo = np.zeros(self.dims)
        self.ob = np.zeros(self.dims, bool)

    def update(self, depth, mask=None):
        depth = depth.cpu().numpy() if torch.is_tensor(depth) else np.asarray(depth)
        c, r = mask if mask is not None else (np.zeros((0, 3)), np.zeros(0))
        cam = self.cam
        pm = oracle.masked_pixels(depth, cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max, cam.pose_r,
                                  cam.pose_t, c, r, 0.01)
        wr, wt = cam.world_to_camera()
        oracle.fuse_voxels(self.lo, self.ob, (0, 0, 0), self.dims, self.origin, 0.02, wr, wt, cam.fx, cam.fy, cam.cx,
                           cam.cy, cam.width, cam.height, cam.d_min, cam.d_max, depth, pm, c, r, 0.05, 0.85, -0.4,
                           -2.0, 3.5)

    def recompute_edt(self):
        return oracle.edt3d(self.lo)


def _mapper_worker(rank, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from oracle import scene as osc
        from paper_2512_22575_b200 import distributed

        n = 48
        frames = osc.moving_obstacle_frames((n, n, n), 3) if rank == 0 else [(None, None)] * 3
        sm = distributed.ShardedMapper(_OracleMapper(n), (120, 160), world=WORLD, rank=rank)
        digests = []
        for depth, mask in frames:  # only rank 0 holds the camera frames
            sm.update(depth, mask=mask)
            sq = sm.recompute_edt()
            digests.append([hashlib.sha1(a.tobytes()).hexdigest() for a in (sq, sm.mapper.lo, sm.mapper.ob)])
        np.savez(os.path.join(out_dir, f"map{rank}.npz"), sq=sq, lo=sm.mapper.lo, digests=np.array(digests))
    finally:
        dist.destroy_process_group()


def test_sharded_mapper_replicas_bitwise_gloo(tmp_path):
    """Rank 0 broadcasts each frame (depth + mask spheres, one block); both
    ranks fuse and transform their own replica: bit-identical fields, and
    equal to a single-process run on the same frames."""
    mp.start_processes(_mapper_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, start_method="fork")
    r0, r1 = (np.load(tmp_path / f"map{r}.npz") for r in range(WORLD))
    np.testing.assert_array_equal(r0["digests"], r1["digests"])
    np.testing.assert_array_equal(r0["sq"], r1["sq"])
    from oracle import scene as osc

    ref = _OracleMapper(48)
    for depth, mask in osc.moving_obstacle_frames((48, 48, 48), 3):
        ref.update(depth, mask=mask)
    np.testing.assert_array_equal(r0["sq"], ref.recompute_edt())
    np.testing.assert_array_equal(r1["lo"], ref.lo)
    assert np.isfinite(r0["sq"]).any() and (r0["sq"] == 0).any()
