"""Rollouts sharded across GPUs.

Each rank evaluates its own slice of the candidate batch (global sample index
offset rank * M_local; global sample 0, the nominal, lives on rank 0) and
reduces it on the device to one softmin partial

    [m_r, Z_r = sum exp(-(S - m_r)/lam), nonfinite_r, best_index_r, N_r = sum exp(...) eps]

The only data-path collective is one all-gather of these partials
((4 + H n) doubles per rank, 1.8 KB at H = 64) over NCCL; every rank then
merges them in fixed rank order (shift invariance of the softmin,
t/test_planner.py:369-377) and finishes the step on its own device, so all
ranks hold bit-identical commands without a broadcast.  The distance field is
replicated (each rank runs its own bit-exact fusion + EDT), never sent.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .planner import Planner, StepResult


def exchange_partials(part: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gather one partial per rank -> (world, L) in rank order."""
    if world == 1:
        return part.reshape(1, -1)
    if part.is_cuda and dist.get_backend(group) != "nccl":  # e.g. gloo: gather through the host
        host = exchange_partials(part.cpu(), world, group)
        return host.to(part.device)
    out = torch.empty(world * part.numel(), dtype=part.dtype, device=part.device)
    dist.all_gather_into_tensor(out, part.contiguous(), group=group)
    return out.reshape(world, -1)


class ShardedSMPC:
    """SMPC step over `world` ranks with `samples_per_rank` candidates each
    (weak scaling; defaults to params.samples per rank)."""

    def __init__(self, planner: Planner, world: int = 1, rank: int = 0, samples_per_rank: int | None = None,
                 group=None):
        self.planner = planner
        self.world = int(world)
        self.rank = int(rank)
        self.m_local = int(samples_per_rank or planner.params.samples)
        self.group = group

    @property
    def global_samples(self) -> int:
        return self.world * self.m_local

    def sample_range(self) -> tuple[int, int]:
        """Global sample indices [lo, hi) this rank evaluates (rank 0 holds the nominal, sample 0)."""
        lo = self.rank * self.m_local
        return lo, lo + self.m_local

    def step_device(self, state, goal, snap, nominal_dev: torch.Tensor, rng_seed: int,
                    perturbations: torch.Tensor | None = None) -> torch.Tensor:
        pl = self.planner
        lo = self.sample_range()[0]
        if perturbations is None:  # draws inside the step kernel (vpb_smpc_generate)
            res, _ = pl.smpc_generate_device(state, goal, snap, nominal_dev, rng_seed, samples=self.m_local,
                                             m_offset=lo, partial=self.world > 1)
            if self.world == 1:
                return res
            part = res
        elif self.world == 1:
            return pl.smpc_step_device(state, goal, snap, nominal_dev, perturbations)  # one fused launch
        else:
            part, _, _ = pl.smpc_partial_device(state, goal, snap, nominal_dev, perturbations, m_offset=lo)
        parts = exchange_partials(part, self.world, self.group)
        return pl.smpc_finish_device(state, goal, snap, nominal_dev, parts)

    def step(self, state, goal, snap, nominal, rng_seed: int) -> StepResult:
        """Public-API step with host buffers: nominal in, StepResult out."""
        pl = self.planner
        h, n = pl.params.horizon, pl.chain.dof
        nom = np.zeros((h, n)) if nominal is None else np.ascontiguousarray(nominal, dtype=np.float64)
        nom_dev = torch.from_numpy(nom).to(pl.device, non_blocking=True)
        out = self.step_device(state, goal, snap, nom_dev, rng_seed)
        return pl.unpack_step(out.cpu().numpy(), state, goal, h)


class ShardedGraph:
    """One rank's sharded SMPC step captured as a CUDA graph: H2D of the
    per-call block, the fused draw + rollout + shard-partial kernel, the NCCL
    all-gather of the partial records, the rank-order merge + tail kernel and
    the D2H of the result -- one replay per step, no per-launch host work.
    Raises if the process group cannot be captured (the caller falls back to
    the eager ``ShardedSMPC.step_device``)."""

    def __init__(self, sharded: ShardedSMPC, snap):
        from ._lib import load

        self.sh = sharded
        pl = sharded.planner
        self.pl, self.snap = pl, snap
        p = pl.params
        self.h, self.n = p.horizon, pl.chain.dof
        dev = pl.device
        L = load()
        self.dyn_len = 2 * self.n + 12
        self.block_len = self.dyn_len + 1 + self.h * self.n
        self.host_in = torch.zeros(self.block_len, dtype=torch.float64).pin_memory()
        self.dev_in = torch.zeros(self.block_len, dtype=torch.float64, device=dev)
        self._seed_view = self.dev_in[self.dyn_len:self.dyn_len + 1].view(torch.int64)
        self._nom_view = self.dev_in[self.dyn_len + 1:].view(self.h, self.n)
        self._dyn_view = self.dev_in[:self.dyn_len]
        self.part = torch.empty(int(L.vpb_smpc_partial_len(self.h, self.n)), dtype=torch.float64, device=dev)
        self.parts = torch.empty(sharded.world * self.part.numel(), dtype=torch.float64, device=dev)
        self.out = torch.empty(int(L.vpb_smpc_out_len(self.h, self.n)), dtype=torch.float64, device=dev)
        self.host_out = torch.zeros(self.out.numel(), dtype=torch.float64).pin_memory()
        self.eps = torch.empty((sharded.m_local, self.h, self.n), dtype=pl._eps_dtype, device=dev)
        for _ in range(2):  # warm: workspaces, kernel attributes, NCCL communicator
            self._enqueue(copy_out=False)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            with torch.cuda.graph(self.graph, stream=s):
                self._enqueue(copy_out=True)
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize(dev)

    def _enqueue(self, copy_out: bool):
        sh, pl = self.sh, self.pl
        self.dev_in.copy_(self.host_in, non_blocking=True)
        pl.smpc_generate_device(None, None, self.snap, self._nom_view, 0, samples=sh.m_local,
                                m_offset=sh.sample_range()[0], partial=True, seed_dev=self._seed_view,
                                dyn=self._dyn_view, eps_out=self.eps, out=self.part)
        dist.all_gather_into_tensor(self.parts, self.part, group=sh.group)
        pl.smpc_finish_device(None, None, self.snap, self._nom_view, self.parts.view(sh.world, -1),
                              dyn=self._dyn_view, out=self.out)
        if copy_out:
            self.host_out.copy_(self.out, non_blocking=True)

    def stage(self, state, goal, nominal, rng_seed: int) -> None:
        n = self.n
        h = self.host_in.numpy()
        h[:n] = np.asarray(state.q, dtype=float)
        h[n:2 * n] = np.asarray(state.qd, dtype=float)
        h[2 * n:2 * n + 9] = np.asarray(goal.rotation.matrix, dtype=float).reshape(-1)
        h[2 * n + 9:2 * n + 12] = np.asarray(goal.translation, dtype=float)
        h[self.dyn_len:self.dyn_len + 1].view(np.uint64)[0] = np.uint64(int(rng_seed) & 0xFFFFFFFFFFFFFFFF)
        nom = np.zeros((self.h, n)) if nominal is None else np.asarray(nominal, dtype=float)
        h[self.dyn_len + 1:] = nom.reshape(-1)

    def replay(self) -> None:
        self.graph.replay()

    def step(self, state, goal, nominal, rng_seed: int) -> StepResult:
        self.stage(state, goal, nominal, rng_seed)
        self.graph.replay()
        torch.cuda.current_stream(self.pl.device).synchronize()
        return self.pl.unpack_step(self.host_out.numpy().copy(), state, goal, self.h)


class ShardedMapper:
    """The map side of SURVEY.md 8e, option 1: every rank keeps its own
    replica of the occupancy grid and distance field, and per map update only
    the source rank's input frame travels -- the depth image (160 x 120 f64 =
    154 KB) and the body-mask spheres, in ONE broadcast of a fixed-size block.
    Fusion and the EDT are deterministic and exact (bitwise the reference's),
    so every replica is bit-identical and the 67 MB (256^3) / 537 MB (512^3)
    field is never sent.  `mapper` is any object with the OccupancyMapper
    interface (update(depth, mask=...), recompute_edt()); `cam_hw` is the
    camera's (height, width) (known on every rank).

    Block layout (float64): [H*W depth | n_mask | 3 * MAX centers | MAX radii]."""

    MAX_SPHERES = 64

    def __init__(self, mapper, cam_hw, world: int = 1, rank: int = 0, src: int = 0, group=None, device=None):
        self.mapper = mapper
        self.h, self.w = int(cam_hw[0]), int(cam_hw[1])
        self.world, self.rank, self.src, self.group = int(world), int(rank), int(src), group
        self.device = device
        n = self.h * self.w + 1 + 4 * self.MAX_SPHERES
        on_dev = device is not None and (world == 1 or dist.get_backend(group) == "nccl")
        self._block = torch.zeros(n, dtype=torch.float64, device=device if on_dev else "cpu")

    def _pack(self, depth, mask) -> None:
        b = self._block
        hw = self.h * self.w
        d = depth.data if hasattr(depth, "data") and not torch.is_tensor(depth) else depth
        d = d.reshape(-1).to(torch.float64) if torch.is_tensor(d) else np.asarray(d, dtype=np.float64).reshape(-1)
        b[:hw] = torch.as_tensor(d, device=b.device)
        if mask is None:
            b[hw] = 0.0
            return
        centers = np.asarray(mask[0], dtype=np.float64).reshape(-1, 3)
        radii = np.asarray(mask[1], dtype=np.float64).reshape(-1)
        k = centers.shape[0]
        if k > self.MAX_SPHERES or radii.shape[0] != k:
            raise ValueError(f"mask must hold <= {self.MAX_SPHERES} spheres with one radius each")
        b[hw] = float(k)
        m = self.MAX_SPHERES
        b[hw + 1:hw + 1 + 3 * k] = torch.as_tensor(centers.reshape(-1), device=b.device)
        b[hw + 1 + 3 * m:hw + 1 + 3 * m + k] = torch.as_tensor(radii, device=b.device)

    def _unpack(self):
        b = self._block
        hw = self.h * self.w
        m = self.MAX_SPHERES
        depth = b[:hw].reshape(self.h, self.w)
        k = int(b[hw].item())
        mask = None
        if k > 0:
            host = b[hw + 1:].cpu().numpy()
            mask = (host[:3 * k].reshape(k, 3).copy(), host[3 * m:3 * m + k].copy())
        return depth, mask

    def broadcast_frame(self, depth=None, mask=None):
        """Source rank: pack (depth, mask); every rank: receive the same block.
        Returns this rank's (depth (H, W) f64 tensor, mask or None)."""
        if self.rank == self.src:
            if depth is None:
                raise ValueError("the source rank must provide the depth frame")
            self._pack(depth, mask)
        if self.world > 1:
            dist.broadcast(self._block, src=self.src, group=self.group)
        return self._unpack()

    def update(self, depth=None, mask=None) -> None:
        """One map update on this rank's replica from the source rank's frame
        (depth handed to the mapper as an (H, W) f64 tensor)."""
        d, m = self.broadcast_frame(depth, mask)
        self.mapper.update(d, mask=m)

    def recompute_edt(self):
        return self.mapper.recompute_edt()
