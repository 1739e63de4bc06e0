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
