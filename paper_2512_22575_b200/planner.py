"""Sampling MPC on the device: rollout/cost kernel, softmin, weighted update.

Drop-in counterpart of vp/planner.py.  ``Planner.evaluate`` replaces the
numba ``evaluate_batch`` call (vp/planner.py:504-592, vp/batch.py:161-336);
``Planner.smpc_step`` (vp/planner.py:594-630) runs sampling (optional), the
fused rollout + per-CTA softmin partial, the fixed-order merge, U*, the M=1
re-evaluation, clip and shift on the device and returns to the host once.
``soft_weights`` / ``update_controls`` keep the reference's validation and
exceptions.  Precision: ``"fp32"`` (production: fp32 arithmetic, fp64 cost
sums and softmin) or ``"fp64"`` (parity mode).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from ._lib import (DTYPE_F32, DTYPE_F64, MAX_JOINTS, MAX_PAIRS, MAX_SPHERES, PREC_F32, PREC_F64, VpbField,
                   VpbProblem, check, fill, load)
from .errors import DegenerateRotation, DimensionMismatch, WeightMismatch
from .geometry import RigidTransform
from .mapping import DistanceField, MapSnapshot
from .robot import JointState, KinematicChain, SphereModel

TERM_NAMES = ("pose", "collision", "limits", "smoothness", "nullspace", "terminal")


@dataclass(frozen=True)
class PlannerParams:
    """vp/planner.py:38-102 (same validation)."""

    horizon: int
    samples: int
    dt: float
    lam: float
    sigma: np.ndarray
    noise_window: int
    pose_weight: np.ndarray
    terminal_weight: np.ndarray
    w_env: float
    w_self: float
    w_q: float
    w_qd: float
    w_qdd: float
    w_s: float
    w_ns: float
    d_act: float
    margin_frac: float
    q_ref: np.ndarray

    def __post_init__(self):
        if self.horizon < 1 or self.samples < 1:
            raise ValueError("horizon and samples must be >= 1")
        if self.dt <= 0.0 or self.lam <= 0.0:
            raise ValueError("dt and lam must be positive")
        q_ref = np.asarray(self.q_ref, dtype=float).reshape(-1).copy()
        sigma = np.broadcast_to(np.asarray(self.sigma, dtype=float), q_ref.shape).copy()
        if (sigma < 0.0).any():
            raise ValueError("sigma must be non-negative")
        for name, arr in (("q_ref", q_ref), ("sigma", sigma)):
            arr.flags.writeable = False
            object.__setattr__(self, name, arr)
        for name, psd_only in (("pose_weight", True), ("terminal_weight", False)):
            w = np.asarray(getattr(self, name), dtype=float)
            if w.shape != (6, 6):
                raise ValueError(f"{name} must be 6x6, got {w.shape}")
            if np.abs(w - w.T).max() > 1e-9:
                raise ValueError(f"{name} must be symmetric")
            eigs = np.linalg.eigvalsh(w)
            if psd_only and eigs.min() < -1e-9:
                raise ValueError(f"{name} must be positive semidefinite")
            if not psd_only and eigs.min() <= 1e-12:
                raise ValueError(f"{name} must be positive definite")
            w = w.copy()
            w.flags.writeable = False
            object.__setattr__(self, name, w)
        for name in ("w_env", "w_self", "w_q", "w_qd", "w_qdd", "w_s", "w_ns"):
            if getattr(self, name) < 0.0:
                raise ValueError(f"{name} must be non-negative")
        if self.d_act < 0.0 or not 0.0 <= self.margin_frac < 0.5:
            raise ValueError("d_act must be >= 0 and margin_frac in [0, 0.5)")

    @property
    def dof(self) -> int:
        return self.q_ref.shape[0]


@dataclass(frozen=True)
class CostBreakdown:
    pose: float
    collision: float
    limits: float
    smoothness: float
    nullspace: float
    terminal: float

    @property
    def total(self) -> float:
        return self.pose + self.collision + self.limits + self.smoothness + self.nullspace + self.terminal

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in TERM_NAMES}


@dataclass
class RolloutBatch:
    controls: np.ndarray
    perturbations: np.ndarray
    costs: np.ndarray
    terms: np.ndarray
    traj_q: np.ndarray | None = None
    traj_qd: np.ndarray | None = None
    sphere_positions: np.ndarray | None = None


@dataclass(frozen=True)
class StepDiagnostics:
    best_cost: float
    weighted_cost: float
    breakdown: CostBreakdown
    e_pos: float
    e_ori: float


@dataclass(frozen=True)
class StepResult:
    command: np.ndarray
    next_nominal: np.ndarray
    diagnostics: StepDiagnostics


def tightened_limits(chain: KinematicChain, margin_frac: float):
    """vp/planner.py:291-306."""
    pos_lo, pos_hi = chain.position_limits()
    eps_q = margin_frac * (pos_hi - pos_lo)
    vel = chain.velocity_limits()
    eps_v = margin_frac * 2.0 * vel
    acc = chain.acceleration_limits()
    eps_a = margin_frac * 2.0 * acc
    return pos_lo + eps_q, pos_hi - eps_q, -vel + eps_v, vel - eps_v, -acc + eps_a, acc - eps_a


def _field_of(snap) -> DistanceField | None:
    if snap is None:
        return None
    return snap.field if isinstance(snap, MapSnapshot) else snap


def _field_struct(snap) -> VpbField:
    f = _field_of(snap)
    if f is None:
        return VpbField()  # sq = NULL: every query reports inf (vp/planner.py:429-441)
    return f._struct()


def _as_device(x, dev, dtype) -> torch.Tensor:
    if torch.is_tensor(x):
        return x.to(device=dev, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev).to(dtype)


def pack_problem(chain: KinematicChain, model: SphereModel, params: PlannerParams) -> VpbProblem:
    """Flat robot + objective block for the kernel (vp/planner.py:461-499).

    Spheres are stably sorted by link so the kernel can emit sphere centres
    while walking the chain; ``sph_orig`` maps them back to caller order and
    self pairs are remapped accordingly."""
    ch, md, p = chain, model, params
    P = VpbProblem()
    n = ch.dof
    P.n_joints, P.horizon, P.dt = n, p.horizon, p.dt
    fill(P.base_r, ch.base_pose.rotation.matrix)
    fill(P.base_t, ch.base_pose.translation)
    for i, j in enumerate(ch.joints):
        P.off_r[9 * i:9 * i + 9] = list(np.asarray(j.parent_offset.rotation.matrix, float).reshape(-1))
        P.off_t[3 * i:3 * i + 3] = list(np.asarray(j.parent_offset.translation, float))
        P.axes[3 * i:3 * i + 3] = list(np.asarray(j.axis, float))
    order = sorted(range(md.count), key=lambda s: md.spheres[s].link)
    pos = {s: k for k, s in enumerate(order)}
    P.n_spheres = md.count
    for k, s in enumerate(order):
        sp = md.spheres[s]
        P.sph_link[k] = int(sp.link)
        P.sph_orig[k] = int(s)
        P.sph_loc[3 * k:3 * k + 3] = list(np.asarray(sp.center, float))
        P.sph_r[k] = float(sp.radius)
    P.n_pairs = len(md.self_pairs)
    for q, (a, b) in enumerate(md.self_pairs):
        P.pairs[2 * q], P.pairs[2 * q + 1] = pos[a], pos[b]
    fill(P.pose_weight, p.pose_weight)
    fill(P.terminal_weight, p.terminal_weight)
    lims = tightened_limits(ch, p.margin_frac)
    for name, arr in zip(("pos_lo", "pos_hi", "vel_lo", "vel_hi", "acc_lo", "acc_hi"), lims):
        fill(getattr(P, name), arr)
    fill(P.acc_limit, ch.acceleration_limits())
    fill(P.q_ref, p.q_ref)
    P.w_env, P.w_self, P.w_q, P.w_qd = p.w_env, p.w_self, p.w_q, p.w_qd
    P.w_qdd, P.w_s, P.w_ns, P.d_act, P.lam = p.w_qdd, p.w_s, p.w_ns, p.d_act, p.lam
    return P


class Planner:
    """One manipulator's sampling MPC (vp/planner.py:458-636), device-resident."""

    def __init__(self, chain: KinematicChain, model: SphereModel, params: PlannerParams,
                 precision: str = "fp32", device=None):
        if params.dof != chain.dof:
            raise DimensionMismatch(f"params are for {params.dof} joints, chain has {chain.dof}")
        model.validate_links(chain)
        if chain.dof > MAX_JOINTS or model.count > MAX_SPHERES or len(model.self_pairs) > MAX_PAIRS:
            raise ValueError("robot exceeds the kernel limits (16 joints, 64 spheres, 256 pairs)")
        if precision not in ("fp32", "fp64"):
            raise ValueError("precision must be 'fp32' or 'fp64'")
        self.chain = chain
        self.model = model
        self.params = params
        self.precision = precision
        self._prec = PREC_F32 if precision == "fp32" else PREC_F64
        self._eps_dtype = torch.float32 if precision == "fp32" else torch.float64
        self.device = D.device(device)
        self._acc_limits = chain.acceleration_limits()
        self._base = pack_problem(chain, model, params)
        self._sessions: dict = {}
        self._last_session = None
        self._ws: dict = {}

    def problem(self, state: JointState | None, goal: RigidTransform | None, horizon: int | None = None,
                dyn: torch.Tensor | None = None) -> VpbProblem:
        P = VpbProblem()
        ctypes.memmove(ctypes.byref(P), ctypes.byref(self._base), ctypes.sizeof(VpbProblem))
        if horizon is not None:
            P.horizon = int(horizon)
        if dyn is not None:
            P.dyn_state = D.ptr(dyn)
        if state is None:
            return P
        q0 = np.asarray(state.q, dtype=float).reshape(-1)
        qd0 = np.asarray(state.qd, dtype=float).reshape(-1)
        if q0.shape != (self.chain.dof,) or qd0.shape != (self.chain.dof,):
            raise DimensionMismatch("state does not match the chain's dof")
        fill(P.q0, q0)
        fill(P.qd0, qd0)
        fill(P.goal_r, np.asarray(goal.rotation.matrix, float))
        fill(P.goal_t, np.asarray(goal.translation, float))
        return P

    def zero_nominal(self) -> np.ndarray:
        return np.zeros((self.params.horizon, self.chain.dof))

    # -- evaluate --------------------------------------------------------------
    def evaluate_device(self, state, goal, snap, controls: torch.Tensor, nominal: torch.Tensor | None = None,
                        keep_trajectories: bool = False, keep_spheres: bool = False):
        """Kernel launch on device tensors; returns device outputs, no sync.

        controls: (M, H, n) f32/f64 CUDA tensor (perturbations when
        ``nominal`` (H, n) f64 is given)."""
        dev = self.device
        m, h, n = controls.shape
        if n != self.chain.dof:
            raise DimensionMismatch(f"controls carry {n} joints, chain has {self.chain.dof}")
        P = self.problem(state, goal, horizon=h)
        dtype = DTYPE_F32 if controls.dtype == torch.float32 else DTYPE_F64
        costs = torch.empty(m, dtype=torch.float64, device=dev)
        terms = torch.empty((m, 6), dtype=torch.float64, device=dev)
        flags = torch.empty(m, dtype=torch.uint8, device=dev)
        tq = torch.empty((m, h + 1, n), dtype=torch.float64, device=dev) if keep_trajectories else None
        tqd = torch.empty((m, h + 1, n), dtype=torch.float64, device=dev) if keep_trajectories else None
        sp = torch.empty((m, h, self.model.count, 3), dtype=torch.float64, device=dev) if keep_spheres else None
        check(load().vpb_evaluate_batch(
            P, _field_struct(snap), D.ptr(controls), D.ptr(nominal), dtype, m, self._prec, D.ptr(costs),
            D.ptr(terms), D.ptr(flags), D.ptr(tq), D.ptr(tqd), D.ptr(sp), D.stream(dev)), "evaluate_batch")
        return costs, terms, flags, tq, tqd, sp

    def evaluate(self, state: JointState, goal: RigidTransform, snap, controls, perturbations=None,
                 keep_trajectories: bool = False, keep_spheres: bool = False) -> RolloutBatch:
        """Score a batch of control sequences (vp/planner.py:504-592)."""
        host = not torch.is_tensor(controls)
        c_np = np.ascontiguousarray(controls, dtype=float) if host else None
        shape = c_np.shape if host else tuple(controls.shape)
        if len(shape) != 3:
            raise DimensionMismatch(f"controls must be (M, H, n), got {shape}")
        m, h, n = shape
        if n != self.chain.dof:
            raise DimensionMismatch(f"controls carry {n} joints, chain has {self.chain.dof}")
        if host and not np.isfinite(c_np).all():
            raise ValueError("control sequences must be finite")
        c_dev = _as_device(c_np if host else controls, self.device, torch.float64)
        if not host and not bool(torch.isfinite(c_dev).all()):
            raise ValueError("control sequences must be finite")
        costs, terms, flags, tq, tqd, sp = self.evaluate_device(state, goal, snap, c_dev, None,
                                                                 keep_trajectories, keep_spheres)
        flags_h = flags.cpu().numpy()
        if flags_h.any():
            bad = int(np.nonzero(flags_h)[0][0])
            raise DegenerateRotation(f"sample {bad} reached a pose error with rotation angle at pi")
        ctrl_out = c_np if host else controls
        if perturbations is None:
            perturbations = np.zeros_like(c_np) if host else torch.zeros_like(controls)
        return RolloutBatch(
            controls=ctrl_out, perturbations=perturbations, costs=costs.cpu().numpy(), terms=terms.cpu().numpy(),
            traj_q=None if tq is None else tq.cpu().numpy(), traj_qd=None if tqd is None else tqd.cpu().numpy(),
            sphere_positions=None if sp is None else sp.cpu().numpy(),
        )

    # -- smpc step -------------------------------------------------------------
    def sample_device(self, rng_seed: int, m_offset: int = 0, samples: int | None = None,
                      seed_dev: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
        """On-device perturbations (M, H, n) in the planner's noise dtype."""
        p = self.params
        m = p.samples if samples is None else int(samples)
        if out is None:
            out = torch.empty((m, p.horizon, self.chain.dof), dtype=self._eps_dtype, device=self.device)
        sig = np.ascontiguousarray(p.sigma, dtype=np.float64)
        check(load().vpb_sample_perturbations(
            int(rng_seed) & 0xFFFFFFFFFFFFFFFF, D.ptr(seed_dev), int(m_offset), m, p.horizon, self.chain.dof,
            p.noise_window, D.host_ptr(sig), DTYPE_F32 if out.dtype == torch.float32 else DTYPE_F64, D.ptr(out),
            D.stream(self.device)), "sample_perturbations")
        return out

    def _smpc_ws(self, m: int, h: int) -> torch.Tensor:
        """This planner's step workspace for (M, H): owned by the planner (not
        shared between planners or graphs), fixed size per key, so a captured
        graph's pointers into it stay valid for the planner's lifetime."""
        ws = self._ws.get((m, h))
        if ws is None:
            nbytes = int(load().vpb_smpc_workspace_bytes(m, h, self.chain.dof))
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            self._ws[(m, h)] = ws
        return ws

    def _finish_ws(self, n_parts: int, h: int) -> torch.Tensor:
        ws = self._ws.get(("finish", n_parts, h))
        if ws is None:
            nbytes = int(load().vpb_smpc_finish_workspace_bytes(n_parts, h, self.chain.dof))
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            self._ws[("finish", n_parts, h)] = ws
        return ws

    def smpc_weights_device(self, m: int, h: int) -> torch.Tensor:
        """Softmin weights (M,) f64 of the last single-device step run with M
        samples and horizon H, as the fused merge computed them (debug export,
        vpb_smpc_debug_weights)."""
        ws = self._smpc_ws(m, h)
        w = torch.empty(m, dtype=torch.float64, device=self.device)
        P = self.problem(None, None, horizon=h)
        check(load().vpb_smpc_debug_weights(P, m, D.ptr(ws), ws.numel(), D.ptr(w), D.stream(self.device)),
              "smpc_debug_weights")
        return w

    def smpc_partial_device(self, state, goal, snap, nominal_dev: torch.Tensor, eps_dev: torch.Tensor,
                            m_offset: int = 0, dyn: torch.Tensor | None = None):
        """Rollout + this shard's merged softmin partial in one launch (device,
        no sync).  Returns (partial (L,) f64, costs (M,), flags (M,))."""
        m, h, n = eps_dev.shape
        P = self.problem(state, goal, horizon=h, dyn=dyn)
        L = load()
        part = torch.empty(int(L.vpb_smpc_partial_len(h, n)), dtype=torch.float64, device=self.device)
        costs = torch.empty(m, dtype=torch.float64, device=self.device)
        flags = torch.empty(m, dtype=torch.uint8, device=self.device)
        ws = self._smpc_ws(m, h)
        dtype = DTYPE_F32 if eps_dev.dtype == torch.float32 else DTYPE_F64
        check(L.vpb_smpc_partial(P, _field_struct(snap), D.ptr(eps_dev), dtype, D.ptr(nominal_dev), m, int(m_offset),
                                 self._prec, D.ptr(costs), D.ptr(flags), D.ptr(part), D.ptr(ws), ws.numel(),
                                 D.stream(self.device)), "smpc_partial")
        return part, costs, flags

    def smpc_step_device(self, state, goal, snap, nominal_dev: torch.Tensor, eps_dev: torch.Tensor,
                         out: torch.Tensor | None = None, costs: torch.Tensor | None = None,
                         dyn: torch.Tensor | None = None) -> torch.Tensor:
        """Whole single-device step in ONE kernel launch (rollout, softmin
        partials, fixed-order merges, U*, clip, shift, re-evaluation).
        Returns the packed output vector (vpb_smpc_out_len doubles)."""
        m, h, n = eps_dev.shape
        P = self.problem(state, goal, horizon=h, dyn=dyn)
        L = load()
        if out is None:
            out = torch.empty(int(L.vpb_smpc_out_len(h, n)), dtype=torch.float64, device=self.device)
        ws = self._smpc_ws(m, h)
        dtype = DTYPE_F32 if eps_dev.dtype == torch.float32 else DTYPE_F64
        check(L.vpb_smpc_step(P, _field_struct(snap), D.ptr(eps_dev), dtype, D.ptr(nominal_dev), m, self._prec,
                              D.ptr(costs), None, D.ptr(out), D.ptr(ws), ws.numel(), D.stream(self.device)),
              "smpc_step")
        return out

    def smpc_generate_device(self, state, goal, snap, nominal_dev: torch.Tensor, rng_seed: int,
                             samples: int | None = None, m_offset: int = 0, partial: bool = False,
                             seed_dev: torch.Tensor | None = None, dyn: torch.Tensor | None = None,
                             eps_out: torch.Tensor | None = None, out: torch.Tensor | None = None):
        """Draw + step in one call (vpb_smpc_generate): the perturbations of
        ``sample_device`` with the same seed / offset, then the fused step
        (``partial=False``: the packed step output) or this shard's softmin
        partial (``partial=True``).  Returns (result, eps)."""
        p = self.params
        m = p.samples if samples is None else int(samples)
        h, n = p.horizon, self.chain.dof
        P = self.problem(state, goal, horizon=h, dyn=dyn)
        L = load()
        if eps_out is None:
            eps_out = torch.empty((m, h, n), dtype=self._eps_dtype, device=self.device)
        if out is None:
            length = L.vpb_smpc_partial_len(h, n) if partial else L.vpb_smpc_out_len(h, n)
            out = torch.empty(int(length), dtype=torch.float64, device=self.device)
        ws = self._smpc_ws(m, h)
        sig = np.ascontiguousarray(np.broadcast_to(np.asarray(p.sigma, dtype=float), (n,)))
        check(L.vpb_smpc_generate(P, _field_struct(snap), int(rng_seed) & 0xFFFFFFFFFFFFFFFF, D.ptr(seed_dev),
                                  int(m_offset), p.noise_window, D.host_ptr(sig), D.ptr(nominal_dev), m, self._prec,
                                  None, None, D.ptr(eps_out), D.ptr(out) if partial else None,
                                  None if partial else D.ptr(out), D.ptr(ws), ws.numel(), D.stream(self.device)),
              "smpc_generate")
        return out, eps_out

    def smpc_finish_device(self, state, goal, snap, nominal_dev: torch.Tensor, partials: torch.Tensor,
                           dyn: torch.Tensor | None = None, out: torch.Tensor | None = None):
        """Merge rank partials (R, L) in rank order and finish the step on the
        device.  Returns the packed output vector (vpb_smpc_out_len)."""
        h, n = nominal_dev.shape
        P = self.problem(state, goal, horizon=h, dyn=dyn)
        L = load()
        if out is None:
            out = torch.empty(int(L.vpb_smpc_out_len(h, n)), dtype=torch.float64, device=self.device)
        parts = partials.reshape(-1, int(L.vpb_smpc_partial_len(h, n))).contiguous()
        ws = self._finish_ws(parts.shape[0], h)
        check(L.vpb_smpc_finish(P, _field_struct(snap), D.ptr(parts), parts.shape[0], D.ptr(nominal_dev),
                                self._prec, D.ptr(out), D.ptr(ws), ws.numel(), D.stream(self.device)),
              "smpc_finish")
        return out

    def unpack_step(self, out_host: np.ndarray, state: JointState, goal: RigidTransform, h: int) -> StepResult:
        """StepResult from the packed step output (vpb_smpc_out_len doubles;
        e_pos / e_ori come from the device, vp/planner.py:620-629)."""
        n = self.chain.dof
        hn = h * n
        base = 2 * hn + n
        # [cost(U*), 5 sums, terminal, best, Z, non-finite, best index, e_pos, e_ori] as Python floats
        v = out_host[base:base + 13].tolist()
        wcost = v[0]
        # non-finite count = flagged samples + 2^32 x other non-finite costs (rollout.cu)
        flagged = math.fmod(v[9], 4294967296.0)
        if flagged > 0 or not math.isfinite(wcost):
            raise DegenerateRotation("a sample reached a pose error with rotation angle at pi")
        if v[9] > 0:
            raise ValueError("costs must be finite")  # vp/planner.py:377-378 (soft_weights)
        if not math.isfinite(v[11]):  # device-step output: diagnostics on the host
            q0 = np.ascontiguousarray(state.q, dtype=np.float64)
            gr = np.ascontiguousarray(goal.rotation.matrix, dtype=np.float64)
            gt = np.ascontiguousarray(goal.translation, dtype=np.float64)
            e = np.zeros(2)
            check(load().vpb_ee_errors(self._base, D.host_ptr(q0), D.host_ptr(gr), D.host_ptr(gt), D.host_ptr(e[:1]),
                                       D.host_ptr(e[1:])), "ee_errors")
            v[11], v[12] = e.tolist()
        diag = StepDiagnostics(best_cost=v[7], weighted_cost=wcost, breakdown=CostBreakdown(*v[1:7]), e_pos=v[11],
                               e_ori=v[12])
        return StepResult(command=out_host[hn:hn + n].copy(),
                          next_nominal=out_host[hn + n:2 * hn + n].reshape(h, n).copy(), diagnostics=diag)

    def smpc_step(self, state: JointState, goal: RigidTransform, snap, nominal, rng_seed: int,
                  perturbations=None) -> StepResult:
        """One cycle: sample, roll out, weight, update, shift (vp/planner.py:594-630).

        ``perturbations`` (M, H, n), if given, replaces the on-device sampler
        (parity runs feed the reference's own noise)."""
        p = self.params
        h, n = p.horizon, self.chain.dof
        nom = self.zero_nominal() if nominal is None else np.asarray(nominal, dtype=float)
        if nom.shape != (h, n):
            raise DimensionMismatch(f"nominal must be {(h, n)}, got {nom.shape}")
        if perturbations is None:  # the production path: one native call per step
            return self.session(snap).step(state, goal, nom, rng_seed, snap)
        nom_dev = _as_device(nom, self.device, torch.float64)
        eps_dev = _as_device(perturbations, self.device, self._eps_dtype)
        if tuple(eps_dev.shape) != (eps_dev.shape[0], h, n):
            raise DimensionMismatch("perturbations must be (M, H, n)")
        out = self.smpc_step_device(state, goal, snap, nom_dev, eps_dev)
        return self.unpack_step(out.cpu().numpy(), state, goal, h)

    def session(self, snap, samples: int | None = None) -> "SmpcSession":
        """The cached native step session for this field geometry."""
        f = _field_of(snap)
        m = int(samples or self.params.samples)
        last = self._last_session
        if last is not None and last[0] is f and last[1] == m:  # same field object: no key building
            return last[2]
        key = (m, None if f is None else (tuple(f.volume.lo), f.volume.shape, tuple(np.asarray(f.origin).tolist()),
                                         float(f.voxel_size), float(f.outside_default), str(f.sq_device.device)))
        sess = self._sessions.get(key)
        if sess is None:
            sess = SmpcSession(self, snap, m)
            self._sessions[key] = sess
        self._last_session = (f, m, sess)
        return sess

    def integrate(self, state: JointState, command: np.ndarray) -> JointState:
        """vp/planner.py:632-636."""
        qd = state.qd + command * self.params.dt
        q = state.q + qd * self.params.dt
        return JointState(q, qd, np.asarray(command, dtype=float).copy())


# -- module-level softmin / update (vp/planner.py:373-400) ------------------------
def soft_weights(costs, lam: float):
    """Softmin weights on the device; numpy in -> numpy out, tensor in -> tensor out."""
    host = not torch.is_tensor(costs)
    c = np.asarray(costs, dtype=float) if host else costs
    if (c.size if host else c.numel()) == 0:
        raise ValueError("cost batch is empty")
    if host and not np.isfinite(c).all():
        raise ValueError("costs must be finite")
    if not host and not bool(torch.isfinite(c).all()):
        raise ValueError("costs must be finite")
    if lam <= 0.0:
        raise ValueError(f"temperature must be positive, got {lam}")
    dev = D.device()
    c_dev = _as_device(c.reshape(-1) if host else c.reshape(-1), dev, torch.float64)
    m = c_dev.numel()
    w = torch.empty(m, dtype=torch.float64, device=dev)
    stats = torch.empty(4, dtype=torch.float64, device=dev)
    L = load()
    ws = D.Workspace.get(dev, "softmin", int(L.vpb_soft_weights_workspace_bytes(m)))
    check(L.vpb_soft_weights(D.ptr(c_dev), m, float(lam), D.ptr(w), D.ptr(stats), D.ptr(ws), ws.numel(),
                             D.stream(dev)), "soft_weights")
    return w.cpu().numpy() if host else w


def update_controls(nominal, perturbations, weights):
    """nominal + sum_m w_m eps_m on the device, with the reference's checks."""
    host = not torch.is_tensor(perturbations)
    w_np = weights.detach().cpu().numpy() if torch.is_tensor(weights) else np.asarray(weights, dtype=float)
    if abs(w_np.sum() - 1.0) > 1e-9:
        raise WeightMismatch(f"weights sum to {w_np.sum()!r}, expected 1")
    m = perturbations.shape[0]
    if w_np.shape[0] != m:
        raise WeightMismatch(f"{w_np.shape[0]} weights for {m} samples")
    dev = D.device()
    nom = _as_device(nominal, dev, torch.float64)
    eps = perturbations.to(dev).contiguous() if not host else _as_device(perturbations, dev, torch.float64)
    hn = nom.numel()
    w_dev = _as_device(w_np, dev, torch.float64)
    out = torch.empty_like(nom)
    L = load()
    ws = D.Workspace.get(dev, "update", int(L.vpb_update_controls_workspace_bytes(m, hn)))
    dtype = DTYPE_F32 if eps.dtype == torch.float32 else DTYPE_F64
    check(L.vpb_update_controls(D.ptr(nom), D.ptr(eps), dtype, D.ptr(w_dev), m, hn, D.ptr(out), D.ptr(ws),
                                ws.numel(), D.stream(dev)), "update_controls")
    return out.cpu().numpy() if host else out


def sample_perturbations(params: PlannerParams, rng_seed: int, device=None, dtype=torch.float64) -> torch.Tensor:
    """On-device counterpart of vp/planner.py:199-219 ((M, H, n) CUDA tensor).
    Statistically equivalent to the reference's numpy stream, not bitwise."""
    dev = D.device(device)
    out = torch.empty((params.samples, params.horizon, params.dof), dtype=dtype, device=dev)
    sig = np.ascontiguousarray(params.sigma, dtype=np.float64)
    check(load().vpb_sample_perturbations(
        int(rng_seed) & 0xFFFFFFFFFFFFFFFF, None, 0, params.samples, params.horizon, params.dof, params.noise_window,
        D.host_ptr(sig), DTYPE_F32 if dtype == torch.float32 else DTYPE_F64, D.ptr(out), D.stream(dev)),
        "sample_perturbations")
    return out


class SmpcGraph:
    """One single-device SMPC step captured as a CUDA graph.

    The graph holds: host->device copy of the per-call block (start state,
    goal, seed, nominal) from pinned memory, the on-device sampler, the fused
    one-kernel SMPC step and the device->host copy of the packed result.  A
    call writes the pinned block, replays the graph and waits for the result,
    so the host does no per-launch work.  The distance field is part of the
    captured launch; use one graph per field buffer (the mapper's pipeline
    keeps its field buffer fixed).
    """

    def __init__(self, planner: Planner, snap, samples: int | None = None):
        self.pl = planner
        p = planner.params
        self.m = int(samples or p.samples)
        self.h, self.n = p.horizon, planner.chain.dof
        dev = planner.device
        n = self.n
        L = load()
        self.dyn_len = 2 * n + 12
        # [dyn (2n + 12) | seed (1, as uint64 bits) | nominal (H n)]
        self.block_len = self.dyn_len + 1 + self.h * n
        self.host_in = torch.zeros(self.block_len, dtype=torch.float64).pin_memory()
        self.dev_in = torch.zeros(self.block_len, dtype=torch.float64, device=dev)
        self.out_len = int(L.vpb_smpc_out_len(self.h, n))
        self.dev_out = torch.zeros(self.out_len, dtype=torch.float64, device=dev)
        self.host_out = torch.zeros(self.out_len, dtype=torch.float64).pin_memory()
        self.eps = torch.empty((self.m, self.h, n), dtype=planner._eps_dtype, device=dev)
        self.snap = snap
        self._seed_view = self.dev_in[self.dyn_len:self.dyn_len + 1].view(torch.int64)
        self._nom_view = self.dev_in[self.dyn_len + 1:].view(self.h, n)
        self._dyn_view = self.dev_in[:self.dyn_len]
        self.planner_ws = planner._smpc_ws(self.m, self.h)
        # warm once outside capture (workspace, kernel attributes)
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
        self.dev_in.copy_(self.host_in, non_blocking=True)
        self.pl.smpc_generate_device(None, None, self.snap, self._nom_view, 0, samples=self.m,
                                     seed_dev=self._seed_view, dyn=self._dyn_view, eps_out=self.eps,
                                     out=self.dev_out)
        if copy_out:
            self.host_out.copy_(self.dev_out, non_blocking=True)

    def stage(self, state: JointState, goal: RigidTransform, nominal, rng_seed: int) -> None:
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

    def step(self, state: JointState, goal: RigidTransform, nominal, rng_seed: int) -> StepResult:
        """Public-API step with host buffers (same contract as Planner.smpc_step)."""
        self.stage(state, goal, nominal, rng_seed)
        self.graph.replay()
        torch.cuda.current_stream(self.pl.device).synchronize()
        return self.pl.unpack_step(self.host_out.numpy().copy(), state, goal, self.h)


def _raw_stream(device_index: int) -> int:
    """Current CUDA stream handle of the device (the cheap torch binding)."""
    return torch._C._cuda_getCurrentRawStream(device_index)


class SmpcSession:
    """Native single-device step (``vpb_smpc_session_*``): the per-call block
    goes to pinned memory, one captured CUDA graph runs H2D -> sampler ->
    fused step -> D2H on the caller's stream, and the host reads the packed
    result.  The field geometry is fixed per session; its buffer may change
    from step to step (the mapper rebuilds the EDT into a new tensor)."""

    def __init__(self, planner: Planner, snap, samples: int):
        self.pl = planner
        p = planner.params
        self.h, self.n, self.m = p.horizon, planner.chain.dof, int(samples)
        L = load()
        self._lib = L
        _release_pending_sessions()
        P = planner.problem(None, None)
        self._sigma = np.ascontiguousarray(np.broadcast_to(np.asarray(p.sigma, dtype=float), (self.n,)))
        handle = ctypes.c_void_p()
        torch.cuda.set_device(planner.device)
        check(L.vpb_smpc_session_create(P, _field_struct(snap), self.m, p.noise_window, D.host_ptr(self._sigma),
                                        planner._prec, ctypes.byref(handle)), "smpc_session_create")
        self._h = handle
        self.out = np.zeros(int(L.vpb_smpc_session_out_len(self.h, self.n)))
        # [q0 (n) | qd0 (n) | goal R (9) | goal t (3)]: filled by one concatenate per step
        self._blk = np.zeros(2 * self.n + 12)
        self._q0, self._qd0 = self._blk[:self.n], self._blk[self.n:2 * self.n]
        self._gr, self._gt = self._blk[2 * self.n:2 * self.n + 9], self._blk[2 * self.n + 9:]
        self._nom = np.zeros((self.h, self.n))
        # the per-step call passes plain integers (no per-call ctypes objects)
        self._p_q0, self._p_qd0 = self._q0.ctypes.data, self._qd0.ctypes.data
        self._p_gr, self._p_gt, self._p_out = self._gr.ctypes.data, self._gt.ctypes.data, self.out.ctypes.data
        self._p_nom = self._nom.ctypes.data
        self._step = L.vpb_smpc_session_step
        self._dev_index = planner.device.index if planner.device.index is not None else torch.cuda.current_device()

    def step(self, state: JointState, goal: RigidTransform, nominal: np.ndarray, rng_seed: int, snap) -> StepResult:
        n = self.n
        q0, qd0 = state.q, state.qd
        if q0.shape != (n,) or qd0.shape != (n,):
            raise DimensionMismatch("state does not match the chain's dof")
        np.concatenate((q0, qd0, goal.rotation.matrix.reshape(-1), goal.translation), out=self._blk)
        self._nom[...] = nominal
        f = _field_of(snap)
        sq = f._sq_ptr if f is not None else None
        rc = self._step(self._h, self._p_q0, self._p_qd0, self._p_gr, self._p_gt, self._p_nom,
                        int(rng_seed) & 0xFFFFFFFFFFFFFFFF, sq, self._p_out, _raw_stream(self._dev_index))
        if rc:
            check(rc, "smpc_session_step")
        return self.pl.unpack_step(self.out, state, goal, self.h)

    def launch(self) -> None:
        """Replay the step graph asynchronously with the last staged inputs
        (device-side timing, no result).  The next ``step`` or ``launch`` waits
        for this replay before it restages the inputs."""
        check(self._lib.vpb_smpc_session_launch(self._h, D.stream(self.pl.device)), "smpc_session_launch")

    def close(self) -> None:
        """Release the native session now (not during a stream capture)."""
        h = getattr(self, "_h", None)
        self._h = None
        if h is not None and h.value:
            check(self._lib.vpb_smpc_session_destroy(h), "smpc_session_destroy")

    def __del__(self):
        # The garbage collector may run this while some stream is capturing a
        # CUDA graph, where the cudaFree / cudaStreamDestroy of the native
        # destroy would invalidate that capture: park the handle and release
        # it at the next session creation instead.
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _PENDING_DESTROY.append((self._lib, h))
            self._h = None


_PENDING_DESTROY: list = []


def _release_pending_sessions() -> None:
    while _PENDING_DESTROY:
        lib, h = _PENDING_DESTROY.pop()
        lib.vpb_smpc_session_destroy(h)
