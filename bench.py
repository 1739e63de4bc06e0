"""Benchmark of the B200 mapping-and-planning hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0.  The headline `value` is SMPC rollouts/s (7-DoF,
H=32): each step is one full SMPC iteration per rank (on-device noise,
fused rollout + cost kernel, per-CTA softmin partials, fixed-order merge,
NCCL all-gather of the shard partials when N > 1, U*, M=1 re-evaluation,
clip/shift) with M=4096 samples per rank (weak scaling) on the distance
field of the C2 scene (256^3 bench grid, 7-DoF body mask).  The same run
also times the C2 map update (masked fusion + exact EDT, EDT Mvoxel/s) and
the replan (fusion + EDT + SMPC, p50 ms).  L2 is flushed between timed
steps; every timing uses CUDA events on the launching stream, max over
ranks.  `e2e` repeats the SMPC step through the public Planner.smpc_step API
with host-resident nominal in and the step result out.

`--impl reference` times the CPU restatement of the reference's own path
(oracle/: numpy sampler identical to the reference's + C float64 rollout
with all host threads + softmin/update + M=1 re-evaluation) on the same
config; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SMPC rollouts/s (7-DoF, H=32)"
UNIT = "rollouts/s"
# algorithmic cost figures
FLOP_PER_ROLLOUT_STEP = 2294.0
FLOP_PER_ROLLOUT_TERMINAL = 1217.0
EDT_BYTES_PER_VOXEL = 5.0
FUSION_BYTES_PER_TOUCHED = 18.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--samples", type=int, default=4096, help="rollouts per rank")
    ap.add_argument("--horizon", type=int, default=32)
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1 / C5 replan measurements")
    ap.add_argument("--c5-frames", type=int, default=100)
    ap.add_argument("--dist-backend", default="nccl",
                    help="nccl (one GPU per rank); gloo lets several ranks share one GPU to exercise the sharded "
                         "path on a 1-GPU box")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.idx), "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        finally:
            if self.path:
                try:
                    os.unlink(self.path)
                except OSError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ncu_traffic() -> dict:
    """DRAM bytes per launch of the step's kernels from the committed ncu
    capture (profiles/r1_ncu_traffic.json, tools/ncu_traffic.py)."""
    p = ROOT / "profiles" / "r1_ncu_traffic.json"
    if p.exists():
        return {k: v["bytes"] for k, v in json.loads(p.read_text()).items()}
    return {}


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


# ----------------------------------------------------------------------------- scene
def make_scene(args, dev):
    from paper_2512_22575_b200 import config, mapping, planner, robot, scene

    chain, model = config.robot_7dof()
    q_mask = np.full(7, 0.3)
    centers, radii = robot.sphere_positions(chain, q_mask, model)
    n = args.grid
    grid, cam, depth = scene.bench_edt_scene((n, n, n), robot_spheres=(centers, radii), device=dev)
    mapper = mapping.OccupancyMapper(grid, cam, outside_default=0.8)
    # touched voxels per update (fresh grid, one update): the fusion roofline unit
    mapper.update(depth, mask=(centers, radii))
    touched = int(grid.observed.sum().item())
    mapper.update(depth, mask=(centers, radii))  # 2 hits -> occupied surface
    field = mapper.recompute_edt()
    params = config.planner_params(7, {"samples": args.samples, "horizon": args.horizon})
    pl = planner.Planner(chain, model, params, precision=args.precision, device=dev)
    state = robot.JointState.resting(np.full(7, 0.05))
    goal = robot.forward_kinematics(chain, np.full(7, 0.35))[-1]
    return dict(chain=chain, model=model, centers=centers, radii=radii, grid=grid, cam=cam, depth=depth,
                mapper=mapper, field=field, params=params, planner=pl, state=state, goal=goal, touched=touched)


# ----------------------------------------------------------------------------- closed loop (C1, C5)
def closed_loop(dev, dims, samples, horizon, frames, warm=3):
    """p50 replan ms over `frames` frames of a moving-obstacle scene: per frame
    the masked update of a rendered depth image (host render, untimed), the
    exact EDT of the whole grid and one SMPC step through the public API
    (native session; the field buffer changes every frame), then the
    executed command is integrated.  SURVEY.md 8d C1 / C5."""
    import torch

    from paper_2512_22575_b200 import config, mapping, planner, robot, scene

    chain, model = config.robot_7dof()
    grid, cam, _ = scene.bench_edt_scene(dims, device=dev)
    mapper = mapping.OccupancyMapper(grid, cam, outside_default=0.8)
    params = config.planner_params(7, {"samples": samples, "horizon": horizon})
    pl = planner.Planner(chain, model, params, device=dev)
    state = robot.JointState.resting(np.full(7, 0.05))
    goal = robot.forward_kinematics(chain, np.full(7, 0.35))[-1]
    nominal = np.zeros((horizon, 7))
    seq = scene.moving_obstacle_frames(cam, dims, frames + warm, chain, model)
    depths = [mapping.DepthImage(d) for d, _ in seq]
    masks = [m for _, m in seq]
    stream = torch.cuda.current_stream(dev)
    times = []
    for f in range(frames + warm):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        mapper.update(depths[f], mask=masks[f])
        field = mapper.recompute_edt()
        res = pl.smpc_step(state, goal, field, nominal, f)
        e1.record(stream)
        e1.synchronize()
        if f >= warm:
            times.append(e0.elapsed_time(e1))
        state = pl.integrate(state, res.command)
        nominal = res.next_nominal
    return {"metric": "p50 replan ms", "value": statistics.median(times), "unit": "ms",
            "p90": float(np.percentile(times, 90)), "frames": frames, "grid": list(dims), "samples": samples,
            "horizon": horizon,
            "per_frame": "masked fusion (160x120 depth, 11-sphere body mask) + exact EDT of the whole grid + "
                         "Planner.smpc_step (host in/out); depth rendered on the host, untimed"}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2512_22575_b200 import _lib, distributed

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dist_backend != "nccl":
        local = local % torch.cuda.device_count()  # ranks may share a device (path check, not a measurement)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    S = make_scene(args, dev)
    pl, state, goal, field, mapper = S["planner"], S["state"], S["goal"], S["field"], S["mapper"]
    M, H, n = args.samples, args.horizon, 7
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    nominal = torch.zeros((H, n), dtype=torch.float64, device=dev)
    sharded = distributed.ShardedSMPC(pl, world=world, rank=rank)

    def smpc_iteration(seed):
        return sharded.step_device(state, goal, field, nominal, seed)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps, warmup, flush_between=True):
        for w in range(warmup):
            fn(w)
        barrier()
        times = []
        l0 = lib.vpb_launch_count()
        for k in range(steps):
            if flush_between:
                flush.fill_(k & 0xFF)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(1000 + k)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        launches = lib.vpb_launch_count() - l0
        barrier()
        return times, launches

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local]) if \
        os.environ.get("CUDA_VISIBLE_DEVICES") else local

    # --- A: SMPC iterations (headline) ---------------------------------------
    # single device: the step is captured once as a CUDA graph (staged state
    # copy + sampler + one fused SMPC kernel + result copy) and replayed;
    # multi-device: sampler + fused partial kernel + NCCL all-gather + finish.
    graph = None
    if world == 1:
        # the production path: the native session's captured step graph
        # (H2D of the 1.8 KB per-call block -> fused step kernel that draws the
        # noise and writes the result into pinned host memory), replayed on
        # the stream with the inputs staged by one public-API step
        graph = pl.session(field, M)
        graph.step(state, goal, np.zeros((H, n)), 0, field)

        def smpc_iteration(seed):
            graph.launch()
    elif args.dist_backend == "nccl":
        # one CUDA graph per rank: draw + rollout + shard partial, NCCL
        # all-gather, rank-order merge + tail (eager fallback if capture fails)
        try:
            graph = distributed.ShardedGraph(sharded, field)
            graph.stage(state, goal, None, 0)

            def smpc_iteration(seed):
                graph.replay()
        except Exception as exc:  # pragma: no cover - depends on the NCCL build
            graph = None
            print(f"sharded graph capture failed, eager step: {exc}", file=sys.stderr)
    with ClockSampler(gpu_index) as clk:
        t_smpc, launches_smpc = timed(smpc_iteration, args.steps, args.warmup)
    clocks = clk.summary()
    ms_smpc = max_over_ranks(statistics.mean(t_smpc))
    value = world * M / (ms_smpc * 1e-3)
    t_direct, _ = timed(lambda k: sharded.step_device(state, goal, field, nominal, k), args.steps, args.warmup)
    ms_direct = max_over_ranks(statistics.mean(t_direct))
    if graph is not None:
        # per replay: the fused SMPC kernel (N=1); fused partial + finish kernels (N>1)
        launches_smpc = args.steps * (1 if world == 1 else 2)

    # rollout kernel alone (dominant kernel) for the roofline
    eps = pl.sample_device(7, m_offset=rank * M, samples=M)

    def rollout_only(k):
        pl.evaluate_device(state, goal, field, eps, nominal)

    t_roll, _ = timed(rollout_only, args.steps, args.warmup)
    ms_roll = statistics.mean(t_roll)

    # the step's dominant kernel alone: the fused SMPC kernel (draws + rollout +
    # softmin + merge + U* + re-evaluation), one launch (+ its counter memset)
    gen_eps = torch.empty((M, H, n), dtype=torch.float32 if args.precision == "fp32" else torch.float64, device=dev)
    gen_out = torch.empty(int(lib.vpb_smpc_out_len(H, n)), dtype=torch.float64, device=dev)

    def fused_only(k):
        pl.smpc_generate_device(state, goal, field, nominal, k, samples=M, m_offset=rank * M, eps_out=gen_eps,
                                out=gen_out)

    t_fused, _ = timed(fused_only, args.steps, args.warmup)
    ms_fused = statistics.mean(t_fused)


    # --- B: map update (C2): masked fusion and EDT timed separately -----------
    depth_dev = S["depth"]
    depth_dev.device_tensor(dev)
    mask = (S["centers"], S["radii"])

    def fusion(k):
        mapper.update(depth_dev, mask=mask)

    def edt(k):
        mapper.recompute_edt()

    t_fus, _ = timed(fusion, args.steps, args.warmup)
    t_edt, launches_edt = timed(edt, args.steps, args.warmup)
    ms_fus, ms_edt = max_over_ranks(statistics.mean(t_fus)), max_over_ranks(statistics.mean(t_edt))
    vox = args.grid ** 3

    # --- C: full replan (fusion + EDT + SMPC) ----------------------------------
    def replan(k):
        mapper.update(depth_dev, mask=mask)
        f = mapper.recompute_edt()
        sharded.step_device(state, goal, f, nominal, k)

    t_replan, launches_replan = timed(replan, args.steps, args.warmup)
    p50_replan = max_over_ranks(statistics.median(t_replan))

    # --- e2e: public API, host buffers ------------------------------------------
    nominal_host = np.zeros((H, n))

    def e2e_step(k):
        if world == 1:
            pl.smpc_step(state, goal, field, nominal_host, k)
        else:
            sharded.step(state, goal, field, nominal_host, k)

    t_e2e, _ = timed(e2e_step, args.steps, args.warmup)
    ms_e2e = max_over_ranks(statistics.mean(t_e2e))
    ms_e2e_graph = None
    h2d = nominal_host.nbytes
    d2h = int(lib.vpb_smpc_out_len(H, n)) * 8

    peaks = measured_peaks()
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = sm_count * 128 * 2 * clk_mhz * 1e6 / 1e12  # TFLOP/s at max clock
    roll_flops = (FLOP_PER_ROLLOUT_STEP * H + FLOP_PER_ROLLOUT_TERMINAL) * M
    roll_tflops = roll_flops / (ms_roll * 1e-3) / 1e12
    fused_tflops = roll_flops / (ms_fused * 1e-3) / 1e12
    traffic = ncu_traffic()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    edt_gbs = EDT_BYTES_PER_VOXEL * vox / (ms_edt * 1e-3) / 1e9
    fus_gbs = FUSION_BYTES_PER_TOUCHED * S["touched"] / (ms_fus * 1e-3) / 1e9

    configs = {}
    if rank == 0 and world == 1 and not args.no_configs:
        configs["c1"] = closed_loop(dev, (64, 64, 64), 256, 20, 20)
        configs["c5"] = closed_loop(dev, (512, 512, 512), 16384, 32, args.c5_frames)
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, S)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_smpc, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
            "data": "synthetic (CLI bench scene 256^3 + 7-DoF body mask; on-device smoothed Gaussian noise)",
            "config": {
                "workload": f"C3: SMPC iteration M={M}/rank x H={H}, 7-DoF robot_7dof, field = C2 256^3 masked map",
                "samples_per_rank": M, "horizon": H, "grid": [args.grid] * 3, "precision": args.precision,
                "l2": "flushed between timed steps (256 MiB write)",
                "parallelism": f"rollouts sharded over {world} GPU(s); NCCL all-gather of softmin partials",
            },
            "edt": {"metric": "EDT Mvoxel/s at 256^3", "value": vox / (ms_edt * 1e-3) / 1e6, "unit": "Mvoxel/s",
                    "ms": ms_edt},
            "fusion": {"metric": "masked fusion Mvoxel/s at 256^3", "value": vox / (ms_fus * 1e-3) / 1e6,
                       "unit": "Mvoxel/s", "ms": ms_fus, "touched_voxels": S["touched"]},
            "replan": {"metric": "p50 replan ms (fusion + EDT 256^3 + SMPC M x H)", "value": p50_replan,
                       "unit": "ms", "launches_per_step": launches_replan / max(1, args.steps)},
            "roofline": {"kernel": "smpc_kernel (fused step: draws + rollout + softmin + U* + re-evaluation)",
                         "bound": "fp32", "achieved": fused_tflops, "peak": fp32_peak, "unit": "TFLOP/s",
                         "frac": fused_tflops / fp32_peak, "traffic": traffic.get("smpc_kernel"),
                         "traffic_unit": "bytes/launch", "ms": ms_fused,
                         "note": "FP32-issue-bound: achieved = (2294 FLOP/rollout-step x H + 1217/rollout) x M "
                                 "(SURVEY.md 8d) / CUDA-event time of one fused launch, L2 flushed; peak = SMs x "
                                 "128 x 2 x sm_max_mhz (no FP32 entry in MEASURED_PEAKS.json); traffic = ncu "
                                 "dram__bytes_read+write of the kernel (profiles/r1_ncu_traffic.json)"},
            "rooflines": [
                {"kernel": "rollout_kernel (evaluate_batch alone)", "bound": "fp32", "achieved": roll_tflops,
                 "peak": fp32_peak, "unit": "TFLOP/s", "frac": roll_tflops / fp32_peak, "ms": ms_roll},
                {"kernel": "edt (line table + Z+Y FH + X FH)", "bound": "hbm", "achieved": edt_gbs, "peak": hbm,
                 "unit": "GB/s", "frac": edt_gbs / hbm, "bytes_per_voxel": EDT_BYTES_PER_VOXEL,
                 "traffic": traffic.get("edt"), "traffic_unit": "bytes/call"},
                {"kernel": "fuse+masked_pixels", "bound": "hbm", "achieved": fus_gbs, "peak": hbm, "unit": "GB/s",
                 "frac": fus_gbs / hbm, "bytes_per_touched_voxel": FUSION_BYTES_PER_TOUCHED,
                 "traffic": traffic.get("fuse_kernel"), "traffic_unit": "bytes/call"},
            ],
            "e2e": {"value": world * M / (ms_e2e * 1e-3), "unit": UNIT, "ms": ms_e2e, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "api": "Planner.smpc_step (N=1: native session, vpb_smpc_session_step) / ShardedSMPC.step "
                           "(N>1): host state / goal / nominal in, StepResult out"},
            "launch_mode": ("native session CUDA graph" if world == 1 else "per-rank CUDA graph with NCCL all-gather")
                           if graph is not None else "direct",
            "direct_launch_ms_per_step": ms_direct,
            "gpu_launches": int(launches_smpc),
            "clocks": clocks,
            "peaks_source": "MEASURED_PEAKS.json (measured)" if not peaks.get("_fallback") else "fallback",
        }
        if configs:
            line["configs"] = configs
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- CPU port
def _oracle_args(S, field_sq, field_lo, field_origin, voxel, outside):
    from paper_2512_22575_b200 import planner

    chain, model, params, state, goal = S["chain"], S["model"], S["params"], S["state"], S["goal"]
    args = {
        "q0": state.q, "qd0": state.qd, "dt": params.dt, "base_r": chain.base_pose.rotation.matrix,
        "base_t": chain.base_pose.translation,
        "off_r": np.array([j.parent_offset.rotation.matrix for j in chain.joints]),
        "off_t": np.array([j.parent_offset.translation for j in chain.joints]),
        "axes": np.array([j.axis for j in chain.joints]), "sph_link": np.array([s.link for s in model.spheres]),
        "sph_loc": np.array([s.center for s in model.spheres]), "sph_r": model.radii(),
        "pairs": np.array(model.self_pairs), "goal_r": goal.rotation.matrix, "goal_t": goal.translation,
        "pose_weight": params.pose_weight, "terminal_weight": params.terminal_weight, "w_env": params.w_env,
        "w_self": params.w_self, "w_q": params.w_q, "w_qd": params.w_qd, "w_qdd": params.w_qdd, "w_s": params.w_s,
        "w_ns": params.w_ns, "d_act": params.d_act, "q_ref": params.q_ref, "field_sq": field_sq,
        "field_lo0": field_lo[0], "field_lo1": field_lo[1], "field_lo2": field_lo[2],
        "field_origin0": field_origin[0], "field_origin1": field_origin[1], "field_origin2": field_origin[2],
        "field_voxel": voxel, "field_outside": outside,
    }
    for k, v in zip(("pos_lo", "pos_hi", "vel_lo", "vel_hi", "acc_lo", "acc_hi"),
                    planner.tightened_limits(chain, params.margin_frac)):
        args[k] = v
    return args


def cpu_smpc_port(S, field_sq, reps: int, seed0: int = 0):
    """Reference smpc_step restated on the host (numpy sampler + C rollout)."""
    import oracle

    p = S["params"]
    args = _oracle_args(S, field_sq, (0, 0, 0), S["grid"].origin, S["grid"].voxel_size, 0.8)
    times = []
    for r in range(reps):
        t0 = time.perf_counter()
        eps = oracle.sample_perturbations(p.samples, p.horizon, 7, p.sigma, p.noise_window, seed0 + r)
        oracle.smpc_step(args, np.zeros((p.horizon, 7)), eps, p.lam, S["chain"].acceleration_limits())
        times.append(time.perf_counter() - t0)
    return times


def cpu_baseline(args, S):
    import oracle

    oracle.build()
    oracle.set_threads(0)
    threads = oracle.get_threads()
    field_sq = S["field"].sq
    times = cpu_smpc_port(S, field_sq, reps=3)
    t = statistics.median(times)
    # C2 map stages on the same host (1 rep each; fusion is serial like the reference)
    lo = S["grid"].log_odds_host().copy()
    ob = S["grid"].observed_host().copy()
    cam, depth = S["cam"], S["depth"]
    pm = oracle.masked_pixels(depth.data, cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max,
                              cam.pose.rotation.matrix, cam.pose.translation, S["centers"], S["radii"], 0.01)
    r, tt = cam.world_to_camera()
    t0 = time.perf_counter()
    oracle.fuse_voxels(lo, ob, (0, 0, 0), S["grid"].dims, S["grid"].origin, S["grid"].voxel_size, r, tt, cam.fx,
                       cam.fy, cam.cx, cam.cy, cam.width, cam.height, cam.d_min, cam.d_max, depth.data, pm,
                       S["centers"], S["radii"], S["grid"].tau, 0.85, -0.4, -2.0, 3.5)
    t_fus = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.edt3d(lo)
    t_edt = time.perf_counter() - t0
    vox = args.grid ** 3
    return {
        "value": args.samples / t, "unit": UNIT, "cores": threads, "kind": "port",
        "sample": f"3 smpc_step reps at M={args.samples}, H={args.horizon} (numpy Philox sampler as the "
                  f"reference + C fp64 rollout on {threads} threads); 1 rep each of serial masked fusion and "
                  f"EDT at {args.grid}^3",
        "smpc_step_ms": t * 1e3, "fusion_ms": t_fus * 1e3, "edt_ms": t_edt * 1e3,
        "edt_mvoxel_s": vox / t_edt / 1e6, "cpu": cpu_model(),
    }


def run_reference(args):
    """--impl reference: the reference's path restated on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import torch

    oracle.build()
    oracle.set_threads(0)
    threads = oracle.get_threads()
    # the same scene, built on the GPU for convenience and copied to the host
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else None
    if dev is None:
        print(json.dumps({"impl": "reference", "unavailable": "scene generation needs the CUDA grid"}))
        return
    args.samples = args.samples * max(1, args.gpus)  # the whole job's rollouts per step
    S = make_scene(args, dev)
    field_sq = S["field"].sq
    cpu_smpc_port(S, field_sq, reps=max(1, min(args.warmup, 3)))
    times = cpu_smpc_port(S, field_sq, reps=args.steps, seed0=1000)
    t = statistics.mean(times)
    value = args.samples / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C3: SMPC iteration M={args.samples} x H={args.horizon}, 7-DoF, C2 256^3 field",
                   "samples_per_rank": args.samples, "horizon": args.horizon, "grid": [args.grid] * 3},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full smpc_step iterations (numpy sampler identical to the "
                                   f"reference + C fp64 rollout/softmin/update on {threads} threads)",
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
