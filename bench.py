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

Also in the line (N=1 unless noted): `c4` = C4 strong scaling (65,536
rollouts x H=64 split over the ranks; every N), `c2` = the EDT at random
occupancy 0.01/0.1/0.5 and the full-coverage fusion scene, the other
arithmetic precision of the same step (`fp64`), `c3_converged` = C3 in the
converged many-weights regime, `configs` = C1/C5 closed loops, and
`cpu_baseline` = the reference path restated on the host cores.

`--impl reference` times the CPU restatement of the reference's own path
(oracle/: numpy sampler identical to the reference's + C float64 rollout
with all host threads + softmin/update + M=1 re-evaluation) on the same
config, with the scene also built on the host by the oracle (no product
code is imported); rank 0 only.
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
FUSION_FLOP_PER_BOX_VOXEL = 30.0  # fp64 projection ~30 flop per voxel of the box


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
    ap.add_argument("--c4-samples", type=int, default=65536, help="C4 total rollouts, split over the ranks")
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
    capture (profiles/ncu_traffic.json, tools/ncu_traffic.py)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
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
        mapper.recompute_edt()
        snap = mapper.snapshot()  # inside map_ms like vp/sim.py:476-480 (O(1): copy-on-write)
        res = pl.smpc_step(state, goal, snap, nominal, f)
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
                         "mapper.snapshot() + Planner.smpc_step on the snapshot (host in/out); depth rendered on "
                         "the host, untimed"}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2512_22575_b200 import _lib, config, distributed, mapping, planner, robot, scene

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
    single = world == 1
    S = make_scene(args, dev)
    pl, state, goal, field, mapper = S["planner"], S["state"], S["goal"], S["field"], S["mapper"]
    M, H, n = args.samples, args.horizon, 7
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    nominal = torch.zeros((H, n), dtype=torch.float64, device=dev)
    sharded = distributed.ShardedSMPC(pl, world=world, rank=rank)

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

    def step_runner(p_, fld, st, gl, nom_host, m_local):
        """One SMPC iteration per call, as production launches it: N=1 the
        native session's captured graph (H2D of the per-call block -> fused
        draw + rollout + softmin + U* + re-evaluation -> result into pinned
        host memory); N>1 one CUDA graph per rank (fused draw + shard partial,
        NCCL all-gather, rank-order merge + tail).  Inputs staged once."""
        if single:
            sess = p_.session(fld, m_local)
            sess.step(st, gl, nom_host, 0, fld)
            return (lambda k: sess.launch()), "native session CUDA graph", 1
        sh = distributed.ShardedSMPC(p_, world=world, rank=rank, samples_per_rank=m_local)
        if args.dist_backend == "nccl":
            try:
                g = distributed.ShardedGraph(sh, fld)
                g.stage(st, gl, nom_host, 0)
                return (lambda k: g.replay()), "per-rank CUDA graph with NCCL all-gather", 2
            except Exception as exc:  # pragma: no cover - depends on the NCCL build
                print(f"sharded graph capture failed, eager step: {exc}", file=sys.stderr)
        nom_dev = torch.from_numpy(np.ascontiguousarray(nom_host)).to(dev)
        return (lambda k: sh.step_device(st, gl, fld, nom_dev, k)), "direct", 2

    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local]) if \
        os.environ.get("CUDA_VISIBLE_DEVICES") else local

    # --- A: SMPC iterations (headline, C3 per rank) ----------------------------
    smpc_iteration, launch_mode, kernels_per_step = step_runner(pl, field, state, goal, np.zeros((H, n)), M)
    with ClockSampler(gpu_index) as clk:
        t_smpc, _ = timed(smpc_iteration, args.steps, args.warmup)
    clocks = clk.summary()
    ms_smpc = max_over_ranks(statistics.mean(t_smpc))
    value = world * M / (ms_smpc * 1e-3)
    launches_smpc = args.steps * kernels_per_step
    t_direct, _ = timed(lambda k: sharded.step_device(state, goal, field, nominal, k), args.steps, args.warmup)
    ms_direct = max_over_ranks(statistics.mean(t_direct))

    # rollout kernel alone (evaluate_batch seam) and the fused step kernel alone
    eps = pl.sample_device(7, m_offset=rank * M, samples=M)
    t_roll, _ = timed(lambda k: pl.evaluate_device(state, goal, field, eps, nominal), args.steps, args.warmup)
    ms_roll = statistics.mean(t_roll)
    gen_eps = torch.empty((M, H, n), dtype=torch.float32 if args.precision == "fp32" else torch.float64, device=dev)
    gen_out = torch.empty(int(lib.vpb_smpc_out_len(H, n)), dtype=torch.float64, device=dev)

    def fused_only(k):
        pl.smpc_generate_device(state, goal, field, nominal, k, samples=M, m_offset=rank * M, eps_out=gen_eps,
                                out=gen_out)

    t_fused, _ = timed(fused_only, args.steps, args.warmup)
    ms_fused = statistics.mean(t_fused)

    # --- C4: 65,536 rollouts x H = 64 split over the ranks (strong scaling) ----
    c4 = None
    if not args.no_configs:
        m4 = args.c4_samples // world
        p4 = config.planner_params(7, {"samples": m4, "horizon": 64})
        pl4 = planner.Planner(S["chain"], S["model"], p4, precision=args.precision, device=dev)
        fn4, mode4, k4 = step_runner(pl4, field, state, goal, np.zeros((64, n)), m4)
        t4, _ = timed(fn4, args.steps, args.warmup)
        ms4 = max_over_ranks(statistics.mean(t4))
        c4 = {"metric": "SMPC rollouts/s (7-DoF, H=64), C4 strong scaling", "value": m4 * world / (ms4 * 1e-3),
              "unit": UNIT, "ms_per_step": ms4, "total_samples": m4 * world, "samples_per_rank": m4, "horizon": 64,
              "n_gpus": world, "scaling": "strong", "launch_mode": mode4,
              "note": "efficiency = T1 / (N * T_N) from the per-N lines (driver-computed)"}
        del pl4
        torch.cuda.empty_cache()

    # --- B: map update (C2): masked fusion and EDT timed separately -----------
    depth_dev = S["depth"]
    depth_dev.device_tensor(dev)
    mask = (S["centers"], S["radii"])
    t_fus, _ = timed(lambda k: mapper.update(depth_dev, mask=mask), args.steps, args.warmup)
    t_edt, launches_edt = timed(lambda k: mapper.recompute_edt(), args.steps, args.warmup)
    ms_fus, ms_edt = max_over_ranks(statistics.mean(t_fus)), max_over_ranks(statistics.mean(t_edt))
    vox = args.grid ** 3

    c2 = None
    if single and not args.no_configs:
        # EDT on random occupancy (t/test_acceptance.py:60-68 style) and the
        # full-coverage fusion variant (a backdrop behind the volume)
        sweep = {}
        g_r = mapping.VoxelGrid((0, 0, 0), 0.02, (args.grid,) * 3, device=dev)
        for dens in (0.01, 0.1, 0.5):
            gen = torch.Generator(device=dev).manual_seed(int(dens * 1000))
            occ = torch.rand((args.grid,) * 3, device=dev, generator=gen) < dens
            g_r.set_log_odds(torch.where(occ, 3.5, 0.0).double())
            mapping.edt_3d(g_r)
            t_d, _ = timed(lambda k: mapping.edt_3d(g_r), args.steps, args.warmup)
            md = statistics.mean(t_d)
            sweep[str(dens)] = {"ms": md, "mvoxel_s": vox / (md * 1e-3) / 1e6,
                                "hbm_frac": EDT_BYTES_PER_VOXEL * vox / (md * 1e-3) / 1e9 / hbm_peak()}
        del g_r, occ
        grid_f, cam_f, depth_f = scene.bench_edt_scene((args.grid,) * 3, backdrop=True, robot_spheres=mask,
                                                       device=dev)
        mapper_f = mapping.OccupancyMapper(grid_f, cam_f, outside_default=0.8)
        depth_f.device_tensor(dev)
        mapper_f.update(depth_f, mask=mask)
        touched_f = int(grid_f.observed.sum().item())
        t_ff, _ = timed(lambda k: mapper_f.update(depth_f, mask=mask), args.steps, args.warmup)
        t_fe, _ = timed(lambda k: mapper_f.recompute_edt(), args.steps, args.warmup)
        del grid_f, mapper_f
        torch.cuda.empty_cache()
        c2 = {"edt_random_occupancy": sweep,
              "full_coverage": {"fusion_ms": statistics.mean(t_ff), "edt_ms": statistics.mean(t_fe),
                                "touched_voxels": touched_f, "touched_fraction": touched_f / vox},
              "bench_scene": {"fusion_ms": ms_fus, "edt_ms": ms_edt, "touched_voxels": S["touched"],
                              "touched_fraction": S["touched"] / vox}}

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
        if single:
            pl.smpc_step(state, goal, field, nominal_host, k)
        else:
            sharded.step(state, goal, field, nominal_host, k)

    t_e2e, _ = timed(e2e_step, args.steps, args.warmup)
    ms_e2e = max_over_ranks(statistics.mean(t_e2e))
    # per step: the session's per-call block [q0, qd0, goal R, goal t | seed | field ptr | nominal]
    # host -> device, the packed step result device -> host
    h2d = (2 * n + 12 + 2 + H * n) * 8 if single else nominal_host.nbytes
    d2h = int(lib.vpb_smpc_out_len(H, n)) * 8

    # --- same-precision leg and the converged regime (single device) -------------
    extra = {}
    if single and not args.no_configs:
        prec_other = "fp64" if args.precision == "fp32" else "fp32"
        pl_o = planner.Planner(S["chain"], S["model"], S["params"], precision=prec_other, device=dev)
        fn_o, _, _ = step_runner(pl_o, field, state, goal, np.zeros((H, n)), M)
        t_o, _ = timed(fn_o, args.steps, args.warmup)
        extra[prec_other] = {"metric": METRIC, "value": M / (statistics.mean(t_o) * 1e-3), "unit": UNIT,
                             "ms_per_step": statistics.mean(t_o), "dtype": "f64" if prec_other == "fp64" else "f32",
                             "note": "same step, other arithmetic precision (fp64 = the reference's)"}
        extra["c3_converged"] = converged_c3(dev, args, timed, step_runner)

    peaks = measured_peaks()
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = sm_count * 128 * 2 * clk_mhz * 1e6 / 1e12  # TFLOP/s at max clock
    roll_flops = (FLOP_PER_ROLLOUT_STEP * H + FLOP_PER_ROLLOUT_TERMINAL) * M
    roll_tflops = roll_flops / (ms_roll * 1e-3) / 1e12
    fused_tflops = roll_flops / (ms_fused * 1e-3) / 1e12
    traffic = ncu_traffic()
    hbm = hbm_peak()
    edt_gbs = EDT_BYTES_PER_VOXEL * vox / (ms_edt * 1e-3) / 1e9
    fus_gbs = FUSION_BYTES_PER_TOUCHED * S["touched"] / (ms_fus * 1e-3) / 1e9
    # roofline = max(bytes / BW, flops / FP64 peak); the flop
    # term dominates (30 flop x every box voxel vs 18 B x the touched ones)
    fp64_peak = sm_count * 64 * 2 * clk_mhz * 1e6 / 1e12  # 64 FP64 FMA / clk / SM (nominal; not in MEASURED_PEAKS)
    fus_tflops = FUSION_FLOP_PER_BOX_VOXEL * args.grid ** 3 / (ms_fus * 1e-3) / 1e12

    configs = {}
    if rank == 0 and single and not args.no_configs:
        configs["c1"] = closed_loop(dev, (64, 64, 64), 256, 20, 20)
        configs["c5"] = closed_loop(dev, (512, 512, 512), 16384, 32, args.c5_frames)
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and single and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, S)

    if rank == 0:
        wl = "C3" if (M, H) == (4096, 32) else "custom"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_smpc, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
            "data": "synthetic (CLI bench scene 256^3 + 7-DoF body mask; on-device smoothed Gaussian noise)",
            "config": {
                "workload": f"{wl}: SMPC iteration M={M}/rank x H={H}, 7-DoF robot_7dof, field = C2 "
                            f"{args.grid}^3 masked map",
                "samples_per_rank": M, "horizon": H, "grid": [args.grid] * 3, "precision": args.precision,
                "l2": "flushed between timed steps (256 MiB write)",
                "parallelism": f"rollouts sharded over {world} GPU(s); NCCL all-gather of softmin partials",
            },
            "edt": {"metric": f"EDT Mvoxel/s at {args.grid}^3", "value": vox / (ms_edt * 1e-3) / 1e6,
                    "unit": "Mvoxel/s", "ms": ms_edt},
            "fusion": {"metric": f"masked fusion Mvoxel/s at {args.grid}^3", "value": vox / (ms_fus * 1e-3) / 1e6,
                       "unit": "Mvoxel/s", "ms": ms_fus, "touched_voxels": S["touched"]},
            "replan": {"metric": f"p50 replan ms (fusion + EDT {args.grid}^3 + SMPC M x H)", "value": p50_replan,
                       "unit": "ms", "launches_per_step": launches_replan / max(1, args.steps)},
            "roofline": {"kernel": "smpc_kernel (fused step: draws + rollout + softmin + U* + re-evaluation)",
                         "bound": "fp32", "achieved": fused_tflops, "peak": fp32_peak, "unit": "TFLOP/s",
                         "frac": fused_tflops / fp32_peak, "traffic": traffic.get("smpc_kernel"),
                         "traffic_unit": "bytes/launch", "ms": ms_fused,
                         "note": "FP32-issue-bound: achieved = (2294 FLOP/rollout-step x H + 1217/rollout) x M "
                                 "(SURVEY.md 8d) / CUDA-event time of one fused launch, L2 flushed; peak = SMs x "
                                 "128 x 2 x sm_max_mhz (no FP32 entry in MEASURED_PEAKS.json); traffic = ncu "
                                 "dram__bytes_read+write of the kernel (profiles/ncu_traffic.json)"},
            "rooflines": [
                {"kernel": "rollout_kernel (evaluate_batch alone)", "bound": "fp32", "achieved": roll_tflops,
                 "peak": fp32_peak, "unit": "TFLOP/s", "frac": roll_tflops / fp32_peak, "ms": ms_roll},
                {"kernel": "edt (all EDT launches of one edt_3d)", "bound": "hbm", "achieved": edt_gbs,
                 "peak": hbm, "unit": "GB/s", "frac": edt_gbs / hbm, "bytes_per_voxel": EDT_BYTES_PER_VOXEL,
                 "traffic": traffic.get("edt"), "traffic_unit": "bytes/call"},
                {"kernel": "fuse+masked_pixels", "bound": "fp64", "achieved": fus_tflops, "peak": fp64_peak,
                 "unit": "TFLOP/s", "frac": fus_tflops / fp64_peak, "flop_per_box_voxel": FUSION_FLOP_PER_BOX_VOXEL,
                 "hbm_gbs": fus_gbs, "hbm_frac": fus_gbs / hbm, "bytes_per_touched_voxel": FUSION_BYTES_PER_TOUCHED,
                 "note": "algorithmic work = the reference's (every box voxel projected in fp64); the kernel culls "
                         "to the frustum footprint and decides most voxels in fp32, so frac > 1 is possible",
                 "traffic": traffic.get("fuse_kernel"), "traffic_unit": "bytes/call"},
            ],
            "e2e": {"value": world * M / (ms_e2e * 1e-3), "unit": UNIT, "ms": ms_e2e, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "api": "Planner.smpc_step (N=1: native session, vpb_smpc_session_step) / ShardedSMPC.step "
                           "(N>1): host state / goal / nominal in, StepResult out"},
            "launch_mode": launch_mode,
            "direct_launch_ms_per_step": ms_direct,
            "gpu_launches": int(launches_smpc),
            "clocks": clocks,
            "peaks_source": "MEASURED_PEAKS.json (measured)" if not peaks.get("_fallback") else "fallback",
        }
        if c4 is not None:
            line["c4"] = c4
        if c2 is not None:
            line["c2"] = c2
        line.update(extra)
        if configs:
            line["configs"] = configs
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def hbm_peak() -> float:
    return float(measured_peaks().get("hbm_gbs", 6650.0))


def converged_c3(dev, args, timed, step_runner):
    """C3 (4096 x 32) in the converged regime: the reach_static board scene
    after 30 closed-loop replans (thousands of nonzero weights; the merge's
    helper-CTA path), next to the headline's single-weight regime."""
    import torch

    from paper_2512_22575_b200 import config, mapping, planner, robot, scene
    from paper_2512_22575_b200.geometry import RigidTransform

    chain, model = config.robot_7dof()
    origin, voxel, occ = scene.reach_static_occupancy()
    grid = mapping.VoxelGrid(origin, voxel, occ.shape, device=dev)
    grid.set_log_odds(np.where(occ, 3.5, 0.0))
    field = mapping.edt_3d(grid, outside_default=0.8)
    params = config.planner_params(7, {"samples": args.samples, "horizon": args.horizon,
                                       "q_ref": scene.REACH_STATIC_QREF})
    pl = planner.Planner(chain, model, params, precision=args.precision, device=dev)
    goal = RigidTransform.from_vec7(scene.REACH_STATIC_GOAL)
    state = robot.JointState.resting(scene.REACH_STATIC_START)
    nominal = np.zeros((args.horizon, 7))
    for f in range(30):
        res = pl.smpc_step(state, goal, field, nominal, 1000 + f)
        state = pl.integrate(state, res.command)
        nominal = res.next_nominal
    nom_dev = torch.from_numpy(nominal).to(dev)
    pl.smpc_generate_device(state, goal, field, nom_dev, 0, samples=args.samples)
    nnz = int((pl.smpc_weights_device(args.samples, args.horizon) > 0).sum().item())
    fn, _, _ = step_runner(pl, field, state, goal, nominal, args.samples)
    t, _ = timed(fn, args.steps, args.warmup)
    ms = statistics.mean(t)
    return {"metric": METRIC, "value": args.samples / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "nonzero_weights": nnz, "samples": args.samples, "horizon": args.horizon,
            "scene": "reach_static board (vp/data/reach_static.yaml) after 30 closed-loop replans"}


# ----------------------------------------------------------------------------- CPU port
def _median_s(fn, reps):
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return statistics.median(times)


def cpu_smpc_port(args_o, samples, horizon, reps: int, seed0: int = 0, nominal=None):
    """Reference smpc_step restated on the host (numpy sampler identical to
    vp/planner.py:199-219 + C fp64 rollout / softmin / update / M=1 tail)."""
    import oracle
    from oracle import scene as osc

    d = osc.DEFAULTS
    nom = np.zeros((horizon, 7)) if nominal is None else nominal
    times, last = [], None
    for r in range(reps):
        t0 = time.perf_counter()
        eps = oracle.sample_perturbations(samples, horizon, 7, d["sigma"], d["noise_window"], seed0 + r)
        last = oracle.smpc_step(args_o, nom, eps, d["lam"], osc.ACC_LIMIT)
        times.append(time.perf_counter() - t0)
    return times, last


def cpu_closed_loop(dims, samples, horizon, frames):
    """Host restatement of one closed-loop replan per frame (SURVEY.md 8d
    C1/C5): serial masked fusion (like the reference), EDT, smpc_step on all
    threads, integrate.  Returns the per-frame seconds."""
    import oracle
    from oracle import scene as osc

    voxel = 0.02
    extent = np.array(dims) * voxel
    origin = np.array([-extent[0] / 2.0, -extent[1] / 2.0, 0.0])
    cam = osc.Camera()
    r, t = cam.world_to_camera()
    lo = np.zeros(dims)
    ob = np.zeros(dims, bool)
    d = osc.DEFAULTS
    q, qd = np.full(7, 0.05), np.zeros(7)
    nominal = np.zeros((horizon, 7))
    times = []
    for f, (depth, (centers, radii)) in enumerate(osc.moving_obstacle_frames(dims, frames)):
        t0 = time.perf_counter()
        pm = oracle.masked_pixels(depth, cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max, cam.pose_r,
                                  cam.pose_t, centers, radii, 0.01)
        oracle.fuse_voxels(lo, ob, (0, 0, 0), dims, origin, voxel, r, t, cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                           cam.height, cam.d_min, cam.d_max, depth, pm, centers, radii, 2.5 * voxel, 0.85, -0.4,
                           -2.0, 3.5)
        sq = oracle.edt3d(lo)
        a = osc.rollout_args(sq, origin, voxel)
        a["q0"], a["qd0"] = q, qd
        eps = oracle.sample_perturbations(samples, horizon, 7, d["sigma"], d["noise_window"], f)
        res = oracle.smpc_step(a, nominal, eps, d["lam"], osc.ACC_LIMIT)
        times.append(time.perf_counter() - t0)
        qd = qd + res["command"] * d["dt"]
        q = q + qd * d["dt"]
        nominal = res["next_nominal"]
    return times


def cpu_baseline(args, S):
    """The reference path restated on this box's host cores (kind "port":
    the reference is Python + numba and cannot travel to the GPU box; its
    restatement is oracle/).  Medians of 3 repetitions per stage, at all
    threads and at 8 threads (the reference's acceptance setting,
    t/test_acceptance.py:50-54); fusion and sampling are serial in the
    reference regardless of threads."""
    import oracle
    from oracle import scene as osc

    oracle.build()
    oracle.set_threads(0)
    threads = oracle.get_threads()
    field_sq = S["field"].sq
    a3 = osc.rollout_args(field_sq, S["grid"].origin, S["grid"].voxel_size)
    times, _ = cpu_smpc_port(a3, args.samples, args.horizon, reps=3)
    t = statistics.median(times)
    oracle.set_threads(8)
    times8, _ = cpu_smpc_port(a3, args.samples, args.horizon, reps=3)
    oracle.set_threads(0)
    # C2 map stages
    lo = S["grid"].log_odds_host().copy()
    ob = S["grid"].observed_host().copy()
    cam, depth = S["cam"], S["depth"]
    pm = oracle.masked_pixels(depth.data, cam.fx, cam.fy, cam.cx, cam.cy, cam.d_min, cam.d_max,
                              cam.pose.rotation.matrix, cam.pose.translation, S["centers"], S["radii"], 0.01)
    r, tt = cam.world_to_camera()
    t_fus = _median_s(lambda: oracle.fuse_voxels(
        lo, ob, (0, 0, 0), S["grid"].dims, S["grid"].origin, S["grid"].voxel_size, r, tt, cam.fx, cam.fy, cam.cx,
        cam.cy, cam.width, cam.height, cam.d_min, cam.d_max, depth.data, pm, S["centers"], S["radii"],
        S["grid"].tau, 0.85, -0.4, -2.0, 3.5), 3)
    t_edt = _median_s(lambda: oracle.edt3d(lo), 3)
    oracle.set_threads(8)
    t_edt8 = _median_s(lambda: oracle.edt3d(lo), 3)
    oracle.set_threads(0)
    vox = args.grid ** 3
    out = {
        "value": args.samples / t, "unit": UNIT, "cores": threads, "kind": "port",
        "sample": f"median of 3 smpc_step reps at M={args.samples}, H={args.horizon} (numpy Philox sampler as the "
                  f"reference + C fp64 rollout on {threads} threads); medians of 3 reps of serial masked fusion "
                  f"and EDT at {args.grid}^3; C1 and C5 closed loops over 3 frames each",
        "smpc_step_ms": t * 1e3, "smpc_step_ms_8threads": statistics.median(times8) * 1e3,
        "fusion_ms": t_fus * 1e3, "edt_ms": t_edt * 1e3, "edt_ms_8threads": t_edt8 * 1e3,
        "edt_mvoxel_s": vox / t_edt / 1e6, "cpu": cpu_model(), "host_cpus": os.cpu_count(),
        "note": "the C port is faster than the numba reference on the same host (survey box: reference EDT "
                "538 ms at 256^3, 8 threads); the ratios against it are conservative",
    }
    if not args.no_configs:
        c1 = cpu_closed_loop((64, 64, 64), 256, 20, 3)
        c5 = cpu_closed_loop((512, 512, 512), 16384, 32, 3)
        out["c1_replan_p50_ms"] = statistics.median(c1) * 1e3
        out["c5_replan_p50_ms"] = statistics.median(c5) * 1e3
        out["closed_loop_frames"] = 3
    return out


def _import_reference():
    """The unmodified reference (voxplan, Python + numba) from baseline/_ref
    (pip --target install), or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "voxplan").is_dir():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import voxplan  # noqa: F401
        from voxplan import config as vconfig, mapping as vmapping, parallel as vparallel, planner as vplanner
        from voxplan import robot as vrobot
    except Exception as exc:  # pragma: no cover - depends on the box
        print(f"reference not importable ({exc}); timing the oracle port instead", file=sys.stderr)
        return None
    return vconfig, vmapping, vparallel, vplanner, vrobot


def run_reference_stock(args, mods) -> bool:
    """--impl reference through the reference's own public API and stock code
    path: voxplan.planner.Planner.smpc_step (numba, all host threads) on the C3
    workload, the field from voxplan.mapping.edt_3d of the C2 bench map (whose
    log-odds the host oracle fuses: bitwise the reference's fusion, pinned by
    tests/test_oracle_golden.py), the warm start fed back every step as the
    reference's own CLI bench and closed loop do (vp/cli.py:286-292,
    vp/sim.py:484-488)."""
    vconfig, vmapping, vparallel, vplanner, vrobot = mods
    from oracle import scene as osc

    m = args.samples * max(1, args.gpus)
    scene_map = osc.bench_map(args.grid)  # host fusion x2 of the C2 scene (input data, untimed)
    grid = vmapping.VoxelGrid(scene_map["origin"], scene_map["voxel"], (args.grid,) * 3)
    grid.log_odds[...] = scene_map["log_odds"]
    field = vmapping.edt_3d(grid, outside_default=0.8)
    chain, model = vrobot.load_robot(vconfig.bundled_scenario_path("robot_7dof"))
    params = vconfig.planner_params(chain.dof, {"samples": m, "horizon": args.horizon})
    planner = vplanner.Planner(chain, model, params)
    state = vrobot.JointState.resting(np.full(7, 0.05))
    goal = vrobot.forward_kinematics(chain, np.full(7, 0.35))[-1]
    threads = vparallel.set_threads(os.cpu_count() or 1)
    nominal = None
    for k in range(max(1, args.warmup)):  # the first call JIT-compiles the numba kernels
        nominal = planner.smpc_step(state, goal, field, nominal, k).next_nominal
    times = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        nominal = planner.smpc_step(state, goal, field, nominal, 1000 + k).next_nominal
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    value = m / t
    wl = "C3" if (args.samples, args.horizon) == (4096, 32) else "custom"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (CLI bench scene 256^3 + 7-DoF body mask fused on the host; the reference's own edt_3d "
                "and Planner.smpc_step)",
        "config": {"workload": f"{wl}: SMPC iteration M={args.samples}/rank x H={args.horizon}, 7-DoF robot_7dof, "
                               f"field = C2 {args.grid}^3 masked map",
                   "samples_per_rank": args.samples, "horizon": args.horizon, "grid": [args.grid] * 3,
                   "total_samples": m},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{args.steps} full smpc_step iterations of M={m} through the unmodified "
                                   f"reference (baseline/_ref, numba parallel on {threads} threads), warm start "
                                   f"fed back, after {max(1, args.warmup)} warm-up steps (JIT)",
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_modules_loaded": sorted(k for k in sys.modules if k.startswith("paper_2512_22575_b200")),
    }
    print(json.dumps(line), flush=True)
    return True


def run_reference(args):
    """--impl reference: the reference's path restated on the host cores
    (oracle/: C fp64 restatement + the reference's numpy sampler), on the
    same workload as our arm.  Imports nothing from the product package."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    mods = None if os.environ.get("VPB_REFERENCE_PORT") else _import_reference()
    if mods is not None and run_reference_stock(args, mods):
        return
    import oracle
    from oracle import scene as osc

    oracle.build()
    oracle.set_threads(0)
    threads = oracle.get_threads()
    m = args.samples * max(1, args.gpus)  # the whole job's rollouts per step (weak scaling, like our arm)
    scene_map = osc.bench_map(args.grid)  # host fusion x2 + EDT of the C2 scene
    a = osc.rollout_args(scene_map["sq"], scene_map["origin"], scene_map["voxel"])
    cpu_smpc_port(a, m, args.horizon, reps=max(1, min(args.warmup, 3)))
    times, _ = cpu_smpc_port(a, m, args.horizon, reps=args.steps, seed0=1000)
    t = statistics.mean(times)
    value = m / t
    wl = "C3" if (args.samples, args.horizon) == (4096, 32) else "custom"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (CLI bench scene 256^3 + 7-DoF body mask built on the host by the oracle; reference "
                "numpy Philox noise)",
        "config": {"workload": f"{wl}: SMPC iteration M={args.samples}/rank x H={args.horizon}, 7-DoF robot_7dof, "
                               f"field = C2 {args.grid}^3 masked map",
                   "samples_per_rank": args.samples, "horizon": args.horizon, "grid": [args.grid] * 3,
                   "total_samples": m},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full smpc_step iterations of M={m} (numpy sampler identical to "
                                   f"the reference + C fp64 rollout/softmin/update on {threads} threads)",
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        # evidence that this arm ran no product code
        "product_modules_loaded": sorted(k for k in sys.modules if k.startswith("paper_2512_22575_b200")),
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
