"""A/B timing of library builds on the C3 step (fused SMPC kernel and the
native-session step, L2 flushed before every timed launch).

    python tools/ab_time.py ab/libA.so ab/libB.so [--rounds 4]
    python tools/ab_time.py lib.so lib.so@VPB_NO_DRY_MERGE=1   (same build, env A/B)

Each round runs every build in its own process (VPB_LIB_PATH), interleaved
A B A B ... so clock and thermal drift hit all builds alike; prints the
median over rounds of each build's per-run median."""
import argparse
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def worker(iters: int, grid: int, samples: int) -> None:
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch

    import bench
    from paper_2512_22575_b200 import _lib

    args = argparse.Namespace(samples=samples, horizon=32, grid=grid, precision="fp32")
    dev = torch.device("cuda", 0)
    S = bench.make_scene(args, dev)
    pl, st, goal, field = S["planner"], S["state"], S["goal"], S["field"]
    nom = torch.zeros((32, 7), dtype=torch.float64, device=dev)
    lib = _lib.load()
    eps = torch.empty((samples, 32, 7), dtype=torch.float32, device=dev)
    out = torch.empty(int(lib.vpb_smpc_out_len(32, 7)), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sess = pl.session(field, samples)
    sess.step(st, goal, np.zeros((32, 7)), 0, field)
    stream = torch.cuda.current_stream(dev)

    def run(fn):
        for k in range(5):
            fn(k)
        ts = []
        for k in range(iters):
            flush.fill_(k & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(k)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        cut = len(ts) // 10  # 10 % trimmed mean (event timestamps are ~1 us quantized)
        return statistics.mean(ts[cut:len(ts) - cut])

    res = {
        "fused_us": run(lambda k: pl.smpc_generate_device(st, goal, field, nom, k, eps_out=eps, out=out)),
        "session_us": run(lambda k: sess.launch()),
        "rollout_us": run(lambda k: pl.evaluate_device(st, goal, field, eps, nom)),
    }
    print(json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="*")
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--worker", action="store_true")
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--samples", type=int, default=4096)
    a = ap.parse_args()
    if a.worker:
        worker(a.iters, a.grid, a.samples)
        return
    per = {lib: [] for lib in a.libs}
    for _ in range(a.rounds):
        for lib in a.libs:
            path, _, extra = lib.partition("@")
            env = dict(os.environ, VPB_LIB_PATH=str(Path(path).resolve()))
            if extra:
                k, _, v = extra.partition("=")
                env[k] = v
            r = subprocess.run([sys.executable, __file__, "--worker", "--iters", str(a.iters), "--grid", str(a.grid),
                                "--samples", str(a.samples)], env=env,
                               capture_output=True, text=True, check=True)
            per[lib].append(json.loads(r.stdout.strip().splitlines()[-1]))
    summary = {lib: {k: round(statistics.median(x[k] for x in v), 2) for k in v[0]} for lib, v in per.items()}
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
