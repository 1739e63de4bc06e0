"""Host-side cost of one public-API SMPC step (native session), C3 scene."""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def best(fn, n=200):
    for _ in range(n):  # warm-up pass (CPU clocks, caches): the first timed series ran ~9 us slow
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e6


def main():
    import bench
    from paper_2512_22575_b200 import _device as D

    args = argparse.Namespace(samples=4096, horizon=32, grid=256, precision="fp32")
    S = bench.make_scene(args, torch.device("cuda", 0))
    pl, st, goal, field = S["planner"], S["state"], S["goal"], S["field"]
    nom = np.zeros((32, 7))
    sess = pl.session(field)
    sess.step(st, goal, nom, 0, field)
    L = sess._lib
    q0 = np.ascontiguousarray(st.q, dtype=np.float64)
    qd0 = np.ascontiguousarray(st.qd, dtype=np.float64)
    gr = np.ascontiguousarray(goal.rotation.matrix, dtype=np.float64).reshape(-1)
    gt = np.ascontiguousarray(goal.translation, dtype=np.float64)
    ptrs = [D.host_ptr(a) for a in (q0, qd0, gr, gt, nom)]
    sq = D.ptr(field.sq_device)
    out = sess.out
    optr = D.host_ptr(out)
    strm = D.stream(pl.device)
    res = {
        "public_step_us": best(lambda: pl.smpc_step(st, goal, field, nom, 3)),
        "session_step_us": best(lambda: sess.step(st, goal, nom, 3, field)),
        "raw_c_call_us": best(lambda: L.vpb_smpc_session_step(sess._h, *ptrs[:4], ptrs[4], 3, sq, optr, strm)),
        "unpack_us": best(lambda: pl.unpack_step(out, st, goal, 32)),
    }
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
