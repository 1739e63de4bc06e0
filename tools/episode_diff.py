"""Stock reference run_episode vs the same with the seams rebound to libvpb200
(integration/voxplan_shim.py): per-cycle deviation of the closed loop.
Needs the reference in baseline/_ref.  Usage: python tools/episode_diff.py [cycles] [scenario]"""
import dataclasses
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
sys.path.insert(0, str(ROOT / "integration"))
sys.path.insert(0, str(ROOT))

import voxplan  # noqa: E402
import voxplan.sim  # noqa: E402
from voxplan import parallel  # noqa: E402
from voxplan.config import bundled_scenario_path, load_scenario  # noqa: E402
from voxplan.sim import run_episode  # noqa: E402

import voxplan_shim  # noqa: E402


def main():
    cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    name = sys.argv[2] if len(sys.argv) > 2 else "reach_static"
    parallel.set_threads(8)
    scn = dataclasses.replace(load_scenario(bundled_scenario_path(name)), timeout_cycles=cycles)
    a = run_episode(scn)
    voxplan_shim.install(voxplan)
    b = run_episode(scn)
    rows = []
    for ra, rb in zip(a.records, b.records):
        rows.append({"cycle": ra.cycle,
                     "q": float(np.max(np.abs(ra.q - rb.q))),
                     "command": float(np.max(np.abs(ra.command - rb.command))),
                     "weighted_cost_rel": abs(ra.weighted_cost - rb.weighted_cost) / abs(ra.weighted_cost),
                     "best_cost_rel": abs(ra.best_cost - rb.best_cost) / abs(ra.best_cost),
                     "clearance": abs(ra.clearance - rb.clearance)})
    print(json.dumps({"scenario": name, "cycles": len(rows), "success": [a.success, b.success],
                      "goal_cycles": [a.goal_cycles, b.goal_cycles], "per_cycle": rows}))


if __name__ == "__main__":
    main()
