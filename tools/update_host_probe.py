"""Host cost of the pieces of mapping.update_occupancy (64^3 scene, 160x120 depth)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def t(fn, n=200):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return round((t1 - t0) / n * 1e6, 1)


def main():
    from paper_2512_22575_b200 import _device as D, config, mapping, robot, scene
    from paper_2512_22575_b200._lib import load

    dev = torch.device("cuda", 0)
    chain, model = config.robot_7dof()
    grid, cam, depth = scene.bench_edt_scene((64, 64, 64), device=dev)
    centers, radii = robot.sphere_positions(chain, np.full(7, 0.3), model)
    host = depth.data.copy()
    mapper = mapping.OccupancyMapper(grid, cam, outside_default=0.8)
    res = {}
    res["DepthImage+upload"] = t(lambda: mapping.DepthImage(host).device_tensor(dev))
    res["stream"] = t(lambda: D.stream(dev))
    res["mask_arrays"] = t(lambda: mapping._mask_arrays((centers, radii)))
    res["update(host depth)"] = t(lambda: mapper.update(mapping.DepthImage(host), mask=(centers, radii)))
    dd = mapping.DepthImage(host)
    dd.device_tensor(dev)
    res["update(device depth)"] = t(lambda: mapper.update(dd, mask=(centers, radii)))
    res["update(device, no mask)"] = t(lambda: mapper.update(dd))
    snap = mapper.snapshot()
    res["update(device) w/ live snapshot"] = t(lambda: mapper.update(dd, mask=(centers, radii)))
    del snap
    res["recompute_edt"] = t(lambda: mapper.recompute_edt())
    res["snapshot"] = t(lambda: mapper.snapshot())
    print(res)


if __name__ == "__main__" and "--detail" not in sys.argv:
    main()


def detail():
    from paper_2512_22575_b200 import _device as D, config, mapping, robot, scene
    from paper_2512_22575_b200._lib import load

    dev = torch.device("cuda", 0)
    grid, cam, depth = scene.bench_edt_scene((64, 64, 64), device=dev)
    mapper = mapping.OccupancyMapper(grid, cam, outside_default=0.8)
    mapper.update(depth)
    f = mapper.recompute_edt()
    box = grid.full_box()
    L = load()
    blo, n = box.native()
    ws = D.Workspace.get(dev, "edt", int(L.vpb_edt3d_workspace_bytes(n)))
    out = torch.empty(box.shape, dtype=torch.float32, device=dev)
    st = grid._struct()
    s = D.stream(dev)
    res = {}
    res["edt C call only"] = t(lambda: L.vpb_edt3d(st, blo, n, 1.0, 1, D.ptr(out), D.ptr(ws), ws.numel(), s))
    res["torch.empty field"] = t(lambda: torch.empty(box.shape, dtype=torch.float32, device=dev))
    res["DistanceField ctor"] = t(lambda: mapping.DistanceField(grid.origin, grid.voxel_size, grid.dims, box, out, 0.8))
    res["edt_3d total"] = t(lambda: mapping.edt_3d(grid, None, 0.8))
    j = mapping._Journal(grid)
    j._grow(100000)
    res["journal zero_"] = t(lambda: j.count.zero_())
    res["journal starts copy"] = t(lambda: j.starts[3:4].copy_(j.count))
    snap_cycle = []

    def cyc():
        sn = mapper.snapshot()
        mapper.update(depth)
        snap_cycle.append(sn)
        if len(snap_cycle) > 1:
            snap_cycle.pop(0)
    res["update w/ previous snapshot alive (closed loop)"] = t(cyc)
    print(res)


if __name__ == "__main__" and "--detail" in sys.argv:
    detail()
