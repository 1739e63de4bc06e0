import argparse, sys, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
args = argparse.Namespace(samples=4096, horizon=32, grid=256, precision="fp32")
S = bench.make_scene(args, torch.device("cuda", 0))
pl, st, goal, field = S["planner"], S["state"], S["goal"], S["field"]
nom = torch.zeros((32, 7), dtype=torch.float64, device="cuda")
for seed in (0, 1, 2):
    eps = pl.sample_device(seed)
    c, t, f, *_ = pl.evaluate_device(st, goal, field, eps, nom)
    c = c.cpu().numpy()
    w = np.exp(-(c - c.min()) / pl.params.lam)
    ctam = c.reshape(-1, 4).min(1)
    print(json.dumps({"min": float(c.min()), "p50": float(np.median(c)), "nonzero_w": int((w > 0).sum()),
                      "w_gt_1e-300": int((w > 1e-300).sum()), "nonzero_cta": int((np.exp(-(ctam - c.min()) / pl.params.lam) > 0).sum()),
                      "spread_p10_p90": [float(np.percentile(c, 10)), float(np.percentile(c, 90))]}))
