"""A few cycles of every path at small sizes, for compute-sanitizer (memcheck / racecheck / synccheck).
Usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I, shard  # noqa: E402

cfg = I.config("cfg2", width=128, height=96, nu=40_000, nu_b=4_000, beams=300, movers=3, peds=2, boxes=6)
sc = I.scene(cfg)
f = dog.Filter.from_config(cfg, debug=False)
for k in range(3):
    f.step(sc.frame(k, device="cuda").contiguous(), cfg.dt)
for k in range(3, 5):
    m = sc.frame(k, device="cuda").contiguous()
    dop, pA = sc.doppler(k, m, frac=0.7)
    f.step_doppler(m, dop.cuda().contiguous(), pA.cuda().contiguous(), cfg.dt)
f.ego_scroll(0.35, -0.21)
for k in range(5, 7):
    f.step_exact(I.Scene.exact_obs(sc.frame(k, device="cuda")), cfg.dt)
r = f.evaluate(labels=torch.ones(cfg.C, dtype=torch.uint8, device="cuda"), thresholds=[0.5, 2.0])
lb = shard.LocalBands.from_config(cfg, 2)
for k in range(3):
    lb.step(sc.frame(k, device="cuda").contiguous(), cfg.dt)
lb.rebalance(min_rows=8, rows=[(0, 30), (30, 96)])
lb.step(sc.frame(3, device="cuda").contiguous(), cfg.dt)
torch.cuda.synchronize()
print("sanitize run ok")
