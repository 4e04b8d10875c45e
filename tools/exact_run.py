"""cfg T: settle with plain cycles, then n exact PHD/MIB cycles (NEXT-3) -- for ncu launch lists of the
exact path, including its later cycles (births spread the particles over the whole grid, so runs per
sort tile grow).  Usage: python tools/exact_run.py [n_exact_cycles] [settle]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I  # noqa: E402

cfg = I.CONFIGS["cfgT"]
sc = I.scene(cfg)
f = dog.Filter.from_config(cfg)
settle = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for k in range(settle):
    f.step(sc.frame(k, device="cuda").contiguous(), cfg.dt)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ms = []
for k in range(settle, settle + n):
    obs = I.Scene.exact_obs(sc.frame(k, device="cuda").contiguous())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    last = k == settle + n - 1
    if last:
        torch.cuda.nvtx.range_push("capture")   # ncu --nvtx --nvtx-include "capture/": the last cycle only
    f.step_exact(obs, cfg.dt)
    if last:
        torch.cuda.nvtx.range_pop()
    e1.record()
    torch.cuda.synchronize()
    ms.append(round(e0.elapsed_time(e1), 3))
print("exact cycle ms:", ms)
